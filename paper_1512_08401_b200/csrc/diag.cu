// Diagnostics: cost of the grid barrier used by the persistent solver (wbx_diag.h).
#include "device_util.cuh"
#include "internal.hpp"
#include "wbx_diag.h"

namespace {
__global__ void __launch_bounds__(256) barrier_kernel(unsigned* bar, int iters) {
    for (int i = 0; i < iters; ++i) wbx::grid_sync(bar, gridDim.x);
}
}  // namespace

extern "C" void wbx_set_last_error(const char* msg);

extern "C" int wbx_diag_barrier_us(int device, int iters, int blocks_per_sm, double* us) {
    try {
        WBX_CUDA(cudaSetDevice(device));
        int sms = 0;
        WBX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        wbx::DevBuf<unsigned> bar(2);
        WBX_CUDA(cudaMemset(bar.p, 0, 8));
        dim3 grid(sms * blocks_per_sm);
        void* args[] = {&bar.p, &iters};
        cudaEvent_t a, b;
        WBX_CUDA(cudaEventCreate(&a));
        WBX_CUDA(cudaEventCreate(&b));
        WBX_CUDA(cudaLaunchCooperativeKernel((void*)barrier_kernel, grid, dim3(256), args, 0, 0));
        WBX_CUDA(cudaEventRecord(a));
        WBX_CUDA(cudaLaunchCooperativeKernel((void*)barrier_kernel, grid, dim3(256), args, 0, 0));
        WBX_CUDA(cudaEventRecord(b));
        WBX_CUDA(cudaEventSynchronize(b));
        float ms = 0;
        WBX_CUDA(cudaEventElapsedTime(&ms, a, b));
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        *us = ms * 1e3 / iters;
        return WBX_OK;
    } catch (const wbx::Error& e) {
        wbx_set_last_error(e.what());
        return e.status;
    }
}

#include "stream.cuh"

namespace {
// mode 0: each warp streams its chunks (strided over the buffer) through a smem ring by
// bulk copies; mode 1: lanes stream with 16-B loads.
__global__ void __launch_bounds__(256) stream_kernel(const uint4* buf, uint64_t n16, int reps, int mode,
                                                     int chunk16, int inflight, unsigned long long* sink) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t gwarp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * blockDim.x / 32;
    unsigned long long acc = 0;
    const uint64_t pol = wbx::l2_keep_policy();
    if (mode == 0) {
        uint64_t* bars = reinterpret_cast<uint64_t*>(sm + wib * (128 + inflight * chunk16 * 16));
        uint4* slots = reinterpret_cast<uint4*>(sm + wib * (128 + inflight * chunk16 * 16) + 128);
        if (lane == 0)
            for (int i = 0; i < inflight; ++i) wbx::mbar_init(bars + i, 1);
        wbx::mbar_fence_init();
        __syncwarp();
        const uint64_t nchunks = n16 / chunk16;
        const uint64_t mine = nchunks > gwarp ? (nchunks - gwarp + nw - 1) / nw : 0;
        const uint64_t total = mine * reps;
        uint64_t issued = 0;
        auto issue = [&]() {
            const uint64_t c = gwarp + (issued % mine) * nw;
            if (lane == 0) {
                const int s = static_cast<int>(issued % inflight);
                wbx::mbar_expect_tx(bars + s, chunk16 * 16);
                wbx::bulk_g2s(slots + s * chunk16, buf + c * chunk16, chunk16 * 16, bars + s, pol);
            }
            ++issued;
        };
        while (issued < total && issued < static_cast<uint64_t>(inflight)) issue();
        for (uint64_t e = 0; e < total; ++e) {
            const int s = static_cast<int>(e % inflight);
            wbx::mbar_wait(bars + s, static_cast<unsigned>((e / inflight) & 1));
            acc += slots[s * chunk16 + lane].x;
            __syncwarp();
            if (issued < total) issue();
        }
    } else {
        const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
        const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
        for (int r = 0; r < reps; ++r)
            for (uint64_t i = t0; i < n16; i += 8 * nthreads) {
                uint4 v[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) v[j] = i + j * nthreads < n16 ? wbx::ld_stream(buf + i + j * nthreads, pol) : make_uint4(0, 0, 0, 0);
#pragma unroll
                for (int j = 0; j < 8; ++j) acc += v[j].x;
            }
    }
    if (acc == 0x1234567ull) sink[0] = acc;
}
}  // namespace

extern "C" int wbx_diag_stream_gbs(int device, int mode, uint64_t bytes, int reps, int chunk, int inflight,
                                   int blocks_per_sm, double* gbs) {
    try {
        WBX_CUDA(cudaSetDevice(device));
        int sms = 0;
        WBX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        const uint64_t n16 = bytes / 16;
        wbx::DevBuf<uint4> buf(n16);
        wbx::DevBuf<unsigned long long> sink(1);
        WBX_CUDA(cudaMemset(buf.p, 1, n16 * 16));
        const int chunk16 = chunk / 16;
        const unsigned smem = mode == 0 ? 8u * (128u + inflight * chunk) : 0u;
        if (smem)
            WBX_CUDA(cudaFuncSetAttribute((const void*)stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        const dim3 grid(sms * blocks_per_sm);
        cudaEvent_t a, b;
        WBX_CUDA(cudaEventCreate(&a));
        WBX_CUDA(cudaEventCreate(&b));
        stream_kernel<<<grid, 256, smem>>>(buf.p, n16, 1, mode, chunk16, inflight, sink.p);  // warm (L2 fill)
        WBX_CUDA(cudaEventRecord(a));
        stream_kernel<<<grid, 256, smem>>>(buf.p, n16, reps, mode, chunk16, inflight, sink.p);
        WBX_CUDA(cudaEventRecord(b));
        WBX_CUDA(cudaEventSynchronize(b));
        WBX_CUDA(cudaGetLastError());
        float ms = 0;
        WBX_CUDA(cudaEventElapsedTime(&ms, a, b));
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        *gbs = static_cast<double>(n16 * 16) * reps / (ms * 1e-3) / 1e9;
        return WBX_OK;
    } catch (const wbx::Error& e) {
        wbx_set_last_error(e.what());
        return e.status;
    }
}
