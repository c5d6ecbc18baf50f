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
