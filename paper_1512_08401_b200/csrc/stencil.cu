// Circulant-compressed Theta_K as a stencil SpMV: y = Theta x and Theta^T x
// straight from the kept generator groups of the reference's top-K walk (678 records at
// 1024^2, K = 3N) - no CSR: the only streams are x and y.
//
// A record (block = (out band, in band), generator index v, count c, value) stands for the
// first c positions, row-major, of the smaller band (theta.cpp:236-275):
//   in band finer or equal (s = in/out per dim): row n of the out band (flat(n) < c) has
//     column m = (v + s n) mod in.shape;
//   in band coarser (s = out/in):                column m (flat(m) < c) feeds row
//     n = (v + s m) mod out.shape, i.e. row n is hit iff (n - v) mod out.shape is a
//     multiple of s, by m = ((n - v) mod out.shape) / s.
// One thread per output coordinate scans the records of its band (sorted by band on the
// host) and accumulates in record order. Band shapes are powers of two (the reference's
// dyadic images), so every div/mod is a shift/mask. The row sums are in record order, not
// in the CSR's ascending-column order: equal to wbx_spmv within rounding (fp64 ~1e-16).
#include <algorithm>
#include <vector>

#include "internal.hpp"

extern "C" void wbx_set_last_error(const char* msg);

struct wbx_stencil {
    wbx_ctx* ctx = nullptr;
    uint64_t n = 0;
    uint32_t nb = 0, d = 2;
    wbx::DevBuf<uint4> rec_fwd, rec_adj;  // {other band, v0 | v1 << 16, count (low 32), value index}
    wbx::DevBuf<uint32_t> off_fwd, off_adj;  // per band: record range
    wbx::DevBuf<double> val64;
    wbx::DevBuf<float> val32;
    wbx::DevBuf<uint4> band;  // {offset, log2 shape0, log2 shape1, level}
};

namespace wbx {
namespace {

__device__ __forceinline__ uint32_t find_band(const uint4* band, uint32_t nb, uint64_t i) {
    uint32_t b = 0;  // bands are ordered by offset: last band with offset <= i
    for (uint32_t k = 1; k < nb; ++k)
        if (band[k].x <= i) b = k;
    return b;
}

template <typename T, bool ADJ>
__global__ void stencil_kernel(uint64_t n, uint32_t nb, const uint4* __restrict__ band, const uint4* __restrict__ rec,
                               const uint32_t* __restrict__ off, const T* __restrict__ val, const T* __restrict__ x,
                               T* __restrict__ y) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t b = find_band(band, nb, i);
    const uint4 me = band[b];
    const uint32_t p = static_cast<uint32_t>(i - me.x);  // position in my band
    const uint32_t l1 = me.z;
    const uint32_t p0 = p >> l1, p1 = p & ((1u << l1) - 1u);
    T acc = T(0);
    for (uint32_t r = off[b]; r < off[b + 1]; ++r) {
        const uint4 R = rec[r];
        const uint4 ob = band[R.x];  // the other band of the block
        const uint32_t v0 = R.y & 0xffffu, v1 = R.y >> 16;
        // forward: me = out band, ob = in band; adjoint: me = in band, ob = out band
        const uint4 bo = ADJ ? ob : me, bi = ADJ ? me : ob;
        const bool in_finer = bi.w <= bo.w;  // level
        uint32_t q0, q1;  // the other coordinate (column for forward, row for adjoint)
        uint32_t small_flat;
        bool hit = true;
        if (in_finer) {  // positions walk the out band: n (rows); m = (v + s n) mod in
            const uint32_t s0 = bi.y - bo.y, s1 = bi.z - bo.z;  // log2 scale
            if (!ADJ) {  // n = p
                small_flat = p;
                q0 = (v0 + (p0 << s0)) & ((1u << bi.y) - 1u);
                q1 = (v1 + (p1 << s1)) & ((1u << bi.z) - 1u);
            } else {  // m = p: n = ((m - v) mod in) / s when divisible
                const uint32_t t0 = (p0 - v0) & ((1u << bi.y) - 1u), t1 = (p1 - v1) & ((1u << bi.z) - 1u);
                hit = !(t0 & ((1u << s0) - 1u)) && !(t1 & ((1u << s1) - 1u));
                q0 = t0 >> s0;
                q1 = t1 >> s1;
                small_flat = (q0 << bo.z) + q1;
            }
        } else {  // positions walk the in band: m; n = (v + s m) mod out
            const uint32_t s0 = bo.y - bi.y, s1 = bo.z - bi.z;
            if (!ADJ) {  // n = p: m = ((n - v) mod out) / s when divisible
                const uint32_t t0 = (p0 - v0) & ((1u << bo.y) - 1u), t1 = (p1 - v1) & ((1u << bo.z) - 1u);
                hit = !(t0 & ((1u << s0) - 1u)) && !(t1 & ((1u << s1) - 1u));
                q0 = t0 >> s0;
                q1 = t1 >> s1;
                small_flat = (q0 << bi.z) + q1;
            } else {  // m = p
                small_flat = p;
                q0 = (v0 + (p0 << s0)) & ((1u << bo.y) - 1u);
                q1 = (v1 + (p1 << s1)) & ((1u << bo.z) - 1u);
            }
        }
        if (hit && small_flat < R.z) {
            const uint64_t j = static_cast<uint64_t>(ob.x) + (static_cast<uint64_t>(q0) << ob.z) + q1;
            acc = fma(val[R.w], x[j], acc);
        }
    }
    y[i] = acc;
}

}  // namespace
}  // namespace wbx

extern "C" {

int wbx_stencil_create(wbx_ctx* ctx, uint32_t ndim, const uint64_t* dims, uint32_t J, uint64_t n_gens,
                       const uint32_t* blocks, const uint32_t* gen_index, const uint64_t* counts, const double* values,
                       wbx_stencil** out) {
    wbx_stencil* s = nullptr;
    try {
        if (!ctx || !dims || !out || (n_gens && (!blocks || !gen_index || !counts || !values)))
            wbx::fail(WBX_INVALID_ARGUMENT, "null argument to wbx_stencil_create");
        if (ndim != 1 && ndim != 2) wbx::fail(WBX_BAD_SPEC, "stencil: 1-D or 2-D layouts");
        std::vector<wbx_band> bands;
        wbx::make_layout(ndim, dims, J, bands);
        s = new wbx_stencil;
        s->ctx = ctx;
        s->d = ndim;
        s->nb = static_cast<uint32_t>(bands.size());
        s->n = dims[0] * (ndim == 2 ? dims[1] : 1);
        if (s->n > 0xffffffffull) wbx::fail(WBX_TOO_LARGE, "stencil: more than 2^32 coordinates");
        auto lg = [](uint64_t v) {
            if (!v || (v & (v - 1))) wbx::fail(WBX_BAD_SPEC, "stencil: band shapes must be powers of two");
            uint32_t l = 0;
            while ((1ull << l) < v) ++l;
            return l;
        };
        std::vector<uint4> hb(s->nb);
        for (uint32_t b = 0; b < s->nb; ++b) {
            // 1-D layouts: shape = {count, 1} -> treated as a count x 1 "image" (column index 0)
            hb[b] = make_uint4(static_cast<uint32_t>(bands[b].offset), lg(bands[b].shape[0]),
                               ndim == 2 ? lg(bands[b].shape[1]) : 0u, bands[b].level);
        }
        struct R {
            uint32_t band, other, vpack, count, vi;
        };
        std::vector<R> fw, ad;
        std::vector<double> v64(std::max<uint64_t>(n_gens, 1));
        for (uint64_t g = 0; g < n_gens; ++g) {
            const uint32_t out_b = blocks[g] / s->nb, in_b = blocks[g] % s->nb;
            if (out_b >= s->nb) wbx::fail(WBX_BAD_SPEC, "stencil: block index out of range");
            const wbx_band& bi = bands[in_b];
            const wbx_band& bo = bands[out_b];
            const uint64_t* gs = bi.level <= bo.level ? bi.shape : bo.shape;
            const uint64_t g1 = ndim == 2 ? gs[1] : 1;
            const uint64_t v0 = gen_index[g] / g1, v1 = gen_index[g] % g1;
            if (v0 > 0xffff || v1 > 0xffff || counts[g] > 0xffffffffull)
                wbx::fail(WBX_TOO_LARGE, "stencil: generator index or count too large");
            const uint32_t vp = static_cast<uint32_t>(v0 | (v1 << 16));
            fw.push_back({out_b, in_b, vp, static_cast<uint32_t>(counts[g]), static_cast<uint32_t>(g)});
            ad.push_back({in_b, out_b, vp, static_cast<uint32_t>(counts[g]), static_cast<uint32_t>(g)});
            v64[g] = values[g];
        }
        auto pack = [&](std::vector<R>& v, wbx::DevBuf<uint4>& rec, wbx::DevBuf<uint32_t>& off) {
            std::stable_sort(v.begin(), v.end(), [](const R& a, const R& b) { return a.band < b.band; });
            std::vector<uint32_t> o(s->nb + 1, 0);
            std::vector<uint4> h(std::max<size_t>(v.size(), 1));
            for (size_t k = 0; k < v.size(); ++k) {
                ++o[v[k].band + 1];
                h[k] = make_uint4(v[k].other, v[k].vpack, v[k].count, v[k].vi);
            }
            for (uint32_t b = 0; b < s->nb; ++b) o[b + 1] += o[b];
            rec.upload(h, ctx->stream);
            off.upload(o, ctx->stream);
        };
        pack(fw, s->rec_fwd, s->off_fwd);
        pack(ad, s->rec_adj, s->off_adj);
        std::vector<float> v32(v64.begin(), v64.end());
        s->val64.upload(v64, ctx->stream);
        s->val32.upload(v32, ctx->stream);
        s->band.upload(hb, ctx->stream);
        WBX_CUDA(cudaStreamSynchronize(ctx->stream));
        *out = s;
        return WBX_OK;
    } catch (const wbx::Error& e) {
        delete s;
        wbx_set_last_error(e.what());
        return e.status;
    }
}

int wbx_stencil_destroy(wbx_stencil* s) {
    delete s;
    return WBX_OK;
}

// y = Theta x (transpose = 0) or Theta^T x on device buffers; precision WBX_FP64 or WBX_FP32
int wbx_stencil_spmv_dev(wbx_stencil* s, int transpose, int precision, const void* x_dev, void* y_dev) {
    try {
        if (!s || !x_dev || !y_dev) wbx::fail(WBX_INVALID_ARGUMENT, "null argument to wbx_stencil_spmv_dev");
        const unsigned grid = static_cast<unsigned>((s->n + 255) / 256);
        cudaStream_t st = s->ctx->stream;
        const uint4* rec = transpose ? s->rec_adj.p : s->rec_fwd.p;
        const uint32_t* off = transpose ? s->off_adj.p : s->off_fwd.p;
        if (precision == WBX_FP64) {
            auto k = transpose ? wbx::stencil_kernel<double, true> : wbx::stencil_kernel<double, false>;
            k<<<grid, 256, 0, st>>>(s->n, s->nb, s->band.p, rec, off, s->val64.p, static_cast<const double*>(x_dev),
                                     static_cast<double*>(y_dev));
        } else {
            auto k = transpose ? wbx::stencil_kernel<float, true> : wbx::stencil_kernel<float, false>;
            k<<<grid, 256, 0, st>>>(s->n, s->nb, s->band.p, rec, off, s->val32.p, static_cast<const float*>(x_dev),
                                     static_cast<float*>(y_dev));
        }
        wbx::count_launch(s->ctx);
        WBX_CUDA(cudaGetLastError());
        return WBX_OK;
    } catch (const wbx::Error& e) {
        wbx_set_last_error(e.what());
        return e.status;
    }
}

}  // extern "C"
