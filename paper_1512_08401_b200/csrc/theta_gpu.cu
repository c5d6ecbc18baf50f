// Theta_K construction on the device: build_theta_conv (theta.cpp:40-79) + the global
// weighted top-K walk of threshold_impl (theta.cpp:206-276), producing the kept generator
// groups (block, generator index, positions kept, value) that wbx_theta_expand turns into
// the CSR (assemble, theta.cpp:180-201).
//
// Arithmetic is the oracle build's, operation by operation, so the generators, the keys and
// hence the index set are BITWISE those of the reference built against the oracle's FFT
// ("pinned to the oracle build, not to FFTW"):
//  * convolve_spectral (operators.cpp:20-77): r2c of the image and of the kernel, half-
//    spectrum product (std::complex multiply: re = ac - bd, im = ad + bc, no contraction),
//    c2r that rebuilds the full spectrum by Hermitian symmetry, scale by 1/size;
//  * the FFT is the oracle shim's radix-2 (oracle/shim/fftw_shim.cpp): complex transform of
//    rows then columns, bit reversal, butterflies u + v, u - v with v = b * w[k * n/len]
//    (conjugated twiddle for the inverse), twiddles cos/sin(-2 pi k / n) from the host libm;
//  * single_wavelet and analyze are the library's bitwise DWT kernels.
// Selection: keys |g| * w_in (> 0) of all ~22 M generator entries (1024^2) are reduced to the
// boundary key by a weighted radix select (each entry stands for `multiplicity` positions);
// only the entries at or above it (a few hundred) go to the host, where they are sorted with
// the reference comparator and walked to K positions.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "fft.cuh"
#include "internal.hpp"

extern "C" void wbx_set_last_error(const char* msg);

namespace wbx {
namespace {

__global__ void unit_kernel(double* x, uint64_t n, uint64_t pos) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) x[i] = i == pos ? 1.0 : 0.0;
}

// ---------------------------------------------------------------- candidates / selection
struct BlockDesc {
    const double* gen;  // generator values (slice of fwd[in] or adj[out])
    uint64_t size;      // generator entries
    uint64_t base;      // first global candidate index
    uint64_t mult;      // positions per entry (the smaller band's count)
    double w;           // column-band weight
};

__device__ __forceinline__ uint32_t block_of(const BlockDesc* bd, uint32_t nblk, uint64_t g) {
    uint32_t lo = 0, hi = nblk;  // last block with base <= g
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) / 2;
        if (bd[mid].base <= g) lo = mid;
        else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ uint64_t key_bits(const BlockDesc& b, uint64_t v) {
    const double key = __dmul_rn(fabs(b.gen[v]), b.w);  // std::abs(g) * w
    return key > 0.0 ? static_cast<uint64_t>(__double_as_longlong(key)) : 0ull;  // 0 = not a candidate
}

// weighted histogram of digit `shift` over the candidates whose higher digits equal `prefix`
__global__ void radix_hist_kernel(const BlockDesc* bd, uint32_t nblk, uint64_t total, uint64_t prefix,
                                  uint64_t mask, int shift, unsigned long long* hist) {
    __shared__ unsigned long long h[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    for (uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < total;
         g += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t b = block_of(bd, nblk, g);
        const uint64_t k = key_bits(bd[b], g - bd[b].base);
        if (k != 0 && (k & mask) == prefix) atomicAdd(&h[(k >> shift) & 0xff], bd[b].mult);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
        if (h[i]) atomicAdd(&hist[i], h[i]);
}

struct Sel {
    uint64_t key;
    uint32_t block;
    uint32_t gen_index;
};

__global__ void collect_kernel(const BlockDesc* bd, uint32_t nblk, uint64_t total, uint64_t kmin, Sel* out,
                               unsigned long long cap, unsigned long long* count) {
    for (uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < total;
         g += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t b = block_of(bd, nblk, g);
        const uint64_t k = key_bits(bd[b], g - bd[b].base);
        if (k != 0 && k >= kmin) {
            const unsigned long long slot = atomicAdd(count, 1ull);
            if (slot < cap) out[slot] = Sel{k, b, static_cast<uint32_t>(g - bd[b].base)};
        }
    }
}

unsigned blocks_of(uint64_t n, unsigned t = 256) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace

}  // namespace wbx

extern "C" {

// gaussian_kernel (operators.cpp:100-120) + normalize_sum: host, the reference's expressions
int wbx_psf_gaussian(uint32_t ndim, const uint64_t* dims, double sigma, double* k) {
    try {
        if ((ndim != 1 && ndim != 2) || !dims || !k) wbx::fail(WBX_INVALID_ARGUMENT, "wbx_psf_gaussian: bad arguments");
        if (!(sigma > 0.0)) wbx::fail(WBX_BAD_SPEC, "Gaussian sigma must be positive");
        const uint64_t n0 = dims[0], n1 = ndim == 2 ? dims[1] : 1;
        auto wrapped = [](uint64_t i, uint64_t n) {
            return i < n / 2 ? static_cast<double>(i) : static_cast<double>(i) - static_cast<double>(n);
        };
        if (sigma < 1.0) {  // sub-pixel width degenerates to a delta (no normalisation pass)
            std::fill(k, k + n0 * n1, 0.0);
            k[0] = 1.0;
            return WBX_OK;
        }
        if (ndim == 1) {
            for (uint64_t i = 0; i < n0; ++i) {
                const double t = wrapped(i, n0);
                k[i] = std::exp(-t * t / (2.0 * sigma * sigma));
            }
        } else {
            for (uint64_t r = 0; r < n0; ++r)
                for (uint64_t c = 0; c < n1; ++c) {
                    const double t1 = wrapped(r, n0), t2 = wrapped(c, n1);
                    k[r * n1 + c] = std::exp(-(t1 * t1 + t2 * t2) / (2.0 * sigma * sigma));
                }
        }
        double s = 0.0;
        for (uint64_t i = 0; i < n0 * n1; ++i) s += k[i];
        if (s <= 0.0) wbx::fail(WBX_BAD_SPEC, "PSF has nonpositive mass");
        for (uint64_t i = 0; i < n0 * n1; ++i) k[i] /= s;
        return WBX_OK;
    } catch (const wbx::Error& e) {
        wbx_set_last_error(e.what());
        return e.status;
    }
}

int wbx_theta_conv_topk(wbx_ctx* ctx, wbx_basis* basis, const double* psf, const double* band_weight, uint64_t K,
                        uint64_t max_records, uint32_t* gen_block, uint32_t* gen_index, uint64_t* gen_count,
                        double* gen_value, uint64_t* n_records) {
    using namespace wbx;
    try {
        if (!ctx || !basis || !psf || !band_weight || !gen_block || !gen_index || !gen_count || !gen_value ||
            !n_records)
            fail(WBX_INVALID_ARGUMENT, "null argument to wbx_theta_conv_topk");
        cudaStream_t st = ctx->stream;
        const auto& bands = basis->bands;
        const uint32_t nb = static_cast<uint32_t>(bands.size()), d = basis->ndim;
        const uint64_t n = basis->n;
        const uint64_t n0 = d == 2 ? basis->dims[0] : 1, n1 = d == 2 ? basis->dims[1] : basis->dims[0];
        for (uint32_t b = 0; b < nb; ++b)
            if (!(band_weight[b] > 0.0)) fail(WBX_BAD_SPEC, "threshold_weighted: sigma must be positive");
        Fft2 fft(n0, n1, st);
        const uint64_t hs = n0 * fft.h;
        DevBuf<double> img(n), u(n);
        DevBuf<double2> sk(hs), su(hs);
        img.upload(psf, n, st);
        fft.r2c(img.p, sk.p);  // kernel spectrum
        // fwd[i] = analyze(convolve(w_i, psf)), adj[i] = analyze(apply_adjoint(w_i, psf))
        DevBuf<double> fwd(static_cast<uint64_t>(nb) * n), adj(static_cast<uint64_t>(nb) * n);
        for (uint32_t i = 0; i < nb; ++i) {
            unit_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(img.p, n, bands[i].offset);
            synthesize_dev(basis, img.p, u.p, st);  // single_wavelet(level, orientation)
            fft.r2c(u.p, su.p);
            fft.conv_c2r(su.p, sk.p, 0, img.p);
            analyze_dev(basis, img.p, fwd.p + static_cast<uint64_t>(i) * n, st);
            fft.conv_c2r(su.p, sk.p, 1, img.p);
            analyze_dev(basis, img.p, adj.p + static_cast<uint64_t>(i) * n, st);
        }
        // blocks b = out * nb + in (CirculantTheta::blocks order)
        auto count_of = [&](const wbx_band& b) { return b.shape[0] * (d == 2 ? b.shape[1] : 1); };
        std::vector<BlockDesc> bd(static_cast<size_t>(nb) * nb);
        uint64_t total = 0;
        for (uint32_t out = 0; out < nb; ++out)
            for (uint32_t in = 0; in < nb; ++in) {
                const wbx_band& bi = bands[in];
                const wbx_band& bo = bands[out];
                BlockDesc& x = bd[out * nb + in];
                if (bi.level <= bo.level) {  // input grid finer or equal: slice of adj[out] on the input band
                    x.gen = adj.p + static_cast<uint64_t>(out) * n + bi.offset;
                    x.size = count_of(bi);
                    x.mult = count_of(bo);
                } else {  // output grid finer: slice of fwd[in] on the output band
                    x.gen = fwd.p + static_cast<uint64_t>(in) * n + bo.offset;
                    x.size = count_of(bo);
                    x.mult = count_of(bi);
                }
                x.w = band_weight[in];
                x.base = total;
                total += x.size;
            }
        DevBuf<BlockDesc> dbd(bd.size());
        dbd.upload(bd, st);
        // weighted radix select of the boundary key: the largest key kb with
        // sum_{key >= kb} mult >= K (all candidates when their total is below K)
        DevBuf<unsigned long long> hist(256);
        const unsigned grid = 4u * static_cast<unsigned>(ctx->num_sms);
        uint64_t prefix = 0, mask = 0, above = 0;  // above: positions of keys > current prefix range
        bool all = false;
        for (int shift = 56; shift >= 0; shift -= 8) {
            WBX_CUDA(cudaMemsetAsync(hist.p, 0, 256 * sizeof(unsigned long long), st));
            radix_hist_kernel<<<grid, 256, 0, st>>>(dbd.p, nb * nb, total, prefix, mask, shift, hist.p);
            unsigned long long h[256];
            WBX_CUDA(cudaMemcpyAsync(h, hist.p, sizeof h, cudaMemcpyDeviceToHost, st));
            WBX_CUDA(cudaStreamSynchronize(st));
            int digit = -1;
            for (int dgt = 255; dgt >= 0; --dgt) {
                if (above + h[dgt] >= K) {
                    digit = dgt;
                    break;
                }
                above += h[dgt];
            }
            if (digit < 0) {  // fewer than K positions in total: keep every candidate
                all = true;
                break;
            }
            prefix |= static_cast<uint64_t>(digit) << shift;
            mask |= 0xffull << shift;
        }
        const uint64_t kmin = all ? 1ull : prefix;
        const unsigned long long cap = std::max<unsigned long long>(max_records * 4 + 1024, 1ull << 16);
        DevBuf<Sel> sel(cap);
        DevBuf<unsigned long long> cnt(1);
        WBX_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), st));
        collect_kernel<<<grid, 256, 0, st>>>(dbd.p, nb * nb, total, kmin, sel.p, cap, cnt.p);
        unsigned long long ns = 0;
        WBX_CUDA(cudaMemcpyAsync(&ns, cnt.p, sizeof ns, cudaMemcpyDeviceToHost, st));
        WBX_CUDA(cudaStreamSynchronize(st));
        if (ns > cap) fail(WBX_TOO_LARGE, "theta build: too many candidates at the selection boundary");
        std::vector<Sel> hsel(ns);
        if (ns) WBX_CUDA(cudaMemcpy(hsel.data(), sel.p, ns * sizeof(Sel), cudaMemcpyDeviceToHost));
        // the reference's order: key descending, then block, then generator index
        std::sort(hsel.begin(), hsel.end(), [](const Sel& a, const Sel& b) {
            if (a.key != b.key) return a.key > b.key;
            if (a.block != b.block) return a.block < b.block;
            return a.gen_index < b.gen_index;
        });
        uint64_t kept = 0, nrec = 0;
        for (const Sel& c : hsel) {
            if (kept >= K) break;
            if (nrec >= max_records) fail(WBX_TOO_LARGE, "theta build: more kept generator groups than max_records");
            const uint64_t take = std::min<uint64_t>(bd[c.block].mult, K - kept);
            double v = 0.0;
            WBX_CUDA(cudaMemcpy(&v, bd[c.block].gen + c.gen_index, sizeof v, cudaMemcpyDeviceToHost));
            gen_block[nrec] = c.block;
            gen_index[nrec] = c.gen_index;
            gen_count[nrec] = take;
            gen_value[nrec] = v;
            ++nrec;
            kept += take;
        }
        *n_records = nrec;
        count_launch(ctx, 8 + 8 * nb);
        return WBX_OK;
    } catch (const wbx::Error& e) {
        wbx_set_last_error(e.what());
        return e.status;
    }
}

}  // extern "C"
