// Internal declarations of libwbx (not part of the ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "wbx.h"

namespace wbx {

// Exception carrying a wbx_status; converted to a status code at the C-ABI edge.
struct Error : std::runtime_error {
    int status;
    Error(int s, const std::string& msg) : std::runtime_error(msg), status(s) {}
};

[[noreturn]] inline void fail(int status, const std::string& msg) { throw Error(status, msg); }

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        fail(WBX_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}
#define WBX_CUDA(call) ::wbx::cuda_check((call), #call)

// Device buffer owned by RAII.
template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            n = o.n;
            o.p = nullptr;
            o.n = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t count) {
        release();
        n = count;
        if (count) WBX_CUDA(cudaMalloc(&p, count * sizeof(T)));
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    size_t bytes() const { return n * sizeof(T); }
    void upload(const T* h, size_t count, cudaStream_t s) {
        if (count) WBX_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    void upload(const std::vector<T>& h, cudaStream_t s) {
        if (n < h.size()) alloc(h.size());
        upload(h.data(), h.size(), s);
    }
};

// winlayout.cu: per-CTA window layout of one operator side (win.cuh)
struct WinSide {
    uint32_t G = 0, max_u = 0, max_win = 0, max_rows = 0, max_slices = 0, max_dict = 0;
    uint32_t src_len = 0;  // length of the gathered vector (set by the solver)
    bool chunk = false;    // chunk layout (win.cuh WinView::chunk)
    DevBuf<uint32_t> u_off, u_idx, s_off, r_off, d_off;
    DevBuf<uint16_t> u_slot;
    DevBuf<uint4> s_tab, rec;
    DevBuf<float> d_val;
    uint64_t bytes = 0;
};
struct StencilPlan;  // stencil_plan.cu
struct CircPlan;     // circ_tau.cu

// both sides for one grid size G; ok == false when a window exceeds 16-bit local indices
struct WinPair {
    WinSide A, T;
    bool ok = false;
};

}  // namespace wbx

struct wbx_ctx {
    int device = 0;
    int num_sms = 0;
    cudaStream_t stream = nullptr;
    uint64_t launches = 0;
    // standalone SpMV: compacted input / output of the calling context
    wbx::DevBuf<double> scratch64[2];
    wbx::DevBuf<float> scratch32[2];
};

// Wavelet layout + filters (WaveletBasis, wavelet.hpp:68-74).
struct wbx_basis {
    wbx_ctx* ctx = nullptr;
    uint32_t family = 0, order = 0, ndim = 2, J = 1;
    uint64_t dims[2] = {1, 1};
    std::vector<wbx_band> bands;
    double lo[20] = {0}, hi[20] = {0};
    uint32_t len = 0;
    uint64_t n = 0;
    wbx::DevBuf<double> work_a, work_b, io;  // ping-pong scratch + staging
};

// Compacted sliced-ELL (SELL-32) operator. Rows of the slice structure are the
// NONEMPTY rows of the matrix, sorted by descending length; columns are remapped to
// positions in the compacted column space of the consuming vector.
struct wbx_sell {
    uint64_t rows = 0;     // real rows
    // exact fp64 layout (one lane per row, element-major): slice s, element j, lane l at
    // xslice_ptr[s] + 32*j + l
    uint64_t xslices = 0;
    wbx::DevBuf<uint64_t> xslice_ptr;
    wbx::DevBuf<uint32_t> xslice_len;
    wbx::DevBuf<double> val64;
    wbx::DevBuf<uint32_t> col;
    wbx::DevBuf<uint32_t> row_len;
    // segmented fp32 layout (rows split into <= 16-element segments, one lane each); absent
    // (seg_ok false, fp64 entry points only) when a row is longer than 31 segments
    bool seg_ok = true;
    uint64_t slices = 0;
    uint64_t pairs = 0;               // uint4 element pairs incl. padding
    wbx::DevBuf<uint64_t> slice_ptr;  // pair offset of each slice
    wbx::DevBuf<uint32_t> slice_np;   // pairs per lane in the slice (<= 8)
    wbx::DevBuf<uint4> pk;            // {val0,col0,val1,col1} fp32 pairs
    wbx::DevBuf<uint32_t> lane_info;  // head lane: row | nseg << 27; else 0xffffffff
    // the same slices as contiguous records for TMA staging: [lane_info x32][pairs]
    wbx::DevBuf<uint64_t> rec_off;    // uint4 offset of each record
    wbx::DevBuf<uint4> rec;
    // row-per-lane fp32 layout (the standalone SpMV, spmv.cu sell_row_kernel): the xslices
    // of the exact layout (32 consecutive sorted rows, one per lane), element-major, packed as
    // {val, col, val, col} pairs [np x 32 x uint4] followed, for an odd slice length L, by the
    // last element [32 x uint2]. Row sums run in element order. No per-lane row word: rows of
    // slice s are s*32 + lane; no segment padding (rows of a slice have ~equal length, they
    // are sorted). rslice[s] = {uint4 offset, L}.
    wbx::DevBuf<uint2> rslice;
    wbx::DevBuf<uint4> rpk;
    uint64_t rpk_u4 = 0;
};

// A compacted operator side on the host: rows in the solver's sorted order, columns as
// positions in the compacted space of the vector they multiply.
struct HostCompact {
    std::vector<uint64_t> ptr;
    std::vector<uint32_t> col;
    std::vector<double> val;
    uint64_t rows() const { return ptr.empty() ? 0 : ptr.size() - 1; }
};

struct wbx_op {
    wbx_ctx* ctx = nullptr;
    HostCompact hA, hT;           // host copies of the two compacted sides
    uint64_t n = 0, nnz = 0;
    uint64_t nR = 0, nC = 0;      // nonempty rows / nonempty columns
    wbx_sell A;                   // Theta   : rows = R (sorted), cols -> C positions
    wbx_sell T;                   // Theta^T : rows = C (sorted), cols -> R positions
    wbx::DevBuf<uint32_t> R_glob; // R position -> original row
    wbx::DevBuf<uint32_t> C_glob; // C position -> original column
    wbx::DevBuf<uint32_t> isC;    // bitmask over n: column nonempty
    wbx::DevBuf<uint32_t> isR;    // bitmask over n: row nonempty
    std::vector<uint32_t> h_R_glob, h_C_glob;
    // host copy of the CSR (for the exact host-side setup routines: Gram diagonals)
    std::vector<uint64_t> h_rowptr;
    std::vector<uint32_t> h_col;
    std::vector<double> h_val;
    uint64_t device_bytes = 0;
    // window layouts per solver grid size, built once per operator and shared by every solver
    // on it (a host loop calling fista() on one operator pays the layout build once)
    mutable std::mutex win_mu;
    mutable std::map<uint32_t, std::shared_ptr<wbx::WinPair>> win_cache;
    // the operator as the reference's kept generator groups (stationary Theta_K), when the
    // caller attached them (wbx_op_set_generators, checked against the CSR): the stencil engine
    bool has_gens = false;
    uint32_t g_ndim = 0;
    std::vector<wbx_band> g_bands;
    std::vector<uint32_t> g_block, g_index;
    std::vector<uint64_t> g_count;
    std::vector<double> g_val;
    mutable std::map<uint64_t, std::shared_ptr<wbx::StencilPlan>> st_cache;  // by (CTA warps, G)
    // the wavelet layout the operator acts on (SparseOperator::layout, theta.hpp:55), when the
    // caller attached it (wbx_op_set_layout / wbx_op_set_generators)
    bool has_layout = false;
    uint32_t l_ndim = 0, l_J = 0;
    uint64_t l_dims[2] = {1, 1};
    std::vector<wbx_band> l_bands;
    // block-Fourier step-estimate plans (circ_tau.cu) per wavelet layout (ndim, dims, J)
    mutable std::map<std::vector<uint64_t>, std::shared_ptr<wbx::CircPlan>> circ_cache;
};

namespace wbx {

constexpr uint64_t kSegElems = 16;  // max elements per lane segment (8 uint4 pairs)
constexpr uint32_t kInfoShift = 27;

// Kernel-launch accounting (gpu_launches in bench.py).
inline void count_launch(wbx_ctx* ctx, uint64_t k = 1) { ctx->launches += k; }

// dwt.cu
void analyze_dev(wbx_basis* b, const double* u, double* x, cudaStream_t s);
// nimg images back to back (n doubles apart, work buffers n doubles per image each)
void analyze_dev_n(wbx_basis* b, const double* u, double* x, uint32_t nimg, double* work_a, double* work_b,
                   cudaStream_t s);
void synthesize_dev_n(wbx_basis* b, const double* x, double* u, uint32_t nimg, double* work_a, double* work_b,
                      cudaStream_t s, int clamp = 0);
// clamp: the deblur's final clamp to [0, 1] fused into the last level
void synthesize_dev(wbx_basis* b, const double* x, double* u, cudaStream_t s, int clamp = 0);
void make_layout(uint32_t ndim, const uint64_t* dims, uint32_t J, std::vector<wbx_band>& bands);
void make_filters(uint32_t family, uint32_t order, double* lo, double* hi, uint32_t* len);

// spmv.cu
// mode: the fp32 SELL kernel (-1: WBX_SPMV / default row kernel; see spmv.cu spmv_mode)
template <typename T>
void spmv_compact(wbx_ctx* ctx, const wbx_sell& M, const T* x, T* y, cudaStream_t s, int mode = -1);
void spmv_full_fp64(wbx_ctx* ctx, const wbx_op* op, int transpose, const double* x_dev, double* y_dev);
void spmv_full_fp32(wbx_ctx* ctx, const wbx_op* op, int transpose, const float* x_dev, float* y_dev);
void set_spmv_pf_bytes(long long bytes);  // row kernel's L2 prefetch distance (-1: default)

// op_build.cu
struct SellView;
SellView view_of(const wbx_sell& m);

void build_op(wbx_op* op, uint64_t n, const uint64_t* rowptr, const uint32_t* col,
              const double* val);
// SELL layouts (both the segmented fp32 and the exact fp64 one) of `nrows` rows given by
// len(i) and get(i, j, col, val), uploaded into `out`.
void build_sell(wbx_sell& out, uint64_t nrows, const std::function<uint64_t(uint64_t)>& len,
                const std::function<void(uint64_t, uint64_t, uint32_t&, double&)>& get, cudaStream_t s,
                uint64_t& bytes);

// winlayout.cu: per-CTA window layout of one operator side (WinSide, above)
// side 'A' or 'T'; chunk: the chunk layout (fp32 sources, 16-byte window copies)
void build_win(WinSide& out, const HostCompact& M, uint32_t G, cudaStream_t st, char side, bool chunk);
struct WinView;
WinView view_of(const WinSide& w);

// gram.cu: Gram diagonals on the device (shared-memory tables, global-memory second pass for
// columns whose 2-hop set overflows them)
void gram_device(wbx_ctx* ctx, const wbx_op* op, uint64_t cap_factor, double* diagM, double* diagM2);

// stencil_plan.cu: the stencil engine's plan for grid G (ok == false when it does not apply)
std::shared_ptr<StencilPlan> build_stencil_plan(const std::vector<wbx_band>& bands, uint32_t ndim, uint64_t n,
                                                const std::vector<uint32_t>& gblock, const std::vector<uint32_t>& gidx,
                                                const std::vector<uint64_t>& gcount, const std::vector<double>& gval,
                                                uint32_t G, uint32_t cta_warps, uint32_t smem_budget_floats);
void upload_stencil_plan(StencilPlan& p, cudaStream_t st);
bool stencil_plan_ok(const StencilPlan& p, std::string* why);
void stencil_apply_host(const StencilPlan& p, int ph, const double* src, double* out);
struct StencilView;
StencilView view_of(const StencilPlan& p);
// the operator's plan for grid G (built from its generator groups, uploaded, cached on it)
std::shared_ptr<StencilPlan> stencil_plan_for(const wbx_op* op, uint32_t G, uint32_t cta_warps, cudaStream_t st);

// solver.cu: wbx_pgd's solver cache (drop entries of a context / an operator)
void pgd_purge(const wbx_ctx* ctx, const wbx_op* op);

// circ_tau.cu: the step estimate of translation-invariant operators, block-diagonal in the
// Fourier domain of the translation group (ok == false when it does not apply)
std::shared_ptr<CircPlan> circ_analyze(const wbx_op* op, uint32_t ndim, const uint64_t* dims, uint32_t J,
                                       const std::vector<wbx_band>& bands);
bool circ_plan_ok(const CircPlan& p, std::string* why, uint32_t* info5);  // {ok, nRo, nCo, g0, g1}
bool circ_check_p(const CircPlan& p, const double* p_full, std::vector<double>& isp, std::string* why);
void circ_upload(CircPlan& p, cudaStream_t st);
uint64_t circ_work_doubles(const CircPlan& p);
void circ_tau_launch(wbx_ctx* ctx, const CircPlan& p, const double* isp_dev, double step_safety, double* work,
                     double2* gram, double* out, cudaStream_t st, cudaStream_t aux, cudaEvent_t ev_fork,
                     cudaEvent_t ev_join);
uint64_t circ_gram_doubles(const CircPlan& p);
void circ_gram_launch(wbx_ctx* ctx, const CircPlan& p, double2* gram, cudaStream_t st);
// the spectral FISTA engine (fp64 iterations, gradient in the Fourier domain of the group)
struct CircProblem {
    const double* x0_full;
    const double* w_full;
    const double* p_full;
    double* x_full;
    const uint32_t* isC;
    const double* beta64;
    double lambda;
    int K;
    const double* out;  // tau at out[0]
    // energy / support tracking (no ref_energy rule): work buffer (circ_track_doubles) and outputs
    double* track_work = nullptr;
    double* energies = nullptr;
    unsigned long long* supports = nullptr;
    // images in this launch (C5 batches, untracked): x0_full / x_full hold nimg images back to
    // back, T nimg exchange buffers (circ_exchange_doubles each), counter 32 words per image
    uint32_t nimg = 1;
};
// images of a batch the spectral engine solves in one launch (NB spectral CTAs per image, the
// rest of the SMs for the decoupled coordinates)
uint32_t circ_fista_slots(const CircPlan& p, int num_sms, uint32_t batch);
bool circ_fista_ok(const CircPlan& p, std::string* why);
uint64_t circ_track_doubles(const CircPlan& p, int K, int num_sms);
uint64_t circ_exchange_doubles(const CircPlan& p);
uint32_t circ_fista_blocks(const CircPlan& p);
void circ_fista_launch(wbx_ctx* ctx, const CircPlan& p, const CircProblem& pr, const double2* gram, double2* T,
                       unsigned* counter, cudaStream_t st);

// theta_build.cu (host): CSR assembly of thresholded circulant operators
struct HostCsr {
    std::vector<uint64_t> rowptr;
    std::vector<uint32_t> col;
    std::vector<double> val;
};
HostCsr expand_generators(const std::vector<wbx_band>& bands, uint32_t ndim, uint64_t n, uint64_t n_gens,
                          const uint32_t* blocks, const uint32_t* gen_index, const uint64_t* counts,
                          const double* values);

}  // namespace wbx
