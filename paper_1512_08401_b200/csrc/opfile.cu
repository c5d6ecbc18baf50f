// Operator files (SURVEY §8f #3, §5 "checkpoint / operator cache").
//
// * WTHETA01 (write_operator / read_operator, theta.cpp:413-490): the reference's bit-exact
//   operator file — magic, u32 header {ndim, dims, J, family, order, nnz}, u64 row offsets,
//   u32 columns, f64 values — with the reference's validation and IoError messages. This is
//   how a C/C++ host hands the device path an operator the reference built (or cached under
//   WAVEBLUR_CACHE, tools/waveblur.cpp:110-151).
// * WBXOP001 (device-ready operator cache, no reference counterpart): the wbx_op exactly as
//   wbx_op_create leaves it — the CSR, the compacted row/column orders, the exact fp64 SELL,
//   the segmented and row-per-lane fp32 layouts of Theta and Theta^T, the window layouts the
//   solvers built so far — plus optional per-operator setup results (the preconditioner p and
//   the step tau). Loading uploads the arrays; nothing is recomputed (no transpose, sort or
//   layout build), so a deployment pays the operator setup once per operator, not per process.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "internal.hpp"

extern "C" void wbx_set_last_error(const char* msg);

namespace wbx {
namespace {

constexpr char kMagic[8] = {'W', 'T', 'H', 'E', 'T', 'A', '0', '1'};
constexpr char kDevMagic[8] = {'W', 'B', 'X', 'O', 'P', '0', '0', '1'};

struct File {
    std::FILE* f = nullptr;
    std::string path;
    File(const char* p, const char* mode) : f(std::fopen(p, mode)), path(p) {}
    ~File() {
        if (f) std::fclose(f);
    }
    void write(const void* p, size_t bytes) {
        if (bytes && std::fwrite(p, 1, bytes, f) != bytes) fail(WBX_IO_ERROR, "write failed: " + path);
    }
    void read(void* p, size_t bytes) {
        if (bytes && std::fread(p, 1, bytes, f) != bytes) fail(WBX_IO_ERROR, "operator file truncated");
    }
    uint32_t u32() {
        uint32_t v;
        read(&v, 4);
        return v;
    }
    uint64_t u64() {
        uint64_t v;
        read(&v, 8);
        return v;
    }
    void put32(uint32_t v) { write(&v, 4); }
    void put64(uint64_t v) { write(&v, 8); }
};

// ---- WBXOP001 record helpers: host vectors and device buffers as (count, raw bytes)
template <typename T>
void put_vec(File& f, const std::vector<T>& v) {
    f.put64(v.size());
    f.write(v.data(), v.size() * sizeof(T));
}
template <typename T>
void get_vec(File& f, std::vector<T>& v, uint64_t max_count) {
    const uint64_t n = f.u64();
    if (n > max_count) fail(WBX_IO_ERROR, f.path + ": corrupt device operator cache (array length)");
    v.resize(n);
    f.read(v.data(), n * sizeof(T));
}
template <typename T>
void put_dev(File& f, const DevBuf<T>& b) {
    std::vector<T> h(b.n);
    if (b.n) WBX_CUDA(cudaMemcpy(h.data(), b.p, b.bytes(), cudaMemcpyDeviceToHost));
    put_vec(f, h);
}
template <typename T>
void get_dev(File& f, DevBuf<T>& b, uint64_t max_count, cudaStream_t s) {
    std::vector<T> h;
    get_vec(f, h, max_count);
    b.alloc(h.size());
    b.upload(h.data(), h.size(), s);
    WBX_CUDA(cudaStreamSynchronize(s));
}

void put_sell(File& f, const wbx_sell& m) {
    f.put64(m.rows);
    f.put64(m.xslices);
    f.put32(m.seg_ok ? 1u : 0u);
    f.put64(m.slices);
    f.put64(m.pairs);
    f.put64(m.rpk_u4);
    put_dev(f, m.xslice_ptr);
    put_dev(f, m.xslice_len);
    put_dev(f, m.val64);
    put_dev(f, m.col);
    put_dev(f, m.row_len);
    put_dev(f, m.slice_ptr);
    put_dev(f, m.slice_np);
    put_dev(f, m.pk);
    put_dev(f, m.lane_info);
    put_dev(f, m.rec_off);
    put_dev(f, m.rec);
    put_dev(f, m.rslice);
    put_dev(f, m.rpk);
}

void get_sell(File& f, wbx_sell& m, uint64_t cap, cudaStream_t s, uint64_t& bytes) {
    m.rows = f.u64();
    m.xslices = f.u64();
    m.seg_ok = f.u32() != 0;
    m.slices = f.u64();
    m.pairs = f.u64();
    m.rpk_u4 = f.u64();
    get_dev(f, m.xslice_ptr, cap, s);
    get_dev(f, m.xslice_len, cap, s);
    get_dev(f, m.val64, cap, s);
    get_dev(f, m.col, cap, s);
    get_dev(f, m.row_len, cap, s);
    get_dev(f, m.slice_ptr, cap, s);
    get_dev(f, m.slice_np, cap, s);
    get_dev(f, m.pk, cap, s);
    get_dev(f, m.lane_info, cap, s);
    get_dev(f, m.rec_off, cap, s);
    get_dev(f, m.rec, cap, s);
    get_dev(f, m.rslice, cap, s);
    get_dev(f, m.rpk, cap, s);
    bytes += m.xslice_ptr.bytes() + m.xslice_len.bytes() + m.val64.bytes() + m.col.bytes() + m.row_len.bytes() +
             m.slice_ptr.bytes() + m.slice_np.bytes() + m.pk.bytes() + m.lane_info.bytes() + m.rec_off.bytes() +
             m.rec.bytes() + m.rslice.bytes() + m.rpk.bytes();
}

void put_compact(File& f, const HostCompact& h) {
    put_vec(f, h.ptr);
    put_vec(f, h.col);
    put_vec(f, h.val);
}
void get_compact(File& f, HostCompact& h, uint64_t cap) {
    get_vec(f, h.ptr, cap);
    get_vec(f, h.col, cap);
    get_vec(f, h.val, cap);
}

void put_win(File& f, const WinSide& w) {
    // src_len < 2^31; its top bit carries the chunk-layout flag
    const uint32_t hdr[7] = {w.G, w.max_u, w.max_win, w.max_rows, w.max_slices, w.max_dict,
                             w.src_len | (w.chunk ? 0x80000000u : 0u)};
    f.write(hdr, sizeof hdr);
    f.put64(w.bytes);
    put_dev(f, w.u_off);
    put_dev(f, w.u_idx);
    put_dev(f, w.s_off);
    put_dev(f, w.r_off);
    put_dev(f, w.d_off);
    put_dev(f, w.u_slot);
    put_dev(f, w.s_tab);
    put_dev(f, w.rec);
    put_dev(f, w.d_val);
}
void get_win(File& f, WinSide& w, uint64_t cap, cudaStream_t s) {
    uint32_t hdr[7];
    f.read(hdr, sizeof hdr);
    w.G = hdr[0];
    w.max_u = hdr[1];
    w.max_win = hdr[2];
    w.max_rows = hdr[3];
    w.max_slices = hdr[4];
    w.max_dict = hdr[5];
    w.src_len = hdr[6] & 0x7fffffffu;
    w.chunk = (hdr[6] >> 31) != 0;
    w.bytes = f.u64();
    get_dev(f, w.u_off, cap, s);
    get_dev(f, w.u_idx, cap, s);
    get_dev(f, w.s_off, cap, s);
    get_dev(f, w.r_off, cap, s);
    get_dev(f, w.d_off, cap, s);
    get_dev(f, w.u_slot, cap, s);
    get_dev(f, w.s_tab, cap, s);
    get_dev(f, w.rec, cap, s);
    get_dev(f, w.d_val, cap, s);
}

}  // namespace
}  // namespace wbx

extern "C" {

int wbx_write_operator(const char* path, uint32_t ndim, const uint64_t* dims, uint32_t J, uint32_t family,
                       uint32_t order, uint64_t n, const uint64_t* row_offsets, const uint32_t* col_indices,
                       const double* values) {
    using namespace wbx;
    try {
        if (!path || !dims || !row_offsets || (row_offsets[n] > 0 && (!col_indices || !values)))
            fail(WBX_INVALID_ARGUMENT, "null argument to wbx_write_operator");
        const uint64_t nnz = row_offsets[n];
        File f(path, "wb");
        if (!f.f) fail(WBX_IO_ERROR, std::string("cannot write operator file ") + path);
        f.write(kMagic, 8);  // theta.cpp:428-443
        f.put32(ndim);
        for (uint32_t d = 0; d < ndim; ++d) f.put32(static_cast<uint32_t>(dims[d]));
        f.put32(J);
        f.put32(family);
        f.put32(order);
        f.put32(static_cast<uint32_t>(nnz));
        f.write(row_offsets, (n + 1) * sizeof(uint64_t));
        f.write(col_indices, nnz * sizeof(uint32_t));
        f.write(values, nnz * sizeof(double));
        if (std::fflush(f.f) != 0) fail(WBX_IO_ERROR, std::string("write failed: ") + path);
        return WBX_OK;
    } catch (const wbx::Error& e) {
        wbx_set_last_error(e.what());
        return e.status;
    }
}

int wbx_read_operator(const char* path, uint32_t* ndim, uint64_t* dims, uint32_t* J, uint32_t* family,
                      uint32_t* order, uint64_t* n_out, uint64_t* nnz_out, uint64_t** row_offsets,
                      uint32_t** col_indices, double** values) {
    using namespace wbx;
    uint64_t* ro = nullptr;
    uint32_t* ci = nullptr;
    double* va = nullptr;
    try {
        if (!path || !ndim || !dims || !J || !family || !order || !n_out || !nnz_out || !row_offsets ||
            !col_indices || !values)
            fail(WBX_INVALID_ARGUMENT, "null argument to wbx_read_operator");
        const std::string p(path);
        File f(path, "rb");
        if (!f.f) fail(WBX_IO_ERROR, "cannot open operator file " + p);  // theta.cpp:445-490
        char magic[8];
        f.read(magic, 8);
        if (std::memcmp(magic, kMagic, 8) != 0) fail(WBX_IO_ERROR, p + ": not a WTHETA01 operator file");
        const uint32_t d = f.u32();
        if (d < 1 || d > 2) fail(WBX_IO_ERROR, p + ": bad dimension count");
        uint64_t dd[2] = {1, 1};
        for (uint32_t k = 0; k < d; ++k) dd[k] = f.u32();
        const uint32_t j = f.u32(), fam = f.u32(), ord = f.u32(), nnz = f.u32();
        if (fam > 2) fail(WBX_IO_ERROR, p + ": bad filter family id");
        std::vector<wbx_band> bands;
        make_layout(d, dd, j, bands);  // the reference's make_layout checks (ShapeMismatch / BadSpec)
        const uint64_t n = d == 2 ? dd[0] * dd[1] : dd[0];
        ro = static_cast<uint64_t*>(std::malloc((n + 1) * sizeof(uint64_t)));
        ci = static_cast<uint32_t*>(std::malloc(std::max<uint64_t>(nnz, 1) * sizeof(uint32_t)));
        va = static_cast<double*>(std::malloc(std::max<uint64_t>(nnz, 1) * sizeof(double)));
        if (!ro || !ci || !va) fail(WBX_MEMORY_GUARD, "operator file: host allocation failed");
        f.read(ro, (n + 1) * sizeof(uint64_t));
        f.read(ci, uint64_t(nnz) * sizeof(uint32_t));
        f.read(va, uint64_t(nnz) * sizeof(double));
        if (ro[0] != 0 || ro[n] != nnz) fail(WBX_IO_ERROR, p + ": inconsistent row offsets");
        for (uint64_t r = 0; r < n; ++r) {
            if (ro[r] > ro[r + 1]) fail(WBX_IO_ERROR, p + ": row offsets not nondecreasing");
            for (uint64_t k = ro[r]; k < ro[r + 1]; ++k) {
                if (ci[k] >= n) fail(WBX_IO_ERROR, p + ": column index out of range");
                if (k > ro[r] && ci[k] <= ci[k - 1]) fail(WBX_IO_ERROR, p + ": columns not strictly increasing in a row");
            }
        }
        *ndim = d;
        dims[0] = dd[0];
        if (d == 2) dims[1] = dd[1];
        *J = j;
        *family = fam;
        *order = ord;
        *n_out = n;
        *nnz_out = nnz;
        *row_offsets = ro;
        *col_indices = ci;
        *values = va;
        return WBX_OK;
    } catch (const wbx::Error& e) {
        std::free(ro);
        std::free(ci);
        std::free(va);
        wbx_set_last_error(e.what());
        return e.status;
    }
}

int wbx_op_get_csr(const wbx_op* op, uint64_t* row_offsets, uint32_t* col_indices, double* values) {
    using namespace wbx;
    try {
        if (!op || !row_offsets || (op->nnz > 0 && (!col_indices || !values)))
            fail(WBX_INVALID_ARGUMENT, "null argument to wbx_op_get_csr");
        std::memcpy(row_offsets, op->h_rowptr.data(), (op->n + 1) * sizeof(uint64_t));
        if (op->nnz) {
            std::memcpy(col_indices, op->h_col.data(), op->nnz * sizeof(uint32_t));
            std::memcpy(values, op->h_val.data(), op->nnz * sizeof(double));
        }
        return WBX_OK;
    } catch (const wbx::Error& e) {
        wbx_set_last_error(e.what());
        return e.status;
    }
}

int wbx_op_save(const wbx_op* op, const char* path, const double* p, double tau) {
    using namespace wbx;
    try {
        if (!op || !path) fail(WBX_INVALID_ARGUMENT, "null argument to wbx_op_save");
        File f(path, "wb");
        if (!f.f) fail(WBX_IO_ERROR, std::string("cannot write device operator cache ") + path);
        WBX_CUDA(cudaSetDevice(op->ctx->device));
        WBX_CUDA(cudaStreamSynchronize(op->ctx->stream));
        f.write(kDevMagic, 8);
        f.put32(WBX_ABI_VERSION);
        f.put64(op->n);
        f.put64(op->nnz);
        f.put64(op->nR);
        f.put64(op->nC);
        put_vec(f, op->h_rowptr);
        put_vec(f, op->h_col);
        put_vec(f, op->h_val);
        put_vec(f, op->h_R_glob);
        put_vec(f, op->h_C_glob);
        put_compact(f, op->hA);
        put_compact(f, op->hT);
        put_sell(f, op->A);
        put_sell(f, op->T);
        put_dev(f, op->isC);
        put_dev(f, op->isR);
        {  // the window layouts the solvers built so far
            std::lock_guard<std::mutex> g(op->win_mu);
            uint32_t cnt = 0;
            for (const auto& kv : op->win_cache) cnt += kv.second->ok ? 1u : 0u;
            f.put32(cnt);
            for (const auto& kv : op->win_cache)
                if (kv.second->ok) {
                    f.put32(kv.first);
                    put_win(f, kv.second->A);
                    put_win(f, kv.second->T);
                }
        }
        // per-operator setup results (optional)
        f.put32(p ? 1u : 0u);
        if (p) f.write(p, op->n * sizeof(double));
        f.write(&tau, sizeof tau);
        if (std::fflush(f.f) != 0) fail(WBX_IO_ERROR, std::string("write failed: ") + path);
        return WBX_OK;
    } catch (const wbx::Error& e) {
        wbx_set_last_error(e.what());
        return e.status;
    }
}

int wbx_op_load(wbx_ctx* ctx, const char* path, wbx_op** out, double* p, int* has_p, double* tau) {
    using namespace wbx;
    wbx_op* op = nullptr;
    try {
        if (!ctx || !path || !out) fail(WBX_INVALID_ARGUMENT, "null argument to wbx_op_load");
        File f(path, "rb");
        if (!f.f) fail(WBX_IO_ERROR, std::string("cannot open device operator cache ") + path);
        char magic[8];
        f.read(magic, 8);
        if (std::memcmp(magic, kDevMagic, 8) != 0)
            fail(WBX_IO_ERROR, std::string(path) + ": not a WBXOP001 device operator cache");
        if (f.u32() != WBX_ABI_VERSION) fail(WBX_IO_ERROR, std::string(path) + ": device operator cache of another ABI");
        WBX_CUDA(cudaSetDevice(ctx->device));
        op = new wbx_op();
        op->ctx = ctx;
        cudaStream_t s = ctx->stream;
        op->n = f.u64();
        op->nnz = f.u64();
        op->nR = f.u64();
        op->nC = f.u64();
        const uint64_t n = op->n, nnz = op->nnz;
        if (n == 0 || n > 0xffffffffull || op->nR > n || op->nC > n)
            fail(WBX_IO_ERROR, std::string(path) + ": corrupt device operator cache (header)");
        const uint64_t cap = std::max<uint64_t>(64, 64 * (n + nnz));  // generous bound on any array
        get_vec(f, op->h_rowptr, n + 1);
        get_vec(f, op->h_col, nnz);
        get_vec(f, op->h_val, nnz);
        get_vec(f, op->h_R_glob, n);
        get_vec(f, op->h_C_glob, n);
        if (op->h_rowptr.size() != n + 1 || op->h_col.size() != nnz || op->h_R_glob.size() != op->nR ||
            op->h_C_glob.size() != op->nC || op->h_rowptr[n] != nnz)
            fail(WBX_IO_ERROR, std::string(path) + ": corrupt device operator cache (CSR)");
        get_compact(f, op->hA, cap);
        get_compact(f, op->hT, cap);
        uint64_t bytes = 0;
        get_sell(f, op->A, cap, s, bytes);
        get_sell(f, op->T, cap, s, bytes);
        get_dev(f, op->isC, cap, s);
        get_dev(f, op->isR, cap, s);
        op->R_glob.upload(op->h_R_glob, s);
        op->C_glob.upload(op->h_C_glob, s);
        bytes += op->R_glob.bytes() + op->C_glob.bytes() + op->isC.bytes() + op->isR.bytes();
        const uint32_t nwin = f.u32();
        for (uint32_t i = 0; i < nwin; ++i) {
            const uint32_t G = f.u32();
            auto wp = std::make_shared<WinPair>();
            get_win(f, wp->A, cap, s);
            get_win(f, wp->T, cap, s);
            wp->ok = true;
            op->win_cache[G] = wp;
        }
        const uint32_t hp = f.u32();
        std::vector<double> pv;
        if (hp) {
            pv.resize(n);
            f.read(pv.data(), n * sizeof(double));
        }
        double t = 0.0;
        f.read(&t, sizeof t);
        op->device_bytes = bytes;
        WBX_CUDA(cudaStreamSynchronize(s));
        if (has_p) *has_p = hp ? 1 : 0;
        if (p && hp) std::memcpy(p, pv.data(), n * sizeof(double));
        if (tau) *tau = t;
        *out = op;
        return WBX_OK;
    } catch (const wbx::Error& e) {
        delete op;
        wbx_set_last_error(e.what());
        return e.status;
    }
}

}  // extern "C"
