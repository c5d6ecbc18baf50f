// The stencil engine's persistent FISTA kernel (included by solver.cu inside its anonymous
// namespace: it shares SolveArgs, the grid barrier, the decoupled pass and the FISTA
// arithmetic with the window engine). Plan and data layout: stencil_engine.cuh.
//
// Per phase a CTA
//   1. bulk-copies the windows of its tiles into shared memory (one 16-byte aligned copy per
//      window row piece, all completing on one mbarrier),
//   2. runs its warp entry lists (per lane: window base from the entry + its class-grid
//      position, per tap one shared load and one fma; the warp's sum for a tile goes to the
//      part-sum slots),
//   3. folds the parts in order and applies the phase's epilogue (A: res = Theta y - x0;
//      T: the window engine's gradient / prox / momentum update, same fmaf expressions).
// Per-output state (x0 of the CTA's A outputs, {y, x_prev, tau/p, threshold} of its T
// outputs) stays in shared memory for the whole solve, as in the window engine.

constexpr int kStBlock = 512;  // one CTA per SM; tiles are 256 thread slots (8 warp slots)
constexpr int kStWarps = kStBlock / 32;
constexpr int kStTileSlots = 8;

// shared-memory footprint (host and device agree on it)
struct StSmemLayout {
    uint32_t taps[2], segs[2], ents[2], outs[2], tasks[2], bands[2], grp[2], red, x0s, cs, win, total;
};

__host__ __device__ inline uint32_t st_a16(uint32_t b) { return (b + 15u) & ~15u; }

__host__ __device__ inline StSmemLayout st_smem_layout(const StencilView& v) {
    StSmemLayout L{};
    uint32_t o = 0;
    auto take = [&](uint32_t bytes) {
        const uint32_t at = o;
        o += st_a16(bytes);
        return at;
    };
    for (int ph = 0; ph < 2; ++ph) {
        const StPhaseView& P = v.ph[ph];
        L.taps[ph] = take(P.ntaps * static_cast<uint32_t>(sizeof(StTap)));
        L.segs[ph] = take(P.max_segs * static_cast<uint32_t>(sizeof(StSeg)));
        L.ents[ph] = take(P.max_rows * static_cast<uint32_t>(sizeof(StEntry)));
        L.grp[ph] = take(P.max_tasks * kStTileSlots * 4u);
        L.outs[ph] = take(P.max_outs * static_cast<uint32_t>(sizeof(StOut)));
        L.tasks[ph] = take(P.max_tasks * static_cast<uint32_t>(sizeof(StTask)));
        L.bands[ph] = take(P.nbands * static_cast<uint32_t>(sizeof(StBand)));
    }
    const uint32_t mt = v.ph[0].max_rows > v.ph[1].max_rows ? v.ph[0].max_rows : v.ph[1].max_rows;
    const uint32_t mw = v.ph[0].max_win > v.ph[1].max_win ? v.ph[0].max_win : v.ph[1].max_win;
    L.red = take(mt * 32u * 4u);
    L.x0s = take(v.ph[0].max_outs * 4u);
    L.cs = take(v.ph[1].max_outs * 16u);
    L.win = take(mw * 4u);
    L.total = o;
    return L;
}

struct StSmemPhase {
    const StTap* taps;
    const StSeg* segs;
    const StEntry* ents;
    const StOut* outs;
    const StTask* tasks;
    const StBand* bands;
    const uint32_t* grp;
    const StTapX* tapx;  // global (partial walks only)
    uint32_t nseg, nout, ent_beg, ent_end, bytes;  // ent_*: the calling warp's entries
};

struct StSmem {
    StSmemPhase ph[2];
    float* red;
    float* x0s;
    float4* cs;
    float* win;
};

__device__ __forceinline__ void st_copy(unsigned char* dst, const void* src, uint32_t bytes) {
    const uint32_t* s = static_cast<const uint32_t*>(src);
    uint32_t* d = reinterpret_cast<uint32_t*>(dst);
    for (uint32_t i = threadIdx.x; i < bytes / 4u; i += kStBlock) d[i] = s[i];
}

template <typename T>
__device__ __forceinline__ const T* st_stage(unsigned char* base, uint32_t at, const T* src, uint32_t count) {
    st_copy(base + at, src, count * static_cast<uint32_t>(sizeof(T)));
    return reinterpret_cast<const T*>(base + at);
}

__device__ __forceinline__ StSmem st_smem_init(unsigned char* base, const StencilView& v) {
    const StSmemLayout L = st_smem_layout(v);
    const uint32_t b = blockIdx.x, w = threadIdx.x >> 5;
    StSmem S;
    for (int ph = 0; ph < 2; ++ph) {
        const StPhaseView& P = v.ph[ph];
        StSmemPhase& Q = S.ph[ph];
        Q.taps = st_stage(base, L.taps[ph], P.taps, P.ntaps);
        Q.bands = st_stage(base, L.bands[ph], P.bands, P.nbands);
        Q.nseg = P.seg_off[b + 1] - P.seg_off[b];
        Q.nout = P.out_off[b + 1] - P.out_off[b];
        Q.segs = st_stage(base, L.segs[ph], P.segs + P.seg_off[b], Q.nseg);
        Q.outs = st_stage(base, L.outs[ph], P.outs + P.out_off[b], Q.nout);
        Q.tasks = st_stage(base, L.tasks[ph], P.tasks + P.task_off[b], P.task_off[b + 1] - P.task_off[b]);
        const uint32_t e0 = P.ent_off[b * kStWarps];
        Q.ents = st_stage(base, L.ents[ph], P.ents + e0, P.ent_off[(b + 1) * kStWarps] - e0);
        Q.grp = st_stage(base, L.grp[ph], P.grp + P.task_off[b] * kStTileSlots,
                         (P.task_off[b + 1] - P.task_off[b]) * kStTileSlots);
        Q.ent_beg = P.ent_off[b * kStWarps + w] - e0;
        Q.ent_end = P.ent_off[b * kStWarps + w + 1] - e0;
        Q.bytes = P.win_bytes[b];
        Q.tapx = P.tapx;
    }
    S.red = reinterpret_cast<float*>(base + L.red);
    S.x0s = reinterpret_cast<float*>(base + L.x0s);
    S.cs = reinterpret_cast<float4*>(base + L.cs);
    S.win = reinterpret_cast<float*>(base + L.win);
    __syncthreads();
    return S;
}

// Output position of pixel e of a tile: class-major (the 2^smax x 2^smax residue classes one
// after the other, each a row-major sub-grid), so a half warp's outputs share one class.
__device__ __forceinline__ void st_out_pos(const StBand& b, uint32_t a0, uint32_t a1, uint32_t e, uint32_t& q0,
                                           uint32_t& q1) {
    const uint32_t per_class_l = b.lTH + b.lTW - 2u * b.smax;
    const uint32_t c = e >> per_class_l, wi = e & ((1u << per_class_l) - 1u);
    const uint32_t ltwm = b.lTW - b.smax;
    q0 = a0 + ((wi >> ltwm) << b.smax) + (c >> b.smax);
    q1 = a1 + ((wi & ((1u << ltwm) - 1u)) << b.smax) + (c & ((1u << b.smax) - 1u));
}

// WBX_PROFILE=3 (diagnostics build): per-warp cycles [A fill, A taps, A epilogue, A barrier,
// T fill, ...] summed into g_prof (tools/st_profile.py)
template <typename Epi>
__device__ __forceinline__ void st_phase(const StSmem& S, const StSmemPhase& Q, const float* __restrict__ src,
                                         uint64_t* bar, unsigned& parity, int fill, Epi epi,
                                         unsigned long long* pc = nullptr) {
    const uint32_t tid = threadIdx.x, lane = tid & 31u;
    const long long c0 = WBX_PROFILE == 3 ? clock64() : 0;
    // 1. windows (the grid barrier ordered the producers' stores before this CTA's acquire; the
    // proxy fence orders them, and this CTA's last reads of the window, before the bulk copies)
    if (fill == 2) {  // cp.async 16 B, L2 only: warp w copies pieces w, w + 8, ...
        for (uint32_t k = tid >> 5; k < Q.nseg; k += kStWarps) {
            const StSeg sg = Q.segs[k];
            const unsigned dst = smem_u32(S.win + sg.dst);
            const float* sp = src + sg.src;
            for (uint32_t c = lane; c < sg.bytes / 16u; c += 32u)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16u * c), "l"(sp + 4u * c) : "memory");
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
        __syncthreads();
    } else {
        if (tid == 0) mbar_expect_tx(bar, Q.bytes);
        if (fill == 0 && tid < Q.nseg) asm volatile("fence.proxy.async;" ::: "memory");
        for (uint32_t k = tid; k < Q.nseg; k += kStBlock) {
            const StSeg sg = Q.segs[k];
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             smem_u32(S.win + sg.dst)),
                         "l"(src + sg.src), "r"(sg.bytes), "r"(smem_u32(bar))
                         : "memory");
        }
        mbar_wait(bar, parity);
        parity ^= 1u;
    }
    const long long c1 = WBX_PROFILE == 3 ? clock64() : 0;
    // 2. warp entries: each writes its 32 sums to its part-sum row
    uint32_t cur = 0xffffffffu, kr = 0, kc = 0, e = 0;
    const uint32_t h = lane >> 4;
    for (uint32_t k = Q.ent_beg; k < Q.ent_end; ++k) {
        const StEntry en = Q.ents[k];
        const uint32_t key = (static_cast<uint32_t>(en.task) << 8) | en.slot;
        if (key != cur) {
            cur = key;
            const StBand& b = Q.bands[Q.tasks[en.task].band];
            const uint32_t lnp = b.lTH + b.lTW;
            e = ((static_cast<uint32_t>(en.slot) << 5) + lane) & ((1u << lnp) - 1u);
            const uint32_t wi = e & ((1u << (lnp - 2u * b.smax)) - 1u);
            const uint32_t ltwm = b.lTW - b.smax;
            kr = wi >> ltwm;
            kc = wi & ((1u << ltwm) - 1u);
        }
        const int base = (h ? en.base[1] : en.base[0]) + static_cast<int>(kr * en.rstride + (kc << en.cshift));
        const uint32_t rng = h ? en.rng[1] : en.rng[0];
        const uint32_t lo = rng & 0xffffu, hi = rng >> 16;
        const float* w = S.win + base;
        float acc = 0.f;
        if (!(en.flags & kStPartial)) {
            uint32_t r = lo;
#pragma unroll 1
            for (; r + 4 <= hi; r += 4) {
                const StTap t0 = Q.taps[r], t1 = Q.taps[r + 1], t2 = Q.taps[r + 2], t3 = Q.taps[r + 3];
                const float v0 = w[t0.off], v1 = w[t1.off], v2 = w[t2.off], v3 = w[t3.off];
                acc = fmaf(t0.val, v0, acc);
                acc = fmaf(t1.val, v1, acc);
                acc = fmaf(t2.val, v2, acc);
                acc = fmaf(t3.val, v3, acc);
            }
            for (; r < hi; ++r) {
                const StTap t0 = Q.taps[r];
                acc = fmaf(t0.val, w[t0.off], acc);
            }
        } else {  // a tap of the range covers only the first `count` small-band positions
            const StTask tk = Q.tasks[en.task];
            const StBand& b = Q.bands[tk.band];
            uint32_t q0, q1;
            st_out_pos(b, static_cast<uint32_t>(tk.t0) << b.lTH, static_cast<uint32_t>(tk.t1) << b.lTW, e, q0, q1);
            const int sl0 = en.job_sl >> 4, sl1 = en.job_sl & 15;
            const int m0 = (1 << sl0) - 1, m1 = (1 << sl1) - 1;
            const int dflat = static_cast<int>((q0 << b.l1) + q1);
            const int sq0 = static_cast<int>(q0 >> en.job_s), sq1 = static_cast<int>(q1 >> en.job_s);
            for (uint32_t r = lo; r < hi; ++r) {
                const StTap t0 = Q.taps[r];
                const StTapX x = Q.tapx[r];
                float v = w[t0.off];
                if (x.count >= 0) {
                    const int flat = en.job_up ? (((sq0 - x.j0) & m0) << sl1) + ((sq1 - x.j1) & m1) : dflat;
                    if (flat >= x.count) v = 0.f;
                }
                acc = fmaf(t0.val, v, acc);
            }
        }
        S.red[(static_cast<uint32_t>(en.row) << 5) + lane] = acc;
    }
    const long long c2 = WBX_PROFILE == 3 ? clock64() : 0;
    __syncthreads();
    // 3. parts in order, epilogue (every thread: outputs tid, tid + 256, ...)
    for (uint32_t k = tid; k < Q.nout; k += kStBlock) {
        const StOut o = Q.outs[k];
        float total = 0.f;
        for (uint32_t p = 0; p < o.P; ++p) {  // parts in order, each its rows in order
            const uint32_t x = (p << o.lnp) + o.e;
            const uint32_t g = Q.grp[o.task * kStTileSlots + (x >> 5)];
            for (uint32_t r = g & 0xffffu; r < (g >> 16); ++r) total += S.red[(r << 5) + (x & 31u)];
        }
        epi(k, o.idx, total);
    }
    if (WBX_PROFILE == 3 && pc) {
        const long long c3 = clock64();
        pc[0] += c1 - c0;
        pc[1] += c2 - c1;
        pc[2] += c3 - c2;
    }
}

__global__ void __launch_bounds__(kStBlock, 1) fista_stencil_kernel(SolveArgs a) {
    __shared__ double smem[kStWarps + 1];
    __shared__ __align__(8) uint64_t bar;
    extern __shared__ __align__(16) unsigned char dsmem[];
    const uint64_t gthread = static_cast<uint64_t>(blockIdx.x) * kStBlock + threadIdx.x;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * kStBlock;
    const unsigned epoch0 = *reinterpret_cast<volatile unsigned*>(a.sync.gen);
    Epoch epoch{epoch0, epoch0};
    const double tau = a.tau_from_device ? a.out[OUT_TAU] : a.tau_given;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_fence_init();
    }
    const StSmem S = st_smem_init(dsmem, a.st);
    float* yP = a.yF;     // phase A source
    float* resP = a.resF; // phase T source
    unsigned parity = 0;
    for (uint32_t k = threadIdx.x; k < S.ph[1].nout; k += kStBlock) {
        const uint32_t i = S.ph[1].outs[k].idx;
        const float v = static_cast<float>(a.x0_full[i]);
        yP[i] = v;
        S.cs[k] = make_float4(v, v, static_cast<float>(tau / a.p_full[i]),
                              static_cast<float>(thr_exact(tau, a.lambda, a.w_full[i], a.p_full[i])));
    }
    for (uint32_t k = threadIdx.x; k < S.ph[0].nout; k += kStBlock)
        S.x0s[k] = static_cast<float>(a.x0_full[S.ph[0].outs[k].idx]);
    // coordinates outside the Theta^T output bands (a.isC = the plan's coupled mask here)
    if (a.decoupled_inline) decoupled_pass<float>(a, tau, a.max_iters, 0, gthread, nthreads, nullptr, nullptr, 0);
    grid_sync(a.sync, epoch, smem);
    unsigned long long pc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    auto sync = [&](int side) {
        const long long b0 = WBX_PROFILE == 3 ? clock64() : 0;
        grid_sync(a.sync, epoch, smem);
        if (WBX_PROFILE == 3) pc[side + 3] += clock64() - b0;
    };
    for (int k = 1; k <= a.max_iters; ++k) {
        st_phase(S, S.ph[0], yP, &bar, parity, a.st_fill, [&](uint32_t o, uint32_t i, float acc) {
            resP[i] = acc - S.x0s[o];
        }, pc);
        sync(0);
        const float beta = a.beta32[k - 1];
        st_phase(S, S.ph[1], resP, &bar, parity, a.st_fill, [&](uint32_t o, uint32_t i, float g) {
            float4& s = S.cs[o];
            const float z0 = fmaf(-s.z, g, s.x);
            const float xn = Prec<float>::prox(z0, s.w);
            const float yn = fmaf(beta, xn - s.y, xn);
            s.x = yn;
            s.y = xn;
            yP[i] = yn;
        }, pc + 4);
        sync(4);
    }
    if (WBX_PROFILE == 3 && (threadIdx.x & 31) == 0)
        for (int i = 0; i < 8; ++i) atomicAdd(&g_prof[i], pc[i]);
    if (gthread == 0) a.out[OUT_ITERS_USED] = a.max_iters;
    for (uint32_t k = threadIdx.x; k < S.ph[1].nout; k += kStBlock)
        a.x_full[S.ph[1].outs[k].idx] = static_cast<double>(S.cs[k].y);
}
