// Host planner of the stencil engine (stencil_engine.cuh): from the kept generator groups of a
// stationary Theta_K, the per-(phase, output band) tilings, the blocks with their window
// geometry and class-split tap lists, the tile -> CTA assignment and
// each CTA's window copies, warp entry lists and outputs; plus a host execution of the plan
// through exactly those tables (the tests compare it with the CSR products).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <queue>
#include <string>
#include <tuple>
#include <vector>

#include "internal.hpp"
#include "stencil_engine.cuh"

extern "C" void wbx_set_last_error(const char* msg);

namespace wbx {

struct StHostPhase {
    std::vector<StBand> bands;
    std::vector<StTap> taps;
    std::vector<StTapX> tapx;
    std::vector<uint32_t> task_off, seg_off, ent_off, out_off, win_bytes;
    std::vector<uint32_t> grp;  // per (task, warp slot): canonical entry range lo | hi << 16
    std::vector<StTask> tasks;
    std::vector<StSeg> segs;
    std::vector<StEntry> ents;
    std::vector<StOut> outs;
    uint32_t max_tasks = 0, max_segs = 0, max_ents = 0, max_outs = 0, max_win = 0, max_rows = 0;
    uint32_t cta_warps = 0;
    double work_max = 0.0, work_mean = 0.0;
};

struct StencilPlan {
    bool ok = false;
    std::string why;
    uint32_t G = 0;
    StHostPhase h[2];
    std::vector<uint32_t> coupled;  // bitmask over n
    struct Dev {
        DevBuf<StBand> bands;
        DevBuf<StTap> taps;
        DevBuf<StTapX> tapx;
        DevBuf<uint32_t> task_off, seg_off, ent_off, out_off, win_bytes, grp;
        DevBuf<StTask> tasks;
        DevBuf<StSeg> segs;
        DevBuf<StEntry> ents;
        DevBuf<StOut> outs;
    } d[2];
    DevBuf<uint32_t> d_coupled;
};

namespace {

constexpr int kStThreads = 256;                  // thread slots of a tile (P parts x pixels)
constexpr int kStSlots = kStThreads / 32;        // warp slots of a tile
constexpr double kTapsPerThread = 24.0;  // target taps per thread before an output is split in parts

uint32_t lg2(uint64_t v) {
    uint32_t l = 0;
    while ((1ull << l) < v) ++l;
    return l;
}

int64_t floor_shift(int64_t x, uint32_t s) { return x >= 0 ? (x >> s) : -((-x + (1ll << s) - 1) >> s); }
int64_t pmod(int64_t x, int64_t m) { return ((x % m) + m) % m; }
uint32_t up4(int64_t v) { return static_cast<uint32_t>((v + 3) & ~3ll); }

struct RecIn {
    uint32_t block, o, i;
    int64_t vs0, vs1;   // signed generator offset in the large band
    uint64_t v0, v1;
    uint64_t count, full;
    double val;
};

// a block of a (phase, output band) while planning
struct PBlock {
    bool up;
    uint32_t s, src;
    double taps;                              // taps per output (UP: per class on average)
    int64_t c0, c1;
    uint32_t R0, R1, R1p, woff;
    std::vector<std::pair<uint32_t, uint32_t>> cls;  // per class: tap range [lo, hi) in the phase's taps
};
struct PJob {                                 // a part's share of a block: per class tap range
    uint32_t blk;
    std::vector<std::pair<uint32_t, uint32_t>> cls;
};
struct PBand {
    uint32_t band;                            // layout band
    std::vector<PBlock> blocks;
    std::vector<std::vector<PJob>> parts;
    uint32_t win;                             // window floats of one tile
    double work;                              // cost model of one tile
};

// class-major pixel order of a tile (the kernel's st_out_pos)
inline void st_output(const StBand& b, uint32_t a0, uint32_t a1, uint32_t e, uint32_t& q0, uint32_t& q1) {
    const uint32_t per_class_l = b.lTH + b.lTW - 2u * b.smax;
    const uint32_t c = e >> per_class_l, wi = e & ((1u << per_class_l) - 1u);
    const uint32_t ltwm = b.lTW - b.smax;
    q0 = a0 + ((wi >> ltwm) << b.smax) + (c >> b.smax);
    q1 = a1 + ((wi & ((1u << ltwm) - 1u)) << b.smax) + (c & ((1u << b.smax) - 1u));
}
// position of pixel e inside its class grid (the kernel's krow / kcol)
inline void st_kpos(const StBand& b, uint32_t e, uint32_t& krow, uint32_t& kcol) {
    const uint32_t per_class_l = b.lTH + b.lTW - 2u * b.smax;
    const uint32_t wi = e & ((1u << per_class_l) - 1u);
    const uint32_t ltwm = b.lTW - b.smax;
    krow = wi >> ltwm;
    kcol = wi & ((1u << ltwm) - 1u);
}
int64_t win_base0(const PBlock& b, int64_t a0) { return (b.up ? (a0 >> b.s) : (a0 << b.s)) + b.c0; }
int64_t win_base1(const PBlock& b, int64_t a1) { return (b.up ? (a1 >> b.s) : (a1 << b.s)) + b.c1; }

// window offset (relative to the window origin, pitch R1p, data from column delta) of the tap
// base of output (q0, q1) of the tile at (a0, a1)
int64_t tap_base(const PBlock& b, uint32_t a0, uint32_t a1, uint32_t q0, uint32_t q1, int64_t delta) {
    if (!b.up) return (static_cast<int64_t>(q0 - a0) << b.s) * b.R1p + (static_cast<int64_t>(q1 - a1) << b.s) + delta;
    return (static_cast<int64_t>(q0 >> b.s) - static_cast<int64_t>(a0 >> b.s) - b.c0) * b.R1p +
           (static_cast<int64_t>(q1 >> b.s) - static_cast<int64_t>(a1 >> b.s) - b.c1) + delta;
}

}  // namespace

// Build the plan for grid G; returns it with ok == false (and why) when the operator does not
// suit the engine (1-D layouts, non-power-of-two bands, scales above 2, windows too large).
std::shared_ptr<StencilPlan> build_stencil_plan(const std::vector<wbx_band>& bands, uint32_t ndim, uint64_t n,
                                                const std::vector<uint32_t>& gblock, const std::vector<uint32_t>& gidx,
                                                const std::vector<uint64_t>& gcount, const std::vector<double>& gval,
                                                uint32_t G, uint32_t cta_warps, uint32_t smem_budget_floats) {
    auto plan = std::make_shared<StencilPlan>();
    plan->G = G;
    plan->h[0].cta_warps = plan->h[1].cta_warps = cta_warps;
    auto reject = [&](const std::string& w) {
        plan->ok = false;
        plan->why = w;
        return plan;
    };
    if (ndim != 2) return reject("stencil engine: 2-D layouts only");
    if (cta_warps == 0 || cta_warps > 32) return reject("stencil engine: bad CTA size");
    if (n > 0x7fffffffull) return reject("stencil engine: more than 2^31 coefficients");
    const uint32_t nb = static_cast<uint32_t>(bands.size());
    if (nb > 255) return reject("stencil engine: too many bands");
    for (const auto& b : bands) {
        const uint64_t h = b.shape[0], w = b.shape[1];
        if (!h || !w || (h & (h - 1)) || (w & (w - 1))) return reject("stencil engine: band shapes must be powers of two");
    }
    std::vector<RecIn> rin;
    for (size_t g = 0; g < gblock.size(); ++g) {
        RecIn r{};
        r.block = gblock[g];
        r.o = gblock[g] / nb;
        r.i = gblock[g] % nb;
        if (r.o >= nb) return reject("stencil engine: block out of range");
        const wbx_band& bo = bands[r.o];
        const wbx_band& bi = bands[r.i];
        const bool in_finer = bi.level <= bo.level;
        const wbx_band& large = in_finer ? bi : bo;
        const wbx_band& small = in_finer ? bo : bi;
        r.v0 = gidx[g] / large.shape[1];
        r.v1 = gidx[g] % large.shape[1];
        r.vs0 = r.v0 < large.shape[0] / 2 ? static_cast<int64_t>(r.v0) : static_cast<int64_t>(r.v0) - static_cast<int64_t>(large.shape[0]);
        r.vs1 = r.v1 < large.shape[1] / 2 ? static_cast<int64_t>(r.v1) : static_cast<int64_t>(r.v1) - static_cast<int64_t>(large.shape[1]);
        r.count = gcount[g];
        r.full = small.shape[0] * small.shape[1];
        r.val = gval[g];
        if (r.count > r.full || r.count > 0x7fffffffull) return reject("stencil engine: bad record count");
        rin.push_back(r);
    }
    std::vector<PBand> pb[2];
    // ---- 1. per phase: output bands, blocks, windows, taps, parts
    for (int ph = 0; ph < 2; ++ph) {
        StHostPhase& H = plan->h[ph];
        std::vector<std::vector<uint32_t>> blocks_of_band(nb);
        std::vector<std::vector<std::vector<size_t>>> recs_of(nb);
        for (size_t g = 0; g < rin.size(); ++g) {
            const RecIn& r = rin[g];
            const uint32_t out = ph == 0 ? r.o : r.i;
            auto& bl = blocks_of_band[out];
            auto it = std::find(bl.begin(), bl.end(), r.block);
            size_t k;
            if (it == bl.end()) {
                bl.push_back(r.block);
                recs_of[out].emplace_back();
                k = bl.size() - 1;
            } else {
                k = static_cast<size_t>(it - bl.begin());
            }
            recs_of[out][k].push_back(g);
        }
        for (uint32_t B = 0; B < nb; ++B) {
            if (blocks_of_band[B].empty()) continue;
            const wbx_band& ob = bands[B];
            const uint32_t l0 = lg2(ob.shape[0]), l1 = lg2(ob.shape[1]);
            PBand band{};
            band.band = B;
            uint32_t smax = 0;
            double taps = 0.0;
            for (size_t k = 0; k < blocks_of_band[B].size(); ++k) {
                const RecIn& r0 = rin[recs_of[B][k][0]];
                const bool in_finer = bands[r0.i].level <= bands[r0.o].level;
                PBlock b{};
                b.up = ph == 0 ? !in_finer : in_finer;
                b.s = static_cast<uint32_t>(std::abs(static_cast<int>(bands[r0.o].level) - static_cast<int>(bands[r0.i].level)));
                if (b.s > static_cast<uint32_t>(kStMaxScale)) return reject("stencil engine: band scale above 4");
                b.src = ph == 0 ? r0.i : r0.o;
                b.taps = static_cast<double>(recs_of[B][k].size()) / (b.up ? static_cast<double>(1u << (2 * b.s)) : 1.0);
                if (b.up) smax = std::max(smax, b.s);
                taps += b.taps;
                band.blocks.push_back(std::move(b));
            }
            // parts per output and tile shape; every half warp must lie in one residue class
            const uint32_t M = 1u << smax;
            uint32_t P = 1;
            while (taps / P > kTapsPerThread && P < static_cast<uint32_t>(kStMaxParts) && kStThreads / (2 * P) >= 16 * M * M) P *= 2;
            const uint64_t band_px = ob.shape[0] * ob.shape[1];
            while (static_cast<uint64_t>(kStThreads / P) > band_px && P < static_cast<uint32_t>(kStMaxParts)) P *= 2;
            const uint32_t npix = kStThreads / P;
            if (npix > band_px) return reject("stencil engine: band smaller than a tile");
            if (npix < 16 * M * M || ob.shape[0] < M || ob.shape[1] < M) return reject("stencil engine: tile smaller than its classes");
            uint32_t lnp = lg2(npix), lTW = std::min<uint32_t>(l1, std::min<uint32_t>(5, lnp)), lTH = lnp - lTW;
            while (lTH > l0) {
                --lTH;
                ++lTW;
            }
            if (lTW > l1 || (1u << lTH) < M || (1u << lTW) < M) return reject("stencil engine: no tile shape");
            const uint32_t TH = 1u << lTH, TW = 1u << lTW;
            StBand sb{};
            sb.out_off = static_cast<uint32_t>(ob.offset);
            sb.l0 = static_cast<uint8_t>(l0);
            sb.l1 = static_cast<uint8_t>(l1);
            sb.lTH = static_cast<uint8_t>(lTH);
            sb.lTW = static_cast<uint8_t>(lTW);
            sb.P = static_cast<uint8_t>(P);
            sb.smax = static_cast<uint8_t>(smax);
            sb.band = static_cast<uint8_t>(B);
            const uint32_t nt1 = 1u << (l1 - lTW);
            uint32_t win = 0;
            for (size_t k = 0; k < band.blocks.size(); ++k) {
                PBlock& b = band.blocks[k];
                const auto& ids = recs_of[B][k];
                int64_t mn0 = INT64_MAX, mx0 = INT64_MIN, mn1 = INT64_MAX, mx1 = INT64_MIN;
                for (size_t g : ids) {
                    mn0 = std::min(mn0, rin[g].vs0);
                    mx0 = std::max(mx0, rin[g].vs0);
                    mn1 = std::min(mn1, rin[g].vs1);
                    mx1 = std::max(mx1, rin[g].vs1);
                }
                int64_t R0, R1;
                if (!b.up) {
                    b.c0 = mn0;
                    b.c1 = mn1;
                    R0 = ((static_cast<int64_t>(TH) - 1) << b.s) + (mx0 - mn0) + 1;
                    R1 = ((static_cast<int64_t>(TW) - 1) << b.s) + (mx1 - mn1) + 1;
                } else {
                    b.c0 = floor_shift(-mx0, b.s);
                    b.c1 = floor_shift(-mx1, b.s);
                    R0 = floor_shift(static_cast<int64_t>(TH) - 1 - mn0, b.s) - b.c0 + 1;
                    R1 = floor_shift(static_cast<int64_t>(TW) - 1 - mn1, b.s) - b.c1 + 1;
                }
                int64_t dmax = 0;  // largest alignment shift of a tile's window row start
                for (uint32_t t1 = 0; t1 < nt1; ++t1) dmax = std::max(dmax, pmod(win_base1(b, static_cast<int64_t>(t1) << lTW), 4));
                const int64_t R1p = up4(R1 + dmax);
                if (R0 <= 0 || R1 <= 0 || R0 > 4096 || R1p > 4096 || R0 * R1p > (1 << 20))
                    return reject("stencil engine: window too large");
                b.R0 = static_cast<uint32_t>(R0);
                b.R1 = static_cast<uint32_t>(R1);
                b.R1p = static_cast<uint32_t>(R1p);
                b.woff = win;
                win += b.R0 * b.R1p;
                const uint32_t ncls = b.up ? (1u << (2 * b.s)) : 1u;
                std::vector<std::vector<std::pair<StTap, StTapX>>> bycls(ncls);
                // record order within a class = the reference's walk order
                for (size_t g : ids) {
                    const RecIn& r = rin[g];
                    StTap t{};
                    StTapX x{};
                    t.val = static_cast<float>(r.val);
                    x.count = r.count < r.full ? static_cast<int32_t>(r.count) : -1;
                    uint32_t cls = 0;
                    if (!b.up) {
                        t.off = static_cast<int32_t>((r.vs0 - b.c0) * R1p + (r.vs1 - b.c1));
                    } else {
                        const uint32_t mask = (1u << b.s) - 1u;
                        const uint32_t k0 = static_cast<uint32_t>(r.v0) & mask, k1 = static_cast<uint32_t>(r.v1) & mask;
                        cls = (k0 << b.s) | k1;
                        const int64_t j0 = (r.vs0 - static_cast<int64_t>(k0)) >> b.s;
                        const int64_t j1 = (r.vs1 - static_cast<int64_t>(k1)) >> b.s;
                        x.j0 = static_cast<int16_t>(j0);
                        x.j1 = static_cast<int16_t>(j1);
                        t.off = static_cast<int32_t>(-j0 * R1p - j1);
                    }
                    bycls[cls].push_back({t, x});
                }
                for (uint32_t c = 0; c < ncls; ++c) {  // each class list contiguous in the phase's taps
                    const uint32_t lo = static_cast<uint32_t>(H.taps.size());
                    for (const auto& tx : bycls[c]) {
                        H.taps.push_back(tx.first);
                        H.tapx.push_back(tx.second);
                    }
                    b.cls.push_back({lo, static_cast<uint32_t>(H.taps.size())});
                }
            }
            if (H.taps.size() > 0xffffu) return reject("stencil engine: more than 65535 taps per phase");
            band.win = win;
            // parts: the band's taps (blocks in order) cut into P ranges of equal length; a cut
            // inside a block splits every class list of it at the same fraction
            const double per = taps / P;
            double start = 0.0;
            band.parts.assign(P, {});
            for (size_t k = 0; k < band.blocks.size(); ++k) {
                const PBlock& b = band.blocks[k];
                const double s0b = start, s1b = start + b.taps;
                start = s1b;
                for (uint32_t p = 0; p < P; ++p) {
                    const double lo = p * per, hi = p + 1 == P ? taps + 1.0 : (p + 1) * per;
                    const double s0 = std::max(lo, s0b), s1 = std::min(hi, s1b);
                    if (s1 <= s0) continue;
                    const double f0 = (s0 - s0b) / b.taps, f1 = (s1 - s0b) / b.taps;
                    PJob j{static_cast<uint32_t>(k), {}};
                    bool any = false;
                    for (const auto& cr : b.cls) {
                        const double len = static_cast<double>(cr.second - cr.first);
                        const uint32_t a = f0 <= 0.0 ? 0u : static_cast<uint32_t>(std::min(len, std::floor(len * f0 + 0.5)));
                        const uint32_t e = f1 >= 1.0 ? static_cast<uint32_t>(len) : static_cast<uint32_t>(std::min(len, std::floor(len * f1 + 0.5)));
                        j.cls.push_back({cr.first + a, cr.first + std::max(a, e)});
                        any |= e > a;
                    }
                    if (any) band.parts[p].push_back(std::move(j));
                }
            }
            // per-thread cost model of a tile: the longest part's taps + entries + its window rows
            double worst = 0.0;
            for (uint32_t p = 0; p < P; ++p) {
                double t = 0.0;
                for (const PJob& j : band.parts[p]) {
                    double len = 0.0;
                    for (const auto& cr : j.cls) len += static_cast<double>(cr.second - cr.first);
                    t += 3.0 * len / static_cast<double>(j.cls.size()) + 12.0;
                }
                worst = std::max(worst, t);
            }
            double rows = 0.0;
            for (const PBlock& b : band.blocks) rows += b.R0;
            band.work = worst + 2.0 * rows / kStThreads + 4.0 * P + 24.0;
            H.bands.push_back(sb);
            pb[ph].push_back(std::move(band));
        }
        if (H.bands.size() > 255) return reject("stencil engine: too many output bands");
    }
    // ---- 2. source bands: rows of 16-byte multiples (a window row is one or more aligned copies)
    for (int ph = 0; ph < 2; ++ph)
        for (const PBand& band : pb[ph])
            for (const PBlock& b : band.blocks)
                if (bands[b.src].shape[1] % 4 != 0) return reject("stencil engine: source band narrower than 4 columns");
    // ---- 3. tiles -> CTAs and each CTA's tables
    for (int ph = 0; ph < 2; ++ph) {
        StHostPhase& H = plan->h[ph];
        // cost model (warp cycles): an entry ~ 3 per tap of its longer half + 16; a tile ~ its
        // entries spread over the CTA's warps + its window rows + its part sums
        std::vector<double> tile_cost(H.bands.size(), 0.0);
        for (uint32_t bi = 0; bi < H.bands.size(); ++bi) {
            const StBand& sb = H.bands[bi];
            const PBand& band = pb[ph][bi];
            const uint32_t lnp = sb.lTH + sb.lTW, npix = 1u << lnp;
            double c = 0.0, rows = 0.0;
            for (uint32_t w = 0; w < static_cast<uint32_t>(kStSlots); ++w) {
                const uint32_t part = (w * 32u) >> lnp, e0 = (w * 32u) & (npix - 1u);
                for (const PJob& j : band.parts[part]) {
                    const PBlock& b = band.blocks[j.blk];
                    double mx = 0.0;
                    for (uint32_t h = 0; h < 2; ++h) {
                        uint32_t q0, q1;
                        st_output(sb, 0, 0, e0 + 16 * h, q0, q1);
                        const uint32_t mask = (1u << b.s) - 1u;
                        const uint32_t cls = b.up ? (((q0 & mask) << b.s) | (q1 & mask)) : 0u;
                        mx = std::max(mx, static_cast<double>(j.cls[cls].second - j.cls[cls].first));
                    }
                    c += 3.0 * mx + 16.0;
                }
            }
            for (const PBlock& b : band.blocks) rows += b.R0;
            tile_cost[bi] = c / cta_warps + 2.0 * rows / cta_warps + 6.0 * npix * sb.P / (32.0 * cta_warps);
        }
        struct Work {
            double w;
            uint32_t band, t0, t1;
        };
        std::vector<Work> work;
        for (uint32_t bi = 0; bi < H.bands.size(); ++bi) {
            const StBand& sb = H.bands[bi];
            for (uint32_t t0 = 0; t0 < (1u << (sb.l0 - sb.lTH)); ++t0)
                for (uint32_t t1 = 0; t1 < (1u << (sb.l1 - sb.lTW)); ++t1) work.push_back({tile_cost[bi], bi, t0, t1});
        }
        std::stable_sort(work.begin(), work.end(), [](const Work& a, const Work& b) { return a.w > b.w; });
        using Slot = std::pair<double, uint32_t>;
        std::priority_queue<Slot, std::vector<Slot>, std::greater<Slot>> pq;
        for (uint32_t b = 0; b < G; ++b) pq.push({0.0, b});
        std::vector<std::vector<const Work*>> per(G);
        std::vector<double> load(G, 0.0);
        for (const Work& w : work) {
            Slot sl = pq.top();
            pq.pop();
            per[sl.second].push_back(&w);
            sl.first += w.w;
            load[sl.second] = sl.first;
            pq.push(sl);
        }
        H.work_max = *std::max_element(load.begin(), load.end());
        H.work_mean = std::accumulate(load.begin(), load.end(), 0.0) / G;
        H.task_off.assign(G + 1, 0);
        H.seg_off.assign(G + 1, 0);
        H.out_off.assign(G + 1, 0);
        H.ent_off.assign(static_cast<size_t>(G) * cta_warps + 1, 0);
        H.win_bytes.assign(G, 0);
        for (uint32_t cta = 0; cta < G; ++cta) {
            if (per[cta].size() > 255) return reject("stencil engine: more than 255 tiles per CTA");
            std::sort(per[cta].begin(), per[cta].end(), [](const Work* a, const Work* b) {
                return std::make_tuple(a->band, a->t0, a->t1) < std::make_tuple(b->band, b->t0, b->t1);
            });
            uint32_t wbase = 0;
            std::vector<StEntry> canon;  // the CTA's entries in canonical order (task, slot, job) = red rows
            std::vector<double> ecost;
            for (size_t t = 0; t < per[cta].size(); ++t) {
                const Work& w = *per[cta][t];
                const StBand& sb = H.bands[w.band];
                const PBand& band = pb[ph][w.band];
                H.tasks.push_back(StTask{static_cast<uint16_t>(w.band), static_cast<uint16_t>(w.t0), static_cast<uint16_t>(w.t1), 0});
                const uint32_t a0 = w.t0 << sb.lTH, a1 = w.t1 << sb.lTW;
                std::vector<int64_t> delta(band.blocks.size());
                for (size_t k = 0; k < band.blocks.size(); ++k) {
                    const PBlock& b = band.blocks[k];
                    const wbx_band& sbnd = bands[b.src];
                    const int64_t S0 = static_cast<int64_t>(sbnd.shape[0]), S1 = static_cast<int64_t>(sbnd.shape[1]);
                    const int64_t b0 = win_base0(b, a0), b1 = win_base1(b, a1);
                    delta[k] = pmod(b1, 4);
                    for (uint32_t r = 0; r < b.R0; ++r) {
                        const int64_t p0 = pmod(b0 + r, S0);
                        int64_t c = pmod(b1 - delta[k], S1);  // a multiple of 4, as S1 is
                        for (uint32_t done = 0; done < b.R1p;) {  // wrapped pieces, 16-byte multiples
                            const uint32_t len = static_cast<uint32_t>(std::min<int64_t>(b.R1p - done, S1 - c));
                            H.segs.push_back(StSeg{static_cast<uint32_t>(sbnd.offset + p0 * S1 + c),
                                                   wbase + b.woff + r * b.R1p + done, len * 4u});
                            H.win_bytes[cta] += len * 4u;
                            done += len;
                            c = 0;
                        }
                    }
                }
                // entries: one per (warp slot of the tile, job of the slot's part)
                const uint32_t lnp = sb.lTH + sb.lTW, npix = 1u << lnp;
                for (uint32_t wp = 0; wp < static_cast<uint32_t>(kStSlots); ++wp) {
                    const uint32_t part = (wp * 32u) >> lnp;
                    const uint32_t e0 = (wp * 32u) & (npix - 1u);
                    const uint32_t beg = static_cast<uint32_t>(canon.size());
                    for (const PJob& j : band.parts[part]) {
                        const PBlock& b = band.blocks[j.blk];
                        StEntry en{};
                        en.task = static_cast<uint8_t>(t);
                        en.slot = static_cast<uint8_t>(wp);
                        en.row = static_cast<uint16_t>(canon.size());
                        en.job_up = b.up ? 1 : 0;
                        en.job_s = static_cast<uint8_t>(b.s);
                        en.job_sl = static_cast<uint8_t>((lg2(bands[b.src].shape[0]) << 4) | lg2(bands[b.src].shape[1]));
                        const uint32_t cs = b.up ? sb.smax - b.s : sb.smax + b.s;
                        const int64_t rstride = static_cast<int64_t>(b.R1p) << cs;
                        if (rstride > 65535) return reject("stencil engine: window row stride too large");
                        en.rstride = static_cast<uint16_t>(rstride);
                        en.cshift = static_cast<uint8_t>(cs);
                        double mx = 0.0;
                        for (uint32_t h = 0; h < 2; ++h) {
                            uint32_t cls0 = 0;
                            for (uint32_t l = 16 * h; l < 16 * h + 16; ++l) {
                                const uint32_t e = e0 + l;
                                uint32_t q0, q1, kr, kc;
                                st_output(sb, a0, a1, e, q0, q1);
                                st_kpos(sb, e, kr, kc);
                                const uint32_t mask = (1u << b.s) - 1u;
                                const uint32_t cls = b.up ? (((q0 & mask) << b.s) | (q1 & mask)) : 0u;
                                const int64_t tb = static_cast<int64_t>(wbase + b.woff) + tap_base(b, a0, a1, q0, q1, delta[j.blk]);
                                const int64_t lane_part = static_cast<int64_t>(kr) * rstride + (static_cast<int64_t>(kc) << cs);
                                if (l == 16 * h) {
                                    cls0 = cls;
                                    en.base[h] = static_cast<int32_t>(tb - lane_part);
                                    en.rng[h] = j.cls[cls].first | (j.cls[cls].second << 16);
                                } else if (cls != cls0 || tb - lane_part != en.base[h]) {
                                    return reject("stencil engine: a half warp spans two classes");
                                }
                            }
                            for (uint32_t r = en.rng[h] & 0xffffu; r < (en.rng[h] >> 16); ++r)
                                if (H.tapx[r].count >= 0) en.flags |= kStPartial;
                            mx = std::max(mx, static_cast<double>((en.rng[h] >> 16) - (en.rng[h] & 0xffffu)));
                        }
                        canon.push_back(en);
                        ecost.push_back(3.0 * mx + 16.0);
                    }
                    H.grp.push_back(beg | (static_cast<uint32_t>(canon.size()) << 16));
                }
                for (uint32_t e = 0; e < npix; ++e) {
                    uint32_t q0, q1;
                    st_output(sb, a0, a1, e, q0, q1);
                    H.outs.push_back(StOut{sb.out_off + (q0 << sb.l1) + q1, static_cast<uint16_t>(e), static_cast<uint8_t>(t), sb.P,
                                           static_cast<uint8_t>(lnp), {0, 0, 0}});
                }
                wbase += band.win;
            }
            if (canon.size() > 0xffffu) return reject("stencil engine: too many entries per CTA");
            // entries -> warps: longest first to the least loaded warp; each warp's list in
            // canonical order (tile / slot locality)
            std::vector<size_t> order(canon.size());
            std::iota(order.begin(), order.end(), 0);
            std::stable_sort(order.begin(), order.end(), [&](size_t x, size_t y) { return ecost[x] > ecost[y]; });
            std::vector<std::vector<size_t>> wl(cta_warps);
            std::vector<double> wload(cta_warps, 0.0);
            for (size_t k : order) {
                const size_t wmin = static_cast<size_t>(std::min_element(wload.begin(), wload.end()) - wload.begin());
                wl[wmin].push_back(k);
                wload[wmin] += ecost[k];
            }
            for (uint32_t wp = 0; wp < cta_warps; ++wp) {
                std::sort(wl[wp].begin(), wl[wp].end());
                for (size_t k : wl[wp]) H.ents.push_back(canon[k]);
                H.ent_off[static_cast<size_t>(cta) * cta_warps + wp + 1] = static_cast<uint32_t>(H.ents.size());
                H.max_ents = std::max<uint32_t>(H.max_ents, static_cast<uint32_t>(wl[wp].size()));
            }
            H.max_rows = std::max<uint32_t>(H.max_rows, static_cast<uint32_t>(canon.size()));
            H.task_off[cta + 1] = static_cast<uint32_t>(H.tasks.size());
            H.seg_off[cta + 1] = static_cast<uint32_t>(H.segs.size());
            H.out_off[cta + 1] = static_cast<uint32_t>(H.outs.size());
            H.max_tasks = std::max<uint32_t>(H.max_tasks, H.task_off[cta + 1] - H.task_off[cta]);
            H.max_segs = std::max<uint32_t>(H.max_segs, H.seg_off[cta + 1] - H.seg_off[cta]);
            H.max_outs = std::max<uint32_t>(H.max_outs, H.out_off[cta + 1] - H.out_off[cta]);
            H.max_win = std::max<uint32_t>(H.max_win, wbase);
        }
    }
    if (std::getenv("WBX_ST_DEBUG")) {
        for (int ph = 0; ph < 2; ++ph) {
            const StHostPhase& H = plan->h[ph];
            std::fprintf(stderr,
                         "phase %d: %zu bands %zu taps %zu tasks %zu entries; per CTA max tasks %u segs %u outs %u win %u; "
                         "per warp max entries %u; work max/mean %.1f/%.1f\n",
                         ph, H.bands.size(), H.taps.size(), H.tasks.size(), H.ents.size(), H.max_tasks, H.max_segs,
                         H.max_outs, H.max_win, H.max_ents, H.work_max, H.work_mean);
            for (size_t bi = 0; bi < H.bands.size(); ++bi) {
                const StBand& b = H.bands[bi];
                std::fprintf(stderr, "  band off %u %ux%u tile %ux%u P %u smax %u win %u work %.1f\n", b.out_off, 1u << b.l0,
                             1u << b.l1, 1u << b.lTH, 1u << b.lTW, b.P, b.smax, pb[ph][bi].win, pb[ph][bi].work);
            }
        }
    }
    if (std::max(plan->h[0].max_win, plan->h[1].max_win) > smem_budget_floats)
        return reject("stencil engine: windows exceed shared memory");
    // coupled coordinates: the outputs of phase T (whole bands)
    plan->coupled.assign((n + 31) / 32, 0);
    for (const StBand& b : plan->h[1].bands) {
        const uint64_t cnt = 1ull << (b.l0 + b.l1);
        for (uint64_t k = 0; k < cnt; ++k) {
            const uint64_t i = b.out_off + k;
            plan->coupled[i >> 5] |= 1u << (i & 31);
        }
    }
    plan->ok = true;
    return plan;
}

bool stencil_plan_ok(const StencilPlan& p, std::string* why) {
    if (why) *why = p.why;
    return p.ok;
}

void upload_stencil_plan(StencilPlan& p, cudaStream_t st) {
    for (int ph = 0; ph < 2; ++ph) {
        const StHostPhase& H = p.h[ph];
        auto& D = p.d[ph];
        D.bands.upload(H.bands, st);
        D.taps.upload(H.taps, st);
        D.tapx.upload(H.tapx, st);
        D.task_off.upload(H.task_off, st);
        D.tasks.upload(H.tasks, st);
        D.seg_off.upload(H.seg_off, st);
        D.segs.upload(H.segs, st);
        D.ent_off.upload(H.ent_off, st);
        D.grp.upload(H.grp, st);
        D.ents.upload(H.ents, st);
        D.out_off.upload(H.out_off, st);
        D.outs.upload(H.outs, st);
        D.win_bytes.upload(H.win_bytes, st);
    }
    p.d_coupled.upload(p.coupled, st);
    WBX_CUDA(cudaStreamSynchronize(st));
}

StencilView view_of(const StencilPlan& p) {
    StencilView v{};
    for (int ph = 0; ph < 2; ++ph) {
        const StHostPhase& H = p.h[ph];
        const auto& D = p.d[ph];
        StPhaseView& V = v.ph[ph];
        V.bands = D.bands.p;
        V.taps = D.taps.p;
        V.tapx = D.tapx.p;
        V.task_off = D.task_off.p;
        V.tasks = D.tasks.p;
        V.seg_off = D.seg_off.p;
        V.segs = D.segs.p;
        V.ent_off = D.ent_off.p;
        V.grp = D.grp.p;
        V.ents = D.ents.p;
        V.out_off = D.out_off.p;
        V.outs = D.outs.p;
        V.win_bytes = D.win_bytes.p;
        V.nbands = static_cast<uint32_t>(H.bands.size());
        V.ntaps = static_cast<uint32_t>(H.taps.size());
        V.max_tasks = H.max_tasks;
        V.max_segs = H.max_segs;
        V.max_ents = H.max_ents;
        V.max_outs = H.max_outs;
        V.max_win = H.max_win;
        V.max_rows = H.max_rows;
        V.cta_warps = H.cta_warps;
    }
    v.coupled = p.d_coupled.p;
    return v;
}

std::shared_ptr<StencilPlan> stencil_plan_for(const wbx_op* op, uint32_t G, uint32_t cta_warps, cudaStream_t st) {
    std::lock_guard<std::mutex> g(op->win_mu);
    const uint64_t key = (static_cast<uint64_t>(cta_warps) << 32) | G;
    auto it = op->st_cache.find(key);
    if (it != op->st_cache.end()) return it->second;
    std::shared_ptr<StencilPlan> p;
    if (!op->has_gens) {
        p = std::make_shared<StencilPlan>();
        p->why = "stencil engine: no generator groups attached";
    } else {
        p = build_stencil_plan(op->g_bands, op->g_ndim, op->n, op->g_block, op->g_index, op->g_count, op->g_val, G,
                               cta_warps, 1u << 30);
        if (p->ok) upload_stencil_plan(*p, st);
    }
    op->st_cache[key] = p;
    return p;
}

// Host execution of one phase of the plan, CTA by CTA, through the kernel's tables: the window
// row copies, the warp entries per lane, the part sums in order and
// the output list; out = the phase's product of src (natural layout), in double.
void stencil_apply_host(const StencilPlan& p, int ph, const double* src, double* out) {
    const StHostPhase& H = p.h[ph];
    std::vector<double> win, red;
    for (uint32_t cta = 0; cta < p.G; ++cta) {
        win.assign(static_cast<size_t>(H.max_win) + 4, std::nan(""));
        for (uint32_t k = H.seg_off[cta]; k < H.seg_off[cta + 1]; ++k)
            for (uint32_t e = 0; e < H.segs[k].bytes / 4; ++e) win[H.segs[k].dst + e] = src[H.segs[k].src + e];
        const uint32_t W = H.cta_warps;
        const uint32_t nrows = H.ent_off[static_cast<size_t>(cta + 1) * W] - H.ent_off[static_cast<size_t>(cta) * W];
        red.assign(static_cast<size_t>(nrows) * 32, std::nan(""));
        for (size_t k = H.ent_off[static_cast<size_t>(cta) * W]; k < H.ent_off[static_cast<size_t>(cta + 1) * W]; ++k) {
            const StEntry& en = H.ents[k];
            const StTask& tk = H.tasks[H.task_off[cta] + en.task];
            const StBand& b = H.bands[tk.band];
            const uint32_t lnp = b.lTH + b.lTW;
            for (uint32_t lane = 0; lane < 32; ++lane) {
                const uint32_t e = (en.slot * 32u + lane) & ((1u << lnp) - 1u);
                uint32_t kr, kc;
                st_kpos(b, e, kr, kc);
                const uint32_t h = lane >> 4;
                const int64_t base = en.base[h] + static_cast<int64_t>(kr) * en.rstride + (static_cast<int64_t>(kc) << en.cshift);
                double acc = 0.0;
                for (uint32_t r = en.rng[h] & 0xffffu; r < (en.rng[h] >> 16); ++r) {
                    const StTap& T = H.taps[r];
                    const StTapX& X = H.tapx[r];
                    if ((en.flags & kStPartial) && X.count >= 0) {
                        uint32_t q0, q1;
                        st_output(b, static_cast<uint32_t>(tk.t0) << b.lTH, static_cast<uint32_t>(tk.t1) << b.lTW, e, q0, q1);
                        int64_t flat;
                        if (!en.job_up) {
                            flat = (static_cast<int64_t>(q0) << b.l1) + q1;
                        } else {
                            const int64_t sl0 = en.job_sl >> 4, sl1 = en.job_sl & 15;
                            flat = (((static_cast<int64_t>(q0 >> en.job_s) - X.j0) & ((1ll << sl0) - 1)) << sl1) +
                                   ((static_cast<int64_t>(q1 >> en.job_s) - X.j1) & ((1ll << sl1) - 1));
                        }
                        if (flat >= X.count) continue;
                    }
                    acc += static_cast<double>(T.val) * win[static_cast<size_t>(base + T.off)];
                }
                red[static_cast<size_t>(en.row) * 32 + lane] = acc;
            }
        }
        for (uint32_t k = H.out_off[cta]; k < H.out_off[cta + 1]; ++k) {
            const StOut& o = H.outs[k];
            double total = 0.0;
            for (uint32_t q = 0; q < o.P; ++q) {
                const uint32_t x = (q << o.lnp) + o.e;
                const uint32_t g = H.grp[(static_cast<size_t>(H.task_off[cta]) + o.task) * kStSlots + (x >> 5)];
                for (uint32_t r = g & 0xffffu; r < (g >> 16); ++r) total += red[static_cast<size_t>(r) * 32 + (x & 31u)];
            }
            out[o.idx] = total;
        }
    }
}

}  // namespace wbx

extern "C" {

// Attach the kept generator groups of a stationary Theta_K to its operator (they must expand
// to the operator's CSR exactly): lets the solver run the stencil engine.
int wbx_op_set_generators(wbx_op* op, uint32_t ndim, const uint64_t* dims, uint32_t J, uint64_t n_gens,
                          const uint32_t* blocks, const uint32_t* gen_index, const uint64_t* counts,
                          const double* values) {
    using namespace wbx;
    try {
        if (!op || !dims || (n_gens && (!blocks || !gen_index || !counts || !values)))
            fail(WBX_INVALID_ARGUMENT, "null argument to wbx_op_set_generators");
        std::vector<wbx_band> bands;
        make_layout(ndim, dims, J, bands);
        const uint64_t n = dims[0] * (ndim == 2 ? dims[1] : 1);
        if (n != op->n) fail(WBX_SHAPE_MISMATCH, "generator layout and operator sizes differ");
        const uint64_t nb = bands.size();
        for (uint64_t g = 0; g < n_gens; ++g)
            if (blocks[g] >= nb * nb) fail(WBX_BAND_NOT_FOUND, "block index out of range");
        HostCsr csr = expand_generators(bands, ndim, n, n_gens, blocks, gen_index, counts, values);
        if (csr.rowptr != op->h_rowptr || csr.col != op->h_col || csr.val != op->h_val)
            fail(WBX_BAD_SPEC, "generator groups do not expand to the operator's CSR");
        wbx::pgd_purge(nullptr, op);  // cached wbx_pgd solvers chose engines without the generators
        std::lock_guard<std::mutex> g(op->win_mu);
        op->has_gens = true;
        op->g_ndim = ndim;
        op->g_bands = bands;
        op->g_block.assign(blocks, blocks + n_gens);
        op->g_index.assign(gen_index, gen_index + n_gens);
        op->g_count.assign(counts, counts + n_gens);
        op->g_val.assign(values, values + n_gens);
        op->st_cache.clear();
        op->has_layout = true;  // the generators' layout is the operator's
        op->l_ndim = ndim;
        op->l_J = J;
        op->l_dims[0] = dims[0];
        op->l_dims[1] = ndim == 2 ? dims[1] : 1;
        op->l_bands = bands;
        op->circ_cache.clear();
        return WBX_OK;
    } catch (const wbx::Error& e) {
        wbx_set_last_error(e.what());
        return e.status;
    }
}

// Host execution of the stencil engine's plan for grid G (diagnostics / tests; no GPU needed):
// y = Theta x (phase 0) or Theta^T x (phase 1) for the operator given by its kept generator
// groups, over full-length fp64 vectors; outputs outside the phase's output bands are left
// untouched. WBX_BAD_SPEC with the reason when the plan does not apply.
int wbx_diag_stencil_apply_host(uint32_t ndim, const uint64_t* dims, uint32_t J, uint64_t n_gens,
                                const uint32_t* blocks, const uint32_t* gen_index, const uint64_t* counts,
                                const double* values, int phase, uint32_t G, const double* x, double* y) {
    using namespace wbx;
    try {
        if (!dims || !x || !y || phase < 0 || phase > 1 || G == 0) fail(WBX_INVALID_ARGUMENT, "bad arguments");
        std::vector<wbx_band> bands;
        make_layout(ndim, dims, J, bands);
        const uint64_t n = dims[0] * (ndim == 2 ? dims[1] : 1);
        auto plan = build_stencil_plan(bands, ndim, n, std::vector<uint32_t>(blocks, blocks + n_gens),
                                       std::vector<uint32_t>(gen_index, gen_index + n_gens),
                                       std::vector<uint64_t>(counts, counts + n_gens),
                                       std::vector<double>(values, values + n_gens), G, 16, 1u << 30);
        std::string why;
        if (!stencil_plan_ok(*plan, &why)) fail(WBX_BAD_SPEC, why);
        stencil_apply_host(*plan, phase, x, y);
        return WBX_OK;
    } catch (const wbx::Error& e) {
        wbx_set_last_error(e.what());
        return e.status;
    }
}

}  // extern "C"
