// The stencil engine (stationary operators): plan structures shared by the host planner
// (stencil_plan.cu) and the persistent FISTA kernel (stencil_kernel.cuh).
//
// A stationary Theta_K is the reference's kept generator groups (theta.cpp:236-275): a record
// (block = (out band o, in band i), generator offset v in the finer band of the pair, count c,
// value g) stands for the entries (small band position p, large band position
// q = (v + (p << s)) mod S_large) of the first c positions p (row-major) of the smaller band,
// s = |level_o - level_i|. So a product needs no index stream: every entry is an affine
// function of its output position. Per phase the engine sees each block as
//   DOWN: the output band is the small one: out[p] += g * src[(v + (p << s)) mod S_src]
//   UP:   the output band is the large one: out[q] += g * src[(q - v) >> s] for q = v (mod 2^s)
// (phase A = Theta: in finer or equal -> DOWN, coarser -> UP; phase T = Theta^T: in finer or
// equal -> UP, coarser -> DOWN).
//
// Data layout. Vectors stay in the natural band layout (fp32 y and residual): a window row of
// a tile is one or two (wrapped) 16-byte aligned bulk copies, as every source band has a row
// width that is a multiple of 4 floats and a window row starts at a multiple of 4 (the
// offset delta of its first useful column is folded into the lane bases).
//
// Work. Outputs are cut into tiles (a band's tiles share one shape); a CTA owns a fixed set of
// tiles per phase. Per phase it bulk-copies the windows of all its tiles (one per contributing
// block and tile) into shared memory (one mbarrier, one round trip), then every warp runs its
// precomputed entry list: an entry = one block's tap range for the warp's 32 outputs of one
// tile (a part of them when an output's taps are split into P parts): per lane a window base
// base[half] + krow * rstride + (kcol << cshift) (krow, kcol: the lane's position in its
// residue class grid), per tap one shared load and one fma. UP blocks are class-split: the
// records with v = k (mod 2^s) serve the outputs q = k (mod 2^s); pixels are ordered
// class-major so each half warp shares one class.
#pragma once

#include <cstdint>

namespace wbx {

constexpr int kStMaxParts = 8;
constexpr int kStMaxScale = 2;                                    // 2^s x 2^s classes, s <= 2
constexpr int kStMaxClass = (1 << kStMaxScale) * (1 << kStMaxScale);

struct StTap {          // hot tap entry (8 B)
    int32_t off;        // window offset relative to the lane's base
    float val;
};
struct StTapX {         // partial-walk data of a tap (8 B)
    int32_t count;      // < 0: full walk; else only small-band positions with flat index < count
    int16_t j0, j1;     // UP: (v_signed - class) >> s per dim
};

struct StBand {                               // a (phase, output band): tiling
    uint32_t out_off;                         // offset of the output band (natural layout)
    uint8_t l0, l1;                           // log2 output band shape
    uint8_t lTH, lTW;                         // log2 tile shape
    uint8_t P;                                // thread parts per output (256 = P * tile pixels)
    uint8_t smax;                             // class-major output order modulus 2^smax
    uint8_t band;                             // layout band index
    uint8_t pad;
};

struct StTask {                               // one tile of a CTA
    uint16_t band, t0, t1, pad;               // phase band index, tile coordinates
};

struct StSeg {                                // one window row: a 16-byte aligned bulk copy
    uint32_t src, dst, bytes;                 // source float index, window float index
};

enum : uint8_t { kStPartial = 1 };

// One tap range (one block's share of a part) for the 32 outputs of one warp slot of a tile
// (28 B). Its 32 sums go to row `row` of the CTA's part-sum table; the entries of a CTA are
// spread over its warps by cost (any warp may run any entry).
struct StEntry {
    int32_t base[2];                          // lane window base per half warp (window floats)
    uint32_t rng[2];                          // tap range per half warp: lo | hi << 16
    uint16_t rstride;                         // window floats per class-grid row
    uint16_t row;                             // part-sum row (canonical entry index in the CTA)
    uint8_t cshift;                           // log2 window floats per class-grid column
    uint8_t flags;                            // kStPartial: some tap covers only `count` positions
    uint8_t task, slot;                       // the CTA's tile index, warp slot in the tile (0..7)
    uint8_t job_up, job_s, job_sl, pad;       // partial walks: UP, scale, log2 source band shape (l0 << 4 | l1)
};

struct StOut {                                // one output of a CTA (epilogue order)
    uint32_t idx;                             // natural coordinate
    uint16_t e;                               // pixel in its tile
    uint8_t task, P, lnp;                     // tile, parts, log2 tile pixels (part stride)
    uint8_t pad[3];
};

struct StPhaseView {
    const StBand* bands;
    const StTap* taps;
    const StTapX* tapx;
    const uint32_t* task_off;                 // [G + 1]
    const StTask* tasks;
    const uint32_t* seg_off;                  // [G + 1]
    const StSeg* segs;
    const uint32_t* ent_off;                  // [G * cta_warps + 1]: entries per (CTA, warp)
    const StEntry* ents;
    const uint32_t* grp;                      // per (task, warp slot): part-sum rows lo | hi << 16
    const uint32_t* out_off;                  // [G + 1]
    const StOut* outs;
    const uint32_t* win_bytes;                // [G]: bulk-copy bytes of the CTA's windows
    uint32_t nbands, ntaps;
    uint32_t max_tasks, max_segs, max_ents, max_outs, max_win, max_rows, cta_warps;
};

struct StencilView {
    StPhaseView ph[2];                        // 0: phase A (Theta), 1: phase T (Theta^T)
    const uint32_t* coupled;                  // bitmask over n: outputs of phase T
};

}  // namespace wbx
