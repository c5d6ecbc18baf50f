// Per-block "window" layout of one operator side (Theta rows R, or Theta^T rows C) for the
// persistent solver.
//
// The compacted rows are cut into one contiguous, nonzero-balanced range per CTA. Because
// rows are sorted by length and, within a length class, by position, a CTA's rows are a
// spatially coherent strip, and the vector entries they reference form a small set U_b
// (at 1024^2, 296 CTAs: <= 5k entries for ~10.6k nonzeros). Each phase the CTA gathers
// x[U_b] ONCE into shared memory (one coalesced, fully parallel round trip) and its rows
// then read the window with LDS through 16-bit local column indices, so the per-slice
// dependency chain no longer contains a global gather, and global loads drop ~4x.
//
// Slice records (segmented, segment-major lanes as in sell.cuh, <= 16 nonzeros per lane
// segment = 4 quads): [info: 32 x u32][vals: nq x 32 lanes x 4 fp32][cols: nq x 32 lanes x
// 4 u16] -> 6 bytes per nonzero.
#pragma once

#include <cstdint>

namespace wbx {

struct WinView {
    const uint32_t* u_off;   // [G+1] window offsets into u_idx
    const uint32_t* u_idx;   // window entries: positions in the source vector
    const uint32_t* s_off;   // [G+1] slice offsets of each CTA
    const uint64_t* s_rec;   // record offset (uint4 units) of each slice
    const uint32_t* s_meta;  // nq | lane stride m << 8
    const uint32_t* r_off;   // [G+1] first compacted row of each CTA (rows are contiguous)
    const uint4* rec;
    uint32_t max_u;          // largest window of any CTA
    uint32_t max_rows;       // most rows of any CTA (per-row state owned in shared memory)
};

}  // namespace wbx
