// Per-block "window" layout of one operator side (Theta rows R, or Theta^T rows C) for the
// persistent solver.
//
// The compacted rows are cut into one contiguous, cost-balanced range per CTA. Because rows
// are sorted by length and, within a length class, by position, a CTA's rows are a
// spatially coherent strip, and the vector entries they reference form a small set U_b
// (at 1024^2, 296 CTAs: <= 4.3k entries). Each phase the CTA gathers x[U_b] ONCE into
// shared memory (one coalesced, fully parallel round trip) and its rows then read the
// window with LDS through 16-bit local column indices.
//
// Slices (segmented, segment-major lanes as in sell.cuh, <= 16 nonzeros per lane segment
// = 4 quads) hold `cnt` CONSECUTIVE rows of equal segment count q: lane = t*m + i holds
// segment t of row first_row + i, so no per-lane row word is stored.
//
// Values come in one of two formats, chosen per operator side:
//  * dictionary (kWinDict): the rows of a CTA have very few DISTINCT value sequences (a
//    stationary operator: rows of one band pair repeat the same generator values; at
//    1024^2 <= 26 per CTA, ~10 KB). Each distinct sequence is stored once per CTA as q
//    zero-padded 16-value segment blocks in shared memory (loaded once per solve); a slice
//    record then carries only a 16-bit dictionary offset per lane and the columns:
//    [pb: 32 x u16][cols: nq x 32 lanes x 4 u16] -> ~2 bytes per nonzero streamed.
//  * full: [vals: nq x 32 lanes x 4 fp32][cols: nq x 32 lanes x 4 u16] -> 6 bytes per
//    nonzero (used when some CTA's dictionary exceeds the shared-memory budget).
#pragma once

#include <cstdint>

namespace wbx {

constexpr uint32_t kWinDictBudget = 16384;  // bytes of dictionary per CTA and side

struct WinView {
    const uint32_t* u_off;   // [G+1] window offsets into u_idx
    const uint32_t* u_idx;   // window entries: positions in the source vector (chunk layout: the
                             // 16-byte chunk index)
    const uint16_t* u_slot;  // shared-memory slot of each window entry (bank-aware placement;
                             // chunk layout: chunk slot, the chunk fills window floats 4 slot ..)
    const uint32_t* s_off;   // [G+1] slice offsets of each CTA
    const uint4* s_tab;      // per slice {record offset (uint4), meta, first row, 0}
    const uint32_t* r_off;   // [G+1] first compacted row of each CTA (rows are contiguous)
    const uint32_t* d_off;   // [G+1] dictionary offsets (floats) of each CTA (dictionary format)
    const float* d_val;      // dictionaries: per CTA a zero block then q x 16-value blocks per sequence
    const uint4* rec;
    uint32_t max_u;          // most window entries of any CTA
    uint32_t max_win;        // largest window slot extent of any CTA (>= max_u)
    uint32_t max_rows;       // most rows of any CTA (per-row state owned in shared memory)
    uint32_t max_slices;     // most slices of any CTA
    uint32_t max_dict;       // largest dictionary of any CTA (floats; 0 = full format)
    uint32_t src_len;        // length of the vector the windows gather from (debug checks)
    uint32_t chunk;          // 1: chunk layout (fp32 sources; one 16-byte copy per chunk)
};

// slice meta word: nq (quads per lane) | m (lane stride) << 8 | q (segments per row) << 16 |
// cnt (rows) << 24
__host__ __device__ constexpr uint32_t win_meta(uint32_t nq, uint32_t m, uint32_t q, uint32_t cnt) {
    return nq | (m << 8) | (q << 16) | (cnt << 24);
}

}  // namespace wbx
