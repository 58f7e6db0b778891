// plan.hpp -- plan structures shared by the host planner and the sm_100a
// kernels.  Everything is plain data passed by value as __grid_constant__
// kernel parameters (no device allocation on the conversion path).
#pragma once

#include <cstdint>

#ifndef __CUDACC__
#define LL_HD
#else
#define LL_HD __host__ __device__
#endif

#define LL_MAX_VEC 16    // 16-byte global vectors per thread per side
#define LL_MAX_GRAN 64   // shared-memory granules per thread per side
#define LL_MAX_TBITS 8   // thread bits inside a tile group: 5 lane + <= 3 warp
#define LL_MAX_SWAPS 8

namespace ll {

// Tile index t -> byte offsets of the tile in src and dst.  t = inst * 2^n_bits
// + r; the bits of r (in the planner's tile order) each add a fixed offset.
// The planner tabulates r in chunks of LL_TAB_BITS bits (tab[k][v] = offsets
// of chunk k having value v); the tables live in the kernel parameters
// (constant bank) and are indexed warp-uniformly, so a tile costs n_tab
// constant loads and adds.
#define LL_MAX_OUTER 24
#define LL_TAB_BITS 8
#define LL_MAX_TAB 3
struct TileTab {
  int64_t src, dst;
};
struct TileMap {
  int64_t n_tiles;                               // tiles incl. batch
  int32_t n_bits;                                // outer bits per layout instance
  int32_t n_tab;                                 // ceil(n_bits / LL_TAB_BITS)
  int64_t batch_stride_src, batch_stride_dst;    // bytes per layout instance
  TileTab tab[LL_MAX_TAB][1 << LL_TAB_BITS];     // bytes
};

// Shared-memory conversion plan (LL_PATH_SMEM): a tile group of 2^gw warps
// loads a tile with coalesced 16-byte vectors in the planner's load layout,
// fixes the sub-word order with prmt where needed, stores granules to shared
// memory through the swizzled layout S (paper's optimal swizzling) -- the
// granule's words are picked at compile time from the word bits gsel_a/b --
// synchronises, loads granules in the store layout and writes coalesced
// 16-byte vectors.  All in-tile offsets are in BYTES (32-bit).
//
// Scheduling: grid-stride loop over tile indices (planner's tile order).
struct SmemPlan {
  TileMap tile;
  int32_t gw;           // log2 warps per tile group
  int32_t tile_bytes;   // bytes per tile (smem per buffer)
  int32_t n_swaps;      // sub-word register-bit swaps (prmt), swap_a < sub-word bits
  int8_t swap_a[LL_MAX_SWAPS], swap_b[LL_MAX_SWAPS];
  int8_t gsel_a, gsel_b;          // register word bits forming a write granule (-1: unused)
  uint32_t ld_thr[LL_MAX_TBITS];  // src byte offset per thread bit (lane 0-4, warp-in-group)
  uint32_t st_thr[LL_MAX_TBITS];  // dst byte offset per thread bit
  uint32_t ld_vec[LL_MAX_VEC];    // src byte offset of 16-B load u
  uint32_t st_vec[LL_MAX_VEC];    // dst byte offset of 16-B store u
  uint32_t sw_thr[LL_MAX_TBITS];  // smem byte offset (xor) per thread bit, write side
  uint32_t sr_thr[LL_MAX_TBITS];  // read side
  uint32_t sw_gran[LL_MAX_GRAN];  // smem byte offset (xor) of write granule j
  uint32_t sr_gran[LL_MAX_GRAN];  // read granule j
};

// Warp-shuffle conversion plan (LL_PATH_SHUFFLE), warp-local tiles.  Word-
// granular exchange (32-bit payload): per round k every lane sends
// word k of its (lane-permuted) register file and receives into word k; the
// lane-dependent parts are XOR masks on the word index.
struct ShufflePlan {
  TileMap tile;
  int32_t n_swaps_ld;
  int8_t swap_a[LL_MAX_SWAPS], swap_b[LL_MAX_SWAPS];   // load-side register-bit swaps
  int64_t ld_thr[5], st_thr[5];
  int64_t ld_vec[LL_MAX_VEC], st_vec[LL_MAX_VEC];
  // send side: word index of round k = k ^ send_xor(lane)
  int32_t send_lane_xor[5];        // per lane bit: xor into the send word index
  // source lane of round k for lane l = src_lane_base(l) ^ src_lane_round(k)
  int32_t srcl_lane[5];            // per lane bit
  int32_t srcl_round[LL_MAX_GRAN]; // per round (word index)
  // receive: word k received lands at word dst_word(k, lane) = k ^ recv_xor(lane) after
  // the final permutation given by the store-side word map
  int32_t recv_lane_xor[5];
  int32_t recv_perm[LL_MAX_GRAN];  // uniform word permutation after the exchange
  int32_t send_perm[LL_MAX_GRAN];  // uniform word permutation before the exchange
};

// Generic pull kernel (LL_PATH_GENERIC): dst[h] = src[X h] for every h.
struct GenericPlan {
  int64_t n_vec;           // number of destination 16-byte vectors (incl. batch)
  int32_t nB;              // dst index bits (per batch element)
  int32_t n_x;             // columns of X used (= nB)
  int64_t batch_stride_src, batch_stride_dst;
  int64_t x[64];           // X columns: src index of each dst index bit
};

// Gather plan: out[h] = src[(h ^ clear(h)) ^ Y(idx[h])], i.e. h with its axis
// coordinate replaced (bijective layouts; see planner).
struct GatherPlan {
  int64_t n_vec;           // 16-byte output vectors (incl. batch)
  int32_t nbits;           // buffer index bits per batch element
  int64_t batch_stride;
  int32_t ax_shift, ax_bits;       // axis field in the flat tensor index
  int64_t L[64];                   // layout columns (buffer bit -> tensor flat)
  int64_t Y[32];                   // buffer vector of each axis bit (L^{-1} e_axis_k)
  int32_t y_contig;                // Y_k = 1 << (y_base + k)
  int32_t y_base;
  int64_t axis_mask_buf;           // buffer bits carrying the axis (contiguous case)
  int32_t check;                   // bounds-check indices
  // shuffle path: the warp-local part (buffer bits < vb + 5)
  int32_t vb;                      // log2 elements per 16-byte vector
  int32_t cand_mask;               // register bits touched by Y (candidate shuffles)
};

}  // namespace ll
