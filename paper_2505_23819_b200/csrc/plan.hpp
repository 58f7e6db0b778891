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
  int64_t sc;   // mxfp4 upcast: scale-index contribution (0 otherwise)
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
  int32_t tile_bytes;   // bytes per tile (smem per buffer, padding included)
  int32_t pad;          // 1: unswizzled + 16 B padding per 128 B (legacy heuristic, ablation)
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
  // fused mxfp4 dequantisation (NEXT #1): scale index (row-major [M][K/32])
  // contributions of the destination bits, split like the offsets above
  int32_t upcast;
  uint32_t sc_thr[LL_MAX_TBITS];
  uint32_t sc_vec[LL_MAX_VEC];
  uint32_t sc_e[16];              // byte e of a 16-byte destination vector
  int32_t sc_nz;                  // vector bits moving the scale (<= 2: 4-slot fast path)
  uint32_t sc_c[2];               // their scale-index contributions
  uint8_t sc_slot[16];            // slot (0..3) of byte e among the 4 loaded scales
  uint32_t sc_sel[16];            // prmt selector: bf16x2 factor of byte e's slot
  uint32_t sc_psel;               // prmt: slots of bytes e + 4 from those of bytes e
};

// Warp-shuffle conversion plan (LL_PATH_SHUFFLE): warp-local tiles exchanged
// with shfl.sync.  The payload is one 32-bit word; the
// load side first makes each word hold the same sub-word elements as on the
// store side (prmt swaps), so the exchange is word-granular.  Round k of the
// paper's 2^|R| rounds moves, for every lane l, the word
//   send  S[k] = R[alpha(k) ^ beta(l)]        from lane  gamma(k) ^ delta(l)
//   recv  Q[eps(k) ^ zeta(l)] = received word
// alpha and eps^{-1} are uniform linear maps of the word index, applied as a
// short list of elementary register operations (bit swaps / bit xors);
// beta(l), zeta(l) are lane-dependent XOR masks applied with selects.
#define LL_MAX_LINOPS 12
struct ShufflePlan {
  TileMap tile;
  int32_t n_swaps;
  int8_t swap_a[LL_MAX_SWAPS], swap_b[LL_MAX_SWAPS];   // sub-word swaps (as SmemPlan)
  uint32_t ld_thr[5], st_thr[5];                       // byte offsets per lane bit
  uint32_t ld_vec[LL_MAX_VEC], st_vec[LL_MAX_VEC];     // byte offsets per 16-B vector
  int32_t n_pre, n_post;                               // elementary ops (word-index bits)
  int8_t pre_op[LL_MAX_LINOPS], pre_a[LL_MAX_LINOPS], pre_b[LL_MAX_LINOPS];
  int8_t post_op[LL_MAX_LINOPS], post_a[LL_MAX_LINOPS], post_b[LL_MAX_LINOPS];
  uint32_t beta_lane[5], zeta_lane[5], delta_lane[5];  // per lane bit
  uint32_t beta_any, zeta_any;                         // OR of the masks (which bits can flip)
  uint8_t gamma[LL_MAX_GRAN];                          // per round: xor into the source lane
};

// TMA-fed smem path (LL_PATH_SMEM_TMA): the source tile is one box of a
// <= 5-D tensor view of the source buffer whose dims are runs of source index
// bits (dim i = element bits [shift[i], shift[i] + size_bits[i]), box =
// the low box_bits[i] of them; the top dim also carries the batch).  The box
// lands in shared memory densely (tile bits in ascending source order) and
// permuted by the hardware swizzle `swizzle` (0 none, 1/2/3 = 32/64/128 B:
// byte-address bits [4, 4+m) ^= bits [7, 7+m)).  The reader side reuses the
// SmemPlan fields (sr_thr / sr_gran / swaps / st_*).
struct TmaDesc {
  int32_t ndim;
  int32_t swizzle;
  int32_t shift[5];
  int32_t box_bits[5];
  int32_t size_bits[5];   // top dim: ignored (computed from the launch range)
};

// Register-faithful conversion plan (LL_PATH_REGS): threads ARE the layouts'
// lanes and warps (one CTA per block index), each thread holds its own
// registers (2^reg elements, contiguous in the buffers' hardware order), and
// the exchange goes registers -> shared memory (layout S, the paper's optimal
// swizzle) -> registers, as in the paper's in-kernel convert_layout.  Each
// side uses vectorised st/ld.shared or, when its layout is divisible by the
// tile id^{reg,offset}_k x id^{thread,offset}_2, stmatrix /
// ldmatrix (m8n8 b16 rows of 16 bytes).  Offsets are bytes, XOR-combined.
#define LL_REGS_MAX_INST 64
struct RegsPlan {
  int32_t nw;            // log2 warps per CTA
  int32_t nwords;        // 32-bit words per thread
  int64_t tile_bytes;    // bytes per CTA tile (= per block index)
  int64_t n_tiles;       // blocks x batch
  int32_t wr_mat, rd_mat;    // 1: stmatrix / ldmatrix; 0: st/ld.shared
  int32_t wr_gw, rd_gw;      // words per thread per instruction (1, 2, 4)
  int32_t n_swaps;           // load-side element-bit swaps (A's word order -> B's)
  int8_t swap_a[LL_MAX_SWAPS], swap_b[LL_MAX_SWAPS];
  // word-bit transpositions bringing each side's instruction words to word
  // bits 0 (and 1): applied to the source registers once before the exchange
  // (write side), and in reverse to the received registers (read side), so the
  // exchange itself has one fixed operand pattern
  int32_t n_wsw, n_rsw;
  int8_t wsw_a[4], wsw_b[4], rsw_a[4], rsw_b[4];
  uint32_t sw_thr[LL_MAX_TBITS], sr_thr[LL_MAX_TBITS];  // per lane / address-provider bit, warp bit
  uint32_t sw_inst[LL_REGS_MAX_INST], sr_inst[LL_REGS_MAX_INST];  // per instruction
};

// A contiguous range of tile indices [t0, t1) of a smem / shuffle plan, with
// the byte offsets of the caller's slices (multi-GPU shards: each rank holds
// only its slice of src and dst).
struct TileRange {
  int64_t t0, t1;
  int64_t src_shift, dst_shift;
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
