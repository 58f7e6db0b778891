// kernels.cu -- sm_100a kernels for layout conversion and gather.
//
// Pure data movement: no tensor cores (no dense contraction on this path).
// Every kernel is persistent-style (grid sized from the SM count, loop over
// work items) and moves HBM data with 128-bit coalesced loads / stores.
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>
#include <cstdlib>
#include <string>
#include <algorithm>

#include "kernels.hpp"
#include "plan.hpp"

namespace ll {

// ------------------------------------------------------------------ PTX helpers

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void stg_stream(void* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}

template <int G>
__device__ __forceinline__ void sts(uint32_t addr, const uint32_t* r) {
  if constexpr (G == 16)
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(r[0]), "r"(r[1]),
                 "r"(r[2]), "r"(r[3])
                 : "memory");
  else if constexpr (G == 8)
    asm volatile("st.shared.v2.b32 [%0], {%1,%2};" ::"r"(addr), "r"(r[0]), "r"(r[1]) : "memory");
  else
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(r[0]) : "memory");
}

template <int G>
__device__ __forceinline__ void lds(uint32_t addr, uint32_t* r) {
  if constexpr (G == 16)
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr)
                 : "memory");
  else if constexpr (G == 8)
    asm volatile("ld.shared.v2.b32 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(addr) : "memory");
  else
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(r[0]) : "r"(addr) : "memory");
}

__device__ __forceinline__ void group_sync(int gw, int group) {
  if (gw == 0) {
    __syncwarp();
  } else {
    // named barrier per tile group (id 0 is __syncthreads)
    asm volatile("bar.sync %0, %1;" ::"r"(group + 1), "r"(32 << gw) : "memory");
  }
}

__host__ __device__ constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x >> 1); }

// ----------------------------------------------------------- register-bit swaps
//
// The thread's register file R[] holds 2^r elements of W bytes in element
// order rho.  swap(a, b) exchanges element-index bits a < b.  Word-level
// bits are register renames; a sub-word bit against a word bit is a 2x2
// transpose with prmt (byte permute, the FlashAttention-3 trick of P:62).
// (a, b) are warp-uniform plan data; every case below is unrolled with
// compile-time register indices so R[] stays in registers.

template <int NW>
__device__ __forceinline__ void swap_word_bits(uint32_t (&R)[NW], int a, int b) {
  constexpr int LB = ilog2(NW);
#pragma unroll
  for (int A = 0; A < LB; ++A) {
#pragma unroll
    for (int B = A + 1; B < LB; ++B) {
      if (a == A && b == B) {
#pragma unroll
        for (int i = 0; i < NW; ++i) {
          if (((i >> A) & 1) == 0 && ((i >> B) & 1) == 1) {
            const int j = i ^ ((1 << A) | (1 << B));
            uint32_t t = R[i];
            R[i] = R[j];
            R[j] = t;
          }
        }
      }
    }
  }
}

template <int NW>
__device__ __forceinline__ void swap_sub_word(uint32_t (&R)[NW], int wb, uint32_t sel_lo,
                                              uint32_t sel_hi) {
  constexpr int LB = ilog2(NW);
#pragma unroll
  for (int B = 0; B < LB; ++B) {
    if (wb == B) {
#pragma unroll
      for (int i = 0; i < NW; ++i) {
        if (((i >> B) & 1) == 0) {
          const int j = i | (1 << B);
          uint32_t lo = prmt(R[i], R[j], sel_lo);
          uint32_t hi = prmt(R[i], R[j], sel_hi);
          R[i] = lo;
          R[j] = hi;
        }
      }
    }
  }
}

template <int W, int NW>
__device__ __forceinline__ void apply_swap(uint32_t (&R)[NW], int a, int b) {
  if constexpr (W == 8) {
    swap_word_bits<NW>(R, a + 1, b + 1);
  } else if constexpr (W == 4) {
    swap_word_bits<NW>(R, a, b);
  } else if constexpr (W == 2) {
    if (a == 0)
      swap_sub_word<NW>(R, b - 1, 0x5410u, 0x7632u);
    else
      swap_word_bits<NW>(R, a - 1, b - 1);
  } else {  // W == 1
    if (a == 0 && b == 1) {
#pragma unroll
      for (int i = 0; i < NW; ++i) R[i] = prmt(R[i], 0u, 0x3120u);
    } else if (a == 0) {
      swap_sub_word<NW>(R, b - 2, 0x6240u, 0x7351u);
    } else if (a == 1) {
      swap_sub_word<NW>(R, b - 2, 0x5410u, 0x7632u);
    } else {
      swap_word_bits<NW>(R, a - 2, b - 2);
    }
  }
}

// ------------------------------------------------------------- smem kernel

// ------------------------------------------------ compile-time granule selection
//
// A write granule is GW consecutive 32-bit words of shared memory.  Its words
// come from the register file R[NW] at word indices that deposit the
// granule-internal index k into word bits (A, B) and the granule number j
// into the remaining word bits (ascending).  (A, B) are plan data; every
// case is instantiated so the STS operands are compile-time registers.

__host__ __device__ constexpr int deposit_word(int j, int k, int LB, int A, int B) {
  int idx = 0, q = 0;
  for (int bit = 0; bit < LB; ++bit) {
    if (bit == A) {
      idx |= (k & 1) << bit;
    } else if (bit == B) {
      idx |= ((k >> 1) & 1) << bit;
    } else {
      idx |= ((j >> q) & 1) << bit;
      ++q;
    }
  }
  return idx;
}

// wbase: (region base + buffer); wx: the thread's xor offset; the swizzled
// offsets are combined by XOR *within* the region, then added to the base
// (the dynamic shared window need not be aligned to the tile size).
template <int NW, int GW, int A, int B, bool PAD = false>
__device__ __forceinline__ void sts_granules(const uint32_t (&R)[NW], uint32_t wbase, uint32_t wx,
                                             const uint32_t* gran) {
  constexpr int LB = ilog2(NW);
  constexpr int NG = NW / GW;
#pragma unroll
  for (int j = 0; j < NG; ++j) {
    uint32_t v[GW];
#pragma unroll
    for (int k = 0; k < GW; ++k) v[k] = R[deposit_word(j, k, LB, A, B)];
    const uint32_t o = wx ^ gran[j];
    sts<GW * 4>(wbase + (PAD ? o + ((o >> 7) << 4) : o), v);
  }
}

template <int NW, int GW, int A, int B, bool PAD>
__device__ __forceinline__ bool sts_try_b(int a, int b, const uint32_t (&R)[NW], uint32_t wbase,
                                          uint32_t wx, const uint32_t* gran) {
  constexpr int LB = ilog2(NW);
  if constexpr (B >= LB) {
    return false;
  } else {
    if constexpr (A != B) {
      if (a == A && b == B) {
        sts_granules<NW, GW, A, B, PAD>(R, wbase, wx, gran);
        return true;
      }
    }
    return sts_try_b<NW, GW, A, B + 1, PAD>(a, b, R, wbase, wx, gran);
  }
}

template <int NW, int GW, int A, bool PAD>
__device__ __forceinline__ bool sts_try_a(int a, int b, const uint32_t (&R)[NW], uint32_t wbase,
                                          uint32_t wx, const uint32_t* gran) {
  constexpr int LB = ilog2(NW);
  if constexpr (A >= LB) {
    return false;
  } else {
    bool done;
    if constexpr (GW == 2) {
      done = false;
      if (a == A) {
        sts_granules<NW, 2, A, -1, PAD>(R, wbase, wx, gran);
        done = true;
      }
    } else {
      done = sts_try_b<NW, GW, A, 0, PAD>(a, b, R, wbase, wx, gran);
    }
    if (done) return true;
    return sts_try_a<NW, GW, A + 1, PAD>(a, b, R, wbase, wx, gran);
  }
}

template <int NW, int GW, bool PAD = false>
__device__ __forceinline__ void sts_dispatch(int a, int b, const uint32_t (&R)[NW], uint32_t wbase,
                                             uint32_t wx, const uint32_t* gran) {
  if constexpr (GW == 1) {
    sts_granules<NW, 1, -1, -1, PAD>(R, wbase, wx, gran);
  } else {
    sts_try_a<NW, GW, 0, PAD>(a, b, R, wbase, wx, gran);
  }
}

// ------------------------------------------------------------- smem kernel
//
// W: element bytes; NV: 16-byte vectors per thread per side; G: granule
// bytes; PIPE: the loads of the group's next tile are issued right after the
// current tile's STS (before the exchange completes).
template <int NV>
__device__ __forceinline__ void load_tile(uint32_t (&R)[NV * 4], const uint8_t* sp,
                                          const uint32_t* ld_vec) {
#pragma unroll
  for (int u = 0; u < NV; ++u) {
    uint4 v = ldg_stream(sp + ld_vec[u]);
    R[4 * u + 0] = v.x;
    R[4 * u + 1] = v.y;
    R[4 * u + 2] = v.z;
    R[4 * u + 3] = v.w;
  }
}

// PAD: the legacy padding heuristic (ablation, LL_PATH_SMEM_PADDED): the
// staging offsets are unswizzled and 16 bytes of padding follow every 128 B.
__device__ __forceinline__ uint32_t pad_off(uint32_t o) { return o + ((o >> 7) << 4); }

template <int W, int NV, int G, bool PIPE, bool PAD>
__global__ void __launch_bounds__(256) convert_smem_kernel(const __grid_constant__ SmemPlan p,
                                                           const uint8_t* __restrict__ src,
                                                           uint8_t* __restrict__ dst,
                                                           int64_t n_groups, TileRange rg) {
  constexpr int NW = NV * 4;          // 32-bit words per thread
  constexpr int NG = NV * 16 / G;     // granules per thread
  constexpr int GW = G / 4;           // words per granule
  extern __shared__ __align__(16) uint8_t smem[];

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int gw = p.gw;
  const int group = warp >> gw;
  const int tb = lane | ((warp & ((1 << gw) - 1)) << 5);
  const int gpc = (blockDim.x >> 5) >> gw;
  const int tbits = 5 + gw;

  const int64_t gid = (int64_t)blockIdx.x * gpc + group;
  if (gid >= n_groups) return;  // idle group (whole warps: barriers stay consistent)

  uint32_t ld_off = 0, st_off = 0, swx = 0, srx = 0;
#pragma unroll
  for (int b = 0; b < LL_MAX_TBITS; ++b) {
    if (b < tbits && ((tb >> b) & 1)) {
      ld_off += p.ld_thr[b];
      st_off += p.st_thr[b];
      swx ^= p.sw_thr[b];
      srx ^= p.sr_thr[b];
    }
  }
  const uint8_t* sthr = src + ld_off - rg.src_shift;
  uint8_t* dthr = dst + st_off - rg.dst_shift;
  const int n_bits = p.tile.n_bits;
  const int n_tab = p.tile.n_tab;
  const int64_t rmask = (int64_t(1) << n_bits) - 1;
  auto tile_off = [&](int64_t t, int64_t& so, int64_t& dof) {
    const int64_t inst = t >> n_bits;
    const int64_t r = t & rmask;
    so = inst * p.tile.batch_stride_src;
    dof = inst * p.tile.batch_stride_dst;
#pragma unroll
    for (int k = 0; k < LL_MAX_TAB; ++k) {
      if (k < n_tab) {
        const TileTab& e = p.tile.tab[k][(int)((r >> (k * LL_TAB_BITS)) & ((1 << LL_TAB_BITS) - 1))];
        so += e.src;
        dof += e.dst;
      }
    }
  };

  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem) + group * 2 * p.tile_bytes;
  uint32_t buf = 0;
  const int ga = p.gsel_a, gb = p.gsel_b;
  const int64_t n_tiles = rg.t1;

  uint32_t R[NW];
  int64_t so, dof;
  int64_t t = rg.t0 + gid;
  if (PIPE && t < n_tiles) {
    tile_off(t, so, dof);
    load_tile<NV>(R, sthr + so, p.ld_vec);
  }
  for (; t < n_tiles; t += n_groups) {
    if (!PIPE) tile_off(t, so, dof);
    if (!PIPE) load_tile<NV>(R, sthr + so, p.ld_vec);
    const int64_t dcur = dof;
    for (int s = 0; s < p.n_swaps; ++s) apply_swap<W, NW>(R, p.swap_a[s], p.swap_b[s]);
    sts_dispatch<NW, GW, PAD>(ga, gb, R, sbase + buf, swx, p.sw_gran);
    if (PIPE) {
      const int64_t tn = t + n_groups;
      if (tn < n_tiles) {
        tile_off(tn, so, dof);
        load_tile<NV>(R, sthr + so, p.ld_vec);
      }
    }
    group_sync(gw, group);
    uint32_t Q[NW];
#pragma unroll
    for (int j = 0; j < NG; ++j) {
      const uint32_t o = srx ^ p.sr_gran[j];
      lds<G>(sbase + buf + (PAD ? pad_off(o) : o), &Q[j * GW]);
    }
    uint8_t* dp = dthr + dcur;
#pragma unroll
    for (int u = 0; u < NV; ++u)
      stg_stream(dp + p.st_vec[u], make_uint4(Q[4 * u + 0], Q[4 * u + 1], Q[4 * u + 2], Q[4 * u + 3]));
    buf ^= p.tile_bytes;
  }
}

// ------------------------------------------------------ cp.async smem kernel
//
// LL_PATH_SMEM_ASYNC: HBM -> shared memory by cp.async (16-byte source
// vectors written straight to their swizzled granule, no registers), NS
// tiles in flight per group; readers load 16-byte granules, fix the sub-word
// order with prmt and pick destination vectors at compile time.

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int NW, int A, int B>
__device__ __forceinline__ void stg_vectors(const uint32_t (&Q)[NW], uint8_t* dp,
                                            const uint32_t* st_vec) {
  constexpr int LB = ilog2(NW);
#pragma unroll
  for (int u = 0; u < NW / 4; ++u)
    stg_stream(dp + st_vec[u], make_uint4(Q[deposit_word(u, 0, LB, A, B)], Q[deposit_word(u, 1, LB, A, B)],
                                          Q[deposit_word(u, 2, LB, A, B)], Q[deposit_word(u, 3, LB, A, B)]));
}

template <int NW, int A, int B>
__device__ __forceinline__ bool stg_try_b(int a, int b, const uint32_t (&Q)[NW], uint8_t* dp,
                                          const uint32_t* st_vec) {
  constexpr int LB = ilog2(NW);
  if constexpr (B >= LB) {
    return false;
  } else {
    if constexpr (A != B) {
      if (a == A && b == B) {
        stg_vectors<NW, A, B>(Q, dp, st_vec);
        return true;
      }
    }
    return stg_try_b<NW, A, B + 1>(a, b, Q, dp, st_vec);
  }
}

template <int NW, int A>
__device__ __forceinline__ bool stg_try_a(int a, int b, const uint32_t (&Q)[NW], uint8_t* dp,
                                          const uint32_t* st_vec) {
  constexpr int LB = ilog2(NW);
  if constexpr (A >= LB) {
    return false;
  } else {
    if (stg_try_b<NW, A, 0>(a, b, Q, dp, st_vec)) return true;
    return stg_try_a<NW, A + 1>(a, b, Q, dp, st_vec);
  }
}

template <int W, int NV, int NS>
__global__ void __launch_bounds__(256) convert_async_kernel(const __grid_constant__ SmemPlan p,
                                                            const uint8_t* __restrict__ src,
                                                            uint8_t* __restrict__ dst,
                                                            int64_t n_groups, TileRange rg) {
  constexpr int NW = NV * 4;
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int gw = p.gw;
  const int group = warp >> gw;
  const int tb = lane | ((warp & ((1 << gw) - 1)) << 5);
  const int gpc = (blockDim.x >> 5) >> gw;
  const int tbits = 5 + gw;
  const int64_t gid = (int64_t)blockIdx.x * gpc + group;
  if (gid >= n_groups) return;
  uint32_t ld_off = 0, st_off = 0, swx = 0, srx = 0;
#pragma unroll
  for (int b = 0; b < LL_MAX_TBITS; ++b) {
    if (b < tbits && ((tb >> b) & 1)) {
      ld_off += p.ld_thr[b];
      st_off += p.st_thr[b];
      swx ^= p.sw_thr[b];
      srx ^= p.sr_thr[b];
    }
  }
  const uint8_t* sthr = src + ld_off - rg.src_shift;
  uint8_t* dthr = dst + st_off - rg.dst_shift;
  const int n_bits = p.tile.n_bits;
  const int n_tab = p.tile.n_tab;
  const int64_t rmask = (int64_t(1) << n_bits) - 1;
  auto tile_off = [&](int64_t t, int64_t& so, int64_t& dof) {
    const int64_t inst = t >> n_bits;
    const int64_t r = t & rmask;
    so = inst * p.tile.batch_stride_src;
    dof = inst * p.tile.batch_stride_dst;
#pragma unroll
    for (int k = 0; k < LL_MAX_TAB; ++k) {
      if (k < n_tab) {
        const TileTab& e = p.tile.tab[k][(int)((r >> (k * LL_TAB_BITS)) & ((1 << LL_TAB_BITS) - 1))];
        so += e.src;
        dof += e.dst;
      }
    }
  };
  const uint32_t tb_bytes = (uint32_t)p.tile_bytes;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem) + group * NS * tb_bytes;
  auto issue = [&](int64_t t, int stg) {
    if (t < rg.t1) {
      int64_t so, dof;
      tile_off(t, so, dof);
      const uint8_t* sp = sthr + so;
      const uint32_t st_base = sbase + stg * tb_bytes;
#pragma unroll
      for (int u = 0; u < NV; ++u) cp_async16(st_base + (swx ^ p.sw_gran[u]), sp + p.ld_vec[u]);
    }
    cp_async_commit();
  };
  const int64_t t_first = rg.t0 + gid;
#pragma unroll
  for (int s = 0; s < NS - 1; ++s) issue(t_first + s * n_groups, s);
  int stage = 0;
  const int ga = p.gsel_a, gb = p.gsel_b;
  for (int64_t t = t_first; t < rg.t1; t += n_groups) {
    cp_async_wait<NS - 2>();
    group_sync(gw, group);
    issue(t + (NS - 1) * n_groups, stage == 0 ? NS - 1 : stage - 1);
    uint32_t Q[NW];
    const uint32_t rb = sbase + stage * tb_bytes;
#pragma unroll
    for (int j = 0; j < NV; ++j) lds<16>(rb + (srx ^ p.sr_gran[j]), &Q[4 * j]);
    for (int s = 0; s < p.n_swaps; ++s) apply_swap<W, NW>(Q, p.swap_a[s], p.swap_b[s]);
    int64_t so, dof;
    tile_off(t, so, dof);
    stg_try_a<NW, 0>(ga, gb, Q, dthr + dof, p.st_vec);
    stage = stage == NS - 1 ? 0 : stage + 1;
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------- shuffle kernel
//
// Warp-shuffle conversion (reading A11): the paper's 2^|R| rounds,
// one 32-bit word per lane per round.  The lane-dependent part of the send /
// receive word index is a XOR mask applied with selects; the uniform part is
// a linear map of the word index applied as elementary register operations
// (plan data, every case unrolled so the register file stays in registers).

template <int NW>
__device__ __forceinline__ void lane_xor(uint32_t (&T)[NW], uint32_t m, uint32_t any) {
  constexpr int LB = ilog2(NW);
#pragma unroll
  for (int b = 0; b < LB; ++b) {
    if ((any >> b) & 1) {
      const bool q = (m >> b) & 1;
#pragma unroll
      for (int k = 0; k < NW; ++k) {
        if (((k >> b) & 1) == 0) {
          const uint32_t x = T[k], y = T[k | (1 << b)];
          T[k] = q ? y : x;
          T[k | (1 << b)] = q ? x : y;
        }
      }
    }
  }
}

// op 0: T'[k] = T[k with bits a, b swapped]; op 1: T'[k] = T[k ^ (bit a of k) << b]
template <int NW>
__device__ __forceinline__ void lin_op(uint32_t (&T)[NW], int op, int a, int b) {
  constexpr int LB = ilog2(NW);
#pragma unroll
  for (int A = 0; A < LB; ++A) {
#pragma unroll
    for (int B = 0; B < LB; ++B) {
      if (A != B && a == A && b == B) {
        if (op == 0) {
#pragma unroll
          for (int k = 0; k < NW; ++k) {
            if (((k >> A) & 1) == 0 && ((k >> B) & 1) == 1) {
              const int j = k ^ ((1 << A) | (1 << B));
              const uint32_t t = T[k];
              T[k] = T[j];
              T[j] = t;
            }
          }
        } else {
#pragma unroll
          for (int k = 0; k < NW; ++k) {
            if (((k >> A) & 1) == 1 && ((k >> B) & 1) == 0) {
              const int j = k | (1 << B);
              const uint32_t t = T[k];
              T[k] = T[j];
              T[j] = t;
            }
          }
        }
      }
    }
  }
}

template <int W, int NV, bool PIPE>
__global__ void __launch_bounds__(256) convert_shuffle_kernel(const __grid_constant__ ShufflePlan p,
                                                              const uint8_t* __restrict__ src,
                                                              uint8_t* __restrict__ dst,
                                                              int64_t n_groups, TileRange rg) {
  constexpr int NW = NV * 4;
  const int lane = threadIdx.x & 31;
  const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (gid >= n_groups) return;
  uint32_t ld_off = 0, st_off = 0, beta = 0, zeta = 0, delta = 0;
#pragma unroll
  for (int b = 0; b < 5; ++b) {
    if ((lane >> b) & 1) {
      ld_off += p.ld_thr[b];
      st_off += p.st_thr[b];
      beta ^= p.beta_lane[b];
      zeta ^= p.zeta_lane[b];
      delta ^= p.delta_lane[b];
    }
  }
  const uint8_t* sthr = src + ld_off - rg.src_shift;
  uint8_t* dthr = dst + st_off - rg.dst_shift;
  const int n_bits = p.tile.n_bits;
  const int n_tab = p.tile.n_tab;
  const int64_t rmask = (int64_t(1) << n_bits) - 1;
  auto tile_off = [&](int64_t t, int64_t& so, int64_t& dof) {
    const int64_t inst = t >> n_bits;
    const int64_t r = t & rmask;
    so = inst * p.tile.batch_stride_src;
    dof = inst * p.tile.batch_stride_dst;
#pragma unroll
    for (int k = 0; k < LL_MAX_TAB; ++k) {
      if (k < n_tab) {
        const TileTab& e = p.tile.tab[k][(int)((r >> (k * LL_TAB_BITS)) & ((1 << LL_TAB_BITS) - 1))];
        so += e.src;
        dof += e.dst;
      }
    }
  };
  const int64_t n_tiles = rg.t1;
  uint32_t R[NW];
  int64_t so, dof;
  int64_t t = rg.t0 + gid;
  if (PIPE && t < n_tiles) {
    tile_off(t, so, dof);
    load_tile<NV>(R, sthr + so, p.ld_vec);
  }
  for (; t < n_tiles; t += n_groups) {
    if (!PIPE) tile_off(t, so, dof);
    if (!PIPE) load_tile<NV>(R, sthr + so, p.ld_vec);
    const int64_t dcur = dof;
    for (int s = 0; s < p.n_swaps; ++s) apply_swap<W, NW>(R, p.swap_a[s], p.swap_b[s]);
    lane_xor<NW>(R, beta, p.beta_any);
    for (int i = 0; i < p.n_pre; ++i) lin_op<NW>(R, p.pre_op[i], p.pre_a[i], p.pre_b[i]);
    uint32_t X[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) X[k] = __shfl_sync(0xffffffffu, R[k], (int)(p.gamma[k] ^ delta));
    if (PIPE) {
      const int64_t tn = t + n_groups;
      if (tn < n_tiles) {
        tile_off(tn, so, dof);
        load_tile<NV>(R, sthr + so, p.ld_vec);
      }
    }
    for (int i = 0; i < p.n_post; ++i) lin_op<NW>(X, p.post_op[i], p.post_a[i], p.post_b[i]);
    lane_xor<NW>(X, zeta, p.zeta_any);
    uint8_t* dp = dthr + dcur;
#pragma unroll
    for (int u = 0; u < NV; ++u)
      stg_stream(dp + p.st_vec[u], make_uint4(X[4 * u + 0], X[4 * u + 1], X[4 * u + 2], X[4 * u + 3]));
  }
}

// ------------------------------------------------------------ generic kernel

// dst[h] = src[X h]: each thread writes one 16-byte destination vector; the
// source elements are fetched one by one (the slow, always-applicable path).
template <int W>
__global__ void __launch_bounds__(256) convert_generic_kernel(const __grid_constant__ GenericPlan p,
                                                              const uint8_t* __restrict__ src,
                                                              uint8_t* __restrict__ dst) {
  constexpr int NE = 16 / W;
  constexpr int VB = ilog2(NE);
  using T = typename std::conditional<W == 1, uint8_t,
            typename std::conditional<W == 2, uint16_t,
            typename std::conditional<W == 4, uint32_t, uint64_t>::type>::type>::type;
  const int64_t per_batch = (p.nB >= VB) ? (int64_t(1) << (p.nB - VB)) : 1;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < p.n_vec;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = v / per_batch;
    const uint64_t h0 = (uint64_t)(v - b * per_batch) << VB;
    uint64_t x0 = 0;
    for (int k = VB; k < p.nB; ++k)
      if ((h0 >> k) & 1) x0 ^= (uint64_t)p.x[k];
    const T* s = reinterpret_cast<const T*>(src) + b * p.batch_stride_src;
    T* d = reinterpret_cast<T*>(dst) + b * p.batch_stride_dst + h0;
    union {
      uint4 v4;
      T e[NE];
    } out;
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      uint64_t x = x0;
#pragma unroll
      for (int k = 0; k < VB; ++k)
        if ((e >> k) & 1) x ^= (uint64_t)p.x[k];
      out.e[e] = (e < (1 << (p.nB < VB ? p.nB : VB))) ? __ldg(s + x) : T(0);
    }
    if (p.nB >= VB) {
      *reinterpret_cast<uint4*>(d) = out.v4;
    } else {
      for (int e = 0; e < (1 << p.nB); ++e) d[e] = out.e[e];
    }
  }
}

// ------------------------------------------------------------ gather kernels

// Direct gather: each thread produces one 16-byte output vector; source
// elements are read through L1 (the rows a warp gathers from are the rows it
// covers, so L1 absorbs the reuse).  Works for any axis placement.
template <int W>
__global__ void __launch_bounds__(256) gather_direct_kernel(const __grid_constant__ GatherPlan p,
                                                            const uint8_t* __restrict__ src,
                                                            const int32_t* __restrict__ idx,
                                                            uint8_t* __restrict__ out,
                                                            int* __restrict__ err) {
  constexpr int NE = 16 / W;
  constexpr int VB = ilog2(NE);
  using T = typename std::conditional<W == 1, uint8_t,
            typename std::conditional<W == 2, uint16_t,
            typename std::conditional<W == 4, uint32_t, uint64_t>::type>::type>::type;
  const int64_t per_batch = int64_t(1) << (p.nbits - VB);
  const uint32_t amask = (1u << p.ax_bits) - 1;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < p.n_vec;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = v / per_batch;
    const uint64_t h0 = (uint64_t)(v - b * per_batch) << VB;
    const T* s = reinterpret_cast<const T*>(src) + b * p.batch_stride;
    const int32_t* ip = idx + b * p.batch_stride + h0;
    // warm L1 with this thread's own source vector while the indices load: for
    // row-local axes the warp's gathers then hit lines already in flight
    asm volatile("prefetch.global.L1 [%0];" ::"l"(s + h0));
    int32_t iv[NE];
    if constexpr (NE >= 4) {
#pragma unroll
      for (int q = 0; q < NE / 4; ++q) {
        int4 t = __ldg(reinterpret_cast<const int4*>(ip) + q);
        iv[4 * q] = t.x; iv[4 * q + 1] = t.y; iv[4 * q + 2] = t.z; iv[4 * q + 3] = t.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < NE; ++q) iv[q] = __ldg(ip + q);
    }
    union {
      uint4 v4;
      T e[NE];
    } o;
    // axis coordinate of h0's elements and the "cleared" base
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const uint64_t h = h0 | (uint64_t)e;
      uint64_t hs;
      uint32_t i = (uint32_t)iv[e];
      if (p.check && i > amask) atomicExch(err, 1);
      i &= amask;
      if (p.y_contig) {
        hs = (h & ~(uint64_t)p.axis_mask_buf) | ((uint64_t)i << p.y_base);
      } else {
        // h* = h ^ Y(axis(h) ^ idx)
        uint64_t t = 0;
        for (int k = 0; k < p.nbits; ++k)
          if ((h >> k) & 1) t ^= (uint64_t)p.L[k];
        uint32_t a = (uint32_t)(t >> p.ax_shift) & amask;
        uint32_t dlt = a ^ i;
        hs = h;
        for (int k = 0; k < p.ax_bits; ++k)
          if ((dlt >> k) & 1) hs ^= (uint64_t)p.Y[k];
      }
      o.e[e] = __ldg(s + hs);
    }
    *reinterpret_cast<uint4*>(reinterpret_cast<T*>(out) + b * p.batch_stride + h0) = o.v4;
  }
}

// Warp-shuffle gather (reading A19): each lane holds one 16-byte
// vector of src (registers = the vector's elements, lanes = the next five
// buffer bits).  For each output element the source (register, lane) comes
// from h* = (h with axis replaced); one shuffle per candidate register
// (2^|L_reg^axis|, mask `cand_mask`), keeping the value whose register
// matches.  Requires the axis to live in the warp's buffer bits (vb + 5).
// ALLC: the axis covers every register bit (cand_mask = NE-1): all NE words
// are shuffled from the source lane and a select tree picks the element.
template <int W, bool ALLC>
__global__ void __launch_bounds__(256) gather_shuffle_kernel(const __grid_constant__ GatherPlan p,
                                                             const uint8_t* __restrict__ src,
                                                             const int32_t* __restrict__ idx,
                                                             uint8_t* __restrict__ out,
                                                             int* __restrict__ err) {
  constexpr int NE = 16 / W;
  constexpr int VB = ilog2(NE);
  using T = typename std::conditional<W == 1, uint8_t,
            typename std::conditional<W == 2, uint16_t,
            typename std::conditional<W == 4, uint32_t, uint64_t>::type>::type>::type;
  const int lane = threadIdx.x & 31;
  const int64_t per_batch = int64_t(1) << (p.nbits - VB);
  const uint32_t amask = (1u << p.ax_bits) - 1;
  const int64_t nwarps_total = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n_wvec = p.n_vec >> 5;  // warps' worth of vectors
  const uint32_t clear32 = ~(uint32_t)p.axis_mask_buf;
  const int ybase = p.y_base;
  for (int64_t wv = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wv < n_wvec;
       wv += nwarps_total) {
    const int64_t v = (wv << 5) | lane;
    const int64_t b = v / per_batch;
    const uint64_t h0 = (uint64_t)(v - b * per_batch) << VB;
    const uint8_t* sbase = src + (b * p.batch_stride) * W;
    union {
      uint4 v4;
      T e[NE];
      uint32_t w[4];
    } sv, o;
    sv.v4 = ldg_stream(sbase + h0 * W);
    const int32_t* ip = idx + b * p.batch_stride + h0;
    int32_t iv[NE];
    if constexpr (NE >= 4) {
#pragma unroll
      for (int q = 0; q < NE / 4; ++q) {
        int4 t = __ldg(reinterpret_cast<const int4*>(ip) + q);
        iv[4 * q] = t.x; iv[4 * q + 1] = t.y; iv[4 * q + 2] = t.z; iv[4 * q + 3] = t.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < NE; ++q) iv[q] = __ldg(ip + q);
    }
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      // only the warp-local bits (VB + 5) of h* matter here: 32-bit arithmetic
      uint32_t i = (uint32_t)iv[e];
      if (p.check && i > amask) atomicExch(err, 1);
      i &= amask;
      const uint32_t hl = (((uint32_t)lane << VB) | (uint32_t)e) & clear32;
      const uint32_t hs = hl | (i << ybase);
      const int src_lane = (int)((hs >> VB) & 31);
      const int src_reg = (int)(hs & (NE - 1));
      if constexpr (ALLC && W == 4) {
        // four shuffles, then a 2-level select on the register index
        const uint32_t g0 = __shfl_sync(0xffffffffu, sv.w[0], src_lane);
        const uint32_t g1 = __shfl_sync(0xffffffffu, sv.w[1], src_lane);
        const uint32_t g2 = __shfl_sync(0xffffffffu, sv.w[2], src_lane);
        const uint32_t g3 = __shfl_sync(0xffffffffu, sv.w[3], src_lane);
        const uint32_t lo = (src_reg & 1) ? g1 : g0;
        const uint32_t hi = (src_reg & 1) ? g3 : g2;
        o.e[e] = (T)((src_reg & 2) ? hi : lo);
      } else {
        T val = 0;
        // candidate rounds: every register index the axis can select, i.e. the
        // registers that agree with e outside cand_mask (2^|L_reg^axis| shuffles)
#pragma unroll
        for (int c = 0; c < NE; ++c) {
          if (ALLC || ((c ^ e) & ~p.cand_mask) == 0) {
            T got;
            if constexpr (W == 8) {
              uint32_t lo = __shfl_sync(0xffffffffu, sv.w[2 * c], src_lane);
              uint32_t hi = __shfl_sync(0xffffffffu, sv.w[2 * c + 1], src_lane);
              got = (T)(((uint64_t)hi << 32) | lo);
            } else if constexpr (W == 4) {
              got = (T)__shfl_sync(0xffffffffu, sv.w[c], src_lane);
            } else {
              // sub-word elements: shuffle the containing word, then extract
              uint32_t wd = __shfl_sync(0xffffffffu, sv.w[(c * W) >> 2], src_lane);
              got = (T)(wd >> (((c * W) & 3) * 8));
            }
            if (src_reg == c) val = got;
          }
        }
        o.e[e] = val;
      }
    }
    stg_stream(out + (b * p.batch_stride + h0) * W, o.v4);
  }
}

// ------------------------------------------------------------------ launchers

static int g_num_sms = 0;
static int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

static int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

// Launch configuration knobs (env, read once): LL_TPG = target tiles per tile
// group (0 = persistent grid at full occupancy), LL_PIPE = 1 for the
// software-pipelined kernel.
struct LaunchKnobs {
  int tpg, pipe, gather_tpt, carveout, pow2, stages, async_tpg;
  LaunchKnobs()
      : tpg(env_int("LL_TPG", 2)), pipe(env_int("LL_PIPE", 1)),
        gather_tpt(env_int("LL_GATHER_VPT", 0)), carveout(env_int("LL_CARVEOUT", -1)),
        pow2(env_int("LL_POW2", 0)), stages(env_int("LL_STAGES", 3)),
        async_tpg(env_int("LL_ASYNC_TPG", 8)) {}
};
static LaunchKnobs& knobs() {
  static LaunchKnobs k;
  return k;
}

int set_knob(const char* name, int value) {
  std::string n(name ? name : "");
  if (n == "tpg") { knobs().tpg = value; return 0; }
  if (n == "pipe") { knobs().pipe = value; return 0; }
  if (n == "gather_vpt") { knobs().gather_tpt = value; return 0; }
  if (n == "carveout") { knobs().carveout = value; return 0; }
  if (n == "pow2") { knobs().pow2 = value; return 0; }
  if (n == "stages") { knobs().stages = value; return 0; }
  if (n == "async_tpg") { knobs().async_tpg = value; return 0; }
  return -1;
}

template <int W, int NV, int G, bool PIPE, bool PAD>
static cudaError_t launch_smem_p(const SmemPlan& p, const void* src, void* dst, int max_ctas,
                                 cudaStream_t st, const TileRange& rg) {
  auto k = convert_smem_kernel<W, NV, G, PIPE, PAD>;
  const int threads = 256;
  const int gpc = (threads / 32) >> p.gw;
  const size_t smem = (size_t)gpc * 2 * p.tile_bytes;  // tile_bytes includes any padding
  static int occ_cache = -1;
  static size_t occ_smem = 0;
  static int occ_carve = -2;
  if (occ_cache < 0 || occ_smem != smem || occ_carve != knobs().carveout) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, knobs().carveout);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_cache, k, threads, smem);
    occ_smem = smem;
    occ_carve = knobs().carveout;
  }
  if (occ_cache <= 0) return cudaErrorInvalidConfiguration;
  const int64_t n_tiles = rg.t1 - rg.t0;
  if (n_tiles <= 0) return cudaSuccess;
  // tile groups: n_tiles / tpg (the hardware block scheduler balances the
  // tail), or the resident capacity when tpg = 0 (persistent)
  const int tpg = knobs().tpg;
  int64_t groups = tpg > 0 ? (n_tiles + tpg - 1) / tpg : (int64_t)occ_cache * num_sms() * gpc;
  if (max_ctas > 0) groups = std::min<int64_t>(groups, (int64_t)max_ctas * gpc);
  groups = std::max<int64_t>(1, std::min<int64_t>(groups, n_tiles));
  const int64_t grid = (groups + gpc - 1) / gpc;
  if (grid > 0x7fffffff) return cudaErrorInvalidConfiguration;
  k<<<(unsigned)grid, threads, smem, st>>>(p, (const uint8_t*)src, (uint8_t*)dst, groups, rg);
  return cudaGetLastError();
}

template <int W, int NV, int G>
static cudaError_t launch_smem_t(const SmemPlan& p, const void* src, void* dst, int max_ctas,
                                 cudaStream_t st, const TileRange& rg) {
  if (p.pad) return launch_smem_p<W, NV, G, true, true>(p, src, dst, max_ctas, st, rg);
  if (knobs().pipe) return launch_smem_p<W, NV, G, true, false>(p, src, dst, max_ctas, st, rg);
  return launch_smem_p<W, NV, G, false, false>(p, src, dst, max_ctas, st, rg);
}

template <int W>
static cudaError_t launch_smem_w(const SmemPlan& p, int nv, int g, const void* src, void* dst,
                                 int max_ctas, cudaStream_t st, const TileRange& rg) {
#define LL_CASE(NV_, G_) \
  if (nv == NV_ && g == G_) return launch_smem_t<W, NV_, G_>(p, src, dst, max_ctas, st, rg);
  LL_CASE(1, 4) LL_CASE(1, 8) LL_CASE(1, 16)
  LL_CASE(2, 4) LL_CASE(2, 8) LL_CASE(2, 16)
  LL_CASE(4, 4) LL_CASE(4, 8) LL_CASE(4, 16)
  LL_CASE(8, 4) LL_CASE(8, 8) LL_CASE(8, 16)
#undef LL_CASE
  return cudaErrorNotSupported;
}

cudaError_t launch_convert_smem(const SmemPlan& p, int w, int nv, int g, const void* src, void* dst,
                                int max_ctas, cudaStream_t st, const TileRange& rg) {
  switch (w) {
    case 1: return launch_smem_w<1>(p, nv, g, src, dst, max_ctas, st, rg);
    case 2: return launch_smem_w<2>(p, nv, g, src, dst, max_ctas, st, rg);
    case 4: return launch_smem_w<4>(p, nv, g, src, dst, max_ctas, st, rg);
    case 8: return launch_smem_w<8>(p, nv, g, src, dst, max_ctas, st, rg);
  }
  return cudaErrorNotSupported;
}

template <int W, int NV, int NS>
static cudaError_t launch_async_p(const SmemPlan& p, const void* src, void* dst, int max_ctas,
                                  cudaStream_t st, const TileRange& rg) {
  auto k = convert_async_kernel<W, NV, NS>;
  const int threads = 256;
  const int gpc = (threads / 32) >> p.gw;
  const size_t smem = (size_t)gpc * NS * p.tile_bytes;
  if (smem > 200 * 1024) return cudaErrorInvalidConfiguration;
  static int occ_cache = -1;
  static size_t occ_smem = 0;
  if (occ_cache < 0 || occ_smem != smem) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_cache, k, threads, smem);
    occ_smem = smem;
  }
  if (occ_cache <= 0) return cudaErrorInvalidConfiguration;
  const int64_t n_tiles = rg.t1 - rg.t0;
  if (n_tiles <= 0) return cudaSuccess;
  const int tpg = knobs().async_tpg;
  int64_t groups = tpg > 0 ? (n_tiles + tpg - 1) / tpg : (int64_t)occ_cache * num_sms() * gpc;
  if (max_ctas > 0) groups = std::min<int64_t>(groups, (int64_t)max_ctas * gpc);
  groups = std::max<int64_t>(1, std::min<int64_t>(groups, n_tiles));
  const int64_t grid = (groups + gpc - 1) / gpc;
  if (grid > 0x7fffffff) return cudaErrorInvalidConfiguration;
  k<<<(unsigned)grid, threads, smem, st>>>(p, (const uint8_t*)src, (uint8_t*)dst, groups, rg);
  return cudaGetLastError();
}

template <int W>
static cudaError_t launch_async_w(const SmemPlan& p, int nv, const void* src, void* dst,
                                  int max_ctas, cudaStream_t st, const TileRange& rg) {
  const int ns = knobs().stages;
#define LL_ACASE(NV_)                                                        \
  if (nv == NV_) {                                                           \
    if (ns <= 2) return launch_async_p<W, NV_, 2>(p, src, dst, max_ctas, st, rg); \
    if (ns == 3) return launch_async_p<W, NV_, 3>(p, src, dst, max_ctas, st, rg); \
    return launch_async_p<W, NV_, 4>(p, src, dst, max_ctas, st, rg);         \
  }
  LL_ACASE(1) LL_ACASE(2) LL_ACASE(4) LL_ACASE(8)
#undef LL_ACASE
  return cudaErrorNotSupported;
}

cudaError_t launch_convert_async(const SmemPlan& p, int w, int nv, const void* src, void* dst,
                                 int max_ctas, cudaStream_t st, const TileRange& rg) {
  switch (w) {
    case 1: return launch_async_w<1>(p, nv, src, dst, max_ctas, st, rg);
    case 2: return launch_async_w<2>(p, nv, src, dst, max_ctas, st, rg);
    case 4: return launch_async_w<4>(p, nv, src, dst, max_ctas, st, rg);
    case 8: return launch_async_w<8>(p, nv, src, dst, max_ctas, st, rg);
  }
  return cudaErrorNotSupported;
}

template <int W, int NV, bool PIPE>
static cudaError_t launch_shuffle_p(const ShufflePlan& p, const void* src, void* dst, int max_ctas,
                                    cudaStream_t st, const TileRange& rg) {
  auto k = convert_shuffle_kernel<W, NV, PIPE>;
  const int threads = 256;
  const int gpc = threads / 32;
  const int64_t n_tiles = rg.t1 - rg.t0;
  if (n_tiles <= 0) return cudaSuccess;
  static int occ_cache = -1;
  if (occ_cache < 0) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_cache, k, threads, 0);
  const int tpg = knobs().tpg;
  int64_t groups = tpg > 0 ? (n_tiles + tpg - 1) / tpg : (int64_t)std::max(1, occ_cache) * num_sms() * gpc;
  if (max_ctas > 0) groups = std::min<int64_t>(groups, (int64_t)max_ctas * gpc);
  groups = std::max<int64_t>(1, std::min<int64_t>(groups, n_tiles));
  const int64_t grid = (groups + gpc - 1) / gpc;
  if (grid > 0x7fffffff) return cudaErrorInvalidConfiguration;
  k<<<(unsigned)grid, threads, 0, st>>>(p, (const uint8_t*)src, (uint8_t*)dst, groups, rg);
  return cudaGetLastError();
}

template <int W>
static cudaError_t launch_shuffle_w(const ShufflePlan& p, int nv, const void* src, void* dst,
                                    int max_ctas, cudaStream_t st, const TileRange& rg) {
  const bool pipe = knobs().pipe != 0;
#define LL_SCASE(NV_) \
  if (nv == NV_) return pipe ? launch_shuffle_p<W, NV_, true>(p, src, dst, max_ctas, st, rg) \
                             : launch_shuffle_p<W, NV_, false>(p, src, dst, max_ctas, st, rg);
  LL_SCASE(1) LL_SCASE(2) LL_SCASE(4) LL_SCASE(8)
#undef LL_SCASE
  return cudaErrorNotSupported;
}

cudaError_t launch_convert_shuffle(const ShufflePlan& p, int w, int nv, const void* src, void* dst,
                                   int max_ctas, cudaStream_t st, const TileRange& rg) {
  switch (w) {
    case 1: return launch_shuffle_w<1>(p, nv, src, dst, max_ctas, st, rg);
    case 2: return launch_shuffle_w<2>(p, nv, src, dst, max_ctas, st, rg);
    case 4: return launch_shuffle_w<4>(p, nv, src, dst, max_ctas, st, rg);
  }
  return cudaErrorNotSupported;
}

template <int W>
static cudaError_t launch_generic_t(const GenericPlan& p, const void* src, void* dst, int max_ctas,
                                    cudaStream_t st) {
  const int threads = 256;
  int64_t want = (p.n_vec + threads - 1) / threads;
  int64_t cap = (int64_t)num_sms() * 8;
  if (max_ctas > 0 && cap > max_ctas) cap = max_ctas;
  int grid = (int)(want < cap ? want : cap);
  if (grid < 1) grid = 1;
  convert_generic_kernel<W><<<grid, threads, 0, st>>>(p, (const uint8_t*)src, (uint8_t*)dst);
  return cudaGetLastError();
}

cudaError_t launch_convert_generic(const GenericPlan& p, int w, const void* src, void* dst,
                                   int max_ctas, cudaStream_t st) {
  switch (w) {
    case 1: return launch_generic_t<1>(p, src, dst, max_ctas, st);
    case 2: return launch_generic_t<2>(p, src, dst, max_ctas, st);
    case 4: return launch_generic_t<4>(p, src, dst, max_ctas, st);
    case 8: return launch_generic_t<8>(p, src, dst, max_ctas, st);
  }
  return cudaErrorNotSupported;
}

template <int W>
static cudaError_t launch_gather_t(const GatherPlan& p, bool shuffle, const void* src,
                                   const int32_t* idx, void* out, int* err, int max_ctas,
                                   cudaStream_t st) {
  const int threads = 256;
  // 16-byte output vectors per thread (measured on B200: 4 for the shuffle
  // kernel, 1 for the direct kernel); the knob overrides
  const int vpt = knobs().gather_tpt > 0 ? knobs().gather_tpt : (shuffle ? 4 : 1);
  int64_t want = (p.n_vec + (int64_t)threads * vpt - 1) / ((int64_t)threads * vpt);
  if (max_ctas > 0 && want > max_ctas) want = max_ctas;
  int grid = (int)(want < 0x7fffffff ? want : 0x7fffffff);
  if (grid < 1) grid = 1;
  if (shuffle && p.cand_mask == (16 / W) - 1)
    gather_shuffle_kernel<W, true><<<grid, threads, 0, st>>>(p, (const uint8_t*)src, idx,
                                                            (uint8_t*)out, err);
  else if (shuffle)
    gather_shuffle_kernel<W, false><<<grid, threads, 0, st>>>(p, (const uint8_t*)src, idx,
                                                             (uint8_t*)out, err);
  else
    gather_direct_kernel<W><<<grid, threads, 0, st>>>(p, (const uint8_t*)src, idx, (uint8_t*)out,
                                                     err);
  return cudaGetLastError();
}

cudaError_t launch_gather(const GatherPlan& p, int w, bool shuffle, const void* src,
                          const int32_t* idx, void* out, int* err, int max_ctas, cudaStream_t st) {
  switch (w) {
    case 1: return launch_gather_t<1>(p, shuffle, src, idx, out, err, max_ctas, st);
    case 2: return launch_gather_t<2>(p, shuffle, src, idx, out, err, max_ctas, st);
    case 4: return launch_gather_t<4>(p, shuffle, src, idx, out, err, max_ctas, st);
    case 8: return launch_gather_t<8>(p, shuffle, src, idx, out, err, max_ctas, st);
  }
  return cudaErrorNotSupported;
}

int device_sm_count() { return num_sms(); }

}  // namespace ll
