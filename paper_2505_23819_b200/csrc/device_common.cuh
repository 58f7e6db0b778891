// device_common.cuh -- device helpers shared by the sm_100a kernels (PTX
// wrappers, register-bit swaps, compile-time operand selection) and the
// launch-configuration knobs.  Included by the kernel translation units.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <map>
#include <mutex>
#include <tuple>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "kernels.hpp"
#include "plan.hpp"

namespace ll {

// ------------------------------------------------------------------ PTX helpers

// LL_LDG_HINT (build-time experiment): 0 = L1::no_allocate; 1 = + L2::256B
// prefetch; 2 = + L2::evict_first; 3 = both.  LL_STG_HINT: 0 = .cs
// (streaming); 1 = default (.wb); 2 = L2::evict_last ... (see the sweep).
#ifndef LL_LDG_HINT
#define LL_LDG_HINT 0
#endif
#ifndef LL_STG_HINT
#define LL_STG_HINT 0
#endif
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 v;
#if LL_LDG_HINT == 1
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
#elif LL_LDG_HINT == 2
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.u32 {%0,%1,%2,%3}, [%4];"
#elif LL_LDG_HINT == 3
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
#else
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
#endif
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void stg_stream(void* p, uint4 v) {
#if LL_STG_HINT == 1
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
#elif LL_STG_HINT == 2
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
#else
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
#endif
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


// ------------------------------------------------------------- launch knobs
int num_sms();

// Resident CTAs per SM of `kernel` for (threads, dynamic smem, carveout),
// computed once per key (thread-safe: several host threads may launch).  The
// kernel's max dynamic smem (220 KB) and carveout (if != -1) are set first.
int cached_occupancy(const void* kernel, int threads, size_t smem, int carveout);
struct LaunchKnobs {
  int tpg, pipe, gather_tpt, carveout, pow2, stages, async_tpg, up_tpg, tma_tpg, tma_stages, gather_v8,
      gather_shfl_u;
  LaunchKnobs();
};
LaunchKnobs& knobs();

}  // namespace ll
