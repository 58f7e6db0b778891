// kernel_regs.cu -- register-faithful conversion (LL_PATH_REGS): the paper's
// in-kernel convert_layout with the layouts' own lanes and warps.
//
// One CTA per block index (grid-stride over blocks x batch); thread t =
// lane + 32 warp loads its 2^reg elements (contiguous in the source's
// hardware order), fixes the sub-word order with prmt, writes them to shared
// memory through S (st.shared.v{1,2,4} or stmatrix.x{1,2,4}), bar.sync,
// reads its destination registers (ld.shared.v{1,2,4} or ldmatrix.x{1,2,4})
// and stores them contiguously.  `reps` > 1 repeats the register -> smem ->
// register exchange inside the kernel and thread 0 of each CTA records the
// clock64 cycles of the repeated section (the paper's microbenchmarks time
// the conversion inside one CTA).
#include "device_common.cuh"

namespace ll {

// MAT: 0 = st/ld.shared vectors, 1 = stmatrix / ldmatrix, 2 = their .trans
// forms, 3 = the sm_100a 8-bit forms stmatrix.m16n8.trans.b8 /
// ldmatrix.m16n16.trans.b8 (G = words per thread: 1 / 2 / 4 matrices for the
// store, 2 / 4 words = x1 / x2 for the load)
template <int G, int MAT>
__device__ __forceinline__ void smem_put(uint32_t addr, const uint32_t* r) {
  if constexpr (MAT == 0) {
    sts<G * 4>(addr, r);
  } else if constexpr (MAT == 3 && G == 4) {
    asm volatile("stmatrix.sync.aligned.m16n8.x4.trans.shared.b8 [%0], {%1, %2, %3, %4};" ::"r"(addr),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3])
                 : "memory");
  } else if constexpr (MAT == 3 && G == 2) {
    asm volatile("stmatrix.sync.aligned.m16n8.x2.trans.shared.b8 [%0], {%1, %2};" ::"r"(addr), "r"(r[0]),
                 "r"(r[1])
                 : "memory");
  } else if constexpr (MAT == 3) {
    asm volatile("stmatrix.sync.aligned.m16n8.x1.trans.shared.b8 [%0], {%1};" ::"r"(addr), "r"(r[0])
                 : "memory");
  } else if constexpr (MAT == 2 && G == 4) {
    asm volatile("stmatrix.sync.aligned.m8n8.x4.trans.shared.b16 [%0], {%1, %2, %3, %4};" ::"r"(addr),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3])
                 : "memory");
  } else if constexpr (MAT == 2 && G == 2) {
    asm volatile("stmatrix.sync.aligned.m8n8.x2.trans.shared.b16 [%0], {%1, %2};" ::"r"(addr), "r"(r[0]),
                 "r"(r[1])
                 : "memory");
  } else if constexpr (MAT == 2) {
    asm volatile("stmatrix.sync.aligned.m8n8.x1.trans.shared.b16 [%0], {%1};" ::"r"(addr), "r"(r[0])
                 : "memory");
  } else if constexpr (G == 4) {
    asm volatile("stmatrix.sync.aligned.m8n8.x4.shared.b16 [%0], {%1, %2, %3, %4};" ::"r"(addr),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3])
                 : "memory");
  } else if constexpr (G == 2) {
    asm volatile("stmatrix.sync.aligned.m8n8.x2.shared.b16 [%0], {%1, %2};" ::"r"(addr), "r"(r[0]),
                 "r"(r[1])
                 : "memory");
  } else {
    asm volatile("stmatrix.sync.aligned.m8n8.x1.shared.b16 [%0], {%1};" ::"r"(addr), "r"(r[0])
                 : "memory");
  }
}

template <int G, int MAT>
__device__ __forceinline__ void smem_get(uint32_t addr, uint32_t* r) {
  if constexpr (MAT == 0) {
    lds<G * 4>(addr, r);
  } else if constexpr (MAT == 3 && G == 4) {
    asm volatile("ldmatrix.sync.aligned.m16n16.x2.trans.shared.b8 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr)
                 : "memory");
  } else if constexpr (MAT == 3 && G == 2) {
    asm volatile("ldmatrix.sync.aligned.m16n16.x1.trans.shared.b8 {%0, %1}, [%2];"
                 : "=r"(r[0]), "=r"(r[1])
                 : "r"(addr)
                 : "memory");
  } else if constexpr (MAT == 3) {
    static_assert(G != 1, "ldmatrix.b8 returns at least two words");
  } else if constexpr (MAT == 2 && G == 4) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr)
                 : "memory");
  } else if constexpr (MAT == 2 && G == 2) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];"
                 : "=r"(r[0]), "=r"(r[1])
                 : "r"(addr)
                 : "memory");
  } else if constexpr (MAT == 2) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x1.trans.shared.b16 {%0}, [%1];" : "=r"(r[0]) : "r"(addr) : "memory");
  } else if constexpr (G == 4) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr)
                 : "memory");
  } else if constexpr (G == 2) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0, %1}, [%2];"
                 : "=r"(r[0]), "=r"(r[1])
                 : "r"(addr)
                 : "memory");
  } else {
    asm volatile("ldmatrix.sync.aligned.m8n8.x1.shared.b16 {%0}, [%1];" : "=r"(r[0]) : "r"(addr) : "memory");
  }
}

// all instructions of one side with compile-time operand selection: the GW
// words of instruction j are R[deposit_word(j, k, LB, A, B)], k < GW
template <int NW, int GW, int MAT, bool PUT, int A, int B>
__device__ __forceinline__ void xfer_all(uint32_t (&R)[NW], uint32_t base, uint32_t tx,
                                         const uint32_t* inst) {
  constexpr int LB = ilog2(NW);
#pragma unroll
  for (int j = 0; j < NW / GW; ++j) {
    uint32_t v[GW];
    const uint32_t addr = base + (tx ^ inst[j]);
    if constexpr (PUT) {
#pragma unroll
      for (int k = 0; k < GW; ++k) v[k] = R[deposit_word(j, k, LB, A, B)];
      smem_put<GW, MAT>(addr, v);
    } else {
      smem_get<GW, MAT>(addr, v);
#pragma unroll
      for (int k = 0; k < GW; ++k) R[deposit_word(j, k, LB, A, B)] = v[k];
    }
  }
}

// the exchange with fixed operand patterns (instruction words at word bits
// 0, 1 -- the planner permuted the registers so); the side kinds are
// dispatched once, outside the repetition loop
template <int NW, int GWW, int MW, int GWR, int MR>
__device__ __forceinline__ void exchange(uint32_t (&R)[NW], uint32_t (&Q)[NW], int reps,
                                         uint32_t sbase, uint32_t wx, uint32_t rx,
                                         const RegsPlan& p) {
  constexpr int WA = GWW >= 2 ? 0 : -1, WB = GWW >= 4 ? 1 : -1;
  constexpr int RA = GWR >= 2 ? 0 : -1, RB = GWR >= 4 ? 1 : -1;
  for (int rep = 0; rep < reps; ++rep) {
    xfer_all<NW, GWW, MW, true, WA, WB>(R, sbase, wx, p.sw_inst);
    __syncthreads();
    xfer_all<NW, GWR, MR, false, RA, RB>(Q, sbase, rx, p.sr_inst);
    __syncthreads();
  }
}

template <int W, int NW, int GWW, int MW>
__device__ __forceinline__ void exchange_r(uint32_t (&R)[NW], uint32_t (&Q)[NW], int reps,
                                           uint32_t sbase, uint32_t wx, uint32_t rx,
                                           const RegsPlan& p) {
  const int k = p.rd_gw * 4 + p.rd_mat;
  if (k == 4) exchange<NW, GWW, MW, 1, 0>(R, Q, reps, sbase, wx, rx, p);
  else if (k == 5) exchange<NW, GWW, MW, 1, 1>(R, Q, reps, sbase, wx, rx, p);
  else if (W == 2 && k == 6) exchange<NW, GWW, MW, 1, W == 2 ? 2 : 0>(R, Q, reps, sbase, wx, rx, p);
  if constexpr (NW >= 2) {
    if (k == 8) exchange<NW, GWW, MW, 2, 0>(R, Q, reps, sbase, wx, rx, p);
    else if (k == 9) exchange<NW, GWW, MW, 2, 1>(R, Q, reps, sbase, wx, rx, p);
    else if (W == 2 && k == 10) exchange<NW, GWW, MW, 2, W == 2 ? 2 : 0>(R, Q, reps, sbase, wx, rx, p);
    else if (W == 1 && k == 11) exchange<NW, GWW, MW, 2, W == 1 ? 3 : 0>(R, Q, reps, sbase, wx, rx, p);
  }
  if constexpr (NW >= 4) {
    if (k == 16) exchange<NW, GWW, MW, 4, 0>(R, Q, reps, sbase, wx, rx, p);
    else if (k == 17) exchange<NW, GWW, MW, 4, 1>(R, Q, reps, sbase, wx, rx, p);
    else if (W == 2 && k == 18) exchange<NW, GWW, MW, 4, W == 2 ? 2 : 0>(R, Q, reps, sbase, wx, rx, p);
    else if (W == 1 && k == 19) exchange<NW, GWW, MW, 4, W == 1 ? 3 : 0>(R, Q, reps, sbase, wx, rx, p);
  }
}

template <int W, int NW>
__device__ __forceinline__ void exchange_w(uint32_t (&R)[NW], uint32_t (&Q)[NW], int reps,
                                           uint32_t sbase, uint32_t wx, uint32_t rx,
                                           const RegsPlan& p) {
  const int k = p.wr_gw * 4 + p.wr_mat;
  if (k == 4) exchange_r<W, NW, 1, 0>(R, Q, reps, sbase, wx, rx, p);
  else if (k == 5) exchange_r<W, NW, 1, 1>(R, Q, reps, sbase, wx, rx, p);
  else if (W == 2 && k == 6) exchange_r<W, NW, 1, W == 2 ? 2 : 0>(R, Q, reps, sbase, wx, rx, p);
  else if (W == 1 && k == 7) exchange_r<W, NW, 1, W == 1 ? 3 : 0>(R, Q, reps, sbase, wx, rx, p);
  if constexpr (NW >= 2) {
    if (k == 8) exchange_r<W, NW, 2, 0>(R, Q, reps, sbase, wx, rx, p);
    else if (k == 9) exchange_r<W, NW, 2, 1>(R, Q, reps, sbase, wx, rx, p);
    else if (W == 2 && k == 10) exchange_r<W, NW, 2, W == 2 ? 2 : 0>(R, Q, reps, sbase, wx, rx, p);
    else if (W == 1 && k == 11) exchange_r<W, NW, 2, W == 1 ? 3 : 0>(R, Q, reps, sbase, wx, rx, p);
  }
  if constexpr (NW >= 4) {
    if (k == 16) exchange_r<W, NW, 4, 0>(R, Q, reps, sbase, wx, rx, p);
    else if (k == 17) exchange_r<W, NW, 4, 1>(R, Q, reps, sbase, wx, rx, p);
    else if (W == 2 && k == 18) exchange_r<W, NW, 4, W == 2 ? 2 : 0>(R, Q, reps, sbase, wx, rx, p);
    else if (W == 1 && k == 19) exchange_r<W, NW, 4, W == 1 ? 3 : 0>(R, Q, reps, sbase, wx, rx, p);
  }
}

template <int W, int NW>
__global__ void __launch_bounds__(256) convert_regs_kernel(const __grid_constant__ RegsPlan p,
                                                           const uint8_t* __restrict__ src,
                                                           uint8_t* __restrict__ dst, int reps,
                                                           long long* __restrict__ cycles) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int TB = NW * 4;  // bytes per thread
  const int tid = threadIdx.x;
  const int tbits = 5 + p.nw;
  uint32_t wx = 0, rx = 0;
#pragma unroll
  for (int b = 0; b < LL_MAX_TBITS; ++b) {
    if (b < tbits && ((tid >> b) & 1)) {
      wx ^= p.sw_thr[b];
      rx ^= p.sr_thr[b];
    }
  }
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  for (int64_t t = blockIdx.x; t < p.n_tiles; t += gridDim.x) {
    const uint8_t* sp = src + t * p.tile_bytes + (int64_t)tid * TB;
    uint8_t* dp = dst + t * p.tile_bytes + (int64_t)tid * TB;
    uint32_t R[NW];
    if constexpr (TB >= 16) {
#pragma unroll
      for (int u = 0; u < NW / 4; ++u) {
        const uint4 v = ldg_stream(sp + 16 * u);
        R[4 * u] = v.x; R[4 * u + 1] = v.y; R[4 * u + 2] = v.z; R[4 * u + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int u = 0; u < NW; ++u) R[u] = __ldg(reinterpret_cast<const uint32_t*>(sp) + u);
    }
    for (int s = 0; s < p.n_swaps; ++s) apply_swap<W, NW>(R, p.swap_a[s], p.swap_b[s]);
    for (int s = 0; s < p.n_wsw; ++s) swap_word_bits<NW>(R, p.wsw_a[s], p.wsw_b[s]);
    uint32_t Q[NW];
    long long c0 = 0;
    if (cycles && tid == 0) c0 = clock64();
    exchange_w<W, NW>(R, Q, reps, sbase, wx, rx, p);
    if (cycles && tid == 0 && t == blockIdx.x) cycles[blockIdx.x] = clock64() - c0;
    for (int s = p.n_rsw - 1; s >= 0; --s) swap_word_bits<NW>(Q, p.rsw_a[s], p.rsw_b[s]);
    if constexpr (TB >= 16) {
#pragma unroll
      for (int u = 0; u < NW / 4; ++u) stg_stream(dp + 16 * u, make_uint4(Q[4 * u], Q[4 * u + 1], Q[4 * u + 2], Q[4 * u + 3]));
    } else {
#pragma unroll
      for (int u = 0; u < NW; ++u) reinterpret_cast<uint32_t*>(dp)[u] = Q[u];
    }
  }
}

template <int W, int NW>
static cudaError_t launch_regs_t(const RegsPlan& p, const void* src, void* dst, int max_ctas,
                                 int reps, long long* cycles, cudaStream_t st) {
  auto k = convert_regs_kernel<W, NW>;
  const int threads = 32 << p.nw;
  const size_t smem = (size_t)p.tile_bytes;
  if (smem > 200 * 1024) return cudaErrorInvalidConfiguration;
  const int occ = cached_occupancy((const void*)k, threads, smem, -1);
  if (occ <= 0) return cudaErrorInvalidConfiguration;
  int64_t grid = std::min<int64_t>(p.n_tiles, (int64_t)occ * num_sms() * 8);
  if (max_ctas > 0) grid = std::min<int64_t>(grid, max_ctas);
  if (grid <= 0) return cudaSuccess;
  k<<<(unsigned)grid, threads, smem, st>>>(p, (const uint8_t*)src, (uint8_t*)dst, reps, cycles);
  return cudaGetLastError();
}

template <int W>
static cudaError_t launch_regs_w(const RegsPlan& p, const void* src, void* dst, int max_ctas,
                                 int reps, long long* cycles, cudaStream_t st) {
  switch (p.nwords) {
    case 1: return launch_regs_t<W, 1>(p, src, dst, max_ctas, reps, cycles, st);
    case 2: return launch_regs_t<W, 2>(p, src, dst, max_ctas, reps, cycles, st);
    case 4: return launch_regs_t<W, 4>(p, src, dst, max_ctas, reps, cycles, st);
    case 8: return launch_regs_t<W, 8>(p, src, dst, max_ctas, reps, cycles, st);
    case 16: return launch_regs_t<W, 16>(p, src, dst, max_ctas, reps, cycles, st);
    case 32: return launch_regs_t<W, 32>(p, src, dst, max_ctas, reps, cycles, st);
    case 64: return launch_regs_t<W, 64>(p, src, dst, max_ctas, reps, cycles, st);
  }
  return cudaErrorNotSupported;
}

cudaError_t launch_convert_regs(const RegsPlan& p, int w, const void* src, void* dst,
                                int max_ctas, int reps, long long* cycles, cudaStream_t st) {
  if (reps < 1) return cudaErrorInvalidValue;
  switch (w) {
    case 1: return launch_regs_w<1>(p, src, dst, max_ctas, reps, cycles, st);
    case 2: return launch_regs_w<2>(p, src, dst, max_ctas, reps, cycles, st);
    case 4: return launch_regs_w<4>(p, src, dst, max_ctas, reps, cycles, st);
  }
  return cudaErrorNotSupported;
}

}  // namespace ll
