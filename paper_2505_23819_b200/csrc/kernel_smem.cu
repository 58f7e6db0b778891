// kernel_smem.cu -- shared-memory conversion kernel (paper's optimal swizzle) and launcher.
#include "device_common.cuh"

#ifndef LL_UP_PREFETCH
#define LL_UP_PREFETCH 1  // upcast: load the next tile's scales with its data
#endif
#ifndef LL_UP_V8
#define LL_UP_V8 1  // upcast stores: each lane writes its own 64 B as two 256-bit STG (sm_100)
#endif
#ifndef LL_UP_MINB
#define LL_UP_MINB 2  // resident CTAs the upcast kernel is compiled for (sweep: 2 > 3 > 4 > 1)
#endif
// Resident CTAs (256 threads) the conversion kernel is compiled for, i.e. a
// register cap of 64 (4 CTAs) / 80 (3 CTAs) per thread.  Without it ptxas
// takes 72-116 registers and the occupancy drop costs 3-11 % of HBM bandwidth
// (cfg2/3/5 measured against the 64/80-register build of the same kernel).
// 4-byte granules (G = 4) keep the uncapped allocation: capped, they spill.
#ifndef LL_SMEM_MINB
#define LL_SMEM_MINB 4   // NV <= 4 vectors per thread
#endif
#ifndef LL_SMEM_MINB8
#define LL_SMEM_MINB8 3  // NV = 8
#endif

namespace ll {

// UP: fused mxfp4 dequantisation (NEXT #1; W == 1): every
// destination byte (two E2M1 values, even k in the low nibble) becomes two
// bf16 = e2m1 x 2^(E8M0 scale - 127), computed exactly in fp32 (the products
// are representable; overflow -> inf, scale 0xFF -> NaN) and truncated to bf16.
__device__ __forceinline__ uint32_t mx_scale_f32(uint32_t x) {
  return x == 255u ? 0x7FC00000u : (x == 0u ? 0x00400000u : (x << 23));
}
__device__ __forceinline__ uint32_t e2m1_f32(uint32_t n) {
  const uint32_t e = (n >> 1) & 3u, m = n & 1u;
  const uint32_t b = e ? (((e + 126u) << 23) | (m << 22)) : (m ? 0x3F000000u : 0u);
  return b | ((n & 8u) << 28);
}

// bf16 bits of the e2m1 magnitudes 0, 0.5, 1, 1.5, 2, 3, 4, 6 (index = the
// nibble's low 3 bits), split into low-byte and high-byte permute tables
constexpr uint32_t kE2M1Lo0 = 0xC0800000u, kE2M1Lo1 = 0xC0804000u;
constexpr uint32_t kE2M1Hi0 = 0x3F3F3F00u, kE2M1Hi1 = 0x40404040u;
// exact here: both operands are bf16 and the product is a normal number
__device__ __forceinline__ uint32_t bf16x2_mul(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

template <int W, int NV, int G, bool PIPE, bool PAD, bool UP = false>
__global__ void __launch_bounds__(256, UP ? LL_UP_MINB : (G < 8 ? 1 : (NV >= 8 ? LL_SMEM_MINB8 : LL_SMEM_MINB))) convert_smem_kernel(const __grid_constant__ SmemPlan p,
                                                           const uint8_t* __restrict__ src,
                                                           uint8_t* __restrict__ dst,
                                                           int64_t n_groups, TileRange rg,
                                                           const uint8_t* __restrict__ scales) {
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

  uint32_t ld_off = 0, st_off = 0, swx = 0, srx = 0, sc_off = 0;
#pragma unroll
  for (int b = 0; b < LL_MAX_TBITS; ++b) {
    if (b < tbits && ((tb >> b) & 1)) {
      ld_off += p.ld_thr[b];
      st_off += p.st_thr[b];
      swx ^= p.sw_thr[b];
      srx ^= p.sr_thr[b];
      if (UP) sc_off += p.sc_thr[b];
    }
  }
  const uint8_t* sthr = src + ld_off - rg.src_shift;
  uint8_t* dthr = dst + st_off - rg.dst_shift;
  const int n_bits = p.tile.n_bits;
  const int n_tab = p.tile.n_tab;
  const int64_t rmask = (int64_t(1) << n_bits) - 1;
  int64_t sct = 0;  // scale-index contribution of the current tile (UP)
  auto tile_off = [&](int64_t t, int64_t& so, int64_t& dof) {
    const int64_t inst = t >> n_bits;
    const int64_t r = t & rmask;
    so = inst * p.tile.batch_stride_src;
    dof = inst * p.tile.batch_stride_dst;
    if (UP) sct = 0;
#pragma unroll
    for (int k = 0; k < LL_MAX_TAB; ++k) {
      if (k < n_tab) {
        const TileTab& e = p.tile.tab[k][(int)((r >> (k * LL_TAB_BITS)) & ((1 << LL_TAB_BITS) - 1))];
        so += e.src;
        dof += e.dst;
        if (UP) sct += e.sc;
      }
    }
  };

  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem) + group * 2 * p.tile_bytes;
  uint32_t buf = 0;
  const int ga = p.gsel_a, gb = p.gsel_b;
  const int64_t n_tiles = rg.t1;

  // UP: the 4 distinct scales of each destination vector, packed per vector,
  // and a bit per vector when all four give normal products (fast path);
  // loaded together with the tile so their latency overlaps the staging
  uint32_t PK[UP ? NV : 1];
  uint32_t fastm = 0;
  auto load_scales = [&]() {
    if constexpr (UP) {
      fastm = 0;
      if (p.sc_nz <= 2) {
#pragma unroll
        for (int u = 0; u < NV; ++u) {
          const uint8_t* scp = scales + sct + sc_off + p.sc_vec[u];
          const uint32_t s0 = __ldg(scp), s1 = __ldg(scp + p.sc_c[0]), s2 = __ldg(scp + p.sc_c[1]),
                         s3 = __ldg(scp + p.sc_c[0] + p.sc_c[1]);
          PK[u] = s0 | (s1 << 8) | (s2 << 16) | (s3 << 24);
          // all four scales in [2, 252]: every product is a normal number
          const bool ok = (s0 - 2u < 251u) & (s1 - 2u < 251u) & (s2 - 2u < 251u) & (s3 - 2u < 251u);
          fastm |= (uint32_t)ok << u;
        }
      }
    }
  };

  uint32_t R[NW];
  int64_t so, dof;
  int64_t t = rg.t0 + gid;
  if (PIPE && t < n_tiles) {
    tile_off(t, so, dof);
    load_tile<NV>(R, sthr + so, p.ld_vec);
    if (LL_UP_PREFETCH) load_scales();
  }
  for (; t < n_tiles; t += n_groups) {
    if (!PIPE) tile_off(t, so, dof);
    if (!PIPE) load_tile<NV>(R, sthr + so, p.ld_vec);
    if (!PIPE || !LL_UP_PREFETCH) load_scales();
    const int64_t dcur = dof;
    const int64_t sct_cur = sct;
    uint32_t PKc[UP ? NV : 1];
#pragma unroll
    for (int u = 0; u < (UP ? NV : 1); ++u) PKc[u] = PK[u];
    const uint32_t fastc = fastm;
    for (int s = 0; s < p.n_swaps; ++s) apply_swap<W, NW>(R, p.swap_a[s], p.swap_b[s]);
    sts_dispatch<NW, GW, PAD>(ga, gb, R, sbase + buf, swx, p.sw_gran);
    if (PIPE) {
      const int64_t tn = t + n_groups;
      if (tn < n_tiles) {
        tile_off(tn, so, dof);
        load_tile<NV>(R, sthr + so, p.ld_vec);
        if (LL_UP_PREFETCH) load_scales();
      }
    }
    group_sync(gw, group);
    uint32_t Q[NW];
#pragma unroll
    for (int j = 0; j < NG; ++j) {
      const uint32_t o = srx ^ p.sr_gran[j];
      lds<G>(sbase + buf + (PAD ? pad_off(o) : o), &Q[j * GW]);
    }
    if constexpr (UP) {
      // fused dequantisation: 16 packed bytes -> 32 bf16 (64 bytes) per vector.
      // Lanes l and l^1 form a pair: every store instruction of the pair
      // fills one whole 32-byte sector (the even lane the first 16 bytes, the
      // odd lane the next 16) -- 16 bytes per lane at a 64-byte stride would
      // leave each sector half written per instruction, which runs at half
      // the HBM write rate (tools/bwprobe.cu: r1w4_lane vs r1w4_coal).  The
      // pair trades packed input words (4 bytes -> one 16-byte output chunk)
      // and scales: the even lane converts chunks 0 and 2 of both lanes'
      // vectors, the odd lane chunks 1 and 3.
      const int64_t dbyte = (int64_t)st_off - rg.dst_shift + dcur;
      const int64_t scur = sct_cur + sc_off;
#if LL_UP_V8
      // sm_100 256-bit stores: every lane writes whole 32-byte sectors of its
      // own 64 output bytes, so no lane pairing is needed
#pragma unroll
      for (int u = 0; u < NV; ++u) {
        const uint32_t pk = PKc[u];
        uint8_t* op = dst + 4 * (dbyte + p.st_vec[u]);
        uint32_t o8[2][8];
        if ((fastc >> u) & 1u) {
          const uint32_t plo = (pk << 7) & 0x80808080u, phi = (pk >> 1) & 0x7F7F7F7Fu;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t wq = Q[4 * u + q];
            const uint32_t m = wq & 0x77777777u, mh = m >> 16, x = wq & 0x88888888u;
            const uint32_t L01 = __byte_perm(kE2M1Lo0, kE2M1Lo1, m), H01 = __byte_perm(kE2M1Hi0, kE2M1Hi1, m);
            const uint32_t L23 = __byte_perm(kE2M1Lo0, kE2M1Lo1, mh), H23 = __byte_perm(kE2M1Hi0, kE2M1Hi1, mh);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int e = 4 * q + k;
              const uint32_t mag = __byte_perm(k < 2 ? L01 : L23, k < 2 ? H01 : H23, (k & 1) ? 0x7362 : 0x5140);
              const uint32_t t = __byte_perm(x, 0u, 0x4440 | k) * 0x01001000u;  // bits 3,7 -> 15,31
              const uint32_t v = mag | (t & 0x80008000u);
              o8[q >> 1][4 * (q & 1) + k] = bf16x2_mul(v, __byte_perm(plo, phi, p.sc_sel[e]));
            }
          }
        } else {
          const uint8_t* scp = scales + scur + p.sc_vec[u];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const uint32_t byte = (Q[4 * u + (e >> 2)] >> ((e & 3) * 8)) & 0xFFu;
            const uint32_t sb = p.sc_nz <= 2 ? (pk >> (8 * p.sc_slot[e])) & 0xFFu
                                             : (uint32_t)__ldg(scp + p.sc_e[e]);
            const float sf = __uint_as_float(mx_scale_f32(sb));
            const uint32_t lo = __float_as_uint(__fmul_rn(__uint_as_float(e2m1_f32(byte & 15u)), sf));
            const uint32_t hi = __float_as_uint(__fmul_rn(__uint_as_float(e2m1_f32(byte >> 4)), sf));
            o8[e >> 3][e & 7] = sb == 255u ? 0x7FC07FC0u : ((hi & 0xFFFF0000u) | (lo >> 16));
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
          asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(op + 32 * h),
                       "r"(o8[h][0]), "r"(o8[h][1]), "r"(o8[h][2]), "r"(o8[h][3]), "r"(o8[h][4]),
                       "r"(o8[h][5]), "r"(o8[h][6]), "r"(o8[h][7])
                       : "memory");
      }
#else
      const bool odd = lane & 1;
      const uint32_t fpair = fastc & __shfl_xor_sync(0xFFFFFFFFu, fastc, 1);
#pragma unroll
      for (int u = 0; u < NV; ++u) {
        const uint32_t pk = PKc[u];
        const uint32_t w0 = Q[4 * u], w1 = Q[4 * u + 1], w2 = Q[4 * u + 2], w3 = Q[4 * u + 3];
        const uint32_t r0 = __shfl_xor_sync(0xFFFFFFFFu, odd ? w0 : w1, 1);
        const uint32_t r1 = __shfl_xor_sync(0xFFFFFFFFu, odd ? w2 : w3, 1);
        const uint32_t pkp = __shfl_xor_sync(0xFFFFFFFFu, pk, 1);
        uint8_t* op = dst + 4 * (dbyte + p.st_vec[u]);
        if ((fpair >> u) & 1u) {
          // chunk q of this lane's work: the lane's own vector (A/B) and word
          uint8_t* opp = op + (odd ? -4 * (int64_t)p.st_thr[0] : 4 * (int64_t)p.st_thr[0]);
          uint8_t* oA = (odd ? opp : op) + (odd ? 16 : 0);
          uint8_t* oB = (odd ? op : opp) + (odd ? 16 : 0);
          const uint32_t in[4] = {odd ? r0 : w0, odd ? r1 : w2, odd ? w1 : r0, odd ? w3 : r1};
          // the odd lane's chunks are the even lane's byte indices + 4: the
          // same selectors apply after permuting the packed scales
          const uint32_t psel = odd ? p.sc_psel : 0x3210u;
          const uint32_t pkA = __byte_perm(odd ? pkp : pk, 0u, psel);
          const uint32_t pkB = __byte_perm(odd ? pk : pkp, 0u, psel);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t pq = q < 2 ? pkA : pkB;
            const uint32_t plo = (pq << 7) & 0x80808080u, phi = (pq >> 1) & 0x7F7F7F7Fu;
            const uint32_t wq = in[q];
            const uint32_t m = wq & 0x77777777u, mh = m >> 16, x = wq & 0x88888888u;
            const uint32_t L01 = __byte_perm(kE2M1Lo0, kE2M1Lo1, m), H01 = __byte_perm(kE2M1Hi0, kE2M1Hi1, m);
            const uint32_t L23 = __byte_perm(kE2M1Lo0, kE2M1Lo1, mh), H23 = __byte_perm(kE2M1Hi0, kE2M1Hi1, mh);
            uint32_t o4[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int e = 8 * (q & 1) + k;
              const uint32_t mag = __byte_perm(k < 2 ? L01 : L23, k < 2 ? H01 : H23, (k & 1) ? 0x7362 : 0x5140);
              const uint32_t t = __byte_perm(x, 0u, 0x4440 | k) * 0x01001000u;  // bits 3,7 -> 15,31
              const uint32_t v = mag | (t & 0x80008000u);
              o4[k] = bf16x2_mul(v, __byte_perm(plo, phi, p.sc_sel[e]));
            }
            stg_stream((q < 2 ? oA : oB) + 32 * (q & 1), make_uint4(o4[0], o4[1], o4[2], o4[3]));
          }
        } else {
          const uint8_t* scp = scales + scur + p.sc_vec[u];
          uint32_t ow[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const uint32_t byte = (Q[4 * u + (e >> 2)] >> ((e & 3) * 8)) & 0xFFu;
            const uint32_t sb = p.sc_nz <= 2 ? (pk >> (8 * p.sc_slot[e])) & 0xFFu
                                             : (uint32_t)__ldg(scp + p.sc_e[e]);
            const float sf = __uint_as_float(mx_scale_f32(sb));
            const uint32_t lo = __float_as_uint(__fmul_rn(__uint_as_float(e2m1_f32(byte & 15u)), sf));
            const uint32_t hi = __float_as_uint(__fmul_rn(__uint_as_float(e2m1_f32(byte >> 4)), sf));
            // NaN scale -> the canonical bf16 quiet NaN 0x7FC0 for both values
            ow[e] = sb == 255u ? 0x7FC07FC0u : ((hi & 0xFFFF0000u) | (lo >> 16));
          }
#pragma unroll
          for (int q = 0; q < 4; ++q)
            stg_stream(op + 16 * q, make_uint4(ow[4 * q], ow[4 * q + 1], ow[4 * q + 2], ow[4 * q + 3]));
        }
      }
#endif
    } else {
      uint8_t* dp = dthr + dcur;
#pragma unroll
      for (int u = 0; u < NV; ++u)
        stg_stream(dp + p.st_vec[u], make_uint4(Q[4 * u + 0], Q[4 * u + 1], Q[4 * u + 2], Q[4 * u + 3]));
    }
    buf ^= p.tile_bytes;
  }
}

template <int W, int NV, int G, bool PIPE, bool PAD, bool UP = false>
static cudaError_t launch_smem_p(const SmemPlan& p, const void* src, void* dst, int max_ctas,
                                 cudaStream_t st, const TileRange& rg,
                                 const uint8_t* scales = nullptr) {
  auto k = convert_smem_kernel<W, NV, G, PIPE, PAD, UP>;
  const int threads = 256;
  const int gpc = (threads / 32) >> p.gw;
  const size_t smem = (size_t)gpc * 2 * p.tile_bytes;  // tile_bytes includes any padding
  const int occ_cache = cached_occupancy((const void*)k, threads, smem, knobs().carveout);
  if (occ_cache <= 0) return cudaErrorInvalidConfiguration;
  const int64_t n_tiles = rg.t1 - rg.t0;
  if (n_tiles <= 0) return cudaSuccess;
  // tile groups: n_tiles / tpg (the hardware block scheduler balances the
  // tail), or the resident capacity when tpg = 0 (persistent)
  const int tpg = UP ? knobs().up_tpg : knobs().tpg;
  int64_t groups = tpg > 0 ? (n_tiles + tpg - 1) / tpg : (int64_t)occ_cache * num_sms() * gpc;
  if (max_ctas > 0) groups = std::min<int64_t>(groups, (int64_t)max_ctas * gpc);
  groups = std::max<int64_t>(1, std::min<int64_t>(groups, n_tiles));
  const int64_t grid = (groups + gpc - 1) / gpc;
  if (grid > 0x7fffffff) return cudaErrorInvalidConfiguration;
  k<<<(unsigned)grid, threads, smem, st>>>(p, (const uint8_t*)src, (uint8_t*)dst, groups, rg,
                                           scales);
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

cudaError_t launch_mxfp4_upcast(const SmemPlan& p, int nv, int g, const void* src, void* dst,
                                const uint8_t* scales, int max_ctas, cudaStream_t st,
                                const TileRange& rg) {
#define LL_UCASE(NV_, G_) \
  if (nv == NV_ && g == G_)  \
    return launch_smem_p<1, NV_, G_, true, false, true>(p, src, dst, max_ctas, st, rg, scales);
  LL_UCASE(1, 4) LL_UCASE(1, 8) LL_UCASE(1, 16) LL_UCASE(2, 4) LL_UCASE(2, 8) LL_UCASE(2, 16)
  LL_UCASE(4, 4) LL_UCASE(4, 8) LL_UCASE(4, 16) LL_UCASE(8, 4) LL_UCASE(8, 8) LL_UCASE(8, 16)
#undef LL_UCASE
  return cudaErrorNotSupported;
}

}  // namespace ll
