// kernel_async.cu -- cp.async-fed shared-memory conversion kernel and launcher.
#include "device_common.cuh"

namespace ll {

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

template <int W, int NV, int NS>
static cudaError_t launch_async_p(const SmemPlan& p, const void* src, void* dst, int max_ctas,
                                  cudaStream_t st, const TileRange& rg) {
  auto k = convert_async_kernel<W, NV, NS>;
  const int threads = 256;
  const int gpc = (threads / 32) >> p.gw;
  const size_t smem = (size_t)gpc * NS * p.tile_bytes;
  if (smem > 200 * 1024) return cudaErrorInvalidConfiguration;
  const int occ_cache = cached_occupancy((const void*)k, threads, smem, -1);
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

}  // namespace ll
