// kernel_shuffle.cu -- warp-shuffle conversion kernel and launcher.
#include "device_common.cuh"

namespace ll {

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

template <int W, int NV, bool PIPE>
static cudaError_t launch_shuffle_p(const ShufflePlan& p, const void* src, void* dst, int max_ctas,
                                    cudaStream_t st, const TileRange& rg) {
  auto k = convert_shuffle_kernel<W, NV, PIPE>;
  const int threads = 256;
  const int gpc = threads / 32;
  const int64_t n_tiles = rg.t1 - rg.t0;
  if (n_tiles <= 0) return cudaSuccess;
  const int occ_cache = cached_occupancy((const void*)k, threads, 0, -1);
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

}  // namespace ll
