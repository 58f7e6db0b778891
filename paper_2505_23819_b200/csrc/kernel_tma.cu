// kernel_tma.cu -- TMA-fed shared-memory conversion kernel (LL_PATH_SMEM_TMA)
// and its launcher (tensor-map encoding through the driver entry point).
//
// Per tile group (2^gw warps) an NS-stage ring of shared-memory tiles: the
// group's leader thread issues one cp.async.bulk.tensor per tile (the source
// tile is one box of the planner's <= 5-D view of the source buffer, landing
// densely in shared memory under the hardware swizzle the planner chose) and
// arms the stage's mbarrier with the tile's byte count; the readers wait on
// the mbarrier's phase, load their 16-byte source granules (conflict-free by
// the planner's lane choice), permute registers into destination vectors
// (prmt / compile-time word selection) and store them with st.global.cs.v4.
// No thread issues a global load.
#include <cuda.h>

#include <mutex>

#include "device_common.cuh"

namespace ll {

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "LL_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra LL_WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load(uint32_t sdst, const CUtensorMap* tm, const int32_t* c,
                                         int nd, uint32_t bar) {
  const uint64_t tp = reinterpret_cast<uint64_t>(tm);
  switch (nd) {
    case 1:
      asm volatile(
          "cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];" ::"r"(sdst),
          "l"(tp), "r"(c[0]), "r"(bar)
          : "memory");
      break;
    case 2:
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(sdst),
          "l"(tp), "r"(c[0]), "r"(c[1]), "r"(bar)
          : "memory");
      break;
    case 3:
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(sdst),
          "l"(tp), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(bar)
          : "memory");
      break;
    case 4:
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(sdst),
          "l"(tp), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(bar)
          : "memory");
      break;
    default:
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(sdst),
          "l"(tp), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(bar)
          : "memory");
      break;
  }
}

__device__ __forceinline__ void tma_store(const CUtensorMap* tm, const int32_t* c, int nd,
                                          uint32_t ssrc) {
  const uint64_t tp = reinterpret_cast<uint64_t>(tm);
  switch (nd) {
    case 1:
      asm volatile("cp.async.bulk.tensor.1d.global.shared::cta.bulk_group [%0, {%1}], [%2];" ::"l"(tp),
                   "r"(c[0]), "r"(ssrc)
                   : "memory");
      break;
    case 2:
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(tp),
                   "r"(c[0]), "r"(c[1]), "r"(ssrc)
                   : "memory");
      break;
    case 3:
      asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(tp),
                   "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(ssrc)
                   : "memory");
      break;
    case 4:
      asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(tp),
                   "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(ssrc)
                   : "memory");
      break;
    default:
      asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(tp),
                   "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(ssrc)
                   : "memory");
      break;
  }
}

__device__ __forceinline__ void tile_coords(int64_t e, const TmaDesc& td, int32_t* c) {
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    if (i < td.ndim) {
      const int64_t v = e >> td.shift[i];
      c[i] = (int32_t)(i + 1 < td.ndim ? (v & ((int64_t(1) << td.size_bits[i]) - 1)) : v);
    } else {
      c[i] = 0;
    }
  }
}

#define LL_TMA_MAX_GROUPS 8
#define LL_TMA_MAX_STAGES 4

template <int W, int NV, int NS>
__global__ void __launch_bounds__(256) convert_tma_kernel(const __grid_constant__ SmemPlan p,
                                                          const __grid_constant__ CUtensorMap tmap,
                                                          const TmaDesc td,
                                                          uint8_t* __restrict__ dst,
                                                          int64_t n_groups, TileRange rg) {
  constexpr int NW = NV * 4;
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[LL_TMA_MAX_GROUPS][NS];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int gw = p.gw;
  const int group = warp >> gw;
  const int tb = lane | ((warp & ((1 << gw) - 1)) << 5);
  const int gpc = (blockDim.x >> 5) >> gw;
  const int tbits = 5 + gw;
  const int64_t gid = (int64_t)blockIdx.x * gpc + group;
  if (gid >= n_groups) return;  // whole idle groups only (named barriers stay consistent)
  uint32_t st_off = 0, srx = 0;
#pragma unroll
  for (int b = 0; b < LL_MAX_TBITS; ++b) {
    if (b < tbits && ((tb >> b) & 1)) {
      st_off += p.st_thr[b];
      srx ^= p.sr_thr[b];
    }
  }
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
  // stage buffers aligned to 1024 B (the 128-byte swizzle pattern repeats
  // every 1024 bytes of shared-memory address)
  const uint32_t sraw = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t sbase = ((sraw + 1023u) & ~1023u) + group * NS * tb_bytes;
  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&bars[group][0]);
  const bool leader = tb == 0;
  if (leader) {
#pragma unroll
    for (int s = 0; s < NS; ++s) mbar_init(bar0 + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  group_sync(gw, group);
  constexpr int lw = ilog2(W);
  auto issue = [&](int64_t t, int stg) {
    if (leader && t < rg.t1) {
      int64_t so, dof;
      tile_off(t, so, dof);
      const int64_t e = (so - rg.src_shift) >> lw;  // element offset of the tile origin
      int32_t c[5];
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        if (i < td.ndim) {
          const int64_t v = e >> td.shift[i];
          c[i] = (int32_t)(i + 1 < td.ndim ? (v & ((int64_t(1) << td.size_bits[i]) - 1)) : v);
        } else {
          c[i] = 0;
        }
      }
      const uint32_t bar = bar0 + 8 * stg;
      mbar_expect_tx(bar, tb_bytes);
      tma_load(sbase + stg * tb_bytes, &tmap, c, td.ndim, bar);
    }
  };
  const int64_t t_first = rg.t0 + gid;
#pragma unroll
  for (int s = 0; s < NS - 1; ++s) issue(t_first + s * n_groups, s);
  int stage = 0;
  uint32_t phase = 0;  // bit s: parity of stage s's next completion
  const int ga = p.gsel_a, gb = p.gsel_b;
  for (int64_t t = t_first; t < rg.t1; t += n_groups) {
    mbar_wait(bar0 + 8 * stage, (phase >> stage) & 1u);
    phase ^= 1u << stage;
    // every reader of the group is done with the stage read last iteration;
    // their generic-proxy reads ordered before the leader's TMA refill
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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
}

// TMA load + TMA store (LL_PATH_SMEM_TMA_STORE): as convert_tma_kernel, but
// the readers write their destination vectors into one of two destination
// images (STS.128, conflict-free by the planner's lanes), fence the generic
// proxy against the async proxy, and the leader stores the image with one
// cp.async.bulk.tensor (bulk group); the image is rewritten only after that
// store has finished reading it (cp.async.bulk.wait_group.read 1).
template <int W, int NV, int NS>
__global__ void __launch_bounds__(256) convert_tma_store_kernel(
    const __grid_constant__ SmemPlan p, const __grid_constant__ CUtensorMap tsrc,
    const __grid_constant__ CUtensorMap tdst, const TmaDesc tds, const TmaDesc tdd,
    int64_t n_groups, TileRange rg) {
  constexpr int NW = NV * 4;
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[LL_TMA_MAX_GROUPS][NS];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int gw = p.gw;
  const int group = warp >> gw;
  const int tb = lane | ((warp & ((1 << gw) - 1)) << 5);
  const int gpc = (blockDim.x >> 5) >> gw;
  const int tbits = 5 + gw;
  const int64_t gid = (int64_t)blockIdx.x * gpc + group;
  if (gid >= n_groups) return;
  uint32_t swx = 0, srx = 0;
#pragma unroll
  for (int b = 0; b < LL_MAX_TBITS; ++b) {
    if (b < tbits && ((tb >> b) & 1)) {
      swx ^= p.sw_thr[b];
      srx ^= p.sr_thr[b];
    }
  }
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
  const uint32_t sraw = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t sbase = ((sraw + 1023u) & ~1023u) + group * (NS + 2) * tb_bytes;
  const uint32_t dbase = sbase + NS * tb_bytes;
  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&bars[group][0]);
  const bool leader = tb == 0;
  if (leader) {
#pragma unroll
    for (int s = 0; s < NS; ++s) mbar_init(bar0 + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  group_sync(gw, group);
  constexpr int lw = ilog2(W);
  auto issue = [&](int64_t t, int stg) {
    if (leader && t < rg.t1) {
      int64_t so, dof;
      tile_off(t, so, dof);
      int32_t c[5];
      tile_coords((so - rg.src_shift) >> lw, tds, c);
      const uint32_t bar = bar0 + 8 * stg;
      mbar_expect_tx(bar, tb_bytes);
      tma_load(sbase + stg * tb_bytes, &tsrc, c, tds.ndim, bar);
    }
  };
  const int64_t t_first = rg.t0 + gid;
#pragma unroll
  for (int s = 0; s < NS - 1; ++s) issue(t_first + s * n_groups, s);
  int stage = 0;
  uint32_t phase = 0, it = 0;
  const int ga = p.gsel_a, gb = p.gsel_b;
  for (int64_t t = t_first; t < rg.t1; t += n_groups, ++it) {
    mbar_wait(bar0 + 8 * stage, (phase >> stage) & 1u);
    phase ^= 1u << stage;
    if (leader) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    group_sync(gw, group);
    issue(t + (NS - 1) * n_groups, stage == 0 ? NS - 1 : stage - 1);
    uint32_t Q[NW];
    const uint32_t rb = sbase + stage * tb_bytes;
#pragma unroll
    for (int j = 0; j < NV; ++j) lds<16>(rb + (srx ^ p.sr_gran[j]), &Q[4 * j]);
    for (int s = 0; s < p.n_swaps; ++s) apply_swap<W, NW>(Q, p.swap_a[s], p.swap_b[s]);
    const uint32_t db = dbase + (it & 1u) * tb_bytes;
    sts_dispatch<NW, 4>(ga, gb, Q, db, swx, p.sw_gran);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    group_sync(gw, group);
    if (leader) {
      int64_t so, dof;
      tile_off(t, so, dof);
      int32_t c[5];
      tile_coords((dof - rg.dst_shift) >> lw, tdd, c);
      tma_store(&tdst, c, tdd.ndim, db);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    stage = stage == NS - 1 ? 0 : stage + 1;
  }
  if (leader) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ------------------------------------------------------------ tensor maps

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(f);
  });
  return fn;
}

// The tensor view of the caller's source slice: dim i spans element bits
// [shift[i], shift[i] + size_bits[i]); the top dim spans the rest of the slice.
static cudaError_t encode_src_map(CUtensorMap* tm, const TmaDesc& td, int w, const void* src,
                                  int64_t slice_elems) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  cuuint64_t gdim[5], gstride[5];
  cuuint32_t box[5], estr[5];
  for (int i = 0; i < td.ndim; ++i) {
    gdim[i] = i + 1 < td.ndim ? (cuuint64_t(1) << td.size_bits[i])
                              : (cuuint64_t)(slice_elems >> td.shift[i]);
    if (i > 0) gstride[i - 1] = (cuuint64_t)w << td.shift[i];
    box[i] = 1u << td.box_bits[i];
    estr[i] = 1;
  }
  if (gdim[td.ndim - 1] == 0) return cudaErrorInvalidValue;
  CUtensorMapDataType dt = w == 1   ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                           : w == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                           : w == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32
                                    : CU_TENSOR_MAP_DATA_TYPE_INT64;
  static const CUtensorMapSwizzle sw[4] = {CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                                           CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_SWIZZLE_128B};
  CUresult r = fn(tm, dt, (cuuint32_t)td.ndim, const_cast<void*>(src), gdim, gstride, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, sw[td.swizzle & 3],
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int W, int NV, int NS>
static cudaError_t launch_tma_p(const SmemPlan& p, const TmaDesc& td, const void* src, void* dst,
                                int max_ctas, cudaStream_t st, const TileRange& rg) {
  auto k = convert_tma_kernel<W, NV, NS>;
  const int threads = 256;
  const int gpc = (threads / 32) >> p.gw;
  const size_t smem = (size_t)gpc * NS * p.tile_bytes + 1024;
  if (smem > 220 * 1024) return cudaErrorInvalidConfiguration;
  const int occ_cache = cached_occupancy((const void*)k, threads, smem, -1);
  if (occ_cache <= 0) return cudaErrorInvalidConfiguration;
  const int64_t n_tiles = rg.t1 - rg.t0;
  if (n_tiles <= 0) return cudaSuccess;
  CUtensorMap tm;
  const int64_t slice_elems = n_tiles * (int64_t(p.tile_bytes) / W);
  cudaError_t e = encode_src_map(&tm, td, W, src, slice_elems);
  if (e != cudaSuccess) return e;
  // tiles per group: knob > 0; 0 = persistent; < 0 (default) = 4 tiles per
  // group when that still gives >= 8 waves of resident groups, else
  // persistent (sweep: cfg5 6739 GB/s at 4 vs 5932 persistent; cfg3, 4096
  // tiles of 32 KB, 5746 persistent vs 4844 at 4)
  const int64_t resident = (int64_t)occ_cache * num_sms() * gpc;
  int tpg = knobs().tma_tpg;
  if (tpg < 0) tpg = (n_tiles / 4 >= 8 * resident) ? 4 : 0;
  int64_t groups = tpg > 0 ? (n_tiles + tpg - 1) / tpg : resident;
  if (max_ctas > 0) groups = std::min<int64_t>(groups, (int64_t)max_ctas * gpc);
  groups = std::max<int64_t>(1, std::min<int64_t>(groups, n_tiles));
  const int64_t grid = (groups + gpc - 1) / gpc;
  if (grid > 0x7fffffff) return cudaErrorInvalidConfiguration;
  k<<<(unsigned)grid, threads, smem, st>>>(p, tm, td, (uint8_t*)dst, groups, rg);
  return cudaGetLastError();
}

template <int W, int NV, int NS>
static cudaError_t launch_tma_store_p(const SmemPlan& p, const TmaDesc& tds, const TmaDesc& tdd,
                                      const void* src, void* dst, int max_ctas, cudaStream_t st,
                                      const TileRange& rg) {
  auto k = convert_tma_store_kernel<W, NV, NS>;
  const int threads = 256;
  const int gpc = (threads / 32) >> p.gw;
  const size_t smem = (size_t)gpc * (NS + 2) * p.tile_bytes + 1024;
  if (smem > 220 * 1024) return cudaErrorInvalidConfiguration;
  const int occ_cache = cached_occupancy((const void*)k, threads, smem, -1);
  if (occ_cache <= 0) return cudaErrorInvalidConfiguration;
  const int64_t n_tiles = rg.t1 - rg.t0;
  if (n_tiles <= 0) return cudaSuccess;
  CUtensorMap ms, md;
  const int64_t slice_elems = n_tiles * (int64_t(p.tile_bytes) / W);
  cudaError_t e = encode_src_map(&ms, tds, W, src, slice_elems);
  if (e != cudaSuccess) return e;
  e = encode_src_map(&md, tdd, W, dst, slice_elems);
  if (e != cudaSuccess) return e;
  const int64_t resident = (int64_t)occ_cache * num_sms() * gpc;
  int tpg = knobs().tma_tpg;
  if (tpg < 0) tpg = (n_tiles / 4 >= 8 * resident) ? 4 : 0;
  int64_t groups = tpg > 0 ? (n_tiles + tpg - 1) / tpg : resident;
  if (max_ctas > 0) groups = std::min<int64_t>(groups, (int64_t)max_ctas * gpc);
  groups = std::max<int64_t>(1, std::min<int64_t>(groups, n_tiles));
  const int64_t grid = (groups + gpc - 1) / gpc;
  if (grid > 0x7fffffff) return cudaErrorInvalidConfiguration;
  k<<<(unsigned)grid, threads, smem, st>>>(p, ms, md, tds, tdd, groups, rg);
  return cudaGetLastError();
}

template <int W>
static cudaError_t launch_tma_store_w(const SmemPlan& p, const TmaDesc& tds, const TmaDesc& tdd,
                                      int nv, const void* src, void* dst, int max_ctas,
                                      cudaStream_t st, const TileRange& rg) {
  const int ns = knobs().tma_stages;
#define LL_TSCASE(NV_)                                                                          \
  if (nv == NV_) {                                                                              \
    if (ns <= 2) return launch_tma_store_p<W, NV_, 2>(p, tds, tdd, src, dst, max_ctas, st, rg); \
    return launch_tma_store_p<W, NV_, 3>(p, tds, tdd, src, dst, max_ctas, st, rg);              \
  }
  LL_TSCASE(1) LL_TSCASE(2) LL_TSCASE(4) LL_TSCASE(8)
#undef LL_TSCASE
  return cudaErrorNotSupported;
}

cudaError_t launch_convert_tma_store(const SmemPlan& p, const TmaDesc& tds, const TmaDesc& tdd,
                                     int w, int nv, const void* src, void* dst, int max_ctas,
                                     cudaStream_t st, const TileRange& rg) {
  if (tds.ndim < 1 || tds.ndim > 5 || tdd.ndim < 1 || tdd.ndim > 5) return cudaErrorInvalidValue;
  switch (w) {
    case 1: return launch_tma_store_w<1>(p, tds, tdd, nv, src, dst, max_ctas, st, rg);
    case 2: return launch_tma_store_w<2>(p, tds, tdd, nv, src, dst, max_ctas, st, rg);
    case 4: return launch_tma_store_w<4>(p, tds, tdd, nv, src, dst, max_ctas, st, rg);
    case 8: return launch_tma_store_w<8>(p, tds, tdd, nv, src, dst, max_ctas, st, rg);
  }
  return cudaErrorNotSupported;
}

template <int W>
static cudaError_t launch_tma_w(const SmemPlan& p, const TmaDesc& td, int nv, const void* src,
                                void* dst, int max_ctas, cudaStream_t st, const TileRange& rg) {
  const int ns = knobs().tma_stages;
#define LL_TCASE(NV_)                                                               \
  if (nv == NV_) {                                                                  \
    if (ns <= 2) return launch_tma_p<W, NV_, 2>(p, td, src, dst, max_ctas, st, rg); \
    if (ns == 3) return launch_tma_p<W, NV_, 3>(p, td, src, dst, max_ctas, st, rg); \
    return launch_tma_p<W, NV_, 4>(p, td, src, dst, max_ctas, st, rg);              \
  }
  LL_TCASE(1) LL_TCASE(2) LL_TCASE(4) LL_TCASE(8)
#undef LL_TCASE
  return cudaErrorNotSupported;
}

// The plan-compiled TMA kernels (jit.cpp) encode their maps here too.
cudaError_t encode_tma_map(void* tm, const TmaDesc& td, int w, const void* base, int64_t slice_elems) {
  return encode_src_map(reinterpret_cast<CUtensorMap*>(tm), td, w, base, slice_elems);
}

cudaError_t launch_convert_tma(const SmemPlan& p, const TmaDesc& td, int w, int nv,
                               const void* src, void* dst, int max_ctas, cudaStream_t st,
                               const TileRange& rg) {
  if (td.ndim < 1 || td.ndim > 5) return cudaErrorInvalidValue;
  switch (w) {
    case 1: return launch_tma_w<1>(p, td, nv, src, dst, max_ctas, st, rg);
    case 2: return launch_tma_w<2>(p, td, nv, src, dst, max_ctas, st, rg);
    case 4: return launch_tma_w<4>(p, td, nv, src, dst, max_ctas, st, rg);
    case 8: return launch_tma_w<8>(p, td, nv, src, dst, max_ctas, st, rg);
  }
  return cudaErrorNotSupported;
}

}  // namespace ll
