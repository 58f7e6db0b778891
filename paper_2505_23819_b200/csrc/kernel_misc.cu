// kernel_misc.cu -- generic pull kernel, gather kernels, launch knobs.
#include "device_common.cuh"

namespace ll {

int planner_knob(const char* name, int dflt);   // planner.cpp

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
  // vectors per instance: a power of two, so batch / offset are shift / mask
  const int pb_shift = (p.nB >= VB) ? (p.nB - VB) : 0;
  const int64_t pb_mask = (int64_t(1) << pb_shift) - 1;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < p.n_vec;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = v >> pb_shift;
    const uint64_t h0 = (uint64_t)(v & pb_mask) << VB;
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
template <int W, bool V2 = false>
__global__ void __launch_bounds__(256) gather_direct_kernel(const __grid_constant__ GatherPlan p,
                                                            const uint8_t* __restrict__ src,
                                                            const int32_t* __restrict__ idx,
                                                            uint8_t* __restrict__ out,
                                                            int* __restrict__ err) {
  constexpr int NE = (V2 ? 32 : 16) / W;   // elements per thread per iteration
  constexpr int VB = ilog2(NE);
  using T = typename std::conditional<W == 1, uint8_t,
            typename std::conditional<W == 2, uint16_t,
            typename std::conditional<W == 4, uint32_t, uint64_t>::type>::type>::type;
  // vectors per instance: a power of two, so batch / offset are shift / mask
  const int pb_shift = p.nbits - VB;
  const int64_t pb_mask = (int64_t(1) << pb_shift) - 1;
  const uint32_t amask = (1u << p.ax_bits) - 1;
  const int64_t n_units = V2 ? (p.n_vec >> 1) : p.n_vec;
  // programmatic dependent launch (knob gather_pdl; a no-op otherwise):
  // wait for the preceding grid, let the next one launch at once
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n_units;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = v >> pb_shift;
    const uint64_t h0 = (uint64_t)(v & pb_mask) << VB;
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
      uint4 v4[NE * W / 16];
      uint32_t w[NE * W / 4];
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
    T* op = reinterpret_cast<T*>(out) + b * p.batch_stride + h0;
    if constexpr (V2) {
      // sm_100 256-bit store of the thread's 32 output bytes
      asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(op), "r"(o.w[0]),
                   "r"(o.w[1]), "r"(o.w[2]), "r"(o.w[3]), "r"(o.w[4]), "r"(o.w[5]), "r"(o.w[6]),
                   "r"(o.w[7])
                   : "memory");
    } else {
      *reinterpret_cast<uint4*>(op) = o.v4[0];
    }
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
template <int W, bool ALLC, int U = 1>
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
  // vectors per instance: a power of two, so batch / offset are shift / mask
  const int pb_shift = p.nbits - VB;
  const int64_t pb_mask = (int64_t(1) << pb_shift) - 1;
  const uint32_t amask = (1u << p.ax_bits) - 1;
  const int64_t nwarps_total = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n_wvec = p.n_vec >> 5;  // warps' worth of vectors
  const uint32_t clear32 = ~(uint32_t)p.axis_mask_buf;
  const int ybase = p.y_base;
  union V {
    uint4 v4;
    T e[NE];
    uint32_t w[4];
  };
  // U warp-vectors per iteration: all their loads are issued before the
  // first shuffle (U = 1: the plain loop)
  for (int64_t wv0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wv0 < n_wvec;
       wv0 += nwarps_total * U) {
    V sv[U];
    int32_t iv[U][NE];
    int64_t vv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t wv = wv0 + (int64_t)u * nwarps_total;
      vv[u] = -1;
      if (wv >= n_wvec) continue;  // warp-uniform
      const int64_t v = (wv << 5) | lane;
      vv[u] = v;
      const int64_t b = v >> pb_shift;
      const uint64_t h0 = (uint64_t)(v & pb_mask) << VB;
      sv[u].v4 = ldg_stream(src + (b * p.batch_stride + h0) * W);
      const int32_t* ip = idx + b * p.batch_stride + h0;
      if constexpr (NE >= 4) {
#pragma unroll
        for (int q = 0; q < NE / 4; ++q) {
          int4 t = __ldg(reinterpret_cast<const int4*>(ip) + q);
          iv[u][4 * q] = t.x; iv[u][4 * q + 1] = t.y; iv[u][4 * q + 2] = t.z; iv[u][4 * q + 3] = t.w;
        }
      } else {
#pragma unroll
        for (int q = 0; q < NE; ++q) iv[u][q] = __ldg(ip + q);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (vv[u] < 0) continue;
      const int64_t v = vv[u];
      const int64_t b = v >> pb_shift;
      const uint64_t h0 = (uint64_t)(v & pb_mask) << VB;
      V o;
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        // only the warp-local bits (VB + 5) of h* matter here: 32-bit arithmetic
        uint32_t i = (uint32_t)iv[u][e];
        if (p.check && i > amask) atomicExch(err, 1);
        i &= amask;
        const uint32_t hl = (((uint32_t)lane << VB) | (uint32_t)e) & clear32;
        const uint32_t hs = hl | (i << ybase);
        const int src_lane = (int)((hs >> VB) & 31);
        const int src_reg = (int)(hs & (NE - 1));
        if constexpr (ALLC && W == 4) {
          // four shuffles, then a 2-level select on the register index
          const uint32_t g0 = __shfl_sync(0xffffffffu, sv[u].w[0], src_lane);
          const uint32_t g1 = __shfl_sync(0xffffffffu, sv[u].w[1], src_lane);
          const uint32_t g2 = __shfl_sync(0xffffffffu, sv[u].w[2], src_lane);
          const uint32_t g3 = __shfl_sync(0xffffffffu, sv[u].w[3], src_lane);
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
                uint32_t lo = __shfl_sync(0xffffffffu, sv[u].w[2 * c], src_lane);
                uint32_t hi = __shfl_sync(0xffffffffu, sv[u].w[2 * c + 1], src_lane);
                got = (T)(((uint64_t)hi << 32) | lo);
              } else if constexpr (W == 4) {
                got = (T)__shfl_sync(0xffffffffu, sv[u].w[c], src_lane);
              } else {
                // sub-word elements: shuffle the containing word, then extract
                uint32_t wd = __shfl_sync(0xffffffffu, sv[u].w[(c * W) >> 2], src_lane);
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
}

// ------------------------------------------------------------------ launchers

static int g_num_sms = 0;
int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

int cached_occupancy(const void* kernel, int threads, size_t smem, int carveout) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, size_t, int, int>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(kernel, threads, smem, carveout, dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  if (carveout != -1) cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem) != cudaSuccess) occ = 0;
  cache[key] = occ;
  return occ;
}

static int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

// Launch configuration knobs (env, read once): LL_TPG = target tiles per tile
// group (0 = persistent grid at full occupancy), LL_PIPE = 1 for the
// software-pipelined kernel, LL_UP_TPG = tiles per group of the mxfp4 upcast
// kernel (default 0: persistent; sweep 4.78 vs 4.46 TB/s at 2), LL_TMA_TPG /
// LL_TMA_STAGES = tiles per group (0: persistent, -1: by wave count) and ring
// depth of the TMA path.
LaunchKnobs::LaunchKnobs()
      : tpg(env_int("LL_TPG", 2)), pipe(env_int("LL_PIPE", 1)),
        gather_tpt(env_int("LL_GATHER_VPT", 0)), carveout(env_int("LL_CARVEOUT", -1)),
        pow2(env_int("LL_POW2", 0)), stages(env_int("LL_STAGES", 3)),
        async_tpg(env_int("LL_ASYNC_TPG", 8)), up_tpg(env_int("LL_UP_TPG", 0)),
        tma_tpg(env_int("LL_TMA_TPG", -1)), tma_stages(env_int("LL_TMA_STAGES", 3)),
        gather_v8(env_int("LL_GATHER_V8", 0)), gather_shfl_u(2) {}
LaunchKnobs& knobs() {
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
  if (n == "up_tpg") { knobs().up_tpg = value; return 0; }
  if (n == "tma_tpg") { knobs().tma_tpg = value; return 0; }
  if (n == "tma_stages") { knobs().tma_stages = value; return 0; }
  if (n == "gather_v8") { knobs().gather_v8 = value; return 0; }
  if (n == "gather_shfl_u") { knobs().gather_shfl_u = value; return 0; }
  return -1;
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
  if (shuffle) {
    // warp-vectors whose loads are in flight together (knob gather_shfl_u)
    const int u = knobs().gather_shfl_u;
    const bool allc = p.cand_mask == (16 / W) - 1;
    auto go = [&](auto kern) {
      kern<<<grid, threads, 0, st>>>(p, (const uint8_t*)src, idx, (uint8_t*)out, err);
    };
    if (u >= 4) allc ? go(gather_shuffle_kernel<W, true, 4>) : go(gather_shuffle_kernel<W, false, 4>);
    else if (u == 2) allc ? go(gather_shuffle_kernel<W, true, 2>) : go(gather_shuffle_kernel<W, false, 2>);
    else allc ? go(gather_shuffle_kernel<W, true, 1>) : go(gather_shuffle_kernel<W, false, 1>);
  } else
  {
    // 32 bytes per thread (256-bit stores) when every batch holds an even
    // number of 16-byte vectors (knob gather_v8)
    const bool v2 = knobs().gather_v8 && (p.nbits - ilog2(16 / W)) >= 1 &&
                    (reinterpret_cast<uintptr_t>(out) & 31) == 0;
    auto go = [&](auto kern, int g) {
      if (planner_knob("gather_pdl", 1)) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)g);
        cfg.blockDim = dim3(threads);
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, kern, p, (const uint8_t*)src, idx, (uint8_t*)out, err);
      } else {
        kern<<<g, threads, 0, st>>>(p, (const uint8_t*)src, idx, (uint8_t*)out, err);
      }
    };
    if (v2) {
      int64_t want2 = ((p.n_vec >> 1) + (int64_t)threads * vpt - 1) / ((int64_t)threads * vpt);
      if (max_ctas > 0 && want2 > max_ctas) want2 = max_ctas;
      const int grid2 = (int)std::max<int64_t>(1, std::min<int64_t>(want2, 0x7fffffff));
      go(gather_direct_kernel<W, true>, grid2);
    } else {
      go(gather_direct_kernel<W, false>, grid);
    }
  }
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

// ------------------------------------------------------------- checksum (a12)
// Sum over elements of fmix(v + (base + h + 1) * gamma) (indexed) or fmix(v),
// mod 2^64 (order-free, so a grid-stride reduction with 64-bit atomics).
__device__ __forceinline__ unsigned long long ck_fmix(unsigned long long z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <int W>
__global__ void __launch_bounds__(256) checksum_kernel(const uint8_t* __restrict__ buf, int64_t n,
                                                       bool indexed, int64_t base,
                                                       unsigned long long* result) {
  constexpr int E = 16 / W;  // elements per 16-byte vector
  constexpr unsigned long long G = 0x9E3779B97F4A7C15ull;
  unsigned long long acc = 0;
  const int64_t nvec = n / E;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += stride) {
    const uint4 q = __ldg(reinterpret_cast<const uint4*>(buf) + v);
    const uint32_t wd[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int e = 0; e < E; ++e) {
      unsigned long long x;
      if (W == 8) x = (unsigned long long)wd[2 * e] | ((unsigned long long)wd[2 * e + 1] << 32);
      else x = (wd[(e * W) / 4] >> (8 * ((e * W) % 4))) & (W == 4 ? 0xFFFFFFFFu : (1u << (8 * W)) - 1u);
      const unsigned long long h = (unsigned long long)(v * E + e);
      acc += ck_fmix(indexed ? x + ((unsigned long long)base + h + 1ull) * G : x);
    }
  }
  // ragged tail (n not a multiple of E): the first threads take one element each
  const int64_t tail0 = nvec * E;
  const int64_t ti = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (ti < n - tail0) {
    const uint8_t* ep = buf + (tail0 + ti) * W;
    unsigned long long x = 0;
    for (int b = 0; b < W; ++b) x |= (unsigned long long)ep[b] << (8 * b);
    const unsigned long long h = (unsigned long long)(tail0 + ti);
    acc += ck_fmix(indexed ? x + ((unsigned long long)base + h + 1ull) * G : x);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
  __shared__ unsigned long long part[8];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long s = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += part[i];
    atomicAdd(result, s);
  }
}

cudaError_t launch_checksum(const void* buf, int64_t n, int w, bool indexed, int64_t base,
                            unsigned long long* result, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(result, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess || n == 0) return e;
  const int64_t nvec = std::max<int64_t>(1, n / (16 / w));
  const int64_t grid = std::min<int64_t>((nvec + 255) / 256, (int64_t)num_sms() * 8);
  const uint8_t* b = static_cast<const uint8_t*>(buf);
  switch (w) {
    case 1: checksum_kernel<1><<<(unsigned)grid, 256, 0, st>>>(b, n, indexed, base, result); break;
    case 2: checksum_kernel<2><<<(unsigned)grid, 256, 0, st>>>(b, n, indexed, base, result); break;
    case 4: checksum_kernel<4><<<(unsigned)grid, 256, 0, st>>>(b, n, indexed, base, result); break;
    case 8: checksum_kernel<8><<<(unsigned)grid, 256, 0, st>>>(b, n, indexed, base, result); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace ll
