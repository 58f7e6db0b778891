// jit.cpp -- run-time specialised kernels (NVRTC) for the register-faithful
// warp-shuffle exchange (LL_PATH_REGS_SHUFFLE).
//
// The paper lowers a conversion inside a compiler, so every register index of
// the 2^|R| shuffle rounds is a constant and the uniform word permutations
// (alpha, eps) are free register renames; only the lane-dependent parts
// (beta / zeta selects, delta source lane) cost instructions.  A generic
// kernel would have to apply alpha / eps as run-time register moves, so this
// path generates CUDA source for the plan, compiles it for sm_100a with NVRTC
// once per plan, and launches it through the driver API (entry points from
// cudaGetDriverEntryPoint; no link-time libcuda dependency).
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>

#include "kernels.hpp"
#include "planner.hpp"

namespace ll {

namespace {

int ilog2i(int x) {
  int r = 0;
  while ((1 << (r + 1)) <= x) ++r;
  return r;
}

typedef CUresult (*PFN_LoadData)(CUmodule*, const void*);
typedef CUresult (*PFN_GetFunction)(CUfunction*, CUmodule, const char*);
typedef CUresult (*PFN_FuncSetAttribute)(CUfunction, CUfunction_attribute, int);
typedef CUresult (*PFN_LaunchEx)(const CUlaunchConfig*, CUfunction, void**, void**);
typedef CUresult (*PFN_Occupancy)(int*, CUfunction, int, size_t);
typedef CUresult (*PFN_Launch)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned,
                               unsigned, unsigned, CUstream, void**, void**);

template <class F>
F entry(const char* name) {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &f, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(f);
}

// global load / store instructions of the compiled smem kernel; knobs
// ld_hint / st_hint select the cache qualifiers (ablation of the streaming
// hints): ld 0 = .nc.L1::no_allocate, 1 = + .L2::256B prefetch, 2 = + L2
// evict_first policy, 3 = .cs.nc; st 0 = .cs, 1 = plain (write-back),
// 2 = L2 evict_first policy, 3 = .L1::no_allocate, 4 = L2 evict_last policy.
// Each returns the asm text from the opcode to the end: "op.vN.T {...}, [%a];"
std::string ldg_asm(const std::string& vt, const std::string& regs, int a) {
  const int h = planner_knob("ld_hint", 0);
  const std::string addr = "[%" + std::to_string(a) + "]";
  switch (h) {
    case 1: return "ld.global.nc.L1::no_allocate.L2::256B." + vt + " " + regs + ", " + addr + ";";
    case 2: return "{ .reg .b64 p_; createpolicy.fractional.L2::evict_first.b64 p_, 1.0; "
                   "ld.global.nc.L1::no_allocate.L2::cache_hint." + vt + " " + regs + ", " + addr + ", p_; }";
    case 3: return "ld.global.cs.nc." + vt + " " + regs + ", " + addr + ";";
    default: return "ld.global.nc.L1::no_allocate." + vt + " " + regs + ", " + addr + ";";
  }
}
std::string stg_asm(const std::string& vt, const std::string& regs) {
  const int h = planner_knob("st_hint", 0);
  switch (h) {
    case 1: return "st.global." + vt + " [%0], " + regs + ";";
    case 2: return "{ .reg .b64 p_; createpolicy.fractional.L2::evict_first.b64 p_, 1.0; "
                   "st.global.L2::cache_hint." + vt + " [%0], " + regs + ", p_; }";
    case 3: return "st.global.L1::no_allocate." + vt + " [%0], " + regs + ";";
    case 4: return "{ .reg .b64 p_; createpolicy.fractional.L2::evict_last.b64 p_, 1.0; "
                   "st.global.L2::cache_hint." + vt + " [%0], " + regs + ", p_; }";
    default: return "st.global.cs." + vt + " [%0], " + regs + ";";
  }
}

// CTAs of a launch that can be resident at once (SMs x occupancy of fn):
// the first wave, the only CTAs PDL can start during the preceding grid
long long first_wave_ctas(CUfunction fn, int block, int smem, int sms) {
  static PFN_Occupancy occ = entry<PFN_Occupancy>("cuOccupancyMaxActiveBlocksPerMultiprocessor");
  static PFN_FuncSetAttribute setattr_ = entry<PFN_FuncSetAttribute>("cuFuncSetAttribute");
  // the occupancy query needs the kernel's dynamic shared-memory limit raised first
  if (smem > 48 * 1024 && setattr_) setattr_(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, smem);
  static std::mutex occ_mu;
  static std::map<std::pair<CUfunction, int>, int> occ_cache;
  std::lock_guard<std::mutex> lk(occ_mu);
  auto key = std::make_pair(fn, smem * 2048 + block);
  auto it = occ_cache.find(key);
  if (it == occ_cache.end()) {
    int per_sm = 0;
    if (!occ || occ(&per_sm, fn, block, (size_t)smem) != CUDA_SUCCESS) per_sm = 1;
    it = occ_cache.emplace(key, std::max(1, per_sm)).first;
  }
  return (long long)it->second * sms;
}

// element-bit swap (a < b) of the thread's register file, compile-time
// (same semantics as device_common.cuh apply_swap), emitted as source text
void emit_swap(std::ostringstream& o, int W, int NW, int a, int b, const char* R) {
  auto word_swap = [&](int A, int B) {
    for (int i = 0; i < NW; ++i)
      if (((i >> A) & 1) == 0 && ((i >> B) & 1) == 1) {
        const int j = i ^ ((1 << A) | (1 << B));
        o << "  { unsigned t_ = " << R << "[" << i << "]; " << R << "[" << i << "] = " << R << "[" << j
          << "]; " << R << "[" << j << "] = t_; }\n";
      }
  };
  auto sub_swap = [&](int B, unsigned lo, unsigned hi) {
    for (int i = 0; i < NW; ++i)
      if (((i >> B) & 1) == 0) {
        const int j = i | (1 << B);
        o << "  { unsigned x_ = " << R << "[" << i << "], y_ = " << R << "[" << j << "]; " << R << "["
          << i << "] = __byte_perm(x_, y_, " << lo << "u); " << R << "[" << j
          << "] = __byte_perm(x_, y_, " << hi << "u); }\n";
      }
  };
  if (W == 8) {
    word_swap(a + 1, b + 1);
  } else if (W == 4) {
    word_swap(a, b);
  } else if (W == 2) {
    if (a == 0) sub_swap(b - 1, 0x5410u, 0x7632u);
    else word_swap(a - 1, b - 1);
  } else {
    if (a == 0 && b == 1) {
      for (int i = 0; i < NW; ++i)
        o << "  " << R << "[" << i << "] = __byte_perm(" << R << "[" << i << "], 0u, " << 0x3120u << "u);\n";
    } else if (a == 0) {
      sub_swap(b - 2, 0x6240u, 0x7351u);
    } else if (a == 1) {
      sub_swap(b - 2, 0x5410u, 0x7632u);
    } else {
      word_swap(a - 2, b - 2);
    }
  }
}

// one direction of the exchange: D = exchange(S)
void emit_dir(std::ostringstream& o, const ShuffleDir& d, int NW, const char* S, const char* D,
              const char* pfx) {
  o << "  {\n    unsigned T_[" << NW << "];\n";
  for (int k = 0; k < NW; ++k) o << "    T_[" << k << "] = " << S << "[" << k << "];\n";
  auto lane_xor = [&](const char* A, uint32_t any, const char* mask) {
    for (int b = 0; (1 << b) < NW; ++b) {
      if (!((any >> b) & 1)) continue;
      o << "    { const bool q_ = (" << mask << " >> " << b << ") & 1;\n";
      for (int k = 0; k < NW; ++k)
        if (((k >> b) & 1) == 0) {
          const int j = k | (1 << b);
          o << "      { unsigned x_ = " << A << "[" << k << "], y_ = " << A << "[" << j << "]; " << A
            << "[" << k << "] = q_ ? y_ : x_; " << A << "[" << j << "] = q_ ? x_ : y_; }\n";
        }
      o << "    }\n";
    }
  };
  lane_xor("T_", d.beta_any, (std::string(pfx) + "b").c_str());
  // every round reads the receiving lane itself: a register permutation
  // inside each thread, no shuffle
  bool local = true;
  for (int k = 0; k < NW; ++k) local = local && d.gamma[k] == 0;
  for (int c = 0; c < 5; ++c) local = local && d.delta[c] == (1u << c);
  for (int k = 0; k < NW; ++k) {
    if (local)
      o << "    " << D << "[" << d.eps[k] << "] = T_[" << d.alpha[k] << "];\n";
    else
      o << "    " << D << "[" << d.eps[k] << "] = __shfl_sync(0xffffffffu, T_[" << d.alpha[k] << "], "
        << (int)d.gamma[k] << " ^ " << pfx << "d);\n";
  }
  lane_xor(D, d.zeta_any, (std::string(pfx) + "z").c_str());
  o << "  }\n";
}

std::string regs_shuffle_source(const RegsShufflePlan& p, int W) {
  const int NW = p.nwords, NT = 32 << p.nw, TB = NW * 4;
  std::ostringstream o;
  o << "extern \"C\" __global__ void __launch_bounds__(" << NT << ") ll_regs_shfl(\n"
    << "    const unsigned char* __restrict__ src, unsigned char* __restrict__ dst,\n"
    << "    long long n_tiles, long long tile_bytes, int reps, long long* cycles) {\n"
    << "  const int tid = threadIdx.x, lane = tid & 31;\n"
    << "  unsigned fb = 0, fz = 0, fd = 0, bb = 0, bz = 0, bd = 0;\n";
  for (int c = 0; c < 5; ++c)
    o << "  if (lane & " << (1 << c) << ") { fb ^= " << p.fwd.beta[c] << "u; fz ^= " << p.fwd.zeta[c]
      << "u; fd ^= " << p.fwd.delta[c] << "u; bb ^= " << p.bwd.beta[c] << "u; bz ^= " << p.bwd.zeta[c]
      << "u; bd ^= " << p.bwd.delta[c] << "u; }\n";
  o << "  for (long long t = blockIdx.x; t < n_tiles; t += gridDim.x) {\n"
    << "  const unsigned char* sp = src + t * tile_bytes + (long long)tid * " << TB << ";\n"
    << "  unsigned char* dp = dst + t * tile_bytes + (long long)tid * " << TB << ";\n"
    << "  unsigned R[" << NW << "], Q[" << NW << "];\n";
  if (TB >= 16) {
    for (int u = 0; u < NW / 4; ++u)
      o << "  { uint4 v_ = __ldg(reinterpret_cast<const uint4*>(sp) + " << u << "); R[" << 4 * u
        << "] = v_.x; R[" << 4 * u + 1 << "] = v_.y; R[" << 4 * u + 2 << "] = v_.z; R[" << 4 * u + 3
        << "] = v_.w; }\n";
  } else {
    for (int u = 0; u < NW; ++u)
      o << "  R[" << u << "] = __ldg(reinterpret_cast<const unsigned*>(sp) + " << u << ");\n";
  }
  for (auto& s : p.swaps) emit_swap(o, W, NW, s.first, s.second, "R");
  o << "  long long c0_ = 0;\n  if (cycles && tid == 0) c0_ = clock64();\n"
    << "  for (int rep = 0; rep < reps; ++rep) {\n";
  emit_dir(o, p.fwd, NW, "R", "Q", "f");
  emit_dir(o, p.bwd, NW, "Q", "R", "b");
  o << "  }\n  if (cycles && tid == 0 && t == blockIdx.x) cycles[blockIdx.x] = clock64() - c0_;\n";
  emit_dir(o, p.fwd, NW, "R", "Q", "f");
  if (TB >= 16) {
    for (int u = 0; u < NW / 4; ++u)
      o << "  reinterpret_cast<uint4*>(dp)[" << u << "] = make_uint4(Q[" << 4 * u << "], Q["
        << 4 * u + 1 << "], Q[" << 4 * u + 2 << "], Q[" << 4 * u + 3 << "]);\n";
  } else {
    for (int u = 0; u < NW; ++u) o << "  reinterpret_cast<unsigned*>(dp)[" << u << "] = Q[" << u << "];\n";
  }
  o << "  }\n}\n";
  return o.str();
}

// HBM -> HBM warp-shuffle conversion (LL_PATH_SHUFFLE) specialised for the
// plan: the free-mapped warp tiles of plan_smem (load / store layouts), the
// tile offsets from the plan's tables (kernel parameter, warp-uniform), and
// the exchange with constant register indices.
std::string shuffle_hbm_source(const ConvertPlan& P) {
  const ShufflePlan& p = P.shp;
  const int W = P.w, NV = P.nv, NW = NV * 4;
  std::ostringstream o;
  o << "struct TileTab { long long src, dst, sc; };\n"
    << "struct TileMap { long long n_tiles; int n_bits; int n_tab; long long bss, bsd; TileTab tab["
    << LL_MAX_TAB << "][" << (1 << LL_TAB_BITS) << "]; };\n"
    << "extern \"C\" __global__ void __launch_bounds__(256) ll_shfl_hbm(\n"
    << "    const __grid_constant__ TileMap tm, const unsigned char* __restrict__ src,\n"
    << "    unsigned char* __restrict__ dst, long long n_groups, long long t0, long long t1,\n"
    << "    long long src_shift, long long dst_shift, long long pf_ctas) {\n"
    << "  const int lane = threadIdx.x & 31;\n"
    << "  const long long gid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;\n"
    << "  if (gid >= n_groups) return;\n"
    << "  unsigned ld_off = 0, st_off = 0, fb = 0, fz = 0, fd = 0;\n";
  for (int c = 0; c < 5; ++c)
    o << "  if (lane & " << (1 << c) << ") { ld_off += " << p.ld_thr[c] << "u; st_off += " << p.st_thr[c]
      << "u; fb ^= " << P.shd.beta[c] << "u; fz ^= " << P.shd.zeta[c] << "u; fd ^= " << P.shd.delta[c]
      << "u; }\n";
  o << "  const unsigned char* sthr = src + ld_off - src_shift;\n"
    << "  unsigned char* dthr = dst + st_off - dst_shift;\n"
    << "  const long long rmask = (1LL << tm.n_bits) - 1;\n";
  // programmatic dependent launch (knob shuffle_pdl; config 6: 6601 -> 6793
  // GB/s, profiles/r02/s3h) with the first wave's L2 prefetch of its first
  // tile (as the smem kernel, pdl_prefetch)
  if (planner_knob("shuffle_pdl", 1)) {
    if (planner_knob("pdl_prefetch", 1)) {
      // knob shuffle_prefetch_waves = K (default 3): also the tiles of the
      // warps that replace this one in waves 2..K (8 warps per CTA); config
      // 6: 6765 -> 6795 (K = 2) -> 6819 GB/s (K = 3), profiles/r02/s3y
      const int pfk = std::max(1, std::min(4, planner_knob("shuffle_prefetch_waves", 3)));
      for (int kw = 0; kw < pfk; ++kw) {
        o << "  { const long long t = t0 + gid + " << kw << "LL * pf_ctas * 8; if (t < t1 && blockIdx.x < pf_ctas) {\n"
          << "    const long long inst = t >> tm.n_bits, r = t & rmask;\n"
          << "    long long so = inst * tm.bss;\n";
        for (int k = 0; k < p.tile.n_tab; ++k)
          o << "    so += tm.tab[" << k << "][(int)((r >> " << k * LL_TAB_BITS << ") & "
            << ((1 << LL_TAB_BITS) - 1) << ")].src;\n";
        const bool sbulk = planner_knob("shuffle_prefetch_bulk", 1) != 0;   // as pdl_prefetch_bulk (config 6: 6818 -> 6929, s3bb)
        for (int u = 0; u < NV; ++u)
          o << "    { const unsigned char* a_ = sthr + so + " << p.ld_vec[u]
            << "u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile(\""
            << (sbulk ? "cp.async.bulk.prefetch.L2.global [%0], 128;" : "prefetch.global.L2 [%0];")
            << "\" :: \"l\"(a_)); }\n";
        o << "  } }\n";
      }
    }
    o << "  asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");\n"
      << "  asm volatile(\"griddepcontrol.launch_dependents;\");\n";
  }
  o << "  for (long long t = t0 + gid; t < t1; t += n_groups) {\n"
    << "    const long long inst = t >> tm.n_bits, r = t & rmask;\n"
    << "    long long so = inst * tm.bss, dof = inst * tm.bsd;\n";
  for (int k = 0; k < p.tile.n_tab; ++k)
    o << "    { const TileTab& e = tm.tab[" << k << "][(int)((r >> " << k * LL_TAB_BITS << ") & "
      << ((1 << LL_TAB_BITS) - 1) << ")]; so += e.src; dof += e.dst; }\n";
  o << "    unsigned R[" << NW << "], Q[" << NW << "];\n";
  for (int u = 0; u < NV; ++u)
    o << "    asm volatile(\"ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\" : \"=r\"(R["
      << 4 * u << "]), \"=r\"(R[" << 4 * u + 1 << "]), \"=r\"(R[" << 4 * u + 2 << "]), \"=r\"(R["
      << 4 * u + 3 << "]) : \"l\"(sthr + so + " << p.ld_vec[u] << "));\n";
  for (int i = 0; i < p.n_swaps; ++i) emit_swap(o, W, NW, p.swap_a[i], p.swap_b[i], "R");
  emit_dir(o, P.shd, NW, "R", "Q", "f");
  for (int u = 0; u < NV; ++u)
    o << "    asm volatile(\"st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};\" :: \"l\"(dthr + dof + "
      << p.st_vec[u] << "), \"r\"(Q[" << 4 * u << "]), \"r\"(Q[" << 4 * u + 1 << "]), \"r\"(Q["
      << 4 * u + 2 << "]), \"r\"(Q[" << 4 * u + 3 << "]) : \"memory\");\n";
  o << "  }\n}\n";
  return o.str();
}

int deposit_word_h(int j, int k, int LB, int A, int B) {
  int idx = 0, q = 0;
  for (int bit = 0; bit < LB; ++bit) {
    if (bit == A) idx |= (k & 1) << bit;
    else if (bit == B) idx |= ((k >> 1) & 1) << bit;
    else { idx |= ((j >> q) & 1) << bit; ++q; }
  }
  return idx;
}

// One 32-bit word from 4 bytes (word expression, byte index), with prmt:
// a copy, one __byte_perm of two words, or two + a merge.
std::string pack_bytes(const std::vector<std::pair<std::string, int>>& b) {
  if (b[0].first == b[1].first && b[0].first == b[2].first && b[0].first == b[3].first &&
      b[0].second == 0 && b[1].second == 1 && b[2].second == 2 && b[3].second == 3)
    return b[0].first;
  std::vector<std::string> words;
  for (auto& x : b)
    if (std::find(words.begin(), words.end(), x.first) == words.end()) words.push_back(x.first);
  auto sel2 = [&](const std::string& w0, int i0, int i1, int i2, int i3) {
    // selector over (w0, w1): index < 4 from w0, else w1
    unsigned sel = 0;
    const int ii[4] = {i0, i1, i2, i3};
    for (int k = 0; k < 4; ++k) sel |= (unsigned)(ii[k] & 7) << (4 * k);
    (void)w0;
    return sel;
  };
  if (words.size() <= 2) {
    const std::string& w0 = words[0];
    const std::string& w1 = words.size() > 1 ? words[1] : words[0];
    int ii[4];
    for (int k = 0; k < 4; ++k) ii[k] = (b[k].first == w0 ? 0 : 4) + b[k].second;
    std::ostringstream e;
    e << "__byte_perm(" << w0 << ", " << w1 << ", " << sel2(w0, ii[0], ii[1], ii[2], ii[3]) << "u)";
    return e.str();
  }
  // two halves, then merge: t0 = [b0 b1 . .], t1 = [b2 b3 . .]
  auto half = [&](int k0) {
    const std::string& a = b[k0].first;
    const std::string& c = b[k0 + 1].first;
    std::ostringstream e;
    e << "__byte_perm(" << a << ", " << c << ", " << sel2(a, b[k0].second, 4 + b[k0 + 1].second, 0, 0) << "u)";
    return e.str();
  };
  return "__byte_perm(" + half(0) + ", " + half(2) + ", 0x5410u)";
}

// HBM -> HBM shared-memory conversion (LL_PATH_SMEM) specialised for the
// plan: the same schedule as convert_smem_kernel (software-pipelined loads,
// swizzled STS, group barrier, LDS, streaming stores), with every offset,
// granule operand and register permutation a compile-time constant.
//
// single: every group converts exactly one tile (the launch has at least as
// many groups as tiles), so the group needs one staging buffer instead of
// two and no prefetch; half the shared memory per CTA.
std::string smem_hbm_source(const ConvertPlan& P, bool single) {
  const SmemPlan& p = P.sp;
  const int W = P.w, NV = P.nv, NW = NV * 4, G = P.g, GWd = G / 4, NG = NV * 16 / G;
  const int gw = p.gw, LB = ilog2i(NW);
  const int minb_knob = planner_knob("smem_jit_minb", 0);
  const int minb = minb_knob > 0 ? minb_knob : (G < 8 ? 1 : (NV >= 8 ? 3 : 4));
  std::ostringstream o;
  o << "struct TileTab { long long src, dst, sc; };\n"
    << "struct TileMap { long long n_tiles; int n_bits; int n_tab; long long bss, bsd; TileTab tab["
    << LL_MAX_TAB << "][" << (1 << LL_TAB_BITS) << "]; };\n"
    << "extern \"C\" __global__ void __launch_bounds__(256, " << minb << ") ll_smem_hbm(\n"
    << "    const __grid_constant__ TileMap tm, const unsigned char* __restrict__ src,\n"
    << "    unsigned char* __restrict__ dst, long long n_groups, long long t0, long long t1,\n"
    << "    long long src_shift, long long dst_shift, long long pf_ctas) {\n"
    << "  extern __shared__ __align__(16) unsigned char smem[];\n"
    << "  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;\n"
    << "  const int group = warp >> " << gw << ";\n"
    << "  const int tb = lane | ((warp & " << ((1 << gw) - 1) << ") << 5);\n"
    << "  const long long gid = (long long)blockIdx.x * " << (8 >> gw) << " + group;\n"
    << "  if (gid >= n_groups) return;\n"
    << "  unsigned ld_off = 0, st_off = 0, swx = 0, srx = 0;\n";
  for (int b = 0; b < 5 + gw; ++b)
    o << "  if (tb & " << (1 << b) << ") { ld_off += " << p.ld_thr[b] << "u; st_off += " << p.st_thr[b]
      << "u; swx ^= " << p.sw_thr[b] << "u; srx ^= " << p.sr_thr[b] << "u; }\n";
  o << "  const unsigned char* sthr = src + ld_off - src_shift;\n"
    << "  unsigned char* dthr = dst + st_off - dst_shift;\n"
    << "  const long long rmask = (1LL << tm.n_bits) - 1;\n"
    << "  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem) + group * "
    << (single ? 1 : 2) * p.tile_bytes << "u;\n"
    << "  unsigned buf = 0;\n  unsigned R[" << NW << "], Q[" << NW << "];\n"
    << "  long long so = 0, dof = 0;\n";
  // knob tile_xor = L (sweep): the tile -> CTA order XORs L bits of the tile
  // index (from bit tile_xor_skip up) into its top L bits, so consecutive
  // tiles of a column walk also hop across the outer dimension ("diagonal"
  // order against DRAM channel camping of power-of-two strides).  A
  // bijection on each instance's tiles; only for full-range launches (a
  // shard's tile range is not closed under it).
  const int txl = std::max(0, std::min(planner_knob("tile_xor", 0), p.tile.n_bits / 2));
  const int txs = std::max(0, planner_knob("tile_xor_skip", 1));
  const bool twist = txl > 0 && txs + txl <= p.tile.n_bits - txl;
  if (twist) o << "  const bool twist = t0 == 0 && t1 == tm.n_tiles;\n";
  o << "  auto tile_off = [&](long long t) {\n"
    << "    const long long inst = t >> tm.n_bits;\n"
    << "    long long r = t & rmask;\n";
  if (twist)
    o << "    if (twist) r ^= ((r >> " << txs << ") & " << ((1 << txl) - 1) << "LL) << " << p.tile.n_bits - txl << ";\n";
  o << "    so = inst * tm.bss; dof = inst * tm.bsd;\n";
  for (int k = 0; k < p.tile.n_tab; ++k)
    o << "    { const TileTab& e = tm.tab[" << k << "][(int)((r >> " << k * LL_TAB_BITS << ") & "
      << ((1 << LL_TAB_BITS) - 1) << ")]; so += e.src; dof += e.dst; }\n";
  o << "  };\n";
  // 256-bit accesses where a thread's vectors u, u + 1 are contiguous (knob vec32)
  bool ld32 = NV >= 2, st32 = NV >= 2;
  for (int u = 0; u + 1 < NV; u += 2) {
    ld32 = ld32 && p.ld_vec[u + 1] == p.ld_vec[u] + 16;
    st32 = st32 && p.st_vec[u + 1] == p.st_vec[u] + 16;
  }
  const bool noload = planner_knob("smem_jit_noload", 0) != 0;   // test hook: no global loads
  const bool nostore = planner_knob("smem_jit_nostore", 0) != 0; // test hook: no global stores
  const bool noxchg = planner_knob("smem_jit_noxchg", 0) != 0;   // test hook: no exchange
  auto load = [&](const char* ind, const std::string& R) {
    if (noload) {
      for (int i = 0; i < NW; ++i)
        o << ind << R << "[" << i << "] = (unsigned)so * 2654435761u + tb * " << 4 * NW + 1 << "u + " << i << "u;\n";
      return;
    }
    if (P.ld_span > 0) {
      // broadcast dedup: a virtual vector's elements come from 2^ld_span
      // physical vectors (source copy bits inside them are dropped)
      const int C = 1 << P.ld_span, NEl = 16 / W, vbl = ilog2i(NEl);
      std::vector<char> ref(C, 0);     // physical vectors holding virtual elements
      for (int e = 0; e < NEl; ++e) {
        int ph = 0;
        for (int b = 0; b < vbl; ++b) if ((e >> b) & 1) ph |= 1 << P.src_phys[b];
        ref[ph >> vbl] = 1;
      }
      for (int u = 0; u < NV; ++u) {
        o << ind << "{ unsigned PL[" << 4 * C << "];\n";
        for (int c = 0; c < C; ++c)
          if (ref[c])
            o << ind << "  asm volatile(\"" << ldg_asm("v4.u32", "{%0,%1,%2,%3}", 4) << "\" : \"=r\"(PL["
              << 4 * c << "]), \"=r\"(PL[" << 4 * c + 1 << "]), \"=r\"(PL[" << 4 * c + 2 << "]), \"=r\"(PL["
              << 4 * c + 3 << "]) : \"l\"(sthr + so + " << p.ld_vec[u] + 16u * c << "));\n";
        auto src_byte = [&](int byte) {   // byte of the virtual vector -> (word, byte) of PL
          const int e = byte / W, eb = byte % W;
          int ph = 0;
          for (int b = 0; b < vbl; ++b) if ((e >> b) & 1) ph |= 1 << P.src_phys[b];
          const int pbyte = (ph & (NEl - 1)) * W + eb + 16 * (ph >> vbl);
          return std::make_pair("PL[" + std::to_string(pbyte >> 2) + "]", pbyte & 3);
        };
        for (int q = 0; q < 4; ++q) {
          std::vector<std::pair<std::string, int>> bs;
          for (int k = 0; k < 4; ++k) bs.push_back(src_byte(4 * q + k));
          o << ind << "  " << R << "[" << 4 * u + q << "] = " << pack_bytes(bs) << ";\n";
        }
        o << ind << "}\n";
      }
      return;
    }
    for (int u = 0; u < NV; u += ld32 ? 2 : 1) {
      if (ld32) {
        o << ind << "asm volatile(\"" << ldg_asm("v8.u32", "{%0,%1,%2,%3,%4,%5,%6,%7}", 8) << "\" : ";
        for (int q = 0; q < 8; ++q) o << (q ? ", " : "") << "\"=r\"(" << R << "[" << 4 * u + q << "])";
        o << " : \"l\"(sthr + so + " << p.ld_vec[u] << "));\n";
        continue;
      }
      o << ind << "asm volatile(\"" << ldg_asm("v4.u32", "{%0,%1,%2,%3}", 4) << "\" : \"=r\"(" << R << "["
        << 4 * u << "]), \"=r\"(" << R << "[" << 4 * u + 1 << "]), \"=r\"(" << R << "[" << 4 * u + 2
        << "]), \"=r\"(" << R << "[" << 4 * u + 3 << "]) : \"l\"(sthr + so + " << p.ld_vec[u] << "));\n";
    }
  };
  const int ga = GWd >= 2 ? p.gsel_a : -1, gb = GWd >= 4 ? p.gsel_b : -1;
  // one tile: swaps, STS, prefetch of tile t + ahead * n_groups into the same
  // registers, group barrier, LDS, streaming stores
  auto body = [&](const std::string& R, const std::string& dv, int ahead) {
    o << "    { const long long dcur = " << dv << ";\n";
    for (int i = 0; i < p.n_swaps; ++i) emit_swap(o, W, NW, p.swap_a[i], p.swap_b[i], R.c_str());
    // test hook (knob smem_jit_noxchg): no shared-memory exchange at all --
    // the loaded words are stored as they are, so the kernel keeps exactly
    // the global access pattern of the plan (the pattern's own ceiling)
    if (noxchg) for (int i = 0; i < NW; ++i) o << "    Q[" << i << "] = " << R << "[" << i << "];\n";
    for (int j = 0; j < NG && !noxchg; ++j) {
      o << "    asm volatile(\"st.shared.";
      if (GWd == 4) o << "v4.b32 [%0], {%1,%2,%3,%4};\"";
      else if (GWd == 2) o << "v2.b32 [%0], {%1,%2};\"";
      else o << "b32 [%0], %1;\"";
      o << " :: \"r\"(sbase + buf + (swx ^ " << p.sw_gran[j] << "u))";
      for (int k = 0; k < GWd; ++k) o << ", \"r\"(" << R << "[" << deposit_word_h(j, k, LB, ga, gb) << "])";
      o << " : \"memory\");\n";
    }
    if (ahead > 0) {
      o << "    { const long long tn = t + " << ahead << " * n_groups; if (tn < t1) { tile_off(tn); "
        << dv << " = dof;\n";
      load("      ", R);
      o << "    } }\n";
    }
    if (noxchg) {
    } else if (gw == 0) o << "    __syncwarp();\n";
    else o << "    asm volatile(\"bar.sync %0, %1;\" :: \"r\"(group + 1), \"r\"(" << (32 << gw) << ") : \"memory\");\n";
    for (int j = 0; j < NG && !noxchg; ++j) {
      o << "    asm volatile(\"ld.shared.";
      if (GWd == 4) o << "v4.b32 {%0,%1,%2,%3}, [%4];\" : \"=r\"(Q[" << 4 * j << "]), \"=r\"(Q[" << 4 * j + 1
                      << "]), \"=r\"(Q[" << 4 * j + 2 << "]), \"=r\"(Q[" << 4 * j + 3 << "])";
      else if (GWd == 2) o << "v2.b32 {%0,%1}, [%2];\" : \"=r\"(Q[" << 2 * j << "]), \"=r\"(Q[" << 2 * j + 1 << "])";
      else o << "b32 %0, [%1];\" : \"=r\"(Q[" << j << "])";
      o << " : \"r\"(sbase + buf + (srx ^ " << p.sr_gran[j] << "u)) : \"memory\");\n";
    }
    if (nostore) {   // test hook: keep the LDS results alive without global stores
      o << "    { unsigned x_ = 0;";
      for (int i = 0; i < NW; ++i) o << " x_ ^= Q[" << i << "];";
      o << " if (x_ == 0x9e3779b9u && dcur < 0) dthr[0] = 1; }\n";
    }
    if (!nostore && (P.st_span > 0 || P.copy_off.size() > 1)) {
      // broadcast dedup: each virtual vector becomes 2^st_span physical
      // vectors (destination copy bits inside them duplicated in registers),
      // each stored at every copy offset
      const int C = 1 << P.st_span, NEl = 16 / W, vbl = ilog2i(NEl);
      for (int u = 0; u < NV; ++u) {
        for (int c = 0; c < C; ++c) {
          std::string wexpr[4];
          for (int q = 0; q < 4; ++q) {
            std::vector<std::pair<std::string, int>> bs;
            for (int k = 0; k < 4; ++k) {
              const int pbyte = 4 * q + k, pe = (c << vbl) | (pbyte / W);
              int e = 0;   // virtual element: the bits at the virtual vector's physical positions
              for (int b = 0; b < vbl; ++b) if ((pe >> P.dst_phys[b]) & 1) e |= 1 << b;
              const int vbyte = e * W + pbyte % W;
              bs.push_back(std::make_pair("Q[" + std::to_string(4 * u + (vbyte >> 2)) + "]", vbyte & 3));
            }
            wexpr[q] = pack_bytes(bs);
          }
          o << "    { const unsigned S0 = " << wexpr[0] << ", S1 = " << wexpr[1] << ", S2 = " << wexpr[2]
            << ", S3 = " << wexpr[3] << ";\n";
          const std::vector<uint32_t> offs = P.copy_off.empty() ? std::vector<uint32_t>{0u} : P.copy_off;
          for (uint32_t co : offs)
            o << "      asm volatile(\"" << stg_asm("v4.u32", "{%1,%2,%3,%4}") << "\" :: \"l\"(dthr + dcur + "
              << p.st_vec[u] + 16u * c + co << "u), \"r\"(S0), \"r\"(S1), \"r\"(S2), \"r\"(S3) : \"memory\");\n";
          o << "    }\n";
        }
      }
    }
    for (int u = 0; u < NV && !nostore && !(P.st_span > 0 || P.copy_off.size() > 1); u += st32 ? 2 : 1) {
      if (st32) {
        o << "    asm volatile(\"" << stg_asm("v8.b32", "{%1,%2,%3,%4,%5,%6,%7,%8}") << "\" :: \"l\"(dthr + dcur + "
          << p.st_vec[u] << ")";
        for (int q = 0; q < 8; ++q) o << ", \"r\"(Q[" << 4 * u + q << "])";
        o << " : \"memory\");\n";
        continue;
      }
      o << "    asm volatile(\"" << stg_asm("v4.u32", "{%1,%2,%3,%4}") << "\" :: \"l\"(dthr + dcur + "
        << p.st_vec[u] << "), \"r\"(Q[" << 4 * u << "]), \"r\"(Q[" << 4 * u + 1 << "]), \"r\"(Q["
        << 4 * u + 2 << "]), \"r\"(Q[" << 4 * u + 3 << "]) : \"memory\");\n";
    }
    o << "    buf ^= " << p.tile_bytes << "u; }\n";
  };
  const int depth = std::max(1, std::min(2, planner_knob("smem_jit_depth", 1)));
  const bool pdl = planner_knob("pdl", 1) != 0;
  // programmatic dependent launch: wait for the preceding grid (its writes
  // visible) before the first global access; let the next grid launch once
  // this CTA's first loads are issued (its CTAs then wait at their own
  // griddepcontrol.wait), hiding launch latency and the tail wave
  // L2 prefetch of the first tile's source lines before the wait (knob
  // pdl_prefetch): a CTA that PDL makes resident during the preceding grid's
  // tail starts pulling its source into L2 then, so the DRAM pipe stays full
  // across the launch boundary.  Only the first wave (blockIdx < pf_ctas =
  // SMs x resident CTAs) can be early; later CTAs skip it (2: every CTA
  // prefetches, the A/B variant).  Safe whatever the
  // preceding grid writes: L2 is the device's point of coherence (its writes
  // land in the same lines), and nothing enters L1 before the wait.
  if (pdl && P.ld_span == 0 && !noload && planner_knob("pdl_prefetch", 1)) {
    // knob pdl_prefetch_waves = K (default 2): a first-wave CTA also
    // prefetches the first tiles of the CTAs that replace it in waves 2..K
    // (one-pass launches: tile + k * pf_ctas * groups per CTA).  K = 2:
    // config 2 6845 -> 6893 GB/s, config 5's N = 8 shard 6676 -> 6801,
    // configs 3 / 5 -0.2 % (profiles/r02/s3p); K = 3 loses
    const int pfk = std::max(1, std::min(4, planner_knob("pdl_prefetch_waves", 2)));
    for (int k = 0; k < pfk; ++k) {
      o << "  { const long long tp = t0 + gid + " << k << "LL * pf_ctas * " << (8 >> gw) << "; if (tp < t1"
        << (planner_knob("pdl_prefetch", 1) == 2 ? "" : " && blockIdx.x < pf_ctas") << ") { tile_off(tp);\n";
      // knob pdl_prefetch_bulk (default 1): the same lines through the
      // bulk-copy engine (cp.async.bulk.prefetch.L2, 128 B) instead of
      // prefetch.global.L2 -- config 3 6270 -> 6464 GB/s, config 2 6889 ->
      // 6914, config 5 unchanged, config 5's N = 8 shard 6936
      // (profiles/r02/s3aa)
      const bool bulk = planner_knob("pdl_prefetch_bulk", 1) != 0;
      for (int u = 0; u < NV; ++u)
        o << "    { const unsigned char* a_ = sthr + so + " << p.ld_vec[u]
          << "u; if ((((unsigned long long)a_) & 127ull) == 0) asm volatile(\""
          << (bulk ? "cp.async.bulk.prefetch.L2.global [%0], 128;" : "prefetch.global.L2 [%0];")
          << "\" :: \"l\"(a_)); }\n";
      o << "  } }\n";
    }
  }
  if (pdl) o << "  asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");\n";
  o << "  long long t = t0 + gid;\n";
  if (single) {
    o << "  if (t >= t1) return;\n  tile_off(t);\n  long long da = dof;\n";
    load("  ", "R");
    if (pdl) o << "  asm volatile(\"griddepcontrol.launch_dependents;\");\n";
    body("R", "da", 0);
    o << "}\n";
  } else if (depth == 1) {
    o << "  long long da = 0;\n  if (t < t1) { tile_off(t); da = dof;\n";
    load("    ", "R");
    o << "  }\n";
    if (pdl) o << "  asm volatile(\"griddepcontrol.launch_dependents;\");\n";
    o << "  for (; t < t1; t += n_groups) {\n";
    body("R", "da", 1);
    o << "  }\n}\n";
  } else {
    // two tiles in flight per group: registers Ra / Rb alternate
    o << "  unsigned Ra[" << NW << "], Rb[" << NW << "];\n  long long da = 0, db = 0;\n"
      << "  if (t < t1) { tile_off(t); da = dof;\n";
    load("    ", "Ra");
    o << "  }\n  if (t + n_groups < t1) { tile_off(t + n_groups); db = dof;\n";
    load("    ", "Rb");
    o << "  }\n  while (t < t1) {\n";
    body("Ra", "da", 2);
    o << "    t += n_groups;\n    if (t >= t1) break;\n";
    body("Rb", "db", 2);
    o << "    t += n_groups;\n  }\n}\n";
  }
  return o.str();
}

// The fused mxfp4 upcast (NEXT 1) compiled per plan: the smem schedule of
// smem_hbm_source with the tile's scales loaded with the tile, and the store
// stage decoding each 16-byte packed vector into 64 bytes of bf16 written as
// two 256-bit stores (same arithmetic as the template kernel's UP path).
std::string upcast_hbm_source(const ConvertPlan& P) {
  const SmemPlan& p = P.sp;
  const int NV = P.nv, NW = NV * 4, G = P.g, GWd = G / 4, NG = NV * 16 / G;
  const int gw = p.gw, LB = ilog2i(NW);
  std::ostringstream o;
  o << "struct TileTab { long long src, dst, sc; };\n"
    << "struct TileMap { long long n_tiles; int n_bits; int n_tab; long long bss, bsd; TileTab tab["
    << LL_MAX_TAB << "][" << (1 << LL_TAB_BITS) << "]; };\n"
    << "__device__ __forceinline__ unsigned mx_scale_f32(unsigned x) {\n"
    << "  return x == 255u ? 0x7FC00000u : (x == 0u ? 0x00400000u : (x << 23)); }\n"
    << "__device__ __forceinline__ unsigned e2m1_f32(unsigned n) {\n"
    << "  const unsigned e = (n >> 1) & 3u, m = n & 1u;\n"
    << "  const unsigned b = e ? (((e + 126u) << 23) | (m << 22)) : (m ? 0x3F000000u : 0u);\n"
    << "  return b | ((n & 8u) << 28); }\n"
    << "__device__ __forceinline__ unsigned bf16x2_mul(unsigned a, unsigned b) {\n"
    << "  unsigned d; asm(\"mul.rn.bf16x2 %0, %1, %2;\" : \"=r\"(d) : \"r\"(a), \"r\"(b)); return d; }\n"
    << "extern \"C\" __global__ void __launch_bounds__(256, 2) ll_upcast_hbm(\n"
    << "    const __grid_constant__ TileMap tm, const unsigned char* __restrict__ src,\n"
    << "    unsigned char* __restrict__ dst, long long n_groups, long long t0, long long t1,\n"
    << "    long long src_shift, long long dst_shift, const unsigned char* __restrict__ scales) {\n"
    << "  extern __shared__ __align__(16) unsigned char smem[];\n"
    << "  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;\n"
    << "  const int group = warp >> " << gw << ";\n"
    << "  const int tb = lane | ((warp & " << ((1 << gw) - 1) << ") << 5);\n"
    << "  const long long gid = (long long)blockIdx.x * " << (8 >> gw) << " + group;\n"
    << "  if (gid >= n_groups) return;\n"
    << "  unsigned ld_off = 0, st_off = 0, swx = 0, srx = 0, sc_off = 0;\n";
  for (int b = 0; b < 5 + gw; ++b)
    o << "  if (tb & " << (1 << b) << ") { ld_off += " << p.ld_thr[b] << "u; st_off += " << p.st_thr[b]
      << "u; swx ^= " << p.sw_thr[b] << "u; srx ^= " << p.sr_thr[b] << "u; sc_off += " << p.sc_thr[b]
      << "u; }\n";
  o << "  const unsigned char* sthr = src + ld_off - src_shift;\n"
    << "  const long long dbase = (long long)st_off - dst_shift;\n"
    << "  const long long rmask = (1LL << tm.n_bits) - 1;\n"
    << "  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem) + group * "
    << 2 * p.tile_bytes << "u;\n"
    << "  unsigned buf = 0;\n  unsigned R[" << NW << "], Q[" << NW << "], PK[" << NV << "], fastm = 0;\n"
    << "  long long so = 0, dof = 0, sct = 0;\n"
    << "  auto tile_off = [&](long long t) {\n"
    << "    const long long inst = t >> tm.n_bits, r = t & rmask;\n"
    << "    so = inst * tm.bss; dof = inst * tm.bsd; sct = 0;\n";
  for (int k = 0; k < p.tile.n_tab; ++k)
    o << "    { const TileTab& e = tm.tab[" << k << "][(int)((r >> " << k * LL_TAB_BITS << ") & "
      << ((1 << LL_TAB_BITS) - 1) << ")]; so += e.src; dof += e.dst; sct += e.sc; }\n";
  o << "  };\n";
  auto load = [&](const char* ind) {
    for (int u = 0; u < NV; ++u)
      o << ind << "asm volatile(\"ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\" : \"=r\"(R["
        << 4 * u << "]), \"=r\"(R[" << 4 * u + 1 << "]), \"=r\"(R[" << 4 * u + 2 << "]), \"=r\"(R["
        << 4 * u + 3 << "]) : \"l\"(sthr + so + " << p.ld_vec[u] << "));\n";
    o << ind << "fastm = 0;\n";
    for (int u = 0; u < NV; ++u) {
      o << ind << "{ const unsigned char* scp = scales + sct + sc_off + " << p.sc_vec[u] << ";\n"
        << ind << "  const unsigned s0 = __ldg(scp), s1 = __ldg(scp + " << p.sc_c[0] << "), s2 = __ldg(scp + "
        << p.sc_c[1] << "), s3 = __ldg(scp + " << p.sc_c[0] + p.sc_c[1] << ");\n"
        << ind << "  PK[" << u << "] = s0 | (s1 << 8) | (s2 << 16) | (s3 << 24);\n"
        << ind << "  fastm |= (unsigned)((s0 - 2u < 251u) & (s1 - 2u < 251u) & (s2 - 2u < 251u) & (s3 - 2u < 251u)) << "
        << u << "; }\n";
    }
  };
  // programmatic dependent launch (knob upcast_pdl): wait for the preceding
  // grid before the first global access, let the next one launch once this
  // CTA's first loads are issued
  const bool pdl = planner_knob("upcast_pdl", 0) != 0;
  if (pdl) o << "  asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");\n";
  o << "  long long t = t0 + gid;\n  if (t < t1) { tile_off(t);\n";
  load("    ");
  o << "  }\n";
  if (pdl) o << "  asm volatile(\"griddepcontrol.launch_dependents;\");\n";
  o << "  for (; t < t1; t += n_groups) {\n"
    << "    const long long dcur = dof, scur = sct + sc_off;\n"
    << "    unsigned PKc[" << NV << "];\n";
  for (int u = 0; u < NV; ++u) o << "    PKc[" << u << "] = PK[" << u << "];\n";
  o << "    const unsigned fastc = fastm;\n";
  for (int i = 0; i < p.n_swaps; ++i) emit_swap(o, 1, NW, p.swap_a[i], p.swap_b[i], "R");
  const int ga = GWd >= 2 ? p.gsel_a : -1, gb = GWd >= 4 ? p.gsel_b : -1;
  for (int j = 0; j < NG; ++j) {
    o << "    asm volatile(\"st.shared.";
    if (GWd == 4) o << "v4.b32 [%0], {%1,%2,%3,%4};\"";
    else if (GWd == 2) o << "v2.b32 [%0], {%1,%2};\"";
    else o << "b32 [%0], %1;\"";
    o << " :: \"r\"(sbase + buf + (swx ^ " << p.sw_gran[j] << "u))";
    for (int k = 0; k < GWd; ++k) o << ", \"r\"(R[" << deposit_word_h(j, k, LB, ga, gb) << "])";
    o << " : \"memory\");\n";
  }
  o << "    { const long long tn = t + n_groups; if (tn < t1) { tile_off(tn);\n";
  load("      ");
  o << "    } }\n";
  if (gw == 0) o << "    __syncwarp();\n";
  else o << "    asm volatile(\"bar.sync %0, %1;\" :: \"r\"(group + 1), \"r\"(" << (32 << gw) << ") : \"memory\");\n";
  for (int j = 0; j < NG; ++j) {
    o << "    asm volatile(\"ld.shared.";
    if (GWd == 4) o << "v4.b32 {%0,%1,%2,%3}, [%4];\" : \"=r\"(Q[" << 4 * j << "]), \"=r\"(Q[" << 4 * j + 1
                    << "]), \"=r\"(Q[" << 4 * j + 2 << "]), \"=r\"(Q[" << 4 * j + 3 << "])";
    else if (GWd == 2) o << "v2.b32 {%0,%1}, [%2];\" : \"=r\"(Q[" << 2 * j << "]), \"=r\"(Q[" << 2 * j + 1 << "])";
    else o << "b32 %0, [%1];\" : \"=r\"(Q[" << j << "])";
    o << " : \"r\"(sbase + buf + (srx ^ " << p.sr_gran[j] << "u)) : \"memory\");\n";
  }
  // decode + two 256-bit stores per packed vector
  for (int u = 0; u < NV; ++u) {
    o << "    { unsigned char* op = dst + 4 * (dbase + dcur + " << p.st_vec[u] << ");\n"
      << "      unsigned o8[16]; const unsigned pk = PKc[" << u << "];\n"
      << "      if ((fastc >> " << u << ") & 1u) {\n"
      << "        const unsigned plo = (pk << 7) & 0x80808080u, phi = (pk >> 1) & 0x7F7F7F7Fu;\n";
    for (int q = 0; q < 4; ++q) {
      o << "        { const unsigned wq = Q[" << 4 * u + q << "];\n"
        << "          const unsigned m = wq & 0x77777777u, mh = m >> 16, x = wq & 0x88888888u;\n"
        << "          const unsigned L01 = __byte_perm(0xC0800000u, 0xC0804000u, m), H01 = __byte_perm(0x3F3F3F00u, 0x40404040u, m);\n"
        << "          const unsigned L23 = __byte_perm(0xC0800000u, 0xC0804000u, mh), H23 = __byte_perm(0x3F3F3F00u, 0x40404040u, mh);\n";
      for (int k = 0; k < 4; ++k) {
        const int e = 4 * q + k;
        o << "          { const unsigned mag = __byte_perm(" << (k < 2 ? "L01" : "L23") << ", "
          << (k < 2 ? "H01" : "H23") << ", " << ((k & 1) ? 0x7362 : 0x5140) << ");\n"
          << "            const unsigned tt = __byte_perm(x, 0u, " << (0x4440 | k) << ") * 0x01001000u;\n"
          << "            o8[" << 4 * q + k << "] = bf16x2_mul(mag | (tt & 0x80008000u), __byte_perm(plo, phi, "
          << p.sc_sel[e] << "u)); }\n";
      }
      o << "        }\n";
    }
    o << "      } else {\n";
    for (int e = 0; e < 16; ++e)
      o << "        { const unsigned byte = (Q[" << 4 * u + (e >> 2) << "] >> " << (e & 3) * 8
        << ") & 0xFFu; const unsigned sb = (pk >> " << 8 * p.sc_slot[e]
        << ") & 0xFFu; const float sf = __uint_as_float(mx_scale_f32(sb));\n"
        << "          const unsigned lo = __float_as_uint(__fmul_rn(__uint_as_float(e2m1_f32(byte & 15u)), sf));\n"
        << "          const unsigned hi = __float_as_uint(__fmul_rn(__uint_as_float(e2m1_f32(byte >> 4)), sf));\n"
        << "          o8[" << e << "] = sb == 255u ? 0x7FC07FC0u : ((hi & 0xFFFF0000u) | (lo >> 16)); }\n";
    o << "      }\n";
    for (int h = 0; h < 2; ++h)
      o << "      asm volatile(\"st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\" :: \"l\"(op + "
        << 32 * h << "), \"r\"(o8[" << 8 * h << "]), \"r\"(o8[" << 8 * h + 1 << "]), \"r\"(o8[" << 8 * h + 2
        << "]), \"r\"(o8[" << 8 * h + 3 << "]), \"r\"(o8[" << 8 * h + 4 << "]), \"r\"(o8[" << 8 * h + 5
        << "]), \"r\"(o8[" << 8 * h + 6 << "]), \"r\"(o8[" << 8 * h + 7 << "]) : \"memory\");\n";
    o << "    }\n";
  }
  o << "    buf ^= " << p.tile_bytes << "u;\n  }\n}\n";
  return o.str();
}

struct JitEntry {
  CUmodule mod = nullptr;
  CUfunction fn = nullptr;
  std::string error;   // non-empty: compiling / loading failed (not retried)
};
std::mutex g_jit_mu;
std::map<std::pair<int, std::string>, JitEntry> g_jit;

cudaError_t get_kernel(const std::string& src, CUfunction* fn, std::string* err,
                       const char* name = "ll_regs_shfl") {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_jit_mu);
  auto key = std::make_pair(dev, src);
  auto it = g_jit.find(key);
  if (it != g_jit.end()) {
    if (!it->second.error.empty()) {
      *err = it->second.error;
      return cudaErrorUnknown;
    }
    *fn = it->second.fn;
    return cudaSuccess;
  }
  auto failed = [&](const std::string& m) {
    JitEntry bad;
    bad.error = m;
    g_jit[key] = bad;
    *err = m;
    return cudaErrorUnknown;
  };
  // test hook: make every compile fail (the template-kernel fallback path);
  // not cached
  if (planner_knob("jit_force_fail", 0)) {
    *err = "jit_force_fail";
    return cudaErrorUnknown;
  }
  static PFN_LoadData load = entry<PFN_LoadData>("cuModuleLoadData");
  static PFN_GetFunction getf = entry<PFN_GetFunction>("cuModuleGetFunction");
  if (!load || !getf) return failed("driver entry points unavailable");
  cudaFree(nullptr);  // make sure the runtime's primary context is current
  // LL_JIT_SOURCE_DIR: write each generated source there and name the
  // program after it, so the line table (-lineinfo) points at a real file
  // and `ncu --import-source on` can show the generated code.
  std::string pname = "ll_jit.cu";
  if (const char* dir = std::getenv("LL_JIT_SOURCE_DIR")) {
    unsigned long long h = 1469598103934665603ull;
    for (unsigned char c : src) h = (h ^ c) * 1099511628211ull;
    char buf[64];
    std::snprintf(buf, sizeof buf, "/%s_%016llx.cu", name, h);
    pname = std::string(dir) + buf;
    if (FILE* f = std::fopen(pname.c_str(), "w")) {
      std::fwrite(src.data(), 1, src.size(), f);
      std::fclose(f);
    }
  }
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), pname.c_str(), 0, nullptr, nullptr) != NVRTC_SUCCESS)
    return failed("nvrtcCreateProgram failed");
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-default-device", "-lineinfo"};
  nvrtcResult r = nvrtcCompileProgram(prog, 4, opts);
  if (r != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, &log[0]);
    nvrtcDestroyProgram(&prog);
    return failed("NVRTC: " + log.substr(0, 400));
  }
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  std::string cubin(n, '\0');
  nvrtcGetCUBIN(prog, &cubin[0]);
  nvrtcDestroyProgram(&prog);
  JitEntry e;
  if (load(&e.mod, cubin.data()) != CUDA_SUCCESS || getf(&e.fn, e.mod, name) != CUDA_SUCCESS)
    return failed("cuModuleLoadData / cuModuleGetFunction failed");
  g_jit[key] = e;
  *fn = e.fn;
  return cudaSuccess;
}

}  // namespace

// First-wave CTA count of a compiled kernel (for gather.cpp's prefetch).
long long jit_first_wave_ctas(void* fn, int block, int smem) {
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return first_wave_ctas((CUfunction)fn, block, smem, sms);
}

// Compile (cached per source) and fetch a kernel of a generated source; the
// gather kernels (gather.cpp) use these too.
cudaError_t jit_kernel(const std::string& src, const char* name, void** fn, std::string* err) {
  CUfunction f = nullptr;
  cudaError_t e = get_kernel(src, &f, err, name);
  *fn = (void*)f;
  return e;
}

cudaError_t jit_launch(void* fn, unsigned grid, unsigned block, unsigned smem, cudaStream_t st,
                       void** args, std::string* err, bool pdl) {
  static PFN_Launch launch = entry<PFN_Launch>("cuLaunchKernel");
  static PFN_LaunchEx launch_ex = entry<PFN_LaunchEx>("cuLaunchKernelEx");
  static PFN_FuncSetAttribute setattr = entry<PFN_FuncSetAttribute>("cuFuncSetAttribute");
  if (!launch || !setattr) {
    *err = "driver entry points unavailable";
    return cudaErrorNotSupported;
  }
  if (smem > 48 * 1024) setattr((CUfunction)fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)smem);
  if (pdl && launch_ex) {
    // programmatic dependent launch: the kernel itself waits (griddepcontrol.wait)
    CUlaunchAttribute attr[1];
    attr[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
    attr[0].value.programmaticStreamSerializationAllowed = 1;
    CUlaunchConfig cfg = {};
    cfg.gridDimX = grid;
    cfg.gridDimY = cfg.gridDimZ = 1;
    cfg.blockDimX = block;
    cfg.blockDimY = cfg.blockDimZ = 1;
    cfg.sharedMemBytes = smem;
    cfg.hStream = (CUstream)st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (launch_ex(&cfg, (CUfunction)fn, args, nullptr) != CUDA_SUCCESS) {
      *err = "cuLaunchKernel failed";
      return cudaErrorLaunchFailure;
    }
    return cudaSuccess;
  }
  if (launch((CUfunction)fn, grid, 1, 1, block, 1, 1, smem, (CUstream)st, args, nullptr) != CUDA_SUCCESS) {
    *err = "cuLaunchKernel failed";
    return cudaErrorLaunchFailure;
  }
  return cudaSuccess;
}

// Compile only (no device needed): NVRTC log / status for tests.
bool nvrtc_compile_check(const std::string& src, std::string* log, size_t* cubin_bytes) {
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), "ll_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
    return false;
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-default-device"};
  const bool ok = nvrtcCompileProgram(prog, 3, opts) == NVRTC_SUCCESS;
  size_t n = 0;
  nvrtcGetProgramLogSize(prog, &n);
  log->assign(n, '\0');
  if (n) nvrtcGetProgramLog(prog, &(*log)[0]);
  *cubin_bytes = 0;
  if (ok) nvrtcGetCUBINSize(prog, cubin_bytes);
  nvrtcDestroyProgram(&prog);
  return ok;
}

std::string regs_shuffle_kernel_source(const RegsShufflePlan& p, int w) {
  return regs_shuffle_source(p, w);
}

cudaError_t launch_regs_shuffle(const RegsShufflePlan& p, int w, const void* src, void* dst,
                                int max_ctas, int reps, long long* cycles, cudaStream_t st,
                                std::string* err) {
  if (reps < 1 || w > 4) return cudaErrorInvalidValue;
  CUfunction fn = nullptr;
  cudaError_t e = get_kernel(regs_shuffle_source(p, w), &fn, err);
  if (e != cudaSuccess) return e;
  static PFN_Launch launch = entry<PFN_Launch>("cuLaunchKernel");
  if (!launch) return cudaErrorNotSupported;
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int64_t grid = std::min<int64_t>(p.n_tiles, (int64_t)sms * 16);
  if (max_ctas > 0) grid = std::min<int64_t>(grid, max_ctas);
  if (grid <= 0) return cudaSuccess;
  long long nt = p.n_tiles, tb = p.tile_bytes;
  const void* s = src;
  void* d = dst;
  void* args[] = {(void*)&s, (void*)&d, (void*)&nt, (void*)&tb, (void*)&reps, (void*)&cycles};
  if (launch(fn, (unsigned)grid, 1, 1, 32u << p.nw, 1, 1, 0, (CUstream)st, args, nullptr) !=
      CUDA_SUCCESS) {
    *err = "cuLaunchKernel failed";
    return cudaErrorLaunchFailure;
  }
  return cudaSuccess;  // launched by the driver API: no runtime error state to read
}

cudaError_t launch_shuffle_jit(const ConvertPlan& P, const void* src, void* dst, int max_ctas,
                               cudaStream_t st, const TileRange& rg, std::string* err) {
  if (!P.shuffle_ok || P.w > 4) return cudaErrorInvalidValue;
  CUfunction fn = nullptr;
  cudaError_t e = get_kernel(shuffle_hbm_source(P), &fn, err, "ll_shfl_hbm");
  if (e != cudaSuccess) return e;
  static PFN_Launch launch = entry<PFN_Launch>("cuLaunchKernel");
  if (!launch) return cudaErrorNotSupported;
  const int64_t n_tiles = rg.t1 - rg.t0;
  if (n_tiles <= 0) return cudaSuccess;
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int tpg = planner_knob("shuffle_jit_tpg", 1);  // sweep: 1 > 2 > 4 > 8
  int64_t groups = tpg > 0 ? (n_tiles + tpg - 1) / tpg : (int64_t)sms * 64;
  if (max_ctas > 0) groups = std::min<int64_t>(groups, (int64_t)max_ctas * 8);
  groups = std::max<int64_t>(1, std::min<int64_t>(groups, n_tiles));
  const int64_t grid = (groups + 7) / 8;
  long long ng = groups, t0 = rg.t0, t1 = rg.t1, ss = rg.src_shift, ds = rg.dst_shift;
  const void* s = src;
  void* d = dst;
  const bool pdl = planner_knob("shuffle_pdl", 1) != 0;
  long long pf = pdl && planner_knob("pdl_prefetch", 1) ? first_wave_ctas(fn, 256, 0, sms) : 0;
  void* args[] = {(void*)&P.shp.tile, (void*)&s, (void*)&d, (void*)&ng, (void*)&t0, (void*)&t1,
                  (void*)&ss, (void*)&ds, (void*)&pf};
  return jit_launch((void*)fn, (unsigned)grid, 256, 0, st, args, err, pdl);
}

// Register permutation (LL_PATH_REGPERM): thread c loads chunk c (2^rp_bits
// elements, contiguous in both buffers: 16-byte or 256-bit accesses),
// rebuilds it in destination order with renames / prmt (compile time) and
// stores it.  No shared memory, no shuffles.
std::string regperm_kernel_source(const ConvertPlan& P) {
  const int W = P.w, CB = W << P.rp_bits, NW = CB / 4;
  // 256-bit accesses for 64-byte chunks (lanes 64 B apart: 128-bit accesses
  // would leave every instruction half of each sector, 5157-5541 vs
  // 6376-6846 GB/s, profiles/r02/s2r vs s2f); 128-bit for 32-byte chunks
  // (1.7 % faster for 1-byte elements, equal for 4-byte); knob regperm_v8:
  // 1 = always (>= 32-byte chunks), 0 = never
  const int v8k = planner_knob("regperm_v8", -1);
  const bool v8 = CB >= 32 && (v8k < 0 ? CB >= 64 : v8k != 0);
  const int step = v8 ? 32 : 16;
  // U chunks per thread and iteration, all loads issued first: >= 64 bytes
  // in flight per thread (one 32-byte chunk alone ran at 0.89 of the smem
  // path, profiles/r02/classify)
  const int U = planner_knob("regperm_u", 0) > 0 ? planner_knob("regperm_u", 0) : std::max(1, 64 / CB);
  std::ostringstream o;
  o << "extern \"C\" __global__ void __launch_bounds__(256) ll_regperm(\n"
    << "    const unsigned char* __restrict__ src, unsigned char* __restrict__ dst, long long t0,\n"
    << "    long long t1, long long src_shift, long long dst_shift, long long pf_ctas) {\n";
  const bool pdl = planner_knob("pdl", 1) != 0;
  // the first wave's L2 prefetch of its first chunks before the wait (knob
  // regperm_prefetch, as the smem kernel's pdl_prefetch): one prefetch per
  // 128-byte line.  Off by default: measured 0.8-1.2 % slower at every
  // element width (profiles/r02/s3h/ab_regperm.jsonl)
  if (pdl && planner_knob("regperm_prefetch", 0)) {
    o << "  if (blockIdx.x < pf_ctas) {\n";
    for (int u = 0; u < U; ++u)
      for (int off = 0; off < CB; off += 128)
        o << "    { const long long c = t0 + (long long)blockIdx.x * " << U << " * blockDim.x + threadIdx.x + "
          << u << "LL * blockDim.x; const unsigned char* a_ = src + c * " << CB << " + " << off
          << " - src_shift; if (c < t1 && (((unsigned long long)a_) & 127ull) == 0) "
          << "asm volatile(\"prefetch.global.L2 [%0];\" :: \"l\"(a_)); }\n";
    o << "  }\n";
  }
  if (pdl) o << "  asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");\n";
  o << "  for (long long c0 = t0 + (long long)blockIdx.x * " << U << " * blockDim.x + threadIdx.x; c0 < t1;\n"
    << "       c0 += (long long)gridDim.x * " << U << " * blockDim.x) {\n"
    << "    unsigned R[" << U << "][" << NW << "];\n";
  for (int u = 0; u < U; ++u) {
    o << "    { const long long c = c0 + " << u << "LL * blockDim.x; if (c < t1) {\n"
      << "      const unsigned char* s = src + c * " << CB << " - src_shift;\n";
    for (int off = 0; off < CB; off += step) {
      const int k = off / 4, nw = step / 4;
      o << "      asm volatile(\"ld.global.nc.L1::no_allocate.v" << nw << ".u32 {";
      for (int q = 0; q < nw; ++q) o << (q ? "," : "") << "%" << q;
      o << "}, [%" << nw << "];\" : ";
      for (int q = 0; q < nw; ++q) o << (q ? ", " : "") << "\"=r\"(R[" << u << "][" << k + q << "])";
      o << " : \"l\"(s + " << off << "));\n";
    }
    o << "    } }\n";
  }
  if (pdl) o << "    asm volatile(\"griddepcontrol.launch_dependents;\");\n";
  for (int u = 0; u < U; ++u) {
    o << "    { const long long c = c0 + " << u << "LL * blockDim.x; if (c < t1) {\n"
      << "      unsigned char* d = dst + c * " << CB << " - dst_shift;\n";
    const std::string Ru = "R[" + std::to_string(u) + "]";
    for (int q = 0; q < NW; ++q) {
      std::vector<std::pair<std::string, int>> bs;
      for (int b = 0; b < 4; ++b) {
        const int byte = 4 * q + b, e = byte / W, eb = byte % W;
        const int sbyte = P.rp_src[e] * W + eb;
        bs.push_back(std::make_pair(Ru + "[" + std::to_string(sbyte >> 2) + "]", sbyte & 3));
      }
      o << "      const unsigned Q" << q << " = " << pack_bytes(bs) << ";\n";
    }
    for (int off = 0; off < CB; off += step) {
      const int k = off / 4, nw = step / 4;
      o << "      asm volatile(\"st.global.cs.v" << nw << ".b32 [%0], {";
      for (int q = 0; q < nw; ++q) o << (q ? "," : "") << "%" << q + 1;
      o << "};\" :: \"l\"(d + " << off << ")";
      for (int q = 0; q < nw; ++q) o << ", \"r\"(Q" << k + q << ")";
      o << " : \"memory\");\n";
    }
    o << "    } }\n";
  }
  o << "  }\n}\n";
  return o.str();
}

cudaError_t launch_regperm_jit(const ConvertPlan& P, const void* src, void* dst, int max_ctas,
                               cudaStream_t st, const TileRange& rg, std::string* err) {
  CUfunction fn = nullptr;
  cudaError_t e = get_kernel(regperm_kernel_source(P), &fn, err, "ll_regperm");
  if (e != cudaSuccess) return e;
  const int64_t n = rg.t1 - rg.t0;
  if (n <= 0) return cudaSuccess;
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int U = planner_knob("regperm_u", 0) > 0 ? planner_knob("regperm_u", 0)
                                                 : std::max(1, 64 / (P.w << P.rp_bits));
  // knob regperm_waves: CTAs per SM of a grid-stride launch; 0 (default):
  // one pass, every thread U chunks (profiles/r02/s2e/regperm_sweep.jsonl:
  // 6804-6814 vs 6235 GB/s with 8 CTAs per SM striding, w = 4)
  const int waves = planner_knob("regperm_waves", 0);
  int64_t grid = (n + 256 * U - 1) / (256 * U);
  if (waves > 0) grid = std::min<int64_t>(grid, (int64_t)sms * waves);
  if (max_ctas > 0) grid = std::min<int64_t>(grid, max_ctas);
  grid = std::max<int64_t>(1, std::min<int64_t>(grid, 0x7fffffff));
  long long t0 = rg.t0, t1 = rg.t1, ss = rg.src_shift, ds = rg.dst_shift;
  const void* s = src;
  void* d = dst;
  // knob regperm_occ: CTAs per SM (occupancy capped through dynamic shared
  // memory the kernel does not use; 0 = no cap)
  const int occ = planner_knob("regperm_occ", 0);
  unsigned smem = occ > 0 ? (unsigned)std::min(227 * 1024, 228 * 1024 / occ - 1024) : 0u;
  long long pf = planner_knob("pdl", 1) && planner_knob("regperm_prefetch", 0)
                     ? first_wave_ctas(fn, 256, (int)smem, sms) : 0;
  void* args[] = {(void*)&s, (void*)&d, (void*)&t0, (void*)&t1, (void*)&ss, (void*)&ds, (void*)&pf};
  static PFN_FuncSetAttribute setattr = entry<PFN_FuncSetAttribute>("cuFuncSetAttribute");
  if (smem > 48 * 1024 && setattr) setattr(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)smem);
  static PFN_LaunchEx launch_ex = entry<PFN_LaunchEx>("cuLaunchKernelEx");
  if (planner_knob("pdl", 1) && launch_ex) {
    CUlaunchAttribute attr[1];
    attr[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
    attr[0].value.programmaticStreamSerializationAllowed = 1;
    CUlaunchConfig cfg = {};
    cfg.gridDimX = (unsigned)grid;
    cfg.gridDimY = cfg.gridDimZ = 1;
    cfg.blockDimX = 256;
    cfg.blockDimY = cfg.blockDimZ = 1;
    cfg.sharedMemBytes = smem;
    cfg.hStream = (CUstream)st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (launch_ex(&cfg, fn, args, nullptr) != CUDA_SUCCESS) {
      *err = "cuLaunchKernel failed";
      return cudaErrorLaunchFailure;
    }
    return cudaSuccess;
  }
  void* f = (void*)fn;
  return jit_launch(f, (unsigned)grid, 256, smem, st, args, err);
}

std::string shuffle_hbm_kernel_source(const ConvertPlan& P) { return shuffle_hbm_source(P); }
std::string smem_hbm_kernel_source(const ConvertPlan& P) {
  return smem_hbm_source(P, planner_knob("smem_jit_single", 0) != 0);
}
std::string upcast_hbm_kernel_source(const ConvertPlan& P) { return upcast_hbm_source(P); }

cudaError_t launch_upcast_jit(const ConvertPlan& P, const void* src, void* dst,
                              const uint8_t* scales, int max_ctas, cudaStream_t st,
                              const TileRange& rg, std::string* err) {
  if (P.op != 1 || P.sp.sc_nz > 2 || P.w != 1) return cudaErrorInvalidValue;
  {
    // the 256-bit stores need NVRTC >= 12.9 (the process may have loaded an
    // older libnvrtc.so.12 first, e.g. PyTorch's bundled copy)
    int major = 0, minor = 0;
    nvrtcVersion(&major, &minor);
    if (major < 12 || (major == 12 && minor < 9)) {
      *err = "NVRTC " + std::to_string(major) + "." + std::to_string(minor) + " < 12.9";
      return cudaErrorNotSupported;
    }
  }
  CUfunction fn = nullptr;
  cudaError_t e = get_kernel(upcast_hbm_source(P), &fn, err, "ll_upcast_hbm");
  if (e != cudaSuccess) return e;
  static PFN_Launch launch = entry<PFN_Launch>("cuLaunchKernel");
  static PFN_FuncSetAttribute setattr = entry<PFN_FuncSetAttribute>("cuFuncSetAttribute");
  if (!launch || !setattr) return cudaErrorNotSupported;
  const int64_t n_tiles = rg.t1 - rg.t0;
  if (n_tiles <= 0) return cudaSuccess;
  const int gpc = 8 >> P.sp.gw;
  const int smem = gpc * 2 * P.sp.tile_bytes;
  if (smem > 48 * 1024) setattr(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, smem);
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // tiles per group (sweep on B200: 4-8 -> 6.49-6.50 TB/s, persistent 5.81)
  const int tpg = planner_knob("upcast_jit_tpg", 4);
  int64_t groups = tpg > 0 ? (n_tiles + tpg - 1) / tpg : (int64_t)sms * 2 * gpc;
  if (max_ctas > 0) groups = std::min<int64_t>(groups, (int64_t)max_ctas * gpc);
  groups = std::max<int64_t>(1, std::min<int64_t>(groups, n_tiles));
  const int64_t grid = (groups + gpc - 1) / gpc;
  long long ng = groups, t0 = rg.t0, t1 = rg.t1, ss = rg.src_shift, ds = rg.dst_shift;
  const void* s = src;
  void* d = dst;
  const void* sc = scales;
  void* args[] = {(void*)&P.sp.tile, (void*)&s, (void*)&d, (void*)&ng, (void*)&t0, (void*)&t1,
                  (void*)&ss, (void*)&ds, (void*)&sc};
  return jit_launch((void*)fn, (unsigned)grid, 256, (unsigned)smem, st, args, err,
                    planner_knob("upcast_pdl", 0) != 0);
}

cudaError_t launch_smem_jit(const ConvertPlan& P, const void* src, void* dst, int max_ctas,
                            cudaStream_t st, const TileRange& rg, std::string* err) {
  if (P.sp.pad || P.op != 0) return cudaErrorInvalidValue;
  static PFN_Launch launch = entry<PFN_Launch>("cuLaunchKernel");
  static PFN_FuncSetAttribute setattr = entry<PFN_FuncSetAttribute>("cuFuncSetAttribute");
  if (!launch || !setattr) return cudaErrorNotSupported;
  const int64_t n_tiles = rg.t1 - rg.t0;
  if (n_tiles <= 0) return cudaSuccess;
  const int gpc = 8 >> P.sp.gw;
  const int tpg = planner_knob("smem_jit_tpg", 1);  // sweep: 1 > 2 > 4
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int64_t groups = tpg > 0 ? (n_tiles + tpg - 1) / tpg : (int64_t)sms * 4 * gpc;
  if (max_ctas > 0) groups = std::min<int64_t>(groups, (int64_t)max_ctas * gpc);
  groups = std::max<int64_t>(1, std::min<int64_t>(groups, n_tiles));
  const int64_t grid = (groups + gpc - 1) / gpc;
  const bool single = groups >= n_tiles && planner_knob("smem_jit_single", 0);
  CUfunction fn = nullptr;
  cudaError_t e = get_kernel(smem_hbm_source(P, single), &fn, err, "ll_smem_hbm");
  if (e != cudaSuccess) return e;
  const int smem = gpc * (single ? 1 : 2) * P.sp.tile_bytes;
  if (smem > 48 * 1024) setattr(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, smem);
  long long ng = groups, t0 = rg.t0, t1 = rg.t1, ss = rg.src_shift, ds = rg.dst_shift;
  // the first wave: CTAs that can be resident at once (pdl_prefetch)
  long long pf = planner_knob("pdl_prefetch", 1) ? first_wave_ctas(fn, 256, smem, sms) : 0;
  // knob pdl_prefetch_short: every CTA prefetches in launches of <= 2 waves
  // (strong-scaling shards).  Off: config 5's N = 8 shard measured 6751 vs
  // 6690 GB/s in one run (profiles/r02/s3f) and 6603 vs 6689 in the next
  // (s3k) -- inside the run-to-run spread
  if (pf > 0 && grid <= 2 * pf && planner_knob("pdl_prefetch_short", 0)) pf = grid;
  const void* s = src;
  void* d = dst;
  void* args[] = {(void*)&P.sp.tile, (void*)&s, (void*)&d, (void*)&ng, (void*)&t0, (void*)&t1,
                  (void*)&ss, (void*)&ds, (void*)&pf};
  static PFN_LaunchEx launch_ex = entry<PFN_LaunchEx>("cuLaunchKernelEx");
  CUresult r;
  if (planner_knob("pdl", 1) && launch_ex) {
    CUlaunchAttribute attr[1];
    attr[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
    attr[0].value.programmaticStreamSerializationAllowed = 1;
    CUlaunchConfig cfg = {};
    cfg.gridDimX = (unsigned)grid;
    cfg.gridDimY = cfg.gridDimZ = 1;
    cfg.blockDimX = 256;
    cfg.blockDimY = cfg.blockDimZ = 1;
    cfg.sharedMemBytes = (unsigned)smem;
    cfg.hStream = (CUstream)st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    r = launch_ex(&cfg, fn, args, nullptr);
  } else {
    r = launch(fn, (unsigned)grid, 1, 1, 256, 1, 1, (unsigned)smem, (CUstream)st, args, nullptr);
  }
  if (r != CUDA_SUCCESS) {
    *err = "cuLaunchKernel failed";
    return cudaErrorLaunchFailure;
  }
  return cudaSuccess;  // launched by the driver API: no runtime error state to read
}

// ------------------------------------------------------------------------
// TMA-fed conversion compiled per plan (LL_PATH_SMEM_TMA / _TMA_STORE,
// knob tma_jit).  Warp-specialised and persistent: one producer warp per CTA
// (one elected lane) streams the CTA's source tiles into an NS-stage ring
// with cp.async.bulk.tensor (one box per tile, mbarrier complete_tx); K
// consumer groups of 2^gw warps each own one slot per stage, wait on the
// slot's full barrier, read their 16-byte granules (the planner's
// conflict-free reader lanes), release the slot on its empty barrier (one
// arrival per warp) and then either store their destination vectors with
// st.global.cs (tma_store = false) or write them into one of two
// destination images and let one lane store the image with a TMA tensor
// store (tma_store = true).  Every offset, permutation, box coordinate
// shift and stage count is a compile-time constant.
std::string tma_hbm_source(const ConvertPlan& P, bool tma_store, int NS, int K, int NI) {
  const SmemPlan& p = P.sp;
  const int W = P.w, NV = P.nv, NW = NV * 4, gw = p.gw, LB = ilog2i(NW), lw = ilog2i(W);
  const int NC = K << gw;   // consumer warps
  const TmaDesc& ts = P.td;
  const TmaDesc& tq = P.td_dst;
  const uint32_t TB = (uint32_t)p.tile_bytes;
  const int ga = p.gsel_a, gb = p.gsel_b;
  const bool pdl = planner_knob("pdl", 1) != 0;
  std::ostringstream o;
  o << "struct TileTab { long long src, dst, sc; };\n"
    << "struct TileMap { long long n_tiles; int n_bits; int n_tab; long long bss, bsd; TileTab tab["
    << LL_MAX_TAB << "][" << (1 << LL_TAB_BITS) << "]; };\n"
    << "struct __align__(64) TMap { unsigned long long v[16]; };\n"
    << "__device__ __forceinline__ void mwait(unsigned b, unsigned ph) {\n"
    << "  asm volatile(\"{\\n.reg .pred p;\\nW_%=:\\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\\n@!p bra W_%=;\\n}\\n\" :: \"r\"(b), \"r\"(ph) : \"memory\");\n}\n"
    << "extern \"C\" __global__ void __launch_bounds__(" << 32 * (NC + 1) << ", 1) ll_tma_hbm(\n"
    << "    const __grid_constant__ TileMap tm, const __grid_constant__ TMap tsrc,\n"
    << "    const __grid_constant__ TMap tdst, unsigned char* __restrict__ dst,\n"
    << "    long long t0, long long t1, long long src_shift, long long dst_shift) {\n"
    << "  extern __shared__ __align__(16) unsigned char smem[];\n"
    << "  __shared__ __align__(8) unsigned long long bars[" << 2 * NS * K << "];\n"
    << "  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;\n"
    << "  const unsigned sb = (((unsigned)__cvta_generic_to_shared(smem)) + 1023u) & ~1023u;\n"
    << "  const unsigned full0 = (unsigned)__cvta_generic_to_shared(bars), empty0 = full0 + "
    << 8 * NS * K << "u;\n"
    << "  if (threadIdx.x == 0) {\n"
    << "    for (int i = 0; i < " << NS * K << "; ++i) {\n"
    << "      asm volatile(\"mbarrier.init.shared::cta.b64 [%0], 1;\" :: \"r\"(full0 + 8 * i) : \"memory\");\n"
    << "      asm volatile(\"mbarrier.init.shared::cta.b64 [%0], " << (1 << gw)
    << ";\" :: \"r\"(empty0 + 8 * i) : \"memory\");\n"
    << "    }\n"
    << "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n"
    << "  }\n"
    << "  __syncthreads();\n";
  if (pdl) o << "  asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");\n";
  o << "  const long long rmask = (1LL << tm.n_bits) - 1;\n"
    << "  auto tile_off = [&](long long t, long long& so, long long& dof) {\n"
    << "    const long long inst = t >> tm.n_bits, r = t & rmask;\n"
    << "    so = inst * tm.bss; dof = inst * tm.bsd;\n";
  for (int k = 0; k < p.tile.n_tab; ++k)
    o << "    { const TileTab& e = tm.tab[" << k << "][(int)((r >> " << k * LL_TAB_BITS << ") & "
      << ((1 << LL_TAB_BITS) - 1) << ")]; so += e.src; dof += e.dst; }\n";
  o << "  };\n";
  auto regs = [&](int nd, int first) {
    std::ostringstream c;
    c << "{";
    for (int i = 0; i < nd; ++i) c << (i ? ", " : "") << "%" << first + i;
    c << "}";
    return c.str();
  };
  // producer: the last warp, one lane
  o << "  if (warp == " << NC << ") {\n"
    << "    if (lane == 0) {\n"
    << "      int s = 0; unsigned ph = 0;\n"
    << "      for (long long base = t0 + (long long)blockIdx.x * " << K << "; base < t1; base += (long long)gridDim.x * "
    << K << ") {\n";
  for (int g = 0; g < K; ++g) {
    o << "        { const long long t = base + " << g << "; if (t < t1) {\n"
      << "          const unsigned fb = full0 + 8u * (s * " << K << " + " << g << "), eb = empty0 + 8u * (s * " << K
      << " + " << g << ");\n"
      << "          mwait(eb, ph ^ 1u);\n"   // first pass: the preceding phase counts as complete
      << "          long long so, dof; tile_off(t, so, dof);\n"
      << "          const long long e = (so - src_shift) >> " << lw << ";\n"
      << "          asm volatile(\"mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\" :: \"r\"(fb), \"r\"("
      << TB << "u) : \"memory\");\n"
      << "          asm volatile(\"cp.async.bulk.tensor." << ts.ndim
      << "d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, " << regs(ts.ndim, 2) << "], [%"
      << 2 + ts.ndim << "];\" :: \"r\"(sb + (unsigned)(s * " << K << " + " << g << ") * " << TB
      << "u), \"l\"(&tsrc), ";
    {
      // each coordinate as its own operand
      for (int i = 0; i < ts.ndim; ++i) {
        o << "\"r\"((int)((e >> " << ts.shift[i] << ")";
        if (i + 1 < ts.ndim) o << " & " << ((1LL << ts.size_bits[i]) - 1) << "LL";
        o << ")), ";
      }
    }
    o << "\"r\"(fb) : \"memory\");\n"
      << "        } }\n";
  }
  o << "        if (++s == " << NS << ") { s = 0; ph ^= 1u; }\n";
  if (pdl) o << "        if (base == t0 + (long long)blockIdx.x * " << K << ") asm volatile(\"griddepcontrol.launch_dependents;\");\n";
  o << "      }\n"
    << "    }\n"
    << "    return;\n"
    << "  }\n";
  // consumers
  o << "  const int g = warp >> " << gw << ";\n"
    << "  const int tb = lane | ((warp & " << ((1 << gw) - 1) << ") << 5);\n"
    << "  unsigned st_off = 0, srx = 0, swx = 0;\n";
  for (int b = 0; b < 5 + gw; ++b)
    o << "  if (tb & " << (1 << b) << ") { st_off += " << p.st_thr[b] << "u; srx ^= " << p.sr_thr[b]
      << "u; swx ^= " << p.sw_thr[b] << "u; }\n";
  o << "  unsigned char* dthr = dst + st_off - dst_shift;\n"
    << "  (void)dthr; (void)swx;\n";
  if (tma_store)
    o << "  const unsigned db0 = sb + " << NS * K << "u * " << TB << "u + (unsigned)g * " << NI * TB << "u;\n"
      << "  unsigned it = 0;\n";
  o << "  int s = 0; unsigned ph = 0;\n"
    << "  for (long long t = t0 + (long long)blockIdx.x * " << K << " + g; t < t1; t += (long long)gridDim.x * " << K
    << ") {\n"
    << "    const unsigned slot = (unsigned)(s * " << K << ") + (unsigned)g;\n"
    << "    mwait(full0 + 8u * slot, ph);\n"
    << "    unsigned Q[" << NW << "];\n"
    << "    const unsigned rb = sb + slot * " << TB << "u;\n";
  for (int j = 0; j < NV; ++j)
    o << "    asm volatile(\"ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];\" : \"=r\"(Q[" << 4 * j << "]), \"=r\"(Q["
      << 4 * j + 1 << "]), \"=r\"(Q[" << 4 * j + 2 << "]), \"=r\"(Q[" << 4 * j + 3 << "]) : \"r\"(rb + (srx ^ "
      << p.sr_gran[j] << "u)) : \"memory\");\n";
  // release the slot: the warp's generic-proxy reads (LDS) are ordered
  // before the producer's next async-proxy write (TMA) into it by
  // fence.proxy.async, then one arrival per warp.  Without the fence the
  // refill overwrote slots still being read (full-size mismatches on configs
  // 2 / 3 / 5, scripts/tma_diag.py, profiles/r02/diag); knob tmaj_late
  // releases only after the tile's stores were issued
  const bool fence = planner_knob("tmaj_fence", 1) != 0, late = planner_knob("tmaj_late", 0) != 0;
  auto release = [&]() {
    if (fence) o << "    asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n";
    o << "    __syncwarp();\n"
      << "    if (lane == 0) asm volatile(\"mbarrier.arrive.shared::cta.b64 _, [%0];\" :: \"r\"(empty0 + 8u * slot) : \"memory\");\n";
  };
  if (!late) release();
  for (int i = 0; i < p.n_swaps; ++i) emit_swap(o, W, NW, p.swap_a[i], p.swap_b[i], "Q");
  o << "    long long so, dof; tile_off(t, so, dof);\n";
  if (!tma_store) {
    // 256-bit stores where a thread's destination vectors u, u + 1 are
    // adjacent: the TMA swizzle modes often force reader lanes whose 16-byte
    // vectors leave 16-byte gaps between lanes (config 2: 16-byte runs),
    // which one 32-byte store per pair closes (knob tmaj_v8)
    bool st32 = NV >= 2 && planner_knob("tmaj_v8", 1) != 0;
    for (int u = 0; st32 && u + 1 < NV; u += 2) st32 = p.st_vec[u + 1] == p.st_vec[u] + 16;
    for (int u = 0; u < NV; u += st32 ? 2 : 1) {
      if (st32) {
        o << "    asm volatile(\"st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\" :: \"l\"(dthr + dof + "
          << p.st_vec[u] << ")";
        for (int q = 0; q < 2; ++q)
          for (int k = 0; k < 4; ++k) o << ", \"r\"(Q[" << deposit_word_h(u + q, k, LB, ga, gb) << "])";
        o << " : \"memory\");\n";
        continue;
      }
      o << "    asm volatile(\"st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};\" :: \"l\"(dthr + dof + " << p.st_vec[u] << ")";
      for (int k = 0; k < 4; ++k) o << ", \"r\"(Q[" << deposit_word_h(u, k, LB, ga, gb) << "])";
      o << " : \"memory\");\n";
    }
  } else {
    const std::string gbar = gw == 0 ? std::string("__syncwarp();")
                                     : "asm volatile(\"bar.sync %0, %1;\" :: \"r\"(g + 1), \"r\"(" +
                                           std::to_string(32 << gw) + ") : \"memory\");";
    o << "    const unsigned db = db0 + (it % " << NI << "u) * " << TB << "u;\n"
      << "    if (tb == 0) asm volatile(\"cp.async.bulk.wait_group.read " << NI - 1 << ";\" ::: \"memory\");\n"
      << "    " << gbar << "\n";
    for (int j = 0; j < NV; ++j) {
      o << "    asm volatile(\"st.shared.v4.b32 [%0], {%1,%2,%3,%4};\" :: \"r\"(db + (swx ^ " << p.sw_gran[j] << "u))";
      for (int k = 0; k < 4; ++k) o << ", \"r\"(Q[" << deposit_word_h(j, k, LB, ga, gb) << "])";
      o << " : \"memory\");\n";
    }
    o << "    asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n"
      << "    " << gbar << "\n"
      << "    if (tb == 0) {\n"
      << "      const long long e = (dof - dst_shift) >> " << lw << ";\n"
      << "      asm volatile(\"cp.async.bulk.tensor." << tq.ndim << "d.global.shared::cta.bulk_group [%0, "
      << regs(tq.ndim, 1) << "], [%" << 1 + tq.ndim << "];\" :: \"l\"(&tdst), ";
    for (int i = 0; i < tq.ndim; ++i) {
      o << "\"r\"((int)((e >> " << tq.shift[i] << ")";
      if (i + 1 < tq.ndim) o << " & " << ((1LL << tq.size_bits[i]) - 1) << "LL";
      o << ")), ";
    }
    o << "\"r\"(db) : \"memory\");\n"
      << "      asm volatile(\"cp.async.bulk.commit_group;\" ::: \"memory\");\n"
      << "    }\n"
      << "    ++it;\n";
  }
  if (late) release();
  o << "    if (++s == " << NS << ") { s = 0; ph ^= 1u; }\n";
  o << "  }\n";
  if (tma_store) o << "  if (tb == 0) asm volatile(\"cp.async.bulk.wait_group 0;\" ::: \"memory\");\n";
  o << "}\n";
  return o.str();
}

namespace {
// stages / groups of the compiled TMA kernel: K consumer groups (8 consumer
// warps by default), tmaj_stages ring stages (default 2) and, for the store
// variant, two destination images per group (one when two do not fit),
// sized for tmaj_cps CTAs per SM (default 2; fewer when the tiles do not
// fit, e.g. the 32 KB tiles of config 3)
bool tma_jit_shape(const ConvertPlan& P, bool tma_store, int* ns, int* k, int* cps, size_t* smem,
                   int* ni) {
  const int gw = P.sp.gw;
  int K = planner_knob("tmaj_k", 0);
  if (K <= 0) K = std::max(1, 8 >> gw);
  if ((K << gw) > 16) return false;
  const size_t tb = (size_t)P.sp.tile_bytes;
  // default 2 stages with the non-persistent launch (tmaj_tpc = 2 tiles per
  // group and CTA; profiles/r02/s2f: config 5 6952 GB/s vs 6692 for the
  // best persistent shape, 3 stages at one CTA per SM, profiles/r02/s2d;
  // deeper rings lost up to 10 % there)
  const int want = std::min(16, planner_knob("tmaj_stages", 0) > 0 ? planner_knob("tmaj_stages", 0) : 2);
  const int img_knob = planner_knob("tmaj_images", 0);
  for (int c = std::max(1, std::min(4, planner_knob("tmaj_cps", 0) > 0 ? planner_knob("tmaj_cps", 0) : 2));
       c >= 1; --c) {
    for (int im = tma_store ? (img_knob > 0 ? std::min(2, img_knob) : 2) : 0;
         im >= (tma_store ? (img_knob > 0 ? std::min(2, img_knob) : 1) : 0); --im) {
      const size_t budget = (size_t)(227 * 1024) / c - 1024 - 1024;   // per CTA: alignment slack, reserved
      const size_t fixed = (size_t)im * K * tb;
      if (budget <= fixed) continue;
      const int n = std::min(want, (int)((budget - fixed) / (K * tb)));
      if (n < 2) continue;
      *ns = n;
      *k = K;
      *cps = c;
      *ni = std::max(1, im);
      *smem = (size_t)n * K * tb + fixed + 1024;
      return true;
    }
  }
  return false;
}
}  // namespace

std::string tma_hbm_kernel_source(const ConvertPlan& P, bool tma_store) {
  int ns, k, cps, ni;
  size_t smem;
  if (!tma_jit_shape(P, tma_store, &ns, &k, &cps, &smem, &ni)) return std::string();
  return tma_hbm_source(P, tma_store, ns, k, ni);
}

cudaError_t launch_tma_jit(const ConvertPlan& P, bool tma_store, const void* src, void* dst, int max_ctas,
                           cudaStream_t st, const TileRange& rg, std::string* err) {
  static PFN_Launch launch = entry<PFN_Launch>("cuLaunchKernel");
  static PFN_LaunchEx launch_ex = entry<PFN_LaunchEx>("cuLaunchKernelEx");
  static PFN_FuncSetAttribute setattr = entry<PFN_FuncSetAttribute>("cuFuncSetAttribute");
  if (!launch || !setattr) return cudaErrorNotSupported;
  const int64_t n_tiles = rg.t1 - rg.t0;
  if (n_tiles <= 0) return cudaSuccess;
  int ns, K, cps, ni;
  size_t smem;
  if (!tma_jit_shape(P, tma_store, &ns, &K, &cps, &smem, &ni)) {
    *err = "tma_jit: tile does not fit two stages";
    return cudaErrorInvalidConfiguration;
  }
  // tensor maps over the launch's slices (as the template kernels)
  alignas(64) unsigned char ms[128], md[128];
  std::memset(md, 0, sizeof md);
  const int64_t slice_elems = n_tiles * (int64_t(P.sp.tile_bytes) / P.w);
  cudaError_t e = encode_tma_map(ms, P.td, P.w, src, slice_elems);
  if (e == cudaSuccess && tma_store) e = encode_tma_map(md, P.td_dst, P.w, dst, slice_elems);
  if (e != cudaSuccess) {
    *err = "tma_jit: tensor map encoding failed";
    return e;
  }
  CUfunction fn = nullptr;
  e = get_kernel(tma_hbm_source(P, tma_store, ns, K, ni), &fn, err, "ll_tma_hbm");
  if (e != cudaSuccess) return e;
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // tmaj_tpc (default 2) tiles per consumer group and CTA in as many waves
  // as that takes -- several CTAs per SM, and the next launch's CTAs fill
  // SMs while this one drains (PDL); tmaj_tpc < 0: persistent, tmaj_cps
  // CTAs per SM (the persistent grid's drain cost 4-7 %, profiles/r02/s2d)
  const int tpc = planner_knob("tmaj_tpc", 0) != 0 ? planner_knob("tmaj_tpc", 0) : 2;
  int64_t grid = (n_tiles + K - 1) / K;
  if (tpc > 0) grid = (grid + tpc - 1) / tpc;
  else grid = std::min<int64_t>(grid, (int64_t)sms * cps);
  if (max_ctas > 0) grid = std::min<int64_t>(grid, max_ctas);
  grid = std::min<int64_t>(grid, 0x7fffffff);
  grid = std::max<int64_t>(1, grid);
  if (smem > 48 * 1024) setattr(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)smem);
  long long t0 = rg.t0, t1 = rg.t1, ss = rg.src_shift, ds = rg.dst_shift;
  void* d = dst;
  void* args[] = {(void*)&P.sp.tile, (void*)ms, (void*)md, (void*)&d, (void*)&t0, (void*)&t1,
                  (void*)&ss, (void*)&ds};
  const unsigned threads = 32u * ((unsigned)(K << P.sp.gw) + 1u);
  CUresult r;
  if (planner_knob("pdl", 1) && launch_ex) {
    CUlaunchAttribute attr[1];
    attr[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
    attr[0].value.programmaticStreamSerializationAllowed = 1;
    CUlaunchConfig cfg = {};
    cfg.gridDimX = (unsigned)grid;
    cfg.gridDimY = cfg.gridDimZ = 1;
    cfg.blockDimX = threads;
    cfg.blockDimY = cfg.blockDimZ = 1;
    cfg.sharedMemBytes = (unsigned)smem;
    cfg.hStream = (CUstream)st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    r = launch_ex(&cfg, fn, args, nullptr);
  } else {
    r = launch(fn, (unsigned)grid, 1, 1, threads, 1, 1, (unsigned)smem, (CUstream)st, args, nullptr);
  }
  if (r != CUDA_SUCCESS) {
    *err = "cuLaunchKernel failed";
    return cudaErrorLaunchFailure;
  }
  return cudaSuccess;
}

}  // namespace ll
