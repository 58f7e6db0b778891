// gather.cpp -- tl.gather: planning and the kernels compiled per
// plan (NVRTC) for the warp-shuffle and shared-memory gathers.
//
// out[h] = src[h*],  h* = L^{-1}( L(h) with coordinate `axis` := idx[h] ).
// With a(h) the axis coordinate of L(h) (the XOR of acol over h's bits) and
// Y the buffer vectors of the axis bits (Y_k = L^{-1} e_{axis,k}),
//     h* = h ^ Y(a(h) ^ idx[h]),
// so a gather never leaves the aligned unit of 2^U buffer elements spanned by
// the Y's low bits (U = top bit of span(Y) + 1).  Where that unit lives
// decides the executor (the shuffle gather needs L_warp^axis = 0;
// reading A20: and L_block^axis = 0):
//   * shuffle: the unit fits a warp's registers in the free (coalesced)
//     mapping -- lane l holds the 16-byte vectors l, l + 32, ... of the unit;
//     every output takes 2^|Y_reg| candidate shuffles from the lane that owns
//     its source (reading A19), every register index a compile-time constant;
//   * smem: the unit fits a CTA's shared memory -- one cp.async.bulk (TMA
//     1-D bulk copy) per unit into a 2-stage ring, then one LDS per output;
//   * direct (kernel_misc.cu): sources read through L1, any layout.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <sstream>

#include "planner.hpp"
#include "planner_internal.hpp"

namespace ll {

using detail::ilog2i;

namespace {

constexpr int kMaxWarpVec = 16;          // 16-byte vectors per lane per warp unit
constexpr int kSmemUnitMax = 96 * 1024;  // bytes per stage (source + indices) of the smem gather

int top_bit(u64 x) { return x ? 63 - __builtin_clzll(x) : -1; }

std::vector<u64> span_of(const std::vector<u64>& gens) {
  std::vector<u64> s{0};
  F2Basis b;
  for (u64 g : gens) {
    if (!g || !b.add(g)) continue;
    const size_t n0 = s.size();
    for (size_t i = 0; i < n0; ++i) s.push_back(s[i] ^ g);
  }
  return s;
}

}  // namespace

std::shared_ptr<GatherPlanHost> build_gather_plan(const Layout& L, int axis, int w, int path_req,
                                                  int64_t batch) {
  if (axis < 0 || axis >= (int)L.out.size()) throw Error(LL_ERR_ARG, "gather: axis out of range");
  const int n = L.in_bits();
  if (n != L.out_bits() || !L.surjective())
    throw Error(LL_ERR_UNSUPPORTED, "gather: the layout must be a bijection (no broadcasting)");
  auto P = std::make_shared<GatherPlanHost>();
  P->w = w;
  P->n = n;
  P->batch = batch;
  GatherPlan& g = P->gp;
  g = GatherPlan{};
  const int vb = ilog2i(16 / w);
  P->vb = vb;
  if (n < vb) throw Error(LL_ERR_UNSUPPORTED, "gather: tensor smaller than one 16-byte vector");
  g.nbits = n;
  g.batch_stride = int64_t(1) << n;
  g.ax_shift = L.out_shift(axis);
  g.ax_bits = L.out[axis].bits;
  if (g.ax_bits > 31) throw Error(LL_ERR_UNSUPPORTED, "gather: axis too long");
  for (int k = 0; k < n; ++k) g.L[k] = (int64_t)L.cols[k];
  auto Linv = f2_right_inverse(L.cols, L.out_bits());
  bool contig = true;
  int64_t amask = 0;
  const uint32_t mask = g.ax_bits >= 32 ? 0xFFFFFFFFu : ((1u << g.ax_bits) - 1);
  for (int k = 0; k < g.ax_bits; ++k) {
    g.Y[k] = (int64_t)Linv[g.ax_shift + k];
    P->Y.push_back(Linv[g.ax_shift + k]);
    amask |= g.Y[k];
    if (g.Y[k] != (int64_t(1) << (ctz64(Linv[g.ax_shift]) + k))) contig = false;
  }
  for (int b = 0; b < n; ++b) P->acol.push_back((uint32_t)(L.cols[b] >> g.ax_shift) & mask);
  // the direct kernel's field insert h* = (h & ~M) | (idx << y_base) needs
  // a(h) to be exactly that field: contiguous unit Y and no other column
  // with an axis component
  bool onehot = contig;
  for (int b = 0; b < n && onehot; ++b) {
    const int y0 = g.ax_bits ? ctz64(Linv[g.ax_shift]) : 0;
    const bool in_field = b >= y0 && b < y0 + g.ax_bits;
    onehot = P->acol[b] == (in_field ? (1u << (b - y0)) : 0u);
  }
  g.y_contig = onehot ? 1 : 0;
  g.y_base = g.ax_bits ? ctz64(Linv[g.ax_shift]) : 0;
  g.axis_mask_buf = amask;
  g.vb = vb;
  g.cand_mask = (int32_t)(amask & ((1 << vb) - 1));
  g.n_vec = (int64_t(1) << (n - vb)) * batch;
  // the unit closed under the gather, and the two unit-local executors
  P->unit_bits = top_bit((u64)amask) + 1;
  P->warp_bits = std::max(P->unit_bits, vb + 5);
  P->cta_bits = std::max(P->unit_bits, vb + 8 + std::max(0, planner_knob("gather_cta_extra", 0)));
  P->shuffle_ok = n >= P->warp_bits && P->warp_bits - vb - 5 <= ilog2i(kMaxWarpVec) && w <= 8;
  P->smem_ok = n >= P->cta_bits && (int64_t(w + 4) << P->cta_bits) <= kSmemUnitMax;
  // the paper's criterion by the labels: no warp or block bit moves the axis
  {
    bool ok = true;
    int b0 = 0;
    for (const Dim& d : L.in) {
      if (d.name == "warp" || d.name == "block")
        for (int k = 0; k < d.bits; ++k) ok = ok && P->acol[b0 + k] == 0;
      b0 += d.bits;
    }
    P->paper_criterion = ok;
  }
  int path = path_req;
  // AUTO (measured on B200): the shared-memory gather whenever
  // the unit fits a CTA -- one-pass launches with PDL: config 4 6688 vs 6459
  // direct / 6580 shuffle GB/s, the full 4096 axis 6551 vs 4750 direct
  // (profiles/r02/s3g) -- else the direct (L1) gather.  Knob
  // gather_auto_smem: 2 = the round-1 rule (direct for warp-local units),
  // 0 = always direct.
  if (path == LL_PATH_AUTO) {
    const int ak = planner_knob("gather_auto_smem", 1);
    path = !P->smem_ok || ak == 0 || (ak == 2 && P->unit_bits <= vb + 5) ? LL_PATH_GENERIC : LL_PATH_SMEM;
  }
  if (path == LL_PATH_SHUFFLE && !P->shuffle_ok)
    throw Error(LL_ERR_UNSUPPORTED,
                "gather: shuffle path needs the axis inside one warp's registers and lanes "
                "(span of the axis vectors within the low " + std::to_string(vb + 9) +
                " buffer bits; P:722 L_warp^axis = 0)");
  if (path == LL_PATH_SMEM && !P->smem_ok)
    throw Error(LL_ERR_UNSUPPORTED,
                "gather: smem path needs the axis inside one CTA's unit of <= 96 KiB of source + indices "
                "(L_block^axis = 0, reading A20)");
  if (path != LL_PATH_SHUFFLE && path != LL_PATH_SMEM && path != LL_PATH_GENERIC)
    throw Error(LL_ERR_UNSUPPORTED, "gather: path must be auto, shuffle, smem or generic");
  P->path = path;
  std::vector<u64> yreg;
  for (u64 y : P->Y) yreg.push_back((y & ((1ull << vb) - 1)) | ((y >> (vb + 5)) << vb));
  const int d_reg = ilog2i((int)span_of(yreg).size());
  std::ostringstream js;
  js << "{\"path\":\""
     << (path == LL_PATH_SHUFFLE ? "shuffle" : path == LL_PATH_SMEM ? "smem" : "direct")
     << "\",\"nbits\":" << n << ",\"elem_bytes\":" << w << ",\"axis_bits\":" << g.ax_bits << ",\"Y\":[";
  for (int k = 0; k < g.ax_bits; ++k) js << (k ? "," : "") << g.Y[k];
  js << "],\"y_contig\":" << g.y_contig << ",\"unit_bits\":" << P->unit_bits
     << ",\"warp_unit_bits\":" << P->warp_bits << ",\"cta_unit_bits\":" << P->cta_bits
     << ",\"shuffle_ok\":" << (P->shuffle_ok ? "true" : "false")
     << ",\"smem_ok\":" << (P->smem_ok ? "true" : "false")
     << ",\"paper_criterion\":" << (P->paper_criterion ? "true" : "false")
     << ",\"cand_mask\":" << g.cand_mask << ",\"candidate_shuffles\":" << (1 << d_reg)
     << ",\"batch\":" << batch << "}";
  P->json = js.str();
  return P;
}

namespace {

// shared pieces of the generated sources ------------------------------------

const char* kElemT[] = {"", "unsigned char", "unsigned short", "", "unsigned", "", "", "",
                        "unsigned long long"};

// a_unit: the axis contribution of the unit index bits (compile-time table)
void emit_unit_axis(std::ostringstream& o, const GatherPlanHost& P, int ubits, const char* t) {
  o << "    unsigned a_unit = 0; { const long long r_ = " << t << " & " << ((1LL << (P.n - ubits)) - 1)
    << "LL;\n";
  for (int j = 0; j < P.n - ubits; ++j)
    if (P.acol[ubits + j]) o << "      if ((r_ >> " << j << ") & 1) a_unit ^= " << P.acol[ubits + j] << "u;\n";
  o << "    }\n";
}

// idx: NE int32 per 16-byte vector, loaded as 16 / 8-byte vectors
void emit_idx_load(std::ostringstream& o, int NE, const std::string& dst, const std::string& ptr) {
  if (NE >= 4) {
    for (int q = 0; q < NE / 4; ++q)
      o << "      { int4 t_ = __ldg(reinterpret_cast<const int4*>(" << ptr << ") + " << q << "); " << dst
        << "[" << 4 * q << "] = t_.x; " << dst << "[" << 4 * q + 1 << "] = t_.y; " << dst << "["
        << 4 * q + 2 << "] = t_.z; " << dst << "[" << 4 * q + 3 << "] = t_.w; }\n";
  } else {
    o << "      { int2 t_ = __ldg(reinterpret_cast<const int2*>(" << ptr << ")); " << dst << "[0] = t_.x; "
      << dst << "[1] = t_.y; }\n";
  }
}

// h* from the in-unit index hl (runtime expression) and d = a ^ idx: the
// contiguous one-hot case is a field insert, else one conditional XOR per
// axis bit
std::string hstar_expr(const GatherPlanHost& P, const std::string& hl, const std::string& d) {
  std::ostringstream e;
  bool contig = !P.Y.empty();
  for (size_t k = 0; k < P.Y.size(); ++k) contig = contig && P.Y[k] == (P.Y[0] << k) && P.Y[0] && !(P.Y[0] & (P.Y[0] - 1));
  if (contig) {
    // Y_k = 1 << (y0 + k): Y(d) = d << y0
    e << "(" << hl << " ^ (" << d << " << " << ctz64(P.Y[0]) << "))";
  } else {
    e << "(" << hl;
    for (size_t k = 0; k < P.Y.size(); ++k)
      e << " ^ (((" << d << " >> " << k << ") & 1u) ? " << (uint32_t)P.Y[k] << "u : 0u)";
    e << ")";
  }
  return e.str();
}

}  // namespace

// Warp-shuffle gather.  Warp unit = 2^WU elements (WU = warp_bits):
// lane l holds the NV 16-byte vectors u = 0..NV-1 at unit offsets
// (u << (vb + 5)) | (l << vb), i.e. register slot s = e | (u << vb) of lane l
// is element e | (l << vb) | (u << (vb + 5)).  For each output slot the
// source (lane, slot) follows from h*; the candidate source slots are
// s ^ span(Y_slot) (compile time), one shuffle per candidate word, the
// matching one selected.  MU warp units per iteration: all their loads are
// issued before the first shuffle.
std::string gather_shfl_source(const GatherPlanHost& P, int timed) {
  const int W = P.w, NE = 16 / W, vb = P.vb, WU = P.warp_bits;
  const int NV = 1 << (WU - vb - 5);
  const int NS = NV * NE;                 // element slots per lane
  const int NWD = NV * 4;                 // 32-bit words per lane
  const int mu_knob = planner_knob("gather_shfl_mu", 0);
  const int MU = timed ? 1 : mu_knob > 0 ? mu_knob : std::max(1, std::min(4 / NV, 64 / (NV * NE)));
  const uint32_t mask = (uint32_t)((1ull << P.gp.ax_bits) - 1);
  std::vector<u64> yslot;
  for (u64 y : P.Y) yslot.push_back((y & (u64)(NE - 1)) | ((y >> (vb + 5)) << vb));
  const std::vector<u64> D = span_of(yslot);
  auto aslot = [&](int s) {
    uint32_t a = 0;
    for (int b = 0; b < vb; ++b) if ((s >> b) & 1) a ^= P.acol[b];
    for (int b = 0; b < WU - vb - 5; ++b) if ((s >> (vb + b)) & 1) a ^= P.acol[vb + 5 + b];
    return a;
  };
  std::ostringstream o;
  o << "extern \"C\" __global__ void __launch_bounds__(256) ll_gather_shfl(\n"
    << "    const unsigned char* __restrict__ src, const int* __restrict__ idx,\n"
    << "    unsigned char* __restrict__ out, long long n_units, int* err, int check";
  if (timed) o << ", int reps, long long* cycles";
  o << ") {\n"
    << "  typedef " << kElemT[W] << " T;\n"
    << "  const int lane = threadIdx.x & 31;\n"
    << "  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;\n"
    << "  const long long tw = ((long long)gridDim.x * blockDim.x) >> 5;\n"
    << "  unsigned a_lane = 0;\n";
  for (int c = 0; c < 5; ++c)
    if (P.acol[vb + c]) o << "  if (lane & " << (1 << c) << ") a_lane ^= " << P.acol[vb + c] << "u;\n";
  // programmatic dependent launch (knob gather_pdl): wait for the preceding
  // grid before the first global access, let the next one launch at once
  if (!timed && planner_knob("gather_pdl", 1))
    o << "  asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");\n"
      << "  asm volatile(\"griddepcontrol.launch_dependents;\");\n";
  o << "  for (long long t0 = gw * " << MU << "; t0 < n_units; t0 += tw * " << MU << ") {\n"
    << "    unsigned V[" << MU << "][" << NWD << "]; int I[" << MU << "][" << NS << "];\n";
  for (int m = 0; m < MU; ++m) {
    o << "    if (t0 + " << m << " < n_units) { const long long base = (t0 + " << m << ") << " << WU << ";\n";
    for (int u = 0; u < NV; ++u) {
      o << "      asm volatile(\"ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\" : \"=r\"(V["
        << m << "][" << 4 * u << "]), \"=r\"(V[" << m << "][" << 4 * u + 1 << "]), \"=r\"(V[" << m << "]["
        << 4 * u + 2 << "]), \"=r\"(V[" << m << "][" << 4 * u + 3 << "]) : \"l\"(src + (base + "
        << (u << (vb + 5)) << " + (lane << " << vb << ")) * " << W << "));\n";
      std::ostringstream dst;
      dst << "(&I[" << m << "][" << u * NE << "])";
      std::ostringstream ptr;
      ptr << "idx + base + " << (u << (vb + 5)) << " + (lane << " << vb << ")";
      emit_idx_load(o, NE, dst.str(), ptr.str());
    }
    o << "    }\n";
  }
  if (timed) o << "    long long c0 = clock64(); unsigned acc = 0;\n    for (int rep = 0; rep < reps; ++rep) {\n"
               << "    unsigned z_; asm volatile(\"mov.b32 %0, 0;\" : \"=r\"(z_));\n";
  for (int m = 0; m < MU; ++m) {
    o << "    if (t0 + " << m << " < n_units) { const long long t = t0 + " << m << ";\n";
    emit_unit_axis(o, P, WU, "t");
    o << "      unsigned O[" << NWD << "];\n";
    for (int s = 0; s < NS; ++s) {
      const int e = s & (NE - 1), u = s >> vb;
      const uint32_t hl_c = (uint32_t)(e | (u << (vb + 5)));
      o << "      { int ix = I[" << m << "][" << s << "]" << (timed ? " ^ (int)z_" : "") << ";\n"
        << "        if (check && (unsigned)ix > " << mask << "u) atomicExch(err, 1);\n"
        << "        const unsigned d = (a_unit ^ a_lane ^ " << aslot(s) << "u ^ (unsigned)ix) & " << mask << "u;\n"
        << "        const unsigned hl = " << hl_c << "u | ((unsigned)lane << " << vb << ");\n"
        << "        const unsigned hs = " << hstar_expr(P, "hl", "d") << ";\n"
        << "        const int sl = (int)((hs >> " << vb << ") & 31u);\n"
        << "        const unsigned ss = (hs & " << (NE - 1) << "u) | ((hs >> " << vb + 5 << ") << " << vb << ");\n";
      // candidate slots and the words holding them
      std::vector<int> cands;
      for (u64 dv : D) cands.push_back(s ^ (int)dv);
      std::sort(cands.begin(), cands.end());
      if (W >= 4) {
        const int wpe = W / 4;
        o << "        unsigned v0 = 0" << (wpe == 2 ? ", v1 = 0" : "") << ";\n";
        for (int c : cands) {
          for (int q = 0; q < wpe; ++q)
            o << "        { const unsigned g_ = __shfl_sync(0xffffffffu, V[" << m << "][" << c * wpe + q
              << "], sl); if (ss == " << c << "u) v" << q << " = g_; }\n";
        }
        o << "        O[" << s * wpe << "] = v0;";
        if (wpe == 2) o << " O[" << s * wpe + 1 << "] = v1;";
        o << "\n";
      } else {
        const int epw = 4 / W;   // elements per word
        std::vector<int> words;
        for (int c : cands) if (std::find(words.begin(), words.end(), c / epw) == words.end()) words.push_back(c / epw);
        o << "        unsigned wd = 0; const unsigned sw = ss / " << epw << "u;\n";
        for (int q : words)
          o << "        { const unsigned g_ = __shfl_sync(0xffffffffu, V[" << m << "][" << q
            << "], sl); if (sw == " << q << "u) wd = g_; }\n";
        o << "        const unsigned val = (wd >> ((ss % " << epw << "u) * " << 8 * W << "u)) & "
          << (W == 1 ? "0xFFu" : "0xFFFFu") << ";\n";
        const int word = s / epw, sh = (s % epw) * 8 * W;
        if (s % epw == 0) o << "        O[" << word << "] = val;\n";
        else o << "        O[" << word << "] |= val << " << sh << ";\n";
      }
      o << "      }\n";
    }
    if (timed) {
      o << "      for (int q = 0; q < " << NWD << "; ++q) acc ^= O[q];\n";
      o << "      if (rep == reps - 1) {\n";
    }
    o << "      const long long base = t << " << WU << ";\n";
    for (int u = 0; u < NV; ++u)
      o << "      asm volatile(\"st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};\" :: \"l\"(out + (base + "
        << (u << (vb + 5)) << " + (lane << " << vb << ")) * " << W << "), \"r\"(O[" << 4 * u << "]), \"r\"(O["
        << 4 * u + 1 << "]), \"r\"(O[" << 4 * u + 2 << "]), \"r\"(O[" << 4 * u + 3 << "]) : \"memory\");\n";
    if (timed) o << "      }\n";
    o << "    }\n";
  }
  if (timed)
    o << "    }\n    long long c1 = clock64();\n"
      << "    if (threadIdx.x == 0 && cycles) cycles[blockIdx.x] = c1 - c0;\n"
      << "    if (acc == 0x9e3779b9u && reps < 0) err[1] = 1;\n";
  o << "  }\n}\n";
  return o.str();
}

// Shared-memory gather: a CTA unit of 2^CU elements (CU = cta_bits) and its
// 2^CU indices are copied into shared memory by two cp.async.bulk (1-D TMA,
// one mbarrier with complete_tx) into a 2-stage ring; each thread then takes
// its NVT 16-byte output vectors of the unit: indices by ld.shared (16-byte,
// conflict-free), one ld.shared per output element at h* (in-unit),
// streaming 16-byte stores.  No thread issues a global load.
//
// timed: the one-CTA in-kernel study from REGISTERS (the paper's setting:
// the tensor is distributed over the threads): every repetition stores the
// thread's vectors of the unit to shared memory, synchronises, gathers with
// ld.shared and synchronises again -- the legacy staging round trip the
// shuffle gather avoids.
std::string gather_smem_source(const GatherPlanHost& P, int timed) {
  const int W = P.w, NE = 16 / W, vb = P.vb, CU = P.cta_bits;
  const int NVT = 1 << (CU - vb - 8);
  const uint32_t UB = (uint32_t)W << CU;       // source bytes per unit
  const uint32_t IB = 4u << CU;                // index bytes per unit
  const uint32_t SB = UB + IB;                 // stage bytes
  const uint32_t mask = (uint32_t)((1ull << P.gp.ax_bits) - 1);
  auto aconst = [&](int e, int j) {   // axis contribution of element bits and vector-index bits >= 8
    uint32_t a = 0;
    for (int b = 0; b < vb; ++b) if ((e >> b) & 1) a ^= P.acol[b];
    for (int b = 0; b < CU - vb - 8; ++b) if ((j >> b) & 1) a ^= P.acol[vb + 8 + b];
    return a;
  };
  std::ostringstream o;
  o << "extern \"C\" __global__ void __launch_bounds__(256) ll_gather_smem(\n"
    << "    const unsigned char* __restrict__ src, const int* __restrict__ idx,\n"
    << "    unsigned char* __restrict__ out, long long n_units, int* err, int check";
  if (timed) o << ", int reps, long long* cycles";
  else o << ", long long pf_ctas";
  o << ") {\n"
    << "  extern __shared__ __align__(128) unsigned char smem[];\n"
    << "  const int tid = threadIdx.x;\n"
    << "  const unsigned sb = (unsigned)__cvta_generic_to_shared(smem);\n"
    << "  const unsigned bar0 = sb + " << 2 * SB << "u;\n"
    << "  unsigned a_tid = 0;\n";
  for (int c = 0; c < 8; ++c)
    if (P.acol[vb + c]) o << "  if (tid & " << (1 << c) << ") a_tid ^= " << P.acol[vb + c] << "u;\n";
  o << "  if (tid == 0) {\n"
    << "    asm volatile(\"mbarrier.init.shared::cta.b64 [%0], 1;\" :: \"r\"(bar0) : \"memory\");\n"
    << "    asm volatile(\"mbarrier.init.shared::cta.b64 [%0], 1;\" :: \"r\"(bar0 + 8u) : \"memory\");\n"
    << "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n"
    << "  }\n"
    << "  __syncthreads();\n"
    << "  auto issue = [&](long long t, int s) {\n"
    << "    const unsigned bar = bar0 + 8u * s, st = sb + " << SB << "u * s;\n"
    << "    asm volatile(\"mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\" :: \"r\"(bar), \"r\"(" << SB
    << "u) : \"memory\");\n"
    << "    asm volatile(\"cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\" "
       ":: \"r\"(st), \"l\"(src + (t << " << CU << ") * " << W << "), \"r\"(" << UB << "u), \"r\"(bar) : \"memory\");\n"
    << "    asm volatile(\"cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\" "
       ":: \"r\"(st + " << UB << "u), \"l\"(idx + (t << " << CU << ")), \"r\"(" << IB << "u), \"r\"(bar) : \"memory\");\n"
    << "  };\n"
    << "  const long long g0 = blockIdx.x, gs = gridDim.x;\n";
  // first-wave L2 prefetch of the units of this CTA and the CTAs replacing
  // it in waves 2..K (knob gather_prefetch_waves, default 1; one bulk
  // prefetch per unit's source and indices) before the PDL wait, as the smem
  // conversion: config 4 6689 -> 6770 GB/s, the full axis 6550 -> 6853
  // (profiles/r02/s3z; K = 2, 3 lose part of it)
  const int gpk = std::max(0, std::min(4, planner_knob("gather_prefetch_waves", 1)));
  if (!timed && planner_knob("gather_pdl", 1) && gpk > 0) {
    o << "  if (tid == 0 && blockIdx.x < pf_ctas) {\n";
    for (int k = 0; k < gpk; ++k)
      o << "    { const long long t = g0 + " << k << "LL * pf_ctas; if (t < n_units) {\n"
        << "      asm volatile(\"cp.async.bulk.prefetch.L2.global [%0], %1;\" :: \"l\"(src + (t << " << CU << ") * " << W
        << "), \"r\"(" << UB << "u) : \"memory\");\n"
        << "      asm volatile(\"cp.async.bulk.prefetch.L2.global [%0], %1;\" :: \"l\"(idx + (t << " << CU
        << ")), \"r\"(" << IB << "u) : \"memory\"); } }\n";
    o << "  }\n";
  }
  if (!timed && planner_knob("gather_pdl", 1))   // programmatic dependent launch (knob gather_pdl)
    o << "  asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");\n"
      << "  asm volatile(\"griddepcontrol.launch_dependents;\");\n";
  o << "  if (tid == 0) { if (g0 < n_units) issue(g0, 0); if (g0 + gs < n_units) issue(g0 + gs, 1); }\n"
    << "  int k = 0;\n"
    << "  for (long long t = g0; t < n_units; t += gs, ++k) {\n"
    << "    const int s = k & 1;\n"
    << "    const unsigned ph = (unsigned)(k >> 1) & 1u;\n"
    << "    asm volatile(\"{\\n.reg .pred p;\\nLL_GW_%=:\\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\\n@!p bra LL_GW_%=;\\n}\\n\" :: \"r\"(bar0 + 8u * s), \"r\"(ph) : \"memory\");\n"
    << "    const unsigned su = sb + " << SB << "u * s, si = su + " << UB << "u;\n"
    << "    const long long base = t << " << CU << ";\n";
  emit_unit_axis(o, P, CU, "t");
  o << "    int I[" << NVT << "][" << NE << "];\n";
  for (int j = 0; j < NVT; ++j)
    for (int q = 0; q < NE; q += (NE >= 4 ? 4 : 2)) {
      if (NE >= 4)
        o << "    asm volatile(\"ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\" : \"=r\"(I[" << j << "][" << q
          << "]), \"=r\"(I[" << j << "][" << q + 1 << "]), \"=r\"(I[" << j << "][" << q + 2 << "]), \"=r\"(I["
          << j << "][" << q + 3 << "]) : \"r\"(si + ((((unsigned)tid + " << (j << 8) << "u) << " << vb << ") + "
          << q << "u) * 4u));\n";
      else
        o << "    asm volatile(\"ld.shared.v2.u32 {%0,%1}, [%2];\" : \"=r\"(I[" << j << "][" << q
          << "]), \"=r\"(I[" << j << "][" << q + 1 << "]) : \"r\"(si + ((((unsigned)tid + " << (j << 8)
          << "u) << " << vb << ") + " << q << "u) * 4u));\n";
    }
  if (timed) {
    // registers-resident input: the thread's own vectors of the unit
    o << "    unsigned RV[" << NVT << "][4];\n";
    for (int j = 0; j < NVT; ++j)
      o << "    asm volatile(\"ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\" : \"=r\"(RV[" << j << "][0]), \"=r\"(RV["
        << j << "][1]), \"=r\"(RV[" << j << "][2]), \"=r\"(RV[" << j << "][3]) : \"r\"(su + (((unsigned)tid + "
        << (j << 8) << "u) << 4)));\n";
    o << "    __syncthreads();\n"
      << "    long long c0 = clock64(); unsigned acc = 0;\n    for (int rep = 0; rep < reps; ++rep) {\n"
      << "    unsigned z_; asm volatile(\"mov.b32 %0, 0;\" : \"=r\"(z_));\n";
    for (int j = 0; j < NVT; ++j)
      o << "    asm volatile(\"st.shared.v4.u32 [%0], {%1,%2,%3,%4};\" :: \"r\"(su + (((unsigned)tid + " << (j << 8)
        << "u) << 4)), \"r\"(RV[" << j << "][0] ^ z_), \"r\"(RV[" << j << "][1]), \"r\"(RV[" << j << "][2]), \"r\"(RV["
        << j << "][3]) : \"memory\");\n";
    o << "    __syncthreads();\n";
  }
  for (int j = 0; j < NVT; ++j) {
    o << "    { unsigned O[4] = {0, 0, 0, 0};\n";
    for (int e = 0; e < NE; ++e) {
      o << "      { int ix = I[" << j << "][" << e << "]" << (timed ? " ^ (int)z_" : "") << ";\n"
        << "        if (check && (unsigned)ix > " << mask << "u) atomicExch(err, 1);\n"
        << "        const unsigned d = (a_unit ^ a_tid ^ " << aconst(e, j) << "u ^ (unsigned)ix) & " << mask << "u;\n"
        << "        const unsigned hl = " << (uint32_t)(e | (j << (vb + 8))) << "u | ((unsigned)tid << " << vb << ");\n"
        << "        const unsigned hs = " << hstar_expr(P, "hl", "d") << ";\n";
      if (W == 8) {
        o << "        unsigned lo, hi; asm volatile(\"ld.shared.v2.u32 {%0,%1}, [%2];\" : \"=r\"(lo), \"=r\"(hi) : \"r\"(su + hs * 8u));\n"
          << "        O[" << 2 * e << "] = lo; O[" << 2 * e + 1 << "] = hi; }\n";
      } else if (W == 4) {
        o << "        unsigned v; asm volatile(\"ld.shared.u32 %0, [%1];\" : \"=r\"(v) : \"r\"(su + hs * 4u));\n"
          << "        O[" << e << "] = v; }\n";
      } else {
        const int epw = 4 / W, word = e / epw, sh = (e % epw) * 8 * W;
        o << "        unsigned v; asm volatile(\"ld.shared." << (W == 2 ? "u16" : "u8") << " %0, [%1];\" : \"=r\"(v) : \"r\"(su + hs * "
          << W << "u));\n"
          << "        O[" << word << "] |= v << " << sh << "; }\n";
      }
    }
    if (timed) o << "      acc ^= O[0] ^ O[1] ^ O[2] ^ O[3];\n      if (rep == reps - 1)\n";
    o << "      asm volatile(\"st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};\" :: \"l\"(out + (base + (((long long)tid + "
      << (j << 8) << ") << " << vb << ")) * " << W << "), \"r\"(O[0]), \"r\"(O[1]), \"r\"(O[2]), \"r\"(O[3]) : \"memory\");\n"
      << "    }\n";
  }
  if (timed)
    o << "    __syncthreads();\n    }\n    long long c1 = clock64();\n"
      << "    if (tid == 0 && cycles) cycles[blockIdx.x] = c1 - c0;\n"
      << "    if (acc == 0x9e3779b9u && reps < 0) err[1] = 1;\n";
  // every thread is done with stage s; its generic-proxy reads ordered
  // before the async-proxy refill (fence.proxy.async, as the TMA kernels)
  o << "    asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n"
    << "    __syncthreads();   // every thread is done with stage s\n"
    << "    if (tid == 0 && t + 2 * gs < n_units) issue(t + 2 * gs, s);\n"
    << "  }\n}\n";
  return o.str();
}

cudaError_t launch_gather_jit(const GatherPlanHost& P, const void* src, const int32_t* idx,
                              void* out, int* err_flag, int max_ctas, cudaStream_t st,
                              std::string* err, int reps, long long* cycles) {
  const bool shfl = P.path == LL_PATH_SHUFFLE;
  if (!shfl && P.path != LL_PATH_SMEM) return cudaErrorInvalidValue;
  const int timed = reps > 0 ? 1 : 0;
  const std::string source = shfl ? gather_shfl_source(P, timed) : gather_smem_source(P, timed);
  void* fn = nullptr;
  cudaError_t e = jit_kernel(source, shfl ? "ll_gather_shfl" : "ll_gather_smem", &fn, err);
  if (e != cudaSuccess) return e;
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int ub = shfl ? P.warp_bits : P.cta_bits;
  long long n_units = (P.batch << P.n) >> ub;
  int check = P.gp.check;
  int grid;
  unsigned smem = 0;
  if (shfl) {
    const int NV = 1 << (P.warp_bits - P.vb - 5);
    const int mu_knob = planner_knob("gather_shfl_mu", 0);
    const int MU = mu_knob > 0 ? mu_knob : std::max(1, std::min(4 / NV, 64 / (NV * (16 / P.w))));
    const long long warps = (n_units + MU - 1) / MU;
    // knob gather_shfl_waves: CTAs per SM of a grid-stride launch; < 0
    // (default): one pass, every warp MU units (config 4: 6460 vs 6084 GB/s
    // striding over 8 CTAs per SM, profiles/r02/s2l)
    const int waves = planner_knob("gather_shfl_waves", -1);
    long long g = (warps + 7) / 8;
    if (waves > 0) g = std::min<long long>(g, (long long)sms * waves);
    grid = (int)std::max<long long>(1, std::min<long long>(g, 0x7fffffff));
  } else {
    smem = 2u * ((unsigned)(P.w + 4) << P.cta_bits) + 16u;
    const int per_sm = std::max(1, std::min(8, (int)((200u * 1024u) / smem)));
    // knob gather_smem_upc: units per CTA (grid = units / upc, several
    // waves; default 1: config 4full 6464 vs 6132 GB/s for the persistent
    // grid, profiles/r02/s2l); 0: persistent, every resident CTA slot
    // striding over the units
    const int upc = planner_knob("gather_smem_upc", 1);
    const long long g = upc > 0 ? (n_units + upc - 1) / upc : std::min<long long>(n_units, (long long)sms * per_sm);
    grid = (int)std::max<long long>(1, std::min<long long>(g, 0x7fffffff));
  }
  if (timed) {
    // one CTA: 8 warp units (one per warp) for the shuffle gather, one CTA
    // unit for the shared-memory gather
    n_units = std::min<long long>(n_units, shfl ? 8 : 1);
    grid = 1;
  }
  if (max_ctas > 0) grid = std::min(grid, max_ctas);
  long long nu = n_units;
  int* ef = err_flag;
  const void* s = src;
  const int32_t* ix = idx;
  void* d = out;
  long long pf = 0;
  if (!shfl && !timed && planner_knob("gather_prefetch_waves", 1) > 0)
    pf = jit_first_wave_ctas(fn, 256, (int)smem);
  void* args_t[] = {(void*)&s, (void*)&ix, (void*)&d, (void*)&nu, (void*)&ef, (void*)&check,
                    (void*)&reps, (void*)&cycles};
  // the non-timed smem gather takes pf_ctas after check (the shuffle gather
  // reads the first six only)
  void* args_s[] = {(void*)&s, (void*)&ix, (void*)&d, (void*)&nu, (void*)&ef, (void*)&check, (void*)&pf};
  void** args = (!shfl && !timed) ? args_s : args_t;
  return jit_launch(fn, (unsigned)grid, 256, smem, st, args, err,
                    !timed && planner_knob("gather_pdl", 1) != 0);
}

}  // namespace ll
