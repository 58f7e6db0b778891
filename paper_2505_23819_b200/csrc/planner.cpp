// planner.cpp -- conversion / gather planning on the host.
//
// The conversion B^{-1} o A is executed as a pull:
// dst[h] = src[X h] with X = A^{-1} o B (reading A6).  When X is a
// permutation of index bits the tensor splits into independent tiles; the
// planner picks a coalesced load layout and a coalesced store layout for one
// tile (the "free mapping" of DESIGN.md), and the exchange between them goes
// through shared memory laid out by the paper's optimal swizzle.
#include "planner.hpp"
#include "planner_internal.hpp"

#include <algorithm>
#include <array>
#include <cstdio>
#include <map>
#include <mutex>
#include <sstream>
#include <tuple>

namespace ll {

namespace detail {

int ilog2i(int x) {
  int r = 0;
  while ((1 << (r + 1)) <= x) ++r;
  return r;
}

std::string vec_json(const std::vector<u64>& v) {
  std::ostringstream o;
  o << "[";
  for (size_t i = 0; i < v.size(); ++i) o << (i ? "," : "") << v[i];
  o << "]";
  return o.str();
}
std::string u32_json(const uint32_t* v, int n) {
  std::ostringstream o;
  o << "[";
  for (int i = 0; i < n; ++i) o << (i ? "," : "") << v[i];
  o << "]";
  return o.str();
}
std::string ivec_json(const std::vector<int>& v) {
  std::ostringstream o;
  o << "[";
  for (size_t i = 0; i < v.size(); ++i) o << (i ? "," : "") << v[i];
  o << "]";
  return o.str();
}

}  // namespace detail
using namespace detail;

// ------------------------------------------------------------ optimal swizzle
SwizzleResult optimal_swizzle(const std::vector<u64>& A_lane, const std::vector<u64>& B_lane,
                              const std::vector<u64>& V, int d, int elem_bytes) {
  SwizzleResult s;
  s.v = (int)V.size();
  const int gbytes = (1 << s.v) * elem_bytes;
  // b = log2(128 / (2^v w))
  s.b = gbytes <= 128 ? ilog2i(128 / gbytes) : 0;
  s.b = std::min(s.b, d - s.v);
  s.ell = d - s.v - s.b;
  // A_bank, B_bank: drop the last log2 max(1, 2^v w / 4) thread vectors (reading A13)
  const int drop = ilog2i(std::max(1, gbytes / 4));
  std::vector<u64> At, Bt;
  for (u64 x : A_lane) if (x) At.push_back(x);
  for (u64 x : B_lane) if (x) Bt.push_back(x);
  s.A_bank.assign(At.begin(), At.end() - std::min<int>(drop, (int)At.size()));
  s.B_bank.assign(Bt.begin(), Bt.end() - std::min<int>(drop, (int)Bt.size()));
  // E = A_bank \ B_bank, F = B_bank \ A_bank, ascending; |E| <= |F|
  for (u64 x : s.A_bank)
    if (std::find(s.B_bank.begin(), s.B_bank.end(), x) == s.B_bank.end()) s.E.push_back(x);
  for (u64 x : s.B_bank)
    if (std::find(s.A_bank.begin(), s.A_bank.end(), x) == s.A_bank.end()) s.F.push_back(x);
  std::sort(s.E.begin(), s.E.end());
  std::sort(s.F.begin(), s.F.end());
  if (s.E.size() > s.F.size()) std::swap(s.E, s.F);
  for (size_t i = 0; i < s.E.size(); ++i) s.H.push_back(s.E[i] ^ s.F[i]);
  // C: complement of span(S_vect u A_bank u B_bank)
  {
    F2Basis bs;
    for (u64 x : V) bs.add(x);
    for (u64 x : s.A_bank) bs.add(x);
    for (u64 x : s.B_bank) bs.add(x);
    for (int k = 0; k < d && bs.n < d; ++k)
      if (bs.add(u64(1) << k)) s.C.push_back(u64(1) << k);
  }
  // S_idx: ell vectors from H then C (reading A15); pad from A_bank (A16)
  std::vector<u64> hc = s.H;
  hc.insert(hc.end(), s.C.begin(), s.C.end());
  if ((int)hc.size() >= s.ell) {
    s.idx.assign(hc.begin(), hc.begin() + s.ell);
  } else {
    s.idx = hc;
    s.unavoidable = true;
    F2Basis bs;
    for (u64 x : V) bs.add(x);
    for (u64 x : s.idx) bs.add(x);
    for (u64 x : s.A_bank) {
      if ((int)s.idx.size() == s.ell) break;
      if (bs.add(x)) s.idx.push_back(x);
    }
  }
  s.vect = V;
  // S_bank completes S_vect u S_idx to a basis of F2^d
  {
    F2Basis bs;
    for (u64 x : V) bs.add(x);
    for (u64 x : s.idx) bs.add(x);
    for (int k = 0; k < d && bs.n < d; ++k)
      if (bs.add(u64(1) << k)) s.bank.push_back(u64(1) << k);
  }
  return s;
}

int lemma_wavefronts(const SwizzleResult& s, const std::vector<u64>& lanes, int elem_bytes) {
  const int gbytes = (1 << s.v) * elem_bytes;
  const int n = std::max(1, gbytes / 4);
  const int drop = ilog2i(n);
  std::vector<u64> bank(lanes.begin(), lanes.end() - std::min<int>(drop, (int)lanes.size()));
  std::vector<u64> vi = s.vect;
  vi.insert(vi.end(), s.idx.begin(), s.idx.end());
  std::vector<u64> all = vi;
  all.insert(all.end(), bank.begin(), bank.end());
  int inter = f2_rank(vi) + f2_rank(bank) - f2_rank(all);
  return n * (1 << inter);
}

// ------------------------------------------------------------- planner knobs
namespace {
std::mutex g_knob_mu;
std::map<std::string, int> g_knobs;
int g_knob_version = 0;
}  // namespace

int planner_knob(const char* name, int dflt) {
  std::lock_guard<std::mutex> lk(g_knob_mu);
  auto it = g_knobs.find(name);
  return it == g_knobs.end() ? dflt : it->second;
}
int planner_knob_version() {
  std::lock_guard<std::mutex> lk(g_knob_mu);
  return g_knob_version;
}
bool set_planner_knob(const std::string& name, int value) {
  if (name != "thread_bytes" && name != "thread_bytes_max" && name != "max_granule" &&
      name != "run_bytes" && name != "tile_order" && name != "host_chunk_mb" &&
      name != "host_slots" && name != "host_2d" && name != "tma_run_bytes" && name != "tma_thread_bytes" &&
      name != "tma_tile_bytes" && name != "tma_force_swizzle" && name != "regs_matrix" &&
      name != "regs_shuffle_max_rounds" && name != "shuffle_jit" && name != "shuffle_jit_tpg" &&
      name != "auto_shuffle" && name != "smem_jit" && name != "smem_jit_tpg" &&
      name != "upcast_jit" && name != "upcast_jit_tpg" && name != "smem_jit_minb" &&
      name != "regs_trans" && name != "smem_jit_depth" && name != "smem_jit_single" && name != "jit_force_fail" &&
      name != "pdl" && name != "run_bytes_dst" && name != "run_bytes_src" &&
      name != "auto_asym" && name != "tma_run_bytes_dst" && name != "gather_shfl_mu" &&
      name != "gather_cta_extra" && name != "gather_auto_smem" && name != "vec32" &&
      name != "smem_jit_noload" && name != "smem_jit_nostore" && name != "bcast_dedup" &&
      name != "smem_jit_noxchg" &&
      name != "auto_regperm" && name != "tma_jit" && name != "tmaj_k" && name != "tmaj_stages" &&
      name != "tmaj_cps" && name != "regs_b8" && name != "regperm_u" && name != "tmaj_fence" && name != "tmaj_late" &&
      name != "auto_small_granule_shuffle" && name != "regperm_v8" && name != "regperm_waves" && name != "tmaj_tpc" && name != "tmaj_images" && name != "tmaj_v8" &&
      name != "gather_shfl_waves" && name != "gather_smem_upc" && name != "regperm_occ" &&
      name != "ld_hint" && name != "st_hint" && name != "pdl_prefetch" && name != "gather_pdl" &&
      name != "shuffle_pdl" && name != "regperm_prefetch" &&
      name != "auto_regperm_shuffle" && name != "pdl_prefetch_short" && name != "upcast_pdl" &&
      name != "tile_xor" && name != "tile_xor_skip" && name != "host_ramp" && name != "pdl_prefetch_waves" && name != "shuffle_prefetch_waves" && name != "gather_prefetch_waves" && name != "pdl_prefetch_bulk" && name != "shuffle_prefetch_bulk")
    return false;
  std::lock_guard<std::mutex> lk(g_knob_mu);
  g_knobs[name] = value;
  ++g_knob_version;
  return true;
}

// ------------------------------------------------------------- conversion plan
namespace {

// X = A^{-1} o B as columns (one per dst index bit): the src index of each
// dst basis bit.
std::vector<u64> quotient(const Layout& A, const Layout& B) {
  auto Ainv = f2_right_inverse(A.cols, A.out_bits());
  std::vector<u64> X;
  X.reserve(B.cols.size());
  for (u64 c : B.cols) X.push_back(f2_apply(Ainv, c));
  return X;
}

void fill_generic(ConvertPlan& P, const std::vector<u64>& X) {
  GenericPlan& g = P.gp;
  g = GenericPlan{};
  const int vb = ilog2i(16 / P.w);
  g.nB = P.nB;
  g.n_x = P.nB;
  for (int k = 0; k < P.nB; ++k) g.x[k] = (int64_t)X[k];
  g.batch_stride_src = int64_t(1) << P.nA;
  g.batch_stride_dst = int64_t(1) << P.nB;
  const int64_t per = P.nB >= vb ? (int64_t(1) << (P.nB - vb)) : 1;
  g.n_vec = per * P.batch;
}


// ------------------------------------------------ word-index linear maps
// Column-reduce an invertible LB x LB matrix M (columns = images of unit
// vectors) to the identity; returns the elementary array operations E1..Em
// such that applying them in order to an array T (T'[k] = T[E k]) yields
// T'[k] = T[M k].  op 0 = swap bits (a, b); op 1 = "if bit a set, flip bit b".
bool linop_factor(std::vector<u64> M, int LB, std::vector<std::array<int, 3>>& ops) {
  std::vector<std::array<int, 3>> F;  // recorded column operations, in order
  for (int j = 0; j < LB; ++j) {
    int piv = -1;
    for (int c = j; c < LB; ++c)
      if ((M[c] >> j) & 1) { piv = c; break; }
    if (piv < 0) return false;
    if (piv != j) { std::swap(M[piv], M[j]); F.push_back({0, j, piv}); }
    for (int q = 0; q < LB; ++q)
      if (q != j && ((M[q] >> j) & 1)) { M[q] ^= M[j]; F.push_back({1, q, j}); }
  }
  ops.assign(F.rbegin(), F.rend());
  return true;
}

u64 linop_apply_index(const std::array<int, 3>& op, u64 k) {
  if (op[0] == 0) {
    u64 ba = (k >> op[1]) & 1, bb = (k >> op[2]) & 1;
    if (ba != bb) k ^= (u64(1) << op[1]) | (u64(1) << op[2]);
    return k;
  }
  if ((k >> op[1]) & 1) k ^= u64(1) << op[2];
  return k;
}

// mxfp4 upcast: scale-index contribution of destination (byte-layout) index
// bit k, for scales stored row-major [M][K/32] = [M][KB/16] -- column k of
// the scale layout S = (m, kb -> m, kb >> 4) o B (ll_mxfp4_scale_layout),
// flattened; zero for the kb bits 0-3 (one scale per 16 bytes)
int64_t scale_contrib(const ConvertPlan& P, int k) {
  const u64 c = P.dst_cols[k];
  if (!c) return 0;
  const int pos = ctz64(c);                 // flat (m, kb) bit; kb is the fastest dim
  if (pos >= P.kb_bits) return P.scale_row << (pos - P.kb_bits);   // m bit
  return pos >= 4 ? (int64_t(1) << (pos - 4)) : 0;                 // kb bit (32 fp4 = 16 bytes per scale)
}

}  // namespace

namespace detail {

// The paper's warp-shuffle exchange between two warp-local
// thread layouts given by their word-level register vectors (Aw / Bw, word
// order) and lane vectors (Al5 / Bl5): V is the word, I, E, F (ascending),
// G = {e_i ^ f_i}, R completes span(I u G); round k sends
// R[alpha(k) ^ beta(l)] to lane gamma(k) ^ delta(l), which stores it at word
// eps(k) ^ zeta(l).  ok = false if the exchange is not expressible so.
ShuffleCore shuffle_core(const std::vector<u64>& Aw, const std::vector<u64>& Al5,
                         const std::vector<u64>& Bw, const std::vector<u64>& Bl5, int LB) {
  ShuffleCore sc;
  // I, E, F (ascending), G = {e_i ^ f_i}, R completes span(I u G)
  std::vector<u64>& I = sc.I;
  std::vector<u64>& E = sc.E;
  std::vector<u64>& F = sc.F;
  std::vector<u64>& Gv = sc.Gv;
  std::vector<u64>& R = sc.R;
  for (u64 x : Al5) if (std::find(Bl5.begin(), Bl5.end(), x) != Bl5.end()) I.push_back(x);
  for (u64 x : Al5) if (std::find(I.begin(), I.end(), x) == I.end()) E.push_back(x);
  for (u64 x : Bl5) if (std::find(I.begin(), I.end(), x) == I.end()) F.push_back(x);
  std::sort(I.begin(), I.end());
  std::sort(E.begin(), E.end());
  std::sort(F.begin(), F.end());
  for (size_t i = 0; i < E.size() && i < F.size(); ++i) Gv.push_back(E[i] ^ F[i]);
  {
    F2Basis bs;
    for (u64 x : I) bs.add(x);
    for (u64 x : Gv) bs.add(x);
    std::vector<u64> units;
    for (u64 x : Aw) units.push_back(x);
    for (u64 x : Al5) units.push_back(x);
    std::sort(units.begin(), units.end());
    for (u64 x : units) if (bs.add(x)) R.push_back(x);
  }
  const int NWd = 1 << LB;
  bool ok = E.size() == F.size() && (int)R.size() == LB && NWd <= LL_MAX_GRAN;
  // decompose word-level vectors in the ld and st bases
  auto decomp = [&](u64 x, const std::vector<u64>& wv, const std::vector<u64>& lv, int& word,
                    int& lane) {
    word = 0; lane = 0;
    for (int b = 0; b < (int)wv.size(); ++b) if (x & wv[b]) word |= 1 << b;
    for (int c = 0; c < 5; ++c) if (x & lv[c]) lane |= 1 << c;
  };
  std::vector<u64> span5;
  if (ok) {
    std::vector<u64> gen = I;
    gen.insert(gen.end(), Gv.begin(), Gv.end());
    span5.push_back(0);
    for (u64 gvec : gen) {
      size_t n0 = span5.size();
      for (size_t i = 0; i < n0; ++i) span5.push_back(span5[i] ^ gvec);
    }
    ok = span5.size() == 32;
  }
  std::vector<int> ws(32 * NWd, -1), sl(32 * NWd, -1), wr(32 * NWd, -1);
  for (int k = 0; ok && k < NWd; ++k) {
    u64 Rk = 0;
    for (int j = 0; j < LB; ++j) if ((k >> j) & 1) Rk ^= R[j];
    for (u64 y : span5) {
      const u64 x = Rk ^ y;
      int aw, al, bw, bl;
      decomp(x, Aw, Al5, aw, al);
      decomp(x, Bw, Bl5, bw, bl);
      if (ws[al * NWd + k] >= 0 || wr[bl * NWd + k] >= 0) { ok = false; break; }  // one send / recv per lane
      ws[al * NWd + k] = aw;
      sl[bl * NWd + k] = al;
      wr[bl * NWd + k] = bw;
    }
  }
  std::vector<u64>& alpha = sc.alpha;
  std::vector<u64>& epsm = sc.epsm;
  alpha.assign(LB, 0);
  epsm.assign(LB, 0);
  if (ok) {
    // linear decomposition: ws(l,k) = alpha(k) ^ beta(l), etc. (checked)
    for (int l = 0; l < 32 && ok; ++l)
      for (int k = 0; k < NWd && ok; ++k) {
        ok = ws[l * NWd + k] == (ws[k] ^ ws[l * NWd]) && sl[l * NWd + k] == (sl[k] ^ sl[l * NWd]) &&
             wr[l * NWd + k] == (wr[k] ^ wr[l * NWd]);
      }
  }
  std::vector<std::array<int, 3>>& pre = sc.pre;
  std::vector<std::array<int, 3>>& post = sc.post;
  if (ok) {
    for (int j = 0; j < LB; ++j) { alpha[j] = (u64)ws[1 << j]; epsm[j] = (u64)wr[1 << j]; }
    // eps^{-1}
    std::vector<u64> einv(LB, 0);
    for (int m = 0; m < NWd; ++m) {
      int e = 0;
      for (int j = 0; j < LB; ++j) if ((m >> j) & 1) e ^= (int)epsm[j];
      for (int j = 0; j < LB; ++j) if (e == (1 << j)) einv[j] = (u64)m;
    }
    ok = linop_factor(alpha, LB, pre) && linop_factor(einv, LB, post) &&
         (int)pre.size() <= LL_MAX_LINOPS && (int)post.size() <= LL_MAX_LINOPS;
    // verify the factorisations by applying them to index arrays
    for (int pass = 0; ok && pass < 2; ++pass) {
      const auto& ops = pass ? post : pre;
      std::vector<int> T(NWd);
      for (int k = 0; k < NWd; ++k) T[k] = k;
      for (const auto& op : ops) {
        std::vector<int> T2(NWd);
        for (int k = 0; k < NWd; ++k) T2[k] = T[(int)linop_apply_index(op, (u64)k)];
        T = T2;
      }
      for (int k = 0; k < NWd && ok; ++k) {
        int want = 0;
        for (int j = 0; j < LB; ++j) if ((k >> j) & 1) want ^= (int)(pass ? einv[j] : alpha[j]);
        ok = T[k] == want;
      }
    }
  }
  if (ok) {
    for (int c = 0; c < 5; ++c) {
      sc.beta[c] = (uint32_t)ws[(1 << c) * NWd];
      sc.delta[c] = (uint32_t)sl[(1 << c) * NWd];
      sc.zeta[c] = (uint32_t)wr[(1 << c) * NWd];
      sc.beta_any |= sc.beta[c];
      sc.zeta_any |= sc.zeta[c];
    }
    for (int k = 0; k < NWd; ++k) sc.gamma.push_back((uint8_t)sl[k]);
  }
  sc.ok = ok;
  sc.rounds = NWd;
  return sc;
}

}  // namespace detail

namespace {

// Try to build the shared-memory tile plan; returns false if X is not a bit
// permutation or the tile does not fit.
bool plan_smem(ConvertPlan& P, const std::vector<u64>& X, bool swizzle, std::ostringstream& js,
               bool warp_tile = false) {
  // virtual index spaces (broadcast dedup, build_convert_plan): X is over
  // the destination bits that are not copies and the source bits that are
  // read; SP / DP give their physical buffer positions (identity otherwise)
  const bool virt = !P.dst_phys.empty();
  const int n = virt ? (int)P.dst_phys.size() : P.nB, nA = virt ? (int)P.src_phys.size() : P.nA, w = P.w;
  auto SP = [&](int p) { return virt ? P.src_phys[p] : p; };
  auto DP = [&](int k) { return virt ? P.dst_phys[k] : k; };
  if (n > 62 || nA > 62) return false;
  // sigma: dst bit -> src bit; -1 for destination broadcast bits (zero columns
  // of X: the min-weight quotient makes every copy read the same source,
  // P:607-610).  Source bits outside the image of sigma are source broadcast
  // copies that are never read.
  std::vector<int> sigma(n, -1), sinv(nA, -1), Zd;
  for (int k = 0; k < n; ++k) {
    if (X[k] == 0) { Zd.push_back(k); continue; }
    if (popcount64(X[k]) != 1) return false;
    sigma[k] = ctz64(X[k]);
    if (sinv[sigma[k]] >= 0) return false;
    sinv[sigma[k]] = k;
  }
  auto contains = [](const std::vector<int>& v, int x) {
    return std::find(v.begin(), v.end(), x) != v.end();
  };
  const int vb = ilog2i(16 / w);
  const int neff = n - (int)Zd.size();  // bits of distinct elements
  if (neff < vb + 5 || nA < vb) return false;
  std::vector<int> VD, VS, CD, CS;
  for (int k = 0; k < vb; ++k) {
    if (sigma[k] < 0 || sinv[k] < 0) return false;  // vectors must be broadcast-free
    VD.push_back(k);
    VS.push_back(sinv[k]);
  }
  int r_max = ilog2i(std::max(16, std::min(128, planner_knob("thread_bytes_max", 128))) / w);
  if (P.r_cap > 0) r_max = std::min(r_max, P.r_cap);
  const int r_pref = std::min(r_max, ilog2i(std::max(16, planner_knob("thread_bytes", 64)) / w));
  int G = 0, gbits = 0, r = 0, g = -1;
  std::vector<int> V, need, T;
  // coalescing run: run_bytes contiguous bytes on both sides (skipping broadcast
  // bits); shortened (down to 128 B) when the tile would not fit 8 warps
  int cbits = warp_tile ? 3 : std::max(0, ilog2i(std::max(16, planner_knob("run_bytes", 256)) / 16));
  // asymmetric runs: when the tile needs a group of >= 4 warps (transposes),
  // the destination run is cut to 64 B -- stores merge in L2, loads need the
  // long runs -- which halves the group (config 3: 6232 -> 6316 GB/s;
  // configs 2 / 5 keep 2- / 1-warp groups and are unchanged)
  bool asym = false;
  for (; cbits >= std::min(cbits, 3); --cbits) {
    CD.clear();
    CS.clear();
    // per-side run lengths (knobs run_bytes_dst / run_bytes_src override the
    // shared run_bytes for one side)
    const int rd_knob = planner_knob("run_bytes_dst", 0), rs_knob = planner_knob("run_bytes_src", 0);
    const int cbits_d = rd_knob > 0 && !warp_tile ? std::min(cbits, ilog2i(std::max(16, rd_knob) / 16))
                        : asym ? std::min(cbits, 2) : cbits;
    const int cbits_s = rs_knob > 0 && !warp_tile ? std::min(cbits, ilog2i(std::max(16, rs_knob) / 16)) : cbits;
    for (int k = vb; k < n && (int)CD.size() < cbits_d; ++k) if (sigma[k] >= 0) CD.push_back(k);
    for (int k = vb; k < nA && (int)CS.size() < cbits_s; ++k) if (sinv[k] >= 0) CS.push_back(sinv[k]);
    G = 0;
    // Granule choice: the largest prefix of the destination vector that the
    // load side can also hold in registers; prefer choices that keep the
    // source coalescing bits out of the registers.
    for (int pass = 0; pass < 2 && !G; ++pass) {
      for (int Gc : {16, 8, 4}) {
        if (Gc < w || Gc < 4 || Gc > planner_knob("max_granule", 16)) continue;
        int gb = ilog2i(Gc / w);
        std::vector<int> Vc(VD.begin(), VD.begin() + gb);
        std::vector<int> nd = VS;
        for (int x : Vc) if (!contains(nd, x)) nd.push_back(x);
        int rn = (int)nd.size();
        if (rn > r_max || rn + 5 > neff) continue;
        bool clash = false;
        for (int x : nd) if (contains(CS, x)) clash = true;
        if (clash && pass == 0) continue;
        G = Gc; gbits = gb; V = Vc; need = nd;
        r = std::min(std::max(rn, r_pref), std::min(r_max, neff - 5));
        break;
      }
    }
    if (!G) return false;
    // tile bits T (dst bit ids)
    T = VD;
    for (auto* s : {&VS, &CD, &CS, &need})
      for (int x : *s) if (!contains(T, x)) T.push_back(x);
    for (int k = 0; (int)T.size() < r + 5 && k < n; ++k)
      if (!contains(T, k) && sigma[k] >= 0) T.push_back(k);
    g = (int)T.size() - r - 5;
    if (g > 3) {
      int r2 = std::min(r_max, (int)T.size() - 5 - 3);
      if (r2 > r) { r = r2; g = (int)T.size() - r - 5; }
    }
    if (!asym && !warp_tile && rd_knob == 0 && g >= 2 && cbits > 2 &&
        planner_knob("auto_asym", 1)) {
      asym = true;
      ++cbits;  // the same run length again, with the shorter destination run
      continue;
    }
    if (g >= 0 && g <= 3) break;
    if (cbits <= 3) break;
  }
  if (g < 0 || g > 3) return false;
  std::sort(T.begin(), T.end());
  // ---- load layout: rho order = VS, need \ VS (src order), extra (highest src)
  std::vector<int> ld_reg = VS;
  {
    std::vector<int> rest;
    for (int x : need) if (!contains(ld_reg, x)) rest.push_back(x);
    std::sort(rest.begin(), rest.end(), [&](int a, int b) { return sigma[a] < sigma[b]; });
    ld_reg.insert(ld_reg.end(), rest.begin(), rest.end());
    std::vector<int> cand;
    for (int x : T) if (!contains(ld_reg, x) && !contains(CS, x)) cand.push_back(x);
    std::sort(cand.begin(), cand.end(), [&](int a, int b) { return sigma[a] > sigma[b]; });
    for (int x : cand) { if ((int)ld_reg.size() == r) break; ld_reg.push_back(x); }
    if ((int)ld_reg.size() != r) return false;
  }
  std::vector<int> ld_lane, ld_warp;
  {
    std::vector<int> cand;
    for (int x : T) if (!contains(ld_reg, x)) cand.push_back(x);
    std::sort(cand.begin(), cand.end(), [&](int a, int b) { return sigma[a] < sigma[b]; });
    for (int x : cand) (ld_lane.size() < 5 ? ld_lane : ld_warp).push_back(x);
  }
  // ---- store layout: rho order = VD, extra (highest dst)
  std::vector<int> st_reg = VD;
  {
    std::vector<int> cand;
    for (int x : T) if (!contains(st_reg, x) && !contains(CD, x)) cand.push_back(x);
    std::sort(cand.begin(), cand.end(), [](int a, int b) { return a > b; });
    for (int x : cand) { if ((int)st_reg.size() == r) break; st_reg.push_back(x); }
    if ((int)st_reg.size() != r) return false;
  }
  std::vector<int> st_lane(CD.begin(), CD.begin() + std::min<size_t>(5, CD.size())), st_warp;
  {
    std::vector<int> cand;
    for (int x : T) if (!contains(st_reg, x) && !contains(st_lane, x)) cand.push_back(x);
    std::sort(cand.begin(), cand.end());
    for (int x : cand) (st_lane.size() < 5 ? st_lane : st_warp).push_back(x);
  }
  if (ld_lane.size() != 5 || st_lane.size() != 5 || (int)ld_warp.size() != g ||
      (int)st_warp.size() != g)
    return false;
  // 32-byte thread vectors (knob vec32; sm_100 256-bit LDG / STG): the first
  // register bit above the 16-byte vector becomes the next buffer bit, so a
  // thread's vectors u and u ^ 1 are contiguous -- on the load side the source
  // bit vb, on the store side the destination bit vb.  The bit trades places
  // with a register bit the granule does not need; lanes and warps are
  // re-sorted (lowest buffer bits first, the coalescing order).
  if (planner_knob("vec32", 0) && r > vb) {
    auto to32 = [&](std::vector<int>& reg, std::vector<int>& lane, std::vector<int>& warp, int bit,
                    const std::vector<int>& keep, auto key) {
      if (bit < 0 || !contains(T, bit)) return false;
      auto it = std::find(reg.begin(), reg.end(), bit);
      if (it == reg.end()) {
        int x = -1;
        for (int q = (int)reg.size() - 1; q >= vb; --q)
          if (!contains(keep, reg[q])) { x = q; break; }
        if (x < 0) return false;
        std::vector<int>* side = contains(lane, bit) ? &lane : &warp;
        *std::find(side->begin(), side->end(), bit) = reg[x];
        reg.erase(reg.begin() + x);
        std::vector<int> tw = lane;
        tw.insert(tw.end(), warp.begin(), warp.end());
        std::sort(tw.begin(), tw.end(), [&](int a, int b) { return key(a) < key(b); });
        lane.assign(tw.begin(), tw.begin() + 5);
        warp.assign(tw.begin() + 5, tw.end());
      } else {
        reg.erase(it);
      }
      reg.insert(reg.begin() + vb, bit);
      return true;
    };
    std::vector<int> keep_ld = need, keep_st = VD;
    to32(ld_reg, ld_lane, ld_warp, sinv[vb], keep_ld, [&](int k) { return sigma[k]; });
    if (sigma[vb] >= 0) to32(st_reg, st_lane, st_warp, vb, keep_st, [&](int k) { return k; });
  }
  // ---- sub-word register-bit swaps on the load side (prmt): the first sw
  // positions of rho must hold V's sub-word bits; V's word-level bits are
  // then picked at compile time by the STS operand selection (gsel).
  const int nsub = w >= 4 ? 0 : ilog2i(4 / w);
  std::vector<int> order = ld_reg;
  std::vector<std::pair<int, int>> swaps;
  for (int t = 0; t < std::min(nsub, gbits); ++t) {
    int s = (int)(std::find(order.begin(), order.end(), V[t]) - order.begin());
    if (s != t) { swaps.push_back({t, s}); std::swap(order[t], order[s]); }
  }
  if ((int)swaps.size() > LL_MAX_SWAPS) return false;
  // register word bit of each rho position (w = 8: word bit 0 = element half)
  auto wordbit = [&](int rho) { return w == 8 ? rho + 1 : rho - nsub; };
  const int LB = w == 8 ? r + 1 : r - nsub;   // word-index bits
  std::vector<int> gsel;                    // word bits forming a granule
  if (w == 8) gsel.push_back(0);
  for (int t = (w == 8 ? 0 : nsub); t < gbits; ++t) {
    int pos = (int)(std::find(order.begin(), order.end(), V[t]) - order.begin());
    gsel.push_back(wordbit(pos));
  }
  if ((int)gsel.size() > 2) return false;
  std::vector<int> rest_rho;                // rho positions of the remaining word bits (ascending word bit)
  for (int wb = 0; wb < LB; ++wb) {
    if (std::find(gsel.begin(), gsel.end(), wb) != gsel.end()) continue;
    rest_rho.push_back(w == 8 ? wb - 1 : wb + nsub);
  }
  // ---- tile-local space
  const int d = (int)T.size();
  auto loc = [&](int k) -> u64 {
    return u64(1) << (std::find(T.begin(), T.end(), k) - T.begin());
  };
  std::vector<u64> Al, Bl, Vl;
  for (int x : ld_lane) Al.push_back(loc(x));
  for (int x : st_lane) Bl.push_back(loc(x));
  for (int x : V) Vl.push_back(loc(x));
  SwizzleResult sw;
  std::vector<u64> Scols;
  if (swizzle) {
    sw = optimal_swizzle(Al, Bl, Vl, d, w);
    Scols = sw.vect;
    Scols.insert(Scols.end(), sw.bank.begin(), sw.bank.end());
    Scols.insert(Scols.end(), sw.idx.begin(), sw.idx.end());
  } else {
    // unswizzled staging (ablation): offsets = store order (rho, lane, warp)
    sw.v = (int)Vl.size();
    for (int k : st_reg) Scols.push_back(loc(k));
    for (int k : st_lane) Scols.push_back(loc(k));
    for (int k : st_warp) Scols.push_back(loc(k));
    sw.vect = Vl;
    sw.bank.assign(Scols.begin() + Vl.size(), Scols.end());
  }
  auto Sinv = f2_right_inverse(Scols, d);  // square, invertible
  auto off = [&](int k) -> int32_t { return (int32_t)f2_apply(Sinv, loc(k)); };
  // ---- fill the device plan (all offsets in bytes)
  SmemPlan& sp = P.sp;
  sp = SmemPlan{};
  const int lw = ilog2i(w);
  for (int k : T)
    if (SP(sigma[k]) + lw >= 31 || DP(k) + lw >= 31) return false;  // 32-bit in-tile byte offsets
  sp.gw = g;
  sp.tile_bytes = w << d;
  if (P.padded) {
    sp.pad = 1;
    sp.tile_bytes += sp.tile_bytes / 8;
  }
  sp.n_swaps = (int)swaps.size();
  for (size_t i = 0; i < swaps.size(); ++i) {
    sp.swap_a[i] = (int8_t)swaps[i].first;
    sp.swap_b[i] = (int8_t)swaps[i].second;
  }
  sp.gsel_a = gsel.size() > 0 ? (int8_t)gsel[0] : (int8_t)-1;
  sp.gsel_b = gsel.size() > 1 ? (int8_t)gsel[1] : (int8_t)-1;
  auto boff = [&](int k) -> uint32_t { return (uint32_t)off(k) << lw; };
  for (int b = 0; b < 5; ++b) {
    sp.ld_thr[b] = uint32_t(w) << SP(sigma[ld_lane[b]]);
    sp.st_thr[b] = uint32_t(w) << DP(st_lane[b]);
    sp.sw_thr[b] = boff(ld_lane[b]);
    sp.sr_thr[b] = boff(st_lane[b]);
  }
  for (int b = 0; b < g; ++b) {
    sp.ld_thr[5 + b] = uint32_t(w) << SP(sigma[ld_warp[b]]);
    sp.st_thr[5 + b] = uint32_t(w) << DP(st_warp[b]);
    sp.sw_thr[5 + b] = boff(ld_warp[b]);
    sp.sr_thr[5 + b] = boff(st_warp[b]);
  }
  const int nvec = 1 << (r - vb);
  if (nvec > LL_MAX_VEC) return false;
  for (int u = 0; u < nvec; ++u) {
    uint32_t lo = 0, so = 0;
    for (int q = 0; q < r - vb; ++q)
      if ((u >> q) & 1) { lo += uint32_t(w) << SP(sigma[ld_reg[vb + q]]); so += uint32_t(w) << DP(st_reg[vb + q]); }
    sp.ld_vec[u] = lo;
    sp.st_vec[u] = so;
  }
  const int ngran = 1 << (r - gbits);
  if (ngran > LL_MAX_GRAN || (int)rest_rho.size() != r - gbits) return false;
  for (int j = 0; j < ngran; ++j) {
    uint32_t wo = 0, ro = 0;
    for (int q = 0; q < r - gbits; ++q)
      if ((j >> q) & 1) { wo ^= boff(order[rest_rho[q]]); ro ^= boff(st_reg[gbits + q]); }
    sp.sw_gran[j] = wo;
    sp.sr_gran[j] = ro;
  }
  if (P.op == 1) {
    // mxfp4 upcast: the scale of destination byte (m, kb) is scales[m][kb >> 4]
    sp.upcast = 1;
    for (int b = 0; b < 5; ++b) sp.sc_thr[b] = (uint32_t)scale_contrib(P, st_lane[b]);
    for (int b = 0; b < g; ++b) sp.sc_thr[5 + b] = (uint32_t)scale_contrib(P, st_warp[b]);
    for (int u = 0; u < nvec; ++u) {
      int64_t c = 0;
      for (int q = 0; q < r - vb; ++q)
        if ((u >> q) & 1) c += scale_contrib(P, st_reg[vb + q]);
      sp.sc_vec[u] = (uint32_t)c;
    }
    for (int e = 0; e < (1 << vb); ++e) {
      int64_t c = 0;
      for (int q = 0; q < vb; ++q)
        if ((e >> q) & 1) c += scale_contrib(P, st_reg[q]);
      sp.sc_e[e] = (uint32_t)c;
    }
    // the scale of byte e depends only on the vector bits with a nonzero
    // contribution: <= 2 such bits -> 4 scale loads per vector + byte select
    std::vector<int> nzq;
    for (int q = 0; q < vb; ++q)
      if (scale_contrib(P, st_reg[q])) nzq.push_back(q);
    sp.sc_nz = (int)nzq.size();
    for (size_t i = 0; i < nzq.size() && i < 2; ++i) sp.sc_c[i] = (uint32_t)scale_contrib(P, st_reg[nzq[i]]);
    // byte e + 4 (vector bit 2 set) has the slot of byte e with the slot bit
    // of vector bit 2 (if it moves the scale) flipped
    sp.sc_psel = 0x3210u;
    for (size_t i = 0; i < nzq.size() && i < 2; ++i)
      if (nzq[i] == 2) {
        sp.sc_psel = 0;
        for (int q = 0; q < 4; ++q) sp.sc_psel |= (uint32_t)(q ^ (1 << i)) << (4 * q);
      }
    for (int e = 0; e < (1 << vb); ++e) {
      int slot = 0;
      for (size_t i = 0; i < nzq.size() && i < 2; ++i) slot |= ((e >> nzq[i]) & 1) << i;
      sp.sc_slot[e] = (uint8_t)slot;
      sp.sc_sel[e] = (uint32_t)(slot | (4 + slot) << 4 | slot << 8 | (4 + slot) << 12);
    }
  }
  // ---- tile map: outer dst bits in the planner's tile order.  Order 0
  // (default): destination order, so consecutive tiles complete destination
  // runs and lines (measured best on every config); 1: source order; 2:
  // "next lowest destination bit" and "next lowest source bit" interleaved
  // (the tiles in flight form a 2-D block contiguous in both buffers).
  std::vector<int> O;
  for (int k = 0; k < n; ++k) if (!contains(T, k)) O.push_back(k);
  if ((int)O.size() > LL_MAX_OUTER) return false;
  std::vector<int> by_dst = O, by_src = O;
  std::sort(by_src.begin(), by_src.end(), [&](int a, int b) { return sigma[a] < sigma[b]; });
  const int order_knob = planner_knob("tile_order", 0);
  // destination broadcast bits first: consecutive tiles then reuse the same
  // source tile from L2 (each copy of a broadcast element is written, its
  // source is fetched from HBM once)
  std::vector<int> torder(Zd.begin(), Zd.end());
  by_dst.erase(std::remove_if(by_dst.begin(), by_dst.end(), [&](int k) { return sigma[k] < 0; }), by_dst.end());
  by_src.erase(std::remove_if(by_src.begin(), by_src.end(), [&](int k) { return sigma[k] < 0; }), by_src.end());
  if (order_knob == 0) {
    torder.insert(torder.end(), by_dst.begin(), by_dst.end());
  } else if (order_knob == 1) {
    torder.insert(torder.end(), by_src.begin(), by_src.end());
  } else if (order_knob >= 10 && order_knob < 30) {
    // sweep: the k lowest bits of one buffer's order (10 + k: destination,
    // 20 + k: source), then the other buffer's order
    const int k = order_knob % 10;
    const auto& first = order_knob < 20 ? by_dst : by_src;
    const auto& second = order_knob < 20 ? by_src : by_dst;
    for (int i = 0; i < (int)first.size() && i < k; ++i) torder.push_back(first[i]);
    for (int x : second) if (!contains(torder, x)) torder.push_back(x);
    for (int x : first) if (!contains(torder, x)) torder.push_back(x);
  } else {
    size_t i = 0, j = 0;
    while (torder.size() < O.size()) {
      while (i < by_dst.size() && contains(torder, by_dst[i])) ++i;
      if (i < by_dst.size()) torder.push_back(by_dst[i]);
      while (j < by_src.size() && contains(torder, by_src[j])) ++j;
      if (j < by_src.size() && torder.size() < O.size()) torder.push_back(by_src[j]);
    }
  }
  TileMap& tm = sp.tile;
  tm.n_bits = (int)torder.size();
  tm.n_tab = (tm.n_bits + LL_TAB_BITS - 1) / LL_TAB_BITS;
  for (int k = 0; k < tm.n_tab; ++k) {
    for (int v = 0; v < (1 << LL_TAB_BITS); ++v) {
      int64_t so = 0, dof = 0, sc = 0;
      for (int q = 0; q < LL_TAB_BITS; ++q) {
        const int bit = k * LL_TAB_BITS + q;
        if (((v >> q) & 1) && bit < tm.n_bits) {
          if (sigma[torder[bit]] >= 0) so += int64_t(w) << SP(sigma[torder[bit]]);
          dof += int64_t(w) << DP(torder[bit]);
          if (P.op == 1) sc += scale_contrib(P, torder[bit]);
        }
      }
      tm.tab[k][v].src = so;
      tm.tab[k][v].dst = dof;
      tm.tab[k][v].sc = sc;
    }
  }
  tm.batch_stride_src = int64_t(w) << P.nA;
  tm.batch_stride_dst = int64_t(w) << P.nB;
  tm.n_tiles = (int64_t(1) << O.size()) * P.batch;
  P.tile_bit_src.clear();
  P.tile_bit_dst.clear();
  for (int q = 0; q < tm.n_bits; ++q) {
    P.tile_bit_src.push_back(sigma[torder[q]] >= 0 ? SP(sigma[torder[q]]) : -1);
    P.tile_bit_dst.push_back(DP(torder[q]));
  }
  P.nv = nvec;
  P.g = G;
  P.tile_bits = d;
  P.r = r;
  P.gw = g;
  std::vector<u64> Bw;
  for (int k : st_lane) Bw.push_back(loc(k));
  P.pred_wf_ld = lemma_wavefronts(sw, Al, w);
  P.pred_wf_st = lemma_wavefronts(sw, Bw, w);
  if (!swizzle) { P.pred_wf_ld = -1; P.pred_wf_st = -1; }
  // ---- warp-shuffle exchange, warp tiles only (g == 0), word payload
  P.shuffle_ok = false;
  std::ostringstream sjs;
  if (g == 0 && w <= 4 && swizzle && !virt) {
    // word-level coordinates: tile-local unit vectors of the word bits / lanes
    std::vector<u64> Aw, Al5, Bw, Bl5;
    for (int b = 0; b < LB; ++b) Aw.push_back(loc(order[b + nsub]));
    for (int b = 0; b < LB; ++b) Bw.push_back(loc(st_reg[b + nsub]));
    for (int c = 0; c < 5; ++c) { Al5.push_back(loc(ld_lane[c])); Bl5.push_back(loc(st_lane[c])); }
    ShuffleCore sc = shuffle_core(Aw, Al5, Bw, Bl5, LB);
    const bool ok = sc.ok;
    const int NWd = sc.rounds;
    const auto& I = sc.I; const auto& E = sc.E; const auto& F = sc.F; const auto& Gv = sc.Gv;
    const auto& R = sc.R; const auto& alpha = sc.alpha; const auto& epsm = sc.epsm;
    const auto& pre = sc.pre; const auto& post = sc.post;
    ShufflePlan& sh = P.shp;
    sh = ShufflePlan{};
    if (ok) {
      sh.tile = sp.tile;
      sh.n_swaps = sp.n_swaps;
      for (int i = 0; i < LL_MAX_SWAPS; ++i) { sh.swap_a[i] = sp.swap_a[i]; sh.swap_b[i] = sp.swap_b[i]; }
      for (int c = 0; c < 5; ++c) {
        sh.ld_thr[c] = sp.ld_thr[c];
        sh.st_thr[c] = sp.st_thr[c];
        sh.beta_lane[c] = sc.beta[c];
        sh.delta_lane[c] = sc.delta[c];
        sh.zeta_lane[c] = sc.zeta[c];
      }
      sh.beta_any = sc.beta_any;
      sh.zeta_any = sc.zeta_any;
      for (int u = 0; u < LL_MAX_VEC; ++u) { sh.ld_vec[u] = sp.ld_vec[u]; sh.st_vec[u] = sp.st_vec[u]; }
      sh.n_pre = (int)pre.size();
      sh.n_post = (int)post.size();
      for (size_t i = 0; i < pre.size(); ++i) {
        sh.pre_op[i] = (int8_t)pre[i][0]; sh.pre_a[i] = (int8_t)pre[i][1]; sh.pre_b[i] = (int8_t)pre[i][2];
      }
      for (size_t i = 0; i < post.size(); ++i) {
        sh.post_op[i] = (int8_t)post[i][0]; sh.post_a[i] = (int8_t)post[i][1]; sh.post_b[i] = (int8_t)post[i][2];
      }
      for (int k = 0; k < NWd; ++k) sh.gamma[k] = sc.gamma[k];
      P.shd = ShuffleDir{};
      for (int k = 0; k < NWd; ++k) {
        int a = 0, e = 0;
        for (int j = 0; j < LB; ++j)
          if ((k >> j) & 1) { a ^= (int)alpha[j]; e ^= (int)epsm[j]; }
        P.shd.alpha.push_back(a);
        P.shd.eps.push_back(e);
        P.shd.gamma.push_back(sc.gamma[k]);
      }
      for (int c = 0; c < 5; ++c) { P.shd.beta[c] = sc.beta[c]; P.shd.zeta[c] = sc.zeta[c]; P.shd.delta[c] = sc.delta[c]; }
      P.shd.beta_any = sc.beta_any;
      P.shd.zeta_any = sc.zeta_any;
      P.shuffle_ok = true;
      P.shuffle_rounds = NWd;
    }
    auto ops_json = [](const std::vector<std::array<int, 3>>& ops) {
      std::ostringstream o;
      o << "[";
      for (size_t i = 0; i < ops.size(); ++i)
        o << (i ? "," : "") << "[" << ops[i][0] << "," << ops[i][1] << "," << ops[i][2] << "]";
      o << "]";
      return o.str();
    };
    sjs << ",\"shuffle\":{\"ok\":" << (ok ? "true" : "false") << ",\"I\":" << vec_json(I)
        << ",\"E\":" << vec_json(E) << ",\"F\":" << vec_json(F) << ",\"G\":" << vec_json(Gv)
        << ",\"R\":" << vec_json(R) << ",\"rounds\":" << NWd << ",\"word_bits_ld\":" << vec_json(Aw)
        << ",\"word_bits_st\":" << vec_json(Bw) << ",\"lanes_ld\":" << vec_json(Al5)
        << ",\"lanes_st\":" << vec_json(Bl5);
    if (ok) {
      sjs << ",\"alpha\":" << vec_json(alpha) << ",\"eps\":" << vec_json(epsm)
          << ",\"pre_ops\":" << ops_json(pre) << ",\"post_ops\":" << ops_json(post)
          << ",\"beta_lane\":" << u32_json(sh.beta_lane, 5) << ",\"zeta_lane\":" << u32_json(sh.zeta_lane, 5)
          << ",\"delta_lane\":" << u32_json(sh.delta_lane, 5) << ",\"gamma\":[";
      for (int k = 0; k < NWd; ++k) sjs << (k ? "," : "") << (int)sh.gamma[k];
      sjs << "]";
    }
    sjs << "}";
  }
  // ---- description
  auto srcpos = [&](const std::vector<int>& v) {
    std::vector<int> o;
    for (int x : v) o.push_back(sigma[x]);
    return o;
  };
  js << ",\"tile_dst_bits\":" << ivec_json(T) << ",\"gsel\":" << ivec_json(gsel) << ",\"r\":" << r << ",\"group_warps_log2\":" << g
     << ",\"granule_bytes\":" << G << ",\"granule_dst_bits\":" << ivec_json(V)
     << ",\"vectors_per_thread\":" << nvec << ",\"swaps\":[";
  for (size_t i = 0; i < swaps.size(); ++i)
    js << (i ? "," : "") << "[" << swaps[i].first << "," << swaps[i].second << "]";
  js << "],\"ld_reg_dst\":" << ivec_json(ld_reg) << ",\"ld_reg_src\":" << ivec_json(srcpos(ld_reg))
     << ",\"ld_lane_dst\":" << ivec_json(ld_lane) << ",\"ld_lane_src\":" << ivec_json(srcpos(ld_lane))
     << ",\"ld_warp_dst\":" << ivec_json(ld_warp) << ",\"ld_rho_after_swaps\":" << ivec_json(order)
     << ",\"st_reg\":" << ivec_json(st_reg) << ",\"st_lane\":" << ivec_json(st_lane)
     << ",\"st_warp\":" << ivec_json(st_warp) << ",\"swizzled\":" << (swizzle ? "true" : "false")
     << ",\"S_vect\":" << vec_json(sw.vect) << ",\"S_bank\":" << vec_json(sw.bank)
     << ",\"S_idx\":" << vec_json(sw.idx) << ",\"H\":" << vec_json(sw.H)
     << ",\"C\":" << vec_json(sw.C) << ",\"E\":" << vec_json(sw.E) << ",\"F\":" << vec_json(sw.F)
     << ",\"unavoidable\":" << (sw.unavoidable ? "true" : "false")
     << ",\"pred_wavefronts_per_sts\":" << P.pred_wf_ld
     << ",\"pred_wavefronts_per_lds\":" << P.pred_wf_st << ",\"n_tiles\":" << tm.n_tiles
     << ",\"smem_bytes\":{\"sw_thr\":" << u32_json(sp.sw_thr, 5 + g) << ",\"sr_thr\":"
     << u32_json(sp.sr_thr, 5 + g) << ",\"sw_gran\":" << u32_json(sp.sw_gran, ngran)
     << ",\"sr_gran\":" << u32_json(sp.sr_gran, ngran) << "}"
     << ",\"tile_order_dst_bits\":" << ivec_json(torder) << sjs.str();
  return true;
}

std::shared_ptr<ConvertPlan> build_convert_plan(const Layout& A, const Layout& B, int w,
                                                int path_req, int64_t batch, int op) {
  if (!A.same_tensor(B)) throw Error(LL_ERR_SHAPE, "convert: source and destination layouts map to different tensors");
  if (!A.surjective()) throw Error(LL_ERR_NOT_SURJECTIVE, "convert: the source layout is not surjective");
  auto P = std::make_shared<ConvertPlan>();
  P->op = op;
  if (op == 1) {
    if (w != 1 || B.out.size() != 2 || B.out[1].bits < 4)
      throw Error(LL_ERR_ARG, "mxfp4 upcast: byte layouts over (m, kb) with >= 16 bytes per row");
    if (path_req != LL_PATH_AUTO && path_req != LL_PATH_SMEM)
      throw Error(LL_ERR_UNSUPPORTED, "mxfp4 upcast: only the smem path");
    P->kb_bits = B.out[1].bits;
    P->scale_row = int64_t(1) << (B.out[1].bits - 4);
    P->dst_cols = B.cols;
    path_req = LL_PATH_SMEM;
  }
  P->w = w;
  P->nA = A.in_bits();
  P->nB = B.in_bits();
  P->batch = batch;
  auto X = quotient(A, B);
  bool ident = P->nA == P->nB;
  for (int k = 0; ident && k < P->nB; ++k) ident = X[k] == (u64(1) << k);
  P->identity = ident;
  std::ostringstream js;
  js << "{\"nA\":" << P->nA << ",\"nB\":" << P->nB << ",\"elem_bytes\":" << w
     << ",\"batch\":" << batch << ",\"X\":" << vec_json(X) << ",\"identity\":"
     << (ident ? "true" : "false");
  int path = path_req;
  bool planned = false;
  // register permutation: X is the identity above the low q
  // bits and permutes them among themselves -> each thread permutes its own
  // chunk, no exchange.  Chunk = max(q, 16-byte vector) <= 64 bytes.
  if (!ident && op == 0 && (path == LL_PATH_AUTO || path == LL_PATH_REGPERM) && P->nA == P->nB &&
      planner_knob("auto_regperm", 1) | (path == LL_PATH_REGPERM)) {
    int q = P->nB;
    while (q > 0 && X[q - 1] == (u64(1) << (q - 1))) --q;
    const int vb = ilog2i(16 / w);
    const int cb = std::max(q, vb);
    bool ok = (int64_t(w) << cb) <= 64 && cb <= P->nB;
    for (int k = 0; ok && k < q; ++k) ok = popcount64(X[k]) == 1 && X[k] < (u64(1) << q);
    // AUTO (knob auto_regperm = 1): the register permutation unless the smem
    // plan exchanges granules of >= 8 bytes -- measured on register-only
    // pairs (profiles/r02/s2f classify, s2q): smem ahead by 0.7-2.6 % there
    // (6464-6915 vs 6323-6819 GB/s), the register permutation ahead by 15-19 %
    // where the smem plan falls back to 4-byte granules; 2 = always
    // With PDL on the compiled shuffle kernel (session 3) the warp-shuffle
    // exchange ties or beats the register permutation wherever it applies
    // (w <= 4: 6671 vs 6371 GB/s for 1-byte elements with 6 register bits,
    // 6685-6847 vs 6684-6845 otherwise, profiles/r02/s3i/classify_rows.jsonl),
    // so AUTO leaves those pairs to the small-granule shuffle rule below
    // (knob auto_regperm_shuffle = 0: keep the register permutation)
    if (ok && path == LL_PATH_AUTO && planner_knob("auto_regperm", 1) == 1) {
      auto trial = std::make_shared<ConvertPlan>(*P);
      std::ostringstream js2;
      if (plan_smem(*trial, X, true, js2) && trial->g >= 8) ok = false;
      if (ok && w <= 4 && planner_knob("auto_regperm_shuffle", 1) && planner_knob("shuffle_jit", 1) &&
          planner_knob("auto_small_granule_shuffle", 1)) {
        auto strial = std::make_shared<ConvertPlan>(*P);
        std::ostringstream js3;
        if (plan_smem(*strial, X, true, js3, true) && strial->shuffle_ok && strial->g <= 4) ok = false;
      }
    }
    if (ok) {
      P->rp_bits = cb;
      for (int e = 0; e < (1 << cb); ++e) {
        u64 x = 0;
        for (int k = 0; k < cb; ++k) if ((e >> k) & 1) x ^= X[k];
        P->rp_src.push_back((int)x);
      }
      js << ",\"regperm\":{\"chunk_bits\":" << cb << ",\"chunk_bytes\":" << (w << cb) << "}";
      path = LL_PATH_REGPERM;
      planned = true;
    } else if (path == LL_PATH_REGPERM) {
      throw Error(LL_ERR_UNSUPPORTED, "regperm path requested but the quotient moves data between "
                                      "chunks of <= 64 bytes (an exchange is needed)");
    }
  }
  if (path == LL_PATH_AUTO) {
    path = ident ? LL_PATH_COPY : LL_PATH_SMEM;
    // cost model (measured on B200, profiles/r01/shuffle_jit, smem_jit): with
    // both exchanges compiled for the plan, the swizzled shared-memory path
    // (config 2 6703 GB/s, config 5 6993) edges out the paper's warp shuffles
    // (6601 / 6900), so AUTO takes shared memory; auto_shuffle=1 prefers
    // shuffles whenever the planner's warp tile makes the exchange warp-local
    if (!ident && op == 0 && w <= 4 && planner_knob("auto_shuffle", 0) && planner_knob("shuffle_jit", 1)) {
      auto trial = std::make_shared<ConvertPlan>(*P);
      std::ostringstream js2;
      if (plan_smem(*trial, X, true, js2, true) && trial->shuffle_ok) {
        *P = *trial;
        js << js2.str();
        path = LL_PATH_SHUFFLE;
        planned = true;
      }
    }
  }
  // broadcast dedup (SMEM / AUTO): zero columns of X (destination copies) and
  // source bits X never reads are removed from the index spaces the tile plan
  // works in, so each distinct element crosses shared memory once; copies
  // are made in registers (inside a 16-byte vector) or by extra stores
  // (above it), unread source copies are dropped in registers after the load
  if (!ident && op == 0 && (path == LL_PATH_AUTO || path == LL_PATH_SMEM) &&
      planner_knob("bcast_dedup", 1)) {
    const int vb = ilog2i(16 / w);
    std::vector<int> srcbit(P->nB, -1);
    std::vector<char> read(P->nA, 0);
    bool perm = true;
    for (int k = 0; k < P->nB && perm; ++k) {
      if (!X[k]) continue;
      perm = popcount64(X[k]) == 1;
      if (perm) { srcbit[k] = ctz64(X[k]); perm = !read[srcbit[k]]; read[srcbit[k]] = 1; }
    }
    int zd = 0, zs = 0;
    for (int k = 0; k < P->nB; ++k) zd += srcbit[k] < 0;
    for (int p = 0; p < P->nA; ++p) zs += !read[p];
    if (perm && (zd || zs)) {
      auto trial = std::make_shared<ConvertPlan>(*P);
      std::vector<int> svirt(P->nA, -1);
      for (int p = 0; p < P->nA; ++p)
        if (read[p]) { svirt[p] = (int)trial->src_phys.size(); trial->src_phys.push_back(p); }
      std::vector<u64> Xv;
      for (int k = 0; k < P->nB; ++k)
        if (srcbit[k] >= 0) { trial->dst_phys.push_back(k); Xv.push_back(u64(1) << svirt[srcbit[k]]); }
      const int nv = (int)Xv.size();
      bool ok = nv >= vb + 5;
      if (ok) {
        trial->ld_span = std::max(0, trial->src_phys[vb - 1] + 1 - vb);
        trial->st_span = std::max(0, trial->dst_phys[vb - 1] + 1 - vb);
        std::vector<int> high;   // destination copy bits above the virtual vector's range
        for (int k = trial->dst_phys[vb - 1] + 1; k < P->nB; ++k) if (srcbit[k] < 0) high.push_back(k);
        // loads: only the physical vectors holding virtual elements (chunks
        // of copies are skipped); stores: every physical vector of the range
        int ld_chunks = 0;
        {
          std::vector<char> ref(size_t(1) << trial->ld_span, 0);
          for (int e = 0; e < (1 << vb); ++e) {
            int ph = 0;
            for (int b = 0; b < vb; ++b) if ((e >> b) & 1) ph |= 1 << trial->src_phys[b];
            ref[ph >> vb] = 1;
          }
          for (char r : ref) ld_chunks += r;
        }
        trial->ld_chunks = ld_chunks;
        ok = trial->ld_span <= 6 && trial->st_span <= 6 && high.size() <= 4 && ld_chunks <= 16;
        for (int j = 0; ok && j < (1 << high.size()); ++j) {
          int64_t off = 0;
          for (size_t q = 0; q < high.size(); ++q) if ((j >> q) & 1) off += int64_t(w) << high[q];
          ok = off < (int64_t(1) << 31);
          trial->copy_off.push_back((uint32_t)off);
        }
      }
      std::ostringstream js2;
      // sparse sources (many copy bits inside the vectors) take fewer vectors
      // per thread: at most 16 physical 16-byte loads per thread and tile
      bool fit = false;
      for (int rc = 0; ok && !fit && rc >= 0; ) {
        trial->r_cap = rc;
        js2.str("");
        fit = plan_smem(*trial, Xv, true, js2) && trial->nv * trial->ld_chunks <= 16 &&
              (trial->nv << trial->st_span) * (int)std::max<size_t>(1, trial->copy_off.size()) <= 256;
        if (!fit) rc = rc == 0 ? trial->r - 1 : rc - 1;
        if (rc > 0 && rc < vb) rc = -1;
      }
      // AUTO keeps the dedup plan where it measured as fast as the alternatives
      // (profiles/r02/bcast_smem_counts.json: copies above or inside short
      // vector spans, enough tiles for every SM); sparse sliced layouts (long
      // spans, few tiles) ran 2-10x slower than the element-wise kernel
      if (ok && fit && path_req == LL_PATH_AUTO &&
          (trial->ld_span > 2 || trial->st_span > 2 || trial->sp.tile.n_tiles < 148))
        fit = false;
      if (ok && fit) {
        trial->jit_only = true;
        *P = *trial;
        fill_generic(*P, X);    // fallback when the plan cannot be compiled
        js << js2.str() << ",\"bcast_dedup\":{\"src_phys\":" << ivec_json(P->src_phys)
           << ",\"dst_phys\":" << ivec_json(P->dst_phys) << ",\"ld_span\":" << P->ld_span
           << ",\"st_span\":" << P->st_span << ",\"copies\":" << P->copy_off.size() << "}";
        path = LL_PATH_SMEM;
        planned = true;
      }
    }
  }
  if (path == LL_PATH_COPY && !ident)
    throw Error(LL_ERR_UNSUPPORTED, "copy path requested but the quotient is not the identity");
  if (path == LL_PATH_SMEM_PADDED) P->padded = true;
  if (!planned && (path == LL_PATH_SMEM || path == LL_PATH_SMEM_NOSWIZZLE ||
                   path == LL_PATH_SHUFFLE || path == LL_PATH_SMEM_PADDED)) {
    std::ostringstream js2;
    if (plan_smem(*P, X, path == LL_PATH_SMEM || path == LL_PATH_SHUFFLE, js2,
                  path == LL_PATH_SHUFFLE)) {
      // AUTO with a small shared-memory granule (<= 4 bytes: NV * 16 / G
      // STS + LDS per thread and tile) takes the warp-shuffle exchange when
      // the pair is warp-local on the planner's warp tile (config 6, the
      // pre-shuffle: smem 5293 vs shuffles 6470 GB/s, profiles/r02/s2b;
      // 16-byte granules keep smem: configs 2 / 5, 6700 / 6986 vs 6595 / 6900)
      if (path_req == LL_PATH_AUTO && path == LL_PATH_SMEM && P->g <= 4 && op == 0 && w <= 4 &&
          planner_knob("shuffle_jit", 1) && planner_knob("auto_small_granule_shuffle", 1)) {
        auto trial = std::make_shared<ConvertPlan>(*P);
        std::ostringstream js3;
        if (plan_smem(*trial, X, true, js3, true) && trial->shuffle_ok) {
          *P = *trial;
          js2.str(js3.str());
          path = LL_PATH_SHUFFLE;
        }
      }
      js << js2.str();
      if (path == LL_PATH_SHUFFLE && !P->shuffle_ok)
        throw Error(LL_ERR_UNSUPPORTED,
                    "shuffle path requested but the exchange is not warp-local with a word payload "
                    "((B^-1 o A)_warp must be the identity on the planner's warp tile, P:624)");
    } else {
      if (path_req != LL_PATH_AUTO)
        throw Error(LL_ERR_UNSUPPORTED, "smem/shuffle path requested but the quotient is not a tileable bit permutation");
      path = LL_PATH_GENERIC;
    }
  }
  if (path == LL_PATH_SMEM_ASYNC) {
    std::ostringstream js2;
    if (plan_async(*P, X, js2)) {
      js << js2.str();
    } else {
      throw Error(LL_ERR_UNSUPPORTED, "smem_async path requested but the quotient is not a tileable bit permutation");
    }
  }
  if (path == LL_PATH_SMEM_TMA) {
    std::ostringstream js2;
    if (plan_tma(*P, X, js2)) {
      js << js2.str();
    } else {
      throw Error(LL_ERR_UNSUPPORTED, "smem_tma path requested but the quotient is not a tileable "
                                      "bit permutation or the source tile needs more than 5 TMA box dims");
    }
  }
  if (path == LL_PATH_SMEM_TMA_STORE) {
    std::ostringstream js2;
    if (plan_tma_store(*P, X, js2)) {
      js << js2.str();
    } else {
      throw Error(LL_ERR_UNSUPPORTED, "smem_tma_store path requested but the quotient is not a tileable "
                                      "bit permutation or a tile needs more than 5 TMA box dims");
    }
  }
  if (path == LL_PATH_REGS_SHUFFLE) {
    std::ostringstream js2;
    if (plan_regs_shuffle(*P, A, B, X, js2)) {
      js << js2.str();
    } else {
      throw Error(LL_ERR_UNSUPPORTED,
                  "regs_shuffle path requested but the pair is not a warp-local register-faithful "
                  "exchange ((B^-1 o A)_warp must be the identity, P:624)");
    }
  }
  if (path == LL_PATH_REGS) {
    // cost model (measured in-kernel on B200,
    // profiles/r01/regs2): the paper's shuffle exchange beats the
    // shared-memory round trip up to 4 rounds (26-30 vs 30-46 cycles) and
    // loses from 8 rounds on (16 rounds: 166 vs 47; 64: 1100 vs 559); a
    // warp-local pair with identical lanes is a register permutation
    const int max_rounds = planner_knob("regs_shuffle_max_rounds", 4);
    if (max_rounds > 0) {
      std::ostringstream js2;
      if (plan_regs_shuffle(*P, A, B, X, js2) && P->shuffle_rounds <= max_rounds) {
        js << js2.str();
        path = LL_PATH_REGS_SHUFFLE;
      }
    }
  }
  if (path == LL_PATH_REGS) {
    std::ostringstream js2;
    if (plan_regs(*P, A, B, X, js2)) {
      js << js2.str();
    } else {
      throw Error(LL_ERR_UNSUPPORTED,
                  "regs path requested but the layouts are not register-faithful compatible "
                  "(reg/lane/warp/block dims with 5 lane and <= 3 warp bits on both sides, "
                  "identical block columns, elements of <= 4 bytes)");
    }
  }
  if (op == 1 && path != LL_PATH_SMEM)
    throw Error(LL_ERR_UNSUPPORTED, "mxfp4 upcast: the layouts are not a tileable bit permutation");
  if (path == LL_PATH_GENERIC || path == LL_PATH_REGPERM) fill_generic(*P, X);
  P->path = path;
  static const char* names[] = {"auto", "copy", "smem", "shuffle", "generic", "smem_noswizzle",
                                "smem_async", "smem_padded", "smem_tma", "regs", "smem_tma_store",
                                "regs_shuffle", "regperm"};
  js << ",\"path\":\"" << names[path] << "\"}";
  P->json = js.str();
  return P;
}

// Exact cache key: the full layouts (dims and columns), not a hash of them,
// so two different layouts can never share a plan.
void append_sig(std::vector<u64>& s, const Layout& L) {
  auto dims = [&](const std::vector<Dim>& ds) {
    s.push_back(0x5eedull << 32 | ds.size());
    for (auto& d : ds) {
      s.push_back(((u64)d.bits << 32) | d.name.size());
      for (char ch : d.name) s.push_back((unsigned char)ch);
    }
  };
  dims(L.in);
  dims(L.out);
  s.insert(s.end(), L.cols.begin(), L.cols.end());
}

struct Key {
  std::vector<u64> sig;
  int w, path;
  int64_t batch;
  int knobs;
  bool operator<(const Key& o) const {
    return std::tie(w, path, batch, knobs, sig) < std::tie(o.w, o.path, o.batch, o.knobs, o.sig);
  }
};

Key make_key(const Layout& A, const Layout* B, u64 extra, int w, int path, int64_t batch) {
  Key k{{}, w, path, batch, planner_knob_version()};
  k.sig.reserve(160);
  append_sig(k.sig, A);
  if (B) append_sig(k.sig, *B);
  k.sig.push_back(extra);
  return k;
}
constexpr size_t kMaxCached = 4096;

std::mutex g_mu;
std::map<Key, std::shared_ptr<const ConvertPlan>> g_cache;
std::map<Key, std::shared_ptr<const GatherPlanHost>> g_gcache;

}  // namespace

std::shared_ptr<const ConvertPlan> get_convert_plan(const Layout& A, const Layout& B, int w,
                                                    int path_req, int64_t batch, int op) {
  Key k = make_key(A, &B, 0, w, path_req + 1000 * op, batch);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_cache.find(k);
    if (it != g_cache.end()) return it->second;
  }
  auto P = build_convert_plan(A, B, w, path_req, batch, op);
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_cache.size() >= kMaxCached) g_cache.clear();
  g_cache[k] = P;
  return P;
}

TileRange shard_range(const ConvertPlan& P, int n_shards, int shard) {
  if (n_shards < 1 || (n_shards & (n_shards - 1)) || shard < 0 || shard >= n_shards)
    throw Error(LL_ERR_ARG, "shard: n_shards must be a power of two and 0 <= shard < n_shards");
  int sb = 0;
  while ((1 << sb) < n_shards) ++sb;
  const int64_t w = P.w;
  TileRange rg{};
  if (P.batch != 1) throw Error(LL_ERR_UNSUPPORTED, "shard: batch must be 1 (shard the layout's own block bits)");
  if (P.path == LL_PATH_COPY) {
    rg.t0 = (int64_t)shard;
    rg.t1 = (int64_t)shard + 1;
    rg.src_shift = (int64_t)shard * ((w << P.nA) >> sb);
    rg.dst_shift = (int64_t)shard * ((w << P.nB) >> sb);
    return rg;
  }
  if (P.path == LL_PATH_REGPERM) {
    // chunks are contiguous in both buffers: shard = a contiguous chunk range
    const int64_t chunks = (int64_t(1) << P.nB) >> P.rp_bits;
    if ((int64_t)n_shards > chunks) throw Error(LL_ERR_UNSUPPORTED, "shard: more shards than chunks");
    rg.t0 = chunks / n_shards * shard;
    rg.t1 = chunks / n_shards * (shard + 1);
    rg.src_shift = (int64_t)shard * ((w << P.nA) >> sb);
    rg.dst_shift = (int64_t)shard * ((w << P.nB) >> sb);
    return rg;
  }
  if (P.path != LL_PATH_SMEM && P.path != LL_PATH_SHUFFLE && P.path != LL_PATH_SMEM_NOSWIZZLE &&
      P.path != LL_PATH_SMEM_ASYNC && P.path != LL_PATH_SMEM_PADDED && P.path != LL_PATH_SMEM_TMA &&
      P.path != LL_PATH_SMEM_TMA_STORE)
    throw Error(LL_ERR_UNSUPPORTED, "shard: only tiled (smem / shuffle) plans are shardable");
  const int nb = (int)P.tile_bit_src.size();
  if (sb > nb) throw Error(LL_ERR_UNSUPPORTED, "shard: more shards than tiles");
  for (int j = 0; j < sb; ++j) {
    const int q = nb - sb + j;
    if (P.tile_bit_src[q] != P.nA - sb + j || P.tile_bit_dst[q] != P.nB - sb + j)
      throw Error(LL_ERR_UNSUPPORTED,
                  "shard: the top index bits are not block bits shared by both layouts "
                  "(a rank's shard would not be a contiguous slice of both buffers)");
  }
  const int64_t per = (int64_t(1) << nb) >> sb;
  rg.t0 = per * shard;
  rg.t1 = per * (shard + 1);
  rg.src_shift = (int64_t)shard * ((w << P.nA) >> sb);
  rg.dst_shift = (int64_t)shard * ((w << P.nB) >> sb);
  return rg;
}

TileRange shard_range_2d(const ConvertPlan& P, int n_shards, int shard, int* side, int* r0) {
  if (n_shards < 2 || (n_shards & (n_shards - 1)) || shard < 0 || shard >= n_shards)
    throw Error(LL_ERR_ARG, "shard_2d: n_shards must be a power of two >= 2 and 0 <= shard < n_shards");
  int sb = 0;
  while ((1 << sb) < n_shards) ++sb;
  if (P.batch != 1) throw Error(LL_ERR_UNSUPPORTED, "shard_2d: batch must be 1");
  if (P.path != LL_PATH_SMEM && P.path != LL_PATH_SHUFFLE && P.path != LL_PATH_SMEM_NOSWIZZLE &&
      P.path != LL_PATH_SMEM_ASYNC && P.path != LL_PATH_SMEM_PADDED && P.path != LL_PATH_SMEM_TMA &&
      P.path != LL_PATH_SMEM_TMA_STORE)
    throw Error(LL_ERR_UNSUPPORTED, "shard_2d: only tiled (smem / shuffle) plans are shardable");
  const int nb = (int)P.tile_bit_src.size();
  if (sb > nb) throw Error(LL_ERR_UNSUPPORTED, "shard_2d: more shards than tiles");
  const int64_t w = P.w;
  for (int s = 0; s < 2; ++s) {
    const std::vector<int>& top = s == 0 ? P.tile_bit_src : P.tile_bit_dst;
    const std::vector<int>& oth = s == 0 ? P.tile_bit_dst : P.tile_bit_src;
    const int ntop = s == 0 ? P.nA : P.nB;
    const int base = oth[nb - sb];
    bool ok = true;
    for (int j = 0; j < sb && ok; ++j)
      ok = top[nb - sb + j] == ntop - sb + j && oth[nb - sb + j] == base + j;
    if (!ok) continue;
    *side = s;
    *r0 = base;
    TileRange rg{};
    const int64_t per = (int64_t(1) << nb) >> sb;
    rg.t0 = per * shard;
    rg.t1 = per * (shard + 1);
    const int64_t slice = (int64_t)shard * ((w << ntop) >> sb);
    rg.src_shift = s == 0 ? slice : 0;
    rg.dst_shift = s == 0 ? 0 : slice;
    return rg;
  }
  throw Error(LL_ERR_UNSUPPORTED,
              "shard_2d: the top tile bits are not the top bits of one side and a contiguous run "
              "of the other's");
}

// ------------------------------------------------------------------ gather
std::shared_ptr<const GatherPlanHost> get_gather_plan(const Layout& L, int axis, int w,
                                                      int path_req, int64_t batch) {
  Key k = make_key(L, nullptr, (u64)axis, w, path_req, batch);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_gcache.find(k);
    if (it != g_gcache.end()) return it->second;
  }
  auto P = build_gather_plan(L, axis, w, path_req, batch);
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_gcache.size() >= kMaxCached) g_gcache.clear();
  g_gcache[k] = P;
  return P;
}

}  // namespace ll
