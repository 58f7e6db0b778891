// planner_regs.cpp -- register-faithful plans (LL_PATH_REGS, LL_PATH_REGS_SHUFFLE).
#include <algorithm>
#include <array>
#include <sstream>

#include "planner_internal.hpp"

namespace ll {
namespace detail {

// Common frame of the register-faithful plans: both layouts are reg / lane /
// warp / block with 5 lane bits, equal reg and warp bits and identical block
// columns; tile vectors in A's (reg, lane, warp) index space; B's word must
// hold elements A holds in registers (load-side prmt swaps).
struct RegsFrame {
  int w, lw, nr, nw, d, n, kw, LB, NW;
  bool words_ok;        // B's word elements are among A's registers (swaps below)
  std::vector<std::pair<int, int>> swaps;
  std::vector<u64> WB, Aw, Bw, Al, Bl, Awp, Bwp;
  std::vector<u64> Aw0;  // A's word-level columns without the swaps
};

bool regs_frame(const ConvertPlan& P, const Layout& A, const Layout& B, const std::vector<u64>& X,
                RegsFrame& f) {
  const int w = P.w;
  if (w > 4 || P.nA != P.nB) return false;
  auto dims_ok = [](const Layout& L) {
    static const char* order[] = {"reg", "lane", "warp", "block"};
    size_t k = 0;
    for (auto& d : L.in) {
      while (k < 4 && d.name != order[k]) ++k;
      if (k == 4) return false;
      ++k;
    }
    return true;
  };
  if (!dims_ok(A) || !dims_ok(B)) return false;
  const int nr = A.in_size("reg"), nw = A.in_size("warp");
  if (B.in_size("reg") != nr || B.in_size("warp") != nw || A.in_size("lane") != 5 ||
      B.in_size("lane") != 5 || nw > 3)
    return false;
  const int d = nr + 5 + nw;
  const int n = P.nB;
  for (int k = d; k < n; ++k)
    if (X[k] != (u64(1) << k)) return false;  // block bits: identical columns
  const u64 tmask = (u64(1) << d) - 1;
  for (int k = 0; k < d; ++k)
    if (!X[k] || (X[k] & ~tmask)) return false;
  {
    std::vector<u64> xt(X.begin(), X.begin() + d);
    if (f2_rank(xt) != d) return false;
  }
  const int lw = ilog2i(w);
  const int kw = ilog2i(4 / w);             // element bits inside a 32-bit word
  if (nr < kw) return false;
  const int LB = nr - kw;                   // word-index bits
  const int NW = 1 << LB;
  if (NW > 64) return false;
  auto e = [](int i) { return u64(1) << i; };
  // word bits: B's word must hold the same elements as A's (prmt swaps on load)
  // (any of A's register bits can be moved into the word by prmt / renames
  // on load, the paper's register permutation P_reg)
  std::vector<u64> WB(X.begin(), X.begin() + kw);
  std::vector<std::pair<int, int>> swaps;
  std::vector<u64> cur;  // A's register columns in register order after the swaps
  for (int t = 0; t < nr; ++t) cur.push_back(e(t));
  const std::vector<u64> cur0 = cur;
  bool words_ok = true;
  for (int t = 0; t < kw && words_ok; ++t) {
    auto it = std::find(cur.begin(), cur.end(), WB[t]);
    int s = it == cur.end() ? -1 : (int)(it - cur.begin());
    if (s < t) { words_ok = false; break; }
    if (s != t) { swaps.push_back({t, s}); std::swap(cur[t], cur[s]); }
  }
  if (!words_ok) {  // only ldmatrix / stmatrix .trans options can serve (plan_regs)
    swaps.clear();
    cur = cur0;
  }
  // word-level columns, lanes, warps of both sides (tile vectors)
  std::vector<u64> Aw, Bw, Al, Bl, Awp, Bwp;
  for (int u = 0; u < LB; ++u) { Aw.push_back(cur[kw + u]); Bw.push_back(X[kw + u]); }
  for (int b = 0; b < 5; ++b) { Al.push_back(e(nr + b)); Bl.push_back(X[nr + b]); }
  for (int b = 0; b < nw; ++b) { Awp.push_back(e(nr + 5 + b)); Bwp.push_back(X[nr + 5 + b]); }
  f.w = w; f.lw = lw; f.nr = nr; f.nw = nw; f.d = d; f.n = n; f.kw = kw; f.LB = LB; f.NW = NW;
  f.words_ok = words_ok;
  f.swaps = swaps;
  f.WB = WB; f.Aw = Aw; f.Bw = Bw; f.Al = Al; f.Bl = Bl; f.Awp = Awp; f.Bwp = Bwp;
  for (int u = 0; u < LB; ++u) f.Aw0.push_back(cur0[kw + u]);
  return true;
}

// Register-faithful plan (LL_PATH_REGS): the paper's in-kernel conversion.
// Tile-local vectors live in A's (reg, lane, warp) index space: A's input bit
// i is e_i, B's input bit k is X[k].  Shared memory S = the paper's optimal
// swizzle for the two sides' bank-relevant thread vectors with S_vect =
// [word bits, granule bits]; each side writes / reads either vectors
// (generalised vectorisation) or stmatrix / ldmatrix rows when its
// layout divided by the tile T = id^{reg,offset}_k x id^{thread,offset}_2
// (left division P:354-362) exists -- checked on S^{-1} o L.
bool plan_regs(ConvertPlan& P, const Layout& A, const Layout& B, const std::vector<u64>& X,
               std::ostringstream& js) {
  RegsFrame f;
  if (!regs_frame(P, A, B, X, f)) return false;
  const int w = f.w, lw = f.lw, nr = f.nr, nw = f.nw, d = f.d, n = f.n, kw = f.kw, LB = f.LB, NW = f.NW;
  (void)nr;
  auto e = [](int i) { return u64(1) << i; };
  const auto &WB = f.WB, &Bw = f.Bw, &Al = f.Al, &Bl = f.Bl, &Awp = f.Awp, &Bwp = f.Bwp;
  // per option: with the load-side swaps (A's words = B's words) or without
  // (the .trans options, where each side keeps its own words)
  std::vector<std::pair<int, int>> swaps;
  std::vector<u64> Aw;
  auto pos = [](const std::vector<u64>& v, u64 x) {
    auto it = std::find(v.begin(), v.end(), x);
    return it == v.end() ? -1 : (int)(it - v.begin());
  };
  const bool allow_mat = planner_knob("regs_matrix", 1) != 0;
  // candidate granule rows: (extra S_vect vectors beyond the word, side kinds)
  struct Opt {
    std::vector<u64> gv;     // granule vectors after the word bits (<= 2)
    std::vector<u64> svect;  // .trans options: the full S_vect (else WB + gv)
    int wr_mat = 0, rd_mat = 0, wr_gw = 1, rd_gw = 1;   // mat: 0 vector, 1 matrix, 2 matrix.trans
    int wa = -1, wb = -1, ra = -1, rb = -1;
    int cost = 1 << 30;
  };
  std::vector<Opt> opts;
  auto side = [&](const std::vector<u64>& gv, const std::vector<u64>& W, const std::vector<u64>& L,
                  int& mat, int& gw, int& a, int& b) {
    // matrix: the granule rows are exactly the side's lanes 0, 1
    if (allow_mat && gv.size() == 2 && L[0] == gv[0] && L[1] == gv[1]) {
      mat = 1;
      gw = std::min(4, NW);
      a = LB > 0 ? 0 : -1;
      b = LB > 1 ? 1 : -1;
      return;
    }
    // vector: the longest prefix of gv the side holds as word bits
    mat = 0;
    int q = 0;
    a = b = -1;
    if (q < (int)gv.size() && pos(W, gv[0]) >= 0) { a = pos(W, gv[0]); ++q; }
    if (q == 1 && q < (int)gv.size() && pos(W, gv[1]) >= 0) { b = pos(W, gv[1]); ++q; }
    gw = 1 << q;
  };
  auto consider = [&](const std::vector<u64>& gv) {
    Opt o;
    o.gv = gv;
    side(gv, Aw, Al, o.wr_mat, o.wr_gw, o.wa, o.wb);
    side(gv, Bw, Bl, o.rd_mat, o.rd_gw, o.ra, o.rb);
    o.cost = NW / o.wr_gw + NW / o.rd_gw;
    opts.push_back(o);
  };
  if (f.words_ok) {
    swaps = f.swaps;
    Aw = f.Aw;
    {  // generalised vectorisation: word-level columns common to both sides
      std::vector<u64> gv;
      for (u64 x : Aw) if (pos(Bw, x) >= 0 && gv.size() < 2) gv.push_back(x);
      consider(gv);
    }
    if (allow_mat) {
      consider({Al[0], Al[1]});
      consider({Bl[0], Bl[1]});
    }
  }
  // ldmatrix / stmatrix .trans (b16): the 16-byte row is the side's lanes
  // 2..4 (thread t holds rows 2(t%4), 2(t%4)+1 of column t/4), so each side
  // keeps its own word and no load-side swap is needed -- the transposes
  if (w == 2 && allow_mat && planner_knob("regs_trans", 1)) {
    const std::vector<u64> TA = {Al[2], Al[3], Al[4]}, TB = {Bl[2], Bl[3], Bl[4]};
    const u64 a0 = e(0), b0 = X[0];  // each side's word element bit
    auto side_t = [&](const std::vector<u64>& T, u64 w0, const std::vector<u64>& W,
                      const std::vector<u64>& L, int& mat, int& gw, int& a, int& b) -> bool {
      a = b = -1;
      if (T == std::vector<u64>{L[2], L[3], L[4]}) {   // .trans too
        mat = 2; gw = std::min(4, NW); a = LB > 0 ? 0 : -1; b = LB > 1 ? 1 : -1;
        return true;
      }
      if (w0 != T[0]) return false;                    // the side's word must be the row's pair
      if (T[1] == L[0] && T[2] == L[1]) {              // plain matrix
        mat = 1; gw = std::min(4, NW); a = LB > 0 ? 0 : -1; b = LB > 1 ? 1 : -1;
        return true;
      }
      mat = 0;
      int q = 0;
      if (pos(W, T[1]) >= 0) { a = pos(W, T[1]); ++q; }
      if (q == 1 && pos(W, T[2]) >= 0) { b = pos(W, T[2]); ++q; }
      gw = 1 << q;
      return true;
    };
    for (int which = 0; which < 2; ++which) {
      const std::vector<u64>& T = which ? TB : TA;
      Opt o;
      o.svect = T;
      if (!side_t(T, a0, f.Aw0, Al, o.wr_mat, o.wr_gw, o.wa, o.wb)) continue;
      if (!side_t(T, b0, Bw, Bl, o.rd_mat, o.rd_gw, o.ra, o.rb)) continue;
      if (o.wr_mat != 2 && o.rd_mat != 2) continue;
      o.cost = NW / o.wr_gw + NW / o.rd_gw;
      opts.push_back(o);
    }
  }
  // sm_100a 8-bit matrix tiles (w = 1; measured on the B200, tools/b8_probe.cu,
  // pinned in test_b8_matrix_tiles_measured_on_b200_are_linear_layouts):
  //   stmatrix.m16n8.x{1,2,4}.trans.b8: word bytes (e0, e1) -> (row 1, col 8),
  //     lanes 0..4 -> (row 2, row 4, col 1, 2, 4); 8 rows of 16 B per matrix,
  //     row r of matrix m addressed by lane 8m + r
  //   ldmatrix.m16n16.x{1,2}.trans.b8: two words per matrix; bytes (e0, e1)
  //     -> (row 1, row 2), word 1 -> col 8, lanes -> (row 4, row 8, col 1,
  //     2, 4); 16 rows of 16 B, row r of matrix m addressed by lane 16m + r
  // The tile's 16-byte row (the smem granule S_vect) is the side's lanes
  // 2..4 plus element bit 1 (store) or an instruction word bit (load); left
  // division of S^{-1} o L by the tile is checked
  // below.  Either side may instead use vectors whose word bytes are the
  // row's first two vectors (the other side's transposition).
  if (w == 1 && planner_knob("regs_b8", 1)) {
    const std::vector<u64> RA = {Al[2], Al[3], Al[4], e(1)};
    auto vec_side = [&](const std::vector<u64>& row, u64 e0, u64 e1, const std::vector<u64>& W,
                        int& gw, int& a, int& b) -> bool {
      a = b = -1;
      if (e0 != row[0] || e1 != row[1]) return false;
      int q = 0;
      if (pos(W, row[2]) >= 0) { a = pos(W, row[2]); ++q; }
      if (q == 1 && pos(W, row[3]) >= 0) { b = pos(W, row[3]); ++q; }
      gw = 1 << q;
      return true;
    };
    // A writes with stmatrix.b8
    {
      Opt o;
      o.svect = RA;
      o.wr_mat = 3;
      o.wr_gw = std::min(4, NW);
      o.wa = LB > 0 ? 0 : -1;
      o.wb = LB > 1 ? 1 : -1;
      bool ok = false;
      for (int u = 0; u < LB && !ok; ++u) {
        if (NW < 2 || !(Bl[2] == RA[0] && Bl[3] == RA[1] && Bl[4] == RA[2] && Bw[u] == RA[3])) continue;
        o.rd_mat = 3; o.rd_gw = std::min(4, NW); o.ra = u; o.rb = -1;
        for (int v = 0; v < LB && o.rd_gw == 4; ++v) if (v != u) { o.rb = v; break; }
        ok = true;
      }
      if (!ok) ok = vec_side(RA, X[0], X[1], Bw, o.rd_gw, o.ra, o.rb);
      if (ok) {
        o.cost = NW / o.wr_gw + NW / o.rd_gw;
        opts.push_back(o);
      }
    }
    // B reads with ldmatrix.b8 (column-8 word bit u), A writes vectors
    for (int u = 0; u < LB && NW >= 2; ++u) {
      Opt o;
      o.svect = {Bl[2], Bl[3], Bl[4], Bw[u]};
      o.rd_mat = 3;
      o.rd_gw = std::min(4, NW);
      o.ra = u;
      o.rb = -1;
      for (int v = 0; v < LB && o.rd_gw == 4; ++v) if (v != u) { o.rb = v; break; }
      if (!vec_side(o.svect, e(0), e(1), f.Aw0, o.wr_gw, o.wa, o.wb)) continue;
      o.cost = NW / o.wr_gw + NW / o.rd_gw;
      opts.push_back(o);
    }
  }
  if (opts.empty()) return false;
  // options by cost (instructions per thread), matrix instructions first on
  // ties (the paper's preference for hardware primitives); an option
  // whose layouts turn out not divisible by the matrix tile under the
  // constructed S is dropped for the next one
  std::stable_sort(opts.begin(), opts.end(), [](const Opt& x, const Opt& y) {
    if (x.cost != y.cost) return x.cost < y.cost;
    return x.wr_mat + x.rd_mat > y.wr_mat + y.rd_mat;
  });
  SwizzleResult sw;
  std::vector<u64> At, Bt, V;
  Opt best;
  auto build = [&](const Opt& o) -> bool {
    best = o;
    const bool own = !o.svect.empty();   // .trans option: no load-side swaps
    swaps = own ? std::vector<std::pair<int, int>>{} : f.swaps;
    Aw = own ? f.Aw0 : f.Aw;
    const u64 wA = own ? e(0) : (WB.empty() ? 0 : WB[0]), wB = X[0];
    if (own) {
      V = o.svect;
    } else {
      V = WB;  // S_vect: word bits (B's order), then the granule rows
      for (u64 x : best.gv) V.push_back(x);
    }
    // bank-relevant thread vectors per side (phase order): lanes for vector
    // accesses; the address providers (rows = lanes 2..4, then the matrix
    // select word bits) for stmatrix / ldmatrix
    auto thr_vecs = [&](int mat, const std::vector<u64>& W, const std::vector<u64>& L, int a, int b,
                        u64 w0, bool ld) {
      std::vector<u64> t;
      if (!mat) return L;
      if (mat == 3) {
        // b8 address providers: rows (element bits, lanes 0, 1), then the matrix selects
        t = ld ? std::vector<u64>{w0, X[1], L[0], L[1]} : std::vector<u64>{w0, L[0], L[1]};
        if (!ld && a >= 0) t.push_back(W[a]);
        if (b >= 0) t.push_back(W[b]);
        while (t.size() < 5) t.push_back(L[2]);
        return t;
      }
      t = mat == 2 ? std::vector<u64>{w0, L[0], L[1]} : std::vector<u64>{L[2], L[3], L[4]};
      if (a >= 0) t.push_back(W[a]);
      if (b >= 0) t.push_back(W[b]);
      while (t.size() < 5) t.push_back(L[2]);  // padding (dropped by the phase rule)
      return t;
    };
    At = thr_vecs(best.wr_mat, Aw, Al, best.wa, best.wb, wA, false);
    Bt = thr_vecs(best.rd_mat, Bw, Bl, best.ra, best.rb, wB, true);
    sw = optimal_swizzle(At, Bt, V, d, w);
    std::vector<u64> Scols = sw.vect;
    Scols.insert(Scols.end(), sw.bank.begin(), sw.bank.end());
    Scols.insert(Scols.end(), sw.idx.begin(), sw.idx.end());
    if (f2_rank(Scols) != d) return false;
    auto Sinv = f2_right_inverse(Scols, d);
    if (d + lw > 31) return false;
    auto boff = [&](u64 v) -> uint32_t { return (uint32_t)f2_apply(Sinv, v) << lw; };
    // tile matching by left division of S^{-1} o L by the matrix tile: the
    // word bits and lanes 0, 1 must be offset bits 0..k+1 and no other column
    // may touch them
    auto divisible = [&](const std::vector<u64>& W0, const std::vector<u64>& L,
                         const std::vector<u64>& rest) {
      const u64 low = (u64(1) << (kw + 2)) - 1;
      for (int t = 0; t < kw; ++t)
        if (f2_apply(Sinv, W0[t]) != e(t)) return false;
      if (f2_apply(Sinv, L[0]) != e(kw) || f2_apply(Sinv, L[1]) != e(kw + 1)) return false;
      for (u64 c : rest)
        if (f2_apply(Sinv, c) & low) return false;
      return true;
    };
    auto rest_of = [&](const std::vector<u64>& W, const std::vector<u64>& L, const std::vector<u64>& Wp) {
      std::vector<u64> r(W);
      r.insert(r.end(), L.begin() + 2, L.end());
      r.insert(r.end(), Wp.begin(), Wp.end());
      return r;
    };
    // .trans tile: the row's 8 elements are lanes 2..4 (offset bits 0..2); the
    // word bit and lanes 0, 1 select rows, like every other column
    auto divisible_t = [&](u64 w0, const std::vector<u64>& W, const std::vector<u64>& L,
                           const std::vector<u64>& Wp) {
      for (int t = 0; t < 3; ++t)
        if (f2_apply(Sinv, L[2 + t]) != e(t)) return false;
      std::vector<u64> rest(W);
      rest.push_back(w0);
      rest.push_back(L[0]);
      rest.push_back(L[1]);
      rest.insert(rest.end(), Wp.begin(), Wp.end());
      for (u64 c : rest)
        if (f2_apply(Sinv, c) & 7u) return false;
      return true;
    };
    if (best.wr_mat == 1 && !divisible(own ? std::vector<u64>{wA} : WB, Al, rest_of(Aw, Al, Awp))) return false;
    if (best.rd_mat == 1 && !divisible(own ? std::vector<u64>{wB} : WB, Bl, rest_of(Bw, Bl, Bwp))) return false;
    if (best.wr_mat == 2 && !divisible_t(wA, Aw, Al, Awp)) return false;
    if (best.rd_mat == 2 && !divisible_t(wB, Bw, Bl, Bwp)) return false;
    if (w == 1 && (best.wr_mat == 3 || best.rd_mat == 3)) {
      // b8 tiles: the row vectors are offset bits 0..3 and no other column of
      // the side touches them; vector sides: bytes, then the granule's words,
      // at the low offset bits, nothing else below the granule
      auto b8_ok = [&](int mat, const std::vector<u64>& row, const std::vector<u64>& others) {
        for (int t = 0; t < 4; ++t)
          if (mat == 3 && f2_apply(Sinv, row[t]) != e(t)) return false;
        for (u64 c : others)
          if (f2_apply(Sinv, c) & 15u) return false;
        return true;
      };
      auto vec_ok = [&](u64 e0, u64 e1, const std::vector<u64>& W, int a, int b, int gw,
                        const std::vector<u64>& L, const std::vector<u64>& Wp) {
        std::vector<u64> gran = {e0, e1};
        if (gw >= 2) gran.push_back(W[a]);
        if (gw >= 4) gran.push_back(W[b]);
        for (size_t t = 0; t < gran.size(); ++t)
          if (f2_apply(Sinv, gran[t]) != e((int)t)) return false;
        const u64 low = (u64(1) << gran.size()) - 1;
        std::vector<u64> rest(L);
        rest.insert(rest.end(), Wp.begin(), Wp.end());
        for (int u = 0; u < (int)W.size(); ++u)
          if (!(gw >= 2 && u == a) && !(gw >= 4 && u == b)) rest.push_back(W[u]);
        for (u64 c : rest)
          if (f2_apply(Sinv, c) & low) return false;
        return true;
      };
      const std::vector<u64>& row = best.svect;
      if (best.wr_mat == 3) {
        std::vector<u64> oth = {e(0), Al[0], Al[1]};
        oth.insert(oth.end(), Aw.begin(), Aw.end());
        oth.insert(oth.end(), Awp.begin(), Awp.end());
        if (!b8_ok(3, row, oth)) return false;
      } else if (!vec_ok(e(0), e(1), Aw, best.wa, best.wb, best.wr_gw, Al, Awp)) {
        return false;
      }
      if (best.rd_mat == 3) {
        std::vector<u64> oth = {X[0], X[1], Bl[0], Bl[1]};
        for (int u = 0; u < LB; ++u) if (u != best.ra) oth.push_back(Bw[u]);
        oth.insert(oth.end(), Bwp.begin(), Bwp.end());
        if (!b8_ok(3, row, oth)) return false;
      } else if (!vec_ok(X[0], X[1], Bw, best.ra, best.rb, best.rd_gw, Bl, Bwp)) {
        return false;
      }
    }
    // vector sides read / write whole words: their word must be offset bit 0
    if (own && w == 2 && best.wr_mat == 0 && f2_apply(Sinv, wA) != 1) return false;
    if (own && w == 2 && best.rd_mat == 0 && f2_apply(Sinv, wB) != 1) return false;
    RegsPlan& rp = P.rp;
    rp = RegsPlan{};
    rp.nw = nw;
    rp.nwords = NW;
    rp.tile_bytes = int64_t(w) << d;
    rp.n_tiles = (int64_t(1) << (n - d)) * P.batch;
    rp.wr_mat = best.wr_mat;
    rp.rd_mat = best.rd_mat;
    rp.wr_gw = best.wr_gw;
    rp.rd_gw = best.rd_gw;
    rp.n_swaps = (int)swaps.size();
    for (size_t i = 0; i < swaps.size(); ++i) {
      rp.swap_a[i] = (int8_t)swaps[i].first;
      rp.swap_b[i] = (int8_t)swaps[i].second;
    }
    // canonical word order per side: the instruction's words at word bits 0
    // (and 1), realised by transpositions (recorded for the kernel)
    auto canon = [&](std::vector<u64> W, int a, int b, int gw, int& ns, int8_t* sa, int8_t* sb) {
      ns = 0;
      std::vector<u64> sel;
      if (gw >= 2 && a >= 0) sel.push_back(W[a]);
      if (gw >= 4 && b >= 0) sel.push_back(W[b]);
      for (size_t t = 0; t < sel.size(); ++t) {
        const int s2 = pos(W, sel[t]);
        if (s2 != (int)t) {
          sa[ns] = (int8_t)std::min<int>((int)t, s2);
          sb[ns] = (int8_t)std::max<int>((int)t, s2);
          ++ns;
          std::swap(W[t], W[s2]);
        }
      }
      return W;
    };
    const std::vector<u64> Awc = canon(Aw, best.wa, best.wb, best.wr_gw, rp.n_wsw, rp.wsw_a, rp.wsw_b);
    const std::vector<u64> Bwc = canon(Bw, best.ra, best.rb, best.rd_gw, rp.n_rsw, rp.rsw_a, rp.rsw_b);
    auto fill = [&](int mat, const std::vector<u64>& W, const std::vector<u64>& L,
                    const std::vector<u64>& Wp, int a, int b, int gw, uint32_t* thr, uint32_t* inst,
                    u64 wrow0, bool ld) {
      if (mat == 3) {
        // b8: address provider lane p; store: p bits 0..2 = rows (e0, lanes
        // 0, 1), bits 3, 4 = matrix (words a, b); load: p bits 0..3 = rows
        // (e0, e1, lanes 0, 1), bit 4 = matrix (word b)
        thr[0] = boff(wrow0);
        if (ld) {
          thr[1] = boff(X[1]);
          thr[2] = boff(L[0]);
          thr[3] = boff(L[1]);
          thr[4] = b >= 0 && gw >= 4 ? boff(W[b]) : 0;
        } else {
          thr[1] = boff(L[0]);
          thr[2] = boff(L[1]);
          thr[3] = a >= 0 && gw >= 2 ? boff(W[a]) : 0;
          thr[4] = b >= 0 && gw >= 4 ? boff(W[b]) : 0;
        }
      } else if (mat) {
        // address provider lane p: rows = p bits 0..2 (the data lanes 2..4;
        // .trans: the word bit and lanes 0, 1), matrix = p bits 3, 4 (the
        // selected word bits)
        thr[0] = boff(mat == 2 ? wrow0 : L[2]);
        thr[1] = boff(mat == 2 ? L[0] : L[3]);
        thr[2] = boff(mat == 2 ? L[1] : L[4]);
        thr[3] = a >= 0 && gw >= 2 ? boff(W[a]) : 0;
        thr[4] = b >= 0 && gw >= 4 ? boff(W[b]) : 0;
      } else {
        for (int q = 0; q < 5; ++q) thr[q] = boff(L[q]);
      }
      for (int q = 0; q < nw; ++q) thr[5 + q] = boff(Wp[q]);
      // instruction j: the word bits other than the selected ones, ascending
      const int ninst = NW / gw;
      if (ninst > LL_REGS_MAX_INST) return false;
      std::vector<int> other;
      for (int u = 0; u < LB; ++u)
        if (!(u == a && gw >= 2) && !(u == b && gw >= 4)) other.push_back(u);
      for (int j = 0; j < ninst; ++j) {
        uint32_t o = 0;
        for (size_t q = 0; q < other.size(); ++q)
          if ((j >> q) & 1) o ^= boff(W[other[q]]);
        inst[j] = o;
      }
      return true;
    };
    if (!fill(rp.wr_mat, Awc, Al, Awp, LB > 0 ? 0 : -1, LB > 1 ? 1 : -1, rp.wr_gw, rp.sw_thr, rp.sw_inst, wA, false))
      return false;
    if (!fill(rp.rd_mat, Bwc, Bl, Bwp, LB > 0 ? 0 : -1, LB > 1 ? 1 : -1, rp.rd_gw, rp.sr_thr, rp.sr_inst, wB, true))
      return false;
    P.nv = NW;
    P.tile_bits = d;
    P.pred_wf_ld = lemma_wavefronts(sw, At, w);
    P.pred_wf_st = lemma_wavefronts(sw, Bt, w);
    return true;
  };
  bool ok = false;
  for (auto& o : opts)
    if ((ok = build(o))) break;
  if (!ok) return false;
  RegsPlan& rp = P.rp;
  static const char* kinds[] = {"st.shared", "stmatrix", "stmatrix.trans", "stmatrix.m16n8.trans.b8",
                                "ld.shared", "ldmatrix", "ldmatrix.trans", "ldmatrix.m16n16.trans.b8"};
  js << ",\"regs\":{\"warps_log2\":" << nw << ",\"words_per_thread\":" << NW
     << ",\"write\":\"" << kinds[rp.wr_mat] << "\",\"write_words\":" << rp.wr_gw
     << ",\"read\":\"" << kinds[4 + rp.rd_mat] << "\",\"read_words\":" << rp.rd_gw
     << ",\"write_instr_per_thread\":" << NW / rp.wr_gw
     << ",\"read_instr_per_thread\":" << NW / rp.rd_gw << ",\"n_tiles\":" << rp.n_tiles
     << ",\"swaps\":" << swaps.size() << ",\"sw_thr\":" << u32_json(rp.sw_thr, 5 + nw)
     << ",\"sr_thr\":" << u32_json(rp.sr_thr, 5 + nw)
     << ",\"wsw\":[";
  for (int i = 0; i < rp.n_wsw; ++i) js << (i ? "," : "") << "[" << int(rp.wsw_a[i]) << "," << int(rp.wsw_b[i]) << "]";
  js << "],\"rsw\":[";
  for (int i = 0; i < rp.n_rsw; ++i) js << (i ? "," : "") << "[" << int(rp.rsw_a[i]) << "," << int(rp.rsw_b[i]) << "]";
  js << "],\"sw_inst\":" << u32_json(rp.sw_inst, NW / rp.wr_gw)
     << ",\"sr_inst\":" << u32_json(rp.sr_inst, NW / rp.rd_gw) << "},\"S_vect\":" << vec_json(sw.vect)
     << ",\"S_bank\":" << vec_json(sw.bank) << ",\"S_idx\":" << vec_json(sw.idx)
     << ",\"granule_bytes\":" << ((w << (int)V.size()))
     << ",\"pred_wavefronts_per_sts\":" << P.pred_wf_ld
     << ",\"pred_wavefronts_per_lds\":" << P.pred_wf_st;
  return true;
}

// Register-faithful warp-shuffle plan (LL_PATH_REGS_SHUFFLE): warp-local
// pairs only ((B^{-1} o A)_warp = I): both directions of the paper's
// exchange on the layouts' own registers and lanes.
bool plan_regs_shuffle(ConvertPlan& P, const Layout& A, const Layout& B,
                       const std::vector<u64>& X, std::ostringstream& js) {
  RegsFrame f;
  if (!regs_frame(P, A, B, X, f) || !f.words_ok) return false;
  if (f.NW > LL_MAX_GRAN) return false;
  for (int b = 0; b < f.nw; ++b)
    if (f.Bwp[b] != f.Awp[b]) return false;
  const u64 wmask = (u64(1) << (f.nr + 5)) - 1;  // (reg, lane) space of one warp
  for (u64 v : f.Bw) if (v & ~wmask) return false;
  for (u64 v : f.Bl) if (v & ~wmask) return false;
  ShuffleCore fw = shuffle_core(f.Aw, f.Al, f.Bw, f.Bl, f.LB);
  ShuffleCore bw = shuffle_core(f.Bw, f.Bl, f.Aw, f.Al, f.LB);
  if (!fw.ok || !bw.ok) return false;
  RegsShufflePlan& q = P.rsp;
  q = RegsShufflePlan{};
  q.nw = f.nw;
  q.nwords = f.NW;
  q.tile_bytes = int64_t(f.w) << f.d;
  q.n_tiles = (int64_t(1) << (f.n - f.d)) * P.batch;
  q.swaps = f.swaps;
  auto fill = [&](const ShuffleCore& c, ShuffleDir& dd) {
    for (int k = 0; k < c.rounds; ++k) {
      int a = 0, e = 0;
      for (int j = 0; j < f.LB; ++j)
        if ((k >> j) & 1) { a ^= (int)c.alpha[j]; e ^= (int)c.epsm[j]; }
      dd.alpha.push_back(a);
      dd.eps.push_back(e);
      dd.gamma.push_back(c.gamma[k]);
    }
    for (int b = 0; b < 5; ++b) { dd.beta[b] = c.beta[b]; dd.zeta[b] = c.zeta[b]; dd.delta[b] = c.delta[b]; }
    dd.beta_any = c.beta_any;
    dd.zeta_any = c.zeta_any;
  };
  fill(fw, q.fwd);
  fill(bw, q.bwd);
  P.nv = f.NW;
  P.tile_bits = f.d;
  // a register permutation (identical lanes) costs no shuffle round
  P.shuffle_rounds = f.Al == f.Bl ? 0 : fw.rounds;
  js << ",\"regs_shuffle\":{\"warps_log2\":" << f.nw << ",\"words_per_thread\":" << f.NW
     << ",\"rounds\":" << fw.rounds << ",\"I\":" << vec_json(fw.I) << ",\"E\":" << vec_json(fw.E)
     << ",\"F\":" << vec_json(fw.F) << ",\"G\":" << vec_json(fw.Gv) << ",\"R\":" << vec_json(fw.R)
     << ",\"beta_lane\":" << u32_json(q.fwd.beta, 5) << ",\"zeta_lane\":" << u32_json(q.fwd.zeta, 5)
     << ",\"delta_lane\":" << u32_json(q.fwd.delta, 5) << ",\"swaps\":" << f.swaps.size()
     << ",\"exchange\":\"" << (f.Al == f.Bl ? "register permutation" : "warp shuffles") << "\""
     << ",\"n_tiles\":" << q.n_tiles << "}";
  return true;
}

}  // namespace detail
}  // namespace ll
