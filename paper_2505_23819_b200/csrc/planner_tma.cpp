// planner_tma.cpp -- cp.async / TMA-fed shared-memory plans (LL_PATH_SMEM_ASYNC,
// LL_PATH_SMEM_TMA, LL_PATH_SMEM_TMA_STORE).
#include <algorithm>
#include <array>
#include <sstream>

#include "planner_internal.hpp"

namespace ll {
namespace detail {

// Asynchronous-copy variant of the shared-memory path (LL_PATH_SMEM_ASYNC):
// the source tile goes HBM -> shared memory with cp.async (16-byte chunks,
// no registers, several tiles in flight per group), so the shared-memory
// granule is the *source* 16-byte vector V = VS; the reading side holds
// VS u VD in registers and permutes into destination vectors (prmt for the
// sub-word bits, compile-time STG operand selection for the word bits).  The
// swizzle S is the paper's construction for (writer, reader) with V = VS.
bool plan_async(ConvertPlan& P, const std::vector<u64>& X, std::ostringstream& js) {
  const int n = P.nB, w = P.w;
  if (P.nA != P.nB || n > 62 || w > 8) return false;
  std::vector<int> sigma(n), sinv(n, -1);
  for (int k = 0; k < n; ++k) {
    if (popcount64(X[k]) != 1) return false;
    sigma[k] = ctz64(X[k]);
    if (sinv[sigma[k]] >= 0) return false;
    sinv[sigma[k]] = k;
  }
  const int vb = ilog2i(16 / w);
  if (n < vb + 5) return false;
  auto contains = [](const std::vector<int>& v, int x) {
    return std::find(v.begin(), v.end(), x) != v.end();
  };
  std::vector<int> VD, VS, CD, CS;
  for (int k = 0; k < vb; ++k) { VD.push_back(k); VS.push_back(sinv[k]); }
  const int cbits = std::max(0, ilog2i(std::max(16, planner_knob("run_bytes", 256)) / 16));
  for (int k = vb; k < std::min(n, vb + cbits); ++k) { CD.push_back(k); CS.push_back(sinv[k]); }
  const int r_max = ilog2i(std::max(16, std::min(128, planner_knob("thread_bytes_max", 128))) / w);
  const int r_pref = std::min(r_max, ilog2i(std::max(16, planner_knob("thread_bytes", 64)) / w));
  std::vector<int> need = VS;
  for (int x : VD) if (!contains(need, x)) need.push_back(x);
  if ((int)need.size() > r_max || (int)need.size() + 5 > n) return false;
  int r = std::min(std::max((int)need.size(), r_pref), std::min(r_max, n - 5));
  std::vector<int> T = VD;
  for (auto* s : {&VS, &CD, &CS, &need})
    for (int x : *s) if (!contains(T, x)) T.push_back(x);
  for (int k = 0; (int)T.size() < r + 5 && k < n; ++k)
    if (!contains(T, k)) T.push_back(k);
  int g = (int)T.size() - r - 5;
  if (g > 3) {
    int r2 = std::min(r_max, (int)T.size() - 5 - 3);
    if (r2 > r) { r = r2; g = (int)T.size() - r - 5; }
  }
  if (g < 0 || g > 3) return false;
  std::sort(T.begin(), T.end());
  // reader (store side): rho = VS (granule order), VD \ VS, extra (highest dst, not CD)
  std::vector<int> rd_reg = VS;
  for (int x : VD) if (!contains(rd_reg, x)) rd_reg.push_back(x);
  {
    std::vector<int> cand;
    for (int x : T) if (!contains(rd_reg, x) && !contains(CD, x)) cand.push_back(x);
    std::sort(cand.begin(), cand.end(), [](int a, int b) { return a > b; });
    for (int x : cand) { if ((int)rd_reg.size() == r) break; rd_reg.push_back(x); }
    if ((int)rd_reg.size() != r) return false;
  }
  std::vector<int> rd_lane, rd_warp;
  {
    for (int x : CD) if (!contains(rd_reg, x) && rd_lane.size() < 5) rd_lane.push_back(x);
    std::vector<int> cand;
    for (int x : T) if (!contains(rd_reg, x) && !contains(rd_lane, x)) cand.push_back(x);
    std::sort(cand.begin(), cand.end());
    for (int x : cand) (rd_lane.size() < 5 ? rd_lane : rd_warp).push_back(x);
  }
  // writer (cp.async): rho = VS + unroll (highest src, not CS); lanes lowest src
  std::vector<int> wr_reg = VS;
  {
    std::vector<int> cand;
    for (int x : T) if (!contains(wr_reg, x) && !contains(CS, x)) cand.push_back(x);
    std::sort(cand.begin(), cand.end(), [&](int a, int b) { return sigma[a] > sigma[b]; });
    for (int x : cand) { if ((int)wr_reg.size() == r) break; wr_reg.push_back(x); }
    if ((int)wr_reg.size() != r) return false;
  }
  std::vector<int> wr_lane, wr_warp;
  {
    std::vector<int> cand;
    for (int x : T) if (!contains(wr_reg, x)) cand.push_back(x);
    std::sort(cand.begin(), cand.end(), [&](int a, int b) { return sigma[a] < sigma[b]; });
    for (int x : cand) (wr_lane.size() < 5 ? wr_lane : wr_warp).push_back(x);
  }
  if (rd_lane.size() != 5 || wr_lane.size() != 5 || (int)rd_warp.size() != g ||
      (int)wr_warp.size() != g)
    return false;
  // reader sub-word swaps (prmt): rho positions 0..nsub-1 must hold VD[0..nsub)
  const int nsub = w >= 4 ? 0 : ilog2i(4 / w);
  std::vector<int> order = rd_reg;
  std::vector<std::pair<int, int>> swaps;
  for (int t = 0; t < nsub; ++t) {
    int s = (int)(std::find(order.begin(), order.end(), VD[t]) - order.begin());
    if (s != t) { swaps.push_back({t, s}); std::swap(order[t], order[s]); }
  }
  if ((int)swaps.size() > LL_MAX_SWAPS) return false;
  auto wordbit = [&](int rho) { return w == 8 ? rho + 1 : rho - nsub; };
  const int LB = w == 8 ? r + 1 : r - nsub;
  std::vector<int> ssel;  // word bits forming a 16-byte store vector (2 word bits)
  if (w == 8) ssel.push_back(0);
  for (int t = (w == 8 ? 0 : nsub); t < vb; ++t) {
    int pos = (int)(std::find(order.begin(), order.end(), VD[t]) - order.begin());
    ssel.push_back(wordbit(pos));
  }
  if (ssel.size() != 2) return false;
  std::vector<int> rest_rho;  // rho positions of the remaining word bits, ascending word bit
  for (int wb = 0; wb < LB; ++wb) {
    if (std::find(ssel.begin(), ssel.end(), wb) != ssel.end()) continue;
    rest_rho.push_back(w == 8 ? wb - 1 : wb + nsub);
  }
  // swizzle: paper's construction, V = VS (source vector), writer A, reader B
  const int d = (int)T.size();
  auto loc = [&](int k) -> u64 {
    return u64(1) << (std::find(T.begin(), T.end(), k) - T.begin());
  };
  std::vector<u64> Al, Bl, Vl;
  for (int x : wr_lane) Al.push_back(loc(x));
  for (int x : rd_lane) Bl.push_back(loc(x));
  for (int x : VS) Vl.push_back(loc(x));
  SwizzleResult sw = optimal_swizzle(Al, Bl, Vl, d, w);
  std::vector<u64> Scols = sw.vect;
  Scols.insert(Scols.end(), sw.bank.begin(), sw.bank.end());
  Scols.insert(Scols.end(), sw.idx.begin(), sw.idx.end());
  auto Sinv = f2_right_inverse(Scols, d);
  const int lw = ilog2i(w);
  for (int k : T)
    if (sigma[k] + lw >= 31 || k + lw >= 31) return false;
  auto boff = [&](int k) -> uint32_t { return (uint32_t)f2_apply(Sinv, loc(k)) << lw; };
  SmemPlan& sp = P.sp;
  sp = SmemPlan{};
  sp.gw = g;
  sp.tile_bytes = w << d;
  sp.n_swaps = (int)swaps.size();
  for (size_t i = 0; i < swaps.size(); ++i) {
    sp.swap_a[i] = (int8_t)swaps[i].first;
    sp.swap_b[i] = (int8_t)swaps[i].second;
  }
  sp.gsel_a = (int8_t)ssel[0];
  sp.gsel_b = (int8_t)ssel[1];
  for (int b = 0; b < 5; ++b) {
    sp.ld_thr[b] = uint32_t(w) << sigma[wr_lane[b]];
    sp.st_thr[b] = uint32_t(w) << rd_lane[b];
    sp.sw_thr[b] = boff(wr_lane[b]);
    sp.sr_thr[b] = boff(rd_lane[b]);
  }
  for (int b = 0; b < g; ++b) {
    sp.ld_thr[5 + b] = uint32_t(w) << sigma[wr_warp[b]];
    sp.st_thr[5 + b] = uint32_t(w) << rd_warp[b];
    sp.sw_thr[5 + b] = boff(wr_warp[b]);
    sp.sr_thr[5 + b] = boff(rd_warp[b]);
  }
  const int nvec = 1 << (r - vb);
  if (nvec > LL_MAX_VEC || nvec > LL_MAX_GRAN) return false;
  for (int u = 0; u < nvec; ++u) {
    uint32_t lo = 0, wo = 0, ro = 0, so = 0;
    for (int q = 0; q < r - vb; ++q) {
      if ((u >> q) & 1) {
        lo += uint32_t(w) << sigma[wr_reg[vb + q]];   // chunk u: source offset
        wo ^= boff(wr_reg[vb + q]);                    //          smem offset
        ro ^= boff(rd_reg[vb + q]);                    // granule u read offset
        so += uint32_t(w) << order[rest_rho[q]];       // store vector u: dst offset
      }
    }
    sp.ld_vec[u] = lo;
    sp.sw_gran[u] = wo;
    sp.sr_gran[u] = ro;
    sp.st_vec[u] = so;
  }
  // tile map (dst order; top bits last)
  std::vector<int> O;
  for (int k = 0; k < n; ++k) if (!contains(T, k)) O.push_back(k);
  if ((int)O.size() > LL_MAX_OUTER) return false;
  TileMap& tm = sp.tile;
  tm.n_bits = (int)O.size();
  tm.n_tab = (tm.n_bits + LL_TAB_BITS - 1) / LL_TAB_BITS;
  for (int k = 0; k < tm.n_tab; ++k)
    for (int v = 0; v < (1 << LL_TAB_BITS); ++v) {
      int64_t so = 0, dof = 0;
      for (int q = 0; q < LL_TAB_BITS; ++q) {
        const int bit = k * LL_TAB_BITS + q;
        if (((v >> q) & 1) && bit < tm.n_bits) {
          so += int64_t(w) << sigma[O[bit]];
          dof += int64_t(w) << O[bit];
        }
      }
      tm.tab[k][v].src = so;
      tm.tab[k][v].dst = dof;
    }
  tm.batch_stride_src = int64_t(w) << P.nA;
  tm.batch_stride_dst = int64_t(w) << P.nB;
  tm.n_tiles = (int64_t(1) << O.size()) * P.batch;
  P.tile_bit_src.clear();
  P.tile_bit_dst.clear();
  for (int q = 0; q < tm.n_bits; ++q) {
    P.tile_bit_src.push_back(sigma[O[q]]);
    P.tile_bit_dst.push_back(O[q]);
  }
  P.nv = nvec;
  P.g = 16;
  P.tile_bits = d;
  P.r = r;
  P.gw = g;
  P.pred_wf_ld = lemma_wavefronts(sw, Al, w);
  P.pred_wf_st = lemma_wavefronts(sw, Bl, w);
  auto srcpos = [&](const std::vector<int>& v) {
    std::vector<int> o;
    for (int x : v) o.push_back(sigma[x]);
    return o;
  };
  js << ",\"tile_dst_bits\":" << ivec_json(T) << ",\"r\":" << r << ",\"group_warps_log2\":" << g
     << ",\"granule_bytes\":16,\"granule_dst_bits\":" << ivec_json(VS)
     << ",\"vectors_per_thread\":" << nvec << ",\"swaps\":[";
  for (size_t i = 0; i < swaps.size(); ++i)
    js << (i ? "," : "") << "[" << swaps[i].first << "," << swaps[i].second << "]";
  js << "],\"stg_sel\":" << ivec_json(ssel) << ",\"wr_reg_dst\":" << ivec_json(wr_reg)
     << ",\"wr_reg_src\":" << ivec_json(srcpos(wr_reg)) << ",\"wr_lane_dst\":" << ivec_json(wr_lane)
     << ",\"wr_lane_src\":" << ivec_json(srcpos(wr_lane)) << ",\"wr_warp_dst\":" << ivec_json(wr_warp)
     << ",\"rd_reg\":" << ivec_json(rd_reg) << ",\"rd_rho_after_swaps\":" << ivec_json(order)
     << ",\"rd_lane\":" << ivec_json(rd_lane) << ",\"rd_warp\":" << ivec_json(rd_warp)
     << ",\"S_vect\":" << vec_json(sw.vect) << ",\"S_bank\":" << vec_json(sw.bank)
     << ",\"S_idx\":" << vec_json(sw.idx) << ",\"H\":" << vec_json(sw.H) << ",\"C\":" << vec_json(sw.C)
     << ",\"unavoidable\":" << (sw.unavoidable ? "true" : "false")
     << ",\"pred_wavefronts_per_cp_async\":" << P.pred_wf_ld
     << ",\"pred_wavefronts_per_lds\":" << P.pred_wf_st << ",\"n_tiles\":" << tm.n_tiles
     << ",\"smem_bytes\":{\"sw_thr\":" << u32_json(sp.sw_thr, 5 + g) << ",\"sr_thr\":"
     << u32_json(sp.sr_thr, 5 + g) << ",\"sw_gran\":" << u32_json(sp.sw_gran, nvec)
     << ",\"sr_gran\":" << u32_json(sp.sr_gran, nvec) << "}";
  return true;
}

// TMA-fed variant of the shared-memory path (LL_PATH_SMEM_TMA).  The source
// tile is fetched by one cp.async.bulk.tensor per tile into a dense image
// (tile bits in ascending source order) permuted by a hardware swizzle mode
// m in {none, 32 B, 64 B, 128 B}: byte-address bits [4, 4+m) ^= [7, 7+m).
// That map is Def. 5 with vec = 16 bytes, per_phase = 1 and
// max_phase = 2^m on rows of 16 << m bytes (tests: test_oracle_swizzle.py),
// i.e. a fixed member of the family the paper's construction searches; the
// planner therefore cannot choose S, but chooses (a) the mode and (b) the
// reader's lanes so that the reader's 16-byte granules are conflict-free
// under it (wavefronts = 4 * 2^(rank(phase cols) - rank(bank projection)),
// the lemma P:1083-1089 for 16-byte granules), and among conflict-free
// choices the one with the longest coalesced destination runs.  The reader
// holds VS u VD in registers and permutes into destination vectors exactly
// as the cp.async path does.
bool plan_tma(ConvertPlan& P, const std::vector<u64>& X, std::ostringstream& js) {
  const int n = P.nB, w = P.w;
  if (P.nA != P.nB || n > 62 || w > 8) return false;
  std::vector<int> sigma(n), sinv(n, -1);
  for (int k = 0; k < n; ++k) {
    if (popcount64(X[k]) != 1) return false;
    sigma[k] = ctz64(X[k]);
    if (sinv[sigma[k]] >= 0) return false;
    sinv[sigma[k]] = k;
  }
  const int vb = ilog2i(16 / w);
  const int lw = ilog2i(w);
  if (n < vb + 5) return false;
  auto contains = [](const std::vector<int>& v, int x) {
    return std::find(v.begin(), v.end(), x) != v.end();
  };
  std::vector<int> VD, VS, CD, CS;
  for (int k = 0; k < vb; ++k) { VD.push_back(k); VS.push_back(sinv[k]); }
  const int cbits = std::max(0, ilog2i(std::max(16, planner_knob("tma_run_bytes", 256)) / 16));
  // destination run (knob tma_run_bytes_dst; the stores are merged in L2)
  const int cbits_d = planner_knob("tma_run_bytes_dst", 0) > 0
                          ? std::min(cbits, ilog2i(std::max(16, planner_knob("tma_run_bytes_dst", 0)) / 16))
                          : cbits;
  for (int k = vb; k < std::min(n, vb + cbits_d); ++k) CD.push_back(k);
  for (int k = vb; k < std::min(n, vb + cbits); ++k) CS.push_back(sinv[k]);
  const int r_max = ilog2i(std::max(16, std::min(128, planner_knob("thread_bytes_max", 128))) / w);
  const int r_pref = std::min(r_max, ilog2i(std::max(16, planner_knob("tma_thread_bytes", 64)) / w));
  std::vector<int> need = VS;
  for (int x : VD) if (!contains(need, x)) need.push_back(x);
  if ((int)need.size() > r_max || (int)need.size() + 5 > n) return false;
  int r = std::min(std::max((int)need.size(), r_pref), std::min(r_max, n - 5));
  // tile: the vectors and coalescing runs of both sides, then the lowest
  // destination bits; at least tma_tile_bytes (several KB in flight per TMA)
  const int tile_min = ilog2i(std::max(1024, planner_knob("tma_tile_bytes", 8192)) / w);
  std::vector<int> T = VD;
  for (auto* s : {&VS, &CD, &CS, &need})
    for (int x : *s) if (!contains(T, x)) T.push_back(x);
  for (int k = 0; (int)T.size() < std::max(r + 5, std::min(n, tile_min)) && k < n; ++k)
    if (!contains(T, k)) T.push_back(k);
  int g = (int)T.size() - r - 5;
  if (g > 3) {
    int r2 = std::min(r_max, (int)T.size() - 5 - 3);
    if (r2 > r) { r = r2; g = (int)T.size() - r - 5; }
  }
  if (g < 0 || g > 3) return false;
  std::sort(T.begin(), T.end());
  const int d = (int)T.size();
  // dense image: rank of the source bit among the tile's source bits
  std::vector<int> Ts;
  for (int k : T) Ts.push_back(sigma[k]);
  std::sort(Ts.begin(), Ts.end());
  auto dense = [&](int k) -> uint32_t {
    return uint32_t(w) << (std::find(Ts.begin(), Ts.end(), sigma[k]) - Ts.begin());
  };
  for (int k : T)
    if (sigma[k] + lw >= 40 || d + lw > 20) return false;
  // reader registers: VS (granule order), VD \ VS, extra (highest dst, not CD)
  std::vector<int> rd_reg = VS;
  for (int x : VD) if (!contains(rd_reg, x)) rd_reg.push_back(x);
  {
    std::vector<int> cand;
    for (int x : T) if (!contains(rd_reg, x) && !contains(CD, x)) cand.push_back(x);
    std::sort(cand.begin(), cand.end(), [](int a, int b) { return a > b; });
    for (int x : cand) { if ((int)rd_reg.size() == r) break; rd_reg.push_back(x); }
    if ((int)rd_reg.size() != r) return false;
  }
  // TMA box dims for swizzle mode m: runs of consecutive source bits; the
  // first run is split at the swizzle span (16 << m bytes), every box dim is
  // at most 256 elements; <= 5 dims
  auto make_desc = [&](int m, TmaDesc& td) -> bool {
    td = TmaDesc{};
    td.swizzle = m;
    std::vector<std::pair<int, int>> runs;  // (first source bit, length)
    for (int b : Ts) {
      if (!runs.empty() && runs.back().first + runs.back().second == b) ++runs.back().second;
      else runs.push_back({b, 1});
    }
    if (runs.empty() || runs[0].first != 0) return false;
    const int span_bits = m ? ilog2i((16 << m) / w) : 8;
    std::vector<std::pair<int, int>> dims;  // (shift, box bits)
    for (size_t i = 0; i < runs.size(); ++i) {
      int a = runs[i].first, len = runs[i].second;
      if (i == 0 && m) {
        if (len < span_bits) return false;
        dims.push_back({a, span_bits});
        a += span_bits;
        len -= span_bits;
      }
      while (len > 0) {
        const int piece = std::min(len, 8);
        dims.push_back({a, piece});
        a += piece;
        len -= piece;
      }
    }
    if (dims.size() > 5) return false;
    if (!m && dims[0].second > 8) return false;
    td.ndim = (int)dims.size();
    for (int i = 0; i < td.ndim; ++i) {
      td.shift[i] = dims[i].first;
      td.box_bits[i] = dims[i].second;
      td.size_bits[i] = i + 1 < td.ndim ? dims[i + 1].first - dims[i].first : 0;
      if (i > 0 && (dims[i].first + lw) < 4) return false;  // strides: multiples of 16 B
    }
    return true;
  };
  auto swz = [](uint32_t a, int m) -> uint32_t {
    return m ? a ^ (((a >> 7) & ((1u << m) - 1)) << 4) : a;
  };
  struct Choice {
    int m = -1, wf = 1 << 30, run = -1;
    std::vector<int> lane, warp;
    TmaDesc td{};
  } best;
  const int force = planner_knob("tma_force_swizzle", -1);
  for (int m = 0; m <= 3; ++m) {
    if (force >= 0 && m != force) continue;
    Choice c;
    c.m = m;
    if (!make_desc(m, c.td)) continue;
    auto addr = [&](int k) { return swz(dense(k), m); };
    std::vector<int> cand;
    for (int x : T) if (!contains(rd_reg, x)) cand.push_back(x);
    std::sort(cand.begin(), cand.end());
    // phase lanes (lane bits 0-2 of a 16-byte access): independent bank
    // projections (address bits 4-6), lowest destination bits first
    std::vector<int> phase;
    std::vector<u64> proj;
    for (int x : cand) {
      if (phase.size() == 3) break;
      std::vector<u64> p2 = proj;
      p2.push_back((addr(x) >> 4) & 7u);
      if (f2_rank(p2) > f2_rank(proj)) { phase.push_back(x); proj = p2; }
    }
    for (int x : cand) {
      if (phase.size() == 3) break;
      if (!contains(phase, x)) phase.push_back(x);
    }
    c.lane = phase;
    for (int x : cand) {
      if (c.lane.size() == 5) break;
      if (!contains(c.lane, x)) c.lane.push_back(x);
    }
    for (int x : cand) if (!contains(c.lane, x)) c.warp.push_back(x);
    std::vector<u64> pc, pp;
    for (int i = 0; i < 3; ++i) {
      pc.push_back(addr(c.lane[i]));
      pp.push_back((addr(c.lane[i]) >> 4) & 7u);
    }
    c.wf = 4 << (f2_rank(pc) - f2_rank(pp));
    // destination run of one store instruction: 16 B x 2^(lane bits that
    // extend the vector contiguously, in lane order)
    std::vector<int> sl = c.lane;
    int run = 0;
    for (int q = 0;; ++q) {
      if (!contains(sl, vb + q)) break;
      ++run;
    }
    c.run = run;
    if (c.wf < best.wf || (c.wf == best.wf && c.run > best.run)) best = c;
  }
  if (best.m < 0 || (int)best.warp.size() != g) return false;
  const int m = best.m;
  std::vector<int> rd_lane = best.lane, rd_warp = best.warp;
  // reader sub-word swaps / store selection: as in plan_async
  const int nsub = w >= 4 ? 0 : ilog2i(4 / w);
  std::vector<int> order = rd_reg;
  std::vector<std::pair<int, int>> swaps;
  for (int t = 0; t < nsub; ++t) {
    int s = (int)(std::find(order.begin(), order.end(), VD[t]) - order.begin());
    if (s != t) { swaps.push_back({t, s}); std::swap(order[t], order[s]); }
  }
  if ((int)swaps.size() > LL_MAX_SWAPS) return false;
  auto wordbit = [&](int rho) { return w == 8 ? rho + 1 : rho - nsub; };
  const int LB = w == 8 ? r + 1 : r - nsub;
  std::vector<int> ssel;
  if (w == 8) ssel.push_back(0);
  for (int t = (w == 8 ? 0 : nsub); t < vb; ++t) {
    int pos = (int)(std::find(order.begin(), order.end(), VD[t]) - order.begin());
    ssel.push_back(wordbit(pos));
  }
  if (ssel.size() != 2) return false;
  std::vector<int> rest_rho;
  for (int wb = 0; wb < LB; ++wb) {
    if (std::find(ssel.begin(), ssel.end(), wb) != ssel.end()) continue;
    rest_rho.push_back(w == 8 ? wb - 1 : wb + nsub);
  }
  auto boff = [&](int k) -> uint32_t { return swz(dense(k), m); };
  SmemPlan& sp = P.sp;
  sp = SmemPlan{};
  sp.gw = g;
  sp.tile_bytes = w << d;
  sp.n_swaps = (int)swaps.size();
  for (size_t i = 0; i < swaps.size(); ++i) {
    sp.swap_a[i] = (int8_t)swaps[i].first;
    sp.swap_b[i] = (int8_t)swaps[i].second;
  }
  sp.gsel_a = (int8_t)ssel[0];
  sp.gsel_b = (int8_t)ssel[1];
  for (int b = 0; b < 5 + g; ++b) {
    const int k = b < 5 ? rd_lane[b] : rd_warp[b - 5];
    sp.st_thr[b] = uint32_t(w) << k;
    sp.sr_thr[b] = boff(k);
  }
  const int nvec = 1 << (r - vb);
  if (nvec > LL_MAX_VEC || nvec > LL_MAX_GRAN) return false;
  for (int u = 0; u < nvec; ++u) {
    uint32_t ro = 0, so = 0;
    for (int q = 0; q < r - vb; ++q) {
      if ((u >> q) & 1) {
        ro ^= boff(rd_reg[vb + q]);
        so += uint32_t(w) << order[rest_rho[q]];
      }
    }
    sp.sr_gran[u] = ro;
    sp.st_vec[u] = so;
  }
  std::vector<int> O;
  for (int k = 0; k < n; ++k) if (!contains(T, k)) O.push_back(k);
  if ((int)O.size() > LL_MAX_OUTER) return false;
  TileMap& tm = sp.tile;
  tm.n_bits = (int)O.size();
  tm.n_tab = (tm.n_bits + LL_TAB_BITS - 1) / LL_TAB_BITS;
  for (int k = 0; k < tm.n_tab; ++k)
    for (int v = 0; v < (1 << LL_TAB_BITS); ++v) {
      int64_t so = 0, dof = 0;
      for (int q = 0; q < LL_TAB_BITS; ++q) {
        const int bit = k * LL_TAB_BITS + q;
        if (((v >> q) & 1) && bit < tm.n_bits) {
          so += int64_t(w) << sigma[O[bit]];
          dof += int64_t(w) << O[bit];
        }
      }
      tm.tab[k][v].src = so;
      tm.tab[k][v].dst = dof;
    }
  tm.batch_stride_src = int64_t(w) << P.nA;
  tm.batch_stride_dst = int64_t(w) << P.nB;
  tm.n_tiles = (int64_t(1) << O.size()) * P.batch;
  P.tile_bit_src.clear();
  P.tile_bit_dst.clear();
  for (int q = 0; q < tm.n_bits; ++q) {
    P.tile_bit_src.push_back(sigma[O[q]]);
    P.tile_bit_dst.push_back(O[q]);
  }
  P.td = best.td;
  P.nv = nvec;
  P.g = 16;
  P.tile_bits = d;
  P.r = r;
  P.gw = g;
  P.pred_wf_ld = 0;  // the TMA write has no bank conflicts to predict
  P.pred_wf_st = best.wf;
  std::vector<int> shifts, boxes;
  for (int i = 0; i < P.td.ndim; ++i) {
    shifts.push_back(P.td.shift[i]);
    boxes.push_back(P.td.box_bits[i]);
  }
  static const char* mode_names[] = {"none", "32B", "64B", "128B"};
  js << ",\"tile_dst_bits\":" << ivec_json(T) << ",\"r\":" << r << ",\"group_warps_log2\":" << g
     << ",\"granule_bytes\":16,\"granule_dst_bits\":" << ivec_json(VS)
     << ",\"vectors_per_thread\":" << nvec << ",\"swaps\":[";
  for (size_t i = 0; i < swaps.size(); ++i)
    js << (i ? "," : "") << "[" << swaps[i].first << "," << swaps[i].second << "]";
  js << "],\"stg_sel\":" << ivec_json(ssel) << ",\"rd_reg\":" << ivec_json(rd_reg)
     << ",\"rd_rho_after_swaps\":" << ivec_json(order) << ",\"rd_lane\":" << ivec_json(rd_lane)
     << ",\"rd_warp\":" << ivec_json(rd_warp) << ",\"tma\":{\"swizzle\":\"" << mode_names[m]
     << "\",\"ndim\":" << P.td.ndim << ",\"dim_src_shift\":" << ivec_json(shifts)
     << ",\"box_bits\":" << ivec_json(boxes) << ",\"store_run_bytes\":" << (16 << best.run)
     << "},\"pred_wavefronts_per_lds\":" << P.pred_wf_st << ",\"n_tiles\":" << tm.n_tiles
     << ",\"smem_bytes\":{\"sr_thr\":" << u32_json(sp.sr_thr, 5 + g)
     << ",\"sr_gran\":" << u32_json(sp.sr_gran, nvec) << "}";
  return true;
}

// TMA load + TMA store variant (LL_PATH_SMEM_TMA_STORE).  As plan_tma, but
// the readers write their destination vectors into a second shared-memory
// image (the destination tile, dense in destination-bit order, hardware
// swizzle md) that one cp.async.bulk.tensor store sends to HBM.  The
// readers' lanes are then free of global coalescing and must make BOTH the
// 16-byte reads of the source image and the 16-byte writes of the
// destination image conflict-free; when no set of single tile bits does,
// XOR combinations are used (a lane bit then moves along a "diagonal" of the
// tile -- the paper's swizzling idea applied to the thread layout).
bool plan_tma_store(ConvertPlan& P, const std::vector<u64>& X, std::ostringstream& js) {
  const int n = P.nB, w = P.w;
  if (P.nA != P.nB || n > 62 || w > 8) return false;
  std::vector<int> sigma(n), sinv(n, -1);
  for (int k = 0; k < n; ++k) {
    if (popcount64(X[k]) != 1) return false;
    sigma[k] = ctz64(X[k]);
    if (sinv[sigma[k]] >= 0) return false;
    sinv[sigma[k]] = k;
  }
  const int vb = ilog2i(16 / w);
  const int lw = ilog2i(w);
  if (n < vb + 5) return false;
  auto contains = [](const std::vector<int>& v, int x) {
    return std::find(v.begin(), v.end(), x) != v.end();
  };
  std::vector<int> VD, VS, CD, CS;
  for (int k = 0; k < vb; ++k) { VD.push_back(k); VS.push_back(sinv[k]); }
  const int cbits = std::max(0, ilog2i(std::max(16, planner_knob("tma_run_bytes", 256)) / 16));
  // destination run (knob tma_run_bytes_dst; the stores are merged in L2)
  const int cbits_d = planner_knob("tma_run_bytes_dst", 0) > 0
                          ? std::min(cbits, ilog2i(std::max(16, planner_knob("tma_run_bytes_dst", 0)) / 16))
                          : cbits;
  for (int k = vb; k < std::min(n, vb + cbits_d); ++k) CD.push_back(k);
  for (int k = vb; k < std::min(n, vb + cbits); ++k) CS.push_back(sinv[k]);
  const int r_max = ilog2i(std::max(16, std::min(128, planner_knob("thread_bytes_max", 128))) / w);
  const int r_pref = std::min(r_max, ilog2i(std::max(16, planner_knob("tma_thread_bytes", 64)) / w));
  std::vector<int> need = VS;
  for (int x : VD) if (!contains(need, x)) need.push_back(x);
  if ((int)need.size() > r_max || (int)need.size() + 5 > n) return false;
  int r = std::min(std::max((int)need.size(), r_pref), std::min(r_max, n - 5));
  const int tile_min = ilog2i(std::max(1024, planner_knob("tma_tile_bytes", 8192)) / w);
  std::vector<int> T = VD;
  for (auto* s : {&VS, &CD, &CS, &need})
    for (int x : *s) if (!contains(T, x)) T.push_back(x);
  for (int k = 0; (int)T.size() < std::max(r + 5, std::min(n, tile_min)) && k < n; ++k)
    if (!contains(T, k)) T.push_back(k);
  int g = (int)T.size() - r - 5;
  if (g > 3) {
    int r2 = std::min(r_max, (int)T.size() - 5 - 3);
    if (r2 > r) { r = r2; g = (int)T.size() - r - 5; }
  }
  if (g < 0 || g > 3) return false;
  std::sort(T.begin(), T.end());
  const int d = (int)T.size();
  if (d + lw > 20) return false;
  std::vector<int> Ts;
  for (int k : T) Ts.push_back(sigma[k]);
  std::sort(Ts.begin(), Ts.end());
  // dense images (byte offsets before the swizzle), linear in tile vectors
  auto dense_s = [&](u64 v) -> uint32_t {
    uint32_t o = 0;
    for (int k = 0; k < n; ++k)
      if ((v >> k) & 1) o ^= uint32_t(w) << (std::find(Ts.begin(), Ts.end(), sigma[k]) - Ts.begin());
    return o;
  };
  auto dense_d = [&](u64 v) -> uint32_t {
    uint32_t o = 0;
    for (int k = 0; k < n; ++k)
      if ((v >> k) & 1) o ^= uint32_t(w) << (std::find(T.begin(), T.end(), k) - T.begin());
    return o;
  };
  auto swz = [](uint32_t a, int m) -> uint32_t {
    return m ? a ^ (((a >> 7) & ((1u << m) - 1)) << 4) : a;
  };
  std::vector<int> rd_reg = VS;
  for (int x : VD) if (!contains(rd_reg, x)) rd_reg.push_back(x);
  {
    std::vector<int> cand;
    for (int x : T) if (!contains(rd_reg, x) && !contains(CD, x)) cand.push_back(x);
    std::sort(cand.begin(), cand.end(), [](int a, int b) { return a > b; });
    for (int x : cand) { if ((int)rd_reg.size() == r) break; rd_reg.push_back(x); }
    if ((int)rd_reg.size() != r) return false;
  }
  auto make_desc = [&](const std::vector<int>& bits, int m, TmaDesc& td) -> bool {
    td = TmaDesc{};
    td.swizzle = m;
    std::vector<std::pair<int, int>> runs;
    for (int b : bits) {
      if (!runs.empty() && runs.back().first + runs.back().second == b) ++runs.back().second;
      else runs.push_back({b, 1});
    }
    if (runs.empty() || runs[0].first != 0) return false;
    const int span_bits = m ? ilog2i((16 << m) / w) : 8;
    std::vector<std::pair<int, int>> dims;
    for (size_t i = 0; i < runs.size(); ++i) {
      int a = runs[i].first, len = runs[i].second;
      if (i == 0 && m) {
        if (len < span_bits) return false;
        dims.push_back({a, span_bits});
        a += span_bits;
        len -= span_bits;
      }
      while (len > 0) {
        const int piece = std::min(len, 8);
        dims.push_back({a, piece});
        a += piece;
        len -= piece;
      }
    }
    if (dims.size() > 5) return false;
    td.ndim = (int)dims.size();
    for (int i = 0; i < td.ndim; ++i) {
      td.shift[i] = dims[i].first;
      td.box_bits[i] = dims[i].second;
      td.size_bits[i] = i + 1 < td.ndim ? dims[i + 1].first - dims[i].first : 0;
      if (i > 0 && (dims[i].first + lw) < 4) return false;
    }
    return true;
  };
  // candidate lane vectors: single non-register tile bits (lowest
  // destination bit first), then their pairwise XORs
  std::vector<u64> singles, cands;
  for (int x : T) if (!contains(rd_reg, x)) singles.push_back(u64(1) << x);
  cands = singles;
  for (size_t i = 0; i < singles.size(); ++i)
    for (size_t j = i + 1; j < singles.size(); ++j) cands.push_back(singles[i] | singles[j]);
  struct Choice {
    int ms = -1, md = -1, wf = 1 << 30, diag = 0;
    std::vector<u64> thr;   // 5 lanes then g warps
    TmaDesc tds{}, tdd{};
  } best;
  for (int ms = 0; ms <= 3; ++ms) {
    for (int md = 0; md <= 3; ++md) {
      Choice c;
      c.ms = ms;
      c.md = md;
      if (!make_desc(Ts, ms, c.tds) || !make_desc(T, md, c.tdd)) continue;
      auto ps = [&](u64 v) -> u64 { return (swz(dense_s(v), ms) >> 4) & 7u; };
      auto pd = [&](u64 v) -> u64 { return (swz(dense_d(v), md) >> 4) & 7u; };
      std::vector<u64> phase, prs, prd;
      F2Basis span;
      for (u64 v : cands) {
        if (phase.size() == 3) break;
        if (span.in_span(v)) continue;
        std::vector<u64> a = prs, b = prd;
        a.push_back(ps(v));
        b.push_back(pd(v));
        if (f2_rank(a) > f2_rank(prs) && f2_rank(b) > f2_rank(prd)) {
          phase.push_back(v);
          prs = a;
          prd = b;
          span.add(v);
        }
      }
      for (u64 v : singles) {
        if (phase.size() == 3) break;
        if (span.add(v)) phase.push_back(v);
      }
      c.thr = phase;
      for (u64 v : singles)
        if (span.add(v)) c.thr.push_back(v);
      if ((int)c.thr.size() != 5 + g) continue;
      std::vector<u64> as, ad, qs, qd;
      for (int i = 0; i < 3; ++i) {
        as.push_back(swz(dense_s(c.thr[i]), ms));
        ad.push_back(swz(dense_d(c.thr[i]), md));
        qs.push_back(ps(c.thr[i]));
        qd.push_back(pd(c.thr[i]));
      }
      c.wf = (4 << (f2_rank(as) - f2_rank(qs))) + (4 << (f2_rank(ad) - f2_rank(qd)));
      for (u64 v : c.thr) c.diag += popcount64(v) > 1;
      if (c.wf < best.wf || (c.wf == best.wf && c.diag < best.diag)) best = c;
    }
  }
  if (best.ms < 0) return false;
  const int nsub = w >= 4 ? 0 : ilog2i(4 / w);
  std::vector<int> order = rd_reg;
  std::vector<std::pair<int, int>> swaps;
  for (int t = 0; t < nsub; ++t) {
    int s = (int)(std::find(order.begin(), order.end(), VD[t]) - order.begin());
    if (s != t) { swaps.push_back({t, s}); std::swap(order[t], order[s]); }
  }
  if ((int)swaps.size() > LL_MAX_SWAPS) return false;
  auto wordbit = [&](int rho) { return w == 8 ? rho + 1 : rho - nsub; };
  const int LB = w == 8 ? r + 1 : r - nsub;
  std::vector<int> ssel;
  if (w == 8) ssel.push_back(0);
  for (int t = (w == 8 ? 0 : nsub); t < vb; ++t) {
    int pos = (int)(std::find(order.begin(), order.end(), VD[t]) - order.begin());
    ssel.push_back(wordbit(pos));
  }
  if (ssel.size() != 2) return false;
  std::vector<int> rest_rho;
  for (int wb = 0; wb < LB; ++wb) {
    if (std::find(ssel.begin(), ssel.end(), wb) != ssel.end()) continue;
    rest_rho.push_back(w == 8 ? wb - 1 : wb + nsub);
  }
  auto roff = [&](u64 v) -> uint32_t { return swz(dense_s(v), best.ms); };
  auto woff = [&](u64 v) -> uint32_t { return swz(dense_d(v), best.md); };
  SmemPlan& sp = P.sp;
  sp = SmemPlan{};
  sp.gw = g;
  sp.tile_bytes = w << d;
  sp.n_swaps = (int)swaps.size();
  for (size_t i = 0; i < swaps.size(); ++i) {
    sp.swap_a[i] = (int8_t)swaps[i].first;
    sp.swap_b[i] = (int8_t)swaps[i].second;
  }
  sp.gsel_a = (int8_t)ssel[0];
  sp.gsel_b = (int8_t)ssel[1];
  for (int b = 0; b < 5 + g; ++b) {
    sp.sr_thr[b] = roff(best.thr[b]);
    sp.sw_thr[b] = woff(best.thr[b]);
  }
  const int nvec = 1 << (r - vb);
  if (nvec > LL_MAX_VEC || nvec > LL_MAX_GRAN) return false;
  for (int u = 0; u < nvec; ++u) {
    uint32_t ro = 0, wo = 0;
    for (int q = 0; q < r - vb; ++q) {
      if ((u >> q) & 1) {
        ro ^= roff(u64(1) << rd_reg[vb + q]);            // source granule u
        wo ^= woff(u64(1) << order[rest_rho[q]]);        // destination vector u
      }
    }
    sp.sr_gran[u] = ro;
    sp.sw_gran[u] = wo;
  }
  std::vector<int> O;
  for (int k = 0; k < n; ++k) if (!contains(T, k)) O.push_back(k);
  if ((int)O.size() > LL_MAX_OUTER) return false;
  TileMap& tm = sp.tile;
  tm.n_bits = (int)O.size();
  tm.n_tab = (tm.n_bits + LL_TAB_BITS - 1) / LL_TAB_BITS;
  for (int k = 0; k < tm.n_tab; ++k)
    for (int v = 0; v < (1 << LL_TAB_BITS); ++v) {
      int64_t so = 0, dof = 0;
      for (int q = 0; q < LL_TAB_BITS; ++q) {
        const int bit = k * LL_TAB_BITS + q;
        if (((v >> q) & 1) && bit < tm.n_bits) {
          so += int64_t(w) << sigma[O[bit]];
          dof += int64_t(w) << O[bit];
        }
      }
      tm.tab[k][v].src = so;
      tm.tab[k][v].dst = dof;
    }
  tm.batch_stride_src = int64_t(w) << P.nA;
  tm.batch_stride_dst = int64_t(w) << P.nB;
  tm.n_tiles = (int64_t(1) << O.size()) * P.batch;
  P.tile_bit_src.clear();
  P.tile_bit_dst.clear();
  for (int q = 0; q < tm.n_bits; ++q) {
    P.tile_bit_src.push_back(sigma[O[q]]);
    P.tile_bit_dst.push_back(O[q]);
  }
  P.td = best.tds;
  P.td_dst = best.tdd;
  P.nv = nvec;
  P.g = 16;
  P.tile_bits = d;
  P.r = r;
  P.gw = g;
  std::vector<u64> as, ad, qs, qd;
  for (int i = 0; i < 3; ++i) {
    as.push_back(roff(best.thr[i]));
    ad.push_back(woff(best.thr[i]));
    qs.push_back((roff(best.thr[i]) >> 4) & 7u);
    qd.push_back((woff(best.thr[i]) >> 4) & 7u);
  }
  P.pred_wf_st = 4 << (f2_rank(as) - f2_rank(qs));   // LDS of the source image
  P.pred_wf_ld = 4 << (f2_rank(ad) - f2_rank(qd));   // STS of the destination image
  static const char* mode_names[] = {"none", "32B", "64B", "128B"};
  auto td_json = [&](const TmaDesc& t) {
    std::vector<int> sh, bx;
    for (int i = 0; i < t.ndim; ++i) { sh.push_back(t.shift[i]); bx.push_back(t.box_bits[i]); }
    std::ostringstream o;
    o << "{\"swizzle\":\"" << mode_names[t.swizzle] << "\",\"ndim\":" << t.ndim
      << ",\"dim_shift\":" << ivec_json(sh) << ",\"box_bits\":" << ivec_json(bx) << "}";
    return o.str();
  };
  js << ",\"tile_dst_bits\":" << ivec_json(T) << ",\"r\":" << r << ",\"group_warps_log2\":" << g
     << ",\"granule_bytes\":16,\"vectors_per_thread\":" << nvec << ",\"rd_reg\":" << ivec_json(rd_reg)
     << ",\"thread_vecs_dst_bits\":" << vec_json(best.thr) << ",\"diagonal_lanes\":" << best.diag
     << ",\"tma\":{\"src\":" << td_json(best.tds) << ",\"dst\":" << td_json(best.tdd) << "}"
     << ",\"pred_wavefronts_per_lds\":" << P.pred_wf_st << ",\"pred_wavefronts_per_sts\":" << P.pred_wf_ld
     << ",\"n_tiles\":" << tm.n_tiles << ",\"smem_bytes\":{\"sr_thr\":" << u32_json(sp.sr_thr, 5 + g)
     << ",\"sw_thr\":" << u32_json(sp.sw_thr, 5 + g) << ",\"sr_gran\":" << u32_json(sp.sr_gran, nvec)
     << ",\"sw_gran\":" << u32_json(sp.sw_gran, nvec) << "}";
  return true;
}

}  // namespace detail
}  // namespace ll
