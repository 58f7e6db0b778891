// core.cpp -- F2 algebra and labeled layouts (host).  See core.hpp.
#include "core.hpp"

#include <algorithm>
#include <map>

namespace ll {

std::vector<u64> f2_right_inverse(const std::vector<u64>& cols, int m) {
  const int n = (int)cols.size();
  if (m > 63 || n > 63) throw Error(LL_ERR_ARG, "right inverse: more than 63 bits");
  // rows of M as n-bit ints, augmented with I_m
  std::vector<u64> rows(m, 0), aug(m, 0);
  for (int r = 0; r < m; ++r) {
    aug[r] = u64(1) << r;
    for (int j = 0; j < n; ++j)
      if ((cols[j] >> r) & 1) rows[r] |= u64(1) << j;
  }
  std::vector<int> pivcol;
  int p = 0;
  for (int j = 0; j < n && p < m; ++j) {
    int sel = -1;
    for (int r = p; r < m; ++r)
      if ((rows[r] >> j) & 1) { sel = r; break; }
    if (sel < 0) continue;
    std::swap(rows[p], rows[sel]);
    std::swap(aug[p], aug[sel]);
    for (int q = 0; q < m; ++q)
      if (q != p && ((rows[q] >> j) & 1)) { rows[q] ^= rows[p]; aug[q] ^= aug[p]; }
    pivcol.push_back(j);
    ++p;
  }
  if (p < m)
    throw Error(LL_ERR_NOT_SURJECTIVE, "layout is not surjective (rank " + std::to_string(p) +
                                           " < " + std::to_string(m) + " output bits)");
  std::vector<u64> x(m, 0);
  for (int c = 0; c < m; ++c)
    for (int i = 0; i < (int)pivcol.size(); ++i)
      if ((aug[i] >> c) & 1) x[c] |= u64(1) << pivcol[i];
  return x;
}

std::vector<u64> f2_complete(const std::vector<u64>& vecs, int d) {
  F2Basis b;
  for (u64 v : vecs)
    if (!b.add(v)) throw Error(LL_ERR_ARG, "basis completion: dependent input");
  std::vector<u64> out;
  for (int k = 0; k < d && b.n < d; ++k)
    if (b.add(u64(1) << k)) out.push_back(u64(1) << k);
  return out;
}

int Layout::in_bits() const {
  int s = 0;
  for (auto& d : in) s += d.bits;
  return s;
}
int Layout::out_bits() const {
  int s = 0;
  for (auto& d : out) s += d.bits;
  return s;
}
int Layout::in_offset(const std::string& name) const {
  int off = 0;
  for (auto& d : in) {
    if (d.name == name) return off;
    off += d.bits;
  }
  return -1;
}
int Layout::in_size(const std::string& name) const {
  for (auto& d : in)
    if (d.name == name) return d.bits;
  return 0;
}
int Layout::out_index(const std::string& name) const {
  for (size_t i = 0; i < out.size(); ++i)
    if (out[i].name == name) return (int)i;
  return -1;
}
int Layout::out_shift(int d) const {
  int s = 0;
  for (size_t i = d + 1; i < out.size(); ++i) s += out[i].bits;
  return s;
}
std::vector<u64> Layout::sub(const std::string& name) const {
  int off = in_offset(name);
  if (off < 0) return {};
  return std::vector<u64>(cols.begin() + off, cols.begin() + off + in_size(name));
}
u64 Layout::flatten(const std::vector<int64_t>& c) const {
  u64 x = 0;
  for (size_t d = 0; d < out.size(); ++d) x |= u64(c[d]) << out_shift((int)d);
  return x;
}
std::vector<int64_t> Layout::unflatten(u64 x) const {
  std::vector<int64_t> c(out.size());
  for (size_t d = 0; d < out.size(); ++d)
    c[d] = (int64_t)((x >> out_shift((int)d)) & ((u64(1) << out[d].bits) - 1));
  return c;
}
bool Layout::surjective() const { return f2_rank(cols) == out_bits(); }
bool Layout::distributed() const {
  // Definition "Distributed Layout"
  for (auto& d : in)
    if (d.name != "reg" && d.name != "lane" && d.name != "thread" && d.name != "warp" &&
        d.name != "block")
      return false;
  std::vector<u64> nz;
  for (u64 c : cols) {
    if (popcount64(c) > 1) return false;
    if (c) nz.push_back(c);
  }
  std::sort(nz.begin(), nz.end());
  if (std::adjacent_find(nz.begin(), nz.end()) != nz.end()) return false;
  return surjective();
}
bool Layout::memory() const {
  // Definition "Memory Layout"
  if (in.size() != 1 || in[0].name != "offset") return false;
  if ((int)cols.size() != out_bits() || f2_rank(cols) != out_bits()) return false;
  for (u64 c : cols)
    if (popcount64(c) < 1 || popcount64(c) > 2) return false;
  return true;
}
u64 Layout::hash() const {
  u64 h = 0xcbf29ce484222325ull;
  auto mix = [&](u64 v) {
    h ^= v;
    h *= 0x100000001b3ull;
    h ^= h >> 29;
  };
  for (auto& d : in) {
    for (char ch : d.name) mix((u64)(unsigned char)ch);
    mix(0x100 + d.bits);
  }
  mix(0xabcdef);
  for (auto& d : out) {
    for (char ch : d.name) mix((u64)(unsigned char)ch);
    mix(0x200 + d.bits);
  }
  for (u64 c : cols) mix(c);
  return h;
}
bool Layout::same_tensor(const Layout& o) const {
  if (out.size() != o.out.size()) return false;
  for (size_t i = 0; i < out.size(); ++i)
    if (out[i].name != o.out[i].name || out[i].bits != o.out[i].bits) return false;
  return true;
}

Layout compose(const Layout& outer, const Layout& inner) {
  // Definition "Composition": label-wise product, matched by name.
  if (outer.in.size() != inner.out.size())
    throw Error(LL_ERR_LABEL, "compose: inner has " + std::to_string(inner.out.size()) +
                                  " output dims, outer has " + std::to_string(outer.in.size()) +
                                  " input dims");
  for (auto& d : inner.out)
    if (outer.in_size(d.name) != d.bits || outer.in_offset(d.name) < 0)
      throw Error(LL_ERR_LABEL, "compose: inner output dim '" + d.name +
                                    "' does not match an outer input dim of the same size");
  Layout r;
  r.in = inner.in;
  r.out = outer.out;
  for (u64 c : inner.cols) {
    auto coords = inner.unflatten(c);
    u64 h = 0;
    for (size_t d = 0; d < inner.out.size(); ++d)
      h |= u64(coords[d]) << outer.in_offset(inner.out[d].name);
    r.cols.push_back(f2_apply(outer.cols, h));
  }
  return r;
}

Layout right_inverse(const Layout& l) {
  Layout r;
  r.cols = f2_right_inverse(l.cols, l.out_bits());
  r.in.assign(l.out.rbegin(), l.out.rend());
  r.out.assign(l.in.rbegin(), l.in.rend());
  return r;
}

Layout product(const Layout& a, const Layout& b) {
  // Definition "Product": label-wise block diagonal, a low / b high.
  Layout r;
  r.in = a.in;
  for (auto& d : b.in) {
    bool found = false;
    for (auto& e : r.in)
      if (e.name == d.name) { e.bits += d.bits; found = true; }
    if (!found) r.in.push_back(d);
  }
  r.out = a.out;
  for (auto& d : b.out) {
    bool found = false;
    for (auto& e : r.out)
      if (e.name == d.name) { e.bits += d.bits; found = true; }
    if (!found) r.out.push_back(d);
  }
  if (r.in_bits() > 62 || r.out_bits() > 62) throw Error(LL_ERR_ARG, "product: too many bits");
  auto embed = [&](const Layout& src, u64 c, bool high) {
    auto coords = src.unflatten(c);
    std::vector<int64_t> rc(r.out.size(), 0);
    for (size_t d = 0; d < src.out.size(); ++d) {
      int idx = r.out_index(src.out[d].name);
      int shift = high ? std::max(0, a.out_index(src.out[d].name) >= 0
                                         ? a.out[a.out_index(src.out[d].name)].bits
                                         : 0)
                       : 0;
      rc[idx] = coords[d] << shift;
    }
    return r.flatten(rc);
  };
  for (auto& d : r.in) {
    auto av = a.sub(d.name), bv = b.sub(d.name);
    for (u64 c : av) r.cols.push_back(embed(a, c, false));
    for (u64 c : bv) r.cols.push_back(embed(b, c, true));
  }
  return r;
}

Layout left_divide(const Layout& m, const Layout& m1) {
  // Definition "Left Division", label-wise: m = [[m1, 0], [0, m2]]
  // -- for every input label the first m1.in_size bits are m1's columns
  // (embedded at the low bits of each output dim) and the other bits have
  // zero m1 block; m2 = the remaining columns shifted down.
  for (auto& d : m1.out) {
    int i = m.out_index(d.name);
    if (i < 0 || m.out[i].bits < d.bits)
      throw Error(LL_ERR_SHAPE, "left_divide: output dim " + d.name + " missing or too small");
  }
  for (auto& d : m1.in)
    if (m.in_size(d.name) < d.bits && !(m.in_offset(d.name) >= 0 && d.bits == 0))
      throw Error(LL_ERR_SHAPE, "left_divide: input dim " + d.name + " missing or too small");
  auto low_bits = [&](const std::string& name) {
    int i = m1.out_index(name);
    return i < 0 ? 0 : m1.out[i].bits;
  };
  Layout r;
  for (auto& d : m.out) r.out.push_back({d.name, d.bits - low_bits(d.name)});
  for (auto& d : m.in) {
    const int k1 = m1.in_size(d.name);
    auto mv = m.sub(d.name);
    auto m1v = m1.sub(d.name);
    for (int k = 0; k < k1; ++k) {
      auto c1 = m1.unflatten(m1v[k]);
      std::vector<int64_t> want(m.out.size(), 0);
      for (size_t o = 0; o < m1.out.size(); ++o) want[m.out_index(m1.out[o].name)] = c1[o];
      if (mv[k] != m.flatten(want))
        throw Error(LL_ERR_SHAPE, "left_divide: " + d.name + " bit " + std::to_string(k) +
                                      " is not the divisor's column");
    }
    for (int k = k1; k < d.bits; ++k) {
      auto c = m.unflatten(mv[k]);
      std::vector<int64_t> rc(m.out.size(), 0);
      for (size_t o = 0; o < m.out.size(); ++o) {
        const int lb = low_bits(m.out[o].name);
        if (c[o] & ((int64_t(1) << lb) - 1))
          throw Error(LL_ERR_SHAPE, "left_divide: " + d.name + " bit " + std::to_string(k) +
                                        " has a non-zero divisor block");
        rc[o] = c[o] >> lb;
      }
      r.cols.push_back(r.flatten(rc));
    }
    r.in.push_back({d.name, d.bits - k1});
  }
  return r;
}

}  // namespace ll

namespace ll {

// tt.trans: permute the output dims; every column keeps its coordinates.
Layout shape_transpose(const Layout& l, const std::vector<int>& perm) {
  const int r = (int)l.out.size();
  if ((int)perm.size() != r) throw Error(LL_ERR_ARG, "transpose: permutation size != rank");
  std::vector<int> seen(r, 0);
  for (int p : perm) {
    if (p < 0 || p >= r || seen[p]++) throw Error(LL_ERR_ARG, "transpose: not a permutation");
  }
  Layout o;
  o.in = l.in;
  for (int i = 0; i < r; ++i) o.out.push_back(l.out[perm[i]]);
  for (u64 c : l.cols) {
    auto x = l.unflatten(c);
    std::vector<int64_t> y(r);
    for (int i = 0; i < r; ++i) y[i] = x[perm[i]];
    o.cols.push_back(o.flatten(y));
  }
  return o;
}

// tt.reshape: row-major flattening is preserved, so the flat columns
// are unchanged; only the split of the flat index into dims changes.
Layout shape_reshape(const Layout& l, const std::vector<Dim>& new_out) {
  int t = 0;
  for (auto& d : new_out) {
    if (d.bits < 0) throw Error(LL_ERR_ARG, "reshape: negative dim");
    t += d.bits;
  }
  if (t != l.out_bits()) throw Error(LL_ERR_SHAPE, "reshape: element count changes");
  Layout o;
  o.in = l.in;
  o.out = new_out;
  o.cols = l.cols;
  return o;
}

// tt.expand_dims: a new size-1 dim at position `axis`.
Layout shape_expand_dims(const Layout& l, int axis, const std::string& name) {
  if (axis < 0 || axis > (int)l.out.size()) throw Error(LL_ERR_ARG, "expand_dims: axis out of range");
  if (l.out_index(name) >= 0) throw Error(LL_ERR_ARG, "expand_dims: duplicate dim name");
  Layout o;
  o.in = l.in;
  o.out = l.out;
  o.out.insert(o.out.begin() + axis, Dim{name, 0});
  o.cols = l.cols;  // a 0-bit dim adds no flat bits
  return o;
}

// tt.broadcast: a size-1 dim grows to 2^bits.  Hardware
// indices that held copies (zero columns, lowest first) now index the new
// dim; if there are fewer copies than new bits, registers are added.
Layout shape_broadcast(const Layout& l, int axis, int bits) {
  if (axis < 0 || axis >= (int)l.out.size()) throw Error(LL_ERR_ARG, "broadcast: axis out of range");
  if (l.out[axis].bits != 0) throw Error(LL_ERR_SHAPE, "broadcast: the dim must have size 1");
  if (bits < 0 || l.out_bits() + bits > 62) throw Error(LL_ERR_ARG, "broadcast: bad size");
  Layout o;
  o.in = l.in;
  o.out = l.out;
  o.out[axis].bits = bits;
  int used = 0;
  for (u64 c : l.cols) {
    auto x = l.unflatten(c);
    if (c == 0 && used < bits) x[axis] = int64_t(1) << used++;
    o.cols.push_back(o.flatten(x));
  }
  // remaining new bits: extra register bits (appended at the top of "reg")
  if (used < bits) {
    int roff = o.in_offset("reg");
    int rbits = o.in_size("reg");
    if (roff < 0) {
      o.in.insert(o.in.begin(), Dim{"reg", 0});
      roff = 0;
      rbits = 0;
    }
    std::vector<u64> add;
    for (; used < bits; ++used) {
      std::vector<int64_t> x(o.out.size(), 0);
      x[axis] = int64_t(1) << used;
      add.push_back(o.flatten(x));
    }
    o.cols.insert(o.cols.begin() + roff + rbits, add.begin(), add.end());
    for (auto& d : o.in)
      if (d.name == "reg") d.bits += (int)add.size();
  }
  return o;
}

// tt.join: two tensors of the same layout become a new fastest dim of
// size 2, the two values of a hardware index sitting in adjacent registers:
// a new register bit 0 maps to the new dim; existing register bits shift up.
Layout shape_join(const Layout& l, const std::string& name) {
  if (l.out_index(name) >= 0) throw Error(LL_ERR_ARG, "join: duplicate dim name");
  Layout o;
  o.in = l.in;
  o.out = l.out;
  o.out.push_back(Dim{name, 1});
  int roff = o.in_offset("reg");
  if (roff < 0) {
    o.in.insert(o.in.begin(), Dim{"reg", 0});
    roff = 0;
  }
  for (u64 c : l.cols) o.cols.push_back(c << 1);  // the new dim is the lowest flat bit
  o.cols.insert(o.cols.begin() + roff, u64(1));
  for (auto& d : o.in)
    if (d.name == "reg") d.bits += 1;
  return o;
}

// tt.split: inverse of join -- the last dim (size 2) must be held by
// exactly one register bit, which is removed together with the dim.
Layout shape_split(const Layout& l) {
  if (l.out.empty() || l.out.back().bits != 1) throw Error(LL_ERR_SHAPE, "split: the last dim must have size 2");
  const int roff = l.in_offset("reg");
  const int rbits = l.in_size("reg");
  int hold = -1;
  for (int k = 0; k < (int)l.cols.size(); ++k) {
    if (l.cols[k] & 1) {
      if (hold >= 0 || l.cols[k] != 1 || roff < 0 || k < roff || k >= roff + rbits)
        throw Error(LL_ERR_UNSUPPORTED, "split: the size-2 dim is not held by a single register bit");
      hold = k;
    }
  }
  if (hold < 0) throw Error(LL_ERR_UNSUPPORTED, "split: the size-2 dim is not held by any register");
  Layout o;
  o.in = l.in;
  o.out.assign(l.out.begin(), l.out.end() - 1);
  for (int k = 0; k < (int)l.cols.size(); ++k)
    if (k != hold) o.cols.push_back(l.cols[k] >> 1);
  for (auto& d : o.in)
    if (d.name == "reg") d.bits -= 1;
  return o;
}

// Sliced layouts: removing the output dim `axis` (the result of a
// reduction along it) is a linear map; the matrix loses that dim's rows, so
// columns that only reached it become zero (broadcast) -- still surjective.
Layout shape_slice(const Layout& l, int axis) {
  if (axis < 0 || axis >= (int)l.out.size()) throw Error(LL_ERR_ARG, "slice: axis out of range");
  Layout o;
  o.in = l.in;
  o.out = l.out;
  o.out.erase(o.out.begin() + axis);
  for (u64 c : l.cols) {
    auto x = l.unflatten(c);
    x.erase(x.begin() + axis);
    o.cols.push_back(o.flatten(x));
  }
  return o;
}

namespace {
// Product of identity tiles id^{in,out}_k in order (Appendix notation,
// P:1005): each factor maps the next k bits of input dim `in` onto the next k
// bits of output dim `out` (a shared label's earlier factors are the low bits,
// Definition "Product").
struct TileBuilder {
  std::vector<std::string> in_names;
  std::vector<std::vector<std::pair<int, int>>> in_cols;  // per input dim: (out dim, out bit)
  std::vector<int> out_used;
  explicit TileBuilder(int n_out) : out_used(n_out, 0) {}
  void id(const std::string& in, int out, int k) {
    auto it = std::find(in_names.begin(), in_names.end(), in);
    size_t d = it - in_names.begin();
    if (it == in_names.end()) {
      in_names.push_back(in);
      in_cols.emplace_back();
    }
    for (int i = 0; i < k; ++i) in_cols[d].push_back({out, out_used[out]++});
  }
  Layout build(const std::vector<std::string>& order, const std::vector<int>& out_bits) {
    Layout L;
    for (size_t o = 0; o < out_bits.size(); ++o) L.out.push_back({"dim" + std::to_string(o), out_bits[o]});
    for (const std::string& nm : order) {
      auto it = std::find(in_names.begin(), in_names.end(), nm);
      const int d = it == in_names.end() ? -1 : (int)(it - in_names.begin());
      const int bits = d < 0 ? 0 : (int)in_cols[d].size();
      L.in.push_back({nm, bits});
      for (int i = 0; i < bits; ++i) {
        std::vector<int64_t> x(out_bits.size(), 0);
        x[in_cols[d][i].first] = int64_t(1) << in_cols[d][i].second;
        L.cols.push_back(L.flatten(x));
      }
    }
    return L;
  }
};
}  // namespace

// Blocked layouts (Appendix proposition):
// sigma_o^{-1} o (id_R^o x id_T^o x id_W^o), id_R^o = id^{reg,o_1}_{r_{o_1}} x
// ... x id^{reg,o_l}_{r_{o_l}}; order[0] = the fastest dim.
Layout make_blocked(const std::vector<int>& shape_bits, const std::vector<int>& R,
                    const std::vector<int>& T, const std::vector<int>& W,
                    const std::vector<int>& order) {
  const size_t rank = shape_bits.size();
  if (rank == 0 || R.size() != rank || T.size() != rank || W.size() != rank || order.size() != rank)
    throw Error(LL_ERR_ARG, "blocked: R, T, W, order must have one entry per dim");
  std::vector<int> seen(rank, 0);
  for (int o : order) {
    if (o < 0 || o >= (int)rank || seen[o]++) throw Error(LL_ERR_ARG, "blocked: order must be a permutation");
  }
  for (size_t i = 0; i < rank; ++i)
    if (R[i] < 0 || T[i] < 0 || W[i] < 0 || R[i] + T[i] + W[i] != shape_bits[i])
      throw Error(LL_ERR_SHAPE, "blocked: R_i + T_i + W_i must equal d_i (P:1012)");
  TileBuilder tb((int)rank);
  for (int o : order) tb.id("reg", o, R[o]);
  for (int o : order) tb.id("lane", o, T[o]);
  for (int o : order) tb.id("warp", o, W[o]);
  return tb.build({"reg", "lane", "warp"}, shape_bits);
}

// mma tiles (Appendix proposition): lhs / output
// id^{reg,1}_{log2(32/b)} x id^{thread,1}_2 x id^{thread,0}_3 x id^{reg,0}_1 x
// id^{reg,1}_1; rhs id^{reg,0}_{log2(32/b)} x id^{thread,0}_2 x id^{thread,1}_3 x
// id^{reg,0}_1 (reading A8: the printed trailing id^{reg,1}_1 contradicts the
// PTX m16n8k16 B fragment); output = the first four factors of the b = 16 lhs
// tile (the m16n8 accumulator fragment).  operand 0 = lhs, 1 = rhs, 2 = out.
Layout make_mma_tile(int operand, int bitwidth) {
  if (bitwidth != 8 && bitwidth != 16 && bitwidth != 32) throw Error(LL_ERR_ARG, "mma: bitwidth must be 8, 16 or 32");
  int kreg = 0;
  while ((32 / bitwidth) > (1 << kreg)) ++kreg;
  TileBuilder tb(2);
  if (operand == 0) {
    tb.id("reg", 1, kreg); tb.id("lane", 1, 2); tb.id("lane", 0, 3); tb.id("reg", 0, 1); tb.id("reg", 1, 1);
  } else if (operand == 1) {
    tb.id("reg", 0, kreg); tb.id("lane", 0, 2); tb.id("lane", 1, 3); tb.id("reg", 0, 1);
  } else if (operand == 2) {
    tb.id("reg", 1, 1); tb.id("lane", 1, 2); tb.id("lane", 0, 3); tb.id("reg", 0, 1);
  } else {
    throw Error(LL_ERR_ARG, "mma: operand must be 0 (lhs), 1 (rhs) or 2 (out)");
  }
  return tb.build({"reg", "lane"}, {tb.out_used[0], tb.out_used[1]});
}

}  // namespace ll
