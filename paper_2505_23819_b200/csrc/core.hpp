// core.hpp -- host-side F2 algebra and labeled linear layouts (C++17).
//
// Vectors of F2^d are uint64_t with bit k = coordinate k (LSB-first, PAPER.md
// P:305 footnote).  A matrix is the vector of its columns: column k is the
// image of input bit k (P:283-295 shows layout A this way), so M v is the
// XOR of the columns selected by v.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ll.h"

namespace ll {

using u64 = uint64_t;

// Internal error carrying an ll_status; converted at the C-ABI boundary.
struct Error : std::runtime_error {
  ll_status code;
  Error(ll_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline int popcount64(u64 x) { return __builtin_popcountll(x); }
inline int ctz64(u64 x) { return __builtin_ctzll(x); }

// M v: XOR of the columns picked by the set bits of v.
inline u64 f2_apply(const std::vector<u64>& cols, u64 v) {
  u64 out = 0;
  for (size_t k = 0; v && k < cols.size(); ++k, v >>= 1)
    if (v & 1) out ^= cols[k];
  return out;
}

// Incremental row-echelon basis keyed by highest set bit.
struct F2Basis {
  u64 piv[64] = {0};
  int n = 0;
  // reduce x against the basis; returns residue (0 iff x in span)
  u64 reduce(u64 x) const {
    for (int b = 63; b >= 0 && x; --b)
      if (((x >> b) & 1) && piv[b]) x ^= piv[b];
    return x;
  }
  bool in_span(u64 x) const { return reduce(x) == 0; }
  bool add(u64 x) {  // true if x was independent
    x = reduce(x);
    if (!x) return false;
    piv[63 - __builtin_clzll(x)] = x;
    ++n;
    return true;
  }
};

inline int f2_rank(const std::vector<u64>& v) {
  F2Basis b;
  for (u64 x : v) b.add(x);
  return b.n;
}

// Right inverse of a surjective m-row matrix: Gauss-Jordan on
// [M | I], columns in order, pivot = first remaining row with a one, free
// variables zero.  Returns m columns of n bits.  Throws
// LL_ERR_NOT_SURJECTIVE when rank < m.
std::vector<u64> f2_right_inverse(const std::vector<u64>& cols, int m);

// Lowest standard vectors completing `vecs` to a basis of F2^d.
std::vector<u64> f2_complete(const std::vector<u64>& vecs, int d);

struct Dim {
  std::string name;
  int bits = 0;
};

// A labeled linear layout.  Input dims minor -> major (first-listed at the
// lowest flat bits); output dims dim0..dimN-1, row-major (last dim fastest).
struct Layout {
  std::vector<Dim> in, out;
  std::vector<u64> cols;  // flat out vector per flat input bit

  int in_bits() const;
  int out_bits() const;
  int in_offset(const std::string& name) const;  // -1 if absent
  int in_size(const std::string& name) const;    // 0 if absent
  int out_index(const std::string& name) const;  // -1 if absent
  int out_shift(int d) const;                    // flat position of bit 0 of out dim d
  std::vector<u64> sub(const std::string& name) const;
  u64 flatten(const std::vector<int64_t>& coords) const;
  std::vector<int64_t> unflatten(u64 x) const;
  bool surjective() const;
  bool distributed() const;
  bool memory() const;
  u64 hash() const;
  bool same_tensor(const Layout& o) const;
};

Layout compose(const Layout& outer, const Layout& inner);
Layout right_inverse(const Layout& l);
Layout product(const Layout& a, const Layout& b);
// Left division: m = [[m1, 0], [0, m2]] label-wise -> m2; throws
// LL_ERR_SHAPE when m has no such structure.
Layout left_divide(const Layout& m, const Layout& m1);

}  // namespace ll

namespace ll {
// Shape-operation transfer functions on layouts (Appendix theorem
// P:1057-1064): for a distributed input layout, the output layout for which
// the shape operation moves no data between hardware indices.
Layout shape_transpose(const Layout& l, const std::vector<int>& perm);
Layout shape_reshape(const Layout& l, const std::vector<Dim>& new_out);
Layout shape_expand_dims(const Layout& l, int axis, const std::string& name);
Layout shape_broadcast(const Layout& l, int axis, int bits);
Layout shape_join(const Layout& l, const std::string& name);
Layout shape_split(const Layout& l);
Layout shape_slice(const Layout& l, int axis);
Layout make_blocked(const std::vector<int>& shape_bits, const std::vector<int>& R,
                    const std::vector<int>& T, const std::vector<int>& W,
                    const std::vector<int>& order);
Layout make_mma_tile(int operand, int bitwidth);
}  // namespace ll
