"""Labeled linear layouts -- oracle (test infrastructure only).

Definition "Linear Layouts": a linear map between labeled vector
spaces over F2.  Conventions (reading A1/A2):

* input dims are listed minor -> major; the flattened input index puts the
  first-listed dim at the lowest bits (v_{0:1} = reg, v_{2:6} = thread,
  v_7 = warp);
* output dims are tensor dims dim0..dimN-1 flattened row-major, last dim
  fastest ("w_{0:3} = j and w_{4:7} = i, given that j is the fastest
  moving dimension");
* every basis vector is stored both as per-dim coordinates and as a flat int.
"""

from . import f2


class Layout:
    """A labeled linear layout given by the images of its input basis bits.

    ``bases[name][k]`` is the tuple of output coordinates (one per out dim) of
    input bit k of input dim ``name`` -- exactly the paper's columns (P:283-295
    displays them as the columns of A).  A zero tuple is a zero column
    (broadcast).
    """

    def __init__(self, in_dims, out_dims, bases):
        self.in_dims = [(str(n), int(b)) for n, b in in_dims]
        self.out_dims = [(str(n), int(b)) for n, b in out_dims]
        names = [n for n, _ in self.in_dims]
        if len(set(names)) != len(names):
            raise ValueError("duplicate input dim names")
        onames = [n for n, _ in self.out_dims]
        if len(set(onames)) != len(onames):
            raise ValueError("duplicate output dim names")
        self.bases = {}
        for n, b in self.in_dims:
            vecs = [tuple(int(c) for c in v) for v in bases.get(n, [])]
            if len(vecs) != b:
                raise ValueError("dim %s: %d bases given, %d expected" % (n, len(vecs), b))
            for v in vecs:
                if len(v) != len(self.out_dims):
                    raise ValueError("basis arity mismatch")
                for c, (_, ob) in zip(v, self.out_dims):
                    if c < 0 or c >= (1 << ob):
                        raise ValueError("basis coordinate out of range")
            self.bases[n] = vecs

    # --- sizes and flattening -------------------------------------------
    @property
    def in_bits(self):
        return sum(b for _, b in self.in_dims)

    @property
    def out_bits(self):
        return sum(b for _, b in self.out_dims)

    def in_offset(self, name):
        off = 0
        for n, b in self.in_dims:
            if n == name:
                return off
            off += b
        raise KeyError(name)

    def in_size(self, name):
        for n, b in self.in_dims:
            if n == name:
                return b
        return 0

    def out_shift(self, d):
        """Flat bit position of bit 0 of output dim index d (row-major)."""
        return sum(b for _, b in self.out_dims[d + 1:])

    def flatten(self, coords):
        x = 0
        for d, c in enumerate(coords):
            x |= int(c) << self.out_shift(d)
        return x

    def unflatten(self, x):
        return tuple((x >> self.out_shift(d)) & ((1 << b) - 1)
                     for d, (_, b) in enumerate(self.out_dims))

    @property
    def cols(self):
        """Flat matrix: column k = flat image of flattened input bit k."""
        out = []
        for n, _ in self.in_dims:
            out.extend(self.flatten(v) for v in self.bases[n])
        return out

    def sub(self, name):
        """L_name: flat images of the basis bits of input dim ``name``."""
        return [self.flatten(v) for v in self.bases.get(name, [])]

    # --- evaluation ---------------------------------------------------------
    def apply_flat(self, h):
        """Tensor flat index of flattened input index h ("w = Av")."""
        return f2.apply(self.cols, h)

    def apply(self, point):
        """``point`` maps input dim name -> coordinate; returns out coords.

        P:273-277: the location is the XOR of the per-level locations."""
        h = 0
        for n, b in self.in_dims:
            c = int(point.get(n, 0))
            if c < 0 or c >= (1 << b):
                raise ValueError("coordinate %s=%d out of range" % (n, c))
            h |= c << self.in_offset(n)
        return self.unflatten(self.apply_flat(h))

    # --- predicates -----------------------------------------------------------
    def is_surjective(self):
        return f2.rank(self.cols) == self.out_bits

    def is_distributed(self, allowed=("reg", "lane", "thread", "warp", "block")):
        """Definition "Distributed Layout": surjective, every column
        has at most one non-zero bit, no two non-zero columns repeated."""
        if any(n not in allowed for n, _ in self.in_dims):
            return False
        cols = self.cols
        nz = [c for c in cols if c]
        return (self.is_surjective() and all(f2.popcount(c) <= 1 for c in cols)
                and len(set(nz)) == len(nz))

    def is_memory(self):
        """Definition "Memory Layout": invertible, columns of weight
        1 or 2 (single input dim ``offset``)."""
        if [n for n, _ in self.in_dims] != ["offset"]:
            return False
        cols = self.cols
        return (len(cols) == self.out_bits and f2.rank(cols) == len(cols)
                and all(f2.popcount(c) in (1, 2) for c in cols))

    def broadcast_mask(self, name):
        """Zero columns of input dim ``name``."""
        m = 0
        for k, v in enumerate(self.bases.get(name, [])):
            if not any(v):
                m |= 1 << k
        return m

    def __eq__(self, other):
        return (isinstance(other, Layout) and self.in_dims == other.in_dims
                and self.out_dims == other.out_dims and self.bases == other.bases)

    def __repr__(self):
        parts = []
        for n, _ in self.in_dims:
            parts.append("%s=%s" % (n, self.bases[n]))
        return "Layout(out=%s, %s)" % (self.out_dims, ", ".join(parts))


def from_flat(in_dims, out_dims, cols):
    """Build a Layout from a flat column list (inverse of ``Layout.cols``)."""
    tmp = Layout(in_dims, out_dims, {n: [(0,) * len(out_dims)] * b for n, b in in_dims})
    bases = {}
    k = 0
    for n, b in in_dims:
        bases[n] = [tmp.unflatten(cols[k + i]) for i in range(b)]
        k += b
    return Layout(in_dims, out_dims, bases)


def compose(outer, inner):
    """Definition "Composition": (L2 o L1)(u) = L2(L1(u)); the matrix
    is the label-wise product M2 M1.  inner's output dims must equal outer's
    input dims (names and sizes); matching is by name."""
    o_in = dict(outer.in_dims)
    i_out = dict(inner.out_dims)
    if o_in != i_out:
        raise ValueError("compose: label mismatch %s vs %s" % (outer.in_dims, inner.out_dims))
    bases = {}
    for n, _ in inner.in_dims:
        vecs = []
        for v in inner.bases[n]:
            pt = {name: c for (name, _), c in zip(inner.out_dims, v)}
            vecs.append(outer.apply(pt))
        bases[n] = vecs
    return Layout(inner.in_dims, outer.out_dims, bases)


def product(l1, l2):
    """Definition "Product": label-wise block-diagonal matrix.

    For a label shared by both, l1's bits come first (low) and l2's after
    (high), on inputs and on outputs alike; new labels are appended."""
    in_dims = list(l1.in_dims)
    for n, b in l2.in_dims:
        if n in dict(in_dims):
            in_dims = [(m, c + b) if m == n else (m, c) for m, c in in_dims]
        else:
            in_dims.append((n, b))
    out_names = [n for n, _ in l1.out_dims] + [n for n, _ in l2.out_dims
                                               if n not in dict(l1.out_dims)]
    o1 = dict(l1.out_dims)
    o2 = dict(l2.out_dims)
    out_dims = [(n, o1.get(n, 0) + o2.get(n, 0)) for n in out_names]

    def embed(layout, v, shift):
        coords = dict(zip([n for n, _ in layout.out_dims], v))
        return tuple((coords.get(n, 0) << shift.get(n, 0)) for n in out_names)

    bases = {}
    for n, _ in in_dims:
        vecs = [embed(l1, v, {}) for v in l1.bases.get(n, [])]
        vecs += [embed(l2, v, o1) for v in l2.bases.get(n, [])]
        bases[n] = vecs
    return Layout(in_dims, out_dims, bases)


def with_out_order(layout, names):
    """Same map with output dims listed in ``names`` order (changes flattening)."""
    od = dict(layout.out_dims)
    idx = [[n for n, _ in layout.out_dims].index(m) for m in names]
    bases = {n: [tuple(v[i] for i in idx) for v in vs] for n, vs in layout.bases.items()}
    return Layout(layout.in_dims, [(m, od[m]) for m in names], bases)


def left_divide(m, m1):
    """Definition "Left Division": M = [[M1, 0], [0, M2]] label-wise
    gives M // M1 = M2; otherwise ValueError.  Inverse of ``product``."""
    o1 = dict(m1.out_dims)
    om = dict(m.out_dims)
    for n, b in m1.out_dims:
        if om.get(n, -1) < b:
            raise ValueError("left_divide: output dim %s too small" % n)
    out_names = [n for n, _ in m.out_dims]
    in2 = []
    bases2 = {}
    for n, b in m.in_dims:
        k1 = m1.in_size(n)
        if k1 > b:
            raise ValueError("left_divide: input dim %s too small" % n)
        vecs = m.bases[n]
        for k in range(k1):
            want = tuple(dict(zip([x for x, _ in m1.out_dims], m1.bases[n][k])).get(d, 0)
                         for d in out_names)
            if vecs[k] != want:
                raise ValueError("left_divide: %s bit %d is not M1's column" % (n, k))
        rest = []
        for k in range(k1, b):
            v = vecs[k]
            for d, c in zip(out_names, v):
                if c & ((1 << o1.get(d, 0)) - 1):
                    raise ValueError("left_divide: %s bit %d has a non-zero M1 block" % (n, k))
            rest.append(tuple(c >> o1.get(d, 0) for d, c in zip(out_names, v)))
        if b - k1 > 0 or n in dict(m.in_dims):
            in2.append((n, b - k1))
            bases2[n] = rest
    for n in m1.in_dims:
        if n[0] not in dict(m.in_dims):
            raise ValueError("left_divide: unknown input dim %s" % n[0])
    out2 = [(d, om[d] - o1.get(d, 0)) for d in out_names]
    return Layout(in2, out2, bases2)


def right_inverse(layout):
    """Definition "Right Inverse" applied label-wise: the returned
    layout maps the tensor (input dims = the out dims, listed fastest first so
    the flat index is unchanged) to the hardware dims (out dims = the in dims,
    listed major first so the flat index is unchanged)."""
    xcols = f2.right_inverse(layout.cols, layout.out_bits)
    in_dims = list(reversed(layout.out_dims))
    out_dims = list(reversed(layout.in_dims))
    return from_flat(in_dims, out_dims, xcols)
