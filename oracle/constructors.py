"""Layout constructors from the paper -- oracle (test infrastructure only).

* ``identity``      id^{i,j}_k of the Appendix notation.
* ``blocked``       Proposition "Blocked layouts are linear layouts", proof
                    P:1011-1025: sigma_o^{-1} o (id_R^o x id_T^o x id_W^o).
* ``mma_tile``      Proposition on mma layouts, proof P:1031-1047 (with the
                    reading A8 for the rhs tile).
* ``mma_swizzle_*`` Definition 5 "mma swizzling" and the matrix
                    structure [[I_n, C], [0, I_m]] stated after it.
"""

from .layout import Layout, product, with_out_order


def dim_names(rank):
    return ["dim%d" % d for d in range(rank)]


def identity(k, in_name, out_name):
    """id^{in,out}_k: the first k bits of ``in_name`` map identically onto the
    first k bits of output dim ``out_name``."""
    return Layout([(in_name, k)], [(out_name, k)], {in_name: [(1 << i,) for i in range(k)]})


def empty(out_names=()):
    return Layout([], [(n, 0) for n in out_names], {})


def blocked(shape_bits, R, T, W, order, thread_name="lane"):
    """Blocked layout of the Appendix proof.

    shape_bits[i] = d_i = log2 of dim i, R/T/W = log2 of registers/threads/warps
    per dim with R_i + T_i + W_i = d_i, ``order`` lists dims fastest first
    (o_1 is the fastest).  id_R^o = id^{reg,o_1}_{r_{o_1}} x ... x id^{reg,o_l}_{r_{o_l}}
    and likewise for T, W; sigma_o^{-1} restores the dim order.  Output dims are
    dim0..dim{l-1} (dim0 slowest).
    """
    rank = len(shape_bits)
    for i in range(rank):
        if R[i] + T[i] + W[i] != shape_bits[i]:
            raise ValueError("blocked: R_i + T_i + W_i must equal d_i (P:1012)")
    names = dim_names(rank)
    lay = empty()
    for label, sizes in (("reg", R), (thread_name, T), ("warp", W)):
        for o in order:
            lay = product(lay, identity(sizes[o], label, names[o]))
    for label in ("reg", thread_name, "warp"):
        if label not in dict(lay.in_dims):
            lay = product(lay, Layout([(label, 0)], [], {label: []}))
    # drop size-0 out dims bookkeeping: rebuild with all dims in order
    lay = _ensure_out_dims(lay, names)
    return with_out_order(lay, names)


def _ensure_out_dims(lay, names):
    have = dict(lay.out_dims)
    if all(n in have for n in names):
        return lay
    return product(lay, Layout([], [(n, 0) for n in names if n not in have], {}))


def mma_tile(operand, bitwidth, thread_name="lane", rhs_reading="A8"):
    """Register/thread tile of NVIDIA ``mma`` operands (Appendix).

    lhs (and output) tile:  id^{reg,1}_{log2(32/b)} x id^{thread,1}_2 x
                            id^{thread,0}_3 x id^{reg,0}_1 x id^{reg,1}_1
    rhs tile, as printed:   id^{reg,0}_{log2(32/b)} x id^{thread,0}_2 x
                            id^{thread,1}_3 x id^{reg,1}_1
    Reading A8: the printed trailing id^{reg,1}_1 of the rhs contradicts the
    PTX m16n8k16 B fragment; we read id^{reg,0}_1 (``rhs_reading="A8"``);
    ``rhs_reading="printed"`` gives the literal text.  The output (accumulator)
    tile is the first four factors of the b=16 lhs formula (reading A8).
    Output dims: dim0 = rows (m for lhs/out, k for rhs), dim1 = columns.
    """
    import math
    names = dim_names(2)
    if bitwidth not in (8, 16, 32):
        raise ValueError("mma_tile: bitwidth must be 8, 16 or 32")
    kreg = int(math.log2(32 // bitwidth))
    t = thread_name
    if operand == "lhs":
        factors = [identity(kreg, "reg", "dim1"), identity(2, t, "dim1"),
                   identity(3, t, "dim0"), identity(1, "reg", "dim0"),
                   identity(1, "reg", "dim1")]
    elif operand == "out":
        factors = [identity(1, "reg", "dim1"), identity(2, t, "dim1"),
                   identity(3, t, "dim0"), identity(1, "reg", "dim0")]
    elif operand == "rhs":
        last = identity(1, "reg", "dim0") if rhs_reading == "A8" else identity(1, "reg", "dim1")
        factors = [identity(kreg, "reg", "dim0"), identity(2, t, "dim0"),
                   identity(3, t, "dim1"), last]
    else:
        raise ValueError("operand must be lhs, rhs or out")
    lay = empty()
    for f in factors:
        lay = product(lay, f)
    lay = _ensure_out_dims(lay, names)
    return with_out_order(lay, names)


# --- Definition 5: mma swizzling ------------------------------------------------

def mma_swizzle_offset(i, j, n, vec, per_phase, max_phase):
    """Def. 5: offset of element (i, j) of a 2^m x 2^n tensor,
    counted in elements:  ((i/per_phase mod max_phase) XOR j/vec) . vec XOR
    (j mod vec), placed in row i.  Reading A7: per_phase, max_phase >= 1 and
    the swizzled column is reduced mod 2^n."""
    col = ((((i // per_phase) % max_phase) ^ (j // vec)) * vec) ^ (j % vec)
    return i * (1 << n) + (col % (1 << n))


def mma_swizzle_layout(m, n, vec, per_phase, max_phase):
    """Memory layout offset -> (i, j) from the matrix structure printed after
    Def. 5: [[I_n, C], [0, I_m]] with (reading A7) the k-th
    *column* of C, i.e. the image of row bit k, equal to
    c_k = (vec . ((2^k / per_phase) mod max_phase)) mod 2^n."""
    bases = []
    for k in range(n):                       # offset bit k (< n) -> column bit k
        bases.append((0, 1 << k))
    for k in range(m):                       # offset bit n+k -> row bit k plus C's column
        c = (vec * (((1 << k) // per_phase) % max_phase)) % (1 << n)
        bases.append((1 << k, c))
    return Layout([("offset", m + n)], [("dim0", m), ("dim1", n)], {"offset": bases})
