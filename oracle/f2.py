"""F2 (GF(2)) vectors and matrices -- oracle (test infrastructure only).

Representation (P:305 footnote, "The least significant bits come first in the
vector"): a vector of F2^d is a Python int whose bit k is coordinate k.  A
matrix M in F2^{m x n} is the list of its n columns, each an int of m bits, so
that ``M v`` is the XOR of the columns selected by the set bits of v
(c_ij = XOR_k a_ik . b_kj; "w = A v").
"""


def popcount(x):
    return bin(x).count("1")


def apply(cols, v):
    """M v for M given by columns (P:298, P:305-306 worked example)."""
    out = 0
    k = 0
    while v:
        if v & 1:
            out ^= cols[k]
        v >>= 1
        k += 1
    return out


def matmul(cols2, cols1):
    """(M2 M1) as columns: column j of M2 M1 is M2 (column j of M1)."""
    return [apply(cols2, c) for c in cols1]


def rank(vectors):
    """Rank over F2 by elimination on a copy of the vectors."""
    basis = {}  # highest set bit -> basis vector
    for v in vectors:
        while v:
            h = v.bit_length() - 1
            if h in basis:
                v ^= basis[h]
            else:
                basis[h] = v
                break
    return len(basis)


def in_span(v, vectors):
    return rank(list(vectors) + [v]) == rank(vectors)


def span(vectors):
    """All elements of span(vectors), as a set.  Small inputs only."""
    out = {0}
    for v in vectors:
        out |= {x ^ v for x in out}
    return out


def intersection_dim(U, V):
    """dim(span U  cap  span V) = dim U + dim V - dim(U + V)."""
    return rank(U) + rank(V) - rank(list(U) + list(V))


def complete_basis(vectors, d):
    """Extend independent ``vectors`` to a basis of F2^d by appending the
    lowest-index standard vectors not yet in the span (the deterministic
    completion used for R in P:649-650 and for C / S_bank in P:706)."""
    out = list(vectors)
    if rank(out) != len(out):
        raise ValueError("complete_basis: input vectors are dependent")
    for k in range(d):
        if rank(out) == d:
            break
        e = 1 << k
        if not in_span(e, out):
            out.append(e)
    return out[len(vectors):]


def right_inverse(cols, m):
    """Right inverse of a surjective M (m x n, given by its n columns).

    Definition "Right Inverse": M^{-1} is the n x m solution of
    M X = I_m, "computed via Gaussian elimination over F2".  Free (slack)
    variables are set to zero ("we set the slack variables in the
    linear system to zeros").  Pivot rule (reading A4): columns are processed
    in order 0..n-1 and the pivot is the first remaining row with a 1 in that
    column; so basic variables are the earliest independent columns.

    Returns the m columns of X, each an int of n bits.  Raises ValueError if M
    is not surjective (rank < m).
    """
    n = len(cols)
    # rows of [M | I]: row r of M is the n-bit int of bit r of every column
    rows = []
    for r in range(m):
        row = 0
        for j, c in enumerate(cols):
            if (c >> r) & 1:
                row |= 1 << j
        rows.append(row)
    aug = [1 << r for r in range(m)]
    pivcol = []
    p = 0
    for j in range(n):
        sel = None
        for r in range(p, m):
            if (rows[r] >> j) & 1:
                sel = r
                break
        if sel is None:
            continue
        rows[p], rows[sel] = rows[sel], rows[p]
        aug[p], aug[sel] = aug[sel], aug[p]
        for q in range(m):
            if q != p and (rows[q] >> j) & 1:
                rows[q] ^= rows[p]
                aug[q] ^= aug[p]
        pivcol.append(j)
        p += 1
        if p == m:
            break
    if p < m:
        raise ValueError("right_inverse: matrix is not surjective (rank %d < %d)" % (p, m))
    # X row pivcol[i] = aug[i] (an m-bit row); free rows are zero.
    xcols = []
    for c in range(m):
        col = 0
        for i, j in enumerate(pivcol):
            if (aug[i] >> c) & 1:
                col |= 1 << j
        xcols.append(col)
    return xcols


def solve_all(cols, target):
    """All x with M x = target (brute force; small n only). Test helper."""
    n = len(cols)
    return [x for x in range(1 << n) if apply(cols, x) == target]
