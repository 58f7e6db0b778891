"""Shape-operation transfer functions -- oracle (tests only).

P:491-498 ("For every input distributed layout, there exists an output layout
from the same family such that the operation effectively becomes a no-op") and
the Appendix theorem.  Each function returns the output layout
for which every hardware index keeps the value it held, written directly from
the operation's effect on tensor coordinates:

* trans(perm):     coordinate c -> (c[perm[0]], ..., c[perm[r-1]])
* reshape(dims):   row-major flat index preserved
* expand_dims:     a size-1 coordinate inserted
* broadcast:       a size-1 dim grows; hardware copies (zero columns) index it
* join:            two tensors -> new fastest dim of size 2 (adjacent registers)
* split:           inverse of join
"""

from .layout import Layout


def trans(L, perm):
    out = [L.out_dims[p] for p in perm]
    bases = {n: [tuple(v[p] for p in perm) for v in vs] for n, vs in L.bases.items()}
    return Layout(L.in_dims, out, bases)


def reshape(L, new_dims):
    new = Layout([], new_dims, {})
    if new.out_bits != L.out_bits:
        raise ValueError("reshape changes the element count")
    bases = {n: [new.unflatten(L.flatten(v)) for v in vs] for n, vs in L.bases.items()}
    return Layout(L.in_dims, new_dims, bases)


def expand_dims(L, axis, name):
    out = list(L.out_dims)
    out.insert(axis, (name, 0))
    bases = {n: [tuple(v[:axis]) + (0,) + tuple(v[axis:]) for v in vs] for n, vs in L.bases.items()}
    return Layout(L.in_dims, out, bases)


def broadcast(L, axis, bits):
    """The first `bits` zero columns (input order) become the new dim's bits;
    registers are appended for the rest."""
    if L.out_dims[axis][1] != 0:
        raise ValueError("broadcast needs a size-1 dim")
    out = list(L.out_dims)
    out[axis] = (out[axis][0], bits)
    used = 0
    bases = {}
    for n, _ in L.in_dims:
        vs = []
        for v in L.bases[n]:
            if not any(v) and used < bits:
                v = tuple((1 << used) if d == axis else 0 for d in range(len(out)))
                used += 1
            vs.append(tuple(v))
        bases[n] = vs
    in_dims = list(L.in_dims)
    if used < bits:
        extra = [tuple((1 << u) if d == axis else 0 for d in range(len(out))) for u in range(used, bits)]
        if "reg" not in dict(in_dims):
            in_dims.insert(0, ("reg", 0))
            bases["reg"] = []
        bases["reg"] = bases["reg"] + extra
        in_dims = [(n, b + len(extra)) if n == "reg" else (n, b) for n, b in in_dims]
    return Layout(in_dims, out, bases)


def join(L, name):
    out = list(L.out_dims) + [(name, 1)]
    bases = {n: [tuple(v) + (0,) for v in vs] for n, vs in L.bases.items()}
    in_dims = list(L.in_dims)
    if "reg" not in dict(in_dims):
        in_dims.insert(0, ("reg", 0))
        bases["reg"] = []
    bases["reg"] = [tuple(0 for _ in L.out_dims) + (1,)] + bases["reg"]
    in_dims = [(n, b + 1) if n == "reg" else (n, b) for n, b in in_dims]
    return Layout(in_dims, out, bases)


def split(L):
    if L.out_dims[-1][1] != 1:
        raise ValueError("split needs a last dim of size 2")
    holders = [(n, k) for n, vs in L.bases.items() for k, v in enumerate(vs) if v[-1]]
    if len(holders) != 1 or holders[0][0] != "reg":
        raise ValueError("the size-2 dim is not held by one register bit")
    n0, k0 = holders[0]
    if any(L.bases[n0][k0][:-1]):
        raise ValueError("the holding register also moves other coordinates")
    bases = {}
    for n, vs in L.bases.items():
        bases[n] = [tuple(v[:-1]) for k, v in enumerate(vs) if not (n == n0 and k == k0)]
    in_dims = [(n, b - 1) if n == n0 else (n, b) for n, b in L.in_dims]
    return Layout(in_dims, L.out_dims[:-1], bases)


def slice_(L, axis):
    """Sliced layout: "Removing a dimension is a linear map" --
    the output dim ``axis`` is dropped from every basis vector, so the matrix
    loses that dim's rows; columns that only reached it become
    zero."""
    out = [d for i, d in enumerate(L.out_dims) if i != axis]
    bases = {n: [tuple(c for i, c in enumerate(v) if i != axis) for v in vs]
             for n, vs in L.bases.items()}
    return Layout(L.in_dims, out, bases)
