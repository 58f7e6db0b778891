"""CPU oracle for Linear Layouts (arXiv 2505.23819) -- TEST INFRASTRUCTURE ONLY.

This package is the plain, slow, obviously-correct reference that the CUDA path
is checked against.  It is *not* part of the product:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import it;
* it shares no code with ``paper_2505_23819_b200`` (neither imports the other);
  the only common module is ``workloads`` (seeded inputs + literal layout
  tables, no layout arithmetic).

Citations ``P:n`` are lines of the paper's LaTeX source, with the
section / equation they fall in.  Every function states the passage it follows.

Modules
-------
f2           F2 vectors and matrices: product, rank, span, Gauss-Jordan right
             inverse.
layout       Labeled linear layouts: apply, compose, product, left division,
             right inverse, predicates.
constructors identity tiles, blocked (Appendix), mma tiles
             (Appendix, reading A8), mma swizzling (Def. 5,
             P:435-463).
convert      element-by-element layout conversion and gather (P:599-611,
             P:719-727) -- the plain definition.
banks        brute-force shared-memory bank / wavefront counter (P:679-689,
             Appendix lemma).
swizzle      the paper's optimal swizzling construction step by step
             (Appendix) + brute-force optimum.
shuffle      the paper's warp-shuffle construction V, I, E, F, G, R
              + a round-by-round simulator.
contig       contiguity / vector width.

Parity status of each function is recorded in DESIGN.md ("oracle pins").
"""
