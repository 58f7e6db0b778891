"""Seeded synthetic inputs shared by the oracle side and the product side.

This is the ONLY module both sides import.  It holds no layout arithmetic:
``values`` is a counter-based hash (splitmix64) that fills buffers, and
``configs`` lists the five BASELINE.json workloads as literal tables of basis
vectors (taken from SURVEY.md 8(d)), in the C-ABI's bases format.  Whether a
table really is "mma C fragment" or "blocked [1,8]x[2,16]x[4,1]" is checked by
tests against the oracle's constructors and the PTX fragment formulas.
"""
