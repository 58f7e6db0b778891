"""B200-native Linear Layouts (arXiv 2505.23819): Python binding of libll_b200.so.

A thin ctypes layer over the C ABI declared in ``include/ll.h``: argument
marshalling only.  Every step of a conversion or gather runs in the library
(host planner in C++, data movement in sm_100a kernels).  There is no CPU or
PyTorch fallback: if the shared library is missing the import fails loudly.

    import paper_2505_23819_b200 as ll
    A = ll.Layout(in_dims, out_dims, bases)       # per-dimension bases
    ll.convert(src, A, dst, B, elem_bits=16)      # device tensors (torch)
"""

from ._lib import (LLError, Layout, broadcast, checksum, compose, convert, convert_host, convert_host_shard, convert_regs_timed,
                   convert_shard, jit_source, left_divide,
                   expand_dims, join, mxfp4_upcast, reshape, shard_describe, shard_describe_2d, gather_host, split, transpose, gather, gather_describe,
                   invert, launch_count, lib_path, plan_describe, product, tune, version, PATHS,
                   gather_jit_source, gather_timed, slice_layout, blocked, mma_tile, mxfp4_scale_layout)

__all__ = ["LLError", "Layout", "broadcast", "checksum", "compose", "convert", "convert_host", "convert_host_shard",
           "convert_regs_timed", "convert_shard", "jit_source", "left_divide",
           "expand_dims", "join", "mxfp4_upcast", "reshape", "split", "transpose",
           "shard_describe", "shard_describe_2d", "gather_host", "gather", "gather_describe",
           "invert", "launch_count", "lib_path", "plan_describe", "product", "tune", "version",
           "PATHS", "gather_jit_source", "gather_timed", "slice_layout", "blocked", "mma_tile", "mxfp4_scale_layout"]
