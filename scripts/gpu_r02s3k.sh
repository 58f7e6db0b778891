#!/bin/bash
# Upcast PDL A/B, all-CTA prefetch for short launches (shard projection),
# parity tests of both.
O=gpurun_out/r02s3k
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "upcast or hint_and_order or shard" > $O/pytest.txt 2>&1
timeout 900 python scripts/ab_upcast_pdl.py > $O/ab_upcast_pdl.jsonl 2> $O/ab.err
timeout 600 python scripts/shard_projection.py "" > $O/proj_default.jsonl 2>> $O/ab.err
timeout 600 python scripts/shard_projection.py "pdl_prefetch_short=0" > $O/proj_noshort.jsonl 2>> $O/ab.err
echo done > $O/done.txt
