#!/bin/bash
# usage: bash scripts/l2_check.sh TAG — quick loop for the small-config work: the L2-pass and
# parity tests, graph-replayed µs/sweep of C1–C4/C2r (default vs the streaming walk), and the
# per-block launch times of C2/C3/C4.
TAG=${1:-x}
python -m pytest tests/test_gpu_l2pass.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -15 > gpurun_out/l2tests_$TAG.log
tail -4 gpurun_out/l2tests_$TAG.log
python scripts/ab_flags.py C1,C2,C3,C4,C2r 0,128 1 2>&1 | tee gpurun_out/l2ab_$TAG.log
for c in C2 C3 C4; do python scripts/block_split.py $c; done 2>&1 | tee gpurun_out/l2blocks_$TAG.log
