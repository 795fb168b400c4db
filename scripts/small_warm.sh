#!/bin/bash
# usage: bash scripts/small_warm.sh OUTDIR — warm-cache per-kernel durations of graph-replayed
# sweeps of C1–C4 (ncu --cache-control none: L2 keeps the working set, as in the bench), to
# split each config's µs/sweep into kernel time and launch gaps.
OUT=${1:-gpurun_out}
mkdir -p $OUT
for CFG in C1 C2 C3 C4 C2r; do
  ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv \
      --log-file $OUT/warm_$CFG.csv python scripts/ncu_target.py --config $CFG --sweeps 3 > $OUT/warm_$CFG.log 2>&1
done
