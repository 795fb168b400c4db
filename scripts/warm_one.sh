#!/bin/bash
# usage: bash scripts/warm_one.sh OUT CFG[,CFG..] — warm-cache per-kernel durations (ncu, --cache-control none)
# of graph-free sweeps, printed as a per-launch table of the last sweep
OUT=${1:-gpurun_out}; mkdir -p $OUT
for CFG in ${2//,/ }; do
  ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv \
      --log-file $OUT/warm_$CFG.csv python scripts/ncu_target.py --config $CFG --sweeps 3 > $OUT/warm_$CFG.log 2>&1
  python - $OUT/warm_$CFG.csv $CFG <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0].isdigit()]
per = len(rows) // 3
tot = 0.0
print("==", sys.argv[2], per, "launches per sweep")
for r in rows[-per:]:
    t = float(r[-1].replace(",", "")) / 1000.0
    tot += t
    print(f"  {r[4].split('(')[0][:44]:44s} grid {r[8]:14s} {t:7.2f} us")
print(f"  sum {tot:.1f} us")
PY
done
