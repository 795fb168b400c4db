#!/bin/bash
# usage: bash scripts/kept_fixed_cost.sh CFG — ncu warm durations of the l2_kept launches for the
# experiment builds that skip the main loop and/or the table staging (results are wrong there:
# timing only): exp/nomain.so, exp/nostage.so, exp/noboth.so (scripts/variants.sh)
CFG=${1:-C3}
for lib in default nomain nostage noboth; do
  if [ "$lib" != default ]; then export IFCTN_LIB=$PWD/exp/$lib.so; else unset IFCTN_LIB; fi
  ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv -k regex:l2_kept \
      --log-file gpurun_out/fc_$lib.csv python scripts/ncu_target.py --config $CFG --sweeps 2 > /dev/null 2>&1
  python - gpurun_out/fc_$lib.csv $lib <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0].isdigit()]
h = len(rows) // 2
print(f"{sys.argv[2]:8s}", " ".join(f"{float(r[-1].replace(',', '')) / 1000:6.2f}" for r in rows[h:]))
PY
done
