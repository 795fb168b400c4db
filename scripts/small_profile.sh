#!/bin/bash
# usage: bash scripts/small_profile.sh OUTDIR — `ncu --set full` of every launch of one
# plain-launch sweep of C1–C4 (per-kernel DRAM/L2/pipe figures for each config),
# summarised on the box with ncu_per_launch.py + ncu_summary.py; the .ncu-rep files are deleted.
OUT=${1:-gpurun_out}
mkdir -p $OUT
for CFG in C1 C2 C3 C4; do
  python scripts/ncu_target.py --config $CFG --sweeps 1 > $OUT/ncu_target_$CFG.log 2>&1 || exit 1
  ncu --set full --clock-control none -k regex:"fiber_pass|reduce_partials|block_solve|finalize" \
      -c 64 -o $OUT/sweep_$CFG -f python scripts/ncu_target.py --config $CFG --sweeps 1 > $OUT/ncu_$CFG.log 2>&1
  python scripts/ncu_per_launch.py $OUT/sweep_$CFG.ncu-rep > $OUT/ncu_${CFG}_per_launch.txt 2>&1
  ncu -i $OUT/sweep_$CFG.ncu-rep --page raw --csv --print-units base 2>/dev/null | python -c "
import csv, sys, re
rows = list(csv.reader(sys.stdin)); h = rows[0]
keys = ['gpu__time_duration.sum', 'lts__t_bytes.sum', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'dram__bytes_read.sum', 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active']
print('#', 'kernel', *[k.split('.')[0] for k in keys])
for i, r in enumerate(rows[2:]):
    d = dict(zip(h, r))
    print(i, re.sub(r'\(.*', '', d['Kernel Name']).replace('void ', '')[:40], *[d.get(k, '') for k in keys])
" > $OUT/ncu_${CFG}_l2_pipes.txt 2>&1
  rm -f $OUT/sweep_$CFG.ncu-rep
done
