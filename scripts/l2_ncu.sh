#!/bin/bash
# usage: bash scripts/l2_ncu.sh OUT CFG [REGEX] — warm-cache `ncu --set full` of the L2-pass (or REGEX)
# kernels of the second plain-launch sweep of CFG: duration, activity, L1/L2 throughput, stalls
OUT=${1:-gpurun_out}; CFG=${2:-C3}; RX=${3:-l2_}
mkdir -p $OUT
ncu --set full --cache-control none --clock-control none --import-source on -k regex:"$RX" -c 40 -o $OUT/l2ncu_$CFG -f \
    python scripts/ncu_target.py --config $CFG --sweeps 2 > $OUT/l2ncu_$CFG.log 2>&1
ncu -i $OUT/l2ncu_$CFG.ncu-rep --page raw --csv --print-units base 2>/dev/null | python -c "
import csv, sys, re
rows = list(csv.reader(sys.stdin)); h = rows[0]
half = (len(rows) - 2) // 2
for i, r in enumerate(rows[2 + half:]):
    d = dict(zip(h, r))
    f = lambda k: float(d.get(k) or 0)
    name = re.sub(r'\(.*', '', d['Kernel Name']).replace('void ', '').replace('ifctn::', '')
    el = f('sm__cycles_elapsed.avg')
    print(f\"{i:2d} {name[:22]:22s} grid {d['Grid Size']:14s} {f('gpu__time_duration.sum')/1e3:6.2f} us regs {d.get('launch__registers_per_thread','')} \"
          f\"act {100*f('sm__cycles_active.avg')/el:4.0f}% issue {f('smsp__issue_active.avg.pct_of_peak_sustained_active'):4.1f}% \"
          f\"warps {f('sm__warps_active.avg.pct_of_peak_sustained_active'):4.1f}% \"
          f\"L1 {f('l1tex__throughput.avg.pct_of_peak_sustained_active'):4.1f}% L2 {f('lts__throughput.avg.pct_of_peak_sustained_elapsed'):4.1f}% \"
          f\"ltsMB {f('lts__t_bytes.sum')/1e6:6.1f} dramMB {f('dram__bytes_read.sum')/1e6:5.1f} \"
          f\"l1hit {f('l1tex__t_sector_hit_rate.pct'):4.1f}\")
    st = sorted(((float(v or 0), k) for k, v in d.items() if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio')), reverse=True)[:4]
    print('     stalls:', ', '.join(f\"{k.split('stalled_')[1].split('_per_')[0]} {v:.1f}\" for v, k in st))
" > $OUT/l2ncu_$CFG.txt 2>&1
cat $OUT/l2ncu_$CFG.txt
