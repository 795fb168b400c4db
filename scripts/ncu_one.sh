#!/bin/bash
# usage: bash scripts/ncu_one.sh TAG CONFIG KERNEL_REGEX [SKIP]  — one --set full capture,
# summarised on the box (raw metrics + source hot spots + stall reasons), report deleted.
TAG=$1; CFG=$2; RX=$3; SKIP=${4:-0}
python scripts/ncu_target.py --config $CFG --sweeps 1 > gpurun_out/ncu_plain_$TAG.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"$RX" -s $SKIP -c 1 -o gpurun_out/$TAG -f \
    python scripts/ncu_target.py --config $CFG --sweeps 1 > gpurun_out/ncu_$TAG.log 2>&1
python scripts/ncu_summary.py gpurun_out/$TAG.ncu-rep 0 > gpurun_out/sum_$TAG.txt 2>&1
ncu -i gpurun_out/$TAG.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; d=dict(zip(h,rows[2]))
st=sorted(((int(float(v)),k.replace('smsp__pcsamp_warps_issue_stalled_','')) for k,v in d.items()
          if k.startswith('smsp__pcsamp_warps_issue_stalled') and not k.endswith('not_issued') and v not in ('','0')), reverse=True)
print('stalls', st[:10])
for k in ('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active','smsp__issue_active.avg.pct_of_peak_sustained_active',
          'sm__warps_active.avg.pct_of_peak_sustained_active','gpu__time_duration.sum','launch__grid_size','launch__block_size',
          'smsp__inst_executed.sum','sm__cycles_active.avg'):
    print(k, d.get(k))
" >> gpurun_out/sum_$TAG.txt 2>&1
rm -f gpurun_out/$TAG.ncu-rep
