#!/bin/bash
# ncu --set full captures of the C5 contraction passes (blocks (0,1)..(1,2), and the plain
# RED1 block (2,3)) and the refill; run from the repo root under gpurun.
TAG=${1:-k2}
python scripts/ncu_target.py --config C5 --sweeps 1 > gpurun_out/ncu_plain_$TAG.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:fiber_pass -s 0 -c 6 -o gpurun_out/${TAG}_a -f python scripts/ncu_target.py --config C5 --sweeps 1 > gpurun_out/ncu_${TAG}_a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fiber_pass -s 10 -c 1 -o gpurun_out/${TAG}_b -f python scripts/ncu_target.py --config C5 --sweeps 1 > gpurun_out/ncu_${TAG}_b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fiber_pass -s 20 -c 1 -o gpurun_out/${TAG}_r -f python scripts/ncu_target.py --config C5 --sweeps 1 > gpurun_out/ncu_${TAG}_r.log 2>&1
ls -la gpurun_out | grep $TAG
for r in a b r; do
  for l in 0 1 2 3 4 5; do
    [ -f gpurun_out/${TAG}_$r.ncu-rep ] || continue
    python scripts/ncu_summary.py gpurun_out/${TAG}_$r.ncu-rep $l > gpurun_out/sum_${TAG}_${r}$l.txt 2>&1
    [ $r != a ] && break
  done
done
ncu -i gpurun_out/${TAG}_a.ncu-rep --page details --csv > gpurun_out/details_${TAG}_a.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_r.ncu-rep --page details --csv > gpurun_out/details_${TAG}_r.csv 2>/dev/null
rm -f gpurun_out/${TAG}_b.ncu-rep gpurun_out/${TAG}_r.ncu-rep
