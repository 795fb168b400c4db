#!/bin/bash
# ncu --set full capture of the fused refill+contraction pass (C5, 2 plain-launch sweeps).
TAG=${1:-fz}
python scripts/ncu_target.py --config C5 --sweeps 2 > gpurun_out/ncu_plain_$TAG.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"fiber_pass_vb<float, \(int\)5" -c 1 -o gpurun_out/${TAG} -f python scripts/ncu_target.py --config C5 --sweeps 2 > gpurun_out/ncu_${TAG}.log 2>&1
python scripts/ncu_summary.py gpurun_out/${TAG}.ncu-rep 0 > gpurun_out/sum_${TAG}.txt 2>&1
ncu -i gpurun_out/${TAG}.ncu-rep --page details --csv > gpurun_out/details_${TAG}.csv 2>/dev/null
