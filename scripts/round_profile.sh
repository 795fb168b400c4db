#!/bin/bash
# Full bench + ncu evidence for profiles/: launch list of the bench command and a --set full
# capture of the top kernels (one plain a2 pass, one tiled a2 pass, the refill).
TAG=${1:-r1}
python bench.py > gpurun_out/bench_full_$TAG.json 2> gpurun_out/bench_full_$TAG.err
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-extras > gpurun_out/bench_short_$TAG.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-extras > gpurun_out/ncu_launches_$TAG.log 2>&1
python scripts/ncu_target.py --config C5 --sweeps 1 > gpurun_out/ncu_plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fiber_pass -s 0 -c 2 -o gpurun_out/full_$TAG python scripts/ncu_target.py --config C5 --sweeps 1 > gpurun_out/ncu_full_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fiber_pass -s 20 -c 1 -o gpurun_out/full_refill_$TAG python scripts/ncu_target.py --config C5 --sweeps 1 >> gpurun_out/ncu_full_$TAG.log 2>&1
ls -la gpurun_out | tail -12
