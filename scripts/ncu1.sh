set -x
python scripts/ncu_target.py --config C5 --sweeps 1 > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fiber_pass -s 0 -c 6 -o gpurun_out/prof_c5_k2 python scripts/ncu_target.py --config C5 --sweeps 1 > gpurun_out/ncu_k2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fiber_pass -s 20 -c 1 -o gpurun_out/prof_c5_refill python scripts/ncu_target.py --config C5 --sweeps 1 > gpurun_out/ncu_refill.log 2>&1
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-extras > gpurun_out/bench_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-extras > gpurun_out/ncu_launches.log 2>&1
ls -la gpurun_out/
