python scripts/ncu_target.py --config C5 --sweeps 1 > gpurun_out/ncu_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fiber_pass -s 0 -c 6 -o gpurun_out/prof2_c5_k2 python scripts/ncu_target.py --config C5 --sweeps 1 > gpurun_out/ncu2_k2.log 2>&1
ls -la gpurun_out | tail -3
