python scripts/ncu_target.py --config C5 --sweeps 1 > gpurun_out/ncu_plain5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fiber_pass -s 0 -c 2 -o gpurun_out/prof5_c5_k2 python scripts/ncu_target.py --config C5 --sweeps 1 > gpurun_out/ncu5_k2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fiber_pass -s 20 -c 1 -o gpurun_out/prof5_c5_refill python scripts/ncu_target.py --config C5 --sweeps 1 > gpurun_out/ncu5_refill.log 2>&1
