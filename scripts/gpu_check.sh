#!/bin/bash
# usage: bash scripts/gpu_check.sh TAG  — GPU tests + bench, logs under gpurun_out/
TAG=${1:-x}
python -m pytest tests -m gpu -q -p no:cacheprovider --maxfail=20 2>&1 | tail -40 > gpurun_out/tests_$TAG.log
python bench.py ${BENCH_ARGS} > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -3 gpurun_out/tests_$TAG.log
python - << PY
import json
d=json.load(open('gpurun_out/bench_$TAG.json'))
print('value', d['value'], 'ms/step', d['ms_per_step'], 'k2 frac', d['roofline']['frac'], 'refill frac', d['refill']['frac'])
print('kernels', d['kernels_ms_per_sweep'])
for k,v in d.get('other_configs',{}).items(): print(k, round(v['us_per_sweep'],1), 'us/sweep')
PY
