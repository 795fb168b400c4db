for c in 0 1; do
  IFCTN_TUNE_CTAS=$c python bench.py --no-cpu --no-e2e --no-extras > gpurun_out/tune_$c.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/tune_$c.json')); print('ctas', $c, round(d['value'],2), round(d['roofline']['frac'],3), round(d['refill']['frac'],3), d['a2_ms_by_block'])"
done
