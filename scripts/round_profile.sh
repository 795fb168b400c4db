#!/bin/bash
# Evidence for profiles/<TAG>/ (run from the repo root under gpurun, one GPU):
#   1. full bench line (stdout JSON) and its stderr
#   2. ncu launch list of the short bench command (gpu__time_duration per launch)
#   3. ncu --set full of every launch of one plain-launch C5 sweep (20 a2 passes, reduces,
#      solves, refill) -> per-kernel raw metrics + source hot spots of the top kernels;
#      the .ncu-rep files are summarised on the box and deleted (size cap on gpurun_out/)
TAG=${1:-r1}
OUT=gpurun_out/prof_$TAG
mkdir -p $OUT
python bench.py > $OUT/bench_full.json 2> $OUT/bench_full.err
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-extras > $OUT/bench_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-extras > $OUT/ncu_launches.log 2>&1
python scripts/launch_summary.py $OUT/launches.csv > $OUT/launches.txt 2>&1
python scripts/ncu_target.py --config C5 --sweeps 1 > $OUT/ncu_target_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fiber_pass|reduce_partials|block_solve|finalize" \
    -c 62 -o $OUT/sweep -f python scripts/ncu_target.py --config C5 --sweeps 1 > $OUT/ncu_sweep.log 2>&1
python scripts/ncu_summary.py $OUT/sweep.ncu-rep 0 > $OUT/ncu_sweep_summary.txt 2>&1
python scripts/ncu_per_launch.py $OUT/sweep.ncu-rep > $OUT/ncu_sweep_per_launch.txt 2>&1
# source hot spots of: the first tiled pass, the first plain pass, the first solve, the refill
PICK=$(python - "$OUT/ncu_sweep_per_launch.txt" << 'PY'
import sys
rows = [l.split() for l in open(sys.argv[1]) if l[:4].strip().isdigit()]
def first(pred):
    for r in rows:
        if pred(r[1] + " " + r[2]):
            return r[0]
    return None
picks = [first(lambda n: n.startswith("fiber_pass_vb")), first(lambda n: n.startswith("fiber_pass<") and "2," not in n),
         first(lambda n: n.startswith("block_solve")), first(lambda n: n.startswith("fiber_pass<float, 2"))]
print(" ".join(p for p in picks if p is not None))
PY
)
for l in $PICK; do
  python scripts/ncu_summary.py $OUT/sweep.ncu-rep $l > $OUT/ncu_src_launch$l.txt 2>&1
done
rm -f $OUT/sweep.ncu-rep
ls -la $OUT
