"""Summarise an ncu report: key raw metrics per kernel and top source lines of one launch."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
launch = int(sys.argv[2]) if len(sys.argv) > 2 else 0
WANT = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__registers_per_thread',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__grid_size',
        'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'lts__t_bytes.sum', 'l1tex__t_bytes.sum']
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print({w.split('__')[-1] if '__' in w else w: d.get(w) for w in WANT})
src = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source=cuda,sass',
                      '--launch-skip', str(launch), '--launch-count', '1'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
cur, hdr, agg = None, None, []
for r in rows:
    if len(r) == 2 and r[0] in ('File Path', 'File Name'):
        cur = r[1]
        continue
    if len(r) >= 2 and r[0] == 'Line No':
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or r[0] == '':
        continue
    d = dict(zip(hdr, r))
    try:
        ie = int(d['Instructions Executed'] or 0)
        st = int(d['Warp Stall Sampling (All Samples)'] or 0)
    except Exception:
        continue
    agg.append((ie, st, cur.split('/')[-1], r[0], r[1][:100]))
tot = sum(a[0] for a in agg) or 1
tots = sum(a[1] for a in agg) or 1
print('launch', launch, 'warp-inst', tot, 'stall samples', tots)
for a in sorted(agg, key=lambda a: -a[int(sys.argv[3]) if len(sys.argv) > 3 else 1])[:int(sys.argv[4]) if len(sys.argv) > 4 else 25]:
    print(f"{a[0]:>10} {100*a[0]/tot:5.1f}% stall{100*a[1]/tots:5.1f}% {a[2]}:{a[3]} {a[4]}")
