"""Instruction and stall share per source-line range of one file in an ncu report (dev tool).
usage: ncu_ranges.py REPORT FILE name:a-b [name:a-b ...]"""
import csv, io, subprocess, sys
rep, fname = sys.argv[1], sys.argv[2]
ranges = []
for spec in sys.argv[3:]:
    name, ab = spec.split(":")
    a, b = ab.split("-")
    ranges.append((name, int(a), int(b)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur = None; agg = {}
for r in rows:
    if not r: continue
    if r[0] == 'File Path': cur = r[1].split('/')[-1]; continue
    try: ln = int(r[0])
    except ValueError: continue
    if r[2] != '-': continue
    v = agg.setdefault((cur, ln), [0.0, 0.0])
    v[0] += float(r[4] or 0); v[1] += float(r[7] or 0)
ts = sum(v[0] for v in agg.values()) or 1; ti = sum(v[1] for v in agg.values()) or 1
seen = 0.0
for name, a, b in ranges:
    st = sum(v[0] for k, v in agg.items() if k[0] == fname and a <= k[1] <= b)
    it = sum(v[1] for k, v in agg.items() if k[0] == fname and a <= k[1] <= b)
    seen += it
    print(f"{name:14s} {a:5d}-{b:<5d} stall {100*st/ts:5.1f}%  inst {100*it/ti:5.1f}%  ({it:.3g} inst)")
print(f"other: inst {100*(ti-seen)/ti:5.1f}%  total {ti:.3g}")
