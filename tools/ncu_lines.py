"""Top source lines by stall samples + stall-reason totals for an ncu report (dev tool)."""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
if rep.endswith(".csv"):   # a saved `--page source --csv --print-source cuda,sass` export
    out = open(rep).read()
else:
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur = None; hdr = None; agg = {}; tot = {}
for r in rows:
    if not r: continue
    if r[0] == 'File Path': cur = r[1].split('/')[-1]; continue
    if r[0] == 'Function Name': continue
    if r[0] == 'Line No': hdr = r; idx = {h: i for i, h in enumerate(hdr)}; continue
    try: ln = int(r[0])
    except ValueError: continue
    if r[2] != '-': continue
    v = agg.setdefault((cur, ln), [0.0, 0.0, r[1][:95]])
    v[0] += float(r[4] or 0); v[1] += float(r[7] or 0)
    for h in hdr:
        if h.startswith('stall_') and '(Not' not in h:
            try: tot[h] = tot.get(h, 0) + float(r[idx[h]] or 0)
            except ValueError: pass
ts = sum(v[0] for v in agg.values()) or 1; ti = sum(v[1] for v in agg.values()) or 1
s = sum(tot.values()) or 1
print("stall reasons:", {k[6:]: round(100 * v / s, 1) for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:7]})
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*v[0]/ts:5.1f}% stall {100*v[1]/ti:5.1f}% inst {k[0]}:{k[1]} {v[2]}")
if len(sys.argv) > 3 and sys.argv[3] == "inst":
    print("-- by instructions")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{100*v[1]/ti:5.1f}% inst {100*v[0]/ts:5.1f}% stall {k[0]}:{k[1]} {v[2]}")
