"""Per-region totals of an ncu source page (warp-stall samples, executed warp
instructions): python scripts/ncu_regions.py rep 'name:lo-hi,name:lo-hi,...'"""
import csv, io, subprocess, sys
rep, spec = sys.argv[1], sys.argv[2]
regs = []
for part in spec.split(","):
    n, r = part.split(":")
    lo, hi = r.split("-")
    regs.append((n, int(lo), int(hi)))
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = None; cur = None; agg = {}; ts = ti = 0
num = lambda x: int(x) if x.strip().isdigit() else 0
for r in rows:
    if len(r) > 4 and r[0] == "Line No":
        hdr = r; continue
    if not hdr or len(r) < len(hdr) - 1:
        continue
    if r[0]:
        cur = int(r[0]); continue
    if cur is None:
        continue
    name = next((n for n, lo, hi in regs if lo <= cur <= hi), "other")
    a = agg.setdefault(name, [0, 0])
    a[0] += num(r[4]); a[1] += num(r[7]); ts += num(r[4]); ti += num(r[7])
for n, (s, i) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{n:14s} {100*s/ts:5.1f}% samples {100*i/ti:5.1f}% inst  {i:,}")
