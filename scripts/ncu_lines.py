"""Summarise an ncu report's source page per CUDA line: warp-stall samples and
executed warp instructions (needs -lineinfo).  python scripts/ncu_lines.py rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = None
agg = {}
cur = None
tot_s = tot_i = 0
for r in rows:
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < len(hdr) - 1:
        continue
    if r[0]:
        cur = (int(r[0]), r[1].strip()[:110])
        continue
    if cur is None:
        continue
    num = lambda x: int(x) if x.strip().isdigit() else 0
    s = num(r[4])
    i = num(r[7])
    a = agg.setdefault(cur, [0, 0])
    a[0] += s
    a[1] += i
    tot_s += s
    tot_i += i
print(f"total samples {tot_s}, warp instructions {tot_i}")
for (ln, src), (s, i) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{ln:5d} {100*s/max(tot_s,1):5.1f}% samp {100*i/max(tot_i,1):5.1f}% inst  {src}")
