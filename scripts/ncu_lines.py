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
tot_st = {}
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
    a = agg.setdefault(cur, [0, 0, {}])
    a[0] += s
    a[1] += i
    for ci, name in enumerate(hdr):
        if name.startswith("stall_") and "Not Issued" not in name and ci < len(r):
            a[2][name[6:]] = a[2].get(name[6:], 0) + num(r[ci])
            tot_st[name[6:]] = tot_st.get(name[6:], 0) + num(r[ci])
    tot_s += s
    tot_i += i
print(f"total samples {tot_s}, warp instructions {tot_i}")
print("stalls:", ", ".join(f"{k} {100*v/max(tot_s,1):.1f}%" for k, v in sorted(tot_st.items(), key=lambda kv: -kv[1])[:8]))
for (ln, src), (s, i, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    top2 = ",".join(f"{k}:{v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:2])
    print(f"{ln:5d} {100*s/max(tot_s,1):5.1f}% samp {100*i/max(tot_i,1):5.1f}% inst  [{top2:28s}] {src[:80]}")
