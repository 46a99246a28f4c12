"""Summarise an ncu --set full capture of the rollout kernel into profiles/:
    python scripts/ncu_summary.py <config> <report.ncu-rep> [round-tag]
writes profiles/<tag>_ncu_<config>.txt (the headline metrics) and updates
profiles/ncu_summary.json[config] (read by bench.py for roofline.traffic)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfg, rep = sys.argv[1], sys.argv[2]
tag = sys.argv[3] if len(sys.argv) > 3 else "r01"

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
M = {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def num(name, scale=1.0):
    v, u = M[name]
    x = float(v.replace(",", ""))
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3,
            "second": 1.0}.get(u, 1.0)
    return x * mult * scale


keys = {
    "kernel": "Kernel Name", "block": "Block Size", "grid": "Grid Size",
}
out = {k: M[v][0] for k, v in keys.items() if v in M}
rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
dur = num("gpu__time_duration.sum")
out.update({
    "duration_s": dur,
    "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
    "issue_active_pct": float(M["smsp__issue_active.avg.pct_of_peak_sustained_active"][0]),
    "warp_inst_executed": float(M["smsp__inst_executed.sum"][0].replace(",", "")),
    "ipc": float(M["sm__inst_executed.avg.per_cycle_active"][0]),
    "warps_active_pct": float(M["sm__warps_active.avg.pct_of_peak_sustained_active"][0]),
    "registers": int(float(M["launch__registers_per_thread"][0])),
    "smem_wavefronts": float(M["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"][0].replace(",", "")),
    "alu_pipe_pct": float(M["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"][0]),
    "fma_pipe_pct": float(M["sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"][0]),
    "lsu_pipe_pct": float(M["sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"][0]),
    "thread_inst_per_inst": float(M["smsp__thread_inst_executed_per_inst_executed.ratio"][0]),
    "theoretical_occupancy_pct": float(M["sm__maximum_warps_per_active_cycle_pct"][0]),
    "occupancy_limit_registers": float(M["launch__occupancy_limit_registers"][0]),
    "occupancy_limit_shared_mem": float(M["launch__occupancy_limit_shared_mem"][0]),
    "report": os.path.basename(rep), "round": tag,
})
# evaluations in the captured launch: the bench line of the same run (plain_<cfg>.log)
try:
    plain = os.path.join(os.path.dirname(rep), f"plain_forced_{cfg}.log")
    if not os.path.exists(plain):
        plain = os.path.join(os.path.dirname(rep), f"plain_{cfg}.log")
    line = json.loads(open(plain).read().strip().splitlines()[-1])
    out["evals_per_launch"] = line["config"]["rollouts_per_step_per_gpu"]
    out["warps_per_batch"] = line["config"].get("warps_per_batch")
except Exception:
    pass
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
p = os.path.join(ROOT, "profiles", "ncu_summary.json")
allp = json.load(open(p)) if os.path.exists(p) else {}
allp[cfg] = out
json.dump(allp, open(p, "w"), indent=1, sort_keys=True)
with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_{cfg}.txt"), "w") as f:
    det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
    f.write(det)
    f.write("\n# summary\n" + json.dumps(out, indent=1) + "\n")
print(json.dumps(out, indent=1))
