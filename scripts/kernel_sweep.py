"""Build kernel variants (launch bounds / register caps) and time each on the
GPU: `python scripts/kernel_sweep.py build` here, `... run` on the box."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VAR = os.path.join(ROOT, "paper_2508_15010_b200", "lib", "variants")
VARIANTS = {
    "b3": ["-DTOAST_MAX_THREADS=256", "-DTOAST_MIN_BLOCKS=3"],
    "t128b7": ["-DTOAST_MAX_THREADS=128", "-DTOAST_MIN_BLOCKS=7"],
    "t128b8": ["-DTOAST_MAX_THREADS=128", "-DTOAST_MIN_BLOCKS=8"],
    "t128b7np": ["-DTOAST_MAX_THREADS=128", "-DTOAST_MIN_BLOCKS=7", "-DTOAST_H4_PREFETCH=0"],
    "sigpf": ["-DTOAST_SIG_PREFETCH=1"],
    "smemtab": ["-DTOAST_SMEM_TABLES=1"],
    "stcs": ["-DTOAST_STREAM_STORES=1"],
    "na3b3": ["-DTOAST_NA3_MIN_BLOCKS=3"],
    "na3b4": ["-DTOAST_NA3_MIN_BLOCKS=4"],
}
if os.environ.get("SWEEP_ONLY"):
    VARIANTS = {k: v for k, v in VARIANTS.items() if k in os.environ["SWEEP_ONLY"].split(",")}
KS = [int(k) for k in os.environ.get("SWEEP_KS", "1,2").split(",")]


def build_all():
    from paper_2508_15010_b200 import build as b
    os.makedirs(VAR, exist_ok=True)
    for tag, fl in VARIANTS.items():
        b.build(force=True, lib=os.path.join(VAR, f"libtoast_{tag}.so"), obj=os.path.join(ROOT, "paper_2508_15010_b200", "build", tag), extra=fl)
        print("built", tag, flush=True)


def run_all(config="gpt24", n=1 << 18):
    out = {}
    for tag in VARIANTS:
        for K in KS:
            lib = os.path.join(VAR, f"libtoast_{tag}.so")
            r = subprocess.run([sys.executable, __file__, "one", lib, config, str(n)], capture_output=True, text=True,
                               env=dict(os.environ, TOAST_LIB=lib, TOAST_FORCE_K=str(K)))
            out[f"{tag}K{K}"] = r.stdout.strip().splitlines()[-1] if r.returncode == 0 else ("ERR " + r.stderr[-300:])
            print(f"{tag}K{K}", out[f"{tag}K{K}"], flush=True)
    return out


def one(lib, config, n):
    import torch
    from paper_2508_15010_b200 import toast as T
    from workloads import configs
    c = configs.get(config)
    a = T.build_analysis(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth, cuda_device=0)
    pre = torch.zeros((n, 32), dtype=torch.int16, device="cuda")
    seq = torch.empty_like(pre)
    out = torch.empty((n, 256), dtype=torch.uint8, device="cuda")
    for w in range(3):
        T.rollout_batch(a, pre, 1, w * n, seq, out)
    torch.cuda.synchronize()
    ts = []
    for s in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        T.rollout_batch(a, pre, 1, s * n, seq, out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    print(json.dumps({"config": config, "n": n, "ms": ms, "evals_per_s": n / ms * 1e3}))


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build_all()
    elif sys.argv[1] == "run":
        for cfg in (sys.argv[2:] or ["gpt24"]):
            run_all(cfg)
    else:
        one(sys.argv[2], sys.argv[3], int(sys.argv[4]))
