"""Time-to-best-partition: GPU toast_search vs the CPU oracle search.

1. S*: the best score a long GPU search finds under a fixed evaluation budget
   (patience disabled), re-evaluated bit-exactly by the oracle; for mlp_c,
   S* = the brute-force optimum (C17).
2. GPU: the same search with target S* -> wall time to the first round whose
   best <= S*.
3. CPU: the oracle's search (same C16 spec, same seed -> the same trajectory)
   on all host cores with target S* and a time limit; if it does not get there,
   the ratio is reported as a lower bound.

    python scripts/time_to_best.py --config gpt24 [--budget 20000000] [--cpu-seconds 120]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(config="gpt24", budget=20_000_000, cpu_seconds=120.0, L=64, R=256, seed=0, device=0):
    import numpy as np
    import torch
    from oracle.oracle import Oracle
    from paper_2508_15010_b200 import toast as T
    from workloads import configs

    c = configs.get(config)
    torch.cuda.set_device(device)
    a = T.build_analysis(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth, cuda_device=device)
    o = Oracle(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth)
    big = 1 << 62
    if config == "mlp_c":
        _, best_seq, best = o.bruteforce()
        s_star = float(best["score"])
        s_star_src = "brute-force optimum (C17)"
    else:
        r = T.search(a, T.SearchOptions(seed=seed, max_evals=budget, leaves_per_round=L, rollouts_per_leaf=R,
                                        patience=big >> 32))
        s_star = float(r["best"]["score"])
        best_seq = np.array(r["best_seq"], dtype=np.uint16)
        s_star_src = f"best of a {int(r['evals'])}-eval GPU search (seed {seed}, L={L}, R={R})"
    # the oracle re-evaluates the target state bit-exactly
    oc = o.eval(best_seq.reshape(1, 32))[0]
    assert oc["score"] == s_star, (oc["score"], s_star)
    opts = T.SearchOptions(seed=seed, max_evals=budget, leaves_per_round=L, rollouts_per_leaf=R, patience=big >> 32,
                           target_score=s_star)
    g = T.search(a, opts)
    gpu_t = float(g["time_to_target_s"])
    gpu_evals = int(g["evals"])
    cores = os.cpu_count() or 1
    ro, trace = o.search(seed=seed, max_evals=budget, time_limit_s=cpu_seconds, L=L, R=R, patience=big >> 32,
                         target_score=s_star, threads=cores)
    cpu_hit = bool(ro["hit_target"])
    cpu_t = float(ro["time_to_target_s"]) if cpu_hit else float(ro["wall_s"])
    cpu_rate = int(ro["evals"]) / max(float(ro["wall_s"]), 1e-9)
    out = {
        "config": config, "target_score": s_star, "target_source": s_star_src,
        "search": {"leaves_per_round": L, "rollouts_per_leaf": R, "seed": seed, "budget_evals": budget},
        "gpu": {"time_to_target_s": gpu_t, "hit": bool(g["hit_target"]), "evals": gpu_evals, "rounds": int(g["rounds"])},
        "cpu_oracle": {"time_to_target_s": cpu_t if cpu_hit else None, "hit": cpu_hit, "evals": int(ro["evals"]),
                       "wall_s": float(ro["wall_s"]), "cores": cores, "evals_per_s": cpu_rate,
                       "extrapolated_time_to_target_s": gpu_evals / cpu_rate},
        "speedup": (cpu_t / gpu_t) if cpu_hit else None,
        "speedup_lower_bound": None if cpu_hit else cpu_t / gpu_t,
        "speedup_extrapolated": (gpu_evals / cpu_rate) / gpu_t if gpu_t > 0 else None,
    }
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="gpt24")
    ap.add_argument("--budget", type=int, default=20_000_000)
    ap.add_argument("--cpu-seconds", type=float, default=120.0)
    ap.add_argument("--L", type=int, default=64)
    ap.add_argument("--R", type=int, default=256)
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    print(json.dumps(run(a.config, a.budget, a.cpu_seconds, a.L, a.R, a.seed)))
