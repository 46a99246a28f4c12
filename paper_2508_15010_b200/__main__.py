"""Partition a program with the GPU search ("find a sequence of sharding
decisions"): toast_nda, toast_search on one GPU, then the best state's cost
record and its device-local program (toast_lower, Fig. 2c / 5b notation).

    python -m paper_2508_15010_b200 --ir prog.ir --mesh data=8:5e10,model=4:9e11
    python -m paper_2508_15010_b200 --config gpt24 --cost-model cp --grouping contraction

Machine defaults are the B200-class target of SURVEY §8(d)."""
from __future__ import annotations

import argparse
import sys

from . import toast as T


def _mesh(spec: str):
    axes = []
    for item in spec.split(","):
        name, rest = item.split("=")
        size, bw = rest.split(":")
        axes.append((name, int(size), float(bw)))
    return axes


def main(argv=None) -> int:
    p = argparse.ArgumentParser(prog="python -m paper_2508_15010_b200", description=__doc__.split("\n\n")[0])
    src = p.add_mutually_exclusive_group(required=True)
    src.add_argument("--ir", help="text-IR file (include/toast.h toast_load_graph)")
    src.add_argument("--config", help="a built-in workload (workloads/configs.py: gpt24, unet, gns16, llama80, ...)")
    p.add_argument("--mesh", help="name=size:bytes_per_sec,... in mesh order (required with --ir)")
    p.add_argument("--flops", type=float, default=2.25e15, help="matmul-class FLOP/s")
    p.add_argument("--dm", type=float, default=180e9, help="device memory bytes (DM)")
    p.add_argument("--penalty", type=float, default=100.0, help="memory penalty C")
    p.add_argument("--min-dims", type=int, default=10, help="P:1417 minimum value dims per super-color")
    p.add_argument("--cost-model", choices=["sum", "cp"], default="sum", help="G14 straight-line sum or R22 critical path")
    p.add_argument("--grouping", choices=["compat", "contraction"], default="compat", help="C4/C5 or R23")
    p.add_argument("--dedup", action="store_true", help="cost each distinct state of a rollout launch once (NEXT-3)")
    p.add_argument("--transpositions", action="store_true", help="each materialised state once in the tree (R24)")
    p.add_argument("--budget", type=int, default=2_000_000, help="evaluations")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--no-program", action="store_true", help="do not print the lowered program")
    args = p.parse_args(argv)

    if args.config:
        import os
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from workloads import configs
        c = configs.get(args.config)
        ir, axes, flops, dm, pen, min_dims = c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims
    else:
        if not args.mesh:
            p.error("--mesh is required with --ir")
        ir = open(args.ir).read()
        axes, flops, dm, pen, min_dims = _mesh(args.mesh), args.flops, int(args.dm), args.penalty, args.min_dims
    a = T.build_analysis(ir, axes, flops, int(dm), pen, min_dims, 30, cuda_device=0,
                         cost_model=T.COST_CRITICAL_PATH if args.cost_model == "cp" else T.COST_SUM,
                         grouping=T.GROUP_CONTRACTION if args.grouping == "contraction" else T.GROUP_COMPAT,
                         dedup=T.DEDUP_ON if args.dedup else T.DEDUP_AUTO)
    acts = a.actions()
    r = T.search(a, T.SearchOptions(seed=args.seed, max_evals=args.budget, patience=1 << 30,
                                    transpositions=int(args.transpositions)))
    best = r["best"]
    seq = [int(x) for x in r["best_seq"] if x]
    print(f"evaluations {int(r['evals'])} in {int(r['rounds'])} rounds, {float(r['wall_s']) * 1e3:.2f} ms")
    print(f"best score {float(best['score']):.6g} (runtime {float(best['runtime_s']):.6g} s, "
          f"peak {int(best['peak_bytes'])} B, baseline runtime {float(a.baseline()['runtime_s']):.6g} s)")
    print("actions: " + (", ".join(f"#{i}(super-color {acts[i][0]}, r={acts[i][1]}, axis {axes[acts[i][2]][0]})"
                                    for i in seq) or "none (the unsharded program is best)"))
    if not args.no_program:
        print(T.lower(a, seq))
    return 0


if __name__ == "__main__":
    sys.exit(main())
