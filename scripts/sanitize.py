"""Drive every kernel instantiation the parity suite uses, small, under a
checking tool:

    TOAST_LIB=paper_2508_15010_b200/lib/libtoast_checked.so python scripts/sanitize.py

The checked library (kernels.cu TOAST_CHECKED) bounds-checks every shared-memory
access and table index (a violation traps), poisons every region the moment it
dies and sleeps pseudo-random times at every barrier and cross-lane exchange,
so a race or a stale read breaks the bit-exact comparison below.  (The same
driver runs under compute-sanitizer — `compute-sanitizer --tool racecheck
--kernel-name kns=toast_ python scripts/sanitize.py` — where it is available;
this pool's GPU boxes refuse it.)

Per config (1-4 axes, power-of-two and not) x cost model (sum, critical path)
x K in {1, 2, 4, 8} warps per batch (TOAST_FORCE_K, read when the analysis is
built): one rollout launch and one eval launch of a ragged batch (3 full
batches + a 13-candidate tail), full 256-B and compact 16-B records.  The
results are also compared with the oracle (test infrastructure), so a run
that is hazard-free is also a parity run of every instantiation.
"""
from __future__ import annotations

import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle.oracle import Oracle  # noqa: E402
from workloads import configs  # noqa: E402

CONFIGS = ["mlp_c", "attn_toy", "gpt2", "gpt2_np2", "gpt2_3ax", "gpt2_3ax_np2", "gpt2_4ax", "gpt2_4ax_np2"]


def main():
    from paper_2508_15010_b200 import toast as T
    quick = "--quick" in sys.argv
    names = [a for a in sys.argv[1:] if not a.startswith("--")] or CONFIGS
    n = 32 * 3 + 13
    ks = (1, 8) if quick else (1, 2, 4, 8)
    torch.cuda.set_device(0)
    done = 0
    for name in names:
        c = configs.get(name)
        for cm in (T.COST_SUM, T.COST_CRITICAL_PATH):
            o = Oracle(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth, cost_model=cm)
            o_seqs, oc = o.rollout(np.zeros((n, 32), np.uint16), seed=5, id_base=0)
            for K in ks:
                os.environ["TOAST_FORCE_K"] = str(K)
                a = T.build_analysis(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth,
                                     cuda_device=0, cost_model=cm, dedup=T.DEDUP_OFF)
                pre = torch.zeros((n, 32), dtype=torch.int16, device="cuda")
                seqs = torch.empty_like(pre)
                out = torch.empty((n, 256), dtype=torch.uint8, device="cuda")
                try:
                    T.rollout_batch(a, pre, 5, 0, seqs, out)
                    torch.cuda.synchronize()
                    out2 = torch.empty_like(out)
                    T.eval_batch(a, seqs, out2)
                    sc = torch.empty((n, 16), dtype=torch.uint8, device="cuda")
                    T.eval_scores(a, seqs, sc)
                    torch.cuda.synchronize()
                except Exception:
                    f = getattr(T._lib, "toast_checked_failure_line", None)
                    if f is not None:
                        f.restype = ctypes.c_uint
                        print(f"{name} cost_model={cm} K={K}: CHECK FAILED at kernels.cu:{f()}", flush=True)
                    raise
                g_seqs = seqs.cpu().numpy().view(np.uint16)
                ok = (np.array_equal(g_seqs, o_seqs) and T.as_costs(out).tobytes() == oc.tobytes()
                      and T.as_costs(out2).tobytes() == oc.tobytes())
                print(f"{name} cost_model={cm} K={K}: {'ok' if ok else 'MISMATCH'}", flush=True)
                if not ok:
                    sys.exit(1)
                done += 1
                del a
        # the dedup pipeline (front / back / scatter kernels), both cost models
        for cm in (T.COST_SUM, T.COST_CRITICAL_PATH):
            os.environ.pop("TOAST_FORCE_K", None)
            o = Oracle(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth, cost_model=cm)
            o_seqs, oc = o.rollout(np.zeros((n, 32), np.uint16), seed=5, id_base=0)
            a = T.build_analysis(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth,
                                 cuda_device=0, cost_model=cm, dedup=1)
            pre = torch.zeros((n, 32), dtype=torch.int16, device="cuda")
            seqs = torch.empty_like(pre)
            out = torch.empty((n, 256), dtype=torch.uint8, device="cuda")
            T.rollout_batch(a, pre, 5, 0, seqs, out)
            torch.cuda.synchronize()
            ok = np.array_equal(seqs.cpu().numpy().view(np.uint16), o_seqs) and T.as_costs(out).tobytes() == oc.tobytes()
            print(f"{name} cost_model={cm} dedup: {'ok' if ok else 'MISMATCH'}", flush=True)
            if not ok:
                sys.exit(1)
            done += 1
    os.environ.pop("TOAST_FORCE_K", None)
    print(f"sanitize driver: {done} (config, cost model, K) runs, all bit-identical to the oracle")


if __name__ == "__main__":
    main()
