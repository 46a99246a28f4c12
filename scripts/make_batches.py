"""Write the committed candidate batches (SURVEY §8(d) "Candidate inputs")
using ONLY the oracle (test infrastructure):

  workloads/batches/<config>_oracle_n65536.npz
      seqs      uint16[65536][32]  the oracle's C15 rollouts from the empty
                                   prefix (seed 0, ids 0..65535)
      worst     uint16[4096][32]   a worst-case batch: every row 30 legal
                                   actions, STOP disabled (the C15 kill rule
                                   restated over the oracle's action table)
      sample_idx / sample_rec      the oracle's 256-B records of 64 sampled
      worst_idx / worst_rec        rows of each batch (bench.py checks them)

    python scripts/make_batches.py [config ...]     (default: gpt24)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle.oracle import Oracle  # noqa: E402
from workloads import configs  # noqa: E402

OUT = os.path.join(ROOT, "workloads", "batches")


def legal_long(o: Oracle, n: int, seed: int, length: int = 30) -> np.ndarray:
    d = o.dump()
    acts = d["actions"]
    groups = [sc[2] for sc in d["scolors"]]
    rng = np.random.default_rng(seed)

    def kills(x, y):
        cx, rx, ax = acts[x - 1]
        cy, ry, ay = acts[y - 1]
        if cx == cy and ax == ay:
            return True
        return any(gx == gy and ((rx >> i) ^ (ry >> j)) & 1 for i, gx in enumerate(groups[cx])
                   for j, gy in enumerate(groups[cy]))
    K = len(acts) + 1
    kill = np.zeros((K, K), bool)
    for x in range(1, K):
        for y in range(1, K):
            kill[x, y] = kills(x, y)
    out = np.zeros((n, 32), np.uint16)
    for r in range(n):
        legal = np.ones(K, bool)
        legal[0] = False
        k = 0
        while legal.any() and k < length:
            c = np.flatnonzero(legal)
            a = int(c[rng.integers(len(c))])
            out[r, k] = a
            k += 1
            legal &= ~kill[a]
    return out


def main():
    names = sys.argv[1:] or ["gpt24"]
    os.makedirs(OUT, exist_ok=True)
    cores = os.cpu_count() or 1
    for name in names:
        c = configs.get(name)
        o = Oracle(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth)
        n = 1 << 16
        seqs, _ = o.rollout(np.zeros((n, 32), np.uint16), seed=0, id_base=0, threads=cores)
        worst = legal_long(o, 4096, seed=1)
        rng = np.random.default_rng(2)
        si = np.sort(rng.choice(n, 64, replace=False))
        wi = np.sort(rng.choice(len(worst), 64, replace=False))
        srec = o.eval(seqs[si], threads=cores)
        wrec = o.eval(worst[wi], threads=cores)
        assert (wrec["status"] == 0).all()
        path = os.path.join(OUT, f"{name}_oracle_n{n}.npz")
        np.savez_compressed(path, seqs=seqs, worst=worst, sample_idx=si, sample_rec=srec.view(np.uint8).reshape(-1, 256),
                            worst_idx=wi, worst_rec=wrec.view(np.uint8).reshape(-1, 256))
        print(path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
