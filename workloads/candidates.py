"""Seeded random candidate sequences (uint16[n][32]) — input generation only.

`uniform` draws raw action ids with no legality knowledge (exercises the
status paths).  Legal rollout batches come from the oracle's C15 policy in
the tests (SURVEY §8(d) "Candidate inputs").
"""
from __future__ import annotations

import numpy as np


def uniform(n: int, n_actions: int, seed: int, max_len: int = 30, bad_frac: float = 0.0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    out = np.zeros((n, 32), dtype=np.uint16)
    lens = rng.integers(0, max_len + 1, size=n)
    for i in range(n):
        L = int(lens[i])
        if L:
            out[i, :L] = rng.integers(1, max(2, n_actions), size=L)
    if bad_frac > 0:
        k = int(n * bad_frac)
        idx = rng.choice(n, size=k, replace=False)
        out[idx, 31] = rng.integers(1, 65535, size=k)   # nonzero after STOP (or a bad id)
    return out
