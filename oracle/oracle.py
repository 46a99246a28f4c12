"""ctypes wrapper around the TOAST oracle (oracle/toast_oracle.cpp).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module.  The product
package (paper_2508_15010_b200) never imports it and shares no code with it.
"""
from __future__ import annotations

import ctypes
import json
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "toast_oracle.cpp")
_LIB = os.path.join(_HERE, "build", "liboracle.so")

# the oracle's own view of the 256-byte cost record
COST_DTYPE = np.dtype([
    ("runtime_s", "<f8"), ("score", "<f8"),
    ("peak_bytes", "<u8"), ("flops", "<u8"), ("state_key", "<u8"),
    ("status", "<u4"), ("n_collectives", "<u4"),
    ("payload", "<u8", (4, 4)),
    ("count", "<u2", (4, 4)),
    ("flops_hi", "<u8"),
    ("pad", "u1", (40,)),
])
assert COST_DTYPE.itemsize == 256

SEARCH_DTYPE = np.dtype([
    ("best_seq", "<u2", (32,)), ("best", COST_DTYPE),
    ("evals", "<i8"), ("rounds", "<i4"), ("hit_target", "<i4"),
    ("wall_s", "<f8"), ("time_to_target_s", "<f8"),
])

AG, RS, AR, A2A = 0, 1, 2, 3


def build(force: bool = False) -> str:
    """Compile the oracle with g++ (plain C++17, no FMA contraction)."""
    os.makedirs(os.path.dirname(_LIB), exist_ok=True)
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call([
            "g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fPIC", "-shared", "-pthread",
            "-o", _LIB, _SRC])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        L.orc_new.restype = ctypes.c_void_p
        L.orc_new.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_double, ctypes.c_uint64,
                              ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.orc_last_error.restype = ctypes.c_char_p
        L.orc_free.argtypes = [ctypes.c_void_p]
        for f in ("orc_n_actions", "orc_n_loops", "orc_n_ops"):
            getattr(L, f).argtypes = [ctypes.c_void_p]
            getattr(L, f).restype = ctypes.c_int
        L.orc_eval.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int]
        L.orc_rollout.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64,
                                  ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        L.orc_materialize.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.orc_profile.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.orc_bruteforce.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.orc_bruteforce.restype = ctypes.c_int64
        L.orc_philox.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.orc_baseline.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                                   ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)]
        L.orc_dump.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int64]
        L.orc_dump.restype = ctypes.c_int64
        for f in ("orc_use_loop",):
            getattr(L, f).argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.orc_def_loop.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
        for f in ("orc_n_names", "orc_n_identities", "orc_n_map"):
            getattr(L, f).argtypes = [ctypes.c_void_p]
        L.orc_edges.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        L.orc_search.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int64, ctypes.c_double,
                                 ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                 ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
    return _lib


class OracleError(Exception):
    def __init__(self, msg: str):
        super().__init__(msg)
        self.code = msg.split(":", 1)[0]


def mesh_spec(axes) -> str:
    """axes: list of (name, size, bytes_per_sec)."""
    return ",".join(f"{n}={s}:{bw!r}" for n, s, bw in axes)


class Oracle:
    def __init__(self, ir: str, axes, flops_per_sec: float, dm: int, penalty_c: float = 100.0,
                 min_dims: int = 10, max_depth: int = 30, cost_model: int = 0, grouping: int = 0):
        """cost_model: 0 = straight-line sum (reading G14), 1 = critical path (reading R22).
        grouping: 0 = compatibility sets (C4/C5), 1 = graph contraction heuristic (reading R23)."""
        L = lib()
        self.axes = list(axes)
        self.max_depth = max_depth
        h = L.orc_new(ir.encode(), mesh_spec(axes).encode(), float(flops_per_sec), int(dm),
                      float(penalty_c), int(min_dims), int(max_depth), int(cost_model), int(grouping))
        if not h:
            raise OracleError(L.orc_last_error().decode())
        self.h = ctypes.c_void_p(h)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_free(self.h)
            self.h = None

    @property
    def n_actions(self) -> int:
        return lib().orc_n_actions(self.h)

    @property
    def n_loops(self) -> int:
        return lib().orc_n_loops(self.h)

    @property
    def n_ops(self) -> int:
        return lib().orc_n_ops(self.h)

    def use_loop(self, t: int, k: int, i: int) -> int:
        return lib().orc_use_loop(self.h, t, k, i)

    def def_loop(self, t: int, i: int) -> int:
        return lib().orc_def_loop(self.h, t, i)

    def edges(self) -> np.ndarray:
        """The deduplicated M edges over loops (C1): int32[n][2] (def loop, use loop)."""
        L = lib()
        n = L.orc_edges(self.h, None, 0)
        e = np.zeros((max(n, 1), 2), np.int32)
        L.orc_edges(self.h, e.ctypes.data, n)
        return e[:n]

    def nda_sizes(self):
        L = lib()
        return L.orc_n_names(self.h), L.orc_n_map(self.h), L.orc_n_identities(self.h)

    def _dump_all(self) -> dict:
        L = lib()
        n = L.orc_dump(self.h, None, 0)
        buf = ctypes.create_string_buffer(int(n))
        L.orc_dump(self.h, buf, n)
        return json.loads(buf.value.decode())

    def dump(self) -> dict:
        """The H0 analysis (the part comparable with the library's dump)."""
        d = self._dump_all()
        d.pop("set_graphs", None)
        return d

    def set_graphs(self) -> list:
        """Per compatibility set, the labelled graph its C6 signature hashes: nodes
        [loop, op kind, role, loop type, side mask], directed M edges, conflict edges."""
        return self._dump_all()["set_graphs"]

    def baseline(self):
        t0, p0, f0 = ctypes.c_double(), ctypes.c_uint64(), ctypes.c_uint64()
        lib().orc_baseline(self.h, ctypes.byref(t0), ctypes.byref(p0), ctypes.byref(f0))
        return t0.value, p0.value, f0.value

    @staticmethod
    def seqs(rows) -> np.ndarray:
        a = np.zeros((len(rows), 32), dtype=np.uint16)
        for i, r in enumerate(rows):
            a[i, :len(r)] = r
        return a

    def eval(self, seqs, threads: int = 1) -> np.ndarray:
        seqs = np.ascontiguousarray(seqs, dtype=np.uint16).reshape(-1, 32)
        out = np.zeros(len(seqs), dtype=COST_DTYPE)
        lib().orc_eval(self.h, seqs.ctypes.data, len(seqs), out.ctypes.data, int(threads))
        return out

    def rollout(self, prefixes, seed: int, id_base: int = 0, threads: int = 1):
        prefixes = np.ascontiguousarray(prefixes, dtype=np.uint16).reshape(-1, 32)
        out_seqs = np.zeros_like(prefixes)
        out = np.zeros(len(prefixes), dtype=COST_DTYPE)
        lib().orc_rollout(self.h, prefixes.ctypes.data, len(prefixes), int(seed), int(id_base),
                          out_seqs.ctypes.data, out.ctypes.data, int(threads))
        return out_seqs, out

    def materialize(self, seq) -> np.ndarray:
        s = np.zeros(32, dtype=np.uint16)
        s[:len(seq)] = seq
        m = np.zeros(self.n_loops, dtype=np.uint8)
        lib().orc_materialize(self.h, s.ctypes.data, m.ctypes.data)
        return m

    def profile(self, seq) -> np.ndarray:
        """M_t of every op t for one sequence (C12: peak = max_t M_t)."""
        s = np.zeros(32, dtype=np.uint16)
        s[:len(seq)] = seq
        out = np.zeros(lib().orc_n_ops(self.h), dtype=np.int64)
        lib().orc_profile(self.h, s.ctypes.data, out.ctypes.data)
        return out

    def bruteforce(self):
        best = np.zeros(32, dtype=np.uint16)
        cost = np.zeros(1, dtype=COST_DTYPE)
        n = lib().orc_bruteforce(self.h, best.ctypes.data, cost.ctypes.data)
        return n, best, cost[0]

    def search(self, seed=0, max_evals=0, time_limit_s=0.0, L=16, R=16, patience=1, uct_c=2 ** 0.5,
               target_score=float("nan"), threads=1, trace_cap=4096, transpositions=0):
        """C16; transpositions=1: each materialised state once in the tree (reading R24)."""
        res = np.zeros(1, dtype=SEARCH_DTYPE)
        trace = np.zeros(trace_cap, dtype=np.float64)
        lib().orc_search(self.h, int(seed), int(max_evals), float(time_limit_s), int(L), int(R), int(patience),
                         float(uct_c), float(target_score), int(threads), res.ctypes.data, trace.ctypes.data,
                         int(trace_cap), int(transpositions))
        r = res[0]
        return r, trace[:min(int(r["rounds"]), trace_cap)].copy()


def philox4x32_10(ctr, key):
    c = (ctypes.c_uint32 * 4)(*ctr)
    k = (ctypes.c_uint32 * 2)(*key)
    o = (ctypes.c_uint32 * 4)()
    lib().orc_philox(c, k, o)
    return list(o)
