"""Thin ctypes binding of libtoast (include/toast.h) — argument marshalling only.

Every step of the hot path runs in libtoast's sm_100a kernels; this module
turns Python objects into pointers and back.  There is no CPU fallback: if
libtoast.so is missing the import fails loudly, and evaluation calls on a
graph without device tables raise ToastError(TOAST_E_CUDA).

Buffers: torch tensors (CUDA tensors -> asynchronous on the given stream;
CPU / pinned tensors -> the library stages through device scratch) or numpy
arrays (host).  Candidate sequences are uint16[n][32] (torch: int16 viewed as
uint16, or torch.uint16); cost records are 256-byte rows (torch.uint8[n,256]
or a numpy COST_DTYPE array).
"""
from __future__ import annotations

import ctypes
import json
import math
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TOAST_LIB") or os.path.join(_HERE, "lib", "libtoast.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libtoast.so not built ({LIB_PATH}); run `python -m paper_2508_15010_b200.build`")

_lib = ctypes.CDLL(LIB_PATH)

STATUS = {0: "TOAST_OK", 1: "TOAST_E_INVALID_ARG", 2: "TOAST_E_PARSE", 3: "TOAST_E_SHAPE", 4: "TOAST_E_UNDEFINED",
          5: "TOAST_E_DUPLICATE", 6: "TOAST_E_MESH", 7: "TOAST_E_MACHINE", 8: "TOAST_E_DEGENERATE", 9: "TOAST_E_LIMIT",
          10: "TOAST_E_CUDA", 11: "TOAST_E_NCCL", 12: "TOAST_E_OOM"}
ST_BAD_ACTION_ID, ST_DUP_COLOR_AXIS, ST_RES_MISMATCH, ST_NONZERO_AFTER_STOP = 1, 2, 4, 8
AG, RS, AR, A2A = 0, 1, 2, 3

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


class _Axis(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("size", ctypes.c_int32), ("bytes_per_sec", ctypes.c_double)]


class _Machine(ctypes.Structure):
    _fields_ = [("flops_per_sec", ctypes.c_double), ("device_memory_bytes", ctypes.c_uint64),
                ("penalty_c", ctypes.c_double)]


class _NdaOpts(ctypes.Structure):
    _fields_ = [("min_unique_dims", ctypes.c_int32), ("max_depth", ctypes.c_int32), ("cost_model", ctypes.c_int32),
                ("conflict_grouping", ctypes.c_int32), ("dedup", ctypes.c_int32)]


COST_SUM, COST_CRITICAL_PATH = 0, 1
GROUP_COMPAT, GROUP_CONTRACTION = 0, 1


class _ActionInfo(ctypes.Structure):
    _fields_ = [("super_color", ctypes.c_int32), ("resolution", ctypes.c_int32), ("axis", ctypes.c_int32),
                ("n_value_dims", ctypes.c_int32)]


class _SearchOpts(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("max_evals", ctypes.c_int64), ("time_limit_s", ctypes.c_double),
                ("leaves_per_round", ctypes.c_int32), ("rollouts_per_leaf", ctypes.c_int32),
                ("patience", ctypes.c_int32), ("transpositions", ctypes.c_int32), ("uct_c", ctypes.c_double),
                ("target_score", ctypes.c_double), ("cuda_stream", ctypes.c_void_p)]


SEARCH_RESULT_DTYPE = np.dtype([
    ("best_seq", "<u2", (32,)), ("best", COST_DTYPE), ("evals", "<i8"), ("rounds", "<i4"), ("hit_target", "<i4"),
    ("wall_s", "<f8"), ("time_to_target_s", "<f8")])

ROOT_STAT_DTYPE = np.dtype([("visits", "<i8"), ("value_sum", "<f8")])

# toast_score (include/toast.h): score, or NaN with the status in state_key
SCORE_DTYPE = np.dtype([("score", "<f8"), ("state_key", "<u8")])
assert SCORE_DTYPE.itemsize == 16

_P = ctypes.c_void_p
_sigs = {
    "toast_load_graph": [ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(_Axis), ctypes.c_int32,
                         ctypes.POINTER(_Machine), ctypes.c_int32, ctypes.POINTER(_P)],
    "toast_nda": [_P, ctypes.POINTER(_NdaOpts), ctypes.POINTER(_P)],
    "toast_num_actions": [_P, ctypes.POINTER(ctypes.c_int32)],
    "toast_query_actions": [_P, ctypes.POINTER(_ActionInfo), ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)],
    "toast_query_baseline": [_P, _P],
    "toast_preferred_batch": [_P, ctypes.POINTER(ctypes.c_int64)],
    "toast_dump_analysis": [_P, ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)],
    "toast_eval_batch": [_P, _P, ctypes.c_int64, _P, _P],
    "toast_rollout_batch": [_P, _P, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, _P, _P, _P],
    "toast_eval_scores": [_P, _P, ctypes.c_int64, _P, _P],
    "toast_rollout_scores": [_P, _P, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, _P, _P, _P],
    "toast_materialize": [_P, _P, _P, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)],
    "toast_lower": [_P, _P, _P, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)],
    "toast_search_root_stats": [_P, _P, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)],
    "toast_search": [_P, ctypes.POINTER(_SearchOpts), _P],
    "toast_search_begin": [_P, ctypes.POINTER(_SearchOpts), ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(_P)],
    "toast_search_round": [_P, _P],
    "toast_search_import": [_P, _P, ctypes.POINTER(ctypes.c_int32)],
    "toast_search_round_dev": [_P, _P, _P],
    "toast_search_import_dev": [_P, _P, ctypes.POINTER(ctypes.c_int32), _P],
    "toast_search_end": [_P, _P],
}
for _n, _a in _sigs.items():
    getattr(_lib, _n).argtypes = _a
    getattr(_lib, _n).restype = ctypes.c_int
_lib.toast_last_error.restype = ctypes.c_char_p
_lib.toast_last_error.argtypes = []
_lib.toast_search_export_bytes.restype = ctypes.c_size_t
_lib.toast_search_export_bytes.argtypes = [_P]
_lib.toast_free_graph.argtypes = [_P]
_lib.toast_free_graph.restype = None
_lib.toast_free_analysis.argtypes = [_P]
_lib.toast_free_analysis.restype = None

EXPORTED = sorted(list(_sigs) + ["toast_last_error", "toast_search_export_bytes", "toast_free_graph",
                                 "toast_free_analysis"])


class ToastError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.code = STATUS.get(status, str(status))


def _check(st: int):
    if st != 0:
        raise ToastError(st, _lib.toast_last_error().decode(errors="replace"))


def _ptr(x):
    """(address, nbytes) of a torch tensor or numpy array (contiguous)."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        assert x.is_contiguous(), "tensor must be contiguous"
        return x.data_ptr()
    assert isinstance(x, np.ndarray) and x.flags["C_CONTIGUOUS"], "numpy array must be C-contiguous"
    return x.ctypes.data


def _len(x, row_bytes):
    if hasattr(x, "data_ptr"):
        return x.numel() * x.element_size() // row_bytes
    return x.nbytes // row_bytes


def _stream(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except Exception:
            pass
        return None
    return getattr(stream, "cuda_stream", stream)


# ----------------------------------------------------------------- graph / analysis
class Graph:
    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.toast_free_graph(self._h)
            self._h = None


def load_graph(ir_text: str, axes, flops_per_sec: float, device_memory_bytes: int, penalty_c: float = 100.0,
               cuda_device: int = 0) -> Graph:
    """toast_load_graph.  axes: [(name, size, bytes_per_sec), ...] in mesh order."""
    b = ir_text.encode()
    arr = (_Axis * len(axes))(*[_Axis(n.encode(), int(s), float(bw)) for n, s, bw in axes])
    m = _Machine(float(flops_per_sec), int(device_memory_bytes), float(penalty_c))
    h = _P()
    _check(_lib.toast_load_graph(b, len(b), arr, len(axes), ctypes.byref(m), int(cuda_device), ctypes.byref(h)))
    return Graph(h)


class Analysis:
    def __init__(self, handle, graph_axes):
        self._h = handle
        self.axes = graph_axes

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:   # (module globals are gone at interpreter exit)
            _lib.toast_free_analysis(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def n_actions(self) -> int:
        n = ctypes.c_int32()
        _check(_lib.toast_num_actions(self._h, ctypes.byref(n)))
        return n.value

    def actions(self):
        n = self.n_actions
        arr = (_ActionInfo * n)()
        k = ctypes.c_int32()
        _check(_lib.toast_query_actions(self._h, arr, n, ctypes.byref(k)))
        return [(a.super_color, a.resolution, a.axis, a.n_value_dims) for a in arr]

    def baseline(self):
        out = np.zeros(1, dtype=COST_DTYPE)
        _check(_lib.toast_query_baseline(self._h, out.ctypes.data))
        return out[0]

    def preferred_batch(self) -> int:
        n = ctypes.c_int64()
        _check(_lib.toast_preferred_batch(self._h, ctypes.byref(n)))
        return n.value

    def _dump_all(self) -> dict:
        need = ctypes.c_size_t()
        _check(_lib.toast_dump_analysis(self._h, None, 0, ctypes.byref(need)))
        buf = ctypes.create_string_buffer(need.value)
        _check(_lib.toast_dump_analysis(self._h, buf, need.value, ctypes.byref(need)))
        return json.loads(buf.value.decode())

    def dump(self) -> dict:
        """The H0 analysis (the part comparable with the oracle's own dump)."""
        d = self._dump_all()
        d.pop("kernel_tables", None)
        return d

    def kernel_tables(self) -> dict:
        """Sizes of the per-candidate tables (signatures, edge templates, the
        peak-memory frontier) and the op index of every frontier point."""
        return self._dump_all()["kernel_tables"]


DEDUP_OFF, DEDUP_ON, DEDUP_AUTO = 0, 1, 2


def nda(graph: Graph, min_unique_dims: int = 10, max_depth: int = 30, cost_model: int = COST_SUM,
        grouping: int = GROUP_COMPAT, dedup: int = DEDUP_AUTO) -> Analysis:
    """toast_nda (H0).  grouping: GROUP_COMPAT (C4/C5) or GROUP_CONTRACTION (reading R23);
    dedup: rollout launches cost each distinct state once (NEXT-3, same results) —
    DEDUP_ON, DEDUP_OFF, or DEDUP_AUTO (on under the critical-path model only)."""
    o = _NdaOpts(int(min_unique_dims), int(max_depth), int(cost_model), int(grouping), int(dedup))
    h = _P()
    _check(_lib.toast_nda(graph._h, ctypes.byref(o), ctypes.byref(h)))
    return Analysis(h, None)


def build_analysis(ir_text, axes, flops_per_sec, device_memory_bytes, penalty_c=100.0, min_unique_dims=10,
                   max_depth=30, cuda_device=0, cost_model=COST_SUM, grouping=GROUP_COMPAT, dedup=DEDUP_AUTO) -> Analysis:
    g = load_graph(ir_text, axes, flops_per_sec, device_memory_bytes, penalty_c, cuda_device)
    a = nda(g, min_unique_dims, max_depth, cost_model, grouping, dedup)
    a.axes = list(axes)
    return a


# ----------------------------------------------------------------- hot path
def eval_batch(a: Analysis, seqs, out, stream=None, n: int | None = None):
    """toast_eval_batch: seqs uint16[n][32] -> out 256-B records (same memory kind)."""
    n = _len(seqs, 64) if n is None else n
    assert _len(out, 256) >= n
    _check(_lib.toast_eval_batch(a._h, _ptr(seqs), int(n), _ptr(out), _stream(stream)))
    return out


def rollout_batch(a: Analysis, prefixes, seed: int, id_base: int, out_seqs, out, stream=None, n: int | None = None):
    """toast_rollout_batch: extend each prefix with Philox draws (H8), then cost it."""
    n = _len(prefixes, 64) if n is None else n
    assert _len(out, 256) >= n and _len(out_seqs, 64) >= n, "output buffers hold fewer than n rows"
    _check(_lib.toast_rollout_batch(a._h, _ptr(prefixes), int(n), int(seed), int(id_base), _ptr(out_seqs),
                                    _ptr(out), _stream(stream)))
    return out_seqs, out


def eval_scores(a: Analysis, seqs, out, stream=None, n: int | None = None):
    """toast_eval_scores: seqs uint16[n][32] -> out 16-B toast_score records (same memory kind)."""
    n = _len(seqs, 64) if n is None else n
    assert _len(out, 16) >= n
    _check(_lib.toast_eval_scores(a._h, _ptr(seqs), int(n), _ptr(out), _stream(stream)))
    return out


def rollout_scores(a: Analysis, prefixes, seed: int, id_base: int, out_seqs, out, stream=None, n: int | None = None):
    """toast_rollout_scores: toast_rollout_batch with 16-B toast_score results."""
    n = _len(prefixes, 64) if n is None else n
    assert _len(out, 16) >= n and _len(out_seqs, 64) >= n, "output buffers hold fewer than n rows"
    _check(_lib.toast_rollout_scores(a._h, _ptr(prefixes), int(n), int(seed), int(id_base), _ptr(out_seqs),
                                     _ptr(out), _stream(stream)))
    return out_seqs, out


def as_scores(out) -> np.ndarray:
    """View a torch uint8[n,16] / numpy buffer of toast_score records as SCORE_DTYPE."""
    if hasattr(out, "data_ptr"):
        out = out.detach().cpu().contiguous().numpy()
    return np.ascontiguousarray(out).view(SCORE_DTYPE).reshape(-1)


def materialize(a: Analysis, seq) -> np.ndarray:
    s = np.zeros(32, dtype=np.uint16)
    s[:len(seq)] = seq
    n = ctypes.c_int64()
    _check(_lib.toast_materialize(a._h, s.ctypes.data, None, 0, ctypes.byref(n)))
    m = np.zeros(n.value, dtype=np.uint8)
    _check(_lib.toast_materialize(a._h, s.ctypes.data, m.ctypes.data, n.value, ctypes.byref(n)))
    return m


def lower(a: Analysis, seq) -> str:
    """The device-local program of one action sequence (toast_lower)."""
    s = np.zeros(32, dtype=np.uint16)
    s[:len(seq)] = seq
    need = ctypes.c_size_t()
    _check(_lib.toast_lower(a._h, s.ctypes.data, None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    _check(_lib.toast_lower(a._h, s.ctypes.data, buf, need.value, ctypes.byref(need)))
    return buf.value.decode()


def as_costs(out) -> np.ndarray:
    """View a torch uint8[n,256] / numpy buffer of records as COST_DTYPE (copies device tensors to host)."""
    if hasattr(out, "data_ptr"):
        out = out.detach().cpu().contiguous().numpy()
    return np.ascontiguousarray(out).view(COST_DTYPE).reshape(-1)


# ----------------------------------------------------------------- search
@dataclass
class SearchOptions:
    seed: int = 0
    max_evals: int = 0
    time_limit_s: float = 0.0
    leaves_per_round: int = 64
    rollouts_per_leaf: int = 64
    patience: int = 1
    uct_c: float = math.sqrt(2.0)
    target_score: float = float("nan")
    transpositions: int = 0   # 1: each materialised state once in the tree (reading R24)

    def c(self, stream):
        return _SearchOpts(int(self.seed), int(self.max_evals), float(self.time_limit_s), int(self.leaves_per_round),
                           int(self.rollouts_per_leaf), int(self.patience), int(self.transpositions), float(self.uct_c),
                           float(self.target_score), _stream(stream))


def search(a: Analysis, opts: SearchOptions, stream=None):
    """toast_search (single GPU)."""
    o = opts.c(stream)
    res = np.zeros(1, dtype=SEARCH_RESULT_DTYPE)
    _check(_lib.toast_search(a._h, ctypes.byref(o), res.ctypes.data))
    return res[0]


def search_export_bytes(a: Analysis) -> int:
    return int(_lib.toast_search_export_bytes(a._h))


class SearchState:
    """Root-parallel search driver state (toast_search_begin/round/import/end)."""

    def __init__(self, a: Analysis, opts: SearchOptions, rank: int, world: int, stream=None):
        self.a = a
        self._o = opts.c(stream)
        h = _P()
        _check(_lib.toast_search_begin(a._h, ctypes.byref(self._o), int(rank), int(world), ctypes.byref(h)))
        self._h = h
        self.export_bytes = search_export_bytes(a)

    def round(self) -> np.ndarray:
        buf = np.zeros(self.export_bytes, dtype=np.uint8)
        _check(_lib.toast_search_round(self._h, buf.ctypes.data))
        return buf

    def round_dev(self, export_dev, stream=None):
        """toast_search_round_dev: the round's record into a device tensor (uint8[export_bytes])."""
        assert _len(export_dev, 1) >= self.export_bytes
        _check(_lib.toast_search_round_dev(self._h, _ptr(export_dev), _stream(stream)))
        return export_dev

    def import_dev(self, gathered_dev, stream=None) -> bool:
        """toast_search_import_dev: the all-gathered records ([world][export_bytes], device)."""
        stop = ctypes.c_int32()
        _check(_lib.toast_search_import_dev(self._h, _ptr(gathered_dev), ctypes.byref(stop), _stream(stream)))
        return bool(stop.value)

    def import_(self, gathered: np.ndarray) -> bool:
        g = np.ascontiguousarray(gathered, dtype=np.uint8)
        stop = ctypes.c_int32()
        _check(_lib.toast_search_import(self._h, g.ctypes.data, ctypes.byref(stop)))
        return bool(stop.value)

    def root_stats(self) -> np.ndarray:
        """Root-child (visits, value_sum) per action id, summed over the ranks at the last import."""
        n = ctypes.c_int32()
        _check(_lib.toast_search_root_stats(self._h, None, 0, ctypes.byref(n)))
        out = np.zeros(n.value, dtype=ROOT_STAT_DTYPE)
        _check(_lib.toast_search_root_stats(self._h, out.ctypes.data, n.value, ctypes.byref(n)))
        return out

    def end(self):
        res = np.zeros(1, dtype=SEARCH_RESULT_DTYPE)
        _check(_lib.toast_search_end(self._h, res.ctypes.data))
        self._h = None
        return res[0]

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.toast_search_end(self._h, None)
            self._h = None
