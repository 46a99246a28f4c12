"""The five BASELINE.json configs as (IR text, mesh, machine, options).

Input generation only.  Default machine = B200-class target:
F = 2.25e15 flop/s, innermost axis 9.0e11 B/s (NVLink 5), other axes 5.0e10 B/s,
DM = 180e9 B, C = 100.
"""
from __future__ import annotations

import functools
import os
from dataclasses import dataclass

from . import models

F_B200 = 2.25e15
BW_NVLINK = 9.0e11
BW_NIC = 5.0e10
DM_B200 = 180 * 10 ** 9

_HERE = os.path.dirname(os.path.abspath(__file__))
_GOLDEN = os.path.join(os.path.dirname(_HERE), "tests", "golden")


@dataclass(frozen=True)
class Config:
    name: str
    ir: str
    axes: tuple          # ((name, size, bytes_per_sec), ...) in mesh order
    flops_per_sec: float
    dm: int
    penalty_c: float
    min_dims: int
    max_depth: int = 30
    description: str = ""


def _golden(name: str) -> str:
    with open(os.path.join(_GOLDEN, name)) as f:
        return f.read()


def _b200_mesh(*axes):
    """axes: (name, size); the last axis is the innermost (NVLink)."""
    out = []
    for i, (n, s) in enumerate(axes):
        out.append((n, s, BW_NVLINK if i == len(axes) - 1 else BW_NIC))
    return tuple(out)


@functools.lru_cache(maxsize=None)
def get(name: str, **kw) -> Config:
    if name == "mlp_c":
        return Config("mlp_c", _golden("mlp_c.ir"), (("b", 2, 1e10), ("m", 2, 1e11)), 1e12, 131072, 100.0, 1,
                      description="M1 MLP-c, mesh {b:2,m:2}, exhaustive-checkable")
    if name == "attn_toy":
        return Config("attn_toy", _golden("attn_fig5.ir"), (("s", 2, 1e10),), 1e12, 1 << 40, 100.0, 1,
                      description="Fig. 5a attention, S=8, mesh {s:2}")
    if name == "gpt24":
        return Config("gpt24", models.gpt(), _b200_mesh(("data", 8), ("model", 4)), F_B200, DM_B200, 100.0, 10,
                      description="M2 GPT-24 decoder (T2B-like widths), mesh {data:8, model:4}")
    if name == "gpt2":
        # a 2-layer GPT at reduced widths: several tiles, fast for the oracle
        return Config("gpt2", models.gpt(layers=2, B=8, S=64, D=64, H=4, Dh=16, F=256, V=512, name="gpt2"),
                      _b200_mesh(("data", 8), ("model", 4)), F_B200, 1 << 22, 100.0, 10,
                      description="2-layer GPT (small widths), mesh {data:8, model:4}")
    if name == "gpt2_np2":
        # non-power-of-two mesh {data:3, model:6}: exact division by odd products
        return Config("gpt2_np2", models.gpt(layers=2, B=12, S=48, D=96, H=6, Dh=16, F=384, V=384, name="gpt2np2"),
                      (("data", 3, BW_NIC), ("model", 6, BW_NVLINK)), F_B200, 1 << 22, 100.0, 10,
                      description="2-layer GPT on a non-power-of-two mesh {data:3, model:6}")
    if name == "gpt2_1ax_np2":
        # the 2-layer GPT on one non-power-of-two axis (the kernels' NA = 1, P2 = false instantiation)
        return Config("gpt2_1ax_np2", models.gpt(layers=2, B=12, S=48, D=96, H=6, Dh=16, F=384, V=384, name="gpt2np2"),
                      (("model", 3, BW_NVLINK),), F_B200, 1 << 22, 100.0, 10,
                      description="2-layer GPT on a one-axis non-power-of-two mesh {model:3}")
    if name == "gpt2_3ax":
        # the 2-layer GPT on a three-axis mesh (the kernels' NA = 3 instantiation, Llama-80's mesh shape)
        return Config("gpt2_3ax", models.gpt(layers=2, B=8, S=64, D=64, H=4, Dh=16, F=256, V=512, name="gpt2"),
                      _b200_mesh(("data", 2), ("fsdp", 2), ("tensor", 2)), F_B200, 1 << 22, 100.0, 10,
                      description="2-layer GPT on a three-axis mesh {data:2, fsdp:2, tensor:2}")
    if name == "gpt2_3ax_np2":
        return Config("gpt2_3ax_np2", models.gpt(layers=2, B=12, S=48, D=96, H=6, Dh=16, F=384, V=384, name="gpt2np2"),
                      _b200_mesh(("data", 2), ("fsdp", 3), ("tensor", 2)), F_B200, 1 << 22, 100.0, 10,
                      description="2-layer GPT on a three-axis non-power-of-two mesh {data:2, fsdp:3, tensor:2}")
    if name == "gpt2_4ax":
        # the same 2-layer GPT on a four-axis mesh (the kernels' NA = 4 instantiation)
        return Config("gpt2_4ax", models.gpt(layers=2, B=8, S=64, D=64, H=4, Dh=16, F=256, V=512, name="gpt2"),
                      _b200_mesh(("pod", 2), ("data", 2), ("fsdp", 2), ("model", 4)), F_B200, 1 << 22, 100.0, 10,
                      description="2-layer GPT on a four-axis mesh {pod:2, data:2, fsdp:2, model:4}")
    if name == "gpt2_4ax_np2":
        return Config("gpt2_4ax_np2", models.gpt(layers=2, B=12, S=48, D=96, H=6, Dh=16, F=384, V=384, name="gpt2np2"),
                      _b200_mesh(("pod", 2), ("data", 3), ("fsdp", 2), ("model", 2)), F_B200, 1 << 22, 100.0, 10,
                      description="2-layer GPT on a four-axis non-power-of-two mesh {pod:2, data:3, fsdp:2, model:2}")
    if name == "unet":
        return Config("unet", models.unet(), _b200_mesh(("batch", 4), ("model", 8)), F_B200, DM_B200, 100.0, 10,
                      description="M3 U-Net, mesh {batch:4, model:8}")
    if name == "gns16":
        return Config("gns16", models.gns(), _b200_mesh(("edges", 8), ("features", 4)), F_B200, DM_B200, 100.0, 10,
                      description="M4 GNS-16, mesh {edges:8, features:4}")
    if name == "llama80":
        return Config("llama80", models.llama(), _b200_mesh(("data", 4), ("fsdp", 8), ("tensor", 8)), F_B200,
                      DM_B200, 100.0, 10, description="M5 Llama-80L, mesh {data:4, fsdp:8, tensor:8}")
    raise KeyError(name)


ALL = ("mlp_c", "gpt24", "unet", "gns16", "llama80")
