"""Kernel timeline of one dedup rollout launch (torch.profiler / CUPTI): which
kernel or gap the step's time goes to.  python scripts/dedup_timeline.py <config>"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2508_15010_b200 import toast as T
from workloads import configs
name = sys.argv[1] if len(sys.argv) > 1 else "unet"
c = configs.get(name)
for dd in (0, 1):
    a = T.build_analysis(c.ir, c.axes, c.flops_per_sec, c.dm, c.penalty_c, c.min_dims, c.max_depth, cuda_device=0, dedup=dd)
    wave = a.preferred_batch()
    n = max(wave, ((1 << 18) // wave) * wave)
    pre = torch.zeros((n, 32), dtype=torch.int16, device="cuda")
    seq = torch.empty_like(pre)
    out = torch.empty((n, 256), dtype=torch.uint8, device="cuda")
    for w in range(3):
        T.rollout_batch(a, pre, 1, w * n, seq, out)
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as prof:
        for s in range(3):
            T.rollout_batch(a, pre, 1, (5 + s) * n, seq, out)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start if evs else 0
    print(f"== {name} dedup={dd} n={n}")
    for e in evs:
        print(f"  {e.time_range.start - t0:10.1f} us  {e.time_range.end - e.time_range.start:9.1f} us  {e.name[:70]}")
