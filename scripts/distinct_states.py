import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
"""Distinct final states and sequences in one bench-sized rollout batch per config (NEXT-3 dedup potential)."""
import numpy as np, torch
from workloads import configs
from paper_2508_15010_b200 import toast as T
for n in ['gpt24','unet','gns16','llama80']:
    c=configs.get(n)
    a=T.build_analysis(c.ir,c.axes,c.flops_per_sec,c.dm,c.penalty_c,c.min_dims,c.max_depth,cuda_device=0)
    N=189440
    pre=torch.zeros((N,32),dtype=torch.int16,device='cuda'); seqs=torch.empty_like(pre); out=torch.empty((N,256),dtype=torch.uint8,device='cuda')
    T.rollout_batch(a,pre,2024,0,seqs,out); torch.cuda.synchronize()
    k=T.as_costs(out)['state_key']; s=seqs.cpu().numpy().view(np.uint16)
    print(n, 'rollouts', N, 'distinct states', len(np.unique(k)), 'distinct sequences', len(np.unique(s, axis=0)))
