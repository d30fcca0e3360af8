#!/usr/bin/env python3
"""Device time of one sph_lpv_eval (objective + gradient) for R restarts x S sequences x K."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2604_12505_b200.lpv import LpvProblem, init_params
for R, S, K in [(8, 1, 2200), (1, 1, 2200), (8, 2, 300), (64, 1, 2200)]:
    r = np.random.Generator(np.random.Philox(1))
    us = [r.normal(size=(K, 3)).astype(np.float32) for _ in range(S)]
    ys = [r.normal(size=(K, 3)).astype(np.float32) for _ in range(S)]
    p = LpvProblem(R, us, ys)
    p.set_params(init_params(R, S, 3))
    for _ in range(3): p.eval()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); n = 20
    for _ in range(n): p.eval()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    e0.record()
    for _ in range(n): p.eval(grad=False)
    e1.record(); torch.cuda.synchronize()
    ms_f = e0.elapsed_time(e1) / n
    print(f"R={R} S={S} K={K}: eval+grad {ms:.3f} ms ({ms*1e6/K:.0f} ns/step), objective only {ms_f:.3f} ms", flush=True)
