#!/usr/bin/env python3
"""One sph_jacobian call per workload (for an ncu launch list)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import sph_inputs as si
from paper_2604_12505_b200 import SphContext
name = sys.argv[1] if len(sys.argv) > 1 else "P0"
tk = {"C1": lambda: si.make_tank(1.0), "P0": lambda: si.make_tank(1.0, n_first=666), "C2": lambda: si.make_tank(4.0)}[name]()
c = SphContext(tk.params, tk.pv32(), tk.ghost_b, n_rollouts=1)
for _ in range(2):
    A, B = c.jacobian(0, device=True)
torch.cuda.synchronize()
print(name, "ok", float(A.abs().max()))
