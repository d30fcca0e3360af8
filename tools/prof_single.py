"""One C2 (or C1) tank, W warm-up ticks then T ticks through sph_rollout_batch on the auto path
(resident clusters) -- for ncu captures of k_resident in the latency-bound regime."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import sph_inputs as si
from paper_2604_12505_b200 import SphContext
ell = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
W = int(sys.argv[2]) if len(sys.argv) > 2 else 3
T = int(sys.argv[3]) if len(sys.argv) > 3 else 10
t = si.make_tank(ell)
sp = t.params
pv = (np.ascontiguousarray(np.load(os.path.join(ROOT, "bench_data", "settled_ell4.npz"))["pv"], np.float32)
      if ell == 4.0 else t.pv32())
u = torch.from_numpy(np.ascontiguousarray(si.ensemble_inputs([0], 2200)[0][:, :W + T])).cuda()
ctx = SphContext(sp, pv, t.ghost_b, n_rollouts=1, rebin_every=0, skin=0.15 * sp.h, skin_max=0.5 * sp.h)
ctx.rollout(u[:, :W].contiguous())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(ctx.stream)
ctx.rollout(u[:, W:].contiguous())
e1.record(ctx.stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / T
print(f"{ctx.exec_path()} {ms:.3f} ms/tick = {1e3 * ms / sp.n_sub:.2f} us/substep, rebuilds {ctx.counters()[1][0]}", flush=True)
