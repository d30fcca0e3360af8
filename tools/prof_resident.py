"""k_resident on the C3 workload shape (B rollouts of the settled C2 tank, excitation inputs):
W warm-up ticks then T ticks, each one launch (for ncu: -k regex:k_resident -s W)."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import sph_inputs as si
from paper_2604_12505_b200 import SphContext

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
W = int(sys.argv[2]) if len(sys.argv) > 2 else 2
T = int(sys.argv[3]) if len(sys.argv) > 3 else 1
ex = int(sys.argv[4]) if len(sys.argv) > 4 else 3
t = si.make_tank(4.0)
sp = t.params
pv = np.ascontiguousarray(np.load(os.path.join(ROOT, "bench_data", "settled_ell4.npz"))["pv"], np.float32)
u = torch.from_numpy(si.ensemble_inputs(range(B), W + T)[0]).cuda()
ctx = SphContext(sp, pv, t.ghost_b, n_rollouts=B, rebin_every=0, skin=0.15 * sp.h, exec_path=ex)
y = torch.empty((B, W + T, 6), device="cuda")
ua = torch.empty((B, W + T, 3), device="cuda")
ctx.rollout(u[:, :W].contiguous(), y_out=y[:, :W].contiguous(), u_applied=ua[:, :W].contiguous())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(ctx.stream)
ctx.rollout(u[:, W:].contiguous(), y_out=y[:, W:].contiguous(), u_applied=ua[:, W:].contiguous())
e1.record(ctx.stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"B={B} exec={ex} {ctx.exec_path()} ticks={T}: {ms / T:.3f} ms/tick, "
      f"{B * t.n_fluid * sp.n_sub * T / ms / 1e6:.3f} G updates/s, rebuilds {ctx.counters()[1].mean():.1f}",
      flush=True)
