"""The bench's C3 configuration (1024 rollouts, settled C2 start, excitation train, default skin
policy), W ticks then T ticks through sph_rollout_batch -- for ncu captures of the production
launches (e.g. -k regex:"k_force|k_density" -s <n> -c <m>)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import sph_inputs as si
from paper_2604_12505_b200 import SphContext

W = int(sys.argv[1]) if len(sys.argv) > 1 else 2
T = int(sys.argv[2]) if len(sys.argv) > 2 else 1
B = 1024
t = si.make_tank(4.0)
sp = t.params
pv = np.ascontiguousarray(np.load(os.path.join(ROOT, "bench_data", "settled_ell4.npz"))["pv"], np.float32)
u = torch.from_numpy(np.ascontiguousarray(si.ensemble_inputs(range(B), 2200)[0][:, :W + T])).cuda()
ctx = SphContext(sp, pv, t.ghost_b, n_rollouts=B, rebin_every=0, skin=0.15 * sp.h, skin_max=0.5 * sp.h)
ctx.rollout(u[:, :W].contiguous())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(ctx.stream)
ctx.rollout(u[:, W:].contiguous())
e1.record(ctx.stream)
torch.cuda.synchronize()
print(f"{e0.elapsed_time(e1) / T:.2f} ms/tick, rebuilds {ctx.counters()[1].mean():.1f}", flush=True)
