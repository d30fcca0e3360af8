"""Fluid speed distribution relative to the body translation at the steady state of the C3
horizon (diagnostic): which particles trip the Verlet bound."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import sph_inputs as si
from paper_2604_12505_b200 import SphContext
T0 = int(sys.argv[1]) if len(sys.argv) > 1 else 300
B = 64
t = si.make_tank(4.0)
sp = t.params
pv = np.ascontiguousarray(np.load(os.path.join(ROOT, "bench_data", "settled_ell4.npz"))["pv"], np.float32)
u = torch.from_numpy(si.ensemble_inputs(range(B), 2200)[0][:, :T0]).cuda()
ctx = SphContext(sp, pv, t.ghost_b, n_rollouts=B, rebin_every=0, skin=0.15 * sp.h)
ctx.rollout(u.contiguous())
body = ctx.get_body_state()
for b in range(0, B, 8):
    p = ctx.get_particles(b)
    v = np.hypot(p[:, 2] - body[b, 3], p[:, 3] - body[b, 4])
    vs = np.sort(v)[::-1]
    r = np.hypot(p[:, 0] - body[b, 0], p[:, 1] - body[b, 1])
    i = np.argsort(-v)[:5]
    print(f"b{b}: vmax {vs[0]:.3f} v2 {vs[1]:.3f} v10 {vs[9]:.3f} v100 {vs[99]:.3f} p50 {np.median(v):.3f} "
          f"n>vmax/2 {(v > vs[0] / 2).sum()}  r of top5 {np.round(r[i] / sp.R, 3)}", flush=True)
