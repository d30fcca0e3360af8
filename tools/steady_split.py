"""Kernel split at the steady state of the C3 data-generation horizon (diagnostic): run T0 ticks of
the 2200-sample train, then sph_profile_substeps (each kernel alone, events)."""
import os, sys, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import sph_inputs as si
from paper_2604_12505_b200 import SphContext

skin = float(sys.argv[1]); T0 = int(sys.argv[2]); B = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
t = si.make_tank(4.0)
sp = t.params
pv = np.ascontiguousarray(np.load(os.path.join(ROOT, "bench_data", "settled_ell4.npz"))["pv"], np.float32)
u = torch.from_numpy(si.ensemble_inputs(range(B), 2200)[0][:, :T0 + 1]).cuda()
ctx = SphContext(sp, pv, t.ghost_b, n_rollouts=B, rebin_every=0, skin=skin * sp.h)
ctx.rollout(u[:, :T0].contiguous())
s0, r0 = ctx.counters()
prof = ctx.profile(20)
s1, r1 = ctx.counters()
print(json.dumps({"skin": skin, "T0": T0, "ms": prof, "rebuilt_fraction_per_substep": float((r1 - r0).mean() / 20)}), flush=True)
