#!/usr/bin/env python3
"""Short driver for ncu captures: the bench's workload and launch configuration (C3 by default),
a brief GPU settle, then a few substeps through the C ABI (sph_step, direct launches)."""
import argparse
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import sph_inputs as si  # noqa: E402
from bench import WORKLOADS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C3")
ap.add_argument("--rollouts", type=int, default=0)
ap.add_argument("--substeps", type=int, default=6)
ap.add_argument("--settle-steps", type=int, default=400)
ap.add_argument("--rebin-every", type=int, default=0)
ap.add_argument("--skin", type=float, default=0.3)
a = ap.parse_args()

import torch  # noqa: E402
from paper_2604_12505_b200 import SphContext  # noqa: E402

ell, B, _ = WORKLOADS[a.workload]
B = a.rollouts or B
t = si.make_tank(ell)
sp = t.params
snap = os.path.join(ROOT, "bench_data", f"settled_ell{ell:g}.npz")
if a.settle_steps < 0 and os.path.exists(snap):      # the bench's oracle-settled start
    pv = np.load(snap)["pv"].astype(np.float32)
else:
    one = SphContext(sp, t.pv32(), t.ghost_b, n_rollouts=1)
    one.settle(math.exp(-10 * sp.dt), max(a.settle_steps, 0))
    pv = one.get_particles(0)
    one.close()
ctx = SphContext(sp, pv, t.ghost_b, n_rollouts=B, rebin_every=a.rebin_every, skin=a.skin * sp.h)
u = si.ensemble_inputs(range(B), 1)[0][:, 0]
ctx.step(u, a.substeps)
torch.cuda.synchronize()
print("status max", ctx.get_status()[0].max(), "profile", ctx.profile(3))
ctx.close()
