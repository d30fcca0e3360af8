"""Batch / call-path invariance of one C2 rollout (diagnostic, GPU): B=2 rollout vs B=1 rollout vs
B=1 steps, for the per-substep kernels (1) and the resident clusters (3)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O
import sph_inputs as si
from paper_2604_12505_b200 import SphContext

t = si.make_tank(4.0)
sp = t.params
pv = np.ascontiguousarray(np.load(os.path.join(ROOT, "bench_data", "settled_ell4.npz"))["pv"], np.float32)
u2 = si.ensemble_inputs([5, 6], 3)[0]
ref = O.State(sp, pv[:, :2].astype(np.float64), pv[:, 2:].astype(np.float64), t.ghost_b)
ref.rollout(u2[1].astype(np.float64), sp.n_sub)
for ex in (1, 3):
    kw = dict(rebin_every=0, skin=0.15 * sp.h, exec_path=ex)
    a = SphContext(sp, pv, t.ghost_b, n_rollouts=2, **kw)
    ya, _ = a.rollout(u2)
    pa = a.get_particles(1)
    b = SphContext(sp, pv, t.ghost_b, n_rollouts=1, **kw)
    yb, _ = b.rollout(u2[1:2])
    pb = b.get_particles(0)
    c = SphContext(sp, pv, t.ghost_b, n_rollouts=1, **kw)
    for k in range(3):
        c.step(u2[1:2, k], sp.n_sub)
    pc = c.get_particles(0)
    e = lambda p: np.abs(p[:, :2] - ref.pos).max()
    print(f"ex{ex}: B2-rollout {e(pa):.3e}  B1-rollout {e(pb):.3e}  B1-step {e(pc):.3e}  "
          f"eq(B2,B1) {np.array_equal(pa, pb)} eq(B1r,B1s) {np.array_equal(pb, pc)} "
          f"reb {a.counters()[1].tolist()} {b.counters()[1].tolist()} {c.counters()[1].tolist()}", flush=True)
