"""Error statistics vs the oracle over several C2 rollouts (3 ticks of excitation), per-substep
kernels (1) vs resident clusters (3) -- diagnostic, GPU."""
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
B = 8
u = si.ensemble_inputs(range(B), 3)[0]
P = {}
for ex in (1, 3):
    c = SphContext(sp, pv, t.ghost_b, n_rollouts=B, rebin_every=0, skin=0.15 * sp.h, exec_path=ex)
    c.rollout(u)
    P[ex] = [c.get_particles(b) for b in range(B)]
    print(ex, c.counters()[1].tolist(), flush=True)
    c.close()
for b in range(B):
    ref = O.State(sp, pv[:, :2].astype(np.float64), pv[:, 2:].astype(np.float64), t.ghost_b)
    ref.rollout(u[b].astype(np.float64), sp.n_sub)
    row = [f"b{b}"]
    for ex in (1, 3):
        e = np.abs(P[ex][b][:, :2] - ref.pos).max(1)
        row.append(f"ex{ex} max {e.max():.2e} p99 {np.percentile(e, 99):.2e} med {np.median(e):.2e}")
    e = np.abs(P[1][b][:, :2] - P[3][b][:, :2]).max(1)
    row.append(f"1v3 max {e.max():.2e} p99 {np.percentile(e, 99):.2e} med {np.median(e):.2e}")
    print(" | ".join(row), flush=True)
