"""Resident vs per-substep kernels vs oracle on the C2 tank: per-particle position error growth
(diagnostic, GPU)."""
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
gid = int(sys.argv[1]) if len(sys.argv) > 1 else 6
u = si.ensemble_inputs([gid], 3)[0]
ctxs = {ex: SphContext(sp, pv, t.ghost_b, n_rollouts=1, rebin_every=0, skin=0.15 * sp.h, exec_path=ex) for ex in (1, 3)}
ref = O.State(sp, pv[:, :2].astype(np.float64), pv[:, 2:].astype(np.float64), t.ghost_b)
done = 0
for n in (1, 1, 8, 10, 30, 50, 100, 200, 200):
    for ex, c in ctxs.items():
        c.step(u[:, min(done // sp.n_sub, 2)], n)
    ref.step(tuple(float(x) for x in u[0, min(done // sp.n_sub, 2)]), n=n)
    done += n
    out = [f"step {done:4d}"]
    P = {ex: c.get_particles(0) for ex, c in ctxs.items()}
    for ex in (1, 3):
        e = np.abs(P[ex][:, :2] - ref.pos).max(1)
        i = int(e.argmax())
        out.append(f"ex{ex}: max {e.max():.2e} at id {i} pos ({ref.pos[i,0]:+.4f},{ref.pos[i,1]:+.4f}) "
                   f"|v| {np.hypot(*ref.vel[i]):.3f} rho? reb {ctxs[ex].counters()[1][0]}")
    e13 = np.abs(P[1][:, :2] - P[3][:, :2]).max(1)
    out.append(f"ex1-ex3 max {e13.max():.2e} at id {int(e13.argmax())}")
    print(" | ".join(out), flush=True)
# top deviating particles at the end
e = np.abs(P[3][:, :2] - ref.pos).max(1)
top = np.argsort(-e)[:12]
for i in top:
    print(i, e[i], ref.pos[i], np.hypot(*ref.pos[i]), np.abs(P[1][i, :2] - ref.pos[i]).max())
