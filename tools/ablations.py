#!/usr/bin/env python3
"""SURVEY 8(f) f4 / DESIGN.md readings A1, A4, F4: the P0 tank (666 particles) from its rest
lattice, 3 s without actuation, body pinned, under each reading, on the GPU (and, with --oracle,
the float64 oracle of the same input).  Reports particles outside the wall at the end and, on
the GPU side, the status / substep at which a particle left the cell grid (status 3)."""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import sph_inputs as si  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seconds", type=float, default=3.0)
ap.add_argument("--oracle", action="store_true")
a = ap.parse_args()

from paper_2604_12505_b200 import SphContext  # noqa: E402

s0 = si.D_PAPER
READINGS = {
    "adopted (R1, A1 normalised, A4 repulsive)": {},
    "A4 literal ghost-pressure sign (+)": {"ghost_pressure_sign": 1.0},
    "A1 printed cubic constant 15/(14 pi)": {"w_cb_const": si.W_CB_CONST_PRINTED},
    "R0 lattice dx = 6 mm, m = rho0 dx^2, printed constant": {
        "spacing": s0, "mass": si.RHO0 * s0 * s0, "w_cb_const": si.W_CB_CONST_PRINTED},
    "R0 lattice, normalised constant": {"spacing": s0, "mass": si.RHO0 * s0 * s0},
}
out = []
for name, over in READINGS.items():
    t = si.make_tank(1.0, n_first=666, **over).snapped()
    sp = t.params
    n = int(round(a.seconds / sp.dt))
    ctx = SphContext(sp, t.pv32(), t.ghost_b, n_rollouts=1)
    c0 = time.perf_counter()
    ctx.settle(1.0, n)
    st, bad_step, bad_p = ctx.get_status()
    pv = ctx.get_particles(0).astype(np.float64)
    ctx.close()
    r = np.hypot(pv[:, 0], pv[:, 1])
    rec = {"reading": name, "n_fluid": t.n_fluid, "gpu_status": int(st[0]),
           "gpu_tunnel_time_s": float(bad_step[0] * sp.dt) if st[0] == 3 else None,
           "gpu_outside_wall": int((r > sp.R).sum()), "gpu_max_speed": float(np.abs(pv[:, 2:]).max())}
    if a.oracle:
        import oracle as O
        s = O.State.from_tank(t)
        s.step(n=n, pin_body=True)
        ro = np.hypot(s.pos[:, 0], s.pos[:, 1])
        rec["oracle_outside_wall"] = int((ro > sp.R).sum())
        rec["oracle_max_speed"] = float(np.abs(s.vel).max())
    out.append(rec)
    print(json.dumps(rec), flush=True)
