#!/usr/bin/env python3
"""Parity margins and timing of sph_jacobian (GPU) vs the oracle FD Jacobian."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import oracle as O
import sph_inputs as si
from paper_2604_12505_b200 import SphContext

BODY = [0.05, -0.03, 0.4, 0.01, -0.02, 0.05]
t = si.moving_tank(1.0, seed=3, vel=0.02, body=BODY)
ctx = SphContext(t.params, t.pv32(), t.ghost_b, n_rollouts=1)
ctx.set_body_state(np.array([BODY]))
pv = ctx.get_particles(0).astype(np.float64)
x = O.state_vector(pv[:, :2], pv[:, 2:], ctx.get_body_state()[0])
A, B = ctx.jacobian(0)
Ao, Bo = O.jacobian_fd(t.params, x, t.ghost_b)
n = t.n_fluid
print("C1 parity: max|dA|/max|A| = %.3e (acc rows %.3e, body rows %.3e)" % (
    np.abs(A - Ao).max() / np.abs(Ao).max(),
    np.abs(A[2*n:4*n] - Ao[2*n:4*n]).max() / np.abs(Ao[2*n:4*n]).max(),
    np.abs(A[4*n:] - Ao[4*n:]).max() / np.abs(Ao[4*n:]).max()))
ctx.close()
for name, tk in [("C1", si.make_tank(1.0)), ("P0", si.make_tank(1.0, n_first=666)), ("C2", si.make_tank(4.0))]:
    c = SphContext(tk.params, tk.pv32(), tk.ghost_b, n_rollouts=1)
    c.jacobian(0, device=True)
    torch.cuda.synchronize()
    reps = 5 if name != "C2" else 2
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(c.stream)
    for _ in range(reps):
        Ad, Bd = c.jacobian(0, device=True)
    e1.record(c.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    nx = 4 * tk.n_fluid + 6
    t0 = time.time(); ev = torch.linalg.eigvals(Ad) if name != "C2" else None; torch.cuda.synchronize(); te = time.time() - t0
    print(f"{name}: N={tk.n_fluid} n_x={nx} jacobian {ms:.3f} ms ({(nx+3)/ms*1e3:.3e} columns/s), eigvals {te*1e3:.1f} ms")
    c.close()
