"""Eigen-trace of the linearized open-loop dynamics along a trajectory.

P:408-413: "linearizations of the continuous-time nonlinear dynamic model are computed along the
simulated trajectories ... performed on the open-loop system dynamics, i.e., excluding the
controller", and Figs. 5-6 plot the eigenvalues at different time instances.  The trajectory runs
on the GPU (sph_rollout_batch, one slow tick per call), the Jacobian at each sampled tick is the
GPU forward-mode linearization (sph_jacobian, float64, device-resident), and the spectrum is the
GPU library eigensolver (sph_eigenvalues: cuSOLVER Xgeev) applied to that device matrix.
"""
from __future__ import annotations

import numpy as np


def eigen_trace(ctx, u_seq, stride: int = 1, rollout: int = 0, theta_ref=None, Kp: float = 0.0,
                Kd: float = 0.0):
    """Advance every rollout of ``ctx`` through ``u_seq`` [B, K, 3] (one slow tick per sample,
    optional PD law as in sph_rollout_batch) and return (times [s], spectra): at ticks
    k = 0, stride, 2 stride, ... the eigenvalues of A = df/dx of ``rollout`` at t = k T_s, i.e.
    before u_k is applied (the sampling convention of P:97-100).  The controller is not part of
    A (u is exogenous)."""
    u_seq = np.ascontiguousarray(u_seq, np.float32)
    B, K, _ = u_seq.shape
    dt = float(ctx.tp.dt) * int(ctx.tp.substeps_per_sample)
    times, spectra = [], []
    for k in range(K):
        if k % max(int(stride), 1) == 0:
            A, _ = ctx.jacobian(rollout, device=True)
            spectra.append(ctx.eigenvalues(A).cpu().numpy())
            times.append(k * dt)
        th = None if theta_ref is None else np.ascontiguousarray(np.asarray(theta_ref)[:, k:k + 1])
        ctx.rollout(u_seq[:, k:k + 1], theta_ref=th, Kp=Kp, Kd=Kd)
    return times, spectra
