"""Thin ctypes binding over libsphb200.so (include/sph.h).  Argument marshalling only:
every step of the SPH path runs in the library's sm_100a kernels.  PyTorch provides the device
workspace, the CUDA stream and device tensors for inputs / outputs.

There is no CPU fallback: if the CUDA library is missing, ``lib()`` raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPH_LIB_PATH") or os.path.join(_HERE, "libsphb200.so")

SPH_OK, SPH_EINVAL, SPH_ENOMEM, SPH_ECUDA, SPH_EBLOWUP, SPH_ESTATE = 0, 1, 2, 3, 4, 6
TIMER_NAMES = ["rebuild", "density", "force", "body", "substep", "sort"]
LIVE_NAMES = ["density", "force", "substep", "tick"]   # SPH_LIVE_* order


class FluidParams(C.Structure):
    _fields_ = [("rho0", C.c_double), ("k", C.c_double), ("alpha", C.c_double),
                ("beta", C.c_double), ("gamma1", C.c_double), ("eps", C.c_double),
                ("h", C.c_double), ("mass", C.c_double), ("w_cb_const", C.c_double),
                ("ghost_pressure_sign", C.c_double), ("gravity", C.c_double * 2),
                ("clamp_negative_pressure", C.c_double)]


class BodyParams(C.Structure):
    _fields_ = [("m", C.c_double), ("J", C.c_double), ("tank_radius", C.c_double)]


class TimeParams(C.Structure):
    _fields_ = [("dt", C.c_double), ("substeps_per_sample", C.c_int), ("rebin_every", C.c_int),
                ("skin", C.c_double), ("rebuild_path", C.c_int), ("exec_path", C.c_int),
                ("skin_max", C.c_double), ("skin_mode", C.c_int)]


class PdAttitude(C.Structure):
    _fields_ = [("Kp", C.c_double), ("Kd", C.c_double), ("theta_ref", C.c_void_p)]


class SphError(RuntimeError):
    pass


_lib = None


def lib():
    """Load libsphb200.so (fails loudly when the CUDA extension was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise SphError(f"CUDA extension missing: {LIB_PATH} (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, dbl = C.c_void_p, C.c_int, C.c_int64, C.c_double
        sig = {
            "sph_workspace_bytes": (C.c_size_t, [vp, vp, vp, i32, i32, i32]),
            "sph_init_tank": (i32, [vp, vp, vp, i32, vp, i32, vp, i32, vp, vp, C.c_size_t, vp]),
            "sph_set_state": (i32, [vp, i32, vp, vp]),
            "sph_set_body_state": (i32, [vp, vp]),
            "sph_get_particles": (i32, [vp, i32, vp, vp]),
            "sph_get_ghosts": (i32, [vp, i32, vp]),
            "sph_step": (i32, [vp, vp, i32, i32]),
            "sph_rollout_batch": (i32, [vp, vp, i32, vp, vp, vp, i32]),
            "sph_get_body_state": (i32, [vp, vp]),
            "sph_settle": (i32, [vp, dbl, i32]),
            "sph_get_status": (i32, [vp, vp, vp, vp]),
            "sph_debug_cells": (i32, [vp, i32, vp, vp]),
            "sph_debug_neighbours": (i32, [vp, i32, vp, vp, i64, vp, vp, i64, vp, vp, i64]),
            "sph_profile_substeps": (i32, [vp, i32, vp]),
            "sph_set_live_timing": (i32, [vp, i32]),
            "sph_get_live_timing": (i32, [vp, vp, vp, i32]),
            "sph_launches_per_substep": (i32, [vp]),
            "sph_launches_per_tick": (i32, [vp]),
            "sph_exec_path": (i32, [vp, vp, vp, vp, vp]),
            "sph_jacobian": (i32, [vp, i32, vp, vp, i32]),
            "sph_eigenvalues": (i32, [vp, i32, vp, vp, i32]),
            "sph_gamma1_estimate": (i32, [vp, i32, dbl, vp, vp, vp]),
            "sph_set_domain": (i32, [vp, i32, i32]),
            "sph_settle_until": (i32, [vp, dbl, dbl, i32, i32, vp, vp]),
            "sph_dd_phase": (i32, [vp, i32, vp, vp, vp, vp]),
            "sph_lpv_scratch_bytes": (C.c_size_t, [i32, i32, i32]),
            "sph_lpv_eval": (i32, [i32, i32, i32, vp, vp, vp, dbl, dbl, vp, vp, vp, vp, C.c_size_t, vp]),
            "sph_lpv_adam": (i32, [i32, i32, vp, vp, vp, vp, dbl, dbl, dbl, dbl, i32, vp, vp]),
            "sph_get_counters": (i32, [vp, vp, vp]),
            "sph_get_sizes": (None, [vp, vp, vp, vp, vp]),
            "sph_last_error": (C.c_char_p, [vp]),
            "sph_destroy": (None, [vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return ["sph_workspace_bytes", "sph_init_tank", "sph_set_state", "sph_set_body_state",
            "sph_get_particles", "sph_get_ghosts", "sph_step", "sph_rollout_batch",
            "sph_get_body_state", "sph_settle", "sph_get_status", "sph_debug_cells",
            "sph_debug_neighbours", "sph_profile_substeps", "sph_set_live_timing", "sph_get_live_timing",
            "sph_launches_per_substep", "sph_launches_per_tick", "sph_exec_path", "sph_get_counters", "sph_jacobian", "sph_eigenvalues",
            "sph_gamma1_estimate", "sph_lpv_scratch_bytes", "sph_lpv_eval", "sph_lpv_adam",
            "sph_set_domain", "sph_dd_phase", "sph_settle_until",
            "sph_get_sizes", "sph_last_error", "sph_destroy"]


def fluid_params(sp) -> FluidParams:
    g = FluidParams(sp.rho0, sp.k, sp.alpha, sp.beta, sp.gamma1, sp.eps, sp.h, sp.mass,
                    sp.w_cb_const, sp.ghost_pressure_sign)
    g.gravity[0] = sp.gx
    g.gravity[1] = sp.gy
    g.clamp_negative_pressure = float(getattr(sp, "clamp_negative_pressure", 0.0))
    return g


def body_params(sp) -> BodyParams:
    return BodyParams(sp.m_body, sp.J_body, sp.R)


def time_params(sp, rebin_every: int = 1, skin: float = 0.0, rebuild_path: int = 0,
                exec_path: int = 0, skin_max: float = 0.0, skin_mode: int = 0) -> TimeParams:
    return TimeParams(sp.dt, int(sp.n_sub), int(rebin_every), float(skin), int(rebuild_path),
                      int(exec_path), float(skin_max), int(skin_mode))


def _ptr(a):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


def _host(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


class SphContext:
    """One batched ensemble of B identical tanks on one GPU (sph_init_tank)."""

    def __init__(self, sp, fluid_pv, ghost_b, n_rollouts: int = 1, rebin_every: int = 1,
                 skin: float = 0.0, device: int = 0, rebuild_path: int = 0, exec_path: int = 0,
                 skin_max: float = 0.0, skin_mode: int = 0):
        import torch
        self.torch = torch
        self.L = lib()
        self.device = torch.device("cuda", device)
        self.fp, self.bp = fluid_params(sp), body_params(sp)
        self.tp = time_params(sp, rebin_every, skin, rebuild_path, exec_path, skin_max, skin_mode)
        pv = _host(fluid_pv, np.float32).reshape(-1, 4)
        gb = _host(ghost_b, np.float64).reshape(-1, 2)
        self.N, self.G, self.B = pv.shape[0], gb.shape[0], int(n_rollouts)
        nbytes = self.L.sph_workspace_bytes(C.byref(self.fp), C.byref(self.bp), C.byref(self.tp),
                                            self.N, self.G, self.B)
        if nbytes == 0:
            raise SphError("invalid parameters (sph_workspace_bytes returned 0)")
        with torch.cuda.device(self.device):
            self.stream = torch.cuda.Stream(self.device)
            self.workspace = torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)
        self.workspace_bytes = int(nbytes)
        ctx = C.c_void_p()
        st = self.L.sph_init_tank(C.byref(self.fp), C.byref(self.bp), C.byref(self.tp), self.N,
                                  pv.ctypes.data, self.G, gb.ctypes.data, self.B,
                                  self.stream.cuda_stream, self.workspace.data_ptr(), nbytes,
                                  C.byref(ctx))
        if st != SPH_OK:
            raise SphError(f"sph_init_tank: {st}: {self.L.sph_last_error(None).decode()}")
        self.ctx = ctx
        self.n_sub = int(sp.n_sub)
        nc = C.c_int()
        self.L.sph_get_sizes(self.ctx, None, None, None, C.byref(nc))
        self.n_cells = nc.value

    # -- helpers ------------------------------------------------------------------------
    def _check(self, st, what):
        if st != SPH_OK:
            msg = self.L.sph_last_error(self.ctx).decode()
            raise SphError(f"{what}: status {st}: {msg}")

    def _dev_in(self, t):
        """Order the context stream after torch's current stream (device inputs)."""
        self.stream.wait_stream(self.torch.cuda.current_stream(self.device))
        return t

    def _dev_out(self):
        self.torch.cuda.current_stream(self.device).wait_stream(self.stream)

    def close(self):
        if getattr(self, "ctx", None):
            self.L.sph_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- state ---------------------------------------------------------------------------
    def set_state(self, fluid_pv, rollout: int = -1, body=None):
        pv = _host(fluid_pv, np.float32).reshape(self.N, 4)
        bd = None if body is None else _host(body, np.float64).reshape(6)
        self._check(self.L.sph_set_state(self.ctx, rollout, pv.ctypes.data,
                                         None if bd is None else bd.ctypes.data), "sph_set_state")

    def set_body_state(self, body):
        bd = _host(body, np.float64).reshape(self.B, 6)
        self._check(self.L.sph_set_body_state(self.ctx, bd.ctypes.data), "sph_set_body_state")

    def get_particles(self, rollout: int = 0, with_rho: bool = False):
        pv = np.zeros((self.N, 4), np.float32)
        rho = np.zeros(self.N, np.float32) if with_rho else None
        self._check(self.L.sph_get_particles(self.ctx, rollout, pv.ctypes.data,
                                             None if rho is None else rho.ctypes.data),
                    "sph_get_particles")
        return (pv, rho) if with_rho else pv

    def get_ghosts(self, rollout: int = 0):
        g = np.zeros((self.G, 4), np.float32)
        self._check(self.L.sph_get_ghosts(self.ctx, rollout, g.ctypes.data), "sph_get_ghosts")
        return g

    def get_body_state(self):
        out = np.zeros((self.B, 6), np.float64)
        self._check(self.L.sph_get_body_state(self.ctx, out.ctypes.data), "sph_get_body_state")
        return out

    def get_status(self):
        st = np.zeros(self.B, np.int32)
        bs = np.zeros(self.B, np.int64)
        bp = np.zeros(self.B, np.int32)
        self._check(self.L.sph_get_status(self.ctx, st.ctypes.data, bs.ctypes.data, bp.ctypes.data),
                    "sph_get_status")
        return st, bs, bp

    # -- dynamics ------------------------------------------------------------------------
    def step(self, u, n_substeps: int = 1):
        """u: [B,3] (numpy -> host path; cuda tensor -> device path)."""
        if hasattr(u, "is_cuda") and u.is_cuda:
            u = self._dev_in(u.contiguous().float())
            self._check(self.L.sph_step(self.ctx, u.data_ptr(), int(n_substeps), 1), "sph_step")
            self._dev_out()
        else:
            uu = _host(np.broadcast_to(np.asarray(u, np.float32), (self.B, 3)), np.float32)
            self._check(self.L.sph_step(self.ctx, uu.ctypes.data, int(n_substeps), 0), "sph_step")

    def settle(self, damping: float, n_steps: int):
        self._check(self.L.sph_settle(self.ctx, float(damping), int(n_steps)), "sph_settle")

    def settle_until(self, damping: float, v_tol: float, max_steps: int, check_every: int = 500):
        """Damped settle until every rollout's largest fluid speed < v_tol; returns
        (substeps taken, final largest speed per rollout)."""
        n = C.c_int(0)
        sp = np.zeros(self.B, np.float32)
        self._check(self.L.sph_settle_until(self.ctx, float(damping), float(v_tol), int(max_steps),
                                            int(check_every), C.byref(n), sp.ctypes.data),
                    "sph_settle_until")
        return n.value, sp

    def rollout(self, u_seq, theta_ref=None, Kp: float = 0.0, Kd: float = 0.0, y_out=None,
                u_applied=None):
        """Multi-rate rollout.  Device tensors -> device path (outputs must be given or are
        allocated as cuda tensors); numpy -> host path.  Returns (y, u_applied)."""
        torch = self.torch
        on_dev = hasattr(u_seq, "is_cuda") and u_seq.is_cuda
        if on_dev:
            K = int(u_seq.shape[1])
            u_seq = self._dev_in(u_seq.contiguous().float())
            if tuple(u_seq.shape) != (self.B, K, 3):
                raise SphError(f"u_seq must be [B, K, 3] = [{self.B}, K, 3], got {tuple(u_seq.shape)}")
            if y_out is None:
                y_out = torch.empty((self.B, K, 6), dtype=torch.float32, device=self.device)
            if u_applied is None:
                u_applied = torch.empty((self.B, K, 3), dtype=torch.float32, device=self.device)
            for nm, t_, shp in (("y_out", y_out, (self.B, K, 6)), ("u_applied", u_applied, (self.B, K, 3))):
                if not (t_.is_cuda and t_.dtype == torch.float32 and t_.is_contiguous() and tuple(t_.shape) == shp):
                    raise SphError(f"{nm} must be a contiguous float32 cuda tensor of shape {shp}")
            th = None if theta_ref is None else theta_ref.contiguous().float()
            if th is not None and tuple(th.shape) != (self.B, K):
                raise SphError(f"theta_ref must be [B, K] = [{self.B}, {K}]")
            pd = None if th is None else PdAttitude(Kp, Kd, th.data_ptr())
            self._check(self.L.sph_rollout_batch(self.ctx, u_seq.data_ptr(), K,
                                                 None if pd is None else C.byref(pd),
                                                 y_out.data_ptr(), u_applied.data_ptr(), 1),
                        "sph_rollout_batch")
            self._dev_out()
            return y_out, u_applied
        u_seq = _host(u_seq, np.float32)
        K = u_seq.shape[1]
        if u_seq.shape != (self.B, K, 3):
            raise SphError(f"u_seq must be [B, K, 3] = [{self.B}, K, 3], got {u_seq.shape}")
        y = y_out if y_out is not None else np.zeros((self.B, K, 6), np.float32)
        ua = u_applied if u_applied is not None else np.zeros((self.B, K, 3), np.float32)
        for nm, a_, shp in (("y_out", y, (self.B, K, 6)), ("u_applied", ua, (self.B, K, 3))):
            if not (isinstance(a_, np.ndarray) and a_.dtype == np.float32 and a_.flags.c_contiguous
                    and a_.shape == shp):
                raise SphError(f"{nm} must be a C-contiguous float32 array of shape {shp}")
        th = None if theta_ref is None else _host(theta_ref, np.float32)
        if th is not None and th.shape != (self.B, K):
            raise SphError(f"theta_ref must be [B, K] = [{self.B}, {K}]")
        pd = None if th is None else PdAttitude(Kp, Kd, _ptr(th))
        self._check(self.L.sph_rollout_batch(self.ctx, _ptr(u_seq), K,
                                             None if pd is None else C.byref(pd), _ptr(y),
                                             _ptr(ua), 0), "sph_rollout_batch")
        return y, ua

    # -- parity / debug -----------------------------------------------------------------
    def debug_cells(self, rollout: int = 0):
        cells = np.zeros((self.N, 2), np.int32)
        grid = np.zeros(4, np.float32)
        self._check(self.L.sph_debug_cells(self.ctx, rollout, cells.ctypes.data, grid.ctypes.data),
                    "sph_debug_cells")
        return cells, grid

    def debug_neighbours(self, rollout: int = 0, cap: int | None = None):
        cap = cap or max(64, 40 * self.N)
        arrs = []
        args = []
        for _ in range(3):
            off = np.zeros(self.N + 1, np.int64)
            idx = np.zeros(cap, np.int32)
            arrs.append((off, idx))
            args += [off.ctypes.data, idx.ctypes.data, cap]
        self._check(self.L.sph_debug_neighbours(self.ctx, rollout, *args), "sph_debug_neighbours")
        return [(off, idx[:off[-1]].copy()) for off, idx in arrs]

    def profile(self, n_substeps: int = 10):
        ms = np.zeros(len(TIMER_NAMES), np.float32)
        self._check(self.L.sph_profile_substeps(self.ctx, int(n_substeps), ms.ctypes.data),
                    "sph_profile_substeps")
        return dict(zip(TIMER_NAMES, ms.tolist()))

    def set_live_timing(self, every: int):
        """Event-record nodes in the tick graph around density / force / substep of every
        `every`-th substep (0 = off); see sph_set_live_timing."""
        self._check(self.L.sph_set_live_timing(self.ctx, int(every)), "sph_set_live_timing")

    def live_timing(self, reset: bool = True):
        """Mean in-situ ms per sample: {"density", "force", "substep", "tick", "samples"}
        (per-substep path: per sampled substep; resident path: "tick" = ms per k_resident
        launch = one slow tick, samples = ticks)."""
        ms = np.zeros(len(LIVE_NAMES), np.float64)
        n = np.zeros(1, np.int64)
        self._check(self.L.sph_get_live_timing(self.ctx, ms.ctypes.data, n.ctypes.data,
                                               1 if reset else 0), "sph_get_live_timing")
        k = int(n[0])
        out = {name: (float(v) / k if k else None) for name, v in zip(LIVE_NAMES, ms)}
        out["samples"] = k
        return out

    def jacobian(self, rollout: int = 0, device: bool = False):
        """Linearization of the continuous-time model at the rollout's current state
        (sph_jacobian): returns (A [n_x, n_x], B [n_x, 3]) float64, x = [pos, vel, r, theta,
        rd, thd].  device=True: CUDA tensors (no host round trip), else numpy arrays."""
        nx = 4 * self.N + 6
        if device:
            torch = self.torch
            A = torch.empty((nx, nx), dtype=torch.float64, device=self.device)
            B = torch.empty((nx, 3), dtype=torch.float64, device=self.device)
            self._dev_in(A)
            self._check(self.L.sph_jacobian(self.ctx, int(rollout), A.data_ptr(), B.data_ptr(), 1),
                        "sph_jacobian")
            self._dev_out()
            return A, B
        A = np.empty((nx, nx), np.float64)
        B = np.empty((nx, 3), np.float64)
        self._check(self.L.sph_jacobian(self.ctx, int(rollout), A.ctypes.data, B.ctypes.data, 0),
                    "sph_jacobian")
        return A, B

    def eigenvalues(self, A):
        """Eigenvalues of a square float64 matrix (sph_eigenvalues, cuSOLVER Xgeev on the
        context stream).  A: CUDA tensor (copied; the result stays on the device) or numpy."""
        torch = self.torch
        if hasattr(A, "is_cuda") and A.is_cuda:
            n = int(A.shape[0])
            work = self._dev_in(A.to(torch.float64).contiguous().clone())
            w = torch.empty((n, 2), dtype=torch.float64, device=self.device)
            self._check(self.L.sph_eigenvalues(self.ctx, n, work.data_ptr(), w.data_ptr(), 1),
                        "sph_eigenvalues")
            self._dev_out()
            return torch.complex(w[:, 0], w[:, 1])
        a = np.array(A, dtype=np.float64, order="C", copy=True)
        n = a.shape[0]
        w = np.empty((n, 2), np.float64)
        self._check(self.L.sph_eigenvalues(self.ctx, n, a.ctypes.data, w.ctypes.data, 0),
                    "sph_eigenvalues")
        return w[:, 0] + 1j * w[:, 1]

    def gamma1_estimate(self, rollout: int = 0, rho_target=None):
        """Analytic gamma1 estimate (Eq. gamma1; sph_gamma1_estimate) on the current
        state of ``rollout``: (gamma1_wall, gamma1_i [N] canonical order, NaN away from the
        wall, sums [N, 2] = (sum_f W, sum_g W) in units of C/h^2)."""
        n = self.N
        g = np.empty(n, np.float32)
        sums = np.empty((n, 2), np.float32)
        wall = C.c_double(0.0)
        rt = float(self.fp.rho0 if rho_target is None else rho_target)
        self._check(self.L.sph_gamma1_estimate(self.ctx, int(rollout), rt, g.ctypes.data,
                                               sums.ctypes.data, C.byref(wall)),
                    "sph_gamma1_estimate")
        return wall.value, g, sums

    def counters(self):
        steps = np.zeros(self.B, np.int64)
        reb = np.zeros(self.B, np.int32)
        self._check(self.L.sph_get_counters(self.ctx, steps.ctypes.data, reb.ctypes.data),
                    "sph_get_counters")
        return steps, reb

    def launches_per_substep(self):
        return int(self.L.sph_launches_per_substep(self.ctx))

    def launches_per_tick(self):
        return int(self.L.sph_launches_per_tick(self.ctx))

    def exec_path(self):
        """(path, {cluster_ctas, threads, slots_per_cta, smem_bytes}) -- path 1 per-substep
        kernels, 2 cooperative tick, 3 resident clusters."""
        v = [C.c_int(0) for _ in range(4)]
        p = int(self.L.sph_exec_path(self.ctx, *[C.byref(x) for x in v]))
        return p, dict(zip(["cluster_ctas", "threads", "slots_per_cta", "smem_bytes"], [x.value for x in v]))
