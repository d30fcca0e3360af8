"""Spatial domain decomposition of one tank over several GPUs.

Replicated-data decomposition (include/sph.h, "Spatial domain decomposition"): every process
holds the whole tank and sorts it by cell identically; process r computes densities, forces and
the integration of its slab of the cell-sorted slots (a band of cell rows), and three all-gathers
per substep make every process's copy whole again:

    phase 0  rebuild if due + densities (own slots)   -> all-gather aux   (8 B / particle)
    phase 1  forces + integration (own slots)         -> all-gather state (16 B / particle)
                                                         and body partials (32 B / warp)
    phase 2  body reduction + body step (every process, identical)

The trajectories are bitwise identical to the single-GPU path (same per-slot arithmetic, same
fixed-order body sum).  The all-gathers run over NCCL (NVLink / NVSwitch) in place on padded
buffers: rank r's slab lives at [r chunk, (r + 1) chunk) of each buffer.  ``LocalGroup`` runs W
slabs in one process on one device with shared buffers (no collective), for tests.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from .binding import SPH_OK, SphError

DD_ALIGN = 1024   # SPH_DD_ALIGN


def slab_ranges(n: int, world: int):
    """Slot ranges of the W slabs: equal chunks, multiples of DD_ALIGN (the last one shorter)."""
    chunk = max(1, math.ceil(math.ceil(n / world) / DD_ALIGN)) * DD_ALIGN
    rng = [(r * chunk, min((r + 1) * chunk, n)) for r in range(world)]
    if any(lo >= hi for lo, hi in rng):
        raise ValueError(f"{n} particles are too few for {world} slabs of {DD_ALIGN}-slot multiples")
    return chunk, rng


def n_partials(n: int) -> int:
    return 8 * math.ceil(n / 256)


class Buffers:
    """Padded exchange buffers on one device: aux [W chunk, 2] f32, state [W chunk, 4] f32,
    part [W chunk / 32, 4] f64."""

    def __init__(self, torch, device, chunk, world):
        self.chunk, self.world = chunk, world
        self.aux = torch.zeros((world * chunk, 2), dtype=torch.float32, device=device)
        self.state = torch.zeros((world * chunk, 4), dtype=torch.float32, device=device)
        self.part = torch.zeros((world * chunk // 32, 4), dtype=torch.float64, device=device)

    def views(self, rank):
        c, p = self.chunk, self.chunk // 32
        return (self.aux[rank * c:(rank + 1) * c], self.state[rank * c:(rank + 1) * c],
                self.part[rank * p:(rank + 1) * p])


def all_gather_inplace(dist, full, rank, group=None):
    """In-place all-gather of rank-ordered equal chunks of ``full`` (NCCL in-place form)."""
    world = dist.get_world_size(group)
    n = full.shape[0] // world
    dist.all_gather_into_tensor(full, full[rank * n:(rank + 1) * n].clone(), group=group)


class DomainPart:
    """One slab of a tank held by a SphContext (single rollout)."""

    def __init__(self, ctx, rank, world, bufs=None):
        if ctx.B != 1:
            raise SphError("domain decomposition needs a single rollout")
        self.ctx, self.rank, self.world = ctx, rank, world
        self.chunk, rngs = slab_ranges(ctx.N, world)
        self.lo, self.hi = rngs[rank]
        st = ctx.L.sph_set_domain(ctx.ctx, self.lo, self.hi)
        if st != SPH_OK:
            raise SphError(f"sph_set_domain: status {st}: {ctx.L.sph_last_error(ctx.ctx).decode()}")
        self.bufs = bufs or Buffers(ctx.torch, ctx.device, self.chunk, world)

    def phase(self, k, u=None):
        uh = None
        if u is not None:
            uh = np.ascontiguousarray(np.asarray(u, np.float32).reshape(3))
        b = self.bufs
        st = self.ctx.L.sph_dd_phase(self.ctx.ctx, k, None if uh is None else uh.ctypes.data,
                                     b.aux.data_ptr(), b.state.data_ptr(), b.part.data_ptr())
        if st != SPH_OK:
            raise SphError(f"sph_dd_phase({k}): status {st}: {self.ctx.L.sph_last_error(self.ctx.ctx).decode()}")


class DistributedTank:
    """The tank decomposed over the processes of a torch.distributed group (one GPU each;
    backend nccl on GPUs).  ``substep(u)`` advances one fast step on every process."""

    def __init__(self, ctx, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        rank = dist.get_rank(group)
        world = dist.get_world_size(group)
        self.part = DomainPart(ctx, rank, world)
        self.torch = ctx.torch
        self.host_staged = dist.get_backend(group) == "gloo"

    def _gather(self, *tensors):
        ctx = self.part.ctx
        cur = self.torch.cuda.current_stream(ctx.device)
        cur.wait_stream(ctx.stream)
        for t in tensors:
            if self.host_staged:      # gloo: control-flow checks only (host copies)
                h = t.cpu()
                all_gather_inplace(self.dist, h, self.part.rank, self.group)
                t.copy_(h)
            else:
                all_gather_inplace(self.dist, t, self.part.rank, self.group)
        ctx.stream.wait_stream(cur)

    def substep(self, u=None):
        b = self.part.bufs
        self.part.phase(0, u)
        self._gather(b.aux)
        self.part.phase(1)
        self._gather(b.state, b.part)
        self.part.phase(2)


class LocalGroup:
    """W slabs of one tank in one process on one device (W contexts sharing the exchange
    buffers; the all-gathers reduce to each context writing its own chunk).  For tests: the
    contexts run one after another, so nothing waits on another process."""

    def __init__(self, ctxs):
        W = len(ctxs)
        self.parts = []
        bufs = None
        for r, c in enumerate(ctxs):
            p = DomainPart(c, r, W, bufs)
            bufs = p.bufs
            self.parts.append(p)
        self.torch = ctxs[0].torch

    def substep(self, u=None):
        for k in range(3):
            for p in self.parts:
                p.phase(k, u if k == 0 else None)
            if len(self.parts) > 1:     # one part: its phases are ordered on its own stream
                self.torch.cuda.synchronize()
