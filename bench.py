#!/usr/bin/env python3
"""Benchmark of the B200-native SPH hot path (contract: see DESIGN.md "Measurement").

Metric (BASELINE.json): particle-updates/s, device-timed, whole job.  One fluid particle
advanced one fast substep = one particle-update.  A bench "step" is one slow tick of the
multi-rate loop: the sample/control kernel plus n_sub = 200 fast substeps
(rebin, density, forces + wall + integration, body) for every rollout of the batch.

Default workload (N = 1): C3 of SURVEY 8(d) -- 1024 independent rollouts of the C2 tank
(ell = 4: 9,261 fluid + 944 ghosts), open-loop excitation inputs, settled start.
With --gpus N (torchrun) each rank runs 1024 rollouts with global-id seeded inputs (weak
scaling, config C5 layout) and the trajectories are gathered to rank 0 with NCCL.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import sph_inputs as si  # noqa: E402

WORKLOADS = {
    # name: (ell, rollouts per GPU, description)
    "C3": (4.0, 1024, "C3: 1024 rollouts per GPU x C2 tank (ell=4, 9261 fluid + 944 ghosts), open-loop excitation"),
    "C2": (4.0, 1, "C2: single C2 tank (9261 + 944), excitation, latency-bound"),
    "C4": (42.0, 1, "C4: single ell=42 tank (1,025,788 + 9,912)"),
    "C1": (1.0, 1, "C1: single ell=1 tank (569 + 236)"),
    "C5": (4.0, 8192, "C5: 8192 rollouts of the C2 tank, manoeuvre profiles 1 and 2 under the PD "
                      "law (P:364-386), sharded by global id, dataset (y, u_applied, status) gathered"),
}
K_TRAIN = 2200   # samples of the identification input train: the C3 horizon, 110 s
METRIC = "particle-updates/sec (device-timed) at 1/2/4/8 B200; % HBM roofline"
UNIT = "particle-updates/s"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--eos-clamp", action="store_true",
                    help="LPV / SETTLE workloads: clamp negative pressures (ablation E1, DESIGN.md)")
    ap.add_argument("--lpv-seqs", type=int, default=1,
                    help="LPV workload: training sequences (the paper: 1)")
    ap.add_argument("--workload", default="C3", choices=sorted(WORKLOADS) + ["LIN", "P0", "C2CL", "SETTLE", "LPV", "C4DD"],
                    help="LIN: linearization (SURVEY 8(f) f1) of the paper's P0 tank; P0: the paper's "
                         "Table 3 benchmark (30 s closed loop); C2CL: the same manoeuvre on the C2 tank (configs[1]); "
                         "none of them is the north-star line")
    ap.add_argument("--rollouts", type=int, default=0, help="override rollouts per GPU")
    ap.add_argument("--window-start", type=int, default=0,
                    help="C3: first tick (within the 2200-sample train, P:431) of the warm-up; the "
                         "timed window is ticks [start + W, start + W + K)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="C5: weak = 1024 rollouts per GPU, strong = 8192 in total")
    ap.add_argument("--long-horizon", action="store_true",
                    help="C3: run the whole 2200-tick train, report the rate per 100-tick window")
    ap.add_argument("--horizon-ticks", type=int, default=2200, help="--long-horizon: ticks to run")
    ap.add_argument("--skin-max", type=float, default=None,
                    help="adaptive Verlet skin upper bound in units of h (DESIGN.md B5; 0 = fixed skin)")
    ap.add_argument("--skin-mode", type=int, default=None, choices=[0, 1],
                    help="with --skin-max > --skin: 0 per-rollout adaptive skin (B5), 1 per-particle (B6)")
    ap.add_argument("--rebuild-path", type=int, default=0, choices=[0, 1, 2],
                    help="sph_time_params.rebuild_path: 0 auto, 1 per-rollout CTA sort, 2 grid-wide kernels")
    ap.add_argument("--exec-path", type=int, default=0, choices=[0, 1, 2, 3],
                    help="sph_time_params.exec_path: 0 auto, 1 per-substep kernels + CUDA graph, "
                         "2 cooperative tick, 3 rollout-resident clusters (opt-in)")
    ap.add_argument("--rebin-every", type=int, default=0,
                    help="1: rebuild cell list + neighbour lists every substep; 0: adaptive (skin)")
    ap.add_argument("--skin", type=float, default=None,
                    help="Verlet skin in units of h (adaptive); default 0.15 for the open-loop ensembles, "
                         "0.5 for the closed-loop manoeuvre runs (P0, C2CL: energetic flow, see DESIGN.md), "
                         "0.8 for C4 (wall-layer particles at 0.3-0.5 m/s trip a small skin every 2 substeps)")
    ap.add_argument("--live-every", type=int, default=16,
                    help="live kernel timing: event nodes every N-th substep of the timed ticks (0 = off)")
    ap.add_argument("--settle-seconds", type=float, default=None,
                    help="damped settle of the initial tank (reading A17; ell=4 needs >= 4 s); default 4 s, "
                         "C4: 1,000 damped substeps (SURVEY 8(d)) when no settled snapshot exists")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-substeps", type=int, default=20)
    return ap.parse_args(argv)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # control-flow check of the multi-rank path on a 1-GPU box (tools/check_multirank_bench.sh):
    # every rank on device 0, gloo collectives; never used for a measured number
    if os.environ.get("BENCH_SINGLE_DEVICE_CHECK") == "1":
        local = 0
    return rank, world, local


# ------------------------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ------------------------------------------------------------------------------------------
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.index)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ------------------------------------------------------------------------------------------
# workload construction
# ------------------------------------------------------------------------------------------
def make_workload(name):
    ell, _, _ = WORKLOADS[name]
    t = si.make_tank(ell)
    return t


def settled_start(t, seconds, device):
    """Settled start state: the committed oracle-settled snapshot when one exists for this
    refinement (tools/make_settled.py; independent of the CUDA path, so the benchmark input
    does not change with the kernels), else a damped settle on the GPU."""
    ell = t.params.ell
    path = os.path.join(ROOT, "bench_data", f"settled_ell{ell:g}.npz")
    if os.path.exists(path):
        d = np.load(path)
        pv = np.ascontiguousarray(d["pv"], dtype=np.float32)
        if pv.shape == (t.n_fluid, 4):
            SETTLE_INFO.update(source=os.path.relpath(path, ROOT), seconds=float(d["seconds"]),
                               residual_max_speed=float(np.abs(pv[:, 2:]).max()))
            return pv
    SETTLE_INFO["source"] = "GPU damped settle"
    return settle_on_gpu(t, seconds, device)


def settle_on_gpu(t, seconds, device):
    """Damped settle (reading A17) of one tank on the GPU (product path, untimed)."""
    from paper_2604_12505_b200 import SphContext
    ctx = SphContext(t.params, t.pv32(), t.ghost_b, n_rollouts=1, device=device, rebin_every=0,
                     skin=0.1 * t.params.h)
    n = int(round(seconds / t.params.dt))
    ctx.settle(math.exp(-10.0 * t.params.dt), n)
    pv = ctx.get_particles(0)
    st = ctx.get_status()[0]
    ctx.close()
    if st[0] != 0:
        raise RuntimeError(f"settle failed with status {st[0]}")
    SETTLE_INFO["residual_max_speed"] = float(np.abs(pv[:, 2:]).max())
    SETTLE_INFO["seconds"] = seconds
    return pv


SETTLE_INFO = {}


def inputs_for(global_ids, K):
    return si.ensemble_inputs(global_ids, K)[0]           # [B, K, 3] float32, seed 1000 + id


# ------------------------------------------------------------------------------------------
# oracle baselines (test infrastructure; only here and in tests)
# ------------------------------------------------------------------------------------------
def _oracle_sample(args):
    """Run the float64 oracle on one rollout of the workload for n substeps; returns
    (particle-updates, seconds)."""
    name, pv, gid, n_sub_total, u_seq_row = args
    import oracle as O
    t = make_workload(name)
    s = O.State(t.params, pv[:, :2].astype(np.float64), pv[:, 2:].astype(np.float64), t.ghost_b)
    n_sub = t.params.n_sub
    t0 = time.perf_counter()
    done = 0
    k = 0
    while done < n_sub_total:
        m = min(n_sub, n_sub_total - done)
        s.step(tuple(float(x) for x in u_seq_row[k % len(u_seq_row)]), n=m)
        done += m
        k += 1
    dt = time.perf_counter() - t0
    return t.n_fluid * n_sub_total, dt


def cpu_baseline(name, pv, budget_s=15.0):
    """Oracle timed on the host cores: independent rollouts of the same workload, one process
    per core, each sized to ~budget_s of CPU work (bounded sample)."""
    import concurrent.futures as cf
    import oracle as O
    O.build()
    cores = max(1, min(os.cpu_count() or 1, 32))
    u = inputs_for([0], 8)[0]
    # calibrate on a few substeps
    upd, sec = _oracle_sample((name, pv, 0, 4, u))
    per_sub = sec / 4
    n = max(4, int(budget_s / per_sub))
    with cf.ProcessPoolExecutor(max_workers=cores) as ex:
        t0 = time.perf_counter()
        res = list(ex.map(_oracle_sample, [(name, pv, g, n, u) for g in range(cores)]))
        wall = time.perf_counter() - t0
    total = sum(r[0] for r in res)
    return {"value": total / wall, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{cores} independent rollouts x {n} substeps of the {name} tank "
                      f"({WORKLOADS[name][0]:g}-refined, {int(res[0][0] / n)} fluid particles), "
                      f"float64 C oracle, one process per core, {wall:.1f} s wall"}


def run_reference(a):
    """--impl reference: the oracle as it stands on the host cores, same metric/config."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle as O
    O.build()
    name = a.workload
    t = make_workload(name)
    pv = t.pv32()      # lattice start (the settle is untimed and not part of the metric)
    u = inputs_for([0], 8)[0]
    import concurrent.futures as cf
    cores = max(1, min(os.cpu_count() or 1, 32))
    n_per = 20 if name != "C4" else 1
    times = []
    total_upd = 0
    with cf.ProcessPoolExecutor(max_workers=cores) as ex:
        for it in range(a.warmup + a.steps):
            t0 = time.perf_counter()
            res = list(ex.map(_oracle_sample, [(name, pv, g, n_per, u) for g in range(cores)]))
            dt = time.perf_counter() - t0
            if it >= a.warmup:
                times.append(dt)
                total_upd += sum(r[0] for r in res)
    wall = sum(times)
    value = total_upd / wall
    ell, Bg, desc = WORKLOADS[name]
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": 1e3 * wall / max(a.steps, 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": desc, "sample": f"{cores} rollouts x {n_per} substeps per step"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{cores} independent rollouts x {n_per} substeps per step, "
                                       f"{a.steps} steps"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------
def algorithmic_bytes(kernel, N, G, B, n_sub=1):
    """Bytes the method must move per launch: float32 SoA arrays
    touched once.  density: read x (8) write (rho, P/rho^2) (8) per particle + ghosts (16);
    force: read x, v (16) + aux (8), write x, v (16) per particle + ghosts (16 + 8).
    Neighbour-list bytes are implementation overhead and are not credited."""
    if kernel == "density":
        return B * (16 * N + 16 * G)
    if kernel == "force":
        return B * (40 * N + 24 * G)
    if kernel == "resident":   # one launch = n_sub whole substeps (density + force) of every rollout
        return B * n_sub * (56 * N + 40 * G)
    return None


def traffic_from_profiles(kernel, workload):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        d = json.load(open(p))
        return d.get(workload, {}).get(kernel)
    except Exception:
        return None


def run_ours(a):
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    if world > 1 and not dist.is_initialized():
        if os.environ.get("BENCH_SINGLE_DEVICE_CHECK") == "1":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2604_12505_b200 import SphContext
    name = a.workload
    ell, B, desc = WORKLOADS[name]
    c5 = name == "C5"
    if c5:   # strong: 8192 rollouts in total; weak: 1024 per GPU
        n_total = B if a.scaling == "strong" else 1024 * world
        from paper_2604_12505_b200.ensemble import shard
        gids = list(shard(n_total, world, rank))
        B = len(gids)
    if a.rollouts:
        B = a.rollouts
    if not c5:
        gids = list(range(rank * B, (rank + 1) * B))
        n_total = world * B
    t = make_workload(name)
    sp = t.params
    pv0 = settled_start(t, a.settle_seconds, local)
    K_all = a.warmup + a.steps
    w0 = a.window_start
    th_host = None
    if c5:   # profiles 1 / 2 from their start, PD attitude law
        from paper_2604_12505_b200.ensemble import ensemble_inputs_for
        u_host, th_host = ensemble_inputs_for(gids, K_all, "profiles", n_total)
        w0 = 0
        window = {"ticks": [a.warmup, K_all], "seconds": [a.warmup * 0.05, K_all * 0.05],
                  "inputs": "manoeuvre profiles 1 (ids < n/2) and 2, PD law"}
    else:    # the 2200-sample identification train; the timed window is a slice of it
        if w0 + K_all > K_TRAIN:
            raise SystemExit(f"window [{w0}, {w0 + K_all}) exceeds the {K_TRAIN}-sample train")
        u_host = np.ascontiguousarray(inputs_for(gids, K_TRAIN)[:, w0:w0 + K_all])
        window = {"ticks": [w0 + a.warmup, w0 + K_all], "train_samples": K_TRAIN,
                  "seconds": [(w0 + a.warmup) * 0.05, (w0 + K_all) * 0.05],
                  "inputs": "open-loop multisine + pulse train (P:430-432)"}
    skin = a.skin * sp.h if a.rebin_every == 0 else 0.0
    ctx = SphContext(sp, pv0, t.ghost_b, n_rollouts=B, rebin_every=a.rebin_every,
                     skin=skin, device=local, exec_path=a.exec_path, rebuild_path=a.rebuild_path, skin_max=a.skin_max * sp.h, skin_mode=a.skin_mode)
    u_dev = torch.from_numpy(u_host).to(dev)
    th_dev = torch.from_numpy(th_host).to(dev) if th_host is not None else None
    pdkw = dict(Kp=sp.Kp, Kd=sp.Kd) if th_host is not None else {}
    y_dev = torch.empty((B, K_all, 6), dtype=torch.float32, device=dev)
    ua_dev = torch.empty((B, K_all, 3), dtype=torch.float32, device=dev)
    # live kernel timing: event-record nodes in the tick graph around density / force of every
    # LIVE_EVERY-th substep of the timed rollout (enabled before the warm-up, which captures
    # the graph; accumulators reset after it)
    ctx.set_live_timing(a.live_every)
    # warm-up (also captures the per-tick CUDA graph)
    if a.warmup:
        ctx.rollout(u_dev[:, :a.warmup].contiguous(), y_out=y_dev[:, :a.warmup].contiguous(),
                    u_applied=ua_dev[:, :a.warmup].contiguous(),
                    theta_ref=th_dev[:, :a.warmup].contiguous() if th_dev is not None else None, **pdkw)
    torch.cuda.synchronize(dev)
    ctx.live_timing(reset=True)
    steps0, reb0 = ctx.counters()
    u_timed = u_dev[:, a.warmup:].contiguous()
    th_timed = th_dev[:, a.warmup:].contiguous() if th_dev is not None else None
    y_timed = torch.empty((B, a.steps, 6), dtype=torch.float32, device=dev)
    ua_timed = torch.empty((B, a.steps, 3), dtype=torch.float32, device=dev)
    clocks = Clocks(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.nvtx.range_push("timed")   # ncu --nvtx-include "timed/" selects these launches
    e0.record(ctx.stream)
    ctx.rollout(u_timed, y_out=y_timed, u_applied=ua_timed, theta_ref=th_timed, **pdkw)
    e1.record(ctx.stream)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ck = clocks.stop()
    ms = e0.elapsed_time(e1)
    live = ctx.live_timing(reset=True)
    ctx.set_live_timing(0)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    st = ctx.get_status()[0]
    n_failed = int((st != 0).sum())
    steps_done, rebuilds = ctx.counters()
    win_steps, win_reb = steps_done - steps0, rebuilds - reb0   # the timed window only
    y_checksum = float(y_timed.double().abs().sum().item())   # determinism monitor
    updates = n_total * t.n_fluid * sp.n_sub * a.steps
    value = updates / (ms_max / 1e3)
    # NCCL gather of the trajectory dataset (y, u_applied, status; config C5 -- the only
    # collective on the path), timed separately after the timed region
    gather_ms = None
    if world > 1:
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        from paper_2604_12505_b200.ensemble import gather_dataset
        g0.record()
        yg, uag, stg = gather_dataset(y_timed, ua_timed, torch.from_numpy(st).to(dev))
        g1.record()
        torch.cuda.synchronize(dev)
        gather_ms = g0.elapsed_time(g1)
        assert yg.shape[0] == n_total
    # ---- per-kernel device times (CUDA events on the context stream, same data) -----------
    prof = ctx.profile(a.profile_substeps)
    kern = {k: v for k, v in prof.items() if k != "substep"}
    # dominant kernel and its duration per substep: live in-graph events of the timed region
    # (k_force = the sum of its launches in a substep); isolated timings as context.
    # Resident path: the tick is ONE launch (k_resident), timed live around every launch.
    exec_path, res_shape = ctx.exec_path()
    if exec_path == 3:
        top = "resident"
        kms = live["tick"] if live["samples"] else prof["substep"] * sp.n_sub
        kms_src = (f"live: CUDA events around every k_resident launch of the timed region "
                   f"({live['samples']} launches = ticks)" if live["samples"] else
                   "isolated: sph_profile_substeps after the timed region")
    elif live["samples"]:
        top = max(("density", "force"), key=lambda k: live[k])
        kms, kms_src = live[top], f"live: CUDA event nodes in the timed tick graph, every {a.live_every}th substep ({live['samples']} samples)"
    else:
        top = max(("density", "force"), key=lambda k: kern[k])
        kms, kms_src = kern[top], "isolated: sph_profile_substeps after the timed region"
    alg = algorithmic_bytes(top, t.n_fluid, t.n_ghost, B, sp.n_sub)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = peaks.get("hbm_gbs", 6650.0)
    achieved = alg / (kms / 1e3) / 1e9
    roof = {"bound": "hbm", "kernel": f"k_{top}", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": traffic_from_profiles(top, name),
            "exec_path": exec_path, "resident_shape": res_shape if exec_path == 3 else None,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if peaks else "fallback 6.65 TB/s",
            "algorithmic_bytes_per_launch": alg, "kernel_ms": kms, "kernel_ms_source": kms_src,
            "kernel_share_of_step": (kms * a.steps / ms_max if exec_path == 3 else
                                     (kms / live["substep"] if live["samples"] else kms / prof["substep"])),
            "live_ms": {k: live[k] for k in ("density", "force", "substep", "tick")},
            "isolated_ms": kern, "substep_ms_isolated": prof["substep"]}
    # the resource that binds these kernels: instruction issue.  Warp
    # instructions per launch from the committed ncu capture, over the same live time, against
    # 4 issue slots per SM per cycle at the SM clock measured during the timed region
    inst = traffic_from_profiles(top + "_inst", name)
    if inst:
        ipk = inst / (kms / 1e3) / 1e9
        ipeak = 148 * 4 * ck.get("sm_mhz", 1965.0) / 1e3 if isinstance(ck, dict) and ck.get("sm_mhz") else 148 * 4 * 1.965
        roof["issue"] = {"bound": "issue", "achieved": ipk, "peak": ipeak, "unit": "G warp-instructions/s",
                         "frac": ipk / ipeak, "instructions_per_launch": inst,
                         "source": "smsp__inst_executed.sum per launch, profiles/traffic.json (ncu --set full)"}
    launches = a.steps * ctx.launches_per_tick()
    ctx.close()
    del ctx
    # ---- e2e: the same ticks through the public API with HOST buffers ----------------------
    # A fresh context from the same start runs the W warm-up ticks (device path, untimed, also
    # captures the tick graph), then the K timed ticks one sph_rollout_batch call per tick with
    # pinned host buffers: the H2D copy of u_k and the D2H read of y_k and u_applied inside.
    K_e2e = a.steps
    u_pin = [torch.from_numpy(np.ascontiguousarray(u_host[:, a.warmup + k:a.warmup + k + 1])).pin_memory()
             for k in range(K_e2e)]
    th_pin = [torch.from_numpy(np.ascontiguousarray(th_host[:, a.warmup + k:a.warmup + k + 1])).pin_memory()
              for k in range(K_e2e)] if th_host is not None else None
    y_pin = [torch.empty((B, 1, 6), dtype=torch.float32).pin_memory() for _ in range(K_e2e)]
    ua_pin = [torch.empty((B, 1, 3), dtype=torch.float32).pin_memory() for _ in range(K_e2e)]
    ctx2 = SphContext(sp, pv0, t.ghost_b, n_rollouts=B, rebin_every=a.rebin_every, skin=skin,
                      device=local, exec_path=a.exec_path, rebuild_path=a.rebuild_path, skin_max=a.skin_max * sp.h, skin_mode=a.skin_mode)
    if a.warmup > 1:
        ctx2.rollout(u_dev[:, :a.warmup - 1].contiguous(), y_out=y_dev[:, :a.warmup - 1].contiguous(),
                     u_applied=ua_dev[:, :a.warmup - 1].contiguous(),
                     theta_ref=th_dev[:, :a.warmup - 1].contiguous() if th_dev is not None else None, **pdkw)
    if a.warmup:   # the last warm-up tick through the host-pointer path (allocates its staging)
        uw = torch.from_numpy(np.ascontiguousarray(u_host[:, a.warmup - 1:a.warmup])).pin_memory()
        thw = (np.ascontiguousarray(th_host[:, a.warmup - 1:a.warmup]) if th_host is not None else None)
        ctx2.rollout(uw.numpy(), y_out=torch.empty((B, 1, 6)).pin_memory().numpy(),
                     u_applied=torch.empty((B, 1, 3)).pin_memory().numpy(), theta_ref=thw, **pdkw)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    x0 = torch.cuda.Event(enable_timing=True)
    x1 = torch.cuda.Event(enable_timing=True)
    x0.record(ctx2.stream)
    for k in range(K_e2e):
        ctx2.rollout(u_pin[k].numpy(), y_out=y_pin[k].numpy(), u_applied=ua_pin[k].numpy(),
                     theta_ref=th_pin[k].numpy() if th_pin is not None else None, **pdkw)
    x1.record(ctx2.stream)
    torch.cuda.synchronize(dev)
    e2e_ms = x0.elapsed_time(x1)
    e2e_t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = n_total * t.n_fluid * sp.n_sub * K_e2e / (float(e2e_t.item()) / 1e3)
    y_e2e = np.concatenate([y.numpy() for y in y_pin], axis=1)
    e2e_matches = bool(np.array_equal(y_e2e, y_timed.cpu().numpy()))
    ctx2.close()
    if rank != 0:
        return
    cpu = None
    if world == 1 and not a.no_cpu_baseline:
        try:
            cpu = cpu_baseline(name, pv0)
        except Exception as ex:  # never fail the bench line on the baseline
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "oracle", "sample": f"failed: {ex}"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms_max / a.steps, "higher_is_better": True,
        "scaling": a.scaling if c5 else "weak", "vs_baseline": None, "dtype": "f32 (body f64)",
        "data": "synthetic (seeded lattice tank, " + ("oracle-settled snapshot" if SETTLE_INFO.get("source", "").startswith("bench_data") else "GPU damped settle") + (", manoeuvre profiles 1/2 + PD law)" if c5 else ", multisine+pulse excitation)"),
        "config": {"workload": desc, "rollouts_per_gpu": B, "fluid_per_rollout": t.n_fluid,
                   "ghosts_per_rollout": t.n_ghost, "substeps_per_step": sp.n_sub,
                   "dt": sp.dt, "rebin_every": a.rebin_every, "skin_h": a.skin, "skin_max_h": a.skin_max,
                   "parallelism": f"ensemble dp{world}",
                   "l2": (f"no flush: working set {ctx_bytes_gb(t, B):.2f} GB > 126 MB L2"
                          if ctx_bytes_gb(t, B) > 0.126 else
                          f"working set {ctx_bytes_gb(t, B):.3f} GB fits the 126 MB L2 (not flushed)"),
                   "failed_rollouts": n_failed, "gather_ms": gather_ms, "settle": SETTLE_INFO,
                   "timed_window": window, "rollouts_total": n_total,
                   "substeps_per_rebuild": float(win_steps.mean() / max(win_reb.mean(), 1e-9)),
                   "y_checksum": y_checksum},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": B * (3 + (1 if c5 else 0)) * 4,
                "d2h_bytes_per_step": B * (6 + 3) * 4, "steps": K_e2e,
                "same_ticks_as_timed_region": True, "y_bitwise_equal_to_timed_region": e2e_matches},
        "gpu_launches": launches,
        "clocks": ck,
        "roofline": roof,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def run_horizon(a):
    """--long-horizon: the C3 batch over the WHOLE 2200-sample identification train (110 s,
    P:431), timed per 100-tick window with CUDA events (one host sync per window), with the
    rebuild count per window: how the rate moves as the excitation proceeds."""
    import torch
    from paper_2604_12505_b200 import SphContext
    _, _, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    ell, B, desc = WORKLOADS["C3"]
    if a.rollouts:
        B = a.rollouts
    t = make_workload("C3")
    sp = t.params
    pv0 = settled_start(t, a.settle_seconds, local)
    u = torch.from_numpy(inputs_for(range(B), K_TRAIN)).to(dev)
    ctx = SphContext(sp, pv0, t.ghost_b, n_rollouts=B, rebin_every=0, skin=a.skin * sp.h,
                     device=local, exec_path=a.exec_path, rebuild_path=a.rebuild_path, skin_max=a.skin_max * sp.h, skin_mode=a.skin_mode)
    y = torch.empty((B, K_TRAIN, 6), dtype=torch.float32, device=dev)
    ua = torch.empty((B, K_TRAIN, 3), dtype=torch.float32, device=dev)
    win = 100
    rows = []
    clocks = Clocks(local)
    clocks.start()
    n_ticks = min(K_TRAIN, a.horizon_ticks)
    for w0 in range(0, n_ticks, win):
        s0, r0 = ctx.counters()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        yw, uaw = y[:, w0:w0 + win].contiguous(), ua[:, w0:w0 + win].contiguous()
        ctx.rollout(u[:, w0:w0 + win].contiguous(), y_out=yw, u_applied=uaw)
        e1.record(ctx.stream)
        torch.cuda.synchronize(dev)
        y[:, w0:w0 + win] = yw
        ms = e0.elapsed_time(e1)
        s1, r1 = ctx.counters()
        st = ctx.get_status()[0]
        rows.append({"ticks": [w0, w0 + win], "seconds": [w0 * 0.05, (w0 + win) * 0.05],
                     "value": B * t.n_fluid * sp.n_sub * win / (ms / 1e3), "ms_per_tick": ms / win,
                     "substeps_per_rebuild": float((s1 - s0).mean() / max((r1 - r0).mean(), 1e-9)),
                     "failed_rollouts": int((st != 0).sum())})
        print(json.dumps(rows[-1]), flush=True)
    ck = clocks.stop()
    # isolated per-kernel times in the state the horizon ends in (after the timed windows)
    prof_end = ctx.profile(a.profile_substeps)
    tot_ms = sum(r["ms_per_tick"] * win for r in rows)
    line = {"metric": METRIC, "mode": "long-horizon", "workload": desc, "rollouts": B,
            "train_ticks": n_ticks, "value": B * t.n_fluid * sp.n_sub * n_ticks / (tot_ms / 1e3),
            "unit": UNIT, "exec_path": ctx.exec_path()[0], "skin_h": a.skin, "skin_max_h": a.skin_max,
            "windows": rows, "isolated_ms_at_end": prof_end,
            "clocks": ck, "y_finite": bool(torch.isfinite(y).all().item())}
    ctx.close()
    print(json.dumps(line), flush=True)


def ctx_bytes_gb(t, B):
    return B * t.n_fluid * 64 / 1e9


# ------------------------------------------------------------------------------------------
# Linearization: full Jacobians of the continuous-time model
# ------------------------------------------------------------------------------------------
LIN_METRIC = "Jacobians/s (A = df/dx, B = df/du, float64 forward mode) of the P0 tank"


def lin_point(device):
    """P0 tank (the paper's 666-particle benchmark) after 0.2 s of actuation
    u = (5 N, 2 N, 1 N m) from the lattice: an active operating point (GPU product path)."""
    from paper_2604_12505_b200 import SphContext
    t = si.make_tank(1.0, n_first=666)
    ctx = SphContext(t.params, t.pv32(), t.ghost_b, n_rollouts=1, device=device)
    ctx.step(np.array([[5.0, 2.0, 1.0]], np.float32), 200)
    return t, ctx


def run_linearize(a):
    import torch
    rank, world, local = dist_env()
    if rank != 0:
        return
    torch.cuda.set_device(local)
    t, ctx = lin_point(local)
    nx = 4 * t.n_fluid + 6
    for _ in range(max(a.warmup, 1)):
        A, B = ctx.jacobian(0, device=True)
    torch.cuda.synchronize()
    clocks = Clocks(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ctx.stream)
    for _ in range(a.steps):
        A, B = ctx.jacobian(0, device=True)
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    ck = clocks.stop()
    ms = e0.elapsed_time(e1) / a.steps
    # e2e: host buffers through the C ABI (D2H of A and B inside)
    x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    x0.record(ctx.stream)
    for _ in range(2):
        Ah, Bh = ctx.jacobian(0)
    x1.record(ctx.stream)
    torch.cuda.synchronize()
    e2e_ms = x0.elapsed_time(x1) / 2
    # eigenvalues of the device matrix (sph_eigenvalues: cuSOLVER Xgeev, a library call)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev = ctx.eigenvalues(A)
    torch.cuda.synchronize()
    eig_ms = (time.perf_counter() - t0) * 1e3
    out_bytes = 8.0 * (nx * nx + 3 * nx)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = peaks.get("hbm_gbs", 6650.0)
    achieved = out_bytes / (ms / 1e3) / 1e9
    cpu = None
    if not a.no_cpu_baseline:
        import oracle as O
        pv = ctx.get_particles(0).astype(np.float64)
        x = O.state_vector(pv[:, :2], pv[:, 2:], ctx.get_body_state()[0])
        c0 = time.perf_counter()
        O.jacobian_fd(t.params, x, t.ghost_b)
        dt = time.perf_counter() - c0
        cpu = {"value": 1.0 / dt, "unit": "Jacobians/s", "cores": 1, "kind": "oracle",
               "sample": f"1 central-difference Jacobian of the same P0 point (2 x {nx + 3} evaluations of f), float64 C oracle, 1 thread, {dt:.1f} s"}
    ctx.close()
    line = {
        "metric": LIN_METRIC, "value": 1e3 / ms, "unit": "Jacobians/s", "n_gpus": 1, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "none",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (P0 lattice tank, 0.2 s actuated)",
        "config": {"workload": f"LIN: P0 tank (666 fluid + 236 ghosts), n_x = {nx}, columns {nx + 3}",
                   "columns_per_s": (nx + 3) * 1e3 / ms, "eig_ms_cusolver_xgeev": eig_ms,
                   "spectral_radius": float(ev.abs().max())},
        "e2e": {"value": 1e3 / e2e_ms, "unit": "Jacobians/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": int(out_bytes)},
        "gpu_launches": a.steps * 6,
        "clocks": ck,
        "roofline": {"bound": "hbm", "kernel": "sph_jacobian (all launches)", "achieved": achieved,
                     "peak": hbm, "unit": "GB/s", "frac": achieved / hbm, "traffic": None,
                     "note": "algorithmic bytes = the dense float64 A and B written once; at P0 size the call is launch/latency bound"},
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# P0: the paper's own benchmark (Table 3): 666 + 236 particles, manoeuvre profile 1
# under the PD attitude law, 30 s of simulated time at dt = 1 ms
# ------------------------------------------------------------------------------------------
P0_METRIC = "SPH simulation time of manoeuvre profile 1, 30 s closed loop (paper Table 3)"
P0_PAPER_S = 9.9093   # RTX 2000 Ada laptop GPU, JAX (context, not the target)


def run_p0(a, closed_loop_c2=False):
    """P0 (the paper's Table 3 tank) or, with closed_loop_c2, the C2 tank (configs[1]: paper
    resolution x4, one manoeuvre, closed loop): profile 1 + PD law over 30 s."""
    import torch
    rank, world, local = dist_env()
    if rank != 0:
        return
    torch.cuda.set_device(local)
    from paper_2604_12505_b200 import SphContext
    t = si.make_tank(4.0) if closed_loop_c2 else si.make_tank(1.0, n_first=666)
    sp = t.params
    K = int(round(30.0 / (sp.dt * sp.n_sub)))                # 600 slow ticks of 50 ms
    u, th = si.profile(1, K)
    u = u.astype(np.float32)[None]
    th = th.astype(np.float32)[None]
    # damped settle (reading A17, untimed): the oracle-settled C2 snapshot, else 2 s on the GPU
    if closed_loop_c2:
        pv0 = settled_start(t, a.settle_seconds, local)
    else:
        ctx = SphContext(sp, t.pv32(), t.ghost_b, n_rollouts=1, rebin_every=0, skin=a.skin * sp.h,
                         device=local)
        ctx.settle(math.exp(-10.0 * sp.dt), int(2.0 / sp.dt))
        pv0 = ctx.get_particles(0)
        ctx.close()
    ctx = SphContext(sp, pv0, t.ghost_b, n_rollouts=1, rebin_every=0, skin=a.skin * sp.h, device=local,
                     exec_path=a.exec_path)
    dev = torch.device("cuda", local)
    ud, thd = torch.from_numpy(u).to(dev), torch.from_numpy(th).to(dev)
    y = torch.empty((1, K, 6), dtype=torch.float32, device=dev)
    ua = torch.empty((1, K, 3), dtype=torch.float32, device=dev)
    # warm-up: capture the tick graph with 2 ticks on a throwaway copy of the state
    ctx.rollout(ud[:, :2].contiguous(), theta_ref=thd[:, :2].contiguous(), Kp=sp.Kp, Kd=sp.Kd)
    ctx.set_state(pv0, rollout=0, body=np.zeros(6))
    torch.cuda.synchronize()
    clocks = Clocks(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ctx.stream)
    ctx.rollout(ud, theta_ref=thd, Kp=sp.Kp, Kd=sp.Kd, y_out=y, u_applied=ua)
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    ck = clocks.stop()
    secs = e0.elapsed_time(e1) / 1e3
    steps = K * sp.n_sub
    st = ctx.get_status()[0]
    n_steps, n_reb = ctx.counters()
    lps = ctx.launches_per_substep()
    theta_end = float(y[0, -1, 2])
    cpu = None
    if not a.no_cpu_baseline:
        import oracle as O
        s = O.State(sp, pv0[:, :2].astype(np.float64), pv0[:, 2:].astype(np.float64), t.ghost_b)
        n_t = 4 if closed_loop_c2 else 40                         # a bounded sample, 1 thread
        c0 = time.perf_counter()
        s.rollout(u[0, :n_t], sp.n_sub, theta_ref=th[0, :n_t], Kp=sp.Kp, Kd=sp.Kd)
        dt = time.perf_counter() - c0
        cpu = {"value": dt * K / n_t, "unit": "s", "cores": 1, "kind": "oracle",
               "sample": f"first {n_t} of {K} ticks ({n_t * sp.n_sub} steps), float64 C oracle, 1 thread, "
                         f"{dt:.1f} s, extrapolated to the 30 s horizon"}
    ctx.close()
    if closed_loop_c2:
        metric, vsb = "SPH simulation time of manoeuvre profile 1, 30 s closed loop, C2 tank", None
        data = "synthetic (C2 lattice tank, oracle-settled snapshot, profile 1 + PD law)"
        wl = f"C2CL: C2 tank (9261 fluid + 944 ghosts), dt 0.25 ms, {K} ticks x {sp.n_sub} substeps (configs[1])"
    else:
        metric, vsb = P0_METRIC, secs / P0_PAPER_S
        data = "synthetic (P0 lattice tank, 2 s GPU damped settle, profile 1 + PD law)"
        wl = "P0: paper tank, 666 fluid + 236 ghosts, dt 1 ms, 600 ticks x 50 substeps"
    line = {
        "metric": metric, "value": secs, "unit": "s", "n_gpus": 1, "steps": 1, "warmup": 1,
        "ms_per_step": secs * 1e3, "higher_is_better": False, "scaling": "none",
        "vs_baseline": vsb, "dtype": "f32 (body f64)",
        "data": data,
        "config": {"workload": wl, "steps_per_s": steps / secs, "skin_h": a.skin,
                   "substeps": steps, "us_per_substep": secs * 1e6 / steps,
                   "particle_updates_per_s": t.n_fluid * steps / secs,
                   "paper_seconds": P0_PAPER_S, "paper_hardware": "RTX 2000 Ada laptop GPU, JAX (P:391, P:490)",
                   "status": int(st[0]), "theta_end_rad": theta_end,
                   "substeps_per_rebuild": float(n_steps[0] / max(int(n_reb[0]), 1)),
                   "path": "cooperative tick" if lps == 0 else f"{lps} kernels per substep"},
        "gpu_launches": K * (1 + (sp.n_sub * lps if lps > 0 else 1)),
        "clocks": ck,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def run_settle(a):
    """--workload SETTLE: the paper's initialisation -- fluid
    spawned at random in the C2 tank, damped settle (reading A17, body pinned) for 3 s of model
    time until the velocities vanish -- then the gamma1 estimate (Eq. gamma1) of the
    settled wall layer.  Both device-timed on the context stream; the oracle's settle of the
    same spawn timed beside it on a bounded sample."""
    import torch
    rank, world, local = dist_env()
    if rank != 0:
        return
    torch.cuda.set_device(local)
    from paper_2604_12505_b200 import SphContext
    t = si.random_spawn(4.0, seed=0)
    sp = t.params
    n = int(round(6.0 / sp.dt))
    damp = math.exp(-10.0 * sp.dt)
    ctx = SphContext(sp, t.pv32(), t.ghost_b, n_rollouts=1, rebin_every=0, skin=a.skin * sp.h,
                     device=local)
    ctx.settle(damp, 8)                                   # warm-up (first-call allocations)
    ctx.set_state(t.pv32(), rollout=0, body=np.zeros(6))
    torch.cuda.synchronize()
    clocks = Clocks(local)
    clocks.start()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record(ctx.stream)
    n_done, vmax = ctx.settle_until(damp, 2e-4, n, 500)   # until the velocities vanish
    ev[1].record(ctx.stream)
    wall, g, sums = ctx.gamma1_estimate(0)
    ev[2].record(ctx.stream)
    torch.cuda.synchronize()
    ck = clocks.stop()
    settle_s = ev[0].elapsed_time(ev[1]) / 1e3
    g1_ms = ev[1].elapsed_time(ev[2])
    st = ctx.get_status()[0]
    pv = ctx.get_particles(0)
    n_steps, n_reb = ctx.counters()
    lps = ctx.launches_per_substep()
    ctx.close()
    r = np.hypot(pv[:, 0], pv[:, 1])
    cpu = None
    if not a.no_cpu_baseline:
        import oracle as O
        s = O.State.from_tank(t)
        m = 400                                                # a bounded sample, 1 thread
        c0 = time.perf_counter()
        s.step(n=m, damping=damp, pin_body=True)
        dt = time.perf_counter() - c0
        cpu = {"value": dt * n_done / m, "unit": "s", "cores": 1, "kind": "oracle",
               "sample": f"first {m} settle substeps of the same spawn, float64 C oracle, "
                         f"1 thread, {dt:.1f} s, extrapolated to the GPU's {n_done} substeps"}
    line = {
        "metric": "random-spawn damped settle of the C2 tank until max |v| < 2e-4 m/s (P:323-324)",
        "value": settle_s, "unit": "s", "n_gpus": 1, "steps": 1, "warmup": 1,
        "ms_per_step": settle_s * 1e3, "higher_is_better": False, "scaling": "none",
        "vs_baseline": None, "dtype": "f32 (body f64)",
        "data": "synthetic (uniform random spawn, Philox seed 0, C2 fill region)",
        "config": {"workload": f"SETTLE: C2 tank ({t.n_fluid} fluid + {t.n_ghost} ghosts), "
                               f"damped substeps (at most {n}) until max |v| < 2e-4 m/s + gamma1 estimate",
                   "substeps": n_done, "model_seconds_to_converge": n_done * sp.dt,
                   "us_per_substep": settle_s * 1e6 / max(n_done, 1),
                   "particle_updates_per_s": t.n_fluid * n_done / settle_s,
                   "substeps_per_rebuild": float(n_steps[0] / max(int(n_reb[0]), 1)),
                   "status": int(st[0]), "max_speed_end": float(np.abs(pv[:, 2:]).max()),
                   "max_r_over_R": float(r.max() / sp.R),
                   "gamma1_estimate_wall": wall, "gamma1_estimate_ms": g1_ms,
                   "gamma1_wall_particles": int(np.isfinite(g).sum()),
                   "path": "cooperative tick" if lps == 0 else f"{lps} kernels per substep"},
        "gpu_launches": (n_done // 500) * 2 + 1 + 2 if lps == 0 else n_done * lps + n_done // 500 + 3,
        "clocks": ck,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def run_lpv(a):
    """--workload LPV: the paper's surrogate identification on data
    the simulator generates.  Dataset: the P0 tank (GPU damped settle), the open-loop excitation
    train of P:430-432 (2200 samples, multisine [0, 2) Hz + pulses) -> velocities (rd_x, rd_y,
    thd).  Identification (timed, wall clock with the device synchronised): LTI
    initialisation (reading LPV2), 8 LPV restarts x (2000 Adam + up to 6000 L-BFGS iterations),
    best training BFR.  Validation: the closed-loop manoeuvre profiles 1 and 2 on the SPH
    simulator, their applied inputs replayed through the surrogate (open loop, reading LPV5)."""
    import torch
    rank, world, local = dist_env()
    if rank != 0:
        return
    torch.cuda.set_device(local)
    from paper_2604_12505_b200 import SphContext
    from paper_2604_12505_b200 import lpv as LP
    t = si.make_tank(1.0, n_first=666, clamp_negative_pressure=1.0 if a.eos_clamp else 0.0)
    sp = t.params
    Ts = sp.dt * sp.n_sub
    ctx = SphContext(sp, t.pv32(), t.ghost_b, n_rollouts=1, rebin_every=0, skin=0.5 * sp.h,
                     device=local)
    ctx.settle(math.exp(-10.0 * sp.dt), int(2.0 / sp.dt))
    pv0 = ctx.get_particles(0)
    K = 2200
    S = int(a.lpv_seqs)
    # the identification data IS the ensemble dataset: S rollouts of the
    # excitation train (seed 1000 + global id) run as one batch through the product ensemble path
    # (shard -> sph_rollout_batch -> gather of (y, u_applied, status)), velocities as outputs
    from paper_2604_12505_b200.ensemble import run_ensemble
    g0 = time.perf_counter()
    yd, uad, std = run_ensemble(sp, pv0, t.ghost_b, S, K, "excitation", device=local, rebin_every=0,
                                skin=0.5 * sp.h)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - g0
    # a rollout whose particle tunnelled through the ghost wall (status 3: 3 of 8 seeds within the
    # 110 s train on this tank, on every execution path -- a property of the model as read, A4)
    # is not identification data: only status-0 rollouts are used, and the count is reported
    ok = [sidx for sidx in range(S) if int(std[sidx].item()) == 0]
    if not ok:
        raise SystemExit("every rollout of the identification ensemble failed")
    yd, uad = yd.cpu().numpy(), uad.cpu().numpy()
    us = [uad[sidx].astype(np.float64) for sidx in ok]
    ys = [yd[sidx, :, 3:6].astype(np.float64) for sidx in ok]
    S = len(ok)
    val = {}
    for pid in (1, 2):
        Kv = int(round(30.0 / Ts))
        uv, th = si.profile(pid, Kv)
        ctx.set_state(pv0, rollout=0, body=np.zeros(6))
        yv, ua = ctx.rollout(uv.astype(np.float32)[None], theta_ref=th.astype(np.float32)[None],
                             Kp=sp.Kp, Kd=sp.Kd)
        val[pid] = (np.asarray(ua)[0].astype(np.float64), np.asarray(yv)[0].astype(np.float64))
    ctx.close()
    un, yn, (um, usd, ym, ysd) = LP.normalise(us, ys)
    torch.cuda.synchronize()
    clocks = Clocks(local)
    clocks.start()
    c0 = time.perf_counter()
    res = LP.identify(un, yn, restarts=8, adam_iters=2000, lbfgs_iters=6000, lti_iters=2000,
                      seed=0, lr=1e-3, device=local)
    torch.cuda.synchronize()
    train_s = time.perf_counter() - c0
    ck = clocks.stop()
    # validation: replay the closed-loop runs' applied inputs through the surrogate
    vbfr, sim_ms = {}, {}
    for pid, (ua, yv) in val.items():
        ua_n = ((ua - um) / usd).astype(np.float32)
        prob = LP.LpvProblem(1, [ua_n], None, device=local)
        P = np.concatenate([res["theta"], np.zeros(4)])[None]
        prob.set_params(P)
        prob.simulate()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        yh = prob.simulate()
        e1.record()
        torch.cuda.synchronize()
        sim_ms[pid] = e0.elapsed_time(e1)
        vel = yh[0, 0].cpu().numpy().astype(np.float64) * ysd + ym
        pos = LP.augment_positions(vel, Ts)
        b_pos = LP.bfr(yv[:, 0:3], pos)
        b_vel = LP.bfr(yv[:, 3:6], vel)
        vbfr[pid] = dict(zip(["r_x", "r_y", "theta", "rd_x", "rd_y", "thd"],
                             [round(float(v), 2) for v in np.concatenate([b_pos, b_vel])]))
    cpu = None
    if not a.no_cpu_baseline:
        from oracle import lpv as OL
        th0 = np.concatenate([res["theta"]])
        x0 = np.zeros((S, 4))
        c1 = time.perf_counter()
        OL.objective(th0, x0, [u.astype(np.float64) for u in un], [y.astype(np.float64) for y in yn])
        one = time.perf_counter() - c1
        n_obj = res["n_evals"] * (2 * (LP.NT + 4 * S) + 1)
        cpu = {"value": one * n_obj, "unit": "s", "cores": 1, "kind": "oracle",
               "sample": f"1 objective evaluation ({S} x {K} samples, float64 numpy oracle, 1 thread, "
                         f"{one * 1e3:.0f} ms) x {n_obj} (the {res['n_evals']} gradient evaluations "
                         f"of the run by central differences over {LP.NT + 4 * S} parameters)"}
    line = {
        "metric": "LPV surrogate identification time: LTI init + 8 restarts x (2000 Adam + <= 6000 L-BFGS) (P:441-446)",
        "value": train_s, "unit": "s", "n_gpus": 1, "steps": 1, "warmup": 0,
        "ms_per_step": train_s * 1e3, "higher_is_better": False, "scaling": "none",
        "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (SPH simulator: P0 tank, open-loop excitation train, {S} x {K} samples"
                f"{', clamped EOS (ablation E1)' if a.eos_clamp else ''})",
        "config": {"workload": f"LPV: n_x 4, n_u 3, n_y 3, n_p 1, theta 137 + x0; {S} sequence(s) x {K} samples",
                   "dataset_generation_s": gen_s, "n_evals": res["n_evals"],
                   "ensemble_rollouts": int(a.lpv_seqs), "used_rollouts (status 0)": S,
                   "ms_per_eval": train_s * 1e3 / max(res["n_evals"] / 8, 1),
                   "train_bfr_lti": round(res["bfr_lti"], 2), "train_bfr_lpv": round(res["bfr"], 2),
                   "train_bfr_restarts": [round(v, 2) for v in res["bfr_all"]],
                   "validation_bfr_replay": vbfr, "surrogate_sim_ms": sim_ms,
                   "paper": {"train_s": 48.0, "bfr_lti": 82.16, "bfr_lpv": 98.66,
                             "surrogate_sim_s": {"1": 0.0242, "2": 0.0056},
                             "hardware": "RTX 2000 Ada laptop GPU, JAX (P:391, P:446)"}},
        "gpu_launches": None,
        "clocks": ck,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def run_dd(a):
    """--workload C4DD: the single 1M-particle C4 tank decomposed over the
    torchrun ranks (one GPU each) -- slabs of the cell-sorted slots, three NCCL all-gathers per
    substep (paper_2604_12505_b200.parallel).  One bench step = 50 substeps; value = particle-
    updates/s of the one tank (strong scaling: the tank is the same at every N)."""
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    from paper_2604_12505_b200 import SphContext
    from paper_2604_12505_b200.parallel import DistributedTank, LocalGroup, slab_ranges
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("gloo" if os.environ.get("BENCH_SINGLE_DEVICE_CHECK") == "1" else "nccl",
                                device_id=torch.device("cuda", local))
    t = si.make_tank(42.0)
    sp = t.params
    ctx = SphContext(sp, t.pv32(), t.ghost_b, n_rollouts=1, rebin_every=0, skin=a.skin * sp.h,
                     device=local)
    tank = DistributedTank(ctx) if world > 1 else LocalGroup([ctx])
    SUB = 50
    u = np.array([5.0, 2.0, 1.0], np.float32)

    def step():
        tank.substep(u)                 # input held (ZOH) for the remaining substeps
        for _ in range(SUB - 1):
            tank.substep(None)
    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = Clocks(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ctx.stream)
    for _ in range(a.steps):
        step()
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    ck = clocks.stop()
    ms = e0.elapsed_time(e1)
    if world > 1:
        tm = torch.tensor([ms], dtype=torch.float64, device=ctx.device)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        ms = float(tm.item())
    n_sub = a.steps * SUB
    st = ctx.get_status()[0]
    n_steps, n_reb = ctx.counters()
    chunk, rng = slab_ranges(t.n_fluid, world)
    ctx.close()
    if rank != 0:
        return
    value = t.n_fluid * n_sub / (ms / 1e3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32 (body f64)",
        "data": "synthetic (C4 lattice tank, constant input)",
        "config": {"workload": f"C4DD: one C4 tank ({t.n_fluid} fluid + {t.n_ghost} ghosts) decomposed "
                               f"over {world} GPU(s), {SUB} substeps per step",
                   "slabs": rng, "exchange_bytes_per_substep": 40 * t.n_fluid,
                   "us_per_substep": ms * 1e3 / n_sub, "status": int(st[0]),
                   "substeps_per_rebuild": float(n_steps[0] / max(int(n_reb[0]), 1)),
                   "path": "per-substep phases (sph_dd_phase), NCCL in-place all-gathers"},
        "gpu_launches": None, "clocks": ck, "cpu_baseline": None,
    }
    print(json.dumps(line), flush=True)


def resolve_defaults(a):
    """Per-workload defaults of the skin policy and the settle (the measured configuration is
    entirely in these arguments; tests/test_bench_defaults.py pins the defaults)."""
    skin_default = a.skin is None
    if a.skin is None:
        a.skin = {"P0": 0.5, "C2CL": 0.5, "SETTLE": 0.5, "C3": 0.10, "C5": 0.10}.get(a.workload, 0.15)
    # Verlet skin policy (B4-B6): C3/C5 per-rollout adaptive skin 0.10h -> 0.7h (B5;
    # calm start and sloshing steady state of the 110 s train, profiles/horizon*_r02*, r02.36 /
    # r02.43); C4 per-particle half-skins 0.15h / 0.8h (B6: the bulk keeps short lists, the wall
    # layer wide).  An explicit --skin without --skin-max is a fixed skin (B4).
    if a.skin_max is None:
        a.skin_max = {"C3": 0.7, "C5": 0.7, "C4": 0.8}.get(a.workload, 0.0) if skin_default or a.workload == "C4" else 0.0
    if a.skin_mode is None:
        a.skin_mode = 1 if a.workload == "C4" else 0
    if a.settle_seconds is None:
        # C4: lattice start + 1,000 untimed damped warm-up substeps; dt = 1 ms / 42
        a.settle_seconds = 1000 * 1e-3 / 42.0 if a.workload == "C4" else 4.0
    return a


def main():
    a = resolve_defaults(parse())
    if a.workload == "LIN":
        run_linearize(a)
        return
    if a.workload in ("P0", "C2CL"):
        run_p0(a, closed_loop_c2=a.workload == "C2CL")
        return
    if a.workload == "SETTLE":
        run_settle(a)
        return
    if a.workload == "LPV":
        run_lpv(a)
        return
    if a.workload == "C4DD":
        run_dd(a)
        return
    if a.long_horizon:
        run_horizon(a)
        return
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
    try:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()
    except Exception:
        pass


if __name__ == "__main__":
    main()
