#!/usr/bin/env python
"""Benchmark of the B200 DG advection hot path (hyper.deal, arXiv 2002.08110).

One "step" = one LSRK(5,4) time step (5 fused stages: M^-1 A + 2N update) over the whole synthetic
workload. Metric (BASELINE.json): GDoF/s per RK stage = DoFs * 5 * steps / time, whole job over all
ranks, plus the HBM-roofline fraction of the dominant kernel (the fused stage kernel).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 6d] [--impl reference]

N > 1 is launched by torchrun (one rank per GPU, x-slab partition, NCCL halo). Rank 0 prints ONE
JSON line. ``--impl reference`` times the CPU oracle (test infrastructure) on the same workload,
as the reference arm.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GDoF/s per RK stage (A + M^-1) and % of HBM roofline at 1/2/4/8 B200"
UNIT = "GDoF/s"
FALLBACK_HBM_GBS = 6650.0


def load_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def load_traffic(workload):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled DURING the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.active", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def workload_config(name, spec, ndofs, nranks):
    return {"workload": name, "d_x": spec["d_x"], "d_v": spec["d_v"], "k": spec["k"], "cells": spec["cells"],
            "dofs": ndofs, "field": "vlasov-like" if any(any(r) for r in spec["a_lin"]) else "constant",
            "flux": "upwind", "basis": "Lagrange on Gauss points (collocation)",
            "l2_policy": "inputs larger than L2 (%.1f GB per vector)" % (ndofs * 8 / 1e9),
            "parallelism": f"x-slab x{nranks}" if nranks > 1 else "single GPU"}


# ------------------------------------------------------------------------------------------------
def cpu_oracle_sample(name, target_s=15.0, stage_only=True):
    """Time the CPU oracle (O2, C++/OpenMP, as it stands) on a bounded sample of the workload: the
    merged operator of one RK stage plus its 2N update on consecutive cells, chunk by chunk, until
    ~target_s seconds of oracle time. Returns (GDoF/s, cores, sample description)."""
    from oracle import capi
    from paper_2002_08110_b200 import configs, inputs
    cfg = configs.CONFIGS[name]
    spec = cfg["spec"]
    seed = configs.seed_of(name)
    d = spec["d_x"] + spec["d_v"]
    nd = (spec["k"] + 1) ** d
    ncell = int(np.prod(spec["cells"]))
    # one chunk of consecutive cells (inputs generated once, untimed), evaluated repeatedly
    chunk = max(1, min(ncell, (1 << 23) // nd))
    A = capi.rk_coefficients()[0]
    B = capi.rk_coefficients()[1]
    dt = configs.time_step(spec, cfg["cfl"])
    ids = np.arange(0, chunk, dtype=np.int64)
    nb = inputs.neighbour_ids(spec, ids)
    own = inputs.cell_values(spec, cfg["recipe"], seed, ids)
    nbv = inputs.cell_values(spec, cfg["recipe"], seed, nb.reshape(-1)).reshape(len(ids), 2 * d, nd)
    cells = np.concatenate([own[:, None, :], nbv], axis=1)
    du0 = np.zeros_like(own)
    done, t_or, reps = 0, 0.0, 0
    while t_or < target_s:
        t0 = time.perf_counter()
        r = capi.apply_advection_cells(spec, ids, cells, merged=True)
        du = A[1] * du0 + dt * r          # stage 2 form: reads dU, writes dU and U'
        _ = own + B[1] * du
        t_or += time.perf_counter() - t0
        done += len(ids) * nd
        reps += 1
    cores = capi.num_threads()
    desc = (f"cells 0..{chunk - 1} of the {name} workload ({chunk * nd} DoFs) x {reps} repetitions: one RK "
            f"stage each (merged operator, oracle O2, + 2N update), {t_or:.1f} s of oracle time; input "
            f"generation untimed")
    return done / t_or / 1e9, cores, desc


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_2002_08110_b200 import configs
    cfg = configs.CONFIGS[args.config]
    spec = cfg["spec"]
    ndofs = configs.dof_count(spec)
    per_step_budget = max(2.0, 60.0 / max(1, args.steps + args.warmup))
    for _ in range(args.warmup):
        cpu_oracle_sample(args.config, target_s=min(per_step_budget, 3.0))
    vals, cores, desc = [], 0, ""
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v, cores, desc = cpu_oracle_sample(args.config, target_s=per_step_budget)
        vals.append(v)
    wall = time.perf_counter() - t0
    value = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * ndofs * 5 / (value * 1e9),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args.config, spec, ndofs, 1),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": f"CPU oracle; ms_per_step extrapolated to the full workload; wall {wall:.1f} s"}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------------
def run_gpu(args):
    import torch
    import torch.distributed as dist
    from paper_2002_08110_b200 import Mesh, configs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = configs.CONFIGS[args.config]
    spec = cfg["spec"]
    nccl_id = None
    if world > 1:
        nccl_id = _bcast_nccl_id(rank)
    mesh = Mesh(spec, rank=rank, nranks=world, nccl_id=nccl_id)
    N = mesh.owned_dofs
    ndofs = configs.dof_count(spec)
    seed = configs.seed_of(args.config)
    dt = configs.time_step(spec, cfg["cfl"])
    stream = torch.cuda.current_stream()
    bufs = [torch.empty(N, dtype=torch.float64, device="cuda") for _ in range(3)]
    mesh.fill_initial(bufs[0], cfg["recipe"], seed)
    sol = 0

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- warm-up (untimed)
    for _ in range(args.warmup):
        sol = mesh.rk_step(bufs, sol, 0.0, dt, 1, stream)
    barrier()
    # ---- timed region: exactly K steps, CUDA events on the launching stream
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    l0 = mesh.launch_count
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    for _ in range(args.steps):
        sol = mesh.rk_step(bufs, sol, 0.0, dt, 1, stream)
    e1.record(stream)
    barrier()
    clocks = sampler.stop()
    launches = mesh.launch_count - l0
    ms = max_over_ranks(e0.elapsed_time(e1))
    ms_per_step = ms / args.steps
    value = ndofs * 5 * args.steps / (ms * 1e-3) / 1e9
    ok = bool(torch.isfinite(bufs[sol][:: max(1, N // 4096)]).all())

    # roofline of the dominant kernel: the fused stage kernel is every launch of the step.
    # Algorithmic bytes per launch: stage 1 reads U, writes dU and U' (24 B/DoF);
    # stages 2..5 also read dU (32 B/DoF) -> (24 + 4*32)/5 = 30.4 B/DoF per launch on average.
    peak, peak_kind = load_peak()
    bytes_per_launch = N * 8 * (3 + 4 * 4) / 5.0
    launch_ms = ms_per_step / 5.0
    achieved = bytes_per_launch / (launch_ms * 1e-3) / 1e9
    traffic = load_traffic(args.config)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak * (1 if world == 1 else 1), "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": "cell_kernel<6,4,RK> (fused M^-1 A + LSRK stage)" if args.config == "6d" else
                "cell_kernel (fused M^-1 A + LSRK stage)",
                "algorithmic_bytes_per_dof": 30.4, "peak_kind": f"of {peak_kind} (MEASURED_PEAKS.json hbm_gbs)"}

    # ---- the two operators of the metric name, timed alone (same workload, 16 B/DoF each)
    extra = {}
    if not args.no_ops:
        v = bufs[(sol + 1) % 3]
        u = bufs[sol]
        reps = max(3, args.steps)
        for _ in range(2):
            mesh.apply_advection(u, v, 0.0, stream)
        barrier()
        e0.record(stream)
        for _ in range(reps):
            mesh.apply_advection(u, v, 0.0, stream)
        e1.record(stream)
        barrier()
        a_ms = max_over_ranks(e0.elapsed_time(e1)) / reps
        w = bufs[(sol + 2) % 3]
        for _ in range(2):
            mesh.apply_inv_mass(w, stream)
        barrier()
        e0.record(stream)
        for _ in range(reps):
            mesh.apply_inv_mass(w, stream)
        e1.record(stream)
        barrier()
        m_ms = max_over_ranks(e0.elapsed_time(e1)) / reps
        a_gdofs = ndofs / (a_ms * 1e-3) / 1e9
        m_gdofs = ndofs / (m_ms * 1e-3) / 1e9
        extra = {
            "apply_advection": {"gdofs": a_gdofs, "ms": a_ms, "hbm_frac_of_8tbs": a_gdofs * 16 / 8000 / world,
                                "hbm_frac_of_measured": a_gdofs * 16 / peak / world},
            "apply_inv_mass": {"gdofs": m_gdofs, "ms": m_ms, "hbm_frac_of_8tbs": m_gdofs * 16 / 8000 / world,
                               "hbm_frac_of_measured": m_gdofs * 16 / peak / world},
            "rk_stage": {"gdofs": value, "hbm_frac_of_8tbs": value * 32 / 8000 / world,
                         "hbm_frac_of_measured_32B": value * 32 / peak / world},
        }
        # keep the solution buffer intact for e2e: u, v, w are distinct
        mesh.fill_initial(bufs[0], cfg["recipe"], seed)
        sol = 0

    # ---- end to end through the C ABI with HOST buffers (H2D + steps + D2H inside the timed region)
    e2e = None
    if not args.no_e2e:
        hbuf = torch.empty(N, dtype=torch.float64, pin_memory=True)
        hbuf.copy_(bufs[0])  # initial state on the host (untimed)
        torch.cuda.synchronize()
        mesh.rk_step_host(hbuf, hbuf, bufs, 0.0, dt, 1, stream)  # warm-up
        e2e_steps = args.e2e_steps
        barrier()
        t0 = time.perf_counter()
        e0.record(stream)
        for _ in range(e2e_steps):
            mesh.rk_step_host(hbuf, hbuf, bufs, 0.0, dt, 1, stream)
        e1.record(stream)
        barrier()
        e_ms = max_over_ranks(e0.elapsed_time(e1)) / e2e_steps
        e2e = {"value": ndofs * 5 / (e_ms * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": N * 8 * world,
               "d2h_bytes_per_step": N * 8 * world, "ms_per_step": e_ms, "steps": e2e_steps,
               "api": "hd_rk_step_host (pinned host in/out, one step per call)"}
        del hbuf

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            v_c, cores, desc = cpu_oracle_sample(args.config, target_s=args.cpu_seconds)
            cpu = {"value": v_c, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc}
        except Exception as ex:  # the oracle is test infrastructure; report, do not fail the bench
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "oracle", "sample": f"failed: {ex}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": workload_config(args.config, spec, ndofs, world),
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clocks, "finite": ok, **extra}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def _bcast_nccl_id(rank):
    import torch
    import torch.distributed as dist
    from paper_2002_08110_b200 import _binding
    if rank == 0:
        uid = _binding.nccl_unique_id()
        t = torch.tensor(list(uid), dtype=torch.uint8, device="cuda")
    else:
        t = torch.empty(128, dtype=torch.uint8, device="cuda")
    dist.broadcast(t, 0)
    return bytes(t.cpu().tolist())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="6d", choices=["2d", "3d", "4d", "5d", "6d"])
    ap.add_argument("--impl", default="gpu", choices=["gpu", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-ops", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "gpu":
        print("warning: contract requires >= 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
