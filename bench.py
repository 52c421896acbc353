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


def host_cpu_meta():
    """lscpu model, sockets, nproc and OMP_NUM_THREADS of the host the CPU oracle runs on (BASELINE.md plan)."""
    meta = {"nproc": os.cpu_count(), "omp_num_threads": os.environ.get("OMP_NUM_THREADS")}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            k, _, v = ln.partition(":")
            if k.strip() == "Model name":
                meta["cpu_model"] = v.strip()
            elif k.strip() == "Socket(s)":
                meta["sockets"] = v.strip()
    except Exception:
        pass
    return meta


def workload_config(name, spec, ndofs, nranks):
    return {"workload": name, "d_x": spec["d_x"], "d_v": spec["d_v"], "k": spec["k"], "cells": spec["cells"],
            "dofs": ndofs, "field": "vlasov-like" if any(any(r) for r in spec["a_lin"]) else "constant",
            "flux": "upwind", "basis": "Lagrange on Gauss points (collocation)",
            "l2_policy": ("inputs larger than L2 (%.2f GB per vector)" % (ndofs * 8 / 1e9) if ndofs * 8 > 2 * 126e6 else
                          "L2-resident inputs (%.3f GB per vector; --l2-flush for an HBM claim)" % (ndofs * 8 / 1e9)),
            "parallelism": f"x-partition x{nranks}" if nranks > 1 else "single GPU"}


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
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args.config, spec, ndofs, 1),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc,
                             **host_cpu_meta()},
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
    xparts = None
    if world > 1 and args.partition == "slabs":
        xparts = [1] * (spec["d_x"] - 1) + [world]  # x-slabs of the slowest x dim (north star)
    mesh = Mesh(spec, rank=rank, nranks=world, nccl_id=nccl_id, xparts=xparts)
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

    flush_buf = None
    if args.l2_flush:
        # 2 x L2 of scratch written between timed repetitions (outside their events)
        l2 = torch.cuda.get_device_properties(local).L2_cache_size
        flush_buf = torch.empty(2 * l2 // 8, dtype=torch.float64, device="cuda")

    def timed(fn, reps):
        """Device time (ms) of reps calls of fn on the stream, CUDA events around each call; with --l2-flush
        an L2 flush runs between the calls outside the events. Max over ranks."""
        total = 0.0
        if flush_buf is None:
            e0.record(stream)
            for _ in range(reps):
                fn()
            e1.record(stream)
            barrier()
            total = e0.elapsed_time(e1)
        else:
            for _ in range(reps):
                flush_buf.fill_(1.0)
                e0.record(stream)
                fn()
                e1.record(stream)
                barrier()
                total += e0.elapsed_time(e1)
        return max_over_ranks(total)

    # ---- warm-up (untimed)
    for _ in range(args.warmup):
        sol = mesh.rk_step(bufs, sol, 0.0, dt, 1, stream)
    barrier()
    # ---- timed region: exactly K steps, CUDA events on the launching stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    l0 = mesh.launch_count
    barrier()
    state = {"sol": sol}

    def one_step():
        state["sol"] = mesh.rk_step(bufs, state["sol"], 0.0, dt, 1, stream)

    ms = timed(one_step, args.steps)
    sol = state["sol"]
    clocks = sampler.stop()
    launches = mesh.launch_count - l0
    ms_per_step = ms / args.steps
    value = ndofs * 5 * args.steps / (ms * 1e-3) / 1e9
    ok = bool(torch.isfinite(bufs[sol][:: max(1, N // 4096)]).all())

    # roofline of the dominant kernel: the fused stage kernel is every launch of the step (multi-rank: plus
    # the halo pack). Algorithmic bytes per DoF: stage 1 reads U and
    # writes dU and U' (24 B/DoF); stages 2..5 also read dU (32 B/DoF) -> 30.4 B/DoF per launch on average;
    # the 32 B/DoF of SURVEY 8(d) is reported beside it. Whole-job bytes over the whole-job peak (N x HBM).
    peak, peak_kind = load_peak()
    launch_ms = ms_per_step / 5.0
    achieved = ndofs * 30.4 / (launch_ms * 1e-3) / 1e9
    traffic = load_traffic(args.config)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak * world, "unit": "GB/s",
                "frac": achieved / (peak * world), "traffic": traffic,
                "frac_32B": ndofs * 32.0 / (launch_ms * 1e-3) / 1e9 / (peak * world),
                "kernel": f"cell_kernel<{spec['d_x'] + spec['d_v']},{spec['k'] + 1},RK> (fused M^-1 A + LSRK stage)",
                "algorithmic_bytes_per_dof": 30.4,
                "peak_kind": f"{peak_kind} copy bandwidth (MEASURED_PEAKS.json hbm_gbs) x {world} GPU(s)"}

    # ---- the two operators of the metric name, timed alone (same workload, 16 B/DoF each)
    extra = {}
    if not args.no_ops:
        v = bufs[(sol + 1) % 3]
        u = bufs[sol]
        reps = max(3, args.steps)
        for _ in range(2):
            mesh.apply_advection(u, v, 0.0, stream)
        barrier()
        a_ms = timed(lambda: mesh.apply_advection(u, v, 0.0, stream), reps) / reps
        w = bufs[(sol + 2) % 3]
        for _ in range(2):
            mesh.apply_inv_mass(w, stream)
        barrier()
        m_ms = timed(lambda: mesh.apply_inv_mass(w, stream), reps) / reps
        a_gdofs = ndofs / (a_ms * 1e-3) / 1e9
        m_gdofs = ndofs / (m_ms * 1e-3) / 1e9

        def op_roofline(gdofs, kernel, key):
            ach = gdofs * 16.0
            return {"bound": "hbm", "achieved": ach, "peak": peak * world, "unit": "GB/s",
                    "frac": ach / (peak * world), "frac_of_8tbs": ach / (8000.0 * world),
                    "traffic": load_traffic(args.config + "_" + key), "algorithmic_bytes_per_dof": 16.0,
                    "kernel": kernel}
        extra = {
            "apply_advection": {"gdofs": a_gdofs, "ms": a_ms,
                                "roofline": op_roofline(a_gdofs, "cell_kernel<..,A> (v <- A(u), weak form)", "adv")},
            "apply_inv_mass": {"gdofs": m_gdofs, "ms": m_ms,
                               "roofline": op_roofline(m_gdofs, "mass_kernel (u <- M^-1 u in place)", "mass")},
            "rk_stage": {"gdofs": value, "hbm_frac_of_8tbs_32B": value * 32 / 8000 / world,
                         "hbm_frac_of_measured_32B": value * 32 / peak / world,
                         "hbm_frac_of_measured_30.4B": value * 30.4 / peak / world},
        }
        # the face-centric loop comparison path (hd_apply_advection_fcl) where its
        # face buffers (3 d n^(d-1) doubles per cell) fit beside the product path's buffers
        dd, nn = spec["d_x"] + spec["d_v"], spec["k"] + 1
        fcl_bytes = 3 * dd * (N // nn) * 8
        if world == 1 and not args.no_fcl:
            free = torch.cuda.mem_get_info()[0]
            if fcl_bytes < free - (1 << 30):
                for _ in range(2):
                    mesh.apply_advection_fcl(u, v, 0.0, stream)
                barrier()
                f_ms = timed(lambda: mesh.apply_advection_fcl(u, v, 0.0, stream), reps) / reps
                f_gdofs = ndofs / (f_ms * 1e-3) / 1e9
                design = 32.0 + 6 * dd * 8.0 / nn
                extra["apply_advection_fcl"] = {
                    "gdofs": f_gdofs, "ms": f_ms, "ecl_over_fcl": a_gdofs / f_gdofs,
                    "roofline": dict(op_roofline(f_gdofs, "fcl_cell + fcl_face + fcl_lift (v <- A(u), face-centric loop)",
                                                 "fcl"),
                                     design_bytes_per_dof=design, frac_design=f_gdofs * design / (peak * world))}
            else:
                extra["apply_advection_fcl"] = {"skipped": f"face buffers ({fcl_bytes / 1e9:.1f} GB) do not fit the "
                                                           f"{free / 1e9:.1f} GB left beside the product path's buffers"}
        # the GLL <-> Gauss basis change (hd_basis_change, "quantify the overhead
        # resulting from the basis change") alone (16 B/DoF) and around the operator (T, A, T^T: 3 launches)
        try:
            for _ in range(2):
                mesh.basis_change(u, v, "gll_to_gauss", stream)
            barrier()
            b_ms = timed(lambda: mesh.basis_change(u, v, "gll_to_gauss", stream), reps) / reps
            b_gdofs = ndofs / (b_ms * 1e-3) / 1e9
            for _ in range(2):
                mesh.apply_advection_gll(u, v, w, 0.0, stream)
            barrier()
            g_ms = timed(lambda: mesh.apply_advection_gll(u, v, w, 0.0, stream), reps) / reps
            extra["basis_change"] = {"gdofs": b_gdofs, "ms": b_ms,
                                     "roofline": op_roofline(b_gdofs, "basis_kernel (v <- (T x ... x T) u per cell)", "basis")}
            extra["apply_advection_gll"] = {"gdofs": ndofs / (g_ms * 1e-3) / 1e9, "ms": g_ms,
                                            "overhead_vs_gauss_collocation": g_ms / a_ms,
                                            "launches": "basis_kernel(T) + cell_kernel<A> + basis_kernel(T^T)"}
        except Exception as ex:  # noqa: BLE001 -- (d, n) whose cell does not fit the basis kernel
            extra["basis_change"] = {"skipped": str(ex)}
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
            cpu = {"value": v_c, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc, **host_cpu_meta()}
        except Exception as ex:  # the oracle is test infrastructure; report, do not fail the bench
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "oracle", "sample": f"failed: {ex}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": dict(workload_config(args.config, spec, ndofs, world),
                               l2_policy=("L2 flushed (2 x L2 scratch write) between timed repetitions"
                                          if args.l2_flush else workload_config(args.config, spec, ndofs, world)["l2_policy"]),
                               xparts=mesh.xparts[:spec["d_x"]]),
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
    ap.add_argument("--no-fcl", action="store_true", help="skip the face-centric loop comparison timing")
    ap.add_argument("--l2-flush", action="store_true", help="flush L2 between timed repetitions (3D/4D)")
    ap.add_argument("--partition", default="auto", choices=["auto", "slabs"],
                    help="multi-GPU x partition: smallest halo (auto) or x-slabs of the slowest x dim")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (rank 0 prints the line)
        port = 29500 + (os.getpid() % 2000)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
        return subprocess.call(cmd)
    if args.warmup < 3 and args.impl == "gpu":
        print("warning: contract requires >= 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
