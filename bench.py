#!/usr/bin/env python
"""Benchmark: sketched-LSLU iterations/s at 2048^2 tomography (BASELINE.json
config 4) and the achieved HBM bandwidth of the dominant kernel.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one complete sLSLU solve of the config (K=300 iterations on the
720 x 2897-ray, 2048^2-pixel exact-chord tomography operator, fp32 CSR with
~3.8e9 nonzeros, sparse-sign S2 with ell=1200, zeta=8); the metric is
iterations/s = 300 * steps / time.  ``value`` times the device loop with all
inputs resident (CUDA events on the library's stream, max over ranks);
``e2e`` times the public ``slslu(...)`` call with host b / x_true, including
host<->device copies and the solver setup.  Inputs (A + A^T = 61 GB) are far
larger than L2, so no flush is needed between steps.

Multi-GPU (torchrun, one rank per GPU): the operator is built row-sharded
(rank r holds its rays of A and its image rows of A^T) and all ranks run ONE
solve together over NCCL (all-gathers of the two Krylov vectors per
iteration, tiny owner-pick exchanges, sketch all-reduce): strong scaling.

``--impl reference`` times the CPU port of the reference loop
(oracle/coracle.c, all host threads) on a bounded sample of the same
workload (rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sketched-LSLU iterations/sec at 2048^2 tomography; achieved HBM GB/s"
UNIT = "iterations/s"


# BASELINE.json's configs (paper_2502_02721_b200.problems.CONFIGS; restated here so the
# reference arm names its workload without importing the device package)
WORKLOADS = {
    1: "1D deblurring, dense fp64 1024^2 Toeplitz (sigma=0.02 n), sCMRH K=100, Gaussian s=400",
    2: "2D deblurring 256^2, 15x15 PSF (sigma=2), fp32, sCMRH K=200, Gaussian s=800",
    3: "tomography 512^2, 180 angles x 725 bins, CSR fp32, sLSLU lam=1e-3 K=200, sparse-sign s=800 zeta=8",
    4: "tomography 2048^2, 720 angles x 2897 bins, CSR fp32, sLSLU K=300, sparse-sign s=1200 zeta=8",
    5: "deblurring 4096^2, 31x31 PSF (sigma=4), bf16 basis / fp32 work, sCMRH K=150, Gaussian s=600",
}


def workload_config(args, grid, angles, bins, nnz, K, ell, ws):
    """The `config` object of both arms' JSON lines (identical for the same
    workload and N; how each arm executes it goes into its own keys)."""
    return {
        "workload": f"cfg{args.config}: " + WORKLOADS[args.config],
        "grid": grid, "angles": angles, "bins": bins, "nnz": nnz, "maxiter": K,
        "sketch": "sparse-sign ell=%d zeta=8" % ell,
        "step": "one full sLSLU solve (maxiter iterations)",
        "l2": "inputs (A + A^T) far larger than L2; no flush",
        "parallelism": f"rowshard{ws}" if ws > 1 else "single",
    }


def _traffic(args, which):
    """DRAM bytes per launch of one SpMV direction ("A" / "AT") from the committed ncu
    --set full capture (config 4 only; profiles/r2/traffic.json)."""
    if args.config != 4 or args.scale:
        return None
    try:
        with open(os.path.join(ROOT, "profiles", "r2", "traffic.json")) as fh:
            return float(json.load(fh)["per_launch"][which])
    except Exception:
        return None


def _spmv_roofline(args, name, st, nnz, peak, loop_ms_total, single):
    """Roofline entry of one SpMV direction: encoded (algorithmic) bytes per launch over the mean
    launch time from the CUDA events inside the timed region."""
    if not st or not st.get("launches") or st["ms"] <= 0:
        return None
    bpl = st["bytes"] / st["launches"]
    ms = st["ms"] / st["launches"]
    ach = bpl / (ms / 1e3) / 1e9
    bpn = bpl / nnz if nnz else None
    if name == "spmv_A":
        kern = ("sell_spmv_c2_kernel (A: 2-bit step codes, 4.25 B/nonzero)" if bpn and bpn < 5.0
                else "sell_spmv_d16_kernel (A: 16-bit deltas, 6 B/nonzero)")
    else:
        kern = ("sell_spmv_t8_kernel (A^T: 8-bit step codes, 5 B/nonzero)" if bpn and bpn < 5.5
                else "sell_spmv_d16_kernel (A^T: 16-bit deltas, 6 B/nonzero)")
    return {
        "bound": "hbm", "kernel": kern,
        "bytes_per_launch": round(bpl), "bytes_per_nonzero": round(bpn, 3) if bpn else None,
        "ms_per_launch": round(ms, 4),
        "achieved": round(ach, 1), "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4),
        "achieved_csr8_equiv": round(8.0 * nnz / (ms / 1e3) / 1e9, 1) if nnz and single else None,
        "traffic": _traffic(args, "A" if name == "spmv_A" else "AT"),
        "share_of_step": round(st["ms"] / loop_ms_total, 4) if loop_ms_total else None,
    }


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    smax = float(parts[2])
                except ValueError:
                    continue
                for name, flag in zip(names, parts[5:9]):
                    if flag.lower() in ("active", "0x1", "1"):
                        reasons.add(name)
        except Exception:
            pass
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def max_over_ranks(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(x)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_ranks(x, ws):
    """Per-rank values (rank order) on every rank."""
    if ws == 1:
        return [x]
    import torch.distributed as dist

    out = [None] * ws
    dist.all_gather_object(out, x)
    return out


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()


def run_ours(args, ws, rank, local):
    import numpy as np

    import paper_2502_02721_b200 as hs
    from paper_2502_02721_b200 import _lib
    from paper_2502_02721_b200.problems import make_workload

    os.environ["HS_DEVICE"] = str(local)
    _lib.load()
    ctx = _lib.context(local)
    if ws > 1:
        # row-sharded solve over NCCL: operators are built per rank, one problem for all ranks
        from paper_2502_02721_b200 import dist as hsd

        hsd.init_comm(ctx)
    t_setup = time.perf_counter()
    w = make_workload(args.config, seed=args.seed, scale=args.scale, maxiter=args.maxiter)
    setup_s = time.perf_counter() - t_setup
    K = w.cfg.maxiter
    solve = hs.slslu if w.solver == "slslu" else hs.scmrh
    op = w.operator
    inf = op.info() if hasattr(op, "info") else {}

    # the step's host inputs live in pinned memory (the e2e contract: host->device
    # copies of each step's inputs from pinned host buffers, inside the timed region)
    def pinned(a):
        import torch

        t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
        t.numpy()[...] = a
        return t.numpy()

    b_host, xt_host = pinned(w.b), pinned(w.x_true)

    def one_step(x_true):
        return solve(op, b_host, w.cfg, x_true=x_true, sketch=w.sketch)

    for _ in range(args.warmup):
        one_step(xt_host)
    ctx.synchronize()
    barrier(ws)
    ctx.reset_stats()
    ctx.set_profiling(True)
    launches0 = _lib.load().hs_launch_count()
    loop_ms, wall_s, iters = [], [], 0
    with ClockSampler(local) as clk:
        barrier(ws)
        for _ in range(args.steps):
            t0 = time.perf_counter()
            res = one_step(xt_host)  # host b / x_true in (pinned), host x / trace out
            wall_s.append(time.perf_counter() - t0)
            loop_ms.append(res.loop_ms)
            iters += len(res.trace.records)
        ctx.synchronize()
        barrier(ws)
    launches = _lib.load().hs_launch_count() - launches0
    ctx.set_profiling(False)
    stats = ctx.kernel_stats()
    clocks = clk.summary()

    per_rank = gather_ranks(round(sum(loop_ms), 3), ws)
    tot_ms = max_over_ranks(sum(loop_ms), ws)
    tot_wall = max_over_ranks(sum(wall_s), ws)
    iters_all = iters  # one sharded solve across all ranks (strong scaling)
    value = iters_all / (tot_ms / 1e3)
    e2e = iters_all / tot_wall
    peak, peak_kind = _peaks()
    # the two order-faithful CSR SpMVs (A and A^T) are separate kernels with separate
    # encodings: the roofline is the one with the larger share of the step, the other rides along
    rl = {k: _spmv_roofline(args, k, stats.get(k), inf.get("nnz"), peak, sum(loop_ms), ws == 1)
          for k in ("spmv_A", "spmv_AT")}
    dom = max((k for k in rl if rl[k]), key=lambda k: rl[k]["share_of_step"] or 0.0, default=None)
    step_ms = tot_ms / args.steps
    kernels = {k: {"launches": v["launches"], "ms_total": round(v["ms"], 3),
                   "GBps": round(v["bytes"] / (v["ms"] / 1e3) / 1e9, 1) if v["ms"] > 0 and v["bytes"] > 0 else None}
               for k, v in stats.items()}
    out = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": UNIT,
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(step_ms, 3),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (seeded random-ellipse phantom, 1% noise; device-built exact-chord operator)",
        "config": workload_config(args, w.meta.get("grid"), w.meta.get("angles"), w.meta.get("bins"),
                                  w.meta.get("nnz"), K, w.cfg.sketch_rows, ws),
        "parallelism_detail": ("row-sharded operator and bases, NCCL all-gathers of l_k / d_{k+1} and of the "
                               "sketch partials, owner-picked pivot rows, merged argmax candidates"
                               if ws > 1 else "one GPU"),
        "per_rank_loop_ms": per_rank,
        "e2e": {"value": round(e2e, 3), "unit": UNIT,
                "h2d_bytes_per_step": int(w.b.nbytes + w.x_true.nbytes),
                "d2h_bytes_per_step": int(w.x_true.nbytes + 8 * 12 * K)},
        "roofline": (dict(rl[dom], peak_source=peak_kind,
                          other_spmv=rl["spmv_A" if dom == "spmv_AT" else "spmv_AT"])
                     if dom else None),
        "storage": ({"A": op.storage(False), "AT": op.storage(True)} if hasattr(op, "storage") else None),
        "gpu_launches": int(launches),
        "clocks": clocks,
        "kernels": kernels,
        "kernels_note": ("CUDA-event spans per kernel name; aux-stream kernels (sketch_*, qr_step) are timed on "
                         "the aux stream, so their span includes waiting for SM residency behind the main-stream "
                         "SpMV they overlap"),
        "setup_s": round(setup_s, 2),
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args, w)
    return out


def cpu_baseline(args, w, seconds=None):
    """Oracle port (oracle/coracle.c, OpenMP over host cores) on a bounded sample."""
    try:
        from oracle import cpu_baseline as cb

        return cb.run(w, budget_s=seconds or args.cpu_seconds)
    except Exception as e:  # reported, never fatal for the GPU number
        return {"value": None, "unit": UNIT, "cores": None, "kind": "port", "sample": f"unavailable: {e}"}


def _python_reference_note():
    """The measured seconds per iteration of the unmodified Python reference at
    a reduced size (tools/ref_python_scaled.py, run where /root/reference
    exists; the committed measurement travels, the reference does not)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2", "reference_python_scaled.json")) as fh:
            r = json.load(fh)
        return {k: r[k] for k in ("grid", "angles", "bins", "nnz", "maxiter", "python_reference_s_per_iter",
                                  "c_port_s_per_iter", "python_over_c_port",
                                  "python_reference_full_size_estimate_s_per_iter", "host_threads")}
    except Exception:
        return None


def run_reference(args, ws, rank):
    if rank != 0:
        return None
    from types import SimpleNamespace

    from oracle import cpu_baseline as cb

    if args.config not in (3, 4):
        return {"impl": "reference", "unavailable": "CPU reference arm implemented for the tomography configs only"}
    grid, angles, bins, K, ell = (512, 180, 725, 200, 800) if args.config == 3 else (2048, 720, 2897, 300, 1200)
    if args.scale:
        f = args.scale / grid
        grid, angles, bins = args.scale, max(2, round(angles * f)), max(2, round(bins * f))
    K = args.maxiter or K
    ell = max(ell, K + 1)
    # host-only workload description (the operator, phantom and b are built on the host by oracle/)
    w = SimpleNamespace(meta={"grid": grid, "angles": angles, "bins": bins},
                        cfg=SimpleNamespace(maxiter=K, sketch_rows=ell))
    vals, last = [], None
    t_all = time.perf_counter()
    for i in range(args.warmup + args.steps):
        r = cb.run(w, real_iters=4 if i == 0 else 0)
        if i >= args.warmup:
            vals.append(r["value"])
        if last is None or i == 0:
            first = r
        last = r
    value = statistics.mean(vals) if vals else None
    sample = (first["sample"] + f"; {args.steps} timed steps (+{args.warmup} warm-up), each the same {K}-step "
              f"profile: rate mean {value:.4f}, min {min(vals):.4f}, max {max(vals):.4f} it/s; "
              f"{time.perf_counter() - t_all:.0f}s in all")
    return {
        "metric": METRIC, "impl": "reference", "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded random-ellipse phantom, 1% noise; host-built exact-chord operator)",
        "config": workload_config(args, grid, angles, bins, last.get("nnz") if last else None, K, ell, ws),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": last["cores"] if last else None, "kind": "port",
                         "sample": sample},
        "python_reference": _python_reference_note(),
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--scale", type=int, default=None, help="image side override (testing)")
    ap.add_argument("--maxiter", type=int, default=None)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: relaunch this command under torchrun
        import socket

        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        os.execv(sys.executable, cmd)
    ws, rank, local = dist_env()
    if ws != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
    if ws > 1:
        import torch
        import torch.distributed as dist

        # host-side plumbing only (NCCL id broadcast, barriers, max over ranks);
        # the data path uses the library's own NCCL communicator on each GPU
        dist.init_process_group(backend="gloo")
    if args.impl == "reference":
        out = run_reference(args, ws, rank)
    else:
        out = run_ours(args, ws, rank, local)
    if rank == 0 and out is not None:
        print(json.dumps(out), flush=True)
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
