#!/usr/bin/env python
"""Benchmark: voxel-steps/s of forward + adjoint geodesic shooting (grad()).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2]

Workload (BASELINE.json configs[1]): 2D LDDMM, 64 independent pairs of 512^2
fp32, T=20, Gaussian sigma=6 (r=24), seeded synthetic inputs.
A step = one grad() of every pair (forward shoot + explicit adjoint).  Pairs
shard over ranks (torchrun, one process per GPU) with no collective on the hot
path; the max-over-ranks device time is reported.  The timed region starts
with every input resident in HBM; ``e2e`` re-measures through the public API
with pinned host buffers and the H2D/D2H copies inside the timed region.

``--impl reference`` times the reference algorithm's CPU implementation (the
float64 numpy port in oracle/, the reference itself being pure Python that
cannot travel to the GPU box) on all host cores, on the same config.
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

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

# algorithmic bytes per voxel-step per kernel (fp32, store-all-states)
def alg_bytes(d: int) -> dict:
    return {
        "velocity": 4 * (2 + d),          # read I, z; write v
        "sl_step": 4 * (d + 4),           # read v, I, z; write I', z'
        "sl_adjoint": 4 * (2 * d + 6),    # read ibar', zbar', v, I, z; write ib, zb, vbar
        "velocity_adjoint": 4 * (d + 6),  # read vbar, I, z, ib, zb; write ibar, zbar
    }


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", type=int, default=2)
    p.add_argument("--scheme", default="semi-lagrangian",
                   choices=["semi-lagrangian", "eulerian", "hybrid"],
                   help="shooting scheme (2D configs; the hot path is semi-lagrangian)")
    p.add_argument("--groups", type=int, default=None,
                   help="pair groups on concurrent streams (default 2 for 2D batches >= 8)")
    p.add_argument("--shard-of", type=int, default=None,
                   help="builder aid: time rank 0's shard of a W-rank job on this one GPU "
                        "(no process group; predicts the per-rank step of --gpus W)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=None)
    p.add_argument("--e2e-chunks", type=str, default=None,
                   help="pair groups of the host-buffer pipeline: a count or comma-separated "
                        "group sizes (default: the API's choice)")
    p.add_argument("--no-graph", action="store_true", help="launch kernels directly (no CUDA graph)")
    p.add_argument("--mu", type=float, default=None,
                   help="override the config's metamorphosis weight (e.g. --config 5 --mu 0)")
    p.add_argument("--deterministic", action="store_true",
                   help="fixed-point adjoint scatters (bitwise run-to-run reproducible)")
    p.add_argument("--print-launch", action="store_true",
                   help="print the multi-rank launch command --gpus N would exec, then exit")
    return p.parse_args()


def launch_cmd(argv, n: int, port: int) -> list:
    """torch.distributed.run command that starts one rank per GPU."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
            f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={port}",
            os.path.abspath(__file__)] + list(argv)


def maybe_relaunch(args) -> bool:
    """`python bench.py --gpus N` outside torchrun: re-exec as N ranks (one per GPU).
    Returns True when this process only launched (and waited for) the ranks."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    import socket

    with socket.socket() as sk:  # a free local port for the rendezvous
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = launch_cmd(sys.argv[1:], args.gpus, port)
    if args.print_launch:
        print(json.dumps({"launch": cmd}))
        return True
    rc = subprocess.call(cmd)
    if rc != 0:
        sys.exit(rc)
    return True


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def shard(n: int, rank: int, world: int) -> list:
    """Contiguous split of n independent pairs over ranks."""
    lo = (n * rank) // world
    hi = (n * (rank + 1)) // world
    return list(range(lo, hi))


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled (every 100 ms) during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._p = None

    def __enter__(self):
        try:
            self._p = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # let the first sample land inside the region
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is None:
            return
        self._p.terminate()
        try:
            out, _ = self._p.communicate(timeout=5)
        except Exception:
            self._p.kill()
            out, _ = self._p.communicate()
        for line in out.splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2106_08817_b200 import _lib, engine
    from paper_2106_08817_b200.synthetic import CONFIGS, make_config

    rank, world, local = dist_env()
    if world != args.gpus and rank == 0:
        print(f"bench: {world} rank(s) from the launcher, --gpus {args.gpus}; using {world}",
              file=sys.stderr)
    if local >= torch.cuda.device_count():
        raise SystemExit(f"bench: rank {rank} needs GPU {local}, only "
                         f"{torch.cuda.device_count()} visible")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    spec = CONFIGS[args.config]
    B_global = spec["batch"]
    pairs = shard(B_global, rank, world)
    if args.shard_of and world == 1:
        pairs = shard(B_global, 0, args.shard_of)
    c = make_config(args.config, pairs=pairs, mu=args.mu)
    d = len(c.shape)
    if d == 3 or args.scheme != "semi-lagrangian":
        # untimed input preparation: keep shoots finite (the explicit
        # Eulerian continuity step is CFL-limited at the SL configs' 1 px/step)
        from paper_2106_08817_b200.calibrate import calibrate_no_divergence

        calibrate_no_divergence(c, scheme=args.scheme)
    N = int(np.prod(c.shape))
    T = c.n_steps
    w = c.weights()
    dtype = torch.float32
    sl = args.scheme == "semi-lagrangian"
    # pair groups on concurrent streams (2D batches): FIR and transport kernels overlap
    groups = args.groups if args.groups is not None else (2 if d == 2 and len(pairs) >= 8 else 1)
    bg = engine.GroupedBatchGrad(len(pairs), c.shape, T, c.mu, w, c.lam, c.rho, dtype,
                                 scheme=args.scheme, groups=groups,
                                 deterministic=args.deterministic)
    bg.load(torch.as_tensor(c.source, dtype=dtype), torch.as_tensor(c.target, dtype=dtype),
            torch.as_tensor(c.z0, dtype=dtype))
    stream = torch.cuda.current_stream()

    # the whole grad (2T+1 forward + 2T+2 adjoint launches) replays as one CUDA graph
    step = bg.run
    if not args.no_graph:
        bg.capture_graph()
        step = bg.replay
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    vsteps_total = B_global * N * T
    value = vsteps_total / (ms_max * 1e-3)
    # the only collective: final gather of the per-pair CostReports (not timed)
    terms = bg.terms.clone()
    if world > 1:
        from paper_2106_08817_b200.distributed import gather_terms

        terms = gather_terms(terms, B_global)
    diverged = bool(engine.diverged_pairs(bg.guard).any())

    # ---- per-kernel device time (same stream, same buffers, live) ----
    ab = alg_bytes(d)
    Bl = len(pairs)
    hbm_peak, peak_kind = peaks()
    step_bytes = sum(ab.values()) * Bl * N * T
    step_achieved = step_bytes / (ms * 1e-3) / 1e9
    if d == 2 and sl:
        # each kernel as the step launches it: on one pair group's buffers (groups
        # run concurrently, so the shares are of serialised time and may sum > 1)
        g0 = bg.parts[0]
        kt = kernel_times(g0, w, stream)
        launches = {"velocity": T + 1, "sl_step": T, "sl_adjoint": T, "velocity_adjoint": T}
        share = {k: kt[k] * launches[k] * len(bg.parts) / ms for k in kt}
        dom = max(share, key=share.get)
        achieved = ab[dom] * g0.traj.batch * N / (kt[dom] * 1e-3) / 1e9
    else:  # 3D / Eulerian / Hybrid: report the whole step against HBM
        kt, share, dom = {}, {"step": 1.0}, "step"
        achieved = step_achieved
        kt["step"] = ms

    # ---- e2e through the public API with pinned host buffers ----
    e2e = run_e2e(c, args, dtype, world)

    line = {
        "metric": "voxel-steps/sec (fwd+adjoint shooting)",
        "value": value,
        "unit": "voxel-steps/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_max,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": f"synthetic (seeded cfg-{args.config} generator, calibrated z0; SURVEY §8(d))",
        "config": {
            "workload": f"{c.name}: {B_global} pairs x {'x'.join(map(str, c.shape))}, T={T}, "
                        f"sigma={c.sigma}, r={c.radius}, mu={c.mu}, grad() = shoot + adjoint"
                        + ("" if sl else f", scheme={args.scheme}"),
            "scheme": args.scheme,
            "momentum_scale": c.manifest.get("momentum_scale"),
            "offset_vox_per_step": c.manifest.get("offset_achieved"),
            "cuda_graph": not args.no_graph,
            "deterministic": bool(args.deterministic),
            "global_batch": B_global,
            "shape": list(c.shape),
            "n_steps": T,
            "parallelism": f"pairs sharded over {world} rank(s); no collective on the hot path",
            "l2": "inputs larger than L2 (trajectory %.1f GB per rank)" % (
                bg.trajectory_bytes() / 1e9),
        },
        "roofline": {
            "bound": "hbm",
            "kernel": dom,
            "achieved": achieved,
            "peak": hbm_peak,
            "unit": "GB/s",
            "frac": achieved / hbm_peak,
            "peak_kind": peak_kind,
            "alg_bytes_per_voxel": ab[dom] if dom in ab else sum(ab.values()) * T,
            "avg_launch_ms": kt[dom],
            "share_of_step": share[dom],
            "traffic": kernel_traffic(dom),
            "traffic_unit": "bytes per launch (dram read+write, ncu --set full, profiles/r02_traffic.json)",
        },
        "step_roofline": {
            "alg_bytes_per_voxel_step": sum(ab.values()),
            "achieved": step_achieved,
            "peak": hbm_peak,
            "unit": "GB/s",
            "frac": step_achieved / hbm_peak,
        },
        "kernels_ms": kt,
        "kernel_share": share,
        "gpu_launches": args.steps * bg.launches_per_run(),
        "pair_groups": len(bg.parts),
        "clocks": clk.summary(),
        "e2e": e2e,
        "diverged_pairs": diverged,
        "mean_cost": float(terms[:, 0].mean()),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_sample(c, w, args.scheme)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# kernels each bench operation launches (split FIR operations are two kernels)
NCU_NAMES = {"velocity": ("k_vel_a<", "k_vel_b<"),
             "velocity_adjoint": ("k_fir_axis0_f32<24, 1, 0>", "k_velocity_adj2d_h<"),
             "sl_adjoint": ("k_sl_adjoint2d_tma",), "sl_step": ("k_sl_step2d_tma",)}


def kernel_traffic(kernel: str):
    """DRAM bytes per launch of a bench kernel from the committed ncu capture."""
    try:
        with open(os.path.join(REPO, "profiles", "r02_traffic.json")) as f:
            tr = json.load(f)
    except Exception:
        return None
    keys = NCU_NAMES.get(kernel, ())
    found = [d["dram_bytes"] for key in keys for name, d in tr.items() if key in name]
    return sum(found) if keys and len(found) == len(keys) else None


def kernel_times(bg, w, stream, reps: int = 1) -> dict:
    """Average device time of one launch of each kernel, by CUDA events around
    a loop of its T launches on the bench's own stream and buffers."""
    import torch

    from paper_2106_08817_b200 import _lib

    lib = _lib.load_library()
    traj = bg.traj
    T = traj.n_steps
    B = traj.batch
    shape = traj.shape
    g = _lib.make_grid(B, shape)
    kern = _lib.KernelHandle(w)
    dt = _lib.dtype_code(traj.I.dtype)
    sp = _lib.stream_ptr(stream)
    P = _lib.ptr
    sI = torch.empty_like(traj.I[0])
    sz = torch.empty_like(traj.z[0])
    sv = torch.empty_like(traj.v[0])
    ws = torch.empty_like(traj.v[0])  # 2 scalars per pixel: the split kernels the step runs
    out = {}

    def timed(name, fn, n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fn(0)
        e0.record(stream)
        for k in range(n):
            fn(k)
        e1.record(stream)
        torch.cuda.synchronize()
        out[name] = e0.elapsed_time(e1) / n

    timed("velocity", lambda k: _lib.check(lib.mr_velocity(
        dt, g, kern.struct, P(traj.I[k]), P(traj.z[k]), P(sv), None, P(ws), sp)), T + 1)
    timed("sl_step", lambda k: _lib.check(lib.mr_sl_step(
        dt, g, 1.0 / T, bg.mu, P(traj.I[k]), P(traj.z[k]), P(traj.v[k]), P(sI), P(sz), None,
        None, sp)), T)
    timed("sl_adjoint", lambda k: _lib.check(lib.mr_sl_step_adjoint(
        dt, g, 1.0 / T, bg.mu, P(traj.I[k]), P(traj.z[k]), P(traj.v[k]), P(traj.I[k + 1]),
        P(traj.z[k + 1]), P(sI), P(sz), P(sv), sp)), T)
    timed("velocity_adjoint", lambda k: _lib.check(lib.mr_velocity_adjoint(
        dt, g, kern.struct, P(traj.I[k]), P(traj.z[k]), P(traj.v[k]), P(sI), P(sz), P(ws), sp)), T)
    return out


def run_e2e(c, args, dtype, world):
    """Same metric through the public API (objective.cost_and_grad_batch) called with
    pinned HOST tensors: every step uploads (I0, z0, J) and returns dH/dz0, the cost
    rows and the guard in host memory (the API pipelines the batch in pair groups so
    the PCIe copies overlap the other groups' shooting)."""
    import torch

    import paper_2106_08817_b200 as mr

    cfg = mr.ShootingConfig(mr.Scheme(args.scheme), c.n_steps, c.mu,
                            mr.GaussianKernel(c.sigma, c.radius),
                            deterministic=args.deterministic)
    src = torch.as_tensor(c.source, dtype=dtype).pin_memory()
    tgt = torch.as_tensor(c.target, dtype=dtype).pin_memory()
    z0 = torch.as_tensor(c.z0, dtype=dtype).pin_memory()
    stream = torch.cuda.current_stream()

    chunks = args.e2e_chunks
    if chunks is not None:
        chunks = [int(n) for n in chunks.split(",")] if "," in chunks else int(chunks)

    def step():
        zbar, terms, _ = mr.cost_and_grad_batch(src, tgt, z0, cfg, c.lam, c.rho, chunks=chunks)
        return zbar, terms

    steps = args.e2e_steps if args.e2e_steps is not None else max(3, min(args.steps, 10))
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    es = torch.finfo(dtype).bits // 8
    npair = c.batch
    Nv = int(np.prod(c.shape))
    from paper_2106_08817_b200.synthetic import CONFIGS

    B_global = CONFIGS[args.config]["batch"]
    return {
        "value": B_global * Nv * c.n_steps / (ms * 1e-3),
        "unit": "voxel-steps/s",
        "ms_per_step": ms,
        "steps": steps,
        "api": "paper_2106_08817_b200.cost_and_grad_batch",
        "h2d_bytes_per_step": 3 * npair * Nv * es,
        "d2h_bytes_per_step": npair * Nv * es + npair * 4 * 8 + npair * (c.n_steps + 1) * 4,
        "chunks": args.e2e_chunks,
    }


# ---------------------------------------------------------------------------------
def _oracle_grad_task(args):
    """One oracle grad() (float64 numpy port of the reference) on one pair."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import morphreg_oracle as O

    src, tgt, z0, T, mu, lam, rho, w = args[:8]
    scheme = args[8] if len(args) > 8 else "semi-lagrangian"
    t0 = time.perf_counter()
    O.grad(src, tgt, z0, lam, rho, T, mu, w, scheme=scheme)
    return time.perf_counter() - t0


def cpu_baseline_sample(c, w, scheme="semi-lagrangian"):
    """Oracle port on 1 host core, one pair: ~10-30 s of CPU work (2D: full T;
    3D: T truncated to 1 step -- the cost per voxel-step is T-independent)."""
    src, tgt, z0 = c.source[0], c.target[0], c.z0[0]
    T = c.n_steps if len(c.shape) == 2 else 1
    crop = ""
    if src.size > 8_000_000:  # cfg5 (256^3): the central 128^3 block keeps the sample ~10 s
        sl = tuple(slice((n - 128) // 2, (n - 128) // 2 + 128) for n in src.shape)
        src, tgt, z0 = src[sl], tgt[sl], z0[sl]
        crop = " (central 128^3 crop)"
    sec = _oracle_grad_task((src, tgt, z0, T, c.mu, c.lam, c.rho, w, scheme))
    vs = int(src.size) * T
    return {"value": vs / sec, "unit": "voxel-steps/s", "cores": 1, "kind": "port",
            "sample": f"oracle grad() of 1 pair {'x'.join(map(str, src.shape))}{crop}, T={T}, "
                      f"float64 numpy, 1 thread: {sec:.2f} s"}


def run_reference(args):
    """Reference arm: the reference algorithm's CPU implementation on all host cores."""
    import multiprocessing as mp

    from paper_2106_08817_b200.synthetic import CONFIGS, make_config

    rank, world, _ = dist_env()
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    spec = CONFIGS[args.config]
    # 2D: the full T of the config (same_config); 3D: one step (cost per voxel-step is
    # T-independent and a full-T 3D oracle grad takes minutes per pair)
    T_sample = spec["n_steps"] if len(spec["shape"]) == 2 else 1
    P = min(cores, spec["batch"])
    c = make_config(args.config, batch=P, mu=args.mu)
    w = c.weights()
    tasks = [(c.source[i], c.target[i], c.z0[i], T_sample, c.mu, c.lam, c.rho, w, args.scheme)
             for i in range(P)]
    Nv = int(np.prod(c.shape))
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        for _ in range(args.warmup):
            pool.map(_oracle_grad_task, tasks, chunksize=1)
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            pool.map(_oracle_grad_task, tasks, chunksize=1)
            times.append(time.perf_counter() - t0)
    sec = sum(times) / len(times)
    value = P * Nv * T_sample / sec
    line = {
        "impl": "reference",
        "metric": "voxel-steps/sec (fwd+adjoint shooting)",
        "value": value,
        "unit": "voxel-steps/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": sec * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": f"synthetic (seeded cfg-{args.config} generator, same as the GPU arm)",
        "config": {"workload": f"{c.name}: {P} of {spec['batch']} pairs per step, T={T_sample}"
                               + ("" if T_sample == spec["n_steps"] else
                                  f" (truncated from {spec['n_steps']}; cost is linear in T)"),
                   "global_batch": spec["batch"], "shape": list(c.shape)},
        "cpu_baseline": {"value": value, "unit": "voxel-steps/s", "cores": cores, "kind": "port",
                         "sample": f"{P} pairs x T={T_sample} per step, one pair per process, "
                                   f"oracle/morphreg_oracle.py (float64 numpy restatement of the "
                                   f"reference, bitwise-equal in 2D)"},
        "e2e": {"value": value, "unit": "voxel-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse()
    if maybe_relaunch(a):
        sys.exit(0)
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
