"""Benchmark of the MPO·MPS apply + simplify hot path.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C4]

Default workload: BASELINE.json config 4 (random D=8 MPO applied to an n=30,
chi=512 MPS, simplified back to chi=512 over 2 sweeps), the largest
apply+simplify config and the one the FP64 tensor-peak target is set on.
One step = one full `apply(MPO, MPS, Strategy)` call (blas.hpp:8-11): MPO
expansion + exact QR pass + truncating R->L pass + variational sweeps, with the
inputs already resident in HBM.  `e2e` repeats the step through the public host
API (host tensors in, host tensors out: H2D + call + D2H).

Multi-GPU: `--gpus N` without a torchrun environment re-launches itself under
`torch.distributed.run` with N ranks (one per GPU).  Single-chain configs do
not shard (the sweep is sequential along sites), so every rank compresses its
own independent chain (seed + 1000*rank, weak scaling).  `c5_scaling` adds the
batched config 5 (1024 chains) sharded over the N ranks with one NCCL
all-gather of per-chain (norm, error, sweeps) per batch.

`--impl reference` times the CPU restatement of the reference (oracle/; the
reference itself cannot be built here: it needs Eigen3) on the host cores.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MPO·MPS apply+simplify sweeps/sec; achieved FP64 TFLOP/s vs tensor-core peak"
FP64_DMMA_PEAK_TFLOPS = 37.07  # measured on this pool's B200: tools/fp64_peak (profiles/r01_fp64_peak.txt)
L2_FLUSH_BYTES = 512 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--chains", type=int, default=None, help="batch configs: total chains (default: config)")
    ap.add_argument("--no-c5", action="store_true", help="skip the c5_scaling measurement")
    ap.add_argument("--ref-step-s", type=float, default=10.0, help="reference arm: CPU seconds sampled per step")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
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
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def workload(cfg_name, rank, world=1, chains=None):
    from paper_2601_16734_b200 import inputs as I
    from paper_2601_16734_b200.batch import shard_range
    cfg = I.CONFIGS[cfg_name]
    if cfg.kind == "batch":
        total = chains or cfg.batch
        lo, hi = shard_range(total, world, rank)
        workers = max(1, (os.cpu_count() or 1) // world)
        return cfg, I.batch_inputs(cfg, lo, hi, workers), None
    import dataclasses
    cfg_r = dataclasses.replace(cfg, seed=cfg.seed + 1000 * rank)
    mps, W = I.config_inputs(cfg_r)
    return cfg, mps, W


def _call(ttlab, cfg, mps, W, strat, rep=None):
    """One call of the config's hot path (device objects or host tensors)."""
    if cfg.kind == "apply":
        return ttlab.apply(W, mps[0], strat, report=rep)
    if cfg.kind == "hadamard":
        return ttlab.simplify(ttlab.hadamard(mps[0], mps[1]), strat, report=rep)
    return ttlab.simplify(mps[0], strat, report=rep)


def _target_bonds(cfg, mps, W):
    if cfg.kind == "apply":
        return [1] + [w.shape[3] * a.shape[2] for w, a in zip(W, mps[0])]
    if cfg.kind == "hadamard":
        return [1] + [a.shape[2] * b.shape[2] for a, b in zip(mps[0], mps[1])]
    return [1] + [a.shape[2] for a in mps[0]]


LARGE = ("C3", "C4")  # configs whose full CPU call takes minutes: timed through oracle.cpu_model


def _output_bonds(cfg, t_bonds):
    """Output bond profile of the call: min(chi_out, d^k, d^(n-k), exact-pass rank)."""
    from paper_2601_16734_b200 import flops as F
    q = F.qr_pass_bonds(t_bonds, [cfg.d] * cfg.n)
    return [max(1, min(cfg.out_chi, cfg.d ** k, cfg.d ** (cfg.n - k), q[k])) for k in range(cfg.n + 1)]


def cpu_call_model(cfg, mps, W, threads, sweeps):
    """Unit model of one full call in reference arithmetic (oracle/cpu_model.py)."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(threads))
    from oracle.cpu_model import CallModel
    t_b = _target_bonds(cfg, mps, W)
    return CallModel(t_b, _output_bonds(cfg, t_b), [cfg.d] * cfg.n, sweeps, seed=cfg.seed)


def _model_sample(cfg, model, wall):
    return (f"unit model of one full {cfg.name} call in reference arithmetic (complex128, pair-first "
            f"project_pair, scprod <T,T>; oracle/cpu_model.py): {model.units_timed()} units timed "
            f"({wall:.0f} s, random operands of the exact unit shapes), covering {100 * model.coverage():.0f}% "
            f"of the call's estimated work directly; the {model.total_units()} units of the call are summed "
            "(untimed groups extrapolated from their kind's measured rate) - partial")


def cpu_reference(cfg, mps, W, steps, warmup, threads):
    """Time the oracle restatement (reference arithmetic: complex128 promotion,
    pair-first project_pair, scprod <T,T>) on the host cores."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(threads))
    from oracle import ttlab_oracle as O
    strat = O.Strategy(max_bond=cfg.out_chi, tolerance=cfg.tolerance, max_sweeps=cfg.max_sweeps)
    ms = [O.MPS(m) for m in mps]

    def once(rep=None):
        if cfg.kind == "apply":
            return O.apply(O.MPO(W), ms[0], strat, promote=True, report=rep)
        if cfg.kind == "hadamard":
            return O.simplify(O.hadamard(ms[0], ms[1]), strat, promote=True, report=rep)
        return O.simplify(ms[0], strat, promote=True, report=rep)

    for _ in range(warmup):
        once()
    sweeps, t0 = 0, time.perf_counter()
    for _ in range(steps):
        rep = {}
        once(rep)
        sweeps += rep["sweeps"]
    dt = time.perf_counter() - t0
    return sweeps / dt, dt, sweeps


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    from paper_2601_16734_b200 import inputs as I
    cfg = I.CONFIGS[args.config]
    if cfg.kind == "batch":  # each step: `threads` chains on a pool of single-threaded workers
        t_all, sw_all = 0.0, 0.0
        for _ in range(args.steps):
            v, cps, dt = cpu_reference_batch(cfg, threads, threads)
            t_all += dt
            sw_all += v * dt
        val, dt = sw_all / t_all, t_all
        line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "sweeps/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": 0, "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
                "config": {"workload": f"{cfg.name} batched simplify (sample of {threads} chains per step)",
                           "parallelism": f"{threads} single-threaded host workers"},
                "cpu_baseline": {"value": val, "unit": "sweeps/s", "cores": threads, "kind": "port",
                                 "sample": f"{args.steps} x {threads} chains, oracle/ in reference arithmetic"},
                "e2e": {"value": val, "unit": "sweeps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    cfg, mps, W = workload(args.config, 0)
    if cfg.name in LARGE:
        model = cpu_call_model(cfg, mps, W, threads, cfg.max_sweeps)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            model.measure(args.ref_step_s)
        wall = time.perf_counter() - t0
        t_call = model.estimate()
        val = cfg.max_sweeps / t_call
        line = {
            "impl": "reference", "metric": METRIC, "value": val, "unit": "sweeps/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": 0, "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic", "partial": True,
            "config": {"workload": _workload_desc(cfg), "parallelism": "host threads"},
            "full_call_s_estimate": t_call, "sweeps_per_call": cfg.max_sweeps,
            "cpu_baseline": {"value": val, "unit": "sweeps/s", "cores": threads, "kind": "port",
                             "sample": f"{args.steps} steps of ~{args.ref_step_s:.0f} s: " + _model_sample(cfg, model, wall)},
            "e2e": {"value": val, "unit": "sweeps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return
    val, dt, sweeps = cpu_reference(cfg, mps, W, args.steps, min(args.warmup, 1), threads)
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "sweeps/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": min(args.warmup, 1), "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": _workload_desc(cfg), "parallelism": "host threads"},
        "cpu_baseline": {"value": val, "unit": "sweeps/s", "cores": threads, "kind": "port",
                         "sample": f"{args.steps} full {cfg.name} apply+simplify calls, numpy/scipy restatement "
                                   "(oracle/) in reference arithmetic (complex128, pair-first projection)"},
        "e2e": {"value": val, "unit": "sweeps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _workload_desc(cfg):
    tail = f"simplify to chi={cfg.out_chi}, tol {cfg.tolerance:g}, max {cfg.max_sweeps} sweeps"
    if cfg.kind == "apply":
        mpo = "QTT Laplacian D=3" if cfg.mpo_D == 3 else f"random MPO D={cfg.mpo_D}"
        return (f"{cfg.name}: {mpo} applied to n={cfg.n} d={cfg.d} chi={cfg.chi} f64 MPS (seed {cfg.seed}+1000*rank), "
                + tail)
    if cfg.kind == "hadamard":
        return (f"{cfg.name}: Hadamard product of two n={cfg.n} d={cfg.d} chi={cfg.chi} complex128 MPS "
                f"(seeds {cfg.seed}/{cfg.seed + 1}), " + tail)
    return f"{cfg.name}: n={cfg.n} d={cfg.d} chi={cfg.chi} f64 MPS (seed {cfg.seed}+1000*rank), " + tail


# DRAM bytes per launch of the dominant SVD kernel (dram__bytes_read.sum + dram__bytes_write.sum,
# ncu --clock-control none, profiles/r01_dram_svd.txt): the split matrices stay L2-resident, so
# traffic is about one read of the matrix per launch
_SVD_TRAFFIC = {"C2": {"kernel": "jacobi_cluster_kernel<double,16,8,128,2>", "bytes": 204117},
                # round 2: block-Gram Jacobi on a 1024 x 1024 split (profiles/r02_jbg_c4.raw.csv: 8.46 MB read +
                # 1.92 MB written for the 8 MiB matrix, 14.0 ms)
                "C4": {"kernel": "jacobi_bg_kernel<16,256>", "bytes": 10379520}}


def _roofline(prof, cfg_name=None):
    """Roofline of the dominant kernel class of a profiled call (CUDA events around
    every launch, executed flops from the live bond table)."""
    dom = max(("gemm", "svd", "qr"), key=lambda k: prof[k]["ms"])
    p = prof[dom]
    achieved = p["flops"] / (p["ms"] / 1e3) / 1e12 if p["ms"] > 0 else 0.0
    return {
        "bound": "tensor",  # the FP64 tensor pipe (DMMA); on B200 the FP64 FMA pipe has the same peak
        "pipe": "fp64 (DMMA m16n8k4 / DFMA)",
        "kernel": {"gemm": "ttg::gemm_kernel (DMMA m16n8k4)",
                   "svd": "ttg::" + (_SVD_TRAFFIC[cfg_name]["kernel"] if cfg_name in _SVD_TRAFFIC
                                     else "jacobi_svd_kernel"),
                   "qr": "ttg::qr_panel_cl_kernel + DMMA updates"}[dom],
        "achieved": achieved, "peak": FP64_DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
        "frac": achieved / FP64_DMMA_PEAK_TFLOPS,
        "traffic": (_SVD_TRAFFIC[cfg_name]["bytes"] if dom == "svd" and cfg_name in _SVD_TRAFFIC else None),
        "traffic_unit": "bytes per launch of the dominant kernel (ncu dram__bytes_read+write)",
        "per_launch": {"launches_per_step": p["launches"], "avg_us": 1e3 * p["ms"] / max(1, p["launches"]),
                       "flops_per_launch": p["flops"] / max(1, p["launches"])},
        "share_of_step": {k: v["ms"] / max(1e-9, sum(x["ms"] for x in prof.values())) for k, v in prof.items()},
        "peak_source": "measured FP64 DMMA (mma.sync m16n8k4) 37.07 TF/s on this pool, tools/fp64_peak; "
                       "MEASURED_PEAKS.json has no FP64 entry; DFMA measured 36.8 TF/s, cuBLAS DGEMM 35.5",
        "flops_model": "executed flops: 2MNK per GEMM from the live bond table; SVD = Golub-Van Loan "
                       "4m^2n+8mn^2+9n^3; QR = 4n^2(m-n/3)",
    }


def _need_gpus(torch, world):
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        raise SystemExit(f"bench.py: needs {world} CUDA device(s) (one rank per GPU), "
                         f"found {torch.cuda.device_count() if torch.cuda.is_available() else 0}; no CPU fallback")


def _context_comm(ctx, torch, dist, rank, world):
    """Give the library context its NCCL communicator (ttg_comm_init; id shipped by torch.distributed) and
    agree over the ranks whether every one got it; otherwise the stats collective goes through
    torch.distributed's NCCL all-gather."""
    if world == 1:
        return True
    n, _ = ctx.comm_info()
    ok = 1
    if n != world:
        try:
            from paper_2601_16734_b200.batch import init_context_comm
            init_context_comm(ctx, world, rank)
        except Exception as e:  # noqa: BLE001 - reported, then the torch collective is used on every rank
            print(f"bench.py[rank {rank}]: context communicator unavailable ({e}); using torch.distributed",
                  file=sys.stderr)
            ok = 0
    flag = torch.tensor([ok], dtype=torch.int32, device=torch.device("cuda", torch.cuda.current_device()))
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    return bool(flag.item())


def c5_scaling(ttlab, torch, dist, ctx, stream, rank, world, steps=3):
    """Config 5 (1024 chains, chi 128 -> 64) sharded over the ranks: chains/s at
    this N and T1/(N T_N), T1 timed on rank 0 with the whole batch."""
    import numpy as np
    from paper_2601_16734_b200.batch import gather_chain_stats, gather_chain_stats_ctx
    native = _context_comm(ctx, torch, dist, rank, world)
    cfg, chains, _ = workload("C5", rank, world)
    total = cfg.batch
    strat = ttlab.Strategy(max_bond=cfg.out_chi, tolerance=cfg.tolerance, max_sweeps=cfg.max_sweeps)
    dev = torch.device("cuda", torch.cuda.current_device())

    def timed(batch, nsteps, collective):
        ttlab.simplify(batch, strat)  # warm-up
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sweeps = 0
        e0.record(stream)
        for _ in range(nsteps):
            reps = []
            ttlab.simplify(batch, strat, report=reps)
            if native:  # the collective on the communicator the library context owns (ttg_comm_allgather_f64)
                st = np.array([[r["norm"], r["error"], float(r["sweeps"])] for r in reps])
                allst = gather_chain_stats_ctx(ctx, st, total, world) if collective else st
                sweeps += int(allst[:, 2].sum())
            else:
                st = torch.tensor([[r["norm"], r["error"], float(r["sweeps"])] for r in reps], dtype=torch.float64,
                                  device=dev)
                allst = gather_chain_stats(st, total, world) if collective else st
                sweeps += int(allst[:, 2].sum().item())
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / nsteps, sweeps / nsteps

    batch = ttlab.DeviceMPS.from_batch(chains, ctx=ctx)
    if world > 1:
        dist.barrier()
    ms, sweeps = timed(batch, steps, True)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_n = float(t[0])
    del batch
    t_1 = t_n
    if world > 1:
        if rank == 0:
            _, full, _ = workload("C5", 0, 1)
            fb = ttlab.DeviceMPS.from_batch(full, ctx=ctx)
            t_1, _ = timed(fb, steps, False)
            del fb
        t1 = torch.tensor([t_1], dtype=torch.float64, device=dev)
        dist.broadcast(t1, 0)
        t_1 = float(t1[0])
    return {"workload": f"C5: {total} chains n={cfg.n} chi={cfg.chi}->{cfg.out_chi}, {total // world} per GPU, "
                        "NCCL all-gather of per-chain (norm, error, sweeps) per batch",
            "n_gpus": world, "ms_per_batch": t_n, "chains_per_s": total / (t_n / 1e3),
            "sweeps_per_batch": sweeps, "t1_ms_per_batch": t_1, "efficiency_t1_over_n_tn": t_1 / (world * t_n),
            "collective": ("ttg_comm_allgather_f64 on the context's own NCCL communicator" if native
                           else "torch.distributed all_gather_into_tensor (NCCL)"),
            "steps": steps}


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2601_16734_b200 import flops as F
    from paper_2601_16734_b200 import ttlab

    rank, world, local = dist_env()
    _need_gpus(torch, world)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    cfg, mps, W = workload(args.config, rank)
    strat = ttlab.Strategy(max_bond=cfg.out_chi, tolerance=cfg.tolerance, max_sweeps=cfg.max_sweeps)

    ctx = ttlab.context(local)
    stream = torch.cuda.Stream(dev)  # a real stream: the library and the events share it
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    Wd = ttlab.DeviceMPO(W, ctx=ctx) if W is not None else None
    mpsd = [ttlab.DeviceMPS.from_tensors(m, ctx=ctx) for m in mps]
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    # warm-up
    for _ in range(args.warmup):
        out = _call(ttlab, cfg, mpsd, Wd, strat)
    torch.cuda.synchronize()

    # ---- timed: device-resident inputs
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    sweeps = 0
    launches0 = ctx.kernel_launches
    reps = []
    for i in range(args.steps):
        flush.zero_()  # L2 flush between timed steps (outside the events)
        rep = []
        ev[i][0].record(stream)
        out = _call(ttlab, cfg, mpsd, Wd, strat, rep)
        ev[i][1].record(stream)
        sweeps += rep[0]["sweeps"]
        reps.append(rep[0])
    torch.cuda.synchronize()
    barrier()
    launches = ctx.kernel_launches - launches0
    clk = clocks.stop()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    out_bonds = out.bond_dimensions()

    # ---- e2e through the public host API (H2D + call + D2H every step)
    for _ in range(1):
        _call(ttlab, cfg, mps, W, strat).to_tensors()
    torch.cuda.synchronize()
    barrier()
    e2e_sweeps, t_e2e = 0, 0.0
    h2d = sum(a.nbytes for m in mps for a in m) + (sum(np.asarray(w).nbytes for w in W) if W is not None else 0)
    d2h = 0
    for i in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = []
        res = _call(ttlab, cfg, mps, W, strat, rep).to_tensors()
        t_e2e += time.perf_counter() - t0
        e2e_sweeps += rep[0]["sweeps"]
        d2h = sum(a.nbytes for a in res)
    barrier()

    # ---- max over ranks; gather per-chain scalars over NCCL
    stats = torch.tensor([ms, t_e2e * 1e3, float(sweeps), float(e2e_sweeps), reps[-1]["residual"],
                          reps[-1]["norm"]], dtype=torch.float64, device=dev)
    if world > 1:
        allst = [torch.empty_like(stats) for _ in range(world)]
        dist.all_gather(allst, stats)
        allst = torch.stack(allst).cpu().numpy()
    else:
        allst = stats.cpu().numpy()[None]
    ms_max = float(allst[:, 0].max())
    e2e_ms_max = float(allst[:, 1].max())
    total_sweeps = float(allst[:, 2].sum())
    total_e2e_sweeps = float(allst[:, 3].sum())
    value = total_sweeps / (ms_max / 1e3)
    e2e_value = total_e2e_sweeps / (e2e_ms_max / 1e3)

    # ---- algorithmic work and roofline (profiled pass, separate from the timed one)
    t_b = _target_bonds(cfg, mps, W)
    fl = F.algorithmic_flops(t_b, out_bonds, [2] * cfg.n, int(round(sweeps / args.steps)), complex_=cfg.complex_)
    f_alg = fl["F_alg"]
    tflops = f_alg / (ms / args.steps / 1e3) / 1e12
    roofline = None
    prof = None
    if not args.no_profile:
        ctx.profile_enable(True)
        _call(ttlab, cfg, mpsd, Wd, strat)
        prof = ctx.profile_read()
        ctx.profile_enable(False)
        roofline = _roofline(prof, cfg.name)

    if roofline is not None:
        roofline["call"] = {"F_alg_tflop": f_alg / 1e12, "achieved": tflops, "frac": tflops / FP64_DMMA_PEAK_TFLOPS,
                            "note": "whole call: algorithmic flops (SURVEY §8d F_alg) / device time per call"}
    c5 = None
    if not args.no_c5:
        c5 = c5_scaling(ttlab, torch, dist, ctx, stream, rank, world)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        if cfg.name in LARGE:
            model = cpu_call_model(cfg, mps, W, threads, int(round(sweeps / args.steps)))
            t0 = time.perf_counter()
            model.measure(25.0)
            wall = time.perf_counter() - t0
            v = int(round(sweeps / args.steps)) / model.estimate()
            cpu = {"value": v, "unit": "sweeps/s", "cores": threads, "kind": "port", "partial": True,
                   "full_call_s_estimate": model.estimate(), "sample": _model_sample(cfg, model, wall)}
        else:
            v, dt, sw = cpu_reference(cfg, mps, W, 1, 0, threads)
            cpu = {"value": v, "unit": "sweeps/s", "cores": threads, "kind": "port",
                   "sample": f"1 full {cfg.name} call ({sw} sweeps, {dt:.1f} s), numpy/scipy restatement "
                             "(oracle/) in reference arithmetic (complex128 promotion, pair-first projection)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "sweeps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128" if cfg.complex_ else "f64", "data": "synthetic",
            "config": {"workload": _workload_desc(cfg), "global_batch": world, "chains_per_gpu": 1,
                       "parallelism": f"dp{world} (independent chains)", "l2": "flushed between steps (512 MiB write)",
                       "output_bonds_max": max(out_bonds)},
            "fp64_tflops": tflops, "fp64_frac_of_peak": tflops / FP64_DMMA_PEAK_TFLOPS,
            "work": {"F_alg_gflop_per_step": f_alg / 1e9, **{k: v / 1e9 for k, v in fl.items()}},
            "e2e": {"value": e2e_value, "unit": "sweeps/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches),
            "roofline": roofline,
            "profile": prof,
            "cpu_baseline": cpu,
            "clocks": clk,
            "c5_scaling": c5,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _cpu_chain(args_):
    """One chain of the batched config through the oracle (single-threaded worker)."""
    chain, cfgname = args_
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from oracle import ttlab_oracle as O
    from paper_2601_16734_b200 import inputs as I
    cfg = I.CONFIGS[cfgname]
    (psi,), _ = I.config_inputs(cfg, chain=chain)
    rep = {}
    t0 = time.perf_counter()
    O.simplify(O.MPS(psi), O.Strategy(max_bond=cfg.out_chi, tolerance=cfg.tolerance, max_sweeps=cfg.max_sweeps),
               promote=True, report=rep)
    return rep["sweeps"], time.perf_counter() - t0


def cpu_reference_batch(cfg, nchains, threads):
    """A pool of `threads` single-threaded oracle workers over `nchains` chains
    (BASELINE.md CPU plan for config 5); returns (sweeps/s, chains/s, seconds)."""
    import multiprocessing as mpr
    t0 = time.perf_counter()
    with mpr.get_context("spawn").Pool(threads, initializer=_pin_blas) as pool:
        res = pool.map(_cpu_chain, [(c, cfg.name) for c in range(nchains)])
    dt = time.perf_counter() - t0
    return sum(r[0] for r in res) / dt, nchains / dt, dt


def _pin_blas():
    os.environ["OPENBLAS_NUM_THREADS"] = "1"


def run_ours_batch(args):
    """Config 5: independent chains sharded over ranks, one batched simplify per
    step on each GPU, per-chain (norm, error, sweeps) all-gathered over NCCL."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2601_16734_b200 import ttlab
    from paper_2601_16734_b200.batch import gather_chain_stats

    rank, world, local = dist_env()
    _need_gpus(torch, world)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    total = args.chains or None
    cfg, chains, _ = workload(args.config, rank, world, total)
    total = args.chains or cfg.batch
    strat = ttlab.Strategy(max_bond=cfg.out_chi, tolerance=cfg.tolerance, max_sweeps=cfg.max_sweeps)
    ctx = ttlab.context(local)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    batch = ttlab.DeviceMPS.from_batch(chains, ctx=ctx)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def step(target):
        reps = []
        out = ttlab.simplify(target, strat, report=reps)
        st = torch.tensor([[r["norm"], r["error"], float(r["sweeps"])] for r in reps], dtype=torch.float64,
                          device=dev)
        allst = gather_chain_stats(st, total, world)
        return out, reps, allst

    for _ in range(args.warmup):
        step(batch)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = ctx.kernel_launches
    sweeps = 0
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record(stream)
        out, reps, allst = step(batch)
        ev[i][1].record(stream)
        sweeps += int(allst[:, 2].sum().item())
    torch.cuda.synchronize()
    barrier()
    launches = ctx.kernel_launches - launches0
    clk = clocks.stop()
    ms = sum(a.elapsed_time(b) for a, b in ev)

    # e2e: host chains in, host chains out
    h2d = sum(a.nbytes for ch in chains for a in ch)
    barrier()
    t_e2e, e2e_sweeps, d2h = 0.0, 0, 0
    for i in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out, reps, allst = step(ttlab.DeviceMPS.from_batch(chains, ctx=ctx))
        res = out.to_tensors_batch()
        t_e2e += time.perf_counter() - t0
        e2e_sweeps += int(allst[:, 2].sum().item())
        d2h = sum(a.nbytes for ch in res for a in ch)
    ms_t = torch.tensor([ms, t_e2e * 1e3], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max, e2e_ms_max = float(ms_t[0]), float(ms_t[1])
    value = sweeps / (ms_max / 1e3)
    e2e_value = e2e_sweeps / (e2e_ms_max / 1e3)
    prof = None
    if not args.no_profile:
        ctx.profile_enable(True)
        step(batch)
        prof = ctx.profile_read()
        ctx.profile_enable(False)
    roofline = _roofline(prof, cfg.name) if prof else None
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        v, cps, dt = cpu_reference_batch(cfg, threads, threads)
        cpu = {"value": v, "unit": "sweeps/s", "cores": threads, "kind": "port", "chains_per_s": cps,
               "sample": f"{threads} chains of {cfg.name} on a pool of {threads} single-threaded workers "
                         f"({dt:.1f} s), oracle/ in reference arithmetic (complex128)"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "sweeps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak" if args.chains is None and world == 1 else "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{cfg.name}: {total} independent n={cfg.n} d={cfg.d} chi={cfg.chi} f64 MPS "
                                   f"(seeds {cfg.seed}+i), simplify to chi={cfg.out_chi}, tol {cfg.tolerance:g}, "
                                   f"max {cfg.max_sweeps} sweeps", "global_batch": total,
                       "chains_per_gpu": len(chains), "parallelism": f"dp{world} (chain shards, NCCL all-gather "
                                                                      "of per-chain norm/error/sweeps)",
                       "l2": "flushed between steps (512 MiB write)"},
            "chains_per_s": total * args.steps / (ms_max / 1e3),
            "e2e": {"value": e2e_value, "unit": "sweeps/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches), "roofline": roofline, "profile": prof, "cpu_baseline": cpu, "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(args) -> int:
    """`--gpus N` outside torchrun: re-launch this script with N ranks (one per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    rank, world, _ = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    from paper_2601_16734_b200 import inputs as I
    batch = I.CONFIGS[args.config].kind == "batch"
    if args.impl == "reference":
        run_reference(args)
    elif batch:
        run_ours_batch(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
