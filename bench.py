#!/usr/bin/env python
"""Benchmark of the B200 PSCA hot path (driver contract).

Workload (BASELINE.json configs[1], the config the metric is quoted on):
PSCA-MLE with unknown pathloss (ml-ud), N=1000 devices, L=40, M=128, K=50
active, T=100 iterations from gamma=0 with the default step rule, a batch of
4096 independent instances per GPU (weak scaling: rank r solves instances
r*4096 .. r*4096+4095; no collective on the data path).  One "step" = one
batched solve of the whole batch.

  value  instances/s over all ranks, inputs resident in HBM, device-timed
         (CUDA events, barrier + synchronize on both sides, max over ranks)
  e2e    the same through the public API (psca_run_batch) from pinned HOST
         buffers: H2D of the step's pilots / Sigma_hat / noise and D2H of the
         estimates inside the timed region
  roofline  the dominant kernel (the warp-streamed column kernel): the FP64
         DMMA flops it EXECUTES per launch (closed form per 8-column block +
         the moving columns of the rebuild, counted exactly in an untimed
         iterate-recording pass) / its mean SERIALISED launch time (one solve
         with every launch on one stream, CUDA events around each launch),
         against the FP64 peak measured live (cuBLAS DGEMM); the algorithmic
         24 N L^2 ratio is reported beside it as algorithmic_frac
  cpu_baseline  the CPU oracle (numpy/OpenBLAS restatement of the reference)
         on this host's cores, one process per core, bounded sample

``--config`` selects another BASELINE configuration (c0, c2, c2net, c3_l20,
c3_l40, c3_l80, c4); the driver's default line is c1.  ``--impl reference``
times the reference algorithm's CPU implementation (the oracle port; the
reference is pure Python and cannot travel to the box) on the same workload
with all host cores (scene generation untimed) and prints the same JSON line.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import pathlib
import statistics
import sys
import threading
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "detection instances/sec and PSCA iters/sec at N=1000,L=40,M=128; % of roofline"
UNIT = "instances/s"
CONFIGS = ["c0", "c1", "c2", "c2net", "c3_l20", "c3_l40", "c3_l80", "c4"]
DMMA_FLOPS = 512.0   # mma.m8n8k4.f64: 8 x 8 x 4 multiply-adds


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=0, help="instances per GPU (default: config)")
    ap.add_argument("--iters", type=int, default=0, help="PSCA iterations (default: config)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="CPU-baseline sample budget (seconds of solve time per worker)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-executed", action="store_true",
                    help="skip the untimed iterate-recording pass that counts executed DMMAs")
    ap.add_argument("--config", default="c1", choices=CONFIGS,
                    help="BASELINE configuration: c1 (headline, default), c0, c2, c2net (the "
                         "PSCA-Net forward of c2), c3_l20/l40/l80, or c4 (one N=100000, L=256 "
                         "instance, devices column-sharded over the ranks, NCCL all-reduce per "
                         "iteration)")
    return ap.parse_args()


class Workload:
    """One BASELINE configuration as the bench runs it."""

    def __init__(self, name: str, iters: int = 0, batch: int = 0):
        from paper_2503_15259_b200 import estimators, scenes
        self.name = name
        self.scene_name = "c2" if name == "c2net" else name
        self.cfg = scenes.BASELINE_CONFIGS[self.scene_name]
        self.net = name == "c2net"
        if self.net:
            self.steps = scenes.net_steps(self.cfg.net_blocks)
            self.iters = iters or self.cfg.net_blocks
            self.schedule = estimators.StepSchedule.explicit(self.steps)
        else:
            self.iters = iters or self.cfg.n_iter
            self.schedule = estimators.StepSchedule.default()
            self.steps = self.schedule.materialize(self.iters)
        self.batch = batch or self.cfg.batch
        self.problem = scenes.problem_for(self.cfg)
        self.known = self.cfg.kind in ("ml-k", "map-k")
        c = self.cfg
        what = {"ml-k": "PSCA-MLE known pathloss (ml-k)", "ml-ud": "PSCA-MLE unknown pathloss (ml-ud)",
                "map-k": "PSCA-MAPE known pathloss (map-k, p=0.05)",
                "map-ur": "PSCA-MAPE unknown pathloss (map-ur, smoothed effective-pathloss prior)"}
        step_rule = ("PSCA-Net forward, T=10 seeded per-layer steps" if self.net
                     else "default step rule")
        self.description = (f"{name}: {what[c.kind]}, N={c.n_devices}, L={c.pilot_len}, "
                             f"M={c.n_antennas}, K={c.n_active} active, T={self.iters} iterations, "
                             f"{step_rule}, complex128")
        self.metric = METRIC if name == "c1" else \
            f"detection instances/sec and PSCA iters/sec at {name} (N={c.n_devices},L={c.pilot_len},M={c.n_antennas}); % of roofline"

    def config_block(self, batch, per_gpu=True, world=1):
        c = self.cfg
        pil = 16 * c.pilot_len * c.n_devices
        return {"workload": self.description,
                "instances_per_gpu" if per_gpu else "instances_per_step": batch,
                "N": c.n_devices, "L": c.pilot_len, "M": c.n_antennas, "T": self.iters,
                "kind": c.kind,
                "l2": (f"inputs larger than L2 (pilots {pil // 1024} KB/instance, "
                       f"{pil * batch / 1e9:.2f} GB per GPU vs 126 MB L2)") if pil * batch > 126e6
                      else "inputs smaller than L2: every timed step re-reads them from L2 "
                           "(latency-bound single instance)",
                "parallelism": (f"instance sharding over {world} GPU(s), no collective"
                                if batch > 1 else "one instance (replicas only)")}


# ---------------------------------------------------------------------------
# inputs
# ---------------------------------------------------------------------------

def _gen_chunk(args):
    name, ids = args
    from paper_2503_15259_b200 import scenes
    cfg = scenes.BASELINE_CONFIGS[name]
    samples = [scenes.make_scene(cfg, i) for i in ids]
    return scenes.stack_batch(samples)


def generate(name: str, ids: list[int], workers: int):
    """Seeded scenes for instance ids (parallel over host processes)."""
    import multiprocessing as mp
    import numpy as np
    chunks = [ids[i:i + 64] for i in range(0, len(ids), 64)]
    if workers > 1 and len(chunks) > 1:
        ctx = mp.get_context("fork")
        with ctx.Pool(min(workers, len(chunks))) as pool:
            parts = pool.map(_gen_chunk, [(name, c) for c in chunks])
    else:
        parts = [_gen_chunk((name, c)) for c in chunks]
    out = {k: np.concatenate([p[k] for p in parts]) for k in ("pilots", "gains", "emp_cov",
                                                              "noise", "activities")}
    out["n_antennas"] = parts[0]["n_antennas"]
    return out


def _draw_chunk(args):
    name, ids = args
    from paper_2503_15259_b200 import scenes
    cfg = scenes.BASELINE_CONFIGS[name]
    return [scenes.draw_scene(cfg, i) for i in ids]


def generate_device(name: str, ids: list[int], workers: int):
    """Seeded scenes with the covariances formed on the GPU: the Philox draws in
    host processes, Y = S_A diag(sqrt(g_A)) H + Z and Sigma_hat = Y Y^H / M on
    DMMA (scenes.make_batch_device).  Returns (device batch, host arrays for
    the e2e arm, timing dict)."""
    import multiprocessing as mp
    import numpy as np
    import torch
    from paper_2503_15259_b200 import scenes
    cfg = scenes.BASELINE_CONFIGS[name]
    t0 = time.perf_counter()
    chunks = [ids[i:i + 64] for i in range(0, len(ids), 64)]
    if workers > 1 and len(chunks) > 1:
        with mp.get_context("fork").Pool(min(workers, len(chunks))) as pool:
            parts = pool.map(_draw_chunk, [(name, c) for c in chunks])
    else:
        parts = [_draw_chunk((name, c)) for c in chunks]
    draws = [d for part in parts for d in part]
    t_draw = time.perf_counter() - t0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dev = scenes.make_batch_device(cfg, ids, draws=draws)
    e1.record()
    torch.cuda.synchronize()
    host = {"pilots": np.stack([d["pilots"] for d in draws]),
            "gains": np.stack([d["gains"] for d in draws]),
            "emp_cov": dev["emp_cov"].cpu().numpy(), "noise": dev["noise"].cpu().numpy(),
            "activities": dev["activities"], "n_antennas": cfg.n_antennas}
    timing = {"host_draws_s": t_draw, "host_draw_workers": workers,
              "device_cov_ms": e0.elapsed_time(e1),
              "note": "Philox draws on the host (the scene contract), Y and Sigma_hat on the "
                      "FP64 tensor pipe incl. the host-to-device copy of the draws "
                      "(psca_received + psca_empirical_cov); outside the timed solve region"}
    return dev, host, timing


# ---------------------------------------------------------------------------
# CPU baseline (oracle, one process per core, OPENBLAS_NUM_THREADS=1)
# ---------------------------------------------------------------------------

def _oracle_solve(wl, s):
    import numpy as np
    from oracle import psca_oracle as orc
    cfg = wl.cfg
    kw = {}
    if cfg.kind == "map-k":
        kw["indep_p"] = np.full(cfg.n_devices, cfg.p)
    elif cfg.kind == "map-ur":
        kw["eff"] = orc.EffPrior.from_reference(wl.problem.prior)
    return orc.psca(cfg.kind, s.pilots, s.gains, s.emp_cov, s.noise_power, s.n_antennas,
                    wl.steps, wl.iters, **kw)


def _cpu_worker(args):
    """Solve instances of the workload on one core: scene generation untimed, the
    oracle solve timed.  per_step > 0: exactly that many instances; else until
    budget_s of solve time."""
    wid, nworkers, budget_s, name, iters, per_step, base = args
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from paper_2503_15259_b200 import scenes
    wl = Workload(name, iters)
    done, solve_s = 0, 0.0
    i = wid
    while (per_step and done < per_step) or (not per_step and solve_s < budget_s):
        s = scenes.make_scene(wl.cfg, base + i)
        t0 = time.perf_counter()
        _oracle_solve(wl, s)
        solve_s += time.perf_counter() - t0
        done += 1
        i += nworkers
    return done, solve_s


def _cpu_pool(workers):
    import multiprocessing as mp
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    return mp.get_context("spawn").Pool(workers)


def cpu_baseline(name: str, iters: int, budget_s: float) -> dict:
    workers = os.cpu_count() or 1
    with _cpu_pool(workers) as pool:
        pool.map(_cpu_worker, [(w, workers, 0.0, name, 2, 1, 10_000_000) for w in range(workers)])
        res = pool.map(_cpu_worker, [(w, workers, budget_s, name, iters, 0, 10_000_000)
                                     for w in range(workers)])
    n = sum(r[0] for r in res)
    rate = sum(r[0] / r[1] for r in res if r[1] > 0)
    return {"value": rate, "unit": UNIT, "cores": workers, "kind": "port",
            "sample": f"{n} {name} instances (T={iters}) solved by the numpy/OpenBLAS oracle, "
                      f"{workers} processes x 1 BLAS thread, ~{budget_s:.0f} s of solve time each; "
                      "scene generation excluded"}


# ---------------------------------------------------------------------------
# clocks (NVML, sampled during the timed region)
# ---------------------------------------------------------------------------

_REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
            0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
            0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
            0x100: "display_clock_setting"}


class ClockSampler:
    def __init__(self, index: int):
        self.samples, self.reasons = [], 0
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                fn = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    nv.nvmlDeviceGetCurrentClocksThrottleReasons
                self.reasons |= int(fn(self.h))
            except Exception:
                pass
            time.sleep(0.2)

    def __enter__(self):
        if self.nv is not None:
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": [n for b, n in _REASONS.items() if self.reasons & b and b != 0x1],
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# FP64 peak (cuBLAS DGEMM, measured live)
# ---------------------------------------------------------------------------

def fp64_peak_tflops(torch) -> float:
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = math.inf
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


def ncu_pipe(name: str = "column_kernel"):
    """DMMA sub-pipe busy fraction of the kernel's committed full ncu capture, if any."""
    p = ROOT / "profiles" / "ncu_summary.json"
    try:
        return json.loads(p.read_text())[name]["dmma_pipe_active_pct_full_capture"] / 100.0
    except Exception:
        return None


def ncu_traffic(name: str = "column_kernel"):
    """dram bytes per launch of the column kernel from the committed ncu summary, if any."""
    p = ROOT / "profiles" / "ncu_summary.json"
    try:
        d = json.loads(p.read_text())
        return d[name]["dram_bytes_per_launch"]
    except Exception:
        return None


# ---------------------------------------------------------------------------
# arms
# ---------------------------------------------------------------------------

def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def instance_ids(rank: int, per_rank: int) -> list[int]:
    """Instance sharding (c1-c3): rank r owns the scene seeds [r B, (r + 1) B) -- disjoint
    blocks, no data-path collective."""
    return list(range(rank * per_rank, (rank + 1) * per_rank))


def rank_barrier(world: int) -> None:
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v: float, world: int, dev) -> float:
    """The slowest rank's device time (the only collective of the instance-sharded arms)."""
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_rate(world: int, per_rank: int, steps: int, ms: float) -> float:
    """instances/s of the whole job: every rank's instances over the slowest rank's time."""
    return world * per_rank * steps / (ms * 1e-3)


REF_PER_CORE = 4


def reference_arm(args):
    """The reference algorithm's CPU implementation (the oracle port) on all host cores.

    Each step: every core solves PER_CORE instances of the workload (scene
    generation untimed, as the GPU arms exclude it); the step's time is the
    slowest core's solve time, so value = instances / sum of step times.  Several
    instances per core per step keep the slowest-core term close to the mean."""
    world, rank, _ = dist_setup(args)
    if rank != 0:
        return 0
    if args.config == "c4":
        print(json.dumps({"impl": "reference", "unavailable": "c4 reference arm: ~80 s per "
                          "instance on the host; see DESIGN.md section 6"}), flush=True)
        return 0
    wl = Workload(args.config, args.iters)
    workers = os.cpu_count() or 1
    with _cpu_pool(workers) as pool:
        for _ in range(args.warmup):
            pool.map(_cpu_worker, [(w, workers, 0, wl.name, wl.iters, 1, 20_000_000)
                                   for w in range(workers)])
        n, wall = 0, 0.0
        for st in range(args.steps):
            res = pool.map(_cpu_worker, [(w, workers, 0, wl.name, wl.iters, REF_PER_CORE,
                                          30_000_000 + st * workers * REF_PER_CORE)
                                         for w in range(workers)])
            n += sum(r[0] for r in res)
            wall += max(r[1] for r in res)
    value = n / wall
    line = {
        "impl": "reference", "metric": wl.metric, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": wall / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": wl.config_block(workers * REF_PER_CORE, per_gpu=False),
        "psca_iters_per_s": value * wl.iters,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "port",
                         "sample": f"each step: {workers * REF_PER_CORE} {wl.name} instances "
                                   f"(T={wl.iters}), {REF_PER_CORE} per host core, numpy/OpenBLAS oracle (restatement of the "
                                   "reference; the reference is pure Python and cannot be "
                                   "installed on the box); scene generation excluded, step time "
                                   "= slowest core's solve"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def executed_column_flops(wl, problem, pil_d, emp_d, noi_d, gain_d, m):
    """Executed DMMA flops of the column launches of one solve, exactly.

    Untimed pass with iterate recording.  Per instance-iteration the
    warp-streamed column kernel issues 2 NRB (NRB + 1) DMMAs per 8-column
    block for the two quadratic forms (lower block triangle of P' and A') and,
    for its moving columns (non-zero rebuild weight rho cand g: exactly the
    devices with x_{k+1} != (1 - rho_k) x_k), NBLK DMMAs per pair of listed
    columns in rounds of 16 (psca_wcol.cuh wc_rebuild) -- unless the list has at
    most MOV_CAP = 160 entries on the warp factor path (L <= 40): those increments
    are summed by the instance's factor warp (fac_sweep_w, deferred rebuild) and
    are not column-kernel work.  Returns (flops per column launch, quad share,
    mean moving columns per iteration, share of instance-iterations deferred)."""
    import torch
    from paper_2503_15259_b200 import device, estimators
    cfg = wl.cfg
    nrb = next(r for r in (2, 3, 4, 5, 6, 8, 10, 12, 16, 20) if 4 * r >= cfg.pilot_len)
    nblk = sum((4 * i + 3) // 8 + 1 for i in range(nrb))
    B, N, T = pil_d.shape[0], cfg.n_devices, wl.iters
    kw = estimators.prior_arrays(problem, N, m)
    res = device.solve(cfg.kind, pil_d, emp_d, noi_d, m, wl.steps, gains=gain_d, max_iter=T,
                       record_iterates=True, n_chunks=1, **kw)
    its = res["iterates"]
    n_iter = res["n_iter"].to(torch.int64)
    quad_blk = 2 * nrb * (nrb + 1) * (-(-N // 8))
    defer = nrb <= 10 and B >= device.sm_count() and os.environ.get("PSCA_DEFER_REBUILD") != "0"
    mov_cap = 160
    quad_total, rebuild_total, moving_total, deferred, live_total = 0, 0, 0, 0, 0
    for k in range(T):
        live = n_iter > k
        omr = 1.0 - float(wl.steps[k])
        mv = (its[:, k + 1] != omr * its[:, k]).sum(dim=1).to(torch.int64)
        mv = torch.where(live, mv, torch.zeros_like(mv))
        moving_total += int(mv.sum())
        live_total += int(live.sum())
        if defer:
            deferred += int((live & (mv <= mov_cap)).sum())
            mv = torch.where(mv <= mov_cap, torch.zeros_like(mv), mv)
        full, rest = mv // 16, mv % 16
        rebuild_total += int((nblk * (8 * full + (rest + 1) // 2)).sum())
        quad_total += int(live.sum()) * quad_blk
    del its, res
    torch.cuda.empty_cache()
    flops = DMMA_FLOPS * (quad_total + rebuild_total) / T
    return (flops, quad_total / max(quad_total + rebuild_total, 1), moving_total / (B * T),
            deferred / max(live_total, 1))


def serial_launch_times(run):
    """Mean serialised (single stream, no half-batch split) column and factor launch
    times of one solve, from CUDA events around every launch."""
    from paper_2503_15259_b200 import device
    import torch
    device.set_serial(True)
    try:
        torch.cuda.synchronize()
        device.profile_begin()
        run()
        recs = device.profile_launches()
        device.profile_end()
    finally:
        device.set_serial(False)
    col = [ms for k, ms in recs if k == 0]
    fac = [ms for k, ms in recs if k == 1]
    return (sum(col) / max(len(col), 1), len(col), sum(fac) / max(len(fac), 1), len(fac),
            sum(col), sum(fac))


def ours_arm(args):
    import numpy as np
    import torch
    world, rank, local = dist_setup(args)
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        torch.cuda.set_device(0)
    import __graft_entry__
    __graft_entry__.build()
    from paper_2503_15259_b200 import device, estimators

    wl = Workload(args.config, args.iters, args.batch)
    cfg, problem = wl.cfg, wl.problem
    B, iters = wl.batch, wl.iters
    ids = instance_ids(rank, B)
    devb, host, gen_timing = generate_device(wl.scene_name, ids, os.cpu_count() or 1)
    dev = torch.device("cuda", torch.cuda.current_device())
    pil_h = torch.from_numpy(host["pilots"]).pin_memory()
    emp_h = torch.from_numpy(host["emp_cov"]).pin_memory()
    noi_h = torch.from_numpy(host["noise"]).pin_memory()
    gain_h = torch.from_numpy(host["gains"]).pin_memory() if wl.known else None
    pil_d, emp_d, noi_d = devb["pilots"], devb["emp_cov"], devb["noise"]
    gain_d = devb["gains"] if wl.known else None
    del devb
    m = int(host["n_antennas"])

    def barrier():
        rank_barrier(world)

    def solve(out):
        return estimators.psca_run_batch(problem, pil_d, emp_d, noi_d, m, gains=gain_d,
                                         schedule=wl.schedule, max_iter=iters, out=out)

    out = {}
    for _ in range(max(args.warmup, 3)):
        out = solve(out)
    torch.cuda.synchronize()
    peak = fp64_peak_tflops(torch)

    # ---- device-resident timed region -------------------------------------
    launches = 0
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        e0.record()
        for _ in range(args.steps):
            out = solve(out)
            launches += out["launches"]
        e1.record()
        torch.cuda.synchronize()
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1), world, dev)
    value = whole_job_rate(world, B, args.steps, ms)
    x_check = out["x"]
    finite = bool(torch.isfinite(x_check).all().item())

    # ---- roofline of the dominant kernel (untimed passes) -------------------
    col_ms, n_col, fac_ms, n_fac, col_tot, fac_tot = serial_launch_times(lambda: solve({}))
    algo_launch = 24.0 * cfg.n_devices * cfg.pilot_len ** 2 * B * iters / max(n_col, 1)
    algo_tflops = algo_launch / (col_ms * 1e-3) / 1e12
    executed = None
    if not args.no_executed and out.get("path") != "persistent" and B >= 2 * device.sm_count():
        ex_launch, quad_share, moving, deferred = executed_column_flops(
            wl, problem, pil_d, emp_d, noi_d, gain_d, m)
        executed = {"flops_per_launch": ex_launch, "quad_share": quad_share,
                    "moving_columns_per_iteration": moving, "deferred_share": deferred}
    if executed is not None:
        ach = executed["flops_per_launch"] / (col_ms * 1e-3) / 1e12
        nrb = next(r for r in (2, 3, 4, 5, 6, 8, 10, 12, 16, 20) if 4 * r >= cfg.pilot_len)
        roofline = {
            "bound": "tensor", "kernel": f"column_kernel_w<{nrb}>", "achieved": ach,
            "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
            "flops_per_unit": "EXECUTED FP64 DMMA flops (m8n8k4 = 512 flops): 2 NRB(NRB+1) "
                              "per 8-column block for the quadratic forms + NBLK per pair of "
                              "moving columns for the rebuilds the column CTA does itself "
                              "(lists longer than 160; shorter lists are summed by the factor "
                              "warp and not counted here), counted exactly from an "
                              "iterate-recording pass of the same batch",
            "executed_flops_per_launch": executed["flops_per_launch"],
            "quad_share_of_executed": executed["quad_share"],
            "moving_columns_per_iteration": executed["moving_columns_per_iteration"],
            "rebuild_deferred_share": executed["deferred_share"],
        }
    else:
        roofline = {"bound": "tensor", "kernel": "column_kernel (tile path, chunked instance)",
                    "achieved": algo_tflops, "peak": peak, "unit": "TFLOP/s",
                    "frac": algo_tflops / peak,
                    "flops_per_unit": "algorithmic 24 N L^2 per instance-iteration"}
    roofline.update({
        "traffic": ncu_traffic() if wl.name == "c1" else None,
        "peak_source": "FP64 cuBLAS DGEMM 8192^3 measured live in this run "
                       "(MEASURED_PEAKS.json has no FP64 entry)",
        "timing": "serialised: one solve with every launch on one stream (psca_set_serial), "
                  "CUDA events around each launch; mean column launch time",
        "column_ms_per_launch": col_ms, "factor_ms_per_launch": fac_ms,
        "column_launches": n_col, "factor_launches": n_fac,
        "column_share_serial": col_tot / max(col_tot + fac_tot, 1e-12),
        "algorithmic_flops_per_launch": algo_launch,
        "algorithmic_achieved": algo_tflops, "algorithmic_frac": algo_tflops / peak,
        "algorithmic_note": "24 N L^2 per instance-iteration (SURVEY.md 8(d): the reference's "
                            "three dense ZGEMMs); the kernel executes fewer flops (Hermitian "
                            "lower-triangle forms, incremental rebuild over moving columns), so "
                            "this ratio can exceed 1 and is not a roofline",
        "dmma_pipe_busy_ncu": ncu_pipe() if wl.name == "c1" else None,
        "path": out.get("path"),
    })

    # ---- end to end through the public API from pinned host buffers ----------
    e2e = None
    if not args.no_e2e:
        h2d = pil_h.numel() * 16 + emp_h.numel() * 16 + noi_h.numel() * 8 + \
            (gain_h.numel() * 8 if gain_h is not None else 0)
        d2h = B * cfg.n_devices * 8 + 2 * B * 4

        e2e_out = [None]

        def e2e_step():
            e2e_out[0] = estimators.psca_run_batch_host(problem, pil_h, emp_h, noi_h, m,
                                                        gains=gain_h, schedule=wl.schedule,
                                                        max_iter=iters, out=e2e_out[0])
            return e2e_out[0]

        e2e_step()
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(args.steps):
            r = e2e_step()
        f1.record()
        torch.cuda.synchronize()
        barrier()
        ems = max_over_ranks(f0.elapsed_time(f1), world, dev)
        e2e = {"value": whole_job_rate(world, B, args.steps, ems), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": ems / args.steps,
               "api": "paper_2503_15259_b200.psca_run_batch_host (pinned host in, pinned host "
                      "out; growing chunks of 1, 2, 4 and the remaining waves of instances on "
                      "four rotating compute streams, each chunk's H2D overlapped with the "
                      "previous chunks' solves; result buffers reused across steps)",
               "x_matches_device_run": bool(torch.equal(r["x"], out["x"].cpu()))}

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(wl.name, iters, args.cpu_seconds)
        line = {
            "metric": wl.metric, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic (seeded BASELINE {wl.scene_name} scenes, "
                    "paper_2503_15259_b200/scenes.py)",
            "config": wl.config_block(B, world=world),
            "psca_iters_per_s": value * iters,
            "ms_per_iteration": ms / args.steps / iters,
            "roofline": roofline,
            "generation": gen_timing,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
            "finite": finite,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def c4_arm(args):
    """BASELINE config 4: one huge instance, columns sharded over the ranks."""
    import numpy as np
    import torch
    world, rank, local = dist_setup(args)
    group = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
        group = dist.group.WORLD
    else:
        torch.cuda.set_device(0)
    import __graft_entry__
    __graft_entry__.build()
    from paper_2503_15259_b200 import estimators, large, scenes
    cfg = scenes.BASELINE_CONFIGS["c4"]
    T = args.iters or cfg.n_iter
    sl = large.column_shard(cfg.n_devices, rank, world)
    steps = estimators.default_steps(T)
    # scene: host Philox draws, Y (256 x 2500 x 512 complex GEMM) and Sigma_hat on DMMA
    t0 = time.perf_counter()
    draws = [scenes.draw_scene(cfg, 0)]
    t_draw = time.perf_counter() - t0
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record()
    dv = scenes.make_batch_device(cfg, [0], draws=draws)
    g1.record()
    torch.cuda.synchronize()
    gen_timing = {"host_draws_s": t_draw, "device_cov_ms": g0.elapsed_time(g1)}
    S = dv["pilots"][0][:, sl].contiguous()
    g = dv["gains"][0][sl].contiguous()
    E = dv["emp_cov"][0].contiguous()
    del dv, draws

    def run():
        st = large.GpuLargeStepper("ml-k", S, g, E, 1.0, cfg.n_antennas, steps, max_iter=T)
        return large.ShardedDriver(st, group=group).run(T), st.launches

    for _ in range(max(args.warmup, 1)):
        run()
    torch.cuda.synchronize()
    times = []
    launches = 0
    for _ in range(args.steps):
        if group is not None:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res, nl = run()
        e1.record()
        torch.cuda.synchronize()
        launches += nl
        times.append(max_over_ranks(e0.elapsed_time(e1), world,
                                    torch.device("cuda", torch.cuda.current_device())))
    ms = sum(times) / len(times)
    if rank == 0:
        flops = 24.0 * cfg.n_devices * cfg.pilot_len ** 2 * T
        print(json.dumps({
            "metric": "c4 solve time (one instance, N=100000, L=256, T=50)",
            "value": 1e3 / ms, "unit": "instances/s", "ms_per_step": ms,
            "ms_per_iteration": ms / T, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded BASELINE c4 scene)",
            "config": {"workload": "c4: PSCA-MLE known pathloss, N=100000, L=256, M=512, "
                                   "K=2500, T=50; devices column-sharded, NCCL all-reduce of "
                                   "the Sigma increment per iteration",
                       "parallelism": f"column shards x{world}"},
            "algorithmic_tflops": flops / (ms * 1e-3) / 1e12,
            "algorithmic_note": "24 N L^2 per iteration (SURVEY.md 8(d)) over the device "
                                "time of the whole step loop",
            "generation": gen_timing,
            "gpu_launches": launches, "status": res["status"], "n_iter": res["n_iter"]}),
            flush=True)
    if group is not None:
        torch.distributed.destroy_process_group()
    return 0


def main():
    args = parse_args()
    if args.impl == "reference":
        return reference_arm(args)
    if args.config == "c4":
        return c4_arm(args)
    return ours_arm(args)


if __name__ == "__main__":
    sys.exit(main())
