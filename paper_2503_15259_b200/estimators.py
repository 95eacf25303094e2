"""PSCA engine entry points (mirror of actdet.estimators, GPU-backed).

``psca_run`` keeps the reference signature (estimators.py:239-289) and
returns the same ``DetectorTrace``; the whole iteration loop runs on the GPU
as 1 + 2T kernel launches (csrc/psca.cu: factor_kernel / column_kernel).
``psca_run_batch`` is the throughput entry: B independent instances in one
call, device tensors in and out.
"""

from __future__ import annotations

import json
import time
from dataclasses import dataclass, field

import os

import numpy as np

from . import covlinalg, device, priors
from .sysmodel import DomainError

KINDS = ("ml-k", "map-k", "ml-ud", "map-ur")


@dataclass(frozen=True)
class Problem:
    """Which objective is minimised; MAP kinds carry their prior (estimators.py:30-63)."""

    kind: str
    prior: object | None = None

    def __post_init__(self):
        if self.kind not in KINDS:
            raise DomainError(f"unknown problem kind {self.kind!r}")
        if self.kind in ("map-k", "map-ur") and self.prior is None:
            raise DomainError(f"{self.kind} requires a prior")
        if self.kind in ("ml-k", "ml-ud") and self.prior is not None:
            raise DomainError(f"{self.kind} does not take a prior")

    @classmethod
    def ml_k(cls):
        return cls("ml-k")

    @classmethod
    def map_k(cls, prior):
        return cls("map-k", prior)

    @classmethod
    def ml_ud(cls):
        return cls("ml-ud")

    @classmethod
    def map_ur(cls, prior):
        return cls("map-ur", prior)

    @property
    def known_pathloss(self) -> bool:
        return self.kind in ("ml-k", "map-k")


def default_schedule(k: int) -> float:
    """k-th step of rho <- rho (1 - rho/2), rho_0 = 1/2 (estimators.py:66-73)."""
    if k < 0:
        raise DomainError("iteration index must be >= 0")
    rho = 0.5
    for _ in range(k):
        rho = rho * (1.0 - 0.5 * rho)
    return rho


def default_steps(n: int) -> np.ndarray:
    """First n steps of the default schedule (estimators.py:76-83)."""
    out = np.empty(n)
    rho = 0.5
    for i in range(n):
        out[i] = rho
        rho = rho * (1.0 - 0.5 * rho)
    return out


@dataclass
class StepSchedule:
    """Per-iteration steps: a rule k -> rho or an explicit vector (estimators.py:86-128)."""

    fn: object | None = None
    steps: np.ndarray | None = None

    def __post_init__(self):
        if (self.fn is None) == (self.steps is None):
            raise DomainError("provide exactly one of fn or steps")
        if self.steps is not None:
            self.steps = np.asarray(self.steps, dtype=float)
            if np.any(self.steps <= 0.0) or np.any(self.steps > 1.0):
                raise DomainError("every step must lie in (0,1]")

    @classmethod
    def default(cls) -> "StepSchedule":
        return cls(fn=default_schedule)

    @classmethod
    def polynomial(cls, offset: float = 4.0, exponent: float = 0.8) -> "StepSchedule":
        if not 0.5 < exponent <= 1.0:
            raise DomainError("exponent must lie in (0.5, 1] for admissibility")
        return cls(fn=lambda k: (1.0 + k / offset) ** -exponent)

    @classmethod
    def explicit(cls, steps) -> "StepSchedule":
        return cls(steps=steps)

    def __call__(self, k: int) -> float:
        if self.steps is not None:
            return float(self.steps[k])
        rho = float(self.fn(k))
        if not 0.0 < rho <= 1.0:
            raise DomainError(f"schedule produced step {rho} outside (0,1]")
        return rho

    def materialize(self, n: int) -> np.ndarray:
        """rho_0..rho_{n-1} as the device step vector.

        The default rule uses the recursion directly (bitwise the values
        ``default_schedule(k)`` returns); other rules are evaluated eagerly, so
        an invalid step anywhere in the first n raises up front.
        """
        if self.steps is not None:
            return np.asarray(self.steps[:n], dtype=float)
        if self.fn is default_schedule:
            return default_steps(n)
        return np.array([self(k) for k in range(n)], dtype=float)


@dataclass
class DetectorTrace:
    """Per-iteration record of one run (estimators.py:131-164).

    wall_times: device time of each iteration's kernels (the factorisation
    that opens it plus its column pass), from CUDA events recorded around
    every launch of the solve (psca_profile_launches).
    """

    iterates: list = field(default_factory=list)
    objective: list = field(default_factory=list)
    update_norm: list = field(default_factory=list)
    wall_times: list = field(default_factory=list)
    final: np.ndarray | None = None
    meta: dict = field(default_factory=dict)

    @property
    def n_iterations(self) -> int:
        return len(self.update_norm)

    def dump_jsonl(self, path, method: str = ""):
        with open(path, "a", encoding="utf-8") as fh:
            for k in range(self.n_iterations):
                rec = {
                    "method": method or self.meta.get("method", ""),
                    "iteration": k + 1,
                    "update_norm": self.update_norm[k],
                    "objective": self.objective[k] if k < len(self.objective) else None,
                    "wall_time_s": self.wall_times[k],
                }
                fh.write(json.dumps(rec) + "\n")


def bounds_for(problem, sample=None) -> tuple[float, float]:
    """Coordinate box (estimators.py:167-173)."""
    if problem.kind in ("ml-k", "map-k"):
        return 0.0, 1.0
    if problem.kind == "ml-ud":
        return 0.0, np.inf
    return 0.0, problem.prior.g_high


def prior_arrays(problem, n_devices: int, n_antennas: int) -> dict:
    """Device-side prior inputs for ``device.solve`` from a Problem."""
    if problem.kind == "map-k":
        if hasattr(problem.prior, "c2"):   # pairwise MVB (priors.py:56-106)
            pr = problem.prior
            if not isinstance(pr, priors.PairwiseMvbPrior):
                pr = priors.PairwiseMvbPrior(pr.c1, pr.c2)
            return {"prior_c1": np.broadcast_to(pr.c1, (n_devices,)).astype(float),
                    "prior_c2": pr.csr_arrays()}
        return {"prior_lin": priors.known_prior_gradient(problem.prior, n_antennas, n_devices)}
    if problem.kind == "map-ur":
        p = np.broadcast_to(np.asarray(problem.prior.p, dtype=float), (n_devices,)).copy()
        return {"prior_p": p, "eff_prior": problem.prior}
    return {}


def _iteration_times(launch_times, k_done: int, fallback: float) -> list:
    """Per-iteration device seconds from the solve's launch record: iteration k =
    the factor launch that opens it + its column launch (launch order: factor 0,
    then column k, factor k+1 for every k)."""
    if launch_times and len(launch_times) >= 2 * k_done + 1 and launch_times[0][0] == 1:
        out = []
        for k in range(k_done):
            (kf, tf), (kc, tc) = launch_times[2 * k], launch_times[2 * k + 1]
            if kf != 1 or kc != 0:
                return [fallback] * k_done
            out.append((tf + tc) * 1e-3)
        return out
    return [fallback] * k_done


def _conditioning_message(problem, sample, x, cond) -> str:
    """The reference's abort text for a failed factorisation at iterate x
    (covlinalg.py:78-88 via estimators.py:263-266)."""
    try:
        import torch
        xt = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x))
        w = xt.cpu().numpy() * (np.asarray(sample.gains) if problem.known_pathloss else 1.0)
        sigma = covlinalg.cov_unknown(sample.pilots, w, sample.noise_power)
        return str(covlinalg.conditioning_error(sigma))
    except Exception:   # pragma: no cover - message only
        return str(covlinalg.ConditioningError("Re(Sigma) is numerically singular",
                                               float(cond)))


def _components_engine(engine: str) -> bool:
    if engine not in ("auto", "fused", "components"):
        raise DomainError(f"unknown engine {engine!r}")
    if engine == "auto":
        return covlinalg.CovState.__dict__.get("build") is not covlinalg.NATIVE_BUILD
    return engine == "components"


def _psca_run_components(problem, sample, steps, n_steps, tol, record_objective, trace,
                         max_iter, schedule):
    """The reference loop (estimators.py:239-289) over the component entry points."""
    import torch
    n = sample.n_devices
    x = np.zeros(n)
    lo, hi = bounds_for(problem, sample)
    pilots_conj = np.asarray(sample.pilots).conj()
    trace.iterates.append(x.copy())
    for k in range(n_steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        try:
            state = build_state(problem, x, sample, pilots_conj)
        except covlinalg.ConditioningError as exc:
            trace.meta["abort"] = str(exc)
            trace.final = x.copy()
            return trace
        step = _coord_step(problem, x, state, sample, float(steps[k]), hi, guard=True)
        e1.record()
        if int(step["status"][0].item()) == device.STATUS_QFLOOR:
            trace.meta["abort"] = ABORT_QFLOOR
            trace.final = x.copy()
            return trace
        x_new = step["x_new"][0].cpu().numpy()
        if record_objective:
            trace.objective.append(objective_value(problem, x, sample, state))
        torch.cuda.synchronize()
        trace.wall_times.append(e0.elapsed_time(e1) * 1e-3)
        trace.update_norm.append(float(step["update_norm"][0].item()))
        x = x_new
        trace.iterates.append(x.copy())
        if trace.update_norm[-1] < tol:
            break
    if schedule.steps is not None and len(schedule.steps) < max_iter and \
            trace.n_iterations == n_steps:
        raise IndexError("explicit schedule shorter than max_iter")
    trace.final = x.copy()
    return trace


def _prior_kwargs(problem, n: int, n_antennas: int) -> dict:
    kind, kw = priors._device_prior_args(problem.prior, n, n_antennas)
    return kw


def _coord_step(problem, x, state, sample, rho: float, hi: float, guard: bool = False):
    """psca_coord_step at x from a CovState (device); returns device tensors."""
    torch = device._torch()
    dev = torch.device("cuda", torch.cuda.current_device())
    as_d = (lambda a: torch.as_tensor(np.ascontiguousarray(a), device=dev).reshape(1, -1))  # noqa: E731
    n = x.shape[-1]
    X, Q, R = as_d(np.asarray(x, float)), as_d(state.q), as_d(state.r)
    g = as_d(np.asarray(sample.gains, float)) if problem.known_pathloss else None
    pg = None
    if problem.kind in ("map-k", "map-ur"):
        if problem.kind == "map-ur":
            priors._check_range(x, problem.prior)
        pg, _, _ = device.prior_terms_t(problem.kind, X, sample.n_antennas,
                                        **_prior_kwargs(problem, n, sample.n_antennas))
    sig = (torch.as_tensor(np.ascontiguousarray(state.sigma), device=dev)[None]
           if guard else None)
    return device.coord_step_t(problem.kind, X, Q, R, rho,
                               hi if np.isfinite(hi) else np.finfo(float).max,
                               gains=g, prior_grad=pg, sigma=sig)


def gradient(problem, x, state, gains, n_antennas: int) -> np.ndarray:
    """Objective gradient at x from the covariance state built there (estimators.py:176-186):
    g (q - r) [known] or q - r [unknown] plus the prior term, on the device."""
    from types import SimpleNamespace
    smp = SimpleNamespace(gains=gains, n_antennas=n_antennas)
    out = _coord_step(problem, np.asarray(x, float), state, smp, 1.0, np.finfo(float).max)
    return out["grad"][0].cpu().numpy()


def objective_value(problem, x, sample, state) -> float:
    """Covariance fit plus the prior penalty (estimators.py:203-211), on the device."""
    val = covlinalg.eval_objective(state.sigma, state.sigma_inv, sample.emp_cov)
    if problem.kind == "map-k":
        val += priors.log_prior_value_known(x, problem.prior, sample.n_antennas)
    elif problem.kind == "map-ur":
        val += priors.log_prior_value_unknown(x, problem.prior, sample.n_antennas)
    return val


def _cov_weights(problem, x, gains) -> np.ndarray:
    """x g (known pathloss) or x (estimators.py:214-215)."""
    return x * gains if problem.known_pathloss else x


def build_state(problem, x, sample, pilots_conj=None):
    """CovState at x (estimators.py:218-222): Sigma, Sigma^-1, q, r on the GPU."""
    weights = _cov_weights(problem, np.asarray(x, float), sample.gains)
    return covlinalg.CovState.build(sample.pilots, weights, sample.noise_power, sample.emp_cov,
                                    pilots_conj)


def stationarity_residual(problem, x, sample) -> float:
    """||x - clip(x - grad, lo, hi)||_inf, the projected-gradient residual (estimators.py:225-230)."""
    state = build_state(problem, x, sample)
    grad = gradient(problem, x, state, sample.gains, sample.n_antennas)
    lo, hi = bounds_for(problem, sample)
    return float(np.max(np.abs(x - np.clip(x - grad, lo, hi))))


ABORT_COND = "Sigma is numerically singular (estimated condition number {:.3e})"
# The compiled / generic batched kernels cover L <= 128; larger pilot lengths
# (BASELINE config 4: L = 256) run the GEMM-tiled step loop of large.py.
MAX_L_BATCHED = 128


ABORT_QFLOOR = "quadratic form underflow; inverse inconsistent"


def use_large_path(pilot_len: int) -> bool:
    import os
    return pilot_len > MAX_L_BATCHED or os.environ.get("PSCA_FORCE_LARGE") == "1"


def psca_run(problem, sample, schedule: StepSchedule | None = None, max_iter: int = 30,
             tol: float = 1e-4, record_objective: bool = True, *, engine: str = "auto",
             fault_iter: int = 0) -> DetectorTrace:
    """Run the PSCA iteration from the all-zero start on the GPU (estimators.py:239-289).

    Same stopping rules and trace contents as the reference: stops at
    max_iter or when the update norm drops below tol; a singular covariance
    or a q-floor violation ends the run with ``meta["abort"]`` set and
    ``final`` = the last accepted iterate.

    engine: "fused" -- the whole loop in one device call (psca_solve, the
    product path); "components" -- the reference's loop structure, one
    ``build_state`` (cov_unknown, frobenius_inverse, quad_forms on the GPU) and
    one ``psca_coord_step`` per iteration; "auto" (default) -- fused, unless
    ``covlinalg.CovState.build`` has been replaced (the reference test seam
    test_estimators.py:268-279 monkeypatches it to inject a failure), in which
    case the components engine runs so the replacement takes effect.
    fault_iter: k >= 1 forces the factorisation opening iteration k-1 to fail
    on the fused engine (psca_solve_args.fault_iter; a device-side test seam).
    """
    import torch

    if schedule is None:
        schedule = StepSchedule.default()
    n = sample.n_devices
    trace = DetectorTrace(meta={"kind": problem.kind, "tol": tol})
    if problem.kind == "map-ur":
        trace.meta["dead_zone_grad"] = problem.prior.dead_zone_grad
    n_steps = max_iter
    if schedule.steps is not None and len(schedule.steps) < max_iter:
        n_steps = len(schedule.steps)    # the reference would IndexError at k = len(steps)
    steps = schedule.materialize(n_steps)
    m = sample.n_antennas
    if _components_engine(engine):
        return _psca_run_components(problem, sample, steps, n_steps, tol, record_objective,
                                    trace, max_iter, schedule)
    kw = prior_arrays(problem, n, m)
    t0 = torch.cuda.Event(enable_timing=True) if torch.cuda.is_available() else None
    t1 = torch.cuda.Event(enable_timing=True) if torch.cuda.is_available() else None
    if t0 is not None:
        t0.record()
    gains = np.asarray(sample.gains, dtype=float) if problem.known_pathloss else None
    launch_times = None
    if use_large_path(sample.pilot_len):
        from .large import psca_run_large
        r = psca_run_large(problem.kind, np.asarray(sample.pilots), gains,
                           np.asarray(sample.emp_cov), sample.noise_power, m, steps,
                           max_iter=n_steps, tol=tol, record_objective=record_objective,
                           record_iterates=True, **kw)
        status, k_done = r["status"], r["n_iter"]
        its_t, un_t, obj_t, x_t, cond = (r["iterates"], r["update_norm"], r["objective"],
                                         r["x"], r["cond_est"])
    else:
        device.profile_begin()
        try:
            res = device.solve(problem.kind, np.asarray(sample.pilots)[None],
                               np.asarray(sample.emp_cov)[None],
                               np.array([sample.noise_power], float), m, steps,
                               gains=gains[None] if gains is not None else None,
                               max_iter=n_steps, tol=tol, record_objective=record_objective,
                               record_iterates=True, fault_iter=fault_iter, **kw)
            launch_times = device.profile_launches()
        finally:
            device.profile_end()
        status = int(res["status"][0].item())
        k_done = int(res["n_iter"][0].item())
        its_t, un_t = res["iterates"][0, :k_done + 1], res["update_norm"][0, :k_done]
        obj_t = res["objective"][0, :k_done] if record_objective else None
        x_t, cond = res["x"][0], float(res["cond_est"][0].item())
    if t1 is not None:
        t1.record()
    its = its_t.cpu().numpy()
    trace.iterates = [its[i].copy() for i in range(k_done + 1)]
    trace.update_norm = [float(v) for v in un_t.cpu().numpy()]
    if record_objective:
        trace.objective = [float(v) for v in obj_t.cpu().numpy()]
    torch.cuda.synchronize()
    per = (t0.elapsed_time(t1) * 1e-3 / max(k_done, 1)) if t0 is not None else 0.0
    trace.wall_times = _iteration_times(launch_times, k_done, per)
    if status == device.STATUS_CHOL_FAIL:
        trace.meta["abort"] = _conditioning_message(problem, sample, x_t, cond)
    elif status == device.STATUS_QFLOOR:
        trace.meta["abort"] = ABORT_QFLOOR
    trace.final = x_t.cpu().numpy().copy()
    if (status in (device.STATUS_RUNNING,) and schedule.steps is not None
            and len(schedule.steps) < max_iter):
        raise IndexError("explicit schedule shorter than max_iter")
    return trace


def psca_run_batch(problem, pilots, emp_cov, noise, n_antennas: int, gains=None,
                   schedule: StepSchedule | None = None, max_iter: int = 30, tol: float = 0.0,
                   record_objective: bool = False, n_chunks: int = 0, out=None) -> dict:
    """B independent PSCA runs in one device call.

    pilots (B,L,N), emp_cov (B,L,L), noise (B,), gains (B,N); numpy arrays
    or CUDA tensors.  Returns device tensors (see ``device.solve``).
    """
    if schedule is None:
        schedule = StepSchedule.default()
    steps = schedule.materialize(max_iter)
    n = pilots.shape[-1]
    kw = prior_arrays(problem, n, n_antennas)
    if problem.known_pathloss and gains is None:
        raise DomainError("known-pathloss problems need the gains")
    if use_large_path(pilots.shape[-2]):
        return _batch_via_large(problem, pilots, emp_cov, noise, n_antennas, gains, steps,
                                max_iter, tol, record_objective, kw)
    return device.solve(problem.kind, pilots, emp_cov, noise, n_antennas, steps,
                        gains=gains if problem.known_pathloss else None, max_iter=max_iter,
                        tol=tol, record_objective=record_objective, n_chunks=n_chunks, out=out,
                        **kw)


_COPY_STREAMS = {}


def _host_chunk_bounds(B: int, chunks: int) -> list:
    if chunks <= 0:
        wave = 2 * device.sm_count()           # column CTAs resident at once
        if B >= 8 * wave:
            return [0, wave, 3 * wave, 7 * wave, B]
        chunks = 4 if B >= 4 * wave else (2 if B >= 2 * wave else 1)
    chunks = max(1, min(chunks, B))
    return [(B * c) // chunks for c in range(chunks + 1)]


def psca_run_batch_host(problem, pilots, emp_cov, noise, n_antennas: int, gains=None,
                        schedule: StepSchedule | None = None, max_iter: int = 30,
                        tol: float = 0.0, chunks: int = 0, out: dict | None = None) -> dict:
    """B independent PSCA runs from HOST arrays, with H2D / compute / D2H overlap.

    pilots (B,L,N) complex128, emp_cov (B,L,L), noise (B,), gains (B,N): numpy
    arrays or CPU tensors (pinned memory for full copy/compute overlap).  The
    batch is cut into sub-batches; the host-to-device copy of chunk c+1 runs
    on a copy stream while chunk c is solved on the current stream, and each
    chunk's estimates are copied back as soon as it is solved.  ``chunks`` = 0
    picks growing chunks: one wave of column CTAs first (its upload is the only
    copy not hidden), then two and four waves (each uploaded while the previous
    chunk solves, with margin for a slower host link), then the rest
    (tools/e2e_sweep.py compares schedules); ``chunks`` > 0 cuts equal chunks.
    Returns host tensors x (B,N), status (B,), n_iter (B,).  ``out`` = the dict a
    previous call of the same shape returned: its (pinned) result tensors are
    written again instead of allocating new ones (a pinned allocation per call
    costs milliseconds).
    """
    import torch
    if schedule is None:
        schedule = StepSchedule.default()
    dev = torch.device("cuda", torch.cuda.current_device())
    as_t = lambda a: a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))  # noqa: E731
    S, E, nz = as_t(pilots), as_t(emp_cov), as_t(np.asarray(noise, dtype=float))
    G = as_t(gains) if (gains is not None and problem.known_pathloss) else None
    B, L, N = S.shape
    bounds = _host_chunk_bounds(B, chunks)
    chunks = len(bounds) - 1
    user = torch.cuda.current_stream()
    copy = _COPY_STREAMS.setdefault(dev.index, torch.cuda.Stream(device=dev))
    # consecutive chunks solve on rotating streams (4: c1 e2e 242.8 ms with two,
    # 239.7 with three, 238.1 with four), so the next chunks' launches fill the
    # SMs while the previous chunks are in their latency-bound stages
    ns = max(2, int(os.environ.get("PSCA_HOST_STREAMS", "4")))
    alts = [_COPY_STREAMS.setdefault(("alt", i, dev.index), torch.cuda.Stream(device=dev))
            for i in range(1, ns)]
    start = torch.cuda.Event()
    start.record(user)
    for alt in alts:
        alt.wait_event(start)
    copy.wait_event(start)
    comps = [user] + alts
    pin = S.is_pinned()
    if (out is not None and tuple(out["x"].shape) == (B, N) and out["x"].is_pinned() == pin
            and out["status"].numel() == B and out["n_iter"].numel() == B):
        x_h, st_h, ni_h = out["x"], out["status"], out["n_iter"]
    else:
        x_h = torch.empty((B, N), dtype=torch.float64, pin_memory=pin)
        st_h = torch.empty(B, dtype=torch.int32, pin_memory=pin)
        ni_h = torch.empty(B, dtype=torch.int32, pin_memory=pin)
    bufs = [None] * ns
    free = [torch.cuda.Event() for _ in range(ns)]
    outs = [{} for _ in range(ns)]
    for c in range(chunks):
        lo, hi = bounds[c], bounds[c + 1]
        k = c % ns
        comp = comps[k]
        with torch.cuda.stream(copy):
            if c >= ns:
                copy.wait_event(free[k])           # chunk c-ns finished with this buffer
            bufs[k] = [t[lo:hi].to(dev, non_blocking=True) if t is not None else None
                       for t in (S, E, nz, G)]
            copied = torch.cuda.Event()
            copied.record(copy)
        comp.wait_event(copied)
        Sd, Ed, nd, gd = bufs[k]
        for t in (Sd, Ed, nd, gd):
            if t is not None:
                t.record_stream(comp)
        # one column chunk per instance once a chunk fills a wave, so results do
        # not depend on how the batch was cut
        nck = 1 if hi - lo >= 2 * device.sm_count() else 0
        with torch.cuda.stream(comp):
            res = psca_run_batch(problem, Sd, Ed, nd, n_antennas, gains=gd, schedule=schedule,
                                 max_iter=max_iter, tol=tol, n_chunks=nck, out=outs[k])
            outs[k] = {"x": res["x"], "_ws": res.get("_ws"), "_bufs": res.get("_bufs")}
            x_h[lo:hi].copy_(res["x"], non_blocking=True)
            st_h[lo:hi].copy_(res["status"], non_blocking=True)
            ni_h[lo:hi].copy_(res["n_iter"], non_blocking=True)
        free[k].record(comp)
    for alt in alts:
        done = torch.cuda.Event()
        done.record(alt)
        user.wait_event(done)
    user.synchronize()
    return {"x": x_h, "status": st_h, "n_iter": ni_h}


def _batch_via_large(problem, pilots, emp_cov, noise, n_antennas, gains, steps, max_iter, tol,
                     record_objective, kw):
    """Large-L batches: one step-loop solve per instance (device tensors out)."""
    import torch
    from .large import psca_run_large
    B = pilots.shape[0]
    outs = []
    for b in range(B):
        g = gains[b] if gains is not None else None
        outs.append(psca_run_large(problem.kind, pilots[b], g, emp_cov[b], float(noise[b]),
                                   n_antennas, steps, max_iter=max_iter, tol=tol,
                                   record_objective=record_objective, **kw))
    dev = outs[0]["x"].device
    un = torch.zeros((B, max_iter), dtype=torch.float64, device=dev)
    for b, o in enumerate(outs):
        un[b, :o["n_iter"]] = o["update_norm"]
    return {"x": torch.stack([o["x"] for o in outs]), "update_norm": un,
            "objective": None, "iterates": None,
            "status": torch.tensor([o["status"] for o in outs], dtype=torch.int32, device=dev),
            "n_iter": torch.tensor([o["n_iter"] for o in outs], dtype=torch.int32, device=dev),
            "cond_est": torch.tensor([o["cond_est"] for o in outs], dtype=torch.float64, device=dev),
            "launches": sum(o["launches"] for o in outs), "path": "large"}


# -- elementwise helpers kept for API parity (estimators.py:176-200); the
#    solver never calls them: the same arithmetic is fused in column_kernel.

def surrogate_coef(problem, state, gains):
    if problem.known_pathloss:
        return (gains * state.q) ** 2
    return state.q ** 2


def coord_solution(x, grad, coef, lo, hi):
    return np.clip(x - grad / coef, lo, hi)
