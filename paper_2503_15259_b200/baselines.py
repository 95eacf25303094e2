"""First-order reference detector on GPU batches (mirror of actdet.baselines.pg_ml).

PG (baselines.py:156-252) is the parallel first-order counterpart of PSCA:
one projected-gradient step per iteration on the covariance-fit objective,
with a fixed step, a Barzilai-Borwein ("spectral") step, or a BB-seeded
Grippo non-monotone backtracking line search.  Here every sample of a batch
runs the reference's per-sample control flow in lock step: the covariance,
its inverse, the quadratic forms and the objective of all samples come from
the batched C-ABI kernels (psca_cov_unknown, psca_hpd_inverse,
psca_quad_forms, psca_eval_objective); each backtracking try evaluates the
objective of the samples that have not accepted yet, in one batched call.
The per-sample scalars (BB step, Grippo reference value, acceptance) are
device-tensor arithmetic between those calls.

BCD (baselines.py:54-150) sweeps the devices in order with exact coordinate
minimisers and Sherman-Morrison updates of Sigma^-1: one CTA per instance
runs a whole sweep in the ``psca_bcd_sweep`` kernel (csrc/psca_bcd.cuh), the
per-sweep trace objective comes from the batched covariance / objective
kernels.
"""

from __future__ import annotations

import ctypes
import time

import numpy as np

from . import device
from .covlinalg import ConditioningError, SingularUpdateError
from .estimators import DetectorTrace, Problem
from .sysmodel import DomainError

SUFF_DEC = 1e-4          # baselines.py:194
MAX_BACKTRACKS = 30      # baselines.py:241


def _stack(samples, torch, dev):
    st = lambda f, dt: torch.from_numpy(np.ascontiguousarray(   # noqa: E731
        np.stack([np.asarray(getattr(s, f)) for s in samples]).astype(dt))).to(dev)
    noise = torch.tensor([float(s.noise_power) for s in samples], dtype=torch.float64, device=dev)
    return st("pilots", np.complex128), st("emp_cov", np.complex128), st("gains", np.float64), noise


def _bb_step(x, grad, prev_x, prev_grad, torch):
    """Shorter BB step s.y / y.y when s.y > 0, else the unit-max-move step; clipped
    to [1e-12, 1e12] (baselines.py:226-239).  Per sample, (B,) tensor."""
    gmax = torch.clamp(grad.abs().amax(dim=1), min=1e-12)
    first = 1.0 / gmax
    if prev_x is None:
        d = first
    else:
        s = x - prev_x
        y = grad - prev_grad
        sy = (s * y).sum(dim=1)
        yy = (y * y).sum(dim=1)
        d = torch.where(sy > 0, sy / yy, first)
    return torch.clamp(d, 1e-12, 1e12)


def pg_ml_batch(samples, known: bool = True, max_iter: int = 30, step_mode: str = "nonmonotone",
                d0: float | None = None, window: int = 10) -> list:
    """``pg_ml`` for a list of same-shape samples; returns one DetectorTrace each."""
    if step_mode not in ("fixed", "nonmonotone", "spectral"):
        raise DomainError(f"unknown step mode {step_mode!r}")
    if step_mode == "fixed" and d0 is None:
        raise DomainError("fixed step mode requires d0")
    problem = Problem.ml_k() if known else Problem.ml_ud()
    torch = device._torch()
    dev = torch.device("cuda", torch.cuda.current_device())
    S, E, G, noise = _stack(samples, torch, dev)
    B, _, N = S.shape
    hi = 1.0 if known else float("inf")
    x = torch.zeros((B, N), dtype=torch.float64, device=dev)
    traces = [DetectorTrace(meta={"kind": problem.kind, "algorithm": "pg", "step_mode": step_mode,
                                  "line_search_failures": 0}) for _ in range(B)]
    iterates = [[np.zeros(N)] for _ in range(B)]
    hist = torch.full((B, window), -float("inf"), dtype=torch.float64, device=dev)
    prev_x = prev_grad = None
    last_safe = torch.full((B,), float("nan"), dtype=torch.float64, device=dev)
    failures = torch.zeros(B, dtype=torch.int64, device=dev)

    def weights(xv, idx=None):
        g = G if idx is None else G[idx]
        return xv * g if known else xv

    def objective(xv, idx):
        """f(x) of the samples idx (baselines.py:142-153), one batched evaluation."""
        sig = device.cov_unknown_t(S[idx], weights(xv, idx).contiguous(), noise[idx])
        inv, status, cond, _ = device.hpd_inverse_t(sig)
        if bool((status != 0).any()):
            raise np.linalg.LinAlgError("covariance is not positive definite")
        val, _ = device.eval_objective_t(sig, inv, E[idx])
        return val

    proj = lambda v: torch.clamp(v, 0.0, hi)   # noqa: E731
    for it in range(max_iter):
        t0 = time.perf_counter()
        sig = device.cov_unknown_t(S, weights(x).contiguous(), noise)
        inv, status, cond, _ = device.hpd_inverse_t(sig)
        if bool((status != 0).any()):
            b = int(torch.nonzero(status != 0)[0, 0])
            raise ConditioningError("Sigma is numerically singular", float(cond[b]))
        q, r = device.quad_forms_t(S, inv, E)
        grad = q - r
        if known:
            grad = G * grad
        f_cur, _ = device.eval_objective_t(sig, inv, E)
        hist[:, it % window] = f_cur

        if step_mode == "fixed":
            d = torch.full((B,), float(d0), dtype=torch.float64, device=dev)
            x_new = proj(x - d[:, None] * grad)
        elif step_mode == "spectral":
            d = _bb_step(x, grad, prev_x, prev_grad, torch)
            x_new = proj(x - d[:, None] * grad)
        else:
            d = _bb_step(x, grad, prev_x, prev_grad, torch)
            d = torch.where(~torch.isnan(last_safe) & ~torch.isfinite(d), last_safe, d)
            f_ref = hist.amax(dim=1)
            x_new = x.clone()
            ok = torch.zeros(B, dtype=torch.bool, device=dev)
            for _ in range(MAX_BACKTRACKS):
                idx = torch.nonzero(~ok).flatten()
                if idx.numel() == 0:
                    break
                trial = proj(x[idx] - d[idx, None] * grad[idx])
                decrease = (grad[idx] * (trial - x[idx])).sum(dim=1)
                acc = objective(trial, idx) <= f_ref[idx] + SUFF_DEC * decrease
                x_new[idx[acc]] = trial[acc]
                ok[idx[acc]] = True
                d[idx[~acc]] = d[idx[~acc]] * 0.5
            bad = ~ok
            if bool(bad.any()):
                failures += bad.to(torch.int64)
                # the last halved step, or the last accepted step when there is one
                d_fail = torch.where(torch.isnan(last_safe), d, last_safe)
                x_new[bad] = proj(x[bad] - d_fail[bad, None] * grad[bad])
            last_safe = torch.where(ok, d, last_safe)
        torch.cuda.synchronize()
        elapsed = (time.perf_counter() - t0) / B
        un = torch.linalg.vector_norm(x_new - x, dim=1).cpu().numpy()
        fc = f_cur.cpu().numpy()
        prev_x, prev_grad = x, grad
        x = x_new
        xh = x.cpu().numpy()
        for b in range(B):
            traces[b].wall_times.append(elapsed)
            traces[b].objective.append(float(fc[b]))
            traces[b].update_norm.append(float(un[b]))
            iterates[b].append(xh[b].copy())
    fails = failures.cpu().numpy()
    xf = x.cpu().numpy()
    for b in range(B):
        traces[b].iterates = iterates[b]
        traces[b].final = xf[b].copy()
        traces[b].meta["line_search_failures"] = int(fails[b])
    return traces


def pg_ml(sample, known: bool = True, max_iter: int = 30, step_mode: str = "nonmonotone",
          d0: float | None = None, window: int = 10) -> DetectorTrace:
    """Projected gradient on one sample (baselines.py:156-223)."""
    return pg_ml_batch([sample], known, max_iter, step_mode, d0, window)[0]


# ---------------------------------------------------------------------------
# block coordinate descent (baselines.py:54-150)
# ---------------------------------------------------------------------------

def _bcd_batch(problem: Problem, samples, max_iter: int) -> list:
    from .estimators import prior_arrays
    torch = device._torch()
    lib = device.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    S, E, G, noise = _stack(samples, torch, dev)
    B, L, N = S.shape
    m = samples[0].received.shape[1]
    known = problem.known_pathloss
    kw = prior_arrays(problem, N, m)
    keep = []

    def put(v, dt):
        if v is None:
            return 0
        t = torch.as_tensor(np.ascontiguousarray(v), device=dev).to(dt)
        keep.append(t)
        return t.data_ptr()

    c2 = kw.get("prior_c2")
    x = torch.zeros((B, N), dtype=torch.float64, device=dev)
    pinv = torch.zeros((B, L, L), dtype=torch.complex128, device=dev)
    status = torch.zeros(B, dtype=torch.int32, device=dev)
    args = device.BcdArgsC(
        kind=device.KIND_CODES[problem.kind], B=B, N=N, L=L, n_antennas=m, init=1,
        pilots=S.data_ptr(), gains=G.data_ptr() if known else 0, emp_cov=E.data_ptr(),
        noise=noise.data_ptr(), prior_lin=put(kw.get("prior_lin"), torch.float64),
        prior_c1=put(kw.get("prior_c1"), torch.float64),
        prior_c2_indptr=put(c2[0], torch.int32) if c2 is not None else 0,
        prior_c2_indices=put(c2[1] if c2[1].size else np.zeros(1, np.int32), torch.int32)
        if c2 is not None else 0,
        prior_c2_data=put(c2[2] if c2[2].size else np.zeros(1), torch.float64)
        if c2 is not None else 0,
        x=x.data_ptr(), sigma_inv=pinv.data_ptr(), status=status.data_ptr())
    traces = [DetectorTrace(meta={"kind": problem.kind, "algorithm": "bcd"}) for _ in range(B)]
    prev = np.zeros((B, N))
    for b in range(B):
        traces[b].iterates.append(prev[b].copy())
    w_gain = G if known else torch.ones_like(G)
    for sweep in range(max_iter):
        t0 = time.perf_counter()
        args.init = 1 if sweep == 0 else 0
        device._check(lib.psca_bcd_sweep(ctypes.byref(args), device._stream(torch)),
                      "psca_bcd_sweep")
        st = status.cpu().numpy()
        if st.any():
            raise SingularUpdateError("rank-1 update denominator below tolerance")
        elapsed = (time.perf_counter() - t0) / B
        sig = device.cov_unknown_t(S, (x * w_gain).contiguous(), noise)
        obj, _ = device.eval_objective_t(sig, pinv, E)
        obj = obj.cpu().numpy()
        xh = x.cpu().numpy()
        if problem.kind == "map-k":
            obj = obj + _known_prior_value(problem.prior, xh, m)
        for b in range(B):
            traces[b].wall_times.append(elapsed)
            traces[b].update_norm.append(float(np.linalg.norm(xh[b] - prev[b])))
            traces[b].objective.append(float(obj[b]))
            traces[b].iterates.append(xh[b].copy())
        prev = xh
    for b in range(B):
        traces[b].final = prev[b].copy()
    return traces


def _known_prior_value(prior, xh, m) -> np.ndarray:
    """Per-sample -(1/M) log p(alpha) (priors.py:146-151)."""
    if hasattr(prior, "c2"):
        c2 = prior.c2
        return np.array([-(float(prior.c1 @ a) + 0.5 * float(a @ (c2 @ a))) / m for a in xh])
    lo = np.log(prior.p / (1.0 - prior.p))
    return np.array([-float(lo @ a) / m for a in xh])


def bcd_ml_batch(samples, known: bool = True, max_iter: int = 5) -> list:
    """Sequential exact coordinate descent on the covariance-fit objective for a
    batch of same-shape samples (baselines.py:54-63); one trace per sample."""
    return _bcd_batch(Problem.ml_k() if known else Problem.ml_ud(), samples, max_iter)


def bcd_map_k_batch(samples, prior, max_iter: int = 5) -> list:
    """Coordinate descent on the known-pathloss MAP objective (baselines.py:66-71)."""
    return _bcd_batch(Problem.map_k(prior), samples, max_iter)


def bcd_ml(sample, known: bool = True, max_iter: int = 5) -> DetectorTrace:
    return bcd_ml_batch([sample], known, max_iter)[0]


def bcd_map_k(sample, prior, max_iter: int = 5) -> DetectorTrace:
    return bcd_map_k_batch([sample], prior, max_iter)[0]
