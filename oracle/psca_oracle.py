"""CPU oracle for the PSCA hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this module,
and only as the checker / the timed CPU baseline.  The product package
(``paper_2503_15259_b200``) never imports it: its solver runs on the CUDA
extension or raises.

This is a numpy/scipy restatement of the reference algorithm in
``/root/reference/pkg/src/actdet`` (the upstream is pure Python, so there is
nothing to compile into ``oracle/_ref``).  Every function names the reference
lines it restates.  It uses the same primitive operations as the reference
(an OpenBLAS ZGEMM for the covariance rebuild and the two contractions,
LAPACK ``dpotrf``/``dpotrs`` for the Frobenius inversion) so that it is also a
faithful CPU baseline.

Parity pin: ``tests/golden/make_golden.py`` runs the *reference itself*
(imported from /root/reference in the build container) on seeded cases and
stores inputs + outputs under ``tests/golden/*.npz``; ``tests/test_oracle.py``
checks this restatement against those fixtures (``not gpu`` suite).
"""

from __future__ import annotations

import math

import numpy as np
import scipy.linalg

KINDS = ("ml-k", "map-k", "ml-ud", "map-ur")
DENSITY_FLOOR = 1e-300          # priors.py:32
Q_GUARD = 0.5                   # estimators.py:236


class OracleConditioningError(np.linalg.LinAlgError):
    """Cholesky failure inside the Frobenius inversion (covlinalg.py:31-36)."""

    def __init__(self, what: str, cond: float):
        super().__init__(f"{what} is numerically singular (estimated condition number {cond:.3e})")
        self.cond_estimate = cond


# ---------------------------------------------------------------------------
# Numeric core (covlinalg.py)
# ---------------------------------------------------------------------------

def emp_cov(y: np.ndarray) -> np.ndarray:
    """Sigma_hat = Y Y^H / M  (sysmodel.py:244-248)."""
    return (y @ y.conj().T) / y.shape[1]


def model_cov(pilots: np.ndarray, weights: np.ndarray, noise: float,
              pilots_conj: np.ndarray | None = None) -> np.ndarray:
    """S diag(w) S^H + sigma^2 I as one full ZGEMM (covlinalg.py:43-57)."""
    pc = pilots.conj() if pilots_conj is None else pilots_conj
    out = (pilots * weights) @ pc.T
    idx = np.arange(pilots.shape[0])
    out[idx, idx] += noise
    return out


def _chol_solve(mat: np.ndarray, rhs: np.ndarray, what: str) -> np.ndarray:
    """SPD solve via LAPACK Cholesky (covlinalg.py:78-88)."""
    try:
        fac = scipy.linalg.cho_factor(mat, lower=True, check_finite=False)
    except np.linalg.LinAlgError as exc:
        ev = np.linalg.eigvalsh(0.5 * (mat + mat.T))
        cond = math.inf if ev[0] <= 0 else float(ev[-1] / ev[0])
        raise OracleConditioningError(what, cond) from exc
    return scipy.linalg.cho_solve(fac, rhs, check_finite=False)


def herm_inverse(sigma: np.ndarray) -> np.ndarray:
    """Frobenius inversion of a Hermitian PD matrix (covlinalg.py:91-115).

    Re(S^-1) = (A + B A^-1 B)^-1, Im(S^-1) = -A^-1 B Re(S^-1), with the
    real-only shortcut when B == 0 and the (anti)symmetrisation of the result.
    """
    re = np.ascontiguousarray(sigma.real)
    im = np.ascontiguousarray(sigma.imag)
    eye = np.eye(re.shape[0])
    if not im.any():
        inv = _chol_solve(re, eye, "Re(Sigma)")
        return (0.5 * (inv + inv.T)).astype(complex)
    x = _chol_solve(re, im, "Re(Sigma)")
    schur = re + im @ x
    rinv = _chol_solve(schur, eye, "A + B A^-1 B")
    rinv = 0.5 * (rinv + rinv.T)
    iinv = -x @ rinv
    iinv = 0.5 * (iinv - iinv.T)
    return rinv + 1j * iinv


def quad(pilots: np.ndarray, sigma_inv: np.ndarray, emp: np.ndarray,
         pilots_conj: np.ndarray | None = None):
    """q_n = s^H P s, r_n = s^H P Sh P s via t = P S (covlinalg.py:134-156)."""
    pc = pilots.conj() if pilots_conj is None else pilots_conj
    t = sigma_inv @ pilots
    q = np.einsum("ln,ln->n", pc, t).real.copy()
    r = np.einsum("ln,ln->n", t.conj(), emp @ t).real.copy()
    return q, r


def objective_cov(sigma: np.ndarray, sigma_inv: np.ndarray, emp: np.ndarray) -> float:
    """log|Sigma| + tr(Sigma^-1 Sigma_hat) (covlinalg.py:159-172)."""
    fac = scipy.linalg.cho_factor(sigma, lower=True, check_finite=False)
    logdet = 2.0 * float(np.sum(np.log(np.real(np.diag(fac[0])))))
    return logdet + float(np.real(np.sum(sigma_inv * emp.T)))


# ---------------------------------------------------------------------------
# Priors (priors.py)
# ---------------------------------------------------------------------------

class EffPrior:
    """Parameters of the smoothed effective-pathloss prior (priors.py:173-281).

    Stores the scalars the gradient needs; ``from_law`` recomputes g_low,
    g_high, the Hermite targets and the default dead-zone gradient exactly as
    ``EffPathlossPrior.__post_init__``/``from_config`` do.
    """

    def __init__(self, p, eps, d_inner, d_outer, eta, wavelength, tx_power_dbm,
                 dead_zone_grad=None):
        self.p = np.asarray(p, dtype=float)
        self.eps = float(eps)
        self.d_inner, self.d_outer = float(d_inner), float(d_outer)
        self.eta = float(eta)
        self.wavelength = float(wavelength)
        self.tx_power_dbm = float(tx_power_dbm)
        self.p_lin = 10.0 ** (self.tx_power_dbm / 10.0)
        self.k = 4.0 * np.pi / self.wavelength
        self.g_low = float(self.p_lin * (self.k * np.asarray(self.d_outer)) ** (-self.eta))
        self.g_high = float(self.p_lin * (self.k * np.asarray(self.d_inner)) ** (-self.eta))
        self.dead_zone_grad = 2.0 / self.g_low if dead_zone_grad is None else float(dead_zone_grad)
        self.area2 = self.d_outer ** 2 - self.d_inner ** 2

    @classmethod
    def from_reference(cls, prior) -> "EffPrior":
        """Copy the fields of an actdet/mirror EffPathlossPrior object."""
        return cls(prior.p, prior.eps, prior.d_inner, prior.d_outer, prior.pathloss_exp,
                   prior.wavelength, prior.tx_power_dbm, prior.dead_zone_grad)

    # phi^-1 and derivatives (priors.py:249-263)
    def _inv(self, g):
        return (1.0 / self.k) * (g / self.p_lin) ** (-1.0 / self.eta)

    def _dinv(self, g):
        return -(1.0 / (self.k * self.eta * self.p_lin)) * (g / self.p_lin) ** (-1.0 / self.eta - 1.0)

    def _d2inv(self, g):
        return ((1.0 + self.eta) / (self.k * self.eta ** 2 * self.p_lin ** 2)) * \
            (g / self.p_lin) ** (-1.0 / self.eta - 2.0)

    def pg(self, g):       # priors.py:269-271
        return -2.0 * self._inv(g) * self._dinv(g) / self.area2

    def dpg(self, g):      # priors.py:273-275
        return -2.0 * (self._dinv(g) ** 2 + self._inv(g) * self._d2inv(g)) / self.area2

    def hermite(self):     # priors.py:277-281
        return self.pg(self.g_low), self.dpg(self.g_low)


def smooth_density(gamma: np.ndarray, pr: EffPrior):
    """(density, derivative) of the 4-piece smoothed law (priors.py:313-367)."""
    eps, gl = pr.eps, pr.g_low
    p = pr.p
    cv, cw = pr.hermite()
    in_bump = gamma < eps
    in_bridge = (gamma >= gl - eps) & (gamma < gl)
    in_tail = gamma >= gl
    gb = np.where(in_bump, gamma, 0.0)
    t = np.where(in_bridge, gamma - gl, 0.0)
    u = (t + eps) / eps
    gt = np.where(in_tail, gamma, gl)
    dens = np.zeros_like(gamma)
    dens = np.where(in_bump, (1.0 - p) * (1.0 + 2.0 * gb / eps) * ((gb - eps) / eps) ** 2, dens)
    dens = np.where(in_bridge, p * (cv * (1.0 - 2.0 * t / eps) * u ** 2 + cw * t * u ** 2), dens)
    dens = np.where(in_tail, p * pr.pg(gt), dens)
    der = np.zeros_like(gamma)
    der = np.where(in_bump, 6.0 * (1.0 - p) * gb * (gb - eps) / eps ** 3, der)
    der = np.where(in_bridge, p * (-6.0 * cv * t * (t + eps) / eps ** 3
                                   + cw * (t + eps) * (3.0 * t + eps) / eps ** 2), der)
    der = np.where(in_tail, p * pr.dpg(gt), der)
    return dens, der


def eff_prior_grad(gamma: np.ndarray, pr: EffPrior, m: int) -> np.ndarray:
    """-(1/M) p'/p clipped, dead-zone push (priors.py:377-399)."""
    dens, der = smooth_density(gamma, pr)
    dead = dens <= DENSITY_FLOOR
    safe = np.where(dead, 1.0, dens)
    mag = pr.dead_zone_grad
    grad = -np.clip(der / safe, -mag, mag) / m
    push = np.where(gamma <= pr.g_low / 2.0, 1.0, -1.0) * (mag / m)
    return np.where(dead, push, grad)


def eff_prior_value(gamma: np.ndarray, pr: EffPrior, m: int) -> float:
    """-(1/M) sum log max(p_eps, floor) (priors.py:370-374)."""
    dens, _ = smooth_density(gamma, pr)
    return -float(np.sum(np.log(np.maximum(dens, DENSITY_FLOOR)))) / m


def indep_prior_grad(p: np.ndarray, m: int, n: int) -> np.ndarray:
    """Independent Bernoulli: constant -log(p/(1-p))/M (priors.py:154-158)."""
    lo = np.log(p / (1.0 - p))
    return np.broadcast_to(-lo / m, (n,)).copy()


def indep_prior_value(p: np.ndarray, alpha: np.ndarray, m: int) -> float:
    """-(log_odds . alpha)/M (priors.py:145-149)."""
    return -float(np.log(p / (1.0 - p)) @ alpha) / m


# ---------------------------------------------------------------------------
# Step schedules (estimators.py:66-128)
# ---------------------------------------------------------------------------

def pairwise_prior_grad(c1: np.ndarray, c2, alpha: np.ndarray, m: int) -> np.ndarray:
    """Pairwise MVB gradient -(c1 + c2 alpha)/M (priors.py:154-159); c2 = (indptr,
    indices, data) CSR, each row summed in index order like scipy's csr matvec."""
    indptr, indices, data = c2
    s = np.zeros(alpha.shape[0])
    for n in range(alpha.shape[0]):
        acc = 0.0
        for j in range(indptr[n], indptr[n + 1]):
            acc += data[j] * alpha[indices[j]]
        s[n] = acc
    return -(c1 + s) / m


def pairwise_prior_value(c1: np.ndarray, c2, alpha: np.ndarray, m: int) -> float:
    """-(c1.alpha + alpha.(c2 alpha)/2)/M (priors.py:146-151)."""
    cs = -pairwise_prior_grad(np.zeros_like(c1), c2, alpha, 1)
    return -(float(c1 @ alpha) + 0.5 * float(alpha @ cs)) / m


def default_steps(n: int) -> np.ndarray:
    """rho_0 = 1/2, rho <- rho (1 - rho/2)  (estimators.py:66-83)."""
    out = np.empty(n)
    rho = 0.5
    for i in range(n):
        out[i] = rho
        rho = rho * (1.0 - 0.5 * rho)
    return out


def polynomial_steps(n: int, offset: float = 4.0, exponent: float = 0.8) -> np.ndarray:
    """(1 + k/offset)^-exponent (estimators.py:105-116)."""
    return np.array([(1.0 + k / offset) ** -exponent for k in range(n)])


# ---------------------------------------------------------------------------
# The PSCA loop (estimators.py:176-289)
# ---------------------------------------------------------------------------

def psca(kind: str, pilots: np.ndarray, gains: np.ndarray, emp: np.ndarray, noise: float,
         n_antennas: int, steps: np.ndarray, max_iter: int, tol: float = 0.0,
         indep_p: np.ndarray | None = None, eff: EffPrior | None = None,
         record_objective: bool = False, pairwise=None) -> dict:
    """One PSCA run from x = 0; returns the trace fields of DetectorTrace.

    kind in KINDS; ``steps`` holds rho_k for k < max_iter (explicit schedule).
    Known-pathloss kinds estimate activities in [0,1]; unknown-pathloss kinds
    estimate gamma in [0, inf) (ml-ud) or [0, g_high] (map-ur).
    ``pairwise`` = (c1, (indptr, indices, data)) selects the pairwise MAP-K
    prior instead of ``indep_p``.
    """
    assert kind in KINDS
    n = pilots.shape[1]
    l = pilots.shape[0]
    known = kind in ("ml-k", "map-k")
    hi = 1.0 if known else (np.inf if kind == "ml-ud" else eff.g_high)
    x = np.zeros(n)
    pc = pilots.conj()
    out = {"iterates": [x.copy()], "update_norm": [], "objective": [], "abort": None}
    prior_const = (indep_prior_grad(indep_p, n_antennas, n)
                   if kind == "map-k" and pairwise is None else None)
    for k in range(max_iter):
        w = x * gains if known else x
        sigma = model_cov(pilots, w, noise, pc)
        try:
            p = herm_inverse(sigma)
        except OracleConditioningError as exc:
            out["abort"] = "conditioning: " + str(exc)
            break
        q, r = quad(pilots, p, emp, pc)
        if np.min(q) < Q_GUARD * l / np.linalg.norm(sigma):
            out["abort"] = "quadratic form underflow; inverse inconsistent"
            break
        d = q - r
        if kind == "ml-k":
            grad = gains * d
        elif kind == "map-k":
            pg = prior_const if pairwise is None else pairwise_prior_grad(*pairwise, x, n_antennas)
            grad = gains * d + pg
        elif kind == "ml-ud":
            grad = d
        else:
            grad = d + eff_prior_grad(x, eff, n_antennas)
        coef = (gains * q) ** 2 if known else q ** 2
        cand = np.clip(x - grad / coef, 0.0, hi)
        rho = float(steps[k])
        x_new = (1.0 - rho) * x + rho * cand
        if record_objective:
            val = objective_cov(sigma, p, emp)
            if kind == "map-k" and pairwise is not None:
                val += pairwise_prior_value(*pairwise, x, n_antennas)
            elif kind == "map-k":
                val += indep_prior_value(indep_p, x, n_antennas)
            elif kind == "map-ur":
                val += eff_prior_value(x, eff, n_antennas)
            out["objective"].append(val)
        out["update_norm"].append(float(np.linalg.norm(x_new - x)))
        x = x_new
        out["iterates"].append(x.copy())
        if out["update_norm"][-1] < tol:
            break
    out["final"] = x.copy()
    return out


# ---------------------------------------------------------------------------
# Thresholding (unroll.py:305-352)
# ---------------------------------------------------------------------------

def calibrate(scores, truths) -> float:
    """Error-minimising threshold, ties to the smallest candidate (unroll.py:305-333)."""
    s = np.concatenate([np.ravel(np.asarray(v, dtype=float)) for v in scores])
    t = np.concatenate([np.ravel(np.asarray(v, dtype=float)) for v in truths])
    uniq = np.unique(s)
    mids = (uniq[:-1] + uniq[1:]) / 2.0 if uniq.size > 1 else np.empty(0)
    cands = np.unique(np.concatenate([mids, [0.5]]))
    order = np.argsort(s, kind="stable")
    ss, st = s[order], t[order]
    pref = np.concatenate([[0.0], np.cumsum(st)])
    cut = np.searchsorted(ss, cands, side="left")
    err = (pref[cut] + (s.size - cut) - (pref[-1] - pref[cut])) / s.size
    return float(cands[int(np.argmin(err))])


def decide(scores, theta: float) -> np.ndarray:
    """score >= theta (unroll.py:350-352)."""
    return (np.asarray(scores) >= theta).astype(float)


# ---------------------------------------------------------------------------
# Sensitivity floor (used by the parity tests to set per-instance tolerances)
# ---------------------------------------------------------------------------

def perturbation_floor(kind, pilots, gains, emp, noise, n_antennas, steps, max_iter, tol=0.0,
                       indep_p=None, eff=None, n_trials: int = 3, rel: float = 4e-16,
                       seed: int = 0) -> float:
    """Max relative spread of the final iterate under rounding-size perturbations.

    Re-runs the PSCA loop with the pilots perturbed by a relative 4e-16
    (two ulps) per trial, i.e. by as much as any two valid float64
    evaluation orders differ, and returns max_trials max|x' - x| / max|x|.
    Well-conditioned kinds give ~1e-14; map-ur near the Hermite bridge of
    the prior is locally expanding and gives up to ~1e-5:
    a GPU result cannot be held to a bound tighter than the reference's own.
    """
    base = psca(kind, pilots, gains, emp, noise, n_antennas, steps, max_iter, tol,
                indep_p, eff)["final"]
    rng = np.random.default_rng(seed)
    worst = 0.0
    scale = max(float(np.max(np.abs(base))), 1e-300)
    for _ in range(n_trials):
        pert = pilots * (1.0 + rel * rng.standard_normal(pilots.shape))
        x = psca(kind, pert, gains, emp, noise, n_antennas, steps, max_iter, tol, indep_p,
                 eff)["final"]
        worst = max(worst, float(np.max(np.abs(x - base))) / scale)
    return worst
