"""Prior parameter objects for the MAP kinds (mirror of actdet.priors, host side).

Only parameter handling lives here: the per-iteration prior gradient is fused
into the column kernel (csrc/psca.cu ``eff_grad``) and never evaluated on the
CPU.  Field names, defaults and validation follow priors.py:39-281 so that
reference prior objects can be passed to this package unchanged.
"""

from __future__ import annotations

import dataclasses
import math
from dataclasses import dataclass, field

import numpy as np

from .sysmodel import DomainError

DENSITY_FLOOR = 1e-300   # priors.py:32


@dataclass
class IndependentPrior:
    """Independent Bernoulli activities with probabilities p_n (priors.py:39-52)."""

    p: np.ndarray

    def __post_init__(self):
        self.p = np.asarray(self.p, dtype=float)
        if np.any(self.p <= 0.0) or np.any(self.p >= 1.0):
            raise DomainError("activation probabilities must lie strictly in (0,1)")

    @property
    def log_odds(self) -> np.ndarray:
        return np.log(self.p / (1.0 - self.p))


@dataclass
class PairwiseMvbPrior:
    """Order-2 multivariate-Bernoulli prior exp(c1.a + sum_{n<m} c2_nm a_n a_m)/Z
    (priors.py:56-106).  c2 is kept as a symmetric CSR matrix with zero
    diagonal; one given triangle is mirrored.  On the GPU path the MAP-K
    gradient -(c1 + c2 x)/M is evaluated at every iterate by the factor kernel
    (CSR passed through ``psca_solve_args.prior_c2_*``)."""

    c1: np.ndarray
    c2: object

    def __post_init__(self):
        import scipy.sparse as sp
        self.c1 = np.asarray(self.c1, dtype=float)
        c2 = sp.csr_matrix(self.c2)
        c2.setdiag(0.0)
        c2.eliminate_zeros()
        if (c2 != c2.T).nnz:
            upper = sp.triu(c2, k=1)
            c2 = upper + upper.T
        self.c2 = sp.csr_matrix(c2)

    def scaled(self, s: float) -> "PairwiseMvbPrior":
        return PairwiseMvbPrior(self.c1 * s, self.c2 * s)

    @classmethod
    def from_independent(cls, prior: IndependentPrior) -> "PairwiseMvbPrior":
        import scipy.sparse as sp
        n = prior.p.shape[0]
        return cls(prior.log_odds, sp.csr_matrix((n, n)))

    @classmethod
    def from_group_model(cls, n_devices: int, group_size: int, p_group: float,
                         coeff_cap: float = 12.0) -> "PairwiseMvbPrior":
        """Coefficients for contiguous groups of ``group_size`` devices that are
        active together with probability p_group (priors.py:84-106)."""
        import scipy.sparse as sp
        if n_devices % group_size:
            raise DomainError("group_size must divide n_devices")
        a, b = fit_group_coefficients(group_size, p_group, coeff_cap)
        c1 = np.full(n_devices, a)
        if group_size == 1:
            return cls(c1, sp.csr_matrix((n_devices, n_devices)))
        block = b * (np.ones((group_size, group_size)) - np.eye(group_size))
        c2 = sp.block_diag([sp.csr_matrix(block)] * (n_devices // group_size), format="csr")
        return cls(c1, c2)

    def csr_arrays(self):
        """(indptr, indices, data) of c2, int32 / float64, rows in index order."""
        c2 = self.c2.tocsr()
        c2.sort_indices()
        return (c2.indptr.astype(np.int32), c2.indices.astype(np.int32),
                c2.data.astype(np.float64))


class _GroupCountLaw:
    """Exchangeable pairwise model of one group of G devices, reduced to the
    active count k = 0..G: log P(k) = log C(G, k) + a k + b k(k-1)/2 - log Z.
    Its sufficient statistics are (k, pairs(k)); under the true group law
    (every device active with prob. p, all together) their means are G p and
    C(G, 2) p."""

    def __init__(self, g: int, p: float):
        self.count = np.arange(g + 1)
        self.pairs = self.count * (self.count - 1) / 2.0
        lg = math.lgamma
        self.log_mult = np.array([lg(g + 1) - lg(c + 1) - lg(g - c + 1) for c in self.count])
        self.target = (g * p, g * (g - 1) / 2.0 * p)

    def neg_loglik(self, nat):
        """-(E_true[log P]) and its gradient in the natural parameters (a, b)."""
        import scipy.special
        a, b = nat
        z = self.log_mult + a * self.count + b * self.pairs
        log_norm = scipy.special.logsumexp(z)
        prob = np.exp(z - log_norm)
        tk, tp = self.target
        return (-(tk * a + tp * b - log_norm),
                -np.array([tk - float(prob @ self.count), tp - float(prob @ self.pairs)]))


def fit_group_coefficients(group_size: int, p: float, cap: float) -> tuple[float, float]:
    """(a, b) of the pairwise MVB prior for one group (reference
    priors.py:109-139): the maximum-expected-likelihood fit of
    ``_GroupCountLaw`` by box-constrained L-BFGS-B from (logit p, 0), with
    |a| <= cap and |b| <= 2 cap + 8.  A single-device group is independent:
    a = logit p clipped to the cap, b = 0."""
    import scipy.optimize
    logit = math.log(p / (1.0 - p))
    if group_size == 1:
        return float(np.clip(logit, -cap, cap)), 0.0
    law = _GroupCountLaw(group_size, p)
    fit = scipy.optimize.minimize(law.neg_loglik, x0=np.array([logit, 0.0]), jac=True,
                                  method="L-BFGS-B",
                                  bounds=[(-cap, cap), (-2 * cap - 8, 2 * cap + 8)])
    return float(fit.x[0]), float(fit.x[1])


def known_prior_gradient(prior, n_antennas: int, n: int) -> np.ndarray:
    """Constant MAP-K gradient term -log(p/(1-p))/M (priors.py:154-158).

    Evaluated once on the host with the same operations as the reference, so
    the value the kernel adds is bitwise the reference's.
    """
    if hasattr(prior, "c2"):
        raise DomainError("a pairwise prior has an iterate-dependent gradient (prior_c1/prior_c2)")
    log_odds = np.log(prior.p / (1.0 - prior.p))
    return np.broadcast_to(-log_odds / n_antennas, (n,)).copy()


@dataclass
class EffPathlossPrior:
    """Smoothed effective-pathloss prior (priors.py:173-281)."""

    p: np.ndarray
    eps: float
    d_inner: float
    d_outer: float
    pathloss_exp: float
    wavelength: float
    tx_power_dbm: float
    dead_zone_grad: float | None = None
    g_low: float = field(init=False)
    g_high: float = field(init=False)

    def __post_init__(self):
        self.p = np.asarray(self.p, dtype=float)
        if np.any(self.p <= 0.0) or np.any(self.p >= 1.0):
            raise DomainError("activation probabilities must lie strictly in (0,1)")
        if not self.d_inner < self.d_outer or self.d_inner <= 0:
            raise DomainError("need 0 < d_inner < d_outer")
        self.g_low = float(self.phi(self.d_outer))
        self.g_high = float(self.phi(self.d_inner))
        if not 0.0 < 2.0 * self.eps <= self.g_low:
            raise DomainError("need 0 < 2*eps <= g_low so the smoothed pieces don't overlap")
        if self.dead_zone_grad is None:
            self.dead_zone_grad = 2.0 / self.g_low

    @classmethod
    def from_config(cls, cfg, eps_frac: float = 0.1) -> "EffPathlossPrior":
        p = np.full(cfg.n_devices, cfg.activity.marginal_p())
        p_lin = 10.0 ** (cfg.tx_power_dbm / 10.0)
        k = 4.0 * np.pi / cfg.wavelength
        g_low = p_lin * (k * cfg.d_outer) ** (-cfg.pathloss_exp)
        return cls(p=p, eps=eps_frac * g_low, d_inner=cfg.d_inner, d_outer=cfg.d_outer,
                   pathloss_exp=cfg.pathloss_exp, wavelength=cfg.wavelength,
                   tx_power_dbm=cfg.tx_power_dbm)

    def whitened(self, noise_power: float) -> "EffPathlossPrior":
        return dataclasses.replace(self, eps=self.eps / noise_power, dead_zone_grad=None,
                                   tx_power_dbm=self.tx_power_dbm - 10.0 * math.log10(noise_power))

    @property
    def _p_lin(self) -> float:
        return 10.0 ** (self.tx_power_dbm / 10.0)

    @property
    def _k(self) -> float:
        return 4.0 * np.pi / self.wavelength

    def phi(self, d):
        return self._p_lin * (self._k * np.asarray(d, dtype=float)) ** (-self.pathloss_exp)

    def phi_inv(self, g):
        g = np.asarray(g, dtype=float)
        return (1.0 / self._k) * (g / self._p_lin) ** (-1.0 / self.pathloss_exp)

    def dphi_inv(self, g):
        g = np.asarray(g, dtype=float)
        eta = self.pathloss_exp
        return -(1.0 / (self._k * eta * self._p_lin)) * (g / self._p_lin) ** (-1.0 / eta - 1.0)

    def d2phi_inv(self, g):
        g = np.asarray(g, dtype=float)
        eta = self.pathloss_exp
        return ((1.0 + eta) / (self._k * eta ** 2 * self._p_lin ** 2)) * \
            (g / self._p_lin) ** (-1.0 / eta - 2.0)

    def _pg(self, g):
        return -2.0 * self.phi_inv(g) * self.dphi_inv(g) / (self.d_outer ** 2 - self.d_inner ** 2)

    def _dpg(self, g):
        return -2.0 * (self.dphi_inv(g) ** 2 + self.phi_inv(g) * self.d2phi_inv(g)) \
            / (self.d_outer ** 2 - self.d_inner ** 2)

    def _hermite_coeffs(self):
        return float(self._pg(self.g_low)), float(self._dpg(self.g_low))


# ---------------------------------------------------------------------------
# Prior penalty terms at an iterate (priors.py:145-159, 313-399).  Evaluated
# on the GPU by psca_prior_terms -- the same device code the solver runs at
# every iterate -- for numpy or CUDA-tensor inputs (numpy in, numpy out).
# ---------------------------------------------------------------------------

def _device_prior_args(prior, n: int, n_antennas: int) -> tuple[str, dict]:
    if isinstance(prior, EffPathlossPrior) or hasattr(prior, "g_low"):
        p = np.broadcast_to(np.asarray(prior.p, dtype=float), (n,)).copy()
        return "map-ur", {"prior_p": p, "eff_prior": prior}
    if hasattr(prior, "c2"):
        pr = prior if isinstance(prior, PairwiseMvbPrior) else PairwiseMvbPrior(prior.c1, prior.c2)
        return "map-k", {"prior_c1": np.broadcast_to(pr.c1, (n,)).astype(float),
                         "prior_c2": pr.csr_arrays()}
    return "map-k", {"prior_lin": known_prior_gradient(prior, n_antennas, n)}


def _prior_terms(x, prior, n_antennas: int, value=False, density=False):
    import torch
    from . import device
    xt = x if isinstance(x, torch.Tensor) else None
    xa = np.atleast_1d(np.asarray(x, dtype=float)) if xt is None else None
    X = device._dev(device._torch(), xt if xt is not None else xa, torch.float64,
                    torch.device("cuda", torch.cuda.current_device()))
    single = X.dim() == 1
    X2 = X.reshape(1, -1) if single else X
    kind, kw = _device_prior_args(prior, X2.shape[1], n_antennas)
    g, v, d = device.prior_terms_t(kind, X2, n_antennas, want_value=value, want_density=density,
                                   **kw)
    if xt is not None:
        return g, v, d
    cvt = (lambda t: None if t is None else (t[0] if single else t).cpu().numpy())
    return cvt(g), cvt(v), cvt(d)


def _check_range(gamma, prior):
    """gamma in [0, g_high (1 + 1e-12)] or DomainError (priors.py:300-304)."""
    g = np.asarray(gamma, dtype=float) if not hasattr(gamma, "cpu") else gamma.cpu().numpy()
    if np.any(g < 0.0) or np.any(g > prior.g_high * (1.0 + 1e-12)):
        raise DomainError("gamma outside [0, g_high]")


def log_prior_grad_known(alpha, prior, n_antennas: int):
    """-(1/M) d log p(alpha) / d alpha_n (priors.py:154-159), on the device."""
    return _prior_terms(alpha, prior, n_antennas)[0]


def log_prior_value_known(alpha, prior, n_antennas: int) -> float:
    """-(1/M) log p(alpha) up to the normaliser (priors.py:145-151), on the device."""
    return float(_prior_terms(alpha, prior, n_antennas, value=True)[1])


def log_prior_grad_unknown(gamma, prior, n_antennas: int):
    """-(1/M) clip(p'/p) with the dead-zone push (priors.py:377-399), on the device."""
    _check_range(gamma, prior)
    return _prior_terms(gamma, prior, n_antennas)[0]


def log_prior_value_unknown(gamma, prior, n_antennas: int) -> float:
    """-(1/M) sum log max(p^eps(gamma), 1e-300) (priors.py:370-374), on the device."""
    _check_range(gamma, prior)
    return float(_prior_terms(gamma, prior, n_antennas, value=True)[1])


def pdf_eff_smooth(gamma, prior, n: int | None = None):
    """Smoothed effective-pathloss density (priors.py:313-336), on the device."""
    _check_range(gamma, prior)
    g = np.atleast_1d(np.asarray(gamma, dtype=float))
    pr = prior
    if n is not None:
        pr = dataclasses.replace(prior, p=np.full(g.shape[-1], float(np.asarray(prior.p)[n])),
                                 dead_zone_grad=prior.dead_zone_grad)
    out = _prior_terms(g, pr, 1, density=True)[2]
    return float(out[0]) if np.ndim(gamma) == 0 else out
