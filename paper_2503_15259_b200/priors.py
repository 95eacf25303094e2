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


def known_prior_gradient(prior, n_antennas: int, n: int) -> np.ndarray:
    """Constant MAP-K gradient term -log(p/(1-p))/M (priors.py:154-158).

    Evaluated once on the host with the same operations as the reference, so
    the value the kernel adds is bitwise the reference's.
    """
    if hasattr(prior, "c2"):
        raise NotImplementedError(
            "PairwiseMvbPrior (group activity) is not on the GPU path yet (SURVEY.md 8(f) item 4)")
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
