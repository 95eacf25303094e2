"""Numeric core entry points (mirror of actdet.covlinalg, GPU-backed).

Each function keeps the reference signature and error behaviour and runs the
corresponding sm_100a kernel through the C ABI (include/psca.h):

=====================  ===============================  ======================
reference              here                             C ABI
=====================  ===============================  ======================
cov_unknown  :43-57    cov_unknown                      psca_cov_unknown
cov_known    :60-67    cov_known (delegates, bitwise)   psca_cov_unknown
frobenius_inverse      frobenius_inverse                psca_hpd_inverse
  :91-115
quad_forms   :134-156  quad_forms                       psca_quad_forms
eval_objective         eval_objective                   psca_eval_objective
  :159-172
CovState.build :184-192 CovState.build                  the three above
=====================  ===============================  ======================
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import device
from .sysmodel import DomainError


class ConditioningError(np.linalg.LinAlgError):
    """Numerically singular matrix; carries an estimated condition number (covlinalg.py:31-36)."""

    def __init__(self, message: str, cond_estimate: float):
        super().__init__(f"{message} (estimated condition number {cond_estimate:.3e})")
        self.cond_estimate = cond_estimate


class SingularUpdateError(np.linalg.LinAlgError):
    """Rank-1 inverse update denominator fell below tolerance (covlinalg.py:39-40)."""


def cov_unknown(pilots: np.ndarray, gamma: np.ndarray, noise_power: float,
                pilots_conj: np.ndarray | None = None) -> np.ndarray:
    """S diag(gamma) S^H + sigma^2 I (covlinalg.py:43-57); ``pilots_conj`` is accepted and unused."""
    if noise_power <= 0:
        raise DomainError("noise power must be strictly positive")
    return device.cov_unknown(pilots, np.asarray(gamma, dtype=float), float(noise_power))


def cov_known(pilots: np.ndarray, alpha: np.ndarray, gains: np.ndarray,
              noise_power: float) -> np.ndarray:
    """S diag(alpha g) S^H + sigma^2 I via cov_unknown, so both are bit-identical (:60-67)."""
    return cov_unknown(pilots, alpha * gains, noise_power)


def frobenius_inverse(sigma: np.ndarray) -> np.ndarray:
    """Inverse of a Hermitian PD matrix (covlinalg.py:91-115); exactly Hermitian.

    Raises ConditioningError when a pivot of the factorisation is not positive.
    """
    inv, status, cond, _ = device.hpd_inverse(np.asarray(sigma, dtype=complex))
    if int(status) != 0:
        raise conditioning_error(sigma)
    return inv


def conditioning_error(sigma) -> ConditioningError:
    """The ConditioningError the reference raises for this singular Sigma
    (covlinalg.py:78-88, 104-110): which real SPD factor fails Cholesky --
    Re(Sigma), or A + B A^-1 B -- and the eigenvalue-ratio condition estimate
    of that factor.  Error path only (never on the solve path): it runs after a
    device factorisation has reported a non-positive pivot, on the GPU through
    torch.linalg (cuSOLVER)."""
    torch = device._torch()
    dev = torch.device("cuda", torch.cuda.current_device())
    S = torch.as_tensor(np.asarray(sigma, dtype=complex), device=dev)
    a, b = S.real.contiguous(), S.imag.contiguous()

    def cond(m):
        e = torch.linalg.eigvalsh((m + m.T) / 2.0)
        return float("inf") if float(e[0]) <= 0.0 else float(e[-1] / e[0])

    if not bool(torch.any(b != 0)) or int(torch.linalg.cholesky_ex(a).info) != 0:
        return ConditioningError("Re(Sigma) is numerically singular", cond(a))
    c = a + b @ torch.linalg.solve(a, b)
    return ConditioningError("A + B A^-1 B is numerically singular", cond(c))


def quad_forms(pilots: np.ndarray, sigma_inv: np.ndarray, emp_cov: np.ndarray,
               pilots_conj: np.ndarray | None = None) -> tuple[np.ndarray, np.ndarray]:
    """q_n = s^H P s and r_n = s^H P Sigma_hat P s (covlinalg.py:134-156)."""
    return device.quad_forms(pilots, sigma_inv, emp_cov)


def eval_objective(sigma: np.ndarray, sigma_inv: np.ndarray, emp_cov: np.ndarray) -> float:
    """log|Sigma| + tr(Sigma^-1 Sigma_hat) (covlinalg.py:159-172)."""
    val, status = device.eval_objective(sigma, sigma_inv, emp_cov)
    if int(status) != 0:
        raise DomainError("objective requires a positive definite covariance")
    return float(val)


@dataclass
class CovState:
    """Covariance, its inverse and the quadratic forms at one iterate (covlinalg.py:175-192)."""

    sigma: np.ndarray
    sigma_inv: np.ndarray
    q: np.ndarray
    r: np.ndarray

    @classmethod
    def build(cls, pilots: np.ndarray, weights: np.ndarray, noise_power: float,
              emp_cov: np.ndarray, pilots_conj: np.ndarray | None = None) -> "CovState":
        sigma = cov_unknown(pilots, weights, noise_power)
        sigma_inv = frobenius_inverse(sigma)
        q, r = quad_forms(pilots, sigma_inv, emp_cov)
        return cls(sigma=sigma, sigma_inv=sigma_inv, q=q, r=r)


# the library's own CovState.build; estimators.psca_run(engine="auto") runs the
# components engine when this has been replaced (the reference test seam)
NATIVE_BUILD = CovState.__dict__["build"]
