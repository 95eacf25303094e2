"""Scene containers and the sample-covariance entry point (mirror of actdet.sysmodel).

Host-side types follow the reference field-for-field (sysmodel.py:28-179) so
that reference ``Sample`` objects and these are interchangeable (duck-typed).
``empirical_cov`` is the reference entry point sysmodel.py:244-248; here it
runs the batched HERK kernel ``psca_herk_emp_cov`` on the GPU.
"""

from __future__ import annotations

from dataclasses import asdict, dataclass, field

import numpy as np


class DomainError(ValueError):
    """Raised when an argument leaves an operation's mathematical domain (sysmodel.py:28-29)."""


@dataclass(frozen=True)
class ActivityModel:
    """Activity law (sysmodel.py:36-71)."""

    variant: str = "iid"
    p: float = 0.05
    group_size: int = 1
    p_group: float = 0.05

    def __post_init__(self):
        if self.variant not in ("iid", "group"):
            raise DomainError(f"unknown activity variant {self.variant!r}")
        prob = self.p if self.variant == "iid" else self.p_group
        if not 0.0 < prob < 1.0:
            raise DomainError("activity probability must lie in (0,1)")
        if self.variant == "group" and self.group_size < 1:
            raise DomainError("group_size must be >= 1")

    @classmethod
    def iid(cls, p: float) -> "ActivityModel":
        return cls(variant="iid", p=p)

    @classmethod
    def group(cls, group_size: int, p_group: float) -> "ActivityModel":
        return cls(variant="group", group_size=group_size, p_group=p_group)

    def marginal_p(self) -> float:
        return self.p if self.variant == "iid" else self.p_group


@dataclass(frozen=True)
class SystemConfig:
    """Scenario scalars (sysmodel.py:74-117); used here to build priors."""

    n_devices: int = 1000
    pilot_len: int = 40
    n_antennas: int = 256
    noise_power: float = 10.0 ** -11.4
    tx_power_dbm: float = 23.0
    d_inner: float = 20.0
    d_outer: float = 200.0
    pathloss_exp: float = 2.5
    wavelength: float = 0.086
    activity: ActivityModel = field(default_factory=ActivityModel)
    seed: int = 0
    freeze_pilots: bool = False

    def __post_init__(self):
        if not self.pilot_len < self.n_devices:
            raise DomainError("pilot_len must be < n_devices (non-orthogonal regime)")
        for name in ("noise_power", "d_inner", "d_outer", "wavelength"):
            if getattr(self, name) <= 0:
                raise DomainError(f"{name} must be strictly positive")
        if not self.d_inner < self.d_outer:
            raise DomainError("d_inner must be < d_outer")

    @property
    def tx_power_mw(self) -> float:
        return 10.0 ** (self.tx_power_dbm / 10.0)

    def replace(self, **kwargs) -> "SystemConfig":
        d = asdict(self)
        d["activity"] = self.activity
        d.update(kwargs)
        return SystemConfig(**d)


@dataclass
class Sample:
    """One realisation (sysmodel.py:153-179).  ``n_antennas`` comes from ``received``."""

    pilots: np.ndarray
    gains: np.ndarray
    activities: np.ndarray
    eff_pathloss: np.ndarray
    received: np.ndarray
    emp_cov: np.ndarray
    noise_power: float

    @property
    def n_devices(self) -> int:
        return self.pilots.shape[1]

    @property
    def pilot_len(self) -> int:
        return self.pilots.shape[0]

    @property
    def n_antennas(self) -> int:
        return self.received.shape[1]


def normalize_noise(sample) -> Sample:
    """Unit-noise reparametrisation (sysmodel.py:251-264)."""
    s2 = sample.noise_power
    return Sample(pilots=sample.pilots, gains=sample.gains / s2,
                  activities=sample.activities, eff_pathloss=sample.eff_pathloss / s2,
                  received=sample.received / np.sqrt(s2), emp_cov=sample.emp_cov / s2,
                  noise_power=1.0)


def empirical_cov(y: np.ndarray, n_antennas: int) -> np.ndarray:
    """(1/M) Y Y^H on the GPU (sysmodel.py:244-248).

    ``y`` is (L, M) or a batch (B, L, M) of complex128; the result has the
    matching (L, L) / (B, L, L) shape.
    """
    if n_antennas < 1:
        raise DomainError("n_antennas must be >= 1")
    from . import device
    return device.empirical_cov(np.asarray(y), int(n_antennas))
