"""Scene containers, seeded scene generation and the sample covariance
(mirror of actdet.sysmodel).

Host-side types follow the reference field-for-field (sysmodel.py:28-179) so
that reference ``Sample`` objects and these are interchangeable (duck-typed).
Scene draws (pilots, distances, activities, H, Z) are host numpy calls in the
reference's order on the same Philox streams (sysmodel.py:182-281), so a
seeded dataset holds the same pilots, gains, activities and received signals
as the reference's; ``empirical_cov`` (sysmodel.py:244-248) and the dataset's
covariances run the batched HERK kernel on the GPU.
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
        if self.activity.variant == "group" and self.n_devices % self.activity.group_size:
            raise DomainError("group_size must divide n_devices")

    @property
    def tx_power_mw(self) -> float:
        return 10.0 ** (self.tx_power_dbm / 10.0)

    def replace(self, **kwargs) -> "SystemConfig":
        d = asdict(self)
        d["activity"] = self.activity
        if isinstance(kwargs.get("activity"), dict):
            kwargs["activity"] = ActivityModel(**kwargs["activity"])
        d.update(kwargs)
        return SystemConfig(**d)


# ---------------------------------------------------------------------------
# pathloss law (sysmodel.py:120-147)
# ---------------------------------------------------------------------------

def _positive_distance(d) -> np.ndarray:
    d = np.asarray(d, dtype=float)
    if np.any(d <= 0):
        raise DomainError("distance must be strictly positive")
    return d


def pathloss_db(d, eta: float, wavelength: float):
    """10 eta log10(4 pi d / lambda) (sysmodel.py:120-125)."""
    return 10.0 * eta * np.log10(4.0 * np.pi * _positive_distance(d) / wavelength)


def raw_pathloss_gain(d, eta: float, wavelength: float):
    """(4 pi d / lambda)^-eta (sysmodel.py:128-133)."""
    return (4.0 * np.pi * _positive_distance(d) / wavelength) ** (-eta)


def pathloss_gain(d, cfg: SystemConfig):
    """Gain with the transmit power folded in (sysmodel.py:136-143)."""
    return cfg.tx_power_mw * raw_pathloss_gain(d, cfg.pathloss_exp, cfg.wavelength)


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


# ---------------------------------------------------------------------------
# seeded draws (sysmodel.py:182-241, 267-281): same generator, same calls,
# same order as the reference, so the streams agree bit for bit
# ---------------------------------------------------------------------------

def make_rng(seed) -> np.random.Generator:
    """Philox generator from an int, an entropy list or a SeedSequence."""
    ss = seed if isinstance(seed, np.random.SeedSequence) else np.random.SeedSequence(seed)
    return np.random.Generator(np.random.Philox(ss))


def _cn(rng: np.random.Generator, shape, scale: float = 1.0) -> np.ndarray:
    """CN(0, scale) entries: independent N(0, scale/2) real and imaginary parts."""
    re = rng.standard_normal(shape)
    im = rng.standard_normal(shape)
    return (re + 1j * im) * np.sqrt(scale / 2.0)


def draw_pilots(rng, pilot_len: int, n_devices: int) -> np.ndarray:
    """Gaussian pilots, every column rescaled to norm sqrt(L)."""
    s = _cn(rng, (pilot_len, n_devices))
    return s * (np.sqrt(pilot_len) / np.linalg.norm(s, axis=0))


def draw_distances(rng, n: int, d_inner: float, d_outer: float) -> np.ndarray:
    """Area-uniform distances in the annulus [d_inner, d_outer]."""
    u = rng.random(n)
    return np.sqrt(d_inner ** 2 + u * (d_outer ** 2 - d_inner ** 2))


def draw_activities(rng, n: int, model: ActivityModel) -> np.ndarray:
    """i.i.d. Bernoulli(p), or whole contiguous groups switched on together."""
    if model.variant == "iid":
        return (rng.random(n) < model.p).astype(float)
    on = rng.random(n // model.group_size) < model.p_group
    return np.repeat(on, model.group_size).astype(float)


def draw_received(rng, pilots: np.ndarray, eff_pathloss: np.ndarray, noise_power: float,
                  n_antennas: int) -> np.ndarray:
    """Y = S diag(gamma)^1/2 H + Z for fresh H, Z (sysmodel.py:210-217, without Sigma_hat)."""
    h = _cn(rng, (pilots.shape[1], n_antennas))
    z = _cn(rng, (pilots.shape[0], n_antennas), scale=noise_power)
    return (pilots * np.sqrt(eff_pathloss)) @ h + z


def _draw_scene(cfg: SystemConfig, rng, pilots=None) -> dict:
    if pilots is None:
        pilots = draw_pilots(rng, cfg.pilot_len, cfg.n_devices)
    d = draw_distances(rng, cfg.n_devices, cfg.d_inner, cfg.d_outer)
    alpha = draw_activities(rng, cfg.n_devices, cfg.activity)
    g = pathloss_gain(d, cfg)
    gamma = alpha * g
    y = draw_received(rng, pilots, gamma, cfg.noise_power, cfg.n_antennas)
    return dict(pilots=pilots, gains=g, activities=alpha, eff_pathloss=gamma, received=y)


def sample_scene(cfg: SystemConfig, rng, pilots=None) -> Sample:
    """One scene; draw order pilots, distances, activities, H, Z (sysmodel.py:220-241)."""
    f = _draw_scene(cfg, rng, pilots)
    return Sample(emp_cov=empirical_cov(f["received"], cfg.n_antennas),
                  noise_power=cfg.noise_power, **f)


def draw_dataset(cfg: SystemConfig, n_samples: int, base_seed) -> list:
    """The host draws of ``gen_dataset`` (dicts without the covariance)."""
    children = np.random.SeedSequence(base_seed).spawn(n_samples + 1)
    pilots = None
    if cfg.freeze_pilots:
        pilots = draw_pilots(make_rng(children[0]), cfg.pilot_len, cfg.n_devices)
    return [_draw_scene(cfg, make_rng(children[i + 1]), pilots) for i in range(n_samples)]


def gen_dataset(cfg: SystemConfig, n_samples: int, base_seed) -> list:
    """Scenes on per-sample Philox streams spawned from SeedSequence(base_seed);
    child 0 is reserved for a frozen pilot matrix (sysmodel.py:267-281).  The
    draws run on the host; all covariances come from one batched GPU HERK."""
    scenes = draw_dataset(cfg, n_samples, base_seed)
    if not scenes:
        return []
    covs = empirical_cov(np.stack([f["received"] for f in scenes]), cfg.n_antennas)
    return [Sample(emp_cov=covs[i], noise_power=cfg.noise_power, **f)
            for i, f in enumerate(scenes)]


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
