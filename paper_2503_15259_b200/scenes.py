"""Seeded synthetic scenes for the BASELINE configurations (host-side data prep).

This is not on the hot path: it produces the inputs that the GPU solver and
the CPU oracle both consume.  It restates BASELINE.json's generation recipe
(SURVEY.md section 8(d)), which differs from the reference generator
``actdet.sysmodel.sample_scene`` (sysmodel.py:226-241) in three documented
ways:

* pilots are i.i.d. CN(0,1) and are NOT column-normalised to sqrt(L)
  (the reference rescales them, sysmodel.py:195-199);
* the active set is a uniform random K-subset (BASELINE), not Bernoulli(p);
* H is drawn only for the K active rows (rows of inactive devices are
  multiplied by zero anyway; this keeps config 4 tractable).

The draw order mirrors sample_scene: pilots, distances, active set, H, Z.
Randomness: Philox seeded by SeedSequence([config_id, instance]), as
``make_rng``/``gen_dataset`` do (sysmodel.py:182-186, 267-281).

Pathloss: PL = 128.1 + 37.6 log10(d_km); g = 10^((23 - PL + 99)/10), noise
normalised to sigma^2 = 1.  This equals the reference law
phi(d) = P (4 pi d / lambda)^-eta with tx_power_dbm = -6.1, lambda = 4 pi,
eta = 3.76, d in km on [0.05, 0.5].
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .sysmodel import Sample

D_INNER_KM = 0.05
D_OUTER_KM = 0.5
PATHLOSS_EXP = 3.76
TX_POWER_DBM_EQUIV = 23.0 + 99.0 - 128.1   # = -6.1: folds PL intercept and noise
WAVELENGTH_EQUIV = 4.0 * np.pi             # makes 4 pi d / lambda = d


@dataclass(frozen=True)
class SceneConfig:
    """One BASELINE configuration (BASELINE.json ``configs``)."""

    config_id: int
    kind: str
    n_devices: int
    pilot_len: int
    n_antennas: int
    n_active: int
    n_iter: int
    batch: int
    p: float = 0.05           # activity prior (MAP kinds)
    net_blocks: int = 0       # PSCA-Net depth (config 2)


BASELINE_CONFIGS = {
    "c0": SceneConfig(0, "ml-k", 1000, 40, 64, 50, 100, 1),
    "c1": SceneConfig(1, "ml-ud", 1000, 40, 128, 50, 100, 4096),
    "c2": SceneConfig(2, "map-k", 1000, 40, 128, 50, 100, 4096, net_blocks=10),
    "c3_l20": SceneConfig(3, "map-ur", 2000, 20, 128, 100, 100, 2048),
    "c3_l40": SceneConfig(3, "map-ur", 2000, 40, 128, 100, 100, 2048),
    "c3_l80": SceneConfig(3, "map-ur", 2000, 80, 128, 100, 100, 2048),
    "c4": SceneConfig(4, "ml-k", 100_000, 256, 512, 2500, 50, 1),
}


def gains_from_distance(d_km: np.ndarray) -> np.ndarray:
    """g = 10^((23 - PL + 99)/10), PL = 128.1 + 37.6 log10 d (BASELINE.json)."""
    pl = 128.1 + 37.6 * np.log10(d_km)
    return 10.0 ** ((23.0 - pl + 99.0) / 10.0)


def _cn(rng: np.random.Generator, shape) -> np.ndarray:
    """i.i.d. CN(0,1): real and imaginary parts N(0, 1/2) (sysmodel.py:189-192)."""
    z = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    return z * np.sqrt(0.5)


def draw_scene(cfg: SceneConfig, instance: int, pilot_len: int | None = None) -> dict:
    """The host random draws of instance ``instance`` (the scene contract: one
    Philox stream per instance, draw order pilots, distances, active set, H, Z)."""
    l = cfg.pilot_len if pilot_len is None else pilot_len
    n, m, k = cfg.n_devices, cfg.n_antennas, cfg.n_active
    seed = np.random.SeedSequence([cfg.config_id, l, instance])
    rng = np.random.Generator(np.random.Philox(seed))
    pilots = _cn(rng, (l, n))
    u = rng.random(n)
    d = np.sqrt(D_INNER_KM ** 2 + u * (D_OUTER_KM ** 2 - D_INNER_KM ** 2))
    active = np.sort(rng.choice(n, size=k, replace=False))
    h = _cn(rng, (k, m))
    z = _cn(rng, (l, m))
    return {"pilots": pilots, "gains": gains_from_distance(d), "active": active, "h": h, "z": z}


def make_scene(cfg: SceneConfig, instance: int, pilot_len: int | None = None) -> Sample:
    """Instance ``instance`` of configuration ``cfg`` (deterministic; host arithmetic,
    used by the golden-fixture generator and as the CPU-side reference of
    ``make_batch_device``)."""
    f = draw_scene(cfg, instance, pilot_len)
    pilots, g, active, h, z = f["pilots"], f["gains"], f["active"], f["h"], f["z"]
    n, m = cfg.n_devices, cfg.n_antennas
    alpha = np.zeros(n)
    alpha[active] = 1.0
    y = (pilots[:, active] * np.sqrt(g[active])) @ h + z
    emp = (y @ y.conj().T) / m
    return Sample(pilots=pilots, gains=g, activities=alpha, eff_pathloss=alpha * g,
                  received=y, emp_cov=emp, noise_power=1.0)


def make_batch_device(cfg: SceneConfig, instances, draws=None) -> dict:
    """A batch of instances with the covariances formed on the GPU.

    The random draws stay on the host (``draw_scene``; pass ``draws`` to reuse
    draws made elsewhere, e.g. in worker processes); Y = S_A diag(sqrt(g_A)) H + Z
    and Sigma_hat = Y Y^H / M run on the FP64 tensor pipe (psca_received,
    psca_empirical_cov).  Returns device tensors pilots, gains, emp_cov, noise,
    received and the host activities."""
    import torch
    from . import device
    if draws is None:
        draws = [draw_scene(cfg, int(i)) for i in instances]
    dev = torch.device("cuda", torch.cuda.current_device())
    st = lambda key, dt: torch.from_numpy(np.ascontiguousarray(   # noqa: E731
        np.stack([f[key] for f in draws]).astype(dt))).to(dev)
    S, g, H, Z = (st("pilots", np.complex128), st("gains", np.float64), st("h", np.complex128),
                  st("z", np.complex128))
    A = st("active", np.int32)
    Y = device.received_t(S, A, g, H, Z)
    E = device.empirical_cov_t(Y, cfg.n_antennas)
    act = np.zeros((len(draws), cfg.n_devices))
    for b, f in enumerate(draws):
        act[b, f["active"]] = 1.0
    return {"pilots": S, "gains": g, "emp_cov": E, "received": Y,
            "noise": torch.ones(len(draws), dtype=torch.float64, device=dev),
            "activities": act, "n_antennas": cfg.n_antennas}


def net_steps(n_blocks: int, seed: int = 2) -> np.ndarray:
    """Config-2 PSCA-Net per-layer steps: 1 - U[0,1), i.e. uniform in (0,1]."""
    rng = np.random.Generator(np.random.Philox(np.random.SeedSequence([seed, 10])))
    return 1.0 - rng.random(n_blocks)


def stack_batch(samples) -> dict:
    """Stack samples into contiguous batch arrays (the HBM layout)."""
    return {
        "pilots": np.ascontiguousarray(np.stack([s.pilots for s in samples])),
        "gains": np.ascontiguousarray(np.stack([s.gains for s in samples])),
        "emp_cov": np.ascontiguousarray(np.stack([s.emp_cov for s in samples])),
        "noise": np.array([s.noise_power for s in samples], dtype=float),
        "activities": np.stack([s.activities for s in samples]),
        "n_antennas": samples[0].n_antennas,
    }


def system_config(cfg: SceneConfig, pilot_len: int | None = None):
    """The reference-law SystemConfig equivalent to the BASELINE generator."""
    from .sysmodel import ActivityModel, SystemConfig
    return SystemConfig(n_devices=cfg.n_devices,
                        pilot_len=cfg.pilot_len if pilot_len is None else pilot_len,
                        n_antennas=cfg.n_antennas, noise_power=1.0,
                        tx_power_dbm=TX_POWER_DBM_EQUIV, d_inner=D_INNER_KM, d_outer=D_OUTER_KM,
                        pathloss_exp=PATHLOSS_EXP, wavelength=WAVELENGTH_EQUIV,
                        activity=ActivityModel.iid(cfg.p))


def problem_for(cfg: SceneConfig):
    """Problem (with its prior) of a BASELINE configuration."""
    from .estimators import Problem
    from .priors import EffPathlossPrior, IndependentPrior
    if cfg.kind == "ml-k":
        return Problem.ml_k()
    if cfg.kind == "ml-ud":
        return Problem.ml_ud()
    if cfg.kind == "map-k":
        return Problem.map_k(IndependentPrior(np.full(cfg.n_devices, cfg.p)))
    return Problem.map_ur(EffPathlossPrior.from_config(system_config(cfg)))
