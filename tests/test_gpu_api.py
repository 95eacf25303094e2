"""The standalone estimator / prior API on the GPU (reference estimators.py:176-230,
priors.py:145-159, 313-399, covlinalg.py:78-115) and the two test seams.

These follow the reference's own tests of the same functions
(tests/test_estimators.py TestGradient, TestStationarity,
test_abort_on_inversion_failure; tests/test_priors.py unknown-prior grid),
pointed at this package; the prior grid is compared with the reference's
outputs stored in golden_components.npz.
"""

import numpy as np
import pytest

from psca_testutil import max_rel

pytestmark = pytest.mark.gpu


def _cfg(n=40, l=8, m=32, p=0.1):
    from paper_2503_15259_b200 import sysmodel
    return sysmodel.SystemConfig(n_devices=n, pilot_len=l, n_antennas=m, noise_power=1.0,
                                 tx_power_dbm=0.0, d_inner=1.0, d_outer=2.0, pathloss_exp=2.5,
                                 wavelength=4.0 * np.pi, activity=sysmodel.ActivityModel.iid(p))


def _sample(seed, **kw):
    from paper_2503_15259_b200 import sysmodel
    cfg = _cfg(**kw)
    return cfg, sysmodel.gen_dataset(cfg, 1, seed)[0]


def _problems(cfg):
    from paper_2503_15259_b200 import Problem
    from paper_2503_15259_b200.priors import EffPathlossPrior, IndependentPrior
    return {"ml-k": Problem.ml_k(),
            "map-k": Problem.map_k(IndependentPrior(np.full(cfg.n_devices,
                                                            cfg.activity.marginal_p()))),
            "ml-ud": Problem.ml_ud(),
            "map-ur": Problem.map_ur(EffPathlossPrior.from_config(cfg))}


def _interior(problem, sample, rng):
    n = sample.n_devices
    if problem.known_pathloss:
        return rng.uniform(0.2, 0.8, n)
    if problem.kind == "ml-ud":
        return rng.uniform(0.05, 1.2, n) * np.mean(sample.gains)
    pr = problem.prior
    return rng.uniform(1.05 * pr.g_low, 0.95 * pr.g_high, n)


# ---------------------------------------------------------------------------
# gradient / objective_value / build_state / stationarity_residual
# ---------------------------------------------------------------------------

def test_gradient_cold_start(cuda_device):
    from paper_2503_15259_b200 import Problem, estimators as est
    _, s = _sample(1, n=15, l=6)
    s.emp_cov[:] = 0.0
    st = est.build_state(Problem.ml_k(), np.zeros(15), s)
    g = est.gradient(Problem.ml_k(), np.zeros(15), st, s.gains, 32)
    np.testing.assert_allclose(g, s.gains * 6.0, rtol=1e-10)


def test_gradient_zero_at_generating_covariance(cuda_device):
    from paper_2503_15259_b200 import Problem, covlinalg, estimators as est
    _, s = _sample(2, n=15, l=6)
    x = np.random.default_rng(5).uniform(0.1, 0.9, 15)
    s.emp_cov = covlinalg.cov_unknown(s.pilots, x * s.gains, 1.0)
    st = est.build_state(Problem.ml_k(), x, s)
    np.testing.assert_allclose(est.gradient(Problem.ml_k(), x, st, s.gains, 32), 0.0, atol=1e-9)


@pytest.mark.parametrize("kind", ["ml-k", "map-k", "ml-ud", "map-ur"])
def test_gradient_matches_finite_differences(cuda_device, kind):
    from paper_2503_15259_b200 import estimators as est
    cfg, s = _sample(3, n=20, l=8, m=32)
    problem = _problems(cfg)[kind]
    rng = np.random.default_rng(77)
    for _ in range(2):
        x = _interior(problem, s, rng)
        g = est.gradient(problem, x, est.build_state(problem, x, s), s.gains, s.n_antennas)
        h = 1e-5
        fd = np.empty_like(x)
        for i in range(x.size):
            xp, xm = x.copy(), x.copy()
            xp[i] += h
            xm[i] -= h
            fp = est.objective_value(problem, xp, s, est.build_state(problem, xp, s))
            fm = est.objective_value(problem, xm, s, est.build_state(problem, xm, s))
            fd[i] = (fp - fm) / (2 * h)
        assert np.linalg.norm(fd - g) / np.linalg.norm(g) <= 1e-6


@pytest.mark.parametrize("kind", ["ml-k", "map-k", "ml-ud", "map-ur"])
def test_stationarity_residual_after_long_run(cuda_device, kind):
    from paper_2503_15259_b200 import StepSchedule, estimators as est, sysmodel
    cfg = _cfg(n=100, l=16, m=64, p=0.05)
    s = sysmodel.gen_dataset(cfg, 1, 100)[0]
    problem = _problems(cfg)[kind]
    tr = est.psca_run(problem, s, StepSchedule.polynomial(), max_iter=200, tol=0.0,
                      record_objective=False)
    assert est.stationarity_residual(problem, tr.final, s) <= 1e-3


@pytest.mark.parametrize("kind", ["ml-k", "map-k", "ml-ud", "map-ur"])
def test_components_engine_matches_fused(cuda_device, kind):
    """The reference loop over the component entry points == the fused solve."""
    from paper_2503_15259_b200 import StepSchedule, estimators as est
    cfg, s = _sample(9, n=60, l=12, m=24)
    problem = _problems(cfg)[kind]
    a = est.psca_run(problem, s, StepSchedule.default(), max_iter=20, tol=0.0, engine="fused")
    b = est.psca_run(problem, s, StepSchedule.default(), max_iter=20, tol=0.0,
                     engine="components")
    assert a.n_iterations == b.n_iterations == 20
    assert max_rel(b.final, a.final) <= 1e-10
    assert max_rel(b.update_norm, a.update_norm) <= 1e-9
    assert max_rel(b.objective, a.objective) <= 1e-11
    assert len(a.wall_times) == 20 and all(t > 0 for t in a.wall_times)
    assert len(set(a.wall_times)) > 1     # measured per iteration, not one mean


# ---------------------------------------------------------------------------
# abort paths and the test seams
# ---------------------------------------------------------------------------

def test_abort_when_covstate_build_is_monkeypatched(cuda_device, monkeypatch):
    """test_estimators.py:268-279 pointed at this package."""
    from paper_2503_15259_b200 import Problem, covlinalg, estimators as est
    _, s = _sample(15, n=15, l=6)
    monkeypatch.setattr("paper_2503_15259_b200.estimators.covlinalg.CovState.build",
                        lambda *a, **k: (_ for _ in ()).throw(
                            covlinalg.ConditioningError("forced", 1e99)))
    tr = est.psca_run(Problem.ml_k(), s, max_iter=5)
    assert tr.meta["abort"] == "forced (estimated condition number 1.000e+99)"
    np.testing.assert_array_equal(tr.final, np.zeros(15))


@pytest.mark.parametrize("k", [1, 4])
def test_device_fault_seam(cuda_device, k):
    """psca_solve_args.fault_iter: the factorisation opening iteration k-1 fails."""
    from paper_2503_15259_b200 import Problem, StepSchedule, estimators as est
    _, s = _sample(16, n=40, l=8)
    ref = est.psca_run(Problem.ml_k(), s, StepSchedule.default(), max_iter=8, tol=0.0)
    tr = est.psca_run(Problem.ml_k(), s, StepSchedule.default(), max_iter=8, tol=0.0,
                      fault_iter=k)
    assert tr.n_iterations == k - 1
    np.testing.assert_array_equal(tr.final, ref.iterates[k - 1])
    assert tr.meta["abort"].startswith(("Re(Sigma) is numerically singular",
                                        "A + B A^-1 B is numerically singular"))
    # at x = 0 Sigma is real: the reference fails on Re(Sigma)
    if k == 1:
        assert tr.meta["abort"].startswith("Re(Sigma)")


def test_conditioning_error_messages(cuda_device):
    """Which factor fails and the eigenvalue-ratio estimate, as covlinalg.py:78-115."""
    from paper_2503_15259_b200 import ConditioningError, frobenius_inverse
    with pytest.raises(ConditioningError) as e1:
        frobenius_inverse(np.diag([1.0, 1.0, 0.0]).astype(complex))   # test_covlinalg.py:91-95
    assert str(e1.value).startswith("Re(Sigma) is numerically singular (estimated condition")
    assert e1.value.cond_estimate > 1e12
    # Re(Sigma) = I is PD but Sigma = [[1, i], [-i, 1]] is singular: the reference's
    # second factor A + B A^-1 B = 0 fails
    with pytest.raises(ConditioningError) as e2:
        frobenius_inverse(np.array([[1.0, 1j], [-1j, 1.0]]))
    assert str(e2.value).startswith("A + B A^-1 B is numerically singular")
    assert e2.value.cond_estimate > 1e12


# ---------------------------------------------------------------------------
# priors on the device vs the reference grid (golden_components.npz)
# ---------------------------------------------------------------------------

def _golden_eff(g):
    from paper_2503_15259_b200.priors import EffPathlossPrior
    f = g["eff_fields"]
    n = g["eff_gamma"].size
    return EffPathlossPrior(np.full(n, 0.1), f[0], f[1], f[2], f[3], f[4], f[5],
                            dead_zone_grad=f[6])


def test_unknown_prior_grid_matches_reference(cuda_device, golden_components):
    """Every piece of the smoothed density (bump, gap/dead zone with its sign flip at
    g_low/2, Hermite bridge, exact tail, the +-dzg clip): device == reference."""
    from paper_2503_15259_b200 import priors
    g = golden_components
    eff = _golden_eff(g)
    gam = g["eff_gamma"]
    assert eff.g_low == pytest.approx(g["eff_fields"][7], rel=1e-15)
    grad = priors.log_prior_grad_unknown(gam, eff, 32)
    dens = priors.pdf_eff_smooth(gam, eff)
    val = priors.log_prior_value_unknown(gam, eff, 32)
    assert max_rel(grad, g["eff_grad_m32"]) <= 1e-13
    assert max_rel(dens, g["eff_dens"]) <= 1e-13
    assert abs(val - float(g["eff_value_m32"])) <= 1e-13 * abs(float(g["eff_value_m32"]))
    # the dead zone push is exactly +-dzg/M with the sign flip at g_low/2
    dead = g["eff_dens"] <= 1e-300
    np.testing.assert_array_equal(grad[dead], g["eff_grad_m32"][dead])
    with pytest.raises(priors.DomainError):
        priors.log_prior_grad_unknown(np.array([eff.g_high * 1.01]), eff, 32)


def test_known_prior_terms(cuda_device, golden_components):
    from paper_2503_15259_b200 import priors
    ind = priors.IndependentPrior(np.full(3, 0.05))
    np.testing.assert_array_equal(priors.log_prior_grad_known(np.zeros(3), ind, 64),
                                  golden_components["known_grad_p005_m64"])
    x = np.array([0.2, 0.0, 1.0])
    assert priors.log_prior_value_known(x, ind, 64) == pytest.approx(
        -float(ind.log_odds @ x) / 64, rel=1e-14)
    pw = priors.PairwiseMvbPrior.from_group_model(12, 3, 0.2)
    a = np.random.default_rng(0).uniform(0, 1, 12)
    np.testing.assert_allclose(priors.log_prior_grad_known(a, pw, 16),
                               -(pw.c1 + pw.c2 @ a) / 16, rtol=1e-14, atol=1e-16)
    assert priors.log_prior_value_known(a, pw, 16) == pytest.approx(
        -(pw.c1 @ a + 0.5 * a @ (pw.c2 @ a)) / 16, rel=1e-13)


# ---------------------------------------------------------------------------
# per-instance step schedules (psca_solve_args.steps_stride)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("kind", ["ml-k", "map-k", "ml-ud", "map-ur"])
@pytest.mark.parametrize("n_chunks", [1, 0])
def test_per_instance_steps_match_separate_solves(cuda_device, kind, n_chunks):
    """One call with a (B, T) step matrix == B calls with one schedule each, bit
    for bit on the same column kernel (what the PSCA-Net trainer's batched
    probe groups rely on)."""
    import torch
    from paper_2503_15259_b200 import device, estimators as est, sysmodel
    cfg = _cfg(n=60, l=12, m=32)
    samples = sysmodel.gen_dataset(cfg, 3, 11)
    prob = _problems(cfg)[kind]
    rng = np.random.default_rng(5)
    T = 7
    steps = rng.uniform(0.05, 1.0, (6, T))
    # every sample twice, with two different schedules
    idx = [0, 1, 2, 0, 1, 2]
    pil = np.stack([samples[i].pilots for i in idx])
    cov = np.stack([samples[i].emp_cov for i in idx])
    noise = np.array([samples[i].noise_power for i in idx])
    gains = np.stack([samples[i].gains for i in idx])
    kw = est.prior_arrays(prob, cfg.n_devices, cfg.n_antennas)
    g = gains if prob.known_pathloss else None
    res = device.solve(kind, pil, cov, noise, cfg.n_antennas, steps, gains=g, max_iter=T,
                       n_chunks=n_chunks, **kw)
    x = res["x"].cpu().numpy()
    un = res["update_norm"].cpu().numpy()
    for b in range(6):
        one = device.solve(kind, pil[b:b + 1], cov[b:b + 1], noise[b:b + 1], cfg.n_antennas,
                           steps[b], gains=None if g is None else g[b:b + 1], max_iter=T,
                           n_chunks=1 if n_chunks == 1 else n_chunks, **kw)
        if n_chunks == 1:
            assert np.array_equal(one["x"].cpu().numpy()[0], x[b])
            assert np.array_equal(one["update_norm"].cpu().numpy()[0], un[b])
        else:
            assert max_rel(one["x"].cpu().numpy()[0], x[b]) < 1e-10
    # the two schedules of the same sample really differ
    assert not np.array_equal(x[0], x[3])
    torch.cuda.synchronize()


def test_per_instance_steps_rejects_short_stride(cuda_device):
    from paper_2503_15259_b200 import device
    cfg = _cfg(n=40, l=8)
    _, s = _sample(2)
    with pytest.raises(ValueError):
        device.solve("ml-ud", s.pilots[None], s.emp_cov[None], np.array([1.0]), cfg.n_antennas,
                     np.full((2, 5), 0.5), max_iter=5)
