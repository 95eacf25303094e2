"""The CPU oracle pinned against the reference's own outputs (golden fixtures).

tests/golden/*.npz were produced by running the reference implementation
(/root/reference/pkg/src/actdet) via tests/golden/make_golden.py.  These tests
run on the CPU (no GPU marker) and establish that oracle/psca_oracle.py is a
faithful restatement before it is used as the checker of the CUDA path.
"""

import numpy as np
import pytest

from oracle import psca_oracle as orc
from psca_testutil import max_rel


def _case(g, i):
    pre = f"case{i}_"
    return {k[len(pre):]: v for k, v in g.items() if k.startswith(pre)}


def _eff(c, n):
    f = c["eff"]
    return orc.EffPrior(np.full(n, float(c["p"])), f[0], f[1], f[2], f[3], f[4], f[5], f[6])


def _run(c, steps, max_iter, tol=0.0, record_objective=True):
    kind = str(c["kind"])
    n = c["pilots"].shape[1]
    return orc.psca(kind, c["pilots"], c["gains"], c["emp_cov"], float(c["noise"]),
                    c["received"].shape[1], steps, max_iter, tol=tol,
                    indep_p=np.full(n, float(c["p"])) if kind == "map-k" else None,
                    eff=_eff(c, n) if kind == "map-ur" else None,
                    record_objective=record_objective)


def test_schedule_known_answers():
    # test_estimators.py:61-64
    s = orc.default_steps(3)
    assert s[0] == 0.5 and s[1] == 0.375
    assert s[2] == pytest.approx(0.3046875, abs=1e-12)


@pytest.mark.parametrize("i", range(32))
def test_oracle_matches_reference_trace(golden_small, i):
    if i >= int(golden_small["n_cases"]):
        pytest.skip("fewer cases")
    c = _case(golden_small, i)
    out = _run(c, orc.default_steps(int(c["max_iter"])), int(c["max_iter"]))
    assert (out["abort"] is not None) == bool(c["abort"])
    # same primitive operations as the reference: agreement to rounding level
    assert max_rel(out["final"], c["final"]) <= 1e-12
    assert max_rel(out["update_norm"], c["update_norm"]) <= 1e-12
    assert max_rel(out["objective"], c["objective"]) <= 1e-12
    assert max_rel(np.array(out["iterates"]), c["iterates"]) <= 1e-12


@pytest.mark.parametrize("i", range(0, 32, 3))
def test_oracle_polynomial_schedule_with_tolerance_stop(golden_small, i):
    c = _case(golden_small, i)
    out = _run(c, orc.polynomial_steps(60), 60, tol=1e-4, record_objective=False)
    assert len(out["update_norm"]) == len(c["poly_update_norm"])
    assert max_rel(out["final"], c["poly_final"]) <= 1e-11


@pytest.mark.parametrize("i", range(1, 32, 4))
def test_oracle_net_forward(golden_small, i):
    c = _case(golden_small, i)
    steps = c["net_steps"]
    out = _run(c, steps, len(steps), record_objective=False)
    assert max_rel(out["final"], c["net_out"]) <= 1e-12


def test_oracle_components(golden_components):
    g = golden_components
    for j in range(int(g["n_comp"])):
        p = f"comp{j}_"
        s = g[p + "pilots"]
        assert max_rel(orc.emp_cov(g[p + "y"]), g[p + "emp"]) <= 1e-14
        sigma = orc.model_cov(s, g[p + "gamma"], float(g[p + "noise"]))
        assert max_rel(sigma, g[p + "sigma"]) <= 1e-14
        inv = orc.herm_inverse(sigma)
        assert max_rel(inv, g[p + "inv"]) <= 1e-13
        q, r = orc.quad(s, inv, g[p + "emp"])
        assert max_rel(q, g[p + "q"]) <= 1e-13 and max_rel(r, g[p + "r"]) <= 1e-13
        obj = orc.objective_cov(sigma, inv, g[p + "emp"])
        assert obj == pytest.approx(float(g[p + "obj"]), rel=1e-13)


def test_oracle_prior_gradients(golden_components):
    g = golden_components
    f = g["eff_fields"]
    gam = g["eff_gamma"]
    eff = orc.EffPrior(np.full(gam.size, 0.1), f[0], f[1], f[2], f[3], f[4], f[5])
    assert eff.g_low == pytest.approx(f[7], rel=1e-15)
    assert eff.g_high == pytest.approx(f[8], rel=1e-15)
    assert eff.dead_zone_grad == pytest.approx(f[6], rel=1e-15)
    grad = orc.eff_prior_grad(gam, eff, 32)
    np.testing.assert_allclose(grad, g["eff_grad_m32"], rtol=1e-13, atol=1e-300)
    dens, _ = orc.smooth_density(gam, eff)
    np.testing.assert_allclose(dens, g["eff_dens"], rtol=1e-13, atol=1e-300)
    assert orc.eff_prior_value(gam, eff, 32) == pytest.approx(float(g["eff_value_m32"]), rel=1e-13)
    # priors.py known-answer (test_priors.py:192-195)
    kg = orc.indep_prior_grad(np.full(3, 0.05), 64, 3)
    np.testing.assert_allclose(kg, g["known_grad_p005_m64"], rtol=0, atol=0)
    np.testing.assert_allclose(kg, 0.0460068590495, rtol=1e-10)


def test_oracle_threshold(golden_components):
    g = golden_components
    theta = orc.calibrate(list(g["thr_scores"]), list(g["thr_truths"]))
    assert theta == float(g["thr_theta"])


def test_oracle_singular_raises():
    # test_covlinalg.py:89-95
    with pytest.raises(orc.OracleConditioningError) as err:
        orc.herm_inverse(np.diag([1.0, 1.0, 0.0]).astype(complex))
    assert err.value.cond_estimate > 1e12
