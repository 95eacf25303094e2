"""SURVEY.md 8(f) rows on the host: pairwise prior (oracle + construction),
seeded scene draws, harness formats and trainer helpers, against golden
vectors produced by the reference (tests/golden/make_golden.py ext)."""

import pathlib

import numpy as np
import pytest

from oracle import psca_oracle as orc   # checker only

GOLD = pathlib.Path(__file__).parent / "golden" / "golden_ext.npz"


@pytest.fixture(scope="module")
def ext():
    return np.load(GOLD)


def _pair(ext, i):
    pre = f"pair{i}_"
    return pre, (ext[pre + "indptr"], ext[pre + "indices"], ext[pre + "data"])


@pytest.mark.parametrize("i", range(3))
def test_oracle_pairwise_prior_matches_reference(ext, i):
    pre, c2 = _pair(ext, i)
    m = ext[pre + "received"].shape[1]
    r = orc.psca("map-k", ext[pre + "pilots"], ext[pre + "gains"], ext[pre + "emp_cov"],
                 float(ext[pre + "noise"]), m, orc.default_steps(25), 25, record_objective=True,
                 pairwise=(ext[pre + "c1"], c2))
    f = ext[pre + "final"]
    assert np.max(np.abs(r["final"] - f)) <= 1e-12 * np.max(np.abs(f))
    np.testing.assert_allclose(r["objective"], ext[pre + "objective"], rtol=1e-12)
    np.testing.assert_allclose(r["update_norm"], ext[pre + "update_norm"], rtol=1e-10)


@pytest.mark.parametrize("i", range(3))
def test_group_prior_construction_matches_reference(ext, i):
    from paper_2503_15259_b200.priors import PairwiseMvbPrior
    pre, c2 = _pair(ext, i)
    n = ext[pre + "pilots"].shape[1]
    pr = PairwiseMvbPrior.from_group_model(n, int(ext[pre + "group"]), 0.15)
    np.testing.assert_array_equal(pr.c1, ext[pre + "c1"])
    ip, ix, dv = pr.csr_arrays()
    np.testing.assert_array_equal(ip, c2[0])
    np.testing.assert_array_equal(ix, c2[1])
    np.testing.assert_array_equal(dv, c2[2])


@pytest.mark.parametrize("name", ["iid", "group", "frozen"])
def test_scene_draws_match_reference_bitwise(ext, name):
    from paper_2503_15259_b200 import sysmodel as sm
    cfgs = {
        "iid": sm.SystemConfig(n_devices=50, pilot_len=10, n_antennas=12),
        "group": sm.SystemConfig(n_devices=48, pilot_len=8, n_antennas=10,
                                 activity=sm.ActivityModel.group(4, 0.2)),
        "frozen": sm.SystemConfig(n_devices=30, pilot_len=6, n_antennas=8, freeze_pilots=True),
    }
    ds = sm.draw_dataset(cfgs[name], 3, [5, 6, 7])
    for f in ("pilots", "gains", "activities", "eff_pathloss", "received"):
        np.testing.assert_array_equal(np.stack([d[f] for d in ds]), ext[f"ds_{name}_{f}"])


def test_harness_formats_and_models(ext):
    from paper_2503_15259_b200 import harness as h
    assert h.flop_model("psca-ml-k", 64, 8) == 40 * 64 * 64
    assert h.flop_model("bcd-ml-k", 64, 8) == 56 * 64 * 64
    assert h.flop_model("psca-map-k", 64, 8, True, True) == 40 * 64 * 64 + 2 ** 64
    assert h.flop_model("psca-map-k", 64, 8, True, False) == 40 * 64 * 64
    assert h.error_rate([np.array([1.0, 0.0])], [np.array([1.0, 1.0])]) == 0.5
    header = str(ext["grid_csv"]).splitlines()[0]
    rows = [{"method": "psca-ml-k", "N": 1, "error_rate": 0.25, "threshold": 0.1,
             "mean_wall_time_s": 1.0, "error": ""}]
    assert h.strip_wall_time_columns(h.rows_to_csv(rows)).splitlines()[0] == header
    with pytest.raises(h.DomainError):
        h.ExperimentGrid(methods=["psca-ml-k-net"], sweep_name="L", sweep_values=[8])
    with pytest.raises(h.DomainError):
        h.ExperimentGrid(methods=["nope"], sweep_name="L", sweep_values=[8])
    g = h.ExperimentGrid(methods=["psca-ml-k"], sweep_name="group_size", sweep_values=[4])
    assert g.config_at(4).activity.group_size == 4
    assert g.iterations_for("psca-ml-k", 4) == 30 and g.iterations_for("pg-ml-k", 4) == 60


def test_trainer_helpers():
    from paper_2503_15259_b200 import unroll
    x, f = unroll._golden_section(lambda v: (v - 0.3) ** 2, -1.0, 1.0, n_iter=40)
    assert abs(x - 0.3) < 1e-6
    soft = np.array([[0.2, 0.9], [0.0, 1.0]])
    truth = np.array([[0.0, 1.0], [0.0, 1.0]])
    u = np.clip(soft, 1e-6, 1 - 1e-6)
    ref = float(np.mean(-(truth * np.log(u) + (1 - truth) * np.log(1 - u))))
    assert unroll.bce_loss(soft, truth, True) == ref
    assert unroll.bce_loss(soft * 2.0, truth, False, gains=np.full((2, 2), 2.0)) == ref
    th = unroll._clip_theta(np.array([1.0, -9.0, 7.0]), 2, np.log(1e-3), 0.0)
    np.testing.assert_array_equal(th, [0.0, np.log(1e-3), 4.0])
