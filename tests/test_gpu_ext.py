"""SURVEY.md 8(f) rows on the GPU: pairwise MAP-K prior, GPU covariances of the
seeded datasets, the batched experiment harness and the batched-forward net
trainer, against the reference's outputs (tests/golden/golden_ext.npz)."""

import csv
import io
import pathlib

import numpy as np
import pytest

from psca_testutil import max_rel

pytestmark = pytest.mark.gpu
GOLD = pathlib.Path(__file__).parent / "golden" / "golden_ext.npz"


@pytest.fixture(scope="module")
def ext():
    return np.load(GOLD)


@pytest.mark.parametrize("i", range(3))
def test_pairwise_map_k_matches_reference(cuda_device, ext, i):
    from paper_2503_15259_b200 import estimators as est, priors, sysmodel
    import scipy.sparse as sp
    pre = f"pair{i}_"
    n = ext[pre + "pilots"].shape[1]
    c2 = sp.csr_matrix((ext[pre + "data"], ext[pre + "indices"], ext[pre + "indptr"]),
                       shape=(n, n))
    prob = est.Problem.map_k(priors.PairwiseMvbPrior(ext[pre + "c1"], c2))
    s = sysmodel.Sample(pilots=ext[pre + "pilots"], gains=ext[pre + "gains"],
                        activities=ext[pre + "activities"], eff_pathloss=ext[pre + "gains"],
                        received=ext[pre + "received"], emp_cov=ext[pre + "emp_cov"],
                        noise_power=float(ext[pre + "noise"]))
    tr = est.psca_run(prob, s, est.StepSchedule.default(), max_iter=25, tol=0.0,
                      record_objective=True)
    assert max_rel(tr.final, ext[pre + "final"]) <= 1e-9
    np.testing.assert_allclose(tr.objective, ext[pre + "objective"], rtol=1e-10)
    np.testing.assert_allclose(tr.update_norm, ext[pre + "update_norm"], rtol=1e-8)


@pytest.mark.parametrize("name", ["iid", "group", "frozen"])
def test_dataset_covariances_on_gpu(cuda_device, ext, name):
    from paper_2503_15259_b200 import sysmodel as sm
    cfgs = {
        "iid": sm.SystemConfig(n_devices=50, pilot_len=10, n_antennas=12),
        "group": sm.SystemConfig(n_devices=48, pilot_len=8, n_antennas=10,
                                 activity=sm.ActivityModel.group(4, 0.2)),
        "frozen": sm.SystemConfig(n_devices=30, pilot_len=6, n_antennas=8, freeze_pilots=True),
    }
    ds = sm.gen_dataset(cfgs[name], 3, [5, 6, 7])
    got = np.stack([d.emp_cov for d in ds])
    ref = ext[f"ds_{name}_emp_cov"]
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))
    np.testing.assert_array_equal(np.stack([d.received for d in ds]), ext[f"ds_{name}_received"])


def _rows(text):
    return list(csv.DictReader(io.StringIO(text)))


def _compare_grid(ours_csv, ref_csv, thr_tol=1e-8):
    ours, ref = _rows(ours_csv), _rows(ref_csv)
    assert len(ours) == len(ref)
    for a, b in zip(ours, ref):
        for col in ("method", "N", "L", "M", "P_dbm", "group_size", "iterations", "seed",
                    "flop_model_count", "flop_model_impl_count", "error"):
            assert a[col] == b[col], (col, a, b)
        assert float(a["error_rate"]) == float(b["error_rate"]), (a, b)
        assert abs(float(a["threshold"]) - float(b["threshold"])) <= thr_tol * max(
            1.0, abs(float(b["threshold"]))), (a, b)


def test_experiment_grid_matches_reference(cuda_device, ext):
    """run_grid on GPU batches: same rows, error rates and thresholds as the reference."""
    from paper_2503_15259_b200 import harness as h, sysmodel as sm
    grid = h.ExperimentGrid(
        methods=["psca-ml-k", "psca-map-k", "psca-ml-ud", "psca-map-ur", "psca-ml-k-net"],
        sweep_name="L", sweep_values=[8, 10],
        base=sm.SystemConfig(n_devices=64, pilot_len=8, n_antennas=16, tx_power_dbm=5.0,
                             activity=sm.ActivityModel.iid(0.15)),
        n_train=6, n_val=6, n_test=8, seeds=[0], train_budget=40)
    rows = h.run_grid(grid)
    assert all(r["mean_wall_time_s"] > 0 for r in rows)
    _compare_grid(h.strip_wall_time_columns(h.rows_to_csv(rows)), str(ext["grid_csv"]))


def test_group_prior_grid_matches_reference(cuda_device, ext):
    from paper_2503_15259_b200 import harness as h, sysmodel as sm
    grid = h.ExperimentGrid(
        methods=["psca-map-k"], sweep_name="group_size", sweep_values=[1, 4],
        base=sm.SystemConfig(n_devices=64, pilot_len=8, n_antennas=16, tx_power_dbm=5.0,
                             activity=sm.ActivityModel.iid(0.15)),
        n_val=6, n_test=8, seeds=[1])
    _compare_grid(h.strip_wall_time_columns(h.rows_to_csv(h.run_grid(grid))),
                  str(ext["ggrid_csv"]))


@pytest.mark.parametrize("kind", ["ml-k", "ml-ud", "map-k", "map-k-pair"])
def test_bcd_baseline_matches_reference(cuda_device, ext, kind):
    """Block coordinate descent sweeps (baselines.py:54-150) against the reference."""
    from paper_2503_15259_b200 import baselines, priors
    smp = _pg_samples(ext)
    if kind == "map-k":
        trs = baselines.bcd_map_k_batch(smp, priors.IndependentPrior(np.full(40, 0.1)), 5)
    elif kind == "map-k-pair":
        trs = baselines.bcd_map_k_batch(smp, priors.PairwiseMvbPrior.from_group_model(40, 4, 0.1),
                                        5)
    else:
        trs = baselines.bcd_ml_batch(smp, known=kind == "ml-k", max_iter=5)
    key = "bcd_" + kind.replace("-", "_")
    for b, t in enumerate(trs):
        assert max_rel(t.final, ext[key + "_final"][b]) <= 1e-9
        np.testing.assert_allclose(t.objective, ext[key + "_objective"][b], rtol=1e-10)
        np.testing.assert_allclose(t.update_norm, ext[key + "_update_norm"][b], rtol=1e-8)
        assert len(t.iterates) == 6
    one = baselines.bcd_ml(smp[2], known=True, max_iter=5) if kind == "ml-k" else None
    if one is not None:
        np.testing.assert_allclose(one.final, trs[2].final, rtol=1e-13, atol=1e-15)


def _pg_samples(ext):
    from paper_2503_15259_b200 import sysmodel as sm
    return [sm.Sample(pilots=ext["pg_pilots"][i], gains=ext["pg_gains"][i],
                      activities=ext["pg_activities"][i], eff_pathloss=ext["pg_gains"][i],
                      received=ext["pg_received"][i], emp_cov=ext["pg_emp_cov"][i],
                      noise_power=1.0) for i in range(ext["pg_pilots"].shape[0])]


@pytest.mark.parametrize("known", [True, False])
@pytest.mark.parametrize("mode", ["nonmonotone", "spectral", "fixed"])
def test_pg_baseline_matches_reference(cuda_device, ext, known, mode):
    """Batched projected gradient (baselines.py:156-252) against the reference."""
    from paper_2503_15259_b200 import baselines
    key = f"pg_{'k' if known else 'u'}_{mode}"
    d0 = (0.05 if known else 0.01) if mode == "fixed" else None
    trs = baselines.pg_ml_batch(_pg_samples(ext), known=known, max_iter=25, step_mode=mode, d0=d0)
    for b, t in enumerate(trs):
        assert max_rel(t.final, ext[key + "_final"][b]) <= 1e-8
        np.testing.assert_allclose(t.objective, ext[key + "_objective"][b], rtol=1e-10)
        np.testing.assert_allclose(t.update_norm, ext[key + "_update_norm"][b], rtol=1e-6,
                                   atol=1e-12)
        assert t.meta["line_search_failures"] == int(ext[key + "_failures"][b])
    # one sample through the single-sample entry gives the batch result
    one = baselines.pg_ml(_pg_samples(ext)[1], known=known, max_iter=25, step_mode=mode, d0=d0)
    np.testing.assert_allclose(one.final, trs[1].final, rtol=1e-12, atol=1e-15)


def test_baseline_grid_matches_reference(cuda_device, ext):
    """PG and BCD rows of run_grid (bench.py:244-281) against the reference."""
    from paper_2503_15259_b200 import harness as h, sysmodel as sm
    grid = h.ExperimentGrid(
        methods=["pg-ml-k", "pg-ml-ud", "bcd-ml-k", "bcd-map-k", "bcd-ml-ud"], sweep_name="L", sweep_values=[8],
        base=sm.SystemConfig(n_devices=64, pilot_len=8, n_antennas=16, tx_power_dbm=5.0,
                             activity=sm.ActivityModel.iid(0.15)),
        n_val=6, n_test=8, seeds=[0])
    # PG is first-order: 60 iterations with a line search carry rounding-level
    # differences of the objective further than PSCA does (threshold to 1e-6)
    _compare_grid(h.strip_wall_time_columns(h.rows_to_csv(h.run_grid(grid))),
                  str(ext["pgrid_csv"]), thr_tol=1e-6)


def test_trainer_matches_reference(cuda_device, ext):
    """unroll.train with batched GPU forwards follows the reference's search."""
    from paper_2503_15259_b200 import estimators as est, sysmodel as sm, unroll

    def samples(prefix):
        k = ext[prefix + "pilots"].shape[0]
        return [sm.Sample(pilots=ext[prefix + "pilots"][i], gains=ext[prefix + "gains"][i],
                          activities=ext[prefix + "activities"][i],
                          eff_pathloss=ext[prefix + "gains"][i],
                          received=ext[prefix + "received"][i],
                          emp_cov=ext[prefix + "emp_cov"][i], noise_power=1.0)
                for i in range(k)]

    net = unroll.UnrolledConfig.with_default_schedule(est.Problem.ml_k(), 5)
    rep = unroll.train(net, samples("train_tr_"), samples("train_va_"), budget=80, seed=3)
    assert rep.stopped_epoch == int(ext["train_stopped_epoch"])
    assert rep.budget_exhausted == bool(ext["train_budget_exhausted"])
    np.testing.assert_allclose(rep.best_steps, ext["train_best_steps"], rtol=1e-7)
    np.testing.assert_allclose(rep.val_loss_curve, ext["train_val_curve"], rtol=1e-9)
    assert abs(rep.threshold - float(ext["train_threshold"])) <= 1e-8
