"""Solver behaviour the reference tests pin (tests/test_estimators.py:207-330),
the q-floor abort path against the reference, per-instance isolation inside a
batch, and edge shapes -- all on the CUDA path."""

import json
import pathlib

import numpy as np
import pytest

from oracle import psca_oracle as orc   # checker only
from psca_testutil import max_rel

pytestmark = pytest.mark.gpu
GOLD = pathlib.Path(__file__).parent / "golden" / "golden_ext.npz"


def unit_cfg(n_devices, pilot_len, n_antennas=32, p=0.1):
    from paper_2503_15259_b200 import sysmodel as sm
    return sm.SystemConfig(n_devices=n_devices, pilot_len=pilot_len, n_antennas=n_antennas,
                           noise_power=1.0, tx_power_dbm=0.0, d_inner=1.0, d_outer=2.0,
                           pathloss_exp=2.5, wavelength=4.0 * np.pi,
                           activity=sm.ActivityModel.iid(p))


def unit_sample(seed, n_devices, pilot_len, n_antennas=32):
    from paper_2503_15259_b200 import sysmodel as sm
    cfg = unit_cfg(n_devices, pilot_len, n_antennas)
    return cfg, sm.gen_dataset(cfg, 1, seed)[0]


def problems_for(cfg):
    from paper_2503_15259_b200 import Problem, priors
    return {"ml-k": Problem.ml_k(), "ml-ud": Problem.ml_ud(),
            "map-k": Problem.map_k(priors.IndependentPrior(np.full(cfg.n_devices, 0.1))),
            "map-ur": Problem.map_ur(priors.EffPathlossPrior.from_config(cfg))}


def test_zero_iterations(cuda_device):
    from paper_2503_15259_b200 import Problem, psca_run
    _, s = unit_sample(8, 15, 6)
    tr = psca_run(Problem.ml_k(), s, max_iter=0)
    np.testing.assert_array_equal(tr.final, np.zeros(15))
    assert tr.n_iterations == 0 and len(tr.iterates) == 1


def test_trace_lengths_and_update_norms(cuda_device):
    from paper_2503_15259_b200 import Problem, psca_run
    _, s = unit_sample(9, 15, 6)
    tr = psca_run(Problem.ml_k(), s, max_iter=12, tol=0.0)
    assert tr.n_iterations == 12
    assert len(tr.iterates) == 13 and len(tr.objective) == 12 and len(tr.wall_times) == 12
    for i in range(12):
        manual = np.linalg.norm(tr.iterates[i + 1] - tr.iterates[i])
        assert tr.update_norm[i] == pytest.approx(manual, rel=1e-12)


def test_objective_decreases_and_tolerance_stop(cuda_device):
    from paper_2503_15259_b200 import Problem, psca_run
    _, s = unit_sample(10, 30, 8)
    tr = psca_run(Problem.ml_k(), s, max_iter=30, tol=0.0)
    assert tr.objective[-1] < tr.objective[0]
    _, s = unit_sample(11, 15, 6)
    tr = psca_run(Problem.ml_k(), s, max_iter=500, tol=1e-4)
    assert tr.n_iterations < 500 and tr.update_norm[-1] < 1e-4
    assert all(u >= 1e-4 for u in tr.update_norm[:-1])


@pytest.mark.parametrize("kind", ["ml-k", "map-k", "ml-ud", "map-ur"])
def test_box_feasibility(cuda_device, kind):
    from paper_2503_15259_b200 import bounds_for, psca_run
    cfg, s = unit_sample(12, 25, 8)
    prob = problems_for(cfg)[kind]
    lo, hi = bounds_for(prob, s)
    tr = psca_run(prob, s, max_iter=25, tol=0.0)
    for it in tr.iterates:
        assert np.all(it >= lo) and np.all(it <= hi)


def test_noiseless_orthogonal_toy(cuda_device):
    from paper_2503_15259_b200 import Problem, Sample, psca_run
    l = 8
    pilots = np.sqrt(l) * np.eye(l, dtype=complex)
    gamma = np.zeros(l)
    gamma[3] = 1.0
    rng = np.random.Generator(np.random.Philox(np.random.SeedSequence(13)))
    h = (rng.standard_normal((l, 512)) + 1j * rng.standard_normal((l, 512))) / np.sqrt(2)
    y = (pilots * np.sqrt(gamma)) @ h
    s = Sample(pilots=pilots, gains=np.ones(l), activities=gamma.copy(),
               eff_pathloss=gamma.copy(), received=y, emp_cov=y @ y.conj().T / 512,
               noise_power=1e-3)
    tr = psca_run(Problem.ml_k(), s, max_iter=30, tol=0.0)
    assert np.max(np.abs(tr.final - gamma)) <= 0.05


def test_map_k_even_odds_is_iterate_identical_to_ml(cuda_device):
    from paper_2503_15259_b200 import Problem, psca_run
    from paper_2503_15259_b200.priors import IndependentPrior
    _, s = unit_sample(14, 20, 8)
    a = psca_run(Problem.ml_k(), s, max_iter=15, tol=0.0)
    b = psca_run(Problem.map_k(IndependentPrior(np.full(20, 0.5))), s, max_iter=15, tol=0.0)
    for x, y in zip(a.iterates, b.iterates):
        np.testing.assert_array_equal(x, y)


def test_trace_jsonl_dump(cuda_device, tmp_path):
    from paper_2503_15259_b200 import Problem, psca_run
    _, s = unit_sample(16, 15, 6)
    tr = psca_run(Problem.ml_k(), s, max_iter=5, tol=0.0)
    path = tmp_path / "trace.jsonl"
    tr.dump_jsonl(path, method="psca-ml-k")
    recs = [json.loads(line) for line in path.read_text().splitlines()]
    assert len(recs) == 5 and recs[0]["method"] == "psca-ml-k" and recs[2]["iteration"] == 3
    assert recs[1]["update_norm"] == pytest.approx(tr.update_norm[1])


@pytest.mark.parametrize("kind", ["ml-k", "map-k", "ml-ud", "map-ur"])
def test_stationarity_after_long_run(cuda_device, kind):
    """Projected-gradient residual <= 1e-3 after 200 polynomial-schedule steps; the
    residual is evaluated by the oracle at the GPU's final iterate."""
    from paper_2503_15259_b200 import StepSchedule, psca_run, sysmodel as sm
    cfg = unit_cfg(100, 16, 64, 0.05)
    s = sm.gen_dataset(cfg, 1, 100)[0]
    prob = problems_for(cfg)[kind]
    tr = psca_run(prob, s, schedule=StepSchedule.polynomial(), max_iter=200, tol=0.0,
                  record_objective=False)
    x = tr.final
    known = kind in ("ml-k", "map-k")
    w = x * s.gains if known else x
    sigma = orc.model_cov(s.pilots, w, s.noise_power)
    q, r = orc.quad(s.pilots, orc.herm_inverse(sigma), s.emp_cov)
    grad = (s.gains * (q - r)) if known else (q - r)
    if kind == "map-k":
        grad = grad + orc.indep_prior_grad(np.full(100, 0.1), s.n_antennas, 100)
    elif kind == "map-ur":
        grad = grad + orc.eff_prior_grad(x, orc.EffPrior.from_reference(prob.prior), s.n_antennas)
    hi = 1.0 if known else (np.inf if kind == "ml-ud" else prob.prior.g_high)
    assert np.max(np.abs(x - np.clip(x - grad, 0.0, hi))) <= 1e-3


@pytest.fixture(scope="module")
def ext():
    return np.load(GOLD)


def _abort_sample(ext, j):
    from paper_2503_15259_b200 import Sample
    pre = f"abort{j}_"
    return Sample(pilots=ext[pre + "pilots"], gains=ext[pre + "gains"],
                  activities=ext[pre + "activities"], eff_pathloss=ext[pre + "gains"],
                  received=ext[pre + "received"], emp_cov=ext[pre + "emp_cov"], noise_power=1.0)


@pytest.mark.parametrize("j", range(4))
def test_qfloor_abort_matches_reference(cuda_device, ext, j):
    """psca_run never raises on numerical failure: meta['abort'] carries the
    reference's message and final is the last accepted iterate (estimators.py:263-271)."""
    from paper_2503_15259_b200 import Problem, StepSchedule, psca_run
    pre = f"abort{j}_"
    prob = Problem.ml_k() if str(ext[pre + "kind"]) == "ml-k" else Problem.ml_ud()
    tr = psca_run(prob, _abort_sample(ext, j), StepSchedule.default(), max_iter=40, tol=0.0,
                  record_objective=False)
    assert tr.meta.get("abort") == str(ext[pre + "message"])
    assert tr.n_iterations == int(ext[pre + "n_iter"])
    f = ext[pre + "final"]
    assert np.max(np.abs(tr.final - f)) <= 1e-9 * max(np.max(np.abs(f)), 1e-300)


def test_abort_is_isolated_to_its_instance(cuda_device, ext):
    """One aborting instance in a batch leaves the others' results unchanged."""
    from paper_2503_15259_b200 import Problem, StepSchedule, device, psca_run, psca_run_batch
    bad = _abort_sample(ext, 0)
    _, good = unit_sample(21, 24, 6)
    good.gains = good.gains * 100
    samples = [good, bad, good]
    out = psca_run_batch(Problem.ml_k(), np.stack([s.pilots for s in samples]),
                         np.stack([s.emp_cov for s in samples]), np.ones(3), 32,
                         gains=np.stack([s.gains for s in samples]),
                         schedule=StepSchedule.default(), max_iter=40)
    status = out["status"].cpu().numpy()
    assert status[1] == device.STATUS_QFLOOR and status[0] == status[2] == 0
    assert int(out["n_iter"][1]) == int(ext["abort0_n_iter"])
    x = out["x"].cpu().numpy()
    single = psca_run(Problem.ml_k(), good, StepSchedule.default(), max_iter=40, tol=0.0).final
    assert max_rel(x[0], single) <= 1e-13 and np.array_equal(x[0], x[2])
    assert np.max(np.abs(x[1] - ext["abort0_final"])) <= 1e-9 * np.max(np.abs(ext["abort0_final"]))


@pytest.mark.parametrize("n,l", [(5, 3), (7, 1), (33, 2), (77, 11), (130, 17), (64, 32)])
def test_edge_shapes_match_oracle(cuda_device, n, l):
    """Ragged N (not a multiple of the 32-column tile, fewer than one tile), odd
    and minimal L, against the oracle."""
    from paper_2503_15259_b200 import Problem, StepSchedule, psca_run
    for kind in ("ml-k", "ml-ud"):
        cfg, s = unit_sample([n, l], n, l, 16)
        prob = Problem.ml_k() if kind == "ml-k" else Problem.ml_ud()
        tr = psca_run(prob, s, StepSchedule.default(), max_iter=20, tol=0.0)
        ref = orc.psca(kind, s.pilots, s.gains, s.emp_cov, 1.0, 16, orc.default_steps(20), 20)
        assert max_rel(tr.final, ref["final"]) <= 1e-9, (n, l, kind)


@pytest.mark.parametrize("n,l", [(5, 3), (7, 1), (33, 2), (77, 11), (130, 17), (2600, 72)])
def test_one_chunk_shapes_match_oracle(cuda_device, n, l):
    """One column chunk per instance (the warp-streamed column kernel; a chunk
    too wide for its SMEM lists, N = 2600 at L = 72, falls back to the tile
    kernel): ragged and minimal shapes against the oracle."""
    from paper_2503_15259_b200 import Problem, StepSchedule, psca_run_batch
    T = 6 if n > 1000 else 20
    for kind in ("ml-k", "ml-ud"):
        ss = [unit_sample([n, l, i], n, l, 16)[1] for i in range(2)]
        prob = Problem.ml_k() if kind == "ml-k" else Problem.ml_ud()
        out = psca_run_batch(prob, np.stack([s.pilots for s in ss]), np.stack([s.emp_cov for s in ss]),
                             np.ones(2), 16, gains=np.stack([s.gains for s in ss]),
                             schedule=StepSchedule.default(), max_iter=T, n_chunks=1)
        x = out["x"].cpu().numpy()
        for i, s in enumerate(ss):
            ref = orc.psca(kind, s.pilots, s.gains, s.emp_cov, 1.0, 16, orc.default_steps(T), T)
            assert max_rel(x[i], ref["final"]) <= 1e-9, (n, l, kind, i)


def test_empty_batch(cuda_device):
    from paper_2503_15259_b200 import Problem, psca_run_batch
    out = psca_run_batch(Problem.ml_ud(), np.zeros((0, 4, 10), complex), np.zeros((0, 4, 4), complex),
                         np.zeros(0), 8, max_iter=5)
    assert tuple(out["x"].shape) == (0, 10)


@pytest.mark.parametrize("B,chunks", [(2400, 0), (700, 0), (5, 0), (9, 3)])
def test_host_batch_api_matches_device_batch(cuda_device, B, chunks):
    """psca_run_batch_host (pinned host in / out, chunked uploads overlapped with
    the solves on alternating streams) returns the device batch's estimates."""
    import torch
    from paper_2503_15259_b200 import Problem, psca_run_batch, psca_run_batch_host
    cfg = unit_cfg(40, 6, 16)
    from paper_2503_15259_b200 import sysmodel as sm
    base = sm.draw_dataset(cfg, 7, [77])
    idx = np.arange(B) % 7
    pil = np.stack([base[i]["pilots"] for i in idx])
    gains = np.stack([base[i]["gains"] for i in idx])
    rec = np.stack([base[i]["received"] for i in idx])
    emp = np.einsum("blm,bkm->blk", rec, rec.conj()) / 16
    noise = np.ones(B)
    host = psca_run_batch_host(Problem.ml_k(), torch.from_numpy(pil).pin_memory(),
                               torch.from_numpy(emp).pin_memory(), noise, 16,
                               gains=torch.from_numpy(gains).pin_memory(), max_iter=10,
                               chunks=chunks)
    dev = psca_run_batch(Problem.ml_k(), pil, emp, noise, 16, gains=gains, max_iter=10,
                         n_chunks=1)
    xd = dev["x"].cpu().numpy()
    xh = host["x"].numpy()
    assert xh.shape == (B, 40) and np.all(host["status"].numpy() == 0)
    assert np.all(host["n_iter"].numpy() == 10)
    if B >= 2 * torch.cuda.get_device_properties(0).multi_processor_count:
        np.testing.assert_array_equal(xh, xd)
    else:
        assert np.max(np.abs(xh - xd)) <= 1e-12 * np.max(np.abs(xd))
