"""Large-L step-loop path (csrc/psca_large.cuh, large.py) on the GPU.

PSCA_FORCE_LARGE=1 routes any L through the large path (read per call), so
it is checked against the reference traces and the compiled small-L path on
shapes the small path also covers, and against the oracle / golden c4 at
L = 160 and L = 256 (BASELINE config 4 is in test_gpu_baseline.py).
"""

import os

import numpy as np
import pytest

from oracle import psca_oracle as orc   # checker only
from psca_testutil import case, max_rel

pytestmark = pytest.mark.gpu


@pytest.fixture
def force_large(monkeypatch):
    monkeypatch.setenv("PSCA_FORCE_LARGE", "1")


def _pkg():
    from paper_2503_15259_b200 import estimators, priors
    import paper_2503_15259_b200 as pkg
    return pkg, estimators, priors


@pytest.mark.parametrize("i", [0, 1, 2, 3, 9, 12, 21, 22, 24, 26, 27, 29, 30, 31])
def test_large_path_matches_reference_traces(cuda_device, golden_small, force_large, i):
    import test_gpu_parity as tp
    pkg, est, _ = _pkg()
    c = case(golden_small, i)
    tr = est.psca_run(tp._problem(c), tp._sample(c), est.StepSchedule.default(),
                      max_iter=int(c["max_iter"]), tol=0.0, record_objective=True)
    tol = tp._tol(c, orc.default_steps(int(c["max_iter"])), int(c["max_iter"]))
    assert tr.n_iterations == len(c["update_norm"])
    assert max_rel(tr.final, c["final"]) <= tol
    assert max_rel(np.array(tr.iterates), c["iterates"]) <= tol
    assert max_rel(tr.objective, c["objective"]) <= 1e-10


@pytest.mark.parametrize("L,kind", [(40, "ml-ud"), (64, "map-k"), (72, "ml-k"), (96, "ml-ud")])
def test_large_path_equals_batched_path(cuda_device, L, kind, monkeypatch):
    pkg, est, _ = _pkg()
    from paper_2503_15259_b200 import scenes
    cfg = scenes.SceneConfig(11, kind, 700, L, 96, 30, 30, 2)
    ss = [scenes.make_scene(cfg, i) for i in range(2)]
    b = scenes.stack_batch(ss)
    problem = scenes.problem_for(cfg)
    small = est.psca_run_batch(problem, b["pilots"], b["emp_cov"], b["noise"], 96,
                               gains=b["gains"], max_iter=30)["x"].cpu().numpy()
    monkeypatch.setenv("PSCA_FORCE_LARGE", "1")
    large = est.psca_run_batch(problem, b["pilots"], b["emp_cov"], b["noise"], 96,
                               gains=b["gains"], max_iter=30)
    assert large["path"] == "large"
    xl = large["x"].cpu().numpy()
    for k in range(2):
        assert max_rel(xl[k], small[k]) <= 1e-11


@pytest.mark.parametrize("L,kind", [(160, "ml-k"), (130, "map-ur"), (131, "ml-ud")])
def test_large_l_matches_oracle(cuda_device, L, kind):
    pkg, est, _ = _pkg()
    from paper_2503_15259_b200 import scenes
    cfg = scenes.SceneConfig(12, kind, 900, L, 200, 40, 20, 1)
    s = scenes.make_scene(cfg, 0)
    problem = scenes.problem_for(cfg)
    tr = est.psca_run(problem, s, est.StepSchedule.default(), max_iter=20, tol=0.0,
                      record_objective=False)
    kw = {}
    if kind == "map-ur":
        kw["eff"] = orc.EffPrior.from_reference(problem.prior)
    ref = orc.psca(kind, s.pilots, s.gains, s.emp_cov, 1.0, 200, orc.default_steps(20), 20, **kw)
    tol = 1e-9
    if kind == "map-ur":
        tol = max(tol, 10 * orc.perturbation_floor(kind, s.pilots, s.gains, s.emp_cov, 1.0, 200,
                                                   orc.default_steps(20), 20, **kw))
    assert max_rel(tr.final, ref["final"]) <= tol
    assert max_rel(tr.update_norm, ref["update_norm"]) <= 1e-8


def test_large_l_pairwise_map_k_matches_oracle(cuda_device):
    """Pairwise MVB prior (priors.py:56-159) on the large-L path (L = 136 > 128):
    estimates, update norms and the recorded objective against the oracle."""
    pkg, est, _ = _pkg()
    from paper_2503_15259_b200 import priors, scenes
    from paper_2503_15259_b200.large import psca_run_large
    N, L, M, T = 600, 136, 160, 15
    cfg = scenes.SceneConfig(14, "map-k", N, L, M, 30, T, 1)
    s = scenes.make_scene(cfg, 0)
    pr = priors.PairwiseMvbPrior.from_group_model(N, 4, 0.1)
    problem = est.Problem.map_k(pr)
    tr = est.psca_run(problem, s, est.StepSchedule.default(), max_iter=T, tol=0.0,
                      record_objective=True)
    assert tr.meta.get("abort") is None
    c1 = np.broadcast_to(pr.c1, (N,)).astype(float)
    ref = orc.psca("map-k", s.pilots, s.gains, s.emp_cov, 1.0, M, orc.default_steps(T), T,
                   record_objective=True, pairwise=(c1, pr.csr_arrays()))
    assert max_rel(tr.final, ref["final"]) <= 1e-9
    assert max_rel(tr.update_norm, ref["update_norm"]) <= 1e-8
    assert max_rel(np.asarray(tr.objective), np.asarray(ref["objective"])) <= 1e-10
    # the prior really acts: the independent prior gives a different estimate
    ind = est.psca_run(scenes.problem_for(cfg), s, est.StepSchedule.default(), max_iter=T)
    assert max_rel(ind.final, tr.final) > 1e-6
    # missing half of the pairwise arguments is an error, not a silent fallback
    with pytest.raises(ValueError):
        psca_run_large("map-k", s.pilots, s.gains, s.emp_cov, 1.0, M, orc.default_steps(T),
                       max_iter=T, prior_c1=c1)


def _run_shards(kind, S, g, E, M, steps, T, nshard, **kw):
    """Column-sharded GPU steppers on ONE GPU, the all-reduces done by hand
    (sum of the [increment | dx2 | prior] blocks, min of min q): the sharded
    semantics of large.ShardedDriver without a second GPU."""
    import torch
    from paper_2503_15259_b200.large import GpuLargeStepper, column_shard
    N = S.shape[1]
    sls = [column_shard(N, r, nshard) for r in range(nshard)]
    sts = [GpuLargeStepper(kind, np.ascontiguousarray(S[:, sl]),
                           np.ascontiguousarray(g[sl]) if g is not None else None, E, 1.0, M,
                           steps, max_iter=T, **{k: (v[sl] if k in ("prior_p", "prior_lin") else v)
                                                 for k, v in kw.items()})
           for sl in sls]
    for st in sts:
        st.begin()
    for k in range(T):
        for st in sts:
            st.columns(k)
        ex = [st.exchange() for st in sts]
        tot = torch.stack([e[0] for e in ex]).sum(0)
        mn = torch.stack([e[1] for e in ex]).min(0).values
        for e in ex:
            e[0].copy_(tot)
            e[1].copy_(mn)
        for st in sts:
            st.factor(k)
    res = [st.result() for st in sts]
    x = np.concatenate([r["x"].cpu().numpy() for r in res])
    return x, res


@pytest.mark.parametrize("nshard", [2, 4])
def test_c4_column_sharded_steppers_match_reference(cuda_device, golden_baseline, nshard):
    """BASELINE c4 (N = 100,000, L = 256, T = 50) solved as 2 / 4 column shards with the
    exchange reduced by hand: every shard's replicated factorisation sees the same
    reduced increment, and the assembled estimate matches the reference at 1e-9."""
    from paper_2503_15259_b200 import scenes
    cfg = scenes.BASELINE_CONFIGS["c4"]
    s = scenes.make_scene(cfg, 0)
    steps = orc.default_steps(cfg.n_iter)
    x, res = _run_shards("ml-k", s.pilots, s.gains, s.emp_cov, cfg.n_antennas, steps,
                         cfg.n_iter, nshard)
    assert all(r["status"] == 0 and r["n_iter"] == cfg.n_iter for r in res)
    for r in res[1:]:   # replicated scalars agree bitwise across shards
        np.testing.assert_array_equal(r["update_norm"].cpu().numpy(),
                                      res[0]["update_norm"].cpu().numpy())
    assert max_rel(x, golden_baseline["c4_i0_final"]) <= 1e-9
    assert max_rel(res[0]["update_norm"].cpu().numpy(),
                   golden_baseline["c4_i0_update_norm"]) <= 1e-8


def test_sharded_map_ur_objective_sums_prior_over_shards(cuda_device):
    """map-ur with the objective recorded: each shard's prior penalty rides in the summed
    exchange block, so the sharded objective equals the one-shard objective."""
    from paper_2503_15259_b200 import scenes
    from paper_2503_15259_b200.large import psca_run_large
    cfg = scenes.SceneConfig(3, "map-ur", 600, 160, 128, 30, 12, 1)
    s = scenes.make_scene(cfg, 5)
    prior = scenes.problem_for(cfg).prior
    steps = orc.default_steps(12)
    p = np.full(cfg.n_devices, float(np.asarray(prior.p).ravel()[0]))
    one = psca_run_large("map-ur", s.pilots, None, s.emp_cov, 1.0, cfg.n_antennas, steps,
                         max_iter=12, prior_p=p, eff_prior=prior, record_objective=True)
    x, res = _run_shards("map-ur", s.pilots, None, s.emp_cov, cfg.n_antennas, steps, 12, 3,
                         prior_p=p, eff_prior=prior, record_objective=True)
    assert max_rel(x, one["x"].cpu().numpy()) <= 1e-10
    for r in res:
        assert max_rel(r["objective"].cpu().numpy(), one["objective"].cpu().numpy()) <= 1e-12


def test_sharded_driver_stops_without_per_iteration_sync(cuda_device):
    """tol stop: the driver checks the device flag every 8 iterations; the gated kernels
    leave the stopped state untouched, so the result equals the reference's early stop."""
    from paper_2503_15259_b200 import scenes
    from paper_2503_15259_b200.large import GpuLargeStepper, ShardedDriver
    cfg = scenes.SceneConfig(3, "ml-ud", 500, 136, 96, 25, 40, 1)
    s = scenes.make_scene(cfg, 2)
    steps = orc.default_steps(40)
    ref = orc.psca("ml-ud", s.pilots, s.gains, s.emp_cov, 1.0, 96, steps, 40, tol=20.0)
    st = GpuLargeStepper("ml-ud", s.pilots, None, s.emp_cov, 1.0, 96, steps, max_iter=40,
                         tol=20.0)
    res = ShardedDriver(st, check_every=8).run(40)
    assert res["n_iter"] == len(ref["update_norm"]) < 40
    assert max_rel(res["x"].cpu().numpy(), ref["final"]) <= 1e-9
