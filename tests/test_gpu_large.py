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
