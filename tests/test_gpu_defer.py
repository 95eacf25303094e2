"""The batched warp-factor path against the CTA factor path and the oracle.

Batches of at least one instance per SM (B >= 148) with L <= 40 run the
warp-per-instance factor sweep (fac_sweep_w) with the deferred covariance
rebuild (the factor warp sums the short moving-column lists the column kernel
leaves) and, for map-ur / pairwise map-k without objective recording, the
full-grid prior-gradient kernel (prior_grad_kernel).  Small batches of the same
instances run factor_solve_t (one CTA per instance) with the rebuild in the
column CTA.  Same iteration, different summation orders: rounding-level
agreement.  Shapes cover L not a multiple of 4 (zero-filled gather rows), odd L
(identity padding pivot), every kind, the pairwise prior, a tol stop, lists
longer than the deferral capacity and the PSCA_DEFER_REBUILD=0 /
PSCA_PRIOR_KERNEL=0 switches.
"""

import json
import os
import pathlib
import subprocess
import sys

import numpy as np
import pytest

from psca_testutil import max_rel

pytestmark = pytest.mark.gpu
ROOT = pathlib.Path(__file__).resolve().parent.parent
REPS = 40          # 4 scenes x 40 = 160 instances >= 148 SMs

CASES = [(40, "ml-ud", 300), (33, "map-k", 300), (20, "map-ur", 300), (38, "ml-k", 300),
         (17, "map-ur", 260), (24, "ml-ud", 200), (8, "ml-k", 120), (12, "map-k", 150)]


def _scenes(L, kind, N, n_active=15):
    from paper_2503_15259_b200 import scenes
    cfg = scenes.SceneConfig(11, kind, N, L, 64, n_active, 25, 4)
    return cfg, scenes.stack_batch([scenes.make_scene(cfg, i) for i in range(4)])


def _tile(b, reps):
    return {k: (np.tile(v, (reps,) + (1,) * (v.ndim - 1)) if v is not None else None)
            for k, v in b.items() if k in ("pilots", "emp_cov", "noise", "gains")}


@pytest.mark.parametrize("L,kind,N", CASES)
def test_warp_factor_path_matches_cta_factor_path(cuda_device, L, kind, N):
    from paper_2503_15259_b200 import estimators, scenes
    cfg, b = _scenes(L, kind, N)
    prob = scenes.problem_for(cfg)
    big_in = _tile(b, REPS)
    tol = 1e-7 if kind == "map-ur" else 1e-10
    for rec in (False, True):   # False: prior_grad_kernel; True: in-kernel prior + penalty value
        small = estimators.psca_run_batch(prob, b["pilots"], b["emp_cov"], b["noise"], 64,
                                          gains=b["gains"], max_iter=25, n_chunks=1,
                                          record_objective=rec)
        big = estimators.psca_run_batch(prob, big_in["pilots"], big_in["emp_cov"], big_in["noise"],
                                        64, gains=big_in["gains"], max_iter=25,
                                        record_objective=rec)
        xs, xb = small["x"].cpu().numpy(), big["x"].cpu().numpy()
        assert xb.shape == (4 * REPS, N)
        for r in (0, 1, REPS // 2, REPS - 1):
            assert max_rel(xb[4 * r:4 * r + 4], xs) <= tol, (L, kind, rec, r)
        # replicas of one instance take the same path: bit-identical
        np.testing.assert_array_equal(xb[:4], xb[-4:])
        un_s, un_b = small["update_norm"].cpu().numpy(), big["update_norm"].cpu().numpy()
        assert max_rel(un_b[:4], un_s) <= (1e-5 if kind == "map-ur" else 1e-8)
        if rec:
            assert max_rel(big["objective"].cpu().numpy()[:4],
                           small["objective"].cpu().numpy()) <= (1e-7 if kind == "map-ur" else 1e-10)


def test_warp_factor_path_matches_oracle(cuda_device):
    """The deferred path against the CPU oracle directly (ml-ud and map-k, L = 30)."""
    from oracle import psca_oracle as orc
    from paper_2503_15259_b200 import estimators, scenes
    for kind in ("ml-ud", "map-k"):
        cfg, b = _scenes(30, kind, 220)
        prob = scenes.problem_for(cfg)
        big_in = _tile(b, REPS)
        big = estimators.psca_run_batch(prob, big_in["pilots"], big_in["emp_cov"], big_in["noise"],
                                        64, gains=big_in["gains"], max_iter=25)
        xb = big["x"].cpu().numpy()
        steps = orc.default_steps(25)
        kw = {}
        if kind == "map-k":
            kw["indep_p"] = np.full(220, cfg.p)
        for i in range(4):
            ref = orc.psca(kind, b["pilots"][i], b["gains"][i], b["emp_cov"][i], 1.0, 64, steps,
                           25, **kw)["final"]
            assert max_rel(xb[4 * (REPS - 1) + i], ref) <= 1e-9, (kind, i)


def test_pairwise_prior_and_tol_stop_on_warp_factor_path(cuda_device):
    from paper_2503_15259_b200 import device, estimators, priors, scenes
    cfg, b = _scenes(24, "ml-ud", 240, n_active=12)
    big_in = _tile(b, REPS)
    steps = estimators.default_steps(15)
    pr = priors.PairwiseMvbPrior.from_group_model(240, 4, 0.1)
    c1 = np.broadcast_to(pr.c1, (240,)).astype(float)
    un = device.solve("ml-k", b["pilots"], b["emp_cov"], b["noise"], 64, steps, gains=b["gains"],
                      max_iter=15)["update_norm"].cpu().numpy()
    cases = {
        "pairwise": dict(kind="map-k", prior_c1=c1, prior_c2=pr.csr_arrays()),
        "tol": dict(kind="ml-k", tol=float(np.median(un[:, 6]))),
    }
    for name, kw in cases.items():
        kind = kw.pop("kind")
        small = device.solve(kind, b["pilots"], b["emp_cov"], b["noise"], 64, steps,
                             gains=b["gains"], max_iter=15, n_chunks=1, **kw)
        big = device.solve(kind, big_in["pilots"], big_in["emp_cov"], big_in["noise"], 64, steps,
                           gains=big_in["gains"], max_iter=15, **kw)
        assert max_rel(big["x"].cpu().numpy()[-4:], small["x"].cpu().numpy()) <= 1e-10, name
        np.testing.assert_array_equal(big["n_iter"].cpu().numpy()[-4:],
                                      small["n_iter"].cpu().numpy(), err_msg=name)
        np.testing.assert_array_equal(big["status"].cpu().numpy()[-4:],
                                      small["status"].cpu().numpy(), err_msg=name)
    assert int(small["n_iter"].min()) < 15   # the tol case stopped early


SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2503_15259_b200 import device, estimators, scenes
out = {}
# many active devices: the moving lists straddle the deferral capacity (160),
# so some instance-iterations are deferred and others rebuilt by the column CTA
for L, kind, N, K in ((40, "map-k", 1200, 260), (20, "map-ur", 900, 170), (36, "ml-k", 1000, 220)):
    cfg = scenes.SceneConfig(13, kind, N, L, 64, K, 20, 4)
    b = scenes.stack_batch([scenes.make_scene(cfg, i) for i in range(4)])
    t = lambda v: np.tile(v, (40,) + (1,) * (v.ndim - 1))
    prob = scenes.problem_for(cfg)
    steps = estimators.default_steps(20)
    res = device.solve(kind, t(b["pilots"]), t(b["emp_cov"]), t(b["noise"]), 64, steps,
                       gains=t(b["gains"]) if prob.known_pathloss else None, max_iter=20,
                       record_iterates=True, **estimators.prior_arrays(prob, N, 64))
    its = res["iterates"].cpu().numpy()[:4]
    moving = [[int(np.count_nonzero(its[i, k + 1] != (1.0 - steps[k]) * its[i, k]))
               for k in range(20)] for i in range(4)]
    out[f"{L}-{kind}"] = {"x": res["x"].cpu().numpy()[:8].tolist(), "path": res["path"],
                          "un": res["update_norm"].cpu().numpy()[:8].tolist(), "moving": moving}
print(json.dumps(out))
"""


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    p = subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT)], env=env, capture_output=True,
                       text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-2000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


def test_deferral_switches_and_capacity_boundary(cuda_device):
    """Default (deferred rebuild + prior kernel) against PSCA_DEFER_REBUILD=0 and
    PSCA_PRIOR_KERNEL=0 on scenes whose moving lists fall on both sides of the
    160-entry capacity."""
    on = _run({})
    off = _run({"PSCA_DEFER_REBUILD": "0", "PSCA_PRIOR_KERNEL": "0"})
    straddle, seen = False, {}
    for key in on:
        mv = np.array(on[key]["moving"])[:, 1:]
        seen[key] = (int(mv.min()), int(mv.max()))
        straddle |= bool((mv > 160).any() and (mv <= 160).any())
        tol = 1e-7 if "map-ur" in key else 1e-10
        assert max_rel(np.array(on[key]["x"]), np.array(off[key]["x"])) <= tol, key
        assert max_rel(np.array(on[key]["un"]), np.array(off[key]["un"])) <= 1e-5, key
    assert straddle, f"no case had lists on both sides of the capacity: {seen}"
