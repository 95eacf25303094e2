"""The compiled-shape kernels and the generic runtime-shape kernels agree.

PSCA_GENERIC_COLUMN=1 forces the generic column/factor kernels (read once
per process), so the comparison runs the generic path in a subprocess.
Also covers shapes whose L is padded up to a compiled row-block count.
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

SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2503_15259_b200 import estimators, scenes
out = {}
for L, kind in ((40, "ml-ud"), (33, "map-k"), (20, "map-ur"), (52, "ml-k"), (72, "map-ur")):
    cfg = scenes.SceneConfig(7, kind, 300, L, 64, 15, 25, 3)
    ss = [scenes.make_scene(cfg, i) for i in range(3)]
    b = scenes.stack_batch(ss)
    res = estimators.psca_run_batch(scenes.problem_for(cfg), b["pilots"], b["emp_cov"], b["noise"],
                                    64, gains=b["gains"], max_iter=25, record_objective=True,
                                    n_chunks=1)
    out[f"{L}-{kind}"] = {"x": res["x"].cpu().numpy().tolist(), "path": res["path"],
                          "obj": res["objective"].cpu().numpy().tolist(),
                          "un": res["update_norm"].cpu().numpy().tolist()}
print(json.dumps(out))
"""


def run_script(env_extra):
    env = dict(os.environ, **env_extra)
    p = subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT)], env=env, capture_output=True,
                       text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


def test_generic_and_compiled_kernels_agree(cuda_device):
    fast = run_script({"PSCA_GENERIC_COLUMN": "0"})
    slow = run_script({"PSCA_GENERIC_COLUMN": "1"})
    for key in fast:
        xf, xs = np.array(fast[key]["x"]), np.array(slow[key]["x"])
        tol = 1e-9 if "map-ur" not in key else 1e-7
        assert max_rel(xf, xs) <= tol, key
        assert max_rel(np.array(fast[key]["obj"]), np.array(slow[key]["obj"])) <= 1e-10, key


def test_warp_streamed_and_tile_column_kernels_agree(cuda_device):
    """The warp-streamed column kernel (default, L <= 40) and the tile-pipelined one
    compute the same pass with different summation orders: rounding-level agreement."""
    warp = run_script({"PSCA_TILE_COLUMN": "0"})
    tile = run_script({"PSCA_TILE_COLUMN": "1"})
    for key in warp:
        xw, xt = np.array(warp[key]["x"]), np.array(tile[key]["x"])
        tol = 1e-10 if "map-ur" not in key else 1e-7
        assert max_rel(xw, xt) <= tol, key
        assert max_rel(np.array(warp[key]["obj"]), np.array(tile[key]["obj"])) <= 1e-11, key


def test_persistent_equals_two_kernel_bitwise(cuda_device):
    """One chunk per instance: the persistent kernel and the two-kernel path with the
    tile-pipelined column kernel run the same device functions, so the iterates are
    bit-identical."""
    pers = run_script({"PSCA_PERSISTENT": "1", "PSCA_TILE_COLUMN": "1"})
    two = run_script({"PSCA_PERSISTENT": "0", "PSCA_TILE_COLUMN": "1"})
    assert any(v["path"] == "persistent" for v in pers.values())
    assert all(v["path"] == "two-kernel" for v in two.values())
    for key in pers:
        for field in ("x", "un"):
            np.testing.assert_array_equal(np.array(pers[key][field]), np.array(two[key][field]),
                                          err_msg=f"{key} {field}")
        # the objective's trace / Frobenius reductions run over different CTA sizes
        assert max_rel(np.array(pers[key]["obj"]), np.array(two[key]["obj"])) <= 1e-13


def test_warp_kernel_options_match_tile_kernel(cuda_device):
    """Options the batch path exercises rarely, with one chunk per instance (the
    warp-streamed column kernel) against column chunks (the tile kernel): iterate
    recording, a pairwise MAP-K prior, and a tol stop."""
    from paper_2503_15259_b200 import device, estimators, priors, scenes
    cfg = scenes.SceneConfig(5, "ml-ud", 240, 24, 48, 12, 15, 4)
    ss = [scenes.make_scene(cfg, i) for i in range(4)]
    b = scenes.stack_batch(ss)
    steps = estimators.default_steps(15)
    pr = priors.PairwiseMvbPrior.from_group_model(240, 4, 0.1)
    c1 = np.broadcast_to(pr.c1, (240,)).astype(float)
    un = device.solve("ml-k", b["pilots"], b["emp_cov"], b["noise"], 48, steps, gains=b["gains"],
                      max_iter=15)["update_norm"].cpu().numpy()
    cases = {
        "iterates": dict(kind="ml-ud", record_iterates=True),
        "pairwise": dict(kind="map-k", gains=b["gains"], prior_c1=c1, prior_c2=pr.csr_arrays(),
                         record_objective=True),
        # stops some instances around iteration 6
        "tol": dict(kind="ml-k", gains=b["gains"], tol=float(np.median(un[:, 6]))),
    }
    for name, kw in cases.items():
        kind = kw.pop("kind")
        res = {}
        for nck in (1, 0):
            r = device.solve(kind, b["pilots"], b["emp_cov"], b["noise"], 48, steps, max_iter=15,
                             n_chunks=nck, **kw)
            res[nck] = {k: v.cpu().numpy() for k, v in r.items()
                        if k in ("x", "iterates", "objective", "n_iter", "status") and v is not None}
        assert max_rel(res[1]["x"], res[0]["x"]) <= 1e-10, name
        np.testing.assert_array_equal(res[1]["n_iter"], res[0]["n_iter"], err_msg=name)
        np.testing.assert_array_equal(res[1]["status"], res[0]["status"], err_msg=name)
        if "iterates" in res[0]:
            assert max_rel(res[1]["iterates"], res[0]["iterates"]) <= 1e-10, name
        if "objective" in res[0]:
            assert max_rel(res[1]["objective"], res[0]["objective"]) <= 1e-11, name
    assert int(res[0]["n_iter"].min()) < 15   # the tol case stopped early


CLUSTER_SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2503_15259_b200 import estimators, scenes
out = {}
for L, kind, B, tol in ((40, "ml-k", 1, 0.0), (33, "map-k", 3, 0.0), (20, "map-ur", 2, 0.0),
                        (52, "ml-ud", 1, 0.0), (72, "map-ur", 2, 0.0), (40, "ml-ud", 4, 1.0)):
    cfg = scenes.SceneConfig(11, kind, 600, L, 64, 20, 30, B)
    ss = [scenes.make_scene(cfg, i) for i in range(B)]
    b = scenes.stack_batch(ss)
    if tol > 0:   # a tol some instances reach mid-run: the 10th update norm of the first
        r0 = estimators.psca_run_batch(scenes.problem_for(cfg), b["pilots"], b["emp_cov"],
                                       b["noise"], 64, gains=b["gains"], max_iter=30)
        tol = float(r0["update_norm"].cpu().numpy()[0, 10])
    res = estimators.psca_run_batch(scenes.problem_for(cfg), b["pilots"], b["emp_cov"], b["noise"],
                                    64, gains=b["gains"], max_iter=30, tol=tol,
                                    record_objective=True)
    out[f"{L}-{kind}-{B}"] = {"x": res["x"].cpu().numpy().tolist(),
                              "obj": res["objective"].cpu().numpy().tolist(),
                              "un": res["update_norm"].cpu().numpy().tolist(),
                              "n_iter": res["n_iter"].cpu().numpy().tolist(),
                              "status": res["status"].cpu().numpy().tolist()}
print(json.dumps(out))
"""


def test_cluster_factor_equals_single_cta_factor_bitwise(cuda_device):
    """Few instances: the factor stage on a cluster of eight CTAs (factor_cluster_t:
    chunk partials summed by slices, the sweep on CTA 0, the products by column
    tiles) against one wide CTA per instance (PSCA_FAC_CLUSTER=0).  Same summation
    orders in every phase, so iterates, update norms, objectives, stop iterations
    and statuses are bit-identical (only the Frobenius norm of the q-floor guard
    is summed in another order)."""
    env = dict(os.environ)

    def run(extra):
        p = subprocess.run([sys.executable, "-c", CLUSTER_SCRIPT, str(ROOT)],
                           env=dict(env, **extra), capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        return json.loads(p.stdout.strip().splitlines()[-1])

    clus = run({"PSCA_FAC_CLUSTER": "1"})
    one = run({"PSCA_FAC_CLUSTER": "0"})
    assert any(min(v["n_iter"]) < 30 for v in clus.values())   # the tol stop is exercised
    for key in clus:
        for field in ("x", "un", "obj", "n_iter", "status"):
            np.testing.assert_array_equal(np.array(clus[key][field]), np.array(one[key][field]),
                                          err_msg=f"{key} {field}")


FAIL_SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2503_15259_b200 import estimators, scenes
cfg = scenes.SceneConfig(13, "ml-ud", 400, 24, 32, 12, 12, 3)
ss = [scenes.make_scene(cfg, i) for i in range(3)]
b = scenes.stack_batch(ss)
b["pilots"][1, 3, 7] = np.nan          # instance 1: Sigma is NaN from the second factorisation on
res = estimators.psca_run_batch(scenes.problem_for(cfg), b["pilots"], b["emp_cov"], b["noise"],
                                32, gains=b["gains"], max_iter=12)
x = res["x"].cpu().numpy()
print(json.dumps({"status": res["status"].cpu().numpy().tolist(),
                  "n_iter": res["n_iter"].cpu().numpy().tolist(),
                  "x0": x[0].tolist(), "x2": x[2].tolist()}))
"""


def test_cluster_factor_pivot_failure_stops_only_that_instance(cuda_device):
    """A sweep that meets a non-positive pivot on CTA 0 must release the other seven
    CTAs of its cluster (outcome flag + barrier) and freeze that instance only."""
    def run(extra):
        p = subprocess.run([sys.executable, "-c", FAIL_SCRIPT, str(ROOT)],
                           env=dict(os.environ, **extra), capture_output=True, text=True,
                           timeout=180)
        assert p.returncode == 0, p.stderr[-2000:]
        return json.loads(p.stdout.strip().splitlines()[-1])

    clus = run({"PSCA_FAC_CLUSTER": "1"})
    one = run({"PSCA_FAC_CLUSTER": "0"})
    assert clus["status"][1] == 1 and clus["n_iter"][1] < 12      # PSCA_CHOL_FAIL, stopped early
    assert clus["status"][0] == 0 and clus["status"][2] == 0 and clus["n_iter"][0] == 12
    assert clus == one
