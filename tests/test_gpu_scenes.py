"""Scene covariances on the FP64 tensor pipe.

The random draws stay on the host (one Philox stream per instance, the scene
contract); Y = S_A diag(sqrt(g_A)) H + Z (psca_received) and
Sigma_hat = Y Y^H / M (psca_empirical_cov, DMMA) run on the GPU and are
checked against the host arithmetic of ``scenes.make_scene`` -- the generator
the golden fixtures were produced with (make_golden.py) -- at 1e-13.
"""

import numpy as np
import pytest

from psca_testutil import max_rel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,ids", [("c0", [0, 1]), ("c1", list(range(6))),
                                      ("c3_l20", [3, 4]), ("c3_l80", [0, 7]), ("c4", [0])])
def test_device_scene_batch_matches_host_generator(cuda_device, name, ids):
    from paper_2503_15259_b200 import scenes
    cfg = scenes.BASELINE_CONFIGS[name]
    dev = scenes.make_batch_device(cfg, ids)
    E = dev["emp_cov"].cpu().numpy()
    Y = dev["received"].cpu().numpy()
    for k, i in enumerate(ids):
        s = scenes.make_scene(cfg, i)
        assert max_rel(Y[k], s.received) <= 1e-13
        assert max_rel(E[k], s.emp_cov) <= 1e-13
        np.testing.assert_array_equal(E[k], E[k].conj().T)           # exactly Hermitian
        np.testing.assert_array_equal(dev["activities"][k], s.activities)
        np.testing.assert_array_equal(dev["pilots"][k].cpu().numpy(), s.pilots)


def test_device_scene_batch_solves_like_the_host_batch(cuda_device, golden_baseline):
    """A c1 batch built on the device solves to the reference outputs (golden_baseline)."""
    from paper_2503_15259_b200 import estimators, scenes
    cfg = scenes.BASELINE_CONFIGS["c1"]
    dev = scenes.make_batch_device(cfg, [0, 1])
    res = estimators.psca_run_batch(scenes.problem_for(cfg), dev["pilots"], dev["emp_cov"],
                                    dev["noise"], cfg.n_antennas, max_iter=cfg.n_iter)
    x = res["x"].cpu().numpy()
    for k in range(2):
        assert max_rel(x[k], golden_baseline[f"c1_i{k}_final"]) <= 1e-9


def test_empirical_cov_ragged_shapes(cuda_device):
    """Odd L, M (partial tiles) and M < L (a singular Sigma_hat)."""
    from paper_2503_15259_b200 import sysmodel
    rng = np.random.default_rng(4)
    for (L, M) in [(5, 3), (33, 40), (13, 7), (1, 9), (80, 128)]:
        y = rng.standard_normal((3, L, M)) + 1j * rng.standard_normal((3, L, M))
        got = sysmodel.empirical_cov(y, M)
        for b in range(3):
            ref = (y[b] @ y[b].conj().T) / M
            assert max_rel(got[b], ref) <= 1e-13
