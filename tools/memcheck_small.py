"""Small solve for compute-sanitizer (one tool per run; see B200_PROFILING.md)."""
import sys
sys.path.insert(0, ".")
import __graft_entry__
__graft_entry__.build()
from paper_2503_15259_b200 import estimators, scenes
for L, kind in ((40, "ml-ud"), (20, "map-ur"), (72, "map-k"), (33, "ml-k")):
    cfg = scenes.SceneConfig(7, kind, 100, L, 64, 10, 4, 2)
    ss = [scenes.make_scene(cfg, i) for i in range(2)]
    b = scenes.stack_batch(ss)
    for nck in (0, 1):   # chunked (tile column kernel) and one chunk (warp-streamed)
        res = estimators.psca_run_batch(scenes.problem_for(cfg), b["pilots"], b["emp_cov"], b["noise"],
                                        64, gains=b["gains"], max_iter=4, record_objective=True,
                                        n_chunks=nck)
        print(L, kind, nck, float(res["x"].sum()))

# the batched warp-factor path (B >= SM count): deferred rebuild, prior-gradient
# kernel, the column kernel's cp.async landing zone
import numpy as np
for L, kind in ((40, "ml-ud"), (18, "map-ur"), (33, "map-k")):
    cfg = scenes.SceneConfig(7, kind, 100, L, 64, 10, 4, 2)
    b = scenes.stack_batch([scenes.make_scene(cfg, i) for i in range(2)])
    t = lambda v: np.tile(v, (80,) + (1,) * (v.ndim - 1))
    res = estimators.psca_run_batch(scenes.problem_for(cfg), t(b["pilots"]), t(b["emp_cov"]), t(b["noise"]),
                                    64, gains=t(b["gains"]), max_iter=4)
    print(L, kind, "B=160", float(res["x"].sum()), res["path"])
