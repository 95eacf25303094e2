"""c0 latency: one N=1000, L=40, M=64 ml-k instance, T=100 (BASELINE configs[0])."""
import json, sys, time
sys.path.insert(0, ".")
import torch
import __graft_entry__
if len(sys.argv) > 1:   # A/B: time an alternative build of _psca.so
    import pathlib
    from paper_2503_15259_b200 import device
    device.LIB_PATH = pathlib.Path(sys.argv[1]).resolve()
else:
    __graft_entry__.build()
from paper_2503_15259_b200 import estimators, scenes
cfg = scenes.BASELINE_CONFIGS["c0"]
s = scenes.make_scene(cfg, 0)
b = scenes.stack_batch([s])
dev = torch.device("cuda", 0)
args = [torch.from_numpy(b[k]).to(dev) for k in ("pilots", "emp_cov", "noise", "gains")]
prob = scenes.problem_for(cfg)
out = {}
for _ in range(5):
    out = estimators.psca_run_batch(prob, args[0], args[1], args[2], 64, gains=args[3], max_iter=100, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
R = 20
for _ in range(R):
    out = estimators.psca_run_batch(prob, args[0], args[1], args[2], 64, gains=args[3], max_iter=100, out=out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / R
t0 = time.perf_counter()
tr = estimators.psca_run(prob, s, estimators.StepSchedule.default(), max_iter=100, tol=0.0, record_objective=False)
wall = time.perf_counter() - t0
print(json.dumps({"lib": sys.argv[1] if len(sys.argv) > 1 else "in-tree", "c0_device_ms_per_solve": ms, "us_per_iteration": ms * 10, "launches": out["launches"],
                  "psca_run_wall_ms": wall * 1e3}))
