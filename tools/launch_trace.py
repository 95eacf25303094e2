"""Per-iteration launch times of one serialised solve (experiment driver).

usage: [AB_LIB=variant.so] [AB_CONFIG=c1] [AB_BATCH=4096] [AB_ITERS=100] python tools/launch_trace.py
Prints, for selected iterations, the device ms of the column launch and of the
factor launches that follow it (sweep, products on the warp factor path).
"""
import json, os, sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_2503_15259_b200 import device
if os.environ.get("AB_LIB"):
    device.LIB_PATH = pathlib.Path(os.environ["AB_LIB"]).resolve()
import torch
import bench
from paper_2503_15259_b200 import estimators, scenes
name, nb, T = os.environ.get("AB_CONFIG", "c1"), int(os.environ.get("AB_BATCH", "4096")), int(os.environ.get("AB_ITERS", "100"))
cfg = scenes.BASELINE_CONFIGS[name]
host = bench.generate(name, list(range(nb)), 16)
dev = torch.device("cuda", 0)
p, e, n, g = (torch.from_numpy(host[k]).to(dev) for k in ("pilots", "emp_cov", "noise", "gains"))
prob = scenes.problem_for(cfg)
run = lambda out: estimators.psca_run_batch(prob, p, e, n, cfg.n_antennas, gains=g, max_iter=T, out=out)
out = run({})
torch.cuda.synchronize()
device.set_serial(True)
device.profile_begin()
run({})
recs = device.profile_launches()
device.profile_end()
device.set_serial(False)
col = [ms for k, ms in recs if k == 0]
fr = [ms for k, ms in recs if k == 1]
pg = [ms for k, ms in recs if k == 2]   # prior_grad_kernel launches
sweep, prod = fr[0::2], fr[1::2]
rows = []
for k in (0, 1, 2, 3, 5, 8, 12, 20, 30, 50, 70, 99):
    if k < len(col):
        rows.append({"k": k, "col_ms": round(col[k], 4), "sweep_after_ms": round(sweep[k + 1], 4) if k + 1 < len(sweep) else None,
                     "prod_after_ms": round(prod[k + 1], 4) if k + 1 < len(prod) else None})
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("PSCA_")}, "col_mean": sum(col) / len(col),
                  "sweep_mean": sum(sweep) / len(sweep), "prod_mean": sum(prod) / max(len(prod), 1), "prior_mean": sum(pg) / max(len(pg), 1), "rows": rows}))
