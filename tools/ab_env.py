"""A/B timing of one build under different PSCA_* environment settings.

usage: [AB_CONFIG=c1] [AB_BATCH=4096] python tools/ab_env.py "PSCA_FAC_WARP=0" "" ...
Each argument is a space-separated list of NAME=VALUE settings (empty = default);
prints ms per solve (30 iterations) and the per-iteration column / factor launch
times of one serialised solve.
"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, json
sys.path.insert(0, sys.argv[1])
import torch
import bench
from paper_2503_15259_b200 import device, estimators, scenes
name, nb = sys.argv[2], int(sys.argv[3])
cfg = scenes.BASELINE_CONFIGS[name]
host = bench.generate(name, list(range(nb)), 16)
dev = torch.device("cuda", 0)
p, e, n, g = (torch.from_numpy(host[k]).to(dev) for k in ("pilots", "emp_cov", "noise", "gains"))
prob = scenes.problem_for(cfg)
T = 30
run = lambda out: estimators.psca_run_batch(prob, p, e, n, cfg.n_antennas, gains=g, max_iter=T, out=out)
out = {}
for _ in range(2):
    out = run(out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    out = run(out)
e1.record()
torch.cuda.synchronize()
device.set_serial(True)
device.profile_begin()
run({})
recs = device.profile_launches()
device.profile_end()
device.set_serial(False)
col = sum(ms for k, ms in recs if k == 0)
fac = sum(ms for k, ms in recs if k != 0)
fr = [ms for k, ms in recs if k == 1]
pg = [ms for k, ms in recs if k == 2]   # prior_grad_kernel launches
# warp factor path: per iteration a sweep launch then a product launch
fac_even, fac_odd = sum(fr[0::2]), sum(fr[1::2])
print(json.dumps({"env": sys.argv[4], "ms_per_solve_30it": e0.elapsed_time(e1) / 3,
                  "col_ms_per_iter": col / T, "fac_ms_per_iter": fac / T,
                  "fac_launches": len(fr), "fac_even_ms_per_iter": fac_even / T,
                  "fac_odd_ms_per_iter": fac_odd / T,
                  "x_sum": float(out["x"].sum())}))
'''
for spec in sys.argv[1:]:
    env = dict(os.environ)
    for kv in spec.split():
        k, v = kv.split("=", 1)
        env[k] = v
    r = subprocess.run([sys.executable, "-c", CODE, ROOT, os.environ.get("AB_CONFIG", "c1"),
                        os.environ.get("AB_BATCH", "4096"), spec], env=env,
                       capture_output=True, text=True, cwd=ROOT)
    print(r.stdout.strip() or r.stderr[-1500:])
