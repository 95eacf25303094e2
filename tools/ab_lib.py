"""A/B timing of alternative builds of _psca.so (experiment driver).

usage: python tools/ab_lib.py lib1.so lib2.so ...
c1 workload (2048 instances, 30 iterations); each library is loaded by pointing
device.LIB_PATH at it before the first load; prints per-launch device ms of the
column and factor kernels scaled to 4096 instances.
"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, json
sys.path.insert(0, sys.argv[1])
from paper_2503_15259_b200 import device
import pathlib
device.LIB_PATH = pathlib.Path(sys.argv[2])
import torch
from paper_2503_15259_b200 import estimators, scenes
cfg = scenes.BASELINE_CONFIGS["c1"]
import bench
host = bench.generate("c1", list(range(2048)), 16)
dev = torch.device("cuda", 0)
p, e, n = (torch.from_numpy(host[k]).to(dev) for k in ("pilots", "emp_cov", "noise"))
prob = scenes.problem_for(cfg)
out = {}
for _ in range(2):
    out = estimators.psca_run_batch(prob, p, e, n, 128, max_iter=30, out=out)
torch.cuda.synchronize()
device.profile_begin()
for _ in range(3):
    out = estimators.psca_run_batch(prob, p, e, n, 128, max_iter=30, out=out)
torch.cuda.synchronize()
pr = device.profile_end()
print(json.dumps({"lib": sys.argv[2], "col_ms": pr["column_ms"] / pr["column_launches"] * 2,
                  "fac_ms": pr["factor_ms"] / max(pr["factor_launches"], 1) * 2}))
'''
for lib in sys.argv[1:]:
    env = dict(os.environ)
    r = subprocess.run([sys.executable, "-c", CODE, ROOT, os.path.abspath(lib)], env=env,
                       capture_output=True, text=True, cwd=ROOT)
    print(r.stdout.strip() or r.stderr[-800:])
