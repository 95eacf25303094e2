"""A/B timing of alternative builds of _psca.so (experiment driver).

usage: [AB_CONFIG=c1] [AB_BATCH=2048] python tools/ab_lib.py lib1.so lib2.so ...
BASELINE workload AB_CONFIG (AB_BATCH instances, 30 iterations); each library
is loaded by pointing device.LIB_PATH at it before the first load; prints
per-launch device ms of the column and factor kernels and ms per solve
(scaled to 2 x AB_BATCH instances, as the split-stream halves of a full batch).
Build variants with e.g.
  nvcc <__graft_entry__.NVCC_FLAGS> -DPSCA_FAC_WIDE=128 -o /tmp/v.so csrc/psca.cu
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
name, nb = sys.argv[3], int(sys.argv[4])
cfg = scenes.BASELINE_CONFIGS[name]
import bench
host = bench.generate(name, list(range(nb)), 16)
dev = torch.device("cuda", 0)
p, e, n, g = (torch.from_numpy(host[k]).to(dev) for k in ("pilots", "emp_cov", "noise", "gains"))
prob = scenes.problem_for(cfg)
out = {}
for _ in range(2):
    out = estimators.psca_run_batch(prob, p, e, n, cfg.n_antennas, gains=g, max_iter=30, out=out)
torch.cuda.synchronize()
device.profile_begin()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    out = estimators.psca_run_batch(prob, p, e, n, cfg.n_antennas, gains=g, max_iter=30, out=out)
e1.record()
torch.cuda.synchronize()
pr = device.profile_end()
print(json.dumps({"lib": sys.argv[2], "col_ms": pr["column_ms"] / pr["column_launches"] * 2,
                  "fac_ms": pr["factor_ms"] / max(pr["factor_launches"], 1) * 2,
                  "ms_per_solve_30it": e0.elapsed_time(e1) / 3}))
'''
for lib in sys.argv[1:]:
    env = dict(os.environ)
    r = subprocess.run([sys.executable, "-c", CODE, ROOT, os.path.abspath(lib),
                        os.environ.get("AB_CONFIG", "c1"), os.environ.get("AB_BATCH", "2048")],
                       env=env,
                       capture_output=True, text=True, cwd=ROOT)
    print(r.stdout.strip() or r.stderr[-800:])
