"""A/B timing of alternative builds of _psca.so (experiment driver).

usage: [AB_CONFIG=c1] [AB_BATCH=2048] [AB_ITERS=30] python tools/ab_lib.py lib1.so lib2.so ...
BASELINE workload AB_CONFIG (AB_BATCH instances, AB_ITERS iterations); each library
is loaded by pointing device.LIB_PATH at it before the first load; prints
ms per solve (default launch schedule) and the mean per-launch
device ms of the column kernel and of the even / odd factor launches (sweep /
products on the warp factor path) of one serialised solve.
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
name, nb, T = sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
cfg = scenes.BASELINE_CONFIGS[name]
import bench
host = bench.generate(name, list(range(nb)), 16)
dev = torch.device("cuda", 0)
p, e, n, g = (torch.from_numpy(host[k]).to(dev) for k in ("pilots", "emp_cov", "noise", "gains"))
prob = scenes.problem_for(cfg)
out = {}
for _ in range(2):
    out = estimators.psca_run_batch(prob, p, e, n, cfg.n_antennas, gains=g, max_iter=T, out=out)
torch.cuda.synchronize()
device.profile_begin()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    out = estimators.psca_run_batch(prob, p, e, n, cfg.n_antennas, gains=g, max_iter=T, out=out)
e1.record()
torch.cuda.synchronize()
pr = device.profile_end()
# one serialised solve (every launch on one stream): per-launch times by kind;
# on the warp factor path the factor launches alternate sweep, products
device.set_serial(True)
device.profile_begin()
estimators.psca_run_batch(prob, p, e, n, cfg.n_antennas, gains=g, max_iter=T, out={})
recs = device.profile_launches()
device.profile_end()
device.set_serial(False)
col = [ms for k, ms in recs if k == 0]
fr = [ms for k, ms in recs if k == 1]
pg = [ms for k, ms in recs if k == 2]   # prior_grad_kernel launches
print(json.dumps({"lib": sys.argv[2], "ms_per_solve": e0.elapsed_time(e1) / 3,
                  "serial_col_ms": sum(col) / max(len(col), 1),
                  "serial_fac_even_ms": sum(fr[0::2]) / max(len(fr[0::2]), 1),
                  "serial_fac_odd_ms": sum(fr[1::2]) / max(len(fr[1::2]), 1),
                  "serial_prior_ms": sum(pg) / max(len(pg), 1),
                  "n_col": len(col), "n_fac": len(fr), "n_prior": len(pg)}))
'''
for lib in sys.argv[1:]:
    env = dict(os.environ)
    r = subprocess.run([sys.executable, "-c", CODE, ROOT, os.path.abspath(lib),
                        os.environ.get("AB_CONFIG", "c1"), os.environ.get("AB_BATCH", "2048"),
                        os.environ.get("AB_ITERS", "30")],
                       env=env,
                       capture_output=True, text=True, cwd=ROOT)
    print(r.stdout.strip() or r.stderr[-800:])
