"""clock64 phase probes of the factor kernel (experiment driver).

usage: python tools/probe_factor.py lib_built_with_-DPSCA_PROBE=1.so [config] [batch]
Runs one batched solve (30 iterations) and prints the cycle deltas between the
PROBE points of block 0 of the LAST factor launch (factor_solve_t):
0 start, 1 finalize, 2 prior terms, 3 assembly, 4 Frobenius norm, 5 sweep,
6 P write + trace, 7 Sigma_hat wait, 8 G = Sigma_hat P, 9 A = P G + pack.
"""
import ctypes, json, pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_2503_15259_b200 import device
device.LIB_PATH = pathlib.Path(sys.argv[1]).resolve()
import torch
import bench
from paper_2503_15259_b200 import estimators, scenes
name = sys.argv[2] if len(sys.argv) > 2 else "c0"
cfg = scenes.BASELINE_CONFIGS[name]
B = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.batch
host = bench.generate(name, list(range(B)), 16)
dev = torch.device("cuda", 0)
p, e, n, g = (torch.from_numpy(host[k]).to(dev) for k in ("pilots", "emp_cov", "noise", "gains"))
prob = scenes.problem_for(cfg)
lib = device.load()
lib.psca_debug_probes.argtypes = [ctypes.POINTER(ctypes.c_longlong), ctypes.c_int]
out = {}
res = []
for rep in range(3):
    out = estimators.psca_run_batch(prob, p, e, n, cfg.n_antennas, gains=g, max_iter=30, out=out)
    torch.cuda.synchronize()
    buf = (ctypes.c_longlong * 32)()
    lib.psca_debug_probes(buf, 32)
    v = list(buf)[:32]
    res.append([v[i + 1] - v[i] for i in range(9)] + [v[9] - v[0]] +
               [v[i + 1] - v[i] for i in range(10, 29)])
names = ["finalize", "prior", "assembly", "frob", "sweep", "P+trace", "emp_wait", "G", "A+pack",
         "total"] + [f"step{i}" for i in range(19)]
print(json.dumps({"raw_10_24": [v[i] - v[10] for i in range(10, 24)]}))
print(json.dumps({"config": name, "B": B, "lib": sys.argv[1],
                  "cycles": {k: res[-1][i] for i, k in enumerate(names)}}))
