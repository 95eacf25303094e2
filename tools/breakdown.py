"""Per-kernel breakdown of one batched solve (experiment driver).

usage: [BD_CONFIG=c1] [BD_BATCH=4096] [BD_ITERS=30] python tools/breakdown.py
Prints device ms per solve, ms per iteration, and the mean CUDA-event duration
of the column and factor launches (psca_profile_begin/end).  Run it under
different PSCA_* environment settings (PSCA_NO_SPLIT=1, ...) to compare paths.
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__
__graft_entry__.build()
import bench
from paper_2503_15259_b200 import device, estimators, scenes

name = os.environ.get("BD_CONFIG", "c1")
cfg = scenes.BASELINE_CONFIGS[name]
B = int(os.environ.get("BD_BATCH", cfg.batch))
T = int(os.environ.get("BD_ITERS", "30"))
host = bench.generate(name, list(range(B)), os.cpu_count() or 1)
dev = torch.device("cuda", 0)
P, E, Nz, G = (torch.from_numpy(host[k]).to(dev) for k in ("pilots", "emp_cov", "noise", "gains"))
prob = scenes.problem_for(cfg)
out = {}


def run():
    global out
    out = estimators.psca_run_batch(prob, P, E, Nz, cfg.n_antennas, gains=G, max_iter=T, out=out)


for _ in range(2):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
R = 3
e0.record()
for _ in range(R):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / R
device.profile_begin()
run()
torch.cuda.synchronize()
p = device.profile_end()
env = {k: v for k, v in os.environ.items() if k.startswith("PSCA_")}
print(json.dumps({"config": name, "B": B, "T": T, "env": env, "ms_per_solve": round(ms, 3),
                  "ms_per_iter": round(ms / T, 4), "inst_per_s_T100": round(B / (ms / T * 100) * 1e3, 1),
                  "col_ms_per_launch": round(p["column_ms"] / max(1, p["column_launches"]), 4),
                  "col_launches": p["column_launches"],
                  "fac_ms_per_launch": round(p["factor_ms"] / max(1, p["factor_launches"]), 4),
                  "fac_launches": p["factor_launches"], "path": device.load().psca_last_path()}))
