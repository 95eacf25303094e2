"""Device time of a c1 solve cut into sub-batches (experiment driver): how much of
the end-to-end gap of psca_run_batch_host is the small chunks' lower efficiency.

usage: python tools/chunk_cost.py
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2503_15259_b200 import device, estimators, scenes

cfg = scenes.BASELINE_CONFIGS["c1"]
B, T = 4096, 100
host = bench.generate("c1", list(range(B)), os.cpu_count() or 1)
dev = {k: torch.from_numpy(host[k]).cuda() for k in ("pilots", "emp_cov", "noise", "gains")}
prob = scenes.problem_for(cfg)
w = 2 * device.sm_count()


def run(lo, hi, out):
    nck = 1 if hi - lo >= 2 * device.sm_count() else 0
    return estimators.psca_run_batch(prob, dev["pilots"][lo:hi], dev["emp_cov"][lo:hi], dev["noise"][lo:hi],
                                     128, gains=dev["gains"][lo:hi], max_iter=T, n_chunks=nck, out=out)


def timed(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


outs = {}
for name, bnd in {"whole": [0, B], "w,3w,7w,B": [0, w, 3 * w, 7 * w, B], "2w,7w,B": [0, 2 * w, 7 * w, B],
                  "7w,B": [0, 7 * w, B]}.items():
    per = []
    for lo, hi in zip(bnd[:-1], bnd[1:]):
        o = outs.setdefault((lo, hi), {})
        per.append(round(timed(lambda: outs.__setitem__((lo, hi), run(lo, hi, outs[(lo, hi)]))), 2))
    print(json.dumps({"bounds": name, "chunk_ms": per, "sum_ms": round(sum(per), 2),
                      "us_per_instance": [round(1e3 * m / (hi - lo), 1) for m, lo, hi in zip(per, bnd[:-1], bnd[1:])]}), flush=True)
