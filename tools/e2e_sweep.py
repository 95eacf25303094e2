"""End-to-end (host in / host out) timing of psca_run_batch_host under different
chunk schedules (experiment driver for the e2e bench key).

usage: python tools/e2e_sweep.py   (c1, B = 4096, T = 100)
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__
__graft_entry__.build()
import bench
from paper_2503_15259_b200 import device, estimators, scenes

cfg = scenes.BASELINE_CONFIGS["c1"]
B, T = 4096, 100
host = bench.generate("c1", list(range(B)), os.cpu_count() or 1)
pin = {k: torch.from_numpy(host[k]).pin_memory() for k in ("pilots", "emp_cov", "noise", "gains")}
prob = scenes.problem_for(cfg)
w = 2 * device.sm_count()
orig = estimators._host_chunk_bounds
schedules = {
    "default": None,
    "w,3w,7w,B": [0, w, 3 * w, 7 * w, B],
    "w,B": [0, w, B],
    "w/2,w,7w,B": [0, w // 2, w, 7 * w, B],
    "2w,7w,B": [0, 2 * w, 7 * w, B],
    "equal4": [(B * c) // 4 for c in range(5)],
    "2w,B": [0, 2 * w, B],
    "w,3w,B": [0, w, 3 * w, B],
    "2w,6w,B": [0, 2 * w, 6 * w, B],
    "w,2w,4w,8w,B": [0, w, 2 * w, 4 * w, 8 * w, B],
    "2w,4w,8w,B": [0, 2 * w, 4 * w, 8 * w, B],
    "w/2,3w/2,7w/2,B": [0, w // 2, 3 * w // 2, 7 * w // 2, B],
    "w,2w,4w,7w,B": [0, w, 2 * w, 4 * w, 7 * w, B],
    "w,2w,3w,5w,8w,B": [0, w, 2 * w, 3 * w, 5 * w, 8 * w, B],
}
if os.environ.get("E2E_ONLY"):
    schedules = {k: v for k, v in schedules.items() if k in os.environ["E2E_ONLY"].split(";")}


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


dev = {k: v.cuda() for k, v in pin.items()}
out = {}


def devrun():
    global out
    out = estimators.psca_run_batch(prob, dev["pilots"], dev["emp_cov"], dev["noise"], 128,
                                    gains=dev["gains"], max_iter=T, out=out)


print(json.dumps({"device_ms": timed(devrun)}), flush=True)
del dev, out
for name, bnd in schedules.items():
    estimators._host_chunk_bounds = (lambda B_, c_, b=bnd: b) if bnd else orig
    ms = timed(lambda: estimators.psca_run_batch_host(prob, pin["pilots"], pin["emp_cov"], pin["noise"],
                                                      128, gains=pin["gains"], max_iter=T))
    print(json.dumps({"schedule": name, "e2e_ms": ms, "inst_per_s": B / ms * 1e3}), flush=True)
