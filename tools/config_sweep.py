"""Device throughput of every BASELINE config (c0..c3 batched path, c2 net, c4 large path).

Prints one JSON line per config: instances/s, ms per solve, PSCA iterations/s,
algorithmic TFLOP/s (24 N L^2 per instance-iteration).  Inputs resident in HBM.
"""
import json, os, sys
sys.path.insert(0, ".")
import numpy as np
import torch
import __graft_entry__
__graft_entry__.build()
import bench
from paper_2503_15259_b200 import estimators, large, scenes, unroll

dev = torch.device("cuda", 0)


def timed(fn, reps=3, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def batched(name, net=False):
    cfg = scenes.BASELINE_CONFIGS[name]
    B = cfg.batch
    host = bench.generate(name, list(range(B)), os.cpu_count() or 1)
    P, E, Nz, G = (torch.from_numpy(host[k]).to(dev) for k in ("pilots", "emp_cov", "noise", "gains"))
    prob = scenes.problem_for(cfg)
    T = cfg.net_blocks if net else cfg.n_iter
    sched = estimators.StepSchedule.explicit(scenes.net_steps(T)) if net else None
    out = {}

    def run():
        nonlocal out
        kw = {"n_chunks": int(os.environ["SWEEP_CHUNKS"])} if os.environ.get("SWEEP_CHUNKS") else {}
        out = estimators.psca_run_batch(prob, P, E, Nz, cfg.n_antennas, gains=G, schedule=sched,
                                        max_iter=T, out=out, **kw)
    ms = timed(run)
    prof = None
    if os.environ.get("SWEEP_PROFILE"):
        from paper_2503_15259_b200 import device
        device.profile_begin()
        run()
        torch.cuda.synchronize()
        p = device.profile_end()
        prof = {"column_ms_per_launch": p["column_ms"] / max(1, p["column_launches"]),
                "factor_ms_per_launch": p["factor_ms"] / max(1, p["factor_launches"]),
                "column_ms": p["column_ms"], "factor_ms": p["factor_ms"]}
    flops = 24.0 * cfg.n_devices * cfg.pilot_len ** 2 * B * T
    return {"config": name + ("_net" if net else ""), "kind": cfg.kind, "B": B, "N": cfg.n_devices,
            "L": cfg.pilot_len, "T": T, "ms_per_solve": ms, "instances_per_s": B / (ms * 1e-3),
            "psca_iters_per_s": B * T / (ms * 1e-3), "algorithmic_tflops": flops / (ms * 1e-3) / 1e12,
            "path": out.get("path"), "profile": prof}


only = set(sys.argv[1:])
want = lambda n: not only or n in only   # noqa: E731
rows = [batched(n) for n in ("c0", "c1", "c2", "c3_l20", "c3_l40", "c3_l80") if want(n)]
if want("c2_net"):
    rows.append(batched("c2", net=True))
for r in rows:
    print(json.dumps(r), flush=True)
if not want("c4"):
    sys.exit(0)
rows = []
cfg = scenes.BASELINE_CONFIGS["c4"]
s = scenes.make_scene(cfg, 0)
S = torch.from_numpy(s.pilots).to(dev)
g = torch.from_numpy(s.gains).to(dev)
Em = torch.from_numpy(s.emp_cov).to(dev)
steps = estimators.default_steps(cfg.n_iter)
ms = timed(lambda: large.psca_run_large("ml-k", S, g, Em, 1.0, cfg.n_antennas, steps,
                                        max_iter=cfg.n_iter), reps=2, warm=1)
rows.append({"config": "c4", "kind": "ml-k", "B": 1, "N": cfg.n_devices, "L": 256, "T": cfg.n_iter,
             "ms_per_solve": ms, "instances_per_s": 1e3 / ms,
             "psca_iters_per_s": cfg.n_iter * 1e3 / ms,
             "algorithmic_tflops": 24.0 * cfg.n_devices * 256 ** 2 * cfg.n_iter / (ms * 1e-3) / 1e12,
             "path": "large"})
for r in rows:
    print(json.dumps(r), flush=True)
