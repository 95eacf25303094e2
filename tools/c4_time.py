"""c4 (one instance, N = 100000, L = 256, T = 50) device time per solve; optional arg: an alternative _psca.so."""
import sys, pathlib, json
sys.path.insert(0, ".")
import torch
from paper_2503_15259_b200 import device
if len(sys.argv) > 1:
    device.LIB_PATH = pathlib.Path(sys.argv[1]).resolve()
from paper_2503_15259_b200 import estimators, large, scenes
cfg = scenes.BASELINE_CONFIGS["c4"]
s = scenes.make_scene(cfg, 0)
dev = torch.device("cuda", 0)
S = torch.from_numpy(s.pilots).to(dev); g = torch.from_numpy(s.gains).to(dev); Em = torch.from_numpy(s.emp_cov).to(dev)
steps = estimators.default_steps(cfg.n_iter)
run = lambda: large.psca_run_large("ml-k", S, g, Em, 1.0, cfg.n_antennas, steps, max_iter=cfg.n_iter)
x = run(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); x = run(); e1.record(); torch.cuda.synchronize()
xx = x["x"] if isinstance(x, dict) else x
print(json.dumps({"lib": sys.argv[1] if len(sys.argv) > 1 else "", "ms_per_solve": e0.elapsed_time(e1), "xsum": float(xx.sum())}))
