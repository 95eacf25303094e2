"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv) into profiles/ncu_summary.json, which bench.py reads for
roofline.traffic.

usage: python tools/ncu_summary.py launches.csv "command that produced it" [instances_per_launch]

Kernel groups: the column pass (column_kernel*) and the factor stage, which is
either factor_solve_t (one kernel) or the fac_sweep_w + fac_prod_t pair; each
group is summarised per launch of its kernels, and the step share of every
kernel is listed.
"""
import collections, csv, json, pathlib, re, sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
src, cmd = sys.argv[1], sys.argv[2]
per_launch = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
rows = [r for r in csv.reader(open(src)) if len(r) > 14 and r[0].isdigit()]
launch = collections.defaultdict(dict)
for r in rows:
    launch[int(r[0])]["kernel"] = r[4]
    launch[int(r[0])][r[12]] = float(r[14].replace(",", ""))


def short(name):
    m = re.search(r"(\w+)<([^>]*)>", name)
    return f"{m.group(1)}<{m.group(2)}>" if m else name.split("(")[0]


def group(ls):
    rd = sum(v.get("dram__bytes_read.sum", 0) for v in ls) / len(ls)
    wr = sum(v.get("dram__bytes_write.sum", 0) for v in ls) / len(ls)
    dur = sum(v.get("gpu__time_duration.sum", 0) for v in ls) / len(ls)
    return {"kernel": short(ls[0]["kernel"]), "instances_per_launch": per_launch,
            "launches": len(ls), "dram_bytes_per_launch": int(rd + wr),
            "dram_read_bytes_per_launch": int(rd), "dram_write_bytes_per_launch": int(wr),
            "mean_duration_ns_cold": int(dur)}


out = {"_source": f"{pathlib.Path(src).name}: ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                  f"dram__bytes_write.sum --clock-control none, command `{cmd}`"}
total = sum(v.get("gpu__time_duration.sum", 0) for v in launch.values())
by_kernel = collections.defaultdict(list)
for v in launch.values():
    by_kernel[short(v["kernel"])].append(v)
out["step_share_by_kernel"] = {
    k: {"launches": len(ls), "mean_ns": int(sum(v.get("gpu__time_duration.sum", 0) for v in ls) / len(ls)),
        "share": round(sum(v.get("gpu__time_duration.sum", 0) for v in ls) / total, 4)}
    for k, ls in sorted(by_kernel.items(), key=lambda kv: -sum(v.get("gpu__time_duration.sum", 0)
                                                               for v in kv[1]))}
for key, pats in (("column_kernel", ("column_kernel",)),
                  ("factor_kernel", ("factor_solve",)),
                  ("factor_sweep", ("fac_sweep",)),
                  ("factor_products", ("fac_prod",))):
    ls = [v for v in launch.values() if any(p in v["kernel"] for p in pats)]
    if ls:
        out[key] = group(ls)
if "column_kernel" in out:
    out["column_kernel"]["algorithmic_pilot_bytes_per_launch"] = per_launch * 1000 * 40 * 16
# keep the full-capture figures (pipe utilisation of one --set full launch) already recorded
try:
    prev = json.loads((ROOT / "profiles" / "ncu_summary.json").read_text())
    for key in out:
        if isinstance(out[key], dict):
            for k, v in prev.get(key, {}).items():
                if "full_capture" in k:
                    out[key].setdefault(k, v)
except Exception:
    pass
(ROOT / "profiles" / "ncu_summary.json").write_text(json.dumps(out, indent=2) + "\n")
print(json.dumps(out, indent=2))
