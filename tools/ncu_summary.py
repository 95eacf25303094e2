"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv) into profiles/ncu_summary.json, which bench.py reads for
roofline.traffic.

usage: python tools/ncu_summary.py launches.csv "command that produced it" [instances_per_launch]
"""
import collections, csv, json, pathlib, re, sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
src, cmd = sys.argv[1], sys.argv[2]
per_launch = int(sys.argv[3]) if len(sys.argv) > 3 else 2048
rows = [r for r in csv.reader(open(src)) if len(r) > 14 and r[0].isdigit()]
launch = collections.defaultdict(dict)
for r in rows:
    launch[int(r[0])]["kernel"] = r[4]
    launch[int(r[0])][r[12]] = float(r[14].replace(",", ""))


def short(name):
    m = re.search(r"::(\w+)<([^>]*)>", name)
    return f"{m.group(1)}<{m.group(2)}>" if m else name


out = {"_source": f"{pathlib.Path(src).name}: ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                  f"dram__bytes_write.sum --clock-control none, command `{cmd}`"}
for key, pat in (("column_kernel", "column_kernel"), ("factor_kernel", "factor_solve")):
    ls = [v for v in launch.values() if pat in v["kernel"]]
    if not ls:
        continue
    rd = sum(v.get("dram__bytes_read.sum", 0) for v in ls) / len(ls)
    wr = sum(v.get("dram__bytes_write.sum", 0) for v in ls) / len(ls)
    dur = sum(v.get("gpu__time_duration.sum", 0) for v in ls) / len(ls)
    out[key] = {"kernel": short(ls[0]["kernel"]), "instances_per_launch": per_launch, "launches": len(ls),
                "dram_bytes_per_launch": int(rd + wr), "dram_read_bytes_per_launch": int(rd),
                "dram_write_bytes_per_launch": int(wr), "mean_duration_ns_cold": int(dur)}
    if key == "column_kernel":
        out[key]["algorithmic_pilot_bytes_per_launch"] = per_launch * 1000 * 40 * 16
# keep the full-capture figures (pipe utilisation of one --set full launch) already recorded
try:
    prev = json.loads((ROOT / "profiles" / "ncu_summary.json").read_text())
    for key in ("column_kernel", "factor_kernel"):
        for k, v in prev.get(key, {}).items():
            if "full_capture" in k and key in out:
                out[key][k] = v
except Exception:
    pass
(ROOT / "profiles" / "ncu_summary.json").write_text(json.dumps(out, indent=2) + "\n")
print(json.dumps(out, indent=2))
