"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch count, mean/total device time and share of the total."""
import collections
import csv
import io
import json
import sys


def summarize(path, only_after=None):
    text = open(path).read()
    start = text.index('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    launches = []
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        t = float(d["Metric Value"])
        t_ns = t * (1000.0 if d["Metric Unit"] == "us" else 1e6 if d["Metric Unit"] == "ms" else 1.0)
        launches.append((d["Kernel Name"], t_ns, d["Grid Size"], d["Block Size"]))
    agg = collections.OrderedDict()
    for name, t, grid, block in launches:
        short = name.split("(")[0][:120]
        a = agg.setdefault(short, {"launches": 0, "total_us": 0.0, "grid": grid, "block": block})
        a["launches"] += 1
        a["total_us"] += t / 1e3
    tot = sum(a["total_us"] for a in agg.values())
    out = []
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["total_us"]):
        out.append({"kernel": k, **a, "mean_us": round(a["total_us"] / a["launches"], 2),
                    "total_us": round(a["total_us"], 2), "share": round(a["total_us"] / tot, 4)})
    return {"launches": len(launches), "total_us": round(tot, 2), "kernels": out}


if __name__ == "__main__":
    print(json.dumps(summarize(sys.argv[1]), indent=1))
