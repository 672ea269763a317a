"""profiles/ncu_summary.json from the committed round-2 ncu summaries
(profiles/r02/ncu_*_summary.json, written by scripts/ncu_capture.sh +
scripts/ncu_raw_summary.py): the per-launch DRAM traffic bench.py reports as
roofline.traffic, keyed spmm_<dtype>_<config>.

    python scripts/make_profile_summary.py
"""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
R02 = os.path.join(ROOT, "profiles", "r02")
UNITS = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1.0, "us": 1e-3, "ns": 1e-6}
# bench key -> capture (current default kernel of that path)
SOURCES = {
    "spmm_f32_products": "ncu_f32_summary.json",
    "spmm_int8_products": "ncu_q8_batch_default_summary.json",
    "spmm_int8-row_products": "ncu_q8f_row_summary.json",
    "spmm_int8-feature_products": "ncu_q8f_feat_summary.json",
    "spmm_f32_reddit": "ncu_f32_reddit_summary.json",
    "spmm_int8_reddit": "ncu_q8b_reddit_summary.json",
    "spmm_int8-row_reddit": "ncu_q8f_row_reddit_summary.json",
    "spmm_int8-feature_reddit": "ncu_q8f_feat_reddit_summary.json",
}


def val(v):
    x, u = v.split()
    return float(x) * UNITS[u]


out = {"_note": "ncu --set full --clock-control none, one launch each (W=32); dram bytes per launch = "
                "dram__bytes_read.sum + dram__bytes_write.sum; sources profiles/r02/<file>"}
for key, f in SOURCES.items():
    p = os.path.join(R02, f)
    if not os.path.exists(p):
        continue
    rec = json.load(open(p))[0]
    t = val(rec["dram__bytes_read.sum"]) + val(rec["dram__bytes_write.sum"])
    ms = val(rec["gpu__time_duration.sum"])
    out[key] = {"kernel": rec["kernel"].split("(")[0], "source": "profiles/r02/" + f,
                "dram_bytes_per_launch": int(t), "duration_ms_under_ncu": round(ms, 4),
                "dram_GBps_under_ncu": round(t / ms / 1e6, 1),
                "registers": rec.get("launch__registers_per_thread"),
                "issue_active": rec.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                "instructions": rec.get("smsp__inst_executed.sum")}
json.dump(out, open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
