"""profiles/ncu_summary.json from profiles/rNN_ncu_full_spmm.json (the per-launch
DRAM traffic bench.py reports as roofline.traffic)."""
import json
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "profiles/r01_ncu_full_spmm.json"
s = json.load(open(src))
UNITS = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1.0, "us": 1e-3, "ns": 1e-6}


def val(v):
    x, u = v.split()
    return float(x) * UNITS[u]


out = {"_note": "ncu --set full --clock-control none, one launch each (products W=32, F=128); "
                "dram bytes per launch = dram__bytes_read.sum + dram__bytes_write.sum; source " + src}
for f, key in [("prof_spmm_f32.ncu-rep", "spmm_f32_products"), ("prof_spmm_int8.ncu-rep", "spmm_int8_products")]:
    rec = s[f][0]
    t = val(rec["dram__bytes_read.sum"]) + val(rec["dram__bytes_write.sum"])
    ms = val(rec["gpu__time_duration.sum"])
    out[key] = {"kernel": rec["kernel"].split("(")[0], "dram_bytes_per_launch": int(t),
                "dram_read": rec["dram__bytes_read.sum"], "dram_write": rec["dram__bytes_write.sum"],
                "duration_ms_under_ncu": round(ms, 4), "dram_GBps_under_ncu": round(t / ms / 1e6, 1),
                "registers": rec["launch__registers_per_thread"],
                "warps_active_per_cycle": rec["sm__warps_active.avg.per_cycle_active"],
                "issue_active": rec["smsp__issue_active.avg.pct_of_peak_sustained_active"],
                "lts_hit_rate": rec["lts__t_sector_hit_rate.pct"], "instructions": rec["smsp__inst_executed.sum"]}
json.dump(out, open("profiles/ncu_summary.json", "w"), indent=1)
print(json.dumps(out, indent=1))
