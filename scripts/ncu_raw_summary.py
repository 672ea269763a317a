"""Key metrics per kernel from an `ncu --page raw --csv` export (the
*_raw.csv files scripts/ncu_capture.sh writes on the GPU box).

    python scripts/ncu_raw_summary.py gpurun_out/ncu_q8b_raw.csv [--json]
"""
import csv
import json
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warp_latency_per_inst_issued.ratio",
]
STALLS = ["long_scoreboard", "short_scoreboard", "wait", "barrier", "mio_throttle", "lg_throttle",
          "math_pipe_throttle", "not_selected", "selected", "no_instructions", "branch_resolving", "membar",
          "dispatch_stall", "drain", "sleeping", "tex_throttle"]


def summarize(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        item = {"kernel": d.get("Kernel Name", "")[:120]}
        for k in KEYS:
            if k in d:
                item[k] = f"{d[k]} {u.get(k, '')}".strip()
        st = {}
        for s in STALLS:
            k = f"smsp__pcsamp_warps_issue_stalled_{s}"
            if k in d and d[k] not in ("", "0"):
                st[s] = d[k]
        item["stall_samples"] = st
        out.append(item)
    return out


if __name__ == "__main__":
    res = summarize(sys.argv[1])
    if "--json" in sys.argv:
        print(json.dumps(res, indent=1))
    else:
        for it in res:
            print(it["kernel"])
            for k, v in it.items():
                if k != "kernel":
                    print(f"   {k:60s} {v}")
