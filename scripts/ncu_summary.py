"""Summarise an ncu --set full report (run here, no GPU needed)."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__inst_executed.sum", "smsp__inst_executed.sum",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__warps_active.avg.per_cycle_active"]


def summarize(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        rec = {"kernel": d.get("Kernel Name", "")[:160]}
        for k in KEYS:
            if k in d:
                rec[k] = d[k] + (" " + units[hdr.index(k)] if units[hdr.index(k)] else "")
        # stall breakdown (warp-state)
        stalls = {k.split("warp_state_")[-1]: d[k] for k in hdr
                  if k.startswith("smsp__average_warp_latency_per_inst_issued") or
                  ("smsp__pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"))}
        rec["stalls"] = {k: v for k, v in stalls.items() if v not in ("", "0")}
        out.append(rec)
    return out


if __name__ == "__main__":
    print(json.dumps({p.split("/")[-1]: summarize(p) for p in sys.argv[1:]}, indent=1))
