#!/bin/bash
# ncu --set full capture of one kernel, summarised ON THE BOX (raw metrics csv
# + per-SASS-line stall samples) so gpurun_out stays small; the .ncu-rep is
# kept only when KEEP_REP=1.
#   scripts/ncu_capture.sh NAME KERNEL_REGEX SKIP COUNT -- command...
name=$1; kre=$2; skip=$3; cnt=$4; shift 5
out=gpurun_out/ncu_$name
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$kre" -s $skip -c $cnt -o /tmp/ncu_$name -f "$@" > /tmp/ncu_$name.log 2>&1
tail -2 /tmp/ncu_$name.log
ncu -i /tmp/ncu_$name.ncu-rep --page raw --csv > ${out}_raw.csv 2>/dev/null
ncu -i /tmp/ncu_$name.ncu-rep --page source --csv --print-source sass > /tmp/ncu_${name}_src.csv 2>/dev/null
python3 - /tmp/ncu_${name}_src.csv ${out}_hot.txt <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
out = open(sys.argv[2], "w")
cur = None; hdr = None; items = []
def flush():
    if not items: return
    tot = sum(v for v, *_ in items) or 1
    out.write(f"== {cur}  total samples {tot:.0f}\n")
    keys = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
    for v, src, r in sorted(items, key=lambda t: -t[0])[:40]:
        reasons = sorted(((float(r[hdr.index(k)] or 0), k) for k in keys), reverse=True)[:3]
        out.write(f"{v:7.0f} {100*v/tot:5.1f}%  {src[:70]:70s} " + " ".join(f"{k[6:]}={x:.0f}" for x, k in reasons if x) + "\n")
for r in rows:
    if len(r) == 2 and r[0] == "Kernel Name":
        flush(); cur = r[1][:90]; items = []; hdr = None; continue
    if r and r[0] == "Address":
        hdr = r; continue
    if hdr and len(r) == len(hdr):
        try: v = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except ValueError: continue
        items.append((v, r[hdr.index("Source")], r))
flush()
PY
[ "$KEEP_REP" = "1" ] && cp /tmp/ncu_$name.ncu-rep gpurun_out/
rm -f /tmp/ncu_${name}_src.csv
