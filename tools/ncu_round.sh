#!/bin/bash
# ncu evidence for one round (run on the GPU box from the repo root):
#   1. launch list of one bench step (graphs on, --clock-control none)
#   2. --set full capture of the step's largest gemm_batched_kernel launch
# Outputs under gpurun_out/ (launches.csv, gemm_top.ncu-rep, gemm_top_*.csv).
set -e
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-clocks > gpurun_out/ncu_list.log 2>&1
SKIP=$(python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/launches.csv")))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hd = rows[hi]
ki, mi, vi, ii = (hd.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
dur, order = {}, []
for r in rows[hi + 1:]:
    if len(r) > vi and "gemm_batched_kernel" in r[ki] and r[mi] == "gpu__time_duration.sum":
        order.append(r[ii]); dur[r[ii]] = float(r[vi].replace(",", ""))
print(max(range(len(order)), key=lambda j: dur[order[j]]))
PY
)
echo "largest gemm launch index: $SKIP"
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:gemm_batched_kernel \
    --launch-skip $SKIP -c 1 -o gpurun_out/gemm_top -f \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-clocks > gpurun_out/ncu_full.log 2>&1
ncu -i gpurun_out/gemm_top.ncu-rep --page details --csv > gpurun_out/gemm_top_details.csv
ncu -i gpurun_out/gemm_top.ncu-rep --page raw --csv > gpurun_out/gemm_top_raw.csv
echo "skip=$SKIP" > gpurun_out/gemm_top_skip.txt
