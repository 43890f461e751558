#!/bin/bash
# ncu evidence for one round (run on the GPU box from the repo root):
#   1. launch list of one bench step (graphs on, --clock-control none)
#   2. --set full capture of the step's longest launch of each kernel named
#      in KERNELS (default: the GEMM)
# Usage: CONFIG=C3 TAG=r02 KERNELS="gemm_batched_kernel panel_loop_kernel" tools/ncu_round.sh
# Outputs under gpurun_out/: ${TAG}_launches.csv, ${TAG}_<kernel>.ncu-rep + _raw.csv / _details.csv.
set -e
CONFIG=${CONFIG:-C3}
TAG=${TAG:-r02}
KERNELS=${KERNELS:-gemm_batched_kernel}
BENCH="python bench.py --config $CONFIG --steps 1 --warmup 3 --no-cpu-baseline --no-clocks --no-accuracy"
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $BENCH > gpurun_out/${TAG}_ncu_list.log 2>&1
for K in $KERNELS; do
  SKIP=$(python - "$K" "$TAG" <<'PY'
import csv, sys
k, tag = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(f"gpurun_out/{tag}_launches.csv")))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hd = rows[hi]
ki, mi, vi, ii = (hd.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
dur, order = {}, []
for r in rows[hi + 1:]:
    if len(r) > vi and r[ki].split("(")[0].split("<")[0].strip().endswith(k) and r[mi] == "gpu__time_duration.sum":
        order.append(r[ii]); dur[r[ii]] = float(r[vi].replace(",", ""))
print(max(range(len(order)), key=lambda j: dur[order[j]]) if order else -1)
PY
)
  echo "$K: longest launch index $SKIP"
  [ "$SKIP" -ge 0 ] || continue
  ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"$K" \
      --launch-skip $SKIP -c 1 -o gpurun_out/${TAG}_$K -f $BENCH > gpurun_out/${TAG}_${K}_full.log 2>&1
  ncu -i gpurun_out/${TAG}_$K.ncu-rep --page details --csv > gpurun_out/${TAG}_${K}_details.csv
  ncu -i gpurun_out/${TAG}_$K.ncu-rep --page raw --csv > gpurun_out/${TAG}_${K}_raw.csv
done
