#!/bin/bash
# Build tools/kbench (kernel micro-benchmark) against the in-tree objects.
set -e
cd "$(dirname "$0")/.."
make -s -C paper_1701_02324_b200/csrc >/dev/null
O=paper_1701_02324_b200/_lib/obj
OBJS="$O/capi.o $O/eval.o $O/gemm.o $O/knn.o $O/lu.o $O/lu_fused.o $O/plan.o $O/qrcp.o $O/sample.o $O/tree.o $O/tsqr.o $O/vec.o"
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr"
$NV -o tools/kbench tools/kbench.cu $OBJS $O/lu2.o
