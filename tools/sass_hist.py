"""Per-kernel SASS instruction histograms of libhks.so (static counts of the
mnemonics that identify the data path): python tools/sass_hist.py OUT.json"""
import collections
import json
import re
import subprocess
import sys

LIB = "paper_1701_02324_b200/_lib/libhks.so"
HOT = ("gemm_batched_kernel", "gemm_skinny_kernel", "trsm_kernel", "panel_loop_kernel", "getrs_fused_kernel",
       "gather_rows_kernel", "gecon_warp_kernel", "eval_kernel", "eval_mma_kernel", "ksum_kernel", "ksum_mma_kernel",
       "knn_kernel", "knn_stream_kernel", "knn_chunk_kernel", "tsqr_absorb_kernel", "qr_update", "qr_wpart",
       "qr_id_rows")
KEEP = ("DMMA", "DFMA", "DADD", "DMUL", "LDGSTS", "UBLKCP", "UTMALDG", "SYNCS", "LDG", "STG", "LDS", "STS", "SHFL",
        "BAR", "MUFU", "REDUX", "LDGDEPBAR")

out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
kernels, cur = {}, None
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        name = m.group(1)
        cur = collections.Counter() if any(h in name for h in HOT) else None
        if cur is not None:
            kernels[name] = cur
        continue
    if cur is None:
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\d+\s+)?([A-Z][A-Za-z0-9_.]*)", line)
    if not m:
        continue
    op = m.group(1)
    cur["total_instructions"] += 1
    base = op.split(".")[0]
    if base in KEEP:
        key = op if base in ("DMMA", "LDGSTS", "UBLKCP", "UTMALDG", "SYNCS") else base
        cur[key] += 1
note = ("cuobjdump -sass of paper_1701_02324_b200/_lib/libhks.so (sm_100a): per-kernel static instruction histograms "
        "of the hot kernels (tools/sass_hist.py).  DMMA.8x8x4 = FP64 mma.sync m8n8k4 (the FP64 tensor path; sm_100a "
        "has no FP64 tcgen05 kind in CUDA 12.9); LDGSTS.E.64 / .E.128 = 8- / 16-byte cp.async; UBLKCP = "
        "cp.async.bulk (TMA bulk copy, the kNN candidate tiles) with SYNCS = its mbarrier operations.  No UTMALDG: "
        "tensor-map TMA is not used (the batched operands are ragged per-node descriptors with run-time strides, "
        "most of them not 16-byte multiples).")
json.dump({"note": note, "kernels": {k: dict(sorted(v.items())) for k, v in sorted(kernels.items())}},
          open(sys.argv[1], "w"), indent=1)
print(len(kernels), "kernels")
