"""Pretty-print an HKS_TRACE dump (tools/level_times.py stderr)."""
import sys
names = ("gemm", "copy", "getrf", "getrs", "gecon", "eval", "eval_rm", "ksum", "panel", "swap", "trsm_l", "trsm_u",
         "norm1", "lu_fused", "gather", "getrs_fused")
sec = None
for line in open(sys.argv[1]):
    if line.startswith("MARK"):
        print(line.strip())
        continue
    if not line.startswith("HKS_TRACE"):
        continue
    _, k, ms, fl, by = line.split()
    ms, fl, by = float(ms), float(fl), float(by)
    print(f"{names[int(k)]:12s} {ms * 1e3:8.1f} us  {fl / 1e9:8.3f} GF {fl / ms / 1e9 if ms else 0:6.2f} TF/s"
          f"  {by / 1e6:8.2f} MB {by / ms / 1e6 if ms else 0:7.1f} GB/s")
