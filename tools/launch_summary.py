"""Summarise an ncu --metrics gpu__time_duration.sum launch list of one
factorize (tools/ncu_fact.py): per-kind totals for the leaf level (launches
before the first norm1_kernel) and for the whole factorization."""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hd = rows[hi]
ki, vi, gi = hd.index("Kernel Name"), hd.index("Metric Value"), hd.index("Grid Size")
out = []
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    n = r[ki].split("(")[0].replace("void ", "").replace("unnamed>::", "").split("<")[0]
    out.append((n, float(r[vi].replace(",", "")) / 1e3, r[gi]))
ends = [i for i, (n, _, _) in enumerate(out) if n == "norm1_kernel"]
end = ends[0] if ends else len(out)
for title, seg in (("leaf level", out[:end]), ("all", out)):
    agg = collections.defaultdict(float)
    for n, us, _ in seg:
        agg[n] += us
    print(title, {k: round(v / 1e3, 3) for k, v in sorted(agg.items(), key=lambda kv: -kv[1])},
          "total ms", round(sum(agg.values()) / 1e3, 3))
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 150
for i, (n, us, g) in enumerate(out[:end]):
    if us > thr:
        print(i, n, round(us, 1), g)
