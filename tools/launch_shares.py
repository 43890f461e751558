"""Summarise an ncu launch list (gpu__time_duration.sum + dram bytes per
launch) into per-kernel totals: python tools/launch_shares.py CSV > TXT."""
import collections
import csv
import json
import sys

SCALE = {"ms": 1e6, "us": 1e3, "ns": 1, "msecond": 1e6, "usecond": 1e3, "nsecond": 1,
         "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hd = rows[hi]
    ki, mi, vi, ii, ui = (hd.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Metric Unit"))
    per, names = collections.defaultdict(dict), {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        try:
            val = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1)
        except ValueError:
            continue
        per[r[ii]][r[mi]] = val
        names[r[ii]] = r[ki].split("(")[0].replace("void ", "").split("::")[-1].split("<")[0]
    return per, names


def main():
    per, names = load(sys.argv[1])
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in per.items():
        a = agg[names[i]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"# launches {len(per)}  sum of launch times {tot / 1e6:.3f} ms (ncu: serialised, cold caches)")
    print(f"{'kernel':26s} {'launches':>8s} {'ms':>9s} {'share':>6s} {'DRAM MB':>10s} {'MB/launch':>10s}")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:26s} {a[0]:8d} {a[1] / 1e6:9.3f} {a[1] / tot:6.3f} {a[2] / 1e6:10.1f} {a[2] / a[0] / 1e6:10.2f}")
    if len(sys.argv) > 2:
        g = agg["gemm_batched_kernel"]
        json.dump({"gemm": round(g[2] / g[0]), "source": sys.argv[1],
                   "note": "mean dram__bytes_read.sum + dram__bytes_write.sum per gemm_batched_kernel launch "
                           "over one bench step"}, open(sys.argv[2], "w"), indent=1)


if __name__ == "__main__":
    main()
