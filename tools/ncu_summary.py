"""Summarise `ncu --page raw --csv` dumps of single-launch full captures into
one JSON: python tools/ncu_summary.py OUT.json NOTE raw1.csv raw2.csv ..."""
import csv
import json
import sys

KEYS = {
    "duration_ms": ("gpu__time_duration.sum", None),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "dmma_pipe_pct": ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", None),
    "fp64_pipe_pct": ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", None),
    "lsu_pipe_pct": ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", None),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", None),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", None),
    "regs": ("launch__registers_per_thread", None),
    "shared_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", None),
    "shared_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", None),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", None),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", None),
    "grid": ("launch__grid_size", None),
    "block": ("launch__block_size", None),
    "smem_per_block_bytes": ("launch__shared_mem_per_block_dynamic", None),
}
SCALE = {"ms": 1.0, "us": 1e-3, "ns": 1e-6, "msecond": 1.0, "usecond": 1e-3, "nsecond": 1e-6, "s": 1e3, "second": 1e3,
         "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}


def one(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    head, units, vals = rows[hi], rows[hi + 1], rows[hi + 2]
    out = {"kernel": vals[head.index("Kernel Name")].split("(")[0].replace("void ", "").split("::")[-1]}
    for name, (metric, _) in KEYS.items():
        if metric not in head:
            continue
        i = head.index(metric)
        try:
            v = float(vals[i].replace(",", ""))
        except ValueError:
            continue
        out[name] = round(v * SCALE.get(units[i], 1.0), 6)
    return out


if __name__ == "__main__":
    json.dump({"note": sys.argv[2], "captures": [one(p) for p in sys.argv[3:]]}, open(sys.argv[1], "w"), indent=1)
