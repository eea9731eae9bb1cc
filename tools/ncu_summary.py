"""Per-kernel table from an ncu raw page (ncu -i X.ncu-rep --page raw --csv > raw.csv):
duration, DRAM bytes, pipe / issue utilisation, active warps, top stall reasons.
Usage: python tools/ncu_summary.py raw.csv [fp64]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
fp64 = len(sys.argv) > 2 and sys.argv[2] == "fp64"
h = rows[0]
ix = {c: i for i, c in enumerate(h)}
pipe = ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active" if fp64 else
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active")
stalls = [c for c in h if c.startswith("smsp__average_warps_issue_stalled_") and c.endswith("_per_issue_active.ratio")]


def f(r, c, scale=1.0, nd=1):
    try:
        return f"{float(r[ix[c]].replace(',', '')) * scale:.{nd}f}"
    except (KeyError, ValueError):
        return "-"


print(f"| kernel | duration ms | DRAM R / W GB | {'fp64' if fp64 else 'FMA'} pipe % | issue % | warps active % | "
      "shared wavefronts M | top stalls (per issue) |")
print("|---|---|---|---|---|---|---|---|")
for r in rows[2:]:
    if len(r) < len(h):
        continue
    name = r[ix["Kernel Name"]].split("(")[0].split("::")[-1]
    unit = rows[1][ix["gpu__time_duration.sum"]]
    dur = float(r[ix["gpu__time_duration.sum"]].replace(",", "")) * {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "usecond": 1e-3,
                                                                     "msecond": 1.0, "nsecond": 1e-6}.get(unit, 1.0)
    ub = rows[1][ix["dram__bytes_read.sum"]]
    bs = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}.get(ub, 1e-9)
    st = sorted(((float(r[ix[c]] or 0), c[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")])
                 for c in stalls if r[ix[c]]), reverse=True)
    st = [x for x in st if x[1] != "selected"][:3]
    print(f"| `{name}` | {dur:.3f} | {f(r, 'dram__bytes_read.sum', bs, 2)} / {f(r, 'dram__bytes_write.sum', bs, 2)} | "
          f"{f(r, pipe)} | {f(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active')} | "
          f"{f(r, 'sm__warps_active.avg.pct_of_peak_sustained_active')} | "
          f"{f(r, 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 1e-6, 0)} | "
          + ", ".join(f"{n.replace('_', ' ')} {v:.2f}" for v, n in st) + " |")
