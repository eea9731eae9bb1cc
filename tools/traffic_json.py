"""ncu per-launch DRAM bytes (CSV of --metrics dram__bytes_read.sum,dram__bytes_write.sum,
gpu__time_duration.sum over tools/one_frame.py W ss 1) -> profiles/ncu_traffic.json,
summed per bench stage (col_carry = k_seed + the carry kernel). Usage:
  python tools/traffic_json.py gpurun_out/r02_traffic.csv profiles/ncu_traffic.json 8192 [tag]"""
import csv
import json
import sys

STAGES = [("k_mean", "mean"), ("k_seed", "col_carry"), ("k_col_carry", "col_carry"),
          ("k_colpass", "colpass"), ("k_row_scan", "row_scan"), ("k_rowpass", "rowpass")]


def main():
    src, dst, w = sys.argv[1], sys.argv[2], int(sys.argv[3])
    tag = sys.argv[4] if len(sys.argv) > 4 else ""
    lines = [l for l in open(src) if l.startswith('"')]
    per_launch = {}
    for row in csv.DictReader(lines):
        key = (row["ID"], row["Kernel Name"])
        per_launch.setdefault(key, {})[row["Metric Name"]] = float(row["Metric Value"].replace(",", ""))
    out_b, out_t = {}, {}
    for (_, name), m in per_launch.items():
        stage = next((s for k, s in STAGES if k in name), None)
        if stage is None:
            continue
        out_b[stage] = out_b.get(stage, 0) + int(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0))
        out_t[stage] = out_t.get(stage, 0) + int(m.get("gpu__time_duration.sum", 0))
    px = w * w
    json.dump({"source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                         "--clock-control none (one launch per kernel, cold cache), tools/one_frame.py "
                         f"{w} 5 1 -> {src.split('/')[-1]} {tag}; col_carry = k_seed + k_col_carry_tma",
               "width": w, "height": w, "degree": 20, "bytes_per_launch": out_b, "duration_ns": out_t,
               "bytes_per_px": {k: round(v / px, 1) for k, v in out_b.items()},
               "total_bytes_per_px": round(sum(out_b.values()) / px, 1)},
              open(dst, "w"), indent=1)
    print(json.load(open(dst)))


if __name__ == "__main__":
    main()
