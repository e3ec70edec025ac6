"""Summarise an `ncu --set full` capture (raw page CSV) into profiles/.

  ncu -i rep.ncu-rep --page raw --csv > raw.csv
  python -m paper_1906_01211_b200.tools.ncu_summary raw.csv [more.csv ...] --out profiles/r1_vN_ncu_summary.csv \
      [--traffic profiles/ncu_traffic.json] [--fp64 profiles/ncu_fp64_executed.json]

One row per captured launch (kernel name, duration, DRAM bytes, pipe and
issue utilisation, hit rates, stalls, registers, executed FP64 flops). The
JSON side files feed bench.py's roofline.traffic / ncu_executed_fp64 (first
launch of each bench kernel name)."""
from __future__ import annotations

import argparse
import csv
import json

COLS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_sector_hit_rate.pct",
    "lts__t_sector_hit_rate.pct",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "launch__registers_per_thread",
    "smsp__inst_executed.sum",
    "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "sm__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "sm__sass_thread_inst_executed_op_dfma_pred_on.sum",
]

# bench kernel names (MDG_LAUNCH names) <- device function name prefixes
BENCH_NAME = [("k_tmatvec_pre<1>", "tmatvec_pcg"), ("k_tmatvec_pre<0>", "tmatvec_pre"),
              ("k_perm_field", "field_tpre"), ("k_mpole", "mpole"), ("k_halgren", "halgren"),
              ("k_polar_force", "polar_force"), ("k_nlist_cells", "nlist_cells"),
              ("k_nlist_build", "nlist_build"), ("k_sort_rows", "sort_rows")]

SCALE = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
         "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def to_num(v: str) -> float:
    return float(v.replace(",", ""))


def summarise(hdr, units, r):
    """One launch's row of the raw page -> the COLS it has, times in ms,
    DRAM in bytes, plus executed FP64 TFLOP/s when the op counts are there."""
    idx = {h: k for k, h in enumerate(hdr)}
    rec = {"kernel": r[idx["Kernel Name"]]}
    for col in COLS:
        if col not in idx:
            continue
        v = to_num(r[idx[col]])
        scale = SCALE.get(units[idx[col]], 1.0)
        if col == "gpu__time_duration.sum":
            rec["time_ms"] = v * scale
        elif col.startswith("dram__bytes"):
            rec[col] = v * scale
        else:
            rec[col] = v
    if all(k in rec for k in COLS[-3:]):
        fl = rec[COLS[-3]] + rec[COLS[-2]] + 2.0 * rec[COLS[-1]]
        rec["fp64_executed_tflops"] = fl / (rec["time_ms"] * 1e-3) / 1e12
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("raw", nargs="+", help="one or more raw-page CSVs")
    ap.add_argument("--out", required=True)
    ap.add_argument("--traffic")
    ap.add_argument("--fp64")
    ap.add_argument("--fp64-peak", type=float, default=36.56,
                    help="TFLOP/s, the DFMA-chain probe (mdg_probe_fp64_peak)")
    a = ap.parse_args()
    tables = []
    for path in a.raw:
        with open(path) as f:
            rows = list(csv.reader(f))
        tables.append((rows[0], rows[1], rows[2:]))
    out_rows, traffic, fp64 = [], {}, {}
    for hdr, units, data in tables:
        for r in data:
            rec = summarise(hdr, units, r)
            out_rows.append(rec)
            base = rec["kernel"].removeprefix("void ")
            bench = next((b for p, b in BENCH_NAME if base.startswith(p)), None)
            if bench is None or bench in traffic:
                continue
            traffic[bench] = int(rec.get("dram__bytes_read.sum", 0) +
                                 rec.get("dram__bytes_write.sum", 0))
            if "fp64_executed_tflops" in rec:
                fp64[bench] = {"executed_tflops": round(rec["fp64_executed_tflops"], 3),
                               "frac": round(rec["fp64_executed_tflops"] / a.fp64_peak, 4),
                               "fp64_pipe_pct": round(rec.get(COLS[3], 0.0), 2)}
    keys = ["kernel", "time_ms"] + [c for c in COLS[1:] if any(c in r for r in out_rows)] + \
        ["fp64_executed_tflops"]
    with open(a.out, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=keys, extrasaction="ignore")
        w.writeheader()
        for r in out_rows:
            w.writerow(r)
    src = f"{a.out} (ncu --set full --clock-control none, config 4, first launch of each kernel)"
    if a.traffic:
        with open(a.traffic, "w") as f:
            json.dump({"source": src + "; dram__bytes_read.sum + dram__bytes_write.sum",
                       "kernels": traffic}, f, indent=1)
    if a.fp64:
        with open(a.fp64, "w") as f:
            json.dump({"source": src + "; (dadd + dmul + 2 dfma) / duration",
                       "fp64_peak_tflops": a.fp64_peak, "kernels": fp64}, f, indent=1)
    for r in out_rows:
        print(f"{r['kernel'][:48]:48s} {r['time_ms']:8.3f} ms")


if __name__ == "__main__":
    main()
