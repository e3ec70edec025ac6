"""Executed FP64 flops of one config-4 AMOEBA step from an ncu metrics pass
(one step incl. a list rebuild, host-driven PCG loop):

  ncu --metrics gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,\
sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum \
      --clock-control none --csv --log-file LAUNCHES.csv python tools/one_step.py 4 1
  python tools/fp64_step.py LAUNCHES.csv PCG_ITERATIONS > profiles/r2_ncu_fp64_step.json

flops = dadd + dmul + 2 dfma per kernel; split into the list rebuild, the
per-PCG-iteration kernels and the fixed rest (bench.py fp64_step_fraction)."""
import collections
import csv
import io
import json
import sys

REBUILD = ("k_nlist_cells", "k_cut_rows", "k_sort_rows", "k_scan", "k_cell_", "k_row_union",
           "k_cluster_union", "k_cluster_gen", "k_list_motion", "k_moved")
PER_ITER = ("k_tmatvec_pre<true", "k_tmatvec_pre<1", "k_tmatvec_cl<true", "k_tmatvec_cl<1",
            "k_cg_update", "k_cg_dir", "k_cg_finish", "k_cg_scalars")


def main(path, iters):
    lines = open(path).read().splitlines()
    k0 = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[k0:]))))
    h = rows[0]
    iid, iname, imet, ival = (h.index(k) for k in ("ID", "Kernel Name", "Metric Name",
                                                   "Metric Value"))
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        per[r[iid]][r[imet]] = float(r[ival].replace(",", "") or 0)
        names[r[iid]] = r[iname]
    kern = collections.defaultdict(lambda: {"launches": 0, "fp64_flops": 0.0, "ncu_ms": 0.0})
    parts = {"rebuild": 0.0, "iter": 0.0, "fixed": 0.0}
    for lid, m in per.items():
        name = names[lid].replace("void ", "").replace("mdg::", "")
        fl = (m.get("sm__sass_thread_inst_executed_op_dadd_pred_on.sum", 0.0) +
              m.get("sm__sass_thread_inst_executed_op_dmul_pred_on.sum", 0.0) +
              2.0 * m.get("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", 0.0))
        key = name.split("(")[0]
        kern[key]["launches"] += 1
        kern[key]["fp64_flops"] += fl
        kern[key]["ncu_ms"] += m.get("gpu__time_duration.sum", 0.0) * 1e-6
        if name.startswith(REBUILD):
            parts["rebuild"] += fl
        elif name.startswith(PER_ITER):
            parts["iter"] += fl
        else:
            parts["fixed"] += fl
    out = {"what": "executed FP64 flops (dadd + dmul + 2 dfma, ncu "
                   "sm__sass_thread_inst_executed_op_*_pred_on.sum) of one BASELINE config-4 "
                   "AMOEBA step incl. one list rebuild (python tools/one_step.py 4 1 under ncu "
                   "--metrics, --clock-control none), round 2 session 2 HEAD",
           "pcg_iterations": iters,
           "per_eval_fixed_flops": parts["fixed"],
           "per_pcg_iteration_flops": parts["iter"] / max(1, iters),
           "per_rebuild_flops": parts["rebuild"],
           "kernels": dict(sorted(kern.items(), key=lambda kv: -kv[1]["fp64_flops"]))}
    json.dump(out, sys.stdout, indent=1)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
