"""Summarise an ncu report: python tools/ncu_summary.py REPORT.ncu-rep"""
import csv, io, subprocess, sys

WANT = [("gpu__time_duration.sum", "ms"), ("dram__bytes_read.sum", "rd"), ("dram__bytes_write.sum", "wr"),
        ("launch__registers_per_thread", "regs"), ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%"),
        ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "l1wf%"),
        ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1%"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%")]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
SCALE = {("ms", "usecond"): 1e-3, ("ms", "us"): 1e-3, ("ms", "nsecond"): 1e-6, ("ms", "ns"): 1e-6, ("rd", "Mbyte"): 1e-3, ("wr", "Mbyte"): 1e-3,
         ("rd", "Kbyte"): 1e-6, ("wr", "Kbyte"): 1e-6}
for r in rows[2:]:
    name = r[h.index("Kernel Name")][:60]
    vals = []
    for k, lab in WANT:
        if k in h:
            i = h.index(k)
            v = r[i]
            f = SCALE.get((lab, units[i]))
            if f is not None:
                v = "%g" % (float(v.replace(",", "")) * f)
            vals.append("%s=%s" % (lab, v))
    print(name, " ".join(vals), "(ms, GB)")
