"""Warp-stall breakdown (per issued instruction) + key throughput numbers of an ncu report."""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
for v in rows[2:]:
    d = dict(zip(h, v))
    def f(k):
        try: return float(d.get(k, "nan").replace(",", ""))
        except ValueError: return float("nan")
    print(d.get("Kernel Name", "?")[:40], "dur_ms", f("gpu__time_duration.sum"),
          "fp64%", f("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
          "ipc", f("sm__inst_executed.avg.per_cycle_active"), "regs", d.get("launch__registers_per_thread"))
    st = [(f(k), k.split("stalled_")[1].split("_per")[0]) for k in h
          if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
    print("  " + "  ".join(f"{n}={x:.2f}" for x, n in sorted(st, reverse=True) if x >= 0.02))
