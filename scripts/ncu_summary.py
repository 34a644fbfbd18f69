"""Summarise an ncu report: key metrics + SASS opcode histogram (run here, no GPU)."""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
def page(p, extra=()):
    return subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(page("details"))))
hdr = rows[0]; ix = {h: i for i, h in enumerate(hdr)}
want = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Registers Per Thread", "Achieved Occupancy", "Executed Instructions", "L1/TEX Hit Rate",
        "Warp Cycles Per Issued Instruction", "No Eligible", "Dynamic Shared Memory Per Block"]
seen = set()
for r in rows[1:]:
    name = r[ix["Metric Name"]]
    if name in want and (r[ix["ID"]], name) not in seen:
        seen.add((r[ix["ID"]], name))
        print(f"[{r[ix['ID']]}] {name:40s} {r[ix['Metric Unit']]:12s} {r[ix['Metric Value']]}")
raw = list(csv.reader(io.StringIO(page("raw"))))
rh = raw[0]
for key in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "smsp__inst_executed.sum",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"):
    for i, h in enumerate(rh):
        if h == key:
            print(f"{key:60s}", raw[1][i], [r[i] for r in raw[2:]])
sass = list(csv.reader(io.StringIO(page("source", ["--print-source", "sass"]))))
hi = [i for i, r in enumerate(sass) if r and r[0] == "Address"]
if hi:
    h = sass[hi[0]]; ix = {k: i for i, k in enumerate(h)}
    cnt = collections.Counter(); stall = collections.Counter(); tot = 0
    for r in sass[hi[0] + 1:]:
        if len(r) < len(h) or not r[ix["Instructions Executed"]].isdigit():
            continue
        toks = r[ix["Source"]].strip().split()
        op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        n = int(r[ix["Instructions Executed"]]); cnt[op] += n; tot += n
        stall[op] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    print("warp-instructions executed", tot)
    for op, n in cnt.most_common(22):
        print(f"  {op:10s} {n:14d} {100 * n / tot:5.1f}%  stall-samples {stall[op]}")
