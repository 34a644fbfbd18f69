"""Turn a scripts/round_measure.sh run (gpurun_out/) into the committed profiles/<round>/ files.

  python scripts/make_profiles.py r02
Writes: launches.csv + launches_summary.txt (ncu launch list of one warm-up + one timed C2 step,
per-launch time and DRAM bytes), ncu_full_pass<k>.txt (metrics, SASS mix, stall reasons of the
captured passes), bench_*.json (every bench line), bench_reference.json (the reference arm).
"""
import collections, csv, json, shutil, subprocess, sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
out = ROOT / "profiles" / sys.argv[1]
src = ROOT / "gpurun_out"
out.mkdir(parents=True, exist_ok=True)

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
         "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}

# launch list
if (src / "launches.csv").exists():
    shutil.copy(src / "launches.csv", out / "launches.csv")
    rows = [r for r in csv.reader(open(src / "launches.csv")) if len(r) > 10]
    h = {k: i for i, k in enumerate(rows[0])}
    per = collections.OrderedDict()
    for r in rows[1:]:
        d = per.setdefault(int(r[h["ID"]]), {"kernel": r[h["Kernel Name"]].split("(")[0]})
        d[r[h["Metric Name"]]] = float(r[h["Metric Value"]].replace(",", "")) * SCALE.get(r[h["Metric Unit"]], 1.0)
    plain = json.loads((src / "plain.json").read_text()) if (src / "plain.json").exists() else {}
    npass = plain.get("config", {}).get("passes", len(per) // 2)
    tot = sum(d.get("gpu__time_duration.sum", 0.0) for d in per.values())
    lines = ["ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none",
             "(cold-cache, serialised launches: compare the SHARE of each pass, not the absolute time)",
             "command: python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --traffic off  (C2: n=30 RQC)",
             f"{len(per)} launches = warm-up step + timed step, {npass} passes each", "",
             f"{'id':>3s} {'kernel':10s} {'ms':>8s} {'share':>7s} {'DRAM GB':>8s} {'GB/s':>7s}"]
    for i, d in per.items():
        ms = d.get("gpu__time_duration.sum", 0.0)
        b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        lines.append(f"{i:3d} {d['kernel']:10s} {ms:8.3f} {100 * ms / tot:6.1f}% {b / 1e9:8.2f} {b / ms / 1e6:7.0f}")
    (out / "launches_summary.txt").write_text("\n".join(lines) + "\n")

# full captures
for rep in sorted(src.glob("prof_pass*.ncu-rep")):
    k = rep.stem.replace("prof_pass", "")
    summ = subprocess.run([sys.executable, str(ROOT / "scripts/ncu_summary.py"), str(rep)], capture_output=True,
                          text=True).stdout
    stalls = subprocess.run([sys.executable, str(ROOT / "scripts/ncu_stalls.py"), str(rep)], capture_output=True,
                            text=True).stdout
    head = (f"ncu --set full --clock-control none --import-source on -k regex:qsv_pass -s <passes + {k}> -c 1 "
            f"python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --traffic off\n"
            f"(pass {k} of the timed C2 step; scripts/ncu_passes.sh)\n\n")
    (out / f"ncu_full_pass{k}.txt").write_text(head + stalls + "\n" + summ)

# bench lines (last JSON line of each file)
for f in sorted(src.glob("bench*.json")):
    txt = [ln for ln in f.read_text().splitlines() if ln.startswith("{")]
    if txt:
        name = "bench_c2.json" if f.name == "bench_full.json" else f.name
        (out / name).write_text(json.dumps(json.loads(txt[-1]), indent=1) + "\n")
print("wrote", out)
