"""Turn a scripts/round_measure.sh run (gpurun_out/) into the committed profiles/<round>/ files.

  python scripts/make_profiles.py r01 [--skip-full N]
Writes: launches.csv (raw ncu launch list), launches_summary.txt, ncu_full_qsv_pass.txt
(metrics, SASS mix, stall reasons of the captured pass), traffic.json, bench.json.
"""
import collections, csv, io, json, shutil, subprocess, sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
out = ROOT / "profiles" / sys.argv[1]
skip = int(sys.argv[sys.argv.index("--skip-full") + 1]) if "--skip-full" in sys.argv else 11
src = ROOT / "gpurun_out"
out.mkdir(parents=True, exist_ok=True)

# launch list
shutil.copy(src / "launches.csv", out / "launches.csv")
rows = [r for r in csv.reader(open(src / "launches.csv")) if len(r) > 10]
h = rows[0]; ix = {k: i for i, k in enumerate(h)}
per = [(r[ix["Kernel Name"]].split("(")[0], float(r[ix["Metric Value"]].replace(",", "")) / 1e6)
       for r in rows[1:] if r[ix["Metric Name"]] == "gpu__time_duration.sum"]
tot = collections.defaultdict(float); cnt = collections.Counter()
for k, ms in per:
    tot[k] += ms; cnt[k] += 1
allms = sum(tot.values())
lines = ["ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches)",
         "command: python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline   (C2: n=30 RQC)", "",
         f"{'kernel':32s} {'launches':>8s} {'total ms':>10s} {'avg ms':>8s} {'share':>7s}"]
for k in sorted(tot, key=lambda k: -tot[k]):
    lines.append(f"{k:32s} {cnt[k]:8d} {tot[k]:10.2f} {tot[k] / cnt[k]:8.3f} {100 * tot[k] / allms:6.1f}%")
lines += ["", "per launch (ms):"] + [f"  {k:30s} {ms:7.3f}" for k, ms in per]
(out / "launches_summary.txt").write_text("\n".join(lines) + "\n")

# full capture of one pass
rep = str(src / "prof_full.ncu-rep")
summ = subprocess.run([sys.executable, str(ROOT / "scripts/ncu_summary.py"), rep], capture_output=True, text=True).stdout
stalls = subprocess.run([sys.executable, str(ROOT / "scripts/ncu_stalls.py"), rep], capture_output=True, text=True).stdout
head = (f"ncu --set full --clock-control none --import-source on -k regex:qsv_pass -s {skip} -c 1 "
        f"python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline\n"
        f"(launch {skip} of the qsv_pass kernels = one pass of the timed step)\n\n")
(out / "ncu_full_qsv_pass.txt").write_text(head + summ + "\nwarp stalls per issued instruction:\n" + stalls)
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                                   capture_output=True, text=True).stdout)))
rh = raw[0]; rv = raw[2]
val = lambda k: float(rv[rh.index(k)].replace(",", ""))
unit = lambda k: raw[1][rh.index(k)]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd = val("dram__bytes_read.sum") * scale[unit("dram__bytes_read.sum")]
wr = val("dram__bytes_write.sum") * scale[unit("dram__bytes_write.sum")]
bench = json.loads((src / "bench_full.json").read_text())
n = bench["config"]["n_qubits"]
(out / "traffic.json").write_text(json.dumps({
    "kernel": f"qsv_pass (runtime-specialised fused pass, C2 launch {skip})",
    "capture": f"ncu --set full --clock-control none -k regex:qsv_pass -s {skip} -c 1 (profiles/{sys.argv[1]}/ncu_full_qsv_pass.txt)",
    "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
    "algorithmic_bytes_per_launch": 32 * 2 ** n, "round": int(sys.argv[1][1:])}, indent=1) + "\n")
(out / "bench.json").write_text(json.dumps(bench, indent=1) + "\n")
# the other configs' bench lines (scripts/round_measure.sh)
for name in ("bench_qft", "bench_traj", "bench_traj_dedup", "bench_n32", "bench_partial", "bench_noisy"):
    f = src / f"{name}.json"
    if f.exists() and f.read_text().strip():
        (out / f"{name}.json").write_text(json.dumps(json.loads(f.read_text().strip().splitlines()[-1]), indent=1) + "\n")
# batched noisy-trajectory kernel: launch list + one full capture
if (src / "noisy_launches.csv").exists():
    shutil.copy(src / "noisy_launches.csv", out / "noisy_launches.csv")
    agg = collections.defaultdict(list)
    nrows = [r for r in csv.reader(open(src / "noisy_launches.csv")) if len(r) > 10]
    nh = {k: i for i, k in enumerate(nrows[0])}
    for r in nrows[1:]:
        agg[(r[nh["Kernel Name"]].split("(")[0], r[nh["Metric Name"]])].append(float(r[nh["Metric Value"]].replace(",", "")))
    nl = ["ncu launch list: python bench.py --workload noisy --steps 1 --warmup 1 --no-cpu-baseline --trajectories 256",
          "(first 60 noisy_batch* launches, --clock-control none; 2 groups of 128 trajectories x 2^20 amplitudes:",
          " algorithmic bytes per apply+reduce launch = 2 x 16 x 2^27 = 4.29 GB)", "",
          "kernel | launches | avg us | avg dram read+write GB | GB/s"]
    for k in sorted({k for k, _ in agg}):
        t = agg[(k, "gpu__time_duration.sum")]; rr = agg[(k, "dram__bytes_read.sum")]; ww = agg[(k, "dram__bytes_write.sum")]
        T = sum(t) / len(t); Bb = sum(rr) / len(rr) + sum(ww) / len(ww)
        nl.append(f"{k} | {len(t)} | {T / 1e3:.1f} | {Bb / 1e9:.3f} | {Bb / T:.0f}")
    (out / "noisy_launches_summary.txt").write_text("\n".join(nl) + "\n")
if (src / "prof_noisy.ncu-rep").exists():
    summ = subprocess.run([sys.executable, str(ROOT / "scripts/ncu_summary.py"), str(src / "prof_noisy.ncu-rep")],
                          capture_output=True, text=True).stdout
    (out / "ncu_full_noisy_batch.txt").write_text(
        "ncu --set full --clock-control none -k regex:noisy_batch_kernel -s 30 -c 1 "
        "python bench.py --workload noisy --steps 1 --warmup 1 --no-cpu-baseline --trajectories 256\n\n" + summ)
if (src / "exchange_pass.log").exists():
    shutil.copy(src / "exchange_pass.log", out / "exchange_pass.log")
print("wrote", out)
