# per-pass kernel times (ncu launch list) with 32 vs 16 amplitudes per thread
mkdir -p gpurun_out
for w in rqc qft; do for r in 5 4; do
  CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --workload $w --regs $r"
  $CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pr_${w}_$r.csv $CMD > /dev/null 2>&1; echo "$w $r rc=$?"
done; done
