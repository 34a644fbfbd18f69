# full measurement: GPU tests, smoke, bench line, ncu launch list + full capture of the top kernel
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"; cat gpurun_out/bench_full.json
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_l.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"
CMD1="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD1 > gpurun_out/plain_f.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:qsv_pass -s ${NCU_SKIP_FULL:-15} -c 1 -o gpurun_out/prof_full -f $CMD1 > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
