# full measurement: GPU tests, smoke, bench line, ncu launch list + full capture of the top kernel
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"; cat gpurun_out/bench_full.json
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_l.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"
CMD1="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD1 > gpurun_out/plain_f.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:qsv_pass -s ${NCU_SKIP_FULL:-11} -c 1 -o gpurun_out/prof_full -f $CMD1 > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
# the other BASELINE configs on this one GPU (bench lines kept under profiles/<round>/)
timeout 900 python bench.py --workload qft --no-e2e --no-cpu-baseline > gpurun_out/bench_qft.json 2>> gpurun_out/bench_full.err; echo "qft rc=$?"
timeout 900 python bench.py --workload traj > gpurun_out/bench_traj.json 2>> gpurun_out/bench_full.err; echo "traj rc=$?"
timeout 900 python bench.py --workload traj --dedup > gpurun_out/bench_traj_dedup.json 2>> gpurun_out/bench_full.err; echo "traj dedup rc=$?"
timeout 900 python bench.py --qubits 32 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_n32.json 2>> gpurun_out/bench_full.err; echo "n32 rc=$?"
timeout 900 python bench.py --workload partial > gpurun_out/bench_partial.json 2>> gpurun_out/bench_full.err; echo "partial rc=$?"
timeout 900 python bench.py --workload noisy > gpurun_out/bench_noisy.json 2>> gpurun_out/bench_full.err; echo "noisy rc=$?"
NCMD="python bench.py --workload noisy --steps 1 --warmup 1 --no-cpu-baseline --trajectories 256"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:noisy_batch -c 60 --log-file gpurun_out/noisy_launches.csv $NCMD > gpurun_out/ncu_noisy_l.log 2>&1; echo "noisy launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:noisy_batch_kernel -s 30 -c 1 -o gpurun_out/prof_noisy -f $NCMD > gpurun_out/ncu_noisy_full.log 2>&1; echo "noisy full rc=$?"
timeout 600 python scripts/exchange_pass_bench.py > gpurun_out/exchange_pass.log 2>&1; echo "exchange rc=$?"
