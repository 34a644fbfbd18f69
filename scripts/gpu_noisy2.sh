mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_noisy_batch.py -m gpu -x -q > gpurun_out/pytest_nb.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_nb.log
timeout 600 python bench.py --workload noisy --steps 3 --warmup 1 > gpurun_out/bench_noisy.json 2> gpurun_out/bench_noisy.err; echo "bench rc=$?"; cat gpurun_out/bench_noisy.json
CMD="python bench.py --workload noisy --steps 1 --warmup 1 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:noisy_batch -c 60 --log-file gpurun_out/noisy_launches.csv $CMD > gpurun_out/ncu_noisy_l.log 2>&1; echo "launches rc=$?"
