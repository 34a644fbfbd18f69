mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_noisy_batch.py tests/test_partition.py tests/test_cli.py -m gpu -x -q > gpurun_out/pytest_nbp.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_nbp.log
timeout 600 python bench.py --workload noisy --steps 3 --warmup 1 > gpurun_out/bench_noisy.json 2> gpurun_out/bench_noisy.err; echo "noisy bench rc=$?"; cat gpurun_out/bench_noisy.json
timeout 600 python bench.py --workload partial > gpurun_out/bench_partial.json 2>gpurun_out/bench_partial.err; echo "partial bench rc=$?"; cat gpurun_out/bench_partial.json
