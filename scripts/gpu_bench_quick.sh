# one default bench line + the interpreted-kernel C2 timing (diagnostic)
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
timeout 600 python bench.py --jit -1 --no-e2e --no-cpu-baseline --traffic off > gpurun_out/bench_interp.json 2>> gpurun_out/bench.err; echo "interp rc=$?"
cat gpurun_out/bench_interp.json
