# full GPU test suite + default bench line + an A/B line (args: extra bench flags for the B line)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep "\[parity\]" gpurun_out/pytest_gpu.log | head -40; tail -25 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
if [ -n "$1" ]; then
timeout 600 python bench.py --no-e2e --no-cpu-baseline --traffic off "$@" > gpurun_out/bench_b.json 2>> gpurun_out/bench.err; echo "bench B rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_b.json'));print('B', d['ms_per_step'], [p['ms'] for p in d['roofline']['per_pass']], d['clocks'])"
fi
