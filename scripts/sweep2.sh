mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for args in "" "--tile 11" "--tile 10"; do
  timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline $args > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json;d=json.load(open('gpurun_out/sw.json'));print('$args',round(d['ms_per_step'],1),d['config']['passes'],d['config']['stages'],round(d['roofline']['frac'],3))" || tail -3 gpurun_out/sw.err
done
