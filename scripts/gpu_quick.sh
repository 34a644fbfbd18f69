mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for w in rqc qft; do timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --workload $w > gpurun_out/sw.json 2>gpurun_out/sw.err
python -c "import json;d=json.load(open('gpurun_out/sw.json'));print('$w',round(d['ms_per_step'],1),'%.3g'%d['value'],d['config']['passes'],round(d['roofline']['avg_launch_ms'],2),round(d['roofline']['frac'],3),d['gpu_launches'])" || tail -3 gpurun_out/sw.err; done
