mkdir -p gpurun_out
for v in "" "QSV_JIT_GRID_TILES=1"; do
 env $v timeout 900 python bench.py --workload traj > gpurun_out/bench_traj.json 2>gpurun_out/bench_traj.err; echo "$v traj rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench_traj.json'));print(d['ms_per_step'], '%.3g'%d['value'])"
 env $v timeout 900 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/b.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b.json'));print('C2', round(d['ms_per_step'],2))"
 env $v timeout 900 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --workload qft > gpurun_out/b.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b.json'));print('QFT', round(d['ms_per_step'],2))"
done
