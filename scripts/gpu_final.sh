# final check at HEAD: all GPU tests, smoke, C5 lines with the trajectory defaults
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --workload traj > gpurun_out/bench_traj.json 2>gpurun_out/bench_traj.err; echo "traj rc=$?"
timeout 900 python bench.py --workload traj --dedup > gpurun_out/bench_traj_dedup.json 2>>gpurun_out/bench_traj.err; echo "dedup rc=$?"
for f in bench_traj bench_traj_dedup; do python -c "import json;d=json.load(open('gpurun_out/$f.json'));print('$f', round(d['ms_per_step'],1), '%.3g'%d['value'])"; done
