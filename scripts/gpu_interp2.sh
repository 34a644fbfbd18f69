mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "golden_programs or traj or c1_twenty" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for s in 2 1; do QSV_TRAJ_STREAMS=$s timeout 900 python bench.py --workload traj > gpurun_out/bench_traj.json 2>gpurun_out/bench_traj.err; echo "streams=$s traj rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench_traj.json'));print(d['ms_per_step'], '%.3g'%d['value'])"; done
timeout 600 python scripts/traj_profile.py > gpurun_out/traj_profile.log 2>&1; grep "jit=-1" gpurun_out/traj_profile.log
