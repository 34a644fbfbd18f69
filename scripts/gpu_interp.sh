mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --workload traj > gpurun_out/bench_traj.json 2>gpurun_out/bench_traj.err; echo "traj rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench_traj.json'));print(d['ms_per_step'], '%.3g'%d['value'])"
timeout 600 python scripts/traj_profile.py > gpurun_out/traj_profile.log 2>&1; grep "jit=-1" gpurun_out/traj_profile.log
python bench.py --workload traj --trajectories 64 > /dev/null 2>&1; ncu --set full --clock-control none -k regex:pass_kernel -s 3 -c 1 -o gpurun_out/prof_interp2 -f python bench.py --workload traj --trajectories 64 > gpurun_out/ncu_interp.log 2>&1; echo ncu rc=$?
