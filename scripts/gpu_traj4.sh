mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --workload traj > gpurun_out/bench_traj.json 2>gpurun_out/bench_traj.err; echo "traj rc=$?"; cat gpurun_out/bench_traj.json; tail -3 gpurun_out/bench_traj.err
timeout 900 python bench.py --workload traj --dedup > gpurun_out/bench_traj2.json 2>>gpurun_out/bench_traj.err; cat gpurun_out/bench_traj2.json
timeout 600 python scripts/traj_profile.py > gpurun_out/traj_profile.log 2>&1; echo "prof rc=$?"; grep -v "jit=1" gpurun_out/traj_profile.log | tail -4
