mkdir -p gpurun_out
timeout 600 python scripts/traj_profile.py > gpurun_out/traj_profile.log 2>&1; echo "prof rc=$?"; cat gpurun_out/traj_profile.log | tail -20
timeout 900 python bench.py --workload traj > gpurun_out/bench_traj.json 2>gpurun_out/bench_traj.err; echo "traj rc=$?"; cat gpurun_out/bench_traj.json; tail -3 gpurun_out/bench_traj.err
