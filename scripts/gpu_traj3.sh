mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "traj or noise or pauli or readout or measure" > gpurun_out/traj_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/traj_pytest.log
timeout 900 python bench.py --workload traj > gpurun_out/bench_traj.json 2>gpurun_out/bench_traj.err; echo "traj rc=$?"; cat gpurun_out/bench_traj.json; tail -3 gpurun_out/bench_traj.err
timeout 600 python scripts/traj_profile.py > gpurun_out/traj_profile.log 2>&1; echo "prof rc=$?"; grep -v "jit=1" gpurun_out/traj_profile.log | tail -8
