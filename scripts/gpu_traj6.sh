mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "probe_out or traj or noise or pauli" > gpurun_out/traj_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/traj_pytest.log
timeout 900 python bench.py --workload traj > gpurun_out/bench_traj.json 2>gpurun_out/bench_traj.err; echo "traj rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench_traj.json'));print(d['ms_per_step'], '%.3g'%d['value'])"; tail -3 gpurun_out/bench_traj.err
