mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "traj or noise or pauli" > gpurun_out/traj_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/traj_pytest.log
for s in 1 2 3; do QSV_TRAJ_STREAMS=$s timeout 900 python bench.py --workload traj > gpurun_out/bench_traj_$s.json 2>gpurun_out/bench_traj.err; echo "streams=$s rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench_traj_$s.json'));print(d['ms_per_step'], '%.3g'%d['value'])"; done
