mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "traj or noise or pauli or probe" > gpurun_out/traj_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/traj_pytest.log
for v in "" "QSV_PAULI_FRAME=0" "" "QSV_PAULI_FRAME=0"; do
 env $v timeout 900 python bench.py --workload traj > gpurun_out/bench_traj.json 2>gpurun_out/bench_traj.err; python -c "import json;d=json.load(open('gpurun_out/bench_traj.json'));print('$v', d['ms_per_step'], '%.3g'%d['value'])"
done
