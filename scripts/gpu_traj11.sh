# trajectory parity (incl. the explicit-program fallback) + C5 forced-low-qubit A/B
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "traj" > gpurun_out/traj_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/traj_pytest.log
for o in "" "--low 4" "" "--low 4" "" "--low 4" "--super 20"; do
 timeout 300 python bench.py --workload traj $o > gpurun_out/t11.json 2>gpurun_out/t11.err || { echo "$o FAILED"; tail -3 gpurun_out/t11.err; continue; }
 python -c "import json;d=json.load(open('gpurun_out/t11.json'));print('opts=[$o]', round(d['ms_per_step'],1), '%.3g'%d['value'])"
done
