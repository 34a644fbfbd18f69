# lazy sampling + cached clean plan: trajectory parity + C5 series with launch traces
mkdir -p gpurun_out; rm -f gpurun_out/traj_trace.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "traj" > gpurun_out/traj_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/traj_pytest.log
for i in 1 2 3 4 5 6; do
 QSV_TRAJ_TRACE=gpurun_out/traj_trace.txt timeout 300 python bench.py --workload traj > gpurun_out/t15.json 2>gpurun_out/t15.err || { echo "run $i FAILED"; tail -3 gpurun_out/t15.err; continue; }
 python -c "import json;d=json.load(open('gpurun_out/t15.json'));print('run $i', round(d['ms_per_step'],1))"
done
cp gpurun_out/t15.json gpurun_out/bench_traj.json
timeout 300 python bench.py --workload traj --dedup > gpurun_out/bench_traj_dedup.json 2>>gpurun_out/t15.err; echo "dedup rc=$?"
