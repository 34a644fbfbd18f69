mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
run() { timeout 600 env $1 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline $2 > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json;d=json.load(open('gpurun_out/sw.json'));c=d['config'];r=d['roofline'];print('$1','$2',round(d['ms_per_step'],1),'%.3g'%d['value'],c['passes'],c['stages'],c['reg_qubits'],round(r['avg_launch_ms'],2),round(r['fp64']['frac'],3),d['clocks']['sm_mhz'])" || tail -3 gpurun_out/sw.err; }
run "" ""
run "" "--workload qft"
run "" "--qubits 32 --steps 2 --warmup 1"
run "QSV_PLAN_ROLLOUT=0" "--qubits 32 --steps 2 --warmup 1"
run "" "--qubits 31 --steps 2 --warmup 1"
run "QSV_PLAN_ROLLOUT=0" "--qubits 31 --steps 2 --warmup 1"
