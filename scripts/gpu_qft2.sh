mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "qft or golden_programs or c1_twenty" > gpurun_out/qft_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/qft_pytest.log
run() { timeout 600 env $1 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline $2 > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json;d=json.load(open('gpurun_out/sw.json'));c=d['config'];r=d['roofline'];print('$1','$2',round(d['ms_per_step'],1),'%.3g'%d['value'],c['passes'],c['stages'],c['reg_qubits'],round(r['avg_launch_ms'],2),round(r['fp64']['frac'],3),d['clocks']['sm_mhz'])" || tail -3 gpurun_out/sw.err; }
run "" "--workload qft"
run "QSV_JIT_MIN_BLOCKS=2" "--workload qft"
run "" "--workload qft --regs 4"
