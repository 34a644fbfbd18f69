# forced low qubits L (tile must contain qubits 0..L-1): fewer forced => fewer passes
mkdir -p gpurun_out
run() { timeout 600 env $1 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline $2 > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json;d=json.load(open('gpurun_out/sw.json'));c=d['config'];print('$1','$2',round(d['ms_per_step'],1),'%.3g'%d['value'],c['passes'],c['stages'],round(d['roofline']['avg_launch_ms'],2),d['clocks']['sm_mhz'])" || tail -3 gpurun_out/sw.err; }
run "" ""
run "" "--low 4"
run "" "--low 3"
run "" "--low 2"
run "" "--workload qft"
run "" "--workload qft --low 4"
run "" "--workload qft --low 3"
