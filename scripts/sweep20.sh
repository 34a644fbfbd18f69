mkdir -p gpurun_out
run() { timeout 600 env $1 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline $2 > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json;d=json.load(open('gpurun_out/sw.json'));c=d['config'];print('$1','$2',round(d['ms_per_step'],1),'%.3g'%d['value'],c['passes'],c['stages'],round(d['roofline']['avg_launch_ms'],2),d['clocks']['sm_mhz'])" || tail -3 gpurun_out/sw.err; }
run "" "--low 3"
run "QSV_JIT_PREFETCH=0" "--low 3"
run "QSV_JIT_PREFETCH=0" "--low 4"
run "QSV_JIT_PREFETCH=0" "--low 2"
run "QSV_JIT_PREFETCH=0 QSV_JIT_MIN_BLOCKS=2" "--low 3"
run "QSV_JIT_PREFETCH=0" "--low 3 --tile 13"
run "QSV_JIT_PREFETCH=0" "--workload qft --low 3"
run "QSV_JIT_PREFETCH=0" "--workload qft --low 2"
run "QSV_JIT_PREFETCH=0" "--workload qft --low 4"
run "QSV_JIT_PREFETCH=0" "--qubits 32 --low 3"
