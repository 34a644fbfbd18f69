# 16 amplitudes per thread (R=4) under one-CTA-per-tile grids
mkdir -p gpurun_out
run() { timeout 600 env $1 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline $2 > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json;d=json.load(open('gpurun_out/sw.json'));c=d['config'];r=d['roofline'];print('$1','$2',round(d['ms_per_step'],1),'%.3g'%d['value'],c['passes'],c['stages'],round(r['avg_launch_ms'],2),round(r['fp64']['frac'],3),d['clocks']['sm_mhz'])" || tail -3 gpurun_out/sw.err; }
run "" "--regs 4"
run "QSV_JIT_MIN_BLOCKS=2" "--regs 4"
run "QSV_JIT_MIN_BLOCKS=3" "--regs 4"
run "QSV_JIT_MIN_BLOCKS=1" "--regs 4"
run "" "--regs 3"
run "" "--regs 4 --low 4"
run "" "--regs 4 --low 2"
run "" "--regs 4 --tile 13"
run "" "--workload qft --regs 4"
run "" "--workload qft --regs 3"
run "" "--qubits 32 --regs 4 --steps 2 --warmup 1"
