# register-qubit / occupancy variants after the FP64 work reached 2 DADD per amplitude per mixing gate
mkdir -p gpurun_out
run() { timeout 600 env $1 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline $2 > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json;d=json.load(open('gpurun_out/sw.json'));c=d['config'];print('$1','$2',round(d['ms_per_step'],1),'%.3g'%d['value'],c['passes'],c['stages'],round(d['roofline']['avg_launch_ms'],2),d['clocks']['sm_mhz'])" || tail -3 gpurun_out/sw.err; }
run "" ""
run "" "--regs 4"
run "" "--regs 4 --tile 11"
run "QSV_JIT_MIN_BLOCKS=4" "--regs 4 --tile 11"
run "QSV_JIT_MIN_BLOCKS=3" "--regs 4"
run "" "--regs 3 --tile 10"
run "QSV_JIT_MIN_BLOCKS=4" "--regs 4 --tile 10"
