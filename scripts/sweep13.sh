# tile / register-qubit / occupancy sweep of the specialised pass kernels (C2)
mkdir -p gpurun_out
run() { timeout 600 env $1 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline $2 > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json;d=json.load(open('gpurun_out/sw.json'));print('$1','$2',round(d['ms_per_step'],1),'%.3g'%d['value'],d['config']['passes'],d['config']['stages'],round(d['roofline']['avg_launch_ms'],2),d['clocks']['sm_mhz'])" || tail -3 gpurun_out/sw.err; }
run "QSV_JIT_MIN_BLOCKS=2" ""
run "QSV_JIT_MIN_BLOCKS=1" ""
run "QSV_JIT_MIN_BLOCKS=1" "--tile 13"
run "QSV_JIT_MIN_BLOCKS=2" "--regs 4"
run "QSV_JIT_MIN_BLOCKS=3" "--regs 4"
run "QSV_JIT_MIN_BLOCKS=1" "--regs 4 --tile 13"
run "QSV_JIT_MIN_BLOCKS=4" "--regs 4 --tile 11"
run "QSV_JIT_MIN_BLOCKS=4" "--regs 3 --tile 11"
run "QSV_JIT_MIN_BLOCKS=2" "--regs 3 --tile 12"
