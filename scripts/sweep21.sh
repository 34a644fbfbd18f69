# re-tune around the new defaults (L=3, one CTA per tile)
mkdir -p gpurun_out
run() { timeout 600 env $1 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline $2 > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json;d=json.load(open('gpurun_out/sw.json'));c=d['config'];r=d['roofline'];print('$1','$2',round(d['ms_per_step'],1),'%.3g'%d['value'],c['passes'],c['stages'],round(r['avg_launch_ms'],2),round(r['fp64']['frac'],3),d['clocks']['sm_mhz'])" || tail -3 gpurun_out/sw.err; }
run "" ""
run "QSV_JIT_MIN_BLOCKS=2" ""
run "" "--regs 4"
run "" "--tile 11"
run "" "--tile 11 --regs 4"
run "QSV_JIT_GANG=3" ""
run "QSV_JIT_DIAG_L2=1" ""
run "" "--workload qft"
run "" "--workload qft --tile 11"
run "QSV_JIT_MIN_BLOCKS=2" "--workload qft"
