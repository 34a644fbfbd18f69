# L2 prefetch of the tile one residency wave ahead under one-CTA-per-tile grids
mkdir -p gpurun_out
run() { timeout 600 env $1 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline $2 > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json;d=json.load(open('gpurun_out/sw.json'));c=d['config'];r=d['roofline'];print('$1','$2',round(d['ms_per_step'],1),'%.3g'%d['value'],c['passes'],c['reg_qubits'],round(r['avg_launch_ms'],2),round(r['fp64']['frac'],3),d['clocks']['sm_mhz'])" || tail -3 gpurun_out/sw.err; }
run "" ""
run "QSV_JIT_PREFETCH=1" ""
run "QSV_JIT_PREFETCH=1 QSV_JIT_PREFETCH_DIST=148" ""
run "QSV_JIT_PREFETCH=1 QSV_JIT_PREFETCH_DIST=592" ""
run "QSV_JIT_PREFETCH=1 QSV_JIT_PREFETCH_DIST=1184" ""
run "" "--workload qft"
run "QSV_JIT_PREFETCH=1 QSV_JIT_PREFETCH_DIST=444" "--workload qft"
run "QSV_JIT_PREFETCH=1 QSV_JIT_PREFETCH_DIST=888" "--workload qft"
