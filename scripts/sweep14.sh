# super-pass (L2-resident inner passes) sweep after the FP64 reductions (C2)
mkdir -p gpurun_out
run() { timeout 600 env $1 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline $2 > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json;d=json.load(open('gpurun_out/sw.json'));c=d['config'];print('$1','$2',round(d['ms_per_step'],1),'%.3g'%d['value'],c['passes'],c['stages'],c['super_passes'],c['super_qubits'],round(d['roofline']['avg_launch_ms'],2),d['clocks']['sm_mhz'])" || tail -3 gpurun_out/sw.err; }
run "" ""
run "" "--tile 13"
run "" "--super 20"
run "" "--super 21"
run "" "--super 22"
run "" "--tile 13 --super 21"
run "" "--tile 13 --super 22"
