mkdir -p gpurun_out
run() { timeout 600 env $1 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline $2 > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json;d=json.load(open('gpurun_out/sw.json'));print('$1','$2',round(d['ms_per_step'],1),'%.3g'%d['value'],d['config']['passes'],d['config']['super_passes'],round(d['roofline']['avg_launch_ms'],2))" || tail -3 gpurun_out/sw.err; }
run "" "--super 21"
run "QSV_L2_BYTES=100663296" "--super 21"
run "" "--super 20"
run "" "--super 22"
run "" "--workload qft --super 21"
run "" "--workload qft --super 20"
