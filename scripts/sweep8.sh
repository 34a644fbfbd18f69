mkdir -p gpurun_out
run() { timeout 600 env $1 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline $2 > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json;d=json.load(open('gpurun_out/sw.json'));print('$1','$2',round(d['ms_per_step'],1),'%.3g'%d['value'],d['config']['passes'],d['config']['stages'],round(d['roofline']['avg_launch_ms'],2))" || tail -3 gpurun_out/sw.err; }
run "" "--tile 13"
run "QSV_JIT_MIN_BLOCKS=1" "--tile 13"
run "" "--tile 11"
run "QSV_JIT_MIN_BLOCKS=3" "--tile 11"
run "QSV_JIT_MIN_BLOCKS=3" ""
run "" "--workload qft --tile 13"
run "" "--workload qft --tile 11"
