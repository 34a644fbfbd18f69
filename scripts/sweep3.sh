mkdir -p gpurun_out
run() { timeout 300 env $1 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline $2 > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json;d=json.load(open('gpurun_out/sw.json'));print('$1','$2',round(d['ms_per_step'],1),d['config']['passes'],d['config']['super_passes'],round(d['roofline']['avg_launch_ms'],2))" || tail -3 gpurun_out/sw.err; }
run "QSV_L2_BYTES=33554432" ""
run "QSV_L2_BYTES=67108864" ""
run "QSV_L2_BYTES=100663296" ""
run "QSV_L2_BYTES=134217728" ""
run "QSV_L2_BYTES=67108864" "--super 20"
run "QSV_L2_BYTES=100663296" "--super 22"
run "QSV_L2_BYTES=67108864" "--super 12"
