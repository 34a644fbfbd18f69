mkdir -p gpurun_out
run() { timeout 300 env $1 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline $2 > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json;d=json.load(open('gpurun_out/sw.json'));print('$1','$2',round(d['ms_per_step'],1),d['config']['passes'],d['config']['super_passes'],round(d['roofline']['avg_launch_ms'],2))" || tail -3 gpurun_out/sw.err; }
for t in 12 11; do for db in 1 0; do for mb in 1 2 3; do
run "QSV_JIT_DBUF=$db QSV_JIT_MIN_BLOCKS=$mb" "--super 12 --tile $t"
done; done; done
run "QSV_JIT_DBUF=0 QSV_JIT_MIN_BLOCKS=2" ""
run "QSV_JIT_DBUF=0 QSV_JIT_MIN_BLOCKS=3" "--tile 11"
