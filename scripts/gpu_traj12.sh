# C5 back-to-back series with clocks: is the ~1.45 s outlier a clock/power event?
mkdir -p gpurun_out
for i in 1 2 3 4 5 6 7 8; do
 timeout 300 python bench.py --workload traj > gpurun_out/t12.json 2>gpurun_out/t12.err || { echo "run $i FAILED"; tail -3 gpurun_out/t12.err; continue; }
 python -c "import json;d=json.load(open('gpurun_out/t12.json'));print('run $i', round(d['ms_per_step'],1), '%.3g'%d['value'], d['clocks'])"
done
