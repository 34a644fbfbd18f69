# C5 outlier diagnosis: per-trajectory host launch timestamps over 8 back-to-back runs
mkdir -p gpurun_out; rm -f gpurun_out/traj_trace.txt
for i in 1 2 3 4 5 6 7 8; do
 QSV_TRAJ_TRACE=gpurun_out/traj_trace.txt timeout 300 python bench.py --workload traj > gpurun_out/t13.json 2>gpurun_out/t13.err || { echo "run $i FAILED"; tail -3 gpurun_out/t13.err; continue; }
 python -c "import json;d=json.load(open('gpurun_out/t13.json'));print('run $i', round(d['ms_per_step'],1))"
done
