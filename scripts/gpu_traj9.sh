# C5: one-by-one trajectories (default) vs error-free trajectories batched 2^b per state
mkdir -p gpurun_out
for b in 0 6 0 4 0; do
 timeout 900 python bench.py --workload traj --batch-clean $b > gpurun_out/bench_traj_b$b.json 2>gpurun_out/bench_traj.err
 python -c "import json;d=json.load(open('gpurun_out/bench_traj_b$b.json'));print('batch_clean=$b', round(d['ms_per_step'],1), '%.3g'%d['value'])"
done
cp gpurun_out/bench_traj_b0.json gpurun_out/bench_traj.json
