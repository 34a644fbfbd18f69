mkdir -p gpurun_out
for v in "" "QSV_JIT_PREFETCH=0" "" "QSV_JIT_PREFETCH=0" "QSV_PLAN_ROLLOUT=0"; do
 env $v timeout 900 python bench.py --workload traj > gpurun_out/bench_traj.json 2>gpurun_out/bench_traj.err; python -c "import json;d=json.load(open('gpurun_out/bench_traj.json'));print('$v', d['ms_per_step'], '%.3g'%d['value'])"
done
