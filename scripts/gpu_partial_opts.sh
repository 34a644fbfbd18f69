# partial mode (n=36 cut 18) planner options A/B
mkdir -p gpurun_out
for o in "" "--low 4" "--tile 11" "" "--low 4" "--low 5" "--regs 4" ""; do
 timeout 300 python bench.py --workload partial --no-cpu-baseline $o > gpurun_out/p.json 2>gpurun_out/p.err || { echo "$o FAILED"; tail -3 gpurun_out/p.err; continue; }
 python -c "import json;d=json.load(open('gpurun_out/p.json'));print('opts=[$o]', round(d['ms_per_step'],2), '%.3g'%d['value'])"
done
