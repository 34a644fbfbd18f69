# C5 planner options sweep (clean-plan tile / register / low / L2 super-tile qubits)
mkdir -p gpurun_out
for o in "" "--super 20" "--super 22" "--tile 11" "--tile 13" "--low 4" "--low 5" "--regs 5" ""; do
 timeout 300 python bench.py --workload traj $o > gpurun_out/t10.json 2>gpurun_out/t10.err || { echo "$o FAILED"; tail -3 gpurun_out/t10.err; continue; }
 python -c "import json;d=json.load(open('gpurun_out/t10.json'));print('opts=[$o]', round(d['ms_per_step'],1), '%.3g'%d['value'])"
done
