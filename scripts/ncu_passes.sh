# ncu: launch list of one C2 step + full captures of chosen passes of the timed step
#   bash scripts/ncu_passes.sh "2 5" [extra bench args]
mkdir -p gpurun_out
PASSES=${1:-"2"}; shift
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --traffic off $*"
$CMD > gpurun_out/plain.json 2> gpurun_out/plain.err || { echo "plain run failed"; tail -5 gpurun_out/plain.err; exit 1; }
NP=$(python -c "import json;print(json.load(open('gpurun_out/plain.json'))['config']['passes'])")
echo "passes per step: $NP"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:qsv_pass --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_l.log 2>&1; echo "launches rc=$?"
for p in $PASSES; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:qsv_pass -s $((NP + p)) -c 1 \
    -o gpurun_out/prof_pass$p -f $CMD > gpurun_out/ncu_full_$p.log 2>&1; echo "full pass $p rc=$?"
done
