# per-pass kernel durations (ncu launch list, serialised) for the C2 plan under env/flag variants
mkdir -p gpurun_out
i=0
while read -r ENVS ARGS; do
i=$((i+1))
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline $ARGS"
env $ENVS $CMD > gpurun_out/pt_plain.log 2>&1 && env $ENVS ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/pt_$i.csv $CMD > gpurun_out/pt_ncu.log 2>&1; echo "variant $i [$ENVS] [$ARGS] rc=$?"
done < ${VARIANTS:-scripts/pt_variants.txt}
