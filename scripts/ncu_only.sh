mkdir -p gpurun_out
CMD1="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline ${BENCH_ARGS}"
$CMD1 > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-qsv_pass|pass_kernel}" -s ${NCU_SKIP:-3} -c ${NCU_COUNT:-1} -o gpurun_out/prof_iter -f $CMD1 > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu.log
