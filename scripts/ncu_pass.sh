mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pass_kernel -s 3 -c 2 -o gpurun_out/prof_pass $CMD > gpurun_out/ncu.log 2>&1
echo "rc=$?"
tail -5 gpurun_out/ncu.log
