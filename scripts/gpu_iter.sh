# build-measure iteration: GPU parity tests, short bench, ncu of the pass kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
CMD="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline ${BENCH_ARGS}"
timeout 600 $CMD > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err; echo "bench rc=$?"; cat gpurun_out/bench_iter.json; tail -3 gpurun_out/bench_iter.err
if [ "${NCU:-1}" = "1" ]; then
CMD1="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline ${BENCH_ARGS}"
$CMD1 > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"qsv_pass|pass_kernel" -s 3 -c 1 -o gpurun_out/prof_iter -f $CMD1 > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
fi
