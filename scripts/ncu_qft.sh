mkdir -p gpurun_out
C1="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --workload qft --super 12"
C2="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --workload qft"
$C1 > gpurun_out/plain1.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:qsv_pass -s 14 -c 1 -o gpurun_out/prof_qft_flat -f $C1 > gpurun_out/ncu1.log 2>&1; echo "ncu1 rc=$?"
$C2 > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:qsv_super -s 4 -c 1 -o gpurun_out/prof_qft_super -f $C2 > gpurun_out/ncu2.log 2>&1; echo "ncu2 rc=$?"
