# one ncu --set full capture of the heaviest C2 pass (pass 5) with and without lock-step gangs
mkdir -p gpurun_out
CMD1="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD1 > gpurun_out/plain_g.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:qsv_pass -s 15 -c 1 -o gpurun_out/prof_p5 -f $CMD1 > gpurun_out/ncu_p5.log 2>&1; echo "base rc=$?"
QSV_JIT_GANG=3 ncu --set full --clock-control none --import-source on -k regex:qsv_pass -s 15 -c 1 -o gpurun_out/prof_p5_gang3 -f $CMD1 > gpurun_out/ncu_p5g.log 2>&1; echo "gang rc=$?"
