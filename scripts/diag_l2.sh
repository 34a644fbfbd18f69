mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/a.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_mem.csv $CMD > /dev/null 2>&1
QSV_JIT_DIAG_L2=1 $CMD > gpurun_out/b.log 2>&1 && QSV_JIT_DIAG_L2=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_l2.csv $CMD > /dev/null 2>&1
echo done
