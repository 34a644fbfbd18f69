# TMA-fed tiles for compute-bound passes (QSV_JIT_TMA), with independent CTAs and with lock-step gangs
mkdir -p gpurun_out
for v in "QSV_JIT_TMA=1" "QSV_JIT_TMA=1 QSV_JIT_GANG=3"; do
  env $v QSV_JIT_GANG_MIN=0 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "c1_twenty or larger or qft_round or golden_programs" > gpurun_out/tma_pytest.log 2>&1; echo "$v parity rc=$?"; tail -2 gpurun_out/tma_pytest.log
done
run() { timeout 600 env $1 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline $2 > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json;d=json.load(open('gpurun_out/sw.json'));c=d['config'];print('$1','$2',round(d['ms_per_step'],1),'%.3g'%d['value'],c['passes'],c['stages'],round(d['roofline']['avg_launch_ms'],2),d['clocks']['sm_mhz'])" || tail -3 gpurun_out/sw.err; }
run "" ""
run "QSV_JIT_TMA=1" ""
run "QSV_JIT_TMA=1 QSV_JIT_GANG=3" ""
run "QSV_JIT_TMA=1 QSV_JIT_GANG=2" ""
run "QSV_JIT_TMA=1 QSV_JIT_GANG_MIN=0" ""
run "" "--workload qft"
run "QSV_JIT_TMA=1" "--workload qft"
run "QSV_JIT_TMA=1 QSV_JIT_GANG=3" "--workload qft"
