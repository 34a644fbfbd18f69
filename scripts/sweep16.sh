# lock-step multi-tile CTAs (QSV_JIT_GANG) for compute-bound passes: parity first, then timing
mkdir -p gpurun_out
QSV_JIT_GANG=3 QSV_JIT_GANG_MIN=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "c1_twenty or larger or qft_round or golden_programs" > gpurun_out/gang_pytest.log 2>&1; echo "gang3 parity rc=$?"; tail -2 gpurun_out/gang_pytest.log
QSV_JIT_GANG=2 QSV_JIT_GANG_MIN=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "c1_twenty or larger" > gpurun_out/gang2_pytest.log 2>&1; echo "gang2 parity rc=$?"; tail -2 gpurun_out/gang2_pytest.log
run() { timeout 600 env $1 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline $2 > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json;d=json.load(open('gpurun_out/sw.json'));c=d['config'];print('$1','$2',round(d['ms_per_step'],1),'%.3g'%d['value'],c['passes'],c['stages'],round(d['roofline']['avg_launch_ms'],2),d['clocks']['sm_mhz'])" || tail -3 gpurun_out/sw.err; }
run "" ""
run "QSV_JIT_GANG=3" ""
run "QSV_JIT_GANG=2" ""
run "QSV_JIT_GANG=3" "--low 3"
run "QSV_JIT_GANG=3 QSV_JIT_GANG_MIN=40" ""
run "" "--workload qft"
run "QSV_JIT_GANG=3" "--workload qft"
run "QSV_JIT_GANG=3" "--workload qft --low 3"
