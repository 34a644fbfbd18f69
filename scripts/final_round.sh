# End-of-round measurement: GPU tests, every bench line, launch list + full ncu captures (C2 and
# QFT), power log of the C2 step.  Results land in gpurun_out/ (scripts/make_profiles.py copies
# the summaries into profiles/<round>/).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
NCU_PASSES="" SKIP_NCU=1 bash scripts/round_measure.sh
mkdir -p gpurun_out/qft
bash scripts/ncu_passes.sh "0 2" --workload qft > gpurun_out/qft_ncu.log 2>&1
for p in 0 2; do mv gpurun_out/prof_pass$p.ncu-rep gpurun_out/qft/prof_pass$p.ncu-rep; done
mv gpurun_out/launches.csv gpurun_out/qft/launches.csv; mv gpurun_out/plain.json gpurun_out/qft/plain.json
# the C2 launch list and captures again (ncu_passes.sh overwrote them)
NCU_PASSES="0 1 6"; bash scripts/ncu_passes.sh "0 1 6" > gpurun_out/c2_ncu.log 2>&1
nvidia-smi --query-gpu=clocks.sm,power.draw,power.limit,temperature.gpu,clocks_throttle_reasons.active --format=csv,noheader -lms 100 > gpurun_out/power_c2.log & SMI=$!
python bench.py --steps 60 --warmup 3 --no-e2e --no-cpu-baseline --traffic off > gpurun_out/bench_c2_60.json 2>/dev/null
kill $SMI
nvidia-smi --query-gpu=clocks.sm,power.draw,power.limit,temperature.gpu,clocks_throttle_reasons.active --format=csv,noheader -lms 100 > gpurun_out/power_fp64.log & SMI=$!
./scripts/fp64_sustained > gpurun_out/fp64_sustained.log
kill $SMI
./scripts/tile_stream > gpurun_out/tile_stream.log
./scripts/issue_mix > gpurun_out/issue_mix.log
