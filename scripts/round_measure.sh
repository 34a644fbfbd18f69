# Round measurement on one GPU: every bench line kept under profiles/<round>/ (copied from
# gpurun_out/ by scripts/make_profiles.py), the reference arm, the ncu launch list and
# full captures of the first (synthesising) and the heaviest C2 pass.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2>> gpurun_out/bench_full.err; echo "reference rc=$?"
timeout 900 python bench.py --workload qft --no-e2e --no-cpu-baseline > gpurun_out/bench_qft.json 2>> gpurun_out/bench_full.err; echo "qft rc=$?"
timeout 900 python bench.py --qubits 32 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_n32.json 2>> gpurun_out/bench_full.err; echo "n32 rc=$?"
timeout 900 python bench.py --workload traj > gpurun_out/bench_traj.json 2>> gpurun_out/bench_full.err; echo "traj rc=$?"
timeout 900 python bench.py --workload partial > gpurun_out/bench_partial.json 2>> gpurun_out/bench_full.err; echo "partial rc=$?"
timeout 900 python bench.py --workload noisy > gpurun_out/bench_noisy.json 2>> gpurun_out/bench_full.err; echo "noisy rc=$?"
[ -n "$SKIP_NCU" ] || bash scripts/ncu_passes.sh "${NCU_PASSES:-0 3}"
