# Like sweep.sh, but prints the per-pass table (ms, FP64/amp, GB/s) of every configuration.
#   bash scripts/sweep_passes.sh "ENV=..|bench args" ...
mkdir -p gpurun_out
i=0
for cfg in "$@"; do
  envs=${cfg%%|*}; args=${cfg#*|}
  timeout 900 env $envs python bench.py --steps ${STEPS:-3} --warmup ${WARMUP:-3} --no-e2e --no-cpu-baseline --traffic off $args \
    > gpurun_out/swp_$i.json 2> gpurun_out/swp.err
  python - "$envs" "$args" gpurun_out/swp_$i.json <<'PY' || tail -3 gpurun_out/swp.err
import json, sys
d = json.load(open(sys.argv[3])); c = d["config"]; r = d["roofline"]
print(f"== {sys.argv[1] or '-'} | {sys.argv[2] or '-'}: {d['ms_per_step']:.2f} ms passes={c.get('passes')} stages={c.get('stages')} "
      f"frac={r['frac']:.3f} clk={d.get('clocks', {}).get('sm_mhz')}")
print("   ms  ", " ".join(f"{p['ms']:6.2f}" for p in r["per_pass"]))
print("   fp64", " ".join(f"{p['fp64_per_amp']:6.1f}" for p in r["per_pass"]))
PY
  i=$((i+1))
done
