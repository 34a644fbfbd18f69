# Parametrised bench sweep (one gpurun call): each argument is "ENV=... ENV2=...|bench args".
#   bash scripts/sweep.sh "|" "QSV_JIT_PREFETCH=1|" "|--workload qft --regs 4"
# prints one summary line per configuration (ms/step, passes, regs, HBM frac, FP64 frac, SM clock)
mkdir -p gpurun_out
for cfg in "$@"; do
  envs=${cfg%%|*}; args=${cfg#*|}
  timeout 900 env $envs python bench.py --steps ${STEPS:-3} --warmup ${WARMUP:-3} --no-e2e --no-cpu-baseline $args \
    > gpurun_out/sw.json 2> gpurun_out/sw.err
  python - "$envs" "$args" <<'PY' || tail -3 gpurun_out/sw.err
import json, sys
d = json.load(open("gpurun_out/sw.json")); c = d["config"]; r = d["roofline"]
print(sys.argv[1] or "-", sys.argv[2] or "-", round(d["ms_per_step"], 2), "%.3g" % d["value"],
      c.get("passes"), c.get("reg_qubits"), round(r["frac"], 3),
      round(r.get("fp64", {}).get("frac", 0), 3), d.get("clocks", {}).get("sm_mhz"))
PY
done
