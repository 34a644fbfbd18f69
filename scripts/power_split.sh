# Board power / SM clock of 60 back-to-back C2 steps: full kernels vs kernels without gate math
# (QSV_JIT_DIAG_NOOPS=1: loads, re-layouts, barriers, stores only).  Diagnostic for DESIGN.md section 3.4.
mkdir -p gpurun_out
for tag in full noops; do
  [ $tag = noops ] && export QSV_JIT_DIAG_NOOPS=1
  nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 100 > gpurun_out/power_$tag.log & SMI=$!
  python bench.py --steps 60 --warmup 3 --no-e2e --no-cpu-baseline --traffic off 2>/dev/null | python scripts/pp.py $tag
  kill $SMI
  python - $tag <<'PY'
import sys, statistics
rows = [l.split(",") for l in open(f"gpurun_out/power_{sys.argv[1]}.log") if "," in l]
v = [(float(a), float(b)) for a, b in rows]
hot = [x for x in v if x[1] > 0.6 * max(p for _, p in v)]
print(sys.argv[1], "samples under load", len(hot), "median MHz", statistics.median(a for a, _ in hot), "median W", statistics.median(b for _, b in hot), "max W", max(b for _, b in hot))
PY
done
