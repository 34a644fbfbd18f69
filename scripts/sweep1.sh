mkdir -p gpurun_out
for cfg in "1|" "2|" "1|--regs 3" "2|--regs 3" "1|--tile 13" "2|--tile 11"; do
  mb=${cfg%%|*}; args=${cfg#*|}
  QSV_JIT_MIN_BLOCKS=$mb timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline $args > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json;d=json.load(open('gpurun_out/sw.json'));print('$mb','$args',round(d['ms_per_step'],1),d['config']['passes'],d['config']['stages'],round(d['roofline']['frac'],3))" || tail -3 gpurun_out/sw.err
done
