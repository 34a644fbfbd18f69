# BASELINE config 2 "with and without host gate fusion (k = 2..5)": unfused (one kernel per gate,
# the reference's one sweep per gate) and fused passes whose register stages hold k qubits
mkdir -p gpurun_out
run() { timeout 900 env $1 python bench.py $2 --no-e2e --no-cpu-baseline > gpurun_out/fs.json 2>gpurun_out/fs.err
  python -c "import json;d=json.load(open('gpurun_out/fs.json'));c=d['config'];r=d['roofline'];print(json.dumps({'args':'$2','ms_per_step':round(d['ms_per_step'],2),'value':d['value'],'passes':c['passes'],'stages':c['stages'],'tile':c['tile_qubits'],'regs':c['reg_qubits'],'avg_launch_ms':round(r['avg_launch_ms'],3),'frac':round(r['frac'],3),'launches':d['gpu_launches']}))" || tail -3 gpurun_out/fs.err; }
run "" "--unfused --steps 1 --warmup 1"
run "" "--regs 2 --steps 3 --warmup 2"
run "" "--regs 3 --steps 3 --warmup 2"
run "" "--regs 4 --steps 3 --warmup 2"
run "" "--regs 5 --steps 3 --warmup 2"
