# sharded path on the one GPU (2/4 ranks sharing it: gloo-host and CUDA-IPC P2P transports) + C3's n=32 single-GPU point
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sharded" > gpurun_out/dist_pytest.log 2>&1; echo "sharded rc=$?"; tail -25 gpurun_out/dist_pytest.log
timeout 900 python bench.py --qubits 32 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/b32.json 2> gpurun_out/b32.err; echo "n32 rc=$?"; cat gpurun_out/b32.json; tail -3 gpurun_out/b32.err
