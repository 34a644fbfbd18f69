mkdir -p gpurun_out
(nproc; free -g; lscpu | head -20; nvidia-smi; df -h /tmp /dev/shm) > gpurun_out/box.txt 2>&1
timeout 1700 python -m pytest tests/test_gpu_c2_n30.py tests/test_gpu_c4_n30.py tests/test_gpu_c3_n32.py tests/test_gpu_sharded_n28.py -q --durations=20 -rs > gpurun_out/big.log 2>&1; echo "big rc=$?"
tail -30 gpurun_out/big.log
