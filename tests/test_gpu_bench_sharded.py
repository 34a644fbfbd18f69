"""`bench.py --gpus N` contract on this one-GPU box: N = 2 and 4 torchrun ranks share GPU 0
(gloo for the bookkeeping collectives - NCCL refuses two ranks on one device; the
data path is the CUDA-IPC peer-memory exchange of the multi-GPU run).  The N = 2
line must carry what the driver's scaling run needs without a code change: the
weak-scaling ladder (n = n_local + log2 N) or the strong mode (fixed n), per-GPU HBM roofline, clocks, e2e, the
exchange-out pass time with its NVLink rate, cpu_baseline and gpu_launches."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,extra,n_expect,scaling", [(2, ["--local-qubits", "24"], 25, "weak"),
                                                          (2, ["--strong", "--qubits", "24"], 24, "strong"),
                                                          (4, ["--local-qubits", "22"], 24, "weak")])
def test_multi_rank_bench_line(world, extra, n_expect, scaling):
    env = dict(os.environ, QSV_SHARE_GPU="1", QSV_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "bench.py"), "--gpus", str(world),
           "--steps", "2", "--warmup", "1", "--cpu-seconds", "2", *extra]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    line = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == world and line["scaling"] == scaling
    cfg = line["config"]
    g = world.bit_length() - 1
    assert cfg["n_qubits"] == n_expect and cfg["n_local"] == n_expect - g
    assert cfg["swaps_per_step"] >= 1 and cfg["fused_exchanges_per_step"] >= 1
    assert cfg["exchange_pass_ms"] > 0 and cfg["nvlink_gbs_per_rank"] > 0 and "nvlink_frac" in cfg
    rf = line["roofline"]
    assert len(rf["per_gpu_gbs"]) == world and all(x and x > 0 for x in rf["per_gpu_gbs"]) and rf["frac"] > 0
    assert line["clocks"]["sm_max_mhz"]
    assert line["e2e"]["value"] > 0 and line["e2e"]["d2h_bytes_per_step"] == 16 << n_expect
    assert line["cpu_baseline"]["value"] > 0
    assert line["gpu_launches"] > 0 and line["value"] > 0
