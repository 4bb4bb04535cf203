"""GPU: bench.py's multi-process path (torchrun, one process per rank, CUDA-IPC
symmetric heap) end to end, in its shared-GPU test mode (two ranks
time-slicing the test box's one GPU, gloo plumbing).  Guards the N > 1 code
the driver's scaling run takes: world creation + handle exchange, every
timed section, the host-streaming e2e, max-over-ranks, one JSON line."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def test_bench_two_processes_shared_gpu():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, TFB_BENCH_SHARED_GPU="1", TILEFABRIC_WATCHDOG_SECS="60")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2", "--steps", "2",
           "--warmup", "3", "--no-cpu", "--cooldown", "0", "--no-sweep"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["config"]["world_size"] == 2
    assert line["e2e"]["matches_device_run"] is True
    # W > 1: sampled rows of C against an fp32 product of the NCCL(gloo)-gathered operand
    assert line["numerics"]["ag_sampled_rows_norm_err"] <= 4e-3
    assert line["nvlink"]["bytes_per_rank"] > 0
    for k in ("fd_config3_b1_L128k", "fd_config4_b32_L32k"):
        sec = line["secondary"][k]
        assert sec["fused_us"] > 0 and sec["nccl_bsp_us"] > 0
        assert sec["numerics"]["fused_equals_nccl_bsp_bitwise"] is True
        assert sec["numerics"]["bf16"]["head_rel_err"] <= sec["numerics"]["bf16"]["tol"]
        assert sec["numerics"]["f32"]["head_rel_err"] <= sec["numerics"]["f32"]["tol"]
