"""Multi-GPU CP parity under ``pytest -m gpu`` (skipped on boxes with fewer
GPUs than the case needs): tests/cp_multi_gpu_worker.py under torchrun at
N = 2 / 4 / 8, through the copy-engine and NCCL transports, at the full
config-4 shape (128K EMU multi-image mask, GQA 32q/8kv), checked against the
fp32 oracle on sampled rows and against the single-GPU path on every row."""

import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("transport", ["ce", "nccl"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_cp_multi_gpu_config4_parity(world, transport):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs (have {torch.cuda.device_count()})")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1", f"--master-port={_port()}",
           os.path.join(ROOT, "tests", "cp_multi_gpu_worker.py"), "--transport", transport]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert r.returncode == 0 and lines, f"rc={r.returncode}\n{r.stdout[-3000:]}\n{r.stderr[-3000:]}"
    rep = json.loads(lines[-1])
    assert rep["ok"] and rep["world"] == world and rep["transport"] == transport
    out = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, f"cp_multi_n{world}_{transport}.json"), "w") as fh:
        fh.write(lines[-1] + "\n")
