"""Multi-GPU parity (NCCL over NVLink): 1D and every 1.5D grid on the available GPUs, both paths,
against the single-GPU run and the oracle (tools/run_multi.py under torchrun). Skips on boxes
with fewer than 2 GPUs; the schedule itself is pinned on CPU by tests/test_dist_cpu.py."""
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("ngpu,lsa", [(2, False), (4, False), (2, True)], ids=["2", "4", "2-lsa"])
def test_multi_gpu_1d_and_15d(ngpu, lsa):
    """lsa: the opt-in distributed a3/a4 over NCCL symmetric windows (KKM_LSA=1)."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < ngpu:
        pytest.skip(f"needs {ngpu} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={ngpu}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tools", "run_multi.py")]
    env = dict(os.environ, KKM_LSA="1") if lsa else None
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    assert "MULTI OK" in out.stdout, out.stdout[-3000:]
