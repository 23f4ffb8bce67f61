"""Multi-GPU Parareal (NCCL or peer-store hand-off) — runs tools/mgpu_check.py under torchrun
when at least 2 GPUs are visible; W-invariance is bitwise, oracle parity 1e-12."""
import json
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def ngpus():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


CASES = [(2, 32, 4, 2, 0.0), (2, 32, 2, 2, 0.0), (2, 40, 4, 3, 0.0), (4, 32, 4, 2, 0.0), (4, 32, 8, 3, 0.0),
         (8, 32, 8, 3, 0.0), (2, 128, 2, 1, 0.0), (2, 32, 4, 4, 3e-3), (4, 32, 4, 4, 3e-3)]
PEER = [(2, 32, 4, 2, 0.0), (2, 40, 4, 3, 0.0), (4, 32, 8, 3, 0.0), (2, 128, 2, 1, 0.0),
        (2, 32, 4, 4, 3e-3), (4, 32, 4, 4, 3e-3)]


@pytest.mark.parametrize("W,n,Np,K,tol,handoff", [c + ("nccl",) for c in CASES] + [c + ("peer",) for c in PEER])
def test_parareal_multi_gpu(W, n, Np, K, tol, handoff):
    """Each case runs pr_parareal twice (second call: same buffers, next sequence
    epoch) and compares with one GPU (bitwise) and the oracle.  `peer`: the
    correction kernel stores the hand-off into the successor's buffer over
    NVLink (PR_FLAG_PEER_HANDOFF) instead of ncclSend/ncclRecv."""
    if ngpus() < W:
        pytest.skip(f"needs {W} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={W}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "tools", "mgpu_check.py"), str(n), str(Np), str(K), str(tol), handoff]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert res.returncode == 0 and lines, res.stdout[-3000:] + res.stderr[-3000:]
    info = json.loads(lines[-1])
    assert info["ok"] and info["bitwise_equal_to_1gpu"], info


@pytest.mark.parametrize("handoff", ["nccl", "peer"])
@pytest.mark.parametrize("W,K", [(2, 1000), (4, 350)])
def test_multi_gpu_handoff_stress(W, K, handoff):
    """~10^3 hand-offs between processes on different GPUs (n = 32, N_p = W, K iterations on
    a 64-step horizon, two calls): u_T and every d^k bitwise equal to the one-GPU run of the
    same slices, so the NCCL and the peer-store paths agree with each other bit for bit."""
    if ngpus() < W:
        pytest.skip(f"needs {W} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={W}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "tools", "mgpu_check.py"), "32", str(W), str(K), "0", handoff, "stress"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert res.returncode == 0 and lines, res.stdout[-3000:] + res.stderr[-3000:]
    info = json.loads(lines[-1])
    assert info["ok"] and info["bitwise_equal_to_1gpu"] and info["repeat_equal"], \
        {k: info[k] for k in info if k != "defects"}


@pytest.mark.parametrize("handoff", ["nccl"])
def test_stuck_predecessor_nccl(handoff):
    """Rank 0 never sends: rank 1's pr_parareal returns PR_ENCCL with its rank and
    iteration after PR_NCCL_TIMEOUT_S (tools/mgpu_stuck.py)."""
    if ngpus() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "tools", "mgpu_stuck.py"), handoff]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert res.returncode == 0 and lines, res.stdout[-3000:] + res.stderr[-3000:]
    assert json.loads(lines[-1])["ok"]
