"""Runs tests/dist_parity.py under torchrun when >= 2 GPUs are visible (NCCL path)."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("nproc,groups", [(2, 1), (2, 2), (4, 2), (4, 1), (4, 4), (8, 2), (8, 4)])
def test_dist_parity(nproc, groups):
    if not torch.cuda.is_available() or torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={29500 + nproc * 10 + groups}",
           os.path.join(ROOT, "tests", "dist_parity.py"), "--groups", str(groups), "--graph"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("PASS") == nproc, r.stdout


@pytest.mark.parametrize("groups", [None])
def test_dist_parity_fullsize(groups):
    """bench.py's GPT-1.3B workload on every visible GPU (2 x (P/2) split), sampled windows."""
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if n < 2:
        pytest.skip("needs 2 GPUs")
    nproc = 8 if n >= 8 else (4 if n >= 4 else 2)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", "--master-port=29777", os.path.join(ROOT, "tests", "dist_parity.py"), "--full"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("PASS") == nproc, r.stdout


@pytest.mark.parametrize("nproc,groups", [(2, 1), (4, 2)])
def test_dist_parity_memop_waits(nproc, groups):
    """The unbounded stream-memop flag waits (timeout 0) give the same results as the default
    polling-kernel waits."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={29560 + nproc}", os.path.join(ROOT, "tests", "dist_parity.py"),
           "--groups", str(groups), "--transports", "p2p", "--wait", "memop", "--graph"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("PASS") == nproc, r.stdout


@pytest.mark.parametrize("fused_limit", [0, 1 << 40])
def test_dist_wait_timeout(fused_limit):
    """Bounded waits on two GPUs: rank 1 skips a collective call; rank 0's polling waits give
    up at the deadline (its stream drains, no hang) and its next call returns SDP4_ETIMEOUT --
    for the multi-launch path's wait kernels (limit 0) and the one-launch kernel's in-kernel
    waits."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={29590 + (fused_limit > 0)}",
           os.path.join(ROOT, "tests", "dist_parity.py"), "--timeout-test", "--fused-limit", str(fused_limit)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("PASS") == 2, r.stdout
