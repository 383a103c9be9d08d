"""Multi-rank parity of the product P2P transport on ONE GPU (any box with a B200).

P ranks run as P processes sharing cuda:0, bootstrapped over a gloo group
(sdp4_comm_init_p2p, no NCCL), so the exchange steps of the path -- the qWD all-gather
(Alg. 2 l.4) pulled inside K2, the intra / inter all-to-alls of TLq-HS (Alg. 3 l.4 and
l.10) pushed by K3 / K4 and pulled by K4, the ring's P - 1 quantized hops
(sec. 2.3), the flag protocol and the chunked two-stream overlap -- are checked
bit-exactly against the oracle for every M x N split of P in {2, 4, 8} (incl. the paper's
2 x 4 / 4 x 2 nodes).  See tests/dist_parity.py.
"""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(nproc, extra, port, timeout=1200):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "tests", "dist_parity.py"),
           "--shared-gpu"] + extra
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert r.stdout.count("PASS") >= nproc, r.stdout
    return r.stdout


@pytest.mark.parametrize("nproc", [2, 4, 8])
def test_virtual_all_splits(nproc):
    """Every M dividing P: 1x2, 2x1; 1x4, 2x2, 4x1; 1x8, 2x4, 4x2, 8x1 -- push-only and split
    intra all-to-alls, 1 / 2 / 3 chunks, nearest and stochastic rounding, qwd_step and the two
    qWD calls, TLq-HS (bf16 and fp32 gradients), qW and the ring; plus CUDA-graph replays."""
    out = _run(nproc, ["--splits", "all", "--graph"], 29600 + nproc)
    assert "FAIL" not in out, out


def test_virtual_fullsize_2x4():
    """BASELINE config 2 as the paper splits it -- GPT-1.3B-shaped buffer, 8 ranks as 2 x 4
     -- at FULL size on one GPU, bench.py's calls (qwd_step, TLq-HS 8/4 bits,
    G = 128, b = 64), sampled windows of every shard bit-exact against the oracle."""
    out = _run(8, ["--full", "--splits", "2"], 29640, timeout=1800)
    assert "FAIL" not in out, out
