"""NEXT-4: the sharded SGD harness (Alg. 2 / Alg. 4, examples/sgd_harness.py) on a synthetic
least-squares task through the library: TLq-HS gradients + qWD weights converge like the
lossless run, the replica stays close to the main weights (e_t drift) -- much
closer than with direct weight quantization qW -- and replicas stay identical on every rank."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def check(res):
    ex = res["exact+exact"]["final_loss"]
    for k in ("qwd+tlq_hs", "qw+tlq_hs"):
        assert res[k]["final_loss"] < 1.5 * ex, (k, res)
        assert res[k]["replicas_identical"], k
    assert res["qwd+tlq_hs"]["max_drift"] < res["qw+tlq_hs"]["max_drift"] / 3, res


def test_sgd_harness_single_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sys.path.insert(0, ROOT)
    from examples.sgd_harness import run
    from paper_2410_15526_b200 import Comm
    comm = Comm()
    res = {}
    for mode, grad in (("exact", "exact"), ("qwd", "tlq_hs"), ("qw", "tlq_hs")):
        hist, same = run(comm, steps=150, mode=mode, grad=grad)
        res[f"{mode}+{grad}"] = {"final_loss": hist[-1]["loss"], "max_drift": max(h["drift"] for h in hist[5:]),
                                 "replicas_identical": same}
    comm.close()
    check(res)


def test_sgd_harness_two_gpus():
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29791", os.path.join(ROOT, "examples", "sgd_harness.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    check(json.loads(lines[-1]))
