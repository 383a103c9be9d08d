"""The C ABI library loads and exports every symbol include/sdp4.h declares; host-only
entry points (sizes, layout, validation) behave as documented.  No GPU needed."""
import ctypes
import os
import re

import pytest

import oracle
from paper_2410_15526_b200 import sdp4
from paper_2410_15526_b200.topology import default_split, pad_numel

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "sdp4.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sdp4_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = sdp4.lib()
    syms = declared_symbols()
    assert len(syms) >= 17
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(sdp4.SIGNATURES), "binding and header disagree"
    assert L.sdp4_version() >= 100


@pytest.mark.parametrize("n,k,G", [(131072, 4, 2048), (4096, 8, 128), (4096, 4, 32), (1000 * 64, 32, 128)])
def test_wire_unit_bytes_match_oracle(n, k, G):
    assert sdp4.wire_unit_bytes(n, k, G) == oracle.wire_unit_bytes(n, k, G)


@pytest.mark.parametrize("M,N", [(1, 1), (2, 4), (4, 2), (1, 8), (8, 1)])
def test_workspace_layout(M, N):
    P = M * N
    D = P * 128 * 20
    S = D // P
    w8, w4 = oracle.wire_unit_bytes(S, 8, 128), oracle.wire_unit_bytes(S, 4, 128)
    off = [sdp4.tlq_workspace_offset(M, N, D, 8, 4, 128, r) for r in range(4)]
    assert off[0] == 0
    assert off[1] == (0 if N == 1 else N * M * w8)
    one_chunk = (2 if N > 1 else 1) * N * M * w8 + (2 if M > 1 else 1) * M * w4
    total = sdp4.tlq_workspace_bytes(M, N, D, 8, 4, 128)
    # the size covers any pipeline chunk count (<= 16 chunks, each unit padded to 256 B)
    assert one_chunk <= total <= one_chunk + 16 * (2 * N * M + 2 * M) * 256
    q1 = P * w4
    assert q1 <= sdp4.qwd_workspace_bytes(P, D, 4, 128) <= q1 + 16 * P * 256


def test_validation_errors_before_any_launch():
    # world-1 comm (no NCCL); every call below must be rejected by host validation.
    c = sdp4.Comm()
    L = sdp4.lib()
    st = L.sdp4_tlq_hs_reduce_scatter(c._h, None, 0, 4096, 8, 4, 100, 64, 1, 0, 0, None, None, 0, None)
    assert st == sdp4.EINVAL and b"group" in L.sdp4_last_error()
    st = L.sdp4_tlq_hs_reduce_scatter(c._h, None, 0, 4096 + 64, 8, 4, 128, 64, 1, 0, 0, None, None, 0, None)
    assert st == sdp4.EALIGN
    st = L.sdp4_tlq_hs_reduce_scatter(c._h, None, 0, 4096, 8, 4, 64, 128, 1, 0, 0, None, None, 0, None)
    assert st == sdp4.EALIGN                      # G % b != 0
    st = L.sdp4_tlq_hs_reduce_scatter(c._h, None, 0, 4096, 8, 4, 128, 64, 1, 0, 0, None, None, 0, None)
    assert st == sdp4.EINVAL and b"grad" in L.sdp4_last_error()
    st = L.sdp4_tlq_hs_reduce_scatter(c._h, None, 0, 4096, 5, 4, 128, 64, 1, 0, 0, None, None, 0, None)
    assert st == sdp4.EINVAL
    st = L.sdp4_qwd_quantize(c._h, None, None, 1, 4096, 4, 128, 7, 0, None, 0, None)
    assert st == sdp4.EINVAL and b"rounding" in L.sdp4_last_error()   # unknown rounding mode
    st = L.sdp4_qw_quantize(c._h, None, 4096, 3, 128, 0, 0, None, 0, None)
    assert st == sdp4.EINVAL and b"bits" in L.sdp4_last_error()
    st = L.sdp4_ring_reduce_scatter(c._h, None, 0, 4096, 2, 128, 1, None, None, 0, None)
    assert st == sdp4.EINVAL and b"bits" in L.sdp4_last_error()        # int2 is a weight codec only
    assert L.sdp4_ring_workspace_bytes(4, 4096, 4, 128) == 2 * oracle.wire_unit_bytes(1024, 4, 128)
    assert L.sdp4_wire_unit_bytes(4096, 2, 64) == oracle.wire_unit_bytes(4096, 2, 64)
    st = L.sdp4_tlq_hs_reduce_scatter(c._h, None, 0, 0, 8, 4, 128, 64, 1, 0, 0, None, None, 0, None)
    assert st == sdp4.EALIGN and b"nonzero" in L.sdp4_last_error()      # empty buffers are rejected
    assert L.sdp4_qwd_workspace_bytes(1, 0, 4, 128) == 0
    bad = ctypes.c_void_p()
    assert L.sdp4_comm_init(ctypes.byref(bad), None, 0, 8, 3, 3, 0) == sdp4.EINVAL
    assert L.sdp4_comm_set_chunks(c._h, 17) == sdp4.EINVAL
    assert c.chunks(16384 * 64) == 1          # world 1 never pipelines
    c.close()


def test_topology_helpers():
    assert default_split(8) == (2, 4) and default_split(4) == (2, 2) and default_split(1) == (1, 1)
    assert default_split(8, 4) == (4, 2)
    assert pad_numel(1000, 8, 128) == 1024 and pad_numel(1000, 1, 32) == 1024 and pad_numel(5000, 2, 2048) == 8192
