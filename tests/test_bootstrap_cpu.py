"""Host-side bootstrap of the P2P-only comm (sdp4_comm_init_p2p) on CPU, no GPU: the
library's collective host exchanges (reachability records, agreement on one status byte per
rank) run through the Python gloo callback, in real multi-process gloo groups.  Without a
GPU no rank can map another's memory, so every rank must get the same ESTATE -- agreed,
never a hang or a split decision -- and world-1 comms and the new knobs behave as the header
says (include/sdp4.h: sdp4_comm_init_p2p, sdp4_comm_set_timeout, sdp4_comm_check)."""
import ctypes
import os
import socket
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _bootstrap_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    from paper_2410_15526_b200 import Comm, SDP4Error, sdp4
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        try:
            Comm.from_process_group(1, bootstrap="host")
            q.put((rank, "created"))
        except SDP4Error as ex:
            q.put((rank, ex.status, str(ex)))
        # the callback itself: a rank-major byte gather over the group
        cb = sdp4._gloo_allgather(None)
        send = ctypes.create_string_buffer(bytes([rank + 1] * 5), 5)
        recv = ctypes.create_string_buffer(5 * world)
        rc = cb(ctypes.addressof(send), ctypes.addressof(recv), 5, None)
        q.put((rank, "gather", rc, list(recv.raw)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_p2p_bootstrap_agrees_on_failure_without_gpu(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bootstrap_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0, "a rank hung or crashed in the bootstrap"
    res = [q.get(timeout=10) for _ in range(2 * world)]
    inits = sorted(r for r in res if r[1] != "gather")
    gathers = sorted(r for r in res if r[1] == "gather")
    from paper_2410_15526_b200 import sdp4
    assert [r[0] for r in inits] == list(range(world))
    assert all(r[1] == sdp4.ESTATE and "P2P transport unavailable" in r[2] for r in inits), inits
    want = [b for r in range(world) for b in [r + 1] * 5]
    assert all(g[2] == 0 and g[3] == want for g in gathers), gathers


def test_world1_p2p_comm_and_knobs():
    from paper_2410_15526_b200 import sdp4
    L = sdp4.lib()
    h = ctypes.c_void_p()
    assert L.sdp4_comm_init_p2p(ctypes.byref(h), 0, 1, 1, 1, sdp4.HOST_ALLGATHER_FN(), None) == sdp4.OK
    assert L.sdp4_comm_check(h) == sdp4.OK
    assert L.sdp4_comm_set_timeout(h, 0.0) == sdp4.OK
    assert L.sdp4_comm_set_timeout(h, -1.0) == sdp4.EINVAL
    assert L.sdp4_comm_set_transport(h, 1) == sdp4.EINVAL          # world 1: no P2P transport
    assert L.sdp4_comm_destroy(h) == sdp4.OK
    bad = ctypes.c_void_p()
    # world > 1 needs the host allgather callback; M * N must equal world
    assert L.sdp4_comm_init_p2p(ctypes.byref(bad), 0, 2, 1, 2, sdp4.HOST_ALLGATHER_FN(), None) == sdp4.EINVAL
    assert L.sdp4_comm_init_p2p(ctypes.byref(bad), 0, 4, 3, 2, sdp4.HOST_ALLGATHER_FN(), None) == sdp4.EINVAL
    assert L.sdp4_comm_check(None) == sdp4.EINVAL
