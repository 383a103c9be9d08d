"""Thin ctypes binding of libsdp4 (include/sdp4.h).

Argument marshalling only: torch tensors are turned into device pointers and the
current CUDA stream; every step of the hot path runs in libsdp4's kernels and NCCL
calls.  There is no fallback: if libsdp4.so is missing or a call fails, an
exception is raised.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import torch

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libsdp4.so")

OK, EINVAL, EALIGN, ECUDA, ENCCL, ESTATE, ETIMEOUT = range(7)
F32, BF16 = 0, 1
RNE, STOCHASTIC = 0, 1
UNIQUE_ID_BYTES = 128

_DT = {torch.float32: F32, torch.bfloat16: BF16}
_ESZ = {F32: 4, BF16: 2}

_c_size = ctypes.c_size_t
_vp = ctypes.c_void_p
_ci = ctypes.c_int
_u64 = ctypes.c_uint64
# sdp4_host_allgather_fn: int (*)(const void* send, void* recv, size_t bytes, void* ctx)
HOST_ALLGATHER_FN = ctypes.CFUNCTYPE(_ci, _vp, _vp, _c_size, _vp)

# name -> (restype, argtypes): exactly the entry points of include/sdp4.h
SIGNATURES = {
    "sdp4_version": (_ci, []),
    "sdp4_last_error": (ctypes.c_char_p, []),
    "sdp4_get_unique_id": (_ci, [ctypes.c_char_p]),
    "sdp4_comm_init": (_ci, [ctypes.POINTER(_vp), ctypes.c_char_p, _ci, _ci, _ci, _ci, _ci]),
    "sdp4_comm_init_p2p": (_ci, [ctypes.POINTER(_vp), _ci, _ci, _ci, _ci, HOST_ALLGATHER_FN, _vp]),
    "sdp4_comm_destroy": (_ci, [_vp]),
    "sdp4_comm_set_timeout": (_ci, [_vp, ctypes.c_double]),
    "sdp4_comm_check": (_ci, [_vp]),
    "sdp4_comm_set_chunks": (_ci, [_vp, _ci]),
    "sdp4_comm_chunks": (_ci, [_vp, _c_size, _ci]),
    "sdp4_comm_set_transport": (_ci, [_vp, _ci]),
    "sdp4_comm_transport": (_ci, [_vp]),
    "sdp4_comm_set_intra_pull": (_ci, [_vp, _ci, _ci]),
    "sdp4_comm_set_fused_limit": (_ci, [_vp, _c_size]),
    "sdp4_comm_set_local_fusion": (_ci, [_vp, _ci]),
    "sdp4_wire_unit_bytes": (_c_size, [_c_size, _ci, _ci]),
    "sdp4_qwd_workspace_bytes": (_c_size, [_ci, _c_size, _ci, _ci]),
    "sdp4_tlq_workspace_bytes": (_c_size, [_ci, _ci, _c_size, _ci, _ci, _ci]),
    "sdp4_tlq_workspace_offset": (_c_size, [_ci, _ci, _c_size, _ci, _ci, _ci, _ci]),
    "sdp4_qwd_quantize": (_ci, [_vp, _vp, _vp, _ci, _c_size, _ci, _ci, _ci, _u64, _vp, _c_size, _vp]),
    "sdp4_qwd_allgather_apply": (_ci, [_vp, _vp, _c_size, _c_size, _ci, _ci, _vp, _ci, _vp]),
    "sdp4_qwd_step": (_ci, [_vp, _vp, _vp, _ci, _c_size, _ci, _ci, _ci, _u64, _vp, _c_size, _vp]),
    "sdp4_qw_quantize": (_ci, [_vp, _vp, _c_size, _ci, _ci, _ci, _u64, _vp, _c_size, _vp]),
    "sdp4_qw_allgather_apply": (_ci, [_vp, _vp, _c_size, _c_size, _ci, _ci, _vp, _ci, _vp]),
    "sdp4_ring_workspace_bytes": (_c_size, [_ci, _c_size, _ci, _ci]),
    "sdp4_ring_reduce_scatter": (_ci, [_vp, _vp, _ci, _c_size, _ci, _ci, _ci, _vp, _vp, _c_size, _vp]),
    "sdp4_tlq_hs_reduce_scatter": (_ci, [_vp, _vp, _ci, _c_size, _ci, _ci, _ci, _ci, _ci, _ci, _u64, _vp, _vp,
                                         _c_size, _vp]),
    "sdp4_tlq_stage_quantize": (_ci, [_vp, _ci, _c_size, _ci, _ci, _ci, _ci, _ci, _ci, _u64, _ci, _vp, _vp]),
    "sdp4_tlq_stage_quantize_reduce": (_ci, [_vp, _ci, _c_size, _ci, _ci, _ci, _ci, _u64, _ci, _vp, _vp]),
    "sdp4_tlq_stage_reduce": (_ci, [_vp, _c_size, _ci, _ci, _ci, _ci, _ci, _ci, _u64, _ci, _vp, _vp]),
    "sdp4_tlq_stage_final": (_ci, [_vp, _c_size, _ci, _ci, _ci, _ci, _ci, _ci, _vp, _vp]),
    "sdp4_emu_qwd_workspace_bytes": (_c_size, [_ci, _c_size, _ci, _ci]),
    "sdp4_emu_qwd_step": (_ci, [_ci, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _ci, _c_size, _ci, _ci, _ci, _u64,
                                _ci, _vp, _c_size, _vp]),
    "sdp4_emu_tlq_workspace_bytes": (_c_size, [_ci, _ci, _c_size, _ci, _ci, _ci]),
    "sdp4_emu_tlq_hs_reduce_scatter": (_ci, [_ci, _ci, ctypes.POINTER(_vp), _ci, _c_size, _ci, _ci, _ci, _ci, _ci,
                                             _ci, _u64, ctypes.POINTER(_vp), _ci, _vp, _c_size, _vp]),
    "sdp4_launch_count": (_u64, [_vp, _ci]),
    "sdp4_profile_enable": (_ci, [_vp, _ci]),
    "sdp4_profile_read": (_ci, [_vp, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_double),
                                ctypes.POINTER(_u64), _ci, ctypes.POINTER(_ci)]),
    "sdp4_nccl_reduce_scatter": (_ci, [_vp, _vp, _vp, _c_size, _ci, _ci, _vp]),
    "sdp4_nccl_all_gather": (_ci, [_vp, _vp, _vp, _c_size, _ci, _vp]),
}

_lib = None


class SDP4Error(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"libsdp4 status {status}: {msg}")
        self.status = status


def lib() -> ctypes.CDLL:
    """Load libsdp4.so (built in-tree by paper_2410_15526_b200.build).  Fails loudly."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is not built; run `python -m paper_2410_15526_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(status: int):
    if status != OK:
        raise SDP4Error(status, lib().sdp4_last_error().decode())


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_contiguous():
        raise ValueError("tensors passed to libsdp4 must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _nbytes(t: Optional[torch.Tensor]) -> int:
    return 0 if t is None else t.numel() * t.element_size()


def _stream(stream) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def wire_unit_bytes(n: int, bits: int, group: int) -> int:
    return lib().sdp4_wire_unit_bytes(n, bits, group)


def qwd_workspace_bytes(world: int, numel: int, bits: int, group: int) -> int:
    return lib().sdp4_qwd_workspace_bytes(world, numel, bits, group)


def ring_workspace_bytes(world: int, numel: int, bits: int, group: int) -> int:
    return lib().sdp4_ring_workspace_bytes(world, numel, bits, group)


def tlq_workspace_bytes(M: int, N: int, numel: int, bits_intra: int, bits_inter: int, group: int) -> int:
    return lib().sdp4_tlq_workspace_bytes(M, N, numel, bits_intra, bits_inter, group)


def tlq_workspace_offset(M, N, numel, bits_intra, bits_inter, group, region) -> int:
    return lib().sdp4_tlq_workspace_offset(M, N, numel, bits_intra, bits_inter, group, region)


def tlq_stage_quantize(grad: torch.Tensor, intra_send: torch.Tensor, M: int, N: int, bits_intra: int = 8,
                       group: int = 128, hadamard_block: int = 64, seed=None, rank: int = 0, stream=None):
    """K3 alone (Alg. 3 l.2-3) on rank `rank`'s gradient, no communication.  seed: stochastic
    rounding (R14) with that seed; None: round to nearest even."""
    _check(lib().sdp4_tlq_stage_quantize(_ptr(grad), _DT[grad.dtype], grad.numel(), M, N, bits_intra, group,
                                         hadamard_block, RNE if seed is None else STOCHASTIC, seed or 0, rank,
                                         _ptr(intra_send), _stream(stream)))


def tlq_stage_reduce(intra_recv: torch.Tensor, inter_send: torch.Tensor, numel: int, M: int, N: int,
                     bits_intra: int = 8, bits_inter: int = 4, group: int = 128, seed=None, rank: int = 0,
                     stream=None):
    """K4 alone (Alg. 3 l.5, 7, 9) for rank `rank`, no communication."""
    _check(lib().sdp4_tlq_stage_reduce(_ptr(intra_recv), numel, M, N, bits_intra, bits_inter, group,
                                       RNE if seed is None else STOCHASTIC, seed or 0, rank, _ptr(inter_send),
                                       _stream(stream)))


def tlq_stage_quantize_reduce(grad: torch.Tensor, inter_send: torch.Tensor, M: int, group: int = 128,
                              hadamard_block: int = 64, seed=None, rank: int = 0, stream=None):
    """K34 alone (one GPU per group, N = 1, bits 8 / 4): Alg. 3 l.2-9 for node `rank`,
    no communication -- every 4-bit unit into inter_send (M units)."""
    _check(lib().sdp4_tlq_stage_quantize_reduce(_ptr(grad), _DT[grad.dtype], grad.numel(), M, group, hadamard_block,
                                                RNE if seed is None else STOCHASTIC, seed or 0, rank,
                                                _ptr(inter_send), _stream(stream)))


def tlq_stage_final(inter_recv: torch.Tensor, out_shard: torch.Tensor, numel: int, M: int, N: int,
                    bits_inter: int = 4, group: int = 128, hadamard_block: int = 64, average: bool = True,
                    stream=None):
    """K5 alone (Alg. 3 l.11-13) for one rank, no communication."""
    _check(lib().sdp4_tlq_stage_final(_ptr(inter_recv), numel, M, N, bits_inter, group, hadamard_block,
                                      int(bool(average)), _ptr(out_shard), _stream(stream)))


def _ptr_array(ts):
    return (_vp * len(ts))(*[_ptr(t) for t in ts])


def emu_qwd_workspace_bytes(world: int, numel: int, bits: int = 4, group: int = 128) -> int:
    return lib().sdp4_emu_qwd_workspace_bytes(world, numel, bits, group)


def emu_qwd_step(w_main_shards, w_models, workspace: torch.Tensor, bits: int = 4, group: int = 128, seed=None,
                 fresh: bool = True, stream=None):
    """The one-launch qWD step of every rank of an emulated job in one launch on this device
    (sdp4_emu_qwd_step): w_models[q] is updated as rank q's replica."""
    P = len(w_main_shards)
    _check(lib().sdp4_emu_qwd_step(P, _ptr_array(w_main_shards), _ptr_array(w_models), _DT[w_models[0].dtype],
                                   w_models[0].numel(), bits, group, RNE if seed is None else STOCHASTIC, seed or 0,
                                   int(bool(fresh)), _ptr(workspace), _nbytes(workspace), _stream(stream)))


def emu_tlq_workspace_bytes(M: int, N: int, numel: int, bits_intra: int = 8, bits_inter: int = 4,
                            group: int = 128) -> int:
    return lib().sdp4_emu_tlq_workspace_bytes(M, N, numel, bits_intra, bits_inter, group)


def emu_tlq_hs_reduce_scatter(M: int, N: int, grads, out_shards, workspace: torch.Tensor, bits_intra: int = 8,
                              bits_inter: int = 4, group: int = 128, hadamard_block: int = 64,
                              average: bool = True, seed=None, fresh: bool = True, stream=None):
    """The one-launch TLq-HS of every rank of an emulated M x N job in one launch on this device
    (sdp4_emu_tlq_hs_reduce_scatter): out_shards[q] receives rank q's shard."""
    _check(lib().sdp4_emu_tlq_hs_reduce_scatter(M, N, _ptr_array(grads), _DT[grads[0].dtype], grads[0].numel(),
                                                bits_intra, bits_inter, group, hadamard_block, int(bool(average)),
                                                RNE if seed is None else STOCHASTIC, seed or 0,
                                                _ptr_array(out_shards), int(bool(fresh)), _ptr(workspace),
                                                _nbytes(workspace), _stream(stream)))


def get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(UNIQUE_ID_BYTES)
    _check(lib().sdp4_get_unique_id(buf))
    return buf.raw


def _gloo_allgather(group):
    """A sdp4_host_allgather_fn over a torch.distributed process group (the host bootstrap of
    sdp4_comm_init_p2p): byte buffers gathered rank-major.  Argument marshalling only."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else None

    def cb(send, recv, nbytes, ctx):
        try:
            src = torch.frombuffer(bytearray(ctypes.string_at(send, nbytes)), dtype=torch.uint8) if nbytes \
                else torch.zeros(0, dtype=torch.uint8)
            if dev is not None:
                src = src.to(dev)
            outs = [torch.empty_like(src) for _ in range(world)]
            dist.all_gather(outs, src, group=group)
            for r, o in enumerate(outs):
                if nbytes:
                    b = bytes(o.cpu().numpy().tobytes())
                    ctypes.memmove(recv + r * nbytes, b, nbytes)
            return 0
        except Exception as ex:  # noqa: BLE001 -- reported as a nonzero status to the library
            import sys
            print(f"libsdp4 host allgather failed: {ex!r}", file=sys.stderr)
            return 1
    return HOST_ALLGATHER_FN(cb)


class Comm:
    """sdp4_comm_t: world + intra (N) + inter (M) NCCL communicators, or a P2P-only comm
    bootstrapped over a host channel (sdp4_comm_init_p2p).  Destroy it with close() on every
    rank (collective); a Comm that is garbage-collected unclosed is leaked, never destroyed,
    because destruction is a collective."""

    def __init__(self, rank: int = 0, world: int = 1, groups: int = 1, group_size: int = 1,
                 unique_id: Optional[bytes] = None, nccl_ctas: int = 0, chunks: int = 0,
                 host_allgather=None):
        self.rank, self.world, self.M, self.N = rank, world, groups, group_size
        self._h = ctypes.c_void_p()
        self._ag = host_allgather          # keeps the ctypes callback alive
        if host_allgather is not None:
            _check(lib().sdp4_comm_init_p2p(ctypes.byref(self._h), rank, world, groups, group_size, host_allgather,
                                            None))
        else:
            uid = None if unique_id is None else ctypes.create_string_buffer(unique_id, UNIQUE_ID_BYTES)
            _check(lib().sdp4_comm_init(ctypes.byref(self._h), uid, rank, world, groups, group_size, nccl_ctas))
        if chunks:
            self.set_chunks(chunks)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def set_timeout(self, seconds: float):
        """Deadline of the P2P flag waits (0 = unbounded stream-memop waits); see sdp4_comm_set_timeout."""
        _check(lib().sdp4_comm_set_timeout(self._h, float(seconds)))

    def check(self):
        """Raise SDP4Error if an earlier call failed asynchronously (P2P wait timeout, NCCL)."""
        _check(lib().sdp4_comm_check(self._h))

    def set_chunks(self, chunks: int):
        """Pipeline chunk count (0 = automatic, 1 = off); see sdp4_comm_set_chunks."""
        _check(lib().sdp4_comm_set_chunks(self._h, chunks))

    TRANSPORTS = {"nccl": 0, "p2p": 1}

    def set_transport(self, transport):
        """'nccl' or 'p2p' (fused NVLink push); see sdp4_comm_set_transport."""
        _check(lib().sdp4_comm_set_transport(self._h, self.TRANSPORTS.get(transport, transport)))

    def set_intra_pull(self, num: int, den: int):
        """P2P: share num/den of the peer tiles of the intra all-to-all pulled by K4 (the rest
        pushed by K3); see sdp4_comm_set_intra_pull."""
        _check(lib().sdp4_comm_set_intra_pull(self._h, num, den))

    def set_fused_limit(self, numel: int):
        """P2P calls on at most `numel` elements run as one kernel per rank (0: never); see
        sdp4_comm_set_fused_limit."""
        _check(lib().sdp4_comm_set_fused_limit(self._h, numel))

    def set_local_fusion(self, enable: bool):
        """World size 1: TLq-HS (8/4 bits) as one kernel (default) or K3 + K4 + K5; see
        sdp4_comm_set_local_fusion."""
        _check(lib().sdp4_comm_set_local_fusion(self._h, int(bool(enable))))

    @property
    def transport(self) -> str:
        return {0: "nccl", 1: "p2p"}.get(lib().sdp4_comm_transport(self._h), "?")

    def chunks(self, numel: int, group: int = 128) -> int:
        return int(lib().sdp4_comm_chunks(self._h, numel, group))

    @classmethod
    def from_process_group(cls, groups: Optional[int] = None, device=None, nccl_ctas: int = 0,
                           chunks: int = 0, bootstrap: str = "nccl", group=None) -> "Comm":
        """Bootstrap from torch.distributed; groups defaults to the topology of
        topology.default_split.  bootstrap="nccl": rank 0 draws an NCCL unique id and broadcasts
        it (sdp4_comm_init).  bootstrap="host": a P2P-only comm whose CUDA-IPC handles travel over
        the process group (sdp4_comm_init_p2p) -- no NCCL, so several ranks may share one GPU."""
        import torch.distributed as dist
        from .topology import default_split
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        M, N = default_split(world, groups)
        if bootstrap == "host":
            return cls(rank, world, M, N, chunks=chunks, host_allgather=_gloo_allgather(group))
        uid = None
        if world > 1:
            t = torch.zeros(UNIQUE_ID_BYTES, dtype=torch.uint8)
            if rank == 0:
                t = torch.frombuffer(bytearray(get_unique_id()), dtype=torch.uint8)
            if dist.get_backend(group) == "nccl":
                t = t.to(device or torch.device("cuda", torch.cuda.current_device()))
            dist.broadcast(t, dist.get_global_rank(group, 0) if group is not None else 0, group=group)
            uid = bytes(t.cpu().tolist())
        return cls(rank, world, M, N, uid, nccl_ctas, chunks)

    def close(self):
        if self._h:
            _check(lib().sdp4_comm_destroy(self._h))
            self._h = ctypes.c_void_p()

    def __del__(self):
        # sdp4_comm_destroy is collective (a barrier with the peers when symmetric buffers
        # exist): running it from a garbage collector on one rank could hang, so an unclosed
        # multi-rank comm is leaked; a single-rank one is destroyed (nothing collective).
        try:
            if self._h and self.world == 1:
                self.close()
        except Exception:
            pass

    # -- sizes -------------------------------------------------------------------
    def qwd_workspace_bytes(self, numel: int, bits: int = 4, group: int = 128) -> int:
        return qwd_workspace_bytes(self.world, numel, bits, group)

    def tlq_workspace_bytes(self, numel: int, bits_intra: int = 8, bits_inter: int = 4, group: int = 128) -> int:
        return tlq_workspace_bytes(self.M, self.N, numel, bits_intra, bits_inter, group)

    def workspace(self, nbytes: int, device=None) -> torch.Tensor:
        return torch.empty(nbytes, dtype=torch.uint8, device=device or "cuda")

    # -- qWD (Alg. 2 l.2-5) ----------------------------------------------------------
    def qwd_quantize(self, w_main_shard: torch.Tensor, w_model: torch.Tensor, workspace: Optional[torch.Tensor],
                     bits: int = 4, group: int = 128, seed=None, stream=None):
        """seed: stochastic rounding (R14) with this seed; None: round to nearest even."""
        if w_main_shard.dtype != torch.float32:
            raise TypeError("w_main_shard must be fp32 (P:211)")
        _check(lib().sdp4_qwd_quantize(self._h, _ptr(w_main_shard), _ptr(w_model), _DT[w_model.dtype],
                                       w_model.numel(), bits, group, RNE if seed is None else STOCHASTIC,
                                       seed or 0, _ptr(workspace), _nbytes(workspace), _stream(stream)))

    def qwd_allgather_apply(self, workspace: Optional[torch.Tensor], w_model: torch.Tensor, bits: int = 4,
                            group: int = 128, stream=None):
        _check(lib().sdp4_qwd_allgather_apply(self._h, _ptr(workspace), _nbytes(workspace), w_model.numel(), bits,
                                              group, _ptr(w_model), _DT[w_model.dtype], _stream(stream)))

    def qwd_step(self, w_main_shard: torch.Tensor, w_model: torch.Tensor, workspace: Optional[torch.Tensor],
                 bits: int = 4, group: int = 128, seed=None, stream=None):
        """Alg. 2 l.2-5 in one call (qwd_quantize + qwd_allgather_apply, bit-identical), the
        owner's own update fused into K1."""
        if w_main_shard.dtype != torch.float32:
            raise TypeError("w_main_shard must be fp32 (P:211)")
        _check(lib().sdp4_qwd_step(self._h, _ptr(w_main_shard), _ptr(w_model), _DT[w_model.dtype], w_model.numel(),
                                   bits, group, RNE if seed is None else STOCHASTIC, seed or 0, _ptr(workspace),
                                   _nbytes(workspace), _stream(stream)))

    # -- ablation baselines ---------------------------------------------
    def qw_quantize(self, w_main_shard: torch.Tensor, numel: int, workspace: Optional[torch.Tensor], bits: int = 4,
                    group: int = 128, seed=None, stream=None):
        """qW (Alg. 1, QSDP / ZeRO++): quantize the main-weight shard itself."""
        if w_main_shard.dtype != torch.float32:
            raise TypeError("w_main_shard must be fp32 (P:211)")
        _check(lib().sdp4_qw_quantize(self._h, _ptr(w_main_shard), numel, bits, group,
                                      RNE if seed is None else STOCHASTIC, seed or 0, _ptr(workspace),
                                      _nbytes(workspace), _stream(stream)))

    def qw_allgather_apply(self, workspace: Optional[torch.Tensor], w_model: torch.Tensor, bits: int = 4, group: int = 128,
                           stream=None):
        """qW all-gather + dequantize: the replica becomes the gathered quantized weights."""
        _check(lib().sdp4_qw_allgather_apply(self._h, _ptr(workspace), _nbytes(workspace), w_model.numel(), bits,
                                             group, _ptr(w_model), _DT[w_model.dtype], _stream(stream)))

    def ring_workspace_bytes(self, numel: int, bits: int = 4, group: int = 128) -> int:
        return ring_workspace_bytes(self.world, numel, bits, group)

    def ring_reduce_scatter(self, grad: torch.Tensor, out_shard: torch.Tensor, workspace: Optional[torch.Tensor],
                            bits: int = 4, group: int = 128, average: bool = True, stream=None):
        """Ring reduce-scatter with per-hop quantization (sec. 2.3), ablation baseline."""
        if out_shard.dtype != torch.float32:
            raise TypeError("out_shard must be fp32")
        _check(lib().sdp4_ring_reduce_scatter(self._h, _ptr(grad), _DT[grad.dtype], grad.numel(), bits, group,
                                              int(bool(average)), _ptr(out_shard), _ptr(workspace),
                                              _nbytes(workspace), _stream(stream)))

    # -- TLq-HS (Alg. 3) -------------------------------------------------------------
    def tlq_hs_reduce_scatter(self, grad: torch.Tensor, out_shard: torch.Tensor, workspace: Optional[torch.Tensor],
                              bits_intra: int = 8, bits_inter: int = 4, group: int = 128,
                              hadamard_block: int = 64, average: bool = True, seed=None, stream=None):
        """seed: stochastic rounding (R14) of both quantizers with this seed; None: nearest even."""
        if out_shard.dtype != torch.float32:
            raise TypeError("out_shard must be fp32")
        _check(lib().sdp4_tlq_hs_reduce_scatter(self._h, _ptr(grad), _DT[grad.dtype], grad.numel(), bits_intra,
                                                bits_inter, group, hadamard_block, int(bool(average)),
                                                RNE if seed is None else STOCHASTIC, seed or 0,
                                                _ptr(out_shard), _ptr(workspace), _nbytes(workspace),
                                                _stream(stream)))

    # -- instrumentation -------------------------------------------------------------
    def launch_count(self, reset: bool = False) -> int:
        return int(lib().sdp4_launch_count(self._h, int(reset)))

    def profile_enable(self, enable: bool = True):
        _check(lib().sdp4_profile_enable(self._h, int(enable)))

    def profile_read(self) -> dict:
        n = 16
        names = (ctypes.c_char_p * n)()
        ms = (ctypes.c_double * n)()
        cnt = (ctypes.c_uint64 * n)()
        k = ctypes.c_int(0)
        _check(lib().sdp4_profile_read(self._h, names, ms, cnt, n, ctypes.byref(k)))
        return {names[i].decode(): (ms[i], int(cnt[i])) for i in range(k.value)}

    # -- unquantized comparators (sec. 2.1) -----------------------------------
    def nccl_reduce_scatter(self, send: torch.Tensor, recv: torch.Tensor, average: bool = True, stream=None):
        _check(lib().sdp4_nccl_reduce_scatter(self._h, _ptr(send), _ptr(recv), send.numel(), _DT[send.dtype],
                                              int(average), _stream(stream)))

    def nccl_all_gather(self, send: torch.Tensor, recv: torch.Tensor, stream=None):
        _check(lib().sdp4_nccl_all_gather(self._h, _ptr(send), _ptr(recv), recv.numel(), _DT[send.dtype],
                                          _stream(stream)))
