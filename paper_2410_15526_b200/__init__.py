"""paper_2410_15526_b200 -- SDP4Bit (arXiv 2410.15526) data-parallel communication hot path on B200.

qWD all-gather (Alg. 2 l.2-5) and TLq-HS reduce-scatter (Alg. 3) as sm_100a CUDA kernels + NCCL,
behind the C ABI of include/sdp4.h (libsdp4.so, built in-tree by `paper_2410_15526_b200.build`).
This package is a thin ctypes binding; it never computes the method on the CPU.
"""
from .sdp4 import (Comm, SDP4Error, emu_qwd_step, emu_qwd_workspace_bytes, emu_tlq_hs_reduce_scatter,  # noqa: F401
                   emu_tlq_workspace_bytes, get_unique_id, lib, qwd_workspace_bytes, ring_workspace_bytes,
                   tlq_stage_final, tlq_stage_quantize_reduce,
                   tlq_stage_quantize, tlq_stage_reduce, tlq_workspace_bytes, tlq_workspace_offset,
                   wire_unit_bytes)
from .topology import default_split, pad_numel  # noqa: F401

__version__ = "0.1.0"
