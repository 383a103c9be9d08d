"""SDP4Bit CPU oracle -- TEST INFRASTRUCTURE ONLY.

This package is the plain, slow, obviously-correct CPU statement of what the
SDP4Bit hot path computes (arXiv 2410.15526, /root/reference/PAPER.md).  It is
NOT part of the product: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it.  The
CUDA path (``paper_2410_15526_b200``) never imports it and shares no code with
it; the two meet only through seeded inputs from ``synth/``.

Every function cites the PAPER.md line (``P:n``) it follows; readings where the
paper is silent are the R1..R16 of DESIGN.md.
Parity pins: see tests/test_oracle_*.py.  Nothing here is "parity unpinned"
except where a function's docstring says so.
"""
from .sdp4_oracle import *  # noqa: F401,F403
