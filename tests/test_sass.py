"""Static checks on the built sm_100a SASS of libsdp4.so (no GPU needed).

ptxas 12.9 contracts a multiply feeding an add into FFMA2 even with .rn and --fmad=false,
which would change roundings of the numeric contract (R3/R5/R8).  The kernels
issue FFMA2 only for the quantizer's explicit fused RNE(x * inv) (addend 1.5 * 2^23 =
12582912, R3, or 1.5 * 2^23 + 8 = 12582920 for K4's biased 4-bit codes) and for
fusion-barrier products fma(a, b, z) with a scalar addend z = -0.0.  Also checks the Blackwell-native evidence: TMA (UTMALDG /
UTMASTG / UBLKCP) and mbarrier (SYNCS) instructions are present.
"""
import re
import shutil
import subprocess

import pytest

from paper_2410_15526_b200.sdp4 import LIB_PATH


@pytest.fixture(scope="module")
def sass():
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    r = subprocess.run([exe, "-sass", LIB_PATH], capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("cuobjdump unavailable: " + r.stderr[:200])
    return r.stdout


def functions(sass):
    out, name = {}, None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            name = m.group(1)
            out[name] = []
        elif name and re.match(r"\s+/\*[0-9a-f]{4,}\*/", line):
            out[name].append(line)
    return out


def test_no_contracted_products(sass):
    # Allowed FFMA2 forms: the quantizer's fused RNE (immediate addend 12582912 = 1.5*2^23) and
    # the fusion-barrier product fma(a, b, z) whose addend is a broadcast scalar register
    # (".F32").  An FFMA2 with a packed ".F32x2" addend is a product contracted into an
    # accumulation -- a changed rounding of the contract.
    fns = functions(sass)
    assert fns, "no kernels found"
    bad = []
    for name, lines in fns.items():
        for ln in lines:
            if "FFMA2" not in ln:
                continue
            ops = ln.split("FFMA2", 1)[1].split(";")[0].split(",")
            addend = ops[-1].strip()
            if "12582912" in addend or "12582920" in addend or (addend.endswith(".F32") and "F32x2" not in addend):
                continue
            bad.append((name[:80], ln.strip()[:110]))
    assert not bad, bad[:5]


def test_blackwell_async_copy_present(sass):
    fns = functions(sass)
    k3 = [n for n in fns if "k3_tlq_had_quant" in n]
    k5 = [n for n in fns if "k5_tlq_dq_reduce_had" in n]
    k4 = [n for n in fns if "k4_tlq_dq_reduce_q" in n]
    assert k3 and k4 and k5
    for n in k3 + k5:   # TMA tensor loads through an mbarrier ring
        body = "\n".join(fns[n])
        assert "UTMALDG" in body and "SYNCS" in body, n
    for n in k3:        # TMA tensor stores of the local code rows (per warp)
        assert "UTMASTG" in "\n".join(fns[n]), n
    for n in k5:        # the fp32 shard: coalesced 16-byte stores after the smem transpose
        assert "STG.E.128" in "\n".join(fns[n]), n
    for n in k3 + k4:   # 1-D bulk copies (K4 ring loads; K3/K4 staged tile stores, local or peer)
        assert "UBLKCP" in "\n".join(fns[n]), n


def test_fused_kernels_use_tma(sass):
    # the world-1 (K345) and N = 1 (K34) fused kernels keep K3's TMA + mbarrier input ring;
    # K34 bulk-copies its 4-bit tiles (to a peer or locally), K345 writes the fp32 shard with
    # coalesced 16-byte stores
    fns = functions(sass)
    loc = [n for n in fns if "k_tlq_local" in n]
    q84 = [n for n in fns if "k_tlq_q84" in n]
    assert loc and q84
    for n in loc + q84:
        body = "\n".join(fns[n])
        assert "UTMALDG" in body and "SYNCS" in body, n
    for n in q84:
        assert "UBLKCP" in "\n".join(fns[n]), n
    for n in loc:
        assert "STG.E.128" in "\n".join(fns[n]), n
