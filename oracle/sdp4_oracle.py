"""SDP4Bit oracle: qWD all-gather and TLq-HS reduce-scatter, step by step.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain numpy, scalar fp32
semantics: every numpy float32 operation below is one IEEE-754 binary32
operation rounded to nearest-even (numpy never contracts a*b+c into an FMA and
keeps subnormals), so each line is exactly the fp32 arithmetic written in it.
The paper fixes FP32 as the working precision of the reduction ("dequantizes the
received data back to the full precision (i.e., FP32) for local reduction",
P:344, sec. 3.2.1), so the oracle computes in fp32, not fp64; fp64 appears only
in the pins of tests/ (exact sums, dense Hadamard products).

Notation (sec. 2.1, sec. 2.3):  P workers = M groups ("nodes")
x N workers per group; rank r = m*N + l.  D = flattened buffer length, S = D/P
the shard length; shard r is the contiguous range [r*S, (r+1)*S).  G = group
size, k = bits, q_k = 2^(k-1) - 1, b = Hadamard block (0 = no Hadamard).

Readings are cited as R1..R16.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

F32 = np.float32
TINY = F32(2.0 ** -120)     # R2: 0 < s < 2^-120 is a zero group (q/s would overflow)
IDENTITY_BITS = 32          # R12: bits = 32 is the lossless identity codec

__all__ = [
    "F32", "TINY", "q_levels", "bf16_widen", "bf16_round", "hadamard_c",
    "group_scales", "quantize", "dequantize", "fwht_unnormalized", "hadamard_normalized",
    "pack_codes", "unpack_codes", "wire_unit_bytes", "wire_unit", "wire_unit_decode",
    "Topology", "qwd_quantize", "qwd_allgather_apply", "qwd_step", "qw_quantize", "qw_allgather_apply", "qw_step",
    "ring_reduce_scatter", "RingTrace", "unfused_tlq_hs_reduce_scatter",
    "TlqTrace", "tlq_hs_reduce_scatter", "naive_tlq_hs_reduce_scatter", "mix32", "sr_key", "sr_uniform",
    "STAGE_QWD", "STAGE_INTRA", "STAGE_INTER",
    "exact_reduce_scatter_f64", "comm_bits_per_param",
]


# --------------------------------------------------------------------------
# bf16 storage (model weights "in relatively low precision"; BF16
# model weights).  Widening is exact; narrowing is round-to-nearest-even.
# --------------------------------------------------------------------------
def bf16_widen(u16: np.ndarray) -> np.ndarray:
    """bf16 bit patterns (uint16) -> fp32, exact: the bf16 bits are the top half."""
    return (np.asarray(u16, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(F32)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bits, round to nearest, ties to even (R11).  NaN -> 0x7FC0.

    Definition: keep the top 16 bits of the fp32 pattern after adding half an
    ulp of bf16 (0x7FFF) plus the lsb of the kept part (ties to even).
    """
    u = np.asarray(x, dtype=F32).view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    r = ((u + np.uint64(0x7FFF) + lsb) >> np.uint64(16)).astype(np.uint16)
    return np.where(np.isnan(np.asarray(x, dtype=F32)), np.uint16(0x7FC0), r).astype(np.uint16)


# --------------------------------------------------------------------------
# Symmetric linear group-wise quantization (sec. 2.2):
#     x_int = round( x / s * (2^(k-1) - 1) ),   s = max(x)   per group.
# --------------------------------------------------------------------------
def q_levels(k: int) -> int:
    """q_k = 2^(k-1) - 1."""
    return (1 << (k - 1)) - 1


def hadamard_c(b: int) -> np.float32:
    """c_b = rn(1/sqrt(b)): normalization making H = c_b * H_unnorm orthonormal
    (H H^T = I).  b = 0 (no Hadamard) -> 1."""
    if b == 0:
        return F32(1.0)
    return F32(1.0 / math.sqrt(float(b)))


def group_scales(x: np.ndarray, G: int) -> np.ndarray:
    """s = max |x| over each contiguous G-group (P:281 with R2: the absolute max).
    NaN in a group -> NaN; otherwise any +-Inf -> +Inf (numpy max propagates)."""
    X = np.asarray(x, dtype=F32).reshape(-1, G)
    return np.max(np.abs(X), axis=1).astype(F32)


# --------------------------------------------------------------------------
# Stochastic rounding (NEXT-2; reading R14): the convergence theory assumes an
# unbiased gradient compressor E[U(v)] = v (Def. 1; Remark 2).
# Counter-based: the uniform draw of element i is a pure function of (seed, stage,
# rank, i), so any schedule reproduces it.  Stages: qWD = 1, intra = 2, inter = 3.
# --------------------------------------------------------------------------
STAGE_QWD, STAGE_INTRA, STAGE_INTER = 1, 2, 3
_U32 = np.uint32


def mix32(x):
    """32-bit finalizer: x ^= x>>16; x *= 0x7feb352d; x ^= x>>15; x *= 0x846ca68b; x ^= x>>16
    (all arithmetic mod 2^32)."""
    x = np.asarray(x, dtype=np.uint64) & 0xFFFFFFFF
    x ^= x >> 16
    x = (x * 0x7FEB352D) & 0xFFFFFFFF
    x ^= x >> 15
    x = (x * 0x846CA68B) & 0xFFFFFFFF
    x ^= x >> 16
    return x.astype(np.uint32)


def sr_key(seed: int, stage: int, rank: int) -> int:
    lo, hi = seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF
    return int(mix32(lo ^ int(mix32(hi ^ ((stage << 24) & 0xFFFFFFFF) ^ rank))))


def sr_uniform(index: np.ndarray, key: int) -> np.ndarray:
    """U_i = (h_i >> 8) * 2^-24 in [0, 1), h_i = mix32(lo32(i) ^ mix32(hi32(i) ^ key))."""
    i = np.asarray(index, dtype=np.uint64)
    lo = (i & np.uint64(0xFFFFFFFF)).astype(np.uint64)
    hi = (i >> np.uint64(32)).astype(np.uint64)
    h = mix32(lo ^ mix32(hi ^ np.uint64(key)).astype(np.uint64))
    return ((h >> 8).astype(np.float64) * 2.0 ** -24).astype(F32)


def quantize(x: np.ndarray, k: int, G: int, c: np.float32 = F32(1.0), sr=None):
    """Group-wise k-bit quantization of x.

    Returns (codes, scales).  codes: int32 in [-q_k, q_k] (R4: -2^(k-1) is never
    produced); scales: fp32 per group.
      s      = max |x_g|                                   (R2)
      inv    = rn(q_k / s)                                 (R3, one division per group)
      code   = clamp(RNE(x * inv), +-q_k)                  (R3: the exact product x*inv is
               rounded once, to the nearest-even integer -- the single round() of P:281;
               fp64 holds the 24x24-bit product exactly)
      scale  = rn(s * c)                                   (R6: c = c_b folds the
               Hadamard normalization into the scale; c = 1 without Hadamard)
    Zero / tiny groups (s < 2^-120) and non-finite groups get codes 0; the scale
    of a tiny group is stored as 0 and of a non-finite group as rn(s*c) (NaN or
    +Inf), so that dequantization poisons the group (R2, R5).
    k = 32 is the identity codec (R12): returns (rn(x*c) as fp32, None).
    sr = (base_index, key): stochastic rounding (R14) of element j with the uniform draw of
    global index base_index + j: y = rn(x*inv), fl = floor(y), fr = rn(y - fl),
    code = clamp(fl + [U < fr], +-q_k).
    """
    x = np.asarray(x, dtype=F32)
    if k == IDENTITY_BITS:
        return (x * F32(c) if F32(c) != F32(1.0) else x.copy()), None
    q = F32(q_levels(k))
    X = x.reshape(-1, G)
    s = group_scales(x, G)
    ok = np.isfinite(s) & (s >= TINY)
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        inv = np.where(ok, q / np.where(ok, s, F32(1.0)), F32(0.0)).astype(F32)
        if sr is None:
            y = X.astype(np.float64) * inv.astype(np.float64)[:, None]     # exact product
            y = np.where(ok[:, None], y, 0.0)
            codes = np.clip(np.rint(y), -q, q).astype(np.int32)
        else:
            base, key = sr
            y = (X * inv[:, None]).astype(F32)                            # rn(x * inv)
            y = np.where(ok[:, None], y, F32(0.0))
            fl = np.floor(y).astype(F32)
            fr = (y - fl).astype(F32)
            u = sr_uniform(base + np.arange(X.size, dtype=np.uint64), key).reshape(X.shape)
            codes = np.clip(fl + (u < fr).astype(F32), -q, q).astype(np.int32)
        scales = np.where(s < TINY, F32(0.0), s * F32(c)).astype(F32)
    return codes.reshape(-1), scales


def dequantize(codes: np.ndarray, scales, k: int, G: int) -> np.ndarray:
    """x_hat = rn(code * rn(s / q_k)) (R5; inverse of P:281, "Dequantize" P:371/P:377).
    A NaN/Inf scale yields NaN for the whole group (0*Inf = NaN), a 0 scale yields 0."""
    if k == IDENTITY_BITS:
        return np.asarray(codes, dtype=F32).copy()
    q = F32(q_levels(k))
    with np.errstate(invalid="ignore", over="ignore"):
        ds = (np.asarray(scales, dtype=F32) / q).astype(F32)
        C = np.asarray(codes).astype(F32).reshape(-1, G)
        return (C * ds[:, None]).astype(F32).reshape(-1)


# --------------------------------------------------------------------------
# Hadamard smoother (sec. 3.2.2: "H = H^T and H . H^T = I";
# sec. 3.3: blockwise, group size divisible by the Hadamard size).
# --------------------------------------------------------------------------
def fwht_unnormalized(x: np.ndarray, b: int) -> np.ndarray:
    """u = H_b^unnorm x on each aligned block of b elements (Sylvester order, R6).

    Butterfly stages h = 1, 2, 4, ..., b/2 in ascending order; in stage h every
    pair (i, i+h) inside a 2h-chunk becomes (rn(a + c), rn(a - c)).
    """
    X = np.asarray(x, dtype=F32).reshape(-1, b).copy()
    h = 1
    while h < b:
        Y = X.reshape(-1, b // (2 * h), 2, h)
        a = Y[:, :, 0, :].copy()
        c = Y[:, :, 1, :].copy()
        Y[:, :, 0, :] = a + c
        Y[:, :, 1, :] = a - c
        h *= 2
    return X.reshape(-1)


def hadamard_normalized(x: np.ndarray, b: int) -> np.ndarray:
    """H_b x with H_b = c_b H_unnorm (orthonormal): rn(u * c_b)."""
    return (fwht_unnormalized(x, b) * hadamard_c(b)).astype(F32)


# --------------------------------------------------------------------------
# Wire format (R4, R15): one "wire unit" per (shard, bit-width):
#   [codes: n*k/8 bytes][scales: n/G fp32 little-endian] padded to 256 bytes.
#   int8 codes are two's complement; int4 codes are two's-complement nibbles,
#   element 2j in the low nibble; int2 codes (the ternary codec of
#   Counterexample 1, weights only) are two's-complement bit pairs, element
#   4j+i in bits 2i..2i+1 (R4).  k = 32: n fp32 values, no scales.
# --------------------------------------------------------------------------
def pack_codes(codes: np.ndarray, k: int) -> np.ndarray:
    c = np.asarray(codes, dtype=np.int64)
    if k == 8:
        return (c & 0xFF).astype(np.uint8)
    if k == 4:
        nib = (c & 0xF).astype(np.uint8).reshape(-1, 2)
        return (nib[:, 0] | (nib[:, 1] << np.uint8(4))).astype(np.uint8)
    if k == 2:
        two = (c & 0x3).astype(np.uint8).reshape(-1, 4)
        return (two[:, 0] | (two[:, 1] << np.uint8(2)) | (two[:, 2] << np.uint8(4))
                | (two[:, 3] << np.uint8(6))).astype(np.uint8)
    raise ValueError(f"pack_codes: unsupported k={k}")


def unpack_codes(packed: np.ndarray, k: int, n: int) -> np.ndarray:
    p = np.asarray(packed, dtype=np.uint8)
    if k == 8:
        return p[:n].view(np.int8).astype(np.int32)
    if k == 4:
        lo = (p & 0xF).astype(np.int32)
        hi = (p >> 4).astype(np.int32)
        out = np.stack([lo, hi], axis=1).reshape(-1)[:n]
        return np.where(out >= 8, out - 16, out).astype(np.int32)
    if k == 2:
        out = np.stack([(p >> np.uint8(2 * i)) & np.uint8(3) for i in range(4)], axis=1).astype(np.int32)
        out = out.reshape(-1)[:n]
        return np.where(out >= 2, out - 4, out).astype(np.int32)
    raise ValueError(f"unpack_codes: unsupported k={k}")


def _round_up(a: int, m: int) -> int:
    return (a + m - 1) // m * m


def wire_unit_bytes(n: int, k: int, G: int) -> int:
    """Bytes of one wire unit of n elements (R15)."""
    if k == IDENTITY_BITS:
        return _round_up(4 * n, 256)
    return _round_up(n * k // 8 + 4 * (n // G), 256)


def wire_unit(codes, scales, k: int, G: int) -> np.ndarray:
    """Encode (codes, scales) of n elements into the wire-unit bytes (zero padding)."""
    n = len(codes)
    out = np.zeros(wire_unit_bytes(n, k, G), dtype=np.uint8)
    if k == IDENTITY_BITS:
        out[: 4 * n] = np.asarray(codes, dtype="<f4").view(np.uint8)
        return out
    cb = pack_codes(codes, k)
    out[: len(cb)] = cb
    sb = np.asarray(scales, dtype="<f4").view(np.uint8)
    out[len(cb): len(cb) + len(sb)] = sb
    return out


def wire_unit_decode(buf: np.ndarray, n: int, k: int, G: int):
    """Inverse of wire_unit: returns (codes, scales) (scales None for k = 32)."""
    buf = np.asarray(buf, dtype=np.uint8)
    if k == IDENTITY_BITS:
        return buf[: 4 * n].copy().view("<f4").astype(F32), None
    ncb = n * k // 8
    codes = unpack_codes(buf[:ncb], k, n)
    scales = buf[ncb: ncb + 4 * (n // G)].copy().view("<f4").astype(F32)
    return codes, scales


def comm_bits_per_param(k: int, G: int, scale_bits: int = 32) -> float:
    """k + scale_bits / G (group-wise overhead of P:286)."""
    return k + scale_bits / G


# --------------------------------------------------------------------------
# Topology (sec. 2.3): M groups of N workers, rank r = m*N + l.
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class Topology:
    M: int
    N: int

    @property
    def P(self) -> int:
        return self.M * self.N

    def rank(self, m: int, l: int) -> int:
        return m * self.N + l

    def coords(self, r: int):
        return divmod(r, self.N)


# --------------------------------------------------------------------------
# qWD: quantized weight differences (sec. 3.1; Alg. 2 l.2-5)
# --------------------------------------------------------------------------
def qwd_quantize(w_main_shard: np.ndarray, w_model_shard: np.ndarray, k: int, G: int, sr=None):
    """Alg. 2 l.2-3 on worker p:
         d[p] = w_main[p] - w_model[p]                  (fp32, R11)
         d~[p] = QuantizeWeightsDiff(d[p])              (k-bit group quantizer)
    w_model_shard is the fp32 value of the stored model weights (bf16 widened
    exactly, or fp32).  Returns (codes, scales, d)."""
    d = (np.asarray(w_main_shard, dtype=F32) - np.asarray(w_model_shard, dtype=F32)).astype(F32)
    codes, scales = quantize(d, k, G, sr=sr)
    return codes, scales, d


def qwd_allgather_apply(units, w_model: np.ndarray, k: int, G: int, model_bf16: bool):
    """Alg. 2 l.4-5:  d <- AllGather(d~[p]);  w_model <- w_model + d.

    units: the P quantized shards (codes, scales) in rank order (the all-gather
    concatenates them).  w_model: full replica as fp32 values.  Every
    worker adds the dequantized d (its own shard included, R11), so replicas stay
    identical.  Returns the new replica: bf16 bits (uint16) if model_bf16 (the add
    is done in fp32 then rounded RNE to bf16, R11), else fp32."""
    d_hat = np.concatenate([dequantize(c, s, k, G) for (c, s) in units]).astype(F32)
    acc = (np.asarray(w_model, dtype=F32) + d_hat).astype(F32)
    return bf16_round(acc) if model_bf16 else acc


def qwd_step(w_main_shards, w_model, k: int, G: int, model_bf16: bool, seed=None):
    """One qWD iteration over all P simulated workers (Alg. 2 l.2-5).
    w_main_shards: list of P fp32 shards; w_model: replica (uint16 bf16 bits if
    model_bf16 else fp32).  seed: stochastic rounding (R14, stage qWD, element index = the
    global index p*S + j of d).  Returns (units, new_w_model)."""
    wm = bf16_widen(w_model) if model_bf16 else np.asarray(w_model, dtype=F32)
    S = len(w_main_shards[0])
    units = []
    for p, shard in enumerate(w_main_shards):
        sr = None if seed is None else (p * S, sr_key(seed, STAGE_QWD, p))
        c, s, _ = qwd_quantize(shard, wm[p * S:(p + 1) * S], k, G, sr)
        units.append((c, s))
    return units, qwd_allgather_apply(units, wm, k, G, model_bf16)


# --------------------------------------------------------------------------
# qW: direct weight quantization, the comparison codec of QSDP / ZeRO++ (Alg. 1,
# "Quantize weights", "AllGather"; sec. 3.1 P:330-336 and Counterexample 1
# P:412-416 contrast it with qWD).  Ablation baseline, same wire unit.
# --------------------------------------------------------------------------
def qw_quantize(w_main_shard: np.ndarray, k: int, G: int, sr=None):
    """Alg. 1 "Quantize weights" on worker p: codes/scales of w_main[p] itself (no difference)."""
    return quantize(np.asarray(w_main_shard, dtype=F32), k, G, sr=sr)


def qw_allgather_apply(units, k: int, G: int, model_bf16: bool):
    """Alg. 1 "AllGather" + dequantize: the replica BECOMES the gathered dequantized weights
    (w_model <- concat_j Dequantize(unit_j)), stored bf16 (RNE) or fp32 -- no accumulation,
    which is why a biased codec can stall (Counterexample 1)."""
    w = np.concatenate([dequantize(c, s, k, G) for (c, s) in units]).astype(F32)
    return bf16_round(w) if model_bf16 else w


def qw_step(w_main_shards, k: int, G: int, model_bf16: bool, seed=None):
    """One qW iteration over all P simulated workers.  seed: stochastic rounding with the
    qWD stage key (R14), element index = the global index p*S + j."""
    S = len(w_main_shards[0])
    units = []
    for p, shard in enumerate(w_main_shards):
        sr = None if seed is None else (p * S, sr_key(seed, STAGE_QWD, p))
        units.append(qw_quantize(shard, k, G, sr))
    return units, qw_allgather_apply(units, k, G, model_bf16)


# --------------------------------------------------------------------------
# TLq-HS: two-level gradient quantization with Hadamard smoother
# (sec. 3.2.1, sec. 3.2.2, Alg. 3, pruning sec. 3.3
# P:389-390).  b = 0 gives TLq; (k_intra, k_inter, b) = (4, 4, 0) gives ULq
# (ZeRO++'s two all-to-alls).
# --------------------------------------------------------------------------
@dataclass
class TlqTrace:
    """Every message of one TLq-HS reduce-scatter, for stage-by-stage comparison.
    intra_send[r][lp][mp]: (codes, scales) rank r sends to local rank lp for shard mp*N+lp.
    inter_send[r][mp]:     (codes, scales) rank r sends to node mp for shard mp*N+l.
    out[r]:                fp32 output shard r."""
    intra_send: list = field(default_factory=list)
    inter_send: list = field(default_factory=list)
    out: list = field(default_factory=list)


def tlq_hs_reduce_scatter(grads, topo: Topology, G: int, b: int,
                          k_intra: int = 8, k_inter: int = 4, average: bool = True, seed=None) -> TlqTrace:
    """Alg. 3 with the sec. 3.3 pruning, simulated for all P = M*N workers.

    grads: list of P fp32 arrays (the local gradients g^p_model, each of length D).
    seed: stochastic rounding (R14) for both quantizers: the intra message of rank r for
    shard j draws with key (seed, intra, r) at the gradient's global index j*S + e; the inter
    message of rank r for shard j with key (seed, inter, r) at index j*S + e.
    Returns a TlqTrace whose out[r] is g_main[r] (Alg. 2 l.9).
    """
    M, N, P = topo.M, topo.N, topo.P
    D = len(grads[0])
    assert D % P == 0
    S = D // P
    cb = hadamard_c(b)
    tr = TlqTrace()

    # Alg. 3 l.2-3 on every worker: g_hat = Hadamard(grad) blockwise,
    # then Quantize8Bit per G-group.  R6: codes come from the unnormalized u and
    # the stored scale carries c_b, i.e. the quantizer is applied to H x = c_b u.
    # Sent to local rank lp: shards {mp*N + lp : mp = 0..M-1} (R9).
    for r in range(P):
        g = np.asarray(grads[r], dtype=F32)
        u = fwht_unnormalized(g, b) if b else g
        blocks = []
        for lp in range(N):
            sub = []
            for mp in range(M):
                j = mp * N + lp
                sr = None if seed is None else (j * S, sr_key(seed, STAGE_INTRA, r))
                sub.append(quantize(u[j * S:(j + 1) * S], k_intra, G, cb, sr))
            blocks.append(sub)
        tr.intra_send.append(blocks)

    # Alg. 3 l.4 IntraAlltoAll: worker (m, l) receives block l from every
    # (m, l'') of its node.  l.5 Dequantize; l.6 Hadamard pruned;
    # l.7 Reduction in FP32, fixed order l'' = 0..N-1 (R8).
    # l.8 Hadamard pruned; l.9 Quantize4Bit.  Sent to node mp: shard mp*N+l.
    for r in range(P):
        m, l = topo.coords(r)
        sends = []
        for mp in range(M):
            acc = np.zeros(S, dtype=F32)
            for lpp in range(N):
                codes, scales = tr.intra_send[topo.rank(m, lpp)][l][mp]
                acc = (acc + dequantize(codes, scales, k_intra, G)).astype(F32)
            j = mp * N + l
            sr = None if seed is None else (j * S, sr_key(seed, STAGE_INTER, r))
            sends.append(quantize(acc, k_inter, G, sr=sr))
        tr.inter_send.append(sends)

    # Alg. 3 l.10 InterAlltoAll: worker (m, l) receives from (m'', l) the
    # unit for node m.  l.11 Dequantize, l.12 Reduction over m'' = 0..M-1 (R8),
    # l.13 Hadamard moved after the final reduction (sum_i H g_i = H sum_i g_i).
    # Average (R8): kappa = rn(c_b / P) multiplies the unnormalized butterfly output.
    for r in range(P):
        m, l = topo.coords(r)
        acc = np.zeros(S, dtype=F32)
        for mpp in range(M):
            codes, scales = tr.inter_send[topo.rank(mpp, l)][m]
            acc = (acc + dequantize(codes, scales, k_inter, G)).astype(F32)
        if b:
            kappa = F32(cb / F32(P)) if average else cb
            out = (fwht_unnormalized(acc, b) * kappa).astype(F32)
        else:
            out = (acc * F32(F32(1.0) / F32(P))).astype(F32) if average else acc
        tr.out.append(out)
    return tr


def naive_tlq_hs_reduce_scatter(grads, topo: Topology, G: int, b: int,
                                k_intra: int = 8, k_inter: int = 4, average: bool = True):
    """Alg. 3 WITHOUT the sec. 3.3 pruning (test oracle only):
    normalized H before Quantize8Bit (l.2), H after intra Dequantize (l.6, struck
    in the paper), H before Quantize4Bit (l.8, struck), and H after inter
    Dequantize (the pre-move position of l.13) -- four transforms, each
    H = c_b H_unnorm applied explicitly; the reductions then run in the original
    domain.  Mean = division by P after the final reduction.  Returns the P
    output shards."""
    M, N, P = topo.M, topo.N, topo.P
    D = len(grads[0])
    S = D // P

    def H(v):
        return hadamard_normalized(v, b) if b else np.asarray(v, dtype=F32)

    sent = []
    for r in range(P):
        gh = H(grads[r])
        sent.append([quantize(gh[j * S:(j + 1) * S], k_intra, G) for j in range(P)])
    inter = []
    for r in range(P):
        m, l = topo.coords(r)
        row = []
        for mp in range(M):
            j = mp * N + l
            acc = np.zeros(S, dtype=F32)
            for lpp in range(N):
                c, s = sent[topo.rank(m, lpp)][j]
                acc = (acc + H(dequantize(c, s, k_intra, G))).astype(F32)
            row.append(quantize(H(acc), k_inter, G))
        inter.append(row)
    outs = []
    for r in range(P):
        m, l = topo.coords(r)
        acc = np.zeros(S, dtype=F32)
        for mpp in range(M):
            c, s = inter[topo.rank(mpp, l)][m]
            acc = (acc + H(dequantize(c, s, k_inter, G))).astype(F32)
        if average:
            acc = (acc / F32(P)).astype(F32)
        outs.append(acc)
    return outs


@dataclass
class RingTrace:
    """Messages of one ring reduce-scatter: send[t][r] = (codes, scales) rank r sends to rank
    (r+1) mod P at hop t (t = 0..P-2), carrying chunk (r - t - 1) mod P; out[r]: shard r."""
    send: list = field(default_factory=list)
    out: list = field(default_factory=list)


def ring_reduce_scatter(grads, k: int, G: int, average: bool = True) -> RingTrace:
    """Ring reduce-scatter with per-hop quantization, the baseline of sec. 2.3 ("P-1
    rounds, during which each GPU sends local data and aggregates the received data. When
    quantization is applied, this necessitates P-1 rounds of quantization and
    dequantization").  Ablation baseline, nearest rounding.

    Chunk c (= shard c, ending on rank c) starts on rank c+1: acc = g_{c+1}[c].  Hop h =
    1..P-1: rank (c+h) mod P sends Quantize(acc) (k bits, group G); rank (c+h+1) mod P sets
    acc = rn(Dequantize(msg) + g_own[c]) (fp32).  Finally out_c = rn(acc * rn(1/P)) when
    averaging (as R8).  k = 32 is the identity codec (R12)."""
    P = len(grads)
    D = len(grads[0])
    S = D // P
    g = [np.asarray(x, dtype=F32) for x in grads]
    tr = RingTrace(send=[[None] * P for _ in range(max(P - 1, 0))], out=[None] * P)
    for c in range(P):
        acc = g[(c + 1) % P][c * S:(c + 1) * S].copy()
        for h in range(1, P):
            sender, recv = (c + h) % P, (c + h + 1) % P
            codes, scales = quantize(acc, k, G)
            tr.send[h - 1][sender] = (codes, scales)
            acc = (dequantize(codes, scales, k, G) + g[recv][c * S:(c + 1) * S]).astype(F32)
        if average:
            acc = (acc * F32(F32(1.0) / F32(P))).astype(F32)
        tr.out[c] = acc
    return tr


def unfused_tlq_hs_reduce_scatter(grads, topo: Topology, G: int, b: int, k_intra: int = 8, k_inter: int = 4,
                                  average: bool = True):
    """TLq-HS with the Hadamard transforms as separate passes ("SDP4Bit (HS w/o fused)",
    P:645, ablation comparator): h_r = H_b g_r on every rank (normalized),
    the b = 0 two-level reduce-scatter of the h_r, then H_b on each reduced shard (l.13 moved
    after the final reduction; H = H^T = H^-1).  Returns the P output shards."""
    h = [hadamard_normalized(np.asarray(g, dtype=F32), b) for g in grads]
    tr = tlq_hs_reduce_scatter(h, topo, G, 0, k_intra, k_inter, average)
    return [hadamard_normalized(o, b) for o in tr.out]


def exact_reduce_scatter_f64(grads, P: int, average: bool = True):
    """The plain definition the collective approximates (sec. 2.1):
    shard r of (1/P) sum_p g_p, computed in fp64.  Pin for bits = 32 cases."""
    tot = np.zeros(len(grads[0]), dtype=np.float64)
    for g in grads:
        tot += np.asarray(g, dtype=np.float64)
    if average:
        tot /= P
    S = len(tot) // P
    return [tot[r * S:(r + 1) * S] for r in range(P)]
