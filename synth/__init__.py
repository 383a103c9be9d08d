"""Seeded synthetic inputs shared by tests, bench.py and the oracle legs.

This module holds NONE of the method's arithmetic (no quantizer, no Hadamard,
no reduction): it only draws the buffers the paper's workloads consist of, with
their shapes and value distributions (DESIGN.md sec. 4 "input recipe"):

* GPT-shaped flat buffers (P:1018-1037 tab:model_size_params; Megatron layout:
  word embedding V x h, position embedding s x h, L x (12 h^2 + 13 h), final LN 2h;
  V = 50304 (Megatron's padded GPT-2 vocabulary, an assumption), s = 2048).
* model weights w_model ~ N(0, 0.02^2) (Megatron init; assumption), stored bf16.
* main weights w_main = widen(w_model) + lr * U(-1, 1): AdamW-like bounded steps
  ("weight differences are more uniformly distributed in a smaller range");
  lr from tab:e2e_params.
* gradients ~ N(0, 1e-3^2) with outliers: each element x50 with probability 0.01
  ("outliers can significantly amplify quantization errors").
* edge-case buffers (zero groups, exact ties, lattice points, single spikes,
  NaN/Inf groups, subnormal scales, bf16 extremes).

All generators are torch-based (CPU or CUDA) and fully determined by the seed.
"""
from __future__ import annotations

import torch

V_GPT2_PADDED = 50304
SEQ = 2048

# tab:model_size_params: name -> (hidden, layers)
GPT_SHAPES = {
    "125M": (768, 12),
    "350M": (1024, 24),
    "1.3B": (2048, 24),
    "2.7B": (2560, 32),
    "6.7B": (4096, 32),
    "13B": (5120, 40),
    "18B": (6144, 40),
}
# tab:e2e_params; 13B/18B: assumption (1e-4)
GPT_LR = {"125M": 6e-4, "350M": 3e-4, "1.3B": 2e-4, "2.7B": 1.6e-4, "6.7B": 1.2e-4,
          "13B": 1e-4, "18B": 1e-4}


def gpt_numel(name: str) -> int:
    """Flat parameter count of the GPT-shaped buffer (Megatron parameter order)."""
    h, L = GPT_SHAPES[name]
    return V_GPT2_PADDED * h + SEQ * h + L * (12 * h * h + 13 * h) + 2 * h


def padded_numel(numel: int, P: int, align: int) -> int:
    """Zero-pad to a multiple of P * align (zeros are reduction-neutral)."""
    m = P * align
    return (numel + m - 1) // m * m


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


_BIG = 1 << 31   # above this, buffers are generated in 2^30-element pieces (piece seeds seed+k)


def _pieces(n: int, seed: int, dtype, device, fn) -> torch.Tensor:
    """Generate n elements as fn(count, seed) in pieces so that no full-size fp32 temporary
    exists (GPT-13B buffers); small buffers (n <= 2^31) are a single piece, unchanged."""
    if n <= _BIG:
        return fn(n, seed).to(dtype)
    out = torch.empty(n, dtype=dtype, device=device)
    step = 1 << 30
    for k, o in enumerate(range(0, n, step)):
        out[o:o + step] = fn(min(step, n - o), seed * 1000003 + k)
    return out


def gradient(n: int, seed: int, device="cpu", dtype=torch.float32, std: float = 1e-3,
             spike_prob: float = 0.01, spike_scale: float = 50.0) -> torch.Tensor:
    """Spiky gradient: N(0, std^2), each element x spike_scale w.p. spike_prob."""
    def fn(m, sd):
        g = _gen(sd, device)
        x = torch.randn(m, generator=g, device=device, dtype=torch.float32) * std
        if spike_prob > 0:
            mask = torch.rand(m, generator=g, device=device) < spike_prob
            x = torch.where(mask, x * spike_scale, x)
        return x
    return _pieces(n, seed, dtype, device, fn)


def model_weights(n: int, seed: int, device="cpu", dtype=torch.bfloat16, std: float = 0.02) -> torch.Tensor:
    def fn(m, sd):
        return torch.randn(m, generator=_gen(sd, device), device=device, dtype=torch.float32) * std
    return _pieces(n, seed, dtype, device, fn)


def main_weights(w_model_shard: torch.Tensor, seed: int, lr: float = 2e-4) -> torch.Tensor:
    """fp32 main weights one optimizer step away from the stored model weights."""
    n, dev = w_model_shard.numel(), w_model_shard.device
    if n <= _BIG:
        u = torch.rand(n, generator=_gen(seed, dev), device=dev) * 2.0 - 1.0
        return w_model_shard.to(torch.float32) + lr * u
    out = w_model_shard.to(torch.float32)
    step = 1 << 30
    for k, o in enumerate(range(0, n, step)):
        m = min(step, n - o)
        out[o:o + m] += lr * (torch.rand(m, generator=_gen(seed * 1000003 + k, dev), device=dev) * 2.0 - 1.0)
    return out


def uniform_ints(n: int, seed: int, lo: int = -8, hi: int = 8, device="cpu") -> torch.Tensor:
    """Small integers as fp32 (every fp32 sum of a few of them is exact)."""
    g = _gen(seed, device)
    return torch.randint(lo, hi + 1, (n,), generator=g, device=device).to(torch.float32)


def edge_case_groups(G: int, seed: int = 0) -> torch.Tensor:
    """A buffer of 16 G-groups, each exercising one edge case of the quantizer."""
    g = _gen(seed, "cpu")
    rows = []
    base = torch.randn(G, generator=g) * 0.01
    rows.append(torch.zeros(G))                                   # zero group
    r = torch.zeros(G); r[G // 2] = 3.0; rows.append(r)            # single spike
    r = base.clone(); r[0] = 1.0; rows.append(r)                  # spike + small values
    r = torch.full((G,), -2.5); rows.append(r)                    # constant negative
    r = torch.arange(G, dtype=torch.float32) - G / 2; rows.append(r)  # lattice-ish ramp
    r = base.clone() * 1e-30; rows.append(r)                      # tiny but normal
    r = base.clone() * 1e-38; rows.append(r)                      # subnormal values
    r = torch.zeros(G); r[1] = 2.0 ** -125; rows.append(r)        # tiny scale (< 2^-120)
    r = base.clone(); r[3] = float("nan"); rows.append(r)         # NaN group
    r = base.clone(); r[5] = float("inf"); rows.append(r)         # +Inf group
    r = base.clone(); r[7] = float("-inf"); rows.append(r)        # -Inf group
    r = base.clone() * 1e30; rows.append(r)                       # huge values
    # exact ties for k=4 and k=8: s = q_k so y = x; x = j + 0.5
    r = torch.zeros(G); r[0] = 7.0; r[1:9] = torch.tensor([0.5, 1.5, 2.5, -0.5, -1.5, -2.5, 3.5, -3.5]); rows.append(r)
    r = torch.zeros(G); r[0] = 127.0; r[1:9] = torch.tensor([0.5, 1.5, 2.5, -0.5, -1.5, -2.5, 64.5, -64.5]); rows.append(r)
    r = torch.randn(G, generator=g); rows.append(r)               # plain gaussian
    r = torch.randn(G, generator=g) * 1e4; rows.append(r)         # large gaussian
    return torch.cat(rows)


def bf16_bits(t: torch.Tensor):
    """uint16 view (numpy) of a bf16 tensor (for the oracle, which stores bf16 as bits)."""
    return t.contiguous().view(torch.int16).cpu().numpy().view("uint16")


def spiky_numpy(n: int, seed: int, std: float = 1.0, spike_prob: float = 0.01, spike_scale: float = 50.0):
    """numpy fp32 spiky gradient (CPU convenience for the oracle pins)."""
    return gradient(n, seed, "cpu", torch.float32, std, spike_prob, spike_scale).numpy()


def lr_for(name: str) -> float:
    return GPT_LR[name]


def describe() -> str:
    return ("gradients N(0,1e-3^2) x50 w.p. 0.01; w_model N(0,0.02^2) bf16; "
            "w_main = w_model + lr*U(-1,1); torch.Generator seeds 2410+1000*rank+tensor_id")


def seed_for(rank: int, tensor_id: int, base: int = 2410) -> int:
    return base + 1000 * rank + tensor_id

