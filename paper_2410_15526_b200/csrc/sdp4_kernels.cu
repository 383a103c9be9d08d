// sdp4_kernels.cu -- sm_100a kernels of the SDP4Bit hot path (arXiv 2410.15526).
//
// All five kernels are HBM-streaming: the method has no dense contraction (the
// Hadamard block is "memory-bound", sec. 3.3), so tensor cores are not used.
// Arithmetic is fp32 with every operation an explicit round-to-nearest intrinsic
// (__fadd_rn / __fmul_rn / __fdiv_rn; the library is also built with --fmad=false)
// so codes and scales are bit-identical to the numeric contract R1-R16.
//
//  K1 qwd_quantize      Alg. 2 l.2-3          vector layout, 8 el/thread
//  K2 qwd_apply         Alg. 2 l.5              vector layout, 16 el/thread
//  K3 tlq_had_quant     Alg. 3 l.2-3, fused   row layout (64 el/thread),
//                       Hadamard + quantize    smem-staged (cp.async)
//  K4 tlq_dq_reduce_q   Alg. 3 l.5,7,9        vector layout, 16 el/thread
//  K5 tlq_dq_reduce_had Alg. 3 l.11-13 row layout, smem-staged output
//
// Integer rounding uses the magic-number identity: for |y| <= 2^22,
// rn(y + 1.5*2^23) is the nearest-even integer of y and its low mantissa bits
// hold that integer in two's complement, so a code is one FADD (not a quarter-rate
// F2I) and packing is byte/nibble selection.  Decoding inverts it with PRMT + FADD.
#include "sdp4_kernels.cuh"

#include <cfloat>
#include <cuda_bf16.h>

namespace sdp4 {
namespace {

constexpr float kTiny = 0x1p-120f;        // R2: 0 < s < 2^-120 is a zero group
constexpr float kMagic = 12582912.0f;     // 1.5 * 2^23
constexpr float kDec8 = 8388736.0f;       // 2^23 + 128: float(0x4B0000xx) - kDec8 = (int8)(xx ^ 0x80)
constexpr float kDec4 = 8388616.0f;       // 2^23 + 8

__device__ __forceinline__ float max_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);  // cvt.rn.bf16x2.f32: RNE (R11)
  return *reinterpret_cast<uint32_t*>(&v);
}

// Per-group quantizer parameters (R2, R3): ok <=> s finite and >= 2^-120.
struct QP {
  float inv;
  bool ok;
};
__device__ __forceinline__ QP qparam(float s, float q) {
  QP p;
  p.ok = (s >= kTiny) && (s <= FLT_MAX);
  p.inv = p.ok ? __fdiv_rn(q, s) : 0.f;
  return p;
}
// Stored scale (R2, R6): 0 for tiny/zero groups, rn(s * c) otherwise (NaN/Inf kept).
__device__ __forceinline__ float stored_scale(float s, float c) {
  return (s < kTiny) ? 0.f : __fmul_rn(s, c);
}
// rn(x * inv) rounded to the nearest-even integer, as magic-number bits.
__device__ __forceinline__ uint32_t rq(float x, float inv) {
  return __float_as_uint(__fadd_rn(__fmul_rn(x, inv), kMagic));
}
__device__ __forceinline__ uint32_t pack8x4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}
__device__ __forceinline__ uint32_t pack4x8(const uint32_t* r) {
  uint32_t p01 = (r[0] & 0xFu) | (r[1] << 4);
  uint32_t p23 = (r[2] & 0xFu) | (r[3] << 4);
  uint32_t p45 = (r[4] & 0xFu) | (r[5] << 4);
  uint32_t p67 = (r[6] & 0xFu) | (r[7] << 4);
  return __byte_perm(__byte_perm(p01, p23, 0x0040), __byte_perm(p45, p67, 0x0040), 0x5410);
}
// Decode 4 int8 codes of w into exact floats (code values, not yet scaled).
__device__ __forceinline__ void dec8x4(uint32_t w, float* f) {
  const uint32_t x = w ^ 0x80808080u;
  f[0] = __fsub_rn(__uint_as_float(__byte_perm(x, 0x4B000000u, 0x7540)), kDec8);
  f[1] = __fsub_rn(__uint_as_float(__byte_perm(x, 0x4B000000u, 0x7541)), kDec8);
  f[2] = __fsub_rn(__uint_as_float(__byte_perm(x, 0x4B000000u, 0x7542)), kDec8);
  f[3] = __fsub_rn(__uint_as_float(__byte_perm(x, 0x4B000000u, 0x7543)), kDec8);
}
// Decode 8 int4 codes of w (element 2j = low nibble of byte j).
__device__ __forceinline__ void dec4x8(uint32_t w, float* f) {
  const uint32_t x = w ^ 0x88888888u;
  const uint32_t lo = x & 0x0F0F0F0Fu, hi = (x >> 4) & 0x0F0F0F0Fu;
  f[0] = __fsub_rn(__uint_as_float(__byte_perm(lo, 0x4B000000u, 0x7540)), kDec4);
  f[1] = __fsub_rn(__uint_as_float(__byte_perm(hi, 0x4B000000u, 0x7540)), kDec4);
  f[2] = __fsub_rn(__uint_as_float(__byte_perm(lo, 0x4B000000u, 0x7541)), kDec4);
  f[3] = __fsub_rn(__uint_as_float(__byte_perm(hi, 0x4B000000u, 0x7541)), kDec4);
  f[4] = __fsub_rn(__uint_as_float(__byte_perm(lo, 0x4B000000u, 0x7542)), kDec4);
  f[5] = __fsub_rn(__uint_as_float(__byte_perm(hi, 0x4B000000u, 0x7542)), kDec4);
  f[6] = __fsub_rn(__uint_as_float(__byte_perm(lo, 0x4B000000u, 0x7543)), kDec4);
  f[7] = __fsub_rn(__uint_as_float(__byte_perm(hi, 0x4B000000u, 0x7543)), kDec4);
}

// NaN-propagating max over the `tpg` consecutive threads of a group (tpg a power of
// two).  tpg > 32 reduces across warps through `red` (CTA-uniform branch).
__device__ __forceinline__ float group_max(float v, int tpg, float* red) {
  const int lim = tpg < 32 ? tpg : 32;
  for (int off = 1; off < lim; off <<= 1) v = max_nan(v, __shfl_xor_sync(0xffffffffu, v, off));
  if (tpg > 32) {
    const int warp = threadIdx.x >> 5, wpg = tpg >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[warp] = v;
    __syncthreads();
    const int base = warp & ~(wpg - 1);
    v = red[base];
    for (int w = 1; w < wpg; ++w) v = max_nan(v, red[base + w]);
  }
  return v;
}

// Physical 16-byte chunk index of logical chunk c of row `row` in a smem tile whose
// rows are `cpr` chunks long.  XOR swizzle: conflict-free both for one-row-per-thread
// access (8 consecutive rows per quarter-warp) and for linear (coalescing) access.
// For cpr = 2/4/8 it equals the TMA SWIZZLE_32B/64B/128B patterns.
__device__ __forceinline__ int swz(int row, int c, int cpr) {
  const int f = (cpr >= 8) ? (row & 7) : ((row / (8 / cpr)) & (cpr - 1));
  return row * cpr + (c ^ f);
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem_src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// In-register butterfly stages h = 1..min(b,64)/2 of the unnormalized Sylvester
// Hadamard (R6): pairs (i, i+h) -> (a + c, a - c), ascending h.
__device__ __forceinline__ void fwht_row(float* v, int b) {
#pragma unroll
  for (int h = 1; h < 64; h <<= 1) {
    if (b > h) {
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        if ((i & h) == 0) {
          const float a = v[i], c = v[i + h];
          v[i] = __fadd_rn(a, c);
          v[i + h] = __fsub_rn(a, c);
        }
      }
    }
  }
  // b = 128, 256: stages h = 64, 128 pair row t with row t ^ (h / 64) (lanes of one warp).
  for (int hx = 1; 64 * hx < b; hx <<= 1) {
    const bool upper = (threadIdx.x & hx) != 0;
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      const float o = __shfl_xor_sync(0xffffffffu, v[i], hx);
      v[i] = upper ? __fsub_rn(o, v[i]) : __fadd_rn(v[i], o);
    }
  }
}

// =====================================================================================
// K1  qWD quantize (Alg. 2 l.2-3): d = rn(w_main - widen(w_model)),
// per G-group s = max|d|, codes = RNE(d * rn(q/s)).  8 elements per thread, a group is
// G/8 consecutive threads.  Output: one wire unit [codes][scales].
// =====================================================================================
template <typename TM, int BITS>
__global__ void __launch_bounds__(256) k1_qwd_quantize(const float* __restrict__ w_main,
                                                       const TM* __restrict__ w_model, size_t S,
                                                       int G, uint8_t* __restrict__ unit) {
  __shared__ float red[8];
  constexpr float q = float((1 << (BITS == 32 ? 1 : BITS - 1)) - 1);
  const int tpg = G >> 3;
  const size_t ntiles = (S + 2047) / 2048;
  float* scales = reinterpret_cast<float*>(unit + S * (BITS == 32 ? 4 : BITS) / 8);
  for (size_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const size_t e0 = tile * 2048 + threadIdx.x * 8;
    const bool act = e0 < S;
    float d[8];
    if (act) {
      const float4 a0 = *reinterpret_cast<const float4*>(w_main + e0);
      const float4 a1 = *reinterpret_cast<const float4*>(w_main + e0 + 4);
      float m[8];
      if constexpr (sizeof(TM) == 2) {
        const uint4 u = *reinterpret_cast<const uint4*>(w_model + e0);
        m[0] = bf16_lo(u.x); m[1] = bf16_hi(u.x); m[2] = bf16_lo(u.y); m[3] = bf16_hi(u.y);
        m[4] = bf16_lo(u.z); m[5] = bf16_hi(u.z); m[6] = bf16_lo(u.w); m[7] = bf16_hi(u.w);
      } else {
        const float4 b0 = *reinterpret_cast<const float4*>(w_model + e0);
        const float4 b1 = *reinterpret_cast<const float4*>(w_model + e0 + 4);
        m[0] = b0.x; m[1] = b0.y; m[2] = b0.z; m[3] = b0.w;
        m[4] = b1.x; m[5] = b1.y; m[6] = b1.z; m[7] = b1.w;
      }
      d[0] = __fsub_rn(a0.x, m[0]); d[1] = __fsub_rn(a0.y, m[1]);
      d[2] = __fsub_rn(a0.z, m[2]); d[3] = __fsub_rn(a0.w, m[3]);
      d[4] = __fsub_rn(a1.x, m[4]); d[5] = __fsub_rn(a1.y, m[5]);
      d[6] = __fsub_rn(a1.z, m[6]); d[7] = __fsub_rn(a1.w, m[7]);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) d[i] = 0.f;
    }
    if constexpr (BITS == 32) {  // identity codec (R12): the wire carries d itself
      if (act) {
        float4* o = reinterpret_cast<float4*>(unit + e0 * 4);
        o[0] = make_float4(d[0], d[1], d[2], d[3]);
        o[1] = make_float4(d[4], d[5], d[6], d[7]);
      }
      continue;
    } else {
      float a = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) a = max_nan(a, fabsf(d[i]));
      a = group_max(a, tpg, red);
      const QP p = qparam(a, q);
      if (act) {
        uint32_t r[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) r[i] = rq(d[i], p.inv);
        if constexpr (BITS == 4) {
          uint32_t w = pack4x8(r);
          if (!p.ok) w = 0u;
          *reinterpret_cast<uint32_t*>(unit + e0 / 2) = w;
        } else {
          uint2 w = make_uint2(pack8x4(r[0], r[1], r[2], r[3]), pack8x4(r[4], r[5], r[6], r[7]));
          if (!p.ok) w = make_uint2(0u, 0u);
          *reinterpret_cast<uint2*>(unit + e0) = w;
        }
        if ((threadIdx.x & (tpg - 1)) == 0) scales[e0 / G] = stored_scale(a, 1.f);
      }
    }
  }
}

// =====================================================================================
// K2  qWD apply (Alg. 2 l.5): w_model[jS + e] = bf16_rn(widen(w) + code*rn(s/q))
// for every shard j (blockIdx.y) of the gathered units.  16 elements per thread.
// =====================================================================================
template <typename TM, int BITS>
__global__ void __launch_bounds__(256) k2_qwd_apply(const uint8_t* __restrict__ units,
                                                    size_t unit_bytes, size_t S, int G,
                                                    TM* __restrict__ w_model) {
  constexpr float q = float((1 << (BITS == 32 ? 1 : BITS - 1)) - 1);
  const int j = blockIdx.y;
  const uint8_t* unit = units + (size_t)j * unit_bytes;
  const float* scales = reinterpret_cast<const float*>(unit + S * (BITS == 32 ? 4 : BITS) / 8);
  TM* wm = w_model + (size_t)j * S;
  const size_t ntiles = (S + 4095) / 4096;
  for (size_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const size_t e0 = tile * 4096 + threadIdx.x * 16;
    if (e0 >= S) continue;
    float x[16];
    if constexpr (BITS == 32) {
      const float4* src = reinterpret_cast<const float4*>(unit + e0 * 4);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4 t = src[i];
        x[4 * i] = t.x; x[4 * i + 1] = t.y; x[4 * i + 2] = t.z; x[4 * i + 3] = t.w;
      }
    } else {
      const float ds = __fdiv_rn(scales[e0 / G], q);
      float f[16];
      if constexpr (BITS == 4) {
        const uint2 w = *reinterpret_cast<const uint2*>(unit + e0 / 2);
        dec4x8(w.x, f);
        dec4x8(w.y, f + 8);
      } else {
        const uint4 w = *reinterpret_cast<const uint4*>(unit + e0);
        dec8x4(w.x, f); dec8x4(w.y, f + 4); dec8x4(w.z, f + 8); dec8x4(w.w, f + 12);
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) x[i] = __fmul_rn(f[i], ds);
    }
    if constexpr (sizeof(TM) == 2) {
      uint4* p = reinterpret_cast<uint4*>(wm + e0);
      uint4 u0 = p[0], u1 = p[1];
      uint32_t* w0 = &u0.x;
      uint32_t* w1 = &u1.x;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        w0[i] = pack_bf16x2(__fadd_rn(bf16_lo(w0[i]), x[2 * i]), __fadd_rn(bf16_hi(w0[i]), x[2 * i + 1]));
        w1[i] = pack_bf16x2(__fadd_rn(bf16_lo(w1[i]), x[8 + 2 * i]),
                            __fadd_rn(bf16_hi(w1[i]), x[8 + 2 * i + 1]));
      }
      p[0] = u0;
      p[1] = u1;
    } else {
      float4* p = reinterpret_cast<float4*>(wm + e0);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float4 t = p[i];
        t.x = __fadd_rn(t.x, x[4 * i]);
        t.y = __fadd_rn(t.y, x[4 * i + 1]);
        t.z = __fadd_rn(t.z, x[4 * i + 2]);
        t.w = __fadd_rn(t.w, x[4 * i + 3]);
        p[i] = t;
      }
    }
  }
}

// =====================================================================================
// K3  TLq-HS Hadamard + quantize (Alg. 3 l.2-3; fused per P:394-395).
// One thread owns one 64-element row; a CTA tile is 256 rows of one shard j, staged
// global -> smem with cp.async (double-buffered, XOR-swizzled), butterflied in
// registers, quantized, staged in smem and written coalesced to block l' = j % N,
// unit m' = j / N of the intra send buffer (R9).
// =====================================================================================
template <typename TG, int BITS>
__global__ void __launch_bounds__(kTileRows) k3_tlq_had_quant(const TG* __restrict__ grad, size_t S,
                                                             int M, int N, int G, int b, float cb,
                                                             uint8_t* __restrict__ intra_send,
                                                             size_t unit_bytes, size_t tiles_per_shard,
                                                             size_t ntiles) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int IN_CPR = kRowElems * (int)sizeof(TG) / 16;    // 8 (bf16) or 16 (fp32)
  constexpr int IN_TILE = kTileRows * IN_CPR * 16;
  constexpr int OUT_CPR = kRowElems * BITS / 8 / 16;          // 2, 4 or 16
  constexpr float q = float((1 << (BITS == 32 ? 1 : BITS - 1)) - 1);
  uint8_t* out_buf = smem + 2 * IN_TILE;
  const int t = threadIdx.x;
  const size_t rows_per_shard = S / kRowElems;

  auto issue_load = [&](size_t tile, int buf) {
    if (tile < ntiles) {
      const size_t j = tile / tiles_per_shard, ts = tile % tiles_per_shard;
      const size_t row0 = ts * kTileRows;
      const int rows = (int)min((size_t)kTileRows, rows_per_shard - row0);
      const uint8_t* src = reinterpret_cast<const uint8_t*>(grad + j * S + row0 * kRowElems);
      uint8_t* dst = smem + buf * IN_TILE;
      for (int i = t; i < rows * IN_CPR; i += kTileRows)
        cp_async16(dst + 16 * swz(i / IN_CPR, i % IN_CPR, IN_CPR), src + 16 * (size_t)i);
    }
    cp_async_commit();
  };

  int buf = 0;
  issue_load(blockIdx.x, 0);
  for (size_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, buf ^= 1) {
    issue_load(tile + gridDim.x, buf ^ 1);
    cp_async_wait<1>();
    __syncthreads();
    const size_t j = tile / tiles_per_shard, ts = tile % tiles_per_shard;
    const size_t row0 = ts * kTileRows;
    const int rows = (int)min((size_t)kTileRows, rows_per_shard - row0);
    const bool act = t < rows;

    float v[64];
    const uint8_t* in = smem + buf * IN_TILE;
    if (act) {
#pragma unroll
      for (int c = 0; c < IN_CPR; ++c) {
        const uint4 u = *reinterpret_cast<const uint4*>(in + 16 * swz(t, c, IN_CPR));
        if constexpr (sizeof(TG) == 2) {
          v[8 * c + 0] = bf16_lo(u.x); v[8 * c + 1] = bf16_hi(u.x);
          v[8 * c + 2] = bf16_lo(u.y); v[8 * c + 3] = bf16_hi(u.y);
          v[8 * c + 4] = bf16_lo(u.z); v[8 * c + 5] = bf16_hi(u.z);
          v[8 * c + 6] = bf16_lo(u.w); v[8 * c + 7] = bf16_hi(u.w);
        } else {
          v[4 * c + 0] = __uint_as_float(u.x); v[4 * c + 1] = __uint_as_float(u.y);
          v[4 * c + 2] = __uint_as_float(u.z); v[4 * c + 3] = __uint_as_float(u.w);
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 64; ++i) v[i] = 0.f;
    }
    fwht_row(v, b);

    const size_t lp = j % N, mp = j / N;
    uint8_t* unit = intra_send + (lp * M + mp) * unit_bytes;
    if constexpr (BITS == 32) {  // identity codec (R12): rn(u * c_b)
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const float4 o = make_float4(__fmul_rn(v[4 * c], cb), __fmul_rn(v[4 * c + 1], cb),
                                     __fmul_rn(v[4 * c + 2], cb), __fmul_rn(v[4 * c + 3], cb));
        *reinterpret_cast<float4*>(out_buf + 16 * swz(t, c, OUT_CPR)) = o;
      }
    } else {
      float* scales = reinterpret_cast<float*>(unit + S * BITS / 8) + row0 * kRowElems / G;
      // group maxima: G >= 64 -> one group spans G/64 rows (lanes); G == 32 -> two per row
      float a0 = 0.f, a1 = 0.f;
#pragma unroll
      for (int i = 0; i < 32; ++i) a0 = max_nan(a0, fabsf(v[i]));
#pragma unroll
      for (int i = 32; i < 64; ++i) a1 = max_nan(a1, fabsf(v[i]));
      QP p0, p1;
      if (G >= 64) {
        a0 = max_nan(a0, a1);
        for (int off = 1; off < G / 64; off <<= 1)
          a0 = max_nan(a0, __shfl_xor_sync(0xffffffffu, a0, off));
        a1 = a0;
        p0 = qparam(a0, q);
        p1 = p0;
        if (act && (t & (G / 64 - 1)) == 0) scales[t / (G / 64)] = stored_scale(a0, cb);
      } else {
        p0 = qparam(a0, q);
        p1 = qparam(a1, q);
        if (act)
          *reinterpret_cast<float2*>(scales + 2 * t) =
              make_float2(stored_scale(a0, cb), stored_scale(a1, cb));
      }
      uint32_t r[64];
#pragma unroll
      for (int i = 0; i < 32; ++i) r[i] = rq(v[i], p0.inv);
#pragma unroll
      for (int i = 32; i < 64; ++i) r[i] = rq(v[i], p1.inv);
      if constexpr (BITS == 8) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint4 w = make_uint4(pack8x4(r[16 * c], r[16 * c + 1], r[16 * c + 2], r[16 * c + 3]),
                               pack8x4(r[16 * c + 4], r[16 * c + 5], r[16 * c + 6], r[16 * c + 7]),
                               pack8x4(r[16 * c + 8], r[16 * c + 9], r[16 * c + 10], r[16 * c + 11]),
                               pack8x4(r[16 * c + 12], r[16 * c + 13], r[16 * c + 14], r[16 * c + 15]));
          if (!(c < 2 ? p0.ok : p1.ok)) w = make_uint4(0u, 0u, 0u, 0u);
          *reinterpret_cast<uint4*>(out_buf + 16 * swz(t, c, OUT_CPR)) = w;
        }
      } else {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint4 w = make_uint4(pack4x8(r + 32 * c), pack4x8(r + 32 * c + 8), pack4x8(r + 32 * c + 16),
                               pack4x8(r + 32 * c + 24));
          if (!(c == 0 ? p0.ok : p1.ok)) w = make_uint4(0u, 0u, 0u, 0u);
          *reinterpret_cast<uint4*>(out_buf + 16 * swz(t, c, OUT_CPR)) = w;
        }
      }
    }
    __syncthreads();
    // coalesced write-out of the tile's codes
    uint8_t* dst = unit + row0 * kRowElems * BITS / 8;
    for (int i = t; i < rows * OUT_CPR; i += kTileRows)
      *reinterpret_cast<uint4*>(dst + 16 * (size_t)i) =
          *reinterpret_cast<const uint4*>(out_buf + 16 * swz(i / OUT_CPR, i % OUT_CPR, OUT_CPR));
  }
  cp_async_wait<0>();
}

// =====================================================================================
// K4  TLq dequantize + reduce + requantize (Alg. 3 l.5, 7, 9, FP32 reduce
// P:344).  Sub-block m' = blockIdx.y; sources l'' = 0..N-1 summed in order (R8).
// 16 elements per thread; a group is G/16 consecutive threads.
// =====================================================================================
template <int BIN, int BOUT>
__global__ void __launch_bounds__(256) k4_tlq_dq_reduce_q(const uint8_t* __restrict__ recv,
                                                          size_t in_unit_bytes, int N, int M,
                                                          size_t S, int G,
                                                          uint8_t* __restrict__ send,
                                                          size_t out_unit_bytes) {
  __shared__ float red[8];
  constexpr float qin = float((1 << (BIN == 32 ? 1 : BIN - 1)) - 1);
  constexpr float qout = float((1 << (BOUT == 32 ? 1 : BOUT - 1)) - 1);
  const int mp = blockIdx.y;
  const int tpg = G >> 4;
  uint8_t* out = send + (size_t)mp * out_unit_bytes;
  float* oscales = reinterpret_cast<float*>(out + S * BOUT / 8);
  const size_t ntiles = (S + 4095) / 4096;
  for (size_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const size_t e0 = tile * 4096 + threadIdx.x * 16;
    const bool act = e0 < S;
    float acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0.f;
    if (act) {
      for (int l = 0; l < N; ++l) {
        const uint8_t* unit = recv + ((size_t)l * M + mp) * in_unit_bytes;
        float x[16];
        if constexpr (BIN == 32) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint4 u = ldg_stream(unit + (e0 + 4 * i) * 4);
            x[4 * i] = __uint_as_float(u.x); x[4 * i + 1] = __uint_as_float(u.y);
            x[4 * i + 2] = __uint_as_float(u.z); x[4 * i + 3] = __uint_as_float(u.w);
          }
        } else {
          const float s = reinterpret_cast<const float*>(unit + S * BIN / 8)[e0 / G];
          const float ds = __fdiv_rn(s, qin);
          float f[16];
          if constexpr (BIN == 8) {
            const uint4 w = ldg_stream(unit + e0);
            dec8x4(w.x, f); dec8x4(w.y, f + 4); dec8x4(w.z, f + 8); dec8x4(w.w, f + 12);
          } else {
            const uint2 w = *reinterpret_cast<const uint2*>(unit + e0 / 2);
            dec4x8(w.x, f); dec4x8(w.y, f + 8);
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) x[i] = __fmul_rn(f[i], ds);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = __fadd_rn(acc[i], x[i]);
      }
    }
    if constexpr (BOUT == 32) {
      if (act) {
        float4* o = reinterpret_cast<float4*>(out + e0 * 4);
#pragma unroll
        for (int i = 0; i < 4; ++i) o[i] = make_float4(acc[4 * i], acc[4 * i + 1], acc[4 * i + 2], acc[4 * i + 3]);
      }
    } else {
      float a = 0.f;
#pragma unroll
      for (int i = 0; i < 16; ++i) a = max_nan(a, fabsf(acc[i]));
      a = group_max(a, tpg, red);
      const QP p = qparam(a, qout);
      if (act) {
        uint32_t r[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) r[i] = rq(acc[i], p.inv);
        if constexpr (BOUT == 4) {
          uint2 w = make_uint2(pack4x8(r), pack4x8(r + 8));
          if (!p.ok) w = make_uint2(0u, 0u);
          *reinterpret_cast<uint2*>(out + e0 / 2) = w;
        } else {
          uint4 w = make_uint4(pack8x4(r[0], r[1], r[2], r[3]), pack8x4(r[4], r[5], r[6], r[7]),
                               pack8x4(r[8], r[9], r[10], r[11]), pack8x4(r[12], r[13], r[14], r[15]));
          if (!p.ok) w = make_uint4(0u, 0u, 0u, 0u);
          *reinterpret_cast<uint4*>(out + e0) = w;
        }
        if ((threadIdx.x & (tpg - 1)) == 0) oscales[e0 / G] = stored_scale(a, 1.f);
      }
    }
  }
}

// =====================================================================================
// K5  TLq-HS dequantize + reduce + inverse Hadamard (Alg. 3 l.11-13; the H
// moved after the final reduction).  Row layout (64 elements per thread);
// sources m'' = 0..M-1 in order (R8); out = rn(H_unnorm(acc) * kappa) (R8).
// =====================================================================================
template <int BIN>
__global__ void __launch_bounds__(kTileRows) k5_tlq_dq_reduce_had(const uint8_t* __restrict__ recv,
                                                                 size_t in_unit_bytes, int M, size_t S,
                                                                 int G, int b, float kappa,
                                                                 float* __restrict__ out,
                                                                 size_t ntiles) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr float qin = float((1 << (BIN == 32 ? 1 : BIN - 1)) - 1);
  constexpr int ROW_BYTES = kRowElems * BIN / 8;
  const int t = threadIdx.x;
  const size_t rows_per_shard = S / kRowElems;
  for (size_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const size_t row0 = tile * kTileRows;
    const int rows = (int)min((size_t)kTileRows, rows_per_shard - row0);
    const bool act = t < rows;
    const size_t row = row0 + t;
    float v[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) v[i] = 0.f;
    if (act) {
      for (int m = 0; m < M; ++m) {
        const uint8_t* unit = recv + (size_t)m * in_unit_bytes;
        const uint8_t* src = unit + row * ROW_BYTES;
        if constexpr (BIN == 32) {
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const uint4 u = ldg_stream(src + 16 * c);
            v[4 * c] = __fadd_rn(v[4 * c], __uint_as_float(u.x));
            v[4 * c + 1] = __fadd_rn(v[4 * c + 1], __uint_as_float(u.y));
            v[4 * c + 2] = __fadd_rn(v[4 * c + 2], __uint_as_float(u.z));
            v[4 * c + 3] = __fadd_rn(v[4 * c + 3], __uint_as_float(u.w));
          }
        } else {
          const float* sc = reinterpret_cast<const float*>(unit + S * BIN / 8);
          float ds0, ds1;
          if (G >= 64) {
            ds0 = ds1 = __fdiv_rn(sc[row * kRowElems / G], qin);
          } else {
            const float2 s2 = *reinterpret_cast<const float2*>(sc + 2 * row);
            ds0 = __fdiv_rn(s2.x, qin);
            ds1 = __fdiv_rn(s2.y, qin);
          }
#pragma unroll
          for (int c = 0; c < ROW_BYTES / 16; ++c) {
            const uint4 u = ldg_stream(src + 16 * c);
            const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              if constexpr (BIN == 4) {
                float f[8];
                dec4x8(w[k], f);
                const int base = 32 * c + 8 * k;
                const float ds = base < 32 ? ds0 : ds1;
#pragma unroll
                for (int i = 0; i < 8; ++i) v[base + i] = __fadd_rn(v[base + i], __fmul_rn(f[i], ds));
              } else {
                float f[4];
                dec8x4(w[k], f);
                const int base = 16 * c + 4 * k;
                const float ds = base < 32 ? ds0 : ds1;
#pragma unroll
                for (int i = 0; i < 4; ++i) v[base + i] = __fadd_rn(v[base + i], __fmul_rn(f[i], ds));
              }
            }
          }
        }
      }
    }
    fwht_row(v, b);
    __syncthreads();  // previous tile's write-out finished reading smem
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const float4 o = make_float4(__fmul_rn(v[4 * c], kappa), __fmul_rn(v[4 * c + 1], kappa),
                                   __fmul_rn(v[4 * c + 2], kappa), __fmul_rn(v[4 * c + 3], kappa));
      *reinterpret_cast<float4*>(smem + 16 * swz(t, c, 16)) = o;
    }
    __syncthreads();
    uint8_t* dst = reinterpret_cast<uint8_t*>(out + row0 * kRowElems);
    for (int i = t; i < rows * 16; i += kTileRows)
      *reinterpret_cast<uint4*>(dst + 16 * (size_t)i) =
          *reinterpret_cast<const uint4*>(smem + 16 * swz(i / 16, i % 16, 16));
  }
}

inline int grid_for(size_t ntiles, int cap) {
  return (int)(ntiles < (size_t)cap ? (ntiles == 0 ? 1 : ntiles) : (size_t)cap);
}

template <typename K>
cudaError_t set_smem(K kernel, int bytes) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

}  // namespace

// ------------------------------- launchers -------------------------------------------
cudaError_t launch_qwd_quantize(const float* w_main, const void* w_model_shard, int model_dtype,
                                size_t S, int bits, int G, uint8_t* unit, int grid_cap,
                                cudaStream_t st) {
  const int grid = grid_for((S + 2047) / 2048, grid_cap);
#define K1(TM, B) \
  k1_qwd_quantize<TM, B><<<grid, 256, 0, st>>>(w_main, static_cast<const TM*>(w_model_shard), S, G, unit)
  if (model_dtype == kBF16) {
    if (bits == 4) K1(uint16_t, 4); else if (bits == 8) K1(uint16_t, 8); else K1(uint16_t, 32);
  } else {
    if (bits == 4) K1(float, 4); else if (bits == 8) K1(float, 8); else K1(float, 32);
  }
#undef K1
  return cudaGetLastError();
}

cudaError_t launch_qwd_apply(const uint8_t* units, size_t unit_bytes, int P, size_t S, int bits,
                             int G, void* w_model, int model_dtype, int grid_cap, cudaStream_t st) {
  const int gx = grid_for((S + 4095) / 4096, (grid_cap + P - 1) / P);
  const dim3 grid(gx, P);
#define K2(TM, B) \
  k2_qwd_apply<TM, B><<<grid, 256, 0, st>>>(units, unit_bytes, S, G, static_cast<TM*>(w_model))
  if (model_dtype == kBF16) {
    if (bits == 4) K2(uint16_t, 4); else if (bits == 8) K2(uint16_t, 8); else K2(uint16_t, 32);
  } else {
    if (bits == 4) K2(float, 4); else if (bits == 8) K2(float, 8); else K2(float, 32);
  }
#undef K2
  return cudaGetLastError();
}

cudaError_t launch_tlq_had_quant(const void* grad, int grad_dtype, size_t S, int M, int N, int G,
                                 int b, float cb, int bits, uint8_t* intra_send, size_t unit_bytes,
                                 int grid_cap, cudaStream_t st) {
  const size_t tps = (S / kRowElems + kTileRows - 1) / kTileRows;
  const size_t ntiles = tps * (size_t)M * N;
  const int grid = grid_for(ntiles, grid_cap);
  cudaError_t e = cudaSuccess;
#define K3(TG, B)                                                                              \
  do {                                                                                         \
    const int smem = 2 * kTileRows * kRowElems * (int)sizeof(TG) + kTileRows * kRowElems * B / 8; \
    e = set_smem(k3_tlq_had_quant<TG, B>, smem);                                               \
    if (e != cudaSuccess) return e;                                                            \
    k3_tlq_had_quant<TG, B><<<grid, kTileRows, smem, st>>>(static_cast<const TG*>(grad), S, M, N, \
                                                           G, b, cb, intra_send, unit_bytes, tps, \
                                                           ntiles);                            \
  } while (0)
  if (grad_dtype == kBF16) {
    if (bits == 4) K3(uint16_t, 4); else if (bits == 8) K3(uint16_t, 8); else K3(uint16_t, 32);
  } else {
    if (bits == 4) K3(float, 4); else if (bits == 8) K3(float, 8); else K3(float, 32);
  }
#undef K3
  return cudaGetLastError();
}

cudaError_t launch_tlq_dq_reduce_q(const uint8_t* intra_recv, size_t in_unit_bytes, int bits_in,
                                   int N, int M, size_t S, int G, uint8_t* inter_send,
                                   size_t out_unit_bytes, int bits_out, int grid_cap,
                                   cudaStream_t st) {
  const int gx = grid_for((S + 4095) / 4096, (grid_cap + M - 1) / M);
  const dim3 grid(gx, M);
#define K4(BI, BO)                                                                          \
  k4_tlq_dq_reduce_q<BI, BO><<<grid, 256, 0, st>>>(intra_recv, in_unit_bytes, N, M, S, G, \
                                                    inter_send, out_unit_bytes)
#define K4O(BI) \
  if (bits_out == 4) K4(BI, 4); else if (bits_out == 8) K4(BI, 8); else K4(BI, 32)
  if (bits_in == 4) { K4O(4); } else if (bits_in == 8) { K4O(8); } else { K4O(32); }
#undef K4O
#undef K4
  return cudaGetLastError();
}

cudaError_t launch_tlq_dq_reduce_had(const uint8_t* inter_recv, size_t in_unit_bytes, int bits_in,
                                     int M, size_t S, int G, int b, float kappa, float* out,
                                     int grid_cap, cudaStream_t st) {
  const size_t ntiles = (S / kRowElems + kTileRows - 1) / kTileRows;
  const int grid = grid_for(ntiles, grid_cap);
  const int smem = kTileRows * kRowElems * 4;
  cudaError_t e = cudaSuccess;
#define K5(BI)                                                                                 \
  do {                                                                                         \
    e = set_smem(k5_tlq_dq_reduce_had<BI>, smem);                                              \
    if (e != cudaSuccess) return e;                                                            \
    k5_tlq_dq_reduce_had<BI><<<grid, kTileRows, smem, st>>>(inter_recv, in_unit_bytes, M, S, G, b, \
                                                            kappa, out, ntiles);               \
  } while (0)
  if (bits_in == 4) K5(4); else if (bits_in == 8) K5(8); else K5(32);
#undef K5
  return cudaGetLastError();
}

}  // namespace sdp4
