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
//  K3 tlq_had_quant     Alg. 3 l.2-3, fused   row layout (64 el/thread, f32x2),
//                       Hadamard + quantize    TMA tensor ring in, TMA store out
//  K4 tlq_dq_reduce_q   Alg. 3 l.5,7,9        vector layout, 1-D bulk-copy ring
//  K5 tlq_dq_reduce_had Alg. 3 l.11-13 row layout, TMA ring in, TMA store out
//
// Integer rounding uses the magic-number identity: for |y| <= 2^22,
// rn(y + 1.5*2^23) is the nearest-even integer of y and its low mantissa bits
// hold that integer in two's complement, so a code is one FADD (not a quarter-rate
// F2I) and packing is byte/nibble selection.  Decoding inverts it with PRMT + FADD.
#include "sdp4_kernels.cuh"

#include <cfloat>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <cuda.h>
#include <cudaTypedefs.h>
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
// 3-input form (sm_100 FMNMX3): max|.| of two more elements per instruction
__device__ __forceinline__ float max3_abs_nan(float a, float b, float c) {
  float r;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(fabsf(b)), "f"(fabsf(c)));
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
// RNE(x * inv) of the exact product (R3: one rounding), as magic-number bits:
// fma(x, inv, 1.5*2^23) rounds the exact x*inv + 1.5*2^23 once, to an integer.
__device__ __forceinline__ uint32_t rq(float x, float inv) { return __float_as_uint(__fmaf_rn(x, inv, kMagic)); }

// Stochastic rounding (NEXT-2, R14): counter-based uniform U_i = (h >> 8) * 2^-24 with
// h = mix32(lo32(i) ^ mix32(hi32(i) ^ key)); y = rn(x*inv), fl = floor(y), fr = rn(y - fl),
// code = clamp(fl + [U < fr], +-q) -- unbiased (Def. 1).
__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}
__device__ __forceinline__ float sr_u(uint64_t i, uint32_t key) {
  const uint32_t h = mix32((uint32_t)i ^ mix32((uint32_t)(i >> 32) ^ key));
  return __uint2float_rn(h >> 8) * 0x1p-24f;  // exact: 24-bit integer times 2^-24
}
__device__ __forceinline__ uint32_t rq_sr(float x, float inv, float u, float q) {
  const float y = __fmul_rn(x, inv);
  const float fl = floorf(y);
  const float fr = __fsub_rn(y, fl);
  const float c = fminf(fmaxf(__fadd_rn(fl, u < fr ? 1.f : 0.f), -q), q);
  return __float_as_uint(__fadd_rn(c, kMagic));  // c is a small integer: exact magic bits
}
struct SR {
  int on;        // 0: round to nearest even (R3)
  uint32_t key;  // per (seed, stage, rank)
};
__device__ __forceinline__ uint32_t pack8x4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}
// int2 (ternary weight codec, R4): element 4j+i in bits 2i..2i+1 of byte j.
__device__ __forceinline__ uint32_t pack2x8(const uint32_t* r) {
  uint32_t w = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) w |= (r[i] & 3u) << (2 * i);
  return w;
}
__device__ __forceinline__ void dec2x16(uint32_t w, float* f) {
#pragma unroll
  for (int i = 0; i < 16; ++i) f[i] = float((int)(((w >> (2 * i)) & 3u) ^ 2u) - 2);
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

// =====================================================================================
// TMA (cp.async.bulk[.tensor]) + mbarrier primitives (sm_90+ PTX, used on sm_100a).
// =====================================================================================
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n\tfence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(map), "r"(c0),
               "r"(c1), "r"(c2), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(map),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(src))
               : "memory");
}
// 1-D bulk copy global -> shared (16-byte aligned, size a multiple of 16)
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// 1-D bulk copy shared -> global (local or peer memory over NVLink; 16-byte aligned,
// size a multiple of 16)
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// Store a finished output tile staged in smem -- `cbytes` code bytes and `nsc` fp32 scales
// -- to one destination unit with 1-D bulk copies issued by thread 0 (the 16-byte multiple
// prefix of the scales; the < 4 trailing scales are stored by lanes of warp 1).  The caller
// has done fence_proxy_async + __syncthreads, and thread 0 commits the bulk group after
// the last destination.  Contiguous bulk stores keep NVLink transfers at full efficiency.
__device__ __forceinline__ void store_tile(const uint8_t* s_codes, uint32_t cbytes, const float* s_sc, uint32_t nsc,
                                           uint8_t* g_codes, float* g_sc) {
  const uint32_t n16 = nsc & ~3u;
  if (threadIdx.x == 0) {
    bulk_store(g_codes, s_codes, cbytes);
    if (n16) bulk_store(g_sc, s_sc, n16 * 4);
  }
  const int k = (int)threadIdx.x - 32;
  if (k >= 0 && k < (int)(nsc - n16)) g_sc[n16 + k] = s_sc[n16 + k];
}

// Row tiles: kTileRows rows of R bytes of one unit.  R <= 128: one TMA box {R, 256, 1},
// smem [256][R] with the hardware swizzle of width R (SWIZZLE_32B/64B/128B: 16-byte chunk
// index XOR address bits 7..); R == 256: two boxes (halves) {128, 1, 256, 1}, smem
// [2][256][128], SWIZZLE_128B.  Thread r touching chunk c of its own row is conflict-free
// (8 consecutive rows of a quarter-warp hit 8 distinct bank groups).
template <int R, int ROWS = kTileRows>
__device__ __forceinline__ uint32_t tile_off(int r, int c) {
  if constexpr (R == 256) return (c >> 3) * (ROWS * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4);
  else if constexpr (R == 128) return r * 128 + ((c ^ (r & 7)) << 4);
  else if constexpr (R == 64) return r * 64 + ((c ^ ((r >> 1) & 3)) << 4);
  else return r * 32 + ((c ^ ((r >> 2) & 1)) << 4);
}
template <int R, int ROWS = kTileRows>
__device__ __forceinline__ void tma_load_tile(void* dst, const CUtensorMap* map, uint64_t* bar, int row, int unit) {
  if constexpr (R == 256) {
    tma_load_4d(dst, map, bar, 0, 0, row, unit);
    tma_load_4d(static_cast<uint8_t*>(dst) + ROWS * 128, map, bar, 0, 1, row, unit);
  } else {
    tma_load_3d(dst, map, bar, 0, row, unit);
  }
}
template <int R, int ROWS = kTileRows>
__device__ __forceinline__ void tma_store_tile(const CUtensorMap* map, const void* src, int row, int unit) {
  if constexpr (R == 256) {
    tma_store_4d(map, src, 0, 0, row, unit);
    tma_store_4d(map, static_cast<const uint8_t*>(src) + ROWS * 128, 0, 1, row, unit);
  } else {
    tma_store_3d(map, src, 0, row, unit);
  }
}

// ---- packed fp32x2 (sm_100a FADD2 / FMUL2: two IEEE round-to-nearest ops per instruction).
// Inline PTX with an explicit .rn: never contracted into FFMA2 (the __fmul2_rn/__fadd2_rn
// builtins were observed to fuse into FFMA2 under nvcc 12.9, which changes roundings).
__device__ __forceinline__ float2 f2op_add(float2 a, float2 b) {
  float2 r;
  asm("{\n\t.reg .b64 pa, pb, pd;\n\tmov.b64 pa, {%2, %3};\n\tmov.b64 pb, {%4, %5};\n\t"
      "add.rn.f32x2 pd, pa, pb;\n\tmov.b64 {%0, %1}, pd;\n\t}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 f2sub(float2 a, float2 b) {
  float2 r;
  asm("{\n\t.reg .b64 pa, pb, pd;\n\tmov.b64 pa, {%2, %3};\n\tmov.b64 pb, {%4, %5};\n\t"
      "sub.rn.f32x2 pd, pa, pb;\n\tmov.b64 {%0, %1}, pd;\n\t}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 f2mul(float2 a, float2 b) {
  float2 r;
  asm("{\n\t.reg .b64 pa, pb, pd;\n\tmov.b64 pa, {%2, %3};\n\tmov.b64 pb, {%4, %5};\n\t"
      "mul.rn.f32x2 pd, pa, pb;\n\tmov.b64 {%0, %1}, pd;\n\t}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 f2add(float2 a, float2 b) { return f2op_add(a, b); }
// Packed rq: RNE(x * inv) bits for two elements (explicit FFMA2, exact product).
__device__ __forceinline__ float2 f2rq(float2 a, float2 inv) {
  float2 r;
  asm("{\n\t.reg .b64 pa, pb, pc, pd;\n\tmov.b64 pa, {%2, %3};\n\tmov.b64 pb, {%4, %5};\n\t"
      "mov.b64 pc, {%6, %6};\n\tfma.rn.f32x2 pd, pa, pb, pc;\n\tmov.b64 {%0, %1}, pd;\n\t}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(inv.x), "f"(inv.y), "f"(kMagic));
  return r;
}
// NOTE: ptxas (12.9) contracts a multiply feeding an add into FFMA2 even with .rn and
// --fmad=false (it also re-vectorizes scalar __fmul_rn/__fadd_rn pairs and then fuses them).
// Every product that is later added is therefore computed as fma(a, b, z) with z = -0.0f
// passed as a kernel argument: bit-identical to rn(a*b) (x + -0 == x, +0 + -0 == +0), and
// ptxas can neither drop the unknown addend nor fuse an FMA into the following add.
// tests/test_sass.py rejects any FFMA2 whose addend is a packed accumulator.
__device__ __forceinline__ float2 f2mulz(float2 a, float2 b, float z) {
  float2 r;
  asm("{\n\t.reg .b64 pa, pb, pc, pd;\n\tmov.b64 pa, {%2, %3};\n\tmov.b64 pb, {%4, %5};\n\t"
      "mov.b64 pc, {%6, %6};\n\tfma.rn.f32x2 pd, pa, pb, pc;\n\tmov.b64 {%0, %1}, pd;\n\t}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(z));
  return r;
}
__device__ __forceinline__ float mulz(float a, float b, float z) { return __fmaf_rn(a, b, z); }

// A 64-element row lives in 32 f32x2 registers p[i] = {v[i], v[i+32]}.
//
// Unnormalized Sylvester butterfly of one b-block (R6): stages h = 1, 2, ..., B/2 in
// ascending order, pairs (i, i+h) -> (a + c, a - c).  Stages h < 32 act on whole pairs
// (elements i and i+32 play the same role), h = 32 inside each pair, and h = 64, 128 pair
// row t with row t ^ (h / 64) of the same warp.
template <int B>
__device__ __forceinline__ void fwht_pairs(float2* p) {
#pragma unroll
  for (int h = 1; h < 32 && h < B; h <<= 1) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if ((i & h) == 0) {
        const float2 a = p[i], c = p[i + h];
        p[i] = f2add(a, c);
        p[i + h] = f2sub(a, c);
      }
    }
  }
  if constexpr (B >= 64) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float a = p[i].x, c = p[i].y;
      p[i] = make_float2(__fadd_rn(a, c), __fsub_rn(a, c));
    }
  }
#pragma unroll
  for (int hx = 1; 64 * hx < B; hx <<= 1) {
    const bool upper = (threadIdx.x & hx) != 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float2 o = make_float2(__shfl_xor_sync(0xffffffffu, p[i].x, hx), __shfl_xor_sync(0xffffffffu, p[i].y, hx));
      p[i] = upper ? f2sub(o, p[i]) : f2add(p[i], o);
    }
  }
}

// Code decoding with the exact magic subtraction done by FADD2 (add -> mul cannot contract).
__device__ __forceinline__ void dec8x4_2(uint32_t w, float* f) {
  const uint32_t x = w ^ 0x80808080u;
  const float2 d = make_float2(-kDec8, -kDec8);
  const float2 a = f2add(make_float2(__uint_as_float(__byte_perm(x, 0x4B000000u, 0x7540)),
                                     __uint_as_float(__byte_perm(x, 0x4B000000u, 0x7541))), d);
  const float2 b = f2add(make_float2(__uint_as_float(__byte_perm(x, 0x4B000000u, 0x7542)),
                                     __uint_as_float(__byte_perm(x, 0x4B000000u, 0x7543))), d);
  f[0] = a.x; f[1] = a.y; f[2] = b.x; f[3] = b.y;
}
__device__ __forceinline__ void dec4x8_2(uint32_t w, float* f) {
  const uint32_t x = w ^ 0x88888888u;
  const uint32_t lo = x & 0x0F0F0F0Fu, hi = (x >> 4) & 0x0F0F0F0Fu;
  const float2 d = make_float2(-kDec4, -kDec4);
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const float2 v = f2add(make_float2(__uint_as_float(__byte_perm(lo, 0x4B000000u, 0x7540 + b)),
                                       __uint_as_float(__byte_perm(hi, 0x4B000000u, 0x7540 + b))), d);
    f[2 * b] = v.x;
    f[2 * b + 1] = v.y;
  }
}

// K5's row layout: 32 f32x2 registers p[j] = {v[2j], v[2j+1]} (adjacent elements), so the
// decoded pairs come straight out of one FADD2 each and four consecutive elements are one
// 16-byte store -- no re-pairing moves.
//
// Decode the 64 codes of row t of a row tile (R = 64*BIN/8 bytes) and dequantize:
// x[j] = {code_2j, code_2j+1} * ds (ds0 for elements 0..31, ds1 for 32..63).
template <int BIN, int R, int ROWS>
__device__ __forceinline__ void dequant_row_adj(const uint8_t* tile, int t, float ds0, float ds1, float z,
                                                float2* x) {
#pragma unroll
  for (int c = 0; c < R / 16; ++c) {
    const uint4 u = *reinterpret_cast<const uint4*>(tile + tile_off<R, ROWS>(t, c));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
    if constexpr (BIN == 32) {  // chunk c: elements 4c..4c+3
      x[2 * c] = make_float2(__uint_as_float(w[0]), __uint_as_float(w[1]));
      x[2 * c + 1] = make_float2(__uint_as_float(w[2]), __uint_as_float(w[3]));
    } else if constexpr (BIN == 8) {  // chunk c: elements 16c..16c+15 (word q: 16c + 4q + k)
      const float d = c < 2 ? ds0 : ds1;
      const float2 dd = make_float2(d, d), m = make_float2(-kDec8, -kDec8);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t xw = w[q] ^ 0x80808080u;
        const float2 v0 = f2add(make_float2(__uint_as_float(__byte_perm(xw, 0x4B000000u, 0x7540)),
                                            __uint_as_float(__byte_perm(xw, 0x4B000000u, 0x7541))), m);
        const float2 v1 = f2add(make_float2(__uint_as_float(__byte_perm(xw, 0x4B000000u, 0x7542)),
                                            __uint_as_float(__byte_perm(xw, 0x4B000000u, 0x7543))), m);
        x[8 * c + 2 * q] = f2mulz(v0, dd, z);
        x[8 * c + 2 * q + 1] = f2mulz(v1, dd, z);
      }
    } else {  // BIN == 4: chunk c: elements 32c..32c+31 (word q: 32c + 8q + 2k + {0, 1})
      const float d = c == 0 ? ds0 : ds1;
      const float2 dd = make_float2(d, d), m = make_float2(-kDec4, -kDec4);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t xw = w[q] ^ 0x88888888u;
        const uint32_t lo = xw & 0x0F0F0F0Fu, hi = (xw >> 4) & 0x0F0F0F0Fu;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 v = f2add(make_float2(__uint_as_float(__byte_perm(lo, 0x4B000000u, 0x7540 + k)),
                                             __uint_as_float(__byte_perm(hi, 0x4B000000u, 0x7540 + k))), m);
          x[16 * c + 4 * q + k] = f2mulz(v, dd, z);
        }
      }
    }
  }
}

// Unnormalized Sylvester butterfly (R6) on the adjacent-pair layout: stage h = 1 inside each
// pair, h = 2..32 between pairs j and j + h/2, h = 64, 128 across lanes (row t ^ h/64).
template <int B>
__device__ __forceinline__ void fwht_adj(float2* p) {
  if constexpr (B >= 2) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float a = p[j].x, c = p[j].y;
      p[j] = make_float2(__fadd_rn(a, c), __fsub_rn(a, c));
    }
  }
#pragma unroll
  for (int h2 = 1; h2 < 32 && 2 * h2 < B; h2 <<= 1) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if ((j & h2) == 0) {
        const float2 a = p[j], c = p[j + h2];
        p[j] = f2add(a, c);
        p[j + h2] = f2sub(a, c);
      }
    }
  }
#pragma unroll
  for (int hx = 1; 64 * hx < B; hx <<= 1) {
    const bool upper = (threadIdx.x & hx) != 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float2 o = make_float2(__shfl_xor_sync(0xffffffffu, p[i].x, hx), __shfl_xor_sync(0xffffffffu, p[i].y, hx));
      p[i] = upper ? f2sub(o, p[i]) : f2add(p[i], o);
    }
  }
}

// Quantize a 64-element row held as pairs (R2, R3) into codes in an output row tile (LINEAR:
// row-major for a 1-D bulk store to a peer; else the TMA-swizzled layout for a tensor store);
// the group's first row writes the scale rn(s * c) (R6) to scales_tile.  lg = log2 G:
// G >= 64 -> a group spans G/64 rows (lanes); G == 32 -> two groups per row (one per half).
template <int BITS, int R, bool LINEAR, bool STOCH>
__device__ __forceinline__ void quant_row(const float2* p, int t, int lg, float c, bool act, uint8_t* out_tile,
                                          float* scales_tile, const SR& sr, uint64_t i0) {
  constexpr float q = float((1 << (BITS - 1)) - 1);
  float a0 = 0.f, a1 = 0.f;
#pragma unroll
  for (int i = 0; i < 32; i += 2) {
    a0 = max3_abs_nan(a0, p[i].x, p[i + 1].x);
    a1 = max3_abs_nan(a1, p[i].y, p[i + 1].y);
  }
  QP p0, p1;
  if (lg >= 6) {
    a0 = max_nan(a0, a1);
    const int rpg = 1 << (lg - 6);
    for (int off = 1; off < rpg; off <<= 1) a0 = max_nan(a0, __shfl_xor_sync(0xffffffffu, a0, off));
    p0 = qparam(a0, q);
    p1 = p0;
    if (act && (t & (rpg - 1)) == 0) scales_tile[t >> (lg - 6)] = stored_scale(a0, c);
  } else {
    p0 = qparam(a0, q);
    p1 = qparam(a1, q);
    if (act) *reinterpret_cast<float2*>(scales_tile + 2 * t) = make_float2(stored_scale(a0, c), stored_scale(a1, c));
  }
  const float2 inv = make_float2(p0.inv, p1.inv);
  uint32_t rx[32], ry[32];
  if constexpr (STOCH) {  // element i of the row has global index i0 + i (stochastic rounding, R14)
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      rx[i] = rq_sr(p[i].x, inv.x, sr_u(i0 + i, sr.key), q);
      ry[i] = rq_sr(p[i].y, inv.y, sr_u(i0 + 32 + i, sr.key), q);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float2 y = f2rq(p[i], inv);
      rx[i] = __float_as_uint(y.x);
      ry[i] = __float_as_uint(y.y);
    }
  }
  if constexpr (BITS == 8) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t* r = (k < 2 ? rx : ry) + 16 * (k & 1);
      uint4 w = make_uint4(pack8x4(r[0], r[1], r[2], r[3]), pack8x4(r[4], r[5], r[6], r[7]),
                           pack8x4(r[8], r[9], r[10], r[11]), pack8x4(r[12], r[13], r[14], r[15]));
      if (!(k < 2 ? p0.ok : p1.ok)) w = make_uint4(0u, 0u, 0u, 0u);
      *reinterpret_cast<uint4*>(out_tile + (LINEAR ? t * R + 16 * k : tile_off<R>(t, k))) = w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const uint32_t* r = k == 0 ? rx : ry;
      uint4 w = make_uint4(pack4x8(r), pack4x8(r + 8), pack4x8(r + 16), pack4x8(r + 24));
      if (!(k == 0 ? p0.ok : p1.ok)) w = make_uint4(0u, 0u, 0u, 0u);
      *reinterpret_cast<uint4*>(out_tile + (LINEAR ? t * R + 16 * k : tile_off<R>(t, k))) = w;
    }
  }
}

// Incremental (unit, tile-in-unit) coordinates of tile = blockIdx.x + i * gridDim.x with the
// unit index fastest (tile = ts * U + unit): consecutive tiles go to different destinations,
// so local (HBM) and peer (NVLink) stores of a pushing kernel overlap instead of forming
// phases.
struct TileIter {
  uint32_t unit, ts, U, gq, gr;
  __device__ explicit TileIter(uint32_t units) : U(units) {
    ts = blockIdx.x / U;
    unit = blockIdx.x - ts * U;
    gq = gridDim.x / U;
    gr = gridDim.x - gq * U;
  }
  __device__ void next() {
    unit += gr;
    ts += gq;
    if (unit >= U) {
      unit -= U;
      ++ts;
    }
  }
};

// =====================================================================================
// K1  qWD quantize (Alg. 2 l.2-3): d = rn(w_main - widen(w_model)),
// per G-group s = max|d|, codes = RNE(d * rn(q/s)) (R3: fused, exact product).  8 elements per
// thread, a group is G/8 consecutive threads.  Output: one wire unit [codes][scales].
// DIFF = false is the qW ablation codec (Alg. 1, QSDP / ZeRO++): d = w_main itself.
// APPLY: the owner also applies its own unit to its replica shard here (Alg. 2 l.5 for
// j = rank), decoding the codes it just packed with K2's exact arithmetic, so the replica
// shard it already holds in registers is not read again by K2 (sdp4_qwd_step).
// =====================================================================================
constexpr int kVecThreads = 256;  // K1 / K2: 256-thread CTAs, kVecCtas per SM (persistent)

// w[i] = rn(m[i] + x[i]) for 8 replica elements (m = widen(w) already in registers), stored
// with one 16-byte (bf16) or two 16-byte (fp32) stores -- K2's update, element by element.
template <typename TM>
__device__ __forceinline__ void apply_own(TM* w, const float* m, const float* x) {
  if constexpr (sizeof(TM) == 2) {
    uint4 o;
    uint32_t* ow = &o.x;
#pragma unroll
    for (int i = 0; i < 4; ++i) ow[i] = pack_bf16x2(__fadd_rn(m[2 * i], x[2 * i]), __fadd_rn(m[2 * i + 1], x[2 * i + 1]));
    *reinterpret_cast<uint4*>(w) = o;
  } else {
    reinterpret_cast<float4*>(w)[0] = make_float4(__fadd_rn(m[0], x[0]), __fadd_rn(m[1], x[1]), __fadd_rn(m[2], x[2]),
                                                  __fadd_rn(m[3], x[3]));
    reinterpret_cast<float4*>(w)[1] = make_float4(__fadd_rn(m[4], x[4]), __fadd_rn(m[5], x[5]), __fadd_rn(m[6], x[6]),
                                                  __fadd_rn(m[7], x[7]));
  }
}
constexpr int kVecCtas = 8;

template <typename TM, int BITS, bool DIFF, bool APPLY>
__global__ void __launch_bounds__(kVecThreads) k1_qwd_quantize(const float* __restrict__ w_main,
                                                                   TM* __restrict__ w_model, size_t S,
                                                                   int lg, const Dests dst, const SR sr,
                                                                   uint64_t idx0, float z) {
  static_assert(!APPLY || DIFF, "the owner's apply is the qWD update");
  constexpr int TILE = kVecThreads * 8;
  __shared__ float red[kVecThreads / 32];
  constexpr float q = float((1 << (BITS == 32 ? 1 : BITS - 1)) - 1);
  const int tpg = (1 << lg) >> 3;
  const size_t ntiles = (S + TILE - 1) / TILE;
  const size_t sc_off = S * (BITS == 32 ? 4 : BITS) / 8;
  const int t = threadIdx.x;
  // the next tile's inputs are loaded before this tile's arithmetic (one tile of prefetch)
  float4 na0, na1;
  uint4 nu0, nu1;
  auto load = [&](size_t tile) {
    const size_t e = tile * TILE + t * 8;
    if (tile < ntiles && e < S) {
      na0 = *reinterpret_cast<const float4*>(w_main + e);
      na1 = *reinterpret_cast<const float4*>(w_main + e + 4);
      if constexpr (DIFF) {
        nu0 = *reinterpret_cast<const uint4*>(w_model + e);
        if constexpr (sizeof(TM) == 4) nu1 = *reinterpret_cast<const uint4*>(w_model + e + 4);
      }
    }
  };
  load(blockIdx.x);
  for (size_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const size_t e0 = tile * TILE + t * 8;
    const bool act = e0 < S;
    const float4 a0 = na0, a1 = na1;
    const uint4 u0 = nu0, u1 = nu1;
    load(tile + gridDim.x);
    float d[8], m[8];
    if (act) {
      if constexpr (!DIFF) {
#pragma unroll
        for (int i = 0; i < 8; ++i) m[i] = 0.f;
      } else if constexpr (sizeof(TM) == 2) {
        m[0] = bf16_lo(u0.x); m[1] = bf16_hi(u0.x); m[2] = bf16_lo(u0.y); m[3] = bf16_hi(u0.y);
        m[4] = bf16_lo(u0.z); m[5] = bf16_hi(u0.z); m[6] = bf16_lo(u0.w); m[7] = bf16_hi(u0.w);
      } else {
        m[0] = __uint_as_float(u0.x); m[1] = __uint_as_float(u0.y); m[2] = __uint_as_float(u0.z);
        m[3] = __uint_as_float(u0.w); m[4] = __uint_as_float(u1.x); m[5] = __uint_as_float(u1.y);
        m[6] = __uint_as_float(u1.z); m[7] = __uint_as_float(u1.w);
      }
      if constexpr (DIFF) {
        d[0] = __fsub_rn(a0.x, m[0]); d[1] = __fsub_rn(a0.y, m[1]);
        d[2] = __fsub_rn(a0.z, m[2]); d[3] = __fsub_rn(a0.w, m[3]);
        d[4] = __fsub_rn(a1.x, m[4]); d[5] = __fsub_rn(a1.y, m[5]);
        d[6] = __fsub_rn(a1.z, m[6]); d[7] = __fsub_rn(a1.w, m[7]);
      } else {
        d[0] = a0.x; d[1] = a0.y; d[2] = a0.z; d[3] = a0.w;
        d[4] = a1.x; d[5] = a1.y; d[6] = a1.z; d[7] = a1.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) d[i] = 0.f;
    }
    if constexpr (BITS == 32) {  // identity codec (R12): the wire carries d itself
      if (act)
        for (int k = 0; k < dst.n; ++k) {
          float4* o = reinterpret_cast<float4*>(dst.p[k] + e0 * 4);
          o[0] = make_float4(d[0], d[1], d[2], d[3]);
          o[1] = make_float4(d[4], d[5], d[6], d[7]);
        }
      if constexpr (APPLY) {
        if (act) apply_own<TM>(w_model + e0, m, d);
      }
    } else {
      float a = 0.f;
#pragma unroll
      for (int i = 0; i < 8; i += 2) a = max3_abs_nan(a, d[i], d[i + 1]);
      a = group_max(a, tpg, red);
      const QP p = qparam(a, q);
      if (act) {
        uint32_t r[8];
        if (sr.on) {
#pragma unroll
          for (int i = 0; i < 8; ++i) r[i] = rq_sr(d[i], p.inv, sr_u(idx0 + e0 + i, sr.key), q);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) r[i] = rq(d[i], p.inv);
        }
        // every destination unit (all-gather push, Alg. 2 l.4): warp-contiguous stores
        if constexpr (BITS == 2) {
          uint32_t w = pack2x8(r);
          if (!p.ok) w = 0u;
          for (int k = 0; k < dst.n; ++k) *reinterpret_cast<uint16_t*>(dst.p[k] + e0 / 4) = (uint16_t)w;
        } else if constexpr (BITS == 4) {
          uint32_t w = pack4x8(r);
          if (!p.ok) w = 0u;
          for (int k = 0; k < dst.n; ++k) *reinterpret_cast<uint32_t*>(dst.p[k] + e0 / 2) = w;
        } else {
          uint2 w = make_uint2(pack8x4(r[0], r[1], r[2], r[3]), pack8x4(r[4], r[5], r[6], r[7]));
          if (!p.ok) w = make_uint2(0u, 0u);
          for (int k = 0; k < dst.n; ++k) *reinterpret_cast<uint2*>(dst.p[k] + e0) = w;
        }
        if ((t & (tpg - 1)) == 0) {
          const float sv = stored_scale(a, 1.f);
          for (int k = 0; k < dst.n; ++k) reinterpret_cast<float*>(dst.p[k] + sc_off)[e0 >> lg] = sv;
        }
        if constexpr (APPLY) {  // K2's update from the codes just packed: x = mulz(code, rn(s/q)), w += x
          // r[i] holds code + 1.5*2^23 exactly (|code| <= q when p.ok), so code = r - 1.5*2^23:
          // the value K2 decodes from the packed word; !p.ok packs zero codes
          const float ds = __fdiv_rn(stored_scale(a, 1.f), q);
          float f[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) f[i] = mulz(p.ok ? __fsub_rn(__uint_as_float(r[i]), kMagic) : 0.f, ds, z);
          apply_own<TM>(w_model + e0, m, f);
        }
      }
    }
  }
}

// =====================================================================================
// K2  qWD apply (Alg. 2 l.5): w_model[jS + e] = bf16_rn(widen(w) + code*rn(s/q))
// for every shard j (w_model shard j at w_model + j*stride), unit j read through units.p[j]:
// the gathered local copy (NCCL transport) or, with the P2P transport, rank j's own buffer
// over NVLink -- the all-gather (Alg. 2 l.4) fused into the consumer as a pull, so the
// NVLink ingress overlaps the HBM-bound replica update.  ADD = false is the qW ablation codec
// (Alg. 1): the replica becomes the dequantized weights.
// =====================================================================================
// Thread 0 streams each tile's codes and scales from the unit's buffer (local, or rank j's own
// buffer over NVLink) into a STAGES-deep shared-memory ring with 1-D bulk copies (4 KB per
// copy for 4-bit codes: large requests, many in flight), while every thread runs K1's
// 8-element layout on the replica (four rounds per 8192-element tile, the four 16-byte replica
// loads issued before the wait).  Measured faster than plain per-thread code loads both
// locally (0.94 vs 0.98 ms at P = 1) and over NVLink (0.95 vs 1.11 ms at P = 4).
constexpr int kK2rTile = 8192;
constexpr int kK2rStages = 6;
template <int BITS>
struct K2rCfg {
  static constexpr int CODE_BYTES = kK2rTile * (BITS == 32 ? 32 : BITS) / 8;
  static constexpr int SC_BYTES = BITS == 32 ? 0 : kK2rTile / 32 * 4;  // G >= 32
  static constexpr int STAGE = CODE_BYTES + SC_BYTES;
  static constexpr int SMEM = kK2rStages * STAGE + kK2rStages * 8 + 128;
};

template <typename TM, int BITS, bool ADD>
__global__ void __launch_bounds__(kVecThreads) k2_qwd_apply_ring(const Dests units, size_t S, size_t stride, int P,
                                                                    int rot, int U, int lg, TM* __restrict__ w_model,
                                                                    float z) {
  using C = K2rCfg<BITS>;
  constexpr int ROUNDS = kK2rTile / (kVecThreads * 8);
  constexpr float q = float((1 << (BITS == 32 ? 1 : BITS - 1)) - 1);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kK2rStages * C::STAGE);
  const int t = threadIdx.x;
  // U units (U = P, or P - 1 when the owner applied its own in K1), unit fastest, starting at rot
  const size_t tpu = (S + kK2rTile - 1) / kK2rTile, ntiles = tpu * U;
  const size_t sc_off = S * (BITS == 32 ? 4 : BITS) / 8;
  auto tile_of = [&](size_t tile, size_t& ts, size_t& j) {
    ts = tile / U;
    j = tile - ts * U + rot;
    if (j >= (size_t)P) j -= P;
  };
  if (t == 0) {
    for (int s = 0; s < kK2rStages; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](uint32_t k) {  // thread 0: tile k of this CTA into stage k % STAGES
    const size_t tile = blockIdx.x + (size_t)k * gridDim.x;
    if (tile >= ntiles) return;
    size_t ts, j;
    tile_of(tile, ts, j);
    const size_t e0 = ts * kK2rTile;
    const uint32_t n = (uint32_t)min((size_t)kK2rTile, S - e0);
    const uint32_t cb = n * (BITS == 32 ? 32 : BITS) / 8;
    uint32_t sb = 0;
    if constexpr (BITS != 32) sb = ((((n >> lg) * 4) + 15) & ~15u);
    const int s = k % kK2rStages;
    mbar_arrive_tx(&bar[s], cb + sb);
    const uint8_t* unit = units.p[j];
    bulk_load(smem + s * C::STAGE, unit + e0 * (BITS == 32 ? 32 : BITS) / 8, cb, &bar[s]);
    if constexpr (BITS != 32)
      bulk_load(smem + s * C::STAGE + C::CODE_BYTES, unit + sc_off + (e0 >> lg) * 4, sb, &bar[s]);
  };
  if (t == 0)
    for (int k = 0; k < kK2rStages; ++k) issue(k);
  for (uint32_t k = 0;; ++k) {
    const size_t tile = blockIdx.x + (size_t)k * gridDim.x;
    if (tile >= ntiles) break;
    size_t ts, j;
    tile_of(tile, ts, j);
    TM* wm = w_model + j * stride;
    const size_t e0 = ts * kK2rTile;
    // replica loads first (local HBM), then wait for the pulled codes
    uint4 m0[ROUNDS], m1[ROUNDS];
#pragma unroll
    for (int r = 0; r < ROUNDS; ++r) {
      const size_t e = e0 + r * (kVecThreads * 8) + t * 8;
      m0[r] = m1[r] = make_uint4(0u, 0u, 0u, 0u);
      if (ADD && e < S) {
        m0[r] = *reinterpret_cast<const uint4*>(wm + e);
        if constexpr (sizeof(TM) == 4) m1[r] = *reinterpret_cast<const uint4*>(wm + e + 4);
      }
    }
    const int s = k % kK2rStages;
    mbar_wait(&bar[s], (k / kK2rStages) & 1);
    const uint8_t* st = smem + s * C::STAGE;
#pragma unroll
    for (int r = 0; r < ROUNDS; ++r) {
      const uint32_t el = r * (kVecThreads * 8) + t * 8;  // element offset within the tile
      const size_t e = e0 + el;
      if (e >= S) continue;
      float x[8];
      if constexpr (BITS == 32) {
        const uint4 a = *reinterpret_cast<const uint4*>(st + el * 4);
        const uint4 b = *reinterpret_cast<const uint4*>(st + el * 4 + 16);
        x[0] = __uint_as_float(a.x); x[1] = __uint_as_float(a.y); x[2] = __uint_as_float(a.z); x[3] = __uint_as_float(a.w);
        x[4] = __uint_as_float(b.x); x[5] = __uint_as_float(b.y); x[6] = __uint_as_float(b.z); x[7] = __uint_as_float(b.w);
      } else {
        float f[8];
        if constexpr (BITS == 8) {
          const uint2 w = *reinterpret_cast<const uint2*>(st + el);
          dec8x4(w.x, f);
          dec8x4(w.y, f + 4);
        } else if constexpr (BITS == 4) {
          dec4x8(*reinterpret_cast<const uint32_t*>(st + el / 2), f);
        } else {
          const uint32_t w = *reinterpret_cast<const uint16_t*>(st + el / 4);
#pragma unroll
          for (int i = 0; i < 8; ++i) f[i] = float((int)(((w >> (2 * i)) & 3u) ^ 2u) - 2);
        }
        const float ds = __fdiv_rn(reinterpret_cast<const float*>(st + C::CODE_BYTES)[el >> lg], q);
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = ADD ? mulz(f[i], ds, z) : __fmul_rn(f[i], ds);  // added next: barrier
      }
      if constexpr (sizeof(TM) == 2) {
        uint32_t* w = &m0[r].x;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          w[i] = ADD ? pack_bf16x2(__fadd_rn(bf16_lo(w[i]), x[2 * i]), __fadd_rn(bf16_hi(w[i]), x[2 * i + 1]))
                     : pack_bf16x2(x[2 * i], x[2 * i + 1]);
        *reinterpret_cast<uint4*>(wm + e) = m0[r];
      } else {
        float4 a, b;
        if constexpr (ADD) {
          a = make_float4(__fadd_rn(__uint_as_float(m0[r].x), x[0]), __fadd_rn(__uint_as_float(m0[r].y), x[1]),
                          __fadd_rn(__uint_as_float(m0[r].z), x[2]), __fadd_rn(__uint_as_float(m0[r].w), x[3]));
          b = make_float4(__fadd_rn(__uint_as_float(m1[r].x), x[4]), __fadd_rn(__uint_as_float(m1[r].y), x[5]),
                          __fadd_rn(__uint_as_float(m1[r].z), x[6]), __fadd_rn(__uint_as_float(m1[r].w), x[7]));
        } else {
          a = make_float4(x[0], x[1], x[2], x[3]);
          b = make_float4(x[4], x[5], x[6], x[7]);
        }
        reinterpret_cast<float4*>(wm + e)[0] = a;
        reinterpret_cast<float4*>(wm + e + 4)[0] = b;
      }
    }
    __syncthreads();  // every thread is done with stage s
    if (t == 0) issue(k + kK2rStages);
  }
}

// =====================================================================================
// K6  one hop of the ring reduce-scatter with per-hop quantization (sec. 2.3) -- the
// ablation baseline TLq-HS is measured against.  acc = rn(dequant(recv) + g) (RECV) or g;
// then either quantize acc into the next rank's wire unit (local or peer memory; K1's
// vector layout, so a warp stores 128 contiguous code bytes) or, on the last hop,
// out = rn(acc * kappa).
// =====================================================================================
template <typename TG, int BITS, bool RECV, bool LAST>
__global__ void __launch_bounds__(kVecThreads) k6_ring_hop(const TG* __restrict__ g, const uint8_t* __restrict__ recv,
                                                               uint8_t* __restrict__ dst, float* __restrict__ out,
                                                               float kappa, size_t S, int lg, float z) {
  constexpr int TILE = kVecThreads * 8;
  __shared__ float red[kVecThreads / 32];
  constexpr float q = float((1 << (BITS == 32 ? 1 : BITS - 1)) - 1);
  const int tpg = (1 << lg) >> 3;
  const size_t ntiles = (S + TILE - 1) / TILE;
  const size_t sc_off = S * (BITS == 32 ? 4 : BITS) / 8;
  const int t = threadIdx.x;
  for (size_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const size_t e0 = tile * TILE + t * 8;
    const bool act = e0 < S;
    float a[8];
    if (act) {
      if constexpr (sizeof(TG) == 2) {
        const uint4 u = *reinterpret_cast<const uint4*>(g + e0);
        a[0] = bf16_lo(u.x); a[1] = bf16_hi(u.x); a[2] = bf16_lo(u.y); a[3] = bf16_hi(u.y);
        a[4] = bf16_lo(u.z); a[5] = bf16_hi(u.z); a[6] = bf16_lo(u.w); a[7] = bf16_hi(u.w);
      } else {
        const float4 b0 = *reinterpret_cast<const float4*>(g + e0);
        const float4 b1 = *reinterpret_cast<const float4*>(g + e0 + 4);
        a[0] = b0.x; a[1] = b0.y; a[2] = b0.z; a[3] = b0.w;
        a[4] = b1.x; a[5] = b1.y; a[6] = b1.z; a[7] = b1.w;
      }
      if constexpr (RECV) {
        float x[8];
        if constexpr (BITS == 32) {
          const float4 r0 = *reinterpret_cast<const float4*>(recv + e0 * 4);
          const float4 r1 = *reinterpret_cast<const float4*>(recv + e0 * 4 + 16);
          x[0] = r0.x; x[1] = r0.y; x[2] = r0.z; x[3] = r0.w;
          x[4] = r1.x; x[5] = r1.y; x[6] = r1.z; x[7] = r1.w;
        } else {
          const float ds = __fdiv_rn(reinterpret_cast<const float*>(recv + sc_off)[e0 >> lg], q);
          float f[8];
          if constexpr (BITS == 4) {
            dec4x8(*reinterpret_cast<const uint32_t*>(recv + e0 / 2), f);
          } else {
            const uint2 w = *reinterpret_cast<const uint2*>(recv + e0);
            dec8x4(w.x, f);
            dec8x4(w.y, f + 4);
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) x[i] = mulz(f[i], ds, z);  // added next: fusion barrier
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = __fadd_rn(x[i], a[i]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = 0.f;
    }
    if constexpr (LAST) {
      if (act) {
        float4* o = reinterpret_cast<float4*>(out + e0);
        o[0] = make_float4(__fmul_rn(a[0], kappa), __fmul_rn(a[1], kappa), __fmul_rn(a[2], kappa),
                           __fmul_rn(a[3], kappa));
        o[1] = make_float4(__fmul_rn(a[4], kappa), __fmul_rn(a[5], kappa), __fmul_rn(a[6], kappa),
                           __fmul_rn(a[7], kappa));
      }
    } else if constexpr (BITS == 32) {
      if (act) {
        float4* o = reinterpret_cast<float4*>(dst + e0 * 4);
        o[0] = make_float4(a[0], a[1], a[2], a[3]);
        o[1] = make_float4(a[4], a[5], a[6], a[7]);
      }
    } else {
      float m = 0.f;
#pragma unroll
      for (int i = 0; i < 8; i += 2) m = max3_abs_nan(m, a[i], a[i + 1]);
      m = group_max(m, tpg, red);
      const QP p = qparam(m, q);
      if (act) {
        uint32_t r[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) r[i] = rq(a[i], p.inv);
        if constexpr (BITS == 4) {
          *reinterpret_cast<uint32_t*>(dst + e0 / 2) = p.ok ? pack4x8(r) : 0u;
        } else {
          *reinterpret_cast<uint2*>(dst + e0) = p.ok ? make_uint2(pack8x4(r[0], r[1], r[2], r[3]),
                                                                  pack8x4(r[4], r[5], r[6], r[7]))
                                                     : make_uint2(0u, 0u);
        }
        if ((t & (tpg - 1)) == 0) reinterpret_cast<float*>(dst + sc_off)[e0 >> lg] = stored_scale(m, 1.f);
      }
    }
  }
}

template <int IN_R, int OUT_R>
struct K3Cfg {
  static constexpr int IN_TILE = kTileRows * IN_R;
  static constexpr int OUT_TILE = kTileRows * OUT_R + kTileElems / 32 * 4;  // codes + scales (G >= 32)
  static constexpr int BUDGET = 200 * 1024;
  static constexpr int OUTB = OUT_TILE <= 20 * 1024 ? 4 : 2;  // output tiles in flight (stores not yet read out)
  static constexpr int S0 = (BUDGET - OUTB * OUT_TILE) / IN_TILE;
  static constexpr int STAGES = S0 > 4 ? 4 : (S0 < 1 ? 1 : S0);
  static constexpr int SMEM = STAGES * IN_TILE + OUTB * OUT_TILE + 64 + 1024;
  static_assert(SMEM <= 227 * 1024, "K3 tile configuration exceeds the per-CTA shared memory");
};

// =====================================================================================
// K3  TLq-HS Hadamard + quantize (Alg. 3 l.2-3; fused per P:394-395).
// Persistent CTAs (one per SM); tile = 256 rows of 64 elements of one shard j.  Thread 0
// keeps a STAGES-deep ring of TMA tensor loads in flight (mbarrier complete_tx); every
// thread butterflies its own row in f32x2 registers, quantizes it and writes its codes and
// scales into a double-buffered linear smem tile that thread 0 bulk-stores to unit m' = j / N
// of the block for local rank l' = j % N (R9) -- with the P2P transport that block is the
// peer's receive buffer, so the store IS the intra all-to-all (Alg. 3 l.4) over NVLink.
// =====================================================================================
// Output of K3: per destination local rank l', the block this rank sends to l' (peer
// receive buffer or local send buffer); unit m' at blk + m' * unit_bytes.
struct K3Out {
  CUtensorMap map[kMaxN];   // valid for local blocks: M units of that block
  CUtensorMap omap[kMaxN];  // outbox blocks (pulled tiles, IntraPull), local memory
  uint8_t* blk[kMaxN];
  uint8_t* oblk[kMaxN];
  uint32_t remote;          // bit l': block l' lives in a peer's memory (P2P push)
  uint32_t pmask;           // bit l': some tiles for l' are pulled (IntraPull)
  uint32_t pnum, pden;
};

template <int IN_R, int BITS, int B, bool STOCH>
__global__ void __launch_bounds__(kTileRows, 1)
    k3_tlq_had_quant(const __grid_constant__ CUtensorMap in_map, const __grid_constant__ K3Out out, size_t S, int M,
                     int N, int lg, float cb, size_t unit_bytes, uint32_t tps, uint32_t ntiles, const SR sr,
                     size_t sr_stride, size_t sr_off) {
  constexpr int OUT_R = kRowElems * BITS / 8;
  using C = K3Cfg<IN_R, OUT_R>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* in_buf = smem;
  uint8_t* out_buf = smem + STAGES * C::IN_TILE;
  uint64_t* bar = reinterpret_cast<uint64_t*>(out_buf + C::OUTB * C::OUT_TILE);
  const int t = threadIdx.x;
  const uint32_t rows_per_shard = (uint32_t)(S / kRowElems);

  if (t == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](uint32_t i) {
    const uint32_t tile = blockIdx.x + i * gridDim.x;
    if (tile < ntiles) {
      const int s = i % STAGES;
      mbar_arrive_tx(&bar[s], C::IN_TILE);
      tma_load_tile<IN_R>(in_buf + s * C::IN_TILE, &in_map, &bar[s], (int)((tile / (uint32_t)(M * N)) * kTileRows),
                          (int)(tile % (uint32_t)(M * N)));
    }
  };
  if (t == 0)
    for (int i = 0; i < STAGES; ++i) issue(i);

  TileIter it((uint32_t)(M * N));
  for (uint32_t i = 0; blockIdx.x + i * gridDim.x < ntiles; ++i, it.next()) {
    const int s = i % STAGES;
    const uint32_t j = it.unit, ts = it.ts;
    const bool act = (int)(ts * kTileRows) + t < (int)rows_per_shard;
    mbar_wait(&bar[s], (i / STAGES) & 1);
    float2 p[32];
    const uint8_t* in = in_buf + s * C::IN_TILE;
#pragma unroll
    for (int c = 0; c < IN_R / 16; ++c) {
      const uint4 u = *reinterpret_cast<const uint4*>(in + tile_off<IN_R>(t, c));
      if constexpr (IN_R == 128) {  // bf16: chunk c = elements 8c..8c+7
        const int b0 = 8 * (c & 3);
        float2* d = p + b0;
        if (c < 4) {
          d[0].x = bf16_lo(u.x); d[1].x = bf16_hi(u.x); d[2].x = bf16_lo(u.y); d[3].x = bf16_hi(u.y);
          d[4].x = bf16_lo(u.z); d[5].x = bf16_hi(u.z); d[6].x = bf16_lo(u.w); d[7].x = bf16_hi(u.w);
        } else {
          d[0].y = bf16_lo(u.x); d[1].y = bf16_hi(u.x); d[2].y = bf16_lo(u.y); d[3].y = bf16_hi(u.y);
          d[4].y = bf16_lo(u.z); d[5].y = bf16_hi(u.z); d[6].y = bf16_lo(u.w); d[7].y = bf16_hi(u.w);
        }
      } else {  // fp32: chunk c = elements 4c..4c+3
        float2* d = p + 4 * (c & 7);
        if (c < 8) {
          d[0].x = __uint_as_float(u.x); d[1].x = __uint_as_float(u.y);
          d[2].x = __uint_as_float(u.z); d[3].x = __uint_as_float(u.w);
        } else {
          d[0].y = __uint_as_float(u.x); d[1].y = __uint_as_float(u.y);
          d[2].y = __uint_as_float(u.z); d[3].y = __uint_as_float(u.w);
        }
      }
    }
    if (t == 0) bulk_wait_read<C::OUTB - 1>();  // the store of tile i - OUTB has left out_buf[i % OUTB]
    __syncthreads();                  // stage s fully consumed -> refill it
    if (t == 0) issue(i + STAGES);

    fwht_pairs<B>(p);

    const uint32_t lp = j % N, mp = j / N;  // shard j = m'N + l' goes to local rank l', unit m' (R9)
    uint8_t* ot = out_buf + (i % C::OUTB) * C::OUT_TILE;
    float* osc = reinterpret_cast<float*>(ot + kTileRows * OUT_R);
    const bool pull = ((out.pmask >> lp) & 1u) && ts % out.pden < out.pnum;  // kept in the outbox
    uint8_t* unit = (pull ? out.oblk[lp] : out.blk[lp]) + mp * unit_bytes;
    const bool remote = !pull && ((out.remote >> lp) & 1u);  // CTA-uniform
    if constexpr (BITS == 32) {  // identity codec (R12): rn(u * c_b)
      const float2 cc = make_float2(cb, cb);
#pragma unroll
      for (int i2 = 0; i2 < 32; ++i2) p[i2] = f2mul(p[i2], cc);
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const float2* q = p + 4 * (c & 7);
        *reinterpret_cast<float4*>(ot + (remote ? t * 256 + 16 * c : tile_off<256>(t, c))) =
            c < 8 ? make_float4(q[0].x, q[1].x, q[2].x, q[3].x) : make_float4(q[0].y, q[1].y, q[2].y, q[3].y);
      }
    } else {
      const uint64_t i0 = (uint64_t)j * sr_stride + sr_off + ((uint64_t)ts * kTileRows + t) * kRowElems;
      if (remote) {  // peer block: linear tile, codes + scales bulk-stored over NVLink
        quant_row<BITS, OUT_R, true, STOCH>(p, t, lg, cb, act, ot, osc, sr, i0);
      } else {       // local block: swizzled tile for the TMA tensor store, scales direct
        float* gsc = reinterpret_cast<float*>(unit + S * BITS / 8) + (((size_t)ts * kTileElems) >> lg);
        quant_row<BITS, OUT_R, false, STOCH>(p, t, lg, cb, act, ot, gsc, sr, i0);
      }
    }
    fence_proxy_async();
    __syncthreads();
    if (remote) {
      const uint32_t rows = min((uint32_t)kTileRows, rows_per_shard - ts * kTileRows);
      const uint32_t nsc = BITS == 32 ? 0u : ((rows * kRowElems) >> lg);
      store_tile(ot, rows * OUT_R, osc, nsc, unit + (size_t)ts * kTileRows * OUT_R,
                 reinterpret_cast<float*>(unit + S * BITS / 8) + (((size_t)ts * kTileElems) >> lg));
      if (t == 0) bulk_commit();
    } else if (t == 0) {
      tma_store_tile<OUT_R>(pull ? &out.omap[lp] : &out.map[lp], ot, (int)(ts * kTileRows), (int)mp);
      bulk_commit();
    }
  }
  if (t == 0) bulk_wait<0>();
}

// =====================================================================================
// K4  TLq dequantize + reduce + requantize (Alg. 3 l.5, 7, 9, FP32 reduce P:344).
// Vector layout: a tile is 8192 elements of sub-block m'; thread t owns the 64 contiguous
// elements [64t, 64t+64), read from smem as 16-byte chunks in XOR-permuted order
// (slot c <- chunk c ^ f(t): conflict-free; the permutation is undone by the store
// addresses).  Thread 0 streams (tile, source l'') items through a STAGES-deep ring of 1-D
// bulk copies (codes + scales); sources are summed in order l'' = 0..N-1 (R8); the sum is
// requantized (one division per group) into a staged smem tile that thread 0 bulk-stores to
// unit m' (P2P transport: the receive slot of node m' itself -- the inter all-to-all).
// =====================================================================================
constexpr int kK4Threads = 128;
constexpr int kK4Ctas = 4;
constexpr int kK4Tile = kK4Threads * 64;

template <int BIN, int BOUT>
struct K4Cfg {
  static constexpr int CODE_BYTES = kK4Tile * BIN / 8;
  static constexpr int SC_BYTES = BIN == 32 ? 0 : kK4Tile / 32 * 4;
  static constexpr int STAGE = CODE_BYTES + SC_BYTES;
  static constexpr int OUT_TILE = kK4Tile * BOUT / 8 + kK4Tile / 32 * 4;  // staged output: codes + scales
  static constexpr int OUTB = OUT_TILE <= 8 * 1024 ? 4 : 2;  // staged remote output tiles in flight
  static constexpr int S0 = (54 * 1024 - OUTB * OUT_TILE) / STAGE;  // ~54 KB per CTA: kK4Ctas per SM
  static constexpr int STAGES = S0 > 8 ? 8 : (S0 < 1 ? 1 : S0);
  static constexpr int SMEM = STAGES * STAGE + OUTB * OUT_TILE + 64 + 128;
  static_assert(SMEM <= 227 * 1024, "K4 tile configuration exceeds the per-CTA shared memory");
  static constexpr int CPT = 64 * BIN / 8 / 16;   // 16-byte chunks per thread
  static constexpr int EPC = 64 / CPT;            // elements per chunk
};

// Producer cursor over (tile, source) items of this CTA, advanced without divisions.
struct ItemCursor {
  uint32_t l;
  TileIter it;
  __device__ explicit ItemCursor(uint32_t units) : l(0), it(units) {}
  __device__ void next(uint32_t n_src) {
    if (++l == n_src) {
      l = 0;
      it.next();
    }
  }
};

// K4 helper: decode + dequantize the thread's 64 codes of one source (slot order; chunk c holds
// elements of half ((c ^ f) * EPC) >> 5) and fold them into acc.  FIRST: acc = x (for quantized
// inputs 0 + x_0 == x_0 since a dequantized code is never -0; the identity codec keeps the add
// so that -0 becomes +0 as in R8's acc = 0; acc += x); else acc += x.
template <int BIN, int CPT, int EPC, bool FIRST>
__device__ __forceinline__ void k4_item(const uint8_t* codes, float ds0, float ds1, int f, float z, float2* acc) {
  constexpr float kDec = BIN == 8 ? kDec8 : kDec4;
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    const uint4 u = *reinterpret_cast<const uint4*>(codes + 16 * (c ^ f));
    float2* ac = acc + c * (EPC / 2);
    if constexpr (BIN == 32) {
      const float2 x0 = make_float2(__uint_as_float(u.x), __uint_as_float(u.y));
      const float2 x1 = make_float2(__uint_as_float(u.z), __uint_as_float(u.w));
      ac[0] = f2add(FIRST ? make_float2(0.f, 0.f) : ac[0], x0);
      ac[1] = f2add(FIRST ? make_float2(0.f, 0.f) : ac[1], x1);
    } else {
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
      const float2 dec = make_float2(-kDec, -kDec);
      const float d = (((c ^ f) * EPC) >> 5) ? ds1 : ds0;
      const float2 dd = make_float2(d, d);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float2 v[BIN == 8 ? 2 : 4];
        if constexpr (BIN == 8) {  // 4 codes
          const uint32_t xw = w[q] ^ 0x80808080u;
          v[0] = f2add(make_float2(__uint_as_float(__byte_perm(xw, 0x4B000000u, 0x7540)),
                                   __uint_as_float(__byte_perm(xw, 0x4B000000u, 0x7541))), dec);
          v[1] = f2add(make_float2(__uint_as_float(__byte_perm(xw, 0x4B000000u, 0x7542)),
                                   __uint_as_float(__byte_perm(xw, 0x4B000000u, 0x7543))), dec);
        } else {  // 8 codes
          const uint32_t xw = w[q] ^ 0x88888888u;
          const uint32_t lo = xw & 0x0F0F0F0Fu, hi = (xw >> 4) & 0x0F0F0F0Fu;
#pragma unroll
          for (int b = 0; b < 4; ++b)
            v[b] = f2add(make_float2(__uint_as_float(__byte_perm(lo, 0x4B000000u, 0x7540 + b)),
                                     __uint_as_float(__byte_perm(hi, 0x4B000000u, 0x7540 + b))), dec);
        }
        constexpr int NV = BIN == 8 ? 2 : 4;
#pragma unroll
        for (int b = 0; b < NV; ++b) {
          const float2 x = f2mulz(v[b], dd, z);  // rn(code * ds) (R5); added next: fusion barrier
          if constexpr (FIRST) ac[NV * q + b] = x;
          else ac[NV * q + b] = f2add(ac[NV * q + b], x);
        }
      }
    }
  }
}

struct K4Pull {  // IntraPull, K4 side: tiles of source l with ts % den < num come from src[l]
  const uint8_t* src[kMaxN];
  uint32_t mask, num, den;
};

template <int BIN, int BOUT, bool STOCH>
__global__ void __launch_bounds__(kK4Threads, kK4Ctas) k4_tlq_dq_reduce_q(const uint8_t* __restrict__ recv, size_t in_unit_bytes,
                                                          int N, int M, size_t S, int lg, const Dests dst,
                                                          uint32_t tpu, uint32_t ntiles, float z, const SR sr,
                                                          int l_self, size_t sr_stride, size_t sr_off,
                                                          const K4Pull pull) {
  using C = K4Cfg<BIN, BOUT>;
  constexpr int STAGES = C::STAGES, CPT = C::CPT, EPC = C::EPC;
  constexpr float qin = float((1 << (BIN == 32 ? 1 : BIN - 1)) - 1);
  constexpr float qout = float((1 << (BOUT == 32 ? 1 : BOUT - 1)) - 1);
  constexpr float kDec = BIN == 8 ? kDec8 : kDec4;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  uint8_t* out_buf = smem + STAGES * C::STAGE;
  uint64_t* bar = reinterpret_cast<uint64_t*>(out_buf + C::OUTB * C::OUT_TILE);
  const int t = threadIdx.x;
  if (t == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  ItemCursor pc((uint32_t)M);
  uint32_t pk = 0;
  auto issue = [&]() {  // thread 0: next item of the producer cursor into its ring slot
    if (pc.it.ts < tpu) {
      const int s = pk % STAGES;
      const size_t e0 = (size_t)pc.it.ts * kK4Tile;
      const uint32_t n = (uint32_t)min((size_t)kK4Tile, S - e0);
      // K3 tile (kTileElems) holding these elements: pulled from the source's outbox or pushed
      const bool pulled = ((pull.mask >> pc.l) & 1u) && (uint32_t)(e0 / kTileElems) % pull.den < pull.num;
      const uint8_t* unit = pulled ? pull.src[pc.l] + (size_t)pc.it.unit * in_unit_bytes
                                   : recv + ((size_t)pc.l * M + pc.it.unit) * in_unit_bytes;
      const uint32_t cb = n * BIN / 8;
      uint32_t sb = 0;
      if constexpr (BIN != 32) sb = (((n >> lg) * 4) + 15) & ~15u;
      mbar_arrive_tx(&bar[s], cb + sb);
      bulk_load(smem + s * C::STAGE, unit + e0 * BIN / 8, cb, &bar[s]);
      if constexpr (BIN != 32)
        bulk_load(smem + s * C::STAGE + C::CODE_BYTES, unit + S * BIN / 8 + (e0 >> lg) * 4, sb, &bar[s]);
    }
    ++pk;
    pc.next(N);
  };
  if (t == 0)
    for (int k = 0; k < STAGES; ++k) issue();

  // slot c of this thread holds chunk c ^ f (f = 0 for the fp32 identity path)
  const int f = BIN == 32 ? 0 : (CPT >= 8 ? (t & 7) : ((t / (8 / CPT)) & (CPT - 1)));
  const int tpg = lg >= 6 ? (1 << (lg - 6)) : 1;  // threads per group
  TileIter it((uint32_t)M);
  uint32_t k = 0;
  for (uint32_t i = 0; blockIdx.x + i * gridDim.x < ntiles; ++i, it.next()) {
    const uint32_t mp = it.unit;
    const size_t e0 = (size_t)it.ts * kK4Tile;
    const bool act = e0 + 64 * t < S;
    float2 acc[32];  // slot order: acc[i] = elements (2i, 2i+1) of the slot-ordered 64
    // one (tile, source) item: wait for its ring slot, dequantize, fold into acc (R8), release
    auto consume = [&](auto first) {
      const int s = k % STAGES;
      mbar_wait(&bar[s], (k / STAGES) & 1);
      const uint8_t* codes = smem + s * C::STAGE + t * (64 * BIN / 8);
      float ds0 = 1.f, ds1 = 1.f;
      if constexpr (BIN != 32) {
        const float* sc = reinterpret_cast<const float*>(smem + s * C::STAGE + C::CODE_BYTES);
        if (lg >= 6) {
          ds0 = ds1 = __fdiv_rn(sc[(64 * t) >> lg], qin);
        } else {
          ds0 = __fdiv_rn(sc[2 * t], qin);
          ds1 = __fdiv_rn(sc[2 * t + 1], qin);
        }
      }
      k4_item<BIN, CPT, EPC, decltype(first)::value>(codes, ds0, ds1, f, z, acc);
      __syncthreads();
      if (t == 0) issue();
      ++k;
    };
    // the first source is dequantized straight into acc (no copies); the rest are added in
    // source order l'' = 1..N-1
    consume(std::true_type{});
    for (int l = 1; l < N; ++l) consume(std::false_type{});

    // ---- requantize at BOUT bits into the staged output tile; 16-element vectors v = 0..3
    // in slot order, written at their element positions (undoing the slot permutation)
    // local destination: write global memory directly (L2 merges the partial sectors);
    // peer destination: stage the tile in smem and bulk-store it (contiguous NVLink writes)
    const bool remote = (dst.remote >> mp) & 1ull;  // CTA-uniform
    uint8_t* gout = dst.p[mp];
    uint8_t* ot = remote ? out_buf + (i % C::OUTB) * C::OUT_TILE : gout + e0 * BOUT / 8;
    float* osc = remote ? reinterpret_cast<float*>(ot + kK4Tile * BOUT / 8)
                        : reinterpret_cast<float*>(gout + S * BOUT / 8) + (e0 >> lg);
    if (remote) {
      if (t == 0) bulk_wait_read<C::OUTB - 1>();  // the stores of tile i - OUTB have left out_buf[i % OUTB]
      __syncthreads();
    }
    auto vbase = [&](int v) {  // element offset (within the thread's 64) of slot-order vector v
      if constexpr (EPC >= 16) return (((16 * v) / EPC) ^ f) * EPC + (16 * v) % EPC;
      else return 16 * v;
    };
    if constexpr (BOUT == 32) {
      if (act) {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          float4* o = reinterpret_cast<float4*>(ot + (64 * t + vbase(v)) * 4);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            o[q] = make_float4(acc[8 * v + 2 * q].x, acc[8 * v + 2 * q].y, acc[8 * v + 2 * q + 1].x,
                               acc[8 * v + 2 * q + 1].y);
        }
      }
    } else {
      float am[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        float a = 0.f;
#pragma unroll
        for (int q = 0; q < 8; ++q) a = max3_abs_nan(a, acc[8 * v + q].x, acc[8 * v + q].y);
        am[v] = a;
      }
      QP p0, p1;
      float a0, a1;
      if (lg >= 6) {
        a0 = max_nan(max_nan(am[0], am[1]), max_nan(am[2], am[3]));
#pragma unroll
        for (int off = 1; off < 32; off <<= 1)
          if (off < tpg) a0 = max_nan(a0, __shfl_xor_sync(0xffffffffu, a0, off));
        a1 = a0;
        p0 = qparam(a0, qout);
        p1 = p0;
      } else {  // G == 32: two groups per thread (element halves)
        a0 = 0.f;
        a1 = 0.f;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          if (vbase(v) >> 5) a1 = max_nan(a1, am[v]);
          else a0 = max_nan(a0, am[v]);
        }
        p0 = qparam(a0, qout);
        p1 = qparam(a1, qout);
      }
      if (act) {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const bool h = (vbase(v) >> 5) != 0;
          const float iv = h ? p1.inv : p0.inv;
          uint32_t r[16];
          const int e = 64 * t + vbase(v);
          if constexpr (STOCH) {  // global index of the shard element (mp*N + l)*S_full + off + e0 + e (R14)
            const uint64_t i0 = (uint64_t)(mp * N + l_self) * sr_stride + sr_off + e0 + e;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              r[2 * q] = rq_sr(acc[8 * v + q].x, iv, sr_u(i0 + 2 * q, sr.key), qout);
              r[2 * q + 1] = rq_sr(acc[8 * v + q].y, iv, sr_u(i0 + 2 * q + 1, sr.key), qout);
            }
          } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float2 y = f2rq(acc[8 * v + q], make_float2(iv, iv));
              r[2 * q] = __float_as_uint(y.x);
              r[2 * q + 1] = __float_as_uint(y.y);
            }
          }
          const bool okv = h ? p1.ok : p0.ok;
          if constexpr (BOUT == 4) {
            uint2 w = make_uint2(pack4x8(r), pack4x8(r + 8));
            if (!okv) w = make_uint2(0u, 0u);
            *reinterpret_cast<uint2*>(ot + e / 2) = w;
          } else {
            uint4 w = make_uint4(pack8x4(r[0], r[1], r[2], r[3]), pack8x4(r[4], r[5], r[6], r[7]),
                                 pack8x4(r[8], r[9], r[10], r[11]), pack8x4(r[12], r[13], r[14], r[15]));
            if (!okv) w = make_uint4(0u, 0u, 0u, 0u);
            *reinterpret_cast<uint4*>(ot + e) = w;
          }
        }
        if (lg >= 6) {
          if ((t & (tpg - 1)) == 0) osc[(64 * t) >> lg] = stored_scale(a0, 1.f);
        } else {
          *reinterpret_cast<float2*>(osc + 2 * t) = make_float2(stored_scale(a0, 1.f), stored_scale(a1, 1.f));
        }
      }
    }
    if (remote) {  // unit m' -> node m' (P2P: the peer's receive slot -- Alg. 3 l.10)
      fence_proxy_async();
      __syncthreads();
      const uint32_t n = (uint32_t)min((size_t)kK4Tile, S - e0);
      store_tile(ot, n * BOUT / 8, osc, BOUT == 32 ? 0u : (n >> lg), gout + e0 * BOUT / 8,
                 reinterpret_cast<float*>(gout + S * BOUT / 8) + (e0 >> lg));
      if (t == 0) bulk_commit();
    }
  }
  if (t == 0) bulk_wait<0>();
}

// =====================================================================================
// K5  TLq-HS dequantize + reduce + inverse Hadamard (Alg. 3 l.11-13; H after
// the final reduction).  Row layout; thread 0 streams (tile, source m'') items
// through a STAGES-deep ring (TMA tensor load of the codes + 1-D bulk copy of the scales);
// sources summed in order m'' = 0..M-1 (R8); out = rn(H_unnorm(acc) * kappa) (R8) is
// written into a double-buffered swizzled smem tile that thread 0 TMA-stores.
// =====================================================================================
constexpr int kK5Rows = 128;  // K5 tile rows = threads per CTA (two CTAs per SM)
constexpr int kK5Ctas = 2;

template <int IN_R>
struct K5Cfg {
  static constexpr int IN_TILE = kK5Rows * IN_R;
  static constexpr int SC_BYTES = kK5Rows * 64 / 32 * 4;  // G >= 32
  static constexpr int STAGE = IN_TILE + SC_BYTES;
  static constexpr int OUT_TILE = kK5Rows * 256;
  static constexpr int S0 = (100 * 1024 - 2 * OUT_TILE) / STAGE;
  static constexpr int STAGES = S0 > 6 ? 6 : (S0 < 1 ? 1 : S0);
  static constexpr int SMEM = STAGES * STAGE + 2 * OUT_TILE + 64 + 1024;
  static_assert(SMEM <= 227 * 1024, "K5 tile configuration exceeds the per-CTA shared memory");
};

template <int IN_R, int B>
__global__ void __launch_bounds__(kK5Rows, kK5Ctas)
    k5_tlq_dq_reduce_had(const __grid_constant__ CUtensorMap in_map, const __grid_constant__ CUtensorMap out_map,
                         const uint8_t* __restrict__ recv, size_t in_unit_bytes, int M, size_t S, int lg, float kappa,
                         uint32_t ntiles, float z) {
  constexpr int BIN = IN_R * 8 / kRowElems;
  using C = K5Cfg<IN_R>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* out_buf = smem + STAGES * C::STAGE;
  uint64_t* bar = reinterpret_cast<uint64_t*>(out_buf + 2 * C::OUT_TILE);
  const int t = threadIdx.x;
  const uint32_t rows_per_shard = (uint32_t)(S / kRowElems);
  if (t == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](uint32_t k) {
    const uint32_t i = k / M, m = k % M;
    const uint32_t tile = blockIdx.x + i * gridDim.x;
    if (tile < ntiles) {
      const int s = k % STAGES;
      uint32_t sb = 0;
      if constexpr (BIN != 32) {
        const uint32_t rows = min((uint32_t)kK5Rows, rows_per_shard - tile * kK5Rows);
        sb = (((rows * kRowElems) >> lg) * 4 + 15) & ~15u;
      }
      mbar_arrive_tx(&bar[s], C::IN_TILE + sb);
      tma_load_tile<IN_R, kK5Rows>(smem + s * C::STAGE, &in_map, &bar[s], (int)(tile * kK5Rows), (int)m);
      if constexpr (BIN != 32)
        bulk_load(smem + s * C::STAGE + C::IN_TILE,
                  recv + (size_t)m * in_unit_bytes + S * BIN / 8 + (((size_t)tile * kK5Rows * kRowElems) >> lg) * 4, sb,
                  &bar[s]);
    }
  };
  if (t == 0)
    for (int k = 0; k < STAGES; ++k) issue(k);

  constexpr float qin = float((1 << (BIN == 32 ? 1 : BIN - 1)) - 1);
  uint32_t k = 0;
  for (uint32_t i = 0;; ++i) {
    const uint32_t tile = blockIdx.x + i * gridDim.x;
    if (tile >= ntiles) break;
    float2 acc[32];
    for (int m = 0; m < M; ++m, ++k) {
      const int s = k % STAGES;
      mbar_wait(&bar[s], (k / STAGES) & 1);
      const uint8_t* st = smem + s * C::STAGE;
      float ds0 = 0.f, ds1 = 0.f;
      if constexpr (BIN != 32) {
        const float* sc = reinterpret_cast<const float*>(st + C::IN_TILE);
        if (lg >= 6) {
          ds0 = ds1 = __fdiv_rn(sc[t >> (lg - 6)], qin);
        } else {
          const float2 s2 = *reinterpret_cast<const float2*>(sc + 2 * t);
          ds0 = __fdiv_rn(s2.x, qin);
          ds1 = __fdiv_rn(s2.y, qin);
        }
      }
      float2 x[32];
      dequant_row_adj<BIN, IN_R, kK5Rows>(st, t, ds0, ds1, z, x);
      // R8 order; the first add 0 + x_0 is exact for quantized inputs (x_0 != -0).
      if (m == 0 && BIN != 32) {
#pragma unroll
        for (int q = 0; q < 32; ++q) acc[q] = x[q];
      } else {
        if (m == 0) {
#pragma unroll
          for (int q = 0; q < 32; ++q) acc[q] = make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int q = 0; q < 32; ++q) acc[q] = f2add(acc[q], x[q]);
      }
      if (t == 0 && m == M - 1) bulk_wait_read<1>();  // out_buf[i & 1] released by the store of tile i-2
      __syncthreads();
      if (t == 0) issue(k + STAGES);
    }
    fwht_adj<B>(acc);
    const float2 kk = make_float2(kappa, kappa);
#pragma unroll
    for (int q = 0; q < 32; ++q) acc[q] = f2mul(acc[q], kk);
    uint8_t* ot = out_buf + (i & 1) * C::OUT_TILE;
#pragma unroll
    for (int c = 0; c < 16; ++c)  // chunk c = elements 4c..4c+3 = pairs 2c, 2c+1
      *reinterpret_cast<float4*>(ot + tile_off<256, kK5Rows>(t, c)) =
          make_float4(acc[2 * c].x, acc[2 * c].y, acc[2 * c + 1].x, acc[2 * c + 1].y);
    fence_proxy_async();
    __syncthreads();
    if (t == 0) {
      tma_store_tile<256, kK5Rows>(&out_map, ot, (int)(tile * kK5Rows), 0);
      bulk_commit();
    }
  }
  if (t == 0) bulk_wait<0>();
}

// =====================================================================================
// P2P completion-flag wait (the sync protocol of sdp4_api.cu): one warp, lane i polls flags
// i, i + 32, ... of this rank's own symmetric buffer with system-scope acquire loads until each
// is non-zero (raised by a peer's stream memory operation after its producing kernel), then
// resets it to 0.  With a timeout, a flag still missing at the deadline writes its code into a
// host-mapped error word and the lane gives up, so a dead peer cannot hang the stream.
// =====================================================================================
__global__ void __launch_bounds__(32, 1) k_wait_flags(const FlagWait w) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = threadIdx.x; i < w.n; i += 32) {
    uint32_t* f = w.flag[i];
    for (;;) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
      if (v) break;
      if (w.timeout_ns) {
        unsigned long long now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        if (now - t0 > w.timeout_ns) {
          if (w.err) *reinterpret_cast<volatile uint32_t*>(w.err) = w.code[i];
          return;
        }
      }
      __nanosleep(32);
    }
    asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(f), "r"(0u) : "memory");
  }
}

inline int grid_for(size_t ntiles, int cap) {
  return (int)(ntiles < (size_t)cap ? (ntiles == 0 ? 1 : ntiles) : (size_t)cap);
}

template <typename K>
int occ_blocks(K kernel, int threads, size_t smem = 0) {
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, threads, smem) != cudaSuccess || nb < 1) nb = 1;
  return nb;
}

template <typename K>
cudaError_t set_smem(K kernel, int bytes) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// Tensor map over `units` units of `rows` rows of R bytes (row tiles of kTileRows rows).
cudaError_t make_row_map(CUtensorMap* map, const void* base, int R, uint64_t rows, uint64_t units,
                         uint64_t unit_stride, int box_rows = kTileRows) {
  auto fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r;
  if (R <= 128) {
    const CUtensorMapSwizzle sw =
        R == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : (R == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B);
    cuuint64_t dims[3] = {(cuuint64_t)R, rows, units};
    cuuint64_t strides[2] = {(cuuint64_t)R, unit_stride};
    cuuint32_t box[3] = {(cuuint32_t)R, (cuuint32_t)box_rows, 1};
    r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    cuuint64_t dims[4] = {128, 2, rows, units};
    cuuint64_t strides[3] = {128, (cuuint64_t)R, unit_stride};
    cuuint32_t box[4] = {128, 1, (cuuint32_t)box_rows, 1};
    r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void*>(base), dims, strides, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

#define SDP4_B_SWITCH(b, ...)                                   \
  switch (b) {                                                  \
    case 0: { constexpr int BB = 0; __VA_ARGS__; } break;       \
    case 2: { constexpr int BB = 2; __VA_ARGS__; } break;       \
    case 4: { constexpr int BB = 4; __VA_ARGS__; } break;       \
    case 8: { constexpr int BB = 8; __VA_ARGS__; } break;       \
    case 16: { constexpr int BB = 16; __VA_ARGS__; } break;     \
    case 32: { constexpr int BB = 32; __VA_ARGS__; } break;     \
    case 64: { constexpr int BB = 64; __VA_ARGS__; } break;     \
    case 128: { constexpr int BB = 128; __VA_ARGS__; } break;   \
    case 256: { constexpr int BB = 256; __VA_ARGS__; } break;   \
    default: return cudaErrorInvalidValue;                      \
  }

template <int IN_R, int BITS, int B, bool STOCH>
cudaError_t k3_launch_t(const CUtensorMap& in_map, const K3Out& out, size_t S, int M, int N, int G, float cb,
                        size_t unit_bytes, uint32_t tps, uint32_t ntiles, int grid, const SR& sr, size_t sr_stride,
                        size_t sr_off, cudaStream_t st) {
  constexpr int SMEM = K3Cfg<IN_R, kRowElems * BITS / 8>::SMEM;
  cudaError_t e = set_smem(k3_tlq_had_quant<IN_R, BITS, B, STOCH>, SMEM);
  if (e != cudaSuccess) return e;
  k3_tlq_had_quant<IN_R, BITS, B, STOCH><<<grid, kTileRows, SMEM, st>>>(in_map, out, S, M, N, __builtin_ctz(G), cb,
                                                                         unit_bytes, tps, ntiles, sr, sr_stride, sr_off);
  return cudaGetLastError();
}
template <int IN_R, int BITS, int B>
cudaError_t k3_launch(const CUtensorMap& in_map, const K3Out& out, size_t S, int M, int N, int G, float cb,
                      size_t unit_bytes, uint32_t tps, uint32_t ntiles, int grid, const SR& sr, size_t sr_stride,
                      size_t sr_off, cudaStream_t st) {
  if constexpr (BITS != 32) {
    if (sr.on)
      return k3_launch_t<IN_R, BITS, B, true>(in_map, out, S, M, N, G, cb, unit_bytes, tps, ntiles, grid, sr, sr_stride,
                                              sr_off, st);
  }
  return k3_launch_t<IN_R, BITS, B, false>(in_map, out, S, M, N, G, cb, unit_bytes, tps, ntiles, grid, sr, sr_stride,
                                           sr_off, st);
}

template <int IN_R, int B>
cudaError_t k5_launch(const CUtensorMap& in_map, const CUtensorMap& out_map, const uint8_t* recv, size_t unit_bytes,
                      int M, size_t S, int G, float kappa, uint32_t ntiles, int grid, cudaStream_t st) {
  constexpr int SMEM = K5Cfg<IN_R>::SMEM;
  cudaError_t e = set_smem(k5_tlq_dq_reduce_had<IN_R, B>, SMEM);
  if (e != cudaSuccess) return e;
  k5_tlq_dq_reduce_had<IN_R, B><<<grid, kK5Rows, SMEM, st>>>(in_map, out_map, recv, unit_bytes, M, S, __builtin_ctz(G), kappa,
                                                                ntiles, -0.0f);
  return cudaGetLastError();
}

template <int BIN, int BOUT, bool STOCH>
cudaError_t k4_launch_t(const uint8_t* recv, size_t in_unit_bytes, int N, int M, size_t S, int G, const Dests& dst,
                        const SR& sr, int l_self, size_t sr_stride, size_t sr_off, int sms, cudaStream_t st,
                        const K4Pull& pull) {
  constexpr int SMEM = K4Cfg<BIN, BOUT>::SMEM;
  cudaError_t e = set_smem(k4_tlq_dq_reduce_q<BIN, BOUT, STOCH>, SMEM);
  if (e != cudaSuccess) return e;
  const uint32_t tpu = (uint32_t)((S + kK4Tile - 1) / kK4Tile);
  const uint32_t ntiles = tpu * (uint32_t)M;
  const int grid = grid_for(ntiles, sms * kK4Ctas);
  k4_tlq_dq_reduce_q<BIN, BOUT, STOCH><<<grid, kK4Threads, SMEM, st>>>(recv, in_unit_bytes, N, M, S, __builtin_ctz(G),
                                                                dst, tpu, ntiles, -0.0f, sr, l_self, sr_stride, sr_off,
                                                                pull);
  return cudaGetLastError();
}
template <int BIN, int BOUT>
cudaError_t k4_launch(const uint8_t* recv, size_t in_unit_bytes, int N, int M, size_t S, int G, const Dests& dst,
                      const SR& sr, int l_self, size_t sr_stride, size_t sr_off, int sms, cudaStream_t st,
                      const K4Pull& pull) {
  if constexpr (BOUT != 32) {
    if (sr.on)
      return k4_launch_t<BIN, BOUT, true>(recv, in_unit_bytes, N, M, S, G, dst, sr, l_self, sr_stride, sr_off, sms, st,
                                          pull);
  }
  return k4_launch_t<BIN, BOUT, false>(recv, in_unit_bytes, N, M, S, G, dst, sr, l_self, sr_stride, sr_off, sms, st,
                                       pull);
}

}  // namespace

// ------------------------------- launchers -------------------------------------------
cudaError_t launch_qwd_quantize(const float* w_main, const void* w_model_shard, int model_dtype,
                                size_t S, int bits, int G, const Dests& dst, int sr_on, uint32_t sr_key,
                                uint64_t idx0, int sms, cudaStream_t st, bool apply_own) {
  const SR sr{sr_on, sr_key};
  if (apply_own && !w_model_shard) return cudaErrorInvalidValue;
  void* wm = const_cast<void*>(w_model_shard);  // written only by the APPLY variants
  const size_t ntiles = (S + kVecThreads * 8 - 1) / (kVecThreads * 8);
  // persistent grid: as many CTAs per SM as the variant's registers allow (at most kVecCtas)
#define K1(TM, B, DF, AP)                                                                                    \
  do {                                                                                                       \
    static const int nb = std::min(kVecCtas, occ_blocks(k1_qwd_quantize<TM, B, DF, AP>, kVecThreads));      \
    k1_qwd_quantize<TM, B, DF, AP><<<grid_for(ntiles, sms * nb), kVecThreads, 0, st>>>(                      \
        w_main, static_cast<TM*>(wm), S, __builtin_ctz(G), dst, sr, idx0, -0.0f);                            \
  } while (0)
#define K1B(TM, DF, AP)                 \
  if (bits == 2) K1(TM, 2, DF, AP);     \
  else if (bits == 4) K1(TM, 4, DF, AP); \
  else if (bits == 8) K1(TM, 8, DF, AP); \
  else K1(TM, 32, DF, AP)
  if (!w_model_shard) {
    K1B(float, false, false);
  } else if (model_dtype == kBF16) {
    if (apply_own) { K1B(uint16_t, true, true); } else { K1B(uint16_t, true, false); }
  } else {
    if (apply_own) { K1B(float, true, true); } else { K1B(float, true, false); }
  }
#undef K1B
#undef K1
  return cudaGetLastError();
}

cudaError_t launch_qwd_apply(const Dests& units, int P, size_t S, size_t stride, int bits, int G, void* w_model,
                             int model_dtype, bool add, int sms, cudaStream_t st, int rot, bool skip_rot) {
  const int U = skip_rot ? P - 1 : P;  // skip_rot: unit `rot` was applied by its owner's K1
  if (skip_rot) rot = (rot + 1) % P;
  if (U <= 0 || S == 0) return cudaSuccess;
  const int grid_r = grid_for((S + kK2rTile - 1) / kK2rTile * U, sms * 4);
#define K2(TM, B, AD)                                                                          \
  do {                                                                                                 \
    set_smem(k2_qwd_apply_ring<TM, B, AD>, K2rCfg<B>::SMEM);                                           \
    k2_qwd_apply_ring<TM, B, AD><<<grid_r, kVecThreads, K2rCfg<B>::SMEM, st>>>(                         \
        units, S, stride, P, rot % P, U, __builtin_ctz(G), static_cast<TM*>(w_model), -0.0f);          \
  } while (0)
#define K2B(TM, AD) \
  if (bits == 2) K2(TM, 2, AD); else if (bits == 4) K2(TM, 4, AD); else if (bits == 8) K2(TM, 8, AD); else K2(TM, 32, AD)
  if (model_dtype == kBF16) {
    if (add) { K2B(uint16_t, true); } else { K2B(uint16_t, false); }
  } else {
    if (add) { K2B(float, true); } else { K2B(float, false); }
  }
#undef K2B
#undef K2
  return cudaGetLastError();
}

cudaError_t launch_ring_hop(const void* grad_chunk, int grad_dtype, const uint8_t* recv, uint8_t* dst, float* out,
                            float kappa, size_t S, int bits, int G, int sms, cudaStream_t st) {
  const int grid = grid_for((S + kVecThreads * 8 - 1) / (kVecThreads * 8), sms * kVecCtas);
#define K6(TG, B, RV, LS)                                                                                 \
  k6_ring_hop<TG, B, RV, LS><<<grid, kVecThreads, 0, st>>>(static_cast<const TG*>(grad_chunk), recv, dst, out, \
                                                           kappa, S, __builtin_ctz(G), -0.0f)
#define K6B(TG, RV, LS) \
  if (bits == 4) K6(TG, 4, RV, LS); else if (bits == 8) K6(TG, 8, RV, LS); else K6(TG, 32, RV, LS)
#define K6T(TG)                                                         \
  if (recv) {                                                           \
    if (dst) { K6B(TG, true, false); } else { K6B(TG, true, true); }    \
  } else {                                                              \
    if (dst) { K6B(TG, false, false); } else { K6B(TG, false, true); }  \
  }
  if (grad_dtype == kBF16) {
    K6T(uint16_t)
  } else {
    K6T(float)
  }
#undef K6T
#undef K6B
#undef K6
  return cudaGetLastError();
}

cudaError_t launch_tlq_had_quant(const void* grad, size_t grad_stride, int grad_dtype, size_t S, int M, int N,
                                 int G, int b, float cb, int bits, uint8_t* const* blocks, uint32_t remote_mask,
                                 size_t unit_bytes, int sr_on, uint32_t sr_key, size_t sr_off, int sms,
                                 cudaStream_t st, const IntraPull* pull) {
  const SR sr{sr_on, sr_key};
  if (N > kMaxN) return cudaErrorInvalidValue;
  const uint64_t rows = S / kRowElems;
  const uint32_t tps = (uint32_t)((rows + kTileRows - 1) / kTileRows);
  const uint32_t ntiles = tps * (uint32_t)(M * N);
  const int grid = grid_for(ntiles, sms);
  const int in_r = grad_dtype == kBF16 ? 128 : 256;
  const int out_r = kRowElems * bits / 8;
  CUtensorMap in_map;
  K3Out out;
  memset(&out, 0, sizeof(out));
  cudaError_t e = make_row_map(&in_map, grad, in_r, rows, (uint64_t)M * N, (uint64_t)grad_stride * (in_r / kRowElems));
  if (e != cudaSuccess) return e;
  out.remote = remote_mask;
  out.pmask = pull && pull->num > 0 ? pull->mask : 0u;
  out.pnum = pull ? (uint32_t)pull->num : 0u;
  out.pden = pull && pull->den > 0 ? (uint32_t)pull->den : 1u;
  for (int lp = 0; lp < N; ++lp) {
    out.blk[lp] = blocks[lp];
    if (!((remote_mask >> lp) & 1u)) {
      e = make_row_map(&out.map[lp], blocks[lp], out_r, rows, (uint64_t)M, unit_bytes);
      if (e != cudaSuccess) return e;
    }
    if ((out.pmask >> lp) & 1u) {
      out.oblk[lp] = pull->outbox[lp];
      e = make_row_map(&out.omap[lp], pull->outbox[lp], out_r, rows, (uint64_t)M, unit_bytes);
      if (e != cudaSuccess) return e;
    }
  }
#define K3(IR, BT) SDP4_B_SWITCH(b, return (k3_launch<IR, BT, BB>(in_map, out, S, M, N, G, cb, unit_bytes, tps, ntiles, \
                                                                  grid, sr, grad_stride, sr_off, st)))
  if (in_r == 128) {
    if (bits == 4) { K3(128, 4); } else if (bits == 8) { K3(128, 8); } else { K3(128, 32); }
  } else {
    if (bits == 4) { K3(256, 4); } else if (bits == 8) { K3(256, 8); } else { K3(256, 32); }
  }
#undef K3
  return cudaErrorInvalidValue;
}

cudaError_t launch_tlq_dq_reduce_q(const uint8_t* intra_recv, size_t in_unit_bytes, int bits_in,
                                   int N, int M, size_t S, int G, const Dests& dst, int bits_out, int sr_on,
                                   uint32_t sr_key, int l_self, size_t sr_stride, size_t sr_off, int sms,
                                   cudaStream_t st, const IntraPull* pull) {
  if (M > kMaxDests || N > kMaxN) return cudaErrorInvalidValue;
  const SR sr{sr_on, sr_key};
  K4Pull kp;
  memset(&kp, 0, sizeof(kp));
  kp.den = 1;
  if (pull && pull->num > 0) {
    kp.mask = pull->mask;
    kp.num = (uint32_t)pull->num;
    kp.den = (uint32_t)pull->den;
    for (int l = 0; l < N; ++l) kp.src[l] = pull->src[l];
  }
#define K4(BI, BO) return k4_launch<BI, BO>(intra_recv, in_unit_bytes, N, M, S, G, dst, sr, l_self, sr_stride, sr_off, \
                                            sms, st, kp)
#define K4O(BI) \
  if (bits_out == 4) { K4(BI, 4); } else if (bits_out == 8) { K4(BI, 8); } else { K4(BI, 32); }
  if (bits_in == 4) { K4O(4); } else if (bits_in == 8) { K4O(8); } else { K4O(32); }
#undef K4O
#undef K4
}

cudaError_t launch_tlq_dq_reduce_had(const uint8_t* inter_recv, size_t in_unit_bytes, int bits_in,
                                     int M, size_t S, int G, int b, float kappa, float* out,
                                     int sms, cudaStream_t st) {
  const uint64_t rows = S / kRowElems;
  const uint32_t ntiles = (uint32_t)((rows + kK5Rows - 1) / kK5Rows);
  const int grid = grid_for(ntiles, sms * kK5Ctas);
  const int in_r = kRowElems * bits_in / 8;
  CUtensorMap in_map, out_map;
  cudaError_t e = make_row_map(&in_map, inter_recv, in_r, rows, (uint64_t)M, in_unit_bytes, kK5Rows);
  if (e != cudaSuccess) return e;
  e = make_row_map(&out_map, out, 256, rows, 1, (uint64_t)S * 4, kK5Rows);
  if (e != cudaSuccess) return e;
#define K5(IR) SDP4_B_SWITCH(b, return (k5_launch<IR, BB>(in_map, out_map, inter_recv, in_unit_bytes, M, S, G, \
                                                          kappa, ntiles, grid, st)))
  if (in_r == 32) { K5(32); } else if (in_r == 64) { K5(64); } else { K5(256); }
#undef K5
  return cudaErrorInvalidValue;
}

cudaError_t launch_wait_flags(const FlagWait& w, cudaStream_t st) {
  if (w.n <= 0) return cudaSuccess;
  if (w.n > kMaxWait) return cudaErrorInvalidValue;
  k_wait_flags<<<1, 32, 0, st>>>(w);
  return cudaGetLastError();
}

}  // namespace sdp4
