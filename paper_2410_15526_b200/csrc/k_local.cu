// k_local.cu -- TLq-HS at world size 1 as ONE kernel: K3 -> K4 -> K5 fused (Alg. 3 with
// M = N = 1).  With one rank both all-to-alls are the identity, so the 8-bit codes
// K3 would write, K4 read back, requantize to 4 bits and write, and K5 read back never need to
// leave the registers: a row is loaded once (2 or 4 B per element) and the fp32 output written
// once (4 B), 6 B per element instead of K3 + K4 + K5's 9.1 (bf16 gradients).  Every
// quantize / dequantize / reduce / butterfly is the same operation, in the same order, on the
// same element as in the three kernels (and the oracle), so the output is bit-identical.
#include "sdp4_device.cuh"

namespace sdp4 {
namespace {

constexpr int kLBlock = kTileRows + 32;  // 256 consumer threads (one row each) + producer warp
constexpr int kLChunk = 2;               // tiles per scheduler claim
constexpr uint32_t kLNoTile = 0xffffffffu;

template <int IN_R>
struct LCfg {
  static constexpr int IN_TILE = kTileRows * IN_R;
  static constexpr int OUT_WARP = 32 * 256;                        // a warp's 32 fp32 rows
  static constexpr int OUT_BYTES = (kTileRows / 32) * OUT_WARP;    // one transpose tile per warp
  static constexpr int S0 = (200 * 1024 - OUT_BYTES) / IN_TILE;
  static constexpr int STAGES = S0 > 4 ? 4 : (S0 < 2 ? 2 : S0);
  static constexpr int SMEM = STAGES * IN_TILE + OUT_BYTES + 2 * 8 * STAGES + 4 * STAGES + 1024;
  static_assert(SMEM <= 227 * 1024, "local TLq-HS tile configuration exceeds the per-CTA shared memory");
};

// Quantize a row held as pairs p[i] = {v[i], v[i+32]} at BITS (quant_row's arithmetic: group
// max, qparam, RNE or stochastic codes, stored scale rn(s * c)) and replace it by what the
// consumer of the wire unit decodes: code * div_by_q(stored scale, q) (K4's / K5's
// dequantization; zero codes for groups that are not ok).  i0: stochastic index of element 0.
//
// `known` (the 4-bit step after the 8-bit one, nearest rounding, every group of the warp ok at
// 8 bits): the group max is rn(127 * d8) without a pass over the row -- the 8-bit code of the
// max element is +-127 and |rn(c8 * d8)| is monotone in |c8| (K34's argument, k_local34.cu,
// DESIGN.md sec. 7).
struct DQR {
  float d0, d1;
  bool ok;
};
template <int BITS, bool STOCH>
__device__ __forceinline__ DQR quant_dequant_row(float2* p, int t, int lg, float c, const SR& sr, uint64_t i0,
                                                 float z, const DQR* known = nullptr) {
  constexpr float q = float((1 << (BITS - 1)) - 1);
  const float rq_ = __fdiv_rn(1.f, q);
  float a0 = 0.f, a1 = 0.f;
  const bool kn = !STOCH && known && __all_sync(0xffffffffu, known->ok);
  if (kn) {
    a0 = __fmul_rn(127.f, known->d0);
    a1 = __fmul_rn(127.f, known->d1);
  } else {
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      a0 = max3_abs_nan(a0, p[i].x, p[i + 1].x);
      a1 = max3_abs_nan(a1, p[i].y, p[i + 1].y);
    }
  }
  QP p0, p1;
  if (lg >= 6) {  // a group spans G/64 rows (lanes)
    if (!kn) {
      a0 = max_nan(a0, a1);
      const int rpg = 1 << (lg - 6);
      for (int off = 1; off < rpg; off <<= 1) a0 = max_nan(a0, __shfl_xor_sync(0xffffffffu, a0, off));
    }
    a1 = a0;
    p0 = qparam(a0, q);
    p1 = p0;
  } else {  // G == 32: two groups per row (element halves)
    p0 = qparam(a0, q);
    p1 = qparam(a1, q);
  }
  const float d0 = div_by_q(stored_scale(a0, c), q, rq_), d1 = div_by_q(stored_scale(a1, c), q, rq_);
  const float2 inv = make_float2(p0.inv, p1.inv);
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    float2 y;
    if constexpr (STOCH) {
      y.x = __uint_as_float(rq_sr(p[i].x, inv.x, sr_u(i0 + i, sr.key), q));
      y.y = __uint_as_float(rq_sr(p[i].y, inv.y, sr_u(i0 + 32 + i, sr.key), q));
    } else {
      y = f2rq(p[i], inv);
    }
    // the code value (exact: magic bits minus the magic constant), zero for a group that is
    // not ok; then rn(code * ds) as K4 / K5 decode it
    const float2 cv = f2add(y, make_float2(-kMagic, -kMagic));
    if constexpr (STOCH) {
      p[i] = f2mulz(make_float2(p0.ok ? cv.x : 0.f, p1.ok ? cv.y : 0.f), make_float2(d0, d1), z);
    } else {
      // no select needed: a group that is not ok has inv = 0, so cv is +0 for finite
      // elements and NaN for non-finite ones -- and such a group's d is 0 (tiny) or
      // non-finite (NaN / Inf max), where code 0 * d gives the same +0 / NaN
      p[i] = f2mulz(cv, make_float2(d0, d1), z);
    }
  }
  return DQR{d0, d1, p0.ok && p1.ok};
}

template <int IN_R, int B, bool STOCH>
__global__ void __launch_bounds__(kLBlock, 1)
    k_tlq_local(const __grid_constant__ CUtensorMap in_map, size_t S, int lg, float cb, float kappa, uint32_t ntiles,
                const SR sr8, const SR sr4, float z, float* __restrict__ out, uint32_t* sched) {
  using C = LCfg<IN_R>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* in_buf = smem;
  uint8_t* out_buf = smem + STAGES * C::IN_TILE;
  uint64_t* full = reinterpret_cast<uint64_t*>(out_buf + C::OUT_BYTES);
  uint64_t* empty = full + STAGES;
  uint32_t* tile_of = reinterpret_cast<uint32_t*>(empty + STAGES);
  const int t = threadIdx.x;
  const uint32_t rows_per_shard = (uint32_t)(S / kRowElems);
  if (t == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTileRows / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();  // the only CTA-wide barrier
  if (t >= kTileRows) {  // ---- producer warp (K3's)
    if (t == kTileRows) {
      uint32_t k = 0;
      for (;;) {
        const uint32_t t0 = sched_claim(sched, kLChunk);
        if (t0 >= ntiles) break;
        const uint32_t t1 = min(t0 + kLChunk, ntiles);
        for (uint32_t tile = t0; tile < t1; ++tile, ++k) {
          const int s = k % STAGES;
          mbar_wait(&empty[s], ((k / STAGES) & 1) ^ 1);
          tile_of[s] = tile;
          mbar_arrive_tx(&full[s], C::IN_TILE);
          tma_load_tile<IN_R>(in_buf + s * C::IN_TILE, &in_map, &full[s], (int)(tile * kTileRows), 0);
        }
      }
      const int s = k % STAGES;
      mbar_wait(&empty[s], ((k / STAGES) & 1) ^ 1);
      tile_of[s] = kLNoTile;
      mbar_arrive(&full[s]);
      sched_done(sched);
    }
    return;
  }
  const int lane = t & 31, warp = t >> 5;
  uint8_t* ob = out_buf + warp * C::OUT_WARP;  // this warp's transpose tile
  for (uint32_t i = 0;; ++i) {
    const int s = i % STAGES;
    mbar_wait(&full[s], (i / STAGES) & 1);
    const uint32_t tile = tile_of[s];
    if (tile == kLNoTile) break;
    const uint32_t row = tile * kTileRows + t;
    const bool act = row < rows_per_shard;
    float2 p[32];
    const uint8_t* in = in_buf + s * C::IN_TILE;
#pragma unroll
    for (int c = 0; c < IN_R / 16; ++c) {  // K3's row load
      const uint4 u = *reinterpret_cast<const uint4*>(in + tile_off<IN_R>(t, c));
      if constexpr (IN_R == 128) {
        const int b0 = 8 * (c & 3);
        float2* d = p + b0;
        if (c < 4) {
          d[0].x = bf16_lo(u.x); d[1].x = bf16_hi(u.x); d[2].x = bf16_lo(u.y); d[3].x = bf16_hi(u.y);
          d[4].x = bf16_lo(u.z); d[5].x = bf16_hi(u.z); d[6].x = bf16_lo(u.w); d[7].x = bf16_hi(u.w);
        } else {
          d[0].y = bf16_lo(u.x); d[1].y = bf16_hi(u.x); d[2].y = bf16_lo(u.y); d[3].y = bf16_hi(u.y);
          d[4].y = bf16_lo(u.z); d[5].y = bf16_hi(u.z); d[6].y = bf16_lo(u.w); d[7].y = bf16_hi(u.w);
        }
      } else {
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
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // this warp's rows of stage s are in registers
    if (!act) {
#pragma unroll
      for (int k = 0; k < 32; ++k) p[k] = make_float2(0.f, 0.f);
    }
    const uint64_t i0 = (uint64_t)row * kRowElems;  // stochastic index of the row (shard 0 = the buffer)
    fwht_pairs<B>(p);                                           // K3: H (unnormalized)
    const DQR r8 = quant_dequant_row<8, STOCH>(p, t, lg, cb, sr8, i0, z);  // K3: Q8 (scale * c_b); K4: DQ8 (N = 1)
    quant_dequant_row<4, STOCH>(p, t, lg, 1.f, sr4, i0, z, &r8);            // K4: Q4; K5: DQ4 (M = 1)
    fwht_pairs<B>(p);                                           // K5: H after the reduction
    const float2 kk = make_float2(kappa, kappa);
#pragma unroll
    for (int k = 0; k < 32; ++k) p[k] = f2mul(p[k], kk);
    // K5's epilogue: transpose through the warp's smem tile, coalesced 16-byte stores
    // (the warp's 32 rows are 8 KB of contiguous output); pairs hold {v[k], v[k+32]}
#pragma unroll
    for (int c = 0; c < 16; ++c) {  // chunk c = elements 4c..4c+3
      const float2* q = p + 4 * (c & 7);
      *reinterpret_cast<float4*>(ob + tile_off<256, 32>(lane, c)) =
          c < 8 ? make_float4(q[0].x, q[1].x, q[2].x, q[3].x) : make_float4(q[0].y, q[1].y, q[2].y, q[3].y);
    }
    __syncwarp();
    const uint32_t row0 = tile * kTileRows + warp * 32;
    const uint32_t nrow = row0 < rows_per_shard ? min(32u, rows_per_shard - row0) : 0u;
    float* gout = out + (size_t)row0 * kRowElems;
#pragma unroll
    for (int j = 0; j < 16; ++j) {  // store j: bytes [512 j, 512 j + 512) of the warp's rows
      const int r = 2 * j + (lane >> 4), c = lane & 15;
      const float4 v = *reinterpret_cast<const float4*>(ob + tile_off<256, 32>(r, c));
      if ((uint32_t)r < nrow) *reinterpret_cast<float4*>(gout + r * kRowElems + 4 * c) = v;
    }
    __syncwarp();  // ob is rewritten by the next tile
  }
}

template <int IN_R, int B>
cudaError_t local_launch(const CUtensorMap& in_map, size_t S, int G, float cb, float kappa, uint32_t ntiles,
                         const SR& sr8, const SR& sr4, float* out, int sms, cudaStream_t st) {
  constexpr int SMEM = LCfg<IN_R>::SMEM;
  uint32_t* sched = sched_counter(st);
  if (!sched) return cudaErrorMemoryAllocation;
  const int grid = grid_for(ntiles, sms);
  cudaError_t e;
  if (sr8.on) {
    if ((e = set_smem(k_tlq_local<IN_R, B, true>, SMEM)) != cudaSuccess) return e;
    k_tlq_local<IN_R, B, true><<<grid, kLBlock, SMEM, st>>>(in_map, S, __builtin_ctz(G), cb, kappa, ntiles, sr8, sr4,
                                                            -0.0f, out, sched);
  } else {
    if ((e = set_smem(k_tlq_local<IN_R, B, false>, SMEM)) != cudaSuccess) return e;
    k_tlq_local<IN_R, B, false><<<grid, kLBlock, SMEM, st>>>(in_map, S, __builtin_ctz(G), cb, kappa, ntiles, sr8, sr4,
                                                             -0.0f, out, sched);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_tlq_local(const void* grad, int grad_dtype, size_t S, int G, int b, float cb, float kappa,
                             int sr_on, uint32_t key8, uint32_t key4, float* out, int sms, cudaStream_t st) {
  const uint64_t rows = S / kRowElems;
  const uint32_t ntiles = (uint32_t)((rows + kTileRows - 1) / kTileRows);
  const int in_r = grad_dtype == kBF16 ? 128 : 256;
  CUtensorMap in_map;
  cudaError_t e = make_row_map(&in_map, grad, in_r, rows, 1, (uint64_t)S * (in_r / kRowElems));
  if (e != cudaSuccess) return e;
  const SR sr8{sr_on, key8}, sr4{sr_on, key4};
#define KL(IR) SDP4_B_SWITCH(b, return (local_launch<IR, BB>(in_map, S, G, cb, kappa, ntiles, sr8, sr4, out, sms, st)))
  if (in_r == 128) {
    KL(128);
  } else {
    KL(256);
  }
#undef KL
  return cudaErrorInvalidValue;
}

}  // namespace sdp4
