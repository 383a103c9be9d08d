// k_local34.cu -- TLq-HS with one GPU per group (N = 1, M > 1): K3 and K4 fused (Alg. 3 l.2-9,
// P:368-375).  With N = 1 the intra all-to-all (l.4) is the identity and K4 reduces a single
// source, so the 8-bit codes K3 would write and K4 read back stay in registers: a row is
// loaded once, butterflied, quantized to 8 bits and dequantized (K4's decode of the one
// source), requantized to 4 bits, and the 4-bit unit of shard j = m' goes straight to slot m
// of node m''s inter receive region -- a peer's over NVLink (the inter all-to-all, l.10) or
// this rank's own.  Same operations, same order, same elements as K3 + K4: bit-identical.
#include "sdp4_device.cuh"

namespace sdp4 {
namespace {

constexpr int kQBlock = kTileRows + 32;  // 256 consumer threads (one row each) + producer warp
constexpr int kQChunk = 2;
constexpr uint32_t kQNoTile = 0xffffffffu;
constexpr int kQOutR = kRowElems * 4 / 8;  // 32 bytes of 4-bit codes per row

template <int IN_R>
struct QCfg {
  static constexpr int CTAS = IN_R == 128 ? 2 : 1;  // bf16 gradients: two CTAs per SM (K3's)
  static constexpr int IN_TILE = kTileRows * IN_R;
  static constexpr int OUT_W = (32 * kQOutR + 256 + 1023) / 1024 * 1024;  // a warp's codes + scales
  static constexpr int OB = 2;                                              // output tiles per warp
  static constexpr int OUT_BYTES = OB * (kTileRows / 32) * OUT_W;
  static constexpr int BUDGET = CTAS == 2 ? 110 * 1024 : 200 * 1024;
  static constexpr int S0 = (BUDGET - OUT_BYTES) / IN_TILE;
  static constexpr int STAGES = S0 > 4 ? 4 : (S0 < 2 ? 2 : S0);
  static constexpr int SMEM = STAGES * IN_TILE + OUT_BYTES + 2 * 8 * STAGES + 4 * STAGES + 1024;
  static_assert(SMEM <= 227 * 1024, "K34 tile configuration exceeds the per-CTA shared memory");
};

struct Q4Out {
  uint8_t* unit[kMaxDests];  // unit m' (shard j = m'): slot m of node m''s inter receive region
  uint64_t remote;           // bit m': peer memory
};

// The 8-bit step's dequantization steps d and whether both of the row's groups are ok.
struct DQ8 {
  float d0, d1;
  bool ok;
};

// quant_dequant_row (k_local.cu): the row quantized at BITS and replaced by its dequantization
template <int BITS, bool STOCH>
__device__ __forceinline__ DQ8 quant_dequant_row34(float2* p, int lg, float c, const SR& sr, uint64_t i0, float z) {
  constexpr float q = float((1 << (BITS - 1)) - 1);
  const float rq_ = __fdiv_rn(1.f, q);
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
    a1 = a0;
    p0 = qparam(a0, q);
    p1 = p0;
  } else {
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
  return DQ8{d0, d1, p0.ok && p1.ok};
}

// K4's 4-bit requantization of a row held as pairs (quant_row<4>'s arithmetic: group max,
// qparam, RNE / stochastic codes, stored scale rn(s * 1)) with K4's packing: biased magic
// bits (kMagicB4) and pack4x8_b (4 ALU instructions per 8 codes instead of pack4x8's 11).
// Codes of the row at out_tile + t * 32 (linear), scales as quant_row places them.
//
// The 4-bit group is the 8-bit group (one G), so when that group was ok its max |x| is known
// without a pass over the row: the element of max |u| got code +-127 (|u| * rn(127/|u|) =
// 127 (1 + d), |d| <= 2^-24, rounds to 127), every |x| = rn(|code| * d8) is monotone in |code|,
// so max |x| = rn(127 * d8) -- bit for bit the max the pass would find.  Nearest rounding
// only (a stochastic code of the max element can be 126); a warp with any group not ok (zero,
// tiny, Inf, NaN: the ragged tail or edge groups) takes the pass.
template <bool STOCH>
__device__ __forceinline__ void quant_row4_b(const float2* p, int t, int lg, bool act, uint8_t* out_tile,
                                             float* scales_tile, const SR& sr, uint64_t i0, uint32_t m16,
                                             const DQ8& r8) {
  constexpr float q = 7.f;
  float a0 = 0.f, a1 = 0.f;
  const bool known = !STOCH && __all_sync(0xffffffffu, r8.ok);
  if (known) {
    a0 = __fmul_rn(127.f, r8.d0);
    a1 = __fmul_rn(127.f, r8.d1);
  } else {
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      a0 = max3_abs_nan(a0, p[i].x, p[i + 1].x);
      a1 = max3_abs_nan(a1, p[i].y, p[i + 1].y);
    }
  }
  QP p0, p1;
  if (lg >= 6) {
    const int rpg = 1 << (lg - 6);
    if (!known) {
      a0 = max_nan(a0, a1);
      for (int off = 1; off < rpg; off <<= 1) a0 = max_nan(a0, __shfl_xor_sync(0xffffffffu, a0, off));
    }
    p0 = qparam(a0, q);
    p1 = p0;
    if (act && (t & (rpg - 1)) == 0) scales_tile[t >> (lg - 6)] = stored_scale(a0, 1.f);
  } else {
    p0 = qparam(a0, q);
    p1 = qparam(a1, q);
    if (act) *reinterpret_cast<float2*>(scales_tile + 2 * t) = make_float2(stored_scale(a0, 1.f), stored_scale(a1, 1.f));
  }
  const float2 inv = make_float2(p0.inv, p1.inv);
  uint32_t rx[32], ry[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    if constexpr (STOCH) {
      rx[i] = rq_sr(p[i].x, inv.x, sr_u(i0 + i, sr.key), q, kMagicB4);
      ry[i] = rq_sr(p[i].y, inv.y, sr_u(i0 + 32 + i, sr.key), q, kMagicB4);
    } else {
      const float2 y = f2rq(p[i], inv, kMagicB4);
      rx[i] = __float_as_uint(y.x);
      ry[i] = __float_as_uint(y.y);
    }
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const uint32_t* r = k == 0 ? rx : ry;
    uint4 w = make_uint4(pack4x8_b(r, m16), pack4x8_b(r + 8, m16), pack4x8_b(r + 16, m16), pack4x8_b(r + 24, m16));
    if (!(k == 0 ? p0.ok : p1.ok)) w = make_uint4(0u, 0u, 0u, 0u);
    *reinterpret_cast<uint4*>(out_tile + t * 32 + 16 * k) = w;
  }
}

template <int IN_R, int B, bool STOCH>
__global__ void __launch_bounds__(kQBlock, QCfg<IN_R>::CTAS)
    k_tlq_q84(const __grid_constant__ CUtensorMap in_map, const __grid_constant__ Q4Out out, size_t S, int M, int lg,
              float cb, uint32_t ntiles, const SR sr8, const SR sr4, float z, uint32_t m16, uint32_t* sched) {
  using C = QCfg<IN_R>;
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
  const uint32_t U = (uint32_t)M;  // shards; tile = ts * U + j (shard fastest, K3's order)
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
        const uint32_t t0 = sched_claim(sched, kQChunk);
        if (t0 >= ntiles) break;
        const uint32_t t1 = min(t0 + kQChunk, ntiles);
        for (uint32_t tile = t0; tile < t1; ++tile, ++k) {
          const int s = k % STAGES;
          mbar_wait(&empty[s], ((k / STAGES) & 1) ^ 1);
          tile_of[s] = tile;
          mbar_arrive_tx(&full[s], C::IN_TILE);
          tma_load_tile<IN_R>(in_buf + s * C::IN_TILE, &in_map, &full[s], (int)((tile / U) * kTileRows),
                              (int)(tile % U));
        }
      }
      const int s = k % STAGES;
      mbar_wait(&empty[s], ((k / STAGES) & 1) ^ 1);
      tile_of[s] = kQNoTile;
      mbar_arrive(&full[s]);
      sched_done(sched);
    }
    return;
  }
  const int lane = t & 31, warp = t >> 5;
  uint8_t* ob0 = out_buf + warp * C::OB * C::OUT_W;  // this warp's output tiles
  for (uint32_t i = 0;; ++i) {
    const int s = i % STAGES;
    mbar_wait(&full[s], (i / STAGES) & 1);
    const uint32_t tile = tile_of[s];
    if (tile == kQNoTile) break;
    const uint32_t ts = tile / U, j = tile - ts * U;
    const uint32_t row = ts * kTileRows + t;
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
    if (lane == 0) mbar_arrive(&empty[s]);
    if (!act) {
#pragma unroll
      for (int k = 0; k < 32; ++k) p[k] = make_float2(0.f, 0.f);
    }
    const uint64_t i0 = (uint64_t)j * S + (uint64_t)row * kRowElems;  // global index (shard j, R14)
    fwht_pairs<B>(p);                                      // K3: H (unnormalized)
    const DQ8 r8 = quant_dequant_row34<8, STOCH>(p, lg, cb, sr8, i0, z);  // K3: Q8; K4: DQ8 of the one source
    // K4: requantize at 4 bits into the warp's linear output tile (K3's quantizer with c = 1:
    // the same codes and scales as K4's requantization), then to the destination unit
    uint8_t* ot = ob0 + (i % C::OB) * C::OUT_W;
    float* osc = reinterpret_cast<float*>(ot + 32 * kQOutR);
    if (lane == 0) bulk_wait_read<C::OB - 1>();  // this warp's store of tile i - OB has left ot
    __syncwarp();
    quant_row4_b<STOCH>(p, lane, lg, act, ot, osc, sr4, i0, m16, r8);
    fence_proxy_async();
    __syncwarp();
    const uint32_t wrow0 = ts * kTileRows + 32 * warp;
    if (wrow0 < rows_per_shard) {
      uint8_t* unit = out.unit[j];
      const uint32_t rows = min(32u, rows_per_shard - wrow0);
      const uint32_t nsc = (rows * kRowElems) >> lg;
      const bool sc_bulk = nsc && ((nsc & 3u) == 0);
      float* g_sc = reinterpret_cast<float*>(unit + S / 2) + (((size_t)wrow0 * kRowElems) >> lg);
      if (lane == 0) {
        bulk_store(unit + (size_t)wrow0 * kQOutR, ot, rows * kQOutR);
        if (sc_bulk && ((reinterpret_cast<uintptr_t>(g_sc) & 15u) == 0)) bulk_store(g_sc, osc, nsc * 4);
        bulk_commit();
      }
      if (!(sc_bulk && ((reinterpret_cast<uintptr_t>(g_sc) & 15u) == 0)))
        for (uint32_t k = lane; k < nsc; k += 32) g_sc[k] = osc[k];
    }
  }
  if (lane == 0) bulk_wait<0>();
}

template <int IN_R, int B>
cudaError_t q84_launch(const CUtensorMap& in_map, const Q4Out& out, size_t S, int M, int G, float cb, uint32_t ntiles,
                       const SR& sr8, const SR& sr4, int sms, cudaStream_t st) {
  constexpr int SMEM = QCfg<IN_R>::SMEM;
  uint32_t* sched = sched_counter(st);
  if (!sched) return cudaErrorMemoryAllocation;
  const int grid = grid_for(ntiles, sms * QCfg<IN_R>::CTAS);
  cudaError_t e;
  if (sr8.on) {
    if ((e = set_smem(k_tlq_q84<IN_R, B, true>, SMEM)) != cudaSuccess) return e;
    k_tlq_q84<IN_R, B, true><<<grid, kQBlock, SMEM, st>>>(in_map, out, S, M, __builtin_ctz(G), cb, ntiles, sr8, sr4,
                                                          -0.0f, 16u, sched);
  } else {
    if ((e = set_smem(k_tlq_q84<IN_R, B, false>, SMEM)) != cudaSuccess) return e;
    k_tlq_q84<IN_R, B, false><<<grid, kQBlock, SMEM, st>>>(in_map, out, S, M, __builtin_ctz(G), cb, ntiles, sr8, sr4,
                                                           -0.0f, 16u, sched);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_tlq_q84(const void* grad, size_t grad_stride, int grad_dtype, size_t S, int M, int G, int b,
                           float cb, uint8_t* const* units, uint64_t remote_mask, int sr_on, uint32_t key8,
                           uint32_t key4, int sms, cudaStream_t st) {
  if (M < 1 || M > kMaxDests) return cudaErrorInvalidValue;
  const uint64_t rows = S / kRowElems;
  const uint32_t tps = (uint32_t)((rows + kTileRows - 1) / kTileRows);
  const uint32_t ntiles = tps * (uint32_t)M;
  const int in_r = grad_dtype == kBF16 ? 128 : 256;
  CUtensorMap in_map;
  cudaError_t e = make_row_map(&in_map, grad, in_r, rows, (uint64_t)M, (uint64_t)grad_stride * (in_r / kRowElems));
  if (e != cudaSuccess) return e;
  Q4Out out;
  memset(&out, 0, sizeof(out));
  for (int m = 0; m < M; ++m) out.unit[m] = units[m];
  out.remote = remote_mask;
  const SR sr8{sr_on, key8}, sr4{sr_on, key4};
#define KQ(IR) SDP4_B_SWITCH(b, return (q84_launch<IR, BB>(in_map, out, S, M, G, cb, ntiles, sr8, sr4, sms, st)))
  if (in_r == 128) {
    KQ(128);
  } else {
    KQ(256);
  }
#undef KQ
  return cudaErrorInvalidValue;
}

}  // namespace sdp4
