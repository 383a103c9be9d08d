// k_weights.cu -- K1 qwd_quantize, K2 qwd_apply (Alg. 2 l.2-5), K6 ring hop (sec. 2.3 ablation).
#include "sdp4_device.cuh"

namespace sdp4 {
namespace {

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
                                                                   uint64_t idx0, float z, uint32_t tpb) {
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
  // tpb > 0: block b streams its own tpb consecutive tiles (a non-persistent grid: the
  // hardware hands blocks to SMs as they free up -- a static persistent split measured 10-20%
  // slower on B200 streams); tpb == 0: persistent grid-stride
  const size_t t_end = tpb ? min(ntiles, ((size_t)blockIdx.x + 1) * tpb) : ntiles;
  const size_t t_begin = tpb ? (size_t)blockIdx.x * tpb : blockIdx.x;
  const size_t t_step = tpb ? 1 : gridDim.x;
  auto load = [&](size_t tile) {
    const size_t e = tile * TILE + t * 8;
    if (tile < t_end && e < S) {
      na0 = *reinterpret_cast<const float4*>(w_main + e);
      na1 = *reinterpret_cast<const float4*>(w_main + e + 4);
      if constexpr (DIFF) {
        nu0 = *reinterpret_cast<const uint4*>(w_model + e);
        if constexpr (sizeof(TM) == 4) nu1 = *reinterpret_cast<const uint4*>(w_model + e + 4);
      }
    }
  };
  load(t_begin);
  for (size_t tile = t_begin; tile < t_end; tile += t_step) {
    const size_t e0 = tile * TILE + t * 8;
    const bool act = e0 < S;
    const float4 a0 = na0, a1 = na1;
    const uint4 u0 = nu0, u1 = nu1;
    load(tile + t_step);
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
          const float ds = div_by_q(stored_scale(a, 1.f), q, __fdiv_rn(1.f, q));
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
constexpr int kK2Chunk = 4;  // tiles per scheduler claim
constexpr uint32_t kNoTileW = 0xffffffffu;
template <int BITS>
struct K2rCfg {
  static constexpr int CODE_BYTES = kK2rTile * (BITS == 32 ? 32 : BITS) / 8;
  static constexpr int SC_BYTES = BITS == 32 ? 0 : kK2rTile / 32 * 4;  // G >= 32
  static constexpr int STAGE = CODE_BYTES + SC_BYTES;
  static constexpr int SMEM = kK2rStages * STAGE + kK2rStages * 12 + 128;
};

template <typename TM, int BITS, bool ADD>
__global__ void __launch_bounds__(kVecThreads) k2_qwd_apply_ring(const Dests units, size_t S, size_t stride, int P,
                                                                    int rot, int U, int lg, TM* __restrict__ w_model,
                                                                    float z, uint32_t* sched) {
  using C = K2rCfg<BITS>;
  constexpr int ROUNDS = kK2rTile / (kVecThreads * 8);
  constexpr float q = float((1 << (BITS == 32 ? 1 : BITS - 1)) - 1);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem<128>(smem_raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kK2rStages * C::STAGE);
  uint32_t* tile_of = reinterpret_cast<uint32_t*>(bar + kK2rStages);  // tile carried by each stage
  const int t = threadIdx.x;
  // U units (U = P, or P - 1 when the owner applied its own in K1), unit fastest, starting at rot
  const size_t tpu = (S + kK2rTile - 1) / kK2rTile, ntiles = tpu * U;
  const size_t sc_off = S * (BITS == 32 ? 4 : BITS) / 8;
  auto tile_of_fn = [&](size_t tile, size_t& ts, size_t& j) {
    ts = tile / U;
    j = tile - ts * U + rot;
    if (j >= (size_t)P) j -= P;
  };
  if (t == 0) {
    for (int s = 0; s < kK2rStages; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // thread 0 claims tiles from the dynamic scheduler, kK2Chunk at a time (sched_counter)
  uint32_t c_next = 0, c_end = 0;
  bool done = false;
  auto issue = [&](uint32_t k) {  // thread 0: the next claimed tile into stage k % STAGES
    const int s = k % kK2rStages;
    if (c_next == c_end && !done) {
      c_next = sched_claim(sched, kK2Chunk);
      c_end = (uint32_t)min((size_t)c_next + kK2Chunk, ntiles);
      if (c_next >= ntiles) {
        done = true;
        sched_done(sched);
      }
    }
    if (done) {  // no more work: complete the stage's phase with no data
      tile_of[s] = kNoTileW;
      mbar_arrive(&bar[s]);
      return;
    }
    const size_t tile = c_next++;
    tile_of[s] = (uint32_t)tile;
    size_t ts, j;
    tile_of_fn(tile, ts, j);
    const size_t e0 = ts * kK2rTile;
    const uint32_t n = (uint32_t)min((size_t)kK2rTile, S - e0);
    const uint32_t cb = n * (BITS == 32 ? 32 : BITS) / 8;
    uint32_t sb = 0;
    if constexpr (BITS != 32) sb = ((((n >> lg) * 4) + 15) & ~15u);
    mbar_arrive_tx(&bar[s], cb + sb);
    const uint8_t* unit = units.p[j];
    bulk_load(smem + s * C::STAGE, unit + e0 * (BITS == 32 ? 32 : BITS) / 8, cb, &bar[s]);
    if constexpr (BITS != 32)
      bulk_load(smem + s * C::STAGE + C::CODE_BYTES, unit + sc_off + (e0 >> lg) * 4, sb, &bar[s]);
  };
  if (t == 0)
    for (int k = 0; k < kK2rStages; ++k) issue(k);
  __syncthreads();  // tile_of[] of the first stages is visible (later ones: after the per-tile barrier)
  for (uint32_t k = 0;; ++k) {
    const uint32_t tid = tile_of[k % kK2rStages];  // written by thread 0 before an earlier barrier
    if (tid == kNoTileW) break;
    size_t ts, j;
    tile_of_fn(tid, ts, j);
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
        const float ds = div_by_q(reinterpret_cast<const float*>(st + C::CODE_BYTES)[el >> lg], q, __fdiv_rn(1.f, q));
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
          const float ds = div_by_q(reinterpret_cast<const float*>(recv + sc_off)[e0 >> lg], q, __fdiv_rn(1.f, q));
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


}  // namespace

cudaError_t launch_qwd_quantize(const float* w_main, const void* w_model_shard, int model_dtype,
                                size_t S, int bits, int G, const Dests& dst, int sr_on, uint32_t sr_key,
                                uint64_t idx0, int sms, cudaStream_t st, bool apply_own) {
  const SR sr{sr_on, sr_key};
  if (apply_own && !w_model_shard) return cudaErrorInvalidValue;
  void* wm = const_cast<void*>(w_model_shard);  // written only by the APPLY variants
  const size_t ntiles = (S + kVecThreads * 8 - 1) / (kVecThreads * 8);
  static const uint32_t tpb = [] {  // tiles per block (measurement override: SDP4_K1_TPB, 0 = persistent)
    const char* e = getenv("SDP4_K1_TPB");
    return e ? (uint32_t)atoi(e) : 8u;
  }();
  // persistent grid: as many CTAs per SM as the variant's registers allow (at most kVecCtas)
#define K1(TM, B, DF, AP)                                                                                    \
  do {                                                                                                       \
    static const int nb = std::min(kVecCtas, occ_blocks(k1_qwd_quantize<TM, B, DF, AP>, kVecThreads));      \
    const int grid = tpb ? (int)((ntiles + tpb - 1) / tpb) : grid_for(ntiles, sms * nb);                     \
    k1_qwd_quantize<TM, B, DF, AP><<<grid, kVecThreads, 0, st>>>(                                            \
        w_main, static_cast<TM*>(wm), S, __builtin_ctz(G), dst, sr, idx0, -0.0f, tpb);                       \
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
  uint32_t* sched = sched_counter(st);
  if (!sched) return cudaErrorMemoryAllocation;
#define K2(TM, B, AD)                                                                          \
  do {                                                                                                 \
    set_smem(k2_qwd_apply_ring<TM, B, AD>, K2rCfg<B>::SMEM);                                           \
    k2_qwd_apply_ring<TM, B, AD><<<grid_r, kVecThreads, K2rCfg<B>::SMEM, st>>>(                         \
        units, S, stride, P, rot % P, U, __builtin_ctz(G), static_cast<TM*>(w_model), -0.0f, sched);   \
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


}  // namespace sdp4
