// k_fused.cu -- the one-launch P2P paths for small messages: a whole qWD step
// (Alg. 2 l.2-5) or a whole TLq-HS reduce-scatter (Alg. 3) as ONE kernel per rank, the P2P sync
// protocol's waits and raises done in-kernel.  The multi-launch path costs two to three
// stream-ordered hand-offs per call (wait kernel / memop + kernel + flag raise, ~8-15 us each,
// tools/latency_probe.cu); one kernel pays one launch plus a ~2.6 us flag round trip per
// exchange.  The arithmetic is K1/K2 (qWD) and K3/K4/K5 (TLq-HS) operation for operation, on
// the same shared helpers, so results are bit-identical to the multi-launch path and the oracle.
#include "k_fused.cuh"

namespace sdp4 {
namespace {

// =====================================================================================
// One-launch qWD step.  CTA tasks of 2048 elements (K1's tile: 256 threads x 8 elements, a
// group is G/8 consecutive threads): phase A = (vrank v, tile ts) -> K1 with apply_own on the
// own shard, unit written into region[rank]; phase B = (v, tile ts, peer j) -> K2's update of
// shard j from rank j's unit, pulled over NVLink.  Flag stage 0: A waits free[0][q] (every peer
// done reading my previous unit) and its last task raises data[0][me] at every peer; B waits
// data[0][j] and its last task raises free[0][me] at every peer.
// =====================================================================================
constexpr int kFqTile = kFThreads * 8;

struct FqwdArgs {
  const float* w_main[kMaxVr];
  void* w_model[kMaxVr];
  uint32_t key[kMaxVr];
  size_t S;
  int lg, sr_on;
  float z;
};

template <typename TM>
__device__ __forceinline__ void store_replica8(TM* w, const float* m, const float* x) {  // w = rn(m + x)
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
template <typename TM>
__device__ __forceinline__ void load_replica8(const TM* w, float* m) {
  if constexpr (sizeof(TM) == 2) {
    const uint4 u = *reinterpret_cast<const uint4*>(w);
    m[0] = bf16_lo(u.x); m[1] = bf16_hi(u.x); m[2] = bf16_lo(u.y); m[3] = bf16_hi(u.y);
    m[4] = bf16_lo(u.z); m[5] = bf16_hi(u.z); m[6] = bf16_lo(u.w); m[7] = bf16_hi(u.w);
  } else {
    const float4 a = reinterpret_cast<const float4*>(w)[0], b = reinterpret_cast<const float4*>(w)[1];
    m[0] = a.x; m[1] = a.y; m[2] = a.z; m[3] = a.w; m[4] = b.x; m[5] = b.y; m[6] = b.z; m[7] = b.w;
  }
}

template <typename TM, int BITS>
__global__ void __launch_bounds__(kFThreads) kf_qwd_step(const FusedSync fs, const FqwdArgs a) {
  constexpr float q = float((1 << (BITS == 32 ? 1 : BITS - 1)) - 1);
  __shared__ float red[kFThreads / 32];
  __shared__ uint32_t s_task;
  __shared__ uint32_t s_free_ok;   // bit v: the free flags of virtual rank v were seen
  __shared__ uint64_t s_seen[kMaxVr];  // bit j: data[0][j] of virtual rank v was seen
  const int t = threadIdx.x;
  const int nv = fs.nv, P = fs.P;
  const size_t S = a.S;
  const uint32_t tpu = (uint32_t)((S + kFqTile - 1) / kFqTile);
  const uint32_t TA = tpu * nv, TB = tpu * (uint32_t)(P - 1) * nv;
  const size_t sc_off = S * (BITS == 32 ? 4 : BITS) / 8;
  const int tpg = (1 << a.lg) >> 3;
  if (t == 0) {
    s_free_ok = 0;
    for (int v = 0; v < kMaxVr; ++v) s_seen[v] = 0;
  }
  if (t == 0) tstamp(fs, blockIdx.x, 0);
  for (;;) {
    if (t == 0) s_task = atomicAdd(fs.ctr, 1u);
    __syncthreads();
    const uint32_t task = s_task;
    if (task >= TA + TB) break;
    if (task < TA) {  // ---- phase A: K1 + apply_own on (v, ts)
      const int v = (int)(task % nv);
      const uint32_t ts = task / nv;
      const int r = fs.rank[v];
      if (t == 0) tstamp(fs, blockIdx.x, 2);
      if (t == 0 && !((s_free_ok >> v) & 1u)) {
        for (int q2 = 0; q2 < P; ++q2)
          if (q2 != r) wait_flag(fs, flag(fs, r, kFlagFree, 0, q2), wait_code(kFlagFree, 0, q2));
        s_free_ok |= 1u << v;
      }
      __syncthreads();
      uint8_t* unit = fs.region[r];
      TM* wm = static_cast<TM*>(a.w_model[v]) + (size_t)r * S;
      const size_t e0 = (size_t)ts * kFqTile + t * 8;
      const bool act = e0 < S;
      float d[8], m[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) d[i] = m[i] = 0.f;
      if (act) {
        const float4 a0 = *reinterpret_cast<const float4*>(a.w_main[v] + e0);
        const float4 a1 = *reinterpret_cast<const float4*>(a.w_main[v] + e0 + 4);
        load_replica8<TM>(wm + e0, m);
        d[0] = __fsub_rn(a0.x, m[0]); d[1] = __fsub_rn(a0.y, m[1]);
        d[2] = __fsub_rn(a0.z, m[2]); d[3] = __fsub_rn(a0.w, m[3]);
        d[4] = __fsub_rn(a1.x, m[4]); d[5] = __fsub_rn(a1.y, m[5]);
        d[6] = __fsub_rn(a1.z, m[6]); d[7] = __fsub_rn(a1.w, m[7]);
      }
      if constexpr (BITS == 32) {  // identity codec (R12)
        if (act) {
          float4* o = reinterpret_cast<float4*>(unit + e0 * 4);
          o[0] = make_float4(d[0], d[1], d[2], d[3]);
          o[1] = make_float4(d[4], d[5], d[6], d[7]);
          store_replica8<TM>(wm + e0, m, d);
        }
      } else {
        float amax = 0.f;
#pragma unroll
        for (int i = 0; i < 8; i += 2) amax = max3_abs_nan(amax, d[i], d[i + 1]);
        amax = group_max(amax, tpg, red);
        const QP p = qparam(amax, q);
        if (act) {
          uint32_t rr[8];
          if (a.sr_on) {
#pragma unroll
            for (int i = 0; i < 8; ++i) rr[i] = rq_sr(d[i], p.inv, sr_u((uint64_t)r * S + e0 + i, a.key[v]), q);
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) rr[i] = rq(d[i], p.inv);
          }
          if constexpr (BITS == 2) {
            uint32_t w = pack2x8(rr);
            if (!p.ok) w = 0u;
            *reinterpret_cast<uint16_t*>(unit + e0 / 4) = (uint16_t)w;
          } else if constexpr (BITS == 4) {
            uint32_t w = pack4x8(rr);
            if (!p.ok) w = 0u;
            *reinterpret_cast<uint32_t*>(unit + e0 / 2) = w;
          } else {
            uint2 w = make_uint2(pack8x4(rr[0], rr[1], rr[2], rr[3]), pack8x4(rr[4], rr[5], rr[6], rr[7]));
            if (!p.ok) w = make_uint2(0u, 0u);
            *reinterpret_cast<uint2*>(unit + e0) = w;
          }
          if ((t & (tpg - 1)) == 0) reinterpret_cast<float*>(unit + sc_off)[e0 >> a.lg] = stored_scale(amax, 1.f);
          // K2's update from the codes just packed (K1 with apply_own)
          const float ds = div_by_q(stored_scale(amax, 1.f), q, __fdiv_rn(1.f, q));
          float f[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) f[i] = mulz(p.ok ? __fsub_rn(__uint_as_float(rr[i]), kMagic) : 0.f, ds, a.z);
          store_replica8<TM>(wm + e0, m, f);
        }
      }
      __syncthreads();
      if (t == 0) tstamp(fs, blockIdx.x, 3);
      if (t == 0 && finish_task(fs, 0, v, tpu)) {
        for (int q2 = 0; q2 < P; ++q2)
          if (q2 != r) st_relaxed_sys(flag(fs, r, kFlagFree, 0, q2), 0u);
        __threadfence_system();
        for (int q2 = 0; q2 < P; ++q2)
          if (q2 != r) st_relaxed_sys(flag(fs, q2, kFlagData, 0, r), 1u);
      }
    } else {  // ---- phase B: K2 on (v, ts, peer j), the unit pulled from rank j
      const uint32_t b = task - TA;
      const int v = (int)(b % nv);
      const uint32_t rest = b / nv;
      const uint32_t jj = rest % (uint32_t)(P - 1), ts = rest / (uint32_t)(P - 1);
      const int r = fs.rank[v];
      const int j = (r + 1 + (int)jj) % P;
      if (t == 0 && !((s_seen[v] >> j) & 1ull)) {
        wait_flag(fs, flag(fs, r, kFlagData, 0, j), wait_code(kFlagData, 0, j));
        s_seen[v] |= 1ull << j;
      }
      if (t == 0) tstamp(fs, blockIdx.x, 4);
      __syncthreads();
      const uint8_t* unit = fs.region[j];
      TM* wm = static_cast<TM*>(a.w_model[v]) + (size_t)j * S;
      const size_t e = (size_t)ts * kFqTile + t * 8;
      float x[8];
      if (e < S) {
        if constexpr (BITS == 32) {
          const float4 u0 = __ldcg(reinterpret_cast<const float4*>(unit + e * 4));
          const float4 u1 = __ldcg(reinterpret_cast<const float4*>(unit + e * 4 + 16));
          x[0] = u0.x; x[1] = u0.y; x[2] = u0.z; x[3] = u0.w; x[4] = u1.x; x[5] = u1.y; x[6] = u1.z; x[7] = u1.w;
        } else {
          float fv[8];
          if constexpr (BITS == 8) {
            const uint2 w = __ldcg(reinterpret_cast<const uint2*>(unit + e));
            dec8x4(w.x, fv);
            dec8x4(w.y, fv + 4);
          } else if constexpr (BITS == 4) {
            dec4x8(__ldcg(reinterpret_cast<const unsigned int*>(unit + e / 2)), fv);
          } else {
            const uint32_t w = __ldcg(reinterpret_cast<const unsigned short*>(unit + e / 4));
#pragma unroll
            for (int i = 0; i < 8; ++i) fv[i] = float((int)(((w >> (2 * i)) & 3u) ^ 2u) - 2);
          }
          const float ds = div_by_q(__ldcg(reinterpret_cast<const float*>(unit + sc_off) + (e >> a.lg)), q,
                                    __fdiv_rn(1.f, q));
#pragma unroll
          for (int i = 0; i < 8; ++i) x[i] = mulz(fv[i], ds, a.z);
        }
      }
      // every thread's reads of unit j are done (their values are in x): the last task to get
      // here frees every peer's unit -- before the replica update, so the fence and raises
      // overlap it
      __syncthreads();
      if (t == 0 && finish_task(fs, 1, v, tpu * (uint32_t)(P - 1))) {
        for (int q2 = 0; q2 < P; ++q2)
          if (q2 != r) st_relaxed_sys(flag(fs, r, kFlagData, 0, q2), 0u);
        __threadfence_system();
        for (int q2 = 0; q2 < P; ++q2)
          if (q2 != r) st_relaxed_sys(flag(fs, q2, kFlagFree, 0, r), 1u);
      }
      if (e < S) {
        float m[8];
        load_replica8<TM>(wm + e, m);
        store_replica8<TM>(wm + e, m, x);
      }
      __syncthreads();  // (the next task's s_task write waits for every thread)
      if (t == 0) tstamp(fs, blockIdx.x, 5);
    }
  }
  if (t == 0) {
    tstamp(fs, blockIdx.x, 1);
    exit_unit(fs, gridDim.x);
  }
}

__global__ void k_fill32(uint32_t* p, size_t n, uint32_t v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}

}  // namespace

cudaError_t launch_fused_qwd(const FusedSync& fs, const float* const* w_main, void* const* w_model, int model_dtype,
                             size_t S, int bits, int G, int sr_on, const uint32_t* sr_key, int sms, cudaStream_t st) {
  if (fs.nv < 1 || fs.nv > kMaxVr || fs.P < 2 || fs.P > kMaxDests || G > 2048) return cudaErrorInvalidValue;
  FqwdArgs a;
  memset(&a, 0, sizeof(a));
  for (int v = 0; v < fs.nv; ++v) {
    a.w_main[v] = w_main[v];
    a.w_model[v] = w_model[v];
    a.key[v] = sr_key[v];
  }
  a.S = S;
  a.lg = __builtin_ctz(G);
  a.sr_on = sr_on;
  a.z = -0.0f;
  const size_t tasks = (S + kFqTile - 1) / kFqTile * (size_t)fs.P * fs.nv;
  const int grid = grid_for(tasks, sms * 4);
#define KQ(TM, B) kf_qwd_step<TM, B><<<grid, kFThreads, 0, st>>>(fs, a)
#define KQB(TM) \
  if (bits == 2) KQ(TM, 2); else if (bits == 4) KQ(TM, 4); else if (bits == 8) KQ(TM, 8); else KQ(TM, 32)
  if (model_dtype == kBF16) {
    KQB(uint16_t);
  } else {
    KQB(float);
  }
#undef KQB
#undef KQ
  return cudaGetLastError();
}

bool fused_tlq_supported(int bits_intra, int bits_inter, int b) {
  return (bits_intra == 4 || bits_intra == 8) && (bits_inter == 4 || bits_inter == 8) && b >= 0 && b <= 256;
}

cudaError_t launch_fused_tlq(const FusedSync& fs, const void* const* grad, int grad_dtype, float* const* out,
                             int M, int N, size_t S, int G, int b, float cb, float kappa, int bits_intra,
                             int bits_inter, size_t w8, size_t w4, int sr_on, const uint32_t* key8,
                             const uint32_t* key4, int sms, cudaStream_t st) {
  if (fs.nv < 1 || fs.nv > kMaxVr || fs.P != M * N || fs.P < 2 || fs.P > kMaxDests || fs.nv * fs.P > 64 ||
      !fused_tlq_supported(bits_intra, bits_inter, b))
    return cudaErrorInvalidValue;
  FtlqArgs a;
  memset(&a, 0, sizeof(a));
  for (int v = 0; v < fs.nv; ++v) {
    a.grad[v] = grad[v];
    a.out[v] = out[v];
    a.key8[v] = key8[v];
    a.key4[v] = key4[v];
  }
  a.S = S;
  a.w8 = w8;
  a.w4 = w4;
  a.M = M;
  a.N = N;
  a.lg = __builtin_ctz(G);
  a.sr_on = sr_on;
  a.cb = cb;
  a.kappa = kappa;
  a.z = -0.0f;
  a.m16 = 16u;
  static const uint32_t dbg = getenv("SDP4_FUSED_DBG") ? (uint32_t)atoi(getenv("SDP4_FUSED_DBG")) : 0u;
  a.dbg = dbg;
  const size_t rb = (S / kRowElems + kFtRows - 1) / kFtRows;
  const size_t warps = rb * (size_t)fs.P * fs.nv;
  const int grid = grid_for((warps + 7) / 8, sms * 4);
  const bool stoch = sr_on != 0;
  a.grad_bf16 = grad_dtype == kBF16;
  return bits_intra == 8 ? launch_fused_tlq_bi8(fs, a, bits_inter, b, stoch, grid, st)
                         : launch_fused_tlq_bi4(fs, a, bits_inter, b, stoch, grid, st);
}

cudaError_t launch_fill32(uint32_t* p, size_t n, uint32_t v, cudaStream_t st) {
  if (!n) return cudaSuccess;
  k_fill32<<<grid_for((n + 255) / 256, 1024), 256, 0, st>>>(p, n, v);
  return cudaGetLastError();
}

}  // namespace sdp4
