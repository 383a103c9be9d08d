// k_reduce.cu -- K4 tlq_dq_reduce_q: dequantize + fp32 reduce + requantize (Alg. 3 l.5, 7, 9).
#include "sdp4_device.cuh"

namespace sdp4 {
namespace {

// =====================================================================================
// K4  TLq dequantize + reduce + requantize (Alg. 3 l.5, 7, 9, FP32 reduce P:344).
// Vector layout: a tile is 8192 elements of sub-block m'; consumer thread t owns the 64
// contiguous elements [64t, 64t+64), read from smem as 16-byte chunks in XOR-permuted order
// (slot c <- chunk c ^ f(t): conflict-free; the permutation is undone by the store
// addresses).  Warp-specialized: a dedicated producer warp streams (tile, source l'') items
// through a STAGES-deep ring of 1-D bulk copies (codes + scales), each slot guarded by a
// "full" mbarrier (transaction bytes) and an "empty" mbarrier that each of the four consumer
// warps arrives on when it is done with its quarter -- no CTA-wide barrier per item, so warps
// drift within the ring depth.  Sources are summed in order l'' = 0..N-1 (R8); the sum is
// requantized (one division per group; a group spans at most one warp) and stored straight to
// global memory (local unit), or staged in smem and bulk-stored by consumer thread 0 to unit m'
// (P2P transport: the receive slot of node m' itself -- the inter all-to-all), with named
// barriers over the consumer warps only.
// =====================================================================================
constexpr int kK4Threads = 128;                   // consumer threads (four warps)
constexpr int kK4Block = kK4Threads + 32;         // + one producer warp
constexpr int kK4Ctas = 3;        // CTAs per SM with remote output staging
constexpr int kK4CtasLocal = 4;   // without it (every destination local: P = 1, NCCL transport)
constexpr int kK4Tile = kK4Threads * 64;
constexpr int kK4Chunk = 8;  // tiles per scheduler claim
constexpr uint32_t kNoTile = 0xffffffffu;

template <int BIN, int BOUT, bool REMOTE = true>
struct K4Cfg {
  static constexpr int CTAS = REMOTE ? kK4Ctas : kK4CtasLocal;
  static constexpr int CODE_BYTES = kK4Tile * BIN / 8;
  static constexpr int SC_BYTES = BIN == 32 ? 0 : kK4Tile / 32 * 4;
  static constexpr int STAGE = CODE_BYTES + SC_BYTES;
  static constexpr int OUT_TILE = kK4Tile * BOUT / 8 + kK4Tile / 32 * 4;  // staged output: codes + scales
  static constexpr int OUTB = !REMOTE ? 0 : (OUT_TILE <= 8 * 1024 ? 4 : 2);  // staged remote output tiles in flight
  static constexpr int S0 = ((REMOTE ? 74 : 55) * 1024 - OUTB * OUT_TILE) / STAGE;  // per-CTA budget: CTAS per SM
  static constexpr int STAGES = S0 > 8 ? 8 : (S0 < 2 ? 2 : S0);
  static constexpr int SMEM = STAGES * STAGE + OUTB * OUT_TILE + 2 * 8 * STAGES + 4 * STAGES + 128;
  static_assert(SMEM <= 227 * 1024, "K4 tile configuration exceeds the per-CTA shared memory");
  static constexpr int CPT = 64 * BIN / 8 / 16;   // 16-byte chunks per thread
  static constexpr int EPC = 64 / CPT;            // elements per chunk
};

struct K4Pull {  // IntraPull, K4 side: tiles of source l with ts % den < num come from src[l]
  const uint8_t* src[kMaxN];
  uint32_t mask, num, den;
};

// REMOTE: some destination unit is peer memory (P2P inter all-to-all); G64: G >= 64 (a group
// is whole threads).  Both are compile-time so the common local / G >= 64 path carries none
// of the other paths' branches and selects (K4 is issue- and ALU-bound: ~1.56 B per element).
template <int BIN, int BOUT, bool STOCH, bool REMOTE, bool G64>
__global__ void __launch_bounds__(kK4Block, K4Cfg<BIN, BOUT, REMOTE>::CTAS) k4_tlq_dq_reduce_q(const uint8_t* __restrict__ recv, size_t in_unit_bytes,
                                                          int N, int M, size_t S, int lg, const Dests dst,
                                                          uint32_t tpu, uint32_t ntiles, float z, const SR sr,
                                                          int l_self, size_t sr_stride, size_t sr_off,
                                                          const K4Pull pull, uint32_t m16, uint32_t* sched) {
  using C = K4Cfg<BIN, BOUT, REMOTE>;
  constexpr int STAGES = C::STAGES, CPT = C::CPT, EPC = C::EPC;
  constexpr float qin = float((1 << (BIN == 32 ? 1 : BIN - 1)) - 1);
  const float rqin = __fdiv_rn(1.f, qin);  // rn(1/q): div_by_q's reciprocal (constant-folded)
  constexpr float qout = float((1 << (BOUT == 32 ? 1 : BOUT - 1)) - 1);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem<128>(smem_raw);
  uint8_t* out_buf = smem + STAGES * C::STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(out_buf + C::OUTB * C::OUT_TILE);
  uint64_t* empty = full + STAGES;
  uint32_t* tile_of = reinterpret_cast<uint32_t*>(empty + STAGES);  // tile id carried by each slot
  const int t = threadIdx.x;
  if (t == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kK4Threads / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();  // the only CTA-wide barrier
  if (t >= kK4Threads) {  // ---- producer warp: one lane claims tiles and streams their (tile, source) items
    if (t == kK4Threads) {
      uint32_t pk = 0;
      for (;;) {
        const uint32_t t0 = sched_claim(sched, kK4Chunk);
        if (t0 >= ntiles) break;
        const uint32_t t1 = min(t0 + kK4Chunk, ntiles);
        for (uint32_t tile = t0; tile < t1; ++tile) {
          const uint32_t ts = tile / (uint32_t)M, mp = tile - ts * (uint32_t)M;  // unit fastest
          const size_t e0 = (size_t)ts * kK4Tile;
          const uint32_t n = (uint32_t)min((size_t)kK4Tile, S - e0);
          const uint32_t cb = n * BIN / 8;
          uint32_t sb = 0;
          if constexpr (BIN != 32) sb = (((n >> lg) * 4) + 15) & ~15u;
          for (int l = 0; l < N; ++l, ++pk) {  // sources l'' = 0..N-1 (R8)
            const int s = pk % STAGES;
            mbar_wait(&empty[s], ((pk / STAGES) & 1) ^ 1);  // the consumers released this slot
            tile_of[s] = (ts << 6) | mp;  // (tile-in-unit, unit): M <= 64
            // K3 tile (kTileElems) holding these elements: pulled from the source's outbox or pushed
            const bool pulled = ((pull.mask >> l) & 1u) && (uint32_t)(e0 / kTileElems) % pull.den < pull.num;
            const uint8_t* unit = pulled ? pull.src[l] + (size_t)mp * in_unit_bytes
                                         : recv + ((size_t)l * M + mp) * in_unit_bytes;
            mbar_arrive_tx(&full[s], cb + sb);  // release: tile_of[s] is visible with the data
            bulk_load(smem + s * C::STAGE, unit + e0 * BIN / 8, cb, &full[s]);
            if constexpr (BIN != 32)
              bulk_load(smem + s * C::STAGE + C::CODE_BYTES, unit + S * BIN / 8 + (e0 >> lg) * 4, sb, &full[s]);
          }
        }
      }
      const int s = pk % STAGES;  // end of work: a slot carrying no data, tile id kNoTile
      mbar_wait(&empty[s], ((pk / STAGES) & 1) ^ 1);
      tile_of[s] = kNoTile;
      mbar_arrive(&full[s]);
      sched_done(sched);
    }
    return;
  }

  // slot c of this thread holds chunk c ^ f (f = 0 for the fp32 identity path)
  const int f = BIN == 32 ? 0 : (CPT >= 8 ? (t & 7) : ((t / (8 / CPT)) & (CPT - 1)));
  const int tpg = G64 ? (1 << (lg - 6)) : 1;  // threads per group
  uint32_t k = 0;
  for (uint32_t i = 0;; ++i) {
    {  // the tile of the next item (kNoTile: no more work)
      const int s = k % STAGES;
      mbar_wait(&full[s], (k / STAGES) & 1);
    }
    const uint32_t tile = tile_of[k % STAGES];
    if (tile == kNoTile) break;
    const uint32_t ts = tile >> 6, mp = tile & 63u;
    const size_t e0 = (size_t)ts * kK4Tile;
    const bool act = e0 + 64 * t < S;
    float2 acc[32];  // slot order: acc[i] = elements (2i, 2i+1) of the slot-ordered 64
    // one (tile, source) item: wait for its ring slot, dequantize, fold into acc (R8), release
    auto consume = [&](auto first) {
      const int s = k % STAGES;
      mbar_wait(&full[s], (k / STAGES) & 1);
      const uint8_t* codes = smem + s * C::STAGE + t * (64 * BIN / 8);
      float ds0 = 1.f, ds1 = 1.f;
      if constexpr (BIN != 32) {
        const float* sc = reinterpret_cast<const float*>(smem + s * C::STAGE + C::CODE_BYTES);
        if constexpr (G64) {
          ds0 = ds1 = div_by_q(sc[(64 * t) >> lg], qin, rqin);
        } else {
          ds0 = div_by_q(sc[2 * t], qin, rqin);
          ds1 = div_by_q(sc[2 * t + 1], qin, rqin);
        }
      }
      k4_item<BIN, CPT, EPC, decltype(first)::value>(codes, ds0, ds1, f, z, acc);
      __syncwarp();
      if ((t & 31) == 0) mbar_arrive(&empty[s]);  // this warp is done with its quarter of slot s
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
    const bool remote = REMOTE && ((dst.remote >> mp) & 1ull);  // CTA-uniform
    uint8_t* gout = dst.p[mp];
    // output codes / scales: the staged smem tile (remote) or the unit in global memory (local);
    // two explicit address spaces, so stores are STS / STG rather than generic
    constexpr int OB = C::OUTB > 0 ? C::OUTB : 1;  // (no staging in the local-only variant)
    uint8_t* ot_s = out_buf + (i % OB) * C::OUT_TILE;
    uint8_t* ot_g = gout + e0 * BOUT / 8;
    float* osc_s = reinterpret_cast<float*>(ot_s + kK4Tile * BOUT / 8);
    float* osc_g = reinterpret_cast<float*>(gout + S * BOUT / 8) + (e0 >> lg);
    if (remote) {
      if (t == 0) bulk_wait_read<OB - 1>();  // the stores of tile i - OUTB have left out_buf[i % OUTB]
      named_sync(1, kK4Threads);
    }
    auto vbase = [&](int v) {  // element offset (within the thread's 64) of slot-order vector v
      if constexpr (EPC >= 16) return (((16 * v) / EPC) ^ f) * EPC + (16 * v) % EPC;
      else return 16 * v;
    };
    if constexpr (BOUT == 32) {
      if (act) {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 w = make_float4(acc[8 * v + 2 * q].x, acc[8 * v + 2 * q].y, acc[8 * v + 2 * q + 1].x,
                                         acc[8 * v + 2 * q + 1].y);
            const int off = (64 * t + vbase(v)) * 4 + 16 * q;
            if (remote) *reinterpret_cast<float4*>(ot_s + off) = w;
            else *reinterpret_cast<float4*>(ot_g + off) = w;
          }
        }
      }
    } else {
      // 4-bit output codes come out of the quantizer biased by 8 (pack4x8_b)
      constexpr float magic = BOUT == 4 ? kMagicB4 : kMagic;
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
      if constexpr (G64) {
        a0 = max_nan(max_nan(am[0], am[1]), max_nan(am[2], am[3]));
#pragma unroll
        if (tpg == 2) {  // G = 128 (the common case): one exchange
          a0 = max_nan(a0, __shfl_xor_sync(0xffffffffu, a0, 1));
        } else {
#pragma unroll
          for (int off = 1; off < 32; off <<= 1)
            if (off < tpg) a0 = max_nan(a0, __shfl_xor_sync(0xffffffffu, a0, off));
        }
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
              r[2 * q] = rq_sr(acc[8 * v + q].x, iv, sr_u(i0 + 2 * q, sr.key), qout, magic);
              r[2 * q + 1] = rq_sr(acc[8 * v + q].y, iv, sr_u(i0 + 2 * q + 1, sr.key), qout, magic);
            }
          } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float2 y = f2rq(acc[8 * v + q], make_float2(iv, iv), magic);
              r[2 * q] = __float_as_uint(y.x);
              r[2 * q + 1] = __float_as_uint(y.y);
            }
          }
          const bool okv = h ? p1.ok : p0.ok;
          if constexpr (BOUT == 4) {
            uint2 w = make_uint2(pack4x8_b(r, m16), pack4x8_b(r + 8, m16));
            if (!okv) w = make_uint2(0u, 0u);
            if (remote) *reinterpret_cast<uint2*>(ot_s + e / 2) = w;
            else *reinterpret_cast<uint2*>(ot_g + e / 2) = w;
          } else {
            uint4 w = make_uint4(pack8x4(r[0], r[1], r[2], r[3]), pack8x4(r[4], r[5], r[6], r[7]),
                                 pack8x4(r[8], r[9], r[10], r[11]), pack8x4(r[12], r[13], r[14], r[15]));
            if (!okv) w = make_uint4(0u, 0u, 0u, 0u);
            if (remote) *reinterpret_cast<uint4*>(ot_s + e) = w;
            else *reinterpret_cast<uint4*>(ot_g + e) = w;
          }
        }
        if constexpr (G64) {
          if ((t & (tpg - 1)) == 0) {
            if (remote) osc_s[(64 * t) >> lg] = stored_scale(a0, 1.f);
            else osc_g[(64 * t) >> lg] = stored_scale(a0, 1.f);
          }
        } else {
          const float2 w = make_float2(stored_scale(a0, 1.f), stored_scale(a1, 1.f));
          if (remote) *reinterpret_cast<float2*>(osc_s + 2 * t) = w;
          else *reinterpret_cast<float2*>(osc_g + 2 * t) = w;
        }
      }
    }
    if (remote) {  // unit m' -> node m' (P2P: the peer's receive slot -- Alg. 3 l.10)
      fence_proxy_async();
      named_sync(1, kK4Threads);
      const uint32_t n = (uint32_t)min((size_t)kK4Tile, S - e0);
      store_tile(ot_s, n * BOUT / 8, osc_s, BOUT == 32 ? 0u : (n >> lg), ot_g, osc_g);
      if (t == 0) bulk_commit();
    }
  }
  if (t == 0) bulk_wait<0>();
}


template <int BIN, int BOUT, bool STOCH, bool REMOTE, bool G64>
cudaError_t k4_launch_v(const uint8_t* recv, size_t in_unit_bytes, int N, int M, size_t S, int G, const Dests& dst,
                        const SR& sr, int l_self, size_t sr_stride, size_t sr_off, int sms, cudaStream_t st,
                        const K4Pull& pull) {
  constexpr int SMEM = K4Cfg<BIN, BOUT, REMOTE>::SMEM;
  cudaError_t e = set_smem(k4_tlq_dq_reduce_q<BIN, BOUT, STOCH, REMOTE, G64>, SMEM);
  if (e != cudaSuccess) return e;
  uint32_t* sched = sched_counter(st);
  if (!sched) return cudaErrorMemoryAllocation;
  const uint32_t tpu = (uint32_t)((S + kK4Tile - 1) / kK4Tile);
  const uint32_t ntiles = tpu * (uint32_t)M;
  const int grid = grid_for(ntiles, sms * K4Cfg<BIN, BOUT, REMOTE>::CTAS);
  k4_tlq_dq_reduce_q<BIN, BOUT, STOCH, REMOTE, G64><<<grid, kK4Block, SMEM, st>>>(recv, in_unit_bytes, N, M, S, __builtin_ctz(G),
                                                                dst, tpu, ntiles, -0.0f, sr, l_self, sr_stride, sr_off,
                                                                pull, 16u, sched);
  return cudaGetLastError();
}
template <int BIN, int BOUT, bool STOCH>
cudaError_t k4_launch_t(const uint8_t* recv, size_t in_unit_bytes, int N, int M, size_t S, int G, const Dests& dst,
                        const SR& sr, int l_self, size_t sr_stride, size_t sr_off, int sms, cudaStream_t st,
                        const K4Pull& pull) {
#define K4V(RM, GB) return k4_launch_v<BIN, BOUT, STOCH, RM, GB>(recv, in_unit_bytes, N, M, S, G, dst, sr, l_self, \
                                                               sr_stride, sr_off, sms, st, pull)
  if (dst.remote) {
    if (G >= 64) K4V(true, true); else K4V(true, false);
  } else {
    if (G >= 64) K4V(false, true); else K4V(false, false);
  }
#undef K4V
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


}  // namespace sdp4
