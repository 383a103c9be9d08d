// k_had_quant.cu -- K3 tlq_had_quant: blockwise Hadamard + quantize (Alg. 3 l.2-3, fused P:394-395).
#include "sdp4_device.cuh"

namespace sdp4 {
namespace {

constexpr int kK3Warps = kTileRows / 32;          // consumer warps (one row per thread)
constexpr int kK3Block = kTileRows + 32;          // + the producer warp
constexpr int kK3Chunk = 2;                       // tiles per scheduler claim
constexpr uint32_t kK3NoTile = 0xffffffffu;

template <int IN_R, int OUT_R>
struct K3Cfg {
  static constexpr int CTAS = IN_R == 128 ? 2 : 1;  // bf16 gradients: two CTAs per SM
  static constexpr int IN_TILE = kTileRows * IN_R;
  // one warp's output: 32 rows of codes + its scales (G >= 32: at most 64), 1024-aligned
  // (TMA swizzle atoms); double-buffered per warp
  static constexpr int OUT_W = (32 * OUT_R + 256 + 1023) / 1024 * 1024;
  static constexpr int BUDGET = CTAS == 2 ? 110 * 1024 : 200 * 1024;
  static constexpr int OB = 2 * kK3Warps * OUT_W + 2 * IN_TILE <= BUDGET ? 2 : 1;  // output tiles per warp
  static constexpr int OUT_BYTES = OB * kK3Warps * OUT_W;
  static constexpr int S0 = (BUDGET - OUT_BYTES) / IN_TILE;
  static constexpr int STAGES = S0 > 4 ? 4 : (S0 < 2 ? 2 : S0);
  static constexpr int SMEM = STAGES * IN_TILE + OUT_BYTES + 2 * 8 * STAGES + 4 * STAGES + 1024;
  static_assert(SMEM <= 227 * 1024, "K3 tile configuration exceeds the per-CTA shared memory");
};

// =====================================================================================
// K3  TLq-HS Hadamard + quantize (Alg. 3 l.2-3; fused per P:394-395).
// Persistent CTAs (one per SM), warp-specialized: a producer warp claims tiles (256 rows of
// 64 elements of one shard j) from the dynamic scheduler and keeps a STAGES-deep ring of TMA
// tensor loads in flight (full / empty mbarriers); every consumer thread butterflies its own
// row in f32x2 registers and quantizes it into its warp's double-buffered output tile, and
// each warp stores its own 32 rows to unit m' = j / N of the block for local rank l' = j % N
// (R9) -- a TMA tensor store into a local block, or 1-D bulk copies into the receive buffer of
// a peer, where the store IS the intra all-to-all (Alg. 3 l.4) over NVLink.  No barrier spans
// more than one warp after the prologue.
// =====================================================================================
// Output of K3: per destination local rank l', the block this rank sends to l' (peer
// receive buffer or local send buffer); unit m' at blk + m' * unit_bytes.
struct K3Out {
  CUtensorMap map[kMaxN];   // valid for local blocks: M units of that block (32-row boxes)
  CUtensorMap omap[kMaxN];  // outbox blocks (pulled tiles, IntraPull), local memory
  uint8_t* blk[kMaxN];
  uint8_t* oblk[kMaxN];
  uint32_t remote;          // bit l': block l' lives in a peer's memory (P2P push)
  uint32_t pmask;           // bit l': some tiles for l' are pulled (IntraPull)
  uint32_t pnum, pden;
};

// One warp's 32 output rows to a peer (or any linear destination): codes with one 1-D bulk
// copy by lane 0, scales with a bulk copy when 16-byte aligned and sized, else by lanes.
__device__ __forceinline__ void store_warp_linear(const uint8_t* s_codes, uint32_t cbytes, const float* s_sc,
                                                  uint32_t nsc, uint8_t* g_codes, float* g_sc, int lane) {
  const bool sc_bulk = nsc && ((nsc & 3u) == 0) && ((reinterpret_cast<uintptr_t>(g_sc) & 15u) == 0);
  if (lane == 0) {
    if (cbytes) bulk_store(g_codes, s_codes, cbytes);
    if (sc_bulk) bulk_store(g_sc, s_sc, nsc * 4);
    bulk_commit();
  }
  if (!sc_bulk)
    for (uint32_t k = lane; k < nsc; k += 32) g_sc[k] = s_sc[k];
}

template <int IN_R, int BITS, int B, bool STOCH>
__global__ void __launch_bounds__(kK3Block, K3Cfg<IN_R, kRowElems * BITS / 8>::CTAS)
    k3_tlq_had_quant(const __grid_constant__ CUtensorMap in_map, const __grid_constant__ K3Out out, size_t S, int M,
                     int N, int lg, float cb, size_t unit_bytes, uint32_t tps, uint32_t ntiles, const SR sr,
                     size_t sr_stride, size_t sr_off, uint32_t* sched) {
  constexpr int OUT_R = kRowElems * BITS / 8;
  using C = K3Cfg<IN_R, OUT_R>;
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
  const uint32_t U = (uint32_t)(M * N);  // shards; tile = ts * U + j (shard fastest)

  if (t == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kK3Warps);
    }
    fence_mbar_init();
  }
  __syncthreads();  // the only CTA-wide barrier
  if (t >= kTileRows) {  // ---- producer warp
    if (t == kTileRows) {
      uint32_t k = 0;
      for (;;) {
        const uint32_t t0 = sched_claim(sched, kK3Chunk);
        if (t0 >= ntiles) break;
        const uint32_t t1 = min(t0 + kK3Chunk, ntiles);
        for (uint32_t tile = t0; tile < t1; ++tile, ++k) {
          const int s = k % STAGES;
          mbar_wait(&empty[s], ((k / STAGES) & 1) ^ 1);
          tile_of[s] = tile;
          mbar_arrive_tx(&full[s], C::IN_TILE);
          tma_load_tile<IN_R>(in_buf + s * C::IN_TILE, &in_map, &full[s], (int)((tile / U) * kTileRows),
                              (int)(tile % U));
        }
      }
      const int s = k % STAGES;  // end of work
      mbar_wait(&empty[s], ((k / STAGES) & 1) ^ 1);
      tile_of[s] = kK3NoTile;
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
    if (tile == kK3NoTile) break;
    const uint32_t ts = tile / U, j = tile - ts * U;
    const uint32_t row = ts * kTileRows + t;       // this thread's row of shard j
    const bool act = row < rows_per_shard;
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
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // this warp's rows of stage s are in registers

    fwht_pairs<B>(p);

    const uint32_t lp = j % N, mp = j / N;  // shard j = m'N + l' goes to local rank l', unit m' (R9)
    uint8_t* ot = ob0 + (i % C::OB) * C::OUT_W;
    float* osc = reinterpret_cast<float*>(ot + 32 * OUT_R);
    const bool pull = ((out.pmask >> lp) & 1u) && ts % out.pden < out.pnum;  // kept in the outbox
    uint8_t* unit = (pull ? out.oblk[lp] : out.blk[lp]) + mp * unit_bytes;
    const bool remote = !pull && ((out.remote >> lp) & 1u);  // CTA-uniform
    if (lane == 0) bulk_wait_read<C::OB - 1>();  // this warp's store of tile i - OB has left ot
    __syncwarp();
    const uint32_t wrow0 = ts * kTileRows + 32 * warp;  // the warp's first row in the shard
    if constexpr (BITS == 32) {  // identity codec (R12): rn(u * c_b)
      const float2 cc = make_float2(cb, cb);
#pragma unroll
      for (int i2 = 0; i2 < 32; ++i2) p[i2] = f2mul(p[i2], cc);
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const float2* q = p + 4 * (c & 7);
        *reinterpret_cast<float4*>(ot + (remote ? lane * 256 + 16 * c : tile_off<256, 32>(lane, c))) =
            c < 8 ? make_float4(q[0].x, q[1].x, q[2].x, q[3].x) : make_float4(q[0].y, q[1].y, q[2].y, q[3].y);
      }
    } else {
      const uint64_t i0 = (uint64_t)j * sr_stride + sr_off + (uint64_t)row * kRowElems;
      if (remote) {  // peer block: linear rows, codes + scales bulk-stored over NVLink
        quant_row<BITS, OUT_R, true, STOCH>(p, lane, lg, cb, act, ot, osc, sr, i0);
      } else {       // local block: swizzled rows for the TMA tensor store, scales direct
        float* gsc = reinterpret_cast<float*>(unit + S * BITS / 8) + (((size_t)wrow0 * kRowElems) >> lg);
        quant_row<BITS, OUT_R, false, STOCH>(p, lane, lg, cb, act, ot, gsc, sr, i0);
      }
    }
    fence_proxy_async();
    __syncwarp();
    if (wrow0 < rows_per_shard) {
      if (remote) {
        const uint32_t rows = min(32u, rows_per_shard - wrow0);
        const uint32_t nsc = BITS == 32 ? 0u : ((rows * kRowElems) >> lg);
        store_warp_linear(ot, rows * OUT_R, osc, nsc, unit + (size_t)wrow0 * OUT_R,
                          reinterpret_cast<float*>(unit + S * BITS / 8) + (((size_t)wrow0 * kRowElems) >> lg), lane);
      } else if (lane == 0) {
        tma_store_tile<OUT_R, 32>(pull ? &out.omap[lp] : &out.map[lp], ot, (int)wrow0, (int)mp);
        bulk_commit();
      }
    }
  }
  if (lane == 0) bulk_wait<0>();
}


template <int IN_R, int BITS, int B, bool STOCH>
cudaError_t k3_launch_t(const CUtensorMap& in_map, const K3Out& out, size_t S, int M, int N, int G, float cb,
                        size_t unit_bytes, uint32_t tps, uint32_t ntiles, int grid, const SR& sr, size_t sr_stride,
                        size_t sr_off, cudaStream_t st) {
  constexpr int SMEM = K3Cfg<IN_R, kRowElems * BITS / 8>::SMEM;
  cudaError_t e = set_smem(k3_tlq_had_quant<IN_R, BITS, B, STOCH>, SMEM);
  if (e != cudaSuccess) return e;
  uint32_t* sched = sched_counter(st);
  if (!sched) return cudaErrorMemoryAllocation;
  k3_tlq_had_quant<IN_R, BITS, B, STOCH><<<grid, kK3Block, SMEM, st>>>(in_map, out, S, M, N, __builtin_ctz(G), cb,
                                                                        unit_bytes, tps, ntiles, sr, sr_stride, sr_off,
                                                                        sched);
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


}  // namespace

cudaError_t launch_tlq_had_quant(const void* grad, size_t grad_stride, int grad_dtype, size_t S, int M, int N,
                                 int G, int b, float cb, int bits, uint8_t* const* blocks, uint32_t remote_mask,
                                 size_t unit_bytes, int sr_on, uint32_t sr_key, size_t sr_off, int sms,
                                 cudaStream_t st, const IntraPull* pull) {
  const SR sr{sr_on, sr_key};
  if (N > kMaxN) return cudaErrorInvalidValue;
  const uint64_t rows = S / kRowElems;
  const uint32_t tps = (uint32_t)((rows + kTileRows - 1) / kTileRows);
  const uint32_t ntiles = tps * (uint32_t)(M * N);
  const int grid = grid_for(ntiles, sms * (grad_dtype == kBF16 ? 2 : 1));  // K3Cfg::CTAS
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
      e = make_row_map(&out.map[lp], blocks[lp], out_r, rows, (uint64_t)M, unit_bytes, 32);  // per-warp stores
      if (e != cudaSuccess) return e;
    }
    if ((out.pmask >> lp) & 1u) {
      out.oblk[lp] = pull->outbox[lp];
      e = make_row_map(&out.omap[lp], pull->outbox[lp], out_r, rows, (uint64_t)M, unit_bytes, 32);
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


}  // namespace sdp4
