// k_final.cu -- K5 tlq_dq_reduce_had (Alg. 3 l.11-13) and the P2P flag-wait kernel.
#include "sdp4_device.cuh"

#include <atomic>
#include <mutex>

namespace sdp4 {
namespace {

// =====================================================================================
// K5  TLq-HS dequantize + reduce + inverse Hadamard (Alg. 3 l.11-13; H after
// the final reduction).  Row layout, one 64-element row per consumer thread.
// Warp-specialized: a producer warp streams (tile, source m'') items through a STAGES-deep
// ring (TMA tensor load of the 128 code rows + 1-D bulk copy of the scales), each slot
// guarded by a "full" mbarrier (transaction bytes) and an "empty" mbarrier the four consumer
// warps arrive on.  Sources are summed in order m'' = 0..M-1 (R8); out = rn(H_unnorm(acc) *
// kappa) (R8).  Each consumer warp transposes its own 32 output rows through a swizzled smem
// tile and writes them with coalesced 16-byte stores (the warp's rows are 8 KB of contiguous
// output): no barrier spans more than one warp, and the TMA unit carries only the loads (TMA
// stores of the fp32 output, 88% of K5's bytes, back-pressured the loads behind them).
// =====================================================================================
constexpr int kK5Rows = 128;   // rows per input tile = consumer threads per CTA
constexpr int kK5Block = kK5Rows + 32;  // + the producer warp
constexpr int kK5Ctas = 2;
constexpr int kK5WarpRows = 32;  // rows per consumer warp (its own output tile)
constexpr int kK5Chunk = 4;      // tiles per scheduler claim (128 KB of output)
constexpr uint32_t kNoTile = 0xffffffffu;

template <int IN_R>
struct K5Cfg {
  static constexpr int IN_TILE = kK5Rows * IN_R;
  static constexpr int SC_BYTES = kK5Rows * 64 / 32 * 4;  // G >= 32
  static constexpr int STAGE = (IN_TILE + SC_BYTES + 1023) / 1024 * 1024;  // 1024-aligned (TMA swizzle atoms)
  static constexpr int OUT_WARP = kK5WarpRows * 256;  // one warp's output rows (fp32)
  static constexpr int OUT_BYTES = (kK5Rows / kK5WarpRows) * OUT_WARP;   // one transpose tile per warp
  static constexpr int S0 = (110 * 1024 - OUT_BYTES) / STAGE;  // ~110 KB per CTA: kK5Ctas per SM
  static constexpr int STAGES = S0 > 8 ? 8 : (S0 < 2 ? 2 : S0);
  static constexpr int SMEM = STAGES * STAGE + OUT_BYTES + 2 * 8 * STAGES + 4 * STAGES + 1024;
  static_assert(SMEM <= 227 * 1024, "K5 tile configuration exceeds the per-CTA shared memory");
};

template <int IN_R, int B>
__global__ void __launch_bounds__(kK5Block, kK5Ctas)
    k5_tlq_dq_reduce_had(const __grid_constant__ CUtensorMap in_map,
                         const uint8_t* __restrict__ recv, size_t in_unit_bytes, int M, size_t S, int lg, float kappa,
                         uint32_t ntiles, float z, float* __restrict__ out, uint32_t* sched) {
  constexpr int BIN = IN_R * 8 / kRowElems;
  using C = K5Cfg<IN_R>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* out_buf = smem + STAGES * C::STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(out_buf + C::OUT_BYTES);
  uint64_t* empty = full + STAGES;
  uint32_t* tile_of = reinterpret_cast<uint32_t*>(empty + STAGES);  // tile id carried by each slot
  const int t = threadIdx.x;
  const uint32_t rows_per_shard = (uint32_t)(S / kRowElems);
  if (t == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kK5Rows / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();  // the only CTA-wide barrier
  if (t >= kK5Rows) {  // ---- producer warp: one lane claims tiles and streams their (tile, source) items
    if (t == kK5Rows) {
      uint32_t k = 0;
      for (;;) {
        const uint32_t t0 = sched_claim(sched, kK5Chunk);
        if (t0 >= ntiles) break;
        const uint32_t t1 = min(t0 + kK5Chunk, ntiles);
        for (uint32_t tile = t0; tile < t1; ++tile) {
          for (int m = 0; m < M; ++m, ++k) {
            const int s = k % STAGES;
            mbar_wait(&empty[s], ((k / STAGES) & 1) ^ 1);  // the consumers released this slot
            tile_of[s] = tile;
            uint32_t sb = 0;
            if constexpr (BIN != 32) {
              const uint32_t rows = min((uint32_t)kK5Rows, rows_per_shard - tile * kK5Rows);
              sb = (((rows * kRowElems) >> lg) * 4 + 15) & ~15u;
            }
            mbar_arrive_tx(&full[s], C::IN_TILE + sb);  // release: tile_of[s] is visible with the data
            tma_load_tile<IN_R, kK5Rows>(smem + s * C::STAGE, &in_map, &full[s], (int)(tile * kK5Rows), m);
            if constexpr (BIN != 32)
              bulk_load(smem + s * C::STAGE + C::IN_TILE,
                        recv + (size_t)m * in_unit_bytes + S * BIN / 8 +
                            (((size_t)tile * kK5Rows * kRowElems) >> lg) * 4,
                        sb, &full[s]);
          }
        }
      }
      const int s = k % STAGES;  // end of work: a slot carrying no data, tile id kNoTile
      mbar_wait(&empty[s], ((k / STAGES) & 1) ^ 1);
      tile_of[s] = kNoTile;
      mbar_arrive(&full[s]);
      sched_done(sched);
    }
    return;
  }

  constexpr float qin = float((1 << (BIN == 32 ? 1 : BIN - 1)) - 1);
  const float rqin = __fdiv_rn(1.f, qin);  // rn(1/q): div_by_q's reciprocal (constant-folded)
  const int lane = t & 31, warp = t >> 5;
  uint8_t* ob = out_buf + warp * C::OUT_WARP;  // this warp's transpose tile
  uint32_t k = 0;
  for (;;) {
    uint32_t tile = 0;
    float2 acc[32];
    for (int m = 0; m < M; ++m, ++k) {
      const int s = k % STAGES;
      mbar_wait(&full[s], (k / STAGES) & 1);
      if (m == 0) {
        tile = tile_of[s];
        if (tile == kNoTile) break;
      }
      const uint8_t* st = smem + s * C::STAGE;
      float ds0 = 0.f, ds1 = 0.f;
      if constexpr (BIN != 32) {
        const float* sc = reinterpret_cast<const float*>(st + C::IN_TILE);
        if (lg >= 6) {
          ds0 = ds1 = div_by_q(sc[t >> (lg - 6)], qin, rqin);
        } else {
          const float2 s2 = *reinterpret_cast<const float2*>(sc + 2 * t);
          ds0 = div_by_q(s2.x, qin, rqin);
          ds1 = div_by_q(s2.y, qin, rqin);
        }
      }
      // R8 order; the first add 0 + x_0 is exact for quantized inputs (x_0 != -0), so source 0
      // is assigned; the identity codec keeps the add so that -0 becomes +0
      if (m == 0 && BIN != 32) {
        dequant_row_adj<BIN, IN_R, kK5Rows, false>(st, t, ds0, ds1, z, acc);
      } else {
        if (m == 0) {
#pragma unroll
          for (int q = 0; q < 32; ++q) acc[q] = make_float2(0.f, 0.f);
        }
        dequant_row_adj<BIN, IN_R, kK5Rows, true>(st, t, ds0, ds1, z, acc);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);  // this warp is done with its rows of slot s
    }
    if (tile == kNoTile) break;
    fwht_adj<B>(acc);
    const float2 kk = make_float2(kappa, kappa);
#pragma unroll
    for (int q = 0; q < 32; ++q) acc[q] = f2mul(acc[q], kk);
    // transpose through smem: lane = row, 16-byte chunk c at tile_off (conflict-free both ways)
#pragma unroll
    for (int c = 0; c < 16; ++c)  // chunk c = elements 4c..4c+3 = pairs 2c, 2c+1
      *reinterpret_cast<float4*>(ob + tile_off<256, kK5WarpRows>(lane, c)) =
          make_float4(acc[2 * c].x, acc[2 * c].y, acc[2 * c + 1].x, acc[2 * c + 1].y);
    __syncwarp();
    const uint32_t row0 = tile * kK5Rows + warp * kK5WarpRows;
    const uint32_t nrow = row0 < rows_per_shard ? min((uint32_t)kK5WarpRows, rows_per_shard - row0) : 0u;
    float* gout = out + (size_t)row0 * kRowElems;
#pragma unroll
    for (int j = 0; j < 16; ++j) {  // store j: bytes [512 j, 512 j + 512) of the warp's rows
      const int r = 2 * j + (lane >> 4), c = lane & 15;
      const float4 v = *reinterpret_cast<const float4*>(ob + tile_off<256, kK5WarpRows>(r, c));
      if ((uint32_t)r < nrow) *reinterpret_cast<float4*>(gout + r * kRowElems + 4 * c) = v;
    }
    __syncwarp();  // ob is rewritten by the next tile
  }
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


template <int IN_R, int B>
cudaError_t k5_launch(const CUtensorMap& in_map, float* out, const uint8_t* recv, size_t unit_bytes, int M, size_t S,
                      int G, float kappa, uint32_t ntiles, int grid, cudaStream_t st) {
  constexpr int SMEM = K5Cfg<IN_R>::SMEM;
  cudaError_t e = set_smem(k5_tlq_dq_reduce_had<IN_R, B>, SMEM);
  if (e != cudaSuccess) return e;
  uint32_t* sched = sched_counter(st);
  if (!sched) return cudaErrorMemoryAllocation;
  k5_tlq_dq_reduce_had<IN_R, B><<<grid, kK5Block, SMEM, st>>>(in_map, recv, unit_bytes, M, S, __builtin_ctz(G), kappa,
                                                                ntiles, -0.0f, out, sched);
  return cudaGetLastError();
}


}  // namespace

cudaError_t launch_tlq_dq_reduce_had(const uint8_t* inter_recv, size_t in_unit_bytes, int bits_in,
                                     int M, size_t S, int G, int b, float kappa, float* out,
                                     int sms, cudaStream_t st) {
  const uint64_t rows = S / kRowElems;
  const uint32_t ntiles = (uint32_t)((rows + kK5Rows - 1) / kK5Rows);
  const int grid = grid_for(ntiles, sms * kK5Ctas);
  const int in_r = kRowElems * bits_in / 8;
  CUtensorMap in_map;
  cudaError_t e = make_row_map(&in_map, inter_recv, in_r, rows, (uint64_t)M, in_unit_bytes, kK5Rows);
  if (e != cudaSuccess) return e;
#define K5(IR) SDP4_B_SWITCH(b, return (k5_launch<IR, BB>(in_map, out, inter_recv, in_unit_bytes, M, S, G, \
                                                          kappa, ntiles, grid, st)))
  if (in_r == 32) { K5(32); } else if (in_r == 64) { K5(64); } else { K5(256); }
#undef K5
  return cudaErrorInvalidValue;
}

uint32_t* sched_counter(cudaStream_t st) {
  constexpr int kSlots = 64;
  static uint32_t* pool = nullptr;
  static std::atomic<uint32_t> next{0};
  static std::once_flag once;
  std::call_once(once, [] {
    if (cudaMalloc(&pool, kSlots * 2 * sizeof(uint32_t)) == cudaSuccess) cudaMemset(pool, 0, kSlots * 2 * sizeof(uint32_t));
    else pool = nullptr;
  });
  if (!pool) return nullptr;
  uint32_t* slot = pool + 2 * (next++ % kSlots);
  return cudaMemsetAsync(slot, 0, 2 * sizeof(uint32_t), st) == cudaSuccess ? slot : nullptr;
}

cudaError_t launch_wait_flags(const FlagWait& w, cudaStream_t st) {
  if (w.n <= 0) return cudaSuccess;
  if (w.n > kMaxWait) return cudaErrorInvalidValue;
  k_wait_flags<<<1, 32, 0, st>>>(w);
  return cudaGetLastError();
}


}  // namespace sdp4
