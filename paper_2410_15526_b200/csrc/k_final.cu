// k_final.cu -- K5 tlq_dq_reduce_had (Alg. 3 l.11-13) and the P2P flag-wait kernel.
#include "sdp4_device.cuh"

namespace sdp4 {
namespace {

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


}  // namespace

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
