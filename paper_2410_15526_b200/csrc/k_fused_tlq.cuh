// k_fused_tlq.cuh -- the one-launch TLq-HS kernel (instantiated per intra bit width by
// k_fused_tlq8.cu and k_fused_tlq4.cu, compiled in parallel).
#pragma once
#include "k_fused.cuh"

namespace sdp4 {
namespace {

// =====================================================================================
// One-launch TLq-HS.  Warp tasks of 32 rows of 64 elements (2048 elements; lane = one row =
// 64 contiguous elements, which is both K3/K5's row layout and K4's vector layout):
//  A (v, shard j, row block)  K3: rows loaded straight from the gradient, butterfly + quantize
//     (fwht_pairs, quant_row) into the warp's smem tile, copied to unit m' of block l of rank
//     (m, l')'s intra receive region (j = m'N + l');
//  B (v, unit m', block)      K4: N sources l'' in order, dequantize + fp32 reduce + requantize,
//     staged in smem and copied to slot m of rank (m', l)'s inter receive region;
//  C (v, row block)           K5: M sources m'' in order, dequantize + reduce, inverse butterfly,
//     * kappa, the fp32 output rows (through smem, whole-sector stores).
// Degenerate axes skip an exchange and a phase: with N = 1 the intra all-to-all is the identity,
// so an A task feeds its own smem tile straight into B's arithmetic (A+B); with M = 1 the inter
// one is, so a B task feeds C's (B+C).  Same operations in the same order -- bit-identical.
// Flags: stage 1 (intra) and 2 (inter), as the multi-launch P2P path.
// =====================================================================================

// A: one lane's row of shard j (grad dtype bf16 or fp32) -> p[i] = {v[i], v[i+32]}
__device__ __forceinline__ void load_row(const FtlqArgs& a, int v, size_t off, bool act, float2* p) {
  if (act && a.grad_bf16) {
    const uint16_t* g = static_cast<const uint16_t*>(a.grad[v]) + off;
#pragma unroll
    for (int c = 0; c < 8; ++c) {  // 16-byte chunk c = elements 8c..8c+7
      const uint4 u = *reinterpret_cast<const uint4*>(g + 8 * c);
      float2* dd = p + 8 * (c & 3);
      if (c < 4) {
        dd[0].x = bf16_lo(u.x); dd[1].x = bf16_hi(u.x); dd[2].x = bf16_lo(u.y); dd[3].x = bf16_hi(u.y);
        dd[4].x = bf16_lo(u.z); dd[5].x = bf16_hi(u.z); dd[6].x = bf16_lo(u.w); dd[7].x = bf16_hi(u.w);
      } else {
        dd[0].y = bf16_lo(u.x); dd[1].y = bf16_hi(u.x); dd[2].y = bf16_lo(u.y); dd[3].y = bf16_hi(u.y);
        dd[4].y = bf16_lo(u.z); dd[5].y = bf16_hi(u.z); dd[6].y = bf16_lo(u.w); dd[7].y = bf16_hi(u.w);
      }
    }
  } else if (act) {
    const float* g = static_cast<const float*>(a.grad[v]) + off;
#pragma unroll
    for (int c = 0; c < 16; ++c) {  // chunk c = elements 4c..4c+3
      const float4 u = *reinterpret_cast<const float4*>(g + 4 * c);
      float2* dd = p + 4 * (c & 7);
      if (c < 8) {
        dd[0].x = u.x; dd[1].x = u.y; dd[2].x = u.z; dd[3].x = u.w;
      } else {
        dd[0].y = u.x; dd[1].y = u.y; dd[2].y = u.z; dd[3].y = u.w;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i) p[i] = make_float2(0.f, 0.f);
  }
}

// B: fold one source's 64 BI-bit codes of this lane into acc (K4's arithmetic, slot order =
// element order).  codes: the lane's 64 codes; sc: the unit's (or tile's) scale array and el
// the lane's first element index in it.
template <int BI, bool FIRST>
__device__ __forceinline__ void b_source(const uint8_t* codes, const float* sc, size_t el, int lg, float z,
                                         float2* acc) {
  constexpr int CPT = 64 * BI / 8 / 16, EPC = 64 / CPT;
  constexpr float qin = float((1 << (BI - 1)) - 1);
  const float rqin = __fdiv_rn(1.f, qin);
  float ds0, ds1;
  if (lg >= 6) {
    ds0 = ds1 = div_by_q(sc[el >> lg], qin, rqin);
  } else {
    ds0 = div_by_q(sc[el >> 5], qin, rqin);
    ds1 = div_by_q(sc[(el >> 5) + 1], qin, rqin);
  }
  k4_item<BI, CPT, EPC, FIRST>(codes, ds0, ds1, 0, z, acc);
}

// B: requantize acc at BE bits (K4's arithmetic) into the warp's smem staging: the lane's 64
// codes at lane * 64 * BE / 8 (row tile of R = 8 * BE bytes), its group scales at index
// (64 * lane) >> lg.  i0: global stochastic-rounding index of the lane's first element.
template <int BE, bool STOCH>
__device__ __forceinline__ void b_requant(const float2* acc, int lane, int lg, bool act, uint32_t key, uint64_t i0,
                                          uint32_t m16, uint8_t* sc_codes, float* sc_sc) {
  constexpr float qout = float((1 << (BE - 1)) - 1);
  constexpr float magic = BE == 4 ? kMagicB4 : kMagic;
  const int tpg = lg >= 6 ? (1 << (lg - 6)) : 1;
  float am[4];
#pragma unroll
  for (int vq = 0; vq < 4; ++vq) {
    float x = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) x = max3_abs_nan(x, acc[8 * vq + k].x, acc[8 * vq + k].y);
    am[vq] = x;
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
  } else {  // G == 32: elements 0..31 and 32..63 of the lane are two groups
    a0 = max_nan(am[0], am[1]);
    a1 = max_nan(am[2], am[3]);
    p0 = qparam(a0, qout);
    p1 = qparam(a1, qout);
  }
  if (!act) return;
#pragma unroll
  for (int vq = 0; vq < 4; ++vq) {
    const bool h = vq >= 2;
    const float iv = h ? p1.inv : p0.inv;
    uint32_t rr[16];
    if constexpr (STOCH) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        rr[2 * k] = rq_sr(acc[8 * vq + k].x, iv, sr_u(i0 + 16 * vq + 2 * k, key), qout, magic);
        rr[2 * k + 1] = rq_sr(acc[8 * vq + k].y, iv, sr_u(i0 + 16 * vq + 2 * k + 1, key), qout, magic);
      }
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float2 y = f2rq(acc[8 * vq + k], make_float2(iv, iv), magic);
        rr[2 * k] = __float_as_uint(y.x);
        rr[2 * k + 1] = __float_as_uint(y.y);
      }
    }
    const bool okv = h ? p1.ok : p0.ok;
    if constexpr (BE == 4) {
      uint2 w = make_uint2(pack4x8_b(rr, m16), pack4x8_b(rr + 8, m16));
      if (!okv) w = make_uint2(0u, 0u);
      *reinterpret_cast<uint2*>(sc_codes + lane * 32 + 8 * vq) = w;
    } else {
      uint4 w = make_uint4(pack8x4(rr[0], rr[1], rr[2], rr[3]), pack8x4(rr[4], rr[5], rr[6], rr[7]),
                           pack8x4(rr[8], rr[9], rr[10], rr[11]), pack8x4(rr[12], rr[13], rr[14], rr[15]));
      if (!okv) w = make_uint4(0u, 0u, 0u, 0u);
      *reinterpret_cast<uint4*>(sc_codes + lane * 64 + 16 * vq) = w;
    }
  }
  if (lg >= 6) {
    if ((lane & (tpg - 1)) == 0) sc_sc[(64 * lane) >> lg] = stored_scale(a0, 1.f);
  } else {
    *reinterpret_cast<float2*>(sc_sc + 2 * lane) = make_float2(stored_scale(a0, 1.f), stored_scale(a1, 1.f));
  }
}

// Copy a staged tile (cbytes code bytes, nsc scales) to its place in a unit, 16-byte stores.
__device__ __forceinline__ void copy_tile(uint8_t* g_codes, float* g_sc, const uint8_t* s_codes, const float* s_sc,
                                          uint32_t cbytes, uint32_t nsc, int lane) {
  uint4* gc = reinterpret_cast<uint4*>(g_codes);
  const uint4* s4 = reinterpret_cast<const uint4*>(s_codes);
  for (uint32_t k = lane; k < cbytes / 16; k += 32) gc[k] = s4[k];
  for (uint32_t k = lane; k < nsc; k += 32) g_sc[k] = s_sc[k];
}

// C: dequantize one source's row (linear row tile), fold into acc (K5's arithmetic).
template <int BE, bool FIRST>
__device__ __forceinline__ void c_source(const uint8_t* tile, const float* sc, int row, int lg, float z,
                                         float2* acc) {
  constexpr int RE = kRowElems * BE / 8;
  constexpr float qe = float((1 << (BE - 1)) - 1);
  const float rqe = __fdiv_rn(1.f, qe);
  float ds0, ds1;
  if (lg >= 6) {
    ds0 = ds1 = div_by_q(sc[row >> (lg - 6)], qe, rqe);
  } else {
    const float2 s2 = *reinterpret_cast<const float2*>(sc + 2 * row);
    ds0 = div_by_q(s2.x, qe, rqe);
    ds1 = div_by_q(s2.y, qe, rqe);
  }
  dequant_row_adj<BE, RE, kFtRows, !FIRST, true>(tile, row, ds0, ds1, z, acc);
}

// C: inverse butterfly, * kappa, and the warp's rows to the output through the smem tile in
// four passes of 16 elements: a store instruction writes 8 rows x 64 contiguous bytes (whole
// sectors) instead of 32 scattered 16-byte pieces.
template <int B>
__device__ __forceinline__ void c_finish(float2* acc, float kappa, uint8_t* tile, float* orow0, uint32_t nrow,
                                         int lane) {
  fwht_adj<B>(acc);
  const float2 kk = make_float2(kappa, kappa);
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = f2mul(acc[i], kk);
  float4* st4 = reinterpret_cast<float4*>(tile);
#pragma unroll
  for (int qp = 0; qp < 4; ++qp) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = 4 * qp + k;  // elements 4c..4c+3 = pairs 2c, 2c+1
      st4[lane * 4 + k] = make_float4(acc[2 * c].x, acc[2 * c].y, acc[2 * c + 1].x, acc[2 * c + 1].y);
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = 32 * i + lane, rr = k >> 2, pc = k & 3;
      if ((uint32_t)rr < nrow) *reinterpret_cast<float4*>(orow0 + (size_t)rr * kRowElems + 16 * qp + 4 * pc) = st4[k];
    }
    __syncwarp();
  }
}

template <int BI, int BE, int B, bool STOCH>
__global__ void __launch_bounds__(kFThreads) kf_tlq(const FusedSync fs, const FtlqArgs a) {
  constexpr int RI = kRowElems * BI / 8;   // intra row bytes
  constexpr int RE = kRowElems * BE / 8;   // inter row bytes
  constexpr int OUT_W = kFtRows * 64 + 64 * 4;  // a warp's staged codes (<= 8-bit) + scales
  __shared__ __align__(16) uint8_t stage[kFThreads / 32][OUT_W];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nv = fs.nv, M = a.M, N = a.N, P = fs.P;
  const size_t S = a.S;
  const uint32_t rows = (uint32_t)(S / kRowElems);
  const uint32_t RB = (rows + kFtRows - 1) / kFtRows;  // row blocks (= K4 blocks of 2048 elements)
  const bool ab = N == 1, bc = M == 1;                 // fused phases on a degenerate axis
  const uint32_t TA1 = RB * (uint32_t)P, TB1 = ab ? 0u : RB * (uint32_t)M, TC1 = bc ? 0u : RB;
  const uint32_t TA = TA1 * nv, TB = TB1 * nv, TC = TC1 * nv;
  const size_t intra_bytes = (size_t)N * M * a.w8;
  const int lg = a.lg;
  uint64_t free4_ok = 0;  // bit v * P + d: node peer d's free flag seen
  uint32_t free8_ok = 0, data8_ok = 0, data4_ok = 0, doneA_ok = 0, doneB_ok = 0;  // per vrank bits
  uint8_t* ot = stage[warp];
  float* osc = reinterpret_cast<float*>(ot + kFtRows * 64);  // staged scales (A and B layouts)
  const int tunit = blockIdx.x * (kFThreads / 32) + warp;     // trace slot block of this warp
  if (lane == 0) tstamp(fs, tunit, 0);

  // B's tail shared by B tasks and fused A+B tasks: wait until node peer d is done with the
  // previous push, requantize into the staging tile, copy it to slot m of d's inter region
  auto b_out = [&](const float2* acc, int v, int r, int m, int l, uint32_t mp, size_t e0) {
    const int d = (int)mp * N + l;  // destination rank: (m', l)
    if (lane == 0 && d != r && !((free4_ok >> (v * P + d)) & 1ull))
      wait_flag(fs, flag(fs, r, kFlagFree, 2, d), wait_code(kFlagFree, 2, d));
    if (d != r) free4_ok |= 1ull << (v * P + d);
    __syncwarp();  // (also: every lane is done reading the smem tile that b_requant overwrites)
    const bool act = e0 + 64 * lane < S;
    b_requant<BE, STOCH>(acc, lane, lg, act, a.key4[v], (uint64_t)(mp * N + l) * S + e0 + 64 * lane, a.m16, ot, osc);
    __syncwarp();
    uint8_t* unit4 = fs.region[d] + intra_bytes + (size_t)m * a.w4;
    const uint32_t nact = (uint32_t)min((size_t)32, (S - e0) / 64);  // lanes with elements (S % 64 == 0)
    copy_tile(unit4 + e0 * BE / 8, reinterpret_cast<float*>(unit4 + S * BE / 8) + (e0 >> lg), ot, osc,
              nact * 64 * BE / 8, (nact * 64) >> lg, lane);
  };
  // raises of the last task of a phase: resets of this rank's own consumed flags, then one
  // system-scope fence and the peers' flags (release pattern)
  auto raise_intra_data = [&](int r, int m) {  // A done: my blocks are in the group peers' regions
    for (int q2 = 0; q2 < N; ++q2)
      if (m * N + q2 != r) st_relaxed_sys(flag(fs, r, kFlagFree, 1, m * N + q2), 0u);
    __threadfence_system();
    for (int q2 = 0; q2 < N; ++q2)
      if (m * N + q2 != r) st_relaxed_sys(flag(fs, m * N + q2, kFlagData, 1, r), 1u);
  };
  auto raise_b_done = [&](int r, int m, int l) {  // B done: intra region consumed, inter units pushed
    for (int q2 = 0; q2 < N; ++q2)
      if (m * N + q2 != r) st_relaxed_sys(flag(fs, r, kFlagData, 1, m * N + q2), 0u);
    for (int q2 = 0; q2 < M; ++q2)
      if (q2 * N + l != r) st_relaxed_sys(flag(fs, r, kFlagFree, 2, q2 * N + l), 0u);
    __threadfence_system();
    for (int q2 = 0; q2 < N; ++q2)
      if (m * N + q2 != r) st_relaxed_sys(flag(fs, m * N + q2, kFlagFree, 1, r), 1u);
    for (int q2 = 0; q2 < M; ++q2)
      if (q2 * N + l != r) st_relaxed_sys(flag(fs, q2 * N + l, kFlagData, 2, r), 1u);
  };

  for (;;) {
    uint32_t task = 0;
    if (lane == 0) task = atomicAdd(fs.ctr, 1u);
    task = __shfl_sync(0xffffffffu, task, 0);
    if (task >= TA + TB + TC) break;
    if (task < TA) {  // ---------------- phase A (K3), with N = 1 also B (K4)
      const int v = (int)(task % nv);
      const uint32_t rest = task / nv;
      const uint32_t j = rest % (uint32_t)P, rb = rest / (uint32_t)P;
      const int r = fs.rank[v], m = r / N, l = r % N;
      const int lp = (int)j % N, mp = (int)j / N;
      if (lane == 0) tstamp(fs, tunit, 2);
      if (lane == 0 && !((free8_ok >> v) & 1u)) {  // every group peer is done with my previous pushes
        for (int q2 = 0; q2 < N; ++q2)
          if (m * N + q2 != r) wait_flag(fs, flag(fs, r, kFlagFree, 1, m * N + q2), wait_code(kFlagFree, 1, m * N + q2));
      }
      free8_ok |= 1u << v;
      __syncwarp();
      const uint32_t row = rb * kFtRows + lane;
      const bool act = row < rows;
      float2 p[32];
      load_row(a, v, (size_t)j * S + (size_t)row * kRowElems, act, p);
      fwht_pairs<B>(p);
      const SR sr{a.sr_on, a.key8[v]};
      quant_row<BI, RI, true, STOCH>(p, lane, lg, a.cb, act, ot, osc, sr, (uint64_t)j * S + (uint64_t)row * kRowElems);
      __syncwarp();
      const uint32_t nrow = min((uint32_t)kFtRows, rows - rb * kFtRows);
      if (ab) {  // N = 1: the intra exchange is the identity -- B on the tile just quantized
        float2 acc[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[i] = make_float2(0.f, 0.f);
        if (act) b_source<BI, true>(ot + lane * RI, osc, (size_t)64 * lane, lg, a.z, acc);
        b_out(acc, v, r, m, l, (uint32_t)mp, (size_t)rb * kFtTask);
      } else {
        const int d = m * N + lp;  // destination rank: (m, l')
        uint8_t* unit = fs.region[d] + (size_t)l * M * a.w8 + (size_t)mp * a.w8;
        copy_tile(unit + (size_t)rb * kFtRows * RI,
                  reinterpret_cast<float*>(unit + S * BI / 8) + (((size_t)rb * kFtRows * kRowElems) >> lg), ot, osc,
                  nrow * RI, (nrow * kRowElems) >> lg, lane);
      }
      __syncwarp();
      if (lane == 0) tstamp(fs, tunit, 3);
      if (lane == 0 && finish_task(fs, 0, v, TA1)) {
        if (ab) raise_b_done(r, m, l);
        else raise_intra_data(r, m);
      }
      __syncwarp();  // ot is rewritten by the next task
    } else if (task < TA + TB) {  // ---------------- phase B (K4), with M = 1 also C (K5)
      const uint32_t bt = task - TA;
      const int v = (int)(bt % nv);
      const uint32_t rest = bt / nv;
      const uint32_t mp = rest % (uint32_t)M, tb = rest / (uint32_t)M;
      const int r = fs.rank[v], m = r / N, l = r % N;
      if (lane == 0) {
        if (!((data8_ok >> v) & 1u))
          for (int q2 = 0; q2 < N; ++q2)
            if (m * N + q2 != r) wait_flag(fs, flag(fs, r, kFlagData, 1, m * N + q2), wait_code(kFlagData, 1, m * N + q2));
        if (!((doneA_ok >> v) & 1u)) wait_done(fs, 0, v, TA1);  // this rank's own block is written
      }
      data8_ok |= 1u << v;
      doneA_ok |= 1u << v;
      if (lane == 0) tstamp(fs, tunit, 4);
      __syncwarp();
      const size_t e0 = (size_t)tb * kFtTask, e = e0 + 64 * lane;
      const bool act = e < S;
      float2 acc[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) acc[i] = make_float2(0.f, 0.f);
      if (act) {
        for (int ls = 0; ls < N; ++ls) {  // sources l'' = 0..N-1 in order (R8)
          const uint8_t* unit = fs.region[r] + ((size_t)ls * M + mp) * a.w8;
          const float* sc = reinterpret_cast<const float*>(unit + S * BI / 8);
          if (ls == 0) b_source<BI, true>(unit + e * BI / 8, sc, e, lg, a.z, acc);
          else b_source<BI, false>(unit + e * BI / 8, sc, e, lg, a.z, acc);
        }
      }
      if (bc) {  // M = 1: the inter exchange is the identity -- C on the requantized tile
        __syncwarp();
        b_requant<BE, STOCH>(acc, lane, lg, act, a.key4[v], (uint64_t)(mp * N + l) * S + e, a.m16, ot, osc);
        __syncwarp();
        float2 c[32];
        if (act) c_source<BE, true>(ot, osc, lane, lg, a.z, c);
        else {
#pragma unroll
          for (int i = 0; i < 32; ++i) c[i] = make_float2(0.f, 0.f);
        }
        __syncwarp();  // the tile is reused by c_finish's transpose
        c_finish<B>(c, a.kappa, ot, a.out[v] + e0, min((uint32_t)kFtRows, rows - tb * kFtRows), lane);
      } else {
        b_out(acc, v, r, m, l, mp, e0);
      }
      __syncwarp();
      if (lane == 0) tstamp(fs, tunit, 5);
      if (lane == 0 && finish_task(fs, 1, v, TB1)) raise_b_done(r, m, l);
      __syncwarp();
    } else {  // ---------------- phase C (K5)
      const uint32_t ct = task - TA - TB;
      const int v = (int)(ct % nv);
      const uint32_t rb = ct / nv;
      const int r = fs.rank[v], l = r % N;
      if (lane == 0) {
        if (!((data4_ok >> v) & 1u))
          for (int q2 = 0; q2 < M; ++q2)
            if (q2 * N + l != r) wait_flag(fs, flag(fs, r, kFlagData, 2, q2 * N + l), wait_code(kFlagData, 2, q2 * N + l));
        if (!((doneB_ok >> v) & 1u)) {  // this rank's own slot is written (by B, or by A+B)
          if (ab) wait_done(fs, 0, v, TA1);
          else wait_done(fs, 1, v, TB1);
        }
      }
      data4_ok |= 1u << v;
      doneB_ok |= 1u << v;
      if (lane == 0) tstamp(fs, tunit, 6);
      __syncwarp();
      const uint32_t row = rb * kFtRows + lane;
      const bool act = row < rows;
      float2 acc[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) acc[i] = make_float2(0.f, 0.f);
      if (act) {
        for (int ms = 0; ms < M; ++ms) {  // sources m'' = 0..M-1 in order (R8)
          const uint8_t* unit = fs.region[r] + intra_bytes + (size_t)ms * a.w4;
          const float* sc = reinterpret_cast<const float*>(unit + S * BE / 8);
          if (ms == 0) c_source<BE, true>(unit, sc, (int)row, lg, a.z, acc);
          else c_source<BE, false>(unit, sc, (int)row, lg, a.z, acc);
        }
      }
      // every lane's reads of the inter slots are done (their values are in acc): the last
      // task to get here frees the slots for the peers' next call -- before the butterfly and
      // the stores, so the fence and raises overlap the tail of the kernel
      __syncwarp();
      if (lane == 0 && finish_task(fs, 2, v, TC1)) {
        for (int q2 = 0; q2 < M; ++q2)
          if (q2 * N + l != r) st_relaxed_sys(flag(fs, r, kFlagData, 2, q2 * N + l), 0u);
        __threadfence_system();
        for (int q2 = 0; q2 < M; ++q2)
          if (q2 * N + l != r) st_relaxed_sys(flag(fs, q2 * N + l, kFlagFree, 2, r), 1u);
      }
      c_finish<B>(acc, a.kappa, ot, a.out[v] + (size_t)rb * kFtTask, min((uint32_t)kFtRows, rows - rb * kFtRows),
                  lane);
      __syncwarp();
      if (lane == 0) tstamp(fs, tunit, 7);
    }
  }
  if (lane == 0) {
    tstamp(fs, tunit, 1);
    exit_unit(fs, gridDim.x * (kFThreads / 32));
  }
}

template <int BI, int BE>
cudaError_t fused_tlq_b(const FusedSync& fs, const FtlqArgs& a, int b, bool stoch, int grid, cudaStream_t st) {
#define KT(BB)                                                                  \
  do {                                                                          \
    if (stoch) kf_tlq<BI, BE, BB, true><<<grid, kFThreads, 0, st>>>(fs, a);     \
    else kf_tlq<BI, BE, BB, false><<<grid, kFThreads, 0, st>>>(fs, a);          \
  } while (0)
  switch (b) {
    case 0: KT(0); break;
    case 2: KT(2); break;
    case 4: KT(4); break;
    case 8: KT(8); break;
    case 16: KT(16); break;
    case 32: KT(32); break;
    case 64: KT(64); break;
    case 128: KT(128); break;
    case 256: KT(256); break;
    default: return cudaErrorInvalidValue;
  }
#undef KT
  return cudaGetLastError();
}

}  // namespace
}  // namespace sdp4
