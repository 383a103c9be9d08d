// sdp4_kernels.cuh -- internal launcher interface between the C ABI (sdp4_api.cu)
// and the sm_100a kernels (sdp4_kernels.cu).  Not part of the public ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace sdp4 {

// Every kernel is a persistent grid of at most `sms` CTAs, one CTA per SM (the rest of the
// SMs stay free for concurrent NCCL kernels).
// Rows of 64 elements are the unit of the Hadamard kernels (one row per thread).
constexpr int kRowElems = 64;
constexpr int kTileRows = 256;                       // rows per CTA tile = threads per CTA
constexpr int kTileElems = kTileRows * kRowElems;    // 16384 elements

enum Dtype { kF32 = 0, kBF16 = 1 };

// Destination wire units (or blocks) of a producing kernel: local send buffers for the
// NCCL transport, or peers' receive buffers (CUDA IPC over NVLink) for the fused P2P
// transport, where the producing kernel is the exchange (all-gather / all-to-all push).
constexpr int kMaxDests = 64;
constexpr int kMaxN = 8;  // max local ranks per group (K3 keeps one tensor map per destination)
struct Dests {
  uint8_t* p[kMaxDests];
  int n;
  uint64_t remote;  // bit k: p[k] is peer memory (store via staged 1-D bulk copies)
};

// P2P completion flags (sdp4_api.cu): wait until every listed flag word of this rank's own
// symmetric buffer is non-zero, then reset it to 0 (binary flags, so a captured CUDA graph
// replays correctly).  timeout_ns > 0: give up after that long, write `code` | the index of the
// first missing flag into *err (host-mapped) and return -- the stream is never blocked forever.
constexpr int kMaxWait = 128;
struct FlagWait {
  uint32_t* flag[kMaxWait];
  int n;
  unsigned long long timeout_ns;
  uint32_t* err;  // device view of a host-mapped word
  uint32_t code[kMaxWait];
};
cudaError_t launch_wait_flags(const FlagWait& w, cudaStream_t st);

// Dynamic tile scheduling: a persistent kernel's CTAs claim tiles from a global counter pair
// {next, done} (so faster SMs take more tiles -- a static cyclic split measured 15-20% slower
// on HBM-bound streams).  Counters come from a small per-process pool, one pair per launch
// (round-robin over 64, so concurrent launches on different streams never share one); the
// pair is zeroed on the launch's stream right before the kernel (so it is correct whatever
// the slot's history -- an aborted kernel, a replayed CUDA graph) and the kernel's last CTA
// zeroes it again.  nullptr if the pool could not be allocated.
uint32_t* sched_counter(cudaStream_t st);

// K1: Alg. 2 l.2-3 -- d = w_main - w_model (this shard), k-bit group quantization
// into the wire unit at every destination dst.p[0..n) (n = 1: local; n = P: all-gather push).
// w_model_shard = nullptr: the qW codec (Alg. 1), d = w_main.  bits in {2, 4, 8, 32}.
// sr_on: stochastic rounding (R14) with key sr_key; element e has global index idx0 + e.
// apply_own: also w_model_shard += dequant(own unit) in place (Alg. 2 l.5 for this shard,
// K2's arithmetic); K2 then runs with skip_rot.
cudaError_t launch_qwd_quantize(const float* w_main, const void* w_model_shard, int model_dtype,
                                size_t S, int bits, int G, const Dests& dst, int sr_on, uint32_t sr_key,
                                uint64_t idx0, int sms, cudaStream_t st, bool apply_own = false);

// K2: Alg. 2 l.5 -- for every shard j < P: w_model[j*stride ..+S] += dequant(unit units.p[j])
// (local or peer memory), in place.  add = false (qW): w_model[...] = dequant(unit), no read.
// Tiles are visited unit-fastest, starting at unit `rot` (this rank: spreads the P2P pulls).
// skip_rot: unit `rot` is not applied (its owner did it in K1 with apply_own); P = 1 -> no launch.
cudaError_t launch_qwd_apply(const Dests& units, int P, size_t S, size_t stride, int bits, int G, void* w_model,
                             int model_dtype, bool add, int sms, cudaStream_t st, int rot = 0,
                             bool skip_rot = false);

// K6: one hop of the ring reduce-scatter with per-hop quantization (sec. 2.3, ablation):
// acc = (recv ? rn(dequant(recv) + g) : g) over S elements of one chunk (grad dtype);
// dst != nullptr: quantize acc (bits, G) into the wire unit at dst (local or peer memory);
// else out = rn(acc * kappa).
cudaError_t launch_ring_hop(const void* grad_chunk, int grad_dtype, const uint8_t* recv, uint8_t* dst, float* out,
                            float kappa, size_t S, int bits, int G, int sms, cudaStream_t st);

// Split of the P2P intra all-to-all (Alg. 3 l.4) between push and pull: K3 tile ts (16384
// elements) of a shard bound for local rank l' with bit l' of `mask` set is PULLED iff
// ts % den < num -- K3 stores it into its own outbox block l' (local memory) and K4 on rank l'
// bulk-loads it from there over NVLink; every other peer tile is pushed by K3 into the
// receive block of rank l'.  Spreading the NVLink bytes over K3 and K4 overlaps them with
// both kernels' HBM streams.
struct IntraPull {
  uint8_t* outbox[kMaxN];     // K3: this rank's outbox block for destination l' (M units)
  const uint8_t* src[kMaxN];  // K4: the outbox block of source l'' for this rank (peer memory)
  uint32_t mask;              // K3: destinations with pulled tiles; K4: sources with pulled tiles
  int num, den;
};

// K3: Alg. 3 l.2-3 -- blockwise Hadamard (b, in {0,2,..,256}) + bits_intra quantization
// of S elements of each of the P shards (shard j at grad + j*grad_stride elements); shard
// m'N + l' goes to unit m' of blocks[l'] (M units of unit_bytes; blocks[l'] is the local send
// block or the receive block of local rank l' itself; remote_mask bit l' = peer memory).
// Stochastic rounding: element e of shard j has global index j*grad_stride + sr_off + e.
cudaError_t launch_tlq_had_quant(const void* grad, size_t grad_stride, int grad_dtype, size_t S, int M, int N,
                                 int G, int b, float cb, int bits, uint8_t* const* blocks, uint32_t remote_mask,
                                 size_t unit_bytes, int sr_on, uint32_t sr_key, size_t sr_off, int sms,
                                 cudaStream_t st, const IntraPull* pull = nullptr);

// K4: Alg. 3 l.5,7,9 -- dequantize N received units per sub-block m', fp32 reduce in
// source order, requantize at bits_out into unit dst.p[m'] (local send unit or the
// receive slot of node m' itself).
// Stochastic rounding: element e of unit m' (shard m'*N + l_self) has global index
// (m'*N + l_self)*sr_stride + sr_off + e.
cudaError_t launch_tlq_dq_reduce_q(const uint8_t* intra_recv, size_t in_unit_bytes, int bits_in,
                                   int N, int M, size_t S, int G, const Dests& dst, int bits_out, int sr_on,
                                   uint32_t sr_key, int l_self, size_t sr_stride, size_t sr_off, int sms,
                                   cudaStream_t st, const IntraPull* pull = nullptr);

// K5: Alg. 3 l.11-13 -- dequantize M received units, fp32 reduce in source order,
// inverse blockwise Hadamard, scale by kappa, write the fp32 shard.
cudaError_t launch_tlq_dq_reduce_had(const uint8_t* inter_recv, size_t in_unit_bytes, int bits_in,
                                     int M, size_t S, int G, int b, float kappa, float* out,
                                     int sms, cudaStream_t st);

// ---- P2P flag layout (the sync protocol of sdp4_api.cu): word flag[kind][stage][src] of a
// rank's symmetric buffer; kind 0 = data (src published into my region), 1 = free (src is done
// with the region I wrote / it reads).
constexpr int kFlagStages = 64, kFlagSrcs = 256;
constexpr int kFlagData = 0, kFlagFree = 1;
__host__ __device__ inline size_t flag_word(int kind, int stage, int src) {
  return ((size_t)kind * kFlagStages + stage) * kFlagSrcs + src;
}

// ---- One-launch P2P paths ("small messages").  The whole exchange runs as
// ONE kernel per rank: the producing phase writes its units (peer memory over NVLink), the last
// warp / CTA to finish a phase raises the peers' data flags with system-scope release stores,
// the consuming phase polls its own flags with acquire loads (deadline: timeout_ns, then
// *err = code and carry on), and the last consumer raises the free flags -- the same flags, in
// the same order, as the multi-launch path, so the two paths interoperate call by call.
// Phases are claimed in order from one counter, so a task that waits for another phase finds
// every task of that phase already claimed by a running CTA: no co-residency assumption.
// nv > 1 virtual ranks in one launch emulate a P-rank job on one device (region / flags of
// every virtual rank are then plain device buffers): the parity tests' route on one GPU.
constexpr int kMaxVr = 8;  // virtual ranks per launch
constexpr int kFusedCtrWords = 32;  // per-op counter block: claim, exit, done[phase][vr]
struct FusedSync {
  uint8_t* region[kMaxDests];   // symmetric region of every rank (this process's mapping)
  uint32_t* flags[kMaxDests];   // flag words of every rank
  int rank[kMaxVr];             // ranks this launch acts for
  int nv, P;
  uint32_t* ctr;                // kFusedCtrWords counters, zero between launches
  uint32_t* err;                // host-mapped error word (timeouts), may be null
  unsigned long long timeout_ns;  // 0: wait forever
  unsigned long long* trace;    // debugging (SDP4_FUSED_TRACE): kTraceSlots %globaltimer stamps per unit
};
constexpr int kTraceSlots = 8;    // per warp / CTA: entry, exit, A start, A end, B start, B end, C start, C end
constexpr int kTraceUnits = 4096;  // warps / CTAs traced
// qWD step (Alg. 2 l.2-5): phase A quantizes the own shard into region[rank] and applies it to
// the own replica shard (K1 with apply_own); phase B applies every peer's unit (K2's pull).
// bits in {2, 4, 8, 32}, G <= 2048.  Flag stage 0.
cudaError_t launch_fused_qwd(const FusedSync& fs, const float* const* w_main, void* const* w_model, int model_dtype,
                             size_t S, int bits, int G, int sr_on, const uint32_t* sr_key, int sms, cudaStream_t st);
// TLq-HS (Alg. 3): phase A = K3 (push into the group peers' intra receive blocks), B = K4 (push
// into the node peers' inter slots), C = K5; the push-only single-chunk layout of the P2P path
// ([intra receive: N blocks of M units of w8][inter receive: M units of w4]).  bits_intra and
// bits_inter in {4, 8}; b in {0, 2, ..., 256}.  Flag stages 1 (intra) and 2 (inter).
cudaError_t launch_fused_tlq(const FusedSync& fs, const void* const* grad, int grad_dtype, float* const* out,
                             int M, int N, size_t S, int G, int b, float cb, float kappa, int bits_intra,
                             int bits_inter, size_t w8, size_t w4, int sr_on, const uint32_t* key8,
                             const uint32_t* key4, int sms, cudaStream_t st);
bool fused_tlq_supported(int bits_intra, int bits_inter, int b);

// TLq-HS with N = 1 (M > 1): K3 + K4 fused (k_local34.cu).  Shard j = m' of the gradient
// (at grad + j * grad_stride elements) -> its 4-bit unit at units[m'] (slot m of node m''s
// inter receive region; remote_mask bit m' = peer memory).  bits 8 / 4, any b.
cudaError_t launch_tlq_q84(const void* grad, size_t grad_stride, int grad_dtype, size_t S, int M, int G, int b,
                           float cb, uint8_t* const* units, uint64_t remote_mask, int sr_on, uint32_t key8,
                           uint32_t key4, int sms, cudaStream_t st);

// TLq-HS at world size 1 (M = N = 1) as one kernel, K3 -> K4 -> K5 fused in registers
// (k_local.cu): out[S] from grad[S], bits 8 (intra) / 4 (inter), any b.
cudaError_t launch_tlq_local(const void* grad, int grad_dtype, size_t S, int G, int b, float cb, float kappa,
                             int sr_on, uint32_t key8, uint32_t key4, float* out, int sms, cudaStream_t st);
// Fill n words with v (flag initialization of emulated symmetric buffers).
cudaError_t launch_fill32(uint32_t* p, size_t n, uint32_t v, cudaStream_t st);

}  // namespace sdp4
