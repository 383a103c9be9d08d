/*
 * sdp4.h -- C ABI of libsdp4: the SDP4Bit data-parallel communication hot path
 * (arXiv 2410.15526) on B200 (sm_100a) with NCCL over NVLink 5 / NVSwitch.
 *
 * Citations: "P:n" = line n of the paper text, with its section /
 * algorithm label; "R<k>" = reading k of DESIGN.md sec. 3 (where the paper is
 * silent or ambiguous).  Notation: P = M*N workers (M groups of N, rank
 * r = m*N + l, sec. 2.3); D = numel of the flat buffer; S = D/P the shard
 * length, shard r = [r*S, (r+1)*S) (sec. 2.1); G = quantization group
 * size; k = bits, q_k = 2^(k-1)-1; b = Hadamard block.
 *
 * Conventions (all entry points):
 *  - Data pointers (w_main_shard, w_model_full, grad, out_shard, workspace) are
 *    CUDA DEVICE pointers owned by the caller; the library never allocates,
 *    frees or retains them beyond the call.  They must be 16-byte aligned.
 *  - `stream` is a cudaStream_t (passed as void*).  Every call is stream-ordered
 *    on it: kernels and NCCL calls are enqueued, nothing is synchronized on the
 *    host (except sdp4_comm_init / sdp4_comm_destroy / sdp4_profile_read).
 *  - Validation happens before any launch; on error nothing is enqueued, the
 *    status is returned and sdp4_last_error() describes it.
 *  - Alignment rule (R1): numel % (P * lcm(G, 64)) == 0 (the caller zero-pads;
 *    zeros are reduction-neutral).  Groups never straddle shards.
 *  - Calls on one comm are not reentrant; serialize them on one stream.
 *  - World size 1 is valid: no NCCL traffic, every codec step still runs.
 */
#ifndef SDP4_H
#define SDP4_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SDP4_OK = 0,
  SDP4_EINVAL = 1, /* bad argument (null pointer, unsupported bits/dtype/group, M*N != world) */
  SDP4_EALIGN = 2, /* size/alignment rule violated (numel, G % b, pointer alignment)          */
  SDP4_ECUDA = 3,  /* a CUDA runtime error (launch failure, bad device pointer)                */
  SDP4_ENCCL = 4,  /* an NCCL error, including an asynchronous one from a previous call         */
  SDP4_ESTATE = 5,  /* workspace too small, call out of order, or comm unusable                  */
  SDP4_ETIMEOUT = 6 /* a P2P flag wait of an earlier call passed its deadline (a peer never
                       signalled); the comm is unusable and must be destroyed                     */
} sdp4_status;

typedef enum { SDP4_F32 = 0, SDP4_BF16 = 1 } sdp4_dtype;
/* Rounding of the quantizers.  SDP4_RNE: code = RNE(x * rn(q/s)) of the exact product (R3).
 * SDP4_STOCHASTIC (NEXT-2, R14; unbiased as the convergence theory assumes for gradients,
 * Def. 1): y = rn(x * rn(q/s)), fl = floor(y), fr = rn(y - fl),
 * code = clamp(fl + [U < fr], +-q) with U = (h >> 8) * 2^-24,
 * h = mix32(lo32(i) ^ mix32(hi32(i) ^ key)), key = mix32(seed_lo ^ mix32(seed_hi ^
 * (stage << 24) ^ rank)), stage qWD = 1 / intra = 2 / inter = 3, i = the element's global
 * index (d: rank*S + e; gradient: its index in the full buffer; inter message: its index
 * in the full buffer), rank = the quantizing rank; mix32(x): x ^= x >> 16;
 * x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16.  Pass a new seed per call. */
typedef enum { SDP4_RNE = 0, SDP4_STOCHASTIC = 1 } sdp4_round;

/* Opaque communicator: world + intra (N ranks of group m) + inter (M ranks of
 * local rank l) NCCL communicators, plus profiling state.  P:292 sec. 2.3. */
typedef struct sdp4_comm* sdp4_comm_t;

#define SDP4_UNIQUE_ID_BYTES 128

/* Library version (major*10000 + minor*100 + patch). */
int sdp4_version(void);

/* Thread-local description of the last error of this thread ("" if none).
 * Valid until the next sdp4_* call on the same thread. */
const char* sdp4_last_error(void);

/* Host.  Fill id[128] with a fresh NCCL unique id (call on rank 0, broadcast the
 * bytes to every rank by any means, e.g. torch.distributed). */
sdp4_status sdp4_get_unique_id(unsigned char id[SDP4_UNIQUE_ID_BYTES]);

/* Host, collective over all `world` ranks.  Binds to the CURRENT CUDA device.
 * groups_M * group_size_N must equal world (P = M*N).  For world == 1 the
 * id may be NULL and no NCCL communicator is created.  intra = ncclCommSplit
 * (color = rank / N, key = rank % N); inter = ncclCommSplit(color = rank % N,
 * key = rank / N).  nccl_ctas (0 = default 16): NCCL is capped at that many CTAs
 * (ncclConfig_t.maxCTAs) and, while a call is pipelined, libsdp4's persistent kernels
 * leave that many SMs free so the NCCL exchanges run concurrently.
 * On success *out owns the communicators and an internal high-priority stream. */
sdp4_status sdp4_comm_init(sdp4_comm_t* out, const unsigned char* id, int rank, int world,
                           int groups_M, int group_size_N, int nccl_ctas);

/* Host.  Pipelining: every shard is processed in `chunks` sub-ranges (0 = automatic; 1 = no
 * pipelining; at most 16).  NCCL transport: automatic = about 16M elements per chunk, at
 * most 8; the kernels of chunk c run on the caller's stream while the exchanges of other
 * chunks run on the internal stream.  P2P transport (TLq-HS only): automatic = 1; with C > 1
 * the chunks alternate between the caller's stream and the internal stream, so K4/K5 of
 * one chunk overlap the NVLink-bound K3 of the next.  Results do not depend on the chunk
 * count (R16).  World size 1 never pipelines.  sdp4_comm_chunks returns the chunk count a
 * call with (numel, group) uses. */
sdp4_status sdp4_comm_set_chunks(sdp4_comm_t comm, int chunks);
int sdp4_comm_chunks(sdp4_comm_t comm, size_t numel, int group);

/* Host.  Transport of the exchanges (world > 1):
 *   0 NCCL: kernels write the caller's workspace; ncclAllGather / ncclAlltoAll move it
 *     (with the chunked two-stream pipeline above);
 *   1 P2P (default when every rank can map every other rank's memory with CUDA IPC -- one OS
 *     instance, peer access between the devices or ranks sharing one device -- and N <= 8,
 *     P <= 64; checked collectively by sdp4_comm_init): the exchanges are fused into the
 *     kernels over NVLink: K3 and K4 push their quantized tiles straight into the receive
 *     regions of the ranks that own them; the qWD all-gather is a pull inside K2 (unit j read
 *     from rank j's buffer while the replica update streams HBM).  The receive regions are
 *     library-owned, symmetric and allocated collectively on first use (the caller's workspace
 *     is then unused and may be NULL / 0 bytes).  Completion and reuse are signalled per
 *     (stage, source) with binary flags: a producer raises data[stage][me] in the consumer's
 *     buffer after its kernel, the consumer raises free[stage][me] in the producer's buffer
 *     after consuming; each side waits for (and resets) the flag before its kernel.  No
 *     host-side epoch: a P2P call captured in a CUDA graph replays correctly (make one eager
 *     call of the same size first, so no buffer grows during capture: ESTATE otherwise).
 *     P2P qWD allows one outstanding quantize per comm (quantize, apply, quantize, ...).
 * Results are bit-identical across transports (R16).  sdp4_comm_transport returns the
 * current one.  EINVAL for P2P if it is unavailable, for NCCL on a sdp4_comm_init_p2p comm. */
sdp4_status sdp4_comm_set_transport(sdp4_comm_t comm, int transport);
int sdp4_comm_transport(sdp4_comm_t comm);

/* Host.  Deadline of every P2P flag wait (seconds; default 300, or SDP4_WAIT_TIMEOUT_S).  A
 * wait is a one-warp polling kernel: if a peer has not signalled by the deadline (it died or
 * skipped a collective call), the kernel writes a host-mapped error word and returns instead
 * of blocking the stream forever; the next call on this comm (or sdp4_comm_check) returns
 * SDP4_ETIMEOUT, and results of the timed-out call are garbage.  0: unbounded waits with
 * stream memory operations (cuStreamWaitValue32), no kernel.  Ranks that share one GPU
 * (sdp4_comm_init_p2p emulation) always wait with stream memory operations -- kernels of
 * different processes are not guaranteed to run concurrently, so no kernel may wait for
 * another rank -- and EINVAL is returned for seconds > 0. */
sdp4_status sdp4_comm_set_timeout(sdp4_comm_t comm, double seconds);

/* Host, no synchronization.  SDP4_OK, or the asynchronous error of an earlier call
 * (SDP4_ETIMEOUT from a P2P wait, SDP4_ENCCL from NCCL) visible so far. */
sdp4_status sdp4_comm_check(sdp4_comm_t comm);

/* Host.  P2P transport only: how the intra all-to-all (Alg. 3 l.4) moves over NVLink.  Of
 * the K3 tiles (16384 elements of a shard) bound for another local rank, those with
 * tile_index % den < num are PULLED -- K3 stores them into this rank's own outbox and K4 on
 * the destination bulk-loads them over NVLink -- and the rest are PUSHED by K3 into the
 * destination's receive block.  Splitting the bytes between the two kernels overlaps them
 * with both kernels' HBM streams.  num = 0: push only.  Default (never set): push only when
 * N = 2, 1/2 for N >= 3 (measured).  Results do not depend on the split
 * (R16).  EINVAL unless 0 <= num <= den, 1 <= den <= 64. */
sdp4_status sdp4_comm_set_intra_pull(sdp4_comm_t comm, int num, int den);

/* Host.  Small-message path of the P2P transport: sdp4_qwd_step and
 * sdp4_tlq_hs_reduce_scatter calls on buffers of numel <= limit elements run as ONE kernel per
 * rank -- the producing phase writes peer memory over NVLink, the consuming phase polls its
 * flags in-kernel (same flags, same deadline and SDP4_ETIMEOUT behaviour as the multi-launch
 * path), so a call costs one launch instead of two or three stream-ordered hand-offs (Alg. 2
 * l.2-5; Alg. 3, P:368-379 -- the arithmetic and results are identical, R16).
 * Applies when the ranks are on distinct GPUs, with one chunk, and for TLq-HS when
 * bits_intra and bits_inter are in {4, 8}; other calls take the multi-launch path.  Defaults
 * (the measured crossovers): 8 Mi elements for the qWD step, 16 Mi for TLq-HS; a value set
 * here (or SDP4_FUSED_MAX_NUMEL) applies to both; 0 disables the path. */
sdp4_status sdp4_comm_set_fused_limit(sdp4_comm_t comm, size_t numel);

/* Host.  World size 1: sdp4_tlq_hs_reduce_scatter with bits 8 / 4 runs K3 -> K4 -> K5 as ONE
 * kernel (both all-to-alls of Alg. 3 are the identity with one rank, so the 8- and 4-bit
 * codes never leave the registers: 6 instead of ~9 bytes of HBM traffic per element, same
 * operations, bit-identical results).  enable = 0 selects the three-kernel path (measurement;
 * default 1). */
sdp4_status sdp4_comm_set_local_fusion(sdp4_comm_t comm, int enable);

/* Host, collective (every rank calls it).  Waits for this rank's work, then -- if symmetric
 * buffers were allocated -- barriers with the peers (they may still be pulling from this
 * rank's buffers) before unmapping and freeing them; destroys the NCCL communicators and
 * frees the comm.  Call it explicitly on every rank (not from a garbage collector). */
sdp4_status sdp4_comm_destroy(sdp4_comm_t comm);

/* Host bootstrap callback of sdp4_comm_init_p2p: collective over the `world` ranks, blocking;
 * gathers `bytes` bytes from every rank into recv (rank r's at recv + r * bytes).  Returns 0
 * on success.  Called only from sdp4_comm_init_p2p, from calls that (re)allocate symmetric
 * buffers, and from sdp4_comm_destroy, on the calling thread. */
typedef int (*sdp4_host_allgather_fn)(const void* send, void* recv, size_t bytes, void* ctx);

/* Host, collective.  A P2P-only comm bootstrapped WITHOUT NCCL: `allgather` (e.g. over a
 * torch.distributed gloo group) exchanges the CUDA-IPC handles and reachability records.
 * Every rank must reach every other through CUDA IPC (same OS instance; peer access between
 * the devices) -- ranks may share ONE device, so P ranks (any M x N, N <= 8, P <= 64) run on a
 * single GPU through exactly the product P2P path (NCCL refuses duplicate GPUs).  Binds to the
 * current device.  The transport is P2P and cannot be changed; the NCCL comparators return
 * ESTATE.  ESTATE if some rank cannot reach another. */
sdp4_status sdp4_comm_init_p2p(sdp4_comm_t* out, int rank, int world, int groups_M, int group_size_N,
                               sdp4_host_allgather_fn allgather, void* ctx);

/* ---------------------------------------------------------------------------
 * Sizes and workspace layout (R15).  One "wire unit" carries n elements at k
 * bits: [codes n*k/8 bytes][fp32 scales n/G][zero..255 pad bytes], the unit
 * size rounded up to 256 bytes.  int4 codes are two's-complement nibbles,
 * element 2j in the low nibble; int8 codes two's complement (R4).  k = 32 is
 * the identity codec (R12): n fp32 values, no scales.
 * ------------------------------------------------------------------------- */
size_t sdp4_wire_unit_bytes(size_t n, int bits, int group);

/* qWD workspace (Alg. 2 l.3-4): per chunk (see sdp4_comm_set_chunks) P
 * consecutive wire units W(len_chunk, bits, G), unit r = rank r's quantized weight
 * difference; with one chunk simply P units W(S, bits, G).  The size returned covers any
 * chunk count.  0 on bad args. */
size_t sdp4_qwd_workspace_bytes(int world, size_t numel, int bits, int group);

/* TLq-HS workspace (Alg. 3), per chunk four regions in this order (the size
 * returned covers any chunk count; the offsets below are those of a one-chunk call):
 *   region 0 intra_send: N blocks of M units W(S, bits_intra, G); block l' unit m'
 *            holds shard m'*N + l' of H(grad) quantized (Alg. 3 l.2-3, R9)
 *   region 1 intra_recv: N blocks of M units (block l'' = from local rank l'')
 *            (aliases region 0 when N == 1)
 *   region 2 inter_send: M units W(S, bits_inter, G); unit m' = shard m'*N + l
 *   region 3 inter_recv: M units (unit m'' = from group m''; aliases region 2 when M == 1)
 * sdp4_tlq_workspace_offset(region) gives each region's byte offset.  0 on bad args. */
size_t sdp4_tlq_workspace_bytes(int groups_M, int group_size_N, size_t numel, int bits_intra,
                                int bits_inter, int group);
size_t sdp4_tlq_workspace_offset(int groups_M, int group_size_N, size_t numel, int bits_intra,
                                 int bits_inter, int group, int region);

/* ---------------------------------------------------------------------------
 * qWD -- quantized weight differences (sec. 3.1; Alg. 2).
 * ------------------------------------------------------------------------- */

/* Alg. 2 l.2-3 on this rank r:
 *   d[r] = w_main[r] - w_model[r]   (fp32; w_model widened exactly, R11)
 *   d~[r] = QuantizeWeightsDiff(d[r]): per G-group s = max|d|, codes = RNE(d * rn(q_k/s))
 *           (R2, R3), written as wire unit r of `workspace` (layout above).
 * w_main_shard: fp32[S] (this rank's main weights).  w_model_full: the
 * full replica D elements of model_dtype (bf16 or fp32); only
 * [r*S, (r+1)*S) is read.  bits in {2, 4, 8, 32} (2 = the ternary codec of
 * Counterexample 1, int2 packing R4); G power of two in [32, 2048].
 * rnd / seed: rounding of the codes (see sdp4_round). */
sdp4_status sdp4_qwd_quantize(sdp4_comm_t comm, const float* w_main_shard, const void* w_model_full,
                              sdp4_dtype model_dtype, size_t numel, int bits, int group,
                              sdp4_round rnd, uint64_t seed, void* workspace, size_t workspace_bytes,
                              void* stream);

/* Alg. 2 l.4-5: AllGather of the P wire units in place in
 * `workspace` (ncclAllGather on the world comm), then for all D elements
 *   w_model <- bf16_rn(widen(w_model) + code * rn(s / q_k))   (fp32 add for fp32 models)
 * in place (R5, R11).  Every rank, owner included, applies the dequantized d~,
 * so all replicas stay bit-identical. */
sdp4_status sdp4_qwd_allgather_apply(sdp4_comm_t comm, void* workspace, size_t workspace_bytes,
                                     size_t numel, int bits, int group, void* w_model_full,
                                     sdp4_dtype model_dtype, void* stream);

/* Alg. 2 l.2-5 in one call: the same result as sdp4_qwd_quantize followed by
 * sdp4_qwd_allgather_apply, bit for bit, with the owner's own update fused into the quantize
 * kernel: K1 holds widen(w_model[r]) and the codes of d~[r] in registers, so it also writes
 *   w_model[r] <- bf16_rn(widen(w_model[r]) + code * rn(s / q_k))
 * (K2's arithmetic, element by element) and K2 then applies only the P - 1 other units.
 * Saves one read of the replica shard and of unit r per step (at P = 1, K2 does not run).
 * w_model_full is read and written (shard r by K1, the others by K2); all other arguments,
 * the workspace and the errors are those of the two calls.  The wire unit r is identical. */
sdp4_status sdp4_qwd_step(sdp4_comm_t comm, const float* w_main_shard, void* w_model_full,
                          sdp4_dtype model_dtype, size_t numel, int bits, int group, sdp4_round rnd,
                          uint64_t seed, void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Ablation baselines: the codecs SDP4Bit is compared against.
 * ------------------------------------------------------------------------- */

/* qW -- direct weight quantization of QSDP / ZeRO++ (Alg. 1 P:231-233 "Quantize weights",
 * "AllGather"; contrasted with qWD in sec. 3.1 P:330-336 and Counterexample 1 P:412-416).
 * Same workspace, wire unit, symmetric buffers and rounding as sdp4_qwd_quantize, but the
 * codes are those of w_main[r] itself:  codes = RNE(w_main * rn(q_k/s)), s = max|w_main| per
 * group.  No replica is read.  Errors as sdp4_qwd_quantize. */
sdp4_status sdp4_qw_quantize(sdp4_comm_t comm, const float* w_main_shard, size_t numel, int bits, int group,
                             sdp4_round rnd, uint64_t seed, void* workspace, size_t workspace_bytes,
                             void* stream);

/* qW AllGather + dequantize: for all D elements  w_model <- dtype_rn(code * rn(s / q_k))
 * (assignment, not accumulation: the replica becomes the gathered quantized weights, which
 * is why a biased codec can stall).  w_model_full is only written. */
sdp4_status sdp4_qw_allgather_apply(sdp4_comm_t comm, void* workspace, size_t workspace_bytes, size_t numel,
                                    int bits, int group, void* w_model_full, sdp4_dtype model_dtype,
                                    void* stream);

/* Ring reduce-scatter with per-hop quantization (sec. 2.3: "P-1 rounds of
 * quantization and dequantization, potentially leading to error propagation").  Chunk c
 * (= shard c, ends on rank c) starts on rank c+1: acc = g_{c+1}[c]; at hop h = 1..P-1 rank
 * (c+h) mod P sends Quantize(acc) (bits, group G, nearest, R3) and rank (c+h+1) mod P sets
 * acc = rn(Dequantize(msg) + g_own[c]) in fp32; out_shard = rn(acc * rn(1/P)) if average
 * else acc.  grad: D elements of grad_dtype; out_shard: fp32[S].  bits in {4, 8, 32}.
 * Transport as configured: P2P pushes each hop into the next rank's library-owned slot over
 * NVLink (one flag per hop); NCCL uses ncclSend/ncclRecv on `stream` with `workspace` as
 * the send and receive units.  workspace_bytes >= sdp4_ring_workspace_bytes (2 units). */
size_t sdp4_ring_workspace_bytes(int world, size_t numel, int bits, int group);
sdp4_status sdp4_ring_reduce_scatter(sdp4_comm_t comm, const void* grad, sdp4_dtype grad_dtype, size_t numel,
                                     int bits, int group, int average, float* out_shard, void* workspace,
                                     size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * TLq-HS -- two-level gradient quantization with Hadamard smoother, replacing the
 * ReduceScatter of Alg. 2 l.9: Alg. 3 with the sec. 3.3
 * pruning:
 *   K3  u = H_unnorm(grad) per b-block; per G-group s_u = max|u|; codes =
 *       RNE(u * rn(q/s_u)) at bits_intra; scale = rn(s_u * c_b), c_b = rn(1/sqrt b) (R6)
 *   --  IntraAlltoAll (ncclAlltoAll on the intra comm)                 (l.4)
 *   K4  acc = sum_{l''=0..N-1} code * rn(s/q) in fp32, requantize at
 *       bits_inter                                                       (l.5,7,9)
 *   --  InterAlltoAll (ncclAlltoAll on the inter comm)                 (l.10)
 *   K5  acc = sum_{m''=0..M-1} code * rn(s/q); out = rn(H_unnorm(acc) * kappa),
 *       kappa = rn(c_b / P) if average else c_b (b = 0: rn(1/P) or none)  (l.11-13, R8)
 * grad: D elements of grad_dtype (fp32 or bf16).  out_shard: fp32[S], shard r.
 * hadamard_block b in {0, 2, 4, ..., 256} with G % b == 0; b = 0 gives
 * TLq; (bits_intra, bits_inter, b) = (4, 4, 0) gives ULq.
 * bits_intra, bits_inter in {4, 8, 32}.  workspace_bytes >= sdp4_tlq_workspace_bytes, except
 * with the P2P transport (library-owned buffers) and at world size 1 with bits 8 / 4 and the
 * local fusion on (K3 -> K4 -> K5 as one kernel, sdp4_comm_set_local_fusion), where the
 * workspace is not used and may be NULL. */
sdp4_status sdp4_tlq_hs_reduce_scatter(sdp4_comm_t comm, const void* grad, sdp4_dtype grad_dtype,
                                       size_t numel, int bits_intra, int bits_inter, int group,
                                       int hadamard_block, int average, sdp4_round rnd, uint64_t seed,
                                       float* out_shard, void* workspace, size_t workspace_bytes,
                                       void* stream);

/* Stage entry points: the three kernels of sdp4_tlq_hs_reduce_scatter on ONE rank's
 * buffers, with no communication and no comm object (argument rules as above, with
 * P = groups_M * group_size_N).  They let a caller verify each stage or emulate P ranks
 * on one GPU by moving the blocks itself.  Buffers use the region layouts of
 * sdp4_tlq_workspace_offset: intra_send / intra_recv = N blocks of M units
 * W(S, bits_intra, G); inter_send / inter_recv = M units W(S, bits_inter, G).
 *   stage_quantize  K3: Alg. 3 l.2-3: grad (D) -> intra_send
 *   stage_reduce    K4: Alg. 3 l.5,7,9 for local rank l: intra_recv -> inter_send
 *   stage_final     K5: Alg. 3 l.11-13: inter_recv -> out_shard (S)
 *   stage_quantize_reduce  K34, one GPU per group (N = 1, bits 8 / 4): Alg. 3 l.2-9 for rank
 *                   `rank` = node m: grad (D) -> inter_send, unit m' = shard m' (the 8-bit
 *                   intra units never materialize; sdp4_tlq_hs_reduce_scatter's N = 1 path) */
sdp4_status sdp4_tlq_stage_quantize(const void* grad, sdp4_dtype grad_dtype, size_t numel, int groups_M,
                                    int group_size_N, int bits_intra, int group, int hadamard_block,
                                    sdp4_round rnd, uint64_t seed, int rank, void* intra_send, void* stream);
sdp4_status sdp4_tlq_stage_quantize_reduce(const void* grad, sdp4_dtype grad_dtype, size_t numel, int groups_M,
                                           int group, int hadamard_block, sdp4_round rnd, uint64_t seed, int rank,
                                           void* inter_send, void* stream);
sdp4_status sdp4_tlq_stage_reduce(const void* intra_recv, size_t numel, int groups_M, int group_size_N,
                                  int bits_intra, int bits_inter, int group, sdp4_round rnd, uint64_t seed,
                                  int rank, void* inter_send, void* stream);
sdp4_status sdp4_tlq_stage_final(const void* inter_recv, size_t numel, int groups_M, int group_size_N,
                                 int bits_inter, int group, int hadamard_block, int average, float* out_shard,
                                 void* stream);

/* ---------------------------------------------------------------------------
 * One-launch kernels on an EMULATED job (tests): all P = world (or M * N <= 8) ranks of a job
 * run in ONE launch of the small-message kernels on the current device, each rank's symmetric
 * buffer (flags + region) a slice of `workspace` (device, caller-owned, >= the *_workspace_bytes
 * value; 0 = invalid arguments).  Array arguments are HOST arrays of P device pointers, rank q
 * at index q: w_main_shards[q] (fp32, numel / P), w_model_full[q] (its replica, numel, updated
 * in place as sdp4_qwd_step would on rank q), grads[q] (numel), out_shards[q] (fp32, numel / P,
 * written as sdp4_tlq_hs_reduce_scatter would on rank q).  fresh != 0 resets the emulated flags
 * to their initial state (a first call); fresh == 0 continues from the previous call on the
 * same workspace and sizes (exercises the flag resets between calls).  Stream-ordered on
 * `stream`; a kernel whose waits do not complete within 20 s gives up (wrong results, no hang).
 * Errors: EINVAL (arguments, or bits outside the one-launch set), EALIGN, ESTATE (workspace
 * too small), ECUDA (launch).
 * ------------------------------------------------------------------------- */
size_t sdp4_emu_qwd_workspace_bytes(int world, size_t numel, int bits, int group);
sdp4_status sdp4_emu_qwd_step(int world, const float* const* w_main_shards, void* const* w_model_full,
                              sdp4_dtype model_dtype, size_t numel, int bits, int group, sdp4_round rnd,
                              uint64_t seed, int fresh, void* workspace, size_t workspace_bytes, void* stream);
size_t sdp4_emu_tlq_workspace_bytes(int groups_M, int group_size_N, size_t numel, int bits_intra, int bits_inter,
                                    int group);
sdp4_status sdp4_emu_tlq_hs_reduce_scatter(int groups_M, int group_size_N, const void* const* grads,
                                           sdp4_dtype grad_dtype, size_t numel, int bits_intra, int bits_inter,
                                           int group, int hadamard_block, int average, sdp4_round rnd, uint64_t seed,
                                           float* const* out_shards, int fresh, void* workspace,
                                           size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Instrumentation (measurement only; no effect on results).
 * ------------------------------------------------------------------------- */
/* Count of kernels this comm launched since init (or since the last reset). */
uint64_t sdp4_launch_count(sdp4_comm_t comm, int reset);

/* enable != 0: bracket every kernel launch of this comm with CUDA events on its
 * stream; sdp4_profile_read synchronizes those events and returns, per kernel
 * name, the summed device milliseconds and launch count since the last read.
 * names[i] point to static strings.  *count receives the number of entries. */
sdp4_status sdp4_profile_enable(sdp4_comm_t comm, int enable);
sdp4_status sdp4_profile_read(sdp4_comm_t comm, const char** names, double* ms, uint64_t* launches,
                              int max_entries, int* count);

/* Unquantized comparators on the same comm (bench only, sec. 2.1):
 * ncclReduceScatter(sum, or avg if average) of D elements of dtype into S, and
 * ncclAllGather of S elements of dtype into D. */
sdp4_status sdp4_nccl_reduce_scatter(sdp4_comm_t comm, const void* send, void* recv, size_t numel,
                                     sdp4_dtype dtype, int average, void* stream);
sdp4_status sdp4_nccl_all_gather(sdp4_comm_t comm, const void* send, void* recv, size_t numel,
                                 sdp4_dtype dtype, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SDP4_H */
