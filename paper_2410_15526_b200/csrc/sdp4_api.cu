// sdp4_api.cu -- the C ABI of include/sdp4.h: argument validation, workspace layout,
// NCCL communicators (world + intra + inter via ncclCommSplit, sec. 2.3) and the
// stream-ordered orchestration of Alg. 2 l.2-5 (qWD) and Alg. 3 (TLq-HS).
//
// Pipelining (row p of the hot path; the paper overlaps its two all-to-alls):
// every shard is split into C chunks.  Chunk c is an independent instance of the path on
// the sub-range [off_c, off_c + len_c) of every shard (groups never straddle chunks, R1),
// with its own workspace regions.  Kernels run on the caller's stream, NCCL calls on an
// internal high-priority side stream; CUDA events carry the per-chunk dependencies, and the
// issue order is software-pipelined (K3(c) | K4(c-1) | K5(c-2) against the exchanges of the
// chunks in between), so NVLink transfers overlap kernel work.  Kernels leave
// `nccl_ctas` SMs free and NCCL is capped at that many CTAs, so both make progress.
// Results are bit-identical for every C (tests/test_gpu_dist.py).
//
// Transports.  NCCL: kernels write local send buffers, NCCL moves them (the baseline).
// P2P (default when every rank reaches every other through CUDA IPC): the producing kernel IS
// the exchange -- K1 publishes its unit in its own buffer and every K2 pulls it, K3 stores each
// tile into the receive block of the local rank that owns it, K4 stores each requantized unit
// into its node's receive slot, all through CUDA-IPC-mapped peer memory over NVLink/NVSwitch,
// tile by tile while computing.  Receive regions are library-owned and symmetric across ranks;
// completion and reuse are signalled with binary data/free flags (the sync protocol below):
// raised by stream memory operations after the producing / consuming kernel, awaited by a
// one-warp polling kernel with a deadline (or, with the timeout set to 0, by
// cuStreamWaitValue32).  No host-side epoch: a captured CUDA graph replays correctly.
// Ranks may share one GPU (sdp4_comm_init_p2p with a host bootstrap), which emulates any
// M x N topology on a single device.
#include "sdp4.h"

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include <unistd.h>

#include <cuda.h>
#include <cudaTypedefs.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: host ranges for nsys / ncu (no link dependency)
#include <cuda_runtime.h>
#include <nccl.h>

#include "sdp4_kernels.cuh"

namespace {

constexpr int kMaxChunks = 16;
constexpr int kDefaultNcclCtas = 16;
constexpr double kDefaultTimeoutS = 300.0;  // P2P flag waits (SDP4_WAIT_TIMEOUT_S; 0 = unbounded memop waits)
// P2P calls on buffers of at most this many elements run as one kernel per rank (k_fused.cu);
// SDP4_FUSED_MAX_NUMEL / sdp4_comm_set_fused_limit override (measured crossover)
constexpr size_t kDefaultFusedLimit = (size_t)8 << 20;      // qWD: 32 MB of fp32 (measured crossover,
constexpr size_t kDefaultFusedLimitTlq = (size_t)16 << 20;  // TLq-HS: 64 MB           DESIGN.md sec. 9)

thread_local std::string g_err;

// NVTX range around every data-path entry point (the call's name), so an nsys / ncu timeline
// shows which collective each kernel, memop and NCCL call belongs to (SURVEY sec. 5 tracing).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

sdp4_status fail(sdp4_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

bool is_pow2(long long x) { return x > 0 && (x & (x - 1)) == 0; }
size_t round_up(size_t a, size_t m) { return (a + m - 1) / m * m; }

bool valid_bits(int bits) { return bits == 4 || bits == 8 || bits == 32; }
bool valid_wbits(int bits) { return bits == 2 || valid_bits(bits); }  // weight codecs add int2 (R4)

// Wire unit (R15): [codes n*k/8][fp32 scales n/G] padded to 256 bytes; k = 32: n fp32.
size_t unit_bytes(size_t n, int bits, int group) {
  if (bits == 32) return round_up(4 * n, 256);
  return round_up(n * (size_t)bits / 8 + 4 * (n / (size_t)group), 256);
}

struct Chunk {
  size_t off, len;
};

// Split a shard of S elements into at most C chunks aligned to lcm(G, 64) (and to the 16384-
// element Hadamard tile when the chunks are large enough).
std::vector<Chunk> plan_chunks(size_t S, int C, int group) {
  const size_t a0 = (size_t)std::max(group, 64);
  C = std::max(1, std::min(C, kMaxChunks));
  size_t align = a0;
  if (S / C >= 4 * (size_t)sdp4::kTileElems) align = std::max(a0, (size_t)sdp4::kTileElems);
  const size_t base = round_up((S + C - 1) / C, align);
  std::vector<Chunk> out;
  for (size_t off = 0; off < S; off += base) out.push_back({off, std::min(base, S - off)});
  if (out.empty()) out.push_back({0, S});
  return out;
}

// Per-chunk TLq-HS regions (R9, R15): intra_send N*M units, intra_recv (aliased if N == 1),
// inter_send M units, inter_recv (aliased if M == 1).
struct TlqRegions {
  size_t send8, recv8, send4, recv4, end;
};
TlqRegions tlq_regions(int M, int N, size_t len, int bi, int be, int group, size_t base) {
  const size_t w8 = unit_bytes(len, bi, group), w4 = unit_bytes(len, be, group);
  const size_t intra = (size_t)N * M * w8, inter = (size_t)M * w4;
  TlqRegions r;
  r.send8 = base;
  r.recv8 = N > 1 ? r.send8 + intra : r.send8;
  r.send4 = r.recv8 + intra;
  r.recv4 = M > 1 ? r.send4 + inter : r.send4;
  r.end = r.recv4 + inter;
  return r;
}

size_t tlq_total(int M, int N, size_t S, int bi, int be, int group, int C) {
  size_t base = 0;
  for (const Chunk& ch : plan_chunks(S, C, group)) base = tlq_regions(M, N, ch.len, bi, be, group, base).end;
  return base;
}
size_t qwd_total(int P, size_t S, int bits, int group, int C) {
  size_t t = 0;
  for (const Chunk& ch : plan_chunks(S, C, group)) t += (size_t)P * unit_bytes(ch.len, bits, group);
  return t;
}

}  // namespace

// Library-owned receive buffer, mapped on every rank (CUDA IPC).  Layout:
// [flags: kFlagBytes][region].  Flags are binary words flag[kind][stage][src] (see the sync
// protocol below); one region, reused every call.
using sdp4::kFlagStages;
using sdp4::kFlagSrcs;
constexpr int kDrainStage = kFlagStages - 1;  // TLq-HS layout-change drain (stages 1..2C are per chunk)
constexpr size_t kFlagBytes = 2 * (size_t)kFlagStages * kFlagSrcs * sizeof(uint32_t);
enum FlagKind { kData = sdp4::kFlagData, kFree = sdp4::kFlagFree };
inline size_t flag_off(int kind, int stage, int src) { return sdp4::flag_word(kind, stage, src) * sizeof(uint32_t); }
struct SymBuf {
  uint8_t* local = nullptr;
  size_t bytes = 0, region = 0;
  std::vector<uint8_t*> peer;  // peer[r]: rank r's buffer in this process (peer[rank] = local)
};

enum Transport { kTransportNccl = 0, kTransportP2P = 1 };

// Host-side allgather the library uses for its own bootstrap (IPC handles, reachability,
// barriers): the caller's callback (sdp4_comm_init_p2p), else ncclAllGather on the world comm.
typedef int (*HostAllgather)(const void* send, void* recv, size_t bytes, void* ctx);

// What a rank tells its peers at init so that each can decide whether CUDA IPC reaches them:
// the same OS instance (host name + kernel boot id) and a device this process can map.
struct PeerInfo {
  char host[96];
  unsigned char uuid[16];
  int pid;
};

struct sdp4_comm {
  int rank = 0, world = 1, M = 1, N = 1, m = 0, l = 0;
  int transport = kTransportNccl;
  bool p2p_ok = false;  // every rank reaches every other through CUDA IPC (same host, P2P-capable)
  bool shared_gpu = false;  // some ranks share a device: flag waits must not be polling kernels
  HostAllgather ag_fn = nullptr;
  void* ag_ctx = nullptr;
  SymBuf sym_qwd, sym_tlq, sym_ring;
  struct QwdPending {  // P2P: the unit K1 published and K2 has not yet consumed
    bool valid = false;
    size_t numel = 0;
    int bits = 0, group = 0;
  } qwd_pending;
  uint64_t tlq_layout[6] = {0, 0, 0, 0, 0, 0};  // layout of the last P2P TLq-HS call (drain on change)
  bool tlq_layout_valid = false;
  size_t fused_limit = 0;             // P2P qWD steps with numel <= this run as one kernel (k_fused.cu)
  size_t fused_limit_tlq = 0;         // P2P TLq-HS calls likewise
  bool local_fusion = true;           // world 1: TLq-HS as one kernel (k_local.cu)
  uint32_t* fused_ctr = nullptr;      // counter blocks of the one-launch kernels (qWD, TLq-HS)
  unsigned long long timeout_ns = 0;  // > 0: flag waits are polling kernels with this deadline
  uint32_t* err_host = nullptr;       // host-mapped error word written by a timed-out wait
  uint32_t* err_dev = nullptr;
  PFN_cuStreamWriteValue32_v11070 write_value = nullptr;
  PFN_cuStreamWaitValue32_v11070 wait_value = nullptr;
  PFN_cuStreamBatchMemOp_v11070 batch_memop = nullptr;  // all flag writes / waits of a step in one call
  int device = 0;
  int sm_count = 148;
  int nccl_ctas = kDefaultNcclCtas;
  int chunks_cfg = 0;  // 0 = auto
  int pull_num = -1, pull_den = 2;  // P2P intra all-to-all: share of peer tiles pulled by K4 (IntraPull); -1 = auto
  ncclComm_t world_c = nullptr, intra = nullptr, inter = nullptr;
  cudaStream_t side = nullptr;
  uint64_t launches = 0;
  bool profiling = false;
  struct Pending {
    const char* name;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> pool;
  std::vector<cudaEvent_t> deps;  // dependency events (timing disabled), reused round-robin
  size_t dep_next = 0;
  std::map<std::string, std::pair<double, uint64_t>> acc;
  std::vector<std::string> names_keep;

  cudaEvent_t ev() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  // A dependency event: record on `from`, make `to` wait for it.
  void link(cudaStream_t from, cudaStream_t to) {
    if (deps.empty()) {
      deps.resize(64);
      for (auto& e : deps) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    }
    cudaEvent_t e = deps[dep_next++ % deps.size()];
    cudaEventRecord(e, from);
    cudaStreamWaitEvent(to, e, 0);
  }
  int chunks(size_t S) const {
    if (world == 1) return 1;
    if (chunks_cfg > 0) return std::min(chunks_cfg, kMaxChunks);
    if (transport == kTransportP2P) return 1;  // chunking gains ~2%; opt in with set_chunks
    const size_t c = S / ((size_t)16 << 20);  // ~16M elements per chunk and shard
    return (int)std::max<size_t>(1, std::min<size_t>(c, 8));
  }
  int sms(bool overlap) const { return overlap ? std::max(1, sm_count - nccl_ctas) : sm_count; }
};

namespace {

// Launch wrapper: counts launches and (optionally) brackets them with events.
template <typename F>
sdp4_status launch(sdp4_comm* c, const char* name, cudaStream_t st, F&& f) {
  cudaEvent_t a = nullptr, b = nullptr;
  if (c->profiling) {
    a = c->ev();
    b = c->ev();
    cudaEventRecord(a, st);
  }
  cudaError_t e = f();
  if (e != cudaSuccess) return fail(SDP4_ECUDA, "%s launch failed: %s", name, cudaGetErrorString(e));
  c->launches++;
  if (c->profiling) {
    cudaEventRecord(b, st);
    c->pending.push_back({name, a, b});
  }
  return SDP4_OK;
}

sdp4_status nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) return fail(SDP4_ENCCL, "%s: %s", what, ncclGetErrorString(r));
  return SDP4_OK;
}

// NCCL call on stream `st`, bracketed by profiling events like the kernels.
template <typename F>
sdp4_status nccl_op(sdp4_comm* c, const char* name, cudaStream_t st, F&& f) {
  cudaEvent_t a = nullptr, b = nullptr;
  if (c->profiling) {
    a = c->ev();
    b = c->ev();
    cudaEventRecord(a, st);
  }
  sdp4_status s = nccl_check(f(), name);
  if (s != SDP4_OK) return s;
  if (c->profiling) {
    cudaEventRecord(b, st);
    c->pending.push_back({name, a, b});
  }
  return SDP4_OK;
}

// Errors raised asynchronously by earlier calls: NCCL's, and a P2P flag wait that timed out
// (the comm is then unusable: the exchange it guarded never completed).
sdp4_status async_check(sdp4_comm* c) {
  if (c->err_host) {
    const uint32_t e = *reinterpret_cast<volatile uint32_t*>(c->err_host);
    if (e)
      return fail(SDP4_ETIMEOUT, "a P2P wait timed out: %s flag of stage %u from rank %u never arrived; the comm is "
                                 "unusable (destroy it)",
                  ((e >> 24) & 1) ? "free" : "data", (e >> 16) & 0xff, e & 0xffff);
  }
  ncclComm_t cs[3] = {c->world_c, c->intra, c->inter};
  for (ncclComm_t x : cs) {
    if (!x) continue;
    ncclResult_t ar = ncclSuccess;
    ncclCommGetAsyncError(x, &ar);
    if (ar != ncclSuccess && ar != ncclInProgress)
      return fail(SDP4_ENCCL, "asynchronous NCCL error: %s", ncclGetErrorString(ar));
  }
  return SDP4_OK;
}

// Host allgather of `bytes` per rank (rank-major into recv) over the bootstrap channel.
sdp4_status host_allgather(sdp4_comm* c, const void* send, void* recv, size_t bytes) {
  if (c->world == 1) {
    memcpy(recv, send, bytes);
    return SDP4_OK;
  }
  if (c->ag_fn) {
    if (c->ag_fn(send, recv, bytes, c->ag_ctx) != 0) return fail(SDP4_ESTATE, "host allgather callback failed");
    return SDP4_OK;
  }
  if (!c->world_c) return fail(SDP4_ESTATE, "no bootstrap channel");
  uint8_t* d = nullptr;
  cudaError_t e = cudaMalloc(&d, bytes * c->world);
  if (e != cudaSuccess) return fail(SDP4_ECUDA, "bootstrap buffer: %s", cudaGetErrorString(e));
  cudaMemcpy(d + bytes * c->rank, send, bytes, cudaMemcpyHostToDevice);
  ncclResult_t r = ncclAllGather(d + bytes * c->rank, d, bytes, ncclUint8, c->world_c, c->side);
  cudaStreamSynchronize(c->side);
  e = cudaMemcpy(recv, d, bytes * c->world, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (r != ncclSuccess) return fail(SDP4_ENCCL, "bootstrap allgather: %s", ncclGetErrorString(r));
  return e == cudaSuccess ? SDP4_OK : fail(SDP4_ECUDA, "bootstrap copy: %s", cudaGetErrorString(e));
}
// Host allgather of one status byte per rank; returns the first failing rank or -1.
int host_agree(sdp4_comm* c, bool ok, sdp4_status* st) {
  std::vector<uint8_t> all(c->world);
  const uint8_t mine = ok ? 1 : 0;
  *st = host_allgather(c, &mine, all.data(), 1);
  if (*st != SDP4_OK) return c->rank;
  for (int q = 0; q < c->world; ++q)
    if (!all[q]) return q;
  return -1;
}

PeerInfo my_peer_info(int device) {
  PeerInfo pi;
  memset(&pi, 0, sizeof(pi));
  char host[64] = {0}, boot[40] = {0};
  gethostname(host, sizeof(host) - 1);
  if (FILE* f = fopen("/proc/sys/kernel/random/boot_id", "r")) {
    if (!fgets(boot, sizeof(boot), f)) boot[0] = 0;
    fclose(f);
  }
  for (char* p = boot; *p; ++p)
    if (*p == '\n') *p = 0;
  snprintf(pi.host, sizeof(pi.host), "%s/%s", host, boot);
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) == cudaSuccess) memcpy(pi.uuid, &prop.uuid, 16);
  pi.pid = (int)getpid();
  return pi;
}

// Can this process map the memory of a peer described by `q` (CUDA IPC: same OS instance,
// the peer's device visible here and either this device or peer-accessible from it)?
bool reachable(const PeerInfo& me, const PeerInfo& q, int my_dev) {
  if (strncmp(me.host, q.host, sizeof(me.host)) != 0) return false;
  if (memcmp(me.uuid, q.uuid, 16) == 0) return true;  // ranks sharing one GPU (single-GPU emulation)
  int n = 0;
  cudaGetDeviceCount(&n);
  for (int d = 0; d < n; ++d) {
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, d) != cudaSuccess) continue;
    if (memcmp(&prop.uuid, q.uuid, 16) != 0) continue;
    int can = 0;
    cudaDeviceCanAccessPeer(&can, my_dev, d);
    return can != 0;
  }
  return false;
}

// Collective: decide whether the P2P transport is usable by every rank, and
// whether some ranks share a device.  Ranks sharing a GPU must never wait for one another in
// a kernel (nothing guarantees that kernels of different processes run concurrently; a
// spinning kernel can stall a context switch), so such a comm waits with stream memory
// operations only.
sdp4_status probe_p2p(sdp4_comm* c, bool* ok) {
  const PeerInfo me = my_peer_info(c->device);
  std::vector<PeerInfo> all(c->world);
  sdp4_status s = host_allgather(c, &me, all.data(), sizeof(PeerInfo));
  if (s != SDP4_OK) return s;
  bool mine = c->write_value && c->wait_value && c->N <= sdp4::kMaxN && c->M <= sdp4::kMaxDests &&
              c->world <= sdp4::kMaxDests;
  for (int q = 0; q < c->world && mine; ++q)
    if (q != c->rank && !reachable(me, all[q], c->device)) mine = false;
  for (int q = 0; q < c->world; ++q)
    for (int p = 0; p < q; ++p)
      if (memcmp(all[p].uuid, all[q].uuid, 16) == 0) c->shared_gpu = true;
  if (c->shared_gpu) c->timeout_ns = 0;
  const int bad = host_agree(c, mine, &s);
  if (s != SDP4_OK) return s;
  *ok = bad < 0;
  return SDP4_OK;
}

void sym_release(sdp4_comm* c, SymBuf& b) {
  for (size_t q = 0; q < b.peer.size(); ++q)
    if ((int)q != c->rank && b.peer[q]) cudaIpcCloseMemHandle(b.peer[q]);
  if (b.local) cudaFree(b.local);
  b = SymBuf();
}

bool capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
}

// Collectively (re)allocate a symmetric buffer whose region holds `region` bytes.  Every
// failure is agreed on by all ranks (each reports its status through the bootstrap channel),
// so either every rank returns with a complete mapping or every rank returns the error with
// the buffer released -- never a partial mapping, never a rank left waiting in a barrier.
sdp4_status sym_ensure(sdp4_comm* c, SymBuf& b, size_t region, cudaStream_t st) {
  if (b.local && region <= b.region) return SDP4_OK;
  if (capturing(st))
    return fail(SDP4_ESTATE, "the symmetric buffer must grow to %zu bytes during stream capture: make one eager call "
                             "of the same size before capturing", region);
  region = round_up(region + region / 16, 1 << 21);
  cudaError_t e = cudaDeviceSynchronize();  // no kernel of ours still touches the old buffers
  sdp4_status s;
  if (b.local) {  // every rank synchronized: the peers are done with the old buffers
    int bad = host_agree(c, e == cudaSuccess, &s);
    if (s != SDP4_OK) return s;
    sym_release(c, b);
    if (bad >= 0) return fail(SDP4_ECUDA, "rank %d failed to synchronize before reallocation", bad);
  }
  struct Rec {
    cudaIpcMemHandle_t h;
    int ok;
  } mine;
  memset(&mine, 0, sizeof(mine));
  const size_t bytes = kFlagBytes + region;
  std::string why;
  if ((e = cudaMalloc(&b.local, bytes)) != cudaSuccess) {
    b.local = nullptr;
    why = std::string("cudaMalloc: ") + cudaGetErrorString(e);
  } else {
    // data flags 0 (nothing published), free flags 1 (every receive slot initially free)
    std::vector<uint32_t> init(kFlagBytes / 4, 0u);
    for (size_t i = flag_off(kFree, 0, 0) / 4; i < init.size(); ++i) init[i] = 1u;
    e = cudaMemcpy(b.local, init.data(), kFlagBytes, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(&mine.h, b.local);
    if (e != cudaSuccess) why = std::string("init/ipc handle: ") + cudaGetErrorString(e);
  }
  mine.ok = why.empty();
  b.bytes = bytes;
  b.region = region;
  std::vector<Rec> all(c->world);
  if ((s = host_allgather(c, &mine, all.data(), sizeof(Rec))) != SDP4_OK) {
    sym_release(c, b);
    return s;
  }
  int bad = -1;
  for (int q = 0; q < c->world && bad < 0; ++q)
    if (!all[q].ok) bad = q;
  if (bad < 0) {
    b.peer.assign(c->world, nullptr);
    for (int q = 0; q < c->world; ++q) {
      if (q == c->rank) {
        b.peer[q] = b.local;
        continue;
      }
      void* p = nullptr;
      if ((e = cudaIpcOpenMemHandle(&p, all[q].h, cudaIpcMemLazyEnablePeerAccess)) != cudaSuccess) {
        cudaGetLastError();
        why = "open peer " + std::to_string(q) + " buffer: " + cudaGetErrorString(e);
        break;
      }
      b.peer[q] = static_cast<uint8_t*>(p);
    }
    if (why.empty() && (e = cudaDeviceSynchronize()) != cudaSuccess)  // flags initialized before any peer signals
      why = std::string("sync: ") + cudaGetErrorString(e);
    bad = host_agree(c, why.empty(), &s);
    if (s != SDP4_OK) {
      sym_release(c, b);
      return s;
    }
  }
  if (bad >= 0) {
    sym_release(c, b);
    if (bad == c->rank) return fail(SDP4_ECUDA, "symmetric buffer of %zu bytes: %s", bytes, why.c_str());
    return fail(SDP4_ECUDA, "symmetric buffer of %zu bytes failed on rank %d", bytes, bad);
  }
  return SDP4_OK;
}

uint8_t* sym_region(const SymBuf& b, int rank) { return b.peer[rank] + kFlagBytes; }

// ---- P2P sync protocol --------------------------------------------------------------
// Binary flags, no epochs, so a captured graph replays correctly and the receive regions
// need no double buffering.  For an exchange from producer p to consumer q (q's receive
// region written by p, or p's own region read by q):
//   p: wait free[stage][q] (in p's buffer) -> produce -> raise data[stage][p] in q's buffer;
//   q: wait data[stage][p] (in q's buffer) -> consume -> raise free[stage][q] in p's buffer.
// Each wait resets the flag it saw.  q's reset of data happens before q's consume, which is
// before q raises free, which p waits for before it raises data again -- so a reset never
// erases a newer raise (and symmetrically for free).  Initial state: data 0, free 1.
struct Sig {
  int owner, kind, stage;  // raise owner's flag[kind][stage][me]
};
struct Wt {
  int kind, stage, src;  // wait for my flag[kind][stage][src]
};

sdp4_status raise_flags(sdp4_comm* c, cudaStream_t st, const SymBuf& b, const std::vector<Sig>& sigs) {
  std::vector<CUstreamBatchMemOpParams> ops;
  for (const Sig& g : sigs) {
    if (g.owner == c->rank) continue;
    const CUdeviceptr a = (CUdeviceptr)(b.peer[g.owner] + flag_off(g.kind, g.stage, c->rank));
    if (!c->batch_memop) {
      CUresult r = c->write_value((CUstream)st, a, 1u, CU_STREAM_WRITE_VALUE_DEFAULT);
      if (r != CUDA_SUCCESS) return fail(SDP4_ECUDA, "cuStreamWriteValue32 failed (%d)", (int)r);
      continue;
    }
    CUstreamBatchMemOpParams op;
    memset(&op, 0, sizeof(op));
    op.writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_32;
    op.writeValue.address = a;
    op.writeValue.value = 1u;
    op.writeValue.flags = CU_STREAM_WRITE_VALUE_DEFAULT;  // fenced after the stream's prior work
    ops.push_back(op);
  }
  if (ops.empty()) return SDP4_OK;
  CUresult r = c->batch_memop((CUstream)st, (unsigned)ops.size(), ops.data(), 0);
  return r == CUDA_SUCCESS ? SDP4_OK : fail(SDP4_ECUDA, "cuStreamBatchMemOp (raise) failed (%d)", (int)r);
}

// Wait for (and reset) my flags.  timeout_ns > 0: one polling kernel with a deadline (a missing
// peer sets the comm's error word instead of blocking the stream forever); 0: stream memory
// operations (cuStreamWaitValue32, unbounded).  With profiling on, the wait is timed as `name`.
sdp4_status wait_flags(sdp4_comm* c, cudaStream_t st, const SymBuf& b, const std::vector<Wt>& wts,
                       const char* name = "wait") {
  std::vector<Wt> w;
  for (const Wt& x : wts)
    if (x.src != c->rank) w.push_back(x);
  if (w.empty()) return SDP4_OK;
  cudaEvent_t ea = nullptr, eb = nullptr;
  if (c->profiling) {
    ea = c->ev();
    eb = c->ev();
    cudaEventRecord(ea, st);
  }
  if (c->timeout_ns) {
    if (w.size() > (size_t)sdp4::kMaxWait) return fail(SDP4_EINVAL, "too many flags to wait for");
    sdp4::FlagWait fw;
    memset(&fw, 0, sizeof(fw));
    fw.n = (int)w.size();
    fw.timeout_ns = c->timeout_ns;
    fw.err = c->err_dev;
    for (size_t i = 0; i < w.size(); ++i) {
      fw.flag[i] = reinterpret_cast<uint32_t*>(b.local + flag_off(w[i].kind, w[i].stage, w[i].src));
      fw.code[i] = 0x80000000u | ((uint32_t)w[i].kind << 24) | ((uint32_t)w[i].stage << 16) | (uint32_t)w[i].src;
    }
    cudaError_t e = sdp4::launch_wait_flags(fw, st);  // one of our kernels: counted as a launch
    if (e != cudaSuccess) return fail(SDP4_ECUDA, "flag-wait launch failed: %s", cudaGetErrorString(e));
    c->launches++;
  } else {
    std::vector<CUstreamBatchMemOpParams> waits, resets;
    for (const Wt& x : w) {
      const CUdeviceptr a = (CUdeviceptr)(b.local + flag_off(x.kind, x.stage, x.src));
      if (!c->batch_memop) {
        CUresult r = c->wait_value((CUstream)st, a, 1u, CU_STREAM_WAIT_VALUE_GEQ);
        if (r == CUDA_SUCCESS) r = c->write_value((CUstream)st, a, 0u, CU_STREAM_WRITE_VALUE_DEFAULT);
        if (r != CUDA_SUCCESS) return fail(SDP4_ECUDA, "cuStreamWaitValue32 failed (%d)", (int)r);
        continue;
      }
      CUstreamBatchMemOpParams op;
      memset(&op, 0, sizeof(op));
      op.waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_32;
      op.waitValue.address = a;
      op.waitValue.value = 1u;
      op.waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ;
      waits.push_back(op);
      memset(&op, 0, sizeof(op));
      op.writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_32;
      op.writeValue.address = a;
      op.writeValue.value = 0u;
      op.writeValue.flags = CU_STREAM_WRITE_VALUE_DEFAULT;
      resets.push_back(op);
    }
    if (!waits.empty()) {
      CUresult r = c->batch_memop((CUstream)st, (unsigned)waits.size(), waits.data(), 0);
      if (r == CUDA_SUCCESS) r = c->batch_memop((CUstream)st, (unsigned)resets.size(), resets.data(), 0);
      if (r != CUDA_SUCCESS) return fail(SDP4_ECUDA, "cuStreamBatchMemOp (wait) failed (%d)", (int)r);
    }
  }
  if (c->profiling) {
    cudaEventRecord(eb, st);
    c->pending.push_back({name, ea, eb});
  }
  return SDP4_OK;
}

sdp4_status check_ptr(const void* p, const char* what) {
  if (!p) return fail(SDP4_EINVAL, "%s is NULL", what);
  if (reinterpret_cast<uintptr_t>(p) % 16) return fail(SDP4_EALIGN, "%s is not 16-byte aligned", what);
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(SDP4_EINVAL, "%s: not a CUDA pointer (%s)", what, cudaGetErrorString(e));
  }
  if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged)
    return fail(SDP4_EINVAL, "%s must be a device pointer", what);
  return SDP4_OK;
}

// The caller's workspace is only used by the NCCL transport (and at world 1); with the P2P
// transport the exchanges go through library-owned symmetric buffers, so it may be NULL.
sdp4_status check_workspace(const sdp4_comm* c, const void* ws, size_t bytes, size_t need) {
  if (c->transport == kTransportP2P && c->world > 1) return SDP4_OK;
  sdp4_status s = check_ptr(ws, "workspace");
  if (s != SDP4_OK) return s;
  if (bytes < need) return fail(SDP4_ESTATE, "workspace %zu < %zu bytes", bytes, need);
  return SDP4_OK;
}

// R1: numel % (P * lcm(G, 64)) == 0, G power of two in [32, 2048].
sdp4_status check_sizes(int P, size_t numel, int group) {
  if (!is_pow2(group) || group < 32 || group > 2048)
    return fail(SDP4_EINVAL, "group size %d must be a power of two in [32, 2048]", group);
  const size_t align = (size_t)P * (size_t)(group > 64 ? group : 64);
  if (numel == 0 || numel % align)
    return fail(SDP4_EALIGN, "numel %zu must be a nonzero multiple of P*lcm(G,64) = %zu (zero-pad)", numel,
                align);
  return SDP4_OK;
}

sdp4_status check_tlq_args(int P, size_t numel, int bi, int be, int group, int b) {
  if (!valid_bits(bi) || !valid_bits(be)) return fail(SDP4_EINVAL, "bits (%d, %d) not in {4, 8, 32}", bi, be);
  if (b != 0 && (!is_pow2(b) || b < 2 || b > 256))
    return fail(SDP4_EINVAL, "hadamard_block %d not in {0, 2, 4, ..., 256}", b);
  sdp4_status s = check_sizes(P, numel, group);
  if (s != SDP4_OK) return s;
  if (b > group) return fail(SDP4_EALIGN, "group %d must be divisible by hadamard_block %d (P:395)", group, b);
  return SDP4_OK;
}

// R6/R8 constants: c_b = rn(1/sqrt(b)); kappa = rn(c_b / P) (average) or c_b; b = 0: rn(1/P) or 1.
float hadamard_cb(int b) { return b ? (float)(1.0 / std::sqrt((double)b)) : 1.0f; }
float final_kappa(int b, int P, int average) {
  const float cb = hadamard_cb(b);
  return average ? (b ? cb / (float)P : 1.0f / (float)P) : cb;
}

int sm_count_current() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

size_t esize(sdp4_dtype d) { return d == SDP4_BF16 ? 2 : 4; }

// Stochastic rounding key (R14): key = mix32(seed_lo ^ mix32(seed_hi ^ (stage << 24) ^ rank)).
uint32_t mix32_host(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}
enum { kStageQwd = 1, kStageIntra = 2, kStageInter = 3 };
uint32_t sr_key(uint64_t seed, int stage, int rank) {
  return mix32_host((uint32_t)seed ^ mix32_host((uint32_t)(seed >> 32) ^ ((uint32_t)stage << 24) ^ (uint32_t)rank));
}
bool valid_round(sdp4_round r) { return r == SDP4_RNE || r == SDP4_STOCHASTIC; }

}  // namespace

namespace {
sdp4_status check_topology(sdp4_comm_t* out, int rank, int world, int groups_M, int group_size_N) {
  if (!out) return fail(SDP4_EINVAL, "out is NULL");
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world) return fail(SDP4_EINVAL, "bad rank %d / world %d", rank, world);
  if (groups_M < 1 || group_size_N < 1 || groups_M * group_size_N != world)
    return fail(SDP4_EINVAL, "groups_M (%d) * group_size_N (%d) != world (%d)", groups_M, group_size_N, world);
  return SDP4_OK;
}

sdp4_comm* comm_new(int rank, int world, int groups_M, int group_size_N, int nccl_ctas) {
  sdp4_comm* c = new sdp4_comm();
  c->rank = rank;
  c->world = world;
  c->M = groups_M;
  c->N = group_size_N;
  c->m = rank / group_size_N;
  c->l = rank % group_size_N;
  c->nccl_ctas = nccl_ctas ? nccl_ctas : kDefaultNcclCtas;
  if (getenv("SDP4_NO_LOCAL_FUSION")) c->local_fusion = false;  // measurement: K3 -> K4 -> K5 unfused
  cudaGetDevice(&c->device);
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, c->device);
  if (c->nccl_ctas >= c->sm_count) c->nccl_ctas = c->sm_count / 2;
  if (world > 1) {
    void* fw = nullptr;
    void* fwt = nullptr;
    void* fb = nullptr;
    cudaDriverEntryPointQueryResult q1, q2, q3;
    cudaGetDriverEntryPoint("cuStreamWriteValue32", &fw, cudaEnableDefault, &q1);
    cudaGetDriverEntryPoint("cuStreamWaitValue32", &fwt, cudaEnableDefault, &q2);
    cudaGetDriverEntryPoint("cuStreamBatchMemOp", &fb, cudaEnableDefault, &q3);
    c->write_value = reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(fw);
    c->wait_value = reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(fwt);
    c->batch_memop = reinterpret_cast<PFN_cuStreamBatchMemOp_v11070>(fb);
    if (getenv("SDP4_NO_BATCH_MEMOP")) c->batch_memop = nullptr;  // measurement switch
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, hi);
    // the error word a timed-out flag wait writes (host-mapped: readable without a sync)
    if (cudaHostAlloc(&c->err_host, sizeof(uint32_t), cudaHostAllocMapped) == cudaSuccess) {
      *c->err_host = 0;
      cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->err_dev), c->err_host, 0);
    } else {
      c->err_host = nullptr;
      cudaGetLastError();
    }
    double sec = kDefaultTimeoutS;
    if (const char* e = getenv("SDP4_WAIT_TIMEOUT_S")) sec = atof(e);
    c->timeout_ns = (sec > 0 && c->err_dev) ? (unsigned long long)(sec * 1e9) : 0ull;
    // one-launch small-message path; counters zeroed once, then by the kernels
    if (cudaMalloc(&c->fused_ctr, 2 * sdp4::kFusedCtrWords * sizeof(uint32_t)) == cudaSuccess &&
        cudaMemset(c->fused_ctr, 0, 2 * sdp4::kFusedCtrWords * sizeof(uint32_t)) == cudaSuccess) {
      c->fused_limit = kDefaultFusedLimit;
      c->fused_limit_tlq = kDefaultFusedLimitTlq;
      if (const char* e = getenv("SDP4_FUSED_MAX_NUMEL")) c->fused_limit = c->fused_limit_tlq = strtoull(e, nullptr, 10);
    } else {
      cudaGetLastError();
      if (c->fused_ctr) cudaFree(c->fused_ctr);
      c->fused_ctr = nullptr;
    }
  }
  return c;
}

// SDP4_FUSED_TRACE=1 (debugging only): every one-launch call records %globaltimer stamps of its
// phases (private per warp / CTA), synchronizes, and prints one JSON line to stderr, in us from
// the earliest entry: [last exit, A first start, A last end, B first start, B last end, C first
// start, C last end] (-1: no such phase).
struct FusedTrace {
  unsigned long long* host = nullptr;
  unsigned long long* dev = nullptr;
};
constexpr size_t kTraceWords = (size_t)sdp4::kTraceUnits * sdp4::kTraceSlots;
FusedTrace* fused_trace() {
  static FusedTrace t;
  static bool init = false;
  if (!init) {
    init = true;
    if (getenv("SDP4_FUSED_TRACE") && cudaMalloc(&t.dev, kTraceWords * 8) == cudaSuccess) {
      t.host = static_cast<unsigned long long*>(malloc(kTraceWords * 8));
    } else {
      cudaGetLastError();
      t.dev = nullptr;
    }
  }
  return t.dev ? &t : nullptr;
}
void trace_begin(sdp4::FusedSync& fs) {
  FusedTrace* t = fused_trace();
  if (!t) return;
  cudaMemset(t->dev, 0, kTraceWords * 8);
  fs.trace = t->dev;
}
void trace_end(const char* what, const sdp4::FusedSync& fs, cudaStream_t st) {
  FusedTrace* t = fused_trace();
  if (!t) return;
  cudaStreamSynchronize(st);
  cudaMemcpy(t->host, t->dev, kTraceWords * 8, cudaMemcpyDeviceToHost);
  unsigned long long agg[sdp4::kTraceSlots];
  for (int k = 0; k < sdp4::kTraceSlots; ++k) agg[k] = (k & 1) ? 0ull : ~0ull;
  for (int u = 0; u < sdp4::kTraceUnits; ++u)
    for (int k = 0; k < sdp4::kTraceSlots; ++k) {
      const unsigned long long y = t->host[(size_t)u * sdp4::kTraceSlots + k];
      if (!y) continue;
      agg[k] = (k & 1) ? std::max(agg[k], y) : std::min(agg[k], y);
    }
  std::string line = std::string("{\"fused_trace\": \"") + what + "\", \"rank\": " + std::to_string(fs.rank[0]) +
                     ", \"nv\": " + std::to_string(fs.nv) + ", \"us\": [";
  for (int k = 1; k < sdp4::kTraceSlots; ++k) {
    const unsigned long long y = agg[k];
    char b[32];
    snprintf(b, sizeof(b), "%s%.2f", k > 1 ? ", " : "",
             (y == 0 || y == ~0ull || agg[0] == ~0ull) ? -1.0 : (double)(long long)(y - agg[0]) * 1e-3);
    line += b;
  }
  fprintf(stderr, "%s]}\n", line.c_str());
}

// The one-launch path needs distinct GPUs (its kernels poll for other ranks' kernels, which
// processes sharing one GPU cannot guarantee to run concurrently).
bool use_fused(const sdp4_comm* c, size_t numel, bool tlq) {
  return c->transport == kTransportP2P && c->world > 1 && !c->shared_gpu && c->fused_ctr &&
         numel <= (tlq ? c->fused_limit_tlq : c->fused_limit);
}

void comm_free(sdp4_comm* c) {
  if (c->inter) ncclCommDestroy(c->inter);
  if (c->intra) ncclCommDestroy(c->intra);
  if (c->world_c) ncclCommDestroy(c->world_c);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->err_host) cudaFreeHost(c->err_host);
  if (c->fused_ctr) cudaFree(c->fused_ctr);
  delete c;
}
}  // namespace

extern "C" {

int sdp4_version(void) { return 200; }

const char* sdp4_last_error(void) { return g_err.c_str(); }

sdp4_status sdp4_get_unique_id(unsigned char id[SDP4_UNIQUE_ID_BYTES]) {
  if (!id) return fail(SDP4_EINVAL, "id is NULL");
  static_assert(sizeof(ncclUniqueId) == SDP4_UNIQUE_ID_BYTES, "ncclUniqueId size");
  ncclUniqueId u;
  sdp4_status s = nccl_check(ncclGetUniqueId(&u), "ncclGetUniqueId");
  if (s != SDP4_OK) return s;
  memcpy(id, &u, sizeof(u));
  return SDP4_OK;
}


sdp4_status sdp4_comm_init(sdp4_comm_t* out, const unsigned char* id, int rank, int world, int groups_M,
                           int group_size_N, int nccl_ctas) {
  NvtxRange nvtx_("sdp4_comm_init");
  sdp4_status s = check_topology(out, rank, world, groups_M, group_size_N);
  if (s != SDP4_OK) return s;
  if (world > 1 && !id) return fail(SDP4_EINVAL, "id is NULL with world > 1");
  if (nccl_ctas < 0) return fail(SDP4_EINVAL, "nccl_ctas must be >= 0");
  sdp4_comm* c = comm_new(rank, world, groups_M, group_size_N, nccl_ctas);
  if (world > 1) {
    ncclUniqueId u;
    memcpy(&u, id, sizeof(u));
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.maxCTAs = c->nccl_ctas;
    s = nccl_check(ncclCommInitRankConfig(&c->world_c, world, u, rank, &cfg), "ncclCommInitRankConfig");
    if (s == SDP4_OK && group_size_N > 1) {
      ncclConfig_t cfg2 = NCCL_CONFIG_INITIALIZER;
      cfg2.maxCTAs = c->nccl_ctas;
      s = nccl_check(ncclCommSplit(c->world_c, c->m, c->l, &c->intra, &cfg2), "ncclCommSplit(intra)");
    }
    if (s == SDP4_OK && groups_M > 1) {
      ncclConfig_t cfg3 = NCCL_CONFIG_INITIALIZER;
      cfg3.maxCTAs = c->nccl_ctas;
      s = nccl_check(ncclCommSplit(c->world_c, c->l, c->m, &c->inter, &cfg3), "ncclCommSplit(inter)");
    }
    // P2P (the default) only if every rank reaches every other through CUDA IPC
    if (s == SDP4_OK) s = probe_p2p(c, &c->p2p_ok);
    if (s != SDP4_OK) {
      comm_free(c);
      return s;
    }
    c->transport = c->p2p_ok ? kTransportP2P : kTransportNccl;
  }
  *out = c;
  return SDP4_OK;
}

sdp4_status sdp4_comm_init_p2p(sdp4_comm_t* out, int rank, int world, int groups_M, int group_size_N,
                               sdp4_host_allgather_fn allgather, void* ctx) {
  NvtxRange nvtx_("sdp4_comm_init_p2p");
  sdp4_status s = check_topology(out, rank, world, groups_M, group_size_N);
  if (s != SDP4_OK) return s;
  if (world > 1 && !allgather) return fail(SDP4_EINVAL, "allgather callback is NULL with world > 1");
  sdp4_comm* c = comm_new(rank, world, groups_M, group_size_N, 0);
  c->ag_fn = allgather;
  c->ag_ctx = ctx;
  if (world > 1) {
    s = probe_p2p(c, &c->p2p_ok);
    if (s == SDP4_OK && !c->p2p_ok)
      s = fail(SDP4_ESTATE, "P2P transport unavailable: some rank cannot map another's memory with CUDA IPC "
                            "(different hosts, or no peer access); use sdp4_comm_init (NCCL)");
    if (s != SDP4_OK) {
      comm_free(c);
      return s;
    }
    c->transport = kTransportP2P;
  }
  *out = c;
  return SDP4_OK;
}

sdp4_status sdp4_comm_destroy(sdp4_comm_t c) {
  NvtxRange nvtx_("sdp4_comm_destroy");
  if (!c) return fail(SDP4_EINVAL, "comm is NULL");
  if (c->side) cudaStreamSynchronize(c->side);
  for (auto& p : c->pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : c->pool) cudaEventDestroy(e);
  for (auto e : c->deps) cudaEventDestroy(e);
  sdp4_status s = SDP4_OK;
  if (c->sym_qwd.local || c->sym_tlq.local || c->sym_ring.local) {
    // peers may still be reading this rank's symmetric buffers (K2 / K4 pulls): every rank
    // finishes its own work, then a barrier, then the mappings are closed and freed
    const cudaError_t e = cudaDeviceSynchronize();
    host_agree(c, e == cudaSuccess, &s);
    for (SymBuf* b : {&c->sym_qwd, &c->sym_tlq, &c->sym_ring}) sym_release(c, *b);
  }
  comm_free(c);
  return s;
}

sdp4_status sdp4_comm_set_timeout(sdp4_comm_t c, double seconds) {
  if (!c) return fail(SDP4_EINVAL, "comm is NULL");
  if (!(seconds >= 0)) return fail(SDP4_EINVAL, "timeout must be >= 0");
  if (seconds > 0 && c->world > 1 && !c->err_dev) return fail(SDP4_ESTATE, "no host-mapped error word");
  if (seconds > 0 && c->shared_gpu)
    return fail(SDP4_EINVAL, "ranks share a GPU: flag waits must be stream memory operations (timeout 0), never "
                             "polling kernels");
  c->timeout_ns = (unsigned long long)(seconds * 1e9);
  return SDP4_OK;
}

sdp4_status sdp4_comm_check(sdp4_comm_t c) {
  if (!c) return fail(SDP4_EINVAL, "comm is NULL");
  g_err.clear();
  return async_check(c);
}

sdp4_status sdp4_comm_set_chunks(sdp4_comm_t c, int chunks) {
  if (!c) return fail(SDP4_EINVAL, "comm is NULL");
  if (chunks < 0 || chunks > kMaxChunks) return fail(SDP4_EINVAL, "chunks %d not in [0, %d]", chunks, kMaxChunks);
  c->chunks_cfg = chunks;
  return SDP4_OK;
}

sdp4_status sdp4_comm_set_intra_pull(sdp4_comm_t c, int num, int den) {
  if (!c) return fail(SDP4_EINVAL, "comm is NULL");
  if (den < 1 || den > 64 || num < 0 || num > den) return fail(SDP4_EINVAL, "intra pull %d/%d not in [0, 1]", num, den);
  c->pull_num = num;
  c->pull_den = den;
  return SDP4_OK;
}

sdp4_status sdp4_comm_set_fused_limit(sdp4_comm_t c, size_t numel) {
  if (!c) return fail(SDP4_EINVAL, "comm is NULL");
  c->fused_limit = c->fused_limit_tlq = numel;
  return SDP4_OK;
}

sdp4_status sdp4_comm_set_local_fusion(sdp4_comm_t c, int enable) {
  if (!c) return fail(SDP4_EINVAL, "comm is NULL");
  c->local_fusion = enable != 0;
  return SDP4_OK;
}

sdp4_status sdp4_comm_set_transport(sdp4_comm_t c, int transport) {
  if (!c) return fail(SDP4_EINVAL, "comm is NULL");
  if (transport != kTransportNccl && transport != kTransportP2P) return fail(SDP4_EINVAL, "bad transport %d", transport);
  if (transport == kTransportP2P && (c->world == 1 || !c->p2p_ok))
    return fail(SDP4_EINVAL, "P2P transport unavailable for this comm (world 1, or CUDA IPC does not reach every rank)");
  if (transport == kTransportNccl && c->world > 1 && !c->world_c)
    return fail(SDP4_EINVAL, "this comm has no NCCL communicators (sdp4_comm_init_p2p)");
  c->transport = transport;
  return SDP4_OK;
}

int sdp4_comm_transport(sdp4_comm_t c) { return c ? c->transport : -1; }

int sdp4_comm_chunks(sdp4_comm_t c, size_t numel, int group) {
  if (!c || numel % (size_t)c->world) return 0;
  return (int)plan_chunks(numel / c->world, c->chunks(numel / c->world), group).size();
}

size_t sdp4_wire_unit_bytes(size_t n, int bits, int group) {
  if (!valid_wbits(bits) || !is_pow2(group)) return 0;
  return unit_bytes(n, bits, group);
}

size_t sdp4_qwd_workspace_bytes(int world, size_t numel, int bits, int group) {
  if (world < 1 || !valid_wbits(bits) || !is_pow2(group) || numel % (size_t)world) return 0;
  size_t m = 0;
  for (int C = 1; C <= kMaxChunks; ++C) m = std::max(m, qwd_total(world, numel / world, bits, group, C));
  return m;
}

size_t sdp4_tlq_workspace_bytes(int M, int N, size_t numel, int bi, int be, int group) {
  if (M < 1 || N < 1 || !valid_bits(bi) || !valid_bits(be) || !is_pow2(group) || numel % ((size_t)M * N))
    return 0;
  size_t m = 0;
  for (int C = 1; C <= kMaxChunks; ++C) m = std::max(m, tlq_total(M, N, numel / ((size_t)M * N), bi, be, group, C));
  return m;
}

size_t sdp4_tlq_workspace_offset(int M, int N, size_t numel, int bi, int be, int group, int region) {
  if (region < 0 || region > 3 || sdp4_tlq_workspace_bytes(M, N, numel, bi, be, group) == 0) return 0;
  const TlqRegions r = tlq_regions(M, N, numel / ((size_t)M * N), bi, be, group, 0);
  const size_t offs[4] = {r.send8, r.recv8, r.send4, r.recv4};
  return offs[region];
}

namespace {
// Alg. 2 l.2-3 (qWD, diff) or Alg. 1's "Quantize weights" (qW, !diff: w_model_full unused).
sdp4_status weight_quantize(sdp4_comm_t c, bool diff, const float* w_main_shard, const void* w_model_full,
                            sdp4_dtype model_dtype, size_t numel, int bits, int group, sdp4_round rnd, uint64_t seed,
                            void* workspace, size_t workspace_bytes, void* stream, const char* kname,
                            bool apply_own = false) {
  g_err.clear();
  if (!c) return fail(SDP4_EINVAL, "comm is NULL");
  if (!valid_round(rnd)) return fail(SDP4_EINVAL, "bad rounding mode %d", (int)rnd);
  if (!valid_wbits(bits)) return fail(SDP4_EINVAL, "bits %d not in {2, 4, 8, 32}", bits);
  if (diff && model_dtype != SDP4_F32 && model_dtype != SDP4_BF16) return fail(SDP4_EINVAL, "bad model dtype");
  sdp4_status s = check_sizes(c->world, numel, group);
  if (s != SDP4_OK) return s;
  if ((s = check_ptr(w_main_shard, "w_main_shard")) != SDP4_OK) return s;
  if (diff && (s = check_ptr(w_model_full, "w_model_full")) != SDP4_OK) return s;
  const size_t need = sdp4_qwd_workspace_bytes(c->world, numel, bits, group);
  if ((s = check_workspace(c, workspace, workspace_bytes, need)) != SDP4_OK) return s;
  if ((s = async_check(c)) != SDP4_OK) return s;
  const size_t S = numel / c->world;
  const size_t es = diff ? esize(model_dtype) : 0;
  const auto chunks = plan_chunks(S, c->chunks(S), group);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int sms = c->sms(chunks.size() > 1);
  const int sr = rnd == SDP4_STOCHASTIC;
  const uint32_t key = sr_key(seed, kStageQwd, c->rank);
  auto shard_of = [&](size_t off) -> const void* {
    return diff ? static_cast<const uint8_t*>(w_model_full) + ((size_t)c->rank * S + off) * es : nullptr;
  };
  if (c->transport == kTransportP2P) {
    // Alg. 2 l.2-3: K1 writes unit `rank` into this rank's own symmetric buffer and raises
    // data[0][rank] on every peer; the all-gather (l.4) is the pull inside each rank's K2.
    // Before overwriting the unit, wait until every peer's K2 of the previous call has read it.
    if (c->qwd_pending.valid)
      return fail(SDP4_ESTATE, "P2P: the unit of the previous quantize has not been applied yet (one outstanding "
                               "quantize per comm: call the matching allgather_apply first)");
    const size_t W = unit_bytes(S, bits, group);
    if ((s = sym_ensure(c, c->sym_qwd, W, st)) != SDP4_OK) return s;
    std::vector<Wt> frees;
    std::vector<Sig> datas;
    for (int q = 0; q < c->world; ++q) {
      frees.push_back({kFree, 0, q});
      datas.push_back({q, kData, 0});
    }
    if ((s = wait_flags(c, st, c->sym_qwd, frees, "wait_qwd_free")) != SDP4_OK) return s;
    sdp4::Dests d;
    d.n = 1;
    d.remote = 0;
    d.p[0] = sym_region(c->sym_qwd, c->rank);
    s = launch(c, kname, st, [&] {
      return sdp4::launch_qwd_quantize(w_main_shard, shard_of(0), model_dtype, S, bits, group, d, sr, key,
                                       (uint64_t)c->rank * S, c->sm_count, st, apply_own);
    });
    if (s != SDP4_OK) return s;
    if ((s = raise_flags(c, st, c->sym_qwd, datas)) != SDP4_OK) return s;
    c->qwd_pending.valid = true;
    c->qwd_pending.numel = numel;
    c->qwd_pending.bits = bits;
    c->qwd_pending.group = group;
    return SDP4_OK;
  }
  uint8_t* region = static_cast<uint8_t*>(workspace);
  for (const Chunk& ch : chunks) {  // Alg. 2 l.2-3 per chunk: unit (chunk, rank)
    const size_t W = unit_bytes(ch.len, bits, group);
    sdp4::Dests d;
    d.n = 1;
    d.remote = 0;
    d.p[0] = region + (size_t)c->rank * W;
    s = launch(c, kname, st, [&] {
      return sdp4::launch_qwd_quantize(w_main_shard + ch.off, shard_of(ch.off), model_dtype, ch.len, bits, group, d,
                                       sr, key, (uint64_t)c->rank * S + ch.off, sms, st, apply_own);
    });
    if (s != SDP4_OK) return s;
    region += (size_t)c->world * W;
  }
  return SDP4_OK;
}

// Alg. 2 l.4-5 (qWD: add) or Alg. 1's "AllGather" + dequantize (qW: assign).
sdp4_status weight_apply(sdp4_comm_t c, void* workspace, size_t workspace_bytes, size_t numel, int bits, int group,
                         void* w_model_full, sdp4_dtype model_dtype, void* stream, bool add, const char* kname,
                         bool skip_own = false) {
  g_err.clear();
  if (!c) return fail(SDP4_EINVAL, "comm is NULL");
  if (!valid_wbits(bits)) return fail(SDP4_EINVAL, "bits %d not in {2, 4, 8, 32}", bits);
  if (model_dtype != SDP4_F32 && model_dtype != SDP4_BF16) return fail(SDP4_EINVAL, "bad model dtype");
  sdp4_status s = check_sizes(c->world, numel, group);
  if (s != SDP4_OK) return s;
  if ((s = check_ptr(w_model_full, "w_model_full")) != SDP4_OK) return s;
  const size_t need = sdp4_qwd_workspace_bytes(c->world, numel, bits, group);
  if ((s = check_workspace(c, workspace, workspace_bytes, need)) != SDP4_OK) return s;
  if ((s = async_check(c)) != SDP4_OK) return s;
  const size_t S = numel / c->world;
  const size_t es = esize(model_dtype);
  const auto chunks = plan_chunks(S, c->chunks(S), group);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool overlap = chunks.size() > 1;
  const int sms = c->sms(overlap);
  const int P = c->world;
  if (P > sdp4::kMaxDests) return fail(SDP4_EINVAL, "world %d > %d", P, sdp4::kMaxDests);
  if (skip_own && P == 1) return SDP4_OK;  // the only unit was applied by K1 (flags are >= waits)
  if (c->transport == kTransportP2P) {  // wait for every rank's unit; K2 pulls unit j from rank j
    const auto& pd = c->qwd_pending;
    if (!pd.valid || !c->sym_qwd.local)
      return fail(SDP4_ESTATE, "P2P: no quantized unit is pending (call qwd_quantize / qw_quantize first)");
    if (pd.numel != numel || pd.bits != bits || pd.group != group)
      return fail(SDP4_ESTATE, "P2P: apply (numel %zu, bits %d, G %d) does not match the pending quantize (numel %zu, "
                               "bits %d, G %d)", numel, bits, group, pd.numel, pd.bits, pd.group);
    std::vector<Wt> datas;
    std::vector<Sig> frees;
    for (int q = 0; q < P; ++q) {
      datas.push_back({kData, 0, q});
      frees.push_back({q, kFree, 0});
    }
    if ((s = wait_flags(c, st, c->sym_qwd, datas, "wait_qwd_allgather")) != SDP4_OK) return s;
    sdp4::Dests u;
    u.n = P;
    u.remote = ~0ull >> (64 - P) & ~(1ull << c->rank);  // peers' units (P <= 64)
    for (int q = 0; q < P; ++q) u.p[q] = sym_region(c->sym_qwd, q);
    s = launch(c, kname, st, [&] {
      return sdp4::launch_qwd_apply(u, P, S, S, bits, group, w_model_full, model_dtype, add, c->sm_count, st,
                                    c->rank, skip_own);
    });
    if (s != SDP4_OK) return s;
    c->qwd_pending.valid = false;
    return raise_flags(c, st, c->sym_qwd, frees);  // K2 is done reading every peer's unit
  }
  if (P > 1) c->link(st, c->side);  // the units of every chunk were written on st (K1)
  uint8_t* region = static_cast<uint8_t*>(workspace);
  for (const Chunk& ch : chunks) {
    const size_t W = unit_bytes(ch.len, bits, group);
    if (P > 1) {  // Alg. 2 l.4 AllGather of chunk c, in place, on the side stream
      s = nccl_op(c, "nccl_allgather_qwd", c->side, [&] {
        return ncclAllGather(region + (size_t)c->rank * W, region, W, ncclUint8, c->world_c, c->side);
      });
      if (s != SDP4_OK) return s;
      c->link(c->side, st);
    }
    // Alg. 2 l.5 for chunk c: every shard j's sub-range [j*S + off, +len) of the replica
    uint8_t* wm = static_cast<uint8_t*>(w_model_full) + ch.off * es;
    sdp4::Dests u;
    u.n = P;
    u.remote = 0;
    for (int q = 0; q < P && q < sdp4::kMaxDests; ++q) u.p[q] = region + (size_t)q * W;
    s = launch(c, kname, st, [&] {
      return sdp4::launch_qwd_apply(u, P, ch.len, S, bits, group, wm, model_dtype, add, sms, st,
                                    skip_own ? c->rank : 0, skip_own);
    });
    if (s != SDP4_OK) return s;
    region += (size_t)P * W;
  }
  return SDP4_OK;
}
}  // namespace

sdp4_status sdp4_qwd_quantize(sdp4_comm_t c, const float* w_main_shard, const void* w_model_full,
                              sdp4_dtype model_dtype, size_t numel, int bits, int group, sdp4_round rnd,
                              uint64_t seed, void* workspace, size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_("sdp4_qwd_quantize");
  return weight_quantize(c, true, w_main_shard, w_model_full, model_dtype, numel, bits, group, rnd, seed, workspace,
                         workspace_bytes, stream, "K1_qwd_quantize");
}

sdp4_status sdp4_qwd_allgather_apply(sdp4_comm_t c, void* workspace, size_t workspace_bytes, size_t numel, int bits,
                                     int group, void* w_model_full, sdp4_dtype model_dtype, void* stream) {
  NvtxRange nvtx_("sdp4_qwd_allgather_apply");
  return weight_apply(c, workspace, workspace_bytes, numel, bits, group, w_model_full, model_dtype, stream, true,
                      "K2_qwd_apply");
}

sdp4_status sdp4_qwd_step(sdp4_comm_t c, const float* w_main_shard, void* w_model_full, sdp4_dtype model_dtype,
                          size_t numel, int bits, int group, sdp4_round rnd, uint64_t seed, void* workspace,
                          size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_("sdp4_qwd_step");
  if (c && use_fused(c, numel, false)) {  // small message: the whole step as one kernel per rank
    g_err.clear();
    if (!valid_round(rnd)) return fail(SDP4_EINVAL, "bad rounding mode %d", (int)rnd);
    if (!valid_wbits(bits)) return fail(SDP4_EINVAL, "bits %d not in {2, 4, 8, 32}", bits);
    if (model_dtype != SDP4_F32 && model_dtype != SDP4_BF16) return fail(SDP4_EINVAL, "bad model dtype");
    sdp4_status s = check_sizes(c->world, numel, group);
    if (s != SDP4_OK) return s;
    if ((s = check_ptr(w_main_shard, "w_main_shard")) != SDP4_OK) return s;
    if ((s = check_ptr(w_model_full, "w_model_full")) != SDP4_OK) return s;
    if ((s = async_check(c)) != SDP4_OK) return s;
    if (c->qwd_pending.valid)
      return fail(SDP4_ESTATE, "P2P: the unit of the previous quantize has not been applied yet (one outstanding "
                               "quantize per comm: call the matching allgather_apply first)");
    const size_t S = numel / c->world;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if ((s = sym_ensure(c, c->sym_qwd, unit_bytes(S, bits, group), st)) != SDP4_OK) return s;
    sdp4::FusedSync fs;
    memset(&fs, 0, sizeof(fs));
    for (int q = 0; q < c->world; ++q) {
      fs.region[q] = sym_region(c->sym_qwd, q);
      fs.flags[q] = reinterpret_cast<uint32_t*>(c->sym_qwd.peer[q]);
    }
    fs.rank[0] = c->rank;
    fs.nv = 1;
    fs.P = c->world;
    fs.ctr = c->fused_ctr;
    fs.err = c->err_dev;
    fs.timeout_ns = c->timeout_ns;
    const uint32_t key = sr_key(seed, kStageQwd, c->rank);
    const float* wm = w_main_shard;
    void* wmod = w_model_full;
    trace_begin(fs);
    s = launch(c, "KF_qwd_step", st, [&] {
      return sdp4::launch_fused_qwd(fs, &wm, &wmod, model_dtype, S, bits, group, rnd == SDP4_STOCHASTIC, &key,
                                    c->sm_count, st);
    });
    trace_end("qwd", fs, st);
    return s;
  }
  sdp4_status s = weight_quantize(c, true, w_main_shard, w_model_full, model_dtype, numel, bits, group, rnd, seed,
                                  workspace, workspace_bytes, stream, "K1_qwd_quantize", true);
  if (s != SDP4_OK) return s;
  return weight_apply(c, workspace, workspace_bytes, numel, bits, group, w_model_full, model_dtype, stream, true,
                      "K2_qwd_apply", true);
}

sdp4_status sdp4_qw_quantize(sdp4_comm_t c, const float* w_main_shard, size_t numel, int bits, int group,
                             sdp4_round rnd, uint64_t seed, void* workspace, size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_("sdp4_qw_quantize");
  return weight_quantize(c, false, w_main_shard, nullptr, SDP4_F32, numel, bits, group, rnd, seed, workspace,
                         workspace_bytes, stream, "K1_qw_quantize");
}

sdp4_status sdp4_qw_allgather_apply(sdp4_comm_t c, void* workspace, size_t workspace_bytes, size_t numel, int bits,
                                    int group, void* w_model_full, sdp4_dtype model_dtype, void* stream) {
  NvtxRange nvtx_("sdp4_qw_allgather_apply");
  return weight_apply(c, workspace, workspace_bytes, numel, bits, group, w_model_full, model_dtype, stream, false,
                      "K2_qw_apply");
}

sdp4_status sdp4_tlq_hs_reduce_scatter(sdp4_comm_t c, const void* grad, sdp4_dtype grad_dtype, size_t numel,
                                       int bits_intra, int bits_inter, int group, int hadamard_block, int average,
                                       sdp4_round rnd, uint64_t seed, float* out_shard, void* workspace,
                                       size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_("sdp4_tlq_hs_reduce_scatter");
  g_err.clear();
  if (!c) return fail(SDP4_EINVAL, "comm is NULL");
  if (!valid_round(rnd)) return fail(SDP4_EINVAL, "bad rounding mode %d", (int)rnd);
  if (grad_dtype != SDP4_F32 && grad_dtype != SDP4_BF16) return fail(SDP4_EINVAL, "bad grad dtype");
  const int b = hadamard_block;
  sdp4_status s = check_tlq_args(c->world, numel, bits_intra, bits_inter, group, b);
  if (s != SDP4_OK) return s;
  if ((s = check_ptr(grad, "grad")) != SDP4_OK) return s;
  if ((s = check_ptr(out_shard, "out_shard")) != SDP4_OK) return s;
  const int M = c->M, N = c->N, P = c->world;
  const size_t S = numel / P;
  const auto chunks = plan_chunks(S, c->chunks(S), group);
  const int C = (int)chunks.size();
  // world 1, bits 8 / 4: one kernel (k_local.cu) that needs no workspace
  const bool local_fused = P == 1 && c->local_fusion && C == 1 && bits_intra == 8 && bits_inter == 4;
  const size_t need = sdp4_tlq_workspace_bytes(M, N, numel, bits_intra, bits_inter, group);
  if (!local_fused && (s = check_workspace(c, workspace, workspace_bytes, need)) != SDP4_OK) return s;
  if ((s = async_check(c)) != SDP4_OK) return s;

  const size_t es = esize(grad_dtype);
  const bool overlap = C > 1;
  const int sms = c->sms(overlap);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaStream_t cs = P > 1 ? c->side : st;  // communication stream
  const float cb = hadamard_cb(b), kappa = final_kappa(b, P, average);
  const int sr = rnd == SDP4_STOCHASTIC;
  const uint32_t key8 = sr_key(seed, kStageIntra, c->rank), key4 = sr_key(seed, kStageInter, c->rank);
  if (c->transport == kTransportP2P) {
    // Alg. 3 with both all-to-alls fused into the producing kernels: the intra one (l.4) split
    // between K3 pushes and K4 pulls (IntraPull), the inter one (l.10) pushed by K4.  With
    // C > 1 chunks (sub-ranges of every shard, independent end to end) the chunks alternate
    // between the caller's stream and the side stream, so K4/K5 of chunk k overlap the
    // NVLink-bound K3 of chunk k+1 (the overlap of P:344).  Symmetric region, per chunk:
    // [intra receive: N blocks][inter receive: M units][outbox: N blocks].
    // small messages: the whole reduce-scatter as one kernel per rank (push-only layout)
    const bool fused = C == 1 && use_fused(c, numel, true) && sdp4::fused_tlq_supported(bits_intra, bits_inter, b);
    const int pnum = fused ? 0 : c->pull_num >= 0 ? c->pull_num : (N <= 2 ? 0 : 1);  // auto split
    const int pden = c->pull_num >= 0 ? c->pull_den : 2;
    const bool pulling = N > 1 && pnum > 0;
    if (C > kMaxChunks) return fail(SDP4_EINVAL, "too many chunks");
    std::vector<size_t> base(C + 1, 0);
    for (int k = 0; k < C; ++k) {
      const size_t w8 = unit_bytes(chunks[k].len, bits_intra, group), w4 = unit_bytes(chunks[k].len, bits_inter, group);
      base[k + 1] = base[k] + (size_t)N * M * w8 * (pulling ? 2 : 1) + (size_t)M * w4;
    }
    if ((s = sym_ensure(c, c->sym_tlq, base[C], st)) != SDP4_OK) return s;
    const int m = c->m, l = c->l;
    std::vector<int> group_ranks(N), node_ranks(M);
    for (int q = 0; q < N; ++q) group_ranks[q] = m * N + q;
    for (int q = 0; q < M; ++q) node_ranks[q] = q * N + l;
    const uint32_t remote = ((1u << N) - 1u) & ~(1u << l);
    // Layout drain.  The receive regions are reused call after call, and a call's per-chunk
    // flags only order it against the SAME chunk of the previous call.  When the layout
    // changes (sizes, bit widths, G, chunk count or push/pull split), a region section of this
    // call can overlap a different section of the previous one, still being read by a peer's
    // K4 or K5.  So on a layout change every rank first waits until each exchange peer has
    // finished the previous call: a data/free round on a dedicated stage, raised in stream
    // order after the previous call's K5 (the same handshake as the data stages, so repeated
    // drains are safe and a captured graph replays correctly).
    {
      const uint64_t sig[6] = {numel, (uint64_t)bits_intra, (uint64_t)bits_inter, (uint64_t)group,
                               (uint64_t)C, (uint64_t)(pulling ? (pnum << 8 | pden) : 0)};
      const bool changed = c->tlq_layout_valid && memcmp(sig, c->tlq_layout, sizeof(sig)) != 0;
      memcpy(c->tlq_layout, sig, sizeof(sig));
      c->tlq_layout_valid = true;
      if (changed) {
        std::vector<int> peers;
        for (int q : group_ranks) peers.push_back(q);
        for (int q : node_ranks)
          if (std::find(peers.begin(), peers.end(), q) == peers.end()) peers.push_back(q);
        std::vector<Wt> wf, wd;
        std::vector<Sig> gd, gf;
        for (int q : peers) {
          wf.push_back({kFree, kDrainStage, q});
          gd.push_back({q, kData, kDrainStage});
          wd.push_back({kData, kDrainStage, q});
          gf.push_back({q, kFree, kDrainStage});
        }
        if ((s = wait_flags(c, st, c->sym_tlq, wf, "wait_tlq_drain")) != SDP4_OK) return s;
        if ((s = raise_flags(c, st, c->sym_tlq, gd)) != SDP4_OK) return s;
        if ((s = wait_flags(c, st, c->sym_tlq, wd, "wait_tlq_drain")) != SDP4_OK) return s;
        if ((s = raise_flags(c, st, c->sym_tlq, gf)) != SDP4_OK) return s;
      }
    }
    if (fused) {
      sdp4::FusedSync fs;
      memset(&fs, 0, sizeof(fs));
      for (int q = 0; q < P; ++q) {
        fs.region[q] = sym_region(c->sym_tlq, q);
        fs.flags[q] = reinterpret_cast<uint32_t*>(c->sym_tlq.peer[q]);
      }
      fs.rank[0] = c->rank;
      fs.nv = 1;
      fs.P = P;
      fs.ctr = c->fused_ctr + sdp4::kFusedCtrWords;
      fs.err = c->err_dev;
      fs.timeout_ns = c->timeout_ns;
      const void* g = grad;
      float* o = out_shard;
      trace_begin(fs);
      s = launch(c, "KF_tlq_hs", st, [&] {
        return sdp4::launch_fused_tlq(fs, &g, grad_dtype, &o, M, N, S, group, b, cb, kappa, bits_intra, bits_inter,
                                      unit_bytes(S, bits_intra, group), unit_bytes(S, bits_inter, group), sr, &key8,
                                      &key4, c->sm_count, st);
      });
      trace_end("tlq", fs, st);
      return s;
    }
    if (N == 1 && M > 1 && C == 1 && c->local_fusion && bits_intra == 8 && bits_inter == 4) {
      // one GPU per group: the intra all-to-all is the identity, so K3 and K4 are one kernel
      // (k_local34.cu) that pushes each 4-bit unit straight to its node's inter slot; then K5
      const size_t w8 = unit_bytes(S, bits_intra, group), w4 = unit_bytes(S, bits_inter, group);
      const size_t intra_bytes = (size_t)N * M * w8;
      std::vector<Wt> wf, wd;
      std::vector<Sig> gd, gf;
      for (int q : node_ranks) {
        wf.push_back({kFree, 2, q});  // q's K5 of the previous call is done with my push
        gd.push_back({q, kData, 2});
        wd.push_back({kData, 2, q});
        gf.push_back({q, kFree, 2});
      }
      uint8_t* units[sdp4::kMaxDests];
      for (int mp = 0; mp < M; ++mp) units[mp] = sym_region(c->sym_tlq, mp) + intra_bytes + (size_t)m * w4;
      const uint64_t remote = (~0ull >> (64 - M)) & ~(1ull << m);
      if ((s = wait_flags(c, st, c->sym_tlq, wf, "wait_tlq_free")) != SDP4_OK) return s;
      s = launch(c, "K34_tlq_q84", st, [&] {
        return sdp4::launch_tlq_q84(grad, S, grad_dtype, S, M, group, b, cb, units, remote, sr, key8, key4,
                                    c->sm_count, st);
      });
      if (s != SDP4_OK) return s;
      if ((s = raise_flags(c, st, c->sym_tlq, gd)) != SDP4_OK) return s;
      if ((s = wait_flags(c, st, c->sym_tlq, wd, "wait_tlq_inter")) != SDP4_OK) return s;
      uint8_t* my = sym_region(c->sym_tlq, c->rank);
      s = launch(c, "K5_tlq_dq_reduce_had", st, [&] {
        return sdp4::launch_tlq_dq_reduce_had(my + intra_bytes, w4, bits_inter, M, S, group, b, kappa, out_shard,
                                              c->sm_count, st);
      });
      if (s != SDP4_OK) return s;
      return raise_flags(c, st, c->sym_tlq, gf);
    }
    if (C > 1) c->link(st, c->side);
    for (int k = 0; k < C; ++k) {
      const Chunk& ch = chunks[k];
      cudaStream_t sk = (k & 1) ? c->side : st;
      const size_t w8 = unit_bytes(ch.len, bits_intra, group), w4 = unit_bytes(ch.len, bits_inter, group);
      const size_t intra_bytes = (size_t)N * M * w8, outbox_off = intra_bytes + (size_t)M * w4;
      auto region = [&](int rank) { return sym_region(c->sym_tlq, rank) + base[k]; };
      // K3: shard m'N + l' -> unit m' of block l (this rank) in rank (m, l')'s intra receive region
      uint8_t* blocks[sdp4::kMaxN];
      for (int lp = 0; lp < N; ++lp) blocks[lp] = region(m * N + lp) + (size_t)l * M * w8;
      sdp4::IntraPull pull;
      memset(&pull, 0, sizeof(pull));
      pull.mask = pulling ? remote : 0u;
      pull.num = pulling ? pnum : 0;
      pull.den = pden;
      for (int lp = 0; lp < N; ++lp) {
        pull.outbox[lp] = region(c->rank) + outbox_off + (size_t)lp * M * w8;  // mine, for l'
        pull.src[lp] = region(m * N + lp) + outbox_off + (size_t)l * M * w8;   // l''s, for me
      }
      // flag stages of chunk k; sync protocol: K3 writes the group peers' receive blocks and this
      // rank's outbox (read by their K4), K4 the node peers' inter slots (read by their K5)
      const int st_intra = 1 + 2 * k, st_inter = 2 + 2 * k;
      std::vector<Wt> wq3, wq4, wq5;
      std::vector<Sig> g3, g4, g5;
      for (int q : group_ranks) {
        wq3.push_back({kFree, st_intra, q});  // q's K4 of the previous call is done with my pushes / outbox
        g3.push_back({q, kData, st_intra});
        wq4.push_back({kData, st_intra, q});
        g4.push_back({q, kFree, st_intra});
      }
      for (int q : node_ranks) {
        wq4.push_back({kFree, st_inter, q});  // q's K5 of the previous call is done with my pushes
        g4.push_back({q, kData, st_inter});
        wq5.push_back({kData, st_inter, q});
        g5.push_back({q, kFree, st_inter});
      }
      if ((s = wait_flags(c, sk, c->sym_tlq, wq3, "wait_tlq_free")) != SDP4_OK) return s;
      s = launch(c, "K3_tlq_had_quant", sk, [&] {
        return sdp4::launch_tlq_had_quant(static_cast<const uint8_t*>(grad) + ch.off * es, S, grad_dtype, ch.len, M, N,
                                          group, b, cb, bits_intra, blocks, remote, w8, sr, key8, ch.off, c->sm_count,
                                          sk, &pull);
      });
      if (s != SDP4_OK) return s;
      if ((s = raise_flags(c, sk, c->sym_tlq, g3)) != SDP4_OK) return s;
      if ((s = wait_flags(c, sk, c->sym_tlq, wq4, "wait_tlq_intra")) != SDP4_OK) return s;
      // K4: unit m' -> slot m (this node) of rank (m', l)'s inter receive region
      sdp4::Dests d4;
      d4.n = M;
      d4.remote = ~0ull >> (64 - M) & ~(1ull << m);
      for (int mp = 0; mp < M; ++mp) d4.p[mp] = region(mp * N + l) + intra_bytes + (size_t)m * w4;
      uint8_t* my = region(c->rank);
      s = launch(c, "K4_tlq_dq_reduce_q", sk, [&] {
        return sdp4::launch_tlq_dq_reduce_q(my, w8, bits_intra, N, M, ch.len, group, d4, bits_inter, sr, key4, l, S,
                                            ch.off, c->sm_count, sk, &pull);
      });
      if (s != SDP4_OK) return s;
      if ((s = raise_flags(c, sk, c->sym_tlq, g4)) != SDP4_OK) return s;
      if ((s = wait_flags(c, sk, c->sym_tlq, wq5, "wait_tlq_inter")) != SDP4_OK) return s;
      s = launch(c, "K5_tlq_dq_reduce_had", sk, [&] {
        return sdp4::launch_tlq_dq_reduce_had(my + intra_bytes, w4, bits_inter, M, ch.len, group, b, kappa,
                                              out_shard + ch.off, c->sm_count, sk);
      });
      if (s != SDP4_OK) return s;
      if ((s = raise_flags(c, sk, c->sym_tlq, g5)) != SDP4_OK) return s;
    }
    if (C > 1) c->link(c->side, st);
    return SDP4_OK;
  }
  if (local_fused) {
    // one rank: both all-to-alls are the identity -- K3, K4 and K5 as one kernel (k_local.cu)
    return launch(c, "K345_tlq_local", st, [&] {
      return sdp4::launch_tlq_local(grad, grad_dtype, S, group, b, cb, kappa, sr, key8, key4, out_shard, sms, st);
    });
  }
  std::vector<TlqRegions> reg;
  size_t base = 0;
  for (const Chunk& ch : chunks) {
    reg.push_back(tlq_regions(M, N, ch.len, bits_intra, bits_inter, group, base));
    base = reg.back().end;
  }
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  if (P > 1) c->link(st, cs);  // order the side stream after the caller's prior work

  auto stage_k3 = [&](int k) -> sdp4_status {  // Alg. 3 l.2-3 + l.4 IntraAlltoAll
    const Chunk& ch = chunks[k];
    const size_t w8 = unit_bytes(ch.len, bits_intra, group);
    uint8_t* blocks[sdp4::kMaxN];
    for (int lp = 0; lp < N && lp < sdp4::kMaxN; ++lp) blocks[lp] = ws + reg[k].send8 + (size_t)lp * M * w8;
    sdp4_status r = launch(c, "K3_tlq_had_quant", st, [&] {
      return sdp4::launch_tlq_had_quant(static_cast<const uint8_t*>(grad) + ch.off * es, S, grad_dtype, ch.len, M, N,
                                        group, b, cb, bits_intra, blocks, 0u, w8, sr, key8, ch.off, sms, st);
    });
    if (r != SDP4_OK || N == 1) return r;
    c->link(st, cs);
    r = nccl_op(c, "nccl_alltoall_intra", cs, [&] {
      return ncclAlltoAll(ws + reg[k].send8, ws + reg[k].recv8, (size_t)M * w8, ncclUint8, c->intra, cs);
    });
    if (r == SDP4_OK) c->link(cs, st);
    return r;
  };
  auto stage_k4 = [&](int k) -> sdp4_status {  // Alg. 3 l.5, 7, 9 + l.10 InterAlltoAll
    const Chunk& ch = chunks[k];
    const size_t w8 = unit_bytes(ch.len, bits_intra, group), w4 = unit_bytes(ch.len, bits_inter, group);
    sdp4::Dests d4;
    d4.n = M;
    d4.remote = 0;
    for (int mp = 0; mp < M && mp < sdp4::kMaxDests; ++mp) d4.p[mp] = ws + reg[k].send4 + (size_t)mp * w4;
    sdp4_status r = launch(c, "K4_tlq_dq_reduce_q", st, [&] {
      return sdp4::launch_tlq_dq_reduce_q(ws + reg[k].recv8, w8, bits_intra, N, M, ch.len, group, d4, bits_inter, sr,
                                          key4, c->l, S, ch.off, sms, st);
    });
    if (r != SDP4_OK || M == 1) return r;
    c->link(st, cs);
    r = nccl_op(c, "nccl_alltoall_inter", cs, [&] {
      return ncclAlltoAll(ws + reg[k].send4, ws + reg[k].recv4, w4, ncclUint8, c->inter, cs);
    });
    if (r == SDP4_OK) c->link(cs, st);
    return r;
  };
  auto stage_k5 = [&](int k) -> sdp4_status {  // Alg. 3 l.11-13
    const Chunk& ch = chunks[k];
    const size_t w4 = unit_bytes(ch.len, bits_inter, group);
    return launch(c, "K5_tlq_dq_reduce_had", st, [&] {
      return sdp4::launch_tlq_dq_reduce_had(ws + reg[k].recv4, w4, bits_inter, M, ch.len, group, b, kappa,
                                            out_shard + ch.off, sms, st);
    });
  };
  // Software pipeline: at step i issue K3(i), K4(i-1), K5(i-2).  Each stream executes in
  // order; every wait targets an event recorded earlier in issue order (no cycles).
  for (int i = 0; i < C + 2; ++i) {
    if (i < C && (s = stage_k3(i)) != SDP4_OK) return s;
    if (i - 1 >= 0 && i - 1 < C && (s = stage_k4(i - 1)) != SDP4_OK) return s;
    if (i - 2 >= 0 && i - 2 < C && (s = stage_k5(i - 2)) != SDP4_OK) return s;
  }
  return SDP4_OK;
}

size_t sdp4_ring_workspace_bytes(int world, size_t numel, int bits, int group) {
  if (world < 1 || !valid_bits(bits) || !is_pow2(group) || numel % (size_t)world) return 0;
  return 2 * unit_bytes(numel / world, bits, group);
}

// Ring reduce-scatter with per-hop quantization (sec. 2.3) -- the ablation baseline.
// Hop t on rank r: chunk (r - t - 1) mod P; K6 folds the received partial sum into this rank's
// gradient chunk and quantizes it into the next rank's receive slot; the last hop writes the
// fp32 output shard r.  P2P: slot t of hop t in the library's symmetric buffer, one data flag
// per hop (binary flags, sync protocol above).  NCCL: ncclSend/ncclRecv.
sdp4_status sdp4_ring_reduce_scatter(sdp4_comm_t c, const void* grad, sdp4_dtype grad_dtype, size_t numel, int bits,
                                     int group, int average, float* out_shard, void* workspace,
                                     size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_("sdp4_ring_reduce_scatter");
  g_err.clear();
  if (!c) return fail(SDP4_EINVAL, "comm is NULL");
  if (!valid_bits(bits)) return fail(SDP4_EINVAL, "bits %d not in {4, 8, 32}", bits);
  if (grad_dtype != SDP4_F32 && grad_dtype != SDP4_BF16) return fail(SDP4_EINVAL, "bad grad dtype");
  sdp4_status s = check_sizes(c->world, numel, group);
  if (s != SDP4_OK) return s;
  if ((s = check_ptr(grad, "grad")) != SDP4_OK) return s;
  if ((s = check_ptr(out_shard, "out_shard")) != SDP4_OK) return s;
  const size_t need = sdp4_ring_workspace_bytes(c->world, numel, bits, group);
  if ((s = check_workspace(c, workspace, workspace_bytes, need)) != SDP4_OK) return s;
  if ((s = async_check(c)) != SDP4_OK) return s;
  const int P = c->world, r = c->rank;
  if (P > sdp4::kMaxDests) return fail(SDP4_EINVAL, "world %d > %d", P, sdp4::kMaxDests);
  const size_t S = numel / P, es = esize(grad_dtype), W = unit_bytes(S, bits, group);
  const float kappa = average ? 1.0f / (float)P : 1.0f;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int sms = c->sm_count;
  auto chunk = [&](int j) { return static_cast<const uint8_t*>(grad) + (size_t)j * S * es; };
  auto hop = [&](int j, const uint8_t* recv, uint8_t* dst, float* out) {
    return launch(c, "K6_ring_hop", st, [&] {
      return sdp4::launch_ring_hop(chunk(j), grad_dtype, recv, dst, out, kappa, S, bits, group, sms, st);
    });
  };
  if (P == 1) return hop(0, nullptr, nullptr, out_shard);
  const int next = (r + 1) % P, prev = (r + P - 1) % P;
  if (c->transport == kTransportP2P) {
    // region: P-1 receive slots + one local send slot; K6 writes the hop's unit locally and
    // the copy engine moves it into the next rank's slot (large NVLink writes).  Sync: hop t
    // raises data[t] on next; the final hop consumed every slot, so it raises free[0] on prev,
    // which prev waits for before its first push of the following call.
    if ((s = sym_ensure(c, c->sym_ring, (size_t)P * W, st)) != SDP4_OK) return s;
    auto slot = [&](int owner, int t) { return sym_region(c->sym_ring, owner) + (size_t)t * W; };
    uint8_t* send_local = slot(r, P - 1);
    if ((s = wait_flags(c, st, c->sym_ring, {{kFree, 0, next}}, "wait_ring_free")) != SDP4_OK) return s;
    for (int t = 0; t < P - 1; ++t) {
      if (t > 0 && (s = wait_flags(c, st, c->sym_ring, {{kData, t - 1, prev}}, "wait_ring")) != SDP4_OK) return s;
      if ((s = hop((r - t - 1 + 2 * P) % P, t ? slot(r, t - 1) : nullptr, send_local, nullptr)) != SDP4_OK)
        return s;
      cudaError_t e = cudaMemcpyAsync(slot(next, t), send_local, W, cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) return fail(SDP4_ECUDA, "ring hop copy: %s", cudaGetErrorString(e));
      if ((s = raise_flags(c, st, c->sym_ring, {{next, kData, t}})) != SDP4_OK) return s;
    }
    if ((s = wait_flags(c, st, c->sym_ring, {{kData, P - 2, prev}}, "wait_ring")) != SDP4_OK) return s;
    if ((s = hop(r, slot(r, P - 2), nullptr, out_shard)) != SDP4_OK) return s;
    return raise_flags(c, st, c->sym_ring, {{prev, kFree, 0}});
  }
  uint8_t* send = static_cast<uint8_t*>(workspace);
  uint8_t* recv = send + W;
  for (int t = 0; t < P - 1; ++t) {
    if ((s = hop((r - t - 1 + 2 * P) % P, t ? recv : nullptr, send, nullptr)) != SDP4_OK) return s;
    s = nccl_op(c, "nccl_ring_sendrecv", st, [&] {
      ncclGroupStart();
      ncclSend(send, W, ncclUint8, next, c->world_c, st);
      ncclRecv(recv, W, ncclUint8, prev, c->world_c, st);
      return ncclGroupEnd();
    });
    if (s != SDP4_OK) return s;
  }
  return hop(r, recv, nullptr, out_shard);
}

sdp4_status sdp4_tlq_stage_quantize(const void* grad, sdp4_dtype grad_dtype, size_t numel, int M, int N,
                                    int bits_intra, int group, int hadamard_block, sdp4_round rnd, uint64_t seed,
                                    int rank, void* intra_send, void* stream) {
  NvtxRange nvtx_("sdp4_tlq_stage_quantize");
  g_err.clear();
  if (M < 1 || N < 1) return fail(SDP4_EINVAL, "bad topology %d x %d", M, N);
  if (!valid_round(rnd) || rank < 0 || rank >= M * N) return fail(SDP4_EINVAL, "bad rounding mode or rank");
  if (grad_dtype != SDP4_F32 && grad_dtype != SDP4_BF16) return fail(SDP4_EINVAL, "bad grad dtype");
  sdp4_status s = check_tlq_args(M * N, numel, bits_intra, 4, group, hadamard_block);
  if (s != SDP4_OK) return s;
  if ((s = check_ptr(grad, "grad")) != SDP4_OK) return s;
  if ((s = check_ptr(intra_send, "intra_send")) != SDP4_OK) return s;
  const size_t S = numel / ((size_t)M * N);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (N > sdp4::kMaxN) return fail(SDP4_EINVAL, "group_size_N %d > %d", N, sdp4::kMaxN);
  const size_t w8 = unit_bytes(S, bits_intra, group);
  uint8_t* blocks[sdp4::kMaxN];
  for (int lp = 0; lp < N; ++lp) blocks[lp] = static_cast<uint8_t*>(intra_send) + (size_t)lp * M * w8;
  cudaError_t e = sdp4::launch_tlq_had_quant(grad, S, grad_dtype, S, M, N, group, hadamard_block,
                                             hadamard_cb(hadamard_block), bits_intra, blocks, 0u, w8,
                                             rnd == SDP4_STOCHASTIC, sr_key(seed, kStageIntra, rank), 0,
                                             sm_count_current(), st);
  return e == cudaSuccess ? SDP4_OK : fail(SDP4_ECUDA, "K3 launch failed: %s", cudaGetErrorString(e));
}

sdp4_status sdp4_tlq_stage_quantize_reduce(const void* grad, sdp4_dtype grad_dtype, size_t numel, int M, int group,
                                           int hadamard_block, sdp4_round rnd, uint64_t seed, int rank,
                                           void* inter_send, void* stream) {
  NvtxRange nvtx_("sdp4_tlq_stage_quantize_reduce");
  g_err.clear();
  if (M < 1 || M > sdp4::kMaxDests) return fail(SDP4_EINVAL, "bad groups_M %d", M);
  if (!valid_round(rnd) || rank < 0 || rank >= M) return fail(SDP4_EINVAL, "bad rounding mode or rank");
  if (grad_dtype != SDP4_F32 && grad_dtype != SDP4_BF16) return fail(SDP4_EINVAL, "bad grad dtype");
  sdp4_status s = check_tlq_args(M, numel, 8, 4, group, hadamard_block);
  if (s != SDP4_OK) return s;
  if ((s = check_ptr(grad, "grad")) != SDP4_OK) return s;
  if ((s = check_ptr(inter_send, "inter_send")) != SDP4_OK) return s;
  const size_t S = numel / M;
  const size_t w4 = unit_bytes(S, 4, group);
  uint8_t* units[sdp4::kMaxDests];
  for (int mp = 0; mp < M; ++mp) units[mp] = static_cast<uint8_t*>(inter_send) + (size_t)mp * w4;
  cudaError_t e = sdp4::launch_tlq_q84(grad, S, grad_dtype, S, M, group, hadamard_block, hadamard_cb(hadamard_block),
                                       units, 0ull, rnd == SDP4_STOCHASTIC, sr_key(seed, kStageIntra, rank),
                                       sr_key(seed, kStageInter, rank), sm_count_current(), static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SDP4_OK : fail(SDP4_ECUDA, "K34 launch failed: %s", cudaGetErrorString(e));
}

sdp4_status sdp4_tlq_stage_reduce(const void* intra_recv, size_t numel, int M, int N, int bits_intra,
                                  int bits_inter, int group, sdp4_round rnd, uint64_t seed, int rank,
                                  void* inter_send, void* stream) {
  NvtxRange nvtx_("sdp4_tlq_stage_reduce");
  g_err.clear();
  if (M < 1 || N < 1) return fail(SDP4_EINVAL, "bad topology %d x %d", M, N);
  if (!valid_round(rnd) || rank < 0 || rank >= M * N) return fail(SDP4_EINVAL, "bad rounding mode or rank");
  sdp4_status s = check_tlq_args(M * N, numel, bits_intra, bits_inter, group, 0);
  if (s != SDP4_OK) return s;
  if ((s = check_ptr(intra_recv, "intra_recv")) != SDP4_OK) return s;
  if ((s = check_ptr(inter_send, "inter_send")) != SDP4_OK) return s;
  const size_t S = numel / ((size_t)M * N);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (M > sdp4::kMaxDests) return fail(SDP4_EINVAL, "groups_M %d > %d", M, sdp4::kMaxDests);
  sdp4::Dests d4;
  d4.n = M;
  d4.remote = 0;
  for (int mp = 0; mp < M; ++mp) d4.p[mp] = static_cast<uint8_t*>(inter_send) + (size_t)mp * unit_bytes(S, bits_inter, group);
  cudaError_t e = sdp4::launch_tlq_dq_reduce_q(static_cast<const uint8_t*>(intra_recv),
                                               unit_bytes(S, bits_intra, group), bits_intra, N, M, S, group, d4,
                                               bits_inter, rnd == SDP4_STOCHASTIC, sr_key(seed, kStageInter, rank),
                                               rank % N, S, 0, sm_count_current(), st);
  return e == cudaSuccess ? SDP4_OK : fail(SDP4_ECUDA, "K4 launch failed: %s", cudaGetErrorString(e));
}

sdp4_status sdp4_tlq_stage_final(const void* inter_recv, size_t numel, int M, int N, int bits_inter, int group,
                                 int hadamard_block, int average, float* out_shard, void* stream) {
  NvtxRange nvtx_("sdp4_tlq_stage_final");
  g_err.clear();
  if (M < 1 || N < 1) return fail(SDP4_EINVAL, "bad topology %d x %d", M, N);
  sdp4_status s = check_tlq_args(M * N, numel, 8, bits_inter, group, hadamard_block);
  if (s != SDP4_OK) return s;
  if ((s = check_ptr(inter_recv, "inter_recv")) != SDP4_OK) return s;
  if ((s = check_ptr(out_shard, "out_shard")) != SDP4_OK) return s;
  const size_t S = numel / ((size_t)M * N);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = sdp4::launch_tlq_dq_reduce_had(static_cast<const uint8_t*>(inter_recv),
                                                 unit_bytes(S, bits_inter, group), bits_inter, M, S, group,
                                                 hadamard_block, final_kappa(hadamard_block, M * N, average),
                                                 out_shard, sm_count_current(), st);
  return e == cudaSuccess ? SDP4_OK : fail(SDP4_ECUDA, "K5 launch failed: %s", cudaGetErrorString(e));
}

// ---- One-launch kernels on an emulated P-rank job (every rank's symmetric buffer a slice of
// one device workspace, all ranks in ONE launch): the parity tests' route to the kernels of
// the small-message path on a single GPU.  Workspace: [counters: 256 B][rank 0: flags, region]...
namespace {
constexpr size_t kEmuHead = 256;
size_t emu_rank_bytes(size_t region) { return kFlagBytes + round_up(region, 256); }

sdp4_status emu_prepare(uint8_t* ws, int P, size_t region, int fresh, cudaStream_t st, sdp4::FusedSync* fs) {
  memset(fs, 0, sizeof(*fs));
  const size_t rb = emu_rank_bytes(region);
  for (int q = 0; q < P; ++q) {
    uint8_t* base = ws + kEmuHead + (size_t)q * rb;
    fs->flags[q] = reinterpret_cast<uint32_t*>(base);
    fs->region[q] = base + kFlagBytes;
    fs->rank[q] = q;
    if (fresh) {  // a first call: data flags 0, free flags 1 (sym_ensure's initial state)
      const size_t half = flag_off(kFree, 0, 0) / 4;
      cudaError_t e = sdp4::launch_fill32(fs->flags[q], half, 0u, st);
      if (e == cudaSuccess) e = sdp4::launch_fill32(fs->flags[q] + half, kFlagBytes / 4 - half, 1u, st);
      if (e != cudaSuccess) return fail(SDP4_ECUDA, "flag init: %s", cudaGetErrorString(e));
    }
  }
  fs->nv = P;
  fs->P = P;
  fs->ctr = reinterpret_cast<uint32_t*>(ws);
  fs->err = nullptr;
  fs->timeout_ns = 20ull * 1000000000ull;  // a broken kernel gives up (wrong results, no hang)
  if (fresh && cudaMemsetAsync(ws, 0, kEmuHead, st) != cudaSuccess) return fail(SDP4_ECUDA, "counter init failed");
  return SDP4_OK;
}
}  // namespace

size_t sdp4_emu_qwd_workspace_bytes(int world, size_t numel, int bits, int group) {
  if (world < 2 || world > sdp4::kMaxVr || !valid_wbits(bits) || !is_pow2(group) || numel % (size_t)world) return 0;
  return kEmuHead + (size_t)world * emu_rank_bytes(unit_bytes(numel / world, bits, group));
}

sdp4_status sdp4_emu_qwd_step(int world, const float* const* w_main_shards, void* const* w_model_full,
                              sdp4_dtype model_dtype, size_t numel, int bits, int group, sdp4_round rnd,
                              uint64_t seed, int fresh, void* workspace, size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_("sdp4_emu_qwd_step");
  g_err.clear();
  if (world < 2 || world > sdp4::kMaxVr) return fail(SDP4_EINVAL, "world %d not in [2, %d]", world, sdp4::kMaxVr);
  if (!w_main_shards || !w_model_full) return fail(SDP4_EINVAL, "pointer arrays are NULL");
  if (!valid_round(rnd)) return fail(SDP4_EINVAL, "bad rounding mode %d", (int)rnd);
  if (!valid_wbits(bits)) return fail(SDP4_EINVAL, "bits %d not in {2, 4, 8, 32}", bits);
  if (model_dtype != SDP4_F32 && model_dtype != SDP4_BF16) return fail(SDP4_EINVAL, "bad model dtype");
  sdp4_status s = check_sizes(world, numel, group);
  if (s != SDP4_OK) return s;
  for (int q = 0; q < world; ++q) {
    if ((s = check_ptr(w_main_shards[q], "w_main_shards[q]")) != SDP4_OK) return s;
    if ((s = check_ptr(w_model_full[q], "w_model_full[q]")) != SDP4_OK) return s;
  }
  if ((s = check_ptr(workspace, "workspace")) != SDP4_OK) return s;
  const size_t need = sdp4_emu_qwd_workspace_bytes(world, numel, bits, group);
  if (workspace_bytes < need) return fail(SDP4_ESTATE, "workspace %zu < %zu bytes", workspace_bytes, need);
  const size_t S = numel / world;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  sdp4::FusedSync fs;
  if ((s = emu_prepare(static_cast<uint8_t*>(workspace), world, unit_bytes(S, bits, group), fresh, st, &fs)) != SDP4_OK)
    return s;
  uint32_t keys[sdp4::kMaxVr];
  for (int q = 0; q < world; ++q) keys[q] = sr_key(seed, kStageQwd, q);
  trace_begin(fs);
  cudaError_t e = sdp4::launch_fused_qwd(fs, w_main_shards, w_model_full, model_dtype, S, bits, group,
                                         rnd == SDP4_STOCHASTIC, keys, sm_count_current(), st);
  trace_end("emu_qwd", fs, st);
  return e == cudaSuccess ? SDP4_OK : fail(SDP4_ECUDA, "one-launch qWD failed: %s", cudaGetErrorString(e));
}

size_t sdp4_emu_tlq_workspace_bytes(int M, int N, size_t numel, int bits_intra, int bits_inter, int group) {
  const int P = M * N;
  if (M < 1 || N < 1 || P < 2 || P > sdp4::kMaxVr || !valid_bits(bits_intra) || !valid_bits(bits_inter) ||
      !is_pow2(group) || numel % (size_t)P)
    return 0;
  const size_t S = numel / P;
  return kEmuHead + (size_t)P * emu_rank_bytes((size_t)N * M * unit_bytes(S, bits_intra, group) +
                                               (size_t)M * unit_bytes(S, bits_inter, group));
}

sdp4_status sdp4_emu_tlq_hs_reduce_scatter(int M, int N, const void* const* grads, sdp4_dtype grad_dtype,
                                           size_t numel, int bits_intra, int bits_inter, int group,
                                           int hadamard_block, int average, sdp4_round rnd, uint64_t seed,
                                           float* const* out_shards, int fresh, void* workspace,
                                           size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_("sdp4_emu_tlq_hs_reduce_scatter");
  g_err.clear();
  const int P = M * N, b = hadamard_block;
  if (M < 1 || N < 1 || P < 2 || P > sdp4::kMaxVr) return fail(SDP4_EINVAL, "bad topology %d x %d", M, N);
  if (!grads || !out_shards) return fail(SDP4_EINVAL, "pointer arrays are NULL");
  if (!valid_round(rnd)) return fail(SDP4_EINVAL, "bad rounding mode %d", (int)rnd);
  if (grad_dtype != SDP4_F32 && grad_dtype != SDP4_BF16) return fail(SDP4_EINVAL, "bad grad dtype");
  sdp4_status s = check_tlq_args(P, numel, bits_intra, bits_inter, group, b);
  if (s != SDP4_OK) return s;
  if (!sdp4::fused_tlq_supported(bits_intra, bits_inter, b))
    return fail(SDP4_EINVAL, "the one-launch path takes bits_intra, bits_inter in {4, 8}");
  for (int q = 0; q < P; ++q) {
    if ((s = check_ptr(grads[q], "grads[q]")) != SDP4_OK) return s;
    if ((s = check_ptr(out_shards[q], "out_shards[q]")) != SDP4_OK) return s;
  }
  if ((s = check_ptr(workspace, "workspace")) != SDP4_OK) return s;
  const size_t need = sdp4_emu_tlq_workspace_bytes(M, N, numel, bits_intra, bits_inter, group);
  if (workspace_bytes < need) return fail(SDP4_ESTATE, "workspace %zu < %zu bytes", workspace_bytes, need);
  const size_t S = numel / P;
  const size_t w8 = unit_bytes(S, bits_intra, group), w4 = unit_bytes(S, bits_inter, group);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  sdp4::FusedSync fs;
  if ((s = emu_prepare(static_cast<uint8_t*>(workspace), P, (size_t)N * M * w8 + (size_t)M * w4, fresh, st, &fs)) !=
      SDP4_OK)
    return s;
  uint32_t k8[sdp4::kMaxVr], k4[sdp4::kMaxVr];
  for (int q = 0; q < P; ++q) {
    k8[q] = sr_key(seed, kStageIntra, q);
    k4[q] = sr_key(seed, kStageInter, q);
  }
  trace_begin(fs);
  cudaError_t e = sdp4::launch_fused_tlq(fs, grads, grad_dtype, out_shards, M, N, S, group, b, hadamard_cb(b),
                                         final_kappa(b, P, average), bits_intra, bits_inter, w8, w4,
                                         rnd == SDP4_STOCHASTIC, k8, k4, sm_count_current(), st);
  trace_end("emu_tlq", fs, st);
  return e == cudaSuccess ? SDP4_OK : fail(SDP4_ECUDA, "one-launch TLq-HS failed: %s", cudaGetErrorString(e));
}

uint64_t sdp4_launch_count(sdp4_comm_t c, int reset) {
  if (!c) return 0;
  const uint64_t n = c->launches;
  if (reset) c->launches = 0;
  return n;
}

sdp4_status sdp4_profile_enable(sdp4_comm_t c, int enable) {
  if (!c) return fail(SDP4_EINVAL, "comm is NULL");
  c->profiling = enable != 0;
  return SDP4_OK;
}

sdp4_status sdp4_profile_read(sdp4_comm_t c, const char** names, double* ms, uint64_t* launches, int max_entries,
                              int* count) {
  if (!c || !count) return fail(SDP4_EINVAL, "comm/count is NULL");
  for (auto& p : c->pending) {
    cudaError_t e = cudaEventSynchronize(p.b);
    if (e != cudaSuccess) return fail(SDP4_ECUDA, "event sync: %s", cudaGetErrorString(e));
    float t = 0.f;
    cudaEventElapsedTime(&t, p.a, p.b);
    auto& slot = c->acc[p.name];
    slot.first += t;
    slot.second += 1;
    c->pool.push_back(p.a);
    c->pool.push_back(p.b);
  }
  c->pending.clear();
  int i = 0;
  c->names_keep.clear();
  for (auto& kv : c->acc) c->names_keep.push_back(kv.first);
  for (auto& kv : c->acc) {
    if (i >= max_entries) break;
    if (names) names[i] = c->names_keep[i].c_str();
    if (ms) ms[i] = kv.second.first;
    if (launches) launches[i] = kv.second.second;
    ++i;
  }
  *count = i;
  c->acc.clear();
  return SDP4_OK;
}

sdp4_status sdp4_nccl_reduce_scatter(sdp4_comm_t c, const void* send, void* recv, size_t numel, sdp4_dtype dtype,
                                     int average, void* stream) {
  NvtxRange nvtx_("sdp4_nccl_reduce_scatter");
  if (!c) return fail(SDP4_EINVAL, "comm is NULL");
  if (c->world > 1 && !c->world_c) return fail(SDP4_ESTATE, "this comm has no NCCL communicators");
  if (numel % (size_t)c->world) return fail(SDP4_EALIGN, "numel not divisible by world");
  const ncclDataType_t dt = dtype == SDP4_BF16 ? ncclBfloat16 : ncclFloat32;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (c->world == 1) {
    cudaError_t e = cudaMemcpyAsync(recv, send, numel * esize(dtype), cudaMemcpyDeviceToDevice, st);
    return e == cudaSuccess ? SDP4_OK : fail(SDP4_ECUDA, "%s", cudaGetErrorString(e));
  }
  return nccl_check(ncclReduceScatter(send, recv, numel / c->world, dt, average ? ncclAvg : ncclSum, c->world_c, st),
                    "ncclReduceScatter");
}

sdp4_status sdp4_nccl_all_gather(sdp4_comm_t c, const void* send, void* recv, size_t numel, sdp4_dtype dtype,
                                 void* stream) {
  NvtxRange nvtx_("sdp4_nccl_all_gather");
  if (!c) return fail(SDP4_EINVAL, "comm is NULL");
  if (c->world > 1 && !c->world_c) return fail(SDP4_ESTATE, "this comm has no NCCL communicators");
  if (numel % (size_t)c->world) return fail(SDP4_EALIGN, "numel not divisible by world");
  const ncclDataType_t dt = dtype == SDP4_BF16 ? ncclBfloat16 : ncclFloat32;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (c->world == 1) {
    cudaError_t e = cudaMemcpyAsync(recv, send, numel * esize(dtype), cudaMemcpyDeviceToDevice, st);
    return e == cudaSuccess ? SDP4_OK : fail(SDP4_ECUDA, "%s", cudaGetErrorString(e));
  }
  return nccl_check(ncclAllGather(send, recv, numel / c->world, dt, c->world_c, st), "ncclAllGather");
}

}  // extern "C"
