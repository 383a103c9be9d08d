// sdp4_api.cu -- the C ABI of include/sdp4.h: argument validation, workspace layout,
// NCCL communicators (world + intra + inter via ncclCommSplit, sec. 2.3) and the
// stream-ordered orchestration of Alg. 2 l.2-5 (qWD) and Alg. 3 (TLq-HS).
#include "sdp4.h"

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>

#include "sdp4_kernels.cuh"

namespace {

thread_local std::string g_err;

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

// Wire unit (R15): [codes n*k/8][fp32 scales n/G] padded to 256 bytes; k = 32: n fp32.
size_t unit_bytes(size_t n, int bits, int group) {
  if (bits == 32) return round_up(4 * n, 256);
  return round_up(n * (size_t)bits / 8 + 4 * (n / (size_t)group), 256);
}

}  // namespace

struct sdp4_comm {
  int rank = 0, world = 1, M = 1, N = 1, m = 0, l = 0;
  int device = 0;
  int sm_count = 148;
  ncclComm_t world_c = nullptr, intra = nullptr, inter = nullptr;
  uint64_t launches = 0;
  bool profiling = false;
  struct Pending {
    const char* name;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> pool;
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
  int grid_cap() const { return sm_count * 8; }
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

sdp4_status async_check(sdp4_comm* c) {
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

size_t tlq_region(int M, int N, size_t numel, int bi, int be, int group, int region, size_t* total) {
  const size_t P = (size_t)M * N, S = numel / P;
  const size_t w8 = unit_bytes(S, bi, group), w4 = unit_bytes(S, be, group);
  const size_t intra = (size_t)N * M * w8, inter = (size_t)M * w4;
  size_t off[5];
  off[0] = 0;
  off[1] = off[0] + intra;
  off[2] = off[1] + (N > 1 ? intra : 0);
  off[3] = off[2] + inter;
  off[4] = off[3] + (M > 1 ? inter : 0);
  if (N == 1) off[1] = off[0];
  if (M == 1) off[3] = off[2];
  if (total) *total = off[4];
  return off[region];
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

}  // namespace

extern "C" {

int sdp4_version(void) { return 100; }

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

sdp4_status sdp4_comm_init(sdp4_comm_t* out, const unsigned char* id, int rank, int world,
                           int groups_M, int group_size_N) {
  if (!out) return fail(SDP4_EINVAL, "out is NULL");
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world) return fail(SDP4_EINVAL, "bad rank %d / world %d", rank, world);
  if (groups_M < 1 || group_size_N < 1 || groups_M * group_size_N != world)
    return fail(SDP4_EINVAL, "groups_M (%d) * group_size_N (%d) != world (%d)", groups_M, group_size_N, world);
  if (world > 1 && !id) return fail(SDP4_EINVAL, "id is NULL with world > 1");
  sdp4_comm* c = new sdp4_comm();
  c->rank = rank;
  c->world = world;
  c->M = groups_M;
  c->N = group_size_N;
  c->m = rank / group_size_N;
  c->l = rank % group_size_N;
  cudaGetDevice(&c->device);
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, c->device);
  if (world > 1) {
    ncclUniqueId u;
    memcpy(&u, id, sizeof(u));
    sdp4_status s = nccl_check(ncclCommInitRank(&c->world_c, world, u, rank), "ncclCommInitRank");
    if (s == SDP4_OK && group_size_N > 1)
      s = nccl_check(ncclCommSplit(c->world_c, c->m, c->l, &c->intra, nullptr), "ncclCommSplit(intra)");
    if (s == SDP4_OK && groups_M > 1)
      s = nccl_check(ncclCommSplit(c->world_c, c->l, c->m, &c->inter, nullptr), "ncclCommSplit(inter)");
    if (s != SDP4_OK) {
      if (c->inter) ncclCommDestroy(c->inter);
      if (c->intra) ncclCommDestroy(c->intra);
      if (c->world_c) ncclCommDestroy(c->world_c);
      delete c;
      return s;
    }
  }
  *out = c;
  return SDP4_OK;
}

sdp4_status sdp4_comm_destroy(sdp4_comm_t c) {
  if (!c) return fail(SDP4_EINVAL, "comm is NULL");
  for (auto& p : c->pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : c->pool) cudaEventDestroy(e);
  if (c->inter) ncclCommDestroy(c->inter);
  if (c->intra) ncclCommDestroy(c->intra);
  if (c->world_c) ncclCommDestroy(c->world_c);
  delete c;
  return SDP4_OK;
}

size_t sdp4_wire_unit_bytes(size_t n, int bits, int group) {
  if (!valid_bits(bits) || !is_pow2(group)) return 0;
  return unit_bytes(n, bits, group);
}

size_t sdp4_qwd_workspace_bytes(int world, size_t numel, int bits, int group) {
  if (world < 1 || !valid_bits(bits) || !is_pow2(group) || numel % (size_t)world) return 0;
  return (size_t)world * unit_bytes(numel / world, bits, group);
}

size_t sdp4_tlq_workspace_bytes(int M, int N, size_t numel, int bi, int be, int group) {
  if (M < 1 || N < 1 || !valid_bits(bi) || !valid_bits(be) || !is_pow2(group) || numel % ((size_t)M * N))
    return 0;
  size_t total = 0;
  tlq_region(M, N, numel, bi, be, group, 0, &total);
  return total;
}

size_t sdp4_tlq_workspace_offset(int M, int N, size_t numel, int bi, int be, int group, int region) {
  if (region < 0 || region > 3 || sdp4_tlq_workspace_bytes(M, N, numel, bi, be, group) == 0) return 0;
  return tlq_region(M, N, numel, bi, be, group, region, nullptr);
}

sdp4_status sdp4_qwd_quantize(sdp4_comm_t c, const float* w_main_shard, const void* w_model_full,
                              sdp4_dtype model_dtype, size_t numel, int bits, int group,
                              sdp4_round rnd, uint64_t seed, void* workspace, size_t workspace_bytes,
                              void* stream) {
  (void)seed;
  g_err.clear();
  if (!c) return fail(SDP4_EINVAL, "comm is NULL");
  if (rnd != SDP4_RNE) return fail(SDP4_EINVAL, "only SDP4_RNE rounding is implemented");
  if (!valid_bits(bits)) return fail(SDP4_EINVAL, "bits %d not in {4, 8, 32}", bits);
  if (model_dtype != SDP4_F32 && model_dtype != SDP4_BF16) return fail(SDP4_EINVAL, "bad model dtype");
  sdp4_status s = check_sizes(c->world, numel, group);
  if (s != SDP4_OK) return s;
  if ((s = check_ptr(w_main_shard, "w_main_shard")) != SDP4_OK) return s;
  if ((s = check_ptr(w_model_full, "w_model_full")) != SDP4_OK) return s;
  if ((s = check_ptr(workspace, "workspace")) != SDP4_OK) return s;
  const size_t need = sdp4_qwd_workspace_bytes(c->world, numel, bits, group);
  if (workspace_bytes < need) return fail(SDP4_ESTATE, "workspace %zu < %zu bytes", workspace_bytes, need);
  if ((s = async_check(c)) != SDP4_OK) return s;
  const size_t S = numel / c->world;
  const size_t W = unit_bytes(S, bits, group);
  const size_t esz = model_dtype == SDP4_BF16 ? 2 : 4;
  const void* shard = static_cast<const uint8_t*>(w_model_full) + (size_t)c->rank * S * esz;
  uint8_t* unit = static_cast<uint8_t*>(workspace) + (size_t)c->rank * W;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return launch(c, "K1_qwd_quantize", st, [&] {
    return sdp4::launch_qwd_quantize(w_main_shard, shard, model_dtype, S, bits, group, unit, c->grid_cap(), st);
  });
}

sdp4_status sdp4_qwd_allgather_apply(sdp4_comm_t c, void* workspace, size_t workspace_bytes, size_t numel,
                                     int bits, int group, void* w_model_full, sdp4_dtype model_dtype,
                                     void* stream) {
  g_err.clear();
  if (!c) return fail(SDP4_EINVAL, "comm is NULL");
  if (!valid_bits(bits)) return fail(SDP4_EINVAL, "bits %d not in {4, 8, 32}", bits);
  if (model_dtype != SDP4_F32 && model_dtype != SDP4_BF16) return fail(SDP4_EINVAL, "bad model dtype");
  sdp4_status s = check_sizes(c->world, numel, group);
  if (s != SDP4_OK) return s;
  if ((s = check_ptr(workspace, "workspace")) != SDP4_OK) return s;
  if ((s = check_ptr(w_model_full, "w_model_full")) != SDP4_OK) return s;
  const size_t need = sdp4_qwd_workspace_bytes(c->world, numel, bits, group);
  if (workspace_bytes < need) return fail(SDP4_ESTATE, "workspace %zu < %zu bytes", workspace_bytes, need);
  if ((s = async_check(c)) != SDP4_OK) return s;
  const size_t S = numel / c->world;
  const size_t W = unit_bytes(S, bits, group);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (c->world > 1) {  // Alg. 2 l.4 AllGather, in place
    s = nccl_check(ncclAllGather(ws + (size_t)c->rank * W, ws, W, ncclUint8, c->world_c, st), "ncclAllGather");
    if (s != SDP4_OK) return s;
  }
  return launch(c, "K2_qwd_apply", st, [&] {
    return sdp4::launch_qwd_apply(ws, W, c->world, S, bits, group, w_model_full, model_dtype, c->grid_cap(), st);
  });
}

sdp4_status sdp4_tlq_hs_reduce_scatter(sdp4_comm_t c, const void* grad, sdp4_dtype grad_dtype, size_t numel,
                                       int bits_intra, int bits_inter, int group, int hadamard_block,
                                       int average, sdp4_round rnd, uint64_t seed, float* out_shard,
                                       void* workspace, size_t workspace_bytes, void* stream) {
  (void)seed;
  g_err.clear();
  if (!c) return fail(SDP4_EINVAL, "comm is NULL");
  if (rnd != SDP4_RNE) return fail(SDP4_EINVAL, "only SDP4_RNE rounding is implemented");
  if (grad_dtype != SDP4_F32 && grad_dtype != SDP4_BF16) return fail(SDP4_EINVAL, "bad grad dtype");
  const int b = hadamard_block;
  sdp4_status s = check_tlq_args(c->world, numel, bits_intra, bits_inter, group, b);
  if (s != SDP4_OK) return s;
  if ((s = check_ptr(grad, "grad")) != SDP4_OK) return s;
  if ((s = check_ptr(out_shard, "out_shard")) != SDP4_OK) return s;
  if ((s = check_ptr(workspace, "workspace")) != SDP4_OK) return s;
  const int M = c->M, N = c->N, P = c->world;
  size_t need = 0;
  tlq_region(M, N, numel, bits_intra, bits_inter, group, 0, &need);
  if (workspace_bytes < need) return fail(SDP4_ESTATE, "workspace %zu < %zu bytes", workspace_bytes, need);
  if ((s = async_check(c)) != SDP4_OK) return s;

  const size_t S = numel / P;
  const size_t w8 = unit_bytes(S, bits_intra, group), w4 = unit_bytes(S, bits_inter, group);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  uint8_t* intra_send = ws + tlq_region(M, N, numel, bits_intra, bits_inter, group, 0, nullptr);
  uint8_t* intra_recv = ws + tlq_region(M, N, numel, bits_intra, bits_inter, group, 1, nullptr);
  uint8_t* inter_send = ws + tlq_region(M, N, numel, bits_intra, bits_inter, group, 2, nullptr);
  uint8_t* inter_recv = ws + tlq_region(M, N, numel, bits_intra, bits_inter, group, 3, nullptr);
  cudaStream_t st = static_cast<cudaStream_t>(stream);

  const float cb = hadamard_cb(b), kappa = final_kappa(b, P, average);

  // Alg. 3 l.2-3: Hadamard + Quantize8Bit into the intra send layout (K3)
  s = launch(c, "K3_tlq_had_quant", st, [&] {
    return sdp4::launch_tlq_had_quant(grad, grad_dtype, S, M, N, group, b, cb, bits_intra, intra_send, w8,
                                      c->grid_cap(), st);
  });
  if (s != SDP4_OK) return s;
  // Alg. 3 l.4 IntraAlltoAll
  if (N > 1) {
    s = nccl_check(ncclAlltoAll(intra_send, intra_recv, (size_t)M * w8, ncclUint8, c->intra, st), "ncclAlltoAll(intra)");
    if (s != SDP4_OK) return s;
  }
  // Alg. 3 l.5, 7, 9: Dequantize + Reduction + Quantize4Bit (K4)
  s = launch(c, "K4_tlq_dq_reduce_q", st, [&] {
    return sdp4::launch_tlq_dq_reduce_q(intra_recv, w8, bits_intra, N, M, S, group, inter_send, w4, bits_inter,
                                        c->grid_cap(), st);
  });
  if (s != SDP4_OK) return s;
  // Alg. 3 l.10 InterAlltoAll
  if (M > 1) {
    s = nccl_check(ncclAlltoAll(inter_send, inter_recv, w4, ncclUint8, c->inter, st), "ncclAlltoAll(inter)");
    if (s != SDP4_OK) return s;
  }
  // Alg. 3 l.11-13: Dequantize + Reduction + Hadamard (K5)
  return launch(c, "K5_tlq_dq_reduce_had", st, [&] {
    return sdp4::launch_tlq_dq_reduce_had(inter_recv, w4, bits_inter, M, S, group, b, kappa, out_shard,
                                          c->grid_cap(), st);
  });
}

sdp4_status sdp4_tlq_stage_quantize(const void* grad, sdp4_dtype grad_dtype, size_t numel, int M, int N,
                                    int bits_intra, int group, int hadamard_block, void* intra_send, void* stream) {
  g_err.clear();
  if (M < 1 || N < 1) return fail(SDP4_EINVAL, "bad topology %d x %d", M, N);
  if (grad_dtype != SDP4_F32 && grad_dtype != SDP4_BF16) return fail(SDP4_EINVAL, "bad grad dtype");
  sdp4_status s = check_tlq_args(M * N, numel, bits_intra, 4, group, hadamard_block);
  if (s != SDP4_OK) return s;
  if ((s = check_ptr(grad, "grad")) != SDP4_OK) return s;
  if ((s = check_ptr(intra_send, "intra_send")) != SDP4_OK) return s;
  const size_t S = numel / ((size_t)M * N);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = sdp4::launch_tlq_had_quant(grad, grad_dtype, S, M, N, group, hadamard_block,
                                             hadamard_cb(hadamard_block), bits_intra,
                                             static_cast<uint8_t*>(intra_send), unit_bytes(S, bits_intra, group),
                                             sm_count_current() * 8, st);
  return e == cudaSuccess ? SDP4_OK : fail(SDP4_ECUDA, "K3 launch failed: %s", cudaGetErrorString(e));
}

sdp4_status sdp4_tlq_stage_reduce(const void* intra_recv, size_t numel, int M, int N, int bits_intra,
                                  int bits_inter, int group, void* inter_send, void* stream) {
  g_err.clear();
  if (M < 1 || N < 1) return fail(SDP4_EINVAL, "bad topology %d x %d", M, N);
  sdp4_status s = check_tlq_args(M * N, numel, bits_intra, bits_inter, group, 0);
  if (s != SDP4_OK) return s;
  if ((s = check_ptr(intra_recv, "intra_recv")) != SDP4_OK) return s;
  if ((s = check_ptr(inter_send, "inter_send")) != SDP4_OK) return s;
  const size_t S = numel / ((size_t)M * N);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = sdp4::launch_tlq_dq_reduce_q(static_cast<const uint8_t*>(intra_recv),
                                               unit_bytes(S, bits_intra, group), bits_intra, N, M, S, group,
                                               static_cast<uint8_t*>(inter_send), unit_bytes(S, bits_inter, group),
                                               bits_inter, sm_count_current() * 8, st);
  return e == cudaSuccess ? SDP4_OK : fail(SDP4_ECUDA, "K4 launch failed: %s", cudaGetErrorString(e));
}

sdp4_status sdp4_tlq_stage_final(const void* inter_recv, size_t numel, int M, int N, int bits_inter, int group,
                                 int hadamard_block, int average, float* out_shard, void* stream) {
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
                                                 out_shard, sm_count_current() * 8, st);
  return e == cudaSuccess ? SDP4_OK : fail(SDP4_ECUDA, "K5 launch failed: %s", cudaGetErrorString(e));
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
  if (!c) return fail(SDP4_EINVAL, "comm is NULL");
  if (numel % (size_t)c->world) return fail(SDP4_EALIGN, "numel not divisible by world");
  const ncclDataType_t dt = dtype == SDP4_BF16 ? ncclBfloat16 : ncclFloat32;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (c->world == 1) {
    const size_t bytes = numel * (dtype == SDP4_BF16 ? 2 : 4);
    cudaError_t e = cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, st);
    return e == cudaSuccess ? SDP4_OK : fail(SDP4_ECUDA, "%s", cudaGetErrorString(e));
  }
  return nccl_check(ncclReduceScatter(send, recv, numel / c->world, dt, average ? ncclAvg : ncclSum, c->world_c, st),
                    "ncclReduceScatter");
}

sdp4_status sdp4_nccl_all_gather(sdp4_comm_t c, const void* send, void* recv, size_t numel, sdp4_dtype dtype,
                                 void* stream) {
  if (!c) return fail(SDP4_EINVAL, "comm is NULL");
  if (numel % (size_t)c->world) return fail(SDP4_EALIGN, "numel not divisible by world");
  const ncclDataType_t dt = dtype == SDP4_BF16 ? ncclBfloat16 : ncclFloat32;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (c->world == 1) {
    const size_t bytes = numel * (dtype == SDP4_BF16 ? 2 : 4);
    cudaError_t e = cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, st);
    return e == cudaSuccess ? SDP4_OK : fail(SDP4_ECUDA, "%s", cudaGetErrorString(e));
  }
  return nccl_check(ncclAllGather(send, recv, numel / c->world, dt, c->world_c, st), "ncclAllGather");
}

}  // extern "C"
