// latency_probe.cu -- fixed costs behind the small-message P2P latency.
// One process, two GPUs with peer access:
//  (1) per-node cost of a captured graph: 1 vs 6 empty kernels on one stream;
//  (2) cross-GPU flag ping-pong inside one kernel per GPU (st.release.sys to the peer's flag,
//      ld.acquire.sys polls of the local flag): one-way latency = total / (2 * rounds);
//  (3) the stream-ordered hand-off the multi-launch path uses: GPU0 kernel -> memop write of
//      GPU1's flag -> GPU1 wait kernel -> GPU1 kernel, timed per hand-off.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/latency_probe tools/latency_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));         \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

__global__ void k_empty() {}

__device__ __forceinline__ uint32_t ld_acq(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ping-pong: side 0 starts; each round waits for local == expected, then writes peer
__global__ void k_pingpong(uint32_t* local, uint32_t* peer, int side, int rounds) {
  if (threadIdx.x) return;
  for (int r = 1; r <= rounds; ++r) {
    if (side == 0) {
      st_rel(peer, (uint32_t)r);
      while (ld_acq(local) != (uint32_t)r) {}
    } else {
      while (ld_acq(local) != (uint32_t)r) {}
      st_rel(peer, (uint32_t)r);
    }
  }
}

__global__ void k_wait(uint32_t* f) {
  if (threadIdx.x) return;
  while (ld_acq(f) == 0u) {}
  *f = 0u;
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    printf("{\"error\": \"needs 2 GPUs\"}\n");
    return 0;
  }
  cuInit(0);
  // (1) graph node overhead on GPU 0
  CK(cudaSetDevice(0));
  cudaStream_t s0;
  CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int nodes : {1, 6}) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s0, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < nodes; ++i) k_empty<<<148, 128, 0, s0>>>();
    CK(cudaStreamEndCapture(s0, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    for (int i = 0; i < 20; ++i) CK(cudaGraphLaunch(ge, s0));
    CK(cudaStreamSynchronize(s0));
    const int reps = 200;
    CK(cudaEventRecord(a, s0));
    for (int i = 0; i < reps; ++i) CK(cudaGraphLaunch(ge, s0));
    CK(cudaEventRecord(b, s0));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("{\"probe\": \"graph_empty_kernels\", \"nodes\": %d, \"us_per_graph\": %.2f}\n", nodes, ms * 1e3 / reps);
    // eager launches of the same count
    CK(cudaEventRecord(a, s0));
    for (int i = 0; i < reps; ++i)
      for (int j = 0; j < nodes; ++j) k_empty<<<148, 128, 0, s0>>>();
    CK(cudaEventRecord(b, s0));
    CK(cudaEventSynchronize(b));
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("{\"probe\": \"eager_empty_kernels\", \"nodes\": %d, \"us_per_group\": %.2f}\n", nodes, ms * 1e3 / reps);
    CK(cudaGraphExecDestroy(ge));
    CK(cudaGraphDestroy(g));
  }
  // (2) in-kernel ping-pong
  uint32_t* f[2];
  cudaStream_t st[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    cudaError_t e = cudaDeviceEnablePeerAccess(1 - d, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
    cudaGetLastError();
    CK(cudaMalloc(&f[d], 4096));
    CK(cudaMemset(f[d], 0, 4096));
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
  }
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceSynchronize());
  }
  const int rounds = 20000;
  cudaEvent_t e0, e1;
  CK(cudaSetDevice(0));
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaSetDevice(1));
  k_pingpong<<<1, 32, 0, st[1]>>>(f[1], f[0], 1, rounds);
  CK(cudaSetDevice(0));
  CK(cudaEventRecord(e0, st[0]));
  k_pingpong<<<1, 32, 0, st[0]>>>(f[0], f[1], 0, rounds);
  CK(cudaEventRecord(e1, st[0]));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  printf("{\"probe\": \"in_kernel_pingpong\", \"rounds\": %d, \"one_way_us\": %.3f}\n", rounds, ms * 1e3 / (2.0 * rounds));
  // (3) stream-ordered hand-off: GPU0 empty kernel + memop write to GPU1's flag; GPU1 wait kernel + empty kernel
  CK(cudaSetDevice(1));
  CK(cudaMemset(f[1], 0, 4096));
  CK(cudaDeviceSynchronize());
  cudaEvent_t g1a, g1b;
  CK(cudaEventCreate(&g1a));
  CK(cudaEventCreate(&g1b));
  const int hand = 500;
  // GPU1: hand waits, each followed by an empty kernel
  CK(cudaEventRecord(g1a, st[1]));
  for (int i = 0; i < hand; ++i) {
    k_wait<<<1, 32, 0, st[1]>>>(f[1]);
    k_empty<<<148, 128, 0, st[1]>>>();
  }
  CK(cudaEventRecord(g1b, st[1]));
  CK(cudaSetDevice(0));
  CK(cudaEventRecord(e0, st[0]));
  for (int i = 0; i < hand; ++i) {
    k_empty<<<148, 128, 0, st[0]>>>();
    CUresult r = cuStreamWriteValue32((CUstream)st[0], (CUdeviceptr)f[1], 1u, CU_STREAM_WRITE_VALUE_DEFAULT);
    if (r != CUDA_SUCCESS) {
      printf("memop %d\n", (int)r);
      return 1;
    }
    // wait for GPU1 to consume before the next write (flag back to 0) -- a memop wait here
    cuStreamWaitValue32((CUstream)st[0], (CUdeviceptr)f[1], 0u, CU_STREAM_WAIT_VALUE_EQ);
  }
  CK(cudaEventRecord(e1, st[0]));
  CK(cudaEventSynchronize(e1));
  CK(cudaSetDevice(1));
  CK(cudaEventSynchronize(g1b));
  float ms1;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  CK(cudaEventElapsedTime(&ms1, g1a, g1b));
  printf("{\"probe\": \"stream_handoff\", \"handoffs\": %d, \"gpu0_us_per\": %.2f, \"gpu1_us_per\": %.2f}\n", hand,
         ms * 1e3 / hand, ms1 * 1e3 / hand);
  return 0;
}
