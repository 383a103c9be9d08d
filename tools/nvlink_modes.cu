// nvlink_modes.cu -- NVLink throughput of the access patterns the fused exchanges can use,
// with every GPU active at once (the all-to-all case), one process driving all GPUs:
//   push-bulk : each GPU bulk-stores 16 KB smem tiles into its peers' buffers
//   pull-bulk : each GPU bulk-loads 16 KB tiles from its peers' buffers into smem
//   pull-ldg  : each GPU reads its peers' buffers with ld.global.v4 (grid-stride)
//   push-stg  : each GPU writes its peers' buffers with st.global.v4 (grid-stride)
// Peers are all other GPUs (round-robin tiles).  Prints per-GPU GB/s per direction.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o nvlink_modes tools/nvlink_modes.cu -lcuda
#include <cstdint>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("FAIL %s: %s (line %d)\n", #x, cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int kTile = 16384;
constexpr int kMaxPeers = 8;
struct Peers {
  uint8_t* p[kMaxPeers];
  int n;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// tiles per peer = bytes_per_peer / kTile; CTA b handles tiles b, b+grid, ... over (peer, tile)
__global__ void push_bulk(Peers peers, size_t tiles_per_peer, size_t off) {
  extern __shared__ __align__(128) uint8_t sm[];
  for (int i = threadIdx.x; i < 4 * kTile; i += blockDim.x) sm[i] = (uint8_t)i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x) return;
  const size_t total = tiles_per_peer * peers.n;
  int k = 0;
  for (size_t t = blockIdx.x; t < total; t += gridDim.x, ++k) {
    const int q = (int)(t % peers.n);
    const size_t i = t / peers.n;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(peers.p[q] + off + i * kTile),
                 "r"(smem_u32(sm + (k & 3) * kTile)), "r"(kTile) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void pull_bulk(Peers peers, size_t tiles_per_peer, size_t off, int stages) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[8];
  if (threadIdx.x) return;
  for (int s = 0; s < stages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t total = tiles_per_peer * peers.n;
  uint32_t phase[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  auto issue = [&](size_t t, int s) {
    const int q = (int)(t % peers.n);
    const size_t i = t / peers.n;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(kTile) : "memory");
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(sm + s * kTile)),
                 "l"(peers.p[q] + off + i * kTile), "r"(kTile), "r"(smem_u32(&bar[s])) : "memory");
  };
  size_t t = blockIdx.x;
  int k = 0;
  for (int s = 0; s < stages && t + (size_t)s * gridDim.x < total; ++s) issue(t + (size_t)s * gridDim.x, s);
  for (; t < total; t += gridDim.x, ++k) {
    const int s = k % stages;
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(
                     smem_u32(&bar[s])), "r"(phase[s]) : "memory");
    phase[s] ^= 1;
    const size_t nt = t + (size_t)stages * gridDim.x;
    if (nt < total) issue(nt, s);
  }
}

__global__ void pull_ldg(Peers peers, size_t bytes_per_peer, size_t off, uint4* sink) {
  const size_t n16 = bytes_per_peer / 16;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16 * peers.n; i += (size_t)gridDim.x * blockDim.x) {
    const int q = (int)((i / 1024) % peers.n);
    const size_t j = (i / 1024 / peers.n) * 1024 + (i % 1024);
    const uint4 v = reinterpret_cast<const uint4*>(peers.p[q] + off)[j];
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if (acc.x == 0x12345678u) sink[0] = acc;
}

__global__ void push_stg(Peers peers, size_t bytes_per_peer, size_t off) {
  const size_t n16 = bytes_per_peer / 16;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16 * peers.n; i += (size_t)gridDim.x * blockDim.x) {
    const int q = (int)((i / 1024) % peers.n);
    const size_t j = (i / 1024 / peers.n) * 1024 + (i % 1024);
    reinterpret_cast<uint4*>(peers.p[q] + off)[j] = make_uint4((uint32_t)i, 1, 2, 3);
  }
}

int main(int argc, char** argv) {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) { printf("need >= 2 GPUs\n"); return 1; }
  const int G = n > 8 ? 8 : n;
  const size_t per_peer = (size_t)256 << 20;  // 256 MB from each GPU to each peer
  std::vector<uint8_t*> buf(G);
  std::vector<cudaStream_t> st(G);
  std::vector<uint4*> sink(G);
  for (int d = 0; d < G; ++d) {
    CK(cudaSetDevice(d));
    for (int e = 0; e < G; ++e)
      if (e != d) cudaDeviceEnablePeerAccess(e, 0);
    cudaGetLastError();
    CK(cudaMalloc(&buf[d], per_peer * G));  // slot s = written by / read for GPU s
    CK(cudaMemset(buf[d], 1, per_peer * G));
    CK(cudaMalloc(&sink[d], 64));
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    CK(cudaFuncSetAttribute(push_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * kTile));
    CK(cudaFuncSetAttribute(pull_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * kTile));
  }
  for (int active = 2; active <= G; active *= 2) {
    for (int mode = 0; mode < 4; ++mode) {
      const char* names[4] = {"push-bulk", "pull-bulk", "pull-ldg", "push-stg"};
      for (int ctas : {148, 296}) {
        float best = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {
          std::vector<cudaEvent_t> e0(active), e1(active);
          for (int d = 0; d < active; ++d) {
            cudaSetDevice(d);
            cudaDeviceSynchronize();
          }
          for (int d = 0; d < active; ++d) {
            cudaSetDevice(d);
            cudaEventCreate(&e0[d]);
            cudaEventCreate(&e1[d]);
            Peers p;
            p.n = 0;
            for (int q = 0; q < active; ++q)
              if (q != d) p.p[p.n++] = buf[q];
            // push: write my slot (d) in each peer's buffer; pull: read my slot in each peer
            const size_t off = per_peer * d;
            cudaEventRecord(e0[d], st[d]);
            if (mode == 0) push_bulk<<<ctas, 32, 4 * kTile, st[d]>>>(p, per_peer / kTile, off);
            if (mode == 1) pull_bulk<<<ctas, 32, 8 * kTile, st[d]>>>(p, per_peer / kTile, off, 8);
            if (mode == 2) pull_ldg<<<ctas * 2, 512, 0, st[d]>>>(p, per_peer, off, sink[d]);
            if (mode == 3) push_stg<<<ctas * 2, 512, 0, st[d]>>>(p, per_peer, off);
            cudaEventRecord(e1[d], st[d]);
          }
          float worst = 0.f;
          for (int d = 0; d < active; ++d) {
            cudaSetDevice(d);
            CK(cudaEventSynchronize(e1[d]));
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0[d], e1[d]);
            worst = ms > worst ? ms : worst;
            cudaEventDestroy(e0[d]);
            cudaEventDestroy(e1[d]);
          }
          best = worst < best ? worst : best;
        }
        const double bytes = (double)per_peer * (active - 1);
        printf("gpus=%d %-9s ctas=%d: %.1f GB/s per GPU per direction\n", active, names[mode], ctas,
               bytes / (best * 1e-3) / 1e9);
      }
    }
  }
  printf("DONE\n");
  return 0;
}
