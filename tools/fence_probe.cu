// fence_probe.cu -- cost of memory fences / release operations on B200 (one warp timing itself
// with clock64): after local or peer (NVLink) stores, fence.sc.gpu vs fence.sc.sys vs
// fence.acq_rel.sys vs a release store.  Guides the one-launch kernels' sync (k_fused.cu).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/fence_probe tools/fence_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                            \
  do {                                                                   \
    cudaError_t e_ = (x);                                                \
    if (e_ != cudaSuccess) {                                             \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));  \
      exit(1);                                                           \
    }                                                                    \
  } while (0)

template <int MODE>
__global__ void k_fence(uint4* dst, int nstore, long long* out, int reps) {
  const int lane = threadIdx.x;
  long long tot_store = 0, tot_fence = 0;
  for (int r = 0; r < reps; ++r) {
    const long long t0 = clock64();
    for (int i = 0; i < nstore; ++i) dst[(r * nstore + i) * 32 + lane] = make_uint4(r, i, lane, 1);
    const long long t1 = clock64();
    if (MODE == 0) asm volatile("fence.sc.gpu;" ::: "memory");
    if (MODE == 1) asm volatile("fence.sc.sys;" ::: "memory");
    if (MODE == 2) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    if (MODE == 3) asm volatile("fence.acq_rel.sys;" ::: "memory");
    if (MODE == 4) {
      __syncwarp();
      if (lane == 0) {
        unsigned v;
        asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(v) : "l"(reinterpret_cast<unsigned*>(out + 8)) : "memory");
      }
      __syncwarp();
    }
    if (MODE == 5) {
      __syncwarp();
      if (lane == 0) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(reinterpret_cast<unsigned*>(out + 9)), "r"(1u) : "memory");
      __syncwarp();
    }
    const long long t2 = clock64();
    tot_store += t1 - t0;
    tot_fence += t2 - t1;
  }
  if (lane == 0) {
    out[0] = tot_store / reps;
    out[1] = tot_fence / reps;
  }
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  const int reps = 200, nstore = 4;
  long long* out;
  uint4* loc[2] = {nullptr, nullptr};
  for (int d = 0; d < (n > 1 ? 2 : 1); ++d) {
    CK(cudaSetDevice(d));
    CK(cudaMalloc(&loc[d], (size_t)reps * nstore * 32 * 16));
    if (n > 1) {
      cudaError_t e = cudaDeviceEnablePeerAccess(1 - d, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
      cudaGetLastError();
    }
  }
  CK(cudaSetDevice(0));
  CK(cudaMallocManaged(&out, 16 * sizeof(long long)));
  const char* names[6] = {"fence.sc.gpu", "fence.sc.sys", "fence.acq_rel.gpu", "fence.acq_rel.sys",
                          "lane0 atom.acq_rel.gpu", "lane0 st.release.sys"};
  for (int target = 0; target < (n > 1 ? 2 : 1); ++target) {
    for (int mode = 0; mode < 6; ++mode) {
      for (int w = 0; w < 2; ++w) {  // warm-up, then measure
        switch (mode) {
          case 0: k_fence<0><<<1, 32>>>(loc[target], nstore, out, reps); break;
          case 1: k_fence<1><<<1, 32>>>(loc[target], nstore, out, reps); break;
          case 2: k_fence<2><<<1, 32>>>(loc[target], nstore, out, reps); break;
          case 3: k_fence<3><<<1, 32>>>(loc[target], nstore, out, reps); break;
          case 4: k_fence<4><<<1, 32>>>(loc[target], nstore, out, reps); break;
          case 5: k_fence<5><<<1, 32>>>(loc[target], nstore, out, reps); break;
        }
        CK(cudaDeviceSynchronize());
      }
      printf("{\"stores\": \"%s\", \"op\": \"%s\", \"store_cycles\": %lld, \"op_cycles\": %lld}\n",
             target ? "peer" : "local", names[mode], out[0], out[1]);
    }
  }
  return 0;
}
