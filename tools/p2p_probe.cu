// p2p_probe.cu -- checks the NVLink primitives the fused exchange relies on (2 GPUs, one
// process): (1) TMA tensor store (cp.async.bulk.tensor) from smem to a PEER address,
// (2) 1-D bulk store to a peer address, (3) plain st.global to a peer, (4) stream memops
// cuStreamWriteValue32 to a peer flag + cuStreamWaitValue32 on the owner's stream,
// (5) peer-store bandwidth of a simple kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o p2p_probe tools/p2p_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("FAIL %s: %s (line %d)\n", #x, cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void tma_store_kernel(const __grid_constant__ CUtensorMap map, int pattern) {
  __shared__ __align__(1024) uint8_t tile[256 * 64];
  for (int i = threadIdx.x; i < 256 * 64; i += blockDim.x) tile[i] = (uint8_t)(i * 7 + pattern);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(&map), "r"(0),
                 "r"(256 * blockIdx.x), "r"(0), "r"(smem_u32(tile)) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

__global__ void bulk_store_kernel(uint8_t* dst, int pattern) {
  __shared__ __align__(128) uint8_t tile[16384];
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) tile[i] = (uint8_t)(i * 3 + pattern);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + 16384 * blockIdx.x),
                 "r"(smem_u32(tile)), "r"(16384) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

__global__ void stg_kernel(uint4* dst, size_t n16, uint32_t v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = make_uint4(v, v + 1, v + 2, (uint32_t)i);
}

__global__ void tma_bw_kernel(const __grid_constant__ CUtensorMap map, int tiles) {
  __shared__ __align__(1024) uint8_t tile[2][256 * 64];
  for (int i = threadIdx.x; i < 2 * 256 * 64; i += blockDim.x) (&tile[0][0])[i] = (uint8_t)i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    int k = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++k) {
      asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(&map),
                   "r"(0), "r"(256 * t), "r"(0), "r"(smem_u32(tile[k & 1])) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

__global__ void bulk_bw_kernel(uint8_t* dst, size_t tiles) {
  __shared__ __align__(128) uint8_t tile[2][16384];
  for (int i = threadIdx.x; i < 2 * 16384; i += blockDim.x) (&tile[0][0])[i] = (uint8_t)i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    int k = 0;
    for (size_t t = blockIdx.x; t < tiles; t += gridDim.x, ++k) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + 16384 * t),
                   "r"(smem_u32(tile[k & 1])), "r"(16384) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

// K4-like pattern: each lane stores 8 B per 32 B (4 stores complete a lane's 32 B span)
__global__ void stg64_kernel(uint2* dst, size_t n8) {
  const size_t lanes = (size_t)gridDim.x * blockDim.x;
  for (size_t base = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 4; base < n8; base += lanes * 4)
    for (int k = 0; k < 4; ++k) dst[base + k] = make_uint2((uint32_t)base, k);
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) { printf("need 2 GPUs\n"); return 1; }
  int can = 0;
  CK(cudaDeviceCanAccessPeer(&can, 0, 1));
  printf("canAccessPeer(0->1) = %d\n", can);
  CK(cudaSetDevice(1));
  uint8_t* remote;
  const size_t bytes = size_t(1) << 30;
  CK(cudaMalloc(&remote, bytes));
  CK(cudaMemset(remote, 0, bytes));
  uint32_t* flag1;
  CK(cudaMalloc(&flag1, 256));
  CK(cudaMemset(flag1, 0, 256));
  cudaStream_t s1;
  CK(cudaStreamCreate(&s1));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  cudaStream_t s0;
  CK(cudaStreamCreate(&s0));

  // (1) TMA tensor store to peer
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap map;
  cuuint64_t dims[3] = {64, 256 * 148, 1}, strides[2] = {64, 64ull * 256 * 148};
  cuuint32_t box[3] = {64, 256, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, remote, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode(peer ptr) = %d\n", (int)r);
  tma_store_kernel<<<148, 256, 0, s0>>>(map, 5);
  CK(cudaStreamSynchronize(s0));
  CK(cudaGetLastError());
  uint8_t h[4096];
  CK(cudaMemcpy(h, remote, 4096, cudaMemcpyDefault));
  int nz = 0;
  for (int i = 0; i < 4096; ++i) nz += h[i] != 0;
  printf("(1) TMA tensor store to peer: %s (%d/4096 nonzero)\n", nz > 3000 ? "OK" : "FAILED", nz);

  // (2) bulk store to peer
  CK(cudaMemset(remote, 0, 1 << 20));
  bulk_store_kernel<<<8, 256, 0, s0>>>(remote, 9);
  CK(cudaStreamSynchronize(s0));
  CK(cudaGetLastError());
  CK(cudaMemcpy(h, remote + 16384 * 3, 4096, cudaMemcpyDefault));
  int ok2 = 1;
  for (int i = 0; i < 4096; ++i) ok2 &= h[i] == (uint8_t)(i * 3 + 9);
  printf("(2) bulk store to peer: %s\n", ok2 ? "OK" : "FAILED");

  // (4) stream memops: write a flag on the peer from s0 after a kernel; s1 waits for it
  void* fw = nullptr;
  void* fwait = nullptr;
  CK(cudaGetDriverEntryPoint("cuStreamWriteValue32", &fw, cudaEnableDefault, &q));
  CK(cudaGetDriverEntryPoint("cuStreamWaitValue32", &fwait, cudaEnableDefault, &q));
  auto wv = (PFN_cuStreamWriteValue32_v11070)fw;
  auto wt = (PFN_cuStreamWaitValue32_v11070)fwait;
  stg_kernel<<<148, 512, 0, s0>>>((uint4*)remote, (32u << 20) / 16, 77);
  CUresult r1 = wv((CUstream)s0, (CUdeviceptr)flag1, 42, CU_STREAM_WRITE_VALUE_DEFAULT);
  CK(cudaSetDevice(1));
  CUresult r2 = wt((CUstream)s1, (CUdeviceptr)flag1, 42, CU_STREAM_WAIT_VALUE_GEQ);
  uint32_t* check;
  CK(cudaMalloc(&check, 4));
  CK(cudaMemcpyAsync(check, remote + (32u << 20) - 16 + 12, 4, cudaMemcpyDeviceToDevice, s1));
  uint32_t hv = 0;
  CK(cudaMemcpyAsync(&hv, check, 4, cudaMemcpyDeviceToHost, s1));
  CK(cudaStreamSynchronize(s1));
  printf("(4) stream memops write=%d wait=%d, data after wait %s (%u)\n", (int)r1, (int)r2,
         hv == (32u << 20) / 16 - 1 ? "OK" : "STALE", hv);
  CK(cudaSetDevice(0));

  // (5) peer store bandwidth (plain st.global.v4), 1 GiB, various grids
  cudaEvent_t a, b;  // (also used by (6))
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int g : {16, 32, 64, 148, 296}) {
    stg_kernel<<<g, 512, 0, s0>>>((uint4*)remote, bytes / 16, 1);
    CK(cudaEventRecord(a, s0));
    for (int it = 0; it < 5; ++it) stg_kernel<<<g, 512, 0, s0>>>((uint4*)remote, bytes / 16, it);
    CK(cudaEventRecord(b, s0));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("(5) peer st.global.v4 grid=%d x 512: %.1f GB/s\n", g, 5.0 * bytes / (ms * 1e-3) / 1e9);
  }
  // (6) bandwidth of TMA tensor stores / bulk stores to the peer (1 GiB region, many tiles)
  {
    CUtensorMap bm;
    const uint64_t rows = bytes / 64;
    cuuint64_t d3[3] = {64, rows, 1}, st3[2] = {64, bytes};
    cuuint32_t bx[3] = {64, 256, 1};
    enc(&bm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, remote, d3, st3, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int g : {148, 296}) {
      const int tiles = (int)(rows / 256);
      tma_bw_kernel<<<g, 256, 0, s0>>>(bm, tiles);
      CK(cudaEventRecord(a, s0));
      for (int it = 0; it < 5; ++it) tma_bw_kernel<<<g, 256, 0, s0>>>(bm, tiles);
      CK(cudaEventRecord(b, s0));
      CK(cudaEventSynchronize(b));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, a, b));
      CK(cudaGetLastError());
      printf("(6) peer TMA tensor store (16 KB boxes, SWIZZLE_64B) grid=%d: %.1f GB/s\n", g, 5.0 * bytes / (ms * 1e-3) / 1e9);
      bulk_bw_kernel<<<g, 256, 0, s0>>>(remote, bytes / 16384);
      CK(cudaEventRecord(a, s0));
      for (int it = 0; it < 5; ++it) bulk_bw_kernel<<<g, 256, 0, s0>>>(remote, bytes / 16384);
      CK(cudaEventRecord(b, s0));
      CK(cudaEventSynchronize(b));
      CK(cudaEventElapsedTime(&ms, a, b));
      printf("(6) peer bulk store (16 KB) grid=%d: %.1f GB/s\n", g, 5.0 * bytes / (ms * 1e-3) / 1e9);
      stg64_kernel<<<g, 256, 0, s0>>>((uint2*)remote, bytes / 8);
      CK(cudaEventRecord(a, s0));
      for (int it = 0; it < 5; ++it) stg64_kernel<<<g, 256, 0, s0>>>((uint2*)remote, bytes / 8);
      CK(cudaEventRecord(b, s0));
      CK(cudaEventSynchronize(b));
      CK(cudaEventElapsedTime(&ms, a, b));
      printf("(6) peer st.global.v2 at 32-byte lane stride grid=%d: %.1f GB/s\n", g, 5.0 * bytes / (ms * 1e-3) / 1e9);
    }
  }
  printf("DONE\n");
  return 0;
}
