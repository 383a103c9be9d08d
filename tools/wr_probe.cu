// wr_probe.cu -- which store patterns reach the HBM write ceiling (torch's fill_ measures
// ~7.4 TB/s, a grid-stride 16-byte-per-iteration kernel ~6.2): non-persistent grids with U
// 16-byte stores per thread, grid-stride variants, and cache hints.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int U, int HINT>
__global__ void __launch_bounds__(256) wr_block(uint4* __restrict__ out, size_t n) {
  const size_t base = (size_t)blockIdx.x * 256 * U + threadIdx.x;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const size_t i = base + (size_t)u * 256;
    if (i < n) {
      const uint4 v = make_uint4((uint32_t)i, (uint32_t)i * 3u, 7u, ~(uint32_t)i);
      if (HINT == 0) out[i] = v;
      else if (HINT == 1) __stcs(out + i, v);
      else __stwt(out + i, v);
    }
  }
}
template <int U>
__global__ void __launch_bounds__(256) wr_stride(uint4* __restrict__ out, size_t n) {
  const size_t step = (size_t)gridDim.x * 256 * U;
  for (size_t base = (size_t)blockIdx.x * 256 * U + threadIdx.x; base < n; base += step) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t i = base + (size_t)u * 256;
      if (i < n) out[i] = make_uint4((uint32_t)i, (uint32_t)i * 3u, 7u, ~(uint32_t)i);
    }
  }
}

// persistent cyclic, but the slot within each grid-sized window rotates every iteration
// (CTA k writes tile i*G + (k + i*ROT) mod G): same compact front, no fixed SM->address phase
template <int ROT>
__global__ void __launch_bounds__(256) wr_rot(uint4* __restrict__ out, size_t n) {
  const size_t tiles = (n + 1023) / 1024, G = gridDim.x;
  for (size_t it = 0;; ++it) {
    const size_t t = it * G + (blockIdx.x + it * ROT) % G;
    if (it * G >= tiles) break;
    if (t >= tiles) continue;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const size_t i = t * 1024 + u * 256 + threadIdx.x;
      if (i < n) out[i] = make_uint4((uint32_t)i, (uint32_t)i * 3u, 7u, ~(uint32_t)i);
    }
  }
}
// non-persistent, blocks visit tiles in a scrambled order (tests "compact front" vs "spread")
__global__ void __launch_bounds__(256) wr_scr(uint4* __restrict__ out, size_t n, size_t tiles) {
  const size_t t = ((size_t)blockIdx.x * 2654435761ull) % tiles;  // a bijection when gcd(.., tiles) == 1
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const size_t i = t * 1024 + u * 256 + threadIdx.x;
    if (i < n) out[i] = make_uint4((uint32_t)i, (uint32_t)i * 3u, 7u, ~(uint32_t)i);
  }
}
// persistent, contiguous range per CTA (blocked distribution)
__global__ void __launch_bounds__(256) wr_blocked(uint4* __restrict__ out, size_t n) {
  const size_t tiles = (n + 1023) / 1024, per = (tiles + gridDim.x - 1) / gridDim.x;
  const size_t t0 = blockIdx.x * per, t1 = min(tiles, t0 + per);
  for (size_t t = t0; t < t1; ++t)
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const size_t i = t * 1024 + u * 256 + threadIdx.x;
      if (i < n) out[i] = make_uint4((uint32_t)i, (uint32_t)i * 3u, 7u, ~(uint32_t)i);
    }
}
// persistent, tiles handed out in launch order by a global atomic counter
__global__ void __launch_bounds__(256) wr_dyn(uint4* __restrict__ out, size_t n, unsigned long long* ctr) {
  __shared__ unsigned long long tile;
  const size_t tiles = (n + 1023) / 1024;
  for (;;) {
    if (threadIdx.x == 0) tile = atomicAdd(ctr, 1ull);
    __syncthreads();
    const size_t t = tile;
    __syncthreads();
    if (t >= tiles) break;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const size_t i = t * 1024 + u * 256 + threadIdx.x;
      if (i < n) out[i] = make_uint4((uint32_t)i, (uint32_t)i * 3u, 7u, ~(uint32_t)i);
    }
  }
}
// persistent, dynamic tiles fetched one iteration ahead (the atomic's latency is hidden), one
// warp fetching for the CTA, chunks of C tiles per fetch
template <int C>
__global__ void __launch_bounds__(256) wr_dyn2(uint4* __restrict__ out, size_t n, unsigned long long* ctr) {
  __shared__ unsigned long long nxt[2];
  const size_t tiles = (n + 1023) / 1024;
  if (threadIdx.x == 0) nxt[0] = atomicAdd(ctr, (unsigned long long)C);
  __syncthreads();
  for (int it = 0;; ++it) {
    const size_t t0 = nxt[it & 1];
    if (threadIdx.x == 0) nxt[(it + 1) & 1] = atomicAdd(ctr, (unsigned long long)C);
    if (t0 >= tiles) break;
    for (int c = 0; c < C; ++c) {
      const size_t t = t0 + c;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const size_t i = t * 1024 + u * 256 + threadIdx.x;
        if (i < n) out[i] = make_uint4((uint32_t)i, (uint32_t)i * 3u, 7u, ~(uint32_t)i);
      }
    }
    __syncthreads();
  }
}
// copy 1:1, non-persistent vs persistent cyclic
__global__ void __launch_bounds__(256) cp_block(const uint4* __restrict__ in, uint4* __restrict__ out, size_t n) {
  const size_t base = (size_t)blockIdx.x * 1024 + threadIdx.x;
  uint4 v[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) v[u] = base + u * 256 < n ? in[base + u * 256] : make_uint4(0, 0, 0, 0);
#pragma unroll
  for (int u = 0; u < 4; ++u) if (base + u * 256 < n) out[base + u * 256] = v[u];
}
__global__ void __launch_bounds__(256) cp_stride(const uint4* __restrict__ in, uint4* __restrict__ out, size_t n) {
  for (size_t base = (size_t)blockIdx.x * 1024 + threadIdx.x; base < n; base += (size_t)gridDim.x * 1024) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = base + u * 256 < n ? in[base + u * 256] : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < 4; ++u) if (base + u * 256 < n) out[base + u * 256] = v[u];
  }
}

template <typename F>
void timeit(const char* name, F f, double bytes) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9f;
  for (int r = 0; r < 8; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r && ms < best) best = ms;
  }
  printf("{\"pattern\": \"%s\", \"ms\": %.4f, \"GBps\": %.1f}\n", name, best, bytes / best / 1e6);
}

int main() {
  const size_t bytes = (size_t)5 << 30, n = bytes / 16;
  uint4* out;
  cudaMalloc(&out, bytes);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  timeit("memset", [&] { cudaMemsetAsync(out, 0x3f, bytes); }, bytes);
  timeit("block U=1", [&] { wr_block<1, 0><<<(n + 255) / 256, 256>>>(out, n); }, bytes);
  timeit("block U=4", [&] { wr_block<4, 0><<<(n + 1023) / 1024, 256>>>(out, n); }, bytes);
  timeit("block U=8", [&] { wr_block<8, 0><<<(n + 2047) / 2048, 256>>>(out, n); }, bytes);
  timeit("block U=4 .cs", [&] { wr_block<4, 1><<<(n + 1023) / 1024, 256>>>(out, n); }, bytes);
  timeit("block U=4 .wt", [&] { wr_block<4, 2><<<(n + 1023) / 1024, 256>>>(out, n); }, bytes);
  for (int c : {2, 4, 8, 16})
    for (int u : {1, 4}) {
      char nm[64];
      snprintf(nm, sizeof(nm), "stride %d/SM U=%d", c, u);
      if (u == 1) timeit(nm, [&] { wr_stride<1><<<sms * c, 256>>>(out, n); }, bytes);
      else timeit(nm, [&] { wr_stride<4><<<sms * c, 256>>>(out, n); }, bytes);
    }
  for (int c : {2, 4, 8}) {
    char nm[64];
    snprintf(nm, sizeof(nm), "rotated(97) %d/SM", c);
    timeit(nm, [&] { wr_rot<97><<<sms * c, 256>>>(out, n); }, bytes);
    snprintf(nm, sizeof(nm), "rotated(1) %d/SM", c);
    timeit(nm, [&] { wr_rot<1><<<sms * c, 256>>>(out, n); }, bytes);
  }
  {
    const size_t tiles = (n + 1023) / 1024;
    timeit("scrambled non-persistent", [&] { wr_scr<<<tiles, 256>>>(out, n, tiles); }, bytes);
  }
  for (int c : {2, 4, 8}) {
    char nm[64];
    snprintf(nm, sizeof(nm), "blocked %d/SM", c);
    timeit(nm, [&] { wr_blocked<<<sms * c, 256>>>(out, n); }, bytes);
  }
  unsigned long long* ctr;
  cudaMalloc(&ctr, 8);
  for (int c : {2, 4, 8}) {
    char nm[64];
    snprintf(nm, sizeof(nm), "dynamic %d/SM", c);
    timeit(nm, [&] { cudaMemsetAsync(ctr, 0, 8); wr_dyn<<<sms * c, 256>>>(out, n, ctr); }, bytes);
  }
  for (int c : {1, 2, 4, 8}) {
    char nm[64];
    snprintf(nm, sizeof(nm), "dynamic-ahead %d/SM chunk1", c);
    timeit(nm, [&] { cudaMemsetAsync(ctr, 0, 8); wr_dyn2<1><<<sms * c, 256>>>(out, n, ctr); }, bytes);
    snprintf(nm, sizeof(nm), "dynamic-ahead %d/SM chunk4", c);
    timeit(nm, [&] { cudaMemsetAsync(ctr, 0, 8); wr_dyn2<4><<<sms * c, 256>>>(out, n, ctr); }, bytes);
  }
  uint4* in;
  const size_t cb = (size_t)2 << 30, cn = cb / 16;
  cudaMalloc(&in, cb);
  timeit("copy block (r+w)", [&] { cp_block<<<(cn + 1023) / 1024, 256>>>(in, out, cn); }, 2.0 * cb);
  for (int c : {2, 4, 8}) {
    char nm[64];
    snprintf(nm, sizeof(nm), "copy stride %d/SM (r+w)", c);
    timeit(nm, [&] { cp_stride<<<sms * c, 256>>>(in, out, cn); }, 2.0 * cb);
  }
  return 0;
}
