// k_fused.cuh -- device helpers of the one-launch P2P kernels (k_fused.cu, k_fused_tlq*.cu).
#pragma once
#include "sdp4_device.cuh"

namespace sdp4 {
namespace {


__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Phase timestamps (debugging only, fs.trace != nullptr): even slots keep the earliest stamp,
// odd slots the latest (entry 0 / exit 7 likewise: slot 0 min, slot 7 max).
__device__ __forceinline__ void tstamp(const FusedSync& fs, int v, int slot) {
  if (!fs.trace) return;
  unsigned long long* p = fs.trace + v * kTraceSlots + slot;
  const unsigned long long t = gtimer();
  if (slot & 1) atomicMax(p, t);
  else atomicMin(p, t);
}

// Counter block (FusedSync::ctr): [0] task claims, [1] exits, [2 + ph * kMaxVr + v] tasks of
// phase ph done for virtual rank v.
__device__ __forceinline__ uint32_t* done_ctr(const FusedSync& fs, int ph, int v) { return fs.ctr + 2 + ph * kMaxVr + v; }

// Poll a flag of this rank's own buffer until non-zero (a peer's release store).  Past the
// deadline the code goes to the host-mapped error word and the wait gives up: the call's
// results are then garbage, the stream drains, and the next call returns SDP4_ETIMEOUT.
__device__ __forceinline__ void wait_flag(const FusedSync& fs, const uint32_t* f, uint32_t code) {
  if (ld_acquire_sys(f)) return;
  const unsigned long long t0 = gtimer();
  for (;;) {
    __nanosleep(20);
    if (ld_acquire_sys(f)) return;
    if (fs.timeout_ns && gtimer() - t0 > fs.timeout_ns) {
      if (fs.err) *reinterpret_cast<volatile uint32_t*>(fs.err) = code;
      return;
    }
  }
}
// Wait until `n` tasks of phase ph of virtual rank v are done (same launch).
__device__ __forceinline__ void wait_done(const FusedSync& fs, int ph, int v, uint32_t n) {
  const uint32_t* c = done_ctr(fs, ph, v);
  if (ld_acquire_gpu(c) >= n) return;
  const unsigned long long t0 = gtimer();
  for (;;) {
    __nanosleep(20);
    if (ld_acquire_gpu(c) >= n) return;
    if (fs.timeout_ns && gtimer() - t0 > fs.timeout_ns) {
      if (fs.err) *reinterpret_cast<volatile uint32_t*>(fs.err) = 0x80ff0000u | (uint32_t)ph;
      return;
    }
  }
}
__device__ __forceinline__ uint32_t* flag(const FusedSync& fs, int owner, int kind, int stage, int src) {
  return fs.flags[owner] + flag_word(kind, stage, src);
}
__device__ __forceinline__ uint32_t wait_code(int kind, int stage, int src) {
  return 0x80000000u | ((uint32_t)kind << 24) | ((uint32_t)stage << 16) | (uint32_t)src;
}

// Count one finished task of phase ph (after the caller's system-scope fence); true for the
// last one of virtual rank v, which then owns the phase's flag resets and raises.
__device__ __forceinline__ bool finish_task(const FusedSync& fs, int ph, int v, uint32_t total) {
  const uint32_t old = atomicAdd(done_ctr(fs, ph, v), 1u);
  if (old + 1 == total) {
    __threadfence_system();  // acquire side: every counted task's writes precede the raises
    return true;
  }
  return false;
}
// The last unit of work of the launch resets the counter block for the next launch.
__device__ __forceinline__ void exit_unit(const FusedSync& fs, uint32_t units) {
  if (atomicAdd(fs.ctr + 1, 1u) + 1 == units)
    for (int i = 0; i < kFusedCtrWords; ++i) fs.ctr[i] = 0u;
}


constexpr int kFThreads = 256;
constexpr int kFtRows = 32;                   // one-launch TLq-HS: rows per warp task
constexpr int kFtTask = kFtRows * kRowElems;  // 2048 elements

}  // namespace

struct FtlqArgs {
  const void* grad[kMaxVr];
  float* out[kMaxVr];
  uint32_t key8[kMaxVr], key4[kMaxVr];
  size_t S, w8, w4;
  int M, N, lg, sr_on, grad_bf16;
  float cb, kappa, z;
  uint32_t m16;
};

// per-BI instantiation units of the one-launch TLq-HS kernel (k_fused_tlq8.cu / k_fused_tlq4.cu)
cudaError_t launch_fused_tlq_bi8(const FusedSync& fs, const FtlqArgs& a, int be, int b, bool stoch, int grid,
                                 cudaStream_t st);
cudaError_t launch_fused_tlq_bi4(const FusedSync& fs, const FtlqArgs& a, int be, int b, bool stoch, int grid,
                                 cudaStream_t st);

}  // namespace sdp4
