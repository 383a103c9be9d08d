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

// Phase timestamps (debugging only, fs.trace != nullptr): every warp (TLq-HS) or CTA (qWD)
// owns kTraceSlots private words -- plain stores, no contention that would distort the
// timeline -- entry, exit, and per phase the start of its first task (after the waits) and
// the end of its last; the host takes min / max over units.
__device__ __forceinline__ void tstamp(const FusedSync& fs, int unit, int slot) {
  if (!fs.trace || unit >= kTraceUnits) return;
  unsigned long long* p = fs.trace + (size_t)unit * kTraceSlots + slot;
  if ((slot & 1) || *p == 0ull) *p = gtimer();
}

// Counter block (FusedSync::ctr): [0] task claims, [1] exits, [2 + ph * kMaxVr + v] tasks of
// phase ph done for virtual rank v.
__device__ __forceinline__ uint32_t* done_ctr(const FusedSync& fs, int ph, int v) { return fs.ctr + 2 + ph * kMaxVr + v; }

// Poll a flag of this rank's own buffer until non-zero (a peer's release).  The loop polls with
// relaxed loads and only the final read is an acquire: every acquire load invalidates the SM's
// L1 (CCTL.IVALL), which in a polling loop stalled the whole SM (ncu: 30% of samples).  Past
// the deadline the code goes to the host-mapped error word and the wait gives up: the call's
// results are then garbage, the stream drains, and the next call returns SDP4_ETIMEOUT.
__device__ __forceinline__ uint32_t ld_relaxed_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wait_flag(const FusedSync& fs, const uint32_t* f, uint32_t code) {
  if (!ld_relaxed_sys(f)) {
    const unsigned long long t0 = gtimer();
    for (;;) {
      __nanosleep(20);
      if (ld_relaxed_sys(f)) break;
      if (fs.timeout_ns && gtimer() - t0 > fs.timeout_ns) {
        if (fs.err) *reinterpret_cast<volatile uint32_t*>(fs.err) = code;
        return;
      }
    }
  }
  (void)ld_acquire_sys(f);  // acquire: the peer's writes before its raise are visible
}
// Wait until `n` tasks of phase ph of virtual rank v are done (same launch).
__device__ __forceinline__ void wait_done(const FusedSync& fs, int ph, int v, uint32_t n) {
  const uint32_t* c = done_ctr(fs, ph, v);
  if (ld_relaxed_gpu(c) < n) {
    const unsigned long long t0 = gtimer();
    for (;;) {
      __nanosleep(20);
      if (ld_relaxed_gpu(c) >= n) break;
      if (fs.timeout_ns && gtimer() - t0 > fs.timeout_ns) {
        if (fs.err) *reinterpret_cast<volatile uint32_t*>(fs.err) = 0x80ff0000u | (uint32_t)ph;
        return;
      }
    }
  }
  (void)ld_acquire_gpu(c);
}
__device__ __forceinline__ uint32_t* flag(const FusedSync& fs, int owner, int kind, int stage, int src) {
  return fs.flags[owner] + flag_word(kind, stage, src);
}
__device__ __forceinline__ uint32_t wait_code(int kind, int stage, int src) {
  return 0x80000000u | ((uint32_t)kind << 24) | ((uint32_t)stage << 16) | (uint32_t)src;
}

// Count one finished task of phase ph.  Called by ONE thread after a warp / CTA barrier over
// the task's threads, so this release atomic at gpu scope releases every write of the task --
// to local or peer memory (a gpu-scope fence also waits for NVLink stores, ~0.45 us vs ~1.9 us
// at system scope: tools/fence_probe.cu).  True for the last task of virtual rank v: that
// thread resets its own flags, then one fence.sc.sys (the acquire of every task's release, and
// the release of the raises) and relaxed stores raise the peers' flags.
__device__ __forceinline__ bool finish_task(const FusedSync& fs, int ph, int v, uint32_t total) {
  uint32_t old;
  asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(done_ctr(fs, ph, v)) : "memory");
  return old + 1 == total;
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
  uint32_t dbg;  // measurement switches (SDP4_FUSED_DBG), 0 in normal use
};

// per-BI instantiation units of the one-launch TLq-HS kernel (k_fused_tlq8.cu / k_fused_tlq4.cu)
cudaError_t launch_fused_tlq_bi8(const FusedSync& fs, const FtlqArgs& a, int be, int b, bool stoch, int grid,
                                 cudaStream_t st);
cudaError_t launch_fused_tlq_bi4(const FusedSync& fs, const FtlqArgs& a, int be, int b, bool stoch, int grid,
                                 cudaStream_t st);

}  // namespace sdp4
