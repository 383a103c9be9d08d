// k_fused_tlq8.cu -- one-launch TLq-HS, 8-bit intra codes (see k_fused_tlq.cuh).
#include "k_fused_tlq.cuh"

namespace sdp4 {

cudaError_t launch_fused_tlq_bi8(const FusedSync& fs, const FtlqArgs& a, int be, int b, bool stoch, int grid,
                                 cudaStream_t st) {
  return be == 4 ? fused_tlq_b<8, 4>(fs, a, b, stoch, grid, st) : fused_tlq_b<8, 8>(fs, a, b, stoch, grid, st);
}

}  // namespace sdp4
