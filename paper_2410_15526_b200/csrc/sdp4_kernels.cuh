// sdp4_kernels.cuh -- internal launcher interface between the C ABI (sdp4_api.cu)
// and the sm_100a kernels (sdp4_kernels.cu).  Not part of the public ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace sdp4 {

// Rows of 64 elements are the unit of the Hadamard kernels (one row per thread).
constexpr int kRowElems = 64;
constexpr int kTileRows = 256;                       // rows per CTA tile = threads per CTA
constexpr int kTileElems = kTileRows * kRowElems;    // 16384 elements

enum Dtype { kF32 = 0, kBF16 = 1 };

// K1: Alg. 2 l.2-3 -- d = w_main - w_model (this shard), k-bit group quantization
// into one wire unit.  Returns cudaGetLastError() of the launch.
cudaError_t launch_qwd_quantize(const float* w_main, const void* w_model_shard, int model_dtype,
                                size_t S, int bits, int G, uint8_t* unit, int grid_cap,
                                cudaStream_t st);

// K2: Alg. 2 l.5 -- for every shard j < P: w_model[jS..] += dequant(unit j), in place.
cudaError_t launch_qwd_apply(const uint8_t* units, size_t unit_bytes, int P, size_t S, int bits,
                             int G, void* w_model, int model_dtype, int grid_cap, cudaStream_t st);

// K3: Alg. 3 l.2-3 -- blockwise Hadamard (b, in {0,2,..,256}) + bits_intra quantization
// of the full gradient into the intra send layout (N blocks x M units).
cudaError_t launch_tlq_had_quant(const void* grad, int grad_dtype, size_t S, int M, int N, int G,
                                 int b, float cb, int bits, uint8_t* intra_send, size_t unit_bytes,
                                 int grid_cap, cudaStream_t st);

// K4: Alg. 3 l.5,7,9 -- dequantize N received units per sub-block m', fp32 reduce in
// source order, requantize at bits_out into the inter send layout (M units).
cudaError_t launch_tlq_dq_reduce_q(const uint8_t* intra_recv, size_t in_unit_bytes, int bits_in,
                                   int N, int M, size_t S, int G, uint8_t* inter_send,
                                   size_t out_unit_bytes, int bits_out, int grid_cap,
                                   cudaStream_t st);

// K5: Alg. 3 l.11-13 -- dequantize M received units, fp32 reduce in source order,
// inverse blockwise Hadamard, scale by kappa, write the fp32 shard.
cudaError_t launch_tlq_dq_reduce_had(const uint8_t* inter_recv, size_t in_unit_bytes, int bits_in,
                                     int M, size_t S, int G, int b, float kappa, float* out,
                                     int grid_cap, cudaStream_t st);

}  // namespace sdp4
