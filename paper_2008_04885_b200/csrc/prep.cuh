// Operand preparation: fp32 activations -> the GEMM operand format of the
// active precision. int8 follows the reference's per-call-tensor max-abs
// quantization (quant.cpp:108-122) with one scale per *segment* (the tensor the
// reference's Executor::linear would have received: one sentence in the
// encoder, one hypothesis row in the decoder).
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace mtg {

// Rows [seg_off[s], seg_off[s+1]) of x form segment s; rows are x[r*ld_x ..
// + k). Writes q[r*k_pad + c] (zero pad for c >= k) and row_scale[r] = scale of
// r's segment. nonfinite_flag is set to 1 if any input is NaN/Inf (the
// reference throws ValueError, tensor.cpp:69-72).
void launch_quantize_segments(const float* x, long long ld_x, int k, const int* seg_off,
                              int n_seg, const int* d_n_seg, int8_t* q, int k_pad,
                              float* row_scale, int* nonfinite_flag, cudaStream_t st);

// One segment per row, rows counted on device (*d_rows).
void launch_quantize_rows(const float* x, long long ld_x, int k, int max_rows,
                          const int* d_rows, int8_t* q, int k_pad, float* row_scale,
                          int* nonfinite_flag, cudaStream_t st);

void launch_cast_bf16(const float* x, long long ld_x, int k, int max_rows,
                      const int* d_rows, __nv_bfloat16* out, int k_pad, cudaStream_t st);

// p[0..n) = value.
void launch_fill(float* p, long long n, float value, cudaStream_t st);

// hi = tf32(x) (round to nearest), lo = x - hi.
void launch_split_tf32(const float* x, long long ld_x, int k, int max_rows,
                       const int* d_rows, float* hi, float* lo, int k_pad,
                       cudaStream_t st);

}  // namespace mtg
