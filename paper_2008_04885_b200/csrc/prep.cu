#include "prep.cuh"

#include <cstdint>

#include "errors.hpp"
#include "launch.cuh"

namespace mtg {

namespace {

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// quant.cpp:113-118: scale = 127/max_abs (1 when all zero);
// q = clamp(round_half_away(x*scale), -127, 127).
__device__ __forceinline__ int8_t quant1(float x, float scale) {
  float v = roundf(x * scale);
  v = fminf(127.0f, fmaxf(-127.0f, v));
  return static_cast<int8_t>(v);
}

__device__ __forceinline__ float scale_of(float max_abs) {
  return max_abs == 0.0f ? 1.0f : 127.0f / max_abs;
}

// One CTA per segment: block max-abs, then quantize every row of it.
__global__ void quantize_segments_kernel(const float* __restrict__ x, long long ld_x,
                                         int k, const int* __restrict__ seg_off,
                                         int n_seg, const int* d_n_seg,
                                         int8_t* __restrict__ q, int k_pad,
                                         float* __restrict__ row_scale, int* nonfinite) {
  pdl_wait();
  pdl_trigger();
  const int s = blockIdx.x;
  const int ns = d_n_seg ? *d_n_seg : n_seg;
  if (s >= ns) return;
  const int r0 = seg_off[s], r1 = seg_off[s + 1];
  __shared__ float red[32];
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  float m = 0.0f;
  int local_bad = 0;
  for (int r = r0; r < r1; ++r)
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
      const float v = x[r * ld_x + c];
      if (!isfinite(v)) local_bad = 1;
      m = fmaxf(m, fabsf(v));
    }
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (local_bad) bad = 1;
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0f;
    v = warp_max(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  if (bad && threadIdx.x == 0) atomicExch(nonfinite, 1);
  const float scale = scale_of(red[0]);
  for (int r = r0; r < r1; ++r) {
    for (int c = threadIdx.x; c < k_pad; c += blockDim.x)
      q[static_cast<long long>(r) * k_pad + c] = c < k ? quant1(x[r * ld_x + c], scale) : 0;
    if (threadIdx.x == 0) row_scale[r] = scale;
  }
}

// One warp per row.
__global__ void quantize_rows_kernel(const float* __restrict__ x, long long ld_x, int k,
                                     int max_rows, const int* d_rows,
                                     int8_t* __restrict__ q, int k_pad,
                                     float* __restrict__ row_scale, int* nonfinite) {
  pdl_wait();
  pdl_trigger();
  const int rows = d_rows ? *d_rows : max_rows;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float* xr = x + r * ld_x;
  float m = 0.0f;
  int bad = 0;
  for (int c = lane; c < k; c += 32) {
    const float v = xr[c];
    if (!isfinite(v)) bad = 1;
    m = fmaxf(m, fabsf(v));
  }
  m = warp_max(m);
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicExch(nonfinite, 1);
  const float scale = scale_of(m);
  int8_t* qr = q + static_cast<long long>(r) * k_pad;
  for (int c = lane; c < k_pad; c += 32) qr[c] = c < k ? quant1(xr[c], scale) : 0;
  if (lane == 0) row_scale[r] = scale;
}

// Register-resident variant with float4 loads (k % 4 == 0, k <= 128 * V4,
// 16-byte aligned rows): lane owns elements 4 lane + 128 i, quantizes them
// into one 32-bit store (the FFN-down operand at batch 64: 2048 values).
template <int V4>
__global__ void quantize_rows_vec_kernel(const float* __restrict__ x, long long ld_x, int k,
                                         int max_rows, const int* d_rows,
                                         int8_t* __restrict__ q, int k_pad,
                                         float* __restrict__ row_scale, int* nonfinite) {
  pdl_wait();
  pdl_trigger();
  const int rows = d_rows ? *d_rows : max_rows;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float* xr = x + r * ld_x;
  float4 v[V4];
#pragma unroll
  for (int i = 0; i < V4; ++i) {
    const int c = 4 * lane + 128 * i;
    v[i] = c < k ? *reinterpret_cast<const float4*>(xr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float m = 0.0f;
  int bad = 0;
#pragma unroll
  for (int i = 0; i < V4; ++i) {
    bad |= !isfinite(v[i].x) | !isfinite(v[i].y) | !isfinite(v[i].z) | !isfinite(v[i].w);
    m = fmaxf(fmaxf(m, fmaxf(fabsf(v[i].x), fabsf(v[i].y))), fmaxf(fabsf(v[i].z), fabsf(v[i].w)));
  }
  m = warp_max(m);
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicExch(nonfinite, 1);
  const float scale = scale_of(m);
  int8_t* qr = q + static_cast<long long>(r) * k_pad;
#pragma unroll
  for (int i = 0; i < V4; ++i) {
    const int c = 4 * lane + 128 * i;
    if (c < k_pad) {
      const uint32_t w = static_cast<uint32_t>(static_cast<uint8_t>(quant1(v[i].x, scale))) |
                         (static_cast<uint32_t>(static_cast<uint8_t>(quant1(v[i].y, scale))) << 8) |
                         (static_cast<uint32_t>(static_cast<uint8_t>(quant1(v[i].z, scale))) << 16) |
                         (static_cast<uint32_t>(static_cast<uint8_t>(quant1(v[i].w, scale))) << 24);
      *reinterpret_cast<uint32_t*>(qr + c) = w;  // columns >= k hold 0 (quantized zeros)
    }
  }
  for (int c = 128 * V4 + 4 * lane; c < k_pad; c += 128) *reinterpret_cast<uint32_t*>(qr + c) = 0u;
  if (lane == 0) row_scale[r] = scale;
}

// Register-resident variant (k <= 32*KPL): the row is read once.
template <int KPL>
__global__ void quantize_rows_reg_kernel(const float* __restrict__ x, long long ld_x, int k,
                                         int max_rows, const int* d_rows,
                                         int8_t* __restrict__ q, int k_pad,
                                         float* __restrict__ row_scale, int* nonfinite) {
  pdl_wait();
  pdl_trigger();
  const int rows = d_rows ? *d_rows : max_rows;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float* xr = x + r * ld_x;
  float v[KPL];
#pragma unroll
  for (int i = 0; i < KPL; ++i) v[i] = lane + 32 * i < k ? xr[lane + 32 * i] : 0.0f;
  float m = 0.0f;
  int bad = 0;
#pragma unroll
  for (int i = 0; i < KPL; ++i) {
    bad |= !isfinite(v[i]);
    m = fmaxf(m, fabsf(v[i]));
  }
  m = warp_max(m);
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicExch(nonfinite, 1);
  const float scale = scale_of(m);
  int8_t* qr = q + static_cast<long long>(r) * k_pad;
#pragma unroll
  for (int i = 0; i < KPL; ++i) {
    const int c = lane + 32 * i;
    if (c < k_pad) qr[c] = c < k ? quant1(v[i], scale) : 0;
  }
  for (int c = 32 * KPL + lane; c < k_pad; c += 32) qr[c] = 0;
  if (lane == 0) row_scale[r] = scale;
}

__global__ void cast_bf16_kernel(const float* __restrict__ x, long long ld_x, int k,
                                 int max_rows, const int* d_rows,
                                 __nv_bfloat16* __restrict__ out, int k_pad) {
  pdl_wait();
  pdl_trigger();
  const int rows = d_rows ? *d_rows : max_rows;
  const int r = blockIdx.y;
  if (r >= rows) return;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < k_pad; c += gridDim.x * blockDim.x)
    out[static_cast<long long>(r) * k_pad + c] =
        __float2bfloat16_rn(c < k ? x[r * ld_x + c] : 0.0f);
}

__global__ void split_tf32_kernel(const float* __restrict__ x, long long ld_x, int k,
                                  int max_rows, const int* d_rows, float* __restrict__ hi,
                                  float* __restrict__ lo, int k_pad) {
  pdl_wait();
  pdl_trigger();
  const int rows = d_rows ? *d_rows : max_rows;
  const int r = blockIdx.y;
  if (r >= rows) return;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < k_pad;
       c += gridDim.x * blockDim.x) {
    const float v = c < k ? x[r * ld_x + c] : 0.0f;
    if (!lo) {  // plain fp32 operand (the GEMM splits it)
      hi[static_cast<long long>(r) * k_pad + c] = v;
      continue;
    }
    uint32_t h;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(v));
    const float hf = __uint_as_float(h);
    hi[static_cast<long long>(r) * k_pad + c] = hf;
    lo[static_cast<long long>(r) * k_pad + c] = v - hf;
  }
}

__global__ void fill_kernel(float* __restrict__ p, long long n, float value) {
  pdl_wait();
  pdl_trigger();
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    p[i] = value;
}

}  // namespace

void launch_fill(float* p, long long n, float value, cudaStream_t st) {
  if (n <= 0) return;
  launch_k(fill_kernel, 1184, 256, 0, st, p, n, value);
  MTG_CUDA(cudaGetLastError());
}

void launch_quantize_segments(const float* x, long long ld_x, int k, const int* seg_off,
                              int n_seg, const int* d_n_seg, int8_t* q, int k_pad,
                              float* row_scale, int* nonfinite_flag, cudaStream_t st) {
  if (n_seg <= 0) return;
  launch_k(quantize_segments_kernel, n_seg, 256, 0, st, x, ld_x, k, seg_off, n_seg, d_n_seg, q,
                                                  k_pad, row_scale, nonfinite_flag);
  MTG_CUDA(cudaGetLastError());
}

void launch_quantize_rows(const float* x, long long ld_x, int k, int max_rows,
                          const int* d_rows, int8_t* q, int k_pad, float* row_scale,
                          int* nonfinite_flag, cudaStream_t st) {
  if (max_rows <= 0) return;
  const int wpb = 8;
  const dim3 grid((max_rows + wpb - 1) / wpb), block(wpb * 32);
  const int kpl = (k + 31) / 32;
  const bool vec = k % 4 == 0 && ld_x % 4 == 0 && k_pad % 4 == 0 &&
                   reinterpret_cast<uintptr_t>(x) % 16 == 0 && reinterpret_cast<uintptr_t>(q) % 4 == 0;
  if (vec && k <= 512) {
    const dim3 g4((max_rows + 3) / 4), b4(4 * 32);  // more, smaller CTAs
    launch_k(quantize_rows_vec_kernel<4>, g4, b4, 0, st, x, ld_x, k, max_rows, d_rows, q, k_pad,
             row_scale, nonfinite_flag);
  } else if (vec && k <= 2048) {
    const dim3 g4((max_rows + 3) / 4), b4(4 * 32);
    launch_k(quantize_rows_vec_kernel<16>, g4, b4, 0, st, x, ld_x, k, max_rows, d_rows, q, k_pad,
             row_scale, nonfinite_flag);
  } else if (kpl <= 16)
    launch_k(quantize_rows_reg_kernel<16>, grid, block, 0, st, x, ld_x, k, max_rows, d_rows, q, k_pad,
                                                         row_scale, nonfinite_flag);
  else if (kpl <= 64)
    launch_k(quantize_rows_reg_kernel<64>, grid, block, 0, st, x, ld_x, k, max_rows, d_rows, q, k_pad,
                                                         row_scale, nonfinite_flag);
  else
    launch_k(quantize_rows_kernel, grid, block, 0, st, x, ld_x, k, max_rows, d_rows, q, k_pad,
                                                 row_scale, nonfinite_flag);
  MTG_CUDA(cudaGetLastError());
}

void launch_cast_bf16(const float* x, long long ld_x, int k, int max_rows,
                      const int* d_rows, __nv_bfloat16* out, int k_pad, cudaStream_t st) {
  if (max_rows <= 0) return;
  dim3 grid((k_pad + 255) / 256, max_rows);
  launch_k(cast_bf16_kernel, grid, 256, 0, st, x, ld_x, k, max_rows, d_rows, out, k_pad);
  MTG_CUDA(cudaGetLastError());
}

void launch_split_tf32(const float* x, long long ld_x, int k, int max_rows,
                       const int* d_rows, float* hi, float* lo, int k_pad,
                       cudaStream_t st) {
  if (max_rows <= 0) return;
  dim3 grid((k_pad + 255) / 256, max_rows);
  launch_k(split_tf32_kernel, grid, 256, 0, st, x, ld_x, k, max_rows, d_rows, hi, lo, k_pad);
  MTG_CUDA(cudaGetLastError());
}

}  // namespace mtg
