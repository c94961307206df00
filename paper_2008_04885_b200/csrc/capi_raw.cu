// Raw operator entry points of the C ABI: the reference's quantization and
// GEMM kernels (quant.hpp:45-68, tensor.hpp:150-154) executed on the B200
// tensor cores with host buffers in and out. Used by the parity tests that
// mirror proj/tests/test_quant.cpp and test_tensor.cpp.
#include <cstdint>
#include <string>
#include <vector>

#include <cuda_bf16.h>

#include "../../include/minimt_gpu.h"
#include "capi_util.hpp"
#include "device_buffer.hpp"
#include "gemm.hpp"
#include "prep.cuh"

namespace mtg {

std::string& last_error_slot() {
  thread_local std::string s;
  return s;
}

namespace {

constexpr int kMaxInner = 65536;  // quant.cpp:16

int to_gemm_prec(int p) {
  switch (p) {
    case MTG_PREC_F32: return kPrecTF32x3;
    case MTG_PREC_BF16: return kPrecBF16;
    case MTG_PREC_INT8: return kPrecI8;
  }
  fail(kUsageError, "unknown precision " + std::to_string(p));
}

// Runs C = A.B^T on device where both operands arrive as int8 K-major host
// matrices; row/col scales are uniform (one per tensor).
void run_i8(const std::vector<int8_t>& a_kmaj, float sa, const std::vector<int8_t>& b_kmaj,
            float sb, int m, int k, int n, float* c_host) {
  const int kp = pad_k(k, kPrecI8);
  const int ldc = (n + 3) / 4 * 4;
  DeviceBuffer<int8_t> da(static_cast<size_t>(std::max(m, 1)) * kp),
      db(static_cast<size_t>(std::max(n, 1)) * kp);
  std::vector<int8_t> pa(static_cast<size_t>(std::max(m, 1)) * kp, 0),
      pb(static_cast<size_t>(std::max(n, 1)) * kp, 0);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < k; ++j) pa[size_t(i) * kp + j] = a_kmaj[size_t(i) * k + j];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < k; ++j) pb[size_t(i) * kp + j] = b_kmaj[size_t(i) * k + j];
  da.upload(pa.data(), pa.size());
  db.upload(pb.data(), pb.size());
  DeviceBuffer<float> dsa(std::max(m, 1)), dsb(std::max(n, 1)),
      dc(static_cast<size_t>(std::max(m, 1)) * ldc);
  std::vector<float> hsa(std::max(m, 1), sa), hsb(std::max(n, 1), sb);
  dsa.upload(hsa.data(), hsa.size());
  dsb.upload(hsb.data(), hsb.size());
  Operand oa{da.get(), nullptr, std::max(m, 1), kp, kPrecI8};
  Operand ob{db.get(), nullptr, std::max(n, 1), kp, kPrecI8};
  GemmPlan plan = plan_gemm(oa, ob, m, n);
  GemmEpilogue ep{};
  ep.C = dc.get();
  ep.ldc = ldc;
  ep.a_scale = dsa.get();
  ep.w_seg_scale = dsb.get();  // one weight tensor: a single segment
  ep.seg_width = 0;
  ep.M = m;
  ep.N = n;
  launch_gemm(plan, ep, 0);
  MTG_CUDA(cudaDeviceSynchronize());
  std::vector<float> hc(static_cast<size_t>(std::max(m, 1)) * ldc);
  dc.download(hc.data(), hc.size());
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) c_host[size_t(i) * n + j] = hc[size_t(i) * ldc + j];
}

}  // namespace
}  // namespace mtg

using namespace mtg;

extern "C" {

const char* mtg_last_error(void) { return last_error_slot().c_str(); }

int mtg_abi_version(void) { return MTG_ABI_VERSION; }

int mtg_quantize(const float* x, int64_t n, int8_t* q_out, float* scale_out) {
  return guarded([&] {
    if (n < 0) fail(kShapeError, "quantize: negative size");
    if (n == 0) {
      *scale_out = 1.0f;
      return;
    }
    DeviceBuffer<float> dx(n), ds(1);
    DeviceBuffer<int8_t> dq(n);
    DeviceBuffer<int> off(2), bad(1);
    int h_off[2] = {0, 1};
    off.upload(h_off, 2);
    dx.upload(x, n);
    launch_quantize_segments(dx.get(), n, static_cast<int>(n), off.get(), 1, nullptr,
                             dq.get(), static_cast<int>(n), ds.get(), bad.get(), 0);
    MTG_CUDA(cudaDeviceSynchronize());
    int h_bad = 0;
    bad.download(&h_bad, 1);
    if (h_bad) fail(kValueError, "quantize: non-finite values in tensor");
    dq.download(q_out, n);
    ds.download(scale_out, 1);
  });
}

int mtg_qmatmul(const int8_t* a, float a_scale, const int8_t* b, float b_scale, int m,
                int k, int n, float* c) {
  return guarded([&] {
    if (m < 0 || k < 0 || n < 0) fail(kShapeError, "qmatmul: negative dimension");
    if (k > kMaxInner) fail(kValueError, "qmatmul: inner dimension above 65536");
    if (m == 0 || n == 0) return;
    std::vector<int8_t> av(a, a + size_t(m) * k), bt(size_t(n) * k);
    for (int kk = 0; kk < k; ++kk)
      for (int j = 0; j < n; ++j) bt[size_t(j) * k + kk] = b[size_t(kk) * n + j];
    run_i8(av, a_scale, bt, b_scale, m, k, n, c);
  });
}

int mtg_qmatmul_nt(const int8_t* a, float a_scale, const int8_t* b, float b_scale, int m,
                   int k, int b_rows, const int32_t* row_subset, int n_subset, float* c) {
  return guarded([&] {
    if (m < 0 || k < 0 || b_rows < 0) fail(kShapeError, "qmatmul_nt: negative dimension");
    if (k > kMaxInner) fail(kValueError, "qmatmul_nt: inner dimension above 65536");
    const int n = row_subset ? n_subset : b_rows;
    std::vector<int8_t> bt(size_t(std::max(n, 0)) * k);
    for (int j = 0; j < n; ++j) {
      const int r = row_subset ? row_subset[j] : j;
      if (r < 0 || r >= b_rows) fail(kIndexError, "qmatmul_nt: row out of range");
      for (int kk = 0; kk < k; ++kk) bt[size_t(j) * k + kk] = b[size_t(r) * k + kk];
    }
    if (m == 0 || n == 0) return;
    std::vector<int8_t> av(a, a + size_t(m) * k);
    run_i8(av, a_scale, bt, b_scale, m, k, n, c);
  });
}

int mtg_gemm(int precision, const float* a, const float* b, int m, int k, int n,
             float* c) {
  return guarded([&] {
    if (m < 0 || k < 0 || n < 0) fail(kShapeError, "gemm: negative dimension");
    const int prec = to_gemm_prec(precision);
    if (prec == kPrecI8) fail(kUsageError, "gemm: use mtg_qmatmul for int8");
    if (m == 0 || n == 0) return;
    const int kp = pad_k(k, prec);
    const int ldc = (n + 3) / 4 * 4;
    // B^T (K-major) on host, then device-side operand conversion.
    std::vector<float> bt(size_t(n) * k);
    for (int kk = 0; kk < k; ++kk)
      for (int j = 0; j < n; ++j) bt[size_t(j) * k + kk] = b[size_t(kk) * n + j];
    DeviceBuffer<float> da32(size_t(m) * std::max(k, 1)), db32(size_t(n) * std::max(k, 1));
    if (k) {
      da32.upload(a, size_t(m) * k);
      db32.upload(bt.data(), bt.size());
    }
    DeviceBuffer<float> dc(size_t(m) * ldc);
    Operand oa, ob;
    DeviceBuffer<__nv_bfloat16> a16, b16;
    DeviceBuffer<float> ahi, alo, bhi, blo;
    if (prec == kPrecBF16) {
      a16.resize(size_t(m) * kp);
      b16.resize(size_t(n) * kp);
      launch_cast_bf16(da32.get(), k, k, m, nullptr, a16.get(), kp, 0);
      launch_cast_bf16(db32.get(), k, k, n, nullptr, b16.get(), kp, 0);
      oa = Operand{a16.get(), nullptr, m, kp, prec};
      ob = Operand{b16.get(), nullptr, n, kp, prec};
    } else {
      ahi.resize(size_t(m) * kp);
      alo.resize(size_t(m) * kp);
      bhi.resize(size_t(n) * kp);
      blo.resize(size_t(n) * kp);
      launch_split_tf32(da32.get(), k, k, m, nullptr, ahi.get(), alo.get(), kp, 0);
      launch_split_tf32(db32.get(), k, k, n, nullptr, bhi.get(), blo.get(), kp, 0);
      oa = Operand{ahi.get(), alo.get(), m, kp, prec};
      ob = Operand{bhi.get(), blo.get(), n, kp, prec};
    }
    GemmPlan plan = plan_gemm(oa, ob, m, n);
    GemmEpilogue ep{};
    ep.C = dc.get();
    ep.ldc = ldc;
    ep.M = m;
    ep.N = n;
    launch_gemm(plan, ep, 0);
    MTG_CUDA(cudaDeviceSynchronize());
    std::vector<float> hc(size_t(m) * ldc);
    dc.download(hc.data(), hc.size());
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < n; ++j) c[size_t(i) * n + j] = hc[size_t(i) * ldc + j];
  });
}

}  // extern "C"
