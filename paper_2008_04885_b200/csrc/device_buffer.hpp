// RAII device allocation used by the host engine.
#pragma once

#include <cstddef>
#include <utility>

#include <cuda_runtime.h>

#include "errors.hpp"

namespace mtg {

template <typename T>
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(size_t n) { resize(n); }
  ~DeviceBuffer() { release(); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), n_(o.n_), cap_(o.cap_) {
    o.p_ = nullptr;
    o.n_ = o.cap_ = 0;
  }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_;
      n_ = o.n_;
      cap_ = o.cap_;
      o.p_ = nullptr;
      o.n_ = o.cap_ = 0;
    }
    return *this;
  }

  // Logical size n. Reallocates (zero-filled) only when n exceeds the
  // allocation; shrinking keeps it, so the engine's workspace can follow the
  // batch shape without cudaFree / cudaMalloc round trips. Contents are kept.
  void resize(size_t n) {
    if (p_ && n <= cap_) {
      n_ = n;
      return;
    }
    release();
    if (n) {
      MTG_CUDA(cudaMalloc(&p_, n * sizeof(T)));
      // cudaMemset runs on the legacy default stream, which is not ordered
      // with the engine's non-blocking stream: finish it before returning so
      // it cannot land after later writes.
      MTG_CUDA(cudaMemset(p_, 0, n * sizeof(T)));
      MTG_CUDA(cudaDeviceSynchronize());
    }
    n_ = cap_ = n;
  }
  void release() {
    if (p_) cudaFree(p_);
    p_ = nullptr;
    n_ = cap_ = 0;
  }
  void upload(const T* host, size_t n, size_t offset = 0) {
    MTG_CUDA(cudaMemcpy(p_ + offset, host, n * sizeof(T), cudaMemcpyHostToDevice));
  }
  void download(T* host, size_t n, size_t offset = 0) const {
    MTG_CUDA(cudaMemcpy(host, p_ + offset, n * sizeof(T), cudaMemcpyDeviceToHost));
  }

  // Stream-ordered copies (the engine's stream is non-blocking, so plain
  // cudaMemcpy would not be ordered with its kernels).
  void upload(const T* host, size_t n, cudaStream_t st, size_t offset = 0) {
    if (n) MTG_CUDA(cudaMemcpyAsync(p_ + offset, host, n * sizeof(T), cudaMemcpyHostToDevice, st));
  }
  void download(T* host, size_t n, cudaStream_t st, size_t offset = 0) const {
    if (!n) return;
    MTG_CUDA(cudaMemcpyAsync(host, p_ + offset, n * sizeof(T), cudaMemcpyDeviceToHost, st));
    MTG_CUDA(cudaStreamSynchronize(st));
  }

  T* get() const { return p_; }
  size_t size() const { return n_; }
  size_t bytes() const { return n_ * sizeof(T); }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
  size_t cap_ = 0;
};

}  // namespace mtg
