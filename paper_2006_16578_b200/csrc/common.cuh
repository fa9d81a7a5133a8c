// common.cuh — error plumbing and device-buffer helpers for libbtnn_cuda.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <utility>

#include "btnn_cuda.h"

namespace btnn_gpu {

// Carries one of the C-ABI status codes; the C entry points catch it and return the code,
// the C++ adapter maps the code back to the reference's exception types
// (common.hpp:14-32).
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }
inline void require(bool ok, int code, const std::string& msg) {
  if (!ok) fail(code, msg);
}

#define BT_CUDA(x)                                                                            \
  do {                                                                                        \
    cudaError_t e_ = (x);                                                                     \
    if (e_ != cudaSuccess)                                                                    \
      ::btnn_gpu::fail(BTNN_CUDA_ERROR, std::string(#x) + ": " + cudaGetErrorString(e_));    \
  } while (0)

// Owning device allocation (bytes). Move-only.
class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(size_t bytes) { alloc(bytes); }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(std::exchange(o.p_, nullptr)), n_(std::exchange(o.n_, 0)) {}
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p_ = std::exchange(o.p_, nullptr);
      n_ = std::exchange(o.n_, 0);
    }
    return *this;
  }
  void alloc(size_t bytes) {
    release();
    if (bytes == 0) return;
    BT_CUDA(cudaMalloc(&p_, bytes));
    n_ = bytes;
  }
  void release() {
    if (p_) cudaFree(p_);
    p_ = nullptr;
    n_ = 0;
  }
  template <class T = void>
  T* get() const {
    return static_cast<T*>(p_);
  }
  size_t bytes() const { return n_; }

 private:
  void* p_ = nullptr;
  size_t n_ = 0;
};

// Timing experiments (per-role clock64 stamps, work-skipping switches, geometry overrides)
// exist only in builds made with -DBTNN_TIMING=1 (make TIMING=1). The product build
// compiles them out, so the kernels carry no debug branches and read no environment knobs.
#ifndef BTNN_TIMING
#define BTNN_TIMING 0
#endif
inline int timing_knob(const char* name, int dflt) {
  if (!BTNN_TIMING) return dflt;
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

// Launch with programmatic stream serialization (the kernel calls grid_dep_wait before it
// touches data of earlier kernels): its prologue (barrier init, TMEM allocation, tables,
// static weights) overlaps the previous kernel's tail; in a captured graph the dependency
// becomes a programmatic edge.
template <class... KArgs, class... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  BT_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

template <class T>
DevBuf upload(const T* host, size_t count, cudaStream_t st) {
  DevBuf b(count * sizeof(T));
  if (count) BT_CUDA(cudaMemcpyAsync(b.get(), host, count * sizeof(T), cudaMemcpyHostToDevice, st));
  return b;
}

}  // namespace btnn_gpu
