// Shared helpers of the adaptgear_b200 C ABI: error plumbing, launch checks,
// stream-ordered scratch memory.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>

#include "adaptgear_b200.h"

namespace ag {

// Thread-local last error; ag_last_error() returns it.
std::string &last_error();

inline int fail(int code, const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  last_error() = buf;
  return code;
}

inline int cuda_status(cudaError_t e, const char *where) {
  if (e == cudaSuccess) return AG_OK;
  return fail(AG_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

// A failed runtime call also records itself as the thread's last error;
// clear it (non-sticky errors) so the next launch check does not report it.
#define AG_CUDA(expr)                                        \
  do {                                                       \
    cudaError_t _e = (expr);                                 \
    if (_e != cudaSuccess) {                                 \
      (void)cudaGetLastError();                              \
      return ag::cuda_status(_e, #expr);                     \
    }                                                        \
  } while (0)

// Every kernel launch of the library goes through this check, which also
// counts it (ag_launch_count(): the bench reports how many of OUR kernels ran).
#define AG_LAUNCH_CHECK(name)                                     \
  do {                                                            \
    ag::count_launch();                                           \
    cudaError_t _e = cudaGetLastError();                          \
    if (_e != cudaSuccess) return ag::cuda_status(_e, name);      \
  } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Stream-ordered scratch buffer (cudaMallocAsync pool); freed on scope exit
// in stream order, so it never races the kernels that use it.
struct Scratch {
  void *ptr = nullptr;
  cudaStream_t stream = nullptr;
  Scratch() = default;
  Scratch(const Scratch &) = delete;
  Scratch &operator=(const Scratch &) = delete;
  cudaError_t alloc(size_t bytes, cudaStream_t s) {
    stream = s;
    if (bytes == 0) bytes = 16;
    return cudaMallocAsync(&ptr, bytes, s);
  }
  template <class T>
  T *as() const { return static_cast<T *>(ptr); }
  ~Scratch() {
    if (ptr) cudaFreeAsync(ptr, stream);
  }
};

inline int grid_for(int64_t n, int block, int64_t cap = 148LL * 64) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<int>(g);
}

int sm_count();
void count_launch();

// Bit-packed ReLU masks (AG_RELU_BITS layout, include/adaptgear_b200.h): row r
// of a [rows][feat] activation is ldw = ceil(feat / 32) uint32 words; bit
// (c % 32) of word c / 32 is (h[r][c] > 0).  1/32 of the fp32 bytes.
__host__ __device__ inline int64_t relu_words(int64_t feat) { return (feat + 31) / 32; }
__device__ __forceinline__ bool relu_bit(const uint32_t *bits, int64_t ldw, int64_t r,
                                         int64_t c) {
  return (__ldg(bits + r * ldw + (c >> 5)) >> (c & 31)) & 1u;
}

}  // namespace ag
