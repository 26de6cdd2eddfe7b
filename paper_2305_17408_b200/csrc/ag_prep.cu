// Device preprocessing of the AdaptGear path:
//   ag_canonicalize    Graph.from_edges      graph.py:47-82
//   ag_relabel         apply_reorder         reorder.py:217-228
//   ag_gcn_normalize   gcn_normalize         models.py:57-73
//   ag_in_degrees      Graph.in_degrees      graph.py:94-96
//   ag_decompose_*     decompose             decompose.py:57-75
//   ag_build_row_ptr   to_csr                formats.py:76-88
//   ag_blocks_*        to_dense_blocks       formats.py:105-140
// plus the seeded synthetic generator.
// All integer outputs are bit-exact with the reference; the only floating
// point here is the fp64 duplicate-weight sum (input order, like np.add.at)
// and the fp64 GCN weight 1/sqrt(d_i*d_j) rounded once to fp32.
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>
#include <string>

#include "ag_common.cuh"

namespace ag {

std::string &last_error() {
  static thread_local std::string msg;
  return msg;
}

static std::atomic<unsigned long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int sm_count() {
  static int cached = -1;
  static std::mutex mu;
  std::lock_guard<std::mutex> g(mu);
  if (cached < 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
      cudaGetLastError();
      cached = 148;
    }
  }
  return cached;
}

namespace {

constexpr int kThreads = 256;

inline int bits_for(uint64_t max_value) {
  int b = 0;
  while (b < 64 && (max_value >> b) != 0) ++b;
  return b < 1 ? 1 : b;
}

__global__ void minmax_kernel(int64_t n, const int64_t *a, const int64_t *b,
                              unsigned long long *lo_bits, long long *hi) {
  // lo tracked through an order-preserving unsigned mapping (handles negatives)
  long long mn = LLONG_MAX, mx = LLONG_MIN;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    long long x = a[i], y = b[i];
    mn = min(mn, min(x, y));
    mx = max(mx, max(x, y));
  }
  typedef cub::BlockReduce<long long, kThreads> BR;
  __shared__ typename BR::TempStorage t1;
  __shared__ typename BR::TempStorage t2;
  long long bmn = BR(t1).Reduce(mn, cub::Min());
  long long bmx = BR(t2).Reduce(mx, cub::Max());
  if (threadIdx.x == 0) {
    atomicMin(lo_bits, static_cast<unsigned long long>(bmn) ^ 0x8000000000000000ULL);
    atomicMax(hi, bmx);
  }
}

__global__ void make_keys_kernel(int64_t n, int64_t V, const int64_t *dst, const int64_t *src,
                                 uint64_t *keys, int32_t *idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = static_cast<uint64_t>(dst[i]) * static_cast<uint64_t>(V) + static_cast<uint64_t>(src[i]);
    if (idx) idx[i] = static_cast<int32_t>(i);
  }
}

__global__ void head_flags_kernel(int64_t n, const uint64_t *keys, int32_t *flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

__global__ void emit_unique_kernel(int64_t n, int64_t V, const uint64_t *keys,
                                   const int32_t *flags, const int32_t *pos, int32_t *dst_out,
                                   int32_t *src_out, int32_t *seg_start) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (flags[i]) {
      const int32_t u = pos[i];
      const uint64_t k = keys[i];
      dst_out[u] = static_cast<int32_t>(k / static_cast<uint64_t>(V));
      src_out[u] = static_cast<int32_t>(k % static_cast<uint64_t>(V));
      if (seg_start) seg_start[u] = static_cast<int32_t>(i);
    }
  }
}

// np.add.at(merged, inverse, w.astype(f64)) then .astype(f32): duplicates are
// accumulated in fp64 in input order (the radix sort is stable).
__global__ void merge_weights_kernel(int64_t nu, int64_t n, const int32_t *seg_start,
                                     const int32_t *idx, const float *w, float *w_out) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < nu;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = seg_start[u];
    const int64_t b = (u + 1 < nu) ? seg_start[u + 1] : n;
    double s = 0.0;
    for (int64_t i = a; i < b; ++i) s = __dadd_rn(s, static_cast<double>(w[idx[i]]));
    w_out[u] = __double2float_rn(s);
  }
}

// Sort keys (+ optional payload idx), drop duplicates, emit (dst, src) and the
// start of each run; returns the unique count through *nu_host.
int sort_unique(int64_t V, int64_t n, uint64_t *keys, int32_t *idx, int32_t *dst_out,
                int32_t *src_out, int32_t *seg_start_out, int32_t **idx_sorted_out,
                Scratch &keep_idx, int64_t *nu_host, cudaStream_t st) {
  const int end_bit = bits_for(static_cast<uint64_t>(V) * static_cast<uint64_t>(V) - 1);
  Scratch keys2, idx2, tmp, flags, pos;
  AG_CUDA(keys2.alloc(n * sizeof(uint64_t), st));
  size_t tmp_bytes = 0;
  if (idx) {
    AG_CUDA(idx2.alloc(n * sizeof(int32_t), st));
    AG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys2.as<uint64_t>(), idx,
                                            idx2.as<int32_t>(), (int)n, 0, end_bit, st));
    AG_CUDA(tmp.alloc(tmp_bytes, st));
    AG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.ptr, tmp_bytes, keys, keys2.as<uint64_t>(), idx,
                                            idx2.as<int32_t>(), (int)n, 0, end_bit, st));
  } else {
    AG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, keys, keys2.as<uint64_t>(), (int)n,
                                           0, end_bit, st));
    AG_CUDA(tmp.alloc(tmp_bytes, st));
    AG_CUDA(cub::DeviceRadixSort::SortKeys(tmp.ptr, tmp_bytes, keys, keys2.as<uint64_t>(), (int)n,
                                           0, end_bit, st));
  }
  AG_CUDA(flags.alloc(n * sizeof(int32_t), st));
  AG_CUDA(pos.alloc(n * sizeof(int32_t), st));
  const uint64_t *sk = keys2.as<uint64_t>();
  head_flags_kernel<<<grid_for(n, kThreads), kThreads, 0, st>>>(n, sk, flags.as<int32_t>());
  AG_LAUNCH_CHECK("head_flags_kernel");
  Scratch tmp2;
  size_t scan_bytes = 0;
  AG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, flags.as<int32_t>(),
                                        pos.as<int32_t>(), (int)n, st));
  AG_CUDA(tmp2.alloc(scan_bytes, st));
  AG_CUDA(cub::DeviceScan::ExclusiveSum(tmp2.ptr, scan_bytes, flags.as<int32_t>(),
                                        pos.as<int32_t>(), (int)n, st));
  emit_unique_kernel<<<grid_for(n, kThreads), kThreads, 0, st>>>(
      n, V, sk, flags.as<int32_t>(), pos.as<int32_t>(), dst_out, src_out, seg_start_out);
  AG_LAUNCH_CHECK("emit_unique_kernel");
  int32_t last_pos = 0, last_flag = 0;
  AG_CUDA(cudaMemcpyAsync(&last_pos, pos.as<int32_t>() + n - 1, 4, cudaMemcpyDeviceToHost, st));
  AG_CUDA(cudaMemcpyAsync(&last_flag, flags.as<int32_t>() + n - 1, 4, cudaMemcpyDeviceToHost, st));
  AG_CUDA(cudaStreamSynchronize(st));
  *nu_host = static_cast<int64_t>(last_pos) + last_flag;
  if (idx_sorted_out) {
    // hand the sorted payload to the caller (keeps it alive past this scope)
    std::swap(keep_idx.ptr, idx2.ptr);
    std::swap(keep_idx.stream, idx2.stream);
    *idx_sorted_out = keep_idx.as<int32_t>();
  }
  return AG_OK;
}

__global__ void relabel_kernel(int64_t n, const int64_t *perm, const int32_t *dst,
                               const int32_t *src, int64_t *dst_out, int64_t *src_out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    dst_out[i] = perm[dst[i]];
    src_out[i] = perm[src[i]];
  }
}

__global__ void keys_with_loops_kernel(int64_t E, int64_t V, const int32_t *dst,
                                       const int32_t *src, uint64_t *keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E + V;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t d, s;
    if (i < E) {
      d = static_cast<uint64_t>(dst[i]);
      s = static_cast<uint64_t>(src[i]);
    } else {
      d = s = static_cast<uint64_t>(i - E);
    }
    keys[i] = d * static_cast<uint64_t>(V) + s;
  }
}

__global__ void histogram_kernel(int64_t n, const int32_t *dst, unsigned long long *deg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(deg + dst[i], 1ULL);
}

// models.py:71-72: w = 1.0 / np.sqrt(deg[dst] * deg[src]) in fp64, -> fp32.
__global__ void gcn_weights_kernel(int64_t n, const int32_t *dst, const int32_t *src,
                                   const unsigned long long *deg, float *w) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double a = static_cast<double>(deg[dst[i]]);
    const double b = static_cast<double>(deg[src[i]]);
    w[i] = __double2float_rn(__ddiv_rn(1.0, __dsqrt_rn(__dmul_rn(a, b))));
  }
}

__global__ void count_intra_kernel(int64_t n, const int32_t *dst, const int32_t *src, int64_t B,
                                   unsigned long long *count) {
  int local = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    local += (dst[i] / B == src[i] / B) ? 1 : 0;
  typedef cub::BlockReduce<int, kThreads> BR;
  __shared__ typename BR::TempStorage t;
  int tot = BR(t).Sum(local);
  if (threadIdx.x == 0 && tot) atomicAdd(count, static_cast<unsigned long long>(tot));
}

__global__ void intra_flags_kernel(int64_t n, const int32_t *dst, const int32_t *src, int64_t B,
                                   int32_t *flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = (dst[i] / B == src[i] / B) ? 1 : 0;
}

__global__ void split_kernel(int64_t n, const int32_t *dst, const int32_t *src, const float *w,
                             const int32_t *flags, const int32_t *pos, int32_t *id, int32_t *is,
                             float *iw, int32_t *od, int32_t *os, float *ow) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (flags[i]) {
      const int64_t p = pos[i];
      id[p] = dst[i];
      is[p] = src[i];
      if (w) iw[p] = w[i];
    } else {
      const int64_t p = i - pos[i];
      od[p] = dst[i];
      os[p] = src[i];
      if (w) ow[p] = w[i];
    }
  }
}

// row_ptr from sorted dst: every boundary thread fills the gap it closes.
__global__ void row_ptr_kernel(int64_t V, int64_t E, const int32_t *dst, int32_t *row_ptr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= E;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = (i == 0) ? 0 : static_cast<int64_t>(dst[i - 1]) + 1;
    const int64_t hi = (i == E) ? V : static_cast<int64_t>(dst[i]);
    for (int64_t r = lo; r <= hi; ++r) row_ptr[r] = static_cast<int32_t>(i);
  }
}

__global__ void touched_kernel(int64_t rows, const int32_t *row_ptr, uint8_t *t) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x)
    t[r] = row_ptr[r + 1] > row_ptr[r] ? 1 : 0;
}

__global__ void off_block_kernel(int64_t rows, const int32_t *row_ptr, const int32_t *col,
                                 int64_t B, unsigned long long *first) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    for (int64_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
      if (r / B != col[e] / B) {
        atomicMin(first, static_cast<unsigned long long>(e));
        break;
      }
    }
  }
}

__global__ void block_heads_kernel(int64_t n, const int32_t *dst, int64_t B, int32_t *flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = (i == 0 || dst[i] / B != dst[i - 1] / B) ? 1 : 0;
}

__global__ void block_slots_kernel(int64_t n, const int32_t *dst, int64_t B, const int32_t *flags,
                                   const int32_t *pos, int32_t *community_ids,
                                   int32_t *comm_slot) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (flags[i]) {
      const int32_t c = static_cast<int32_t>(dst[i] / B);
      community_ids[pos[i]] = c;
      comm_slot[c] = pos[i];
    }
  }
}

__global__ void block_scatter_kernel(int64_t n, const int32_t *dst, const int32_t *src,
                                     const float *w, int64_t B, const int32_t *comm_slot,
                                     float *blocks, uint8_t *row_touched) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = dst[i] / B;
    const int64_t slot = comm_slot[c];
    const int64_t li = dst[i] - c * B, lj = src[i] - c * B;
    blocks[(slot * B + li) * B + lj] = w ? w[i] : 1.0f;
    row_touched[slot * B + li] = 1;
  }
}

__global__ void fill_i32_kernel(int64_t n, int32_t *p, int32_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// ------------------------------------------------------------ generator ----
__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__device__ inline double unit53(uint64_t h) {
  return __dmul_rn(static_cast<double>(h >> 11), 1.0 / 9007199254740992.0);
}

__device__ inline int64_t scaled(double u, int64_t n) {
  int64_t v = static_cast<int64_t>(floor(__dmul_rn(u, static_cast<double>(n))));
  return v >= n ? n - 1 : v;
}

struct SynthArgs {
  int64_t V, Bg, window, skew;
  double p_intra, p_global;
  uint64_t seedmix;
  int64_t first, count;
  int64_t *dst, *src;
};

__global__ void synth_kernel(SynthArgs a) {
  const int64_t nb = (a.V + a.Bg - 1) / a.Bg;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < a.count;
       t += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t i = static_cast<uint64_t>(a.first + t);
    double u[6];
    uint64_t h5 = 0;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const uint64_t h = mix64(a.seedmix ^ (i * 8ULL + k));
      u[k] = unit53(h);
      if (k == 5) h5 = h;
    }
    double p = u[0];
    for (int64_t j = 1; j < a.skew; ++j) p = __dmul_rn(p, u[0]);
    const int64_t d = scaled(p, a.V);
    const int64_t c = d / a.Bg;
    const int64_t base = c * a.Bg;
    const int64_t sz = min(a.Bg, a.V - base);
    int64_t s;
    if (u[1] < a.p_intra && sz > 1) {
      const int64_t tt = scaled(u[2], sz - 1);
      s = base + tt + (tt >= d - base ? 1 : 0);
    } else {
      int64_t cs;
      if (u[3] < a.p_global) {
        cs = scaled(u[4], nb);
      } else {
        const int64_t off = 1 + scaled(u[4], a.window);
        const int64_t sgn = (h5 & 1ULL) ? 1 : -1;
        cs = ((c + sgn * off) % nb + nb) % nb;
      }
      const int64_t bs = cs * a.Bg;
      const int64_t szs = min(a.Bg, a.V - bs);
      s = bs + scaled(u[2], szs);
      if (s == d) s = -1;
    }
    a.dst[t] = (s < 0) ? -1 : d;
    a.src[t] = s;
  }
}

__global__ void vertex_keys_kernel(int64_t V, uint64_t seedmix, uint64_t *keys) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x)
    keys[v] = mix64(seedmix ^ static_cast<uint64_t>(v));
}

}  // namespace
}  // namespace ag

using namespace ag;

extern "C" int ag_abi_version(void) { return 1; }
extern "C" uint64_t ag_launch_count(void) { return ag::g_launches.load(); }
extern "C" const char *ag_last_error(void) { return ag::last_error().c_str(); }
extern "C" int ag_device_sm_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return 0;
  }
  return ag::sm_count();
}

extern "C" int ag_canonicalize(int64_t V, int64_t E, const int64_t *dst, const int64_t *src,
                               const float *w, int32_t *dst_out, int32_t *src_out, float *w_out,
                               int64_t *num_out_host, void *stream) {
  *num_out_host = 0;
  if (V < 0 || V > 2147483647LL) return fail(AG_ERR_VALUE, "invalid vertex count %lld", (long long)V);
  if (E == 0) return AG_OK;
  if (E > 2147483647LL) return fail(AG_ERR_VALUE, "too many edges (%lld)", (long long)E);
  cudaStream_t st = as_stream(stream);
  Scratch mm;
  AG_CUDA(mm.alloc(16, st));
  unsigned long long init_lo = 0xFFFFFFFFFFFFFFFFULL;
  long long init_hi = LLONG_MIN;
  AG_CUDA(cudaMemcpyAsync(mm.as<unsigned long long>(), &init_lo, 8, cudaMemcpyHostToDevice, st));
  AG_CUDA(cudaMemcpyAsync(mm.as<long long>() + 1, &init_hi, 8, cudaMemcpyHostToDevice, st));
  minmax_kernel<<<grid_for(E, kThreads, 1024), kThreads, 0, st>>>(
      E, dst, src, mm.as<unsigned long long>(), mm.as<long long>() + 1);
  AG_LAUNCH_CHECK("minmax_kernel");
  unsigned long long lo_bits = 0;
  long long hi = 0;
  AG_CUDA(cudaMemcpyAsync(&lo_bits, mm.as<unsigned long long>(), 8, cudaMemcpyDeviceToHost, st));
  AG_CUDA(cudaMemcpyAsync(&hi, mm.as<long long>() + 1, 8, cudaMemcpyDeviceToHost, st));
  AG_CUDA(cudaStreamSynchronize(st));
  const long long lo = static_cast<long long>(lo_bits ^ 0x8000000000000000ULL);
  if (lo < 0 || hi >= V)
    return fail(AG_ERR_VALUE, "edge endpoint out of range [0, %lld): %lld", (long long)V,
                lo < 0 ? lo : hi);
  Scratch keys, idx, seg, keep;
  AG_CUDA(keys.alloc(E * sizeof(uint64_t), st));
  if (w) {
    AG_CUDA(idx.alloc(E * sizeof(int32_t), st));
    AG_CUDA(seg.alloc(E * sizeof(int32_t), st));
  }
  make_keys_kernel<<<grid_for(E, kThreads), kThreads, 0, st>>>(
      E, V, dst, src, keys.as<uint64_t>(), w ? idx.as<int32_t>() : nullptr);
  AG_LAUNCH_CHECK("make_keys_kernel");
  int32_t *idx_sorted = nullptr;
  int64_t nu = 0;
  if (int rc = sort_unique(V, E, keys.as<uint64_t>(), w ? idx.as<int32_t>() : nullptr, dst_out,
                           src_out, w ? seg.as<int32_t>() : nullptr, w ? &idx_sorted : nullptr,
                           keep, &nu, st))
    return rc;
  if (w) {
    merge_weights_kernel<<<grid_for(nu, kThreads), kThreads, 0, st>>>(
        nu, E, seg.as<int32_t>(), idx_sorted, w, w_out);
    AG_LAUNCH_CHECK("merge_weights_kernel");
  }
  *num_out_host = nu;
  return AG_OK;
}

extern "C" int ag_relabel(int64_t E, const int64_t *perm, const int32_t *dst, const int32_t *src,
                          int64_t *dst_out, int64_t *src_out, void *stream) {
  if (E == 0) return AG_OK;
  relabel_kernel<<<grid_for(E, kThreads), kThreads, 0, as_stream(stream)>>>(E, perm, dst, src,
                                                                            dst_out, src_out);
  AG_LAUNCH_CHECK("relabel_kernel");
  return AG_OK;
}

extern "C" int ag_gcn_normalize(int64_t V, int64_t E, const int32_t *dst, const int32_t *src,
                                int32_t *dst_out, int32_t *src_out, float *w_out,
                                int64_t *num_out_host, void *stream) {
  *num_out_host = 0;
  const int64_t n = E + V;
  if (n == 0) return AG_OK;
  if (n > 2147483647LL) return fail(AG_ERR_VALUE, "too many edges (%lld)", (long long)n);
  cudaStream_t st = as_stream(stream);
  Scratch keys, keep, deg;
  AG_CUDA(keys.alloc(n * sizeof(uint64_t), st));
  keys_with_loops_kernel<<<grid_for(n, kThreads), kThreads, 0, st>>>(E, V, dst, src,
                                                                     keys.as<uint64_t>());
  AG_LAUNCH_CHECK("keys_with_loops_kernel");
  int64_t nu = 0;
  if (int rc = sort_unique(V, n, keys.as<uint64_t>(), nullptr, dst_out, src_out, nullptr, nullptr,
                           keep, &nu, st))
    return rc;
  AG_CUDA(deg.alloc(V * sizeof(unsigned long long), st));
  AG_CUDA(cudaMemsetAsync(deg.ptr, 0, V * sizeof(unsigned long long), st));
  histogram_kernel<<<grid_for(nu, kThreads), kThreads, 0, st>>>(nu, dst_out,
                                                                deg.as<unsigned long long>());
  gcn_weights_kernel<<<grid_for(nu, kThreads), kThreads, 0, st>>>(
      nu, dst_out, src_out, deg.as<unsigned long long>(), w_out);
  AG_LAUNCH_CHECK("gcn_weights_kernel");
  *num_out_host = nu;
  return AG_OK;
}

extern "C" int ag_in_degrees(int64_t V, int64_t E, const int32_t *dst, int64_t *deg_out,
                             void *stream) {
  cudaStream_t st = as_stream(stream);
  if (V == 0) return AG_OK;
  AG_CUDA(cudaMemsetAsync(deg_out, 0, V * sizeof(int64_t), st));
  if (E == 0) return AG_OK;
  histogram_kernel<<<grid_for(E, kThreads), kThreads, 0, st>>>(
      E, dst, reinterpret_cast<unsigned long long *>(deg_out));
  AG_LAUNCH_CHECK("histogram_kernel");
  return AG_OK;
}

extern "C" int ag_decompose_count(int64_t E, const int32_t *dst, const int32_t *src,
                                  int64_t B, int64_t *num_intra_host, void *stream) {
  *num_intra_host = 0;
  if (B < 1) return fail(AG_ERR_VALUE, "block_size must be >= 1");
  if (E == 0) return AG_OK;
  cudaStream_t st = as_stream(stream);
  Scratch cnt;
  AG_CUDA(cnt.alloc(8, st));
  AG_CUDA(cudaMemsetAsync(cnt.ptr, 0, 8, st));
  count_intra_kernel<<<grid_for(E, kThreads, 2048), kThreads, 0, st>>>(
      E, dst, src, B, cnt.as<unsigned long long>());
  AG_LAUNCH_CHECK("count_intra_kernel");
  unsigned long long h = 0;
  AG_CUDA(cudaMemcpyAsync(&h, cnt.ptr, 8, cudaMemcpyDeviceToHost, st));
  AG_CUDA(cudaStreamSynchronize(st));
  *num_intra_host = static_cast<int64_t>(h);
  return AG_OK;
}

extern "C" int ag_decompose_split(int64_t E, const int32_t *dst, const int32_t *src,
                                  const float *w, int64_t B, int32_t *intra_dst,
                                  int32_t *intra_src, float *intra_w, int32_t *inter_dst,
                                  int32_t *inter_src, float *inter_w, void *stream) {
  if (B < 1) return fail(AG_ERR_VALUE, "block_size must be >= 1");
  if (E == 0) return AG_OK;
  cudaStream_t st = as_stream(stream);
  Scratch flags, pos, tmp;
  AG_CUDA(flags.alloc(E * sizeof(int32_t), st));
  AG_CUDA(pos.alloc(E * sizeof(int32_t), st));
  intra_flags_kernel<<<grid_for(E, kThreads), kThreads, 0, st>>>(E, dst, src, B,
                                                                 flags.as<int32_t>());
  size_t bytes = 0;
  AG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, flags.as<int32_t>(), pos.as<int32_t>(),
                                        (int)E, st));
  AG_CUDA(tmp.alloc(bytes, st));
  AG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.ptr, bytes, flags.as<int32_t>(), pos.as<int32_t>(),
                                        (int)E, st));
  split_kernel<<<grid_for(E, kThreads), kThreads, 0, st>>>(
      E, dst, src, w, flags.as<int32_t>(), pos.as<int32_t>(), intra_dst, intra_src, intra_w,
      inter_dst, inter_src, inter_w);
  AG_LAUNCH_CHECK("split_kernel");
  return AG_OK;
}

extern "C" int ag_build_row_ptr(int64_t V, int64_t E, const int32_t *dst, int32_t *row_ptr,
                                void *stream) {
  row_ptr_kernel<<<grid_for(E + 1, kThreads), kThreads, 0, as_stream(stream)>>>(V, E, dst,
                                                                                 row_ptr);
  AG_LAUNCH_CHECK("row_ptr_kernel");
  return AG_OK;
}

extern "C" int ag_row_touched(int64_t rows, const int32_t *row_ptr, uint8_t *touched,
                              void *stream) {
  if (rows == 0) return AG_OK;
  touched_kernel<<<grid_for(rows, kThreads), kThreads, 0, as_stream(stream)>>>(rows, row_ptr,
                                                                               touched);
  AG_LAUNCH_CHECK("touched_kernel");
  return AG_OK;
}

extern "C" int ag_first_off_block(int64_t rows, const int32_t *row_ptr, const int32_t *col_idx,
                                  int64_t B, int64_t *first_bad_host, void *stream) {
  *first_bad_host = -1;
  if (B < 1) return fail(AG_ERR_KERNEL, "block_size must be >= 1");
  if (rows == 0) return AG_OK;
  cudaStream_t st = as_stream(stream);
  Scratch first;
  AG_CUDA(first.alloc(8, st));
  AG_CUDA(cudaMemsetAsync(first.ptr, 0xFF, 8, st));
  off_block_kernel<<<grid_for(rows, kThreads), kThreads, 0, st>>>(
      rows, row_ptr, col_idx, B, first.as<unsigned long long>());
  AG_LAUNCH_CHECK("off_block_kernel");
  unsigned long long h = 0;
  AG_CUDA(cudaMemcpyAsync(&h, first.ptr, 8, cudaMemcpyDeviceToHost, st));
  AG_CUDA(cudaStreamSynchronize(st));
  *first_bad_host = (h == 0xFFFFFFFFFFFFFFFFULL) ? -1 : static_cast<int64_t>(h);
  return AG_OK;
}

extern "C" int ag_blocks_count(int64_t V, int64_t E, const int32_t *dst, int64_t B,
                               int64_t *k_host, void *stream) {
  (void)V;
  *k_host = 0;
  if (B < 1) return fail(AG_ERR_VALUE, "block_size must be >= 1");
  if (E == 0) return AG_OK;
  cudaStream_t st = as_stream(stream);
  Scratch flags, cnt, tmp;
  AG_CUDA(flags.alloc(E * sizeof(int32_t), st));
  AG_CUDA(cnt.alloc(sizeof(int32_t), st));
  block_heads_kernel<<<grid_for(E, kThreads), kThreads, 0, st>>>(E, dst, B, flags.as<int32_t>());
  size_t bytes = 0;
  AG_CUDA(cub::DeviceReduce::Sum(nullptr, bytes, flags.as<int32_t>(), cnt.as<int32_t>(), (int)E, st));
  AG_CUDA(tmp.alloc(bytes, st));
  AG_CUDA(cub::DeviceReduce::Sum(tmp.ptr, bytes, flags.as<int32_t>(), cnt.as<int32_t>(), (int)E, st));
  int32_t h = 0;
  AG_CUDA(cudaMemcpyAsync(&h, cnt.ptr, 4, cudaMemcpyDeviceToHost, st));
  AG_CUDA(cudaStreamSynchronize(st));
  *k_host = h;
  return AG_OK;
}

extern "C" int ag_blocks_fill(int64_t V, int64_t E, const int32_t *dst, const int32_t *src,
                              const float *w, int64_t B, int64_t k, int32_t *community_ids,
                              int32_t *comm_slot, float *blocks, uint8_t *row_touched,
                              void *stream) {
  if (B < 1) return fail(AG_ERR_VALUE, "block_size must be >= 1");
  cudaStream_t st = as_stream(stream);
  const int64_t ncomm = (V + B - 1) / B;
  if (ncomm > 0) {
    fill_i32_kernel<<<grid_for(ncomm, kThreads), kThreads, 0, st>>>(ncomm, comm_slot, -1);
    AG_LAUNCH_CHECK("fill_i32_kernel");
  }
  if (k > 0) {
    AG_CUDA(cudaMemsetAsync(blocks, 0, k * B * B * sizeof(float), st));
    AG_CUDA(cudaMemsetAsync(row_touched, 0, k * B, st));
  }
  if (E == 0) return AG_OK;
  Scratch flags, pos, tmp;
  AG_CUDA(flags.alloc(E * sizeof(int32_t), st));
  AG_CUDA(pos.alloc(E * sizeof(int32_t), st));
  block_heads_kernel<<<grid_for(E, kThreads), kThreads, 0, st>>>(E, dst, B, flags.as<int32_t>());
  size_t bytes = 0;
  AG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, flags.as<int32_t>(), pos.as<int32_t>(),
                                        (int)E, st));
  AG_CUDA(tmp.alloc(bytes, st));
  AG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.ptr, bytes, flags.as<int32_t>(), pos.as<int32_t>(),
                                        (int)E, st));
  block_slots_kernel<<<grid_for(E, kThreads), kThreads, 0, st>>>(
      E, dst, B, flags.as<int32_t>(), pos.as<int32_t>(), community_ids, comm_slot);
  block_scatter_kernel<<<grid_for(E, kThreads), kThreads, 0, st>>>(E, dst, src, w, B, comm_slot,
                                                                   blocks, row_touched);
  AG_LAUNCH_CHECK("block_scatter_kernel");
  return AG_OK;
}

extern "C" int ag_synth_candidates(int64_t V, int64_t block_gen, double p_intra, double p_global,
                                   int64_t window, int64_t skew, uint64_t seed, int64_t first,
                                   int64_t count, int64_t *dst_out, int64_t *src_out,
                                   void *stream) {
  if (V < 2 || block_gen < 1 || window < 1 || skew < 1)
    return fail(AG_ERR_VALUE, "bad generator parameters");
  if (count == 0) return AG_OK;
  SynthArgs a{V, block_gen, window, skew, p_intra, p_global, mix64(seed), first, count,
              dst_out, src_out};
  synth_kernel<<<grid_for(count, kThreads), kThreads, 0, as_stream(stream)>>>(a);
  AG_LAUNCH_CHECK("synth_kernel");
  return AG_OK;
}

extern "C" int ag_synth_vertex_keys(int64_t V, uint64_t seed, uint64_t *keys, void *stream) {
  if (V == 0) return AG_OK;
  vertex_keys_kernel<<<grid_for(V, kThreads), kThreads, 0, as_stream(stream)>>>(
      V, mix64(seed ^ 0xA5A5A5A5A5A5A5A5ULL), keys);
  AG_LAUNCH_CHECK("vertex_keys_kernel");
  return AG_OK;
}
