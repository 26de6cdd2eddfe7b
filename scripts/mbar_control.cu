// Control case for compute-sanitizer racecheck: a minimal, correct mbarrier
// producer/consumer hand-off (the slab kernel's ready/done protocol in
// miniature).  Warp 1 fills a shared buffer (plain stores, then a
// cp.async.bulk copy completing on the barrier), arrives; warp 0 waits on the
// barrier's phase and reads.  Every read is ordered after the write by the
// mbarrier, so any hazard racecheck reports here is a false positive of its
// model, not a race.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t su32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void handoff(const float *src, float *out, int rounds) {
  __shared__ __align__(128) float buf[2][256];
  __shared__ __align__(128) float buf2[2][256];  // written with plain st.shared
  __shared__ __align__(8) uint64_t full[2], empty[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      asm volatile("mbarrier.init.shared.b64 [%0], 2;" ::"r"(su32(&full[i])));
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  float acc = 0.f;
  for (int r = 0; r < rounds; ++r) {
    const int s = r & 1;
    const uint32_t ph = (r >> 1) & 1;
    if (warp == 1) {
      if (r >= 2) {  // wait until the consumer released slot s
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                       : "=r"(ok) : "r"(su32(&empty[s])), "r"(ph ^ 1));
      }
      if (lane == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(1024));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 1024, [%2];"
                     ::"r"(su32(buf[s])), "l"(src + r * 256), "r"(su32(&full[s])) : "memory");
      }
      for (int i = lane; i < 256; i += 32) buf2[s][i] = 2.0f;
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(su32(&full[s])) : "memory");
    } else if (warp == 0) {
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(su32(&full[s])), "r"(ph));
      for (int i = lane; i < 256; i += 32) acc += buf[s][i] + buf2[s][i];
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
    }
  }
  if (warp == 0) out[lane] = acc;
}

int main() {
  const int rounds = 64;
  float *src, *out;
  cudaMalloc(&src, rounds * 256 * sizeof(float));
  cudaMalloc(&out, 32 * sizeof(float));
  float h[256 * rounds];
  for (int i = 0; i < 256 * rounds; ++i) h[i] = 1.0f;
  cudaMemcpy(src, h, sizeof(h), cudaMemcpyHostToDevice);
  handoff<<<1, 64>>>(src, out, rounds);
  float o[32];
  cudaMemcpy(o, out, sizeof(o), cudaMemcpyDeviceToHost);
  float t = 0;
  for (float v : o) t += v;
  std::printf("mbar_control: sum %.0f (expect %d), %s\n", t, 3 * 256 * rounds,
              cudaGetErrorString(cudaGetLastError()));
  return t == 3.0f * 256 * rounds ? 0 : 1;
}
