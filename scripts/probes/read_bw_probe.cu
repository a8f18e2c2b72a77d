// Pure-read HBM bandwidth on sm_100a (what a read-only stream such as the skinny kernel's
// can reach): (a) LDG.128 grid-stride sum, (b) bulk copies (cp.async.bulk) into a per-CTA
// smem ring with an mbarrier full/empty pipeline, no compute.  Also a copy (read + write)
// for comparison with MEASURED_PEAKS.json.  Prints GB/s (CUDA events, best of 5).
#include <cstdio>
#include <cstdint>
__global__ void ldg_sum(const float4* __restrict__ p, int64_t n, float* out) {
  float s = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    float4 a = __ldcs(p + i), b = __ldcs(p + i + stride), c = __ldcs(p + i + 2 * stride), d = __ldcs(p + i + 3 * stride);
    s += a.x + a.y + a.z + a.w + b.x + b.y + b.z + b.w + c.x + c.y + c.z + c.w + d.x + d.y + d.z + d.w;
  }
  for (; i < n; i += stride) { float4 a = p[i]; s += a.x + a.y + a.z + a.w; }
  if (s == 1234.5f) *out = s;
}
__global__ void copy_k(const float4* __restrict__ p, float4* __restrict__ q, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) q[i] = __ldcs(p + i);
}
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void bulk_ring(const char* __restrict__ g, int64_t bytes, int chunk, int stages, float* out) {
  extern __shared__ __align__(128) char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * chunk);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&full[i])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[i])), "r"(blockDim.x / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t nch = bytes / chunk;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  float s = 0.f;
  int64_t issued = blockIdx.x, g_i = 0;
  int slot = 0; uint32_t ph = 0;
  // producer primes the ring
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages && issued < nch; ++i, issued += gridDim.x) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[i])), "r"(chunk) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sa(sm + (size_t)i * chunk)), "l"(g + issued * chunk), "r"(chunk), "r"(sa(&full[i])) : "memory");
    }
  }
  for (int64_t c = blockIdx.x; c < nch; c += gridDim.x, ++g_i) {
    uint32_t ok = 0;
    while (!ok) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                             : "=r"(ok) : "r"(sa(&full[slot])), "r"(ph) : "memory");
    s += reinterpret_cast<const float*>(sm + (size_t)slot * chunk)[threadIdx.x];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[slot])) : "memory");
    if (threadIdx.x == 0 && issued < nch) {
      uint32_t ok2 = 0;
      while (!ok2) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                                : "=r"(ok2) : "r"(sa(&empty[slot])), "r"(ph) : "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[slot])), "r"(chunk) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sa(sm + (size_t)slot * chunk)), "l"(g + issued * chunk), "r"(chunk), "r"(sa(&full[slot])) : "memory");
      issued += gridDim.x;
    }
    if (++slot == stages) { slot = 0; ph ^= 1; }
  }
  if (s == 1234.5f) *out = s;
  (void)warp;
}
template <typename F>
float best_ms(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 6; ++r) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (r > 0 && ms < best) best = ms;
  }
  return best;
}
int main() {
  const int64_t bytes = int64_t(12) << 30;
  char* buf; float* out; char* dst;
  if (cudaMalloc(&buf, bytes) != cudaSuccess || cudaMalloc(&dst, int64_t(2) << 30) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMalloc(&out, 4);
  cudaMemset(buf, 0, bytes);
  const int64_t n4 = bytes / 16;
  for (int bpsm : {2, 4, 8}) for (int thr : {256, 512}) {
    float ms = best_ms([&] { ldg_sum<<<148 * bpsm, thr>>>(reinterpret_cast<const float4*>(buf), n4, out); });
    printf("ldg_sum grid=148x%d threads=%d: %.0f GB/s\n", bpsm, thr, bytes / ms / 1e6);
  }
  {
    const int64_t cb = int64_t(2) << 30;
    float ms = best_ms([&] { copy_k<<<148 * 8, 512>>>(reinterpret_cast<const float4*>(buf), reinterpret_cast<float4*>(dst), cb / 16); });
    printf("copy 2 GiB (read+write): %.0f GB/s\n", 2.0 * cb / ms / 1e6);
  }
  for (int chunk : {16384, 32768, 49152}) for (int stages : {4, 6, 8, 12}) {
    const size_t smem = (size_t)chunk * stages + 16 * stages;
    if (smem > 227 * 1024) continue;
    cudaFuncSetAttribute(bulk_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    float ms = best_ms([&] { bulk_ring<<<148, 512, smem>>>(buf, bytes, chunk, stages, out); });
    printf("bulk_ring chunk=%d stages=%d (%zu KB in ring): %.0f GB/s\n", chunk, stages, smem / 1024, bytes / ms / 1e6);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
