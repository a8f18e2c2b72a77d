// FFMA vs FFMA2 (fma.rn.f32x2) throughput on sm_100a: 16 independent accumulator chains
// per thread, 8 warps per SMSP; prints lane-FMAs per clock per SM for both forms.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint64_t pk(float a, float b) { uint64_t r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void fma2(uint64_t& d, uint64_t a, uint64_t b) { asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b)); }
__global__ void k1(float* out, float a, float b, int n, long long* clk) {
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  float x = a + threadIdx.x * 1e-7f, y = b;
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fmaf(acc[i], x, y);
    x += 1e-9f;
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}
__global__ void k2(float* out, float a, float b, int n, long long* clk) {
  uint64_t acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = pk(threadIdx.x * 1e-3f + i, i * 0.5f);
  uint64_t x = pk(a + threadIdx.x * 1e-7f, a), y = pk(b, b);
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) fma2(acc[i], x, y);
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 16; ++i) { float lo, hi; asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[i])); s += lo + hi; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}
int main() {
  float* out; long long* clk; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&clk, 8);
  const int n = 1 << 16;
  for (int threads : {256, 512, 1024}) {
    for (int v = 0; v < 2; ++v) {
      for (int rep = 0; rep < 2; ++rep) {
        if (v == 0) k1<<<148, threads>>>(out, 1.0001f, 1e-6f, n, clk); else k2<<<148, threads>>>(out, 1.0001f, 1e-6f, n, clk);
      }
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
      double lane_fma = (double)threads * n * 16 * (v ? 2 : 1);
      printf("%s threads=%d: %.1f lane-FMA/clk/SM\n", v ? "FFMA2" : "FFMA ", threads, lane_fma / c);
    }
  }
  cudaError_t e = cudaGetLastError(); printf("%s\n", cudaGetErrorString(e));
}
