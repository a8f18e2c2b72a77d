// FP64 tensor-pipe peak probe: back-to-back mma.sync m16n8k4 f64 from registers (no
// memory traffic), 8 independent accumulator chains per warp, all SMs.  Prints TFLOP/s.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_peak dmma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_loop(double* out, int iters) {
  double c[8][4] = {};
  double a0 = threadIdx.x * 1e-3, a1 = 1.0 - a0, b0 = 0.5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[q][0]), "+d"(c[q][1]), "+d"(c[q][2]), "+d"(c[q][3])
                   : "d"(a0), "d"(a1), "d"(b0));
  }
  double s = 0;
  for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1] + c[q][2] + c[q][3];
  if (s == 12345.678) out[0] = s;
}
int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  for (int warps = 4; warps <= 16; warps *= 2) {
    dmma_loop<<<sms * 2, 32 * warps>>>(out, 100);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    dmma_loop<<<sms * 2, 32 * warps>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 16 * 8 * 4 * 8.0 * iters * (double)(sms * 2) * warps;
    printf("warps/CTA %2d: %.2f TFLOP/s fp64 tensor (%.3f ms)\n", warps, flops / (ms * 1e-3) / 1e12, ms);
  }
  return 0;
}
