// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64) vs DFMA.
// Used to fill the FP64 roofline denominator (MEASURED_PEAKS.json carries only bf16/HBM).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 123.456) out[threadIdx.x] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 123.456) out[threadIdx.x] = s;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int wpb : {4, 8, 16, 32}) {
    for (int cps : {1, 2}) {
      int grid = sms * cps, block = 32 * wpb;
      dmma_loop<<<grid, block>>>(out, 100);
      cudaEventRecord(e0);
      dmma_loop<<<grid, block>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (double)grid * wpb;
      printf("DMMA  warps/blk=%2d ctas/sm=%d : %.2f TFLOP/s\n", wpb, cps, flops / ms / 1e9);
      dfma_loop<<<grid, block>>>(out, 100);
      cudaEventRecord(e0);
      dfma_loop<<<grid, block>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      flops = 2.0 * 8.0 * iters * (double)grid * block;
      printf("DFMA  warps/blk=%2d ctas/sm=%d : %.2f TFLOP/s\n", wpb, cps, flops / ms / 1e9);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
