// Microbenchmark of the DMMA update-tile mainloop structure (development tool):
// 128-thread CTAs, 2 x 2 warps of 32 x 32 (4 x 4 DMMA 8x8x4 fragments), 16-wide
// k chunks through NSTAGE shared stages.  Variants isolate what limits the
// DMMA pipe: MODE 0 = LDS + DMMA only (stages pre-filled), 1 = + per-chunk
// __syncthreads, 2 = + cp.async staging of A / B (8-byte, L2-resident
// source, odd leading dimension like the slab), 3 = 2 with 16-byte cp.async
// (even leading dimension).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mainloop_bench mainloop_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#ifndef NST_
#define NST_ 3
#endif
constexpr int KC = 16, NST = NST_, LDS = 68, TM = 64;
struct Sm {
  double A[NST][KC][LDS];
  double B[NST][KC][LDS];
};
__device__ __forceinline__ void cpa8(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(s)), "l"(g));
}
__device__ __forceinline__ void cpa16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(s)), "l"(g));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void waitg() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int MODE>
__global__ void __launch_bounds__(128, 3) kern(const double* __restrict__ src, long ld, int nch, double* out) {
  extern __shared__ __align__(16) unsigned char raw[];
  Sm& sm = *reinterpret_cast<Sm*>(raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, wm = warp & 1, wn = warp >> 1;
  for (int i = tid; i < NST * KC * LDS; i += 128) {
    (&sm.A[0][0][0])[i] = 1e-3 * (i % 7);
    (&sm.B[0][0][0])[i] = 1e-3 * (i % 5);
  }
  __syncthreads();
  const double* A = MODE == 4 ? src + (long)blockIdx.x * 4096 * ld : src + (long)blockIdx.x * 64 * ld % (1 << 22);
  double acc[4][4][2] = {};
  auto load = [&](int st, int c) {
    if (MODE == 3) {
#pragma unroll
      for (int e = 0; e < (KC * TM / 2) / 128; ++e) {
        const int idx = tid + e * 128, r = (idx % 32) * 2, kk = idx / 32;
        cpa16(&sm.A[st][kk][r], A + (long)(c * KC + kk) * ld + r);
        cpa16(&sm.B[st][kk][r], A + (long)(c * KC + kk) * ld + 64 + r);
      }
    } else {
#pragma unroll
      for (int e = 0; e < (KC * TM) / 128; ++e) {
        const int idx = tid + e * 128, r = idx % 64, kk = idx / 64;
        cpa8(&sm.A[st][kk][r], A + (long)(c * KC + kk) * ld + 1 + r);
        cpa8(&sm.B[st][kk][r], A + (long)(c * KC + kk) * ld + 65 + r);
      }
    }
  };
  if (MODE >= 2) {
    for (int s = 0; s < NST - 1; ++s) { load(s, s); commit(); }
  }
  for (int c = 0; c < nch; ++c) {
    if (MODE >= 2) waitg<NST - 2>();
    if (MODE >= 1) __syncthreads();
    if (MODE >= 2) { if (c + NST - 1 < nch) load((c + NST - 1) % NST, (c + NST - 1) % (MODE == 4 ? 256 : 64)); commit(); }
    const int st = c % NST;
#pragma unroll
    for (int ks = 0; ks < KC / 4; ++ks) {
      const int kr = ks * 4 + (lane & 3);
      double af[4], bf[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) af[mi] = sm.A[st][kr][(wm * 4 + mi) * 8 + (lane >> 2)];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) bf[ni] = sm.B[st][kr][(wn * 4 + ni) * 8 + (lane >> 2)];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
    }
  }
  double s = 0;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) s += acc[mi][ni][0] + acc[mi][ni][1];
  if (s == 1.2345) out[tid] = s;
}

template <int MODE>
void run(const double* src, long ld, double* out, int sms, int cps) {
  const int nch = 4096;
  auto k = kern<MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Sm));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<<<sms * cps, 128, sizeof(Sm)>>>(src, ld, 64, out);
  cudaEventRecord(e0);
  k<<<sms * cps, 128, sizeof(Sm)>>>(src, ld, nch, out);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 2.0 * 64 * 64 * KC * (double)nch * sms * cps;
  printf("mode %d ctas/sm %d ld %ld: %.2f TFLOP/s (%s)\n", MODE, cps, ld, fl / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* src; cudaMalloc(&src, 64l << 20);
  cudaMemset(src, 0, 64l << 20);
  double* out; cudaMalloc(&out, 4096);
  for (int cps : {2, 3}) {
    run<0>(src, 1001, out, sms, cps);
    run<1>(src, 1001, out, sms, cps);
    run<2>(src, 1001, out, sms, cps);
    run<3>(src, 1000, out, sms, cps);
    run<4>(src, 1001, out, sms, cps);
  }
  return 0;
}
