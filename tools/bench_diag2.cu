// Microbenchmark of the blocked diagonal factor + inverse (ps_diag.cuh).
#include <cstdio>
#include <vector>
#include "ps_dataflow.cuh"
using namespace ps;

template <int ABL, int NT = 128>
__global__ void kb(double* blk, double* G, int reps, int nb) {
  __shared__ DiagSmem s;
  for (int it = 0; it < reps; ++it) {
    const int tid = threadIdx.x;
    for (int idx = tid; idx < 64 * 64; idx += NT) {
      const int c = idx / 64, r = idx % 64;
      s.D[c][r] = (r >= c && r < nb && c < nb) ? blk[c * 64 + r] : 0.0;
    }
    if (tid == 0) s.s_fail = -1;
    __syncthreads();
    factor_block_inv<ABL, NT>(s.D, s.rdiag, s.W, nb, false, 0.0, &s.s_fail, &s.s_fpiv, tid);
    __syncthreads();
  }
  store_block_inv<NT>(s.D, s.rdiag, s.W, nb, false, blk, 64, 0, G, threadIdx.x);
}

template <int ABL, int NT = 128>
float run(double* d, double* G, int nb) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  kb<ABL, NT><<<1, NT>>>(d, G, 1, nb);
  cudaEventRecord(a);
  kb<ABL, NT><<<1, NT>>>(d, G, 100, nb);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / 100;
}

int main() {
  std::vector<double> h(64 * 64);
  for (int c = 0; c < 64; ++c) for (int r = 0; r < 64; ++r) h[c * 64 + r] = r == c ? 70.0 : -0.5 / (1 + abs(r - c));
  double *d, *G; cudaMalloc(&d, 8 * 4096); cudaMalloc(&G, 8 * 4096);
  cudaMemcpy(d, h.data(), 8 * 4096, cudaMemcpyHostToDevice);
  printf("per factorization (in-loop, 1 CTA): full %.2f us | shuffle-form warp factor %.2f | no warp factor %.2f | no solve/schur %.2f | no inverse %.2f | nothing %.2f\n",
         run<0>(d, G, 64), run<8>(d, G, 64), run<1>(d, G, 64), run<2>(d, G, 64), run<4>(d, G, 64), run<7>(d, G, 64));
  // bitwise comparison of the two warp-factor forms (one factorization each)
  std::vector<double> o0(8192), o1(8192);
  cudaMemcpy(d, h.data(), 8 * 4096, cudaMemcpyHostToDevice);
  kb<0><<<1, 128>>>(d, G, 1, 64);
  cudaMemcpy(o0.data(), d, 8 * 4096, cudaMemcpyDeviceToHost);
  cudaMemcpy(o0.data() + 4096, G, 8 * 4096, cudaMemcpyDeviceToHost);
  cudaMemcpy(d, h.data(), 8 * 4096, cudaMemcpyHostToDevice);
  kb<8><<<1, 128>>>(d, G, 1, 64);
  cudaMemcpy(o1.data(), d, 8 * 4096, cudaMemcpyDeviceToHost);
  cudaMemcpy(o1.data() + 4096, G, 8 * 4096, cudaMemcpyDeviceToHost);
  int ndiff = 0;
  for (int k = 0; k < 8192; ++k) ndiff += o0[k] != o1[k];
  printf("smem vs shuffle form: %d differing entries of 8192\n", ndiff);
  printf("256 threads: full %.2f us | no warp factor %.2f | no solve/schur %.2f | no inverse %.2f\n",
         run<0, 256>(d, G, 64), run<1, 256>(d, G, 64), run<2, 256>(d, G, 64), run<4, 256>(d, G, 64));
  std::vector<double> o2(8192);
  cudaMemcpy(d, h.data(), 8 * 4096, cudaMemcpyHostToDevice);
  kb<0, 256><<<1, 256>>>(d, G, 1, 64);
  cudaMemcpy(o2.data(), d, 8 * 4096, cudaMemcpyDeviceToHost);
  cudaMemcpy(o2.data() + 4096, G, 8 * 4096, cudaMemcpyDeviceToHost);
  ndiff = 0;
  for (int k = 0; k < 8192; ++k) ndiff += o0[k] != o2[k];
  printf("256 vs 128 threads: %d differing entries of 8192\n", ndiff);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
