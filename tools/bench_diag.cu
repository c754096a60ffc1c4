// Microbenchmark of the wide-panel diagonal kernel variants (development tool).
#include <cstdio>
#include <vector>
#include <cmath>
#include "ps_kernels.cuh"
using namespace ps;

template <int MODE, int VAR>
float run(int reps, FItem* d_items, DevArgs* d_args, PanelDev P, i64* fc, double* fp, int nitems) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k_factor_diag<MODE, VAR><<<nitems, DIAG_THREADS>>>(d_items, d_args, P, fc, fp);
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) k_factor_diag<MODE, VAR><<<nitems, DIAG_THREADS>>>(d_items, d_args, P, fc, fp);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / reps;
}

int main() {
  const int nb = 64, nr = 64;
  std::vector<double> h(nb * nr, 0.0);
  for (int c = 0; c < nb; ++c) for (int r = c; r < nr; ++r) h[c * nr + r] = (r == c) ? 70.0 : -0.5 / (1 + r - c);
  double *store, *scratch; cudaMalloc(&store, 8 * h.size()); cudaMalloc(&scratch, 8 * 4096);
  i64 off = 0; int ld = nr, w = nb; i64 fcol = 0;
  i64 *d_off, *d_fc; int *d_ld, *d_w; cudaMalloc(&d_off, 8); cudaMalloc(&d_fc, 8); cudaMalloc(&d_ld, 4); cudaMalloc(&d_w, 4);
  cudaMemcpy(d_off, &off, 8, cudaMemcpyHostToDevice); cudaMemcpy(d_fc, &fcol, 8, cudaMemcpyHostToDevice);
  cudaMemcpy(d_ld, &ld, 4, cudaMemcpyHostToDevice); cudaMemcpy(d_w, &w, 4, cudaMemcpyHostToDevice);
  PanelDev P{d_off, d_ld, d_w, d_fc};
  FItem it{0, 0, nb, nb, 0, 1, 0, 0};
  FItem* d_items; cudaMalloc(&d_items, sizeof(FItem)); cudaMemcpy(d_items, &it, sizeof it, cudaMemcpyHostToDevice);
  i64* fc; double* fp; cudaMalloc(&fc, 8); cudaMalloc(&fp, 8);
  for (int form = 0; form < 2; ++form) {
    DevArgs args{store, scratch, 0.0, form, 0};
    DevArgs* d_args; cudaMalloc(&d_args, sizeof args); cudaMemcpy(d_args, &args, sizeof args, cudaMemcpyHostToDevice);
    auto reset = [&]() { cudaMemcpy(store, h.data(), 8 * h.size(), cudaMemcpyHostToDevice); };
    reset(); float t30 = run<3, 0>(50, d_items, d_args, P, fc, fp, 1);
    reset(); float t31 = run<3, 1>(50, d_items, d_args, P, fc, fp, 1);
    reset(); float t10 = run<1, 0>(50, d_items, d_args, P, fc, fp, 1);
    reset(); float t11 = run<1, 1>(50, d_items, d_args, P, fc, fp, 1);
    reset(); float t2 = run<2, 1>(50, d_items, d_args, P, fc, fp, 1);
    reset(); float t0 = run<0, 1>(50, d_items, d_args, P, fc, fp, 1);
    reset(); float t32 = run<3, 2>(50, d_items, d_args, P, fc, fp, 1);
    reset(); float t33 = run<3, 3>(50, d_items, d_args, P, fc, fp, 1);
    printf("form %d: fused factor+inverse (v2) %.1f us, balanced (v3) %.1f us\n", form, t32, t33);
    reset(); float a4 = run<3, 4>(50, d_items, d_args, P, fc, fp, 1);
    reset(); float a5 = run<3, 5>(50, d_items, d_args, P, fc, fp, 1);
    reset(); float a6 = run<3, 6>(50, d_items, d_args, P, fc, fp, 1);
    printf("  ablation: no-update %.1f us, no-barrier %.1f us, barriers-only %.1f us\n", a4, a5, a6);
    {
      std::vector<double> g0(4096), g3(4096), f0(h.size()), f3(h.size());
      reset(); k_factor_diag<3, 0><<<1, DIAG_THREADS>>>(d_items, d_args, P, fc, fp); cudaMemcpy(g0.data(), scratch, 8 * 4096, cudaMemcpyDeviceToHost); cudaMemcpy(f0.data(), store, 8 * h.size(), cudaMemcpyDeviceToHost);
      reset(); k_factor_diag<3, 3><<<1, DIAG_THREADS>>>(d_items, d_args, P, fc, fp); cudaMemcpy(g3.data(), scratch, 8 * 4096, cudaMemcpyDeviceToHost); cudaMemcpy(f3.data(), store, 8 * h.size(), cudaMemcpyDeviceToHost);
      double md = 0, mf = 0; for (int i = 0; i < 4096; ++i) md = fmax(md, fabs(g0[i] - g3[i]));
      for (size_t i = 0; i < h.size(); ++i) mf = fmax(mf, fabs(f0[i] - f3[i]));
      printf("  v3: max |G_v0 - G_v3| = %.3e, max |L_v0 - L_v3| = %.3e\n", md, mf);
    }
    {
      // G of v2 vs G of v0 (separate inverse), same input
      std::vector<double> g0(4096), g2(4096);
      reset(); k_factor_diag<3, 0><<<1, DIAG_THREADS>>>(d_items, d_args, P, fc, fp); cudaMemcpy(g0.data(), scratch, 8 * 4096, cudaMemcpyDeviceToHost);
      reset(); k_factor_diag<3, 2><<<1, DIAG_THREADS>>>(d_items, d_args, P, fc, fp); cudaMemcpy(g2.data(), scratch, 8 * 4096, cudaMemcpyDeviceToHost);
      double md = 0, mx = 0; for (int i = 0; i < 4096; ++i) { md = fmax(md, fabs(g0[i] - g2[i])); mx = fmax(mx, fabs(g0[i])); }
      printf("  max |G_v0 - G_v2| = %.3e (max |G| %.3e)\n", md, mx);
    }
    printf("form %d: full(v0) %.1f us  full(v1) %.1f us  factor-only v0 %.1f  v1 %.1f  inverse-only %.1f  load/store-only %.1f\n",
           form, t30, t31, t10, t11, t2, t0);
    // correctness of v1 vs v0 (factor of the same input)
    std::vector<double> r0(h.size()), r1(h.size());
    reset(); k_factor_diag<1, 0><<<1, DIAG_THREADS>>>(d_items, d_args, P, fc, fp); cudaMemcpy(r0.data(), store, 8 * h.size(), cudaMemcpyDeviceToHost);
    reset(); k_factor_diag<1, 1><<<1, DIAG_THREADS>>>(d_items, d_args, P, fc, fp); cudaMemcpy(r1.data(), store, 8 * h.size(), cudaMemcpyDeviceToHost);
    double md = 0; for (size_t i = 0; i < h.size(); ++i) md = fmax(md, fabs(r0[i] - r1[i]));
    printf("  max |v0 - v1| = %.3e\n", md);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
