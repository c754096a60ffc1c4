// GPU supernodal triangular solve: the contract of the
// reference's supernodal_solve (kernels.py:332-382) on the device-resident
// factor, level by level, deterministic (no atomics):
//
//   forward  (levels ascending), one CTA per panel q:
//     z_q = x_q - sum over couples (p -> q), ascending p, of L_p[facing rows] z_p
//           (gather form: the destination pulls its contributions)
//     z_q = L_qq^-1 z_q            (unit lower for LDLt)
//     x_q = z_q / d_q (LDLt)  |  z_q (LLt)
//   backward (levels descending), one CTA per panel p:
//     y = x_p - L_p[rows]^T x[rows]   (rows: ancestors, already final)
//     x_p = L_pp^-T y                 (unit upper for LDLt)
//
// x is in the permuted order (x[perm] = b before, b = x[perm] after).
#pragma once
#include "ps_kernels.cuh"

namespace ps {

struct SolveDev {
  const i64* lvl_ptr;   // panels of level L: lvl_panels[lvl_ptr[L] .. lvl_ptr[L+1])
  const int* lvl_panels;
  const i64* in_ptr;    // couples into q: in_cpl[in_ptr[q] .. in_ptr[q+1]), ascending source
  const int* in_cpl;
  const int* cpl_p;     // per couple: source panel, first facing local row, facing rows
  const int* cpl_loc0;
  const int* cpl_N;
  const i64* rowptr;    // per panel: off-diagonal global rows rows[rowptr[p] .. rowptr[p+1])
  const int* rows;
};

constexpr int SV_THREADS = 256;
constexpr int SV_MAXW = 4096;  // widest panel handled in shared memory (wider: global scratch)

// y (length w, shared) <- L_pp^-1 y  (lower, unit if ldlt), column-major a (ld)
__device__ __forceinline__ void trsv_lower(const double* a, i64 ld, int w, double* y, bool unit,
                                           int tid) {
  const int lane = tid & 31, warp = tid >> 5;
  for (int c0 = 0; c0 < w; c0 += 32) {
    const int nb = min(32, w - c0);
    // warp 0 solves the 32x32 diagonal block (column sweep, shuffles)
    if (warp == 0) {
      double v = lane < nb ? y[c0 + lane] : 0.0;
      for (int j = 0; j < nb; ++j) {
        double xj = __shfl_sync(0xffffffffu, v, j);
        if (!unit) xj = xj / __ldcg(a + (i64)(c0 + j) * ld + c0 + j);
        if (lane == j) v = xj;
        if (lane > j && lane < nb) v -= __ldcg(a + (i64)(c0 + j) * ld + c0 + lane) * xj;
      }
      if (lane < nb) y[c0 + lane] = v;
    }
    __syncthreads();
    // rows below the block: y[r] -= sum_j a[r, c0 + j] y[c0 + j]
    for (int r = c0 + nb + tid; r < w; r += SV_THREADS) {
      double s = 0.0;
      for (int j = 0; j < nb; ++j) s += __ldcg(a + (i64)(c0 + j) * ld + r) * y[c0 + j];
      y[r] -= s;
    }
    __syncthreads();
  }
}

// y <- L_pp^-T y (upper = transpose of the lower factor, unit if ldlt)
__device__ __forceinline__ void trsv_lower_t(const double* a, i64 ld, int w, double* y, bool unit,
                                             int tid) {
  const int lane = tid & 31, warp = tid >> 5;
  for (int c1 = w; c1 > 0; c1 -= 32) {
    const int c0 = max(0, c1 - 32), nb = c1 - c0;
    // warp 0: the diagonal block, backward (row j of L^T = column j of L)
    if (warp == 0) {
      double v = lane < nb ? y[c0 + lane] : 0.0;
      for (int j = nb - 1; j >= 0; --j) {
        double xj = __shfl_sync(0xffffffffu, v, j);
        if (!unit) xj = xj / __ldcg(a + (i64)(c0 + j) * ld + c0 + j);
        if (lane == j) v = xj;
        // unknowns i < j: y_i -= L[j, i] x_j
        if (lane < j) v -= __ldcg(a + (i64)(c0 + lane) * ld + c0 + j) * xj;
      }
      if (lane < nb) y[c0 + lane] = v;
    }
    __syncthreads();
    // columns above the block: y[i] -= sum_j L[c0 + j, i] y[c0 + j], i < c0
    for (int i = tid; i < c0; i += SV_THREADS) {
      const double* col = a + (i64)i * ld + c0;
      double s = 0.0;
      for (int j = 0; j < nb; ++j) s += __ldcg(col + j) * y[c0 + j];
      y[i] -= s;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(SV_THREADS)
k_solve_fwd(int level, SolveDev S, PanelDev P, const double* __restrict__ store, double* x,
            double* z, double* scratch, int ldlt, int maxw) {
  __shared__ double ys[SV_MAXW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = S.lvl_panels[S.lvl_ptr[level] + blockIdx.x];
  const int w = P.width[q];
  const i64 fcq = P.fc[q];
  double* y = w <= maxw ? ys : scratch + fcq;
  for (int j = tid; j < w; j += SV_THREADS) y[j] = x[fcq + j];
  __syncthreads();
  // incoming contributions, ascending source (deterministic): warp per facing row
  for (i64 e = S.in_ptr[q]; e < S.in_ptr[q + 1]; ++e) {
    const int c = S.in_cpl[e];
    const int p = S.cpl_p[c], loc0 = S.cpl_loc0[c], N = S.cpl_N[c];
    const int wp = P.width[p];
    const i64 ldp = P.nrows[p];
    const double* ap = store + P.off[p];
    const double* zp = z + P.fc[p];
    const int* rp = S.rows + S.rowptr[p];
    for (int i = warp; i < N; i += SV_THREADS / 32) {
      const int lr = loc0 + i;
      double s = 0.0;
      for (int k = lane; k < wp; k += 32) s += __ldcg(ap + (i64)k * ldp + lr) * __ldcg(zp + k);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) y[rp[lr - wp] - fcq] -= s;
    }
    __syncthreads();
  }
  trsv_lower(store + P.off[q], P.nrows[q], w, y, ldlt != 0, tid);
  const double* aq = store + P.off[q];
  const i64 ldq = P.nrows[q];
  for (int j = tid; j < w; j += SV_THREADS) {
    const double v = y[j];
    z[fcq + j] = v;
    x[fcq + j] = ldlt ? v / __ldcg(aq + (i64)j * ldq + j) : v;
  }
}

__global__ void __launch_bounds__(SV_THREADS)
k_solve_bwd(int level, SolveDev S, PanelDev P, const double* __restrict__ store, double* x,
            double* scratch, int ldlt, int maxw) {
  __shared__ double ys[SV_MAXW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int p = S.lvl_panels[S.lvl_ptr[level] + blockIdx.x];
  const int w = P.width[p];
  const i64 fcp = P.fc[p], ld = P.nrows[p];
  const double* a = store + P.off[p];
  const int* rp = S.rows + S.rowptr[p];
  const int nr = (int)(S.rowptr[p + 1] - S.rowptr[p]);
  double* y = w <= maxw ? ys : scratch + fcp;
  // y_j = x_j - sum_r L[w + r, j] x[rows[r]]: warp per column
  for (int j = warp; j < w; j += SV_THREADS / 32) {
    double s = 0.0;
    const double* col = a + (i64)j * ld + w;
    for (int r = lane; r < nr; r += 32) s += __ldcg(col + r) * x[rp[r]];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) y[j] = x[fcp + j] - s;
  }
  __syncthreads();
  trsv_lower_t(a, ld, w, y, ldlt != 0, tid);
  for (int j = tid; j < w; j += SV_THREADS) x[fcp + j] = y[j];
}

}  // namespace ps
