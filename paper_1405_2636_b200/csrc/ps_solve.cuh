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
constexpr int SV_MAXW = 2048;  // widest panel handled in shared memory (wider: global scratch)
constexpr int SV_PART_W = 256; // panels up to this width: per-warp partial sums of the gather

// the 32x32 diagonal block [c0, c0+nb) into shared memory (one latency
// instead of a dependent global load per pivot): B[c][r] = a(c0 + r, c0 + c)
__device__ __forceinline__ void load_diag32(double (*B)[33], const double* a, i64 ld, int c0, int nb,
                                            int tid) {
  for (int e = tid; e < 32 * 32; e += SV_THREADS) {
    const int c = e >> 5, r = e & 31;
    B[c][r] = (c < nb && r < nb && r >= c) ? __ldcg(a + (i64)(c0 + c) * ld + c0 + r) : 0.0;
  }
  __syncthreads();
}

// y (length w) <- L_pp^-1 y  (lower, unit if ldlt), column-major a (ld)
__device__ __forceinline__ void trsv_lower(const double* a, i64 ld, int w, double* y, bool unit,
                                           int tid, double (*B)[33]) {
  const int lane = tid & 31, warp = tid >> 5;
  for (int c0 = 0; c0 < w; c0 += 32) {
    const int nb = min(32, w - c0);
    load_diag32(B, a, ld, c0, nb, tid);
    // warp 0 solves the 32x32 diagonal block (column sweep, shuffles)
    if (warp == 0) {
      double v = lane < nb ? y[c0 + lane] : 0.0;
      for (int j = 0; j < nb; ++j) {
        double xj = __shfl_sync(0xffffffffu, v, j);
        if (!unit) xj = xj / B[j][j];
        if (lane == j) v = xj;
        if (lane > j && lane < nb) v -= B[j][lane] * xj;
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
                                             int tid, double (*B)[33]) {
  const int lane = tid & 31, warp = tid >> 5;
  for (int c1 = w; c1 > 0; c1 -= 32) {
    const int c0 = max(0, c1 - 32), nb = c1 - c0;
    load_diag32(B, a, ld, c0, nb, tid);
    // warp 0: the diagonal block, backward (row j of L^T = column j of L)
    if (warp == 0) {
      double v = lane < nb ? y[c0 + lane] : 0.0;
      for (int j = nb - 1; j >= 0; --j) {
        double xj = __shfl_sync(0xffffffffu, v, j);
        if (!unit) xj = xj / B[j][j];
        if (lane == j) v = xj;
        // unknowns i < j: y_i -= L[j, i] x_j
        if (lane < j) v -= B[lane][j] * xj;
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
  // incoming contributions, ascending source (deterministic).  Couple
  // descriptors are staged 128 at a time (two memory latencies per chunk);
  // per couple, lanes run over facing rows (coalesced) and the 8 warps over
  // the source columns, reduced in a fixed order.
  __shared__ int cs_p[128], cs_loc0[128], cs_n[128], cs_w[128], cs_ld[128];
  __shared__ i64 cs_off[128], cs_fc[128], cs_rp[128];
  __shared__ double red[SV_THREADS / 32][32];
  __shared__ double parts[(SV_THREADS / 32) * SV_PART_W];
  if (w <= SV_PART_W)
    for (int j = tid; j < (SV_THREADS / 32) * SV_PART_W; j += SV_THREADS) parts[j] = 0.0;
  for (i64 e0 = S.in_ptr[q]; e0 < S.in_ptr[q + 1]; e0 += 128) {
    const int nch = (int)min((i64)128, S.in_ptr[q + 1] - e0);
    if (tid < nch) {
      const int c = S.in_cpl[e0 + tid];
      const int p = S.cpl_p[c];
      cs_p[tid] = p;
      cs_loc0[tid] = S.cpl_loc0[c];
      cs_n[tid] = S.cpl_N[c];
      cs_w[tid] = P.width[p];
      cs_ld[tid] = P.nrows[p];
      cs_off[tid] = P.off[p];
      cs_fc[tid] = P.fc[p];
      cs_rp[tid] = S.rowptr[p];
    }
    __syncthreads();
    if (w <= SV_PART_W) {
      // warps take couples round-robin, each into its own partial vector;
      // the partials are added in warp order (fixed summation order)
      for (int u = warp; u < nch; u += SV_THREADS / 32) {
        const int loc0 = cs_loc0[u], N = cs_n[u], wp = cs_w[u], ldp = cs_ld[u];
        const double* ap = store + cs_off[u];
        const double* zp = z + cs_fc[u];
        const int* rp = S.rows + cs_rp[u];
        double* part = parts + warp * SV_PART_W;
        for (int i = lane; i < N; i += 32) {
          double sacc = 0.0;
          for (int k = 0; k < wp; ++k) sacc += __ldcg(ap + (i64)k * ldp + loc0 + i) * __ldcg(zp + k);
          part[rp[loc0 + i - wp] - fcq] += sacc;
        }
        __syncwarp();  // couples of one warp may hit the same entries from different lanes
      }
      __syncthreads();
    } else {
      for (int u = 0; u < nch; ++u) {
        const int loc0 = cs_loc0[u], N = cs_n[u], wp = cs_w[u], ldp = cs_ld[u];
        const double* ap = store + cs_off[u];
        const double* zp = z + cs_fc[u];
        const int* rp = S.rows + cs_rp[u];
        for (int i0 = 0; i0 < N; i0 += 32) {
          const int i = i0 + lane;
          double sacc = 0.0;
          if (i < N)
            for (int k = warp; k < wp; k += SV_THREADS / 32)
              sacc += __ldcg(ap + (i64)k * ldp + loc0 + i) * __ldcg(zp + k);
          red[warp][lane] = sacc;
          __syncthreads();
          if (warp == 0 && i < N) {
            double t = 0.0;
#pragma unroll
            for (int v = 0; v < SV_THREADS / 32; ++v) t += red[v][lane];
            y[rp[loc0 + i - wp] - fcq] -= t;
          }
          __syncthreads();
        }
      }
    }
  }
  if (w <= SV_PART_W) {
    for (int j = tid; j < w; j += SV_THREADS) {
      double t = 0.0;
#pragma unroll
      for (int v = 0; v < SV_THREADS / 32; ++v) t += parts[v * SV_PART_W + j];
      y[j] -= t;
    }
    __syncthreads();
  }
  __shared__ double B32[32][33];
  trsv_lower(store + P.off[q], P.nrows[q], w, y, ldlt != 0, tid, B32);
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
  __shared__ double B32[32][33];
  trsv_lower_t(a, ld, w, y, ldlt != 0, tid, B32);
  for (int j = tid; j < w; j += SV_THREADS) x[fcp + j] = y[j];
}

}  // namespace ps
