// Blocked factorization + inverse of one diagonal block (nb <= 64) in shared
// memory, 128 threads.  Used for the 64-column steps of wide panels.
//
// Unit form for both variants: A = Lu D Lu^T (Lu unit lower).  LLt stores
// L = Lu D^1/2 (kernels.py:230-231: sqrt of the pivot, column scaled by it),
// LDLt stores Lu with d on the diagonal (kernels.py:240-244).  Failure
// predicates are the reference's on the pivot d_j (LLt d_j <= thr, LDLt
// |d_j| <= thr, kernels.py:217-244).
//
// Right-looking over 16-column sub-blocks:
//   1. one warp factors the 16x16 diagonal sub-block in registers (lane i
//      holds row i; pivots broadcast by shuffles - no CTA barrier per pivot)
//      and Gauss-Jordan-eliminates the identity alongside: M_tt = Lu_tt^-1;
//   2. the rows below: X = A_rt M_tt^T (= Lu_rt D_t), Lu_rt = X D_t^-1;
//   3. Schur update of the trailing rows/columns: A -= Lu_rt X^T;
//   4. at the end the off-diagonal blocks of M = Lu^-1 (block forward
//      substitution) and the scaled inverse G = S M, S = D^-1/2 (LLt) or D^-1
//      (LDLt), so that the panel TRSM is X = B G^T (a DMMA GEMM).
// Layout: D[c][r] holds A(r, c) for r >= c (lower); M(j, k), k < j, is kept
// in the free upper slot D[j][k]; dv[j] = d_j; rdiag[j] = S_jj.
#pragma once
#include "ps_kernels.cuh"

namespace ps {

constexpr int DB = 16;  // sub-block

struct DiagWork {
  double X[FNB - DB][DB + 1];  // Lu_rt D_t of the current sub-block (also Y in the inverse)
  double dv[FNB];
  double wcol[DB], wrow[DB];   // warp sub-block factor: pivot column / pivot row of M
};

__device__ __forceinline__ double shfl(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }

// factor D (nb x nb lower, nb <= 64) in place; returns via D/rdiag/dv as above.
// s_fail / s_fpiv: first failing local column and its pivot (s_fail < 0: none).
// ABL (microbenchmark ablation only): bit 0 skips the warp sub-block factor,
// bit 1 the panel solve + Schur update, bit 2 the block inverse
template <int ABL = 0, int NT = 128>
__device__ __forceinline__ void factor_block_inv(double (*D)[FNB + 1], double* rdiag, DiagWork& W,
                                                 int nb, bool ldlt, double thr, int* s_fail,
                                                 double* s_fpiv, int tid) {
  const int nbp = (nb + DB - 1) / DB * DB;
  const int nsub = nbp / DB;
  // identity padding of rows / columns nb..nbp
  constexpr int NWP = NT / 32;  // warps sharing the DMMA phases
  for (int c = nb + tid; c < nbp; c += NT) {
    for (int r = c; r < nbp; ++r) D[c][r] = r == c ? 1.0 : 0.0;
    for (int cc = 0; cc < nb; ++cc) D[cc][c] = 0.0;
  }
  __syncthreads();
  const int lane = tid & 31, warp = tid >> 5;
  for (int t = 0; t < nsub; ++t) {
    const int k0 = t * DB;
    // ---- 1. warp 0: the 16x16 sub-block, in registers ----
    // (pivot column and the pivot row of M are broadcast through shared
    // memory: one store + broadcast loads instead of 64-bit shuffles; ABL bit
    // 3 selects the shuffle form for the microbenchmark.)  Failing pivots
    // are checked once after the sweep (first failing column, in order).
    if (warp == 0 && !(ABL & 1)) {
      const int i = lane & (DB - 1);
      double a[DB], m[DB];
#pragma unroll
      for (int c = 0; c < DB; ++c) {
        a[c] = (c <= i) ? D[k0 + c][k0 + i] : 0.0;
        m[c] = 0.0;
      }
      double my_d = 1.0;
#pragma unroll
      for (int j = 0; j < DB; ++j) {
        const double aj = a[j];
        double piv;
        if (ABL & 8) {
          piv = shfl(aj, j);
        } else {
          W.wcol[i] = aj;  // lanes i and i + 16 store the same value
          if (i == j) {
#pragma unroll
            for (int c = 0; c < j; ++c) W.wrow[c] = m[c];
          }
          __syncwarp();
          piv = W.wcol[j];
        }
        const double ip = rcp_nr(piv);
        const double l = (i > j) ? aj * ip : 0.0;
#pragma unroll
        for (int c = j + 1; c < DB; ++c) {
          const double acj = (ABL & 8) ? shfl(aj, c) : W.wcol[c];  // unscaled column j at row c
          a[c] -= l * acj;
        }
#pragma unroll
        for (int c = 0; c < j; ++c) {
          const double mjc = (ABL & 8) ? shfl(m[c], j) : W.wrow[c];
          m[c] -= l * mjc;
        }
        m[j] = (i > j) ? -l : m[j];
        if (i > j) a[j] = l;
        if (i == j) my_d = piv;
        if (!(ABL & 8)) __syncwarp();
      }
      {
        const bool bad = lane < DB && k0 + i < nb && (ldlt ? (fabs(my_d) <= thr) : (my_d <= thr));
        const unsigned bm = __ballot_sync(0xffffffffu, bad);
        const int f = bm ? __ffs(bm) - 1 : 0;
        const double fp = __shfl_sync(0xffffffffu, my_d, f);
        if (lane == 0 && bm && *s_fail < 0) {
          *s_fail = k0 + f;
          *s_fpiv = fp;
        }
      }
      if (lane < DB) {
#pragma unroll
        for (int c = 0; c < DB; ++c) {
          if (c < i) {
            D[k0 + c][k0 + i] = a[c];  // Lu
            D[k0 + i][k0 + c] = m[c];  // M (upper slot)
          }
        }
        D[k0 + i][k0 + i] = my_d;
        W.dv[k0 + i] = my_d;
        rdiag[k0 + i] = ldlt ? rcp_nr(my_d) : rsqrt_nr(my_d);
      }
    }
    __syncthreads();
    const int rb = k0 + DB;      // first row below the sub-block
    const int R = nbp - rb;      // rows below (0, 16, 32, 48)
    if (R <= 0) break;
    if (ABL & 2) continue;
    const int rt_n = R / 8;
    // ---- 2. X = A_rt M_tt^T (DMMA), Lu_rt = X D_t^-1 ----
    {
      double xo[(12 + NWP - 1) / NWP][2];
      int cnt = 0;
      for (int tile = warp; tile < rt_n * 2; tile += NWP, ++cnt) {
        const int rt = tile >> 1, j0 = (tile & 1) * 8;
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int kk = 0; kk < DB; kk += 4) {
          const int k = kk + (lane & 3);
          const double av = D[k0 + k][rb + 8 * rt + (lane >> 2)];
          const int jn = j0 + (lane >> 2);
          const double bv = k < jn ? D[k0 + jn][k0 + k] : (k == jn ? 1.0 : 0.0);
          dmma(c0, c1, av, bv);
        }
        xo[cnt][0] = c0;
        xo[cnt][1] = c1;
      }
      __syncthreads();
      cnt = 0;
      for (int tile = warp; tile < rt_n * 2; tile += NWP, ++cnt) {
        const int rt = tile >> 1, j0 = (tile & 1) * 8;
        const int r = rb + 8 * rt + (lane >> 2);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j = j0 + 2 * (lane & 3) + h;
          W.X[r - rb][j] = xo[cnt][h];
          D[k0 + j][r] = xo[cnt][h] * rcp_nr(W.dv[k0 + j]);
        }
      }
    }
    __syncthreads();
    // ---- 3. Schur (DMMA): A(r, c) -= sum_j Lu(r, j) X(c, j), rb <= c <= r ----
    {
      const int ntl = rt_n * (rt_n + 1) / 2;
      for (int tile = warp; tile < ntl; tile += NWP) {
        int rt = 0, rem = tile;
        while (rem > rt) {
          rem -= rt + 1;
          ++rt;
        }
        const int ct = rem;  // ct <= rt
        const int r = rb + 8 * rt + (lane >> 2);
        const int cA = rb + 8 * ct + 2 * (lane & 3);
        double c0 = D[cA][r], c1 = D[cA + 1][r];
#pragma unroll
        for (int kk = 0; kk < DB; kk += 4) {
          const int k = kk + (lane & 3);
          const double av = -D[k0 + k][rb + 8 * rt + (lane >> 2)];
          const double bv = W.X[8 * ct + (lane >> 2)][k];
          dmma(c0, c1, av, bv);
        }
        if (r >= cA) D[cA][r] = c0;
        if (r >= cA + 1) D[cA + 1][r] = c1;
      }
    }
    __syncthreads();
  }
  // ---- 4. off-diagonal blocks of M = Lu^-1, block row by block row (DMMA) ----
  for (int bi = 1; bi < nsub && !(ABL & 4); ++bi) {
    // Y_t = sum_{k=16t}^{16bi-1} Lu(16bi + q, k) M(k, 16t + c), t < bi, into W.X[16t + q][c]
    for (int tile = warp; tile < bi * 4; tile += NWP) {
      const int t = tile >> 2, tr = (tile >> 1) & 1, tc = tile & 1;
      const int rowb = bi * DB + 8 * tr, colg = t * DB + 8 * tc + (lane >> 2);
      double c0 = 0.0, c1 = 0.0;
      for (int kk = t * DB; kk < bi * DB; kk += 4) {
        const int k = kk + (lane & 3);
        const double av = D[k][rowb + (lane >> 2)];
        const double bv = k == colg ? 1.0 : (k > colg ? D[k][colg] : 0.0);
        dmma(c0, c1, av, bv);
      }
      const int q = 8 * tr + (lane >> 2), c = 8 * tc + 2 * (lane & 3);
      W.X[t * DB + q][c] = c0;
      W.X[t * DB + q][c + 1] = c1;
    }
    __syncthreads();
    // M(16bi + q, 16t + c) = -sum_{q' <= q} M(16bi + q, 16bi + q') Y_t(q', c)
    for (int tile = warp; tile < bi * 4; tile += NWP) {
      const int t = tile >> 2, tr = (tile >> 1) & 1, tc = tile & 1;
      const int qa = 8 * tr + (lane >> 2);
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < DB; kk += 4) {
        const int k = kk + (lane & 3);
        const double av = k < qa ? -D[bi * DB + qa][bi * DB + k] : (k == qa ? -1.0 : 0.0);
        const double bv = W.X[t * DB + k][8 * tc + (lane >> 2)];
        dmma(c0, c1, av, bv);
      }
      const int row = bi * DB + qa, col = t * DB + 8 * tc + 2 * (lane & 3);
      D[row][col] = c0;
      D[row][col + 1] = c1;
    }
    __syncthreads();
  }
}

// write the factor (reference layout) and the scaled inverse G (FNB x FNB,
// column-major, G(j, k) at G[k * FNB + j]) after factor_block_inv
template <int NT = 128>
__device__ __forceinline__ void store_block_inv(double (*D)[FNB + 1], const double* rdiag,
                                                const DiagWork& W, int nb, bool ldlt,
                                                double* base, i64 ld, int c0, double* G, int tid) {
  constexpr int CP = NT / 64;
  const int r = tid & 63, cpar = tid >> 6;
  for (int c = cpar; c < nb; c += CP) {
    if (r < nb && r >= c) {
      double v;
      if (ldlt) v = D[c][r];                                   // Lu, d on the diagonal
      else if (r == c) v = W.dv[c] * rdiag[c];                 // sqrt(d)
      else v = D[c][r] * (W.dv[c] * rdiag[c]);                 // Lu * sqrt(d)
      base[(i64)(c0 + c) * ld + c0 + r] = v;
    }
  }
  if (!G) return;
  for (int k = cpar; k < FNB; k += CP) {
    const int j = r;
    double gv = 0.0;
    if (j < nb && k < nb && k <= j) gv = (k == j) ? rdiag[j] : D[j][k] * rdiag[j];
    G[(i64)k * FNB + j] = gv;
  }
}

struct DiagSmem {
  double D[FNB][FNB + 1];
  double rdiag[FNB];
  DiagWork W;
  int s_fail;
  double s_fpiv;
};

// wide panel step: diagonal factor + scaled inverse G into scratch slot it.g
template <int NT>
__device__ __forceinline__ void diag_step(DiagSmem& s, const FItem& it, double* store,
                                        double* scratch, bool ldlt, double thr, const PanelDev& P,
                                        i64* fail_col, double* fail_piv, int tid) {
  double* base = store + P.off[it.p];
  const i64 ld = P.nrows[it.p];
  const int nb = it.nb, c0 = it.c0;
  {
    constexpr int CP = NT / FNB;
    const int r = tid & 63, cpar = tid >> 6;
    double v[FNB / CP];
#pragma unroll
    for (int u = 0; u < FNB / CP; ++u) {
      const int c = cpar + CP * u;
      v[u] = (c < nb && r < nb && r >= c) ? __ldcg(base + (i64)(c0 + c) * ld + c0 + r) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < FNB / CP; ++u) s.D[cpar + CP * u][r] = v[u];
  }
  if (tid == 0) s.s_fail = -1;
  __syncthreads();
  factor_block_inv<0, NT>(s.D, s.rdiag, s.W, nb, ldlt, thr, &s.s_fail, &s.s_fpiv, tid);
  store_block_inv<NT>(s.D, s.rdiag, s.W, nb, ldlt, base, ld, c0, scratch + (i64)it.g * FNB * FNB, tid);
  if (tid == 0 && s.s_fail >= 0 && fail_col[it.p] == NO_FAIL) {
    fail_col[it.p] = P.fc[it.p] + c0 + s.s_fail;
    fail_piv[it.p] = s.s_fpiv;
  }
}


// one CTA per wide panel of the level: its 64-column step's diagonal block
#ifndef DIAGB_T
#define DIAGB_T 512  // diagonal-block CTA threads (DMMA phases over 16 warps; 60^3: 128 -> 512 = 21.9 -> 21.3 ms)
#endif
__global__ void __launch_bounds__(DIAGB_T)
k_factor_diag_blk(const FItem* __restrict__ items, const DevArgs* __restrict__ args, PanelDev P,
                  i64* __restrict__ fail_col, double* __restrict__ fail_piv) {
  pdl_wait();  // programmatic dependent launch: wait for the previous grid
  pdl_trigger();  // (not persistent: every CTA of the grid has started)
  __shared__ DiagSmem s;
  diag_step<DIAGB_T>(s, items[blockIdx.x], args->store, args->scratch, args->form == FORM_LDLT,
                   args->thr, P, fail_col, fail_piv, threadIdx.x);
}

}  // namespace ps
