// Scalar-generic numeric kernels: LU (real, complex) and complex LLt / LDLt.
//
// The reference factors only real LLt / LDLt (kernels.py:19-22); the north
// star asks for LLt / LDLt / LU in real and complex double.  These kernels
// run the SAME plan as the tuned real LLt / LDLt kernels (level batches,
// factor items, colored update tiles, block-row index maps, the counters'
// atomics-free ordered scatter); they are templated on the scalar T (double
// or cplx = interleaved complex128) and the form F.  The arithmetic is on the
// FP64 CUDA cores (DFMA: 33.9 TFLOP/s measured vs 37.1 for DMMA on this
// part, profiles/r01_fp64_peak.txt) in register-blocked tiles.
//
// LU storage (oracle/panel_oracle_ext.py): the L slab (the PanelStore
// layout) holds L's strict lower part with U's diagonal on the diagonal; the
// U slab, `ustride` elements further, holds U transposed in the same layout
// (u[r, j] = U[fc + j, row r] for local rows r > j).  The symmetric forms
// have U^T = L (LLt) / L D (LDLt) and no U slab.
//
// Factor of a panel (left-looking sweep of kernels.py:208-247, LU version of
// PAPER.md:321-331), right-looking inside the diagonal block:
//   LLt  : L_jj = sqrt(piv), column scaled by 1 / L_jj
//   LDLt : d_j = piv, column scaled by 1 / d_j (unit L)
//   LU   : U_jj = piv, L column scaled by 1 / U_jj, U row unscaled
// Pivot failure: real LLt piv <= thr; every other case |piv| <= thr
// (first failing column per panel, as the tuned kernels).
// Update tile (kernels.py:128-136, twice for LU):
//   L: C_L[map i, map j] -= sum_k A_L[i,k] (d_k) B[j,k],  B = U^T rows (LU)
//   U: C_U[map i, map j] -= sum_k A_U[i,k] A_L[j,k]      (LU, i > j only)
#pragma once
#include "ps_kernels.cuh"
#include "ps_solve.cuh"

namespace ps {


struct __align__(16) cplx {
  double re, im;
};

// ---- scalar arithmetic ----
__device__ __forceinline__ double s_zero(double) { return 0.0; }
__device__ __forceinline__ cplx s_zero(cplx) { return cplx{0.0, 0.0}; }
__device__ __forceinline__ double s_mul(double a, double b) { return a * b; }
__device__ __forceinline__ cplx s_mul(cplx a, cplx b) {
  return cplx{fma(a.re, b.re, -a.im * b.im), fma(a.re, b.im, a.im * b.re)};
}
// acc += a * b
__device__ __forceinline__ void s_fma(double& acc, double a, double b) { acc = fma(a, b, acc); }
__device__ __forceinline__ void s_fma(cplx& acc, cplx a, cplx b) {
  acc.re = fma(a.re, b.re, acc.re);
  acc.re = fma(-a.im, b.im, acc.re);
  acc.im = fma(a.re, b.im, acc.im);
  acc.im = fma(a.im, b.re, acc.im);
}
// acc -= a * b
__device__ __forceinline__ void s_fms(double& acc, double a, double b) { acc = fma(-a, b, acc); }
__device__ __forceinline__ void s_fms(cplx& acc, cplx a, cplx b) {
  acc.re = fma(-a.re, b.re, acc.re);
  acc.re = fma(a.im, b.im, acc.re);
  acc.im = fma(-a.re, b.im, acc.im);
  acc.im = fma(-a.im, b.re, acc.im);
}
__device__ __forceinline__ double s_sub(double a, double b) { return a - b; }
__device__ __forceinline__ cplx s_sub(cplx a, cplx b) { return cplx{a.re - b.re, a.im - b.im}; }
__device__ __forceinline__ double s_div(double a, double b) { return a / b; }
__device__ __forceinline__ cplx s_div(cplx a, cplx b) {
  // Smith's algorithm (no overflow for |b| near the range limits)
  if (fabs(b.re) >= fabs(b.im)) {
    const double r = b.im / b.re, d = b.re + b.im * r;
    return cplx{(a.re + a.im * r) / d, (a.im - a.re * r) / d};
  }
  const double r = b.re / b.im, d = b.re * r + b.im;
  return cplx{(a.re * r + a.im) / d, (a.im * r - a.re) / d};
}
__device__ __forceinline__ double s_sqrt(double a) { return sqrt(a); }
__device__ __forceinline__ cplx s_sqrt(cplx a) {  // principal branch
  const double m = hypot(a.re, a.im);
  double re = sqrt(0.5 * (m + fabs(a.re)));
  double im = re > 0.0 ? 0.5 * a.im / re : 0.0;
  if (a.re < 0.0) {
    const double t = fabs(im);
    im = a.im < 0.0 ? -re : re;
    re = t;
  }
  return cplx{re, im};
}
__device__ __forceinline__ double s_abs(double a) { return fabs(a); }
__device__ __forceinline__ double s_abs(cplx a) { return hypot(a.re, a.im); }
template <class T>
__device__ __forceinline__ bool s_is_real(T) { return sizeof(T) == sizeof(double); }
// the reference's failure predicate, extended to complex and LU
template <class T, int F>
__device__ __forceinline__ bool s_bad(T piv, double thr) {
  if constexpr (sizeof(T) == sizeof(double)) {
    if (F == FORM_LLT) return piv <= thr;
    return fabs(piv) <= thr;
  } else {
    return s_abs(piv) <= thr;
  }
}
template <class T>
__device__ __forceinline__ double s_report(T piv) {  // pivot value in the status record
  if constexpr (sizeof(T) == sizeof(double)) return piv;
  else return s_abs(piv);
}
__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }
__device__ __forceinline__ cplx ldcg(const cplx* p) {
  const double2 v = __ldcg(reinterpret_cast<const double2*>(p));
  return cplx{v.x, v.y};
}
__device__ __forceinline__ void stcg(double* p, double v) { __stcg(p, v); }
__device__ __forceinline__ void stcg(cplx* p, cplx v) {
  __stcg(reinterpret_cast<double2*>(p), make_double2(v.re, v.im));
}

template <class T>
__device__ __forceinline__ T* slab(const DevArgs* a) { return reinterpret_cast<T*>(a->store); }

__device__ __forceinline__ void record_fail(i64* fail_col, double* fail_piv, int p, i64 col,
                                            double piv) {
  if (fail_col[p] == NO_FAIL || col < fail_col[p]) {
    fail_col[p] = col;
    fail_piv[p] = piv;
  }
}

// ---------------------------------------------------------------------------
// width-1 panels: a warp per panel (kernels.py:216-221, 232-239)
template <class T, int F>
__global__ void g_factor_w1(const int* __restrict__ plist, int count, const DevArgs* __restrict__ args,
                            PanelDev P, i64* __restrict__ fail_col, double* __restrict__ fail_piv) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  T* store = slab<T>(args);
  for (int i = gw; i < count; i += nw) {
    const int p = plist[i];
    T* a = store + P.off[p];
    const int nr = P.nrows[p];
    const T piv = a[0];
    __syncwarp();
    const T dv = F == FORM_LLT ? s_sqrt(piv) : piv;
    for (int r = 1 + lane; r < nr; r += 32) a[r] = s_div(a[r], dv);
    if (lane == 0) {
      a[0] = dv;
      if (s_bad<T, F>(piv, args->thr)) record_fail(fail_col, fail_piv, p, P.fc[p], s_report(piv));
    }
  }
}

// ---------------------------------------------------------------------------
// dense factor of an nb x nb diagonal block in shared memory (nb <= NBM),
// right-looking, two barriers per pivot.  D[c][r] = M(r, c) for r >= c;
// LU: E[c][r] = U(c, r) for r > c (the strict upper part, from the U slab).
template <class T, int F, int NBM>
__device__ void block_factor_blocked(T (*D)[NBM + 1], T (*E)[NBM + 1], int nb, double thr,
                                     int* s_fail, T* s_fpiv, int tid, int nt) {
  // Right-looking over 16-column sub-blocks, on the unscaled Schur
  // complements M (D: lower part, column-major; E: LU's strict upper part,
  // row-major).  Every entry receives exactly the pivot-by-pivot updates
  // M(i,c) -= (M(i,j) / piv_j) M(j,c), in pivot order, of the plain sweep -
  // bitwise the same result - with 3 barriers per sub-block instead of 2 per
  // pivot:
  //   1. warp 0: the 16 x 16 diagonal sub-block, pivot by pivot in registers
  //   2. the rows below (their multipliers l = M / piv, kept in lm) and, LU,
  //      the U rows right of the sub-block, thread per row / column
  //   3. the trailing entries: M(i,c) -= sum_j lm(i,j) M(j,c), j ascending
  // then every column is scaled by its pivot (LLt sqrt) once.
  constexpr int SB = 16;
  __shared__ T lm[NBM][SB + 1];
  __shared__ T pv[NBM];
  __shared__ T wv[SB + 1];  // warp-0 broadcast: pivot row (LU) / column (LLt, LDLt) values
  const int lane = tid & 31;
  for (int k0 = 0; k0 < nb; k0 += SB) {
    const int kb = min(SB, nb - k0), rb = k0 + kb;
    // ---- 1. the diagonal sub-block (warp 0; lane = row k0 + lane) ----
    if (tid < 32) {
      T a[SB];
      const int i = lane;
#pragma unroll
      for (int c = 0; c < SB; ++c) {
        a[c] = s_zero(T{});
        if (i < kb && c < kb) {
          if (c <= i) a[c] = D[k0 + c][k0 + i];
          else if (F == FORM_LU) a[c] = E[k0 + i][k0 + c];
        }
      }
#pragma unroll
      for (int j = 0; j < SB; ++j) {
        if (j < kb) {
          if (i == j) pv[k0 + j] = a[j];
          if (F == FORM_LU) {
            if (i == j)
#pragma unroll
              for (int c = 0; c < SB; ++c) wv[c] = a[c];
          } else if (i < kb) {
            wv[i] = a[j];  // column j: M(i, j)
          }
          __syncwarp();
          const T piv = pv[k0 + j];
          if (i == 0 && *s_fail < 0 && s_bad<T, F>(piv, thr)) {
            *s_fail = k0 + j;
            *s_fpiv = piv;
          }
          if (i > j && i < kb) {
            const T l = s_div(a[j], piv);
            lm[k0 + i][j] = l;
#pragma unroll
            for (int c = 0; c < SB; ++c) {
              if (c > j && c < kb) {
                if (F == FORM_LU) s_fms(a[c], l, wv[c]);      // M(j, c): row j
                else if (c <= i) s_fms(a[c], l, wv[c]);       // M(c, j) = M(j, c)
              }
            }
          }
          __syncwarp();
        }
      }
      if (i < kb) {
#pragma unroll
        for (int c = 0; c < SB; ++c) {
          if (c < kb) {
            if (c <= i) D[k0 + c][k0 + i] = a[c];
            else if (F == FORM_LU) E[k0 + i][k0 + c] = a[c];
          }
        }
      }
    }
    __syncthreads();
    // ---- 2a. rows below the sub-block: column values and multipliers ----
    for (int i = rb + tid; i < nb; i += nt) {
      T x[SB];
#pragma unroll
      for (int j = 0; j < SB; ++j) x[j] = j < kb ? D[k0 + j][i] : s_zero(T{});
#pragma unroll
      for (int j = 0; j < SB; ++j) {
        if (j < kb) {
          const T l = s_div(x[j], pv[k0 + j]);
          lm[i][j] = l;
#pragma unroll
          for (int jj = j + 1; jj < SB; ++jj)
            if (jj < kb) s_fms(x[jj], l, F == FORM_LU ? E[k0 + j][k0 + jj] : D[k0 + j][k0 + jj]);
        }
      }
#pragma unroll
      for (int j = 0; j < SB; ++j)
        if (j < kb) D[k0 + j][i] = x[j];
    }
    // ---- 2b. LU: the sub-block's U rows right of it ----
    if (F == FORM_LU) {
      for (int c = rb + tid; c < nb; c += nt) {
        T y[SB];
#pragma unroll
        for (int j = 0; j < SB; ++j) y[j] = j < kb ? E[k0 + j][c] : s_zero(T{});
#pragma unroll
        for (int j = 0; j < SB; ++j)
#pragma unroll
          for (int jj = j + 1; jj < SB; ++jj)
            if (jj < kb) s_fms(y[jj], lm[k0 + jj][j], y[j]);
#pragma unroll
        for (int j = 0; j < SB; ++j)
          if (j < kb) E[k0 + j][c] = y[j];
      }
    }
    __syncthreads();
    // ---- 3. trailing entries (16-wide thread grid) ----
    {
      const int tx = tid & 15, ty = tid >> 4, ny = nt >> 4;
      for (int c = rb + ty; c < nb; c += ny) {
        for (int i = rb + tx; i < nb; i += 16) {
          if (i >= c) {
            T acc = D[c][i];
            for (int j = 0; j < kb; ++j)
              s_fms(acc, lm[i][j], F == FORM_LU ? E[k0 + j][c] : D[k0 + j][c]);
            D[c][i] = acc;
          } else if (F == FORM_LU) {
            T acc = E[i][c];
            for (int j = 0; j < kb; ++j) s_fms(acc, lm[i][j], E[k0 + j][c]);
            E[i][c] = acc;
          }
        }
      }
    }
    __syncthreads();
  }
  // ---- final scaling: L = M / dv (LLt: dv = sqrt(piv)) ----
  for (int e = tid; e < nb * nb; e += nt) {
    const int j = e / nb, i = e % nb;
    if (i >= j) {
      const T dv = F == FORM_LLT ? s_sqrt(pv[j]) : pv[j];
      D[j][i] = i == j ? dv : s_div(D[j][i], dv);
    }
  }
  __syncthreads();
}

template <class T, int F, int NBM>
__device__ void block_factor_pivots(T (*D)[NBM + 1], T (*E)[NBM + 1], int nb, double thr, int* s_fail,
                             T* s_fpiv, int tid, int nt) {
  // per pivot: the scaled column l_i = M(i, j) / piv once (not once per
  // trailing entry), the trailing update on a 16-wide thread grid (no index
  // division), and column j's final scaling folded into the next pivot's
  // first pass; every entry sees the same operations in the same order as
  // the plain right-looking sweep
  __shared__ T lcol[NBM];
  const int tx = tid & 15, ty = tid >> 4, ny = nt >> 4;
  T dv_prev = s_zero(T{});
  for (int j = 0; j < nb; ++j) {
    const T piv = D[j][j];
    const T dv = F == FORM_LLT ? s_sqrt(piv) : piv;
    if (tid == 0 && *s_fail < 0 && s_bad<T, F>(piv, thr)) {
      *s_fail = j;
      *s_fpiv = piv;
    }
    for (int i = j + 1 + tid; i < nb; i += nt) lcol[i] = s_div(D[j][i], piv);
    if (j > 0) {  // column j - 1: L = M / dv (its trailing update is done)
      for (int i = j + tid; i < nb; i += nt) D[j - 1][i] = s_div(D[j - 1][i], dv_prev);
      if (tid == 0) D[j - 1][j - 1] = dv_prev;
    }
    __syncthreads();
    // trailing update with the unscaled column: M(i,c) -= M(i,j) M(j,c) / piv
    for (int c = j + 1 + ty; c < nb; c += ny) {
      for (int i = j + 1 + tx; i < nb; i += 16) {
        if (i >= c) {
          const T u = F == FORM_LU ? E[j][c] : D[j][c];  // M(j, c)
          s_fms(D[c][i], lcol[i], u);
        } else if (F == FORM_LU) {  // strict upper (i < c): U(i, c) -= L(i, j) U(j, c)
          s_fms(E[i][c], lcol[i], E[j][c]);
        }
      }
    }
    __syncthreads();
    dv_prev = dv;
  }
  if (nb > 0) {  // the last column (no rows below)
    if (tid == 0) D[nb - 1][nb - 1] = dv_prev;
    __syncthreads();
  }
}

// real forms: the sub-blocked factor (fewer barriers); complex: the
// pivot-by-pivot sweep (its 4x heavier entries keep more threads busy per
// barrier - 1% faster at 80^3 complex LU).  Bitwise the same results.
template <class T, int F, int NBM>
__device__ __forceinline__ void block_factor(T (*D)[NBM + 1], T (*E)[NBM + 1], int nb, double thr,
                                             int* s_fail, T* s_fpiv, int tid, int nt) {
  if constexpr (sizeof(T) == sizeof(double))
    block_factor_blocked<T, F, NBM>(D, E, nb, thr, s_fail, s_fpiv, tid, nt);
  else
    block_factor_pivots<T, F, NBM>(D, E, nb, thr, s_fail, s_fpiv, tid, nt);
}

// TRSM of one row (x in registers, nb <= NBM) against the factored block:
//   L rows:  LLt x L^T = b ; LDLt x D L^T = b ; LU x U = b
//   U rows (LU, ut): y L^T = b (unit L)
template <class T, int F, int NBM>
__device__ __forceinline__ void row_solve(T* x, const T (*D)[NBM + 1], const T (*E)[NBM + 1], int nb,
                                          bool ut) {
#pragma unroll
  for (int j = 0; j < NBM; ++j) {
    if (j < nb) {
      const T t = x[j];
      T xj = t;
      if (!ut) xj = s_div(t, D[j][j]);
      x[j] = xj;
#pragma unroll
      for (int k = j + 1; k < NBM; ++k) {
        if (k < nb) {
          if (ut) s_fms(x[k], t, D[j][k]);              // L(k, j)
          else if (F == FORM_LU) s_fms(x[k], xj, E[j][k]);  // U(j, k)
          else if (F == FORM_LDLT) s_fms(x[k], t, D[j][k]);  // d_j x_j L(k, j) = t L(k, j)
          else s_fms(x[k], xj, D[j][k]);               // LLt: L(k, j)
        }
      }
    }
  }
}

// small panels (width 2..SNB): diagonal item (factor + first rows) or a
// TRSM-only row item, 128 threads (the plan's FItem, as k_factor_small)
template <class T, int F>
__global__ void __launch_bounds__(FTR)
g_factor_small(const FItem* __restrict__ items, const DevArgs* __restrict__ args, PanelDev P,
               i64* __restrict__ fail_col, double* __restrict__ fail_piv) {
  pdl_wait();
  pdl_trigger();
  __shared__ T D[SNB][SNB + 1];
  __shared__ T E[F == FORM_LU ? SNB : 1][SNB + 1];
  __shared__ int s_fail;
  __shared__ T s_fpiv;
  const FItem it = items[blockIdx.x];
  const int tid = threadIdx.x;
  T* a = slab<T>(args) + P.off[it.p];
  T* u = a + args->ustride;
  const i64 ld = P.nrows[it.p];
  const int nb = it.nb, c0 = it.c0;
  for (int e = tid; e < nb * nb; e += FTR) {
    const int c = e / nb, r = e % nb;
    if (r >= c) D[c][r] = a[(i64)(c0 + c) * ld + c0 + r];
    if (F == FORM_LU && r > c) E[c][r] = u[(i64)(c0 + c) * ld + c0 + r];  // U(c, r) = u[r, c]
  }
  if (tid == 0) s_fail = -1;
  __syncthreads();
  if (it.diag) {
    block_factor<T, F, SNB>(D, (T(*)[SNB + 1])E, nb, args->thr, &s_fail, &s_fpiv, tid, FTR);
    for (int e = tid; e < nb * nb; e += FTR) {
      const int c = e / nb, r = e % nb;
      if (r >= c) a[(i64)(c0 + c) * ld + c0 + r] = D[c][r];
      if (F == FORM_LU && r > c) u[(i64)(c0 + c) * ld + c0 + r] = E[c][r];
    }
    if (tid == 0 && s_fail >= 0)
      record_fail(fail_col, fail_piv, it.p, P.fc[it.p] + c0 + s_fail, s_report(s_fpiv));
  }
  if (it.nr == 0) return;
  __syncthreads();
  const int nrow = F == FORM_LU ? 2 * it.nr : it.nr;
  for (int rr = tid; rr < nrow; rr += FTR) {
    const bool ut = rr >= it.nr;
    T* rowp = (ut ? u : a) + it.r0 + (ut ? rr - it.nr : rr);
    T x[SNB];
#pragma unroll
    for (int k = 0; k < SNB; ++k)
      if (k < nb) x[k] = rowp[(i64)(c0 + k) * ld];
    row_solve<T, F, SNB>(x, D, (const T(*)[SNB + 1])E, nb, ut);
#pragma unroll
    for (int k = 0; k < SNB; ++k)
      if (k < nb) rowp[(i64)(c0 + k) * ld] = x[k];
  }
}

// ---------------------------------------------------------------------------
// wide panels, one 64-column step: factor the diagonal block and store the
// TRSM operators in scratch slot it.g (row-major FNB x FNB each):
//   G0[j][k]: X = B G0^T solves the L rows  (LLt L^-1; LDLt D^-1 L^-1; LU U^-T)
//   G1[j][k]: Y = B G1^T solves the U rows  (LU: L^-1, unit)
template <class T, int F>
struct GDiagSmem {
  T D[FNB][FNB + 1];
  T E[F == FORM_LU ? FNB : 1][FNB + 1];
  T Z[FNB][FNB + 1];
  int s_fail;
  T s_fpiv;
};
constexpr int GD_THREADS = 256;

// Z = inverse of the unit / non-unit lower triangle of D (column-major
// D[c][r]), right-looking: rows of Z finalized one at a time
// Z = L^-1 (unit or not) over 16-row sub-blocks: A) the sub-block's rows,
// column per thread (forward substitution inside the sub-block), B) the rows
// below, 16-wide thread grid.  Per entry the operations and order of the
// row-by-row sweep (Z[i][c] -= L(i, j) Z[j][c], j ascending; row j divided
// by L(j, j) before it is used): bitwise the same, 2 barriers per sub-block.
template <class T, int NBM>
__device__ void lower_inverse_blocked(const T (*D)[NBM + 1], T (*Z)[NBM + 1], int nb, bool unit,
                                      int tid, int nt) {
  // Z[r][c], solve L Z = I
  for (int e = tid; e < NBM * NBM; e += nt) {
    const int r = e / NBM, c = e % NBM;
    T v = s_zero(T{});
    if (r == c && r < nb) {
      if constexpr (sizeof(T) == sizeof(double)) v = 1.0;
      else v = T{1.0, 0.0};
    }
    Z[r][c] = v;
  }
  __syncthreads();
  constexpr int SB = 16;
  const int tx = tid & 15, ty = tid >> 4, ny = nt >> 4;
  for (int k0 = 0; k0 < nb; k0 += SB) {
    const int kb = min(SB, nb - k0), rb = k0 + kb;
    for (int c = tid; c < rb; c += nt) {  // A
      T y[SB];
#pragma unroll
      for (int j = 0; j < SB; ++j) y[j] = j < kb ? Z[k0 + j][c] : s_zero(T{});
#pragma unroll
      for (int j = 0; j < SB; ++j) {
        if (j < kb && c <= k0 + j) {
          if (!unit) y[j] = s_div(y[j], D[k0 + j][k0 + j]);
#pragma unroll
          for (int jj = j + 1; jj < SB; ++jj)
            if (jj < kb) s_fms(y[jj], D[k0 + j][k0 + jj], y[j]);
        }
      }
#pragma unroll
      for (int j = 0; j < SB; ++j)
        if (j < kb) Z[k0 + j][c] = y[j];
    }
    __syncthreads();
    for (int c = ty; c < rb; c += ny)  // B
      for (int i = rb + tx; i < nb; i += 16) {
        T acc = Z[i][c];
        for (int j = 0; j < kb; ++j)
          if (c <= k0 + j) s_fms(acc, D[k0 + j][i], Z[k0 + j][c]);
        Z[i][c] = acc;
      }
    __syncthreads();
  }
}

template <class T, int NBM>
__device__ void lower_inverse_rows(const T (*D)[NBM + 1], T (*Z)[NBM + 1], int nb, bool unit, int tid,
                              int nt) {
  // Z[r][c], solve L Z = I
  for (int e = tid; e < NBM * NBM; e += nt) {
    const int r = e / NBM, c = e % NBM;
    T v = s_zero(T{});
    if (r == c && r < nb) {
      if constexpr (sizeof(T) == sizeof(double)) v = 1.0;
      else v = T{1.0, 0.0};
    }
    Z[r][c] = v;
  }
  __syncthreads();
  const int tx = tid & 15, ty = tid >> 4, ny = nt >> 4;
  for (int j = 0; j < nb; ++j) {
    if (!unit)
      for (int c = tid; c <= j; c += nt) Z[j][c] = s_div(Z[j][c], D[j][j]);
    __syncthreads();
    for (int c = ty; c <= j; c += ny)
      for (int i = j + 1 + tx; i < nb; i += 16) s_fms(Z[i][c], D[j][i], Z[j][c]);
    __syncthreads();
  }
}
template <class T, int NBM>
__device__ __forceinline__ void lower_inverse(const T (*D)[NBM + 1], T (*Z)[NBM + 1], int nb,
                                              bool unit, int tid, int nt) {
  if constexpr (sizeof(T) == sizeof(double)) lower_inverse_blocked<T, NBM>(D, Z, nb, unit, tid, nt);
  else lower_inverse_rows<T, NBM>(D, Z, nb, unit, tid, nt);
}

template <class T, int F>
__global__ void __launch_bounds__(GD_THREADS)
g_factor_diag(const FItem* __restrict__ items, const DevArgs* __restrict__ args, PanelDev P,
              i64* __restrict__ fail_col, double* __restrict__ fail_piv) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char gsm_raw[];
  GDiagSmem<T, F>& s = *reinterpret_cast<GDiagSmem<T, F>*>(gsm_raw);
  const FItem it = items[blockIdx.x];
  const int tid = threadIdx.x;
  T* a = slab<T>(args) + P.off[it.p];
  T* u = a + args->ustride;
  const i64 ld = P.nrows[it.p];
  const int nb = it.nb, c0 = it.c0;
  for (int e = tid; e < nb * nb; e += GD_THREADS) {
    const int c = e / nb, r = e % nb;
    if (r >= c) s.D[c][r] = ldcg(a + (i64)(c0 + c) * ld + c0 + r);
    if (F == FORM_LU && r > c) s.E[c][r] = ldcg(u + (i64)(c0 + c) * ld + c0 + r);
  }
  if (tid == 0) s.s_fail = -1;
  __syncthreads();
  block_factor<T, F, FNB>(s.D, (T(*)[FNB + 1])s.E, nb, args->thr, &s.s_fail, &s.s_fpiv, tid,
                          GD_THREADS);
  for (int e = tid; e < nb * nb; e += GD_THREADS) {
    const int c = e / nb, r = e % nb;
    if (r >= c) a[(i64)(c0 + c) * ld + c0 + r] = s.D[c][r];
    if (F == FORM_LU && r > c) u[(i64)(c0 + c) * ld + c0 + r] = s.E[c][r];
  }
  if (tid == 0 && s.s_fail >= 0)
    record_fail(fail_col, fail_piv, it.p, P.fc[it.p] + c0 + s.s_fail, s_report(s.s_fpiv));
  T* G = reinterpret_cast<T*>(args->scratch) + (i64)it.g * (F == FORM_LU ? 2 : 1) * FNB * FNB;
  __syncthreads();
  if (F == FORM_LU) {
    // G1 = L^-1 (unit), while D still holds L
    lower_inverse<T, FNB>((const T(*)[FNB + 1])s.D, s.Z, nb, true, tid, GD_THREADS);
    for (int e = tid; e < FNB * FNB; e += GD_THREADS)  // column-major: G1(j, k) at k FNB + j
      G[FNB * FNB + e] = s.Z[e % FNB][e / FNB];
    __syncthreads();
    // then D's strict lower part := U^T (U^T(r, c) = U(c, r) = E[c][r]); the
    // diagonal already holds U's
    for (int e = tid; e < FNB * FNB; e += GD_THREADS) {
      const int c = e / FNB, r = e % FNB;
      if (r > c) s.D[c][r] = s.E[c][r];
    }
    __syncthreads();
  }
  // G0 (LLt: L^-1; LDLt: D^-1 L^-1; LU: (U^T)^-1 = U^-T)
  lower_inverse<T, FNB>((const T(*)[FNB + 1])s.D, s.Z, nb, F == FORM_LDLT, tid, GD_THREADS);
  for (int e = tid; e < FNB * FNB; e += GD_THREADS) {  // column-major: G(j, k) at k FNB + j
    const int j = e % FNB, k = e / FNB;
    T v = s.Z[j][k];
    if (F == FORM_LDLT && j < nb) v = s_div(v, s.D[j][j]);
    G[e] = v;
  }
}

// wide-panel TRSM tile: rows [r0, r0 + nr) (nr <= 64) x the step's columns,
// X = B G^T in place (L rows; and U rows with G1 for LU).  G (and G1) are
// column-major FNB x FNB, the layout k_trsm8 reads (real LU runs its TRSM
// on k_trsm8).  256 threads:
// thread (row r = tid % 64, 16 columns from (tid / 64) * 16).
template <class T>
struct GTrsmSmem {
  T G[FNB][FNB + 1];
  T B[FNB][FNB + 1];  // B[k][r]
};
template <class T, int F>
__global__ void __launch_bounds__(GD_THREADS)
g_trsm(const FItem* __restrict__ items, const DevArgs* __restrict__ args, PanelDev P) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char gsm_raw[];
  GTrsmSmem<T>& s = *reinterpret_cast<GTrsmSmem<T>*>(gsm_raw);
  const FItem it = items[blockIdx.x];
  const int tid = threadIdx.x;
  const i64 ld = P.nrows[it.p];
  const int nb = it.nb, c0 = it.c0;
  const int r = tid & 63, jg = (tid >> 6) * 16;
  const T* Gb = reinterpret_cast<const T*>(args->scratch) + (i64)it.g * (F == FORM_LU ? 2 : 1) * FNB * FNB;
  for (int pass = 0; pass < (F == FORM_LU ? 2 : 1); ++pass) {
    T* base = slab<T>(args) + P.off[it.p] + (pass ? args->ustride : 0) + (i64)c0 * ld + it.r0;
    const T* G = Gb + pass * FNB * FNB;
    for (int e = tid; e < FNB * FNB; e += GD_THREADS) s.G[e % FNB][e / FNB] = G[e];
    for (int e = tid; e < nb * FNB; e += GD_THREADS) {
      const int k = e / FNB, rr = e % FNB;
      s.B[k][rr] = rr < it.nr ? ldcg(base + (i64)k * ld + rr) : s_zero(T{});
    }
    __syncthreads();
    T acc[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) acc[q] = s_zero(T{});
    for (int k = 0; k < nb; ++k) {
      const T b = s.B[k][r];
#pragma unroll
      for (int q = 0; q < 16; ++q) s_fma(acc[q], b, s.G[jg + q][k]);
    }
    if (r < it.nr) {
#pragma unroll
      for (int q = 0; q < 16; ++q)
        if (jg + q < nb) base[(i64)(jg + q) * ld + r] = acc[q];
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// update tile (inter-panel couples with the run maps, or intra-panel
// trailing tiles with couple = -1), persistent CTAs taking tiles in list
// order, colored wait / signal as k_update.  256 threads, 4 x 4 register
// block per thread (rows 4 tr.., columns 4 tc..), K in chunks of 16.
constexpr int GU_THREADS = 256, GU_KC = 16;
template <class T>
struct GUpdSmem {
  T A[GU_KC][TM + 1];
  T B[GU_KC][TN + 1];
  int rmap[TM];
  int cmap[TN];
  int wsrc[2][TM];
  int wdst[2][TM];
  int tile;
};

// seg != nullptr: a merged chain tile (ChainSeg, ps_kernels.cuh): the
// operand pointers move to the next piece at its first chunk
template <class T, int F>
__device__ __forceinline__ void gu_mainloop(GUpdSmem<T>& sm, const T* A, const T* B, const T* D,
                                            i64 lds, const UTile& Tl, T acc[4][4], int tid,
                                            const ChainSeg* seg) {
  const int tr = tid & 15, tc = tid >> 4;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = s_zero(T{});
  A += (i64)Tl.k0 * lds;
  B += (i64)Tl.k0 * lds;
  D += (i64)Tl.k0 * (lds + 1);
  i64 ld = lds, ldb = lds, dstr = lds + 1;
  int knext = seg ? 0 : INT_MAX;
  for (int k0 = 0; k0 < Tl.kn; k0 += GU_KC) {
    const int kk = min(GU_KC, Tl.kn - k0);
    chain_advance(seg, knext, k0, A, B, D, ld, ldb, dstr);
    const T* Ac = A + (i64)k0 * ld;
    const T* Bc = B + (i64)k0 * ld;
    const T* Dc = D + (i64)k0 * dstr;
    const int i0 = Tl.i0, j0 = Tl.j0;
    for (int e = tid; e < GU_KC * TM; e += GU_THREADS) {
      const int k = e / TM, r = e % TM;
      T av = s_zero(T{}), bv = s_zero(T{});
      if (k < kk) {
        const i64 col = (i64)k * ld;
        if (r < Tl.ni) av = ldcg(Ac + col + i0 + r);
        if (r < Tl.nj) {
          bv = ldcg(Bc + col + j0 + r);
          if (F == FORM_LDLT) bv = s_mul(bv, ldcg(Dc + (i64)k * dstr));
        }
      }
      sm.A[k][r] = av;
      sm.B[k][r] = bv;
    }
    __syncthreads();
    for (int k = 0; k < kk; ++k) {
      T a4[4], b4[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a4[q] = sm.A[k][tr * 4 + q];
        b4[q] = sm.B[k][tc * 4 + q];
      }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) s_fma(acc[x][y], a4[x], b4[y]);
    }
    __syncthreads();
  }
}

template <class T, int F>
__global__ void __launch_bounds__(GU_THREADS)
g_update(const UTile* __restrict__ tiles, int ntiles, int* __restrict__ work_ctr,
         unsigned* __restrict__ counters, const DevArgs* __restrict__ args,
         const i64* __restrict__ run_ptr, const int* __restrict__ run_src,
         const int* __restrict__ run_dst) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char gsm_raw[];
  GUpdSmem<T>& sm = *reinterpret_cast<GUpdSmem<T>*>(gsm_raw);
  const int tid = threadIdx.x;
  const int tr = tid & 15, tc = tid >> 4;
  T* store = slab<T>(args);
  const i64 us = args->ustride;
  while (true) {
    if (tid == 0) sm.tile = atomicAdd(work_ctr, 1);
    __syncthreads();
    const int t = sm.tile;
    if (t >= ntiles) {
      pdl_trigger();
      break;
    }
    const UTile Tl = tiles[t];
    if (tid < 128) maps_load(sm, Tl.couple, Tl.ri, Tl.rj, run_ptr, run_src, run_dst, tid);
    __syncthreads();
    if (tid < 128) maps_search(sm, Tl.couple, Tl.i0, Tl.ni, Tl.j0, Tl.nj, tid);
    const T* srcL = store + Tl.soff;
    for (int pass = 0; pass < (F == FORM_LU ? 2 : 1); ++pass) {
      // pass 0: L rows x (U^T | L | D L) rows into the L slab (i >= j);
      // pass 1 (LU): U^T rows x L rows into the U slab (i > j)
      const T* A = pass ? srcL + us : srcL;
      const T* B = F == FORM_LU ? (pass ? srcL : srcL + us) : srcL;
      T acc[4][4];
      gu_mainloop<T, F>(sm, A, B, srcL, Tl.lds, Tl, acc, tid, chain_of(args, Tl));
      if (pass == 0 && Tl.wait >= 0 && tid == 0) {
        while (ld_acquire(&counters[Tl.dst]) < (unsigned)Tl.wait) __nanosleep(32);
      }
      __syncthreads();
      T* dst = store + Tl.doff + (pass ? us : 0);
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        const int j = tc * 4 + y;
        if (j >= Tl.nj) continue;
        const i64 dc = (i64)sm.cmap[j] * Tl.ldd;
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          const int i = tr * 4 + x;
          const int gi = Tl.i0 + i, gj = Tl.j0 + j;
          if (i < Tl.ni && (pass ? gi > gj : gi >= gj)) {
            T* pp = dst + dc + sm.rmap[i];
            T v = ldcg(pp);
            v = s_sub(v, acc[x][y]);
            stcg(pp, v);
          }
        }
      }
    }
    __syncthreads();
    if (Tl.signal && tid == 0) {
      signal_add(&counters[Tl.dst]);
    }
  }
}

// device assembly of any form / scalar: store[pos[k]] = vals[k] (pos < 0 skipped)
template <class T>
__global__ void g_assemble(T* __restrict__ store, const i64* __restrict__ pos,
                           const T* __restrict__ vals, i64 n) {
  for (i64 k = blockIdx.x * (i64)blockDim.x + threadIdx.x; k < n; k += (i64)gridDim.x * blockDim.x) {
    const i64 p = pos[k];
    if (p >= 0) store[p] = vals[k];
  }
}

// ---------------------------------------------------------------------------
// triangular solve (the plan's virtual panels, ps_solve.cuh layout), all
// forms: forward L y = b (unit for LDLt / LU), x /= diag (LDLt: d; LU: U's
// diagonal), backward with T = L (LLt / LDLt) or the U slab (LU; its
// off-diagonal products scaled by 1 / U_jj: U = D_U * unit upper).
constexpr int GS_THREADS = 256;

template <class T>
__global__ void __launch_bounds__(GS_THREADS)
gs_freduce(i64 first, int count, SolveDev S, T* x, const T* __restrict__ fpart) {
  const int k = blockIdx.x * GS_THREADS + threadIdx.x;
  const int item = k >> 3;
  if (item >= count) return;
  const int2 it = S.ritems[first + item];
  const int j = it.y + (k & 7);
  if (j >= S.w[it.x]) return;
  const i64 gj = S.fc[it.x] + j;
  T v = s_zero(T{});
  for (i64 e = S.jptr[gj]; e < S.jptr[gj + 1]; ++e) {
    const T f = ldcg(fpart + S.jidx[e]);
    if constexpr (sizeof(T) == sizeof(double)) v += f;
    else v = cplx{v.re + f.re, v.im + f.im};
  }
  x[gj] = s_sub(x[gj], v);
}

template <class T, int F>
__global__ void __launch_bounds__(GS_THREADS)
gs_fdiag(i64 first, SolveDev S, const T* __restrict__ store, T* x) {
  extern __shared__ __align__(16) unsigned char gsm_raw[];
  T* y = reinterpret_cast<T*>(gsm_raw);
  const int tid = threadIdx.x;
  const int v = S.lvl_panels[first + blockIdx.x];
  const int w = S.w[v];
  const i64 fc = S.fc[v], ld = S.ld[v];
  const T* a = store + S.off[v];
  for (int j = tid; j < w; j += GS_THREADS) y[j] = x[fc + j];
  __syncthreads();
  for (int j = 0; j < w; ++j) {
    T yj = y[j];
    if (F == FORM_LLT) yj = s_div(yj, a[(i64)j * ld + j]);
    __syncthreads();
    if (tid == 0) y[j] = yj;
    for (int i = j + 1 + tid; i < w; i += GS_THREADS) s_fms(y[i], a[(i64)j * ld + i], yj);
    __syncthreads();
  }
  for (int j = tid; j < w; j += GS_THREADS) x[fc + j] = y[j];
}

template <class T>
__global__ void __launch_bounds__(GS_THREADS)
gs_fgemv(i64 first, SolveDev S, const T* __restrict__ store, const T* __restrict__ z, T* fpart) {
  const int4 it = S.fitems[first + blockIdx.x];
  const int v = it.x, r0 = it.y, k0 = it.z;
  const int w = S.w[v], nro = S.nro[v];
  const i64 ld = S.ld[v];
  const int kn = min(SV_KC, w - k0);
  for (int r = threadIdx.x; r < SV_FR; r += GS_THREADS) {
    if (r0 + r >= nro) continue;
    const T* a = store + S.off[v] + (i64)k0 * ld + w + r0 + r;
    const T* zz = z + S.fc[v] + k0;
    T s = s_zero(T{});
    for (int k = 0; k < kn; ++k) s_fma(s, ldcg(a + (i64)k * ld), ldcg(zz + k));
    fpart[S.fbase[v] + (i64)(k0 / SV_KC) * nro + r0 + r] = s;
  }
}

// x[j] /= diag(j) over every column (LDLt d_j, LU U_jj), virtual panel per CTA
template <class T>
__global__ void __launch_bounds__(GS_THREADS)
gs_scale(int nv, SolveDev S, const T* __restrict__ store, T* x) {
  for (int v = blockIdx.x; v < nv; v += gridDim.x) {
    const int w = S.w[v];
    const i64 ld = S.ld[v];
    const T* a = store + S.off[v];
    for (int j = threadIdx.x; j < w; j += GS_THREADS) x[S.fc[v] + j] = s_div(x[S.fc[v] + j], a[(i64)j * ld + j]);
  }
}

// backward partials: rows [r0, r0 + SV_BR) x columns [c0, c0 + SV_BC), thread per column
template <class T>
__global__ void __launch_bounds__(GS_THREADS)
gs_bgemv(i64 first, SolveDev S, const T* __restrict__ tstore, const T* __restrict__ x, T* bpart) {
  __shared__ T xs[SV_BR];
  const int4 it = S.bitems[first + blockIdx.x];
  const int v = it.x, r0 = it.y, c0 = it.z;
  const int w = S.w[v], nro = S.nro[v];
  const i64 ld = S.ld[v];
  const int nr = min(SV_BR, nro - r0);
  const int* rp = S.rows + S.rowptr[v] + r0;
  for (int i = threadIdx.x; i < SV_BR; i += GS_THREADS) xs[i] = i < nr ? ldcg(x + rp[i]) : s_zero(T{});
  __syncthreads();
  const int c = c0 + (int)threadIdx.x;
  if (threadIdx.x < SV_BC && c < w) {
    const T* a = tstore + S.off[v] + (i64)c * ld + w + r0;
    T s = s_zero(T{});
    for (int i = 0; i < nr; ++i) s_fma(s, ldcg(a + i), xs[i]);
    bpart[S.bbase[v] + (i64)(r0 / SV_BR) * w + c] = s;
  }
}

template <class T, int F>
__global__ void __launch_bounds__(GS_THREADS)
gs_bdiag(i64 first, SolveDev S, const T* __restrict__ store, const T* __restrict__ tstore, T* x,
         const T* __restrict__ bpart) {
  extern __shared__ __align__(16) unsigned char gsm_raw[];
  T* y = reinterpret_cast<T*>(gsm_raw);
  const int tid = threadIdx.x;
  const int v = S.lvl_panels[first + blockIdx.x];
  const int w = S.w[v];
  const i64 fc = S.fc[v], ld = S.ld[v];
  const int nrc = (S.nro[v] + SV_BR - 1) / SV_BR;
  const T* a = store + S.off[v];
  const T* t = tstore + S.off[v];
  for (int j = tid; j < w; j += GS_THREADS) {
    T s = s_zero(T{});
    for (int rc = 0; rc < nrc; ++rc) {
      const T f = ldcg(bpart + S.bbase[v] + (i64)rc * w + j);
      if constexpr (sizeof(T) == sizeof(double)) s += f;
      else s = cplx{s.re + f.re, s.im + f.im};
    }
    if (F == FORM_LU) s = s_div(s, a[(i64)j * ld + j]);
    y[j] = s_sub(x[fc + j], s);
  }
  __syncthreads();
  for (int j = w - 1; j >= 0; --j) {
    T yj = y[j];
    if (F == FORM_LLT) yj = s_div(yj, a[(i64)j * ld + j]);
    __syncthreads();
    if (tid == 0) y[j] = yj;
    for (int i = tid; i < j; i += GS_THREADS) {
      // T(j, i) = t[i * ld + j]; LU: U(i, j) / U_ii
      T l = t[(i64)i * ld + j];
      if (F == FORM_LU) l = s_div(l, a[(i64)i * ld + i]);
      s_fms(y[i], l, yj);
    }
    __syncthreads();
  }
  for (int j = tid; j < w; j += GS_THREADS) x[fc + j] = y[j];
}

}  // namespace ps
