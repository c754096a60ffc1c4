// GPU supernodal triangular solve: the contract of the
// reference's supernodal_solve (kernels.py:332-382) on the device-resident
// factor, level by level (panel-tree height), deterministic (no atomics:
// every sum is taken in a fixed order).  Two kernels per level and pass:
//
//   forward  (levels ascending):
//     fdiag, one CTA per panel q:
//       y = x_q - (partials landing in q's columns, ascending partial index)
//       z_q = L_qq^-1 y ; x_q = z_q / d_q (LDLt) | z_q (LLt)
//     fgemv, one CTA per (panel, 64 facing rows, 128 columns) item:
//       the partial products L_q[facing rows, k-chunk] z_q[k-chunk], one per
//       (k-chunk, row), for the destinations' later levels (right-looking:
//       a wide panel's off-diagonal block is read by many CTAs at once)
//   backward (levels descending):
//     bgemv, one CTA per (panel, 256 facing rows, 32 columns) item:
//       s_rc[j] = sum_{r in chunk} L_p[r, j] x[rows[r]] (rows: ancestors, final)
//     bdiag, one CTA per panel p:
//       y = x_p - sum_rc s_rc (ascending chunk) ; x_p = L_pp^-T y
//
// x is in the permuted order (x[perm] = b before, b = x[perm] after).
#pragma once
#include "ps_kernels.cuh"

namespace ps {

constexpr int SV_THREADS = 256;  // GEMV items
constexpr int SV_SUB = 512;      // widest virtual panel (wider panels: column slices)
constexpr int SV_NARROW_T = 128; // diagonal solves of narrow virtual panels (w <= SV_WIDE)
constexpr int SV_WIDE_T = 512;   // diagonal solves of wide ones (w <= SV_SUB)
constexpr int SV_WIDE = 96;
constexpr int SV_TINY = 32;      // panels solved by one warp (registers + shuffles)
constexpr int SV_MAXW = SV_SUB;  // right-hand side in shared memory (PS_SOLVE_SMEM_W: scratch path)
constexpr int SV_FR = 64;        // forward item: facing rows
constexpr int SV_KC = 128;       // forward item: columns (one partial per k-chunk and row)
constexpr int SV_BR = 256;       // backward item: facing rows
constexpr int SV_BC = 32;        // backward item: columns
static_assert(SV_WIDE <= SV_NARROW_T + 32 && SV_SUB <= SV_WIDE_T + 32, "one update row per thread");

struct SolveDev {
  const i64* lvl_ptr;    // virtual panels of level L: lvl_panels[lvl_ptr[L] .. lvl_ptr[L+1])
  const int* lvl_panels;
  const int* w;          // per virtual panel: width, facing rows, first global column,
  const int* nro;        //   store offset of its diagonal element, leading dimension
  const i64* fc;
  const i64* off;
  const i64* ld;
  const i64* fbase;      // per virtual panel: forward partials fpart[fbase[v] + kc * nro_v + r]
  const i64* jptr;       // per global column j: jidx[jptr[j] .. jptr[j+1]) = the partials
  const i64* jidx;       //   landing in j, ascending (source, k-chunk): fixed order
  const i64* bbase;      // per virtual panel: backward partials bpart[bbase[v] + rc * w_v + j]
  const int4* fitems;    // forward items (v, r0, k0, -), level L: [fi_ptr[L], fi_ptr[L+1])
  const int4* bitems;    // backward items (v, r0, c0, -)
  const int2* ritems;    // forward reduction items (v, first of 8 columns)
  const i64* rowptr;     // per virtual panel: global rows of its facing rows
  const int* rows;
};

// Diagonal-block triangular solves, one CTA of NT threads, w <= NT + 32.
// Per 32-column block: the next block's diagonal entries and every thread's
// 32 update entries are loaded into registers BEFORE warp 0's shuffle sweep
// of the current block, so no global latency sits on the sequential chain.
// B[2][33][33]: double-buffered diagonal blocks (row 32: pivot reciprocals).
template <int NT>
__device__ __forceinline__ void diag_regs(double* dv, const double* a, i64 ld, int c0, int nb, int tid) {
#pragma unroll
  for (int u = 0; u < 1024 / NT; ++u) {
    const int e = tid + u * NT, c = e >> 5, r = e & 31;
    dv[u] = (c < nb && r < nb && r >= c) ? __ldg(a + (i64)(c0 + c) * ld + c0 + r) : 0.0;
  }
}
template <int NT>
__device__ __forceinline__ void diag_store(double (*B)[33], const double* dv, int nb, int tid) {
#pragma unroll
  for (int u = 0; u < 1024 / NT; ++u) {
    const int e = tid + u * NT, c = e >> 5, r = e & 31;
    B[c][r] = dv[u];
    if (r == c) B[32][c] = c < nb ? 1.0 / dv[u] : 0.0;
  }
}

// y (length w) <- L^-1 y  (lower, unit if ldlt), column-major a (ld)
template <int NT>
__device__ __forceinline__ void trsv_lower(const double* a, i64 ld, int w, double* y, bool unit,
                                           int tid, double (*B)[33][33]) {
  constexpr bool PF = NT > SV_NARROW_T;  // register prefetch (narrow CTAs: occupancy instead)
  const int lane = tid & 31, warp = tid >> 5;
  double dv[1024 / NT];
  diag_regs<NT>(dv, a, ld, 0, min(32, w), tid);
  diag_store<NT>(B[0], dv, min(32, w), tid);
  __syncthreads();
  for (int c0 = 0, bi = 0; c0 < w; c0 += 32, bi ^= 1) {
    const int nb = min(32, w - c0);
    const int r = c0 + 32 + tid;  // this thread's update row
    const double* ar = a + (i64)c0 * ld + r;
    double lv[PF ? 32 : 1];
    if (PF && r < w) {
#pragma unroll
      for (int j = 0; j < 32; ++j) lv[j] = __ldg(ar + (i64)j * ld);
    }
    const int n1 = min(32, w - c0 - 32);
    if (n1 > 0) diag_regs<NT>(dv, a, ld, c0 + 32, n1, tid);
    if (warp == 0) {
      double (*D)[33] = B[bi];
      double v = lane < nb ? y[c0 + lane] : 0.0;
      for (int j = 0; j < nb; ++j) {
        double xj = __shfl_sync(0xffffffffu, v, j);
        if (!unit) xj *= D[32][j];
        if (lane == j) v = xj;
        if (lane > j && lane < nb) v -= D[j][lane] * xj;
      }
      if (lane < nb) y[c0 + lane] = v;
    }
    if (n1 > 0) diag_store<NT>(B[bi ^ 1], dv, n1, tid);
    __syncthreads();
    if (r < w) {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        s0 += (PF ? lv[j] : __ldg(ar + (i64)j * ld)) * y[c0 + j];
        s1 += (PF ? lv[j + 1] : __ldg(ar + (i64)(j + 1) * ld)) * y[c0 + j + 1];
      }
      y[r] -= s0 + s1;
    }
    __syncthreads();
  }
}

// y <- L^-T y (upper = transpose of the lower factor, unit if ldlt)
template <int NT>
__device__ __forceinline__ void trsv_lower_t(const double* a, i64 ld, int w, double* y, bool unit,
                                             int tid, double (*B)[33][33]) {
  constexpr bool PF = NT > SV_NARROW_T;
  const int lane = tid & 31, warp = tid >> 5;
  double dv[1024 / NT];
  {
    const int c0 = (w - 1) / 32 * 32;
    diag_regs<NT>(dv, a, ld, c0, w - c0, tid);
    diag_store<NT>(B[0], dv, w - c0, tid);
  }
  __syncthreads();
  for (int c0 = (w - 1) / 32 * 32, bi = 0; c0 >= 0; c0 -= 32, bi ^= 1) {
    const int nb = min(32, w - c0);
    // update columns i < c0.  PF: warp g owns columns [32g, 32g + 32), lane j
    // holds row c0 + j of them (coalesced 256-byte loads, prefetched before
    // the sweep) and the 32 column sums come out of a shuffle transpose-
    // reduction (lane l: column 32g + l).  Narrow CTAs: thread per column.
    const int g0 = warp * 32;
    double lv[PF ? 32 : 1];
    if (PF && g0 < c0) {
#pragma unroll
      for (int k = 0; k < 32; ++k)
        lv[k] = (lane < nb && g0 + k < c0) ? __ldg(a + (i64)(g0 + k) * ld + c0 + lane) : 0.0;
    }
    if (c0 > 0) diag_regs<NT>(dv, a, ld, c0 - 32, 32, tid);
    if (warp == 0) {
      double (*D)[33] = B[bi];
      double v = lane < nb ? y[c0 + lane] : 0.0;
      for (int j = nb - 1; j >= 0; --j) {
        double xj = __shfl_sync(0xffffffffu, v, j);
        if (!unit) xj *= D[32][j];
        if (lane == j) v = xj;
        if (lane < j) v -= D[lane][j] * xj;  // unknowns i < j: y_i -= L[j, i] x_j
      }
      if (lane < nb) y[c0 + lane] = v;
    }
    if (c0 > 0) diag_store<NT>(B[bi ^ 1], dv, 32, tid);
    __syncthreads();
    if (PF) {
      if (g0 < c0) {
        const double yj = lane < nb ? y[c0 + lane] : 0.0;
#pragma unroll
        for (int k = 0; k < 32; ++k) lv[k] *= yj;
        // transpose-reduce: after the step of width h, lane l keeps the
        // entries whose index agrees with l on bit h (fixed order)
#pragma unroll
        for (int h = 16; h > 0; h >>= 1) {
          const bool up = lane & h;
#pragma unroll
          for (int k = 0; k < h; ++k) {
            const double send = up ? lv[k] : lv[k + h];
            const double keep = up ? lv[k + h] : lv[k];
            lv[k] = keep + __shfl_xor_sync(0xffffffffu, send, h);
          }
        }
        if (g0 + lane < c0) y[g0 + lane] -= lv[0];
      }
    } else {
      const int i = tid;  // thread per column: its 32 entries are one contiguous run
      if (i < c0) {
        const double* col = a + (i64)i * ld + c0;
        double s0 = 0.0;
        for (int j = 0; j < nb; ++j) s0 += __ldg(col + j) * y[c0 + j];
        y[i] -= s0;
      }
    }
    __syncthreads();
  }
}

template <int NT>
__global__ void __launch_bounds__(NT)
k_sv_fdiag(i64 first, SolveDev S, const double* __restrict__ store, double* x, double* z,
           double* scratch, const double* __restrict__ fpart, int ldlt, int maxw) {
  pdl_wait();  // programmatic dependent launch (see ps_kernels.cuh)
  pdl_trigger();
  extern __shared__ double ys[];  // the launch's widest fitting panel (host-sized)
  __shared__ double B32[2][33][33];
  const int tid = threadIdx.x;
  const int q = S.lvl_panels[first + blockIdx.x];
  const int w = S.w[q];
  const i64 fcq = S.fc[q];
  double* y = w <= maxw ? ys : scratch + fcq;
  for (int j = tid; j < w; j += NT) y[j] = x[fcq + j];  // incoming partials: k_sv_freduce
  __syncthreads();
  const double* aq = store + S.off[q];
  const i64 ldq = S.ld[q];
  trsv_lower<NT>(aq, ldq, w, y, ldlt != 0, tid, B32);
  for (int j = tid; j < w; j += NT) {
    const double v = y[j];
    z[fcq + j] = v;
    x[fcq + j] = ldlt ? v / __ldg(aq + (i64)j * ldq + j) : v;
  }
}

// tiny virtual panels (w <= 32): one warp per panel, lane r = row r of the
// diagonal block in registers, the same sweep as trsv_lower (pivot
// reciprocals, shuffles) without shared memory or CTA barriers
__global__ void __launch_bounds__(128)
k_sv_fdiag_w(i64 first, int count, SolveDev S, const double* __restrict__ store, double* x,
             double* z, int ldlt) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (k >= count) return;
  const int q = S.lvl_panels[first + k];
  const int w = S.w[q];
  const i64 fcq = S.fc[q], ld = S.ld[q];
  const double* a = store + S.off[q];
  double row[SV_TINY];
#pragma unroll
  for (int c = 0; c < SV_TINY; ++c) row[c] = (c < w && lane < w && c <= lane) ? __ldg(a + (i64)c * ld + lane) : 0.0;
  double dgl = 0.0;  // this lane's pivot L[lane][lane]
#pragma unroll
  for (int c = 0; c < SV_TINY; ++c)
    if (c == lane) dgl = row[c];
  const double rd = lane < w ? 1.0 / dgl : 0.0;
  double v = lane < w ? x[fcq + lane] : 0.0;
#pragma unroll
  for (int j = 0; j < SV_TINY; ++j) {
    if (j < w) {
      double xj = __shfl_sync(0xffffffffu, v, j);
      if (!ldlt) xj *= __shfl_sync(0xffffffffu, rd, j);
      if (lane == j) v = xj;
      if (lane > j && lane < w) v -= row[j] * xj;
    }
  }
  if (lane < w) {
    z[fcq + lane] = v;
    x[fcq + lane] = ldlt ? v / dgl : v;
  }
}

__global__ void __launch_bounds__(128)
k_sv_bdiag_w(i64 first, int count, SolveDev S, const double* __restrict__ store, double* x,
             const double* __restrict__ bpart, int ldlt) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (k >= count) return;
  const int p = S.lvl_panels[first + k];
  const int w = S.w[p];
  const i64 fcp = S.fc[p], ld = S.ld[p];
  const int nrc = (S.nro[p] + SV_BR - 1) / SV_BR;
  const double* a = store + S.off[p];
  const double* bp = bpart + S.bbase[p];
  // lane i holds column i of the diagonal block: L[j][i], j >= i (contiguous)
  double col[SV_TINY];
#pragma unroll
  for (int j = 0; j < SV_TINY; ++j) col[j] = (lane < w && j < w && j >= lane) ? __ldg(a + (i64)lane * ld + j) : 0.0;
  double dgl = 0.0;
#pragma unroll
  for (int j = 0; j < SV_TINY; ++j)
    if (j == lane) dgl = col[j];
  const double rd = lane < w ? 1.0 / dgl : 0.0;
  double v = 0.0;
  if (lane < w) {
    v = x[fcp + lane];
    for (int rc = 0; rc < nrc; ++rc) v -= __ldcg(bp + (i64)rc * w + lane);
  }
#pragma unroll
  for (int j = SV_TINY - 1; j >= 0; --j) {
    if (j < w) {
      double xj = __shfl_sync(0xffffffffu, v, j);
      if (!ldlt) xj *= __shfl_sync(0xffffffffu, rd, j);
      if (lane == j) v = xj;
      if (lane < j) v -= col[j] * xj;  // y_i -= L[j, i] x_j
    }
  }
  if (lane < w) x[fcp + lane] = v;
}

// incoming forward partials of one item (8 columns of a virtual panel): a
// warp per column, lanes over its partials (fixed lane assignment and
// shuffle tree: a fixed summation order), x[j] -= sum
__global__ void __launch_bounds__(SV_THREADS)
k_sv_freduce(i64 first, SolveDev S, double* x, const double* __restrict__ fpart) {
  pdl_wait();  // programmatic dependent launch (see ps_kernels.cuh)
  pdl_trigger();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int2 it = S.ritems[first + blockIdx.x];
  const int j = it.y + warp;
  if (j >= S.w[it.x]) return;
  const i64 gj = S.fc[it.x] + j;
  const i64 e0 = S.jptr[gj], e1 = S.jptr[gj + 1];
  double v = 0.0;
  for (i64 e = e0 + lane; e < e1; e += 32) v += __ldcg(fpart + S.jidx[e]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0 && e1 > e0) x[gj] -= v;
}

// forward partials of one item: 64 rows x 128 columns, thread (row, k-group
// of 32 columns), the 4 groups added in order
__global__ void __launch_bounds__(SV_THREADS)
k_sv_fgemv(i64 first, SolveDev S, const double* __restrict__ store, const double* __restrict__ z,
           double* fpart) {
  pdl_wait();  // programmatic dependent launch (see ps_kernels.cuh)
  pdl_trigger();
  __shared__ double zs[SV_KC];
  __shared__ double red[SV_THREADS / SV_FR][SV_FR];
  const int tid = threadIdx.x;
  const int4 it = S.fitems[first + blockIdx.x];
  const int v = it.x, r0 = it.y, k0 = it.z;
  const int w = S.w[v], nro = S.nro[v];
  const i64 ld = S.ld[v];
  const int kn = min(SV_KC, w - k0);
  if (tid < SV_KC) zs[tid] = tid < kn ? __ldcg(z + S.fc[v] + k0 + tid) : 0.0;
  __syncthreads();
  const int r = tid % SV_FR, g = tid / SV_FR;
  constexpr int KG = SV_KC / (SV_THREADS / SV_FR);
  double s0 = 0.0, s1 = 0.0;
  if (r0 + r < nro) {
    const double* a = store + S.off[v] + (i64)(k0 + g * KG) * ld + w + r0 + r;
    const int kk = min(KG, kn - g * KG);
    if (kk == KG) {
#pragma unroll
      for (int k = 0; k < KG; k += 2) {
        s0 += __ldcg(a + (i64)k * ld) * zs[g * KG + k];
        s1 += __ldcg(a + (i64)(k + 1) * ld) * zs[g * KG + k + 1];
      }
    } else {
      for (int k = 0; k < kk; ++k) s0 += __ldcg(a + (i64)k * ld) * zs[g * KG + k];
    }
  }
  red[g][r] = s0 + s1;
  __syncthreads();
  if (tid < SV_FR && r0 + tid < nro) {
    double t = 0.0;
#pragma unroll
    for (int u = 0; u < SV_THREADS / SV_FR; ++u) t += red[u][tid];
    fpart[S.fbase[v] + (i64)(k0 / SV_KC) * nro + r0 + tid] = t;
  }
}

// backward partials of one item: 256 rows x 32 columns, a warp per 4
// columns, lanes over rows (coalesced), shuffle-reduced (fixed order)
__global__ void __launch_bounds__(SV_THREADS)
k_sv_bgemv(i64 first, SolveDev S, const double* __restrict__ store, const double* __restrict__ x,
           double* bpart) {
  pdl_wait();  // programmatic dependent launch (see ps_kernels.cuh)
  pdl_trigger();
  __shared__ double xs[SV_BR];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int4 it = S.bitems[first + blockIdx.x];
  const int v = it.x, r0 = it.y, c0 = it.z;
  const int w = S.w[v], nro = S.nro[v];
  const i64 ld = S.ld[v];
  const int nr = min(SV_BR, nro - r0);
  const int* rp = S.rows + S.rowptr[v] + r0;
  for (int i = tid; i < SV_BR; i += SV_THREADS) xs[i] = i < nr ? __ldcg(x + rp[i]) : 0.0;
  __syncthreads();
  constexpr int CPW = SV_BC / (SV_THREADS / 32);
#pragma unroll
  for (int cc = 0; cc < CPW; ++cc) {
    const int c = c0 + warp * CPW + cc;
    if (c >= w) break;
    const double* a = store + S.off[v] + (i64)c * ld + w + r0;
    double s = 0.0;
#pragma unroll
    for (int i = lane; i < SV_BR; i += 32)
      if (i < nr) s += __ldcg(a + i) * xs[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) bpart[S.bbase[v] + (i64)(r0 / SV_BR) * w + c] = s;
  }
}

template <int NT>
__global__ void __launch_bounds__(NT)
k_sv_bdiag(i64 first, SolveDev S, const double* __restrict__ store, double* x, double* scratch,
           const double* __restrict__ bpart, int ldlt, int maxw) {
  pdl_wait();  // programmatic dependent launch (see ps_kernels.cuh)
  pdl_trigger();
  extern __shared__ double ys[];
  __shared__ double B32[2][33][33];
  const int tid = threadIdx.x;
  const int v = S.lvl_panels[first + blockIdx.x];
  const int w = S.w[v];
  const i64 fcv = S.fc[v];
  const int nrc = (S.nro[v] + SV_BR - 1) / SV_BR;
  const double* bp = bpart + S.bbase[v];
  double* y = w <= maxw ? ys : scratch + fcv;
  for (int j = tid; j < w; j += NT) {
    double t = x[fcv + j];
    for (int rc = 0; rc < nrc; ++rc) t -= __ldcg(bp + (i64)rc * w + j);
    y[j] = t;
  }
  __syncthreads();
  trsv_lower_t<NT>(store + S.off[v], S.ld[v], w, y, ldlt != 0, tid, B32);
  for (int j = tid; j < w; j += NT) x[fcv + j] = y[j];
}

}  // namespace ps
