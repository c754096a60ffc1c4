// sm_100a kernels of the numeric factorization.
//
//   k_update      the paper's sparse_gemm: a 64x64 FP64 DMMA tile
//                 (mma.sync.m8n8k4.f64 -> DMMA.8x8x4) of one couple's
//                 contraction A_p[rows] * (d o) A_p[facing rows]^T, staged
//                 through a 3-stage cp.async shared-memory pipeline, whose
//                 epilogue scatter-subtracts straight into the destination
//                 panel through the device-resident block-row index map (no
//                 temporary buffer).  Persistent CTAs take tiles in list
//                 order; tiles of the same destination are ordered by source
//                 rank with per-destination completion counters, so the
//                 scatter is atomics-free and deterministic.
//                 Reference: kernels.py:128-136 (update_scatter_direct),
//                 :249-281 (run_update), :114-117 (LDLt scaling).
//   k_factor_blk  one column block (<= 64 wide) of a panel: diagonal
//                 POTRF / LDLt-without-pivoting in shared memory + the TRSM of
//                 up to 128 panel rows (thread per row, registers).
//                 Reference: kernels.py:208-247 (run_factor), :46-93.
//   k_factor_w1   width-1 panels (93% of panels at 60^3), warp per panel.
//                 Reference: kernels.py:216-221, :232-239.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ps {

typedef int64_t i64;

constexpr int FORM_LLT = 0;
constexpr int FORM_LDLT = 1;

struct DevArgs {
  double* store;
  double thr;
  int form;
  int pad;
};

struct UTile {
  int src, dst;     // source / destination panel
  int i0, j0;       // first source-local row of the A rows / facing (B) rows
  int ni, nj;       // extents (<= TM / TN)
  int k0, kn;       // source column range
  int couple;       // run-map couple id, -1: identity map (intra-panel)
  int wait;         // counters[dst] threshold before the scatter, -1: none
  int signal;       // 1: counters[dst] += 1 after the scatter
  int pad;
};

struct FItem {
  int p;            // panel
  int c0, nb;       // column block [c0, c0 + nb)
  int r0, nr;       // TRSM rows [r0, r0 + nr) (local)
  int diag;         // 1: this CTA writes the factored diagonal block + failure
};

struct PanelDev {
  const i64* off;   // slab offset
  const int* nrows; // leading dimension
  const int* width;
  const i64* fc;    // first column
};

struct Status {
  i64 fail_col;
  double fail_piv;
};

constexpr int TM = 64, TN = 64, KC = 16, NSTAGE = 3, LDS = TM + 4;
constexpr int UPD_THREADS = 128;
constexpr int FNB = 64, FTR = 128;
constexpr i64 NO_FAIL = 0x7f7f7f7f7f7f7f7fLL;

struct UpdSmem {
  double A[NSTAGE][KC][LDS];
  double B[NSTAGE][KC][LDS];
  double D[NSTAGE][KC];
  int rmap[TM];
  int cmap[TN];
  int tile;
};

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// destination-local row of source-local row i through the couple's runs
__device__ __forceinline__ int map_row(int i, int couple, const i64* run_ptr, const int* run_src,
                                       const int* run_dst) {
  if (couple < 0) return i;
  i64 lo = run_ptr[couple], hi = run_ptr[couple + 1] - 1;
  // last run with run_src <= i
  while (lo < hi) {
    i64 mid = (lo + hi + 1) >> 1;
    if (run_src[mid] <= i) lo = mid;
    else hi = mid - 1;
  }
  return run_dst[lo] + (i - run_src[lo]);
}

__device__ __forceinline__ void upd_load_stage(UpdSmem& sm, int st, const double* src, int ld,
                                               const UTile& T, int chunk, bool ldlt, int tid) {
  const int kbase = chunk * KC;
#pragma unroll
  for (int e = 0; e < (KC * TM) / UPD_THREADS; ++e) {
    int idx = tid + e * UPD_THREADS;
    int r = idx % TM;
    int kk = idx / TM;
    int k = kbase + kk;
    bool kv = k < T.kn;
    const double* colp = src + (i64)(T.k0 + (kv ? k : 0)) * ld;
    bool va = kv && r < T.ni;
    cp_async8(&sm.A[st][kk][r], colp + (va ? T.i0 + r : 0), va);
    bool vb = kv && r < T.nj;
    cp_async8(&sm.B[st][kk][r], colp + (vb ? T.j0 + r : 0), vb);
  }
  if (ldlt && tid < KC) {
    int k = kbase + tid;
    bool kv = k < T.kn;
    int kc = T.k0 + (kv ? k : 0);
    cp_async8(&sm.D[st][tid], src + (i64)kc * ld + kc, kv);
  }
}

__global__ void __launch_bounds__(UPD_THREADS, 3)
k_update(const UTile* __restrict__ tiles, int ntiles, int* __restrict__ work_ctr,
         unsigned* __restrict__ counters, const DevArgs* __restrict__ args, PanelDev P,
         const i64* __restrict__ run_ptr, const int* __restrict__ run_src,
         const int* __restrict__ run_dst) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  UpdSmem& sm = *reinterpret_cast<UpdSmem*>(smem_raw);
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  double* store = args->store;
  const bool ldlt = args->form == FORM_LDLT;

  while (true) {
    if (tid == 0) sm.tile = atomicAdd(work_ctr, 1);
    __syncthreads();
    const int t = sm.tile;
    if (t >= ntiles) break;
    const UTile T = tiles[t];
    const double* src = store + P.off[T.src];
    const int lds = P.nrows[T.src];

    // index maps of this tile (source-local -> destination-local)
    if (tid < TM) {
      sm.rmap[tid] = tid < T.ni ? map_row(T.i0 + tid, T.couple, run_ptr, run_src, run_dst) : 0;
    } else {
      int j = tid - TM;
      sm.cmap[j] = j < T.nj ? map_row(T.j0 + j, T.couple, run_ptr, run_src, run_dst) : 0;
    }

    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

    const int nch = (T.kn + KC - 1) / KC;
#pragma unroll
    for (int s = 0; s < NSTAGE - 1; ++s) {
      if (s < nch) upd_load_stage(sm, s, src, lds, T, s, ldlt, tid);
      cp_async_commit();
    }
    for (int c = 0; c < nch; ++c) {
      cp_async_wait<NSTAGE - 2>();
      __syncthreads();
      int nxt = c + NSTAGE - 1;
      if (nxt < nch) upd_load_stage(sm, nxt % NSTAGE, src, lds, T, nxt, ldlt, tid);
      cp_async_commit();
      const int st = c % NSTAGE;
#pragma unroll
      for (int ks = 0; ks < KC / 4; ++ks) {
        const int kr = ks * 4 + (lane & 3);
        double af[4], bf[4];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) af[mi] = sm.A[st][kr][wm * 32 + mi * 8 + (lane >> 2)];
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) bf[ni] = sm.B[st][kr][wn * 32 + ni * 8 + (lane >> 2)];
        if (ldlt) {
          double dk = sm.D[st][kr];
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) bf[ni] *= dk;
        }
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
      }
    }
    cp_async_wait<0>();

    // ordered, atomics-free scatter: wait until every lower-rank source of
    // this destination has finished its scatter
    if (T.wait >= 0 && tid == 0) {
      while (ld_acquire(&counters[T.dst]) < (unsigned)T.wait) __nanosleep(32);
    }
    __syncthreads();
    double* dst = store + P.off[T.dst];
    const i64 ldd = P.nrows[T.dst];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      const int row = wm * 32 + mi * 8 + (lane >> 2);
      if (row >= T.ni) continue;
      const int gi = T.i0 + row;
      const int dr = sm.rmap[row];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = wn * 32 + ni * 8 + (lane & 3) * 2 + e;
          if (col < T.nj && gi >= T.j0 + col) {
            double* ptr = dst + (i64)sm.cmap[col] * ldd + dr;
            __stcg(ptr, __ldcg(ptr) - acc[mi][ni][e]);
          }
        }
      }
    }
    __syncthreads();
    if (T.signal && tid == 0) {
      __threadfence();
      atomicAdd(&counters[T.dst], 1u);
    }
  }
}

// --------------------------------------------------------------------------
// narrow sources (width <= SMALL_W): one warp per tile on CUDA cores.  Same
// tile lists, maps, ordering counters and scatter rule as k_update; no
// shared-memory operand staging (operands are read through L1).
// Reference: kernels.py:283-309 (_run_update_rank1) and :128-136.

constexpr int SMALL_W = 8;
constexpr int SMALL_WARPS = 4;

__global__ void __launch_bounds__(32 * SMALL_WARPS)
k_update_small(const UTile* __restrict__ tiles, int ntiles, int* __restrict__ work_ctr,
               unsigned* __restrict__ counters, const DevArgs* __restrict__ args, PanelDev P,
               const i64* __restrict__ run_ptr, const int* __restrict__ run_src,
               const int* __restrict__ run_dst) {
  __shared__ int s_rmap[SMALL_WARPS][TM];
  __shared__ int s_cmap[SMALL_WARPS][TN];
  __shared__ double s_d[SMALL_WARPS][SMALL_W];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int* rmap = s_rmap[wid];
  int* cmap = s_cmap[wid];
  double* dsc = s_d[wid];
  double* store = args->store;
  const bool ldlt = args->form == FORM_LDLT;
  while (true) {
    int t = 0;
    if (lane == 0) t = atomicAdd(work_ctr, 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= ntiles) break;
    const UTile T = tiles[t];
    const double* src = store + P.off[T.src];
    const i64 lds = P.nrows[T.src];
    for (int r = lane; r < T.ni; r += 32)
      rmap[r] = map_row(T.i0 + r, T.couple, run_ptr, run_src, run_dst);
    for (int c = lane; c < T.nj; c += 32)
      cmap[c] = map_row(T.j0 + c, T.couple, run_ptr, run_src, run_dst);
    if (lane < T.kn) {
      const int k = T.k0 + lane;
      dsc[lane] = ldlt ? __ldg(src + (i64)k * lds + k) : 1.0;
    }
    if (T.wait >= 0 && lane == 0) {
      while (ld_acquire(&counters[T.dst]) < (unsigned)T.wait) __nanosleep(32);
    }
    __syncwarp();
    double* dst = store + P.off[T.dst];
    const i64 ldd = P.nrows[T.dst];
    const int tot = T.ni * T.nj;
    for (int e = lane; e < tot; e += 32) {
      const int i = e % T.ni, j = e / T.ni;
      if (T.i0 + i < T.j0 + j) continue;
      double v = 0.0;
      for (int k = 0; k < T.kn; ++k) {
        const double* col = src + (i64)(T.k0 + k) * lds;
        v += __ldg(col + T.i0 + i) * (__ldg(col + T.j0 + j) * dsc[k]);
      }
      double* ptr = dst + (i64)cmap[j] * ldd + rmap[i];
      __stcg(ptr, __ldcg(ptr) - v);
    }
    __syncwarp();
    if (T.signal && lane == 0) {
      __threadfence();
      atomicAdd(&counters[T.dst], 1u);
    }
    __syncwarp();
  }
}

// --------------------------------------------------------------------------
// column-block factorization: diagonal block in smem, TRSM rows in registers

// it.diag == 1: factor the diagonal block (from the assembled/updated panel),
//               write it back with the failure record, TRSM rows [r0, r0+nr).
// it.diag == 0: the block was factored by an earlier launch; load L (and d)
//               and TRSM rows [r0, r0+nr) only.  (Two launches, so no CTA
//               reads a diagonal block another CTA is rewriting.)
__global__ void __launch_bounds__(FTR)
k_factor_blk(const FItem* __restrict__ items, const DevArgs* __restrict__ args, PanelDev P,
             i64* __restrict__ fail_col, double* __restrict__ fail_piv) {
  // D[col][row]: lower part = factor; the free strict upper part holds
  // D[j][k] = d_k L_jk (LDLt) or L_jk (LLt), k < j, for the row solves
  __shared__ double D[FNB][FNB + 1];
  __shared__ double diag[FNB];
  __shared__ int s_fail;
  __shared__ double s_fpiv;
  const FItem it = items[blockIdx.x];
  const int tid = threadIdx.x;
  double* store = args->store;
  const bool ldlt = args->form == FORM_LDLT;
  const double thr = args->thr;
  double* base = store + P.off[it.p];
  const i64 ld = P.nrows[it.p];
  const int nb = it.nb, c0 = it.c0;

  for (int idx = tid; idx < nb * nb; idx += FTR) {
    int c = idx / nb, r = idx % nb;
    D[c][r] = r >= c ? base[(i64)(c0 + c) * ld + c0 + r] : 0.0;
  }
  if (tid == 0) s_fail = -1;
  __syncthreads();
  if (it.diag) {
    for (int j = 0; j < nb; ++j) {
      const double piv = D[j][j];
      const bool bad = ldlt ? (fabs(piv) <= thr) : (piv <= thr);
      if (bad && tid == 0 && s_fail < 0) {
        s_fail = j;
        s_fpiv = piv;
      }
      const double dv = ldlt ? piv : sqrt(piv);
      for (int r = j + 1 + tid; r < nb; r += FTR) D[j][r] = D[j][r] / dv;
      __syncthreads();
      if (tid == 0) D[j][j] = dv;
      for (int r = j + 1 + tid; r < nb; r += FTR) {
        const double lr = ldlt ? D[j][r] * piv : D[j][r];
        for (int c = j + 1; c <= r; ++c) D[c][r] -= lr * D[j][c];
      }
      __syncthreads();
    }
    for (int idx = tid; idx < nb * nb; idx += FTR) {
      int c = idx / nb, r = idx % nb;
      if (r >= c) base[(i64)(c0 + c) * ld + c0 + r] = D[c][r];
    }
    if (tid == 0 && s_fail >= 0 && fail_col[it.p] == NO_FAIL) {
      fail_col[it.p] = P.fc[it.p] + c0 + s_fail;
      fail_piv[it.p] = s_fpiv;
    }
  }
  for (int j = tid; j < nb; j += FTR) diag[j] = D[j][j];
  __syncthreads();
  // scaled copy for the row solves, into the strict upper triangle
  for (int idx = tid; idx < nb * nb; idx += FTR) {
    int k = idx / nb, j = idx % nb;
    if (j > k) D[j][k] = ldlt ? D[k][j] * diag[k] : D[k][j];
  }
  __syncthreads();
  if (tid < it.nr) {
    double* rowp = base + it.r0 + tid;
    double x[FNB];
#pragma unroll
    for (int k = 0; k < FNB; ++k)
      if (k < nb) x[k] = rowp[(i64)(c0 + k) * ld];
#pragma unroll
    for (int j = 0; j < FNB; ++j) {
      if (j < nb) {
        double s = x[j];
#pragma unroll
        for (int k = 0; k < j; ++k) s -= x[k] * D[j][k];
        x[j] = s / diag[j];
      }
    }
#pragma unroll
    for (int k = 0; k < FNB; ++k)
      if (k < nb) rowp[(i64)(c0 + k) * ld] = x[k];
  }
}

__global__ void k_factor_w1(const int* __restrict__ plist, int count, const DevArgs* __restrict__ args,
                            PanelDev P, i64* __restrict__ fail_col, double* __restrict__ fail_piv) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  double* store = args->store;
  const bool ldlt = args->form == FORM_LDLT;
  const double thr = args->thr;
  for (int i = gw; i < count; i += nw) {
    const int p = plist[i];
    double* a = store + P.off[p];
    const int nr = P.nrows[p];
    const double piv = a[0];
    __syncwarp();
    const bool bad = ldlt ? (fabs(piv) <= thr) : (piv <= thr);
    const double dv = ldlt ? piv : sqrt(piv);
    for (int r = 1 + lane; r < nr; r += 32) a[r] = a[r] / dv;
    if (lane == 0) {
      if (!ldlt) a[0] = dv;
      if (bad && fail_col[p] == NO_FAIL) {
        fail_col[p] = P.fc[p];
        fail_piv[p] = piv;
      }
    }
  }
}

__global__ void k_assemble(double* __restrict__ store, const i64* __restrict__ pos,
                           const double* __restrict__ vals, i64 n) {
  for (i64 k = blockIdx.x * (i64)blockDim.x + threadIdx.x; k < n; k += (i64)gridDim.x * blockDim.x)
    store[pos[k]] = vals[k];
}

__global__ void k_status(const i64* __restrict__ fail_col, const double* __restrict__ fail_piv,
                         i64 np, Status* st) {
  __shared__ i64 sc[1024];
  __shared__ i64 sp[1024];
  i64 best = NO_FAIL, bp = -1;
  for (i64 p = threadIdx.x; p < np; p += blockDim.x) {
    if (fail_col[p] < best) {
      best = fail_col[p];
      bp = p;
    }
  }
  sc[threadIdx.x] = best;
  sp[threadIdx.x] = bp;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s && sc[threadIdx.x + s] < sc[threadIdx.x]) {
      sc[threadIdx.x] = sc[threadIdx.x + s];
      sp[threadIdx.x] = sp[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    st->fail_col = sc[0];
    st->fail_piv = sp[0] >= 0 ? fail_piv[sp[0]] : 0.0;
  }
}

}  // namespace ps
