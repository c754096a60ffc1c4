// sm_100a kernels of the numeric factorization.
//
//   k_update       the paper's sparse_gemm: a 64x64 FP64 DMMA tile
//                  (mma.sync.m8n8k4.f64 -> DMMA.8x8x4) of one couple's
//                  contraction A_p[rows] * (d o) A_p[facing rows]^T, staged
//                  through a 3-stage cp.async shared-memory pipeline, whose
//                  epilogue scatter-subtracts straight into the destination
//                  panel through the device-resident block-row index map (no
//                  temporary buffer).  Persistent CTAs take tiles in list
//                  order; tiles of one destination are ordered by a
//                  column-overlap coloring with per-destination completion
//                  counters, so the scatter is atomics-free and deterministic.
//                  Reference: kernels.py:128-136 (update_scatter_direct),
//                  :249-281 (run_update), :114-117 (LDLt scaling).
//   k_update_small narrow sources (width <= 8): warp per tile, CUDA cores.
//                  Reference: kernels.py:283-309 (_run_update_rank1).
//   k_factor_small panels of width 2..32: diagonal POTRF / LDLt in shared
//                  memory + thread-per-row TRSM.  Reference: kernels.py:208-247.
//   k_factor_diag  one 64-column block of a wide panel: diagonal factor, then
//                  G = scaled inverse of the diagonal factor (scratch).
//   k_trsm         the wide panel's TRSM as a DMMA GEMM X = B G^T (in place).
//   k_factor_w1    width-1 panels (93% of panels at 60^3), warp per panel.
//                  Reference: kernels.py:216-221, :232-239.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ps {

typedef int64_t i64;

constexpr int FORM_LLT = 0;
constexpr int FORM_LDLT = 1;

struct DevArgs {
  double* store;
  double* scratch;  // inverse diagonal blocks of wide panels (FNB x FNB each)
  double thr;
  int form;
  int pad;
  unsigned long long* tile_trace;  // optional (debug): per tile {start, mainloop done, end} ns
  const struct UTile* tile_base;   // tile index base of tile_trace
  double* splitk_ws;               // split-K partial tiles (TM x TN doubles per slot)
  unsigned* splitk_cnt;            // finished partials per reduction tile
};

struct UTile {
  int src, dst;     // source / destination panel
  int i0, j0;       // first source-local row of the A rows / facing (B) rows
  int ni, nj;       // extents (<= TM / TN)
  int k0, kn;       // source column range
  int couple;       // run-map couple id, -1: identity map (intra-panel)
  int wait;         // counters[dst] threshold before the scatter, -1: none
  int signal;       // 1: counters[dst] += 1 after the scatter
  int ri, rj;       // run index covering source row i0 / j0 (map hints)
  int mode;         // 0: tile; 1: split-K partial (k0/kn = its K range, product to
                    //    workspace slot ws, then splitk_cnt[rc] += 1); 2: reduction of
                    //    the nparts partials at slots ws.. (fixed order), then scatter
  int ws, nparts, rc;
  int lds, ldd;     // leading dimensions of src / dst, and their slab offsets (filled
  i64 soff, doff;   //   at plan time: one dependent load less per tile)
};

struct FItem {
  int p;            // panel
  int c0, nb;       // column block [c0, c0 + nb)
  int r0, nr;       // rows [r0, r0 + nr) (local) to solve
  int diag;         // 1: this CTA factors the diagonal block (+ failure record)
  int g;            // scratch slot of the block's scaled inverse (wide panels)
  int pad;
};

// narrow-source gather: one destination tile and its source segments
struct NItem {
  int q;            // destination panel
  int r0, nr;       // destination-local rows [r0, r0 + nr), nr <= TM
  int c0, nc;       // destination columns [c0, c0 + nc), nc <= TN
  int seg0, nseg;   // segments [seg0, seg0 + nseg), in source order
  int pad;
  unsigned long long cmask;  // columns c0 + b the segments touch (bit b); 0 = all
};
struct NSeg {
  int couple, p;    // couple (run map) and source panel
  int s0, s1;       // source-local rows landing in the tile's rows
  int f0, f1;       // source-local facing rows landing in the tile's columns
  int rs, rf;       // run hints for s0 / f0
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

#ifndef UPD_KC
#define UPD_KC 16  // K chunk per pipeline stage
#endif
#ifndef UPD_NSTAGE
#define UPD_NSTAGE 3
#endif
constexpr int TM = 64, TN = 64, KC = UPD_KC, NSTAGE = UPD_NSTAGE, LDS = TM + 4, CLD = TM + 2;
constexpr int UPD_THREADS = 128;
#ifndef UPD_MIN_CTAS
#define UPD_MIN_CTAS 3  // k_update resident CTAs per SM (registers: 168 at 3)
#endif
constexpr int FNB = 64;          // column block of wide panels
constexpr int SNB = 32;          // widest "small" panel
constexpr int FTR = 128;         // rows per small-factor CTA
#ifndef PS_SMALL_W
#define PS_SMALL_W 8
#endif
constexpr int SMALL_W = PS_SMALL_W;  // widest narrow update source
#ifndef SMALL_WARPS
#define SMALL_WARPS 4  // warps per narrow-update CTA
#endif
constexpr i64 NO_FAIL = 0x7f7f7f7f7f7f7f7fLL;

struct UpdSmem {
  double A[NSTAGE][KC][LDS];
  double B[NSTAGE][KC][LDS];
  double D[NSTAGE][KC];
  int rmap[TM];
  int cmap[TN];
  int wsrc[2][TM];  // run windows of the tile's rows / columns (map staging)
  int wdst[2][TM];
  int tile;
};
static_assert(sizeof(double) * NSTAGE * KC * LDS * 2 >= sizeof(double) * TN * CLD,
              "epilogue staging must fit in the operand stages");

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

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Programmatic dependent launch (kernels launched with the PDL attribute):
// pdl_wait blocks until the previous grid on the stream has completed and its
// memory is visible; pdl_trigger (a persistent CTA out of work) lets the next
// grid start launching into the slots of exiting CTAs.  No-ops otherwise.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// destination-local row of source-local row i through the couple's runs,
// scanning forward from the run `k` that covers the tile's first row
__device__ __forceinline__ int map_row(int i, int couple, int k, const i64* run_ptr,
                                       const int* run_src, const int* run_dst) {
  if (couple < 0) return i;
  const i64 end = run_ptr[couple + 1];
  while (k + 1 < end && __ldg(run_src + k + 1) <= i) ++k;
  return __ldg(run_dst + k) + (i - __ldg(run_src + k));
}

// Tile maps, phase 1: stage the couple's runs covering the tile's rows
// (window from run ri) and columns (window from run rj) in shared memory -
// one parallel load instead of a dependent scan per row.  64 runs always
// cover 64 consecutive source rows.
template <class SM>
__device__ __forceinline__ void maps_load(SM& sm, int couple, int ri, int rj, const i64* run_ptr,
                                          const int* run_src, const int* run_dst, int tid) {
  if (couple < 0) return;
  const int w = tid >> 6, k = (w ? rj : ri) + (tid & 63);
  const i64 end = __ldg(run_ptr + couple + 1);
  sm.wsrc[w][tid & 63] = k < end ? __ldg(run_src + k) : 0x7fffffff;
  sm.wdst[w][tid & 63] = k < end ? __ldg(run_dst + k) : 0;
}
// phase 2 (after a barrier): binary search of the window
template <class SM>
__device__ __forceinline__ void maps_search(SM& sm, int couple, int i0, int ni, int j0, int nj,
                                            int tid) {
  const int w = tid >> 6, x = tid & 63;
  const int row = (w ? j0 : i0) + x;
  int v = 0;
  if (x < (w ? nj : ni)) {
    if (couple < 0) {
      v = row;
    } else {
      const int* ws = sm.wsrc[w];
      int lo = 0, hi = 63;
      while (lo < hi) {  // last run start <= row
        const int mid = (lo + hi + 1) >> 1;
        if (ws[mid] <= row) lo = mid;
        else hi = mid - 1;
      }
      v = sm.wdst[w][lo] + (row - ws[lo]);
    }
  }
  (w ? sm.cmap : sm.rmap)[x] = v;
}

// ---------------------------------------------------------------------------
// shared DMMA mainloop: acc[i][j] += sum_k A[ai0+i, k] * (d_k) * B[bj0+j, k]
// for column-major A (lda) and B (ldb), k in [0, kn) (pointers pre-offset to
// the first column).  d_k = dptr[k * dstride] when dptr != nullptr.

struct Operands {
  const double* A;
  i64 lda;
  int ai0, ani;
  const double* B;
  i64 ldb;
  int bj0, bnj;
  int kn;
  const double* dptr;
  i64 dstride;
};

__device__ __forceinline__ void load_stage(UpdSmem& sm, int st, const Operands& O, int chunk, int tid) {
  const int kbase = chunk * KC;
#pragma unroll
  for (int e = 0; e < (KC * TM) / UPD_THREADS; ++e) {
    const int idx = tid + e * UPD_THREADS;
    const int r = idx % TM;
    const int kk = idx / TM;
    const int k = kbase + kk;
    const bool kv = k < O.kn;
    const int kc = kv ? k : 0;
    const bool va = kv && r < O.ani;
    cp_async8(&sm.A[st][kk][r], O.A + (i64)kc * O.lda + (va ? O.ai0 + r : 0), va);
    const bool vb = kv && r < O.bnj;
    cp_async8(&sm.B[st][kk][r], O.B + (i64)kc * O.ldb + (vb ? O.bj0 + r : 0), vb);
  }
  if (O.dptr && tid < KC) {
    const int k = kbase + tid;
    const bool kv = k < O.kn;
    cp_async8(&sm.D[st][tid], O.dptr + (i64)(kv ? k : 0) * O.dstride, kv);
  }
}

__device__ __forceinline__ void dmma_mainloop(UpdSmem& sm, const Operands& O, double acc[4][4][2],
                                              int tid) {
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int nch = (O.kn + KC - 1) / KC;
#pragma unroll
  for (int s = 0; s < NSTAGE - 1; ++s) {
    if (s < nch) load_stage(sm, s, O, s, tid);
    cp_async_commit();
  }
  for (int c = 0; c < nch; ++c) {
    cp_async_wait<NSTAGE - 2>();
    __syncthreads();
    const int nxt = c + NSTAGE - 1;
    if (nxt < nch) load_stage(sm, nxt % NSTAGE, O, nxt, tid);
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
      if (O.dptr) {
        const double dk = sm.D[st][kr];
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
  __syncthreads();  // operand stages free: callers reuse them for the epilogue
}

// 8-warp variant of the mainloop for the wide-panel chain (latency-bound
// launches of few tiles): warps in a 2 x 4 grid, 32 x 16 each, so a tile's
// DMMA issue is spread over twice the warps; the same k order per entry as
// dmma_mainloop (bitwise identical sums).
constexpr int W8_THREADS = 256;
__device__ __forceinline__ void load_stage8(UpdSmem& sm, int st, const Operands& O, int chunk, int tid) {
  const int kbase = chunk * KC;
#pragma unroll
  for (int e = 0; e < (KC * TM) / W8_THREADS; ++e) {
    const int idx = tid + e * W8_THREADS;
    const int r = idx % TM;
    const int kk = idx / TM;
    const int k = kbase + kk;
    const bool kv = k < O.kn;
    const int kc = kv ? k : 0;
    const bool va = kv && r < O.ani;
    cp_async8(&sm.A[st][kk][r], O.A + (i64)kc * O.lda + (va ? O.ai0 + r : 0), va);
    const bool vb = kv && r < O.bnj;
    cp_async8(&sm.B[st][kk][r], O.B + (i64)kc * O.ldb + (vb ? O.bj0 + r : 0), vb);
  }
  if (O.dptr && tid < KC) {
    const int k = kbase + tid;
    const bool kv = k < O.kn;
    cp_async8(&sm.D[st][tid], O.dptr + (i64)(kv ? k : 0) * O.dstride, kv);
  }
}

// acc fragments of the 8-warp layout -> Cs[col][row] (shared, reuses the stages)
__device__ __forceinline__ double (*dmma_tile8(UpdSmem& sm, const Operands& O, int tid))[CLD] {
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  double acc[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int nch = (O.kn + KC - 1) / KC;
#pragma unroll
  for (int s = 0; s < NSTAGE - 1; ++s) {
    if (s < nch) load_stage8(sm, s, O, s, tid);
    cp_async_commit();
  }
  for (int c = 0; c < nch; ++c) {
    cp_async_wait<NSTAGE - 2>();
    __syncthreads();
    const int nxt = c + NSTAGE - 1;
    if (nxt < nch) load_stage8(sm, nxt % NSTAGE, O, nxt, tid);
    cp_async_commit();
    const int st = c % NSTAGE;
#pragma unroll
    for (int ks = 0; ks < KC / 4; ++ks) {
      const int kr = ks * 4 + (lane & 3);
      double af[4], bf[2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) af[mi] = sm.A[st][kr][wm * 32 + mi * 8 + (lane >> 2)];
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) bf[ni] = sm.B[st][kr][wn * 16 + ni * 8 + (lane >> 2)];
      if (O.dptr) {
        const double dk = sm.D[st][kr];
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) bf[ni] *= dk;
      }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  double(*Cs)[CLD] = reinterpret_cast<double(*)[CLD]>(&sm.A[0][0][0]);
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int row = wm * 32 + mi * 8 + (lane >> 2);
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) {
      const int col = wn * 16 + ni * 8 + 2 * (lane & 3);
      Cs[col][row] = acc[mi][ni][0];
      Cs[col + 1][row] = acc[mi][ni][1];
    }
  }
  __syncthreads();
  return Cs;
}

// intra-panel trailing tiles of wide panels (identity maps, no ordering):
// one tile per 256-thread CTA, C(i, j) -= A_i (D) A_j^T for i >= j
__global__ void __launch_bounds__(W8_THREADS, 3)
k_trail8(const UTile* __restrict__ tiles, const DevArgs* __restrict__ args) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  UpdSmem& sm = *reinterpret_cast<UpdSmem*>(smem_raw);
  const int tid = threadIdx.x;
  const UTile T = tiles[blockIdx.x];
  double* store = args->store;
  const bool ldlt = args->form == FORM_LDLT;
  const double* colk = store + T.soff + (i64)T.k0 * T.lds;
  const i64 lds = T.lds;
  Operands O{colk, lds, T.i0, T.ni, colk, lds, T.j0, T.nj, T.kn, ldlt ? colk + T.k0 : nullptr, lds + 1};
  double(*Cs)[CLD] = dmma_tile8(sm, O, tid);
  double* dst = store + T.doff;
  const i64 ldd = T.ldd;
  const int row = tid & (TM - 1), gi = T.i0 + row;
  if (row < T.ni) {
    constexpr int CSTEP = W8_THREADS / TM;  // 4 column phases
    for (int cb = tid >> 6; cb < T.nj; cb += 8 * CSTEP) {
      double v[8];
      double* pp[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int col = cb + u * CSTEP;
        const bool ok = col < T.nj && gi >= T.j0 + col;
        pp[u] = ok ? dst + (i64)(T.j0 + col) * ldd + gi : nullptr;
        v[u] = ok ? __ldcg(pp[u]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (pp[u]) __stcg(pp[u], v[u] - Cs[cb + u * CSTEP][row]);
    }
  }
}

// accumulator fragments -> Cs[col][row] (shared, reuses the operand stages)
__device__ __forceinline__ double (*stage_acc(UpdSmem& sm, double acc[4][4][2], int tid))[CLD] {
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  double(*Cs)[CLD] = reinterpret_cast<double(*)[CLD]>(&sm.A[0][0][0]);
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int row = wm * 32 + mi * 8 + (lane >> 2);
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const int col = wn * 32 + ni * 8 + (lane & 3) * 2;
      Cs[col][row] = acc[mi][ni][0];
      Cs[col + 1][row] = acc[mi][ni][1];
    }
  }
  __syncthreads();
  return Cs;
}

__global__ void __launch_bounds__(UPD_THREADS, UPD_MIN_CTAS)
k_update(const UTile* __restrict__ tiles, int ntiles, int* __restrict__ work_ctr,
         unsigned* __restrict__ counters, const DevArgs* __restrict__ args, PanelDev P,
         const i64* __restrict__ run_ptr, const int* __restrict__ run_src,
         const int* __restrict__ run_dst) {
  pdl_wait();  // programmatic dependent launch: wait for the previous grid
  extern __shared__ __align__(16) unsigned char smem_raw[];
  UpdSmem& sm = *reinterpret_cast<UpdSmem*>(smem_raw);
  const int tid = threadIdx.x;
  double* store = args->store;
  const bool ldlt = args->form == FORM_LDLT;

  while (true) {
    if (tid == 0) sm.tile = atomicAdd(work_ctr, 1);
    __syncthreads();
    const int t = sm.tile;
    if (t >= ntiles) {
      pdl_trigger();
      break;
    }
    const UTile T = tiles[t];
    unsigned long long* ttr = args->tile_trace ? args->tile_trace + 3 * (size_t)(&tiles[t] - args->tile_base) : nullptr;
    if (ttr && tid == 0) ttr[0] = gtimer();
    const double* src = store + T.soff;
    const i64 lds = T.lds;
    if (T.kn <= SMALL_W && T.couple >= 0 && T.mode == 0) {
      // narrow source (joint launch): CUDA-core tile, operands in the stage buffers
      double(*av)[TM] = reinterpret_cast<double(*)[TM]>(&sm.A[0][0][0]);
      double(*bv)[TN] = reinterpret_cast<double(*)[TN]>(&sm.B[0][0][0]);
      double* dsc = &sm.D[0][0];
      maps_load(sm, T.couple, T.ri, T.rj, run_ptr, run_src, run_dst, tid);
      if (tid < T.kn) {
        const int k = T.k0 + tid;
        dsc[tid] = ldlt ? __ldg(src + (i64)k * lds + k) : 1.0;
      }
      for (int idx = tid; idx < T.kn * TM; idx += UPD_THREADS) {
        const int k = idx / TM, r = idx % TM;
        const double* col = src + (i64)(T.k0 + k) * lds;
        if (r < T.ni) av[k][r] = __ldg(col + T.i0 + r);
        if (r < T.nj) bv[k][r] = __ldg(col + T.j0 + r);
      }
      __syncthreads();
      maps_search(sm, T.couple, T.i0, T.ni, T.j0, T.nj, tid);
      if (T.wait >= 0 && tid == 0) {
        while (ld_acquire(&counters[T.dst]) < (unsigned)T.wait) __nanosleep(32);
      }
      __syncthreads();
      double* dst = store + T.doff;
      const i64 ldd = T.ldd;
      const int tot = T.ni * T.nj;
      constexpr int U = 8;
      for (int e0 = tid; e0 < tot; e0 += UPD_THREADS * U) {
        double v[U], old[U];
        double* pp[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = e0 + UPD_THREADS * u;
          const int i = e % T.ni, j = e / T.ni;
          const bool ok = e < tot && T.i0 + i >= T.j0 + j;
          pp[u] = ok ? dst + (i64)sm.cmap[j] * ldd + sm.rmap[i] : nullptr;
          old[u] = ok ? __ldcg(pp[u]) : 0.0;
          double a = 0.0;
          if (ok)
            for (int k = 0; k < T.kn; ++k) a += av[k][i] * (bv[k][j] * dsc[k]);
          v[u] = a;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (pp[u]) __stcg(pp[u], old[u] - v[u]);
      }
      __syncthreads();
      if (T.signal && tid == 0) {
        __threadfence();
        atomicAdd(&counters[T.dst], 1u);
      }
      if (ttr && tid == 0) ttr[1] = ttr[2] = gtimer();
      continue;
    }
    const double* colk = src + (i64)T.k0 * lds;
    Operands O{colk, lds, T.i0, T.ni, colk, lds, T.j0, T.nj, T.kn,
               ldlt ? colk + T.k0 : nullptr, lds + 1};
    double acc[4][4][2];
    if (T.mode == 1) {
      // split-K partial: the product of this K range into the workspace,
      // fragment layout (coalesced: element e of thread tid at e * 128 + tid)
      dmma_mainloop(sm, O, acc, tid);
      double* W = args->splitk_ws + (i64)T.ws * (TM * TN);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int h = 0; h < 2; ++h) __stcg(W + ((a * 4 + b) * 2 + h) * UPD_THREADS + tid, acc[a][b][h]);
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        atomicAdd(&args->splitk_cnt[T.rc], 1u);
      }
      if (ttr && tid == 0) ttr[1] = ttr[2] = gtimer();
      continue;
    }
    maps_load(sm, T.couple, T.ri, T.rj, run_ptr, run_src, run_dst, tid);
    __syncthreads();
    maps_search(sm, T.couple, T.i0, T.ni, T.j0, T.nj, tid);
    if (T.mode == 2) {
      // split-K reduction: the partials in slot order (deterministic)
      if (tid == 0) {
        while (ld_acquire(&args->splitk_cnt[T.rc]) < (unsigned)T.nparts) __nanosleep(64);
      }
      __syncthreads();
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
      for (int sp = 0; sp < T.nparts; ++sp) {
        const double* W = args->splitk_ws + (i64)(T.ws + sp) * (TM * TN);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int h = 0; h < 2; ++h) acc[a][b][h] += __ldcg(W + ((a * 4 + b) * 2 + h) * UPD_THREADS + tid);
      }
    } else {
      if (!(args->pad & 64)) dmma_mainloop(sm, O, acc, tid);  // 64: timing ablation (debug)
    }

    if (ttr && tid == 0) ttr[1] = gtimer();
    // ordered, atomics-free scatter: wait for every lower-color source of
    // this destination
    if (T.wait >= 0 && tid == 0) {
      while (ld_acquire(&counters[T.dst]) < (unsigned)T.wait) __nanosleep(32);
    }
    double(*Cs)[CLD] = stage_acc(sm, acc, tid);
    double* dst = store + T.doff;
    const i64 ldd = T.ldd;
    const int row = tid & (TM - 1);
    const int dr = sm.rmap[row];
    const int gi = T.i0 + row;
    if (row < T.ni) {
      // 8 independent loads in flight per thread, then the 8 stores
      constexpr int CSTEP = UPD_THREADS / TM;
      for (int cb = tid >> 6; cb < T.nj; cb += 8 * CSTEP) {
        double v[8];
        double* pp[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int col = cb + u * CSTEP;
          const bool ok = col < T.nj && gi >= T.j0 + col;
          pp[u] = ok ? dst + (i64)sm.cmap[col] * ldd + dr : nullptr;
          v[u] = ok ? __ldcg(pp[u]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (pp[u]) __stcg(pp[u], v[u] - Cs[cb + u * CSTEP][row]);
        }
      }
    }
    __syncthreads();
    if (T.signal && tid == 0) {
      __threadfence();
      atomicAdd(&counters[T.dst], 1u);
    }
    if (ttr && tid == 0) ttr[2] = gtimer();
  }
}

// ---------------------------------------------------------------------------
// narrow sources (width <= SMALL_W): one CTA per tile on CUDA cores (the
// entries of a tile are independent; 8 loads in flight per thread).

#ifndef NARROW_MIN_CTAS
#define NARROW_MIN_CTAS 7  // resident CTAs per SM: 72 registers, no spills (10 and 12 measured slower)
#endif
__global__ void __launch_bounds__(32 * SMALL_WARPS, NARROW_MIN_CTAS)
k_update_small(const UTile* __restrict__ tiles, int ntiles, int* __restrict__ work_ctr,
               unsigned* __restrict__ counters, const DevArgs* __restrict__ args, PanelDev P,
               const i64* __restrict__ run_ptr, const int* __restrict__ run_src,
               const int* __restrict__ run_dst) {
  pdl_wait();  // programmatic dependent launch: wait for the previous grid
  constexpr int NT = 32 * SMALL_WARPS;
  struct MapSm {
    int rmap[TM], cmap[TN];
    int wsrc[2][TM], wdst[2][TM];
  };
  __shared__ MapSm ms;
  int* rmap = ms.rmap;
  int* cmap = ms.cmap;
  __shared__ double dsc[SMALL_W];
  __shared__ double av[SMALL_W][TM];
  __shared__ double bv[SMALL_W][TN];
  __shared__ int s_tile;
  const int tid = threadIdx.x;
  double* store = args->store;
  const bool ldlt = args->form == FORM_LDLT;
  // in-order tickets, the next one fetched while the current tile runs (a
  // CTA holding tickets t < t2 finishes t first: the smallest unfinished
  // ticket can always progress, as with one ticket at a time)
  if (tid == 0) s_tile = atomicAdd(work_ctr, 1);
  while (true) {
    __syncthreads();
    const int t = s_tile;
    if (t >= ntiles) {
      pdl_trigger();
      break;
    }
    int t_next = 0;
    if (tid == 0) t_next = atomicAdd(work_ctr, 1);
    const UTile T = tiles[t];
    unsigned long long* ttr = args->tile_trace ? args->tile_trace + 3 * (size_t)(&tiles[t] - args->tile_base) : nullptr;
    if (ttr && tid == 0) ttr[0] = gtimer();
    const double* src = store + T.soff;
    const i64 lds = T.lds;
    const int abl = args->pad;  // timing ablations (debug)
    // the wait's counter is read together with the operands: when the lower
    // colors are already done (the common case) it costs no extra latency
    unsigned seen = 0;
    if (T.wait >= 0 && tid == 0) seen = ld_acquire(&counters[T.dst]);
    if (!(abl & 4)) {
    maps_load(ms, T.couple, T.ri, T.rj, run_ptr, run_src, run_dst, tid);
    if (tid < T.kn) {
      const int k = T.k0 + tid;
      dsc[tid] = ldlt ? __ldg(src + (i64)k * lds + k) : 1.0;
    }
    // operands into shared memory (coalesced columns)
    for (int idx = tid; idx < T.kn * TM; idx += NT) {
      const int k = idx / TM, r = idx % TM;
      const double* col = src + (i64)(T.k0 + k) * lds;
      if (r < T.ni) av[k][r] = __ldg(col + T.i0 + r);
      if (r < T.nj) bv[k][r] = __ldg(col + T.j0 + r);
    }
    __syncthreads();
    maps_search(ms, T.couple, T.i0, T.ni, T.j0, T.nj, tid);
    }
    if (ttr && tid == 0) ttr[1] = gtimer();
    if (T.wait >= 0 && tid == 0 && seen < (unsigned)T.wait && !(abl & 256)) {
      while (ld_acquire(&counters[T.dst]) < (unsigned)T.wait) __nanosleep(32);
    }
    __syncthreads();
    double* dst = store + T.doff;
    const i64 ldd = T.ldd;
    const int tot = (abl & 6) ? 0 : T.ni * T.nj;
    constexpr int U = 8;
    for (int e0 = tid; e0 < tot; e0 += NT * U) {
      double v[U], old[U];
      double* pp[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = e0 + NT * u;
        const int i = e % T.ni, j = e / T.ni;
        const bool ok = e < tot && T.i0 + i >= T.j0 + j;
        pp[u] = ok ? dst + (i64)cmap[j] * ldd + rmap[i] : nullptr;
        old[u] = ok ? __ldcg(pp[u]) : 0.0;
        double a = 0.0;
        if (ok)
          for (int k = 0; k < T.kn; ++k) a += av[k][i] * (bv[k][j] * dsc[k]);
        v[u] = a;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (pp[u]) __stcg(pp[u], old[u] - v[u]);
    }
    __syncthreads();
    if (T.signal && tid == 0) {
      __threadfence();
      atomicAdd(&counters[T.dst], 1u);
    }
    if (ttr && tid == 0) ttr[2] = gtimer();
    if (tid == 0) s_tile = t_next;
  }
}



// ---------------------------------------------------------------------------
// narrow sources (width <= SMALL_W), one WARP per tile of <= 32 x 32 entries
// (the plan emits narrow couples in 32 x 32 tiles): four independent tiles per
// 128-thread CTA, warp-level barriers only.  Same protocol as k_update_small
// - in-order tickets (per warp, the next one fetched ahead), the couple's run
// window staged once per tile, the wait counter read with the operands, an
// atomics-free ordered scatter, fence + signal - at four times the tiles in
// flight per SM (the narrow updates are per-tile-latency bound: ~950 k tiles
// of mean width 1 at 60^3).
constexpr int NW_T = 32;
#ifndef NARROW_W_MIN_CTAS
#define NARROW_W_MIN_CTAS 8  // with NW_U 4: 64 registers, no spills (60^3: 6/U8 +0.3 ms, 11 +1.4 ms)
#endif
#ifndef NW_U
#define NW_U 4  // scatter entries in flight per lane
#endif
struct NarrowWarpSm {
  int rmap[NW_T], cmap[NW_T];
  int wsrc[2][NW_T], wdst[2][NW_T];
  double dsc[SMALL_W];
  double av[SMALL_W][NW_T], bv[SMALL_W][NW_T];
};
__global__ void __launch_bounds__(128, NARROW_W_MIN_CTAS)
k_update_narrow_w(const UTile* __restrict__ tiles, int ntiles, int* __restrict__ work_ctr,
                  unsigned* __restrict__ counters, const DevArgs* __restrict__ args,
                  const i64* __restrict__ run_ptr, const int* __restrict__ run_src,
                  const int* __restrict__ run_dst) {
  pdl_wait();
  __shared__ NarrowWarpSm sm_all[4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  NarrowWarpSm& sm = sm_all[warp];
  double* store = args->store;
  const bool ldlt = args->form == FORM_LDLT;
  const int abl = args->pad;  // timing ablations (debug)
  int t = 0;
  if (lane == 0) t = atomicAdd(work_ctr, 1);
  t = __shfl_sync(0xffffffffu, t, 0);
  while (t < ntiles) {
    int t_next = 0;
    if (lane == 0) t_next = atomicAdd(work_ctr, 1);
    const UTile T = tiles[t];
    const double* src = store + T.soff;
    const i64 lds = T.lds;
    unsigned seen = 0;
    if (T.wait >= 0 && lane == 0) seen = ld_acquire(&counters[T.dst]);
    if (!(abl & 4)) {
      if (T.couple >= 0) {
        const i64 end = __ldg(run_ptr + T.couple + 1);
        const int kr = T.ri + lane, kc = T.rj + lane;
        sm.wsrc[0][lane] = kr < end ? __ldg(run_src + kr) : 0x7fffffff;
        sm.wdst[0][lane] = kr < end ? __ldg(run_dst + kr) : 0;
        sm.wsrc[1][lane] = kc < end ? __ldg(run_src + kc) : 0x7fffffff;
        sm.wdst[1][lane] = kc < end ? __ldg(run_dst + kc) : 0;
      }
      for (int k = 0; k < T.kn; ++k) {
        const double* col = src + (i64)(T.k0 + k) * lds;
        if (lane < T.ni) sm.av[k][lane] = __ldg(col + T.i0 + lane);
        if (lane < T.nj) sm.bv[k][lane] = __ldg(col + T.j0 + lane);
      }
      if (lane < T.kn) sm.dsc[lane] = ldlt ? __ldg(src + (i64)(T.k0 + lane) * lds + T.k0 + lane) : 1.0;
      __syncwarp();
      // destination-local row / column of this lane's source row (i0 + lane)
      // and facing row (j0 + lane): last run start <= row in the window
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = (h ? T.j0 : T.i0) + lane;
        int v = row;
        if (T.couple >= 0) {
          const int* ws = sm.wsrc[h];
          int lo = 0, hi = NW_T - 1;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (ws[mid] <= row) lo = mid;
            else hi = mid - 1;
          }
          v = sm.wdst[h][lo] + (row - ws[lo]);
        }
        (h ? sm.cmap : sm.rmap)[lane] = v;
      }
    }
    if (T.wait >= 0 && lane == 0 && seen < (unsigned)T.wait && !(abl & 256)) {
      while (ld_acquire(&counters[T.dst]) < (unsigned)T.wait) __nanosleep(32);
    }
    __syncwarp();
    double* dst = store + T.doff;
    const i64 ldd = T.ldd;
    const int tot = (abl & 6) ? 0 : T.ni * T.nj;
    constexpr int U = NW_U;
    for (int e0 = lane; e0 < tot; e0 += 32 * U) {
      double v[U], old[U];
      double* pp[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = e0 + 32 * u;
        const int i = e % T.ni, j = e / T.ni;
        const bool ok = e < tot && T.i0 + i >= T.j0 + j;
        pp[u] = ok ? dst + (i64)sm.cmap[j] * ldd + sm.rmap[i] : nullptr;
        old[u] = ok ? __ldcg(pp[u]) : 0.0;
        double a = 0.0;
        if (ok)
          for (int k = 0; k < T.kn; ++k) a += sm.av[k][i] * (sm.bv[k][j] * sm.dsc[k]);
        v[u] = a;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (pp[u]) __stcg(pp[u], old[u] - v[u]);
    }
    __syncwarp();
    if (T.signal && lane == 0) {
      __threadfence();
      atomicAdd(&counters[T.dst], 1u);
    }
    t = __shfl_sync(0xffffffffu, t_next, 0);
  }
  pdl_trigger();
}

// ---------------------------------------------------------------------------
// narrow sources (width <= SMALL_W), batched: a work item is up to NB_MAX
// consecutive tiles of ONE color class (so none of them waits on another);
// the CTA issues all their descriptor / map / operand loads together, waits
// once for their lower colors, applies all their updates, then one fence and
// the signals.  About five memory latencies per batch instead of ~seven per
// tile (the narrow updates are latency-bound: tens of thousands of tiny tiles).
constexpr int NB_MAX = 8;
constexpr int NB_OPS = 3072;  // operand doubles per batch (plan-time budget)
struct NBatch {
  int first, count;  // tiles [first, first + count) of the tile array
};
struct NarrowBatchSm {
  UTile T[NB_MAX];
  i64 soff[NB_MAX], doff[NB_MAX];
  int sld[NB_MAX], dld[NB_MAX];
  int opoff[NB_MAX + 1];
  int map[NB_MAX][2][TM];
  int wsrc[NB_MAX][2][TM], wdst[NB_MAX][2][TM];
  double ops[NB_OPS];
  int s_batch;
};

__global__ void __launch_bounds__(UPD_THREADS)
k_update_narrow_batch(const NBatch* __restrict__ batches, int nbatches, const UTile* __restrict__ tiles,
                      int* __restrict__ work_ctr, unsigned* __restrict__ counters,
                      const DevArgs* __restrict__ args, PanelDev P, const i64* __restrict__ run_ptr,
                      const int* __restrict__ run_src, const int* __restrict__ run_dst) {
  pdl_wait();  // programmatic dependent launch: wait for the previous grid
  extern __shared__ __align__(16) unsigned char smem_raw[];
  NarrowBatchSm& sm = *reinterpret_cast<NarrowBatchSm*>(smem_raw);
  const int tid = threadIdx.x;
  double* store = args->store;
  const bool ldlt = args->form == FORM_LDLT;
  while (true) {
    if (tid == 0) sm.s_batch = atomicAdd(work_ctr, 1);
    __syncthreads();
    const int bi = sm.s_batch;
    if (bi >= nbatches) break;
    const NBatch B = batches[bi];
    const int nb = B.count;
    // 1. descriptors + panel offsets
    {
      constexpr int W = sizeof(UTile) / sizeof(int);
      for (int e = tid; e < nb * W; e += UPD_THREADS)
        reinterpret_cast<int*>(sm.T)[e] = reinterpret_cast<const int*>(tiles + B.first)[e];
    }
    __syncthreads();
    if (tid < nb) {
      const UTile& T = sm.T[tid];
      sm.soff[tid] = P.off[T.src];
      sm.sld[tid] = P.nrows[T.src];
      sm.doff[tid] = P.off[T.dst];
      sm.dld[tid] = P.nrows[T.dst];
    }
    if (tid == 0) {
      int o = 0;
      for (int b = 0; b < nb; ++b) {
        sm.opoff[b] = o;
        o += sm.T[b].kn * (sm.T[b].ni + sm.T[b].nj + 1);
      }
      sm.opoff[nb] = o;
    }
    // run windows of every tile (rows: side 0 from ri, columns: side 1 from rj)
    for (int e = tid; e < nb * 2 * TM; e += UPD_THREADS) {
      const int b = e / (2 * TM), h = (e / TM) & 1, x = e % TM;
      const UTile& T = sm.T[b];
      const i64 end = __ldg(run_ptr + T.couple + 1);
      const int k = (h ? T.rj : T.ri) + x;
      sm.wsrc[b][h][x] = k < end ? __ldg(run_src + k) : 0x7fffffff;
      sm.wdst[b][h][x] = k < end ? __ldg(run_dst + k) : 0;
    }
    __syncthreads();
    // 2. operands of all tiles: per tile k-major [a(ni) b(nj)] then d(kn)
    const int nops = sm.opoff[nb];
    for (int e = tid; e < nops; e += UPD_THREADS) {
      int b = 0;
      while (b + 1 < nb && sm.opoff[b + 1] <= e) ++b;
      const UTile& T = sm.T[b];
      const int o = e - sm.opoff[b], span = T.ni + T.nj;
      const double* src = store + sm.soff[b];
      const i64 lds = sm.sld[b];
      double v;
      if (o < T.kn * span) {
        const int k = o / span, r = o - k * span;
        const int row = r < T.ni ? T.i0 + r : T.j0 + (r - T.ni);
        v = __ldg(src + (i64)(T.k0 + k) * lds + row);
      } else {
        const int k = T.k0 + (o - T.kn * span);
        v = ldlt ? __ldg(src + (i64)k * lds + k) : 1.0;
      }
      sm.ops[e] = v;
    }
    // maps (binary search in the windows)
    for (int e = tid; e < nb * 2 * TM; e += UPD_THREADS) {
      const int b = e / (2 * TM), h = (e / TM) & 1, x = e % TM;
      const UTile& T = sm.T[b];
      const int row = (h ? T.j0 : T.i0) + x;
      int v = 0;
      if (x < (h ? T.nj : T.ni)) {
        const int* ws = sm.wsrc[b][h];
        int lo = 0, hi = TM - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (ws[mid] <= row) lo = mid;
          else hi = mid - 1;
        }
        v = sm.wdst[b][h][lo] + (row - ws[lo]);
      }
      sm.map[b][h][x] = v;
    }
    // 3. lower colors of every tile (tiles of one class never wait on each other)
    if (tid < nb && sm.T[tid].wait >= 0) {
      const unsigned* c = &counters[sm.T[tid].dst];
      while (ld_acquire(c) < (unsigned)sm.T[tid].wait) __nanosleep(32);
    }
    __syncthreads();
    // 4. all updates, flattened over the batch, 8 in flight per thread
    {
      int tot = 0;
      for (int b = 0; b < nb; ++b) tot += sm.T[b].ni * sm.T[b].nj;
      constexpr int U = 8;
      for (int e0 = tid; e0 < tot; e0 += UPD_THREADS * U) {
        double v[U], old[U];
        double* pp[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          int e = e0 + UPD_THREADS * u;
          pp[u] = nullptr;
          v[u] = 0.0;
          old[u] = 0.0;
          if (e < tot) {
            int b = 0;
            while (e >= sm.T[b].ni * sm.T[b].nj) {
              e -= sm.T[b].ni * sm.T[b].nj;
              ++b;
            }
            const UTile& T = sm.T[b];
            const int i = e % T.ni, j = e / T.ni;
            if (T.i0 + i >= T.j0 + j) {
              pp[u] = store + sm.doff[b] + (i64)sm.map[b][1][j] * sm.dld[b] + sm.map[b][0][i];
              old[u] = __ldcg(pp[u]);
              const double* o = sm.ops + sm.opoff[b];
              const int span = T.ni + T.nj;
              const double* dk = o + T.kn * span;
              double a = 0.0;
              for (int k = 0; k < T.kn; ++k) a += o[k * span + i] * (o[k * span + T.ni + j] * dk[k]);
              v[u] = a;
            }
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (pp[u]) __stcg(pp[u], old[u] - v[u]);
      }
    }
    __syncthreads();
    // 5. one fence, then the signals
    if (tid == 0) __threadfence();
    __syncthreads();
    if (tid < nb && sm.T[tid].signal) atomicAdd(&counters[sm.T[tid].dst], 1u);
  }
}

// ---------------------------------------------------------------------------
// narrow sources (width <= SMALL_W), destination-tiled gather: a CTA owns one
// 64x64 destination tile in shared memory, applies every narrow segment that
// lands in it (source order, one segment at a time), and writes it back once.
// No inter-CTA ordering, no fences, one read + one write of the destination.

__global__ void __launch_bounds__(UPD_THREADS)
k_gather_narrow(const NItem* __restrict__ items, const NSeg* __restrict__ segs,
                const DevArgs* __restrict__ args, PanelDev P, const i64* __restrict__ run_ptr,
                const int* __restrict__ run_src, const int* __restrict__ run_dst) {
  pdl_wait();  // programmatic dependent launch: wait for the previous grid
  pdl_trigger();  // (not persistent: every CTA of the grid has started)
  __shared__ double T[TN][TM + 1];
  __shared__ double av[SMALL_W][TM];
  __shared__ double bv[SMALL_W][TN];
  __shared__ double dsc[SMALL_W];
  __shared__ int rmap[TM], cmap[TN];
  const int tid = threadIdx.x;
  const NItem it = items[blockIdx.x];
  double* store = args->store;
  const bool ldlt = args->form == FORM_LDLT;
  double* dst = store + P.off[it.q];
  const i64 ldd = P.nrows[it.q];
  {
    const int r = tid & (TM - 1);
    for (int c = tid >> 6; c < it.nc; c += UPD_THREADS / TM)
      if (r < it.nr) T[c][r] = __ldcg(dst + (i64)(it.c0 + c) * ldd + it.r0 + r);
  }
  for (int sidx = 0; sidx < it.nseg; ++sidx) {
    const NSeg g = segs[it.seg0 + sidx];
    const double* src = store + P.off[g.p];
    const i64 lds = P.nrows[g.p];
    const int ni = g.s1 - g.s0, nj = g.f1 - g.f0, kn = P.width[g.p];
    if (tid < TM) {
      if (tid < ni) rmap[tid] = map_row(g.s0 + tid, g.couple, g.rs, run_ptr, run_src, run_dst) - it.r0;
    } else if (tid - TM < nj) {
      cmap[tid - TM] = map_row(g.f0 + tid - TM, g.couple, g.rf, run_ptr, run_src, run_dst) - it.c0;
    }
    if (tid < kn) dsc[tid] = ldlt ? __ldg(src + (i64)tid * lds + tid) : 1.0;
    for (int idx = tid; idx < kn * TM; idx += UPD_THREADS) {
      const int k = idx / TM, r = idx % TM;
      const double* col = src + (i64)k * lds;
      if (r < ni) av[k][r] = __ldg(col + g.s0 + r);
      if (r < nj) bv[k][r] = __ldg(col + g.f0 + r);
    }
    __syncthreads();
    const int tot = ni * nj;
    for (int e = tid; e < tot; e += UPD_THREADS) {
      const int i = e % ni, j = e / ni;
      if (g.s0 + i < g.f0 + j) continue;
      double a = 0.0;
      for (int k = 0; k < kn; ++k) a += av[k][i] * (bv[k][j] * dsc[k]);
      T[cmap[j]][rmap[i]] -= a;
    }
    __syncthreads();
  }
  {
    const int r = tid & (TM - 1);
    for (int c = tid >> 6; c < it.nc; c += UPD_THREADS / TM)
      if (r < it.nr) __stcg(dst + (i64)(it.c0 + c) * ldd + it.r0 + r, T[c][r]);
  }
}

// ---------------------------------------------------------------------------
// diagonal block factorization in shared memory (nb <= NBMAX), one barrier
// per pivot: at step j every row r > j subtracts (A_rj / piv) * A_cj from
// A_rc for c in (j, r] (the LLt and the LDLt update alike); column j is then
// scaled (1/sqrt(piv) or 1/piv).  D[col][row], lower part.  Records the
// first failing pivot (reference predicates: LLt piv <= thr, LDLt |piv| <=
// thr).  rdiag[j] = 1 / stored diagonal (sqrt(piv) or d_j).

template <int NBMAX, int NT>
__device__ __forceinline__ void factor_diag_smem(double (*D)[NBMAX + 1], double* rdiag, int nb,
                                                 bool ldlt, double thr, int* s_fail,
                                                 double* s_fpiv, int tid) {
  const int rr_off = tid >> 1, half = tid & 1;
  for (int j = 0; j < nb; ++j) {
    const double piv = D[j][j];
    const double ipiv = 1.0 / piv;
    const int rr = j + 1 + rr_off;
    if (rr < nb && rr_off < NT / 2) {
      // all shared loads of the step first (independent), then the stores
      const double lr = D[j][rr] * ipiv;
      double cj[NBMAX / 2], dr[NBMAX / 2];
#pragma unroll
      for (int u = 0; u < NBMAX / 2; ++u) {
        const int c = j + 1 + half + 2 * u;
        const bool ok = c <= rr;
        cj[u] = ok ? D[j][c] : 0.0;
        dr[u] = ok ? D[c][rr] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < NBMAX / 2; ++u) {
        const int c = j + 1 + half + 2 * u;
        if (c <= rr) D[c][rr] = dr[u] - lr * cj[u];
      }
    }
    if (tid == 0) {
      const bool bad = ldlt ? (fabs(piv) <= thr) : (piv <= thr);
      if (bad && *s_fail < 0) {
        *s_fail = j;
        *s_fpiv = piv;
      }
    }
    __syncthreads();
    const double dv = ldlt ? piv : sqrt(piv);
    const double inv = 1.0 / dv;
    if (half == 0 && rr < nb) D[j][rr] *= inv;
    if (tid == 0) {
      D[j][j] = dv;
      rdiag[j] = inv;
    }
  }
  __syncthreads();
}

// reciprocal / reciprocal square root: hardware approximation + Newton.
// rcp.approx.f64 (MUFU.RCP64H) is good to ~20 bits; each iteration squares
// the relative error: 2 iterations -> ~2^-80, below double rounding (the
// reciprocal is then within 1 ulp; pivots feed a 1e-12 parity bound).
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.f64 %0, %1;" : "=d"(y) : "d"(x));
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double e = fma(-x * y, y, 1.0);
    y = fma(0.5 * y, e, y);
  }
  return y;
}

// Fused diagonal factorization + inverse (wide panels).  Right-looking with
// one barrier per pivot; row r > j of the Schur complement and row r of
// W = L^-1 (Gauss-Jordan on an identity, held in D's free strict upper
// triangle: W[r][c] at D[r][c], c < r) are updated with unscaled column j
// (coefficient A_rj / piv), so the inverse costs no extra serial steps.
__device__ __forceinline__ void factor_inv_smem(double (*D)[FNB + 1], double* rdiag, int nb,
                                                bool ldlt, double thr, int* s_fail,
                                                double* s_fpiv, int tid) {
  const int rr_off = tid >> 1, half = tid & 1;
  for (int j = 0; j < nb; ++j) {
    const double piv = D[j][j];
    const int rr = j + 1 + rr_off;
    const double arj = rr < nb ? D[j][rr] : 0.0;
    double inv, ipiv;
    if (ldlt) {
      ipiv = rcp_nr(piv);
      inv = ipiv;
    } else {
      inv = rsqrt_nr(piv);
      ipiv = inv * inv;
    }
    if (rr < nb) {
      const double lr = arj * ipiv;
      // Schur complement: columns c in (j, rr] of this thread's parity
      for (int c0 = j + 1 + half; c0 <= rr; c0 += 16) {
        double cj[8], dr[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int c = c0 + 2 * u;
          cj[u] = c <= rr ? D[j][c] : 0.0;
          dr[u] = c <= rr ? D[c][rr] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int c = c0 + 2 * u;
          if (c <= rr) D[c][rr] = dr[u] - lr * cj[u];
        }
      }
      // inverse rows: W[rr][c] -= lr * W~[j][c], c in [0, j] (W~[j][j] = 1)
      for (int c0 = half; c0 <= j; c0 += 16) {
        double wj[8], wr[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int c = c0 + 2 * u;
          wj[u] = c < j ? D[j][c] : (c == j ? 1.0 : 0.0);
          wr[u] = c <= j ? D[rr][c] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int c = c0 + 2 * u;
          if (c <= j) D[rr][c] = wr[u] - lr * wj[u];
        }
      }
    }
    if (tid == 0) {
      const bool bad = ldlt ? (fabs(piv) <= thr) : (piv <= thr);
      if (bad && *s_fail < 0) {
        *s_fail = j;
        *s_fpiv = piv;
      }
    }
    __syncthreads();
    if (half == 0 && rr < nb) D[j][rr] = arj * inv;   // L column j
    if (!ldlt && tid < j) D[j][tid] *= inv;           // W row j (LLt: / L_jj)
    if (tid == 0) {
      D[j][j] = ldlt ? piv : piv * inv;
      rdiag[j] = inv;
    }
  }
  __syncthreads();
}

// Balanced fused factorization + inverse.  At pivot j, row r > j touches
// every entry c <= r of its row: the Schur entry A_rc (c > j, at D[c][r])
// or the inverse entry W_rc (c <= j, at D[r][c]), both as
//   target -= (A_rj / piv) * op,   op = D[j][c] (c != j), 1 (c == j).
// So the work of a row does not depend on j, and a static assignment of
// (row, 10-column chunk) to the 256 threads balances every step (<= 10
// entries per thread per pivot, 8 warps to hide latency).
constexpr int DIAG_THREADS = 256;
constexpr int DIAG_CHUNK = 10;

// ABL: ablation (microbenchmarks only): 1 no update, 2 no barrier, 3 barriers only.
// NT threads, CHUNK columns per thread and pivot: sum_r ceil((r+1)/CHUNK) <= NT
// (256/10 and 128/22).
template <int ABL = 0, int CHUNK = DIAG_CHUNK>
__device__ __forceinline__ void factor_inv_smem_bal(double (*D)[FNB + 1], double* rdiag, int nb,
                                                    bool ldlt, double thr, int* s_fail,
                                                    double* s_fpiv, int tid) {
  constexpr int DIAG_CHUNK = CHUNK;
  // static map: thread -> (row, first column) ; rows need ceil((r+1)/CHUNK) threads
  int my_r = FNB, my_c = 0;
  {
    int t = 0;
    for (int r = 0; r < FNB && my_r == FNB; ++r) {
      const int n = (r + DIAG_CHUNK) / DIAG_CHUNK;
      if (tid < t + n) {
        my_r = r;
        my_c = (tid - t) * DIAG_CHUNK;
      }
      t += n;
    }
  }
  for (int j = 0; j < nb; ++j) {
    if (ABL == 3) {
      __syncthreads();
      continue;
    }
    const double piv = D[j][j];
    double inv, ipiv;
    if (ldlt) {
      ipiv = rcp_nr(piv);
      inv = ipiv;
    } else {
      inv = rsqrt_nr(piv);
      ipiv = inv * inv;
    }
    const int r = my_r;
    double arj = 0.0;
    if (ABL != 1 && r > j && r < nb) {
      // straight-line: shared offsets (no pointer arrays), unconditional
      // loads from clamped in-bounds slots, predicated stores
      double* Df = &D[0][0];
      arj = Df[j * (FNB + 1) + r];
      const double lr = arj * ipiv;
      constexpr int HB = DIAG_CHUNK > 11 ? (DIAG_CHUNK + 1) / 2 : DIAG_CHUNK;  // register batch
#pragma unroll
      for (int h = 0; h < DIAG_CHUNK; h += HB) {
        double op[HB], tv[HB];
        int ti[HB];
#pragma unroll
        for (int u = 0; u < HB; ++u) {
          const int c = min(my_c + h + u, FNB - 1);
          ti[u] = c > j ? c * (FNB + 1) + r : r * (FNB + 1) + c;
          const double o = Df[j * (FNB + 1) + c];
          op[u] = c == j ? 1.0 : o;
          tv[u] = Df[ti[u]];
        }
#pragma unroll
        for (int u = 0; u < HB; ++u)
          if (h + u < DIAG_CHUNK && my_c + h + u <= r) Df[ti[u]] = tv[u] - lr * op[u];
      }
    }
    if (tid == 0) {
      const bool bad = ldlt ? (fabs(piv) <= thr) : (piv <= thr);
      if (bad && *s_fail < 0) {
        *s_fail = j;
        *s_fpiv = piv;
      }
    }
    if (ABL != 2) __syncthreads();
    if (my_c == 0 && r > j && r < nb) D[j][r] = arj * inv;   // L column j
    if (!ldlt && tid < j) D[j][tid] *= inv;                  // W row j (LLt: / L_jj)
    if (tid == 0) {
      D[j][j] = ldlt ? piv : piv * inv;
      rdiag[j] = inv;
    }
  }
  __syncthreads();
}

// Leaner variant of factor_diag_smem: one long-latency op per pivot
// (rsqrt for LLt, reciprocal for LDLt) and work-proportional batches of 8
// columns (all shared loads of a batch issued before its stores).
template <int NBMAX, int NT>
__device__ __forceinline__ void factor_diag_smem2(double (*D)[NBMAX + 1], double* rdiag, int nb,
                                                  bool ldlt, double thr, int* s_fail,
                                                  double* s_fpiv, int tid) {
  const int rr_off = tid >> 1, half = tid & 1;
  for (int j = 0; j < nb; ++j) {
    const double piv = D[j][j];
    const int rr = j + 1 + rr_off;
    double arj = 0.0;
    if (rr < nb) arj = D[j][rr];
    double inv, ipiv, dv;
    if (ldlt) {
      ipiv = rcp_nr(piv);
      inv = ipiv;
      dv = piv;
    } else {
      inv = rsqrt_nr(piv);
      ipiv = inv * inv;
      dv = piv * inv;
    }
    if (rr < nb && rr_off < NT / 2) {
      const double lr = arj * ipiv;
      for (int c0 = j + 1 + half; c0 <= rr; c0 += 16) {
        double cj[8], dr[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int c = c0 + 2 * u;
          cj[u] = c <= rr ? D[j][c] : 0.0;
          dr[u] = c <= rr ? D[c][rr] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int c = c0 + 2 * u;
          if (c <= rr) D[c][rr] = dr[u] - lr * cj[u];
        }
      }
    }
    if (tid == 0) {
      const bool bad = ldlt ? (fabs(piv) <= thr) : (piv <= thr);
      if (bad && *s_fail < 0) {
        *s_fail = j;
        *s_fpiv = piv;
      }
    }
    __syncthreads();
    if (half == 0 && rr < nb) D[j][rr] = arj * inv;
    if (tid == 0) {
      D[j][j] = dv;
      rdiag[j] = inv;
    }
  }
  __syncthreads();
}

// small panels: width 2..SNB, thread per row solve (x[SNB] in registers)
__global__ void __launch_bounds__(FTR)
k_factor_small(const FItem* __restrict__ items, const DevArgs* __restrict__ args, PanelDev P,
               i64* __restrict__ fail_col, double* __restrict__ fail_piv) {
  pdl_wait();  // programmatic dependent launch: wait for the previous grid
  pdl_trigger();  // (not persistent: every CTA of the grid has started)
  if (args->pad & 32) return;  // timing ablation (debug)
  __shared__ double D[SNB][SNB + 1];
  __shared__ double rdiag[SNB];
  __shared__ int s_fail;
  __shared__ double s_fpiv;
  const FItem it = items[blockIdx.x];
  const int tid = threadIdx.x;
  const bool ldlt = args->form == FORM_LDLT;
  double* base = args->store + P.off[it.p];
  const i64 ld = P.nrows[it.p];
  const int nb = it.nb, c0 = it.c0;
  for (int idx = tid; idx < nb * nb; idx += FTR) {
    const int c = idx / nb, r = idx % nb;
    D[c][r] = r >= c ? base[(i64)(c0 + c) * ld + c0 + r] : 0.0;
  }
  if (tid == 0) s_fail = -1;
  __syncthreads();
  if (it.diag) {
    factor_diag_smem2<SNB, FTR>(D, rdiag, nb, ldlt, args->thr, &s_fail, &s_fpiv, tid);
    for (int idx = tid; idx < nb * nb; idx += FTR) {
      const int c = idx / nb, r = idx % nb;
      if (r >= c) base[(i64)(c0 + c) * ld + c0 + r] = D[c][r];
    }
    if (tid == 0 && s_fail >= 0 && fail_col[it.p] == NO_FAIL) {
      fail_col[it.p] = P.fc[it.p] + c0 + s_fail;
      fail_piv[it.p] = s_fpiv;
    }
  } else {
    for (int j = tid; j < nb; j += FTR) rdiag[j] = 1.0 / D[j][j];
  }
  if (it.nr == 0) return;
  __syncthreads();
  // T into the strict upper triangle: D[k][j] = L_kj (LLt) / d_j L_kj (LDLt)
  for (int idx = tid; idx < nb * nb; idx += FTR) {
    const int j = idx / nb, k = idx % nb;
    if (k > j) D[k][j] = ldlt ? D[j][k] * D[j][j] : D[j][k];
  }
  __syncthreads();
  if (tid < it.nr) {
    double* rowp = base + it.r0 + tid;
    double x[SNB];
#pragma unroll
    for (int k = 0; k < SNB; ++k)
      if (k < nb) x[k] = rowp[(i64)(c0 + k) * ld];
#pragma unroll
    for (int j = 0; j < SNB; ++j) {
      if (j < nb) {
        const double xj = x[j] * rdiag[j];
        x[j] = xj;
#pragma unroll
        for (int k = j + 1; k < SNB; ++k)
          if (k < nb) x[k] -= xj * D[k][j];
      }
    }
#pragma unroll
    for (int k = 0; k < SNB; ++k)
      if (k < nb) rowp[(i64)(c0 + k) * ld] = x[k];
  }
}

// wide panels, one 64-column block: factor the diagonal block, write it
// back, and store G (FNB x FNB, column-major) in the scratch slot with
//   LLt : G[j][k] = (L^-1)[j][k]          (X = B L^-T       = B G^T)
//   LDLt: G[j][k] = (L^-1)[j][k] / d_j    (X = B L^-T D^-1  = B G^T)
template <int MODE = 3, int VARIANT = 3>
__global__ void __launch_bounds__(DIAG_THREADS)
k_factor_diag(const FItem* __restrict__ items, const DevArgs* __restrict__ args, PanelDev P,
              i64* __restrict__ fail_col, double* __restrict__ fail_piv) {
  __shared__ double D[FNB][FNB + 1];
  __shared__ double rdiag[FNB];
  __shared__ int s_fail;
  __shared__ double s_fpiv;
  const FItem it = items[blockIdx.x];
  const int tid = threadIdx.x;
  const bool ldlt = args->form == FORM_LDLT;
  double* base = args->store + P.off[it.p];
  const i64 ld = P.nrows[it.p];
  const int nb = it.nb, c0 = it.c0;
  // load: thread t reads rows of column blocks (coalesced), all loads first
  {
    constexpr int CP = DIAG_THREADS / FNB;  // column parities
    const int r = tid & 63, cpar = tid >> 6;
    double v[FNB / CP];
#pragma unroll
    for (int u = 0; u < FNB / CP; ++u) {
      const int c = cpar + CP * u;
      v[u] = (c < nb && r < nb && r >= c) ? __ldg(base + (i64)(c0 + c) * ld + c0 + r) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < FNB / CP; ++u) D[cpar + CP * u][r] = v[u];
  }
  if (tid == 0) s_fail = -1;
  __syncthreads();
  if (VARIANT >= 3) {
    if (VARIANT == 3) factor_inv_smem_bal<0>(D, rdiag, nb, ldlt, args->thr, &s_fail, &s_fpiv, tid);
    if (VARIANT == 4) factor_inv_smem_bal<1>(D, rdiag, nb, ldlt, args->thr, &s_fail, &s_fpiv, tid);
    if (VARIANT == 5) factor_inv_smem_bal<2>(D, rdiag, nb, ldlt, args->thr, &s_fail, &s_fpiv, tid);
    if (VARIANT == 6) factor_inv_smem_bal<3>(D, rdiag, nb, ldlt, args->thr, &s_fail, &s_fpiv, tid);
  } else if (VARIANT == 2) {
    if (tid < 128) factor_inv_smem(D, rdiag, nb, ldlt, args->thr, &s_fail, &s_fpiv, tid);
    else for (int j = 0; j < nb; ++j) { __syncthreads(); }
    __syncthreads();
  } else if (MODE & 1) {
    if (VARIANT == 0) factor_diag_smem<FNB, DIAG_THREADS>(D, rdiag, nb, ldlt, args->thr, &s_fail, &s_fpiv, tid);
    else factor_diag_smem2<FNB, DIAG_THREADS>(D, rdiag, nb, ldlt, args->thr, &s_fail, &s_fpiv, tid);
  } else {
    for (int j = tid; j < nb; j += DIAG_THREADS) rdiag[j] = 1.0 / D[j][j];
    __syncthreads();
  }
  {
    constexpr int CP = DIAG_THREADS / FNB;
    const int r = tid & 63, cpar = tid >> 6;
#pragma unroll 4
    for (int c = cpar; c < nb; c += CP)
      if (r < nb && r >= c) base[(i64)(c0 + c) * ld + c0 + r] = D[c][r];
  }
  if (tid == 0 && s_fail >= 0 && fail_col[it.p] == NO_FAIL) {
    fail_col[it.p] = P.fc[it.p] + c0 + s_fail;
    fail_piv[it.p] = s_fpiv;
  }
  double* G = args->scratch + (i64)it.g * FNB * FNB;
  if (VARIANT >= 2) {
    // G[j][k] = W[j][k] (LLt) or W[j][k] / d_j (LDLt); W[j][j] = rdiag[j] (LLt) or 1
    const int j = tid & 63, kpar = tid >> 6;
    for (int k = kpar; k < FNB; k += DIAG_THREADS / FNB) {
      double g = 0.0;
      if (j < nb && k < nb && k <= j) {
        if (k == j) g = rdiag[j];
        else g = ldlt ? D[j][k] * rdiag[j] : D[j][k];
      }
      G[(i64)k * FNB + j] = g;
    }
    return;
  }
  // inverse of the (unit, for LDLt) lower factor: thread c < nb owns column
  // c: y_r = (delta_rc - sum_{k<r} L_rk y_k) / L_rr, y_k = 0 for k < c
  if ((MODE & 2) && tid < FNB) {
    const int c = tid;
    double y[FNB];
#pragma unroll
    for (int r = 0; r < FNB; ++r) {
      if (r < nb) {
        double s0 = r == c ? 1.0 : 0.0, s1 = 0.0;
#pragma unroll
        for (int k = 0; k + 1 < r; k += 2) {
          s0 -= D[k][r] * y[k];
          s1 -= D[k + 1][r] * y[k + 1];
        }
        if (r & 1) s0 -= D[r - 1][r] * y[r - 1];
        const double rd = ldlt ? 1.0 : rdiag[r];
        y[r] = (r >= c && c < nb) ? (s0 + s1) * rd : 0.0;
      } else {
        y[r] = 0.0;
      }
    }
#pragma unroll
    for (int j = 0; j < FNB; ++j)
      if (j < nb) G[(i64)c * FNB + j] = ldlt ? y[j] * rdiag[j] : y[j];
  }
}

// wide-panel TRSM as a DMMA GEMM, in place: X[r0:r0+nr, c0:c0+nb] =
// B[r0:r0+nr, c0:c0+nb] G^T  (one 64-row tile per CTA)
__global__ void __launch_bounds__(UPD_THREADS, 3)
k_trsm(const FItem* __restrict__ items, const DevArgs* __restrict__ args, PanelDev P) {
  pdl_wait();  // programmatic dependent launch: wait for the previous grid
  pdl_trigger();  // (not persistent: every CTA of the grid has started)
  if (args->pad & 16) return;  // timing ablation (debug)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  UpdSmem& sm = *reinterpret_cast<UpdSmem*>(smem_raw);
  const int tid = threadIdx.x;
  const FItem it = items[blockIdx.x];
  double* base = args->store + P.off[it.p];
  const i64 ld = P.nrows[it.p];
  const double* G = args->scratch + (i64)it.g * FNB * FNB;
  double* colc = base + (i64)it.c0 * ld;
  Operands O{colc, ld, it.r0, it.nr, G, FNB, 0, it.nb, it.nb, nullptr, 0};
  double acc[4][4][2];
  dmma_mainloop(sm, O, acc, tid);
  double(*Cs)[CLD] = stage_acc(sm, acc, tid);
  const int row = tid & (TM - 1);
  if (row < it.nr) {
    for (int col = tid >> 6; col < it.nb; col += UPD_THREADS / TM)
      colc[(i64)col * ld + it.r0 + row] = Cs[col][row];
  }
}

// inter-panel update tiles (mode 0) on 8-warp CTAs: the k_update protocol -
// in-order tickets, the couple's run-window maps, the ordered atomics-free
// scatter behind the color counter, fence + signal - around dmma_tile8
__global__ void __launch_bounds__(W8_THREADS, 3)
k_update8(const UTile* __restrict__ tiles, int ntiles, int* __restrict__ work_ctr,
          unsigned* __restrict__ counters, const DevArgs* __restrict__ args,
          const i64* __restrict__ run_ptr, const int* __restrict__ run_src,
          const int* __restrict__ run_dst) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  UpdSmem& sm = *reinterpret_cast<UpdSmem*>(smem_raw);
  const int tid = threadIdx.x;
  double* store = args->store;
  const bool ldlt = args->form == FORM_LDLT;
  while (true) {
    if (tid == 0) sm.tile = atomicAdd(work_ctr, 1);
    __syncthreads();
    const int t = sm.tile;
    if (t >= ntiles) {
      pdl_trigger();
      break;
    }
    const UTile T = tiles[t];
    const i64 lds = T.lds;
    const double* colk = store + T.soff + (i64)T.k0 * lds;
    if (tid < 128) maps_load(sm, T.couple, T.ri, T.rj, run_ptr, run_src, run_dst, tid);
    __syncthreads();
    if (tid < 128) maps_search(sm, T.couple, T.i0, T.ni, T.j0, T.nj, tid);
    Operands O{colk, lds, T.i0, T.ni, colk, lds, T.j0, T.nj, T.kn, ldlt ? colk + T.k0 : nullptr,
               lds + 1};
    double(*Cs)[CLD] = dmma_tile8(sm, O, tid);  // (its barriers also publish the maps)
    if (T.wait >= 0 && tid == 0) {
      while (ld_acquire(&counters[T.dst]) < (unsigned)T.wait) __nanosleep(32);
    }
    __syncthreads();
    double* dst = store + T.doff;
    const i64 ldd = T.ldd;
    const int row = tid & (TM - 1);
    const int dr = sm.rmap[row];
    const int gi = T.i0 + row;
    if (row < T.ni) {
      constexpr int CSTEP = W8_THREADS / TM;
      for (int cb = tid >> 6; cb < T.nj; cb += 8 * CSTEP) {
        double v[8];
        double* pp[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int col = cb + u * CSTEP;
          const bool ok = col < T.nj && gi >= T.j0 + col;
          pp[u] = ok ? dst + (i64)sm.cmap[col] * ldd + dr : nullptr;
          v[u] = ok ? __ldcg(pp[u]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (pp[u]) __stcg(pp[u], v[u] - Cs[cb + u * CSTEP][row]);
      }
    }
    __syncthreads();
    if (T.signal && tid == 0) {
      __threadfence();
      atomicAdd(&counters[T.dst], 1u);
    }
  }
}

// the same TRSM tile on an 8-warp CTA (dmma_tile8: bitwise identical)
__global__ void __launch_bounds__(W8_THREADS, 3)
k_trsm8(const FItem* __restrict__ items, const DevArgs* __restrict__ args, PanelDev P) {
  pdl_wait();
  pdl_trigger();
  if (args->pad & 16) return;  // timing ablation (debug)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  UpdSmem& sm = *reinterpret_cast<UpdSmem*>(smem_raw);
  const int tid = threadIdx.x;
  const FItem it = items[blockIdx.x];
  double* base = args->store + P.off[it.p];
  const i64 ld = P.nrows[it.p];
  const double* G = args->scratch + (i64)it.g * FNB * FNB;
  double* colc = base + (i64)it.c0 * ld;
  Operands O{colc, ld, it.r0, it.nr, G, FNB, 0, it.nb, it.nb, nullptr, 0};
  double(*Cs)[CLD] = dmma_tile8(sm, O, tid);
  const int row = tid & (TM - 1);
  if (row < it.nr) {
    for (int col = tid >> 6; col < it.nb; col += W8_THREADS / TM)
      colc[(i64)col * ld + it.r0 + row] = Cs[col][row];
  }
}

__global__ void k_factor_w1(const int* __restrict__ plist, int count, const DevArgs* __restrict__ args,
                            PanelDev P, i64* __restrict__ fail_col, double* __restrict__ fail_piv) {
  pdl_wait();  // programmatic dependent launch: wait for the previous grid
  pdl_trigger();  // (not persistent: every CTA of the grid has started)
  if (args->pad & 128) return;  // timing ablation (debug)
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
    const double inv = 1.0 / dv;
    for (int r = 1 + lane; r < nr; r += 32) a[r] = a[r] * inv;
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
  for (i64 k = blockIdx.x * (i64)blockDim.x + threadIdx.x; k < n; k += (i64)gridDim.x * blockDim.x) {
    const i64 p = pos[k];
    if (p >= 0) store[p] = vals[k];  // p < 0: an upper entry of A (not stored)
  }
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
