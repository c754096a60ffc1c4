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
#include <climits>
#include <cuda_runtime.h>

namespace ps {

typedef int64_t i64;

constexpr int FORM_LLT = 0;
constexpr int FORM_LDLT = 1;
constexpr int FORM_LU = 2;  // real LU on the DMMA update tiles (factor tasks: ps_generic.cuh)

// One source of a merged chain tile: consecutive split pieces p_1..p_m of one
// supernode (exactly nested rows) update the same destination entries, so
// their updates into ancestors beyond the chain are one tile with K = sum of
// the widths.  Tile rows are p_m-local; piece i's operand rows sit
// shift_i = w_i + ... + w_{m-1} rows lower in its own storage.  Piece i is
// addressed like an ordinary source through a virtual column-0 pointer
//   A_i = store + off_i + shift_i - kbeg_i lds_i   (entry (r, k) at A_i + k lds_i + r)
//   D_i = store + off_i - kbeg_i (lds_i + 1)       (d_k at D_i + k (lds_i + 1))
// and the entries hold the increments from the previous pointer (entry 0:
// from p_m's own column 0), so the operand loader just moves its pointers
// when its chunk reaches the next piece (chain_advance).  Pieces are
// multiples of the k chunk wide.  CHAIN_GM + 1 entries per group; unused
// entries (and always the last) have kbeg = INT_MAX.
constexpr int CHAIN_GM = 8;
constexpr int CHAIN_STRIDE = CHAIN_GM + 1;
struct ChainSeg {
  i64 step;   // A / B pointer increment (elements)
  i64 dstep;  // D pointer increment (elements)
  int lds;    // the piece's leading dimension (nrows)
  int kbeg;   // first k of the piece in the merged tile (INT_MAX: none)
};

struct DevArgs {
  double* store;
  double* scratch;  // inverse diagonal blocks of wide panels (FNB x FNB each)
  double thr;
  int form;
  int pad;
  unsigned long long* tile_trace;  // optional (debug): per tile {start, mainloop done, end} ns
  const struct UTile* tile_base;   // tile index base of tile_trace
  i64 ustride;                     // LU: elements from the L slab to the U slab (0 otherwise)
  const ChainSeg* chain;           // merged chain tiles: CHAIN_STRIDE entries per group
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
  int mode, ws, nparts, rc;  // reserved (0)
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
#define UPD_MIN_CTAS 3  // k_update resident CTAs per SM (168 registers, no spills; with chain tiles 120^3: 494.0 (4 CTAs) -> 488.3 ms)
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

// completion signal of a tile: every thread's scatter stores are ordered
// before the caller's barrier; the signalling thread's acq_rel fence makes
// them visible (cumulatively) before the counter increment (lighter than
// __threadfence's fence.sc: 60^3 19.17 -> 19.10 ms)
__device__ __forceinline__ void signal_add(unsigned* ctr) {
  asm volatile("fence.acq_rel.gpu;\n red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
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
  const int s = __ldg(run_src + k), d = __ldg(run_dst + k);  // (run arrays are padded)
  sm.wsrc[w][tid & 63] = k < end ? s : 0x7fffffff;
  sm.wdst[w][tid & 63] = k < end ? d : 0;
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
  int lda;
  int ai0, ani;
  const double* B;
  int ldb;
  int bj0, bnj;
  int kn;
  const double* dptr;
  int dstride;
  const ChainSeg* seg = nullptr;  // merged chain tile: the next piece's entry
  int knext = INT_MAX;            // first k of that piece (INT_MAX: no more pieces)
};

// merged chain tile T.mode > 0: its group's entries
__device__ __forceinline__ const ChainSeg* chain_of(const DevArgs* args, const UTile& T) {
  return T.mode > 0 ? args->chain + (i64)(T.mode - 1) * CHAIN_STRIDE : nullptr;
}

// merged chain tiles: move A / B / D to the piece holding chunk k (chunks are
// loaded in ascending order, pieces are whole chunks)
template <class T, class LD>
__device__ __forceinline__ void chain_advance(const ChainSeg*& seg, int& knext, int kbase,
                                              const T*& A, const T*& B, const T*& D, LD& lda,
                                              LD& ldb, LD& dstride) {
  if (kbase >= knext) {
    const ChainSeg g = *seg;
    A += g.step;
    B += g.step;
    if (D) D += g.dstep;
    lda = ldb = g.lds;
    dstride = g.lds + 1;
    knext = seg[1].kbeg;
    ++seg;
  }
}

// Shape-adaptive DMMA tile: WM x WN warps, each FM x FN fragments of 8 x 8,
// covering a (8 WM FM) x (8 WN FN) tile; the caller picks the smallest shape
// that holds the tile's ni x nj extents (tile_shape), so partial tiles issue
// no DMMA on padding.  Only the RA = 8 WM FM operand rows of A and RB = 8 WN
// FN rows of B are staged.  k steps past kn in the last chunk are skipped
// (their operands are zero: the sums are unchanged).  Every entry sees the
// same sequence of DMMA k steps in every shape and CTA size, so all shapes
// give bitwise identical results.  The result is staged to Cs[col][row]
// (shared, reusing the operand stages) behind a barrier.
// one operand (R rows x KC columns of a column-major source) into a stage:
// when R divides NT every thread keeps one row and steps its pointer across
// the columns it stages (no per-element index math); otherwise the general
// element split.  Entries past the extent / past kn are zero-filled.
template <int NT, int R>
__device__ __forceinline__ void stage_operand(double (*S)[LDS], const double* src, int ld, int r0,
                                              int rn, int kbase, int kn, int tid) {
  static_assert((KC * R) % NT == 0, "stage split");
  if constexpr (NT % R == 0) {
    constexpr int SK = NT / R;  // columns apart of one thread's elements
    const int r = tid % R, kk0 = tid / R;
    const bool rv = r < rn;
    const double* p = src + (i64)(kbase + kk0) * ld + r0 + r;
    const i64 step = (i64)SK * ld;
#pragma unroll
    for (int e = 0; e < KC / SK; ++e) {
      const bool v = rv && kbase + kk0 + e * SK < kn;
      cp_async8(&S[kk0 + e * SK][r], v ? p : src, v);
      p += step;
    }
  } else {
#pragma unroll
    for (int e = 0; e < (KC * R) / NT; ++e) {
      const int idx = tid + e * NT;
      const int r = idx % R, kk = idx / R;
      const int k = kbase + kk;
      const bool v = k < kn && r < rn;
      cp_async8(&S[kk][r], src + (i64)(v ? k : 0) * ld + (v ? r0 + r : 0), v);
    }
  }
}

template <int NT, int RA, int RB>
__device__ __forceinline__ void load_stage_t(UpdSmem& sm, int st, Operands& O, int chunk, int tid) {
  const int kbase = chunk * KC;
  chain_advance(O.seg, O.knext, kbase, O.A, O.B, O.dptr, O.lda, O.ldb, O.dstride);
  // extents that do not divide the CTA stage as the next power of two (the
  // extra rows are zero-filled, never read)
  constexpr int SA = NT % RA == 0 ? RA : (RA <= 32 ? 32 : 64);
  constexpr int SB = NT % RB == 0 ? RB : (RB <= 32 ? 32 : 64);
  stage_operand<NT, SA>(sm.A[st], O.A, O.lda, O.ai0, O.ani, kbase, O.kn, tid);
  stage_operand<NT, SB>(sm.B[st], O.B, O.ldb, O.bj0, O.bnj, kbase, O.kn, tid);
  if (O.dptr && tid < KC) {
    const int k = kbase + tid;
    const bool kv = k < O.kn;
    cp_async8(&sm.D[st][tid], O.dptr + (i64)(kv ? k : 0) * O.dstride, kv);
  }
}

template <int NT, int WM, int WN, int FM, int FN>
__device__ __forceinline__ double (*dmma_tile_t(UpdSmem& sm, Operands O, int tid))[CLD] {
  static_assert(WM * WN * 32 == NT, "one warp per WM x WN slot");
  constexpr int RA = 8 * WM * FM, RB = 8 * WN * FN;
  static_assert(RA <= TM && RB <= TN, "tile fits the stages");
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp % WM, wn = warp / WM;
  const bool scaled = O.dptr != nullptr;  // LDLt: B scaled by d_k
  double acc[FM][FN][2];
#pragma unroll
  for (int a = 0; a < FM; ++a)
#pragma unroll
    for (int b = 0; b < FN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int nch = (O.kn + KC - 1) / KC;
#pragma unroll
  for (int s = 0; s < NSTAGE - 1; ++s) {
    if (s < nch) load_stage_t<NT, RA, RB>(sm, s, O, s, tid);
    cp_async_commit();
  }
  for (int c = 0; c < nch; ++c) {
    cp_async_wait<NSTAGE - 2>();
    __syncthreads();
    const int nxt = c + NSTAGE - 1;
    if (nxt < nch) load_stage_t<NT, RA, RB>(sm, nxt % NSTAGE, O, nxt, tid);
    cp_async_commit();
    const int st = c % NSTAGE;
    const int krem = O.kn - c * KC;  // k steps left in this chunk (>= 1)
#pragma unroll
    for (int ks = 0; ks < KC / 4; ++ks) {
      if (ks > 0 && 4 * ks >= krem) break;  // all-zero k steps of the last chunk
      const int kr = ks * 4 + (lane & 3);
      double af[FM], bf[FN];
#pragma unroll
      for (int mi = 0; mi < FM; ++mi) af[mi] = sm.A[st][kr][(wm * FM + mi) * 8 + (lane >> 2)];
#pragma unroll
      for (int ni = 0; ni < FN; ++ni) bf[ni] = sm.B[st][kr][(wn * FN + ni) * 8 + (lane >> 2)];
      if (scaled) {
        const double dk = sm.D[st][kr];
#pragma unroll
        for (int ni = 0; ni < FN; ++ni) bf[ni] *= dk;
      }
#pragma unroll
      for (int mi = 0; mi < FM; ++mi)
#pragma unroll
        for (int ni = 0; ni < FN; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();  // operand stages free: the result is staged over them
  double(*Cs)[CLD] = reinterpret_cast<double(*)[CLD]>(&sm.A[0][0][0]);
#pragma unroll
  for (int mi = 0; mi < FM; ++mi) {
    const int row = (wm * FM + mi) * 8 + (lane >> 2);
#pragma unroll
    for (int ni = 0; ni < FN; ++ni) {
      const int col = (wn * FN + ni) * 8 + 2 * (lane & 3);
      Cs[col][row] = acc[mi][ni][0];
      Cs[col + 1][row] = acc[mi][ni][1];
    }
  }
  __syncthreads();
  return Cs;
}

// Shape dispatch: the smallest warp layout holding the tile's ni x nj
// (partial tiles: the last rows / columns of a couple).  Columns are covered
// at 8-column granularity on tall tiles, 16 on short ones; full tiles keep the
// operand-reuse-optimal layouts (32 x 32 per warp on 4 warps, 32 x 16 on 8).
//
// 4-warp CTAs (k_update):
//   ni > 32, nj > 56 : 2 x 2 warps of 32 x 32
//   ni > 32, nj <= 56: 4 x 1 warps of 16 x 8 FN      (FN = ceil(nj / 8))
//   ni <= 32         : 2 x 2 warps of 16 x 8 FN      (FN = ceil(nj / 16))
#ifndef PS_SHAPES
#define PS_SHAPES 2  // A/B of the dispatch: 0 = 64 x 64 only, 1 = 64|32 x 64|32, 2 = as below
#endif
__device__ __forceinline__ double (*dmma_tile4(UpdSmem& sm, const Operands& O, int tid))[CLD] {
  const int nj = O.bnj;
  if (PS_SHAPES == 0) return dmma_tile_t<128, 2, 2, 4, 4>(sm, O, tid);
  if (PS_SHAPES == 1) {
    switch ((O.ani <= 32 ? 2 : 0) | (nj <= 32 ? 1 : 0)) {
      case 0: return dmma_tile_t<128, 2, 2, 4, 4>(sm, O, tid);
      case 1: return dmma_tile_t<128, 4, 1, 2, 4>(sm, O, tid);
      case 2: return dmma_tile_t<128, 1, 4, 4, 2>(sm, O, tid);
      default: return dmma_tile_t<128, 2, 2, 2, 2>(sm, O, tid);
    }
  }
  if (O.ani > 32) {
    switch (nj > 56 ? 0 : (nj + 7) >> 3) {
      case 0: return dmma_tile_t<128, 2, 2, 4, 4>(sm, O, tid);
      case 1: return dmma_tile_t<128, 4, 1, 2, 1>(sm, O, tid);
      case 2: return dmma_tile_t<128, 4, 1, 2, 2>(sm, O, tid);
      case 3: return dmma_tile_t<128, 4, 1, 2, 3>(sm, O, tid);
      case 4: return dmma_tile_t<128, 4, 1, 2, 4>(sm, O, tid);
      case 5: return dmma_tile_t<128, 4, 1, 2, 5>(sm, O, tid);
      case 6: return dmma_tile_t<128, 4, 1, 2, 6>(sm, O, tid);
      default: return dmma_tile_t<128, 4, 1, 2, 7>(sm, O, tid);
    }
  }
  switch ((nj + 15) >> 4) {
    case 1: return dmma_tile_t<128, 2, 2, 2, 1>(sm, O, tid);
    case 2: return dmma_tile_t<128, 2, 2, 2, 2>(sm, O, tid);
    case 3: return dmma_tile_t<128, 2, 2, 2, 3>(sm, O, tid);
    default: return dmma_tile_t<128, 2, 2, 2, 4>(sm, O, tid);
  }
}

// 8-warp CTAs (the wide-panel chain's latency-bound launches):
//   ni > 32, nj > 48 : 2 x 4 warps of 32 x 16
//   ni > 32, nj <= 48: 4 x 2 warps of 16 x 8 FN      (FN = ceil(nj / 16))
//   ni <= 32         : 4 x 2 warps of  8 x 8 FN      (FN = ceil(nj / 16))
constexpr int W8_THREADS = 256;
__device__ __forceinline__ double (*dmma_tile8(UpdSmem& sm, const Operands& O, int tid))[CLD] {
  const int nf = (O.bnj + 15) >> 4;
  if (PS_SHAPES == 0) return dmma_tile_t<256, 2, 4, 4, 2>(sm, O, tid);
  if (PS_SHAPES == 1) {
    switch ((O.ani <= 32 ? 2 : 0) | (O.bnj <= 32 ? 1 : 0)) {
      case 0: return dmma_tile_t<256, 2, 4, 4, 2>(sm, O, tid);
      case 1: return dmma_tile_t<256, 4, 2, 2, 2>(sm, O, tid);
      case 2: return dmma_tile_t<256, 2, 4, 2, 2>(sm, O, tid);
      default: return dmma_tile_t<256, 4, 2, 1, 2>(sm, O, tid);
    }
  }
  if (O.ani > 32) {
    switch (nf > 3 ? 0 : nf) {
      case 0: return dmma_tile_t<256, 2, 4, 4, 2>(sm, O, tid);
      case 1: return dmma_tile_t<256, 4, 2, 2, 1>(sm, O, tid);
      case 2: return dmma_tile_t<256, 4, 2, 2, 2>(sm, O, tid);
      default: return dmma_tile_t<256, 4, 2, 2, 3>(sm, O, tid);
    }
  }
  switch (nf) {
    case 1: return dmma_tile_t<256, 4, 2, 1, 1>(sm, O, tid);
    case 2: return dmma_tile_t<256, 4, 2, 1, 2>(sm, O, tid);
    case 3: return dmma_tile_t<256, 4, 2, 1, 3>(sm, O, tid);
    default: return dmma_tile_t<256, 4, 2, 1, 4>(sm, O, tid);
  }
}

// Epilogue: C(map i, map j) -= Cs[j][i] for the tile's entries on or below
// the destination diagonal (source-local i0 + i >= j0 + j), rows across
// threads - 32 or 64 of them by the tile's height, so short tiles keep every
// thread busy - and 8 independent loads in flight per thread before the
// stores.  MAPPED: rows / columns through the staged index maps (couple
// tiles); otherwise identity (intra-panel trailing tiles).  strict = 1: only
// entries strictly below the diagonal (LU's U^T slab).
#ifndef PS_EPI_BATCH
#define PS_EPI_BATCH 8  // destination loads in flight per thread in the epilogue
#endif
template <int NT, bool MAPPED>
__device__ __forceinline__ void scatter_sub(double (*Cs)[CLD], double* dst, i64 ldd,
                                            const UTile& T, const int* rmap, const int* cmap,
                                            int tid, int strict = 0) {
  constexpr int B = PS_EPI_BATCH;
  const int lr = T.ni <= 32 ? 5 : 6;
  const int row = tid & ((1 << lr) - 1);
  const int cstep = NT >> lr;
  if (row >= T.ni) return;
  const int gi = T.i0 + row;
  const int dr = MAPPED ? rmap[row] : gi;
  for (int cb = tid >> lr; cb < T.nj; cb += B * cstep) {
    double v[B];
    double* pp[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int col = cb + u * cstep;
      const bool ok = col < T.nj && gi >= T.j0 + col + strict;
      pp[u] = ok ? dst + (i64)(MAPPED ? cmap[col] : T.j0 + col) * ldd + dr : nullptr;
      v[u] = ok ? __ldcg(pp[u]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < B; ++u)
      if (pp[u]) __stcg(pp[u], v[u] - Cs[cb + u * cstep][row]);
  }
}

// L2 prefetch of the tile's destination lines (one per 16 mapped rows of each
// column) before the mainloop, so the epilogue's read-modify-write hits L2
// instead of waiting on HBM.  A hint: discontiguous row runs may leave lines
// out; nothing depends on it.
#ifndef PS_PREFETCH_DST
#define PS_PREFETCH_DST 1
#endif
template <int NT>
__device__ __forceinline__ void prefetch_dst(const double* dst, i64 ldd, const UTile& T,
                                             const int* rmap, const int* cmap, int tid) {
  if (!PS_PREFETCH_DST) return;
  for (int e = tid; e < 4 * TN; e += NT) {
    const int col = e & (TN - 1), row = (e >> 6) * 16;
    if (col < T.nj && row < T.ni && T.i0 + row + 15 >= T.j0 + col) {
      const double* a = dst + (i64)cmap[col] * ldd + rmap[row];
      asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
    }
  }
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
  const bool lu = args->form == FORM_LU;
  const i64 us = args->ustride;
  // LU: pass 0 = L rows x U^T rows into L (i >= j), pass 1 = U^T rows x L
  // rows into U^T (i > j) (oracle/panel_oracle_ext.py)
  for (int pass = 0; pass < (lu ? 2 : 1); ++pass) {
    const double* A = colk + (pass ? us : 0);
    const double* B = colk + (lu && !pass ? us : 0);
    Operands O{A, (int)lds, T.i0, T.ni, B, (int)lds, T.j0, T.nj, T.kn, ldlt ? colk + T.k0 : nullptr, (int)lds + 1};
    double(*Cs)[CLD] = dmma_tile8(sm, O, tid);
    scatter_sub<W8_THREADS, false>(Cs, store + T.doff + (pass ? us : 0), T.ldd, T, nullptr, nullptr,
                                   tid, pass);
    if (lu) __syncthreads();  // Cs (over the operand stages) read before pass 1 loads
  }
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
  const bool lu = args->form == FORM_LU;
  const i64 us = args->ustride;

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
    const double* colk = src + (i64)T.k0 * lds;
    maps_load(sm, T.couple, T.ri, T.rj, run_ptr, run_src, run_dst, tid);
    __syncthreads();
    maps_search(sm, T.couple, T.i0, T.ni, T.j0, T.nj, tid);
    if (PS_PREFETCH_DST) {
      __syncthreads();
      prefetch_dst<UPD_THREADS>(store + T.doff, T.ldd, T, sm.rmap, sm.cmap, tid);
    }
    // LU: pass 0 = L rows x U^T rows into L (i >= j), pass 1 = U^T rows x L
    // rows into U^T (i > j) (oracle/panel_oracle_ext.py)
    for (int pass = 0; pass < (lu ? 2 : 1); ++pass) {
      const double* A = colk + (pass ? us : 0);
      const double* B = colk + (lu && !pass ? us : 0);
      const Operands O{A, (int)lds, T.i0, T.ni, B, (int)lds, T.j0, T.nj, T.kn, ldlt ? colk + T.k0 : nullptr,
                       (int)lds + 1, chain_of(args, T), T.mode > 0 ? 0 : INT_MAX};
      double(*Cs)[CLD] = dmma_tile4(sm, O, tid);  // (its barriers also publish the maps)

      if (ttr && tid == 0 && pass == 0) ttr[1] = gtimer();
      // ordered, atomics-free scatter: wait for every lower-color source of
      // this destination
      if (pass == 0 && T.wait >= 0 && tid == 0) {
        while (ld_acquire(&counters[T.dst]) < (unsigned)T.wait) __nanosleep(32);
      }
      __syncthreads();
      scatter_sub<UPD_THREADS, true>(Cs, store + T.doff + (pass ? us : 0), T.ldd, T, sm.rmap,
                                     sm.cmap, tid, pass);
      __syncthreads();
    }
    if (T.signal && tid == 0) {
      signal_add(&counters[T.dst]);
    }
    if (ttr && tid == 0) ttr[2] = gtimer();
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
    {
      if (T.couple >= 0) {
        const i64 end = __ldg(run_ptr + T.couple + 1);
        const int kr = T.ri + lane, kc = T.rj + lane;
        // whole windows, not waiting for `end` (the run arrays are padded)
        const int s0 = __ldg(run_src + kr), d0 = __ldg(run_dst + kr);
        const int s1 = __ldg(run_src + kc), d1 = __ldg(run_dst + kc);
        sm.wsrc[0][lane] = kr < end ? s0 : 0x7fffffff;
        sm.wdst[0][lane] = kr < end ? d0 : 0;
        sm.wsrc[1][lane] = kc < end ? s1 : 0x7fffffff;
        sm.wdst[1][lane] = kc < end ? d1 : 0;
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
    if (T.wait >= 0 && lane == 0 && seen < (unsigned)T.wait) {
      while (ld_acquire(&counters[T.dst]) < (unsigned)T.wait) __nanosleep(32);
    }
    __syncwarp();
    double* dst = store + T.doff;
    const i64 ldd = T.ldd;
    const int tot = T.ni * T.nj;
    constexpr int U = NW_U;
    // entry e = lane + 32 s is (i, j) = (e % ni, e / ni): one division per
    // tile, then stepped by 32 = qd ni + rd
    const int qd = 32 / T.ni, rd = 32 - qd * T.ni;
    int ci = lane % T.ni, cj = lane / T.ni;
    for (int e0 = lane; e0 < tot; e0 += 32 * U) {
      double v[U], old[U];
      double* pp[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = e0 + 32 * u;
        const int i = ci, j = cj;
        ci += rd;
        cj += qd;
        if (ci >= T.ni) {
          ci -= T.ni;
          ++cj;
        }
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
      signal_add(&counters[T.dst]);
    }
    t = __shfl_sync(0xffffffffu, t_next, 0);
  }
  pdl_trigger();
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
  const bool lu = args->form == FORM_LU;
  const i64 us = args->ustride;
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
    if (PS_PREFETCH_DST) {
      __syncthreads();
      prefetch_dst<W8_THREADS>(store + T.doff, T.ldd, T, sm.rmap, sm.cmap, tid);
    }
    for (int pass = 0; pass < (lu ? 2 : 1); ++pass) {  // LU: L, then U^T (as k_update)
      const double* A = colk + (pass ? us : 0);
      const double* B = colk + (lu && !pass ? us : 0);
      const Operands O{A, (int)lds, T.i0, T.ni, B, (int)lds, T.j0, T.nj, T.kn, ldlt ? colk + T.k0 : nullptr,
                       (int)lds + 1, chain_of(args, T), T.mode > 0 ? 0 : INT_MAX};
      double(*Cs)[CLD] = dmma_tile8(sm, O, tid);  // (its barriers also publish the maps)
      if (pass == 0 && T.wait >= 0 && tid == 0) {
        while (ld_acquire(&counters[T.dst]) < (unsigned)T.wait) __nanosleep(32);
      }
      __syncthreads();
      scatter_sub<W8_THREADS, true>(Cs, store + T.doff + (pass ? us : 0), T.ldd, T, sm.rmap,
                                    sm.cmap, tid, pass);
      __syncthreads();
    }
    if (T.signal && tid == 0) {
      signal_add(&counters[T.dst]);
    }
  }
}

// the same TRSM tile on an 8-warp CTA (dmma_tile8: bitwise identical)
__global__ void __launch_bounds__(W8_THREADS, 3)
k_trsm8(const FItem* __restrict__ items, const DevArgs* __restrict__ args, PanelDev P) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  UpdSmem& sm = *reinterpret_cast<UpdSmem*>(smem_raw);
  const int tid = threadIdx.x;
  const FItem it = items[blockIdx.x];
  const bool lu = args->form == FORM_LU;
  const i64 ld = P.nrows[it.p];
  // LU (G from g_factor_diag, two slots per block): pass 0 = L rows x
  // U^-T, pass 1 = U^T rows x L^-1
  for (int pass = 0; pass < (lu ? 2 : 1); ++pass) {
    double* base = args->store + P.off[it.p] + (pass ? args->ustride : 0);
    const double* G = args->scratch + (i64)it.g * (lu ? 2 : 1) * FNB * FNB + pass * FNB * FNB;
    double* colc = base + (i64)it.c0 * ld;
    Operands O{colc, (int)ld, it.r0, it.nr, G, FNB, 0, it.nb, it.nb, nullptr, 0};
    double(*Cs)[CLD] = dmma_tile8(sm, O, tid);
    const int row = tid & (TM - 1);
    if (row < it.nr) {
      for (int col = tid >> 6; col < it.nb; col += W8_THREADS / TM)
        colc[(i64)col * ld + it.r0 + row] = Cs[col][row];
    }
    if (lu) __syncthreads();  // Cs read before pass 1's loads
  }
}

__global__ void k_factor_w1(const int* __restrict__ plist, int count, const DevArgs* __restrict__ args,
                            PanelDev P, i64* __restrict__ fail_col, double* __restrict__ fail_piv) {
  pdl_wait();  // programmatic dependent launch: wait for the previous grid
  pdl_trigger();  // (not persistent: every CTA of the grid has started)
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

// The reference's default pivot threshold 1e-13 max |diag(A)|
// (kernels.py:32-40) from the assembled slab, on the device (ps_factor with
// a NaN threshold): a warp per panel takes the max over its diagonal; |x| of
// a non-negative double orders like its bit pattern, so the global max is an
// integer atomicMax.  Then k_set_threshold writes it into the call's args.
__global__ void __launch_bounds__(256)
k_diag_absmax(const double* __restrict__ store, PanelDev P, i64 np, int complex_,
              unsigned long long* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const i64 wid = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const i64 nw = ((i64)gridDim.x * blockDim.x) >> 5;
  double m = 0.0;
  for (i64 p = wid; p < np; p += nw) {
    const i64 off = P.off[p], ld = P.nrows[p];
    const int w = P.width[p];
    for (int j = lane; j < w; j += 32) {
      const i64 e = off + (i64)j * ld + j;
      const double a = complex_ ? hypot(store[2 * e], store[2 * e + 1]) : fabs(store[e]);
      m = fmax(m, a);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0 && m > 0.0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}
__global__ void k_set_threshold(DevArgs* args, const unsigned long long* __restrict__ mx) {
  args->thr = 1e-13 * __longlong_as_double((long long)*mx);
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
