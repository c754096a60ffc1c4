// B200 numeric factorization engine: plan construction + C ABI (ps_b200.h).
//
// The reference executes one factor task per panel and one update task per
// (source, destination) couple under a CPU task runtime (taskgraph.py:79-110,
// runtime.py:143-304).  Here the DAG is replaced by level batching: panel p
// sits at level = its height in the panel tree (parent = facing panel of its
// first block, symbolic.py:107-123); every couple's destination is a strict
// ancestor, so "factor level L, then scatter level L's updates" is a valid
// topological order.  Per level the plan holds:
//   * width-1 panels          -> k_factor_w1
//   * wider panels, per 64-column block s
//                              -> k_factor_diag (diagonal + inverse)
//                              -> k_trsm (DMMA) and k_update on intra-panel trailing tiles
//   * couples sourced at L     -> k_update on ordered inter-panel tiles
// The whole sequence is captured once into a CUDA graph and replayed.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <functional>
#include <map>
#include <string>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ps_b200.h"
#include "ps_kernels.cuh"
#include "ps_dataflow.cuh"
#include "ps_dataflow_plan.h"
#include "ps_solve.cuh"

using namespace ps;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      return fail(PS_ECUDA, "%s failed at %s:%d: %s", #x, __FILE__, __LINE__,              \
                  cudaGetErrorString(e_));                                                 \
  } while (0)

enum Kind { K_W1 = 0, K_FACTOR = 1, K_TRAIL = 2, K_UPDATE = 3, K_SMALL = 4, K_FDIAG = 5,
            K_TRSM = 6, K_GATHER = 7, K_GATHER2 = 8, K_JOIN = 9, K_FORK = 10, K_XWAIT = 11,
            K_WSTEP = 12, K_NBATCH = 13 };

struct Launch {
  int kind;
  int level;   // panel-tree level (-1: the deferred fan-in batch)
  i64 first;   // offset into the kind's item array
  int count;
  int grid;
  int stream;  // graph branch: 0 = top / main, g + 1 = subtree group g
  double flops = 0.0;  // arithmetic of the launch (tiles: full 2 ni nj kn incl. masked entries)
  double bytes = 0.0;  // algorithmic HBM bytes: operands read once + destination read + write
};

template <class T>
int upload(T** d, const std::vector<T>& h, i64* bytes) {
  *d = nullptr;
  if (h.empty()) return PS_OK;
  CK(cudaMalloc((void**)d, sizeof(T) * h.size()));
  CK(cudaMemcpy(*d, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice));
  *bytes += (i64)(sizeof(T) * h.size());
  return PS_OK;
}

}  // namespace

struct ps_plan {
  int device = 0;
  int sms = 148;
  int upd_ctas_per_sm = 3;
  i64 n = 0, np = 0, nblocks = 0, ncouples = 0, nruns = 0;
  int nlevels = 0;
  i64 store_elems = 0;
  i64 dev_bytes = 0;
  std::vector<i64> off;                 // npanels + 1
  std::vector<i64> h_fc;
  std::vector<int> h_w, h_nrows;
  // couples (host copy, for per-task entry points)
  std::vector<i64> cpl_first;           // per panel: first couple id
  std::vector<int> cpl_q;               // per couple: destination
  std::vector<int> cpl_loc0, cpl_N;     // per couple
  std::vector<i64> run_ptr_h;
  std::vector<int> run_src_h;
  // device
  i64* d_off = nullptr;
  int* d_nrows = nullptr;
  int* d_w = nullptr;
  i64* d_fc = nullptr;
  i64* d_run_ptr = nullptr;
  int* d_run_src = nullptr;
  int* d_run_dst = nullptr;
  UTile* d_tiles = nullptr;             // inter-panel + trailing tiles
  FItem* d_fitems = nullptr;
  int* d_w1 = nullptr;
  NItem* d_nitems = nullptr;
  NSeg* d_nsegs = nullptr;
  i64 n_nitems = 0, n_nsegs = 0;
  // level-schedule narrow gathers (k_gather_level)
  NItem* d_lg_items = nullptr;
  GSeg* d_lg_segs = nullptr;
  unsigned char* d_lg_gmap = nullptr;
  int* d_lg_region_ptr = nullptr;
  unsigned* d_counters = nullptr;
  int* d_workctr = nullptr;
  i64* d_fail_col = nullptr;
  double* d_fail_piv = nullptr;
  Status* d_status = nullptr;
  DevArgs* d_args = nullptr;
  i64 n_update_tiles = 0, n_trail_tiles = 0, n_fitems = 0;
  std::vector<Launch> launches;
  int n_update_launches = 0;
  int max_colors = 0;
  int ngroups = 0;
  int noffload = 0;                     // wide panels factored on their own graph branch
  int fbranch = 0;                      // branch id of the per-level small-panel factors (0: none)
  int dbranch = 0;                      // branch id of the deferred (non-critical) updates
  // batched narrow tiles (k_update_narrow_batch)
  NBatch* d_nbatches = nullptr;
  // fused wide-panel steps (k_wide_step)
  WItem* d_witems = nullptr;
  unsigned* d_stepctr = nullptr;
  i64 nstepctr = 0;
  int top_begin = 0;
  int phase1_begin = 0;
  std::vector<int> seg_bounds;          // distributed top: launch index after each segment
  std::vector<int> seg_level;           //   (factor / update segment per top level)
  int my_group = -1;
  std::vector<int> group;
  cudaGraphExec_t phase_graph[2] = {nullptr, nullptr};
  std::map<i64, cudaGraphExec_t> range_graphs;  // ps_factor_range graphs by (i0, i1)
  std::vector<cudaStream_t> side;
  std::vector<cudaEvent_t> side_ev;
  i64 scratch_slots = 0;
  double* d_scratch = nullptr;
  // graph
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t graph = nullptr;
  // device task runtime (ps_dataflow.cuh): schedule 1 = one persistent launch
  int schedule = 0;                     // 0: level batches (graph), 1: dataflow
  bool df_built = false;
  i64 df_ntasks = 0, df_ndeps = 0;
  int df_nctr = 0, df_grid = 0;
  i64 df_slots = 0;
  double df_est_us = 0.0;
  DTask* d_df_tasks = nullptr;
  int2* d_df_deps = nullptr;
  UTile* d_df_tiles = nullptr;
  FItem* d_df_fitems = nullptr;
  NItem* d_df_nitems = nullptr;
  GSeg* d_df_gsegs = nullptr;
  unsigned char* d_df_gmap = nullptr;
  int* d_df_w1 = nullptr;
  int* d_df_sigs = nullptr;
  i64* d_cpl_first = nullptr;
  int* d_cpl_q = nullptr;
  int* d_cpl_loc0 = nullptr;
  int* d_cpl_N = nullptr;
  unsigned* d_df_ctr = nullptr;
  int* d_df_head = nullptr;       // queue state (4 ints) + its initial value (4 ints)
  int* d_df_qhi = nullptr;
  int* d_df_qlo = nullptr;
  int* d_df_rem = nullptr;
  int* d_df_rem_init = nullptr;
  int* d_df_qinit_hi = nullptr;
  int* d_df_qinit_lo = nullptr;
  int df_ninit_hi = 0, df_ninit_lo = 0;
  i64* d_df_wl_ptr = nullptr;
  unsigned* d_df_wl_thr = nullptr;
  int* d_df_wl_task = nullptr;
  unsigned char* d_df_prio = nullptr;
  int* d_df_prio_val = nullptr;
  std::vector<int> df_type, df_src, df_dst;
  std::vector<UTile> tiles_h;           // host copy of the level schedule's tiles (analysis)
  std::vector<int2> df_deps_h;          // host copies for analysis exports
  std::vector<int> df_w1_h;             // width-1 panels (scaled after the dataflow kernel)
  std::vector<int> df_dep0_h, df_sigs_h, df_sig0_h;
  std::vector<double> df_flops;
  cudaGraphExec_t df_graph = nullptr;
  unsigned long long* d_tile_trace = nullptr;  // debug: per-tile times (ps_set_tile_trace)
  // triangular solve (ps_solve.cuh)
  i64* d_sv_lvl_ptr = nullptr;
  int* d_sv_lvl_panels = nullptr;
  i64* d_sv_fbase = nullptr;
  i64* d_sv_bbase = nullptr;
  i64* d_sv_jptr = nullptr;
  i64* d_sv_jidx = nullptr;
  int4* d_sv_fitems = nullptr;
  int4* d_sv_bitems = nullptr;
  i64* d_sv_rowptr = nullptr;
  int* d_sv_rows = nullptr;
  int* d_sv_vw = nullptr;          // virtual panels (column slices of <= SV_SUB)
  int* d_sv_vnro = nullptr;
  i64* d_sv_vfc = nullptr;
  i64* d_sv_voff = nullptr;
  i64* d_sv_vld = nullptr;
  std::vector<int> sv_vw_h;
  int sv_nvirt = 0;
  int2* d_sv_ritems = nullptr;
  double* d_sv_x = nullptr;          // the solve graph's right-hand side
  cudaGraphExec_t sv_graph = nullptr;
  const double* sv_graph_store = nullptr;
  int sv_graph_key = -1;
  bool pdl = true;  // programmatic dependent launches (PS_PDL=0: off)
  bool narrow_warp = true;
  bool upd8 = true;    // inter-panel update tiles on 8-warp CTAs (PS_UPD8=0; off with split-K / joint)
  bool trail8 = true;  // trailing / TRSM tiles of wide panels on 8-warp CTAs (PS_TRAIL8=0: 4 warps)
  // factor + overlapped download (ps_factor_download): slab chunks of whole
  // panels, each copied once its last writing launch has run
  std::vector<i64> dl_off, dl_len;   // per chunk: slab element offset / count
  std::vector<int> dl_fin;           // per chunk: last launch writing it
  std::vector<std::vector<int>> dl_fins;  // per chunk: the last writing launch of each of its units
  std::vector<int> dl_order;         // chunks by ascending dl_fin
  cudaStream_t dl_stream = nullptr;
  cudaEvent_t dl_done = nullptr;
  std::vector<std::pair<std::pair<const double*, double*>, cudaGraphExec_t>> dl_graphs;  // narrow updates: warp-per-tile kernel on 32 x 32 tiles (PS_NARROW_WARP=0: CTA per 64 x 64 tile)
  std::vector<i64> sv_ri_ptr_h;
  double* d_sv_z = nullptr;        // forward values before the LDLt diagonal scaling
  double* d_sv_fpart = nullptr;    // forward / backward partial products
  double* d_sv_bpart = nullptr;
  i64 sv_nfpart = 0, sv_nbpart = 0;
  std::vector<i64> sv_fi_ptr_h, sv_bi_ptr_h;
  std::vector<int> sv_lvl_panels_h;
  std::vector<i64> sv_lvl_wide_h;  // per level: first wide panel in sv_lvl_panels_h
  std::vector<i64> sv_lvl_narrow_h;  // per level: first non-tiny (w > SV_TINY) panel
  double* d_sv_scratch = nullptr;  // right-hand sides of panels wider than SV_MAXW
  std::vector<i64> sv_lvl_ptr_h;
  // split-K of huge-K update tiles (level schedule)
  double* d_splitk_ws = nullptr;
  unsigned* d_splitk_cnt = nullptr;
  i64 splitk_slots = 0, splitk_red = 0;
  // scratch for the per-task entry points
  UTile* d_task_tiles = nullptr;
  i64 task_tiles_cap = 0;
  FItem* d_task_items = nullptr;
  i64 task_items_cap = 0;
  int* d_task_w1 = nullptr;
  PanelDev pdev() const { return PanelDev{d_off, d_nrows, d_w, d_fc}; }
};

namespace {

// destination-local row of global row r in panel q, or -1 if absent
inline i64 dst_local(const ps_symbol_desc* s, i64 q, i64 r) {
  const i64 fc = s->starts[q], lc = s->starts[q + 1];
  if (r >= fc && r < lc) return r - fc;
  const i64* b = s->rows + s->rowptr[q];
  const i64* e = s->rows + s->rowptr[q + 1];
  const i64* it = std::lower_bound(b, e, r);
  if (it == e || *it != r) return -1;
  return (lc - fc) + (it - b);
}

// tiles of the lower trapezoid {(i, j): i >= j} of rows [r0, r0+M) x cols [r0', ...)
// run index covering source-local row i of couple c (last run_src <= i)
inline int run_hint(const std::vector<i64>& run_ptr, const std::vector<int>& run_src, int c, int i) {
  if (c < 0) return 0;
  auto b = run_src.begin() + run_ptr[c], e = run_src.begin() + run_ptr[c + 1];
  return (int)((std::upper_bound(b, e, i) - run_src.begin()) - 1);
}

// Narrow couples -> destination-tiled gather items.  For each couple, the
// source rows (and facing rows) are split by the 64-row (64-column) chunks of
// the destination they land in; every (row chunk, column chunk) piece with a
// non-empty lower trapezoid is a segment of that destination tile's item.
struct GatherBuilder {
  std::vector<NItem> items;
  std::vector<NSeg> segs;
};

// pieces of source-local range [lo, hi) by destination chunk (via runs)
inline void chunk_pieces(const std::vector<i64>& run_ptr, const std::vector<int>& run_src,
                         const std::vector<int>& run_dst, int c, int lo, int hi, int src_end,
                         std::vector<std::array<int, 4>>& out /* chunk, s0, s1, run */) {
  out.clear();
  i64 k0 = std::upper_bound(run_src.begin() + run_ptr[c], run_src.begin() + run_ptr[c + 1], lo) -
           run_src.begin() - 1;
  for (i64 k = k0; k < run_ptr[c + 1]; ++k) {
    const int rs = run_src[k];
    const int re = (k + 1 < run_ptr[c + 1]) ? run_src[k + 1] : src_end;
    const int a = std::max(lo, rs), b = std::min(hi, re);
    if (a >= b) {
      if (rs >= hi) break;
      continue;
    }
    // destination rows of [a, b): run_dst[k] + (x - rs), split by chunk
    int x = a;
    while (x < b) {
      const int d = run_dst[k] + (x - rs);
      const int ch = d / TM;
      const int xe = std::min(b, x + (ch + 1) * TM - d);
      if (!out.empty() && out.back()[0] == ch && out.back()[2] == x) out.back()[2] = xe;
      else out.push_back({ch, x, xe, (int)k});
      x = xe;
    }
  }
}

const std::vector<i64> kNoPtr;
const std::vector<int> kNoSrc;

// slab offsets / leading dimensions of every tile's source and destination
void fill_tile_addr(std::vector<UTile>& tl, const std::vector<i64>& off, const std::vector<int>& nrows) {
  for (UTile& u : tl) {
    u.soff = off[u.src];
    u.doff = off[u.dst];
    u.lds = nrows[u.src];
    u.ldd = nrows[u.dst];
  }
}

void emit_tiles(std::vector<UTile>& out, int src, int dst, int i_start, int i_end, int j_start,
                int j_end, int k0, int kn, int couple, int wait, int signal,
                const std::vector<i64>& run_ptr = kNoPtr, const std::vector<int>& run_src = kNoSrc,
                int tm = TM, int tn = TN) {
  for (int j = j_start; j < j_end; j += tn) {
    int nj = std::min(tn, j_end - j);
    int rj = run_hint(run_ptr, run_src, couple, j);
    for (int i = i_start; i < i_end; i += tm) {
      int ni = std::min(tm, i_end - i);
      if (i + ni - 1 < j) continue;  // tile entirely above the diagonal
      out.push_back(UTile{src, dst, i, j, ni, nj, k0, kn, couple, wait, signal,
                          run_hint(run_ptr, run_src, couple, i), rj});
    }
  }
}


// small panel (1 < w <= SNB): diagonal item (factor + first FTR rows), then
// TRSM-only row tiles
void small_items_of_panel(std::vector<FItem>& diag, std::vector<FItem>& trsm, int p, int w,
                          int nrows) {
  const int rows = std::max(0, nrows - w);
  diag.push_back(FItem{p, 0, w, w, std::min(FTR, rows), 1, 0, 0});
  for (int t = 1; t * FTR < rows; ++t)
    trsm.push_back(FItem{p, 0, w, w + t * FTR, std::min(FTR, rows - t * FTR), 0, 0, 0});
}

// wide panel (w > SNB), column block `step`: diagonal+inverse item (scratch
// slot g) and the DMMA TRSM row tiles (TM rows each)
void wide_items_of_panel(std::vector<FItem>& diag, std::vector<FItem>& trsm, int p, int w,
                         int nrows, int step, int g) {
  const int c0 = step * FNB;
  const int nb = std::min(FNB, w - c0);
  const int rbeg = c0 + nb;
  diag.push_back(FItem{p, c0, nb, rbeg, 0, 1, g, 0});
  for (int r = rbeg; r < nrows; r += TM)
    trsm.push_back(FItem{p, c0, nb, r, std::min(TM, nrows - r), 0, g, 0});
}

// Intra-panel trailing updates of a wide panel, two steps at a time: after
// an even step s only the look-ahead column block s+1 is updated (K = 64,
// needed by step s+1's diagonal and TRSM); after the odd step s+1 every
// column block >= s+2 receives both steps at once (K = 128: the two column
// blocks are adjacent in the panel's column-major storage) - twice the
// arithmetic intensity of K = 64 trailing tiles, same flops.
void trailing_tiles_of_panel(std::vector<UTile>& out, int p, int w, int nrows, int step) {
  const int c0 = step * FNB;
  const int nb = std::min(FNB, w - c0);
  const int b = c0 + nb;
  if (b >= w) return;
  if ((step & 1) == 0) {
    emit_tiles(out, p, p, b, nrows, b, std::min(w, b + FNB), c0, nb, -1, -1, 0);
  } else {
    emit_tiles(out, p, p, b, nrows, b, w, c0 - FNB, FNB + nb, -1, -1, 0);
  }
}

int grid_for(const ps_plan* P, int kind, int count) {
  if (kind == K_W1) return std::max(1, std::min((count + 3) / 4, P->sms * 16));  // 4 warps/CTA
  if (kind == K_FACTOR || kind == K_FDIAG || kind == K_TRSM || kind == K_GATHER || kind == K_GATHER2)
    return count;
  if (kind == K_SMALL) {  // 4 tiles per CTA (warp tiles), capped at narrow_ctas per SM
    static const int cap = getenv("PS_NARROW_GRID") ? std::max(1, atoi(getenv("PS_NARROW_GRID"))) : 12;
    return std::max(1, std::min((count + SMALL_WARPS - 1) / SMALL_WARPS, P->sms * cap));
  }
  if (kind == K_WSTEP) return std::max(1, std::min(count, P->sms * 3));
  if (kind == K_NBATCH) return std::max(1, std::min(count, P->sms * 6));  // (emit_fused_step sizes its own)
  return std::max(1, std::min(count, P->sms * P->upd_ctas_per_sm));
}

// kernel launch, optionally as a programmatic dependent launch (PDL): the
// grid may start launching while the previous grid on the stream finishes;
// every kernel opens with pdl_enter() (griddepcontrol.wait) before touching
// memory, so the stream order of results is unchanged
template <typename... KArgs, typename... Args>
static cudaError_t klaunch(bool pdl, void (*k)(KArgs...), int grid, int block, size_t smem,
                           cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

int launch_one(ps_plan* P, const Launch& L, int idx, cudaStream_t s, const UTile* tiles,
               const FItem* fitems, const int* w1) {
  switch (L.kind) {
    case K_JOIN:
    case K_FORK:
    case K_XWAIT:
      return PS_OK;  // branch fork / join markers: handled by enqueue_range
    case K_W1:
      CK(klaunch(P->pdl, k_factor_w1, L.grid, 128, 0, s, w1 + L.first, L.count, P->d_args, P->pdev(), P->d_fail_col,
                                         P->d_fail_piv));
      break;
    case K_FACTOR:
      CK(klaunch(P->pdl, k_factor_small, L.grid, FTR, 0, s, fitems + L.first, P->d_args, P->pdev(), P->d_fail_col,
                                            P->d_fail_piv));
      break;
    case K_FDIAG:
      CK(klaunch(P->pdl, k_factor_diag_blk, L.grid, DIAGB_T, 0, s, fitems + L.first, P->d_args, P->pdev(), P->d_fail_col,
                                               P->d_fail_piv));
      break;
    case K_TRSM:
      if (P->trail8) {
        CK(klaunch(P->pdl, k_trsm8, L.grid, W8_THREADS, sizeof(UpdSmem), s, fitems + L.first,
                   (const DevArgs*)P->d_args, P->pdev()));
        break;
      }
      CK(klaunch(P->pdl, k_trsm, L.grid, UPD_THREADS, sizeof(UpdSmem), s, fitems + L.first, P->d_args, P->pdev()));
      break;
    case K_GATHER:
      CK(klaunch(P->pdl, k_gather_narrow, L.grid, UPD_THREADS, 0, s, P->d_nitems + L.first, P->d_nsegs, P->d_args,
                                                      P->pdev(), P->d_run_ptr, P->d_run_src,
                                                      P->d_run_dst));
      break;
    case K_NBATCH:
      CK(klaunch(P->pdl, k_update_narrow_batch, L.grid, UPD_THREADS, sizeof(NarrowBatchSm), s, 
          P->d_nbatches + L.first, L.count, tiles, P->d_workctr + idx, P->d_counters, P->d_args,
          P->pdev(), P->d_run_ptr, P->d_run_src, P->d_run_dst));
      break;
    case K_WSTEP:
      CK(klaunch(P->pdl, k_wide_step, L.grid, DF_THREADS, DF_SMEM, s, P->d_witems + L.first, L.count,
                                                     P->d_workctr + idx, P->d_stepctr, fitems,
                                                     tiles, P->d_args, P->pdev(), P->d_fail_col,
                                                     P->d_fail_piv));
      break;
    case K_GATHER2:
      CK(klaunch(P->pdl, k_gather_level, L.grid, DF_THREADS, LG_SMEM, s, P->d_lg_region_ptr + L.first, P->d_lg_items,
                                                        P->d_lg_segs, P->d_lg_gmap, P->d_args,
                                                        P->pdev()));
      break;
    case K_SMALL:
      if (P->narrow_warp) {
        CK(klaunch(P->pdl, k_update_narrow_w, L.grid, 128, 0, s, tiles + L.first, L.count,
                   P->d_workctr + idx, P->d_counters, P->d_args, P->d_run_ptr, P->d_run_src,
                   P->d_run_dst));
        break;
      }
      CK(klaunch(P->pdl, k_update_small, L.grid, 32 * SMALL_WARPS, 0, s, 
          tiles + L.first, L.count, P->d_workctr + idx, P->d_counters, P->d_args, P->pdev(),
          P->d_run_ptr, P->d_run_src, P->d_run_dst));
      break;
    case K_TRAIL:
      if (P->trail8 && !P->d_tile_trace) {
        CK(klaunch(P->pdl, k_trail8, L.count, W8_THREADS, sizeof(UpdSmem), s, tiles + L.first,
                   (const DevArgs*)P->d_args));
        break;
      }
      CK(klaunch(P->pdl, k_update, L.grid, UPD_THREADS, sizeof(UpdSmem), s, 
          tiles + L.first, L.count, P->d_workctr + idx, P->d_counters, P->d_args, P->pdev(),
          P->d_run_ptr, P->d_run_src, P->d_run_dst));
      break;
    default:
      if (P->upd8 && L.kind == K_UPDATE && L.count < P->sms * 3 && !P->d_tile_trace) {  // small launches
        CK(klaunch(P->pdl, k_update8, L.grid, W8_THREADS, sizeof(UpdSmem), s, tiles + L.first,
                   L.count, P->d_workctr + idx, P->d_counters, (const DevArgs*)P->d_args,
                   P->d_run_ptr, P->d_run_src, P->d_run_dst));
        break;
      }
      CK(klaunch(P->pdl, k_update, L.grid, UPD_THREADS, sizeof(UpdSmem), s, 
          tiles + L.first, L.count, P->d_workctr + idx, P->d_counters, P->d_args, P->pdev(),
          P->d_run_ptr, P->d_run_src, P->d_run_dst));
      break;
  }
  CK(cudaGetLastError());
  return PS_OK;
}

// launches [i0, i1); `reset` zeroes the per-factorization state first
// download capture (ps_factor_download): the chunks final after each launch,
// copied inside the graph on a copy stream forked off the launch's stream
struct DlCapture {
  const std::vector<std::vector<int>>* after;  // per launch: chunks final after it
  cudaStream_t cs;
  cudaEvent_t ev;
  const double* d;
  double* h;
};

int enqueue_range(ps_plan* P, cudaStream_t s, cudaEvent_t* ev, size_t i0, size_t i1, bool reset,
                  bool status = true, const DlCapture* dl = nullptr) {
  if (reset) {
    if (P->np > 0) {
      CK(cudaMemsetAsync(P->d_counters, 0, sizeof(unsigned) * P->np, s));
      CK(cudaMemsetAsync(P->d_fail_col, 0x7f, sizeof(i64) * P->np, s));
    }
    if (!P->launches.empty())
      CK(cudaMemsetAsync(P->d_workctr, 0, sizeof(int) * P->launches.size(), s));
    if (P->splitk_red) CK(cudaMemsetAsync(P->d_splitk_cnt, 0, sizeof(unsigned) * P->splitk_red, s));
    if (P->nstepctr) CK(cudaMemsetAsync(P->d_stepctr, 0, sizeof(unsigned) * P->nstepctr, s));
  }
  // graph branches (only when capturing without per-launch events): fork the
  // subtree groups off `s`, join them before the top phase
  const bool branches = !ev && P->ngroups > 0;
  if (branches) {
    CK(cudaEventRecord(P->side_ev[0], s));
    for (int g = 0; g < P->ngroups; ++g) CK(cudaStreamWaitEvent(P->side[g], P->side_ev[0], 0));
  }
  // offloaded wide panels: branch b forks off `s` at its first launch (its
  // inputs are complete there) and joins at its K_JOIN marker
  const bool offload = !ev && (P->noffload > 0 || P->fbranch > 0);
  std::vector<char> started(P->noffload + 3, 0);
  for (size_t i = i0; i < i1; ++i) {
    const Launch& L = P->launches[i];
    if (offload && L.kind == K_FORK) {  // explicit fork: branch b starts after this point
      const int b = (int)L.first;
      CK(cudaEventRecord(P->side_ev[2 * b - 2], s));
      CK(cudaStreamWaitEvent(P->side[b - 1], P->side_ev[2 * b - 2], 0));
      started[b] = 1;
      continue;
    }
    if (offload && L.kind == K_XWAIT) {  // branch L.count waits for branch L.first's work so far
      const int b = (int)L.first, t = L.count;
      if (started[b]) {
        CK(cudaEventRecord(P->side_ev[2 * b - 1], P->side[b - 1]));
        CK(cudaStreamWaitEvent(P->side[t - 1], P->side_ev[2 * b - 1], 0));
      }
      continue;
    }
    if (offload && L.kind == K_JOIN) {
      const int b = (int)L.first;
      if (started[b]) {
        CK(cudaEventRecord(P->side_ev[2 * b - 1], P->side[b - 1]));
        CK(cudaStreamWaitEvent(s, P->side_ev[2 * b - 1], 0));
        if (L.count) started[b] = 0;  // reusable branch: the next fork restarts it
      }
      continue;
    }
    if (offload && L.stream > 0 && !started[L.stream]) {
      CK(cudaEventRecord(P->side_ev[2 * L.stream - 2], s));
      CK(cudaStreamWaitEvent(P->side[L.stream - 1], P->side_ev[2 * L.stream - 2], 0));
      started[L.stream] = 1;
    }
    if (branches && (int)i == P->top_begin) {
      for (int g = 0; g < P->ngroups; ++g) {
        CK(cudaEventRecord(P->side_ev[g + 1], P->side[g]));
        CK(cudaStreamWaitEvent(s, P->side_ev[g + 1], 0));
      }
    }
    cudaStream_t ls = ((branches || offload) && L.stream > 0) ? P->side[L.stream - 1] : s;
    if (ev) CK(cudaEventRecord(ev[2 * i], s));
    int rc = launch_one(P, L, (int)i, ls, P->d_tiles, P->d_fitems, P->d_w1);
    if (rc) return rc;
    if (ev) CK(cudaEventRecord(ev[2 * i + 1], s));
    if (dl && !(*dl->after)[i].empty()) {
      // this launch is the last writer of some chunks' units: the copy stream
      // waits for it (stream order of `ls`); a chunk is copied after the wait
      // for the last of its writers (they may sit on different streams)
      CK(cudaEventRecord(dl->ev, ls));
      CK(cudaStreamWaitEvent(dl->cs, dl->ev, 0));
      for (int c : (*dl->after)[i])
        if (P->dl_fin[c] == (int)i)
          CK(cudaMemcpyAsync(dl->h + P->dl_off[c], dl->d + P->dl_off[c],
                             sizeof(double) * P->dl_len[c], cudaMemcpyDeviceToHost, dl->cs));
    }
  }
  if (branches && P->top_begin >= (int)i1) {
    for (int g = 0; g < P->ngroups; ++g) {
      CK(cudaEventRecord(P->side_ev[g + 1], P->side[g]));
      CK(cudaStreamWaitEvent(s, P->side_ev[g + 1], 0));
    }
  }
  if (P->np > 0 && status) {
    k_status<<<1, 1024, 0, s>>>(P->d_fail_col, P->d_fail_piv, P->np, P->d_status);
    CK(cudaGetLastError());
  }
  if (dl) {  // join the copies
    CK(cudaEventRecord(dl->ev, dl->cs));
    CK(cudaStreamWaitEvent(s, dl->ev, 0));
  }
  return PS_OK;
}

int enqueue_all(ps_plan* P, cudaStream_t s, cudaEvent_t* ev) {
  return enqueue_range(P, s, ev, 0, P->launches.size(), true);
}

int set_args(ps_plan* P, double* store, int form, double thr, cudaStream_t s) {
  if (form != PS_FORM_LLT && form != PS_FORM_LDLT) return fail(PS_EARG, "bad form %d", form);
  // pad: timing ablations (debug only, results invalid): PS_ABLATE bit 0 skips
  // the diagonal-block factor arithmetic of wide panels
  static const int ablate = getenv("PS_ABLATE") ? atoi(getenv("PS_ABLATE")) : 0;
  DevArgs a{store, P->d_scratch, thr, form, ablate, P->d_tile_trace, P->d_tiles, P->d_splitk_ws,
            P->d_splitk_cnt};
  // pageable memcpy is stream-ordered and completes the source read on return
  CK(cudaMemcpyAsync(P->d_args, &a, sizeof a, cudaMemcpyHostToDevice, s));
  return PS_OK;
}

// the whole factorization as one persistent launch (ps_dataflow.cuh)

int enqueue_dataflow(ps_plan* P, cudaStream_t s, unsigned long long* d_trace,
                     unsigned long long* d_phase = nullptr) {
  if (P->np > 0) {
    CK(cudaMemsetAsync(P->d_fail_col, 0x7f, sizeof(i64) * P->np, s));
    CK(cudaMemsetAsync(P->d_df_ctr, 0, sizeof(unsigned) * std::max(1, P->df_nctr), s));
  }
  if (P->df_ntasks > 0) {
    const size_t nt = (size_t)P->df_ntasks;
    CK(cudaMemcpyAsync(P->d_df_head, P->d_df_head + 4, sizeof(int) * 4, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(P->d_df_rem, P->d_df_rem_init, sizeof(int) * nt, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemsetAsync(P->d_df_qhi, 0xff, sizeof(int) * nt, s));
    CK(cudaMemsetAsync(P->d_df_qlo, 0xff, sizeof(int) * nt, s));
    if (P->df_ninit_hi)
      CK(cudaMemcpyAsync(P->d_df_qhi, P->d_df_qinit_hi, sizeof(int) * P->df_ninit_hi,
                         cudaMemcpyDeviceToDevice, s));
    if (P->df_ninit_lo)
      CK(cudaMemcpyAsync(P->d_df_qlo, P->d_df_qinit_lo, sizeof(int) * P->df_ninit_lo,
                         cudaMemcpyDeviceToDevice, s));
    DfArgs A{P->d_df_tasks, (int)P->df_ntasks, 0, P->d_df_deps, P->d_df_ctr, P->d_df_head,
             P->d_df_qhi, P->d_df_qlo, P->d_df_rem, P->d_df_wl_ptr, P->d_df_wl_thr, P->d_df_wl_task,
             P->d_df_prio, P->d_df_prio_val,
             P->d_df_tiles, P->d_df_fitems, P->d_df_nitems, P->d_df_gsegs, P->d_df_gmap, P->d_df_w1, d_trace,
             d_phase, P->d_df_sigs};
    const int grid = (int)std::min<i64>(P->df_grid, P->df_ntasks);
    k_dataflow<<<grid, DF_THREADS, DF_SMEM, s>>>(A, P->d_args, P->pdev(), P->d_run_ptr,
                                                 P->d_run_src, P->d_run_dst, P->d_fail_col,
                                                 P->d_fail_piv);
    CK(cudaGetLastError());
  }
  // width-1 panels were read raw by the gathers: scale them now
  // (kernels.py:216-221, 232-239; failure = the reference's pivot predicate)
  if (!P->df_w1_h.empty()) {
    const int cnt = (int)P->df_w1_h.size();
    k_factor_w1<<<grid_for(P, K_W1, cnt), 128, 0, s>>>(P->d_df_w1, cnt, P->d_args, P->pdev(),
                                                      P->d_fail_col, P->d_fail_piv);
    CK(cudaGetLastError());
  }
  if (P->np > 0) {
    k_status<<<1, 1024, 0, s>>>(P->d_fail_col, P->d_fail_piv, P->np, P->d_status);
    CK(cudaGetLastError());
  }
  return PS_OK;
}

}  // namespace

extern "C" {

const char* ps_last_error(void) { return g_err.c_str(); }

static int plan_create_impl(const ps_symbol_desc* S, int device, const int32_t* group_in,
                            int ngroups_in, int my_group, ps_plan** out,
                            const int32_t* top_owner = nullptr) {
  if (!S || !out) return fail(PS_EARG, "null argument");
  *out = nullptr;
  if (S->npanels < 0 || S->n < 0) return fail(PS_EARG, "negative sizes");
  if (S->npanels >= (1LL << 31)) return fail(PS_EARG, "too many panels");
  CK(cudaSetDevice(device));
  auto* P = new ps_plan();
  if (const char* e = getenv("PS_NARROW_WARP")) P->narrow_warp = e[0] != '0';
  if (const char* e = getenv("PS_TRAIL8")) P->trail8 = e[0] != '0';
  if (const char* e = getenv("PS_UPD8")) P->upd8 = e[0] != '0';
  P->device = device;
  cudaDeviceGetAttribute(&P->sms, cudaDevAttrMultiProcessorCount, device);
  const i64 np = S->npanels;
  P->n = S->n;
  P->np = np;
  P->nblocks = np ? S->blkptr[np] : 0;
  P->off.assign(np + 1, 0);
  P->h_fc.resize(np);
  P->h_w.resize(np);
  P->h_nrows.resize(np);
  for (i64 p = 0; p < np; ++p) {
    i64 w = S->starts[p + 1] - S->starts[p];
    i64 nr = w + (S->rowptr[p + 1] - S->rowptr[p]);
    if (w <= 0 || nr >= (1LL << 31)) {
      delete P;
      return fail(PS_STRUCTURAL, "panel %lld has invalid shape", (long long)p);
    }
    P->h_fc[p] = S->starts[p];
    P->h_w[p] = (int)w;
    P->h_nrows[p] = (int)nr;
    P->off[p + 1] = P->off[p] + w * nr;
  }
  P->store_elems = P->off[np];

  // panel tree + levels (height); parent = facing panel of the first block
  std::vector<int> level(np, 0);
  for (i64 p = 0; p < np; ++p) {
    if (S->blkptr[p + 1] > S->blkptr[p]) {
      i64 q = S->blk_facing[S->blkptr[p]];
      if (q <= p || q >= np) {
        delete P;
        return fail(PS_STRUCTURAL, "block of panel %lld faces panel %lld", (long long)p, (long long)q);
      }
      level[q] = std::max(level[q], level[p] + 1);
    }
  }
  int nlev = 0;
  for (i64 p = 0; p < np; ++p) nlev = std::max(nlev, level[p] + 1);
  P->nlevels = nlev;

  // couples + block-row index map (runs)
  std::vector<int> c_p, c_q, c_loc0, c_N;
  std::vector<i64> c_g0, c_g1;  // blocks of p facing q
  std::vector<i64> run_ptr{0};
  std::vector<int> run_src, run_dst;
  P->cpl_first.assign(np + 1, 0);
  for (i64 p = 0; p < np; ++p) {
    P->cpl_first[p] = (i64)c_p.size();
    const i64 b0 = S->blkptr[p], b1 = S->blkptr[p + 1];
    i64 b = b0;
    while (b < b1) {
      const i64 q = S->blk_facing[b];
      if (q <= p || q >= np) {
        delete P;
        return fail(PS_STRUCTURAL, "block of panel %lld faces panel %lld", (long long)p, (long long)q);
      }
      i64 g = b;
      i64 N = 0;
      while (g < b1 && S->blk_facing[g] == q) {
        N += S->blk_lr[g] - S->blk_fr[g];
        ++g;
      }
      c_p.push_back((int)p);
      c_q.push_back((int)q);
      c_loc0.push_back((int)S->blk_loc[b]);
      c_N.push_back((int)N);
      c_g0.push_back(b);
      c_g1.push_back(g);
      for (i64 r = b; r < b1; ++r) {
        i64 dl = dst_local(S, q, S->blk_fr[r]);
        i64 dl_last = dst_local(S, q, S->blk_lr[r] - 1);
        if (dl < 0 || dl_last != dl + (S->blk_lr[r] - 1 - S->blk_fr[r])) {
          delete P;
          return fail(PS_STRUCTURAL, "rows of panel %lld missing from panel %lld", (long long)p,
                      (long long)q);
        }
        run_src.push_back((int)S->blk_loc[r]);
        run_dst.push_back((int)dl);
      }
      run_ptr.push_back((i64)run_src.size());
      b = g;
    }
  }
  P->cpl_first[np] = (i64)c_p.size();
  const i64 nc = (i64)c_p.size();
  P->ncouples = nc;
  P->nruns = (i64)run_src.size();
  P->cpl_q = c_q;
  P->cpl_loc0 = c_loc0;
  P->cpl_N = c_N;
  P->run_ptr_h = run_ptr;
  P->run_src_h = run_src;

  for (i64 c = 0; c < nc; ++c) {
    if (level[c_q[c]] <= level[c_p[c]]) {
      delete P;
      return fail(PS_STRUCTURAL, "couple %lld -> %lld violates the level order", (long long)c_p[c],
                  (long long)c_q[c]);
    }
  }
  // ---- stream-parallel proportional mapping (SURVEY §8(e) inside one GPU) ----
  // Cut the panel tree into up to `nstreams` independent subtree groups
  // (LPT-balanced by flops); each group's level sequence runs on its own graph
  // branch.  Couples from a group into the shared top are deferred to one
  // fan-in update batch after the branches join; the top is level-batched.
  std::vector<int> parent(np, -1);
  for (i64 p = 0; p < np; ++p)
    if (S->blkptr[p + 1] > S->blkptr[p]) parent[p] = (int)S->blk_facing[S->blkptr[p]];
  std::vector<double> sub(np, 0.0);  // subtree flops (factor + update tasks)
  for (i64 p = 0; p < np; ++p) {
    const double w = P->h_w[p], m = P->h_nrows[p] - P->h_w[p];
    double f = w * (w + 1) * (2 * w + 1) / 6.0 + m * w * w;
    for (i64 b = S->blkptr[p]; b < S->blkptr[p + 1]; ++b)
      f += 2.0 * (P->h_nrows[p] - S->blk_loc[b]) * (S->blk_lr[b] - S->blk_fr[b]) * w;
    sub[p] += f;
    if (parent[p] >= 0) sub[parent[p]] += sub[p];
  }
  int nstreams = 1;  // PS_STREAMS=k: k concurrent subtree branches
  if (const char* e = getenv("PS_STREAMS")) nstreams = std::max(1, atoi(e));
  std::vector<int> grp(np, -1);  // -1: top
  int ngroups = 0;
  if (group_in) {
    for (i64 p = 0; p < np; ++p) {
      grp[p] = group_in[p] < ngroups_in ? group_in[p] : -1;
      if (grp[p] >= 0 && parent[p] >= 0 && grp[parent[p]] != grp[p] && grp[parent[p]] != -1) {
        delete P;
        return fail(PS_EARG, "group of panel %lld differs from its parent's", (long long)p);
      }
    }
    // a group panel's parent must be in the same group or the top
    for (i64 p = np - 1; p >= 0; --p)
      if (grp[p] == -1 && parent[p] >= 0 && grp[parent[p]] >= 0) {
        delete P;
        return fail(PS_EARG, "top panel %lld below a group panel", (long long)p);
      }
    ngroups = ngroups_in;
    nstreams = 1;
  }
  if (!group_in && nstreams > 1 && np > 0) {
    std::vector<std::vector<int>> kids(np);
    std::vector<int> cand;
    for (i64 p = 0; p < np; ++p) {
      if (parent[p] >= 0) kids[parent[p]].push_back((int)p);
      else cand.push_back((int)p);
    }
    double tot = 0;
    for (int c : cand) tot += sub[c];
    // split the heaviest candidate while it exceeds its share
    for (int it = 0; it < 100000; ++it) {
      int best = -1;
      for (size_t k = 0; k < cand.size(); ++k)
        if (best < 0 || sub[cand[k]] > sub[cand[best]]) best = (int)k;
      if (best < 0) break;
      double csum = 0;
      for (int c : cand) csum += sub[c];
      if ((int)cand.size() >= 2 * nstreams && sub[cand[best]] <= csum / nstreams) break;
      if (csum < 0.3 * tot) break;  // keep at least the bottom 30% of the work in groups
      const int c = cand[best];
      if (kids[c].empty()) break;
      cand.erase(cand.begin() + best);
      for (int k : kids[c]) cand.push_back(k);
    }
    std::sort(cand.begin(), cand.end(), [&](int x, int y) { return sub[x] > sub[y]; });
    std::vector<double> load(nstreams, 0.0);
    std::vector<int> root_grp(np, -1);
    for (int c : cand) {
      int g = (int)(std::min_element(load.begin(), load.end()) - load.begin());
      load[g] += sub[c];
      root_grp[c] = g;
    }
    // propagate group ids down each candidate subtree (children < parent)
    for (i64 p = np - 1; p >= 0; --p) {
      if (root_grp[p] >= 0) grp[p] = root_grp[p];
      else if (parent[p] >= 0 && grp[parent[p]] >= 0 && root_grp[parent[p]] != -2) grp[p] = grp[parent[p]];
    }
    for (int g = 0; g < nstreams; ++g)
      if (load[g] > 0) ngroups = std::max(ngroups, g + 1);
  }
  P->ngroups = my_group >= 0 ? 0 : ngroups;  // distributed plans run one group, unbranched
  P->my_group = my_group;
  P->group.assign(grp.begin(), grp.end());

  std::vector<UTile> tiles;
  std::vector<FItem> fitems;
  std::vector<int> w1;
  std::vector<i64> base(np, 0);        // signaling tiles into q in completed launches
  std::vector<i64> launch_cnt(np, 0);  // signaling tiles into q in the launch being built
  std::vector<std::vector<int>> colocc(np);  // per destination column: last color
  std::vector<int> topcolor(np, 0);          // highest color into q in the launch
  const char* dbg = getenv("PS_SPLIT_RANKS");
  const bool split_colors = dbg && dbg[0] == '1';
  const char* gdbg = getenv("PS_NARROW_GATHER");
  const bool use_gather = gdbg && gdbg[0] == '1';  // default: colored narrow tiles
  GatherBuilder gb;
  int slot_base = 0, slot_max = 0;           // scratch slots of the current group
  // narrow tiles in batches of one color class (PS_NARROW_BATCH=0: one tile per CTA item)
  std::vector<NBatch> nbatches;
  const char* nbenv = getenv("PS_NARROW_BATCH");
  const bool narrow_batch = nbenv && nbenv[0] == '1';  // measured slower (a batch waits for all its tiles' colors): opt-in
  // huge-K update tiles: split-K (PS_SPLITK_MIN=0 disables)
  int splitk_min = 0, splitk_chunk = 512;  // off by default: no gain measured
  if (const char* e = getenv("PS_SPLITK_MIN")) splitk_min = atoi(e);
  if (const char* e = getenv("PS_SPLITK_CHUNK")) splitk_chunk = std::max(64, atoi(e));
  // narrow and wide sources in one update launch per level (PS_JOINT=0: two launches)
  const char* jmode = getenv("PS_JOINT");
  const bool joint_updates = jmode && jmode[0] == '1';  // measured slower: off by default
  if (joint_updates || splitk_min > 0) P->upd8 = false;  // k_update8 serves plain DMMA tiles only
  // narrow sources: colored tiles (default) or per-level region gathers (PS_NARROW=gather)
  const char* cord = getenv("PS_COLOR_ORDER");
  const bool heavy_first_colors = !(cord && std::string(cord) == "id");  // 60^3 -0.5 ms, 80^3 -0.5 ms
  const char* nmode = getenv("PS_NARROW");
  const bool level_gather = !use_gather && nmode && std::string(nmode) == "gather";
  psdf::Input lin{np, &P->h_w, &P->h_nrows, &P->h_fc, &level, &c_p, &c_q, &c_loc0, &c_N,
                  &c_g0, &c_g1, &run_ptr, &run_src, &run_dst, S->blk_fr, S->blk_lr,
                  &P->cpl_first, &P->off, 1, GMAX};
  psdf::LevelGathers lg;

  // factor launches of one level (panels pl), on graph branch `stream`
  // one fused launch (k_wide_step) for step s of the wide panels `ps_`:
  // [diagonals][TRSM tiles][trailing tiles]
  std::vector<WItem> witems;
  const char* fsenv = getenv("PS_FUSE_STEP");
  const bool fuse_steps = fsenv && fsenv[0] == '1';  // measured slower than 3 launches: opt-in
  auto emit_fused_step = [&](const std::vector<int>& ps_, int s, int L, int stream, int g0) {
    if (ps_.empty()) return;
    const i64 w0 = (i64)witems.size();
    std::vector<int> ctr(ps_.size()), ntr(ps_.size(), 0);
    std::vector<std::vector<FItem>> trs(ps_.size());
    for (size_t k = 0; k < ps_.size(); ++k) {
      const int p = ps_[k];
      std::vector<FItem> dg;
      wide_items_of_panel(dg, trs[k], p, P->h_w[p], P->h_nrows[p], s, g0 + (int)k);
      ctr[k] = (int)P->nstepctr;
      P->nstepctr += 2;
      ntr[k] = (int)trs[k].size();
      witems.push_back(WItem{0, (int)fitems.size(), ctr[k], 0});
      fitems.push_back(dg[0]);
    }
    for (size_t k = 0; k < ps_.size(); ++k)
      for (const FItem& f : trs[k]) {
        witems.push_back(WItem{1, (int)fitems.size(), ctr[k], 0});
        fitems.push_back(f);
      }
    for (size_t k = 0; k < ps_.size(); ++k) {
      const int p = ps_[k];
      const i64 t0 = (i64)tiles.size();
      trailing_tiles_of_panel(tiles, p, P->h_w[p], P->h_nrows[p], s);
      P->n_trail_tiles += (i64)tiles.size() - t0;
      for (i64 t = t0; t < (i64)tiles.size(); ++t) witems.push_back(WItem{2, (int)t, ctr[k], ntr[k]});
    }
    const int cnt = (int)((i64)witems.size() - w0);
    // CTAs that would only spin waiting for the diagonal / TRSM items would
    // hold SM slots the concurrent branches need: one CTA per diagonal / TRSM
    // item (they continue with the trailing tiles), at least 1/SM
    int nft = (int)ps_.size();
    for (auto& v : trs) nft += (int)v.size();
    const int grid = std::min(cnt, std::min(P->sms * 3, std::max(nft, P->sms)));
    P->launches.push_back(Launch{K_WSTEP, L, w0, cnt, grid, stream});
  };
  std::function<void(int)> branch_hook;  // emitted on the factor branch after the small factors
  auto emit_factor = [&](const std::vector<int>& pl, int L, int stream) {
    i64 w1_first = (i64)w1.size();
    int maxw = 0;
    bool has_small = false;
    for (int p : pl) {
      if (P->h_w[p] == 1) w1.push_back(p);
      maxw = std::max(maxw, P->h_w[p]);
      has_small |= P->h_w[p] <= SNB;
    }
    // width <= 32 panels and the wide-panel step chain are independent:
    // the small ones run on a concurrent graph branch, joined before the updates
    const int main_stream = stream;
    const bool fork = P->fbranch > 0 && stream == 0 && has_small && maxw > SNB;
    if (fork) {
      P->launches.push_back(Launch{K_FORK, L, P->fbranch, 0, 0, 0});
      stream = P->fbranch;
    }
    if ((i64)w1.size() > w1_first) {
      int cnt = (int)((i64)w1.size() - w1_first);
      P->launches.push_back(Launch{K_W1, L, w1_first, cnt, grid_for(P, K_W1, cnt), stream});
    }
    {
      std::vector<FItem> dg, tr;
      for (int p : pl)
        if (P->h_w[p] > 1 && P->h_w[p] <= SNB) small_items_of_panel(dg, tr, p, P->h_w[p], P->h_nrows[p]);
      for (auto* v : {&dg, &tr}) {
        if (v->empty()) continue;
        const i64 f0 = (i64)fitems.size();
        fitems.insert(fitems.end(), v->begin(), v->end());
        P->launches.push_back(Launch{K_FACTOR, L, f0, (int)v->size(), (int)v->size(), stream});
      }
    }
    if (fork && branch_hook) branch_hook(stream);
    stream = main_stream;
    const int steps = maxw > SNB ? (maxw + FNB - 1) / FNB : 0;
    for (int s = 0; s < steps && fuse_steps; ++s) {
      std::vector<int> ps_;
      for (int p : pl)
        if (P->h_w[p] > SNB && P->h_w[p] > s * FNB) ps_.push_back(p);
      emit_fused_step(ps_, s, L, stream, slot_base);
      slot_max = std::max(slot_max, slot_base + (int)ps_.size());
    }
    for (int s = 0; s < steps && !fuse_steps; ++s) {
      std::vector<FItem> dg, tr;
      int g = slot_base;
      for (int p : pl)
        if (P->h_w[p] > SNB && P->h_w[p] > s * FNB)
          wide_items_of_panel(dg, tr, p, P->h_w[p], P->h_nrows[p], s, g++);
      slot_max = std::max(slot_max, g);
      if (!dg.empty()) {
        const i64 f0 = (i64)fitems.size();
        fitems.insert(fitems.end(), dg.begin(), dg.end());
        P->launches.push_back(Launch{K_FDIAG, L, f0, (int)dg.size(), (int)dg.size(), stream});
      }
      if (!tr.empty()) {
        const i64 f0 = (i64)fitems.size();
        fitems.insert(fitems.end(), tr.begin(), tr.end());
        P->launches.push_back(Launch{K_TRSM, L, f0, (int)tr.size(), (int)tr.size(), stream});
      }
      const i64 t0 = (i64)tiles.size();
      for (int p : pl)
        if (P->h_w[p] > SNB && P->h_w[p] > (s + 1) * FNB)
          trailing_tiles_of_panel(tiles, p, P->h_w[p], P->h_nrows[p], s);
      const int cnt = (int)((i64)tiles.size() - t0);
      P->n_trail_tiles += cnt;
      if (cnt) P->launches.push_back(Launch{K_TRAIL, L, t0, cnt, grid_for(P, K_TRAIL, cnt), stream});
    }
    if (fork) P->launches.push_back(Launch{K_JOIN, L, P->fbranch, 1, 0, 0});
  };

  // update launches for a set of couples (ascending ids): narrow sources
  // (CUDA-core kernel) then wide sources (DMMA kernel).  Inside a launch,
  // couples into the same destination q are colored by destination-column
  // overlap (two couples touch a common entry iff their column sets
  // intersect - both then touch that column's diagonal entry): color(c) =
  // 1 + max color of the couples colored before it (heaviest first) sharing a column.
  // Tiles are emitted color-major and a tile of color k waits for every
  // tile of colors < k into q, so the scatter is atomics-free,
  // deterministic, and only truly overlapping sources serialize.
  auto emit_updates = [&](const std::vector<int>& couples, int L, int stream, int passes = 3) {
    std::vector<int> lc_small, lc_big;
    for (int c : couples) (P->h_w[c_p[c]] <= SMALL_W ? lc_small : lc_big).push_back(c);
    if (joint_updates && !use_gather && !level_gather) {
      // one jointly colored launch: k_update serves narrow tiles on CUDA cores
      lc_big = couples;
      std::sort(lc_big.begin(), lc_big.end());
      lc_small.clear();
    }
    if (!lc_small.empty() && use_gather) {
      // destination-tiled gather for narrow sources (no ordering needed)
      std::map<std::array<int, 3>, std::vector<NSeg>> tilesegs;  // (q, row chunk, col chunk)
      std::vector<std::array<int, 4>> rp, cp;
      for (int c : lc_small) {
        const int p = c_p[c], q = c_q[c];
        const int loc0 = c_loc0[c], N = c_N[c], nr = P->h_nrows[p];
        chunk_pieces(run_ptr, run_src, run_dst, c, loc0, nr, nr, rp);
        chunk_pieces(run_ptr, run_src, run_dst, c, loc0, loc0 + N, nr, cp);
        for (const auto& cc : cp)
          for (const auto& rr : rp) {
            if (rr[2] - 1 < cc[1]) continue;  // no i >= j in the piece
            tilesegs[{q, rr[0], cc[0]}].push_back(NSeg{c, p, rr[1], rr[2], cc[1], cc[2], rr[3], cc[3]});
          }
      }
      const i64 f0 = (i64)gb.items.size();
      for (auto& kv : tilesegs) {
        const int q = kv.first[0], rch = kv.first[1], cch = kv.first[2];
        NItem it{q, rch * TM, std::min(TM, P->h_nrows[q] - rch * TM), cch * TN,
                 std::min(TN, P->h_w[q] - cch * TN), (int)gb.segs.size(), (int)kv.second.size(), 0};
        gb.segs.insert(gb.segs.end(), kv.second.begin(), kv.second.end());
        gb.items.push_back(it);
      }
      const int cnt = (int)((i64)gb.items.size() - f0);
      if (cnt) P->launches.push_back(Launch{K_GATHER, L, f0, cnt, cnt, stream});
    }
    if (!lc_small.empty() && level_gather) {
      const int r0 = (int)lg.region_ptr.size() - 1;
      const int nreg = psdf::build_level_gathers(lin, lc_small, lg);
      if (nreg) P->launches.push_back(Launch{K_GATHER2, L, r0, nreg, nreg, stream});
    }
    for (int pass = (use_gather || level_gather) ? 1 : 0; pass < 2; ++pass) {
      if (!((passes >> pass) & 1)) continue;
      const std::vector<int>& lc = pass == 0 ? lc_small : lc_big;
      const int kind = pass == 0 ? K_SMALL : K_UPDATE;
      if (lc.empty()) continue;
      std::vector<int> color(lc.size());
      std::vector<int> touched;
      int maxcolor = 0;
      // coloring order: heaviest couple first (default), so that huge-K sources
      // take the low colors and start at once instead of waiting at the end of
      // a destination's chain; PS_COLOR_ORDER=id: ascending couple id
      std::vector<size_t> corder(lc.size());
      for (size_t k = 0; k < lc.size(); ++k) corder[k] = k;
      if (heavy_first_colors) {
        auto wgt = [&](size_t k) {
          const int c = lc[k];
          return (double)(P->h_nrows[c_p[c]] - c_loc0[c]) * c_N[c] * P->h_w[c_p[c]];
        };
        std::stable_sort(corder.begin(), corder.end(), [&](size_t a, size_t b) { return wgt(a) > wgt(b); });
      }
      for (size_t kk = 0; kk < lc.size(); ++kk) {
        const size_t k = corder[kk];
        const int c = lc[k], q = c_q[c];
        auto& occ = colocc[q];
        if (occ.empty()) {
          occ.assign(P->h_w[q], -1);
          touched.push_back(q);
        }
        const i64 qfc = P->h_fc[q];
        int col = 0;
        for (i64 b = c_g0[c]; b < c_g1[c]; ++b)
          for (i64 r = S->blk_fr[b]; r < S->blk_lr[b]; ++r) col = std::max(col, occ[r - qfc] + 1);
        for (i64 b = c_g0[c]; b < c_g1[c]; ++b)
          for (i64 r = S->blk_fr[b]; r < S->blk_lr[b]; ++r) occ[r - qfc] = col;
        color[k] = col;
        maxcolor = std::max(maxcolor, col);
      }
      for (int q : touched) std::vector<int>().swap(colocc[q]);
      for (size_t k = 0; k < lc.size(); ++k) {
        const int q = c_q[lc[k]];
        topcolor[q] = std::max(topcolor[q], color[k]);
      }
      std::vector<std::vector<int>> by_color(maxcolor + 1);
      for (size_t k = 0; k < lc.size(); ++k) by_color[color[k]].push_back(lc[k]);
      for (int q : touched) launch_cnt[q] = 0;
      i64 t0 = (i64)tiles.size();
      std::vector<i64> class_start;
      for (int k = 0; k <= maxcolor; ++k) {
        class_start.push_back((i64)tiles.size());
        if (split_colors && k > 0 && (i64)tiles.size() > t0) {
          int cnt = (int)((i64)tiles.size() - t0);
          P->n_update_tiles += cnt;
          P->launches.push_back(Launch{kind, L, t0, cnt, grid_for(P, kind, cnt), stream});
          t0 = (i64)tiles.size();
          for (int q : touched) { base[q] += launch_cnt[q]; launch_cnt[q] = 0; }
        }
        std::vector<int> waits(by_color[k].size());
        for (size_t u = 0; u < by_color[k].size(); ++u) {
          const int q = c_q[by_color[k][u]];
          waits[u] = launch_cnt[q] == 0 ? -1 : (int)(base[q] + launch_cnt[q]);
        }
        const i64 cbeg = (i64)tiles.size();
        for (size_t u = 0; u < by_color[k].size(); ++u) {
          const int c = by_color[k][u];
          const int p = c_p[c], q = c_q[c];
          const int loc0 = c_loc0[c], N = c_N[c];
          const int nr = P->h_nrows[p];
          const i64 before = (i64)tiles.size();
          const int sig = (split_colors || k < topcolor[q]) ? 1 : 0;
          const int tsz = (kind == K_SMALL && P->narrow_warp) ? NW_T : TM;  // warp tiles: 32 x 32
          emit_tiles(tiles, p, q, loc0, nr, loc0, loc0 + N, 0, P->h_w[p], c, waits[u], sig,
                     run_ptr, run_src, tsz, tsz);
          if (sig) launch_cnt[q] += (i64)tiles.size() - before;
        }
        // heaviest tiles of the color class first: they start while lighter
        // ones fill the remaining CTAs (tiles of one class never wait on each other)
        std::stable_sort(tiles.begin() + cbeg, tiles.end(), [](const UTile& a, const UTile& b) {
          return (double)a.ni * a.nj * a.kn > (double)b.ni * b.nj * b.kn;
        });
      }
      if (getenv("PS_PLAN_STATS")) {
        // per-launch structure: tiles, max K, flops, longest color chain
        // (per destination: sum over its colors of the heaviest tile)
        std::map<std::pair<int, int>, double> heavy;  // (q, color) -> max tile flops
        double fl = 0.0;
        int maxk = 0;
        for (int k = 0; k <= maxcolor; ++k)
          for (int c : by_color[k]) {
            const int pp = c_p[c], qq = c_q[c];
            const double m = P->h_nrows[pp] - c_loc0[c], nn = c_N[c], kk = P->h_w[pp];
            maxk = std::max(maxk, P->h_w[pp]);
            fl += 2.0 * m * nn * kk;
            auto& h = heavy[{qq, k}];
            h = std::max(h, 2.0 * std::min(64.0, m) * std::min(64.0, nn) * kk);
          }
        std::map<int, double> chain;
        for (auto& kv : heavy) chain[kv.first.first] += kv.second;
        double worst = 0.0;
        for (auto& kv : chain) worst = std::max(worst, kv.second);
        fprintf(stderr, "[plan] level %d %s launch: couples %zu tiles %lld colors %d maxK %d flops %.3e "
                "chain %.3e flops (%.0f us at 83 GF/s/CTA)\n", L, kind == K_SMALL ? "narrow" : "dmma", lc.size(),
                (long long)((i64)tiles.size() - t0), maxcolor + 1, maxk, fl, worst, worst / 83e3);
      }
      if (kind == K_UPDATE && splitk_min > 0) {
        // split-K: tiles with K >= splitk_min become partials (listed first:
        // they never wait) + a reduction tile in the original position
        std::vector<UTile> parts, rest;
        i64 slot = 0;
        for (i64 t = t0; t < (i64)tiles.size(); ++t) {
          UTile u = tiles[t];
          if (u.kn >= splitk_min) {
            const int S = (u.kn + splitk_chunk - 1) / splitk_chunk;
            const int ch = (u.kn + S - 1) / S;
            const int rc = (int)P->splitk_red++;
            for (int sp = 0; sp < S; ++sp) {
              UTile pt = u;
              pt.k0 = u.k0 + sp * ch;
              pt.kn = std::min(ch, u.kn - sp * ch);
              pt.wait = -1;
              pt.signal = 0;
              pt.mode = 1;
              pt.ws = (int)(slot + sp);
              pt.rc = rc;
              pt.nparts = 0;
              parts.push_back(pt);
            }
            u.mode = 2;
            u.ws = (int)slot;
            u.nparts = S;
            u.rc = rc;
            slot += S;
          }
          rest.push_back(u);
        }
        if (!parts.empty()) {
          tiles.resize(t0);
          tiles.insert(tiles.end(), parts.begin(), parts.end());
          tiles.insert(tiles.end(), rest.begin(), rest.end());
          P->splitk_slots = std::max(P->splitk_slots, slot);
        }
      }
      for (int q : touched) { base[q] += launch_cnt[q]; launch_cnt[q] = 0; topcolor[q] = 0; }
      int cnt = (int)((i64)tiles.size() - t0);
      P->n_update_tiles += cnt;
      if (cnt && kind == K_SMALL && narrow_batch && !split_colors) {
        // batches of consecutive tiles of one color class (no intra-batch waits)
        class_start.push_back((i64)tiles.size());
        const i64 b0 = (i64)nbatches.size();
        for (size_t k = 0; k + 1 < class_start.size(); ++k) {
          i64 t = class_start[k];
          const i64 te = class_start[k + 1];
          while (t < te) {
            NBatch nb{(int)t, 0};
            int ops = 0;
            while (t < te && nb.count < NB_MAX) {
              const UTile& u = tiles[t];
              const int need = u.kn * (u.ni + u.nj + 1);
              if (nb.count && ops + need > NB_OPS) break;
              ops += need;
              ++nb.count;
              ++t;
            }
            nbatches.push_back(nb);
          }
        }
        const int nbc = (int)((i64)nbatches.size() - b0);
        P->launches.push_back(Launch{K_NBATCH, L, b0, nbc, grid_for(P, K_NBATCH, nbc), stream});
      } else if (cnt) {
        P->launches.push_back(Launch{kind, L, t0, cnt, grid_for(P, kind, cnt), stream});
      }
      ++P->n_update_launches;
      P->max_colors = std::max(P->max_colors, maxcolor + 1);
    }
  };

  // ---- wide panels with long factor chains run on their own graph branch
  //      (single-GPU plans): forked when their inputs are complete, their
  //      couples deferred to the level just below their first destination,
  //      joined there - the chain overlaps the levels in between ----
  std::vector<int> off_branch(np, 0), off_ld(np, -1);
  {
    int min_steps = 6;
    if (const char* e = getenv("PS_OFFLOAD_MIN")) min_steps = atoi(e);
    if (!group_in && ngroups == 0 && min_steps > 0) {
      for (i64 p = 0; p < np; ++p) {
        if (P->h_w[p] <= SNB || (P->h_w[p] + FNB - 1) / FNB < min_steps) continue;
        int ld = nlev;
        for (i64 c = P->cpl_first[p]; c < P->cpl_first[p + 1]; ++c) ld = std::min(ld, level[c_q[c]] - 1);
        if (ld < level[p] + 1) continue;
        off_branch[p] = ++P->noffload;
        off_ld[p] = ld;
      }
    }
  }
  slot_max = P->noffload;  // scratch slots 0..noffload-1: one per offloaded panel
  {
    const char* fb = getenv("PS_FACTOR_BRANCH");
    if (!group_in && ngroups == 0 && !(fb && fb[0] == '0')) P->fbranch = P->noffload + 1;
    const char* db = getenv("PS_DEFER");
    if (P->fbranch && !(db && db[0] == '0')) P->dbranch = P->noffload + 2;
  }
  bool defer_pending = false;  // deferred updates of the previous level still on their branch
  const char* dnenv = getenv("PS_DEFER_NARROW");
  const bool defer_narrow = dnenv && dnenv[0] == '1';
  auto emit_offloaded = [&](int p, int L) {
    const int b = off_branch[p], w = P->h_w[p], nr = P->h_nrows[p];
    const int steps = (w + FNB - 1) / FNB;
    if (fuse_steps) {
      for (int st = 0; st < steps; ++st) emit_fused_step({p}, st, L, b, b - 1);
      return;
    }
    for (int st = 0; st < steps; ++st) {
      std::vector<FItem> dg, tr;
      wide_items_of_panel(dg, tr, p, w, nr, st, b - 1);
      i64 f0 = (i64)fitems.size();
      fitems.insert(fitems.end(), dg.begin(), dg.end());
      P->launches.push_back(Launch{K_FDIAG, L, f0, 1, 1, b});
      if (!tr.empty()) {
        f0 = (i64)fitems.size();
        fitems.insert(fitems.end(), tr.begin(), tr.end());
        P->launches.push_back(Launch{K_TRSM, L, f0, (int)tr.size(), (int)tr.size(), b});
      }
      const i64 t0 = (i64)tiles.size();
      trailing_tiles_of_panel(tiles, p, w, nr, st);
      const int cnt = (int)((i64)tiles.size() - t0);
      P->n_trail_tiles += cnt;
      if (cnt) P->launches.push_back(Launch{K_TRAIL, L, t0, cnt, grid_for(P, K_TRAIL, cnt), b});
    }
  };
  std::vector<std::vector<int>> off_couples(nlev + 1), off_joins(nlev + 1);
  for (i64 p = 0; p < np; ++p)
    if (off_branch[p]) {
      off_joins[off_ld[p]].push_back(off_branch[p]);
      for (i64 c = P->cpl_first[p]; c < P->cpl_first[p + 1]; ++c) off_couples[off_ld[p]].push_back((int)c);
    }

  // groups (graph branches 1..ngroups), then the top (branch 0)
  std::vector<int> deferred;  // couples from a group into the top
  for (int g = 0; g <= ngroups; ++g) {
    const int gid = g < ngroups ? g : -1;  // last pass: the top
    if (my_group >= 0 && gid >= 0 && gid != my_group) continue;
    const int stream = (gid < 0 || my_group >= 0) ? 0 : gid + 1;
    if (gid < 0) {
      P->top_begin = (int)P->launches.size();
      std::sort(deferred.begin(), deferred.end());
      if (!deferred.empty()) emit_updates(deferred, -1, 0);
      P->phase1_begin = (int)P->launches.size();
    }
    slot_base = std::max(slot_max, P->noffload);
    std::vector<std::vector<int>> lvl_panels(nlev);
    for (i64 p = 0; p < np; ++p)
      if (grp[p] == gid) lvl_panels[level[p]].push_back((int)p);
    const bool dist_top = gid < 0 && my_group >= 0 && top_owner != nullptr;
    for (int L = 0; L < nlev; ++L) {
      if (dist_top) {
        // distributed top: factor the owned panels of this level, then (after
        // the host broadcasts every level-L panel from its owner) the updates
        // from level L into the owned destinations
        if (lvl_panels[L].empty()) continue;
        std::vector<int> own;
        for (int p : lvl_panels[L])
          if (top_owner[p] == my_group) own.push_back(p);
        if (!own.empty()) emit_factor(own, L, 0);
        P->seg_bounds.push_back((int)P->launches.size());
        P->seg_level.push_back(L);
        std::vector<int> cl;
        for (int p : lvl_panels[L])
          for (i64 c = P->cpl_first[p]; c < P->cpl_first[p + 1]; ++c)
            if (top_owner[c_q[c]] == my_group) cl.push_back((int)c);
        if (!cl.empty()) emit_updates(cl, L, 0);
        P->seg_bounds.push_back((int)P->launches.size());
        P->seg_level.push_back(L);
        continue;
      }
      std::vector<int> pl;
      for (int p : lvl_panels[L]) {
        if (off_branch[p]) emit_offloaded(p, L);
        else pl.push_back(p);
      }
      std::vector<int> cl;
      for (int p : pl)
        for (i64 c = P->cpl_first[p]; c < P->cpl_first[p + 1]; ++c) {
          if (gid >= 0 && grp[c_q[c]] != gid) deferred.push_back((int)c);
          else cl.push_back((int)c);
        }
      // narrow-source updates depend only on the small factors: on the factor
      // branch they overlap the wide-panel chain (offloaded panels' deferred
      // couples are all wide: they stay in the main-stream DMMA launch)
      std::vector<int> cl_narrow, cl_narrow_defer;
      bool narrow_on_branch = false;
      if (P->fbranch > 0 && stream == 0 && !level_gather && !use_gather && !joint_updates) {
        for (int c : cl)
          if (P->h_w[c_p[c]] <= SMALL_W) {
            // into farther ancestors: the deferred branch (PS_DEFER_NARROW=1)
            if (defer_narrow && P->dbranch && level[c_q[c]] > L + 1) cl_narrow_defer.push_back(c);
            else cl_narrow.push_back(c);
          }
        branch_hook = [&](int bstream) {
          if (!cl_narrow.empty()) {
            // the previous level's deferred updates may touch the same destinations
            if (defer_pending) P->launches.push_back(Launch{K_XWAIT, L, P->dbranch, bstream, 0, 0});
            emit_updates(cl_narrow, L, bstream, 1);
          }
          narrow_on_branch = true;
        };
      }
      if (!pl.empty()) emit_factor(pl, L, stream);
      branch_hook = nullptr;
      if (gid < 0 && !off_couples[L].empty()) {
        for (int b : off_joins[L]) P->launches.push_back(Launch{K_JOIN, L, b, 0, 0, 0});
        cl.insert(cl.end(), off_couples[L].begin(), off_couples[L].end());
        std::sort(cl.begin(), cl.end());
      }
      if (defer_pending) {  // before this level's updates touch the same destinations
        P->launches.push_back(Launch{K_JOIN, L, P->dbranch, 1, 0, 0});
        defer_pending = false;
      }
      if (!cl.empty() && P->dbranch && stream == 0) {
        // DMMA updates into the next level's panels (critical) now; the ones
        // into farther ancestors on the deferred branch, overlapping the next
        // level's factorization (joined before its updates)
        std::vector<int> crit, defr;
        for (int c : cl) {
          if (narrow_on_branch && P->h_w[c_p[c]] <= SMALL_W) continue;
          (level[c_q[c]] <= L + 1 ? crit : defr).push_back(c);
        }
        const int passes = narrow_on_branch ? 2 : 3;
        if (!crit.empty()) emit_updates(crit, L, stream, passes);
        if (!narrow_on_branch) cl_narrow_defer.clear();  // then cl (and defr) holds them
        if (!defr.empty() || !cl_narrow_defer.empty()) {
          P->launches.push_back(Launch{K_FORK, L, P->dbranch, 0, 0, 0});
          if (!cl_narrow_defer.empty()) emit_updates(cl_narrow_defer, L, P->dbranch, 1);
          if (!defr.empty()) emit_updates(defr, L, P->dbranch, passes);
          defer_pending = true;
        }
      } else if (!cl.empty()) {
        emit_updates(cl, L, stream, narrow_on_branch ? 2 : 3);
      }
    }
    if (defer_pending) {
      P->launches.push_back(Launch{K_JOIN, nlev, P->dbranch, 1, 0, 0});
      defer_pending = false;
    }
    if (gid < 0)  // offloaded panels whose couples were never needed (roots)
      for (int b : off_joins[nlev]) P->launches.push_back(Launch{K_JOIN, nlev, b, 0, 0, 0});
  }
  P->scratch_slots = slot_max;

  // ---- device task runtime (single-GPU plans) ----
  psdf::Built dfb;
  {
    const char* sch = getenv("PS_SCHED");
    // built only on request (PS_SCHED=dataflow): the level schedule is the default
    const bool want_df = !group_in && sch && std::string(sch) == "dataflow";
    if (want_df) {
      cudaError_t e0 = cudaFuncSetAttribute(k_dataflow, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)DF_SMEM);
      int occ = 0;
      if (e0 == cudaSuccess)
        e0 = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dataflow, DF_THREADS, DF_SMEM);
      if (e0 != cudaSuccess || occ < 1) {
        delete P;
        return fail(PS_ECUDA, "dataflow kernel occupancy: %s", cudaGetErrorString(e0));
      }
      P->df_grid = P->sms * occ;
      int gmax = GMAX;
      if (const char* e = getenv("PS_GATHER_MAX")) gmax = std::max(1, atoi(e));
      psdf::Input in{np, &P->h_w, &P->h_nrows, &P->h_fc, &level, &c_p, &c_q, &c_loc0, &c_N,
                     &c_g0, &c_g1, &run_ptr, &run_src, &run_dst, S->blk_fr, S->blk_lr,
                     &P->cpl_first, &P->off, P->df_grid, gmax};
      auto df_emit = [&](std::vector<UTile>& o, int src, int dst, int i0, int i1, int j0, int j1,
                         int k0, int kn, int couple) {
        emit_tiles(o, src, dst, i0, i1, j0, j1, k0, kn, couple, -1, 0,
                   couple >= 0 ? run_ptr : kNoPtr, couple >= 0 ? run_src : kNoSrc);
      };
      std::string err;
      if (psdf::build(in, dfb, df_emit, &err)) {
        delete P;
        return fail(PS_STRUCTURAL, "%s", err.c_str());
      }
      P->df_built = true;
      P->schedule = (sch && std::string(sch) == "dataflow") ? 1 : 0;
      P->df_ntasks = (i64)dfb.tasks.size();
      P->df_ndeps = (i64)dfb.deps.size();
      P->df_nctr = dfb.nctr;
      P->df_slots = dfb.scratch_slots;
      P->df_est_us = dfb.est_us;
      P->df_ninit_hi = (int)dfb.init_hi.size();
      P->df_ninit_lo = (int)dfb.init_lo.size();
      P->df_type.swap(dfb.task_type);
      P->df_src.swap(dfb.task_src);
      P->df_dst.swap(dfb.task_dst);
      P->df_flops.swap(dfb.task_flops);
      P->df_deps_h = dfb.deps;
      P->df_w1_h = dfb.w1;
      P->df_sigs_h = dfb.sigs;
      P->df_dep0_h.resize(dfb.tasks.size() + 1);
      P->df_sig0_h.resize(dfb.tasks.size() + 1);
      for (size_t t = 0; t < dfb.tasks.size(); ++t) {
        P->df_dep0_h[t] = dfb.tasks[t].dep0;
        P->df_sig0_h[t] = dfb.tasks[t].sig0;
      }
      P->df_dep0_h[dfb.tasks.size()] = (int)dfb.deps.size();
      P->df_sig0_h[dfb.tasks.size()] = (int)dfb.sigs.size();
    }
  }
  P->n_nitems = (i64)gb.items.size();
  P->n_nsegs = (i64)gb.segs.size();
  P->n_fitems = (i64)fitems.size();
  // arithmetic and algorithmic bytes of every launch (roofline per launch)
  for (auto& L : P->launches) {
    double f = 0.0, b = 0.0;
    if (L.kind == K_UPDATE || L.kind == K_TRAIL || L.kind == K_SMALL) {
      for (i64 t = L.first; t < L.first + L.count; ++t) {
        const UTile& u = tiles[t];
        f += 2.0 * u.ni * u.nj * u.kn;
        b += 8.0 * (u.ni + u.nj) * u.kn + 16.0 * u.ni * u.nj;
      }
    } else if (L.kind == K_FACTOR || L.kind == K_FDIAG || L.kind == K_TRSM) {
      for (i64 t = L.first; t < L.first + L.count; ++t) {
        const FItem& it = fitems[t];
        const double nb = it.nb;
        if (it.diag) {
          f += nb * (nb + 1) * (2 * nb + 1) / 6.0;
          b += 16.0 * nb * nb;
        }
        f += 1.0 * it.nr * nb * nb;
        b += 16.0 * it.nr * nb;
      }
    } else if (L.kind == K_NBATCH) {
      for (i64 bi = L.first; bi < L.first + L.count; ++bi)
        for (int t = nbatches[bi].first; t < nbatches[bi].first + nbatches[bi].count; ++t) {
          const UTile& u = tiles[t];
          f += 2.0 * u.ni * u.nj * u.kn;
          b += 8.0 * (u.ni + u.nj) * u.kn + 16.0 * u.ni * u.nj;
        }
    } else if (L.kind == K_WSTEP) {
      for (i64 t = L.first; t < L.first + L.count; ++t) {
        const WItem& wi = witems[t];
        if (wi.kind == 2) {
          const UTile& u = tiles[wi.idx];
          f += 2.0 * u.ni * u.nj * u.kn;
          b += 8.0 * (u.ni + u.nj) * u.kn + 16.0 * u.ni * u.nj;
        } else {
          const FItem& it = fitems[wi.idx];
          const double nb = it.nb;
          if (it.diag) {
            f += nb * (nb + 1) * (2 * nb + 1) / 6.0;
            b += 16.0 * nb * nb;
          }
          f += 1.0 * it.nr * nb * nb;
          b += 16.0 * it.nr * nb;
        }
      }
    } else if (L.kind == K_W1) {
      for (i64 t = L.first; t < L.first + L.count; ++t) {
        const double nr = P->h_nrows[w1[t]];
        f += nr;
        b += 16.0 * nr;
      }
    }
    L.flops = f;
    L.bytes = b;
  }

  // triangular-solve structures (ps_solve.cuh).  The solve runs on virtual
  // panels: a panel wider than SV_SUB is cut into column slices of <= SV_SUB
  // (slice k's facing rows = the panel's columns right of it, then the
  // panel's rows), so that a wide diagonal block's off-diagonal work goes to
  // the parallel GEMV items instead of one CTA.  Virtual tree: slice k ->
  // slice k+1, the last slice -> the parent panel's first slice; levels are
  // heights in it.  Forward partials (v, k-chunk kc, facing row r) at
  // fbase[v] + kc * nro_v + r, grouped per destination global column in
  // ascending partial index (a fixed summation order); backward partials
  // (v, row chunk rc, column j) at bbase[v] + rc * w_v + j.
  {
    int sub = SV_SUB;
    if (const char* e = getenv("PS_SOLVE_SUB")) sub = std::max(32, std::min(SV_SUB, atoi(e)) / 32 * 32);
    std::vector<int> vw, vnro, vpar, vfirst(np + 1, 0);
    std::vector<i64> vfc, voff, vld, vrowptr{0};
    std::vector<int> vrows;
    for (i64 p = 0; p < np; ++p) {
      vfirst[p] = (int)vw.size();
      const int w = P->h_w[p], nr = P->h_nrows[p];
      for (int c0 = 0; c0 < w; c0 += sub) {
        const int wv = std::min(sub, w - c0);
        vw.push_back(wv);
        vnro.push_back(nr - c0 - wv);
        vfc.push_back(P->h_fc[p] + c0);
        voff.push_back(P->off[p] + (i64)c0 * nr + c0);
        vld.push_back(nr);
        for (int c = c0 + wv; c < w; ++c) vrows.push_back((int)(P->h_fc[p] + c));
        for (i64 k = S->rowptr[p]; k < S->rowptr[p + 1]; ++k) vrows.push_back((int)S->rows[k]);
        vrowptr.push_back((i64)vrows.size());
      }
    }
    const int nv = (int)vw.size();
    vfirst[np] = nv;
    vpar.assign(nv, -1);
    for (i64 p = 0; p < np; ++p) {
      for (int v = vfirst[p]; v + 1 < vfirst[p + 1]; ++v) vpar[v] = v + 1;
      if (S->blkptr[p + 1] > S->blkptr[p]) vpar[vfirst[p + 1] - 1] = vfirst[S->blk_facing[S->blkptr[p]]];
    }
    std::vector<int> vlev(nv, 0);
    for (int v = 0; v < nv; ++v)  // ascending virtual id is a topological order
      if (vpar[v] >= 0) vlev[vpar[v]] = std::max(vlev[vpar[v]], vlev[v] + 1);
    int svl = 0;
    for (int v = 0; v < nv; ++v) svl = std::max(svl, vlev[v] + 1);
    std::vector<i64> sv_lvl_ptr(svl + 1, 0), sv_fbase(nv + 1, 0), sv_bbase(nv + 1, 0),
        sv_jptr(S->n + 1, 0), sv_jidx, sv_fi_ptr(svl + 1, 0), sv_bi_ptr(svl + 1, 0);
    std::vector<int> sv_lvl_panels(nv);
    std::vector<int4> sv_fitems, sv_bitems;
    for (int v = 0; v < nv; ++v) sv_lvl_ptr[vlev[v] + 1]++;
    for (int L = 0; L < svl; ++L) sv_lvl_ptr[L + 1] += sv_lvl_ptr[L];
    std::vector<i64> fill(sv_lvl_ptr.begin(), sv_lvl_ptr.end() - 1);
    for (int v = 0; v < nv; ++v)  // narrow panels first within each level
      if (vw[v] <= SV_TINY) sv_lvl_panels[fill[vlev[v]]++] = v;  // tiny: warp per panel
    P->sv_lvl_narrow_h.assign(fill.begin(), fill.end());
    for (int v = 0; v < nv; ++v)
      if (vw[v] > SV_TINY && vw[v] <= SV_WIDE) sv_lvl_panels[fill[vlev[v]]++] = v;
    P->sv_lvl_wide_h.assign(fill.begin(), fill.end());
    for (int v = 0; v < nv; ++v)
      if (vw[v] > SV_WIDE) sv_lvl_panels[fill[vlev[v]]++] = v;
    for (int v = 0; v < nv; ++v) {
      sv_fbase[v + 1] = sv_fbase[v] + (i64)(vw[v] + SV_KC - 1) / SV_KC * vnro[v];
      sv_bbase[v + 1] = sv_bbase[v] + (i64)(vnro[v] + SV_BR - 1) / SV_BR * vw[v];
    }
    for (int L = 0; L < svl; ++L) {
      for (i64 t = sv_lvl_ptr[L]; t < sv_lvl_ptr[L + 1]; ++t) {
        const int v = sv_lvl_panels[t];
        for (int r0 = 0; r0 < vnro[v]; r0 += SV_FR)
          for (int k0 = 0; k0 < vw[v]; k0 += SV_KC) sv_fitems.push_back(make_int4(v, r0, k0, 0));
        for (int r0 = 0; r0 < vnro[v]; r0 += SV_BR)
          for (int c0 = 0; c0 < vw[v]; c0 += SV_BC) sv_bitems.push_back(make_int4(v, r0, c0, 0));
      }
      sv_fi_ptr[L + 1] = (i64)sv_fitems.size();
      sv_bi_ptr[L + 1] = (i64)sv_bitems.size();
    }
    const i64 npart = sv_fbase[nv];
    std::vector<i64> sv_ri_ptr(svl + 1, 0);
    std::vector<int2> sv_ritems;
    for (int v = 0; v < nv; ++v) {
      const i64 nkc = (vw[v] + SV_KC - 1) / SV_KC;
      for (i64 r = 0; r < vnro[v]; ++r) sv_jptr[vrows[vrowptr[v] + r] + 1] += nkc;
    }
    for (int L = 0; L < svl; ++L) {  // 8-column reduction items with incoming partials
      for (i64 t = sv_lvl_ptr[L]; t < sv_lvl_ptr[L + 1]; ++t) {
        const int v = sv_lvl_panels[t];
        for (int j0 = 0; j0 < vw[v]; j0 += 8) {
          bool any = false;
          for (int j = j0; j < std::min(vw[v], j0 + 8); ++j) any |= sv_jptr[vfc[v] + j + 1] > 0;
          if (any) sv_ritems.push_back(make_int2(v, j0));
        }
      }
      sv_ri_ptr[L + 1] = (i64)sv_ritems.size();
    }
    for (i64 j = 0; j < S->n; ++j) sv_jptr[j + 1] += sv_jptr[j];
    sv_jidx.resize(npart);
    std::vector<i64> f2(sv_jptr.begin(), sv_jptr.end() - 1);
    for (int v = 0; v < nv; ++v) {  // ascending partial index
      const i64 nkc = (vw[v] + SV_KC - 1) / SV_KC;
      for (i64 kc = 0; kc < nkc; ++kc)
        for (i64 r = 0; r < vnro[v]; ++r) sv_jidx[f2[vrows[vrowptr[v] + r]]++] = sv_fbase[v] + kc * vnro[v] + r;
    }
    P->sv_nfpart = npart;
    P->sv_nbpart = sv_bbase[nv];
    P->sv_lvl_ptr_h = sv_lvl_ptr;
    P->sv_fi_ptr_h = sv_fi_ptr;
    P->sv_lvl_panels_h = sv_lvl_panels;
    P->sv_bi_ptr_h = sv_bi_ptr;
    P->sv_ri_ptr_h = sv_ri_ptr;
    P->sv_vw_h = vw;
    P->sv_nvirt = nv;
    int rc0;
    if ((rc0 = upload(&P->d_sv_lvl_ptr, sv_lvl_ptr, &P->dev_bytes)) ||
        (rc0 = upload(&P->d_sv_lvl_panels, sv_lvl_panels, &P->dev_bytes)) ||
        (rc0 = upload(&P->d_sv_vw, vw, &P->dev_bytes)) ||
        (rc0 = upload(&P->d_sv_vnro, vnro, &P->dev_bytes)) ||
        (rc0 = upload(&P->d_sv_vfc, vfc, &P->dev_bytes)) ||
        (rc0 = upload(&P->d_sv_voff, voff, &P->dev_bytes)) ||
        (rc0 = upload(&P->d_sv_vld, vld, &P->dev_bytes)) ||
        (rc0 = upload(&P->d_sv_fbase, sv_fbase, &P->dev_bytes)) ||
        (rc0 = upload(&P->d_sv_bbase, sv_bbase, &P->dev_bytes)) ||
        (rc0 = upload(&P->d_sv_jptr, sv_jptr, &P->dev_bytes)) ||
        (rc0 = upload(&P->d_sv_jidx, sv_jidx, &P->dev_bytes)) ||
        (rc0 = upload(&P->d_sv_fitems, sv_fitems, &P->dev_bytes)) ||
        (rc0 = upload(&P->d_sv_bitems, sv_bitems, &P->dev_bytes)) ||
        (rc0 = upload(&P->d_sv_ritems, sv_ritems, &P->dev_bytes)) ||
        (rc0 = upload(&P->d_sv_rowptr, vrowptr, &P->dev_bytes)) ||
        (rc0 = upload(&P->d_sv_rows, vrows, &P->dev_bytes))) {
      ps_plan_destroy(P);
      return rc0;
    }
  }

  // overlapped download: the last launch writing each panel (its factor /
  // trailing launches; updates into a panel all precede its factor) - for a
  // wide panel per 64-column block (column-major: one contiguous range, final
  // after its own diagonal / TRSM step) - then chunks of >= 4 MB of such
  // consecutive units in slab order
  {
    std::vector<int> fin(np, -1);
    std::map<std::pair<int, int>, int> blk_fin;  // (wide panel, c0) -> launch
    bool known = P->schedule == 0;
    for (size_t i = 0; i < P->launches.size() && known; ++i) {
      const Launch& L = P->launches[i];
      switch (L.kind) {
        case K_W1:
          for (int t = 0; t < L.count; ++t) fin[w1[L.first + t]] = (int)i;
          break;
        case K_FACTOR:
          for (int t = 0; t < L.count; ++t) fin[fitems[L.first + t].p] = (int)i;
          break;
        case K_FDIAG:
        case K_TRSM:
          for (int t = 0; t < L.count; ++t) {
            const FItem& it = fitems[L.first + t];
            fin[it.p] = (int)i;
            blk_fin[{it.p, it.c0}] = (int)i;
          }
          break;
        case K_TRAIL:
          for (int t = 0; t < L.count; ++t) fin[tiles[L.first + t].dst] = (int)i;
          break;
        case K_WSTEP:
          known = false;  // fused steps (opt-in): no per-panel write sets here
          break;
        default:
          break;
      }
    }
    const int last = std::max(0, (int)P->launches.size() - 1);
    struct Unit { i64 off, len; int fin; };
    std::vector<Unit> units;
    for (i64 p = 0; p < np; ++p) {
      const i64 nr = P->h_nrows[p], w = P->h_w[p];
      auto it = known ? blk_fin.find({(int)p, 0}) : blk_fin.end();
      if (it != blk_fin.end()) {
        for (i64 c0 = 0; c0 < w; c0 += FNB) {
          auto jt = blk_fin.find({(int)p, (int)c0});
          const int f = jt != blk_fin.end() ? jt->second : fin[p];
          units.push_back({P->off[p] + c0 * nr, std::min<i64>(FNB, w - c0) * nr, f < 0 ? last : f});
        }
      } else {
        const int f = known ? fin[p] : last;
        units.push_back({P->off[p], P->off[p + 1] - P->off[p], f < 0 ? last : f});
      }
    }
    const i64 target = (i64)(4 << 20) / 8;
    size_t u0 = 0;
    while (u0 < units.size()) {
      size_t u1 = u0;
      i64 len = 0;
      int f = -1;
      std::vector<int> fins;
      while (u1 < units.size() && (len < target || u1 == u0)) {
        len += units[u1].len;
        f = std::max(f, units[u1].fin);
        fins.push_back(std::min(units[u1].fin, last));
        ++u1;
      }
      std::sort(fins.begin(), fins.end());
      fins.erase(std::unique(fins.begin(), fins.end()), fins.end());
      P->dl_off.push_back(units[u0].off);
      P->dl_len.push_back(len);
      P->dl_fin.push_back(std::min(f, last));
      P->dl_fins.push_back(fins);  // every last writer: they may run on different streams
      u0 = u1;
    }
    P->dl_order.resize(P->dl_fin.size());
    for (size_t c = 0; c < P->dl_order.size(); ++c) P->dl_order[c] = (int)c;
    std::stable_sort(P->dl_order.begin(), P->dl_order.end(),
                     [&](int a, int b) { return P->dl_fin[a] < P->dl_fin[b]; });
  }

  // upload
  int rc;
  std::vector<i64> off_h(P->off.begin(), P->off.begin() + np);
  if ((rc = upload(&P->d_off, off_h, &P->dev_bytes)) ||
      (rc = upload(&P->d_nrows, P->h_nrows, &P->dev_bytes)) ||
      (rc = upload(&P->d_w, P->h_w, &P->dev_bytes)) ||
      (rc = upload(&P->d_fc, P->h_fc, &P->dev_bytes)) ||
      (rc = upload(&P->d_run_ptr, run_ptr, &P->dev_bytes)) ||
      (rc = upload(&P->d_run_src, run_src, &P->dev_bytes)) ||
      (rc = upload(&P->d_run_dst, run_dst, &P->dev_bytes)) ||
      (fill_tile_addr(tiles, P->off, P->h_nrows), 0) ||
      (rc = upload(&P->d_tiles, tiles, &P->dev_bytes)) ||
      ((P->tiles_h = getenv("PS_KEEP_TILES") ? tiles : std::vector<UTile>()), 0) ||
      (rc = upload(&P->d_fitems, fitems, &P->dev_bytes)) ||
      (rc = upload(&P->d_w1, w1, &P->dev_bytes)) ||
      (rc = upload(&P->d_nitems, gb.items, &P->dev_bytes)) ||
      (rc = upload(&P->d_nsegs, gb.segs, &P->dev_bytes)) ||
      (rc = upload(&P->d_witems, witems, &P->dev_bytes)) ||
      (rc = upload(&P->d_nbatches, nbatches, &P->dev_bytes)) ||
      (rc = upload(&P->d_lg_items, lg.items, &P->dev_bytes)) ||
      (rc = upload(&P->d_lg_segs, lg.segs, &P->dev_bytes)) ||
      (rc = upload(&P->d_lg_gmap, lg.gmap, &P->dev_bytes)) ||
      (rc = upload(&P->d_lg_region_ptr, lg.region_ptr, &P->dev_bytes)) ||
      (rc = upload(&P->d_df_tasks, dfb.tasks, &P->dev_bytes)) ||
      (rc = upload(&P->d_df_deps, dfb.deps, &P->dev_bytes)) ||
      (fill_tile_addr(dfb.tiles, P->off, P->h_nrows), 0) ||
      (rc = upload(&P->d_df_tiles, dfb.tiles, &P->dev_bytes)) ||
      (rc = upload(&P->d_df_fitems, dfb.fitems, &P->dev_bytes)) ||
      (rc = upload(&P->d_df_nitems, dfb.nitems, &P->dev_bytes)) ||
      (rc = upload(&P->d_df_gsegs, dfb.gsegs, &P->dev_bytes)) ||
      (rc = upload(&P->d_df_gmap, dfb.gmap, &P->dev_bytes)) ||
      (rc = upload(&P->d_df_w1, dfb.w1, &P->dev_bytes)) ||
      (rc = upload(&P->d_df_sigs, dfb.sigs, &P->dev_bytes)) ||
      (rc = upload(&P->d_df_rem_init, dfb.rem_init, &P->dev_bytes)) ||
      (rc = upload(&P->d_df_qinit_hi, dfb.init_hi, &P->dev_bytes)) ||
      (rc = upload(&P->d_df_qinit_lo, dfb.init_lo, &P->dev_bytes)) ||
      (rc = upload(&P->d_df_wl_ptr, dfb.wl_ptr, &P->dev_bytes)) ||
      (rc = upload(&P->d_df_wl_thr, dfb.wl_thr, &P->dev_bytes)) ||
      (rc = upload(&P->d_df_wl_task, dfb.wl_task, &P->dev_bytes)) ||
      (rc = upload(&P->d_df_prio, dfb.prio, &P->dev_bytes)) ||
      (rc = upload(&P->d_df_prio_val, dfb.prio_val, &P->dev_bytes)) ||
      (rc = upload(&P->d_cpl_first, P->cpl_first, &P->dev_bytes)) ||
      (rc = upload(&P->d_cpl_q, P->cpl_q, &P->dev_bytes)) ||
      (rc = upload(&P->d_cpl_loc0, P->cpl_loc0, &P->dev_bytes)) ||
      (rc = upload(&P->d_cpl_N, P->cpl_N, &P->dev_bytes))) {
    ps_plan_destroy(P);
    return rc;
  }
  auto alloc = [&](void** ptr, size_t bytes) -> int {
    *ptr = nullptr;
    if (!bytes) return PS_OK;
    CK(cudaMalloc(ptr, bytes));
    P->dev_bytes += (i64)bytes;
    return PS_OK;
  };
  if ((rc = alloc((void**)&P->d_counters, sizeof(unsigned) * np)) ||
      (rc = alloc((void**)&P->d_workctr, sizeof(int) * std::max<size_t>(1, P->launches.size()))) ||
      (rc = alloc((void**)&P->d_fail_col, sizeof(i64) * np)) ||
      (rc = alloc((void**)&P->d_fail_piv, sizeof(double) * np)) ||
      (rc = alloc((void**)&P->d_status, sizeof(Status))) ||
      (rc = alloc((void**)&P->d_args, sizeof(DevArgs))) ||
      (rc = alloc((void**)&P->d_stepctr, sizeof(unsigned) * P->nstepctr)) ||
      (rc = alloc((void**)&P->d_splitk_ws, sizeof(double) * TM * TN * P->splitk_slots)) ||
      (rc = alloc((void**)&P->d_splitk_cnt, sizeof(unsigned) * P->splitk_red)) ||
      (rc = alloc((void**)&P->d_df_ctr, sizeof(unsigned) * std::max(1, P->df_nctr))) ||
      (rc = alloc((void**)&P->d_df_head, sizeof(int) * 8)) ||
      (rc = alloc((void**)&P->d_df_qhi, sizeof(int) * std::max<i64>(1, P->df_ntasks))) ||
      (rc = alloc((void**)&P->d_df_qlo, sizeof(int) * std::max<i64>(1, P->df_ntasks))) ||
      (rc = alloc((void**)&P->d_df_rem, sizeof(int) * std::max<i64>(1, P->df_ntasks))) ||
      (rc = alloc((void**)&P->d_scratch,
                  sizeof(double) * FNB * FNB *
                      std::max<i64>(1, std::max(P->scratch_slots, P->df_slots))))) {
    ps_plan_destroy(P);
    return rc;
  }
  if (P->df_built) {
    const int nt = (int)P->df_ntasks;
    const int qinit[8] = {0, P->df_ninit_hi, nt, 0, 0, P->df_ninit_hi, nt, 0};
    if (cudaMemcpy(P->d_df_head, qinit, sizeof qinit, cudaMemcpyHostToDevice) != cudaSuccess) {
      ps_plan_destroy(P);
      return fail(PS_ECUDA, "queue init upload failed");
    }
  }
  cudaError_t e = cudaFuncSetAttribute(k_update, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sizeof(UpdSmem));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(UpdSmem));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_trail8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(UpdSmem));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_trsm8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(UpdSmem));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_update8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(UpdSmem));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_gather_level, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LG_SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_wide_step, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DF_SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_update_narrow_batch, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(NarrowBatchSm));
  if (e != cudaSuccess) {
    ps_plan_destroy(P);
    return fail(PS_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_update, UPD_THREADS, sizeof(UpdSmem));
  P->upd_ctas_per_sm = std::max(1, occ);
  int defer_ctas = 8;  // deferred-branch update launches: CTAs per SM (60^3: 3 -> 8 = 26.4 -> 25.1 ms; more: flat)
  if (const char* e = getenv("PS_DEFER_CTAS")) defer_ctas = std::max(1, atoi(e));
  if (const char* e = getenv("PS_PDL")) P->pdl = e[0] != '0';
  for (auto& L : P->launches) {
    if (L.kind == K_UPDATE || L.kind == K_TRAIL) L.grid = grid_for(P, L.kind, L.count);
    if (P->dbranch && L.stream == P->dbranch && (L.kind == K_UPDATE || L.kind == K_SMALL))
      L.grid = std::max(1, std::min(L.grid, P->sms * defer_ctas));
  }
  e = cudaStreamCreateWithFlags(&P->cap_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    ps_plan_destroy(P);
    return fail(PS_ECUDA, "stream create: %s", cudaGetErrorString(e));
  }
  const int nbr = P->noffload + (P->fbranch ? 1 : 0) + (P->dbranch ? 1 : 0);
  const int nside = P->ngroups > 0 ? P->ngroups : nbr;
  const int nev = P->ngroups > 0 ? P->ngroups + 1 : 2 * nbr;
  P->side.assign(nside, nullptr);
  P->side_ev.assign(nev, nullptr);
  for (int g = 0; g < nside && e == cudaSuccess; ++g)
    e = cudaStreamCreateWithFlags(&P->side[g], cudaStreamNonBlocking);
  for (int g = 0; g < nev && e == cudaSuccess; ++g)
    e = cudaEventCreateWithFlags(&P->side_ev[g], cudaEventDisableTiming);
  if (e != cudaSuccess) {
    ps_plan_destroy(P);
    return fail(PS_ECUDA, "side stream create: %s", cudaGetErrorString(e));
  }
  *out = P;
  return PS_OK;
}

int ps_plan_create(const ps_symbol_desc* S, int device, ps_plan** out) {
  return plan_create_impl(S, device, nullptr, 0, -1, out);
}

int ps_plan_create_partitioned(const ps_symbol_desc* S, int device, const int32_t* group,
                               int32_t ngroups, int32_t my_group, ps_plan** out) {
  if (!group || ngroups < 0 || my_group >= ngroups) return fail(PS_EARG, "bad partition");
  return plan_create_impl(S, device, group, ngroups, my_group, out);
}

int ps_plan_create_distributed(const ps_symbol_desc* S, int device, const int32_t* group,
                               int32_t ngroups, int32_t my_group, const int32_t* top_owner,
                               ps_plan** out) {
  if (!group || !top_owner || ngroups < 1 || my_group < 0 || my_group >= ngroups)
    return fail(PS_EARG, "bad distributed partition");
  for (i64 p = 0; p < S->npanels; ++p)
    if (group[p] < 0 && (top_owner[p] < 0 || top_owner[p] >= ngroups))
      return fail(PS_EARG, "top panel %lld has no owner", (long long)p);
  return plan_create_impl(S, device, group, ngroups, my_group, out, top_owner);
}

int ps_plan_segments(const ps_plan* P, int32_t* bounds, int32_t* levels, int32_t* nseg) {
  if (!P || !nseg) return fail(PS_EARG, "null argument");
  if (bounds) {  // nseg + 1 values: the phase-1 start, then the end of each segment
    bounds[0] = P->phase1_begin;
    for (size_t k = 0; k < P->seg_bounds.size(); ++k) bounds[k + 1] = P->seg_bounds[k];
  }
  if (levels)
    for (size_t k = 0; k < P->seg_level.size(); ++k) levels[k] = P->seg_level[k];
  *nseg = (int32_t)P->seg_bounds.size();
  return PS_OK;
}

int ps_factor_range(ps_plan* P, double* d_store, int form, double thr, void* stream, int32_t i0,
                    int32_t i1) {
  if (!P || (!d_store && P->store_elems)) return fail(PS_EARG, "null argument");
  if (i0 < 0 || i1 < i0 || i1 > (int32_t)P->launches.size()) return fail(PS_EARG, "bad range");
  CK(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream;
  int rc = set_args(P, d_store, form, thr, s);
  if (rc) return rc;
  if (i1 == i0) return PS_OK;
  const i64 key = ((i64)i0 << 32) | (i64)i1;
  cudaGraphExec_t& G = P->range_graphs[key];
  if (!G) {
    CK(cudaStreamBeginCapture(P->cap_stream, cudaStreamCaptureModeThreadLocal));
    rc = enqueue_range(P, P->cap_stream, nullptr, (size_t)i0, (size_t)i1, false, false);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(P->cap_stream, &g);
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (e != cudaSuccess) return fail(PS_ECUDA, "graph capture: %s", cudaGetErrorString(e));
    e = cudaGraphInstantiate(&G, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
      G = nullptr;
      return fail(PS_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
    }
  }
  CK(cudaGraphLaunch(G, s));
  return PS_OK;
}

int ps_factor_status_all(ps_plan* P, void* stream) {
  // status reduction only (after ranges)
  if (!P) return fail(PS_EARG, "null argument");
  CK(cudaSetDevice(P->device));
  if (P->np > 0) {
    k_status<<<1, 1024, 0, (cudaStream_t)stream>>>(P->d_fail_col, P->d_fail_piv, P->np, P->d_status);
    CK(cudaGetLastError());
  }
  return PS_OK;
}

int ps_plan_groups(const ps_plan* P, int32_t* group) {
  if (!P || !group) return fail(PS_EARG, "null argument");
  for (i64 p = 0; p < P->np; ++p) group[p] = P->group.empty() ? -1 : P->group[p];
  return PS_OK;
}

void ps_plan_destroy(ps_plan* P) {
  if (!P) return;
  cudaSetDevice(P->device);
  if (P->graph) cudaGraphExecDestroy(P->graph);
  if (P->df_graph) cudaGraphExecDestroy(P->df_graph);
  for (auto g : P->phase_graph)
    if (g) cudaGraphExecDestroy(g);
  for (auto& kv : P->range_graphs)
    if (kv.second) cudaGraphExecDestroy(kv.second);
  if (P->cap_stream) cudaStreamDestroy(P->cap_stream);
  for (auto st : P->side)
    if (st) cudaStreamDestroy(st);
  for (auto ev : P->side_ev)
    if (ev) cudaEventDestroy(ev);
  void* ptrs[] = {P->d_off, P->d_nrows, P->d_w, P->d_fc, P->d_run_ptr, P->d_run_src,
                  P->d_run_dst, P->d_tiles, P->d_fitems, P->d_w1, P->d_counters,
                  P->d_workctr, P->d_fail_col, P->d_fail_piv, P->d_status, P->d_args, P->d_scratch,
                  P->d_task_tiles, P->d_task_items, P->d_task_w1, P->d_nitems, P->d_nsegs,
                  P->d_df_tasks, P->d_df_deps, P->d_df_tiles, P->d_df_fitems, P->d_df_nitems,
                  P->d_df_gsegs, P->d_df_gmap, P->d_df_w1, P->d_df_ctr, P->d_df_head, P->d_df_sigs,
                  P->d_cpl_first, P->d_cpl_q, P->d_cpl_loc0, P->d_cpl_N, P->d_df_qhi,
                  P->d_df_qlo, P->d_df_rem, P->d_df_rem_init, P->d_df_qinit_hi, P->d_df_qinit_lo,
                  P->d_df_wl_ptr, P->d_df_wl_thr, P->d_df_wl_task, P->d_df_prio,
                  P->d_df_prio_val, P->d_lg_items, P->d_lg_segs, P->d_lg_gmap,
                  P->d_lg_region_ptr, P->d_splitk_ws, P->d_splitk_cnt, P->d_sv_lvl_ptr,
                  P->d_sv_lvl_panels, P->d_sv_fbase, P->d_sv_bbase, P->d_sv_fitems,
                  P->d_sv_bitems, P->d_sv_rowptr, P->d_sv_rows, P->d_sv_z, P->d_sv_scratch,
                  P->d_witems, P->d_stepctr, P->d_nbatches, P->d_sv_jptr, P->d_sv_jidx,
                  P->d_sv_fpart, P->d_sv_bpart, P->d_sv_vw, P->d_sv_vnro, P->d_sv_vfc,
                  P->d_sv_voff, P->d_sv_vld, P->d_sv_ritems, P->d_sv_x};
  if (P->sv_graph) cudaGraphExecDestroy(P->sv_graph);
  for (auto& kv : P->dl_graphs) cudaGraphExecDestroy(kv.second);
  if (P->dl_done) cudaEventDestroy(P->dl_done);
  if (P->dl_stream) cudaStreamDestroy(P->dl_stream);
  for (void* q : ptrs)
    if (q) cudaFree(q);
  delete P;
}

int ps_plan_get_info(const ps_plan* P, ps_plan_info* info) {
  if (!P || !info) return fail(PS_EARG, "null argument");
  info->store_elems = P->store_elems;
  info->npanels = P->np;
  info->ncouples = P->ncouples;
  info->nruns = P->nruns;
  info->update_tiles = P->n_update_tiles;
  info->trailing_tiles = P->n_trail_tiles;
  info->factor_items = P->n_fitems;
  info->nlevels = P->nlevels;
  info->nlaunches = P->schedule == 1 ? 1 : (int32_t)P->launches.size();
  info->device_bytes = P->dev_bytes;
  return PS_OK;
}

int ps_plan_offsets(const ps_plan* P, int64_t* offsets) {
  if (!P || !offsets) return fail(PS_EARG, "null argument");
  std::memcpy(offsets, P->off.data(), sizeof(i64) * P->off.size());
  return PS_OK;
}

int ps_assemble(ps_plan* P, double* d_store, const int64_t* d_pos, const double* d_vals,
                int64_t nvals, void* stream) {
  if (!P || (!d_store && P->store_elems)) return fail(PS_EARG, "null argument");
  CK(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream;
  if (P->store_elems) CK(cudaMemsetAsync(d_store, 0, sizeof(double) * P->store_elems, s));
  if (nvals > 0) {
    int grid = (int)std::min<i64>((nvals + 255) / 256, (i64)P->sms * 32);
    k_assemble<<<grid, 256, 0, s>>>(d_store, d_pos, d_vals, nvals);
    CK(cudaGetLastError());
  }
  return PS_OK;
}

int ps_factor_phase(ps_plan* P, double* d_store, int form, double thr, void* stream, int phase) {
  if (!P || (!d_store && P->store_elems)) return fail(PS_EARG, "null argument");
  if (phase < -1 || phase > 1) return fail(PS_EARG, "bad phase %d", phase);
  CK(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream;
  int rc = set_args(P, d_store, form, thr, s);
  if (rc) return rc;
  if (phase < 0 && P->schedule == 1) {
    if (!P->df_graph) {
      CK(cudaStreamBeginCapture(P->cap_stream, cudaStreamCaptureModeThreadLocal));
      rc = enqueue_dataflow(P, P->cap_stream, nullptr);
      cudaGraph_t g = nullptr;
      cudaError_t e = cudaStreamEndCapture(P->cap_stream, &g);
      if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
      }
      if (e != cudaSuccess) return fail(PS_ECUDA, "graph capture: %s", cudaGetErrorString(e));
      e = cudaGraphInstantiate(&P->df_graph, g, 0);
      cudaGraphDestroy(g);
      if (e != cudaSuccess) {
        P->df_graph = nullptr;
        return fail(PS_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
      }
    }
    CK(cudaGraphLaunch(P->df_graph, s));
    return PS_OK;
  }
  cudaGraphExec_t& G = phase < 0 ? P->graph : P->phase_graph[phase];
  if (!G) {
    const size_t n = P->launches.size(), mid = (size_t)P->phase1_begin;
    const size_t i0 = phase == 1 ? mid : 0, i1 = phase == 0 ? mid : n;
    CK(cudaStreamBeginCapture(P->cap_stream, cudaStreamCaptureModeThreadLocal));
    rc = enqueue_range(P, P->cap_stream, nullptr, i0, i1, phase != 1);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(P->cap_stream, &g);
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (e != cudaSuccess) return fail(PS_ECUDA, "graph capture: %s", cudaGetErrorString(e));
    e = cudaGraphInstantiate(&G, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
      G = nullptr;
      return fail(PS_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
    }
  }
  CK(cudaGraphLaunch(G, s));
  return PS_OK;
}

int ps_factor(ps_plan* P, double* d_store, int form, double thr, void* stream) {
  return ps_factor_phase(P, d_store, form, thr, stream, -1);
}

// factorization + download of the factor slab into pinned host memory,
// overlapped: a second graph of the same launches carries the copies as
// memcpy nodes on a copy stream; a chunk's copy waits (captured events) for
// the last writing launch of each of its units - whichever streams those run
// on - and the copies are joined back before the graph ends.
int ps_factor_download(ps_plan* P, double* d_store, int form, double thr, void* stream,
                       double* h_dst) {
  if (!P || (!d_store && P->store_elems) || (!h_dst && P->store_elems))
    return fail(PS_EARG, "null argument");
  CK(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream;
  const size_t nc = P->dl_fin.size();
  if (P->schedule == 1 || nc == 0 || P->launches.empty()) {  // no per-launch structure: copy after
    int rc = ps_factor(P, d_store, form, thr, stream);
    if (rc) return rc;
    if (P->store_elems)
      CK(cudaMemcpyAsync(h_dst, d_store, sizeof(double) * P->store_elems, cudaMemcpyDeviceToHost, s));
    return PS_OK;
  }
  int rc = set_args(P, d_store, form, thr, s);
  if (rc) return rc;
  if (!P->dl_stream) {
    CK(cudaStreamCreateWithFlags(&P->dl_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&P->dl_done, cudaEventDisableTiming));
  }
  // the copies are graph nodes with the slab / host pointers baked in: one
  // cached graph per (device slab, host slab) pair (pools alternate a few)
  auto key = std::make_pair((const double*)d_store, h_dst);
  cudaGraphExec_t G = nullptr;
  for (auto& kv : P->dl_graphs)
    if (kv.first == key) G = kv.second;
  if (!G) {
    std::vector<std::vector<int>> after(P->launches.size());
    for (int c : P->dl_order)
      for (int f : P->dl_fins[c]) after[f].push_back(c);
    DlCapture dl{&after, P->dl_stream, P->dl_done, d_store, h_dst};
    CK(cudaStreamBeginCapture(P->cap_stream, cudaStreamCaptureModeThreadLocal));
    rc = enqueue_range(P, P->cap_stream, nullptr, 0, P->launches.size(), true, true, &dl);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(P->cap_stream, &g);
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (e != cudaSuccess) return fail(PS_ECUDA, "graph capture: %s", cudaGetErrorString(e));
    e = cudaGraphInstantiate(&G, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(PS_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
    if (P->dl_graphs.size() >= 4) {
      cudaGraphExecDestroy(P->dl_graphs.front().second);
      P->dl_graphs.erase(P->dl_graphs.begin());
    }
    P->dl_graphs.push_back({key, G});
  }
  CK(cudaGraphLaunch(G, s));
  return PS_OK;
}

int ps_factor_timed(ps_plan* P, double* d_store, int form, double thr, void* stream,
                    double* ms_by_kind, int32_t* nlaunch, float* per_launch_ms) {
  if (!P || (!d_store && P->store_elems)) return fail(PS_EARG, "null argument");
  CK(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream;
  int rc = set_args(P, d_store, form, thr, s);
  if (rc) return rc;
  if (P->schedule == 1) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, s));
    rc = enqueue_dataflow(P, s, nullptr);
    CK(cudaEventRecord(e1, s));
    CK(cudaStreamSynchronize(s));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    ms_by_kind[0] = ms_by_kind[1] = 0.0;
    ms_by_kind[2] = ms;
    if (nlaunch) *nlaunch = 1;
    if (per_launch_ms) per_launch_ms[0] = ms;
    return rc;
  }
  const size_t nl = P->launches.size();
  std::vector<cudaEvent_t> ev(2 * nl);
  for (auto& e : ev) CK(cudaEventCreate(&e));
  rc = enqueue_all(P, s, ev.data());
  if (!rc) {
    CK(cudaStreamSynchronize(s));
    for (int k = 0; k < 3; ++k) ms_by_kind[k] = 0.0;
    for (size_t i = 0; i < nl; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[2 * i], ev[2 * i + 1]);
      int k = P->launches[i].kind;
      ms_by_kind[(k == K_W1 || k == K_FACTOR || k == K_FDIAG || k == K_TRSM) ? 0 : (k == K_TRAIL ? 1 : 2)] += ms;
      if (per_launch_ms) per_launch_ms[i] = ms;
    }
    if (nlaunch) *nlaunch = (int32_t)nl;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return rc;
}

int ps_plan_launches(const ps_plan* P, int32_t* kind, int32_t* level, int32_t* count,
                     int32_t* branch) {
  if (!P) return fail(PS_EARG, "null argument");
  for (size_t i = 0; i < P->launches.size(); ++i) {
    if (kind) kind[i] = P->launches[i].kind;
    if (level) level[i] = P->launches[i].level;
    if (count) count[i] = P->launches[i].count;
    if (branch) branch[i] = P->launches[i].stream;
  }
  return PS_OK;
}

int ps_factor_status(ps_plan* P, void* stream, int64_t* fail_col, double* fail_piv) {
  if (!P) return fail(PS_EARG, "null argument");
  CK(cudaSetDevice(P->device));
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  Status st{NO_FAIL, 0.0};
  if (P->np > 0) CK(cudaMemcpy(&st, P->d_status, sizeof st, cudaMemcpyDeviceToHost));
  if (st.fail_col != NO_FAIL) {
    if (fail_col) *fail_col = st.fail_col;
    if (fail_piv) *fail_piv = st.fail_piv;
    return PS_NUMERIC;
  }
  return PS_OK;
}

static int ensure(void** ptr, i64* cap, i64 need, size_t elem) {
  if (need <= *cap) return PS_OK;
  if (*ptr) cudaFree(*ptr);
  *ptr = nullptr;
  *cap = 0;
  CK(cudaMalloc(ptr, elem * need));
  *cap = need;
  return PS_OK;
}

int ps_run_factor_task(ps_plan* P, double* d_store, int64_t p, int form, double thr, void* stream) {
  if (!P || p < 0 || p >= P->np) return fail(PS_EARG, "bad panel");
  CK(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream;
  int rc = set_args(P, d_store, form, thr, s);
  if (rc) return rc;
  CK(cudaMemsetAsync(P->d_fail_col, 0x7f, sizeof(i64) * P->np, s));
  const int w = P->h_w[p], nr = P->h_nrows[p];
  std::vector<Launch> seq;            // (kind, items) sequence for this panel
  std::vector<std::vector<FItem>> itemsets;
  std::vector<std::vector<UTile>> tilesets;
  if (w == 1) {
    if (!P->d_task_w1) CK(cudaMalloc((void**)&P->d_task_w1, sizeof(int)));
    int pi = (int)p;
    CK(cudaMemcpyAsync(P->d_task_w1, &pi, sizeof(int), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    k_factor_w1<<<1, 32, 0, s>>>(P->d_task_w1, 1, P->d_args, P->pdev(), P->d_fail_col, P->d_fail_piv);
    CK(cudaGetLastError());
  } else if (w <= SNB) {
    std::vector<FItem> dg, tr;
    small_items_of_panel(dg, tr, (int)p, w, nr);
    seq.push_back(Launch{K_FACTOR, 0, 0, (int)dg.size(), (int)dg.size(), 0});
    itemsets.push_back(dg);
    if (!tr.empty()) {
      seq.push_back(Launch{K_FACTOR, 0, 0, (int)tr.size(), (int)tr.size(), 0});
      itemsets.push_back(tr);
    }
  } else {
    const int steps = (w + FNB - 1) / FNB;
    for (int st = 0; st < steps; ++st) {
      std::vector<FItem> dg, tr;
      wide_items_of_panel(dg, tr, (int)p, w, nr, st, 0);
      seq.push_back(Launch{K_FDIAG, 0, 0, 1, 1, 0});
      itemsets.push_back(dg);
      if (!tr.empty()) {
        seq.push_back(Launch{K_TRSM, 0, 0, (int)tr.size(), (int)tr.size(), 0});
        itemsets.push_back(tr);
      }
      std::vector<UTile> tl;
      trailing_tiles_of_panel(tl, (int)p, w, nr, st);
      if (!tl.empty()) {
        seq.push_back(Launch{K_TRAIL, 0, 0, (int)tl.size(), grid_for(P, K_TRAIL, (int)tl.size()), 0});
        tilesets.push_back(tl);
      }
    }
  }
  size_t fi = 0, ti = 0;
  for (const Launch& L : seq) {
    if (L.kind == K_TRAIL) {
      auto& tl = tilesets[ti++];
      if ((rc = ensure((void**)&P->d_task_tiles, &P->task_tiles_cap, (i64)tl.size(), sizeof(UTile))))
        return rc;
      fill_tile_addr(tl, P->off, P->h_nrows);
      CK(cudaMemcpyAsync(P->d_task_tiles, tl.data(), sizeof(UTile) * tl.size(),
                         cudaMemcpyHostToDevice, s));
      CK(cudaMemsetAsync(P->d_workctr, 0, sizeof(int), s));
      CK(cudaStreamSynchronize(s));
      if ((rc = launch_one(P, L, 0, s, P->d_task_tiles, nullptr, nullptr))) return rc;
    } else {
      const auto& items = itemsets[fi++];
      if ((rc = ensure((void**)&P->d_task_items, &P->task_items_cap, (i64)items.size(), sizeof(FItem))))
        return rc;
      CK(cudaMemcpyAsync(P->d_task_items, items.data(), sizeof(FItem) * items.size(),
                         cudaMemcpyHostToDevice, s));
      CK(cudaStreamSynchronize(s));
      if ((rc = launch_one(P, L, 0, s, nullptr, P->d_task_items, nullptr))) return rc;
    }
    CK(cudaStreamSynchronize(s));
  }
  k_status<<<1, 1024, 0, s>>>(P->d_fail_col, P->d_fail_piv, P->np, P->d_status);
  CK(cudaGetLastError());
  return PS_OK;
}

int ps_run_update_task(ps_plan* P, double* d_store, int64_t p, int64_t q, int form, void* stream) {
  if (!P || p < 0 || p >= P->np || q < 0 || q >= P->np) return fail(PS_EARG, "bad panel");
  CK(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream;
  int rc = set_args(P, d_store, form, 0.0, s);
  if (rc) return rc;
  i64 c = -1;
  for (i64 k = P->cpl_first[p]; k < P->cpl_first[p + 1]; ++k)
    if (P->cpl_q[k] == q) c = k;
  if (c < 0) return fail(PS_STRUCTURAL, "no blocks of panel %lld face panel %lld", (long long)p, (long long)q);
  std::vector<UTile> tl;
  const int loc0 = P->cpl_loc0[c], N = P->cpl_N[c];
  const int tsz = (P->h_w[p] <= SMALL_W && P->narrow_warp) ? NW_T : TM;
  emit_tiles(tl, (int)p, (int)q, loc0, P->h_nrows[p], loc0, loc0 + N, 0, P->h_w[p], (int)c, -1, 0,
             P->run_ptr_h, P->run_src_h, tsz, tsz);
  if (tl.empty()) return PS_OK;
  if ((rc = ensure((void**)&P->d_task_tiles, &P->task_tiles_cap, (i64)tl.size(), sizeof(UTile))))
    return rc;
  fill_tile_addr(tl, P->off, P->h_nrows);
  CK(cudaMemcpyAsync(P->d_task_tiles, tl.data(), sizeof(UTile) * tl.size(), cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(P->d_workctr, 0, sizeof(int), s));
  CK(cudaStreamSynchronize(s));
  const int kind = P->h_w[p] <= SMALL_W ? K_SMALL : K_UPDATE;
  Launch L{kind, 0, 0, (int)tl.size(), grid_for(P, kind, (int)tl.size()), 0};
  int rc2 = launch_one(P, L, 0, s, P->d_task_tiles, nullptr, nullptr);
  if (rc2) return rc2;
  return PS_OK;
}

int ps_solve(ps_plan* P, const double* d_store, double* d_x, int form, void* stream) {
  if (!P || (!d_store && P->store_elems) || (!d_x && P->n)) return fail(PS_EARG, "null argument");
  if (form != PS_FORM_LLT && form != PS_FORM_LDLT) return fail(PS_EARG, "bad form %d", form);
  CK(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream;
  if (!P->d_sv_z && P->n) {
    CK(cudaMalloc((void**)&P->d_sv_z, sizeof(double) * P->n));
    CK(cudaMalloc((void**)&P->d_sv_scratch, sizeof(double) * P->n));
    CK(cudaMalloc((void**)&P->d_sv_fpart, sizeof(double) * std::max<i64>(1, P->sv_nfpart)));
    CK(cudaMalloc((void**)&P->d_sv_bpart, sizeof(double) * std::max<i64>(1, P->sv_nbpart)));
  }
  SolveDev S{P->d_sv_lvl_ptr, P->d_sv_lvl_panels, P->d_sv_vw, P->d_sv_vnro, P->d_sv_vfc,
             P->d_sv_voff, P->d_sv_vld, P->d_sv_fbase, P->d_sv_jptr, P->d_sv_jidx,
             P->d_sv_bbase, P->d_sv_fitems, P->d_sv_bitems, P->d_sv_ritems, P->d_sv_rowptr,
             P->d_sv_rows};
  const int nlev = (int)P->sv_lvl_ptr_h.size() - 1;
  const int ldlt = form == PS_FORM_LDLT;
  int maxw = SV_MAXW;  // widest right-hand side kept in shared memory (PS_SOLVE_SMEM_W: tests)
  if (const char* e = getenv("PS_SOLVE_SMEM_W")) maxw = std::min(SV_MAXW, std::max(0, atoi(e)));
  const bool prof = getenv("PS_SOLVE_PROFILE") != nullptr;  // debug: per-level times to stderr
  const float prof_min = prof ? (float)atof(getenv("PS_SOLVE_PROFILE")) : 0.f;  // ms
  std::vector<cudaEvent_t> ev;
  auto mark = [&]() {
    if (!prof) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    ev.push_back(e);
  };
  static bool attr_set = false;  // per process: dynamic shared memory beyond 48 KB
  if (!attr_set) {
    CK(cudaFuncSetAttribute(k_sv_fdiag<SV_WIDE_T>, cudaFuncAttributeMaxDynamicSharedMemorySize, SV_MAXW * 8));
    CK(cudaFuncSetAttribute(k_sv_bdiag<SV_WIDE_T>, cudaFuncAttributeMaxDynamicSharedMemorySize, SV_MAXW * 8));
    attr_set = true;
  }
  // per level: narrow panels [lvl_ptr[L], lvl_wide[L]) on 128-thread CTAs,
  // wide ones [lvl_wide[L], lvl_ptr[L+1]) on 1024-thread CTAs; the dynamic
  // shared memory holds the launch's widest fitting right-hand side
  auto smem_for = [&](i64 t0, i64 t1) {
    int mw = 0;
    for (i64 t = t0; t < t1; ++t) {
      const int w = P->sv_vw_h[P->sv_lvl_panels_h[t]];
      if (w <= maxw) mw = std::max(mw, w);
    }
    return (size_t)mw * 8;
  };
  auto diag = [&](int L, bool fwd, cudaStream_t s, double* d_x) -> int {
    const i64 tt = P->sv_lvl_ptr_h[L], t0 = P->sv_lvl_narrow_h[L], tw = P->sv_lvl_wide_h[L],
              t1 = P->sv_lvl_ptr_h[L + 1];
    if (t0 > tt && maxw >= SV_TINY) {  // tiny panels: a warp each, four per CTA
      const int nb = (int)((t0 - tt + 3) / 4);
      if (fwd)
        CK(klaunch(P->pdl, k_sv_fdiag_w, nb, 128, 0, s, tt, (int)(t0 - tt), S, d_store, d_x,
                   P->d_sv_z, ldlt));
      else
        CK(klaunch(P->pdl, k_sv_bdiag_w, nb, 128, 0, s, tt, (int)(t0 - tt), S, d_store, d_x,
                   P->d_sv_bpart, ldlt));
    } else if (t0 > tt) {  // (PS_SOLVE_SMEM_W tests: the CTA kernels' scratch path)
      if (fwd)
        CK(klaunch(P->pdl, k_sv_fdiag<SV_NARROW_T>, (int)(t0 - tt), SV_NARROW_T, smem_for(tt, t0), s,
                   tt, S, d_store, d_x, P->d_sv_z, P->d_sv_scratch, P->d_sv_fpart, ldlt, maxw));
      else
        CK(klaunch(P->pdl, k_sv_bdiag<SV_NARROW_T>, (int)(t0 - tt), SV_NARROW_T, smem_for(tt, t0), s,
                   tt, S, d_store, d_x, P->d_sv_scratch, P->d_sv_bpart, ldlt, maxw));
    }
    if (tw > t0) {
      if (fwd)
        CK(klaunch(P->pdl, k_sv_fdiag<SV_NARROW_T>, (int)(tw - t0), SV_NARROW_T, smem_for(t0, tw), s,
                   t0, S, d_store, d_x, P->d_sv_z, P->d_sv_scratch, P->d_sv_fpart, ldlt, maxw));
      else
        CK(klaunch(P->pdl, k_sv_bdiag<SV_NARROW_T>, (int)(tw - t0), SV_NARROW_T, smem_for(t0, tw), s,
                   t0, S, d_store, d_x, P->d_sv_scratch, P->d_sv_bpart, ldlt, maxw));
    }
    if (t1 > tw) {
      if (fwd)
        CK(klaunch(P->pdl, k_sv_fdiag<SV_WIDE_T>, (int)(t1 - tw), SV_WIDE_T, smem_for(tw, t1), s,
                   tw, S, d_store, d_x, P->d_sv_z, P->d_sv_scratch, P->d_sv_fpart, ldlt, maxw));
      else
        CK(klaunch(P->pdl, k_sv_bdiag<SV_WIDE_T>, (int)(t1 - tw), SV_WIDE_T, smem_for(tw, t1), s,
                   tw, S, d_store, d_x, P->d_sv_scratch, P->d_sv_bpart, ldlt, maxw));
    }
    return PS_OK;
  };
  auto enqueue = [&](cudaStream_t s, double* d_x) -> int {
  mark();
  for (int L = 0; L < nlev; ++L) {
    const i64 f0 = P->sv_fi_ptr_h[L], fn = P->sv_fi_ptr_h[L + 1] - f0;
    const i64 r0 = P->sv_ri_ptr_h[L], rn = P->sv_ri_ptr_h[L + 1] - r0;
    if (rn) CK(klaunch(P->pdl, k_sv_freduce, (int)(unsigned)rn, SV_THREADS, 0, s, r0, S, d_x, P->d_sv_fpart));
    if (int rc = diag(L, true, s, d_x)) return rc;
    if (fn) CK(klaunch(P->pdl, k_sv_fgemv, (int)(unsigned)fn, SV_THREADS, 0, s, f0, S, d_store, P->d_sv_z, P->d_sv_fpart));
    mark();
  }
  for (int L = nlev - 1; L >= 0; --L) {
    const i64 b0 = P->sv_bi_ptr_h[L], bn = P->sv_bi_ptr_h[L + 1] - b0;
    if (bn) CK(klaunch(P->pdl, k_sv_bgemv, (int)(unsigned)bn, SV_THREADS, 0, s, b0, S, d_store, d_x, P->d_sv_bpart));
    if (int rc = diag(L, false, s, d_x)) return rc;
    mark();
  }
  return PS_OK;
  };
  // the whole solve (~7 launches per level) is one CUDA graph on the plan's
  // own right-hand-side buffer, cached per (factor store, form)
  const char* ge = getenv("PS_SOLVE_GRAPH");
  if (prof || (ge && ge[0] == '0')) {
    if (int rc = enqueue(s, d_x)) return rc;
  } else {
    if (!P->d_sv_x && P->n) CK(cudaMalloc((void**)&P->d_sv_x, sizeof(double) * P->n));
    if (!P->sv_graph || P->sv_graph_store != d_store || P->sv_graph_key != form * 65536 + maxw) {
      if (P->sv_graph) cudaGraphExecDestroy(P->sv_graph);
      P->sv_graph = nullptr;
      CK(cudaStreamBeginCapture(P->cap_stream, cudaStreamCaptureModeThreadLocal));
      const int erc = enqueue(P->cap_stream, P->d_sv_x);
      cudaGraph_t g;
      CK(cudaStreamEndCapture(P->cap_stream, &g));
      if (erc) {
        cudaGraphDestroy(g);
        return erc;
      }
      cudaError_t e = cudaGraphInstantiate(&P->sv_graph, g, 0);
      cudaGraphDestroy(g);
      if (e != cudaSuccess) return fail(PS_ECUDA, "solve graph: %s", cudaGetErrorString(e));
      P->sv_graph_store = d_store;
      P->sv_graph_key = form * 65536 + maxw;
    }
    CK(cudaMemcpyAsync(P->d_sv_x, d_x, sizeof(double) * P->n, cudaMemcpyDeviceToDevice, s));
    CK(cudaGraphLaunch(P->sv_graph, s));
    CK(cudaMemcpyAsync(d_x, P->d_sv_x, sizeof(double) * P->n, cudaMemcpyDeviceToDevice, s));
  }
  CK(cudaGetLastError());
  if (prof) {
    cudaStreamSynchronize(s);
    for (size_t i = 1; i < ev.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
      const bool fwd = (int)i <= nlev;
      const int L = fwd ? (int)i - 1 : 2 * nlev - (int)i;
      if (ms > prof_min)
        fprintf(stderr, "[solve] %s level %d panels %lld: %.3f ms\n", fwd ? "fwd" : "bwd", L,
                (long long)(P->sv_lvl_ptr_h[L + 1] - P->sv_lvl_ptr_h[L]), ms);
    }
    for (auto e : ev) cudaEventDestroy(e);
  }
  return PS_OK;
}

int ps_set_tile_trace(ps_plan* P, void* d_trace) {
  if (!P) return fail(PS_EARG, "null argument");
  P->d_tile_trace = (unsigned long long*)d_trace;
  if (P->graph) {  // the captured graph holds the old arguments' address only; DevArgs is re-uploaded per call
  }
  return PS_OK;
}

int ps_plan_tiles(const ps_plan* P, int32_t* out /* 24 ints per tile (UTile fields) */) {
  if (!P || !out) return fail(PS_EARG, "null argument");
  if (P->tiles_h.empty()) return fail(PS_EARG, "tiles not kept (create the plan with PS_KEEP_TILES=1)");
  std::memcpy(out, P->tiles_h.data(), sizeof(UTile) * P->tiles_h.size());
  return PS_OK;
}

int ps_plan_tile_count(const ps_plan* P, int64_t* n) {
  if (!P || !n) return fail(PS_EARG, "null argument");
  *n = P->n_update_tiles + P->n_trail_tiles;
  return PS_OK;
}

int ps_plan_launch_work(const ps_plan* P, double* flops, double* bytes) {
  if (!P) return fail(PS_EARG, "null argument");
  for (size_t i = 0; i < P->launches.size(); ++i) {
    if (flops) flops[i] = P->launches[i].flops;
    if (bytes) bytes[i] = P->launches[i].bytes;
  }
  return PS_OK;
}

int ps_plan_set_schedule(ps_plan* P, int schedule) {
  if (!P) return fail(PS_EARG, "null argument");
  if (schedule != 0 && schedule != 1) return fail(PS_EARG, "bad schedule %d", schedule);
  if (schedule == 1 && !P->df_built) return fail(PS_EARG, "plan has no dataflow schedule");
  P->schedule = schedule;
  return PS_OK;
}

int ps_plan_dataflow_info(const ps_plan* P, ps_dataflow_info* info) {
  if (!P || !info) return fail(PS_EARG, "null argument");
  std::memset(info, 0, sizeof *info);
  info->schedule = P->schedule;
  info->built = P->df_built ? 1 : 0;
  info->ntasks = P->df_ntasks;
  info->ndeps = P->df_ndeps;
  info->ncounters = P->df_nctr;
  info->grid = P->df_grid;
  info->scratch_slots = P->df_slots;
  info->est_ms = P->df_est_us * 1e-3;
  for (i64 t = 0; t < P->df_ntasks; ++t) {
    const int k = P->df_type[t];
    if (k >= 0 && k < 8) {
      info->ntasks_by_type[k] += 1;
      info->flops_by_type[k] += P->df_flops[t];
    }
  }
  return PS_OK;
}

int ps_plan_tasks(const ps_plan* P, int32_t* type, int32_t* src, int32_t* dst, double* flops) {
  if (!P) return fail(PS_EARG, "null argument");
  for (i64 t = 0; t < P->df_ntasks; ++t) {
    if (type) type[t] = P->df_type[t];
    if (src) src[t] = P->df_src[t];
    if (dst) dst[t] = P->df_dst[t];
    if (flops) flops[t] = P->df_flops[t];
  }
  return PS_OK;
}

int ps_plan_task_graph(const ps_plan* P, int32_t* dep_ptr, int32_t* dep_ctr, int32_t* dep_target,
                       int32_t* sig_ptr, int32_t* sig_ctr) {
  if (!P) return fail(PS_EARG, "null argument");
  const i64 nt = P->df_ntasks;
  for (i64 t = 0; t <= nt && !P->df_dep0_h.empty(); ++t) {
    if (dep_ptr) dep_ptr[t] = P->df_dep0_h[t];
    if (sig_ptr) sig_ptr[t] = P->df_sig0_h[t];
  }
  for (size_t k = 0; k < P->df_deps_h.size(); ++k) {
    if (dep_ctr) dep_ctr[k] = P->df_deps_h[k].x;
    if (dep_target) dep_target[k] = P->df_deps_h[k].y;
  }
  for (size_t k = 0; k < P->df_sigs_h.size(); ++k)
    if (sig_ctr) sig_ctr[k] = P->df_sigs_h[k];
  return PS_OK;
}

int ps_factor_trace(ps_plan* P, double* d_store, int form, double thr, void* stream,
                    uint64_t* trace) {
  if (!P || (!d_store && P->store_elems) || !trace) return fail(PS_EARG, "null argument");
  if (!P->df_built) return fail(PS_EARG, "plan has no dataflow schedule");
  CK(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream;
  int rc = set_args(P, d_store, form, thr, s);
  if (rc) return rc;
  unsigned long long* d_tr = nullptr;
  const size_t nt = (size_t)std::max<i64>(1, P->df_ntasks);
  const size_t bytes = sizeof(unsigned long long) * 9 * nt;  // 5 trace + 4 phase words per task
  CK(cudaMalloc((void**)&d_tr, bytes));
  CK(cudaMemsetAsync(d_tr, 0, bytes, s));
  rc = enqueue_dataflow(P, s, d_tr, d_tr + 5 * nt);
  if (!rc) {
    cudaError_t e = cudaMemcpyAsync(trace, d_tr, bytes, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = fail(PS_ECUDA, "trace copy: %s", cudaGetErrorString(e));
  }
  cudaFree(d_tr);
  return rc;
}

}  // extern "C"
