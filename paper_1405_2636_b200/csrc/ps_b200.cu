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
#include <tuple>
#include <unordered_map>
#include <string>
#include <cstdarg>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ps_b200.h"
#include "ps_kernels.cuh"
#include "ps_diag.cuh"
#include "ps_generic.cuh"
#include "ps_solve.cuh"
#include "ps_p2p.cuh"
#include "ps_zupdate.cuh"

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
            K_TRSM = 6, K_JOIN = 9, K_FORK = 10, K_XWAIT = 11 };

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
  ChainSeg* d_chain = nullptr;          // merged chain tiles' sources (CHAIN_STRIDE per group)
  int nchain = 0;                       // merged chain groups
  std::unordered_map<int, std::vector<int>> merged_from;  // merged couple -> member couples
  FItem* d_fitems = nullptr;
  int* d_w1 = nullptr;
  unsigned* d_counters = nullptr;
  int* d_workctr = nullptr;
  i64* d_fail_col = nullptr;
  double* d_fail_piv = nullptr;
  Status* d_status = nullptr;
  unsigned long long* d_absmax = nullptr;  // device default pivot threshold: max |diag| bits
  DevArgs* d_args = nullptr;
  i64 n_update_tiles = 0, n_trail_tiles = 0, n_fitems = 0;
  std::vector<Launch> launches;
  int n_update_launches = 0;
  int max_colors = 0;
  int ngroups = 0;
  int noffload = 0;                     // wide panels factored on their own graph branch
  int fbranch = 0;                      // branch id of the per-level small-panel factors (0: none)
  int dbranch = 0;                      // branch id of the deferred (non-critical) updates
  int la_base = 0;                      // look-ahead: companion branch of chain stream X is la_base + X (0: off)
  int prio_hi = 0;                      // greatest stream / graph-node priority of the device
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
  std::vector<i64> lt_ptr, lt_task;     // per launch: the reference tasks it serves
                                        //   (p: factor of p, np + c: update couple c)
  std::vector<UTile> tiles_h;           // host copy of the level schedule's tiles (analysis)
  int cur_form = 0;                     // form code of the current call (ps_b200.h)
  std::map<int, cudaGraphExec_t> kgraphs;  // whole-factorization graphs per kernel family
  double* d_gs_fpart = nullptr;         // generic solve partials (complex-sized)
  double* d_gs_bpart = nullptr;
  cudaEvent_t last_ev = nullptr;        // end of the last call's work (PlanUse)
  cudaStream_t last_stream = nullptr;
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
  // factor + overlapped download (ps_factor_download): slab chunks of whole
  // panels, each copied once its last writing launch has run
  std::vector<i64> dl_off, dl_len;   // per chunk: slab element offset / count
  std::vector<int> dl_fin;           // per chunk: last launch writing it
  std::vector<std::vector<int>> dl_fins;  // per chunk: the last writing launch of each of its units
  std::vector<int> dl_order;         // chunks by ascending dl_fin
  cudaStream_t dl_stream = nullptr;
  cudaEvent_t dl_done = nullptr;
  // download graphs per (device slab, host slab, form): the form selects the kernels
  std::vector<std::pair<std::tuple<const double*, double*, int>, cudaGraphExec_t>> dl_graphs;
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

// panel-tree parent: the panel the first off-diagonal block faces (-1: root)
inline i64 parent_of(const ps_symbol_desc* S, i64 p) {
  return S->blkptr[p + 1] > S->blkptr[p] ? S->blk_facing[S->blkptr[p]] : -1;
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
//
// Look-ahead (part): the odd steps' update splits into the next column block
// (part 1: what step s+2's diagonal and TRSM need) and the column blocks
// beyond it (part 2), which the plan runs on a companion branch concurrently
// with step s+2's diagonal block and TRSM.  Every entry still receives the
// same K = 128 contractions in the same step order: results are unchanged.
#ifndef PS_TRAIL_G
#define PS_TRAIL_G 2  // steps per trailing group (3 / 4 measured: 120^3 -0.2 / -0.3%, 60^3 +0.8 / +1.4%)
#endif
constexpr int TRAIL_G = PS_TRAIL_G;
inline bool trail_group_end(int step) { return step % TRAIL_G == TRAIL_G - 1; }
void trailing_tiles_of_panel(std::vector<UTile>& out, int p, int w, int nrows, int step,
                             int part = 0) {
  const int c0 = step * FNB;
  const int nb = std::min(FNB, w - c0);
  const int b = c0 + nb;
  if (b >= w) return;
  const int g = step % TRAIL_G;  // steps of the group so far: c0 - g FNB .. c0 + nb
  const int k0 = c0 - g * FNB, kn = g * FNB + nb;
  if (!trail_group_end(step)) {
    if (part != 2) emit_tiles(out, p, p, b, nrows, b, std::min(w, b + FNB), k0, kn, -1, -1, 0);
  } else if (part == 0) {
    emit_tiles(out, p, p, b, nrows, b, w, k0, kn, -1, -1, 0);
  } else if (part == 1) {
    emit_tiles(out, p, p, b, nrows, b, std::min(w, b + FNB), k0, kn, -1, -1, 0);
  } else if (b + FNB < w) {
    emit_tiles(out, p, p, b + FNB, nrows, b + FNB, w, k0, kn, -1, -1, 0);
  }
}

int grid_for(const ps_plan* P, int kind, int count) {
  if (kind == K_W1) return std::max(1, std::min((count + 3) / 4, P->sms * 16));  // 4 warps/CTA
  if (kind == K_FACTOR || kind == K_FDIAG || kind == K_TRSM) return count;
  if (kind == K_SMALL)  // 4 warp tiles per CTA, at most 12 CTAs per SM
    return std::max(1, std::min((count + 3) / 4, P->sms * 12));
  return std::max(1, std::min(count, P->sms * P->upd_ctas_per_sm));
}

// kernel launch, optionally as a programmatic dependent launch (PDL): the
// grid may start launching while the previous grid on the stream finishes;
// every kernel opens with pdl_enter() (griddepcontrol.wait) before touching
// memory, so the stream order of results is unchanged
// priority of the kernels being enqueued (0: default); set per launch by
// enqueue_range from the launch's graph branch
static thread_local int g_launch_prio = 0;

template <typename... KArgs, typename... Args>
static cudaError_t klaunch(bool pdl, void (*k)(KArgs...), int grid, int block, size_t smem,
                           cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na++].val.programmaticStreamSerializationAllowed = 1;
  }
  if (g_launch_prio != 0) {  // graph node priority (critical-path launches first)
    at[na].id = cudaLaunchAttributePriority;
    at[na++].val.priority = g_launch_prio;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// form codes: PS_FORM_LLT / LDLT / LU, | PS_FORM_COMPLEX (complex128 values),
// | PS_FORM_GENERIC (real LLt / LDLt on the scalar-generic kernels: tests)
inline int base_form(int f) { return f & 15; }
inline bool form_complex(int f) { return (f & PS_FORM_COMPLEX) != 0; }
inline bool form_generic(int f) {
  return (f & (PS_FORM_COMPLEX | PS_FORM_GENERIC)) != 0 || base_form(f) == PS_FORM_LU;
}
// kernel family of a form (graph cache key): 0 tuned real LLt / LDLt,
// 1 + 3 * complex + base form for the generic kernels
inline int kernel_family(int f) {
  return form_generic(f) ? 1 + 3 * (form_complex(f) ? 1 : 0) + base_form(f) : 0;
}
inline size_t form_elem_bytes(int f) { return form_complex(f) ? 16 : 8; }
inline i64 form_slabs(int f) { return base_form(f) == PS_FORM_LU ? 2 : 1; }

template <class T, int F>
int launch_generic(ps_plan* P, const Launch& L, int idx, cudaStream_t s, const UTile* tiles,
                   const FItem* fitems, const int* w1) {
  switch (L.kind) {
    case K_JOIN:
    case K_FORK:
    case K_XWAIT:
      return PS_OK;
    case K_W1:
      CK(klaunch(P->pdl, g_factor_w1<T, F>, L.grid, 128, 0, s, w1 + L.first, L.count,
                 (const DevArgs*)P->d_args, P->pdev(), P->d_fail_col, P->d_fail_piv));
      break;
    case K_FACTOR:
      CK(klaunch(P->pdl, g_factor_small<T, F>, L.grid, FTR, 0, s, fitems + L.first,
                 (const DevArgs*)P->d_args, P->pdev(), P->d_fail_col, P->d_fail_piv));
      break;
    case K_FDIAG:
      CK(klaunch(P->pdl, g_factor_diag<T, F>, L.grid, GD_THREADS, sizeof(GDiagSmem<T, F>), s,
                 fitems + L.first, (const DevArgs*)P->d_args, P->pdev(), P->d_fail_col,
                 P->d_fail_piv));
      break;
    case K_TRSM:
      CK(klaunch(P->pdl, g_trsm<T, F>, L.grid, GD_THREADS, sizeof(GTrsmSmem<T>), s,
                 fitems + L.first, (const DevArgs*)P->d_args, P->pdev()));
      break;
    default: {  // K_TRAIL / K_UPDATE / K_SMALL: persistent tile CTAs
      if constexpr (sizeof(T) == 16) {
        if (L.kind != K_SMALL) {  // complex DMMA tiles (ps_zupdate.cuh)
          const int zg = std::max(1, std::min(L.count, P->sms * 2));
          CK(klaunch(P->pdl, k_zupdate<F>, zg, ZT, sizeof(ZSmem), s, tiles + L.first, L.count,
                     P->d_workctr + idx, P->d_counters, (const DevArgs*)P->d_args,
                     (const i64*)P->d_run_ptr, (const int*)P->d_run_src,
                     (const int*)P->d_run_dst));
          break;
        }
      }
      const int grid = std::max(1, std::min(L.count, P->sms * 4));
      CK(klaunch(P->pdl, g_update<T, F>, grid, GU_THREADS, sizeof(GUpdSmem<T>), s, tiles + L.first,
                 L.count, P->d_workctr + idx, P->d_counters, (const DevArgs*)P->d_args,
                 (const i64*)P->d_run_ptr, (const int*)P->d_run_src, (const int*)P->d_run_dst));
      break;
    }
  }
  CK(cudaGetLastError());
  return PS_OK;
}

template <class T, int F>
cudaError_t generic_attrs() {
  cudaError_t e = cudaFuncSetAttribute(g_factor_diag<T, F>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sizeof(GDiagSmem<T, F>));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(g_trsm<T, F>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(GTrsmSmem<T>));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(g_update<T, F>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(GUpdSmem<T>));
  if constexpr (sizeof(T) == 16)
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_zupdate<F>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)sizeof(ZSmem));
  return e;
}

// real LU: the DMMA update / trailing / wide-panel TRSM tiles run both passes
// (L and U^T) of each tile; diagonal blocks, small panels and narrow-source
// updates stay on the generic kernels
inline bool lu_on_dmma(int f, int kind) {
  return base_form(f) == PS_FORM_LU && !(f & (PS_FORM_COMPLEX | PS_FORM_GENERIC)) &&
         (kind == K_UPDATE || kind == K_TRAIL || kind == K_TRSM);
}

int launch_one(ps_plan* P, const Launch& L, int idx, cudaStream_t s, const UTile* tiles,
               const FItem* fitems, const int* w1) {
  if (form_generic(P->cur_form) && !lu_on_dmma(P->cur_form, L.kind)) {
    const bool c = form_complex(P->cur_form);
    switch (base_form(P->cur_form)) {
      case PS_FORM_LLT:
        return c ? launch_generic<cplx, FORM_LLT>(P, L, idx, s, tiles, fitems, w1)
                 : launch_generic<double, FORM_LLT>(P, L, idx, s, tiles, fitems, w1);
      case PS_FORM_LDLT:
        return c ? launch_generic<cplx, FORM_LDLT>(P, L, idx, s, tiles, fitems, w1)
                 : launch_generic<double, FORM_LDLT>(P, L, idx, s, tiles, fitems, w1);
      default:
        return c ? launch_generic<cplx, FORM_LU>(P, L, idx, s, tiles, fitems, w1)
                 : launch_generic<double, FORM_LU>(P, L, idx, s, tiles, fitems, w1);
    }
  }
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
      CK(klaunch(P->pdl, k_trsm8, L.grid, W8_THREADS, sizeof(UpdSmem), s, fitems + L.first,
                 (const DevArgs*)P->d_args, P->pdev()));
      break;
    case K_SMALL:
      CK(klaunch(P->pdl, k_update_narrow_w, L.grid, 128, 0, s, tiles + L.first, L.count,
                 P->d_workctr + idx, P->d_counters, P->d_args, P->d_run_ptr, P->d_run_src,
                 P->d_run_dst));
      break;
    case K_TRAIL:
      if (!P->d_tile_trace) {
        CK(klaunch(P->pdl, k_trail8, L.count, W8_THREADS, sizeof(UpdSmem), s, tiles + L.first,
                   (const DevArgs*)P->d_args));
        break;
      }
      CK(klaunch(P->pdl, k_update, L.grid, UPD_THREADS, sizeof(UpdSmem), s,
                 tiles + L.first, L.count, P->d_workctr + idx, P->d_counters, P->d_args, P->pdev(),
                 P->d_run_ptr, P->d_run_src, P->d_run_dst));
      break;
    default:
#ifndef PS_U8_KEFF
#define PS_U8_KEFF 64  // launches of mean tile K below this on the 8-warp kernel (its epilogue has twice the threads; 60^3 18.38 -> 18.19 ms)
#endif
      if (L.kind == K_UPDATE && !P->d_tile_trace &&
          (L.count < P->sms * 3 ||
           L.flops < (double)PS_U8_KEFF * 2.0 * TM * TN * L.count)) {  // small launches
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
  i64 esz = 1;      // doubles per element (complex: 2)
  i64 ustride = 0;  // LU: elements from the L slab to the U slab (the chunk is copied from both)
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
  const int nbr_ids = P->la_base > 0 ? P->la_base + P->noffload + 1 : P->noffload + 3;
  std::vector<char> started(nbr_ids, 0);
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
      const int b = (int)L.first, t = L.count;  // (0: the main stream)
      if (b == 0 || started[b]) {
        cudaEvent_t e = b ? P->side_ev[2 * b - 1] : P->side_ev.back();
        CK(cudaEventRecord(e, b ? P->side[b - 1] : s));
        CK(cudaStreamWaitEvent(t ? P->side[t - 1] : s, e, 0));
        if (t) started[t] = 1;
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
#ifndef PS_PRIO
#define PS_PRIO 1  // main stream + factor branch launches at the highest graph node priority
#endif
    g_launch_prio = 0;
    // (the tuned real LLt / LDLt kernels; LU measured 1.3% slower with them)
    if (PS_PRIO && (branches || offload) && !form_generic(P->cur_form)) {
      // 2 = highest, 1 = middle, 0 = default
#ifndef PS_PRIO_OFF
#define PS_PRIO_OFF 1  // offloaded wide-panel chains
#endif
#ifndef PS_PRIO_LA
#define PS_PRIO_LA 1   // look-ahead companions (bulk trailing updates)
#endif
#ifndef PS_PRIO_D
#define PS_PRIO_D 0    // deferred updates
#endif
      int lv = 2;  // main stream, factor branch
      if (L.stream == P->dbranch) lv = PS_PRIO_D;
      else if (P->la_base > 0 && L.stream >= P->la_base) lv = PS_PRIO_LA;
      else if (L.stream > 0 && L.stream <= P->noffload) lv = PS_PRIO_OFF;
      g_launch_prio = lv == 2 ? P->prio_hi : lv == 1 ? P->prio_hi / 2 : 0;
    }
    int rc = launch_one(P, L, (int)i, ls, P->d_tiles, P->d_fitems, P->d_w1);
    g_launch_prio = 0;
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
          for (i64 u = 0; u < (dl->ustride ? 2 : 1); ++u) {  // LU: the chunk's L and U parts
            const i64 o = (u * dl->ustride + P->dl_off[c]) * dl->esz;
            CK(cudaMemcpyAsync(dl->h + o, dl->d + o, sizeof(double) * P->dl_len[c] * dl->esz,
                               cudaMemcpyDeviceToHost, dl->cs));
          }
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

// A plan's device state (arguments, counters, status, solve buffers, cached
// graphs) serves one call at a time: a call on another stream than the
// previous one first waits for that call's work (event recorded at the end of
// every entry point), so calls on different streams serialize instead of
// corrupting each other.
struct PlanUse {
  ps_plan* P;
  cudaStream_t s;
  PlanUse(ps_plan* P_, cudaStream_t s_) : P(P_), s(s_) {
    if (P->last_ev && P->last_stream != s) cudaStreamWaitEvent(s, P->last_ev, 0);
  }
  ~PlanUse() {
    if (!P->last_ev) cudaEventCreateWithFlags(&P->last_ev, cudaEventDisableTiming);
    if (P->last_ev) cudaEventRecord(P->last_ev, s);
    P->last_stream = s;
  }
};

int set_args(ps_plan* P, double* store, int form, double thr, cudaStream_t s) {
  if (base_form(form) > PS_FORM_LU || (form & ~(15 | PS_FORM_COMPLEX | PS_FORM_GENERIC)))
    return fail(PS_EARG, "bad form %d", form);
  P->cur_form = form;
  DevArgs a{store, P->d_scratch, thr, base_form(form), 0, P->d_tile_trace, P->d_tiles,
            base_form(form) == PS_FORM_LU ? P->store_elems : 0, P->d_chain};
  // pageable memcpy is stream-ordered and completes the source read on return
  const bool dev_thr = std::isnan(thr);
  if (dev_thr) a.thr = 0.0;
  CK(cudaMemcpyAsync(P->d_args, &a, sizeof a, cudaMemcpyHostToDevice, s));
  if (dev_thr) {  // the reference default from the assembled slab, no host round trip
    CK(cudaMemsetAsync(P->d_absmax, 0, sizeof(unsigned long long), s));
    if (P->np > 0)
      k_diag_absmax<<<P->sms * 4, 256, 0, s>>>(store, P->pdev(), P->np,
                                                (form & PS_FORM_COMPLEX) ? 1 : 0, P->d_absmax);
    k_set_threshold<<<1, 1, 0, s>>>(P->d_args, P->d_absmax);
    CK(cudaGetLastError());
  }
  return PS_OK;
}

}  // namespace

extern "C" {

const char* ps_last_error(void) { return g_err.c_str(); }

int ps_host_register(void* ptr, int64_t bytes, int* registered) {
  if (!registered) return fail(PS_EARG, "null argument");
  *registered = 0;
  if (!ptr || bytes <= 0) return PS_OK;
  cudaError_t e = cudaHostRegister(ptr, (size_t)bytes, cudaHostRegisterDefault);
  if (e == cudaSuccess) {
    *registered = 1;
  } else if (e == cudaErrorHostMemoryAlreadyRegistered) {
    *registered = 2;  // page-locked by someone else: usable, not ours to unregister
  }
  cudaGetLastError();  // this library's runtime state only: leave no sticky error behind
  return PS_OK;
}

int ps_host_unregister(void* ptr) {
  if (!ptr) return PS_OK;
  cudaError_t e = cudaHostUnregister(ptr);
  cudaGetLastError();
  return e == cudaSuccess ? PS_OK : fail(PS_ECUDA, "cudaHostUnregister: %s", cudaGetErrorString(e));
}

static int plan_create_impl(const ps_symbol_desc* S, int device, const int32_t* group_in,
                            int ngroups_in, int my_group, ps_plan** out,
                            const int32_t* top_owner = nullptr) {
  if (!S || !out) return fail(PS_EARG, "null argument");
  *out = nullptr;
  if (S->npanels < 0 || S->n < 0) return fail(PS_EARG, "negative sizes");
  if (S->npanels >= (1LL << 31)) return fail(PS_EARG, "too many panels");
  CK(cudaSetDevice(device));
  auto* P = new ps_plan();
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
  // padding: tile kernels load a whole 32 / 64-run window without first
  // reading the couple's end (the loads do not wait for it)
  run_src.insert(run_src.end(), 64, 0x7fffffff);
  run_dst.insert(run_dst.end(), 64, 0);
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
  // ---- merged chain updates (single-GPU plans) ----
  // Split pieces p_1..p_m of one supernode (each the parent of the previous,
  // rows exactly nested: rows(p_i) = cols(p_{i+1}) + rows(p_{i+1})) face the
  // same entries of every ancestor q beyond the chain, so their updates into
  // q are ONE tile of K = w_1 + ... + w_m (sources per 16-wide k chunk,
  // ChainSeg), emitted at p_m's level: the top separators' 128-wide pieces
  // become K = 128 m contractions (fewer epilogues, higher DMMA efficiency).
  // The member couples (p_i -> q, i < m) are not emitted on their own.
  std::vector<int> merged_into(nc, -1), cmerge(nc, -1), ckn(nc, 0);
  for (i64 c = 0; c < nc; ++c) ckn[c] = P->h_w[c_p[c]];
  std::vector<ChainSeg> chain_h;
  {
    int gm = 4;
    if (const char* e = getenv("PS_CHAIN_MERGE")) gm = atoi(e);  // A/B knob: 1 = off
    gm = std::max(1, std::min(gm, CHAIN_GM));
    auto nests = [&](i64 p) -> bool {  // link p -> p + 1
      const i64 q = p + 1;
      if (q >= np || parent_of(S, p) != q) return false;
      if (P->h_w[p] % KC || P->h_w[q] % KC || P->h_w[p] > 256 || P->h_w[q] > 256) return false;
      const int wq = P->h_w[q];
      const i64 rp0 = S->rowptr[p], rp1 = S->rowptr[p + 1], rq0 = S->rowptr[q], rq1 = S->rowptr[q + 1];
      if (rp1 - rp0 != wq + (rq1 - rq0)) return false;
      for (int j = 0; j < wq; ++j)
        if (S->rows[rp0 + j] != S->starts[q] + j) return false;
      for (i64 j = 0; j < rq1 - rq0; ++j)
        if (S->rows[rp0 + wq + j] != S->rows[rq0 + j]) return false;
      return true;
    };
    for (i64 p0 = 0; gm >= 2 && !group_in && p0 < np;) {
      i64 e = p0;
      while (e + 1 < np && nests(e)) ++e;  // chain p0 .. e
      for (i64 a = p0; a < e; a += gm) {
        const i64 last = std::min(e, a + gm - 1);
        const int gid = (int)(chain_h.size() / CHAIN_STRIDE);
        // step form (ps_kernels.cuh ChainSeg): virtual column-0 pointers of
        // each piece, as increments from p_last's column 0
        std::vector<ChainSeg> segs(CHAIN_STRIDE, ChainSeg{0, 0, 0, INT_MAX});
        int kb = 0;
        i64 prev_a = P->off[last], prev_d = P->off[last];
        for (i64 i = a; i <= last; ++i) {
          i64 sh = 0;
          for (i64 t = i; t < last; ++t) sh += P->h_w[t];
          const i64 lds_i = P->h_nrows[i];
          const i64 va = P->off[i] + sh - (i64)kb * lds_i, vd = P->off[i] - (i64)kb * (lds_i + 1);
          segs[i - a] = ChainSeg{va - prev_a, vd - prev_d, (int)lds_i, kb};
          prev_a = va;
          prev_d = vd;
          kb += P->h_w[i];
        }
        bool any = false;
        for (i64 cm = P->cpl_first[last]; cm < P->cpl_first[last + 1]; ++cm) {
          const int q = c_q[cm];
          // the next level's destination stays unmerged: its updates are on the
          // critical path and already run early (deferred at each piece's level)
          if (level[q] <= level[last] + 1) continue;
          std::vector<int> mem;
          bool ok = true;
          for (i64 i = a; i < last && ok; ++i) {
            i64 f = -1;
            for (i64 ci = P->cpl_first[i]; ci < P->cpl_first[i + 1]; ++ci)
              if (c_q[ci] == q) {
                f = ci;
                break;
              }
            ok = f >= 0 && c_N[f] == c_N[cm] && c_g1[f] - c_g0[f] == c_g1[cm] - c_g0[cm];
            for (i64 t = 0; ok && t < c_g1[cm] - c_g0[cm]; ++t)
              ok = S->blk_fr[c_g0[f] + t] == S->blk_fr[c_g0[cm] + t] &&
                   S->blk_lr[c_g0[f] + t] == S->blk_lr[c_g0[cm] + t];
            if (ok) mem.push_back((int)f);
          }
          if (!ok) continue;
          for (int ci : mem) merged_into[ci] = (int)cm;
          cmerge[cm] = gid;
          ckn[cm] = kb;
          P->merged_from[(int)cm] = mem;
          any = true;
        }
        if (any) chain_h.insert(chain_h.end(), segs.begin(), segs.end());
      }
      p0 = e + 1;
    }
    P->nchain = (int)(chain_h.size() / CHAIN_STRIDE);
  }

  // ---- subtree partition (multi-GPU plans): group[p] = rank
  //      of p's subtree, -1 = the shared top ----
  std::vector<int> parent(np, -1);
  for (i64 p = 0; p < np; ++p)
    if (S->blkptr[p + 1] > S->blkptr[p]) parent[p] = (int)S->blk_facing[S->blkptr[p]];
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
  int slot_base = 0, slot_max = 0;           // scratch slots of the current group
  // narrow sources: warp tiles of 32 x 32; couples colored heaviest first
  // factor launches of one level (panels pl), on graph branch `stream`
  std::function<void(int)> branch_hook;  // emitted on the factor branch after the small factors
  // trailing updates of step s of the wide panels pl on chain stream X:
  // with look-ahead (P->la_base > 0) an odd step's update beyond the next
  // column block goes to X's companion branch (forked off X after the TRSM),
  // and X waits for it before its next trailing launch (the even step's
  // update of that block, same entries) or at the end of the chain
  auto emit_trailing = [&](const std::vector<int>& pl, int s, int L, int X, bool& pending) {
    auto wide = [&](int p) { return P->h_w[p] > SNB && P->h_w[p] > (s + 1) * FNB; };
    const bool split = P->la_base > 0 && trail_group_end(s);
    if (split) {
      const i64 t0 = (i64)tiles.size();
      for (int p : pl)
        if (wide(p)) trailing_tiles_of_panel(tiles, p, P->h_w[p], P->h_nrows[p], s, 2);
      const int cnt = (int)((i64)tiles.size() - t0);
      P->n_trail_tiles += cnt;
      if (cnt) {
        const int la = P->la_base + X;
        P->launches.push_back(Launch{K_XWAIT, L, X, la, 0, 0});
        P->launches.push_back(Launch{K_TRAIL, L, t0, cnt, grid_for(P, K_TRAIL, cnt), la});
        pending = true;
      }
    }
    const i64 t0 = (i64)tiles.size();
    for (int p : pl)
      if (wide(p)) trailing_tiles_of_panel(tiles, p, P->h_w[p], P->h_nrows[p], s, split ? 1 : 0);
    const int cnt = (int)((i64)tiles.size() - t0);
    P->n_trail_tiles += cnt;
    if (!cnt) return;
    if (pending && !split) {
      P->launches.push_back(Launch{K_XWAIT, L, P->la_base + X, X, 0, 0});
      pending = false;
    }
    P->launches.push_back(Launch{K_TRAIL, L, t0, cnt, grid_for(P, K_TRAIL, cnt), X});
  };
  bool la_pending = false;
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
    for (int s = 0; s < steps; ++s) {
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
      emit_trailing(pl, s, L, stream, la_pending);
    }
    if (la_pending) {  // the chain stream waits for the last look-ahead update
      P->launches.push_back(Launch{K_XWAIT, L, P->la_base + stream, stream, 0, 0});
      la_pending = false;
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
    for (int pass = 0; pass < 2; ++pass) {
      if (!((passes >> pass) & 1)) continue;
      const std::vector<int>& lc = pass == 0 ? lc_small : lc_big;
      const int kind = pass == 0 ? K_SMALL : K_UPDATE;
      if (lc.empty()) continue;
      std::vector<int> color(lc.size());
      std::vector<int> touched;
      int maxcolor = 0;
      // coloring order: heaviest couple first, so that huge-K sources take the
      // low colors and start at once instead of waiting at the end of a
      // destination's chain (60^3 -0.5 ms, 80^3 -0.5 ms vs ascending ids)
      std::vector<size_t> corder(lc.size());
      for (size_t k = 0; k < lc.size(); ++k) corder[k] = k;
      {
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
          const int sig = k < topcolor[q] ? 1 : 0;
          const int tsz = kind == K_SMALL ? NW_T : TM;  // warp tiles: 32 x 32
          emit_tiles(tiles, p, q, loc0, nr, loc0, loc0 + N, 0, ckn[c], c, waits[u], sig,
                     run_ptr, run_src, tsz, tsz);
          if (cmerge[c] >= 0)  // merged chain tile: its sources per k chunk
            for (i64 t = before; t < (i64)tiles.size(); ++t) tiles[t].mode = cmerge[c] + 1;
          if (sig) launch_cnt[q] += (i64)tiles.size() - before;
        }
        // heaviest tiles of the color class first: they start while lighter
        // ones fill the remaining CTAs (tiles of one class never wait on each other)
        std::stable_sort(tiles.begin() + cbeg, tiles.end(), [](const UTile& a, const UTile& b) {
          return (double)a.ni * a.nj * a.kn > (double)b.ni * b.nj * b.kn;
        });
      }
      for (int q : touched) { base[q] += launch_cnt[q]; launch_cnt[q] = 0; topcolor[q] = 0; }
      int cnt = (int)((i64)tiles.size() - t0);
      P->n_update_tiles += cnt;
      if (cnt) {
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
    const int min_steps = 6;
    if (!group_in) {
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
    if (!group_in) {
      P->fbranch = P->noffload + 1;
      P->dbranch = P->noffload + 2;
      const char* e = getenv("PS_LOOKAHEAD");  // A/B knob: 0 = off
      if (!e || atoi(e) != 0) P->la_base = P->noffload + 3;
    }
  }
  bool defer_pending = false;  // deferred updates of the previous level still on their branch
  auto emit_offloaded = [&](int p, int L) {
    const int b = off_branch[p], w = P->h_w[p], nr = P->h_nrows[p];
    const int steps = (w + FNB - 1) / FNB;
    bool pend = false;
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
      emit_trailing(std::vector<int>{p}, st, L, b, pend);
    }
    if (pend) P->launches.push_back(Launch{K_XWAIT, L, P->la_base + b, b, 0, 0});
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
          if (merged_into[c] >= 0) continue;  // applied by its merged chain tile
          if (gid >= 0 && grp[c_q[c]] != gid) deferred.push_back((int)c);
          else cl.push_back((int)c);
        }
      // narrow-source updates depend only on the small factors: on the factor
      // branch they overlap the wide-panel chain (offloaded panels' deferred
      // couples are all wide: they stay in the main-stream DMMA launch)
      std::vector<int> cl_narrow;
      bool narrow_on_branch = false;
      if (P->fbranch > 0 && stream == 0) {
        for (int c : cl)
          if (P->h_w[c_p[c]] <= SMALL_W) cl_narrow.push_back(c);
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
        if (!defr.empty()) {
          P->launches.push_back(Launch{K_FORK, L, P->dbranch, 0, 0, 0});
          emit_updates(defr, L, P->dbranch, passes);
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

  P->n_fitems = (i64)fitems.size();
  // launch -> reference task ids (taskgraph.py:79-110 numbering: factor
  // tasks 0..np-1, then one update task per couple in panel / block order)
  P->lt_ptr.assign(1, 0);
  for (const Launch& L : P->launches) {
    std::vector<i64> ts;
    for (i64 t = L.first; t < L.first + L.count; ++t) {
      switch (L.kind) {
        case K_W1: ts.push_back(w1[t]); break;
        case K_FACTOR: case K_FDIAG: case K_TRSM: ts.push_back(fitems[t].p); break;
        case K_TRAIL: ts.push_back(tiles[t].dst); break;
        case K_UPDATE: case K_SMALL: {
          ts.push_back(np + tiles[t].couple);
          if (tiles[t].mode > 0)
            for (int m : P->merged_from[tiles[t].couple]) ts.push_back(np + m);
          break;
        }
        default: break;
      }
    }
    std::sort(ts.begin(), ts.end());
    ts.erase(std::unique(ts.begin(), ts.end()), ts.end());
    P->lt_task.insert(P->lt_task.end(), ts.begin(), ts.end());
    P->lt_ptr.push_back((i64)P->lt_task.size());
  }
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
    bool known = true;
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
      (rc = upload(&P->d_chain, chain_h, &P->dev_bytes)) ||
      ((P->tiles_h = getenv("PS_KEEP_TILES") ? tiles : std::vector<UTile>()), 0) ||
      (rc = upload(&P->d_fitems, fitems, &P->dev_bytes)) ||
      (rc = upload(&P->d_w1, w1, &P->dev_bytes)) ||
      0) {
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
      (rc = alloc((void**)&P->d_absmax, sizeof(unsigned long long))) ||
      (rc = alloc((void**)&P->d_args, sizeof(DevArgs))) ||
      (rc = alloc((void**)&P->d_scratch,
                  4 * sizeof(double) * FNB * FNB *  // generic complex LU: 2 complex operators / slot
                      std::max<i64>(1, P->scratch_slots)))) {
    ps_plan_destroy(P);
    return rc;
  }
  cudaError_t e = cudaFuncSetAttribute(k_update, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sizeof(UpdSmem));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_trail8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(UpdSmem));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_trsm8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(UpdSmem));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_update8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(UpdSmem));
  if (e == cudaSuccess) e = generic_attrs<double, FORM_LLT>();
  if (e == cudaSuccess) e = generic_attrs<double, FORM_LDLT>();
  if (e == cudaSuccess) e = generic_attrs<double, FORM_LU>();
  if (e == cudaSuccess) e = generic_attrs<cplx, FORM_LLT>();
  if (e == cudaSuccess) e = generic_attrs<cplx, FORM_LDLT>();
  if (e == cudaSuccess) e = generic_attrs<cplx, FORM_LU>();
  if (e != cudaSuccess) {
    ps_plan_destroy(P);
    return fail(PS_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_update, UPD_THREADS, sizeof(UpdSmem));
  P->upd_ctas_per_sm = std::max(1, occ);
  const int defer_ctas = 8;  // deferred-branch update launches: CTAs per SM (60^3: 3 -> 8 = 26.4 -> 25.1 ms; more: flat)
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
  const int nbr = P->la_base > 0 ? P->la_base + P->noffload
                                 : P->noffload + (P->fbranch ? 1 : 0) + (P->dbranch ? 1 : 0);
  const int nside = P->ngroups > 0 ? P->ngroups : nbr;
  const int nev = P->ngroups > 0 ? P->ngroups + 1 : 2 * nbr + 1;  // (+1: the main stream's)
  P->side.assign(nside, nullptr);
  P->side_ev.assign(nev, nullptr);
  {
    int least = 0, greatest = 0;
    if (cudaDeviceGetStreamPriorityRange(&least, &greatest) == cudaSuccess) P->prio_hi = greatest;
  }
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
  PlanUse use_(P, s);
  int rc = set_args(P, d_store, form, thr, s);
  if (rc) return rc;
  if (form_generic(form)) return fail(PS_EARG, "partitioned (multi-GPU) plans run real LLt / LDLt only");
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
    e = cudaGraphInstantiate(&G, g, PS_PRIO ? cudaGraphInstantiateFlagUseNodePriority : 0);
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
  for (auto& kv : P->kgraphs)
    if (kv.second) cudaGraphExecDestroy(kv.second);
  if (P->d_gs_fpart) cudaFree(P->d_gs_fpart);
  if (P->d_gs_bpart) cudaFree(P->d_gs_bpart);
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
                  P->d_run_dst, P->d_tiles, P->d_chain, P->d_fitems, P->d_w1, P->d_counters,
                  P->d_workctr, P->d_fail_col, P->d_fail_piv, P->d_status, P->d_absmax, P->d_args, P->d_scratch,
                  P->d_task_tiles, P->d_task_items, P->d_task_w1, P->d_sv_lvl_ptr,
                  P->d_sv_lvl_panels, P->d_sv_fbase, P->d_sv_bbase, P->d_sv_fitems,
                  P->d_sv_bitems, P->d_sv_rowptr, P->d_sv_rows, P->d_sv_z, P->d_sv_scratch,
                  P->d_sv_jptr, P->d_sv_jidx,
                  P->d_sv_fpart, P->d_sv_bpart, P->d_sv_vw, P->d_sv_vnro, P->d_sv_vfc,
                  P->d_sv_voff, P->d_sv_vld, P->d_sv_ritems, P->d_sv_x};
  if (P->sv_graph) cudaGraphExecDestroy(P->sv_graph);
  for (auto& kv : P->dl_graphs) cudaGraphExecDestroy(kv.second);
  if (P->dl_done) cudaEventDestroy(P->dl_done);
  if (P->dl_stream) cudaStreamDestroy(P->dl_stream);
  if (P->last_ev) cudaEventDestroy(P->last_ev);
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
  info->nlaunches = (int32_t)P->launches.size();
  info->device_bytes = P->dev_bytes;
  return PS_OK;
}

int ps_plan_offsets(const ps_plan* P, int64_t* offsets) {
  if (!P || !offsets) return fail(PS_EARG, "null argument");
  std::memcpy(offsets, P->off.data(), sizeof(i64) * P->off.size());
  return PS_OK;
}

int ps_assemble_form(ps_plan* P, void* d_store, const int64_t* d_pos, const void* d_vals,
                     int64_t nvals, int form, void* stream) {
  if (!P || (!d_store && P->store_elems)) return fail(PS_EARG, "null argument");
  CK(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream;
  PlanUse use_(P, s);
  const i64 elems = form_slabs(form) * P->store_elems;
  if (elems) CK(cudaMemsetAsync(d_store, 0, form_elem_bytes(form) * elems, s));
  if (nvals > 0) {
    int grid = (int)std::min<i64>((nvals + 255) / 256, (i64)P->sms * 32);
    if (form_complex(form))
      g_assemble<cplx><<<grid, 256, 0, s>>>((cplx*)d_store, d_pos, (const cplx*)d_vals, nvals);
    else
      g_assemble<double><<<grid, 256, 0, s>>>((double*)d_store, d_pos, (const double*)d_vals, nvals);
    CK(cudaGetLastError());
  }
  return PS_OK;
}

int ps_assemble(ps_plan* P, double* d_store, const int64_t* d_pos, const double* d_vals,
                int64_t nvals, void* stream) {
  if (!P || (!d_store && P->store_elems)) return fail(PS_EARG, "null argument");
  CK(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream;
  PlanUse use_(P, s);
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
  PlanUse use_(P, s);
  int rc = set_args(P, d_store, form, thr, s);
  if (rc) return rc;
  if (phase >= 0 && form_generic(form))
    return fail(PS_EARG, "partitioned (multi-GPU) plans run real LLt / LDLt only");
  // one graph per kernel family (the kernels are baked into the graph)
  cudaGraphExec_t& G = phase < 0 ? (kernel_family(form) == 0 ? P->graph : P->kgraphs[kernel_family(form)])
                                 : P->phase_graph[phase];
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
    e = cudaGraphInstantiate(&G, g, PS_PRIO ? cudaGraphInstantiateFlagUseNodePriority : 0);
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
  PlanUse use_(P, s);
  const size_t nc = P->dl_fin.size();
  if (nc == 0 || P->launches.empty()) {  // copy after the factorization
    int rc = ps_factor(P, d_store, form, thr, stream);
    if (rc) return rc;
    if (P->store_elems)
      CK(cudaMemcpyAsync(h_dst, d_store, form_elem_bytes(form) * form_slabs(form) * P->store_elems,
                         cudaMemcpyDeviceToHost, s));
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
  auto key = std::make_tuple((const double*)d_store, h_dst, form);
  cudaGraphExec_t G = nullptr;
  for (auto& kv : P->dl_graphs)
    if (kv.first == key) G = kv.second;
  if (!G) {
    std::vector<std::vector<int>> after(P->launches.size());
    for (int c : P->dl_order)
      for (int f : P->dl_fins[c]) after[f].push_back(c);
    DlCapture dl{&after, P->dl_stream, P->dl_done, d_store, h_dst,
                 form_complex(form) ? 2 : 1, form_slabs(form) == 2 ? P->store_elems : 0};
    CK(cudaStreamBeginCapture(P->cap_stream, cudaStreamCaptureModeThreadLocal));
    rc = enqueue_range(P, P->cap_stream, nullptr, 0, P->launches.size(), true, true, &dl);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(P->cap_stream, &g);
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (e != cudaSuccess) return fail(PS_ECUDA, "graph capture: %s", cudaGetErrorString(e));
    e = cudaGraphInstantiate(&G, g, PS_PRIO ? cudaGraphInstantiateFlagUseNodePriority : 0);
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
  return ps_factor_timeline(P, d_store, form, thr, stream, ms_by_kind, nlaunch, per_launch_ms,
                            nullptr);
}

int ps_factor_timeline(ps_plan* P, double* d_store, int form, double thr, void* stream,
                       double* ms_by_kind, int32_t* nlaunch, float* per_launch_ms,
                       float* start_ms) {
  if (!P || (!d_store && P->store_elems)) return fail(PS_EARG, "null argument");
  CK(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream;
  PlanUse use_(P, s);
  int rc = set_args(P, d_store, form, thr, s);
  if (rc) return rc;
  const size_t nl = P->launches.size();
  std::vector<cudaEvent_t> ev(2 * nl);
  for (auto& e : ev) CK(cudaEventCreate(&e));
  rc = enqueue_all(P, s, ev.data());
  if (!rc) {
    CK(cudaStreamSynchronize(s));
    if (ms_by_kind)
      for (int k = 0; k < 3; ++k) ms_by_kind[k] = 0.0;
    for (size_t i = 0; i < nl; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[2 * i], ev[2 * i + 1]);
      int k = P->launches[i].kind;
      if (ms_by_kind)
        ms_by_kind[(k == K_W1 || k == K_FACTOR || k == K_FDIAG || k == K_TRSM) ? 0 : (k == K_TRAIL ? 1 : 2)] += ms;
      if (per_launch_ms) per_launch_ms[i] = ms;
      if (start_ms) {
        float t0 = 0.f;
        if (i) cudaEventElapsedTime(&t0, ev[0], ev[2 * i]);
        start_ms[i] = t0;
      }
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
    if (branch) {  // markers: the branch they fork / join / wait for
      const Launch& L = P->launches[i];
      const bool marker = L.kind == K_JOIN || L.kind == K_FORK || L.kind == K_XWAIT;
      branch[i] = marker ? (int32_t)L.first : L.stream;
    }
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
  PlanUse use_(P, s);
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
    Launch L{K_W1, 0, 0, 1, 1, 0};
    if ((rc = launch_one(P, L, 0, s, nullptr, nullptr, P->d_task_w1))) return rc;
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
  PlanUse use_(P, s);
  int rc = set_args(P, d_store, form, 0.0, s);
  if (rc) return rc;
  i64 c = -1;
  for (i64 k = P->cpl_first[p]; k < P->cpl_first[p + 1]; ++k)
    if (P->cpl_q[k] == q) c = k;
  if (c < 0) return fail(PS_STRUCTURAL, "no blocks of panel %lld face panel %lld", (long long)p, (long long)q);
  std::vector<UTile> tl;
  const int loc0 = P->cpl_loc0[c], N = P->cpl_N[c];
  const int tsz = P->h_w[p] <= SMALL_W ? NW_T : TM;
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

}  // extern "C"

// triangular solve of the generic forms (ps_generic.cuh gs_*): the same
// virtual panels, levels, items and partial layouts as the tuned solve
template <class T, int F>
int solve_generic(ps_plan* P, const T* store, T* x, cudaStream_t s) {
  if (!P->d_gs_fpart) {
    CK(cudaMalloc((void**)&P->d_gs_fpart, 16 * std::max<i64>(1, P->sv_nfpart)));
    CK(cudaMalloc((void**)&P->d_gs_bpart, 16 * std::max<i64>(1, P->sv_nbpart)));
  }
  T* fpart = reinterpret_cast<T*>(P->d_gs_fpart);
  T* bpart = reinterpret_cast<T*>(P->d_gs_bpart);
  SolveDev S{P->d_sv_lvl_ptr, P->d_sv_lvl_panels, P->d_sv_vw, P->d_sv_vnro, P->d_sv_vfc,
             P->d_sv_voff, P->d_sv_vld, P->d_sv_fbase, P->d_sv_jptr, P->d_sv_jidx,
             P->d_sv_bbase, P->d_sv_fitems, P->d_sv_bitems, P->d_sv_ritems, P->d_sv_rowptr,
             P->d_sv_rows};
  const T* tstore = F == FORM_LU ? store + P->store_elems : store;
  const int nlev = (int)P->sv_lvl_ptr_h.size() - 1;
  auto smem = [&](int L) {
    int mw = 1;
    for (i64 t = P->sv_lvl_ptr_h[L]; t < P->sv_lvl_ptr_h[L + 1]; ++t)
      mw = std::max(mw, P->sv_vw_h[P->sv_lvl_panels_h[t]]);
    return sizeof(T) * (size_t)mw;
  };
  for (int L = 0; L < nlev; ++L) {
    const i64 r0 = P->sv_ri_ptr_h[L], nr = P->sv_ri_ptr_h[L + 1] - r0;
    if (nr > 0) gs_freduce<T><<<(int)((nr * 8 + GS_THREADS - 1) / GS_THREADS), GS_THREADS, 0, s>>>(r0, (int)nr, S, x, fpart);
    const i64 t0 = P->sv_lvl_ptr_h[L], np = P->sv_lvl_ptr_h[L + 1] - t0;
    if (np > 0) gs_fdiag<T, F><<<(int)np, GS_THREADS, smem(L), s>>>(t0, S, store, x);
    const i64 f0 = P->sv_fi_ptr_h[L], nf = P->sv_fi_ptr_h[L + 1] - f0;
    if (nf > 0) gs_fgemv<T><<<(int)nf, GS_THREADS, 0, s>>>(f0, S, store, x, fpart);
    CK(cudaGetLastError());
  }
  if (F != FORM_LLT && P->sv_nvirt > 0)
    gs_scale<T><<<std::min(P->sv_nvirt, P->sms * 8), GS_THREADS, 0, s>>>(P->sv_nvirt, S, store, x);
  for (int L = nlev - 1; L >= 0; --L) {
    const i64 b0 = P->sv_bi_ptr_h[L], nb = P->sv_bi_ptr_h[L + 1] - b0;
    if (nb > 0) gs_bgemv<T><<<(int)nb, GS_THREADS, 0, s>>>(b0, S, tstore, x, bpart);
    const i64 t0 = P->sv_lvl_ptr_h[L], np = P->sv_lvl_ptr_h[L + 1] - t0;
    if (np > 0) gs_bdiag<T, F><<<(int)np, GS_THREADS, smem(L), s>>>(t0, S, store, tstore, x, bpart);
    CK(cudaGetLastError());
  }
  return PS_OK;
}

extern "C" {

int ps_solve(ps_plan* P, const double* d_store, double* d_x, int form, void* stream) {
  if (!P || (!d_store && P->store_elems) || (!d_x && P->n)) return fail(PS_EARG, "null argument");
  if (base_form(form) > PS_FORM_LU || (form & ~(15 | PS_FORM_COMPLEX | PS_FORM_GENERIC)))
    return fail(PS_EARG, "bad form %d", form);
  CK(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream;
  PlanUse use_(P, s);
  if (form_generic(form)) {
    const bool c = form_complex(form);
    switch (base_form(form)) {
      case PS_FORM_LLT:
        return c ? solve_generic<cplx, FORM_LLT>(P, (const cplx*)d_store, (cplx*)d_x, s)
                 : solve_generic<double, FORM_LLT>(P, d_store, d_x, s);
      case PS_FORM_LDLT:
        return c ? solve_generic<cplx, FORM_LDLT>(P, (const cplx*)d_store, (cplx*)d_x, s)
                 : solve_generic<double, FORM_LDLT>(P, d_store, d_x, s);
      default:
        return c ? solve_generic<cplx, FORM_LU>(P, (const cplx*)d_store, (cplx*)d_x, s)
                 : solve_generic<double, FORM_LU>(P, d_store, d_x, s);
    }
  }
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

int ps_plan_launch_tasks(const ps_plan* P, int64_t* ptr, int64_t* task) {
  if (!P || !ptr) return fail(PS_EARG, "null argument");
  std::memcpy(ptr, P->lt_ptr.data(), sizeof(i64) * P->lt_ptr.size());
  if (task && !P->lt_task.empty()) std::memcpy(task, P->lt_task.data(), sizeof(i64) * P->lt_task.size());
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

// ---- peer-to-peer primitives of the multi-GPU factorization (ps_p2p.cuh) ----

int ps_p2p_segment_add(double* d_dst, const double* d_src, const int64_t* d_seg,
                       const int64_t* d_start, int32_t nseg, int64_t total, void* stream) {
  if (total <= 0 || nseg <= 0) return PS_OK;
  if (!d_dst || !d_src || !d_seg || !d_start) return fail(PS_EARG, "null argument");
  int dev = 0, sms = 148;
  CK(cudaGetDevice(&dev));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const i64 want = (total + 255) / 256;
  const int grid = (int)std::max<i64>(1, std::min<i64>(want, (i64)sms * 8));
  k_segment_add<<<grid, 256, 0, (cudaStream_t)stream>>>(d_dst, d_src, d_seg, d_start, nseg, total);
  CK(cudaGetLastError());
  return PS_OK;
}

int ps_p2p_signal(uint64_t* d_flag, uint64_t value, void* stream) {
  if (!d_flag) return fail(PS_EARG, "null argument");
  k_flag_signal<<<1, 1, 0, (cudaStream_t)stream>>>((unsigned long long*)d_flag,
                                                   (unsigned long long)value);
  CK(cudaGetLastError());
  return PS_OK;
}

int ps_p2p_wait(const uint64_t* d_flag, uint64_t value, int32_t* d_timeout, double timeout_s,
                void* stream) {
  if (!d_flag || !d_timeout) return fail(PS_EARG, "null argument");
  const unsigned long long lim = (unsigned long long)(std::max(0.0, timeout_s) * 1e9);
  k_flag_wait<<<1, 1, 0, (cudaStream_t)stream>>>((const unsigned long long*)d_flag,
                                                 (unsigned long long)value, (int*)d_timeout, lim);
  CK(cudaGetLastError());
  return PS_OK;
}

}  // extern "C"
