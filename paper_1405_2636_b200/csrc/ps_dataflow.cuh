// Device-resident task runtime: the whole numeric factorization as ONE
// persistent kernel.
//
// The reference runs its task DAG (taskgraph.py:79-110: factor F(p), update
// U(p->q), F(p) -> U(p->q) -> F(q)) on CPU worker threads with dependency
// counters and a destination-panel guard (runtime.py:189-304).  Here the
// same DAG - refined into tiles - is executed on the GPU:
//
//   * the host orders every task into one list that is a topological order
//     (a list-scheduling simulation with critical-path priorities, see
//     ps_b200.cu: build_dataflow), so tasks come off the list roughly when
//     they become ready;
//   * every dependency is "counter X has reached t"; a finishing task bumps
//     its counters and, for each waiter whose threshold the new value hits,
//     decrements the waiter's unmet-dependency count - the last one pushes
//     the waiter onto a device ready queue (high priority: factor tasks);
//   * persistent CTAs pop READY tasks only, so no CTA ever blocks on an
//     unfinished dependency and no ordering of the list can deadlock.
//
// Scatter conflicts (two updates into the same entries of a destination) are
// ordered by the per-destination counter: update units into q are colored by
// destination-column overlap and a unit of color k waits until every task of
// colors < k into q has finished - atomics-free, deterministic.
#pragma once
#include "ps_kernels.cuh"
#include "ps_diag.cuh"

namespace ps {

enum DType : int {
  DT_W1 = 0,      // batch of width-1 panels (FItem: p = first in w1 list, nb = count)
  DT_SMALL = 1,   // width 2..32 panel: diagonal (+ first rows) or extra TRSM rows (FItem)
  DT_DIAG = 2,    // wide panel, 64-column step: diagonal factor + inverse (FItem)
  DT_TRSM = 3,    // wide panel, 64-row tile of the step's TRSM (FItem)
  DT_UPD = 4,     // 64x64 DMMA update tile (UTile; couple -1 = intra-panel trailing)
  DT_GATHER = 5,  // narrow-source gather into one 64x64 destination region (NItem)
  DT_NTYPES = 6
};

struct DTask {
  int type;
  int idx;        // into the type's payload array
  int dep0;       // deps [dep0, dep0 + ndep) of the dep array: (counter, target)
  int ndep;
  int sig0;       // signals [sig0, sig0 + nsig) of the signal array:
  int nsig;       //   counters incremented on completion
  int pad0, pad1;
};

// narrow-source segment of a gather: source rows [s0, s0+ni) x facing rows
// [f0, f0+nj) of one couple landing in the region; their region rows / columns
// are the bytes gmap[gm .. gm+ni) / gmap[gm+ni .. gm+ni+nj) (host-built)
struct GSeg {
  i64 src;          // slab offset of the source panel
  int lds, kn;      // leading dimension, width
  int s0, ni;
  int f0, nj;
  int gm;           // offset of the maps in gmap (bytes)
  int op0;          // operand offset in the task's shared buffer (doubles)
  int mp0;          // map offset in the task's shared map buffer (bytes)
  int raw;          // 1: width-1 source read before its factor task: the
                    //    contribution a_i a_j / pivot (= l_i d l_j, kernels.py:283-309)
};
struct DfArgs {
  const DTask* tasks;
  int ntasks;
  int pad;
  const int2* deps;
  unsigned* ctr;        // counters (zeroed per factorization)
  int* qstate;          // [0] head (tickets taken) [1] tail (pushed) [2] queue task count
  int* qhi;             // FIFO ready queue (slots -1 until pushed)
  int* qlo;             // unused
  int* remaining;       // unmet dependencies per task
  const i64* wl_ptr;    // per counter: waiters [wl_ptr[X], wl_ptr[X+1]) sorted by threshold
  const unsigned* wl_thr;
  const int* wl_task;
  const unsigned char* prio;  // 1: high-priority queue
  const int* prio_val;        // critical-path priority of each task
  const UTile* tiles;
  const FItem* fitems;
  const NItem* nitems;
  const GSeg* gsegs;
  const unsigned char* gmap;
  const int* w1;
  unsigned long long* trace;  // optional: per task {ticket, deps met, body done, signalled} ns + smid|type
  unsigned long long* phase;  // optional: per task 4 intra-body timestamps (gathers)
  const int* sigs;
};

constexpr int DF_THREADS = 128;
constexpr int DF_READY = 256;  // newly ready tasks collected per release
constexpr int W1_PER_WARP = 8;   // width-1 panels per warp in a DT_W1 batch

struct DiagSmem {
  double D[FNB][FNB + 1];
  double rdiag[FNB];
  DiagWork W;
  int s_fail;
  double s_fpiv;
};
struct SmallSmem {
  double D[SNB][SNB + 1];
  double rdiag[SNB];
  int s_fail;
  double s_fpiv;
};
constexpr int GMAX = 64;            // segments per gather task
constexpr int GATHER_OPS = 3072;    // operand doubles per gather task (after GatherSmem)
constexpr int GATHER_MAPB = 8192;   // map bytes per gather task
template <int GR, int GM, int MAPB>
struct GatherSmemT {
  static constexpr int ROWS = GR;
  double T[TN][GR + 1];
  GSeg seg[GM];
  int clist[TN];
  int ncl;
  alignas(16) unsigned char maps[MAPB];
};
using GatherSmem = GatherSmemT<TM, GMAX, GATHER_MAPB>;
// level schedule: 32-row regions and small chunks -> ~28 KB, 7-8 CTAs / SM
constexpr int LG_ROWS = 32, LG_GMAX = 32, LG_OPS = 1024, LG_MAPB = 2048;
using LevelGatherSmem = GatherSmemT<LG_ROWS, LG_GMAX, LG_MAPB>;
constexpr size_t LG_SMEM = sizeof(LevelGatherSmem) + LG_OPS * sizeof(double);

constexpr size_t cmax(size_t a, size_t b) { return a > b ? a : b; }
constexpr size_t DF_SMEM =
    cmax(cmax(sizeof(UpdSmem), sizeof(DiagSmem)),
         cmax(sizeof(SmallSmem), sizeof(GatherSmem) + GATHER_OPS * sizeof(double)));

__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;\n" ::: "memory"); }

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned s;
  asm volatile("mov.u32 %0, %smid;" : "=r"(s));
  return s;
}


// DMMA mainloop for the persistent kernel: operands are read with L2-only
// loads (ld.global.cg) staged through registers into a 2-stage shared
// buffer.  No L1 allocation: a cache line may also hold entries another CTA
// is still writing (false sharing across row tiles), and an in-flight L1
// fill could outlive the consumer's acquire-time invalidation.
template <class Pro>
__device__ __forceinline__ void df_mainloop(UpdSmem& sm, const Operands& O, double acc[4][4][2],
                                            int tid, Pro prologue) {
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  constexpr int PER = (KC * TM) / DF_THREADS;  // 8 values of A and of B per thread
  const int r = tid & (TM - 1), kq = tid >> 6;
  const bool va_r = r < O.ani, vb_r = r < O.bnj;
  const double* pa = O.A + O.ai0 + (va_r ? r : 0);
  const double* pb = O.B + O.bj0 + (vb_r ? r : 0);
  double ra[PER], rb[PER], rd = 1.0;
  auto gload = [&](int chunk) {
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      const int k = chunk * KC + kq + 2 * e;
      const bool kv = k < O.kn;
      ra[e] = (kv && va_r) ? __ldcg(pa + (i64)k * O.lda) : 0.0;
      rb[e] = (kv && vb_r) ? __ldcg(pb + (i64)k * O.ldb) : 0.0;
    }
    if (O.dptr && tid < KC) {
      const int k = chunk * KC + tid;
      rd = k < O.kn ? __ldcg(O.dptr + (i64)k * O.dstride) : 0.0;
    }
  };
  auto sstore = [&](int st) {
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      sm.A[st][kq + 2 * e][r] = ra[e];
      sm.B[st][kq + 2 * e][r] = rb[e];
    }
    if (O.dptr && tid < KC) sm.D[st][tid] = rd;
  };
  const int nch = (O.kn + KC - 1) / KC;
  gload(0);
  prologue();  // overlaps the first operand fetch (may contain barriers)
  sstore(0);
  __syncthreads();
  for (int c = 0; c < nch; ++c) {
    const int st = c & 1;
    if (c + 1 < nch) gload(c + 1);
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
    if (c + 1 < nch) sstore(st ^ 1);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// task bodies (CTA of DF_THREADS threads).  Store data is read with plain
// (coherent) loads: it may have been written earlier in this same launch.

// 64x64 DMMA update tile + direct scatter (kernels.py:128-136, 249-281)
__device__ __forceinline__ void df_update(UpdSmem& sm, const UTile& T, double* store, bool ldlt,
                                          const PanelDev& P, const i64* run_ptr,
                                          const int* run_src, const int* run_dst, int tid) {
  const double* src = store + P.off[T.src];
  const i64 lds = P.nrows[T.src];
  const double* colk = src + (i64)T.k0 * lds;
  Operands O{colk, lds, T.i0, T.ni, colk, lds, T.j0, T.nj, T.kn,
             ldlt ? colk + T.k0 : nullptr, lds + 1};
  double acc[4][4][2];
  df_mainloop(sm, O, acc, tid, [&]() {
    maps_load(sm, T.couple, T.ri, T.rj, run_ptr, run_src, run_dst, tid);
    __syncthreads();
    maps_search(sm, T.couple, T.i0, T.ni, T.j0, T.nj, tid);
  });
  double(*Cs)[CLD] = stage_acc(sm, acc, tid);
  double* dst = store + P.off[T.dst];
  const i64 ldd = P.nrows[T.dst];
  const int row = tid & (TM - 1);
  const int dr = sm.rmap[row];
  const int gi = T.i0 + row;
  if (row < T.ni) {
    constexpr int CSTEP = DF_THREADS / TM;
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
}

// narrow sources gathered into one destination region (kernels.py:283-309
// for width 1; the same arithmetic for widths <= SMALL_W).  Descriptors, then
// ALL operands, maps and the region's touched columns are fetched with
// independent loads (two memory latencies per task), the segments are applied
// in order to the region in shared memory (all threads on each segment's
// entries), and only the touched columns are written back: other columns of
// the region may be updated concurrently by other tasks.  load_t / store_t:
// a region split into several chunks processed by one CTA keeps the region
// in shared memory between chunks (level schedule).
template <class GS>
__device__ __forceinline__ void df_gather(GS& g, double* ops, const NItem& it,
                                          const GSeg* segs, const unsigned char* gmap,
                                          double* store, bool ldlt, const PanelDev& P, int tid,
                                          unsigned long long* ph = nullptr, bool load_t = true,
                                          bool store_t = true) {
  double* dst = store + P.off[it.q] + it.r0 + (i64)it.c0 * P.nrows[it.q];
  const i64 ldd = P.nrows[it.q];
  const int nseg = it.nseg, nr = it.nr;
  if (tid < nseg) g.seg[tid] = segs[it.seg0 + tid];
  if (tid < 32) {
    const unsigned long long cm = it.cmask ? it.cmask : ~0ULL;
    const unsigned lo = (unsigned)cm, hi = (unsigned)(cm >> 32);
    const unsigned lane_lt = (1u << tid) - 1u;
    const int nlo = __popc(lo);
    if ((lo >> tid) & 1) g.clist[__popc(lo & lane_lt)] = tid;
    if ((hi >> tid) & 1) g.clist[nlo + __popc(hi & lane_lt)] = 32 + tid;
    if (tid == 0) g.ncl = min(nlo + __popc(hi), it.nc);
  }
  __syncthreads();
  if (ph && tid == 0) ph[0] = globaltimer();
  const int ncl = g.ncl;
  const GSeg& last = g.seg[nseg - 1];
  const int nops = last.op0 + last.kn * (last.ni + last.nj) + last.kn;
  const int nmap = last.mp0 + last.ni + last.nj;
  // region columns (touched only), 8 loads in flight per thread
  const int ntv = nr * ncl;
  if (load_t) {
    for (int b = 0; b < ntv; b += 8 * DF_THREADS) {
      double v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int idx = b + tid + e * DF_THREADS;
        if (idx < ntv) {
          const int c = g.clist[idx / nr], r = idx % nr;
          v[e] = __ldcg(dst + (i64)c * ldd + r);
        }
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int idx = b + tid + e * DF_THREADS;
        if (idx < ntv) g.T[g.clist[idx / nr]][idx % nr] = v[e];
      }
    }
  }
  // operands: segment s holds A (kn x ni), B (kn x nj) interleaved per k, then d
  for (int b = 0; b < nops; b += 8 * DF_THREADS) {
    double v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int idx = b + tid + e * DF_THREADS;
      if (idx < nops) {
        int lo = 0, hi = nseg - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (g.seg[mid].op0 <= idx) lo = mid;
          else hi = mid - 1;
        }
        const GSeg& sg = g.seg[lo];
        const int span = sg.ni + sg.nj;
        const int o = idx - sg.op0;
        const double* src = store + sg.src;
        if (o < sg.kn * span) {
          const int k = o / span, rr = o - k * span;
          const int row = rr < sg.ni ? sg.s0 + rr : sg.f0 + (rr - sg.ni);
          v[e] = __ldcg(src + (i64)k * sg.lds + row);
        } else {  // d_k (LDLt) / 1, or 1 / pivot for an unfactored width-1 source
          const int k = o - sg.kn * span;
          if (sg.raw) v[e] = 1.0 / __ldcg(src);
          else v[e] = ldlt ? __ldcg(src + (i64)k * sg.lds + k) : 1.0;
        }
      }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int idx = b + tid + e * DF_THREADS;
      if (idx < nops) ops[idx] = v[e];
    }
  }
  {  // maps: one contiguous 16-byte-aligned area per gather
    const uint4* gm4 = reinterpret_cast<const uint4*>(gmap + g.seg[0].gm);
    uint4* sm4 = reinterpret_cast<uint4*>(g.maps);
    for (int idx = tid; idx < (nmap + 15) / 16; idx += DF_THREADS) sm4[idx] = __ldcg(gm4 + idx);
  }
  __syncthreads();
  if (ph && tid == 0) ph[1] = globaltimer();
  for (int sidx = 0; sidx < nseg; ++sidx) {
    const GSeg& sg = g.seg[sidx];
    const int ni = sg.ni, nj = sg.nj, kn = sg.kn, span = ni + nj;
    const double* o = ops + sg.op0;
    const double* dk = o + kn * span;
    const unsigned char* rm = g.maps + sg.mp0;
    const unsigned char* cm = rm + ni;
    const int tot = ni * nj;
    for (int e = tid; e < tot; e += DF_THREADS) {
      const int j = e / ni, i = e - j * ni;
      if (sg.s0 + i < sg.f0 + j) continue;
      double a = 0.0;
      for (int k = 0; k < kn; ++k) a += o[k * span + i] * (o[k * span + ni + j] * dk[k]);
      g.T[cm[j]][rm[i]] -= a;
    }
    __syncthreads();
  }
  if (ph && tid == 0) ph[2] = ph[3] = globaltimer();
  if (store_t) {
    for (int b = 0; b < ntv; b += DF_THREADS) {
      const int idx = b + tid;
      if (idx < ntv) {
        const int c = g.clist[idx / nr], r = idx % nr;
        __stcg(dst + (i64)c * ldd + r, g.T[c][r]);
      }
    }
  }
}

// level schedule: one CTA per destination region, its chunks in order with
// the region resident in shared memory (regions of one launch are disjoint)
__global__ void __launch_bounds__(DF_THREADS, 7)
k_gather_level(const int* __restrict__ region_ptr, const NItem* __restrict__ items,
               const GSeg* __restrict__ segs, const unsigned char* __restrict__ gmap,
               const DevArgs* __restrict__ args, PanelDev P) {
  pdl_wait();  // programmatic dependent launch: wait for the previous grid
  extern __shared__ __align__(16) unsigned char smem_raw[];
  LevelGatherSmem& g = *reinterpret_cast<LevelGatherSmem*>(smem_raw);
  double* ops = reinterpret_cast<double*>(smem_raw + sizeof(LevelGatherSmem));
  const int c0 = region_ptr[blockIdx.x], c1 = region_ptr[blockIdx.x + 1];
  for (int c = c0; c < c1; ++c) {
    df_gather(g, ops, items[c], segs, gmap, args->store, args->form == FORM_LDLT, P, threadIdx.x,
              nullptr, c == c0, c == c1 - 1);
    __syncthreads();
  }
}

// width-1 panels, warp per panel (kernels.py:216-221, 232-239)
__device__ __forceinline__ void df_w1(const FItem& it, const int* w1, double* store, bool ldlt,
                                      double thr, const PanelDev& P, i64* fail_col,
                                      double* fail_piv, int tid) {
  const int lane = tid & 31, warp = tid >> 5;
  for (int k = warp; k < it.nb; k += DF_THREADS / 32) {
    const int p = w1[it.p + k];
    double* a = store + P.off[p];
    const int nr = P.nrows[p];
    const double piv = __ldcg(a);
    const bool bad = ldlt ? (fabs(piv) <= thr) : (piv <= thr);
    const double dv = ldlt ? piv : sqrt(piv);
    const double inv = 1.0 / dv;
    for (int r = 1 + lane; r < nr; r += 32) a[r] = __ldcg(a + r) * inv;
    if (lane == 0) {
      if (!ldlt) a[0] = dv;
      if (bad && fail_col[p] == NO_FAIL) {
        fail_col[p] = P.fc[p];
        fail_piv[p] = piv;
      }
    }
  }
}

// width 2..SNB: diagonal factor in shared memory + thread-per-row TRSM
// (kernels.py:208-247); it.diag = 0: TRSM rows only (diagonal already final)
__device__ __noinline__ void df_small(SmallSmem& s, const FItem& it, double* store, bool ldlt,
                                         double thr, const PanelDev& P, i64* fail_col,
                                         double* fail_piv, int tid) {
  double* base = store + P.off[it.p];
  const i64 ld = P.nrows[it.p];
  const int nb = it.nb, c0 = it.c0;
  for (int idx = tid; idx < nb * nb; idx += DF_THREADS) {
    const int c = idx / nb, r = idx % nb;
    s.D[c][r] = r >= c ? __ldcg(base + (i64)(c0 + c) * ld + c0 + r) : 0.0;
  }
  if (tid == 0) s.s_fail = -1;
  __syncthreads();
  if (it.diag) {
    factor_diag_smem<SNB, DF_THREADS>(s.D, s.rdiag, nb, ldlt, thr, &s.s_fail, &s.s_fpiv, tid);
    for (int idx = tid; idx < nb * nb; idx += DF_THREADS) {
      const int c = idx / nb, r = idx % nb;
      if (r >= c) base[(i64)(c0 + c) * ld + c0 + r] = s.D[c][r];
    }
    if (tid == 0 && s.s_fail >= 0 && fail_col[it.p] == NO_FAIL) {
      fail_col[it.p] = P.fc[it.p] + c0 + s.s_fail;
      fail_piv[it.p] = s.s_fpiv;
    }
  } else {
    for (int j = tid; j < nb; j += DF_THREADS) s.rdiag[j] = 1.0 / s.D[j][j];
  }
  if (it.nr == 0) return;
  __syncthreads();
  for (int idx = tid; idx < nb * nb; idx += DF_THREADS) {
    const int j = idx / nb, k = idx % nb;
    if (k > j) s.D[k][j] = ldlt ? s.D[j][k] * s.D[j][j] : s.D[j][k];
  }
  __syncthreads();
  if (tid < it.nr) {
    double* rowp = base + it.r0 + tid;
    double x[SNB];
#pragma unroll
    for (int k = 0; k < SNB; ++k)
      if (k < nb) x[k] = __ldcg(rowp + (i64)(c0 + k) * ld);
#pragma unroll
    for (int j = 0; j < SNB; ++j) {
      if (j < nb) {
        const double xj = x[j] * s.rdiag[j];
        x[j] = xj;
#pragma unroll
        for (int k = j + 1; k < SNB; ++k)
          if (k < nb) x[k] -= xj * s.D[k][j];
      }
    }
#pragma unroll
    for (int k = 0; k < SNB; ++k)
      if (k < nb) rowp[(i64)(c0 + k) * ld] = x[k];
  }
}

// wide panel step: diagonal factor + scaled inverse G into scratch slot it.g
template <int NT = DF_THREADS>
__device__ __forceinline__ void df_diag(DiagSmem& s, const FItem& it, double* store,
                                        double* scratch, bool ldlt, double thr, const PanelDev& P,
                                        i64* fail_col, double* fail_piv, int tid, int ablate = 0) {
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
  if (!(ablate & 1))
    factor_block_inv<0, NT>(s.D, s.rdiag, s.W, nb, ldlt, thr, &s.s_fail, &s.s_fpiv, tid);
  store_block_inv<NT>(s.D, s.rdiag, s.W, nb, ldlt, base, ld, c0, scratch + (i64)it.g * FNB * FNB, tid);
  if (tid == 0 && s.s_fail >= 0 && fail_col[it.p] == NO_FAIL) {
    fail_col[it.p] = P.fc[it.p] + c0 + s.s_fail;
    fail_piv[it.p] = s.s_fpiv;
  }
}


// the level schedule's launch of the same body (wide panels, one 64-column block)
#ifndef DIAGB_T
#define DIAGB_T 512  // diagonal-block CTA threads (DMMA phases over 16 warps; 60^3: 128 -> 512 = 21.9 -> 21.3 ms)
#endif
__global__ void __launch_bounds__(DIAGB_T)
k_factor_diag_blk(const FItem* __restrict__ items, const DevArgs* __restrict__ args, PanelDev P,
                  i64* __restrict__ fail_col, double* __restrict__ fail_piv) {
  pdl_wait();  // programmatic dependent launch: wait for the previous grid
  pdl_trigger();  // (not persistent: every CTA of the grid has started)
  __shared__ DiagSmem s;
  df_diag<DIAGB_T>(s, items[blockIdx.x], args->store, args->scratch, args->form == FORM_LDLT,
                   args->thr, P, fail_col, fail_piv, threadIdx.x, args->pad);
}

// wide panel step: 64-row TRSM tile X = B G^T (DMMA), in place
__device__ __forceinline__ void df_trsm(UpdSmem& sm, const FItem& it, double* store,
                                        const double* scratch, const PanelDev& P, int tid) {
  double* base = store + P.off[it.p];
  const i64 ld = P.nrows[it.p];
  const double* G = scratch + (i64)it.g * FNB * FNB;
  double* colc = base + (i64)it.c0 * ld;
  Operands O{colc, ld, it.r0, it.nr, G, FNB, 0, it.nb, it.nb, nullptr, 0};
  double acc[4][4][2];
  df_mainloop(sm, O, acc, tid, []() {});
  double(*Cs)[CLD] = stage_acc(sm, acc, tid);
  const int row = tid & (TM - 1);
  if (row < it.nr) {
    for (int col = tid >> 6; col < it.nb; col += DF_THREADS / TM)
      colc[(i64)col * ld + it.r0 + row] = Cs[col][row];
  }
}


// ---------------------------------------------------------------------------

// ---------------------------------------------------------------------------
// One 64-column step of every wide panel of a level in ONE launch (level
// schedule): items in order [diagonals][TRSM row tiles][trailing tiles];
// persistent CTAs take them in list order; a TRSM tile waits for its
// diagonal (stepctr[2 s] >= 1), a trailing tile for all TRSM tiles of its
// step (stepctr[2 s + 1] >= ntrsm).  Earlier items never wait on later ones:
// no deadlock.  Replaces three dependent launches per step.
struct WItem {
  int kind;   // 0 diagonal (FItem), 1 TRSM tile (FItem), 2 trailing tile (UTile)
  int idx;    // item index in the FItem / UTile array
  int ctr;    // step counter pair base (2 per panel step)
  int need;   // trailing: TRSM tiles of the step to wait for
};

__global__ void __launch_bounds__(DF_THREADS, 3)
k_wide_step(const WItem* __restrict__ items, int nitems, int* __restrict__ work_ctr,
            unsigned* __restrict__ stepctr, const FItem* __restrict__ fitems,
            const UTile* __restrict__ tiles, const DevArgs* __restrict__ args, PanelDev P,
            i64* __restrict__ fail_col, double* __restrict__ fail_piv) {
  pdl_wait();  // programmatic dependent launch: wait for the previous grid
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_item;
  const int tid = threadIdx.x;
  double* store = args->store;
  const bool ldlt = args->form == FORM_LDLT;
  while (true) {
    if (tid == 0) s_item = atomicAdd(work_ctr, 1);
    __syncthreads();
    const int t = s_item;
    if (t >= nitems) break;
    const WItem W = items[t];
    if (W.kind == 0) {
      df_diag(*reinterpret_cast<DiagSmem*>(smem_raw), fitems[W.idx], store, args->scratch, ldlt,
              args->thr, P, fail_col, fail_piv, tid);
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        atomicAdd(&stepctr[W.ctr], 1u);
      }
      continue;
    }
    if (tid == 0) {
      const unsigned* c = &stepctr[W.kind == 1 ? W.ctr : W.ctr + 1];
      const unsigned need = W.kind == 1 ? 1u : (unsigned)W.need;
      while (ld_relaxed(c) < need) __nanosleep(64);
      (void)ld_acquire(c);  // acquire + L1 invalidation: cp.async.ca below reads fresh lines
    }
    __syncthreads();
    UpdSmem& sm = *reinterpret_cast<UpdSmem*>(smem_raw);
    if (W.kind == 1) {
      // TRSM tile X = B G^T (cp.async pipeline; G written by this launch's diagonal item)
      const FItem it = fitems[W.idx];
      double* colc = store + P.off[it.p] + (i64)it.c0 * P.nrows[it.p];
      const i64 ld = P.nrows[it.p];
      const double* G = args->scratch + (i64)it.g * FNB * FNB;
      Operands O{colc, ld, it.r0, it.nr, G, FNB, 0, it.nb, it.nb, nullptr, 0};
      double acc[4][4][2];
      dmma_mainloop(sm, O, acc, tid);
      double(*Cs)[CLD] = stage_acc(sm, acc, tid);
      const int row = tid & (TM - 1);
      if (row < it.nr)
        for (int col = tid >> 6; col < it.nb; col += DF_THREADS / TM)
          colc[(i64)col * ld + it.r0 + row] = Cs[col][row];
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        atomicAdd(&stepctr[W.ctr + 1], 1u);
      }
      continue;
    }
    // trailing tile: identity maps (intra-panel), no ordering
    const UTile T = tiles[W.idx];
    const double* src = store + P.off[T.src];
    const i64 lds = P.nrows[T.src];
    const double* colk = src + (i64)T.k0 * lds;
    Operands O{colk, lds, T.i0, T.ni, colk, lds, T.j0, T.nj, T.kn,
               ldlt ? colk + T.k0 : nullptr, lds + 1};
    double acc[4][4][2];
    dmma_mainloop(sm, O, acc, tid);
    double(*Cs)[CLD] = stage_acc(sm, acc, tid);
    double* dst = store + P.off[T.dst];
    const i64 ldd = P.nrows[T.dst];
    const int row = tid & (TM - 1);
    const int gi = T.i0 + row;
    if (row < T.ni) {
      constexpr int CSTEP = DF_THREADS / TM;
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
    __syncthreads();
  }
}


// push a ready task onto the FIFO ready queue
__device__ __forceinline__ void df_push(const DfArgs& A, int w) {
  __threadfence();  // the releases this thread observed (atomicSub chain) before the push
  const int pos = atomicAdd(&A.qstate[1], 1);
  asm volatile("st.relaxed.gpu.global.s32 [%0], %1;\n" ::"l"(A.qhi + pos), "r"(w) : "memory");
}

// pop: take the next queue ticket (always succeeds) and wait until that slot
// is filled; -1 once every task has been handed out.  qstate[2] = tasks that
// pass through the queue (ntasks minus the direct hand-offs, which decrement
// it).  While a slot below it is unfilled some task is running (else every
// pushed task has completed and the DAG has a ready task left), so every
// ticket below the final count is served and the others exit.  Thread 0 only.
__device__ __forceinline__ int df_pop(const DfArgs& A) {
  const int h = atomicAdd(&A.qstate[0], 1);
  volatile int* lim = A.qstate + 2;  // tasks that go through the queue (shrinks by hand-offs)
  if (h >= *lim) return -1;
  int v;
  if ((v = *(volatile int*)(A.qhi + h)) < 0) {
    do {
      __nanosleep(32);
      if (h >= *lim) return -1;
    } while ((v = *(volatile int*)(A.qhi + h)) < 0);
  }
  return v;
}

// Persistent scheduler: pop a READY task, run it, then signal its counters
// and release the waiters whose threshold the new counter value reaches
// (decrementing their unmet-dependency count; the last one pushes the task).
// No CTA ever waits on a task that is not ready, so the GPU only idles when
// no task is ready (the dependency graph's own critical path).
__global__ void __launch_bounds__(DF_THREADS, 3)
k_dataflow(DfArgs A, const DevArgs* __restrict__ args, PanelDev P, const i64* __restrict__ run_ptr,
           const int* __restrict__ run_src, const int* __restrict__ run_dst,
           i64* __restrict__ fail_col, double* __restrict__ fail_piv) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_task;
  __shared__ unsigned s_val[8];
  __shared__ int s_nready;
  __shared__ unsigned long long s_best;
  __shared__ int s_ready[DF_READY];
  const int tid = threadIdx.x;
  double* store = args->store;
  double* scratch = args->scratch;
  const bool ldlt = args->form == FORM_LDLT;
  const double thr = args->thr;
  __shared__ int s_keep;
  if (tid == 0) s_keep = -1;
  while (true) {
    unsigned long long tw = 0;
    if (tid == 0) {
      if (A.trace) tw = globaltimer();
      // a high-priority task this CTA just made ready runs next, directly
      s_task = s_keep >= 0 ? s_keep : df_pop(A);
      s_keep = -1;
      fence_acq_rel();
    }
    __syncthreads();
    const int t = s_task;
    if (t < 0) break;
    const DTask T = A.tasks[t];
    unsigned long long t0 = 0;
    if (A.trace && tid == 0) t0 = globaltimer();
    switch (T.type) {
      case DT_UPD:
        df_update(*reinterpret_cast<UpdSmem*>(smem_raw), A.tiles[T.idx], store, ldlt, P, run_ptr,
                  run_src, run_dst, tid);
        break;
      case DT_SMALL:
        df_small(*reinterpret_cast<SmallSmem*>(smem_raw), A.fitems[T.idx], store, ldlt, thr, P,
                 fail_col, fail_piv, tid);
        break;
      case DT_DIAG:
        df_diag(*reinterpret_cast<DiagSmem*>(smem_raw), A.fitems[T.idx], store, scratch, ldlt, thr,
                P, fail_col, fail_piv, tid);
        break;
      case DT_TRSM:
        df_trsm(*reinterpret_cast<UpdSmem*>(smem_raw), A.fitems[T.idx], store, scratch, P, tid);
        break;
      case DT_GATHER:
        df_gather(*reinterpret_cast<GatherSmem*>(smem_raw),
                  reinterpret_cast<double*>(smem_raw + sizeof(GatherSmem)), A.nitems[T.idx], A.gsegs,
                  A.gmap, store, ldlt, P, tid, A.phase ? A.phase + 4 * (size_t)t : nullptr);
        break;
      case DT_W1:
        df_w1(A.fitems[T.idx], A.w1, store, ldlt, thr, P, fail_col, fail_piv, tid);
        break;
      default:
        break;
    }
    unsigned long long tb = 0;
    if (A.trace && tid == 0) tb = globaltimer();
    __syncthreads();
    // release: publish the task's writes, bump its counters (chunks of 8)
    if (tid == 0) {
      __threadfence();
      s_nready = 0;
      s_best = 0ULL;
    }
    for (int k0 = 0; k0 < T.nsig; k0 += 8) {
      if (tid == 0)
        for (int k = k0; k < T.nsig && k < k0 + 8; ++k)
          s_val[k - k0] = atomicAdd(&A.ctr[A.sigs[T.sig0 + k]], 1u) + 1u;
      __syncthreads();
      // waiters of threshold == new value: one less unmet dependency each;
      // the newly ready ones are collected (overflow: pushed at once)
      for (int k = k0; k < T.nsig && k < k0 + 8; ++k) {
        const int X = A.sigs[T.sig0 + k];
        const unsigned v = s_val[k - k0];
        i64 lo = A.wl_ptr[X], hi = A.wl_ptr[X + 1];
        while (lo < hi) {  // first waiter with threshold >= v
          const i64 mid = (lo + hi) >> 1;
          if (A.wl_thr[mid] < v) lo = mid + 1;
          else hi = mid;
        }
        for (i64 w = lo + tid; w < A.wl_ptr[X + 1] && A.wl_thr[w] == v; w += DF_THREADS) {
          const int task = A.wl_task[w];
          if (atomicSub(&A.remaining[task], 1) == 1) {
            const int slot = atomicAdd(&s_nready, 1);
            if (slot < DF_READY) {
              s_ready[slot] = task;
              atomicMax(&s_best, ((unsigned long long)(unsigned)A.prio_val[task] << 32) |
                                     (unsigned)task);
            } else {
              df_push(A, task);
            }
          }
        }
      }
      __syncthreads();
    }
    __syncthreads();  // s_nready / s_best final (also when the task has no signals)
    // the most critical newly ready task runs next on this CTA; the others
    // go to the queue
    {
      const int nr = min(s_nready, DF_READY);
      const int keep = nr ? (int)(unsigned)(s_best & 0xffffffffULL) : -1;
      for (int k = tid; k < nr; k += DF_THREADS)
        if (s_ready[k] != keep) df_push(A, s_ready[k]);
      if (tid == 0) {
        s_keep = keep;
        if (keep >= 0) atomicSub(&A.qstate[2], 1);
      }
    }
    if (A.trace && tid == 0) {
      unsigned long long* tr = A.trace + 5 * (size_t)t;
      tr[0] = tw;
      tr[1] = t0;
      tr[2] = tb;
      tr[3] = globaltimer();
      tr[4] = ((unsigned long long)smid() << 8) | (unsigned)T.type;
    }
  }
}

}  // namespace ps
