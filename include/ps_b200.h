/*
 * ps_b200.h - C ABI of the B200 (sm_100a) numeric factorization engine for
 * the supernodal solver of arXiv 1405.2636 (reference package `panelsolve`).
 *
 * The reference has no native code: its numeric path is the Python call
 *     pipeline.factorize(analysis, scheduler, threads, kernel, ...)
 *                                      (pkg/src/panelsolve/pipeline.py:87-117)
 * which runs FactorKernels.run_factor / run_update task by task
 *                                      (pkg/src/panelsolve/kernels.py:185-315)
 * under a CPU task runtime            (pkg/src/panelsolve/runtime.py:143-304).
 * These entry points are what a ctypes binding of that path calls
 * (paper_1405_2636_b200/_abi.py).  Plain pointers and sizes
 * only; device buffers are passed as raw device pointers (the caller - e.g.
 * PyTorch - owns them); streams as `void*` (cudaStream_t).
 *
 * Status codes mirror the reference CLI's exit codes (cli.py:282-298):
 *   PS_OK (0), PS_NUMERIC (2: pivot failure -> NotPositiveDefiniteError /
 *   SingularPivotError, errors.py:14-29, with the global permuted column as
 *   in kernels.py:217-244), PS_STRUCTURAL (4: StructuralError, errors.py:35),
 *   PS_EARG (-1: bad argument), PS_ECUDA (-2: CUDA error; see ps_last_error).
 */
#ifndef PS_B200_H
#define PS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PS_OK 0
#define PS_NUMERIC 2
#define PS_STRUCTURAL 4
#define PS_EARG (-1)
#define PS_ECUDA (-2)

#define PS_FORM_LLT 0
#define PS_FORM_LDLT 1
#define PS_FORM_LU 2         /* no reference counterpart: PAPER.md:321-331 (U slab after L) */
#define PS_FORM_COMPLEX 16   /* flag: complex128 (interleaved) values, any form */
#define PS_FORM_GENERIC 32   /* flag: real LLt / LDLt on the scalar-generic kernels (tests) */

typedef struct ps_plan ps_plan;

/* Block symbolic structure (reference SymbolStructure/Panel/Block,
 * symbolic.py:229-315), flattened.  Panel p owns columns
 * [starts[p], starts[p+1]); its off-diagonal rows are
 * rows[rowptr[p]:rowptr[p+1]] (ascending); its blocks are
 * blkptr[p]..blkptr[p+1] with Block(fr, lr, facing, loc). */
typedef struct ps_symbol_desc {
  int64_t n;
  int64_t npanels;
  const int64_t* starts;     /* [npanels + 1] */
  const int64_t* rowptr;     /* [npanels + 1] */
  const int64_t* rows;       /* [rowptr[npanels]] */
  const int64_t* blkptr;     /* [npanels + 1] */
  const int64_t* blk_fr;     /* [nblocks] */
  const int64_t* blk_lr;
  const int64_t* blk_facing;
  const int64_t* blk_loc;
} ps_symbol_desc;

typedef struct ps_plan_info {
  int64_t store_elems;      /* doubles in the panel slab (PanelStore layout) */
  int64_t npanels;
  int64_t ncouples;         /* (source, destination) update tasks */
  int64_t nruns;            /* entries of the block-row index map */
  int64_t update_tiles;     /* DMMA tiles of inter-panel updates */
  int64_t trailing_tiles;   /* DMMA tiles of intra-panel (wide panel) updates */
  int64_t factor_items;     /* diagonal-factor + TRSM CTAs */
  int32_t nlevels;          /* panel-tree height (batch steps) */
  int32_t nlaunches;        /* kernel launches per factorization */
  int64_t device_bytes;     /* plan-owned device memory */
} ps_plan_info;

/* Build the level schedule, block-row index map and tile lists for one
 * symbol and upload them to `device`.  Replaces the reference's
 * FactorKernels.__init__ (kernels.py:192-203), build_taskgraph
 * (taskgraph.py:79-110) and the runtime's scheduling (runtime.py:48-90). */
int ps_plan_create(const ps_symbol_desc* sym, int device, ps_plan** out);
void ps_plan_destroy(ps_plan* plan);
int ps_plan_get_info(const ps_plan* plan, ps_plan_info* info);

/* Element offset of each panel in the slab (npanels + 1 values); panel p
 * is F-order nrows x width at offsets[p], like PanelStore.data[p]
 * (symbolic.py:318-335). */
int ps_plan_offsets(const ps_plan* plan, int64_t* offsets);

/* Device assembly: zero the slab, then slab[pos[k]] = vals[k]
 * (reference allocate_panels, symbolic.py:338-350). */
int ps_assemble(ps_plan* plan, double* d_store, const int64_t* d_pos,
                const double* d_vals, int64_t nvals, void* stream);

/* ps_assemble for any form code: zero the (form_slabs x store_elems)
 * elements of d_store (LU: L slab then U slab; complex: complex128), then
 * d_store[pos[k]] = vals[k] (pos < 0 skipped). */
int ps_assemble_form(ps_plan* plan, void* d_store, const int64_t* d_pos, const void* d_vals,
                     int64_t nvals, int form, void* stream);

/* Whole numeric factorization, enqueued on `stream` (asynchronous; replays
 * a CUDA graph of the per-level launches).  Replaces pipeline.factorize's
 * timed region (pipeline.py:97-116).  Pivot failures are recorded on the
 * device; read them with ps_factor_status.  pivot_threshold = NaN selects
 * the reference default, 1e-13 max |diag(A)| (kernels.py:32-40), computed on
 * the device from the assembled slab (every ps_factor* entry point). */
int ps_factor(ps_plan* plan, double* d_store, int form, double pivot_threshold,
              void* stream);
/* ps_factor plus the download of the whole factor into pinned host memory
 * h_dst (the form's slabs: store_elems elements each, LU's U slab after the
 * L slab, complex128 elements for complex forms), overlapped with the
 * factorization: each slab chunk (whole panels, >= 4 MB; LU: its L and U
 * parts) is copied on a side stream as soon as its last writing launch has
 * run.  Asynchronous; the copies are joined into `stream`.  Replaces
 * pipeline.factorize + the host PanelStore the reference returns
 * (pipeline.py:97-117). */
int ps_factor_download(ps_plan* plan, double* d_store, int form, double pivot_threshold,
                       void* stream, double* h_dst);

/* Multi-GPU: plan for one rank of a subtree partition.
 * group[p] in [0, ngroups) assigns panel p's subtree to a rank, -1 puts it
 * in the shared top (ancestors of the groups).  The rank plan holds phase 0
 * = its own subtrees (level-batched) + its fan-in contributions into the
 * top, accumulated into its local copy of the top panels; phase 1 = the top.
 * Between the phases the caller sum-reduces the top region of the slabs
 * across ranks (NCCL; every non-top entry is owned by one rank and zero on
 * the others).  Replaces the reference's single-process runtime; the paper's
 * fan-in. */
int ps_plan_create_partitioned(const ps_symbol_desc* sym, int device, const int32_t* group,
                               int32_t ngroups, int32_t my_group, ps_plan** out);
int ps_plan_groups(const ps_plan* plan, int32_t* group);

/* Distributed top separators: like ps_plan_create_partitioned, plus
 * top_owner[p] = the rank that factors top panel p and applies every update
 * into it (-1 for subtree panels).  The top part of the plan is split into
 * two segments per top level (factor of the owned panels; updates into the
 * owned destinations); between them the caller broadcasts every panel of
 * that level from its owner.  Phase 0 is unchanged; the top region is
 * all-reduced before the segments.  bounds has nseg + 1 values: segment i
 * spans launches [bounds[i], bounds[i+1]); levels[i] is its top level. */
int ps_plan_create_distributed(const ps_symbol_desc* sym, int device, const int32_t* group,
                               int32_t ngroups, int32_t my_group, const int32_t* top_owner,
                               ps_plan** out);
int ps_plan_segments(const ps_plan* plan, int32_t* bounds, int32_t* levels, int32_t* nseg);
/* Launches [i0, i1) of the plan (a CUDA graph per range, cached); no status
 * reduction - call ps_factor_status_all then ps_factor_status. */
int ps_factor_range(ps_plan* plan, double* d_store, int form, double pivot_threshold,
                    void* stream, int32_t i0, int32_t i1);
int ps_factor_status_all(ps_plan* plan, void* stream);

/* ps_factor restricted to phase 0 or 1 of the launch sequence (-1: all). */
int ps_factor_phase(ps_plan* plan, double* d_store, int form, double pivot_threshold,
                    void* stream, int phase);

/* Same, launched without the graph with a CUDA event around every launch;
 * per-kind device milliseconds are returned in ms_by_kind[0..2]
 * = {factor (w==1 + diagonal/TRSM), trailing (intra-panel) updates,
 * inter-panel updates}, the launch count in *nlaunch and (if non-null) each
 * launch's milliseconds in per_launch_ms[nlaunches].  Used for the
 * roofline's per-kernel duration and for GPU traces (the reference's
 * TraceEvent CSV, runtime.py:325-336). */
int ps_factor_timed(ps_plan* plan, double* d_store, int form, double pivot_threshold,
                    void* stream, double* ms_by_kind, int32_t* nlaunch, float* per_launch_ms);

/* ps_factor_timed plus each launch's start (start_ms[nlaunches], relative
 * to the first launch's start; NULL allowed for any output).  Launches run
 * serialized on `stream` (no graph branches), so this is a per-launch
 * timeline of the whole factorization. */
int ps_factor_timeline(ps_plan* plan, double* d_store, int form, double pivot_threshold,
                       void* stream, double* ms_by_kind, int32_t* nlaunch, float* per_launch_ms,
                       float* start_ms);

/* Launch table: kind (0 width-1 factor, 1 small-panel factor+TRSM, 2 intra-panel
 * DMMA update, 3 DMMA inter-panel update, 4 narrow-source update, 5 wide-panel
 * diagonal factor + inverse, 6 wide-panel DMMA TRSM; graph markers 9 join,
 * 10 fork, 11 cross-wait), tree level (-1 for the deferred subtree->top fan-in
 * batch), item count and graph branch (0 = main, b > 0 = side branch b, run
 * concurrently) of every launch, in order.  For the markers, branch = the
 * branch joined into the main stream / forked off it / waited for, and for a
 * cross-wait count = the waiting branch (join: count 1 = the branch may be
 * forked again). */
int ps_plan_launches(const ps_plan* plan, int32_t* kind, int32_t* level, int32_t* count,
                     int32_t* branch);

/* The reference tasks (taskgraph.py:79-110 numbering: factor task of panel
 * p = p, update task of couple c = npanels + c, couples in panel then block
 * order) each launch works on: launch i serves task[ptr[i] .. ptr[i+1]).
 * ptr has nlaunches + 1 entries; task may be NULL to size it (ptr[nlaunches]).
 * With ps_factor_timed's per-launch times this gives the reference's
 * TraceEvent timeline (runtime.py:28-36, 325-336). */
int ps_plan_launch_tasks(const ps_plan* plan, int64_t* ptr, int64_t* task);

/* Synchronize `stream` and report the first failing column (minimum over
 * panels, i.e. the reference's sequential first failure).  Returns PS_OK
 * or PS_NUMERIC with *fail_col / *fail_pivot set. */
int ps_factor_status(ps_plan* plan, void* stream, int64_t* fail_col, double* fail_pivot);

/* Task-level operator (the reference plugin protocol run_task(task, ctx),
 * kernels.py:311-315): one factor task of panel p, or one update task of
 * couple (p -> q), on the device slab. */
int ps_run_factor_task(ps_plan* plan, double* d_store, int64_t p, int form,
                       double pivot_threshold, void* stream);
int ps_run_update_task(ps_plan* plan, double* d_store, int64_t p, int64_t q, int form,
                       void* stream);

/* Per launch of the level schedule (ps_plan_launches order): arithmetic
 * (tiles count the full 2 ni nj kn) and algorithmic HBM bytes (operands
 * read once, destination read + written) - the roofline of each launch. */
int ps_plan_launch_work(const ps_plan* plan, double* flops, double* bytes);
/* Debug: per DMMA update tile {start, mainloop done, end} globaltimer ns
 * into a device buffer of 3 * ps_plan_tile_count values (NULL: off). */
int ps_set_tile_trace(ps_plan* plan, void* d_trace);
int ps_plan_tile_count(const ps_plan* plan, int64_t* n);
/* Debug: the tiles (int32 fields: src, dst, i0, j0, ni, nj, k0, kn,
 * couple, wait, signal, ri, rj, 4 reserved, lds, ldd; int64 soff, doff) of
 * a plan created with PS_KEEP_TILES=1 (24 int32 per tile). */
int ps_plan_tiles(const ps_plan* plan, int32_t* out);

/* Supernodal triangular solve on the device-resident factor (reference
 * supernodal_solve, kernels.py:332-382): d_x (n doubles, PERMUTED order,
 * x[perm] = b) is overwritten with the solution (permuted order).  Forward
 * and backward substitution level by level, deterministic. */
int ps_solve(ps_plan* plan, const double* d_store, double* d_x, int form, void* stream);

/* Page-lock a host range for asynchronous uploads (A's values).
 * *registered = 1: registered here (release with ps_host_unregister);
 * 2: already page-locked elsewhere (usable as is); 0: not registrable (the
 * caller stages through its own pinned buffer).  Never leaves a CUDA error
 * pending. */
int ps_host_register(void* ptr, int64_t bytes, int* registered);
int ps_host_unregister(void* ptr);

/* Multi-GPU peer-to-peer primitives; pointers may be peer
 * GPUs' memory mapped through CUDA IPC (NVLink).  They replace the NCCL
 * all-reduce of the top region and the per-panel broadcasts.
 *
 * ps_p2p_segment_add: d_dst[off + i] += d_src[off + i] for every segment
 *   (off, len) = (d_seg[2k], d_seg[2k+1]), k < nseg; d_start = the nseg + 1
 *   prefix sums of the lengths (device), total = d_start[nseg].  The fan-in
 *   of one peer's contributions into the top panels this rank owns.
 * ps_p2p_signal: after every earlier operation on `stream`, store `value` into
 *   the 64-bit flag word d_flag (release, system scope).
 * ps_p2p_wait: later operations on `stream` wait until *d_flag >= value
 *   (acquire, system scope; d_flag typically a peer's flag word).  After
 *   timeout_s seconds the wait gives up and sets *d_timeout = 1. */
int ps_p2p_segment_add(double* d_dst, const double* d_src, const int64_t* d_seg,
                       const int64_t* d_start, int32_t nseg, int64_t total, void* stream);
int ps_p2p_signal(uint64_t* d_flag, uint64_t value, void* stream);
int ps_p2p_wait(const uint64_t* d_flag, uint64_t value, int32_t* d_timeout, double timeout_s,
                void* stream);

/* Last error message of the calling thread. */
const char* ps_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* PS_B200_H */
