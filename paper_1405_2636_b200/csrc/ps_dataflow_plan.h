// Host construction of the device task list (ps_dataflow.cuh).
//
// Tasks and the reference objects they refine:
//   DT_W1 (batches) / DT_SMALL / DT_DIAG + DT_TRSM + intra-panel DT_UPD
//                                       <- F(p) (kernels.py:208-247, taskgraph.py:79-93)
//   DT_UPD (inter-panel, source wider than 8) / DT_GATHER (narrow sources,
//   per 64x64 destination region)       <- U(p -> q)
//                                       (kernels.py:249-309, taskgraph.py:94-110)
// Counters (all start at 0 every factorization):
//   u(q)      = q          update tasks finished into q; F(q) waits for all
//   f(p)      = np + p     factor tasks finished of a panel of width > 1
//   batch b   = 2 np + b   width-1 batch finished
//   step / column counters of wide panels (allocated after)
// The list order is the start order of a list-scheduling simulation on
// `workers` virtual CTAs with critical-path priorities (reference:
// taskgraph.compute_costs_and_priorities, taskgraph.py:113-138), so it is a
// topological order of the dependency graph.
#pragma once
#include <algorithm>
#include <cmath>
#include <array>
#include <map>
#include <string>
#include <queue>
#include <utility>
#include <vector>

#include "ps_dataflow.cuh"

namespace psdf {

using ps::i64;

struct Dep {
  int ctr;
  unsigned target;
};

struct HTask {
  int type, idx, sig0, nsig;
  int dep0, ndep;
  float dur, prio;  // microseconds (cost model)
  int src, dst;     // panels (for traces / analysis)
  double flops;     // reference-model flops attributed to the task
};

struct Built {
  std::vector<ps::DTask> tasks;  // final (list) order
  std::vector<int2> deps;
  std::vector<int> sigs;
  std::vector<ps::UTile> tiles;
  std::vector<ps::FItem> fitems;
  std::vector<ps::NItem> nitems;
  std::vector<ps::GSeg> gsegs;
  std::vector<unsigned char> gmap;
  std::vector<int> w1;
  std::vector<int> task_src, task_dst, task_type;
  // ready-queue scheduler
  std::vector<i64> wl_ptr;          // per counter (nctr + 1)
  std::vector<unsigned> wl_thr;
  std::vector<int> wl_task;
  std::vector<int> rem_init;        // unmet dependencies per task
  std::vector<unsigned char> prio;  // 1: high-priority queue
  std::vector<int> prio_val;        // critical-path priority (higher first)
  std::vector<int> init_hi, init_lo;
  std::vector<double> task_flops;
  int nctr = 0;
  i64 scratch_slots = 0;
  double est_us = 0.0;
};

struct Input {
  i64 np;
  const std::vector<int>* w;
  const std::vector<int>* nrows;
  const std::vector<i64>* fc;  // first column of each panel
  const std::vector<int>* level;
  const std::vector<int>* c_p;
  const std::vector<int>* c_q;
  const std::vector<int>* c_loc0;
  const std::vector<int>* c_N;
  const std::vector<i64>* c_g0;
  const std::vector<i64>* c_g1;
  const std::vector<i64>* run_ptr;
  const std::vector<int>* run_src;
  const std::vector<int>* run_dst;
  const i64* blk_fr;
  const i64* blk_lr;
  const std::vector<i64>* cpl_first;
  const std::vector<i64>* off;  // slab offset of each panel
  int workers;
  int gather_max;   // segments per gather task
};

// destination-local index of source-local row x of couple c (walks the runs)
inline int map_local(const Input& in, int c, int x) {
  const auto& rp = *in.run_ptr;
  const auto& rs = *in.run_src;
  const auto& rd = *in.run_dst;
  i64 k = std::upper_bound(rs.begin() + rp[c], rs.begin() + rp[c + 1], x) - rs.begin() - 1;
  return rd[k] + (x - rs[k]);
}

// pieces of source-local rows [lo, hi) of couple c, one per (run, destination
// chunk of `csz`): {chunk, x0, x1, destination-local index of x0}
inline void run_pieces(const Input& in, int c, int lo, int hi, int src_end, int csz,
                       std::vector<std::array<int, 4>>& out) {
  const auto& rp = *in.run_ptr;
  const auto& rs = *in.run_src;
  const auto& rd = *in.run_dst;
  out.clear();
  i64 k0 = std::upper_bound(rs.begin() + rp[c], rs.begin() + rp[c + 1], lo) - rs.begin() - 1;
  for (i64 k = std::max<i64>(k0, rp[c]); k < rp[c + 1]; ++k) {
    const int r0 = rs[k];
    const int r1 = (k + 1 < rp[c + 1]) ? rs[k + 1] : src_end;
    const int a = std::max(lo, r0), b = std::min(hi, r1);
    if (a >= b) {
      if (r0 >= hi) break;
      continue;
    }
    int x = a;
    while (x < b) {
      const int d = rd[k] + (x - r0);
      const int ch = d / csz;
      const int xe = std::min(b, x + (ch + 1) * csz - d);
      out.push_back({ch, x, xe, d});
      x = xe;
    }
  }
}

// merge pieces of one destination chunk that are contiguous in the source
inline void merge_chunks(std::vector<std::array<int, 4>>& v) {
  size_t o = 0;
  for (size_t k = 0; k < v.size(); ++k) {
    if (o && v[o - 1][0] == v[k][0] && v[o - 1][2] == v[k][1]) v[o - 1][2] = v[k][2];
    else v[o++] = v[k];
  }
  v.resize(o);
}

// Gathers of the level schedule: the narrow couples `cpl` (sources factored,
// width <= SMALL_W) grouped per destination region; each region = a range
// of chunks (GMAX segments / GATHER_OPS operands / GATHER_MAPB map bytes),
// processed in order by one CTA.  Appends to the output vectors; returns the
// number of regions added.
struct LevelGathers {
  std::vector<ps::NItem> items;     // chunks
  std::vector<ps::GSeg> segs;
  std::vector<unsigned char> gmap;
  std::vector<int> region_ptr{0};   // region r = chunks [region_ptr[r], region_ptr[r+1])
};

inline int build_level_gathers(const Input& in, const std::vector<int>& cpl, LevelGathers& out,
                               int rows = ps::LG_ROWS, int gmax = ps::LG_GMAX,
                               int ops_max = ps::LG_OPS, int mapb_max = ps::LG_MAPB) {
  using namespace ps;
  const auto& W = *in.w;
  const auto& NR = *in.nrows;
  std::map<std::array<int, 3>, std::vector<GSeg>> regions;
  std::vector<std::array<int, 4>> rp, cpcs;
  std::vector<unsigned char> tmp;
  for (int c : cpl) {
    const int p = (*in.c_p)[c], q = (*in.c_q)[c];
    const int loc0 = (*in.c_loc0)[c], N = (*in.c_N)[c], nr = NR[p];
    run_pieces(in, c, loc0, nr, nr, rows, rp);
    run_pieces(in, c, loc0, loc0 + N, nr, TN, cpcs);
    merge_chunks(rp);
    merge_chunks(cpcs);
    for (const auto& cc : cpcs)
      for (const auto& rr : rp) {
        if (rr[2] - 1 < cc[1]) continue;
        GSeg g{(*in.off)[p], nr, W[p], rr[1], rr[2] - rr[1], cc[1], cc[2] - cc[1],
               (int)tmp.size(), 0, 0, 0};
        for (int x = rr[1]; x < rr[2]; ++x) tmp.push_back((unsigned char)(map_local(in, c, x) - rr[0] * rows));
        for (int x = cc[1]; x < cc[2]; ++x) tmp.push_back((unsigned char)(map_local(in, c, x) - cc[0] * TN));
        regions[{q, rr[0], cc[0]}].push_back(g);
      }
  }
  int nreg = 0;
  for (auto& kv : regions) {
    const int q = kv.first[0], rch = kv.first[1], cch = kv.first[2];
    auto& v = kv.second;
    unsigned long long cmask = 0;
    for (const GSeg& g : v)
      for (int x = 0; x < g.nj; ++x) cmask |= 1ULL << tmp[g.gm + g.ni + x];
    for (size_t k = 0; k < v.size();) {
      size_t e = k;
      int ops = 0, mb = 0;
      while (e < v.size() && e - k < (size_t)gmax) {
        const int need = v[e].kn * (v[e].ni + v[e].nj) + v[e].kn;
        if (e > k && (ops + need > ops_max || mb + v[e].ni + v[e].nj > mapb_max)) break;
        ops += need;
        mb += v[e].ni + v[e].nj;
        ++e;
      }
      while (out.gmap.size() % 16) out.gmap.push_back(0);
      const int gbase = (int)out.gmap.size();
      NItem it{q, rch * rows, std::min(rows, NR[q] - rch * rows), cch * TN, std::min(TN, W[q] - cch * TN),
               (int)out.segs.size(), (int)(e - k), 0, cmask};
      int op0 = 0, mp0 = 0;
      for (size_t u = k; u < e; ++u) {
        GSeg g = v[u];
        out.gmap.insert(out.gmap.end(), tmp.begin() + g.gm, tmp.begin() + g.gm + g.ni + g.nj);
        g.gm = gbase;
        g.op0 = op0;
        g.mp0 = mp0;
        op0 += g.kn * (g.ni + g.nj) + g.kn;
        mp0 += g.ni + g.nj;
        out.segs.push_back(g);
      }
      out.items.push_back(it);
      k = e;
    }
    out.region_ptr.push_back((int)out.items.size());
    ++nreg;
  }
  while (out.gmap.size() % 16) out.gmap.push_back(0);
  return nreg;
}

// cost model (microseconds per task on one of `workers` CTAs)
constexpr double US_OVH = 1.5;          // ticket + dependency hop + epilogue
constexpr double FLOP_PER_US = 8.0e4;   // DMMA tile rate of one CTA sharing an SM
constexpr double BYTE_PER_US = 2.0e4;   // HBM share of one CTA
constexpr double DIAG_US = 30.0;

inline double tile_us(int ni, int nj, int kn) {
  return US_OVH + 2.0 * ni * nj * kn / FLOP_PER_US + 16.0 * ni * nj / BYTE_PER_US;
}

template <class EmitTiles>
int build(const Input& in, Built& out, EmitTiles emit_tiles, std::string* err) {
  using namespace ps;
  const i64 np = in.np;
  const auto& W = *in.w;
  const auto& NR = *in.nrows;
  const auto& LV = *in.level;
  const auto& cp_ = *in.c_p;
  const auto& cq_ = *in.c_q;
  const i64 nc = (i64)cp_.size();
  int nlev = 0;
  for (i64 p = 0; p < np; ++p) nlev = std::max(nlev, LV[p] + 1);

  std::vector<HTask> T;
  std::vector<Dep> D;
  std::vector<int> SG;  // signal lists (build order)
  auto add_task = [&](int type, int idx, const std::vector<Dep>& deps, const std::vector<int>& sigs,
                      double dur, int src, int dst, double flops) {
    HTask t{type, idx, (int)SG.size(), (int)sigs.size(), (int)D.size(), 0, (float)dur, 0.f, src,
            dst, flops};
    for (const Dep& d : deps)
      if (d.target > 0) {
        D.push_back(d);
        ++t.ndep;
      }
    SG.insert(SG.end(), sigs.begin(), sigs.end());
    T.push_back(t);
    return (int)T.size() - 1;
  };

  // ---- factor completion counters (shape only) ----
  int nctr = (int)(2 * np);
  std::vector<Dep> fdep(np, Dep{0, 0});
  std::vector<std::vector<int>> w1_lv(nlev);
  for (i64 p = 0; p < np; ++p)
    if (W[p] == 1) w1_lv[LV[p]].push_back((int)p);
  struct Batch { int first, count, ctr; };
  std::vector<Batch> batches;
  const int BATCH = (DF_THREADS / 32) * W1_PER_WARP;
  for (int L = 0; L < nlev; ++L)
    for (size_t k = 0; k < w1_lv[L].size(); k += BATCH) {
      Batch b{(int)out.w1.size(), (int)std::min<size_t>(BATCH, w1_lv[L].size() - k), nctr++};
      for (int u = 0; u < b.count; ++u) {
        const int p = w1_lv[L][k + u];
        out.w1.push_back(p);
        fdep[p] = Dep{b.ctr, 1};
      }
      batches.push_back(b);
    }
  // width-1 panels are read unfactored (raw) by the gathers during the whole
  // factorization; one pass after the dataflow kernel scales them all
  auto wide_ntrsm = [&](int p, int s) {
    const int c0 = s * FNB, nb = std::min(FNB, W[p] - c0), rbeg = c0 + nb;
    return NR[p] > rbeg ? (NR[p] - rbeg + TM - 1) / TM : 0;
  };
  for (i64 p = 0; p < np; ++p) {
    if (W[p] == 1) continue;
    unsigned tot;
    if (W[p] <= SNB) {
      const int rows = NR[p] - W[p];
      tot = 1 + (rows > FTR ? (rows + FTR - 1) / FTR - 1 : 0);
    } else {
      const int S = (W[p] + FNB - 1) / FNB;
      tot = S;
      for (int s = 0; s < S; ++s) tot += wide_ntrsm((int)p, s);
    }
    fdep[p] = Dep{(int)(np + p), tot};
  }

  // ---- factor cost estimates and critical-path priorities ----
  std::vector<double> fcost(np), tl(np, 0.0);
  for (i64 p = 0; p < np; ++p) {
    const double w = W[p], m = NR[p] - W[p];
    if (W[p] == 1) fcost[p] = 0.5;  // read raw by the gathers: off the path
    else if (W[p] <= SNB) fcost[p] = 3.0 + 0.3 * w + m * w * w / 4e4;
    else fcost[p] = std::ceil(w / FNB) * (DIAG_US + 2 * tile_us(TM, FNB, FNB) + 3 * US_OVH);
  }
  for (i64 p = np - 1; p >= 0; --p) {
    double best = 0.0;
    for (i64 c = (*in.cpl_first)[p]; c < (*in.cpl_first)[p + 1]; ++c) {
      const int q = cq_[c];
      const double u = (W[p] <= SMALL_W ? 3.0 : tile_us(TM, TN, W[p])) + tl[q];
      best = std::max(best, u);
    }
    tl[p] = fcost[p] + best;
  }

  // ---- update units: narrow-source gathers per destination region, and
  //      wide couples ----
  struct SegRec { int lev, p; GSeg s; };
  std::map<std::array<int, 3>, std::vector<SegRec>> regions;
  std::vector<std::array<int, 4>> rp, cpcs;
  for (i64 c = 0; c < nc; ++c) {
    const int p = cp_[c], q = cq_[c];
    if (W[p] > SMALL_W) continue;
    const int loc0 = (*in.c_loc0)[c], N = (*in.c_N)[c], nr = NR[p];
    run_pieces(in, (int)c, loc0, nr, nr, TM, rp);
    run_pieces(in, (int)c, loc0, loc0 + N, nr, TN, cpcs);
    merge_chunks(rp);
    merge_chunks(cpcs);
    for (const auto& cc : cpcs)
      for (const auto& rr : rp) {
        if (rr[2] - 1 < cc[1]) continue;  // no entry i >= j
        GSeg g{(*in.off)[p], nr, W[p], rr[1], rr[2] - rr[1], cc[1], cc[2] - cc[1],
               (int)out.gmap.size(), 0, 0, W[p] == 1 ? 1 : 0};
        for (int x = rr[1]; x < rr[2]; ++x)
          out.gmap.push_back((unsigned char)(map_local(in, (int)c, x) - rr[0] * TM));
        for (int x = cc[1]; x < cc[2]; ++x)
          out.gmap.push_back((unsigned char)(map_local(in, (int)c, x) - cc[0] * TN));
        regions[{q, rr[0], cc[0]}].push_back(SegRec{LV[p], p, g});
      }
  }
  struct Unit {
    int lev, kind, q;
    i64 id;          // gather item index (kind 0) or couple id (kind 1)
  };
  std::vector<Unit> units;
  std::vector<std::vector<int>> gsrc;  // gather item -> distinct source panels
  std::vector<std::vector<int>> gcols; // gather item -> touched global columns
  std::vector<unsigned char> gmap2;
  for (auto& kv : regions) {
    auto& v = kv.second;
    std::stable_sort(v.begin(), v.end(), [](const SegRec& a, const SegRec& b) {
      return a.lev != b.lev ? a.lev < b.lev : a.p < b.p;
    });
    const int q = kv.first[0], rch = kv.first[1], cch = kv.first[2];
    const i64 qfc = (*in.fc)[q];
    for (size_t k = 0; k < v.size();) {
      // one gather task: at most GMAX segments and GATHER_OPS operand doubles
      size_t e = k;
      int ops = 0, mb = 0;
      // the segments of the region's latest source level get their own
      // gather(s): the last gather into a region then waits only for the
      // last sources and applies only their segments (critical path)
      const int maxlev = v.back().lev;
      while (e < v.size() && e - k < (size_t)std::min(GMAX, in.gather_max) &&
             (v[e].lev == maxlev) == (v[k].lev == maxlev)) {
        const GSeg& g = v[e].s;
        const int need = g.kn * (g.ni + g.nj) + g.kn;
        if (e > k && (ops + need > GATHER_OPS || mb + g.ni + g.nj > GATHER_MAPB)) break;
        ops += need;
        mb += g.ni + g.nj;
        ++e;
      }
      NItem it{q, rch * TM, std::min(TM, NR[q] - rch * TM), cch * TN,
               std::min(TN, W[q] - cch * TN), (int)out.gsegs.size(), (int)(e - k), 0, 0ULL};
      std::vector<int> srcs, cols;
      int lev = 0, op0 = 0, mp0 = 0;
      // this gather's maps, contiguous and 16-byte aligned in gmap2 (one
      // vectorised load per task); GSeg.gm = start of the gather's area
      while (gmap2.size() % 16) gmap2.push_back(0);
      const int gbase = (int)gmap2.size();
      for (size_t u = k; u < e; ++u) {
        GSeg g = v[u].s;
        gmap2.insert(gmap2.end(), out.gmap.begin() + g.gm, out.gmap.begin() + g.gm + g.ni + g.nj);
        g.gm = gbase;
        g.op0 = op0;
        g.mp0 = mp0;
        op0 += g.kn * (g.ni + g.nj) + g.kn;
        mp0 += g.ni + g.nj;
        out.gsegs.push_back(g);
        srcs.push_back(v[u].p);
        lev = std::max(lev, v[u].lev);
        for (int x = 0; x < g.nj; ++x) {
          const int lc = gmap2[gbase + g.mp0 + g.ni + x];
          it.cmask |= 1ULL << lc;
          cols.push_back((int)(qfc + it.c0 + lc));
        }
      }
      std::sort(srcs.begin(), srcs.end());
      srcs.erase(std::unique(srcs.begin(), srcs.end()), srcs.end());
      std::sort(cols.begin(), cols.end());
      cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
      units.push_back(Unit{lev, 0, q, (i64)out.nitems.size()});
      out.nitems.push_back(it);
      gsrc.push_back(std::move(srcs));
      gcols.push_back(std::move(cols));
      k = e;
    }
  }
  std::map<std::array<int, 3>, std::vector<SegRec>>().swap(regions);
  while (gmap2.size() % 16) gmap2.push_back(0);
  out.gmap.swap(gmap2);
  for (i64 c = 0; c < nc; ++c)
    if (W[cp_[c]] > SMALL_W) units.push_back(Unit{LV[cp_[c]], 1, cq_[c], c});
  std::stable_sort(units.begin(), units.end(), [](const Unit& a, const Unit& b) {
    if (a.lev != b.lev) return a.lev < b.lev;
    if (a.kind != b.kind) return a.kind < b.kind;
    return a.id < b.id;
  });

  // ---- color by destination-column overlap in base order, never below the
  //      colors of earlier levels (a unit of color k waits for every task of
  //      colors < k into q; all units are single-destination, so the waits
  //      only link updates into q, whose sources never depend on q: acyclic)
  const i64 ncols_total = np ? (*in.fc)[np - 1] + W[np - 1] : 0;
  std::vector<int> lastcol(ncols_total, -1);
  std::vector<int> ucolor(units.size()), untasks(units.size(), 1);
  std::vector<int> qmax(np, -1), qfloor(np, 0), touched;
  std::vector<std::vector<int>> ccount(np);
  std::vector<int> cols;
  int cur_lev = -1;
  for (size_t k = 0; k < units.size(); ++k) {
    const Unit& u = units[k];
    if (u.lev != cur_lev) {
      for (int q : touched) qfloor[q] = std::max(qfloor[q], qmax[q]);
      touched.clear();
      cur_lev = u.lev;
    }
    const int q = u.q;
    touched.push_back(q);
    cols.clear();
    if (u.kind == 1) {
      for (i64 b = (*in.c_g0)[u.id]; b < (*in.c_g1)[u.id]; ++b)
        for (i64 r = in.blk_fr[b]; r < in.blk_lr[b]; ++r) cols.push_back((int)r);
      const int p = cp_[u.id], loc0 = (*in.c_loc0)[u.id], N = (*in.c_N)[u.id];
      int cnt = 0;  // tiles of the lower trapezoid (emit_tiles' enumeration)
      for (int j = loc0; j < loc0 + N; j += TN)
        for (int i = loc0; i < NR[p]; i += TM)
          if (i + std::min(TM, NR[p] - i) - 1 >= j) ++cnt;
      untasks[k] = cnt;
    } else {
      cols = gcols[u.id];
    }
    int col = qfloor[q];
    for (int r : cols) col = std::max(col, lastcol[r] + 1);
    for (int r : cols) lastcol[r] = col;
    ucolor[k] = col;
    qmax[q] = std::max(qmax[q], col);
    auto& cc = ccount[q];
    if ((int)cc.size() <= col) cc.resize(col + 1, 0);
    cc[col] += untasks[k];
  }
  std::vector<int>().swap(lastcol);
  std::vector<std::vector<int>>().swap(gcols);
  std::vector<std::vector<unsigned>> cpre(np);
  std::vector<unsigned> nin(np, 0);
  for (i64 q = 0; q < np; ++q) {
    auto& cc = ccount[q];
    cpre[q].assign(cc.size() + 1, 0);
    for (size_t k = 0; k < cc.size(); ++k) cpre[q][k + 1] = cpre[q][k] + cc[k];
    nin[q] = cpre[q].back();
  }

  // ---- update tasks ----
  for (size_t k = 0; k < units.size(); ++k) {
    const Unit& u = units[k];
    const int q = u.q;
    const Dep cdep{q, cpre[q][ucolor[k]]};
    if (u.kind == 1) {
      const i64 c = u.id;
      const int p = cp_[c];
      const int loc0 = (*in.c_loc0)[c], N = (*in.c_N)[c];
      std::vector<UTile> tiles;
      emit_tiles(tiles, p, q, loc0, NR[p], loc0, loc0 + N, 0, W[p], (int)c);
      for (const UTile& t : tiles) {
        const int idx = (int)out.tiles.size();
        out.tiles.push_back(t);
        const int ti = add_task(DT_UPD, idx, {fdep[p], cdep}, {q}, tile_us(t.ni, t.nj, t.kn), p, q,
                                2.0 * t.ni * t.nj * t.kn);
        T[ti].prio = (float)(tl[q] + T[ti].dur);
      }
    } else {
      std::vector<Dep> deps{cdep};
      std::map<int, unsigned> byctr;
      for (int p : gsrc[u.id]) {
        const Dep d = W[p] == 1 ? Dep{p, nin[p]} : fdep[p];
        byctr[d.ctr] = std::max(byctr[d.ctr], d.target);
      }
      for (auto& kv : byctr) deps.push_back(Dep{kv.first, kv.second});
      const NItem& it = out.nitems[u.id];
      double fl = 0.0;
      for (int s = it.seg0; s < it.seg0 + it.nseg; ++s) {
        const GSeg& g = out.gsegs[s];
        fl += 2.0 * g.ni * g.nj * g.kn;
      }
      std::vector<int> sigs{q};
      const int ti = add_task(DT_GATHER, (int)u.id, deps, sigs, US_OVH + 1.0 + 0.1 * it.nseg,
                              gsrc[u.id].front(), q, fl);
      T[ti].prio = (float)(tl[q] + T[ti].dur);
    }
  }

  // ---- factor tasks ----
  i64 slot = 0;
  for (i64 p = 0; p < np; ++p) {
    const int w = W[p], nr = NR[p];
    if (w == 1) continue;
    const Dep din{(int)p, nin[p]};
    const int f = (int)(np + p);
    if (w <= SNB) {
      const int rows = nr - w;
      const double wd = w;
      int idx = (int)out.fitems.size();
      out.fitems.push_back(FItem{(int)p, 0, w, w, std::min(FTR, rows), 1, 0, 0});
      double fl = wd * (wd + 1) * (2 * wd + 1) / 6.0 + std::min(FTR, rows) * wd * wd;
      int t = add_task(DT_SMALL, idx, {din}, {f}, fcost[p], (int)p, -1, fl);
      T[t].prio = (float)tl[p];
      for (int k = 1; k * FTR < rows; ++k) {
        idx = (int)out.fitems.size();
        const int r = std::min(FTR, rows - k * FTR);
        out.fitems.push_back(FItem{(int)p, 0, w, w + k * FTR, r, 0, 0, 0});
        t = add_task(DT_SMALL, idx, {Dep{f, 1}}, {f}, 2.0 + r * wd * wd / 4e4, (int)p, -1, r * wd * wd);
        T[t].prio = (float)(tl[p] - 3.0);
      }
      continue;
    }
    const int S = (w + FNB - 1) / FNB;
    std::vector<int> colc(S, -1);
    for (int c = 1; c < S; ++c) colc[c] = nctr++;
    std::vector<unsigned> colcnt(S, 0);  // trailing tiles into column block c so far
    const double step_us = DIAG_US + 2 * tile_us(TM, FNB, FNB) + 3 * US_OVH;
    for (int s = 0; s < S; ++s) {
      const int stp = nctr++;
      const int c0 = s * FNB, nb = std::min(FNB, w - c0), rbeg = c0 + nb;
      const double pr = tl[p] - s * step_us;
      const int g = (int)slot++;
      int idx = (int)out.fitems.size();
      out.fitems.push_back(FItem{(int)p, c0, nb, rbeg, 0, 1, g, 0});
      const Dep d0 = s == 0 ? din : Dep{colc[s], colcnt[s]};
      const double nbd = nb;
      int t = add_task(DT_DIAG, idx, {d0}, {stp, f}, DIAG_US, (int)p, -1,
                       nbd * (nbd + 1) * (2 * nbd + 1) / 6.0);
      T[t].prio = (float)pr;
      const int ntr = wide_ntrsm((int)p, s);
      for (int r = rbeg; r < nr; r += TM) {
        idx = (int)out.fitems.size();
        const int nrr = std::min(TM, nr - r);
        out.fitems.push_back(FItem{(int)p, c0, nb, r, nrr, 0, g, 0});
        t = add_task(DT_TRSM, idx, {Dep{stp, 1}}, {stp, f}, tile_us(nrr, nb, nb), (int)p, -1,
                     (double)nrr * nb * nb);
        T[t].prio = (float)(pr - DIAG_US);
      }
      if (rbeg < w) {
        std::vector<UTile> tl_tiles;
        emit_tiles(tl_tiles, (int)p, (int)p, rbeg, nr, rbeg, w, c0, nb, -1);
        std::vector<unsigned> before(colcnt);
        for (const UTile& u : tl_tiles) {
          const int c = u.j0 / FNB;
          idx = (int)out.tiles.size();
          out.tiles.push_back(u);
          t = add_task(DT_UPD, idx, {Dep{stp, (unsigned)(1 + ntr)}, Dep{colc[c], before[c]}},
                       {colc[c]}, tile_us(u.ni, u.nj, u.kn), (int)p, (int)p,
                       2.0 * u.ni * u.nj * u.kn);
          // the look-ahead column (s + 1) first
          T[t].prio = (float)(pr - DIAG_US - tile_us(TM, FNB, FNB) - (c == s + 1 ? 0.0 : step_us));
          colcnt[c]++;
        }
      }
    }
  }
  out.scratch_slots = slot;
  out.nctr = nctr;

  // ---- list-scheduling simulation -> start order ----
  const int nt = (int)T.size();
  std::vector<int> remaining(nt, 0);
  std::vector<std::vector<std::pair<unsigned, int>>> waiters(nctr);
  for (int t = 0; t < nt; ++t)
    for (int d = T[t].dep0; d < T[t].dep0 + T[t].ndep; ++d) {
      waiters[D[d].ctr].push_back({D[d].target, t});
      ++remaining[t];
    }
  for (auto& w : waiters) std::sort(w.begin(), w.end());
  std::vector<size_t> wptr(nctr, 0);
  std::vector<unsigned> val(nctr, 0);
  std::priority_queue<std::pair<float, int>> ready;
  for (int t = 0; t < nt; ++t)
    if (!remaining[t]) ready.push({T[t].prio, -t});
  std::priority_queue<std::pair<double, int>, std::vector<std::pair<double, int>>,
                      std::greater<std::pair<double, int>>>
      ev;
  std::vector<int> order;
  order.reserve(nt);
  int idle = std::max(1, in.workers);
  double now = 0.0;
  while ((int)order.size() < nt || !ev.empty()) {
    while (idle > 0 && !ready.empty()) {
      const int t = -ready.top().second;
      ready.pop();
      order.push_back(t);
      ev.push({now + T[t].dur, t});
      --idle;
    }
    if (ev.empty()) break;
    const auto e = ev.top();
    ev.pop();
    now = e.first;
    ++idle;
    for (int k = 0; k < T[e.second].nsig; ++k) {
      const int sg = SG[T[e.second].sig0 + k];
      const unsigned v = ++val[sg];
      auto& wl = waiters[sg];
      while (wptr[sg] < wl.size() && wl[wptr[sg]].first <= v) {
        const int t = wl[wptr[sg]].second;
        if (--remaining[t] == 0) ready.push({T[t].prio, -t});
        ++wptr[sg];
      }
    }
  }
  if ((int)order.size() != nt) {
    if (err) *err = "dataflow schedule: dependency cycle (" + std::to_string(nt - (int)order.size()) +
                    " tasks never ready)";
    return -1;
  }
  out.est_us = now;
  out.tasks.resize(nt);
  out.deps.clear();
  out.deps.reserve(D.size());
  out.sigs.clear();
  out.sigs.reserve(SG.size());
  out.task_src.resize(nt);
  out.task_dst.resize(nt);
  out.task_type.resize(nt);
  out.task_flops.resize(nt);
  for (int k = 0; k < nt; ++k) {
    const HTask& h = T[order[k]];
    DTask d{h.type, h.idx, (int)out.deps.size(), h.ndep, (int)out.sigs.size(), h.nsig, 0, 0};
    for (int u = h.dep0; u < h.dep0 + h.ndep; ++u) out.deps.push_back(int2{D[u].ctr, (int)D[u].target});
    for (int u = h.sig0; u < h.sig0 + h.nsig; ++u) out.sigs.push_back(SG[u]);
    out.tasks[k] = d;
    out.task_src[k] = h.src;
    out.task_dst[k] = h.dst;
    out.task_type[k] = h.type;
    out.task_flops[k] = h.flops;
  }
  // waiter lists per counter (final task indices), sorted by threshold
  std::vector<int> pos(nt);
  for (int k = 0; k < nt; ++k) pos[order[k]] = k;
  out.wl_ptr.assign(nctr + 1, 0);
  for (int c = 0; c < nctr; ++c) out.wl_ptr[c + 1] = out.wl_ptr[c] + (i64)waiters[c].size();
  out.wl_thr.resize(out.wl_ptr[nctr]);
  out.wl_task.resize(out.wl_ptr[nctr]);
  for (int c = 0; c < nctr; ++c)
    for (size_t k = 0; k < waiters[c].size(); ++k) {
      out.wl_thr[out.wl_ptr[c] + k] = waiters[c][k].first;
      out.wl_task[out.wl_ptr[c] + k] = pos[waiters[c][k].second];
    }
  out.rem_init.resize(nt);
  out.prio.resize(nt);
  out.prio_val.resize(nt);
  for (int k = 0; k < nt; ++k) {
    const HTask& h = T[order[k]];
    out.rem_init[k] = h.ndep;
    // factor work unblocks everything downstream: high priority
    const bool hi = h.type == DT_W1 || h.type == DT_SMALL || h.type == DT_DIAG ||
                    h.type == DT_TRSM || (h.type == DT_UPD && h.src == h.dst);
    out.prio[k] = hi ? 1 : 0;
    out.prio_val[k] = (int)std::min(2.0e9, std::max(0.0, (double)h.prio * 10.0));
    if (h.ndep == 0) out.init_hi.push_back(k);
  }
  return 0;
}

}  // namespace psdf
