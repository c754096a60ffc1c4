// Complex (complex128) update tiles on the FP64 tensor cores.
//
// The paper's sparse_gemm (kernels.py:128-136, twice for LU: PAPER.md:321-331)
// in complex arithmetic, C(map i, map j) -= sum_k A(i, k) B(j, k), with
//   LLt : B = A (complex symmetric, no conjugation)
//   LDLt: B(j, k) = d_k A(j, k)
//   LU  : pass 0 A = L rows, B = U^T rows into L (i >= j);
//         pass 1 A = U^T rows, B = L rows into U^T (i > j)
// as four real DMMA products per fragment pair (DMMA.8x8x4):
//   Cr += Ar Br^T - Ai Bi^T,   Ci += Ar Bi^T + Ai Br^T.
// Same plan and protocol as k_update: persistent CTAs take tiles in list
// order, the couple's run window is staged for the index maps, the scatter
// waits for the destination's lower colors and signals after (atomics-free,
// deterministic).  Operands are staged as interleaved complex (16-byte
// cp.async per element) through a 3-stage pipeline of 8-wide k chunks; 8 warps
// in a 2 x 4 grid each hold a 32 x 16 complex accumulator (4 x 2 fragments,
// real and imaginary parts); the epilogue scatters straight from the
// accumulator fragments (a lane owns one row and two adjacent columns).
#pragma once
#include "ps_generic.cuh"

namespace ps {

constexpr int ZKC = 8, ZNST = 3, ZT = 256;

struct ZSmem {
  double2 A[ZNST][ZKC][TM + 1];
  double2 B[ZNST][ZKC][TN + 1];
  double2 D[ZNST][ZKC];
  int rmap[TM];
  int cmap[TN];
  int wsrc[2][TM];
  int wdst[2][TM];
  int tile;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}

struct ZOperands {
  const double2* A;
  const double2* B;
  const double2* dptr;  // LDLt: d_k at dptr[k * dstride]
  i64 ld, dstride;
  int i0, ni, j0, nj, kn;
  const ChainSeg* seg = nullptr;  // merged chain tile: the next piece (ps_kernels.cuh)
  int knext = INT_MAX;
};

__device__ __forceinline__ void z_load_stage(ZSmem& sm, int st, ZOperands& O, int chunk, int tid) {
  const int kbase = chunk * ZKC;
  chain_advance(O.seg, O.knext, kbase, O.A, O.B, O.dptr, O.ld, O.ld, O.dstride);
  const i64 ld = O.ld, dstr = O.dstride;
  const int i0 = O.i0, j0 = O.j0;
  const double2* Ac = O.A + (i64)kbase * ld;
  const double2* Bc = O.B + (i64)kbase * ld;
  const double2* Dc = O.dptr ? O.dptr + (i64)kbase * dstr : nullptr;
#pragma unroll
  for (int e = 0; e < (ZKC * TM) / ZT; ++e) {
    const int idx = tid + e * ZT;
    const int r = idx % TM, kk = idx / TM;
    const bool va = kbase + kk < O.kn && r < O.ni;
    cp_async16(&sm.A[st][kk][r], Ac + (i64)(va ? kk : 0) * ld + (va ? i0 + r : 0), va);
    const bool vb = kbase + kk < O.kn && r < O.nj;
    cp_async16(&sm.B[st][kk][r], Bc + (i64)(vb ? kk : 0) * ld + (vb ? j0 + r : 0), vb);
  }
  if (Dc && tid < ZKC) {
    const bool kv = kbase + tid < O.kn;
    cp_async16(&sm.D[st][tid], Dc + (i64)(kv ? tid : 0) * dstr, kv);
  }
}

// acc[mi][ni][0] = real, [1] = imaginary part; each a DMMA 8x8 fragment pair
__device__ __forceinline__ void z_mainloop(ZSmem& sm, ZOperands O, double acc[4][2][2][2],
                                           int tid) {
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int c = 0; c < 2; ++c) acc[a][b][c][0] = acc[a][b][c][1] = 0.0;
  const int nch = (O.kn + ZKC - 1) / ZKC;
#pragma unroll
  for (int s = 0; s < ZNST - 1; ++s) {
    if (s < nch) z_load_stage(sm, s, O, s, tid);
    cp_async_commit();
  }
  for (int c = 0; c < nch; ++c) {
    cp_async_wait<ZNST - 2>();
    __syncthreads();
    const int nxt = c + ZNST - 1;
    if (nxt < nch) z_load_stage(sm, nxt % ZNST, O, nxt, tid);
    cp_async_commit();
    const int st = c % ZNST;
    const int krem = O.kn - c * ZKC;
#pragma unroll
    for (int ks = 0; ks < ZKC / 4; ++ks) {
      if (ks > 0 && 4 * ks >= krem) break;
      const int kr = ks * 4 + (lane & 3);
      double ar[4], ai[4], nai[4], br[2], bi[2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        const double2 v = sm.A[st][kr][wm * 32 + mi * 8 + (lane >> 2)];
        ar[mi] = v.x;
        ai[mi] = v.y;
        nai[mi] = -v.y;
      }
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) {
        double2 v = sm.B[st][kr][wn * 16 + ni * 8 + (lane >> 2)];
        if (O.dptr) {
          const double2 d = sm.D[st][kr];
          v = make_double2(fma(v.x, d.x, -v.y * d.y), fma(v.x, d.y, v.y * d.x));
        }
        br[ni] = v.x;
        bi[ni] = v.y;
      }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) {
          dmma(acc[mi][ni][0][0], acc[mi][ni][0][1], ar[mi], br[ni]);
          dmma(acc[mi][ni][0][0], acc[mi][ni][0][1], nai[mi], bi[ni]);
          dmma(acc[mi][ni][1][0], acc[mi][ni][1][1], ar[mi], bi[ni]);
          dmma(acc[mi][ni][1][0], acc[mi][ni][1][1], ai[mi], br[ni]);
        }
    }
  }
  cp_async_wait<0>();
  __syncthreads();
}

// C(map i, map j) -= acc for the lane's entries (one row, two adjacent
// columns per fragment) on / strictly below the diagonal
__device__ __forceinline__ void z_scatter(const ZSmem& sm, double acc[4][2][2][2], double2* dst,
                                          i64 ldd, const UTile& T, int strict, int tid) {
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
#pragma unroll
  for (int half = 0; half < 2; ++half) {  // 8 entries in flight per lane
    double2* pp[2][2][2];
    double2 old[2][2][2];
#pragma unroll
    for (int m2 = 0; m2 < 2; ++m2) {
      const int row = wm * 32 + (2 * half + m2) * 8 + (lane >> 2);
#pragma unroll
      for (int ni = 0; ni < 2; ++ni)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = wn * 16 + ni * 8 + 2 * (lane & 3) + h;
          const bool ok = row < T.ni && col < T.nj && T.i0 + row >= T.j0 + col + strict;
          pp[m2][ni][h] = ok ? dst + (i64)sm.cmap[col] * ldd + sm.rmap[row] : nullptr;
          old[m2][ni][h] = ok ? __ldcg(pp[m2][ni][h]) : make_double2(0.0, 0.0);
        }
    }
#pragma unroll
    for (int m2 = 0; m2 < 2; ++m2)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (pp[m2][ni][h]) {
            const double* a = acc[2 * half + m2][ni][0];
            const double* b = acc[2 * half + m2][ni][1];
            __stcg(pp[m2][ni][h], make_double2(old[m2][ni][h].x - a[h], old[m2][ni][h].y - b[h]));
          }
  }
}

template <int F>
__global__ void __launch_bounds__(ZT, 2)
k_zupdate(const UTile* __restrict__ tiles, int ntiles, int* __restrict__ work_ctr,
          unsigned* __restrict__ counters, const DevArgs* __restrict__ args,
          const i64* __restrict__ run_ptr, const int* __restrict__ run_src,
          const int* __restrict__ run_dst) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char zsm_raw[];
  ZSmem& sm = *reinterpret_cast<ZSmem*>(zsm_raw);
  const int tid = threadIdx.x;
  double2* store = reinterpret_cast<double2*>(args->store);
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
    const double2* colk = store + T.soff + (i64)T.k0 * lds;
    if (tid < 128) maps_load(sm, T.couple, T.ri, T.rj, run_ptr, run_src, run_dst, tid);
    __syncthreads();
    if (tid < 128) maps_search(sm, T.couple, T.i0, T.ni, T.j0, T.nj, tid);
    for (int pass = 0; pass < (F == FORM_LU ? 2 : 1); ++pass) {
      ZOperands O{colk + (pass ? us : 0), colk + (F == FORM_LU && !pass ? us : 0),
                  F == FORM_LDLT ? colk + T.k0 : nullptr, lds, lds + 1,
                  T.i0, T.ni, T.j0, T.nj, T.kn, chain_of(args, T), T.mode > 0 ? 0 : INT_MAX};
      double acc[4][2][2][2];
      z_mainloop(sm, O, acc, tid);  // (its barriers also publish the maps)
      if (pass == 0 && T.wait >= 0 && tid == 0) {
        while (ld_acquire(&counters[T.dst]) < (unsigned)T.wait) __nanosleep(32);
      }
      __syncthreads();
      z_scatter(sm, acc, store + T.doff + (pass ? us : 0), T.ldd, T, pass, tid);
    }
    __syncthreads();
    if (T.signal && tid == 0) {
      signal_add(&counters[T.dst]);
    }
  }
}

}  // namespace ps
