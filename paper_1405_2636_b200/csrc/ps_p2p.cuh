// Peer-to-peer primitives of the multi-GPU factorization.
//
// The ranks' panel slabs and flag words are mapped into every process
// through CUDA IPC (NVLink peer memory on an NVSwitch box); cross-GPU data
// moves as loads from peer memory inside these kernels - no collective:
//
//   k_segment_add  fan-in of the subtree contributions:
//                  dst[off + i] += src[off + i] over a list of slab segments
//                  (the top panels this rank owns and `src`'s rank contributed
//                  to), src = a peer's slab.  The owner applies its peers one
//                  at a time in rank order: deterministic sums.
//   k_flag_signal  release-store of a 64-bit epoch value into this rank's flag
//                  word, after a system-scope fence (stream order makes every
//                  earlier kernel's slab writes complete before it runs).
//   k_flag_wait    one thread spins (acquire loads, system scope) until a peer's
//                  flag reaches a value; the stream's later work (pulls of the
//                  peer's panels, segment adds) is ordered after it.  Bounded:
//                  after `limit_ns` it raises a timeout word and returns, so a
//                  protocol error can never hang the device.
#pragma once
#include "ps_kernels.cuh"

namespace ps {

__global__ void __launch_bounds__(256)
k_segment_add(double* __restrict__ dst, const double* __restrict__ src, const i64* __restrict__ seg,
              const i64* __restrict__ start, int nseg, i64 total) {
  // seg[2k], seg[2k+1] = (slab offset, length) of segment k; start = prefix
  // sums of the lengths (nseg + 1 values).  Elements are flattened across the
  // segments; each thread handles pairs of consecutive elements.
  const i64 stride = (i64)gridDim.x * blockDim.x;
  int k = 0;
  for (i64 e = (i64)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    if (e >= start[k + 1] || e < start[k]) {  // binary search of the segment
      int lo = 0, hi = nseg - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (start[mid] <= e) lo = mid;
        else hi = mid - 1;
      }
      k = lo;
    }
    const i64 pos = seg[2 * k] + (e - start[k]);
    dst[pos] += __ldcv(src + pos);  // peer memory: no stale L1 line
  }
}

__global__ void k_flag_signal(unsigned long long* flag, unsigned long long value) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(value) : "memory");
}

__global__ void k_flag_wait(const unsigned long long* flag, unsigned long long value,
                            int* timeout, unsigned long long limit_ns) {
  const unsigned long long t0 = gtimer();
  while (true) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
    if (v >= value) break;
    if (gtimer() - t0 > limit_ns) {
      atomicExch(timeout, 1);
      break;
    }
    __nanosleep(256);
  }
  __threadfence_system();
}

}  // namespace ps
