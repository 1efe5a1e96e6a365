// fold_est.cuh - exact sequential FP64 folds (sum_residuals, costmodel.cpp:36-40: s = 0; for i:
// s = fl(s + x_i)) spread over a whole CTA by estimated-start speculation.
//
// A sequential fold is a deterministic function of its start value, so a chain cut into K
// segments can fold segment k from a GUESSED start as soon as the guess is bit-identical to the
// true end of segment k-1; checking that is a comparison. The guess quality decides everything.
// The exact prefix sum P alone misses the chain's accumulated roundings by tens to thousands of
// ulps on long chains. Here the guess adds the estimated rounding error
//     D^ = sum_i e^_i,   e^_i = fl(s^_{i-1} + x_i) - (s^_{i-1} + x_i),   s^_{i-1} = fl(P_{i-1}),
// which is the true chain's error sum EXCEPT at steps where the partial sum grows into a higher
// binade (there the rounding depends on the running sum's last bit): while the binade does not
// grow, fl(s + x) - (s + x) depends only on x and the binade, not on which grid point s is. So
// fl(P + D^) lands within a few ulps of the true prefix even for chains of thousands of adds,
// and a warp of 32 candidate starts around it hits almost always.
//
// cta_fold_est (all threads of the CTA call it; every thread gets the result):
//   per super-segment of up to kFoldE * blockDim elements (sub-blocks of E <= kFoldE elements
//   per thread, held in registers and staged in shared memory):
//     1. every thread sums its sub-block; warp scan + warp totals -> the prefix P at every
//        sub-block start (anchored at the exact start of the super-segment; plain doubles, a few
//        ulps off - the window absorbs that, and a step's rounding error depends only on the
//        running sum's binade and grid, which a few ulps do not change)
//     2. every thread re-walks its sub-block as a rounded fold from its P, accumulating each
//        step's rounding error (TwoSum); warp totals -> D^ at every segment start
//     3. warp k folds segment k (32 sub-blocks) from the 32 doubles fl(P_k + D^_k) - 16 .. +15
//        ulp (warp 0 from the exact start); 16-byte broadcast loads from the stage
//     4. thread 0 walks the segments: the lane whose start is bit-identical to the true end of
//        the previous segment holds the next true end; a miss re-folds that segment alone from
//        the true value (the same adds, so the result is exact either way)
// Every add of the result is the reference's separately rounded one; the estimate only decides
// how much of the work is parallel.
#pragma once

#include "fs_common.cuh"

namespace fs {

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = fs_add(a, b);
  const double bb = fs_sub(s, a);
  e = fs_add(fs_sub(a, fs_sub(s, bb)), fs_sub(b, bb));
}
__device__ __forceinline__ long long dbl_ord(double x) {  // consecutive doubles -> consecutive ints
  const long long b = __double_as_longlong(x);
  return b >= 0 ? b : static_cast<long long>(0x8000000000000000ull) - b;
}
__device__ __forceinline__ double ord_dbl(long long o) {
  return __longlong_as_double(o >= 0 ? o : static_cast<long long>(0x8000000000000000ull) - o);
}
// Stage layout: thread t's sub-block (E <= EMAX elements) at t * (EMAX + 2): the two pad
// doubles keep the sub-block accesses conflict-free while the folds read runs of 16-byte words
// in order.
__host__ __device__ constexpr int fold_est_stage_doubles(int threads, int emax = 16) { return threads * (emax + 2); }
__host__ __device__ constexpr int fold_est_scratch_doubles(int threads) { return threads + 64 + 4 * (threads / 32) + 8; }

// Fold s through `nblk` whole sub-blocks of E elements (pitch P) starting at sb, then `tail`
// more elements; the next sub-block's loads are issued before the current adds.
template <int E, int P>
__device__ __forceinline__ double fold_run(const double* __restrict__ sb, int nblk, int tail, double s) {
  if (nblk > 0) {
    double2 a[E / 2];
#pragma unroll
    for (int u = 0; u < E / 2; ++u) a[u] = reinterpret_cast<const double2*>(sb)[u];
    for (int t = 0; t < nblk; ++t) {
      const double2* nx = reinterpret_cast<const double2*>(sb + min(t + 1, nblk - 1) * P);
      double2 b[E / 2];
#pragma unroll
      for (int u = 0; u < E / 2; ++u) b[u] = nx[u];
#pragma unroll
      for (int u = 0; u < E / 2; ++u) {
        s = fs_add(s, a[u].x);
        s = fs_add(s, a[u].y);
      }
#pragma unroll
      for (int u = 0; u < E / 2; ++u) a[u] = b[u];
    }
  }
  const double* tb = sb + nblk * P;
  for (int u = 0; u < tail; ++u) s = fs_add(s, tb[u]);
  return s;
}
template <int EMAX>
__device__ __forceinline__ double fold_run_e(int E, const double* __restrict__ sb, int nblk, int tail, double s) {
  constexpr int P = EMAX + 2;
  if (EMAX >= 16 && E == 16) return fold_run<(EMAX >= 16 ? 16 : 2), P>(sb, nblk, tail, s);
  if (EMAX >= 8 && E == 8) return fold_run<(EMAX >= 8 ? 8 : 2), P>(sb, nblk, tail, s);
  if (EMAX >= 4 && E == 4) return fold_run<(EMAX >= 4 ? 4 : 2), P>(sb, nblk, tail, s);
  return fold_run<2, P>(sb, nblk, tail, s);
}

// The chain is x_i = v[idx[i]] (idx == nullptr: x_i = v[i]), i < n, folded from `start`.
// stage: fold_est_stage_doubles(blockDim, EMAX) doubles of smem (16-byte aligned); scr:
// fold_est_scratch_doubles(blockDim) doubles. blockDim a multiple of 32, at most 1024; EMAX a
// power of two in [2, 16] (the longest sub-block per thread and super-segment).
// ctr (optional): [0] += segments resolved by a hit, [1] += segments re-folded after a miss.
template <int EMAX, typename CodeT, bool kRec>
__device__ __forceinline__ double cta_fold_est_impl(const double* __restrict__ v, const int32_t* __restrict__ idx, int n,
                                                    double start, const CodeT* __restrict__ codes,
                                                    double* __restrict__ out, double* __restrict__ stage,
                                                    CodeT* __restrict__ cst, double* __restrict__ scr,
                                                    unsigned long long* ctr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = blockDim.x, nw = T >> 5;
  double* res = scr;              // [T] chain results
  double* cen = scr + T;          // [32] candidate centre per segment
  double* wt = cen + 32;          // [2 nw] warp prefix-sum totals (double-double)
  double* dt = wt + 2 * nw;       // [nw] warp rounding-error totals
  double* bcast = dt + 2 * nw;    // [1]
  double* tst = bcast + 8;        // [32] (kRec) true start of every segment
  constexpr int kFoldE = EMAX, kFoldPitch = EMAX + 2;
  double S = start;  // true value at the current super-segment's start (every thread)
  int last_code = -1;  // (kRec) code of the element before the super-segment
#ifdef FOLD_EST_PROBE
  long long tq = clock64();
#define FE_MARK(k)                                                       \
  if (tid == 0 && ctr) {                                                 \
    const long long tn = clock64();                                      \
    atomicAdd(ctr + 2 + (k), static_cast<unsigned long long>(tn - tq)); \
    tq = tn;                                                             \
  }
#else
#define FE_MARK(k)
#endif
  for (int base = 0; base < n;) {
    const int rem = n - base;
    // sub-block length E: a power of two in [2, kFoldE], as small as covers the super-segment
    const int need = (min(rem, T * kFoldE) + T - 1) / T;
    const int E = need <= 2 ? 2 : need <= 4 ? 4 : need <= 8 ? 8 : kFoldE;
    const int lgE = __ffs(E) - 1;
    const int L = min(rem, T * E);
    const int b0 = min(tid * E, L), cnt = min(b0 + E, L) - b0;
    // gather, coalesced: element p = j * T + tid goes to its sub-block slot in the stage
    for (int j0 = 0; j0 < E; j0 += 8) {
      int ii[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int p = (j0 + u) * T + tid;
        ii[u] = base + min(p, L - 1);
      }
      if (idx) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (j0 + u < E) ii[u] = idx[ii[u]];
      }
      double xv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (j0 + u < E) xv[u] = v[ii[u]];
      if (kRec) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int p = (j0 + u) * T + tid;
          if (j0 + u < E && p < L) cst[p] = codes[ii[u]];
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int p = (j0 + u) * T + tid;
        if (j0 + u < E && p < L) stage[(p >> lgE) * kFoldPitch + (p & (E - 1))] = xv[u];
      }
    }
    __syncthreads();
    double x[kFoldE];
    {
      const double2* st2 = reinterpret_cast<const double2*>(stage + tid * kFoldPitch);
#pragma unroll
      for (int u = 0; u < kFoldE; u += 2)
        if (u < E) {
          const double2 a = st2[u >> 1];
          x[u] = a.x;
          x[u + 1] = a.y;
        }
    }
    FE_MARK(0)
    // 1. double-double sum of the sub-block; warp scan + warp totals -> exact prefix at b0
    double h = 0.0;
#pragma unroll
    for (int u = 0; u < kFoldE; ++u)
      if (u < cnt) h = fs_add(h, x[u]);
    double ih = h;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double oh = __shfl_up_sync(0xffffffffu, ih, o);
      if (lane >= o) ih = fs_add(oh, ih);
    }
    if (lane == 31) wt[2 * warp] = ih;
    double xh = __shfl_up_sync(0xffffffffu, ih, 1);
    if (lane == 0) xh = 0.0;
    FE_MARK(1)
    __syncthreads();
    double wh = lane < warp ? wt[2 * lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wh = fs_add(wh, __shfl_xor_sync(0xffffffffu, wh, o));
    const double seg_pre = fs_add(S, wh);
    FE_MARK(2)
    double d = 0.0;
    {
      double q = fs_add(seg_pre, xh);
#pragma unroll
      for (int u = 0; u < kFoldE; ++u) {
        if (u < cnt) {
          double y, err;
          two_sum(q, x[u], y, err);  // the rounding error of this step is -err
          d = fs_sub(d, err);
          q = y;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d = fs_add(d, __shfl_xor_sync(0xffffffffu, d, o));
    if (lane == 0) dt[warp] = d;
    FE_MARK(3)
    __syncthreads();
    double dw = lane < warp ? dt[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dw = fs_add(dw, __shfl_xor_sync(0xffffffffu, dw, o));
    const double est_k = fs_add(seg_pre, dw);
    FE_MARK(4)
    // 3. speculative folds: warp 0 from the exact start, warp k from est_k - 16 .. + 15 ulp
    const int seg0 = min(warp * 32 * E, L), seg_n = min(L - seg0, 32 * E);
    const double cstart = warp == 0 ? S : ord_dbl(dbl_ord(est_k) + (lane - 16));
    const double* sb = stage + warp * 32 * kFoldPitch;
    res[tid] = fold_run_e<EMAX>(E, sb, seg_n / E, seg_n % E, cstart);
    if (lane == 0) cen[warp] = est_k;
    FE_MARK(5)
    __syncthreads();
    FE_MARK(6)
    // 4. resolve segment by segment (thread 0)
    if (tid == 0) {
      double cur = res[0];
      unsigned long long hits = 0, misses = 0;
      if (kRec) tst[0] = S;
      for (int k = 1; k < nw; ++k) {
        const int a0 = k * 32 * E;
        if (a0 >= L) break;
        if (kRec) tst[k] = cur;
        const long long off = dbl_ord(cur) - (dbl_ord(cen[k]) - 16);
        if (off >= 0 && off < 32 && __double_as_longlong(ord_dbl(dbl_ord(cur))) == __double_as_longlong(cur)) {
          cur = res[32 * k + static_cast<int>(off)];
          ++hits;
        } else {  // re-fold segment k from the true value
          const int m = min(L - a0, 32 * E);
          cur = fold_run_e<EMAX>(E, stage + k * 32 * kFoldPitch, m / E, m % E, cur);
          ++misses;
        }
      }
      bcast[0] = cur;
      if (ctr) {
        atomicAdd(ctr, hits);
        atomicAdd(ctr + 1, misses);
      }
    }
    __syncthreads();
    if (kRec) {  // 5. every segment re-folded from its true start by one thread, recording
      // S_i (the fold of x_0..x_{i-1}) at out[c_{i-1}] wherever c_i != c_{i-1}
      const int a0 = warp * 32 * E;
      if (lane == 0 && a0 < L) {
        const int a1 = min(a0 + 32 * E, L);
        double cur = tst[warp];
        int prev = a0 == 0 ? last_code : static_cast<int>(cst[a0 - 1]);
        for (int i = a0; i < a1; ++i) {
          const int c = static_cast<int>(cst[i]);
          if (prev >= 0 && c != prev) out[prev] = cur;
          cur = fs_add(cur, stage[(i >> lgE) * kFoldPitch + (i & (E - 1))]);
          prev = c;
        }
      }
      last_code = static_cast<int>(cst[L - 1]);
      __syncthreads();
    }
    S = bcast[0];
    FE_MARK(7)
    base += L;
  }
#undef FE_MARK
  if (kRec && tid == 0 && n > 0) out[last_code] = S;
  return S;
}

// The chain's fold only (x_i = v[idx[i]], or v[i] when idx is nullptr), from `start`.
template <int EMAX = 16>
__device__ __noinline__ double cta_fold_est(const double* __restrict__ v, const int32_t* __restrict__ idx, int n,
                                            double start, double* __restrict__ stage, double* __restrict__ scr,
                                            unsigned long long* ctr = nullptr) {
  return cta_fold_est_impl<EMAX, uint8_t, false>(v, idx, n, start, nullptr, nullptr, stage, nullptr, scr, ctr);
}

// best_split's recorded fold (costmodel.cpp:50-69): the chain x_i = v[idx[i]] with codes
// c_i = codes[idx[i]] (non-decreasing along the list); out[c] = the fold of every element before
// the first element whose code differs from c, i.e. the left sum at each value boundary, and the
// last code's entry holds the full fold. cst: EMAX * blockDim CodeT of smem. Returns the fold.
template <int EMAX, typename CodeT>
__device__ __noinline__ double cta_fold_est_rec(const double* __restrict__ v, const int32_t* __restrict__ idx, int n,
                                                const CodeT* __restrict__ codes, double* __restrict__ out,
                                                double* __restrict__ stage, CodeT* __restrict__ cst,
                                                double* __restrict__ scr) {
  return cta_fold_est_impl<EMAX, CodeT, true>(v, idx, n, 0.0, codes, out, stage, cst, scr, nullptr);
}

}  // namespace fs
