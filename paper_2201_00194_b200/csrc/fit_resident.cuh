// fit_resident.cuh - the resident trainer: one CTA per family runs every boosting round (C1-C3)
// Part of the trainer translation unit: included once, by fit.cu only (shares its
// anonymous namespace, constants and helpers).
#pragma once


// ==========================================================================================
// resident trainer: one CTA per family runs EVERY boosting round of the fit in a single launch,
// with all per-row state in shared memory. For families of up to a few thousand rows (configs
// C1-C3) the multi-kernel round above is launch- and L2-latency-bound (~40 launches per round);
// here a round is ~30 block barriers. Same algorithm, same arithmetic, same tie handling.
// ==========================================================================================
#ifndef FS_RES_THREADS
#define FS_RES_THREADS 512
#endif
#include <cooperative_groups.h>

namespace fs {
namespace fit {
namespace {

constexpr int kResThreads = FS_RES_THREADS;
constexpr int kResWarps = kResThreads / 32;
constexpr int kPartE = 4;  // partition: consecutive order-0 entries per thread per chunk
constexpr int kSpecBufs = 4;  // warps whose single-candidate exact folds use the speculative split
// Resident histogram precision: FS_RES_LIMBS 3 = the multi-kernel's 62-bit fixed point (three
// 21-bit limbs per update); 2 = 39-bit fixed point (n * max|v| < 2^39, two limbs per update -
// a third fewer shared atomics; the screen bound widens with the quantum, so near-ties are
// re-evaluated exactly as before).
#ifndef FS_RES_LIMBS
#define FS_RES_LIMBS 3
#endif
constexpr int kResLimbs = FS_RES_LIMBS;
constexpr int kResBias = kResLimbs == 3 ? 62 : 40;  // u = v + 2^bias, count = round(U / 2^bias)
constexpr int kResMaxDepth = 7;  // node ids fit in uint8
constexpr int kResClusterMax = 4;  // CTAs per family by default (FAMSEER_RES_CLUSTER overrides)
constexpr int kResClusterMinRows = 1024;  // ... when the largest family has at least this many rows
// Histogram rings: level L's bins live in ring L % 3. With a cluster, the owner of a feature
// pushes its bins into the partners' ring as soon as it folds them; a partner last read that
// ring at level L - 3 (screen, decisions) or L - 2 (as the parent in the sibling subtraction),
// both before it arrived at level L - 1's exchange barrier, which the pusher has passed.
constexpr int kResRings = 3;

// distributed shared memory: the 32-bit shared::cluster address of the same offset in CTA rank
__device__ __forceinline__ uint32_t dsmem_addr(const void* p, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
               : "=r"(r)
               : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))), "r"(rank));
  return r;
}
__device__ __forceinline__ void dsmem_st(uint32_t a, long long v) {
  asm volatile("st.shared::cluster.s64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
__device__ __forceinline__ void dsmem_st(uint32_t a, int v) {
  asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

struct ResNode {
  int32_t n, seg, state, rep, bin, lc, wcount, build;
  int32_t eqf0, pad_;  // lowest window feature when the window may be one tie class, else -1
  double gain, value, total;
  unsigned long long lokey;
  unsigned long long absfix;
};

struct ResLayout {
  int ls, slots, cs;
  size_t codes, resid, pred, predv, targ, fix, node, ord0, scratch, hsum, hcnt, lbuf, nodes, win, items, rep, limb, sbuf, stage, binrep,
      vals, total;
};

__host__ __device__ inline size_t res_align(size_t v) { return (v + 15) & ~size_t(15); }

// groups: private histogram copies used while accumulating one node (threads own
// (feature, group) pairs, so no shared-memory atomics are needed).
__host__ __device__ inline ResLayout res_layout(int n, int nrep, int bins, int depth, int colh, bool pred_smem,
                                                bool pre_smem, int spec_bufs = 0) {
  ResLayout L;
  L.ls = depth > 0 ? (1 << (depth - 1)) : 1;
  L.slots = (1 << (depth + 1)) - 1;
  const size_t nr = nrep > 0 ? static_cast<size_t>(nrep) : 1;
  size_t o = 0;
  // codes [nrep][cs]: cs = 4 (mod 128) so the lanes reading one row's codes of consecutive
  // features fall in consecutive banks
  L.cs = ((n + 127) & ~127) + 4;
  L.codes = o;
  o = res_align(o + static_cast<size_t>(L.cs) * nr);
  L.resid = o;
  o = res_align(o + static_cast<size_t>(n) * 8);
  L.pred = o;  // presorted lists [nrep][n] as u16 (when pre_smem), else empty
  o = res_align(o + (pre_smem ? static_cast<size_t>(n) * nr * 2 : 0));
  L.predv = o;  // running predictions (when pred_smem), else they live in global memory
  o = res_align(o + (pred_smem ? static_cast<size_t>(n) * 8 : 0));
  L.targ = o;  // canonical targets and the root order-0 list, staged with the predictions
  o = res_align(o + (pred_smem ? static_cast<size_t>(n) * 10 : 0));
  L.fix = o;
  o = res_align(o + static_cast<size_t>(n) * 8);
  L.node = o;
  o = res_align(o + static_cast<size_t>(n));
  L.ord0 = o;
  o = res_align(o + static_cast<size_t>(n) * 2);
  L.scratch = o;
  o = res_align(o + static_cast<size_t>(n) * 2);
  L.hsum = o;  // three level rings (kResRings)
  o = res_align(o + static_cast<size_t>(kResRings) * L.ls * bins * 8);
  L.hcnt = o;
  o = res_align(o + static_cast<size_t>(kResRings) * L.ls * bins * 4);
  L.lbuf = o;
  o = res_align(o + static_cast<size_t>(L.ls) * bins * 8);
  L.nodes = o;
  o = res_align(o + static_cast<size_t>(L.slots) * sizeof(ResNode));
  L.win = o;
  o = res_align(o + static_cast<size_t>(L.ls) * nr * sizeof(WinRec));
  L.items = o;
  o = res_align(o + static_cast<size_t>(L.ls) * (nr + 1) * sizeof(int));
  L.rep = o;  // per rep: bin offset, bin count, lane-column offset; per level node: 4 x 16-bit limbs of sum |v|
  o = res_align(o + 3 * nr * sizeof(int) + static_cast<size_t>(L.ls) * 4 * 4);
  L.limb = o;  // lane-column limb histogram [3][colh][32] u32; the tie classes' phi tables
               // between histograms
  o = res_align(o + std::max<size_t>(static_cast<size_t>(3) * colh * 32 * 4, 8 * 512));
  L.sbuf = o;  // speculative exact folds: spec_bufs member lists of up to n rows (u16); during the
               // screen: (gain, bound) doubles and the left count per (node at level, bin)
  o = res_align(o + std::max(static_cast<size_t>(spec_bufs) * n * 2, static_cast<size_t>(L.ls) * bins * 20));
  L.stage = o;  // exact-fold staging: per warp 32 doubles + 32 codes
  o = res_align(o + static_cast<size_t>(kResWarps) * 32 * 9);
  L.binrep = o;  // feature (rep) of every bin, then this CTA's owned bins in order (histogram fold)
  o = res_align(o + static_cast<size_t>(bins) * 4);
  L.vals = o;  // threshold value of every bin + original feature of every rep (split records)
  o = res_align(o + static_cast<size_t>(bins) * 8 + nr * 4);
  L.total = o;
  return L;
}

// sum_residuals (costmodel.cpp:36-40) over a shared-memory index list, by ONE thread: the fold
// order is the list order and every add is rounded separately. Loads of the next 8 elements are
// issued before the current 8 adds, so the loop runs at the FP64 add latency instead of the
// load latency.
__device__ __forceinline__ double fold_seq(const double* __restrict__ v, const uint16_t* __restrict__ idx, int n) {
  double s = 0.0;
  int i = 0;
  if (n >= 8) {
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = v[idx[k]];
    for (i = 8; i + 8 <= n; i += 8) {
      double b[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) b[k] = v[idx[i + k]];
#pragma unroll
      for (int k = 0; k < 8; ++k) s = fs_add(s, a[k]);
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = b[k];
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) s = fs_add(s, a[k]);
  }
  for (; i < n; ++i) s = fs_add(s, v[idx[i]]);
  return s;
}

// Warp-collective exact sequential fold (sum_residuals, costmodel.cpp:36-40) of a long chain in
// about half the dependent-add latency, by speculation on the midpoint value:
//   1. every lane accumulates a strided part of x_0..x_{m-1} in double-double (TwoSum); the warp
//      reduction gives P ~= the EXACT prefix sum (the sequential result differs from it only by
//      the chain's accumulated roundings, typically a few ulps);
//   2. lane 0 folds x_0..x_{m-1} from 0.0 - the true S_m - while lanes 1..31 fold x_m..x_{n-1}
//      from the 31 doubles P-15ulp .. P+15ulp, all in the same loop;
//   3. the lane whose start is bit-identical to S_m holds the exact S_n (the fold is a function
//      of its start); if none is, the warp continues sequentially from S_m (same result, no
//      saving). Every add is still the reference's separately rounded sequential one.
__device__ __forceinline__ double fold_spec(const double* __restrict__ v, const uint16_t* __restrict__ idx, int n) {
  const int lane = threadIdx.x & 31;
  if (n < 192) return fold_seq(v, idx, n);
  const int m = n >> 1;
  double hi = 0.0, lo = 0.0;
  for (int i = lane; i < m; i += 32) {
    double s, e;
    two_sum(hi, v[idx[i]], s, e);
    hi = s;
    lo = fs_add(lo, e);
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double oh = __shfl_xor_sync(0xffffffffu, hi, o), ol = __shfl_xor_sync(0xffffffffu, lo, o);
    double s, e;
    two_sum(hi, oh, s, e);
    hi = s;
    lo = fs_add(fs_add(lo, ol), e);
  }
  const double P = fs_add(hi, lo);
  const double start = lane == 0 ? 0.0 : ord_dbl(dbl_ord(P) + (lane - 16));
  const uint16_t* seq = idx + (lane == 0 ? 0 : m);
  const int len = lane == 0 ? m : n - m;  // n - m is m or m + 1
  double s = start;
  {
    int i = 0;
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = v[seq[k]];
    for (i = 8; i + 8 <= m; i += 8) {
      double b[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) b[k] = v[seq[i + k]];
#pragma unroll
      for (int k = 0; k < 8; ++k) s = fs_add(s, a[k]);
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = b[k];
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) s = fs_add(s, a[k]);
    for (; i < len; ++i) s = fs_add(s, v[seq[i]]);
  }
  const double Sm = __shfl_sync(0xffffffffu, s, 0);
  const unsigned hit = __ballot_sync(0xffffffffu, lane != 0 && __double_as_longlong(start) == __double_as_longlong(Sm));
  if (hit) return __shfl_sync(0xffffffffu, s, __ffs(hit) - 1);
  double t = Sm;  // speculation missed: finish the chain from the true midpoint
  for (int i = m; i < n; ++i) t = fs_add(t, v[idx[i]]);
  return t;
}



// The fold chain s = start + x_0 + x_1 + ... (separately rounded) over a CONTIGUOUS array x[0..n): 16-byte loads (two elements per shared load),
// eight elements in flight ahead of the dependent adds.
__device__ __forceinline__ double fold_c(const double* __restrict__ x, int n, double s) {
  int i = 0;
  if ((reinterpret_cast<uintptr_t>(x) & 15) && n > 0) s = fs_add(s, x[i++]);  // align to 16 bytes
  const double2* x2 = reinterpret_cast<const double2*>(x + i);
  const int n2 = (n - i) >> 1;
  int k = 0;
  if (n2 >= 4) {
    double2 a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] = x2[u];
    for (k = 4; k + 4 <= n2; k += 4) {
      double2 b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) b[u] = x2[k + u];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        s = fs_add(s, a[u].x);
        s = fs_add(s, a[u].y);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] = b[u];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      s = fs_add(s, a[u].x);
      s = fs_add(s, a[u].y);
    }
  }
  for (; k < n2; ++k) {
    const double2 a = x2[k];
    s = fs_add(s, a.x);
    s = fs_add(s, a.y);
  }
  for (i += 2 * n2; i < n; ++i) s = fs_add(s, x[i]);
  return s;
}

// fold_spec over a contiguous array (warp-collective; lane 0 exact first half, lanes 1..31 the
// second half from P - 15 .. P + 15 ulp)
__device__ __forceinline__ double fold_spec_c(const double* __restrict__ x, int n) {
  const int lane = threadIdx.x & 31;
  if (n < 192) return fold_c(x, n, 0.0);
  const int m = n >> 1;
  double hi = 0.0, lo = 0.0;
  for (int i = lane; i < m; i += 32) {
    double s, e;
    two_sum(hi, x[i], s, e);
    hi = s;
    lo = fs_add(lo, e);
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double oh = __shfl_xor_sync(0xffffffffu, hi, o), ol = __shfl_xor_sync(0xffffffffu, lo, o);
    double s, e;
    two_sum(hi, oh, s, e);
    hi = s;
    lo = fs_add(fs_add(lo, ol), e);
  }
  const double P = fs_add(hi, lo);
  const double start = lane == 0 ? 0.0 : ord_dbl(dbl_ord(P) + (lane - 16));
  // one call with per-lane arguments (two call sites would run the halves one after the other)
  const double s = fold_c(lane == 0 ? x : x + m, lane == 0 ? m : n - m, start);
  const double Sm = __shfl_sync(0xffffffffu, s, 0);
  const unsigned hit = __ballot_sync(0xffffffffu, lane != 0 && __double_as_longlong(start) == __double_as_longlong(Sm));
  if (hit) return __shfl_sync(0xffffffffu, s, __ffs(hit) - 1);
  return fold_c(x + m, n - m, Sm);  // speculation missed: finish from the true midpoint
}

// kClu: launched as a thread-block cluster (several CTAs per family); false compiles the
// single-CTA shape without any cluster arithmetic.
template <bool kClu>
__global__ void __launch_bounds__(kResThreads, 1) fit_resident_kernel(
    const FamDesc* __restrict__ fam, FamState* __restrict__ st, const int* __restrict__ fam_list, int Dp,
    const uint8_t* __restrict__ codes_c, const double* __restrict__ target_c, const double* __restrict__ base,
    const int32_t* __restrict__ ord, const int32_t* __restrict__ ord_root, const int32_t* __restrict__ rep_orig,
    const int32_t* __restrict__ rep_nb, const int32_t* __restrict__ rep_boff, const double* __restrict__ vals,
    const int32_t* __restrict__ cle, const int32_t* __restrict__ canon, const double* __restrict__ x, int d,
    TreeRec* __restrict__ trees, double* __restrict__ ebuf, int max_trees, int slots_g,
    unsigned long long* __restrict__ ctr, int pred_smem, double* __restrict__ pred_g, int pre_smem, int spec_bufs) {
  extern __shared__ __align__(16) unsigned char sm[];
  // Optional thread-block cluster of cl_n CTAs per family (FAMSEER_RES_CLUSTER): every CTA holds
  // the whole per-row state and runs every phase identically, except the histogram, whose
  // features are dealt round-robin (feature j -> CTA j % cl_n); after each level's histograms
  // the CTAs pull each other's bins through distributed shared memory. Only CTA rank 0 writes
  // global results.
  cooperative_groups::cluster_group cluster = cooperative_groups::this_cluster();
  const int cl_n = kClu ? static_cast<int>(cluster.num_blocks()) : 1;
  const int cl_r = kClu ? static_cast<int>(cluster.block_rank()) : 0;
  const bool lead = cl_r == 0;
  __shared__ unsigned long long s_red[32];
  __shared__ int s_wsum[32];
  __shared__ int s_nitems, s_ctot;
  __shared__ unsigned long long s_cnt[3];  // screened splits, exact nodes, exact folds
  __shared__ unsigned long long s_why[4];  // exact-node reasons
#ifdef FS_RES_HIST_PROBE
  __shared__ unsigned long long s_probe[4];
  if (threadIdx.x < 4) s_probe[threadIdx.x] = 0;
#endif
  const int f = fam_list[blockIdx.x / cl_n];
  const FamDesc fd = fam[f];
  const int n = fd.n, nrep = fd.nrep, bins = fd.bins, depth = fd.depth;
  const int colh = nrep > 0 ? col_height(nrep, rep_nb + fd.rep0, nullptr) : 1;
  const ResLayout Lo = res_layout(n, nrep, bins, depth, colh, pred_smem != 0, pre_smem != 0, spec_bufs);
  uint16_t* s_sbuf = reinterpret_cast<uint16_t*>(sm + Lo.sbuf);
  uint8_t* s_codes = sm + Lo.codes;  // [nrep][cs]
  const int cs = Lo.cs;
  uint32_t* s_limb = reinterpret_cast<uint32_t*>(sm + Lo.limb);  // [3][colh][32]
  int* s_cofs = reinterpret_cast<int*>(sm + Lo.rep) + 2 * (nrep > 0 ? nrep : 1);       // [nrep]
  uint32_t* s_absl = reinterpret_cast<uint32_t*>(s_cofs + (nrep > 0 ? nrep : 1));      // [level node][4]
  double* s_cand = reinterpret_cast<double*>(sm + Lo.sbuf);  // [level node][bin] x (g, delta), screen only
  int* s_clc = reinterpret_cast<int*>(s_cand + 2 * static_cast<size_t>(Lo.ls) * bins);  // left counts
  uint16_t* s_binrep = reinterpret_cast<uint16_t*>(sm + Lo.binrep);
  uint16_t* s_own = s_binrep + bins;  // bins of this CTA's histogram features (j % cl_n == cl_r)
  __shared__ int s_nown;
  double* s_vals = reinterpret_cast<double*>(sm + Lo.vals);
  int* s_rorig = reinterpret_cast<int*>(s_vals + bins);
  __shared__ int s_neq;
  // phase timers (CTA 0, thread 0): where a round's cycles go (fs_device_counters [4..15])
  __shared__ long long s_ph[12];
  // Phase clock: __syncthreads() is BAR.SYNC.DEFER_BLOCKING - a warp only blocks at the first
  // dependent instruction after it - so a bare clock read right after a barrier would bill the
  // barrier wait to the NEXT phase. The read takes a register input loaded from shared memory
  // after the barrier (the load cannot complete before the barrier does); memory clobber keeps
  // the compiler from moving work across it.
  __shared__ int s_clkdep;
  auto clk = [&]() {
    long long t;
    const int dep = *reinterpret_cast<volatile int*>(&s_clkdep);
    asm volatile("add.s32 %1, %1, 0;\n\tmov.u64 %0, %%clock64;" : "=l"(t) : "r"(dep) : "memory");
    return t;
  };
  if (threadIdx.x == 0) s_clkdep = 0;
  long long t_prev = clock64();
  if (threadIdx.x < 12) s_ph[threadIdx.x] = 0;
#define RES_PHASE(i)                        \
  do {                                      \
    if (tid == 0) {                         \
      const long long t_ = clk();           \
      s_ph[i] += t_ - t_prev;               \
      t_prev = t_;                          \
    }                                       \
  } while (0)
  double* s_resid = reinterpret_cast<double*>(sm + Lo.resid);
  // running predictions: shared memory when they fit, else global (L2-resident); the targets
  // and the root order-0 list are staged with them (read every round)
  double* s_pred = pred_smem ? reinterpret_cast<double*>(sm + Lo.predv) : pred_g + fd.pos0;
  const double* s_targ = target_c + fd.pos0;
  const int32_t* g_ordr = ord_root + fd.pos0;
  uint16_t* s_ordr = nullptr;
  if (pred_smem) {
    double* t = reinterpret_cast<double*>(sm + Lo.targ);
    s_ordr = reinterpret_cast<uint16_t*>(t + n);
    for (int p = threadIdx.x; p < n; p += kResThreads) {
      t[p] = target_c[fd.pos0 + p];
      s_ordr[p] = static_cast<uint16_t>(ord_root[fd.pos0 + p]);
    }
    s_targ = t;
  }
  uint16_t* s_pre = reinterpret_cast<uint16_t*>(sm + Lo.pred);  // presorted lists, if staged
  const int32_t* g_pre = ord + fd.ord0;
  auto pre_at = [&](int j, int i) -> int {
    return pre_smem ? static_cast<int>(s_pre[static_cast<size_t>(j) * n + i]) : g_pre[static_cast<size_t>(j) * n + i];
  };
  long long* s_fix = reinterpret_cast<long long*>(sm + Lo.fix);
  uint8_t* s_node = sm + Lo.node;
  uint16_t* s_ord0 = reinterpret_cast<uint16_t*>(sm + Lo.ord0);
  uint16_t* s_scr = reinterpret_cast<uint16_t*>(sm + Lo.scratch);
  long long* s_hsum = reinterpret_cast<long long*>(sm + Lo.hsum);
  int* s_hcnt = reinterpret_cast<int*>(sm + Lo.hcnt);
  double* s_lbuf = reinterpret_cast<double*>(sm + Lo.lbuf);
  ResNode* s_nodes = reinterpret_cast<ResNode*>(sm + Lo.nodes);
  WinRec* s_win = reinterpret_cast<WinRec*>(sm + Lo.win);
  int* s_items = reinterpret_cast<int*>(sm + Lo.items);
  int* s_repb = reinterpret_cast<int*>(sm + Lo.rep);
  int* s_repn = s_repb + (nrep > 0 ? nrep : 1);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ls = Lo.ls, slots = Lo.slots;
  unsigned long long c_hist_rows = 0;
  if (tid < 3) s_cnt[tid] = 0;
  if (tid < 4) s_why[tid] = 0;

  for (int i = tid; i < n * nrep; i += kResThreads) {
    const int p = i / nrep, j = i - p * nrep;
    s_codes[j * cs + p] = codes_c[(fd.pos0 + p) * Dp + j];
  }
  for (int j = tid; j < nrep; j += kResThreads) {
    s_repb[j] = rep_boff[fd.rep0 + j];
    s_repn[j] = rep_nb[fd.rep0 + j];
    for (int b = 0; b < rep_nb[fd.rep0 + j]; ++b) s_binrep[rep_boff[fd.rep0 + j] + b] = static_cast<uint16_t>(j);
    s_rorig[j] = rep_orig[fd.rep0 + j];
  }
  for (int b = tid; b < bins; b += kResThreads) s_vals[b] = vals[fd.bin0 + b];
  if (tid == 0 && nrep > 0) col_height(nrep, rep_nb + fd.rep0, s_cofs);
  const double b0 = base[f];
  for (int p = tid; p < n; p += kResThreads) s_pred[p] = b0;
  if (pre_smem)
    for (int i = tid; i < n * nrep; i += kResThreads) s_pre[i] = static_cast<uint16_t>(g_pre[i]);
  // limb cells start zeroed; every fold zeroes the cells it reads (and the tie classes' phi
  // tables, which overlay them, are zeroed again), so no zeroing pass per histogram
  for (int i = tid; i < 3 * colh * 32; i += kResThreads) s_limb[i] = 0;
  if (tid == 0) {
    int no = 0;
    for (int j = cl_r; j < nrep; j += cl_n)
      for (int b = 0; b < rep_nb[fd.rep0 + j]; ++b) s_own[no++] = static_cast<uint16_t>(rep_boff[fd.rep0 + j] + b);
    s_nown = no;
  }
  __syncthreads();

  int ntrees = 0;
  bool have_resid = false;
  for (int round = 0; round < fd.trees; ++round) {
    // ---- residuals (costmodel.cpp:204-206), fixed point, per-round reset ----------------
    // (from round 1 on, the previous round's prediction/MSE pass already wrote the residuals,
    // their max |r| per warp and the row resets)
    if (!have_resid) {
      unsigned long long mx = 0;
      for (int p = tid; p < n; p += kResThreads) {
        const double r = fs_sub(s_targ[p], s_pred[p]);
        s_resid[p] = r;
        mx = max(mx, static_cast<unsigned long long>(__double_as_longlong(fabs(r))));
        s_node[p] = 0;
        s_ord0[p] = s_ordr ? s_ordr[p] : static_cast<uint16_t>(g_ordr[p]);
      }
      for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (lane == 0) s_red[warp] = mx;
    }
    if (cl_n > 1) cluster.sync();  // the partners finished pulling last round's histograms
    for (int s = tid; s < slots; s += kResThreads) {
      ResNode z;
      memset(&z, 0, sizeof z);
      if (s == 0) {  // the root's plan (level_plan_kernel, level 0)
        z.n = n;
        if (nrep > 0 && node_needs_split(fd, 0, n)) z.build = 1;
        else z.state = kNodeLeaf;
      }
      s_nodes[s] = z;
    }
    if (tid < 4) s_absl[tid] = 0;  // the root's sum |v| limb counters
    TreeRec* tr = trees + fd.tree0 + static_cast<int64_t>(ntrees) * slots_g;
    for (int s = tid; s < slots_g && lead; s += kResThreads) {
      TreeRec tz;
      memset(&tz, 0, sizeof tz);
      tr[s] = tz;
    }
    __syncthreads();
    // every thread reduces the per-warp maxima itself (broadcast loads): no serial section and
    // no extra barrier
    int shift;
    {
      unsigned long long m = 0;
#pragma unroll
      for (int w = 0; w < kResThreads / 32; ++w) m = max(m, s_red[w]);
      shift = kResLimbs == 3 ? fix_shift(m, n) : fix_shift(m, n) - 22;  // n*|v| < 2^61 resp. 2^39
    }
    const double scale = ldexp(1.0, -shift);
    for (int p = tid; p < n; p += kResThreads) s_fix[p] = __double2ll_rn(ldexp(s_resid[p], shift));
    __syncthreads();
      RES_PHASE(0);

    for (int level = 0; level <= depth; ++level) {
      const int first = (1 << level) - 1, nl = 1 << level;
      // (the level's plan - leaf / build flags - was made when its parents split: split records)
      RES_PHASE(1);
      if (level == depth || nrep == 0) break;
      const int ring = level % kResRings;
      long long* hs = s_hsum + static_cast<size_t>(ring) * ls * bins;
      int* hc = s_hcnt + static_cast<size_t>(ring) * ls * bins;
      // ---- histograms of every directly built node of the level, one node at a time, in lane
      // columns (col_height): every lane of a warp adds into its own bank column, so a 32-lane
      // shared atomic is one wavefront. A row adds the three 21-bit limbs of u = v + 2^62 per
      // feature with native 32-bit shared atomics; every kAtomSub rows the copies' limb sums are
      // folded exactly into the node's 64-bit histogram (see hist_build_atomic_kernel for the
      // arithmetic; the first fold overwrites). sum |v| (the screen bound) is a per-thread
      // 64-bit sum (< 2^61 by the fixed-point shift), warp-reduced, added as 16-bit limbs.
      {
        // this CTA's features: j = jl * cl_n + cl_r (all of them without a cluster)
        const int nown = (nrep - cl_r + cl_n - 1) / cl_n;
        const int rpw = nown <= 32 ? 32 / max(nown, 1) : 1;  // rows per warp step
        const int hjl = nown <= 32 ? lane % max(nown, 1) : lane;
        const int hj = hjl * cl_n + cl_r;
        const int hm = nown <= 32 ? lane / max(nown, 1) : 0;
        const bool hact = nown <= 32 ? nown > 0 && hm < rpw : true;
        for (int k = 0; k < nl; ++k) {
          ResNode& nd = s_nodes[first + k];
          if (nd.build != 1) continue;
          const int nv = nd.n;
          const uint16_t* rows = s_ord0 + nd.seg;
          for (int sub0 = 0; sub0 < nv; sub0 += kAtomSub) {
            const int q_end = min(nv, sub0 + kAtomSub);
            unsigned long long asum = 0;
#ifdef FS_RES_HIST_PROBE
            const long long tp0 = clock64();
#endif
            if (hact) {
              if (nown <= 32) {
                const uint8_t* hcode = s_codes + static_cast<size_t>(hj) * cs;
                uint32_t* colp = s_limb + lane;
#pragma unroll 4
                for (int q = sub0 + warp * rpw + hm; q < q_end; q += kResWarps * rpw) {
                  const int p = rows[q];
                  const long long v = s_fix[p];
                  const uint64_t u = static_cast<uint64_t>(v) + (1ull << kResBias);
                  uint32_t* c = colp + hcode[p] * 32;
                  atomicAdd(c, static_cast<uint32_t>(u) & kLimbMask);
                  atomicAdd(c + colh * 32, static_cast<uint32_t>(u >> 21) & kLimbMask);
                  if (kResLimbs == 3) atomicAdd(c + 2 * colh * 32, static_cast<uint32_t>(u >> 42));
                  if (hjl == 0) asum += static_cast<unsigned long long>(v < 0 ? -v : v);
                }
              } else {
                for (int q = sub0 + warp; q < q_end; q += kResWarps) {
                  const int p = rows[q];
                  const long long v = s_fix[p];
                  const uint64_t u = static_cast<uint64_t>(v) + (1ull << kResBias);
                  const uint32_t l0 = static_cast<uint32_t>(u) & kLimbMask;
                  const uint32_t l1 = static_cast<uint32_t>(u >> 21) & kLimbMask;
                  const uint32_t l2 = static_cast<uint32_t>(u >> 42);
                  for (int j = lane; j < nrep; j += 32) {
                    uint32_t* c = s_limb + lane + (s_cofs[j] + s_codes[static_cast<size_t>(j) * cs + p]) * 32;
                    atomicAdd(c, l0);
                    atomicAdd(c + colh * 32, l1);
                    if (kResLimbs == 3) atomicAdd(c + 2 * colh * 32, l2);
                  }
                  if (lane == 0) asum += static_cast<unsigned long long>(v < 0 ? -v : v);
                }
              }
            }
#ifdef FS_RES_HIST_PROBE
            if (lane == 0 && blockIdx.x == 0) {
              const unsigned long long dt = static_cast<unsigned long long>(clock64() - tp0);
              atomicMax(&s_probe[0], dt);
              atomicAdd(&s_probe[1], dt);
              if (warp == 0) atomicAdd(&s_probe[3], 1ull);
            }
#endif
            for (int o = 16; o > 0; o >>= 1) asum += __shfl_xor_sync(0xffffffffu, asum, o);
            if (lane == 0 && asum) {
#pragma unroll
              for (int t = 0; t < 4; ++t) atomicAdd(s_absl + 4 * k + t, static_cast<uint32_t>(asum >> (16 * t)) & 0xFFFFu);
            }
            __syncthreads();
#ifdef FS_RES_HIST_SPLIT
            RES_PHASE(2);  // accumulate
#endif
            long long* hk = hs + static_cast<size_t>(k) * bins;
            int* ck = hc + static_cast<size_t>(k) * bins;
            // four threads per owned bin, each summing a quarter of the bin's lane copies (the
            // cells are zeroed as they are read), combined by two xor shuffles within the group
            const int nown_b = s_nown;
            for (int i4 = tid; i4 < 4 * nown_b; i4 += kResThreads) {
              const int i = s_own[i4 >> 2], sub = i4 & 3;
              const int j = s_binrep[i], b = i - s_repb[j];
              unsigned long long ulo = 0, uhi = 0;  // 128-bit partial sum of u over the copies
              auto add_cell = [&](uint32_t* c) {
                const unsigned __int128 v = static_cast<unsigned __int128>(c[0]) +
                                            (static_cast<unsigned __int128>(c[colh * 32]) << 21) +
                                            (kResLimbs == 3 ? static_cast<unsigned __int128>(c[2 * colh * 32]) << 42 : 0);
                c[0] = 0;
                c[colh * 32] = 0;
                if (kResLimbs == 3) c[2 * colh * 32] = 0;
                const unsigned __int128 t = ((static_cast<unsigned __int128>(uhi) << 64) | ulo) + v;
                ulo = static_cast<unsigned long long>(t);
                uhi = static_cast<unsigned long long>(t >> 64);
              };
              if (nown <= 32) {
                for (int m = sub; m < rpw; m += 4) add_cell(s_limb + b * 32 + j / cl_n + m * nown);
              } else if (sub == 0) {
                add_cell(s_limb + (s_cofs[j] + b) * 32 + (j & 31));
              }
              // lanes of this warp inside the loop bound (a prefix: whole groups of four)
              const int lim = 4 * nown_b - (i4 - lane);
              const unsigned grp = lim >= 32 ? 0xffffffffu : (1u << lim) - 1u;
#pragma unroll
              for (int o = 1; o < 4; o <<= 1) {
                const unsigned long long olo = __shfl_xor_sync(grp, ulo, o), ohi = __shfl_xor_sync(grp, uhi, o);
                const unsigned __int128 t = ((static_cast<unsigned __int128>(uhi) << 64) | ulo) +
                                            ((static_cast<unsigned __int128>(ohi) << 64) | olo);
                ulo = static_cast<unsigned long long>(t);
                uhi = static_cast<unsigned long long>(t >> 64);
              }
              if (sub == 0) {
                const unsigned __int128 U = (static_cast<unsigned __int128>(uhi) << 64) | ulo;
                const uint64_t cnt =
                    static_cast<uint64_t>((U + (static_cast<unsigned __int128>(1) << (kResBias - 1))) >> kResBias);
                const long long hv =
                    static_cast<long long>(static_cast<uint64_t>(U - (static_cast<unsigned __int128>(cnt) << kResBias)));
                const long long hsv = (sub0 == 0 ? 0ll : hk[i]) + hv;
                const int hcv = (sub0 == 0 ? 0 : ck[i]) + static_cast<int>(cnt);
                hk[i] = hsv;
                ck[i] = hcv;
              }
            }
            if (tid == 0) {  // the node's sum |v| over its chunks so far (counters zeroed by the plan)
              unsigned long long add = 0;
#pragma unroll
              for (int t = 0; t < 4; ++t) add += static_cast<unsigned long long>(s_absl[4 * k + t]) << (16 * t);
              nd.absfix = add;
              if (sub0 == 0) c_hist_rows += nv;
              if (level > 0 && sub0 + kAtomSub >= nv) {  // the derived sibling's sum |v|
                const int s = first + k, sib = (s & 1) ? s + 1 : s - 1;
                if (s_nodes[sib].build == 2) s_nodes[sib].absfix = s_nodes[(s - 1) >> 1].absfix - add;
              }
            }
            __syncthreads();
#ifdef FS_RES_HIST_SPLIT
            RES_PHASE(3);  // limb fold billed to "derive"
#endif
          }
        }
        // prefix form: the owner turns each of its features' bins of every directly built node
        // into inclusive prefix sums over the feature's bins (warp per (node, feature), lanes
        // over bins) and pushes them to the partners. Sums and counts are exact integers and
        // prefix is linear: siblings derive prefix from prefix, the screen reads a candidate's
        // left sum / count and the node total in O(1), the exact decision needs no count scan.
        // The owner also derives the sibling (build 2) of every built node for its features by
        // exact subtraction of prefix sums (parent - built; the parent's prefix of an owned
        // feature is always local) and pushes it too, so no CTA derives after the exchange.
        const int nown_f = (nrep - cl_r + cl_n - 1) / cl_n;
        const int pring = (level + kResRings - 1) % kResRings;
        const long long* hpar = s_hsum + static_cast<size_t>(pring) * ls * bins;
        const int* cpar = s_hcnt + static_cast<size_t>(pring) * ls * bins;
        const int pfirst = level > 0 ? (1 << (level - 1)) - 1 : 0;
        for (int it = warp; it < nl * nown_f; it += kResWarps) {
          const int k = it / nown_f, j = (it - k * nown_f) * cl_n + cl_r;
          const int s = first + k;
          if (s_nodes[s].build != 1) continue;
          const int sib = level > 0 ? ((s & 1) ? s + 1 : s - 1) : -1;
          const bool dsib = sib >= 0 && s_nodes[sib].build == 2;
          const int bo = s_repb[j];
          long long* h = hs + static_cast<size_t>(k) * bins + bo;
          int* c = hc + static_cast<size_t>(k) * bins + bo;
          long long* ho = dsib ? hs + static_cast<size_t>(sib - first) * bins + bo : nullptr;
          int* co = dsib ? hc + static_cast<size_t>(sib - first) * bins + bo : nullptr;
          const size_t pb = dsib ? static_cast<size_t>(((s - 1) >> 1) - pfirst) * bins + bo : 0;
          const int nb = s_repn[j];
          long long hcar = 0;
          int ccar = 0;
          for (int b0 = 0; b0 < nb; b0 += 32) {
            const int b = b0 + lane;
            const long long hv = warp_incl_scan(b < nb ? h[b] : 0ll, lane) + hcar;
            const int cv = warp_incl_scan(b < nb ? c[b] : 0, lane) + ccar;
            if (b < nb) {
              h[b] = hv;
              c[b] = cv;
              long long ov = 0;
              int oc = 0;
              if (dsib) {
                ov = hpar[pb + b] - hv;
                oc = cpar[pb + b] - cv;
                ho[b] = ov;
                co[b] = oc;
              }
              if (kClu)
                for (int r = 1; r < cl_n; ++r) {
                  const int rr = (cl_r + r) % cl_n;
                  dsmem_st(dsmem_addr(h + b, rr), hv);
                  dsmem_st(dsmem_addr(c + b, rr), cv);
                  if (dsib) {
                    dsmem_st(dsmem_addr(ho + b, rr), ov);
                    dsmem_st(dsmem_addr(co + b, rr), oc);
                  }
                }
            }
            hcar = __shfl_sync(0xffffffffu, hv, 31);
            ccar = __shfl_sync(0xffffffffu, cv, 31);
          }
        }
        // the partners' pushed prefix sums visible (arrive.release / wait.acquire)
        if (cl_n > 1) cluster.sync();
        else __syncthreads();
      }
      RES_PHASE(2);
      // (siblings were derived by the feature owners, above)
      RES_PHASE(3);
      // ---- screen: thread per candidate (level node k, bin). Pass 0: the feature's prefix
      // count / sum up to the bin by a short loop over its bins, the screened gain and its bound
      // (cached), the node's max lower bound (segmented warp max, then one 64-bit atomicMax per
      // node segment of the warp). Pass 1: window membership {hi >= LO, hi > 0} with 32-bit
      // atomics: per (node, feature) window count and largest left count; the candidate's data
      // is written racily, which is exact whenever the feature has ONE window candidate - the
      // only case that reads it.
      {
        const int ncand = nl * bins;
        for (int pass = 0; pass < 2; ++pass) {
          for (int c0 = 0; c0 < ncand; c0 += kResThreads) {
            const int ci = c0 + tid;
            int k = ci < ncand ? ci / bins : nl;
            const int bi = ci - k * bins;
            bool live = k < nl;
            ResNode* ndp = live ? &s_nodes[first + k] : nullptr;
            if (live && (ndp->state != 0 || ndp->build == 0)) live = false;
            int j = 0, b = 0, ic = 0;
            double lo = -INFINITY;
            if (live) {
              j = s_binrep[bi];
              b = bi - s_repb[j];
            }
            if (pass == 0) {
              if (live) {
                const int nb = s_repn[j];
                const long long* h = hs + static_cast<size_t>(k) * bins + s_repb[j];
                const int* c = hc + static_cast<size_t>(k) * bins + s_repb[j];
                if (b == 0) {
                  WinRec z;
                  memset(&z, 0, sizeof z);
                  z.best_bin = -1;
                  s_win[k * nrep + j] = z;
                }
                const long long is = h[b], ts = h[nb - 1];  // prefix form
                ic = c[b];
                const int cb = ic - (b > 0 ? c[b - 1] : 0);
                s_clc[ci] = ic;
                const int nv = ndp->n;
                if (cb > 0 && ic < nv) {
                  const double S = static_cast<double>(ndp->absfix) * scale * (1.0 + 1e-12);
                  double g, hi;
                  screen_gain(is, ts, ic, nv, scale, S, g, lo, hi);
                  s_cand[2 * ci] = g;
                  s_cand[2 * ci + 1] = hi - g;
                } else {
                  s_cand[2 * ci] = NAN;
                }
              }
              // segmented (by node) warp max of the lower bounds; lanes' nodes are non-decreasing
              const int kk = live ? k : -1;
              double m = lo;
              for (int o = 1; o < 32; o <<= 1) {
                const double om = __shfl_up_sync(0xffffffffu, m, o);
                const int ok_ = __shfl_up_sync(0xffffffffu, kk, o);
                if (lane >= o && ok_ == kk) m = fmax(m, om);
              }
              const int knext = __shfl_down_sync(0xffffffffu, kk, 1);
              if (kk >= 0 && (lane == 31 || knext != kk) && m > -INFINITY) atomicMax(&ndp->lokey, lo_key(m));
            } else if (live) {
              const double g = s_cand[2 * ci];
              if (!isnan(g)) {
                const double dl = s_cand[2 * ci + 1];
                const double hi = g + dl;
                if (hi >= lo_from_key(ndp->lokey) && hi > 0.0) {
                  WinRec& w = s_win[k * nrep + j];
                  ic = s_clc[ci];
                  atomicAdd(&w.count, 1);
                  atomicMax(&w.maxlc, ic);
                  atomicAdd(&ndp->wcount, 1);
                  w.flag = 1;
                  w.best_g = g;
                  w.best_lo = g - dl;
                  w.best_bin = b;
                  w.best_lc = ic;
                }
              }
            }
          }
          __syncthreads();
#ifdef FS_RES_SCREEN_SPLIT
          RES_PHASE(pass == 0 ? 4 : 3);  // A/B probe: pass 1 billed to "derive"
#endif
        }
      }
      RES_PHASE(4);
      // ---- tie classes: a window whose candidates (one per feature, equal left counts) come
      // from features whose presorted orders coincide on the node's rows has one reference
      // gain for all of them (identical folds), so the lowest feature wins by strict > without
      // any fold. Check order equivalence against the lowest window feature in parallel.
      if (tid == 0) s_neq = 0;
      __syncthreads();
      // warp per node, lanes over its features: the window is one candidate per feature, all at
      // the same left count, and the lowest window feature's lower bound is positive
      for (int k = warp; k < nl; k += kResWarps) {
        ResNode& nd = s_nodes[first + k];
        if (!(nd.state == 0 && nd.build != 0 && nd.wcount >= 2)) {
          if (lane == 0) nd.eqf0 = -1;
          continue;
        }
        const WinRec* w = s_win + k * nrep;
        int f0 = -1;
        for (int j0 = 0; j0 < nrep && f0 < 0; j0 += 32) {
          const unsigned m = __ballot_sync(0xffffffffu, j0 + lane < nrep && w[j0 + lane].flag);
          if (m) f0 = j0 + __ffs(m) - 1;
        }
        const int lc0 = f0 >= 0 ? w[f0].best_lc : -1;
        bool bad = false;
        for (int j0 = 0; j0 < nrep; j0 += 32) {
          const int j = j0 + lane;
          const bool fl = j < nrep && w[j].flag;
          bad |= __any_sync(0xffffffffu, fl && (w[j].count != 1 || w[j].best_lc != lc0));
        }
        const bool ok = !bad && f0 >= 0 && w[f0].best_lo > 0.0;
        if (lane == 0) nd.eqf0 = ok ? f0 : -1;
        if (!ok) continue;
        for (int j0 = 0; j0 < nrep; j0 += 32) {
          const int j = j0 + lane;
          const bool put = j < nrep && j > f0 && w[j].flag;
          const unsigned m = __ballot_sync(0xffffffffu, put);
          int base = 0;
          if (lane == 0 && m) base = atomicAdd(&s_neq, __popc(m));
          base = __shfl_sync(0xffffffffu, base, 0);
          if (put) s_items[base + __popc(m & ((1u << lane) - 1u))] = (first + k) << 16 | j;
        }
      }
      __syncthreads();
      // Order equivalence of g with f0 on the node's rows <=> the map code_f0 -> code_g over
      // those rows is a function that is strictly increasing (ties align and the stable sorts
      // by (code, canonical position) then coincide). Checked without any ordered scan: phi[a] =
      // the g code of some row with f0 code a (racy plain stores), then every row must agree
      // with phi and phi must increase over the present a. Rows come from the node's order-0
      // segment in any order; items are batched through the (free) limb scratch.
      {
        uint16_t* phi = reinterpret_cast<uint16_t*>(s_limb);
        const int cap = static_cast<int>((Lo.stage - Lo.limb) / 512);  // items of 256 u16 (>= 8)
        const int neq = s_neq;
        for (int b0 = 0; b0 < neq; b0 += cap) {
          const int nb_items = min(cap, neq - b0);
          for (int i = tid; i < nb_items * 256; i += kResThreads) phi[i] = 0xFFFFu;
          if (tid < nb_items) {
            const int s = s_items[b0 + tid] >> 16, g = s_items[b0 + tid] & 0xFFFF;
            s_win[(s - first) * nrep + g].eq = 1;
          }
          __syncthreads();
          for (int pass = 0; pass < 2; ++pass) {
            for (int q = 0; q < nb_items; ++q) {
              const int s = s_items[b0 + q] >> 16, g = s_items[b0 + q] & 0xFFFF;
              const ResNode& nd = s_nodes[s];
              const uint8_t* cf = s_codes + static_cast<size_t>(nd.eqf0) * cs;
              const uint8_t* cg = s_codes + static_cast<size_t>(g) * cs;
              uint16_t* ph = phi + q * 256;
              bool bad = false;
              for (int i = tid; i < nd.n; i += kResThreads) {
                const int pr = s_ord0[nd.seg + i];
                if (pass == 0) ph[cf[pr]] = cg[pr];
                else bad |= ph[cf[pr]] != cg[pr];
              }
              if (pass == 1 && bad) s_win[(s - first) * nrep + g].eq = 0;
            }
            __syncthreads();
          }
          // phi strictly increasing over the present f0 codes (warp per item)
          for (int q = warp; q < nb_items; q += kResThreads / 32) {
            const int s = s_items[b0 + q] >> 16, g = s_items[b0 + q] & 0xFFFF;
            const int nb = s_repn[s_nodes[s].eqf0];
            const uint16_t* ph = phi + q * 256;
            int carry = -1;
            bool bad = false;
            for (int a0 = 0; a0 < nb; a0 += 32) {
              const int a = a0 + lane;
              const int v = a < nb ? ph[a] : 0xFFFF;
              const bool present = v != 0xFFFF;
              const unsigned m = __ballot_sync(0xffffffffu, present);
              const unsigned lt = m & ((1u << lane) - 1u);
              int pv = __shfl_sync(0xffffffffu, v, lt ? 31 - __clz(lt) : 0);
              if (!lt) pv = carry;
              if (present && pv >= 0 && v <= pv) bad = true;
              if (m) carry = __shfl_sync(0xffffffffu, v, 31 - __clz(m));
            }
            if (__any_sync(0xffffffffu, bad) && lane == 0) s_win[(s - first) * nrep + g].eq = 0;
          }
          __syncthreads();
        }
        // the phi tables overlaid the limb cells: zero them again for the next histograms (the
        // decide phase's barriers order these stores before any accumulate)
        if (neq > 0)
          for (int i = tid; i < min(3 * colh * 32, min(cap, neq) * 128); i += kResThreads) s_limb[i] = 0;
      }
      RES_PHASE(5);
      // ---- decide (decide_kernel) ------------------------------------------------------------
      if (tid == 0) s_nitems = 0;
      __syncthreads();
      // warp per node, lanes over the node's features (window records read in parallel)
      for (int k = warp; k < nl; k += kResWarps) {
        ResNode& nd = s_nodes[first + k];
        if (nd.state != 0 || nd.build == 0) continue;
        const WinRec* w = s_win + k * nrep;
        if (nd.wcount == 0) {
          if (lane == 0) nd.state = kNodeLeaf;
          continue;
        }
        int pick = -1, nflag = 0, f0 = -1;
        bool multi = false, notall = false;
        for (int j0 = 0; j0 < nrep; j0 += 32) {
          const int j = j0 + lane;
          const bool fl = j < nrep && w[j].flag;
          const unsigned m = __ballot_sync(0xffffffffu, fl);
          nflag += __popc(m);
          if (m && f0 < 0) f0 = j0 + __ffs(m) - 1;
          multi |= __any_sync(0xffffffffu, fl && w[j].count > 1);
          notall |= __any_sync(0xffffffffu, fl && j > nd.eqf0 && !w[j].eq);
        }
        if (nd.wcount == 1) {
          if (f0 >= 0 && w[f0].best_lo > 0.0) pick = f0;
        } else if (nd.eqf0 >= 0 && !notall) {
          pick = nd.eqf0;
        }
        if (pick >= 0) {
          if (lane == 0) {
            nd.state = kNodeSplit;
            nd.rep = pick;
            nd.bin = w[pick].best_bin;
            nd.gain = w[pick].best_g;
            nd.lc = w[pick].best_lc;
            atomicAdd(&s_cnt[0], 1ull);
          }
          continue;
        }
        // exact re-evaluation: why the screen could not decide (diagnostics, device counters)
        int why = 3;  // sign of the only candidate uncertain
        if (nd.wcount >= 2) {
          const int lc0 = w[f0].best_lc;
          bool diff = false;
          for (int j0 = 0; j0 < nrep; j0 += 32) {
            const int j = j0 + lane;
            diff |= __any_sync(0xffffffffu, j < nrep && w[j].flag && w[j].best_lc != lc0);
          }
          why = multi ? 0 : diff ? 1 : 2;  // several candidates on a feature / partitions / orders
        }
        int base = 0;
        if (lane == 0) {
          nd.state = kNodeExact;
          atomicAdd(&s_cnt[1], 1ull);
          atomicAdd(&s_why[why], 1ull);
          base = atomicAdd(&s_nitems, nflag + 1);
          s_items[base] = (first + k) << 16 | 0xFFFF;
          atomicAdd(&s_cnt[2], static_cast<unsigned long long>(nflag + 1));
        }
        base = __shfl_sync(0xffffffffu, base, 0) + 1;
        for (int j0 = 0; j0 < nrep; j0 += 32) {
          const int j = j0 + lane;
          const bool fl = j < nrep && w[j].flag;
          const unsigned m = __ballot_sync(0xffffffffu, fl);
          if (fl) s_items[base + __popc(m & ((1u << lane) - 1u))] = (first + k) << 16 | j;
          base += __popc(m);
        }
      }
      __syncthreads();
      RES_PHASE(6);
      // ---- reference-order folds (exact_kernel) ------------------------------------------------
      // Warp per item. The node total is one fold over its order-0 segment. A window feature's
      // fold walks the feature's presorted list: lanes test 32 entries for node membership, the
      // members are compacted (ballot rank) into the warp's staging slots, and lane 0 folds them
      // in list order, recording the left sum at every value boundary - but only up to the
      // largest window left count (candidates beyond it cannot win, costmodel.cpp:65 strict >).
      {
        double* st_v = reinterpret_cast<double*>(sm + Lo.stage) + warp * 32;
        uint8_t* st_c = sm + Lo.stage + static_cast<size_t>(kResThreads / 32) * 32 * 8 + warp * 32;
        for (int it = warp; it < s_nitems; it += kResThreads / 32) {
          const int s = s_items[it] >> 16, j = s_items[it] & 0xFFFF;
          ResNode& nd = s_nodes[s];
          const int nv = nd.n;
          if (j == 0xFFFF) {  // every lane runs the same chain (broadcast loads): no divergence
            const double t = fold_spec(s_resid, s_ord0 + nd.seg, nv);
            if (lane == 0) nd.total = t;
            continue;
          }
          const int need = s_win[(s - first) * nrep + j].maxlc;
          double* out = s_lbuf + static_cast<size_t>(s - first) * bins + s_repb[j];
          const uint8_t* cj = s_codes + static_cast<size_t>(j) * cs;
          if (warp < spec_bufs && s_win[(s - first) * nrep + j].count == 1) {
            // one window candidate: only L at its left count is needed. Compact the node's
            // members of the feature's presorted list (in list order) into this warp's buffer,
            // then fold them with the speculative midpoint split (fold_spec).
            uint16_t* buf = s_sbuf + static_cast<size_t>(warp) * n;
            int got = 0;
            int p_nx = lane < n ? pre_at(j, lane) : 0;
            for (int i0 = 0; i0 < n && got < need; i0 += 32) {
              const int i = i0 + lane;
              const int p = p_nx;
              p_nx = i + 32 < n ? pre_at(j, i + 32) : 0;
              const bool mem = i < n && s_node[p] == s;
              const unsigned m = __ballot_sync(0xffffffffu, mem);
              const int dst = got + __popc(m & ((1u << lane) - 1u));
              if (mem && dst < need) buf[dst] = static_cast<uint16_t>(p);
              got += __popc(m);
            }
            __syncwarp();
            const double L = fold_spec(s_resid, buf, need);
            if (lane == 0) out[s_win[(s - first) * nrep + j].best_bin] = L;
            continue;
          }
          double left = 0.0;
          int prev = -1, seen = 0;
          int p_next = lane < n ? pre_at(j, lane) : 0;
          for (int i0 = 0; i0 < n && seen < need; i0 += 32) {
            const int i = i0 + lane;
            const int p = p_next;
            p_next = i + 32 < n ? pre_at(j, i + 32) : 0;
            const bool mem = i < n && s_node[p] == s;
            const unsigned m = __ballot_sync(0xffffffffu, mem);
            if (mem) {
              const int dst = __popc(m & ((1u << lane) - 1u));
              st_v[dst] = s_resid[p];
              st_c[dst] = cj[p];
            }
            __syncwarp();
            const int cnt = min(__popc(m), need - seen);
#pragma unroll 8
            for (int t = 0; t < cnt; ++t) {  // all lanes fold identically (broadcast loads)
              const int c = st_c[t];
              if (c != prev && prev >= 0 && lane == 0) out[prev] = left;
              left = fs_add(left, st_v[t]);
              prev = c;
            }
            seen += cnt;
            __syncwarp();
          }
          if (lane == 0 && prev >= 0) out[prev] = left;
        }
      }
      __syncthreads();
      RES_PHASE(7);
      // ---- exact decision (exact_decide_kernel): warp per node, lanes over a window feature's
      // bins; the reference's strict > over (feature asc, threshold asc) = first occurrence of
      // the maximum, so the warp reduction keeps the largest gain and, on equal gains, the
      // earliest (feature, bin).
      for (int k = warp; k < nl; k += kResWarps) {
        ResNode& nd = s_nodes[first + k];
        if (nd.state != kNodeExact) continue;
        const WinRec* w = s_win + k * nrep;
        const int nv = nd.n;
        const double T = nd.total;
        const double parent = fs_div(fs_mul(T, T), static_cast<double>(nv));
        double best = 0.0;
        int bj = -1, bbin = -1, blc = 0;
        // features with one window candidate (the common case): lane per feature, the only
        // candidate that can win on that feature is its window candidate (best_bin / best_lc:
        // every other candidate's gain is provably below LO, costmodel.cpp:65 strict >)
        for (int j0 = 0; j0 < nrep; j0 += 32) {
          const int j = j0 + lane;
          if (j < nrep && w[j].flag && w[j].count == 1) {
            const int cum = w[j].best_lc;
            const double L = s_lbuf[static_cast<size_t>(k) * bins + s_repb[j] + w[j].best_bin];
            const double R = fs_sub(T, L);
            const double a = fs_div(fs_mul(L, L), static_cast<double>(cum));
            const double r = fs_div(fs_mul(R, R), static_cast<double>(nv - cum));
            const double g = fs_sub(fs_add(a, r), parent);
            if (g > best) {  // first candidate of this lane: no earlier (feature, bin) to beat
              best = g;
              bj = j;
              bbin = w[j].best_bin;
              blc = cum;
            }
          }
        }
        for (int j = 0; j < nrep; ++j) {
          if (!w[j].flag || w[j].count == 1) continue;
          const int* c = hc + static_cast<size_t>(k) * bins + s_repb[j];
          const double* lb = s_lbuf + static_cast<size_t>(k) * bins + s_repb[j];
          const int nb = s_repn[j], lim = w[j].maxlc;
          int carry = 0;
          for (int b0 = 0; b0 < nb && carry < lim; b0 += 32) {
            const int b = b0 + lane;
            const int cum = b < nb ? c[b] : 0;  // prefix form
            const int cb = b < nb ? cum - (b > 0 ? c[b - 1] : 0) : 0;
            if (cb > 0 && cum < nv && cum <= lim) {  // folds stop at the last window candidate
              const double L = lb[b];
              const double R = fs_sub(T, L);
              const double a = fs_div(fs_mul(L, L), static_cast<double>(cum));
              const double r = fs_div(fs_mul(R, R), static_cast<double>(nv - cum));
              const double g = fs_sub(fs_add(a, r), parent);
              // a lane's candidates do not arrive in (feature, bin) order: full tie-break
              if (g > best || (g == best && bj >= 0 && (j < bj || (j == bj && b < bbin)))) {
                best = g;
                bj = j;
                bbin = b;
                blc = cum;
              }
            }
            carry = c[min(b0 + 31, nb - 1)];
          }
        }
        for (int o = 16; o > 0; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
          const int obin = __shfl_xor_sync(0xffffffffu, bbin, o);
          const int olc = __shfl_xor_sync(0xffffffffu, blc, o);
          const bool take = oj >= 0 && (bj < 0 || ob > best || (ob == best && (oj < bj || (oj == bj && obin < bbin))));
          if (take) {
            best = ob;
            bj = oj;
            bbin = obin;
            blc = olc;
          }
        }
        if (lane == 0) {
          if (bj < 0) {
            nd.state = kNodeLeaf;
          } else {
            nd.state = kNodeSplit;
            nd.rep = bj;
            nd.bin = bbin;
            nd.gain = best;
            nd.lc = blc;
          }
        }
      }
      __syncthreads();
      // ---- split records: threshold, tree record, children and their plan -----------------------
      if (level + 1 < depth && tid < 8 * nl) s_absl[tid] = 0;  // the next level's sum |v| counters
      if (tid < nl) {
        const int s = first + tid;
        ResNode& nd = s_nodes[s];
        if (nd.state == kNodeSplit) {
          const int j = nd.rep;
          const int orig = s_rorig[j];
          double thr = s_vals[s_repb[j] + nd.bin];
          if (thr == 0.0 && fd.negz) {  // +0.0 / -0.0 share a bin: the last left element's own value
            const int32_t* L = ord + fd.ord0 + static_cast<int64_t>(j) * n;
            for (int i = cle[fd.bin0 + s_repb[j] + nd.bin] - 1; i >= 0; --i)
              if (s_node[L[i]] == s) {
                thr = x[(fd.row0 + canon[fd.pos0 + L[i]]) * d + orig];
                break;
              }
          }
          TreeRec r;
          r.kind = kNodeSplit;
          r.feature = orig;
          r.threshold = thr;
          r.value = 0.0;
          r.gain = nd.gain;
          r.rep = j;
          r.bin = nd.bin;
          if (lead) tr[s] = r;
          ResNode& a = s_nodes[2 * s + 1];
          ResNode& b = s_nodes[2 * s + 2];
          a.n = nd.lc;
          a.seg = nd.seg;
          b.n = nd.n - nd.lc;
          b.seg = nd.seg + nd.lc;
          // the children's plan (level_plan_kernel): a child that cannot split is a leaf; when
          // either can, the smaller is built directly (1) and the other derived (2)
          const bool na = nrep > 0 && node_needs_split(fd, level + 1, a.n);
          const bool nb2 = nrep > 0 && node_needs_split(fd, level + 1, b.n);
          if (!na) a.state = kNodeLeaf;
          if (!nb2) b.state = kNodeLeaf;
          if (na || nb2) {
            ResNode& small = a.n <= b.n ? a : b;
            ResNode& big = a.n <= b.n ? b : a;
            small.build = 1;
            big.build = 2;
          }
        }
      }
      __syncthreads();
      RES_PHASE(8);
      // ---- stable partition of every split node's order-0 segment (costmodel.cpp:94-105 for
      // list 0) in one sweep over the whole list: a block-wide exclusive scan of "goes left"
      // flags; its value at the node's segment start turns it into the rank inside the node
      // (segments are contiguous). Elements are read once into registers (kPartE consecutive per
      // thread per chunk), scattered into the other order buffer, and the buffers swap.
      {
        int nsplit = 0;
        for (int k = 0; k < nl; ++k) nsplit += s_nodes[first + k].state == kNodeSplit;
        if (nsplit) {
          int base = 0;  // exclusive scan carried across chunks (uniform)
          for (int c0 = 0; c0 < n; c0 += kResThreads * kPartE) {
            int pe[kPartE], ve[kPartE];
            bool le[kPartE];
            int cnt = 0;
#pragma unroll
            for (int e = 0; e < kPartE; ++e) {
              const int i = c0 + tid * kPartE + e;
              pe[e] = 0;
              ve[e] = -1;
              le[e] = false;
              if (i < n) {
                pe[e] = s_ord0[i];
                const int v = s_node[pe[e]];
                if (s_nodes[v].state == kNodeSplit) {
                  ve[e] = v;
                  le[e] = s_codes[static_cast<size_t>(s_nodes[v].rep) * cs + pe[e]] <= s_nodes[v].bin;
                }
              }
              cnt += le[e];
            }
            const int incl = warp_incl_scan(cnt, lane);
            if (lane == 31) s_wsum[warp] = incl;
            __syncthreads();
            if (warp == 0) {
              const int wv = lane < kResWarps ? s_wsum[lane] : 0;
              const int inc = warp_incl_scan(wv, lane);
              s_wsum[lane] = inc - wv;
              if (lane == 31) s_ctot = inc;
            }
            __syncthreads();
            int P = base + s_wsum[warp] + incl - cnt;  // exclusive scan at this thread's first element
            const int chunk_total = s_ctot;
            int Pe[kPartE];
#pragma unroll
            for (int e = 0; e < kPartE; ++e) {
              Pe[e] = P;
              P += le[e];
              const int i = c0 + tid * kPartE + e;
              if (ve[e] >= 0 && i == s_nodes[ve[e]].seg) s_nodes[ve[e]].pad_ = Pe[e];
            }
            __syncthreads();
#pragma unroll
            for (int e = 0; e < kPartE; ++e) {
              const int i = c0 + tid * kPartE + e;
              if (i >= n) continue;
              if (ve[e] < 0) {
                s_scr[i] = static_cast<uint16_t>(pe[e]);
                continue;
              }
              const ResNode& nd = s_nodes[ve[e]];
              const int lrank = Pe[e] - nd.pad_;
              const int dst = le[e] ? nd.seg + lrank : nd.seg + nd.lc + (i - nd.seg) - lrank;
              s_scr[dst] = static_cast<uint16_t>(pe[e]);
              s_node[pe[e]] = static_cast<uint8_t>(le[e] ? 2 * ve[e] + 1 : 2 * ve[e] + 2);
            }
            base += chunk_total;
            __syncthreads();
          }
          uint16_t* t = s_ord0;
          s_ord0 = s_scr;
          s_scr = t;
        }
      }
      RES_PHASE(9);
    }
      RES_PHASE(1);
    // ---- leaves (leaf_kernel): reference-order total / n, prediction update ------------------
    // residuals in order-0 list order, contiguous (every leaf's rows are a contiguous segment of
    // the list): the chains read two elements per 16-byte load instead of two loads per element.
    // The fixed-point residuals' buffer is free after the last histogram.
    double* s_gath = reinterpret_cast<double*>(s_fix);
    for (int i = tid; i < n; i += kResThreads) s_gath[i] = s_resid[s_ord0[i]];
    __syncthreads();
    for (int s = warp; s < slots; s += kResWarps) {
      ResNode& nd = s_nodes[s];
      if (nd.state != kNodeLeaf || nd.n == 0) continue;
      if (s > 0 && s_nodes[(s - 1) >> 1].state != kNodeSplit) continue;
      const int nv = nd.n;
      const double sum = fold_spec_c(s_gath + nd.seg, nv);  // warp-collective
      const double value = fs_div(sum, static_cast<double>(nv));
      if (lane == 0) {
        nd.value = value;
        TreeRec r;
        r.kind = kNodeLeaf;
        r.feature = -1;
        r.threshold = 0.0;
        r.value = value;
        r.gain = 0.0;
        r.rep = -1;
        r.bin = 0;
        if (lead) tr[s] = r;
      }
    }
    __syncthreads();
      RES_PHASE(10);
    // ---- prediction update (costmodel.cpp:88-90: pred += lr * leaf value, every row through
    // its final leaf slot, all threads) fused with the MSE (:215-220); commit or early stop
    // (:212 - the update happens before the reference's stop test too)
    const bool stop = s_nodes[0].state == kNodeLeaf && s_nodes[0].value == 0.0;  // uniform (smem)
    // e of this round in the family's block of ebuf ([rounds][n] at pos0 * max_trees): the
    // sequential MSE fold over canonical rows runs after the fit (mse_fold_kernel)
    double* eb = ebuf + fd.pos0 * max_trees + static_cast<int64_t>(ntrees) * n;
    unsigned long long mx = 0;
    for (int p = tid; p < n; p += kResThreads) {
      const double pr = fs_add(s_pred[p], fs_mul(fd.lr, s_nodes[s_node[p]].value));
      s_pred[p] = pr;
      const double e = fs_sub(s_targ[p], pr);  // = the next round's residual (costmodel.cpp:204-206)
      if (lead && !stop) eb[p] = e;
      s_resid[p] = e;
      mx = max(mx, static_cast<unsigned long long>(__double_as_longlong(fabs(e))));
      s_node[p] = 0;
      s_ord0[p] = s_ordr ? s_ordr[p] : static_cast<uint16_t>(g_ordr[p]);
    }
    if (stop) break;
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) s_red[warp] = mx;
    have_resid = true;
    __syncthreads();
    ++ntrees;
    __syncthreads();
      RES_PHASE(11);
  }
  if (cl_n > 1) cluster.sync();  // no CTA leaves while a partner may still read its shared memory
  if (tid == 0 && lead) {
    st[f].ntrees = ntrees;
    st[f].active = 0;
    st[f].screened += s_cnt[0];
    st[f].exact += s_cnt[1];
    atomicAdd(ctr + kCtrHistRows, c_hist_rows);
    atomicAdd(ctr + kCtrHistBytes, c_hist_rows * (static_cast<unsigned long long>(nrep) + 12ull));
    atomicAdd(ctr + kCtrExactChains, s_cnt[2]);
    atomicAdd(ctr + kCtrExactNodes, s_cnt[1]);
    if (blockIdx.x == 0)
      for (int i = 0; i < 12; ++i) atomicAdd(ctr + kCtrPhase0 + i, static_cast<unsigned long long>(s_ph[i]));
    for (int i = 0; i < 4; ++i) atomicAdd(ctr + kCtrPhase0 + 12 + i, s_why[i]);
#ifdef FS_RES_HIST_PROBE
    if (blockIdx.x == 0)
      for (int i = 0; i < 4; ++i) atomicAdd(ctr + kCtrProbe + i, s_probe[i]);
#endif
  }
}

}  // namespace
}  // namespace fit
}  // namespace fs
