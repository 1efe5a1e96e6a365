// Kernel (3): the boosting trainer - fit (costmodel.cpp:152-222) for F families in one call.
// Design and bit-exactness argument: fit.cuh. Phases:
//   prep    distinct values + codes per feature, feature dedup, canonical row order
//           (costmodel.cpp:161-173), per-feature presorts (:193-201), base (:185-188)
//   rounds  residual -> fixed point -> per level: histograms (smaller child built, sibling by
//           exact subtraction), screen, exact reference-order re-evaluation where needed,
//           stable partition of the order-0 list -> leaves (reference-order totals) ->
//           prediction update -> commit / early stop (:212) -> MSE (:215-220)
// The host only launches; no host<->device synchronisation happens inside the boosting loop.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <climits>
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <numeric>
#include <vector>

#include "fit.cuh"

namespace fs {
void launch_featurize(fs_device* dev, const fs_spaces* sp, int64_t n, const int32_t* space_of_d,
                      const int32_t* assign_d, int32_t pad, double* out_d);
}  // namespace fs

namespace fs {
namespace fit {
namespace {

// ------------------------------------------------------------------------------------------
// small device helpers
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t value_key(double v) {  // order-preserving, -0.0 == +0.0
  uint64_t b = static_cast<uint64_t>(__double_as_longlong(v));
  if (b == 0x8000000000000000ull) b = 0;
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_value(uint64_t k) {
  const uint64_t b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double(static_cast<long long>(b));
}
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}
__device__ __forceinline__ uint64_t lo_key(double v) {  // order-preserving key for atomicMax
  const uint64_t b = static_cast<uint64_t>(__double_as_longlong(v));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double lo_from_key(uint64_t k) {
  const uint64_t b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double(static_cast<long long>(b));
}

__device__ __forceinline__ int family_of_pos(const FamDesc* fam, int F, int64_t p) {
  int lo = 0, hi = F;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (fam[mid].pos0 <= p) lo = mid;
    else hi = mid;
  }
  return lo;
}

// Block-level stable counting sort by an 8-bit digit (blockDim == kSortThreads).
// out[...] = in indices ordered by (digit, position in `in`). Returns false (and writes nothing)
// when every element has the same digit, so callers can skip the pass.
struct SortSmem {
  int cnt[256];
  int tot[256];
  int wc[32 * 256];
  int uniform;
};

template <class In, class Digit>
__device__ bool stable_digit_pass(In in, int32_t* __restrict__ out, int n, Digit digit, SortSmem& sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 256; i += blockDim.x) sm.cnt[i] = 0;
  __syncthreads();
  for (int i = tid; i < n; i += blockDim.x) atomicAdd(&sm.cnt[digit(in(i))], 1);
  __syncthreads();
  if (tid == 0) sm.uniform = n == 0 || sm.cnt[digit(in(0))] == n;
  __syncthreads();
  if (sm.uniform) return false;
  if (warp == 0) {  // exclusive scan of 256 counts
    int v[8], s = 0;
    for (int k = 0; k < 8; ++k) {
      v[k] = sm.cnt[lane * 8 + k];
      s += v[k];
    }
    int incl = s;
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    int run = incl - s;
    for (int k = 0; k < 8; ++k) {
      sm.cnt[lane * 8 + k] = run;
      run += v[k];
    }
  }
  __syncthreads();
  for (int t0 = 0; t0 < n; t0 += blockDim.x) {
    const int i = t0 + tid;
    const bool valid = i < n;
    const int idx = valid ? in(i) : 0;
    const int dg = valid ? digit(idx) : 256;
    const unsigned peers = __match_any_sync(0xffffffffu, dg);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    if (valid && rank == 0) sm.wc[warp * 256 + dg] = __popc(peers);
    __syncthreads();
    if (tid < 256) {
      int run = 0;
      for (int w = 0; w < 32; ++w) {
        const int c = sm.wc[w * 256 + tid];
        sm.wc[w * 256 + tid] = run;
        run += c;
      }
      sm.tot[tid] = run;
    }
    __syncthreads();
    if (valid) out[sm.cnt[dg] + sm.wc[warp * 256 + dg] + rank] = idx;
    __syncthreads();
    if (tid < 256) {
      for (int w = 0; w < 32; ++w) sm.wc[w * 256 + tid] = 0;
      sm.cnt[tid] += sm.tot[tid];
    }
    __syncthreads();
  }
  return true;
}

__device__ void sort_smem_init(SortSmem& sm) {
  for (int i = threadIdx.x; i < 32 * 256; i += blockDim.x) sm.wc[i] = 0;
  __syncthreads();
}

// ------------------------------------------------------------------------------------------
// prep 1: distinct values and codes per (family, feature) - hash path (<= 256 distinct)
// ------------------------------------------------------------------------------------------
constexpr int kHashSlots = 512;

__global__ void __launch_bounds__(256) distinct_small_kernel(const double* __restrict__ x, int d,
                                                             const FamDesc* __restrict__ fam,
                                                             uint16_t* __restrict__ codes_all,
                                                             double* __restrict__ vals_all,
                                                             int32_t* __restrict__ nb_all,
                                                             uint64_t* __restrict__ hash_all, uint32_t* err,
                                                             int* __restrict__ negz) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* tab = reinterpret_cast<uint64_t*>(smem);                 // [32][512]
  uint64_t* sorted = tab + 32 * kHashSlots;                          // [32][256]
  int* cnt = reinterpret_cast<int*>(sorted + 32 * kSmallBins);       // [32]
  int* ovf = cnt + 32;                                               // [32]
  unsigned long long* hsh = reinterpret_cast<unsigned long long*>(ovf + 32);  // [32]
  const FamDesc fd = fam[blockIdx.y];
  const int j0 = blockIdx.x * 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 32 * kHashSlots; i += blockDim.x) tab[i] = 0;
  if (tid < 32) {
    cnt[tid] = 0;
    ovf[tid] = 0;
    hsh[tid] = 0;
  }
  __syncthreads();
  const int j = j0 + lane;
  const bool has = j < d;
  bool nonfinite = false, negzero = false;
  if (has) {
    uint64_t* t = tab + lane * kHashSlots;
    for (int r = warp; r < fd.n; r += 8) {
      const double v = x[(fd.row0 + r) * d + j];
      if (!isfinite(v)) {
        nonfinite = true;
        continue;
      }
      negzero |= v == 0.0 && signbit(v);
      if (ovf[lane]) continue;
      const uint64_t k = value_key(v);
      uint32_t h = static_cast<uint32_t>(mix64(k)) & (kHashSlots - 1);
      for (int probe = 0; probe < kHashSlots; ++probe) {
        const uint64_t prev = atomicCAS(reinterpret_cast<unsigned long long*>(t + h), 0ull,
                                        static_cast<unsigned long long>(k));
        if (prev == 0) {
          if (atomicAdd(&cnt[lane], 1) >= kSmallBins) ovf[lane] = 1;
          break;
        }
        if (prev == k) break;
        h = (h + 1) & (kHashSlots - 1);
        if (probe == kHashSlots - 1) ovf[lane] = 1;
      }
    }
  }
  if (__any_sync(0xffffffffu, nonfinite) && lane == 0) atomicOr(err, kErrNonFiniteFit);
  if (__any_sync(0xffffffffu, negzero) && lane == 0) atomicOr(negz + blockIdx.y, 1);
  __syncthreads();
  // rank every present key by counting smaller keys (<= 256 per feature)
  for (int f = warp; f < 32; f += 8) {
    if (j0 + f >= d || ovf[f]) continue;
    const uint64_t* t = tab + f * kHashSlots;
    for (int s = lane; s < kHashSlots; s += 32) {
      const uint64_t k = t[s];
      if (!k) continue;
      int rank = 0;
      for (int o = 0; o < kHashSlots; ++o) {
        const uint64_t q = t[o];
        rank += (q != 0 && q < k);
      }
      sorted[f * kSmallBins + rank] = k;
    }
  }
  __syncthreads();
  for (int f = warp; f < 32; f += 8) {
    if (j0 + f >= d) continue;
    const int64_t fj = static_cast<int64_t>(blockIdx.y) * d + j0 + f;
    if (lane == 0) nb_all[fj] = ovf[f] ? -1 : cnt[f];
    if (!ovf[f])
      for (int i = lane; i < cnt[f]; i += 32) vals_all[fj * kSmallBins + i] = key_value(sorted[f * kSmallBins + i]);
  }
  // codes: binary search in the sorted distinct keys
  if (has && !ovf[lane]) {
    const uint64_t* sk = sorted + lane * kSmallBins;
    const int m = cnt[lane];
    uint64_t hacc = 0;
    for (int r = warp; r < fd.n; r += 8) {
      const double v = x[(fd.row0 + r) * d + j];
      if (!isfinite(v)) continue;
      const uint64_t k = value_key(v);
      int lo = 0, hi = m - 1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (sk[mid] < k) lo = mid + 1;
        else hi = mid;
      }
      codes_all[(fd.row0 + r) * d + j] = static_cast<uint16_t>(lo);
      hacc += mix64((static_cast<uint64_t>(r) << 20) ^ static_cast<uint64_t>(lo) ^ 0x9E3779B97F4A7C15ull);
    }
    atomicAdd(&hsh[lane], static_cast<unsigned long long>(hacc));
  }
  __syncthreads();
  if (tid < 32 && j0 + tid < d && !ovf[tid]) hash_all[static_cast<int64_t>(blockIdx.y) * d + j0 + tid] = hsh[tid];
}

// Same contract, one CTA per (feature, family) and 256 threads over the rows: hash-insert the
// value keys (64-bit CAS into a 512-slot table), compact the <= 256 distinct keys, rank them by
// counting, then code every row by binary search. (The 32-features-per-CTA variant above keeps
// one lane per feature and walks every row serially; at a few thousand rows this one is ~20x
// faster because the row loop is spread over the whole CTA.)
__global__ void __launch_bounds__(256) distinct_col_kernel(const double* __restrict__ x, int d,
                                                           const FamDesc* __restrict__ fam,
                                                           uint16_t* __restrict__ codes_all,
                                                           double* __restrict__ vals_all,
                                                           int32_t* __restrict__ nb_all,
                                                           uint64_t* __restrict__ hash_all, uint32_t* err,
                                                           int* __restrict__ negz) {
  __shared__ unsigned long long tab[kHashSlots];
  __shared__ uint64_t keys[kSmallBins];
  __shared__ uint64_t sorted[kSmallBins];
  __shared__ unsigned long long whash[8];
  __shared__ int cnt, ovf;
  const FamDesc fd = fam[blockIdx.y];
  const int j = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < kHashSlots; i += blockDim.x) tab[i] = 0;
  if (tid == 0) {
    cnt = 0;
    ovf = 0;
  }
  __syncthreads();
  bool nonfinite = false, negzero = false;
  for (int r = tid; r < fd.n; r += blockDim.x) {
    const double v = x[(fd.row0 + r) * d + j];
    if (!isfinite(v)) {
      nonfinite = true;
      continue;
    }
    negzero |= v == 0.0 && signbit(v);
    if (*reinterpret_cast<volatile int*>(&ovf)) continue;
    const uint64_t k = value_key(v);
    uint32_t h = static_cast<uint32_t>(mix64(k)) & (kHashSlots - 1);
    for (int probe = 0; probe < kHashSlots; ++probe) {
      const unsigned long long prev = atomicCAS(tab + h, 0ull, static_cast<unsigned long long>(k));
      if (prev == 0) {
        const int idx = atomicAdd(&cnt, 1);
        if (idx < kSmallBins) keys[idx] = k;
        else ovf = 1;
        break;
      }
      if (prev == k) break;
      h = (h + 1) & (kHashSlots - 1);
      if (probe == kHashSlots - 1) ovf = 1;
    }
  }
  nonfinite = __syncthreads_or(nonfinite);
  negzero = __syncthreads_or(negzero);
  if (tid == 0) {
    if (nonfinite) atomicOr(err, kErrNonFiniteFit);
    if (negzero) atomicOr(negz + blockIdx.y, 1);
  }
  const int64_t fj = static_cast<int64_t>(blockIdx.y) * d + j;
  if (ovf) {  // > 256 distinct: the large path recodes this column
    if (tid == 0) nb_all[fj] = -1;
    return;
  }
  const int m = cnt;
  for (int i = tid; i < m; i += blockDim.x) {
    const uint64_t k = keys[i];
    int rank = 0;
    for (int o = 0; o < m; ++o) rank += keys[o] < k;
    sorted[rank] = k;
  }
  __syncthreads();
  if (tid == 0) nb_all[fj] = m;
  for (int i = tid; i < m; i += blockDim.x) vals_all[fj * kSmallBins + i] = key_value(sorted[i]);
  unsigned long long hacc = 0;
  for (int r = tid; r < fd.n; r += blockDim.x) {
    const double v = x[(fd.row0 + r) * d + j];
    if (!isfinite(v)) continue;
    const uint64_t k = value_key(v);
    int lo = 0, hi = m - 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (sorted[mid] < k) lo = mid + 1;
      else hi = mid;
    }
    codes_all[(fd.row0 + r) * d + j] = static_cast<uint16_t>(lo);
    hacc += mix64((static_cast<uint64_t>(r) << 20) ^ static_cast<uint64_t>(lo) ^ 0x9E3779B97F4A7C15ull);
  }
  for (int o = 16; o > 0; o >>= 1) hacc += __shfl_xor_sync(0xffffffffu, hacc, o);
  if (lane == 0) whash[warp] = hacc;
  __syncthreads();
  if (tid == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += whash[w];
    hash_all[fj] = t;
  }
}

// prep 1b: features with > 256 distinct values - LSD sort of the column by value key, dense rank.
struct LargeItem {
  int32_t fam;
  int32_t feat;
  int64_t vals0;  // offset into vals_large
};

__global__ void __launch_bounds__(kSortThreads) distinct_large_kernel(
    const double* __restrict__ x, int d, const FamDesc* __restrict__ fam, const LargeItem* __restrict__ items,
    int32_t* __restrict__ bufA, int32_t* __restrict__ bufB, int64_t buf_stride, uint16_t* __restrict__ codes_all,
    double* __restrict__ vals_large, int32_t* __restrict__ nb_all, uint64_t* __restrict__ hash_all, uint32_t* err) {
  __shared__ SortSmem sm;
  __shared__ int wsum[32];
  __shared__ int carry;
  __shared__ unsigned long long hsh;
  const LargeItem it = items[blockIdx.x];
  const FamDesc fd = fam[it.fam];
  const int n = fd.n, j = it.feat;
  int32_t* A = bufA + blockIdx.x * buf_stride;
  int32_t* B = bufB + blockIdx.x * buf_stride;
  sort_smem_init(sm);
  auto key = [&](int r) { return value_key(x[(fd.row0 + r) * d + j]); };
  bool first = true;
  for (int byte = 0; byte < 8; ++byte) {
    auto dig = [&](int r) { return static_cast<int>((key(r) >> (8 * byte)) & 255u); };
    bool moved;
    if (first) moved = stable_digit_pass([](int i) { return i; }, B, n, dig, sm);
    else moved = stable_digit_pass([&](int i) { return A[i]; }, B, n, dig, sm);
    if (moved) {
      int32_t* t = A;
      A = B;
      B = t;
      first = false;
    }
    __syncthreads();
  }
  if (first) {  // already sorted (all digit passes were uniform): identity
    for (int i = threadIdx.x; i < n; i += blockDim.x) A[i] = i;
    __syncthreads();
  }
  // dense rank: code = (#distinct keys before)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    carry = 0;
    hsh = 0;
  }
  __syncthreads();
  uint64_t hacc = 0;
  for (int t0 = 0; t0 < n; t0 += blockDim.x) {
    const int i = t0 + tid;
    int flag = 0;
    uint64_t k = 0;
    if (i < n) {
      k = key(A[i]);
      flag = (i == 0) || key(A[i - 1]) != k;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, flag);
    const int in_warp = __popc(bal & ((2u << lane) - 1u));  // inclusive
    if (lane == 31) wsum[warp] = __popc(bal);
    __syncthreads();
    if (warp == 0) {
      const int v = wsum[lane];
      int incl = v;
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      wsum[lane] = incl - v;
    }
    __syncthreads();
    if (i < n) {
      const int code = carry + wsum[warp] + in_warp - 1;
      if (code > kMaxBins - 1) atomicOr(err, kErrInternal);
      const int r = A[i];
      codes_all[(fd.row0 + r) * d + j] = static_cast<uint16_t>(code);
      if (flag) vals_large[it.vals0 + code] = x[(fd.row0 + r) * d + j] == 0.0 ? 0.0 : x[(fd.row0 + r) * d + j];
      hacc += mix64((static_cast<uint64_t>(r) << 20) ^ static_cast<uint64_t>(code) ^ 0x9E3779B97F4A7C15ull);
    }
    __syncthreads();
    if (tid == blockDim.x - 1) carry += wsum[warp] + in_warp;
    __syncthreads();
  }
  atomicAdd(&hsh, static_cast<unsigned long long>(hacc));
  __syncthreads();
  if (tid == 0) {
    nb_all[static_cast<int64_t>(it.fam) * d + j] = carry;
    hash_all[static_cast<int64_t>(it.fam) * d + j] = hsh;
  }
}

// prep 2: exact verification of hash-equal feature pairs (codes identical on every row?)
struct PairItem {
  int32_t fam, a, b, pad;
};

__global__ void verify_pairs_kernel(const uint16_t* __restrict__ codes_all, int d, const FamDesc* __restrict__ fam,
                                    const PairItem* __restrict__ pairs, int32_t* __restrict__ mismatch) {
  const PairItem pr = pairs[blockIdx.x];
  const FamDesc fd = fam[pr.fam];
  int bad = 0;
  for (int r = threadIdx.x; r < fd.n; r += blockDim.x)
    bad |= codes_all[(fd.row0 + r) * d + pr.a] != codes_all[(fd.row0 + r) * d + pr.b];
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) mismatch[blockIdx.x] = bad;
}

// prep 3a: per-rep value tables
__global__ void rep_vals_kernel(const FamDesc* __restrict__ fam, const int32_t* __restrict__ rep_orig,
                                const int32_t* __restrict__ rep_boff, const int32_t* __restrict__ rep_nb,
                                const int64_t* __restrict__ rep_src, const double* __restrict__ vals_all,
                                const double* __restrict__ vals_large, int d, double* __restrict__ vals) {
  const FamDesc fd = fam[blockIdx.y];
  for (int jj = blockIdx.x; jj < fd.nrep; jj += gridDim.x) {
    const int r = fd.rep0 + jj;
    const int64_t src = rep_src[r];
    const int nb = rep_nb[r];
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
      const double v = src >= 0 ? vals_large[src + b]
                                : vals_all[(static_cast<int64_t>(blockIdx.y) * d + rep_orig[r]) * kSmallBins + b];
      vals[fd.bin0 + rep_boff[r] + b] = v;
    }
  }
}

// prep 3b: canonical row order (costmodel.cpp:161-173) - LSD over (rep codes..., target)
__global__ void __launch_bounds__(kSortThreads) canonical_kernel(const double* __restrict__ target,
                                                                 const uint16_t* __restrict__ codes_all, int d,
                                                                 const FamDesc* __restrict__ fam,
                                                                 const int32_t* __restrict__ rep_orig,
                                                                 const int32_t* __restrict__ rep_nb,
                                                                 int32_t* __restrict__ canon,
                                                                 int32_t* __restrict__ tmp,
                                                                 const int* __restrict__ eligible) {
  __shared__ SortSmem sm;
  if (eligible && eligible[blockIdx.x]) return;  // canonical_bitonic_kernel sorts this family
  const FamDesc fd = fam[blockIdx.x];
  const int n = fd.n;
  int32_t* A = canon + fd.pos0;
  int32_t* B = tmp + fd.pos0;
  sort_smem_init(sm);
  for (int i = threadIdx.x; i < n; i += blockDim.x) A[i] = i;
  __syncthreads();
  auto run = [&](auto dig) {
    const bool moved = stable_digit_pass([&](int i) { return A[i]; }, B, n, dig, sm);
    if (moved) {
      int32_t* t = A;
      A = B;
      B = t;
    }
    __syncthreads();
  };
  for (int byte = 0; byte < 8; ++byte)
    run([&](int r) { return static_cast<int>((value_key(target[fd.row0 + r]) >> (8 * byte)) & 255u); });
  for (int jj = fd.nrep - 1; jj >= 0; --jj) {
    const int f = rep_orig[fd.rep0 + jj];
    run([&](int r) { return static_cast<int>(codes_all[(fd.row0 + r) * d + f] & 255u); });
    if (rep_nb[fd.rep0 + jj] > 256) run([&](int r) { return static_cast<int>(codes_all[(fd.row0 + r) * d + f] >> 8); });
  }
  if (A != canon + fd.pos0)
    for (int i = threadIdx.x; i < n; i += blockDim.x) canon[fd.pos0 + i] = A[i];
}

// prep 3c: rows into canonical order (codes of reps only, targets) + row->family map
template <typename CodeT>
__global__ void gather_canonical_kernel(const double* __restrict__ target, const uint16_t* __restrict__ codes_all,
                                        int d, const FamDesc* __restrict__ fam, int F, int64_t n_tot,
                                        const int32_t* __restrict__ rep_orig, const int32_t* __restrict__ canon,
                                        int Dp, CodeT* __restrict__ codes_c, double* __restrict__ target_c,
                                        int32_t* __restrict__ rowfam) {
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < n_tot;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int f = family_of_pos(fam, F, p);
    const FamDesc fd = fam[f];
    const int64_t row = fd.row0 + canon[p];
    rowfam[p] = f;
    target_c[p] = target[row];
    CodeT* o = codes_c + p * Dp;
    for (int jj = 0; jj < Dp; ++jj)
      o[jj] = jj < fd.nrep ? static_cast<CodeT>(codes_all[row * d + rep_orig[fd.rep0 + jj]]) : CodeT(0);
  }
}

// prep 3d: presorted list per rep (costmodel.cpp:193-201): stable by code over canonical positions
template <typename CodeT>
__global__ void __launch_bounds__(kSortThreads) presort_kernel(const FamDesc* __restrict__ fam, int Dp,
                                                               const CodeT* __restrict__ codes_c,
                                                               const int32_t* __restrict__ rep_nb,
                                                               int32_t* __restrict__ ord, int32_t* __restrict__ tmp) {
  __shared__ SortSmem sm;
  const FamDesc fd = fam[blockIdx.y];
  const int jj = blockIdx.x;
  if (jj >= fd.nrep) return;
  const int n = fd.n;
  int32_t* out = ord + fd.ord0 + static_cast<int64_t>(jj) * n;
  int32_t* t = tmp + fd.ord0 + static_cast<int64_t>(jj) * n;
  sort_smem_init(sm);
  const CodeT* cc = codes_c + fd.pos0 * Dp + jj;
  auto lo = [&](int p) { return static_cast<int>(cc[static_cast<int64_t>(p) * Dp] & 255u); };
  if (rep_nb[fd.rep0 + jj] <= 256) {
    if (!stable_digit_pass([](int i) { return i; }, out, n, lo, sm))
      for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = i;
  } else {
    auto hi = [&](int p) { return static_cast<int>(static_cast<uint32_t>(cc[static_cast<int64_t>(p) * Dp]) >> 8); };
    const bool m1 = stable_digit_pass([](int i) { return i; }, t, n, lo, sm);
    if (!m1)
      for (int i = threadIdx.x; i < n; i += blockDim.x) t[i] = i;
    __syncthreads();
    if (!stable_digit_pass([&](int i) { return t[i]; }, out, n, hi, sm))
      for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = t[i];
  }
}

// cumulative bin counts over the whole family (for the signed-zero threshold lookup)
template <typename CodeT>
__global__ void bin_count_kernel(const FamDesc* __restrict__ fam, int F, int64_t n_tot, int Dp,
                                 const CodeT* __restrict__ codes_c, const int32_t* __restrict__ rowfam,
                                 const int32_t* __restrict__ rep_boff, int32_t* __restrict__ cle) {
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < n_tot;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const FamDesc fd = fam[rowfam[p]];
    for (int jj = 0; jj < fd.nrep; ++jj)
      atomicAdd(&cle[fd.bin0 + rep_boff[fd.rep0 + jj] + codes_c[p * Dp + jj]], 1);
  }
}

__global__ void bin_prefix_kernel(const FamDesc* __restrict__ fam, const int32_t* __restrict__ rep_boff,
                                  const int32_t* __restrict__ rep_nb, int32_t* __restrict__ cle) {
  const FamDesc fd = fam[blockIdx.x];
  for (int jj = threadIdx.x; jj < fd.nrep; jj += blockDim.x) {
    int32_t* c = cle + fd.bin0 + rep_boff[fd.rep0 + jj];
    int run = 0;
    for (int b = 0; b < rep_nb[fd.rep0 + jj]; ++b) {
      run += c[b];
      c[b] = run;
    }
  }
}

// prep 3e: base = sequential mean in canonical order (costmodel.cpp:185-188); pred = base;
// pristine order-0 list (presorted[0], or canonical order when feature 0 is constant).
// Canonical row order (costmodel.cpp:161-173) for families whose key rows fit one CTA's shared
// memory and hold no -0.0: rows are ranked by (representative codes in feature order, target) -
// a lexicographic key packed big-endian into 32-bit words (codes preserve each feature's value
// order; constant and duplicate columns cannot change it) - with one bitonic sort. Equal keys are
// bitwise-identical rows (no -0.0), so their relative order is unobservable. Other families
// keep the stable LSD passes of canonical_kernel (which leaves them untouched here: eligible
// families are skipped there).
__device__ __forceinline__ bool key_less(const uint32_t* a, const uint32_t* b, int W) {
  for (int w = 0; w < W; ++w)
    if (a[w] != b[w]) return a[w] < b[w];
  return false;
}

__global__ void __launch_bounds__(kSortThreads) canonical_bitonic_kernel(
    const double* __restrict__ target, const uint16_t* __restrict__ codes_all, int d,
    const FamDesc* __restrict__ fam, const int32_t* __restrict__ rep_orig, const int32_t* __restrict__ rep_nb,
    const int* __restrict__ eligible, int32_t* __restrict__ canon) {
  extern __shared__ __align__(16) uint32_t ks[];  // [P][W] keys, then [P] row ids
  const int f = blockIdx.x;
  if (!eligible[f]) return;
  const FamDesc fd = fam[f];
  const int n = fd.n, nrep = fd.nrep;
  int wide = 0;
  for (int j = 0; j < nrep; ++j) wide |= rep_nb[fd.rep0 + j] > 256;
  const int cb = wide ? 2 : 1;                 // bytes per code
  const int W = (nrep * cb + 3) / 4 + 2;       // code words + 64-bit target key
  int P = 1;
  while (P < n) P <<= 1;
  uint32_t* ids = ks + static_cast<size_t>(P) * W;
  for (int r = threadIdx.x; r < P; r += blockDim.x) {
    uint32_t* k = ks + static_cast<size_t>(r) * W;
    ids[r] = r;
    if (r >= n) {
      for (int w = 0; w < W; ++w) k[w] = 0xFFFFFFFFu;
      continue;
    }
    for (int w = 0; w < W - 2; ++w) k[w] = 0;
    for (int j = 0; j < nrep; ++j) {
      const uint32_t c = codes_all[(fd.row0 + r) * d + rep_orig[fd.rep0 + j]];
      for (int b = cb - 1; b >= 0; --b) {  // big-endian bytes: word compare == lexicographic
        const int byte = j * cb + (cb - 1 - b);
        k[byte >> 2] |= ((c >> (8 * b)) & 255u) << (8 * (3 - (byte & 3)));
      }
    }
    const uint64_t tk = value_key(target[fd.row0 + r]);
    k[W - 2] = static_cast<uint32_t>(tk >> 32);
    k[W - 1] = static_cast<uint32_t>(tk);
  }
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        uint32_t* a = ks + static_cast<size_t>(lo) * W;
        uint32_t* b = ks + static_cast<size_t>(hi) * W;
        if (key_less(b, a, W) == up) {
          for (int w = 0; w < W; ++w) {
            const uint32_t t = a[w];
            a[w] = b[w];
            b[w] = t;
          }
          const uint32_t t = ids[lo];
          ids[lo] = ids[hi];
          ids[hi] = t;
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) canon[fd.pos0 + i] = static_cast<int32_t>(ids[i]);
}

__global__ void base_kernel(const FamDesc* __restrict__ fam, const double* __restrict__ target_c,
                            double* __restrict__ base, double* __restrict__ pred, const int32_t* __restrict__ ord,
                            int32_t* __restrict__ ord_root) {
  const FamDesc fd = fam[blockIdx.x];
  if (threadIdx.x == 0) {  // sequential mean in canonical order (costmodel.cpp:185-188)
    const double* t = target_c + fd.pos0;
    double s = 0.0;
    int i = 0;
    if (fd.n >= 8) {  // the next 8 loads are in flight while 8 dependent adds run
      double a[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = t[k];
      for (i = 8; i + 8 <= fd.n; i += 8) {
        double b[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) b[k] = t[i + k];
#pragma unroll
        for (int k = 0; k < 8; ++k) s = fs_add(s, a[k]);
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = b[k];
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) s = fs_add(s, a[k]);
    }
    for (; i < fd.n; ++i) s = fs_add(s, t[i]);
    base[blockIdx.x] = fd.n ? fs_div(s, static_cast<double>(fd.n)) : 0.0;
  }
  __syncthreads();
  const double b = base[blockIdx.x];
  for (int i = threadIdx.x; i < fd.n; i += blockDim.x) {
    pred[fd.pos0 + i] = b;
    ord_root[fd.pos0 + i] = fd.f0rep >= 0 ? ord[fd.ord0 + static_cast<int64_t>(fd.f0rep) * fd.n + i] : i;
  }
}

// ------------------------------------------------------------------------------------------
// boosting rounds
// ------------------------------------------------------------------------------------------
__global__ void round_init_kernel(const FamDesc* __restrict__ fam, FamState* __restrict__ st, NodeRec* __restrict__ nodes,
                                  int slots, TreeRec* __restrict__ trees) {
  const int f = blockIdx.x;
  const FamDesc fd = fam[f];
  if (!st[f].active) return;
  NodeRec* nd = nodes + fd.node0;
  for (int s = threadIdx.x; s < slots; s += blockDim.x) {
    NodeRec z;
    memset(&z, 0, sizeof z);
    if (s == 0) z.n = fd.n;
    nd[s] = z;
    TreeRec tz;
    memset(&tz, 0, sizeof tz);
    trees[fd.tree0 + static_cast<int64_t>(st[f].ntrees) * slots + s] = tz;
  }
  if (threadIdx.x == 0) st[f].maxabs = 0;
}

__global__ void residual_kernel(const FamDesc* __restrict__ fam, int F, int64_t n_tot, FamState* __restrict__ st,
                                const int32_t* __restrict__ rowfam, const double* __restrict__ target_c,
                                const double* __restrict__ pred, double* __restrict__ resid,
                                const int32_t* __restrict__ ord_root, int32_t* __restrict__ ord_cur,
                                int16_t* __restrict__ nodeid) {
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < n_tot;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int f = rowfam[p];
    if (!st[f].active) continue;
    const double r = fs_sub(target_c[p], pred[p]);  // costmodel.cpp:204-206
    resid[p] = r;
    ord_cur[p] = ord_root[p];
    nodeid[p] = 0;
    // max |r| bits (non-negative doubles order like integers): warp-reduced when the warp's
    // rows share a family (the common case - families are contiguous), else per lane
    unsigned long long m = static_cast<unsigned long long>(__double_as_longlong(fabs(r)));
    const unsigned act = __activemask();
    const int f0 = __shfl_sync(act, f, __ffs(act) - 1);
    if (__all_sync(act, f == f0) && act == 0xffffffffu) {
      for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
      if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<unsigned long long*>(&st[f].maxabs), m);
    } else {
      atomicMax(reinterpret_cast<unsigned long long*>(&st[f].maxabs), m);
    }
  }
}

__device__ __forceinline__ int fix_shift(uint64_t maxabs_bits, int n) {
  const double m = __longlong_as_double(static_cast<long long>(maxabs_bits));
  if (!(m > 0.0)) return 0;
  int lg = 0;
  while ((1 << lg) < n) ++lg;
  const int e = ilogb(m) + 1;  // m < 2^e
  return 61 - e - lg;          // n * |r| * 2^shift < 2^61
}

__global__ void fixed_kernel(const FamDesc* __restrict__ fam, int64_t n_tot, FamState* __restrict__ st,
                             const int32_t* __restrict__ rowfam, const double* __restrict__ resid,
                             int64_t* __restrict__ rfix) {
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < n_tot;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int f = rowfam[p];
    if (!st[f].active) continue;
    const int sh = fix_shift(st[f].maxabs, fam[f].n);
    rfix[p] = __double2ll_rn(ldexp(resid[p], sh));
    if (p == fam[f].pos0) st[f].shift = sh;
  }
}

__device__ __forceinline__ bool node_needs_split(const FamDesc& fd, int level, int n) {
  return level < fd.depth && n >= max(2, fd.min_split);  // costmodel.cpp:78-80 (+ n>=2 for a boundary)
}

// Which nodes at `level` are screened, which histograms are built directly / derived.
__global__ void level_plan_kernel(const FamDesc* __restrict__ fam, const FamState* __restrict__ st,
                                  NodeRec* __restrict__ nodes, int level) {
  const int f = blockIdx.y;
  const FamDesc fd = fam[f];
  if (!st[f].active) return;
  const int first = (1 << level) - 1;
  const int local = blockIdx.x * blockDim.x + threadIdx.x;
  if (local >= (1 << level)) return;
  NodeRec* nd = nodes + fd.node0;
  const int s = first + local;
  if (level == 0) {
    if (fd.nrep > 0 && node_needs_split(fd, 0, nd[0].n)) nd[0].build = 1;
    else nd[0].state = kNodeLeaf;
    return;
  }
  const int parent = (s - 1) >> 1;
  if (nd[parent].state != kNodeSplit) return;
  const bool need = fd.nrep > 0 && node_needs_split(fd, level, nd[s].n);
  if (!need) nd[s].state = kNodeLeaf;
  if (s & 1) {  // left child decides the pair's build plan
    const int sib = s + 1;
    const bool need_sib = fd.nrep > 0 && node_needs_split(fd, level, nd[sib].n);
    if (need || need_sib) {
      const int small = nd[s].n <= nd[sib].n ? s : sib;
      nd[small].build = 1;
      nd[small == s ? sib : s].build = 2;
    }
  }
}

__global__ void hist_zero_kernel(const FamDesc* __restrict__ fam, const FamState* __restrict__ st, int level,
                                 int64_t* __restrict__ hsum, int32_t* __restrict__ hcnt) {
  const int f = blockIdx.y;
  const FamDesc fd = fam[f];
  if (!st[f].active || level >= max(fd.depth, 1)) return;
  const int64_t base = fd.hist0 + static_cast<int64_t>(level & 1) * fd.level_slots * fd.bins;
  const int64_t cnt = static_cast<int64_t>(min(1 << level, fd.level_slots)) * fd.bins;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < cnt;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    hsum[base + i] = 0;
    hcnt[base + i] = 0;
  }
}

constexpr int kHistThreads = 256;
constexpr int kHistTileRows = 64;
constexpr int kHistChunk = 4096;

// Histogram of one directly-built node over one chunk of its rows. Threads own (feature, row
// group) pairs, so shared-memory bins are updated without atomics; the CTA then adds its
// partial histogram to the node's global histogram with integer atomics (exact, order-free).
template <typename CodeT, bool kGlobal>
__global__ void __launch_bounds__(kHistThreads) hist_build_kernel(
    const FamDesc* __restrict__ fam, const FamState* __restrict__ st, const NodeRec* __restrict__ nodes, int level,
    int Dp, const CodeT* __restrict__ codes_c, const int64_t* __restrict__ rfix, const int32_t* __restrict__ ord_cur,
    const int32_t* __restrict__ rep_boff, int64_t* __restrict__ hsum, int32_t* __restrict__ hcnt,
    int64_t* __restrict__ node_abs, int groups, unsigned long long* __restrict__ ctr) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int f = blockIdx.z;
  const FamDesc fd = fam[f];
  if (!st[f].active) return;
  const NodeRec* nd = nodes + fd.node0;
  int s;
  if (level == 0) {
    if (blockIdx.y) return;
    s = 0;
  } else {
    if (blockIdx.y >= (1u << (level - 1))) return;
    const int parent = (1 << (level - 1)) - 1 + blockIdx.y;
    if (nd[parent].state != kNodeSplit) return;
    s = 2 * parent + 1;
    if (nd[s].build != 1) s += 1;
    if (nd[s].build != 1) return;
  }
  const int n_v = nd[s].n;
  const int r0 = blockIdx.x * kHistChunk;
  if (r0 >= n_v) return;
  const int rows = min(kHistChunk, n_v - r0);
  const int seg = nd[s].seg;
  const int local = s - ((1 << level) - 1);
  const int64_t hbase = fd.hist0 + (static_cast<int64_t>(level & 1) * fd.level_slots + local) * fd.bins;
  const int bins = fd.bins, nrep = fd.nrep;

  int64_t* s_sum = reinterpret_cast<int64_t*>(smem);
  int32_t* s_cnt = reinterpret_cast<int32_t*>(s_sum + (kGlobal ? 0 : static_cast<int64_t>(groups) * bins));
  unsigned char* tail = reinterpret_cast<unsigned char*>(s_cnt + (kGlobal ? 0 : static_cast<int64_t>(groups) * bins));
  tail = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tail) + 15) & ~uintptr_t(15));
  CodeT* t_codes = reinterpret_cast<CodeT*>(tail);                          // [kHistTileRows][Dp]
  int64_t* t_fix = reinterpret_cast<int64_t*>(t_codes + kHistTileRows * Dp);  // [kHistTileRows]
  __shared__ unsigned long long s_abs;
  const int tid = threadIdx.x;
  if (!kGlobal)
    for (int i = tid; i < groups * bins; i += kHistThreads) {
      s_sum[i] = 0;
      s_cnt[i] = 0;
    }
  if (tid == 0) s_abs = 0;
  // thread -> (feature, group)
  const int per_group = nrep > 0 ? (nrep < kHistThreads ? nrep : kHistThreads) : 1;
  const int g = tid / per_group;
  const int fj0 = tid - g * per_group;
  const bool worker = g < groups && fj0 < nrep;
  __syncthreads();
  const int vec_per_row = Dp * static_cast<int>(sizeof(CodeT)) / 16;
  for (int t0 = 0; t0 < rows; t0 += kHistTileRows) {
    const int tr = min(kHistTileRows, rows - t0);
    for (int i = tid; i < tr * vec_per_row; i += kHistThreads) {
      const int r = i / vec_per_row, v = i - r * vec_per_row;
      const int64_t p = fd.pos0 + ord_cur[fd.pos0 + seg + r0 + t0 + r];
      reinterpret_cast<uint4*>(t_codes + r * Dp)[v] = reinterpret_cast<const uint4*>(codes_c + p * Dp)[v];
    }
    unsigned long long a = 0;
    if (tid < tr) {
      const int64_t p = fd.pos0 + ord_cur[fd.pos0 + seg + r0 + t0 + tid];
      const int64_t v = rfix[p];
      t_fix[tid] = v;
      a = static_cast<unsigned long long>(v < 0 ? -v : v);
    }
    for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
    if ((tid & 31) == 0 && a) atomicAdd(&s_abs, a);
    __syncthreads();
    if (worker) {
      for (int fj = fj0; fj < nrep; fj += per_group) {
        const int boff = rep_boff[fd.rep0 + fj];
        for (int r = g; r < tr; r += groups) {
          const int bin = boff + static_cast<int>(t_codes[r * Dp + fj]);
          if (kGlobal) {
            atomicAdd(reinterpret_cast<unsigned long long*>(hsum + hbase + bin),
                      static_cast<unsigned long long>(t_fix[r]));
            atomicAdd(hcnt + hbase + bin, 1);
          } else {
            s_sum[g * bins + bin] += t_fix[r];
            s_cnt[g * bins + bin] += 1;
          }
        }
      }
    }
    __syncthreads();
  }
  if (!kGlobal) {
    for (int b = tid; b < bins; b += kHistThreads) {
      int64_t sm = 0;
      int32_t c = 0;
      for (int gg = 0; gg < groups; ++gg) {
        sm += s_sum[gg * bins + b];
        c += s_cnt[gg * bins + b];
      }
      if (c) {
        atomicAdd(reinterpret_cast<unsigned long long*>(hsum + hbase + b), static_cast<unsigned long long>(sm));
        atomicAdd(hcnt + hbase + b, c);
      }
    }
  }
  if (tid == 0 && s_abs)
    atomicAdd(reinterpret_cast<unsigned long long*>(node_abs + fd.node0 + s), s_abs);
  if (tid == 0) {
    atomicAdd(ctr + kCtrHistBytes,
              static_cast<unsigned long long>(rows) * (static_cast<unsigned long long>(nrep) * sizeof(CodeT) + 12ull));
    atomicAdd(ctr + kCtrHistRows, static_cast<unsigned long long>(rows));
  }
}

// Column-layout histogram build (the default shape). Warp w owns feature group fg = w % NFG
// (features 32fg .. 32fg+31, lane = feature) and row group w / NFG. A group's bins live in
// shared memory as [bin][32 lanes], so the 32 updates a warp issues for one row always hit 32
// different banks (no conflicts, no atomics); row groups own private copies that are summed at
// the flush. grp_off[f][fg] = entry offset of feature group fg (entries = bins x 32).
constexpr int kColWarps = 6;

template <typename CodeT>
__global__ void __launch_bounds__(kColWarps * 32) hist_build_col_kernel(
    const FamDesc* __restrict__ fam, const FamState* __restrict__ st, const NodeRec* __restrict__ nodes, int level,
    int Dp, const CodeT* __restrict__ codes_c, const int64_t* __restrict__ rfix, const int32_t* __restrict__ ord_cur,
    const int32_t* __restrict__ rep_boff, const int32_t* __restrict__ rep_nb, const int32_t* __restrict__ grp_off,
    const int32_t* __restrict__ grp_rg, int64_t* __restrict__ hsum, int32_t* __restrict__ hcnt,
    int64_t* __restrict__ node_abs, unsigned long long* __restrict__ ctr) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int f = blockIdx.z;
  const FamDesc fd = fam[f];
  if (!st[f].active) return;
  const NodeRec* nd = nodes + fd.node0;
  int s;
  if (level == 0) {
    if (blockIdx.y) return;
    s = 0;
  } else {
    if (blockIdx.y >= (1u << (level - 1))) return;
    const int parent = (1 << (level - 1)) - 1 + blockIdx.y;
    if (nd[parent].state != kNodeSplit) return;
    s = 2 * parent + 1;
    if (nd[s].build != 1) s += 1;
    if (nd[s].build != 1) return;
  }
  const int n_v = nd[s].n;
  const int r0 = blockIdx.x * kHistChunk;
  if (r0 >= n_v) return;
  const int rows = min(kHistChunk, n_v - r0);
  const int seg = nd[s].seg;
  const int local = s - ((1 << level) - 1);
  const int64_t hbase = fd.hist0 + (static_cast<int64_t>(level & 1) * fd.level_slots + local) * fd.bins;
  const int nrep = fd.nrep;
  const int nfg = (nrep + 31) >> 5;
  const int32_t* go = grp_off + static_cast<int64_t>(f) * (kColWarps + 1);
  const int gsz = go[nfg];            // entries per copy
  const int rg = grp_rg[f];           // row groups (copies)
  int64_t* s_sum = reinterpret_cast<int64_t*>(smem);                        // [rg][gsz]
  int32_t* s_cnt = reinterpret_cast<int32_t*>(s_sum + static_cast<int64_t>(rg) * gsz);
  unsigned char* tail = reinterpret_cast<unsigned char*>(s_cnt + static_cast<int64_t>(rg) * gsz);
  tail = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tail) + 15) & ~uintptr_t(15));
  CodeT* t_codes = reinterpret_cast<CodeT*>(tail);                            // [kHistTileRows][Dp]
  int64_t* t_fix = reinterpret_cast<int64_t*>(t_codes + kHistTileRows * Dp);  // [kHistTileRows]
  __shared__ unsigned long long s_abs;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < rg * gsz; i += kColWarps * 32) {
    s_sum[i] = 0;
    s_cnt[i] = 0;
  }
  if (tid == 0) s_abs = 0;
  const int fg = warp % nfg, rgi = warp / nfg;
  const bool worker = rgi < rg;
  const int j = 32 * fg + lane;
  const bool jv = worker && j < nrep;
  int64_t* my_sum = s_sum + static_cast<int64_t>(rgi) * gsz + go[fg] + lane;
  int32_t* my_cnt = s_cnt + static_cast<int64_t>(rgi) * gsz + go[fg] + lane;
  __syncthreads();
  const int vec_per_row = Dp * static_cast<int>(sizeof(CodeT)) / 16;
  for (int t0 = 0; t0 < rows; t0 += kHistTileRows) {
    const int tr = min(kHistTileRows, rows - t0);
    for (int i = tid; i < tr * vec_per_row; i += kColWarps * 32) {
      const int r = i / vec_per_row, v = i - r * vec_per_row;
      const int64_t p = fd.pos0 + ord_cur[fd.pos0 + seg + r0 + t0 + r];
      reinterpret_cast<uint4*>(t_codes + r * Dp)[v] = reinterpret_cast<const uint4*>(codes_c + p * Dp)[v];
    }
    unsigned long long a = 0;
    for (int r = tid; r < tr; r += kColWarps * 32) {
      const int64_t p = fd.pos0 + ord_cur[fd.pos0 + seg + r0 + t0 + r];
      const int64_t v = rfix[p];
      t_fix[r] = v;
      a += static_cast<unsigned long long>(v < 0 ? -v : v);
    }
    for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
    if (lane == 0 && a) atomicAdd(&s_abs, a);
    __syncthreads();
    if (jv) {
      for (int r = rgi; r < tr; r += rg) {
        const int b = static_cast<int>(t_codes[r * Dp + j]);
        my_sum[b * 32] += t_fix[r];
        my_cnt[b * 32] += 1;
      }
    }
    __syncthreads();
  }
  // flush: entry e = (fg, b, lane) -> global bin boff_j + b
  for (int e = tid; e < gsz; e += kColWarps * 32) {
    int g = 0;
    while (g + 1 < nfg && go[g + 1] <= e) ++g;
    const int within = e - go[g];
    const int b = within >> 5, jj = 32 * g + (within & 31);
    if (jj >= nrep || b >= rep_nb[fd.rep0 + jj]) continue;
    int64_t sm = 0;
    int32_t c = 0;
    for (int k = 0; k < rg; ++k) {
      sm += s_sum[static_cast<int64_t>(k) * gsz + e];
      c += s_cnt[static_cast<int64_t>(k) * gsz + e];
    }
    if (c) {
      const int64_t gb = hbase + rep_boff[fd.rep0 + jj] + b;
      atomicAdd(reinterpret_cast<unsigned long long*>(hsum + gb), static_cast<unsigned long long>(sm));
      atomicAdd(hcnt + gb, c);
    }
  }
  if (tid == 0) {
    if (s_abs) atomicAdd(reinterpret_cast<unsigned long long*>(node_abs + fd.node0 + s), s_abs);
    atomicAdd(ctr + kCtrHistBytes,
              static_cast<unsigned long long>(rows) * (static_cast<unsigned long long>(nrep) * sizeof(CodeT) + 12ull));
    atomicAdd(ctr + kCtrHistRows, static_cast<unsigned long long>(rows));
  }
}

// Lane-column histogram shape (conflict-free shared atomics): lane l of every warp owns bank
// column l. nrep <= 32: lanes l < (32 / nrep) * nrep take feature l % nrep (copy l / nrep of
// it), so the column height is the largest bin count. nrep > 32: lane l takes features l, l+32,
// ... stacked in its column (cofs = offset of a feature's bins in its lane's column).
__host__ __device__ inline int col_height(int nrep, const int32_t* nb, int32_t* cofs) {
  int H = 1;
  if (nrep <= 32) {
    for (int j = 0; j < nrep; ++j) {
      if (cofs) cofs[j] = 0;
      H = nb[j] > H ? nb[j] : H;
    }
    return H;
  }
  for (int l = 0; l < 32; ++l) {
    int h = 0;
    for (int j = l; j < nrep; j += 32) {
      if (cofs) cofs[j] = h;
      h += nb[j];
    }
    H = h > H ? h : H;
  }
  return H;
}

// Limb-atomic histogram build (the default shape). Only 32-bit shared-memory atomics are native
// on sm_100a (64-bit ones compile to CAS spin loops), so each 62-bit fixed-point residual v is
// offset to u = v + 2^62 (in [0, 2^63)) and split into three 21-bit limbs accumulated with
// native 32-bit atomics by ALL 1024 threads (any thread may update any bin). Limb sums over at
// most kAtomSub = 2048 rows stay below 2^32; they are then folded exactly into 64-bit per-bin
// accumulators: U = S0 + S1*2^21 + S2*2^42, count = (U + 2^61) >> 62 (|sum v| < 2^61 by the
// choice of the fixed-point shift), sum = U - count*2^62. No count atomic is needed.
constexpr int kAtomThreads = 1024;
constexpr int kAtomSub = 2048;
constexpr int kAtomChunk = 8192;  // max rows per CTA (fewer when the batch is small: >= 2 CTAs per SM)
constexpr int kAtomTile = 128;
constexpr uint32_t kLimbMask = (1u << 21) - 1u;

template <typename CodeT>
__global__ void __launch_bounds__(kAtomThreads, 2) hist_build_atomic_kernel(
    const FamDesc* __restrict__ fam, const FamState* __restrict__ st, const NodeRec* __restrict__ nodes, int level,
    int Dp, const CodeT* __restrict__ codes_c, const int64_t* __restrict__ rfix, const int32_t* __restrict__ ord_cur,
    const int32_t* __restrict__ rep_boff, int64_t* __restrict__ hsum, int32_t* __restrict__ hcnt,
    int64_t* __restrict__ node_abs, unsigned long long* __restrict__ ctr, int colh_max, int chunk) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int f = blockIdx.z;
  const FamDesc fd = fam[f];
  if (!st[f].active) return;
  const NodeRec* nd = nodes + fd.node0;
  int s;
  if (level == 0) {
    if (blockIdx.y) return;
    s = 0;
  } else {
    if (blockIdx.y >= (1u << (level - 1))) return;
    const int parent = (1 << (level - 1)) - 1 + blockIdx.y;
    if (nd[parent].state != kNodeSplit) return;
    s = 2 * parent + 1;
    if (nd[s].build != 1) s += 1;
    if (nd[s].build != 1) return;
  }
  const int n_v = nd[s].n;
  const int r0 = blockIdx.x * chunk;
  if (r0 >= n_v) return;
  const int rows = min(chunk, n_v - r0);
  const int seg = nd[s].seg;
  const int local = s - ((1 << level) - 1);
  const int64_t hbase = fd.hist0 + (static_cast<int64_t>(level & 1) * fd.level_slots + local) * fd.bins;
  const int nrep = fd.nrep, bins = fd.bins;
  // layout: limbs[3][colh_max][32] u32 (lane columns, see col_height) | acc_sum[bins] i64 |
  // acc_cnt[bins] i32 | binrep[bins] u16 | boff[nrep] | cofs[nrep] | tile codes | tile limbs
  uint32_t* limb = reinterpret_cast<uint32_t*>(smem);
  int64_t* acc_sum =
      reinterpret_cast<int64_t*>(smem + ((static_cast<size_t>(3) * colh_max * 32 * 4 + 15) & ~size_t(15)));
  int32_t* acc_cnt = reinterpret_cast<int32_t*>(acc_sum + bins);
  uint16_t* s_binrep = reinterpret_cast<uint16_t*>(acc_cnt + bins);
  int32_t* s_boff = reinterpret_cast<int32_t*>(s_binrep + ((bins + 1) & ~1));
  int32_t* s_cofs = s_boff + nrep;
  int32_t* s_nbv = s_cofs + nrep;
  unsigned char* tail = reinterpret_cast<unsigned char*>(s_nbv + nrep);
  tail = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tail) + 15) & ~uintptr_t(15));
  CodeT* t_codes = reinterpret_cast<CodeT*>(tail);                              // [kAtomTile][Dp]
  uint32_t* t_limb = reinterpret_cast<uint32_t*>(t_codes + kAtomTile * Dp);     // [kAtomTile][3]
  __shared__ unsigned long long s_abs;
  __shared__ int s_colh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int b = tid; b < bins; b += kAtomThreads) {
    acc_sum[b] = 0;
    acc_cnt[b] = 0;
  }
  for (int j = tid; j < nrep; j += kAtomThreads) {
    const int b0 = rep_boff[fd.rep0 + j];
    const int b1 = j + 1 < nrep ? rep_boff[fd.rep0 + j + 1] : bins;
    s_boff[j] = b0;
    s_nbv[j] = b1 - b0;
    for (int b = b0; b < b1; ++b) s_binrep[b] = static_cast<uint16_t>(j);
  }
  if (tid == 0) s_abs = 0;
  __syncthreads();
  if (tid == 0) s_colh = col_height(nrep, s_nbv, s_cofs);
  __syncthreads();
  const int colh = s_colh;
  const int rpw = nrep <= 32 ? 32 / nrep : 1;  // rows per warp step (lane copies, nrep <= 32)
  const int hj = nrep <= 32 ? lane % nrep : lane;
  const int hm = nrep <= 32 ? lane / nrep : 0;
  const bool hact = nrep <= 32 ? hm < rpw : true;
  const int vec_per_row = Dp * static_cast<int>(sizeof(CodeT)) / 16;
  for (int sub0 = 0; sub0 < rows; sub0 += kAtomSub) {
    for (int i = tid; i < 3 * colh * 32; i += kAtomThreads) limb[i] = 0;
    __syncthreads();
    const int sub_end = min(rows, sub0 + kAtomSub);
    for (int t0 = sub0; t0 < sub_end; t0 += kAtomTile) {
      const int tr = min(kAtomTile, sub_end - t0);
      for (int i = tid; i < tr * vec_per_row; i += kAtomThreads) {
        const int r = i / vec_per_row, v = i - r * vec_per_row;
        const int64_t p = fd.pos0 + ord_cur[fd.pos0 + seg + r0 + t0 + r];
        reinterpret_cast<uint4*>(t_codes + r * Dp)[v] = reinterpret_cast<const uint4*>(codes_c + p * Dp)[v];
      }
      unsigned long long a = 0;
      if (tid < tr) {
        const int64_t p = fd.pos0 + ord_cur[fd.pos0 + seg + r0 + t0 + tid];
        const int64_t v = rfix[p];
        const uint64_t u = static_cast<uint64_t>(v) + (1ull << 62);
        t_limb[3 * tid] = static_cast<uint32_t>(u) & kLimbMask;
        t_limb[3 * tid + 1] = static_cast<uint32_t>(u >> 21) & kLimbMask;
        t_limb[3 * tid + 2] = static_cast<uint32_t>(u >> 42);
        a = static_cast<unsigned long long>(v < 0 ? -v : v);
      }
      if (warp * 32 < tr) {
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0 && a) atomicAdd(&s_abs, a);
      }
      __syncthreads();
      // lane columns: every lane adds into its own bank column -> one wavefront per atomic
      if (hact) {
        uint32_t* colp = limb + lane;
        if (nrep <= 32) {
          for (int r = warp * rpw + hm; r < tr; r += (kAtomThreads / 32) * rpw) {
            const uint32_t* tl = t_limb + 3 * r;
            uint32_t* c = colp + static_cast<int>(t_codes[r * Dp + hj]) * 32;
            atomicAdd(c, tl[0]);
            atomicAdd(c + colh * 32, tl[1]);
            atomicAdd(c + 2 * colh * 32, tl[2]);
          }
        } else {
          for (int r = warp; r < tr; r += kAtomThreads / 32) {
            const uint32_t l0 = t_limb[3 * r], l1 = t_limb[3 * r + 1], l2 = t_limb[3 * r + 2];
            const CodeT* cr = t_codes + r * Dp;
            for (int j = lane; j < nrep; j += 32) {
              uint32_t* c = colp + (s_cofs[j] + static_cast<int>(cr[j])) * 32;
              atomicAdd(c, l0);
              atomicAdd(c + colh * 32, l1);
              atomicAdd(c + 2 * colh * 32, l2);
            }
          }
        }
      }
      __syncthreads();
    }
    for (int b = tid; b < bins; b += kAtomThreads) {
      const int j = s_binrep[b], bb = b - s_boff[j];
      unsigned __int128 U = 0;
      if (nrep <= 32) {
        for (int m = 0; m < rpw; ++m) {
          const uint32_t* c = limb + bb * 32 + j + m * nrep;
          U += static_cast<unsigned __int128>(c[0]) + (static_cast<unsigned __int128>(c[colh * 32]) << 21) +
               (static_cast<unsigned __int128>(c[2 * colh * 32]) << 42);
        }
      } else {
        const uint32_t* c = limb + (s_cofs[j] + bb) * 32 + (j & 31);
        U = static_cast<unsigned __int128>(c[0]) + (static_cast<unsigned __int128>(c[colh * 32]) << 21) +
            (static_cast<unsigned __int128>(c[2 * colh * 32]) << 42);
      }
      const uint64_t c = static_cast<uint64_t>((U + (static_cast<unsigned __int128>(1) << 61)) >> 62);
      const unsigned __int128 sv = U - (static_cast<unsigned __int128>(c) << 62);
      acc_sum[b] += static_cast<int64_t>(static_cast<uint64_t>(sv));
      acc_cnt[b] += static_cast<int32_t>(c);
    }
    __syncthreads();
  }
  for (int b = tid; b < bins; b += kAtomThreads) {
    if (acc_cnt[b]) {
      atomicAdd(reinterpret_cast<unsigned long long*>(hsum + hbase + b), static_cast<unsigned long long>(acc_sum[b]));
      atomicAdd(hcnt + hbase + b, acc_cnt[b]);
    }
  }
  if (tid == 0) {
    if (s_abs) atomicAdd(reinterpret_cast<unsigned long long*>(node_abs + fd.node0 + s), s_abs);
    atomicAdd(ctr + kCtrHistBytes,
              static_cast<unsigned long long>(rows) * (static_cast<unsigned long long>(nrep) * sizeof(CodeT) + 12ull));
    atomicAdd(ctr + kCtrHistRows, static_cast<unsigned long long>(rows));
  }
}

inline size_t hist_atomic_smem(int bins, int nrep, int Dp, int code_bytes, int colh) {
  size_t o = (static_cast<size_t>(3) * colh * 32 * 4 + 15) & ~size_t(15);
  o += static_cast<size_t>(bins) * 14 + static_cast<size_t>(nrep) * 12 + 16;
  o = (o + 15) & ~size_t(15);
  o += static_cast<size_t>(kAtomTile) * Dp * code_bytes + static_cast<size_t>(kAtomTile) * 12 + 16;
  return o;
}

// sibling = parent - built child (exact: integer histograms)
__global__ void hist_derive_kernel(const FamDesc* __restrict__ fam, const FamState* __restrict__ st,
                                   const NodeRec* __restrict__ nodes, int level, int64_t* __restrict__ hsum,
                                   int32_t* __restrict__ hcnt, int64_t* __restrict__ node_abs) {
  const int f = blockIdx.z;
  const FamDesc fd = fam[f];
  if (!st[f].active || level == 0) return;
  const NodeRec* nd = nodes + fd.node0;
  const int k = blockIdx.y;
  if (k >= (1 << (level - 1))) return;
  const int parent = (1 << (level - 1)) - 1 + k;
  if (nd[parent].state != kNodeSplit) return;
  const int c1 = 2 * parent + 1, c2 = c1 + 1;
  int built, other;
  if (nd[c1].build == 1 && nd[c2].build == 2) {
    built = c1;
    other = c2;
  } else if (nd[c2].build == 1 && nd[c1].build == 2) {
    built = c2;
    other = c1;
  } else {
    return;
  }
  const int first = (1 << level) - 1, pfirst = (1 << (level - 1)) - 1;
  const int64_t hb = fd.hist0 + (static_cast<int64_t>(level & 1) * fd.level_slots + (built - first)) * fd.bins;
  const int64_t ho = fd.hist0 + (static_cast<int64_t>(level & 1) * fd.level_slots + (other - first)) * fd.bins;
  const int64_t hp = fd.hist0 + (static_cast<int64_t>((level - 1) & 1) * fd.level_slots + (parent - pfirst)) * fd.bins;
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < fd.bins; b += gridDim.x * blockDim.x) {
    hsum[ho + b] = hsum[hp + b] - hsum[hb + b];
    hcnt[ho + b] = hcnt[hp + b] - hcnt[hb + b];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0)
    node_abs[fd.node0 + other] = node_abs[fd.node0 + parent] - node_abs[fd.node0 + built];
}

// Screened gain of one candidate plus a rigorous bound on |reference gain - screened gain|.
// ls/ts: fixed-point left/total sums; S: sum|r| of the node (real units); scale = 2^-shift.
// The reference folds sums sequentially (error <= gamma_n * S each), R = T - L rounds once,
// then ((L*L)/lc + (R*R)/rc) - (T*T)/n rounds ~5 more times; the screen's sums are exact on
// the quantised residuals (quantisation <= n * scale / 2). Factor 2 covers both sides.
__device__ __forceinline__ void screen_gain(int64_t ls, int64_t ts, int lc, int n, double scale, double S, double& g,
                                            double& lo, double& hi) {
  const double u = 1.1102230246251565e-16;
  const double L = static_cast<double>(ls) * scale, T = static_cast<double>(ts) * scale;
  const double R = static_cast<double>(ts - ls) * scale;
  const int rc = n - lc;
  // three reciprocals instead of nine divisions; their extra rounding (<= 1 ulp per term) is
  // covered by the 6u term below
  const double ilc = 1.0 / lc, irc = 1.0 / rc, in = 1.0 / n;
  const double A = L * L * ilc, B = R * R * irc, P = T * T * in;
  g = (A + B) - P;
  const double nu = static_cast<double>(n) * u;
  const double gam = nu / (1.0 - nu);
  const double q = static_cast<double>(n) * 0.5 * scale;
  const double EL = gam * S + q, ET = gam * S + q, ER = 2.0 * gam * S + 2.0 * q + u * fabs(R);
  const double aL = fabs(L) + EL, aR = fabs(R) + ER, aT = fabs(T) + ET;
  const double dA = ((2.0 * fabs(L) + EL) * EL + 4.0 * u * aL * aL) * ilc;
  const double dB = ((2.0 * fabs(R) + ER) * ER + 4.0 * u * aR * aR) * irc;
  const double dP = ((2.0 * fabs(T) + ET) * ET + 4.0 * u * aT * aT) * in;
  const double delta = 2.0 * (dA + dB + dP + 6.0 * u * (A + B + P)) * (1.0 + 8.0 * u) + 1e-300;
  lo = g - delta;
  hi = g + delta;
}

template <class T>
__device__ __forceinline__ T warp_incl_scan(T v, int lane) {
  for (int o = 1; o < 32; o <<= 1) {
    const T t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// One thread per (family, node at level, rep). pass 0: max lower bound per node. pass 1:
// window membership (hi >= LO and hi > 0), per-feature best candidate, node window count.
__global__ void screen_kernel(const FamDesc* __restrict__ fam, const FamState* __restrict__ st,
                              NodeRec* __restrict__ nodes, int level, const int64_t* __restrict__ hsum,
                              const int32_t* __restrict__ hcnt, const int64_t* __restrict__ node_abs,
                              const int32_t* __restrict__ rep_boff, const int32_t* __restrict__ rep_nb,
                              WinRec* __restrict__ win, int nrep_max, int level_slots_max, int pass) {
  // warp per (node, rep), lanes over the rep's bins: coalesced histogram reads, warp prefix
  // scans for the left count / sum, every candidate's screen in parallel
  const int f = blockIdx.z;
  const FamDesc fd = fam[f];
  if (!st[f].active) return;
  const int local = blockIdx.y;
  if (local >= (1 << level)) return;
  const int lane = threadIdx.x & 31;
  const int jj = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (jj >= fd.nrep) return;
  const int s = (1 << level) - 1 + local;
  NodeRec& nd = nodes[fd.node0 + s];
  if (nd.state != 0 || nd.build == 0) return;
  const int n = nd.n;
  const int64_t hb = fd.hist0 + (static_cast<int64_t>(level & 1) * fd.level_slots + local) * fd.bins +
                     rep_boff[fd.rep0 + jj];
  const int nb = rep_nb[fd.rep0 + jj];
  const double scale = ldexp(1.0, -st[f].shift);
  const double S = static_cast<double>(node_abs[fd.node0 + s]) * scale * (1.0 + 1e-12);
  int64_t ts = 0;
  for (int b = lane; b < nb; b += 32) ts += hsum[hb + b];
  for (int o = 16; o > 0; o >>= 1) ts += __shfl_xor_sync(0xffffffffu, ts, o);
  const double LO = pass ? lo_from_key(nd.lokey) : 0.0;
  double best_lo = -INFINITY, bg = -INFINITY, bl = 0.0;
  int bb = 0x7fffffff, blc = 0, count = 0, mlc = 0, carry_c = 0;
  int64_t carry_s = 0;
  for (int b0 = 0; b0 < nb; b0 += 32) {
    const int b = b0 + lane;
    const int cc = b < nb ? hcnt[hb + b] : 0;
    const int64_t sv = b < nb ? hsum[hb + b] : 0;
    const int ic = warp_incl_scan(cc, lane) + carry_c;
    const int64_t is = warp_incl_scan(sv, lane) + carry_s;
    if (b < nb && cc > 0 && ic < n) {  // a boundary after bin b (a later bin is non-empty)
      double g, lo, hi;
      screen_gain(is, ts, ic, n, scale, S, g, lo, hi);
      if (!pass) {
        best_lo = fmax(best_lo, lo);
      } else if (hi >= LO && hi > 0.0) {
        ++count;
        mlc = max(mlc, ic);
        if (g > bg || (g == bg && b < bb)) {
          bg = g;
          bl = lo;
          bb = b;
          blc = ic;
        }
      }
    }
    carry_c = __shfl_sync(0xffffffffu, ic, 31);
    carry_s = __shfl_sync(0xffffffffu, is, 31);
  }
  if (!pass) {
    for (int o = 16; o > 0; o >>= 1) best_lo = fmax(best_lo, __shfl_xor_sync(0xffffffffu, best_lo, o));
    if (lane == 0 && best_lo > -INFINITY)
      atomicMax(reinterpret_cast<unsigned long long*>(&nd.lokey), lo_key(best_lo));
  } else {
    for (int o = 16; o > 0; o >>= 1) {
      count += __shfl_xor_sync(0xffffffffu, count, o);
      mlc = max(mlc, __shfl_xor_sync(0xffffffffu, mlc, o));
      const double og = __shfl_xor_sync(0xffffffffu, bg, o);
      const double ol = __shfl_xor_sync(0xffffffffu, bl, o);
      const int ob = __shfl_xor_sync(0xffffffffu, bb, o);
      const int olc = __shfl_xor_sync(0xffffffffu, blc, o);
      if (og > bg || (og == bg && ob < bb)) {
        bg = og;
        bl = ol;
        bb = ob;
        blc = olc;
      }
    }
    if (lane == 0) {
      WinRec w;
      w.best_g = bg;
      w.best_lo = bl;
      w.best_bin = count ? bb : -1;
      w.flag = count > 0;
      w.count = count;
      w.best_lc = blc;
      w.eq = 0;
      w.maxlc = mlc;
      win[(static_cast<int64_t>(f) * level_slots_max + local) * nrep_max + jj] = w;
      if (count) atomicAdd(&nd.wcount, count);
    }
  }
}

struct ExactItem {
  int32_t fam;
  int16_t slot;
  int16_t rep;  // -1: node total
};

// Tie classes: a node whose window holds exactly one candidate per feature, all with the same
// left count, is one tie class if every window feature orders the node's rows exactly like the
// lowest one (identical folds, identical reference gains; strict > keeps the lowest feature).
// Prep queues one order-equivalence check per (node, other window feature).
// The per-node decision kernels below run a warp per (family, node) with lanes over the
// node's features (window records read in parallel; ballots replace the serial scans).
__device__ __forceinline__ int first_flag_feature(const WinRec* w, int nrep, int from, bool need_count1,
                                                  bool& multi) {
  // lowest flagged feature >= from; multi = some flagged feature has count != 1 (when asked)
  const int lane = threadIdx.x & 31;
  int first = -1;
  multi = false;
  for (int j0 = from; j0 < nrep; j0 += 32) {
    const int j = j0 + lane;
    const bool fl = j < nrep && w[j].flag;
    const unsigned m = __ballot_sync(0xffffffffu, fl);
    if (need_count1 && __any_sync(0xffffffffu, fl && w[j].count != 1)) multi = true;
    if (m && first < 0) first = j0 + __ffs(m) - 1;
  }
  return first;
}

__global__ void tieclass_prep_kernel(const FamDesc* __restrict__ fam, const FamState* __restrict__ st,
                                     NodeRec* __restrict__ nodes, int level, const WinRec* __restrict__ win,
                                     int nrep_max, int level_slots_max, ExactItem* __restrict__ items,
                                     int* __restrict__ n_items) {
  const int f = blockIdx.y;
  const FamDesc fd = fam[f];
  if (!st[f].active) return;
  const int lane = threadIdx.x & 31;
  const int local = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (local >= (1 << level)) return;
  const int s = (1 << level) - 1 + local;
  NodeRec& nd = nodes[fd.node0 + s];
  if (lane == 0) nd.eqf0 = -1;
  if (nd.state != 0 || nd.build == 0 || nd.wcount < 2) return;
  const WinRec* w = win + (static_cast<int64_t>(f) * level_slots_max + local) * nrep_max;
  bool multi;
  const int f0 = first_flag_feature(w, fd.nrep, 0, true, multi);
  if (multi || f0 < 0 || !(w[f0].best_lo > 0.0)) return;
  const int lc0 = w[f0].best_lc;
  bool diff = false;
  for (int j0 = f0 + 1; j0 < fd.nrep; j0 += 32) {
    const int j = j0 + lane;
    if (__any_sync(0xffffffffu, j < fd.nrep && w[j].flag && w[j].best_lc != lc0)) diff = true;
  }
  if (diff) return;
  if (lane == 0) nd.eqf0 = f0;
  for (int j0 = f0 + 1; j0 < fd.nrep; j0 += 32) {
    const int j = j0 + lane;
    const bool fl = j < fd.nrep && w[j].flag;
    const unsigned m = __ballot_sync(0xffffffffu, fl);
    int base = 0;
    if (lane == 0 && m) base = atomicAdd(n_items, __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (fl) items[base + __popc(m & ((1u << lane) - 1u))] = {f, static_cast<int16_t>(s), static_cast<int16_t>(j)};
  }
}

__global__ void decide_kernel(const FamDesc* __restrict__ fam, const FamState* __restrict__ st,
                              NodeRec* __restrict__ nodes, int level, const int32_t* __restrict__ hcnt,
                              const int32_t* __restrict__ rep_boff, const WinRec* __restrict__ win, int nrep_max,
                              int level_slots_max, ExactItem* __restrict__ items, int* __restrict__ n_items,
                              unsigned long long* __restrict__ ctr) {
  (void)hcnt;
  (void)rep_boff;
  const int f = blockIdx.y;
  const FamDesc fd = fam[f];
  if (!st[f].active) return;
  const int lane = threadIdx.x & 31;
  const int local = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (local >= (1 << level)) return;
  const int s = (1 << level) - 1 + local;
  NodeRec& nd = nodes[fd.node0 + s];
  if (nd.state != 0 || nd.build == 0) return;
  const WinRec* w = win + (static_cast<int64_t>(f) * level_slots_max + local) * nrep_max;
  if (nd.wcount == 0) {  // no candidate can have a positive reference gain
    if (lane == 0) nd.state = kNodeLeaf;
    return;
  }
  int pick = -1;
  if (nd.wcount == 1) {
    bool multi;
    const int j = first_flag_feature(w, fd.nrep, 0, false, multi);
    if (j >= 0 && w[j].best_lo > 0.0) pick = j;
  } else if (nd.eqf0 >= 0) {  // one tie class: the lowest feature wins by strict >
    bool all = true;
    for (int j0 = nd.eqf0 + 1; j0 < fd.nrep; j0 += 32) {
      const int j = j0 + lane;
      if (__any_sync(0xffffffffu, j < fd.nrep && w[j].flag && !w[j].eq)) all = false;
    }
    if (all) pick = nd.eqf0;
  }
  if (pick >= 0) {
    if (lane == 0) {
      nd.state = kNodeSplit;
      nd.rep = pick;
      nd.bin = w[pick].best_bin;
      nd.gain = w[pick].best_g;
      nd.lc = w[pick].best_lc;
      atomicAdd(&const_cast<FamState*>(st)[f].screened, 1ull);
    }
    return;
  }
  const int tot = nd.pad_ ? 0 : 1;  // node total still to fold (not precomputed by totals_kernel)
  int k = tot;
  for (int j0 = 0; j0 < fd.nrep; j0 += 32) {
    const int j = j0 + lane;
    k += __popc(__ballot_sync(0xffffffffu, j < fd.nrep && w[j].flag));
  }
  int base = 0;
  if (lane == 0) {
    nd.state = kNodeExact;
    atomicAdd(&const_cast<FamState*>(st)[f].exact, 1ull);
    base = atomicAdd(n_items, k);
    atomicAdd(ctr + kCtrExactChains, static_cast<unsigned long long>(k));
    atomicAdd(ctr + kCtrExactNodes, 1ull);
    if (tot) items[base] = {f, static_cast<int16_t>(s), static_cast<int16_t>(-1)};
  }
  base = __shfl_sync(0xffffffffu, base, 0) + tot;
  for (int j0 = 0; j0 < fd.nrep; j0 += 32) {
    const int j = j0 + lane;
    const bool fl = j < fd.nrep && w[j].flag;
    const unsigned m = __ballot_sync(0xffffffffu, fl);
    if (fl) items[base + __popc(m & ((1u << lane) - 1u))] = {f, static_cast<int16_t>(s), static_cast<int16_t>(j)};
    base += __popc(m);
  }
}

// One warp per check: walk the lowest window feature's presorted list restricted to the node;
// the other feature must tie exactly where it ties and increase where it increases.
// Order equivalence of g with f0 on the node's rows <=> the map code_f0 -> code_g over those rows
// is a function that strictly increases (ties align, and the stable sorts by (code, canonical
// position) then coincide). CTA per item: phi[a] = the g code of some row with f0 code a (racy
// plain stores), every row must agree with phi, phi must increase over the present a. Rows come
// from the node's order-0 segment, in any order - no scan of the presorted lists.
template <typename CodeT>
__global__ void __launch_bounds__(256) tieclass_phi_kernel(
    const FamDesc* __restrict__ fam, const NodeRec* __restrict__ nodes, const ExactItem* __restrict__ items,
    const int* __restrict__ n_items, int level, int Dp, const CodeT* __restrict__ codes_c,
    const int32_t* __restrict__ ord_cur, const int32_t* __restrict__ rep_nb, WinRec* __restrict__ win,
    int nrep_max, int level_slots_max) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint16_t* phi = reinterpret_cast<uint16_t*>(smem);
  const int tid = threadIdx.x, lane = tid & 31;
  const int total = *n_items;
  for (int wi = blockIdx.x; wi < total; wi += gridDim.x) {
    const ExactItem it = items[wi];
    const FamDesc fd = fam[it.fam];
    const NodeRec& nd = nodes[fd.node0 + it.slot];
    const int f0 = nd.eqf0, g = it.rep, nv = nd.n;
    const int nb = rep_nb[fd.rep0 + f0];
    const int32_t* rows = ord_cur + fd.pos0 + nd.seg;
    const CodeT* cb = codes_c + fd.pos0 * Dp;
    __syncthreads();  // previous item done with phi
    for (int a = tid; a < nb; a += blockDim.x) phi[a] = 0xFFFFu;
    __syncthreads();
    for (int i = tid; i < nv; i += blockDim.x) {
      const int64_t p = rows[i];
      phi[cb[p * Dp + f0]] = static_cast<uint16_t>(cb[p * Dp + g]);
    }
    __syncthreads();
    bool bad = false;
    for (int i = tid; i < nv; i += blockDim.x) {
      const int64_t p = rows[i];
      bad |= phi[cb[p * Dp + f0]] != static_cast<uint16_t>(cb[p * Dp + g]);
    }
    if (tid < 32) {  // phi strictly increasing over the present f0 codes
      int carry = -1;
      for (int a0 = 0; a0 < nb; a0 += 32) {
        const int a = a0 + lane;
        const int v = a < nb ? phi[a] : 0xFFFF;
        const bool present = v != 0xFFFF;
        const unsigned m = __ballot_sync(0xffffffffu, present);
        const unsigned lt = m & ((1u << lane) - 1u);
        int pv = __shfl_sync(0xffffffffu, v, lt ? 31 - __clz(lt) : 0);
        if (!lt) pv = carry;
        if (present && pv >= 0 && v <= pv) bad = true;
        if (m) carry = __shfl_sync(0xffffffffu, v, 31 - __clz(m));
      }
    }
    bad = __syncthreads_or(bad);
    const int local = it.slot - ((1 << level) - 1);
    if (tid == 0) win[(static_cast<int64_t>(it.fam) * level_slots_max + local) * nrep_max + g].eq = !bad;
  }
}

template <typename CodeT>
__global__ void __launch_bounds__(256) tieclass_check_kernel(
    const FamDesc* __restrict__ fam, const NodeRec* __restrict__ nodes, const ExactItem* __restrict__ items,
    const int* __restrict__ n_items, int level, int Dp, const CodeT* __restrict__ codes_c,
    const int32_t* __restrict__ ord, const int16_t* __restrict__ nodeid, WinRec* __restrict__ win, int nrep_max,
    int level_slots_max) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int total = *n_items;
  for (int wi = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; wi < total; wi += warps) {
    const ExactItem it = items[wi];
    const FamDesc fd = fam[it.fam];
    const NodeRec& nd = nodes[fd.node0 + it.slot];
    const int f0 = nd.eqf0, g = it.rep, nv = nd.n, n = fd.n;
    const int32_t* L = ord + fd.ord0 + static_cast<int64_t>(f0) * n;
    int pf = -1, pg = -1, seen = 0;
    bool bad = false;
    int p_next = lane < n ? L[lane] : 0;
    for (int i0 = 0; i0 < n && seen < nv; i0 += 32) {
      const int i = i0 + lane;
      const int p = p_next;
      p_next = i + 32 < n ? L[i + 32] : 0;
      const bool mem = i < n && nodeid[fd.pos0 + p] == it.slot;
      const int a = mem ? static_cast<int>(codes_c[(fd.pos0 + p) * Dp + f0]) : 0;
      const int b = mem ? static_cast<int>(codes_c[(fd.pos0 + p) * Dp + g]) : 0;
      const unsigned m = __ballot_sync(0xffffffffu, mem);
      seen += __popc(m);
      const unsigned lt = m & ((1u << lane) - 1u);
      const int src = lt ? 31 - __clz(lt) : lane;
      int qa = __shfl_sync(0xffffffffu, a, src), qb = __shfl_sync(0xffffffffu, b, src);
      if (!lt) {
        qa = pf;
        qb = pg;
      }
      if (mem && qa >= 0 && ((a == qa) != (b == qb) || b < qb)) bad = true;
      if (m) {
        const int last = 31 - __clz(m);
        pf = __shfl_sync(0xffffffffu, a, last);
        pg = __shfl_sync(0xffffffffu, b, last);
      }
    }
    bad = __any_sync(0xffffffffu, bad);
    const int local = it.slot - ((1 << level) - 1);
    if (lane == 0) win[(static_cast<int64_t>(it.fam) * level_slots_max + local) * nrep_max + g].eq = !bad;
  }
}

// Decide screened nodes; queue the rest for reference-order re-evaluation.
__device__ __forceinline__ double warp_fold_gather(const double* __restrict__ v, const int32_t* __restrict__ idx,
                                                   int n) {
  // Software-pipelined: the next 128 gathers (L2 latency) are in flight while the current 128
  // values are folded in order (the dependent FP64 add chain).
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  double x[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int i = 32 * c + lane;
    x[c] = i < n ? v[idx[i]] : 0.0;
  }
  for (int i0 = 0; i0 < n; i0 += 128) {
    double y[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = i0 + 128 + 32 * c + lane;
      y[c] = i < n ? v[idx[i]] : 0.0;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int base = i0 + 32 * c;
      if (base >= n) break;
      const int m = min(32, n - base);
      if (m == 32) {
#pragma unroll
        for (int l0 = 0; l0 < 32; l0 += 8) {
          double t[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) t[k] = __shfl_sync(0xffffffffu, x[c], l0 + k);
#pragma unroll
          for (int k = 0; k < 8; ++k) s = fs_add(s, t[k]);
        }
      } else {
        for (int l = 0; l < m; ++l) s = fs_add(s, __shfl_sync(0xffffffffu, x[c], l));
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) x[c] = y[c];
  }
  return s;
}

// Node totals (costmodel.cpp:47, sum_residuals over the feature-0 list) for every node of the
// level that will be screened, on a forked stream: the reference-order chains run while the
// histogram / screen / tie-class kernels of the same level do. nd.pad_ = 1 marks the total valid
// (exact decisions and leaf values then reuse it - the same fold over the same segment).
__global__ void totals_kernel(const FamDesc* __restrict__ fam, const FamState* __restrict__ st,
                              NodeRec* __restrict__ nodes, int level, const int32_t* __restrict__ ord_cur,
                              const double* __restrict__ resid) {
  const int f = blockIdx.y;
  const FamDesc fd = fam[f];
  if (!st[f].active) return;
  const int local = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (local >= (1 << level)) return;
  NodeRec& nd = nodes[fd.node0 + (1 << level) - 1 + local];
  if (nd.state != 0 || nd.build == 0 || nd.n <= 0) return;
  const double t = warp_fold_gather(resid + fd.pos0, ord_cur + fd.pos0 + nd.seg, nd.n);
  if ((threadIdx.x & 31) == 0) {
    nd.total = t;
    nd.pad_ = 1;
  }
}


// sum_residuals (costmodel.cpp:36-40) of v[idx[0..n)) in list order by one warp: four chunks of
// 32 gathers are in flight at once, then each chunk's values are added in lane order (shuffles
// hoisted ahead of the dependent add chain). Every lane returns the sum.

// One warp per item: reference-order folds. Item rep < 0: node total over the order-0 list
// (sum_residuals(order[0]), costmodel.cpp:47). Item rep j: best_split's left sums over feature j's
// presorted list restricted to the node (:50-55), recorded at every value boundary.
// exact folds of nodes below a quarter of the family go through exact_small_kernel
__device__ __forceinline__ bool exact_is_small(int nv, int n) { return nv < n; }

// Exact reference-order folds for SMALL nodes (nv * 4 < n): instead of scanning the feature's
// full presorted list for the node's members (exact_kernel; costs O(n) gathers per item however
// small the node), a CTA compacts the node's rows in canonical order (a coalesced scan of the
// node ids), stable-sorts them by the feature's code (the presorted order restricted to the
// node is exactly (code, canonical position) order), and warp 0 folds them - the same adds in
// the same order as best_split (costmodel.cpp:50-69), stopping at the last window candidate.
template <typename CodeT>
__global__ void __launch_bounds__(kSortThreads) exact_small_kernel(
    const FamDesc* __restrict__ fam, NodeRec* __restrict__ nodes, const ExactItem* __restrict__ items,
    const int* __restrict__ n_items, int level, int Dp, const CodeT* __restrict__ codes_c,
    const double* __restrict__ resid, const int16_t* __restrict__ nodeid, const int32_t* __restrict__ rep_boff,
    double* __restrict__ lbuf, const WinRec* __restrict__ win, int nrep_max, int level_slots_max,
    int32_t* __restrict__ scratch, int n_max) {
  __shared__ SortSmem sm;
  __shared__ int wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int total = *n_items;
  sort_smem_init(sm);
  for (int w = blockIdx.x; w < total; w += gridDim.x) {
    const ExactItem it = items[w];
    if (it.rep < 0) continue;
    const FamDesc fd = fam[it.fam];
    const NodeRec& nd = nodes[fd.node0 + it.slot];
    const int nv = nd.n, n = fd.n;
    if (!exact_is_small(nv, n)) continue;
    const int jj = it.rep;
    const int local = it.slot - ((1 << level) - 1);
    const int need = win[(static_cast<int64_t>(it.fam) * level_slots_max + local) * nrep_max + jj].maxlc;
    double* out = lbuf + fd.lbuf0 + static_cast<int64_t>(local) * fd.bins + rep_boff[fd.rep0 + jj];
    int32_t* A = scratch + static_cast<int64_t>(blockIdx.x) * 2 * n_max;
    int32_t* B = A + n_max;
    // 1. the node's rows in canonical order
    int base = 0;
    for (int p0 = 0; p0 < n; p0 += blockDim.x) {
      const int p = p0 + tid;
      const bool mem = p < n && nodeid[fd.pos0 + p] == it.slot;
      const unsigned m = __ballot_sync(0xffffffffu, mem);
      if (lane == 0) wsum[warp] = __popc(m);
      __syncthreads();
      if (warp == 0) {
        const int v = lane < static_cast<int>(blockDim.x >> 5) ? wsum[lane] : 0;
        int incl = v;
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        wsum[lane] = incl - v;
        if (lane == 31) sm.uniform = incl;  // chunk total (borrowed field)
      }
      __syncthreads();
      if (mem) A[base + wsum[warp] + __popc(m & ((1u << lane) - 1u))] = p;
      base += sm.uniform;
      __syncthreads();
    }
    // 2. stable sort by the feature's code: (code, canonical position) = presorted order
    const CodeT* cj = codes_c + static_cast<int64_t>(fd.pos0) * Dp + jj;
    int32_t* src = A;
    int32_t* dst = B;
    if (stable_digit_pass([&](int i) { return src[i]; }, dst, nv,
                          [&](int p) { return static_cast<int>(cj[static_cast<int64_t>(p) * Dp] & 255u); }, sm)) {
      int32_t* t = src;
      src = dst;
      dst = t;
    }
    __syncthreads();
    if (sizeof(CodeT) == 2) {
      if (stable_digit_pass([&](int i) { return src[i]; }, dst, nv,
                            [&](int p) { return static_cast<int>(cj[static_cast<int64_t>(p) * Dp] >> 8); }, sm)) {
        int32_t* t = src;
        src = dst;
        dst = t;
      }
      __syncthreads();
    }
    // 3. the fold (warp 0; members in list order, boundaries at code changes)
    if (warp == 0) {
      double left = 0.0;
      int prev = -1;
      for (int i0 = 0; i0 < need; i0 += 32) {
        const int i = i0 + lane;
        const int p = i < need ? src[i] : 0;
        const int code = i < need ? static_cast<int>(cj[static_cast<int64_t>(p) * Dp]) : 0;
        const double rv = i < need ? resid[fd.pos0 + p] : 0.0;
        const int cnt = min(32, need - i0);
        for (int l0 = 0; l0 < cnt; l0 += 8) {
          int cc[8];
          double vv[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            cc[k] = __shfl_sync(0xffffffffu, code, l0 + k);
            vv[k] = __shfl_sync(0xffffffffu, rv, l0 + k);
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            if (l0 + k < cnt) {
              if (prev >= 0 && cc[k] != prev && lane == 0) out[prev] = left;
              left = fs_add(left, vv[k]);
              prev = cc[k];
            }
          }
        }
      }
      if (lane == 0 && prev >= 0) out[prev] = left;  // the last window boundary
    }
    __syncthreads();
  }
}

template <typename CodeT>
__global__ void __launch_bounds__(256) exact_kernel(const FamDesc* __restrict__ fam, NodeRec* __restrict__ nodes,
                                                    const ExactItem* __restrict__ items, const int* __restrict__ n_items,
                                                    int level, int Dp, const CodeT* __restrict__ codes_c,
                                                    const double* __restrict__ resid, const int32_t* __restrict__ ord,
                                                    const int32_t* __restrict__ ord_cur,
                                                    const int16_t* __restrict__ nodeid,
                                                    const int32_t* __restrict__ rep_boff, double* __restrict__ lbuf,
                                                    const WinRec* __restrict__ win, int nrep_max,
                                                    int level_slots_max, int small_path) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int total = *n_items;
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < total; w += warps) {
    const ExactItem it = items[w];
    const FamDesc fd = fam[it.fam];
    NodeRec& nd = nodes[fd.node0 + it.slot];
    const int n = nd.n;
    if (it.rep < 0) {
      const double s = warp_fold_gather(resid + fd.pos0, ord_cur + fd.pos0 + nd.seg, n);
      if (lane == 0) nd.total = s;
      continue;
    }
    if (exact_is_small(n, fd.n) && small_path) continue;  // exact_small_kernel folds it
    const int jj = it.rep;
    const int32_t* L = ord + fd.ord0 + static_cast<int64_t>(jj) * fd.n;
    const int local = it.slot - ((1 << level) - 1);
    double* out = lbuf + fd.lbuf0 + static_cast<int64_t>(local) * fd.bins + rep_boff[fd.rep0 + jj];
    double left = 0.0;
    int prev = -1, seen = 0, used = 0;
    // candidates past the feature's largest window left count cannot win (costmodel.cpp:65
    // strict >): the fold stops there
    const int need = win[(static_cast<int64_t>(it.fam) * level_slots_max + local) * nrep_max + jj].maxlc;
    // 4 chunks of 32 list entries in flight: index loads, then the dependent gathers
    for (int i0 = 0; i0 < fd.n && seen < need; i0 += 128) {
      int p[4], code[4];
      double rv[4];
      bool mem[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) p[c] = i0 + 32 * c + lane < fd.n ? L[i0 + 32 * c + lane] : -1;
#pragma unroll
      for (int c = 0; c < 4; ++c) mem[c] = p[c] >= 0 && nodeid[fd.pos0 + p[c]] == it.slot;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        code[c] = mem[c] ? static_cast<int>(codes_c[(fd.pos0 + p[c]) * Dp + jj]) : 0;
        rv[c] = mem[c] ? resid[fd.pos0 + p[c]] : 0.0;
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const unsigned m = __ballot_sync(0xffffffffu, mem[c]);
        seen += __popc(m);
        for (int l0 = 0; l0 < 32; l0 += 8) {
          if (!((m >> l0) & 0xFFu)) continue;
          int cc[8];
          double vv[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            cc[k] = __shfl_sync(0xffffffffu, code[c], l0 + k);
            vv[k] = __shfl_sync(0xffffffffu, rv[c], l0 + k);
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            if (((m >> (l0 + k)) & 1u) && used < need) {
              if (prev >= 0 && cc[k] != prev && lane == 0) out[prev] = left;  // boundary after bin `prev`
              left = fs_add(left, vv[k]);
              prev = cc[k];
              ++used;
            }
          }
        }
      }
    }
    if (lane == 0 && prev >= 0 && used == need) out[prev] = left;  // the last window boundary
  }
}

// Reference decision over the exactly folded candidates: gain = ((L*L)/lc + (R*R)/rc) - (T*T)/n,
// R = T - L (costmodel.cpp:58-62), strict > in (feature, threshold) order (:65).
__global__ void exact_decide_kernel(const FamDesc* __restrict__ fam, const FamState* __restrict__ st,
                                    NodeRec* __restrict__ nodes, int level, const int32_t* __restrict__ hcnt,
                                    const int32_t* __restrict__ rep_boff, const int32_t* __restrict__ rep_nb,
                                    const WinRec* __restrict__ win, int nrep_max, int level_slots_max,
                                    const double* __restrict__ lbuf) {
  const int f = blockIdx.y;
  const FamDesc fd = fam[f];
  if (!st[f].active) return;
  const int local = blockIdx.x * blockDim.x + threadIdx.x;
  if (local >= (1 << level)) return;
  const int s = (1 << level) - 1 + local;
  NodeRec& nd = nodes[fd.node0 + s];
  if (nd.state != kNodeExact) return;
  const WinRec* w = win + (static_cast<int64_t>(f) * level_slots_max + local) * nrep_max;
  const int n = nd.n;
  const double T = nd.total;
  const double parent = fs_div(fs_mul(T, T), static_cast<double>(n));
  double best = 0.0;
  int bj = -1, bb = -1, blc = 0;
  for (int jj = 0; jj < fd.nrep; ++jj) {
    if (!w[jj].flag) continue;
    const int64_t hb = fd.hist0 + (static_cast<int64_t>(level & 1) * fd.level_slots + local) * fd.bins +
                       rep_boff[fd.rep0 + jj];
    const double* lb = lbuf + fd.lbuf0 + static_cast<int64_t>(local) * fd.bins + rep_boff[fd.rep0 + jj];
    if (w[jj].count == 1) {  // its window candidate is the only one of this feature that can win
      const int cum = w[jj].best_lc, b = w[jj].best_bin;
      const double L = lb[b];
      const double R = fs_sub(T, L);
      const double a = fs_div(fs_mul(L, L), static_cast<double>(cum));
      const double r = fs_div(fs_mul(R, R), static_cast<double>(n - cum));
      const double g = fs_sub(fs_add(a, r), parent);
      if (g > best) {
        best = g;
        bj = jj;
        bb = b;
        blc = cum;
      }
      continue;
    }
    int cum = 0;
    for (int b = 0; b < rep_nb[fd.rep0 + jj]; ++b) {
      const int c = hcnt[hb + b];
      if (!c) continue;
      cum += c;
      if (cum >= n || cum > w[jj].maxlc) break;  // folds stop at the last window candidate
      const double L = lb[b];
      const double R = fs_sub(T, L);
      const double a = fs_div(fs_mul(L, L), static_cast<double>(cum));
      const double r = fs_div(fs_mul(R, R), static_cast<double>(n - cum));
      const double g = fs_sub(fs_add(a, r), parent);
      if (g > best) {
        best = g;
        bj = jj;
        bb = b;
        blc = cum;
      }
    }
  }
  if (bj < 0) {
    nd.state = kNodeLeaf;
  } else {
    nd.state = kNodeSplit;
    nd.rep = bj;
    nd.bin = bb;
    nd.gain = best;
    nd.lc = blc;
  }
}

// Split nodes: exact threshold, tree record, stable partition of the order-0 segment in place
// (costmodel.cpp:94-105 for list 0), row -> child ids, child records.
template <typename CodeT>
__global__ void __launch_bounds__(1024) partition_kernel(
    const FamDesc* __restrict__ fam, const FamState* __restrict__ st, NodeRec* __restrict__ nodes, int level, int Dp,
    const CodeT* __restrict__ codes_c, int32_t* __restrict__ ord_cur, int32_t* __restrict__ scratch,
    int16_t* __restrict__ nodeid, const int32_t* __restrict__ rep_orig, const int32_t* __restrict__ rep_boff,
    const double* __restrict__ vals, const int32_t* __restrict__ cle, const int32_t* __restrict__ ord,
    const int32_t* __restrict__ canon, const double* __restrict__ x, int d, TreeRec* __restrict__ trees, int slots) {
  __shared__ int wsum[32];
  __shared__ int base_l, base_r;
  const int f = blockIdx.y;
  const FamDesc fd = fam[f];
  if (!st[f].active) return;
  const int local = blockIdx.x;
  if (local >= (1 << level)) return;
  const int s = (1 << level) - 1 + local;
  NodeRec& nd = nodes[fd.node0 + s];
  if (nd.state != kNodeSplit) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int jj = nd.rep, bin = nd.bin, n = nd.n, seg = nd.seg, lc = nd.lc;
  TreeRec* tr = trees + fd.tree0 + static_cast<int64_t>(st[f].ntrees) * slots;
  if (tid == 0) {
    const int orig = rep_orig[fd.rep0 + jj];
    double thr = vals[fd.bin0 + rep_boff[fd.rep0 + jj] + bin];
    if (thr == 0.0 && fd.negz) {  // +0.0 and -0.0 share a bin: take the last left element's own value
      const int32_t* L = ord + fd.ord0 + static_cast<int64_t>(jj) * fd.n;
      for (int i = cle[fd.bin0 + rep_boff[fd.rep0 + jj] + bin] - 1; i >= 0; --i) {
        if (nodeid[fd.pos0 + L[i]] == s) {
          thr = x[(fd.row0 + canon[fd.pos0 + L[i]]) * d + orig];
          break;
        }
      }
    }
    TreeRec r;
    r.kind = kNodeSplit;
    r.feature = orig;
    r.threshold = thr;
    r.value = 0.0;
    r.gain = nd.gain;
    r.rep = jj;
    r.bin = bin;
    tr[s] = r;
    base_l = 0;
    base_r = 0;
    NodeRec& a = nodes[fd.node0 + 2 * s + 1];
    NodeRec& b = nodes[fd.node0 + 2 * s + 2];
    a.n = lc;
    a.seg = seg;
    b.n = n - lc;
    b.seg = seg + lc;
  }
  int32_t* src = scratch + fd.pos0 + seg;
  int32_t* dst = ord_cur + fd.pos0 + seg;
  for (int i = tid; i < n; i += blockDim.x) src[i] = dst[i];
  __syncthreads();
  const int16_t cl = static_cast<int16_t>(2 * s + 1), cr = static_cast<int16_t>(2 * s + 2);
  // the next chunk's index and code gathers are issued before this chunk's scan and scatter
  int p_nx = tid < n ? src[tid] : 0;
  int c_nx = tid < n ? static_cast<int>(codes_c[(fd.pos0 + p_nx) * Dp + jj]) : 0;
  for (int t0 = 0; t0 < n; t0 += blockDim.x) {
    const int i = t0 + tid;
    const int p = p_nx;
    const bool left = i < n && c_nx <= bin;
    if (i + static_cast<int>(blockDim.x) < n) {
      p_nx = src[i + blockDim.x];
      c_nx = static_cast<int>(codes_c[(fd.pos0 + p_nx) * Dp + jj]);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, left);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    if (warp == 0) {
      const int v = wsum[lane];
      int incl = v;
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      wsum[lane] = incl - v;
    }
    __syncthreads();
    const int lrank = wsum[warp] + __popc(bal & ((1u << lane) - 1u));
    if (i < n) {
      if (left) {
        dst[base_l + lrank] = p;
        nodeid[fd.pos0 + p] = cl;
      } else {
        dst[lc + base_r + (i - t0) - lrank] = p;
        nodeid[fd.pos0 + p] = cr;
      }
    }
    __syncthreads();  // every thread has used base_l / base_r for this tile
    if (warp == 31 && lane == 0) {  // tile total = warp 31's exclusive prefix + its own count
      const int tile_left = wsum[31] + __popc(bal);
      const int tile = min(static_cast<int>(blockDim.x), n - t0);
      base_l += tile_left;
      base_r += tile - tile_left;
    }
    __syncthreads();
  }
}

// Leaves: value = (reference-order total) / n (costmodel.cpp:86), prediction += lr * value
// (:88-90); tree record. One warp per (family, slot).
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
// CTA-wide exact sequential fold of a long gathered chain (sum_residuals, costmodel.cpp:36-40) by
// midpoint speculation (the warp version is fold_spec): the block's double-double sum of
// x_0..x_{m-1} estimates the exact prefix P; thread 0 folds x_0..x_{m-1} from 0.0 (the true S_m)
// while threads t = 1..255 fold x_m..x_{n-1} from the doubles P + (t-128) ulp; the thread whose
// start is bit-identical to S_m holds S_n. A miss finishes the chain from S_m (same result).
// All 256 threads must call it; the result is returned to every thread.
__device__ __forceinline__ double warp_fold_gather_from(const double* __restrict__ v, const int32_t* __restrict__ idx,
                                                        int n, double s) {
  // warp_fold_gather with a per-lane start value: every lane folds the same sequence (loaded
  // cooperatively, 128 gathers in flight ahead of the adds) from its own start
  const int lane = threadIdx.x & 31;
  double x[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int i = 32 * c + lane;
    x[c] = i < n ? v[idx[i]] : 0.0;
  }
  for (int i0 = 0; i0 < n; i0 += 128) {
    double y[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = i0 + 128 + 32 * c + lane;
      y[c] = i < n ? v[idx[i]] : 0.0;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int base = i0 + 32 * c;
      if (base >= n) break;
      const int m = min(32, n - base);
      if (m == 32) {
#pragma unroll
        for (int l0 = 0; l0 < 32; l0 += 8) {
          double t[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) t[k] = __shfl_sync(0xffffffffu, x[c], l0 + k);
#pragma unroll
          for (int k = 0; k < 8; ++k) s = fs_add(s, t[k]);
        }
      } else {
        for (int l = 0; l < m; ++l) s = fs_add(s, __shfl_sync(0xffffffffu, x[c], l));
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) x[c] = y[c];
  }
  return s;
}

__device__ __forceinline__ double cta_fold_spec(const double* __restrict__ v, const int32_t* __restrict__ idx, int n,
                                                double* red /* smem [2*8+2] */) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = static_cast<int>(blockDim.x >> 5);
  if (n < 4096 || nw < 2) {  // short chain: warp 0 folds it
    if (warp == 0) {
      const double r = warp_fold_gather_from(v, idx, n, 0.0);
      if (lane == 0) red[16] = r;
    }
    __syncthreads();
    const double r = red[16];
    __syncthreads();
    return r;
  }
  const int m = n >> 1;
  // exact-prefix estimate of x_0..x_{m-1}: double-double partial sums (8 gathers in flight)
  double hi = 0.0, lo = 0.0;
  for (int i0 = tid; i0 < m; i0 += 8 * blockDim.x) {
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = i0 + k * blockDim.x;
      a[k] = i < m ? v[idx[i]] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      double s, e;
      two_sum(hi, a[k], s, e);
      hi = s;
      lo = fs_add(lo, e);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double oh = __shfl_xor_sync(0xffffffffu, hi, o), ol = __shfl_xor_sync(0xffffffffu, lo, o);
    double s, e;
    two_sum(hi, oh, s, e);
    hi = s;
    lo = fs_add(fs_add(lo, ol), e);
  }
  if (lane == 0) {
    red[warp] = hi;
    red[8 + warp] = lo;
  }
  __syncthreads();
  if (tid == 0) {
    double h = 0.0, l = 0.0;
    for (int w = 0; w < nw; ++w) {
      double s, e;
      two_sum(h, red[w], s, e);
      h = s;
      l = fs_add(fs_add(l, red[8 + w]), e);
    }
    red[17] = fs_add(h, l);
  }
  __syncthreads();
  const double P = red[17];
  // warp 0 folds the first half from 0.0 (the true S_m); warps 1.. fold the second half from
  // the candidate starts P + k ulp, k centred on 0 (32 * (nw - 1) candidates)
  const int cand = tid - 32;  // 0 .. 32*(nw-1)-1
  const double start = warp == 0 ? 0.0 : ord_dbl(dbl_ord(P) + (cand - 16 * (nw - 1)));
  const double r = warp == 0 ? warp_fold_gather_from(v, idx, m, 0.0)
                             : warp_fold_gather_from(v, idx + m, n - m, start);
  __shared__ int hit;
  if (tid == 0) {
    red[16] = r;  // S_m
    hit = 0;
  }
  __syncthreads();
  if (warp > 0 && __double_as_longlong(start) == __double_as_longlong(red[16])) {
    red[17] = r;
    hit = 1;
  }
  __syncthreads();
  if (!hit && warp == 0) {  // speculation missed: finish from the true midpoint
    const double t = warp_fold_gather_from(v, idx + m, n - m, red[16]);
    if (lane == 0) red[17] = t;
  }
  __syncthreads();
  const double out = red[17];
  __syncthreads();
  return out;
}

// Leaves (costmodel.cpp:85-91): a CTA per (family, heap slot) - value = reference-order fold of
// the leaf's order-0 segment / n (cta_fold_spec), then pred += lr*value over its rows.
__global__ void __launch_bounds__(256) leaf_cta_kernel(const FamDesc* __restrict__ fam, int F,
                                                       const FamState* __restrict__ st, NodeRec* __restrict__ nodes,
                                                       int slots, const int32_t* __restrict__ ord_cur,
                                                       const double* __restrict__ resid, double* __restrict__ pred,
                                                       TreeRec* __restrict__ trees) {
  __shared__ double red[18];
  const int f = blockIdx.y, s = blockIdx.x;
  if (f >= F) return;
  const FamDesc fd = fam[f];
  if (!st[f].active) return;
  NodeRec& nd = nodes[fd.node0 + s];
  if (nd.state != kNodeLeaf || nd.n == 0) return;
  if (s > 0 && nodes[fd.node0 + ((s - 1) >> 1)].state != kNodeSplit) return;
  const int n = nd.n;
  const int32_t* L = ord_cur + fd.pos0 + nd.seg;
  const double sum = nd.pad_ ? nd.total : cta_fold_spec(resid + fd.pos0, L, n, red);
  const double value = fs_div(sum, static_cast<double>(n));
  const double step = fs_mul(fd.lr, value);
  // prediction update, 8 rows per thread in flight (index and prediction gathers issued before
  // the stores: the compiler cannot prove the arrays do not alias)
  for (int i0 = 0; i0 < n; i0 += 8 * static_cast<int>(blockDim.x)) {
    int64_t pp[8];
    double pv[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = i0 + k * blockDim.x + threadIdx.x;
      pp[k] = i < n ? fd.pos0 + L[i] : -1;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) pv[k] = pp[k] >= 0 ? pred[pp[k]] : 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (pp[k] >= 0) pred[pp[k]] = fs_add(pv[k], step);
  }
  if (threadIdx.x == 0) {
    nd.value = value;
    TreeRec r;
    r.kind = kNodeLeaf;
    r.feature = -1;
    r.threshold = 0.0;
    r.value = value;
    r.gain = 0.0;
    r.rep = -1;
    r.bin = 0;
    trees[fd.tree0 + static_cast<int64_t>(st[f].ntrees) * slots + s] = r;
  }
}

__global__ void leaf_kernel(const FamDesc* __restrict__ fam, int F, const FamState* __restrict__ st,
                            NodeRec* __restrict__ nodes, int slots, const int32_t* __restrict__ ord_cur,
                            const double* __restrict__ resid, double* __restrict__ pred, TreeRec* __restrict__ trees) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int f = static_cast<int>(w / slots), s = static_cast<int>(w % slots);
  if (f >= F) return;
  const FamDesc fd = fam[f];
  if (!st[f].active) return;
  NodeRec& nd = nodes[fd.node0 + s];
  if (nd.state != kNodeLeaf || nd.n == 0) return;
  // a slot is a leaf of this tree only if its parent split (or it is the root)
  if (s > 0 && nodes[fd.node0 + ((s - 1) >> 1)].state != kNodeSplit) return;
  const int n = nd.n;
  const int32_t* L = ord_cur + fd.pos0 + nd.seg;
  // the same fold as the node total when totals_kernel already produced it (costmodel.cpp:86)
  const double sum = nd.pad_ ? nd.total : warp_fold_gather(resid + fd.pos0, L, n);
  const double value = fs_div(sum, static_cast<double>(n));
  const double step = fs_mul(fd.lr, value);
  // prediction update, 8 rows per lane in flight (a plain loop serialises on L2 latency:
  // the compiler cannot prove the index and prediction arrays do not alias)
  for (int i0 = 0; i0 < n; i0 += 256) {
    int64_t pp[8];
    double pv[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = i0 + 32 * k + lane;
      pp[k] = i < n ? fd.pos0 + L[i] : -1;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) pv[k] = pp[k] >= 0 ? pred[pp[k]] : 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (pp[k] >= 0) pred[pp[k]] = fs_add(pv[k], step);
  }
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
    trees[fd.tree0 + static_cast<int64_t>(st[f].ntrees) * slots + s] = r;
  }
}

// Commit the round's tree or stop (costmodel.cpp:212), then MSE over canonical rows (:215-220).
// The MSE is a fixed-order tree reduction: deterministic, within 1e-15 relative of the
// reference's sequential fold (it never feeds back into the model).
// MSE per round (costmodel.cpp:215-220; a fixed-order reduction - it never feeds back):
// blocks of kMseRows rows per family produce partials (block tree reduction), mse_final_kernel
// adds them in block order; it also commits the tree or applies the early stop (:212).
constexpr int kMseRows = 2048;
constexpr int kExactSmallCtas = 64;  // CTAs of exact_small_kernel (items loop over them)
__device__ __forceinline__ bool round_commits(const FamDesc& fd, const FamState& st, const NodeRec* nodes) {
  if (!st.active) return false;
  const NodeRec& root = nodes[fd.node0];
  return !(root.state == kNodeLeaf && root.value == 0.0);
}
__global__ void mse_partial_kernel(const FamDesc* __restrict__ fam, const FamState* __restrict__ st,
                                   const NodeRec* __restrict__ nodes, const double* __restrict__ target_c,
                                   const double* __restrict__ pred, double* __restrict__ part, int max_blocks) {
  __shared__ double red[256];
  const int f = blockIdx.y;
  const FamDesc fd = fam[f];
  const int r0 = blockIdx.x * kMseRows;
  if (r0 >= fd.n || !round_commits(fd, st[f], nodes)) return;
  const int r1 = min(fd.n, r0 + kMseRows);
  double a = 0.0;
  for (int i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
    const double e = fs_sub(target_c[fd.pos0 + i], pred[fd.pos0 + i]);
    a = fs_add(a, fs_mul(e, e));
  }
  red[threadIdx.x] = a;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = fs_add(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) part[static_cast<int64_t>(f) * max_blocks + blockIdx.x] = red[0];
}
__global__ void mse_final_kernel(const FamDesc* __restrict__ fam, FamState* __restrict__ st,
                                 const NodeRec* __restrict__ nodes, const double* __restrict__ part, int max_blocks,
                                 double* __restrict__ mse, int max_trees) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= gridDim.x * blockDim.x) return;
  const FamDesc fd = fam[f];
  if (!st[f].active) return;
  if (!round_commits(fd, st[f], nodes)) {
    st[f].active = 0;  // single leaf of value exactly 0: the reference stops boosting
    return;
  }
  double a = 0.0;
  const int nb = (fd.n + kMseRows - 1) / kMseRows;
  for (int b = 0; b < nb; ++b) a = fs_add(a, part[static_cast<int64_t>(f) * max_blocks + b]);
  const int t = st[f].ntrees;
  mse[static_cast<int64_t>(f) * max_trees + t] = fs_div(a, static_cast<double>(fd.n));
  st[f].ntrees = t + 1;
  if (t + 1 >= fd.trees) st[f].active = 0;
}

}  // namespace
}  // namespace fit
}  // namespace fs

// ==========================================================================================
// resident trainer: one CTA per family runs EVERY boosting round of the fit in a single launch,
// with all per-row state in shared memory. For families of up to a few thousand rows (configs
// C1-C3) the multi-kernel round above is launch- and L2-latency-bound (~40 launches per round);
// here a round is ~30 block barriers. Same algorithm, same arithmetic, same tie handling.
// ==========================================================================================
#ifndef FS_RES_THREADS
#define FS_RES_THREADS 512
#endif
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

struct ResNode {
  int32_t n, seg, state, rep, bin, lc, wcount, build;
  int32_t eqf0, pad_;  // lowest window feature when the window may be one tie class, else -1
  double gain, value, total;
  unsigned long long lokey;
  unsigned long long absfix;
};

struct ResLayout {
  int ls, slots, cs;
  size_t codes, resid, pred, predv, targ, fix, node, ord0, scratch, hsum, hcnt, lbuf, nodes, win, items, rep, limb, sbuf, stage, clc, binrep,
      vals, cand, total;
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
  L.hsum = o;
  o = res_align(o + static_cast<size_t>(2) * L.ls * bins * 8);
  L.hcnt = o;
  o = res_align(o + static_cast<size_t>(2) * L.ls * bins * 4);
  L.lbuf = o;
  o = res_align(o + static_cast<size_t>(L.ls) * bins * 8);
  L.nodes = o;
  o = res_align(o + static_cast<size_t>(L.slots) * sizeof(ResNode));
  L.win = o;
  o = res_align(o + static_cast<size_t>(L.ls) * nr * sizeof(WinRec));
  L.items = o;
  o = res_align(o + static_cast<size_t>(L.ls) * (nr + 1) * sizeof(int));
  L.rep = o;
  o = res_align(o + 2 * nr * sizeof(int));
  L.limb = o;  // lane-column limb histogram [3][colh][32] u32, 4 x 16-bit limbs of sum |v| per level node,
               // column offset per rep
  o = res_align(o + std::max<size_t>(static_cast<size_t>(3) * colh * 32 * 4 + static_cast<size_t>(L.ls) * 4 * 4 + nr * 4,
                                      8 * 512));
  L.sbuf = o;  // speculative exact folds: spec_bufs member lists of up to n rows (u16)
  o = res_align(o + static_cast<size_t>(spec_bufs) * n * 2);
  L.stage = o;  // exact-fold staging: per warp 32 doubles + 32 codes
  o = res_align(o + static_cast<size_t>(kResWarps) * 32 * 9);
  L.clc = o;  // left count per (node at level, bin)
  o = res_align(o + static_cast<size_t>(L.ls) * bins * 4);
  L.binrep = o;  // feature (rep) of every bin
  o = res_align(o + static_cast<size_t>(bins) * 2);
  L.vals = o;  // threshold value of every bin + original feature of every rep (split records)
  o = res_align(o + static_cast<size_t>(bins) * 8 + nr * 4);
  L.cand = o;  // screened (gain, bound) per (node at level, bin)
  o = res_align(o + static_cast<size_t>(L.ls) * bins * 16);
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



__global__ void __launch_bounds__(kResThreads, 1) fit_resident_kernel(
    const FamDesc* __restrict__ fam, FamState* __restrict__ st, const int* __restrict__ fam_list, int Dp,
    const uint8_t* __restrict__ codes_c, const double* __restrict__ target_c, const double* __restrict__ base,
    const int32_t* __restrict__ ord, const int32_t* __restrict__ ord_root, const int32_t* __restrict__ rep_orig,
    const int32_t* __restrict__ rep_nb, const int32_t* __restrict__ rep_boff, const double* __restrict__ vals,
    const int32_t* __restrict__ cle, const int32_t* __restrict__ canon, const double* __restrict__ x, int d,
    TreeRec* __restrict__ trees, double* __restrict__ mse, int max_trees, int slots_g,
    unsigned long long* __restrict__ ctr, int pred_smem, double* __restrict__ pred_g, int pre_smem, int spec_bufs) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ unsigned long long s_red[32];
  __shared__ double s_dred[32];
  __shared__ int s_wsum[32];
  __shared__ int s_shift, s_nitems, s_ctot;
  __shared__ unsigned long long s_cnt[3];  // screened splits, exact nodes, exact folds
  __shared__ unsigned long long s_why[4];  // exact-node reasons
  const int f = fam_list[blockIdx.x];
  const FamDesc fd = fam[f];
  const int n = fd.n, nrep = fd.nrep, bins = fd.bins, depth = fd.depth;
  const int colh = nrep > 0 ? col_height(nrep, rep_nb + fd.rep0, nullptr) : 1;
  const ResLayout Lo = res_layout(n, nrep, bins, depth, colh, pred_smem != 0, pre_smem != 0, spec_bufs);
  uint16_t* s_sbuf = reinterpret_cast<uint16_t*>(sm + Lo.sbuf);
  uint8_t* s_codes = sm + Lo.codes;  // [nrep][cs]
  const int cs = Lo.cs;
  uint32_t* s_limb = reinterpret_cast<uint32_t*>(sm + Lo.limb);  // [3][colh][32]
  uint32_t* s_absl = s_limb + 3 * colh * 32;                      // [level node][4]
  int* s_cofs = reinterpret_cast<int*>(s_absl + Lo.ls * 4);        // [nrep]
  double* s_cand = reinterpret_cast<double*>(sm + Lo.cand);  // [level node][bin] x (g, delta)
  int* s_clc = reinterpret_cast<int*>(sm + Lo.clc);           // [level node][bin] left count
  uint16_t* s_binrep = reinterpret_cast<uint16_t*>(sm + Lo.binrep);
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
  __syncthreads();

  int ntrees = 0;
  for (int round = 0; round < fd.trees; ++round) {
    // ---- residuals (costmodel.cpp:204-206), fixed point, per-round reset ----------------
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
    for (int s = tid; s < slots; s += kResThreads) {
      ResNode z;
      memset(&z, 0, sizeof z);
      if (s == 0) z.n = n;
      s_nodes[s] = z;
    }
    TreeRec* tr = trees + fd.tree0 + static_cast<int64_t>(ntrees) * slots_g;
    for (int s = tid; s < slots_g; s += kResThreads) {
      TreeRec tz;
      memset(&tz, 0, sizeof tz);
      tr[s] = tz;
    }
    __syncthreads();
    if (tid == 0) {
      unsigned long long m = 0;
      for (int w = 0; w < kResThreads / 32; ++w) m = max(m, s_red[w]);
      s_shift = kResLimbs == 3 ? fix_shift(m, n) : fix_shift(m, n) - 22;  // n*|v| < 2^61 resp. 2^39
    }
    __syncthreads();
    const int shift = s_shift;
    const double scale = ldexp(1.0, -shift);
    for (int p = tid; p < n; p += kResThreads) s_fix[p] = __double2ll_rn(ldexp(s_resid[p], shift));
    __syncthreads();
      RES_PHASE(0);

    for (int level = 0; level <= depth; ++level) {
      const int first = (1 << level) - 1, nl = 1 << level;
      // ---- plan (level_plan_kernel) --------------------------------------------------------
      if (tid < nl) {
        const int s = first + tid;
        ResNode& nd = s_nodes[s];
        if (level == 0) {
          if (nrep > 0 && node_needs_split(fd, 0, nd.n)) nd.build = 1;
          else nd.state = kNodeLeaf;
        } else if (s_nodes[(s - 1) >> 1].state == kNodeSplit) {
          const bool need = nrep > 0 && node_needs_split(fd, level, nd.n);
          if (!need) nd.state = kNodeLeaf;
          if (s & 1) {
            const int sib = s + 1;
            const bool need_sib = nrep > 0 && node_needs_split(fd, level, s_nodes[sib].n);
            if (need || need_sib) {
              const int small = nd.n <= s_nodes[sib].n ? s : sib;
              s_nodes[small].build = 1;
              s_nodes[small == s ? sib : s].build = 2;
            }
          }
        }
      }
      __syncthreads();
      RES_PHASE(1);
      if (level == depth || nrep == 0) break;
      const int ring = level & 1;
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
        const int rpw = nrep <= 32 ? 32 / nrep : 1;  // rows per warp step
        const int hj = nrep <= 32 ? lane % nrep : lane;
        const int hm = nrep <= 32 ? lane / nrep : 0;
        const bool hact = nrep <= 32 ? hm < rpw : true;
        const int cpad = 3 * colh * 32;
        for (int k = 0; k < nl; ++k) {
          ResNode& nd = s_nodes[first + k];
          if (nd.build != 1) continue;
          const int nv = nd.n;
          const uint16_t* rows = s_ord0 + nd.seg;
          for (int sub0 = 0; sub0 < nv; sub0 += kAtomSub) {
            for (int i = tid; i < cpad; i += kResThreads) s_limb[i] = 0;
            if (tid < 4) s_absl[4 * k + tid] = 0;
            __syncthreads();
            const int q_end = min(nv, sub0 + kAtomSub);
            unsigned long long asum = 0;
            if (hact) {
              if (nrep <= 32) {
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
                  if (hj == 0) asum += static_cast<unsigned long long>(v < 0 ? -v : v);
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
            for (int o = 16; o > 0; o >>= 1) asum += __shfl_xor_sync(0xffffffffu, asum, o);
            if (lane == 0 && asum) {
#pragma unroll
              for (int t = 0; t < 4; ++t) atomicAdd(s_absl + 4 * k + t, static_cast<uint32_t>(asum >> (16 * t)) & 0xFFFFu);
            }
            __syncthreads();
            long long* hk = hs + static_cast<size_t>(k) * bins;
            int* ck = hc + static_cast<size_t>(k) * bins;
            for (int i = tid; i < bins; i += kResThreads) {
              const int j = s_binrep[i], b = i - s_repb[j];
              unsigned __int128 U = 0;
              if (nrep <= 32) {
                for (int m = 0; m < rpw; ++m) {
                  const uint32_t* c = s_limb + b * 32 + j + m * nrep;
                  U += static_cast<unsigned __int128>(c[0]) + (static_cast<unsigned __int128>(c[colh * 32]) << 21) +
                       (static_cast<unsigned __int128>(c[2 * colh * 32]) << 42);
                }
              } else {
                const uint32_t* c = s_limb + (s_cofs[j] + b) * 32 + (j & 31);
                U = static_cast<unsigned __int128>(c[0]) + (static_cast<unsigned __int128>(c[colh * 32]) << 21) +
                    (static_cast<unsigned __int128>(c[2 * colh * 32]) << 42);
              }
              const uint64_t cnt =
                  static_cast<uint64_t>((U + (static_cast<unsigned __int128>(1) << (kResBias - 1))) >> kResBias);
              const long long hv =
                  static_cast<long long>(static_cast<uint64_t>(U - (static_cast<unsigned __int128>(cnt) << kResBias)));
              hk[i] = (sub0 == 0 ? 0ll : hk[i]) + hv;
              ck[i] = (sub0 == 0 ? 0 : ck[i]) + static_cast<int>(cnt);
            }
            if (tid == 0) {
              unsigned long long add = 0;
#pragma unroll
              for (int t = 0; t < 4; ++t) add += static_cast<unsigned long long>(s_absl[4 * k + t]) << (16 * t);
              nd.absfix = (sub0 == 0 ? 0ull : nd.absfix) + add;
              if (sub0 == 0) c_hist_rows += nv;
            }
            __syncthreads();
          }
        }
      }
      RES_PHASE(2);
      // ---- siblings by exact subtraction --------------------------------------------------------
      if (level > 0) {
        const long long* hp = s_hsum + static_cast<size_t>(ring ^ 1) * ls * bins;
        const int* cp = s_hcnt + static_cast<size_t>(ring ^ 1) * ls * bins;
        const int pfirst = (1 << (level - 1)) - 1;
        for (int k2 = 0; k2 < nl / 2; ++k2) {
          const int parent = pfirst + k2;
          if (s_nodes[parent].state != kNodeSplit) continue;
          const int c1 = 2 * parent + 1, c2 = c1 + 1;
          int built, other;
          if (s_nodes[c1].build == 1 && s_nodes[c2].build == 2) {
            built = c1;
            other = c2;
          } else if (s_nodes[c2].build == 1 && s_nodes[c1].build == 2) {
            built = c2;
            other = c1;
          } else {
            continue;
          }
          const size_t ob = static_cast<size_t>(other - first) * bins, bb = static_cast<size_t>(built - first) * bins;
          const size_t pb = static_cast<size_t>(k2) * bins;
          for (int b = tid; b < bins; b += kResThreads) {
            hs[ob + b] = hp[pb + b] - hs[bb + b];
            hc[ob + b] = cp[pb + b] - hc[bb + b];
          }
          if (tid == 0) s_nodes[other].absfix = s_nodes[parent].absfix - s_nodes[built].absfix;
        }
        __syncthreads();
      RES_PHASE(3);
      }
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
                long long is = 0, ts = 0;
                for (int t = 0; t < nb; ++t) {
                  const long long hv = h[t];
                  ts += hv;
                  if (t <= b) {
                    is += hv;
                    ic += c[t];
                  }
                }
                s_clc[ci] = ic;
                const int nv = ndp->n;
                if (c[b] > 0 && ic < nv) {
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
        }
      }
      RES_PHASE(4);
      // ---- tie classes: a window whose candidates (one per feature, equal left counts) come
      // from features whose presorted orders coincide on the node's rows has one reference
      // gain for all of them (identical folds), so the lowest feature wins by strict > without
      // any fold. Check order equivalence against the lowest window feature in parallel.
      if (tid == 0) s_neq = 0;
      __syncthreads();
      if (tid < nl) {
        const int k = tid;
        ResNode& nd = s_nodes[first + k];
        nd.eqf0 = -1;
        if (nd.state == 0 && nd.build != 0 && nd.wcount >= 2) {
          const WinRec* w = s_win + k * nrep;
          int f0 = -1, lc0 = -1;
          bool ok = true;
          for (int j = 0; j < nrep && ok; ++j) {
            if (!w[j].flag) continue;
            if (w[j].count != 1) ok = false;
            if (f0 < 0) {
              f0 = j;
              lc0 = w[j].best_lc;
            } else if (w[j].best_lc != lc0) {
              ok = false;
            }
          }
          if (ok && f0 >= 0 && w[f0].best_lo > 0.0) {
            nd.eqf0 = f0;
            for (int j = f0 + 1; j < nrep; ++j)
              if (w[j].flag) s_items[atomicAdd(&s_neq, 1)] = (first + k) << 16 | j;
          }
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
            const int cb = b < nb ? c[b] : 0;
            const int cum = warp_incl_scan(cb, lane) + carry;
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
            carry = __shfl_sync(0xffffffffu, cum, 31);
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
      // ---- split records: threshold, tree record, children -------------------------------------
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
          tr[s] = r;
          ResNode& a = s_nodes[2 * s + 1];
          ResNode& b = s_nodes[2 * s + 2];
          a.n = nd.lc;
          a.seg = nd.seg;
          b.n = nd.n - nd.lc;
          b.seg = nd.seg + nd.lc;
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
    for (int s = warp; s < slots; s += kResThreads / 32) {
      ResNode& nd = s_nodes[s];
      if (nd.state != kNodeLeaf || nd.n == 0) continue;
      if (s > 0 && s_nodes[(s - 1) >> 1].state != kNodeSplit) continue;
      const int nv = nd.n;
      const double sum = fold_spec(s_resid, s_ord0 + nd.seg, nv);  // warp-collective
      const double value = fs_div(sum, static_cast<double>(nv));
      const double step = fs_mul(fd.lr, value);
      for (int i = lane; i < nv; i += 32) {
        const int p = s_ord0[nd.seg + i];
        s_pred[p] = fs_add(s_pred[p], step);
      }
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
        tr[s] = r;
      }
    }
    __syncthreads();
      RES_PHASE(10);
    // ---- commit / early stop (costmodel.cpp:212) and MSE (:215-220) --------------------------
    if (s_nodes[0].state == kNodeLeaf && s_nodes[0].value == 0.0) break;  // uniform (smem)
    double a = 0.0;
    for (int p = tid; p < n; p += kResThreads) {
      const double e = fs_sub(s_targ[p], s_pred[p]);
      a = fs_add(a, fs_mul(e, e));
    }
    for (int o = 16; o > 0; o >>= 1) a = fs_add(a, __shfl_down_sync(0xffffffffu, a, o));
    if (lane == 0) s_dred[warp] = a;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < kResThreads / 32; ++w) t = fs_add(t, s_dred[w]);
      mse[static_cast<int64_t>(f) * max_trees + ntrees] = fs_div(t, static_cast<double>(n));
    }
    ++ntrees;
    __syncthreads();
      RES_PHASE(11);
  }
  if (tid == 0) {
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
  }
}

}  // namespace
}  // namespace fit
}  // namespace fs

namespace fs {
namespace fit {
namespace {

constexpr int kCompileSlots = 255;  // heap slots of a depth-7 tree (device compile limit)

// ==========================================================================================
// fit epilogue on the device: per family, the reference pre-order export of every tree
// (costmodel.cpp:82-83 node numbering, :108-111 left before right) and the compiled predict form
// (forest.cuh: complete heap of the family's depth, node = rep | bin << 16 where bin is the
// threshold's rank among the rep's distinct values, early leaves replicated under always-left
// nodes), written straight into the family's model blob - no host round trip after a fit.
// Compiled features are representatives; fmap maps them back to original feature ids.
// ==========================================================================================
struct ExportJob {
  unsigned char* blob;
  DevLayout lay;
  int depth;      // heap depth of the compiled form (the family's tree depth)
  int code_wide;  // codes are u16 (always-left rank 0xFFFF instead of 0xFF)
};

__global__ void __launch_bounds__(128) export_compile_kernel(
    const FamDesc* __restrict__ fam, const FamState* __restrict__ st, const TreeRec* __restrict__ trees,
    int slots, const double* __restrict__ mse, int max_trees, const double* __restrict__ base,
    const int32_t* __restrict__ rep_orig, const int32_t* __restrict__ rep_boff, const double* __restrict__ vals,
    const ExportJob* __restrict__ jobs) {
  const int f = blockIdx.x;
  const FamDesc fd = fam[f];
  const ExportJob jb = jobs[f];
  const DevLayout& L = jb.lay;
  unsigned char* B = jb.blob;
  const int T = fd.n > 0 ? st[f].ntrees : 0;
  if (threadIdx.x == 0) {
    ModelMeta mt;
    mt.base = fd.n > 0 ? base[f] : 0.0;
    mt.n_trees = T;
    mt.pad_ = 0;
    mt.screened = static_cast<int64_t>(st[f].screened);
    mt.exact = static_cast<int64_t>(st[f].exact);
    *reinterpret_cast<ModelMeta*>(B + L.meta) = mt;
  }
  double* uthr = reinterpret_cast<double*>(B + L.uthr);
  int32_t* uoff = reinterpret_cast<int32_t*>(B + L.uoff);
  int32_t* fmap = reinterpret_cast<int32_t*>(B + L.fmap);
  for (int b = threadIdx.x; b < fd.bins; b += blockDim.x) uthr[b] = vals[fd.bin0 + b];
  for (int j = threadIdx.x; j <= fd.nrep; j += blockDim.x) {
    uoff[j] = j < fd.nrep ? rep_boff[fd.rep0 + j] : fd.bins;
    if (j < fd.nrep) fmap[j] = rep_orig[fd.rep0 + j];
  }
  const int D = jb.depth, nint = (1 << D) - 1, nleaf = 1 << D, S = L.slots;
  const uint32_t always_left = jb.code_wide ? 0xFFFFu : 0xFFu;
  uint32_t* nodes = reinterpret_cast<uint32_t*>(B + L.nodes);
  double* leafv = reinterpret_cast<double*>(B + L.leafv);
  uint8_t* leafid = B + L.leafid;
  int32_t* cnt = reinterpret_cast<int32_t*>(B + L.cnt);
  int32_t* feat = reinterpret_cast<int32_t*>(B + L.feat);
  double* thr = reinterpret_cast<double*>(B + L.thr);
  int32_t* lft = reinterpret_cast<int32_t*>(B + L.left);
  int32_t* rgt = reinterpret_cast<int32_t*>(B + L.right);
  double* val = reinterpret_cast<double*>(B + L.val);
  double* gain = reinterpret_cast<double*>(B + L.gain);
  double* mo = reinterpret_cast<double*>(B + L.mse);
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    mo[t] = mse[static_cast<int64_t>(f) * max_trees + t];
    const TreeRec* rec = trees + fd.tree0 + static_cast<int64_t>(t) * slots;
    // subtree sizes bottom-up over the heap slots, then pre-order indices top-down
    int size[kCompileSlots], pidx[kCompileSlots];
    for (int h = S - 1; h >= 0; --h) {
      size[h] = 0;
      if (rec[h].kind == kNodeLeaf) size[h] = 1;
      else if (rec[h].kind == kNodeSplit) size[h] = 1 + size[2 * h + 1] + size[2 * h + 2];
    }
    for (int h = 0; h < S; ++h) pidx[h] = -1;
    pidx[0] = 0;
    const size_t o = static_cast<size_t>(t) * S;
    for (int h = 0; h < S; ++h) {  // parents precede children in heap order
      const int i = pidx[h];
      if (i < 0) continue;
      const TreeRec& r = rec[h];
      const bool sp = r.kind == kNodeSplit;
      feat[o + i] = sp ? r.feature : -1;
      thr[o + i] = sp ? r.threshold : 0.0;
      val[o + i] = sp ? 0.0 : r.value;
      gain[o + i] = sp ? r.gain : 0.0;
      lft[o + i] = -1;
      rgt[o + i] = -1;
      if (sp) {
        pidx[2 * h + 1] = i + 1;
        pidx[2 * h + 2] = i + 1 + size[2 * h + 1];
        lft[o + i] = i + 1;
        rgt[o + i] = i + 1 + size[2 * h + 1];
      }
    }
    cnt[t] = size[0];
    // compiled heap
    for (int h = 0; h < nint; ++h) {
      const TreeRec& r = rec[h];
      nodes[static_cast<size_t>(t) * nint + h] =
          r.kind == kNodeSplit ? static_cast<uint32_t>(r.rep) | (static_cast<uint32_t>(r.bin) << 16) : always_left << 16;
    }
    for (int q = 0; q < nleaf; ++q) {
      int h = nint + q;  // deepest existing ancestor-or-self is the leaf covering this heap leaf
      while (h > 0 && rec[h].kind == 0) h = (h - 1) >> 1;
      leafv[static_cast<size_t>(t) * nleaf + q] = rec[h].value;
      leafid[static_cast<size_t>(t) * nleaf + q] = static_cast<uint8_t>(pidx[h]);
    }
  }
}

}  // namespace
}  // namespace fit
}  // namespace fs

// ==========================================================================================
// host orchestration
// ==========================================================================================
namespace fs {
namespace fit {
namespace {

struct Arena {  // stream-ordered scratch owned by one fit call
  cudaStream_t s;
  std::vector<void*> ptrs;
  explicit Arena(cudaStream_t st) : s(st) {}
  template <class T>
  T* alloc(size_t count) {
    void* p = nullptr;
    FS_CUDA(cudaMallocAsync(&p, std::max<size_t>(count, 1) * sizeof(T), s));
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  template <class T>
  T* upload(const std::vector<T>& v) {
    T* p = alloc<T>(v.size());
    if (!v.empty()) FS_CUDA(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
    return p;
  }
  ~Arena() {
    for (void* p : ptrs) cudaFreeAsync(p, s);
  }
};

template <class T>
std::vector<T> download(const T* d, size_t n, cudaStream_t s) {
  std::vector<T> h(n);
  if (n) FS_CUDA(cudaMemcpyAsync(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, s));
  FS_CUDA(cudaStreamSynchronize(s));
  return h;
}

// Several device->host reads with ONE stream synchronization: async copies into the device's
// pinned staging buffer (plus the deferred-error word), one sync, then unpack. Returns the
// error bits (see fs_device::take_errors).
struct BatchRead {
  struct Item {
    const void* src;
    void* dst;
    size_t bytes;
  };
  std::vector<Item> items;
  template <class T>
  void add(const T* d, std::vector<T>& h, size_t n) {
    h.resize(n);
    if (n) items.push_back({d, h.data(), n * sizeof(T)});
  }
  uint32_t run(fs_device* dev) {
    size_t total = 16;
    for (const auto& it : items) total += (it.bytes + 15) & ~size_t(15);
    auto* st = static_cast<unsigned char*>(dev->pinned(total));
    size_t o = 16;
    FS_CUDA(cudaMemcpyAsync(st, dev->err_d, sizeof(uint32_t), cudaMemcpyDeviceToHost, dev->stream));
    for (const auto& it : items) {
      FS_CUDA(cudaMemcpyAsync(st + o, it.src, it.bytes, cudaMemcpyDeviceToHost, dev->stream));
      o += (it.bytes + 15) & ~size_t(15);
    }
    FS_CUDA(cudaStreamSynchronize(dev->stream));
    o = 16;
    for (const auto& it : items) {
      std::memcpy(it.dst, st + o, it.bytes);
      o += (it.bytes + 15) & ~size_t(15);
    }
    uint32_t bits;
    std::memcpy(&bits, st, sizeof bits);
    if (bits) FS_CUDA(cudaMemsetAsync(dev->err_d, 0, sizeof(uint32_t), dev->stream));
    return bits;
  }
};

inline unsigned grid1(int64_t n, int block, int cap) {
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, block), cap)));
}

struct ResidentPlan {
  bool enabled = false;
  std::vector<int> families;
  size_t smem = 0;
  bool pred_smem = false;
  bool pre_smem = false;
  int spec_bufs = 0;  // warps with a speculative exact-fold member buffer
  // column-layout histogram plan for the multi-kernel path (hist_build_col_kernel)
  bool atomic = false;  // limb-atomic histogram (default)
  int colh_max = 1;     // its lane-column height (col_height), max over families
  size_t phi_smem = 0;  // tie-class phi table bytes (largest per-feature bin count x 2); 0 = ordered scan
  std::vector<int> bitonic_ok;  // per family: canonical order by one bitonic sort (else LSD passes)
  size_t bitonic_smem = 0;
  size_t atomic_smem = 0;
  bool col = false;
  std::vector<int32_t> col_off;  // [F][kColWarps + 1] entry offsets per feature group
  std::vector<int32_t> col_rg;   // [F] row groups (private copies)
  size_t col_smem = 0;
};

template <typename CodeT>
void run_rounds(const ResidentPlan& resident, fs_device* dev, Arena& ar, int F, int d, int Dp, int64_t n_tot,
                int max_trees, int depth_max,
                int slots, int nrep_max, int max_bins, int n_max, int level_slots_max, const FamDesc* fam_d,
                FamState* st_d, const double* x_d, const double* target_d, const uint16_t* codes_all,
                const int32_t* rep_orig_d, const int32_t* rep_nb_d, const int32_t* rep_boff_d, const double* vals_d,
                int64_t total_ord, int64_t total_bins, int64_t total_hist, int64_t total_lbuf, int64_t total_tree,
                TreeRec* trees_d, double* mse_d, double* base_d, int min_nrep_hint) {
  cudaStream_t s = dev->stream;
  const int sm = dev->sm_count;
  const size_t bitonic_smem = resident.bitonic_smem;
  const int* bitonic_ok = bitonic_smem > 0 ? ar.upload(resident.bitonic_ok) : nullptr;
  if (bitonic_smem > 0)
    FS_CUDA(cudaFuncSetAttribute(canonical_bitonic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(bitonic_smem)));
  // rows per histogram CTA: kAtomChunk, shrunk (multiples of kAtomTile) until the root level
  // alone launches >= 2 CTAs per SM - a few large families otherwise leave most SMs idle
  int atom_chunk = kAtomChunk;
  while (atom_chunk > 2 * kAtomTile && static_cast<int64_t>(ceil_div(n_max, atom_chunk)) * F < 2LL * sm)
    atom_chunk /= 2;
  // ---- prep: canonical order, gather, presorts, bin counts, base -------------------------
  int32_t* canon = ar.alloc<int32_t>(n_tot);
  int32_t* tmp = ar.alloc<int32_t>(std::max<int64_t>(n_tot, total_ord));
  {
    ProfScope prof(dev, "fit_canonical");
    if (bitonic_smem > 0) {
      canonical_bitonic_kernel<<<F, kSortThreads, bitonic_smem, s>>>(target_d, codes_all, d, fam_d, rep_orig_d,
                                                                     rep_nb_d, bitonic_ok, canon);
      dev->count_launch();
    }
    canonical_kernel<<<F, kSortThreads, 0, s>>>(target_d, codes_all, d, fam_d, rep_orig_d, rep_nb_d, canon, tmp,
                                                bitonic_ok);
  }
  CodeT* codes_c = ar.alloc<CodeT>(static_cast<size_t>(n_tot) * Dp);
  double* target_c = ar.alloc<double>(n_tot);
  int32_t* rowfam = ar.alloc<int32_t>(n_tot);
  gather_canonical_kernel<CodeT><<<grid1(n_tot, 256, sm * 16), 256, 0, s>>>(
      target_d, codes_all, d, fam_d, F, n_tot, rep_orig_d, canon, Dp, codes_c, target_c, rowfam);
  int32_t* ord = ar.alloc<int32_t>(total_ord);
  if (nrep_max > 0) {
    ProfScope prof(dev, "fit_presort");
    presort_kernel<CodeT><<<dim3(nrep_max, F), kSortThreads, 0, s>>>(fam_d, Dp, codes_c, rep_nb_d, ord, tmp);
  }
  int32_t* cle = ar.alloc<int32_t>(total_bins);
  FS_CUDA(cudaMemsetAsync(cle, 0, std::max<int64_t>(total_bins, 1) * sizeof(int32_t), s));
  bin_count_kernel<CodeT><<<grid1(n_tot, 256, sm * 16), 256, 0, s>>>(fam_d, F, n_tot, Dp, codes_c, rowfam, rep_boff_d, cle);
  bin_prefix_kernel<<<F, 128, 0, s>>>(fam_d, rep_boff_d, rep_nb_d, cle);
  double* pred = ar.alloc<double>(n_tot);
  int32_t* ord_root = ar.alloc<int32_t>(n_tot);
  base_kernel<<<F, 256, 0, s>>>(fam_d, target_c, base_d, pred, ord, ord_root);
  dev->count_launch(8);
  FS_CUDA(cudaGetLastError());

  // ---- resident path: every family fits one CTA's shared memory -> one launch, all rounds ----
  if (std::is_same<CodeT, uint8_t>::value && resident.enabled) {
    int* list_d = ar.upload(resident.families);
    FS_CUDA(cudaFuncSetAttribute(fit_resident_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(resident.smem)));
    {
      ProfScope prof(dev, "fit_resident");
      fit_resident_kernel<<<static_cast<unsigned>(resident.families.size()), kResThreads, resident.smem, s>>>(
          fam_d, st_d, list_d, Dp, reinterpret_cast<const uint8_t*>(codes_c), target_c, base_d, ord, ord_root,
          rep_orig_d, rep_nb_d, rep_boff_d, vals_d, cle, canon, x_d, d, trees_d, mse_d, max_trees, slots, dev->ctr_d,
          resident.pred_smem ? 1 : 0, pred, resident.pre_smem ? 1 : 0, resident.spec_bufs);
    }
    dev->count_launch();
    FS_CUDA(cudaGetLastError());
    return;
  }

  // ---- round state ---------------------------------------------------------------------
  double* resid = ar.alloc<double>(n_tot);
  int64_t* rfix = ar.alloc<int64_t>(n_tot);
  int32_t* ord_cur = ar.alloc<int32_t>(n_tot);
  int32_t* scratch = ar.alloc<int32_t>(n_tot);
  int16_t* nodeid = ar.alloc<int16_t>(n_tot);
  NodeRec* nodes = ar.alloc<NodeRec>(static_cast<size_t>(F) * slots);
  int64_t* node_abs = ar.alloc<int64_t>(static_cast<size_t>(F) * slots);
  int64_t* hsum = ar.alloc<int64_t>(total_hist);
  int32_t* hcnt = ar.alloc<int32_t>(total_hist);
  double* lbuf = ar.alloc<double>(total_lbuf);
  WinRec* win = ar.alloc<WinRec>(static_cast<size_t>(F) * level_slots_max * std::max(nrep_max, 1));
  ExactItem* items = ar.alloc<ExactItem>(static_cast<size_t>(F) * level_slots_max * (nrep_max + 1));
  int* n_items = ar.alloc<int>(1);
  (void)total_tree;

  // histogram launch shape
  const int per_group_min = std::max(1, std::min(min_nrep_hint, kHistThreads));
  const size_t tile_bytes = ((static_cast<size_t>(kHistTileRows) * Dp * sizeof(CodeT) + 15) & ~size_t(15)) +
                            kHistTileRows * sizeof(int64_t) + 64;
  const size_t smem_cap = 200 * 1024;
  int groups = std::max(1, kHistThreads / std::max(1, std::min(nrep_max, kHistThreads)));
  (void)per_group_min;
  while (groups > 1 && static_cast<size_t>(groups) * max_bins * 12 + tile_bytes > smem_cap) --groups;
  const bool hist_global = static_cast<size_t>(max_bins) * 12 + tile_bytes > smem_cap;
  const size_t hist_smem = hist_global ? tile_bytes + 16 : ((static_cast<size_t>(groups) * max_bins * 12 + 15) & ~size_t(15)) + tile_bytes;
  if (hist_global) {
    FS_CUDA(cudaFuncSetAttribute(hist_build_kernel<CodeT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(hist_smem)));
  } else {
    FS_CUDA(cudaFuncSetAttribute(hist_build_kernel<CodeT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(hist_smem)));
  }
  const unsigned chunks = static_cast<unsigned>(std::max<int64_t>(1, ceil_div(n_max, kHistChunk)));
  int32_t* col_off_d = nullptr;
  int32_t* col_rg_d = nullptr;
  if (resident.phi_smem > 0)
    FS_CUDA(cudaFuncSetAttribute(tieclass_phi_kernel<CodeT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(resident.phi_smem)));
  if (resident.atomic)
    FS_CUDA(cudaFuncSetAttribute(hist_build_atomic_kernel<CodeT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(resident.atomic_smem)));
  if (resident.col) {
    col_off_d = ar.upload(resident.col_off);
    col_rg_d = ar.upload(resident.col_rg);
    FS_CUDA(cudaFuncSetAttribute(hist_build_col_kernel<CodeT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(resident.col_smem)));
  }

  // One boosting round = a fixed launch sequence whose arguments never change (the round index
  // lives on the device in FamState::ntrees), so it is captured once as a CUDA graph and replayed
  // max_trees times; families that stopped early skip their work inside the kernels.
  const int64_t l0 = dev->launches;
  const int mse_blocks = static_cast<int>(std::max<int64_t>(1, ceil_div(n_max, kMseRows)));
  double* mse_part = ar.alloc<double>(static_cast<size_t>(F) * mse_blocks);
  const bool fork_totals = std::getenv("FAMSEER_FORK_TOTALS") != nullptr;
  // small-node exact folds (exact_small_kernel): per-CTA scratch of two n_max index buffers
  int32_t* small_scratch = std::getenv("FAMSEER_EXACT_SCAN")
                               ? nullptr
                               : ar.alloc<int32_t>(static_cast<size_t>(kExactSmallCtas) * 2 * std::max(n_max, 1));
  cudaStream_t aux = fork_totals ? dev->aux_stream() : nullptr;
  auto round_body = [&]() {
    round_init_kernel<<<F, 256, 0, s>>>(fam_d, st_d, nodes, slots, trees_d);
    FS_CUDA(cudaMemsetAsync(node_abs, 0, static_cast<size_t>(F) * slots * sizeof(int64_t), s));
    residual_kernel<<<grid1(n_tot, 256, sm * 16), 256, 0, s>>>(fam_d, F, n_tot, st_d, rowfam, target_c, pred, resid,
                                                                 ord_root, ord_cur, nodeid);
    fixed_kernel<<<grid1(n_tot, 256, sm * 16), 256, 0, s>>>(fam_d, n_tot, st_d, rowfam, resid, rfix);
    dev->count_launch(3);
    for (int level = 0; level <= depth_max; ++level) {
      const unsigned lw = 1u << level;
      level_plan_kernel<<<dim3(grid1(lw, 128, 1 << 20), F), 128, 0, s>>>(fam_d, st_d, nodes, level);
      dev->count_launch();
      if (level == depth_max || nrep_max == 0) continue;
      // Optional fork (FAMSEER_FORK_TOTALS=1): every screened node's total on a side stream while
      // this level's histogram..decide kernels run; joined before the exact folds. Measured
      // slower at C4 (the root chain outlasts the level's other kernels and the join then
      // stalls every level, exact or not), so the totals are folded only for exact nodes.
      if (fork_totals) {
        FS_CUDA(cudaEventRecord(dev->ev_fork, s));
        FS_CUDA(cudaStreamWaitEvent(aux, dev->ev_fork, 0));
        totals_kernel<<<dim3(grid1(lw, 4, 1 << 20), F), 128, 0, aux>>>(fam_d, st_d, nodes, level, ord_cur, resid);
        FS_CUDA(cudaEventRecord(dev->ev_join, aux));
        dev->count_launch();
      }
      hist_zero_kernel<<<dim3(grid1(static_cast<int64_t>(lw) * max_bins, 256, 64), F), 256, 0, s>>>(fam_d, st_d, level,
                                                                                                  hsum, hcnt);
      const unsigned pairs = level == 0 ? 1u : (1u << (level - 1));
      {
        ProfScope prof(dev, "fit_hist_build");
        if (resident.atomic)
          hist_build_atomic_kernel<CodeT><<<dim3(static_cast<unsigned>(ceil_div(n_max, atom_chunk)), pairs, F),
                                             kAtomThreads, resident.atomic_smem, s>>>(
              fam_d, st_d, nodes, level, Dp, codes_c, rfix, ord_cur, rep_boff_d, hsum, hcnt, node_abs, dev->ctr_d,
              resident.colh_max, atom_chunk);
        else if (resident.col)
          hist_build_col_kernel<CodeT><<<dim3(chunks, pairs, F), kColWarps * 32, resident.col_smem, s>>>(
              fam_d, st_d, nodes, level, Dp, codes_c, rfix, ord_cur, rep_boff_d, rep_nb_d, col_off_d, col_rg_d, hsum,
              hcnt, node_abs, dev->ctr_d);
        else if (hist_global)
          hist_build_kernel<CodeT, true><<<dim3(chunks, pairs, F), kHistThreads, hist_smem, s>>>(
              fam_d, st_d, nodes, level, Dp, codes_c, rfix, ord_cur, rep_boff_d, hsum, hcnt, node_abs, 1, dev->ctr_d);
        else
          hist_build_kernel<CodeT, false><<<dim3(chunks, pairs, F), kHistThreads, hist_smem, s>>>(
              fam_d, st_d, nodes, level, Dp, codes_c, rfix, ord_cur, rep_boff_d, hsum, hcnt, node_abs, groups,
              dev->ctr_d);
      }
      hist_derive_kernel<<<dim3(grid1(max_bins, 256, 16), pairs, F), 256, 0, s>>>(fam_d, st_d, nodes, level, hsum,
                                                                                  hcnt, node_abs);
      const dim3 sg(grid1(nrep_max, 4, 1 << 20), lw, F);  // 4 warps (reps) per 128-thread block
      {
        ProfScope prof(dev, "fit_screen");
        screen_kernel<<<sg, 128, 0, s>>>(fam_d, st_d, nodes, level, hsum, hcnt, node_abs, rep_boff_d, rep_nb_d, win,
                                          std::max(nrep_max, 1), level_slots_max, 0);
        screen_kernel<<<sg, 128, 0, s>>>(fam_d, st_d, nodes, level, hsum, hcnt, node_abs, rep_boff_d, rep_nb_d, win,
                                          std::max(nrep_max, 1), level_slots_max, 1);
      }
      FS_CUDA(cudaMemsetAsync(n_items, 0, sizeof(int), s));
      tieclass_prep_kernel<<<dim3(grid1(lw, 4, 1 << 20), F), 128, 0, s>>>(  // warp per node
          fam_d, st_d, nodes, level, win, std::max(nrep_max, 1), level_slots_max, items, n_items);
      if (resident.phi_smem > 0)
        tieclass_phi_kernel<CodeT><<<sm * 4, 256, resident.phi_smem, s>>>(fam_d, nodes, items, n_items, level, Dp, codes_c,
                                                                 ord_cur, rep_nb_d, win, std::max(nrep_max, 1),
                                                                 level_slots_max);
      else
        tieclass_check_kernel<CodeT><<<sm * 2, 256, 0, s>>>(fam_d, nodes, items, n_items, level, Dp, codes_c, ord,
                                                             nodeid, win, std::max(nrep_max, 1), level_slots_max);
      dev->count_launch(2);
      FS_CUDA(cudaMemsetAsync(n_items, 0, sizeof(int), s));
      decide_kernel<<<dim3(grid1(lw, 4, 1 << 20), F), 128, 0, s>>>(fam_d, st_d, nodes, level, hcnt, rep_boff_d, win,
                                                                     std::max(nrep_max, 1), level_slots_max, items,
                                                                     n_items, dev->ctr_d);
      if (fork_totals) FS_CUDA(cudaStreamWaitEvent(s, dev->ev_join, 0));  // join: totals ready
      {
        ProfScope prof(dev, "fit_exact");
        exact_kernel<CodeT><<<sm * 2, 256, 0, s>>>(fam_d, nodes, items, n_items, level, Dp, codes_c, resid, ord,
                                                   ord_cur, nodeid, rep_boff_d, lbuf, win, std::max(nrep_max, 1),
                                                   level_slots_max, small_scratch ? 1 : 0);
        if (small_scratch)
          exact_small_kernel<CodeT><<<kExactSmallCtas, kSortThreads, 0, s>>>(
              fam_d, nodes, items, n_items, level, Dp, codes_c, resid, nodeid, rep_boff_d, lbuf, win,
              std::max(nrep_max, 1), level_slots_max, small_scratch, n_max);
      }
      exact_decide_kernel<<<dim3(grid1(lw, 128, 1 << 20), F), 128, 0, s>>>(fam_d, st_d, nodes, level, hcnt,
                                                                           rep_boff_d, rep_nb_d, win,
                                                                           std::max(nrep_max, 1), level_slots_max, lbuf);
      {
        ProfScope prof(dev, "fit_partition");
        partition_kernel<CodeT><<<dim3(lw, F), 1024, 0, s>>>(fam_d, st_d, nodes, level, Dp, codes_c, ord_cur,
                                                              scratch, nodeid, rep_orig_d, rep_boff_d, vals_d, cle, ord,
                                                              canon, x_d, d, trees_d, slots);
      }
      dev->count_launch(10);
    }
    const int64_t leaf_threads = static_cast<int64_t>(F) * slots * 32;
    {
      ProfScope prof(dev, "fit_leaf");
      if (std::getenv("FAMSEER_LEAF_WARP"))
        leaf_kernel<<<static_cast<unsigned>(ceil_div(leaf_threads, 256)), 256, 0, s>>>(fam_d, F, st_d, nodes, slots,
                                                                                         ord_cur, resid, pred, trees_d);
      else
        leaf_cta_kernel<<<dim3(static_cast<unsigned>(slots), F), 256, 0, s>>>(fam_d, F, st_d, nodes, slots, ord_cur,
                                                                               resid, pred, trees_d);
    }
    mse_partial_kernel<<<dim3(static_cast<unsigned>(mse_blocks), F), 256, 0, s>>>(fam_d, st_d, nodes, target_c, pred,
                                                                              mse_part, mse_blocks);
    mse_final_kernel<<<F, 1, 0, s>>>(fam_d, st_d, nodes, mse_part, mse_blocks, mse_d, max_trees);
    dev->count_launch();
    dev->count_launch(2);
    FS_CUDA(cudaGetLastError());
  };
  if (max_trees <= 0) return;
  if (std::getenv("FAMSEER_NO_GRAPH") != nullptr) {
    for (int round = 0; round < max_trees; ++round) round_body();
    return;
  }
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  dev->capturing = true;
  FS_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  try {
    round_body();
  } catch (...) {
    cudaStreamEndCapture(s, &graph);
    dev->capturing = false;
    if (graph) cudaGraphDestroy(graph);
    throw;
  }
  FS_CUDA(cudaStreamEndCapture(s, &graph));
  dev->capturing = false;
  const int64_t per_round = dev->launches - l0;
  FS_CUDA(cudaGraphInstantiate(&exec, graph, 0));
  for (int round = 0; round < max_trees; ++round) FS_CUDA(cudaGraphLaunch(exec, s));
  dev->launches = l0 + per_round * max_trees;
  FS_CUDA(cudaGraphExecDestroy(exec));
  FS_CUDA(cudaGraphDestroy(graph));
}

}  // namespace

// Fit every family segment; results replace fo->fams[f] (pre-order trees + compiled form).
void fit_families(fs_device* dev, fs_forest* fo, int F, const int64_t* seg, int d, const double* x_d,
                  const double* target_d, const fs_gbt_params* params) {
  cudaStream_t s = dev->stream;
  if (F < 1) return;
  if (F > static_cast<int>(fo->fams.size())) fail(FS_ERANGE, "fit: more segments than forest families");
  if (seg[0] != 0) fail(FS_EINVAL, "fit: seg[0] must be 0");
  int depth_max = 0, max_trees = 0, n_max = 0;
  for (int f = 0; f < F; ++f) {
    const int64_t n = seg[f + 1] - seg[f];
    if (n < 0) fail(FS_EINVAL, "fit: segment offsets must be non-decreasing");
    if (n > (1 << 30)) fail(FS_EINVAL, "fit: family larger than 2^30 rows");
    if (params[f].trees < 0) fail(FS_EINVAL, "fit: trees must be >= 0");
    if (params[f].depth < 0 || params[f].depth > kMaxDepth)
      fail(FS_EINVAL, "fit: depth must be in [0, " + std::to_string(kMaxDepth) + "]");
    if (n > 0) {
      depth_max = std::max(depth_max, params[f].depth);
      max_trees = std::max(max_trees, params[f].trees);
      n_max = std::max<int>(n_max, static_cast<int>(n));
    }
  }
  const int64_t n_tot = seg[F];
  // FAMSEER_HOST_TIMING=1: host wall-clock per stage of this call on stderr (diagnostics)
  const bool ht = std::getenv("FAMSEER_HOST_TIMING") != nullptr;
  const auto ht0 = std::chrono::steady_clock::now();
  auto htick = [&](const char* what) {
    if (ht)
      std::fprintf(stderr, "[fit host] %-22s %8.1f us\n", what,
                   std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - ht0).count());
  };
  Arena ar(s);
  // ---- family descriptors (stage 1 needs row0/n only) -----------------------------------
  std::vector<FamDesc> fam(static_cast<size_t>(F));
  for (int f = 0; f < F; ++f) {
    std::memset(&fam[f], 0, sizeof(FamDesc));
    fam[f].row0 = seg[f];
    fam[f].pos0 = seg[f];
    fam[f].n = static_cast<int32_t>(seg[f + 1] - seg[f]);
    fam[f].trees = fam[f].n > 0 ? params[f].trees : 0;
    fam[f].depth = params[f].depth;
    fam[f].min_split = params[f].min_samples_split;
    fam[f].lr = params[f].learning_rate;
  }
  htick("entry");
  FamDesc* fam_d = ar.upload(fam);
  htick("fam uploaded");

  // ---- stage 1: distinct values / codes ---------------------------------------------------
  uint16_t* codes_all = ar.alloc<uint16_t>(static_cast<size_t>(std::max<int64_t>(n_tot, 1)) * std::max(d, 1));
  double* vals_all = ar.alloc<double>(static_cast<size_t>(F) * std::max(d, 1) * kSmallBins);
  int32_t* nb_all = ar.alloc<int32_t>(static_cast<size_t>(F) * std::max(d, 1));
  uint64_t* hash_all = ar.alloc<uint64_t>(static_cast<size_t>(F) * std::max(d, 1));
  FS_CUDA(cudaMemsetAsync(nb_all, 0, static_cast<size_t>(F) * std::max(d, 1) * sizeof(int32_t), s));
  FS_CUDA(cudaMemsetAsync(hash_all, 0, static_cast<size_t>(F) * std::max(d, 1) * sizeof(uint64_t), s));
  int* negz_d = ar.alloc<int>(F);
  FS_CUDA(cudaMemsetAsync(negz_d, 0, F * sizeof(int), s));
  htick("stage-1 buffers");
  if (d > 0) {
    const size_t smem = 32 * kHashSlots * 8 + 32 * kSmallBins * 8 + 32 * 4 * 2 + 32 * 8;
    ProfScope prof(dev, "fit_distinct");
    if (std::getenv("FAMSEER_DISTINCT_WARP")) {
      FS_CUDA(cudaFuncSetAttribute(distinct_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
      distinct_small_kernel<<<dim3(static_cast<unsigned>(ceil_div(d, 32)), F), 256, smem, s>>>(
          x_d, d, fam_d, codes_all, vals_all, nb_all, hash_all, dev->err_d, negz_d);
    } else {
      distinct_col_kernel<<<dim3(static_cast<unsigned>(d), F), 256, 0, s>>>(x_d, d, fam_d, codes_all, vals_all, nb_all,
                                                                            hash_all, dev->err_d, negz_d);
    }
    dev->count_launch();
  }
  std::vector<int32_t> nb;
  std::vector<int> negz;
  std::vector<uint64_t> hh;
  {
    BatchRead br;
    br.add(nb_all, nb, static_cast<size_t>(F) * d);
    br.add(negz_d, negz, static_cast<size_t>(F));
    br.add(hash_all, hh, static_cast<size_t>(F) * d);
    raise_deferred(br.run(dev));
  }
  for (int f = 0; f < F; ++f) fam[static_cast<size_t>(f)].negz = negz[static_cast<size_t>(f)];
  std::vector<LargeItem> large;
  int64_t vl = 0;
  for (int f = 0; f < F; ++f)
    for (int j = 0; j < d; ++j)
      if (nb[static_cast<size_t>(f) * d + j] < 0) {
        large.push_back({f, j, vl});
        vl += fam[f].n;
      }
  double* vals_large = ar.alloc<double>(std::max<int64_t>(vl, 1));
  std::vector<int64_t> large_src(static_cast<size_t>(F) * d, -1);
  if (!large.empty()) {
    LargeItem* items_d = ar.upload(large);
    int32_t* bufA = ar.alloc<int32_t>(large.size() * n_max);
    int32_t* bufB = ar.alloc<int32_t>(large.size() * n_max);
    distinct_large_kernel<<<static_cast<unsigned>(large.size()), kSortThreads, 0, s>>>(
        x_d, d, fam_d, items_d, bufA, bufB, n_max, codes_all, vals_large, nb_all, hash_all, dev->err_d);
    dev->count_launch();
    BatchRead br;
    br.add(nb_all, nb, static_cast<size_t>(F) * d);
    br.add(hash_all, hh, static_cast<size_t>(F) * d);
    raise_deferred(br.run(dev));
    for (const auto& it : large) large_src[static_cast<size_t>(it.fam) * d + it.feat] = it.vals0;
  }
  htick("distinct read");
  for (int v : nb)
    if (v > kMaxBins) fail(FS_EINVAL, "fit: more than 65535 distinct values in one feature");

  // ---- stage 2: representatives (drop constant and duplicate-column features) -------------
  std::vector<PairItem> pairs;
  for (int f = 0; f < F; ++f) {
    std::map<std::pair<int, uint64_t>, std::vector<int>> seen;
    for (int j = 0; j < d; ++j) {
      const int v = nb[static_cast<size_t>(f) * d + j];
      if (v <= 1) continue;
      auto& lst = seen[{v, hh[static_cast<size_t>(f) * d + j]}];
      for (int k : lst) pairs.push_back({f, k, j, 0});
      lst.push_back(j);
    }
  }
  std::vector<int32_t> mismatch;
  if (!pairs.empty()) {
    PairItem* pd = ar.upload(pairs);
    int32_t* mm = ar.alloc<int32_t>(pairs.size());
    verify_pairs_kernel<<<static_cast<unsigned>(pairs.size()), 256, 0, s>>>(codes_all, d, fam_d, pd, mm);
    dev->count_launch();
    mismatch = download(mm, pairs.size(), s);
  }
  htick("pairs verified");
  std::vector<std::vector<char>> dup(static_cast<size_t>(F), std::vector<char>(static_cast<size_t>(d), 0));
  for (size_t i = 0; i < pairs.size(); ++i)
    if (!mismatch[i]) dup[static_cast<size_t>(pairs[i].fam)][static_cast<size_t>(pairs[i].b)] = 1;
  std::vector<int32_t> rep_orig, rep_nb, rep_boff;
  std::vector<int64_t> rep_src;
  int nrep_max = 0, max_bins = 0, max_nb = 0, min_nrep = INT_MAX;
  int64_t total_ord = 0, total_bins = 0, total_hist = 0, total_lbuf = 0, total_tree = 0;
  const int slots = (1 << (depth_max + 1)) - 1;
  const int level_slots_max = std::max(1, 1 << std::max(0, depth_max - 1));
  for (int f = 0; f < F; ++f) {
    FamDesc& fd = fam[static_cast<size_t>(f)];
    fd.rep0 = static_cast<int32_t>(rep_orig.size());
    int bins = 0;
    fd.f0rep = -1;
    if (fd.n > 0)
      for (int j = 0; j < d; ++j) {
        const int v = nb[static_cast<size_t>(f) * d + j];
        if (v <= 1 || dup[static_cast<size_t>(f)][static_cast<size_t>(j)]) continue;
        if (j == 0) fd.f0rep = static_cast<int32_t>(rep_orig.size()) - fd.rep0;
        rep_orig.push_back(j);
        rep_nb.push_back(v);
        rep_boff.push_back(bins);
        rep_src.push_back(large_src[static_cast<size_t>(f) * d + j]);
        bins += v;
        max_nb = std::max(max_nb, v);
      }
    fd.nrep = static_cast<int32_t>(rep_orig.size()) - fd.rep0;
    fd.bins = bins;
    fd.level_slots = std::max(1, 1 << std::max(0, fd.depth - 1));
    fd.ord0 = total_ord;
    fd.bin0 = total_bins;
    fd.hist0 = total_hist;
    fd.lbuf0 = total_lbuf;
    fd.node0 = static_cast<int64_t>(f) * slots;
    fd.tree0 = total_tree;
    total_ord += static_cast<int64_t>(fd.nrep) * fd.n;
    total_bins += bins;
    total_hist += 2LL * fd.level_slots * bins;
    total_lbuf += static_cast<int64_t>(fd.level_slots) * bins;
    total_tree += static_cast<int64_t>(fd.trees) * slots;
    nrep_max = std::max(nrep_max, static_cast<int>(fd.nrep));
    if (fd.n > 0) min_nrep = std::min(min_nrep, static_cast<int>(fd.nrep));
    max_bins = std::max(max_bins, bins);
  }
  if (min_nrep == INT_MAX) min_nrep = 1;
  const int code_bytes = max_nb <= 256 ? 1 : 2;
  const size_t phi_bytes = (static_cast<size_t>(std::max(max_nb, 1)) * 2 + 15) & ~size_t(15);
  // Path choice: FAMSEER_FIT_PATH = auto (default) | resident | multi.
  ResidentPlan res;
  {
    const char* envp = std::getenv("FAMSEER_FIT_PATH");
    const std::string mode = envp ? envp : "auto";
    if (mode != "auto" && mode != "resident" && mode != "multi")
      fail(FS_EINVAL, "FAMSEER_FIT_PATH must be auto, resident or multi");
    if (mode != "multi" && code_bytes == 1 && depth_max <= kResMaxDepth) {
      // Shared-memory staging options, most valuable first: the running predictions (read and
      // updated every round) and the presorted lists (reference-order folds); whatever does not
      // fit stays in global memory (L2-resident).
      const int opts[8][3] = {{1, 1, kSpecBufs}, {1, 1, 0}, {1, 0, kSpecBufs}, {1, 0, 0},
                              {0, 1, kSpecBufs}, {0, 1, 0},  {0, 0, kSpecBufs}, {0, 0, 0}};
      for (const auto& op : opts) {
        const bool pred_smem = op[0] != 0, pre_smem = op[1] != 0;
        const int spec = std::getenv("FAMSEER_NO_SPEC") ? 0 : op[2];
        bool ok = true;
        const size_t budget = 225 * 1024;
        std::vector<int> fams_ok;
        size_t need = 0;
        for (int f = 0; f < F; ++f) {
          const FamDesc& fd = fam[static_cast<size_t>(f)];
          if (fd.n <= 0 || fd.trees <= 0) continue;
          if (fd.n > 65535 || fd.nrep > kResThreads) ok = false;
          const int colh = fd.nrep > 0 ? col_height(fd.nrep, rep_nb.data() + fd.rep0, nullptr) : 1;
          need = std::max(need, res_layout(fd.n, fd.nrep, fd.bins, fd.depth, colh, pred_smem, pre_smem, spec).total);
          fams_ok.push_back(f);
        }
        res.families = fams_ok;
        if (ok && need <= budget && !fams_ok.empty()) {
          res.enabled = true;
          res.smem = need;
          res.pred_smem = pred_smem;
          res.pre_smem = pre_smem;
          res.spec_bufs = spec;
          break;
        }
      }
    }
    if (mode == "resident" && !res.enabled && !res.families.empty())
      fail(FS_EINVAL, "fit: resident path requested but the families do not fit one CTA");
  }
  if (phi_bytes <= 96 * 1024 && !std::getenv("FAMSEER_TIE_SCAN")) res.phi_smem = phi_bytes;
  // canonical order by bitonic sort: families without -0.0 whose packed keys fit shared memory
  if (!std::getenv("FAMSEER_CANON_LSD")) {
    res.bitonic_ok.assign(static_cast<size_t>(F), 0);
    for (int f = 0; f < F; ++f) {
      const FamDesc& fd = fam[static_cast<size_t>(f)];
      if (fd.n <= 1 || fd.negz) continue;
      int wide = 0;
      for (int j = 0; j < fd.nrep; ++j) wide |= rep_nb[static_cast<size_t>(fd.rep0 + j)] > 256;
      const int W = (fd.nrep * (wide ? 2 : 1) + 3) / 4 + 2;
      int P = 1;
      while (P < fd.n) P <<= 1;
      const size_t need = static_cast<size_t>(P) * (W + 1) * 4;
      if (need > 160 * 1024) continue;
      res.bitonic_ok[static_cast<size_t>(f)] = 1;
      res.bitonic_smem = std::max(res.bitonic_smem, need);
    }
  }
  // Column-layout histogram plan (multi-kernel path): per feature group of 32 the largest bin
  // count; row-group copies while they fit the shared-memory budget.
  // Histogram shape for the multi-kernel path: FAMSEER_HIST = atomic (default) | col | rowmajor.
  const char* hist_env = std::getenv("FAMSEER_HIST");
  const std::string hist_mode = hist_env ? hist_env : (std::getenv("FAMSEER_HIST_ROWMAJOR") ? "rowmajor" : "atomic");
  if (hist_mode != "atomic" && hist_mode != "col" && hist_mode != "rowmajor")
    fail(FS_EINVAL, "FAMSEER_HIST must be atomic, col or rowmajor");
  if (!res.enabled && hist_mode == "atomic") {
    const int pv = 16 / code_bytes;
    const int dp = std::max(pv, static_cast<int>(ceil_div(std::max(nrep_max, 1), pv)) * pv);
    int colh_max = 1;
    for (int f = 0; f < F; ++f) {
      const FamDesc& fd = fam[static_cast<size_t>(f)];
      if (fd.nrep > 0) colh_max = std::max(colh_max, col_height(fd.nrep, rep_nb.data() + fd.rep0, nullptr));
    }
    const size_t need = hist_atomic_smem(max_bins, nrep_max, dp, code_bytes, colh_max);
    if (need <= 200 * 1024) {
      res.atomic = true;
      res.atomic_smem = need;
      res.colh_max = colh_max;
    }
  }
  if (!res.enabled && !res.atomic && hist_mode != "rowmajor") {
    const size_t cap = 200 * 1024;
    const int pv = 16 / code_bytes;
    const int dp = std::max(pv, static_cast<int>(ceil_div(std::max(nrep_max, 1), pv)) * pv);
    const size_t tile = ((static_cast<size_t>(kHistTileRows) * dp * code_bytes + 15) & ~size_t(15)) +
                        kHistTileRows * sizeof(int64_t) + 64;
    bool ok = true;
    res.col_off.assign(static_cast<size_t>(F) * (kColWarps + 1), 0);
    res.col_rg.assign(static_cast<size_t>(F), 1);
    size_t need = 0;
    for (int f = 0; f < F && ok; ++f) {
      const FamDesc& fd = fam[static_cast<size_t>(f)];
      const int nfg = (fd.nrep + 31) / 32;
      if (nfg > kColWarps) {
        ok = false;
        break;
      }
      int32_t off = 0;
      for (int g = 0; g < nfg; ++g) {
        int mx = 0;
        for (int j = 32 * g; j < std::min(fd.nrep, 32 * g + 32); ++j)
          mx = std::max(mx, rep_nb[static_cast<size_t>(fd.rep0 + j)]);
        res.col_off[static_cast<size_t>(f) * (kColWarps + 1) + g] = off;
        off += mx * 32;
      }
      for (int g = nfg; g <= kColWarps; ++g) res.col_off[static_cast<size_t>(f) * (kColWarps + 1) + g] = off;
      const size_t per_copy = static_cast<size_t>(off) * 12;
      int rg = std::max(1, kColWarps / std::max(1, nfg));
      while (rg > 1 && rg * per_copy + tile > cap) --rg;
      if (per_copy + tile > cap) ok = false;
      res.col_rg[static_cast<size_t>(f)] = rg;
      need = std::max(need, rg * per_copy + tile);
    }
    if (ok) {
      res.col = true;
      res.col_smem = need;
    }
  }
  const int per_vec = 16 / code_bytes;
  const int Dp = std::max(per_vec, static_cast<int>(ceil_div(std::max(nrep_max, 1), per_vec)) * per_vec);
  FS_CUDA(cudaMemcpyAsync(fam_d, fam.data(), fam.size() * sizeof(FamDesc), cudaMemcpyHostToDevice, s));
  int32_t* rep_orig_d = ar.upload(rep_orig);
  int32_t* rep_nb_d = ar.upload(rep_nb);
  int32_t* rep_boff_d = ar.upload(rep_boff);
  int64_t* rep_src_d = ar.upload(rep_src);
  double* vals_d = ar.alloc<double>(std::max<int64_t>(total_bins, 1));
  if (nrep_max > 0) {
    rep_vals_kernel<<<dim3(static_cast<unsigned>(std::min(nrep_max, 1024)), F), 128, 0, s>>>(
        fam_d, rep_orig_d, rep_boff_d, rep_nb_d, rep_src_d, vals_all, vals_large, d, vals_d);
    dev->count_launch();
  }
  std::vector<FamState> st0(static_cast<size_t>(F));
  for (int f = 0; f < F; ++f) {
    std::memset(&st0[f], 0, sizeof(FamState));
    st0[f].active = fam[f].n > 0 && fam[f].trees > 0;
  }
  FamState* st_d = ar.upload(st0);
  TreeRec* trees_d = ar.alloc<TreeRec>(std::max<int64_t>(total_tree, 1));
  double* mse_d = ar.alloc<double>(static_cast<size_t>(F) * std::max(max_trees, 1));
  double* base_d = ar.alloc<double>(F);
  FS_CUDA(cudaMemsetAsync(base_d, 0, F * sizeof(double), s));

  htick("plan uploaded");
  {
  ProfScope prof_rounds(dev, "fit_rounds");
  if (code_bytes == 1)
    run_rounds<uint8_t>(res, dev, ar, F, d, Dp, n_tot, max_trees, depth_max, slots, nrep_max, max_bins, n_max,
                        level_slots_max, fam_d, st_d, x_d, target_d, codes_all, rep_orig_d, rep_nb_d, rep_boff_d,
                        vals_d, total_ord, total_bins, total_hist, total_lbuf, total_tree, trees_d, mse_d, base_d,
                        min_nrep);
  else
    run_rounds<uint16_t>(res, dev, ar, F, d, Dp, n_tot, max_trees, depth_max, slots, nrep_max, max_bins, n_max,
                         level_slots_max, fam_d, st_d, x_d, target_d, codes_all, rep_orig_d, rep_nb_d, rep_boff_d,
                         vals_d, total_ord, total_bins, total_hist, total_lbuf, total_tree, trees_d, mse_d, base_d,
                         min_nrep);
  }

  // ---- results: heap-slot records -> pre-order CostModelState layout ------------------------
  htick("rounds launched");
  // Epilogue. Default: export + compile on the device straight into each family's model blob
  // (no host round trip; the host pre-order arrays are materialised when first asked for).
  // FAMSEER_HOST_COMPILE=1 (or trees deeper than the device compile handles): read the tree
  // tables back and compile on the host.
  const bool dev_compile = depth_max <= kResMaxDepth && slots <= kCompileSlots && !std::getenv("FAMSEER_HOST_COMPILE");
  if (dev_compile) {
    std::vector<ExportJob> jobs(static_cast<size_t>(F));
    for (int f = 0; f < F; ++f) {
      FamilyModel& m = fo->fams[static_cast<size_t>(f)];
      const FamDesc& fd = fam[static_cast<size_t>(f)];
      const int T = std::max(fd.n > 0 ? fd.trees : 0, 0), D = std::max(fd.depth, 0);
      const int S = (1 << (D + 1)) - 1, nint = (1 << D) - 1, nleaf = 1 << D;
      const int nrep = std::max(static_cast<int>(fd.nrep), 0), bins = std::max(static_cast<int>(fd.bins), 0);
      int max_nb = 0, d_orig = 0;
      for (int j = 0; j < nrep; ++j) {
        max_nb = std::max(max_nb, static_cast<int>(rep_nb[static_cast<size_t>(fd.rep0 + j)]));
        d_orig = std::max(d_orig, static_cast<int>(rep_orig[static_cast<size_t>(fd.rep0 + j)]) + 1);
      }
      DevLayout L;
      size_t o = 0;
      auto put = [&](size_t bytes) {
        const size_t at = o;
        o = (o + bytes + 15) & ~size_t(15);
        return at;
      };
      L.meta = put(sizeof(ModelMeta));
      L.nodes = put(static_cast<size_t>(T) * nint * 4);
      L.leafv = put(static_cast<size_t>(T) * nleaf * 8);
      L.leafid = put(static_cast<size_t>(T) * nleaf);
      L.uthr = put(static_cast<size_t>(bins) * 8);
      L.uoff = put(static_cast<size_t>(nrep + 1) * 4);
      L.fmap = put(static_cast<size_t>(nrep) * 4);
      L.cnt = put(static_cast<size_t>(T) * 4);
      L.feat = put(static_cast<size_t>(T) * S * 4);
      L.thr = put(static_cast<size_t>(T) * S * 8);
      L.left = put(static_cast<size_t>(T) * S * 4);
      L.right = put(static_cast<size_t>(T) * S * 4);
      L.val = put(static_cast<size_t>(T) * S * 8);
      L.gain = put(static_cast<size_t>(T) * S * 8);
      L.mse = put(static_cast<size_t>(T) * 8);
      L.total = o;
      L.max_trees = T;
      L.slots = S;
      if (L.total > m.blob_cap) {
        if (m.blob_d) FS_CUDA(cudaFree(m.blob_d));
        m.blob_d = nullptr;
        const size_t cap = std::max<size_t>(L.total + L.total / 2, 4096);
        FS_CUDA(cudaMalloc(&m.blob_d, cap));
        m.blob_cap = cap;
      }
      const bool wide = max_nb > 255;
      jobs[static_cast<size_t>(f)] = {m.blob_d, L, D, wide ? 1 : 0};
      m.lr = fd.lr;
      m.compiled = true;
      m.generic = false;
      m.pending = true;
      m.lay = L;
      m.depth = D;
      m.d_model = nrep;
      m.d_orig = d_orig;
      m.code_bytes = wide ? 2 : 1;
      m.n_uthr = bins;
      m.n_trees = T;  // upper bound until materialised (the device meta holds the count)
      m.nodes_d = reinterpret_cast<uint32_t*>(m.blob_d + L.nodes);
      m.leafv_d = reinterpret_cast<double*>(m.blob_d + L.leafv);
      m.leafid_d = m.blob_d + L.leafid;
      m.uthr_d = reinterpret_cast<double*>(m.blob_d + L.uthr);
      m.uoff_d = reinterpret_cast<int32_t*>(m.blob_d + L.uoff);
      m.fmap_d = reinterpret_cast<const int32_t*>(m.blob_d + L.fmap);
      m.meta_d = reinterpret_cast<const ModelMeta*>(m.blob_d + L.meta);
      m.g_off_d = m.g_feat_d = m.g_left_d = m.g_right_d = nullptr;
      m.g_thr_d = m.g_val_d = nullptr;
    }
    ExportJob* jobs_d = ar.upload(jobs);
    export_compile_kernel<<<F, 128, 0, s>>>(fam_d, st_d, trees_d, slots, mse_d, std::max(max_trees, 1), base_d,
                                            rep_orig_d, rep_boff_d, vals_d, jobs_d);
    dev->count_launch();
    FS_CUDA(cudaGetLastError());
    htick("device export launched");
    return;
  }
  std::vector<FamState> st_h;
  std::vector<TreeRec> trees_h;
  std::vector<double> mse_h, base_h;
  {
    BatchRead br;
    br.add(st_d, st_h, static_cast<size_t>(F));
    br.add(trees_d, trees_h, static_cast<size_t>(std::max<int64_t>(total_tree, 1)));
    br.add(mse_d, mse_h, static_cast<size_t>(F) * std::max(max_trees, 1));
    br.add(base_d, base_h, static_cast<size_t>(F));
    raise_deferred(br.run(dev));
  }
  htick("results read");
  UploadBatch batch;
  for (int f = 0; f < F; ++f) {
    FamilyModel& m = fo->fams[static_cast<size_t>(f)];
    const FamDesc& fd = fam[static_cast<size_t>(f)];
    m.lr = fd.lr;
    m.base = fd.n > 0 ? base_h[static_cast<size_t>(f)] : 0.0;
    m.offsets.assign(1, 0);
    m.feature.clear();
    m.threshold.clear();
    m.left.clear();
    m.right.clear();
    m.value.clear();
    m.gain.clear();
    m.mse.clear();
    const int T = st_h[static_cast<size_t>(f)].ntrees;
    m.offsets.reserve(static_cast<size_t>(T) + 1);
    for (auto* v : {&m.feature, &m.left, &m.right}) v->reserve(static_cast<size_t>(T) * slots);
    for (auto* v : {&m.threshold, &m.value, &m.gain}) v->reserve(static_cast<size_t>(T) * slots);
    struct Emit {
      int slot, parent, side;  // parent: global index of the parent node (-1 root), side 0 left / 1 right
    };
    std::vector<Emit> es;
    for (int t = 0; t < T; ++t) {
      const TreeRec* rec = trees_h.data() + fd.tree0 + static_cast<int64_t>(t) * slots;
      const int base_idx = static_cast<int>(m.feature.size());
      es.assign(1, {0, -1, 0});
      while (!es.empty()) {  // pre-order: left subtree before right (costmodel.cpp:108-111)
        const Emit e = es.back();
        es.pop_back();
        const int gidx = static_cast<int>(m.feature.size());
        const TreeRec& r = rec[e.slot];
        if (r.kind != kNodeSplit && r.kind != kNodeLeaf) fail(FS_ECUDA, "fit: internal error (missing tree node)");
        m.feature.push_back(r.kind == kNodeSplit ? r.feature : -1);
        m.threshold.push_back(r.kind == kNodeSplit ? r.threshold : 0.0);
        m.left.push_back(-1);
        m.right.push_back(-1);
        m.value.push_back(r.kind == kNodeSplit ? 0.0 : r.value);
        m.gain.push_back(r.kind == kNodeSplit ? r.gain : 0.0);
        if (e.parent >= 0) (e.side ? m.right : m.left)[static_cast<size_t>(e.parent)] = gidx - base_idx;
        if (r.kind == kNodeSplit) {
          es.push_back({2 * e.slot + 2, gidx, 1});
          es.push_back({2 * e.slot + 1, gidx, 0});
        }
      }
      m.offsets.push_back(static_cast<int32_t>(m.feature.size()));
      m.mse.push_back(mse_h[static_cast<size_t>(f) * max_trees + t]);
    }
    m.screened = static_cast<int64_t>(st_h[static_cast<size_t>(f)].screened);
    m.exact = static_cast<int64_t>(st_h[static_cast<size_t>(f)].exact);
    compile_model(dev, m, &batch);
  }
  batch.flush(dev);
  htick("models compiled");
}

}  // namespace fit
}  // namespace fs

extern "C" {

int fs_fit_d(fs_device* dev, fs_forest* fo, int32_t nseg, const int64_t* seg, int32_t d, const double* x_d,
             const double* target_d, const fs_gbt_params* params) {
  return fs::guard([&] {
    if (!dev || !fo || nseg < 0 || !seg || d < 0 || !params) fs::fail(FS_EINVAL, "fs_fit: bad arguments");
    dev->activate();
    fs::fit::fit_families(dev, fo, nseg, seg, d, x_d, target_d, params);
  });
}

int fs_fit(fs_device* dev, fs_forest* fo, int32_t nseg, const int64_t* seg, int32_t d, const double* x,
           const double* target, const fs_gbt_params* params) {
  return fs::guard([&] {
    if (!dev || !fo || nseg < 0 || !seg || d < 0 || !params) fs::fail(FS_EINVAL, "fs_fit: bad arguments");
    dev->activate();
    const int64_t n = seg[nseg];
    auto* xd = static_cast<double*>(dev->scratch(fs::kSlotH2D0, std::max<int64_t>(n * d, 1) * sizeof(double)));
    auto* yd = static_cast<double*>(dev->scratch(fs::kSlotH2D1, std::max<int64_t>(n, 1) * sizeof(double)));
    if (n * d > 0) FS_CUDA(cudaMemcpyAsync(xd, x, n * d * sizeof(double), cudaMemcpyHostToDevice, dev->stream));
    if (n) FS_CUDA(cudaMemcpyAsync(yd, target, n * sizeof(double), cudaMemcpyHostToDevice, dev->stream));
    fs::fit::fit_families(dev, fo, nseg, seg, d, xd, yd, params);
  });
}

int fs_fit_records_d(fs_device* dev, fs_forest* fo, const fs_spaces* sp, int32_t nseg, const int64_t* seg,
                     const int32_t* space_of_d, const int32_t* assign_d, int32_t pad, const double* target_d,
                     const fs_gbt_params* params) {
  return fs::guard([&] {
    if (!dev || !fo || !sp || nseg < 0 || !seg || pad < 0 || !params)
      fs::fail(FS_EINVAL, "fs_fit_records: bad arguments");
    dev->activate();
    const int64_t n = seg[nseg];
    auto* xd = static_cast<double*>(dev->scratch(fs::kSlotFitX, std::max<int64_t>(n * pad, 1) * sizeof(double)));
    fs::launch_featurize(dev, sp, n, space_of_d, assign_d, pad, xd);
    fs::fit::fit_families(dev, fo, nseg, seg, pad, xd, target_d, params);
  });
}

int fs_fit_records(fs_device* dev, fs_forest* fo, const fs_spaces* sp, int32_t nseg, const int64_t* seg,
                   const int32_t* space_of, const int32_t* assign, int32_t pad, const double* target,
                   const fs_gbt_params* params) {
  return fs::guard([&] {
    if (!dev || !fo || !sp || nseg < 0 || !seg || pad < 0 || !params)
      fs::fail(FS_EINVAL, "fs_fit_records: bad arguments");
    dev->activate();
    const int64_t n = seg[nseg];
    // the reference validates every record's dimension on the host (searchspace.cpp:94-101)
    for (int64_t i = 0; i < n; ++i) {
      const int s = space_of[i];
      if (s < 0 || s >= sp->n) fs::fail(FS_EINVAL, "fit_records: unknown space id");
      if (pad < fs_feature_dim(sp->k_h[static_cast<size_t>(s)])) fs::fail(FS_EINVAL, "fit_records: pad_dim too small");
    }
    const size_t b_so = static_cast<size_t>(std::max<int64_t>(n, 1)) * sizeof(int32_t);
    const size_t b_a = static_cast<size_t>(std::max<int64_t>(n, 1)) * FS_MAX_KNOBS * sizeof(int32_t);
    const size_t b_t = static_cast<size_t>(std::max<int64_t>(n, 1)) * sizeof(double);
    auto* in = static_cast<unsigned char*>(dev->scratch(fs::kSlotFitIn, b_t + b_so + b_a + 32));
    auto* td = reinterpret_cast<double*>(in);
    auto* sd = reinterpret_cast<int32_t*>(in + b_t);
    auto* ad = reinterpret_cast<int32_t*>(in + b_t + b_so);
    if (n) {
      FS_CUDA(cudaMemcpyAsync(td, target, n * sizeof(double), cudaMemcpyHostToDevice, dev->stream));
      FS_CUDA(cudaMemcpyAsync(sd, space_of, n * sizeof(int32_t), cudaMemcpyHostToDevice, dev->stream));
      FS_CUDA(cudaMemcpyAsync(ad, assign, n * FS_MAX_KNOBS * sizeof(int32_t), cudaMemcpyHostToDevice, dev->stream));
    }
    auto* xd = static_cast<double*>(dev->scratch(fs::kSlotFitX, std::max<int64_t>(n * pad, 1) * sizeof(double)));
    fs::launch_featurize(dev, sp, n, sd, ad, pad, xd);
    fs::fit::fit_families(dev, fo, nseg, seg, pad, xd, td, params);
  });
}

int fs_forest_fit_stats(const fs_forest* fo, int32_t family, int64_t* screened, int64_t* exact) {
  return fs::guard([&] {
    if (!fo || family < 0 || family >= static_cast<int32_t>(fo->fams.size()))
      fs::fail(FS_ERANGE, "fs_forest_fit_stats: unknown family id");
    const auto& m = fo->fams[static_cast<size_t>(family)];
    fs::materialize(fo->dev, m);
    if (screened) *screened = m.screened;
    if (exact) *exact = m.exact;
  });
}

}  // extern "C"
