// fit_prep.cuh - per-fit preparation kernels: distinct values / codes, feature dedup, canonical order, presorts, base
// Part of the trainer translation unit: included once, by fit.cu only (shares its
// anonymous namespace, constants and helpers).
#pragma once

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

// prep 3b': canonical order exchanged with the caller's training store (FitRows::io): 1 = the
// store's maintained order is the family's canonical order (its sort was skipped), 2 = record
// the order just computed in the store.
__global__ void canon_io_kernel(const FamDesc* __restrict__ fam, int F, int64_t n_tot, const int* __restrict__ io,
                                int32_t* __restrict__ store_canon, int32_t* __restrict__ canon) {
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < n_tot;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int f = family_of_pos(fam, F, p);
    const int m = io[f];
    if (m == 0) continue;
    const int64_t r = fam[f].row0 + (p - fam[f].pos0);
    if (m == 1) canon[p] = store_canon[r];
    else store_canon[r] = canon[p];
  }
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

constexpr int kBitonicE = 4;  // canonical_bitonic_kernel: sequence elements per thread in registers (P <= 4 T)

__global__ void __launch_bounds__(kSortThreads) canonical_bitonic_kernel(
    const double* __restrict__ target, const uint16_t* __restrict__ codes_all, int d,
    const FamDesc* __restrict__ fam, const int32_t* __restrict__ rep_orig, const int32_t* __restrict__ rep_nb,
    const int* __restrict__ eligible, int32_t* __restrict__ canon) {
  extern __shared__ __align__(16) uint32_t ks[];  // [P][W] keys, then [P] row ids
  const int f = blockIdx.x;
  if (eligible[f] != 1) return;  // 0: LSD passes, 2: order given by the caller (fs_store)
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
  // Bitonic sort of ROW IDS (the keys stay in place): element i of the sequence lives in thread
  // i % T, register slot i / T (E = P / T slots, E <= kBitonicE). A compare-exchange keeps the
  // smaller or larger of (key, row) - a total order, so both partners agree. Partners within a
  // warp exchange by shuffle, partners in the same thread by register, others through shared
  // memory (ids[] doubles as the exchange buffer): barriers only for strides in [32, T).
  const int T = blockDim.x, E = P / T;
  if (E >= 1 && E <= kBitonicE && (T & 31) == 0) {
    const int lane = threadIdx.x & 31;
    uint32_t v[kBitonicE];
#pragma unroll
    for (int e = 0; e < kBitonicE; ++e) v[e] = e < E ? static_cast<uint32_t>(threadIdx.x + e * T) : 0u;
    auto less_rows = [&](uint32_t a, uint32_t b) {  // (key, row) order
      const uint32_t* ka = ks + static_cast<size_t>(a) * W;
      const uint32_t* kb = ks + static_cast<size_t>(b) * W;
      for (int w = 0; w < W; ++w)
        if (ka[w] != kb[w]) return ka[w] < kb[w];
      return a < b;
    };
    for (int size = 2; size <= P; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        uint32_t pv[kBitonicE];
        if (stride < 32) {
#pragma unroll
          for (int e = 0; e < kBitonicE; ++e) pv[e] = __shfl_xor_sync(0xffffffffu, v[e], stride);
        } else if (stride >= T) {
          const int es = stride / T;
#pragma unroll
          for (int e = 0; e < kBitonicE; ++e) {
            pv[e] = v[0];
#pragma unroll
            for (int q = 0; q < kBitonicE; ++q)
              if (q == (e ^ es)) pv[e] = v[q];
          }
        } else {
#pragma unroll
          for (int e = 0; e < kBitonicE; ++e)
            if (e < E) ids[threadIdx.x + e * T] = v[e];
          __syncthreads();
#pragma unroll
          for (int e = 0; e < kBitonicE; ++e)
            if (e < E) pv[e] = ids[(threadIdx.x + e * T) ^ stride];
          __syncthreads();
        }
#pragma unroll
        for (int e = 0; e < kBitonicE; ++e) {
          if (e >= E) continue;
          const int i = threadIdx.x + e * T;
          const bool up = (i & size) == 0, lower = (i & stride) == 0;
          const bool pl = less_rows(pv[e], v[e]);  // partner smaller
          // the lower position of an ascending pair keeps the smaller element, etc.
          if (pl == (up == lower)) v[e] = pv[e];
        }
      }
    }
#pragma unroll
    for (int e = 0; e < kBitonicE; ++e)
      if (e < E) ids[threadIdx.x + e * T] = v[e];
    __syncthreads();
    (void)lane;
  } else {
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
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) canon[fd.pos0 + i] = static_cast<int32_t>(ids[i]);
}

__global__ void base_kernel(const FamDesc* __restrict__ fam, const double* __restrict__ target_c,
                            double* __restrict__ base, double* __restrict__ pred, const int32_t* __restrict__ ord,
                            int32_t* __restrict__ ord_root) {
  // sequential mean in canonical order (costmodel.cpp:185-188): the targets are staged into
  // shared memory 2,048 at a time by the whole CTA (coalesced), and thread 0 folds each stage
  // from shared memory (L2 latency only once per stage instead of once per 8 elements)
  constexpr int kStage = 2048;
  __shared__ double st[kStage];
  const FamDesc fd = fam[blockIdx.x];
  const double* t = target_c + fd.pos0;
  double s = 0.0;
  for (int c0 = 0; c0 < fd.n; c0 += kStage) {
    const int m = min(kStage, fd.n - c0);
    for (int i = threadIdx.x; i < m; i += blockDim.x) st[i] = t[c0 + i];
    __syncthreads();
    if (threadIdx.x == 0) {
      int i = 0;
      if (m >= 8) {  // the next 8 loads are in flight while 8 dependent adds run
        double a[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = st[k];
        for (i = 8; i + 8 <= m; i += 8) {
          double b[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) b[k] = st[i + k];
#pragma unroll
          for (int k = 0; k < 8; ++k) s = fs_add(s, a[k]);
#pragma unroll
          for (int k = 0; k < 8; ++k) a[k] = b[k];
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) s = fs_add(s, a[k]);
      }
      for (; i < m; ++i) s = fs_add(s, st[i]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) base[blockIdx.x] = fd.n ? fs_div(s, static_cast<double>(fd.n)) : 0.0;
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
                                  int slots, TreeRec* __restrict__ trees, int64_t* __restrict__ node_abs) {
  FS_PDL_WAIT();
  const int f = blockIdx.x;
  const FamDesc fd = fam[f];
  for (int s = threadIdx.x; s < slots; s += blockDim.x) node_abs[fd.node0 + s] = 0;
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
  FS_PDL_WAIT();
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
  FS_PDL_WAIT();
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

}  // namespace
}  // namespace fit
}  // namespace fs
