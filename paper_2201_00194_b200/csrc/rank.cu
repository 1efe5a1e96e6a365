// Ranking (scheduler.cpp:187-192): the full ascending order of (score, pool index) pairs per
// family segment - what std::sort gives vector<pair<double, size_t>>. The epsilon picks of
// tune_step index into the sorted tail (scheduler.cpp:202-213), so the whole permutation is
// produced, not just a top-k.
//
// Keys: FP64 scores mapped to order-preserving u64 (-0.0 canonicalised to +0.0 so the two
// compare equal, as with operator<); ties broken by the segment-local index, which is unique,
// so every comparison below is a strict total order.
//   1. chunk sort: each CTA bitonic-sorts up to kChunk (key, index) pairs in shared memory;
//   2. merge passes: runs double in length; every output element finds its merge-path split by
//      binary search and writes itself (fully parallel, no atomics), ping-ponging two buffers.
#include <algorithm>
#include <vector>

#include "fs_common.cuh"

namespace {

constexpr int kChunk = 4096;
constexpr int kSortThreads = 1024;

__device__ __forceinline__ uint64_t order_key(double s) {
  uint64_t b = static_cast<uint64_t>(__double_as_longlong(s));
  if (b == 0x8000000000000000ull) b = 0;  // -0.0 == +0.0
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ bool less_kv(uint64_t ka, uint32_t ia, uint64_t kb, uint32_t ib) {
  return ka < kb || (ka == kb && ia < ib);
}

struct ChunkDesc {
  int64_t start;  // global element offset
  int32_t len;
  int32_t pad;
};

__global__ void make_keys_kernel(const double* __restrict__ scores, const int64_t* __restrict__ seg, int nseg,
                                 int64_t n, uint64_t* __restrict__ keys, uint32_t* __restrict__ idx) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int lo = 0, hi = nseg;  // segment containing i: last s with seg[s] <= i
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (seg[mid] <= i) lo = mid;
      else hi = mid;
    }
    keys[i] = order_key(scores[i]);
    idx[i] = static_cast<uint32_t>(i - seg[lo]);
  }
}

__global__ void __launch_bounds__(kSortThreads) chunk_sort_kernel(const ChunkDesc* __restrict__ chunks,
                                                                  uint64_t* __restrict__ keys,
                                                                  uint32_t* __restrict__ idx) {
  __shared__ uint64_t sk[kChunk];
  __shared__ uint32_t si[kChunk];
  const ChunkDesc c = chunks[blockIdx.x];
  int npow = 1;
  while (npow < c.len) npow <<= 1;
  for (int i = threadIdx.x; i < npow; i += blockDim.x) {
    if (i < c.len) {
      sk[i] = keys[c.start + i];
      si[i] = idx[c.start + i];
    } else {
      sk[i] = ~0ull;
      si[i] = 0xFFFFFFFFu;
    }
  }
  __syncthreads();
  for (int k = 2; k <= npow; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < npow; i += blockDim.x) {
        const int p = i ^ j;
        if (p > i) {
          const bool up = (i & k) == 0;
          const uint64_t ka = sk[i], kb = sk[p];
          const uint32_t ia = si[i], ib = si[p];
          const bool swap = up ? less_kv(kb, ib, ka, ia) : less_kv(ka, ia, kb, ib);
          if (swap) {
            sk[i] = kb;
            sk[p] = ka;
            si[i] = ib;
            si[p] = ia;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < c.len; i += blockDim.x) {
    keys[c.start + i] = sk[i];
    idx[c.start + i] = si[i];
  }
}

// One merge pass over every segment: runs of length `run` (segment-local) merge pairwise.
__global__ void merge_pass_kernel(const int64_t* __restrict__ seg, int nseg, int64_t n, int64_t run,
                                  const uint64_t* __restrict__ ki, const uint32_t* __restrict__ ii,
                                  uint64_t* __restrict__ ko, uint32_t* __restrict__ io) {
  for (int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < n;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int lo = 0, hi = nseg;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (seg[mid] <= g) lo = mid;
      else hi = mid;
    }
    const int64_t s0 = seg[lo], ns = seg[lo + 1] - s0, o = g - s0;
    const int64_t b = (o / (2 * run)) * (2 * run);
    const int64_t a0 = b, a1 = min(b + run, ns), b0 = a1, b1 = min(b + 2 * run, ns);
    const int64_t la = a1 - a0, lb = b1 - b0, k = o - b;
    const uint64_t* KA = ki + s0 + a0;
    const uint32_t* IA = ii + s0 + a0;
    const uint64_t* KB = ki + s0 + b0;
    const uint32_t* IB = ii + s0 + b0;
    // merge path: number i of A-elements among the first k outputs
    int64_t l = k - lb > 0 ? k - lb : 0, h = k < la ? k : la;
    while (l < h) {
      const int64_t m = (l + h) >> 1;
      // take A[m] before B[k-1-m]?
      if (less_kv(KA[m], IA[m], KB[k - 1 - m], IB[k - 1 - m])) l = m + 1;
      else h = m;
    }
    const int64_t i = l, j = k - i;
    bool take_a;
    if (i >= la) take_a = false;
    else if (j >= lb) take_a = true;
    else take_a = less_kv(KA[i], IA[i], KB[j], IB[j]);
    ko[g] = take_a ? KA[i] : KB[j];
    io[g] = take_a ? IA[i] : IB[j];
  }
}

__global__ void write_perm_kernel(const uint32_t* __restrict__ idx, int64_t n, int32_t* __restrict__ perm) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    perm[i] = static_cast<int32_t>(idx[i]);
}

}  // namespace

namespace fs {

void launch_rank(fs_device* dev, int32_t nseg, const int64_t* seg_h, const double* scores_d, int32_t* perm_d) {
  const int64_t n = seg_h[nseg] - seg_h[0];
  if (n <= 0) return;
  if (seg_h[0] != 0) fail(FS_EINVAL, "rank: seg[0] must be 0");
  int64_t max_len = 0;
  std::vector<ChunkDesc> chunks;
  for (int s = 0; s < nseg; ++s) {
    const int64_t len = seg_h[s + 1] - seg_h[s];
    if (len < 0) fail(FS_EINVAL, "rank: segment offsets must be non-decreasing");
    if (len > 0x7FFFFFFF) fail(FS_EINVAL, "rank: segment longer than 2^31-1");
    max_len = std::max(max_len, len);
    for (int64_t c = 0; c < len; c += kChunk)
      chunks.push_back({seg_h[s] + c, static_cast<int32_t>(std::min<int64_t>(kChunk, len - c)), 0});
  }
  // scratch: seg table + chunk table + 2x (keys, idx)
  const size_t seg_bytes = (static_cast<size_t>(nseg) + 1) * sizeof(int64_t);
  const size_t ch_bytes = chunks.size() * sizeof(ChunkDesc);
  auto* meta = static_cast<unsigned char*>(dev->scratch(kSlotRankKeys, seg_bytes + ch_bytes + 16 + n * 12));
  auto* seg_d = reinterpret_cast<int64_t*>(meta);
  auto* ch_d = reinterpret_cast<ChunkDesc*>(meta + seg_bytes);
  auto* ka = reinterpret_cast<uint64_t*>(meta + ((seg_bytes + ch_bytes + 15) & ~size_t(15)));
  auto* ia = reinterpret_cast<uint32_t*>(ka + n);
  auto* kb = static_cast<uint64_t*>(dev->scratch(kSlotRankKeys2, n * sizeof(uint64_t)));
  auto* ib = static_cast<uint32_t*>(dev->scratch(kSlotRankIdx2, n * sizeof(uint32_t)));
  FS_CUDA(cudaMemcpyAsync(seg_d, seg_h, seg_bytes, cudaMemcpyHostToDevice, dev->stream));
  FS_CUDA(cudaMemcpyAsync(ch_d, chunks.data(), ch_bytes, cudaMemcpyHostToDevice, dev->stream));
  const int grid = static_cast<int>(std::min<int64_t>(ceil_div(n, 256), dev->sm_count * 16));
  ProfScope prof(dev, "rank");
  make_keys_kernel<<<grid, 256, 0, dev->stream>>>(scores_d, seg_d, nseg, n, ka, ia);
  chunk_sort_kernel<<<static_cast<int>(chunks.size()), kSortThreads, 0, dev->stream>>>(ch_d, ka, ia);
  dev->count_launch(2);
  for (int64_t run = kChunk; run < max_len; run *= 2) {
    merge_pass_kernel<<<grid, 256, 0, dev->stream>>>(seg_d, nseg, n, run, ka, ia, kb, ib);
    dev->count_launch();
    std::swap(ka, kb);
    std::swap(ia, ib);
  }
  write_perm_kernel<<<grid, 256, 0, dev->stream>>>(ia, n, perm_d);
  dev->count_launch();
  FS_CUDA(cudaGetLastError());
}

}  // namespace fs

extern "C" {

int fs_rank_d(fs_device* dev, int32_t nseg, const int64_t* seg_h, const double* scores_d, int32_t* perm_d) {
  return fs::guard([&] {
    if (!dev || nseg < 0 || !seg_h) fs::fail(FS_EINVAL, "fs_rank: bad arguments");
    dev->activate();
    fs::launch_rank(dev, nseg, seg_h, scores_d, perm_d);
  });
}

int fs_rank(fs_device* dev, int32_t nseg, const int64_t* seg, const double* scores, int32_t* perm) {
  return fs::guard([&] {
    if (!dev || nseg < 0 || !seg) fs::fail(FS_EINVAL, "fs_rank: bad arguments");
    dev->activate();
    const int64_t n = seg[nseg] - seg[0];
    if (n <= 0) return;
    auto* sd = static_cast<double*>(dev->scratch(fs::kSlotH2D0, n * sizeof(double)));
    auto* pd = static_cast<int32_t*>(dev->scratch(fs::kSlotD2H0, n * sizeof(int32_t)));
    FS_CUDA(cudaMemcpyAsync(sd, scores, n * sizeof(double), cudaMemcpyHostToDevice, dev->stream));
    fs::launch_rank(dev, nseg, seg, sd, pd);
    FS_CUDA(cudaMemcpyAsync(perm, pd, n * sizeof(int32_t), cudaMemcpyDeviceToHost, dev->stream));
    fs::raise_deferred(dev->take_errors());
  });
}

}  // extern "C"
