// fs_score: the batched scoring block of tune_step (scheduler.cpp:187-192) in one call -
// featurize every pool candidate (searchspace.cpp:90-118), predict it with its family's model
// (costmodel.cpp:237-246), then rank each family's pool by (score, index). The feature matrix
// lives only in device scratch.
#include <algorithm>
#include <string>
#include <vector>
#include <cstdlib>

#include "forest.cuh"

namespace fs {
void launch_featurize(fs_device* dev, const fs_spaces* sp, int64_t n, const int32_t* space_of_d,
                      const int32_t* assign_d, int32_t pad, double* out_d);
void launch_predict(fs_device* dev, const fs_forest* fo, int32_t nseg, const int64_t* seg, int32_t d,
                    const double* x, double* scores, uint16_t* leaf_out);
void launch_rank(fs_device* dev, int32_t nseg, const int64_t* seg_h, const double* scores_d, int32_t* perm_d);
void launch_score_fused(fs_device* dev, const fs_spaces* spc, const fs_forest* fo, int32_t nseg, const int64_t* seg,
                        const int32_t* space_of_d, const int32_t* assign_d, int32_t pad, double* scores,
                        const uint64_t* index_d);

// candidate_from_index (searchspace.cpp:56-66) on the device: assignment[j] = (idx / prod_{k>j}
// m_k) % m_j, thread per (candidate, knob). Only the unfused fallback needs the assignments.
__global__ void decode_index_kernel(const int32_t* __restrict__ space_of, const uint64_t* __restrict__ index, int64_t n,
                                    const int32_t* __restrict__ k_d, const int32_t* __restrict__ nval,
                                    const uint64_t* __restrict__ stride, int n_spaces, int32_t* __restrict__ assign) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n * FS_MAX_KNOBS) return;
  const int64_t c = i / FS_MAX_KNOBS;
  const int j = static_cast<int>(i - c * FS_MAX_KNOBS);
  const int s = space_of[c];
  int a = 0;
  if (s >= 0 && s < n_spaces && j < k_d[s])
    a = static_cast<int>((index[c] / stride[s * FS_MAX_KNOBS + j]) % static_cast<uint64_t>(nval[s * FS_MAX_KNOBS + j]));
  assign[i] = a;
}

// index_d != nullptr: candidates are (space id, linear_index) descriptors (SURVEY.md 8f row 1:
// 4 + 8 bytes per candidate in, instead of the 4 + 64 of an int32[16] assignment)
void score_device(fs_device* dev, const fs_spaces* sp, const fs_forest* fo, int32_t nseg, const int64_t* seg,
                  const int32_t* space_of_d, const int32_t* assign_d, int32_t pad, double* scores_d, int32_t* perm_d,
                  const uint64_t* index_d) {
  const int64_t n = seg[nseg];
  if (n <= 0) return;
  if (seg[0] != 0) fail(FS_EINVAL, "score: seg[0] must be 0");
  // Fused by default: every tested feature is computed from the descriptor inside the predict
  // tile (no pad*8-byte feature row per candidate in HBM). FAMSEER_SCORE_UNFUSED=1 (or a
  // deeper-than-heap model) takes featurize -> predict through a device feature matrix.
  bool fused = std::getenv("FAMSEER_SCORE_UNFUSED") == nullptr;
  for (int f = 0; f < nseg && fused; ++f)
    if (f < static_cast<int32_t>(fo->fams.size()) && fo->fams[static_cast<size_t>(f)].generic) fused = false;
  if (fused) {
    launch_score_fused(dev, sp, fo, nseg, seg, space_of_d, assign_d, pad, scores_d, index_d);
  } else {
    if (index_d) {
      auto* as = static_cast<int32_t*>(dev->scratch(kSlotScoreA, static_cast<size_t>(n) * FS_MAX_KNOBS * sizeof(int32_t)));
      decode_index_kernel<<<static_cast<unsigned>(ceil_div(n * FS_MAX_KNOBS, 256)), 256, 0, dev->stream>>>(
          space_of_d, index_d, n, sp->k_d, sp->nval_d, sp->stride_d, sp->n, as);
      dev->count_launch();
      FS_CUDA(cudaGetLastError());
      assign_d = as;
    }
    auto* x = static_cast<double*>(dev->scratch(kSlotScoreX, static_cast<size_t>(n) * pad * sizeof(double)));
    launch_featurize(dev, sp, n, space_of_d, assign_d, pad, x);
    launch_predict(dev, fo, nseg, seg, pad, x, scores_d, nullptr);
  }
  if (perm_d) launch_rank(dev, nseg, seg, scores_d, perm_d);  // perm NULL: scores only
}

// pairwise_accuracy's pair count (costmodel.cpp:255-276): credit is counted in half units, so
// the device sum is an exact integer and the result is independent of summation order.
__global__ void pair_count_kernel(const double* __restrict__ s, const double* __restrict__ lat, int64_t m,
                                  unsigned long long* __restrict__ acc) {
  unsigned long long half = 0, counted = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double li = lat[i], si = s[i];
    for (int64_t j = i + 1; j < m; ++j) {
      const double lj = lat[j];
      const double rel = fs_div(fabs(fs_sub(li, lj)), li < lj ? lj : li);
      if (rel < 1e-6) continue;
      ++counted;
      const double sj = s[j];
      if (si == sj) half += 1;
      else if ((si < sj) == (li < lj)) half += 2;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    half += __shfl_down_sync(0xffffffffu, half, o);
    counted += __shfl_down_sync(0xffffffffu, counted, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(acc, half);
    atomicAdd(acc + 1, counted);
  }
}

// Batched pair counts: blockIdx.y = segment, counts in half units per segment (exact integers,
// order-independent).
__global__ void pair_count_seg_kernel(const double* __restrict__ s, const double* __restrict__ lat,
                                      const int64_t* __restrict__ seg, unsigned long long* __restrict__ acc) {
  const int k = blockIdx.y;
  const int64_t a = seg[k], m = seg[k + 1] - seg[k];
  unsigned long long half = 0, counted = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double li = lat[a + i], si = s[a + i];
    for (int64_t j = i + 1; j < m; ++j) {
      const double lj = lat[a + j];
      const double rel = fs_div(fabs(fs_sub(li, lj)), li < lj ? lj : li);
      if (rel < 1e-6) continue;
      ++counted;
      const double sj = s[a + j];
      if (si == sj) half += 1;
      else if ((si < sj) == (li < lj)) half += 2;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    half += __shfl_down_sync(0xffffffffu, half, o);
    counted += __shfl_down_sync(0xffffffffu, counted, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(acc + 2 * k, half);
    atomicAdd(acc + 2 * k + 1, counted);
  }
}

}  // namespace fs

extern "C" {

int fs_pairwise_accuracy_batch(fs_device* dev, int32_t nseg, const int64_t* seg, const double* scores,
                               const double* latency, double* out) {
  return fs::guard([&] {
    if (!dev || !out || nseg < 0 || (nseg > 0 && (!seg || !scores || !latency)))
      fs::fail(FS_EINVAL, "fs_pairwise_accuracy_batch: bad arguments");
    if (nseg == 0) return;
    if (seg[0] != 0) fs::fail(FS_EINVAL, "fs_pairwise_accuracy_batch: seg[0] must be 0");
    int64_t mmax = 0;
    for (int k = 0; k < nseg; ++k) {
      const int64_t m = seg[k + 1] - seg[k];
      if (m < 2)
        fs::fail(FS_EINVAL, "pairwise_accuracy: segment " + std::to_string(k) + " has fewer than two records");
      mmax = std::max(mmax, m);
    }
    dev->activate();
    const int64_t n = seg[nseg];
    auto* buf = static_cast<unsigned char*>(
        dev->scratch(fs::kSlotH2D0, static_cast<size_t>(n) * 16 + static_cast<size_t>(nseg + 1) * 8 + nseg * 16 + 64));
    auto* sd = reinterpret_cast<double*>(buf);
    auto* ld = sd + n;
    auto* segd = reinterpret_cast<int64_t*>(ld + n);
    auto* acc = reinterpret_cast<unsigned long long*>(segd + nseg + 1);
    FS_CUDA(cudaMemcpyAsync(sd, scores, n * sizeof(double), cudaMemcpyHostToDevice, dev->stream));
    FS_CUDA(cudaMemcpyAsync(ld, latency, n * sizeof(double), cudaMemcpyHostToDevice, dev->stream));
    FS_CUDA(cudaMemcpyAsync(segd, seg, (nseg + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, dev->stream));
    FS_CUDA(cudaMemsetAsync(acc, 0, 2 * nseg * sizeof(unsigned long long), dev->stream));
    const unsigned gx = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(fs::ceil_div(mmax, 256), 64)));
    fs::pair_count_seg_kernel<<<dim3(gx, static_cast<unsigned>(nseg)), 256, 0, dev->stream>>>(sd, ld, segd, acc);
    dev->count_launch();
    FS_CUDA(cudaGetLastError());
    std::vector<unsigned long long> h(2 * static_cast<size_t>(nseg));
    FS_CUDA(cudaMemcpyAsync(h.data(), acc, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, dev->stream));
    FS_CUDA(cudaStreamSynchronize(dev->stream));
    for (int k = 0; k < nseg; ++k) {
      if (h[2 * k + 1] == 0)
        fs::fail(FS_EDOMAIN, "pairwise_accuracy: segment " + std::to_string(k) + ": all validation pairs excluded as ties");
      out[k] = (static_cast<double>(h[2 * k]) * 0.5) / static_cast<double>(h[2 * k + 1]);
    }
  });
}


int fs_pairwise_accuracy(fs_device* dev, int64_t m, const double* scores, const double* latency, double* out) {
  return fs::guard([&] {
    if (!dev || !out || m < 0) fs::fail(FS_EINVAL, "fs_pairwise_accuracy: bad arguments");
    if (m < 2) fs::fail(FS_EINVAL, "pairwise_accuracy: need at least two validation records");
    dev->activate();
    auto* buf = static_cast<unsigned char*>(dev->scratch(fs::kSlotH2D0, static_cast<size_t>(m) * 16 + 64));
    auto* sd = reinterpret_cast<double*>(buf);
    auto* ld = sd + m;
    auto* acc = reinterpret_cast<unsigned long long*>(ld + m);
    FS_CUDA(cudaMemcpyAsync(sd, scores, m * sizeof(double), cudaMemcpyHostToDevice, dev->stream));
    FS_CUDA(cudaMemcpyAsync(ld, latency, m * sizeof(double), cudaMemcpyHostToDevice, dev->stream));
    FS_CUDA(cudaMemsetAsync(acc, 0, 2 * sizeof(unsigned long long), dev->stream));
    const int grid = static_cast<int>(std::min<int64_t>(fs::ceil_div(m, 256), dev->sm_count * 8));
    fs::pair_count_kernel<<<grid, 256, 0, dev->stream>>>(sd, ld, m, acc);
    dev->count_launch();
    FS_CUDA(cudaGetLastError());
    unsigned long long h[2] = {0, 0};
    FS_CUDA(cudaMemcpyAsync(h, acc, sizeof h, cudaMemcpyDeviceToHost, dev->stream));
    FS_CUDA(cudaStreamSynchronize(dev->stream));
    if (h[1] == 0) fs::fail(FS_EDOMAIN, "pairwise_accuracy: all validation pairs excluded as ties");
    *out = (static_cast<double>(h[0]) * 0.5) / static_cast<double>(h[1]);
  });
}

int fs_score_d(fs_device* dev, const fs_spaces* sp, const fs_forest* fo, int32_t nseg, const int64_t* seg_h,
               const int32_t* space_of_d, const int32_t* assign_d, int32_t pad_dim, double* scores_d,
               int32_t* perm_d) {
  return fs::guard([&] {
    if (!dev || !sp || !fo || nseg < 0 || !seg_h || pad_dim < 0) fs::fail(FS_EINVAL, "fs_score: bad arguments");
    dev->activate();
    fs::score_device(dev, sp, fo, nseg, seg_h, space_of_d, assign_d, pad_dim, scores_d, perm_d, nullptr);
  });
}

int fs_score(fs_device* dev, const fs_spaces* sp, const fs_forest* fo, int32_t nseg, const int64_t* seg,
             const int32_t* space_of, const int32_t* assign, int32_t pad_dim, double* scores, int32_t* perm) {
  return fs::guard([&] {
    if (!dev || !sp || !fo || nseg < 0 || !seg || pad_dim < 0) fs::fail(FS_EINVAL, "fs_score: bad arguments");
    dev->activate();
    const int64_t n = seg[nseg];
    if (n <= 0) return;
    auto* so = static_cast<int32_t*>(dev->scratch(fs::kSlotH2D0, n * sizeof(int32_t)));
    auto* as = static_cast<int32_t*>(dev->scratch(fs::kSlotH2D1, n * FS_MAX_KNOBS * sizeof(int32_t)));
    auto* sd = static_cast<double*>(dev->scratch(fs::kSlotScoreS, n * sizeof(double)));
    auto* pd = static_cast<int32_t*>(dev->scratch(fs::kSlotScoreP, n * sizeof(int32_t)));
    FS_CUDA(cudaMemcpyAsync(so, space_of, n * sizeof(int32_t), cudaMemcpyHostToDevice, dev->stream));
    FS_CUDA(cudaMemcpyAsync(as, assign, n * FS_MAX_KNOBS * sizeof(int32_t), cudaMemcpyHostToDevice, dev->stream));
    fs::score_device(dev, sp, fo, nseg, seg, so, as, pad_dim, sd, pd, nullptr);
    if (scores) FS_CUDA(cudaMemcpyAsync(scores, sd, n * sizeof(double), cudaMemcpyDeviceToHost, dev->stream));
    if (perm) FS_CUDA(cudaMemcpyAsync(perm, pd, n * sizeof(int32_t), cudaMemcpyDeviceToHost, dev->stream));
    fs::raise_deferred(dev->take_errors());
  });
}

int fs_score_index_d(fs_device* dev, const fs_spaces* sp, const fs_forest* fo, int32_t nseg, const int64_t* seg_h,
                     const int32_t* space_of_d, const uint64_t* index_d, int32_t pad_dim, double* scores_d,
                     int32_t* perm_d) {
  return fs::guard([&] {
    if (!dev || !sp || !fo || nseg < 0 || !seg_h || pad_dim < 0) fs::fail(FS_EINVAL, "fs_score_index: bad arguments");
    dev->activate();
    fs::score_device(dev, sp, fo, nseg, seg_h, space_of_d, nullptr, pad_dim, scores_d, perm_d, index_d);
  });
}

int fs_score_index(fs_device* dev, const fs_spaces* sp, const fs_forest* fo, int32_t nseg, const int64_t* seg,
                   const int32_t* space_of, const uint64_t* index, int32_t pad_dim, double* scores, int32_t* perm) {
  return fs::guard([&] {
    if (!dev || !sp || !fo || nseg < 0 || !seg || pad_dim < 0) fs::fail(FS_EINVAL, "fs_score_index: bad arguments");
    dev->activate();
    const int64_t n = seg[nseg];
    if (n <= 0) return;
    auto* so = static_cast<int32_t*>(dev->scratch(fs::kSlotH2D0, n * sizeof(int32_t)));
    auto* ix = static_cast<uint64_t*>(dev->scratch(fs::kSlotH2D1, n * sizeof(uint64_t)));
    auto* sd = static_cast<double*>(dev->scratch(fs::kSlotScoreS, n * sizeof(double)));
    auto* pd = static_cast<int32_t*>(dev->scratch(fs::kSlotScoreP, n * sizeof(int32_t)));
    FS_CUDA(cudaMemcpyAsync(so, space_of, n * sizeof(int32_t), cudaMemcpyHostToDevice, dev->stream));
    FS_CUDA(cudaMemcpyAsync(ix, index, n * sizeof(uint64_t), cudaMemcpyHostToDevice, dev->stream));
    fs::score_device(dev, sp, fo, nseg, seg, so, nullptr, pad_dim, sd, pd, ix);
    if (scores) FS_CUDA(cudaMemcpyAsync(scores, sd, n * sizeof(double), cudaMemcpyDeviceToHost, dev->stream));
    if (perm) FS_CUDA(cudaMemcpyAsync(perm, pd, n * sizeof(int32_t), cudaMemcpyDeviceToHost, dev->stream));
    fs::raise_deferred(dev->take_errors());
  });
}

}  // extern "C"
