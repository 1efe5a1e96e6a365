// fs_score: the batched scoring block of tune_step (scheduler.cpp:187-192) in one call -
// featurize every pool candidate (searchspace.cpp:90-118), predict it with its family's model
// (costmodel.cpp:237-246), then rank each family's pool by (score, index). The feature matrix
// lives only in device scratch.
#include <algorithm>

#include "forest.cuh"

namespace fs {
void launch_featurize(fs_device* dev, const fs_spaces* sp, int64_t n, const int32_t* space_of_d,
                      const int32_t* assign_d, int32_t pad, double* out_d);
void launch_predict(fs_device* dev, const fs_forest* fo, int32_t nseg, const int64_t* seg, int32_t d,
                    const double* x, double* scores, uint8_t* leaf_out);
void launch_rank(fs_device* dev, int32_t nseg, const int64_t* seg_h, const double* scores_d, int32_t* perm_d);

static void score_device(fs_device* dev, const fs_spaces* sp, const fs_forest* fo, int32_t nseg, const int64_t* seg,
                         const int32_t* space_of_d, const int32_t* assign_d, int32_t pad, double* scores_d,
                         int32_t* perm_d) {
  const int64_t n = seg[nseg];
  if (n <= 0) return;
  if (seg[0] != 0) fail(FS_EINVAL, "score: seg[0] must be 0");
  auto* x = static_cast<double*>(dev->scratch(kSlotScoreX, static_cast<size_t>(n) * pad * sizeof(double)));
  launch_featurize(dev, sp, n, space_of_d, assign_d, pad, x);
  launch_predict(dev, fo, nseg, seg, pad, x, scores_d, nullptr);
  launch_rank(dev, nseg, seg, scores_d, perm_d);
}

}  // namespace fs

extern "C" {

int fs_score_d(fs_device* dev, const fs_spaces* sp, const fs_forest* fo, int32_t nseg, const int64_t* seg_h,
               const int32_t* space_of_d, const int32_t* assign_d, int32_t pad_dim, double* scores_d,
               int32_t* perm_d) {
  return fs::guard([&] {
    if (!dev || !sp || !fo || nseg < 0 || !seg_h || pad_dim < 0) fs::fail(FS_EINVAL, "fs_score: bad arguments");
    dev->activate();
    fs::score_device(dev, sp, fo, nseg, seg_h, space_of_d, assign_d, pad_dim, scores_d, perm_d);
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
    fs::score_device(dev, sp, fo, nseg, seg, so, as, pad_dim, sd, pd);
    if (scores) FS_CUDA(cudaMemcpyAsync(scores, sd, n * sizeof(double), cudaMemcpyDeviceToHost, dev->stream));
    if (perm) FS_CUDA(cudaMemcpyAsync(perm, pd, n * sizeof(int32_t), cudaMemcpyDeviceToHost, dev->stream));
    fs::raise_deferred(dev->take_errors());
  });
}

}  // extern "C"
