// fs_forest: the family model store (scheduler.cpp:123-130 models_) and its compiled predict
// form. See forest.cuh for the layout.
#include <algorithm>
#include <cmath>
#include <functional>
#include <memory>

#include "forest.cuh"

namespace fs {

void FamilyModel::release_device() {
  for (void* p : {static_cast<void*>(nodes_d), static_cast<void*>(leafv_d), static_cast<void*>(leafid_d),
                  static_cast<void*>(uthr_d), static_cast<void*>(uoff_d), static_cast<void*>(g_off_d),
                  static_cast<void*>(g_feat_d), static_cast<void*>(g_thr_d), static_cast<void*>(g_left_d),
                  static_cast<void*>(g_right_d), static_cast<void*>(g_val_d)})
    if (p) cudaFree(p);
  nodes_d = nullptr;
  leafv_d = nullptr;
  leafid_d = nullptr;
  uthr_d = nullptr;
  uoff_d = nullptr;
  g_off_d = g_feat_d = g_left_d = g_right_d = nullptr;
  g_thr_d = g_val_d = nullptr;
  compiled = false;
}

namespace {

template <class T>
T* upload(const std::vector<T>& v, cudaStream_t s) {
  T* p = nullptr;
  FS_CUDA(cudaMalloc(&p, std::max<size_t>(1, v.size()) * sizeof(T)));
  if (!v.empty()) FS_CUDA(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  return p;
}

}  // namespace

void compile_model(fs_device* dev, FamilyModel& m) {
  m.release_device();
  const int T = m.num_trees();
  m.n_trees = T;
  // Validate structure and find depth / feature range.
  int depth = 0, dmodel = 0;
  std::function<int(int, int, int)> walk = [&](int o, int idx, int lvl) -> int {
    const int n = m.offsets[static_cast<size_t>(o) + 1] - m.offsets[static_cast<size_t>(o)];
    if (idx < 0 || idx >= n || lvl > 64) fail(FS_EINVAL, "forest: malformed tree (child index out of range)");
    const size_t g = static_cast<size_t>(m.offsets[static_cast<size_t>(o)] + idx);
    if (m.feature[g] < 0) return lvl;
    dmodel = std::max(dmodel, m.feature[g] + 1);
    return std::max(walk(o, m.left[g], lvl + 1), walk(o, m.right[g], lvl + 1));
  };
  for (int t = 0; t < T; ++t) {
    if (m.offsets[static_cast<size_t>(t) + 1] <= m.offsets[static_cast<size_t>(t)])
      fail(FS_EINVAL, "forest: empty tree");
    depth = std::max(depth, walk(t, 0, 0));
  }
  if (dmodel > 65535) fail(FS_EINVAL, "forest: feature index exceeds 65535");
  m.depth = depth;
  m.d_model = dmodel;
  m.generic = depth > kMaxHeapDepth;

  if (m.generic) {
    m.g_off_d = upload(m.offsets, dev->stream);
    m.g_feat_d = upload(m.feature, dev->stream);
    m.g_thr_d = upload(m.threshold, dev->stream);
    m.g_left_d = upload(m.left, dev->stream);
    m.g_right_d = upload(m.right, dev->stream);
    m.g_val_d = upload(m.value, dev->stream);
    FS_CUDA(cudaStreamSynchronize(dev->stream));
    m.compiled = true;
    return;
  }

  // Unique thresholds per feature (== equality, so -0.0 and +0.0 share a rank).
  std::vector<std::vector<double>> uq(static_cast<size_t>(dmodel));
  for (size_t g = 0; g < m.feature.size(); ++g)
    if (m.feature[g] >= 0) uq[static_cast<size_t>(m.feature[g])].push_back(m.threshold[g]);
  size_t max_u = 0;
  std::vector<int32_t> uoff(static_cast<size_t>(dmodel) + 1, 0);
  std::vector<double> uthr;
  for (int f = 0; f < dmodel; ++f) {
    auto& u = uq[static_cast<size_t>(f)];
    std::sort(u.begin(), u.end());
    u.erase(std::unique(u.begin(), u.end(), [](double a, double b) { return a == b; }), u.end());
    uoff[static_cast<size_t>(f)] = static_cast<int32_t>(uthr.size());
    uthr.insert(uthr.end(), u.begin(), u.end());
    max_u = std::max(max_u, u.size());
  }
  uoff[static_cast<size_t>(dmodel)] = static_cast<int32_t>(uthr.size());
  if (max_u > 65534) fail(FS_EINVAL, "forest: more than 65534 distinct thresholds on one feature");
  m.code_bytes = max_u <= 254 ? 1 : 2;
  const uint32_t always_left_rank = m.code_bytes == 1 ? 0xFFu : 0xFFFFu;

  const int nint = (1 << depth) - 1;
  const int nleaf = 1 << depth;
  std::vector<uint32_t> nodes(static_cast<size_t>(T) * nint, 0);
  std::vector<double> leafv(static_cast<size_t>(T) * nleaf, 0.0);
  std::vector<uint8_t> leafid(static_cast<size_t>(T) * nleaf, 0);
  for (int t = 0; t < T; ++t) {
    const int o = m.offsets[static_cast<size_t>(t)];
    std::function<void(int, int, int)> place = [&](int idx, int heap, int lvl) {
      const size_t g = static_cast<size_t>(o + idx);
      if (lvl == depth) {
        leafv[static_cast<size_t>(t) * nleaf + (heap - nint)] = m.value[g];
        leafid[static_cast<size_t>(t) * nleaf + (heap - nint)] = static_cast<uint8_t>(idx);
        return;
      }
      uint32_t node;
      int li, ri;
      if (m.feature[g] < 0) {  // early leaf: replicate down an always-left path
        node = always_left_rank << 16;
        li = ri = idx;
      } else {
        const int f = m.feature[g];
        const auto& u = uq[static_cast<size_t>(f)];
        const auto rank = static_cast<uint32_t>(std::lower_bound(u.begin(), u.end(), m.threshold[g]) - u.begin());
        node = static_cast<uint32_t>(f) | (rank << 16);
        li = m.left[g];
        ri = m.right[g];
      }
      nodes[static_cast<size_t>(t) * nint + heap] = node;
      place(li, 2 * heap + 1, lvl + 1);
      place(ri, 2 * heap + 2, lvl + 1);
    };
    place(0, 0, 0);
  }
  m.nodes_d = upload(nodes, dev->stream);
  m.leafv_d = upload(leafv, dev->stream);
  m.leafid_d = upload(leafid, dev->stream);
  m.uthr_d = upload(uthr, dev->stream);
  m.n_uthr = static_cast<int>(uthr.size());
  m.uoff_d = upload(uoff, dev->stream);
  FS_CUDA(cudaStreamSynchronize(dev->stream));
  m.compiled = true;
}

}  // namespace fs

extern "C" {

int fs_forest_create(fs_device* dev, int32_t n_families, fs_forest** out) {
  return fs::guard([&] {
    if (!dev || !out || n_families < 1) fs::fail(FS_EINVAL, "fs_forest_create: bad arguments");
    auto fo = std::make_unique<fs_forest>();
    fo->dev = dev;
    fo->fams.resize(static_cast<size_t>(n_families));
    *out = fo.release();
  });
}

int fs_forest_destroy(fs_forest* fo) {
  return fs::guard([&] {
    if (!fo) return;
    fo->dev->activate();
    cudaStreamSynchronize(fo->dev->stream);
    for (auto& m : fo->fams) m.release_device();
    delete fo;
  });
}

int fs_forest_upload(fs_forest* fo, int32_t family, double base, double lr, int32_t n_trees,
                     const int32_t* offsets, const int32_t* feature, const double* threshold,
                     const int32_t* left, const int32_t* right, const double* value) {
  return fs::guard([&] {
    if (!fo || family < 0 || family >= static_cast<int32_t>(fo->fams.size()) || n_trees < 0)
      fs::fail(FS_ERANGE, "fs_forest_upload: unknown family id " + std::to_string(family));
    fo->dev->activate();
    auto& m = fo->fams[static_cast<size_t>(family)];
    m.base = base;
    m.lr = lr;
    m.offsets.assign(offsets, offsets + n_trees + 1);
    if (m.offsets.front() != 0) fs::fail(FS_EINVAL, "forest: offsets[0] must be 0");
    const int32_t nn = m.offsets.back();
    m.feature.assign(feature, feature + nn);
    m.threshold.assign(threshold, threshold + nn);
    m.left.assign(left, left + nn);
    m.right.assign(right, right + nn);
    m.value.assign(value, value + nn);
    m.gain.assign(static_cast<size_t>(nn), 0.0);
    m.mse.clear();
    fs::compile_model(fo->dev, m);
  });
}

int fs_forest_export(const fs_forest* fo, int32_t family, double* base, int32_t* n_trees, int32_t* n_nodes,
                     int32_t* offsets, int32_t* feature, double* threshold, int32_t* left, int32_t* right,
                     double* value, double* gain, double* mse) {
  return fs::guard([&] {
    if (!fo || family < 0 || family >= static_cast<int32_t>(fo->fams.size()))
      fs::fail(FS_ERANGE, "fs_forest_export: unknown family id " + std::to_string(family));
    const auto& m = fo->fams[static_cast<size_t>(family)];
    const int T = m.num_trees();
    const int N = m.offsets.back();
    if (base) *base = m.base;
    if (n_trees) *n_trees = T;
    if (n_nodes) *n_nodes = N;
    if (offsets) std::copy(m.offsets.begin(), m.offsets.end(), offsets);
    if (feature) std::copy(m.feature.begin(), m.feature.end(), feature);
    if (threshold) std::copy(m.threshold.begin(), m.threshold.end(), threshold);
    if (left) std::copy(m.left.begin(), m.left.end(), left);
    if (right) std::copy(m.right.begin(), m.right.end(), right);
    if (value) std::copy(m.value.begin(), m.value.end(), value);
    if (gain) {
      std::fill(gain, gain + N, 0.0);
      std::copy(m.gain.begin(), m.gain.begin() + std::min<size_t>(m.gain.size(), N), gain);
    }
    if (mse) std::copy(m.mse.begin(), m.mse.end(), mse);
  });
}

}  // extern "C"
