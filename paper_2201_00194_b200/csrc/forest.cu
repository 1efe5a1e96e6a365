// fs_forest: the family model store (scheduler.cpp:123-130 models_) and its compiled predict
// form. See forest.cuh for the layout.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <memory>

#include "forest.cuh"

namespace fs {

void FamilyModel::release_device() {
  if (blob_d) cudaFree(blob_d);
  blob_d = nullptr;
  blob_cap = 0;
  pending = false;
  fmap_d = nullptr;
  meta_d = nullptr;
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

// Packs host arrays into one staging buffer (16-byte aligned parts) and copies it into the
// model's grow-only device blob with a single async copy. Pageable-source cudaMemcpyAsync
// returns once the bytes are staged, so the host vectors may die right after.
struct BlobPacker {
  std::vector<unsigned char> host;
  std::vector<size_t> offs;
  template <class T>
  void add(const std::vector<T>& v) {
    const size_t o = (host.size() + 15) & ~size_t(15);
    offs.push_back(o);
    host.resize(o + std::max<size_t>(1, v.size()) * sizeof(T), 0);
    if (!v.empty()) std::memcpy(host.data() + o, v.data(), v.size() * sizeof(T));
  }
  void commit(FamilyModel& m, fs_device* dev, UploadBatch* batch) {
    if (host.size() > m.blob_cap) {
      if (m.blob_d) FS_CUDA(cudaFree(m.blob_d));
      m.blob_d = nullptr;
      const size_t cap = std::max<size_t>(host.size() + host.size() / 2, 4096);
      FS_CUDA(cudaMalloc(&m.blob_d, cap));
      m.blob_cap = cap;
    }
    if (batch) {
      batch->add(m.blob_d, host.data(), host.size());
      return;
    }
    // through pinned staging: a truly asynchronous copy (no pageable-staging stream sync)
    void* st = dev->pinned_upload(host.size());
    std::memcpy(st, host.data(), host.size());
    FS_CUDA(cudaMemcpyAsync(m.blob_d, st, host.size(), cudaMemcpyHostToDevice, dev->stream));
    dev->upload_done();
  }
  template <class T>
  T* at(const FamilyModel& m, int i) const {
    return reinterpret_cast<T*>(m.blob_d + offs[static_cast<size_t>(i)]);
  }
};

}  // namespace

void UploadBatch::add(unsigned char* dst, const unsigned char* src, size_t bytes) {
  const size_t o = (host.size() + 15) & ~size_t(15);
  host.resize(o + bytes);
  std::memcpy(host.data() + o, src, bytes);
  items.push_back({dst, {o, bytes}});
}

void UploadBatch::flush(fs_device* dev) {
  if (items.empty()) return;
  auto* st = static_cast<unsigned char*>(dev->pinned_upload(host.size()));
  std::memcpy(st, host.data(), host.size());
  for (const auto& it : items)
    FS_CUDA(cudaMemcpyAsync(it.first, st + it.second.first, it.second.second, cudaMemcpyHostToDevice, dev->stream));
  dev->upload_done();
  items.clear();
  host.clear();
}

void materialize(fs_device* dev, const FamilyModel& m) { materialize(dev, const_cast<FamilyModel&>(m)); }

namespace {
// the pre-order arrays of a pending model from its device export region, already on the host
void materialize_from(FamilyModel& m, const unsigned char* h) {
  const DevLayout& L = m.lay;
  auto at = [&](size_t off) { return h + (off - L.meta); };
  ModelMeta meta;
  std::memcpy(&meta, at(L.meta), sizeof meta);
  const int T = meta.n_trees, S = L.slots;
  const auto* cnt = reinterpret_cast<const int32_t*>(at(L.cnt));
  const auto* feat = reinterpret_cast<const int32_t*>(at(L.feat));
  const auto* thr = reinterpret_cast<const double*>(at(L.thr));
  const auto* lft = reinterpret_cast<const int32_t*>(at(L.left));
  const auto* rgt = reinterpret_cast<const int32_t*>(at(L.right));
  const auto* val = reinterpret_cast<const double*>(at(L.val));
  const auto* gn = reinterpret_cast<const double*>(at(L.gain));
  const auto* mse = reinterpret_cast<const double*>(at(L.mse));
  m.base = meta.base;
  m.screened = meta.screened;
  m.exact = meta.exact;
  m.offsets.assign(1, 0);
  m.feature.clear();
  m.threshold.clear();
  m.left.clear();
  m.right.clear();
  m.value.clear();
  m.gain.clear();
  for (int t = 0; t < T; ++t) {
    const size_t o = static_cast<size_t>(t) * S;
    const int c = cnt[t];
    m.feature.insert(m.feature.end(), feat + o, feat + o + c);
    m.threshold.insert(m.threshold.end(), thr + o, thr + o + c);
    m.left.insert(m.left.end(), lft + o, lft + o + c);
    m.right.insert(m.right.end(), rgt + o, rgt + o + c);
    m.value.insert(m.value.end(), val + o, val + o + c);
    m.gain.insert(m.gain.end(), gn + o, gn + o + c);
    m.offsets.push_back(static_cast<int32_t>(m.feature.size()));
  }
  m.mse.assign(mse, mse + T);
  m.n_trees = T;
  m.pending = false;
}
}  // namespace

void materialize(fs_device* dev, FamilyModel& m) {
  if (!m.pending) return;
  const size_t bytes = m.lay.total - m.lay.meta;
  std::vector<unsigned char> h(bytes);
  FS_CUDA(cudaMemcpyAsync(h.data(), m.blob_d + m.lay.meta, bytes, cudaMemcpyDeviceToHost, dev->stream));
  FS_CUDA(cudaStreamSynchronize(dev->stream));
  materialize_from(m, h.data());
}

// Every pending family of a forest in one pinned device->host read and one synchronisation
// (a fit leaves all its families pending; the first export of any of them fetches them all).
// Split in two so a caller that synchronises anyway (fs_tune_step) can enqueue the read before
// its own synchronisation: materialize_enqueue stages the copies in the device's pinned buffer
// (nothing else may use it until materialize_parse), materialize_parse reads them afterwards.
bool materialize_enqueue(fs_device* dev, std::vector<FamilyModel>& fams) {
  size_t tot = 0;
  for (const auto& m : fams)
    if (m.pending) tot += (m.lay.total - m.lay.meta + 15) & ~size_t(15);
  if (tot == 0) return false;
  auto* h = static_cast<unsigned char*>(dev->pinned(tot));
  size_t o = 0;
  for (const auto& m : fams) {
    if (!m.pending) continue;
    const size_t bytes = m.lay.total - m.lay.meta;
    FS_CUDA(cudaMemcpyAsync(h + o, m.blob_d + m.lay.meta, bytes, cudaMemcpyDeviceToHost, dev->stream));
    o += (bytes + 15) & ~size_t(15);
  }
  return true;
}
void materialize_parse(fs_device* dev, std::vector<FamilyModel>& fams) {
  const auto* h = static_cast<const unsigned char*>(dev->pinned_h);
  size_t o = 0;
  for (auto& m : fams) {
    if (!m.pending) continue;
    const size_t bytes = m.lay.total - m.lay.meta;
    materialize_from(m, h + o);
    o += (bytes + 15) & ~size_t(15);
  }
}
void materialize_all(fs_device* dev, std::vector<FamilyModel>& fams) {
  if (!materialize_enqueue(dev, fams)) return;
  FS_CUDA(cudaStreamSynchronize(dev->stream));
  materialize_parse(dev, fams);
}

void compile_model(fs_device* dev, FamilyModel& m, UploadBatch* batch) {
  m.compiled = false;
  m.pending = false;
  m.fmap_d = nullptr;
  m.meta_d = nullptr;
  const int T = m.num_trees();
  m.n_trees = T;
  // Validate structure and find depth / feature range.
  int depth = 0, dmodel = 0;
  std::vector<std::pair<int, int>> stk;  // (node index in tree, level)
  for (int t = 0; t < T; ++t) {
    const int o = m.offsets[static_cast<size_t>(t)];
    const int n = m.offsets[static_cast<size_t>(t) + 1] - o;
    if (n <= 0) fail(FS_EINVAL, "forest: empty tree");
    stk.assign(1, {0, 0});
    while (!stk.empty()) {
      const auto [idx, lvl] = stk.back();
      stk.pop_back();
      if (idx < 0 || idx >= n || lvl > 64) fail(FS_EINVAL, "forest: malformed tree (child index out of range)");
      const size_t g = static_cast<size_t>(o + idx);
      if (m.feature[g] < 0) {
        depth = std::max(depth, lvl);
        continue;
      }
      dmodel = std::max(dmodel, m.feature[g] + 1);
      stk.push_back({m.left[g], lvl + 1});
      stk.push_back({m.right[g], lvl + 1});
    }
  }
  if (dmodel > 65535) fail(FS_EINVAL, "forest: feature index exceeds 65535");
  m.depth = depth;
  m.d_model = dmodel;
  m.generic = depth > kMaxHeapDepth;

  if (m.generic) {
    BlobPacker pk;
    pk.add(m.offsets);
    pk.add(m.feature);
    pk.add(m.threshold);
    pk.add(m.left);
    pk.add(m.right);
    pk.add(m.value);
    pk.commit(m, dev, batch);
    m.g_off_d = pk.at<int32_t>(m, 0);
    m.g_feat_d = pk.at<int32_t>(m, 1);
    m.g_thr_d = pk.at<double>(m, 2);
    m.g_left_d = pk.at<int32_t>(m, 3);
    m.g_right_d = pk.at<int32_t>(m, 4);
    m.g_val_d = pk.at<double>(m, 5);
    m.nodes_d = nullptr;
    m.compiled = true;
    return;
  }

  // Unique thresholds per feature (== equality, so -0.0 and +0.0 share a rank): one sort of all
  // (feature, threshold) pairs, then per-feature slices.
  std::vector<std::pair<int, double>> ft;
  ft.reserve(m.feature.size());
  for (size_t g = 0; g < m.feature.size(); ++g)
    if (m.feature[g] >= 0) ft.push_back({m.feature[g], m.threshold[g]});
  std::sort(ft.begin(), ft.end(), [](const std::pair<int, double>& a, const std::pair<int, double>& b) {
    return a.first != b.first ? a.first < b.first : a.second < b.second;
  });
  std::vector<int32_t> uoff(static_cast<size_t>(dmodel) + 1, 0);
  std::vector<double> uthr;
  uthr.reserve(ft.size());
  size_t max_u = 0;
  {
    size_t i = 0;
    for (int f = 0; f < dmodel; ++f) {
      uoff[static_cast<size_t>(f)] = static_cast<int32_t>(uthr.size());
      const size_t start = uthr.size();
      for (; i < ft.size() && ft[i].first == f; ++i)
        if (uthr.size() == start || !(uthr.back() == ft[i].second)) uthr.push_back(ft[i].second);
      max_u = std::max(max_u, uthr.size() - start);
    }
  }
  uoff[static_cast<size_t>(dmodel)] = static_cast<int32_t>(uthr.size());
  if (max_u > 65534) fail(FS_EINVAL, "forest: more than 65534 distinct thresholds on one feature");
  m.code_bytes = max_u <= 254 ? 1 : 2;
  const uint32_t always_left_rank = m.code_bytes == 1 ? 0xFFu : 0xFFFFu;

  const int nint = (1 << depth) - 1;
  const int nleaf = 1 << depth;
  std::vector<uint32_t> nodes(static_cast<size_t>(T) * nint, 0);
  std::vector<double> leafv(static_cast<size_t>(T) * nleaf, 0.0);
  std::vector<uint16_t> leafid(static_cast<size_t>(T) * nleaf, 0);
  struct Place {
    int idx, heap, lvl;
  };
  std::vector<Place> ps;
  for (int t = 0; t < T; ++t) {
    const int o = m.offsets[static_cast<size_t>(t)];
    ps.assign(1, {0, 0, 0});
    while (!ps.empty()) {
      const Place c = ps.back();
      ps.pop_back();
      const size_t g = static_cast<size_t>(o + c.idx);
      if (c.lvl == depth) {
        leafv[static_cast<size_t>(t) * nleaf + (c.heap - nint)] = m.value[g];
        leafid[static_cast<size_t>(t) * nleaf + (c.heap - nint)] = static_cast<uint16_t>(c.idx);
        continue;
      }
      uint32_t node;
      int li, ri;
      if (m.feature[g] < 0) {  // early leaf: replicate down an always-left path
        node = always_left_rank << 16;
        li = ri = c.idx;
      } else {
        const int f = m.feature[g];
        const double* u0 = uthr.data() + uoff[static_cast<size_t>(f)];
        const double* u1 = uthr.data() + uoff[static_cast<size_t>(f) + 1];
        const auto rank = static_cast<uint32_t>(std::lower_bound(u0, u1, m.threshold[g]) - u0);
        node = static_cast<uint32_t>(f) | (rank << 16);
        li = m.left[g];
        ri = m.right[g];
      }
      nodes[static_cast<size_t>(t) * nint + c.heap] = node;
      ps.push_back({li, 2 * c.heap + 1, c.lvl + 1});
      ps.push_back({ri, 2 * c.heap + 2, c.lvl + 1});
    }
  }
  BlobPacker pk;
  pk.add(nodes);
  pk.add(leafv);
  pk.add(leafid);
  pk.add(uthr);
  pk.add(uoff);
  pk.commit(m, dev, batch);
  m.nodes_d = pk.at<uint32_t>(m, 0);
  m.leafv_d = pk.at<double>(m, 1);
  m.leafid_d = pk.at<uint16_t>(m, 2);
  m.uthr_d = pk.at<double>(m, 3);
  m.n_uthr = static_cast<int>(uthr.size());
  m.uoff_d = pk.at<int32_t>(m, 4);
  m.g_off_d = m.g_feat_d = m.g_left_d = m.g_right_d = nullptr;
  m.g_thr_d = m.g_val_d = nullptr;
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
    if (m.pending) fs::materialize_all(fo->dev, const_cast<fs_forest*>(fo)->fams);
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
