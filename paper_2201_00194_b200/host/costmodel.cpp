// famtune cost-model API (include/famtune/costmodel.hpp, searchspace.hpp) implemented over the C
// ABI of libfamseer.so. Every numeric operation of the hot path - featurize, predict/eval, fit,
// ranking, pairwise accuracy - runs on the B200; this file only validates arguments with the
// reference's messages (costmodel.cpp:175-183, 224-231, 238-240, 248-277; searchspace.cpp:94-100),
// packs std::vector-based states into flat buffers and maps status codes back to the reference's
// exception types. There is no CPU fallback: if the device or the library is missing, calls throw.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <list>
#include <mutex>
#include <sstream>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "famseer.h"
#include "famtune/costmodel.hpp"

namespace famtune {
namespace {

std::recursive_mutex g_mu;

[[noreturn]] void raise(int rc) {
  const std::string msg = fs_last_error();
  switch (rc) {
    case FS_EINVAL:
      throw std::invalid_argument(msg);
    case FS_EDOMAIN:
      throw std::domain_error(msg);
    case FS_ERANGE:
      throw std::out_of_range(msg);
    default:
      throw std::runtime_error("famseer: " + msg);
  }
}

inline void ck(int rc) {
  if (rc != FS_OK) raise(rc);
}

std::uint64_t fnv(const void* data, std::size_t n, std::uint64_t h = 14695981039346656037ULL) {
  const auto* p = static_cast<const unsigned char*>(data);
  for (std::size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 1099511628211ULL;
  }
  return h;
}

std::uint64_t model_digest(const CostModelState& m) {
  std::uint64_t h = fnv(&m.base_prediction, sizeof(double));
  h = fnv(&m.params.learning_rate, sizeof(double), h);
  const std::size_t t = m.trees.size();
  h = fnv(&t, sizeof t, h);
  for (const auto& tree : m.trees) {
    const std::size_t k = tree.nodes.size();
    h = fnv(&k, sizeof k, h);
    for (const auto& nd : tree.nodes) {
      h = fnv(&nd.feature, sizeof nd.feature, h);
      h = fnv(&nd.threshold, sizeof nd.threshold, h);
      h = fnv(&nd.left, sizeof nd.left, h);
      h = fnv(&nd.right, sizeof nd.right, h);
      h = fnv(&nd.value, sizeof nd.value, h);
    }
  }
  return h;
}

struct Flat {
  std::vector<int32_t> off{0}, feat, left, right;
  std::vector<double> thr, val;
};

Flat flatten(const std::vector<RegressionTree>& trees) {
  Flat f;
  for (const auto& t : trees) {
    for (const auto& nd : t.nodes) {
      f.feat.push_back(nd.feature);
      f.thr.push_back(nd.threshold);
      f.left.push_back(nd.left);
      f.right.push_back(nd.right);
      f.val.push_back(nd.value);
    }
    f.off.push_back(static_cast<int32_t>(f.feat.size()));
  }
  return f;
}

bool same_bits(double a, double b) { return std::memcmp(&a, &b, sizeof(double)) == 0; }

struct Runtime {
  fs_device* dev = nullptr;
  // Compiled device copies of the models predict()/eval() have seen, keyed by a content digest.
  // A digest hit is confirmed against the full model content (a 64-bit collision must never
  // predict with another model); least recently used entries are evicted beyond kCacheCap.
  static constexpr std::size_t kCacheCap = 512;
  struct Entry {
    fs_forest* forest = nullptr;
    double base = 0.0, lr = 0.0;
    Flat flat;  // the uploaded trees, for the exact comparison on a digest hit
    std::vector<double> gains;  // from the fit that produced this model, if any
    std::list<std::uint64_t>::iterator lru;
  };
  std::unordered_map<std::uint64_t, Entry> models;  // digest -> compiled model
  std::list<std::uint64_t> lru;                      // most recently used first
  std::unordered_map<std::uint64_t, fs_spaces*> spaces;

  Runtime() { ck(fs_device_create(gpu::device_ordinal(), &dev)); }
  ~Runtime() {
    for (auto& kv : models) fs_forest_destroy(kv.second.forest);
    for (auto& kv : spaces) fs_spaces_destroy(kv.second);
    fs_device_destroy(dev);
  }

  static bool same_model(const Entry& e, const CostModelState& m) {
    if (!same_bits(e.base, m.base_prediction) || !same_bits(e.lr, m.params.learning_rate)) return false;
    if (e.flat.off.size() != m.trees.size() + 1) return false;
    std::size_t i = 0;
    for (std::size_t t = 0; t < m.trees.size(); ++t) {
      const auto& nodes = m.trees[t].nodes;
      if (static_cast<std::size_t>(e.flat.off[t + 1] - e.flat.off[t]) != nodes.size()) return false;
      for (const auto& nd : nodes) {
        if (e.flat.feat[i] != nd.feature || e.flat.left[i] != nd.left || e.flat.right[i] != nd.right ||
            !same_bits(e.flat.thr[i], nd.threshold) || !same_bits(e.flat.val[i], nd.value))
          return false;
        ++i;
      }
    }
    return true;
  }

  // Compiled device copy of `m`, uploaded on first use (keyed by content).
  fs_forest* forest_for(const CostModelState& m) {
    const std::uint64_t dg = model_digest(m);
    auto it = models.find(dg);
    if (it != models.end()) {
      lru.splice(lru.begin(), lru, it->second.lru);
      if (same_model(it->second, m)) return it->second.forest;
      upload(it->second, m);  // digest collision: the slot now holds this model
      return it->second.forest;
    }
    while (models.size() >= kCacheCap) {  // evict the least recently used model
      const std::uint64_t victim = lru.back();
      lru.pop_back();
      fs_forest_destroy(models[victim].forest);
      models.erase(victim);
    }
    Entry e;
    ck(fs_forest_create(dev, 1, &e.forest));
    try {
      upload(e, m);
    } catch (...) {
      fs_forest_destroy(e.forest);
      throw;
    }
    lru.push_front(dg);
    e.lru = lru.begin();
    return (models[dg] = std::move(e)).forest;
  }

  // the cache entry holding exactly `m`, or nullptr
  Entry* find(const CostModelState& m) {
    auto it = models.find(model_digest(m));
    return it != models.end() && same_model(it->second, m) ? &it->second : nullptr;
  }

  void upload(Entry& e, const CostModelState& m) {
    e.gains.clear();
    e.flat = flatten(m.trees);
    e.base = m.base_prediction;
    e.lr = m.params.learning_rate;
    ck(fs_forest_upload(e.forest, 0, m.base_prediction, m.params.learning_rate, static_cast<int32_t>(m.trees.size()),
                        e.flat.off.data(), e.flat.feat.data(), e.flat.thr.data(), e.flat.left.data(),
                        e.flat.right.data(), e.flat.val.data()));
  }

  fs_spaces* spaces_for(const SpaceDescriptor& space) {
    std::vector<int32_t> nk{static_cast<int32_t>(space.knobs.size())};
    std::vector<int32_t> nv(kMaxKnobs, 0);
    std::vector<int64_t> vals;
    if (space.knobs.size() > static_cast<std::size_t>(kMaxKnobs) || space.knobs.empty())
      throw std::invalid_argument("knob space: knob count must be in [1, 16], got " + std::to_string(space.knobs.size()));
    for (std::size_t k = 0; k < space.knobs.size(); ++k) {
      nv[k] = static_cast<int32_t>(space.knobs[k].values.size());
      vals.insert(vals.end(), space.knobs[k].values.begin(), space.knobs[k].values.end());
    }
    std::uint64_t dg = fnv(nv.data(), nv.size() * sizeof(int32_t));
    dg = fnv(vals.data(), vals.size() * sizeof(int64_t), dg);
    auto it = spaces.find(dg);
    if (it != spaces.end()) return it->second;
    fs_spaces* sp = nullptr;
    ck(fs_spaces_create(dev, 1, nk.data(), nv.data(), vals.empty() ? nullptr : vals.data(), &sp));
    spaces[dg] = sp;
    return sp;
  }
};

Runtime& rt() {
  static Runtime r;
  return r;
}

void export_into(fs_forest* fo, int family, CostModelState& m, std::vector<double>* gains) {
  double base = 0.0;
  int32_t nt = 0, nn = 0;
  ck(fs_forest_export(fo, family, &base, &nt, &nn, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                      nullptr));
  std::vector<int32_t> off(static_cast<std::size_t>(nt) + 1), feat(static_cast<std::size_t>(nn)),
      left(static_cast<std::size_t>(nn)), right(static_cast<std::size_t>(nn));
  std::vector<double> thr(static_cast<std::size_t>(nn)), val(static_cast<std::size_t>(nn)),
      gain(static_cast<std::size_t>(nn)), mse(static_cast<std::size_t>(nt));
  ck(fs_forest_export(fo, family, &base, nullptr, nullptr, off.data(), feat.data(), thr.data(), left.data(),
                      right.data(), val.data(), gain.data(), mse.data()));
  m.base_prediction = base;
  m.trees.assign(static_cast<std::size_t>(nt), RegressionTree{});
  for (int t = 0; t < nt; ++t) {
    auto& nodes = m.trees[static_cast<std::size_t>(t)].nodes;
    for (int32_t i = off[static_cast<std::size_t>(t)]; i < off[static_cast<std::size_t>(t) + 1]; ++i)
      nodes.push_back({feat[static_cast<std::size_t>(i)], thr[static_cast<std::size_t>(i)],
                       left[static_cast<std::size_t>(i)], right[static_cast<std::size_t>(i)],
                       val[static_cast<std::size_t>(i)]});
  }
  m.train_mse_by_round = std::move(mse);
  if (gains) *gains = std::move(gain);
}

fs_gbt_params to_params(const GbtParams& p) {
  return fs_gbt_params{p.trees, p.depth, p.learning_rate, p.min_samples_split};
}

// Pack one model's training set; reference check order (costmodel.cpp:175-183).
int pack(const CostModelState& m, std::vector<double>& x, std::vector<double>& y) {
  const int d = static_cast<int>(m.training_set.front().features.size());
  for (const auto& s : m.training_set)
    if (static_cast<int>(s.features.size()) != d)
      throw std::invalid_argument("cost model: inconsistent feature dimensions in training set");
  for (const auto& s : m.training_set) {
    x.insert(x.end(), s.features.begin(), s.features.end());
    y.push_back(s.target);
  }
  return d;
}

void fit_group(std::vector<CostModelState*>& group) {
  Runtime& r = rt();
  std::vector<double> x, y;
  std::vector<int64_t> seg{0};
  std::vector<fs_gbt_params> params;
  int d = -1;
  for (auto* m : group) {
    d = pack(*m, x, y);
    seg.push_back(static_cast<int64_t>(y.size()));
    params.push_back(to_params(m->params));
  }
  fs_forest* fo = nullptr;
  ck(fs_forest_create(r.dev, static_cast<int32_t>(group.size()), &fo));
  const int rc = fs_fit(r.dev, fo, static_cast<int32_t>(group.size()), seg.data(), d, x.data(), y.data(),
                        params.data());
  if (rc != FS_OK) {
    fs_forest_destroy(fo);
    raise(rc);
  }
  for (std::size_t g = 0; g < group.size(); ++g) {
    std::vector<double> gains;
    export_into(fo, static_cast<int>(g), *group[g], &gains);
    // keep the compiled model for predict: re-upload into a 1-family forest keyed by content
    r.forest_for(*group[g]);
    if (auto* e = r.find(*group[g])) e->gains = std::move(gains);
  }
  fs_forest_destroy(fo);
}

}  // namespace

// ---- searchspace ------------------------------------------------------------------------
int feature_dim(int k) { return fs_feature_dim(k); }

std::uint64_t linear_index(const SpaceDescriptor& space, std::span<const std::int32_t> assignment) {
  std::uint64_t idx = 0;  // mixed radix, most significant knob first (searchspace.cpp:48-54)
  for (std::size_t k = 0; k < space.knobs.size(); ++k)
    idx = idx * space.knobs[k].values.size() + static_cast<std::uint64_t>(assignment[k]);
  return idx;
}

Candidate candidate_from_index(const SpaceDescriptor& space, int subgraph_id, std::uint64_t index) {
  Candidate c;
  c.subgraph_id = subgraph_id;
  c.assignment.resize(space.knobs.size());
  for (std::size_t k = space.knobs.size(); k-- > 0;) {
    const std::uint64_t m = space.knobs[k].values.size();
    c.assignment[k] = static_cast<std::int32_t>(index % m);
    index /= m;
  }
  return c;
}

std::vector<double> featurize(const SpaceDescriptor& space, std::span<const std::int32_t> assignment, int pad_dim) {
  const int k = static_cast<int>(space.knobs.size());
  if (assignment.size() != static_cast<std::size_t>(k))
    throw std::invalid_argument("featurize: assignment length does not match knob count");
  const int d = feature_dim(k);
  if (pad_dim < d)
    throw std::invalid_argument("featurize: pad_dim " + std::to_string(pad_dim) + " smaller than feature dim " +
                                std::to_string(d));
  return gpu::featurize_batch(space, assignment, pad_dim);
}

namespace gpu {

int device_ordinal() {
  const char* e = std::getenv("FAMSEER_DEVICE");
  return e ? std::atoi(e) : 0;
}

std::vector<double> featurize_batch(const SpaceDescriptor& space, std::span<const std::int32_t> assignments,
                                    int pad_dim) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  const int k = static_cast<int>(space.knobs.size());
  if (k < 1 || assignments.size() % static_cast<std::size_t>(k) != 0)
    throw std::invalid_argument("featurize: assignment length does not match knob count");
  const int64_t n = static_cast<int64_t>(assignments.size()) / k;
  std::vector<int32_t> so(static_cast<std::size_t>(n), 0), asg(static_cast<std::size_t>(n) * kMaxKnobs, 0);
  for (int64_t i = 0; i < n; ++i)
    for (int j = 0; j < k; ++j)
      asg[static_cast<std::size_t>(i * kMaxKnobs + j)] = assignments[static_cast<std::size_t>(i * k + j)];
  std::vector<double> out(static_cast<std::size_t>(n) * pad_dim);
  Runtime& r = rt();
  ck(fs_featurize(r.dev, r.spaces_for(space), n, so.data(), asg.data(), pad_dim, out.data()));
  return out;
}

void fit_many(std::span<CostModelState* const> models) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  std::unordered_map<int, std::vector<CostModelState*>> by_dim;  // one device pass per row width
  for (CostModelState* m : models) {
    m->trees.clear();
    m->train_mse_by_round.clear();
    if (m->training_set.empty()) {
      m->base_prediction = 0.0;  // costmodel.cpp:156-159
      continue;
    }
    by_dim[static_cast<int>(m->training_set.front().features.size())].push_back(m);
  }
  for (auto& kv : by_dim) fit_group(kv.second);
}

std::vector<double> predict_batch(const CostModelState& model, std::span<const double> rows, int d) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  if (d < 0 || (d == 0 && !rows.empty()) || (d > 0 && rows.size() % static_cast<std::size_t>(d)))
    throw std::invalid_argument("predict: row width mismatch");
  const int64_t n = d ? static_cast<int64_t>(rows.size()) / d : 0;
  std::vector<double> out(static_cast<std::size_t>(n));
  if (!n) return out;
  Runtime& r = rt();
  const int64_t seg[2] = {0, n};
  ck(fs_predict(r.dev, r.forest_for(model), 1, seg, d, rows.data(), out.data(), nullptr));
  return out;
}

std::vector<std::int32_t> rank(std::span<const double> scores) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  std::vector<std::int32_t> perm(scores.size());
  if (scores.empty()) return perm;
  const int64_t seg[2] = {0, static_cast<int64_t>(scores.size())};
  ck(fs_rank(rt().dev, 1, seg, scores.data(), perm.data()));
  return perm;
}

std::vector<double> split_gains(const CostModelState& model) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  const auto* e = rt().find(model);
  if (!e) return {};
  return e->gains;
}

}  // namespace gpu

// ---- cost model ---------------------------------------------------------------------------
CostModelState initialize_cost_model(int family_id, GbtParams params) {
  CostModelState m;
  m.family_id = family_id;
  m.params = params;
  return m;
}

void fit(CostModelState& model) {
  CostModelState* one[1] = {&model};
  gpu::fit_many(one);
}

void train_cost_model(std::span<const MeasurementRecord> records, CostModelState& model) {
  if (records.empty()) throw std::invalid_argument("train_cost_model: empty record batch");
  for (const auto& rec : records) {  // records before a bad one stay appended, as in the reference
    if (!(rec.latency_ms > 0.0)) throw std::invalid_argument("train_cost_model: non-positive latency");
    model.training_set.push_back({rec.features, std::log(rec.latency_ms)});
  }
  fit(model);
}

double predict(const CostModelState& model, std::span<const double> features) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  double out = 0.0;
  Runtime& r = rt();
  const int64_t seg[2] = {0, 1};
  ck(fs_predict(r.dev, r.forest_for(model), 1, seg, static_cast<int32_t>(features.size()), features.data(), &out,
                nullptr));
  return out;
}

double RegressionTree::eval(std::span<const double> features) const {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  CostModelState one;
  one.trees.push_back(*this);
  Runtime& r = rt();
  double score = 0.0;
  uint16_t leaf = 0;
  const int64_t seg[2] = {0, 1};
  if (nodes.size() > 65536) {  // leaf ids are uint16; larger trees: the value through lr = 1, base 0
    one.params.learning_rate = 1.0;
    ck(fs_predict(r.dev, r.forest_for(one), 1, seg, static_cast<int32_t>(features.size()), features.data(), &score,
                  nullptr));
    return score;
  }
  ck(fs_predict(r.dev, r.forest_for(one), 1, seg, static_cast<int32_t>(features.size()), features.data(), &score,
                &leaf));
  return nodes[leaf].value;
}

double pairwise_accuracy(const CostModelState& model, std::span<const MeasurementRecord> validation) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  if (validation.size() < 2)
    throw std::invalid_argument("pairwise_accuracy: need at least two validation records");
  const int d = static_cast<int>(validation.front().features.size());
  std::vector<double> x, lat;
  for (const auto& v : validation) {
    if (static_cast<int>(v.features.size()) != d)
      throw std::invalid_argument("pairwise_accuracy: inconsistent feature dimensions");
    x.insert(x.end(), v.features.begin(), v.features.end());
    lat.push_back(v.latency_ms);
  }
  const std::vector<double> scores = gpu::predict_batch(model, x, d);
  double acc = 0.0;
  ck(fs_pairwise_accuracy(rt().dev, static_cast<int64_t>(scores.size()), scores.data(), lat.data(), &acc));
  return acc;
}

std::string dump_model(const CostModelState& model) {
  std::ostringstream out;
  out << "cost model family=" << model.family_id << " trees=" << model.trees.size()
      << " base=" << model.base_prediction << " lr=" << model.params.learning_rate << '\n';
  for (std::size_t t = 0; t < model.trees.size(); ++t) {
    out << "tree " << t << ":\n";
    const auto& nodes = model.trees[t].nodes;
    struct Frame {
      int idx, indent;
    };
    std::vector<Frame> stack{{0, 1}};
    while (!stack.empty()) {  // pre-order, left before right
      const Frame fr = stack.back();
      stack.pop_back();
      const auto& nd = nodes[static_cast<std::size_t>(fr.idx)];
      out << std::string(static_cast<std::size_t>(fr.indent) * 2, ' ');
      if (nd.is_leaf()) {
        out << "leaf value=" << nd.value << '\n';
        continue;
      }
      out << "x[" << nd.feature << "] <= " << nd.threshold << '\n';
      stack.push_back({nd.right, fr.indent + 1});
      stack.push_back({nd.left, fr.indent + 1});
    }
  }
  return out.str();
}

}  // namespace famtune
