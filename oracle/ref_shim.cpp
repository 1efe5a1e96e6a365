// TEST INFRASTRUCTURE ONLY - an extern "C" face over the unmodified reference core so pytest
// (ctypes) can run the reference's own hot path on the same inputs as the CUDA path. Built by
// oracle/Makefile into oracle/_ref/ and never linked into the product.
//
// Every function is a thin marshalling wrapper around the reference API:
//   featurize            proj/core/src/searchspace.cpp:90-118
//   train_cost_model     proj/core/src/costmodel.cpp:224-235
//   fit                  proj/core/src/costmodel.cpp:152-222
//   predict              proj/core/src/costmodel.cpp:237-246
//   pairwise_accuracy    proj/core/src/costmodel.cpp:248-277
//   dump_model           proj/core/src/costmodel.cpp:279-288
//   tune_step ranking    proj/core/src/scheduler.cpp:187-192  (std::sort of (score, index))
//   build_registry       proj/core/src/family.cpp:126-136
//   TuningEngine / foresee_tune / baseline_tune   proj/core/src/scheduler.cpp:102-305
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "famtune/costmodel.hpp"
#include "famtune/experiment.hpp"
#include "famtune/family.hpp"
#include "famtune/graph.hpp"
#include "famtune/rng.hpp"
#include "famtune/scheduler.hpp"
#include "famtune/searchspace.hpp"
#include "famtune/simbackend.hpp"

using namespace famtune;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

SpaceDescriptor space_from(int k, const int32_t* nvals, const int64_t* values) {
  SpaceDescriptor s;
  int64_t off = 0;
  for (int i = 0; i < k; ++i) {
    Knob kb;
    kb.name = "k" + std::to_string(i);
    kb.values.assign(values + off, values + off + nvals[i]);
    off += nvals[i];
    s.knobs.push_back(std::move(kb));
  }
  return s;
}

int64_t copy_string(const std::string& s, char* buf, int64_t cap) {
  if (buf && cap > 0) {
    const auto n = std::min<int64_t>(cap - 1, static_cast<int64_t>(s.size()));
    std::memcpy(buf, s.data(), static_cast<std::size_t>(n));
    buf[n] = '\0';
  }
  return static_cast<int64_t>(s.size()) + 1;
}

ClusterAlgo algo_from(int a) {
  return a == 1 ? ClusterAlgo::ByOpCount : a == 2 ? ClusterAlgo::ByOpSequence : ClusterAlgo::ByCoreOp;
}
}  // namespace

struct ref_model {
  CostModelState state;
};

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_featurize(int k, const int32_t* nvals, const int64_t* values, const int32_t* assign,
                  int64_t p, int assign_stride, int pad_dim, double* out) {
  return guarded([&] {
    const auto space = space_from(k, nvals, values);
    for (int64_t i = 0; i < p; ++i) {
      std::span<const int32_t> a(assign + i * assign_stride, static_cast<std::size_t>(k));
      const auto f = featurize(space, a, pad_dim);
      std::copy(f.begin(), f.end(), out + i * pad_dim);
    }
  });
}

int ref_featurize_checked(int k, const int32_t* nvals, const int64_t* values,
                          const int32_t* assign, int assign_len, int pad_dim, double* out) {
  return guarded([&] {
    const auto space = space_from(k, nvals, values);
    const auto f = featurize(space, std::span<const int32_t>(assign, static_cast<std::size_t>(assign_len)),
                             pad_dim);
    std::copy(f.begin(), f.end(), out);
  });
}

int ref_feature_dim(int k) { return feature_dim(k); }

int ref_linear_index(int k, const int32_t* nvals, const int64_t* values, const int32_t* assign, int64_t p,
                     int assign_stride, uint64_t* out) {
  return guarded([&] {
    const auto space = space_from(k, nvals, values);
    for (int64_t i = 0; i < p; ++i)
      out[i] = linear_index(space, std::span<const int32_t>(assign + i * assign_stride, static_cast<std::size_t>(k)));
  });
}

int ref_candidate_from_index(int k, const int32_t* nvals, const int64_t* values, const uint64_t* index, int64_t p,
                             int assign_stride, int32_t* out) {
  return guarded([&] {
    const auto space = space_from(k, nvals, values);
    for (int64_t i = 0; i < p; ++i) {
      const auto c = candidate_from_index(space, 0, index[i]);
      std::copy(c.assignment.begin(), c.assignment.end(), out + i * assign_stride);
    }
  });
}

ref_model* ref_model_new(int family_id, int trees, int depth, double lr, int min_split) {
  auto* m = new ref_model;
  GbtParams p;
  p.trees = trees;
  p.depth = depth;
  p.learning_rate = lr;
  p.min_samples_split = min_split;
  m->state = initialize_cost_model(family_id, p);
  return m;
}

void ref_model_free(ref_model* m) { delete m; }

// Appends raw (features, target) rows to training_set (the experiment-harness path).
int ref_model_add_samples(ref_model* m, int64_t n, int d, const double* x, const double* target) {
  return guarded([&] {
    for (int64_t i = 0; i < n; ++i) {
      TrainingSample s;
      s.features.assign(x + i * d, x + (i + 1) * d);
      s.target = target[i];
      m->state.training_set.push_back(std::move(s));
    }
  });
}

int ref_model_fit(ref_model* m) { return guarded([&] { fit(m->state); }); }

// train_cost_model(records, state): log(latency) targets, validation, refit.
int ref_model_train(ref_model* m, int64_t n, int d, const double* x, const double* latency_ms) {
  return guarded([&] {
    std::vector<MeasurementRecord> recs(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
      recs[i].features.assign(x + i * d, x + (i + 1) * d);
      recs[i].latency_ms = latency_ms[i];
    }
    train_cost_model(recs, m->state);
  });
}

int ref_model_num_trees(const ref_model* m) { return static_cast<int>(m->state.trees.size()); }

int ref_model_num_nodes(const ref_model* m) {
  int total = 0;
  for (const auto& t : m->state.trees) total += static_cast<int>(t.nodes.size());
  return total;
}

int ref_model_num_samples(const ref_model* m) {
  return static_cast<int>(m->state.training_set.size());
}

int ref_model_export(const ref_model* m, double* base, int32_t* offsets, int32_t* feature,
                     double* threshold, int32_t* left, int32_t* right, double* value,
                     double* mse) {
  return guarded([&] {
    *base = m->state.base_prediction;
    int32_t off = 0;
    for (std::size_t t = 0; t < m->state.trees.size(); ++t) {
      offsets[t] = off;
      for (const auto& nd : m->state.trees[t].nodes) {
        feature[off] = nd.feature;
        threshold[off] = nd.threshold;
        left[off] = nd.left;
        right[off] = nd.right;
        value[off] = nd.value;
        ++off;
      }
    }
    offsets[m->state.trees.size()] = off;
    for (std::size_t r = 0; r < m->state.train_mse_by_round.size(); ++r) mse[r] = m->state.train_mse_by_round[r];
  });
}

// Replace the ensemble with hand-built trees (costmodel_test.cpp:98-105 style).
int ref_model_import(ref_model* m, double base, int n_trees, const int32_t* offsets,
                     const int32_t* feature, const double* threshold, const int32_t* left,
                     const int32_t* right, const double* value) {
  return guarded([&] {
    m->state.base_prediction = base;
    m->state.trees.clear();
    for (int t = 0; t < n_trees; ++t) {
      RegressionTree tree;
      for (int32_t i = offsets[t]; i < offsets[t + 1]; ++i) {
        TreeNode nd;
        nd.feature = feature[i];
        nd.threshold = threshold[i];
        nd.left = left[i];
        nd.right = right[i];
        nd.value = value[i];
        tree.nodes.push_back(nd);
      }
      m->state.trees.push_back(std::move(tree));
    }
  });
}

int ref_predict(const ref_model* m, int64_t p, int d, const double* x, double* out) {
  return guarded([&] {
    for (int64_t i = 0; i < p; ++i) {
      out[i] = predict(m->state, std::span<const double>(x + i * d, static_cast<std::size_t>(d)));
    }
  });
}

int ref_pairwise_accuracy(const ref_model* m, int64_t n, int d, const double* x,
                          const double* latency_ms, double* out) {
  return guarded([&] {
    std::vector<MeasurementRecord> recs(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
      recs[i].features.assign(x + i * d, x + (i + 1) * d);
      recs[i].latency_ms = latency_ms[i];
    }
    *out = pairwise_accuracy(m->state, recs);
  });
}

int64_t ref_dump_model(const ref_model* m, char* buf, int64_t cap) {
  return copy_string(dump_model(m->state), buf, cap);
}

// The exact ordering tune_step builds before selection: std::sort over (score, pool index).
int ref_rank(int64_t p, const double* scores, int64_t* perm) {
  return guarded([&] {
    std::vector<std::pair<double, std::size_t>> scored(static_cast<std::size_t>(p));
    for (int64_t i = 0; i < p; ++i) scored[i] = {scores[i], static_cast<std::size_t>(i)};
    std::sort(scored.begin(), scored.end());
    for (int64_t i = 0; i < p; ++i) perm[i] = static_cast<int64_t>(scored[i].second);
  });
}

// ---- model files, families, simulator-generated datasets ----------------------------------

int ref_model_info(const char* path, int* n_subgraphs, int* pad_dim) {
  return guarded([&] {
    const auto model = load_model(path);
    *n_subgraphs = static_cast<int>(model.subgraphs.size());
    *pad_dim = max_feature_dim(model);
  });
}

// family_of[n_subgraphs]; returns the registry CSV through buf (two-call size query).
int64_t ref_cluster(const char* path, int algo, int32_t* family_of, char* buf, int64_t cap) {
  int64_t need = -1;
  const int rc = guarded([&] {
    const auto model = load_model(path);
    const auto reg = build_registry(algo_from(algo), model.subgraphs);
    for (int s = 0; s < reg.subgraph_count(); ++s) family_of[s] = reg.family_of(s);
    need = copy_string(reg.to_csv(), buf, cap);
  });
  return rc == 0 ? need : -rc;
}

// Subgraph knob spaces (for driving featurize with the same spaces): counts then values.
int ref_subgraph_space(const char* path, int sid, int* k, int32_t* nvals, int64_t* values) {
  return guarded([&] {
    const auto model = load_model(path);
    const auto& sg = model.subgraphs.at(static_cast<std::size_t>(sid));
    *k = static_cast<int>(sg.knob_space.knobs.size());
    int64_t off = 0;
    for (std::size_t i = 0; i < sg.knob_space.knobs.size(); ++i) {
      nvals[i] = static_cast<int32_t>(sg.knob_space.knobs[i].values.size());
      for (auto v : sg.knob_space.knobs[i].values) values[off++] = v;
    }
  });
}

// Subgraph attributes after the reference's dedup/reorder (graph.cpp:265-310): op-kind
// sequence, full serialization, core op and weight, as "seq\tfull\tcore\tweight".
int64_t ref_subgraph_info(const char* path, int sid, char* buf, int64_t cap) {
  int64_t need = -1;
  const int rc = guarded([&] {
    const auto model = load_model(path);
    const auto& sg = model.subgraphs.at(static_cast<std::size_t>(sid));
    need = copy_string(serialize_op_sequence(sg) + "\t" + serialize_ops(sg) + "\t" +
                           std::string(to_string(sg.core_op)) + "\t" + std::to_string(sg.weight),
                       buf, cap);
  });
  return rc == 0 ? need : -rc;
}

// Fresh random candidates for every member of `family`, measured by the simulator: the
// experiment-harness data path (experiment.cpp:24-43 with generate_candidates). Rows are written
// up to `cap`; *n_out is the row count; subgraph ids and assignments are returned too.
int ref_family_dataset(const char* path, int algo, int family, uint64_t seed, int per_subgraph,
                       int pad_dim, int64_t cap, double* x, double* latency, int32_t* sid_out,
                       int32_t* assign_out, int64_t* n_out) {
  return guarded([&] {
    const auto model = load_model(path);
    const auto reg = build_registry(algo_from(algo), model.subgraphs);
    const auto land = make_landscape(model, reg, seed);
    int64_t n = 0;
    for (int sid : reg.family(family).member_ids) {
      const auto& sg = model.subgraphs[static_cast<std::size_t>(sid)];
      auto rng = make_rng(seed, 0x5A, static_cast<std::uint64_t>(sid));
      MeasuredSet none;
      auto pool = generate_candidates(sg.knob_space, sid, none, per_subgraph, 0, rng);
      for (const auto& c : pool) {
        if (n >= cap) throw std::out_of_range("ref_family_dataset: capacity exceeded");
        const auto f = featurize(sg.knob_space, c.assignment, pad_dim);
        std::copy(f.begin(), f.end(), x + n * pad_dim);
        latency[n] = measure(land, sg, c, rng);
        sid_out[n] = sid;
        for (int k = 0; k < kMaxKnobs; ++k) {
          assign_out[n * kMaxKnobs + k] =
              k < static_cast<int>(c.assignment.size()) ? c.assignment[static_cast<std::size_t>(k)] : 0;
        }
        ++n;
      }
    }
    *n_out = n;
  });
}

// Run the reference tuning loop (Algorithm 1) and export (a) the curve CSV and (b) one family
// model's accumulated "purified" training set - the realistic inputs fit() sees.
int64_t ref_tune(const char* path, int algo, int foresee, int64_t budget, double p, uint64_t seed,
                 int trees, int depth, double lr, int min_split, int export_family, int64_t cap,
                 double* x, double* target, int64_t* n_out, int* d_out, char* csv, int64_t csv_cap) {
  int64_t need = -1;
  const int rc = guarded([&] {
    const auto model = load_model(path);
    const auto truth = build_registry(ClusterAlgo::ByCoreOp, model.subgraphs);
    auto land = make_landscape(model, truth, seed);
    SimBackend backend(model, std::move(land), seed);
    TuneOptions opt;
    opt.budget = budget;
    opt.foresee_p = p;
    opt.seed = seed;
    opt.cost_model.trees = trees;
    opt.cost_model.depth = depth;
    opt.cost_model.learning_rate = lr;
    opt.cost_model.min_samples_split = min_split;
    Policy pol = foresee ? make_foresee_policy(algo_from(algo)) : make_baseline_policy(algo_from(algo));
    TuningEngine engine(backend, pol, opt);
    const auto state = engine.run();
    need = copy_string(curve_to_csv(state), csv, csv_cap);
    *n_out = 0;
    *d_out = 0;
    if (export_family >= 0 && export_family < static_cast<int>(engine.models().size())) {
      const auto& ts = engine.models()[static_cast<std::size_t>(export_family)].training_set;
      int64_t n = 0;
      const int d = ts.empty() ? 0 : static_cast<int>(ts.front().features.size());
      for (const auto& s : ts) {
        if (n >= cap) break;
        std::copy(s.features.begin(), s.features.end(), x + n * d);
        target[n] = s.target;
        ++n;
      }
      *n_out = n;
      *d_out = d;
    }
  });
  return rc == 0 ? need : -rc;
}

// mt19937_64 seeded through mix_seed (rng.hpp:26-33) - lets tests pin the host RNG replay.
uint64_t ref_rng_draws(uint64_t seed, uint64_t a, uint64_t b, int n, uint64_t bound, uint64_t* out) {
  auto rng = make_rng(seed, a, b);
  for (int i = 0; i < n; ++i) out[i] = bound ? uniform_below(rng, bound) : rng();
  return static_cast<uint64_t>(n);
}

}  // extern "C"
