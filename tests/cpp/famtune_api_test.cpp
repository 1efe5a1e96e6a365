// The reference's cost-model / featurize test expectations (costmodel_test.cpp,
// searchspace_test.cpp, acceptance C7) re-run against the DROP-IN C++ API
// (include/famtune/*.hpp -> libfamtune_b200.so -> B200). A caller written against the reference
// headers sees the same values and the same exception types. gtest is not installed, so this is
// a minimal self-registering harness; pytest runs the binary (tests/test_cpp_api.py).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "famtune/costmodel.hpp"
#include "famtune/searchspace.hpp"

using namespace famtune;

namespace {

struct Case {
  const char* name;
  std::function<void()> fn;
};
std::vector<Case>& cases() {
  static std::vector<Case> c;
  return c;
}
int g_fail = 0;
const char* g_cur = "";

struct Reg {
  Reg(const char* n, std::function<void()> f) { cases().push_back({n, std::move(f)}); }
};
#define CASE(name)                         \
  static void name();                      \
  static Reg reg_##name(#name, name);      \
  static void name()
#define CHECK(cond)                                                                 \
  do {                                                                              \
    if (!(cond)) {                                                                  \
      ++g_fail;                                                                     \
      std::printf("  FAIL %s:%d [%s] %s\n", __FILE__, __LINE__, g_cur, #cond);       \
    }                                                                               \
  } while (0)
#define CHECK_THROWS(expr, T)                 \
  do {                                        \
    bool caught = false;                      \
    try {                                     \
      (void)(expr);                           \
    } catch (const T&) {                      \
      caught = true;                          \
    } catch (...) {                           \
    }                                         \
    CHECK(caught && #T);                      \
  } while (0)

MeasurementRecord rec(std::vector<double> f, double lat) {
  MeasurementRecord r;
  r.features = std::move(f);
  r.latency_ms = lat;
  return r;
}

SpaceDescriptor space(std::vector<std::vector<std::int64_t>> v) {
  SpaceDescriptor s;
  for (std::size_t i = 0; i < v.size(); ++i) s.knobs.push_back({"k" + std::to_string(i), v[i]});
  return s;
}

// Noise-free samples of one 3-knob space from a quadratic bowl (the landscape shape of
// simbackend.cpp:80-102); exact latencies, so their order is the ground-truth order.
std::vector<MeasurementRecord> bowl_samples(int count, unsigned seed) {
  const auto sp = space({{1, 2, 4, 8, 16, 32, 64, 128}, {1, 2, 4, 8, 16, 32, 64, 128}, {1, 2, 4, 8, 16, 32}});
  std::mt19937_64 rng(seed);
  std::vector<std::uint64_t> idx(8 * 8 * 6);
  std::iota(idx.begin(), idx.end(), 0);
  std::shuffle(idx.begin(), idx.end(), rng);
  std::vector<MeasurementRecord> out;
  for (int i = 0; i < count; ++i) {
    const auto c = candidate_from_index(sp, 0, idx[static_cast<std::size_t>(i)]);
    double q = 0.0;
    const double opt[3] = {0.4, 0.3, 0.6};
    for (int k = 0; k < 3; ++k) {
      const double z = c.assignment[static_cast<std::size_t>(k)] / double(sp.knobs[static_cast<std::size_t>(k)].values.size() - 1);
      q += 1.3 * (z - opt[k]) * (z - opt[k]);
    }
    MeasurementRecord r;
    r.candidate = c;
    r.features = featurize(sp, c.assignment, feature_dim(3));
    r.latency_ms = 0.8 * (1.0 + q);
    out.push_back(std::move(r));
  }
  return out;
}

double spearman(const std::vector<double>& a, const std::vector<double>& b) {
  auto ranks = [](const std::vector<double>& v) {
    std::vector<std::size_t> o(v.size());
    std::iota(o.begin(), o.end(), 0);
    std::sort(o.begin(), o.end(), [&](std::size_t x, std::size_t y) { return v[x] < v[y]; });
    std::vector<double> r(v.size());
    for (std::size_t i = 0; i < o.size(); ++i) r[o[i]] = double(i);
    return r;
  };
  const auto ra = ranks(a), rb = ranks(b);
  const double m = (double(a.size()) - 1) / 2;
  double num = 0, da = 0, db = 0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    num += (ra[i] - m) * (rb[i] - m);
    da += (ra[i] - m) * (ra[i] - m);
    db += (rb[i] - m) * (rb[i] - m);
  }
  return num / std::sqrt(da * db);
}

}  // namespace

CASE(fresh_model_predicts_zero) {  // costmodel_test.cpp:77-83
  const auto m = initialize_cost_model(0);
  CHECK(predict(m, std::vector<double>{1, 2, 3}) == 0.0);
  CHECK(predict(m, std::vector<double>{9, -4, 0.5}) == 0.0);
}

CASE(independent_states_per_family) {  // :85-96
  auto a = initialize_cost_model(0), b = initialize_cost_model(1), mono = initialize_cost_model(kMonolithicModel);
  CHECK(a.family_id == 0 && b.family_id == 1 && mono.family_id == kMonolithicModel);
  train_cost_model(std::vector<MeasurementRecord>{rec({1.0}, 2.0), rec({2.0}, 1.0)}, a);
  CHECK(a.trained() && !b.trained());
}

CASE(single_leaf_arithmetic) {  // :98-105
  auto m = initialize_cost_model(0);
  RegressionTree t;
  t.nodes.push_back({-1, 0.0, -1, -1, 7.0});
  m.trees.push_back(t);
  CHECK(predict(m, std::vector<double>{1.0}) == 0.1 * 7.0);
  CHECK(t.eval(std::vector<double>{1.0}) == 7.0);
}

CASE(rejects_non_finite) {  // :107-111
  const auto m = initialize_cost_model(0);
  CHECK_THROWS(predict(m, std::vector<double>{std::numeric_limits<double>::quiet_NaN()}), std::invalid_argument);
}

CASE(two_point_ranking) {  // :113-119
  auto m = initialize_cost_model(0);
  const std::vector<MeasurementRecord> r = {rec({0.0, 1.0}, 1.0), rec({3.0, 2.0}, 2.0)};
  train_cost_model(r, m);
  CHECK(predict(m, r[0].features) < predict(m, r[1].features));
}

CASE(retrain_identical_and_permutation_invariant) {  // :121-145
  auto recs = bowl_samples(128, 21);
  auto a = initialize_cost_model(0), b = initialize_cost_model(0);
  train_cost_model(recs, a);
  std::mt19937_64 rng(22);
  std::shuffle(recs.begin(), recs.end(), rng);
  train_cost_model(recs, b);
  for (const auto& r : recs) CHECK(predict(a, r.features) == predict(b, r.features));
  CHECK(a.trees.size() == b.trees.size());
}

CASE(degenerate_targets_constant_model) {  // :147-158
  auto m = initialize_cost_model(0);
  std::vector<MeasurementRecord> r;
  for (int i = 0; i < 8; ++i) r.push_back(rec({double(i)}, 2.5));
  train_cost_model(r, m);
  const double p1 = predict(m, std::vector<double>{-3.0}), p2 = predict(m, std::vector<double>{42.0});
  CHECK(p1 == p2);
  CHECK(std::abs(p1 - std::log(2.5)) < 1e-12);
}

CASE(in_sample_accuracy) {  // :160-165
  const auto r = bowl_samples(256, 31);
  auto m = initialize_cost_model(0);
  train_cost_model(r, m);
  CHECK(pairwise_accuracy(m, r) >= 0.95);
}

CASE(held_out_spearman) {  // :167-183
  auto r = bowl_samples(256, 41);
  const std::vector<MeasurementRecord> train(r.begin(), r.begin() + 200), held(r.begin() + 200, r.end());
  auto m = initialize_cost_model(0);
  train_cost_model(train, m);
  std::vector<double> p, a;
  for (const auto& h : held) {
    p.push_back(predict(m, h.features));
    a.push_back(h.latency_ms);
  }
  CHECK(spearman(p, a) > 0.8);
}

CASE(mse_non_increasing) {  // :185-202, acceptance C7
  std::mt19937_64 rng(51);
  std::uniform_real_distribution<double> u(0, 1);
  std::normal_distribution<double> nrm(0, 0.3);
  for (int ds = 0; ds < 10; ++ds) {
    auto m = initialize_cost_model(0);
    const int n = 32 + int(rng() % 200);
    for (int i = 0; i < n; ++i) {
      std::vector<double> x = {u(rng) * 8, u(rng) * 8, u(rng)};
      m.training_set.push_back({x, x[0] * 0.5 - x[1] * x[2] + nrm(rng)});
    }
    fit(m);
    CHECK(!m.train_mse_by_round.empty());
    for (std::size_t k = 1; k < m.train_mse_by_round.size(); ++k)
      CHECK(m.train_mse_by_round[k] <= m.train_mse_by_round[k - 1] + 1e-12);
  }
}

CASE(input_validation) {  // :204-209
  auto m = initialize_cost_model(0);
  CHECK_THROWS(train_cost_model(std::span<const MeasurementRecord>{}, m), std::invalid_argument);
  CHECK_THROWS(train_cost_model(std::vector<MeasurementRecord>{rec({1.0}, 0.0)}, m), std::invalid_argument);
  auto bad = initialize_cost_model(0);
  bad.training_set.push_back({{1.0, 2.0}, 0.0});
  bad.training_set.push_back({{1.0}, 0.0});
  CHECK_THROWS(fit(bad), std::invalid_argument);
}

CASE(pairwise_conventions) {  // :211-238
  auto perfect = initialize_cost_model(0);
  std::vector<MeasurementRecord> r;
  for (int i = 0; i < 8; ++i) r.push_back(rec({double(i)}, 1.0 + i));
  train_cost_model(r, perfect);
  CHECK(pairwise_accuracy(perfect, r) == 1.0);
  const auto constant = initialize_cost_model(0);
  std::vector<MeasurementRecord> four;
  for (int i = 0; i < 4; ++i) four.push_back(rec({double(i)}, 1.0 + i));
  CHECK(pairwise_accuracy(constant, four) == 0.5);
  std::vector<MeasurementRecord> same;
  for (int i = 0; i < 4; ++i) same.push_back(rec({double(i)}, 3.0));
  CHECK_THROWS(pairwise_accuracy(constant, same), std::domain_error);
  CHECK_THROWS(pairwise_accuracy(constant, std::span<const MeasurementRecord>{}), std::invalid_argument);
}

CASE(dump_lists_trees) {  // :295-304
  auto m = initialize_cost_model(3);
  train_cost_model(std::vector<MeasurementRecord>{rec({0.0}, 1.0), rec({1.0}, 2.0), rec({2.0}, 4.0), rec({3.0}, 8.0)},
                   m);
  const auto d = dump_model(m);
  CHECK(d.find("family=3") != std::string::npos);
  CHECK(d.find("tree 0:") != std::string::npos);
  CHECK(d.find("leaf value=") != std::string::npos);
}

CASE(featurize_layouts) {  // searchspace_test.cpp:59-100
  const auto f = featurize(space({{8, 16, 32}}), std::vector<std::int32_t>{0}, 6);
  CHECK(f.size() == 6 && f[0] == 3.0 && f[1] == 0.0);
  for (int i = 2; i < 6; ++i) CHECK(f[static_cast<std::size_t>(i)] == 0.0);
  const auto g = featurize(space({{4, 8}, {2, 16}}), std::vector<std::int32_t>{0, 0}, feature_dim(2));
  CHECK(g.size() == 5 && g[0] == 2.0 && g[1] == 1.0 && g[4] == 2.0);
  const auto sp = space({{1, 2, 4}, {1, 2, 4, 8}});
  CHECK(featurize(sp, std::vector<std::int32_t>{2, 1}, 8) == featurize(sp, std::vector<std::int32_t>{2, 1}, 8));
  const auto s2 = space({{1, 2}, {1, 2}});
  CHECK_THROWS(featurize(s2, std::vector<std::int32_t>{0}, 8), std::invalid_argument);
  CHECK_THROWS(featurize(s2, std::vector<std::int32_t>{0, 0}, feature_dim(2) - 1), std::invalid_argument);
  const auto s3 = space({{1, 2, 4, 8}, {1, 3, 9}, {2, 4}});
  std::vector<std::vector<double>> seen;
  for (std::uint64_t i = 0; i < 24; ++i) {
    const auto c = candidate_from_index(s3, 0, i);
    CHECK(linear_index(s3, c.assignment) == i);
    seen.push_back(featurize(s3, c.assignment, feature_dim(3)));
  }
  std::sort(seen.begin(), seen.end());
  CHECK(std::adjacent_find(seen.begin(), seen.end()) == seen.end());
}

CASE(batched_entry_points) {
  auto r1 = bowl_samples(150, 5), r2 = bowl_samples(90, 6);
  auto a = initialize_cost_model(0), b = initialize_cost_model(1);
  for (const auto& r : r1) a.training_set.push_back({r.features, std::log(r.latency_ms)});
  for (const auto& r : r2) b.training_set.push_back({r.features, std::log(r.latency_ms)});
  auto a1 = a, b1 = b;
  CostModelState* both[2] = {&a, &b};
  gpu::fit_many(both);
  fit(a1);
  fit(b1);
  CHECK(a.trees.size() == a1.trees.size() && b.trees.size() == b1.trees.size());
  std::vector<double> rows;
  for (const auto& r : r1) rows.insert(rows.end(), r.features.begin(), r.features.end());
  const auto s = gpu::predict_batch(a, rows, feature_dim(3));
  for (std::size_t i = 0; i < r1.size(); ++i) CHECK(s[i] == predict(a1, r1[i].features));
  const auto perm = gpu::rank(s);
  std::vector<std::pair<double, std::size_t>> ref(s.size());
  for (std::size_t i = 0; i < s.size(); ++i) ref[i] = {s[i], i};
  std::sort(ref.begin(), ref.end());
  for (std::size_t i = 0; i < s.size(); ++i) CHECK(perm[i] == static_cast<std::int32_t>(ref[i].second));
  CHECK(!gpu::split_gains(a).empty());
}

int main() {
  for (const auto& c : cases()) {
    g_cur = c.name;
    const int before = g_fail;
    try {
      c.fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("  FAIL [%s] unexpected exception: %s\n", c.name, e.what());
    }
    std::printf("%s %s\n", g_fail == before ? "PASS" : "FAIL", c.name);
  }
  std::printf("%zu cases, %d failed checks\n", cases().size(), g_fail);
  return g_fail ? 1 : 0;
}
