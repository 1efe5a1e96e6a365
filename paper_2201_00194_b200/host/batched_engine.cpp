// famtune::gpu::BatchedTuningEngine (include/famtune/batched_engine.hpp): the reference's tuning
// loop with the per-candidate scoring block and the per-batch retrain replaced by batched device
// calls. Control flow restates scheduler.cpp line by line (cited per function) so the curve is
// byte-identical; the hot blocks go through the C ABI (include/famseer.h).
#include "famtune/batched_engine.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <numeric>
#include <stdexcept>
#include <string>

namespace famtune {
namespace gpu {
namespace {

constexpr std::uint64_t kGenStream = 0xD4;  // candidate-generation stream tag (scheduler.cpp:12)

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

int device_ordinal() {
  const char* e = std::getenv("FAMSEER_DEVICE");
  return e ? std::atoi(e) : 0;
}

// descriptors of a candidate list: space id = subgraph id, value indices padded to 16
void pack(std::span<const Candidate> cands, std::vector<std::int32_t>& space_of, std::vector<std::int32_t>& assign) {
  space_of.assign(cands.size(), 0);
  assign.assign(cands.size() * FS_MAX_KNOBS, 0);
  for (std::size_t i = 0; i < cands.size(); ++i) {
    space_of[i] = cands[i].subgraph_id;
    std::copy(cands[i].assignment.begin(), cands[i].assignment.end(), assign.begin() + i * FS_MAX_KNOBS);
  }
}

}  // namespace

// TuningEngine::TuningEngine (scheduler.cpp:102-136), plus the device-side model store.
BatchedTuningEngine::BatchedTuningEngine(SimBackend& backend, Policy policy, TuneOptions options)
    : backend_(backend),
      model_(backend.model()),
      policy_(policy),
      options_(options),
      registry_(build_registry(policy.cluster_algo, model_.subgraphs)) {
  if (!(options_.foresee_p > 0.0 && options_.foresee_p < 1.0)) {
    throw std::invalid_argument("foresee proportion must satisfy 0 < p < 1");
  }
  const auto n = static_cast<std::int64_t>(model_.subgraphs.size());
  if (options_.budget < n) {
    throw std::invalid_argument("budget " + std::to_string(options_.budget) + " smaller than subgraph count " +
                                std::to_string(n));
  }
  if (options_.pool_random + options_.pool_evolved < 1) {
    throw std::invalid_argument("candidate pool must be non-empty");
  }
  if (!(options_.epsilon_explore >= 0.0 && options_.epsilon_explore < 1.0)) {
    throw std::invalid_argument("epsilon share must be in [0, 1)");
  }
  if (policy_.granularity == ModelGranularity::Monolithic) {
    models_.push_back(initialize_cost_model(kMonolithicModel, options_.cost_model));
  } else {
    models_.reserve(static_cast<std::size_t>(registry_.family_count()));
    for (int fam = 0; fam < registry_.family_count(); ++fam) {
      models_.push_back(initialize_cost_model(fam, options_.cost_model));
    }
  }
  gen_streams_.reserve(model_.subgraphs.size());
  for (std::size_t sid = 0; sid < model_.subgraphs.size(); ++sid) {
    gen_streams_.push_back(make_rng(options_.seed, kGenStream, sid));
  }

  // device: every subgraph's knob space, an (empty) model and an empty training set per slot
  const int S = static_cast<int>(models_.size());
  ck(fs_device_create(device_ordinal(), &dev_));
  std::vector<std::int32_t> nk, nv;
  std::vector<std::int64_t> vals;
  for (const auto& sg : model_.subgraphs) {
    nk.push_back(static_cast<std::int32_t>(sg.knob_space.knobs.size()));
    for (int k = 0; k < FS_MAX_KNOBS; ++k) {
      const bool has = k < static_cast<int>(sg.knob_space.knobs.size());
      nv.push_back(has ? static_cast<std::int32_t>(sg.knob_space.knobs[static_cast<std::size_t>(k)].values.size()) : 0);
      if (has) {
        const auto& v = sg.knob_space.knobs[static_cast<std::size_t>(k)].values;
        vals.insert(vals.end(), v.begin(), v.end());
      }
    }
  }
  ck(fs_spaces_create(dev_, static_cast<std::int32_t>(nk.size()), nk.data(), nv.data(), vals.data(), &spaces_));
  ck(fs_forest_create(dev_, S, &forest_));
  const std::int32_t off0 = 0;
  for (int s = 0; s < S; ++s)
    ck(fs_forest_upload(forest_, s, 0.0, options_.cost_model.learning_rate, 0, &off0, nullptr, nullptr, nullptr,
                        nullptr, nullptr));
  ck(fs_store_create(dev_, S, backend_.feature_pad_dim(), &store_));
  stale_.assign(static_cast<std::size_t>(S), 0);
  init_state();
}

BatchedTuningEngine::~BatchedTuningEngine() {
  if (store_) fs_store_destroy(store_);
  if (forest_) fs_forest_destroy(forest_);
  if (spaces_) fs_spaces_destroy(spaces_);
  if (dev_) fs_device_destroy(dev_);
}

int BatchedTuningEngine::slot_of(const CostModelState& model) const {
  const auto i = &model - models_.data();
  if (i < 0 || i >= static_cast<std::ptrdiff_t>(models_.size()))
    throw std::invalid_argument("BatchedTuningEngine: model does not belong to this engine");
  return static_cast<int>(i);
}

// CostModelState stays authoritative: pull the device model into the host trees when it moved.
void BatchedTuningEngine::sync(int slot) {
  if (!stale_[static_cast<std::size_t>(slot)]) return;
  auto& m = models_[static_cast<std::size_t>(slot)];
  double base = 0.0;
  std::int32_t nt = 0, nn = 0;
  ck(fs_forest_export(forest_, slot, &base, &nt, &nn, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                      nullptr));
  std::vector<std::int32_t> off(static_cast<std::size_t>(nt) + 1), feat(static_cast<std::size_t>(nn)),
      left(static_cast<std::size_t>(nn)), right(static_cast<std::size_t>(nn));
  std::vector<double> thr(static_cast<std::size_t>(nn)), val(static_cast<std::size_t>(nn)),
      mse(static_cast<std::size_t>(nt));
  ck(fs_forest_export(forest_, slot, &base, nullptr, nullptr, off.data(), feat.data(), thr.data(), left.data(),
                      right.data(), val.data(), nullptr, mse.data()));
  m.base_prediction = base;
  m.trees.assign(static_cast<std::size_t>(nt), RegressionTree{});
  for (int t = 0; t < nt; ++t) {
    auto& nodes = m.trees[static_cast<std::size_t>(t)].nodes;
    for (std::int32_t i = off[static_cast<std::size_t>(t)]; i < off[static_cast<std::size_t>(t) + 1]; ++i) {
      const auto k = static_cast<std::size_t>(i);
      nodes.push_back({feat[k], thr[k], left[k], right[k], val[k]});
    }
  }
  m.train_mse_by_round = std::move(mse);
  stale_[static_cast<std::size_t>(slot)] = 0;
}

std::span<CostModelState> BatchedTuningEngine::models() {
  for (int s = 0; s < static_cast<int>(models_.size()); ++s) sync(s);
  return models_;
}

// TuningEngine::model_for (scheduler.cpp:138-141)
CostModelState& BatchedTuningEngine::model_for(int subgraph_id) {
  const int slot = policy_.granularity == ModelGranularity::Monolithic ? 0 : registry_.family_of(subgraph_id);
  sync(slot);
  return models_[static_cast<std::size_t>(slot)];
}

// TuningEngine::init_state (scheduler.cpp:143-157)
void BatchedTuningEngine::init_state() {
  state_ = TunerState{};
  state_.budget = options_.budget;
  state_.p = options_.foresee_p;
  state_.g = static_cast<int>(
      std::min<std::int64_t>(64, options_.budget / static_cast<std::int64_t>(model_.subgraphs.size())));
  state_.per_subgraph.resize(model_.subgraphs.size());
  for (const auto& sg : model_.subgraphs) {
    auto& st = state_.per_subgraph[static_cast<std::size_t>(sg.id)];
    st.best_candidate = default_candidate(sg.knob_space, sg.id);
    st.best_latency_ms = backend_.default_latency(sg.id);
    st.prev_best_latency_ms = st.best_latency_ms;
  }
  record_point("init", -1);
}

// TuningEngine::record_point (scheduler.cpp:159-167)
void BatchedTuningEngine::record_point(const char* phase, int subgraph_id) {
  CurvePoint point;
  point.b = state_.b;
  point.wall_seconds = backend_.clock().now;
  point.model_latency_ms = state_.model_latency_now(model_);
  point.phase = phase;
  point.tuned_subgraph = subgraph_id;
  state_.curve.push_back(std::move(point));
}

// TuningEngine::tune_step (scheduler.cpp:169-231). The scoring block (:187-192, featurize +
// predict per candidate, then std::sort of (score, index)) is one fs_score call: the pool goes to
// the device as descriptors, the family's resident model scores it, and the device returns the
// full (score, index) permutation - std::sort's order, -0.0 == +0.0.
std::vector<MeasurementRecord> BatchedTuningEngine::tune_step(int subgraph_id, CostModelState& cm, int g_eff) {
  if (g_eff < 1) throw std::invalid_argument("tune_step: g_eff must be >= 1");
  const auto& sg = model_.subgraphs[static_cast<std::size_t>(subgraph_id)];
  auto& st = state_.per_subgraph[static_cast<std::size_t>(subgraph_id)];
  auto& rng = gen_streams_[static_cast<std::size_t>(subgraph_id)];

  auto pool = generate_candidates(sg.knob_space, subgraph_id, st.measured, options_.pool_random,
                                  options_.pool_evolved, rng);
  if (pool.empty()) {
    st.exhausted = true;
    return {};
  }

  std::vector<Candidate> batch;
  if (static_cast<int>(pool.size()) <= g_eff) {
    batch = std::move(pool);
  } else {
    const int slot = slot_of(cm);
    std::vector<std::int32_t> space_of, assign;
    pack(pool, space_of, assign);
    // segment `slot` holds the pool (earlier segments empty): scored with forest slot `slot`
    std::vector<std::int64_t> seg(static_cast<std::size_t>(slot) + 2, 0);
    seg.back() = static_cast<std::int64_t>(pool.size());
    std::vector<std::int32_t> perm(pool.size());
    ck(fs_score(dev_, spaces_, forest_, slot + 1, seg.data(), space_of.data(), assign.data(),
                backend_.feature_pad_dim(), nullptr, perm.data()));

    // Epsilon slots come uniformly from the pool's tail (scheduler.cpp:194-213, host RNG).
    const int explore = static_cast<int>(static_cast<double>(g_eff) * options_.epsilon_explore);
    const int by_score = g_eff - explore;
    batch.reserve(static_cast<std::size_t>(g_eff));
    for (int i = 0; i < by_score; ++i) batch.push_back(pool[static_cast<std::size_t>(perm[static_cast<std::size_t>(i)])]);
    if (explore > 0) {
      std::vector<std::size_t> tail;
      tail.reserve(perm.size() - static_cast<std::size_t>(by_score));
      for (std::size_t i = static_cast<std::size_t>(by_score); i < perm.size(); ++i)
        tail.push_back(static_cast<std::size_t>(perm[i]));
      for (int e = 0; e < explore; ++e) {
        const auto pick = uniform_below(rng, tail.size() - static_cast<std::size_t>(e));
        batch.push_back(pool[tail[pick]]);
        std::swap(tail[pick], tail[tail.size() - 1 - static_cast<std::size_t>(e)]);
      }
    }
  }

  auto records = backend_.run_batch(batch);
  for (const auto& rec : records) {
    const auto key = linear_index(sg.knob_space, rec.candidate.assignment);
    st.measured.add(key, rec.latency_ms);
    st.spent += 1;
    st.measured_any = true;
    if (rec.latency_ms < st.best_latency_ms) {
      st.best_latency_ms = rec.latency_ms;
      st.best_candidate = rec.candidate;
      st.last_improvement_spent = st.spent;
    }
  }
  st.records.insert(st.records.end(), records.begin(), records.end());
  if (st.measured.size() == space_size(sg.knob_space)) st.exhausted = true;
  return records;
}

// TuningEngine::train_and_charge (scheduler.cpp:233-238): train_cost_model (costmodel.cpp:224-235)
// = append {features, log(latency)} to the family's training set, refit from scratch. Here the
// batch's descriptors go to the device store (featurized there, canonical order merged) and the
// store refits the family into its forest slot; the host training set is kept in step so
// CostModelState::training_set stays authoritative.
void BatchedTuningEngine::train_and_charge(std::span<const MeasurementRecord> records, CostModelState& cm) {
  const int slot = slot_of(cm);
  std::vector<Candidate> cands;
  std::vector<double> lat;
  cands.reserve(records.size());
  for (const auto& rec : records) {
    cands.push_back(rec.candidate);
    lat.push_back(rec.latency_ms);
  }
  std::vector<std::int32_t> space_of, assign;
  pack(cands, space_of, assign);
  const std::int64_t seg[2] = {0, static_cast<std::int64_t>(records.size())};
  // FS_EINVAL (-> std::invalid_argument) on an empty batch or latency <= 0, nothing appended
  // (costmodel.cpp:225-231)
  ck(fs_store_append_records(store_, spaces_, 1, &slot, seg, space_of.data(), assign.data(), lat.data()));
  for (const auto& rec : records) cm.training_set.push_back({rec.features, std::log(rec.latency_ms)});
  const fs_gbt_params p{cm.params.trees, cm.params.depth, cm.params.learning_rate, cm.params.min_samples_split};
  ck(fs_store_fit(store_, forest_, 1, &slot, &p));
  stale_[static_cast<std::size_t>(slot)] = 1;
  backend_.charge_training(static_cast<std::int64_t>(cm.training_set.size()), options_.cm_accelerated);
}

// TuningEngine::run (scheduler.cpp:240-290)
TunerState BatchedTuningEngine::run() {
  std::vector<int> all_ids(model_.subgraphs.size());
  std::iota(all_ids.begin(), all_ids.end(), 0);

  while (state_.b < state_.budget) {
    const int s_cur = select_bottleneck(all_ids, state_, model_, policy_.potential);
    if (s_cur < 0) break;  // every space exhausted

    auto& st_cur_before = state_.per_subgraph[static_cast<std::size_t>(s_cur)];
    const double prev_best = st_cur_before.best_latency_ms;
    auto& cm = models_[static_cast<std::size_t>(
        policy_.granularity == ModelGranularity::Monolithic ? 0 : registry_.family_of(s_cur))];
    const auto records = tune_step(s_cur, cm, state_.g);
    if (!records.empty()) {
      auto& st = state_.per_subgraph[static_cast<std::size_t>(s_cur)];
      st.prev_best_latency_ms = prev_best;
      st.last_step_measurements = static_cast<std::int64_t>(records.size());
      state_.b += static_cast<std::int64_t>(records.size());
      st.best_history.emplace_back(state_.b, st.best_latency_ms);
      train_and_charge(records, cm);
      record_point("main", s_cur);
    }

    if (!policy_.foresee_phase) continue;
    const auto& family = find_family(s_cur, registry_);
    if (family.member_ids.size() <= 1) continue;

    std::vector<int> siblings;
    siblings.reserve(family.member_ids.size() - 1);
    for (int sid : family.member_ids) {
      if (sid != s_cur) siblings.push_back(sid);
    }
    const int s_next = select_bottleneck(siblings, state_, model_, policy_.potential);
    if (s_next < 0) continue;

    const int g_foresee = std::max(1, static_cast<int>(static_cast<double>(state_.g) * options_.foresee_p));
    const double prev_best_next = state_.per_subgraph[static_cast<std::size_t>(s_next)].best_latency_ms;
    const auto foresee_records = tune_step(s_next, cm, g_foresee);
    if (!foresee_records.empty()) {
      auto& st = state_.per_subgraph[static_cast<std::size_t>(s_next)];
      st.prev_best_latency_ms = prev_best_next;
      st.last_step_measurements = static_cast<std::int64_t>(foresee_records.size());
      state_.b += static_cast<std::int64_t>(foresee_records.size());
      st.best_history.emplace_back(state_.b, st.best_latency_ms);
      train_and_charge(foresee_records, cm);
      record_point("foresee", s_next);
    }
  }
  for (int s = 0; s < static_cast<int>(models_.size()); ++s) sync(s);
  return state_;
}

}  // namespace gpu
}  // namespace famtune
