// famtune/costmodel.hpp - drop-in declarations of the reference's per-family cost-model API
// (/root/reference/proj/core/include/famtune/costmodel.hpp:18-80) backed by the B200 kernels of
// libfamseer.so. Same types, same layouts, same semantics and exceptions:
//   fit / train_cost_model  -> kernel 3 (bit-identical trees)
//   predict / eval          -> kernel 2
//   pairwise_accuracy       -> kernel 2 + an on-device pair count
// plus batched entry points in famtune::gpu for callers that score or retrain many candidates /
// families at once (the modified tune_step / train_and_charge of SURVEY.md 8b).
#pragma once

#include <cstdint>
#include <span>
#include <string>
#include <vector>

#include "famtune/searchspace.hpp"

namespace famtune {

inline constexpr int kMonolithicModel = -1;

struct GbtParams {
  int trees = 50;
  int depth = 3;
  double learning_rate = 0.1;
  int min_samples_split = 2;
};

struct TreeNode {
  int feature = -1;  // < 0: leaf
  double threshold = 0.0;
  int left = -1;
  int right = -1;
  double value = 0.0;

  bool is_leaf() const { return feature < 0; }
};

struct RegressionTree {
  std::vector<TreeNode> nodes;  // pre-order, nodes[0] = root

  double eval(std::span<const double> features) const;
};

struct TrainingSample {
  std::vector<double> features;
  double target = 0.0;  // log latency
};

struct CostModelState {
  int family_id = kMonolithicModel;
  GbtParams params;
  double base_prediction = 0.0;
  std::vector<RegressionTree> trees;
  std::vector<TrainingSample> training_set;
  std::vector<double> train_mse_by_round;

  bool trained() const { return !training_set.empty(); }
};

CostModelState initialize_cost_model(int family_id, GbtParams params = {});
void train_cost_model(std::span<const MeasurementRecord> records, CostModelState& model);
void fit(CostModelState& model);
double predict(const CostModelState& model, std::span<const double> features);
double pairwise_accuracy(const CostModelState& model, std::span<const MeasurementRecord> validation);
std::string dump_model(const CostModelState& model);

namespace gpu {

/// Refit several family models in ONE device pass (all families' boosting rounds run
/// concurrently). Equivalent to calling fit() on each.
void fit_many(std::span<CostModelState* const> models);

/// Scores of `rows` feature vectors of width d (row-major) under `model`.
std::vector<double> predict_batch(const CostModelState& model, std::span<const double> rows, int d);

/// The ascending (score, index) order std::sort gives vector<pair<double,size_t>>
/// (scheduler.cpp:192), computed on the device.
std::vector<std::int32_t> rank(std::span<const double> scores);

/// Split gain of every node of the last fit of `model` (0 for leaves), in pre-order per tree -
/// the value best_split compared (costmodel.cpp:58-65), which the reference does not store.
std::vector<double> split_gains(const CostModelState& model);

/// Device ordinal the process-wide runtime uses (env FAMSEER_DEVICE, default 0).
int device_ordinal();

}  // namespace gpu
}  // namespace famtune
