// famtune::gpu::BatchedTuningEngine - the reference's tuning loop (TuningEngine, Algorithm 1,
// scheduler.hpp:97-126 / scheduler.cpp:102-290) with its two hot blocks batched onto the B200:
//
//   * tune_step's scoring block (scheduler.cpp:187-192: featurize + predict once PER CANDIDATE,
//     then std::sort) is ONE fs_score call per pool - fused featurize -> predict -> rank on the
//     device, the family's model already resident there;
//   * train_and_charge (scheduler.cpp:233-238: train_cost_model = append the batch to the
//     family's training set and refit from scratch) is fs_store_append_records + fs_store_fit:
//     the training set stays on the device, only the new batch's descriptors travel, and the
//     canonical row order is merged instead of re-sorted.
//
// Everything else - bottleneck selection, candidate generation (mt19937_64 replay), the epsilon
// picks from the pool's tail, measurement, the simulated clock, the curve - is the reference's
// own code or a line-by-line restatement of its control flow, so the curve, registry and models
// are byte-identical to TuningEngine's (tests/test_engine_e2e.py). CostModelState stays the
// authoritative model: models()/model_for() refresh the host trees from the device on access.
//
// Compile against the reference's headers (famtune/scheduler.hpp, simbackend.hpp) - this is the
// caller-side integration of the drop-in, built as libfamtune_b200_tuner.so
// (paper_2201_00194_b200/host/Makefile, target `tuner`).
#pragma once

#include <span>
#include <vector>

#include "famseer.h"
#include "famtune/scheduler.hpp"

namespace famtune {
namespace gpu {

class BatchedTuningEngine {
 public:
  BatchedTuningEngine(SimBackend& backend, Policy policy, TuneOptions options);
  ~BatchedTuningEngine();
  BatchedTuningEngine(const BatchedTuningEngine&) = delete;
  BatchedTuningEngine& operator=(const BatchedTuningEngine&) = delete;

  /// TuningEngine::run (scheduler.cpp:240-290).
  TunerState run();
  /// TuningEngine::tune_step (scheduler.cpp:169-231) with the pool scored by one fs_score.
  std::vector<MeasurementRecord> tune_step(int subgraph_id, CostModelState& model, int g_eff);

  TunerState& state() { return state_; }
  const FamilyRegistry& registry() const { return registry_; }
  std::span<CostModelState> models();
  CostModelState& model_for(int subgraph_id);

 private:
  void init_state();
  void record_point(const char* phase, int subgraph_id);
  void train_and_charge(std::span<const MeasurementRecord> records, CostModelState& model);
  int slot_of(const CostModelState& model) const;
  void sync(int slot);

  SimBackend& backend_;
  const ModelGraph& model_;
  Policy policy_;
  TuneOptions options_;
  FamilyRegistry registry_;
  std::vector<CostModelState> models_;  // one per family, or a single entry
  std::vector<Rng> gen_streams_;        // candidate generation, one per subgraph
  TunerState state_;
  // device side: one forest slot and one store family per model
  fs_device* dev_ = nullptr;
  fs_spaces* spaces_ = nullptr;  // one knob space per subgraph
  fs_forest* forest_ = nullptr;
  fs_store* store_ = nullptr;
  std::vector<char> stale_;  // device model newer than models_[slot].trees
};

}  // namespace gpu
}  // namespace famtune
