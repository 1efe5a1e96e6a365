// famtune/searchspace.hpp - drop-in declarations of the candidate-descriptor and featurization
// part of the reference API (/root/reference/proj/core/include/famtune/searchspace.hpp:18-68),
// implemented by libfamtune_b200.so on the B200 (featurize runs as kernel 1 through the C ABI in
// include/famseer.h). Type layouts match the reference so its unchanged callers link against
// this library. Candidate generation (generate_candidates, MeasuredSet) is host RNG logic that
// stays in the caller.
#pragma once

#include <cstdint>
#include <span>
#include <string>
#include <vector>

namespace famtune {

inline constexpr int kMaxKnobs = 16;

struct Knob {
  std::string name;
  std::vector<std::int64_t> values;  // distinct, >= 1
};

struct SpaceDescriptor {
  std::vector<Knob> knobs;  // 1..kMaxKnobs
};

struct Candidate {
  int subgraph_id = -1;
  std::vector<std::int32_t> assignment;  // one value index per knob

  friend bool operator==(const Candidate&, const Candidate&) = default;
};

struct MeasurementRecord {
  Candidate candidate;
  std::vector<double> features;
  double latency_ms = 0.0;
  double measured_at = 0.0;
};

/// 2K + K(K-1)/2 (searchspace.cpp:86-88).
int feature_dim(int knob_count);

/// Mixed-radix rank / unrank of an assignment (searchspace.cpp:48-66).
std::uint64_t linear_index(const SpaceDescriptor& space, std::span<const std::int32_t> assignment);
Candidate candidate_from_index(const SpaceDescriptor& space, int subgraph_id, std::uint64_t index);

/// Same contract as the reference (searchspace.cpp:90-118); computed on the GPU. Throws
/// std::invalid_argument on a length mismatch or pad_dim < feature_dim(K).
std::vector<double> featurize(const SpaceDescriptor& space, std::span<const std::int32_t> assignment,
                              int pad_dim);

namespace gpu {
/// Batched featurize: rows[i] = featurize(space, assignments[i*K .. +K], pad_dim), K knobs each.
std::vector<double> featurize_batch(const SpaceDescriptor& space, std::span<const std::int32_t> assignments,
                                    int pad_dim);
}  // namespace gpu

}  // namespace famtune
