// famtune/graph.hpp - the subgraph description types the family grouping keys on, layout-
// compatible with the reference (/root/reference/proj/core/include/famtune/graph.hpp:16-66).
// Model-file parsing (load_model / parse_model) is out of scope for this library (SURVEY.md 2:
// one-time host ingestion); callers keep the reference's loader.
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <string>
#include <string_view>
#include <vector>

#include "famtune/searchspace.hpp"

namespace famtune {

// Closed operator vocabulary, in the reference's declaration order (the enum values are ABI).
enum class OpKind : std::uint8_t {
  Conv1d,
  Conv2d,
  Conv3d,
  DepthwiseConv2d,
  Dense,
  BatchMatmul,
  Softmax,
  Pooling,
  Relu,
  Gelu,
  Sigmoid,
  Tanh,
  Add,
  Multiply,
  LayerNorm,
  BatchNorm,
  Embedding,
  Transpose,
  Reshape,
  Reduce,
};

std::string_view to_string(OpKind kind);
std::optional<OpKind> op_kind_from_string(std::string_view name);

struct OperatorNode {
  OpKind op_kind = OpKind::Add;
  std::vector<std::int64_t> input_shape;
  std::map<std::string, std::int64_t> attrs;

  friend bool operator==(const OperatorNode&, const OperatorNode&) = default;
};

struct Subgraph {
  int id = -1;
  std::vector<OperatorNode> ops;
  OpKind core_op = OpKind::Add;
  std::int64_t weight = 1;
  SpaceDescriptor knob_space;
};

struct ModelGraph {
  std::string name;
  std::vector<Subgraph> subgraphs;
};

/// Operator kinds joined with ',' (graph.cpp serialize_op_sequence) - the op-sequence key.
std::string serialize_op_sequence(const Subgraph& sg);

}  // namespace famtune
