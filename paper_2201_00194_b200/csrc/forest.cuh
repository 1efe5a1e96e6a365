// Family model store: one ensemble per family (TuningEngine::models_, scheduler.cpp:123-130),
// kept in two forms.
//   * pre-order host arrays - the CostModelState layout (costmodel.hpp:27-57), authoritative and
//     exported unchanged so callers' CostModelState stays the source of truth;
//   * a compiled device form for predict: every tree expanded to a complete heap of depth
//     `depth` (early leaves replicated under always-left nodes), node = feature | rank<<16 where
//     rank is the threshold's index among the sorted unique thresholds the ensemble uses for that
//     feature. A row's feature value x becomes code(x) = #{unique thresholds < x}, and
//     x <= t_rank  <=>  code(x) <= rank  exactly (SURVEY.md "Bit-exactness rules" 2), so the
//     traversal compares small integers instead of FP64 values.
#pragma once

#include <vector>

#include "fs_common.cuh"

namespace fs {

constexpr int kMaxHeapDepth = 8;  // deeper ensembles take the generic pre-order kernel

// Device-side header of a compiled model (first bytes of the blob when the fit compiled it on
// the device): predict reads n_trees / base from here, so fs_fit needs no host round trip.
struct ModelMeta {
  double base;
  int32_t n_trees;
  int32_t pad_;
  int64_t screened, exact;  // fit diagnostics
};

// Offsets (bytes into blob_d) of a device-compiled fit result: the compiled predict form and the
// reference pre-order export, both written by the fit's export kernel.
struct DevLayout {
  size_t meta, nodes, leafv, leafid, uthr, uoff, fmap;  // compiled
  size_t cnt, feat, thr, left, right, val, gain, mse;   // pre-order export (per tree: S slots)
  size_t total;
  int max_trees = 0, slots = 0;  // S = nodes per tree slot block
};

struct FamilyModel {
  // ---- pre-order form (host) ----
  double base = 0.0;
  double lr = 0.1;
  std::vector<int32_t> offsets{0};
  std::vector<int32_t> feature, left, right;
  std::vector<double> threshold, value, gain, mse;
  int64_t screened = 0, exact = 0;  // fit diagnostics

  // ---- compiled form (device) ----
  bool compiled = false;
  int n_trees = 0;
  int depth = 0;       // heap depth (max leaf depth over trees)
  int d_model = 0;     // 1 + max feature index referenced
  int code_bytes = 1;  // 1: codes fit uint8, 2: uint16
  bool generic = false;  // depth > kMaxHeapDepth: pre-order device arrays instead of heaps
  uint32_t* nodes_d = nullptr;   // [T][2^depth - 1]
  double* leafv_d = nullptr;     // [T][2^depth]
  uint16_t* leafid_d = nullptr;  // [T][2^depth] pre-order node index of each heap leaf
  double* uthr_d = nullptr;      // unique thresholds, feature-major
  int n_uthr = 0;
  int32_t* uoff_d = nullptr;     // [d_model + 1]
  // generic form
  int32_t* g_off_d = nullptr;
  int32_t* g_feat_d = nullptr;
  double* g_thr_d = nullptr;
  int32_t* g_left_d = nullptr;
  int32_t* g_right_d = nullptr;
  double* g_val_d = nullptr;

  // all compiled arrays live in one grow-only device blob (refits reuse it: no cudaMalloc /
  // cudaFree per fit, one copy per compile)
  unsigned char* blob_d = nullptr;
  size_t blob_cap = 0;
  // fit compiled on the device: host pre-order arrays are materialised on first use
  bool pending = false;
  DevLayout lay;
  const int32_t* fmap_d = nullptr;    // compiled feature -> original feature (nullptr = identity)
  int d_orig = 0;                     // 1 + largest original feature referenced (row-width check)
  const ModelMeta* meta_d = nullptr;  // device n_trees / base (nullptr = host fields)

  int num_trees() const { return static_cast<int>(offsets.size()) - 1; }
  void release_device();
};

// Host->device copies of several compiled models gathered into one pinned staging pass.
struct UploadBatch {
  std::vector<unsigned char> host;
  std::vector<std::pair<unsigned char*, std::pair<size_t, size_t>>> items;  // dst, (offset, bytes)
  void add(unsigned char* dst, const unsigned char* src, size_t bytes);
  void flush(fs_device* dev);  // one pinned staging fill, async copies, no host wait
};

// Download a device-compiled fit's pre-order export into the host arrays (no-op otherwise).
void materialize(fs_device* dev, FamilyModel& m);
void materialize(fs_device* dev, const FamilyModel& m);
void materialize_all(fs_device* dev, std::vector<FamilyModel>& fams);
bool materialize_enqueue(fs_device* dev, std::vector<FamilyModel>& fams);  // copies into dev->pinned; true if any
void materialize_parse(fs_device* dev, std::vector<FamilyModel>& fams);    // after the stream synchronised

// Build the compiled device form from the pre-order arrays (host transformation of the tree
// table; O(nodes)). With a batch, the device copy is deferred to batch->flush().
void compile_model(fs_device* dev, FamilyModel& m, UploadBatch* batch = nullptr);

}  // namespace fs

struct fs_forest {
  fs_device* dev = nullptr;
  std::vector<fs::FamilyModel> fams;
};
