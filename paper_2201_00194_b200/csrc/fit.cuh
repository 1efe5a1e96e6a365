// Kernel (3): the boosting trainer - fit (costmodel.cpp:152-222) for many families at once.
//
// Bit-exact design (SURVEY.md 7 "Hard parts" 1-2 and Appendix A P3-P5):
//   * every value that reaches a tree - base, node totals, leaf values, predictions - is folded
//     in the reference's order with separately rounded FP64 adds (chains over the canonical /
//     feature-0-presorted row order);
//   * split search is a histogram SCREEN in exact 62-bit fixed point (integer sums: associative,
//     deterministic, exactly subtractable for the sibling trick), with a rigorous per-candidate
//     bound on how far the reference's own FP64 gain can sit from the screened one;
//   * when more than one candidate (or one of uncertain sign) survives the bound, the node is
//     re-evaluated in the reference's order: one warp per (node, surviving feature) folds the
//     residuals over that feature's presorted list restricted to the node, exactly as
//     best_split (costmodel.cpp:42-71) does, and the decision applies its strict-> rule.
// Features that are constant over a family's training set, or whose code column equals an
// earlier feature's (same order and ties, e.g. log2(v) and v's list position), are dropped up
// front: the reference can never pick them (strict > keeps the earlier, identical gain).
#pragma once

#include "forest.cuh"

namespace fs {
namespace fit {

constexpr int kMaxDepth = 10;                 // 2047 node slots per tree
constexpr int kSmallBins = 256;               // hash-path distinct-value limit per feature
constexpr int kMaxBins = 65535;               // per feature (u16 codes)
constexpr int kSortThreads = 1024;            // stable counting sort CTA
constexpr int kNodeLeaf = 1, kNodeSplit = 2, kNodeExact = 3;

// Per-family constants (device array).
struct FamDesc {
  int64_t row0;   // first caller row (x/target)
  int64_t pos0;   // first slot in the per-row canonical arrays
  int64_t ord0;   // first entry of this family's presorted lists (nrep * n)
  int64_t bin0;   // first bin of this family in per-bin tables
  int64_t hist0;  // first bin of this family's histogram ring (2 * level_slots * bins)
  int64_t node0;  // first node slot of this family in per-node tables
  int64_t lbuf0;  // first entry of this family's exact-fold buffer (level_slots * bins)
  int64_t tree0;  // first record of this family's tree table (trees * slots)
  int32_t n;
  int32_t nrep;
  int32_t rep0;   // first entry in per-rep tables
  int32_t bins;   // total bins over reps
  int32_t trees;
  int32_t depth;
  int32_t min_split;
  int32_t f0rep;  // rep index of original feature 0, -1 if feature 0 is constant
  int32_t level_slots;  // 2^(depth-1) (max histogrammed nodes per level), >= 1
  int32_t negz;         // some feature value is -0.0 (thresholds then need the exact row value)
  double lr;
};

// Per-family mutable scalars.
struct FamState {
  int32_t active;   // still boosting
  int32_t ntrees;   // committed trees
  int32_t shift;    // fixed-point exponent of this round
  int32_t pad_;
  uint64_t maxabs;  // bits of max |residual| (non-negative doubles order like integers)
  unsigned long long screened;  // splits decided by the histogram screen alone
  unsigned long long exact;     // nodes re-evaluated in reference order
};

// Per node slot (per family, kSlots = 2^(depth_max+1)-1).
struct NodeRec {
  int32_t n;        // rows
  int32_t seg;      // start of its rows in the order-0 list (family-relative)
  int32_t state;    // 0 absent/undecided, kNodeLeaf, kNodeSplit, kNodeExact
  int32_t rep;      // split feature (rep index)
  int32_t bin;      // split bin (left = code <= bin)
  int32_t lc;       // left count
  int32_t wcount;   // screen window candidates
  int32_t build;    // 1 if its histogram is accumulated directly this level
  int32_t eqf0;     // lowest window feature when the window may be one tie class, else -1
  int32_t pad_;
  double gain;      // split gain (reference's value)
  double value;     // leaf value
  double total;     // exact reference-order node total (exact nodes / leaves)
  uint64_t lokey;   // max lower bound over candidates (order-preserving key)
};

// Tree table record (per family, per round, per slot).
struct TreeRec {
  int32_t kind;     // 0 absent, kNodeLeaf, kNodeSplit
  int32_t feature;  // original feature index
  double threshold;
  double value;
  double gain;
  int32_t rep;      // split: representative feature index (compiled model feature)
  int32_t bin;      // split: bin of the threshold among the rep's distinct values (its rank)
};

// Window bookkeeping per (node, rep): screen lower/upper bound of the feature's best candidate.
struct WinRec {
  double best_g;    // screened gain of the feature's best candidate
  double best_lo;
  int32_t best_bin;
  int32_t flag;     // feature has >= 1 candidate in the node's window
  int32_t count;    // window candidates of this feature
  int32_t best_lc;  // left count of the best candidate
  int32_t eq;       // order-equivalent (within the node) to the node's lowest window feature
  int32_t maxlc;    // largest left count among the feature's window candidates
};

// Where a fit's rows live when they do not come packed by seg (fs_store):
// segment f's rows are x/target rows [row0[f], row0[f] + n[f]) (seg still gives the counts),
// fam_id[f] is the forest family it refits, and canon (indexed like x rows) holds each family's
// canonical row order (costmodel.cpp:161-173) as family-relative row ids: io[f] = 1 takes it
// from there (the sort is skipped), 2 writes the fit's order back, 0 neither.
struct FitRows {
  const int64_t* row0 = nullptr;
  const int32_t* fam_id = nullptr;
  int64_t span = 0;  // rows addressable in x
  int32_t* canon = nullptr;
  const int* io = nullptr;
  int* negz_out = nullptr;  // per segment: the family holds a -0.0 (its canonical order is not taken)
};

void fit_families(fs_device* dev, fs_forest* fo, int F, const int64_t* seg, int d, const double* x_d,
                  const double* target_d, const fs_gbt_params* params, const FitRows* rows = nullptr);

}  // namespace fit
}  // namespace fs
