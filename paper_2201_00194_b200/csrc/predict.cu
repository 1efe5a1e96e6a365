// Kernel (2): GBDT ensemble predict - predict (costmodel.cpp:237-246) with RegressionTree::eval
// (:135-143) for a whole candidate population, one launch per family segment.
//
// CTA = a tile of 256 candidates, one per thread.
//   1. Stage: warps stream the tile's FP64 rows from HBM with coalesced loads (lanes over
//      features), check finiteness (the reference throws on any non-finite feature) and convert
//      each value the ensemble actually tests into its threshold code (binary search in the
//      feature's sorted unique thresholds). Codes land in shared memory transposed
//      [feature][candidate] so a warp reading one feature hits consecutive bytes.
//   2. Trees are staged through shared memory in chunks; each thread walks its candidate down
//      every tree of the chunk (fixed-depth heap, no divergence in trip count) and folds
//      score = score + lr*leaf in tree order with separately rounded __dmul_rn/__dadd_rn - the
//      reference's `score += learning_rate * tree.eval(x)` without FMA.
// HBM traffic per candidate = 8*d (row) + 8 (score) [+ T leaf ids]; the model is read once per
// CTA from L2.
#include <algorithm>

#include "forest.cuh"

namespace {

constexpr int kTile = 256;
constexpr int kChunk = 64;

// One family's compiled ensemble, as the batched kernel sees it.
struct PredModel {
  const uint32_t* nodes;
  const double* leafv;
  const uint8_t* leafid;
  const double* uthr;
  const int32_t* uoff;
  double base, lr;
  int depth, n_trees, d_model, n_uthr;
  const int32_t* fmap;       // compiled feature -> original feature (nullptr: identity)
  const fs::ModelMeta* meta;  // device-compiled fit: n_trees / base live on the device
};

// Candidate descriptors for the fused score path (kFused): the kernel computes each tested
// feature from the assignment exactly as featurize does (searchspace.cpp:90-118; log2/position
// tables built on the host, pair products one __dmul_rn) instead of reading a feature row.
struct SpaceTabs {
  const int32_t* space_of;  // [P]
  const int32_t* assign;    // [P][16] value indices
  const int32_t* k;         // [n_spaces] knobs
  const int32_t* nval;      // [n_spaces][16]
  const int32_t* off;       // [n_spaces][16] offset into log/pos
  const double* log;
  const double* pos;
  int n_spaces;
  int pad;
};

// One CTA's work: a tile of up to kTile rows of one family segment.
struct PredJob {
  int32_t model, rows;
  int64_t row0;   // first row (into x / scores)
  int64_t leaf0;  // byte offset of row0's leaf ids
};

// Every family segment of a predict call is scored by ONE launch (a family is typically a few
// hundred tiles; one launch per family left most of the 148 SMs idle). Shared memory is laid out
// for the largest model of the launch; each CTA uses its own model's shape.
template <typename CodeT, bool kLeaves, bool kSmemThr, bool kFused>
__global__ void __launch_bounds__(kTile) predict_heap_kernel(
    const double* __restrict__ x, int d, const PredModel* __restrict__ models, const PredJob* __restrict__ jobs,
    int max_dmodel, int max_depth, int max_uthr, double* __restrict__ scores, uint8_t* __restrict__ leaf_out,
    uint32_t* err, SpaceTabs sp) {
  extern __shared__ __align__(16) unsigned char smem[];
  const PredJob job = jobs[blockIdx.x];
  const PredModel M = models[job.model];
  const int depth = M.depth, d_model = M.d_model;
  const int n_trees = M.meta ? M.meta->n_trees : M.n_trees;
  const int32_t* fmap = M.fmap;
  const int nint = (1 << depth) - 1;
  const int nleaf = 1 << depth;
  const int mnint = (1 << max_depth) - 1, mnleaf = 1 << max_depth;
  CodeT* codes = reinterpret_cast<CodeT*>(smem);  // [d_model][kTile]
  size_t off = (static_cast<size_t>(max_dmodel) * kTile * sizeof(CodeT) + 15) & ~size_t(15);
  double* s_leafv = reinterpret_cast<double*>(smem + off);  // [kChunk][nleaf]
  off += static_cast<size_t>(kChunk) * mnleaf * sizeof(double);
  uint32_t* s_nodes = reinterpret_cast<uint32_t*>(smem + off);  // [kChunk][nint]
  off += static_cast<size_t>(kChunk) * mnint * sizeof(uint32_t);
  uint8_t* s_leafid = smem + off;  // [kChunk][nleaf]
  off += static_cast<size_t>(kChunk) * mnleaf;
  uint8_t* s_lbuf = smem + off;  // [kTile][kChunk]
  off += kLeaves ? static_cast<size_t>(kTile) * kChunk : 0;
  off = (off + 15) & ~size_t(15);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  // The threshold tables the codes are searched in: staged in shared memory when they fit
  // (binary-search steps then cost a shared load instead of an L2 round trip).
  const double* uthr = M.uthr;
  const int32_t* uoff = M.uoff;
  if (kSmemThr) {
    double* su = reinterpret_cast<double*>(smem + off);
    int32_t* so = reinterpret_cast<int32_t*>(su + max_uthr);
    for (int i = tid; i < M.n_uthr; i += kTile) su[i] = __ldg(M.uthr + i);
    for (int i = tid; i <= d_model; i += kTile) so[i] = __ldg(M.uoff + i);
    __syncthreads();
    uthr = su;
    uoff = so;
  }
  const int64_t row0 = job.row0;
  const int tile_rows = job.rows;

  auto code_of = [&](int f, double v) {
    int lo = uoff[f], hi = uoff[f + 1];
    const int first = lo;
    while (lo < hi) {  // count of unique thresholds strictly below v
      const int mid = (lo + hi) >> 1;
      if (uthr[mid] < v) lo = mid + 1;
      else hi = mid;
    }
    return static_cast<CodeT>(lo - first);
  };
  if constexpr (kFused) {
    // warp per candidate: lane k < K fetches knob k's log2 / position; every tested feature is
    // formed from shuffles (featurize_kernel's arithmetic) and coded - no feature row in HBM
    for (int c = warp; c < tile_rows; c += kTile / 32) {
      const int64_t cand = row0 + c;
      const int s = __ldg(sp.space_of + cand);
      const bool bad_space = s < 0 || s >= sp.n_spaces;
      const int k = bad_space ? 0 : __ldg(sp.k + s);
      const int dim = 2 * k + k * (k - 1) / 2;
      double lg = 0.0, ps = 0.0;
      bool bad = false;
      if (lane < k) {
        const int a = __ldg(sp.assign + cand * FS_MAX_KNOBS + lane);
        const int m = __ldg(sp.nval + s * FS_MAX_KNOBS + lane);
        if (a < 0 || a >= m) {
          bad = true;
        } else {
          const int off = __ldg(sp.off + s * FS_MAX_KNOBS + lane);
          lg = __ldg(sp.log + off + a);
          ps = __ldg(sp.pos + off + a);
        }
      }
      const unsigned any_bad = __ballot_sync(0xffffffffu, bad);
      if (lane == 0) {
        if (bad_space) atomicOr(err, fs::kErrSpaceId);
        if (any_bad) atomicOr(err, fs::kErrKnobRange);
        if (sp.pad < dim) atomicOr(err, fs::kErrPadDim);
      }
      for (int base = 0; base < d_model; base += 32) {
        const int f = base + lane;
        const int g = f < d_model && fmap ? __ldg(fmap + f) : f;  // the original feature index
        int src_a = 0, src_b = 0, kind = 0;  // 0 zero (padding), 1 log, 2 pos, 3 product
        if (g < k) {
          kind = 1;
          src_a = g;
        } else if (g < 2 * k) {
          kind = 2;
          src_a = g - k;
        } else if (g < dim) {
          kind = 3;
          fs::pair_of(k, g - 2 * k, src_a, src_b);
        }
        const double la = __shfl_sync(0xffffffffu, lg, src_a);
        const double lb = __shfl_sync(0xffffffffu, lg, src_b);
        const double pa = __shfl_sync(0xffffffffu, ps, src_a);
        double v = 0.0;
        if (kind == 1) v = la;
        else if (kind == 2) v = pa;
        else if (kind == 3) v = fs_mul(la, lb);
        if (f < d_model) codes[f * kTile + c] = code_of(f, v);
      }
    }
  } else {
    bool nonfinite = false;
    for (int c = warp; c < tile_rows; c += kTile / 32) {
      const double* xr = x + (row0 + c) * d;
      for (int f = lane; f < d; f += 32) {
        const double v = __ldcs(xr + f);  // streamed once
        nonfinite |= !isfinite(v);
        if (!fmap && f < d_model) codes[f * kTile + c] = code_of(f, v);
      }
      if (fmap)  // compiled features are representatives: gather their original columns (L1 hits)
        for (int f = lane; f < d_model; f += 32) codes[f * kTile + c] = code_of(f, xr[__ldg(fmap + f)]);
    }
    if (__any_sync(0xffffffffu, nonfinite) && lane == 0) atomicOr(err, fs::kErrNonFinitePredict);
  }

  double score = M.meta ? M.meta->base : M.base;
  const double lr = M.lr;
  const bool active = tid < tile_rows;
  for (int t0 = 0; t0 < n_trees; t0 += kChunk) {
    const int ch = min(kChunk, n_trees - t0);
    __syncthreads();  // codes ready / previous chunk consumed
    for (int i = tid; i < ch * nint; i += kTile) s_nodes[i] = __ldg(M.nodes + static_cast<size_t>(t0) * nint + i);
    for (int i = tid; i < ch * nleaf; i += kTile) {
      s_leafv[i] = __ldg(M.leafv + static_cast<size_t>(t0) * nleaf + i);
      s_leafid[i] = __ldg(M.leafid + static_cast<size_t>(t0) * nleaf + i);
    }
    __syncthreads();
    if (active) {
      for (int t = 0; t < ch; ++t) {
        const uint32_t* tn = s_nodes + t * nint;
        int idx = 0;
        for (int lv = 0; lv < depth; ++lv) {
          const uint32_t nd = tn[idx];
          const uint32_t cv = codes[(nd & 0xFFFFu) * kTile + tid];
          idx = 2 * idx + 1 + (cv > (nd >> 16) ? 1 : 0);
        }
        const int slot = idx - nint;
        score = fs_add(score, fs_mul(lr, s_leafv[t * nleaf + slot]));
        if (kLeaves) s_lbuf[tid * kChunk + t] = s_leafid[t * nleaf + slot];
      }
    }
    if (kLeaves) {
      __syncthreads();
      for (int i = tid; i < tile_rows * ch; i += kTile) {
        const int c = i / ch, t = i - c * ch;
        leaf_out[job.leaf0 + static_cast<int64_t>(c) * n_trees + t0 + t] = s_lbuf[c * kChunk + t];
      }
    }
  }
  if (active) scores[row0 + tid] = score;
}

// Trees deeper than kMaxHeapDepth: walk the pre-order arrays directly (rare; hand-built models).
__global__ void predict_generic_kernel(const double* __restrict__ x, int64_t rows, int d, int n_trees, double base,
                                       double lr, const int32_t* __restrict__ off, const int32_t* __restrict__ feat,
                                       const double* __restrict__ thr, const int32_t* __restrict__ left,
                                       const int32_t* __restrict__ right, const double* __restrict__ val,
                                       double* __restrict__ scores, uint8_t* __restrict__ leaf_out, uint32_t* err) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const double* xr = x + r * d;
  bool nonfinite = false;
  for (int f = 0; f < d; ++f) nonfinite |= !isfinite(xr[f]);
  if (nonfinite) atomicOr(err, fs::kErrNonFinitePredict);
  double score = base;
  for (int t = 0; t < n_trees; ++t) {
    const int o = off[t];
    int idx = 0;
    while (feat[o + idx] >= 0) idx = xr[feat[o + idx]] <= thr[o + idx] ? left[o + idx] : right[o + idx];
    score = fs_add(score, fs_mul(lr, val[o + idx]));
    if (leaf_out) leaf_out[r * n_trees + t] = static_cast<uint8_t>(idx);
  }
  scores[r] = score;
}

struct HeapGroup {
  std::vector<PredModel> models;
  std::vector<PredJob> jobs;
  int max_dmodel = 0, max_depth = 0, max_uthr = 0;
};

template <typename CodeT, bool kLeaves, bool kSmemThr, bool kFused>
void launch_group(fs_device* dev, const HeapGroup& g, const double* x, int d, double* scores, uint8_t* leaf_out,
                  const SpaceTabs& sp) {
  if (g.jobs.empty()) return;
  const int mnint = (1 << g.max_depth) - 1, mnleaf = 1 << g.max_depth;
  size_t smem = (static_cast<size_t>(g.max_dmodel) * kTile * sizeof(CodeT) + 15) & ~size_t(15);
  smem += static_cast<size_t>(kChunk) * (mnleaf * sizeof(double) + mnint * sizeof(uint32_t) + mnleaf);
  if (kLeaves) smem += static_cast<size_t>(kTile) * kChunk;
  smem = (smem + 15) & ~size_t(15);
  if (kSmemThr) smem += static_cast<size_t>(g.max_uthr) * sizeof(double) + (g.max_dmodel + 1) * sizeof(int32_t);
  auto* fn = predict_heap_kernel<CodeT, kLeaves, kSmemThr, kFused>;
  if (smem > 227 * 1024) fs::fail(FS_EINVAL, "predict: model too wide for the shared-memory tile");
  FS_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const size_t mb = g.models.size() * sizeof(PredModel), jb = g.jobs.size() * sizeof(PredJob);
  auto* buf = static_cast<unsigned char*>(dev->scratch(fs::kSlotPredictSeg, mb + jb + 16));
  auto* md = reinterpret_cast<PredModel*>(buf);
  auto* jd = reinterpret_cast<PredJob*>(buf + ((mb + 15) & ~size_t(15)));
  FS_CUDA(cudaMemcpyAsync(md, g.models.data(), mb, cudaMemcpyHostToDevice, dev->stream));
  FS_CUDA(cudaMemcpyAsync(jd, g.jobs.data(), jb, cudaMemcpyHostToDevice, dev->stream));
  fs::ProfScope prof(dev, kFused ? "score_fused" : "predict");
  fn<<<static_cast<unsigned>(g.jobs.size()), kTile, smem, dev->stream>>>(
      x, d, md, jd, g.max_dmodel, g.max_depth, g.max_uthr, scores, leaf_out, dev->err_d, sp);
  dev->count_launch();
  FS_CUDA(cudaGetLastError());
}

}  // namespace

namespace fs {

// Scores rows [seg[f], seg[f+1]) with family f. Leaf ids of segment f start at byte
// sum_{g<f} rows_g * T_g of leaf_out. All heap-form families go out in one launch (per code width
// / threshold-table placement, normally one); deeper-than-heap models use the generic kernel.
template <bool kFused>
void launch_predict_impl(fs_device* dev, const fs_forest* fo, int32_t nseg, const int64_t* seg, int32_t d,
                         const double* x, double* scores, uint8_t* leaf_out, const SpaceTabs& sp) {
  int64_t leaf_off = 0;
  HeapGroup groups[2][2];  // [code_bytes == 2][thresholds in smem]
  for (int f = 0; f < nseg; ++f) {
    const int64_t r0 = seg[f], rows = seg[f + 1] - seg[f];
    if (f >= static_cast<int32_t>(fo->fams.size())) fail(FS_ERANGE, "predict: segment names an unknown family");
    const auto& m = fo->fams[static_cast<size_t>(f)];
    if (!m.compiled) fail(FS_EINVAL, "predict: family " + std::to_string(f) + " has no compiled model");
    if ((m.fmap_d ? m.d_orig : m.d_model) > d) fail(FS_EINVAL, "predict: model references feature beyond the row width");
    if (leaf_out && m.pending) materialize(dev, m);  // leaf-id layout needs the true tree count
    if (rows <= 0) continue;
    const int64_t lo = leaf_off;
    leaf_off += rows * m.n_trees;
    if (m.generic) {
      if (kFused) fail(FS_EINVAL, "score: fused path needs heap-form models");
      predict_generic_kernel<<<static_cast<int>(ceil_div(rows, 128)), 128, 0, dev->stream>>>(
          x + r0 * d, rows, d, m.n_trees, m.base, m.lr, m.g_off_d, m.g_feat_d, m.g_thr_d, m.g_left_d, m.g_right_d,
          m.g_val_d, scores + r0, leaf_out ? leaf_out + lo : nullptr, dev->err_d);
      dev->count_launch();
      FS_CUDA(cudaGetLastError());
      continue;
    }
    const bool smem_thr = static_cast<size_t>(m.n_uthr) * sizeof(double) <= 48 * 1024;
    HeapGroup& g = groups[m.code_bytes == 2][smem_thr];
    const int mi = static_cast<int>(g.models.size());
    g.models.push_back({m.nodes_d, m.leafv_d, m.leafid_d, m.uthr_d, m.uoff_d, m.base, m.lr, m.depth, m.n_trees,
                        m.fmap_d ? m.d_model : std::min(m.d_model, d), m.n_uthr, m.fmap_d, m.meta_d});
    g.max_dmodel = std::max(g.max_dmodel, m.fmap_d ? m.d_model : std::min(m.d_model, d));
    g.max_depth = std::max(g.max_depth, m.depth);
    g.max_uthr = std::max(g.max_uthr, m.n_uthr);
    for (int64_t t = 0; t < rows; t += kTile)
      g.jobs.push_back({mi, static_cast<int32_t>(std::min<int64_t>(kTile, rows - t)), r0 + t, lo + t * m.n_trees});
  }
  for (int cb = 0; cb < 2; ++cb)
    for (int st = 0; st < 2; ++st) {
      const HeapGroup& g = groups[cb][st];
      if (g.jobs.empty()) continue;
      if (cb == 0) {
        if (leaf_out) st ? launch_group<uint8_t, true, true, kFused>(dev, g, x, d, scores, leaf_out, sp)
                         : launch_group<uint8_t, true, false, kFused>(dev, g, x, d, scores, leaf_out, sp);
        else st ? launch_group<uint8_t, false, true, kFused>(dev, g, x, d, scores, nullptr, sp)
                : launch_group<uint8_t, false, false, kFused>(dev, g, x, d, scores, nullptr, sp);
      } else {
        if (leaf_out) st ? launch_group<uint16_t, true, true, kFused>(dev, g, x, d, scores, leaf_out, sp)
                         : launch_group<uint16_t, true, false, kFused>(dev, g, x, d, scores, leaf_out, sp);
        else st ? launch_group<uint16_t, false, true, kFused>(dev, g, x, d, scores, nullptr, sp)
                : launch_group<uint16_t, false, false, kFused>(dev, g, x, d, scores, nullptr, sp);
      }
    }
}

void launch_predict(fs_device* dev, const fs_forest* fo, int32_t nseg, const int64_t* seg, int32_t d,
                    const double* x, double* scores, uint8_t* leaf_out) {
  launch_predict_impl<false>(dev, fo, nseg, seg, d, x, scores, leaf_out, SpaceTabs{});
}

// Fused featurize -> predict: candidates come as (space id, value indices)
// descriptors; no feature matrix is written or read. pad plays the row width d.
void launch_score_fused(fs_device* dev, const fs_spaces* spc, const fs_forest* fo, int32_t nseg, const int64_t* seg,
                        const int32_t* space_of_d, const int32_t* assign_d, int32_t pad, double* scores) {
  const SpaceTabs sp{space_of_d, assign_d, spc->k_d, spc->nval_d, spc->off_d, spc->log_d, spc->pos_d, spc->n, pad};
  launch_predict_impl<true>(dev, fo, nseg, seg, pad, nullptr, scores, nullptr, sp);
}

int64_t leaf_bytes(const fs_forest* fo, int32_t nseg, const int64_t* seg) {
  int64_t b = 0;
  for (int f = 0; f < nseg && f < static_cast<int32_t>(fo->fams.size()); ++f) {
    materialize(fo->dev, fo->fams[static_cast<size_t>(f)]);
    b += (seg[f + 1] - seg[f]) * fo->fams[static_cast<size_t>(f)].n_trees;
  }
  return b;
}

}  // namespace fs

extern "C" {

int fs_predict_d(fs_device* dev, const fs_forest* fo, int32_t nseg, const int64_t* seg, int32_t d, const double* x_d,
                 double* scores_d, uint8_t* leaf_d) {
  return fs::guard([&] {
    if (!dev || !fo || nseg < 0 || !seg || d < 0) fs::fail(FS_EINVAL, "fs_predict: bad arguments");
    dev->activate();
    fs::launch_predict(dev, fo, nseg, seg, d, x_d, scores_d, leaf_d);
  });
}

int fs_predict(fs_device* dev, const fs_forest* fo, int32_t nseg, const int64_t* seg, int32_t d, const double* x,
               double* scores, uint8_t* leaf_ids) {
  return fs::guard([&] {
    if (!dev || !fo || nseg < 0 || !seg || d < 0) fs::fail(FS_EINVAL, "fs_predict: bad arguments");
    dev->activate();
    const int64_t n = seg[nseg] - seg[0];
    if (n <= 0) return;
    if (seg[0] != 0) fs::fail(FS_EINVAL, "fs_predict: seg[0] must be 0");
    auto* xd = static_cast<double*>(dev->scratch(fs::kSlotH2D0, n * d * sizeof(double)));
    auto* sd = static_cast<double*>(dev->scratch(fs::kSlotD2H0, n * sizeof(double)));
    const int64_t lb = leaf_ids ? fs::leaf_bytes(fo, nseg, seg) : 0;
    auto* ld = leaf_ids ? static_cast<uint8_t*>(dev->scratch(fs::kSlotD2H1, std::max<int64_t>(lb, 1))) : nullptr;
    FS_CUDA(cudaMemcpyAsync(xd, x, n * d * sizeof(double), cudaMemcpyHostToDevice, dev->stream));
    fs::launch_predict(dev, fo, nseg, seg, d, xd, sd, ld);
    FS_CUDA(cudaMemcpyAsync(scores, sd, n * sizeof(double), cudaMemcpyDeviceToHost, dev->stream));
    if (leaf_ids && lb) FS_CUDA(cudaMemcpyAsync(leaf_ids, ld, lb, cudaMemcpyDeviceToHost, dev->stream));
    fs::raise_deferred(dev->take_errors());
  });
}

}  // extern "C"
