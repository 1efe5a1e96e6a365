// Kernel (2): GBDT ensemble predict - predict (costmodel.cpp:237-246) with RegressionTree::eval
// (:135-143) for a whole candidate population; every family segment of a call in ONE launch.
//
// CTA = 256 threads and a tile of TC candidates (TC = 256 .. 32: the host shrinks the tile until
// the launch covers every SM). Per tile:
//   1. Stage codes. Each candidate's tested features become threshold codes in shared memory,
//      row-major [candidate][feature]: code(x) = #{model thresholds of that feature < x}, so
//      `x <= t_rank` <=> `code(x) <= rank` exactly (SURVEY.md "Bit-exactness rules" 2).
//      * predict: the tile's FP64 feature rows stream HBM -> shared memory by bulk async copies
//        (cp.async.bulk, TMA engine, 16 rows per stage, mbarrier-tracked, double-buffered), so
//        the next stage lands while warps code the current one; every feature of every row is
//        checked for finiteness (the reference throws on any, costmodel.cpp:238-240);
//      * score (fused): no feature row exists - a warp per candidate forms
//        every tested feature from the descriptor exactly as featurize does
//        (searchspace.cpp:90-118: log2 / position tables built on the host, pair products one
//        __dmul_rn).
//   2. Warp-cooperative traversal, 32 trees per pass: the pass's trees are staged in shared
//      memory (node words transposed [heap node][tree] so 32 lanes at different nodes never
//      share a bank; lr*leaf precomputed with __dmul_rn), then LANE = TREE: each warp walks its
//      candidates down the 32 trees at once, the top three levels from registers, and records
//      the leaf slot (u8) per (tree, candidate).
//   3. Tree-order fold: thread = candidate adds the 32 leaf values in tree order,
//      score = score + lr*leaf, separately rounded - the reference's
//      `score += learning_rate * tree.eval(x)` without FMA.
// HBM traffic per candidate: 8*d (row) + 8 (score) [+ 2*T leaf ids] for predict, 4*16 + 4 + 8
// for the fused score; the model is read from L2 once per tile.
#include <algorithm>
#include <cstdlib>

#include "forest.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kStageRows = 16;  // rows per bulk-copy stage (predict)
constexpr int kStages = 2;

// One family's compiled ensemble, as the batched kernel sees it.
struct PredModel {
  const uint32_t* nodes;
  const double* leafv;
  const uint16_t* leafid;
  const double* uthr;
  const int32_t* uoff;
  double base, lr;
  int depth, n_trees, d_model, n_uthr;
  const int32_t* fmap;       // compiled feature -> original feature (nullptr: identity)
  const fs::ModelMeta* meta;  // device-compiled fit: n_trees / base live on the device
};

// Candidate descriptors for the fused score path.
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
  const uint64_t* index = nullptr;   // [P] linear_index descriptors (nullptr: assign)
  const uint64_t* stride = nullptr;  // [n_spaces][16]
};

// One CTA's work: a tile of up to TC rows of one family segment.
struct PredJob {
  int32_t model, rows;
  int64_t row0;   // first row (into x / scores)
  int64_t leaf0;  // element offset of row0's leaf ids
};

// Shared-memory carve-up, identical on host and device.
struct Smem {
  size_t codes, nodes, lrleaf, leafid, slots, uthr, uoff, rows, bars, fsrc, total;
  __host__ __device__ static size_t al(size_t o) { return (o + 15) & ~size_t(15); }
  __host__ __device__ Smem(int tc, int ds, int code_bytes, int max_depth, bool leaves, int max_uthr, int max_dmodel,
                           bool smem_thr, int row_doubles, bool fused = false) {
    const size_t mnint = (size_t{1} << max_depth) - 1, mnleaf = size_t{1} << max_depth;
    size_t o = 0;
    codes = o;
    o = al(o + static_cast<size_t>(tc) * ds * code_bytes);
    nodes = o;  // [heap node][32 trees]
    o = al(o + mnint * 32 * 4);
    lrleaf = o;  // [32 trees][leaf]
    o = al(o + 32 * mnleaf * 8);
    leafid = o;
    o = al(o + (leaves ? 32 * mnleaf * 2 : 0));
    slots = o;  // [32 trees][tc + 4]
    o = al(o + 32 * static_cast<size_t>(tc + 4));
    uthr = o;
    o = al(o + (smem_thr ? static_cast<size_t>(max_uthr) * 8 : 0));
    uoff = o;  // per compiled feature: (row column, threshold segment start, length, top step)
    o = al(o + static_cast<size_t>(max_dmodel + 1) * 16);
    rows = o;  // predict: kStages x kStageRows feature rows
    o = al(o + static_cast<size_t>(row_doubles) * 8);
    bars = o;
    o = al(o + kStages * 8);
    fsrc = o;  // fused score: per warp, every model feature's descriptor sources for one knob count
    o = al(o + (fused ? static_cast<size_t>(kWarps) * ds * 4 : 0));
    total = o;
  }
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// TMA-engine bulk copy global -> shared, completion counted on the mbarrier (bytes % 16 == 0).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// kBulk: predict rows arrive by bulk async copies (rows 16-byte aligned, d even); otherwise warps
// read them with coalesced loads.
template <typename CodeT, bool kLeaves, bool kSmemThr, bool kFused, bool kBulk>
__global__ void __launch_bounds__(kThreads) predict_kernel(const double* __restrict__ x, int d,
                                                           const PredModel* __restrict__ models,
                                                           const PredJob* __restrict__ jobs, int tc, int ds,
                                                           int max_dmodel, int max_depth, int max_uthr,
                                                           double* __restrict__ scores, uint16_t* __restrict__ leaf_out,
                                                           uint32_t* err, SpaceTabs sp, int fast) {
  extern __shared__ __align__(16) unsigned char smem[];
  const PredJob job = jobs[blockIdx.x];
  const PredModel M = models[job.model];
  const Smem L(tc, ds, sizeof(CodeT), max_depth, kLeaves, max_uthr, max_dmodel, kSmemThr,
               kFused || !kBulk ? 0 : kStages * kStageRows * d, kFused);
  CodeT* codes = reinterpret_cast<CodeT*>(smem + L.codes);  // [tc][ds]
  uint32_t* s_nodes = reinterpret_cast<uint32_t*>(smem + L.nodes);
  double* s_lrleaf = reinterpret_cast<double*>(smem + L.lrleaf);
  uint16_t* s_leafid = reinterpret_cast<uint16_t*>(smem + L.leafid);
  uint8_t* s_slot = smem + L.slots;
  // depth-3 register walk: every model of the launch has depth 3, u8 codes and rows <= 256 bytes
  const bool kFast = sizeof(CodeT) == 1 && fast != 0;

  const int depth = M.depth, d_model = M.d_model;
  const int n_trees = M.meta ? M.meta->n_trees : M.n_trees;
  const int32_t* fmap = M.fmap;
  const int nint = (1 << depth) - 1, nleaf = 1 << depth;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t row0 = job.row0;
  const int rows = job.rows;

  // threshold tables the codes are searched in: staged in shared memory when they fit
  const double* uthr = M.uthr;
  if (kSmemThr) {
    double* su = reinterpret_cast<double*>(smem + L.uthr);
    for (int i = tid; i < M.n_uthr; i += kThreads) su[i] = __ldg(M.uthr + i);
    uthr = su;
  }
  // per compiled feature f: its row column, its unique-threshold segment [lo, lo + n) and the
  // highest power of two <= n, one 16-byte shared load per code
  int4* s_meta = reinterpret_cast<int4*>(smem + L.uoff);
  for (int f = tid; f < d_model; f += kThreads) {
    const int lo = __ldg(M.uoff + f), n = __ldg(M.uoff + f + 1) - lo;
    s_meta[f] = make_int4(fmap ? __ldg(fmap + f) : f, lo, n, n > 0 ? 1 << (31 - __clz(n)) : 0);
  }
  // code(v) = #{unique thresholds of the feature < v} by branchless binary lifting over the
  // sorted segment (the same step sequence for every value of one feature, so searches of
  // several rows interleave without divergence)
  auto code_of = [&](const int4 m, double v) {
    int pos = 0;
    for (int step = m.w; step > 0; step >>= 1) {
      const int q = pos + step;
      if (q <= m.z && uthr[m.y + q - 1] < v) pos = q;
    }
    return static_cast<CodeT>(pos);
  };

  // ---- 1. codes ---------------------------------------------------------------------------
  if constexpr (kFused) {
    __syncthreads();  // thresholds / feature table staged
    // Warp per TWO candidates (their descriptor loads and code searches interleaved). Lane l
    // holds one table entry per candidate: lanes 0..15 knob l's log2(value), lanes 16..31 knob
    // (l - 16)'s list position (searchspace.cpp:106-109), so a feature is at most two shuffles:
    // log / position = one entry, pair product (:111-116) = entry(i) * entry(j) with one
    // __dmul_rn. Which entries a feature takes depends only on the knob count K: the warp keeps
    // that map for the K it last saw (shared memory, rebuilt when K changes).
    int* wsrc = reinterpret_cast<int*>(smem + L.fsrc) + warp * ds;
    int wk = -1;
    auto build_src = [&](int k) {
      __syncwarp();  // every lane is done with the previous map
      const int dim = 2 * k + k * (k - 1) / 2;
      for (int f = lane; f < d_model; f += 32) {
        const int g = fmap ? __ldg(fmap + f) : f;  // the original feature index
        int a = 0, b = 0, kind = 0;                // 0 zero (padding), 1 one entry, 2 product
        if (g < k) {
          kind = 1;
          a = g;
        } else if (g < 2 * k) {
          kind = 1;
          a = 16 + g - k;
        } else if (g < dim) {
          kind = 2;
          fs::pair_of(k, g - 2 * k, a, b);
        }
        wsrc[f] = kind | a << 2 | b << 8;
      }
      __syncwarp();
      wk = k;
    };
    struct Desc {
      double tab;
      int k;
    };
    auto load_desc = [&](int64_t cand) {  // the candidate's table entry in this lane + its K
      const int s = __ldg(sp.space_of + cand);
      const bool bad_space = s < 0 || s >= sp.n_spaces;
      const int k = bad_space ? 0 : __ldg(sp.k + s);
      const int j = lane & 15;
      double t = 0.0;
      bool bad = false;
      if (j < k) {
        const int m = __ldg(sp.nval + s * FS_MAX_KNOBS + j);
        int a;
        if (sp.index) {  // candidate_from_index (searchspace.cpp:56-66): a_j = (idx / stride_j) % m_j
          const uint64_t idx = __ldg(reinterpret_cast<const unsigned long long*>(sp.index) + cand);
          const uint64_t q = idx / __ldg(reinterpret_cast<const unsigned long long*>(sp.stride) + s * FS_MAX_KNOBS + j);
          a = static_cast<int>(q % static_cast<uint64_t>(m));
        } else {
          a = __ldg(sp.assign + cand * FS_MAX_KNOBS + j);
        }
        if (a < 0 || a >= m) {
          bad = true;
        } else {
          const int off = __ldg(sp.off + s * FS_MAX_KNOBS + j);
          t = lane < 16 ? __ldg(sp.log + off + a) : __ldg(sp.pos + off + a);
        }
      }
      const unsigned any_bad = __ballot_sync(0xffffffffu, bad);
      if (lane == 0) {
        if (bad_space) atomicOr(err, fs::kErrSpaceId);
        if (any_bad) atomicOr(err, fs::kErrKnobRange);
        if (sp.pad < 2 * k + k * (k - 1) / 2) atomicOr(err, fs::kErrPadDim);
      }
      return Desc{t, k};
    };
    auto value = [&](int e, double tab) {
      const int kind = e & 3;
      const double x1 = __shfl_sync(0xffffffffu, tab, (e >> 2) & 63);
      const double x2 = __shfl_sync(0xffffffffu, tab, e >> 8);
      return kind == 0 ? 0.0 : kind == 1 ? x1 : fs_mul(x1, x2);
    };
    for (int c = warp; c < rows; c += 2 * kWarps) {
      const int c2 = c + kWarps;
      const bool two = c2 < rows;
      const Desc A = load_desc(row0 + c);
      const Desc B = two ? load_desc(row0 + c2) : A;
      CodeT* ra = codes + static_cast<size_t>(c) * ds;
      CodeT* rb = codes + static_cast<size_t>(two ? c2 : c) * ds;
      if (A.k == B.k) {
        if (A.k != wk) build_src(A.k);
        for (int fb = 0; fb < d_model; fb += 32) {
          const int f = fb + lane;
          const int e = f < d_model ? wsrc[f] : 0;
          const double va = value(e, A.tab), vb = value(e, B.tab);
          if (f < d_model) {
            const int4 m = s_meta[f];
            int pa = 0, pb = 0;
            for (int step = m.w; step > 0; step >>= 1) {
              const int qa = pa + step, qb = pb + step;
              if (qa <= m.z && uthr[m.y + qa - 1] < va) pa = qa;
              if (qb <= m.z && uthr[m.y + qb - 1] < vb) pb = qb;
            }
            ra[f] = static_cast<CodeT>(pa);
            rb[f] = static_cast<CodeT>(pb);
          }
        }
      } else {  // different knob counts: one candidate after the other
        for (int h = 0; h < 2; ++h) {
          const Desc& D = h ? B : A;
          CodeT* r = h ? rb : ra;
          if (D.k != wk) build_src(D.k);
          for (int fb = 0; fb < d_model; fb += 32) {
            const int f = fb + lane;
            const int e = f < d_model ? wsrc[f] : 0;
            const double v = value(e, D.tab);
            if (f < d_model) r[f] = code_of(s_meta[f], v);
          }
          __syncwarp();
        }
      }
    }
  } else {
    bool nonfinite = false;
    double* rbuf = reinterpret_cast<double*>(smem + L.rows);  // [kStages][kStageRows][d]
    const int nst = (rows + kStageRows - 1) / kStageRows;
    // warp w codes rows ca and (when cb >= 0) cb of a stage held in shared memory at sa / sb: every
    // value checked for finiteness, every model feature coded, the two rows' searches interleaved
    auto code_rows = [&](const double* sa, int ca, const double* sb, int cb) {
      if (!kBulk || (d & 1)) {
        for (int f = lane; f < d; f += 32) nonfinite |= !isfinite(sa[f]) || (cb >= 0 && !isfinite(sb[f]));
      } else {  // 16-byte aligned rows (bulk stages, d even)
        const double2* a2 = reinterpret_cast<const double2*>(sa);
        const double2* b2 = reinterpret_cast<const double2*>(cb >= 0 ? sb : sa);
        for (int f = lane; f < d / 2; f += 32) {
          const double2 u = a2[f], w = b2[f];
          nonfinite |= !isfinite(u.x) || !isfinite(u.y) || !isfinite(w.x) || !isfinite(w.y);
        }
      }
      CodeT* ra = codes + static_cast<size_t>(ca) * ds;
      CodeT* rb = codes + static_cast<size_t>(cb >= 0 ? cb : ca) * ds;
      const double* sb_ = cb >= 0 ? sb : sa;
      for (int f = lane; f < d_model; f += 32) {
        const int4 m = s_meta[f];
        const double va = sa[m.x], vb = sb_[m.x];
        int pa = 0, pb = 0;
        for (int step = m.w; step > 0; step >>= 1) {
          const int qa = pa + step, qb = pb + step;
          if (qa <= m.z && uthr[m.y + qa - 1] < va) pa = qa;
          if (qb <= m.z && uthr[m.y + qb - 1] < vb) pb = qb;
        }
        ra[f] = static_cast<CodeT>(pa);
        rb[f] = static_cast<CodeT>(pb);
      }
    };
    if constexpr (kBulk) {
      uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
      auto issue = [&](int st) {
        const int r0 = st * kStageRows, nr = min(kStageRows, rows - r0);
        const uint32_t bytes = static_cast<uint32_t>(nr) * d * 8;
        uint64_t* bar = bars + (st % kStages);
        mbar_expect_tx(bar, bytes);
        bulk_g2s(rbuf + static_cast<size_t>(st % kStages) * kStageRows * d, x + (row0 + r0) * d, bytes, bar);
      };
      if (tid == 0) {
        for (int b = 0; b < kStages; ++b) mbar_init(bars + b, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int st = 0; st < min(kStages, nst); ++st) issue(st);
      }
      __syncthreads();  // barriers initialised (and staged thresholds visible)
      for (int st = 0; st < nst; ++st) {
        mbar_wait(bars + (st % kStages), static_cast<uint32_t>((st / kStages) & 1));
        const double* buf = rbuf + static_cast<size_t>(st % kStages) * kStageRows * d;
        const int r0 = st * kStageRows, nr = min(kStageRows, rows - r0);
        for (int r = warp; r < nr; r += 2 * kWarps) {
          const int r2 = r + kWarps < nr ? r + kWarps : -1;
          code_rows(buf + static_cast<size_t>(r) * d, r0 + r, r2 >= 0 ? buf + static_cast<size_t>(r2) * d : nullptr,
                    r2 >= 0 ? r0 + r2 : -1);
        }
        __syncthreads();  // every warp is done with this buffer
        if (tid == 0 && st + kStages < nst) issue(st + kStages);
      }
    } else {
      __syncthreads();  // thresholds / feature table staged
      // rows read in place: coalesced finiteness pass, tested columns gathered (L1 hits)
      for (int c = warp; c < rows; c += 2 * kWarps) {
        const int c2 = c + kWarps < rows ? c + kWarps : -1;
        code_rows(x + (row0 + c) * d, c, c2 >= 0 ? x + (row0 + c2) * d : nullptr, c2);
      }
    }
    if (__any_sync(0xffffffffu, nonfinite) && lane == 0) atomicOr(err, fs::kErrNonFinitePredict);
  }

  // ---- 2./3. passes of 32 trees -------------------------------------------------------------
  double score = M.meta ? M.meta->base : M.base;
  const double lr = M.lr;
  // depth <= 3: a pass's tree tables (<= 7 x 32 node words, <= 8 x 32 leaves) are one item per
  // thread, loaded from global memory one pass ahead into registers so the L2 latency hides
  // behind the current pass's walk and fold
  const bool pf = depth <= 3;
  uint32_t pf_node = 0;
  double pf_leaf = 0.0;
  uint16_t pf_id = 0;
  auto prefetch = [&](int tn) {
    const int chn = min(32, n_trees - tn);
    const int h = tid >> 5, t = tid & 31;
    if (h < nint && t < chn) pf_node = __ldg(M.nodes + static_cast<size_t>(tn + t) * nint + h);
    if (tid < chn * nleaf) {
      pf_leaf = __ldg(M.leafv + static_cast<size_t>(tn) * nleaf + tid);
      if (kLeaves) pf_id = __ldg(M.leafid + static_cast<size_t>(tn) * nleaf + tid);
    }
  };
  if (pf && n_trees > 0) prefetch(0);
  for (int t0 = 0; t0 < n_trees; t0 += 32) {
    const int ch = min(32, n_trees - t0);
    __syncthreads();  // codes ready / the previous pass's fold is done with the tree tables
    if (pf) {
      const int h = tid >> 5, t = tid & 31;
      if (h < nint && t < ch) s_nodes[h * 32 + t] = pf_node;  // [node][tree]
      if (tid < ch * nleaf) {
        s_lrleaf[tid] = fs_mul(lr, pf_leaf);
        if (kLeaves) s_leafid[tid] = pf_id;
      }
      if (t0 + 32 < n_trees) prefetch(t0 + 32);
    } else {
      for (int i = tid; i < ch * nint; i += kThreads) {  // [node][tree]
        const int h = i / ch, t = i - h * ch;
        s_nodes[h * 32 + t] = __ldg(M.nodes + static_cast<size_t>(t0 + t) * nint + h);
      }
      for (int i = tid; i < ch * nleaf; i += kThreads) {
        s_lrleaf[i] = fs_mul(lr, __ldg(M.leafv + static_cast<size_t>(t0) * nleaf + i));
        if (kLeaves) s_leafid[i] = __ldg(M.leafid + static_cast<size_t>(t0) * nleaf + i);
      }
    }
    __syncthreads();
    if (lane < ch) {
      // lane = tree: the top three levels' node words live in registers for the whole pass
      const uint32_t w0 = nint > 0 ? s_nodes[lane] : 0u;
      const uint32_t w1 = nint > 1 ? s_nodes[32 + lane] : 0u, w2 = nint > 2 ? s_nodes[64 + lane] : 0u;
      const uint32_t w3 = nint > 3 ? s_nodes[96 + lane] : 0u, w4 = nint > 4 ? s_nodes[128 + lane] : 0u;
      const uint32_t w5 = nint > 5 ? s_nodes[160 + lane] : 0u, w6 = nint > 6 ? s_nodes[192 + lane] : 0u;
      auto walk = [&](const CodeT* r) {
        if (depth == 0) return 0;
        const uint32_t b0 = static_cast<uint32_t>(r[w0 & 0xFFFFu]) > (w0 >> 16);
        if (depth == 1) return static_cast<int>(b0);
        const uint32_t n1 = b0 ? w2 : w1;
        const uint32_t b1 = static_cast<uint32_t>(r[n1 & 0xFFFFu]) > (n1 >> 16);
        if (depth == 2) return static_cast<int>(2 * b0 + b1);
        const uint32_t n2 = b0 ? (b1 ? w6 : w5) : (b1 ? w4 : w3);
        const uint32_t b2 = static_cast<uint32_t>(r[n2 & 0xFFFFu]) > (n2 >> 16);
        int idx = 7 + static_cast<int>(4 * b0 + 2 * b1 + b2);
        for (int lv = 3; lv < depth; ++lv) {
          const uint32_t nd = s_nodes[idx * 32 + lane];
          idx = 2 * idx + 1 + (static_cast<uint32_t>(r[nd & 0xFFFFu]) > (nd >> 16) ? 1 : 0);
        }
        return idx - nint;
      };
      uint8_t* srow = s_slot + lane;  // slots [candidate][32 trees]: lane t writes byte 32c + t
      int c = warp;
      if (kFast) {
        // depth-3 trees, u8 codes, rows of <= 256 bytes: the seven node words become byte-packed
        // (code offset, rank) tables in registers, so a level is one byte-permute select, one
        // shared load and one compare; eight candidates' walks are interleaved level by level
        const uint32_t o0 = w0 & 0xFFu, k0 = w0 >> 16;
        const uint32_t o12 = (w1 & 0xFFu) | (w2 & 0xFFu) << 8, k12 = (w1 >> 16) | (w2 >> 16) << 8;
        const uint32_t o36 = (w3 & 0xFFu) | (w4 & 0xFFu) << 8 | (w5 & 0xFFu) << 16 | (w6 & 0xFFu) << 24;
        const uint32_t k36 = (w3 >> 16) | (w4 >> 16) << 8 | (w5 >> 16) << 16 | (w6 >> 16) << 24;
        const uint32_t cb = smem_u32(codes) + static_cast<uint32_t>(c * ds);
        constexpr int G = 8;
        for (; c + (G - 1) * kWarps < rows; c += G * kWarps) {
          const uint32_t rb = cb + static_cast<uint32_t>((c - warp) * ds);
          uint32_t b0[G], b1[G], v[G];
#pragma unroll
          for (int g = 0; g < G; ++g) v[g] = lds_u8(rb + static_cast<uint32_t>(g * kWarps * ds) + o0);
#pragma unroll
          for (int g = 0; g < G; ++g) {
            b0[g] = v[g] > k0 ? 1u : 0u;
            const uint32_t sel = 0x4440u | b0[g];
            v[g] = lds_u8(rb + static_cast<uint32_t>(g * kWarps * ds) + __byte_perm(o12, 0, sel));
            b1[g] = v[g] > __byte_perm(k12, 0, sel) ? 1u : 0u;
          }
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const uint32_t i = 2 * b0[g] + b1[g], sel = 0x4440u | i;
            v[g] = lds_u8(rb + static_cast<uint32_t>(g * kWarps * ds) + __byte_perm(o36, 0, sel));
            srow[(c + g * kWarps) * 32] = static_cast<uint8_t>(2 * i + (v[g] > __byte_perm(k36, 0, sel) ? 1u : 0u));
          }
        }
      }
      for (; c + 3 * kWarps < rows; c += 4 * kWarps) {  // four independent walks in flight
        const int q0 = walk(codes + static_cast<size_t>(c) * ds);
        const int q1 = walk(codes + static_cast<size_t>(c + kWarps) * ds);
        const int q2 = walk(codes + static_cast<size_t>(c + 2 * kWarps) * ds);
        const int q3 = walk(codes + static_cast<size_t>(c + 3 * kWarps) * ds);
        srow[c * 32] = static_cast<uint8_t>(q0);
        srow[(c + kWarps) * 32] = static_cast<uint8_t>(q1);
        srow[(c + 2 * kWarps) * 32] = static_cast<uint8_t>(q2);
        srow[(c + 3 * kWarps) * 32] = static_cast<uint8_t>(q3);
      }
      for (; c < rows; c += kWarps) srow[c * 32] = static_cast<uint8_t>(walk(codes + static_cast<size_t>(c) * ds));
    }
    __syncthreads();
    if (tid < rows) {  // thread = candidate: tree-order fold of the pass's leaf values
      // the candidate's 32 slots in two 16-byte loads; the leaf loads run ahead of the add chain
      const uint4* s4 = reinterpret_cast<const uint4*>(s_slot + tid * 32);
      const uint4 sa = s4[0], sb = s4[1];
      auto fold4 = [&](uint32_t w, int t) {  // trees t .. t+3, slots in the bytes of w
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (t + u < ch) {
            const int q = static_cast<int>((w >> (8 * u)) & 0xFFu);
            score = fs_add(score, s_lrleaf[(t + u) * nleaf + q]);
            if (kLeaves)
              leaf_out[job.leaf0 + static_cast<int64_t>(tid) * n_trees + t0 + t + u] = s_leafid[(t + u) * nleaf + q];
          }
        }
      };
      fold4(sa.x, 0);
      fold4(sa.y, 4);
      fold4(sa.z, 8);
      fold4(sa.w, 12);
      fold4(sb.x, 16);
      fold4(sb.y, 20);
      fold4(sb.z, 24);
      fold4(sb.w, 28);
    }
  }
  if (tid < rows) scores[row0 + tid] = score;
}

// Trees deeper than kMaxHeapDepth: walk the pre-order arrays directly (rare; hand-built models).
__global__ void predict_generic_kernel(const double* __restrict__ x, int64_t rows, int d, int n_trees, double base,
                                       double lr, const int32_t* __restrict__ off, const int32_t* __restrict__ feat,
                                       const double* __restrict__ thr, const int32_t* __restrict__ left,
                                       const int32_t* __restrict__ right, const double* __restrict__ val,
                                       double* __restrict__ scores, uint16_t* __restrict__ leaf_out, uint32_t* err) {
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
    if (leaf_out) leaf_out[r * n_trees + t] = static_cast<uint16_t>(idx);
  }
  scores[r] = score;
}

struct HeapGroup {
  std::vector<PredModel> models;
  std::vector<int64_t> r0, rows, leaf0;  // per model's segment
  int max_dmodel = 0, max_depth = 0, max_uthr = 0;
  bool all_depth3 = true;
};

template <typename CodeT, bool kLeaves, bool kSmemThr, bool kFused>
void launch_group(fs_device* dev, const HeapGroup& g, const double* x, int d, double* scores, uint16_t* leaf_out,
                  const SpaceTabs& sp) {
  if (g.models.empty()) return;
  // tile: the largest of 256 / 128 / 64 / 32 candidates whose tiles still cover every SM
  int tc = 256;
  if (const char* e = std::getenv("FAMSEER_PREDICT_TC")) tc = std::max(32, std::min(256, std::atoi(e)));  // A/B
  int64_t rows_all = 0;
  for (int64_t r : g.rows) rows_all += r;
  while (tc > 32) {
    int64_t tiles = 0;
    for (int64_t r : g.rows) tiles += fs::ceil_div(r, tc);
    if (tiles >= dev->sm_count) break;
    tc /= 2;
  }
  const int ds = std::max(4, (g.max_dmodel + 3) & ~3);  // row pitch (elements); >= 4 so feature 0 exists
  const bool bulk = !kFused && d > 0 && d % 2 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
                    static_cast<size_t>(kStages) * kStageRows * d * 8 <= 96 * 1024;
  const int row_doubles = bulk ? kStages * kStageRows * d : 0;
  size_t smem = Smem(tc, ds, sizeof(CodeT), g.max_depth, kLeaves, g.max_uthr, g.max_dmodel, kSmemThr, row_doubles, kFused).total;
  while (smem > 227 * 1024 && tc > 32) {
    tc /= 2;
    smem = Smem(tc, ds, sizeof(CodeT), g.max_depth, kLeaves, g.max_uthr, g.max_dmodel, kSmemThr, row_doubles, kFused).total;
  }
  if (smem > 227 * 1024) fs::fail(FS_EINVAL, "predict: model too wide for the shared-memory tile");
  std::vector<PredJob> jobs;
  jobs.reserve(static_cast<size_t>(fs::ceil_div(rows_all, tc)) + g.models.size());
  for (size_t mi = 0; mi < g.models.size(); ++mi) {
    const int T = g.models[mi].n_trees;
    for (int64_t t = 0; t < g.rows[mi]; t += tc)
      jobs.push_back({static_cast<int32_t>(mi), static_cast<int32_t>(std::min<int64_t>(tc, g.rows[mi] - t)),
                      g.r0[mi] + t, g.leaf0[mi] + t * T});
  }
  const size_t mb = g.models.size() * sizeof(PredModel), jb = jobs.size() * sizeof(PredJob);
  auto* buf = static_cast<unsigned char*>(dev->scratch(fs::kSlotPredictSeg, mb + jb + 16));
  auto* md = reinterpret_cast<PredModel*>(buf);
  auto* jd = reinterpret_cast<PredJob*>(buf + ((mb + 15) & ~size_t(15)));
  FS_CUDA(cudaMemcpyAsync(md, g.models.data(), mb, cudaMemcpyHostToDevice, dev->stream));
  FS_CUDA(cudaMemcpyAsync(jd, jobs.data(), jb, cudaMemcpyHostToDevice, dev->stream));
  fs::ProfScope prof(dev, kFused ? "score_fused" : "predict");
  auto launch = [&](auto* fn) {
    FS_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    fn<<<static_cast<unsigned>(jobs.size()), kThreads, smem, dev->stream>>>(
        x, d, md, jd, tc, ds, g.max_dmodel, g.max_depth, g.max_uthr, scores, leaf_out, dev->err_d, sp,
        sizeof(CodeT) == 1 && g.all_depth3 && ds <= 256 ? 1 : 0);
  };
  if (bulk) launch(predict_kernel<CodeT, kLeaves, kSmemThr, kFused, true>);
  else launch(predict_kernel<CodeT, kLeaves, kSmemThr, kFused, false>);
  dev->count_launch();
  FS_CUDA(cudaGetLastError());
}

}  // namespace

namespace fs {

// Scores rows [seg[f], seg[f+1]) with family f. Leaf ids of segment f start at element
// sum_{g<f} rows_g * T_g of leaf_out. All heap-form families go out in one launch (per code width
// / threshold-table placement, normally one); deeper-than-heap models use the generic kernel.
template <bool kFused>
void launch_predict_impl(fs_device* dev, const fs_forest* fo, int32_t nseg, const int64_t* seg, int32_t d,
                         const double* x, double* scores, uint16_t* leaf_out, const SpaceTabs& sp) {
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
      if (leaf_out)
        for (int t = 0; t < m.num_trees(); ++t)
          if (m.offsets[static_cast<size_t>(t) + 1] - m.offsets[static_cast<size_t>(t)] > 65536)
            fail(FS_EINVAL, "predict: leaf ids are uint16; a tree holds more than 65,536 nodes");
      predict_generic_kernel<<<static_cast<int>(ceil_div(rows, 128)), 128, 0, dev->stream>>>(
          x + r0 * d, rows, d, m.n_trees, m.base, m.lr, m.g_off_d, m.g_feat_d, m.g_thr_d, m.g_left_d, m.g_right_d,
          m.g_val_d, scores + r0, leaf_out ? leaf_out + lo : nullptr, dev->err_d);
      dev->count_launch();
      FS_CUDA(cudaGetLastError());
      continue;
    }
    const bool smem_thr = static_cast<size_t>(m.n_uthr) * sizeof(double) <= 48 * 1024;
    HeapGroup& g = groups[m.code_bytes == 2][smem_thr];
    const int dm = m.fmap_d ? m.d_model : std::min(m.d_model, d);
    g.models.push_back({m.nodes_d, m.leafv_d, m.leafid_d, m.uthr_d, m.uoff_d, m.base, m.lr, m.depth, m.n_trees, dm,
                        m.n_uthr, m.fmap_d, m.meta_d});
    g.r0.push_back(r0);
    g.rows.push_back(rows);
    g.leaf0.push_back(lo);
    g.max_dmodel = std::max(g.max_dmodel, dm);
    g.max_depth = std::max(g.max_depth, m.depth);
    g.all_depth3 = g.all_depth3 && m.depth == 3;
    g.max_uthr = std::max(g.max_uthr, m.n_uthr);
  }
  for (int cb = 0; cb < 2; ++cb)
    for (int st = 0; st < 2; ++st) {
      const HeapGroup& g = groups[cb][st];
      if (g.models.empty()) continue;
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
                    const double* x, double* scores, uint16_t* leaf_out) {
  launch_predict_impl<false>(dev, fo, nseg, seg, d, x, scores, leaf_out, SpaceTabs{});
}

// Fused featurize -> predict: candidates come as (space id, value indices)
// descriptors; no feature matrix is written or read. pad plays the row width d.
void launch_score_fused(fs_device* dev, const fs_spaces* spc, const fs_forest* fo, int32_t nseg, const int64_t* seg,
                        const int32_t* space_of_d, const int32_t* assign_d, int32_t pad, double* scores,
                        const uint64_t* index_d) {
  const SpaceTabs sp{space_of_d, assign_d, spc->k_d, spc->nval_d, spc->off_d, spc->log_d,
                     spc->pos_d, spc->n,   pad,      index_d,     spc->stride_d};
  launch_predict_impl<true>(dev, fo, nseg, seg, pad, nullptr, scores, nullptr, sp);
}

int64_t leaf_count(const fs_forest* fo, int32_t nseg, const int64_t* seg) {
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
                 double* scores_d, uint16_t* leaf_d) {
  return fs::guard([&] {
    if (!dev || !fo || nseg < 0 || !seg || d < 0) fs::fail(FS_EINVAL, "fs_predict: bad arguments");
    dev->activate();
    fs::launch_predict(dev, fo, nseg, seg, d, x_d, scores_d, leaf_d);
  });
}

int fs_predict(fs_device* dev, const fs_forest* fo, int32_t nseg, const int64_t* seg, int32_t d, const double* x,
               double* scores, uint16_t* leaf_ids) {
  return fs::guard([&] {
    if (!dev || !fo || nseg < 0 || !seg || d < 0) fs::fail(FS_EINVAL, "fs_predict: bad arguments");
    dev->activate();
    const int64_t n = seg[nseg] - seg[0];
    if (n <= 0) return;
    if (seg[0] != 0) fs::fail(FS_EINVAL, "fs_predict: seg[0] must be 0");
    auto* xd = static_cast<double*>(dev->scratch(fs::kSlotH2D0, n * d * sizeof(double)));
    auto* sd = static_cast<double*>(dev->scratch(fs::kSlotD2H0, n * sizeof(double)));
    const int64_t lc = leaf_ids ? fs::leaf_count(fo, nseg, seg) : 0;
    auto* ld = leaf_ids ? static_cast<uint16_t*>(dev->scratch(fs::kSlotD2H1, std::max<int64_t>(lc, 1) * 2)) : nullptr;
    FS_CUDA(cudaMemcpyAsync(xd, x, n * d * sizeof(double), cudaMemcpyHostToDevice, dev->stream));
    fs::launch_predict(dev, fo, nseg, seg, d, xd, sd, ld);
    FS_CUDA(cudaMemcpyAsync(scores, sd, n * sizeof(double), cudaMemcpyDeviceToHost, dev->stream));
    if (leaf_ids && lc) FS_CUDA(cudaMemcpyAsync(leaf_ids, ld, lc * 2, cudaMemcpyDeviceToHost, dev->stream));
    fs::raise_deferred(dev->take_errors());
  });
}

}  // extern "C"
