// fit_epilogue.cuh - the device-side fit epilogue: pre-order export + compiled predict form
// Part of the trainer translation unit: included once, by fit.cu only (shares its
// anonymous namespace, constants and helpers).
#pragma once


namespace fs {
namespace fit {
namespace {

constexpr int kCompileSlots = 255;  // heap slots of a depth-7 tree (device compile limit)

// ==========================================================================================
// fit epilogue on the device: per family, the reference pre-order export of every tree
// (costmodel.cpp:82-83 node numbering, :108-111 left before right) and the compiled predict form
// (forest.cuh: complete heap of the family's depth, node = rep | bin << 16 where bin is the
// threshold's rank among the rep's distinct values, early leaves replicated under always-left
// nodes), written straight into the family's model blob - no host round trip after a fit.
// Compiled features are representatives; fmap maps them back to original feature ids.
// ==========================================================================================
struct ExportJob {
  unsigned char* blob;
  DevLayout lay;
  int depth;      // heap depth of the compiled form (the family's tree depth)
  int code_wide;  // codes are u16 (always-left rank 0xFFFF instead of 0xFF)
};

__global__ void __launch_bounds__(128) export_compile_kernel(
    const FamDesc* __restrict__ fam, const FamState* __restrict__ st, const TreeRec* __restrict__ trees,
    int slots, const double* __restrict__ mse, int max_trees, const double* __restrict__ base,
    const int32_t* __restrict__ rep_orig, const int32_t* __restrict__ rep_boff, const double* __restrict__ vals,
    const ExportJob* __restrict__ jobs) {
  const int f = blockIdx.x;
  const FamDesc fd = fam[f];
  const ExportJob jb = jobs[f];
  const DevLayout& L = jb.lay;
  unsigned char* B = jb.blob;
  const int T = fd.n > 0 ? st[f].ntrees : 0;
  if (threadIdx.x == 0) {
    ModelMeta mt;
    mt.base = fd.n > 0 ? base[f] : 0.0;
    mt.n_trees = T;
    mt.pad_ = 0;
    mt.screened = static_cast<int64_t>(st[f].screened);
    mt.exact = static_cast<int64_t>(st[f].exact);
    *reinterpret_cast<ModelMeta*>(B + L.meta) = mt;
  }
  double* uthr = reinterpret_cast<double*>(B + L.uthr);
  int32_t* uoff = reinterpret_cast<int32_t*>(B + L.uoff);
  int32_t* fmap = reinterpret_cast<int32_t*>(B + L.fmap);
  for (int b = threadIdx.x; b < fd.bins; b += blockDim.x) uthr[b] = vals[fd.bin0 + b];
  for (int j = threadIdx.x; j <= fd.nrep; j += blockDim.x) {
    uoff[j] = j < fd.nrep ? rep_boff[fd.rep0 + j] : fd.bins;
    if (j < fd.nrep) fmap[j] = rep_orig[fd.rep0 + j];
  }
  const int D = jb.depth, nint = (1 << D) - 1, nleaf = 1 << D, S = L.slots;
  const uint32_t always_left = jb.code_wide ? 0xFFFFu : 0xFFu;
  uint32_t* nodes = reinterpret_cast<uint32_t*>(B + L.nodes);
  double* leafv = reinterpret_cast<double*>(B + L.leafv);
  uint16_t* leafid = reinterpret_cast<uint16_t*>(B + L.leafid);
  int32_t* cnt = reinterpret_cast<int32_t*>(B + L.cnt);
  int32_t* feat = reinterpret_cast<int32_t*>(B + L.feat);
  double* thr = reinterpret_cast<double*>(B + L.thr);
  int32_t* lft = reinterpret_cast<int32_t*>(B + L.left);
  int32_t* rgt = reinterpret_cast<int32_t*>(B + L.right);
  double* val = reinterpret_cast<double*>(B + L.val);
  double* gain = reinterpret_cast<double*>(B + L.gain);
  double* mo = reinterpret_cast<double*>(B + L.mse);
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    mo[t] = mse[static_cast<int64_t>(f) * max_trees + t];
    const TreeRec* rec = trees + fd.tree0 + static_cast<int64_t>(t) * slots;
    // subtree sizes bottom-up over the heap slots, then pre-order indices top-down
    int size[kCompileSlots], pidx[kCompileSlots];
    for (int h = S - 1; h >= 0; --h) {
      size[h] = 0;
      if (rec[h].kind == kNodeLeaf) size[h] = 1;
      else if (rec[h].kind == kNodeSplit) size[h] = 1 + size[2 * h + 1] + size[2 * h + 2];
    }
    for (int h = 0; h < S; ++h) pidx[h] = -1;
    pidx[0] = 0;
    const size_t o = static_cast<size_t>(t) * S;
    for (int h = 0; h < S; ++h) {  // parents precede children in heap order
      const int i = pidx[h];
      if (i < 0) continue;
      const TreeRec& r = rec[h];
      const bool sp = r.kind == kNodeSplit;
      feat[o + i] = sp ? r.feature : -1;
      thr[o + i] = sp ? r.threshold : 0.0;
      val[o + i] = sp ? 0.0 : r.value;
      gain[o + i] = sp ? r.gain : 0.0;
      lft[o + i] = -1;
      rgt[o + i] = -1;
      if (sp) {
        pidx[2 * h + 1] = i + 1;
        pidx[2 * h + 2] = i + 1 + size[2 * h + 1];
        lft[o + i] = i + 1;
        rgt[o + i] = i + 1 + size[2 * h + 1];
      }
    }
    cnt[t] = size[0];
    // compiled heap
    for (int h = 0; h < nint; ++h) {
      const TreeRec& r = rec[h];
      nodes[static_cast<size_t>(t) * nint + h] =
          r.kind == kNodeSplit ? static_cast<uint32_t>(r.rep) | (static_cast<uint32_t>(r.bin) << 16) : always_left << 16;
    }
    for (int q = 0; q < nleaf; ++q) {
      int h = nint + q;  // deepest existing ancestor-or-self is the leaf covering this heap leaf
      while (h > 0 && rec[h].kind == 0) h = (h - 1) >> 1;
      leafv[static_cast<size_t>(t) * nleaf + q] = rec[h].value;
      leafid[static_cast<size_t>(t) * nleaf + q] = static_cast<uint16_t>(pidx[h]);
    }
  }
}

}  // namespace
}  // namespace fit
}  // namespace fs
