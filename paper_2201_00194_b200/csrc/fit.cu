// Kernel (3): the boosting trainer - fit (costmodel.cpp:152-222) for F families in one call.
// Design and bit-exactness argument: fit.cuh. Phases:
//   prep    distinct values + codes per feature, feature dedup, canonical row order
//           (costmodel.cpp:161-173), per-feature presorts (:193-201), base (:185-188)
//   rounds  residual -> fixed point -> per level: histograms (smaller child built, sibling by
//           exact subtraction), screen, exact reference-order re-evaluation where needed,
//           stable partition of the order-0 list -> leaves (reference-order totals) ->
//           prediction update -> commit / early stop (:212) -> MSE (:215-220)
// The host only launches; no host<->device synchronisation happens inside the boosting loop.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <climits>
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <numeric>
#include <vector>

#include "fit.cuh"
#include "fold_est.cuh"

namespace fs {
void launch_featurize(fs_device* dev, const fs_spaces* sp, int64_t n, const int32_t* space_of_d,
                      const int32_t* assign_d, int32_t pad, double* out_d);
}  // namespace fs

#include "fit_prep.cuh"
#include "fit_round.cuh"
#include "fit_resident.cuh"
#include "fit_epilogue.cuh"


// ==========================================================================================
// host orchestration
// ==========================================================================================
namespace fs {
namespace fit {
namespace {

struct Arena {  // stream-ordered scratch owned by one fit call
  cudaStream_t s;
  std::vector<void*> ptrs;
  explicit Arena(cudaStream_t st) : s(st) {}
  template <class T>
  T* alloc(size_t count) {
    void* p = nullptr;
    FS_CUDA(cudaMallocAsync(&p, std::max<size_t>(count, 1) * sizeof(T), s));
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  template <class T>
  T* upload(const std::vector<T>& v) {
    T* p = alloc<T>(v.size());
    if (!v.empty()) FS_CUDA(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
    return p;
  }
  ~Arena() {
    for (void* p : ptrs) cudaFreeAsync(p, s);
  }
};

template <class T>
std::vector<T> download(const T* d, size_t n, cudaStream_t s) {
  std::vector<T> h(n);
  if (n) FS_CUDA(cudaMemcpyAsync(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, s));
  FS_CUDA(cudaStreamSynchronize(s));
  return h;
}

// Several device->host reads with ONE stream synchronization: async copies into the device's
// pinned staging buffer (plus the deferred-error word), one sync, then unpack. Returns the
// error bits (see fs_device::take_errors).
struct BatchRead {
  struct Item {
    const void* src;
    void* dst;
    size_t bytes;
  };
  std::vector<Item> items;
  template <class T>
  void add(const T* d, std::vector<T>& h, size_t n) {
    h.resize(n);
    if (n) items.push_back({d, h.data(), n * sizeof(T)});
  }
  uint32_t run(fs_device* dev) {
    size_t total = 16;
    for (const auto& it : items) total += (it.bytes + 15) & ~size_t(15);
    auto* st = static_cast<unsigned char*>(dev->pinned(total));
    size_t o = 16;
    FS_CUDA(cudaMemcpyAsync(st, dev->err_d, sizeof(uint32_t), cudaMemcpyDeviceToHost, dev->stream));
    for (const auto& it : items) {
      FS_CUDA(cudaMemcpyAsync(st + o, it.src, it.bytes, cudaMemcpyDeviceToHost, dev->stream));
      o += (it.bytes + 15) & ~size_t(15);
    }
    FS_CUDA(cudaStreamSynchronize(dev->stream));
    o = 16;
    for (const auto& it : items) {
      std::memcpy(it.dst, st + o, it.bytes);
      o += (it.bytes + 15) & ~size_t(15);
    }
    uint32_t bits;
    std::memcpy(&bits, st, sizeof bits);
    if (bits) FS_CUDA(cudaMemsetAsync(dev->err_d, 0, sizeof(uint32_t), dev->stream));
    return bits;
  }
};

inline unsigned grid1(int64_t n, int block, int cap) {
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, block), cap)));
}

// A boosting round's kernels go out with programmatic stream serialization (PDL): the next kernel
// is scheduled while its predecessor drains and waits in FS_PDL_WAIT() for its completion, which
// hides the launch gap between the round's ~40 small dependent kernels (inside the CUDA graph the
// dependencies become programmatic edges). FAMSEER_NO_PDL=1 launches them plainly.
template <class... KArgs, class... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  const bool off = std::getenv("FAMSEER_NO_PDL") != nullptr;  // read per launch (a test toggles it)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = off ? 0 : 1;
  FS_CUDA(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
}

struct ResidentPlan {
  bool enabled = false;
  std::vector<int> families;
  size_t smem = 0;
  bool pred_smem = false;
  bool pre_smem = false;
  int spec_bufs = 0;  // warps with a speculative exact-fold member buffer
  int cluster = 1;    // CTAs per family (thread-block cluster sharing the histogram work)
  // column-layout histogram plan for the multi-kernel path (hist_build_col_kernel)
  bool atomic = false;  // limb-atomic histogram (default)
  int colh_max = 1;     // its lane-column height (col_height), max over families
  size_t phi_smem = 0;  // tie-class phi table bytes (largest per-feature bin count x 2); 0 = ordered scan
  std::vector<int> bitonic_ok;  // per family: 1 = canonical order by one bitonic sort, 2 = given (fs_store), 0 = LSD passes
  size_t bitonic_smem = 0;
  std::vector<int> canon_io;    // per family: FitRows::io (empty: none)
  int32_t* store_canon = nullptr;
  size_t atomic_smem = 0;
  bool col = false;
  std::vector<int32_t> col_off;  // [F][kColWarps + 1] entry offsets per feature group
  std::vector<int32_t> col_rg;   // [F] row groups (private copies)
  size_t col_smem = 0;
};

template <typename CodeT>
void run_rounds(const ResidentPlan& resident, fs_device* dev, Arena& ar, int F, int d, int Dp, int64_t n_tot,
                int max_trees, int depth_max,
                int slots, int nrep_max, int max_bins, int n_max, int level_slots_max, const FamDesc* fam_d,
                FamState* st_d, const double* x_d, const double* target_d, const uint16_t* codes_all,
                const int32_t* rep_orig_d, const int32_t* rep_nb_d, const int32_t* rep_boff_d, const double* vals_d,
                int64_t total_ord, int64_t total_bins, int64_t total_hist, int64_t total_lbuf, int64_t total_tree,
                TreeRec* trees_d, double* mse_d, double* base_d, int min_nrep_hint) {
  cudaStream_t s = dev->stream;
  const int sm = dev->sm_count;
  const size_t bitonic_smem = resident.bitonic_smem;
  const bool have_io = !resident.canon_io.empty();
  const int* bitonic_ok = bitonic_smem > 0 || have_io ? ar.upload(resident.bitonic_ok) : nullptr;
  if (bitonic_smem > 0)
    FS_CUDA(cudaFuncSetAttribute(canonical_bitonic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(bitonic_smem)));
  // rows per histogram CTA: kAtomChunk, shrunk (multiples of kAtomTile) until the root level
  // alone launches >= 2 CTAs per SM - a few large families otherwise leave most SMs idle
  int atom_chunk = kAtomChunk;
  while (atom_chunk > 2 * kAtomTile && static_cast<int64_t>(ceil_div(n_max, atom_chunk)) * F < 2LL * sm)
    atom_chunk /= 2;
  // ---- prep: canonical order, gather, presorts, bin counts, base -------------------------
  int32_t* canon = ar.alloc<int32_t>(n_tot);
  int32_t* tmp = ar.alloc<int32_t>(std::max<int64_t>(n_tot, total_ord));
  {
    ProfScope prof(dev, "fit_canonical");
    if (bitonic_smem > 0) {
      canonical_bitonic_kernel<<<F, kSortThreads, bitonic_smem, s>>>(target_d, codes_all, d, fam_d, rep_orig_d,
                                                                     rep_nb_d, bitonic_ok, canon);
      dev->count_launch();
    }
    canonical_kernel<<<F, kSortThreads, 0, s>>>(target_d, codes_all, d, fam_d, rep_orig_d, rep_nb_d, canon, tmp,
                                                bitonic_ok);
    if (have_io) {
      const int* io_d = ar.upload(resident.canon_io);
      canon_io_kernel<<<grid1(n_tot, 256, sm * 8), 256, 0, s>>>(fam_d, F, n_tot, io_d, resident.store_canon, canon);
      dev->count_launch();
    }
  }
  CodeT* codes_c = ar.alloc<CodeT>(static_cast<size_t>(n_tot) * Dp);
  double* target_c = ar.alloc<double>(n_tot);
  int32_t* rowfam = ar.alloc<int32_t>(n_tot);
  gather_canonical_kernel<CodeT><<<grid1(n_tot, 256, sm * 16), 256, 0, s>>>(
      target_d, codes_all, d, fam_d, F, n_tot, rep_orig_d, canon, Dp, codes_c, target_c, rowfam);
  int32_t* ord = ar.alloc<int32_t>(total_ord);
  if (nrep_max > 0) {
    ProfScope prof(dev, "fit_presort");
    presort_kernel<CodeT><<<dim3(nrep_max, F), kSortThreads, 0, s>>>(fam_d, Dp, codes_c, rep_nb_d, ord, tmp);
  }
  int32_t* cle = ar.alloc<int32_t>(total_bins);
  FS_CUDA(cudaMemsetAsync(cle, 0, std::max<int64_t>(total_bins, 1) * sizeof(int32_t), s));
  bin_count_kernel<CodeT><<<grid1(n_tot, 256, sm * 16), 256, 0, s>>>(fam_d, F, n_tot, Dp, codes_c, rowfam, rep_boff_d, cle);
  bin_prefix_kernel<<<F, 128, 0, s>>>(fam_d, rep_boff_d, rep_nb_d, cle);
  double* pred = ar.alloc<double>(n_tot);
  int32_t* ord_root = ar.alloc<int32_t>(n_tot);
  base_kernel<<<F, 256, 0, s>>>(fam_d, target_c, base_d, pred, ord, ord_root);
  dev->count_launch(8);
  FS_CUDA(cudaGetLastError());

  // ---- resident path: every family fits one CTA's shared memory -> one launch, all rounds ----
  if (std::is_same<CodeT, uint8_t>::value && resident.enabled) {
    int* list_d = ar.upload(resident.families);
    // every round's e = target - pred, [rounds][n] per family, for the exact MSE fold afterwards
    double* ebuf = ar.alloc<double>(static_cast<size_t>(n_tot) * std::max(max_trees, 1));
    auto* kfn = resident.cluster > 1 ? fit_resident_kernel<true> : fit_resident_kernel<false>;
    FS_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(resident.smem)));
    {
      ProfScope prof(dev, "fit_resident");
      const int cl = resident.cluster;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(static_cast<unsigned>(resident.families.size() * cl));
      cfg.blockDim = dim3(kResThreads);
      cfg.dynamicSmemBytes = resident.smem;
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = static_cast<unsigned>(cl);
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = cl > 1 ? 1 : 0;  // no cluster attribute for one CTA per family
      FS_CUDA(cudaLaunchKernelEx(&cfg, kfn, static_cast<const FamDesc*>(fam_d), st_d,
                                 static_cast<const int*>(list_d), Dp, reinterpret_cast<const uint8_t*>(codes_c),
                                 static_cast<const double*>(target_c), static_cast<const double*>(base_d),
                                 static_cast<const int32_t*>(ord), static_cast<const int32_t*>(ord_root),
                                 rep_orig_d, rep_nb_d, rep_boff_d, static_cast<const double*>(vals_d),
                                 static_cast<const int32_t*>(cle), static_cast<const int32_t*>(canon), x_d, d, trees_d,
                                 ebuf, max_trees, slots, dev->ctr_d, resident.pred_smem ? 1 : 0, pred,
                                 resident.pre_smem ? 1 : 0, resident.spec_bufs));
    }
    dev->count_launch();
    FS_CUDA(cudaGetLastError());
    if (max_trees > 0) {
      const int64_t chains = static_cast<int64_t>(F) * max_trees;
      ProfScope prof(dev, "fit_mse");
      mse_fold_kernel<<<static_cast<unsigned>(ceil_div(chains, 4)), 128, 0, s>>>(fam_d, st_d, F, ebuf, max_trees, 0, 0,
                                                                                 max_trees, mse_d, max_trees);
      dev->count_launch();
      FS_CUDA(cudaGetLastError());
    }
    return;
  }

  // ---- round state ---------------------------------------------------------------------
  double* resid = ar.alloc<double>(n_tot);
  int64_t* rfix = ar.alloc<int64_t>(n_tot);
  int32_t* ord_cur = ar.alloc<int32_t>(n_tot);
  int32_t* scratch = ar.alloc<int32_t>(n_tot);
  int16_t* nodeid = ar.alloc<int16_t>(n_tot);
  NodeRec* nodes = ar.alloc<NodeRec>(static_cast<size_t>(F) * slots);
  int64_t* node_abs = ar.alloc<int64_t>(static_cast<size_t>(F) * slots);
  int64_t* hsum = ar.alloc<int64_t>(total_hist);
  int32_t* hcnt = ar.alloc<int32_t>(total_hist);
  // screen pass 0's per-candidate (gain, bound) and left count, read by pass 1 (same cells)
  double2* scr_gd = ar.alloc<double2>(total_hist);
  int32_t* scr_ic = ar.alloc<int32_t>(total_hist);
  double* lbuf = ar.alloc<double>(total_lbuf);
  WinRec* win = ar.alloc<WinRec>(static_cast<size_t>(F) * level_slots_max * std::max(nrep_max, 1));
  ExactItem* items = ar.alloc<ExactItem>(static_cast<size_t>(F) * level_slots_max * (nrep_max + 1));
  int* n_items = ar.alloc<int>(2);  // [0] tie-class items, [1] exact items (zeroed by level_prep_kernel)
  (void)total_tree;
  // column-major codes (the presorted lists' layout) for the kernels that read one feature's code
  // of scattered rows: tie classes, exact folds, partition
  CodeT* codes_cm = ar.alloc<CodeT>(static_cast<size_t>(std::max<int64_t>(total_ord, 1)));
  if (total_ord > 0) {
    const size_t tsm = static_cast<size_t>(128) * (Dp + 1) * sizeof(CodeT);
    FS_CUDA(cudaFuncSetAttribute(codes_colmajor_kernel<CodeT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(tsm)));
    codes_colmajor_kernel<CodeT><<<dim3(static_cast<unsigned>(ceil_div(n_max, 128)), F), 256, tsm, s>>>(
        fam_d, Dp, codes_c, codes_cm);
    dev->count_launch();
    FS_CUDA(cudaGetLastError());
  }

  // histogram launch shape
  const int per_group_min = std::max(1, std::min(min_nrep_hint, kHistThreads));
  const size_t tile_bytes = ((static_cast<size_t>(kHistTileRows) * Dp * sizeof(CodeT) + 15) & ~size_t(15)) +
                            kHistTileRows * sizeof(int64_t) + 64;
  const size_t smem_cap = 200 * 1024;
  int groups = std::max(1, kHistThreads / std::max(1, std::min(nrep_max, kHistThreads)));
  (void)per_group_min;
  while (groups > 1 && static_cast<size_t>(groups) * max_bins * 12 + tile_bytes > smem_cap) --groups;
  const bool hist_global = static_cast<size_t>(max_bins) * 12 + tile_bytes > smem_cap;
  const size_t hist_smem = hist_global ? tile_bytes + 16 : ((static_cast<size_t>(groups) * max_bins * 12 + 15) & ~size_t(15)) + tile_bytes;
  if (hist_global) {
    FS_CUDA(cudaFuncSetAttribute(hist_build_kernel<CodeT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(hist_smem)));
  } else {
    FS_CUDA(cudaFuncSetAttribute(hist_build_kernel<CodeT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(hist_smem)));
  }
  const unsigned chunks = static_cast<unsigned>(std::max<int64_t>(1, ceil_div(n_max, kHistChunk)));
  int32_t* col_off_d = nullptr;
  int32_t* col_rg_d = nullptr;
  if (resident.phi_smem > 0)
    FS_CUDA(cudaFuncSetAttribute(tieclass_phi_kernel<CodeT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(resident.phi_smem)));
  if (resident.atomic) {
    FS_CUDA(cudaFuncSetAttribute(hist_build_atomic_kernel<CodeT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(resident.atomic_smem)));
    FS_CUDA(cudaFuncSetAttribute(hist_build_atomic_kernel<CodeT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(resident.atomic_smem)));
  }
  if (resident.col) {
    col_off_d = ar.upload(resident.col_off);
    col_rg_d = ar.upload(resident.col_rg);
    FS_CUDA(cudaFuncSetAttribute(hist_build_col_kernel<CodeT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(resident.col_smem)));
  }

  // One boosting round = a fixed launch sequence whose arguments never change (the round index
  // lives on the device in FamState::ntrees), so it is captured once as a CUDA graph and replayed
  // max_trees times; families that stopped early skip their work inside the kernels.
  const int64_t l0 = dev->launches;
  // train_mse_by_round: ring of K rounds of e = target - pred, folded every K rounds (mse_fold_kernel)
  const int mse_k = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>(std::min(max_trees, 64), (int64_t{1} << 30) / std::max<int64_t>(1, n_tot * 8))));
  double* ebuf = ar.alloc<double>(static_cast<size_t>(mse_k) * n_tot);
  const bool fork_totals = std::getenv("FAMSEER_FORK_TOTALS") != nullptr;
  // chunked partition: left-row count per (family, node at level, 1,024-row chunk)
  const int part_chunks = static_cast<int>(std::max<int64_t>(1, ceil_div(n_max, kPartChunk)));
  int32_t* part_cnt = ar.alloc<int32_t>(static_cast<size_t>(F) * level_slots_max * part_chunks);
  // small-node exact folds (exact_small_kernel): per-CTA scratch of two n_max index buffers
  int32_t* small_scratch = std::getenv("FAMSEER_EXACT_SCAN")
                               ? nullptr
                               : ar.alloc<int32_t>(static_cast<size_t>(kExactSmallCtas) * 2 * std::max(n_max, 1));
  if (small_scratch)
    FS_CUDA(cudaFuncSetAttribute(exact_small_kernel<CodeT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(exact_small_smem<CodeT>())));
  cudaStream_t aux = fork_totals ? dev->aux_stream() : nullptr;
  auto round_body = [&]() {
    launch_pdl(round_init_kernel, dim3(F), dim3(256), 0, s, fam_d, st_d, nodes, slots, trees_d, node_abs);
    launch_pdl(residual_kernel, dim3(grid1(n_tot, 256, sm * 16)), dim3(256), 0, s, fam_d, F, n_tot, st_d, rowfam,
               target_c, pred, resid, ord_root, ord_cur, nodeid);
    launch_pdl(fixed_kernel, dim3(grid1(n_tot, 256, sm * 16)), dim3(256), 0, s, fam_d, n_tot, st_d, rowfam, resid, rfix);
    dev->count_launch(3);
    for (int level = 0; level <= depth_max; ++level) {
      const unsigned lw = 1u << level;
      if (level == depth_max || nrep_max == 0) {
        launch_pdl(level_plan_kernel, dim3(grid1(lw, 128, 1 << 20), F), dim3(128), 0, s, fam_d, st_d, nodes, level);
        dev->count_launch();
        continue;
      }
      // the level's plan, zeroed histogram slots and work-list counters
      launch_pdl(level_prep_kernel, dim3(grid1(static_cast<int64_t>(lw) * max_bins, 256, 64), F), dim3(256), 0, s,
                 fam_d, st_d, nodes, level, hsum, hcnt, n_items);
      dev->count_launch();
      // Optional fork (FAMSEER_FORK_TOTALS=1): every screened node's total on a side stream while
      // this level's histogram..decide kernels run; joined before the exact folds. Measured
      // slower at C4 (the root chain outlasts the level's other kernels and the join then
      // stalls every level, exact or not), so the totals are folded only for exact nodes.
      if (fork_totals) {
        FS_CUDA(cudaEventRecord(dev->ev_fork, s));
        FS_CUDA(cudaStreamWaitEvent(aux, dev->ev_fork, 0));
        totals_kernel<<<dim3(grid1(lw, 4, 1 << 20), F), 128, 0, aux>>>(fam_d, st_d, nodes, level, ord_cur, resid);
        FS_CUDA(cudaEventRecord(dev->ev_join, aux));
        dev->count_launch();
      }
      const unsigned pairs = level == 0 ? 1u : (1u << (level - 1));
      {
        ProfScope prof(dev, "fit_hist_build");
        if (resident.atomic) {
          const dim3 grid(static_cast<unsigned>(ceil_div(n_max, atom_chunk)), pairs, F);
          if (atom_chunk >= kAtomPipeChunk)
            launch_pdl(hist_build_atomic_kernel<CodeT, true>, grid, dim3(kAtomThreads), resident.atomic_smem, s, fam_d,
                       st_d, nodes, level, Dp, codes_c, rfix, ord_cur, rep_boff_d, hsum, hcnt, node_abs, dev->ctr_d,
                       resident.colh_max, atom_chunk);
          else
            launch_pdl(hist_build_atomic_kernel<CodeT, false>, grid, dim3(kAtomThreads), resident.atomic_smem, s, fam_d,
                       st_d, nodes, level, Dp, codes_c, rfix, ord_cur, rep_boff_d, hsum, hcnt, node_abs, dev->ctr_d,
                       resident.colh_max, atom_chunk);
        }
        else if (resident.col)
          hist_build_col_kernel<CodeT><<<dim3(chunks, pairs, F), kColWarps * 32, resident.col_smem, s>>>(
              fam_d, st_d, nodes, level, Dp, codes_c, rfix, ord_cur, rep_boff_d, rep_nb_d, col_off_d, col_rg_d, hsum,
              hcnt, node_abs, dev->ctr_d);
        else if (hist_global)
          hist_build_kernel<CodeT, true><<<dim3(chunks, pairs, F), kHistThreads, hist_smem, s>>>(
              fam_d, st_d, nodes, level, Dp, codes_c, rfix, ord_cur, rep_boff_d, hsum, hcnt, node_abs, 1, dev->ctr_d);
        else
          hist_build_kernel<CodeT, false><<<dim3(chunks, pairs, F), kHistThreads, hist_smem, s>>>(
              fam_d, st_d, nodes, level, Dp, codes_c, rfix, ord_cur, rep_boff_d, hsum, hcnt, node_abs, groups,
              dev->ctr_d);
      }
      const dim3 sg(grid1(nrep_max, 4, 1 << 20), lw, F);  // 4 warps (reps) per 128-thread block
      {
        ProfScope prof(dev, "fit_screen");
        launch_pdl(screen_kernel, sg, dim3(128), 0, s, fam_d, st_d, nodes, level, hsum, hcnt, node_abs, rep_boff_d,
                   rep_nb_d, win, std::max(nrep_max, 1), level_slots_max, 0, scr_gd, scr_ic);
        launch_pdl(screen_kernel, sg, dim3(128), 0, s, fam_d, st_d, nodes, level, hsum, hcnt, node_abs, rep_boff_d,
                   rep_nb_d, win, std::max(nrep_max, 1), level_slots_max, 1, scr_gd, scr_ic);
      }
      // (n_items[0]: tie-class items, n_items[1]: exact items; both zeroed by level_prep_kernel)
      launch_pdl(tieclass_prep_kernel, dim3(grid1(lw, 4, 1 << 20), F), dim3(128), 0, s,  // warp per node
                 fam_d, st_d, nodes, level, win, std::max(nrep_max, 1), level_slots_max, items, n_items);
      if (resident.phi_smem > 0)
        launch_pdl(tieclass_phi_kernel<CodeT>, dim3(sm * 4), dim3(256), resident.phi_smem, s, fam_d, nodes, items,
                   n_items, level, Dp, codes_cm, ord_cur, rep_nb_d, win, std::max(nrep_max, 1), level_slots_max);
      else
        launch_pdl(tieclass_check_kernel<CodeT>, dim3(sm * 2), dim3(256), 0, s, fam_d, nodes, items, n_items, level, Dp,
                   codes_cm, ord, nodeid, win, std::max(nrep_max, 1), level_slots_max);
      dev->count_launch(2);
      launch_pdl(decide_kernel, dim3(grid1(lw, 4, 1 << 20), F), dim3(128), 0, s, fam_d, st_d, nodes, level, hcnt,
                 rep_boff_d, win, std::max(nrep_max, 1), level_slots_max, items, n_items + 1, dev->ctr_d);
      if (fork_totals) FS_CUDA(cudaStreamWaitEvent(s, dev->ev_join, 0));  // join: totals ready
      {
        ProfScope prof(dev, "fit_exact");
        launch_pdl(exact_kernel<CodeT>, dim3(sm * 2), dim3(256), 0, s, fam_d, nodes, items, n_items + 1, level, Dp,
                   codes_cm, resid, ord, ord_cur, nodeid, rep_boff_d, lbuf, win, std::max(nrep_max, 1), level_slots_max,
                   small_scratch ? 1 : 0);
        if (small_scratch)
          launch_pdl(exact_small_kernel<CodeT>, dim3(kExactSmallCtas), dim3(kSortThreads), exact_small_smem<CodeT>(), s, fam_d, nodes, items,
                     n_items + 1, level, Dp, codes_cm, resid, ord, ord_cur, nodeid, rep_boff_d, lbuf, win,
                     std::max(nrep_max, 1), level_slots_max, small_scratch, n_max);
      }
      launch_pdl(exact_decide_kernel, dim3(grid1(lw, 128, 1 << 20), F), dim3(128), 0, s, fam_d, st_d, nodes, level,
                 hcnt, rep_boff_d, rep_nb_d, win, std::max(nrep_max, 1), level_slots_max, lbuf);
      {
        ProfScope prof(dev, "fit_partition");
        // few large nodes (C4): a CTA per (node, 1,024-row chunk), two passes; many nodes (C5):
        // a CTA per node walking its tiles with the next tile's gathers in flight
        const int64_t p_items = static_cast<int64_t>(F) * lw * part_chunks;
        if (static_cast<int64_t>(F) * lw * 4 < sm) {
          const dim3 pg(static_cast<unsigned>(p_items));
          launch_pdl(partition_count_kernel<CodeT>, pg, dim3(kPartChunk), 0, s, fam_d, st_d, nodes, level, Dp, codes_cm,
                     ord_cur, scratch, nodeid, rep_orig_d, rep_boff_d, vals_d, cle, ord, canon, x_d, d, trees_d, slots,
                     part_cnt, part_chunks, level_slots_max, F);
          launch_pdl(partition_scatter_kernel<CodeT>, pg, dim3(kPartChunk), 0, s, fam_d, st_d, nodes, level, Dp,
                     codes_cm, ord_cur, scratch, nodeid, part_cnt, part_chunks, level_slots_max, F);
        } else {
          launch_pdl(partition_kernel<CodeT>, dim3(lw, F), dim3(1024), 0, s, fam_d, st_d, nodes, level, Dp, codes_cm,
                     ord_cur, scratch, nodeid, rep_orig_d, rep_boff_d, vals_d, cle, ord, canon, x_d, d, trees_d, slots);
        }
      }
      dev->count_launch(8);
    }
    {
      ProfScope prof(dev, "fit_leaf");
      launch_pdl(leaf_cta_kernel, dim3(static_cast<unsigned>(slots), F), dim3(kLeafThreads), 0, s, fam_d, F, st_d, nodes,
                 slots, ord_cur, resid, pred, trees_d, target_c, ebuf, mse_k, n_tot);
    }
    launch_pdl(commit_kernel, dim3(static_cast<unsigned>(ceil_div(F, 128))), dim3(128), 0, s, fam_d, st_d, nodes, F);
    dev->count_launch(2);
    FS_CUDA(cudaGetLastError());
  };
  // after round `round` (0-based): fold the ring once it is full or the fit is over
  auto mse_fold = [&](int round) {
    if ((round + 1) % mse_k != 0 && round + 1 != max_trees) return;
    const int t_lo = (round / mse_k) * mse_k, t_hi = round + 1;
    const int64_t chains = static_cast<int64_t>(F) * (t_hi - t_lo);
    ProfScope prof(dev, "fit_mse");
    mse_fold_kernel<<<static_cast<unsigned>(ceil_div(chains, 4)), 128, 0, s>>>(fam_d, st_d, F, ebuf, mse_k, n_tot,
                                                                               t_lo, t_hi, mse_d, max_trees);
    dev->count_launch();
    FS_CUDA(cudaGetLastError());
  };
  if (max_trees <= 0) return;
  if (std::getenv("FAMSEER_NO_GRAPH") != nullptr) {
    for (int round = 0; round < max_trees; ++round) {
      round_body();
      mse_fold(round);
    }
    return;
  }
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  dev->capturing = true;
  FS_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  try {
    round_body();
  } catch (...) {
    cudaStreamEndCapture(s, &graph);
    dev->capturing = false;
    if (graph) cudaGraphDestroy(graph);
    throw;
  }
  FS_CUDA(cudaStreamEndCapture(s, &graph));
  dev->capturing = false;
  const int64_t per_round = dev->launches - l0;
  FS_CUDA(cudaGraphInstantiate(&exec, graph, 0));
  const int64_t l1 = dev->launches;
  for (int round = 0; round < max_trees; ++round) {
    FS_CUDA(cudaGraphLaunch(exec, s));
    mse_fold(round);
  }
  dev->launches = l0 + per_round * max_trees + (dev->launches - l1);
  FS_CUDA(cudaGraphExecDestroy(exec));
  FS_CUDA(cudaGraphDestroy(graph));
}

}  // namespace

// Fit every family segment; results replace fo->fams[f] (pre-order trees + compiled form).
void fit_families(fs_device* dev, fs_forest* fo, int F, const int64_t* seg, int d, const double* x_d,
                  const double* target_d, const fs_gbt_params* params, const FitRows* rows) {
  cudaStream_t s = dev->stream;
  if (F < 1) return;
  auto fam_id = [&](int f) { return rows && rows->fam_id ? rows->fam_id[f] : f; };
  for (int f = 0; f < F; ++f)
    if (fam_id(f) < 0 || fam_id(f) >= static_cast<int>(fo->fams.size()))
      fail(FS_ERANGE, "fit: more segments than forest families");
  if (seg[0] != 0) fail(FS_EINVAL, "fit: seg[0] must be 0");
  int depth_max = 0, max_trees = 0, n_max = 0;
  for (int f = 0; f < F; ++f) {
    const int64_t n = seg[f + 1] - seg[f];
    if (n < 0) fail(FS_EINVAL, "fit: segment offsets must be non-decreasing");
    if (n > (1 << 30)) fail(FS_EINVAL, "fit: family larger than 2^30 rows");
    if (params[f].trees < 0) fail(FS_EINVAL, "fit: trees must be >= 0");
    if (params[f].depth < 0 || params[f].depth > kMaxDepth)
      fail(FS_EINVAL, "fit: depth must be in [0, " + std::to_string(kMaxDepth) + "]");
    if (n > 0) {
      depth_max = std::max(depth_max, params[f].depth);
      max_trees = std::max(max_trees, params[f].trees);
      n_max = std::max<int>(n_max, static_cast<int>(n));
    }
  }
  const int64_t n_tot = seg[F];
  // FAMSEER_HOST_TIMING=1: host wall-clock per stage of this call on stderr (diagnostics)
  const bool ht = std::getenv("FAMSEER_HOST_TIMING") != nullptr;
  const auto ht0 = std::chrono::steady_clock::now();
  auto htick = [&](const char* what) {
    if (ht)
      std::fprintf(stderr, "[fit host] %-22s %8.1f us\n", what,
                   std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - ht0).count());
  };
  Arena ar(s);
  // ---- family descriptors (stage 1 needs row0/n only) -----------------------------------
  std::vector<FamDesc> fam(static_cast<size_t>(F));
  for (int f = 0; f < F; ++f) {
    std::memset(&fam[f], 0, sizeof(FamDesc));
    fam[f].row0 = rows && rows->row0 ? rows->row0[f] : seg[f];
    fam[f].pos0 = seg[f];
    fam[f].n = static_cast<int32_t>(seg[f + 1] - seg[f]);
    fam[f].trees = fam[f].n > 0 ? params[f].trees : 0;
    fam[f].depth = params[f].depth;
    fam[f].min_split = params[f].min_samples_split;
    fam[f].lr = params[f].learning_rate;
  }
  htick("entry");
  FamDesc* fam_d = ar.upload(fam);
  htick("fam uploaded");

  // ---- stage 1: distinct values / codes ---------------------------------------------------
  const int64_t span = rows && rows->row0 ? rows->span : n_tot;  // rows addressable in x
  uint16_t* codes_all = ar.alloc<uint16_t>(static_cast<size_t>(std::max<int64_t>(span, 1)) * std::max(d, 1));
  double* vals_all = ar.alloc<double>(static_cast<size_t>(F) * std::max(d, 1) * kSmallBins);
  int32_t* nb_all = ar.alloc<int32_t>(static_cast<size_t>(F) * std::max(d, 1));
  uint64_t* hash_all = ar.alloc<uint64_t>(static_cast<size_t>(F) * std::max(d, 1));
  FS_CUDA(cudaMemsetAsync(nb_all, 0, static_cast<size_t>(F) * std::max(d, 1) * sizeof(int32_t), s));
  FS_CUDA(cudaMemsetAsync(hash_all, 0, static_cast<size_t>(F) * std::max(d, 1) * sizeof(uint64_t), s));
  int* negz_d = ar.alloc<int>(F);
  FS_CUDA(cudaMemsetAsync(negz_d, 0, F * sizeof(int), s));
  htick("stage-1 buffers");
  if (d > 0) {
    const size_t smem = 32 * kHashSlots * 8 + 32 * kSmallBins * 8 + 32 * 4 * 2 + 32 * 8;
    ProfScope prof(dev, "fit_distinct");
    if (std::getenv("FAMSEER_DISTINCT_WARP")) {
      FS_CUDA(cudaFuncSetAttribute(distinct_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
      distinct_small_kernel<<<dim3(static_cast<unsigned>(ceil_div(d, 32)), F), 256, smem, s>>>(
          x_d, d, fam_d, codes_all, vals_all, nb_all, hash_all, dev->err_d, negz_d);
    } else {
      distinct_col_kernel<<<dim3(static_cast<unsigned>(d), F), 256, 0, s>>>(x_d, d, fam_d, codes_all, vals_all, nb_all,
                                                                            hash_all, dev->err_d, negz_d);
    }
    dev->count_launch();
  }
  std::vector<int32_t> nb;
  std::vector<int> negz;
  std::vector<uint64_t> hh;
  {
    BatchRead br;
    br.add(nb_all, nb, static_cast<size_t>(F) * d);
    br.add(negz_d, negz, static_cast<size_t>(F));
    br.add(hash_all, hh, static_cast<size_t>(F) * d);
    raise_deferred(br.run(dev));
  }
  for (int f = 0; f < F; ++f) fam[static_cast<size_t>(f)].negz = negz[static_cast<size_t>(f)];
  if (rows && rows->negz_out)
    for (int f = 0; f < F; ++f) rows->negz_out[f] = negz[static_cast<size_t>(f)];
  std::vector<LargeItem> large;
  int64_t vl = 0;
  for (int f = 0; f < F; ++f)
    for (int j = 0; j < d; ++j)
      if (nb[static_cast<size_t>(f) * d + j] < 0) {
        large.push_back({f, j, vl});
        vl += fam[f].n;
      }
  double* vals_large = ar.alloc<double>(std::max<int64_t>(vl, 1));
  std::vector<int64_t> large_src(static_cast<size_t>(F) * d, -1);
  if (!large.empty()) {
    LargeItem* items_d = ar.upload(large);
    int32_t* bufA = ar.alloc<int32_t>(large.size() * n_max);
    int32_t* bufB = ar.alloc<int32_t>(large.size() * n_max);
    distinct_large_kernel<<<static_cast<unsigned>(large.size()), kSortThreads, 0, s>>>(
        x_d, d, fam_d, items_d, bufA, bufB, n_max, codes_all, vals_large, nb_all, hash_all, dev->err_d);
    dev->count_launch();
    BatchRead br;
    br.add(nb_all, nb, static_cast<size_t>(F) * d);
    br.add(hash_all, hh, static_cast<size_t>(F) * d);
    raise_deferred(br.run(dev));
    for (const auto& it : large) large_src[static_cast<size_t>(it.fam) * d + it.feat] = it.vals0;
  }
  htick("distinct read");
  for (int v : nb)
    if (v > kMaxBins) fail(FS_EINVAL, "fit: more than 65535 distinct values in one feature");

  // ---- stage 2: representatives (drop constant and duplicate-column features) -------------
  std::vector<PairItem> pairs;
  for (int f = 0; f < F; ++f) {
    std::map<std::pair<int, uint64_t>, std::vector<int>> seen;
    for (int j = 0; j < d; ++j) {
      const int v = nb[static_cast<size_t>(f) * d + j];
      if (v <= 1) continue;
      auto& lst = seen[{v, hh[static_cast<size_t>(f) * d + j]}];
      for (int k : lst) pairs.push_back({f, k, j, 0});
      lst.push_back(j);
    }
  }
  std::vector<int32_t> mismatch;
  if (!pairs.empty()) {
    PairItem* pd = ar.upload(pairs);
    int32_t* mm = ar.alloc<int32_t>(pairs.size());
    verify_pairs_kernel<<<static_cast<unsigned>(pairs.size()), 256, 0, s>>>(codes_all, d, fam_d, pd, mm);
    dev->count_launch();
    mismatch = download(mm, pairs.size(), s);
  }
  htick("pairs verified");
  std::vector<std::vector<char>> dup(static_cast<size_t>(F), std::vector<char>(static_cast<size_t>(d), 0));
  for (size_t i = 0; i < pairs.size(); ++i)
    if (!mismatch[i]) dup[static_cast<size_t>(pairs[i].fam)][static_cast<size_t>(pairs[i].b)] = 1;
  std::vector<int32_t> rep_orig, rep_nb, rep_boff;
  std::vector<int64_t> rep_src;
  int nrep_max = 0, max_bins = 0, max_nb = 0, min_nrep = INT_MAX;
  int64_t total_ord = 0, total_bins = 0, total_hist = 0, total_lbuf = 0, total_tree = 0;
  const int slots = (1 << (depth_max + 1)) - 1;
  const int level_slots_max = std::max(1, 1 << std::max(0, depth_max - 1));
  for (int f = 0; f < F; ++f) {
    FamDesc& fd = fam[static_cast<size_t>(f)];
    fd.rep0 = static_cast<int32_t>(rep_orig.size());
    int bins = 0;
    fd.f0rep = -1;
    if (fd.n > 0)
      for (int j = 0; j < d; ++j) {
        const int v = nb[static_cast<size_t>(f) * d + j];
        if (v <= 1 || dup[static_cast<size_t>(f)][static_cast<size_t>(j)]) continue;
        if (j == 0) fd.f0rep = static_cast<int32_t>(rep_orig.size()) - fd.rep0;
        rep_orig.push_back(j);
        rep_nb.push_back(v);
        rep_boff.push_back(bins);
        rep_src.push_back(large_src[static_cast<size_t>(f) * d + j]);
        bins += v;
        max_nb = std::max(max_nb, v);
      }
    fd.nrep = static_cast<int32_t>(rep_orig.size()) - fd.rep0;
    fd.bins = bins;
    fd.level_slots = std::max(1, 1 << std::max(0, fd.depth - 1));
    fd.ord0 = total_ord;
    fd.bin0 = total_bins;
    fd.hist0 = total_hist;
    fd.lbuf0 = total_lbuf;
    fd.node0 = static_cast<int64_t>(f) * slots;
    fd.tree0 = total_tree;
    total_ord += static_cast<int64_t>(fd.nrep) * fd.n;
    total_bins += bins;
    total_hist += 2LL * fd.level_slots * bins;
    total_lbuf += static_cast<int64_t>(fd.level_slots) * bins;
    total_tree += static_cast<int64_t>(fd.trees) * slots;
    nrep_max = std::max(nrep_max, static_cast<int>(fd.nrep));
    if (fd.n > 0) min_nrep = std::min(min_nrep, static_cast<int>(fd.nrep));
    max_bins = std::max(max_bins, bins);
  }
  if (min_nrep == INT_MAX) min_nrep = 1;
  const int code_bytes = max_nb <= 256 ? 1 : 2;
  const size_t phi_bytes = (static_cast<size_t>(std::max(max_nb, 1)) * 2 + 15) & ~size_t(15);
  // Path choice: FAMSEER_FIT_PATH = auto (default) | resident | multi.
  ResidentPlan res;
  {
    const char* envp = std::getenv("FAMSEER_FIT_PATH");
    const std::string mode = envp ? envp : "auto";
    if (mode != "auto" && mode != "resident" && mode != "multi")
      fail(FS_EINVAL, "FAMSEER_FIT_PATH must be auto, resident or multi");
    // (the resident fit keeps every round's residuals for the MSE fold: n_tot * trees doubles)
    const bool ebuf_fits = static_cast<double>(seg[F]) * std::max(max_trees, 1) * 8.0 <= 2.0 * (1 << 30);
    if (mode != "multi" && code_bytes == 1 && depth_max <= kResMaxDepth && ebuf_fits) {
      // Shared-memory staging options, most valuable first: the running predictions (read and
      // updated every round) and the presorted lists (reference-order folds); whatever does not
      // fit stays in global memory (L2-resident).
      const int opts[8][3] = {{1, 1, kSpecBufs}, {1, 1, 0}, {1, 0, kSpecBufs}, {1, 0, 0},
                              {0, 1, kSpecBufs}, {0, 1, 0},  {0, 0, kSpecBufs}, {0, 0, 0}};
      for (const auto& op : opts) {
        const bool pred_smem = op[0] != 0, pre_smem = op[1] != 0;
        const int spec = std::getenv("FAMSEER_NO_SPEC") ? 0 : op[2];
        bool ok = true;
        const size_t budget = 225 * 1024;
        std::vector<int> fams_ok;
        size_t need = 0;
        for (int f = 0; f < F; ++f) {
          const FamDesc& fd = fam[static_cast<size_t>(f)];
          if (fd.n <= 0 || fd.trees <= 0) continue;
          if (fd.n > 65535 || fd.nrep > kResThreads) ok = false;
          const int colh = fd.nrep > 0 ? col_height(fd.nrep, rep_nb.data() + fd.rep0, nullptr) : 1;
          need = std::max(need, res_layout(fd.n, fd.nrep, fd.bins, fd.depth, colh, pred_smem, pre_smem, spec).total);
          fams_ok.push_back(f);
        }
        res.families = fams_ok;
        if (ok && need <= budget && !fams_ok.empty()) {
          res.enabled = true;
          res.smem = need;
          res.pred_smem = pred_smem;
          res.pre_smem = pre_smem;
          res.spec_bufs = spec;
          break;
        }
      }
    }
    // FAMSEER_RES_CLUSTER = CTAs per family (1, 2 or 4): the histogram's features are dealt over a
    // thread-block cluster (needs the running predictions in shared memory and <= 32 features
    // per CTA)
    if (res.enabled) {
      const char* ce = std::getenv("FAMSEER_RES_CLUSTER");
      // default: the largest of 4 / 2 whose clusters all fit the SMs at once, for families large
      // enough that the histogram outweighs the per-level cluster exchange (C1's 512 rows: slower)
      int cl = 1;
      int nbig = 0;
      for (int f : res.families) nbig = std::max(nbig, static_cast<int>(fam[static_cast<size_t>(f)].n));
      if (ce) {
        cl = std::atoi(ce);
      } else if (nbig >= kResClusterMinRows) {
        const int nf = static_cast<int>(res.families.size());
        for (int c : {kResClusterMax, 2})
          if (c * nf <= dev->sm_count) {
            cl = c;
            break;
          }
      }
      if (cl != 1 && cl != 2 && cl != 4 && cl != 8) fail(FS_EINVAL, "FAMSEER_RES_CLUSTER must be 1, 2, 4 or 8");
      bool ok = res.pred_smem;
      for (int f : res.families) ok = ok && ceil_div(fam[static_cast<size_t>(f)].nrep, cl) <= 32;
      res.cluster = ok ? cl : 1;
    }
    if (mode == "resident" && !res.enabled && !res.families.empty())
      fail(FS_EINVAL, "fit: resident path requested but the families do not fit one CTA");
  }
  if (phi_bytes <= 96 * 1024 && !std::getenv("FAMSEER_TIE_SCAN")) res.phi_smem = phi_bytes;
  // canonical order by bitonic sort: families without -0.0 whose packed keys fit shared memory
  if (!std::getenv("FAMSEER_CANON_LSD")) {
    res.bitonic_ok.assign(static_cast<size_t>(F), 0);
    for (int f = 0; f < F; ++f) {
      const FamDesc& fd = fam[static_cast<size_t>(f)];
      if (fd.n <= 1 || fd.negz) continue;
      int wide = 0;
      for (int j = 0; j < fd.nrep; ++j) wide |= rep_nb[static_cast<size_t>(fd.rep0 + j)] > 256;
      const int W = (fd.nrep * (wide ? 2 : 1) + 3) / 4 + 2;
      int P = 1;
      while (P < fd.n) P <<= 1;
      const size_t need = static_cast<size_t>(P) * (W + 1) * 4;
      if (need > 160 * 1024) continue;
      res.bitonic_ok[static_cast<size_t>(f)] = 1;
      res.bitonic_smem = std::max(res.bitonic_smem, need);
    }
  }
  // canonical order supplied by / returned to the caller's store (FitRows::io); a family holding
  // a -0.0 always sorts (its ties are not bitwise-identical rows) and returns nothing
  if (rows && rows->io && rows->canon) {
    res.canon_io.assign(static_cast<size_t>(F), 0);
    res.bitonic_ok.resize(static_cast<size_t>(F), 0);
    res.store_canon = rows->canon;
    for (int f = 0; f < F; ++f) {
      if (fam[static_cast<size_t>(f)].n <= 0 || fam[static_cast<size_t>(f)].negz) continue;
      res.canon_io[static_cast<size_t>(f)] = rows->io[f];
      if (rows->io[f] == 1) res.bitonic_ok[static_cast<size_t>(f)] = 2;
    }
  }
  // Column-layout histogram plan (multi-kernel path): per feature group of 32 the largest bin
  // count; row-group copies while they fit the shared-memory budget.
  // Histogram shape for the multi-kernel path: FAMSEER_HIST = atomic (default) | col | rowmajor.
  const char* hist_env = std::getenv("FAMSEER_HIST");
  const std::string hist_mode = hist_env ? hist_env : (std::getenv("FAMSEER_HIST_ROWMAJOR") ? "rowmajor" : "atomic");
  if (hist_mode != "atomic" && hist_mode != "col" && hist_mode != "rowmajor")
    fail(FS_EINVAL, "FAMSEER_HIST must be atomic, col or rowmajor");
  if (!res.enabled && hist_mode == "atomic") {
    const int pv = 16 / code_bytes;
    const int dp = std::max(pv, static_cast<int>(ceil_div(std::max(nrep_max, 1), pv)) * pv);
    int colh_max = 1;
    for (int f = 0; f < F; ++f) {
      const FamDesc& fd = fam[static_cast<size_t>(f)];
      if (fd.nrep > 0) colh_max = std::max(colh_max, col_height(fd.nrep, rep_nb.data() + fd.rep0, nullptr));
    }
    const size_t need = hist_atomic_smem(max_bins, nrep_max, dp, code_bytes, colh_max);
    if (need <= 200 * 1024) {
      res.atomic = true;
      res.atomic_smem = need;
      res.colh_max = colh_max;
    }
  }
  if (!res.enabled && !res.atomic && hist_mode != "rowmajor") {
    const size_t cap = 200 * 1024;
    const int pv = 16 / code_bytes;
    const int dp = std::max(pv, static_cast<int>(ceil_div(std::max(nrep_max, 1), pv)) * pv);
    const size_t tile = ((static_cast<size_t>(kHistTileRows) * dp * code_bytes + 15) & ~size_t(15)) +
                        kHistTileRows * sizeof(int64_t) + 64;
    bool ok = true;
    res.col_off.assign(static_cast<size_t>(F) * (kColWarps + 1), 0);
    res.col_rg.assign(static_cast<size_t>(F), 1);
    size_t need = 0;
    for (int f = 0; f < F && ok; ++f) {
      const FamDesc& fd = fam[static_cast<size_t>(f)];
      const int nfg = (fd.nrep + 31) / 32;
      if (nfg > kColWarps) {
        ok = false;
        break;
      }
      int32_t off = 0;
      for (int g = 0; g < nfg; ++g) {
        int mx = 0;
        for (int j = 32 * g; j < std::min(fd.nrep, 32 * g + 32); ++j)
          mx = std::max(mx, rep_nb[static_cast<size_t>(fd.rep0 + j)]);
        res.col_off[static_cast<size_t>(f) * (kColWarps + 1) + g] = off;
        off += mx * 32;
      }
      for (int g = nfg; g <= kColWarps; ++g) res.col_off[static_cast<size_t>(f) * (kColWarps + 1) + g] = off;
      const size_t per_copy = static_cast<size_t>(off) * 12;
      int rg = std::max(1, kColWarps / std::max(1, nfg));
      while (rg > 1 && rg * per_copy + tile > cap) --rg;
      if (per_copy + tile > cap) ok = false;
      res.col_rg[static_cast<size_t>(f)] = rg;
      need = std::max(need, rg * per_copy + tile);
    }
    if (ok) {
      res.col = true;
      res.col_smem = need;
    }
  }
  const int per_vec = 16 / code_bytes;
  const int Dp = std::max(per_vec, static_cast<int>(ceil_div(std::max(nrep_max, 1), per_vec)) * per_vec);
  FS_CUDA(cudaMemcpyAsync(fam_d, fam.data(), fam.size() * sizeof(FamDesc), cudaMemcpyHostToDevice, s));
  int32_t* rep_orig_d = ar.upload(rep_orig);
  int32_t* rep_nb_d = ar.upload(rep_nb);
  int32_t* rep_boff_d = ar.upload(rep_boff);
  int64_t* rep_src_d = ar.upload(rep_src);
  double* vals_d = ar.alloc<double>(std::max<int64_t>(total_bins, 1));
  if (nrep_max > 0) {
    rep_vals_kernel<<<dim3(static_cast<unsigned>(std::min(nrep_max, 1024)), F), 128, 0, s>>>(
        fam_d, rep_orig_d, rep_boff_d, rep_nb_d, rep_src_d, vals_all, vals_large, d, vals_d);
    dev->count_launch();
  }
  std::vector<FamState> st0(static_cast<size_t>(F));
  for (int f = 0; f < F; ++f) {
    std::memset(&st0[f], 0, sizeof(FamState));
    st0[f].active = fam[f].n > 0 && fam[f].trees > 0;
  }
  FamState* st_d = ar.upload(st0);
  TreeRec* trees_d = ar.alloc<TreeRec>(std::max<int64_t>(total_tree, 1));
  double* mse_d = ar.alloc<double>(static_cast<size_t>(F) * std::max(max_trees, 1));
  double* base_d = ar.alloc<double>(F);
  FS_CUDA(cudaMemsetAsync(base_d, 0, F * sizeof(double), s));

  htick("plan uploaded");
  {
  ProfScope prof_rounds(dev, "fit_rounds");
  if (code_bytes == 1)
    run_rounds<uint8_t>(res, dev, ar, F, d, Dp, n_tot, max_trees, depth_max, slots, nrep_max, max_bins, n_max,
                        level_slots_max, fam_d, st_d, x_d, target_d, codes_all, rep_orig_d, rep_nb_d, rep_boff_d,
                        vals_d, total_ord, total_bins, total_hist, total_lbuf, total_tree, trees_d, mse_d, base_d,
                        min_nrep);
  else
    run_rounds<uint16_t>(res, dev, ar, F, d, Dp, n_tot, max_trees, depth_max, slots, nrep_max, max_bins, n_max,
                         level_slots_max, fam_d, st_d, x_d, target_d, codes_all, rep_orig_d, rep_nb_d, rep_boff_d,
                         vals_d, total_ord, total_bins, total_hist, total_lbuf, total_tree, trees_d, mse_d, base_d,
                         min_nrep);
  }

  // ---- results: heap-slot records -> pre-order CostModelState layout ------------------------
  htick("rounds launched");
  // a forked reader of the current models (fs_tune_step's scoring) must finish first
  if (dev->epilogue_wait) {
    FS_CUDA(cudaStreamWaitEvent(s, dev->epilogue_wait, 0));
    dev->epilogue_wait = nullptr;
  }
  // Epilogue. Default: export + compile on the device straight into each family's model blob
  // (no host round trip; the host pre-order arrays are materialised when first asked for).
  // FAMSEER_HOST_COMPILE=1 (or trees deeper than the device compile handles): read the tree
  // tables back and compile on the host.
  const bool dev_compile = depth_max <= kResMaxDepth && slots <= kCompileSlots && !std::getenv("FAMSEER_HOST_COMPILE");
  if (dev_compile) {
    std::vector<ExportJob> jobs(static_cast<size_t>(F));
    for (int f = 0; f < F; ++f) {
      FamilyModel& m = fo->fams[static_cast<size_t>(fam_id(f))];
      const FamDesc& fd = fam[static_cast<size_t>(f)];
      const int T = std::max(fd.n > 0 ? fd.trees : 0, 0), D = std::max(fd.depth, 0);
      const int S = (1 << (D + 1)) - 1, nint = (1 << D) - 1, nleaf = 1 << D;
      const int nrep = std::max(static_cast<int>(fd.nrep), 0), bins = std::max(static_cast<int>(fd.bins), 0);
      int max_nb = 0, d_orig = 0;
      for (int j = 0; j < nrep; ++j) {
        max_nb = std::max(max_nb, static_cast<int>(rep_nb[static_cast<size_t>(fd.rep0 + j)]));
        d_orig = std::max(d_orig, static_cast<int>(rep_orig[static_cast<size_t>(fd.rep0 + j)]) + 1);
      }
      DevLayout L;
      size_t o = 0;
      auto put = [&](size_t bytes) {
        const size_t at = o;
        o = (o + bytes + 15) & ~size_t(15);
        return at;
      };
      L.meta = put(sizeof(ModelMeta));
      L.nodes = put(static_cast<size_t>(T) * nint * 4);
      L.leafv = put(static_cast<size_t>(T) * nleaf * 8);
      L.leafid = put(static_cast<size_t>(T) * nleaf * 2);
      L.uthr = put(static_cast<size_t>(bins) * 8);
      L.uoff = put(static_cast<size_t>(nrep + 1) * 4);
      L.fmap = put(static_cast<size_t>(nrep) * 4);
      L.cnt = put(static_cast<size_t>(T) * 4);
      L.feat = put(static_cast<size_t>(T) * S * 4);
      L.thr = put(static_cast<size_t>(T) * S * 8);
      L.left = put(static_cast<size_t>(T) * S * 4);
      L.right = put(static_cast<size_t>(T) * S * 4);
      L.val = put(static_cast<size_t>(T) * S * 8);
      L.gain = put(static_cast<size_t>(T) * S * 8);
      L.mse = put(static_cast<size_t>(T) * 8);
      L.total = o;
      L.max_trees = T;
      L.slots = S;
      if (L.total > m.blob_cap) {
        if (m.blob_d) FS_CUDA(cudaFree(m.blob_d));
        m.blob_d = nullptr;
        const size_t cap = std::max<size_t>(L.total + L.total / 2, 4096);
        FS_CUDA(cudaMalloc(&m.blob_d, cap));
        m.blob_cap = cap;
      }
      const bool wide = max_nb > 255;
      jobs[static_cast<size_t>(f)] = {m.blob_d, L, D, wide ? 1 : 0};
      m.lr = fd.lr;
      m.compiled = true;
      m.generic = false;
      m.pending = true;
      m.lay = L;
      m.depth = D;
      m.d_model = nrep;
      m.d_orig = d_orig;
      m.code_bytes = wide ? 2 : 1;
      m.n_uthr = bins;
      m.n_trees = T;  // upper bound until materialised (the device meta holds the count)
      m.nodes_d = reinterpret_cast<uint32_t*>(m.blob_d + L.nodes);
      m.leafv_d = reinterpret_cast<double*>(m.blob_d + L.leafv);
      m.leafid_d = reinterpret_cast<uint16_t*>(m.blob_d + L.leafid);
      m.uthr_d = reinterpret_cast<double*>(m.blob_d + L.uthr);
      m.uoff_d = reinterpret_cast<int32_t*>(m.blob_d + L.uoff);
      m.fmap_d = reinterpret_cast<const int32_t*>(m.blob_d + L.fmap);
      m.meta_d = reinterpret_cast<const ModelMeta*>(m.blob_d + L.meta);
      m.g_off_d = m.g_feat_d = m.g_left_d = m.g_right_d = nullptr;
      m.g_thr_d = m.g_val_d = nullptr;
    }
    ExportJob* jobs_d = ar.upload(jobs);
    export_compile_kernel<<<F, 128, 0, s>>>(fam_d, st_d, trees_d, slots, mse_d, std::max(max_trees, 1), base_d,
                                            rep_orig_d, rep_boff_d, vals_d, jobs_d);
    dev->count_launch();
    FS_CUDA(cudaGetLastError());
    htick("device export launched");
    return;
  }
  std::vector<FamState> st_h;
  std::vector<TreeRec> trees_h;
  std::vector<double> mse_h, base_h;
  {
    BatchRead br;
    br.add(st_d, st_h, static_cast<size_t>(F));
    br.add(trees_d, trees_h, static_cast<size_t>(std::max<int64_t>(total_tree, 1)));
    br.add(mse_d, mse_h, static_cast<size_t>(F) * std::max(max_trees, 1));
    br.add(base_d, base_h, static_cast<size_t>(F));
    raise_deferred(br.run(dev));
  }
  htick("results read");
  UploadBatch batch;
  for (int f = 0; f < F; ++f) {
    FamilyModel& m = fo->fams[static_cast<size_t>(fam_id(f))];
    const FamDesc& fd = fam[static_cast<size_t>(f)];
    m.lr = fd.lr;
    m.base = fd.n > 0 ? base_h[static_cast<size_t>(f)] : 0.0;
    m.offsets.assign(1, 0);
    m.feature.clear();
    m.threshold.clear();
    m.left.clear();
    m.right.clear();
    m.value.clear();
    m.gain.clear();
    m.mse.clear();
    const int T = st_h[static_cast<size_t>(f)].ntrees;
    m.offsets.reserve(static_cast<size_t>(T) + 1);
    for (auto* v : {&m.feature, &m.left, &m.right}) v->reserve(static_cast<size_t>(T) * slots);
    for (auto* v : {&m.threshold, &m.value, &m.gain}) v->reserve(static_cast<size_t>(T) * slots);
    struct Emit {
      int slot, parent, side;  // parent: global index of the parent node (-1 root), side 0 left / 1 right
    };
    std::vector<Emit> es;
    for (int t = 0; t < T; ++t) {
      const TreeRec* rec = trees_h.data() + fd.tree0 + static_cast<int64_t>(t) * slots;
      const int base_idx = static_cast<int>(m.feature.size());
      es.assign(1, {0, -1, 0});
      while (!es.empty()) {  // pre-order: left subtree before right (costmodel.cpp:108-111)
        const Emit e = es.back();
        es.pop_back();
        const int gidx = static_cast<int>(m.feature.size());
        const TreeRec& r = rec[e.slot];
        if (r.kind != kNodeSplit && r.kind != kNodeLeaf) fail(FS_ECUDA, "fit: internal error (missing tree node)");
        m.feature.push_back(r.kind == kNodeSplit ? r.feature : -1);
        m.threshold.push_back(r.kind == kNodeSplit ? r.threshold : 0.0);
        m.left.push_back(-1);
        m.right.push_back(-1);
        m.value.push_back(r.kind == kNodeSplit ? 0.0 : r.value);
        m.gain.push_back(r.kind == kNodeSplit ? r.gain : 0.0);
        if (e.parent >= 0) (e.side ? m.right : m.left)[static_cast<size_t>(e.parent)] = gidx - base_idx;
        if (r.kind == kNodeSplit) {
          es.push_back({2 * e.slot + 2, gidx, 1});
          es.push_back({2 * e.slot + 1, gidx, 0});
        }
      }
      m.offsets.push_back(static_cast<int32_t>(m.feature.size()));
      m.mse.push_back(mse_h[static_cast<size_t>(f) * max_trees + t]);
    }
    m.screened = static_cast<int64_t>(st_h[static_cast<size_t>(f)].screened);
    m.exact = static_cast<int64_t>(st_h[static_cast<size_t>(f)].exact);
    compile_model(dev, m, &batch);
  }
  batch.flush(dev);
  htick("models compiled");
}

}  // namespace fit
}  // namespace fs

extern "C" {

int fs_fit_d(fs_device* dev, fs_forest* fo, int32_t nseg, const int64_t* seg, int32_t d, const double* x_d,
             const double* target_d, const fs_gbt_params* params) {
  return fs::guard([&] {
    if (!dev || !fo || nseg < 0 || !seg || d < 0 || !params) fs::fail(FS_EINVAL, "fs_fit: bad arguments");
    dev->activate();
    fs::fit::fit_families(dev, fo, nseg, seg, d, x_d, target_d, params);
  });
}

int fs_fit(fs_device* dev, fs_forest* fo, int32_t nseg, const int64_t* seg, int32_t d, const double* x,
           const double* target, const fs_gbt_params* params) {
  return fs::guard([&] {
    if (!dev || !fo || nseg < 0 || !seg || d < 0 || !params) fs::fail(FS_EINVAL, "fs_fit: bad arguments");
    dev->activate();
    const int64_t n = seg[nseg];
    auto* xd = static_cast<double*>(dev->scratch(fs::kSlotH2D0, std::max<int64_t>(n * d, 1) * sizeof(double)));
    auto* yd = static_cast<double*>(dev->scratch(fs::kSlotH2D1, std::max<int64_t>(n, 1) * sizeof(double)));
    if (n * d > 0) FS_CUDA(cudaMemcpyAsync(xd, x, n * d * sizeof(double), cudaMemcpyHostToDevice, dev->stream));
    if (n) FS_CUDA(cudaMemcpyAsync(yd, target, n * sizeof(double), cudaMemcpyHostToDevice, dev->stream));
    fs::fit::fit_families(dev, fo, nseg, seg, d, xd, yd, params);
  });
}

int fs_fit_records_d(fs_device* dev, fs_forest* fo, const fs_spaces* sp, int32_t nseg, const int64_t* seg,
                     const int32_t* space_of_d, const int32_t* assign_d, int32_t pad, const double* target_d,
                     const fs_gbt_params* params) {
  return fs::guard([&] {
    if (!dev || !fo || !sp || nseg < 0 || !seg || pad < 0 || !params)
      fs::fail(FS_EINVAL, "fs_fit_records: bad arguments");
    dev->activate();
    const int64_t n = seg[nseg];
    auto* xd = static_cast<double*>(dev->scratch(fs::kSlotFitX, std::max<int64_t>(n * pad, 1) * sizeof(double)));
    fs::launch_featurize(dev, sp, n, space_of_d, assign_d, pad, xd);
    fs::fit::fit_families(dev, fo, nseg, seg, pad, xd, target_d, params);
  });
}

int fs_fit_records(fs_device* dev, fs_forest* fo, const fs_spaces* sp, int32_t nseg, const int64_t* seg,
                   const int32_t* space_of, const int32_t* assign, int32_t pad, const double* target,
                   const fs_gbt_params* params) {
  return fs::guard([&] {
    if (!dev || !fo || !sp || nseg < 0 || !seg || pad < 0 || !params)
      fs::fail(FS_EINVAL, "fs_fit_records: bad arguments");
    dev->activate();
    const int64_t n = seg[nseg];
    // the reference validates every record's dimension on the host (searchspace.cpp:94-101)
    for (int64_t i = 0; i < n; ++i) {
      const int s = space_of[i];
      if (s < 0 || s >= sp->n) fs::fail(FS_EINVAL, "fit_records: unknown space id");
      if (pad < fs_feature_dim(sp->k_h[static_cast<size_t>(s)])) fs::fail(FS_EINVAL, "fit_records: pad_dim too small");
    }
    const size_t b_so = static_cast<size_t>(std::max<int64_t>(n, 1)) * sizeof(int32_t);
    const size_t b_a = static_cast<size_t>(std::max<int64_t>(n, 1)) * FS_MAX_KNOBS * sizeof(int32_t);
    const size_t b_t = static_cast<size_t>(std::max<int64_t>(n, 1)) * sizeof(double);
    auto* in = static_cast<unsigned char*>(dev->scratch(fs::kSlotFitIn, b_t + b_so + b_a + 32));
    auto* td = reinterpret_cast<double*>(in);
    auto* sd = reinterpret_cast<int32_t*>(in + b_t);
    auto* ad = reinterpret_cast<int32_t*>(in + b_t + b_so);
    if (n) {
      FS_CUDA(cudaMemcpyAsync(td, target, n * sizeof(double), cudaMemcpyHostToDevice, dev->stream));
      FS_CUDA(cudaMemcpyAsync(sd, space_of, n * sizeof(int32_t), cudaMemcpyHostToDevice, dev->stream));
      FS_CUDA(cudaMemcpyAsync(ad, assign, n * FS_MAX_KNOBS * sizeof(int32_t), cudaMemcpyHostToDevice, dev->stream));
    }
    auto* xd = static_cast<double*>(dev->scratch(fs::kSlotFitX, std::max<int64_t>(n * pad, 1) * sizeof(double)));
    fs::launch_featurize(dev, sp, n, sd, ad, pad, xd);
    fs::fit::fit_families(dev, fo, nseg, seg, pad, xd, td, params);
  });
}

}  // extern "C"

namespace fs {
void score_device(fs_device* dev, const fs_spaces* sp, const fs_forest* fo, int32_t nseg, const int64_t* seg,
                  const int32_t* space_of_d, const int32_t* assign_d, int32_t pad, double* scores_d, int32_t* perm_d,
                  const uint64_t* index_d);
namespace {
__global__ void merge_err_kernel(uint32_t* err, uint32_t* err_aux) {
  if (*err_aux) {
    *err |= *err_aux;
    *err_aux = 0;
  }
}

// One tuning round (tune_step's scoring, scheduler.cpp:187-192, and train_and_charge's refit,
// :233-238) with the two halves overlapped: the pools are scored with the forest's CURRENT
// models on the device's aux stream (forked after the main stream's prior work, own error word)
// while the main stream runs the refit; the refit's epilogue - the first write of any model
// blob - waits for the scoring. `prefix` (host-pointer variant: the pool's H2D copies) and
// `suffix` (its D2H copies) run on the aux stream around the scoring; `fit` runs on the main
// stream. On return the main stream is joined with the fork and the fork's deferred errors are
// merged into the device's error word.
template <class Pre, class Score, class Post, class Fit>
void tune_step(fs_device* dev, Pre prefix, Score score, Post suffix, Fit fit) {
  cudaStream_t main = dev->stream, aux = dev->aux_stream();
  uint32_t* err_main = dev->err_d;
  FS_CUDA(cudaEventRecord(dev->ev_fork, main));
  FS_CUDA(cudaStreamWaitEvent(aux, dev->ev_fork, 0));
  dev->stream = aux;
  dev->err_d = dev->err_aux_d;
  try {
    prefix();
    score();
    suffix();
  } catch (...) {
    dev->stream = main;
    dev->err_d = err_main;
    FS_CUDA(cudaEventRecord(dev->ev_join, aux));
    FS_CUDA(cudaStreamWaitEvent(main, dev->ev_join, 0));
    throw;
  }
  dev->stream = main;
  dev->err_d = err_main;
  FS_CUDA(cudaEventRecord(dev->ev_join, aux));
  dev->epilogue_wait = dev->ev_join;
  auto join = [&] {
    dev->epilogue_wait = nullptr;
    FS_CUDA(cudaStreamWaitEvent(main, dev->ev_join, 0));
    merge_err_kernel<<<1, 1, 0, main>>>(dev->err_d, dev->err_aux_d);
    FS_CUDA(cudaGetLastError());
  };
  try {
    fit();
  } catch (...) {
    join();
    throw;
  }
  join();
}
}  // namespace
}  // namespace fs

extern "C" {

int fs_tune_step_d(fs_device* dev, const fs_spaces* sp, fs_forest* fo, int32_t n_pool_segments,
                   const int64_t* pool_seg_h, const int32_t* pool_space_of_d, const int32_t* pool_assign_d,
                   int32_t pad_dim, double* scores_d, int32_t* perm_d, int32_t n_fit_segments,
                   const int64_t* fit_seg_h, const double* x_d, const double* target_d,
                   const fs_gbt_params* params) {
  return fs::guard([&] {
    if (!dev || !sp || !fo || n_pool_segments < 0 || !pool_seg_h || pad_dim < 0 || n_fit_segments < 0 ||
        !fit_seg_h || !params)
      fs::fail(FS_EINVAL, "fs_tune_step: bad arguments");
    dev->activate();
    fs::tune_step(
        dev, [] {},
        [&] {
          if (pool_seg_h[n_pool_segments] > 0)
            fs::score_device(dev, sp, fo, n_pool_segments, pool_seg_h, pool_space_of_d, pool_assign_d, pad_dim,
                             scores_d, perm_d, nullptr);
        },
        [] {}, [&] { fs::fit::fit_families(dev, fo, n_fit_segments, fit_seg_h, pad_dim, x_d, target_d, params); });
  });
}

int fs_tune_step(fs_device* dev, const fs_spaces* sp, fs_forest* fo, int32_t n_pool_segments, const int64_t* pool_seg,
                 const int32_t* pool_space_of, const int32_t* pool_assign, int32_t pad_dim, double* scores,
                 int32_t* perm, int32_t n_fit_segments, const int64_t* fit_seg, const int32_t* fit_space_of,
                 const int32_t* fit_assign, const double* fit_target, const fs_gbt_params* params) {
  return fs::guard([&] {
    if (!dev || !sp || !fo || n_pool_segments < 0 || !pool_seg || pad_dim < 0 || n_fit_segments < 0 || !fit_seg ||
        !params)
      fs::fail(FS_EINVAL, "fs_tune_step: bad arguments");
    if (pool_seg[0] != 0 || fit_seg[0] != 0) fs::fail(FS_EINVAL, "fs_tune_step: seg[0] must be 0");
    dev->activate();
    const int64_t P = pool_seg[n_pool_segments], n = fit_seg[n_fit_segments];
    for (int64_t i = 0; i < n; ++i) {  // the reference validates every record's dimension (searchspace.cpp:94-101)
      const int s = fit_space_of[i];
      if (s < 0 || s >= sp->n) fs::fail(FS_EINVAL, "fit_records: unknown space id");
      if (pad_dim < fs_feature_dim(sp->k_h[static_cast<size_t>(s)])) fs::fail(FS_EINVAL, "fit_records: pad_dim too small");
    }
    int32_t *so = nullptr, *as = nullptr, *pd = nullptr;
    double* sd = nullptr;
    fs::tune_step(
        dev,
        [&] {  // pool descriptors in, on the fork
          if (P <= 0) return;
          so = static_cast<int32_t*>(dev->scratch(fs::kSlotH2D0, P * sizeof(int32_t)));
          as = static_cast<int32_t*>(dev->scratch(fs::kSlotH2D1, P * FS_MAX_KNOBS * sizeof(int32_t)));
          sd = static_cast<double*>(dev->scratch(fs::kSlotScoreS, P * sizeof(double)));
          pd = static_cast<int32_t*>(dev->scratch(fs::kSlotScoreP, P * sizeof(int32_t)));
          FS_CUDA(cudaMemcpyAsync(so, pool_space_of, P * sizeof(int32_t), cudaMemcpyHostToDevice, dev->stream));
          FS_CUDA(cudaMemcpyAsync(as, pool_assign, P * FS_MAX_KNOBS * sizeof(int32_t), cudaMemcpyHostToDevice,
                                  dev->stream));
        },
        [&] {
          if (P > 0) fs::score_device(dev, sp, fo, n_pool_segments, pool_seg, so, as, pad_dim, sd, pd, nullptr);
        },
        [&] {  // scores and permutation out, on the fork
          if (P <= 0) return;
          if (scores) FS_CUDA(cudaMemcpyAsync(scores, sd, P * sizeof(double), cudaMemcpyDeviceToHost, dev->stream));
          if (perm) FS_CUDA(cudaMemcpyAsync(perm, pd, P * sizeof(int32_t), cudaMemcpyDeviceToHost, dev->stream));
        },
        [&] {  // records in, featurized on the device (simbackend.cpp:185), refit (costmodel.cpp:224-235)
          const size_t b_so = static_cast<size_t>(std::max<int64_t>(n, 1)) * sizeof(int32_t);
          const size_t b_a = static_cast<size_t>(std::max<int64_t>(n, 1)) * FS_MAX_KNOBS * sizeof(int32_t);
          const size_t b_t = static_cast<size_t>(std::max<int64_t>(n, 1)) * sizeof(double);
          auto* in = static_cast<unsigned char*>(dev->scratch(fs::kSlotFitIn, b_t + b_so + b_a + 32));
          auto* td = reinterpret_cast<double*>(in);
          auto* tsd = reinterpret_cast<int32_t*>(in + b_t);
          auto* tad = reinterpret_cast<int32_t*>(in + b_t + b_so);
          if (n) {
            FS_CUDA(cudaMemcpyAsync(td, fit_target, n * sizeof(double), cudaMemcpyHostToDevice, dev->stream));
            FS_CUDA(cudaMemcpyAsync(tsd, fit_space_of, n * sizeof(int32_t), cudaMemcpyHostToDevice, dev->stream));
            FS_CUDA(cudaMemcpyAsync(tad, fit_assign, n * FS_MAX_KNOBS * sizeof(int32_t), cudaMemcpyHostToDevice,
                                    dev->stream));
          }
          auto* xd = static_cast<double*>(dev->scratch(fs::kSlotFitX, std::max<int64_t>(n * pad_dim, 1) * sizeof(double)));
          fs::launch_featurize(dev, sp, n, tsd, tad, pad_dim, xd);
          fs::fit::fit_families(dev, fo, n_fit_segments, fit_seg, pad_dim, xd, td, params);
        });
    // the refit models' host copies ride on the same synchronisation (the next export reads them
    // without another round trip)
    const bool staged = fs::materialize_enqueue(dev, fo->fams);
    const uint32_t bits = dev->take_errors();  // the host outputs are complete (main joined the fork)
    if (staged && !bits) fs::materialize_parse(dev, fo->fams);
    fs::raise_deferred(bits);
  });
}

int fs_forest_fit_stats(const fs_forest* fo, int32_t family, int64_t* screened, int64_t* exact) {
  return fs::guard([&] {
    if (!fo || family < 0 || family >= static_cast<int32_t>(fo->fams.size()))
      fs::fail(FS_ERANGE, "fs_forest_fit_stats: unknown family id");
    const auto& m = fo->fams[static_cast<size_t>(family)];
    fs::materialize(fo->dev, m);
    if (screened) *screened = m.screened;
    if (exact) *exact = m.exact;
  });
}

}  // extern "C"
