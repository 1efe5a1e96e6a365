/* famseer.h - C ABI of the B200-native FamilySeer cost-model hot path (libfamseer.so).
 *
 * The reference (/root/reference/proj, "famtune") has no plugin ABI: its hot path is the static
 * C++ API in namespace famtune. This header is the thin extern "C" layer
 * underneath the drop-in C++ API (include/famtune/ headers): plain pointers and sizes, no C++ or
 * torch types, int status codes, one thread-local error string. Each entry point names the
 * reference function it replaces.
 *
 * Conventions
 *   - Every call is ordered on the device's stream. Entry points taking HOST pointers copy in,
 *     run, copy out and synchronize before returning (the reference's value semantics). Entry
 *     points with the suffix _d take DEVICE pointers and are asynchronous; call
 *     fs_device_check() to synchronize and surface deferred kernel-side errors (non-finite
 *     features, out-of-range knob indices) as FS_EINVAL.
 *   - Status: FS_OK on success, otherwise the code of the reference exception it stands for:
 *       FS_EINVAL  std::invalid_argument  (costmodel.cpp:178-182,226-231,239; searchspace.cpp:95-100)
 *       FS_EDOMAIN std::domain_error      (costmodel.cpp:273-275)
 *       FS_ERANGE  std::out_of_range      (family.cpp:81-93)
 *     plus FS_ECUDA / FS_ENOMEM / FS_ENCCL for device failures. fs_last_error() returns the
 *     message of the last failing call on this thread.
 *   - Model layout (costmodel.hpp:27-57): trees concatenated in pre-order; tree t owns nodes
 *     [offsets[t], offsets[t+1]); feature < 0 marks a leaf; left/right are tree-local.
 *   - Feature matrices are row-major FP64 [rows][d]; candidate assignments are int32
 *     [rows][FS_MAX_KNOBS] (knob value indices, unused slots ignored).
 */
#ifndef FAMSEER_H
#define FAMSEER_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FS_MAX_KNOBS 16 /* searchspace.hpp:18 kMaxKnobs */

enum fs_status {
  FS_OK = 0,
  FS_EINVAL = 1,
  FS_EDOMAIN = 2,
  FS_ERANGE = 3,
  FS_ECUDA = 4,
  FS_ENOMEM = 5,
  FS_ENCCL = 6
};

typedef struct fs_device fs_device;   /* one per GPU: stream, scratch arena, error word */
typedef struct fs_spaces fs_spaces;   /* device-resident knob-space table */
typedef struct fs_forest fs_forest;   /* device-resident ensembles, one per family */

/* GbtParams (costmodel.hpp:20-25). */
typedef struct fs_gbt_params {
  int32_t trees;             /* default 50 */
  int32_t depth;             /* default 3 */
  double learning_rate;      /* default 0.1 */
  int32_t min_samples_split; /* default 2 */
} fs_gbt_params;

const char* fs_last_error(void);
const char* fs_version(void);

/* ---- device ------------------------------------------------------------------------------ */
int fs_device_create(int ordinal, fs_device** out);
int fs_device_destroy(fs_device* dev);
/* Use an external cudaStream_t (e.g. torch's current stream); NULL restores the own stream. */
int fs_device_set_stream(fs_device* dev, void* cuda_stream);
void* fs_device_stream(fs_device* dev);
/* Synchronize the stream and report deferred kernel-side errors. */
int fs_device_check(fs_device* dev);
/* Kernels launched by this device since creation (evidence counter for bench.py). */
int64_t fs_device_launches(const fs_device* dev);
/* Device-side work counters since the last reset: [0] histogram algorithmic bytes, [1]
 * histogram rows, [2] reference-order folds, [3] nodes re-evaluated in reference order. */
int fs_device_counters(fs_device* dev, int64_t* out, int32_t n, int32_t reset);
/* Per-kernel CUDA-event timing on the device's stream. `kernels` is a comma-separated list of
 * kernel names ("*" = all, NULL/"" = off); enabling resets the accumulators. */
int fs_device_profile(fs_device* dev, const char* kernels);
int fs_device_profile_read(fs_device* dev, const char* kernel, int64_t* count, double* total_ms);
/* Comma-separated names seen so far (two-call size query; returns bytes needed incl. NUL). */
int64_t fs_device_profile_names(fs_device* dev, char* buf, int64_t cap);

/* ---- knob spaces + featurize (searchspace.cpp:90-118, feature_dim :86-88) -------------------
 * n_knobs[s] in [1,16]; n_values[s*16+k] = |values| of knob k; values concatenated space by
 * space, knob by knob. log2 tables are computed once on the host with the C library's log2, the
 * function the reference calls, so features are bit-identical. */
int fs_feature_dim(int32_t knob_count);
int fs_spaces_create(fs_device* dev, int32_t n_spaces, const int32_t* n_knobs,
                     const int32_t* n_values, const int64_t* values, fs_spaces** out);
int fs_spaces_destroy(fs_spaces* sp);
int32_t fs_spaces_max_feature_dim(const fs_spaces* sp); /* max_feature_dim (graph.cpp:346-352) */

/* out[i*pad_dim + j] = featurize(space[space_of[i]], assign[i*16 .. +K], pad_dim)[j].
 * FS_EINVAL when pad_dim < feature_dim(K) of any referenced space or an index is out of range. */
int fs_featurize(fs_device* dev, const fs_spaces* sp, int64_t n, const int32_t* space_of,
                 const int32_t* assign, int32_t pad_dim, double* out);
int fs_featurize_d(fs_device* dev, const fs_spaces* sp, int64_t n, const int32_t* space_of_d,
                   const int32_t* assign_d, int32_t pad_dim, double* out_d);

/* ---- forests (CostModelState trees, costmodel.hpp:48-57) -------------------------------------
 * A forest holds F family ensembles. fs_forest_upload replaces family f's ensemble with
 * host-built trees (the tests' hand-built models, or a CostModelState the caller owns). */
int fs_forest_create(fs_device* dev, int32_t n_families, fs_forest** out);
int fs_forest_destroy(fs_forest* fo);
int fs_forest_upload(fs_forest* fo, int32_t family, double base, double learning_rate,
                     int32_t n_trees, const int32_t* offsets, const int32_t* feature,
                     const double* threshold, const int32_t* left, const int32_t* right,
                     const double* value);
/* Two-call export: pass NULL arrays to learn n_trees / n_nodes, then fill. gain (per node, 0
 * for leaves) and mse (train_mse_by_round) are only produced by fs_fit; may be NULL. */
int fs_forest_export(const fs_forest* fo, int32_t family, double* base, int32_t* n_trees,
                     int32_t* n_nodes, int32_t* offsets, int32_t* feature, double* threshold,
                     int32_t* left, int32_t* right, double* value, double* gain, double* mse);

/* ---- predict (costmodel.cpp:135-143, 237-246) ------------------------------------------------
 * Rows [seg[f], seg[f+1]) are scored with family f's ensemble: score = base, then for every tree
 * in order score = score + lr*leaf (separately rounded, no FMA). leaf_ids (optional, uint16
 * [rows][n_trees_of_family]: the tree-local pre-order index of the leaf RegressionTree::eval
 * stops at) is written row-major, segment after segment (segment f starts at element
 * sum_{g<f} rows_g * n_trees_g). A tree of more than 65,536 nodes cannot report leaf ids
 * (FS_EINVAL). Non-finite features -> FS_EINVAL. */
int fs_predict(fs_device* dev, const fs_forest* fo, int32_t n_segments, const int64_t* seg,
               int32_t d, const double* x, double* scores, uint16_t* leaf_ids);
int fs_predict_d(fs_device* dev, const fs_forest* fo, int32_t n_segments, const int64_t* seg_h,
                 int32_t d, const double* x_d, double* scores_d, uint16_t* leaf_ids_d);

/* ---- rank (scheduler.cpp:187-192) ------------------------------------------------------------
 * perm[seg[f] + i] = segment-local index of the i-th smallest (score, index) pair: the order
 * std::sort gives vector<pair<double,size_t>>. -0.0 and +0.0 compare equal. */
int fs_rank(fs_device* dev, int32_t n_segments, const int64_t* seg, const double* scores,
            int32_t* perm);
int fs_rank_d(fs_device* dev, int32_t n_segments, const int64_t* seg_h, const double* scores_d,
              int32_t* perm_d);

/* ---- score: the batched tune_step scoring block (scheduler.cpp:187-192) ---------------------
 * featurize -> predict -> rank in one call; the feature matrix never leaves the device.
 * scores[i] and perm[seg[f] + k] as for fs_predict / fs_rank. Either output may be NULL on the
 * host-pointer variant; fs_score_d with perm_d NULL scores without ranking. */
int fs_score(fs_device* dev, const fs_spaces* sp, const fs_forest* fo, int32_t n_segments,
             const int64_t* seg, const int32_t* space_of, const int32_t* assign, int32_t pad_dim,
             double* scores, int32_t* perm);
int fs_score_d(fs_device* dev, const fs_spaces* sp, const fs_forest* fo, int32_t n_segments,
               const int64_t* seg_h, const int32_t* space_of_d, const int32_t* assign_d,
               int32_t pad_dim, double* scores_d, int32_t* perm_d);

/* ---- one tuning round: score + refit, overlapped (scheduler.cpp:187-192 + :233-238) ---------
 * fs_score of the pools with the forest's CURRENT models and a refit of every fit segment, as
 * one call: the scoring runs on the device's second stream concurrently with the refit's
 * preparation and boosting rounds, and the refit writes the new models only after the scoring
 * has read the old ones - results identical to fs_score followed by fs_fit_d / fs_fit_records.
 * fs_tune_step_d: device pointers, training rows as features (fs_fit_d's x/target); returns
 * like fs_fit_d (deferred errors of the scoring surface at the next fs_device_check).
 * fs_tune_step: host pointers, training rows as measurement records featurized on the device
 * (fs_fit_records); scores/perm are complete and every error raised on return, and the refit
 * models' host copies were fetched in the same synchronisation (fs_forest_export right after
 * needs no device round trip). */
int fs_tune_step_d(fs_device* dev, const fs_spaces* sp, fs_forest* fo, int32_t n_pool_segments,
                   const int64_t* pool_seg_h, const int32_t* pool_space_of_d, const int32_t* pool_assign_d,
                   int32_t pad_dim, double* scores_d, int32_t* perm_d, int32_t n_fit_segments,
                   const int64_t* fit_seg_h, const double* x_d, const double* target_d,
                   const fs_gbt_params* params);
int fs_tune_step(fs_device* dev, const fs_spaces* sp, fs_forest* fo, int32_t n_pool_segments,
                 const int64_t* pool_seg, const int32_t* pool_space_of, const int32_t* pool_assign,
                 int32_t pad_dim, double* scores, int32_t* perm, int32_t n_fit_segments,
                 const int64_t* fit_seg, const int32_t* fit_space_of, const int32_t* fit_assign,
                 const double* fit_target, const fs_gbt_params* params);

/* ---- score from linear_index descriptors -------------------------------
 * As fs_score, but candidate i is (space_of[i], index[i]) with index[i] =
 * linear_index(space, assignment) (searchspace.cpp:48-54), decoded on the device exactly as
 * candidate_from_index (:56-66) does (mixed radix, last knob fastest): 4 + 8 bytes per candidate
 * in instead of 4 + 64. Replaces the per-candidate featurize + predict calls of
 * scheduler.cpp:187-191 for callers that keep MeasuredSet's u64 keys (reference searchspace.hpp:71-84). */
int fs_score_index(fs_device* dev, const fs_spaces* sp, const fs_forest* fo, int32_t n_segments,
                   const int64_t* seg, const int32_t* space_of, const uint64_t* index, int32_t pad_dim,
                   double* scores, int32_t* perm);
int fs_score_index_d(fs_device* dev, const fs_spaces* sp, const fs_forest* fo, int32_t n_segments,
                     const int64_t* seg_h, const int32_t* space_of_d, const uint64_t* index_d,
                     int32_t pad_dim, double* scores_d, int32_t* perm_d);

/* ---- multi-GPU: family-parallel tuning on the GPUs of one node ---------------
 * Families share nothing (scheduler.cpp:123-130), so each rank (one process per GPU) owns a
 * deterministic set of families and calls fs_score / fs_fit / fs_tune_step on its own device;
 * per-family results are bit-identical on any rank. fs_shard_families: LPT partition on
 * rows*T + pool*T (ties: lower family id first, then the least-loaded lower rank), host only.
 * fs_comm: an NCCL communicator (libnccl.so.2 loaded at run time; FS_ENCCL when it is missing or
 * a call fails): rank 0 makes the id with fs_comm_id and the caller broadcasts the
 * FS_COMM_ID_BYTES bytes to every rank (any side channel). fs_topk_allgather: the per-round
 * exchange - every local family's first g ranked candidates (tune_step's by-score picks,
 * scheduler.cpp:196-201) as records {family id, pool index, score} (float64), all-gathered over
 * NVLink and merged on the device into merged_d[n_families][g][3] in family-id order (missing
 * entries -1). fam_cap: the largest local family count of any rank (the same on every rank).
 * Stream-ordered on the device's stream. */
#define FS_COMM_ID_BYTES 128
typedef struct fs_comm fs_comm;
int fs_shard_families(int32_t n_families, const int64_t* rows, const int64_t* pool, const int32_t* trees,
                      int32_t world, int32_t* owner);
int fs_comm_id(uint8_t* id /* FS_COMM_ID_BYTES */);
int fs_comm_create(fs_device* dev, int32_t world, int32_t rank, const uint8_t* id, fs_comm** out);
int fs_comm_destroy(fs_comm* comm);
int fs_topk_allgather(fs_comm* comm, int32_t n_local, const int32_t* family_ids, const int64_t* seg_h,
                      const double* scores_d, const int32_t* perm_d, int32_t g, int32_t fam_cap,
                      int32_t n_families, double* merged_d);

/* ---- pairwise accuracy (costmodel.cpp:248-277) over precomputed scores ---------------------
 * Pairs with relative latency difference < 1e-6 are excluded, predicted ties score 1/2.
 * FS_EINVAL for m < 2, FS_EDOMAIN when every pair is excluded. */
int fs_pairwise_accuracy(fs_device* dev, int64_t m, const double* scores, const double* latency,
                         double* out);
/* Batched form (the heatmap's n x n model/validation-set grid,
 * experiment.cpp:135-167): out[k] = pairwise accuracy of segment k = [seg[k], seg[k+1]) of
 * scores/latency, one launch for all segments. FS_EINVAL if a segment holds < 2 records,
 * FS_EDOMAIN if a segment excludes every pair (fs_last_error names the first such segment). */
int fs_pairwise_accuracy_batch(fs_device* dev, int32_t n_segments, const int64_t* seg, const double* scores,
                               const double* latency, double* out);

/* ---- fit (costmodel.cpp:152-222; train_cost_model :224-235 appends log-latency rows first) ---
 * Refit family f's ensemble from scratch on rows [seg[f], seg[f+1]) of x/target with params[f].
 * Trees are bit-identical to the reference's (canonical row order, reference-order sums for every
 * value that reaches a tree, exact tie resolution). gains: the reference's split gain per
 * internal node. Non-finite features -> FS_EINVAL. */
int fs_fit(fs_device* dev, fs_forest* fo, int32_t n_segments, const int64_t* seg, int32_t d,
           const double* x, const double* target, const fs_gbt_params* params);
int fs_fit_d(fs_device* dev, fs_forest* fo, int32_t n_segments, const int64_t* seg_h, int32_t d,
             const double* x_d, const double* target_d, const fs_gbt_params* params);

/* fit from measurement records (MeasurementRecord: candidate + log latency, searchspace.hpp:52-57):
 * each record's features are featurize(space_of[i], assign[i], pad_dim) computed on the device
 * (the reference featurizes them at measurement time, simbackend.cpp:185) - the host sends 68
 * bytes per record instead of pad_dim*8. target[i] = log(latency_ms) as the caller computes it
 * (costmodel.cpp:228-233). Otherwise identical to fs_fit. */
int fs_fit_records(fs_device* dev, fs_forest* fo, const fs_spaces* sp, int32_t n_segments, const int64_t* seg,
                   const int32_t* space_of, const int32_t* assign, int32_t pad_dim, const double* target,
                   const fs_gbt_params* params);
int fs_fit_records_d(fs_device* dev, fs_forest* fo, const fs_spaces* sp, int32_t n_segments,
                     const int64_t* seg_h, const int32_t* space_of_d, const int32_t* assign_d, int32_t pad_dim,
                     const double* target_d, const fs_gbt_params* params);

/* ---- device-resident training store -----------------------------------
 * CostModelState::training_set (costmodel.hpp:48-57) of F families kept on the device across
 * retrains: train_cost_model's append (costmodel.cpp:224-233) sends only the new batch, and each
 * family's canonical row order (:161-173) is maintained by merge-insert instead of a full re-sort
 * per fit. A refit from the store is bit-identical to fs_fit on the family's rows in append order.
 * Rows [seg[k], seg[k+1]) of an append go to family[k]; target = log(latency_ms) (:232), computed
 * on the host like the reference. Empty batch or latency <= 0 -> FS_EINVAL (:225-231, nothing is
 * appended); unknown family -> FS_ERANGE. */
typedef struct fs_store fs_store;
int fs_store_create(fs_device* dev, int32_t n_families, int32_t d, fs_store** out);
int fs_store_destroy(fs_store* st);
int fs_store_append(fs_store* st, int32_t n_segments, const int32_t* family, const int64_t* seg,
                    const double* x, const double* latency_ms);
/* the same from measurement records (candidate descriptors, featurized on the device at d) */
int fs_store_append_records(fs_store* st, const fs_spaces* sp, int32_t n_segments,
                            const int32_t* family, const int64_t* seg, const int32_t* space_of,
                            const int32_t* assign, const double* latency_ms);
int fs_store_rows(const fs_store* st, int32_t family, int64_t* rows);
/* rows / targets in append order; canonical = family-relative row ids in canonical order when
 * *canonical_valid (a bulk append leaves it to the next fit). Any pointer may be NULL. */
int fs_store_read(const fs_store* st, int32_t family, double* x, double* target, int32_t* canonical,
                  int32_t* canonical_valid);
/* fit(model) (costmodel.cpp:152-222) of the listed store families on everything they hold;
 * results replace forest family families[k] with params[k]. */
int fs_store_fit(fs_store* st, fs_forest* fo, int32_t n_families, const int32_t* families,
                 const fs_gbt_params* params);

/* Fit diagnostics of the last fs_fit on this forest family: internal nodes resolved by the
 * histogram screen alone / by exact reference-order re-evaluation of the tie window. */
int fs_forest_fit_stats(const fs_forest* fo, int32_t family, int64_t* screened,
                        int64_t* exact_resolved);

#ifdef __cplusplus
}
#endif
#endif /* FAMSEER_H */
