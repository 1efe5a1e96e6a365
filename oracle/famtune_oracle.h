/* TEST INFRASTRUCTURE ONLY - CPU restatement of the reference hot path (famtune, the FamilySeer
 * reference), used exclusively as the parity checker by tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py. Never linked into, or called by, the product path.
 *
 * Pinned against: the reference's own exact-value tests (searchspace_test.cpp:59-76,
 * costmodel_test.cpp:77-158) via tests/golden/, and differentially against the unmodified
 * reference core compiled into oracle/_ref/ (tests/test_oracle.py).
 *
 * Model layout (shared with the product C ABI): trees are concatenated in pre-order, tree t owns
 * nodes [offsets[t], offsets[t+1]); feature < 0 marks a leaf; left/right are tree-local indices
 * (costmodel.hpp:27-41). */
#ifndef FAMTUNE_ORACLE_H
#define FAMTUNE_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_EDOMAIN = 2, ORC_ERANGE = 3 };

const char* orc_last_error(void);

int orc_feature_dim(int k);

void orc_linear_index(int k, const int32_t* nvals, const int32_t* assign, int64_t p, int assign_stride,
                      uint64_t* out);
void orc_candidate_from_index(int k, const int32_t* nvals, const uint64_t* index, int64_t p, int assign_stride,
                              int32_t* out);
int orc_featurize(int k, const int32_t* nvals, const int64_t* values, const int32_t* assign,
                  int64_t p, int assign_stride, int pad_dim, double* out);

int orc_predict(double base, double lr, int n_trees, const int32_t* offsets,
                const int32_t* feature, const double* threshold, const int32_t* left,
                const int32_t* right, const double* value, int64_t p, int d, const double* x,
                double* out, uint16_t* leaf_out);

int orc_rank(int64_t p, const double* scores, int64_t* perm);

int orc_fit(int64_t n, int d, const double* x, const double* target, int trees, int depth,
            double lr, int min_split, double* base, int* n_trees_out, int32_t* offsets,
            int32_t* feature, double* threshold, int32_t* left, int32_t* right, double* value,
            double* gain, double* mse, int64_t node_cap);

int orc_pairwise_accuracy(const double* scores, const double* latency, int64_t n, double* out);

/* tune_step selection (scheduler.cpp:184-213) over an already-ranked pool. rng_state is an
 * mt19937_64 stream seeded with `stream_seed` (the caller derives it with mix_seed). Writes
 * g_eff pool indices to picks; returns the count. */
int orc_select(int64_t p, const int64_t* perm, int g_eff, double epsilon, uint64_t stream_seed,
               int64_t* picks);

uint64_t orc_mix_seed(uint64_t seed, uint64_t a, uint64_t b);

#ifdef __cplusplus
}
#endif
#endif
