// Device-resident family training store.
//
// The reference keeps every family's training set inside its CostModelState
// (costmodel.hpp:48-57), appends each measured batch (train_cost_model, costmodel.cpp:224-233)
// and refits from scratch, re-sorting the whole set into canonical row order (:161-173) every
// time although only g <= 64 rows arrive per tuning step (scheduler.cpp:228,235). fs_store keeps
// the rows on the device across retrains (the host sends only the new batch) and maintains each
// family's canonical order incrementally: a batch is ranked among itself, every new row finds
// its place in the stored order by binary search, and one merge pass writes the new order. A
// refit then skips the O(n log n * d) sort (fit.cuh FitRows); codes, duplicate-feature detection
// and the per-feature presorted lists are linear passes the fit recomputes.
//
// Rows stay in append order in x/target (one region per family, grown geometrically); only the
// int32 order moves. Equal keys are bitwise-identical rows unless the family holds a -0.0
// (+0.0 == -0.0 in the comparison): such a family is always re-sorted by the fit from its
// append-order rows, exactly as fs_fit would (its order is never taken from the store).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "fit.cuh"
#include "fs_common.cuh"

namespace fs {
void launch_featurize(fs_device* dev, const fs_spaces* sp, int64_t n, const int32_t* space_of_d,
                      const int32_t* assign_d, int32_t pad, double* out_d);
}  // namespace fs

struct fs_store {
  fs_device* dev = nullptr;
  int32_t F = 0, d = 0;
  std::vector<int64_t> row0, n, cap;  // per family: region start / rows held / region capacity
  std::vector<char> sorted;           // canon holds the family's canonical order
  int64_t cap_total = 0;
  double* x = nullptr;       // [cap_total][d] rows, append order within each region
  double* y = nullptr;       // [cap_total] targets (log latency)
  int32_t* canon = nullptr;  // [cap_total] family-relative row ids in canonical order
  void* stage_h = nullptr;   // pinned staging of one append (grow-only), reusable once up_evt passed
  size_t stage_cap = 0;
  cudaEvent_t up_evt = nullptr;
};

namespace fs {
namespace store {
namespace {

constexpr int kMergeMax = 4096;  // larger batches are left to the fit's sort (order saved back)

struct MergeJob {
  int64_t row0;  // family region
  int32_t n_old, g;
  int64_t a0;  // offset of the job's new-row entries in the A / L scratch
  int64_t b0;  // offset of the job's merged order in the B scratch
};

// lexicographic (features..., target), the reference's canonical key (costmodel.cpp:161-173)
__device__ __forceinline__ int row_cmp(const double* __restrict__ x, const double* __restrict__ y, int d, int64_t a,
                                       int64_t b) {
  const double* ra = x + a * d;
  const double* rb = x + b * d;
  for (int j = 0; j < d; ++j) {
    const double u = ra[j], v = rb[j];
    if (u < v) return -1;
    if (v < u) return 1;
  }
  const double u = y[a], v = y[b];
  if (u < v) return -1;
  if (v < u) return 1;
  return 0;
}

// Every new row of a job (one warp each): its rank among the batch (ties by arrival; lanes over
// the other batch rows) and its insertion point in the stored order (first stored row not below
// it) by a 32-ary search - each lane compares one pivot, the ballot count narrows the range ~33x
// per step, so a few dependent row compares replace log2(n) of them. In rank order: A =
// family-relative row id, L = insertion point (non-decreasing: lower_bound is monotone in the key).
__global__ void rank_insert_kernel(const MergeJob* __restrict__ jobs, const double* __restrict__ x,
                                   const double* __restrict__ y, int d, const int32_t* __restrict__ canon,
                                   int32_t* __restrict__ A, int32_t* __restrict__ L) {
  const MergeJob jb = jobs[blockIdx.y];
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= jb.g) return;
  const int64_t ri = jb.row0 + jb.n_old + i;
  int rank = 0;
  for (int j = lane; j < jb.g; j += 32) {
    if (j == i) continue;
    const int c = row_cmp(x, y, d, jb.row0 + jb.n_old + j, ri);
    rank += c < 0 || (c == 0 && j < i);
  }
  rank = __reduce_add_sync(0xffffffffu, rank);
  int lo = 0, hi = jb.n_old;
  while (hi > lo) {
    const int m = hi - lo;
    if (m <= 32) {
      const bool lt = lane < m && row_cmp(x, y, d, jb.row0 + canon[jb.row0 + lo + lane], ri) < 0;
      lo += __popc(__ballot_sync(0xffffffffu, lt));
      break;
    }
    const int q = lo + static_cast<int>((static_cast<int64_t>(lane) + 1) * m / 33);
    const bool lt = row_cmp(x, y, d, jb.row0 + canon[jb.row0 + q], ri) < 0;
    const int c = __popc(__ballot_sync(0xffffffffu, lt));  // the pivots below the key form a prefix
    const int qlo = __shfl_sync(0xffffffffu, q, c > 0 ? c - 1 : 0);
    const int qhi = __shfl_sync(0xffffffffu, q, c < 32 ? c : 31);
    if (c > 0) lo = qlo + 1;
    if (c < 32) hi = qhi;
  }
  if (lane == 0) {
    A[jb.a0 + rank] = jb.n_old + i;
    L[jb.a0 + rank] = lo;
  }
}

struct SegDst {
  int64_t src0;  // first row of the segment in the staged batch
  int64_t dst;   // its first store row
};

// staged batch rows (features, targets) into their families' store regions
__global__ void place_kernel(const SegDst* __restrict__ segs, int nseg, int64_t n, int d, const double* __restrict__ xs,
                             const double* __restrict__ ys, double* __restrict__ x, double* __restrict__ y) {
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n * (d + 1);
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e / (d + 1);
    const int j = static_cast<int>(e - i * (d + 1));
    int lo = 0, hi = nseg - 1;  // last segment with src0 <= i
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (segs[mid].src0 <= i) lo = mid;
      else hi = mid - 1;
    }
    const int64_t r = segs[lo].dst + (i - segs[lo].src0);
    if (j < d) x[r * d + j] = xs[i * d + j];
    else y[r] = ys[i];
  }
}

// merged order: stored row k moves up by the new rows inserted at or before it; new row r lands
// at L[r] + r (L is non-decreasing in r)
__global__ void merge_kernel(const MergeJob* __restrict__ jobs, const int32_t* __restrict__ canon,
                             const int32_t* __restrict__ A, const int32_t* __restrict__ L, int32_t* __restrict__ B) {
  const MergeJob jb = jobs[blockIdx.y];
  const int tot = jb.n_old + jb.g;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < tot; q += gridDim.x * blockDim.x) {
    if (q < jb.n_old) {
      int lo = 0, hi = jb.g;  // #{r : L[r] <= q}
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (L[jb.a0 + mid] <= q) lo = mid + 1;
        else hi = mid;
      }
      B[jb.b0 + q + lo] = canon[jb.row0 + q];
    } else {
      const int r = q - jb.n_old;
      B[jb.b0 + L[jb.a0 + r] + r] = A[jb.a0 + r];
    }
  }
}

__global__ void merge_store_kernel(const MergeJob* __restrict__ jobs, const int32_t* __restrict__ B,
                                   int32_t* __restrict__ canon) {
  const MergeJob jb = jobs[blockIdx.y];
  const int tot = jb.n_old + jb.g;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < tot; q += gridDim.x * blockDim.x)
    canon[jb.row0 + q] = B[jb.b0 + q];
}

template <class T>
T* dev_alloc(fs_device* dev, size_t count) {
  void* p = nullptr;
  FS_CUDA(cudaMallocAsync(&p, std::max<size_t>(count, 1) * sizeof(T), dev->stream));
  return static_cast<T*>(p);
}

// room for `need[f]` rows in every family: regions are re-laid out with geometric growth
void reserve(fs_store* st, const std::vector<int64_t>& need) {
  bool grow = false;
  for (int f = 0; f < st->F; ++f) grow |= need[static_cast<size_t>(f)] > st->cap[static_cast<size_t>(f)];
  if (!grow) return;
  fs_device* dev = st->dev;
  cudaStream_t s = dev->stream;
  std::vector<int64_t> cap(st->cap), row0(static_cast<size_t>(st->F));
  int64_t tot = 0;
  for (int f = 0; f < st->F; ++f) {
    int64_t& c = cap[static_cast<size_t>(f)];
    const int64_t want = need[static_cast<size_t>(f)];
    if (want > c) c = std::max<int64_t>(want, c + c / 2 + 64);
    row0[static_cast<size_t>(f)] = tot;
    tot += c;
  }
  const size_t d = static_cast<size_t>(std::max(st->d, 1));
  double* x = dev_alloc<double>(dev, static_cast<size_t>(tot) * d);
  double* y = dev_alloc<double>(dev, static_cast<size_t>(tot));
  int32_t* canon = dev_alloc<int32_t>(dev, static_cast<size_t>(tot));
  for (int f = 0; f < st->F; ++f) {
    const int64_t n = st->n[static_cast<size_t>(f)];
    if (n == 0) continue;
    const int64_t o = st->row0[static_cast<size_t>(f)], p = row0[static_cast<size_t>(f)];
    if (st->d > 0)
      FS_CUDA(cudaMemcpyAsync(x + p * st->d, st->x + o * st->d, static_cast<size_t>(n) * st->d * sizeof(double),
                              cudaMemcpyDeviceToDevice, s));
    FS_CUDA(cudaMemcpyAsync(y + p, st->y + o, static_cast<size_t>(n) * sizeof(double), cudaMemcpyDeviceToDevice, s));
    FS_CUDA(cudaMemcpyAsync(canon + p, st->canon + o, static_cast<size_t>(n) * sizeof(int32_t),
                            cudaMemcpyDeviceToDevice, s));
  }
  if (st->x) FS_CUDA(cudaFreeAsync(st->x, s));
  if (st->y) FS_CUDA(cudaFreeAsync(st->y, s));
  if (st->canon) FS_CUDA(cudaFreeAsync(st->canon, s));
  st->x = x;
  st->y = y;
  st->canon = canon;
  st->cap = cap;
  st->row0 = row0;
  st->cap_total = tot;
}

inline size_t al16(size_t v) { return (v + 15) & ~size_t(15); }

// Rows [seg[k], seg[k+1]) of the call belong to family fam[k]. One pinned staging buffer carries
// the batch (targets, segment table, merge jobs and either the feature rows or the record
// descriptors) in one copy; `records` featurizes the descriptors on the device. Then one kernel
// places the rows and three kernels merge every appended family's canonical order.
void append(fs_store* st, int32_t nseg, const int32_t* fam, const int64_t* seg, const double* latency,
            const double* x_h, const fs_spaces* sp, const int32_t* so_h, const int32_t* a_h) {
  fs_device* dev = st->dev;
  cudaStream_t s = dev->stream;
  if (nseg < 1 || !fam || !seg || !latency) fail(FS_EINVAL, "fs_store_append: bad arguments");
  if (seg[0] != 0) fail(FS_EINVAL, "fs_store_append: seg[0] must be 0");
  std::vector<int64_t> add(static_cast<size_t>(st->F), 0);
  for (int k = 0; k < nseg; ++k) {
    if (fam[k] < 0 || fam[k] >= st->F) fail(FS_ERANGE, "fs_store_append: unknown family id");
    const int64_t g = seg[k + 1] - seg[k];
    if (g <= 0) fail(FS_EINVAL, "train_cost_model: empty record batch");  // costmodel.cpp:225-227
    add[static_cast<size_t>(fam[k])] += g;
  }
  const int64_t n_in = seg[nseg];
  for (int64_t i = 0; i < n_in; ++i)
    if (!(latency[i] > 0.0)) fail(FS_EINVAL, "train_cost_model: non-positive latency");  // :229-231
  std::vector<int64_t> need(st->n);
  for (int f = 0; f < st->F; ++f) {
    need[static_cast<size_t>(f)] += add[static_cast<size_t>(f)];
    if (need[static_cast<size_t>(f)] > (1 << 30)) fail(FS_EINVAL, "fs_store_append: family larger than 2^30 rows");
  }
  reserve(st, need);
  const int d = st->d;
  // segment destinations, merge jobs
  std::vector<SegDst> segs(static_cast<size_t>(nseg));
  std::vector<int64_t> at(st->n);
  for (int k = 0; k < nseg; ++k) {
    const int f = fam[k];
    segs[static_cast<size_t>(k)] = {seg[k], st->row0[static_cast<size_t>(f)] + at[static_cast<size_t>(f)]};
    at[static_cast<size_t>(f)] += seg[k + 1] - seg[k];
  }
  std::vector<MergeJob> jobs;
  int64_t a_tot = 0, b_tot = 0;
  int gmax = 0, tmax = 0;
  for (int f = 0; f < st->F; ++f) {
    const int64_t g = add[static_cast<size_t>(f)];
    if (g == 0) continue;
    const int64_t n_old = st->n[static_cast<size_t>(f)];
    st->n[static_cast<size_t>(f)] += g;
    if (!st->sorted[static_cast<size_t>(f)]) continue;
    if (g > kMergeMax) {  // a bulk load: the next fit sorts and records the order
      st->sorted[static_cast<size_t>(f)] = 0;
      continue;
    }
    MergeJob jb;
    jb.row0 = st->row0[static_cast<size_t>(f)];
    jb.n_old = static_cast<int32_t>(n_old);
    jb.g = static_cast<int32_t>(g);
    jb.a0 = a_tot;
    jb.b0 = b_tot;
    a_tot += g;
    b_tot += jb.n_old + g;
    gmax = std::max(gmax, jb.g);
    tmax = std::max(tmax, jb.n_old + jb.g);
    jobs.push_back(jb);
  }
  // staging layout (16-byte aligned sections), mirrored on the device
  const bool rec = sp != nullptr;
  const size_t o_y = 0, o_seg = al16(o_y + n_in * sizeof(double));
  const size_t o_job = al16(o_seg + segs.size() * sizeof(SegDst));
  const size_t o_in = al16(o_job + jobs.size() * sizeof(MergeJob));
  const size_t in_bytes = rec ? static_cast<size_t>(n_in) * (1 + FS_MAX_KNOBS) * sizeof(int32_t)
                              : static_cast<size_t>(n_in) * d * sizeof(double);
  const size_t staged = al16(o_in + in_bytes);
  if (st->up_evt) FS_CUDA(cudaEventSynchronize(st->up_evt));
  if (staged > st->stage_cap) {
    if (st->stage_h) FS_CUDA(cudaFreeHost(st->stage_h));
    st->stage_h = nullptr;
    st->stage_cap = std::max<size_t>(staged + staged / 2, 1 << 16);
    FS_CUDA(cudaHostAlloc(&st->stage_h, st->stage_cap, cudaHostAllocDefault));
  }
  auto* h = static_cast<unsigned char*>(st->stage_h);
  auto* yh = reinterpret_cast<double*>(h + o_y);
  for (int64_t i = 0; i < n_in; ++i) yh[i] = std::log(latency[i]);  // costmodel.cpp:232 (std::log, host)
  std::memcpy(h + o_seg, segs.data(), segs.size() * sizeof(SegDst));
  if (!jobs.empty()) std::memcpy(h + o_job, jobs.data(), jobs.size() * sizeof(MergeJob));
  if (rec) {
    std::memcpy(h + o_in, so_h, static_cast<size_t>(n_in) * sizeof(int32_t));
    std::memcpy(h + o_in + static_cast<size_t>(n_in) * sizeof(int32_t), a_h,
                static_cast<size_t>(n_in) * FS_MAX_KNOBS * sizeof(int32_t));
  } else if (in_bytes) {
    std::memcpy(h + o_in, x_h, in_bytes);
  }
  const size_t o_x = al16(staged);  // featurized rows (records form)
  const size_t o_A = al16(o_x + (rec ? static_cast<size_t>(n_in) * d * sizeof(double) : 0));
  const size_t o_L = al16(o_A + a_tot * sizeof(int32_t));
  const size_t o_B = al16(o_L + a_tot * sizeof(int32_t));
  const size_t dev_bytes = al16(o_B + b_tot * sizeof(int32_t));
  unsigned char* D = dev_alloc<unsigned char>(dev, dev_bytes);
  FS_CUDA(cudaMemcpyAsync(D, h, staged, cudaMemcpyHostToDevice, s));
  if (!st->up_evt) FS_CUDA(cudaEventCreateWithFlags(&st->up_evt, cudaEventDisableTiming));
  FS_CUDA(cudaEventRecord(st->up_evt, s));
  const double* xs = reinterpret_cast<const double*>(D + (rec ? o_x : o_in));
  if (rec) {
    const auto* so_d = reinterpret_cast<const int32_t*>(D + o_in);
    launch_featurize(dev, sp, n_in, so_d, so_d + n_in, d, reinterpret_cast<double*>(D + o_x));
  }
  const int64_t work = n_in * (d + 1);
  place_kernel<<<static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, dev->sm_count * 8))),
                 256, 0, s>>>(reinterpret_cast<const SegDst*>(D + o_seg), nseg, n_in, d, xs,
                              reinterpret_cast<const double*>(D + o_y), st->x, st->y);
  dev->count_launch();
  if (!jobs.empty()) {
    const auto* jobs_d = reinterpret_cast<const MergeJob*>(D + o_job);
    auto* A = reinterpret_cast<int32_t*>(D + o_A);
    auto* L = reinterpret_cast<int32_t*>(D + o_L);
    auto* B = reinterpret_cast<int32_t*>(D + o_B);
    const unsigned J = static_cast<unsigned>(jobs.size());
    rank_insert_kernel<<<dim3(static_cast<unsigned>((gmax + 7) / 8), J), 256, 0, s>>>(jobs_d, st->x, st->y, d,
                                                                                      st->canon, A, L);
    const unsigned tb = static_cast<unsigned>(std::min(64, (tmax + 255) / 256));
    merge_kernel<<<dim3(tb, J), 256, 0, s>>>(jobs_d, st->canon, A, L, B);
    merge_store_kernel<<<dim3(tb, J), 256, 0, s>>>(jobs_d, B, st->canon);
    dev->count_launch(3);
  }
  FS_CUDA(cudaGetLastError());
  FS_CUDA(cudaFreeAsync(D, s));
}

}  // namespace
}  // namespace store
}  // namespace fs

extern "C" {

int fs_store_create(fs_device* dev, int32_t n_families, int32_t d, fs_store** out) {
  return fs::guard([&] {
    if (!dev || n_families < 0 || d < 0 || !out) fs::fail(FS_EINVAL, "fs_store_create: bad arguments");
    dev->activate();
    auto* st = new fs_store();
    st->dev = dev;
    st->F = n_families;
    st->d = d;
    st->row0.assign(static_cast<size_t>(n_families), 0);
    st->n.assign(static_cast<size_t>(n_families), 0);
    st->cap.assign(static_cast<size_t>(n_families), 0);
    st->sorted.assign(static_cast<size_t>(n_families), 1);  // the empty order is sorted
    *out = st;
  });
}

int fs_store_destroy(fs_store* st) {
  return fs::guard([&] {
    if (!st) return;
    st->dev->activate();
    cudaStream_t s = st->dev->stream;
    if (st->x) FS_CUDA(cudaFreeAsync(st->x, s));
    if (st->y) FS_CUDA(cudaFreeAsync(st->y, s));
    if (st->canon) FS_CUDA(cudaFreeAsync(st->canon, s));
    if (st->up_evt) {
      FS_CUDA(cudaEventSynchronize(st->up_evt));
      FS_CUDA(cudaEventDestroy(st->up_evt));
    }
    if (st->stage_h) FS_CUDA(cudaFreeHost(st->stage_h));
    delete st;
  });
}

int fs_store_append(fs_store* st, int32_t n_segments, const int32_t* family, const int64_t* seg, const double* x,
                    const double* latency_ms) {
  return fs::guard([&] {
    if (!st || (!x && st->d > 0)) fs::fail(FS_EINVAL, "fs_store_append: bad arguments");
    st->dev->activate();
    fs::store::append(st, n_segments, family, seg, latency_ms, x, nullptr, nullptr, nullptr);
  });
}

int fs_store_append_records(fs_store* st, const fs_spaces* sp, int32_t n_segments, const int32_t* family,
                            const int64_t* seg, const int32_t* space_of, const int32_t* assign,
                            const double* latency_ms) {
  return fs::guard([&] {
    if (!st || !sp || !space_of || !assign || !seg || n_segments < 1)
      fs::fail(FS_EINVAL, "fs_store_append_records: bad arguments");
    st->dev->activate();
    const int64_t n = seg[n_segments];
    for (int64_t i = 0; i < n; ++i) {  // searchspace.cpp:94-101, checked on the host as fs_fit_records does
      const int s = space_of[i];
      if (s < 0 || s >= sp->n) fs::fail(FS_EINVAL, "fs_store_append_records: unknown space id");
      if (st->d < fs_feature_dim(sp->k_h[static_cast<size_t>(s)]))
        fs::fail(FS_EINVAL, "fs_store_append_records: pad_dim too small");
    }
    fs::store::append(st, n_segments, family, seg, latency_ms, nullptr, sp, space_of, assign);
  });
}

int fs_store_rows(const fs_store* st, int32_t family, int64_t* rows) {
  return fs::guard([&] {
    if (!st || !rows) fs::fail(FS_EINVAL, "fs_store_rows: bad arguments");
    if (family < 0 || family >= st->F) fs::fail(FS_ERANGE, "fs_store_rows: unknown family id");
    *rows = st->n[static_cast<size_t>(family)];
  });
}

int fs_store_read(const fs_store* st, int32_t family, double* x, double* target, int32_t* canonical,
                  int32_t* canonical_valid) {
  return fs::guard([&] {
    if (!st) fs::fail(FS_EINVAL, "fs_store_read: bad arguments");
    if (family < 0 || family >= st->F) fs::fail(FS_ERANGE, "fs_store_read: unknown family id");
    st->dev->activate();
    cudaStream_t s = st->dev->stream;
    const int64_t n = st->n[static_cast<size_t>(family)], r = st->row0[static_cast<size_t>(family)];
    if (n > 0 && x && st->d > 0)
      FS_CUDA(cudaMemcpyAsync(x, st->x + r * st->d, static_cast<size_t>(n) * st->d * sizeof(double),
                              cudaMemcpyDeviceToHost, s));
    if (n > 0 && target)
      FS_CUDA(cudaMemcpyAsync(target, st->y + r, static_cast<size_t>(n) * sizeof(double), cudaMemcpyDeviceToHost, s));
    const bool ok = st->sorted[static_cast<size_t>(family)] != 0;
    if (n > 0 && canonical && ok)
      FS_CUDA(cudaMemcpyAsync(canonical, st->canon + r, static_cast<size_t>(n) * sizeof(int32_t),
                              cudaMemcpyDeviceToHost, s));
    if (canonical_valid) *canonical_valid = ok ? 1 : 0;
    FS_CUDA(cudaStreamSynchronize(s));
  });
}

int fs_store_fit(fs_store* st, fs_forest* fo, int32_t n_families, const int32_t* families,
                 const fs_gbt_params* params) {
  return fs::guard([&] {
    if (!st || !fo || n_families < 0 || (n_families > 0 && (!families || !params)))
      fs::fail(FS_EINVAL, "fs_store_fit: bad arguments");
    if (n_families == 0) return;
    st->dev->activate();
    std::vector<char> seen(static_cast<size_t>(st->F), 0);
    std::vector<int64_t> seg(static_cast<size_t>(n_families) + 1, 0), row0(static_cast<size_t>(n_families));
    std::vector<int> io(static_cast<size_t>(n_families)), negz(static_cast<size_t>(n_families), 0);
    for (int k = 0; k < n_families; ++k) {
      const int f = families[k];
      if (f < 0 || f >= st->F) fs::fail(FS_ERANGE, "fs_store_fit: unknown family id");
      if (seen[static_cast<size_t>(f)]) fs::fail(FS_EINVAL, "fs_store_fit: family listed twice");
      seen[static_cast<size_t>(f)] = 1;
      seg[static_cast<size_t>(k) + 1] = seg[static_cast<size_t>(k)] + st->n[static_cast<size_t>(f)];
      row0[static_cast<size_t>(k)] = st->row0[static_cast<size_t>(f)];
      io[static_cast<size_t>(k)] = st->sorted[static_cast<size_t>(f)] ? 1 : 2;
    }
    fs::fit::FitRows rows;
    rows.row0 = row0.data();
    rows.fam_id = families;
    rows.span = st->cap_total;
    rows.canon = st->canon;
    rows.io = io.data();
    rows.negz_out = negz.data();
    fs::fit::fit_families(st->dev, fo, n_families, seg.data(), st->d, st->x, st->y, params, &rows);
    for (int k = 0; k < n_families; ++k)
      if (io[static_cast<size_t>(k)] == 2 && !negz[static_cast<size_t>(k)] && seg[k + 1] > seg[k])
        st->sorted[static_cast<size_t>(families[k])] = 1;
  });
}

}  // extern "C"
