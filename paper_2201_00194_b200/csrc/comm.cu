// Family-parallel tuning across the GPUs of one node: families share nothing
// (scheduler.cpp:123-130 - one CostModelState, training set and pool each), so each rank owns a
// deterministic set of families and scores / refits them on its own device exactly as one GPU
// would. The one exchange per tuning round is an all-gather of every family's top-g records
// (tune_step's by-score picks, scheduler.cpp:196-201), merged in family-id order on every rank.
//
//   fs_shard_families  deterministic LPT partition (host; ties by family id / rank)
//   fs_comm_*          an NCCL communicator per rank (libnccl.so.2 resolved at run time, so the
//                      library links without NCCL and a process may bring its own copy)
//   fs_topk_allgather  pack (device) -> ncclAllGather over NVLink / NVSwitch -> merge (device)
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "fs_common.cuh"

namespace {

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
  static Nccl n = [] {
    Nccl x;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      x.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (x.h) break;
    }
    if (!x.h) return x;
    x.get_unique_id = reinterpret_cast<decltype(x.get_unique_id)>(dlsym(x.h, "ncclGetUniqueId"));
    x.comm_init_rank = reinterpret_cast<decltype(x.comm_init_rank)>(dlsym(x.h, "ncclCommInitRank"));
    x.all_gather = reinterpret_cast<decltype(x.all_gather)>(dlsym(x.h, "ncclAllGather"));
    x.comm_destroy = reinterpret_cast<decltype(x.comm_destroy)>(dlsym(x.h, "ncclCommDestroy"));
    x.error_string = reinterpret_cast<decltype(x.error_string)>(dlsym(x.h, "ncclGetErrorString"));
    return x;
  }();
  if (!n.h || !n.get_unique_id || !n.comm_init_rank || !n.all_gather || !n.comm_destroy)
    fs::fail(FS_ENCCL, "NCCL (libnccl.so.2) is not available");
  return n;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const auto& n = nccl();
    fs::fail(FS_ENCCL, std::string(what) + ": " + (n.error_string ? n.error_string(r) : "NCCL error"));
  }
}

constexpr int kRec = 3;  // {family id, segment-local pool index, score} as float64

// Thread per (local family, record): the family's first g ranked candidates; short pools (and
// the unused family slots up to fam_cap) pad with family -1.
__global__ void topk_pack_kernel(int n_local, const int32_t* __restrict__ fam_ids, const int64_t* __restrict__ seg,
                                 const double* __restrict__ scores, const int32_t* __restrict__ perm, int g,
                                 int fam_cap, double* __restrict__ send) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<int64_t>(fam_cap) * g) return;
  const int i = static_cast<int>(t / g), k = static_cast<int>(t - static_cast<int64_t>(i) * g);
  double* r = send + t * kRec;
  if (i < n_local && seg[i] + k < seg[i + 1]) {
    const int32_t p = perm[seg[i] + k];
    r[0] = static_cast<double>(fam_ids[i]);
    r[1] = static_cast<double>(p);
    r[2] = scores[seg[i] + p];
  } else {
    r[0] = r[1] = r[2] = -1.0;
  }
}

__global__ void fill_kernel(double* __restrict__ a, int64_t n, double v) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < n) a[t] = v;
}

// Gathered records [world][fam_cap][g] -> merged [n_families][g][3] in family-id order (each family
// lives on exactly one rank; absent families keep the -1 fill).
__global__ void topk_scatter_kernel(const double* __restrict__ recv, int64_t n_rec, int g, int n_families,
                                    double* __restrict__ merged) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n_rec) return;
  const double* r = recv + t * kRec;
  const int f = static_cast<int>(r[0]);
  if (f < 0 || f >= n_families) return;
  const int k = static_cast<int>(t % g);
  double* o = merged + (static_cast<int64_t>(f) * g + k) * kRec;
  o[0] = r[0];
  o[1] = r[1];
  o[2] = r[2];
}

}  // namespace

struct fs_comm {
  fs_device* dev = nullptr;
  int world = 1, rank = 0;
  ncclComm_t comm = nullptr;
  double* send_d = nullptr;
  double* recv_d = nullptr;
  size_t cap = 0;  // records per rank the buffers hold
};

extern "C" {

int fs_shard_families(int32_t n_families, const int64_t* rows, const int64_t* pool, const int32_t* trees,
                      int32_t world, int32_t* owner) {
  return fs::guard([&] {
    if (n_families < 0 || world < 1 || (n_families > 0 && (!rows || !pool || !trees || !owner)))
      fs::fail(FS_EINVAL, "fs_shard_families: bad arguments");
    // cost = boosting work + scoring work (rows * T + pool * T); LPT: families by descending cost
    // (ties: lower id first), each to the least-loaded rank (ties: lower rank)
    std::vector<double> cost(static_cast<size_t>(n_families));
    for (int f = 0; f < n_families; ++f)
      cost[static_cast<size_t>(f)] = static_cast<double>(rows[f]) * trees[f] + static_cast<double>(pool[f]) * trees[f];
    std::vector<int> order(static_cast<size_t>(n_families));
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[static_cast<size_t>(a)] > cost[static_cast<size_t>(b)]; });
    std::vector<double> load(static_cast<size_t>(world), 0.0);
    for (int f : order) {
      int r = 0;
      for (int k = 1; k < world; ++k)
        if (load[static_cast<size_t>(k)] < load[static_cast<size_t>(r)]) r = k;
      owner[f] = r;
      load[static_cast<size_t>(r)] += cost[static_cast<size_t>(f)];
    }
  });
}

int fs_comm_id(uint8_t* id) {
  return fs::guard([&] {
    if (!id) fs::fail(FS_EINVAL, "fs_comm_id: NULL id");
    static_assert(sizeof(ncclUniqueId) <= FS_COMM_ID_BYTES, "NCCL unique id does not fit");
    ncclUniqueId u;
    nccl_check(nccl().get_unique_id(&u), "ncclGetUniqueId");
    std::memset(id, 0, FS_COMM_ID_BYTES);
    std::memcpy(id, &u, sizeof u);
  });
}

int fs_comm_create(fs_device* dev, int32_t world, int32_t rank, const uint8_t* id, fs_comm** out) {
  return fs::guard([&] {
    if (!dev || world < 1 || rank < 0 || rank >= world || !id || !out) fs::fail(FS_EINVAL, "fs_comm_create: bad arguments");
    dev->activate();
    auto c = std::make_unique<fs_comm>();
    c->dev = dev;
    c->world = world;
    c->rank = rank;
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    nccl_check(nccl().comm_init_rank(&c->comm, world, u, rank), "ncclCommInitRank");
    *out = c.release();
  });
}

int fs_comm_destroy(fs_comm* c) {
  return fs::guard([&] {
    if (!c) return;
    c->dev->activate();
    FS_CUDA(cudaStreamSynchronize(c->dev->stream));
    if (c->comm) nccl().comm_destroy(c->comm);
    if (c->send_d) cudaFree(c->send_d);
    if (c->recv_d) cudaFree(c->recv_d);
    delete c;
  });
}

int fs_topk_allgather(fs_comm* c, int32_t n_local, const int32_t* family_ids, const int64_t* seg_h,
                      const double* scores_d, const int32_t* perm_d, int32_t g, int32_t fam_cap, int32_t n_families,
                      double* merged_d) {
  return fs::guard([&] {
    if (!c || n_local < 0 || g < 1 || fam_cap < n_local || n_families < 0 || !merged_d ||
        (n_local > 0 && (!family_ids || !seg_h || !scores_d || !perm_d)))
      fs::fail(FS_EINVAL, "fs_topk_allgather: bad arguments");
    for (int i = 0; i < n_local; ++i)
      if (family_ids[i] < 0 || family_ids[i] >= n_families) fs::fail(FS_ERANGE, "fs_topk_allgather: family id out of range");
    fs_device* dev = c->dev;
    dev->activate();
    cudaStream_t s = dev->stream;
    const size_t per_rank = static_cast<size_t>(std::max(fam_cap, 1)) * g;
    if (per_rank > c->cap) {
      FS_CUDA(cudaStreamSynchronize(s));
      if (c->send_d) cudaFree(c->send_d);
      if (c->recv_d) cudaFree(c->recv_d);
      FS_CUDA(cudaMalloc(&c->send_d, per_rank * kRec * sizeof(double)));
      FS_CUDA(cudaMalloc(&c->recv_d, per_rank * c->world * kRec * sizeof(double)));
      c->cap = per_rank;
    }
    // the local families' segments and ids travel with the launch (tiny)
    std::vector<int64_t> segv(seg_h, seg_h + n_local + 1);
    auto* md = static_cast<int64_t*>(dev->scratch(fs::kSlotPredictSeg, segv.size() * sizeof(int64_t)));
    FS_CUDA(cudaMemcpyAsync(md, segv.data(), segv.size() * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    std::vector<int32_t> ids32(static_cast<size_t>(std::max(n_local, 1)), 0);
    for (int i = 0; i < n_local; ++i) ids32[static_cast<size_t>(i)] = family_ids[i];
    auto* idd = static_cast<int32_t*>(dev->scratch(fs::kSlotH2D2, ids32.size() * sizeof(int32_t)));
    FS_CUDA(cudaMemcpyAsync(idd, ids32.data(), ids32.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    const int64_t n_send = static_cast<int64_t>(fam_cap) * g;
    topk_pack_kernel<<<static_cast<unsigned>(fs::ceil_div(std::max<int64_t>(n_send, 1), 256)), 256, 0, s>>>(
        n_local, idd, md, scores_d, perm_d, g, fam_cap, c->send_d);
    dev->count_launch();
    FS_CUDA(cudaGetLastError());
    nccl_check(nccl().all_gather(c->send_d, c->recv_d, per_rank * kRec, ncclDouble, c->comm, s), "ncclAllGather");
    const int64_t n_out = static_cast<int64_t>(n_families) * g * kRec;
    if (n_out > 0) {
      fill_kernel<<<static_cast<unsigned>(fs::ceil_div(n_out, 256)), 256, 0, s>>>(merged_d, n_out, -1.0);
      const int64_t n_rec = static_cast<int64_t>(per_rank) * c->world;
      topk_scatter_kernel<<<static_cast<unsigned>(fs::ceil_div(n_rec, 256)), 256, 0, s>>>(c->recv_d, n_rec, g,
                                                                                        n_families, merged_d);
      dev->count_launch(2);
      FS_CUDA(cudaGetLastError());
    }
  });
}

}  // extern "C"
