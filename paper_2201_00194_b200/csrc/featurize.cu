// Kernel (1): batched feature extraction - featurize (searchspace.cpp:90-118) for a whole
// candidate population at once.
//
// Layout: one warp per candidate row. Lane k < K looks up knob k's log2(value) and normalized
// position from the space table; every output feature is then formed from warp shuffles, so the
// row is written as full 256-byte coalesced stores (the write of pad_dim*8 bytes per candidate is
// the only real HBM traffic; algorithmic bytes = 4*16 + 8*pad_dim per candidate).
//
// Bit-exactness: log2 tables are built on the host with the C library's log2 (the function
// std::log2 dispatches to in the reference); positions are IEEE divisions idx/(m-1) (also done
// on the host); pair products are single __dmul_rn roundings - the reference's
// `logs[i] * logs[j]` (searchspace.cpp:114) compiled without FMA.
#include <algorithm>
#include <cmath>
#include <memory>
#include <type_traits>
#include <vector>

#include "fs_common.cuh"


namespace {

__global__ void __launch_bounds__(256) featurize_kernel(const int32_t* __restrict__ space_of,
                                                        const int32_t* __restrict__ assign, int64_t n,
                                                        int pad, int n_spaces,
                                                        const int32_t* __restrict__ k_tab,
                                                        const int32_t* __restrict__ nval_tab,
                                                        const int32_t* __restrict__ off_tab,
                                                        const double* __restrict__ log_tab,
                                                        const double* __restrict__ pos_tab,
                                                        double* __restrict__ out, uint32_t* err) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t c = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; c < n; c += warps) {
    const int s = __ldg(space_of + c);
    double* o = out + c * pad;
    if (s < 0 || s >= n_spaces) {
      if (lane == 0) atomicOr(err, fs::kErrSpaceId);
      for (int j = lane; j < pad; j += 32) o[j] = 0.0;
      continue;
    }
    const int k = __ldg(k_tab + s);
    const int dim = 2 * k + k * (k - 1) / 2;
    double lg = 0.0, ps = 0.0;
    bool bad = false;
    if (lane < k) {
      const int a = __ldg(assign + c * FS_MAX_KNOBS + lane);
      const int m = __ldg(nval_tab + s * FS_MAX_KNOBS + lane);
      if (a < 0 || a >= m) {
        bad = true;
      } else {
        const int off = __ldg(off_tab + s * FS_MAX_KNOBS + lane);
        lg = __ldg(log_tab + off + a);
        ps = __ldg(pos_tab + off + a);
      }
    }
    const unsigned any_bad = __ballot_sync(0xffffffffu, bad);
    if (lane == 0) {
      if (any_bad) atomicOr(err, fs::kErrKnobRange);
      if (pad < dim) atomicOr(err, fs::kErrPadDim);
    }
    for (int base = 0; base < pad; base += 32) {
      const int j = base + lane;
      int src_a = 0, src_b = 0, kind = 0;  // 0 zero, 1 log, 2 pos, 3 product
      if (j < k) {
        kind = 1;
        src_a = j;
      } else if (j < 2 * k) {
        kind = 2;
        src_a = j - k;
      } else if (j < dim) {
        kind = 3;
        fs::pair_of(k, j - 2 * k, src_a, src_b);
      }
      const double la = __shfl_sync(0xffffffffu, lg, src_a);
      const double lb = __shfl_sync(0xffffffffu, lg, src_b);
      const double pa = __shfl_sync(0xffffffffu, ps, src_a);
      double v = 0.0;
      if (kind == 1) v = la;
      else if (kind == 2) v = pa;
      else if (kind == 3) v = fs_mul(la, lb);
      if (j < pad) o[j] = v;
    }
  }
}

}  // namespace

namespace fs {

void launch_featurize(fs_device* dev, const fs_spaces* sp, int64_t n, const int32_t* space_of_d,
                      const int32_t* assign_d, int32_t pad, double* out_d) {
  if (n <= 0) return;
  const int block = 256;
  const int64_t want = ceil_div(n, block / 32);
  const int grid = static_cast<int>(std::min<int64_t>(want, static_cast<int64_t>(dev->sm_count) * 8));
  ProfScope prof(dev, "featurize");
  featurize_kernel<<<grid, block, 0, dev->stream>>>(space_of_d, assign_d, n, pad, sp->n, sp->k_d, sp->nval_d,
                                                     sp->off_d, sp->log_d, sp->pos_d, out_d, dev->err_d);
  dev->count_launch();
  FS_CUDA(cudaGetLastError());
}

}  // namespace fs

extern "C" {

int fs_spaces_create(fs_device* dev, int32_t n_spaces, const int32_t* n_knobs, const int32_t* n_values,
                     const int64_t* values, fs_spaces** out) {
  return fs::guard([&] {
    if (!dev || !out || n_spaces < 1 || !n_knobs || !n_values || !values)
      fs::fail(FS_EINVAL, "fs_spaces_create: bad arguments");
    dev->activate();
    auto sp = std::make_unique<fs_spaces>();
    sp->dev = dev;
    sp->n = n_spaces;
    std::vector<int32_t> nval(static_cast<size_t>(n_spaces) * FS_MAX_KNOBS, 0);
    std::vector<int32_t> off(static_cast<size_t>(n_spaces) * FS_MAX_KNOBS, 0);
    std::vector<double> lg, ps;
    int64_t src = 0;
    for (int s = 0; s < n_spaces; ++s) {
      const int k = n_knobs[s];
      // validate_space (searchspace.cpp:21-45): 1..16 knobs, non-empty lists, values >= 1.
      if (k < 1 || k > FS_MAX_KNOBS) fs::fail(FS_EINVAL, "knob space: knob count must be in [1, 16]");
      sp->k_h.push_back(k);
      sp->max_fd = std::max(sp->max_fd, fs_feature_dim(k));
      for (int i = 0; i < k; ++i) {
        const int m = n_values[s * FS_MAX_KNOBS + i];
        if (m < 1) fs::fail(FS_EINVAL, "knob space: knob has no values");
        nval[static_cast<size_t>(s) * FS_MAX_KNOBS + i] = m;
        off[static_cast<size_t>(s) * FS_MAX_KNOBS + i] = static_cast<int32_t>(lg.size());
        for (int a = 0; a < m; ++a) {
          const int64_t v = values[src++];
          if (v < 1) fs::fail(FS_EINVAL, "knob space: non-positive value");
          lg.push_back(std::log2(static_cast<double>(v)));  // searchspace.cpp:103
          ps.push_back(m > 1 ? static_cast<double>(a) / static_cast<double>(m - 1) : 0.0);  // :106
        }
      }
    }
    // mixed-radix strides of linear_index (searchspace.cpp:48-54): idx = sum_j a_j * prod_{k>j} m_k
    // (wraps modulo 2^64 like the reference's unsigned arithmetic once a space exceeds 2^64)
    std::vector<uint64_t> stride(static_cast<size_t>(n_spaces) * FS_MAX_KNOBS, 0);
    for (int s = 0; s < n_spaces; ++s) {
      uint64_t st = 1;
      for (int i = sp->k_h[static_cast<size_t>(s)] - 1; i >= 0; --i) {
        stride[static_cast<size_t>(s) * FS_MAX_KNOBS + i] = st;
        st *= static_cast<uint64_t>(nval[static_cast<size_t>(s) * FS_MAX_KNOBS + i]);
      }
    }
    auto up = [&](auto*& dst, const auto& vec) {
      using T = std::remove_reference_t<decltype(*dst)>;
      FS_CUDA(cudaMalloc(&dst, std::max<size_t>(1, vec.size()) * sizeof(T)));
      if (!vec.empty())
        FS_CUDA(cudaMemcpyAsync(dst, vec.data(), vec.size() * sizeof(T), cudaMemcpyHostToDevice, dev->stream));
    };
    up(sp->k_d, sp->k_h);
    up(sp->nval_d, nval);
    up(sp->off_d, off);
    up(sp->log_d, lg);
    up(sp->pos_d, ps);
    up(sp->stride_d, stride);
    FS_CUDA(cudaStreamSynchronize(dev->stream));
    *out = sp.release();
  });
}

int fs_spaces_destroy(fs_spaces* sp) {
  return fs::guard([&] {
    if (!sp) return;
    sp->dev->activate();
    FS_CUDA(cudaStreamSynchronize(sp->dev->stream));
    cudaFree(sp->k_d);
    cudaFree(sp->nval_d);
    cudaFree(sp->off_d);
    cudaFree(sp->log_d);
    cudaFree(sp->pos_d);
    cudaFree(sp->stride_d);
    delete sp;
  });
}

int32_t fs_spaces_max_feature_dim(const fs_spaces* sp) { return sp ? sp->max_fd : -1; }

int fs_featurize_d(fs_device* dev, const fs_spaces* sp, int64_t n, const int32_t* space_of_d,
                   const int32_t* assign_d, int32_t pad_dim, double* out_d) {
  return fs::guard([&] {
    if (!dev || !sp || n < 0 || pad_dim < 0) fs::fail(FS_EINVAL, "fs_featurize: bad arguments");
    dev->activate();
    fs::launch_featurize(dev, sp, n, space_of_d, assign_d, pad_dim, out_d);
  });
}

int fs_featurize(fs_device* dev, const fs_spaces* sp, int64_t n, const int32_t* space_of,
                 const int32_t* assign, int32_t pad_dim, double* out) {
  return fs::guard([&] {
    if (!dev || !sp || n < 0 || pad_dim < 0) fs::fail(FS_EINVAL, "fs_featurize: bad arguments");
    if (n == 0) return;
    dev->activate();
    // Host-side the reference checks pad_dim before touching the assignment (searchspace.cpp:96).
    for (int64_t i = 0; i < n; ++i) {
      const int s = space_of[i];
      if (s < 0 || s >= sp->n) fs::fail(FS_EINVAL, "featurize: unknown space id");
      if (pad_dim < fs_feature_dim(sp->k_h[static_cast<size_t>(s)]))
        fs::fail(FS_EINVAL, "featurize: pad_dim " + std::to_string(pad_dim) + " smaller than feature dim " +
                                std::to_string(fs_feature_dim(sp->k_h[static_cast<size_t>(s)])));
    }
    auto* sd = static_cast<int32_t*>(dev->scratch(fs::kSlotH2D0, n * sizeof(int32_t)));
    auto* ad = static_cast<int32_t*>(dev->scratch(fs::kSlotH2D1, n * FS_MAX_KNOBS * sizeof(int32_t)));
    auto* od = static_cast<double*>(dev->scratch(fs::kSlotD2H0, n * pad_dim * sizeof(double)));
    FS_CUDA(cudaMemcpyAsync(sd, space_of, n * sizeof(int32_t), cudaMemcpyHostToDevice, dev->stream));
    FS_CUDA(cudaMemcpyAsync(ad, assign, n * FS_MAX_KNOBS * sizeof(int32_t), cudaMemcpyHostToDevice, dev->stream));
    fs::launch_featurize(dev, sp, n, sd, ad, pad_dim, od);
    FS_CUDA(cudaMemcpyAsync(out, od, n * pad_dim * sizeof(double), cudaMemcpyDeviceToHost, dev->stream));
    fs::raise_deferred(dev->take_errors());
  });
}

}  // extern "C"
