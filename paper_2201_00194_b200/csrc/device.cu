// fs_device: one context per GPU (stream, scratch arena, deferred-error word, launch counter).
#include <algorithm>
#include <cstdio>
#include <string>

#include "fs_common.cuh"

namespace fs {

static thread_local std::string g_last_error;

void set_last_error(const std::string& msg) { g_last_error = msg; }

void raise_deferred(uint32_t bits) {
  if (bits & kErrNonFinitePredict) fail(FS_EINVAL, "predict: non-finite feature");
  if (bits & kErrNonFiniteFit) fail(FS_EINVAL, "cost model: non-finite feature");
  if (bits & kErrPadDim) fail(FS_EINVAL, "featurize: pad_dim smaller than feature dim");
  if (bits & kErrKnobRange) fail(FS_EINVAL, "featurize: knob value index out of range");
  if (bits & kErrSpaceId) fail(FS_EINVAL, "featurize: unknown space id");
  if (bits & kErrInternal) fail(FS_ECUDA, "internal trainer invariant violated");
}

}  // namespace fs

void fs_device::activate() const { FS_CUDA(cudaSetDevice(ordinal)); }

void* fs_device::scratch(int slot, size_t bytes) {
  if (slot >= static_cast<int>(slots.size())) slots.resize(static_cast<size_t>(slot) + 1);
  auto& b = slots[static_cast<size_t>(slot)];
  if (b.bytes < bytes) {
    if (b.p) FS_CUDA(cudaFreeAsync(b.p, stream));
    b.p = nullptr;
    b.bytes = 0;
    const size_t want = bytes + bytes / 4 + 256;
    FS_CUDA(cudaMallocAsync(&b.p, want, stream));
    b.bytes = want;
  }
  return b.p;
}

bool fs_device::prof_wants(const char* name) const {
  if (prof_filter.empty()) return false;
  if (prof_filter == "*") return true;
  const std::string n(name);
  size_t pos = 0;
  while (pos <= prof_filter.size()) {
    const size_t e = prof_filter.find(',', pos);
    const std::string tok = prof_filter.substr(pos, e == std::string::npos ? std::string::npos : e - pos);
    if (tok == n) return true;
    if (e == std::string::npos) break;
    pos = e + 1;
  }
  return false;
}

cudaEvent_t fs_device::prof_event() {
  if (!prof_pool.empty()) {
    cudaEvent_t e = prof_pool.back();
    prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  FS_CUDA(cudaEventCreate(&e));
  return e;
}

void fs_device::prof_resolve() {
  if (prof_pending.empty()) return;
  FS_CUDA(cudaStreamSynchronize(stream));
  for (auto& pe : prof_pending) {
    float ms = 0.f;
    FS_CUDA(cudaEventElapsedTime(&ms, pe.a, pe.b));
    bool found = false;
    for (auto& kv : prof_acc)
      if (kv.first == pe.name) {
        kv.second.first += 1;
        kv.second.second += ms;
        found = true;
        break;
      }
    if (!found) prof_acc.push_back({pe.name, {1, static_cast<double>(ms)}});
    prof_pool.push_back(pe.a);
    prof_pool.push_back(pe.b);
  }
  prof_pending.clear();
}

void* fs_device::pinned(size_t bytes) {
  if (bytes > pinned_cap) {
    FS_CUDA(cudaStreamSynchronize(stream));
    if (pinned_h) FS_CUDA(cudaFreeHost(pinned_h));
    pinned_h = nullptr;
    const size_t cap = std::max<size_t>(bytes + bytes / 2, 1 << 16);
    FS_CUDA(cudaHostAlloc(&pinned_h, cap, cudaHostAllocDefault));
    pinned_cap = cap;
  }
  return pinned_h;
}

void* fs_device::pinned_upload(size_t bytes) {
  if (up_evt) FS_CUDA(cudaEventSynchronize(up_evt));
  if (bytes > up_cap) {
    if (up_h) FS_CUDA(cudaFreeHost(up_h));
    up_h = nullptr;
    const size_t cap = std::max<size_t>(bytes + bytes / 2, 1 << 16);
    FS_CUDA(cudaHostAlloc(&up_h, cap, cudaHostAllocDefault));
    up_cap = cap;
  }
  return up_h;
}

cudaStream_t fs_device::aux_stream() {
  if (!aux) {
    FS_CUDA(cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking));
    FS_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    FS_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    FS_CUDA(cudaMalloc(&err_aux_d, sizeof(uint32_t)));
    FS_CUDA(cudaMemsetAsync(err_aux_d, 0, sizeof(uint32_t), stream));
  }
  return aux;
}

void fs_device::upload_done() {
  if (!up_evt) FS_CUDA(cudaEventCreateWithFlags(&up_evt, cudaEventDisableTiming));
  FS_CUDA(cudaEventRecord(up_evt, stream));
}

uint32_t fs_device::take_errors() {
  FS_CUDA(cudaMemcpyAsync(err_h, err_d, sizeof(uint32_t), cudaMemcpyDeviceToHost, stream));
  FS_CUDA(cudaStreamSynchronize(stream));
  const uint32_t bits = *err_h;
  if (bits) FS_CUDA(cudaMemsetAsync(err_d, 0, sizeof(uint32_t), stream));
  return bits;
}

extern "C" {

const char* fs_last_error(void) { return fs::g_last_error.c_str(); }

const char* fs_version(void) { return "famseer-b200 0.1 (sm_100a)"; }

int fs_device_create(int ordinal, fs_device** out) {
  return fs::guard([&] {
    if (!out) fs::fail(FS_EINVAL, "fs_device_create: out is NULL");
    int n = 0;
    FS_CUDA(cudaGetDeviceCount(&n));
    if (ordinal < 0 || ordinal >= n) fs::fail(FS_EINVAL, "fs_device_create: no such CUDA device");
    auto* d = new fs_device;
    d->ordinal = ordinal;
    try {
      d->activate();
      cudaDeviceProp prop{};
      FS_CUDA(cudaGetDeviceProperties(&prop, ordinal));
      if (prop.major != 10) {
        fs::fail(FS_ECUDA, "libfamseer is built for sm_100a (B200); device reports sm_" +
                               std::to_string(prop.major) + std::to_string(prop.minor));
      }
      d->sm_count = prop.multiProcessorCount;
      FS_CUDA(cudaStreamCreateWithFlags(&d->own, cudaStreamNonBlocking));
      d->stream = d->own;
      // Keep stream-ordered allocations mapped across synchronizations: the default release
      // threshold (0) returns freed pool memory to the driver at every sync, and the next fit's
      // cudaMallocAsync then pays the remapping (~0.25 ms per call at C2).
      cudaMemPool_t pool = nullptr;
      if (cudaDeviceGetDefaultMemPool(&pool, ordinal) == cudaSuccess && pool) {
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      FS_CUDA(cudaMalloc(&d->err_d, sizeof(uint32_t)));
      FS_CUDA(cudaMalloc(&d->ctr_d, fs::kCtrCount * sizeof(unsigned long long)));
      FS_CUDA(cudaMemsetAsync(d->ctr_d, 0, fs::kCtrCount * sizeof(unsigned long long), d->stream));
      FS_CUDA(cudaMemsetAsync(d->err_d, 0, sizeof(uint32_t), d->stream));
      FS_CUDA(cudaMallocHost(&d->err_h, sizeof(uint32_t)));
      FS_CUDA(cudaStreamSynchronize(d->stream));
    } catch (...) {
      delete d;
      throw;
    }
    *out = d;
  });
}

int fs_device_destroy(fs_device* d) {
  return fs::guard([&] {
    if (!d) return;
    d->activate();
    cudaStreamSynchronize(d->stream);
    for (auto& b : d->slots)
      if (b.p) cudaFreeAsync(b.p, d->stream);
    cudaStreamSynchronize(d->stream);
    if (d->err_d) cudaFree(d->err_d);
    if (d->err_aux_d) cudaFree(d->err_aux_d);
    if (d->ctr_d) cudaFree(d->ctr_d);
    if (d->err_h) cudaFreeHost(d->err_h);
    if (d->pinned_h) cudaFreeHost(d->pinned_h);
    if (d->up_evt) {
      cudaEventSynchronize(d->up_evt);
      cudaEventDestroy(d->up_evt);
    }
    if (d->up_h) cudaFreeHost(d->up_h);
    if (d->aux) {
      cudaStreamSynchronize(d->aux);
      cudaStreamDestroy(d->aux);
      cudaEventDestroy(d->ev_fork);
      cudaEventDestroy(d->ev_join);
    }
    if (d->own) cudaStreamDestroy(d->own);
    delete d;
  });
}

int fs_device_set_stream(fs_device* d, void* s) {
  return fs::guard([&] {
    if (!d) fs::fail(FS_EINVAL, "fs_device_set_stream: NULL device");
    d->activate();
    // Scratch buffers were allocated stream-ordered on the previous stream: fence it first.
    FS_CUDA(cudaStreamSynchronize(d->stream));
    d->stream = s ? static_cast<cudaStream_t>(s) : d->own;
  });
}

void* fs_device_stream(fs_device* d) { return d ? static_cast<void*>(d->stream) : nullptr; }

int fs_device_check(fs_device* d) {
  return fs::guard([&] {
    if (!d) fs::fail(FS_EINVAL, "fs_device_check: NULL device");
    d->activate();
    FS_CUDA(cudaGetLastError());
    fs::raise_deferred(d->take_errors());
  });
}

int64_t fs_device_launches(const fs_device* d) { return d ? d->launches : 0; }

int fs_device_counters(fs_device* d, int64_t* out, int32_t n, int32_t reset) {
  return fs::guard([&] {
    if (!d || (n > 0 && !out)) fs::fail(FS_EINVAL, "fs_device_counters: bad arguments");
    d->activate();
    unsigned long long h[fs::kCtrCount] = {};
    FS_CUDA(cudaMemcpyAsync(h, d->ctr_d, sizeof h, cudaMemcpyDeviceToHost, d->stream));
    FS_CUDA(cudaStreamSynchronize(d->stream));
    for (int i = 0; i < n && i < fs::kCtrCount; ++i) out[i] = static_cast<int64_t>(h[i]);
    if (reset) FS_CUDA(cudaMemsetAsync(d->ctr_d, 0, sizeof h, d->stream));
  });
}

int fs_device_profile(fs_device* d, const char* kernels) {
  return fs::guard([&] {
    if (!d) fs::fail(FS_EINVAL, "fs_device_profile: NULL device");
    d->activate();
    d->prof_resolve();
    d->prof_acc.clear();
    d->prof_filter = kernels ? kernels : "";
  });
}

int fs_device_profile_read(fs_device* d, const char* kernel, int64_t* count, double* total_ms) {
  return fs::guard([&] {
    if (!d || !kernel) fs::fail(FS_EINVAL, "fs_device_profile_read: bad arguments");
    d->activate();
    d->prof_resolve();
    if (count) *count = 0;
    if (total_ms) *total_ms = 0.0;
    for (const auto& kv : d->prof_acc)
      if (kv.first == kernel) {
        if (count) *count = kv.second.first;
        if (total_ms) *total_ms = kv.second.second;
      }
  });
}

int64_t fs_device_profile_names(fs_device* d, char* buf, int64_t cap) {
  if (!d) return -1;
  try {
    d->prof_resolve();
  } catch (...) {
    return -1;
  }
  std::string s;
  for (const auto& kv : d->prof_acc) {
    if (!s.empty()) s += ',';
    s += kv.first;
  }
  if (buf && cap > 0) {
    const int64_t n = std::min<int64_t>(cap - 1, static_cast<int64_t>(s.size()));
    std::memcpy(buf, s.data(), static_cast<size_t>(n));
    buf[n] = '\0';
  }
  return static_cast<int64_t>(s.size()) + 1;
}

int fs_feature_dim(int32_t k) { return 2 * k + k * (k - 1) / 2; }

}  // extern "C"
