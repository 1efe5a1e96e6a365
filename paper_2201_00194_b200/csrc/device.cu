// fs_device: one context per GPU (stream, scratch arena, deferred-error word, launch counter).
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
      FS_CUDA(cudaMalloc(&d->err_d, sizeof(uint32_t)));
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
    if (d->err_h) cudaFreeHost(d->err_h);
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

int fs_feature_dim(int32_t k) { return 2 * k + k * (k - 1) / 2; }

}  // extern "C"
