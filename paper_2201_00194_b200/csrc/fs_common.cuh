// Internal plumbing shared by the libfamseer translation units: error mapping, the device
// context (stream, stream-ordered scratch, deferred-error word, launch counter) and the FP64
// helpers that keep every reference sum separately rounded (no FMA contraction).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "famseer.h"

namespace fs {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    if (e == cudaErrorMemoryAllocation) fail(FS_ENOMEM, std::string(what) + ": " + cudaGetErrorString(e));
    fail(FS_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
}
#define FS_CUDA(x) ::fs::cuda_check((x), #x)
// Programmatic dependent launch (PDL): a kernel launched with programmatic stream serialization
// may be scheduled while its predecessor drains; it waits here for the predecessor's completion
// (and memory visibility) before touching anything it produced. A no-op for a normal launch.
// Programmatic dependent launch: wait for the preceding kernel on the stream to complete (and its
// writes to be visible), then let the next PDL launch start scheduling (its CTAs park in their
// own FS_PDL_WAIT). Harmless no-ops when the launch carried no PDL attribute.
#define FS_PDL_WAIT() asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory")

template <class F>
int guard(F&& f) {
  try {
    f();
    return FS_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return FS_ENOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return FS_ECUDA;
  }
}

// Deferred kernel-side error bits (reported by fs_device_check / the host-pointer entry points).
enum ErrBits : uint32_t {
  kErrNonFinitePredict = 1u << 0,  // costmodel.cpp:238-240
  kErrNonFiniteFit = 1u << 1,      // costmodel.cpp:178-182
  kErrKnobRange = 1u << 2,         // assignment index outside the knob's value list
  kErrPadDim = 1u << 3,            // searchspace.cpp:96-100
  kErrSpaceId = 1u << 4,           // candidate names an unknown space
  kErrInternal = 1u << 5,          // trainer invariant violated (must never fire)
};

// Device work counters (algorithmic traffic the host cannot know in advance).
enum Counter : int {
  kCtrHistBytes = 0,  // histogram build: rows * (nrep * code bytes + 8 residual + 4 list index)
  kCtrHistRows,       // rows histogrammed
  kCtrExactChains,    // reference-order folds run (node totals + feature scans)
  kCtrExactNodes,     // nodes re-evaluated in reference order
  kCtrPhase0,         // resident trainer: SM cycles per phase (kResPhases entries, CTA 0's view)
  kCtrProbe = kCtrPhase0 + 16,  // resident trainer A/B probes (FS_RES_HIST_PROBE builds), 4 entries
  kCtrCount = kCtrProbe + 4
};

// Grows-only stream-ordered device buffer.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

}  // namespace fs

struct fs_device {
  int ordinal = 0;
  int sm_count = 148;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  uint32_t* err_d = nullptr;     // device error word
  unsigned long long* ctr_d = nullptr;  // device work counters (fs_device_counters)
  uint32_t* err_h = nullptr;     // pinned mirror
  int64_t launches = 0;
  bool capturing = false;  // inside CUDA-graph capture: no event timing
  std::vector<fs::DevBuf> slots;  // scratch, indexed by purpose

  // Optional per-kernel CUDA-event timing (fs_device_profile): event pairs recorded on the
  // launching stream around the kernels whose names are enabled, resolved on read.
  std::string prof_filter;  // comma-separated kernel names, "*" = all, empty = off
  struct ProfEvent {
    const char* name;
    cudaEvent_t a, b;
  };
  std::vector<ProfEvent> prof_pending;
  std::vector<cudaEvent_t> prof_pool;
  std::vector<std::pair<std::string, std::pair<int64_t, double>>> prof_acc;  // name -> (count, ms)

  void* pinned_h = nullptr;     // pinned host staging for batched device->host reads (grow-only)
  size_t pinned_cap = 0;
  void* pinned(size_t bytes);      // grow-only; synchronizes the stream when it has to grow
  void* up_h = nullptr;            // pinned host staging for async host->device model uploads
  size_t up_cap = 0;
  cudaEvent_t up_evt = nullptr;    // recorded after the last upload from up_h
  void* pinned_upload(size_t bytes);  // waits until the previous upload from it has been read
  void upload_done();                 // record up_evt on the stream after issuing the copies
  cudaStream_t aux = nullptr;      // forked work: trainer node totals / the tune step's scoring
  cudaEvent_t epilogue_wait = nullptr;  // fit_families waits for it before writing any model blob
  uint32_t* err_aux_d = nullptr;   // error word of the tune step's forked scoring
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaStream_t aux_stream();       // lazily created (non-blocking) + its fork/join events
  void* scratch(int slot, size_t bytes);  // stream-ordered grow; contents undefined
  void count_launch(int n = 1) { launches += n; }
  void activate() const;                  // cudaSetDevice(ordinal)
  uint32_t take_errors();                 // sync + read and clear the error word
  bool prof_wants(const char* name) const;
  cudaEvent_t prof_event();
  void prof_resolve();
};

namespace fs {
// Scoped timer: `{ ProfScope p(dev, "hist_build"); kernel<<<...>>>(...); }`
struct ProfScope {
  fs_device* dev;
  const char* name;
  cudaEvent_t a = nullptr;
  ProfScope(fs_device* d, const char* n) : dev(d), name(n) {
    if (!dev->capturing && dev->prof_wants(name)) {
      a = dev->prof_event();
      cudaEventRecord(a, dev->stream);
    }
  }
  ~ProfScope() {
    if (a) {
      cudaEvent_t b = dev->prof_event();
      cudaEventRecord(b, dev->stream);
      dev->prof_pending.push_back({name, a, b});
    }
  }
};
}  // namespace fs

namespace fs {

// Scratch slot ids (each purpose owns one growable buffer).
enum Slot : int {
  kSlotH2D0 = 0,
  kSlotH2D1,
  kSlotH2D2,
  kSlotD2H0,
  kSlotD2H1,
  kSlotRankKeys,
  kSlotRankKeys2,
  kSlotRankIdx2,
  kSlotPredictSeg,
  kSlotScoreX,
  kSlotScoreS,
  kSlotScoreP,
  kSlotScoreA,  // assignments decoded from linear_index descriptors (unfused score fallback)
  kSlotFitX,    // featurized training records (fs_fit_records)
  kSlotFitIn,   // their descriptors / targets (host-pointer form)
  kSlotCount
};

// Throws FS_EINVAL with the reference's message for the deferred bits that are set.
void raise_deferred(uint32_t bits);

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace fs

// FP64 arithmetic in the reference's rounding order. The library is also compiled with
// -fmad=false, but the hot sums spell the rounding out so no compiler flag can change them.
__device__ __forceinline__ double fs_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double fs_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double fs_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double fs_div(double a, double b) { return __ddiv_rn(a, b); }

// Device-resident knob-space tables (fs_spaces_create): per (space, knob, value index) the
// reference's log2(value) and list position, both computed on the host (searchspace.cpp:103-109).
struct fs_spaces {
  fs_device* dev = nullptr;
  int32_t n = 0;
  int32_t max_fd = 0;
  std::vector<int32_t> k_h;  // knobs per space
  int32_t* k_d = nullptr;    // [n]
  int32_t* nval_d = nullptr; // [n*16]
  int32_t* off_d = nullptr;  // [n*16] offset into log/pos tables
  double* log_d = nullptr;
  double* pos_d = nullptr;
  // linear_index descriptors (searchspace.cpp:48-66): stride[s][j] = prod_{k>j} m_k
  uint64_t* stride_d = nullptr;  // [n*16]
};

namespace fs {
// Pair q of K knobs in the reference's row-major i<j order (searchspace.cpp:111-116).
__device__ __forceinline__ void pair_of(int k, int q, int& i, int& j) {
  int row = 0;
  int remaining = q;
  while (remaining >= k - 1 - row) {
    remaining -= k - 1 - row;
    ++row;
  }
  i = row;
  j = row + 1 + remaining;
}
}  // namespace fs
