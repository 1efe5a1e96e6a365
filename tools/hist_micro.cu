// Microbenchmark of the resident trainer's histogram accumulate loop (one CTA, 512 threads,
// 2048 rows x 12 features, lane-column limb layout), with variants that remove one ingredient
// at a time to find what bounds it:
//   0 full loop (index -> value/code -> 3 limb atomics)
//   1 no atomics (loads only, values folded into a register)
//   2 identity rows (no index indirection)
//   3 two limbs
//   4 plain shared stores instead of atomics (racy; timing only)
//   5 full loop, 1024 threads
//   6 full loop, two histogram copies (even / odd warps)
// each mode runs with codes uniform over 14, 4 and 2 values per feature (same-address pressure)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/hist_micro tools/hist_micro.cu
#include <cstdio>
#include <cstdint>

constexpr int kN = 2048, kNrep = 12, kColh = 37, kCs = 2048 + 4;

template <int kMode, int kThreads>
__global__ void __launch_bounds__(kThreads, 1) hist_loop(const uint16_t* g_rows, const long long* g_fix,
                                                         const uint8_t* g_codes, unsigned long long* cyc,
                                                         unsigned* sink) {
  extern __shared__ __align__(16) unsigned char smem[];
  long long* fix = reinterpret_cast<long long*>(smem);
  uint32_t* limb = reinterpret_cast<uint32_t*>(fix + kN);
  uint16_t* rows = reinterpret_cast<uint16_t*>(limb + 2 * 3 * kColh * 32);
  uint8_t* codes = reinterpret_cast<uint8_t*>(rows + kN);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < kN; i += kThreads) {
    rows[i] = kMode == 2 ? static_cast<uint16_t>(i) : g_rows[i];
    fix[i] = g_fix[i];
  }
  for (int i = tid; i < kNrep * kCs; i += kThreads) codes[i] = g_codes[i];
  for (int i = tid; i < 2 * 3 * kColh * 32; i += kThreads) limb[i] = 0;
  __syncthreads();
  const int rpw = 32 / kNrep, hj = lane % kNrep, hm = lane / kNrep;
  const bool hact = hm < rpw;
  const uint8_t* hcode = codes + hj * kCs;
  uint32_t* colp = limb + lane + (kMode == 6 ? (warp & 1) * 3 * kColh * 32 : 0);
  unsigned acc = 0;
  const long long t0 = clock64();
  for (int rep = 0; rep < 10; ++rep) {
    if (hact) {
      for (int q = warp * rpw + hm; q < kN; q += (kThreads / 32) * rpw) {
        const int p = rows[q];
        const long long v = fix[p];
        const uint64_t u = static_cast<uint64_t>(v) + (1ull << 62);
        const int cd = hcode[p];
        uint32_t* c = colp + cd * 96;  // [code][limb][32] as in the trainer
        if (kMode == 1) {
          acc += static_cast<uint32_t>(u) + cd;
        } else if (kMode == 4) {
          c[0] = static_cast<uint32_t>(u) & 0x1FFFFF;
          c[32] = static_cast<uint32_t>(u >> 21) & 0x1FFFFF;
          c[64] = static_cast<uint32_t>(u >> 42);
        } else {
          atomicAdd(c, static_cast<uint32_t>(u) & 0x1FFFFF);
          atomicAdd(c + 32, static_cast<uint32_t>(u >> 21) & 0x1FFFFF);
          if (kMode != 3) atomicAdd(c + 64, static_cast<uint32_t>(u >> 42));
        }
      }
    }
    __syncthreads();
  }
  const long long t1 = clock64();
  if (tid == 0) *cyc = (t1 - t0) / 10;
  if (acc == 12345) sink[0] = acc + limb[tid];
}

template <int kMode, int kThreads>
void run(const char* name, const uint16_t* r, const long long* f, const uint8_t* c, unsigned long long* cyc,
         unsigned* sink, int mod) {
  const int sm = kN * 8 + 2 * 3 * kColh * 32 * 4 + kN * 2 + kNrep * kCs;
  cudaFuncSetAttribute(hist_loop<kMode, kThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  hist_loop<kMode, kThreads><<<1, kThreads, sm>>>(r, f, c, cyc, sink);
  hist_loop<kMode, kThreads><<<1, kThreads, sm>>>(r, f, c, cyc, sink);
  cudaDeviceSynchronize();
  unsigned long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  std::printf("%-40s codes%%%-2d %8llu cycles per 2048x12 pass (%.2f per row-feature)\n", name, mod, h,
              double(h) / (kN * kNrep));
}

int main() {
  uint16_t hr[kN];
  long long hf[kN];
  static uint8_t hc[kNrep * kCs];
  unsigned s = 12345;
  for (int i = 0; i < kN; ++i) hr[i] = static_cast<uint16_t>(i);
  for (int i = kN - 1; i > 0; --i) {
    s = s * 1103515245u + 12345u;
    const int j = static_cast<int>((s >> 8) % (i + 1));
    const uint16_t t = hr[i];
    hr[i] = hr[j];
    hr[j] = t;
  }
  for (int i = 0; i < kN; ++i) {
    s = s * 1103515245u + 12345u;
    hf[i] = (static_cast<long long>(s) << 20) - (1ll << 40);
  }
  for (int i = 0; i < kNrep * kCs; ++i) {
    s = s * 1103515245u + 12345u;
    hc[i] = static_cast<uint8_t>((s >> 8) % 14);
  }
  uint16_t* dr;
  long long* df;
  uint8_t* dc;
  unsigned long long* cyc;
  unsigned* sink;
  cudaMalloc(&dr, sizeof hr);
  cudaMalloc(&df, sizeof hf);
  cudaMalloc(&dc, sizeof hc);
  cudaMalloc(&cyc, 8);
  cudaMalloc(&sink, 4096);
  cudaMemcpy(dr, hr, sizeof hr, cudaMemcpyHostToDevice);
  cudaMemcpy(df, hf, sizeof hf, cudaMemcpyHostToDevice);
  cudaMemcpy(dc, hc, sizeof hc, cudaMemcpyHostToDevice);
  for (int mod : {14, 4, 2}) {
    for (int i = 0; i < kNrep * kCs; ++i) {
      s = s * 1103515245u + 12345u;
      hc[i] = static_cast<uint8_t>((s >> 8) % mod);
    }
    cudaMemcpy(dc, hc, sizeof hc, cudaMemcpyHostToDevice);
    run<0, 512>("0 full (index, 3 limb atomics)", dr, df, dc, cyc, sink, mod);
    run<1, 512>("1 loads only", dr, df, dc, cyc, sink, mod);
    run<2, 512>("2 identity rows", dr, df, dc, cyc, sink, mod);
    run<3, 512>("3 two limbs", dr, df, dc, cyc, sink, mod);
    run<4, 512>("4 plain stores", dr, df, dc, cyc, sink, mod);
    run<0, 1024>("5 full, 1024 threads", dr, df, dc, cyc, sink, mod);
    run<6, 512>("6 full, two copies", dr, df, dc, cyc, sink, mod);
  }
  return 0;
}
