// Microbenchmark guiding the histogram design on sm_100a (results in profiles/README.md):
// cycles per histogram update for (a) native 32-bit shared atomics from every thread,
// (b) 3 x 32-bit limb atomics (exact 63-bit sums), (c) lane-private 64-bit read-modify-write
// chains in a bank-conflict-free column layout, (d) the same with two interleaved copies.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_hist_micro tools/smem_hist_micro.cu
#include <cstdio>
#include <cstdint>

constexpr int kIters = 4096;

__device__ __forceinline__ unsigned hashu(unsigned x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

template <int kMode, int kBins>
__global__ void __launch_bounds__(1024, 1) bench(unsigned long long* cycles, unsigned long long* sink) {
  __shared__ unsigned int h32[3 * 32 * kBins];
  __shared__ long long h64[2 * 32 * kBins];
  for (int i = threadIdx.x; i < 3 * 32 * kBins; i += blockDim.x) h32[i] = 0;
  for (int i = threadIdx.x; i < 2 * 32 * kBins; i += blockDim.x) h64[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  unsigned seed = hashu(threadIdx.x * 7919u + blockIdx.x);
  const long long t0 = clock64();
  if (kMode == 0) {  // one native 32-bit atomic per update, any thread -> any bin
    for (int it = 0; it < kIters; ++it) {
      seed = hashu(seed);
      atomicAdd(&h32[(seed % kBins) * 32 + lane], seed & 0xFFu);
    }
  } else if (kMode == 1) {  // three limb atomics per update
    for (int it = 0; it < kIters; ++it) {
      seed = hashu(seed);
      const unsigned b = (seed % kBins) * 32 + lane;
      atomicAdd(&h32[b], seed & 0x1FFFFFu);
      atomicAdd(&h32[32 * kBins + b], (seed >> 3) & 0x1FFFFFu);
      atomicAdd(&h32[64 * kBins + b], (seed >> 7) & 0x1FFFFFu);
    }
  } else if (kMode == 2) {  // lane-private RMW chain, 64-bit (only warp 0..31 each own a column)
    long long* col = h64 + lane;
    for (int it = 0; it < kIters; ++it) {
      seed = hashu(seed);
      col[(seed % kBins) * 32] += seed;
    }
  } else {  // two interleaved private copies
    long long* c0 = h64 + lane;
    long long* c1 = h64 + 32 * kBins + lane;
    for (int it = 0; it < kIters; it += 2) {
      seed = hashu(seed);
      const unsigned s2 = hashu(seed);
      c0[(seed % kBins) * 32] += seed;
      c1[(s2 % kBins) * 32] += s2;
      seed = s2;
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  unsigned long long acc = 0;
  for (int i = threadIdx.x; i < 32 * kBins; i += blockDim.x) acc += h32[i] + h64[i];
  if (acc == 42) sink[0] = acc;
}

template <int kMode, int kBins>
void run(const char* name, int threads) {
  unsigned long long *c, *s;
  cudaMalloc(&c, 8 * 148);
  cudaMalloc(&s, 8);
  bench<kMode, kBins><<<148, threads>>>(c, s);
  bench<kMode, kBins><<<148, threads>>>(c, s);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double updates = double(threads) * kIters;
  std::printf("%-28s threads=%4d bins=%3d  cycles/update/SM = %.3f\n", name, threads, kBins, avg / updates);
  cudaFree(c);
  cudaFree(s);
}

// dependent FP64 add chain (the reference-order fold's latency floor)
__global__ void dadd_chain(const double* v, double* out, unsigned long long* cycles) {
  double s = 0.0, a = v[threadIdx.x], b = v[threadIdx.x + 1];
  const long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < 65536; ++i) {
    s = __dadd_rn(s, a);
    a = __dadd_rn(a, b) * 0.0 + a;  // keep a live without lengthening the chain
  }
  const long long t1 = clock64();
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[0] = t1 - t0;
}

int main() {
  {
    double *v, *o;
    unsigned long long* c;
    cudaMalloc(&v, 64 * 8);
    cudaMalloc(&o, 64 * 8);
    cudaMalloc(&c, 8);
    cudaMemset(v, 0, 64 * 8);
    dadd_chain<<<1, 32>>>(v, o, c);
    dadd_chain<<<1, 32>>>(v, o, c);
    unsigned long long h = 0;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    std::printf("dependent DADD chain: %.2f cycles per add (upper bound, includes the side chain)\n",
                double(h) / 65536.0);
  }
  run<0, 32>("atomic32 x1", 1024);
  run<1, 32>("atomic32 x3 limbs", 1024);
  run<2, 32>("private rmw64 chain", 1024);
  run<3, 32>("private rmw64 x2 copies", 1024);
  run<2, 32>("private rmw64 chain", 256);
  run<0, 8>("atomic32 x1 (8 bins)", 1024);
  return 0;
}
