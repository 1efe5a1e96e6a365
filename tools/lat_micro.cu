// Latency microbenchmarks behind the resident trainer's design choices (run on the B200):
//   (a) dependent FP64 add chain (__dadd_rn) - the reference-order fold's floor per element;
//   (b) the same chain fed from shared memory through a u16 index list (fold_seq's shape);
//   (c) dependent shared-memory load chain (pointer chasing) - smem load-to-use latency;
//   (d) __syncthreads() round trip in a 1024-thread CTA.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/lat_micro tools/lat_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dadd_chain(const double* v, double* out, long long* cyc, int n) {
  double a = v[threadIdx.x], b = v[32 + threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) a = __dadd_rn(a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void smem_fold(const double* v, double* out, long long* cyc, int n) {
  __shared__ double r[4096];
  __shared__ unsigned short idx[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) {
    r[i] = v[i & 63];
    idx[i] = static_cast<unsigned short>((i * 1237) & 4095);
  }
  __syncthreads();
  double s = 0.0;
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = r[idx[k]];
    for (int i = 8; i + 8 <= n; i += 8) {
      double b[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) b[k] = r[idx[i + k]];
#pragma unroll
      for (int k = 0; k < 8; ++k) s = __dadd_rn(s, a[k]);
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = b[k];
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    out[0] = s;
    *cyc = t1 - t0;
  }
}

__global__ void smem_chase(double* out, long long* cyc, int n) {
  __shared__ int nxt[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) nxt[i] = (i * 1237 + 11) & 4095;
  __syncthreads();
  int p = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) p = nxt[p];
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    out[0] = p;
    *cyc = t1 - t0;
  }
}

__global__ void sync_rt(double* out, long long* cyc, int n) {
  __shared__ int x;
  if (threadIdx.x == 0) x = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (threadIdx.x == (i & 1023)) x += 1;
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    out[0] = x;
    *cyc = t1 - t0;
  }
}

int main() {
  double *v, *o;
  long long* c;
  cudaMalloc(&v, 4096 * 8);
  cudaMalloc(&o, 4096 * 8);
  cudaMallocManaged(&c, 8);
  double h[64];
  for (int i = 0; i < 64; ++i) h[i] = 1.0 + i * 1e-3;
  cudaMemcpy(v, h, sizeof h, cudaMemcpyHostToDevice);
  const int n = 4096;
  for (int rep = 0; rep < 2; ++rep) dadd_chain<<<1, 32>>>(v, o, c, n / 16);
  cudaDeviceSynchronize();
  std::printf("(a) dependent DADD chain        : %.2f cycles/add\n", double(*c) / n);
  for (int rep = 0; rep < 2; ++rep) smem_fold<<<1, 256>>>(v, o, c, n);
  cudaDeviceSynchronize();
  std::printf("(b) smem-fed indexed fold      : %.2f cycles/element\n", double(*c) / n);
  for (int rep = 0; rep < 2; ++rep) smem_chase<<<1, 32>>>(o, c, n);
  cudaDeviceSynchronize();
  std::printf("(c) smem load-to-use latency   : %.2f cycles\n", double(*c) / n);
  for (int rep = 0; rep < 2; ++rep) sync_rt<<<1, 1024>>>(o, c, n);
  cudaDeviceSynchronize();
  std::printf("(d) __syncthreads, 1024 threads: %.2f cycles\n", double(*c) / n);
  for (int rep = 0; rep < 2; ++rep) sync_rt<<<1, 256>>>(o, c, n);
  cudaDeviceSynchronize();
  std::printf("(d) __syncthreads,  256 threads: %.2f cycles\n", double(*c) / n);
  return 0;
}
