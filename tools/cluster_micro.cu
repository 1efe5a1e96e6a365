// Cost of a thread-block-cluster barrier (barrier.cluster.arrive.release + wait.acquire) and of a
// DSMEM read, against __syncthreads, for 512-thread CTAs in clusters of 1, 2 and 4 on sm_100a.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/cluster_micro tools/cluster_micro.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void bar_kernel(unsigned long long* out, int mode) {
  __shared__ double buf[512];
  cg::cluster_group cl = cg::this_cluster();
  buf[threadIdx.x] = threadIdx.x;
  cl.sync();
  const unsigned rank = cl.block_rank();
  const double* peer = cl.map_shared_rank(buf, (rank + 1) % cl.num_blocks());
  double acc = 0;
  const long long t0 = clock64();
  for (int i = 0; i < 1000; ++i) {
    if (mode == 0) {
      __syncthreads();
    } else if (mode == 1) {
      asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    } else {
      acc += peer[(threadIdx.x + i) & 511];  // DSMEM read, then a cluster barrier
      asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    }
  }
  const long long t1 = clock64();
  cl.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / 1000 + (acc == -1.0 ? 1 : 0);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64 * 8);
  for (int cs : {1, 2, 4}) {
    for (int mode = 0; mode < 3; ++mode) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs * 2);
      cfg.blockDim = dim3(512);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, bar_kernel, d, mode);
      cudaLaunchKernelEx(&cfg, bar_kernel, d, mode);
      cudaDeviceSynchronize();
      unsigned long long h[8];
      cudaMemcpy(h, d, 8 * 8, cudaMemcpyDeviceToHost);
      printf("cluster %d mode %s: %llu cycles per iteration (%s)\n", cs,
             mode == 0 ? "syncthreads" : mode == 1 ? "cluster barrier" : "dsmem read + cluster barrier", h[0],
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
