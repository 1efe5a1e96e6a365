// Bit-exactness check + cycle count of fold_est.cuh's CTA folds against a one-thread sequential
// fold (the reference's sum_residuals / best_split recording, costmodel.cpp:36-69), over
// adversarial chains: drifting and zero-mean random walks, near-zero totals, mixed magnitudes,
// subnormals, half-ulp ties, signed zeros and infinities, lengths around every internal size
// boundary. Built and run by tests/test_fold_est_gpu.py:
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false -DLB=256 -DEM=16
//        -I paper_2201_00194_b200/csrc -I include -o fold_bench tools/fold_bench.cu
//   ./fold_bench 256      -> "... bad 0" and exit 0 when every result is bit-identical
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "fold_est.cuh"

#ifndef LB
#define LB 256
#endif
#ifndef EM
#define EM 16
#endif

using namespace fs;

constexpr int kMaxN = 70000;

__global__ void __launch_bounds__(LB) fold_kernel(const double* v, const int32_t* idx, const uint16_t* codes,
                                                   const int* nlist, const int* mode, int nchains, double* out,
                                                   double* ref, double* rec, double* rec_ref, long long* cyc,
                                                   unsigned long long* ctr, int ncodes) {
  extern __shared__ __align__(16) double sm[];
  double* stage = sm;
  double* scr = sm + fold_est_stage_doubles(blockDim.x, EM);
  uint16_t* cst = reinterpret_cast<uint16_t*>(scr + fold_est_scratch_doubles(blockDim.x));
  const int c = blockIdx.x;
  if (c >= nchains) return;
  const int n = nlist[c], m = mode[c];
  const int32_t* id = idx + static_cast<long long>(c) * kMaxN;
  double* ro = rec + static_cast<long long>(c) * ncodes;
  __syncthreads();
  const long long t0 = clock64();
  double r;
  if (m == 0) r = cta_fold_est<EM>(v, id, n, 0.0, stage, scr, ctr);
  else if (m == 1) r = cta_fold_est<EM>(v + static_cast<long long>(c) * 1024, nullptr, n, 0.0, stage, scr, ctr);
  else r = cta_fold_est_rec<EM, uint16_t>(v, id, n, codes, ro, stage, cst, scr);
  const long long t1 = clock64();
  if (threadIdx.x == 0) {
    out[c] = r;
    cyc[c] = t1 - t0;
    double s = 0.0;
    double* rr = rec_ref + static_cast<long long>(c) * ncodes;
    int prev = -1;
    for (int i = 0; i < n; ++i) {
      const double x = m == 1 ? v[static_cast<long long>(c) * 1024 + i] : v[id[i]];
      if (m == 2) {
        const int cc = codes[id[i]];
        if (prev >= 0 && cc != prev) rr[prev] = s;
        prev = cc;
      }
      s = __dadd_rn(s, x);
    }
    if (m == 2 && prev >= 0) rr[prev] = s;
    ref[c] = s;
  }
}

int main(int argc, char** argv) {
  const int T = argc > 1 ? atoi(argv[1]) : LB;
  const int NV = 1 << 21, NCODES = 256;
  std::mt19937_64 g(11);
  std::normal_distribution<double> nd(0.0, 1.0);
  std::vector<double> hv(NV);
  const int kDists = 10;
  auto draw = [&](int dist, int i) -> double {
    switch (dist) {
      case 0: return 0.02 + 0.3 * nd(g);                     // drifting walk
      case 1: return 0.3 * nd(g);                            // zero-mean walk (near-zero totals)
      case 2: return 1e-3 * nd(g) + (i % 2 ? 1e3 : -1e3);    // large cancelling pairs
      case 3: return std::ldexp(nd(g), static_cast<int>(g() % 80) - 40);  // mixed magnitudes
      case 4: return (g() % 2 ? 1.0 : -1.0) * std::ldexp(1.0, -53 + static_cast<int>(g() % 3));  // half-ulp ties
      case 5: return 4.9e-324 * static_cast<double>(g() % 1000) - 2.4e-321;  // subnormals
      case 6: return g() % 7 == 0 ? -0.0 : (g() % 5 == 0 ? 0.0 : 1e-300 * nd(g));  // signed zeros, tiny
      case 7: return 0.3 + 0.1 * nd(g);                      // strong drift
      case 8: return g() % 9973 == 0 ? (g() % 2 ? INFINITY : -INFINITY) : nd(g);  // rare infinities
      default: return 0.001 * nd(g) + 1e-7;                  // tiny drift
    }
  };
  for (int i = 0; i < NV; ++i) hv[i] = draw((i >> 17) % kDists, i);
  const int sizes[] = {1, 2, 31, 33, 200, 383, 384, 1023, 1024, 1600, 2047, 2049, 4095, 4096, 4097,
                       5200, 8191, 8193, 12000, 16384, 16385, 40000, 65536, kMaxN};
  const int NS = sizeof(sizes) / sizeof(int);
  std::vector<int> nl, md;
  std::vector<int32_t> hidx;
  std::vector<uint16_t> hcodes(NV);
  for (int i = 0; i < NV; ++i) hcodes[i] = 0;
  for (int s = 0; s < NS; ++s)
    for (int dist = 0; dist < kDists; ++dist)
      for (int m = 0; m < 3; ++m) {
        nl.push_back(sizes[s]);
        md.push_back(m == 1 && sizes[s] > 1024 * 1 ? 0 : m);  // contiguous mode: short chains only
      }
  const int nch = static_cast<int>(nl.size());
  hidx.resize(static_cast<size_t>(nch) * kMaxN);
  // per chain: rows drawn from its distribution block; codes non-decreasing along the list
  // (assigned per row: a row appears once per chain list, codes are per row and global, so the
  // recording chains use disjoint row ranges sorted by code)
  for (int c = 0; c < nch; ++c) {
    const int dist = (c / 3) % kDists;
    const int base = dist << 17;
    int32_t* id = hidx.data() + static_cast<size_t>(c) * kMaxN;
    if (md[c] == 2) {  // a sorted run of distinct rows in [base, base + 2^17)
      const int n = nl[c];
      const int start = static_cast<int>(g() % static_cast<unsigned>((1 << 17) - n + 1));
      for (int i = 0; i < n; ++i) id[i] = base + start + i;
    } else {
      for (int i = 0; i < kMaxN; ++i) id[i] = base + static_cast<int>(g() % (1u << 17));
    }
  }
  // codes: non-decreasing along every recording list (rows of a block in increasing order)
  for (int b = 0; b < kDists; ++b) {
    int code = 0;
    for (int i = 0; i < (1 << 17); ++i) {
      if (g() % 97 == 0) code = (code + 1) % NCODES;
      if (code == 0 && i > 0 && hcodes[(b << 17) + i - 1] != 0) code = NCODES - 1;  // never wrap down
      hcodes[(b << 17) + i] = static_cast<uint16_t>(code);
    }
  }
  double *v, *out, *ref, *rec, *rec_ref;
  int32_t* idx;
  uint16_t* codes;
  int *nlist, *mode;
  long long* cyc;
  unsigned long long* ctr;
  cudaMalloc(&v, NV * 8);
  cudaMalloc(&idx, hidx.size() * 4);
  cudaMalloc(&codes, NV * 2);
  cudaMalloc(&nlist, nch * 4);
  cudaMalloc(&mode, nch * 4);
  cudaMalloc(&out, nch * 8);
  cudaMalloc(&ref, nch * 8);
  cudaMalloc(&rec, static_cast<size_t>(nch) * NCODES * 8);
  cudaMalloc(&rec_ref, static_cast<size_t>(nch) * NCODES * 8);
  cudaMalloc(&cyc, nch * 8);
  cudaMalloc(&ctr, 80);
  cudaMemcpy(v, hv.data(), NV * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(idx, hidx.data(), hidx.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(codes, hcodes.data(), NV * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(nlist, nl.data(), nch * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(mode, md.data(), nch * 4, cudaMemcpyHostToDevice);
  cudaMemset(rec, 0xff, static_cast<size_t>(nch) * NCODES * 8);
  cudaMemset(rec_ref, 0xff, static_cast<size_t>(nch) * NCODES * 8);
  cudaMemset(ctr, 0, 80);
  const size_t smem = (fold_est_stage_doubles(T, EM) + fold_est_scratch_doubles(T)) * 8 + EM * T * 2;
  cudaFuncSetAttribute(fold_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  fold_kernel<<<nch, T, smem>>>(v, idx, codes, nlist, mode, nch, out, ref, rec, rec_ref, cyc, ctr, NCODES);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    printf("CUDA error %s\n", cudaGetErrorString(e));
    return 2;
  }
  std::vector<double> ho(nch), hr(nch), hrec(static_cast<size_t>(nch) * NCODES), hrr(hrec.size());
  std::vector<long long> hc(nch);
  unsigned long long hctr[10];
  cudaMemcpy(ho.data(), out, nch * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hr.data(), ref, nch * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hrec.data(), rec, hrec.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hrr.data(), rec_ref, hrr.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hc.data(), cyc, nch * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hctr, ctr, 80, cudaMemcpyDeviceToHost);
  int bad = 0, bad_rec = 0;
  for (int s = 0; s < NS; ++s) {
    double cy = 0;
    int cnt = 0, b = 0;
    for (int k = 0; k < kDists * 3; ++k) {
      const int c = s * kDists * 3 + k;
      if (std::memcmp(&ho[c], &hr[c], 8) != 0) ++b;
      if (md[c] == 2 && std::memcmp(&hrec[static_cast<size_t>(c) * NCODES], &hrr[static_cast<size_t>(c) * NCODES],
                                    NCODES * 8) != 0)
        ++bad_rec;
      if (md[c] == 0) {
        cy += static_cast<double>(hc[c]);
        ++cnt;
      }
    }
    bad += b;
    printf("T=%d EM=%d n=%6d cycles %9.0f cyc/elem %6.2f mismatches %d\n", T, EM, sizes[s], cy / cnt,
           cy / cnt / sizes[s], b);
  }
  printf("hits %llu misses %llu bad %d bad_rec %d\n", hctr[0], hctr[1], bad, bad_rec);
  return bad != 0 || bad_rec != 0;
}
