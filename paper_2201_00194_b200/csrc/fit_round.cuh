// fit_round.cuh - the multi-kernel boosting round (families too large for one CTA: C4/C5)
// Part of the trainer translation unit: included once, by fit.cu only (shares its
// anonymous namespace, constants and helpers).
#pragma once

namespace fs {
namespace fit {
namespace {

// Which nodes at `level` are screened, which histograms are built directly / derived (one node).
__device__ __forceinline__ void plan_node(const FamDesc& fd, NodeRec* __restrict__ nodes, int level, int local) {
  const int first = (1 << level) - 1;
  NodeRec* nd = nodes + fd.node0;
  const int s = first + local;
  if (level == 0) {
    if (fd.nrep > 0 && node_needs_split(fd, 0, nd[0].n)) nd[0].build = 1;
    else nd[0].state = kNodeLeaf;
    return;
  }
  const int parent = (s - 1) >> 1;
  if (nd[parent].state != kNodeSplit) return;
  const bool need = fd.nrep > 0 && node_needs_split(fd, level, nd[s].n);
  if (!need) nd[s].state = kNodeLeaf;
  if (s & 1) {  // left child decides the pair's build plan
    const int sib = s + 1;
    const bool need_sib = fd.nrep > 0 && node_needs_split(fd, level, nd[sib].n);
    if (need || need_sib) {
      const int small = nd[s].n <= nd[sib].n ? s : sib;
      nd[small].build = 1;
      nd[small == s ? sib : s].build = 2;
    }
  }
}

__global__ void level_plan_kernel(const FamDesc* __restrict__ fam, const FamState* __restrict__ st,
                                  NodeRec* __restrict__ nodes, int level) {
  FS_PDL_WAIT();
  const int f = blockIdx.y;
  const FamDesc fd = fam[f];
  if (!st[f].active) return;
  const int local = blockIdx.x * blockDim.x + threadIdx.x;
  if (local < (1 << level)) plan_node(fd, nodes, level, local);
}

// A level's preparation in one launch: the node plan (block 0 of each family), the level's
// histogram slots zeroed, the level's two work-list counters (tie-class items, exact items).
__global__ void level_prep_kernel(const FamDesc* __restrict__ fam, const FamState* __restrict__ st,
                                  NodeRec* __restrict__ nodes, int level, int64_t* __restrict__ hsum,
                                  int32_t* __restrict__ hcnt, int* __restrict__ n_items) {
  FS_PDL_WAIT();
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x < 2) n_items[threadIdx.x] = 0;
  const int f = blockIdx.y;
  const FamDesc fd = fam[f];
  if (!st[f].active) return;
  if (blockIdx.x == 0)
    for (int local = threadIdx.x; local < (1 << level); local += blockDim.x) plan_node(fd, nodes, level, local);
  if (level >= max(fd.depth, 1)) return;
  const int64_t base = fd.hist0 + static_cast<int64_t>(level & 1) * fd.level_slots * fd.bins;
  const int64_t cnt = static_cast<int64_t>(min(1 << level, fd.level_slots)) * fd.bins;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < cnt;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    hsum[base + i] = 0;
    hcnt[base + i] = 0;
  }
}

constexpr int kHistThreads = 256;
constexpr int kHistTileRows = 64;
constexpr int kHistChunk = 4096;

// Histogram of one directly-built node over one chunk of its rows. Threads own (feature, row
// group) pairs, so shared-memory bins are updated without atomics; the CTA then adds its
// partial histogram to the node's global histogram with integer atomics (exact, order-free).
template <typename CodeT, bool kGlobal>
__global__ void __launch_bounds__(kHistThreads) hist_build_kernel(
    const FamDesc* __restrict__ fam, const FamState* __restrict__ st, const NodeRec* __restrict__ nodes, int level,
    int Dp, const CodeT* __restrict__ codes_c, const int64_t* __restrict__ rfix, const int32_t* __restrict__ ord_cur,
    const int32_t* __restrict__ rep_boff, int64_t* __restrict__ hsum, int32_t* __restrict__ hcnt,
    int64_t* __restrict__ node_abs, int groups, unsigned long long* __restrict__ ctr) {
  FS_PDL_WAIT();
  extern __shared__ __align__(16) unsigned char smem[];
  const int f = blockIdx.z;
  const FamDesc fd = fam[f];
  if (!st[f].active) return;
  const NodeRec* nd = nodes + fd.node0;
  int s;
  if (level == 0) {
    if (blockIdx.y) return;
    s = 0;
  } else {
    if (blockIdx.y >= (1u << (level - 1))) return;
    const int parent = (1 << (level - 1)) - 1 + blockIdx.y;
    if (nd[parent].state != kNodeSplit) return;
    s = 2 * parent + 1;
    if (nd[s].build != 1) s += 1;
    if (nd[s].build != 1) return;
  }
  const int n_v = nd[s].n;
  const int r0 = blockIdx.x * kHistChunk;
  if (r0 >= n_v) return;
  const int rows = min(kHistChunk, n_v - r0);
  const int seg = nd[s].seg;
  const int local = s - ((1 << level) - 1);
  const int64_t hbase = fd.hist0 + (static_cast<int64_t>(level & 1) * fd.level_slots + local) * fd.bins;
  const int bins = fd.bins, nrep = fd.nrep;

  int64_t* s_sum = reinterpret_cast<int64_t*>(smem);
  int32_t* s_cnt = reinterpret_cast<int32_t*>(s_sum + (kGlobal ? 0 : static_cast<int64_t>(groups) * bins));
  unsigned char* tail = reinterpret_cast<unsigned char*>(s_cnt + (kGlobal ? 0 : static_cast<int64_t>(groups) * bins));
  tail = smem + ((static_cast<size_t>(tail - smem) + 15) & ~size_t(15));  // (stays a shared-space pointer: LDS, not generic loads)
  CodeT* t_codes = reinterpret_cast<CodeT*>(tail);                          // [kHistTileRows][Dp]
  int64_t* t_fix = reinterpret_cast<int64_t*>(t_codes + kHistTileRows * Dp);  // [kHistTileRows]
  __shared__ unsigned long long s_abs;
  const int tid = threadIdx.x;
  if (!kGlobal)
    for (int i = tid; i < groups * bins; i += kHistThreads) {
      s_sum[i] = 0;
      s_cnt[i] = 0;
    }
  if (tid == 0) s_abs = 0;
  // thread -> (feature, group)
  const int per_group = nrep > 0 ? (nrep < kHistThreads ? nrep : kHistThreads) : 1;
  const int g = tid / per_group;
  const int fj0 = tid - g * per_group;
  const bool worker = g < groups && fj0 < nrep;
  __syncthreads();
  const int vec_per_row = Dp * static_cast<int>(sizeof(CodeT)) / 16;
  for (int t0 = 0; t0 < rows; t0 += kHistTileRows) {
    const int tr = min(kHistTileRows, rows - t0);
    for (int i = tid; i < tr * vec_per_row; i += kHistThreads) {
      const int r = i / vec_per_row, v = i - r * vec_per_row;
      const int64_t p = fd.pos0 + ord_cur[fd.pos0 + seg + r0 + t0 + r];
      reinterpret_cast<uint4*>(t_codes + r * Dp)[v] = reinterpret_cast<const uint4*>(codes_c + p * Dp)[v];
    }
    unsigned long long a = 0;
    if (tid < tr) {
      const int64_t p = fd.pos0 + ord_cur[fd.pos0 + seg + r0 + t0 + tid];
      const int64_t v = rfix[p];
      t_fix[tid] = v;
      a = static_cast<unsigned long long>(v < 0 ? -v : v);
    }
    for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
    if ((tid & 31) == 0 && a) atomicAdd(&s_abs, a);
    __syncthreads();
    if (worker) {
      for (int fj = fj0; fj < nrep; fj += per_group) {
        const int boff = rep_boff[fd.rep0 + fj];
        for (int r = g; r < tr; r += groups) {
          const int bin = boff + static_cast<int>(t_codes[r * Dp + fj]);
          if (kGlobal) {
            atomicAdd(reinterpret_cast<unsigned long long*>(hsum + hbase + bin),
                      static_cast<unsigned long long>(t_fix[r]));
            atomicAdd(hcnt + hbase + bin, 1);
          } else {
            s_sum[g * bins + bin] += t_fix[r];
            s_cnt[g * bins + bin] += 1;
          }
        }
      }
    }
    __syncthreads();
  }
  if (!kGlobal) {
    for (int b = tid; b < bins; b += kHistThreads) {
      int64_t sm = 0;
      int32_t c = 0;
      for (int gg = 0; gg < groups; ++gg) {
        sm += s_sum[gg * bins + b];
        c += s_cnt[gg * bins + b];
      }
      if (c) {
        atomicAdd(reinterpret_cast<unsigned long long*>(hsum + hbase + b), static_cast<unsigned long long>(sm));
        atomicAdd(hcnt + hbase + b, c);
      }
    }
  }
  if (tid == 0 && s_abs)
    atomicAdd(reinterpret_cast<unsigned long long*>(node_abs + fd.node0 + s), s_abs);
  if (tid == 0) {
    atomicAdd(ctr + kCtrHistBytes,
              static_cast<unsigned long long>(rows) * (static_cast<unsigned long long>(nrep) * sizeof(CodeT) + 12ull));
    atomicAdd(ctr + kCtrHistRows, static_cast<unsigned long long>(rows));
  }
}

// Column-layout histogram build (the default shape). Warp w owns feature group fg = w % NFG
// (features 32fg .. 32fg+31, lane = feature) and row group w / NFG. A group's bins live in
// shared memory as [bin][32 lanes], so the 32 updates a warp issues for one row always hit 32
// different banks (no conflicts, no atomics); row groups own private copies that are summed at
// the flush. grp_off[f][fg] = entry offset of feature group fg (entries = bins x 32).
constexpr int kColWarps = 6;

template <typename CodeT>
__global__ void __launch_bounds__(kColWarps * 32) hist_build_col_kernel(
    const FamDesc* __restrict__ fam, const FamState* __restrict__ st, const NodeRec* __restrict__ nodes, int level,
    int Dp, const CodeT* __restrict__ codes_c, const int64_t* __restrict__ rfix, const int32_t* __restrict__ ord_cur,
    const int32_t* __restrict__ rep_boff, const int32_t* __restrict__ rep_nb, const int32_t* __restrict__ grp_off,
    const int32_t* __restrict__ grp_rg, int64_t* __restrict__ hsum, int32_t* __restrict__ hcnt,
    int64_t* __restrict__ node_abs, unsigned long long* __restrict__ ctr) {
  FS_PDL_WAIT();
  extern __shared__ __align__(16) unsigned char smem[];
  const int f = blockIdx.z;
  const FamDesc fd = fam[f];
  if (!st[f].active) return;
  const NodeRec* nd = nodes + fd.node0;
  int s;
  if (level == 0) {
    if (blockIdx.y) return;
    s = 0;
  } else {
    if (blockIdx.y >= (1u << (level - 1))) return;
    const int parent = (1 << (level - 1)) - 1 + blockIdx.y;
    if (nd[parent].state != kNodeSplit) return;
    s = 2 * parent + 1;
    if (nd[s].build != 1) s += 1;
    if (nd[s].build != 1) return;
  }
  const int n_v = nd[s].n;
  const int r0 = blockIdx.x * kHistChunk;
  if (r0 >= n_v) return;
  const int rows = min(kHistChunk, n_v - r0);
  const int seg = nd[s].seg;
  const int local = s - ((1 << level) - 1);
  const int64_t hbase = fd.hist0 + (static_cast<int64_t>(level & 1) * fd.level_slots + local) * fd.bins;
  const int nrep = fd.nrep;
  const int nfg = (nrep + 31) >> 5;
  const int32_t* go = grp_off + static_cast<int64_t>(f) * (kColWarps + 1);
  const int gsz = go[nfg];            // entries per copy
  const int rg = grp_rg[f];           // row groups (copies)
  int64_t* s_sum = reinterpret_cast<int64_t*>(smem);                        // [rg][gsz]
  int32_t* s_cnt = reinterpret_cast<int32_t*>(s_sum + static_cast<int64_t>(rg) * gsz);
  unsigned char* tail = reinterpret_cast<unsigned char*>(s_cnt + static_cast<int64_t>(rg) * gsz);
  tail = smem + ((static_cast<size_t>(tail - smem) + 15) & ~size_t(15));  // (stays a shared-space pointer: LDS, not generic loads)
  CodeT* t_codes = reinterpret_cast<CodeT*>(tail);                            // [kHistTileRows][Dp]
  int64_t* t_fix = reinterpret_cast<int64_t*>(t_codes + kHistTileRows * Dp);  // [kHistTileRows]
  __shared__ unsigned long long s_abs;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < rg * gsz; i += kColWarps * 32) {
    s_sum[i] = 0;
    s_cnt[i] = 0;
  }
  if (tid == 0) s_abs = 0;
  const int fg = warp % nfg, rgi = warp / nfg;
  const bool worker = rgi < rg;
  const int j = 32 * fg + lane;
  const bool jv = worker && j < nrep;
  int64_t* my_sum = s_sum + static_cast<int64_t>(rgi) * gsz + go[fg] + lane;
  int32_t* my_cnt = s_cnt + static_cast<int64_t>(rgi) * gsz + go[fg] + lane;
  __syncthreads();
  const int vec_per_row = Dp * static_cast<int>(sizeof(CodeT)) / 16;
  for (int t0 = 0; t0 < rows; t0 += kHistTileRows) {
    const int tr = min(kHistTileRows, rows - t0);
    for (int i = tid; i < tr * vec_per_row; i += kColWarps * 32) {
      const int r = i / vec_per_row, v = i - r * vec_per_row;
      const int64_t p = fd.pos0 + ord_cur[fd.pos0 + seg + r0 + t0 + r];
      reinterpret_cast<uint4*>(t_codes + r * Dp)[v] = reinterpret_cast<const uint4*>(codes_c + p * Dp)[v];
    }
    unsigned long long a = 0;
    for (int r = tid; r < tr; r += kColWarps * 32) {
      const int64_t p = fd.pos0 + ord_cur[fd.pos0 + seg + r0 + t0 + r];
      const int64_t v = rfix[p];
      t_fix[r] = v;
      a += static_cast<unsigned long long>(v < 0 ? -v : v);
    }
    for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
    if (lane == 0 && a) atomicAdd(&s_abs, a);
    __syncthreads();
    if (jv) {
      for (int r = rgi; r < tr; r += rg) {
        const int b = static_cast<int>(t_codes[r * Dp + j]);
        my_sum[b * 32] += t_fix[r];
        my_cnt[b * 32] += 1;
      }
    }
    __syncthreads();
  }
  // flush: entry e = (fg, b, lane) -> global bin boff_j + b
  for (int e = tid; e < gsz; e += kColWarps * 32) {
    int g = 0;
    while (g + 1 < nfg && go[g + 1] <= e) ++g;
    const int within = e - go[g];
    const int b = within >> 5, jj = 32 * g + (within & 31);
    if (jj >= nrep || b >= rep_nb[fd.rep0 + jj]) continue;
    int64_t sm = 0;
    int32_t c = 0;
    for (int k = 0; k < rg; ++k) {
      sm += s_sum[static_cast<int64_t>(k) * gsz + e];
      c += s_cnt[static_cast<int64_t>(k) * gsz + e];
    }
    if (c) {
      const int64_t gb = hbase + rep_boff[fd.rep0 + jj] + b;
      atomicAdd(reinterpret_cast<unsigned long long*>(hsum + gb), static_cast<unsigned long long>(sm));
      atomicAdd(hcnt + gb, c);
    }
  }
  if (tid == 0) {
    if (s_abs) atomicAdd(reinterpret_cast<unsigned long long*>(node_abs + fd.node0 + s), s_abs);
    atomicAdd(ctr + kCtrHistBytes,
              static_cast<unsigned long long>(rows) * (static_cast<unsigned long long>(nrep) * sizeof(CodeT) + 12ull));
    atomicAdd(ctr + kCtrHistRows, static_cast<unsigned long long>(rows));
  }
}

// Lane-column histogram shape (conflict-free shared atomics): lane l of every warp owns bank
// column l. nrep <= 32: lanes l < (32 / nrep) * nrep take feature l % nrep (copy l / nrep of
// it), so the column height is the largest bin count. nrep > 32: lane l takes features l, l+32,
// ... stacked in its column (cofs = offset of a feature's bins in its lane's column).
__host__ __device__ inline int col_height(int nrep, const int32_t* nb, int32_t* cofs) {
  int H = 1;
  if (nrep <= 32) {
    for (int j = 0; j < nrep; ++j) {
      if (cofs) cofs[j] = 0;
      H = nb[j] > H ? nb[j] : H;
    }
    return H;
  }
  for (int l = 0; l < 32; ++l) {
    int h = 0;
    for (int j = l; j < nrep; j += 32) {
      if (cofs) cofs[j] = h;
      h += nb[j];
    }
    H = h > H ? h : H;
  }
  return H;
}

// Limb-atomic histogram build (the default shape). Only 32-bit shared-memory atomics are native
// on sm_100a (64-bit ones compile to CAS spin loops), so each 62-bit fixed-point residual v is
// offset to u = v + 2^62 (in [0, 2^63)) and split into three 21-bit limbs accumulated with
// native 32-bit atomics by ALL 1024 threads (any thread may update any bin). Limb sums over at
// most kAtomSub = 2048 rows stay below 2^32; they are then folded exactly into 64-bit per-bin
// accumulators: U = S0 + S1*2^21 + S2*2^42, count = (U + 2^61) >> 62 (|sum v| < 2^61 by the
// choice of the fixed-point shift), sum = U - count*2^62. No count atomic is needed.
constexpr int kAtomThreads = 1024;
constexpr int kAtomSub = 2048;
constexpr int kAtomChunk = 8192;  // max rows per CTA (fewer when the batch is small: >= 2 CTAs per SM)
constexpr int kAtomTile = 128;
constexpr int kAtomPre = 2;  // uint4 of the next tile's code rows held in registers per thread (kPipe)
constexpr int kAtomCofRegs = 8;  // lane column offsets kept in registers (nrep <= 256)
constexpr int kAtomPipeChunk = 8 * kAtomTile;  // rows per CTA from which the pipelined shape is used
constexpr int kAtomPipeTile = 224;  // pipelined shape: rows per tile (fewer barriers; 224 x 9 uint4 fit 2 per thread)
constexpr uint32_t kLimbMask = (1u << 21) - 1u;

// kPipe: one CTA per SM (64 registers per thread) holding the next tile's gathers in registers
// (for launches whose CTAs walk many tiles, C5-sized); otherwise two CTAs per SM overlap each
// other's gather latency (few tiles per CTA, C4-sized).
template <typename CodeT, bool kPipe>
__global__ void __launch_bounds__(kAtomThreads, kPipe ? 1 : 2) hist_build_atomic_kernel(
    const FamDesc* __restrict__ fam, const FamState* __restrict__ st, const NodeRec* __restrict__ nodes, int level,
    int Dp, const CodeT* __restrict__ codes_c, const int64_t* __restrict__ rfix, const int32_t* __restrict__ ord_cur,
    const int32_t* __restrict__ rep_boff, int64_t* __restrict__ hsum, int32_t* __restrict__ hcnt,
    int64_t* __restrict__ node_abs, unsigned long long* __restrict__ ctr, int colh_max, int chunk) {
  FS_PDL_WAIT();
  extern __shared__ __align__(16) unsigned char smem[];
  const int f = blockIdx.z;
  const FamDesc fd = fam[f];
  if (!st[f].active) return;
  const NodeRec* nd = nodes + fd.node0;
  int s;
  if (level == 0) {
    if (blockIdx.y) return;
    s = 0;
  } else {
    if (blockIdx.y >= (1u << (level - 1))) return;
    const int parent = (1 << (level - 1)) - 1 + blockIdx.y;
    if (nd[parent].state != kNodeSplit) return;
    s = 2 * parent + 1;
    if (nd[s].build != 1) s += 1;
    if (nd[s].build != 1) return;
  }
  const int n_v = nd[s].n;
  const int r0 = blockIdx.x * chunk;
  if (r0 >= n_v) return;
  const int rows = min(chunk, n_v - r0);
  const int seg = nd[s].seg;
  const int local = s - ((1 << level) - 1);
  const int64_t hbase = fd.hist0 + (static_cast<int64_t>(level & 1) * fd.level_slots + local) * fd.bins;
  const int nrep = fd.nrep, bins = fd.bins;
  // the i-th row of the node: at the root every row belongs, and integer sums do not depend on
  // the order, so the root streams rows in canonical order (coalesced tiles) instead of
  // gathering them through the order-0 list
  auto row_at = [&](int i) -> int64_t { return level == 0 ? i : ord_cur[fd.pos0 + i]; };
  // layout: limbs[colh_max][3][32] u32 (lane columns, see col_height; a cell's three limbs 128 B
  // apart, so one address + immediate offsets per (row, feature)) | acc_sum[bins] i64 |
  // acc_cnt[bins] i32 | binrep[bins] u16 | boff[nrep] | cofs[nrep] | tile codes | tile limbs
  uint32_t* limb = reinterpret_cast<uint32_t*>(smem);
  int64_t* acc_sum =
      reinterpret_cast<int64_t*>(smem + ((static_cast<size_t>(3) * colh_max * 32 * 4 + 15) & ~size_t(15)));
  int32_t* acc_cnt = reinterpret_cast<int32_t*>(acc_sum + bins);
  uint16_t* s_binrep = reinterpret_cast<uint16_t*>(acc_cnt + bins);
  int32_t* s_boff = reinterpret_cast<int32_t*>(s_binrep + ((bins + 1) & ~1));
  int32_t* s_cofs = s_boff + nrep;
  int32_t* s_nbv = s_cofs + nrep;
  unsigned char* tail = reinterpret_cast<unsigned char*>(s_nbv + nrep);
  tail = smem + ((static_cast<size_t>(tail - smem) + 15) & ~size_t(15));  // (stays a shared-space pointer: LDS, not generic loads)
  CodeT* t_codes = reinterpret_cast<CodeT*>(tail);                              // [kAtomTile][Dp]
  uint32_t* t_limb = reinterpret_cast<uint32_t*>(t_codes + kAtomTile * Dp);     // [kAtomTile][4] (3 limbs + pad: one 16-byte load)
  __shared__ unsigned long long s_abs;
  __shared__ int s_colh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int b = tid; b < bins; b += kAtomThreads) {
    acc_sum[b] = 0;
    acc_cnt[b] = 0;
  }
  for (int j = tid; j < nrep; j += kAtomThreads) {
    const int b0 = rep_boff[fd.rep0 + j];
    const int b1 = j + 1 < nrep ? rep_boff[fd.rep0 + j + 1] : bins;
    s_boff[j] = b0;
    s_nbv[j] = b1 - b0;
    for (int b = b0; b < b1; ++b) s_binrep[b] = static_cast<uint16_t>(j);
  }
  if (tid == 0) s_abs = 0;
  __syncthreads();
  if (tid == 0) s_colh = col_height(nrep, s_nbv, s_cofs);
  __syncthreads();
  const int colh = s_colh;
  const int rpw = nrep <= 32 ? 32 / nrep : 1;  // rows per warp step (lane copies, nrep <= 32)
  const int hj = nrep <= 32 ? lane % nrep : lane;
  const int hm = nrep <= 32 ? lane / nrep : 0;
  const bool hact = nrep <= 32 ? hm < rpw : true;
  const int vec_per_row = Dp * static_cast<int>(sizeof(CodeT)) / 16;
  // per-lane column offsets of the lane's features (nrep > 32: features lane, lane + 32, ...)
  int cofr[kAtomCofRegs];
#pragma unroll
  for (int t = 0; t < kAtomCofRegs; ++t) cofr[t] = kPipe && lane + 32 * t < nrep ? s_cofs[lane + 32 * t] : 0;
  // one row of the tile into the lane columns (hact lanes; r = the tile row)
  auto add_rows = [&](const CodeT* tc, const uint32_t* tl_all, int tr) {
    if (!hact) return;
    uint32_t* colp = limb + lane;
    if (nrep <= 32) {
      for (int r = warp * rpw + hm; r < tr; r += (kAtomThreads / 32) * rpw) {
        const uint4 lv = reinterpret_cast<const uint4*>(tl_all)[r];
        uint32_t* c = colp + static_cast<int>(tc[r * Dp + hj]) * 96;
        atomicAdd(c, lv.x);
        atomicAdd(c + 32, lv.y);
        atomicAdd(c + 64, lv.z);
      }
    } else if (kPipe && nrep <= 32 * kAtomCofRegs) {  // (registers to spare only in the 1-CTA shape)
      for (int r = warp; r < tr; r += kAtomThreads / 32) {
        const uint4 lv = reinterpret_cast<const uint4*>(tl_all)[r];
        const uint32_t l0 = lv.x, l1 = lv.y, l2 = lv.z;
        const CodeT* cr = tc + r * Dp;
#pragma unroll
        for (int t = 0; t < kAtomCofRegs; ++t) {
          const int j = lane + 32 * t;
          if (j >= nrep) break;
          uint32_t* c = colp + (cofr[t] + static_cast<int>(cr[j])) * 96;
          atomicAdd(c, l0);
          atomicAdd(c + 32, l1);
          atomicAdd(c + 64, l2);
        }
      }
    } else {
      for (int r = warp; r < tr; r += kAtomThreads / 32) {
        const uint4 lv = reinterpret_cast<const uint4*>(tl_all)[r];
        const uint32_t l0 = lv.x, l1 = lv.y, l2 = lv.z;
        const CodeT* cr = tc + r * Dp;
        for (int j = lane; j < nrep; j += 32) {
          uint32_t* c = colp + (s_cofs[j] + static_cast<int>(cr[j])) * 96;
          atomicAdd(c, l0);
          atomicAdd(c + 32, l1);
          atomicAdd(c + 64, l2);
        }
      }
    }
  };
  for (int sub0 = 0; sub0 < rows; sub0 += kAtomSub) {
    for (int i = tid; i < 3 * colh * 32; i += kAtomThreads) limb[i] = 0;
    __syncthreads();
    const int sub_end = min(rows, sub0 + kAtomSub);
    const bool pipe = kPipe && kAtomPipeTile * vec_per_row <= kAtomPre * kAtomThreads;
    if (pipe) {
      // Software pipeline, one barrier per tile: registers hold tile t+1's gathered code rows
      // (and residual); they go to the other tile buffer, tile t+2's gathers are issued into the
      // same registers, then tile t is accumulated. The buffer written at tile t was last read
      // at tile t-1, and tile t's buffer was written at tile t-1: the barrier closing each tile
      // orders both.
      uint4 pv[kAtomPre];
      int64_t pfix = 0;
#define FS_ATOM_PREFETCH(T0)                                                        \
  do {                                                                              \
    const int tr_ = min(kAtomPipeTile, sub_end - (T0));                                 \
    _Pragma("unroll") for (int q = 0; q < kAtomPre; ++q) {                          \
      const int i = tid + q * kAtomThreads;                                         \
      if (i < tr_ * vec_per_row) {                                                  \
        const int r = i / vec_per_row, v = i - r * vec_per_row;                     \
        const int64_t p = fd.pos0 + row_at(seg + r0 + (T0) + r);                      \
        pv[q] = reinterpret_cast<const uint4*>(codes_c + p * Dp)[v];               \
      }                                                                             \
    }                                                                               \
    if (tid < tr_) pfix = rfix[fd.pos0 + row_at(seg + r0 + (T0) + tid)];           \
  } while (0)
      // the registers' tile into buffer b (codes, limbs, |v| into s_abs)
#define FS_ATOM_STAGE(T0, B)                                                                        \
  do {                                                                                              \
    const int tr_ = min(kAtomPipeTile, sub_end - (T0));                                                 \
    CodeT* tc_ = t_codes + (B) * (kAtomPipeTile * Dp + 16 * kAtomPipeTile / static_cast<int>(sizeof(CodeT)));  \
    uint32_t* tl_ = reinterpret_cast<uint32_t*>(tc_ + kAtomPipeTile * Dp);                              \
    _Pragma("unroll") for (int q = 0; q < kAtomPre; ++q) {                                          \
      const int i = tid + q * kAtomThreads;                                                         \
      if (i < tr_ * vec_per_row) {                                                                  \
        const int r = i / vec_per_row, v = i - r * vec_per_row;                                     \
        reinterpret_cast<uint4*>(tc_ + r * Dp)[v] = pv[q];                                          \
      }                                                                                             \
    }                                                                                               \
    unsigned long long a_ = 0;                                                                      \
    if (tid < tr_) {                                                                                \
      const uint64_t u = static_cast<uint64_t>(pfix) + (1ull << 62);                                \
      reinterpret_cast<uint4*>(tl_)[tid] = make_uint4(static_cast<uint32_t>(u) & kLimbMask,          \
                                                      static_cast<uint32_t>(u >> 21) & kLimbMask,    \
                                                      static_cast<uint32_t>(u >> 42), 0u);           \
      a_ = static_cast<unsigned long long>(pfix < 0 ? -pfix : pfix);                                \
    }                                                                                               \
    if (warp * 32 < tr_) {                                                                          \
      for (int o = 16; o > 0; o >>= 1) a_ += __shfl_xor_sync(0xffffffffu, a_, o);                   \
      if (lane == 0 && a_) atomicAdd(&s_abs, a_);                                                   \
    }                                                                                               \
  } while (0)
      FS_ATOM_PREFETCH(sub0);
      FS_ATOM_STAGE(sub0, 0);
      if (sub0 + kAtomPipeTile < sub_end) FS_ATOM_PREFETCH(sub0 + kAtomPipeTile);
      __syncthreads();
      int buf = 0;
      for (int t0 = sub0; t0 < sub_end; t0 += kAtomPipeTile) {
        const int tr = min(kAtomPipeTile, sub_end - t0);
        if (t0 + kAtomPipeTile < sub_end) {
          FS_ATOM_STAGE(t0 + kAtomPipeTile, buf ^ 1);
          if (t0 + 2 * kAtomPipeTile < sub_end) FS_ATOM_PREFETCH(t0 + 2 * kAtomPipeTile);
        }
        const CodeT* tc = t_codes + buf * (kAtomPipeTile * Dp + 16 * kAtomPipeTile / static_cast<int>(sizeof(CodeT)));
        add_rows(tc, reinterpret_cast<const uint32_t*>(tc + kAtomPipeTile * Dp), tr);
        __syncthreads();
        buf ^= 1;
      }
#undef FS_ATOM_PREFETCH
#undef FS_ATOM_STAGE
    } else {
      for (int t0 = sub0; t0 < sub_end; t0 += kAtomTile) {
        const int tr = min(kAtomTile, sub_end - t0);
        for (int i = tid; i < tr * vec_per_row; i += kAtomThreads) {
          const int r = i / vec_per_row, v = i - r * vec_per_row;
          const int64_t p = fd.pos0 + row_at(seg + r0 + t0 + r);
          reinterpret_cast<uint4*>(t_codes + r * Dp)[v] = reinterpret_cast<const uint4*>(codes_c + p * Dp)[v];
        }
        unsigned long long a = 0;
        if (tid < tr) {
          const int64_t v = rfix[fd.pos0 + row_at(seg + r0 + t0 + tid)];
          const uint64_t u = static_cast<uint64_t>(v) + (1ull << 62);
          reinterpret_cast<uint4*>(t_limb)[tid] = make_uint4(static_cast<uint32_t>(u) & kLimbMask,
                                                             static_cast<uint32_t>(u >> 21) & kLimbMask,
                                                             static_cast<uint32_t>(u >> 42), 0u);
          a = static_cast<unsigned long long>(v < 0 ? -v : v);
        }
        if (warp * 32 < tr) {
          for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
          if (lane == 0 && a) atomicAdd(&s_abs, a);
        }
        __syncthreads();
        add_rows(t_codes, t_limb, tr);
        __syncthreads();
      }
    }
    for (int b = tid; b < bins; b += kAtomThreads) {
      const int j = s_binrep[b], bb = b - s_boff[j];
      unsigned __int128 U = 0;
      if (nrep <= 32) {
        for (int m = 0; m < rpw; ++m) {
          const uint32_t* c = limb + bb * 96 + j + m * nrep;
          U += static_cast<unsigned __int128>(c[0]) + (static_cast<unsigned __int128>(c[32]) << 21) +
               (static_cast<unsigned __int128>(c[64]) << 42);
        }
      } else {
        const uint32_t* c = limb + (s_cofs[j] + bb) * 96 + (j & 31);
        U = static_cast<unsigned __int128>(c[0]) + (static_cast<unsigned __int128>(c[32]) << 21) +
            (static_cast<unsigned __int128>(c[64]) << 42);
      }
      const uint64_t c = static_cast<uint64_t>((U + (static_cast<unsigned __int128>(1) << 61)) >> 62);
      const unsigned __int128 sv = U - (static_cast<unsigned __int128>(c) << 62);
      acc_sum[b] += static_cast<int64_t>(static_cast<uint64_t>(sv));
      acc_cnt[b] += static_cast<int32_t>(c);
    }
    __syncthreads();
  }
  for (int b = tid; b < bins; b += kAtomThreads) {
    if (acc_cnt[b]) {
      atomicAdd(reinterpret_cast<unsigned long long*>(hsum + hbase + b), static_cast<unsigned long long>(acc_sum[b]));
      atomicAdd(hcnt + hbase + b, acc_cnt[b]);
    }
  }
  if (tid == 0) {
    if (s_abs) atomicAdd(reinterpret_cast<unsigned long long*>(node_abs + fd.node0 + s), s_abs);
    atomicAdd(ctr + kCtrHistBytes,
              static_cast<unsigned long long>(rows) * (static_cast<unsigned long long>(nrep) * sizeof(CodeT) + 12ull));
    atomicAdd(ctr + kCtrHistRows, static_cast<unsigned long long>(rows));
  }
}

inline size_t hist_atomic_smem(int bins, int nrep, int Dp, int code_bytes, int colh) {
  size_t o = (static_cast<size_t>(3) * colh * 32 * 4 + 15) & ~size_t(15);
  o += static_cast<size_t>(bins) * 14 + static_cast<size_t>(nrep) * 12 + 16;
  o = (o + 15) & ~size_t(15);
  const size_t tile = static_cast<size_t>(std::max(kAtomTile, kAtomPipeTile));
  o += 2 * (tile * Dp * code_bytes + tile * 16) + 16;  // 2 tiles
  return o;
}

// Screened gain of one candidate plus a rigorous bound on |reference gain - screened gain|.
// ls/ts: fixed-point left/total sums; S: sum|r| of the node (real units); scale = 2^-shift.
// The reference folds sums sequentially (error <= gamma_n * S each), R = T - L rounds once,
// then ((L*L)/lc + (R*R)/rc) - (T*T)/n rounds ~5 more times; the screen's sums are exact on
// the quantised residuals (quantisation <= n * scale / 2). Factor 2 covers both sides.
__device__ __forceinline__ void screen_gain_d(int64_t ls, int64_t ts, int lc, int n, double scale, double S, double& g,
                                              double& delta) {
  const double u = 1.1102230246251565e-16;
  const double L = static_cast<double>(ls) * scale, T = static_cast<double>(ts) * scale;
  const double R = static_cast<double>(ts - ls) * scale;
  const int rc = n - lc;
  // three reciprocals instead of nine divisions; their extra rounding (<= 1 ulp per term) is
  // covered by the 6u term below
  const double ilc = 1.0 / lc, irc = 1.0 / rc, in = 1.0 / n;
  const double A = L * L * ilc, B = R * R * irc, P = T * T * in;
  g = (A + B) - P;
  const double nu = static_cast<double>(n) * u;
  const double gam = nu / (1.0 - nu);
  const double q = static_cast<double>(n) * 0.5 * scale;
  const double EL = gam * S + q, ET = gam * S + q, ER = 2.0 * gam * S + 2.0 * q + u * fabs(R);
  const double aL = fabs(L) + EL, aR = fabs(R) + ER, aT = fabs(T) + ET;
  const double dA = ((2.0 * fabs(L) + EL) * EL + 4.0 * u * aL * aL) * ilc;
  const double dB = ((2.0 * fabs(R) + ER) * ER + 4.0 * u * aR * aR) * irc;
  const double dP = ((2.0 * fabs(T) + ET) * ET + 4.0 * u * aT * aT) * in;
  delta = 2.0 * (dA + dB + dP + 6.0 * u * (A + B + P)) * (1.0 + 8.0 * u) + 1e-300;
}

__device__ __forceinline__ void screen_gain(int64_t ls, int64_t ts, int lc, int n, double scale, double S, double& g,
                                            double& lo, double& hi) {
  double delta;
  screen_gain_d(ls, ts, lc, n, scale, S, g, delta);
  lo = g - delta;
  hi = g + delta;
}

template <class T>
__device__ __forceinline__ T warp_incl_scan(T v, int lane) {
  for (int o = 1; o < 32; o <<= 1) {
    const T t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// One thread per (family, node at level, rep). pass 0: max lower bound per node. pass 1:
// window membership (hi >= LO and hi > 0), per-feature best candidate, node window count.
__global__ void screen_kernel(const FamDesc* __restrict__ fam, const FamState* __restrict__ st,
                              NodeRec* __restrict__ nodes, int level, int64_t* __restrict__ hsum,
                              int32_t* __restrict__ hcnt, int64_t* __restrict__ node_abs,
                              const int32_t* __restrict__ rep_boff, const int32_t* __restrict__ rep_nb,
                              WinRec* __restrict__ win, int nrep_max, int level_slots_max, int pass,
                              double2* __restrict__ gcache, int32_t* __restrict__ icache) {
  FS_PDL_WAIT();
  // warp per (node, rep), lanes over the rep's bins: coalesced histogram reads, warp prefix
  // scans for the left count / sum, every candidate's screen in parallel (pass 0); pass 1 reads
  // each candidate's (gain, bound) and left count back from pass 0's cache (the histogram's cells)
  const int f = blockIdx.z;
  const FamDesc fd = fam[f];
  if (!st[f].active) return;
  const int local = blockIdx.y;
  if (local >= (1 << level)) return;
  const int lane = threadIdx.x & 31;
  const int jj = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (jj >= fd.nrep) return;
  const int s = (1 << level) - 1 + local;
  NodeRec& nd = nodes[fd.node0 + s];
  if (nd.state != 0 || nd.build == 0) return;
  const int n = nd.n;
  const int64_t hb = fd.hist0 + (static_cast<int64_t>(level & 1) * fd.level_slots + local) * fd.bins +
                     rep_boff[fd.rep0 + jj];
  const int nb = rep_nb[fd.rep0 + jj];
  const double scale = ldexp(1.0, -st[f].shift);
  int64_t nabs = node_abs[fd.node0 + s];
  if (pass == 0 && nd.build == 2) {
    // the sibling-derived histogram (parent - built sibling), this warp's feature: written here
    // for the pass-1 screen and the next level's derivations (no separate derive launch)
    const int parent = (s - 1) >> 1, sib = (s & 1) ? s + 1 : s - 1;
    const int first = (1 << level) - 1, pfirst = (1 << (level - 1)) - 1;
    const int64_t hs = fd.hist0 + (static_cast<int64_t>(level & 1) * fd.level_slots + (sib - first)) * fd.bins +
                       rep_boff[fd.rep0 + jj];
    const int64_t hp = fd.hist0 + (static_cast<int64_t>((level - 1) & 1) * fd.level_slots + (parent - pfirst)) * fd.bins +
                       rep_boff[fd.rep0 + jj];
    for (int b = lane; b < nb; b += 32) {
      hsum[hb + b] = hsum[hp + b] - hsum[hs + b];
      hcnt[hb + b] = hcnt[hp + b] - hcnt[hs + b];
    }
    __syncwarp();
    nabs = node_abs[fd.node0 + parent] - node_abs[fd.node0 + sib];
    if (jj == 0 && lane == 0) node_abs[fd.node0 + s] = nabs;
  }
  double best_lo = -INFINITY, bg = -INFINITY, bl = 0.0;
  int bb = 0x7fffffff, blc = 0, count = 0, mlc = 0;
  if (!pass) {
    const double S = static_cast<double>(nabs) * scale * (1.0 + 1e-12);
    int64_t ts = 0;
    for (int b = lane; b < nb; b += 32) ts += hsum[hb + b];
    for (int o = 16; o > 0; o >>= 1) ts += __shfl_xor_sync(0xffffffffu, ts, o);
    int carry_c = 0;
    int64_t carry_s = 0;
    for (int b0 = 0; b0 < nb; b0 += 32) {
      const int b = b0 + lane;
      const int cc = b < nb ? hcnt[hb + b] : 0;
      const int64_t sv = b < nb ? hsum[hb + b] : 0;
      const int ic = warp_incl_scan(cc, lane) + carry_c;
      const int64_t is = warp_incl_scan(sv, lane) + carry_s;
      if (b < nb) {
        double g = NAN, delta = 0.0;
        if (cc > 0 && ic < n) {  // a boundary after bin b (a later bin is non-empty)
          screen_gain_d(is, ts, ic, n, scale, S, g, delta);
          best_lo = fmax(best_lo, g - delta);
        }
        gcache[hb + b] = make_double2(g, delta);
        icache[hb + b] = ic;
      }
      carry_c = __shfl_sync(0xffffffffu, ic, 31);
      carry_s = __shfl_sync(0xffffffffu, is, 31);
    }
  } else {
    const double LO = lo_from_key(nd.lokey);
    for (int b = lane; b < nb; b += 32) {
      const double2 gd = gcache[hb + b];
      const double g = gd.x;
      if (isnan(g)) continue;
      const double lo = g - gd.y, hi = g + gd.y;  // = screen_gain's lo / hi
      if (hi >= LO && hi > 0.0) {
        const int ic = icache[hb + b];
        ++count;
        mlc = max(mlc, ic);
        if (g > bg || (g == bg && b < bb)) {
          bg = g;
          bl = lo;
          bb = b;
          blc = ic;
        }
      }
    }
  }
  if (!pass) {
    for (int o = 16; o > 0; o >>= 1) best_lo = fmax(best_lo, __shfl_xor_sync(0xffffffffu, best_lo, o));
    if (lane == 0 && best_lo > -INFINITY)
      atomicMax(reinterpret_cast<unsigned long long*>(&nd.lokey), lo_key(best_lo));
  } else {
    for (int o = 16; o > 0; o >>= 1) {
      count += __shfl_xor_sync(0xffffffffu, count, o);
      mlc = max(mlc, __shfl_xor_sync(0xffffffffu, mlc, o));
      const double og = __shfl_xor_sync(0xffffffffu, bg, o);
      const double ol = __shfl_xor_sync(0xffffffffu, bl, o);
      const int ob = __shfl_xor_sync(0xffffffffu, bb, o);
      const int olc = __shfl_xor_sync(0xffffffffu, blc, o);
      if (og > bg || (og == bg && ob < bb)) {
        bg = og;
        bl = ol;
        bb = ob;
        blc = olc;
      }
    }
    if (lane == 0) {
      WinRec w;
      w.best_g = bg;
      w.best_lo = bl;
      w.best_bin = count ? bb : -1;
      w.flag = count > 0;
      w.count = count;
      w.best_lc = blc;
      w.eq = 0;
      w.maxlc = mlc;
      win[(static_cast<int64_t>(f) * level_slots_max + local) * nrep_max + jj] = w;
      if (count) atomicAdd(&nd.wcount, count);
    }
  }
}

// Column-major copy of the canonical codes for the multi-kernel round: codes_cm[ord0 + j * n + p]
// (the presorted lists' layout). Tiles of 128 rows come in as 16-byte row vectors and go out as
// 128-byte column runs.
template <typename CodeT>
__global__ void __launch_bounds__(256) codes_colmajor_kernel(const FamDesc* __restrict__ fam, int Dp,
                                                             const CodeT* __restrict__ codes_c,
                                                             CodeT* __restrict__ codes_cm) {
  extern __shared__ __align__(16) unsigned char tile_raw[];
  CodeT* tile = reinterpret_cast<CodeT*>(tile_raw);  // [128][Dp + 1]
  const FamDesc fd = fam[blockIdx.y];
  const int r0 = blockIdx.x * 128;
  if (r0 >= fd.n || fd.nrep <= 0) return;
  const int rows = min(128, fd.n - r0), pitch = Dp + 1;
  for (int i = threadIdx.x; i < rows * Dp; i += blockDim.x) {
    const int r = i / Dp, j = i - r * Dp;
    tile[r * pitch + j] = codes_c[(fd.pos0 + r0 + r) * Dp + j];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < fd.nrep * rows; i += blockDim.x) {
    const int j = i / rows, r = i - j * rows;
    codes_cm[fd.ord0 + static_cast<int64_t>(j) * fd.n + r0 + r] = tile[r * pitch + j];
  }
}

struct ExactItem {
  int32_t fam;
  int16_t slot;
  int16_t rep;  // -1: node total
};

// Tie classes: a node whose window holds exactly one candidate per feature, all with the same
// left count, is one tie class if every window feature orders the node's rows exactly like the
// lowest one (identical folds, identical reference gains; strict > keeps the lowest feature).
// Prep queues one order-equivalence check per (node, other window feature).
// The per-node decision kernels below run a warp per (family, node) with lanes over the
// node's features (window records read in parallel; ballots replace the serial scans).
__device__ __forceinline__ int first_flag_feature(const WinRec* w, int nrep, int from, bool need_count1,
                                                  bool& multi) {
  // lowest flagged feature >= from; multi = some flagged feature has count != 1 (when asked)
  const int lane = threadIdx.x & 31;
  int first = -1;
  multi = false;
  for (int j0 = from; j0 < nrep; j0 += 32) {
    const int j = j0 + lane;
    const bool fl = j < nrep && w[j].flag;
    const unsigned m = __ballot_sync(0xffffffffu, fl);
    if (need_count1 && __any_sync(0xffffffffu, fl && w[j].count != 1)) multi = true;
    if (m && first < 0) first = j0 + __ffs(m) - 1;
  }
  return first;
}

__global__ void tieclass_prep_kernel(const FamDesc* __restrict__ fam, const FamState* __restrict__ st,
                                     NodeRec* __restrict__ nodes, int level, const WinRec* __restrict__ win,
                                     int nrep_max, int level_slots_max, ExactItem* __restrict__ items,
                                     int* __restrict__ n_items) {
  FS_PDL_WAIT();
  const int f = blockIdx.y;
  const FamDesc fd = fam[f];
  if (!st[f].active) return;
  const int lane = threadIdx.x & 31;
  const int local = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (local >= (1 << level)) return;
  const int s = (1 << level) - 1 + local;
  NodeRec& nd = nodes[fd.node0 + s];
  if (lane == 0) nd.eqf0 = -1;
  if (nd.state != 0 || nd.build == 0 || nd.wcount < 2) return;
  const WinRec* w = win + (static_cast<int64_t>(f) * level_slots_max + local) * nrep_max;
  bool multi;
  const int f0 = first_flag_feature(w, fd.nrep, 0, true, multi);
  if (multi || f0 < 0 || !(w[f0].best_lo > 0.0)) return;
  const int lc0 = w[f0].best_lc;
  bool diff = false;
  for (int j0 = f0 + 1; j0 < fd.nrep; j0 += 32) {
    const int j = j0 + lane;
    if (__any_sync(0xffffffffu, j < fd.nrep && w[j].flag && w[j].best_lc != lc0)) diff = true;
  }
  if (diff) return;
  if (lane == 0) nd.eqf0 = f0;
  for (int j0 = f0 + 1; j0 < fd.nrep; j0 += 32) {
    const int j = j0 + lane;
    const bool fl = j < fd.nrep && w[j].flag;
    const unsigned m = __ballot_sync(0xffffffffu, fl);
    int base = 0;
    if (lane == 0 && m) base = atomicAdd(n_items, __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (fl) items[base + __popc(m & ((1u << lane) - 1u))] = {f, static_cast<int16_t>(s), static_cast<int16_t>(j)};
  }
}

__global__ void decide_kernel(const FamDesc* __restrict__ fam, const FamState* __restrict__ st,
                              NodeRec* __restrict__ nodes, int level, const int32_t* __restrict__ hcnt,
                              const int32_t* __restrict__ rep_boff, const WinRec* __restrict__ win, int nrep_max,
                              int level_slots_max, ExactItem* __restrict__ items, int* __restrict__ n_items,
                              unsigned long long* __restrict__ ctr) {
  FS_PDL_WAIT();
  (void)hcnt;
  (void)rep_boff;
  const int f = blockIdx.y;
  const FamDesc fd = fam[f];
  if (!st[f].active) return;
  const int lane = threadIdx.x & 31;
  const int local = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (local >= (1 << level)) return;
  const int s = (1 << level) - 1 + local;
  NodeRec& nd = nodes[fd.node0 + s];
  if (nd.state != 0 || nd.build == 0) return;
  const WinRec* w = win + (static_cast<int64_t>(f) * level_slots_max + local) * nrep_max;
  if (nd.wcount == 0) {  // no candidate can have a positive reference gain
    if (lane == 0) nd.state = kNodeLeaf;
    return;
  }
  int pick = -1;
  if (nd.wcount == 1) {
    bool multi;
    const int j = first_flag_feature(w, fd.nrep, 0, false, multi);
    if (j >= 0 && w[j].best_lo > 0.0) pick = j;
  } else if (nd.eqf0 >= 0) {  // one tie class: the lowest feature wins by strict >
    bool all = true;
    for (int j0 = nd.eqf0 + 1; j0 < fd.nrep; j0 += 32) {
      const int j = j0 + lane;
      if (__any_sync(0xffffffffu, j < fd.nrep && w[j].flag && !w[j].eq)) all = false;
    }
    if (all) pick = nd.eqf0;
  }
  if (pick >= 0) {
    if (lane == 0) {
      nd.state = kNodeSplit;
      nd.rep = pick;
      nd.bin = w[pick].best_bin;
      nd.gain = w[pick].best_g;
      nd.lc = w[pick].best_lc;
      atomicAdd(&const_cast<FamState*>(st)[f].screened, 1ull);
    }
    return;
  }
  const int tot = nd.pad_ ? 0 : 1;  // node total still to fold (not precomputed by totals_kernel)
  int k = tot;
  for (int j0 = 0; j0 < fd.nrep; j0 += 32) {
    const int j = j0 + lane;
    k += __popc(__ballot_sync(0xffffffffu, j < fd.nrep && w[j].flag));
  }
  int base = 0;
  if (lane == 0) {
    nd.state = kNodeExact;
    atomicAdd(&const_cast<FamState*>(st)[f].exact, 1ull);
    base = atomicAdd(n_items, k);
    atomicAdd(ctr + kCtrExactChains, static_cast<unsigned long long>(k));
    atomicAdd(ctr + kCtrExactNodes, 1ull);
    if (tot) items[base] = {f, static_cast<int16_t>(s), static_cast<int16_t>(-1)};
  }
  base = __shfl_sync(0xffffffffu, base, 0) + tot;
  for (int j0 = 0; j0 < fd.nrep; j0 += 32) {
    const int j = j0 + lane;
    const bool fl = j < fd.nrep && w[j].flag;
    const unsigned m = __ballot_sync(0xffffffffu, fl);
    if (fl) items[base + __popc(m & ((1u << lane) - 1u))] = {f, static_cast<int16_t>(s), static_cast<int16_t>(j)};
    base += __popc(m);
  }
}

// One warp per check: walk the lowest window feature's presorted list restricted to the node;
// the other feature must tie exactly where it ties and increase where it increases.
// Order equivalence of g with f0 on the node's rows <=> the map code_f0 -> code_g over those rows
// is a function that strictly increases (ties align, and the stable sorts by (code, canonical
// position) then coincide). CTA per item: phi[a] = the g code of some row with f0 code a (racy
// plain stores), every row must agree with phi, phi must increase over the present a. Rows come
// from the node's order-0 segment, in any order - no scan of the presorted lists.
template <typename CodeT>
__global__ void __launch_bounds__(256) tieclass_phi_kernel(
    const FamDesc* __restrict__ fam, const NodeRec* __restrict__ nodes, const ExactItem* __restrict__ items,
    const int* __restrict__ n_items, int level, int Dp, const CodeT* __restrict__ codes_cm,
    const int32_t* __restrict__ ord_cur, const int32_t* __restrict__ rep_nb, WinRec* __restrict__ win,
    int nrep_max, int level_slots_max) {
  FS_PDL_WAIT();
  extern __shared__ __align__(16) unsigned char smem[];
  uint16_t* phi = reinterpret_cast<uint16_t*>(smem);
  const int tid = threadIdx.x, lane = tid & 31;
  const int total = *n_items;
  for (int wi = blockIdx.x; wi < total; wi += gridDim.x) {
    const ExactItem it = items[wi];
    const FamDesc fd = fam[it.fam];
    const NodeRec& nd = nodes[fd.node0 + it.slot];
    const int f0 = nd.eqf0, g = it.rep, nv = nd.n;
    const int nb = rep_nb[fd.rep0 + f0];
    const int32_t* rows = ord_cur + fd.pos0 + nd.seg;
    // column-major codes (codes_cm[ord0 + rep * n + row], built once per fit): a node's rows
    // gather from one feature's column (L2-resident) instead of one 32-byte sector per row
    const CodeT* cm_f0 = codes_cm + fd.ord0 + static_cast<int64_t>(f0) * fd.n;
    const CodeT* cm_g = codes_cm + fd.ord0 + static_cast<int64_t>(g) * fd.n;
    __syncthreads();  // previous item done with phi
    for (int a = tid; a < nb; a += blockDim.x) phi[a] = 0xFFFFu;
    __syncthreads();
    // 8 rows per thread in flight (index gathers, then both code gathers, then the table)
    for (int i0 = tid; i0 < nv; i0 += 8 * blockDim.x) {
      int64_t p[8];
      int cf[8], cg[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int i = i0 + k * static_cast<int>(blockDim.x);
        p[k] = i < nv ? rows[i] : -1;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        cf[k] = p[k] >= 0 ? static_cast<int>(cm_f0[p[k]]) : 0;
        cg[k] = p[k] >= 0 ? static_cast<int>(cm_g[p[k]]) : 0;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (p[k] >= 0) phi[cf[k]] = static_cast<uint16_t>(cg[k]);
    }
    __syncthreads();
    bool bad = false;
    for (int i0 = tid; i0 < nv; i0 += 8 * blockDim.x) {
      int64_t p[8];
      int cf[8], cg[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int i = i0 + k * static_cast<int>(blockDim.x);
        p[k] = i < nv ? rows[i] : -1;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        cf[k] = p[k] >= 0 ? static_cast<int>(cm_f0[p[k]]) : 0;
        cg[k] = p[k] >= 0 ? static_cast<int>(cm_g[p[k]]) : 0;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (p[k] >= 0) bad |= phi[cf[k]] != static_cast<uint16_t>(cg[k]);
    }
    if (tid < 32) {  // phi strictly increasing over the present f0 codes
      int carry = -1;
      for (int a0 = 0; a0 < nb; a0 += 32) {
        const int a = a0 + lane;
        const int v = a < nb ? phi[a] : 0xFFFF;
        const bool present = v != 0xFFFF;
        const unsigned m = __ballot_sync(0xffffffffu, present);
        const unsigned lt = m & ((1u << lane) - 1u);
        int pv = __shfl_sync(0xffffffffu, v, lt ? 31 - __clz(lt) : 0);
        if (!lt) pv = carry;
        if (present && pv >= 0 && v <= pv) bad = true;
        if (m) carry = __shfl_sync(0xffffffffu, v, 31 - __clz(m));
      }
    }
    bad = __syncthreads_or(bad);
    const int local = it.slot - ((1 << level) - 1);
    if (tid == 0) win[(static_cast<int64_t>(it.fam) * level_slots_max + local) * nrep_max + g].eq = !bad;
  }
}

template <typename CodeT>
__global__ void __launch_bounds__(256) tieclass_check_kernel(
    const FamDesc* __restrict__ fam, const NodeRec* __restrict__ nodes, const ExactItem* __restrict__ items,
    const int* __restrict__ n_items, int level, int Dp, const CodeT* __restrict__ codes_cm,
    const int32_t* __restrict__ ord, const int16_t* __restrict__ nodeid, WinRec* __restrict__ win, int nrep_max,
    int level_slots_max) {
  FS_PDL_WAIT();
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int total = *n_items;
  for (int wi = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; wi < total; wi += warps) {
    const ExactItem it = items[wi];
    const FamDesc fd = fam[it.fam];
    const NodeRec& nd = nodes[fd.node0 + it.slot];
    const int f0 = nd.eqf0, g = it.rep, nv = nd.n, n = fd.n;
    const int32_t* L = ord + fd.ord0 + static_cast<int64_t>(f0) * n;
    int pf = -1, pg = -1, seen = 0;
    bool bad = false;
    int p_next = lane < n ? L[lane] : 0;
    for (int i0 = 0; i0 < n && seen < nv; i0 += 32) {
      const int i = i0 + lane;
      const int p = p_next;
      p_next = i + 32 < n ? L[i + 32] : 0;
      const bool mem = i < n && nodeid[fd.pos0 + p] == it.slot;
      const int a = mem ? static_cast<int>(codes_cm[fd.ord0 + static_cast<int64_t>(f0) * n + p]) : 0;
      const int b = mem ? static_cast<int>(codes_cm[fd.ord0 + static_cast<int64_t>(g) * n + p]) : 0;
      const unsigned m = __ballot_sync(0xffffffffu, mem);
      seen += __popc(m);
      const unsigned lt = m & ((1u << lane) - 1u);
      const int src = lt ? 31 - __clz(lt) : lane;
      int qa = __shfl_sync(0xffffffffu, a, src), qb = __shfl_sync(0xffffffffu, b, src);
      if (!lt) {
        qa = pf;
        qb = pg;
      }
      if (mem && qa >= 0 && ((a == qa) != (b == qb) || b < qb)) bad = true;
      if (m) {
        const int last = 31 - __clz(m);
        pf = __shfl_sync(0xffffffffu, a, last);
        pg = __shfl_sync(0xffffffffu, b, last);
      }
    }
    bad = __any_sync(0xffffffffu, bad);
    const int local = it.slot - ((1 << level) - 1);
    if (lane == 0) win[(static_cast<int64_t>(it.fam) * level_slots_max + local) * nrep_max + g].eq = !bad;
  }
}

// Decide screened nodes; queue the rest for reference-order re-evaluation.
__device__ __forceinline__ double warp_fold_gather(const double* __restrict__ v, const int32_t* __restrict__ idx,
                                                   int n) {
  // Software-pipelined: the next 128 gathers (L2 latency) are in flight while the current 128
  // values are folded in order (the dependent FP64 add chain).
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  double x[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int i = 32 * c + lane;
    x[c] = i < n ? v[idx[i]] : 0.0;
  }
  for (int i0 = 0; i0 < n; i0 += 128) {
    double y[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = i0 + 128 + 32 * c + lane;
      y[c] = i < n ? v[idx[i]] : 0.0;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int base = i0 + 32 * c;
      if (base >= n) break;
      const int m = min(32, n - base);
      if (m == 32) {
#pragma unroll
        for (int l0 = 0; l0 < 32; l0 += 8) {
          double t[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) t[k] = __shfl_sync(0xffffffffu, x[c], l0 + k);
#pragma unroll
          for (int k = 0; k < 8; ++k) s = fs_add(s, t[k]);
        }
      } else {
        for (int l = 0; l < m; ++l) s = fs_add(s, __shfl_sync(0xffffffffu, x[c], l));
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) x[c] = y[c];
  }
  return s;
}

// Node totals (costmodel.cpp:47, sum_residuals over the feature-0 list) for every node of the
// level that will be screened, on a forked stream: the reference-order chains run while the
// histogram / screen / tie-class kernels of the same level do. nd.pad_ = 1 marks the total valid
// (exact decisions and leaf values then reuse it - the same fold over the same segment).
__global__ void totals_kernel(const FamDesc* __restrict__ fam, const FamState* __restrict__ st,
                              NodeRec* __restrict__ nodes, int level, const int32_t* __restrict__ ord_cur,
                              const double* __restrict__ resid) {
  FS_PDL_WAIT();
  const int f = blockIdx.y;
  const FamDesc fd = fam[f];
  if (!st[f].active) return;
  const int local = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (local >= (1 << level)) return;
  NodeRec& nd = nodes[fd.node0 + (1 << level) - 1 + local];
  if (nd.state != 0 || nd.build == 0 || nd.n <= 0) return;
  const double t = warp_fold_gather(resid + fd.pos0, ord_cur + fd.pos0 + nd.seg, nd.n);
  if ((threadIdx.x & 31) == 0) {
    nd.total = t;
    nd.pad_ = 1;
  }
}


// (two_sum, dbl_ord, ord_dbl and the CTA-wide folds: fold_est.cuh)

// One warp per item: reference-order folds. Item rep < 0: node total over the order-0 list
// (sum_residuals(order[0]), costmodel.cpp:47). Item rep j: best_split's left sums over feature j's
// presorted list restricted to the node (:50-55), recorded at every value boundary.
// exact folds of nodes below a quarter of the family go through exact_small_kernel
__device__ __forceinline__ bool exact_is_small(int nv, int n) { return nv < n; }
#ifndef FS_EXACT_SPEC_MIN
#define FS_EXACT_SPEC_MIN 128
#endif
constexpr int kExactSpecMin = FS_EXACT_SPEC_MIN;  // chains from this length fold in a CTA (cta_fold_est / cta_fold_est_rec); 1,024 / 512 / 256 measured slower

// Exact reference-order folds for SMALL nodes (nv * 4 < n): instead of scanning the feature's
// full presorted list for the node's members (exact_kernel; costs O(n) gathers per item however
// small the node), a CTA compacts the node's rows in canonical order (a coalesced scan of the
// node ids), stable-sorts them by the feature's code (the presorted order restricted to the
// node is exactly (code, canonical position) order), and warp 0 folds them - the same adds in
// the same order as best_split (costmodel.cpp:50-69), stopping at the last window candidate.
#ifndef FS_EXACT_FOLD_E
#define FS_EXACT_FOLD_E 8
#endif
constexpr int kExactFoldE = FS_EXACT_FOLD_E;  // exact_small's fold sub-blocks (8 elements x 1,024 threads per super-segment)
template <typename CodeT>
constexpr size_t exact_small_smem() {
  const size_t fold = (static_cast<size_t>(fold_est_stage_doubles(kSortThreads, kExactFoldE)) +
                       fold_est_scratch_doubles(kSortThreads)) * 8 + static_cast<size_t>(kExactFoldE) * kSortThreads * sizeof(CodeT);
  return fold > sizeof(SortSmem) ? fold : sizeof(SortSmem);
}
template <typename CodeT>
__global__ void __launch_bounds__(kSortThreads) exact_small_kernel(
    const FamDesc* __restrict__ fam, NodeRec* __restrict__ nodes, const ExactItem* __restrict__ items,
    const int* __restrict__ n_items, int level, int Dp, const CodeT* __restrict__ codes_cm,
    const double* __restrict__ resid, const int32_t* __restrict__ ord, const int32_t* __restrict__ ord_cur,
    const int16_t* __restrict__ nodeid, const int32_t* __restrict__ rep_boff,
    double* __restrict__ lbuf, const WinRec* __restrict__ win, int nrep_max, int level_slots_max,
    int32_t* __restrict__ scratch, int n_max) {
  FS_PDL_WAIT();
  // the sort's and the speculative folds' shared memory overlap (never live together; the sort
  // state is re-initialised after a fold)
  union FoldOrSort {
    SortSmem sort;
    struct {
      double stage[fold_est_stage_doubles(kSortThreads, kExactFoldE)];
      double scr[fold_est_scratch_doubles(kSortThreads)];
      CodeT cst[kExactFoldE * kSortThreads];
    } fold;
  };
  extern __shared__ __align__(16) unsigned char xs_raw[];  // exact_small_smem<CodeT>() bytes
  FoldOrSort& u = *reinterpret_cast<FoldOrSort*>(xs_raw);
  SortSmem& sm = u.sort;
  __shared__ int wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int total = *n_items;
  sort_smem_init(sm);
  auto fold_at = [&](int64_t pos0, const int32_t* list, int len) {
    __syncthreads();  // the sort state is dead
    const double r = cta_fold_est<kExactFoldE>(resid + pos0, list, len, 0.0, u.fold.stage, u.fold.scr);
    sort_smem_init(sm);
    return r;
  };
  auto fold_rec = [&](int64_t pos0, const int32_t* list, int len, const CodeT* cj, double* out) {
    __syncthreads();
    cta_fold_est_rec<kExactFoldE, CodeT>(resid + pos0, list, len, cj, out, u.fold.stage, u.fold.cst, u.fold.scr);
    sort_smem_init(sm);
  };
  for (int w = blockIdx.x; w < total; w += gridDim.x) {
    const ExactItem it = items[w];
    const FamDesc fd = fam[it.fam];
    NodeRec& nd = nodes[fd.node0 + it.slot];
    const int nv = nd.n, n = fd.n;
    if (it.rep < 0) {  // a long node total: speculative CTA fold (exact_kernel folds the short ones)
      if (nv < kExactSpecMin) continue;
      const double t = fold_at(fd.pos0, ord_cur + fd.pos0 + nd.seg, nv);
      if (tid == 0) nd.total = t;
      continue;
    }
    const int jj = it.rep;
    const int local = it.slot - ((1 << level) - 1);
    const WinRec& wr = win[(static_cast<int64_t>(it.fam) * level_slots_max + local) * nrep_max + jj];
    const int need = wr.maxlc;
    double* out = lbuf + fd.lbuf0 + static_cast<int64_t>(local) * fd.bins + rep_boff[fd.rep0 + jj];
    // one window candidate: only L at its left count is read (exact_decide_kernel), so a long
    // fold needs only the fold up to that count (cta_fold_est, bit-exact)
    const bool spec_one = wr.count == 1 && need >= kExactSpecMin;
    const CodeT* cj = codes_cm + fd.ord0 + static_cast<int64_t>(jj) * fd.n;  // column-major
    if (!exact_is_small(nv, n)) {
      if (need < kExactSpecMin) continue;  // exact_kernel scans the presorted list
      // the root: every row is a member, the presorted list is the member list
      const int32_t* lst = ord + fd.ord0 + static_cast<int64_t>(jj) * fd.n;
      if (spec_one) {
        const double L = fold_at(fd.pos0, lst, need);
        if (tid == 0) out[wr.best_bin] = L;
      } else {
        fold_rec(fd.pos0, lst, need, cj, out);
      }
      continue;
    }
    int32_t* A = scratch + static_cast<int64_t>(blockIdx.x) * 2 * n_max;
    int32_t* B = A + n_max;
    // 1. the node's rows in canonical order: each thread tests 8 consecutive rows per pass (8x
    // fewer block scans than one row per thread), then a block scan of the per-thread counts
    int base = 0;
    for (int p0 = 0; p0 < n; p0 += 8 * static_cast<int>(blockDim.x)) {
      const int pb = p0 + 8 * tid;
      unsigned bits = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (pb + k < n && nodeid[fd.pos0 + pb + k] == it.slot) bits |= 1u << k;
      const int cnt = __popc(bits);
      int incl = cnt;  // warp inclusive scan of the per-thread counts
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (lane == 31) wsum[warp] = incl;
      __syncthreads();
      if (warp == 0) {
        const int v = lane < static_cast<int>(blockDim.x >> 5) ? wsum[lane] : 0;
        int wi = v;
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, wi, o);
          if (lane >= o) wi += t;
        }
        wsum[lane] = wi - v;
        if (lane == 31) sm.uniform = wi;  // pass total (borrowed field)
      }
      __syncthreads();
      int dst = base + wsum[warp] + incl - cnt;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (bits >> k & 1u) A[dst++] = pb + k;
      base += sm.uniform;
      __syncthreads();
    }
    // 2. stable sort by the feature's code: (code, canonical position) = presorted order
    int32_t* src = A;
    int32_t* dst = B;
    if (stable_digit_pass([&](int i) { return src[i]; }, dst, nv,
                          [&](int p) { return static_cast<int>(cj[p] & 255u); }, sm)) {
      int32_t* t = src;
      src = dst;
      dst = t;
    }
    __syncthreads();
    if (sizeof(CodeT) == 2) {
      if (stable_digit_pass([&](int i) { return src[i]; }, dst, nv,
                            [&](int p) { return static_cast<int>(cj[p] >> 8); }, sm)) {
        int32_t* t = src;
        src = dst;
        dst = t;
      }
      __syncthreads();
    }
    // 3. the fold (warp 0; members in list order, boundaries at code changes)
    if (spec_one) {
      const double L = fold_at(fd.pos0, src, need);
      if (tid == 0) out[wr.best_bin] = L;
    } else if (need >= kExactSpecMin) {
      fold_rec(fd.pos0, src, need, cj, out);
    } else if (warp == 0) {
      double left = 0.0;
      int prev = -1;
      for (int i0 = 0; i0 < need; i0 += 32) {
        const int i = i0 + lane;
        const int p = i < need ? src[i] : 0;
        const int code = i < need ? static_cast<int>(cj[p]) : 0;
        const double rv = i < need ? resid[fd.pos0 + p] : 0.0;
        const int cnt = min(32, need - i0);
        for (int l0 = 0; l0 < cnt; l0 += 8) {
          int cc[8];
          double vv[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            cc[k] = __shfl_sync(0xffffffffu, code, l0 + k);
            vv[k] = __shfl_sync(0xffffffffu, rv, l0 + k);
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            if (l0 + k < cnt) {
              if (prev >= 0 && cc[k] != prev && lane == 0) out[prev] = left;
              left = fs_add(left, vv[k]);
              prev = cc[k];
            }
          }
        }
      }
      if (lane == 0 && prev >= 0) out[prev] = left;  // the last window boundary
    }
    __syncthreads();
  }
}

template <typename CodeT>
__global__ void __launch_bounds__(256) exact_kernel(const FamDesc* __restrict__ fam, NodeRec* __restrict__ nodes,
                                                    const ExactItem* __restrict__ items, const int* __restrict__ n_items,
                                                    int level, int Dp, const CodeT* __restrict__ codes_cm,
                                                    const double* __restrict__ resid, const int32_t* __restrict__ ord,
                                                    const int32_t* __restrict__ ord_cur,
                                                    const int16_t* __restrict__ nodeid,
                                                    const int32_t* __restrict__ rep_boff, double* __restrict__ lbuf,
                                                    const WinRec* __restrict__ win, int nrep_max,
                                                    int level_slots_max, int small_path) {
  FS_PDL_WAIT();
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int total = *n_items;
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < total; w += warps) {
    const ExactItem it = items[w];
    const FamDesc fd = fam[it.fam];
    NodeRec& nd = nodes[fd.node0 + it.slot];
    const int n = nd.n;
    if (it.rep < 0) {
      if (small_path && n >= kExactSpecMin) continue;  // exact_small_kernel: speculative CTA fold
      const double s = warp_fold_gather(resid + fd.pos0, ord_cur + fd.pos0 + nd.seg, n);
      if (lane == 0) nd.total = s;
      continue;
    }
    if (exact_is_small(n, fd.n) && small_path) continue;  // exact_small_kernel folds it
    if (small_path) {
      const WinRec& wr = win[(static_cast<int64_t>(it.fam) * level_slots_max + (it.slot - ((1 << level) - 1))) *
                                 nrep_max + it.rep];
      if (wr.maxlc >= kExactSpecMin) continue;  // exact_small_kernel: CTA fold of the presorted list
    }
    const int jj = it.rep;
    const int32_t* L = ord + fd.ord0 + static_cast<int64_t>(jj) * fd.n;
    const int local = it.slot - ((1 << level) - 1);
    double* out = lbuf + fd.lbuf0 + static_cast<int64_t>(local) * fd.bins + rep_boff[fd.rep0 + jj];
    double left = 0.0;
    int prev = -1, seen = 0, used = 0;
    // candidates past the feature's largest window left count cannot win (costmodel.cpp:65
    // strict >): the fold stops there
    const int need = win[(static_cast<int64_t>(it.fam) * level_slots_max + local) * nrep_max + jj].maxlc;
    // 4 chunks of 32 list entries in flight: index loads, then the dependent gathers
    for (int i0 = 0; i0 < fd.n && seen < need; i0 += 128) {
      int p[4], code[4];
      double rv[4];
      bool mem[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) p[c] = i0 + 32 * c + lane < fd.n ? L[i0 + 32 * c + lane] : -1;
#pragma unroll
      for (int c = 0; c < 4; ++c) mem[c] = p[c] >= 0 && nodeid[fd.pos0 + p[c]] == it.slot;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        code[c] = mem[c] ? static_cast<int>(codes_cm[fd.ord0 + static_cast<int64_t>(jj) * fd.n + p[c]]) : 0;
        rv[c] = mem[c] ? resid[fd.pos0 + p[c]] : 0.0;
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const unsigned m = __ballot_sync(0xffffffffu, mem[c]);
        seen += __popc(m);
        for (int l0 = 0; l0 < 32; l0 += 8) {
          if (!((m >> l0) & 0xFFu)) continue;
          int cc[8];
          double vv[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            cc[k] = __shfl_sync(0xffffffffu, code[c], l0 + k);
            vv[k] = __shfl_sync(0xffffffffu, rv[c], l0 + k);
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            if (((m >> (l0 + k)) & 1u) && used < need) {
              if (prev >= 0 && cc[k] != prev && lane == 0) out[prev] = left;  // boundary after bin `prev`
              left = fs_add(left, vv[k]);
              prev = cc[k];
              ++used;
            }
          }
        }
      }
    }
    if (lane == 0 && prev >= 0 && used == need) out[prev] = left;  // the last window boundary
  }
}

// Reference decision over the exactly folded candidates: gain = ((L*L)/lc + (R*R)/rc) - (T*T)/n,
// R = T - L (costmodel.cpp:58-62), strict > in (feature, threshold) order (:65).
__global__ void exact_decide_kernel(const FamDesc* __restrict__ fam, const FamState* __restrict__ st,
                                    NodeRec* __restrict__ nodes, int level, const int32_t* __restrict__ hcnt,
                                    const int32_t* __restrict__ rep_boff, const int32_t* __restrict__ rep_nb,
                                    const WinRec* __restrict__ win, int nrep_max, int level_slots_max,
                                    const double* __restrict__ lbuf) {
  FS_PDL_WAIT();
  const int f = blockIdx.y;
  const FamDesc fd = fam[f];
  if (!st[f].active) return;
  const int local = blockIdx.x * blockDim.x + threadIdx.x;
  if (local >= (1 << level)) return;
  const int s = (1 << level) - 1 + local;
  NodeRec& nd = nodes[fd.node0 + s];
  if (nd.state != kNodeExact) return;
  const WinRec* w = win + (static_cast<int64_t>(f) * level_slots_max + local) * nrep_max;
  const int n = nd.n;
  const double T = nd.total;
  const double parent = fs_div(fs_mul(T, T), static_cast<double>(n));
  double best = 0.0;
  int bj = -1, bb = -1, blc = 0;
  for (int jj = 0; jj < fd.nrep; ++jj) {
    if (!w[jj].flag) continue;
    const int64_t hb = fd.hist0 + (static_cast<int64_t>(level & 1) * fd.level_slots + local) * fd.bins +
                       rep_boff[fd.rep0 + jj];
    const double* lb = lbuf + fd.lbuf0 + static_cast<int64_t>(local) * fd.bins + rep_boff[fd.rep0 + jj];
    if (w[jj].count == 1) {  // its window candidate is the only one of this feature that can win
      const int cum = w[jj].best_lc, b = w[jj].best_bin;
      const double L = lb[b];
      const double R = fs_sub(T, L);
      const double a = fs_div(fs_mul(L, L), static_cast<double>(cum));
      const double r = fs_div(fs_mul(R, R), static_cast<double>(n - cum));
      const double g = fs_sub(fs_add(a, r), parent);
      if (g > best) {
        best = g;
        bj = jj;
        bb = b;
        blc = cum;
      }
      continue;
    }
    int cum = 0;
    for (int b = 0; b < rep_nb[fd.rep0 + jj]; ++b) {
      const int c = hcnt[hb + b];
      if (!c) continue;
      cum += c;
      if (cum >= n || cum > w[jj].maxlc) break;  // folds stop at the last window candidate
      const double L = lb[b];
      const double R = fs_sub(T, L);
      const double a = fs_div(fs_mul(L, L), static_cast<double>(cum));
      const double r = fs_div(fs_mul(R, R), static_cast<double>(n - cum));
      const double g = fs_sub(fs_add(a, r), parent);
      if (g > best) {
        best = g;
        bj = jj;
        bb = b;
        blc = cum;
      }
    }
  }
  if (bj < 0) {
    nd.state = kNodeLeaf;
  } else {
    nd.state = kNodeSplit;
    nd.rep = bj;
    nd.bin = bb;
    nd.gain = best;
    nd.lc = blc;
  }
}

// Split nodes: exact threshold, tree record, stable partition of the order-0 segment in place
// (costmodel.cpp:94-105 for list 0), row -> child ids, child records.
template <typename CodeT>
__global__ void __launch_bounds__(1024) partition_kernel(
    const FamDesc* __restrict__ fam, const FamState* __restrict__ st, NodeRec* __restrict__ nodes, int level, int Dp,
    const CodeT* __restrict__ codes_cm, int32_t* __restrict__ ord_cur, int32_t* __restrict__ scratch,
    int16_t* __restrict__ nodeid, const int32_t* __restrict__ rep_orig, const int32_t* __restrict__ rep_boff,
    const double* __restrict__ vals, const int32_t* __restrict__ cle, const int32_t* __restrict__ ord,
    const int32_t* __restrict__ canon, const double* __restrict__ x, int d, TreeRec* __restrict__ trees, int slots) {
  FS_PDL_WAIT();
  __shared__ int wsum[32];
  __shared__ int base_l, base_r;
  const int f = blockIdx.y;
  const FamDesc fd = fam[f];
  if (!st[f].active) return;
  const int local = blockIdx.x;
  if (local >= (1 << level)) return;
  const int s = (1 << level) - 1 + local;
  NodeRec& nd = nodes[fd.node0 + s];
  if (nd.state != kNodeSplit) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int jj = nd.rep, bin = nd.bin, n = nd.n, seg = nd.seg, lc = nd.lc;
  TreeRec* tr = trees + fd.tree0 + static_cast<int64_t>(st[f].ntrees) * slots;
  if (tid == 0) {
    const int orig = rep_orig[fd.rep0 + jj];
    double thr = vals[fd.bin0 + rep_boff[fd.rep0 + jj] + bin];
    if (thr == 0.0 && fd.negz) {  // +0.0 and -0.0 share a bin: take the last left element's own value
      const int32_t* L = ord + fd.ord0 + static_cast<int64_t>(jj) * fd.n;
      for (int i = cle[fd.bin0 + rep_boff[fd.rep0 + jj] + bin] - 1; i >= 0; --i) {
        if (nodeid[fd.pos0 + L[i]] == s) {
          thr = x[(fd.row0 + canon[fd.pos0 + L[i]]) * d + orig];
          break;
        }
      }
    }
    TreeRec r;
    r.kind = kNodeSplit;
    r.feature = orig;
    r.threshold = thr;
    r.value = 0.0;
    r.gain = nd.gain;
    r.rep = jj;
    r.bin = bin;
    tr[s] = r;
    base_l = 0;
    base_r = 0;
    NodeRec& a = nodes[fd.node0 + 2 * s + 1];
    NodeRec& b = nodes[fd.node0 + 2 * s + 2];
    a.n = lc;
    a.seg = seg;
    b.n = n - lc;
    b.seg = seg + lc;
  }
  int32_t* src = scratch + fd.pos0 + seg;
  int32_t* dst = ord_cur + fd.pos0 + seg;
  for (int i = tid; i < n; i += blockDim.x) src[i] = dst[i];
  __syncthreads();
  const int16_t cl = static_cast<int16_t>(2 * s + 1), cr = static_cast<int16_t>(2 * s + 2);
  // the next chunk's index and code gathers are issued before this chunk's scan and scatter
  int p_nx = tid < n ? src[tid] : 0;
  int c_nx = tid < n ? static_cast<int>(codes_cm[fd.ord0 + static_cast<int64_t>(jj) * fd.n + p_nx]) : 0;
  for (int t0 = 0; t0 < n; t0 += blockDim.x) {
    const int i = t0 + tid;
    const int p = p_nx;
    const bool left = i < n && c_nx <= bin;
    if (i + static_cast<int>(blockDim.x) < n) {
      p_nx = src[i + blockDim.x];
      c_nx = static_cast<int>(codes_cm[fd.ord0 + static_cast<int64_t>(jj) * fd.n + p_nx]);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, left);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    if (warp == 0) {
      const int v = wsum[lane];
      int incl = v;
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      wsum[lane] = incl - v;
    }
    __syncthreads();
    const int lrank = wsum[warp] + __popc(bal & ((1u << lane) - 1u));
    if (i < n) {
      if (left) {
        dst[base_l + lrank] = p;
        nodeid[fd.pos0 + p] = cl;
      } else {
        dst[lc + base_r + (i - t0) - lrank] = p;
        nodeid[fd.pos0 + p] = cr;
      }
    }
    __syncthreads();  // every thread has used base_l / base_r for this tile
    if (warp == 31 && lane == 0) {  // tile total = warp 31's exclusive prefix + its own count
      const int tile_left = wsum[31] + __popc(bal);
      const int tile = min(static_cast<int>(blockDim.x), n - t0);
      base_l += tile_left;
      base_r += tile - tile_left;
    }
    __syncthreads();
  }
}

// Chunked stable partition (costmodel.cpp:94-105 for list 0) for few large nodes (C4): a CTA per
// (node, 1,024-row chunk) - launched with one CTA per (family, node, chunk) item (the loop then
// runs once; it also serves a persistent grid). Pass 1 counts each chunk's left rows (and copies the chunk's order-0
// entries to scratch); pass 2 offsets each chunk by its predecessors' counts and scatters with a
// block scan - so a 65,536-row root partitions with 64 CTAs instead of one walking 64 tiles.
constexpr int kPartChunk = 1024;

template <typename CodeT>
__global__ void __launch_bounds__(kPartChunk) partition_count_kernel(
    const FamDesc* __restrict__ fam, const FamState* __restrict__ st, NodeRec* __restrict__ nodes, int level,
    int Dp, const CodeT* __restrict__ codes_cm, const int32_t* __restrict__ ord_cur, int32_t* __restrict__ scratch,
    const int16_t* __restrict__ nodeid, const int32_t* __restrict__ rep_orig, const int32_t* __restrict__ rep_boff,
    const double* __restrict__ vals, const int32_t* __restrict__ cle, const int32_t* __restrict__ ord,
    const int32_t* __restrict__ canon, const double* __restrict__ x, int d, TreeRec* __restrict__ trees, int slots,
    int32_t* __restrict__ part_cnt, int chunks_max, int level_slots_max, int F) {
  FS_PDL_WAIT();
  __shared__ int wsum[32];
  const int nl = 1 << level;
  const int64_t items = static_cast<int64_t>(F) * nl * chunks_max;  // (family, node, chunk)
  for (int64_t w = blockIdx.x; w < items; w += gridDim.x) {
  const int f = static_cast<int>(w / (static_cast<int64_t>(nl) * chunks_max));
  const int local = static_cast<int>((w / chunks_max) % nl);
  const int c = static_cast<int>(w % chunks_max);
  const FamDesc fd = fam[f];
  if (!st[f].active) continue;
  const int s = nl - 1 + local;
  const NodeRec& nd = nodes[fd.node0 + s];
  if (nd.state != kNodeSplit) continue;
  const int r0 = c * kPartChunk;
  const int jj = nd.rep, bin = nd.bin, n = nd.n, seg = nd.seg, lc = nd.lc;
  if (r0 >= nd.n) continue;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // (before any row moves: the -0.0 threshold lookup reads the parent's node ids)
  if (c == 0 && tid == 0) {  // exact threshold, tree record, child records
    const int orig = rep_orig[fd.rep0 + jj];
    double thr = vals[fd.bin0 + rep_boff[fd.rep0 + jj] + bin];
    if (thr == 0.0 && fd.negz) {  // +0.0 and -0.0 share a bin: take the last left element's own value
      const int32_t* L = ord + fd.ord0 + static_cast<int64_t>(jj) * fd.n;
      for (int i = cle[fd.bin0 + rep_boff[fd.rep0 + jj] + bin] - 1; i >= 0; --i) {
        if (nodeid[fd.pos0 + L[i]] == s) {
          thr = x[(fd.row0 + canon[fd.pos0 + L[i]]) * d + orig];
          break;
        }
      }
    }
    TreeRec r;
    r.kind = kNodeSplit;
    r.feature = orig;
    r.threshold = thr;
    r.value = 0.0;
    r.gain = nd.gain;
    r.rep = jj;
    r.bin = bin;
    trees[fd.tree0 + static_cast<int64_t>(st[f].ntrees) * slots + s] = r;
    NodeRec& a = nodes[fd.node0 + 2 * s + 1];
    NodeRec& b = nodes[fd.node0 + 2 * s + 2];
    a.n = lc;
    a.seg = seg;
    b.n = n - lc;
    b.seg = seg + lc;
  }

  const int i = r0 + tid;
  bool left = false;
  if (i < nd.n) {
    const int p = ord_cur[fd.pos0 + nd.seg + i];
    scratch[fd.pos0 + nd.seg + i] = p;
    left = static_cast<int>(codes_cm[fd.ord0 + static_cast<int64_t>(nd.rep) * fd.n + p]) <= nd.bin;
  }
  const unsigned bal = __ballot_sync(0xffffffffu, left);
  if (lane == 0) wsum[warp] = __popc(bal);
  __syncthreads();
  if (warp == 0) {
    int v = lane < static_cast<int>(blockDim.x >> 5) ? wsum[lane] : 0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) part_cnt[(static_cast<int64_t>(f) * level_slots_max + local) * chunks_max + c] = v;
  }
  __syncthreads();  // wsum is reused by the next item
  }
}

template <typename CodeT>
__global__ void __launch_bounds__(kPartChunk) partition_scatter_kernel(
    const FamDesc* __restrict__ fam, const FamState* __restrict__ st, NodeRec* __restrict__ nodes, int level, int Dp,
    const CodeT* __restrict__ codes_cm, int32_t* __restrict__ ord_cur, const int32_t* __restrict__ scratch,
    int16_t* __restrict__ nodeid, const int32_t* __restrict__ part_cnt, int chunks_max, int level_slots_max, int F) {
  FS_PDL_WAIT();
  __shared__ int wsum[32];
  __shared__ int s_off;
  const int nl = 1 << level;
  const int64_t items = static_cast<int64_t>(F) * nl * chunks_max;  // (family, node, chunk)
  for (int64_t w = blockIdx.x; w < items; w += gridDim.x) {
  const int f = static_cast<int>(w / (static_cast<int64_t>(nl) * chunks_max));
  const int local = static_cast<int>((w / chunks_max) % nl);
  const int c = static_cast<int>(w % chunks_max);
  const FamDesc fd = fam[f];
  if (!st[f].active) continue;
  const int s = nl - 1 + local;
  NodeRec& nd = nodes[fd.node0 + s];
  if (nd.state != kNodeSplit) continue;
  const int r0 = c * kPartChunk;
  const int jj = nd.rep, bin = nd.bin, n = nd.n, seg = nd.seg, lc = nd.lc;
  if (r0 >= n) continue;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (warp == 0) {  // left rows of the preceding chunks
    const int32_t* cnt = part_cnt + (static_cast<int64_t>(f) * level_slots_max + local) * chunks_max;
    int v = 0;
    for (int k = lane; k < c; k += 32) v += cnt[k];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) s_off = v;
  }
  const int i = r0 + tid;
  int p = 0;
  bool left = false;
  if (i < n) {
    p = scratch[fd.pos0 + seg + i];
    left = static_cast<int>(codes_cm[fd.ord0 + static_cast<int64_t>(jj) * fd.n + p]) <= bin;
  }
  const unsigned bal = __ballot_sync(0xffffffffu, left);
  if (lane == 0) wsum[warp] = __popc(bal);
  __syncthreads();
  if (warp == 0) {
    const int v = lane < static_cast<int>(blockDim.x >> 5) ? wsum[lane] : 0;
    int incl = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    wsum[lane] = incl - v;
  }
  __syncthreads();
  if (i < n) {
    const int lrank = wsum[warp] + __popc(bal & ((1u << lane) - 1u));
    int32_t* dst = ord_cur + fd.pos0 + seg;
    const int off_l = s_off, off_r = r0 - s_off;
    if (left) {
      dst[off_l + lrank] = p;
      nodeid[fd.pos0 + p] = static_cast<int16_t>(2 * s + 1);
    } else {
      dst[lc + off_r + (i - r0) - lrank] = p;
      nodeid[fd.pos0 + p] = static_cast<int16_t>(2 * s + 2);
    }
  }
  __syncthreads();  // wsum / s_off are reused by the next item
  }
}

#ifndef FS_LEAF_EST_MIN
#define FS_LEAF_EST_MIN 384
#endif
constexpr int kLeafEstMin = FS_LEAF_EST_MIN;   // leaf chains from this length fold through cta_fold_est (fold_est.cuh)
constexpr int kLeafThreads = 256;  // leaf CTA (1,024 threads with four speculated segments measured slower: C5 leaves 0.59 -> 0.82 s)
// Leaves (costmodel.cpp:85-91): a CTA per (family, heap slot) - value = reference-order fold of
// the leaf's order-0 segment / n (cta_fold_est), then pred += lr*value over its rows.
__global__ void __launch_bounds__(kLeafThreads) leaf_cta_kernel(const FamDesc* __restrict__ fam, int F,
                                                       const FamState* __restrict__ st, NodeRec* __restrict__ nodes,
                                                       int slots, const int32_t* __restrict__ ord_cur,
                                                       const double* __restrict__ resid, double* __restrict__ pred,
                                                       TreeRec* __restrict__ trees, const double* __restrict__ target_c,
                                                       double* __restrict__ ebuf, int K, int64_t n_tot) {
  FS_PDL_WAIT();
  __shared__ __align__(16) double stage[fold_est_stage_doubles(kLeafThreads)];
  __shared__ double fscr[fold_est_scratch_doubles(kLeafThreads)];
  const int f = blockIdx.y, s = blockIdx.x;
  if (f >= F) return;
  const FamDesc fd = fam[f];
  if (!st[f].active) return;
  NodeRec& nd = nodes[fd.node0 + s];
  if (nd.state != kNodeLeaf || nd.n == 0) return;
  if (s > 0 && nodes[fd.node0 + ((s - 1) >> 1)].state != kNodeSplit) return;
  const int n = nd.n;
  const int32_t* L = ord_cur + fd.pos0 + nd.seg;
  double sum;
  if (nd.pad_) {
    sum = nd.total;
  } else if (n < kLeafEstMin) {  // short chain: warp 0
    if (threadIdx.x < 32) {
      const double t = warp_fold_gather(resid + fd.pos0, L, n);
      if (threadIdx.x == 0) fscr[0] = t;
    }
    __syncthreads();
    sum = fscr[0];
  } else {
    sum = cta_fold_est<16>(resid + fd.pos0, L, n, 0.0, stage, fscr);
  }
  const double value = fs_div(sum, static_cast<double>(n));
  const double step = fs_mul(fd.lr, value);
  // the round commits unless the tree is a single leaf of value exactly 0 (round_commits); then
  // e = target - prediction of each row goes to the MSE ring slot of this round (mse_stash)
  const bool commits = !(s == 0 && value == 0.0);
  double* eb = ebuf + static_cast<int64_t>(st[f].ntrees % K) * n_tot;
  // prediction update, 8 rows per thread in flight (index and prediction gathers issued before
  // the stores: the compiler cannot prove the arrays do not alias)
  for (int i0 = 0; i0 < n; i0 += 8 * static_cast<int>(blockDim.x)) {
    int64_t pp[8];
    double pv[8], tv[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = i0 + k * blockDim.x + threadIdx.x;
      pp[k] = i < n ? fd.pos0 + L[i] : -1;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      pv[k] = pp[k] >= 0 ? pred[pp[k]] : 0.0;
      tv[k] = pp[k] >= 0 ? target_c[pp[k]] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (pp[k] >= 0) {
        const double np = fs_add(pv[k], step);
        pred[pp[k]] = np;
        if (commits) eb[pp[k]] = fs_sub(tv[k], np);  // this round's MSE term (costmodel.cpp:215-220)
      }
  }
  if (threadIdx.x == 0) {
    nd.value = value;
    TreeRec r;
    r.kind = kNodeLeaf;
    r.feature = -1;
    r.threshold = 0.0;
    r.value = value;
    r.gain = 0.0;
    r.rep = -1;
    r.bin = 0;
    trees[fd.tree0 + static_cast<int64_t>(st[f].ntrees) * slots + s] = r;
  }
}


// Commit the round's tree or stop (costmodel.cpp:212), then train_mse_by_round (:215-220).
// The reference folds e*e over the canonical rows sequentially, and so does mse_fold_kernel -
// but off the round's critical path: every committed round stashes its e = target - pred (the
// next round's residual) in a ring of K rounds, and every K rounds one launch folds all
// (family, round) chains of the ring at once, one thread per chain, in canonical order.
#ifndef FS_EXACT_SMALL_CTAS
#define FS_EXACT_SMALL_CTAS 64
#endif
constexpr int kExactSmallCtas = FS_EXACT_SMALL_CTAS;  // CTAs of exact_small_kernel (items loop over them)
__device__ __forceinline__ bool round_commits(const FamDesc& fd, const FamState& st, const NodeRec* nodes) {
  if (!st.active) return false;
  const NodeRec& root = nodes[fd.node0];
  return !(root.state == kNodeLeaf && root.value == 0.0);
}
__global__ void commit_kernel(const FamDesc* __restrict__ fam, FamState* __restrict__ st,
                              const NodeRec* __restrict__ nodes, int F) {
  FS_PDL_WAIT();
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  const FamDesc fd = fam[f];
  if (!st[f].active) return;
  if (!round_commits(fd, st[f], nodes)) {
    st[f].active = 0;  // single leaf of value exactly 0: the reference stops boosting
    return;
  }
  const int t = st[f].ntrees;
  st[f].ntrees = t + 1;
  if (t + 1 >= fd.trees) st[f].active = 0;
}

}  // namespace

// mse[f][t] = (sum over canonical rows p, in order, of e*e) / n (costmodel.cpp:215-220) for
// every committed round t in [t_lo, t_hi) of every family: one WARP per (family, round) chain -
// the warp loads 128 consecutive e's at a time (coalesced, the next 128 in flight), squares them
// in parallel, and adds the squares in row order (shuffled to every lane; every add separately
// rounded, so the chain is the reference's). Round t's e of family f sits at
//   ring   (ring_stride > 0): ebuf[(t % K) * ring_stride + pos0 + p]
//   blocks (ring_stride = 0): ebuf[pos0 * K + (t % K) * n + p]   (K = all rounds, resident fit)
__global__ void mse_fold_kernel(const FamDesc* __restrict__ fam, const FamState* __restrict__ st, int F,
                                const double* __restrict__ ebuf, int K, int64_t ring_stride, int t_lo, int t_hi,
                                double* __restrict__ mse, int max_trees) {
  FS_PDL_WAIT();
  const int W = t_hi - t_lo;
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (W <= 0 || w >= static_cast<int64_t>(F) * W) return;
  const int f = static_cast<int>(w / W), t = t_lo + static_cast<int>(w % W);
  const FamDesc fd = fam[f];
  if (t >= st[f].ntrees || fd.n <= 0) return;
  const int n = fd.n;
  const double* e = ring_stride > 0 ? ebuf + static_cast<int64_t>(t % K) * ring_stride + fd.pos0
                                    : ebuf + fd.pos0 * K + static_cast<int64_t>(t % K) * n;
  double x[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int i = 32 * c + lane;
    x[c] = i < n ? e[i] : 0.0;
  }
  double s = 0.0;
  for (int i0 = 0; i0 < n; i0 += 128) {
    double y[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = i0 + 128 + 32 * c + lane;
      y[c] = i < n ? e[i] : 0.0;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int base = i0 + 32 * c;
      if (base >= n) break;
      const double sq = fs_mul(x[c], x[c]);
      const int m = min(32, n - base);
      if (m == 32) {
#pragma unroll
        for (int l0 = 0; l0 < 32; l0 += 8) {
          double q[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) q[k] = __shfl_sync(0xffffffffu, sq, l0 + k);
#pragma unroll
          for (int k = 0; k < 8; ++k) s = fs_add(s, q[k]);
        }
      } else {
        for (int l = 0; l < m; ++l) s = fs_add(s, __shfl_sync(0xffffffffu, sq, l));
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) x[c] = y[c];
  }
  if (lane == 0) mse[static_cast<int64_t>(f) * max_trees + t] = fs_div(s, static_cast<double>(n));
}

namespace {
}  // namespace
}  // namespace fit
}  // namespace fs
