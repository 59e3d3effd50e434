// K2 tile binning: build_tiles (gsmesh/splat/tiles.py:35-69).
//
// The reference orders tile entries with np.lexsort((kept, depth, tile))
// (tiles.py:65).  Here, with every count kept on the device (one CUDA-graph
// capturable chain of PDL launches):
//   1. compact the visible rows (count > 0) in row order (chained scan),
//      with the min / max of their depth keys; preprocess has already added
//      each row's tile rectangle into 16 privatised 2D difference grids
//   2. tile_counts: per-tile entry counts = 2D prefix sums of those grids;
//      their exclusive scan is the CSR tile_starts, K and the overflow flag
//                                                                 (1 CTA)
//   3. depth order: the fp64 depth bit patterns (positive doubles order like
//      their bits) are remapped to 24-bit keys over [min, max] (digit
//      histograms in the same pass), sorted stably by 3 onesweep LSD passes
//      (sort.cuh), and every run of equal truncated keys is re-ordered by the
//      full 64-bit key -> visible rows in (depth, row) order, exactly
//   4. two-level rectangle binning (tile grids of up to 512 4x4 super-tiles,
//      i.e. 1080p; larger grids use 8x8 super-tiles split into four 4x4
//      fine CTAs): the depth-ordered rows are flattened into (row,
//      super-tile) pairs, partitioned evenly over warps; count / scan /
//      scatter build each super-tile's coarse list in depth order (staged in
//      shared memory for coalesced writes); fine_bin_kernel expands every
//      coarse entry into its tiles of the super-tile (16-bit masks, ballots
//      in order) straight into the final (tile, depth, row) order == the
//      reference's lexsort, with no entry-level sort at all
//   Larger tile grids: exclusive scan of the rows' tile counts in depth
//      order, emission of (tile id, row) pairs, stable LSD sort by tile id.
// On overflow (K > capacity) the scatter / fine kernels and every consumer
// of the bins skip their work; the caller grows the buffer and re-runs.
#include "sort.cuh"

#ifndef HGS_FIXUP_V2
#define HGS_FIXUP_V2 1
#endif
#ifndef HGS_PREP_3K
#define HGS_PREP_3K 0
#endif

namespace hgs {

// Order-preserving compaction of the visible rows' sort keys (chained scan).
// Each thread owns 16 consecutive keys, loaded as 8 x 16 B vectors.
__global__ void __launch_bounds__(SCAN_THREADS) compact_kernel(const uint64_t* __restrict__ keys, int64_t n,
                                                               uint64_t* dkeys, uint32_t* dvals, uint64_t* status,
                                                               uint32_t* part_ctr, int64_t* counters,
                                                               unsigned long long* minmax) {
  pdl_enter();
  __shared__ int s_part;
  unsigned long long nmin = 0, kmax = 0;  // max of ~key (== ~min key) and max key over visible rows
  const int nparts = (int)((n + SCAN_TILE - 1) / SCAN_TILE);
  while (true) {
    if (threadIdx.x == 0) s_part = (int)atomicAdd(part_ctr, 1u);
    __syncthreads();
    const int part = s_part;
    __syncthreads();
    if (part >= nparts) break;
    const int64_t base = (int64_t)part * SCAN_TILE + (int64_t)threadIdx.x * SCAN_IPT;
    uint64_t k[SCAN_IPT];
    if (base + SCAN_IPT <= n) {
#pragma unroll
      for (int j = 0; j < SCAN_IPT; j += 2) {
        const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(keys + base + j));
        k[j] = v.x;
        k[j + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < SCAN_IPT; j++) k[j] = base + j < n ? keys[base + j] : ~0ull;
    }
    uint64_t excl[SCAN_IPT];
    uint64_t total;
    chained_scan_partition(part, n, [&](int64_t i) -> uint64_t { return k[i - base] != ~0ull ? 1ull : 0ull; },
                           status, excl, total);
#pragma unroll
    for (int j = 0; j < SCAN_IPT; j++) {
      if (k[j] != ~0ull) {
        dkeys[excl[j]] = k[j];
        dvals[excl[j]] = (uint32_t)(base + j);
        nmin = max(nmin, (unsigned long long)~k[j]);
        kmax = max(kmax, (unsigned long long)k[j]);
      }
    }
    if (part == nparts - 1 && threadIdx.x == 0) counters[0] = (int64_t)total;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    nmin = max(nmin, __shfl_xor_sync(0xffffffffu, nmin, o));
    kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
  }
  if ((threadIdx.x & 31) == 0 && kmax) {
    atomicMax(&minmax[0], nmin);
    atomicMax(&minmax[1], kmax);
  }
}

// Depth keys -> DEPTH_KEY_BITS bits, order preserving: (bits - min) >> shift, where
// shift drops the low bits the visible range does not need.  Equal 32-bit
// keys from distinct fp64 depths are re-ordered exactly by depth_fixup_kernel.
// Depth keys are sorted on DEPTH_KEY_BITS bits (3 LSD passes); the exact
// order of keys that collide after the shift is restored by
// depth_fixup_kernel (1M keys: ~1e4 short runs).
constexpr int DEPTH_KEY_BITS = 24;
constexpr uint32_t KEY_CULLED = (1u << DEPTH_KEY_BITS) - 1;
// Depth-order front end (hgs_build_tiles step 3):
//  0: compact_kernel (chained-scan compaction of the visible rows), remap
//  1: no compaction -- every row's key is sorted, the culled rows (key ~0)
//     under the reserved largest 24-bit key, i.e. behind the M visible rows
//  2: compaction fused into the remap: depth_stats_kernel counts each
//     partition's visible rows (and M, the key range), the remap places a
//     partition's visible keys after its predecessors' (one read of their
//     counts) -- no look-back chain, no culled keys in the sort
#ifndef HGS_DEPTH_MODE
#define HGS_DEPTH_MODE 2
#endif
#define HGS_SORT_ALL (HGS_DEPTH_MODE == 1)
// depth sort partition (radix_pass_kernel<uint32_t, 8>: 256 threads x 8 keys)
#ifndef HGS_RS_DEPTH_IPT
#define HGS_RS_DEPTH_IPT 8
#endif
constexpr int RS_DEPTH_IPT = HGS_RS_DEPTH_IPT;
constexpr int RS_PART = RS_THREADS * RS_DEPTH_IPT;
constexpr int RS_KPT = RS_PART / 256;  // keys per thread of the 256-thread stats / compaction kernels
// HGS_SORT_RTS=1: reduce-then-scan depth passes (every pass counts the next
// pass's per-partition digits as it scatters; a scan kernel turns them into
// offsets) instead of the onesweep decoupled look-back
#ifndef HGS_SORT_RTS
#define HGS_SORT_RTS 1
#endif
// Modes 1 / 2: M and the min / max of the visible keys (what the compaction
// gathered on the side), per partition of RS_PART rows; mode 2 also stores
// each partition's visible count (vis_cnt).
__global__ void __launch_bounds__(256) depth_stats_kernel(const uint64_t* __restrict__ keys, int64_t n,
                                                          int64_t* counters, unsigned long long* minmax,
                                                          uint32_t* __restrict__ vis_cnt) {
  pdl_enter();
  __shared__ unsigned long long s_min[8], s_max[8];
  __shared__ uint32_t s_cnt[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long nmin = 0, kmax = 0;
  long long total = 0;
  const int64_t nparts = (n + RS_PART - 1) / RS_PART;
  for (int64_t part = blockIdx.x; part < nparts; part += gridDim.x) {
    const int64_t base = part * RS_PART + (int64_t)threadIdx.x * RS_KPT;  // RS_KPT consecutive keys per thread
    uint32_t cnt = 0;
#pragma unroll
    for (int j = 0; j < RS_KPT; j += 2) {
      uint64_t k0 = ~0ull, k1 = ~0ull;
      if (base + j + 1 < n) {
        const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(keys + base + j));
        k0 = v.x, k1 = v.y;
      } else if (base + j < n) {
        k0 = keys[base + j];
      }
      if (k0 != ~0ull) { nmin = max(nmin, (unsigned long long)~k0); kmax = max(kmax, (unsigned long long)k0); cnt++; }
      if (k1 != ~0ull) { nmin = max(nmin, (unsigned long long)~k1); kmax = max(kmax, (unsigned long long)k1); cnt++; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) s_cnt[warp] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t c = 0;
      for (int w = 0; w < 8; w++) c += s_cnt[w];
      if (vis_cnt) vis_cnt[part] = c;
      total += c;
    }
    __syncthreads();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    nmin = max(nmin, __shfl_xor_sync(0xffffffffu, nmin, o));
    kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
  }
  if (lane == 0) s_min[warp] = nmin, s_max[warp] = kmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; w++) nmin = max(nmin, s_min[w]), kmax = max(kmax, s_max[w]);
    if (total) {
      atomicMax(&minmax[0], nmin);
      atomicMax(&minmax[1], kmax);
      atomicAdd((unsigned long long*)&counters[0], (unsigned long long)total);
    }
  }
}

__device__ __forceinline__ int depth_shift(const unsigned long long* minmax) {
  const unsigned long long lo = ~minmax[0], hi = minmax[1];
  const unsigned long long range = hi > lo ? hi - lo : 0;
  const int bits = range ? 64 - __clzll((long long)range) : 0;
  int sh = bits > DEPTH_KEY_BITS ? bits - DEPTH_KEY_BITS : 0;
  if (HGS_SORT_ALL && (range >> sh) >= KEY_CULLED) sh++;  // the top key is reserved for culled rows
  return sh;
}

// ... and the digit histograms of the remapped keys for the LSD passes
// (hist: DEPTH_KEY_BITS / 8 x 256, zeroed), in the same read.
__global__ void __launch_bounds__(256) depth_remap_kernel(const uint64_t* __restrict__ keys, const int64_t* counters,
                                                          const unsigned long long* __restrict__ minmax,
                                                          uint32_t* __restrict__ k32, uint32_t* __restrict__ hist,
                                                          uint32_t* __restrict__ pcnt0, int64_t nkeys) {
  pdl_enter();
  constexpr int NP = DEPTH_KEY_BITS / 8;
  __shared__ uint32_t sh_h[NP][256];
  for (int i = threadIdx.x; i < NP * 256; i += blockDim.x) (&sh_h[0][0])[i] = 0;
  __shared__ uint32_t sh_part[256];
  __syncthreads();
  // nkeys >= 0 (HGS_SORT_ALL): every row's key, culled rows (~0) -> the
  // reserved key KEY_CULLED (depth_shift keeps the visible ones below it)
  const int64_t m = nkeys >= 0 ? nkeys : counters[0];
  const unsigned long long lo = ~minmax[0];
  const int sh = depth_shift(minmax);
  auto remap = [&](uint64_t key) -> uint32_t {
    return (nkeys >= 0 && key == ~0ull) ? KEY_CULLED : (uint32_t)((key - lo) >> sh);
  };
  if (pcnt0) {
    // reduce-then-scan sort: also the first pass's per-partition digit counts
    // (partitions of RS_PART keys, one per CTA iteration)
    const int64_t nparts = (m + RS_PART - 1) / RS_PART;
    for (int64_t part = blockIdx.x; part < nparts; part += gridDim.x) {
      sh_part[threadIdx.x] = 0;
      __syncthreads();
#pragma unroll
      for (int u = 0; u < RS_PART / 256; u++) {
        const int64_t j = part * RS_PART + u * 256 + threadIdx.x;
        if (j < m) {
          const uint32_t k = remap(keys[j]);
          k32[j] = k;
#pragma unroll
          for (int p = 0; p < NP; p++) atomicAdd(&sh_h[p][(k >> (8 * p)) & 255u], 1u);
          atomicAdd(&sh_part[k & 255u], 1u);
        }
      }
      __syncthreads();
      pcnt0[part * RADIX + threadIdx.x] = sh_part[threadIdx.x];
      __syncthreads();
    }
  } else {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
      const uint32_t k = remap(keys[j]);
      k32[j] = k;
#pragma unroll
      for (int p = 0; p < NP; p++) atomicAdd(&sh_h[p][(k >> (8 * p)) & 255u], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NP * 256; i += blockDim.x) {
    const uint32_t c = (&sh_h[0][0])[i];
    if (c) atomicAdd(&hist[i], c);
  }
}

// Mode 2: the compaction fused into the remap.  One CTA per partition of
// RS_PART rows (RS_KPT consecutive per thread): the visible rows before it are the
// sum of its predecessors' counts (depth_stats_kernel), its own are ranked
// by a block scan, staged in shared memory and written out contiguously --
// the remapped key and the row -- together with the digit histograms and
// the first sort pass's per-partition digit counts (the partition's output
// range spans at most two sort partitions: counted in shared memory).
__global__ void __launch_bounds__(256) depth_compact_remap_kernel(
    const uint64_t* __restrict__ keys, int64_t n, const unsigned long long* __restrict__ minmax,
    const uint32_t* __restrict__ vis_cnt, uint32_t* __restrict__ k32, uint32_t* __restrict__ rows,
    uint32_t* __restrict__ hist, uint32_t* __restrict__ pcnt0) {
  pdl_enter();
  constexpr int NP = DEPTH_KEY_BITS / 8;
  __shared__ uint32_t sh_h[NP][256];
  __shared__ uint32_t sh_p[2][256];
  __shared__ uint32_t s_k[RS_PART], s_r[RS_PART];
  __shared__ uint32_t s_warp[8];
  for (int i = threadIdx.x; i < NP * 256; i += blockDim.x) (&sh_h[0][0])[i] = 0;
  const unsigned long long lo = ~minmax[0];
  const int sh = depth_shift(minmax);
  const int64_t nparts = (n + RS_PART - 1) / RS_PART;
  for (int64_t part = blockIdx.x; part < nparts; part += gridDim.x) {
    uint32_t pre = 0;  // visible rows in the earlier partitions
    for (int64_t q = threadIdx.x; q < part; q += blockDim.x) pre += vis_cnt[q];
    sh_p[0][threadIdx.x] = sh_p[1][threadIdx.x] = 0;
    const int64_t base = part * RS_PART + (int64_t)threadIdx.x * RS_KPT;
    uint64_t kk[RS_KPT];
#pragma unroll
    for (int j = 0; j < RS_KPT; j += 2) {
      if (base + j + 1 < n) {
        const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(keys + base + j));
        kk[j] = v.x, kk[j + 1] = v.y;
      } else {
        kk[j] = base + j < n ? keys[base + j] : ~0ull;
        kk[j + 1] = ~0ull;
      }
    }
    uint32_t cnt = 0;
#pragma unroll
    for (int j = 0; j < RS_KPT; j++) cnt += kk[j] != ~0ull;
    uint32_t tot_pre;
    pre = block_exclusive_scan<uint32_t>(pre, s_warp, tot_pre);  // (only the total is used)
    pre = tot_pre;
    uint32_t tot;
    uint32_t r = block_exclusive_scan<uint32_t>(cnt, s_warp, tot);
    const uint32_t p0 = pre / RS_PART;  // first sort partition of this output range
#pragma unroll
    for (int j = 0; j < RS_KPT; j++) {
      if (kk[j] == ~0ull) continue;
      const uint32_t k = (uint32_t)((kk[j] - lo) >> sh);
      s_k[r] = k;
      s_r[r] = (uint32_t)(base + j);
#pragma unroll
      for (int p = 0; p < NP; p++) atomicAdd(&sh_h[p][(k >> (8 * p)) & 255u], 1u);
      atomicAdd(&sh_p[(pre + r) / RS_PART - p0][k & 255u], 1u);
      r++;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < tot; i += blockDim.x) {
      k32[pre + i] = s_k[i];
      rows[pre + i] = s_r[i];
    }
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const uint32_t c = sh_p[h][threadIdx.x];
      if (c) atomicAdd(&pcnt0[(size_t)(p0 + h) * RADIX + threadIdx.x], c);
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < NP * 256; i += blockDim.x) {
    const uint32_t c = (&sh_h[0][0])[i];
    if (c) atomicAdd(&hist[i], c);
  }
}

// After the stable 32-bit sort, rows with equal truncated keys are in row
// order; the reference order is (fp64 depth, row): re-sort each such run by
// the full 64-bit depth key (runs are rare and short; long runs of exactly
// equal depths are already ordered and only verified).  One CTA per chunk of
// FIX_CHUNK sorted positions: the chunk's keys are staged in shared memory,
// its run starts listed, then one thread per run: runs of up to FIX_SHORT
// rows are loaded at once (rows, then their full keys) and sorted in
// registers, longer ones by a Shell sort in place.
constexpr int FIX_CHUNK = 2048, FIX_SHORT = 8;
__global__ void __launch_bounds__(256) depth_fixup_kernel(const uint32_t* __restrict__ k32, uint32_t* __restrict__ rows,
                                                          const uint64_t* __restrict__ sort_keys, const int64_t* counters,
                                                          const unsigned long long* __restrict__ minmax) {
  pdl_enter();
  __shared__ uint32_t sk[FIX_CHUNK + 2];  // [0]: the key before the chunk, [FIX_CHUNK + 1]: the one after
  __shared__ int s_run[FIX_CHUNK / 2];     // run starts of the chunk (chunk offsets)
  __shared__ int s_nrun;
  const int64_t m = counters[0];
  if (depth_shift(minmax) == 0) return;  // keys were exact
  // full keys by row from the 8-byte sort_keys array (the fp64 depth bit
  // pattern preprocess wrote; L2-resident) rather than the 80-byte records
  auto key64 = [&](uint32_t row) { return (unsigned long long)__ldg(sort_keys + row); };
  for (int64_t base = (int64_t)blockIdx.x * FIX_CHUNK; base < m; base += (int64_t)gridDim.x * FIX_CHUNK) {
    if (threadIdx.x == 0) s_nrun = 0;
    for (int i = threadIdx.x; i < FIX_CHUNK + 2; i += blockDim.x) {
      const int64_t j = base + i - 1;
      sk[i] = (j >= 0 && j < m) ? __ldcg(k32 + j) : 0u;
    }
    __syncthreads();
    // the chunk's run starts first, so that the runs are then handled in
    // parallel (one thread each) rather than one position stride at a time
    for (int i = threadIdx.x; i < FIX_CHUNK; i += blockDim.x) {
      const int64_t j = base + i;
      if (j >= m) break;
      const uint32_t kj = sk[i + 1];
      if (j > 0 && sk[i] == kj) continue;            // not a run start
      if (j + 1 >= m || sk[i + 2] != kj) continue;   // singleton
      s_run[atomicAdd(&s_nrun, 1)] = i;
    }
    __syncthreads();
#pragma unroll 1
    for (int ri = threadIdx.x; ri < s_nrun; ri += blockDim.x) {
      const int i = s_run[ri];
      const int64_t j = base + i;
      const uint32_t kj = sk[i + 1];
      int64_t e = j + 1;
      while (e < m && (e - base + 1 <= FIX_CHUNK ? sk[e - base + 1] : __ldcg(k32 + e)) == kj) e++;
      const int64_t len = e - j;
      if (len <= FIX_SHORT) {
        uint32_t r[FIX_SHORT];
        unsigned long long kk[FIX_SHORT];
#pragma unroll
        for (int t = 0; t < FIX_SHORT; t++) r[t] = t < len ? rows[j + t] : 0xffffffffu;
#pragma unroll
        for (int t = 0; t < FIX_SHORT; t++) kk[t] = t < len ? key64(r[t]) : ~0ull;
        bool sorted = true;
#pragma unroll
        for (int t = 1; t < FIX_SHORT; t++) sorted = sorted && (kk[t - 1] < kk[t] || (kk[t - 1] == kk[t] && r[t - 1] < r[t]));
        if (sorted) continue;
        // odd-even transposition sort by (key, row); padding (~0, ~0) stays last
#pragma unroll
        for (int rd = 0; rd < FIX_SHORT; rd++)
#pragma unroll
          for (int t = rd & 1; t + 1 < FIX_SHORT; t += 2) {
            const bool sw = kk[t] > kk[t + 1] || (kk[t] == kk[t + 1] && r[t] > r[t + 1]);
            const unsigned long long ka = sw ? kk[t + 1] : kk[t], kb = sw ? kk[t] : kk[t + 1];
            const uint32_t ra = sw ? r[t + 1] : r[t], rb = sw ? r[t] : r[t + 1];
            kk[t] = ka, kk[t + 1] = kb, r[t] = ra, r[t + 1] = rb;
          }
#pragma unroll
        for (int t = 0; t < FIX_SHORT; t++)
          if (t < len) rows[j + t] = r[t];
        continue;
      }
      bool sorted = true;
      for (int64_t t = j + 1; t < e && sorted; t++) {
        const unsigned long long a = key64(rows[t - 1]), b = key64(rows[t]);
        sorted = a < b || (a == b && rows[t - 1] < rows[t]);
      }
      if (sorted) continue;
      // Shell sort by (key64, row): correct for any run length
      for (int64_t gap = len / 2; gap > 0; gap /= 2)
        for (int64_t t = j + gap; t < e; t++) {
          const uint32_t rr = rows[t];
          const unsigned long long kr = key64(rr);
          int64_t u = t;
          while (u >= j + gap) {
            const uint32_t ru = rows[u - gap];
            const unsigned long long ku = key64(ru);
            if (ku < kr || (ku == kr && ru < rr)) break;
            rows[u] = ru;
            u -= gap;
          }
          rows[u] = rr;
        }
    }
    __syncthreads();
  }
}

#if !HGS_FIXUP_V2
// round-1 fix-up (A/B baseline): one thread per sorted position
// After the stable 32-bit sort, rows with equal truncated keys are in row
// order; the reference order is (fp64 depth, row): re-sort each such run by
// the full 64-bit depth key (runs are rare and short; long runs of exactly
// equal depths are already ordered and only verified).
__global__ void __launch_bounds__(256) depth_fixup_v1_kernel(const uint32_t* __restrict__ k32, uint32_t* __restrict__ rows,
                                                          const uint64_t* __restrict__ sort_keys, const int64_t* counters,
                                                          const unsigned long long* __restrict__ minmax) {
  pdl_enter();
  const int64_t m = counters[0];
  if (depth_shift(minmax) == 0) return;  // keys were exact
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t kj = k32[j];
    if (j > 0 && k32[j - 1] == kj) continue;        // not a run start
    if (j + 1 >= m || k32[j + 1] != kj) continue;   // singleton
    int64_t e = j + 1;
    while (e < m && k32[e] == kj) e++;
    // full keys by row from the 8-byte sort_keys array (the fp64 depth bit
    // pattern preprocess wrote; L2-resident) rather than the 80-byte records
    auto key64 = [&](uint32_t row) { return (unsigned long long)__ldg(sort_keys + row); };
    bool sorted = true;
    for (int64_t t = j + 1; t < e && sorted; t++) {
      const unsigned long long a = key64(rows[t - 1]), b = key64(rows[t]);
      sorted = a < b || (a == b && rows[t - 1] < rows[t]);
    }
    if (sorted) continue;
    // Shell sort by (key64, row): correct for any run length
    const int64_t len = e - j;
    for (int64_t gap = len / 2; gap > 0; gap /= 2)
      for (int64_t t = j + gap; t < e; t++) {
        const uint32_t r = rows[t];
        const unsigned long long kr = key64(r);
        int64_t u = t;
        while (u >= j + gap) {
          const uint32_t ru = rows[u - gap];
          const unsigned long long ku = key64(ru);
          if (ku < kr || (ku == kr && ru < r)) break;
          rows[u] = ru;
          u -= gap;
        }
        rows[u] = r;
      }
  }
}

#endif

// Per-tile counts from the difference grid (2D inclusive prefix sums, in
// shared memory), the CSR starts (exclusive scan), K, the overflow flag, and
// the digit histograms of the tile keys for the LSD passes.  One CTA.
// Grids too large for shared memory (> 200 KB of cells: beyond ~51k tiles)
// are summed into the first difference-grid copy in global memory and
// prefixed there (each thread walks a row / column 32 cells at a time, the
// loads in flight together); preprocess re-zeroes the grids every frame.
__global__ void __launch_bounds__(1024) tile_counts_kernel(int* __restrict__ diff, int tiles_x, int tiles_y,
                                                           int64_t capacity, int64_t* tile_starts, int64_t* counters,
                                                           uint32_t* hist, int in_global, int* ready,
                                                           int publish_quads) {
  pdl_enter();
  // the ready queue of the fine binning -> blend handoff starts empty; with
  // no visible rows there is no fine binning: every quad is published here
  if (ready)
    for (int i = threadIdx.x; i < READY_HDR + READY_MAX_QUADS; i += blockDim.x)
      ready[i] = i == 0 ? publish_quads : (i >= READY_HDR && i < READY_HDR + publish_quads ? i - READY_HDR + 1 : 0);
  extern __shared__ int g_smem[];  // (tiles_x + 1) x (tiles_y + 1)
  int* g = in_global ? diff : g_smem;
  __shared__ uint32_t sh[3][RADIX];
  __shared__ int64_t s_chunk[1024];
  const int gw = tiles_x + 1;
  const int cells = gw * (tiles_y + 1);
  const int n_tiles = tiles_x * tiles_y;
  for (int i = threadIdx.x; i < 3 * RADIX; i += blockDim.x) (&sh[0][0])[i] = 0;
  if (!in_global && (cells & 3) == 0 && cells <= 4 * (int)blockDim.x) {
    // one round: every thread sums four cells of the 16 copies with 16-byte loads
    const int c4 = threadIdx.x * 4;
    if (c4 < cells) {
      int4 v = make_int4(0, 0, 0, 0);
#pragma unroll
      for (int k = 0; k < TILE_DIFF_COPIES; k++) {
        const int4 d = *reinterpret_cast<const int4*>(diff + (size_t)k * cells + c4);
        v.x += d.x, v.y += d.y, v.z += d.z, v.w += d.w;
      }
      g[c4] = v.x, g[c4 + 1] = v.y, g[c4 + 2] = v.z, g[c4 + 3] = v.w;
    }
  } else {
    for (int c = threadIdx.x; c < cells; c += blockDim.x) {
      int v = 0;
#pragma unroll
      for (int k = 0; k < TILE_DIFF_COPIES; k++) v += diff[(size_t)k * cells + c];
      g[c] = v;  // (global path: copy 0 in place -- each cell is read and written by one thread)
    }
  }
  __syncthreads();
  if (!in_global) {
    // warp-parallel prefix sums: a warp scans a row (then a column) 32 cells
    // at a time with shuffles, carrying the running total
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (int y = warp; y < tiles_y; y += nwarps) {  // prefix along x
      int carry = 0;
      for (int x0 = 0; x0 < tiles_x; x0 += 32) {
        const int x = x0 + lane;
        int v = x < tiles_x ? g[y * gw + x] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, v, o);
          if (lane >= o) v += t;
        }
        v += carry;
        if (x < tiles_x) g[y * gw + x] = v;
        carry = __shfl_sync(0xffffffffu, v, 31);
      }
    }
    __syncthreads();
    for (int x = warp; x < tiles_x; x += nwarps) {  // prefix along y
      int carry = 0;
      for (int y0 = 0; y0 < tiles_y; y0 += 32) {
        const int y = y0 + lane;
        int v = y < tiles_y ? g[y * gw + x] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, v, o);
          if (lane >= o) v += t;
        }
        v += carry;
        if (y < tiles_y) g[y * gw + x] = v;
        carry = __shfl_sync(0xffffffffu, v, 31);
      }
    }
  } else {
    for (int y = threadIdx.x; y < tiles_y; y += blockDim.x) {  // prefix along x, 32 cells per round
      int run = 0;
      int* row = g + (size_t)y * gw;
      for (int x0 = 0; x0 < tiles_x; x0 += 32) {
        int v[32];
#pragma unroll
        for (int i = 0; i < 32; i++) v[i] = x0 + i < tiles_x ? row[x0 + i] : 0;
#pragma unroll
        for (int i = 0; i < 32; i++) {
          run += v[i];
          if (x0 + i < tiles_x) row[x0 + i] = run;
        }
      }
    }
    __syncthreads();
    for (int x = threadIdx.x; x < tiles_x; x += blockDim.x) {  // prefix along y
      int run = 0;
      for (int y0 = 0; y0 < tiles_y; y0 += 32) {
        int v[32];
#pragma unroll
        for (int i = 0; i < 32; i++) v[i] = y0 + i < tiles_y ? g[(size_t)(y0 + i) * gw + x] : 0;
#pragma unroll
        for (int i = 0; i < 32; i++) {
          run += v[i];
          if (y0 + i < tiles_y) g[(size_t)(y0 + i) * gw + x] = run;
        }
      }
    }
  }
  __syncthreads();
  const int per = (n_tiles + blockDim.x - 1) / blockDim.x;
  const int t0 = threadIdx.x * per, t1 = min(n_tiles, t0 + per);
  int64_t local_sum = 0;
  for (int t = t0; t < t1; t++) {
    const int c = g[(t / tiles_x) * gw + t % tiles_x];
    local_sum += c;
    if (c && hist) {  // (the tile-key histograms: non-binned grids only)
      atomicAdd(&sh[0][t & 255], (uint32_t)c);
      atomicAdd(&sh[1][(t >> 8) & 255], (uint32_t)c);
      atomicAdd(&sh[2][(t >> 16) & 255], (uint32_t)c);
    }
  }
  // block-wide exclusive scan of the chunk sums
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t x = local_sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_chunk[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int64_t w = lane < (int)(blockDim.x >> 5) ? s_chunk[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    s_chunk[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  int64_t run = (warp > 0 ? s_chunk[warp - 1] : 0) + x - local_sum;
  if (threadIdx.x == blockDim.x - 1) {
    const int64_t total = s_chunk[(blockDim.x >> 5) - 1];
    counters[1] = total;
    counters[2] = total > capacity ? 1 : 0;
    tile_starts[n_tiles] = total;
  }
  for (int t = t0; t < t1; t++) {
    tile_starts[t] = run;
    run += g[(t / tiles_x) * gw + t % tiles_x];
  }
  if (hist)
    for (int i = threadIdx.x; i < 3 * RADIX; i += blockDim.x) hist[i] = (&sh[0][0])[i];
}

__global__ void __launch_bounds__(SCAN_THREADS) offsets_kernel(const int32_t* __restrict__ count,
                                                               const uint32_t* __restrict__ sorted_rows,
                                                               const int64_t* counters_in, uint32_t* offsets,
                                                               uint64_t* status, uint32_t* part_ctr,
                                                               int64_t* counters, int64_t capacity) {
  __shared__ int s_part;
  const int64_t m = counters_in[0];
  const int nparts = (int)((m + SCAN_TILE - 1) / SCAN_TILE);
  if (m == 0) return;
  while (true) {
    if (threadIdx.x == 0) s_part = (int)atomicAdd(part_ctr, 1u);
    __syncthreads();
    const int part = s_part;
    __syncthreads();
    if (part >= nparts) break;
    uint64_t excl[SCAN_IPT];
    uint64_t total;
    chained_scan_partition(part, m, [&](int64_t j) -> uint64_t { return (uint64_t)count[sorted_rows[j]]; }, status,
                           excl, total);
    const int64_t base = (int64_t)part * SCAN_TILE + (int64_t)threadIdx.x * SCAN_IPT;
#pragma unroll
    for (int j = 0; j < SCAN_IPT; j++)
      if (base + j < m) offsets[base + j] = (uint32_t)tmin<uint64_t>(excl[j], 0xffffffffull);
    (void)total;
    (void)capacity;
  }
}

// Warp-cooperative emission: a warp owns 32 consecutive rows of the depth
// order; their entries are contiguous in the output, so lanes stride over
// that span (coalesced stores), each lane advancing its owning row through
// the 32 row offsets staged in shared memory.  Rows with more than
// EMIT_BIG entries (near-camera Gaussians, which the depth order groups
// together) are deferred to emit_big_kernel, one CTA per row, so they cannot
// serialise a warp.
constexpr uint32_t EMIT_BIG = 256;

__device__ __forceinline__ void emit_entry(uint32_t o, uint32_t local, uint32_t x0, uint32_t y0, uint32_t rw,
                                           uint32_t g, int tiles_x, uint16_t* tkeys, uint32_t* tvals) {
  // local / rw with a float reciprocal estimate (exact after one correction: local < 2^21, rw < 2^16)
  uint32_t q = (uint32_t)((float)local * rcp_approx((float)rw));
  int32_t rr = (int32_t)(local - q * rw);
  if (rr < 0) { q--; rr += rw; } else if (rr >= (int32_t)rw) { q++; rr -= rw; }
  tkeys[o] = (uint16_t)((y0 + q) * (uint32_t)tiles_x + x0 + (uint32_t)rr);
  tvals[o] = g;
}
__device__ __forceinline__ void emit_entry(uint32_t o, uint32_t local, uint32_t x0, uint32_t y0, uint32_t rw,
                                           uint32_t g, int tiles_x, uint32_t* tkeys, uint32_t* tvals) {
  uint32_t q = (uint32_t)((float)local * rcp_approx((float)rw));
  int32_t rr = (int32_t)(local - q * rw);
  if (rr < 0) { q--; rr += rw; } else if (rr >= (int32_t)rw) { q++; rr -= rw; }
  tkeys[o] = (y0 + q) * (uint32_t)tiles_x + x0 + (uint32_t)rr;
  tvals[o] = g;
}

template <typename TK>
__global__ void __launch_bounds__(256) emit_kernel(const uint32_t* __restrict__ sorted_rows,
                                                   const uint32_t* __restrict__ offsets,
                                                   const ushort4* __restrict__ rect, const int64_t* counters,
                                                   int tiles_x, int64_t capacity, TK* tkeys, uint32_t* tvals,
                                                   uint32_t* big_rows, uint32_t* big_count) {
  __shared__ uint32_t s_off[8][32];
  __shared__ uint32_t s_end[8][32];
  __shared__ uint32_t s_row[8][32];
  __shared__ uint32_t s_x0w[8][32];  // x0 | (width << 16)
  __shared__ uint32_t s_y0[8][32];
  const int64_t m = counters[0];
  if (counters[1] > capacity) return;  // overflow: flagged in counters[2], nothing valid to emit
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nwarps = (int64_t)gridDim.x * 8;
  for (int64_t j0 = ((int64_t)blockIdx.x * 8 + warp) * 32; j0 < m; j0 += nwarps * 32) {
    const int64_t j = j0 + lane;
    const bool valid = j < m;
    uint32_t off = 0, cnt = 0;
    if (valid) {
      const uint32_t g = sorted_rows[j];
      off = offsets[j];
      const ushort4 rc = rect[g];  // x0, x1, y0, y1
      const uint32_t wdt = rc.y - rc.x + 1;
      cnt = wdt * (uint32_t)(rc.w - rc.z + 1);
      s_row[warp][lane] = g;
      s_x0w[warp][lane] = rc.x | (wdt << 16);
      s_y0[warp][lane] = rc.z;
      if (cnt > EMIT_BIG) {
        big_rows[atomicAdd(big_count, 1u)] = (uint32_t)j;
        cnt = 0;  // emitted by emit_big_kernel
      }
    }
    s_off[warp][lane] = valid ? off : 0xffffffffu;
    s_end[warp][lane] = off + cnt;
    const int last_lane = (int)tmin<int64_t>(31, m - 1 - j0);
    const uint32_t start = __shfl_sync(0xffffffffu, off, 0);
    const uint32_t end = __shfl_sync(0xffffffffu, off + (valid ? cnt : 0), last_lane);
    __syncwarp();
    int r = 0;  // owning row: non-decreasing along this lane's positions
    for (uint32_t o = start + lane; o < end; o += 32) {
      while (r < last_lane && (s_end[warp][r] <= o)) r++;
      if (o < s_off[warp][r]) {  // inside a deferred big row: jump past it, keeping o = start + lane (mod 32)
        o += (s_off[warp][r] - o - 1) / 32 * 32;
        continue;
      }
      const uint32_t x0w = s_x0w[warp][r];
      emit_entry(o, o - s_off[warp][r], x0w & 0xffffu, s_y0[warp][r], x0w >> 16, s_row[warp][r], tiles_x, tkeys,
                 tvals);
    }
    __syncwarp();
  }
}

template <typename TK>
__global__ void __launch_bounds__(256) emit_big_kernel(const uint32_t* __restrict__ sorted_rows,
                                                       const uint32_t* __restrict__ offsets,
                                                       const ushort4* __restrict__ rect, const int64_t* counters,
                                                       int tiles_x, int64_t capacity, TK* tkeys, uint32_t* tvals,
                                                       const uint32_t* __restrict__ big_rows,
                                                       const uint32_t* __restrict__ big_count) {
  if (counters[1] > capacity) return;
  const uint32_t nbig = *big_count;
  for (uint32_t b = blockIdx.x; b < nbig; b += gridDim.x) {
    const uint32_t j = big_rows[b];
    const uint32_t g = sorted_rows[j];
    const uint32_t off = offsets[j];
    const ushort4 rc = rect[g];
    const uint32_t rw = rc.y - rc.x + 1;
    const uint32_t cnt = rw * (uint32_t)(rc.w - rc.z + 1);
    for (uint32_t t = threadIdx.x; t < cnt; t += blockDim.x)
      emit_entry(off + t, t, rc.x, rc.z, rw, g, tiles_x, tkeys, tvals);
  }
}

// ------------------------------------------------------------ rect binning
// Two levels, no entry-level sort:
//  coarse: the depth-ordered rows are scattered, stably, into the lists of
//    the super-tiles (2^ss x 2^ss tiles, at most 256 of them) their
//    rectangles touch.  coarse_hist_kernel counts the (row, super-tile)
//    pairs per super-tile; coarse_bin_kernel takes partitions of BIN_PG rows
//    (8 warps x BIN_SUB) in dynamic order, counts each warp's pairs per
//    super-tile, gets every super-tile's offset from the earlier partitions
//    with a decoupled look-back (one super-tile per thread, as in a radix
//    pass), ranks the pairs in row order (warp match on the super-tile id
//    over the flattened pairs, per-warp counters) and writes (row, tile
//    rectangle) to the slot;
//  fine: fine_bin_kernel, one CTA per super-tile, each warp owning some of
//    its tiles, streams the super-tile's ordered list (coalesced, double
//    buffered) and keeps the rows whose rectangle contains the tile (ballot
//    compaction preserves order), writing them from tile_starts[t] on.
// A row's entries in a tile list are therefore in (depth, row) order, the
// reference's lexsort((kept, depth, tile)).
constexpr int BIN_THREADS = 256;
constexpr int BIN_WARPS = BIN_THREADS / 32;
constexpr int BIN_PG = 1024;                 // depth-ordered rows per partition
constexpr int BIN_SUB = BIN_PG / BIN_WARPS;  // rows per warp
// BIN_MAX_SUPER (common.cuh): super-tile capacity (two per thread in the
// scans); loops run to the frame's super-tile count
static_assert(BIN_MAX_SUPER == 2 * BIN_THREADS, "coarse scans hold two super-tiles per thread");
// warps per fine CTA (two CTAs per SM: the grid is one wave of super-tiles)
__host__ __device__ constexpr int fine_warps(int S) { return S == 4 ? 16 : 8; }
constexpr int FINE_DEPTH = 4;  // rounds of 32 list entries in flight per warp


// tile id of the l-th tile (row-major) of a rectangle of width rw in a grid
// of width gx
__device__ __forceinline__ uint32_t rect_tile(uint32_t l, ushort4 rc, uint32_t rw, int gx) {
  uint32_t q = (uint32_t)((float)l * rcp_approx((float)rw));  // exact after one correction (l < 2^21)
  int32_t rr = (int32_t)(l - q * rw);
  if (rr < 0) { q--; rr += rw; } else if (rr >= (int32_t)rw) { q++; rr -= rw; }
  return (rc.z + q) * (uint32_t)gx + rc.x + (uint32_t)rr;
}

__device__ __forceinline__ ushort4 coarse_rect(ushort4 rc, int ss) {
  return make_ushort4(rc.x >> ss, rc.y >> ss, rc.z >> ss, rc.w >> ss);
}

// ---- coarse level, partitioned by (row, super-tile) pairs ---------------
// The depth-ordered rows are flattened into their coarse pairs; pair
// offsets come from three small prep kernels; then every warp owns exactly
// CP_WARP consecutive pairs and every partition CP_PART (a huge near-camera
// rectangle is spread over many warps instead of stalling one).
constexpr int CP_WARP = 512;
constexpr int CP_PART = CP_WARP * BIN_WARPS;
constexpr int PREP_ROWS = 4096;  // rows per prep block (256 threads x 16)

__device__ __forceinline__ uint32_t coarse_pairs(ushort4 rc, int ss) {
  return (uint32_t)((rc.y >> ss) - (rc.x >> ss) + 1) * (uint32_t)((rc.w >> ss) - (rc.z >> ss) + 1);
}

// prep 1: rectangles in depth order, per-block pair sums
__global__ void __launch_bounds__(256) coarse_prep_sum_kernel(const uint32_t* __restrict__ sorted_rows,
                                                              const ushort4* __restrict__ rect, const int64_t* counters,
                                                              int ss, ushort4* __restrict__ rsort,
                                                              uint32_t* __restrict__ bsum) {
  pdl_enter();
  __shared__ uint32_t s_w[8];
  const int64_t m = counters[0];
  const int64_t b0 = (int64_t)blockIdx.x * PREP_ROWS;
  if (b0 >= m) return;
  uint32_t sum = 0;
  for (int i = threadIdx.x; i < PREP_ROWS; i += 256) {
    const int64_t j = b0 + i;
    if (j < m) {
      const ushort4 rc = rect[sorted_rows[j]];
      rsort[j] = rc;
      sum += coarse_pairs(rc, ss);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < 8; w++) t += s_w[w];
    bsum[blockIdx.x] = t;
  }
}

// prep 2 (one CTA): exclusive scan of the block sums; pair total -> *npairs
__global__ void __launch_bounds__(1024) coarse_prep_scan_kernel(const int64_t* counters, uint32_t* __restrict__ bsum,
                                                                uint32_t* __restrict__ npairs) {
  pdl_enter();
  __shared__ uint32_t s_w[32];
  __shared__ uint32_t s_carry;
  const int64_t m = counters[0];
  const int nblk = (int)((m + PREP_ROWS - 1) / PREP_ROWS);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < nblk; b0 += 1024) {
    const int i = b0 + threadIdx.x;
    const uint32_t v = i < nblk ? bsum[i] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint32_t w = s_w[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      s_w[lane] = w;
    }
    __syncthreads();
    const uint32_t carry = s_carry;
    const uint32_t excl = carry + (warp ? s_w[warp - 1] : 0u) + x - v;
    if (i < nblk) bsum[i] = excl;
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = carry + s_w[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) *npairs = s_carry;
}

// prep 3: pair offset of every row (pair_off[m] = total) and the first row
// of every CP_WARP-pair warp range
__global__ void __launch_bounds__(256) coarse_prep_offsets_kernel(const ushort4* __restrict__ rsort,
                                                                  const int64_t* counters, int ss,
                                                                  const uint32_t* __restrict__ bpre,
                                                                  const uint32_t* __restrict__ npairs,
                                                                  uint32_t* __restrict__ pair_off,
                                                                  uint32_t* __restrict__ wstart) {
  pdl_enter();
  __shared__ uint32_t s_w[8];
  const int64_t m = counters[0];
  const int64_t b0 = (int64_t)blockIdx.x * PREP_ROWS;
  if (b0 >= m) return;
  constexpr int PER = PREP_ROWS / 256;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t c[PER], lsum = 0;
#pragma unroll
  for (int q = 0; q < PER; q++) {
    const int64_t j = b0 + threadIdx.x * PER + q;
    c[q] = j < m ? coarse_pairs(rsort[j], ss) : 0u;
    lsum += c[q];
  }
  uint32_t x = lsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[warp] = x;
  __syncthreads();
  uint32_t run = bpre[blockIdx.x] + x - lsum;
  for (int w = 0; w < warp; w++) run += s_w[w];
#pragma unroll
  for (int q = 0; q < PER; q++) {
    const int64_t j = b0 + threadIdx.x * PER + q;
    if (j < m) {
      pair_off[j] = run;
      for (uint32_t k = (run + CP_WARP - 1) / CP_WARP; k * CP_WARP < run + c[q]; k++) wstart[k] = (uint32_t)j;
    }
    run += c[q];
  }
  if (b0 + PREP_ROWS >= m && threadIdx.x == 0) pair_off[m] = *npairs;
}

// The three prep steps fused: one persistent chained-scan pass (decoupled
// look-back, sort.cuh) gathers the rectangles in depth order, scans the
// rows' coarse pair counts and writes the pair offsets, warp-range starts
// and the total.
__global__ void __launch_bounds__(SCAN_THREADS) coarse_prep_kernel(const uint32_t* __restrict__ sorted_rows,
                                                                   const ushort4* __restrict__ rect,
                                                                   const int64_t* counters, int ss,
                                                                   ushort4* __restrict__ rsort,
                                                                   uint32_t* __restrict__ pair_off,
                                                                   uint32_t* __restrict__ wstart,
                                                                   uint32_t* __restrict__ npairs, uint64_t* status,
                                                                   uint32_t* part_ctr) {
  pdl_enter();
  __shared__ int s_part;
  const int64_t m = counters[0];
  if (m == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      pair_off[0] = 0;
      *npairs = 0;
    }
    return;
  }
  const int nparts = (int)((m + SCAN_TILE - 1) / SCAN_TILE);
  while (true) {
    if (threadIdx.x == 0) s_part = (int)atomicAdd(part_ctr, 1u);
    __syncthreads();
    const int part = s_part;
    __syncthreads();
    if (part >= nparts) break;
    const int64_t base = (int64_t)part * SCAN_TILE + (int64_t)threadIdx.x * SCAN_IPT;
    uint32_t c[SCAN_IPT];
#pragma unroll
    for (int j = 0; j < SCAN_IPT; j++) {
      const int64_t i = base + j;
      c[j] = 0;
      if (i < m) {
        const ushort4 rc = rect[sorted_rows[i]];
        rsort[i] = rc;
        c[j] = coarse_pairs(rc, ss);
      }
    }
    uint64_t excl[SCAN_IPT];
    uint64_t total;
    chained_scan_partition(part, m, [&](int64_t i) -> uint64_t { return (uint64_t)c[i - base]; }, status, excl,
                           total);
#pragma unroll
    for (int j = 0; j < SCAN_IPT; j++) {
      const int64_t i = base + j;
      if (i < m) {
        const uint32_t run = (uint32_t)excl[j];
        pair_off[i] = run;
        for (uint32_t k = (run + CP_WARP - 1) / CP_WARP; k * CP_WARP < run + c[j]; k++) wstart[k] = (uint32_t)i;
      }
    }
    if (part == nparts - 1 && threadIdx.x == 0) {
      pair_off[m] = (uint32_t)total;
      *npairs = (uint32_t)total;
    }
  }
}

// Walk the CP_WARP pairs of warp range k in rounds of 32 (lane = pair):
// f(valid, super-tile, row, fine rectangle).  Lane i looks at row ra + 1 + i
// (coalesced): the row starts inside the round become a bit mask, each
// lane's owner is ra + (starts at or before it), and the owner's data comes
// over a shuffle (every row has at least one pair, so at most 32 rows start
// inside a round).
template <typename F>
__device__ __forceinline__ void walk_pairs(uint32_t k, uint32_t P, int64_t m, const uint32_t* __restrict__ pair_off,
                                           const ushort4* __restrict__ rsort, const uint32_t* __restrict__ sorted_rows,
                                           const uint32_t* __restrict__ wstart, int ss, int sx, int lane, F f) {
  const uint32_t ob = k * CP_WARP, oe = min(P, ob + CP_WARP);
  if (ob >= oe) return;
  int64_t ra = wstart[k];
  uint32_t offA = pair_off[ra], gA = sorted_rows[ra];
  ushort4 rcA = rsort[ra];
  for (uint32_t o0 = ob; o0 < oe; o0 += 32) {
    const int64_t r = ra + 1 + lane;
    const uint32_t st = r <= m ? pair_off[r] : 0xffffffffu;
    ushort4 rcL = make_ushort4(0, 0, 0, 0);
    uint32_t gL = 0;
    if (r < m) {
      rcL = rsort[r];
      gL = sorted_rows[r];
    }
    const uint32_t rel = st - o0;  // >= 1: ra owns o0
    const unsigned bits = __reduce_or_sync(0xffffffffu, rel < 32 ? (1u << rel) : 0u);
    const int kown = __popc(bits & ((2u << lane) - 1u));
    const int src = kown > 0 ? kown - 1 : 0;
    const uint32_t rlo = (uint32_t)rcL.x | ((uint32_t)rcL.y << 16), rhi = (uint32_t)rcL.z | ((uint32_t)rcL.w << 16);
    const uint32_t o_off = __shfl_sync(0xffffffffu, st, src);
    const uint32_t o_g = __shfl_sync(0xffffffffu, gL, src);
    const uint32_t o_lo = __shfl_sync(0xffffffffu, rlo, src), o_hi = __shfl_sync(0xffffffffu, rhi, src);
    const uint32_t off = kown ? o_off : offA, g = kown ? o_g : gA;
    const ushort4 rc = kown ? make_ushort4(o_lo & 0xffffu, o_lo >> 16, o_hi & 0xffffu, o_hi >> 16) : rcA;
    const uint32_t o = o0 + lane;
    const bool valid = o < oe;
    uint32_t sti = 0xffffffffu;
    if (valid) {
      const ushort4 cr = coarse_rect(rc, ss);
      sti = rect_tile(o - off, cr, (uint32_t)(cr.y - cr.x + 1), sx);
    }
    f(valid, sti, g, rc);
    const int adv = __popc(bits) + (__any_sync(0xffffffffu, rel == 32) ? 1 : 0);
    if (adv > 0) {
      offA = __shfl_sync(0xffffffffu, st, adv - 1);
      gA = __shfl_sync(0xffffffffu, gL, adv - 1);
      const uint32_t a_lo = __shfl_sync(0xffffffffu, rlo, adv - 1), a_hi = __shfl_sync(0xffffffffu, rhi, adv - 1);
      rcA = make_ushort4(a_lo & 0xffffu, a_lo >> 16, a_hi & 0xffffu, a_hi >> 16);
      ra += adv;
    }
  }
}

struct CoarseArgs {
  const uint32_t* sorted_rows;
  const ushort4* rsort;
  const uint32_t* pair_off;
  const uint32_t* wstart;
  const uint32_t* npairs;
  const int64_t* counters;
  int64_t capacity;
  int ss, sx, ns;
};

// per-partition super-tile counts -> mat[part][BIN_MAX_SUPER], totals -> hist
__global__ void __launch_bounds__(BIN_THREADS) coarse_count_kernel(CoarseArgs a, uint32_t* __restrict__ mat,
                                                                   uint32_t* __restrict__ wmat,
                                                                   uint32_t* __restrict__ hist) {
  pdl_enter();
  __shared__ uint32_t cnt[BIN_WARPS][BIN_MAX_SUPER];
  const int64_t m = a.counters[0];
  if (a.counters[1] > a.capacity) return;  // overflow: flagged in counters[2]
  const uint32_t P = *a.npairs;
  const int nparts = (int)((P + CP_PART - 1) / CP_PART);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int part = blockIdx.x; part < nparts; part += gridDim.x) {
#pragma unroll
    for (int w = 0; w < BIN_WARPS; w++)
      for (int t = threadIdx.x; t < a.ns; t += BIN_THREADS) cnt[w][t] = 0;
    __syncthreads();
    walk_pairs((uint32_t)part * BIN_WARPS + warp, P, m, a.pair_off, a.rsort, a.sorted_rows, a.wstart, a.ss, a.sx, lane,
               [&](bool valid, uint32_t sti, uint32_t, ushort4) {
                 if (valid) atomicAdd(&cnt[warp][sti], 1u);
               });
    __syncthreads();
    for (int t = threadIdx.x; t < a.ns; t += BIN_THREADS) {  // per-warp exclusive prefix (for the scatter) and total
      uint32_t acc = 0;
#pragma unroll
      for (int w = 0; w < BIN_WARPS; w++) {
        const uint32_t v = cnt[w][t];
        wmat[((size_t)part * BIN_WARPS + w) * BIN_MAX_SUPER + t] = acc;
        acc += v;
      }
      mat[(size_t)part * BIN_MAX_SUPER + t] = acc;
      if (acc) atomicAdd(&hist[t], acc);
    }
    __syncthreads();
  }
}

// List starts (exclusive scan of the histogram) and the slot of every
// (partition, super-tile): one CTA per 32 super-tiles, 32 warps splitting
// the partitions (lane = super-tile).
__global__ void __launch_bounds__(1024) coarse_scan_kernel(const uint32_t* __restrict__ mat,
                                                           const uint32_t* __restrict__ hist, const int64_t* counters,
                                                           int64_t capacity, const uint32_t* __restrict__ npairs,
                                                           int ns, uint32_t* __restrict__ cstart,
                                                           uint32_t* __restrict__ slot) {
  pdl_enter();
  __shared__ uint32_t s_sum[32][33];
  __shared__ uint32_t s_start[32];
  if (counters[1] > capacity) return;
  const int nparts = (int)((*npairs + CP_PART - 1) / CP_PART);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  if (warp == 0) {
    // start of this CTA's first super-tile: sum of the histogram before it
    uint32_t pre = 0;
    for (int t = lane; t < blockIdx.x * 32; t += 32) pre += hist[t];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
    const uint32_t h = c < ns ? hist[c] : 0u;
    uint32_t x = h;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    s_start[lane] = pre + x - h;
    if (c < ns) cstart[c] = pre + x - h;
    if (c == ns - 1) cstart[ns] = pre + x;
  }
  const int per = (nparts + 31) / 32;
  const int p0 = warp * per, p1 = min(nparts, p0 + per);
  uint32_t sum = 0;
  if (c < ns)
    for (int p = p0; p < p1; p++) sum += mat[(size_t)p * BIN_MAX_SUPER + c];
  s_sum[warp][lane] = sum;
  __syncthreads();
  if (c >= ns) return;
  uint32_t run = s_start[lane];
  for (int w = 0; w < warp; w++) run += s_sum[w][lane];
  for (int p = p0; p < p1; p++) {
    slot[(size_t)p * BIN_MAX_SUPER + c] = run;
    run += mat[(size_t)p * BIN_MAX_SUPER + c];
  }
}

// in-order ranking of every warp's pairs and the scatter of (row, tile
// rectangle) into the coarse lists
// The partition's pairs are first placed in shared memory in (super-tile,
// rank) order, then written out as contiguous runs per super-tile
// (coalesced: a random (row, super-tile) scatter would touch a fresh 32 B
// sector per pair).
// Dynamic shared memory: a fixed head followed by arrays sized by the
// frame's super-tile count (nsp = ns rounded up to even), so a small grid
// keeps the occupancy of the old fixed layout: lstart[nsp + 1] (partition-
// local run starts), gslot[nsp] (global slot of each run), cnt[8][nsp]
// (per-warp local positions).
struct ScatterSmem {
  uint4 stage[CP_PART];                      // row, rect lo, rect hi, super-tile
  uint32_t warp_tmp[8];
};
__host__ __device__ inline int scatter_nsp(int ns) { return (ns + 1) & ~1; }
__host__ __device__ inline size_t scatter_smem_bytes(int ns) {
  const int nsp = scatter_nsp(ns);
  return sizeof(ScatterSmem) + sizeof(uint32_t) * (size_t)(nsp + 1 + nsp + BIN_WARPS * nsp);
}

__global__ void __launch_bounds__(BIN_THREADS) coarse_scatter_kernel(CoarseArgs a, const uint32_t* __restrict__ mat,
                                                                     const uint32_t* __restrict__ slot,
                                                                     const uint32_t* __restrict__ wmat,
                                                                     uint32_t* __restrict__ crow,
                                                                     ushort4* __restrict__ crect_out) {
  pdl_enter();
  extern __shared__ __align__(16) unsigned char sc_raw[];
  ScatterSmem& sm = *reinterpret_cast<ScatterSmem*>(sc_raw);
  const int nsp = scatter_nsp(a.ns);
  uint32_t* lstart = reinterpret_cast<uint32_t*>(sc_raw + sizeof(ScatterSmem));
  uint32_t* gslot = lstart + nsp + 1;
  uint32_t* cnt = gslot + nsp;  // [warp * nsp + super-tile]
  const int64_t m = a.counters[0];
  if (a.counters[1] > a.capacity) return;
  const uint32_t P = *a.npairs;
  const int nparts = (int)((P + CP_PART - 1) / CP_PART);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int part = blockIdx.x; part < nparts; part += gridDim.x) {
    const uint32_t k = (uint32_t)part * BIN_WARPS + warp;
    {  // partition-local run starts (exclusive scan over super-tiles; two consecutive per thread)
      const int t0 = 2 * threadIdx.x;
      const size_t row = (size_t)part * BIN_MAX_SUPER;
      const uint32_t c0 = t0 < a.ns ? mat[row + t0] : 0u, c1 = t0 + 1 < a.ns ? mat[row + t0 + 1] : 0u;
      uint32_t tot;
      const uint32_t e = block_exclusive_scan<uint32_t>(c0 + c1, sm.warp_tmp, tot);
      if (t0 < nsp) {
        lstart[t0] = e;
        lstart[t0 + 1] = e + c0;
        gslot[t0] = t0 < a.ns ? slot[row + t0] : 0u;
        gslot[t0 + 1] = t0 + 1 < a.ns ? slot[row + t0 + 1] : 0u;
      }
      if (threadIdx.x == 0) lstart[nsp] = tot;
      __syncthreads();
    }
#pragma unroll
    for (int w = 0; w < BIN_WARPS; w++)
      for (int t = threadIdx.x; t < a.ns; t += BIN_THREADS)
        cnt[w * nsp + t] = lstart[t] + wmat[((size_t)part * BIN_WARPS + w) * BIN_MAX_SUPER + t];
    __syncthreads();
    walk_pairs(k, P, m, a.pair_off, a.rsort, a.sorted_rows, a.wstart, a.ss, a.sx, lane,
               [&](bool valid, uint32_t sti, uint32_t g, ushort4 rc) {
                 static_assert(BIN_MAX_SUPER <= 512, "super-tile index: 9 bits");
                 const unsigned peers = warp_peers<9>(sti, __ballot_sync(0xffffffffu, valid));
                 uint32_t cur = 0;
                 if (valid) cur = cnt[warp * nsp + sti];
                 __syncwarp();
                 if (valid) {
                   const uint32_t pos = cur + __popc(peers & lanemask_lt());
                   sm.stage[pos] = make_uint4(g, (uint32_t)rc.x | ((uint32_t)rc.y << 16),
                                              (uint32_t)rc.z | ((uint32_t)rc.w << 16), sti);
                   if (lane == __ffs(peers) - 1) cnt[warp * nsp + sti] = cur + __popc(peers);
                 }
                 __syncwarp();
               });
    __syncthreads();
    const uint32_t n = lstart[nsp];
    for (uint32_t i = threadIdx.x; i < n; i += BIN_THREADS) {
      const uint4 v = sm.stage[i];
      const uint32_t pos = gslot[v.w] + (i - lstart[v.w]);
      crow[pos] = v.x;
      crect_out[pos] = make_ushort4(v.y & 0xffffu, v.y >> 16, v.z & 0xffffu, v.z >> 16);
    }
    __syncthreads();
  }
}

// Fine level: one CTA per super-tile (S x S tiles, S = 4 or 8).  Every list
// entry becomes the bit mask of the super-tile's tiles its rectangle covers;
// the 16 warps take contiguous parts of the ordered list, count per tile
// (pass 1: byte-packed warp reductions), take their per-tile start from the
// warp prefix, then write (pass 2: one ballot per tile keeps the list order).
__device__ __forceinline__ ushort4 unpack_rect(uint2 r) {
  return make_ushort4((unsigned short)(r.x & 0xFFFFu), (unsigned short)(r.x >> 16), (unsigned short)(r.y & 0xFFFFu),
                      (unsigned short)(r.y >> 16));
}

template <int S>
struct FineMask;
template <>
struct FineMask<4> {
  using T = uint32_t;
  __device__ static T of(ushort4 rc, int sx0, int sy0) {
    const int lx0 = max((int)rc.x - sx0, 0), lx1 = min((int)rc.y - sx0, 3);
    const int ly0 = max((int)rc.z - sy0, 0), ly1 = min((int)rc.w - sy0, 3);
    if (lx0 > lx1 || ly0 > ly1) return 0u;
    const uint32_t rowbits = (2u << lx1) - (1u << lx0);
    const uint32_t ymask = (ly1 == 3 ? 0x10000u : (1u << (4 * (ly1 + 1)))) - (1u << (4 * ly0));
    return (rowbits * 0x1111u) & ymask;
  }
  __device__ static bool bit(T m, int q) { return (m >> q) & 1u; }
  __device__ static uint32_t nibble(T m, int j) { return (m >> (4 * j)) & 0xFu; }
};

template <int S>
__global__ void __launch_bounds__(fine_warps(S) * 32) fine_bin_kernel(
    const uint32_t* __restrict__ crow, const ushort4* __restrict__ crect, const uint32_t* __restrict__ cstart,
    const int64_t* __restrict__ tile_starts, const int64_t* counters, int64_t capacity, int tiles_x, int tiles_y,
    int sx, uint32_t* __restrict__ entries, int qs, int* __restrict__ ready) {
  pdl_enter();
  constexpr int NT = S * S;
  using M = FineMask<S>;
  constexpr int FINE_WARPS = fine_warps(S);
  __shared__ uint32_t s_cnt[FINE_WARPS][NT];
  if (counters[1] > capacity) return;
  // qs > 0: the super-tiles are (S << qs)^2 tiles and 4^qs CTAs share one,
  // each owning an S x S block of its tiles (every CTA reads the whole coarse
  // list, writes only its own tiles' entries: no cross-CTA dependency)
  const int s = blockIdx.x >> (2 * qs), quad = blockIdx.x & ((1 << (2 * qs)) - 1);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sx0 = (s % sx) * (S << qs) + (quad & ((1 << qs) - 1)) * S;
  const int sy0 = (s / sx) * (S << qs) + (quad >> qs) * S;
  const uint32_t b = cstart[s], e = cstart[s + 1];
  const uint32_t per = ((e - b + FINE_WARPS - 1) / FINE_WARPS + 31) & ~31u;
  const uint32_t w0 = min(e, b + warp * per), w1 = min(e, w0 + per);
  // pass 1: per-tile counts of this warp's part (4 tiles per byte-packed
  // reduction); the next FINE_DEPTH rounds' rectangles are in flight
  uint32_t cnt[NT];
#pragma unroll
  for (int q = 0; q < NT; q++) cnt[q] = 0;
  // loads from a clamped index (no select on the loaded value, which would
  // wait for it at once); validity is applied where the rectangle is used
  const uint32_t klast = w1 > w0 ? w1 - 1 : 0u;
  const uint2* __restrict__ crect2 = reinterpret_cast<const uint2*>(crect);
  uint2 rq[FINE_DEPTH];  // raw 64-bit rectangles: fields are unpacked only where used
#pragma unroll
  for (int d = 0; d < FINE_DEPTH; d++) rq[d] = __ldg(crect2 + min(w0 + d * 32 + lane, klast));
  for (uint32_t k0 = w0; k0 < w1; k0 += 32 * FINE_DEPTH) {
#pragma unroll
    for (int d = 0; d < FINE_DEPTH; d++) {
      const bool valid = k0 + d * 32 + lane < w1;
      const typename M::T msk = valid ? M::of(unpack_rect(rq[d]), sx0, sy0) : (typename M::T)0;
      rq[d] = __ldg(crect2 + min(k0 + (d + FINE_DEPTH) * 32 + lane, klast));
#pragma unroll
      for (int j = 0; j < NT / 4; j++) {
        const uint32_t packed = __reduce_add_sync(0xffffffffu, (M::nibble(msk, j) * 0x00204081u) & 0x01010101u);
#pragma unroll
        for (int i = 0; i < 4; i++) cnt[4 * j + i] += (packed >> (8 * i)) & 0xFFu;
      }
    }
  }
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NT; q++) s_cnt[warp][q] = cnt[q];
  __syncthreads();
  uint32_t out[NT];
#pragma unroll
  for (int q = 0; q < NT; q++) {
    const int tx = sx0 + q % S, ty = sy0 + q / S;
    uint32_t o = 0;
    if (tx < tiles_x && ty < tiles_y) {
      o = (uint32_t)tile_starts[ty * tiles_x + tx];
      for (int w = 0; w < warp; w++) o += s_cnt[w][q];
    }
    out[q] = o;
  }
  // pass 2: write (same prefetch ring)
  uint32_t gq[FINE_DEPTH];
#pragma unroll
  for (int d = 0; d < FINE_DEPTH; d++) {
    const uint32_t k = min(w0 + d * 32 + lane, klast);
    rq[d] = __ldg(crect2 + k);
    gq[d] = __ldg(crow + k);
  }
  for (uint32_t k0 = w0; k0 < w1; k0 += 32 * FINE_DEPTH) {
#pragma unroll
    for (int d = 0; d < FINE_DEPTH; d++) {
      const bool valid = k0 + d * 32 + lane < w1;
      const typename M::T msk = valid ? M::of(unpack_rect(rq[d]), sx0, sy0) : (typename M::T)0;
      const uint32_t g = gq[d];
      const uint32_t k = min(k0 + (d + FINE_DEPTH) * 32 + lane, klast);
      rq[d] = __ldg(crect2 + k);
      gq[d] = __ldg(crow + k);
#pragma unroll
      for (int q = 0; q < NT; q++) {
        const bool hit = M::bit(msk, q);
        const unsigned bal = __ballot_sync(0xffffffffu, hit);
        if (hit) entries[out[q] + __popc(bal & lanemask_lt())] = g;
        out[q] += __popc(bal);
      }
    }
  }
  // publish this quad: its tiles' entries are complete
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int k = atomicAdd(&ready[0], 1);
    atomicExch(&ready[READY_HDR + k], (int)blockIdx.x + 1);
  }
}

// ---------------------------------------------------------------- host side

struct TilesScratch {
  uint64_t* dk[2];
  uint32_t* dv[2];
  uint32_t* offsets;
  uint32_t* big_rows;
  void* tk[2];
  uint32_t* tv0;
  uint32_t* tv1;
  // zeroed control block
  uint32_t* rs_status;    // 3 depth passes x 2 parts_n (2048-key partitions) x 256
  uint32_t* rs_tile_status;  // 3 tile passes x parts_k x 256 (outside the zeroed block: zeroed only when used)
  uint64_t* scan_status;  // 2 x (parts_n + 1)
  uint32_t* hist;         // 10 x 256
  uint32_t* part_ctr;     // 32
  uint32_t* bin_mat;      // parts_bin x BIN_MAX_SUPER: per-partition super-tile counts
  uint32_t* bin_slot;     // parts_bin x BIN_MAX_SUPER: slot per (partition, super-tile)
  uint32_t* bin_wmat;     // parts_bin x 8 x BIN_MAX_SUPER: per-warp exclusive counts
  uint32_t* chist;        // BIN_MAX_SUPER (zeroed)
  uint32_t* vis_cnt;      // 2 parts_n: visible rows per RS_PART-row partition (HGS_DEPTH_MODE 2)
  uint32_t* cstart;       // BIN_MAX_SUPER + 1: super-tile list starts
  void* cprog;            // n_tiles x 16 B: blend-only progress per tile (hgs_tiles.coarse_prog)
  ushort4* rsort;         // n: tile rectangles in depth order
  uint32_t* pair_off;     // n + 1: coarse pair offsets in depth order
  uint32_t* bsum;         // prep blocks
  uint32_t* wstart;       // capacity / CP_WARP + 2: first row of every warp range
  uint32_t* npairs;       // 1
  uint32_t* crow;         // capacity: coarse lists (rows)
  ushort4* crect;         // capacity: coarse lists (tile rectangles)
  int* diff;              // (tiles_x + 1) x (tiles_y + 1)
  size_t control_bytes;
  void* control_begin;
  int64_t parts_n, parts_k;
};

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// n_super_hint > 0: size the binning arrays for that many super-tiles (the
// scratch-size query, which only knows the tile count)
static size_t carve(int64_t n, int64_t cap, int tiles_x, int tiles_y, unsigned char* base, TilesScratch* s,
                    int n_super_hint = 0) {
  const int n_tiles = tiles_x * tiles_y;
  const size_t tkw = n_tiles > 65535 ? 4 : 2;
  const int64_t nn = n > 0 ? n : 1, cc = cap > 0 ? cap : 1;
  const int64_t parts_n = (nn + RS_TILE - 1) / RS_TILE, parts_k = (cc + RS_TILE - 1) / RS_TILE;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes, 256);
    return base ? (void*)(base + o) : nullptr;
  };
  TilesScratch t{};
  // the zeroed control block
  const size_t ctl0 = off;
  t.control_begin = base ? base + ctl0 : nullptr;
  t.rs_status = (uint32_t*)take(sizeof(uint32_t) * RADIX * (size_t)(3 * 2 * parts_n));
  t.scan_status = (uint64_t*)take(sizeof(uint64_t) * (size_t)(2 * (parts_n + 1)));
  t.hist = (uint32_t*)take(sizeof(uint32_t) * 11 * RADIX);
  t.part_ctr = (uint32_t*)take(sizeof(uint32_t) * 32);  // [24..27]: depth key min/max (u64 x 2)
  t.diff = (int*)take(sizeof(int) * (size_t)(tiles_x + 1) * (size_t)(tiles_y + 1));
  const bool binned = (n_super_hint > 0 ? n_super_hint <= BIN_MAX_SUPER : super_shift(tiles_x, tiles_y) >= 0);
  t.chist = binned ? (uint32_t*)take(sizeof(uint32_t) * BIN_MAX_SUPER) : nullptr;
  t.control_bytes = off - ctl0;
  t.rs_tile_status = (uint32_t*)take(sizeof(uint32_t) * RADIX * (size_t)(3 * parts_k));
  t.vis_cnt = (uint32_t*)take(sizeof(uint32_t) * (size_t)(2 * parts_n));
  t.dk[0] = (uint64_t*)take(8 * nn);
  t.dk[1] = (uint64_t*)take(8 * nn + 16);  // two 32-bit key arrays, the second 16-B aligned (cp.async staging)
  t.dv[0] = (uint32_t*)take(4 * nn);
  t.dv[1] = (uint32_t*)take(4 * nn);
  t.offsets = (uint32_t*)take(4 * nn);
  t.big_rows = (uint32_t*)take(4 * nn);
  t.tk[0] = take(tkw * cc);
  t.tk[1] = take(tkw * cc);
  t.tv0 = (uint32_t*)take(4 * cc);
  t.tv1 = (uint32_t*)take(4 * cc);
  t.crow = binned ? (uint32_t*)take(sizeof(uint32_t) * (size_t)cc) : nullptr;
  const size_t cparts = (size_t)(cc / CP_PART + 2);
  t.bin_mat = binned ? (uint32_t*)take(sizeof(uint32_t) * BIN_MAX_SUPER * cparts) : nullptr;
  t.bin_slot = binned ? (uint32_t*)take(sizeof(uint32_t) * BIN_MAX_SUPER * cparts) : nullptr;
  t.bin_wmat = binned ? (uint32_t*)take(sizeof(uint32_t) * BIN_MAX_SUPER * BIN_WARPS * cparts) : nullptr;
  t.rsort = binned ? (ushort4*)take(sizeof(ushort4) * (size_t)nn) : nullptr;
  t.pair_off = binned ? (uint32_t*)take(sizeof(uint32_t) * (size_t)(nn + 1)) : nullptr;
  t.bsum = binned ? (uint32_t*)take(sizeof(uint32_t) * (size_t)(nn / PREP_ROWS + 2)) : nullptr;
  t.wstart = binned ? (uint32_t*)take(sizeof(uint32_t) * (size_t)(cc / CP_WARP + 2)) : nullptr;
  t.npairs = binned ? (uint32_t*)take(sizeof(uint32_t) * 4) : nullptr;
  t.crect = binned ? (ushort4*)take(sizeof(ushort4) * (size_t)cc) : nullptr;
  t.cstart = binned ? (uint32_t*)take(sizeof(uint32_t) * (size_t)(BIN_MAX_SUPER + 1)) : nullptr;
  t.cprog = binned ? take(16 * (size_t)n_tiles) : nullptr;
  t.parts_n = parts_n;
  t.parts_k = parts_k;
  if (s) *s = t;
  return off;
}

static int sm_count() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = NUM_SMS;
  }
  return sms;
}

static int persistent_grid(const void* fn, int threads, size_t smem) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem);
  if (per_sm < 1) per_sm = 1;
  return per_sm * sm_count();
}

// Stable LSD radix sort of (key, value) pairs, npasses 8-bit digits from
// shift0: one histogram kernel for all passes, then one single-pass
// (decoupled look-back) kernel per pass.  The last pass writes its values to
// final_vals when given.
// pcnt != nullptr: reduce-then-scan passes (upsweep counts, one scan CTA,
// rank + scatter from precomputed offsets; pcnt holds parts x 256 words)
// instead of the single-pass decoupled look-back.
// implicit_vals: the first pass's values are the input positions (v0 unread).
// counted: reduce-then-scan without upsweeps -- status holds npasses x parts
// x 256 count words, zero except the first pass's, which the
// caller wrote (depth_remap_kernel); each pass counts the next one's as it
// scatters, and radix_scan_kernel turns a pass's counts into offsets.
template <typename K, int IPT = RS_IPT>
static int radix_sort(K* k0, K* k1, uint32_t* v0, uint32_t* v1, uint32_t* final_vals, const int64_t* count_ptr,
                      int64_t cap, int shift0, int npasses, uint32_t* hist, bool hist_ready, uint32_t* status,
                      int64_t parts, uint32_t* part_ctr, cudaStream_t st, K** keys_result, bool last_keys,
                      uint32_t** vals_result = nullptr, uint32_t* pcnt = nullptr, bool counted = false,
                      bool implicit_vals = false) {
  const size_t smem = sizeof(RadixSmem<K, IPT>);
  static int grid = 0;
  if (grid == 0) {
    cudaFuncSetAttribute(radix_pass_kernel<K, IPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    grid = persistent_grid((const void*)radix_pass_kernel<K, IPT>, RS_THREADS, smem);
  }
  const int64_t tile = (int64_t)RS_THREADS * IPT;
  parts = (cap + tile - 1) / tile;  // partitions of this pass width (status sized for RS_TILE partitions)
  if (!hist_ready) {
    radix_hist_kernel<K><<<2 * sm_count(), 256, 0, st>>>(k0, count_ptr, cap, shift0, npasses, hist);
    HGS_CHECK_LAUNCH();
  }
  const int g = (int)tmax<int64_t>(1, tmin<int64_t>(grid, parts));
  K* kin = k0;
  K* kout = k1;
  uint32_t* vin = v0;
  uint32_t* vout = v1;
  for (int p = 0; p < npasses; p++) {
    const bool last = p == npasses - 1;
    uint32_t* vdst = last && final_vals ? final_vals : vout;
    uint32_t* poff = nullptr;
    uint32_t* pnext = nullptr;
    if (counted) {
      // counted reduce-then-scan: pass p's counts were written by the
      // previous kernel (pass 0: the caller) into status[p]; scan them into
      // offsets in place, count pass p + 1's digits while scattering
      poff = status + (size_t)p * parts * RADIX;
      pnext = last ? nullptr : status + (size_t)(p + 1) * parts * RADIX;
      // (16 CTAs: a one-CTA-per-digit scan was 47 us / frame slower in the
      // chain although faster alone -- its CTAs, scheduled early by PDL,
      // hold SM slots while the previous pass runs)
      launch_pdl(radix_scan_kernel, dim3(RADIX / RSCAN_DIGITS), dim3(RSCAN_DIGITS * RSCAN_GROUPS), 0, st,
                 (const uint32_t*)(hist + RADIX * p), count_ptr, cap, (int)tile, poff);
      HGS_CHECK_LAUNCH();
    } else if (pcnt) {
      radix_upsweep_kernel<K, IPT><<<(int)parts, RS_THREADS, 0, st>>>(kin, count_ptr, cap, shift0 + 8 * p, pcnt);
      HGS_CHECK_LAUNCH();
      radix_scan_kernel<<<RADIX / RSCAN_DIGITS, RSCAN_DIGITS * RSCAN_GROUPS, 0, st>>>(hist + RADIX * p, count_ptr, cap,
                                                                                 (int)tile, pcnt);
      HGS_CHECK_LAUNCH();
      poff = pcnt;
    }
    launch_pdl(radix_pass_kernel<K, IPT>, dim3(g), dim3(RS_THREADS), smem, st, kin,
               (const uint32_t*)(p == 0 && implicit_vals ? nullptr : vin), kout, vdst, count_ptr, cap, shift0 + 8 * p,
                                                      (const uint32_t*)(hist + RADIX * p), status + (size_t)p * parts * RADIX, (int)parts,
                                                      part_ctr + p, (!last || last_keys) ? 1 : 0, (const uint32_t*)poff, pnext);
    HGS_CHECK_LAUNCH();
    std::swap(kin, kout);
    vin = vdst;
    vout = (vdst == v1) ? v0 : v1;
  }
  if (keys_result) *keys_result = kin;
  if (vals_result) *vals_result = vin;
  return HGS_OK;
}

}  // namespace hgs

// The fine binning kernel's entry point (hgs_graph_instantiate restores its
// programmatic edge to the blend, abi.cu)
const void* hgs_fine_bin_fn() { return (const void*)hgs::fine_bin_kernel<4>; }

extern "C" size_t hgs_tiles_scratch_bytes(int64_t n, int64_t capacity, int32_t n_tiles) {
  // n_tiles is an upper bound on tiles_x * tiles_y; size the difference grid
  // for the worst aspect ratio (tiles_x + 1) * (tiles_y + 1) <= 2 * n_tiles + 1
  // any grid of n_tiles tiles has at most ceil(n_tiles / 4) super-tiles of 4 x 4 (or is not binned):
  // size the binning arrays whenever some aspect ratio could be binned
  const bool may_bin = n_tiles <= 16 * hgs::BIN_MAX_SUPER * 16;
  return hgs::carve(n, capacity, n_tiles, 1, nullptr, nullptr, may_bin ? 1 : hgs::BIN_MAX_SUPER + 1) +
         8 * (size_t)n_tiles + 4096;
}

extern "C" int hgs_build_tiles(const hgs_projected* proj, int64_t n, hgs_tiles* tiles, void* stream) {
  using namespace hgs;
  if (!proj || !tiles) return hgs_set_error(HGS_ERR_INVALID, "hgs_build_tiles: null argument");
  if (!tiles->entries || !tiles->tile_starts || !tiles->counters)
    return hgs_set_error(HGS_ERR_INVALID, "hgs_build_tiles: missing output pointer");
  if (tiles->tiles_x <= 0 || tiles->tiles_y <= 0) return hgs_set_error(HGS_ERR_INVALID, "hgs_build_tiles: empty tile grid");
  if (!proj->count || !proj->rect || !proj->rec || !proj->sort_keys || !proj->tile_diff)
    return hgs_set_error(HGS_ERR_INVALID, "hgs_build_tiles: projection needs count, rect, rec, sort_keys, tile_diff");
  const int tx = tiles->tiles_x, ty = tiles->tiles_y;
  const int n_tiles = tx * ty;
  if (n > 0xffffffffLL || tiles->capacity > (1LL << 30) || n_tiles > (1 << 24))
    return hgs_set_error(HGS_ERR_INVALID, "hgs_build_tiles: n, capacity or tile grid too large");
  const size_t need = carve(n, tiles->capacity, tx, ty, nullptr, nullptr);
  if (!tiles->scratch || tiles->scratch_bytes < need)
    return hgs_set_error(HGS_ERR_INVALID, "hgs_build_tiles: scratch too small (see hgs_tiles_scratch_bytes)");
  cudaStream_t st = (cudaStream_t)stream;
  TilesScratch s;
  carve(n, tiles->capacity, tx, ty, (unsigned char*)tiles->scratch, &s);
  tiles->coarse_rows = s.crow;
  tiles->coarse_rects = s.crect;
  tiles->coarse_starts = s.cstart;
  tiles->coarse_prog = s.cprog;
  zero_pdl(st, s.control_begin, s.control_bytes, tiles->counters, 4 * sizeof(int64_t));
  HGS_CHECK_LAUNCH();
  // 1. order-preserving compaction of the visible rows' depth keys
  static int scan_grid_cap = 0;
  if (scan_grid_cap == 0) scan_grid_cap = persistent_grid((const void*)compact_kernel, SCAN_THREADS, 0);
  const int scan_grid = (int)tmax<int64_t>(1, tmin<int64_t>(scan_grid_cap, (n + SCAN_TILE - 1) / SCAN_TILE));
  if (n > 0 && HGS_DEPTH_MODE != 0) {
    launch_pdl(depth_stats_kernel, dim3(2 * sm_count()), dim3(256), 0, st, (const uint64_t*)proj->sort_keys, n,
               tiles->counters, reinterpret_cast<unsigned long long*>(s.part_ctr + 24),
               HGS_DEPTH_MODE == 2 ? s.vis_cnt : (uint32_t*)nullptr);
    HGS_CHECK_LAUNCH();
  } else if (n > 0) {
    launch_pdl(compact_kernel, dim3(scan_grid), dim3(SCAN_THREADS), 0, st, proj->sort_keys, n, s.dk[0], s.dv[0], s.scan_status,
                                                       s.part_ctr + 20, tiles->counters,
                                                       reinterpret_cast<unsigned long long*>(s.part_ctr + 24));
    HGS_CHECK_LAUNCH();
  }
  // 2. per-tile counts -> tile_starts, K, overflow, tile-key histograms
  const bool blend_only = (tiles->flags & HGS_TILES_BLEND_ONLY) != 0;
  const int ss_all = super_shift(tx, ty, blend_only);
  const int n_quads_all = ss_all >= 0 ? (((tx + (1 << ss_all) - 1) >> ss_all) * ((ty + (1 << ss_all) - 1) >> ss_all))
                                            << (2 * (ss_all - 2))
                                      : 0;
  const size_t grid_bytes = sizeof(int) * (size_t)(tx + 1) * (size_t)(ty + 1);
  const int tc_global = grid_bytes > 200 * 1024 ? 1 : 0;  // prefix sums in global memory for huge grids
  const size_t grid_smem = tc_global ? 0 : grid_bytes;
  static bool tc_attr = false;
  if (!tc_attr) {
    cudaFuncSetAttribute(tile_counts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    tc_attr = true;
  }
  launch_pdl(tile_counts_kernel, dim3(1), dim3(1024), grid_smem, st, proj->tile_diff, tx, ty, tiles->capacity, tiles->tile_starts,
                                                 tiles->counters, ss_all >= 0 ? (uint32_t*)nullptr : s.hist + 8 * RADIX,
                                                 tc_global, (int*)tiles->ready,
                                                 n == 0 && ss_all >= 0 ? n_quads_all : 0);
  HGS_CHECK_LAUNCH();
  auto join = [&]() -> int {  // the caller's independent branch joins the stream (hgs.h join_event)
    if (!tiles->join_event) return HGS_OK;
    const cudaError_t e = cudaStreamWaitEvent(st, (cudaEvent_t)tiles->join_event, 0);
    return e == cudaSuccess ? HGS_OK : hgs_set_cuda_error(e, __FILE__, __LINE__);
  };
  if (n == 0) return join();
  // 3. stable sort of the visible rows by fp64 depth bits (result in dk[0]/dv[0])
  // order-preserving remap of the depth keys to DEPTH_KEY_BITS, LSD passes, exact fix-up of truncation ties
  uint32_t* k32a = reinterpret_cast<uint32_t*>(s.dk[1]);
  uint32_t* k32b = k32a + ((n + 3) & ~(int64_t)3);  // 16-B aligned: the radix passes stage their input with cp.async
  unsigned long long* minmax = reinterpret_cast<unsigned long long*>(s.part_ctr + 24);
  const bool rts = HGS_SORT_RTS != 0;
  const bool all = HGS_SORT_ALL;  // every row sorted (culled ones last) instead of the compacted visible rows
  if (HGS_DEPTH_MODE == 2) {
    launch_pdl(depth_compact_remap_kernel, dim3(4 * sm_count()), dim3(256), 0, st, (const uint64_t*)proj->sort_keys, n,
               (const unsigned long long*)minmax, (const uint32_t*)s.vis_cnt, k32a, s.dv[0], s.hist,
               rts ? s.rs_status : (uint32_t*)nullptr);
  } else {
    launch_pdl(depth_remap_kernel, dim3(4 * sm_count()), dim3(256), 0, st,
               all ? (const uint64_t*)proj->sort_keys : s.dk[0], tiles->counters, minmax, k32a, s.hist,
               rts ? s.rs_status : (uint32_t*)nullptr, all ? n : (int64_t)-1);
  }
  HGS_CHECK_LAUNCH();
  uint32_t* k32res = nullptr;
  uint32_t* rows = nullptr;  // visible rows in (depth, row) order (then the culled ones)
  int rc = radix_sort<uint32_t, RS_DEPTH_IPT>(k32a, k32b, s.dv[0], s.dv[1], nullptr, all ? nullptr : tiles->counters, n,
                                              0, DEPTH_KEY_BITS / 8, s.hist, true, s.rs_status, s.parts_n, s.part_ctr,
                                              st, &k32res, true, &rows, nullptr, rts, all);
  if (rc) return rc;
  launch_pdl(
#if HGS_FIXUP_V2
      depth_fixup_kernel,
#else
      depth_fixup_v1_kernel,
#endif
      dim3(4 * sm_count()), dim3(256), 0, st, k32res, rows, (const uint64_t*)proj->sort_keys, tiles->counters,
                                                     minmax);
  HGS_CHECK_LAUNCH();
  const int ss = super_shift(tx, ty, blend_only);
  if (ss >= 0) {
    // 4. two-level rect binning straight into the final (tile, depth, row) order
    const int sx = (tx + (1 << ss) - 1) >> ss, sy = (ty + (1 << ss) - 1) >> ss, n_super = sx * sy;
    const int pblk = (int)((n + PREP_ROWS - 1) / PREP_ROWS);  // upper bound: kernels read m on the device
#if HGS_PREP_3K
    launch_pdl(coarse_prep_sum_kernel, dim3(pblk), dim3(256), 0, st, rows, (const ushort4*)proj->rect, tiles->counters, ss, s.rsort,
                                                 s.bsum);
    HGS_CHECK_LAUNCH();
    launch_pdl(coarse_prep_scan_kernel, dim3(1), dim3(1024), 0, st, tiles->counters, s.bsum, s.npairs);
    HGS_CHECK_LAUNCH();
    launch_pdl(coarse_prep_offsets_kernel, dim3(pblk), dim3(256), 0, st, s.rsort, tiles->counters, ss, s.bsum, s.npairs, s.pair_off,
                                                     s.wstart);
    HGS_CHECK_LAUNCH();
#else
    // (the second half of scan_status and part_ctr[21] belong to offsets_kernel, unused on this path)
    static int prep_cap = 0;
    if (prep_cap == 0) prep_cap = persistent_grid((const void*)coarse_prep_kernel, SCAN_THREADS, 0);
    launch_pdl(coarse_prep_kernel, dim3((int)tmax<int64_t>(1, tmin<int64_t>(prep_cap, pblk))), dim3(SCAN_THREADS), 0, st,
               (const uint32_t*)rows, (const ushort4*)proj->rect, (const int64_t*)tiles->counters, ss, s.rsort,
               s.pair_off, s.wstart, s.npairs, s.scan_status + s.parts_n + 1, s.part_ctr + 21);
    HGS_CHECK_LAUNCH();
#endif
    CoarseArgs ca{rows, s.rsort, s.pair_off, s.wstart, s.npairs, tiles->counters, tiles->capacity, ss, sx, n_super};
    static int cgrid = 0, sgrid = 0, sgrid_ns = -1;
    const size_t ssmem = scatter_smem_bytes(n_super);
    if (cgrid == 0) {
      cgrid = persistent_grid((const void*)coarse_count_kernel, BIN_THREADS, 0);
      cudaFuncSetAttribute(coarse_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)scatter_smem_bytes(BIN_MAX_SUPER));
    }
    if (sgrid_ns != n_super) {  // occupancy depends on the super-tile count
      sgrid = persistent_grid((const void*)coarse_scatter_kernel, BIN_THREADS, ssmem);
      sgrid_ns = n_super;
    }
    launch_pdl(coarse_count_kernel, dim3(cgrid), dim3(BIN_THREADS), 0, st, ca, s.bin_mat, s.bin_wmat, s.chist);
    HGS_CHECK_LAUNCH();
    launch_pdl(coarse_scan_kernel, dim3((n_super + 31) / 32), dim3(1024), 0, st, s.bin_mat, s.chist, tiles->counters, tiles->capacity,
                                                             s.npairs, n_super, s.cstart, s.bin_slot);
    HGS_CHECK_LAUNCH();
    launch_pdl(coarse_scatter_kernel, dim3(sgrid), dim3(BIN_THREADS), ssmem, st, ca, s.bin_mat, s.bin_slot, s.bin_wmat,
                                                                          s.crow, s.crect);
    HGS_CHECK_LAUNCH();
    if (ss != 2 && ss != 3) return hgs_set_error(HGS_ERR_INVALID, "hgs_build_tiles: tile grid too large for binning");
    if (const int jr = join()) return jr;  // before the fine binning: the blend then depends on it alone
    // blend-only bins: the blend reads the coarse lists itself (no entries)
    if (tiles->flags & HGS_TILES_BLEND_ONLY) return HGS_OK;
    // 8x8 super-tiles: four 4x4-tile CTAs each (parallelism at 1080p)
    launch_pdl(fine_bin_kernel<4>, dim3(n_super << (2 * (ss - 2))), dim3(fine_warps(4) * 32), 0, st, s.crow,
               s.crect, s.cstart, tiles->tile_starts, tiles->counters, tiles->capacity, tx, ty, sx, tiles->entries,
               ss - 2, (int*)tiles->ready);
    HGS_CHECK_LAUNCH();
    return HGS_OK;
  }
  // 4. offsets of each row's entries in depth order
  offsets_kernel<<<scan_grid, SCAN_THREADS, 0, st>>>(proj->count, rows, tiles->counters, s.offsets,
                                                     s.scan_status + s.parts_n + 1, s.part_ctr + 21, tiles->counters,
                                                     tiles->capacity);
  HGS_CHECK_LAUNCH();
  // 5-6. emission in depth order, stable tile-key sort
  int bits = 1;
  while ((1 << bits) < n_tiles) bits++;
  const int tpasses = (bits + 7) / 8;
  uint32_t* rs_tile_status = s.rs_tile_status;
  if (tpasses > 3) return hgs_set_error(HGS_ERR_INVALID, "hgs_build_tiles: more than 2^24 tiles");
  zero_pdl(st, rs_tile_status, sizeof(uint32_t) * RADIX * (size_t)tpasses * s.parts_k);
  HGS_CHECK_LAUNCH();
  if (n_tiles > 65535) {
    emit_kernel<uint32_t><<<4 * sm_count(), 256, 0, st>>>(rows, s.offsets, (const ushort4*)proj->rect,
                                                          tiles->counters, tx, tiles->capacity, (uint32_t*)s.tk[0],
                                                          s.tv0, s.big_rows, s.part_ctr + 22);
    HGS_CHECK_LAUNCH();
    emit_big_kernel<uint32_t><<<2 * sm_count(), 256, 0, st>>>(rows, s.offsets, (const ushort4*)proj->rect,
                                                              tiles->counters, tx, tiles->capacity, (uint32_t*)s.tk[0],
                                                              s.tv0, s.big_rows, s.part_ctr + 22);
    HGS_CHECK_LAUNCH();
    rc = radix_sort<uint32_t>((uint32_t*)s.tk[0], (uint32_t*)s.tk[1], s.tv0, s.tv1, tiles->entries,
                              tiles->counters + 1, tiles->capacity, 0, tpasses, s.hist + 8 * RADIX, true, rs_tile_status,
                              s.parts_k, s.part_ctr + 8, st, nullptr, false);
  } else {
    emit_kernel<uint16_t><<<4 * sm_count(), 256, 0, st>>>(rows, s.offsets, (const ushort4*)proj->rect,
                                                          tiles->counters, tx, tiles->capacity, (uint16_t*)s.tk[0],
                                                          s.tv0, s.big_rows, s.part_ctr + 22);
    HGS_CHECK_LAUNCH();
    emit_big_kernel<uint16_t><<<2 * sm_count(), 256, 0, st>>>(rows, s.offsets, (const ushort4*)proj->rect,
                                                              tiles->counters, tx, tiles->capacity, (uint16_t*)s.tk[0],
                                                              s.tv0, s.big_rows, s.part_ctr + 22);
    HGS_CHECK_LAUNCH();
    rc = radix_sort<uint16_t>((uint16_t*)s.tk[0], (uint16_t*)s.tk[1], s.tv0, s.tv1, tiles->entries,
                              tiles->counters + 1, tiles->capacity, 0, tpasses, s.hist + 8 * RADIX, true, rs_tile_status,
                              s.parts_k, s.part_ctr + 8, st, nullptr, false);
  }
  if (rc == HGS_OK) rc = join();
  return rc;
}
