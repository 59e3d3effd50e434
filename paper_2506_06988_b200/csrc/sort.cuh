// Device-wide primitives for tile binning: a single-pass chained scan and a
// stable LSD radix sort (8-bit digits, one kernel per pass), both with
// decoupled look-back and dynamic partition assignment so that every count
// can stay on the device (no host round trip between stages).
//
// Radix pass: 256 threads x IPT items per partition (the depth sort uses
// IPT = 8: 2048 keys, 3 passes over 24-bit keys).  Ranking is
// warp-level multisplit (8 ballots per key) with per-warp digit counters in
// shared memory, which preserves input order inside a partition (stability);
// partitions are ordered by their dynamically assigned id, and the look-back
// over predecessor partitions gives each digit's global offset.  Items are
// staged in shared memory in sorted order and written out digit-run by
// digit-run, so global stores are coalesced.
#pragma once
#include "common.cuh"

namespace hgs {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_IPT = 16;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_IPT;

constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_IPT = 16;
constexpr int RS_TILE = RS_THREADS * RS_IPT;
constexpr int RADIX = 256;

constexpr uint64_t SCAN_FLAG_AGG = 1ull << 62;
constexpr uint64_t SCAN_FLAG_INC = 2ull << 62;
constexpr uint64_t SCAN_VALUE_MASK = (1ull << 62) - 1;

constexpr uint32_t SPIN_LIMIT = 1u << 24;
#ifndef HGS_LB_WINDOW
#define HGS_LB_WINDOW 16
#endif
constexpr int LB_WINDOW = HGS_LB_WINDOW;  // predecessors read per look-back round trip
constexpr uint32_t RS_FLAG_AGG = 1u << 30;
constexpr uint32_t RS_FLAG_INC = 2u << 30;
constexpr uint32_t RS_VALUE_MASK = (1u << 30) - 1;

__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}


// Chained-scan partition: every thread owns SCAN_IPT consecutive items.
// Given per-item values, returns the exclusive prefix of each item and the
// grand total (valid in the last partition).  status: one u64 per partition.
template <typename F>
__device__ __forceinline__ void chained_scan_partition(int part, int64_t n, F value_of, uint64_t* status,
                                                       uint64_t* item_excl /*[SCAN_IPT]*/, uint64_t& grand_total) {
  __shared__ uint64_t s_warp[8];
  __shared__ uint64_t s_prefix;
  const int64_t base = (int64_t)part * SCAN_TILE + (int64_t)threadIdx.x * SCAN_IPT;
  uint64_t vals[SCAN_IPT];
  uint64_t tsum = 0;
#pragma unroll
  for (int j = 0; j < SCAN_IPT; j++) {
    const int64_t i = base + j;
    vals[j] = i < n ? value_of(i) : 0;
    tsum += vals[j];
  }
  uint64_t agg;
  uint64_t texcl = block_exclusive_scan<uint64_t>(tsum, s_warp, agg);
  if (threadIdx.x < 32) {
    // warp-wide decoupled look-back: 32 predecessors per round trip
    const int lane = threadIdx.x;
    uint64_t excl = 0;
    if (part == 0) {
      if (lane == 0) st_relaxed(&status[0], SCAN_FLAG_INC | agg);
    } else {
      if (lane == 0) st_relaxed(&status[part], SCAN_FLAG_AGG | agg);
      int p = part - 1;
      for (uint32_t spin = 0; spin <= SPIN_LIMIT; spin++) {  // watchdog: never hang the GPU
        const int q = p - lane;
        const uint64_t sv = q >= 0 ? ld_relaxed(&status[q]) : SCAN_FLAG_INC;
        const uint64_t flag = sv & ~SCAN_VALUE_MASK;
        const unsigned notready = __ballot_sync(0xffffffffu, flag == 0);
        const unsigned inc = __ballot_sync(0xffffffffu, flag == SCAN_FLAG_INC);
        const int first_inc = inc ? __ffs(inc) - 1 : 32;
        const int first_nr = notready ? __ffs(notready) - 1 : 32;
        const int take = first_nr < first_inc ? first_nr : (first_inc < 32 ? first_inc + 1 : 32);
        uint64_t v = lane < take ? (sv & SCAN_VALUE_MASK) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (first_inc < first_nr && first_inc < 32) break;
        p -= take;
      }
      if (lane == 0) st_relaxed(&status[part], SCAN_FLAG_INC | (excl + agg));
    }
    if (lane == 0) s_prefix = excl;
  }
  __syncthreads();
  const uint64_t pre = s_prefix + texcl;
  uint64_t run = pre;
#pragma unroll
  for (int j = 0; j < SCAN_IPT; j++) {
    item_excl[j] = run;
    run += vals[j];
  }
  grand_total = s_prefix + agg;
  __syncthreads();
}

// Lanes of `active` holding the same BITS-bit value v: one ballot per bit
// (MATCH.ANY on a warp of mostly distinct values is a long-latency
// multi-pass instruction; this is BITS votes + selects)
template <int BITS>
__device__ __forceinline__ unsigned warp_peers(uint32_t v, unsigned active) {
  unsigned peers = active;
#pragma unroll
  for (int b = 0; b < BITS; b++) {
    const unsigned bb = __ballot_sync(0xffffffffu, (v >> b) & 1u);
    peers &= ((v >> b) & 1u) ? bb : ~bb;
  }
  return peers;
}

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K k, int shift) {
  return (uint32_t)((k >> shift) & (K)(RADIX - 1));
}

// Histograms of `npasses` consecutive 8-bit digits starting at shift0.
template <typename K>
__global__ void __launch_bounds__(256) radix_hist_kernel(const K* __restrict__ keys, const int64_t* count_ptr,
                                                         int64_t cap, int shift0, int npasses, uint32_t* hist) {
  __shared__ uint32_t sh[8][RADIX];
  for (int i = threadIdx.x; i < 8 * RADIX; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  int64_t n = count_ptr ? *count_ptr : cap;
  if (n > cap) n = cap;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t nround = (n + stride - 1) / stride * stride;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nround; i += stride) {
    const bool valid = i < n;
    const K k = valid ? keys[i] : K(0);
    if (!valid) continue;
    for (int p = 0; p < npasses; p++) atomicAdd(&sh[p][digit_of<K>(k, shift0 + 8 * p)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < npasses * RADIX; i += blockDim.x) {
    uint32_t c = (&sh[0][0])[i];
    if (c) atomicAdd(&hist[i], c);
  }
}

// Reduce-then-scan variant of an LSD pass (no look-back chain: for a
// million keys the decoupled look-back's frontier latency dominates).
// Upsweep: per-partition digit counts -> pcnt[part][256].
template <typename K, int IPT>
__global__ void __launch_bounds__(RS_THREADS) radix_upsweep_kernel(const K* __restrict__ kin, const int64_t* count_ptr,
                                                                   int64_t cap, int shift, uint32_t* __restrict__ pcnt) {
  __shared__ uint32_t h[RS_WARPS][RADIX];
  constexpr int TILE = RS_THREADS * IPT;
  int64_t n = count_ptr ? *count_ptr : cap;
  if (n > cap) n = cap;
  const int64_t base = (int64_t)blockIdx.x * TILE;
  if (base >= n) return;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < RS_WARPS * RADIX; i += RS_THREADS) (&h[0][0])[i] = 0;
  __syncthreads();
#pragma unroll
  for (int j = 0; j < IPT; j++) {
    const int64_t i = base + (int64_t)j * RS_THREADS + threadIdx.x;
    if (i < n) atomicAdd(&h[warp][digit_of<K>(kin[i], shift)], 1u);
  }
  __syncthreads();
  uint32_t c = 0;
#pragma unroll
  for (int w = 0; w < RS_WARPS; w++) c += h[w][threadIdx.x];
  pcnt[(size_t)blockIdx.x * RADIX + threadIdx.x] = c;
}

// Scan: poff[part][d] = digit base (from the pass histogram) + counts of d
// in the earlier partitions.  16 CTAs x 16 digits; 64 partition groups per
// digit (each thread sums a short, independent run of partitions).
constexpr int RSCAN_DIGITS = 16, RSCAN_GROUPS = 64;
__global__ void __launch_bounds__(RSCAN_DIGITS * RSCAN_GROUPS) radix_scan_kernel(const uint32_t* __restrict__ hist,
                                                                                const int64_t* count_ptr, int64_t cap,
                                                                                int tile, uint32_t* __restrict__ pcnt) {
  __shared__ uint32_t s_sum[RSCAN_GROUPS][RSCAN_DIGITS + 1];
  __shared__ uint32_t s_base[RSCAN_DIGITS];
  pdl_enter();
  int64_t n = count_ptr ? *count_ptr : cap;
  if (n > cap) n = cap;
  const int nparts = (int)((n + tile - 1) / tile);
  const int dl = threadIdx.x % RSCAN_DIGITS, grp = threadIdx.x / RSCAN_DIGITS;
  const int d = blockIdx.x * RSCAN_DIGITS + dl;
  if (threadIdx.x < 32) {  // bases of this CTA's digits: histogram sums below them
    const int lane = threadIdx.x;
    uint32_t below = 0;
    for (int t = lane; t < blockIdx.x * RSCAN_DIGITS; t += 32) below += hist[t];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) below += __shfl_xor_sync(0xffffffffu, below, o);
    const uint32_t h = lane < RSCAN_DIGITS ? hist[blockIdx.x * RSCAN_DIGITS + lane] : 0u;
    uint32_t x = h;
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane < RSCAN_DIGITS) s_base[lane] = below + x - h;
  }
  const int per = (nparts + RSCAN_GROUPS - 1) / RSCAN_GROUPS;
  const int p0 = grp * per, p1 = min(nparts, p0 + per);
  uint32_t sum = 0;
#pragma unroll 4
  for (int p = p0; p < p1; p++) sum += pcnt[(size_t)p * RADIX + d];
  s_sum[grp][dl] = sum;
  __syncthreads();
  uint32_t run = s_base[dl];
  for (int g = 0; g < grp; g++) run += s_sum[g][dl];
#pragma unroll 4
  for (int p = p0; p < p1; p++) {
    const uint32_t c = pcnt[(size_t)p * RADIX + d];
    pcnt[(size_t)p * RADIX + d] = run;
    run += c;
  }
}

// 16-byte global -> shared copy; bytes < 16 zero-fills the rest (0: none read)
__device__ __forceinline__ void cp_async16_zfill(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src),
               "r"(bytes)
               : "memory");
}

template <typename K, int IPT = RS_IPT>
struct RadixSmem {
  K keys[RS_THREADS * IPT];
  uint32_t vals[RS_THREADS * IPT];
};

// One stable LSD pass over the digit at `shift`.
template <typename K, int IPT>
__global__ void __launch_bounds__(RS_THREADS, IPT <= 8 ? 4 : (sizeof(K) == 8 ? 2 : 3)) radix_pass_kernel(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                                K* __restrict__ kout, uint32_t* __restrict__ vout,
                                                                const int64_t* count_ptr, int64_t cap, int shift,
                                                                const uint32_t* __restrict__ hist, uint32_t* status,
                                                                int nparts_cap, uint32_t* part_ctr, int write_keys,
                                                                const uint32_t* __restrict__ poff = nullptr,
                                                                uint32_t* __restrict__ pcnt_next = nullptr) {
  pdl_enter();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  RadixSmem<K, IPT>& sm = *reinterpret_cast<RadixSmem<K, IPT>*>(smem_raw);
  constexpr int TILE = RS_THREADS * IPT;
  __shared__ uint32_t whist[RS_WARPS][RADIX];
  __shared__ uint32_t s_digit_base[RADIX];
  __shared__ uint32_t s_gstart[RADIX];
  __shared__ uint32_t s_lstart[RADIX];
  __shared__ uint32_t s_warp[8];
  __shared__ int s_part;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int64_t n = count_ptr ? *count_ptr : cap;
  if (n > cap) n = cap;
  const int nparts = (int)((n + TILE - 1) / TILE);
  {
    uint32_t tot;
    uint32_t e = block_exclusive_scan<uint32_t>(hist[tid], s_warp, tot);
    s_digit_base[tid] = e;
  }
  int iter = 0;
  while (true) {
    // reduce-then-scan mode: static partitions (offsets are precomputed)
    if (tid == 0) s_part = poff ? (int)blockIdx.x + iter * (int)gridDim.x : (int)atomicAdd(part_ctr, 1u);
    iter++;
    for (int i = tid; i < RS_WARPS * RADIX; i += RS_THREADS) (&whist[0][0])[i] = 0;
    __syncthreads();
    const int part = s_part;
    if (part >= nparts) break;
    const int64_t base = (int64_t)part * TILE;
    const int tile_n = (int)tmin<int64_t>(TILE, n - base);

    // the partition's keys and values are staged in shared memory with
    // every copy in flight at once (loaded into registers directly, ptxas
    // sinks the loads into the ranking loop under the 64-register cap and
    // pays the L2 latency item by item)
    {
      constexpr int KV = 16 / (int)sizeof(K);
      for (int c = tid; c < TILE / KV; c += RS_THREADS) {
        const int nv = tile_n - c * KV;
        cp_async16_zfill(&sm.keys[c * KV], kin + base + (nv > 0 ? c * KV : 0), nv <= 0 ? 0u : (unsigned)(min(nv, KV) * sizeof(K)));
      }
      if (vin)  // (NULL: the values are the input positions)
        for (int c = tid; c < TILE / 4; c += RS_THREADS) {
          const int nv = tile_n - c * 4;
          cp_async16_zfill(&sm.vals[c * 4], vin + base + (nv > 0 ? c * 4 : 0), nv <= 0 ? 0u : (unsigned)(min(nv, 4) * 4));
        }
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncthreads();
    }
    K k[IPT];
    uint32_t v[IPT];
    uint32_t rank[IPT];
#pragma unroll
    for (int j = 0; j < IPT; j++) {
      const int li = warp * (IPT * 32) + j * 32 + lane;
      k[j] = sm.keys[li];
      v[j] = vin ? sm.vals[li] : (uint32_t)(base + li);
    }
#pragma unroll
    for (int j = 0; j < IPT; j++) {
      const int li = warp * (IPT * 32) + j * 32 + lane;
      const bool valid = li < tile_n;
      const unsigned active = __ballot_sync(0xffffffffu, valid);
      uint32_t d = 0, peers = 0, base_cnt = 0;
      if (valid) d = digit_of<K>(k[j], shift);
      peers = warp_peers<8>(d, active);
      if (valid) {
        base_cnt = whist[warp][d];
        rank[j] = base_cnt + __popc(peers & lanemask_lt());
      }
      __syncwarp();
      if (valid && lane == __ffs(peers) - 1) whist[warp][d] = base_cnt + __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    // per digit: exclusive prefix over warps, block count
    uint32_t cnt = 0;
#pragma unroll
    for (int w = 0; w < RS_WARPS; w++) {
      uint32_t c = whist[w][tid];
      whist[w][tid] = cnt;
      cnt += c;
    }
    if (poff) {
      s_gstart[tid] = poff[(size_t)part * RADIX + tid];
    } else {
    // decoupled look-back for this digit: status is [partition][digit] (a
    // warp's 32 digits are one 128 B line); each round trip reads a window of
    // 16 predecessors (independent coalesced loads)
    {
      uint32_t* st = status + tid;
      uint32_t excl = 0;
      if (part == 0) {
        st_relaxed(st, RS_FLAG_INC | cnt);
      } else {
        st_relaxed(st + (size_t)part * RADIX, RS_FLAG_AGG | cnt);
        int p = part - 1;
        bool fin = false;
        while (!fin) {
          // wait (one load per poll) until the nearest unread predecessor is
          // published, then read a window of LB_WINDOW and consume its ready prefix
          for (uint32_t spin = 0; (ld_relaxed(st + (size_t)p * RADIX) & ~RS_VALUE_MASK) == 0; spin++)
            if (spin > SPIN_LIMIT) { fin = true; break; }  // watchdog: never hang the GPU
          if (fin) break;
          uint32_t w[LB_WINDOW];
#pragma unroll
          for (int k = 0; k < LB_WINDOW; k++)
            w[k] = (p - k >= 0) ? ld_relaxed(st + (size_t)(p - k) * RADIX) : RS_FLAG_INC;
          int used = 0;
#pragma unroll
          for (int k = 0; k < LB_WINDOW; k++) {
            if (fin || used < k) continue;  // stopped earlier in this window
            const uint32_t flag = w[k] & ~RS_VALUE_MASK;
            if (flag == 0) continue;        // not ready: re-read from here
            excl += w[k] & RS_VALUE_MASK;
            used = k + 1;
            if (flag == RS_FLAG_INC) fin = true;
          }
          p -= used;
        }
        st_relaxed(st + (size_t)part * RADIX, RS_FLAG_INC | (excl + cnt));
      }
      s_gstart[tid] = s_digit_base[tid] + excl;
    }
    }
    {
      uint32_t tot;
      s_lstart[tid] = block_exclusive_scan<uint32_t>(cnt, s_warp, tot);
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < IPT; j++) {
      const int li = warp * (IPT * 32) + j * 32 + lane;
      if (li < tile_n) {
        const uint32_t d = digit_of<K>(k[j], shift);
        const uint32_t pos = s_lstart[d] + whist[warp][d] + rank[j];
        sm.keys[pos] = k[j];
        sm.vals[pos] = v[j];
      }
    }
    __syncthreads();
    for (int i = tid; i < tile_n; i += RS_THREADS) {
      const K key = sm.keys[i];
      const uint32_t d = digit_of<K>(key, shift);
      const uint32_t out = s_gstart[d] + (uint32_t)i - s_lstart[d];
      if (write_keys) kout[out] = key;
      vout[out] = sm.vals[i];
      // reduce-then-scan: the next pass's per-partition digit counts, so that
      // pass needs no upsweep over its input
      if (pcnt_next) atomicAdd(&pcnt_next[(size_t)(out / TILE) * RADIX + digit_of<K>(key, shift + 8)], 1u);
    }
    __syncthreads();
  }
}

}  // namespace hgs
