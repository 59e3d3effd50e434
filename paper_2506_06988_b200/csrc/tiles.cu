// K2 tile binning: build_tiles (gsmesh/splat/tiles.py:35-69).
//
// The reference orders tile entries with np.lexsort((kept, depth, tile))
// (tiles.py:65).  Here:
//   1. compact the visible rows (count > 0) in row order       (chained scan)
//   2. sort them by the fp64 depth bit pattern, stably         (8 LSD passes)
//      -> visible rows in (depth, row) order
//   3. exclusive scan of their tile counts in that order        (chained scan)
//   4. emit (tile id, row) pairs in depth order                 (1 thread/row)
//   5. stable LSD sort by tile id (1-2 passes of 8 bits)
//      -> (tile, depth, row) order == the reference's lexsort, exactly
//   6. CSR tile ranges from the sorted tile ids.
// Positive doubles order like their IEEE bit patterns, so step 2 is exact.
#include "sort.cuh"

namespace hgs {

__global__ void __launch_bounds__(SCAN_THREADS) compact_kernel(const int32_t* __restrict__ count,
                                                               const BlendRec* __restrict__ rec, int64_t n,
                                                               uint64_t* dkeys, uint32_t* dvals, uint64_t* status,
                                                               uint32_t* part_ctr, int64_t* counters) {
  __shared__ int s_part;
  const int nparts = (int)((n + SCAN_TILE - 1) / SCAN_TILE);
  while (true) {
    if (threadIdx.x == 0) s_part = (int)atomicAdd(part_ctr, 1u);
    __syncthreads();
    const int part = s_part;
    __syncthreads();
    if (part >= nparts) break;
    uint64_t excl[SCAN_IPT];
    uint64_t total;
    chained_scan_partition(part, n, [&](int64_t i) -> uint64_t { return count[i] > 0 ? 1ull : 0ull; }, status,
                           excl, total);
    const int64_t base = (int64_t)part * SCAN_TILE + (int64_t)threadIdx.x * SCAN_IPT;
#pragma unroll
    for (int j = 0; j < SCAN_IPT; j++) {
      const int64_t i = base + j;
      if (i < n && count[i] > 0) {
        dkeys[excl[j]] = (uint64_t)__double_as_longlong(rec[i].depth);
        dvals[excl[j]] = (uint32_t)i;
      }
    }
    if (part == nparts - 1 && threadIdx.x == 0) counters[0] = (int64_t)total;
  }
}

__global__ void __launch_bounds__(SCAN_THREADS) offsets_kernel(const int32_t* __restrict__ count,
                                                               const uint32_t* __restrict__ sorted_rows,
                                                               const int64_t* counters_in, uint32_t* offsets,
                                                               uint64_t* status, uint32_t* part_ctr,
                                                               int64_t* counters, int64_t capacity) {
  __shared__ int s_part;
  const int64_t m = counters_in[0];
  const int nparts = (int)((m + SCAN_TILE - 1) / SCAN_TILE);
  if (m == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) counters[1] = 0;
    return;
  }
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
    if (part == nparts - 1 && threadIdx.x == 0) {
      counters[1] = (int64_t)total;
      counters[2] = (int64_t)total > capacity ? 1 : 0;
    }
  }
}

// One thread per visible row in depth order; writes its tile ids row-major
// over the rectangle (the order inside one row is irrelevant: distinct keys).
template <typename TK>
__global__ void __launch_bounds__(256) emit_kernel(const uint32_t* __restrict__ sorted_rows,
                                                   const uint32_t* __restrict__ offsets,
                                                   const ushort4* __restrict__ rect, const int64_t* counters,
                                                   int tiles_x, int64_t capacity, TK* tkeys, uint32_t* tvals) {
  const int64_t m = counters[0];
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t g = sorted_rows[j];
    int64_t o = offsets[j];
    const ushort4 rc = rect[g];
    for (int ty = rc.z; ty <= rc.w; ty++)
      for (int tx = rc.x; tx <= rc.y; tx++) {
        if (o < capacity) {
          tkeys[o] = (TK)(ty * tiles_x + tx);
          tvals[o] = g;
        }
        o++;
      }
  }
}

template <typename TK>
__global__ void __launch_bounds__(256) ranges_kernel(const TK* __restrict__ tkeys, const int64_t* counters,
                                                     int64_t capacity, int n_tiles, int64_t* tile_starts) {
  int64_t k = counters[1];
  if (k > capacity) k = capacity;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (k == 0) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n_tiles; i += stride) tile_starts[i] = 0;
    return;
  }
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < k; p += stride) {
    const int64_t t = tkeys[p];
    const int64_t prev = p > 0 ? (int64_t)tkeys[p - 1] : -1;
    for (int64_t tt = prev + 1; tt <= t; tt++) tile_starts[tt] = p;
    if (p == k - 1)
      for (int64_t tt = t + 1; tt <= n_tiles; tt++) tile_starts[tt] = k;
  }
}

// ---------------------------------------------------------------- host side

struct TilesScratch {
  uint64_t* dk[2];
  uint32_t* dv[2];
  uint32_t* offsets;
  void* tk[2];
  uint32_t* tv0;
  uint32_t* tv1;
  // zeroed control block
  uint32_t* rs_status;  // (8 + 2) passes x parts x 256
  uint64_t* scan_status;  // 2 x parts
  uint32_t* hist;       // 10 x 256
  uint32_t* part_ctr;   // 16
  size_t control_bytes;
  void* control_begin;
  int64_t parts_n, parts_k;
};

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

static size_t carve(int64_t n, int64_t cap, int n_tiles, unsigned char* base, TilesScratch* s) {
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
  t.dk[0] = (uint64_t*)take(8 * nn);
  t.dk[1] = (uint64_t*)take(8 * nn);
  t.dv[0] = (uint32_t*)take(4 * nn);
  t.dv[1] = (uint32_t*)take(4 * nn);
  t.offsets = (uint32_t*)take(4 * nn);
  t.tk[0] = take(tkw * cc);
  t.tk[1] = take(tkw * cc);
  t.tv0 = (uint32_t*)take(4 * cc);
  t.tv1 = (uint32_t*)take(4 * cc);
  const size_t ctl0 = off;
  t.control_begin = base ? base + ctl0 : nullptr;
  t.rs_status = (uint32_t*)take(sizeof(uint32_t) * RADIX * (size_t)(8 * parts_n + 2 * parts_k));
  t.scan_status = (uint64_t*)take(sizeof(uint64_t) * (size_t)(2 * (parts_n + 1)));
  t.hist = (uint32_t*)take(sizeof(uint32_t) * 10 * RADIX);
  t.part_ctr = (uint32_t*)take(sizeof(uint32_t) * 32);
  t.control_bytes = off - ctl0;
  t.parts_n = parts_n;
  t.parts_k = parts_k;
  if (s) *s = t;
  return off;
}

static int persistent_grid(const void* fn, int threads, size_t smem) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem);
  if (per_sm < 1) per_sm = 1;
  int dev = 0, sms = NUM_SMS;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return per_sm * sms;
}

template <typename K>
static int radix_sort(K* k0, K* k1, uint32_t* v0, uint32_t* v1, uint32_t* final_vals, const int64_t* count_ptr,
                      int64_t cap, int shift0, int npasses, uint32_t* hist, uint32_t* status, int64_t parts,
                      uint32_t* part_ctr, cudaStream_t st, K** keys_result) {
  const size_t smem = sizeof(RadixSmem<K>);
  auto pass = radix_pass_kernel<K>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(pass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  radix_hist_kernel<K><<<2 * NUM_SMS, 256, 0, st>>>(k0, count_ptr, cap, shift0, npasses, hist);
  HGS_CHECK_LAUNCH();
  static int grid = 0;
  if (grid == 0) grid = persistent_grid((const void*)pass, RS_THREADS, smem);
  const int g = (int)hgs::tmin<int64_t>(grid, hgs::tmax<int64_t>(parts, 1));
  K* kin = k0;
  K* kout = k1;
  uint32_t* vin = v0;
  uint32_t* vout = v1;
  for (int p = 0; p < npasses; p++) {
    const bool last = p == npasses - 1;
    uint32_t* vdst = last && final_vals ? final_vals : vout;
    pass<<<g, RS_THREADS, smem, st>>>(kin, vin, kout, vdst, count_ptr, cap, shift0 + 8 * p, hist + RADIX * p,
                                      status + (size_t)p * parts * RADIX, part_ctr + p, 1);
    HGS_CHECK_LAUNCH();
    std::swap(kin, kout);
    vin = vdst;
    vout = (vdst == v1) ? v0 : v1;
  }
  if (keys_result) *keys_result = kin;
  return HGS_OK;
}

}  // namespace hgs

extern "C" size_t hgs_tiles_scratch_bytes(int64_t n, int64_t capacity, int32_t n_tiles) {
  return hgs::carve(n, capacity, n_tiles, nullptr, nullptr);
}

extern "C" int hgs_build_tiles(const hgs_projected* proj, int64_t n, hgs_tiles* tiles, void* stream) {
  using namespace hgs;
  if (!proj || !tiles) return hgs_set_error(HGS_ERR_INVALID, "hgs_build_tiles: null argument");
  if (!tiles->entries || !tiles->tile_starts || !tiles->counters)
    return hgs_set_error(HGS_ERR_INVALID, "hgs_build_tiles: missing output pointer");
  const int n_tiles = tiles->tiles_x * tiles->tiles_y;
  if (tiles->tiles_x <= 0 || tiles->tiles_y <= 0) return hgs_set_error(HGS_ERR_INVALID, "hgs_build_tiles: empty tile grid");
  if (n > 0xffffffffLL || tiles->capacity > (1LL << 30))
    return hgs_set_error(HGS_ERR_INVALID, "hgs_build_tiles: n or capacity too large");
  const size_t need = carve(n, tiles->capacity, n_tiles, nullptr, nullptr);
  if (!tiles->scratch || tiles->scratch_bytes < need)
    return hgs_set_error(HGS_ERR_INVALID, "hgs_build_tiles: scratch too small (see hgs_tiles_scratch_bytes)");
  cudaStream_t st = (cudaStream_t)stream;
  TilesScratch s;
  carve(n, tiles->capacity, n_tiles, (unsigned char*)tiles->scratch, &s);
  cudaMemsetAsync(s.control_begin, 0, s.control_bytes, st);
  cudaMemsetAsync(tiles->counters, 0, 4 * sizeof(int64_t), st);
  if (n == 0) {
    ranges_kernel<uint16_t><<<ceil_div(n_tiles + 1, 256), 256, 0, st>>>((const uint16_t*)s.tk[0], tiles->counters,
                                                                       tiles->capacity, n_tiles, tiles->tile_starts);
    HGS_CHECK_LAUNCH();
    return HGS_OK;
  }
  const int scan_grid = (int)hgs::tmin<int64_t>(persistent_grid((const void*)compact_kernel, SCAN_THREADS, 0),
                                               (n + SCAN_TILE - 1) / SCAN_TILE);
  compact_kernel<<<scan_grid, SCAN_THREADS, 0, st>>>(proj->count, (const BlendRec*)proj->rec, n, s.dk[0], s.dv[0],
                                                     s.scan_status, s.part_ctr + 20, tiles->counters);
  HGS_CHECK_LAUNCH();
  // stable sort of the visible rows by fp64 depth bits
  int rc = radix_sort<uint64_t>(s.dk[0], s.dk[1], s.dv[0], s.dv[1], nullptr, tiles->counters, n, 0, 8, s.hist,
                                s.rs_status, s.parts_n, s.part_ctr, st, nullptr);
  if (rc) return rc;
  // 8 passes: result back in dk[0]/dv[0]
  offsets_kernel<<<scan_grid, SCAN_THREADS, 0, st>>>(proj->count, s.dv[0], tiles->counters, s.offsets,
                                                     s.scan_status + s.parts_n + 1, s.part_ctr + 21, tiles->counters,
                                                     tiles->capacity);
  HGS_CHECK_LAUNCH();
  int bits = 1;
  while ((1 << bits) < n_tiles) bits++;
  const int tpasses = (bits + 7) / 8;
  const int emit_grid = ceil_div(n, 256);
  uint32_t* rs_tile_status = s.rs_status + (size_t)8 * s.parts_n * RADIX;
  if (n_tiles > 65535) {
    emit_kernel<uint32_t><<<emit_grid, 256, 0, st>>>(s.dv[0], s.offsets, (const ushort4*)proj->rect, tiles->counters,
                                                     tiles->tiles_x, tiles->capacity, (uint32_t*)s.tk[0], s.tv0);
    HGS_CHECK_LAUNCH();
    uint32_t* kres = nullptr;
    rc = radix_sort<uint32_t>((uint32_t*)s.tk[0], (uint32_t*)s.tk[1], s.tv0, s.tv1, tiles->entries,
                              tiles->counters + 1, tiles->capacity, 0, tpasses, s.hist + 8 * RADIX, rs_tile_status,
                              s.parts_k, s.part_ctr + 8, st, &kres);
    if (rc) return rc;
    ranges_kernel<uint32_t><<<2 * NUM_SMS, 256, 0, st>>>(kres, tiles->counters, tiles->capacity, n_tiles,
                                                         tiles->tile_starts);
  } else {
    emit_kernel<uint16_t><<<emit_grid, 256, 0, st>>>(s.dv[0], s.offsets, (const ushort4*)proj->rect, tiles->counters,
                                                     tiles->tiles_x, tiles->capacity, (uint16_t*)s.tk[0], s.tv0);
    HGS_CHECK_LAUNCH();
    uint16_t* kres = nullptr;
    rc = radix_sort<uint16_t>((uint16_t*)s.tk[0], (uint16_t*)s.tk[1], s.tv0, s.tv1, tiles->entries,
                              tiles->counters + 1, tiles->capacity, 0, tpasses, s.hist + 8 * RADIX, rs_tile_status,
                              s.parts_k, s.part_ctr + 8, st, &kres);
    if (rc) return rc;
    ranges_kernel<uint16_t><<<2 * NUM_SMS, 256, 0, st>>>(kres, tiles->counters, tiles->capacity, n_tiles,
                                                         tiles->tile_starts);
  }
  HGS_CHECK_LAUNCH();
  return HGS_OK;
}
