// radix_sort.cu — stable LSD radix sort of (key, 32-bit value) pairs on
// sm_100a, the sort behind the generic COO -> CSC conversion (SURVEY §8(f2):
// SparseMatrix::from_triplets, proj/src/sparse.cpp:53-70 orders entries by
// (row, col) keeping insertion order on ties; here the column-major key
// col * rows + row with the entry index as value) and the CSC -> CSR
// transpose of the verification kernels.
//
// Per 8-bit digit (only the bits the keys use): three launches
//   k_rs_hist     one CTA per 3072-item tile: digit histogram in SMEM,
//                 written digit-major (counts[d * ntiles + t])
//   scan          exclusive scan of the 256 x ntiles counts -> every
//                 (digit, tile) pair's first output slot (stable by
//                 construction: tiles in order inside a digit)
//   k_rs_scatter  the tile again: stable in-tile ranks (each warp owns a
//                 contiguous chunk and ranks it with __match_any peers +
//                 its own running digit counters in SMEM -- no block barrier
//                 per round; one pass over the warps' counts then gives each
//                 warp's first rank per digit), the tile staged in SMEM in digit
//                 order, then written out so consecutive threads store
//                 consecutive slots of one digit (coalesced runs instead of
//                 one scattered 8-byte store per item)
// Traffic per digit: 8 (hist) + 2 x 12 B per u64 item; HBM-bound.
#include <cstring>

#include "common.cuh"

namespace phfem {

constexpr int kRsThreads = 256;
constexpr int kRsItems = 12;                      // items per thread per tile
constexpr int kRsTile = kRsThreads * kRsItems;    // 3072
constexpr int kRsWarps = kRsThreads / 32;

template <typename K>
__global__ void __launch_bounds__(kRsThreads) k_rs_hist(const K* __restrict__ keys, int64_t n, int shift,
                                                        int ntiles, int32_t* __restrict__ counts) {
  // per-warp digit counters: plain SMEM atomics (a same-digit warp serialises
  // inside one instruction, cheaper than a __match_any per item)
  __shared__ int32_t h[kRsWarps][256];
#pragma unroll
  for (int w = 0; w < kRsWarps; ++w) h[w][threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kRsTile;
  const int warp = threadIdx.x >> 5;
  K k[kRsItems];  // all loads in flight before the first atomic
#pragma unroll
  for (int r = 0; r < kRsItems; ++r) {
    const int64_t i = base + r * kRsThreads + threadIdx.x;
    if (i < n) k[r] = keys[i];
  }
#pragma unroll
  for (int r = 0; r < kRsItems; ++r) {
    const int64_t i = base + r * kRsThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[warp][(unsigned)(k[r] >> shift) & 0xffu], 1);
  }
  __syncthreads();
  int32_t tot = 0;
#pragma unroll
  for (int w = 0; w < kRsWarps; ++w) tot += h[w][threadIdx.x];
  counts[(int64_t)threadIdx.x * ntiles + blockIdx.x] = tot;
}

template <typename K>
struct RsSmem {
  K key[kRsTile];
  uint32_t val[kRsTile];
  int32_t wc[kRsWarps][256];  // per-warp digit counts of the current round
  int32_t run[256];           // items of each digit in the tile so far
  int32_t tstart[256];        // digit starts inside the tile
  int32_t gofs[256];          // digit's first global slot for this tile
  int32_t scan[33];
};

template <typename K>
__global__ void __launch_bounds__(kRsThreads, 3) k_rs_scatter(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                           int64_t n, int shift, int ntiles,
                                                           const int32_t* __restrict__ offs, K* __restrict__ kout,
                                                           uint32_t* __restrict__ vout) {
  extern __shared__ __align__(16) unsigned char rs_raw[];
  RsSmem<K>& sm = *reinterpret_cast<RsSmem<K>*>(rs_raw);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int64_t base = (int64_t)blockIdx.x * kRsTile;
  sm.gofs[tid] = offs[(int64_t)tid * ntiles + blockIdx.x];
#pragma unroll
  for (int w = 0; w < kRsWarps; ++w) sm.wc[w][tid] = 0;
  K k[kRsItems];
  uint32_t v[kRsItems];
  int rk[kRsItems];
  // warp w owns items [32 kRsItems w, 32 kRsItems (w + 1)) of the tile, 32
  // consecutive ones per round: index order = (warp, round, lane)
  const int64_t wbase = base + (int64_t)warp * (kRsItems * 32) + lane_id();
#pragma unroll
  for (int r = 0; r < kRsItems; ++r) {
    const int64_t i = wbase + r * 32;
    if (i < n) {
      k[r] = kin[i];
      v[r] = vin[i];
    }
  }
  __syncthreads();
  const unsigned lt = lanemask_lt();
  // stable ranks inside the warp's chunk: the warp's own digit counters, no
  // block barrier per round
#pragma unroll
  for (int r = 0; r < kRsItems; ++r) {
    const int64_t i = wbase + r * 32;
    const unsigned d = i < n ? (unsigned)(k[r] >> shift) & 0xffu : 0x100u;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    if (d < 256u) rk[r] = sm.wc[warp][d] + __popc(peers & lt);
    __syncwarp();
    if (d < 256u && lane_id() == (unsigned)(__ffs(peers) - 1)) sm.wc[warp][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // digit tid: the warps' counts -> each warp's first rank, and the tile count
  {
    int acc = 0;
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) {
      const int c = sm.wc[w][tid];
      sm.wc[w][tid] = acc;
      acc += c;
    }
    sm.run[tid] = acc;
  }
  // digit starts inside the tile, then the tile in digit order in SMEM
  int32_t total;
  sm.tstart[tid] = block_exclusive_scan<int32_t>(sm.run[tid], sm.scan, &total);
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRsItems; ++r) {
    const int64_t i = wbase + r * 32;
    if (i < n) {
      const unsigned d = (unsigned)(k[r] >> shift) & 0xffu;
      const int p = sm.tstart[d] + sm.wc[warp][d] + rk[r];
      sm.key[p] = k[r];
      sm.val[p] = v[r];
    }
  }
  __syncthreads();
  const int cnt = n - base < kRsTile ? (int)(n - base) : kRsTile;
  for (int p = tid; p < cnt; p += kRsThreads) {
    const K key = sm.key[p];
    const unsigned d = (unsigned)(key >> shift) & 0xffu;
    const int64_t g = (int64_t)sm.gofs[d] + (p - sm.tstart[d]);
    kout[g] = key;
    vout[g] = sm.val[p];
  }
}

template <typename K>
static phfem_status radix_sort_pairs(phfem_ctx* ctx, const K* kin, K* kout, const uint32_t* vin, uint32_t* vout,
                                     int64_t n, int end_bit) {
  if (n <= 0) return PHFEM_OK;
  if (n >= (int64_t(1) << 31))
    return set_error(ctx, PHFEM_ERR_INVALID_ARGUMENT, "radix_sort: more than 2^31 items");
  const int ntiles = (int)((n + kRsTile - 1) / kRsTile);
  const int passes = end_bit <= 0 ? 0 : (end_bit + 7) / 8;
  if (passes == 0) {
    PHFEM_CUDA(ctx, cudaMemcpyAsync(kout, kin, sizeof(K) * n, cudaMemcpyDeviceToDevice, ctx->stream));
    PHFEM_CUDA(ctx, cudaMemcpyAsync(vout, vin, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, ctx->stream));
    return PHFEM_OK;
  }
  const size_t smem = sizeof(RsSmem<K>);
  PHFEM_TRY(smem_optin(ctx, (const void*)k_rs_scatter<K>, smem, "k_rs_scatter smem opt-in"));
  int32_t* counts = nullptr;
  K* ktmp = nullptr;
  uint32_t* vtmp = nullptr;
  PHFEM_TRY(dalloc(ctx, &counts, (int64_t)256 * ntiles));
  if (passes > 1) {
    PHFEM_TRY(dalloc(ctx, &ktmp, n));
    PHFEM_TRY(dalloc(ctx, &vtmp, n));
  }
  // ping-pong so that the last pass lands in (kout, vout)
  const K* ks = kin;
  const uint32_t* vs = vin;
  for (int p = 0; p < passes; ++p) {
    const bool to_out = ((passes - 1 - p) % 2) == 0;
    K* kd = to_out ? kout : ktmp;
    uint32_t* vd = to_out ? vout : vtmp;
    const int shift = 8 * p;
    PHFEM_LAUNCH(ctx, "k_rs_hist", k_rs_hist<K><<<ntiles, kRsThreads, 0, ctx->stream>>>(ks, n, shift, ntiles,
                                                                                        counts));
    PHFEM_TRY(scan_exclusive_i32(ctx, counts, counts, (int64_t)256 * ntiles, nullptr));
    PHFEM_LAUNCH(ctx, "k_rs_scatter", k_rs_scatter<K><<<ntiles, kRsThreads, smem, ctx->stream>>>(
        ks, vs, n, shift, ntiles, counts, kd, vd));
    ks = kd;
    vs = vd;
  }
  dfree(ctx, counts);
  dfree(ctx, ktmp);
  dfree(ctx, vtmp);
  return PHFEM_OK;
}

phfem_status radix_sort_pairs_u64(phfem_ctx* ctx, const uint64_t* kin, uint64_t* kout, const uint32_t* vin,
                                  uint32_t* vout, int64_t n, int end_bit) {
  return radix_sort_pairs<uint64_t>(ctx, kin, kout, vin, vout, n, end_bit);
}

phfem_status radix_sort_pairs_u32(phfem_ctx* ctx, const uint32_t* kin, uint32_t* kout, const uint32_t* vin,
                                  uint32_t* vout, int64_t n, int end_bit) {
  return radix_sort_pairs<uint32_t>(ctx, kin, kout, vin, vout, n, end_bit);
}

}  // namespace phfem
