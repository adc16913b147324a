// edge_gen.cu — build_topology on sm_100a.
//
// Reference: proj/src/edge_topology.cpp:52-143.  The reference emits 3 directed
// occurrences per element (:61-68), sorts them stably by (max node, min node)
// with two counting passes (:74-77) and walks the runs (:82-115): the first
// occurrence of a run is t_plus, ids are handed out in canonical order.
//
// Device algorithm (2 global passes over the occurrences):
//   A  k_eg_count     histogram of occurrences per bucket of 2^bs consecutive
//                     max-node ids (warp-aggregated atomics)
//   B  scan           bucket offsets; k_eg_tile_max = the largest tile (does
//                     every 256-node tile fit in SMEM?)
//   C  k_eg_scatter   each occurrence packed into one 64-bit item
//                       [max-node low bits | min node | occurrence index | dir]
//                     and scattered into its bucket (warp-aggregated cursor)
//   D  k_eg_tile      one CTA per tile of 256 max nodes (256 >> bs buckets):
//                     the items grouped by max node in SMEM, each node's
//                     occurrences sorted (the packed value orders by (max,
//                     min, occurrence) = the reference's stable order), run
//                     detection with the reference's two error checks, one
//                     16-byte record per edge at a tile-local slot (carrying
//                     the tile-local boundary prefix) and per-tile edge /
//                     boundary / Neumann counts.  Column path (every node
//                     <= 16 occurrences: one thread per node, per-node SMEM
//                     columns, insertion sort), item-parallel fast path (<= 32:
//                     counting sort + in-segment rank sort) and a general path
//                     (global scratch for oversized tiles or segments).
//   (fixed-capacity layout, the default for element input: A and B are
//    skipped — k_eg_fixed_init gives bucket b the item slots [b cap, ...),
//    k_eg_scatter_fixed fills them and reports the fullest bucket; over
//    capacity the counted layout above runs instead)
//   E  scans          of the per-tile counts (no look-back: tiny arrays)
//   F  k_eg_emit      one CTA per tile: records -> edge_nodes, edge_elements,
//                     local indices, interior / boundary list slots, elem_edge,
//                     node_edge_start at the scanned tile offsets; on a fused
//                     final level also retained_pos / retained_edges and C.
#include <algorithm>

#include "common.cuh"

namespace phfem {

struct EgParams {
  int32_t nC, nE;  // nodes of the key range (local), elements of the mesh
  int lo_bits, occ_bits, total_bits, bs;
  int nb;
  int32_t node_base;  // first max node of the range (0 for a whole mesh)
  // fixed-capacity bucket layout (0: contiguous): bucket b owns items
  // [b fcap, b fcap + fill_b), tile t's records start at t nsub fcap
  int32_t fcap;
};

static int bits_for(int64_t max_value) {  // bits to represent 0..max_value
  int b = 1;
  while (b < 63 && (int64_t(1) << b) <= max_value) ++b;
  return b;
}

__device__ __forceinline__ uint64_t eg_pack(const EgParams& P, uint32_t hl, uint32_t lo,
                                            uint32_t occ, uint32_t dir) {
  return ((uint64_t)hl << P.total_bits) | ((uint64_t)lo << (P.occ_bits + 1)) |
         ((uint64_t)occ << 1) | dir;
}

// A ------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_eg_count(const int32_t* __restrict__ elements, EgParams P,
                                                  int32_t* __restrict__ bcount,
                                                  phfem_dev_errors* err) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t m0 = (int64_t)blockIdx.x * blockDim.x; m0 < P.nE; m0 += stride) {
    const int64_t m = m0 + threadIdx.x;
    const bool valid = m < P.nE;
    int t[3] = {0, 0, 0};
    if (valid) {
      t[0] = __ldg(elements + 3 * m);
      t[1] = __ldg(elements + 3 * m + 1);
      t[2] = __ldg(elements + 3 * m + 2);
      if ((unsigned)t[0] >= (unsigned)P.nC || (unsigned)t[1] >= (unsigned)P.nC ||
          (unsigned)t[2] >= (unsigned)P.nC)
        atomicMin(&err->misc, (unsigned long long)m);
    }
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const int a = t[s], b = t[(s + 1) % 3];
      const int hi = a > b ? a : b;
      const bool ok = valid && (unsigned)hi < (unsigned)P.nC && a >= 0 && b >= 0;
      const unsigned key = ok ? ((unsigned)hi >> P.bs) : 0xffffffffu;
      const unsigned grp = __match_any_sync(0xffffffffu, key);
      if (ok && lane_id() == (unsigned)(__ffs(grp) - 1)) atomicAdd(&bcount[key], __popc(grp));
    }
  }
}

// C ------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_eg_scatter(const int32_t* __restrict__ elements,
                                                    EgParams P, int32_t* __restrict__ cursor,
                                                    uint64_t* __restrict__ items) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint32_t hl_mask = (1u << P.bs) - 1u;
  for (int64_t m0 = (int64_t)blockIdx.x * blockDim.x; m0 < P.nE; m0 += stride) {
    const int64_t m = m0 + threadIdx.x;
    const bool valid = m < P.nE;
    int t[3] = {0, 0, 0};
    if (valid) {
      t[0] = __ldg(elements + 3 * m);
      t[1] = __ldg(elements + 3 * m + 1);
      t[2] = __ldg(elements + 3 * m + 2);
    }
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const int a = t[s], b = t[(s + 1) % 3];
      const int hi = a > b ? a : b;
      const int lo = a > b ? b : a;
      const unsigned key = valid ? ((unsigned)hi >> P.bs) : 0xffffffffu;
      const unsigned grp = __match_any_sync(0xffffffffu, key);
      const int leader = __ffs(grp) - 1;
      int base = 0;
      if (valid && (int)lane_id() == leader) base = atomicAdd(&cursor[key], __popc(grp));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (valid) {
        const int rank = __popc(grp & lanemask_lt());
        const uint32_t occ = (uint32_t)(3 * m + s);
        items[base + rank] = eg_pack(P, (uint32_t)hi & hl_mask, (uint32_t)lo, occ, a > b ? 1u : 0u);
      }
    }
  }
}

// C (fixed-capacity layout, no count pass): every bucket owns kTileCap / nsub
// slots, its cursor starts at b * fcap; the node-range check of the count
// pass is made here (first bad element -> misc) and the fullest bucket's
// fill is reported (counters[3]) — above fcap the caller falls back to the
// counted layout.
// (measured at L12 before the batched claims: 8 CTAs per SM 0.320 ms, 32 /
// 128 / 512 per SM 0.325 / 0.400 / 0.844 ms — the bucket cursors' atomics,
// not the stores, bound it; the next element's vertex loads prefetched: no
// change; with the batched claims 8 / 16 per SM 0.298 / 0.296 ms)
#ifndef PHFEM_SC_GRID_MULT
#define PHFEM_SC_GRID_MULT 16
#endif
__global__ void __launch_bounds__(256) k_eg_scatter_fixed(const int32_t* __restrict__ elements,
                                                          EgParams P, int32_t* __restrict__ cursor,
                                                          uint64_t* __restrict__ items, phfem_dev_errors* err) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint32_t hl_mask = (1u << P.bs) - 1u;
  unsigned fill_max = 0;
  for (int64_t m0 = (int64_t)blockIdx.x * blockDim.x; m0 < P.nE; m0 += stride) {
    const int64_t m = m0 + threadIdx.x;
    bool valid = m < P.nE;
    int t[3] = {0, 0, 0};
    if (valid) {
      t[0] = __ldg(elements + 3 * m);
      t[1] = __ldg(elements + 3 * m + 1);
      t[2] = __ldg(elements + 3 * m + 2);
      if ((unsigned)t[0] >= (unsigned)P.nC || (unsigned)t[1] >= (unsigned)P.nC ||
          (unsigned)t[2] >= (unsigned)P.nC) {
        atomicMin(&err->misc, (unsigned long long)m);
        valid = false;
      }
    }
    // the three occurrences' bucket claims issued back to back (three global
    // atomics in flight per warp), then their slots (measured: claim -> shuffle
    // -> store per occurrence serialised the atomics' round trips; L12 scatter
    // 0.319 -> 0.296 ms, given L13 1.244 -> 1.147 ms with 16 CTAs per SM)
    unsigned key[3], grp[3];
    int base[3];
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const int a = t[s], b = t[(s + 1) % 3];
      key[s] = valid ? ((unsigned)(a > b ? a : b) >> P.bs) : 0xffffffffu;
      grp[s] = __match_any_sync(0xffffffffu, key[s]);
    }
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      base[s] = 0;
      if (valid && (int)lane_id() == __ffs(grp[s]) - 1) base[s] = atomicAdd(&cursor[key[s]], __popc(grp[s]));
    }
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const int a = t[s], b = t[(s + 1) % 3];
      const int hi = a > b ? a : b;
      const int lo = a > b ? b : a;
      const int bs_ = __shfl_sync(0xffffffffu, base[s], __ffs(grp[s]) - 1);
      if (valid) {
        const int rank = __popc(grp[s] & lanemask_lt());
        const int64_t at = (int64_t)bs_ + rank;
        const int64_t end = ((int64_t)key[s] + 1) * P.fcap;
        if (at < end) {
          const uint32_t occ = (uint32_t)(3 * m + s);
          items[at] = eg_pack(P, (uint32_t)hi & hl_mask, (uint32_t)lo, occ, a > b ? 1u : 0u);
        }
        fill_max = max(fill_max, (unsigned)(at + 1 - (end - P.fcap)));
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) fill_max = max(fill_max, __shfl_xor_sync(0xffffffffu, fill_max, o));
  if (lane_id() == 0 && fill_max) atomicMax(&err->counters[3], (unsigned long long)fill_max);
}

__global__ void k_eg_fixed_init(int32_t* __restrict__ boff, int32_t* __restrict__ cursor, int nb, int fcap) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b <= nb; b += gridDim.x * blockDim.x) {
    boff[b] = b * fcap;
    if (b < nb) cursor[b] = b * fcap;
  }
}

// A'/C' for the distributed dedup: the occurrences arrive as records
// {max node, min node, occurrence 3m+s, dir} of one max-node key range
// (dist.py's key-range all-to-all) instead of being read from elements.
__global__ void __launch_bounds__(256) k_rec_count(const int4* __restrict__ recs, int64_t n,
                                                   EgParams P, int32_t* __restrict__ bcount,
                                                   phfem_dev_errors* err) {
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    bool ok = i < n;
    int hl = 0;
    if (ok) {
      const int4 r = recs[i];
      hl = r.x - P.node_base;
      if (hl < 0 || hl >= P.nC) {
        atomicMin(&err->misc, (unsigned long long)i);
        ok = false;
      }
    }
    const unsigned key = ok ? ((unsigned)hl >> P.bs) : 0xffffffffu;
    const unsigned grp = __match_any_sync(0xffffffffu, key);
    if (ok && lane_id() == (unsigned)(__ffs(grp) - 1)) atomicAdd(&bcount[key], __popc(grp));
  }
}

__global__ void __launch_bounds__(256) k_rec_scatter(const int4* __restrict__ recs, int64_t n,
                                                     EgParams P, int32_t* __restrict__ cursor,
                                                     uint64_t* __restrict__ items) {
  const uint32_t hl_mask = (1u << P.bs) - 1u;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    const bool valid = i < n;
    int4 r = make_int4(0, 0, 0, 0);
    if (valid) r = recs[i];
    const int hl = r.x - P.node_base;
    const unsigned key = valid ? ((unsigned)hl >> P.bs) : 0xffffffffu;
    const unsigned grp = __match_any_sync(0xffffffffu, key);
    const int leader = __ffs(grp) - 1;
    int base = 0;
    if (valid && (int)lane_id() == leader) base = atomicAdd(&cursor[key], __popc(grp));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (valid)
      items[base + __popc(grp & lanemask_lt())] =
          eg_pack(P, (uint32_t)hl & hl_mask, (uint32_t)r.y, (uint32_t)r.z, (uint32_t)r.w);
  }
}

// D ------------------------------------------------------------------------
struct EgOut {
  int32_t* edge_nodes;
  int32_t* edge_elements;
  int32_t* ltp;
  int32_t* ltm;
  int32_t* interior;
  int32_t* boundary;
  int32_t* elem_edge;
  int32_t* node_edge_start;
  int2* pairs;  // non-null: (slot 3m+l, edge or ~edge) per occurrence instead of elem_edge
  // with pairs: slots [self_lo3, self_hi3) of the rank's own elements go to
  // self_ee directly, only the others are appended to pairs (count npairs)
  int32_t* self_ee;
  int64_t self_lo3, self_hi3;
  int32_t* npairs;
  int32_t node_base;
  // fused classification + C (sort-built final topology, pipeline): the
  // Neumann pairs as a hash set of (min << 32 | max) keys; retained_pos /
  // retained_edges / C rows written by the emit pass
  const unsigned long long* neu_keys;
  int neu_cap;
  int32_t* tileN;  // Neumann edges per tile (tile pass), then their prefixes
  int32_t* rpos;
  int32_t* redges;
  int32_t* row_ptr;
  int32_t* col;
  double* val;
  const double2* coords;
  int L;
};

// the elem_edge entries of edge e: slot s0 <- e (T+), s1 <- ~e (T-; s1 < 0: none)
__device__ __forceinline__ void eg_slots(const EgOut& o, int32_t e, int64_t s0, int64_t s1) {
  if (o.self_ee) {
    const bool own0 = s0 >= o.self_lo3 && s0 < o.self_hi3;
    const bool own1 = s1 < 0 || (s1 >= o.self_lo3 && s1 < o.self_hi3);
    if (own0) o.self_ee[s0 - o.self_lo3] = e;
    if (s1 >= 0 && own1) o.self_ee[s1 - o.self_lo3] = ~e;
    const int k = (own0 ? 0 : 1) + (own1 ? 0 : 1);
    // slots of other ranks' elements: one cursor atomic per warp, not per edge
    const unsigned am = __activemask();
    const unsigned b1 = __ballot_sync(am, k >= 1), b2 = __ballot_sync(am, k == 2);
    const int total = __popc(b1) + __popc(b2);
    if (total) {
      const int leader = __ffs(am) - 1;
      int base = 0;
      if ((int)lane_id() == leader) base = atomicAdd(o.npairs, total);
      base = __shfl_sync(am, base, leader);
      const unsigned lt = lanemask_lt();
      int at = base + __popc(b1 & lt) + __popc(b2 & lt);
      if (!own0) o.pairs[at++] = make_int2((int)s0, e);
      if (!own1) o.pairs[at] = make_int2((int)s1, ~e);
    }
  } else if (o.pairs) {
    o.pairs[2 * (int64_t)e] = make_int2((int)s0, e);
    o.pairs[2 * (int64_t)e + 1] = s1 >= 0 ? make_int2((int)s1, ~e) : make_int2(-1, 0);
  } else {
    o.elem_edge[s0] = e;
    if (s1 >= 0) o.elem_edge[s1] = ~e;
  }
}

__device__ __forceinline__ uint32_t neu_pair_hash(unsigned long long key, int cap) {
  return (uint32_t)((key * 0x9E3779B97F4A7C15ull) >> 32) & (uint32_t)(cap - 1);
}

// is (lo, hi) a Neumann pair (either direction in the mesh's list)?
__device__ __forceinline__ bool neu_pair_has(const EgOut& o, int lo, int hi) {
  if (!o.neu_keys) return false;
  const unsigned long long key = (unsigned long long)(uint32_t)lo << 32 | (uint32_t)hi;
  uint32_t h = neu_pair_hash(key, o.neu_cap);
  while (true) {
    const unsigned long long k = o.neu_keys[h];
    if (k == key) return true;
    if (k == ~0ull) return false;
    h = (h + 1) & (uint32_t)(o.neu_cap - 1);
  }
}

__global__ void k_neu_pair_insert(const int32_t* __restrict__ pairs, int n, int cap,
                                  unsigned long long* __restrict__ keys) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int a = pairs[2 * i], b = pairs[2 * i + 1];
    const unsigned long long key =
        (unsigned long long)(uint32_t)min(a, b) << 32 | (uint32_t)max(a, b);
    uint32_t h = neu_pair_hash(key, cap);
    while (true) {
      const unsigned long long prev = atomicCAS(keys + h, ~0ull, key);
      if (prev == ~0ull || prev == key) break;
      h = (h + 1) & (uint32_t)(cap - 1);
    }
  }
}

// Edge record of the sort pass (one per unique edge, at a tile-local slot of
// the tile's item range): {local max node | boundary edges before it in the
// tile << 8, min node, occ_f << 1 | dir, occ_g or -1} — occ = 3 m + slot of
// the t_plus / t_minus occurrence.  Carrying the tile-local boundary prefix
// lets the emit pass run one record per thread with no scan.
__device__ __forceinline__ int4 eg_record(int nd, int bloc, int32_t lo, uint64_t f, uint64_t g,
                                          bool two, int ob, bool neu = false) {
  const uint32_t occ_mask = (uint32_t)((1ull << ob) - 1ull);
  const uint32_t occ_f = (uint32_t)(f >> 1) & occ_mask;
  const uint32_t occ_g = (uint32_t)(g >> 1) & occ_mask;
  return make_int4(nd | bloc << 8, lo, (int)((occ_f << 1) | (uint32_t)(f & 1ull)),
                   two ? (int)occ_g : (neu ? -2 : -1));  // -2: a Neumann boundary edge
}

// One CTA per tile of kTileNodes consecutive max-node ids (= 256 >> bs
// consecutive buckets).  Item-parallel throughout: counting sort by node,
// per-segment rank sort (segments are tiny: ~6 occurrences per node), blocked
// run detection + block scan, look-back, then every run start emits its edge.
constexpr int kTileNodes = 256;
constexpr int kTileThreads = 256;
#ifndef PHFEM_TILE_PER_NODE
#define PHFEM_TILE_PER_NODE 10
#endif
#ifndef PHFEM_TILE_MIN_BLOCKS
#define PHFEM_TILE_MIN_BLOCKS 4  // 4 x 256 threads at <= 64 registers (5 blocks spill)
#endif
constexpr int kTileCap = PHFEM_TILE_PER_NODE * kTileNodes;  // items kept in SMEM (10 per node)

struct TileSmem {
  uint64_t buf1[kTileCap + 4];  // + 4 all-ones keys: the rank loop reads past the last segment
  uint64_t buf2[kTileCap];
  uint8_t node_of[kTileCap];
  uint8_t fl[kTileCap];  // fast path: run start (bit 0) / has a partner (bit 1) per sorted item
  int32_t cnt[kTileNodes];
  int32_t seg[kTileNodes];
  int32_t cur[kTileNodes];
  int32_t nedge[kTileNodes];
  int32_t sbo[kTileNodes + 1];
  unsigned long long scan[33];
  int tile;
};

template <bool kS>
__device__ __forceinline__ void eg_tile(const uint64_t* __restrict__ items, const EgParams& P,
                                        TileSmem& sm, uint64_t* g1, uint64_t* g2, uint8_t* gnode,
                                        int4* __restrict__ rec, int32_t* __restrict__ tileE,
                                        int32_t* __restrict__ tileB, const EgOut& out,
                                        phfem_dev_errors* err) {
  const int tid = threadIdx.x;
  const int T = blockDim.x;
  const int tile = sm.tile;
  const int nsub = kTileNodes >> P.bs;
  const int64_t s = sm.sbo[0];
  const int n = sm.sbo[nsub] - (int)s;
  uint64_t* buf1 = kS ? sm.buf1 : g1 + s;
  uint64_t* buf2 = kS ? sm.buf2 : g2 + s;
  uint8_t* node_of = kS ? sm.node_of : gnode + s;
  const int shift = P.total_bits;
  const uint64_t kmask = (1ull << shift) - 1ull;
  auto local_node = [&](int p, uint64_t it) -> int {
    int sub = 0;
    if (nsub > 1) {  // last sub-bucket whose start <= s + p
      int lo = 0, hi = nsub - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (sm.sbo[mid] - s <= p) lo = mid;
        else hi = mid - 1;
      }
      sub = lo;
    }
    return (sub << P.bs) | (int)(it >> shift);
  };

  // counting sort by max node
  for (int p = tid; p < n; p += T) {
    const uint64_t it = __ldg(items + s + p);
    atomicAdd(&sm.cnt[local_node(p, it)], 1);
  }
  __syncthreads();
  const int c_me = sm.cnt[tid];
  unsigned long long tot;
  const int st_me = (int)block_exclusive_scan((unsigned long long)c_me, sm.scan, &tot);
  sm.seg[tid] = st_me;
  sm.cur[tid] = st_me;
  __syncthreads();
  for (int p = tid; p < n; p += T) {
    const uint64_t it = __ldg(items + s + p);
    const int nd = local_node(p, it);
    const int pos = atomicAdd(&sm.cur[nd], 1);
    buf1[pos] = it;
    node_of[pos] = (uint8_t)nd;
  }
  __syncthreads();
  // rank sort inside each node segment: key = (min node, occurrence, dir)
  for (int p = tid; p < n; p += T) {
    const uint64_t it = buf1[p];
    const uint64_t k = it & kmask;
    const int nd = node_of[p];
    const int st = sm.seg[nd], c = sm.cnt[nd];
    int r = 0;
    for (int q = st; q < st + c; ++q) r += (buf1[q] & kmask) < k;
    buf2[st + r] = it;
  }
  __syncthreads();

  // blocked run detection
  const int lo_shift = P.occ_bits + 1;
  const uint64_t lo_mask = (1ull << P.lo_bits) - 1ull;
  const int K = (n + T - 1) / T;
  const int p0 = min(n, tid * K), p1 = min(n, p0 + K);
  uint32_t ne_i = 0, nb_i = 0;
  for (int p = p0; p < p1; ++p) {
    const int nd = node_of[p];
    const int st = sm.seg[nd], en = st + sm.cnt[nd];
    const uint64_t f = buf2[p];
    const uint64_t lo = (f >> lo_shift) & lo_mask;
    if (p != st && ((buf2[p - 1] >> lo_shift) & lo_mask) == lo) continue;
    int len = 1;
    while (p + len < en && ((buf2[p + len] >> lo_shift) & lo_mask) == lo) ++len;
    if (len > 2 || (len == 2 && ((f ^ buf2[p + 1]) & 1ull) == 0)) {
      const uint64_t v = (uint64_t)P.node_base + (uint64_t)tile * kTileNodes + nd;
      atomicMin(&err->topo, (v << 33) | (lo << 2) | (len > 2 ? 0ull : (2ull | (f & 1ull))));
    }
    ++ne_i;
    nb_i += (len == 1);
    atomicAdd(&sm.nedge[nd], 1);
  }
  unsigned long long agg;
  const unsigned long long ex =
      block_exclusive_scan(((unsigned long long)ne_i << 32) | nb_i, sm.scan, &agg);
  // per-node first edge, tile-local (k_eg_emit adds the tile offset)
  const int ne_node = sm.nedge[tid];
  unsigned long long tot2;
  const int nes_local = (int)block_exclusive_scan((unsigned long long)ne_node, sm.scan, &tot2);
  const int64_t v_me = (int64_t)tile * kTileNodes + tid;
  if (v_me < P.nC) out.node_edge_start[v_me] = nes_local;
  int32_t e = (int32_t)(ex >> 32);  // tile-local edge index
  int32_t bl = (int32_t)(ex & 0xffffffffu);  // tile-local boundary edges before it
  for (int p = p0; p < p1; ++p) {
    const int nd = node_of[p];
    const int st = sm.seg[nd], en = st + sm.cnt[nd];
    const uint64_t f = buf2[p];
    const uint64_t lo = (f >> lo_shift) & lo_mask;
    if (p != st && ((buf2[p - 1] >> lo_shift) & lo_mask) == lo) continue;
    const bool two = p + 1 < en && ((buf2[p + 1] >> lo_shift) & lo_mask) == lo;
    const bool neu =
        !two && out.neu_keys && neu_pair_has(out, (int)lo, P.node_base + tile * kTileNodes + nd);
    if (neu) atomicAdd(&out.tileN[tile], 1);
    rec[s + e] = eg_record(nd, bl, (int32_t)lo, f, two ? buf2[p + 1] : 0, two, P.occ_bits, neu);
    ++e;
    bl += !two;
  }
  if (tid == 0) {
    tileE[tile] = (int32_t)(agg >> 32);
    tileB[tile] = (int32_t)(agg & 0xffffffffu);
  }
}

// Fast tile path (every node <= 32 occurrences): counting sort by max node,
// rank sort inside each node segment (each item counts the smaller keys of
// its segment — ~6 compares on refined meshes, far fewer instructions than a
// 32-wide bitonic network), then per warp run starts / partners / the
// reference's error checks as neighbour tests; edge ranks are ballot/popc
// prefixes, so records of consecutive edges come from consecutive lanes.
constexpr int kTilePer = kTileCap / kTileThreads;  // items per thread in the fast path

__device__ __forceinline__ void eg_tile_fast(const uint64_t* __restrict__ items, const EgParams& P,
                                             TileSmem& sm, int4* __restrict__ rec,
                                             int32_t* __restrict__ tileE, int32_t* __restrict__ tileB,
                                             const EgOut& out, phfem_dev_errors* err,
                                             const uint64_t (&itr)[kTilePer], const int (&ndr)[kTilePer]) {
  const int tid = threadIdx.x;
  const int T = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int tile = sm.tile;
  const int nsub = kTileNodes >> P.bs;
  const int64_t s = sm.sbo[0];
  const int n = sm.sbo[nsub] - (int)s;
  const int ob = P.occ_bits;
  const uint64_t lomask = (1ull << P.lo_bits) - 1ull;
  const unsigned lt = lanemask_lt();

  // counting sort by node (histogram already in sm.cnt)
  const int c_me = sm.cnt[tid];
  unsigned long long tot;
  const int st_me = (int)block_exclusive_scan((unsigned long long)c_me, sm.scan, &tot);
  sm.seg[tid] = st_me;
  sm.cur[tid] = st_me;
  __syncthreads();
  // scatter the items the histogram pass kept in registers
#pragma unroll
  for (int k = 0; k < kTilePer; ++k) {
    if (k * T >= n) break;  // block-uniform: no predicated-off trips for the empty slots
    if (tid + k * T < n) {
      const int pos = atomicAdd(&sm.cur[ndr[k]], 1);
      sm.buf1[pos] = itr[k];
      sm.node_of[pos] = (uint8_t)ndr[k];
    }
  }
  if (tid < 4) sm.buf1[n + tid] = ~0ull;
  __syncthreads();

  // rank sort inside each node segment (<= 32 items, ~6 on refined meshes):
  // key = (min node, occurrence), unique; the reference's stable order
  // (items of one segment share the max-node bits and differ in (min, occ),
  // so the raw 64-bit items compare in key order).  Items are taken in
  // sorted-by-node order, so the lanes of a warp mostly share a segment and
  // its trip count (ranking the register copies in bucket order instead was
  // measured 25 % slower at L12: divergent trip counts).  Four compares per
  // trip read up to 3 items past the segment.  Those are larger — the next
  // nodes' items carry larger max-node bits, the tile ends in ~0 padding —
  // unless the next sub-bucket starts within them: its keys restart at node
  // 0.  Only such segments (tiles of several sub-buckets, bs < 8: e.g. the
  // L13 square's 57-bit items give bs = 7) take the masked compares.
  const int hb = (1 << P.bs) - 1;
  for (int p = tid; p < n; p += T) {
    const uint64_t it = sm.buf1[p];
    const int nd = sm.node_of[p];
    const int st = sm.seg[nd], end = st + sm.cnt[nd];
    int r = 0;
    if (nsub == 1 || end + 3 <= ((nd | hb) + 1 < kTileNodes ? sm.seg[(nd | hb) + 1] : 0x7fffffff)) {
      for (int q = st; q < end; q += 4)
        r += (int)(sm.buf1[q] < it) + (int)(sm.buf1[q + 1] < it) + (int)(sm.buf1[q + 2] < it) +
             (int)(sm.buf1[q + 3] < it);
    } else {
      for (int q = st; q < end; q += 4)
        r += (int)(sm.buf1[q] < it) + (int)((q + 1 < end) & (sm.buf1[q + 1] < it)) +
             (int)((q + 2 < end) & (sm.buf1[q + 2] < it)) + (int)((q + 3 < end) & (sm.buf1[q + 3] < it));
    }
    sm.buf2[st + r] = it;
  }
  __syncthreads();
  // per warp (its 32 nodes): run starts, partners, the reference's two error
  // checks (edge_topology.cpp:82-99) as neighbour tests in the sorted segment
  const int cnt_l = sm.cnt[32 * warp + lane];
  const int wtotal = __shfl_sync(0xffffffffu, warp_inclusive_scan(cnt_l), 31);
  const int wbase = sm.seg[32 * warp];
  uint32_t w_ne = 0, w_nb = 0;
  for (int q = 0; q < wtotal; q += 32) {
    const int pos = wbase + q + lane;
    const bool valid = q + lane < wtotal;
    bool start = false, partner = false, third = false;
    uint64_t f = 0, g = 0;
    int nd = 0;
    if (valid) {
      f = sm.buf2[pos];
      nd = sm.node_of[pos];
      const int st = sm.seg[nd], en = st + sm.cnt[nd];
      const uint64_t lo = (f >> (ob + 1)) & lomask;
      start = pos == st || ((sm.buf2[pos - 1] >> (ob + 1)) & lomask) != lo;
      if (start && pos + 1 < en) {
        g = sm.buf2[pos + 1];
        partner = ((g >> (ob + 1)) & lomask) == lo;
        third = partner && pos + 2 < en && ((sm.buf2[pos + 2] >> (ob + 1)) & lomask) == lo;
      }
      if (start && (third || (partner && ((f ^ g) & 1ull) == 0))) {
        const uint64_t v = (uint64_t)P.node_base + (uint64_t)tile * kTileNodes + nd;
        atomicMin(&err->topo, (v << 33) | (lo << 2) | (third ? 0ull : (2ull | (f & 1ull))));
      }
      if (start) atomicAdd(&sm.nedge[nd], 1);
      sm.fl[pos] = (uint8_t)(start | (partner << 1));
    }
    w_ne += __popc(__ballot_sync(0xffffffffu, start));
    w_nb += __popc(__ballot_sync(0xffffffffu, start && !partner));
  }
  // CTA totals: per-warp offsets
  __shared__ unsigned long long wsum[kTileThreads / 32];
  if (lane == 0) wsum[warp] = ((unsigned long long)w_ne << 32) | w_nb;
  __syncthreads();
  unsigned long long wex = 0, agg = 0;
  for (int w = 0; w < (T >> 5); ++w) {
    if (w < warp) wex += wsum[w];
    agg += wsum[w];
  }
  const int ne_node = sm.nedge[tid];
  unsigned long long tot2;
  const int nes_local = (int)block_exclusive_scan((unsigned long long)ne_node, sm.scan, &tot2);
  const int64_t v_me = (int64_t)tile * kTileNodes + tid;
  if (v_me < P.nC) out.node_edge_start[v_me] = nes_local;  // tile-local

  // records of the tile's edges at tile-local positions (ranks by ballot)
  int32_t e_off = (int32_t)(wex >> 32);
  int32_t b_off = (int32_t)(wex & 0xffffffffu);
  for (int q = 0; q < wtotal; q += 32) {
    const int pos = wbase + q + lane;
    const bool valid = q + lane < wtotal;
    const int fl = valid ? sm.fl[pos] : 0;  // from the detection pass
    const bool start = fl & 1, partner = fl & 2;
    uint64_t f = 0, g = 0;
    int nd = 0;
    if (start) {
      f = sm.buf2[pos];
      nd = sm.node_of[pos];
      if (partner) g = sm.buf2[pos + 1];
    }
    const unsigned sb = __ballot_sync(0xffffffffu, start);
    const unsigned bb = __ballot_sync(0xffffffffu, start && !partner);
    if (start) {
      const int32_t e = e_off + __popc(sb & lt);
      const int32_t lo = (int32_t)((f >> (ob + 1)) & lomask);
      const bool neu = !partner && out.neu_keys && neu_pair_has(out, lo, P.node_base + tile * kTileNodes + nd);
      if (neu) atomicAdd(&out.tileN[tile], 1);
      rec[s + e] = eg_record(nd, b_off + __popc(bb & lt), lo, f, g, partner, ob, neu);
    }
    e_off += __popc(sb);
    b_off += __popc(bb);
  }
  if (tid == 0) {
    tileE[tile] = (int32_t)(agg >> 32);
    tileB[tile] = (int32_t)(agg & 0xffffffffu);
  }
}

// Column fast path (every node <= kColK occurrences — refined meshes have
// <= 12): one thread per max node.  The counting-sort scatter puts node t's
// j-th occurrence at col[j][t] (column-major: the threads of a warp touch
// consecutive words at every step, no bank conflicts), the thread sorts its
// column by insertion (<= 16 keys, ~6 on refined meshes), walks its runs
// (the reference's two error checks, edges, boundary edges), and after one
// packed block scan of (edges, boundary edges) per node emits its records at
// their tile-local slots — no per-item rank loop, no neighbour pass, no
// per-warp ballot pass (half the instructions of eg_tile_fast).
#ifndef PHFEM_TILE_COL
#define PHFEM_TILE_COL 1
#endif
constexpr int kColK = 16;
// row 0 of the aliased region: zero sentinels (no key is below 0), the
// columns start at row 1
static_assert((kColK + 1) * kTileNodes <= 2 * kTileCap + 4, "the columns alias buf1 / buf2");

__device__ __forceinline__ void eg_tile_col(const EgParams& P, TileSmem& sm, int4* __restrict__ rec,
                                            int32_t* __restrict__ tileE, int32_t* __restrict__ tileB,
                                            const EgOut& out, phfem_dev_errors* err, const int c) {
  const int tid = threadIdx.x;
  const int tile = sm.tile;
  const int64_t s = sm.sbo[0];
  const int ob = P.occ_bits;
  const int lsh = ob + 1;
  const uint64_t lomask = (1ull << P.lo_bits) - 1ull;
  // node t's occurrences in column t of rows 1..c (k_eg_tile scattered them),
  // row 0 = zero sentinels (no key is below 0)
  uint64_t* col = sm.buf1 + kTileNodes;
  uint64_t* my = col + tid;
  // insertion sort of the node's occurrences; key = (min node, occurrence,
  // dir) = the reference's stable order (the max-node bits are shared)
  for (int i = 1; i < c; ++i) {
    uint64_t* q = my + i * kTileNodes;
    const uint64_t x = *q;
    uint64_t y = q[-kTileNodes];
    while (y > x) {  // the zero sentinel row ends the walk
      *q = y;
      q -= kTileNodes;
      y = q[-kTileNodes];
    }
    *q = x;
  }
  // runs of equal min node = edges (edge_topology.cpp:82-99 checks)
  const uint64_t v_glob = (uint64_t)P.node_base + (uint64_t)tile * kTileNodes + tid;
  int ne = 0, nb = 0;
  for (int i = 0; i < c;) {
    const uint64_t f = my[i * kTileNodes];
    const uint64_t lo = (f >> lsh) & lomask;
    int len = 1;
    while (i + len < c && ((my[(i + len) * kTileNodes] >> lsh) & lomask) == lo) ++len;
    if (len > 2 || (len == 2 && ((f ^ my[(i + 1) * kTileNodes]) & 1ull) == 0))
      atomicMin(&err->topo, (v_glob << 33) | (lo << 2) | (len > 2 ? 0ull : (2ull | (f & 1ull))));
    ++ne;
    nb += len == 1;
    i += len;
  }
  unsigned long long agg;
  const unsigned long long ex = block_exclusive_scan(((unsigned long long)ne << 32) | nb, sm.scan, &agg);
  int32_t e = (int32_t)(ex >> 32);                // tile-local edge index of the node's first edge
  int32_t bl = (int32_t)(ex & 0xffffffffu);       // tile-local boundary edges before it
  const int64_t v_me = (int64_t)tile * kTileNodes + tid;
  if (v_me < P.nC) out.node_edge_start[v_me] = e;  // tile-local (k_eg_emit adds the tile offset)
  for (int i = 0; i < c;) {
    const uint64_t f = my[i * kTileNodes];
    const uint64_t lo = (f >> lsh) & lomask;
    const uint64_t g = i + 1 < c ? my[(i + 1) * kTileNodes] : 0ull;
    const bool two = i + 1 < c && ((g >> lsh) & lomask) == lo;
    int len = two ? 2 : 1;
    while (i + len < c && ((my[(i + len) * kTileNodes] >> lsh) & lomask) == lo) ++len;  // (error case)
    const bool neu = !two && out.neu_keys && neu_pair_has(out, (int)lo, (int32_t)v_glob);
    if (neu) atomicAdd(&out.tileN[tile], 1);
    rec[s + e] = eg_record(tid, bl, (int32_t)lo, f, two ? g : 0ull, two, ob, neu);
    ++e;
    bl += !two;
    i += len;
  }
  if (tid == 0) {
    tileE[tile] = (int32_t)(agg >> 32);
    tileB[tile] = (int32_t)(agg & 0xffffffffu);
  }
}

// P.nb here = number of tiles; boff has one entry per bucket (+1).
__device__ __forceinline__ void eg_tile_body(TileSmem& sm, int tile, bool try_col,
                                             const uint64_t* __restrict__ items, const int32_t* __restrict__ boff,
                                             int nbuckets, const EgParams& P, uint64_t* g1, uint64_t* g2,
                                             uint8_t* gnode, int4* __restrict__ rec, int32_t* __restrict__ tileE,
                                             int32_t* __restrict__ tileB, const EgOut& out, phfem_dev_errors* err) {
  const int tid = threadIdx.x;
  if (tid == 0) sm.tile = tile;
  sm.cnt[tid] = 0;
  sm.nedge[tid] = 0;
  sm.cur[tid] = 0;  // the column path's per-node cursors
  __syncthreads();
  const int nsub = kTileNodes >> P.bs;
  if (P.fcap) {  // fixed layout, compacted by k_eg_tile_list: boff = the bucket fills
    if (tid == 0) {
      int at = tile * nsub * P.fcap;
      for (int i = 0; i < nsub; ++i) {
        sm.sbo[i] = at;
        const int b = tile * nsub + i;
        if (b < nbuckets) at += boff[b] - b * P.fcap;
      }
      sm.sbo[nsub] = at;
    }
  } else {
    for (int i = tid; i <= nsub; i += blockDim.x)
      sm.sbo[i] = boff[min(sm.tile * nsub + i, nbuckets)];
  }
  __syncthreads();
  const int64_t s = sm.sbo[0];
  const int n = sm.sbo[nsub] - (int)s;
  bool fast = n <= kTileCap;
  // fast path: every item loaded once into registers (all loads in flight
  // together), histogram by node; it needs every node <= 32 occurrences
  uint64_t itr[kTilePer];
  int ndr[kTilePer];
  if (fast) {
#pragma unroll
    for (int k = 0; k < kTilePer; ++k) {
      if (k * kTileThreads >= n) break;  // block-uniform (~6 of the 10 slots hold items on refined meshes)
      const int p = tid + k * kTileThreads;
      itr[k] = p < n ? __ldg(items + s + p) : 0ull;
    }
    const int64_t s_lo = s;
#pragma unroll
    for (int k = 0; k < kTilePer; ++k) {
      if (k * kTileThreads >= n) break;
      const int p = tid + k * kTileThreads;
      ndr[k] = 0;
      if (p < n) {
        int sub = 0;  // sub-bucket of position p (nsub <= 256 >> bs, uniform trip count)
        for (int m = 1; m < nsub; ++m) sub += p >= sm.sbo[m] - (int)s_lo;
        ndr[k] = (sub << P.bs) | (int)(itr[k] >> P.total_bits);
      }
    }
    int cme;
    if (try_col) {
      // straight into the node columns: the per-node cursor is the histogram
      uint64_t* col = sm.buf1 + kTileNodes;
      sm.buf1[tid] = 0ull;  // sentinel row
#pragma unroll
      for (int k = 0; k < kTilePer; ++k) {
        if (k * kTileThreads >= n) break;
        if (tid + k * kTileThreads < n) {
          const int j = atomicAdd(&sm.cur[ndr[k]], 1);
          if (j < kColK) col[j * kTileNodes + ndr[k]] = itr[k];
        }
      }
      __syncthreads();
      cme = sm.cur[tid];
      if (__syncthreads_and(cme <= kColK)) {
        eg_tile_col(P, sm, rec, tileE, tileB, out, err, cme);
        return;
      }
      sm.cnt[tid] = cme;  // the histogram for the paths below
    } else {
#pragma unroll
      for (int k = 0; k < kTilePer; ++k) {
        if (k * kTileThreads >= n) break;
        if (tid + k * kTileThreads < n) atomicAdd(&sm.cnt[ndr[k]], 1);
      }
      __syncthreads();
      cme = sm.cnt[tid];
    }
    fast = __syncthreads_and(cme <= 32);
  }
  if (fast) {
    eg_tile_fast(items, P, sm, rec, tileE, tileB, out, err, itr, ndr);
    return;
  }
  sm.cnt[tid] = 0;
  __syncthreads();
  if (n <= kTileCap)
    eg_tile<true>(items, P, sm, g1, g2, gnode, rec, tileE, tileB, out, err);
  else
    eg_tile<false>(items, P, sm, g1, g2, gnode, rec, tileE, tileB, out, err);
}

// One tile per CTA, every path (PHFEM_TILE_SPLIT=0).
__global__ void __launch_bounds__(kTileThreads, PHFEM_TILE_MIN_BLOCKS) k_eg_tile(const uint64_t* __restrict__ items,
                                                          const int32_t* __restrict__ boff,
                                                          int nbuckets, EgParams P, uint64_t* g1,
                                                          uint64_t* g2, uint8_t* gnode,
                                                          int4* __restrict__ rec,
                                                          int32_t* __restrict__ tileE,
                                                          int32_t* __restrict__ tileB, EgOut out,
                                                          phfem_dev_errors* err) {
  extern __shared__ __align__(16) unsigned char smraw[];
  TileSmem& sm = *reinterpret_cast<TileSmem*>(smraw);
  eg_tile_body(sm, blockIdx.x, PHFEM_TILE_COL != 0, items, boff, nbuckets, P, g1, g2, gnode, rec, tileE, tileB,
               out, err);
}

// The tiles k_eg_tile_col left (a node with > kColK occurrences): a
// persistent grid over the device-side list, the item-parallel / general paths.
__global__ void __launch_bounds__(kTileThreads, PHFEM_TILE_MIN_BLOCKS) k_eg_tile_list(
    const int32_t* __restrict__ list, const int32_t* __restrict__ count, uint64_t* __restrict__ items,
    const int32_t* __restrict__ boff, int nbuckets, EgParams P, uint64_t* g1, uint64_t* g2, uint8_t* gnode,
    int4* __restrict__ rec, int32_t* __restrict__ tileE, int32_t* __restrict__ tileB, EgOut out,
    phfem_dev_errors* err) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char smraw[];
  TileSmem& sm = *reinterpret_cast<TileSmem*>(smraw);
  const int nl = *count;
  const int nsub = kTileNodes >> P.bs;
  for (int w = blockIdx.x; w < nl; w += gridDim.x) {
    const int tile = list[w];
    if (P.fcap) {
      // fixed layout (boff = the bucket fills): close the gaps between the
      // tile's sub-buckets so its items are contiguous (staged through SMEM:
      // the ranges may overlap)
      int at = boff[tile * nsub] - tile * nsub * P.fcap;
      for (int i = 1; i < nsub; ++i) {
        const int b = tile * nsub + i;
        if (b >= nbuckets) break;
        const int cnt = boff[b] - b * P.fcap;
        const int64_t src = (int64_t)b * P.fcap, dst = (int64_t)tile * nsub * P.fcap + at;
        if (src != dst && cnt > 0) {  // block-uniform
          for (int p = threadIdx.x; p < cnt; p += blockDim.x) sm.buf1[p] = items[src + p];
          __syncthreads();
          for (int p = threadIdx.x; p < cnt; p += blockDim.x) items[dst + p] = sm.buf1[p];
          __syncthreads();
        }
        at += cnt;
      }
      __syncthreads();
    }
    eg_tile_body(sm, tile, false, items, boff, nbuckets, P, g1, g2, gnode, rec, tileE, tileB, out, err);
    __syncthreads();
  }
}

// Column kernel (PHFEM_TILE_SPLIT=1, the default): only the column path, in
// 30 KB of SMEM and 32 registers, without the register-staged items of the
// other paths (7 resident CTAs instead of 4); a tile with a node of more than
// kColK2 occurrences is handed to k_eg_tile_list.
#ifndef PHFEM_TILE_SPLIT
#define PHFEM_TILE_SPLIT 1
#endif
#ifndef PHFEM_COL_MIN_BLOCKS
#define PHFEM_COL_MIN_BLOCKS 7
#endif
// item loads in flight per thread in the column scatter (measured at L12 /
// given L13: 1 -> 0.884 / 3.51 ms, 2 -> 0.866 / 3.44, 4 -> 0.855 / 3.40)
#ifndef PHFEM_COL_LD
#define PHFEM_COL_LD 4
#endif
#ifndef PHFEM_COL_K
#define PHFEM_COL_K 13  // occurrences per node (refined meshes: <= 12); 14 rows of 2 KB: 7 CTAs per SM
#endif
constexpr int kColK2 = PHFEM_COL_K;
struct ColSmem {
  uint64_t col[(kColK2 + 1) * kTileNodes];  // row 0: zero sentinels; node t's j-th occurrence at [j + 1][t]
  int32_t cur[kTileNodes];
  int32_t sbo[kTileNodes / 2 + 1];  // bs >= 1: at most 128 sub-buckets per tile
  unsigned long long scan[33];
};

// Thread = node.  (Measured and dropped: slots ordered by occurrence count, so
// that a warp's 32 nodes sort / walk equally many occurrences — an extra
// histogram pass and the slot indirection cost more than the divergence they
// remove: L12 tile 0.885 -> 0.990 ms.)
__device__ __forceinline__ void eg_tile_col_body(
    int tile, ColSmem& sm, const uint64_t* __restrict__ items, const int32_t* __restrict__ boff, int nbuckets,
    const EgParams& P, int4* __restrict__ rec, int32_t* __restrict__ tileE, int32_t* __restrict__ tileB,
    const EgOut& out, phfem_dev_errors* err, int32_t* __restrict__ fb_list, int32_t* __restrict__ fb_count) {
  const int tid = threadIdx.x;
  sm.cur[tid] = 0;
  sm.col[tid] = 0ull;
  const int nsub = kTileNodes >> P.bs;
  for (int i = tid; i <= nsub; i += blockDim.x) sm.sbo[i] = boff[min(tile * nsub + i, nbuckets)];
  __syncthreads();
  int s;  // the tile's first record slot
  if (P.fcap) {
    // fixed layout (boff = the bucket fills): each sub-bucket read from its own slots
    s = tile * nsub * P.fcap;
    for (int sub = 0; sub < nsub; ++sub) {
      const int b = tile * nsub + sub;
      if (b >= nbuckets) break;
      const int base = b * P.fcap;
      const int cnt = sm.sbo[sub] - base;
#if PHFEM_COL_LD > 1
      // PHFEM_COL_LD item loads in flight per thread before their column slots
      for (int p0 = tid; p0 < cnt; p0 += PHFEM_COL_LD * kTileThreads) {
        uint64_t it[PHFEM_COL_LD];
#pragma unroll
        for (int u = 0; u < PHFEM_COL_LD; ++u)
          if (p0 + u * kTileThreads < cnt) it[u] = __ldg(items + base + p0 + u * kTileThreads);
#pragma unroll
        for (int u = 0; u < PHFEM_COL_LD; ++u)
          if (p0 + u * kTileThreads < cnt) {
            const int nd = (sub << P.bs) | (int)(it[u] >> P.total_bits);
            const int j = atomicAdd(&sm.cur[nd], 1);
            if (j < kColK2) sm.col[(j + 1) * kTileNodes + nd] = it[u];
          }
      }
#else
      for (int p = tid; p < cnt; p += kTileThreads) {
        const uint64_t it = __ldg(items + base + p);
        const int nd = (sub << P.bs) | (int)(it >> P.total_bits);
        const int j = atomicAdd(&sm.cur[nd], 1);
        if (j < kColK2) sm.col[(j + 1) * kTileNodes + nd] = it;
      }
#endif
    }
  } else {
    s = sm.sbo[0];
    const int n = sm.sbo[nsub] - s;
    if (n > kColK2 * kTileNodes) {  // block-uniform
      if (tid == 0) fb_list[atomicAdd(fb_count, 1)] = tile;
      return;
    }
    for (int p = tid; p < n; p += kTileThreads) {
      const uint64_t it = __ldg(items + s + p);
      int sub = 0;
      if (nsub > 1) {  // sub-bucket of position p
        int lo = 0, hi = nsub - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (sm.sbo[mid] - s <= p) lo = mid;
          else hi = mid - 1;
        }
        sub = lo;
      }
      const int nd = (sub << P.bs) | (int)(it >> P.total_bits);
      const int j = atomicAdd(&sm.cur[nd], 1);
      if (j < kColK2) sm.col[(j + 1) * kTileNodes + nd] = it;
    }
  }
  __syncthreads();
  const int c = sm.cur[tid];
  if (!__syncthreads_and(c <= kColK2)) {
    if (tid == 0) fb_list[atomicAdd(fb_count, 1)] = tile;
    return;
  }
  const int ob = P.occ_bits;
  const int lsh = ob + 1;
  const uint64_t lomask = (1ull << P.lo_bits) - 1ull;
  uint64_t* my = sm.col + kTileNodes + tid;
  for (int i = 1; i < c; ++i) {  // insertion sort, the zero row ends every walk
    uint64_t* r = my + (i - 1) * kTileNodes;
    const uint64_t x = r[kTileNodes];
    uint64_t y0 = *r;
    // two shifts per trip with alternating registers: no copies of the
    // loop-carried key (the load of the next one is hoisted above the store)
    while (y0 > x) {
      r[kTileNodes] = y0;
      const uint64_t y1 = r[-kTileNodes];
      r -= kTileNodes;
      if (!(y1 > x)) break;
      r[kTileNodes] = y1;
      y0 = r[-kTileNodes];
      r -= kTileNodes;
    }
    r[kTileNodes] = x;
  }
  const uint64_t v_glob = (uint64_t)P.node_base + (uint64_t)tile * kTileNodes + tid;
  int ne = 0, nb = 0;
  for (int i = 0; i < c;) {
    const uint64_t f = my[i * kTileNodes];
    const uint64_t lo = (f >> lsh) & lomask;
    int len = 1;
    while (i + len < c && ((my[(i + len) * kTileNodes] >> lsh) & lomask) == lo) ++len;
    if (len > 2 || (len == 2 && ((f ^ my[(i + 1) * kTileNodes]) & 1ull) == 0))
      atomicMin(&err->topo, (v_glob << 33) | (lo << 2) | (len > 2 ? 0ull : (2ull | (f & 1ull))));
    ++ne;
    nb += len == 1;
    i += len;
  }
  unsigned long long agg;
  const unsigned long long ex = block_exclusive_scan(((unsigned long long)ne << 32) | nb, sm.scan, &agg);
  int32_t e = (int32_t)(ex >> 32);
  int32_t bl = (int32_t)(ex & 0xffffffffu);
  const int64_t v_me = (int64_t)tile * kTileNodes + tid;
  if (v_me < P.nC) out.node_edge_start[v_me] = e;
  for (int i = 0; i < c;) {
    const uint64_t f = my[i * kTileNodes];
    const uint64_t lo = (f >> lsh) & lomask;
    const uint64_t g = i + 1 < c ? my[(i + 1) * kTileNodes] : 0ull;
    const bool two = i + 1 < c && ((g >> lsh) & lomask) == lo;
    int len = two ? 2 : 1;
    while (i + len < c && ((my[(i + len) * kTileNodes] >> lsh) & lomask) == lo) ++len;
    const bool neu = !two && out.neu_keys && neu_pair_has(out, (int)lo, (int32_t)v_glob);
    if (neu) atomicAdd(&out.tileN[tile], 1);
    rec[s + e] = eg_record(tid, bl, (int32_t)lo, f, two ? g : 0ull, two, ob, neu);
    ++e;
    bl += !two;
    i += len;
  }
  if (tid == 0) {
    tileE[tile] = (int32_t)(agg >> 32);
    tileB[tile] = (int32_t)(agg & 0xffffffffu);
  }
}

__global__ void __launch_bounds__(kTileThreads, PHFEM_COL_MIN_BLOCKS) k_eg_tile_col(
    const uint64_t* __restrict__ items, const int32_t* __restrict__ boff, int nbuckets, EgParams P,
    int4* __restrict__ rec, int32_t* __restrict__ tileE, int32_t* __restrict__ tileB, EgOut out,
    phfem_dev_errors* err, int32_t* __restrict__ fb_list, int32_t* __restrict__ fb_count, int ntiles) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char smraw[];
  ColSmem& sm = *reinterpret_cast<ColSmem*>(smraw);
  // one CTA per tile (measured: a grid-stride loop over tiles with 16 / 64 /
  // 256 CTAs per SM, 1.00 / 0.93 / 0.92 ms against 0.89 at L12)
  (void)ntiles;
  eg_tile_col_body(blockIdx.x, sm, items, boff, nbuckets, P, rec, tileE, tileB, out, err, fb_list, fb_count);
}

// E ------------------------------------------------------------------------
// One CTA per tile: the tile's edge records (consecutive, tile-local) become
// the final outputs at the scanned tile offsets — coalesced record reads and
// edge-array writes; ids are canonical because tiles are max-node ranges.
constexpr int kEmitThreads = kTileNodes;
#ifndef PHFEM_EMIT_MIN_BLOCKS
#define PHFEM_EMIT_MIN_BLOCKS 4
#endif
__global__ void __launch_bounds__(kEmitThreads, PHFEM_EMIT_MIN_BLOCKS) k_eg_emit(const int4* __restrict__ rec,
                                                          const int32_t* __restrict__ boff,
                                                          int nbuckets, int nsub,
                                                          const int32_t* __restrict__ tileE,
                                                          const int32_t* __restrict__ tileB, int nC,
                                                          EgOut out, int ntiles) {
  pdl_wait();
  pdl_trigger();
  // one CTA per tile (measured: a grid-stride loop over tiles with 16 / 64 /
  // 256 CTAs per SM, 0.68 / 0.62 / 0.58 ms against 0.57 at L12)
  const int tile = blockIdx.x;
  const int64_t s = boff[min(tile * nsub, nbuckets)];
  const int E0 = tileE[tile], ne = tileE[tile + 1] - E0;
  const int B0 = tileB[tile];
  const int64_t vme = (int64_t)tile * kTileNodes + threadIdx.x;
  if (vme < nC) out.node_edge_start[vme] += E0;
  if (tile == ntiles - 1 && threadIdx.x == 0) out.node_edge_start[nC] = E0 + ne;
  // one record per thread, 4 in flight: no scan (records carry their
  // tile-local boundary prefix); the fused classification + C also needs
  // the Neumann edges before each record: one packed block scan per trip
  const int64_t vbase = (int64_t)out.node_base + (int64_t)tile * kTileNodes;
  const bool fused = out.rpos != nullptr;
  __shared__ unsigned long long nscan[33];
  int nrun = fused ? out.tileN[tile] : 0;  // Neumann edges before the trip (global)
  for (int i00 = 0; i00 < ne; i00 += 4 * kEmitThreads) {
    const int i0 = i00 + threadIdx.x;
    int4 r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * kEmitThreads;
      if (i < ne) r[u] = rec[s + i];
    }
    int nb4[4] = {0, 0, 0, 0};  // Neumann edges before each of the thread's records
    if (fused) {
      unsigned long long f = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i0 + u * kEmitThreads < ne && r[u].w == -2) f |= 1ull << (16 * u);
      unsigned long long tot;
      const unsigned long long ex = block_exclusive_scan(f, nscan, &tot);
      int base = nrun;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        nb4[u] = base + (int)((ex >> (16 * u)) & 0xffff);
        base += (int)((tot >> (16 * u)) & 0xffff);
      }
      nrun = base;
    }
    const int warp = threadIdx.x >> 5;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (i00 + u * kEmitThreads + 32 * warp >= ne) break;  // warp-uniform exit past the tile's records
      const int i = i0 + u * kEmitThreads;
      const bool ok = i < ne;
      const int32_t e = E0 + i;
      int m_f = 0, l_f = 0, m_g = 0, l_g = -1, rs = 0, nn = 0;
      bool row = false;
      double len = 0.0;
      if (ok) {
        const int32_t v = (int32_t)(vbase + (r[u].x & 0xff));
        const int32_t bpos = B0 + (r[u].x >> 8);  // boundary edges before e
        const uint32_t z = (uint32_t)r[u].z;
        const uint32_t occ_f = z >> 1;
        m_f = (int)(occ_f / 3u);
        l_f = (int)((occ_f % 3u + 2u) % 3u);  // slot s -> local (s + 2) % 3
        reinterpret_cast<int2*>(out.edge_nodes)[e] = (z & 1u) ? make_int2(v, r[u].y) : make_int2(r[u].y, v);
        out.ltp[e] = l_f;
        if (r[u].w >= 0) {
          const uint32_t occ_g = (uint32_t)r[u].w;
          m_g = (int)(occ_g / 3u);
          l_g = (int)((occ_g % 3u + 2u) % 3u);
          reinterpret_cast<int2*>(out.edge_elements)[e] = make_int2(m_f, m_g);
          out.ltm[e] = l_g;
          eg_slots(out, e, 3 * (int64_t)m_f + l_f, 3 * (int64_t)m_g + l_g);
          out.interior[e - bpos] = e;
        } else {
          reinterpret_cast<int2*>(out.edge_elements)[e] = make_int2(m_f, -1);
          out.ltm[e] = -1;
          eg_slots(out, e, 3 * (int64_t)m_f + l_f, -1);
          out.boundary[bpos] = e;
        }
        if (fused) {  // classify_edges + assemble_constraint (edge_topology.cpp:165-173; assembly.cpp:144-168)
          const bool neu = r[u].w == -2;
          const int nl = nb4[u];
          if (neu) {
            out.rpos[e] = -1;
          } else {
            const int rp = e - nl;
            rs = 4 * rp - 2 * (bpos - nl);  // retained boundary rows hold 2 entries
            nn = r[u].w >= 0 ? 4 : 2;
            row = true;
            out.rpos[e] = rp;
            out.redges[rp] = e;
            out.row_ptr[rp] = rs;
            if (rp == out.L - 1) out.row_ptr[out.L] = rs + nn;
            const int a = (z & 1u) ? v : r[u].y, b = (z & 1u) ? r[u].y : v;
            const double2 pa = out.coords[a], pb = out.coords[b];
            const double dx = pb.x - pa.x, dy = pb.y - pa.y;
            len = sqrt(dx * dx + dy * dy);  // edge_topology.cpp:183
          }
        }
      }
      if (fused && row) {
        // direct stores: an interior row at a 32-byte aligned entry as one
        // 16-byte column + one 32-byte value store (STG.256); measured against
        // the per-warp SMEM staging of round 2 (whole-line stores): emit on the
        // given L13 mesh 5.15 -> 4.69 ms
        const int c0 = l_f == 0 ? 1 : 0, c1 = l_f == 2 ? 1 : 2;
        const double vp = len * 0.5;  // assembly.cpp:160
        if (nn == 4 && ((reinterpret_cast<uintptr_t>(out.val + rs) & 31) == 0) &&
            ((reinterpret_cast<uintptr_t>(out.col + rs) & 15) == 0)) {
          const int d0 = l_g == 0 ? 1 : 0, d1 = l_g == 2 ? 1 : 2;
          const double vm = -len * 0.5;  // assembly.cpp:164
          *reinterpret_cast<int4*>(out.col + rs) = make_int4(3 * m_f + c0, 3 * m_f + c1, 3 * m_g + d0, 3 * m_g + d1);
          asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(out.val + rs), "d"(vp), "d"(vp),
                       "d"(vm), "d"(vm)
                       : "memory");
        } else {
          out.col[rs] = 3 * m_f + c0;
          out.col[rs + 1] = 3 * m_f + c1;
          out.val[rs] = vp;
          out.val[rs + 1] = vp;
          if (nn == 4) {
            const int d0 = l_g == 0 ? 1 : 0, d1 = l_g == 2 ? 1 : 2;
            const double vm = -len * 0.5;  // assembly.cpp:164
            out.col[rs + 2] = 3 * m_g + d0;
            out.col[rs + 3] = 3 * m_g + d1;
            out.val[rs + 2] = vm;
            out.val[rs + 3] = vm;
          }
        }
      }
    }
  }
}

__global__ void k_eg_tile_max(const int32_t* __restrict__ boff, int nbuckets, int nsub, int ntiles,
                              phfem_dev_errors* err) {
  int mx = 0;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += gridDim.x * blockDim.x)
    mx = max(mx, boff[min((t + 1) * nsub, nbuckets)] - boff[t * nsub]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane_id() == 0) atomicMax(&err->counters[3], (unsigned long long)mx);
}

}  // namespace phfem

using namespace phfem;

PHFEM_API void phfem_topology_release(phfem_ctx* ctx, phfem_topology* t) {
  if (!t) return;
  dfree(ctx, t->edge_nodes);
  dfree(ctx, t->edge_elements);
  dfree(ctx, t->local_in_tplus);
  dfree(ctx, t->local_in_tminus);
  dfree(ctx, t->interior_edges);
  dfree(ctx, t->boundary_edges);
  dfree(ctx, t->elem_edge);
  dfree(ctx, t->node_edge_start);
  t->E = t->n_interior = t->n_boundary = 0;
}

namespace phfem {

// Sort -> records -> emit over nd occurrences of one max-node key range
// (the whole mesh for build_topology, one rank's range for the distributed
// dedup).  source(kind, ...) launches the histogram (kind 0) or the scatter
// (kind 1) of the occurrences into the bucket array.
// Fused classification + C of a sort-built topology (pipeline_impl): the
// Neumann pairs' hash set in, retained arrays and C (CSR) out.
struct EgFuse {
  const unsigned long long* keys;
  int cap;
  const double* coords;
  phfem_classification* cls;  // retained_pos / retained_edges allocated here, L set
  phfem_csr* C;
  int32_t nE;                 // elements (columns of C = 3 nE)
};

// the rank's own element slots of a distributed dedup (eg_slots)
struct EgOwn {
  int32_t* ee;
  int64_t lo3, hi3;
  int32_t* npairs;  // device counter, zeroed by the caller
};

// items already scattered into their buckets by the senders (distributed
// input level with peer windows): the bucket offsets and the item array
struct EgPre {
  const int32_t* boff;  // [nb + 1] exclusive bucket offsets
  uint64_t* items;      // [nd] packed items, bucketed
};

template <typename Source>
#ifndef PHFEM_EG_FIXED
#define PHFEM_EG_FIXED 1
#endif
// fixed_elements: the mesh's elements when the occurrences come from them —
// then the fixed-capacity bucket layout (no count pass) is tried first
static phfem_status eg_core(phfem_ctx* ctx, EgParams P, int64_t nd, Source source,
                            phfem_topology* out, int2* pairs, const char* who,
                            const EgFuse* fuse = nullptr, const EgOwn* own = nullptr,
                            const EgPre* pre = nullptr, const int32_t* fixed_elements = nullptr) {
  const int64_t nC = P.nC;
  const int64_t cap_e = std::max<int64_t>(nd, 1);
  PHFEM_TRY(dalloc(ctx, &out->node_edge_start, nC + 1));
  PHFEM_TRY(dalloc(ctx, &out->edge_nodes, 2 * cap_e));
  PHFEM_TRY(dalloc(ctx, &out->edge_elements, 2 * cap_e));
  PHFEM_TRY(dalloc(ctx, &out->local_in_tplus, cap_e));
  PHFEM_TRY(dalloc(ctx, &out->local_in_tminus, cap_e));
  PHFEM_TRY(dalloc(ctx, &out->interior_edges, cap_e / 2 + 1));
  PHFEM_TRY(dalloc(ctx, &out->boundary_edges, cap_e));
  if (!pairs) PHFEM_TRY(dalloc(ctx, &out->elem_edge, cap_e));
  if (nd == 0) {
    PHFEM_CUDA(ctx, cudaMemsetAsync(out->node_edge_start, 0, sizeof(int32_t) * (nC + 1), ctx->stream));
    return PHFEM_OK;
  }

  PHFEM_TRY(errors_reset(ctx));
  int32_t *bcount = nullptr, *boff = nullptr, *tiles = nullptr;
  const int ntiles = (int)((nC + kTileNodes - 1) / kTileNodes);
  PHFEM_TRY(dalloc(ctx, &bcount, (int64_t)P.nb + 1));
  PHFEM_TRY(dalloc(ctx, &boff, (int64_t)P.nb + 1));
  PHFEM_TRY(dalloc(ctx, &tiles, 2 * ((int64_t)ntiles + 1)));
  int32_t* tileE = tiles;
  int32_t* tileB = tiles + ntiles + 1;
  PHFEM_CUDA(ctx, cudaMemsetAsync(bcount, 0, sizeof(int32_t) * (P.nb + 1), ctx->stream));
  PHFEM_CUDA(ctx, cudaMemsetAsync(tiles, 0, sizeof(int32_t) * 2 * (ntiles + 1), ctx->stream));

  const int nsub = kTileNodes >> P.bs;
  int32_t* cursor = bcount;  // the scatter cursors (fixed layout: also the bucket fills)
  uint64_t* items = nullptr;
  uint64_t *g1 = nullptr, *g2 = nullptr;
  uint8_t* gnode = nullptr;
  int4* rec = nullptr;
  auto range_error = [&]() -> phfem_status {
    const long long m = (long long)ctx->herr->misc;
    dfree(ctx, items); dfree(ctx, rec);
    dfree(ctx, bcount); dfree(ctx, boff); dfree(ctx, tiles);
    phfem_topology_release(ctx, out);
    if (pairs)
      return set_error(ctx, PHFEM_ERR_OUT_OF_RANGE, "%s: occurrence %lld outside the key range", who, m);
    return set_error(ctx, PHFEM_ERR_OUT_OF_RANGE,
                     "build_topology: element %lld has a node index outside 1..%lld", m + 1,
                     (long long)nC);
  };
  // Fixed-capacity layout first (elements as the source, column tile kernel):
  // every bucket owns kTileCap / nsub item slots, so the scatter needs no
  // count pass / scan; a bucket over its capacity (some tile could not be
  // processed in SMEM anyway) falls back to the counted layout below.
  const int fcap = kTileCap / nsub;
  bool fixed = fixed_elements && !pre && PHFEM_EG_FIXED && PHFEM_TILE_SPLIT &&
               (int64_t)P.nb * fcap < (int64_t(1) << 31) - kTileCap;
  if (fixed) {
    const int64_t capn = (int64_t)P.nb * fcap;
    PHFEM_LAUNCH(ctx, "k_eg_fixed_init", k_eg_fixed_init<<<grid_for((int64_t)P.nb + 1, 256, ctx->num_sms * 4), 256, 0,
                                                           ctx->stream>>>(boff, cursor, P.nb, fcap));
    PHFEM_TRY(dalloc(ctx, &items, capn));
    PHFEM_TRY(dalloc(ctx, &rec, capn));
    P.fcap = fcap;
    const int grid_e = grid_for(P.nE, 256, ctx->num_sms * PHFEM_SC_GRID_MULT);
    PHFEM_LAUNCH(ctx, "k_eg_scatter", k_eg_scatter_fixed<<<grid_e, 256, 0, ctx->stream>>>(fixed_elements, P, cursor,
                                                                                         items, ctx->derr));
    PHFEM_TRY(errors_fetch(ctx));
    if (ctx->herr->misc != ~0ull) return range_error();
    if ((int64_t)ctx->herr->counters[3] > fcap) {  // a bucket over capacity: counted layout
      dfree(ctx, items);
      dfree(ctx, rec);
      P.fcap = 0;
      fixed = false;
      PHFEM_CUDA(ctx, cudaMemsetAsync(bcount, 0, sizeof(int32_t) * (P.nb + 1), ctx->stream));
      PHFEM_TRY(errors_reset(ctx));
    }
  }
  if (!fixed) {
    if (pre) {
      PHFEM_CUDA(ctx, cudaMemcpyAsync(boff, pre->boff, sizeof(int32_t) * ((int64_t)P.nb + 1), cudaMemcpyDeviceToDevice,
                                      ctx->stream));
    } else {
      PHFEM_TRY(source(0, bcount, (uint64_t*)nullptr));
      PHFEM_TRY(scan_exclusive_i32(ctx, bcount, boff, (int64_t)P.nb + 1, nullptr));
    }
    PHFEM_LAUNCH(ctx, "k_eg_tile_max", k_eg_tile_max<<<grid_for(ntiles, 256, ctx->num_sms * 4), 256, 0, ctx->stream>>>(
        boff, P.nb, nsub, ntiles, ctx->derr));
    PHFEM_CUDA(ctx, cudaMemcpyAsync(cursor, boff, sizeof(int32_t) * P.nb, cudaMemcpyDeviceToDevice,
                                    ctx->stream));
    PHFEM_TRY(errors_fetch(ctx));
    if (ctx->herr->misc != ~0ull) return range_error();
    const int64_t max_tile = (int64_t)ctx->herr->counters[3];
    if (pre) items = pre->items;
    else PHFEM_TRY(dalloc(ctx, &items, nd));
    PHFEM_TRY(dalloc(ctx, &rec, nd));
    if (max_tile > kTileCap) {  // some tile does not fit SMEM: global scratch
      PHFEM_TRY(dalloc(ctx, &g1, nd));
      PHFEM_TRY(dalloc(ctx, &g2, nd));
      PHFEM_TRY(dalloc(ctx, &gnode, nd));
    }
    if (!pre) PHFEM_TRY(source(1, cursor, items));
  }
  // the tile kernels' bucket array: the fills in the fixed layout, else the offsets
  const int32_t* tboff = fixed ? cursor : boff;

  EgOut o;
  memset(&o, 0, sizeof o);
  o.edge_nodes = out->edge_nodes;
  o.edge_elements = out->edge_elements;
  o.ltp = out->local_in_tplus;
  o.ltm = out->local_in_tminus;
  o.interior = out->interior_edges;
  o.boundary = out->boundary_edges;
  o.elem_edge = out->elem_edge;
  o.node_edge_start = out->node_edge_start;
  o.pairs = pairs;
  if (own) {
    o.self_ee = own->ee;
    o.self_lo3 = own->lo3;
    o.self_hi3 = own->hi3;
    o.npairs = own->npairs;
  }
  o.node_base = P.node_base;
  int32_t* tileN = nullptr;
  if (fuse) {
    PHFEM_TRY(dalloc(ctx, &tileN, (int64_t)ntiles + 2));
    PHFEM_CUDA(ctx, cudaMemsetAsync(tileN, 0, sizeof(int32_t) * (ntiles + 2), ctx->stream));
    o.neu_keys = fuse->keys;
    o.neu_cap = fuse->cap;
    o.tileN = tileN;
    o.coords = (const double2*)fuse->coords;
  }
  EgParams PT = P;
  PT.nb = ntiles;
  const size_t smem = sizeof(TileSmem);
  if (PHFEM_TILE_SPLIT) {
    // column kernel over every tile, then the list of tiles it handed back
    int32_t* fb = nullptr;
    PHFEM_TRY(dalloc(ctx, &fb, (int64_t)ntiles + 1));
    PHFEM_CUDA(ctx, cudaMemsetAsync(fb, 0, sizeof(int32_t), ctx->stream));
    const size_t csmem = sizeof(ColSmem);
    PHFEM_TRY(smem_optin(ctx, (const void*)k_eg_tile_col, csmem, "k_eg_tile_col smem opt-in"));
    PHFEM_LAUNCH_PDL(ctx, "k_eg_tile", k_eg_tile_col, (unsigned)ntiles, kTileThreads, csmem,
        (const uint64_t*)items, tboff, (int)P.nb, PT, rec, tileE, tileB, o, ctx->derr, fb + 1, fb, (int)ntiles);
    PHFEM_TRY(smem_optin(ctx, (const void*)k_eg_tile_list, smem, "k_eg_tile_list smem opt-in"));
    PHFEM_LAUNCH_PDL(ctx, "k_eg_tile_list", k_eg_tile_list, ctx->num_sms * 4, kTileThreads, smem,
        (const int32_t*)(fb + 1), (const int32_t*)fb, items, tboff, (int)P.nb, PT, g1, g2, gnode, rec,
        tileE, tileB, o, ctx->derr);
    dfree(ctx, fb);
  } else {
    PHFEM_TRY(smem_optin(ctx, (const void*)k_eg_tile, smem, "k_eg_tile smem opt-in"));
    PHFEM_LAUNCH(ctx, "k_eg_tile", k_eg_tile<<<ntiles, kTileThreads, smem, ctx->stream>>>(
        items, boff, P.nb, PT, g1, g2, gnode, rec, tileE, tileB, o, ctx->derr));
  }
  {
    const int32_t* in[3] = {tileE, tileB, tileN};
    int32_t* io[3] = {tileE, tileB, tileN};
    PHFEM_TRY(scan_exclusive_i32_set(ctx, fuse ? 3 : 2, in, io, (int64_t)ntiles + 1, nullptr));
  }
  if (fuse) {  // sizes of the classification / C before the emit pass writes them
    int32_t h[3] = {0, 0, 0};
    PHFEM_CUDA(ctx, cudaMemcpyAsync(&h[0], tileE + ntiles, 4, cudaMemcpyDeviceToHost, ctx->stream));
    PHFEM_CUDA(ctx, cudaMemcpyAsync(&h[1], tileB + ntiles, 4, cudaMemcpyDeviceToHost, ctx->stream));
    PHFEM_CUDA(ctx, cudaMemcpyAsync(&h[2], tileN + ntiles, 4, cudaMemcpyDeviceToHost, ctx->stream));
    PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    const int64_t E = h[0], nB = h[1], nneu = h[2];
    const int64_t L = E - nneu;
    phfem_classification* cls = fuse->cls;
    phfem_csr* C = fuse->C;
    cls->E = (int32_t)E;
    cls->L = (int32_t)L;
    PHFEM_TRY(dalloc(ctx, &cls->retained_pos, std::max<int64_t>(E, 1)));
    PHFEM_TRY(dalloc(ctx, &cls->retained_edges, std::max<int64_t>(L, 1)));
    C->rows = (int32_t)L;
    C->cols = 3 * fuse->nE;
    C->nnz = 4 * L - 2 * (nB - nneu);
    PHFEM_TRY(dalloc(ctx, &C->row_ptr, L + 1));
    PHFEM_TRY(dalloc(ctx, &C->col_idx, std::max<int64_t>(C->nnz, 1)));
    PHFEM_TRY(dalloc(ctx, &C->values, std::max<int64_t>(C->nnz, 1)));
    if (L == 0) PHFEM_CUDA(ctx, cudaMemsetAsync(C->row_ptr, 0, sizeof(int32_t), ctx->stream));
    o.rpos = cls->retained_pos;
    o.redges = cls->retained_edges;
    o.row_ptr = C->row_ptr;
    o.col = C->col_idx;
    o.val = C->values;
    o.L = (int)L;
  }
  PHFEM_LAUNCH_PDL(ctx, "k_eg_emit", k_eg_emit, (unsigned)ntiles, kEmitThreads, 0,
      (const int4*)rec, (const int32_t*)boff, (int)P.nb, (int)nsub, (const int32_t*)tileE, (const int32_t*)tileB,
      (int)nC, o, (int)ntiles);
  // totals ride back with the error words (low 32 bits of counters 0 / 2)
  PHFEM_CUDA(ctx, cudaMemcpyAsync(&ctx->derr->counters[0], tileE + ntiles, sizeof(int32_t),
                                  cudaMemcpyDeviceToDevice, ctx->stream));
  PHFEM_CUDA(ctx, cudaMemcpyAsync(&ctx->derr->counters[2], tileB + ntiles, sizeof(int32_t),
                                  cudaMemcpyDeviceToDevice, ctx->stream));
  if (!pre) dfree(ctx, items);
  dfree(ctx, rec);
  dfree(ctx, g1);
  dfree(ctx, g2);
  dfree(ctx, gnode);
  dfree(ctx, bcount);
  dfree(ctx, boff);
  dfree(ctx, tiles);
  dfree(ctx, tileN);
  PHFEM_TRY(errors_fetch(ctx));
  const uint64_t te = ctx->herr->topo;
  if (te != ~0ull) {
    const long long hi = (long long)(te >> 33);
    const long long lo = (long long)((te >> 2) & ((1ull << 31) - 1));
    const bool dup = (te >> 1) & 1ull;
    const bool dir = te & 1ull;
    phfem_topology_release(ctx, out);
    if (dup) {
      const long long from = dir ? hi : lo, to = dir ? lo : hi;
      return set_error(ctx, PHFEM_ERR_DUP_DIRECTED, "build_topology: duplicate directed edge %lld->%lld",
                       from + 1, to + 1);
    }
    return set_error(ctx, PHFEM_ERR_NONMANIFOLD,
                     "build_topology: non-manifold edge (%lld,%lld) shared by more than two elements",
                     lo + 1, hi + 1);
  }
  out->E = (int32_t)(ctx->herr->counters[0] & 0xffffffffu);
  out->n_boundary = (int32_t)(ctx->herr->counters[2] & 0xffffffffu);
  out->n_interior = out->E - out->n_boundary;
  return PHFEM_OK;
}

static phfem_status eg_params(phfem_ctx* ctx, int64_t nC_range, int64_t nC_all, int64_t nE_all,
                              int32_t node_base, EgParams* P) {
  P->nC = (int32_t)nC_range;
  P->nE = (int32_t)nE_all;
  P->node_base = node_base;
  P->fcap = 0;
  P->lo_bits = bits_for(std::max<int64_t>(nC_all - 1, 1));
  P->occ_bits = bits_for(std::max<int64_t>(3 * nE_all - 1, 1));
  P->total_bits = P->lo_bits + P->occ_bits + 1;
  P->bs = std::min(ctx->eg_max_bs, 64 - P->total_bits);
  if (P->bs < 1) return set_error(ctx, PHFEM_ERR_INVALID_ARGUMENT, "build_topology: ids too wide");
  const int NB = 1 << P->bs;
  P->nb = (int)((nC_range + NB - 1) / NB);
  if (P->nb < 1) P->nb = 1;
  return PHFEM_OK;
}

}  // namespace phfem

PHFEM_API phfem_status phfem_build_topology(phfem_ctx* ctx, const phfem_mesh* mesh,
                                            phfem_topology* out) {
  memset(out, 0, sizeof(*out));
  if (!ctx || !mesh) return PHFEM_ERR_INVALID_ARGUMENT;
  if (cudaSetDevice(ctx->device) != cudaSuccess) return cuda_fail(ctx, cudaGetLastError(), "set device");
  const int64_t nE = mesh->nE, nC = mesh->nC;
  if (nE < 0 || nC < 0 || 3 * nE >= (int64_t(1) << 31))
    return set_error(ctx, PHFEM_ERR_INVALID_ARGUMENT, "build_topology: mesh too large for int ids");
  out->nC = (int32_t)nC;
  out->nE = (int32_t)nE;
  EgParams P;
  PHFEM_TRY(eg_params(ctx, nC, nC, nE, 0, &P));
  const int grid_e = grid_for(nE, 256, ctx->num_sms * 8);
  auto source = [&](int kind, int32_t* counts, uint64_t* items) -> phfem_status {
    if (kind == 0)
      PHFEM_LAUNCH(ctx, "k_eg_count", k_eg_count<<<grid_e, 256, 0, ctx->stream>>>(mesh->elements, P, counts, ctx->derr));
    else
      PHFEM_LAUNCH(ctx, "k_eg_scatter", k_eg_scatter<<<grid_e, 256, 0, ctx->stream>>>(mesh->elements, P, counts, items));
    return PHFEM_OK;
  };
  return eg_core(ctx, P, 3 * nE, source, out, nullptr, "build_topology", nullptr, nullptr, nullptr, mesh->elements);
}

PHFEM_API phfem_status phfem_dist_dedup_ex(phfem_ctx* ctx, const int32_t* recs, int64_t n,
                                           int32_t node_lo, int32_t node_hi, int32_t nC_all,
                                           int32_t nE_all, int32_t self_lo, int32_t self_hi,
                                           int32_t* self_elem_edge, phfem_topology* out, int32_t* pairs,
                                           int64_t* n_pairs) {
  memset(out, 0, sizeof(*out));
  if (!ctx || (!recs && n) || !pairs || node_lo < 0 || node_hi < node_lo || node_hi > nC_all ||
      3 * (int64_t)nE_all >= (int64_t(1) << 31))
    return PHFEM_ERR_INVALID_ARGUMENT;
  if (self_elem_edge && (self_lo < 0 || self_hi < self_lo || self_hi > nE_all || !n_pairs))
    return PHFEM_ERR_INVALID_ARGUMENT;
  if (n_pairs) *n_pairs = 0;
  out->nC = node_hi - node_lo;
  out->nE = nE_all;
  EgParams P;
  PHFEM_TRY(eg_params(ctx, (int64_t)node_hi - node_lo, nC_all, nE_all, node_lo, &P));
  const int grid_r = grid_for(n, 256, ctx->num_sms * 8);
  const int4* r4 = reinterpret_cast<const int4*>(recs);
  auto source = [&](int kind, int32_t* counts, uint64_t* items) -> phfem_status {
    if (kind == 0)
      PHFEM_LAUNCH(ctx, "k_rec_count", k_rec_count<<<grid_r, 256, 0, ctx->stream>>>(r4, n, P, counts, ctx->derr));
    else
      PHFEM_LAUNCH(ctx, "k_rec_scatter", k_rec_scatter<<<grid_r, 256, 0, ctx->stream>>>(r4, n, P, counts, items));
    return PHFEM_OK;
  };
  if (!self_elem_edge) {
    PHFEM_TRY(eg_core(ctx, P, n, source, out, reinterpret_cast<int2*>(pairs), "dist_dedup"));
    if (n_pairs) *n_pairs = 2 * (int64_t)out->E;
    return PHFEM_OK;
  }
  EgOwn own{self_elem_edge, 3 * (int64_t)self_lo, 3 * (int64_t)self_hi, nullptr};
  PHFEM_TRY(dalloc(ctx, &own.npairs, 1));
  PHFEM_CUDA(ctx, cudaMemsetAsync(own.npairs, 0, sizeof(int32_t), ctx->stream));
  phfem_status st = eg_core(ctx, P, n, source, out, reinterpret_cast<int2*>(pairs), "dist_dedup", nullptr, &own);
  int32_t np = 0;
  if (st == PHFEM_OK) {
    if (cudaMemcpyAsync(&np, own.npairs, sizeof np, cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess)
      st = cuda_fail(ctx, cudaGetLastError(), "dist_dedup: pair count");
  }
  dfree(ctx, own.npairs);
  *n_pairs = np;
  return st;
}

PHFEM_API phfem_status phfem_dist_dedup(phfem_ctx* ctx, const int32_t* recs, int64_t n,
                                        int32_t node_lo, int32_t node_hi, int32_t nC_all,
                                        int32_t nE_all, phfem_topology* out, int32_t* pairs) {
  return phfem_dist_dedup_ex(ctx, recs, n, node_lo, node_hi, nC_all, nE_all, 0, 0, nullptr, out, pairs, nullptr);
}

namespace phfem {
phfem_status classify_lists(phfem_ctx* ctx, const phfem_topology* topo, const phfem_mesh* mesh,
                            phfem_classification* out, bool with_retained);

// build_topology + classify_edges + assemble_constraint of a mesh in one
// edge-generation pass (pipeline_impl's final, sort-built level): the emit
// pass writes retained_pos / retained_edges and C's rows; classify_lists then
// resolves the boundary pairs (the reference's errors) and must agree on L.
phfem_status build_topology_fused(phfem_ctx* ctx, const phfem_mesh* mesh, phfem_topology* out,
                                  phfem_classification* cls, phfem_csr* C) {
  memset(out, 0, sizeof(*out));
  memset(cls, 0, sizeof(*cls));
  memset(C, 0, sizeof(*C));
  const int64_t nE = mesh->nE, nC = mesh->nC;
  if (nE < 0 || nC < 0 || 3 * nE >= (int64_t(1) << 31))
    return set_error(ctx, PHFEM_ERR_INVALID_ARGUMENT, "build_topology: mesh too large for int ids");
  out->nC = (int32_t)nC;
  out->nE = (int32_t)nE;
  int cap = 64;
  while (cap < 2 * mesh->nN) cap <<= 1;
  unsigned long long* keys = nullptr;
  PHFEM_TRY(dalloc(ctx, &keys, cap));
  PHFEM_CUDA(ctx, cudaMemsetAsync(keys, 0xff, sizeof(unsigned long long) * cap, ctx->stream));
  if (mesh->nN > 0)
    PHFEM_LAUNCH(ctx, "k_neu_pair_insert", k_neu_pair_insert<<<grid_for(mesh->nN, 256, ctx->num_sms), 256, 0,
                                                                ctx->stream>>>(mesh->neumann, mesh->nN, cap, keys));
  EgParams P;
  PHFEM_TRY(eg_params(ctx, nC, nC, nE, 0, &P));
  const int grid_e = grid_for(nE, 256, ctx->num_sms * 8);
  auto source = [&](int kind, int32_t* counts, uint64_t* items) -> phfem_status {
    if (kind == 0)
      PHFEM_LAUNCH(ctx, "k_eg_count", k_eg_count<<<grid_e, 256, 0, ctx->stream>>>(mesh->elements, P, counts, ctx->derr));
    else
      PHFEM_LAUNCH(ctx, "k_eg_scatter", k_eg_scatter<<<grid_e, 256, 0, ctx->stream>>>(mesh->elements, P, counts, items));
    return PHFEM_OK;
  };
  EgFuse fuse{keys, cap, mesh->coords, cls, C, (int32_t)nE};
  phfem_status st = eg_core(ctx, P, 3 * nE, source, out, nullptr, "build_topology", &fuse, nullptr, nullptr,
                            mesh->elements);
  dfree(ctx, keys);
  if (st != PHFEM_OK) return st;
  const int32_t L = cls->L;
  PHFEM_TRY(classify_lists(ctx, out, mesh, cls, false));
  if (cls->L != L)
    return set_error(ctx, PHFEM_ERR_MISMATCH, "build_topology: fused classification disagrees (%d vs %d)", L, cls->L);
  return PHFEM_OK;
}
}  // namespace phfem

// ---------------------------------------------------------------------------
// Distributed input level with peer windows (dist.py _edge_generation, P2P):
// key ranges aligned to 256-node tiles, so a bucket (2^bs max nodes) has one
// owner and the bucket index max >> bs is global.  Every rank histograms its
// own occurrences per global bucket (k_eg_count), the histograms are
// all-gathered, every rank derives its private cursor inside each bucket
// (owner-local bucket start + the lower ranks' counts), and ONE kernel packs
// each occurrence and stores it straight into its slot of the owner's item
// array (mapped peer window) — the MSD bucket scatter fused with the
// exchange.  The owner then runs the tile / emit passes on its items.
namespace phfem {
__global__ void k_dist_bucket_total(const int32_t* __restrict__ hist_all, int W, int64_t NB,
                                    int32_t* __restrict__ total) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < NB; b += (int64_t)gridDim.x * blockDim.x) {
    int32_t t = 0;
    for (int r = 0; r < W; ++r) t += hist_all[(int64_t)r * NB + b];
    total[b] = t;
  }
}

__device__ __forceinline__ int bucket_owner(const int32_t* __restrict__ bsplits, int W, int64_t b) {
  int lo = 0, hi = W;  // last r with bsplits[r] <= b
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(bsplits + mid) <= b) lo = mid;
    else hi = mid;
  }
  return lo;
}

__global__ void k_dist_bucket_cursor(const int32_t* __restrict__ hist_all, int W, int64_t NB, int me,
                                     const int32_t* __restrict__ gp, const int32_t* __restrict__ bsplits,
                                     int32_t* __restrict__ cursor, int32_t* __restrict__ boff_me) {
  const int64_t b0 = bsplits[me], b1 = bsplits[me + 1];
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b <= NB; b += (int64_t)gridDim.x * blockDim.x) {
    if (b < NB) {
      const int d = bucket_owner(bsplits, W, b);
      int32_t c = gp[b] - gp[bsplits[d]];
      for (int r = 0; r < me; ++r) c += hist_all[(int64_t)r * NB + b];
      cursor[b] = c;
    }
    if (b >= b0 && b <= b1) boff_me[b - b0] = gp[b] - gp[b0];
  }
}

__global__ void __launch_bounds__(256) k_dist_scatter_p2p(const int32_t* __restrict__ elements, int64_t n, int elo,
                                                          EgParams P, int32_t* __restrict__ cursor,
                                                          const int32_t* __restrict__ bsplits, int W, int me,
                                                          uint64_t* const* __restrict__ peer_items,
                                                          int32_t* __restrict__ remote) {
  __shared__ int32_t srem[64];  // per-block remote counts (one global atomic per block and rank)
  for (int i = threadIdx.x; i < 64; i += blockDim.x) srem[i] = 0;
  __syncthreads();
  const uint32_t hl_mask = (1u << P.bs) - 1u;
  for (int64_t m0 = (int64_t)blockIdx.x * blockDim.x; m0 < n; m0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = m0 + threadIdx.x;
    const bool valid = m < n;
    int t[3] = {0, 0, 0};
    if (valid) {
      t[0] = __ldg(elements + 3 * m);
      t[1] = __ldg(elements + 3 * m + 1);
      t[2] = __ldg(elements + 3 * m + 2);
    }
    // the three claims in flight together (as in k_eg_scatter_fixed)
    unsigned keys[3], grps[3];
    int bases[3];
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const int a = t[s], b = t[(s + 1) % 3];
      keys[s] = valid ? ((unsigned)(a > b ? a : b) >> P.bs) : 0xffffffffu;
      grps[s] = __match_any_sync(0xffffffffu, keys[s]);
    }
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      bases[s] = 0;
      if (valid && (int)lane_id() == __ffs(grps[s]) - 1) bases[s] = atomicAdd(&cursor[keys[s]], __popc(grps[s]));
    }
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const int a = t[s], b = t[(s + 1) % 3];
      const int hi = a > b ? a : b;
      const int lo = a > b ? b : a;
      const unsigned key = keys[s], grp = grps[s];
      const int leader = __ffs(grp) - 1;
      const int base = __shfl_sync(0xffffffffu, bases[s], leader);
      if (valid) {
        const int d = bucket_owner(bsplits, W, key);
        const uint32_t occ = (uint32_t)(3 * ((int64_t)elo + m) + s);
        peer_items[d][base + __popc(grp & lanemask_lt())] =
            eg_pack(P, (uint32_t)hi & hl_mask, (uint32_t)lo, occ, a > b ? 1u : 0u);
        if (d != me && (int)lane_id() == leader) atomicAdd(srem + (d & 63), __popc(grp));
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < W && i < 64; i += blockDim.x)
    if (srem[i]) atomicAdd(remote + i, srem[i]);
}
}  // namespace phfem

PHFEM_API int phfem_dist_bucket_bits(int32_t nC_all, int32_t nE_all) {
  const int tb = bits_for(std::max<int64_t>((int64_t)nC_all - 1, 1)) + bits_for(std::max<int64_t>(3 * (int64_t)nE_all - 1, 1)) + 1;
  return std::min(8, 64 - tb);
}

PHFEM_API phfem_status phfem_dist_bucket_hist(phfem_ctx* ctx, const int32_t* elements, int32_t n, int32_t elo,
                                              int32_t nC_all, int32_t nE_all, int32_t* hist) {
  if (!ctx || !hist || n < 0 || (n && !elements)) return PHFEM_ERR_INVALID_ARGUMENT;
  EgParams P;
  PHFEM_TRY(eg_params(ctx, nC_all, nC_all, nE_all, 0, &P));
  P.nE = n;
  PHFEM_CUDA(ctx, cudaMemsetAsync(hist, 0, sizeof(int32_t) * P.nb, ctx->stream));
  PHFEM_TRY(errors_reset(ctx));
  if (n > 0)
    PHFEM_LAUNCH(ctx, "k_eg_count", k_eg_count<<<grid_for(n, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
        elements, P, hist, ctx->derr));
  PHFEM_TRY(errors_fetch(ctx));
  if (ctx->herr->misc != ~0ull)
    return set_error(ctx, PHFEM_ERR_OUT_OF_RANGE, "build_topology: element %lld has a node index outside 1..%lld",
                     (long long)ctx->herr->misc + elo + 1, (long long)nC_all);
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_dist_bucket_cursors(phfem_ctx* ctx, const int32_t* hist_all, int32_t W, int64_t NB,
                                                 int32_t me, const int32_t* bsplits, int32_t* cursor,
                                                 int32_t* boff_me, int64_t* n_items_me) {
  if (!ctx || !hist_all || !bsplits || !cursor || !boff_me || !n_items_me || W < 1 || me < 0 || me >= W || NB < 1)
    return PHFEM_ERR_INVALID_ARGUMENT;
  int32_t* gp = nullptr;
  PHFEM_TRY(dalloc(ctx, &gp, NB + 1));
  PHFEM_CUDA(ctx, cudaMemsetAsync(gp + NB, 0, sizeof(int32_t), ctx->stream));
  PHFEM_LAUNCH(ctx, "k_dist_bucket_total", k_dist_bucket_total<<<grid_for(NB, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
      hist_all, W, NB, gp));
  PHFEM_TRY(scan_exclusive_i32(ctx, gp, gp, NB + 1, nullptr));
  PHFEM_LAUNCH(ctx, "k_dist_bucket_cursor", k_dist_bucket_cursor<<<grid_for(NB + 1, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
      hist_all, W, NB, me, gp, bsplits, cursor, boff_me));
  int32_t h[2];
  int32_t b01[2];
  PHFEM_CUDA(ctx, cudaMemcpyAsync(b01, bsplits + me, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
  PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  PHFEM_CUDA(ctx, cudaMemcpyAsync(&h[0], gp + b01[0], sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
  PHFEM_CUDA(ctx, cudaMemcpyAsync(&h[1], gp + b01[1], sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
  PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  *n_items_me = (int64_t)h[1] - h[0];
  dfree(ctx, gp);
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_dist_scatter_p2p(phfem_ctx* ctx, const int32_t* elements, int32_t n, int32_t elo,
                                              int32_t nC_all, int32_t nE_all, int32_t* cursor, const int32_t* bsplits,
                                              int32_t W, int32_t me, uint64_t* const* peer_items, int32_t* remote) {
  if (!ctx || !cursor || !bsplits || !peer_items || !remote || W < 1 || W > 64 || me < 0 || me >= W || n < 0 ||
      (n && !elements))
    return PHFEM_ERR_INVALID_ARGUMENT;
  EgParams P;
  PHFEM_TRY(eg_params(ctx, nC_all, nC_all, nE_all, 0, &P));
  PHFEM_CUDA(ctx, cudaMemsetAsync(remote, 0, sizeof(int32_t) * W, ctx->stream));
  if (n > 0)
    PHFEM_LAUNCH(ctx, "k_dist_scatter_p2p", k_dist_scatter_p2p<<<grid_for(n, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
        elements, n, elo, P, cursor, bsplits, W, me, peer_items, remote));
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_dist_dedup_items(phfem_ctx* ctx, uint64_t* items, int64_t n, const int32_t* boff,
                                              int32_t node_lo, int32_t node_hi, int32_t nC_all, int32_t nE_all,
                                              int32_t self_lo, int32_t self_hi, int32_t* self_elem_edge,
                                              phfem_topology* out, int32_t* pairs, int64_t* n_pairs) {
  memset(out, 0, sizeof(*out));
  if (!ctx || (!items && n) || !boff || !pairs || !self_elem_edge || !n_pairs || node_lo < 0 || node_hi < node_lo ||
      node_hi > nC_all || self_lo < 0 || self_hi < self_lo || self_hi > nE_all ||
      3 * (int64_t)nE_all >= (int64_t(1) << 31))
    return PHFEM_ERR_INVALID_ARGUMENT;
  *n_pairs = 0;
  out->nC = node_hi - node_lo;
  out->nE = nE_all;
  EgParams P;
  PHFEM_TRY(eg_params(ctx, (int64_t)node_hi - node_lo, nC_all, nE_all, node_lo, &P));
  auto none = [&](int, int32_t*, uint64_t*) -> phfem_status { return PHFEM_OK; };
  EgOwn own{self_elem_edge, 3 * (int64_t)self_lo, 3 * (int64_t)self_hi, nullptr};
  EgPre pre{boff, items};
  PHFEM_TRY(dalloc(ctx, &own.npairs, 1));
  PHFEM_CUDA(ctx, cudaMemsetAsync(own.npairs, 0, sizeof(int32_t), ctx->stream));
  phfem_status st = eg_core(ctx, P, n, none, out, reinterpret_cast<int2*>(pairs), "dist_dedup", nullptr, &own, &pre);
  int32_t np = 0;
  if (st == PHFEM_OK) {
    if (cudaMemcpyAsync(&np, own.npairs, sizeof np, cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess)
      st = cuda_fail(ctx, cudaGetLastError(), "dist_dedup: pair count");
  }
  dfree(ctx, own.npairs);
  *n_pairs = np;
  return st;
}
