// dist.cu — device side of the multi-GPU pipeline (host side in
// paper_2401_15557_b200/dist.py).  Elements are partitioned by contiguous
// ranges, nodes (and so edges, which are grouped by max node) by contiguous
// key ranges.  Per-element work needs no communication; the edge dedup is one
// key-range all-to-all of directed occurrences, a local sort (the single-GPU
// tile machinery of edge_gen.cu, phfem_dist_dedup) and a reverse all-to-all
// of (element slot, edge id) pairs.  The kernels here produce and consume the
// exchange buffers and re-base rank-local ids to global ones, so the
// concatenation of the ranks' outputs is bit-identical to the single-GPU run.
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"

// grid of the peer-window exchange kernels (CTAs per SM)
#ifndef PHFEM_P2P_GRID_MULT
#define PHFEM_P2P_GRID_MULT 8
#endif

namespace phfem {

__device__ __forceinline__ int dest_of(const int32_t* __restrict__ splits, int W, int v) {
  int lo = 0, hi = W;  // last r with splits[r] <= v
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(splits + mid) <= v) lo = mid;
    else hi = mid;
  }
  return lo;
}

// Routing by destination with block-level aggregation: every thread owns
// kRouteK items; destinations are counted in SMEM (W <= kMaxDest), one
// global atomic per (block, destination) reserves the block's ranges, items
// go to base[d] + SMEM rank.  (A per-warp global atomic serialised on one
// counter at W = 1-8 and dominated the step.)  Order inside a destination is
// irrelevant: the receiver sorts.
constexpr int kRouteThreads = 256;
constexpr int kRouteK = 8;
constexpr int kMaxDest = 4097;  // also the coarse histogram's bins

template <typename Item, typename Fn>
__device__ __forceinline__ void route_block(int64_t n, int W, Fn item_of, int32_t* __restrict__ cnt,
                                            int32_t* __restrict__ cursor, Item* __restrict__ send) {
  __shared__ int32_t s_cnt[kMaxDest];
  __shared__ int32_t s_base[kMaxDest];
  const int64_t chunk = (int64_t)kRouteThreads * kRouteK;
  for (int64_t c0 = (int64_t)blockIdx.x * chunk; c0 < n; c0 += (int64_t)gridDim.x * chunk) {
    for (int d = threadIdx.x; d < W; d += blockDim.x) s_cnt[d] = 0;
    __syncthreads();
    Item it[kRouteK];
    int dst[kRouteK], rk[kRouteK];
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < kRouteK; ++k) {
      const int64_t i = c0 + (int64_t)k * kRouteThreads + threadIdx.x;
      dst[k] = -1;
      if (i < n) dst[k] = item_of(i, it[k]);
      // warp-aggregated: one SMEM atomic per (warp, destination) — with few
      // destinations every lane would otherwise hit the same counter
      const unsigned peers = __match_any_sync(0xffffffffu, dst[k]);
      const int leader = __ffs(peers) - 1;
      int base = 0;
      if (lane == leader && dst[k] >= 0) base = atomicAdd(&s_cnt[dst[k]], __popc(peers));
      base = __shfl_sync(0xffffffffu, base, leader);
      rk[k] = base + __popc(peers & ((1u << lane) - 1u));
    }
    __syncthreads();
    for (int d = threadIdx.x; d < W; d += blockDim.x) {
      const int c = s_cnt[d];
      if (c) {
        if (send) s_base[d] = atomicAdd(&cursor[d], c);
        else atomicAdd(&cnt[d], c);
      }
    }
    if (send) {
      __syncthreads();
#pragma unroll
      for (int k = 0; k < kRouteK; ++k)
        if (dst[k] >= 0) send[s_base[dst[k]] + rk[k]] = it[k];
    }
    __syncthreads();
  }
}

// directed occurrences of elements [elo, ehi) (elements: the rank's local
// array): slot s of element m is v_s -> v_{s+1} (edge_topology.cpp:61-68);
// record {max, min, 3m+s, dir}, routed to the owner of the max node
__global__ void __launch_bounds__(kRouteThreads) k_dist_occ(const int32_t* __restrict__ elements, int elo, int ehi,
                           const int32_t* __restrict__ splits, int W, int32_t* __restrict__ cnt,
                           int32_t* __restrict__ cursor, int4* __restrict__ send) {
  const int64_t n = 3 * (int64_t)(ehi - elo);
  route_block<int4>(n, W, [&](int64_t i, int4& r) {
    const int64_t ml = i / 3;
    const int s = (int)(i - 3 * ml);
    const int a = elements[3 * ml + s], b = elements[3 * ml + (s == 2 ? 0 : s + 1)];
    r = make_int4(max(a, b), min(a, b), (int)(3 * (elo + ml) + s), a > b ? 1 : 0);
    return dest_of(splits, W, r.x);
  }, cnt, cursor, send);
}

// pairs (slot 3m+l, local edge or ~local edge) -> global edge ids, routed to
// the element owner; slot < 0 marks "no t_minus".  Pairs of the own element
// range [3 lo, 3 hi) (self_lo < self_hi) are applied to self_ee directly (no
// send, no exchange).
__global__ void __launch_bounds__(kRouteThreads) k_dist_pairs(const int2* __restrict__ pairs, int64_t n, int E0,
                             const int32_t* __restrict__ esplits, int W, int32_t* __restrict__ cnt,
                             int32_t* __restrict__ cursor, int2* __restrict__ send, int self_lo,
                             int self_hi, int32_t* __restrict__ self_ee) {
  route_block<int2>(n, W, [&](int64_t i, int2& q) {
    const int2 p = pairs[i];
    if (p.x < 0) return -1;
    q = make_int2(p.x, p.y >= 0 ? p.y + E0 : ~(~p.y + E0));
    const int m = p.x / 3;
    if (m >= self_lo && m < self_hi) {
      if (send) self_ee[p.x - 3 * (int64_t)self_lo] = q.y;  // (once: in the scatter pass)
      return -1;
    }
    return dest_of(esplits, W, m);
  }, cnt, cursor, send);
}

__global__ void k_dist_apply(const int2* __restrict__ recv, int64_t n, int elo,
                             int32_t* __restrict__ elem_edge) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int2 p = recv[i];
    elem_edge[p.x - 3 * (int64_t)elo] = p.y;
  }
}

__global__ void k_add_offset(int32_t* __restrict__ a, int64_t n, int32_t off, int only_nonneg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = a[i];
    if (only_nonneg == 2) a[i] = v >= 0 ? v + off : v - off;  // signed ids e / ~e
    else if (!only_nonneg || v >= 0) a[i] = v + off;
  }
}

// boundary pairs whose max node lies in [nlo, nhi): global id, or the
// reference's errors (edge_topology.cpp:151-157) keyed by list position
__global__ void k_dist_resolve(const int32_t* __restrict__ pairs, int n, int list,
                               const int32_t* __restrict__ nes, const int32_t* __restrict__ edge_nodes,
                               const int32_t* __restrict__ edge_elements, int nlo, int nhi, int E0,
                               int32_t* __restrict__ ids, unsigned long long* __restrict__ err) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int a = pairs[2 * i], b = pairs[2 * i + 1];
    const int hi = max(a, b), lo = min(a, b);
    ids[i] = -1;
    if (hi < nlo || hi >= nhi) continue;
    int e = -1;
    if (lo >= 0) {
      // edges of max node hi (ascending min); nes holds global ids (re-based)
      const int end = nes[hi - nlo + 1] - E0;
      int l = nes[hi - nlo] - E0, r = end;
      while (l < r) {
        const int mid = (l + r) >> 1;
        const int x = edge_nodes[2 * mid], y = edge_nodes[2 * mid + 1];
        if (min(x, y) < lo) l = mid + 1;
        else r = mid;
      }
      if (l < end && min(edge_nodes[2 * l], edge_nodes[2 * l + 1]) == lo) e = l;
    }
    // error key: (global list position << 2) | code (0 not an edge, 1 interior)
    const unsigned long long pos = (unsigned long long)(list + i);
    if (e < 0) atomicMin(err, pos << 2);
    else if (edge_elements[2 * e + 1] >= 0) atomicMin(err, (pos << 2) | 1ull);
    else ids[i] = E0 + e;
  }
}

// Neumann flags of the local edges from the global Neumann id list
__global__ void k_dist_neu_bits(const int32_t* __restrict__ neu_ids, int nN, int E0, int E,
                                uint32_t* __restrict__ bits, unsigned long long* __restrict__ dup) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nN; i += gridDim.x * blockDim.x) {
    const int e = neu_ids[i] - E0;
    if (e < 0 || e >= E) continue;
    const uint32_t bit = 1u << (e & 31);
    if ((atomicOr(&bits[e >> 5], bit) & bit) && dup) *dup = 1;
  }
}

// local ids of the listed edges in [E0, E0 + E), list order kept
__global__ void k_dist_local_ids(const int32_t* __restrict__ ids, int n, int E0, int E,
                                 int32_t* __restrict__ flag) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int e = ids[i] - E0;
    flag[i] = (e >= 0 && e < E) ? 1 : 0;
  }
}
__global__ void k_dist_compact(const int32_t* __restrict__ ids, const int32_t* __restrict__ pos,
                               int n, int E0, int E, int32_t* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int e = ids[i] - E0;
    if (e >= 0 && e < E) out[pos[i]] = e;
  }
}

// Neumann edge table rows {a, b, t_plus, led} for the local Neumann edges
__global__ void k_dist_neu_table(const int32_t* __restrict__ neu_ids, int nN, int E0, int E,
                                 const int32_t* __restrict__ edge_nodes,
                                 const int32_t* __restrict__ edge_elements,
                                 const int32_t* __restrict__ ltp, int32_t* __restrict__ table) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nN; i += gridDim.x * blockDim.x) {
    const int e = neu_ids[i] - E0;
    if (e < 0 || e >= E) continue;
    table[4 * i] = edge_nodes[2 * e];
    table[4 * i + 1] = edge_nodes[2 * e + 1];
    table[4 * i + 2] = edge_elements[2 * e];
    table[4 * i + 3] = ltp[e];
  }
}

// mini topology of the Neumann edges whose t_plus element is local: edge i
// of the table keeps id i; the Neumann list is the owned positions in order
__global__ void k_dist_neu_mini(const int32_t* __restrict__ table, int nN, int elo, int ehi,
                                int32_t* __restrict__ en, int32_t* __restrict__ el,
                                int32_t* __restrict__ ltp, int32_t* __restrict__ flag) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nN; i += gridDim.x * blockDim.x) {
    en[2 * i] = table[4 * i];
    en[2 * i + 1] = table[4 * i + 1];
    el[2 * i] = table[4 * i + 2] - elo;  // local element: the load array is local
    el[2 * i + 1] = -1;
    ltp[i] = table[4 * i + 3];
    flag[i] = (table[4 * i + 2] >= elo && table[4 * i + 2] < ehi) ? 1 : 0;
  }
}
__global__ void k_dist_iota_compact(const int32_t* __restrict__ flag, const int32_t* __restrict__ pos,
                                    int n, int32_t* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (flag[i]) out[pos[i]] = i;
}

// midpoints 0.5 (c[a] + c[b]) of a range of edges (refine.cpp:16-19)
__global__ void k_dist_midpoints(const double2* __restrict__ coords, const int32_t* __restrict__ edge_nodes,
                                 int E, double2* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double2 pa = coords[edge_nodes[2 * e]], pb = coords[edge_nodes[2 * e + 1]];
    out[e] = make_double2(0.5 * (pa.x + pb.x), 0.5 * (pa.y + pb.y));
  }
}

// children 4m..4m+3 of the local elements (refine.cpp:28-37)
__global__ void __launch_bounds__(256) k_dist_children(const int32_t* __restrict__ elements,
                                                       const int32_t* __restrict__ elem_edge, int n, int nc,
                                                       int4* __restrict__ out) {
  // rows staged per warp, stored as contiguous 512-byte warp writes (as k_refine_children)
  __shared__ int4 stage[8][96];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int4* so = stage[warp];
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + warp * 32; base < n;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = base + lane;
    if (m < n) {
      const int p0 = elements[3 * m], p1 = elements[3 * m + 1], p2 = elements[3 * m + 2];
      const int s0 = elem_edge[3 * m], s1 = elem_edge[3 * m + 1], s2 = elem_edge[3 * m + 2];
      const int m0 = nc + (s0 >= 0 ? s0 : ~s0), m1 = nc + (s1 >= 0 ? s1 : ~s1), m2 = nc + (s2 >= 0 ? s2 : ~s2);
      so[3 * lane] = make_int4(m0, m1, m2, p0);
      so[3 * lane + 1] = make_int4(m2, m1, p1, m0);
      so[3 * lane + 2] = make_int4(m2, p2, m1, m0);
    }
    __syncwarp();
    const int64_t rem = n - base;
    const int n4 = 3 * (int)(rem < 32 ? rem : 32);
    for (int i = lane; i < n4; i += 32) out[3 * base + i] = so[i];
    __syncwarp();
  }
}

// Side records of the sort-free distributed refinement: slot k of element m
// (local index i = 3 m_local + k) -> {e << 1 | (m is t_minus of e), the
// partner edges at local k+1 and k+2 (signed), vertex k}, routed to the
// owner of parent edge e (esplits: first global edge id per rank)
__global__ void __launch_bounds__(kRouteThreads) k_dist_side(const int32_t* __restrict__ elements,
                                                             const int32_t* __restrict__ elem_edge, int n,
                                                             const int32_t* __restrict__ esplits, int W,
                                                             int32_t* __restrict__ cnt, int32_t* __restrict__ cursor,
                                                             int4* __restrict__ send) {
  route_block<int4>(3 * (int64_t)n, W, [&](int64_t i, int4& r) {
    const int64_t m = i / 3;
    const int k = (int)(i - 3 * m);
    const int s = elem_edge[i];
    const int e = s >= 0 ? s : ~s;
    r = make_int4(e << 1 | (s < 0 ? 1 : 0), elem_edge[3 * m + (k == 2 ? 0 : k + 1)],
                  elem_edge[3 * m + (k == 0 ? 2 : k - 1)], elements[i]);
    return dest_of(esplits, W, e);
  }, cnt, cursor, send);
}

__global__ void k_dist_side_apply(const int4* __restrict__ recv, int64_t n, int E0, int E, int4* __restrict__ side) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int4 r = recv[i];
    const int le = (r.x >> 1) - E0;
    if (le >= 0 && le < E) side[2 * (int64_t)le + (r.x & 1)] = make_int4(r.y, r.z, r.w, 0);
  }
}

// Group-start records: for every owned parent edge and each of its elements,
// {slot 3 m + local, first fine id of the edge's group (global), rank byte}
// routed to the owner of m (psplits: first parent element per rank)
struct Rec3 {
  int x, y, z;
};
__global__ void __launch_bounds__(kRouteThreads) k_dist_start(const int32_t* __restrict__ edge_elements,
                                                              const int32_t* __restrict__ ltp,
                                                              const int32_t* __restrict__ ltm,
                                                              const int32_t* __restrict__ fine_nes, int nes_off,
                                                              const uint8_t* __restrict__ rk, int E,
                                                              const int32_t* __restrict__ psplits, int W,
                                                              int32_t* __restrict__ cnt, int32_t* __restrict__ cursor,
                                                              Rec3* __restrict__ send) {
  route_block<Rec3>(2 * (int64_t)E, W, [&](int64_t i, Rec3& r) {
    const int64_t le = i >> 1;
    const int sd = (int)(i & 1);
    const int m = edge_elements[2 * le + sd];
    if (m < 0) return -1;
    const int l = sd ? ltm[le] : ltp[le];
    r.x = 3 * m + l;
    r.y = fine_nes[le + nes_off];
    r.z = rk[le];
    return dest_of(psplits, W, m);
  }, cnt, cursor, send);
}

__global__ void k_dist_start_apply(const Rec3* __restrict__ recv, int64_t n, int elo, int32_t* __restrict__ gs,
                                   uint8_t* __restrict__ grk) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const Rec3 r = recv[i];
    const int64_t slot = (int64_t)r.x - 3 * (int64_t)elo;
    gs[slot] = r.y;
    grk[slot] = (uint8_t)r.z;
  }
}

// ---- peer-window forms (fused compute + exchange over NVLink peer memory) --
// The owner's receive array is mapped into every rank (CUDA IPC; on one GPU
// the emulated ranks' arrays): the producing kernel stores each record
// straight into its final slot there — no count pass, no send buffer, no
// all-to-all, no apply pass.  remote[d] counts the records stored into rank
// d's window by this rank (d != self), for the byte accounting.
// (per-block SMEM counters, flushed once per block: one global counter per
// destination hit by every warp serialised the kernels at L2 — 0.3-0.5 ms)
constexpr int kRemoteMax = 64;
__device__ __forceinline__ void count_remote(int d, int self, int32_t* srem) {
  const unsigned peers = __match_any_sync(__activemask(), d);
  if (d != self && lane_id() == (unsigned)(__ffs(peers) - 1)) atomicAdd(srem + (d & (kRemoteMax - 1)), __popc(peers));
}
__device__ __forceinline__ void remote_init(int32_t* srem) {
  for (int i = threadIdx.x; i < kRemoteMax; i += blockDim.x) srem[i] = 0;
  __syncthreads();
}
__device__ __forceinline__ void remote_flush(const int32_t* srem, int W, int32_t* remote) {
  __syncthreads();
  for (int i = threadIdx.x; i < W && i < kRemoteMax; i += blockDim.x)
    if (srem[i]) atomicAdd(remote + i, srem[i]);
}

__global__ void __launch_bounds__(256) k_dist_side_p2p(const int32_t* __restrict__ elements,
                                                       const int32_t* __restrict__ elem_edge, int n,
                                                       const int32_t* __restrict__ esplits, int W, int self,
                                                       int4* const* __restrict__ peer_side, int32_t* remote,
                                                       int skip_self) {
  __shared__ int32_t srem[kRemoteMax];
  remote_init(srem);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 3 * (int64_t)n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / 3;
    const int k = (int)(i - 3 * m);
    const int s = elem_edge[i];
    const int e = s >= 0 ? s : ~s;
    const int d = dest_of(esplits, W, e);
    if (skip_self && d == self) continue;  // local mode: the level kernel gathers it
    const int4 r = make_int4(elem_edge[3 * m + (k == 2 ? 0 : k + 1)], elem_edge[3 * m + (k == 0 ? 2 : k - 1)],
                             elements[i], 0);
    peer_side[d][2 * (int64_t)(e - __ldg(esplits + d)) + (s < 0 ? 1 : 0)] = r;
    count_remote(d, self, srem);
  }
  remote_flush(srem, W, remote);
}

__global__ void __launch_bounds__(256) k_dist_start_p2p(const int32_t* __restrict__ edge_elements,
                                                        const int32_t* __restrict__ ltp,
                                                        const int32_t* __restrict__ ltm,
                                                        const int32_t* __restrict__ fine_nes, int nes_off,
                                                        const uint8_t* __restrict__ rk, int E,
                                                        const int32_t* __restrict__ psplits, int W, int self,
                                                        int32_t* const* __restrict__ peer_gs,
                                                        uint8_t* const* __restrict__ peer_grk, int32_t* remote,
                                                        int skip_self) {
  __shared__ int32_t srem[kRemoteMax];
  remote_init(srem);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 2 * (int64_t)E;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t le = i >> 1;
    const int sd = (int)(i & 1);
    const int m = edge_elements[2 * le + sd];
    int d = -1;
    if (m >= 0) {
      const int l = sd ? ltm[le] : ltp[le];
      d = dest_of(psplits, W, m);
      if (skip_self && d == self) continue;  // local mode: the children pass gathers it
      const int64_t slot = 3 * (int64_t)(m - __ldg(psplits + d)) + l;
      peer_gs[d][slot] = fine_nes[le + nes_off];
      peer_grk[d][slot] = rk[le];
    }
    if (d >= 0) count_remote(d, self, srem);
  }
  remote_flush(srem, W, remote);
}

// reverse pairs of the input level through peer windows: (slot 3m+l, local
// edge or ~edge) of another rank's element -> global id stored straight into
// that element owner's elem_edge (esplits: first element per rank)
__global__ void __launch_bounds__(256) k_dist_pairs_p2p(const int2* __restrict__ pairs, int64_t n, int E0,
                                                        const int32_t* __restrict__ esplits, int W, int self,
                                                        int32_t* const* __restrict__ peer_ee, int32_t* remote) {
  __shared__ int32_t srem[kRemoteMax];
  remote_init(srem);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int2 p = pairs[i];
    int d = -1;
    if (p.x >= 0) {
      const int m = p.x / 3;
      d = dest_of(esplits, W, m);
      peer_ee[d][p.x - 3 * (int64_t)__ldg(esplits + d)] = p.y >= 0 ? p.y + E0 : ~(~p.y + E0);
    }
    if (d >= 0) count_remote(d, self, srem);
  }
  remote_flush(srem, W, remote);
}

// count pass, exclusive offsets, pack pass of a route_block kernel
template <typename Launch>
static phfem_status route_two_pass(phfem_ctx* ctx, int W, int32_t* counts, int32_t* offsets, bool pack,
                                   Launch launch) {
  PHFEM_CUDA(ctx, cudaMemsetAsync(counts, 0, sizeof(int32_t) * W, ctx->stream));
  if (W >= kMaxDest) return PHFEM_ERR_INVALID_ARGUMENT;
  PHFEM_TRY(launch(counts, (int32_t*)nullptr));
  if (!pack) return PHFEM_OK;
  if (!offsets) return PHFEM_ERR_INVALID_ARGUMENT;
  int32_t* cursor = nullptr;
  PHFEM_TRY(dalloc(ctx, &cursor, (int64_t)W + 1));
  PHFEM_CUDA(ctx, cudaMemcpyAsync(cursor, counts, sizeof(int32_t) * W, cudaMemcpyDeviceToDevice, ctx->stream));
  PHFEM_CUDA(ctx, cudaMemsetAsync(cursor + W, 0, sizeof(int32_t), ctx->stream));
  PHFEM_TRY(scan_exclusive_i32(ctx, cursor, cursor, (int64_t)W + 1, nullptr));
  PHFEM_CUDA(ctx, cudaMemcpyAsync(offsets, cursor, sizeof(int32_t) * (W + 1), cudaMemcpyDeviceToDevice, ctx->stream));
  PHFEM_TRY(launch((int32_t*)nullptr, cursor));
  dfree(ctx, cursor);
  return PHFEM_OK;
}

}  // namespace phfem

using namespace phfem;

PHFEM_API phfem_status phfem_dist_midpoints(phfem_ctx* ctx, const double* coords,
                                            const int32_t* edge_nodes, int32_t E, double* out) {
  if (!ctx || (E && (!coords || !edge_nodes || !out))) return PHFEM_ERR_INVALID_ARGUMENT;
  if (E > 0)
    PHFEM_LAUNCH(ctx, "k_dist_midpoints", k_dist_midpoints<<<grid_for(E, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
        (const double2*)coords, edge_nodes, E, (double2*)out));
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_dist_children(phfem_ctx* ctx, const int32_t* elements,
                                           const int32_t* elem_edge, int32_t n, int32_t nC,
                                           int32_t* children) {
  if (!ctx || (n && (!elements || !elem_edge || !children))) return PHFEM_ERR_INVALID_ARGUMENT;
  if (n > 0)
    PHFEM_LAUNCH(ctx, "k_dist_children", k_dist_children<<<grid_for(n, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
        elements, elem_edge, n, nC, reinterpret_cast<int4*>(children)));
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_dist_occurrences(phfem_ctx* ctx, const int32_t* elements, int32_t elo,
                                              int32_t ehi, const int32_t* splits, int32_t W,
                                              int32_t* counts, int32_t* offsets, int32_t* send) {
  if (!ctx || !splits || !counts || W < 1 || elo < 0 || ehi < elo || (ehi > elo && !elements))
    return PHFEM_ERR_INVALID_ARGUMENT;
  PHFEM_CUDA(ctx, cudaMemsetAsync(counts, 0, sizeof(int32_t) * W, ctx->stream));
  const int64_t n = 3 * (int64_t)(ehi - elo);
  if (W >= kMaxDest) return PHFEM_ERR_INVALID_ARGUMENT;
  const int grid = grid_for(n, kRouteThreads * kRouteK, ctx->num_sms * 8);
  if (n > 0)
    PHFEM_LAUNCH(ctx, "k_dist_occ", k_dist_occ<<<grid, kRouteThreads, 0, ctx->stream>>>(
        elements, elo, ehi, splits, W, counts, nullptr, nullptr));
  if (!send) return PHFEM_OK;
  if (!offsets) return PHFEM_ERR_INVALID_ARGUMENT;
  int32_t* cursor = nullptr;
  PHFEM_TRY(dalloc(ctx, &cursor, (int64_t)W + 1));
  PHFEM_CUDA(ctx, cudaMemcpyAsync(cursor, counts, sizeof(int32_t) * W, cudaMemcpyDeviceToDevice, ctx->stream));
  PHFEM_CUDA(ctx, cudaMemsetAsync(cursor + W, 0, sizeof(int32_t), ctx->stream));
  PHFEM_TRY(scan_exclusive_i32(ctx, cursor, cursor, (int64_t)W + 1, nullptr));
  PHFEM_CUDA(ctx, cudaMemcpyAsync(offsets, cursor, sizeof(int32_t) * (W + 1), cudaMemcpyDeviceToDevice, ctx->stream));
  if (n > 0)
    PHFEM_LAUNCH(ctx, "k_dist_occ", k_dist_occ<<<grid, kRouteThreads, 0, ctx->stream>>>(
        elements, elo, ehi, splits, W, nullptr, cursor, reinterpret_cast<int4*>(send)));
  dfree(ctx, cursor);
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_dist_route_pairs(phfem_ctx* ctx, const int32_t* pairs, int64_t n,
                                              int32_t E0, const int32_t* esplits, int32_t W,
                                              int32_t* counts, int32_t* offsets, int32_t* send,
                                              int32_t self_lo, int32_t self_hi, int32_t* self_elem_edge) {
  if (!ctx || (!pairs && n) || !esplits || !counts || W < 1) return PHFEM_ERR_INVALID_ARGUMENT;
  if (self_lo < self_hi && !self_elem_edge) return PHFEM_ERR_INVALID_ARGUMENT;
  PHFEM_CUDA(ctx, cudaMemsetAsync(counts, 0, sizeof(int32_t) * W, ctx->stream));
  if (W >= kMaxDest) return PHFEM_ERR_INVALID_ARGUMENT;
  const int grid = grid_for(n, kRouteThreads * kRouteK, ctx->num_sms * 8);
  const int2* p2 = reinterpret_cast<const int2*>(pairs);
  if (n > 0)
    PHFEM_LAUNCH(ctx, "k_dist_pairs", k_dist_pairs<<<grid, kRouteThreads, 0, ctx->stream>>>(
        p2, n, E0, esplits, W, counts, nullptr, nullptr, self_lo, self_hi, self_elem_edge));
  if (!send) return PHFEM_OK;
  if (!offsets) return PHFEM_ERR_INVALID_ARGUMENT;
  int32_t* cursor = nullptr;
  PHFEM_TRY(dalloc(ctx, &cursor, (int64_t)W + 1));
  PHFEM_CUDA(ctx, cudaMemcpyAsync(cursor, counts, sizeof(int32_t) * W, cudaMemcpyDeviceToDevice, ctx->stream));
  PHFEM_CUDA(ctx, cudaMemsetAsync(cursor + W, 0, sizeof(int32_t), ctx->stream));
  PHFEM_TRY(scan_exclusive_i32(ctx, cursor, cursor, (int64_t)W + 1, nullptr));
  PHFEM_CUDA(ctx, cudaMemcpyAsync(offsets, cursor, sizeof(int32_t) * (W + 1), cudaMemcpyDeviceToDevice, ctx->stream));
  if (n > 0)
    PHFEM_LAUNCH(ctx, "k_dist_pairs", k_dist_pairs<<<grid, kRouteThreads, 0, ctx->stream>>>(
        p2, n, E0, esplits, W, nullptr, cursor, reinterpret_cast<int2*>(send), self_lo, self_hi,
        self_elem_edge));
  dfree(ctx, cursor);
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_dist_apply_pairs(phfem_ctx* ctx, const int32_t* recv, int64_t n,
                                              int32_t elo, int32_t* elem_edge) {
  if (!ctx || (n && (!recv || !elem_edge))) return PHFEM_ERR_INVALID_ARGUMENT;
  if (n > 0)
    PHFEM_LAUNCH(ctx, "k_dist_apply", k_dist_apply<<<grid_for(n, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
        reinterpret_cast<const int2*>(recv), n, elo, elem_edge));
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_dist_add_offset(phfem_ctx* ctx, int32_t* a, int64_t n, int32_t off,
                                             int only_nonneg) {
  if (!ctx || (n && !a)) return PHFEM_ERR_INVALID_ARGUMENT;
  if (n > 0 && off != 0)
    PHFEM_LAUNCH(ctx, "k_add_offset", k_add_offset<<<grid_for(n, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
        a, n, off, only_nonneg));
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_dist_resolve(phfem_ctx* ctx, const phfem_topology* part,
                                          int32_t node_lo, int32_t E0, const int32_t* pairs,
                                          int32_t n, int32_t list_base, int32_t* ids,
                                          unsigned long long* err) {
  if (!ctx || !part || (n && (!pairs || !ids || !err))) return PHFEM_ERR_INVALID_ARGUMENT;
  if (n > 0)
    PHFEM_LAUNCH(ctx, "k_dist_resolve", k_dist_resolve<<<grid_for(n, 256, ctx->num_sms * 4), 256, 0, ctx->stream>>>(
        pairs, n, list_base, part->node_edge_start, part->edge_nodes, part->edge_elements, node_lo,
        node_lo + part->nC, E0, ids, err));
  return PHFEM_OK;
}

namespace phfem {
phfem_status classify_lists_from_bits(phfem_ctx* ctx, const phfem_topology* topo, phfem_classification* out,
                                      int bnd_base, int r_off, int e_off);
}

// dir_ids / neu_ids: the rank's edges, LOCAL ids; E0 = global id of the
// part's first edge (its boundary list holds global ids after re-basing).
PHFEM_API phfem_status phfem_dist_classify_ex(phfem_ctx* ctx, const phfem_topology* part, int32_t E0,
                                              const int32_t* dir_ids, int32_t nD, const int32_t* neu_ids,
                                              int32_t nN, int32_t r_off, int32_t e_off,
                                              phfem_classification* out) {
  memset(out, 0, sizeof(*out));
  if (!ctx || !part) return PHFEM_ERR_INVALID_ARGUMENT;
  const int E = part->E;
  const int nwords = (E + 31) / 32;
  out->E = E;
  PHFEM_TRY(dalloc(ctx, &out->neumann_bits, nwords));
  PHFEM_CUDA(ctx, cudaMemsetAsync(out->neumann_bits, 0, sizeof(uint32_t) * std::max(nwords, 1), ctx->stream));
  unsigned long long* dup = nullptr;
  PHFEM_TRY(dalloc(ctx, &dup, 1));
  PHFEM_CUDA(ctx, cudaMemsetAsync(dup, 0, sizeof(unsigned long long), ctx->stream));
  if (nN > 0)
    PHFEM_LAUNCH(ctx, "k_dist_neu_bits", k_dist_neu_bits<<<grid_for(nN, 256, ctx->num_sms * 4), 256, 0, ctx->stream>>>(
        neu_ids, nN, 0, E, out->neumann_bits, dup));
  // local Dirichlet / Neumann id lists (owned entries, list order)
  auto compact = [&](const int32_t* ids, int n, int32_t** dst, int32_t* count) -> phfem_status {
    int32_t* flag = nullptr;
    PHFEM_TRY(dalloc(ctx, &flag, (int64_t)n + 1));
    PHFEM_CUDA(ctx, cudaMemsetAsync(flag, 0, sizeof(int32_t) * (n + 1), ctx->stream));
    if (n > 0)
      PHFEM_LAUNCH(ctx, "k_dist_local_ids", k_dist_local_ids<<<grid_for(n, 256, ctx->num_sms * 4), 256, 0, ctx->stream>>>(
          ids, n, 0, E, flag));
    PHFEM_TRY(scan_exclusive_i32(ctx, flag, flag, (int64_t)n + 1, nullptr));
    int32_t c = 0;
    PHFEM_CUDA(ctx, cudaMemcpyAsync(&c, flag + n, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
    PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    PHFEM_TRY(dalloc(ctx, dst, c));
    if (n > 0)
      PHFEM_LAUNCH(ctx, "k_dist_compact", k_dist_compact<<<grid_for(n, 256, ctx->num_sms * 4), 256, 0, ctx->stream>>>(
          ids, flag, n, 0, E, *dst));
    *count = c;
    dfree(ctx, flag);
    return PHFEM_OK;
  };
  PHFEM_TRY(compact(dir_ids, nD, &out->dirichlet_edge_ids, &out->nD));
  PHFEM_TRY(compact(neu_ids, nN, &out->neumann_edge_ids, &out->nN));
  unsigned long long hdup = 0;
  PHFEM_CUDA(ctx, cudaMemcpyAsync(&hdup, dup, sizeof hdup, cudaMemcpyDeviceToHost, ctx->stream));
  PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  dfree(ctx, dup);
  out->flags = hdup ? PHFEM_CLS_DUP_NEUMANN : 0;
  return classify_lists_from_bits(ctx, part, out, E0, r_off, e_off);
}

// The same when the (fused) level kernel already wrote retained_pos [part->E]
// / retained_edges [L] (global rows / ids, ctx memory: ownership moves into
// *out): only the Neumann bitmap and the rank's id lists remain.  No host
// synchronisation (the sharded pipeline overlaps it with the element pass);
// flags stay 0 — the caller, which holds the global Neumann list, sets
// PHFEM_CLS_DUP_NEUMANN.
PHFEM_API phfem_status phfem_dist_classify_given(phfem_ctx* ctx, const phfem_topology* part,
                                                 const int32_t* dir_ids, int32_t nD, const int32_t* neu_ids,
                                                 int32_t nN, int32_t* retained_pos, int32_t* retained_edges,
                                                 int32_t L, phfem_classification* out) {
  memset(out, 0, sizeof(*out));
  if (!ctx || !part || L < 0 || L > part->E || (part->E && !retained_pos) || (L && !retained_edges) ||
      (nD && !dir_ids) || (nN && !neu_ids))
    return PHFEM_ERR_INVALID_ARGUMENT;
  const int E = part->E;
  const int nwords = (E + 31) / 32;
  out->E = E;
  out->L = L;
  out->retained_pos = retained_pos;
  out->retained_edges = retained_edges;
  PHFEM_TRY(dalloc(ctx, &out->neumann_bits, nwords));
  PHFEM_CUDA(ctx, cudaMemsetAsync(out->neumann_bits, 0, sizeof(uint32_t) * std::max(nwords, 1), ctx->stream));
  if (nN > 0)
    PHFEM_LAUNCH(ctx, "k_dist_neu_bits", k_dist_neu_bits<<<grid_for(nN, 256, ctx->num_sms * 4), 256, 0, ctx->stream>>>(
        neu_ids, nN, 0, E, out->neumann_bits, nullptr));
  // the ids are the rank's own already (local, list order): plain copies
  PHFEM_TRY(dalloc(ctx, &out->dirichlet_edge_ids, nD));
  PHFEM_TRY(dalloc(ctx, &out->neumann_edge_ids, nN));
  if (nD) PHFEM_CUDA(ctx, cudaMemcpyAsync(out->dirichlet_edge_ids, dir_ids, sizeof(int32_t) * nD,
                                          cudaMemcpyDeviceToDevice, ctx->stream));
  if (nN) PHFEM_CUDA(ctx, cudaMemcpyAsync(out->neumann_edge_ids, neu_ids, sizeof(int32_t) * nN,
                                          cudaMemcpyDeviceToDevice, ctx->stream));
  out->nD = nD;
  out->nN = nN;
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_dist_classify(phfem_ctx* ctx, const phfem_topology* part, int32_t E0,
                                           const int32_t* dir_ids, int32_t nD,
                                           const int32_t* neu_ids, int32_t nN,
                                           phfem_classification* out) {
  return phfem_dist_classify_ex(ctx, part, E0, dir_ids, nD, neu_ids, nN, 0, 0, out);
}

PHFEM_API phfem_status phfem_dist_neumann_table(phfem_ctx* ctx, const phfem_topology* part,
                                                int32_t E0, const int32_t* neu_ids, int32_t nN,
                                                int32_t* table) {
  if (!ctx || !part || (nN && (!neu_ids || !table))) return PHFEM_ERR_INVALID_ARGUMENT;
  if (nN == 0) return PHFEM_OK;
  PHFEM_CUDA(ctx, cudaMemsetAsync(table, 0, sizeof(int32_t) * 4 * (int64_t)nN, ctx->stream));
  PHFEM_LAUNCH(ctx, "k_dist_neu_table", k_dist_neu_table<<<grid_for(nN, 256, ctx->num_sms * 4), 256, 0, ctx->stream>>>(
      neu_ids, nN, E0, part->E, part->edge_nodes, part->edge_elements, part->local_in_tplus, table));
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_dist_neumann_apply(phfem_ctx* ctx, const phfem_mesh* mesh,
                                                const int32_t* table, int32_t nN, int32_t dup,
                                                int32_t elo, int32_t ehi, const phfem_field* g,
                                                double t, double* load_local) {
  if (!ctx || !mesh || !g || (nN && (!table || !load_local))) return PHFEM_ERR_INVALID_ARGUMENT;
  if (nN == 0) return PHFEM_OK;
  phfem_topology mt;
  memset(&mt, 0, sizeof mt);
  phfem_classification mc;
  memset(&mc, 0, sizeof mc);
  int32_t *flag = nullptr, *pos = nullptr;
  PHFEM_TRY(dalloc(ctx, &mt.edge_nodes, 2 * (int64_t)nN));
  PHFEM_TRY(dalloc(ctx, &mt.edge_elements, 2 * (int64_t)nN));
  PHFEM_TRY(dalloc(ctx, &mt.local_in_tplus, nN));
  PHFEM_TRY(dalloc(ctx, &flag, nN));
  PHFEM_TRY(dalloc(ctx, &pos, (int64_t)nN + 1));
  PHFEM_LAUNCH(ctx, "k_dist_neu_mini", k_dist_neu_mini<<<grid_for(nN, 256, ctx->num_sms * 4), 256, 0, ctx->stream>>>(
      table, nN, elo, ehi, mt.edge_nodes, mt.edge_elements, mt.local_in_tplus, flag));
  PHFEM_CUDA(ctx, cudaMemcpyAsync(pos, flag, sizeof(int32_t) * nN, cudaMemcpyDeviceToDevice, ctx->stream));
  PHFEM_CUDA(ctx, cudaMemsetAsync(pos + nN, 0, sizeof(int32_t), ctx->stream));
  PHFEM_TRY(scan_exclusive_i32(ctx, pos, pos, (int64_t)nN + 1, nullptr));
  int32_t c = 0;
  PHFEM_CUDA(ctx, cudaMemcpyAsync(&c, pos + nN, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
  PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  phfem_status st = PHFEM_OK;
  if (c > 0) {
    PHFEM_TRY(dalloc(ctx, &mc.neumann_edge_ids, c));
    PHFEM_LAUNCH(ctx, "k_dist_iota_compact", k_dist_iota_compact<<<grid_for(nN, 256, ctx->num_sms * 4), 256, 0, ctx->stream>>>(
        flag, pos, nN, mc.neumann_edge_ids));
    mt.E = nN;
    mc.nN = c;
    mc.E = nN;
    mc.flags = dup ? PHFEM_CLS_DUP_NEUMANN : 0;
    // coordinates global, load array and the mini topology's elements local
    st = neumann_into(ctx, mesh, &mt, &mc, g, t, load_local, 1, true);
    dfree(ctx, mc.neumann_edge_ids);
  }
  dfree(ctx, flag);
  dfree(ctx, pos);
  dfree(ctx, mt.edge_nodes);
  dfree(ctx, mt.edge_elements);
  dfree(ctx, mt.local_in_tplus);
  return st;
}

PHFEM_API phfem_status phfem_dist_side_records(phfem_ctx* ctx, const int32_t* elements, const int32_t* elem_edge,
                                               int32_t n, const int32_t* esplits, int32_t W, int32_t* counts,
                                               int32_t* offsets, int32_t* send) {
  if (!ctx || !esplits || !counts || W < 1 || n < 0 || (n && (!elements || !elem_edge)))
    return PHFEM_ERR_INVALID_ARGUMENT;
  const int grid = grid_for(3 * (int64_t)n, kRouteThreads * kRouteK, ctx->num_sms * 8);
  return route_two_pass(ctx, W, counts, offsets, send != nullptr, [&](int32_t* c, int32_t* cur) -> phfem_status {
    if (n > 0)
      PHFEM_LAUNCH(ctx, "k_dist_side", k_dist_side<<<grid, kRouteThreads, 0, ctx->stream>>>(
          elements, elem_edge, n, esplits, W, c, cur, cur ? reinterpret_cast<int4*>(send) : nullptr));
    return PHFEM_OK;
  });
}

PHFEM_API phfem_status phfem_dist_side_apply(phfem_ctx* ctx, const int32_t* recv, int64_t n, int32_t E0, int32_t E,
                                             int32_t* side) {
  if (!ctx || (n && (!recv || !side))) return PHFEM_ERR_INVALID_ARGUMENT;
  if (n > 0)
    PHFEM_LAUNCH(ctx, "k_dist_side_apply", k_dist_side_apply<<<grid_for(n, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
        reinterpret_cast<const int4*>(recv), n, E0, E, reinterpret_cast<int4*>(side)));
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_dist_start_records(phfem_ctx* ctx, const phfem_topology* ppart,
                                                const int32_t* fine_nes, int32_t nes_off, const uint8_t* rk,
                                                const int32_t* psplits, int32_t W, int32_t* counts,
                                                int32_t* offsets, int32_t* send) {
  if (!ctx || !ppart || !psplits || !counts || W < 1 || (ppart->E && (!fine_nes || !rk)))
    return PHFEM_ERR_INVALID_ARGUMENT;
  const int E = ppart->E;
  const int grid = grid_for(2 * (int64_t)E, kRouteThreads * kRouteK, ctx->num_sms * 8);
  return route_two_pass(ctx, W, counts, offsets, send != nullptr, [&](int32_t* c, int32_t* cur) -> phfem_status {
    if (E > 0)
      PHFEM_LAUNCH(ctx, "k_dist_start", k_dist_start<<<grid, kRouteThreads, 0, ctx->stream>>>(
          ppart->edge_elements, ppart->local_in_tplus, ppart->local_in_tminus, fine_nes, nes_off, rk, E, psplits, W,
          c, cur, cur ? reinterpret_cast<Rec3*>(send) : nullptr));
    return PHFEM_OK;
  });
}

PHFEM_API phfem_status phfem_dist_start_apply(phfem_ctx* ctx, const int32_t* recv, int64_t n, int32_t elo,
                                              int32_t* gs, uint8_t* grk) {
  if (!ctx || (n && (!recv || !gs || !grk))) return PHFEM_ERR_INVALID_ARGUMENT;
  if (n > 0)
    PHFEM_LAUNCH(ctx, "k_dist_start_apply", k_dist_start_apply<<<grid_for(n, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
        reinterpret_cast<const Rec3*>(recv), n, elo, gs, grk));
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_dist_side_p2p_ex(phfem_ctx* ctx, const int32_t* elements, const int32_t* elem_edge,
                                              int32_t n, const int32_t* esplits, int32_t W, int32_t self,
                                              int32_t* const* peer_side, int32_t* remote, int skip_self) {
  if (!ctx || !esplits || !peer_side || !remote || W < 1 || W > kRemoteMax || self < 0 || self >= W || n < 0 ||
      (n && (!elements || !elem_edge)))
    return PHFEM_ERR_INVALID_ARGUMENT;
  PHFEM_CUDA(ctx, cudaMemsetAsync(remote, 0, sizeof(int32_t) * W, ctx->stream));
  if (n > 0)
    PHFEM_LAUNCH(ctx, "k_dist_side_p2p", k_dist_side_p2p<<<grid_for(3 * (int64_t)n, 256, ctx->num_sms * PHFEM_P2P_GRID_MULT), 256, 0,
                                                           ctx->stream>>>(
        elements, elem_edge, n, esplits, W, self, reinterpret_cast<int4* const*>(peer_side), remote, skip_self));
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_dist_side_p2p(phfem_ctx* ctx, const int32_t* elements, const int32_t* elem_edge,
                                           int32_t n, const int32_t* esplits, int32_t W, int32_t self,
                                           int32_t* const* peer_side, int32_t* remote) {
  return phfem_dist_side_p2p_ex(ctx, elements, elem_edge, n, esplits, W, self, peer_side, remote, 0);
}

PHFEM_API phfem_status phfem_dist_start_p2p_ex(phfem_ctx* ctx, const phfem_topology* ppart, const int32_t* fine_nes,
                                               int32_t nes_off, const uint8_t* rk, const int32_t* psplits, int32_t W,
                                               int32_t self, int32_t* const* peer_gs, uint8_t* const* peer_grk,
                                               int32_t* remote, int skip_self) {
  if (!ctx || !ppart || !psplits || !peer_gs || !peer_grk || !remote || W < 1 || W > kRemoteMax || self < 0 || self >= W ||
      (ppart->E && (!fine_nes || !rk)))
    return PHFEM_ERR_INVALID_ARGUMENT;
  PHFEM_CUDA(ctx, cudaMemsetAsync(remote, 0, sizeof(int32_t) * W, ctx->stream));
  const int E = ppart->E;
  if (E > 0)
    PHFEM_LAUNCH(ctx, "k_dist_start_p2p", k_dist_start_p2p<<<grid_for(2 * (int64_t)E, 256, ctx->num_sms * PHFEM_P2P_GRID_MULT), 256, 0,
                                                             ctx->stream>>>(
        ppart->edge_elements, ppart->local_in_tplus, ppart->local_in_tminus, fine_nes, nes_off, rk, E, psplits, W,
        self, peer_gs, peer_grk, remote, skip_self));
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_dist_start_p2p(phfem_ctx* ctx, const phfem_topology* ppart, const int32_t* fine_nes,
                                            int32_t nes_off, const uint8_t* rk, const int32_t* psplits, int32_t W,
                                            int32_t self, int32_t* const* peer_gs, uint8_t* const* peer_grk,
                                            int32_t* remote) {
  return phfem_dist_start_p2p_ex(ctx, ppart, fine_nes, nes_off, rk, psplits, W, self, peer_gs, peer_grk, remote, 0);
}

PHFEM_API phfem_status phfem_dist_pairs_p2p(phfem_ctx* ctx, const int32_t* pairs, int64_t n, int32_t E0,
                                            const int32_t* esplits, int32_t W, int32_t self, int32_t* const* peer_ee,
                                            int32_t* remote) {
  if (!ctx || (n && !pairs) || !esplits || !peer_ee || !remote || W < 1 || W > kRemoteMax || self < 0 || self >= W)
    return PHFEM_ERR_INVALID_ARGUMENT;
  PHFEM_CUDA(ctx, cudaMemsetAsync(remote, 0, sizeof(int32_t) * W, ctx->stream));
  if (n > 0)
    PHFEM_LAUNCH(ctx, "k_dist_pairs_p2p", k_dist_pairs_p2p<<<grid_for(n, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
        reinterpret_cast<const int2*>(pairs), n, E0, esplits, W, self, peer_ee, remote));
  return PHFEM_OK;
}
