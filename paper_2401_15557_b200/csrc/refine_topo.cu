// refine_topo.cu — topology of the red-refined mesh straight from the parent
// topology, no sort.
//
// Result is bit-identical to build_topology(red_refine(M)) (reference
// edge_topology.cpp:52-143 applied to refine.cpp:7-53's output):
//  * every fine edge has a midpoint node mu(e) = nc + e as its larger node, so
//    the canonical (max, min) order groups fine edges by parent edge e;
//  * group e = [half at min(a,b), half at max(a,b), then the interior edges
//    mu(e')-mu(e) for the e' < e that share a parent element with e, by e'];
//  * halves of e = (a,b): a->mu in child 4tp+1+(l+1)%3 (local 2) / child
//    4tm+1+(l'+2)%3 (local 1); mu->b in 4tp+1+(l+2)%3 (local 1) / 4tm+1+(l'+1)%3
//    (local 2); interior edge opposite M_k of parent m: M_{k+1}->M_{k+2},
//    t_plus = 4m (local k), t_minus = 4m+1+k (local 0).
// (Derived from the child layout refine.cpp:33-36 and the emission order
// edge_topology.cpp:61-68; tests/test_gpu_parity.py checks it against the
// oracle's sort-based build_topology.)
//
// Device algorithm: one main kernel over the parent edges (k_rl_level),
// one thread per parent edge, 128 edges per tile:
//   1. coalesced loads of the parent edge record; gathers of elem_edge and the
//      opposite vertex of t_plus / t_minus (the partner edges of e in each
//      element sit at the local indices next to ltp / ltm: no search);
//   2. group size = 2 + #partners < e; one packed block scan gives the
//      in-tile (fine edges, boundary, Neumann) prefixes; the tile offsets come
//      from a tiny pre-pass (k_rl_tile_init / k_rl_tile_count: per-tile
//      totals from the coalesced parent elem_edge, then scans of one int per
//      tile).  A decoupled look-back was measured slower here: 128-edge
//      tiles finish faster than the look-back frontier advances;
//   3. the 4 coordinates every fine-edge length needs (a, b and the two
//      opposite vertices) are gathered once per parent edge: fine midpoints
//      are 0.5 (x + y) of parent vertices, so lengths are recomputed from the
//      parent geometry with the same bits as edge_lengths on the fine mesh
//      (edge_topology.cpp:179-186) and the midpoint node mu(e) itself is
//      written coalesced here (refine.cpp:16-19);
//   4. fine-edge records are staged in SMEM and stored coalesced; with kFull
//      the retained positions, retained list, CSR rows of C and their
//      (column, value) entries (assembly.cpp:144-168) are emitted in the
//      same pass (the fine Neumann edges are the halves of the parent's);
//   5. the fine elem_edge is NOT scattered from here (two 4-byte stores per
//      fine edge bounded the kernel): one rank byte per parent edge goes
//      out instead, and k_refine_children (one thread per parent element)
//      writes the children rows and their elem_edge as coalesced rows from
//      the group starts and those ranks.  The distributed variant keeps the
//      per-fine-edge stores (own elements in place, others as pairs).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.cuh"

namespace phfem {

#ifndef PHFEM_LV_TILE
#define PHFEM_LV_TILE 128
#endif
constexpr int kLvT = PHFEM_LV_TILE;  // parent edges (= threads) per tile
constexpr int kLvF = 6 * kLvT;     // fine-edge slots per tile (<= 6 per parent edge)

__device__ __forceinline__ int abs_edge(int s) { return s >= 0 ? s : ~s; }

struct LvArgs {
  // parent topology
  const int32_t* edge_nodes;
  const int32_t* edge_elements;
  const int32_t* ltp;
  const int32_t* ltm;
  const int32_t* elem_edge;
  // parent mesh
  const int32_t* elements;
  const double2* coords;
  // parent classification (kFull)
  const uint32_t* neu_bits;
  int E, nc, Ef, L;
  // distributed level (phfem_dist_refine_level): the parent edge arrays hold
  // edges [eb, eb + E) at local indices; node_edge_start covers the fine node
  // range from nlo.  Both 0 on one GPU.
  int eb, nlo;
  // distributed level, side-record mode: side[2 le + s] = {the two partner
  // edges of e in its t_plus (s = 0) / t_minus (s = 1) element at local
  // indices l+1, l+2, the opposite vertex, -} (phfem_dist_side_apply) instead
  // of gathers from elem_edge / elements of every parent element
  const int4* side;
  // local mode (side records of the rank's own element slots not stored):
  // those elements' rows / elem_edge [own_hi - own_lo][3] from own_el / own_ee
  const int32_t* own_el;
  const int32_t* own_ee;
  int own_lo, own_hi;
  // distributed level with the fine offsets known up front: global ids
  // written directly (fine edge ids in the lists and node_edge_start, C row
  // pointers) — no re-basing pass; 0 on one GPU
  int f_off, nnz_off;
  int r_off;  // global retained row of the rank's first row (distributed fused classification)
  // exclusive per-tile prefixes (k_rl_tile_init / k_rl_tile_count + scans):
  // fine edges, parent boundary edges, parent Neumann edges before the tile
  const int32_t* tileF;
  const int32_t* tileB;
  const int32_t* tileN;
};

struct LvOut {
  int32_t* edge_nodes;
  int32_t* edge_elements;
  int32_t* ltp;
  int32_t* ltm;
  int32_t* interior;
  int32_t* boundary;
  int32_t* elem_edge;  // nullable: with rk the element pass (k_refine_children) writes it
  int32_t* node_edge_start;
  // per parent edge e: the in-group ranks of its interior fine edges, 2 bits
  // each (partner at j1 / j2 of t_plus, k1 / k2 of t_minus) — all the
  // element pass needs besides the group starts
  uint8_t* rk;
  double2* mid;  // nullable: mid[nc + e - mid_base] = midpoint of parent edge e
  int64_t mid_base;
  int2* pairs;   // distributed level: (slot 3m+l, f / ~f) per fine edge instead of elem_edge
  // distributed level with an own range: slots [self_lo3, self_hi3) go to
  // self_ee directly (local f / ~f); only the others are appended to pairs
  int32_t* self_ee;
  int64_t self_lo3, self_hi3;
  int32_t* npairs;
  // kFull
  int32_t* rpos;
  int32_t* redges;
  int32_t* row_ptr;
  int32_t* col;
  double* val;
};

template <bool kFull>
struct LvSmem {
  int2 en[kLvF];
  int2 el[kLvF];
  // tile-local list slot << 8 | lp | (lm + 1) << 2; the slot is the interior
  // list index, or ~(boundary list index) — both offsets are added at store time
  int32_t ms[kLvF];
  int32_t rr[kFull ? kLvF : 1];  // retained: local row << 16 | local row start; else -1
  double len[kFull ? kLvF : 1];
  int32_t scan[33];
};

__device__ __forceinline__ double seg_len(double2 p, double2 q) {
  const double dx = q.x - p.x, dy = q.y - p.y;
  return sqrt(dx * dx + dy * dy);  // edge_topology.cpp:183 (Eigen norm)
}

__device__ __forceinline__ double2 midpt(double2 p, double2 q) {
  return make_double2(0.5 * (p.x + q.x), 0.5 * (p.y + q.y));  // refine.cpp:18
}

// Per-tile totals before the scans.  Group e holds 2 halves plus, for every
// parent element with sorted edge ids x < y < z, one interior fine edge in
// group y and two in group z — so the fine-edge count of a tile is
// 2 (edges in tile) + element contributions, accumulated element-parallel
// (coalesced elem_edge reads, warp-aggregated atomics).
__global__ void k_rl_tile_init(int E, int eb, int ntiles, const int32_t* __restrict__ boundary, int nB,
                               const uint32_t* __restrict__ neu_bits, int32_t* __restrict__ tileF,
                               int32_t* __restrict__ tileB, int32_t* __restrict__ tileN) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += gridDim.x * blockDim.x) {
    const int64_t l0 = (int64_t)t * kLvT;
    const int64_t l1 = l0 + kLvT < E ? l0 + kLvT : E;
    const int64_t e0 = eb + l0, e1 = eb + l1;  // global parent edge ids of the tile
    tileF[t] = 2 * (int)(l1 - l0);
    auto lower = [&](int64_t key) {  // ascending boundary list
      int l = 0, r = nB;
      while (l < r) {
        const int mid = (l + r) >> 1;
        if (__ldg(boundary + mid) < key) l = mid + 1;
        else r = mid;
      }
      return l;
    };
    tileB[t] = lower(e1) - lower(e0);
    if (neu_bits) {  // bitmap over the local edge index
      int c = 0;
      for (int64_t w = l0 >> 5; w < (l1 + 31) >> 5; ++w) c += __popc(__ldg(neu_bits + w));
      tileN[t] = c;
    }
  }
}

// side record {partner at l+1, partner at l+2, opposite vertex, -} of parent
// edge le in element t (local index l, sd 0 t_plus / 1 t_minus): the stored
// record, or in local mode a gather from the rank's own element arrays
__device__ __forceinline__ int4 side_of(const int4* __restrict__ side, int64_t le, int sd, int t, int l,
                                        const int32_t* __restrict__ own_el, const int32_t* __restrict__ own_ee,
                                        int own_lo, int own_hi) {
  if (own_el && t >= own_lo && t < own_hi) {
    const int64_t b = 3 * (int64_t)(t - own_lo);
    return make_int4(__ldg(own_ee + b + (l == 2 ? 0 : l + 1)), __ldg(own_ee + b + (l == 0 ? 2 : l - 1)),
                     __ldg(own_el + b + l), 0);
  }
  return side[2 * le + sd];
}

__device__ __forceinline__ void warp_add(int32_t* ctr, int key, int v) {
  const unsigned g = __match_any_sync(__activemask(), key);
  if ((int)lane_id() == __ffs(g) - 1) atomicAdd(ctr + key, v * __popc(g));
}

// (eb, E): only the groups of parent edges [eb, eb + E) count (a rank's range)
__global__ void k_rl_tile_count(const int32_t* __restrict__ elem_edge, int nE, int eb, int E,
                                int32_t* __restrict__ tileF) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < nE; m += stride) {
    const int x = abs_edge(__ldg(elem_edge + 3 * m)), y = abs_edge(__ldg(elem_edge + 3 * m + 1)),
              z = abs_edge(__ldg(elem_edge + 3 * m + 2));
    const int hi = max(x, max(y, z)) - eb;
    const int md = max(min(x, y), min(max(x, y), z)) - eb;
    if (md >= 0 && md < E) warp_add(tileF, md / kLvT, 1);
    if (hi >= 0 && hi < E) warp_add(tileF, hi / kLvT, 2);
  }
}

// k_rl_tile_init + k_rl_tile_count in one launch (blocks [0, blocksA) the
// tile pass, the rest the element pass; tileF accumulated with atomics on
// both sides, zeroed by the caller): one launch less per refinement level —
// the small levels of a deep refinement are launch-bound.
__global__ void k_rl_tile_prep(int E, int ntiles, const int32_t* __restrict__ boundary, int nB,
                               const uint32_t* __restrict__ neu_bits, int32_t* __restrict__ tileF,
                               int32_t* __restrict__ tileB, int32_t* __restrict__ tileN,
                               const int32_t* __restrict__ elem_edge, int nE, int blocksA) {
  pdl_wait();
  pdl_trigger();
  if ((int)blockIdx.x < blocksA) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += blocksA * blockDim.x) {
      const int64_t l0 = (int64_t)t * kLvT;
      const int64_t l1 = l0 + kLvT < E ? l0 + kLvT : E;
      atomicAdd(tileF + t, 2 * (int)(l1 - l0));
      auto lower = [&](int64_t key) {
        int l = 0, r = nB;
        while (l < r) {
          const int mid = (l + r) >> 1;
          if (__ldg(boundary + mid) < key) l = mid + 1;
          else r = mid;
        }
        return l;
      };
      tileB[t] = lower(l1) - lower(l0);
      if (neu_bits) {
        int c = 0;
        for (int64_t w = l0 >> 5; w < (l1 + 31) >> 5; ++w) c += __popc(__ldg(neu_bits + w));
        tileN[t] = c;
      }
    }
    return;
  }
  const int64_t stride = (int64_t)(gridDim.x - blocksA) * blockDim.x;
  for (int64_t m = (blockIdx.x - blocksA) * (int64_t)blockDim.x + threadIdx.x; m < nE; m += stride) {
    const int x = abs_edge(__ldg(elem_edge + 3 * m)), y = abs_edge(__ldg(elem_edge + 3 * m + 1)),
              z = abs_edge(__ldg(elem_edge + 3 * m + 2));
    const int hi = max(x, max(y, z));
    const int md = max(min(x, y), min(max(x, y), z));
    if (md < E) warp_add(tileF, md / kLvT, 1);
    if (hi < E) warp_add(tileF, hi / kLvT, 2);
  }
}

// k_refine_children grid: 64 CTAs per SM (~14 element rows per thread at
// L12 -> L13) — measured 0.827 ms at 16 per SM, 0.753 at 64, 0.757 at 256,
// 0.793 at 1024 (more concurrent store windows, as for k_volume)
#ifndef PHFEM_CH_GRID_MULT
#define PHFEM_CH_GRID_MULT 64
#endif
#ifndef PHFEM_LV_MIN_BLOCKS
#define PHFEM_LV_MIN_BLOCKS 7
#endif
// stage 1: the parent edge record (coalesced)
struct LvRec {
  int2 ab, el;
  int l, l2;
  bool neu;
};
// stage 2: the gathers of the two parent elements: the partner edges of e
// (signed, at local l+1 / l+2 of t_plus and l2+1 / l2+2 of t_minus) and the
// opposite vertices
struct LvGat {
  int pj1, pj2, qk1, qk2;
  int vop, vom;
};
// stage 3: the four parent coordinates
struct LvCrd {
  double2 ca, cb, cop, com;
};

template <bool kFull>
__device__ __forceinline__ LvRec lv_load_rec(const LvArgs& a, int le) {
  LvRec r;
  r.ab = make_int2(0, 0);
  r.el = make_int2(0, -1);
  r.l = r.l2 = 0;
  r.neu = false;
  if (le < a.E) {
    r.ab = reinterpret_cast<const int2*>(a.edge_nodes)[le];
    r.el = reinterpret_cast<const int2*>(a.edge_elements)[le];
    r.l = __ldg(a.ltp + le);
    r.l2 = __ldg(a.ltm + le);  // -1 on the boundary
    if (kFull) r.neu = (__ldg(a.neu_bits + (le >> 5)) >> (le & 31)) & 1u;
  }
  return r;
}

__device__ __forceinline__ LvGat lv_load_gat(const LvArgs& a, const LvRec& r, bool valid, int le) {
  LvGat g;
  g.pj1 = g.pj2 = g.qk1 = g.qk2 = 0;
  g.vop = g.vom = 0;
  if (a.side) {  // distributed: the element owners' side records, coalesced (local mode: own slots gathered)
    if (valid) {
      const int4 sp = side_of(a.side, le, 0, r.el.x, r.l, a.own_el, a.own_ee, a.own_lo, a.own_hi);
      g.pj1 = sp.x;
      g.pj2 = sp.y;
      g.vop = sp.z;
    }
    if (valid && r.el.y >= 0) {
      const int4 sm = side_of(a.side, le, 1, r.el.y, r.l2, a.own_el, a.own_ee, a.own_lo, a.own_hi);
      g.qk1 = sm.x;
      g.qk2 = sm.y;
      g.vom = sm.z;
    }
    return g;
  }
  if (valid) {
    const int64_t tp = 3 * (int64_t)r.el.x;
    const int j1 = r.l == 2 ? 0 : r.l + 1, j2 = r.l == 0 ? 2 : r.l - 1;
    g.pj1 = __ldg(a.elem_edge + tp + j1);
    g.pj2 = __ldg(a.elem_edge + tp + j2);
    g.vop = __ldg(a.elements + tp + r.l);
  }
  if (valid && r.el.y >= 0) {
    const int64_t tm = 3 * (int64_t)r.el.y;
    const int k1 = r.l2 == 2 ? 0 : r.l2 + 1, k2 = r.l2 == 0 ? 2 : r.l2 - 1;
    g.qk1 = __ldg(a.elem_edge + tm + k1);
    g.qk2 = __ldg(a.elem_edge + tm + k2);
    g.vom = __ldg(a.elements + tm + r.l2);
  }
  return g;
}

__device__ __forceinline__ LvCrd lv_load_crd(const LvArgs& a, const LvRec& r, const LvGat& g, bool valid) {
  LvCrd c;
  c.ca = c.cb = c.cop = c.com = make_double2(0.0, 0.0);
  if (valid) {
    c.ca = __ldg(a.coords + r.ab.x);
    c.cb = __ldg(a.coords + r.ab.y);
    c.cop = __ldg(a.coords + g.vop);
  }
  if (valid && r.el.y >= 0) c.com = __ldg(a.coords + g.vom);
  return c;
}

// One tile of 128 parent edges from its three load stages: group sizes, the
// packed block scan, fine edges into SMEM, coalesced stores.
template <bool kFull>
__device__ __forceinline__ void lv_tile(const LvArgs& a, const LvOut& o, LvSmem<kFull>& s, int tile,
                                        const LvRec& r, const LvGat& g, const LvCrd& c) {
  const int tid = threadIdx.x;
  const int64_t e0 = (int64_t)tile * kLvT;
  const int le = (int)(e0 + tid);  // index into the parent edge arrays
  const int e = a.eb + le;         // global parent edge id
  const bool valid = le < a.E;
  const int2 ab = r.ab;
  const int l = r.l;
  const bool neu = r.neu;
  const bool has_m = valid && r.el.y >= 0;
  const int l2 = has_m ? r.l2 : 0;
  const int tp = r.el.x, tm = r.el.y;
  const double2 ca = c.ca, cb = c.cb, cop = c.cop, com = c.com;

  // 2. group size, tile scan, look-back
  const int j1 = l == 2 ? 0 : l + 1, j2 = l == 0 ? 2 : l - 1;      // partners in t_plus
  const int k1 = l2 == 2 ? 0 : l2 + 1, k2 = l2 == 0 ? 2 : l2 - 1;  // partners in t_minus
  const int q0 = abs_edge(g.pj1), q1 = abs_edge(g.pj2);
  const int r0 = abs_edge(g.qk1), r1 = abs_edge(g.qk2);
  const bool v0 = valid && q0 < e, v1 = valid && q1 < e;
  const bool v2 = has_m && r0 < e, v3 = has_m && r1 < e;
  const bool isB = valid && !has_m;
  const int cnt = valid ? 2 + v0 + v1 + v2 + v3 : 0;
  const int packed = cnt | (int)isB << 11 | (int)neu << 20;
  int tot;
  const int ex = block_exclusive_scan(packed, s.scan, &tot);
  const int i0 = ex & 0x7ff;            // first slot of group e in the tile
  const int exB = (ex >> 11) & 0x1ff;   // parent boundary edges before e in the tile
  const int exN = ex >> 20;             // parent Neumann edges before e in the tile

  // 3. the group's fine edges into SMEM, with TILE-LOCAL offsets only: the
  //    global ones are added at store time, so the look-back below overlaps
  //    nothing but its own latency
  const int mu = a.nc + e;
  const double2 me = midpt(ca, cb);
  if (valid) {
    if (o.mid) o.mid[mu - o.mid_base] = me;
    auto emit = [&](int j, int from, int to, int tpf, int lp, int tmf, int lm, double len) {
      const int i = i0 + j;
      s.en[i] = make_int2(from, to);
      s.el[i] = make_int2(tpf, tmf);
      // list slot: boundary list 2 B_e + j, else interior list f - 2 B_e - (2 if isB)
      const int slot = (j < 2 && isB) ? ~(2 * exB + j) : i - 2 * exB - (isB ? 2 : 0);
      s.ms[i] = slot * 256 | lp | (tmf >= 0 ? lm + 1 : 0) << 2;  // local_in_tminus = -1 on the boundary
      if (kFull) {
        int rr = -1;
        if (j >= 2 || !neu) {
          const int rp = i0 - 2 * exN + (neu ? j - 2 : j);
          const int bret = 2 * (exB - exN) + ((isB && !neu) ? (j == 1 ? 1 : (j >= 2 ? 2 : 0)) : 0);
          rr = rp << 16 | (4 * rp - 2 * bret);  // both in [0, 4 kLvF)
          s.len[i] = len;
        }
        s.rr[i] = rr;
      }
    };
    // halves: a -> mu and mu -> b; the one at the smaller old node first
    const int ia = ab.x < ab.y ? 0 : 1;
    emit(ia, ab.x, mu, 4 * tp + 1 + j1, 2, has_m ? 4 * tm + 1 + k2 : -1, 1, kFull ? seg_len(ca, me) : 0.0);
    emit(1 - ia, mu, ab.y, 4 * tp + 1 + j2, 1, has_m ? 4 * tm + 1 + k1 : -1, 2,
         kFull ? seg_len(me, cb) : 0.0);
    // interior edges mu(e') - mu(e), e' < e, ascending e'.  Candidate
    // (partner, element, third local index kk): the edge opposite M_kk of the
    // element's central child runs M_{kk+1} -> M_{kk+2}.
    const int rk0 = (v1 && q1 < q0) + (v2 && r0 < q0) + (v3 && r1 < q0);
    const int rk1 = (v0 && q0 < q1) + (v2 && r0 < q1) + (v3 && r1 < q1);
    const int rk2 = (v0 && q0 < r0) + (v1 && q1 < r0) + (v3 && r1 < r0);
    const int rk3 = (v0 && q0 < r1) + (v1 && q1 < r1) + (v2 && r0 < r1);
    if (o.rk) o.rk[le] = (uint8_t)(rk0 | rk1 << 2 | rk2 << 4 | rk3 << 6);
    // t_plus vertices: V(l) = cop, V(l+1) = ca, V(l+2) = cb; midpoint of the
    // edge at local j = 0.5 (V(j+1) + V(j+2)).  t_minus: W(l2) = com,
    // W(l2+1) = cb, W(l2+2) = ca.
    if (v0)  // partner at j1, kk = j2: mu(e) -> mu(q0)
      emit(2 + rk0, mu, a.nc + q0, 4 * tp, j2, 4 * tp + 1 + j2, 0,
           kFull ? seg_len(me, midpt(cb, cop)) : 0.0);
    if (v1)  // partner at j2, kk = j1: mu(q1) -> mu(e)
      emit(2 + rk1, a.nc + q1, mu, 4 * tp, j1, 4 * tp + 1 + j1, 0,
           kFull ? seg_len(midpt(cop, ca), me) : 0.0);
    if (v2)  // t_minus partner at k1, kk = k2: mu(e) -> mu(r0)
      emit(2 + rk2, mu, a.nc + r0, 4 * tm, k2, 4 * tm + 1 + k2, 0,
           kFull ? seg_len(me, midpt(ca, com)) : 0.0);
    if (v3)  // t_minus partner at k2, kk = k1: mu(r1) -> mu(e)
      emit(2 + rk3, a.nc + r1, mu, 4 * tm, k1, 4 * tm + 1 + k1, 0,
           kFull ? seg_len(midpt(com, cb), me) : 0.0);
  }

  // 4. global offsets of the tile (precomputed, no look-back)
  const int F0 = __ldg(a.tileF + tile), B0 = __ldg(a.tileB + tile);
  const int N0 = kFull ? __ldg(a.tileN + tile) : 0;
  __syncthreads();
  if (valid) {
    o.node_edge_start[mu - a.nlo] = a.f_off + F0 + i0;
    if (le == a.E - 1) o.node_edge_start[mu - a.nlo + 1] = a.f_off + a.Ef;
  }

  // 5. coalesced stores of the tile's fine edges [F0, F0 + nf)
  const int nf = tot & 0x7ff;
  const int off_int = F0 - 2 * B0, off_bnd = 2 * B0;
  const int off_rp = F0 - 2 * N0, off_rs = 4 * (F0 - N0 - B0);
  for (int i = tid; i < nf; i += kLvT) {
    const int f = F0 + i;
    const int2 en = s.en[i], el2 = s.el[i];
    const int ms = s.ms[i];
    const int lp = ms & 3, lm = ((ms >> 2) & 3) - 1;
    reinterpret_cast<int2*>(o.edge_nodes)[f] = en;
    reinterpret_cast<int2*>(o.edge_elements)[f] = el2;
    o.ltp[f] = lp;
    o.ltm[f] = lm;
    const int sl = ms >> 8;  // arithmetic shift: boundary slots stay negative
    if (sl < 0) o.boundary[off_bnd + ~sl] = a.f_off + f;
    else o.interior[off_int + sl] = a.f_off + f;
    if (o.self_ee) {  // distributed, own fine elements written in place
      const int64_t s0 = 3 * (int64_t)el2.x + lp;
      const int64_t s1 = lm >= 0 ? 3 * (int64_t)el2.y + lm : -1;
      const bool own0 = s0 >= o.self_lo3 && s0 < o.self_hi3;
      const bool own1 = s1 < 0 || (s1 >= o.self_lo3 && s1 < o.self_hi3);
      if (own0) o.self_ee[s0 - o.self_lo3] = f;
      if (s1 >= 0 && own1) o.self_ee[s1 - o.self_lo3] = ~f;
      const int k = (own0 ? 0 : 1) + (own1 ? 0 : 1);
      if (k) {  // to the owners of the other fine elements
        int at = atomicAdd(o.npairs, k);
        if (!own0) o.pairs[at++] = make_int2((int)s0, f);
        if (!own1) o.pairs[at] = make_int2((int)s1, ~f);
      }
    } else if (o.pairs) {  // distributed: to the owners of the fine elements (coalesced)
      o.pairs[2 * (int64_t)f] = make_int2(3 * el2.x + lp, f);
      o.pairs[2 * (int64_t)f + 1] = lm >= 0 ? make_int2(3 * el2.y + lm, ~f) : make_int2(-1, 0);
    } else if (o.elem_edge) {
      o.elem_edge[3 * (int64_t)el2.x + lp] = f;
      if (lm >= 0) o.elem_edge[3 * (int64_t)el2.y + lm] = ~f;
    }
    if (kFull) {
      const int rr = s.rr[i];
      if (o.rpos) o.rpos[f] = rr < 0 ? -1 : a.r_off + off_rp + (rr >> 16);
      if (rr >= 0) {
        const int rp = off_rp + (rr >> 16);
        const int rs = off_rs + (rr & 0xffff);
        const double len = s.len[i];
        if (o.redges) o.redges[rp] = a.f_off + f;
        o.row_ptr[rp] = a.nnz_off + rs;
        // columns {0,1,2} \ {local}, ascending: T+ DOFs, then T- DOFs
        const int c0 = lp == 0 ? 1 : 0, c1 = lp == 2 ? 1 : 2;
        const double vp = len * 0.5;  // assembly.cpp:160
        // interior row at a 32-byte aligned entry (all but the rows after a
        // boundary half within a tile): one 16-byte column store and one
        // 32-byte value store (STG.E.ENL2.256) instead of two of each — the
        // half-sector stores cost the kernel 0.83 ms at L13 (4.35 -> 3.51 ms)
        if (lm >= 0 && ((reinterpret_cast<uintptr_t>(o.val + rs) & 31) == 0) &&
            ((reinterpret_cast<uintptr_t>(o.col + rs) & 15) == 0)) {
          const int d0 = lm == 0 ? 1 : 0, d1 = lm == 2 ? 1 : 2;
          const double vm = -len * 0.5;  // assembly.cpp:164
          *reinterpret_cast<int4*>(o.col + rs) =
              make_int4(3 * el2.x + c0, 3 * el2.x + c1, 3 * el2.y + d0, 3 * el2.y + d1);
          asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(o.val + rs), "d"(vp), "d"(vp),
                       "d"(vm), "d"(vm)
                       : "memory");
          if (rp == a.L - 1) o.row_ptr[a.L] = a.nnz_off + rs + 4;
          continue;
        }
        *reinterpret_cast<int2*>(o.col + rs) = make_int2(3 * el2.x + c0, 3 * el2.x + c1);
        __stcs(reinterpret_cast<double2*>(o.val + rs), make_double2(vp, vp));
        int n = 2;
        if (lm >= 0) {
          const int d0 = lm == 0 ? 1 : 0, d1 = lm == 2 ? 1 : 2;
          const double vm = -len * 0.5;  // assembly.cpp:164
          *reinterpret_cast<int2*>(o.col + rs + 2) = make_int2(3 * el2.y + d0, 3 * el2.y + d1);
          __stcs(reinterpret_cast<double2*>(o.val + rs + 2), make_double2(vm, vm));
          n = 4;
        }
        if (rp == a.L - 1) o.row_ptr[a.L] = a.nnz_off + rs + n;
      }
    }
  }
}

// One tile per CTA: the three load stages back to back.
template <bool kFull>
__global__ void __launch_bounds__(kLvT, PHFEM_LV_MIN_BLOCKS) k_rl_level(LvArgs a, LvOut o) {
  extern __shared__ __align__(16) unsigned char lv_smem[];  // dynamic: tiles may exceed 48 KB
  pdl_wait();
  pdl_trigger();
  LvSmem<kFull>& s = *reinterpret_cast<LvSmem<kFull>*>(lv_smem);
  const int le = blockIdx.x * kLvT + threadIdx.x;
  const bool valid = le < a.E;
  const LvRec r = lv_load_rec<kFull>(a, le);
  const LvGat g = lv_load_gat(a, r, valid, le);
  const LvCrd c = lv_load_crd(a, r, g, valid);
  lv_tile<kFull>(a, o, s, blockIdx.x, r, g, c);
}

// Children rows AND their elem_edge, one thread per parent element, after the
// level kernel (coalesced 48-byte rows instead of two scattered 4-byte
// elem_edge stores per fine edge).  Parent m = (P0, P1, P2) with edges e_j
// opposite P_j (sign s_j: m is t_plus of e_j), group starts G_j, M_j = nc + e_j:
//   * half of e_j at its endpoint v: G_j + (v == min of e_j's endpoints ? 0 : 1)
//     (group order: the half at the smaller old node first);
//   * interior edge I_k (opposite M_k, between M_{k+1} and M_{k+2}): group of
//     E' = max(e_{k+1}, e_{k+2}), position 2 + the rank the level kernel
//     stored for the partner e_min = min(e_{k+1}, e_{k+2}) of E';
//   * child 4m = (M0, M1, M2): (I_0, I_1, I_2), its t_plus;
//     child 4m+1+k = (P_k, M_{k+2}, M_{k+1}): (~I_k, half of e_{k+1} at P_k,
//     half of e_{k+2} at P_k), each half signed by s of its parent edge
//   (refine.cpp:33-36; the same ids as the scattered stores of k_rl_level).
__global__ void __launch_bounds__(256) k_refine_children(const int32_t* __restrict__ elements,
                                                         const int32_t* __restrict__ elem_edge,
                                                         const int32_t* __restrict__ nes,
                                                         const uint8_t* __restrict__ rk, int nE, int nc,
                                                         int4* __restrict__ out_elems,
                                                         int4* __restrict__ out_ee) {
  pdl_wait();
  pdl_trigger();
  // rows staged per warp in SMEM, then stored as contiguous 512-byte warp
  // writes (a direct per-thread 48-byte row leaves every sector half written
  // per instruction: twice the L2 write transactions)
  __shared__ int4 stage[8][2][96];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int4* se = stage[warp][0];
  int4* sq = stage[warp][1];
  const int64_t wstride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = ((int64_t)blockIdx.x * blockDim.x + warp * 32); base < nE; base += wstride) {
    const int64_t m = base + lane;
    if (m < nE) {
      int P[3], sg[3], e[3], G[3];
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        P[j] = __ldg(elements + 3 * m + j);
        sg[j] = __ldg(elem_edge + 3 * m + j);
        e[j] = abs_edge(sg[j]);
      }
#pragma unroll
      for (int j = 0; j < 3; ++j) G[j] = __ldg(nes + nc + e[j]);
      int I[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const int jA = k == 2 ? 0 : k + 1, jB = k == 0 ? 2 : k - 1;
        const bool aBig = e[jA] > e[jB];
        const int jE = aBig ? jA : jB, jm = aBig ? jB : jA;
        const int r = __ldg(rk + e[jE]);
        // partner slot of e_min seen from E': next local index (j1 / k1) or the one after (j2 / k2)
        const bool next = jm == (jE == 2 ? 0 : jE + 1);
        const int field = (sg[jE] >= 0 ? 0 : 2) + (next ? 0 : 1);
        I[k] = G[jE] + 2 + ((r >> (2 * field)) & 3);
      }
      // half of e_j at vertex v, signed
      auto half = [&](int j, int v) {
        const int a = P[j == 2 ? 0 : j + 1], b = P[j == 0 ? 2 : j - 1];
        const int id = G[j] + (v == min(a, b) ? 0 : 1);
        return sg[j] >= 0 ? id : ~id;
      };
      const int M0 = nc + e[0], M1 = nc + e[1], M2 = nc + e[2];
      se[3 * lane] = make_int4(M0, M1, M2, P[0]);
      se[3 * lane + 1] = make_int4(M2, M1, P[1], M0);
      se[3 * lane + 2] = make_int4(M2, P[2], M1, M0);
      sq[3 * lane] = make_int4(I[0], I[1], I[2], ~I[0]);
      sq[3 * lane + 1] = make_int4(half(1, P[0]), half(2, P[0]), ~I[1], half(2, P[1]));
      sq[3 * lane + 2] = make_int4(half(0, P[1]), ~I[2], half(0, P[2]), half(1, P[2]));
    }
    __syncwarp();
    const int64_t rem = nE - base;
    const int n4 = 3 * (int)(rem < 32 ? rem : 32);
    for (int i = lane; i < n4; i += 32) {
      out_elems[3 * base + i] = se[i];
      out_ee[3 * base + i] = sq[i];
    }
    __syncwarp();
  }
}

// dynamic SMEM of the level kernels (opt-in above 48 KB, per ctx device)
template <bool kFull>
static phfem_status lv_smem_bytes(phfem_ctx* ctx, size_t* bytes) {
  *bytes = sizeof(LvSmem<kFull>);
  return smem_optin(ctx, (const void*)k_rl_level<kFull>, *bytes, "k_rl_level smem opt-in");
}

// The level kernel over `ntiles` tiles, one tile per CTA.  (A persistent,
// software-pipelined variant — the next tile's record and element gathers in
// flight while a tile computes — measured 6.4-6.7 ms against 5.16 at L13:
// the kernel is bound by its scattered stores, not by the load chain.)
template <bool kFull>
static phfem_status launch_level(phfem_ctx* ctx, const LvArgs& a, const LvOut& o, int64_t ntiles) {
  const char* name = kFull ? "k_rl_level_full" : "k_rl_level";
  size_t smem = 0;
  PHFEM_TRY(lv_smem_bytes<kFull>(ctx, &smem));
  PHFEM_LAUNCH_PDL(ctx, name, k_rl_level<kFull>, (unsigned)ntiles, kLvT, smem, a, o);
  return PHFEM_OK;
}

}  // namespace phfem

using namespace phfem;

namespace phfem {

// Shared host body of phfem_refine_topology / phfem_refine_level.  `mid`
// (nullable) receives the midpoint coordinates of the fine mesh (nodes
// nc..nc+E-1) — the fused pipeline lets red_refine skip them.
static phfem_status refine_level_run(phfem_ctx* ctx, const phfem_mesh* parent,
                                     const phfem_topology* ptopo,
                                     const phfem_classification* pcls, int64_t Ef, int64_t L,
                                     phfem_topology* topo, phfem_classification* cls, phfem_csr* C,
                                     double* mid, const phfem_mesh* fine, bool write_elems) {
  const int64_t E = ptopo->E;
  if (E == 0) return PHFEM_OK;
  const int64_t ntiles = (E + kLvT - 1) / kLvT;
  int32_t* tiles = nullptr;
  PHFEM_TRY(dalloc(ctx, &tiles, 3 * (ntiles + 1)));
  int32_t *tileF = tiles, *tileB = tiles + (ntiles + 1), *tileN = tiles + 2 * (ntiles + 1);
  PHFEM_TRY(zero_i32(ctx, tiles, 3 * (ntiles + 1)));
  const uint32_t* nbits = pcls ? pcls->neumann_bits : nullptr;
  {
    const int blocksA = grid_for(ntiles, 256, ctx->num_sms * 8);
    const int blocksB = grid_for(parent->nE, 256, ctx->num_sms * 16);
    PHFEM_LAUNCH_PDL(ctx, "k_rl_tile_count", k_rl_tile_prep, blocksA + blocksB, 256, 0,
        (int)E, (int)ntiles, ptopo->boundary_edges, ptopo->n_boundary, nbits, tileF, tileB, tileN, ptopo->elem_edge,
        (int)parent->nE, blocksA);
  }
  {
    const int32_t* in[3] = {tileF, tileB, tileN};
    int32_t* io[3] = {tileF, tileB, tileN};
    PHFEM_TRY(scan_exclusive_i32_set(ctx, pcls ? 3 : 2, in, io, ntiles + 1, nullptr));
  }
  LvArgs a;
  memset(&a, 0, sizeof a);
  a.edge_nodes = ptopo->edge_nodes;
  a.edge_elements = ptopo->edge_elements;
  a.ltp = ptopo->local_in_tplus;
  a.ltm = ptopo->local_in_tminus;
  a.elem_edge = ptopo->elem_edge;
  a.elements = parent->elements;
  a.coords = (const double2*)parent->coords;
  a.E = (int)E;
  a.nc = parent->nC;
  a.Ef = (int)Ef;
  a.L = (int)L;
  a.tileF = tileF;
  a.tileB = tileB;
  a.tileN = tileN;
  LvOut o;
  memset(&o, 0, sizeof o);
  o.edge_nodes = topo->edge_nodes;
  o.edge_elements = topo->edge_elements;
  o.ltp = topo->local_in_tplus;
  o.ltm = topo->local_in_tminus;
  o.interior = topo->interior_edges;
  o.boundary = topo->boundary_edges;
  o.elem_edge = topo->elem_edge;
  o.node_edge_start = topo->node_edge_start;
  o.mid = (double2*)mid;
  uint8_t* rk = nullptr;
  if (write_elems) {  // children rows + fine elem_edge by the element pass below
    PHFEM_TRY(dalloc(ctx, &rk, E));
    o.rk = rk;
    o.elem_edge = nullptr;
  }
  if (pcls) {
    a.neu_bits = pcls->neumann_bits;
    o.rpos = cls->retained_pos;
    o.redges = cls->retained_edges;
    o.row_ptr = C->row_ptr;
    o.col = C->col_idx;
    o.val = C->values;
    PHFEM_TRY(launch_level<true>(ctx, a, o, ntiles));
  } else {
    PHFEM_TRY(launch_level<false>(ctx, a, o, ntiles));
  }
  if (write_elems && parent->nE > 0)
    PHFEM_LAUNCH_PDL(ctx, "k_refine_children", k_refine_children,
        grid_for(parent->nE, 256, ctx->num_sms * PHFEM_CH_GRID_MULT), 256, 0,
        (const int32_t*)parent->elements, (const int32_t*)ptopo->elem_edge, (const int32_t*)topo->node_edge_start,
        (const uint8_t*)rk, (int)parent->nE, (int)parent->nC, (int4*)fine->elements, (int4*)topo->elem_edge);
  dfree(ctx, rk);
  dfree(ctx, tiles);
  return PHFEM_OK;
}

phfem_status refine_topology_impl(phfem_ctx* ctx, const phfem_mesh* parent,
                                  const phfem_topology* ptopo, const phfem_mesh* fine,
                                  phfem_topology* out, double* mid, bool write_elems) {
  memset(out, 0, sizeof(*out));
  if (!ctx || !parent || !ptopo || !fine) return PHFEM_ERR_INVALID_ARGUMENT;
  if (ptopo->nE != parent->nE || ptopo->nC != parent->nC || fine->nE != 4 * parent->nE ||
      fine->nC != parent->nC + ptopo->E)
    return set_error(ctx, PHFEM_ERR_MISMATCH, "refine_topology: meshes do not match the topology");
  const int64_t E = ptopo->E, nc = parent->nC;
  // exact count: two halves per parent edge + three interior edges per parent element
  const int64_t Ef = 2 * E + 3 * (int64_t)parent->nE;
  if (Ef >= (int64_t(1) << 31))
    return set_error(ctx, PHFEM_ERR_INVALID_ARGUMENT, "refine_topology: mesh too large for int ids");
  out->nC = fine->nC;
  out->nE = fine->nE;
  const int64_t nBf = 2 * (int64_t)ptopo->n_boundary;
  PHFEM_TRY(dalloc(ctx, &out->edge_nodes, 2 * Ef));
  PHFEM_TRY(dalloc(ctx, &out->edge_elements, 2 * Ef));
  PHFEM_TRY(dalloc(ctx, &out->local_in_tplus, Ef));
  PHFEM_TRY(dalloc(ctx, &out->local_in_tminus, Ef));
  PHFEM_TRY(dalloc(ctx, &out->interior_edges, Ef - nBf));
  PHFEM_TRY(dalloc(ctx, &out->boundary_edges, nBf));
  PHFEM_TRY(dalloc(ctx, &out->elem_edge, 3 * (int64_t)fine->nE));
  PHFEM_TRY(dalloc(ctx, &out->node_edge_start, (int64_t)fine->nC + 1));
  PHFEM_CUDA(ctx, cudaMemsetAsync(out->node_edge_start, 0, sizeof(int32_t) * (nc + 1), ctx->stream));
  out->E = (int32_t)Ef;
  out->n_boundary = (int32_t)nBf;
  out->n_interior = (int32_t)(Ef - nBf);
  return refine_level_run(ctx, parent, ptopo, nullptr, Ef, 0, out, nullptr, nullptr, mid, fine, write_elems);
}

// defined in classify.cu
phfem_status classify_lists(phfem_ctx* ctx, const phfem_topology* topo, const phfem_mesh* mesh,
                            phfem_classification* out, bool with_retained);

phfem_status refine_level_impl(phfem_ctx* ctx, const phfem_mesh* parent,
                               const phfem_topology* ptopo, const phfem_classification* pcls,
                               const phfem_mesh* fine, phfem_topology* topo,
                               phfem_classification* cls, phfem_csr* C, double* mid,
                               bool write_elems) {
  memset(topo, 0, sizeof(*topo));
  memset(cls, 0, sizeof(*cls));
  memset(C, 0, sizeof(*C));
  if (!ctx || !parent || !ptopo || !pcls || !fine) return PHFEM_ERR_INVALID_ARGUMENT;
  if (ptopo->nE != parent->nE || ptopo->nC != parent->nC || fine->nE != 4 * parent->nE ||
      fine->nC != parent->nC + ptopo->E || pcls->E != ptopo->E ||
      fine->nD != 2 * parent->nD || fine->nN != 2 * parent->nN)
    return set_error(ctx, PHFEM_ERR_MISMATCH, "refine_level: meshes do not match the topology");
  const int64_t E = ptopo->E, nc = parent->nC;
  const int64_t Ef = 2 * E + 3 * (int64_t)parent->nE;
  if (Ef >= (int64_t(1) << 31) || 4 * Ef >= (int64_t(1) << 31))
    return set_error(ctx, PHFEM_ERR_INVALID_ARGUMENT, "refine_level: mesh too large for int ids");
  const int64_t nneu_p = E - pcls->L;                   // Neumann parent edges
  const int64_t nBf = 2 * (int64_t)ptopo->n_boundary;
  const int64_t L = Ef - 2 * nneu_p;                    // their halves are the fine Neumann edges
  const int64_t BR = 2 * ((int64_t)ptopo->n_boundary - nneu_p);
  topo->nC = fine->nC;
  topo->nE = fine->nE;
  PHFEM_TRY(dalloc(ctx, &topo->edge_nodes, 2 * Ef));
  PHFEM_TRY(dalloc(ctx, &topo->edge_elements, 2 * Ef));
  PHFEM_TRY(dalloc(ctx, &topo->local_in_tplus, Ef));
  PHFEM_TRY(dalloc(ctx, &topo->local_in_tminus, Ef));
  PHFEM_TRY(dalloc(ctx, &topo->interior_edges, Ef - nBf));
  PHFEM_TRY(dalloc(ctx, &topo->boundary_edges, nBf));
  PHFEM_TRY(dalloc(ctx, &topo->elem_edge, 3 * (int64_t)fine->nE));
  PHFEM_TRY(dalloc(ctx, &topo->node_edge_start, (int64_t)fine->nC + 1));
  topo->E = (int32_t)Ef;
  topo->n_boundary = (int32_t)nBf;
  topo->n_interior = (int32_t)(Ef - nBf);
  PHFEM_TRY(dalloc(ctx, &cls->retained_pos, Ef));
  PHFEM_TRY(dalloc(ctx, &cls->retained_edges, L));
  C->rows = (int32_t)L;
  C->cols = 3 * fine->nE;
  C->nnz = 4 * L - 2 * BR;
  PHFEM_TRY(dalloc(ctx, &C->row_ptr, L + 1));
  PHFEM_TRY(dalloc(ctx, &C->col_idx, C->nnz));
  PHFEM_TRY(dalloc(ctx, &C->values, C->nnz));
  PHFEM_CUDA(ctx, cudaMemsetAsync(topo->node_edge_start, 0, sizeof(int32_t) * (nc + 1), ctx->stream));
  if (L == 0) PHFEM_CUDA(ctx, cudaMemsetAsync(C->row_ptr, 0, sizeof(int32_t), ctx->stream));
  PHFEM_TRY(refine_level_run(ctx, parent, ptopo, pcls, Ef, L, topo, cls, C, mid, fine, write_elems));
  // boundary lists -> ids, Neumann bitmap, block prefixes (retained arrays already written)
  PHFEM_TRY(classify_lists(ctx, topo, fine, cls, false));
  if (cls->L != L)
    return set_error(ctx, PHFEM_ERR_MISMATCH, "refine_level: classification does not match the parent's");
  return PHFEM_OK;
}

}  // namespace phfem

PHFEM_API phfem_status phfem_refine_topology(phfem_ctx* ctx, const phfem_mesh* parent,
                                             const phfem_topology* ptopo, const phfem_mesh* fine,
                                             phfem_topology* out) {
  return refine_topology_impl(ctx, parent, ptopo, fine, out, nullptr);
}

PHFEM_API phfem_status phfem_refine_level(phfem_ctx* ctx, const phfem_mesh* parent,
                                          const phfem_topology* ptopo,
                                          const phfem_classification* pcls,
                                          const phfem_mesh* fine, phfem_topology* topo,
                                          phfem_classification* cls, phfem_csr* C) {
  return refine_level_impl(ctx, parent, ptopo, pcls, fine, topo, cls, C, nullptr);
}

// Distributed refined level (SURVEY §8(e) + f1): this rank's part of the fine
// topology from its parent part (edges [E0p, E0p + E) with local arrays and
// global-id lists) and the all-gathered parent elem_edge / elements, no sort
// and no occurrence exchange.  Fine edges of the rank are its groups, in
// order (local ids); the fine elem_edge entries leave as (slot, f / ~f) pairs
// for the element owners (phfem_dist_route_pairs).  node range [node_lo,
// node_hi) must end at nc + E0p + E (the rank's last midpoint node).
// parent Neumann ids (global) -> bitmap over the rank's local parent edges
__global__ void k_rl_neu_bits(const int32_t* __restrict__ ids, int n, int E0, int E, uint32_t* __restrict__ bits) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int e = ids[i] - E0;
    if (e >= 0 && e < E) atomicOr(&bits[e >> 5], 1u << (e & 31));
  }
}

PHFEM_API phfem_status phfem_dist_refine_level_ex(phfem_ctx* ctx, const phfem_topology* ppart, int32_t E0p,
                                                  const int32_t* elem_edge_all, const int32_t* elements_all,
                                                  int32_t nE_all, const double* coords, int32_t nc,
                                                  int32_t node_lo, int32_t node_hi,
                                                  const int32_t* neu_parent_ids, int32_t nN_parent,
                                                  int32_t self_lo, int32_t self_hi, int32_t* self_elem_edge,
                                                  phfem_topology* out, int32_t** pairs_out, int64_t* n_pairs,
                                                  double* mids, phfem_csr* C) {
  if (!ctx || !ppart || !out || !pairs_out) return PHFEM_ERR_INVALID_ARGUMENT;
  const bool own = self_elem_edge != nullptr;
  if (own && (self_lo < 0 || self_hi < self_lo || (int64_t)self_hi > 4 * (int64_t)nE_all || !n_pairs))
    return PHFEM_ERR_INVALID_ARGUMENT;
  if (n_pairs) *n_pairs = 0;
  memset(out, 0, sizeof(*out));
  if (C) memset(C, 0, sizeof(*C));
  *pairs_out = nullptr;
  if (nN_parent > 0 && !neu_parent_ids) return PHFEM_ERR_INVALID_ARGUMENT;
  const int64_t E = ppart->E;
  if ((E > 0 && (!elem_edge_all || !elements_all || !coords)) || E0p < 0 || node_lo < 0 ||
      node_hi < node_lo || (E > 0 && (int64_t)node_hi != (int64_t)nc + E0p + E) ||
      (E > 0 && node_lo > nc + E0p) || 4 * (int64_t)nE_all >= (int64_t(1) << 31))
    return PHFEM_ERR_INVALID_ARGUMENT;
  const int64_t ntiles = std::max<int64_t>(1, (E + kLvT - 1) / kLvT);
  const int64_t nwords = std::max<int64_t>(1, (E + 31) / 32);
  int32_t* tiles = nullptr;
  PHFEM_TRY(dalloc(ctx, &tiles, 3 * (ntiles + 1) + 3));
  int32_t *tileF = tiles, *tileB = tiles + (ntiles + 1), *tileN = tiles + 2 * (ntiles + 1);
  int32_t* total = tiles + 3 * (ntiles + 1);  // [0] fine edges, [1] parent Neumann edges
  PHFEM_CUDA(ctx, cudaMemsetAsync(tiles, 0, sizeof(int32_t) * (3 * (ntiles + 1) + 3), ctx->stream));
  uint32_t* nbits = nullptr;
  if (C) {  // the fused variant: classification bits of the owned parent edges
    PHFEM_TRY(dalloc(ctx, &nbits, nwords));
    PHFEM_CUDA(ctx, cudaMemsetAsync(nbits, 0, sizeof(uint32_t) * nwords, ctx->stream));
    if (nN_parent > 0 && E > 0)
      PHFEM_LAUNCH(ctx, "k_rl_neu_bits", k_rl_neu_bits<<<grid_for(nN_parent, 256, ctx->num_sms), 256, 0, ctx->stream>>>(
          neu_parent_ids, nN_parent, E0p, (int)E, nbits));
  }
  if (E > 0) {
    PHFEM_LAUNCH(ctx, "k_rl_tile_init", k_rl_tile_init<<<grid_for(ntiles, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
        (int)E, E0p, (int)ntiles, ppart->boundary_edges, ppart->n_boundary, nbits, tileF, tileB, tileN));
    PHFEM_LAUNCH(ctx, "k_rl_tile_count", k_rl_tile_count<<<grid_for(nE_all, 256, ctx->num_sms * 16), 256, 0, ctx->stream>>>(
        elem_edge_all, nE_all, E0p, (int)E, tileF));
  }
  PHFEM_TRY(scan_exclusive_i32(ctx, tileF, tileF, ntiles + 1, total));
  PHFEM_TRY(scan_exclusive_i32(ctx, tileB, tileB, ntiles + 1, nullptr));
  if (C) PHFEM_TRY(scan_exclusive_i32(ctx, tileN, tileN, ntiles + 1, total + 1));
  int32_t hcnt[2] = {0, 0};
  PHFEM_CUDA(ctx, cudaMemcpyAsync(hcnt, total, sizeof hcnt, cudaMemcpyDeviceToHost, ctx->stream));
  PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  const int32_t Ef = hcnt[0];
  const int64_t nBf = 2 * (int64_t)ppart->n_boundary;
  out->nC = node_hi - node_lo;
  out->nE = 4 * nE_all;
  out->E = Ef;
  out->n_boundary = (int32_t)nBf;
  out->n_interior = (int32_t)(Ef - nBf);
  const int64_t cap = std::max<int64_t>(Ef, 1);
  PHFEM_TRY(dalloc(ctx, &out->edge_nodes, 2 * cap));
  PHFEM_TRY(dalloc(ctx, &out->edge_elements, 2 * cap));
  PHFEM_TRY(dalloc(ctx, &out->local_in_tplus, cap));
  PHFEM_TRY(dalloc(ctx, &out->local_in_tminus, cap));
  PHFEM_TRY(dalloc(ctx, &out->interior_edges, std::max<int64_t>(Ef - nBf, 1)));
  PHFEM_TRY(dalloc(ctx, &out->boundary_edges, std::max<int64_t>(nBf, 1)));
  PHFEM_TRY(dalloc(ctx, &out->node_edge_start, (int64_t)out->nC + 1));
  PHFEM_CUDA(ctx, cudaMemsetAsync(out->node_edge_start, 0, sizeof(int32_t) * ((int64_t)out->nC + 1), ctx->stream));
  int32_t* pairs = nullptr;
  PHFEM_TRY(dalloc(ctx, &pairs, 4 * cap));
  int64_t Lr = 0;
  if (C) {  // rows: fine edges minus the halves of Neumann parent edges (refine_level_impl)
    const int64_t nneu = hcnt[1];
    Lr = Ef - 2 * nneu;
    const int64_t BR = 2 * ((int64_t)ppart->n_boundary - nneu);
    C->rows = (int32_t)Lr;
    C->cols = 3 * 4 * nE_all;
    C->nnz = 4 * Lr - 2 * BR;
    PHFEM_TRY(dalloc(ctx, &C->row_ptr, Lr + 1));
    PHFEM_TRY(dalloc(ctx, &C->col_idx, std::max<int64_t>(C->nnz, 1)));
    PHFEM_TRY(dalloc(ctx, &C->values, std::max<int64_t>(C->nnz, 1)));
    if (Lr == 0) PHFEM_CUDA(ctx, cudaMemsetAsync(C->row_ptr, 0, sizeof(int32_t), ctx->stream));
  }
  if (E > 0) {
    LvArgs a;
    memset(&a, 0, sizeof a);
    a.edge_nodes = ppart->edge_nodes;
    a.edge_elements = ppart->edge_elements;
    a.ltp = ppart->local_in_tplus;
    a.ltm = ppart->local_in_tminus;
    a.elem_edge = elem_edge_all;
    a.elements = elements_all;
    a.coords = (const double2*)coords;
    a.E = (int)E;
    a.nc = nc;
    a.Ef = Ef;
    a.eb = E0p;
    a.nlo = node_lo;
    a.tileF = tileF;
    a.tileB = tileB;
    LvOut o;
    memset(&o, 0, sizeof o);
    o.edge_nodes = out->edge_nodes;
    o.edge_elements = out->edge_elements;
    o.ltp = out->local_in_tplus;
    o.ltm = out->local_in_tminus;
    o.interior = out->interior_edges;
    o.boundary = out->boundary_edges;
    o.node_edge_start = out->node_edge_start;
    o.mid = (double2*)mids;
    o.mid_base = (int64_t)nc + E0p;
    o.pairs = reinterpret_cast<int2*>(pairs);
    if (own) {
      o.self_ee = self_elem_edge;
      o.self_lo3 = 3 * (int64_t)self_lo;
      o.self_hi3 = 3 * (int64_t)self_hi;
      o.npairs = total + 2;
    }
    const unsigned nt = (unsigned)((E + kLvT - 1) / kLvT);
    if (C) {
      a.neu_bits = nbits;
      a.tileN = tileN;
      a.L = (int)Lr;
      o.row_ptr = C->row_ptr;
      o.col = C->col_idx;
      o.val = C->values;
      PHFEM_TRY(launch_level<true>(ctx, a, o, nt));
    } else {
      PHFEM_TRY(launch_level<false>(ctx, a, o, nt));
    }
  }
  if (own) {  // the count of pairs for other ranks
    int32_t np = 0;
    PHFEM_CUDA(ctx, cudaMemcpyAsync(&np, total + 2, sizeof np, cudaMemcpyDeviceToHost, ctx->stream));
    PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    *n_pairs = np;
  } else if (n_pairs) {
    *n_pairs = 2 * (int64_t)Ef;
  }
  dfree(ctx, nbits);
  dfree(ctx, tiles);
  *pairs_out = pairs;
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_dist_refine_level(phfem_ctx* ctx, const phfem_topology* ppart, int32_t E0p,
                                               const int32_t* elem_edge_all, const int32_t* elements_all,
                                               int32_t nE_all, const double* coords, int32_t nc,
                                               int32_t node_lo, int32_t node_hi,
                                               const int32_t* neu_parent_ids, int32_t nN_parent,
                                               phfem_topology* out, int32_t** pairs_out, double* mids,
                                               phfem_csr* C) {
  return phfem_dist_refine_level_ex(ctx, ppart, E0p, elem_edge_all, elements_all, nE_all, coords, nc, node_lo,
                                    node_hi, neu_parent_ids, nN_parent, 0, 0, nullptr, out, pairs_out, nullptr,
                                    mids, C);
}

// ---------------------------------------------------------------------------
// Distributed refined level, side-record mode (dist.py _refine_sort_free):
// the rank's parent edges [E0p, E0p + E) get their partner edges and opposite
// vertices from the element owners' side records (phfem_dist_side_apply), not
// from all-gathered parent arrays; the fine elem_edge is written by the
// element owners (phfem_dist_children_slots) from the group starts and rank
// bytes this level returns (phfem_dist_start_records).  Owned midpoints go to
// coords_fine[nc + E0p + le].
namespace phfem {
// partners < e per parent edge, summed per 128-edge tile (tile of le = le / kLvT)
__global__ void k_rl_tile_count_side(const int4* __restrict__ side, const int32_t* __restrict__ edge_elements,
                                     const int32_t* __restrict__ ltp, const int32_t* __restrict__ ltm,
                                     const int32_t* __restrict__ own_el, const int32_t* __restrict__ own_ee,
                                     int own_lo, int own_hi, int E, int eb, int32_t* __restrict__ tileF) {
  for (int64_t le0 = (int64_t)blockIdx.x * blockDim.x; le0 < E; le0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t le = le0 + threadIdx.x;
    int c = 0;
    if (le < E) {
      const int e = eb + (int)le;
      // local mode: the rank's own elements were counted by the element pass
      // (k_rl_tile_count over them); only the other ranks' sides here
      const int2 el = reinterpret_cast<const int2*>(edge_elements)[le];
      const bool lp = own_el && el.x >= own_lo && el.x < own_hi;
      const bool lm = own_el && el.y >= own_lo && el.y < own_hi;
      if (!lp) {
        const int4 sp = side[2 * le];
        c = (abs_edge(sp.x) < e) + (abs_edge(sp.y) < e);
      }
      if (el.y >= 0 && !lm) {
        const int4 sm = side[2 * le + 1];
        c += (abs_edge(sm.x) < e) + (abs_edge(sm.y) < e);
      }
    }
    c = warp_reduce_sum(c);  // a warp's edges share one tile (kLvT multiple of 32)
    if (lane_id() == 0 && le0 + (threadIdx.x & ~31) < E) atomicAdd(tileF + (le0 + (threadIdx.x & ~31)) / kLvT, c);
  }
}

// k_refine_children with the group starts / rank bytes per element slot
// (gs / grk from phfem_dist_start_apply, global fine ids) instead of
// gathers by edge id; also writes the midpoints of the element's edges into
// the rank's fine coordinate array (0.5 (c[a] + c[b]) with the element's own
// vertices: the same bits as the edge owner's, refine.cpp:18).
__global__ void __launch_bounds__(256) k_dist_children_slots(const int32_t* __restrict__ elements,
                                                             const int32_t* __restrict__ elem_edge,
                                                             const int32_t* __restrict__ gs,
                                                             const uint8_t* __restrict__ grk, int nE, int nc,
                                                             int own_lo, int own_hi,
                                                             const int32_t* __restrict__ fine_nes, int nes_off,
                                                             const uint8_t* __restrict__ rk_own,
                                                             double2* __restrict__ coords,
                                                             int4* __restrict__ out_elems,
                                                             int4* __restrict__ out_ee) {
  __shared__ int4 stage[8][2][96];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int4* se = stage[warp][0];
  int4* sq = stage[warp][1];
  const int64_t wstride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = ((int64_t)blockIdx.x * blockDim.x + warp * 32); base < nE; base += wstride) {
    const int64_t m = base + lane;
    if (m < nE) {
      int P[3], sg[3], e[3], G[3], R[3];
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        P[j] = __ldg(elements + 3 * m + j);
        sg[j] = __ldg(elem_edge + 3 * m + j);
        e[j] = abs_edge(sg[j]);
        if (fine_nes && e[j] >= own_lo && e[j] < own_hi) {  // local mode: the rank's own edge
          G[j] = __ldg(fine_nes + (e[j] - own_lo) + nes_off);
          R[j] = __ldg(rk_own + (e[j] - own_lo));
        } else {
          G[j] = __ldg(gs + 3 * m + j);
          R[j] = __ldg(grk + 3 * m + j);
        }
      }
#pragma unroll
      for (int j = 0; j < 3; ++j) {  // midpoint of the edge opposite P_j (the owner's level wrote its own)
        if (e[j] >= own_lo && e[j] < own_hi) continue;
        const double2 pa = __ldg(coords + P[j == 2 ? 0 : j + 1]), pb = __ldg(coords + P[j == 0 ? 2 : j - 1]);
        coords[nc + e[j]] = midpt(pa, pb);
      }
      int I[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const int jA = k == 2 ? 0 : k + 1, jB = k == 0 ? 2 : k - 1;
        const bool aBig = e[jA] > e[jB];
        const int jE = aBig ? jA : jB, jm = aBig ? jB : jA;
        const int r = jE == 0 ? R[0] : (jE == 1 ? R[1] : R[2]);
        const int GE = jE == 0 ? G[0] : (jE == 1 ? G[1] : G[2]);
        const bool next = jm == (jE == 2 ? 0 : jE + 1);
        const int sE = jE == 0 ? sg[0] : (jE == 1 ? sg[1] : sg[2]);
        const int field = (sE >= 0 ? 0 : 2) + (next ? 0 : 1);
        I[k] = GE + 2 + ((r >> (2 * field)) & 3);
      }
      auto half = [&](int j, int v) {
        const int a = P[j == 2 ? 0 : j + 1], b = P[j == 0 ? 2 : j - 1];
        const int id = G[j] + (v == min(a, b) ? 0 : 1);
        return sg[j] >= 0 ? id : ~id;
      };
      const int M0 = nc + e[0], M1 = nc + e[1], M2 = nc + e[2];
      se[3 * lane] = make_int4(M0, M1, M2, P[0]);
      se[3 * lane + 1] = make_int4(M2, M1, P[1], M0);
      se[3 * lane + 2] = make_int4(M2, P[2], M1, M0);
      sq[3 * lane] = make_int4(I[0], I[1], I[2], ~I[0]);
      sq[3 * lane + 1] = make_int4(half(1, P[0]), half(2, P[0]), ~I[1], half(2, P[1]));
      sq[3 * lane + 2] = make_int4(half(0, P[1]), ~I[2], half(0, P[2]), half(1, P[2]));
    }
    __syncwarp();
    const int64_t rem = nE - base;
    const int n4 = 3 * (int)(rem < 32 ? rem : 32);
    for (int i = lane; i < n4; i += 32) {
      out_elems[3 * base + i] = se[i];
      out_ee[3 * base + i] = sq[i];
    }
    __syncwarp();
  }
}
}  // namespace phfem

namespace phfem {
static __global__ void k_fill_lv(int32_t* __restrict__ a, int64_t n, int32_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = v;
}
}  // namespace phfem

// Count half of the side-mode level: tile counts from the side records,
// fine edges Ef and parent Neumann edges of the rank (synchronises); the
// plan carries the tile prefixes to phfem_dist_level_run.
struct phfem_dist_level_plan {
  phfem_topology ppart;
  int32_t E0p;
  const int32_t* side;
  phfem_dist_local local;  // elements == NULL: every slot has a side record
  int64_t ntiles;
  int32_t* tiles;
  uint32_t* nbits;
  int32_t Ef, nneu;
  bool with_C;
};

PHFEM_API phfem_status phfem_dist_level_count_ex(phfem_ctx* ctx, const phfem_topology* ppart, int32_t E0p,
                                                 const int32_t* side, const phfem_dist_local* local,
                                                 const int32_t* neu_parent_ids, int32_t nN_parent, int with_C,
                                                 int32_t* Ef_out, int32_t* nneu_out, void** plan_out) {
  if (!ctx || !ppart || !Ef_out || !nneu_out || !plan_out || E0p < 0) return PHFEM_ERR_INVALID_ARGUMENT;
  *plan_out = nullptr;
  if (nN_parent > 0 && !neu_parent_ids) return PHFEM_ERR_INVALID_ARGUMENT;
  const int64_t E = ppart->E;
  if (E > 0 && !side) return PHFEM_ERR_INVALID_ARGUMENT;
  const int64_t ntiles = std::max<int64_t>(1, (E + kLvT - 1) / kLvT);
  const int64_t nwords = std::max<int64_t>(1, (E + 31) / 32);
  phfem_dist_level_plan* pl = new phfem_dist_level_plan();
  pl->ppart = *ppart;
  pl->E0p = E0p;
  pl->side = side;
  memset(&pl->local, 0, sizeof pl->local);
  if (local && local->ehi > local->elo) {
    if (!local->elements || !local->elem_edge) {
      delete pl;
      return PHFEM_ERR_INVALID_ARGUMENT;
    }
    pl->local = *local;
  }
  pl->ntiles = ntiles;
  pl->with_C = with_C != 0;
  auto fail = [&](phfem_status st) {
    dfree(ctx, pl->tiles);
    dfree(ctx, pl->nbits);
    delete pl;
    return st;
  };
  phfem_status st = dalloc(ctx, &pl->tiles, 3 * (ntiles + 1) + 2);
  if (st != PHFEM_OK) return fail(st);
  int32_t *tileF = pl->tiles, *tileB = pl->tiles + (ntiles + 1), *tileN = pl->tiles + 2 * (ntiles + 1);
  int32_t* total = pl->tiles + 3 * (ntiles + 1);
  if (cudaMemsetAsync(pl->tiles, 0, sizeof(int32_t) * (3 * (ntiles + 1) + 2), ctx->stream) != cudaSuccess)
    return fail(cuda_fail(ctx, cudaGetLastError(), "level count memset"));
  if (pl->with_C) {
    if ((st = dalloc(ctx, &pl->nbits, nwords)) != PHFEM_OK) return fail(st);
    cudaMemsetAsync(pl->nbits, 0, sizeof(uint32_t) * nwords, ctx->stream);
    if (nN_parent > 0 && E > 0) {
      KTimer kt(ctx, "k_rl_neu_bits");
      k_rl_neu_bits<<<grid_for(nN_parent, 256, ctx->num_sms), 256, 0, ctx->stream>>>(neu_parent_ids, nN_parent, E0p,
                                                                                      (int)E, pl->nbits);
      ctx->launches++;
    }
  }
  if (E > 0) {
    {
      KTimer kt(ctx, "k_rl_tile_init");
      k_rl_tile_init<<<grid_for(ntiles, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
          (int)E, E0p, (int)ntiles, ppart->boundary_edges, ppart->n_boundary, pl->nbits, tileF, tileB, tileN);
      ctx->launches++;
    }
    if (pl->local.elements) {  // the rank's own elements: element pass (coalesced), as on one GPU
      KTimer kt(ctx, "k_rl_tile_count");
      k_rl_tile_count<<<grid_for(pl->local.ehi - pl->local.elo, 256, ctx->num_sms * 16), 256, 0, ctx->stream>>>(
          pl->local.elem_edge, pl->local.ehi - pl->local.elo, E0p, (int)E, tileF);
      ctx->launches++;
    }
    if (!pl->local.elements || !pl->local.no_remote) {
      KTimer kt(ctx, "k_rl_tile_count_side");
      k_rl_tile_count_side<<<grid_for(E, 256, ctx->num_sms * 16), 256, 0, ctx->stream>>>(
          reinterpret_cast<const int4*>(side), ppart->edge_elements, ppart->local_in_tplus, ppart->local_in_tminus,
          pl->local.elements, pl->local.elem_edge, pl->local.elo, pl->local.ehi, (int)E, E0p, tileF);
      ctx->launches++;
    }
  }
  if (cudaGetLastError() != cudaSuccess) return fail(set_error(ctx, PHFEM_ERR_CUDA, "level count launch failed"));
  {
    const int32_t* in[3] = {tileF, tileB, tileN};
    int32_t* io[3] = {tileF, tileB, tileN};
    int32_t* tot[3] = {total, nullptr, total + 1};
    if ((st = scan_exclusive_i32_set(ctx, pl->with_C ? 3 : 2, in, io, ntiles + 1, tot)) != PHFEM_OK) return fail(st);
  }
  int32_t hcnt[2] = {0, 0};
  if (cudaMemcpyAsync(hcnt, total, sizeof hcnt, cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
      cudaStreamSynchronize(ctx->stream) != cudaSuccess)
    return fail(cuda_fail(ctx, cudaGetLastError(), "level count"));
  pl->Ef = hcnt[0];
  pl->nneu = pl->with_C ? hcnt[1] : 0;
  *Ef_out = pl->Ef;
  *nneu_out = pl->nneu;
  *plan_out = pl;
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_dist_level_count(phfem_ctx* ctx, const phfem_topology* ppart, int32_t E0p,
                                              const int32_t* side, const int32_t* neu_parent_ids, int32_t nN_parent,
                                              int with_C, int32_t* Ef_out, int32_t* nneu_out, void** plan_out) {
  return phfem_dist_level_count_ex(ctx, ppart, E0p, side, nullptr, neu_parent_ids, nN_parent, with_C, Ef_out,
                                   nneu_out, plan_out);
}

// Run half: the level kernel with the rank's fine offsets (f_off: first
// global fine edge id; nnz_off: first C entry) written straight into the
// fine lists, node_edge_start and C's row pointers; frees the plan.
PHFEM_API phfem_status phfem_dist_level_run_ex(phfem_ctx* ctx, void* plan, const double* coords, int32_t nc,
                                               int32_t node_lo, int32_t node_hi, int32_t nE_all, int32_t f_off,
                                               int32_t nnz_off, int32_t r_off, phfem_topology* out, uint8_t* rk,
                                               double* coords_fine, phfem_csr* C, int32_t* retained_pos,
                                               int32_t* retained_edges) {
  phfem_dist_level_plan* pl = (phfem_dist_level_plan*)plan;
  if (!ctx || !pl || !out) return PHFEM_ERR_INVALID_ARGUMENT;
  memset(out, 0, sizeof(*out));
  if (C) memset(C, 0, sizeof(*C));
  const phfem_topology* ppart = &pl->ppart;
  const int64_t E = ppart->E;
  const int32_t E0p = pl->E0p;
  phfem_status st = PHFEM_OK;
  if ((E > 0 && (!coords || !rk || !coords_fine)) || node_lo < 0 || node_hi < node_lo ||
      (E > 0 && (int64_t)node_hi != (int64_t)nc + E0p + E) || (E > 0 && node_lo > nc + E0p) ||
      4 * (int64_t)nE_all >= (int64_t(1) << 31) || (C != nullptr) != pl->with_C ||
      (retained_pos != nullptr) != (retained_edges != nullptr) || (retained_pos && !C) || r_off < 0)
    st = PHFEM_ERR_INVALID_ARGUMENT;
  const int64_t ntiles = pl->ntiles;
  int32_t *tileF = pl->tiles, *tileB = pl->tiles + (ntiles + 1), *tileN = pl->tiles + 2 * (ntiles + 1);
  const int32_t Ef = pl->Ef;
  const int64_t nBf = 2 * (int64_t)ppart->n_boundary;
  int64_t Lr = 0;
  if (st == PHFEM_OK) {
    out->nC = node_hi - node_lo;
    out->nE = 4 * nE_all;
    out->E = Ef;
    out->n_boundary = (int32_t)nBf;
    out->n_interior = (int32_t)(Ef - nBf);
    const int64_t cap = std::max<int64_t>(Ef, 1);
    auto al = [&](int32_t** p, int64_t n) { if (st == PHFEM_OK) st = dalloc(ctx, p, n); };
    al(&out->edge_nodes, 2 * cap);
    al(&out->edge_elements, 2 * cap);
    al(&out->local_in_tplus, cap);
    al(&out->local_in_tminus, cap);
    al(&out->interior_edges, std::max<int64_t>(Ef - nBf, 1));
    al(&out->boundary_edges, std::max<int64_t>(nBf, 1));
    al(&out->node_edge_start, (int64_t)out->nC + 1);
    if (st == PHFEM_OK) {  // nodes that start no fine edge (rank 0's old nodes; an empty range): f_off
      KTimer kt(ctx, "k_fill_lv");
      k_fill_lv<<<grid_for((int64_t)out->nC + 1, 256, ctx->num_sms * 4), 256, 0, ctx->stream>>>(
          out->node_edge_start, (int64_t)out->nC + 1, f_off);
      ctx->launches++;
    }
    if (st == PHFEM_OK && C) {
      Lr = Ef - 2 * (int64_t)pl->nneu;
      const int64_t BR = 2 * ((int64_t)ppart->n_boundary - pl->nneu);
      C->rows = (int32_t)Lr;
      C->cols = 3 * 4 * nE_all;
      C->nnz = 4 * Lr - 2 * BR;
      al(&C->row_ptr, Lr + 1);
      al(&C->col_idx, std::max<int64_t>(C->nnz, 1));
      if (st == PHFEM_OK) st = dalloc(ctx, &C->values, std::max<int64_t>(C->nnz, 1));
      if (st == PHFEM_OK && Lr == 0) {  // no rows: the one row pointer is the rank's first entry
        KTimer kt(ctx, "k_fill_lv");
        k_fill_lv<<<1, 32, 0, ctx->stream>>>(C->row_ptr, 1, nnz_off);
        ctx->launches++;
      }
    }
  }
  if (st == PHFEM_OK && E > 0) {
    LvArgs a;
    memset(&a, 0, sizeof a);
    a.edge_nodes = ppart->edge_nodes;
    a.edge_elements = ppart->edge_elements;
    a.ltp = ppart->local_in_tplus;
    a.ltm = ppart->local_in_tminus;
    a.side = reinterpret_cast<const int4*>(pl->side);
    a.own_el = pl->local.elements;
    a.own_ee = pl->local.elem_edge;
    a.own_lo = pl->local.elo;
    a.own_hi = pl->local.ehi;
    a.coords = (const double2*)coords;
    a.E = (int)E;
    a.nc = nc;
    a.Ef = Ef;
    a.eb = E0p;
    a.nlo = node_lo;
    a.f_off = f_off;
    a.nnz_off = nnz_off;
    a.r_off = r_off;
    a.tileF = tileF;
    a.tileB = tileB;
    LvOut o;
    memset(&o, 0, sizeof o);
    o.edge_nodes = out->edge_nodes;
    o.edge_elements = out->edge_elements;
    o.ltp = out->local_in_tplus;
    o.ltm = out->local_in_tminus;
    o.interior = out->interior_edges;
    o.boundary = out->boundary_edges;
    o.node_edge_start = out->node_edge_start;
    o.rk = rk;
    o.mid = (double2*)coords_fine;
    o.mid_base = 0;
    const unsigned nt = (unsigned)((E + kLvT - 1) / kLvT);
    if (C) {
      a.neu_bits = pl->nbits;
      a.tileN = tileN;
      a.L = (int)Lr;
      o.row_ptr = C->row_ptr;
      o.col = C->col_idx;
      o.val = C->values;
      o.rpos = retained_pos;      // global rows (r_off) / global edge ids (f_off)
      o.redges = retained_edges;
      st = launch_level<true>(ctx, a, o, nt);
    } else {
      st = launch_level<false>(ctx, a, o, nt);
    }
  }
  dfree(ctx, pl->nbits);
  dfree(ctx, pl->tiles);
  delete pl;
  return st;
}

PHFEM_API phfem_status phfem_dist_level_run(phfem_ctx* ctx, void* plan, const double* coords, int32_t nc,
                                            int32_t node_lo, int32_t node_hi, int32_t nE_all, int32_t f_off,
                                            int32_t nnz_off, phfem_topology* out, uint8_t* rk, double* coords_fine,
                                            phfem_csr* C) {
  return phfem_dist_level_run_ex(ctx, plan, coords, nc, node_lo, node_hi, nE_all, f_off, nnz_off, 0, out, rk,
                                 coords_fine, C, nullptr, nullptr);
}

PHFEM_API phfem_status phfem_dist_refine_level_side(phfem_ctx* ctx, const phfem_topology* ppart, int32_t E0p,
                                                    const int32_t* side, const double* coords, int32_t nc,
                                                    int32_t node_lo, int32_t node_hi, int32_t nE_all,
                                                    const int32_t* neu_parent_ids, int32_t nN_parent,
                                                    phfem_topology* out, uint8_t* rk, double* coords_fine,
                                                    phfem_csr* C) {
  if (!ctx || !ppart || !out) return PHFEM_ERR_INVALID_ARGUMENT;
  int32_t Ef = 0, nneu = 0;
  void* plan = nullptr;
  PHFEM_TRY(phfem_dist_level_count(ctx, ppart, E0p, side, neu_parent_ids, nN_parent, C != nullptr, &Ef, &nneu, &plan));
  return phfem_dist_level_run(ctx, plan, coords, nc, node_lo, node_hi, nE_all, 0, 0, out, rk, coords_fine, C);
}

PHFEM_API phfem_status phfem_dist_children_slots_ex(phfem_ctx* ctx, const int32_t* elements,
                                                    const int32_t* elem_edge, int32_t n, const int32_t* gs,
                                                    const uint8_t* grk, int32_t nc, int32_t own_lo, int32_t own_hi,
                                                    const int32_t* fine_nes, int32_t nes_off, const uint8_t* rk,
                                                    double* coords_fine, int32_t* children, int32_t* fine_elem_edge) {
  if (!ctx || (n && (!elements || !elem_edge || !gs || !grk || !coords_fine || !children || !fine_elem_edge)) ||
      (fine_nes && own_hi > own_lo && !rk))
    return PHFEM_ERR_INVALID_ARGUMENT;
  if (n > 0)
    PHFEM_LAUNCH(ctx, "k_dist_children_slots", k_dist_children_slots<<<grid_for(n, 256, ctx->num_sms * PHFEM_CH_GRID_MULT), 256, 0,
                                                                       ctx->stream>>>(
        elements, elem_edge, gs, grk, n, nc, own_lo, own_hi, fine_nes, nes_off, rk, (double2*)coords_fine,
        reinterpret_cast<int4*>(children), reinterpret_cast<int4*>(fine_elem_edge)));
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_dist_children_slots(phfem_ctx* ctx, const int32_t* elements,
                                                 const int32_t* elem_edge, int32_t n, const int32_t* gs,
                                                 const uint8_t* grk, int32_t nc, double* coords_fine,
                                                 int32_t* children, int32_t* fine_elem_edge) {
  return phfem_dist_children_slots_ex(ctx, elements, elem_edge, n, gs, grk, nc, 0, 0, nullptr, 0, nullptr,
                                      coords_fine, children, fine_elem_edge);
}
