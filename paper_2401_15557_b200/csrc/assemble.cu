// assemble.cu — assembly on sm_100a: element blocks + load (one fused element
// pass), the coupling matrix C (CSR, and the reference's Eigen CSC layout),
// the Neumann and Dirichlet vectors.
//
// Reference: proj/src/assembly.cpp:17-242, sparse.cpp:30-120.
// Values are bit-identical to the reference: the kernels evaluate the same
// expressions in the same order (phfem_fields.h) and the library is built with
// --fmad=false, so no FMA contraction changes a rounding.
#include <algorithm>

#include "common.cuh"
#include "elem.cuh"
#include "kernels.cuh"

namespace phfem {

// ---------------------------------------------------------------------------
// Element pass.  One thread per element; each warp owns 32 consecutive
// elements, so a 3x3 block of the warp is 32 x 72 = 2304 contiguous bytes.
// A block is computed, staged in the warp's SMEM slice (stride 9 doubles:
// conflict-free) and written back with 16-byte coalesced stores, one block at
// a time (low register pressure, no block-wide barrier: warps stream
// independently, so stores of one warp overlap the fp64 work of others).
constexpr int kVolThreads = 128;
constexpr int kVolWarps = kVolThreads / 32;
#ifndef PHFEM_VOL_MIN_BLOCKS
#define PHFEM_VOL_MIN_BLOCKS 6
#endif
constexpr int kVolMinBlocks = PHFEM_VOL_MIN_BLOCKS;
#ifndef PHFEM_VOL_ITERS
#define PHFEM_VOL_ITERS 3
#endif
constexpr int kVolIters = PHFEM_VOL_ITERS;  // 32-element chunks per warp (grid sizing)

__device__ __forceinline__ void warp_store(double* __restrict__ g, int64_t base, int n_valid,
                                           int per, const double* vals, double* buf, int vec) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 9; ++k)
    if (k < per) buf[lane * per + k] = vals[k];
  __syncwarp();
  const int count = n_valid * per;
  double* dst = g + base * per;
#if PHFEM_VOL_ST256
  // 32-byte streaming stores (STG.E.ENL2.256, sm_100): half the store
  // instructions of the 16-byte form; the destination is 32-byte aligned
  // when vec == 2 (chunk spans are multiples of 768 B).  Measured slower
  // (k_volume 7.61 -> 7.87 ms at L13: the 32-byte-stride SMEM reads conflict;
  // the store-only pattern gains nothing either, tools/micro/volpat.cu), so
  // off by default
  if (vec == 2) {
    const int n4 = count >> 2;
    for (int i = lane; i < n4; i += 32) {
      const double2 lo = reinterpret_cast<const double2*>(buf)[2 * i];
      const double2 hi = reinterpret_cast<const double2*>(buf)[2 * i + 1];
      asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(dst + 4 * i), "d"(lo.x), "d"(lo.y),
                   "d"(hi.x), "d"(hi.y)
                   : "memory");
    }
    for (int i = 4 * n4 + lane; i < count; i += 32) dst[i] = buf[i];
    return;
  }
#endif
  if (vec) {
    const double2* src2 = reinterpret_cast<const double2*>(buf);
    double2* dst2 = reinterpret_cast<double2*>(dst);
    for (int i = lane; i < count / 2; i += 32) __stcs(dst2 + i, src2[i]);
    if ((count & 1) && lane == 0) dst[count - 1] = buf[count - 1];
  } else {
    for (int i = lane; i < count; i += 32) dst[i] = buf[i];
  }
}

__device__ __forceinline__ double2 vol_mid(double2 p, double2 q) {
  return make_double2(0.5 * (p.x + q.x), 0.5 * (p.y + q.y));  // refine.cpp:18
}

template <bool kBlocks, bool kLoad, int FK, int CK, bool kParent>
__global__ void __launch_bounds__(kVolThreads, kVolMinBlocks) k_volume(VolArgs a, phfem_dev_errors* err) {
  pdl_wait();
  pdl_trigger();
  __shared__ __align__(16) double wbuf[kVolWarps][32 * 9];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* buf = wbuf[warp];
  const int64_t nchunks = ((int64_t)a.nE + 31) / 32;
  const int64_t step = (int64_t)gridDim.x * kVolWarps;
  // software pipeline: the vertex indices of chunk ch + 2 step and the
  // coordinates of chunk ch + step are in flight while chunk ch computes
  // (two chunks of coordinates in flight measured: config 4 unchanged at
  // 10.27 ms with 5 CTAs/SM, 10.46 at 6; config 5 6.91 -> 7.20 / 7.61 ms).
  // kParent: a chunk is 8 parents x 4 children (nE = 4 x parents, chunk bases
  // are multiples of 32, so a group of 4 lanes is one parent); lane 4q + k
  // (k = 1..3) loads parent vertex p_{k-1} and its coordinates, lane 4q idles;
  // the group shares them by shuffles and recomputes the midpoints
  const int k4 = lane & 3;
  auto ld_idx = [&](int64_t c, int& i0, int& i1, int& i2) {
    const int64_t m = c * 32 + lane;
    if (c < nchunks && m < a.nE) {
      if (kParent) {
        i0 = k4 ? __ldg(a.parents + 3 * (m >> 2) + (k4 - 1)) : -2;
      } else {
        i0 = __ldg(a.elements + 3 * m);
        i1 = __ldg(a.elements + 3 * m + 1);
        i2 = __ldg(a.elements + 3 * m + 2);
      }
    } else {
      i0 = -1;
    }
  };
  auto ld_xy = [&](int i0, int i1, int i2, double2& v0, double2& v1, double2& v2) {
    if (kParent) {  // v0 only: this lane's parent vertex (a unit triangle on padding groups)
      if (i0 >= 0) v0 = __ldg(a.coords + i0);
      else v0 = make_double2(k4 == 2 ? 1.0 : 0.0, k4 == 3 ? 1.0 : 0.0);
    } else if (i0 >= 0) {
      v0 = __ldg(a.coords + i0);
      v1 = __ldg(a.coords + i1);
      v2 = __ldg(a.coords + i2);
    } else {  // padding lanes: a harmless unit triangle
      v0 = make_double2(0.0, 0.0);
      v1 = make_double2(1.0, 0.0);
      v2 = make_double2(0.0, 1.0);
    }
  };
  int64_t ch = (int64_t)blockIdx.x * kVolWarps + warp;
  int i0, i1, i2, n0, n1, n2;
  ld_idx(ch, i0, i1, i2);
  ld_idx(ch + step, n0, n1, n2);
  double2 v0, v1, v2;
  ld_xy(i0, i1, i2, v0, v1, v2);
  for (; ch < nchunks; ch += step) {
    const int64_t base = ch * 32;
    const int n_valid = (int)((int64_t)a.nE - base < 32 ? (int64_t)a.nE - base : 32);
    const int64_t m = base + lane;
    const bool valid = lane < n_valid;
    // next chunk's coordinates, the one after's indices
    double2 w0, w1, w2;
    ld_xy(n0, n1, n2, w0, w1, w2);
    ld_idx(ch + 2 * step, n0, n1, n2);
    double2 c0 = v0, c1 = v1, c2 = v2;
    if (kParent) {
      const int g = lane & ~3;
      const double2 p0 = make_double2(__shfl_sync(0xffffffffu, v0.x, g + 1), __shfl_sync(0xffffffffu, v0.y, g + 1));
      const double2 p1 = make_double2(__shfl_sync(0xffffffffu, v0.x, g + 2), __shfl_sync(0xffffffffu, v0.y, g + 2));
      const double2 p2 = make_double2(__shfl_sync(0xffffffffu, v0.x, g + 3), __shfl_sync(0xffffffffu, v0.y, g + 3));
      const double2 m0 = vol_mid(p1, p2), m1 = vol_mid(p2, p0), m2 = vol_mid(p0, p1);
      c0 = k4 == 0 ? m0 : k4 == 1 ? p0 : k4 == 2 ? p1 : p2;
      c1 = k4 == 0 ? m1 : k4 == 1 ? m2 : k4 == 2 ? m0 : m1;
      c2 = k4 == 0 ? m2 : k4 == 1 ? m1 : k4 == 2 ? m2 : m0;
    }
    if (kLoad) {
      double bl[3];
      element_load_dev<FK>(c0, c1, c2, a.f, a.t, bl, valid, m, err, a.samples);
      warp_store(a.load, base, n_valid, 3, bl, buf, a.vec);
    }
    if (kBlocks) {
      const phfem_geom g = geometry_dev(c0.x, c0.y, c1.x, c1.y, c2.x, c2.y);
      if (valid && !(g.t2 > 0.0)) atomicMin(&err->degenerate, (unsigned long long)m);
      const phfem_coeff_values cv = coeffs_dev<CK>(a.coeffs, c0, c1, c2);
      double x[9];
      if (a.B) {
        phfem_stiffness(&g, &cv, x);
        warp_store(a.B, base, n_valid, 9, x, buf, a.vec);
      }
      if (a.D) {
        convection_dev(&g, &cv, x);
        warp_store(a.D, base, n_valid, 9, x, buf, a.vec);
      }
      if (a.M) {
        phfem_mass(&g, cv.delta, x);
        warp_store(a.M, base, n_valid, 9, x, buf, a.vec);
      }
      if (a.M0) {
        phfem_unit_mass(&g, x);
        warp_store(a.M0, base, n_valid, 9, x, buf, a.vec);
      }
    }
    v0 = w0;
    v1 = w1;
    v2 = w2;
  }
}

phfem_status launch_volume(phfem_ctx* ctx, const VolArgs& a, bool blocks, bool load) {
  if (a.nE == 0) return PHFEM_OK;
  if (a.parents && (a.nE & 3)) return set_error(ctx, PHFEM_ERR_INVALID_ARGUMENT, "k_volume: children count not 4 x parents");
  const int64_t nchunks = ((int64_t)a.nE + 31) / 32;
  // about kVolIters chunks per warp: a grid of many short-lived CTAs spreads
  // the concurrently written addresses over several windows of every output
  // stream — measured at L13: 32 CTAs per SM (36 chunks per warp) 7.62 ms,
  // 1024 / 2048 / 4096 per SM (7 / 3.5 / 1.7 chunks) 6.96 / 6.84 / 7.06 ms,
  // one chunk per warp 8.05 ms (no software pipelining left)
  const int64_t per_cta = (int64_t)kVolWarps * kVolIters;
  const int grid = (int)std::max<int64_t>(std::min<int64_t>((nchunks + kVolWarps - 1) / kVolWarps,
                                                            (int64_t)ctx->num_sms * 8),
                                          (nchunks + per_cta - 1) / per_cta);
  const int fk = !load ? kKindGeneric : (a.samples ? kKindSamples : field_kind_spec(a.f));
  const int ck = a.coeffs.kind == PHFEM_COEFF_CENTROID_POLY ? PHFEM_COEFF_CENTROID_POLY : PHFEM_COEFF_CONST;
#define PHFEM_VOL(B, L, F, K)                                                                      \
  do {                                                                                             \
    if (a.parents) PHFEM_LAUNCH_PDL(ctx, "k_volume", (k_volume<B, L, F, K, true>), grid, kVolThreads, 0, a, ctx->derr); \
    else PHFEM_LAUNCH_PDL(ctx, "k_volume", (k_volume<B, L, F, K, false>), grid, kVolThreads, 0, a, ctx->derr);         \
  } while (0)
#define PHFEM_VOL_CK(B, L, F)                                                            \
  do {                                                                                   \
    if (ck == PHFEM_COEFF_CENTROID_POLY) PHFEM_VOL(B, L, F, PHFEM_COEFF_CENTROID_POLY); \
    else PHFEM_VOL(B, L, F, PHFEM_COEFF_CONST);                                          \
  } while (0)
#define PHFEM_VOL_FK(B, L)                                                               \
  do {                                                                                   \
    if (fk == PHFEM_FIELD_SINSIN) PHFEM_VOL_CK(B, L, PHFEM_FIELD_SINSIN);               \
    else if (fk == PHFEM_FIELD_EXP_SINSIN) PHFEM_VOL_CK(B, L, PHFEM_FIELD_EXP_SINSIN);  \
    else if (fk == PHFEM_FIELD_ZERO) PHFEM_VOL_CK(B, L, PHFEM_FIELD_ZERO);              \
    else if (fk == kKindSamples) PHFEM_VOL_CK(B, L, kKindSamples);                       \
    else PHFEM_VOL_CK(B, L, kKindGeneric);                                               \
  } while (0)
  if (blocks && load) PHFEM_VOL_FK(true, true);
  else if (blocks) PHFEM_VOL_CK(true, false, kKindGeneric);
  else PHFEM_VOL_FK(false, true);
#undef PHFEM_VOL_FK
#undef PHFEM_VOL_CK
#undef PHFEM_VOL
  return PHFEM_OK;
}

static bool aligned16(const void* p) { return p == nullptr || ((uintptr_t)p & 15u) == 0; }
static bool aligned32(const void* p) { return p == nullptr || ((uintptr_t)p & 31u) == 0; }

VolArgs make_vol_args(const phfem_mesh* mesh) {
  VolArgs a;
  memset(&a, 0, sizeof a);
  a.coords = (const double2*)mesh->coords;
  a.elements = mesh->elements;
  a.nE = mesh->nE;
  return a;
}

// ---------------------------------------------------------------------------
// C in CSR (assembly.cpp:144-168).  Row pointers come from the per-block
// boundary / Neumann prefixes of classify_edges (a retained boundary row
// holds 2 entries, an interior row 4).
constexpr int kCsrEdges = 1024;  // the classification's prefix block

// Warp-staged: a CTA of 8 warps owns the 1024-edge block of the
// classification's prefixes, each warp 4 chunks of 32 consecutive edges
// (coalesced 4-byte loads per chunk).  Row starts k = 4 rp - 2 (retained
// boundary rows before) from the block prefixes + ballot counts.  A chunk's
// entries are contiguous: they go out as "pairs" — (3t + c0, 3t + c1) with
// one value, the T+ pair then the T- pair of a row — staged per warp as
// 16-byte records (<= 2-way SMEM conflicts) and stored as int2 / double2 by
// consecutive lanes (the previous layout staged 4 entries per thread at
// stride 4, a 16- to 32-way bank conflict on every staging store).
constexpr int kCsr2Warps = 8;
struct CsrPair {
  int2 col;
  double val;
};

__global__ void __launch_bounds__(32 * kCsr2Warps) k_constraint_csr2(
    const double2* __restrict__ coords, const int32_t* __restrict__ edge_nodes,
    const int32_t* __restrict__ edge_elements, const int32_t* __restrict__ ltp,
    const int32_t* __restrict__ ltm, const int32_t* __restrict__ rpos,
    const int32_t* __restrict__ pre_bnd, const int32_t* __restrict__ pre_neu, int E, int L,
    int32_t* __restrict__ row_ptr, int32_t* __restrict__ col, double* __restrict__ val) {
  __shared__ CsrPair stage[kCsr2Warps][64];
  __shared__ int32_t wcnt[kCsr2Warps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int blk = blockIdx.x;
  const int64_t eb = (int64_t)blk * kCsrEdges + warp * 128;
  int rp[4], tp[4], tm[4], lp[4], lm[4];
  double len[4];
  unsigned rbm[4];
  int c_before[4];
  int own = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int64_t e = eb + 32 * j + lane;
    const bool ok = e < E;
    rp[j] = ok ? __ldg(rpos + e) : -1;
    const int2 el = ok ? reinterpret_cast<const int2*>(edge_elements)[e] : make_int2(0, -1);
    tp[j] = el.x;
    tm[j] = el.y;
    lp[j] = ok ? __ldg(ltp + e) : 0;
    lm[j] = ok ? __ldg(ltm + e) : 0;
    len[j] = 0.0;
    if (rp[j] >= 0) {
      const int2 ab = reinterpret_cast<const int2*>(edge_nodes)[e];
      const double2 pa = __ldg(coords + ab.x), pb = __ldg(coords + ab.y);
      const double dx = pb.x - pa.x, dy = pb.y - pa.y;
      len[j] = sqrt(dx * dx + dy * dy);  // edge_topology.cpp:183
    }
    rbm[j] = __ballot_sync(0xffffffffu, rp[j] >= 0 && tm[j] < 0);
    c_before[j] = own;
    own += __popc(rbm[j]);
  }
  if (lane == 0) wcnt[warp] = own;
  __syncthreads();
  int wpre = 0;
  for (int w = 0; w < warp; ++w) wpre += wcnt[w];
  const int base_b = pre_bnd[blk] - pre_neu[blk] + wpre;  // retained boundary rows before the warp
  CsrPair* st = stage[warp];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int bret = base_b + c_before[j] + __popc(rbm[j] & lanemask_lt());
    const bool ret = rp[j] >= 0;
    const int k = 4 * rp[j] - 2 * bret;
    const int kmin = __reduce_min_sync(0xffffffffu, ret ? k : 0x7fffffff);
    if (kmin == 0x7fffffff) continue;  // no retained edge in the chunk
    const int n = ret ? (tm[j] >= 0 ? 4 : 2) : 0;
    if (ret) {
      row_ptr[rp[j]] = k;
      if (rp[j] == L - 1) row_ptr[L] = k + n;
      const int q = (k - kmin) >> 1;
      const int c0 = lp[j] == 0 ? 1 : 0, c1 = lp[j] == 2 ? 1 : 2;
      st[q] = CsrPair{make_int2(3 * tp[j] + c0, 3 * tp[j] + c1), len[j] * 0.5};  // assembly.cpp:160
      if (tm[j] >= 0) {
        const int d0 = lm[j] == 0 ? 1 : 0, d1 = lm[j] == 2 ? 1 : 2;
        st[q + 1] = CsrPair{make_int2(3 * tm[j] + d0, 3 * tm[j] + d1), -len[j] * 0.5};  // :164
      }
    }
    const int kend = __reduce_max_sync(0xffffffffu, ret ? k + n : 0);
    const int npairs = (kend - kmin) >> 1;
    __syncwarp();
    for (int p = lane; p < npairs; p += 32) {
      const CsrPair r = st[p];
      *reinterpret_cast<int2*>(col + kmin + 2 * p) = r.col;
      __stcs(reinterpret_cast<double2*>(val + kmin + 2 * p), make_double2(r.val, r.val));
    }
    __syncwarp();
  }
}

// C in Eigen CSC (column = primal DOF 3m+c; <= 2 entries, rows ascending).
__device__ __forceinline__ void csc_entries(const double2* __restrict__ coords,
                                            const int32_t* __restrict__ elements,
                                            const int32_t* __restrict__ elem_edge,
                                            const int32_t* __restrict__ rpos, int64_t m,
                                            int rows[3], double vals[3]) {
  const int t[3] = {__ldg(elements + 3 * m), __ldg(elements + 3 * m + 1), __ldg(elements + 3 * m + 2)};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int s = __ldg(elem_edge + 3 * m + k);
    const int e = s >= 0 ? s : ~s;
    rows[k] = rpos[e];
    const double2 pa = __ldg(coords + t[(k + 1) % 3]), pb = __ldg(coords + t[(k + 2) % 3]);
    const double dx = pb.x - pa.x, dy = pb.y - pa.y;
    const double len = sqrt(dx * dx + dy * dy);
    vals[k] = s >= 0 ? len * 0.5 : -len * 0.5;
  }
}

__global__ void k_csc_count(const int32_t* __restrict__ elem_edge, const int32_t* __restrict__ rpos,
                            int nE, int32_t* __restrict__ counts) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < nE; m += stride) {
    int r[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int s = elem_edge[3 * m + k];
      r[k] = rpos[s >= 0 ? s : ~s] >= 0;
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) counts[3 * m + c] = r[(c + 1) % 3] + r[(c + 2) % 3];
  }
}

__global__ void k_csc_fill(const double2* __restrict__ coords, const int32_t* __restrict__ elements,
                           const int32_t* __restrict__ elem_edge, const int32_t* __restrict__ rpos,
                           int nE, const int32_t* __restrict__ outer, int32_t* __restrict__ inner,
                           double* __restrict__ values) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < nE; m += stride) {
    int rows[3];
    double vals[3];
    csc_entries(coords, elements, elem_edge, rpos, m, rows, vals);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      int ka = (c + 1) % 3, kb = (c + 2) % 3;
      if (rows[kb] >= 0 && (rows[ka] < 0 || rows[kb] < rows[ka])) {
        const int x = ka;
        ka = kb;
        kb = x;
      }
      int p = outer[3 * m + c];
      if (rows[ka] >= 0) {
        inner[p] = rows[ka];
        values[p] = vals[ka];
        ++p;
      }
      if (rows[kb] >= 0) {
        inner[p] = rows[kb];
        values[p] = vals[kb];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Neumann: entries grouped by their t_plus element in a small open-addressing
// table (one slot per element carrying Neumann edges).  Per DOF at most two
// entries carry a non-zero term, so the float sum is order independent and
// atomics reproduce scatter_add exactly; a duplicated Neumann pair (more terms)
// switches to a single-thread pass in list order.
__global__ void k_neu_insert(const int32_t* __restrict__ neu_ids, int nN,
                             const int32_t* __restrict__ edge_elements, int cap,
                             int32_t* __restrict__ keys, int32_t* __restrict__ slot_of) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nN;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int m = edge_elements[2 * neu_ids[i]];
    uint32_t h = neu_hash(m, cap);
    while (true) {
      const int prev = atomicCAS(&keys[h], -1, m);
      if (prev == -1 || prev == m) break;
      h = (h + 1) & (uint32_t)(cap - 1);
    }
    slot_of[i] = (int)h;
  }
}

__device__ __forceinline__ void neu_entry(const NeuArgs& a, int64_t i, double t, double v[3],
                                          phfem_dev_errors* err) {
  const int e = a.neu_ids[i];
  const int2 ab = reinterpret_cast<const int2*>(a.edge_nodes)[e];
  const double2 pa = a.coords[ab.x], pb = a.coords[ab.y];
  const double midx = 0.5 * (pa.x + pb.x), midy = 0.5 * (pa.y + pb.y);
  const double dx = pb.x - pa.x, dy = pb.y - pa.y;
  const double length = sqrt(dx * dx + dy * dy);
  const double nx = dy / length, ny = -dx / length;
  const double g = a.samples ? a.samples[i] : phfem_flux_eval(&a.g, midx, midy, nx, ny, t);
  if (!isfinite(g)) atomicMin(&err->flux_nan, (unsigned long long)i);
  const int led = a.ltp[e];
  const double lg = length * g;
#pragma unroll
  for (int c = 0; c < 3; ++c) v[c] = lg * (c == led ? 0.0 : 0.5);  // length*value*kR[led][c]
}

__global__ void k_neu_values(NeuArgs a, double t, int seq, phfem_dev_errors* err) {
  pdl_wait();
  pdl_trigger();
  if (seq) {  // exact list-order accumulation (duplicated pairs)
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    for (int64_t i = 0; i < a.nN; ++i) {
      double v[3];
      neu_entry(a, i, t, v, err);
      const int s = a.slot_of[i];
      for (int c = 0; c < 3; ++c) a.vals[3 * s + c] += v[c];
    }
    return;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.nN;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v[3];
    neu_entry(a, i, t, v, err);
    const int s = a.slot_of[i];
#pragma unroll
    for (int c = 0; c < 3; ++c) atomicAdd(&a.vals[3 * s + c], v[c]);
  }
}

__global__ void k_neu_apply(const int32_t* __restrict__ keys, const double* __restrict__ vals,
                            int cap, double* __restrict__ out, int accumulate) {
  pdl_wait();
  pdl_trigger();
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < cap;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int m = keys[s];
    if (m < 0) continue;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double v = vals[3 * s + c];
      out[3 * (int64_t)m + c] = accumulate ? out[3 * (int64_t)m + c] + v : v;
    }
  }
}

phfem_status neu_table_build(phfem_ctx* ctx, const phfem_topology* topo,
                             const phfem_classification* cls, NeuTable* tab) {
  memset(tab, 0, sizeof(*tab));
  tab->nN = cls->nN;
  if (cls->nN == 0) return PHFEM_OK;
  int cap = 64;
  while (cap < 2 * cls->nN) cap <<= 1;
  tab->cap = cap;
  tab->seq = (cls->flags & PHFEM_CLS_DUP_NEUMANN) ? 1 : 0;
  PHFEM_TRY(dalloc(ctx, &tab->keys, cap));
  PHFEM_TRY(dalloc(ctx, &tab->slot_of, cls->nN));
  PHFEM_TRY(dalloc(ctx, &tab->vals, 3 * (int64_t)cap));
  PHFEM_CUDA(ctx, cudaMemsetAsync(tab->keys, 0xff, sizeof(int32_t) * cap, ctx->stream));
  PHFEM_LAUNCH(ctx, "k_neu_insert", k_neu_insert<<<grid_for(cls->nN, 256, ctx->num_sms * 4), 256, 0, ctx->stream>>>(
      cls->neumann_edge_ids, cls->nN, topo->edge_elements, cap, tab->keys, tab->slot_of));
  return PHFEM_OK;
}

void neu_table_free(phfem_ctx* ctx, NeuTable* tab) {
  dfree(ctx, tab->keys);
  dfree(ctx, tab->slot_of);
  dfree(ctx, tab->vals);
}

phfem_status neu_table_eval(phfem_ctx* ctx, const NeuTable* tab, const phfem_mesh* mesh,
                            const phfem_topology* topo, const phfem_classification* cls,
                            const phfem_field* g, double t, double* vals,
                            const double* samples) {
  if (tab->nN == 0) return PHFEM_OK;
  NeuArgs a;
  a.coords = (const double2*)mesh->coords;
  a.edge_nodes = topo->edge_nodes;
  a.ltp = topo->local_in_tplus;
  a.neu_ids = cls->neumann_edge_ids;
  a.slot_of = tab->slot_of;
  a.nN = tab->nN;
  a.g = *g;
  a.samples = samples;
  a.vals = vals;
  PHFEM_CUDA(ctx, cudaMemsetAsync(vals, 0, sizeof(double) * 3 * tab->cap, ctx->stream));
  PHFEM_LAUNCH(ctx, "k_neu_values", k_neu_values<<<tab->seq ? 1 : grid_for(tab->nN, 256, ctx->num_sms * 4), tab->seq ? 1 : 256, 0,
                 ctx->stream>>>(a, t, tab->seq, ctx->derr));
  return PHFEM_OK;
}

phfem_status neu_flux_error(phfem_ctx* ctx, const phfem_mesh* mesh, const phfem_topology* topo,
                            const phfem_classification* cls) {
  const uint64_t fe = ctx->herr->flux_nan;
  if (fe == ~0ull) return PHFEM_OK;
  int32_t e = 0;
  int32_t ab[2] = {0, 0};
  PHFEM_CUDA(ctx, cudaMemcpyAsync(&e, cls->neumann_edge_ids + fe, sizeof e, cudaMemcpyDeviceToHost,
                                  ctx->stream));
  PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  PHFEM_CUDA(ctx, cudaMemcpyAsync(ab, topo->edge_nodes + 2 * (int64_t)e, sizeof ab,
                                  cudaMemcpyDeviceToHost, ctx->stream));
  PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  (void)mesh;
  return set_error(ctx, PHFEM_ERR_NONFINITE,
                   "assemble_neumann: non-finite flux sample on edge (%d,%d)", ab[0] + 1, ab[1] + 1);
}

phfem_status neumann_into(phfem_ctx* ctx, const phfem_mesh* mesh, const phfem_topology* topo,
                          const phfem_classification* cls, const phfem_field* g, double t,
                          double* out, int accumulate, bool check, const double* samples) {
  if (cls->nN == 0) return PHFEM_OK;
  NeuTable tab;
  PHFEM_TRY(neu_table_build(ctx, topo, cls, &tab));
  if (check) PHFEM_TRY(errors_reset(ctx));
  PHFEM_TRY(neu_table_eval(ctx, &tab, mesh, topo, cls, g, t, tab.vals, samples));
  PHFEM_LAUNCH(ctx, "k_neu_apply", k_neu_apply<<<grid_for(tab.cap, 256, ctx->num_sms * 4), 256, 0, ctx->stream>>>(
      tab.keys, tab.vals, tab.cap, out, accumulate));
  neu_table_free(ctx, &tab);
  if (check) {
    PHFEM_TRY(errors_fetch(ctx));
    PHFEM_TRY(neu_flux_error(ctx, mesh, topo, cls));
  }
  return PHFEM_OK;
}

// ---------------------------------------------------------------------------
__global__ void k_dirichlet(const double2* __restrict__ coords, const int32_t* __restrict__ edge_nodes,
                            const int32_t* __restrict__ dir_ids, int nD,
                            const int32_t* __restrict__ rpos, phfem_field uD, double t,
                            double* __restrict__ out, const double* __restrict__ samples) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nD;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int e = dir_ids[i];
    const int pos = rpos[e];
    if (pos < 0) continue;  // pair listed as both Dirichlet and Neumann
    const int2 ab = reinterpret_cast<const int2*>(edge_nodes)[e];
    const double2 pa = coords[ab.x], pb = coords[ab.y];
    const double midx = 0.5 * (pa.x + pb.x), midy = 0.5 * (pa.y + pb.y);
    const double dx = pb.x - pa.x, dy = pb.y - pa.y;
    const double length = sqrt(dx * dx + dy * dy);
    const double u = samples ? samples[i] : phfem_field_eval(&uD, midx, midy, t);
    out[pos] = -length * u;  // assembly.cpp:239
  }
}

// r_off: the classification's retained positions start at r_off (a rank of
// the distributed pipeline with global positions); out holds rows r_off..
phfem_status dirichlet_into(phfem_ctx* ctx, const phfem_mesh* mesh, const phfem_topology* topo,
                            const phfem_classification* cls, const phfem_field* uD, double t,
                            double* out, const double* samples, int32_t r_off) {
  if (cls->L > 0)
    PHFEM_CUDA(ctx, cudaMemsetAsync(out, 0, sizeof(double) * cls->L, ctx->stream));
  if (cls->nD == 0) return PHFEM_OK;
  PHFEM_LAUNCH(ctx, "k_dirichlet", k_dirichlet<<<grid_for(cls->nD, 256, ctx->num_sms * 4), 256, 0, ctx->stream>>>(
      (const double2*)mesh->coords, topo->edge_nodes, cls->dirichlet_edge_ids, cls->nD,
      cls->retained_pos, *uD, t, out - r_off, samples));
  return PHFEM_OK;
}

phfem_status constraint_csr_into(phfem_ctx* ctx, const phfem_mesh* mesh,
                                 const phfem_topology* topo, const phfem_classification* cls,
                                 phfem_csr* out) {
  memset(out, 0, sizeof(*out));
  const int E = topo->E, L = cls->L;
  const int nblk = (E + 1023) / 1024;
  out->rows = L;
  out->cols = 3 * mesh->nE;
  const int64_t bret_total = (int64_t)topo->n_boundary - (int64_t)(E - L);
  out->nnz = 4 * (int64_t)L - 2 * bret_total;
  PHFEM_TRY(dalloc(ctx, &out->row_ptr, (int64_t)L + 1));
  PHFEM_TRY(dalloc(ctx, &out->col_idx, out->nnz));
  PHFEM_TRY(dalloc(ctx, &out->values, out->nnz));
  if (L == 0) {
    PHFEM_CUDA(ctx, cudaMemsetAsync(out->row_ptr, 0, sizeof(int32_t), ctx->stream));
    return PHFEM_OK;
  }
  // col / val pairs need 8 / 16-byte alignment: true for pool allocations
  PHFEM_LAUNCH(ctx, "k_constraint_csr", k_constraint_csr2<<<nblk, 32 * kCsr2Warps, 0, ctx->stream>>>(
      (const double2*)mesh->coords, topo->edge_nodes, topo->edge_elements, topo->local_in_tplus,
      topo->local_in_tminus, cls->retained_pos, cls->block_prefix, cls->block_prefix + nblk + 1, E,
      L, out->row_ptr, out->col_idx, out->values));
  return PHFEM_OK;
}

phfem_status volume_errors(phfem_ctx* ctx, bool blocks, bool load) {
  if (blocks && ctx->herr->degenerate != ~0ull)
    return set_error(ctx, PHFEM_ERR_DEGENERATE,
                     "local_element_matrices: degenerate or non-CCW triangle");
  if (load && ctx->herr->load_nan != ~0ull)
    return set_error(ctx, PHFEM_ERR_NONFINITE,
                     "assemble_load: non-finite load sample in element %llu",
                     (unsigned long long)ctx->herr->load_nan + 1ull);
  return PHFEM_OK;
}

}  // namespace phfem

using namespace phfem;

PHFEM_API phfem_status phfem_assemble_volume(phfem_ctx* ctx, const phfem_mesh* mesh,
                                             const phfem_coeffs* c, double* B, double* D,
                                             double* M, double* M0) {
  if (!ctx || !mesh || !c) return PHFEM_ERR_INVALID_ARGUMENT;
  VolArgs a = make_vol_args(mesh);
  a.coeffs = *c;
  a.B = B;
  a.D = D;
  a.M = M;
  a.M0 = M0;
  a.vec = aligned16(B) && aligned16(D) && aligned16(M) && aligned16(M0);
  if (a.vec && aligned32(B) && aligned32(D) && aligned32(M) && aligned32(M0)) a.vec = 2;
  PHFEM_TRY(errors_reset(ctx));
  PHFEM_TRY(launch_volume(ctx, a, true, false));
  PHFEM_TRY(errors_fetch(ctx));
  return volume_errors(ctx, true, false);
}

// assemble_volume_operators + assemble_load in one element pass (the fused
// k_volume of the pipeline): same values as the two calls, one read of the mesh
PHFEM_API phfem_status phfem_assemble_volume_load(phfem_ctx* ctx, const phfem_mesh* mesh,
                                                  const phfem_coeffs* c, const phfem_field* f, double t,
                                                  double* B, double* D, double* M, double* M0,
                                                  double* load) {
  if (!ctx || !mesh || !c || !f || (!load && mesh->nE)) return PHFEM_ERR_INVALID_ARGUMENT;
  VolArgs a = make_vol_args(mesh);
  a.coeffs = *c;
  a.B = B;
  a.D = D;
  a.M = M;
  a.M0 = M0;
  a.f = *f;
  a.t = t;
  a.load = load;
  a.vec = aligned16(B) && aligned16(D) && aligned16(M) && aligned16(M0) && aligned16(load);
  if (a.vec && aligned32(B) && aligned32(D) && aligned32(M) && aligned32(M0) && aligned32(load)) a.vec = 2;
  PHFEM_TRY(errors_reset(ctx));
  PHFEM_TRY(launch_volume(ctx, a, true, true));
  PHFEM_TRY(errors_fetch(ctx));
  return volume_errors(ctx, true, true);
}

// phfem_assemble_volume_load in two halves, so that a caller can enqueue
// other work while the element pass runs: _start resets the ctx error block
// and launches (no synchronisation); _finish fetches it and raises the
// reference's errors.  Nothing between the two may use the ctx error block
// (the sharded pipeline runs its classification / bD / Neumann tables there).
PHFEM_API phfem_status phfem_dist_volume_start(phfem_ctx* ctx, const phfem_mesh* mesh, const phfem_coeffs* c,
                                               const phfem_field* f, double t, double* B, double* D, double* M,
                                               double* M0, double* load) {
  if (!ctx || !mesh || !c || !f || (!load && mesh->nE)) return PHFEM_ERR_INVALID_ARGUMENT;
  VolArgs a = make_vol_args(mesh);
  a.coeffs = *c;
  a.B = B;
  a.D = D;
  a.M = M;
  a.M0 = M0;
  a.f = *f;
  a.t = t;
  a.load = load;
  a.vec = aligned16(B) && aligned16(D) && aligned16(M) && aligned16(M0) && aligned16(load);
  if (a.vec && aligned32(B) && aligned32(D) && aligned32(M) && aligned32(M0) && aligned32(load)) a.vec = 2;
  PHFEM_TRY(errors_reset(ctx));
  return launch_volume(ctx, a, true, true);
}

PHFEM_API phfem_status phfem_dist_volume_finish(phfem_ctx* ctx) {
  if (!ctx) return PHFEM_ERR_INVALID_ARGUMENT;
  PHFEM_TRY(errors_fetch(ctx));
  return volume_errors(ctx, true, true);
}

PHFEM_API phfem_status phfem_assemble_load(phfem_ctx* ctx, const phfem_mesh* mesh,
                                           const phfem_field* f, double t, double* out) {
  if (!ctx || !mesh || !f || (!out && mesh->nE)) return PHFEM_ERR_INVALID_ARGUMENT;
  VolArgs a = make_vol_args(mesh);
  a.f = *f;
  a.t = t;
  a.load = out;
  a.vec = aligned16(out);
  if (a.vec && aligned32(out)) a.vec = 2;
  PHFEM_TRY(errors_reset(ctx));
  PHFEM_TRY(launch_volume(ctx, a, false, true));
  PHFEM_TRY(errors_fetch(ctx));
  return volume_errors(ctx, false, true);
}

PHFEM_API phfem_status phfem_assemble_constraint(phfem_ctx* ctx, const phfem_mesh* mesh,
                                                 const phfem_topology* topo,
                                                 const phfem_classification* cls,
                                                 phfem_csr* out) {
  if (!ctx || !mesh || !topo || !cls || !out) return PHFEM_ERR_INVALID_ARGUMENT;
  if (cls->E != topo->E)
    return set_error(ctx, PHFEM_ERR_MISMATCH,
                     "assemble_constraint: classification does not match topology");
  return constraint_csr_into(ctx, mesh, topo, cls, out);
}

PHFEM_API void phfem_csr_release(phfem_ctx* ctx, phfem_csr* m) {
  if (!m) return;
  dfree(ctx, m->row_ptr);
  dfree(ctx, m->col_idx);
  dfree(ctx, m->values);
  m->nnz = 0;
}

PHFEM_API phfem_status phfem_constraint_csc(phfem_ctx* ctx, const phfem_mesh* mesh,
                                            const phfem_topology* topo,
                                            const phfem_classification* cls, phfem_csc* out) {
  memset(out, 0, sizeof(*out));
  if (!ctx || !mesh || !topo || !cls) return PHFEM_ERR_INVALID_ARGUMENT;
  if (cls->E != topo->E)
    return set_error(ctx, PHFEM_ERR_MISMATCH,
                     "assemble_constraint: classification does not match topology");
  const int64_t N = 3 * (int64_t)mesh->nE;
  out->rows = cls->L;
  out->cols = (int32_t)N;
  const int64_t bret_total = (int64_t)topo->n_boundary - (int64_t)(topo->E - cls->L);
  out->nnz = 4 * (int64_t)cls->L - 2 * bret_total;
  PHFEM_TRY(dalloc(ctx, &out->outer, N + 1));
  PHFEM_TRY(dalloc(ctx, &out->inner, out->nnz));
  PHFEM_TRY(dalloc(ctx, &out->values, out->nnz));
  PHFEM_CUDA(ctx, cudaMemsetAsync(out->outer + N, 0, sizeof(int32_t), ctx->stream));
  if (N > 0) {
    PHFEM_LAUNCH(ctx, "k_csc_count", k_csc_count<<<grid_for(mesh->nE, 256, ctx->num_sms * 16), 256, 0, ctx->stream>>>(
        topo->elem_edge, cls->retained_pos, mesh->nE, out->outer));
  }
  PHFEM_TRY(scan_exclusive_i32(ctx, out->outer, out->outer, N + 1, nullptr));
  if (N > 0) {
    PHFEM_LAUNCH(ctx, "k_csc_fill", k_csc_fill<<<grid_for(mesh->nE, 256, ctx->num_sms * 16), 256, 0, ctx->stream>>>(
        (const double2*)mesh->coords, mesh->elements, topo->elem_edge, cls->retained_pos,
        mesh->nE, out->outer, out->inner, out->values));
  }
  return PHFEM_OK;
}

PHFEM_API void phfem_csc_release(phfem_ctx* ctx, phfem_csc* m) {
  if (!m) return;
  dfree(ctx, m->outer);
  dfree(ctx, m->inner);
  dfree(ctx, m->values);
  m->nnz = 0;
}

PHFEM_API phfem_status phfem_assemble_neumann(phfem_ctx* ctx, const phfem_mesh* mesh,
                                              const phfem_topology* topo,
                                              const phfem_classification* cls,
                                              const phfem_field* g, double t, double* out,
                                              int accumulate) {
  if (!ctx || !mesh || !topo || !cls || !g) return PHFEM_ERR_INVALID_ARGUMENT;
  if (!accumulate && mesh->nE > 0)
    PHFEM_CUDA(ctx, cudaMemsetAsync(out, 0, sizeof(double) * 3 * (int64_t)mesh->nE, ctx->stream));
  return neumann_into(ctx, mesh, topo, cls, g, t, out, accumulate, true);
}

PHFEM_API phfem_status phfem_assemble_dirichlet(phfem_ctx* ctx, const phfem_mesh* mesh,
                                                const phfem_topology* topo,
                                                const phfem_classification* cls,
                                                const phfem_field* uD, double t, double* out) {
  if (!ctx || !mesh || !topo || !cls || !uD) return PHFEM_ERR_INVALID_ARGUMENT;
  return dirichlet_into(ctx, mesh, topo, cls, uD, t, out);
}

PHFEM_API phfem_status phfem_dist_dirichlet(phfem_ctx* ctx, const phfem_mesh* mesh, const phfem_topology* part,
                                            const phfem_classification* cls, const phfem_field* uD, double t,
                                            int32_t r_off, double* out) {
  if (!ctx || !mesh || !part || !cls || !uD || (cls->L > 0 && !out) || r_off < 0) return PHFEM_ERR_INVALID_ARGUMENT;
  return phfem::dirichlet_into(ctx, mesh, part, cls, uD, t, out, nullptr, r_off);
}
