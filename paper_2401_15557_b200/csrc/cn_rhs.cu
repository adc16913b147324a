// cn_rhs.cu — the Crank-Nicolson right-hand side on sm_100a.
//
// Reference: solve_parabolic forms, for the step t_n -> t_{n+1}
// (proj/src/parabolic.cpp:95-103),
//     rhs = M_minus * W;  rhs.head += k*0.5 * (((b^n + LN^n) + b^{n+1}) + LN^{n+1});
//     rhs.tail += 0.5 * (bD^n + bD^{n+1})
// with M_minus = step_matrix(ops, k, -1) (parabolic.cpp:21-37): the top block
// M0 + (-(k/2)) ((B + D) + M), the coupling (k/2) C' in the primal rows and
// (1/2) C in the multiplier rows, each entry stored as 0.0 + value by
// from_triplets.  Eigen's column-major SpMV accumulates each row from 0 in
// ascending column order.
//
// Device version.  The plan (phfem_cn_plan_create) stores, once, everything of
// an element that depends on neither t nor W — the M_minus top block as
// from_triplets stores it, the coupling entries, the load weight, sin(pi x) and
// sin(pi y) at the three edge midpoints (sin-sin loads), the multiplier row of
// each edge slot — and one record per multiplier row (T+ / T- DOF bases and
// locals, |E|/2), all computed with the assembly's own expressions.  Per step:
//   * k_cn_tma: the primal rows, one thread per element; the element records
//     and U stream through a 4-stage SMEM ring filled by cp.async.bulk (TMA),
//     the Lambda gathers run two tiles ahead of the arithmetic;
//   * k_cn_rows: the multiplier rows from the row records (coalesced), U of
//     T+ / T- gathered;
//   * k_cn_edges over the Dirichlet list only (the rows with u_D data);
//   * Neumann data through the per-element table of assemble.cu.
// Other load kinds take k_cn_elements (geometry recomputed every step) +
// k_cn_edges over all edges.
#include <algorithm>
#include <cstdlib>
#include <cmath>

#include "bulk.cuh"
#include "common.cuh"
#include "elem.cuh"
#include "kernels.cuh"

struct phfem_cn_plan {
  phfem_mesh mesh;
  phfem_topology topo;
  phfem_classification cls;
  phfem_coeffs c;
  phfem_field f, g, uD;
  double k;
  phfem::NeuTable neu;
  double* neu_vals0 = nullptr;  // [cap][3] LN at t_n
  double* neu_vals1 = nullptr;  // [cap][3] LN at t_{n+1}
  uint32_t* dir_bits = nullptr; // Dirichlet edge bitmap
  // stored-operator path (sin-sin / zero loads): the time-independent parts of
  // every element, computed once by k_cn_pre with the assembly's expressions
  double* top = nullptr;  // [nE][9] M_minus top-block entries as stored: 0.0 + (M0 + s((B+D)+M))
  double* cpl = nullptr;  // [nE][3] C' entries of the element's edge slots: 0.0 + s_ct (+-|E|/2)
  // [nE][3] load factor of each primal row: w (g[i+1] + g[i+2]) with
  // w = (|T|/3) 0.5 and g[k] = sin(pi x_k) sin(pi y_k) at midpoint k, so the
  // sin-sin load of row i at time t is c(t) lq[i] (24 B instead of a 48-B
  // sin table + 8-B weight; reassociated: within 1e-12, no sign change of g
  // inside an element on the configured fields — SURVEY Appendix A)
  double* lq = nullptr;
  int32_t* rp3 = nullptr; // [nE][3] (multiplier row << 1) | (element is T-) per edge slot, -1 if not retained
  // multiplier rows, one record per retained edge l (row order): T+ as
  // 4 t_plus + local, T- as 4 t_minus + local (kRowBnd / kRowDir on the
  // boundary), and |E| * 0.5
  uint2* rowt = nullptr;
  double* rowh = nullptr;
  bool hybrid = false;  // k_cn_hyb (top block + coupling recomputed) instead of k_cn_tma
};

namespace phfem {

struct CnArgs {
  const double2* coords;
  const int32_t* elements;
  const int32_t* elem_edge;
  const int32_t* edge_elements;
  const int32_t* ltm;
  const int32_t* rpos;
  const uint32_t* dir_bits;
  const int32_t* neu_keys;
  const double* neu0;
  const double* neu1;
  int neu_cap;
  int nE;
  int64_t N;
  phfem_coeffs c;
  phfem_field f, uD;
  double s_top;   // sign*(k/2.0), sign = -1        (parabolic.cpp:26)
  double s_ct;    // -sign*(k/2.0)                  (parabolic.cpp:34)
  double s_c;     // -sign*0.5                      (parabolic.cpp:35)
  double kh;      // k*0.5                          (parabolic.cpp:101)
  double t0, t1;
  int vec;
};

constexpr int kCnThreads = 128;
// k_cn_rows grid (measured at L11: 8 CTAs per SM 0.099 ms; 32 / 128 / 1024
// per SM 0.106 / 0.107 / 0.111 ms; two rows per trip with the six U values
// loaded unconditionally: 0.107 ms)
#ifndef PHFEM_CNR_GRID_MULT
#define PHFEM_CNR_GRID_MULT 8
#endif
#ifndef PHFEM_CN_MIN_BLOCKS
#define PHFEM_CN_MIN_BLOCKS 1
#endif

__device__ __forceinline__ int neu_lookup(const int32_t* __restrict__ keys, int cap, int m) {
  if (cap == 0) return -1;
  uint32_t h = neu_hash(m, cap);
  while (true) {
    const int k = keys[h];
    if (k == m) return (int)h;
    if (k < 0) return -1;
    h = (h + 1) & (uint32_t)(cap - 1);
  }
}

// sin(pi x) sin(pi y) at the 3 midpoints is shared by t_n and t_{n+1}: the
// EXP_SINSIN specialisation evaluates it once, then exp(-t) p0 * sx * sy for
// both times in the formula's own order (phfem_fields.h).
template <int FK>
__device__ __forceinline__ void field_pair(const phfem_field& f, double x, double y, double t0,
                                           double t1, double e0, double e1, double& f0, double& f1) {
  if (FK == PHFEM_FIELD_EXP_SINSIN) {
    const double sx = sin_fast(PHFEM_PI * x), sy = sin_fast(PHFEM_PI * y);
    f0 = e0 * sx * sy;
    f1 = e1 * sx * sy;
  } else {
    f0 = field_dev<FK>(f, x, y, t0);
    f1 = field_dev<FK>(f, x, y, t1);
  }
}

template <int FK, int CK>
__global__ void __launch_bounds__(kCnThreads, PHFEM_CN_MIN_BLOCKS) k_cn_elements(CnArgs a, const double* __restrict__ W,
                                                            double* __restrict__ rhs) {
  __shared__ __align__(16) double tile[kCnThreads * 3];
  const int64_t ntiles = ((int64_t)a.nE + kCnThreads - 1) / kCnThreads;
  for (int64_t tb = blockIdx.x; tb < ntiles; tb += gridDim.x) {
    const int64_t base = tb * kCnThreads;
    const int n_valid = (int)((int64_t)a.nE - base < kCnThreads ? (int64_t)a.nE - base : kCnThreads);
    const int64_t m = base + threadIdx.x;
    const bool valid = threadIdx.x < n_valid;
    double out3[3] = {0.0, 0.0, 0.0};
    if (valid) {
      const int t[3] = {__ldg(a.elements + 3 * m), __ldg(a.elements + 3 * m + 1),
                        __ldg(a.elements + 3 * m + 2)};
      const double2 v[3] = {__ldg(a.coords + t[0]), __ldg(a.coords + t[1]), __ldg(a.coords + t[2])};
      const double U[3] = {W[3 * m], W[3 * m + 1], W[3 * m + 2]};
      const phfem_coeff_values cv = coeffs_dev<CK>(a.c, v[0], v[1], v[2]);
      // the M_minus top block is formed entry by entry below (no 4 x 9 block
      // arrays in registers): the same expressions as phfem_stiffness /
      // convection_dev / phfem_mass / phfem_unit_mass, so the same bits
      const phfem_geom g = geometry_dev(v[0].x, v[0].y, v[1].x, v[1].y, v[2].x, v[2].y);
      double rx[3], ry[3], dj[3];
      const double a3 = div3(g.area);
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        rx[i] = cv.a00 * g.gx[i] + cv.a01 * g.gy[i];
        ry[i] = cv.a10 * g.gx[i] + cv.a11 * g.gy[i];
        dj[i] = a3 * (cv.px * g.gx[i] + cv.py * g.gy[i]);
      }
      const double md = cv.delta * g.area * (1.0 / 6.0), mo = cv.delta * g.area * (1.0 / 12.0);
      const double ud = g.area * (1.0 / 6.0), uo = g.area * (1.0 / 12.0);
      auto top = [&](int i, int j) {  // M0(i,j) + s ((B(i,j) + D(i,j)) + M(i,j))
        const int lo = i < j ? i : j, hi = i < j ? j : i;  // B from the upper triangle
        const double bij = g.area * (rx[lo] * g.gx[hi] + ry[lo] * g.gy[hi]);
        const double mij = i == j ? md : mo;
        const double m0ij = i == j ? ud : uo;
        return m0ij + a.s_top * ((bij + dj[j]) + mij);
      };

      // edges of m: id, orientation, multiplier row, length
      int e[3], rp[3];
      bool plus[3];
      double len[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const int s = __ldg(a.elem_edge + 3 * m + k);
        plus[k] = s >= 0;
        e[k] = s >= 0 ? s : ~s;
        rp[k] = a.rpos[e[k]];
        const double2 pa = v[(k + 1) % 3], pb = v[(k + 2) % 3];
        const double dx = pb.x - pa.x, dy = pb.y - pa.y;
        len[k] = sqrt(dx * dx + dy * dy);
      }
      double lam[3], cval[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        lam[k] = rp[k] >= 0 ? W[a.N + rp[k]] : 0.0;
        const double C = plus[k] ? len[k] * 0.5 : -len[k] * 0.5;  // assembly.cpp:160,164
        cval[k] = 0.0 + a.s_ct * C;
      }

      // loads at t_n, t_{n+1} (load_at_time = assemble_load + assemble_neumann)
      double b0[3], b1[3], l0[3] = {0.0, 0.0, 0.0}, l1[3] = {0.0, 0.0, 0.0};
      {
        const double mx[3] = {0.5 * (v[1].x + v[2].x), 0.5 * (v[2].x + v[0].x), 0.5 * (v[0].x + v[1].x)};
        const double my[3] = {0.5 * (v[1].y + v[2].y), 0.5 * (v[2].y + v[0].y), 0.5 * (v[0].y + v[1].y)};
        const double area =
            0.5 * ((v[1].x - v[0].x) * (v[2].y - v[0].y) - (v[1].y - v[0].y) * (v[2].x - v[0].x));
        double f0[3], f1[3];
        const double e0 = exp(-a.t0) * a.f.p[0], e1 = exp(-a.t1) * a.f.p[0];
#pragma unroll
        for (int i = 0; i < 3; ++i) field_pair<FK>(a.f, mx[i], my[i], a.t0, a.t1, e0, e1, f0[i], f1[i]);
        const double w = div3(area) * 0.5;  // area / 3.0 * 0.5 (assembly.cpp:199)
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          b0[i] = 0.0 + w * (f0[(i + 1) % 3] + f0[(i + 2) % 3]);
          b1[i] = 0.0 + w * (f1[(i + 1) % 3] + f1[(i + 2) % 3]);
        }
        const int slot = neu_lookup(a.neu_keys, a.neu_cap, (int)m);
        if (slot >= 0) {
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            l0[i] = a.neu0[3 * slot + i];
            l1[i] = a.neu1[3 * slot + i];
          }
        }
      }

      // primal rows 3m+i
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < 3; ++j) acc += (0.0 + 1.0 * top(i, j)) * U[j];
        int ka = (i + 1) % 3, kb = (i + 2) % 3;  // edges with R[k][i] != 0
        if (rp[kb] >= 0 && (rp[ka] < 0 || rp[kb] < rp[ka])) {
          const int x = ka;
          ka = kb;
          kb = x;
        }
        if (rp[ka] >= 0) acc += cval[ka] * lam[ka];
        if (rp[kb] >= 0) acc += cval[kb] * lam[kb];
        out3[i] = acc + a.kh * (((b0[i] + l0[i]) + b1[i]) + l1[i]);
      }

    }
    // coalesced store of the primal rows
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 3; ++i) tile[threadIdx.x * 3 + i] = out3[i];
    __syncthreads();
    const int count = n_valid * 3;
    double* dst = rhs + base * 3;
    if (a.vec) {
      const double2* s2 = reinterpret_cast<const double2*>(tile);
      double2* d2 = reinterpret_cast<double2*>(dst);
      for (int i = threadIdx.x; i < count / 2; i += blockDim.x) d2[i] = s2[i];
      if ((count & 1) && threadIdx.x == 0) dst[count - 1] = tile[count - 1];
    } else {
      for (int i = threadIdx.x; i < count; i += blockDim.x) dst[i] = tile[i];
    }
  }
}

// ---- stored-operator path ---------------------------------------------------------
// Once per plan: everything of an element that does not depend on t or W.
template <int CK>
__global__ void __launch_bounds__(kCnThreads) k_cn_pre(CnArgs a, double* __restrict__ top,
                                                        double* __restrict__ cpl, double* __restrict__ lq,
                                                        int32_t* __restrict__ rp3) {
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < a.nE;
       m += (int64_t)gridDim.x * blockDim.x) {
    const double2 v[3] = {a.coords[a.elements[3 * m]], a.coords[a.elements[3 * m + 1]],
                          a.coords[a.elements[3 * m + 2]]};
    const phfem_coeff_values cv = coeffs_dev<CK>(a.c, v[0], v[1], v[2]);
    const phfem_geom g = geometry_dev(v[0].x, v[0].y, v[1].x, v[1].y, v[2].x, v[2].y);
    const double a3 = div3(g.area);
    double rx[3], ry[3], dj[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      rx[i] = cv.a00 * g.gx[i] + cv.a01 * g.gy[i];
      ry[i] = cv.a10 * g.gx[i] + cv.a11 * g.gy[i];
      dj[i] = a3 * (cv.px * g.gx[i] + cv.py * g.gy[i]);
    }
    const double md = cv.delta * g.area * (1.0 / 6.0), mo = cv.delta * g.area * (1.0 / 12.0);
    const double ud = g.area * (1.0 / 6.0), uo = g.area * (1.0 / 12.0);
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const int lo = i < j ? i : j, hi = i < j ? j : i;  // B from the upper triangle
        const double bij = g.area * (rx[lo] * g.gx[hi] + ry[lo] * g.gy[hi]);
        const double t = (i == j ? ud : uo) + a.s_top * ((bij + dj[j]) + (i == j ? md : mo));
        top[9 * m + 3 * j + i] = 0.0 + 1.0 * t;  // from_triplets stores 0.0 + value
      }
    double gk[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double2 pa = v[(k + 1) % 3], pb = v[(k + 2) % 3];
      const double dx = pb.x - pa.x, dy = pb.y - pa.y;
      const double len = sqrt(dx * dx + dy * dy);
      const int se = a.elem_edge[3 * m + k];
      const bool plus = se >= 0;
      cpl[3 * m + k] = 0.0 + a.s_ct * (plus ? len * 0.5 : -len * 0.5);  // assembly.cpp:160,164
      const int rp = a.rpos[plus ? se : ~se];
      rp3[3 * m + k] = rp >= 0 ? (rp << 1) | (plus ? 0 : 1) : -1;  // row and the slot's C sign
      const double mx = 0.5 * (pa.x + pb.x), my = 0.5 * (pa.y + pb.y);
      gk[k] = sin_fast(PHFEM_PI * mx) * sin_fast(PHFEM_PI * my);
    }
    const double area = 0.5 * ((v[1].x - v[0].x) * (v[2].y - v[0].y) - (v[1].y - v[0].y) * (v[2].x - v[0].x));
    const double w = div3(area) * 0.5;  // assembly.cpp:199
#pragma unroll
    for (int i = 0; i < 3; ++i) lq[3 * m + i] = w * (gk[(i + 1) % 3] + gk[(i + 2) % 3]);
  }
}

constexpr uint32_t kRowBnd = 0xffffffffu;  // boundary edge, no Dirichlet data
constexpr uint32_t kRowDir = 0xfffffffeu;  // Dirichlet edge: row written by k_cn_edges

// Once per plan: the record of every multiplier row (row order = retained order)
__global__ void k_cn_rows_pre(CnArgs a, const int32_t* __restrict__ edge_nodes,
                              const int32_t* __restrict__ ltp, int E, uint2* __restrict__ rowt,
                              double* __restrict__ rowh) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int rp = a.rpos[e];
    if (rp < 0) continue;
    const int2 ab = reinterpret_cast<const int2*>(edge_nodes)[e];
    const int2 el = reinterpret_cast<const int2*>(a.edge_elements)[e];
    const double2 pa = a.coords[ab.x], pb = a.coords[ab.y];
    const double dx = pb.x - pa.x, dy = pb.y - pa.y;
    const double len = sqrt(dx * dx + dy * dy);  // edge_topology.cpp:183
    uint32_t y;
    if (el.y >= 0) y = 4u * (uint32_t)el.y + (uint32_t)a.ltm[e];
    else y = ((a.dir_bits[e >> 5] >> (e & 31)) & 1u) ? kRowDir : kRowBnd;
    rowt[rp] = make_uint2(4u * (uint32_t)el.x + (uint32_t)ltp[e], y);
    rowh[rp] = len * 0.5;
  }
}

// Primal rows 3m+i of one element from its stored record (shared by the TMA
// and the plain-load kernels: one expression, one set of bits).
__device__ __forceinline__ void cn_primal(const CnArgs& a, int64_t m, const double (&T)[9],
                                          const double (&lq)[3], const double (&cv3)[3], const double (&U)[3],
                                          const int (&rp)[3], const double (&lam)[3], double c0, double c1,
                                          double (&out3)[3]) {
  double l0[3] = {0.0, 0.0, 0.0}, l1[3] = {0.0, 0.0, 0.0};
  // LN data only on elements with a Neumann edge, i.e. a non-retained one
  // (retained = non-Neumann, edge_topology.cpp:165-173): no probe otherwise
  const int slot = (rp[0] < 0 || rp[1] < 0 || rp[2] < 0) ? neu_lookup(a.neu_keys, a.neu_cap, (int)m) : -1;
  if (slot >= 0) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      l0[i] = a.neu0[3 * slot + i];
      l1[i] = a.neu1[3 * slot + i];
    }
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < 3; ++j) acc += T[3 * j + i] * U[j];
    int ka = (i + 1) % 3, kb = (i + 2) % 3;  // edges with R[k][i] != 0, ascending rows
    if (rp[kb] >= 0 && (rp[ka] < 0 || rp[kb] < rp[ka])) {
      const int x = ka;
      ka = kb;
      kb = x;
    }
    if (rp[ka] >= 0) acc += cv3[ka] * lam[ka];
    if (rp[kb] >= 0) acc += cv3[kb] * lam[kb];
    // assemble_load's 0.0 + w (f[i+1] + f[i+2]) at t_n and t_{n+1} (assembly.cpp:199)
    const double b0 = 0.0 + c0 * lq[i];
    const double b1 = 0.0 + c1 * lq[i];
    out3[i] = acc + a.kh * (((b0 + l0[i]) + b1) + l1[i]);
  }
}

struct CnStored {
  const double* top;
  const double* cpl;
  const double* lq;
  const int32_t* rp3;
};

// warp-cooperative coalesced load of a per-element record of `per` elements
// of T for the warp's 32 consecutive elements into SMEM (stride `per`)
template <typename T>
__device__ __forceinline__ void warp_load(const T* __restrict__ g, int64_t base, int n_valid, int per,
                                          T* buf) {
  const int lane = threadIdx.x & 31;
  const int count = n_valid * per;
  const T* src = g + base * per;
  for (int i = lane; i < count; i += 32) buf[i] = __ldg(src + i);
  __syncwarp();
}

// Plain-load variant: elements [m0, nE) by warps of 32 (the tail tile of the
// TMA kernel, or everything when the state / rhs are not 16-byte aligned).
__global__ void __launch_bounds__(kCnThreads) k_cn_stored(CnArgs a, CnStored st, int64_t m0, double c0,
                                                          double c1, const double* __restrict__ W,
                                                          double* __restrict__ rhs) {
  __shared__ __align__(16) double sbuf[kCnThreads / 32][32 * 9];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* buf = sbuf[warp];
  const int64_t nchunks = ((int64_t)a.nE - m0 + 31) / 32;
  for (int64_t ch = (int64_t)blockIdx.x * (kCnThreads / 32) + warp; ch < nchunks;
       ch += (int64_t)gridDim.x * (kCnThreads / 32)) {
    const int64_t base = m0 + ch * 32;
    const int n_valid = (int)((int64_t)a.nE - base < 32 ? (int64_t)a.nE - base : 32);
    const int64_t m = base + lane;
    const bool valid = lane < n_valid;
    __syncwarp();
    warp_load(st.top, base, n_valid, 9, buf);
    double T[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) T[q] = valid ? buf[9 * lane + q] : 0.0;
    __syncwarp();
    warp_load(st.lq, base, n_valid, 3, buf);
    double lq[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) lq[k] = valid ? buf[3 * lane + k] : 0.0;
    __syncwarp();
    warp_load(st.cpl, base, n_valid, 3, buf);
    double cv3[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) cv3[k] = valid ? buf[3 * lane + k] : 0.0;
    __syncwarp();
    warp_load(W, base, n_valid, 3, buf);  // U of the warp's elements
    double out3[3] = {0.0, 0.0, 0.0};
    if (valid) {
      const double U[3] = {buf[3 * lane], buf[3 * lane + 1], buf[3 * lane + 2]};
      int rp[3];
      double lam[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) rp[k] = __ldg(st.rp3 + 3 * m + k) >> 1;  // -1 stays -1
#pragma unroll
      for (int k = 0; k < 3; ++k) lam[k] = rp[k] >= 0 ? W[a.N + rp[k]] : 0.0;
      cn_primal(a, m, T, lq, cv3, U, rp, lam, c0, c1, out3);
    }
    // coalesced store through the warp's SMEM slice
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 3; ++i) buf[3 * lane + i] = out3[i];
    __syncwarp();
    double* dst = rhs + base * 3;
    for (int i = lane; i < n_valid * 3; i += 32) dst[i] = buf[i];
  }
}

// TMA variant over the full 128-element tiles: one elected thread streams each
// tile's stored record (top 72, load factors 24, coupling 24, U 24, rows 12:
// 156 bytes / element) into a kCnStages-deep SMEM ring with cp.async.bulk
// (evict-first), completion on one mbarrier per stage; the threads read their
// element's record from SMEM (odd strides / 16-byte pairs: conflict-free) and
// only the Lambda and Neumann lookups stay as gathers.
constexpr int kCnTile = 128;
constexpr int kCnStages = 4;
struct CnStage {
  double top[9 * kCnTile];
  double lq[3 * kCnTile];
  double cpl[3 * kCnTile];
  double U[3 * kCnTile];
  int32_t rp[3 * kCnTile];
};
static_assert(sizeof(CnStage) % 16 == 0, "bulk copies need 16-byte granules");
constexpr size_t kCnTmaSmem = kCnStages * sizeof(CnStage) + 3 * kCnTile * sizeof(double) +
                              kCnStages * sizeof(uint64_t);

__global__ void __launch_bounds__(kCnTile) k_cn_tma(CnArgs a, CnStored st, int64_t ntiles, double c0,
                                                     double c1, const double* __restrict__ W,
                                                     double* __restrict__ rhs) {
  extern __shared__ __align__(128) unsigned char cn_smem[];
  CnStage* stg = reinterpret_cast<CnStage*>(cn_smem);
  double* outb = reinterpret_cast<double*>(cn_smem + kCnStages * sizeof(CnStage));
  uint64_t* bar = reinterpret_cast<uint64_t*>(outb + 3 * kCnTile);
  const int tid = threadIdx.x;
  const int64_t my = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  uint64_t pol = 0;
  auto issue = [&](int64_t i) {
    const int s = (int)(i % kCnStages);
    const int64_t base = ((int64_t)blockIdx.x + i * gridDim.x) * kCnTile;
    mbar_expect_tx(&bar[s], (unsigned)sizeof(CnStage));
    bulk_load(stg[s].top, st.top + 9 * base, 9 * kCnTile * 8, &bar[s], pol);
    bulk_load(stg[s].lq, st.lq + 3 * base, 3 * kCnTile * 8, &bar[s], pol);
    bulk_load(stg[s].cpl, st.cpl + 3 * base, 3 * kCnTile * 8, &bar[s], pol);
    bulk_load(stg[s].U, W + 3 * base, 3 * kCnTile * 8, &bar[s], pol);
    bulk_load(stg[s].rp, st.rp3 + 3 * base, 3 * kCnTile * 4, &bar[s], pol);
  };
  if (tid == 0) {
    for (int s = 0; s < kCnStages; ++s) mbar_init(&bar[s], 1);
    mbar_fence_init();
    pol = policy_evict_first();
    for (int64_t i = 0; i < my && i < kCnStages; ++i) issue(i);
  }
  __syncthreads();
  // the Lambda gathers run two tiles ahead of the arithmetic (their rows come
  // with the tile's stage), so their latency overlaps two tiles of work
  int rpq[2][3];
  double lamq[2][3];
  auto gather = [&](int64_t j, int (&rp)[3], double (&lam)[3]) {
    const int sj = (int)(j % kCnStages);
    mbar_wait(&bar[sj], (unsigned)((j / kCnStages) & 1));
#pragma unroll
    for (int k = 0; k < 3; ++k) rp[k] = stg[sj].rp[3 * tid + k] >> 1;  // -1 stays -1
#pragma unroll
    for (int k = 0; k < 3; ++k) lam[k] = rp[k] >= 0 ? __ldg(W + a.N + rp[k]) : 0.0;
  };
#pragma unroll
  for (int d = 0; d < 2; ++d)
    if (d < my) gather(d, rpq[d], lamq[d]);
  for (int64_t i = 0; i < my; ++i) {
    const int s = (int)(i % kCnStages);
    const int64_t base = ((int64_t)blockIdx.x + i * gridDim.x) * kCnTile;
    const int64_t m = base + tid;
    const CnStage& S = stg[s];
    int rp[3];
    double lam[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      rp[k] = rpq[0][k];
      lam[k] = lamq[0][k];
      rpq[0][k] = rpq[1][k];
      lamq[0][k] = lamq[1][k];
    }
    if (i + 2 < my) gather(i + 2, rpq[1], lamq[1]);
    double T[9], lq[3], cv3[3];
    const double U[3] = {S.U[3 * tid], S.U[3 * tid + 1], S.U[3 * tid + 2]};
#pragma unroll
    for (int q = 0; q < 9; ++q) T[q] = S.top[9 * tid + q];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      lq[k] = S.lq[3 * tid + k];
      cv3[k] = S.cpl[3 * tid + k];
    }
    double out3[3];
    cn_primal(a, m, T, lq, cv3, U, rp, lam, c0, c1, out3);
#pragma unroll
    for (int q = 0; q < 3; ++q) outb[3 * tid + q] = out3[q];
    __syncthreads();  // stage s consumed, tile results staged
    if (tid == 0 && i + kCnStages < my) issue(i + kCnStages);
    const double2* s2 = reinterpret_cast<const double2*>(outb);
    double2* d2 = reinterpret_cast<double2*>(rhs + 3 * base);
    for (int q = tid; q < 3 * kCnTile / 2; q += kCnTile) __stcs(d2 + q, s2[q]);
    __syncthreads();  // outb free for the next tile
  }
}

// (Measured and dropped at L11: streaming the plan's coupling entries through
// the ring instead of recomputing three edge lengths per element, 0.254 ->
// 0.267 ms; 5 CTAs per SM do not fit the ring.)
// Hybrid variant (the default when the coordinates fit in L2): the M_minus
// top block and the coupling entries are recomputed from the geometry with
// the plan's own expressions (same bits as k_cn_pre), so per element only
// the elements (12 B), the load factors (24), U (24) and the row codes (12)
// stream through the TMA ring — 72 B instead of 156 — and the coordinates
// are gathered (L2-resident: 16 nC bytes).  Coordinates and Lambda of tile
// i + 2 are gathered while tile i computes.
struct CnHStage {
  int32_t el[3 * kCnTile];
  double lq[3 * kCnTile];
  double U[3 * kCnTile];
  int32_t rp[3 * kCnTile];
};
static_assert(sizeof(CnHStage) % 16 == 0, "bulk copies need 16-byte granules");
constexpr int kCnHStages = 4;
constexpr size_t kCnHybSmem = kCnHStages * sizeof(CnHStage) + 3 * kCnTile * sizeof(double) +
                              kCnHStages * sizeof(uint64_t);

struct CnHQueue {
  double2 v[3];
  double lam[3];
  int rpx[3];
};

#ifndef PHFEM_CN_HYB_BLOCKS
#define PHFEM_CN_HYB_BLOCKS 4
#endif
template <int CK>
__global__ void __launch_bounds__(kCnTile, PHFEM_CN_HYB_BLOCKS) k_cn_hyb(CnArgs a, CnStored st, int64_t ntiles, double c0,
                                                     double c1, const double* __restrict__ W,
                                                     double* __restrict__ rhs) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(128) unsigned char cn_smem[];
  CnHStage* stg = reinterpret_cast<CnHStage*>(cn_smem);
  double* outb = reinterpret_cast<double*>(cn_smem + kCnHStages * sizeof(CnHStage));
  uint64_t* bar = reinterpret_cast<uint64_t*>(outb + 3 * kCnTile);
  const int tid = threadIdx.x;
  const int64_t my = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  uint64_t pol = 0, pol_u = 0;
  auto issue = [&](int64_t i) {
    const int s = (int)(i % kCnHStages);
    const int64_t base = ((int64_t)blockIdx.x + i * gridDim.x) * kCnTile;
    mbar_expect_tx(&bar[s], (unsigned)sizeof(CnHStage));
    bulk_load(stg[s].el, a.elements + 3 * base, 3 * kCnTile * 4, &bar[s], pol);
    bulk_load(stg[s].lq, st.lq + 3 * base, 3 * kCnTile * 8, &bar[s], pol);
    bulk_load(stg[s].U, W + 3 * base, 3 * kCnTile * 8, &bar[s], pol_u);
    bulk_load(stg[s].rp, st.rp3 + 3 * base, 3 * kCnTile * 4, &bar[s], pol);
  };
  if (tid == 0) {
    for (int s = 0; s < kCnHStages; ++s) mbar_init(&bar[s], 1);
    mbar_fence_init();
    pol = policy_evict_first();
    // U stays in L2 for the multiplier-row pass that follows (its U gathers:
    // rows 0.099 -> 0.096 ms at L11)
    pol_u = policy_evict_last();
    for (int64_t i = 0; i < my && i < kCnHStages; ++i) issue(i);
  }
  __syncthreads();
  CnHQueue q0, q1;
  auto gather = [&](int64_t j, CnHQueue& q) {
    const int sj = (int)(j % kCnHStages);
    mbar_wait(&bar[sj], (unsigned)((j / kCnHStages) & 1));
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      q.v[k] = __ldg(a.coords + stg[sj].el[3 * tid + k]);
      q.rpx[k] = stg[sj].rp[3 * tid + k];
      q.lam[k] = q.rpx[k] >= 0 ? __ldg(W + a.N + (q.rpx[k] >> 1)) : 0.0;
    }
  };
  if (my > 0) gather(0, q0);
  if (my > 1) gather(1, q1);
  for (int64_t i = 0; i < my; ++i) {
    const int s = (int)(i % kCnHStages);
    const int64_t base = ((int64_t)blockIdx.x + i * gridDim.x) * kCnTile;
    const int64_t m = base + tid;
    const CnHStage& S = stg[s];
    const double2 v[3] = {q0.v[0], q0.v[1], q0.v[2]};
    const double lamv[3] = {q0.lam[0], q0.lam[1], q0.lam[2]};
    const int rpx[3] = {q0.rpx[0], q0.rpx[1], q0.rpx[2]};
    q0 = q1;
    if (i + 2 < my) gather(i + 2, q1);
    // the plan's k_cn_pre expressions (bit-identical top block / coupling)
    const phfem_coeff_values cv = coeffs_dev<CK>(a.c, v[0], v[1], v[2]);
    const phfem_geom g = geometry_dev(v[0].x, v[0].y, v[1].x, v[1].y, v[2].x, v[2].y);
    const double a3 = div3(g.area);
    double rx[3], ry[3], dj[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      rx[k] = cv.a00 * g.gx[k] + cv.a01 * g.gy[k];
      ry[k] = cv.a10 * g.gx[k] + cv.a11 * g.gy[k];
      dj[k] = a3 * (cv.px * g.gx[k] + cv.py * g.gy[k]);
    }
    const double md = cv.delta * g.area * (1.0 / 6.0), mo = cv.delta * g.area * (1.0 / 12.0);
    const double ud = g.area * (1.0 / 6.0), uo = g.area * (1.0 / 12.0);
    double T[9];
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int i2 = 0; i2 < 3; ++i2) {
        const int lo = i2 < j ? i2 : j, hi = i2 < j ? j : i2;  // B from the upper triangle
        const double bij = g.area * (rx[lo] * g.gx[hi] + ry[lo] * g.gy[hi]);
        const double t = (i2 == j ? ud : uo) + a.s_top * ((bij + dj[j]) + (i2 == j ? md : mo));
        // from_triplets stores 0.0 + value; that only turns -0 into +0, and
        // T / cv3 feed nothing but products added to an accumulator that
        // starts at +0.0 — a +-0 product leaves it unchanged either way, so
        // the add is dropped (same bits; hybrid pass
        // 0.254 -> 0.249 ms at L11)
        T[3 * j + i2] = t;
      }
    double cv3[3], lq[3];
    int rp[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double2 pa = v[(k + 1) % 3], pb = v[(k + 2) % 3];
      const double dx = pb.x - pa.x, dy = pb.y - pa.y;
      const double len = sqrt(dx * dx + dy * dy);
      cv3[k] = a.s_ct * ((rpx[k] & 1) ? -len * 0.5 : len * 0.5);  // assembly.cpp:160,164 (0.0 + dropped, above)
      rp[k] = rpx[k] >> 1;  // -1 stays -1
      lq[k] = S.lq[3 * tid + k];
    }
    const double U[3] = {S.U[3 * tid], S.U[3 * tid + 1], S.U[3 * tid + 2]};
    double out3[3];
    cn_primal(a, m, T, lq, cv3, U, rp, lamv, c0, c1, out3);
#pragma unroll
    for (int k = 0; k < 3; ++k) outb[3 * tid + k] = out3[k];
    __syncthreads();  // stage s consumed, tile results staged
    if (tid == 0 && i + kCnHStages < my) issue(i + kCnHStages);
    const double2* s2 = reinterpret_cast<const double2*>(outb);
    double2* d2 = reinterpret_cast<double2*>(rhs + 3 * base);
    for (int k = tid; k < 3 * kCnTile / 2; k += kCnTile) __stcs(d2 + k, s2[k]);
    __syncthreads();  // outb free for the next tile
  }
}

// Multiplier rows from the stored row records (coalesced), except the
// Dirichlet ones: row l = 0.0 + sum over ascending columns — T+ DOFs, then T-
// DOFs — of (0.0 + (-sign/2) C_lj) U_j (Eigen ColMajor SpMV, from_triplets'
// 0.0 +), + 0.5 (0.0 + 0.0) (parabolic.cpp:103 with no Dirichlet data).
__global__ void __launch_bounds__(256) k_cn_rows(const uint2* __restrict__ rowt, const double* __restrict__ rowh,
                                                  int L, double s_c, const double* __restrict__ W,
                                                  double* __restrict__ rhs_rows) {
  pdl_wait();
  pdl_trigger();
  // (measured: walking the rows backwards, towards the element tiles whose U
  // the hybrid pass loaded last, 0.096 -> 0.138 ms)
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < L;
       l += (int64_t)gridDim.x * blockDim.x) {
    const uint2 r = __ldcs(rowt + l);
    if (r.y == kRowDir) continue;
    const double h = __ldcs(rowh + l);
    const double cp = 0.0 + s_c * h;  // assembly.cpp:160
    const int64_t p = 3 * (int64_t)(r.x >> 2);
    const int lp = (int)(r.x & 3u);
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c)
      if (c != lp) acc += cp * __ldg(W + p + c);
    if (r.y != kRowBnd) {
      const int64_t q = 3 * (int64_t)(r.y >> 2);
      const int lm = (int)(r.y & 3u);
      const double cm = 0.0 + s_c * (-h);  // assembly.cpp:164: -len * 0.5 = -(len * 0.5)
#pragma unroll
      for (int c = 0; c < 3; ++c)
        if (c != lm) acc += cm * __ldg(W + q + c);
    }
    const double bdsum = 0.0 + 0.0;
    __stcs(rhs_rows + l, acc + 0.5 * bdsum);
  }
}

// Multiplier rows, one thread per edge (the retained ones write): row l of
// M_minus W is 0.0 + sum over the row's columns ascending — T+ DOFs, then T-
// DOFs (t_plus < t_minus) — of (0.0 + (-sign/2) C_lj) U_j (Eigen ColMajor
// SpMV, from_triplets' 0.0 +), then + 0.5 (bD^n + bD^{n+1}) (parabolic.cpp:103).
// With `ids` the edges are ids[0..E) (the Dirichlet list of the stored path).
__global__ void __launch_bounds__(256) k_cn_edges(CnArgs a, const int32_t* __restrict__ edge_nodes,
                                                   const int32_t* __restrict__ ltp, int E,
                                                   const int32_t* __restrict__ ids,
                                                   const double* __restrict__ W, double* __restrict__ rhs) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = ids ? ids[i] : i;
    const int rp = a.rpos[e];
    if (rp < 0) continue;
    const int2 ab = reinterpret_cast<const int2*>(edge_nodes)[e];
    const int2 el = reinterpret_cast<const int2*>(a.edge_elements)[e];
    const double2 pa = __ldg(a.coords + ab.x), pb = __ldg(a.coords + ab.y);
    const double dx = pb.x - pa.x, dy = pb.y - pa.y;
    const double len = sqrt(dx * dx + dy * dy);  // edge_topology.cpp:183
    const int l = ltp[e];
    const double cp = 0.0 + a.s_c * (len * 0.5);  // assembly.cpp:160
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c)
      if (c != l) acc += cp * W[3 * (int64_t)el.x + c];
    double bdsum = 0.0 + 0.0;
    if (el.y >= 0) {
      const int l2 = a.ltm[e];
      const double cm = 0.0 + a.s_c * (-len * 0.5);  // assembly.cpp:164
#pragma unroll
      for (int c = 0; c < 3; ++c)
        if (c != l2) acc += cm * W[3 * (int64_t)el.y + c];
    } else if ((a.dir_bits[e >> 5] >> (e & 31)) & 1u) {
      const double midx = 0.5 * (pa.x + pb.x), midy = 0.5 * (pa.y + pb.y);
      const double bd0 = -len * phfem_field_eval(&a.uD, midx, midy, a.t0);  // assembly.cpp:239
      const double bd1 = -len * phfem_field_eval(&a.uD, midx, midy, a.t1);
      bdsum = bd0 + bd1;
    }
    rhs[a.N + rp] = acc + 0.5 * bdsum;
  }
}

__global__ void k_set_bits(const int32_t* __restrict__ ids, int n, uint32_t* __restrict__ bits) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int e = ids[i];
    atomicOr(&bits[e >> 5], 1u << (e & 31));
  }
}

}  // namespace phfem

using namespace phfem;

PHFEM_API phfem_status phfem_cn_plan_create(phfem_ctx* ctx, const phfem_mesh* mesh,
                                            const phfem_topology* topo,
                                            const phfem_classification* cls, const phfem_coeffs* c,
                                            const phfem_field* f, const phfem_field* g,
                                            const phfem_field* uD, double k, phfem_cn_plan** out) {
  *out = nullptr;
  if (!ctx || !mesh || !topo || !cls || !c || !f || !g || !uD) return PHFEM_ERR_INVALID_ARGUMENT;
  if (!(k > 0.0))
    return set_error(ctx, PHFEM_ERR_INVALID_ARGUMENT, "step_matrices: k must be positive");
  if (cls->E != topo->E)
    return set_error(ctx, PHFEM_ERR_MISMATCH,
                     "assemble_constraint: classification does not match topology");
  phfem_cn_plan* p = new phfem_cn_plan();
  p->mesh = *mesh;
  p->topo = *topo;
  p->cls = *cls;
  p->c = *c;
  p->f = *f;
  p->g = *g;
  p->uD = *uD;
  p->k = k;
  phfem_status st = neu_table_build(ctx, topo, cls, &p->neu);
  if (st == PHFEM_OK && p->neu.cap > 0) {
    st = dalloc(ctx, &p->neu_vals0, 3 * (int64_t)p->neu.cap);
    if (st == PHFEM_OK) st = dalloc(ctx, &p->neu_vals1, 3 * (int64_t)p->neu.cap);
    if (st == PHFEM_OK) {
      cudaMemsetAsync(p->neu_vals0, 0, sizeof(double) * 3 * p->neu.cap, ctx->stream);
      cudaMemsetAsync(p->neu_vals1, 0, sizeof(double) * 3 * p->neu.cap, ctx->stream);
    }
  }
  const int nwords = (topo->E + 31) / 32;
  if (st == PHFEM_OK) st = dalloc(ctx, &p->dir_bits, std::max(nwords, 1));
  if (st == PHFEM_OK) {
    cudaMemsetAsync(p->dir_bits, 0, sizeof(uint32_t) * std::max(nwords, 1), ctx->stream);
    if (cls->nD > 0) {
      KTimer kt(ctx, "k_set_bits");
      k_set_bits<<<grid_for(cls->nD, 256, ctx->num_sms * 4), 256, 0, ctx->stream>>>(
          cls->dirichlet_edge_ids, cls->nD, p->dir_bits);
      ctx->launches++;
    }
    if (cudaGetLastError() != cudaSuccess) st = set_error(ctx, PHFEM_ERR_CUDA, "cn plan setup failed");
  }
  const bool sinsin = f->kind == PHFEM_FIELD_SINSIN || f->kind == PHFEM_FIELD_EXP_SINSIN ||
                      f->kind == PHFEM_FIELD_ZERO;
  if (st == PHFEM_OK && sinsin && mesh->nE > 0) {
    const int64_t nE = mesh->nE;
    // hybrid when the coordinates stay L2-resident (their gathers are then
    // nearly free); env PHFEM_CN_MODE=stored|hybrid overrides (A/B runs)
    p->hybrid = 16 * (int64_t)mesh->nC <= (int64_t)80 << 20;
    if (const char* md = getenv("PHFEM_CN_MODE")) p->hybrid = md[0] == 'h';

    st = dalloc(ctx, &p->top, 9 * nE);
    if (st == PHFEM_OK) st = dalloc(ctx, &p->cpl, 3 * nE);
    if (st == PHFEM_OK) st = dalloc(ctx, &p->lq, 3 * nE);
    if (st == PHFEM_OK) st = dalloc(ctx, &p->rp3, 3 * nE);
    if (st == PHFEM_OK && cls->L > 0) st = dalloc(ctx, &p->rowt, (int64_t)cls->L);
    if (st == PHFEM_OK && cls->L > 0) st = dalloc(ctx, &p->rowh, (int64_t)cls->L);
    if (st == PHFEM_OK) {
      CnArgs a;
      memset(&a, 0, sizeof a);
      a.coords = (const double2*)mesh->coords;
      a.elements = mesh->elements;
      a.elem_edge = topo->elem_edge;
      a.edge_elements = topo->edge_elements;
      a.ltm = topo->local_in_tminus;
      a.rpos = cls->retained_pos;
      a.dir_bits = p->dir_bits;
      a.nE = mesh->nE;
      a.c = *c;
      const double sign = -1.0;
      a.s_top = sign * (k / 2.0);
      a.s_ct = -sign * (k / 2.0);
      const int grid = grid_for(nE, kCnThreads, ctx->num_sms * 16);
      {
        KTimer kt(ctx, "k_cn_pre");
        if (c->kind == PHFEM_COEFF_CENTROID_POLY)
          k_cn_pre<PHFEM_COEFF_CENTROID_POLY><<<grid, kCnThreads, 0, ctx->stream>>>(a, p->top, p->cpl, p->lq, p->rp3);
        else
          k_cn_pre<PHFEM_COEFF_CONST><<<grid, kCnThreads, 0, ctx->stream>>>(a, p->top, p->cpl, p->lq, p->rp3);
        ctx->launches++;
      }
      if (cls->L > 0) {
        KTimer kt(ctx, "k_cn_rows_pre");
        k_cn_rows_pre<<<grid_for(topo->E, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
            a, topo->edge_nodes, topo->local_in_tplus, topo->E, p->rowt, p->rowh);
        ctx->launches++;
      }
      // (measured: the Dirichlet rows folded into k_cn_rows — a per-plan
      // midpoint table and the u_D evaluation inlined there — made it
      // 0.099 -> 0.138 ms: registers for every row; the 2-row k_cn_edges
      // launch stays)
      if (cudaGetLastError() != cudaSuccess) st = set_error(ctx, PHFEM_ERR_CUDA, "cn plan setup failed");
      if (st == PHFEM_OK) st = smem_optin(ctx, (const void*)k_cn_tma, kCnTmaSmem, "k_cn_tma smem opt-in");
      if (st == PHFEM_OK)
        st = smem_optin(ctx, (const void*)k_cn_hyb<PHFEM_COEFF_CONST>, kCnHybSmem, "k_cn_hyb smem opt-in");
      if (st == PHFEM_OK)
        st = smem_optin(ctx, (const void*)k_cn_hyb<PHFEM_COEFF_CENTROID_POLY>, kCnHybSmem, "k_cn_hyb smem opt-in");
    }
  }
  if (st != PHFEM_OK) {
    phfem_cn_plan_destroy(ctx, p);
    return st;
  }
  *out = p;
  return PHFEM_OK;
}

PHFEM_API void phfem_cn_plan_destroy(phfem_ctx* ctx, phfem_cn_plan* p) {
  if (!p) return;
  neu_table_free(ctx, &p->neu);
  dfree(ctx, p->neu_vals0);
  dfree(ctx, p->neu_vals1);
  dfree(ctx, p->dir_bits);
  dfree(ctx, p->top);
  dfree(ctx, p->cpl);
  dfree(ctx, p->lq);
  dfree(ctx, p->rp3);
  dfree(ctx, p->rowt);
  dfree(ctx, p->rowh);
  delete p;
}

PHFEM_API phfem_status phfem_cn_rhs(phfem_ctx* ctx, phfem_cn_plan* p, int n, const double* state,
                                    double* rhs) {
  if (!ctx || !p || n < 0) return PHFEM_ERR_INVALID_ARGUMENT;
  const double t0 = n * p->k;        // load_at_time: t = n * k (parabolic.cpp:61)
  const double t1 = (n + 1) * p->k;
  // g = 0: LN = (len * 0) kR = +0 every step — the zero-initialised values stand
  if (p->neu.nN > 0 && p->g.kind != PHFEM_FLUX_ZERO) {
    PHFEM_TRY(neu_table_eval(ctx, &p->neu, &p->mesh, &p->topo, &p->cls, &p->g, t0, p->neu_vals0));
    PHFEM_TRY(neu_table_eval(ctx, &p->neu, &p->mesh, &p->topo, &p->cls, &p->g, t1, p->neu_vals1));
  }
  CnArgs a;
  a.coords = (const double2*)p->mesh.coords;
  a.elements = p->mesh.elements;
  a.elem_edge = p->topo.elem_edge;
  a.edge_elements = p->topo.edge_elements;
  a.ltm = p->topo.local_in_tminus;
  a.rpos = p->cls.retained_pos;
  a.dir_bits = p->dir_bits;
  a.neu_keys = p->neu.keys;
  a.neu0 = p->neu_vals0;
  a.neu1 = p->neu_vals1;
  a.neu_cap = p->neu.cap;
  a.nE = p->mesh.nE;
  a.N = 3 * (int64_t)p->mesh.nE;
  a.c = p->c;
  a.f = p->f;
  a.uD = p->uD;
  const double sign = -1.0;
  a.s_top = sign * (p->k / 2.0);
  a.s_ct = -sign * (p->k / 2.0);
  a.s_c = -sign * 0.5;
  a.kh = p->k * 0.5;
  a.t0 = t0;
  a.t1 = t1;
  a.vec = (((uintptr_t)rhs) & 15u) == 0;
  if (a.nE > 0 && p->top) {
    // c = exp(-t) p0 / p0 / 0: the leading factor of the sin-sin formulas
    double c0 = 0.0, c1 = 0.0;
    if (a.f.kind == PHFEM_FIELD_EXP_SINSIN) {
      c0 = std::exp(-t0) * a.f.p[0];
      c1 = std::exp(-t1) * a.f.p[0];
    } else if (a.f.kind == PHFEM_FIELD_SINSIN) {
      c0 = c1 = a.f.p[0];
    }
    const CnStored st{p->top, p->cpl, p->lq, p->rp3};
    // TMA over the full tiles when the state and rhs allow 16-byte bulk copies
    const bool tma = ((((uintptr_t)state) | ((uintptr_t)rhs)) & 15u) == 0;
    const int64_t nfull = tma ? (int64_t)a.nE / kCnTile : 0;
    if (nfull > 0 && p->hybrid) {
      // 4 CTAs (16 warps) per SM: registers (122) and the 4-stage ring allow it;
      // the recompute is latency-bound, so residency matters more than depth
      const int grid = (int)std::min<int64_t>(nfull, (int64_t)ctx->num_sms * PHFEM_CN_HYB_BLOCKS);
      if (a.c.kind == PHFEM_COEFF_CENTROID_POLY)
        PHFEM_LAUNCH_PDL(ctx, "k_cn_hyb", k_cn_hyb<PHFEM_COEFF_CENTROID_POLY>, grid, kCnTile, kCnHybSmem,
            a, st, nfull, c0, c1, state, rhs);
      else
        PHFEM_LAUNCH_PDL(ctx, "k_cn_hyb", k_cn_hyb<PHFEM_COEFF_CONST>, grid, kCnTile, kCnHybSmem,
            a, st, nfull, c0, c1, state, rhs);
    } else if (nfull > 0) {
      const int grid = (int)std::min<int64_t>(nfull, (int64_t)ctx->num_sms * 2);
      PHFEM_LAUNCH(ctx, "k_cn_tma", k_cn_tma<<<grid, kCnTile, kCnTmaSmem, ctx->stream>>>(
          a, st, nfull, c0, c1, state, rhs));
    }
    const int64_t m0 = nfull * kCnTile;
    if (m0 < a.nE) {
      const int64_t nchunks = ((int64_t)a.nE - m0 + 31) / 32;
      const int grid = (int)std::min<int64_t>((nchunks + 3) / 4, (int64_t)ctx->num_sms * 16);
      PHFEM_LAUNCH(ctx, "k_cn_stored", k_cn_stored<<<grid, kCnThreads, 0, ctx->stream>>>(
          a, st, m0, c0, c1, state, rhs));
    }
    // (measured: running the rows on a side stream next to the element pass
    // gains nothing — both are DRAM-bound)
    // (measured: the rows grouped by owner tile at plan time and evaluated
    // inside k_cn_hyb right after their tile, U kept in L2 by an evict-last
    // policy — bit-identical, but the row loads and U gathers add a dependent
    // latency chain to every tile of a kernel with 16 warps per SM: hybrid
    // pass 0.256 + rows 0.097 ms -> 0.457 ms; dropped)
    // (measured: the rows on a side stream beside the hybrid element pass,
    // 3 or 4 element CTAs per SM: step 0.373 ms either way)
    if (p->cls.L > 0)
      PHFEM_LAUNCH_PDL(ctx, "k_cn_rows", k_cn_rows, grid_for(p->cls.L, 256, ctx->num_sms * PHFEM_CNR_GRID_MULT), 256, 0,
          (const uint2*)p->rowt, (const double*)p->rowh, (int)p->cls.L, a.s_c, state, rhs + a.N);
    if (p->cls.nD > 0)
      PHFEM_LAUNCH_PDL(ctx, "k_cn_edges", k_cn_edges, grid_for(p->cls.nD, 256, ctx->num_sms), 256, 0,
          a, (const int32_t*)p->topo.edge_nodes, (const int32_t*)p->topo.local_in_tplus, (int)p->cls.nD,
          (const int32_t*)p->cls.dirichlet_edge_ids, state, rhs);
    return PHFEM_OK;
  } else if (a.nE > 0) {
    const int64_t ntiles = ((int64_t)a.nE + kCnThreads - 1) / kCnThreads;
    const int grid = (int)std::min<int64_t>(ntiles, (int64_t)ctx->num_sms * 16);
    const int fk = (a.f.kind == PHFEM_FIELD_EXP_SINSIN || a.f.kind == PHFEM_FIELD_SINSIN ||
                    a.f.kind == PHFEM_FIELD_ZERO) ? a.f.kind : kKindGeneric;
    const bool cp = a.c.kind == PHFEM_COEFF_CENTROID_POLY;
#define PHFEM_CN(F)                                                                                   \
  do {                                                                                                \
    if (cp)                                                                                           \
      PHFEM_LAUNCH(ctx, "k_cn_elements", (k_cn_elements<F, PHFEM_COEFF_CENTROID_POLY><<<grid, kCnThreads, 0, ctx->stream>>>(a, state, rhs))); \
    else                                                                                              \
      PHFEM_LAUNCH(ctx, "k_cn_elements", (k_cn_elements<F, PHFEM_COEFF_CONST><<<grid, kCnThreads, 0, ctx->stream>>>(a, state, rhs))); \
  } while (0)
    if (fk == PHFEM_FIELD_EXP_SINSIN) PHFEM_CN(PHFEM_FIELD_EXP_SINSIN);
    else if (fk == PHFEM_FIELD_SINSIN) PHFEM_CN(PHFEM_FIELD_SINSIN);
    else if (fk == PHFEM_FIELD_ZERO) PHFEM_CN(PHFEM_FIELD_ZERO);
    else PHFEM_CN(kKindGeneric);
#undef PHFEM_CN
  }
  if (p->topo.E > 0) {
    PHFEM_LAUNCH(ctx, "k_cn_edges", k_cn_edges<<<grid_for(p->topo.E, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
        a, p->topo.edge_nodes, p->topo.local_in_tplus, p->topo.E, nullptr, state, rhs));
  }
  return PHFEM_OK;
}
