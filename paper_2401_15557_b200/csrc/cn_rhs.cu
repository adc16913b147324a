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
// Device version: ONE element pass per step.  Element m recomputes its
// M_minus block from the geometry (the same expressions as the assembly, so
// the same bits — 72 bytes/element of stored blocks are never read), adds its
// coupling terms in ascending multiplier order, evaluates f at the three edge
// midpoints at t_n and t_{n+1}, and — for every edge it owns as t_plus — also
// produces that edge's multiplier row (its own DOFs first, then the t_minus
// DOFs: ascending columns), including the Dirichlet data.  Neumann data enter
// through the per-element table of assemble.cu, evaluated once per step.
#include <algorithm>

#include "common.cuh"
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

__global__ void __launch_bounds__(kCnThreads) k_cn_elements(CnArgs a, const double* __restrict__ W,
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
      const phfem_coeff_values cv =
          phfem_coeffs_eval(&a.c, v[0].x, v[0].y, v[1].x, v[1].y, v[2].x, v[2].y);
      double b[9], d[9], mm[9], m0[9];
      phfem_local_blocks(v[0].x, v[0].y, v[1].x, v[1].y, v[2].x, v[2].y, &cv, b, d, mm, m0);

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
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          f0[i] = phfem_field_eval(&a.f, mx[i], my[i], a.t0);
          f1[i] = phfem_field_eval(&a.f, mx[i], my[i], a.t1);
        }
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          b0[i] = 0.0 + area / 3.0 * 0.5 * (f0[(i + 1) % 3] + f0[(i + 2) % 3]);
          b1[i] = 0.0 + area / 3.0 * 0.5 * (f1[(i + 1) % 3] + f1[(i + 2) % 3]);
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
        for (int j = 0; j < 3; ++j) {
          const int q = 3 * j + i;
          const double top = m0[q] + a.s_top * ((b[q] + d[q]) + mm[q]);
          acc += (0.0 + 1.0 * top) * U[j];
        }
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

      // multiplier rows of the retained edges m owns as t_plus
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        if (!plus[k] || rp[k] < 0) continue;
        const double cp = 0.0 + a.s_c * (len[k] * 0.5);
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < 3; ++c)
          if (c != k) acc += cp * U[c];
        const int tm = a.edge_elements[2 * e[k] + 1];
        double bdsum = 0.0 + 0.0;
        if (tm >= 0) {
          const int ledtn = a.ltm[e[k]];
          const double cm = 0.0 + a.s_c * (-len[k] * 0.5);
          for (int c = 0; c < 3; ++c)
            if (c != ledtn) acc += cm * W[3 * (int64_t)tm + c];
        } else if ((a.dir_bits[e[k] >> 5] >> (e[k] & 31)) & 1u) {
          const double2 pa = v[(k + 1) % 3], pb = v[(k + 2) % 3];
          const double midx = 0.5 * (pa.x + pb.x), midy = 0.5 * (pa.y + pb.y);
          const double bd0 = -len[k] * phfem_field_eval(&a.uD, midx, midy, a.t0);
          const double bd1 = -len[k] * phfem_field_eval(&a.uD, midx, midy, a.t1);
          bdsum = bd0 + bd1;
        }
        rhs[a.N + rp[k]] = acc + 0.5 * bdsum;
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
  delete p;
}

PHFEM_API phfem_status phfem_cn_rhs(phfem_ctx* ctx, phfem_cn_plan* p, int n, const double* state,
                                    double* rhs) {
  if (!ctx || !p || n < 0) return PHFEM_ERR_INVALID_ARGUMENT;
  const double t0 = n * p->k;        // load_at_time: t = n * k (parabolic.cpp:61)
  const double t1 = (n + 1) * p->k;
  if (p->neu.nN > 0) {
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
  if (a.nE > 0) {
    const int64_t ntiles = ((int64_t)a.nE + kCnThreads - 1) / kCnThreads;
    const int grid = (int)std::min<int64_t>(ntiles, (int64_t)ctx->num_sms * 16);
    PHFEM_LAUNCH(ctx, "k_cn_elements", k_cn_elements<<<grid, kCnThreads, 0, ctx->stream>>>(a, state, rhs));
  }
  return PHFEM_OK;
}
