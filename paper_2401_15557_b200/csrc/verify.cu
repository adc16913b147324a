// verify.cu — SURVEY §8(f4): the device verification kernels around the
// (excluded) solve, each with the reference's evaluation order:
//   * constraint residual ||C U + bD||_inf          (tools/main.cpp:205-207)
//   * exact_multiplier                              (analysis.cpp:26-39)
//   * error_h1 / error_l2 (25-point Duffy rule)     (analysis.cpp:41-80;
//                                                    quadrature.cpp:9-53)
//   * error_multiplier                              (analysis.cpp:82-98)
//   * hybrid_midpoint_traces                        (analysis.cpp:113-125)
//   * CSC -> CSR and the Eigen-ordered SpMV y = A x (the M_plus / M_minus
//     products of parabolic.cpp:100 on a stored step matrix)
// Per-entry values are bit-identical to the reference's.  The two error norms
// sum per-element terms over the whole mesh: the reference sums them in
// element order, the device in a fixed tree (deterministic, run to run); the
// terms themselves are bit-identical (optional per-element output), the sum
// agrees to rounding.  Max-reductions (residual, error_multiplier) are exact.

#include <algorithm>
#include <cmath>
#include <cstring>

#include "common.cuh"

namespace phfem {

constexpr int kVfThreads = 256;

// Max-reductions of non-negative doubles run on their bit patterns (the
// unsigned order of IEEE bits equals the numeric order for x >= 0).
template <typename T>
__device__ __forceinline__ T block_reduce_max(T v, T* sm) {
  for (int o = 16; o > 0; o >>= 1) {
    const T w = __shfl_down_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : T(0);
    for (int o = 16; o > 0; o >>= 1) {
      const T w = __shfl_down_sync(0xffffffffu, v, o);
      v = w > v ? w : v;
    }
  }
  return v;
}

// fixed-order block sum (deterministic for a fixed launch shape)
__device__ __forceinline__ double block_reduce_sum(double v, double* sm) {
  sm[threadIdx.x] = v;
  __syncthreads();
  for (int s = blockDim.x >> 1; s > 0; s >>= 1) {
    if (threadIdx.x < s) sm[threadIdx.x] = sm[threadIdx.x] + sm[threadIdx.x + s];
    __syncthreads();
  }
  return sm[0];
}

// ||C U + bD||_inf: row l = 0.0 + sum over ascending columns of C_lj U_j
// (Eigen ColMajor SpMV), then + bD_l, |.|, max (lpNorm<Infinity>)
__global__ void __launch_bounds__(kVfThreads) k_residual(const int32_t* __restrict__ row_ptr,
                                                         const int32_t* __restrict__ col,
                                                         const double* __restrict__ val, int L,
                                                         const double* __restrict__ U,
                                                         const double* __restrict__ bd,
                                                         unsigned long long* __restrict__ out) {
  __shared__ unsigned long long sm[kVfThreads / 32];
  unsigned long long best = 0;
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < L;
       l += (int64_t)gridDim.x * blockDim.x) {
    double r = 0.0;
    for (int k = row_ptr[l]; k < row_ptr[l + 1]; ++k) r += val[k] * U[col[k]];
    if (bd) r = r + bd[l];
    const unsigned long long b = (unsigned long long)__double_as_longlong(fabs(r));
    best = b > best ? b : best;
  }
  best = block_reduce_max(best, sm);
  if (threadIdx.x == 0) atomicMax(out, best);
}

__global__ void k_exact_multiplier(const double2* __restrict__ coords, const int32_t* __restrict__ edge_nodes,
                                   const int32_t* __restrict__ rpos, int E, phfem_problem p, double t,
                                   double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = rpos[e];
    if (r < 0) continue;
    const int2 ab = reinterpret_cast<const int2*>(edge_nodes)[e];
    const double2 a = coords[ab.x], b = coords[ab.y];
    out[r] = phfem_exact_multiplier_value(&p, a.x, a.y, b.x, b.y, t);
  }
}

struct QuadArgs {
  phfem_quad_rule rule;
  phfem_problem p;
  double t;
};

// per-element error terms (bit-identical to the reference's), per-thread
// sequential partials, fixed-order block tree -> part[block]
template <bool kH1>
__global__ void __launch_bounds__(kVfThreads) k_error_terms(const double2* __restrict__ coords,
                                                            const int32_t* __restrict__ elements, int nE,
                                                            const double* __restrict__ U, QuadArgs q,
                                                            double* __restrict__ terms,
                                                            double* __restrict__ part) {
  __shared__ double sm[kVfThreads];
  double acc = 0.0;
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < nE;
       m += (int64_t)gridDim.x * blockDim.x) {
    const double2 v0 = coords[elements[3 * m]], v1 = coords[elements[3 * m + 1]],
                  v2 = coords[elements[3 * m + 2]];
    const double u0 = U[3 * m], u1 = U[3 * m + 1], u2 = U[3 * m + 2];
    const double term = kH1 ? phfem_h1_term(&q.p, &q.rule, v0.x, v0.y, v1.x, v1.y, v2.x, v2.y, u0, u1, u2, q.t)
                            : phfem_l2_term(&q.p, &q.rule, v0.x, v0.y, v1.x, v1.y, v2.x, v2.y, u0, u1, u2, q.t);
    if (terms) terms[m] = term;
    acc += term;
  }
  const double s = block_reduce_sum(acc, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kVfThreads) k_sum_parts(const double* __restrict__ part, int n,
                                                          double* __restrict__ out) {
  __shared__ double sm[kVfThreads];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += part[i];
  const double s = block_reduce_sum(acc, sm);
  if (threadIdx.x == 0) *out = s;
}

// error_multiplier: w = C' (exact - discrete) per primal DOF — the (<= 2)
// retained edges of the element carrying the DOF, ascending rows, C entries
// +-|E|/2 (assembly.cpp:160,164) — then max |w_i| / sqrt(B_ii) over B_ii > 0
__global__ void __launch_bounds__(kVfThreads) k_error_multiplier(
    const double2* __restrict__ coords, const int32_t* __restrict__ elements,
    const int32_t* __restrict__ elem_edge, const int32_t* __restrict__ rpos, int nE,
    const double* __restrict__ B, const double* __restrict__ exact, const double* __restrict__ discrete,
    unsigned long long* __restrict__ out) {
  __shared__ unsigned long long sm[kVfThreads / 32];
  unsigned long long best = 0, any = 0;
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < nE;
       m += (int64_t)gridDim.x * blockDim.x) {
    const double2 v[3] = {coords[elements[3 * m]], coords[elements[3 * m + 1]], coords[elements[3 * m + 2]]};
    int rp[3];
    double c[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int s = elem_edge[3 * m + k];
      rp[k] = rpos[s >= 0 ? s : ~s];
      const double2 pa = v[(k + 1) % 3], pb = v[(k + 2) % 3];
      const double dx = pb.x - pa.x, dy = pb.y - pa.y;
      const double len = sqrt(dx * dx + dy * dy);  // edge_topology.cpp:183
      c[k] = s >= 0 ? len * 0.5 : -len * 0.5;
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double diag = B[9 * m + 4 * i];
      if (diag <= 0.0) continue;  // analysis.cpp:92 (a NaN diagonal counts, its ratio never wins)
      any = 1;
      int ka = (i + 1) % 3, kb = (i + 2) % 3;
      if (rp[kb] >= 0 && (rp[ka] < 0 || rp[kb] < rp[ka])) {
        const int x = ka;
        ka = kb;
        kb = x;
      }
      double w = 0.0;
      if (rp[ka] >= 0) w += c[ka] * (exact[rp[ka]] - discrete[rp[ka]]);
      if (rp[kb] >= 0) w += c[kb] * (exact[rp[kb]] - discrete[rp[kb]]);
      const double ratio = fabs(w) / sqrt(diag);
      if (!(ratio == ratio)) continue;  // std::max(worst, NaN) keeps worst
      const unsigned long long b = (unsigned long long)__double_as_longlong(ratio);
      best = b > best ? b : best;
    }
  }
  best = block_reduce_max(best, sm);
  if (threadIdx.x == 0) atomicMax(out, best);
  __syncthreads();
  any = block_reduce_max(any, sm);
  if (threadIdx.x == 0 && any) atomicMax(out + 1, 1ull);
}

__global__ void k_midpoint_traces(const int32_t* __restrict__ edge_elements, const int32_t* __restrict__ ltp,
                                  int E, const double* __restrict__ U, double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = edge_elements[2 * e];
    const int led = ltp[e];
    const int i = led == 2 ? 0 : led + 1, j = led == 0 ? 2 : led - 1;
    out[e] = 0.5 * (U[3 * m + i] + U[3 * m + j]);
  }
}

// ---- CSC -> CSR (stable by row: columns stay ascending) and the SpMV ------
__global__ void k_csc_cols(const int32_t* __restrict__ outer, int cols, int32_t* __restrict__ colp) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < cols;
       j += (int64_t)gridDim.x * blockDim.x)
    for (int p = outer[j]; p < outer[j + 1]; ++p) colp[p] = (int32_t)j;
}

__global__ void k_iota(int64_t n, int32_t* __restrict__ v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (int32_t)i;
}

__global__ void k_row_count(const int32_t* __restrict__ inner, int64_t n, int32_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + inner[i], 1);
}

__global__ void k_csr_gather(const int32_t* __restrict__ perm, const int32_t* __restrict__ colp,
                             const double* __restrict__ val, int64_t n, int32_t* __restrict__ col,
                             double* __restrict__ out) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int p = perm[q];
    col[q] = colp[p];
    out[q] = val[p];
  }
}

// y_i = 0.0 + sum over ascending columns of A_ij x_j (Eigen ColMajor A * x:
// res.setZero(); res(i) += A_ij * (1.0 * x_j), columns ascending)
__global__ void k_csr_spmv(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                           const double* __restrict__ val, int rows, const double* __restrict__ x,
                           double* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int k = row_ptr[i]; k < row_ptr[i + 1]; ++k) acc += val[k] * x[col[k]];
    y[i] = acc;
  }
}

static phfem_status fetch_u64(phfem_ctx* ctx, const unsigned long long* dev, unsigned long long* host, int n) {
  PHFEM_CUDA(ctx, cudaMemcpyAsync(host, dev, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost, ctx->stream));
  PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return PHFEM_OK;
}

static double bits_to_double(unsigned long long b) {
  double d;
  std::memcpy(&d, &b, sizeof d);
  return d;
}

static bool valid_problem(const phfem_problem* p) {
  return p && (p->kind == PHFEM_PROBLEM_ELLIPTIC_POLY || p->kind == PHFEM_PROBLEM_PARABOLIC_POLY ||
               p->kind == PHFEM_PROBLEM_SINSIN);
}

}  // namespace phfem

using namespace phfem;

PHFEM_API phfem_status phfem_constraint_residual(phfem_ctx* ctx, const phfem_csr* C, const double* primal,
                                                 const double* bd, double* out) {
  if (!ctx || !C || !out || (C->rows > 0 && !primal)) return PHFEM_ERR_INVALID_ARGUMENT;
  *out = 0.0;
  if (C->rows == 0) return PHFEM_OK;
  unsigned long long* d = nullptr;
  PHFEM_TRY(dalloc(ctx, &d, 1));
  PHFEM_CUDA(ctx, cudaMemsetAsync(d, 0, sizeof(unsigned long long), ctx->stream));
  PHFEM_LAUNCH(ctx, "k_residual", k_residual<<<grid_for(C->rows, kVfThreads, ctx->num_sms * 8), kVfThreads, 0,
                                                ctx->stream>>>(C->row_ptr, C->col_idx, C->values, C->rows, primal,
                                                               bd, d));
  unsigned long long h = 0;
  const phfem_status st = fetch_u64(ctx, d, &h, 1);
  dfree(ctx, d);
  if (st != PHFEM_OK) return st;
  *out = bits_to_double(h);
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_exact_multiplier(phfem_ctx* ctx, const phfem_mesh* mesh, const phfem_topology* topo,
                                              const phfem_classification* cls, const phfem_problem* problem,
                                              double t, double* out) {
  if (!ctx || !mesh || !topo || !cls || !valid_problem(problem) || (cls->L > 0 && !out))
    return PHFEM_ERR_INVALID_ARGUMENT;
  if (problem->coeffs.kind != PHFEM_COEFF_CONST)
    return set_error(ctx, PHFEM_ERR_INVALID_ARGUMENT, "exact_multiplier: problem coefficients must be constant");
  if (cls->E != topo->E)
    return set_error(ctx, PHFEM_ERR_MISMATCH, "exact_multiplier: classification does not match topology");
  if (topo->E > 0 && cls->L > 0)
    PHFEM_LAUNCH(ctx, "k_exact_multiplier", k_exact_multiplier<<<grid_for(topo->E, 256, ctx->num_sms * 8), 256, 0,
                                                                ctx->stream>>>(
        (const double2*)mesh->coords, topo->edge_nodes, cls->retained_pos, topo->E, *problem, t, out));
  return PHFEM_OK;
}

static phfem_status error_norm(phfem_ctx* ctx, const phfem_mesh* mesh, const double* primal,
                               const phfem_problem* problem, double t, double* out, double* terms, bool h1) {
  if (!ctx || !mesh || !out || !valid_problem(problem) || (mesh->nE > 0 && !primal))
    return PHFEM_ERR_INVALID_ARGUMENT;
  *out = 0.0;
  if (mesh->nE == 0) return PHFEM_OK;
  QuadArgs q;
  phfem_default_rule(&q.rule);  // host evaluation of quadrature.cpp's rule (no FMA on x86-64)
  q.p = *problem;
  q.t = t;
  const int grid = grid_for(mesh->nE, kVfThreads, ctx->num_sms * 8);
  double* part = nullptr;
  PHFEM_TRY(dalloc(ctx, &part, grid + 1));
  if (h1)
    PHFEM_LAUNCH(ctx, "k_error_terms_h1", k_error_terms<true><<<grid, kVfThreads, 0, ctx->stream>>>(
        (const double2*)mesh->coords, mesh->elements, mesh->nE, primal, q, terms, part));
  else
    PHFEM_LAUNCH(ctx, "k_error_terms_l2", k_error_terms<false><<<grid, kVfThreads, 0, ctx->stream>>>(
        (const double2*)mesh->coords, mesh->elements, mesh->nE, primal, q, terms, part));
  PHFEM_LAUNCH(ctx, "k_sum_parts", k_sum_parts<<<1, kVfThreads, 0, ctx->stream>>>(part, grid, part + grid));
  double s = 0.0;
  PHFEM_CUDA(ctx, cudaMemcpyAsync(&s, part + grid, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  dfree(ctx, part);
  *out = std::sqrt(s);  // analysis.cpp:57 / :79
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_error_l2(phfem_ctx* ctx, const phfem_mesh* mesh, const double* primal,
                                      const phfem_problem* problem, double t, double* out, double* terms) {
  return error_norm(ctx, mesh, primal, problem, t, out, terms, false);
}

PHFEM_API phfem_status phfem_error_h1(phfem_ctx* ctx, const phfem_mesh* mesh, const double* primal,
                                      const phfem_problem* problem, double t, double* out, double* terms) {
  return error_norm(ctx, mesh, primal, problem, t, out, terms, true);
}

PHFEM_API phfem_status phfem_error_multiplier(phfem_ctx* ctx, const phfem_mesh* mesh, const phfem_topology* topo,
                                              const phfem_classification* cls, const double* B,
                                              const double* exact, const double* discrete, int64_t n_exact,
                                              int64_t n_discrete, double* out) {
  if (!ctx || !mesh || !topo || !cls || !out) return PHFEM_ERR_INVALID_ARGUMENT;
  if (n_exact != n_discrete || n_exact != cls->L)
    return set_error(ctx, PHFEM_ERR_INVALID_ARGUMENT, "error_multiplier: size mismatch");
  if (mesh->nE > 0 && !B) return PHFEM_ERR_INVALID_ARGUMENT;
  if (cls->L > 0 && (!exact || !discrete)) return PHFEM_ERR_INVALID_ARGUMENT;
  unsigned long long* d = nullptr;
  PHFEM_TRY(dalloc(ctx, &d, 2));
  PHFEM_CUDA(ctx, cudaMemsetAsync(d, 0, 2 * sizeof(unsigned long long), ctx->stream));
  if (mesh->nE > 0)
    PHFEM_LAUNCH(ctx, "k_error_multiplier", k_error_multiplier<<<grid_for(mesh->nE, kVfThreads, ctx->num_sms * 8),
                                                                kVfThreads, 0, ctx->stream>>>(
        (const double2*)mesh->coords, mesh->elements, topo->elem_edge, cls->retained_pos, mesh->nE, B, exact,
        discrete, d));
  unsigned long long h[2] = {0, 0};
  const phfem_status st = fetch_u64(ctx, d, h, 2);
  dfree(ctx, d);
  if (st != PHFEM_OK) return st;
  if (!h[1])
    return set_error(ctx, PHFEM_ERR_RUNTIME, "error_multiplier: all diagonal entries of B vanish");
  *out = bits_to_double(h[0]);
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_midpoint_traces(phfem_ctx* ctx, const phfem_topology* topo, const double* primal,
                                             double* out) {
  if (!ctx || !topo || (topo->E > 0 && (!primal || !out))) return PHFEM_ERR_INVALID_ARGUMENT;
  if (topo->E > 0)
    PHFEM_LAUNCH(ctx, "k_midpoint_traces", k_midpoint_traces<<<grid_for(topo->E, 256, ctx->num_sms * 8), 256, 0,
                                                              ctx->stream>>>(
        topo->edge_elements, topo->local_in_tplus, topo->E, primal, out));
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_csc_to_csr(phfem_ctx* ctx, const phfem_csc* A, phfem_csr* out) {
  if (!ctx || !A || !out) return PHFEM_ERR_INVALID_ARGUMENT;
  memset(out, 0, sizeof(*out));
  const int64_t n = A->nnz;
  if (n >= (int64_t(1) << 31))
    return set_error(ctx, PHFEM_ERR_INVALID_ARGUMENT, "csc_to_csr: too many entries for int ids");
  out->rows = A->rows;
  out->cols = A->cols;
  out->nnz = n;
  PHFEM_TRY(dalloc(ctx, &out->row_ptr, (int64_t)A->rows + 1));
  PHFEM_TRY(dalloc(ctx, &out->col_idx, std::max<int64_t>(n, 1)));
  PHFEM_TRY(dalloc(ctx, &out->values, std::max<int64_t>(n, 1)));
  PHFEM_CUDA(ctx, cudaMemsetAsync(out->row_ptr, 0, sizeof(int32_t) * ((int64_t)A->rows + 1), ctx->stream));
  if (n == 0) return PHFEM_OK;
  const int grid = grid_for(n, 256, ctx->num_sms * 8);
  int32_t *colp = nullptr, *k1 = nullptr, *i0 = nullptr, *i1 = nullptr;
  PHFEM_TRY(dalloc(ctx, &colp, n));
  PHFEM_TRY(dalloc(ctx, &k1, n));
  PHFEM_TRY(dalloc(ctx, &i0, n));
  PHFEM_TRY(dalloc(ctx, &i1, n));
  if (A->cols > 0)
    PHFEM_LAUNCH(ctx, "k_csc_cols", k_csc_cols<<<grid_for(A->cols, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
        A->outer, A->cols, colp));
  PHFEM_LAUNCH(ctx, "k_iota", k_iota<<<grid, 256, 0, ctx->stream>>>(n, i0));
  PHFEM_LAUNCH(ctx, "k_row_count", k_row_count<<<grid, 256, 0, ctx->stream>>>(A->inner, n, out->row_ptr));
  PHFEM_TRY(scan_exclusive_i32(ctx, out->row_ptr, out->row_ptr, (int64_t)A->rows + 1, nullptr));
  int end_bit = 1;
  while (end_bit < 31 && (1ll << end_bit) < (long long)A->rows) ++end_bit;
  // stable LSD radix sort by row: entries of a row keep the CSC (column) order
  PHFEM_TRY(radix_sort_pairs_u32(ctx, reinterpret_cast<const uint32_t*>(A->inner), reinterpret_cast<uint32_t*>(k1),
                                 reinterpret_cast<const uint32_t*>(i0), reinterpret_cast<uint32_t*>(i1), n, end_bit));
  PHFEM_LAUNCH(ctx, "k_csr_gather", k_csr_gather<<<grid, 256, 0, ctx->stream>>>(i1, colp, A->values, n,
                                                                                out->col_idx, out->values));
  dfree(ctx, colp);
  dfree(ctx, k1);
  dfree(ctx, i0);
  dfree(ctx, i1);
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_csr_spmv(phfem_ctx* ctx, const phfem_csr* A, const double* x, double* y) {
  if (!ctx || !A || (A->rows > 0 && (!x || !y))) return PHFEM_ERR_INVALID_ARGUMENT;
  if (A->rows > 0)
    PHFEM_LAUNCH(ctx, "k_csr_spmv", k_csr_spmv<<<grid_for(A->rows, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
        A->row_ptr, A->col_idx, A->values, A->rows, x, y));
  return PHFEM_OK;
}
