// sparse.cu — SURVEY §8(f2): the generic COO -> compressed conversion of the
// reference (SparseMatrix::from_triplets, proj/src/sparse.cpp:30-97) on the
// device, and the operators it feeds: the elliptic saddle matrix
// (build_saddle_matrix, elliptic.cpp:22-36) and the Crank-Nicolson step
// matrices (step_matrix, parabolic.cpp:21-37) — the inputs of the global
// solve, which itself stays outside the product path.
//
// from_triplets semantics kept exactly:
//   * the first out-of-range entry raises out_of_range with its index;
//   * a buffer already strictly increasing in (row, col) is stored as-is
//     (values untouched, -0.0 included);
//   * otherwise entries are ordered by (row, col), ties by insertion, and each
//     run is summed left to right from 0.0;
//   * output is Eigen's ColMajor CSC, rows ascending inside a column.
// Device algorithm: one stable LSD radix sort (radix_sort.cu, hand-written)
// of the column-major key col * rows + row with the entry index as payload —
// stable, so runs keep insertion order and come out in CSC order directly —
// then run starts by neighbour compare, a scan for run ids, one thread per
// run summing its (short) run sequentially in the reference's order (the
// segmented run-sum), and the column pointer array from the run columns.
#include <algorithm>

#include "common.cuh"

namespace phfem {

__global__ void k_trip_check(const int32_t* __restrict__ ri, const int32_t* __restrict__ ci,
                             int64_t n, int rows, int cols, unsigned long long* __restrict__ bad,
                             unsigned long long* __restrict__ unsorted) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int r = ri[k], c = ci[k];
    if (r < 0 || r >= rows || c < 0 || c >= cols) atomicMin(bad, (unsigned long long)k);
    if (k > 0) {
      const int rp = ri[k - 1], cp = ci[k - 1];
      if (!(rp < r || (rp == r && cp < c))) *unsorted = 1;
    }
  }
}

__global__ void k_trip_keys(const int32_t* __restrict__ ri, const int32_t* __restrict__ ci,
                            int64_t n, int rows, uint64_t* __restrict__ keys,
                            uint32_t* __restrict__ idx) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    keys[k] = (uint64_t)ci[k] * (uint64_t)rows + (uint64_t)ri[k];
    idx[k] = (uint32_t)k;
  }
}

__global__ void k_trip_starts(const uint64_t* __restrict__ keys, int64_t n, int32_t* __restrict__ flag) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    flag[k] = (k == 0 || keys[k] != keys[k - 1]) ? 1 : 0;
}

// pos = exclusive scan of the start flags: run id of every run start
__global__ void k_trip_runs(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ idx,
                            const int32_t* __restrict__ pos, int64_t n, int rows, int raw,
                            const double* __restrict__ v, int32_t* __restrict__ inner,
                            double* __restrict__ vals, int32_t* __restrict__ run_col) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    if (!(k == 0 || keys[k] != keys[k - 1])) continue;
    const uint64_t key = keys[k];
    const int r = pos[k];
    double sum;
    if (raw) {  // sorted, unique buffer: stored as given (sparse.cpp:53)
      sum = v[idx[k]];
    } else {    // run summed left to right from 0.0 (sparse.cpp:67-69)
      sum = 0.0;
      for (int64_t q = k; q < n && keys[q] == key; ++q) sum += v[idx[q]];
    }
    inner[r] = (int32_t)(key % (uint64_t)rows);
    run_col[r] = (int32_t)(key / (uint64_t)rows);
    vals[r] = sum;
  }
}

// outer[c] = first run with column >= c
__global__ void k_trip_outer(const int32_t* __restrict__ run_col, int64_t nnz, int cols,
                             int32_t* __restrict__ outer) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= nnz;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int cprev = r > 0 ? run_col[r - 1] : -1;
    const int ccur = r < nnz ? run_col[r] : cols;
    for (int c = cprev + 1; c <= ccur; ++c) outer[c] = (int32_t)r;
  }
}

phfem_status from_triplets_impl(phfem_ctx* ctx, int rows, int cols, const int32_t* ri,
                                const int32_t* ci, const double* v, int64_t n, phfem_csc* out) {
  memset(out, 0, sizeof(*out));
  out->rows = rows;
  out->cols = cols;
  if (n >= (int64_t(1) << 31))
    return set_error(ctx, PHFEM_ERR_INVALID_ARGUMENT, "from_triplets: more than 2^31 entries");
  PHFEM_TRY(dalloc(ctx, &out->outer, (int64_t)cols + 1));
  unsigned long long* flags = nullptr;
  PHFEM_TRY(dalloc(ctx, &flags, 2));
  const unsigned long long init[2] = {~0ull, 0ull};
  PHFEM_CUDA(ctx, cudaMemcpyAsync(flags, init, sizeof init, cudaMemcpyHostToDevice, ctx->stream));
  const int grid = grid_for(n, 256, ctx->num_sms * 8);
  if (n > 0)
    PHFEM_LAUNCH(ctx, "k_trip_check", k_trip_check<<<grid, 256, 0, ctx->stream>>>(ri, ci, n, rows, cols, flags,
                                                                                  flags + 1));
  unsigned long long h[2];
  PHFEM_CUDA(ctx, cudaMemcpyAsync(h, flags, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
  PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  dfree(ctx, flags);
  if (h[0] != ~0ull) {
    int32_t rc[2];
    PHFEM_CUDA(ctx, cudaMemcpy(&rc[0], ri + h[0], sizeof(int32_t), cudaMemcpyDeviceToHost));
    PHFEM_CUDA(ctx, cudaMemcpy(&rc[1], ci + h[0], sizeof(int32_t), cudaMemcpyDeviceToHost));
    dfree(ctx, out->outer);
    return set_error(ctx, PHFEM_ERR_OUT_OF_RANGE, "TripletBuffer: entry %llu at (%d,%d) outside %dx%d",
                     h[0], rc[0], rc[1], rows, cols);
  }
  const int raw = h[1] ? 0 : 1;
  if (n == 0) {
    PHFEM_CUDA(ctx, cudaMemsetAsync(out->outer, 0, sizeof(int32_t) * ((int64_t)cols + 1), ctx->stream));
    PHFEM_TRY(dalloc(ctx, &out->inner, 1));
    PHFEM_TRY(dalloc(ctx, &out->values, 1));
    return PHFEM_OK;
  }
  uint64_t *k0 = nullptr, *k1 = nullptr;
  uint32_t *i0 = nullptr, *i1 = nullptr;
  PHFEM_TRY(dalloc(ctx, &k0, n));
  PHFEM_TRY(dalloc(ctx, &k1, n));
  PHFEM_TRY(dalloc(ctx, &i0, n));
  PHFEM_TRY(dalloc(ctx, &i1, n));
  PHFEM_LAUNCH(ctx, "k_trip_keys", k_trip_keys<<<grid, 256, 0, ctx->stream>>>(ri, ci, n, rows, k0, i0));
  // only the bits the keys use: ceil(log2(rows * cols))
  int end_bit = 1;
  const unsigned long long maxkey = (unsigned long long)rows * (unsigned long long)cols;
  while (end_bit < 64 && (1ull << end_bit) < maxkey) ++end_bit;
  PHFEM_TRY(radix_sort_pairs_u64(ctx, k0, k1, i0, i1, n, end_bit));
  dfree(ctx, k0);
  dfree(ctx, i0);
  int32_t* pos = nullptr;
  PHFEM_TRY(dalloc(ctx, &pos, n + 1));
  PHFEM_LAUNCH(ctx, "k_trip_starts", k_trip_starts<<<grid, 256, 0, ctx->stream>>>(k1, n, pos));
  PHFEM_CUDA(ctx, cudaMemsetAsync(pos + n, 0, sizeof(int32_t), ctx->stream));
  PHFEM_TRY(scan_exclusive_i32(ctx, pos, pos, n + 1, nullptr));
  int32_t nnz = 0;
  PHFEM_CUDA(ctx, cudaMemcpyAsync(&nnz, pos + n, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
  PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  out->nnz = nnz;
  int32_t* run_col = nullptr;
  PHFEM_TRY(dalloc(ctx, &out->inner, nnz));
  PHFEM_TRY(dalloc(ctx, &out->values, nnz));
  PHFEM_TRY(dalloc(ctx, &run_col, nnz));
  PHFEM_LAUNCH(ctx, "k_trip_runs", k_trip_runs<<<grid, 256, 0, ctx->stream>>>(
      k1, i1, pos, n, rows, raw, v, out->inner, out->values, run_col));
  PHFEM_LAUNCH(ctx, "k_trip_outer", k_trip_outer<<<grid_for((int64_t)nnz + 1, 256, ctx->num_sms * 8), 256, 0,
                                                   ctx->stream>>>(run_col, nnz, cols, out->outer));
  dfree(ctx, run_col);
  dfree(ctx, pos);
  dfree(ctx, k1);
  dfree(ctx, i1);
  return PHFEM_OK;
}

// ---- operator triplets in the reference's append order -----------------------------
struct OpArgs {
  const double *B, *D, *M, *M0;  // [nE][9] column-major blocks
  const int32_t *c_outer, *c_inner;
  const double* c_val;
  int nE, L;
  int64_t nnzC;
  double s_top;   // step: sign * (k / 2.0) (parabolic.cpp:24-27); saddle: unused
  double s_ct;    // scale of C' in the primal rows
  double s_c;     // scale of C in the multiplier rows
  int step;       // 0 saddle, 1 step matrix
};

// K / top block: column-major over the block-diagonal CSC -> triplet t = 9e + 3j + i
__global__ void k_op_block(OpArgs a, int32_t* __restrict__ ri, int32_t* __restrict__ ci,
                           double* __restrict__ v) {
  const int64_t n9 = 9 * (int64_t)a.nE;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n9;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / 9;
    const int q = (int)(t - 9 * e), j = q / 3, i = q - 3 * j;
    // (B + D) + M: Eigen's sum on the (identical) block pattern
    const double k = (a.B[t] + a.D[t]) + a.M[t];
    const double val = a.step ? a.M0[t] + a.s_top * k : k;
    ri[t] = (int32_t)(3 * e + i);
    ci[t] = (int32_t)(3 * e + j);
    v[t] = 1.0 * val;  // append_block(top, scale 1.0)
  }
}

// the two coupling blocks: -C' (transposed, primal rows / multiplier columns)
// then -C, each in C's column-major storage order
__global__ void k_op_coupling(OpArgs a, int N, int32_t* __restrict__ ri, int32_t* __restrict__ ci,
                              double* __restrict__ v) {
  const int64_t base = 9 * (int64_t)a.nE;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < a.nnzC;
       p += (int64_t)gridDim.x * blockDim.x) {
    // column j of C holding entry p (binary search of the column pointers)
    int lo = 0, hi = N;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (a.c_outer[mid] <= p) lo = mid;
      else hi = mid;
    }
    const int j = lo, l = a.c_inner[p];
    const double c = a.c_val[p];
    ri[base + p] = j;
    ci[base + p] = N + l;
    v[base + p] = a.s_ct * c;
    ri[base + a.nnzC + p] = N + l;
    ci[base + a.nnzC + p] = j;
    v[base + a.nnzC + p] = a.s_c * c;
  }
}

}  // namespace phfem

using namespace phfem;

PHFEM_API phfem_status phfem_from_triplets(phfem_ctx* ctx, int32_t rows, int32_t cols,
                                           const int32_t* ri, const int32_t* ci, const double* v,
                                           int64_t n, phfem_csc* out) {
  if (!ctx || !out || rows < 0 || cols < 0 || n < 0 || (n && (!ri || !ci || !v)))
    return PHFEM_ERR_INVALID_ARGUMENT;
  return from_triplets_impl(ctx, rows, cols, ri, ci, v, n, out);
}

static phfem_status operator_matrix(phfem_ctx* ctx, int32_t nE, const double* B, const double* D,
                                    const double* M, const double* M0, const phfem_csc* C, int step,
                                    double k, double sign, phfem_csc* out) {
  memset(out, 0, sizeof(*out));
  if (!ctx || !B || !D || !M || !C || !out || (step && !M0) || nE < 0) return PHFEM_ERR_INVALID_ARGUMENT;
  const int N = 3 * nE, L = C->rows;
  if (C->cols != N)
    return set_error(ctx, PHFEM_ERR_MISMATCH, "operator matrix: C does not match the blocks");
  OpArgs a;
  a.B = B;
  a.D = D;
  a.M = M;
  a.M0 = M0;
  a.c_outer = C->outer;
  a.c_inner = C->inner;
  a.c_val = C->values;
  a.nE = nE;
  a.L = L;
  a.nnzC = C->nnz;
  a.step = step;
  a.s_top = sign * (k / 2.0);
  a.s_ct = step ? -sign * (k / 2.0) : -1.0;
  a.s_c = step ? -sign * 0.5 : -1.0;
  const int64_t n = 9 * (int64_t)nE + 2 * C->nnz;
  int32_t *ri = nullptr, *ci = nullptr;
  double* v = nullptr;
  PHFEM_TRY(dalloc(ctx, &ri, n));
  PHFEM_TRY(dalloc(ctx, &ci, n));
  PHFEM_TRY(dalloc(ctx, &v, n));
  if (nE > 0)
    PHFEM_LAUNCH(ctx, "k_op_block", k_op_block<<<grid_for(9 * (int64_t)nE, 256, ctx->num_sms * 8), 256, 0,
                                                 ctx->stream>>>(a, ri, ci, v));
  if (C->nnz > 0)
    PHFEM_LAUNCH(ctx, "k_op_coupling", k_op_coupling<<<grid_for(C->nnz, 256, ctx->num_sms * 8), 256, 0,
                                                       ctx->stream>>>(a, N, ri, ci, v));
  const phfem_status st = from_triplets_impl(ctx, N + L, N + L, ri, ci, v, n, out);
  dfree(ctx, ri);
  dfree(ctx, ci);
  dfree(ctx, v);
  return st;
}

PHFEM_API phfem_status phfem_saddle_matrix(phfem_ctx* ctx, int32_t nE, const double* B,
                                           const double* D, const double* M, const phfem_csc* C,
                                           phfem_csc* out) {
  return operator_matrix(ctx, nE, B, D, M, nullptr, C, 0, 0.0, 1.0, out);
}

PHFEM_API phfem_status phfem_step_matrix(phfem_ctx* ctx, int32_t nE, const double* B,
                                         const double* D, const double* M, const double* M0,
                                         const phfem_csc* C, double k, double sign,
                                         phfem_csc* out) {
  if (!(k > 0.0)) return set_error(ctx, PHFEM_ERR_INVALID_ARGUMENT, "step_matrices: k must be positive");
  return operator_matrix(ctx, nE, B, D, M, M0, C, 1, k, sign, out);
}
