// selftest.cu — device self-test of the fast-math building blocks
// (fastmath.cuh): division exactness against IEEE '/' and the ulp error of
// sin_fast against CUDA's sin, over counter-based random operands.  Run by
// tests/test_gpu_parity.py; not used by the product path.
#include "common.cuh"
#include "fastmath.cuh"

namespace phfem {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// operand families: 0 random exponents in the safe window; 1 quotients with
// all-ones / all-zeros significand neighbourhoods; 2 mesh-like geometry
// (coordinate differences over twice-areas of tiny triangles)
__device__ __forceinline__ void operands(uint64_t i, uint64_t seed, double* a, double* b) {
  const uint64_t r1 = mix64(seed + 2 * i + 1), r2 = mix64(seed + 2 * i + 2);
  const int fam = (int)(r1 % 3);
  if (fam == 0) {
    const int ea = (int)((r1 >> 8) % 800) - 400, eb = (int)((r2 >> 8) % 800) - 400;
    *a = ldexp(1.0 + (double)(r1 >> 12) * 0x1p-52, ea) * ((r1 & 2) ? -1.0 : 1.0);
    *b = ldexp(1.0 + (double)(r2 >> 12) * 0x1p-52, eb);
  } else if (fam == 1) {
    const double sig = 2.0 - (double)((r1 >> 20) & 0xff) * 0x1p-52;  // near-2 significands
    *b = 1.0 + (double)(r2 >> 12) * 0x1p-52;
    *a = sig * *b;  // rounded: a/b lands next to the binade boundary
  } else {
    const double h = ldexp(1.0, -(int)((r1 >> 4) % 14) - 1);
    *a = h * ((double)(r1 >> 11) * 0x1p-53 - 0.5);
    *b = h * h * (0.25 + (double)(r2 >> 11) * 0x1p-53);
  }
}

__global__ void k_selftest(uint64_t n, uint64_t seed, unsigned long long* out) {
  unsigned long long bad = 0, worst_ulp = 0, worst3 = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    double a, b;
    operands(i, seed, &a, &b);
    if (div_safe(a) && div_safe(b) && b != 0.0) {
      const double q = div_rcp(a, b, __drcp_rn(b));
      if (__double_as_longlong(q) != __double_as_longlong(a / b)) ++bad;
    }
    if (__double_as_longlong(div3(a)) != __double_as_longlong(a / 3.0)) ++worst3;
    const double x = 3.14159265358979323846 * ((double)(mix64(seed ^ (i * 7 + 3)) >> 11) * 0x1p-52 - 1.0);
    const double s1 = sin_fast(x), s0 = sin(x);
    const long long d = __double_as_longlong(s1) - __double_as_longlong(s0);
    const unsigned long long ad = (unsigned long long)(d < 0 ? -d : d);
    if (ad > worst_ulp && (s0 > 0) == (s1 > 0)) worst_ulp = ad;
  }
  atomicAdd(out + 0, bad);
  atomicMax(out + 1, worst_ulp);
  atomicAdd(out + 2, worst3);
}

}  // namespace phfem

using namespace phfem;

// out[0] = division mismatches, out[1] = max ulp distance sin_fast vs sin,
// out[2] = division-by-3 mismatches (host memory, 3 entries)
PHFEM_API phfem_status phfem_selftest_fastmath(phfem_ctx* ctx, int64_t n, uint64_t seed,
                                               unsigned long long* out) {
  if (!ctx || !out || n < 0) return PHFEM_ERR_INVALID_ARGUMENT;
  unsigned long long* d = nullptr;
  PHFEM_TRY(dalloc(ctx, &d, 3));
  PHFEM_CUDA(ctx, cudaMemsetAsync(d, 0, 3 * sizeof(unsigned long long), ctx->stream));
  PHFEM_LAUNCH(ctx, "k_selftest", k_selftest<<<ctx->num_sms * 16, 256, 0, ctx->stream>>>((uint64_t)n, seed, d));
  PHFEM_CUDA(ctx, cudaMemcpyAsync(out, d, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
  PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  dfree(ctx, d);
  return PHFEM_OK;
}
