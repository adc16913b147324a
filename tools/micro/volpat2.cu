// volpat2.cu — why the k_volume store pattern (five output streams, each warp
// writing a 32-element chunk of every stream) reaches ~6.2 TB/s while a
// single sequential sweep writes at ~7 TB/s: occupancy sweep of the chunk
// pattern, the five streams as grid-stride sweeps, and CTA-wide TMA bulk
// stores (cp.async.bulk.global.shared::cta) of 128-element chunks.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 volpat2.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

// (a) chunk pattern of k_volume: warp = 32 elements, per stream 288 / 96 doubles
__global__ void k_chunk(double2* B, double2* D, double2* M, double2* M0, double2* L, long nchunks) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (long c0 = (long)blockIdx.x * nw + warp; c0 < nchunks; c0 += (long)gridDim.x * nw) {
    const double2 v = make_double2((double)c0, 1.0);
    double2* outs[5] = {B, D, M, M0, L};
#pragma unroll
    for (int s = 0; s < 5; ++s) {
      const int n2 = s == 4 ? 48 : 144;
      double2* o = outs[s] + c0 * n2;
      for (int i = lane; i < n2; i += 32) __stcs(o + i, v);
    }
  }
}

// (b) five grid-stride sweeps interleaved (every thread 16 B per stream per trip)
__global__ void k_sweep5(double2* B, double2* D, double2* M, double2* M0, double2* L, long n2) {
  const double2 v = make_double2(1.0, 2.0);
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n2; i += (long)gridDim.x * blockDim.x) {
    __stcs(B + i, v);
    __stcs(D + i, v);
    __stcs(M + i, v);
    __stcs(M0 + i, v);
    if (i < n2 / 3) __stcs(L + i, v);
  }
}

// (c) CTA chunks of 128 elements staged in SMEM, one thread bulk-stores each
// stream's contiguous span (9216 B / 3072 B); NB-deep ring of stage buffers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
template <int NB>
__global__ void __launch_bounds__(128) k_tma(double* B, double* D, double* M, double* M0, double* L, long ntiles) {
  extern __shared__ __align__(128) double sm[];  // NB x (4 x 1152 + 384) doubles
  const int per = 4 * 1152 + 384;
  int slot = 0;
  for (long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    double* buf = sm + slot * per;
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NB - 1) : "memory");
    __syncthreads();
    for (int i = threadIdx.x; i < per; i += 128) buf[i] = (double)(t + i);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      double* outs[5] = {B, D, M, M0, L};
#pragma unroll
      for (int s = 0; s < 5; ++s) {
        const int nd = s == 4 ? 384 : 1152;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(outs[s] + t * nd),
                     "r"(smem_u32(buf + s * 1152)), "r"(nd * 8)
                     : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    slot = (slot + 1) % NB;
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const long nE = 134217728, nchunks = nE / 32;
  double2 *B, *D, *M, *M0, *L;
  cudaMalloc(&B, nE * 72);
  cudaMalloc(&D, nE * 72);
  cudaMalloc(&M, nE * 72);
  cudaMalloc(&M0, nE * 72);
  cudaMalloc(&L, nE * 24);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes5 = nE * (4 * 72.0 + 24.0);
  auto timeit = [&](auto launch) {
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    return best;
  };
  for (int bps : {4, 6, 8, 12, 16}) {
    const float ms = timeit([&] { k_chunk<<<sms * bps, 128>>>(B, D, M, M0, L, nchunks); });
    printf("(a) chunk pattern   %2d x 128 thr/SM  %7.3f ms %8.1f GB/s\n", bps, ms, bytes5 / ms / 1e6);
  }
  for (int bps : {4, 8, 16}) {
    const float ms = timeit([&] { k_sweep5<<<sms * bps, 256>>>(B, D, M, M0, L, nE * 72 / 16); });
    printf("(b) 5 sweeps        %2d x 256 thr/SM  %7.3f ms %8.1f GB/s\n", bps, ms, bytes5 / ms / 1e6);
  }
  const int per_bytes = (4 * 1152 + 384) * 8;
  cudaFuncSetAttribute(k_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * per_bytes);
  cudaFuncSetAttribute(k_tma<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * per_bytes);
  for (int bps : {1, 2, 3, 4}) {
    float ms = timeit([&] { k_tma<2><<<sms * bps, 128, 2 * per_bytes>>>((double*)B, (double*)D, (double*)M, (double*)M0, (double*)L, nE / 128); });
    printf("(c) TMA bulk, ring 2 %d CTA/SM       %7.3f ms %8.1f GB/s\n", bps, ms, bytes5 / ms / 1e6);
    if (bps <= 2) {
      ms = timeit([&] { k_tma<3><<<sms * bps, 128, 3 * per_bytes>>>((double*)B, (double*)D, (double*)M, (double*)M0, (double*)L, nE / 128); });
      printf("(c) TMA bulk, ring 3 %d CTA/SM       %7.3f ms %8.1f GB/s\n", bps, ms, bytes5 / ms / 1e6);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
