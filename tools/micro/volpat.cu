// volpat.cu — the store pattern of k_volume without its arithmetic: every
// warp writes, per 32-element chunk, 288 doubles to each of B, D, M, M0 and
// 96 doubles of load (16-byte stores), optionally reading the 12-byte
// element records.  Bounds what the blocks kernel can reach at this access
// pattern on one B200.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 volpat.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void st256(double2* p, double2 v) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v.x), "d"(v.y), "d"(v.x), "d"(v.y)
               : "memory");
}

// 256-bit stores (STG.256): the same pattern with half the store instructions
__global__ void k_pat256(double2* B, double2* D, double2* M, double2* M0, double2* L, long nchunks) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (long c0 = (long)blockIdx.x * nw + warp; c0 < nchunks; c0 += (long)gridDim.x * nw) {
    const double2 v = make_double2((double)c0, 1.0);
    double2* outs[5] = {B, D, M, M0, L};
#pragma unroll
    for (int s = 0; s < 5; ++s) {
      const int n4 = s == 4 ? 24 : 72;  // 32-byte units per chunk
      double2* o = outs[s] + c0 * 2 * n4;
      for (int i = lane; i < n4; i += 32) st256(o + 2 * i, v);
    }
  }
}

// G: 32-element chunks per warp iteration (the span written per stream)
template <int NS, bool CS>
__global__ void k_pat(double2* B, double2* D, double2* M, double2* M0, double2* L, const int* el, long nchunks,
                      int rd, int G) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double acc = 0;
  for (long c0 = ((long)blockIdx.x * nw + warp) * G; c0 < nchunks; c0 += (long)gridDim.x * nw * G) {
    if (rd)
      for (int g = 0; g < G; ++g) acc += el[(c0 + g) * 96 + lane] + el[(c0 + g) * 96 + 32 + lane] + el[(c0 + g) * 96 + 64 + lane];
    const double2 v = make_double2(acc, 1.0);
    double2* outs[5] = {B, D, M, M0, L};
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int n2 = s == 4 ? 48 : 144;
      double2* o = outs[s] + c0 * n2;
      for (int i = lane; i < n2 * G; i += 32) {
        if (CS) __stcs(o + i, v);
        else o[i] = v;
      }
    }
  }
}

int main() {
  const long nE = 134217728, nchunks = nE / 32;
  double2 *B, *D, *M, *M0, *L;
  int* el;
  cudaMalloc(&B, nE * 72);
  cudaMalloc(&D, nE * 72);
  cudaMalloc(&M, nE * 72);
  cudaMalloc(&M0, nE * 72);
  cudaMalloc(&L, nE * 24);
  cudaMalloc(&el, nE * 12);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes5 = nE * (4 * 72.0 + 24.0);
  for (int rd = 0; rd < 2; ++rd)
    for (int G : {1, 2, 4, 8})
    for (int mult : {6}) {
      for (int v = 0; v < 2; ++v) {
        float best = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {
          cudaEventRecord(e0);
          if (v == 0) k_pat<5, false><<<sms * mult, 128>>>(B, D, M, M0, L, el, nchunks, rd, G);
          else k_pat<5, true><<<sms * mult, 128>>>(B, D, M, M0, L, el, nchunks, rd, G);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (ms < best) best = ms;
        }
        const double moved = bytes5 + (rd ? nE * 12.0 : 0.0);
        printf("read=%d G=%d grid %2dx%d x128 %-6s %7.3f ms %8.1f GB/s\n", rd, G, mult, sms, v ? "st.cs" : "st", best,
               moved / best / 1e6);
      }
    }
  // stream count: the same chunk pattern into 1, 2, 3 or 4 of the block arrays
  for (int ns = 1; ns <= 4; ++ns) {
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(e0);
      if (ns == 1) k_pat<1, true><<<sms * 6, 128>>>(B, D, M, M0, L, el, nchunks, 0, 1);
      if (ns == 2) k_pat<2, true><<<sms * 6, 128>>>(B, D, M, M0, L, el, nchunks, 0, 1);
      if (ns == 3) k_pat<3, true><<<sms * 6, 128>>>(B, D, M, M0, L, el, nchunks, 0, 1);
      if (ns == 4) k_pat<4, true><<<sms * 6, 128>>>(B, D, M, M0, L, el, nchunks, 0, 1);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("streams=%d (72 B/elem each) %7.3f ms %8.1f GB/s\n", ns, best, nE * 72.0 * ns / best / 1e6);
  }
  for (int mult : {4, 6, 8}) {
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(e0);
      k_pat256<<<sms * mult, 128>>>(B, D, M, M0, L, nchunks);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("st.256 grid %2dx%d x128 %7.3f ms %8.1f GB/s\n", mult, sms, best, bytes5 / best / 1e6);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
