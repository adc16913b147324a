// membw.cu — HBM microbenchmark on one B200: write-only, read-only and copy
// streams (16-byte accesses, grid = k x 148 SMs), to bound the write-heavy
// assembly kernels.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 membw.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_write(double2* p, size_t n, int cs) {
  const double2 v = make_double2(1.0, 2.0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    if (cs) __stcs(p + i, v); else p[i] = v;
}
__global__ void k_read(const double2* p, size_t n, double* sink) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldcs(p + i);
    s += v.x;
  }
  if (s == 12345.0) *sink = s;
}
__global__ void k_copy(const double2* a, double2* b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(b + i, __ldcs(a + i));
}

int main() {
  const size_t bytes = size_t(20) << 30, n = bytes / 16;
  double2 *a, *b;
  double* sink;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMalloc(&sink, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int mult : {4, 8, 16, 32}) {
    for (int test = 0; test < 4; ++test) {
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        if (test == 0) k_write<<<sms * mult, 256>>>(a, n, 0);
        if (test == 1) k_write<<<sms * mult, 256>>>(a, n, 1);
        if (test == 2) k_read<<<sms * mult, 256>>>(a, n, sink);
        if (test == 3) k_copy<<<sms * mult, 256>>>(a, b, n);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      const double moved = test == 3 ? 2.0 * bytes : (double)bytes;
      const char* nm[] = {"write", "write_cs", "read", "copy(r+w)"};
      printf("grid %2dx%d  %-10s %8.1f GB/s\n", mult, sms, nm[test], moved / best / 1e6);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
