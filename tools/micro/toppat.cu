// toppat.cu — the store pattern of the fine-topology + C emit (k_rl_level<1>,
// k_eg_emit) without their loads and arithmetic: per fine edge f the
// coalesced streams edge_nodes, edge_elements, ltp, ltm, interior,
// retained_pos, retained_edges, row_ptr, C col (4) and val (4), plus the two
// elem_edge entries of its elements (scattered 4-byte stores).  Scatter
// models: none, local (slots near 2f, as in a refined square), random.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 toppat.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned mix(unsigned x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

__global__ void k_pat(long E, int mode, int2* en, int2* el, int* ltp, int* ltm, int* inter, int* rpos, int* red,
                      int* rptr, int4* col, double2* val, int* ee, long nslots) {
  for (long f = blockIdx.x * (long)blockDim.x + threadIdx.x; f < E; f += (long)gridDim.x * blockDim.x) {
    const int fi = (int)f;
    en[f] = make_int2(fi, fi + 1);
    el[f] = make_int2(fi >> 1, fi >> 2);
    ltp[f] = fi & 3;
    ltm[f] = fi & 1;
    inter[f] = fi;
    rpos[f] = fi;
    red[f] = fi;
    rptr[f] = 4 * fi;
    col[f] = make_int4(fi, fi + 1, fi + 2, fi + 3);
    __stcs(val + 2 * f, make_double2(1.0, 1.0));
    __stcs(val + 2 * f + 1, make_double2(-1.0, -1.0));
    if (mode) {
      long s0, s1;
      if (mode == 1) {  // local: slots within +-192 of 2f (4 fine elements per parent)
        const unsigned h = mix((unsigned)f);
        s0 = 2 * f + (long)(h & 255) - 128;
        s1 = 2 * f + (long)((h >> 8) & 255) - 128;
      } else {          // random over the whole array
        s0 = (long)(mix((unsigned)f) % (unsigned)nslots);
        s1 = (long)(mix((unsigned)f ^ 0x9e3779b9u) % (unsigned)nslots);
      }
      s0 = s0 < 0 ? 0 : (s0 >= nslots ? nslots - 1 : s0);
      s1 = s1 < 0 ? 0 : (s1 >= nslots ? nslots - 1 : s1);
      ee[s0] = fi;
      ee[s1] = ~fi;
    }
  }
}

int main() {
  const long E = 201342976, nslots = 3L * 134217728;
  int2 *en, *el;
  int *ltp, *ltm, *inter, *rpos, *red, *rptr, *ee;
  int4* col;
  double2* val;
  cudaMalloc(&en, E * 8); cudaMalloc(&el, E * 8); cudaMalloc(&ltp, E * 4); cudaMalloc(&ltm, E * 4);
  cudaMalloc(&inter, E * 4); cudaMalloc(&rpos, E * 4); cudaMalloc(&red, E * 4); cudaMalloc(&rptr, E * 4);
  cudaMalloc(&col, E * 16); cudaMalloc(&val, E * 32); cudaMalloc(&ee, nslots * 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; ++mode)
    for (int mult : {4, 8, 16}) {
      float best = 1e30f;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        k_pat<<<sms * mult, 256>>>(E, mode, en, el, ltp, ltm, inter, rpos, red, rptr, col, val, ee, nslots);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      const double bytes = E * (8 + 8 + 4 + 4 + 4 + 4 + 4 + 4 + 16 + 32.0) + (mode ? E * 8.0 : 0.0);
      const char* nm[] = {"no scatter", "local", "random"};
      printf("%-10s grid %2dx%d  %7.3f ms %8.1f GB/s (useful bytes)\n", nm[mode], mult, sms, best, bytes / best / 1e6);
    }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
