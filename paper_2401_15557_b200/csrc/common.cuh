// common.cuh — shared plumbing for the sm_100a kernels behind include/phfem_gpu.h:
// the context (device, stream, stream-ordered pool, device error words), status
// helpers and the block/device scan primitives the edge and element passes use.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/phfem_gpu.h"

#define PHFEM_API extern "C" __attribute__((visibility("default")))

// Device-side error words, one per failure family.  Each holds an ordering
// key (smaller = what the reference would have hit first) and is merged with
// atomicMin, so the host reports exactly the reference's first exception.
struct phfem_dev_errors {
  unsigned long long topo;      // (hi<<33)|(lo<<2)|(dup<<1)|dir, canonical order
  unsigned long long classify;  // (list position<<2)|code
  unsigned long long degenerate;// element id
  unsigned long long load_nan;  // element id
  unsigned long long flux_nan;  // neumann list position
  unsigned long long misc;      // refine mismatch etc.
  unsigned long long counters[10];  // small per-call results (E, nI, nB, max bucket, dup flags...)
};

struct phfem_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaMemPool_t pool = nullptr;
  phfem_dev_errors* derr = nullptr;   // device
  phfem_dev_errors* dderr = nullptr;  // device: errors deferred to the end of a pipeline call
  phfem_dev_errors* herr = nullptr;   // pinned host mirror
  int64_t launches = 0;
  int num_sms = 148;
  std::string message;
  // per-launch CUDA-event timing (phfem_ctx_profile): events recorded on the
  // ctx stream around every kernel, aggregated per kernel name on read
  bool prof = false;
  struct Rec {
    const char* name;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> free_events;
  // size-bucketed cache of freed blocks (stream-ordered reuse on ctx->stream):
  // repeated pipeline calls get the same blocks back instead of growing /
  // remapping the pool (which costs tens of ms per call at L13 sizes)
  std::unordered_map<size_t, std::vector<void*>> cache;
  std::unordered_map<void*, size_t> block_size;
  size_t cached_bytes = 0;
  // dynamic-SMEM opt-ins already applied on this ctx's device (kernel ->
  // bytes); cudaFuncSetAttribute is per device, so the cache lives here
  std::unordered_map<const void*, size_t> smem_optin;
  // upper bound on the edge pass's bucket width bs (bits of max node per
  // bucket; 8 = a tile is one bucket when the packed item leaves 8 bits).
  // Lowered only to exercise the multi-sub-bucket tile path on small meshes
  // (env PHFEM_EG_MAX_BS at ctx creation, or phfem_ctx_set_eg_max_bs)
  int eg_max_bs = 8;
  // guard mode (env PHFEM_GUARD=1 at ctx creation; the device check that
  // stands in for compute-sanitizer, which this pool does not allow): every
  // block gets kGuardBytes red zones on both sides filled with 0xA5 and its
  // payload poisoned (PHFEM_GUARD_POISON, default 0xff: NaN / -1), blocks are
  // never recycled, and every free checks the red zones on the device; the
  // first violated block's serial is reported by errors_fetch / ctx_sync.
  bool guard = false;
  int guard_poison = 0xff;
  unsigned int* guard_bad = nullptr;  // device: min serial of a violated block (~0u: none)
  unsigned int guard_serial = 0;
  struct GuardBlock {
    void* base;
    size_t bytes, total;
    unsigned serial;
  };
  std::unordered_map<void*, GuardBlock> guard_blocks;
  std::unordered_map<unsigned, size_t> guard_sizes;  // serial -> payload bytes (reports)
};

namespace phfem {

phfem_status set_error(phfem_ctx* ctx, phfem_status st, const char* fmt, ...);
phfem_status cuda_fail(phfem_ctx* ctx, cudaError_t e, const char* where);

#define PHFEM_CUDA(ctx, call)                                   \
  do {                                                          \
    cudaError_t _e = (call);                                    \
    if (_e != cudaSuccess) return ::phfem::cuda_fail(ctx, _e, #call); \
  } while (0)

#define PHFEM_CHECK_LAUNCH(ctx)                                         \
  do {                                                                  \
    (ctx)->launches++;                                                  \
    cudaError_t _e = cudaGetLastError();                                \
    if (_e != cudaSuccess) return ::phfem::cuda_fail(ctx, _e, "kernel launch"); \
  } while (0)

// Launch + error check + (when profiling) a CUDA-event pair around the launch.
#define PHFEM_LAUNCH(ctx, name, ...)        \
  do {                                      \
    ::phfem::KTimer _kt(ctx, name);         \
    __VA_ARGS__;                            \
    PHFEM_CHECK_LAUNCH(ctx);                \
  } while (0)

// Programmatic dependent launch (sm_90+).  A kernel launched through
// PHFEM_LAUNCH_PDL may be scheduled while its predecessor on the stream is
// still draining (its CTAs wait in pdl_wait() until the predecessor grid has
// completed and its writes are visible), so the launch latency of a chain of
// short kernels overlaps the previous kernel's tail.  Every kernel launched
// that way calls pdl_wait() before its first global access and then
// pdl_trigger() (its own dependents may launch once all its CTAs started);
// both are no-ops in a normal launch.  PHFEM_PDL=0 turns the attribute off.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
bool pdl_enabled();
// PDL-chained zero fill of int32 / 16-byte-aligned device copy (ctx.cu)
phfem_status zero_i32(phfem_ctx* ctx, int32_t* p, int64_t n);
phfem_status copy_d2d(phfem_ctx* ctx, void* dst, const void* src, size_t bytes);

#define PHFEM_LAUNCH_PDL(ctx, name, kern, grid, block, smem, ...)                               \
  do {                                                                                          \
    ::phfem::KTimer _kt(ctx, name);                                                             \
    cudaLaunchConfig_t _cfg = {};                                                               \
    _cfg.gridDim = dim3(grid);                                                                  \
    _cfg.blockDim = dim3(block);                                                                \
    _cfg.dynamicSmemBytes = (smem);                                                             \
    _cfg.stream = (ctx)->stream;                                                                \
    cudaLaunchAttribute _at[1];                                                                 \
    _at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                             \
    _at[0].val.programmaticStreamSerializationAllowed = ::phfem::pdl_enabled() ? 1 : 0;         \
    _cfg.attrs = _at;                                                                           \
    _cfg.numAttrs = 1;                                                                          \
    cudaLaunchKernelEx(&_cfg, kern, __VA_ARGS__);                                               \
    PHFEM_CHECK_LAUNCH(ctx);                                                                    \
  } while (0)

#define PHFEM_TRY(expr)                 \
  do {                                  \
    phfem_status _s = (expr);           \
    if (_s != PHFEM_OK) return _s;      \
  } while (0)

phfem_status raw_alloc(phfem_ctx* ctx, void** p, size_t bytes);

// Opt a kernel into `bytes` of dynamic shared memory on the ctx's device
// (needed above 48 KB); applied once per (ctx, kernel), errors reported.
phfem_status smem_optin(phfem_ctx* ctx, const void* fn, size_t bytes, const char* name);
void raw_free(phfem_ctx* ctx, void* p);
void cache_flush(phfem_ctx* ctx);

template <typename T>
phfem_status dalloc(phfem_ctx* ctx, T** p, size_t count) {
  if (count == 0) count = 1;
  return raw_alloc(ctx, (void**)p, count * sizeof(T));
}

template <typename T>
void dfree(phfem_ctx* ctx, T*& p) {
  if (p && ctx) raw_free(ctx, (void*)p);
  p = nullptr;
}

// RAII timer: records an event pair around the launches in its scope when
// profiling is enabled on the ctx.
class KTimer {
 public:
  KTimer(phfem_ctx* ctx, const char* name);
  ~KTimer();

 private:
  phfem_ctx* ctx_;
  const char* name_;
  cudaEvent_t a_ = nullptr;
};

// Reset the device error words (async) / fetch them (sync).
phfem_status errors_reset(phfem_ctx* ctx);
phfem_status errors_fetch(phfem_ctx* ctx);
// guard mode: report a red-zone violation seen so far (synchronises)
phfem_status guard_check(phfem_ctx* ctx);

inline int grid_for(int64_t n, int block, int max_blocks) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > max_blocks) g = max_blocks;
  return (int)g;
}

// ---------------------------------------------------------------------------
// Device-wide exclusive scan of int32 counts (3 launches: tile reduce, scan of
// tile sums, downsweep).  out may alias in.  Writes the total to *total_dev.
phfem_status scan_exclusive_i32(phfem_ctx* ctx, const int32_t* in, int32_t* out, int64_t n,
                                int32_t* total_dev);
// up to 4 arrays of the same length, one launch per phase; in[a] == out[a] allowed
phfem_status scan_exclusive_i32_set(phfem_ctx* ctx, int count, const int32_t* const* in, int32_t* const* out,
                                    int64_t n, int32_t* const* total_dev);

// Stable LSD radix sort of (key, u32 value) pairs over key bits [0, end_bit)
// (radix_sort.cu; hand-written, no library sort).  Inputs are not modified.
phfem_status radix_sort_pairs_u64(phfem_ctx* ctx, const uint64_t* kin, uint64_t* kout, const uint32_t* vin,
                                  uint32_t* vout, int64_t n, int end_bit);
phfem_status radix_sort_pairs_u32(phfem_ctx* ctx, const uint32_t* kin, uint32_t* kout, const uint32_t* vin,
                                  uint32_t* vout, int64_t n, int end_bit);

}  // namespace phfem

// ---------------------------------------------------------------------------
// Warp / block helpers usable in every .cu
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(0xffffffffu, v, o);
    if ((int)lane_id() >= o) v += n;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_reduce_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Edge id of the node pair (a, b) through the max-node grouping table of
// build_topology: edges with larger node hi occupy ids [nes[hi], nes[hi+1]),
// ascending by smaller node.  -1 when (a, b) is not an edge (the reference's
// node_pair_to_edge contract, edge_topology.cpp:36-43).
__device__ __forceinline__ int find_edge(const int32_t* __restrict__ nes,
                                         const int32_t* __restrict__ edge_nodes, int nC, int a,
                                         int b) {
  const int lo = a < b ? a : b;
  const int hi = a < b ? b : a;
  if (lo < 0 || hi >= nC) return -1;
  int l = nes[hi], r = nes[hi + 1];  // edges with max node hi, ascending min node
  while (l < r) {
    const int mid = (l + r) >> 1;
    const int x = edge_nodes[2 * mid], y = edge_nodes[2 * mid + 1];
    const int mn = x < y ? x : y;
    if (mn < lo) l = mid + 1;
    else r = mid;
  }
  if (l < nes[hi + 1]) {
    const int x = edge_nodes[2 * l], y = edge_nodes[2 * l + 1];
    if ((x < y ? x : y) == lo) return l;
  }
  return -1;
}


// Block exclusive scan of one value per thread; blockDim.x multiple of 32,
// <= 1024.  `smem` needs 33 slots.  Returns exclusive prefix, *total = sum.
template <typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* smem, T* total) {
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  T inc = warp_inclusive_scan(v);
  if (lane_id() == 31) smem[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = (lane_id() < (unsigned)nwarps) ? smem[lane_id()] : T(0);
    T wi = warp_inclusive_scan(w);
    if (lane_id() < (unsigned)nwarps) smem[lane_id()] = wi - w;
    if (lane_id() == 31) smem[32] = wi;
  }
  __syncthreads();
  T res = smem[warp] + inc - v;
  *total = smem[32];
  __syncthreads();
  return res;
}

// ---------------------------------------------------------------------------
// Decoupled look-back over tiles (single-pass scans of the edge passes).
// Status word per tile: 2 flag bits (0 = not ready, 1 = aggregate, 2 =
// inclusive prefix) + two 31-bit payloads.  Tiles are claimed in launch order
// through an atomic ticket, so every predecessor is running or done.
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagPre = 2ull << 62;
constexpr uint64_t kPay31 = (1ull << 31) - 1;

__device__ __forceinline__ uint64_t ld_volatile_u64(const unsigned long long* p) {
  return *(const volatile unsigned long long*)p;
}
__device__ __forceinline__ void st_volatile_u64(unsigned long long* p, uint64_t v) {
  *(volatile unsigned long long*)p = v;
}

// Decoupled look-back by warp 0 of the CTA owning tile b.  Returns the
// exclusive (first << 32 | second) prefix of the two payloads.
// Wide variant: every lane inspects V consecutive predecessors, so one L2
// round trip covers 32 V tiles — the frontier of inclusive prefixes advances
// 32 V tiles per round trip instead of 32 (the look-back chain otherwise caps
// the throughput of kernels with short tiles).
template <int V>
__device__ __forceinline__ uint64_t lookback_wide(unsigned long long* status, int b, uint32_t agg_e,
                                                  uint32_t agg_b) {
  const unsigned lane = lane_id();
  if (lane == 0) {
    __threadfence();
    st_volatile_u64(&status[b], (b == 0 ? kFlagPre : kFlagAgg) | ((uint64_t)agg_e << 31) | agg_b);
  }
  if (b == 0) return 0;
  uint64_t ex_e = 0, ex_b = 0;
  int top = b - 1;
  while (true) {
    uint64_t w[V];
    while (true) {
      bool ready = true;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int idx = top - (int)lane * V - v;
        w[v] = idx >= 0 ? ld_volatile_u64(&status[idx]) : kFlagPre;
        ready = ready && (w[v] >> 62) != 0;
      }
      if (__all_sync(0xffffffffu, ready)) break;
      __nanosleep(32);
    }
    int vf = V;  // nearest inclusive prefix among this lane's entries
#pragma unroll
    for (int v = V - 1; v >= 0; --v)
      if ((w[v] >> 62) == 2) vf = v;
    const unsigned pmask = __ballot_sync(0xffffffffu, vf < V);
    const int fl = pmask ? __ffs(pmask) - 1 : 32;
    const int upto = (int)lane < fl ? V - 1 : ((int)lane == fl ? vf : -1);
    uint64_t ve = 0, vb = 0;
#pragma unroll
    for (int v = 0; v < V; ++v)
      if (v <= upto) {
        ve += (w[v] >> 31) & kPay31;
        vb += w[v] & kPay31;
      }
    ex_e += warp_reduce_sum(ve);
    ex_b += warp_reduce_sum(vb);
    if (pmask) break;
    top -= 32 * V;
  }
  if (lane == 0) {
    __threadfence();
    st_volatile_u64(&status[b], kFlagPre | ((ex_e + agg_e) << 31) | (ex_b + agg_b));
  }
  return (ex_e << 32) | ex_b;
}

__device__ __forceinline__ uint64_t eg_lookback(unsigned long long* status, int b, uint32_t agg_e,
                                                uint32_t agg_b) {
  const unsigned lane = lane_id();
  if (lane == 0) {
    __threadfence();
    st_volatile_u64(&status[b], (b == 0 ? kFlagPre : kFlagAgg) | ((uint64_t)agg_e << 31) | agg_b);
  }
  if (b == 0) return 0;
  uint64_t ex_e = 0, ex_b = 0;
  int top = b - 1;
  while (true) {
    const int idx = top - (int)lane;
    uint64_t w;
    while (true) {
      w = idx >= 0 ? ld_volatile_u64(&status[idx]) : kFlagPre;
      if (!__any_sync(0xffffffffu, (w >> 62) == 0)) break;
      __nanosleep(32);
    }
    const unsigned pmask = __ballot_sync(0xffffffffu, (w >> 62) == 2);
    const int first_p = pmask ? __ffs(pmask) - 1 : 32;
    const bool take = (int)lane <= first_p;
    const uint64_t ve = take ? ((w >> 31) & kPay31) : 0;
    const uint64_t vb = take ? (w & kPay31) : 0;
    ex_e += warp_reduce_sum(ve);
    ex_b += warp_reduce_sum(vb);
    if (pmask) break;
    top -= 32;
  }
  if (lane == 0) {
    __threadfence();
    st_volatile_u64(&status[b], kFlagPre | ((ex_e + agg_e) << 31) | (ex_b + agg_b));
  }
  return (ex_e << 32) | ex_b;
}
