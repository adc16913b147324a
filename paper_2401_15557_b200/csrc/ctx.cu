// ctx.cu — context, stream-ordered memory, error plumbing and the device-wide
// scan used by the edge / classification passes.
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace phfem {

// Stream-ordered fill / copy as PDL-chained kernels (a memset / memcpy node
// between two kernels would end the programmatic overlap of the chain).
__global__ void k_zero_i32(int32_t* __restrict__ p, int64_t n) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 0;
}
__global__ void k_copy16(int4* __restrict__ dst, const int4* __restrict__ src, int64_t n) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __ldcs(src + i);
}
phfem_status zero_i32(phfem_ctx* ctx, int32_t* p, int64_t n) {
  if (n <= 0) return PHFEM_OK;
  PHFEM_LAUNCH_PDL(ctx, "k_zero_i32", k_zero_i32, grid_for(n, 256, ctx->num_sms * 8), 256, 0, p, n);
  return PHFEM_OK;
}
phfem_status copy_d2d(phfem_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return PHFEM_OK;
  if (((uintptr_t)dst | (uintptr_t)src | bytes) & 15u) {
    PHFEM_CUDA(ctx, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
    return PHFEM_OK;
  }
  const int64_t n = (int64_t)(bytes / 16);
  PHFEM_LAUNCH_PDL(ctx, "k_copy16", k_copy16, grid_for(n, 256, ctx->num_sms * 32), 256, 0, (int4*)dst,
                   (const int4*)src, n);
  return PHFEM_OK;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PHFEM_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}


phfem_status set_error(phfem_ctx* ctx, phfem_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (ctx) ctx->message = buf;
  return st;
}

phfem_status cuda_fail(phfem_ctx* ctx, cudaError_t e, const char* where) {
  cudaGetLastError();
  return set_error(ctx, e == cudaErrorMemoryAllocation ? PHFEM_ERR_OOM : PHFEM_ERR_CUDA,
                   "phfem: CUDA error %s (%s) at %s", cudaGetErrorName(e), cudaGetErrorString(e),
                   where);
}

phfem_status errors_reset(phfem_ctx* ctx) {
  phfem_dev_errors init;
  memset(&init, 0xff, sizeof init);
  memset(init.counters, 0, sizeof init.counters);
  memcpy(ctx->herr, &init, sizeof init);
  PHFEM_CUDA(ctx, cudaMemcpyAsync(ctx->derr, ctx->herr, sizeof init, cudaMemcpyHostToDevice,
                                  ctx->stream));
  return PHFEM_OK;
}

phfem_status errors_fetch(phfem_ctx* ctx) {
  PHFEM_CUDA(ctx, cudaMemcpyAsync(ctx->herr, ctx->derr, sizeof(phfem_dev_errors),
                                  cudaMemcpyDeviceToHost, ctx->stream));
  PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (ctx->guard) return guard_check(ctx);
  return PHFEM_OK;
}

constexpr size_t kGuardBytes = 4096;
constexpr unsigned char kGuardFill = 0xA5;

// red zones [a0, a0 + n0) and [a1, a1 + n1) must still hold kGuardFill
__global__ void k_guard_check(const unsigned char* __restrict__ a0, size_t n0, const unsigned char* __restrict__ a1,
                              size_t n1, unsigned serial, unsigned int* __restrict__ bad) {
  bool ok = true;
  for (size_t i = threadIdx.x; i < n0; i += blockDim.x) ok &= a0[i] == kGuardFill;
  for (size_t i = threadIdx.x; i < n1; i += blockDim.x) ok &= a1[i] == kGuardFill;
  if (!ok) atomicMin(bad, serial);
}

phfem_status guard_check(phfem_ctx* ctx) {
  unsigned int h = ~0u;
  PHFEM_CUDA(ctx, cudaMemcpyAsync(&h, ctx->guard_bad, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
  PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (h != ~0u) {
    auto it = ctx->guard_sizes.find(h);
    return set_error(ctx, PHFEM_ERR_CUDA,
                     "phfem guard: out-of-bounds write into the red zone of device block #%u (%zu bytes)", h,
                     it == ctx->guard_sizes.end() ? (size_t)0 : it->second);
  }
  return PHFEM_OK;
}

static phfem_status guard_alloc(phfem_ctx* ctx, void** p, size_t bytes) {
  const size_t payload = (bytes + 255) / 256 * 256;
  const size_t total = payload + 2 * kGuardBytes;
  void* base = nullptr;
  cudaError_t e = cudaMallocFromPoolAsync(&base, total, ctx->pool, ctx->stream);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_error(ctx, PHFEM_ERR_OOM, "phfem: device allocation of %zu bytes failed (%s)", bytes,
                     cudaGetErrorString(e));
  }
  unsigned char* b = (unsigned char*)base;
  PHFEM_CUDA(ctx, cudaMemsetAsync(b, kGuardFill, total, ctx->stream));
  PHFEM_CUDA(ctx, cudaMemsetAsync(b + kGuardBytes, ctx->guard_poison, bytes, ctx->stream));
  *p = b + kGuardBytes;
  const unsigned serial = ++ctx->guard_serial;
  ctx->guard_blocks[*p] = {base, bytes, total, serial};
  ctx->guard_sizes[serial] = bytes;
  return PHFEM_OK;
}

static bool guard_free(phfem_ctx* ctx, void* p) {
  auto it = ctx->guard_blocks.find(p);
  if (it == ctx->guard_blocks.end()) return false;
  const auto g = it->second;
  const unsigned char* b = (const unsigned char*)g.base;
  const unsigned char* tail = (const unsigned char*)p + g.bytes;
  k_guard_check<<<1, 256, 0, ctx->stream>>>(b, kGuardBytes, tail, g.total - kGuardBytes - g.bytes, g.serial,
                                            ctx->guard_bad);
  cudaFreeAsync(g.base, ctx->stream);
  ctx->guard_blocks.erase(it);
  return true;
}

phfem_status smem_optin(phfem_ctx* ctx, const void* fn, size_t bytes, const char* name) {
  auto it = ctx->smem_optin.find(fn);
  if (it != ctx->smem_optin.end() && it->second >= bytes) return PHFEM_OK;
  if (bytes > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return cuda_fail(ctx, e, name);
  }
  ctx->smem_optin[fn] = bytes;
  return PHFEM_OK;
}

static size_t round_size(size_t bytes) {
  const size_t g = bytes >= (size_t(1) << 20) ? (size_t(2) << 20) : 512;
  return (bytes + g - 1) / g * g;
}

phfem_status raw_alloc(phfem_ctx* ctx, void** p, size_t bytes) {
  *p = nullptr;
  if (ctx->guard) return guard_alloc(ctx, p, bytes);
  const size_t sz = round_size(bytes);
  auto it = ctx->cache.find(sz);
  if (it != ctx->cache.end() && !it->second.empty()) {
    *p = it->second.back();
    it->second.pop_back();
    ctx->cached_bytes -= sz;
    return PHFEM_OK;
  }
  cudaError_t e = cudaMallocFromPoolAsync(p, sz, ctx->pool, ctx->stream);
  if (e != cudaSuccess) {  // give the cached blocks back and retry once
    cudaGetLastError();
    cache_flush(ctx);
    e = cudaMallocFromPoolAsync(p, sz, ctx->pool, ctx->stream);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    *p = nullptr;
    return set_error(ctx, PHFEM_ERR_OOM, "phfem: device allocation of %zu bytes failed (%s)", bytes,
                     cudaGetErrorString(e));
  }
  ctx->block_size[*p] = sz;
  return PHFEM_OK;
}

void raw_free(phfem_ctx* ctx, void* p) {
  if (ctx->guard && guard_free(ctx, p)) return;
  auto it = ctx->block_size.find(p);
  if (it == ctx->block_size.end()) {  // not ours: hand back to the stream-ordered pool
    cudaFreeAsync(p, ctx->stream);
    return;
  }
  ctx->cache[it->second].push_back(p);
  ctx->cached_bytes += it->second;
}

void cache_flush(phfem_ctx* ctx) {
  for (auto& kv : ctx->cache)
    for (void* q : kv.second) {
      cudaFreeAsync(q, ctx->stream);
      ctx->block_size.erase(q);
    }
  ctx->cache.clear();
  ctx->cached_bytes = 0;
  cudaStreamSynchronize(ctx->stream);
  cudaMemPoolTrimTo(ctx->pool, 0);
}

static cudaEvent_t take_event(phfem_ctx* ctx) {
  if (!ctx->free_events.empty()) {
    cudaEvent_t e = ctx->free_events.back();
    ctx->free_events.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

KTimer::KTimer(phfem_ctx* ctx, const char* name) : ctx_(ctx), name_(name) {
  if (ctx_ && ctx_->prof) {
    a_ = take_event(ctx_);
    cudaEventRecord(a_, ctx_->stream);
  }
}

KTimer::~KTimer() {
  if (a_) {
    cudaEvent_t b = take_event(ctx_);
    cudaEventRecord(b, ctx_->stream);
    ctx_->recs.push_back({name_, a_, b});
  }
}

// ---------------------------------------------------------------------------
// Scan: tiles of 4096 int32 (1024 threads x 4).
constexpr int kScanThreads = 1024;
constexpr int kScanPer = 4;
constexpr int kScanTile = kScanThreads * kScanPer;

__global__ void __launch_bounds__(kScanThreads) k_scan_tile_sums(const int32_t* __restrict__ in,
                                                                 int64_t n,
                                                                 int32_t* __restrict__ sums) {
  __shared__ int32_t sm[33];
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  int32_t v = 0;
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    const int64_t i = base + (int64_t)k * kScanThreads + threadIdx.x;
    if (i < n) v += in[i];
  }
  int32_t tot;
  block_exclusive_scan(v, sm, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// Single-block exclusive scan of the tile sums (any length).
__global__ void __launch_bounds__(kScanThreads) k_scan_sums(int32_t* sums, int64_t n,
                                                            int32_t* total) {
  __shared__ int32_t sm[33];
  int32_t carry = 0;
  for (int64_t base = 0; base < n; base += kScanThreads) {
    const int64_t i = base + threadIdx.x;
    const int32_t v = i < n ? sums[i] : 0;
    int32_t tot;
    const int32_t ex = block_exclusive_scan(v, sm, &tot);
    if (i < n) sums[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_down(const int32_t* in, int32_t* out,
                                                            int64_t n,
                                                            const int32_t* __restrict__ sums) {
  __shared__ int32_t sm[33];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanPer;
  int32_t v[kScanPer];
  int32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    const int64_t i = base + k;
    v[k] = i < n ? in[i] : 0;
    s += v[k];
  }
  int32_t tot;
  int32_t ex = block_exclusive_scan(s, sm, &tot) + sums[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    const int64_t i = base + k;
    if (i < n) out[i] = ex;
    ex += v[k];
  }
}

// Small arrays (tile counts, bucket offsets of small meshes): one CTA walks
// the array in 4096-entry chunks with a carry — one launch instead of three
// (the three-launch scan cost ~15 us even for a few hundred entries, 28 of
// them per config-2 pipeline).
constexpr int64_t kScanSmall = 8 * kScanTile;
__global__ void __launch_bounds__(kScanThreads) k_scan_small(const int32_t* in, int32_t* out, int64_t n,
                                                             int32_t* total) {
  pdl_wait();
  pdl_trigger();
  __shared__ int32_t sm[33];
  int32_t carry = 0;
  for (int64_t c0 = 0; c0 < n; c0 += kScanTile) {
    const int64_t base = c0 + (int64_t)threadIdx.x * kScanPer;
    int32_t v[kScanPer];
    int32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanPer; ++k) {
      v[k] = base + k < n ? in[base + k] : 0;
      s += v[k];
    }
    int32_t tot;
    int32_t ex = carry + block_exclusive_scan(s, sm, &tot);
#pragma unroll
    for (int k = 0; k < kScanPer; ++k) {
      if (base + k < n) out[base + k] = ex;
      ex += v[k];
    }
    carry += tot;
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

// Up to kScanSet arrays of the same length scanned by one launch per phase
// (blockIdx.y / blockIdx.x = the array): the per-tile counts of the edge and
// refinement passes come in threes, each scan a few microseconds of launch.
constexpr int kScanSet = 4;
struct ScanSet {
  const int32_t* in[kScanSet];
  int32_t* out[kScanSet];
  int32_t* total[kScanSet];
};

__global__ void __launch_bounds__(kScanThreads) k_scan_small_set(ScanSet S, int64_t n) {
  pdl_wait();
  pdl_trigger();
  const int a = blockIdx.x;
  const int32_t* in = S.in[a];
  int32_t* out = S.out[a];
  __shared__ int32_t sm[33];
  int32_t carry = 0;
  for (int64_t c0 = 0; c0 < n; c0 += kScanTile) {
    const int64_t base = c0 + (int64_t)threadIdx.x * kScanPer;
    int32_t v[kScanPer];
    int32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanPer; ++k) {
      v[k] = base + k < n ? in[base + k] : 0;
      s += v[k];
    }
    int32_t tot;
    int32_t ex = carry + block_exclusive_scan(s, sm, &tot);
#pragma unroll
    for (int k = 0; k < kScanPer; ++k) {
      if (base + k < n) out[base + k] = ex;
      ex += v[k];
    }
    carry += tot;
  }
  if (threadIdx.x == 0 && S.total[a]) *S.total[a] = carry;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_tile_sums_set(ScanSet S, int64_t n, int32_t* __restrict__ sums,
                                                                     int64_t tiles) {
  pdl_wait();
  pdl_trigger();
  __shared__ int32_t sm[33];
  const int a = blockIdx.y;
  const int32_t* in = S.in[a];
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  int32_t v = 0;
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    const int64_t i = base + (int64_t)k * kScanThreads + threadIdx.x;
    if (i < n) v += in[i];
  }
  int32_t tot;
  block_exclusive_scan(v, sm, &tot);
  if (threadIdx.x == 0) sums[a * tiles + blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_sums_set(int32_t* sums, int64_t tiles, ScanSet S) {
  pdl_wait();
  pdl_trigger();
  __shared__ int32_t sm[33];
  const int a = blockIdx.x;
  int32_t* sa = sums + a * tiles;
  int32_t carry = 0;
  for (int64_t base = 0; base < tiles; base += kScanThreads) {
    const int64_t i = base + threadIdx.x;
    const int32_t v = i < tiles ? sa[i] : 0;
    int32_t tot;
    const int32_t ex = block_exclusive_scan(v, sm, &tot);
    if (i < tiles) sa[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0 && S.total[a]) *S.total[a] = carry;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_down_set(ScanSet S, int64_t n,
                                                                const int32_t* __restrict__ sums, int64_t tiles) {
  pdl_wait();
  pdl_trigger();
  __shared__ int32_t sm[33];
  const int a = blockIdx.y;
  const int32_t* in = S.in[a];
  int32_t* out = S.out[a];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanPer;
  int32_t v[kScanPer];
  int32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    const int64_t i = base + k;
    v[k] = i < n ? in[i] : 0;
    s += v[k];
  }
  int32_t tot;
  int32_t ex = block_exclusive_scan(s, sm, &tot) + sums[a * tiles + blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    const int64_t i = base + k;
    if (i < n) out[i] = ex;
    ex += v[k];
  }
}

phfem_status scan_exclusive_i32_set(phfem_ctx* ctx, int count, const int32_t* const* in, int32_t* const* out,
                                    int64_t n, int32_t* const* total_dev) {
  if (count < 1 || count > kScanSet) return set_error(ctx, PHFEM_ERR_INVALID_ARGUMENT, "scan set size");
  ScanSet S;
  memset(&S, 0, sizeof S);
  for (int a = 0; a < count; ++a) {
    S.in[a] = in[a];
    S.out[a] = out[a];
    S.total[a] = total_dev ? total_dev[a] : nullptr;
  }
  if (n == 0) {
    for (int a = 0; a < count; ++a)
      if (S.total[a]) PHFEM_CUDA(ctx, cudaMemsetAsync(S.total[a], 0, sizeof(int32_t), ctx->stream));
    return PHFEM_OK;
  }
  if (n <= kScanSmall) {
    PHFEM_LAUNCH_PDL(ctx, "scan", k_scan_small_set, count, kScanThreads, 0, S, n);
    return PHFEM_OK;
  }
  const int64_t tiles = (n + kScanTile - 1) / kScanTile;
  int32_t* sums = nullptr;
  PHFEM_TRY(dalloc(ctx, &sums, tiles * count));
  PHFEM_LAUNCH_PDL(ctx, "scan", k_scan_tile_sums_set, dim3((unsigned)tiles, count), kScanThreads, 0, S, n, sums, tiles);
  PHFEM_LAUNCH_PDL(ctx, "scan", k_scan_sums_set, count, kScanThreads, 0, sums, tiles, S);
  PHFEM_LAUNCH_PDL(ctx, "scan", k_scan_down_set, dim3((unsigned)tiles, count), kScanThreads, 0, S, n,
                   (const int32_t*)sums, tiles);
  dfree(ctx, sums);
  return PHFEM_OK;
}

phfem_status scan_exclusive_i32(phfem_ctx* ctx, const int32_t* in, int32_t* out, int64_t n,
                                int32_t* total_dev) {
  const int64_t tiles = (n + kScanTile - 1) / kScanTile;
  if (n == 0) {
    if (total_dev) PHFEM_CUDA(ctx, cudaMemsetAsync(total_dev, 0, sizeof(int32_t), ctx->stream));
    return PHFEM_OK;
  }
  if (n <= kScanSmall) {  // in == out is fine: every thread reads its entries before writing them
    PHFEM_LAUNCH_PDL(ctx, "scan", k_scan_small, 1, kScanThreads, 0, in, out, n, total_dev);
    return PHFEM_OK;
  }
  int32_t* sums = nullptr;
  PHFEM_TRY(dalloc(ctx, &sums, tiles));
  // note: the downsweep reads `in` after the tile pass, so in == out is fine
  // (each tile reads its own range before writing it).
  KTimer kt(ctx, "scan");
  k_scan_tile_sums<<<(unsigned)tiles, kScanThreads, 0, ctx->stream>>>(in, n, sums);
  PHFEM_CHECK_LAUNCH(ctx);
  k_scan_sums<<<1, kScanThreads, 0, ctx->stream>>>(sums, tiles, total_dev);
  PHFEM_CHECK_LAUNCH(ctx);
  k_scan_down<<<(unsigned)tiles, kScanThreads, 0, ctx->stream>>>(in, out, n, sums);
  PHFEM_CHECK_LAUNCH(ctx);
  dfree(ctx, sums);
  return PHFEM_OK;
}

}  // namespace phfem

using namespace phfem;

PHFEM_API int phfem_abi_version(void) { return PHFEM_ABI_VERSION; }

PHFEM_API phfem_status phfem_ctx_create(int device, void* stream, phfem_ctx** out) {
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    return PHFEM_ERR_NO_DEVICE;
  }
  if (device < 0 || device >= count) return PHFEM_ERR_INVALID_ARGUMENT;
  phfem_ctx* ctx = new phfem_ctx();
  ctx->device = device;
  if (cudaSetDevice(device) != cudaSuccess) {
    delete ctx;
    cudaGetLastError();
    return PHFEM_ERR_CUDA;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) == cudaSuccess) {
    ctx->num_sms = prop.multiProcessorCount;
    if (prop.major < 10) {
      delete ctx;
      return PHFEM_ERR_NO_DEVICE;  // sm_100a code only
    }
  }
  if (const char* gd = getenv("PHFEM_GUARD")) ctx->guard = gd[0] == '1';
  if (const char* gp = getenv("PHFEM_GUARD_POISON")) ctx->guard_poison = (int)strtol(gp, nullptr, 0) & 0xff;
  if (const char* bs = getenv("PHFEM_EG_MAX_BS")) {
    const int v = atoi(bs);
    if (v >= 1 && v <= 8) ctx->eg_max_bs = v;
  }
  if (stream) {
    ctx->stream = (cudaStream_t)stream;
  } else {
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete ctx;
      cudaGetLastError();
      return PHFEM_ERR_CUDA;
    }
    ctx->own_stream = true;
  }
  // A private stream-ordered pool: freed blocks stay cached across pipeline
  // runs (release threshold = max), and nothing else in the process (torch,
  // other libraries) can trim or reconfigure it.
  cudaMemPoolProps props = {};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = device;
  if (cudaMemPoolCreate(&ctx->pool, &props) != cudaSuccess) {
    delete ctx;
    cudaGetLastError();
    return PHFEM_ERR_CUDA;
  }
  uint64_t threshold = UINT64_MAX;
  cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolAttrReleaseThreshold, &threshold);
  if (cudaMalloc((void**)&ctx->derr, sizeof(phfem_dev_errors)) != cudaSuccess ||
      cudaMalloc((void**)&ctx->dderr, sizeof(phfem_dev_errors)) != cudaSuccess ||
      cudaMallocHost((void**)&ctx->herr, sizeof(phfem_dev_errors)) != cudaSuccess) {
    cudaGetLastError();
    delete ctx;
    return PHFEM_ERR_OOM;
  }
  if (ctx->guard) {
    if (cudaMalloc((void**)&ctx->guard_bad, sizeof(unsigned int)) != cudaSuccess ||
        cudaMemset(ctx->guard_bad, 0xff, sizeof(unsigned int)) != cudaSuccess) {
      cudaGetLastError();
      delete ctx;
      return PHFEM_ERR_OOM;
    }
  }
  *out = ctx;
  return PHFEM_OK;
}

PHFEM_API void phfem_ctx_destroy(phfem_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->guard) {
    std::vector<void*> live;
    for (auto& kv : ctx->guard_blocks) live.push_back(kv.first);
    for (void* q : live) guard_free(ctx, q);
    if (guard_check(ctx) != PHFEM_OK) fprintf(stderr, "%s\n", ctx->message.c_str());
    cudaFree(ctx->guard_bad);
  }
  cache_flush(ctx);
  for (auto& r : ctx->recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : ctx->free_events) cudaEventDestroy(e);
  cudaFree(ctx->derr);
  cudaFree(ctx->dderr);
  cudaFreeHost(ctx->herr);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  cudaStreamSynchronize(nullptr);
  if (ctx->pool) cudaMemPoolDestroy(ctx->pool);
  delete ctx;
}

PHFEM_API const char* phfem_ctx_message(const phfem_ctx* ctx) {
  return ctx ? ctx->message.c_str() : "";
}

PHFEM_API void* phfem_ctx_stream(const phfem_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

PHFEM_API int64_t phfem_ctx_launches(const phfem_ctx* ctx) { return ctx ? ctx->launches : 0; }

PHFEM_API phfem_status phfem_ctx_set_eg_max_bs(phfem_ctx* ctx, int max_bs) {
  if (!ctx || max_bs < 1 || max_bs > 8) return PHFEM_ERR_INVALID_ARGUMENT;
  ctx->eg_max_bs = max_bs;
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_ctx_sync(phfem_ctx* ctx) {
  PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (ctx->guard) return guard_check(ctx);
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_alloc(phfem_ctx* ctx, size_t bytes, void** out) {
  return dalloc(ctx, (char**)out, bytes);
}

PHFEM_API void phfem_free(phfem_ctx* ctx, void* ptr) {
  if (ptr && ctx) raw_free(ctx, ptr);
}

PHFEM_API phfem_status phfem_memcpy_h2d(phfem_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return PHFEM_OK;
  PHFEM_CUDA(ctx, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_memcpy_d2h(phfem_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return PHFEM_OK;
  PHFEM_CUDA(ctx, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_memcpy_d2d(phfem_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return PHFEM_OK;
  PHFEM_CUDA(ctx, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_ctx_profile(phfem_ctx* ctx, int enable) {
  if (!ctx) return PHFEM_ERR_INVALID_ARGUMENT;
  for (auto& r : ctx->recs) {
    ctx->free_events.push_back(r.a);
    ctx->free_events.push_back(r.b);
  }
  ctx->recs.clear();
  ctx->prof = enable != 0;
  return PHFEM_OK;
}

PHFEM_API int phfem_ctx_profile_read(phfem_ctx* ctx, int max_names, const char** names, double* ms,
                                     int64_t* counts) {
  if (!ctx) return -1;
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  int n = 0;
  if (getenv("PHFEM_PROF_TIMELINE") && !ctx->recs.empty()) {  // debug: per-launch start / gap
    float prev_end = 0.f;
    for (auto& r : ctx->recs) {
      float t0 = 0.f, t1 = 0.f;
      cudaEventElapsedTime(&t0, ctx->recs[0].a, r.a);
      cudaEventElapsedTime(&t1, ctx->recs[0].a, r.b);
      fprintf(stderr, "[timeline] %-22s start %9.3f  dur %8.3f  gap %7.3f ms\n", r.name, t0, t1 - t0, t0 - prev_end);
      prev_end = t1;
    }
  }
  for (auto& r : ctx->recs) {
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    int i = 0;
    while (i < n && strcmp(names[i], r.name) != 0) ++i;
    if (i == n) {
      if (n == max_names) continue;
      names[n] = r.name;
      ms[n] = 0.0;
      counts[n] = 0;
      ++n;
    }
    ms[i] += t;
    counts[i] += 1;
  }
  return n;
}
