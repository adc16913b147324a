// dist_run.cu — host orchestration of the sharded pipeline in C++ (SURVEY
// §8(e)): the same phases as paper_2401_15557_b200/dist.py (the Python
// orchestration, kept as the reference / CPU-testable form) without Python
// between the kernels.  One call runs edge generation -> [red refinement +
// refined topology] x levels -> classification, C, bD, blocks, load = b + LN
// for the ranks this process drives:
//   * phfem_dist_comm_local: W ranks emulated in one process on one device
//     (their kernels run one after another; no rank ever waits on another);
//   * phfem_dist_comm_nccl: this process is one rank of an NCCL communicator
//     (ncclUniqueId from rank 0), every bulk exchange a peer-window kernel
//     into CUDA-IPC-mapped buffers of the owners (NVLink), NCCL only for the
//     small collectives and the stream-ordered fences.
// Exchanges (dist.py / DESIGN §5): input level = histogram all-reduce ->
// tile-aligned key ranges -> bucket histograms all-gathered -> occurrences
// stored into the owners' bucket arrays -> owner dedup -> counts all-gathered
// -> reverse (slot, edge) entries stored into the element owners' elem_edge;
// each refinement = side records into the edge owners' side arrays -> level
// count -> fine counts all-gathered -> level run with global ids -> group
// starts into the element owners' slot arrays -> children pass.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "common.cuh"

extern "C" {
phfem_status phfem_dist_occurrences(phfem_ctx*, const int32_t*, int32_t, int32_t, const int32_t*, int32_t, int32_t*,
                                    int32_t*, int32_t*);
int phfem_dist_bucket_bits(int32_t, int32_t);
phfem_status phfem_dist_bucket_hist(phfem_ctx*, const int32_t*, int32_t, int32_t, int32_t, int32_t, int32_t*);
phfem_status phfem_dist_bucket_cursors(phfem_ctx*, const int32_t*, int32_t, int64_t, int32_t, const int32_t*,
                                       int32_t*, int32_t*, int64_t*);
phfem_status phfem_dist_scatter_p2p(phfem_ctx*, const int32_t*, int32_t, int32_t, int32_t, int32_t, int32_t*,
                                    const int32_t*, int32_t, int32_t, uint64_t* const*, int32_t*);
phfem_status phfem_dist_dedup_items(phfem_ctx*, uint64_t*, int64_t, const int32_t*, int32_t, int32_t, int32_t,
                                    int32_t, int32_t, int32_t, int32_t*, phfem_topology*, int32_t*, int64_t*);
phfem_status phfem_dist_add_offset(phfem_ctx*, int32_t*, int64_t, int32_t, int);
phfem_status phfem_dist_pairs_p2p(phfem_ctx*, const int32_t*, int64_t, int32_t, const int32_t*, int32_t, int32_t,
                                  int32_t* const*, int32_t*);
phfem_status phfem_dist_resolve(phfem_ctx*, const phfem_topology*, int32_t, int32_t, const int32_t*, int32_t,
                                int32_t, int32_t*, unsigned long long*);
phfem_status phfem_dist_side_p2p_ex(phfem_ctx*, const int32_t*, const int32_t*, int32_t, const int32_t*, int32_t,
                                    int32_t, int32_t* const*, int32_t*, int);
phfem_status phfem_dist_level_count_ex(phfem_ctx*, const phfem_topology*, int32_t, const int32_t*,
                                       const phfem_dist_local*, const int32_t*, int32_t, int, int32_t*, int32_t*,
                                       void**);
phfem_status phfem_dist_level_run_ex(phfem_ctx*, void*, const double*, int32_t, int32_t, int32_t, int32_t, int32_t,
                                     int32_t, int32_t, phfem_topology*, uint8_t*, double*, phfem_csr*, int32_t*,
                                     int32_t*);
phfem_status phfem_dist_classify_given(phfem_ctx*, const phfem_topology*, const int32_t*, int32_t, const int32_t*,
                                       int32_t, int32_t*, int32_t*, int32_t, phfem_classification*);
phfem_status phfem_dist_children_slots_ex(phfem_ctx*, const int32_t*, const int32_t*, int32_t, const int32_t*,
                                          const uint8_t*, int32_t, int32_t, int32_t, const int32_t*, int32_t,
                                          const uint8_t*, double*, int32_t*, int32_t*);
phfem_status phfem_dist_start_p2p_ex(phfem_ctx*, const phfem_topology*, const int32_t*, int32_t, const uint8_t*,
                                     const int32_t*, int32_t, int32_t, int32_t* const*, uint8_t* const*, int32_t*,
                                     int);
phfem_status phfem_dist_classify_ex(phfem_ctx*, const phfem_topology*, int32_t, const int32_t*, int32_t,
                                    const int32_t*, int32_t, int32_t, int32_t, phfem_classification*);
phfem_status phfem_dist_dirichlet(phfem_ctx*, const phfem_mesh*, const phfem_topology*,
                                  const phfem_classification*, const phfem_field*, double, int32_t, double*);
phfem_status phfem_dist_neumann_table(phfem_ctx*, const phfem_topology*, int32_t, const int32_t*, int32_t,
                                      int32_t*);
phfem_status phfem_dist_volume_start(phfem_ctx*, const phfem_mesh*, const phfem_coeffs*, const phfem_field*, double,
                                     double*, double*, double*, double*, double*);
phfem_status phfem_dist_volume_finish(phfem_ctx*);
phfem_status phfem_dist_neumann_apply(phfem_ctx*, const phfem_mesh*, const int32_t*, int32_t, int32_t, int32_t,
                                      int32_t, const phfem_field*, double, double*);
}

// ---------------------------------------------------------------------------
// NCCL resolved at run time (the process's libnccl.so.2 — torch's when torch
// is loaded): the library itself does not depend on NCCL
namespace {
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  bool ok = false;
};
const NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.get_unique_id = (decltype(a.get_unique_id))dlsym(h, "ncclGetUniqueId");
    a.init_rank = (decltype(a.init_rank))dlsym(h, "ncclCommInitRank");
    a.all_reduce = (decltype(a.all_reduce))dlsym(h, "ncclAllReduce");
    a.all_gather = (decltype(a.all_gather))dlsym(h, "ncclAllGather");
    a.destroy = (decltype(a.destroy))dlsym(h, "ncclCommDestroy");
    a.ok = a.get_unique_id && a.init_rank && a.all_reduce && a.all_gather && a.destroy;
    return a;
  }();
  return api;
}
}  // namespace

// ---------------------------------------------------------------------------
// communicator
struct phfem_dist_comm {
  int world = 1;
  bool local = true;
  int rank = 0;  // NCCL: this process's rank
  ncclComm_t nccl = nullptr;
  int device = 0;
  // peer windows: per key, per local rank a cudaMalloc'd buffer (IPC-able,
  // persistent, grown on demand) and a device array of the W peer pointers
  struct Win {
    std::vector<void*> buf;
    std::vector<size_t> cap;
    std::vector<void**> peers_dev;
    std::vector<void*> opened;  // NCCL: the other ranks' mapped buffers
    bool valid = false;
  };
  std::map<std::string, Win> win;
  int32_t* fence_dev = nullptr;
  void* pin = nullptr;  // pinned host staging of the resolved boundary ids
  size_t pin_cap = 0;
  cudaEvent_t ev = nullptr;
  // exchange statistics (phfem_dist_comm_stats): bytes each local rank
  // RECEIVED per phase — peer-window records the other ranks stored into it,
  // the other ranks' parts of all-gathers, 2 (W-1)/W of all-reduced buffers
  bool stats = false;
  std::string phase = "input";
  std::vector<std::string> phase_names;
  std::vector<std::vector<int64_t>> recv;
  std::string message;
};

namespace {

using Comm = phfem_dist_comm;

phfem_status comm_fail(Comm* c, phfem_ctx* ctx, const char* what, int code) {
  char buf[256];
  snprintf(buf, sizeof buf, "phfem dist: %s failed (%d)", what, code);
  c->message = buf;
  if (ctx) ctx->message = buf;
  return PHFEM_ERR_CUDA;
}

#define DC_NCCL(c, ctx, call)                                        \
  do {                                                               \
    ncclResult_t _r = (call);                                        \
    if (_r != ncclSuccess) return comm_fail(c, ctx, #call, (int)_r); \
  } while (0)
#define DC_CUDA(c, ctx, call)                                        \
  do {                                                               \
    cudaError_t _e = (call);                                         \
    if (_e != cudaSuccess) return comm_fail(c, ctx, #call, (int)_e); \
  } while (0)

// The ranks this process drives: NCCL one (ctx[0]), local all W (ctx[i] may
// all be the same context; every operation of rank i runs on ctx[i]->stream).
struct Ranks {
  Comm* c;
  std::vector<phfem_ctx*> ctx;
  int n() const { return (int)ctx.size(); }
  cudaStream_t st(int i) const { return ctx[i]->stream; }
  // local mode: all the ranks' queued work complete (the emulated collectives
  // move data between the ranks' streams through the host or plain copies)
  phfem_status sync_all() {
    for (int i = 0; i < n(); ++i)
      if (i == 0 || ctx[i]->stream != ctx[i - 1]->stream) DC_CUDA(c, ctx[i], cudaStreamSynchronize(st(i)));
    return PHFEM_OK;
  }
};

void stat_add(Comm* c, int rank, int64_t bytes) {
  if (!c->stats || bytes == 0) return;
  size_t k = 0;
  while (k < c->phase_names.size() && c->phase_names[k] != c->phase) ++k;
  if (k == c->phase_names.size()) {
    c->phase_names.push_back(c->phase);
    c->recv.emplace_back(c->world, 0);
  }
  c->recv[k][rank] += bytes;
}
// peer-window stores: remote[i][d] records of rec_bytes each went to rank d
phfem_status stat_windows(Ranks& R, const std::vector<int32_t*>& remote, int64_t rec_bytes) {
  Comm* c = R.c;
  if (!c->stats) return PHFEM_OK;
  std::vector<int32_t> h(c->world);
  for (int i = 0; i < R.n(); ++i) {
    DC_CUDA(c, R.ctx[i], cudaMemcpy(h.data(), remote[i], sizeof(int32_t) * c->world, cudaMemcpyDeviceToHost));
    for (int d = 0; d < c->world; ++d)
      if (c->local) stat_add(c, d, h[d] * rec_bytes);
      else if (d != c->rank) stat_add(c, d, h[d] * rec_bytes);  // (NCCL: what this rank sent)
  }
  return PHFEM_OK;
}
void stat_collective(Ranks& R, int64_t bytes_per_rank, bool reduce) {
  Comm* c = R.c;
  for (int i = 0; i < R.n(); ++i) {
    const int r = c->local ? i : c->rank;
    stat_add(c, r, reduce ? 2 * (c->world - 1) * bytes_per_rank / c->world : (c->world - 1) * bytes_per_rank);
  }
}

// all-gather of n int64 per rank to the host (every local rank sees all W*n)
phfem_status allgather_host(Ranks& R, const std::vector<std::vector<int64_t>>& in, std::vector<int64_t>& out) {
  Comm* c = R.c;
  const int n = (int)in[0].size();
  stat_collective(R, 8 * (int64_t)n, false);
  out.assign((size_t)c->world * n, 0);
  if (c->local || c->world == 1) {
    for (int r = 0; r < c->world; ++r)
      for (int k = 0; k < n; ++k) out[(size_t)r * n + k] = in[r][k];
    return PHFEM_OK;
  }
  phfem_ctx* x = R.ctx[0];
  int64_t* d = nullptr;
  PHFEM_TRY(phfem::dalloc(x, &d, (size_t)(c->world + 1) * n));
  DC_CUDA(c, x, cudaMemcpyAsync(d, in[0].data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, R.st(0)));
  DC_NCCL(c, x, nccl_api().all_gather(d, d + n, n, ncclInt64, c->nccl, R.st(0)));
  DC_CUDA(c, x, cudaMemcpyAsync(out.data(), d + n, sizeof(int64_t) * c->world * n, cudaMemcpyDeviceToHost, R.st(0)));
  DC_CUDA(c, x, cudaStreamSynchronize(R.st(0)));
  phfem::dfree(x, d);
  return PHFEM_OK;
}

// in-place all-reduce of per-local-rank device buffers (int32 sum / max, or
// uint64 min), the result on every local rank's buffer
enum RedOp { kSum, kMax, kMinU64 };
phfem_status allreduce_dev(Ranks& R, const std::vector<void*>& bufs, int64_t n, RedOp op) {
  Comm* c = R.c;
  stat_collective(R, (op == kMinU64 ? 8 : 4) * n, true);
  if (n == 0 || c->world == 1) return PHFEM_OK;
  if (!c->local) {
    if (op == kMinU64)
      DC_NCCL(c, R.ctx[0], nccl_api().all_reduce(bufs[0], bufs[0], n, ncclUint64, ncclMin, c->nccl, R.st(0)));
    else
      DC_NCCL(c, R.ctx[0], nccl_api().all_reduce(bufs[0], bufs[0], n, ncclInt32, op == kSum ? ncclSum : ncclMax,
                                                 c->nccl, R.st(0)));
    return PHFEM_OK;
  }
  const size_t es = op == kMinU64 ? 8 : 4;
  std::vector<char> acc(es * n), tmp(es * n);
  PHFEM_TRY(R.sync_all());
  for (int r = 0; r < c->world; ++r) {
    DC_CUDA(c, R.ctx[r], cudaMemcpy(r ? tmp.data() : acc.data(), bufs[r], es * n, cudaMemcpyDeviceToHost));
    if (r == 0) continue;
    for (int64_t i = 0; i < n; ++i) {
      if (op == kMinU64) {
        uint64_t& a = reinterpret_cast<uint64_t*>(acc.data())[i];
        a = std::min(a, reinterpret_cast<uint64_t*>(tmp.data())[i]);
      } else {
        int32_t& a = reinterpret_cast<int32_t*>(acc.data())[i];
        const int32_t b = reinterpret_cast<int32_t*>(tmp.data())[i];
        a = op == kSum ? a + b : std::max(a, b);
      }
    }
  }
  for (int r = 0; r < c->world; ++r) DC_CUDA(c, R.ctx[r], cudaMemcpy(bufs[r], acc.data(), es * n, cudaMemcpyHostToDevice));
  return PHFEM_OK;
}

// all-gather of `bytes` per rank into out[W * bytes] on every local rank (device)
phfem_status allgather_dev(Ranks& R, const std::vector<const void*>& in, size_t bytes, const std::vector<void*>& out) {
  Comm* c = R.c;
  stat_collective(R, (int64_t)bytes, false);
  if (c->local || c->world == 1) {
    PHFEM_TRY(R.sync_all());
    for (int d = 0; d < R.n(); ++d)
      for (int r = 0; r < c->world; ++r)
        DC_CUDA(c, R.ctx[d], cudaMemcpyAsync((char*)out[d] + r * bytes, in[c->local ? r : 0], bytes,
                                             cudaMemcpyDeviceToDevice, R.st(d)));
    return R.sync_all();
  }
  DC_NCCL(c, R.ctx[0], nccl_api().all_gather(in[0], out[0], bytes, ncclChar, c->nccl, R.st(0)));
  return PHFEM_OK;
}

// fence: every rank's preceding peer stores complete before the owners' next
// kernels (NCCL: a one-element all-reduce on the stream, no host sync)
phfem_status fence(Ranks& R) {
  Comm* c = R.c;
  if (c->local) return R.sync_all();
  if (c->world == 1) return PHFEM_OK;
  DC_NCCL(c, R.ctx[0], nccl_api().all_reduce(c->fence_dev, c->fence_dev, 1, ncclInt32, ncclSum, c->nccl, R.st(0)));
  return PHFEM_OK;
}

// peer window `key` with bytes[i] per local rank: buffers grown on demand;
// NCCL: IPC handles re-exchanged when any rank's buffer changed
phfem_status window(Ranks& R, const std::string& key, const std::vector<size_t>& bytes, std::vector<void*>& local_buf,
                    std::vector<void**>& peers) {
  Comm* c = R.c;
  Comm::Win& w = c->win[key];
  const int nl = R.n();
  if ((int)w.buf.size() != nl) {
    w.buf.assign(nl, nullptr);
    w.cap.assign(nl, 0);
    w.peers_dev.assign(nl, nullptr);
  }
  int changed = 0;
  for (int i = 0; i < nl; ++i) {
    const size_t need = std::max<size_t>(bytes[i], 256);
    if (w.cap[i] < need) {
      PHFEM_TRY(R.sync_all());
      if (w.buf[i]) cudaFree(w.buf[i]);
      DC_CUDA(c, R.ctx[i], cudaMalloc(&w.buf[i], need + need / 8));  // headroom against regrowth
      w.cap[i] = need + need / 8;
      changed = 1;
    }
    if (!w.peers_dev[i]) {
      DC_CUDA(c, R.ctx[i], cudaMalloc((void**)&w.peers_dev[i], sizeof(void*) * c->world));
      changed = 1;
    }
  }
  if (c->local || c->world == 1) {
    if (changed || !w.valid) {
      for (int i = 0; i < nl; ++i)
        DC_CUDA(c, R.ctx[i], cudaMemcpy(w.peers_dev[i], w.buf.data(), sizeof(void*) * c->world, cudaMemcpyHostToDevice));
      w.valid = true;
    }
  } else {
    // every rank must agree whether to re-exchange
    phfem_ctx* x = R.ctx[0];
    int32_t* flag = c->fence_dev + 1;
    int32_t h = changed || !w.valid ? 1 : 0;
    DC_CUDA(c, x, cudaMemcpyAsync(flag, &h, sizeof h, cudaMemcpyHostToDevice, R.st(0)));
    DC_NCCL(c, x, nccl_api().all_reduce(flag, flag, 1, ncclInt32, ncclMax, c->nccl, R.st(0)));
    DC_CUDA(c, x, cudaMemcpyAsync(&h, flag, sizeof h, cudaMemcpyDeviceToHost, R.st(0)));
    DC_CUDA(c, x, cudaStreamSynchronize(R.st(0)));
    if (h) {
      for (void* p : w.opened)
        if (p) cudaIpcCloseMemHandle(p);
      w.opened.assign(c->world, nullptr);
      cudaIpcMemHandle_t mine;
      DC_CUDA(c, x, cudaIpcGetMemHandle(&mine, w.buf[0]));
      char* dh = nullptr;
      DC_CUDA(c, x, cudaMalloc(&dh, sizeof(cudaIpcMemHandle_t) * (c->world + 1)));
      DC_CUDA(c, x, cudaMemcpyAsync(dh, &mine, sizeof mine, cudaMemcpyHostToDevice, R.st(0)));
      DC_NCCL(c, x, nccl_api().all_gather(dh, dh + sizeof mine, sizeof mine, ncclChar, c->nccl, R.st(0)));
      std::vector<cudaIpcMemHandle_t> all(c->world);
      DC_CUDA(c, x, cudaMemcpyAsync(all.data(), dh + sizeof mine, sizeof mine * c->world, cudaMemcpyDeviceToHost,
                                    R.st(0)));
      DC_CUDA(c, x, cudaStreamSynchronize(R.st(0)));
      cudaFree(dh);
      std::vector<void*> ptrs(c->world);
      for (int r = 0; r < c->world; ++r) {
        if (r == c->rank) {
          ptrs[r] = w.buf[0];
        } else {
          DC_CUDA(c, x, cudaIpcOpenMemHandle(&ptrs[r], all[r], cudaIpcMemLazyEnablePeerAccess));
          w.opened[r] = ptrs[r];
        }
      }
      DC_CUDA(c, x, cudaMemcpy(w.peers_dev[0], ptrs.data(), sizeof(void*) * c->world, cudaMemcpyHostToDevice));
      w.valid = true;
    }
  }
  local_buf = w.buf;
  peers = w.peers_dev;
  return PHFEM_OK;
}

// ---------------------------------------------------------------------------
// per-rank state
struct RS {
  int r = 0;
  double* coords = nullptr;  // replicated parent coordinates (after the last level: the rank's)
  bool own_coords = false;
  int32_t* elements = nullptr;
  bool own_elements = false;
  int elo = 0, ehi = 0;
  phfem_topology part;
  int E0 = 0, B0 = 0;
  int32_t* ee = nullptr;  // own elem_edge (global ids)
  bool own_ee = false;
  phfem_csr C;
  bool have_C = false;
  int R0 = -1;                     // known up front after a fused last level
  int32_t* rpos = nullptr;         // fused last level: retained_pos [E] / retained_edges [L] (global)
  int32_t* redges = nullptr;
  int32_t Lr = 0;
  int64_t mid_lo = 0, mid_hi = 0;  // the rank's owned midpoints in coords (last level)
  int32_t nc_parent = 0;
};

template <typename T>
phfem_status upload(phfem_ctx* ctx, const std::vector<T>& h, T** d) {
  PHFEM_TRY(phfem::dalloc(ctx, d, std::max<size_t>(h.size(), 1)));
  if (!h.empty())
    PHFEM_CUDA(ctx, cudaMemcpyAsync(*d, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, ctx->stream));
  return PHFEM_OK;
}

// dist.py balanced_splits: first cumulative count >= total * r / W
std::vector<int32_t> balanced_splits(const std::vector<int32_t>& hist, const std::vector<int32_t>& bins, int W) {
  std::vector<int64_t> cum(hist.size() + 1, 0);
  for (size_t i = 0; i < hist.size(); ++i) cum[i + 1] = cum[i] + hist[i];
  std::vector<int32_t> out{bins[0]};
  for (int r = 1; r < W; ++r) {
    const double target = (double)cum.back() * r / W;
    size_t k = 0;
    while (k < cum.size() && (double)cum[k] < target) ++k;
    out.push_back(std::max(out.back(), bins[std::min(k, bins.size() - 1)]));
  }
  out.push_back(bins.back());
  return out;
}

}  // namespace

using namespace phfem;

PHFEM_API phfem_status phfem_dist_comm_local(int32_t W, phfem_dist_comm** out) {
  if (!out || W < 1 || W > 64) return PHFEM_ERR_INVALID_ARGUMENT;
  Comm* c = new Comm();
  c->world = W;
  c->local = true;
  *out = c;
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_dist_nccl_unique_id(void* uid128) {
  if (!uid128) return PHFEM_ERR_INVALID_ARGUMENT;
  ncclUniqueId id;
  if (!nccl_api().ok || nccl_api().get_unique_id(&id) != ncclSuccess) return PHFEM_ERR_CUDA;
  memcpy(uid128, &id, sizeof id);
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_dist_comm_nccl(const void* uid128, int32_t rank, int32_t world, int32_t device,
                                            phfem_dist_comm** out) {
  if (!out || !uid128 || world < 1 || world > 64 || rank < 0 || rank >= world) return PHFEM_ERR_INVALID_ARGUMENT;
  if (!nccl_api().ok || cudaSetDevice(device) != cudaSuccess) return PHFEM_ERR_CUDA;
  Comm* c = new Comm();
  c->world = world;
  c->local = false;
  c->rank = rank;
  c->device = device;
  ncclUniqueId id;
  memcpy(&id, uid128, sizeof id);
  if (nccl_api().init_rank(&c->nccl, world, id, rank) != ncclSuccess ||
      cudaMalloc((void**)&c->fence_dev, 2 * sizeof(int32_t)) != cudaSuccess) {
    delete c;
    return PHFEM_ERR_CUDA;
  }
  cudaMemset(c->fence_dev, 0, 2 * sizeof(int32_t));
  *out = c;
  return PHFEM_OK;
}

PHFEM_API void phfem_dist_comm_destroy(phfem_dist_comm* c) {
  if (!c) return;
  cudaDeviceSynchronize();
  for (auto& kv : c->win) {
    for (void* p : kv.second.opened)
      if (p) cudaIpcCloseMemHandle(p);
    for (void* p : kv.second.buf)
      if (p) cudaFree(p);
    for (void** p : kv.second.peers_dev)
      if (p) cudaFree(p);
  }
  if (c->fence_dev) cudaFree(c->fence_dev);
  if (c->pin) cudaFreeHost(c->pin);
  if (c->ev) cudaEventDestroy(c->ev);
  if (c->nccl) nccl_api().destroy(c->nccl);
  delete c;
}

PHFEM_API const char* phfem_dist_comm_message(const phfem_dist_comm* c) { return c ? c->message.c_str() : ""; }

PHFEM_API phfem_status phfem_dist_comm_set_stats(phfem_dist_comm* c, int enable) {
  if (!c) return PHFEM_ERR_INVALID_ARGUMENT;
  c->stats = enable != 0;
  c->phase_names.clear();
  c->recv.clear();
  return PHFEM_OK;
}

PHFEM_API int phfem_dist_comm_stats(const phfem_dist_comm* c, int max_phases, const char** names, int64_t* bytes) {
  if (!c) return -1;
  const int n = std::min<int>(max_phases, (int)c->phase_names.size());
  for (int k = 0; k < n; ++k) {
    names[k] = c->phase_names[k].c_str();
    for (int r = 0; r < c->world; ++r) bytes[(int64_t)k * c->world + r] = c->recv[k][r];
  }
  return n;
}

PHFEM_API void phfem_dist_rank_out_release(phfem_ctx* ctx, phfem_dist_rank_out* o) {
  if (!ctx || !o) return;
  phfem_topology_release(ctx, &o->part);
  phfem_classification_release(ctx, &o->cls);
  phfem_csr_release(ctx, &o->C);
  dfree(ctx, o->bd);
  dfree(ctx, o->B);
  dfree(ctx, o->D);
  dfree(ctx, o->M);
  dfree(ctx, o->M0);
  dfree(ctx, o->load);
  dfree(ctx, o->elem_edge);
  dfree(ctx, o->elements);
  dfree(ctx, o->coords);
  dfree(ctx, o->dirichlet);
  dfree(ctx, o->neumann);
  memset(o, 0, sizeof(*o));
}

namespace {

// phfem_dist_pipeline's body (dist.py distributed_pipeline with the CUDA
// backend, P2P = True, sort_free = True)
phfem_status dist_pipeline(Ranks& R, const phfem_mesh* meshes, int32_t nC_all, int32_t nE_all, int32_t levels,
                           const phfem_coeffs* coeffs, const phfem_field* f, const phfem_field* g,
                           const phfem_field* uD, double t, int32_t hist_sample, int32_t flags,
                           phfem_dist_rank_out* outs, std::vector<RS>& S) {
  Comm* c = R.c;
  // PHFEM_DIST_TRACE=1: host-side phase times (ms since the call started)
  const bool trace = getenv("PHFEM_DIST_TRACE") != nullptr;
  const auto t_start = std::chrono::steady_clock::now();
  auto tr = [&](const char* what) {
    c->phase = std::string("after ") + what;
    if (trace)
      fprintf(stderr, "[dist-trace] %-28s %8.3f ms\n", what,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count());
  };
  c->phase = "start";
  // local mode: slots whose element and edge are this rank's move through no window
  const int local_mode = (flags & PHFEM_DIST_NO_LOCAL) ? 0 : 1;
  const int nl = R.n(), W = c->world;
  auto& ctx = R.ctx;
  int64_t nC = nC_all, nE = nE_all;
  std::vector<int32_t> esp(W + 1);
  for (int r = 0; r <= W; ++r) esp[r] = (int32_t)(nE * r / W);
  // boundary lists (replicated, host copies: O(sqrt N) pairs)
  std::vector<int32_t> hdir(2 * (size_t)meshes[0].nD), hneu(2 * (size_t)meshes[0].nN);
  if (!hdir.empty())
    PHFEM_CUDA(ctx[0], cudaMemcpy(hdir.data(), meshes[0].dirichlet, sizeof(int32_t) * hdir.size(),
                                  cudaMemcpyDeviceToHost));
  if (!hneu.empty())
    PHFEM_CUDA(ctx[0], cudaMemcpy(hneu.data(), meshes[0].neumann, sizeof(int32_t) * hneu.size(),
                                  cudaMemcpyDeviceToHost));
  for (int i = 0; i < nl; ++i) {
    RS& s = S[i];
    s.r = c->local ? i : c->rank;
    s.coords = meshes[i].coords;
    s.elements = meshes[i].elements;
    s.elo = esp[s.r];
    s.ehi = esp[s.r + 1];
    if (meshes[i].nE != s.ehi - s.elo || meshes[i].nC != nC_all)
      return set_error(ctx[i], PHFEM_ERR_INVALID_ARGUMENT,
                       "dist: rank %d holds %d elements, the even split gives %d", s.r, meshes[i].nE, s.ehi - s.elo);
  }
  auto own = [](const RS& s) { return s.ehi - s.elo; };

  // ---- input level: key ranges, occurrences into the owners' buckets, dedup
  std::vector<int32_t> splits(W + 1);
  {
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>({64 * (int64_t)W, 4096, nC}));
    std::vector<int32_t> bins(nb + 1);
    for (int i = 0; i <= nb; ++i) bins[i] = (int32_t)(nC * i / nb);
    // coarse histogram of max nodes (a 1/hist_sample sample of the own elements)
    std::vector<void*> hists(nl);
    for (int i = 0; i < nl; ++i) {
      RS& s = S[i];
      int32_t *binsd = nullptr, *h = nullptr, *smp = nullptr;
      PHFEM_TRY(upload(ctx[i], bins, &binsd));
      PHFEM_TRY(dalloc(ctx[i], &h, nb));
      const int n = own(s), ns = hist_sample > 1 ? (n + hist_sample - 1) / hist_sample : n;
      const int32_t* src = s.elements;
      if (hist_sample > 1 && ns) {
        PHFEM_TRY(dalloc(ctx[i], &smp, 3 * (int64_t)ns));
        PHFEM_CUDA(ctx[i], cudaMemcpy2DAsync(smp, 12, s.elements, 12 * (size_t)hist_sample, 12, ns,
                                             cudaMemcpyDeviceToDevice, R.st(i)));
        src = smp;
      }
      PHFEM_TRY(phfem_dist_occurrences(ctx[i], src, 0, ns, binsd, nb, h, nullptr, nullptr));
      dfree(ctx[i], smp);
      dfree(ctx[i], binsd);
      hists[i] = h;
    }
    PHFEM_TRY(allreduce_dev(R, hists, nb, kSum));
    std::vector<int32_t> hh(nb);
    PHFEM_CUDA(ctx[0], cudaMemcpyAsync(hh.data(), hists[0], sizeof(int32_t) * nb, cudaMemcpyDeviceToHost, R.st(0)));
    PHFEM_CUDA(ctx[0], cudaStreamSynchronize(R.st(0)));
    for (int i = 0; i < nl; ++i) {
      int32_t* h = (int32_t*)hists[i];
      dfree(ctx[i], h);
    }
    const std::vector<int32_t> sp = balanced_splits(hh, bins, W);
    splits[0] = 0;
    for (int r = 1; r < W; ++r) splits[r] = sp[r] / 256 * 256;  // 256-node tiles: one owner per bucket
    splits[W] = (int32_t)nC;
  }
  tr("hist+splits");
  const int bs = phfem_dist_bucket_bits((int32_t)nC, (int32_t)nE);
  const int64_t NB = (nC + (1 << bs) - 1) >> bs;
  std::vector<int32_t> bsp(W + 1);
  for (int r = 0; r < W; ++r) bsp[r] = splits[r] >> bs;
  bsp[W] = (int32_t)NB;
  std::vector<int32_t*> bspd(nl), espd(nl), cursor(nl), boff(nl), histb(nl), hall(nl), remote(nl);
  std::vector<int64_t> nitems(nl);
  for (int i = 0; i < nl; ++i) {
    PHFEM_TRY(upload(ctx[i], bsp, &bspd[i]));
    PHFEM_TRY(upload(ctx[i], esp, &espd[i]));
    PHFEM_TRY(dalloc(ctx[i], &histb[i], NB));
    PHFEM_TRY(dalloc(ctx[i], &hall[i], NB * W));
    PHFEM_TRY(dalloc(ctx[i], &remote[i], W));
    PHFEM_TRY(phfem_dist_bucket_hist(ctx[i], S[i].elements, own(S[i]), S[i].elo, (int32_t)nC, (int32_t)nE, histb[i]));
  }
  PHFEM_TRY(allgather_dev(R, std::vector<const void*>(histb.begin(), histb.end()), sizeof(int32_t) * NB,
                          std::vector<void*>(hall.begin(), hall.end())));
  for (int i = 0; i < nl; ++i) {
    const int r = S[i].r;
    PHFEM_TRY(dalloc(ctx[i], &cursor[i], NB));
    PHFEM_TRY(dalloc(ctx[i], &boff[i], (int64_t)bsp[r + 1] - bsp[r] + 1));
    PHFEM_TRY(phfem_dist_bucket_cursors(ctx[i], hall[i], W, NB, r, bspd[i], cursor[i], boff[i], &nitems[i]));
    dfree(ctx[i], histb[i]);
    dfree(ctx[i], hall[i]);
  }
  tr("bucket cursors");
  std::vector<void*> itbuf, eebuf;
  std::vector<void**> itpeers, eepeers;
  {
    std::vector<size_t> by(nl);
    for (int i = 0; i < nl; ++i) by[i] = 8 * (size_t)nitems[i];
    PHFEM_TRY(window(R, "items", by, itbuf, itpeers));
    for (int i = 0; i < nl; ++i) by[i] = 12 * (size_t)own(S[i]);
    PHFEM_TRY(window(R, "ee", by, eebuf, eepeers));
  }
  for (int i = 0; i < nl; ++i)
    PHFEM_TRY(phfem_dist_scatter_p2p(ctx[i], S[i].elements, own(S[i]), S[i].elo, (int32_t)nC, (int32_t)nE, cursor[i],
                                     bspd[i], W, S[i].r, (uint64_t* const*)itpeers[i], remote[i]));
  PHFEM_TRY(fence(R));
  PHFEM_TRY(stat_windows(R, remote, 8));
  tr("scatter");
  std::vector<int32_t*> pairs(nl);
  std::vector<int64_t> npairs(nl);
  std::vector<std::vector<int64_t>> eb(nl);
  for (int i = 0; i < nl; ++i) {
    RS& s = S[i];
    const int r = s.r;
    PHFEM_TRY(dalloc(ctx[i], &pairs[i], 4 * std::max<int64_t>(nitems[i], 1)));
    PHFEM_TRY(phfem_dist_dedup_items(ctx[i], (uint64_t*)itbuf[i], nitems[i], boff[i], splits[r], splits[r + 1],
                                     (int32_t)nC, (int32_t)nE, s.elo, s.ehi, (int32_t*)eebuf[i], &s.part, pairs[i],
                                     &npairs[i]));
    eb[i] = {s.part.E, s.part.n_boundary};
    dfree(ctx[i], cursor[i]);
    dfree(ctx[i], boff[i]);
  }
  tr("dedup");
  std::vector<int64_t> ebg;
  PHFEM_TRY(allgather_host(R, eb, ebg));
  int64_t Etot = 0, Btot = 0;
  std::vector<int32_t> E0s(W + 1, 0), B0s(W + 1, 0);
  for (int r = 0; r < W; ++r) {
    Etot += ebg[2 * r];
    Btot += ebg[2 * r + 1];
    E0s[r + 1] = E0s[r] + (int32_t)ebg[2 * r];
    B0s[r + 1] = B0s[r] + (int32_t)ebg[2 * r + 1];
  }
  for (int i = 0; i < nl; ++i) {
    RS& s = S[i];
    s.E0 = E0s[s.r];
    s.B0 = B0s[s.r];
    phfem_topology& p = s.part;
    if (s.E0) {  // dist.py rebase_part + rebase_own_ee
      if (p.n_interior) PHFEM_TRY(phfem_dist_add_offset(ctx[i], p.interior_edges, p.n_interior, s.E0, 0));
      if (p.n_boundary) PHFEM_TRY(phfem_dist_add_offset(ctx[i], p.boundary_edges, p.n_boundary, s.E0, 0));
      PHFEM_TRY(phfem_dist_add_offset(ctx[i], p.node_edge_start, (int64_t)p.nC + 1, s.E0, 0));
      if (own(s)) PHFEM_TRY(phfem_dist_add_offset(ctx[i], (int32_t*)eebuf[i], 3 * (int64_t)own(s), s.E0, 2));
    }
  }
  PHFEM_TRY(fence(R));  // own entries global before the peers store theirs
  for (int i = 0; i < nl; ++i)
    PHFEM_TRY(phfem_dist_pairs_p2p(ctx[i], pairs[i], npairs[i], S[i].E0, espd[i], W, S[i].r,
                                   (int32_t* const*)eepeers[i], remote[i]));
  PHFEM_TRY(fence(R));
  PHFEM_TRY(stat_windows(R, remote, 4));
  for (int i = 0; i < nl; ++i) {
    dfree(ctx[i], pairs[i]);
    S[i].ee = (int32_t*)eebuf[i];  // the window (persistent; copied out when it is an output)
    S[i].own_ee = false;
  }

  tr("pairs");
  // ---- boundary pairs -> global ids on every rank + the reference's first error
  // resolve in two halves: _enqueue (kernels, all-reduces, the copy of the
  // ids into pinned host memory, an event) and _wait (the event, the
  // reference's first error) — the last level enqueues the element pass in
  // between, so the host waits for the ids while the GPU keeps working
  struct Resolve {
    std::vector<void*> idd, errd;
    std::vector<int32_t*> prd;
    int n = 0;
  } rv;
  auto resolve_enqueue = [&]() -> phfem_status {
    const int nD = (int)hdir.size() / 2, nN = (int)hneu.size() / 2, n = nD + nN;
    rv.n = n;
    rv.idd.assign(nl, nullptr);
    rv.errd.assign(nl, nullptr);
    rv.prd.assign(nl, nullptr);
    if (n == 0) return PHFEM_OK;
    std::vector<int32_t> pr(hdir);
    pr.insert(pr.end(), hneu.begin(), hneu.end());
    for (int i = 0; i < nl; ++i) {
      PHFEM_TRY(upload(ctx[i], pr, &rv.prd[i]));
      int32_t* d = nullptr;
      unsigned long long* e = nullptr;
      PHFEM_TRY(dalloc(ctx[i], &d, n));
      PHFEM_TRY(dalloc(ctx[i], &e, 1));
      PHFEM_CUDA(ctx[i], cudaMemsetAsync(d, 0xff, sizeof(int32_t) * n, R.st(i)));
      PHFEM_CUDA(ctx[i], cudaMemsetAsync(e, 0xff, sizeof(unsigned long long), R.st(i)));
      PHFEM_TRY(phfem_dist_resolve(ctx[i], &S[i].part, splits[S[i].r], S[i].E0, rv.prd[i], n, 0, d, e));
      rv.idd[i] = d;
      rv.errd[i] = e;
    }
    PHFEM_TRY(allreduce_dev(R, rv.idd, n, kMax));
    PHFEM_TRY(allreduce_dev(R, rv.errd, 1, kMinU64));
    const size_t need = sizeof(int32_t) * n + 16;
    if (c->pin_cap < need) {
      PHFEM_TRY(R.sync_all());
      if (c->pin) cudaFreeHost(c->pin);
      c->pin = nullptr;
      c->pin_cap = 0;
      PHFEM_CUDA(ctx[0], cudaMallocHost(&c->pin, need + need / 2));
      c->pin_cap = need + need / 2;
    }
    if (!c->ev) PHFEM_CUDA(ctx[0], cudaEventCreateWithFlags(&c->ev, cudaEventDisableTiming));
    PHFEM_CUDA(ctx[0], cudaMemcpyAsync(c->pin, rv.errd[0], 8, cudaMemcpyDeviceToHost, R.st(0)));
    PHFEM_CUDA(ctx[0], cudaMemcpyAsync((char*)c->pin + 16, rv.idd[0], sizeof(int32_t) * n, cudaMemcpyDeviceToHost,
                                       R.st(0)));
    PHFEM_CUDA(ctx[0], cudaEventRecord(c->ev, R.st(0)));
    for (int i = 0; i < nl; ++i) {
      int32_t* d = (int32_t*)rv.idd[i];
      unsigned long long* e = (unsigned long long*)rv.errd[i];
      dfree(ctx[i], d);  // stream-ordered: after the copy
      dfree(ctx[i], e);
      dfree(ctx[i], rv.prd[i]);
    }
    return PHFEM_OK;
  };
  auto resolve_wait = [&](std::vector<int32_t>& ids) -> phfem_status {
    const int nD = (int)hdir.size() / 2, n = rv.n;
    ids.assign(n, -1);
    if (n == 0) return PHFEM_OK;
    PHFEM_CUDA(ctx[0], cudaEventSynchronize(c->ev));
    unsigned long long key = 0;
    memcpy(&key, c->pin, 8);
    memcpy(ids.data(), (char*)c->pin + 16, sizeof(int32_t) * n);
    if (key != ~0ull) {
      const int64_t pos = (int64_t)(key >> 2);
      const bool interior = key & 1;
      const bool is_d = pos < nD;
      const int32_t* pp = is_d ? &hdir[2 * pos] : &hneu[2 * (pos - nD)];
      return set_error(ctx[0], interior ? PHFEM_ERR_INTERIOR_BOUNDARY : PHFEM_ERR_NOT_AN_EDGE, "%s pair (%d,%d) %s",
                       is_d ? "dirichlet" : "neumann", pp[0] + 1, pp[1] + 1,
                       interior ? "resolves to an interior edge" : "is not an edge");
    }
    return PHFEM_OK;
  };
  auto resolve = [&](std::vector<int32_t>& ids) -> phfem_status {
    PHFEM_TRY(resolve_enqueue());
    return resolve_wait(ids);
  };

  // ---- refinements: sort-free, halo form through peer windows
  for (int lvl = 0; lvl < levels; ++lvl) {
    const bool last = lvl == levels - 1;
    std::vector<int32_t> ids;
    PHFEM_TRY(resolve(ids));
    const int nD = (int)hdir.size() / 2, nN = (int)hneu.size() / 2;
    // 1. side records into the edge owners' side arrays
    std::vector<void*> sdbuf;
    std::vector<void**> sdpeers;
    std::vector<int32_t*> edgesp(nl);
    const bool no_remote = local_mode && W == 1;  // one rank in local mode: no record to move
    {
      std::vector<size_t> by(nl);
      for (int i = 0; i < nl; ++i) by[i] = no_remote ? 0 : 32 * (size_t)S[i].part.E;
      PHFEM_TRY(window(R, "side", by, sdbuf, sdpeers));
    }
    for (int i = 0; i < nl; ++i) {
      PHFEM_TRY(upload(ctx[i], E0s, &edgesp[i]));
      if (!no_remote)
        PHFEM_TRY(phfem_dist_side_p2p_ex(ctx[i], S[i].elements, S[i].ee, own(S[i]), edgesp[i], W, S[i].r,
                                         (int32_t* const*)sdpeers[i], remote[i], local_mode));
    }
    PHFEM_TRY(fence(R));
    if (!no_remote) PHFEM_TRY(stat_windows(R, remote, 16));
  tr("side");
    // 2. level count -> fine offsets (all-gathered) -> level run with global ids
    std::vector<int64_t> fsp(W + 1);
    fsp[0] = 0;
    for (int r = 1; r < W; ++r) fsp[r] = nC + E0s[r];
    fsp[W] = nC + Etot;
    std::vector<double*> cfine(nl);
    std::vector<void*> plans(nl);
    std::vector<std::vector<int64_t>> cnt(nl);
    const std::vector<int32_t> neu_ids(ids.begin() + nD, ids.end());
    for (int i = 0; i < nl; ++i) {
      RS& s = S[i];
      int32_t* neud = nullptr;
      PHFEM_TRY(dalloc(ctx[i], &cfine[i], 2 * (nC + Etot)));
      PHFEM_CUDA(ctx[i], cudaMemcpyAsync(cfine[i], s.coords, sizeof(double) * 2 * nC, cudaMemcpyDeviceToDevice, R.st(i)));
      if (last && nN) PHFEM_TRY(upload(ctx[i], neu_ids, &neud));
      int32_t Ef = 0, nneu = 0;
      phfem_dist_local loc{s.elements, s.ee, s.elo, s.ehi, W == 1 ? 1 : 0, 0};
      PHFEM_TRY(phfem_dist_level_count_ex(ctx[i], &s.part, s.E0, (const int32_t*)sdbuf[i], local_mode ? &loc : nullptr,
                                          last ? neud : nullptr, last ? nN : 0, last ? 1 : 0, &Ef, &nneu, &plans[i]));
      dfree(ctx[i], neud);
      cnt[i] = {Ef, 2 * (int64_t)s.part.n_boundary, nneu};
    }
  tr("level count");
    std::vector<int64_t> cg;
    PHFEM_TRY(allgather_host(R, cnt, cg));
    std::vector<int32_t> fE0s(W + 1, 0), fB0s(W + 1, 0);
    std::vector<int64_t> fN0s(W + 1, 0);
    for (int r = 0; r < W; ++r) {
      fE0s[r + 1] = fE0s[r] + (int32_t)cg[3 * r];
      fB0s[r + 1] = fB0s[r] + (int32_t)cg[3 * r + 1];
      fN0s[r + 1] = fN0s[r] + 2 * cg[3 * r + 2];  // fine Neumann edges before the rank
    }
    std::vector<phfem_topology> fpart(nl);
    std::vector<uint8_t*> rk(nl);
    for (int i = 0; i < nl; ++i) {
      RS& s = S[i];
      const int r = s.r;
      const int32_t E0f = fE0s[r], B0f = fB0s[r];
      const int64_t N0f = fN0s[r], R0 = E0f - N0f;
      const int32_t nnz0 = last ? (int32_t)(4 * R0 - 2 * ((int64_t)B0f - N0f)) : 0;
      PHFEM_TRY(dalloc(ctx[i], &rk[i], std::max(s.part.E, 1)));
      memset(&fpart[i], 0, sizeof(phfem_topology));
      phfem_csr Cl;
      memset(&Cl, 0, sizeof Cl);
      if (last) {  // the classification's retained arrays too (global rows / ids)
        s.Lr = (int32_t)(cg[3 * r] - 2 * cg[3 * r + 2]);
        PHFEM_TRY(dalloc(ctx[i], &s.rpos, std::max<int64_t>(cg[3 * r], 1)));
        PHFEM_TRY(dalloc(ctx[i], &s.redges, std::max(s.Lr, 1)));
      }
      PHFEM_TRY(phfem_dist_level_run_ex(ctx[i], plans[i], s.coords, (int32_t)nC, (int32_t)fsp[r], (int32_t)fsp[r + 1],
                                        (int32_t)nE, E0f, nnz0, last ? (int32_t)R0 : 0, &fpart[i], rk[i], cfine[i],
                                        last ? &Cl : nullptr, s.rpos, s.redges));
      plans[i] = nullptr;
      if (last) {
        s.C = Cl;
        s.have_C = true;
        s.R0 = (int32_t)R0;
      }
    }
  tr("level run");
    // 3. group starts into the element owners' slot arrays
    std::vector<void*> gsbuf, grbuf;
    std::vector<void**> gspeers, grpeers;
    {
      std::vector<size_t> b4(nl), b1(nl);
      for (int i = 0; i < nl; ++i) {
        b4[i] = no_remote ? 0 : 12 * (size_t)own(S[i]);
        b1[i] = no_remote ? 0 : 3 * (size_t)own(S[i]);
      }
      PHFEM_TRY(window(R, "gs", b4, gsbuf, gspeers));
      PHFEM_TRY(window(R, "grk", b1, grbuf, grpeers));
    }
    for (int i = 0; i < nl && !no_remote; ++i) {
      RS& s = S[i];
      PHFEM_TRY(phfem_dist_start_p2p_ex(ctx[i], &s.part, fpart[i].node_edge_start, (int32_t)(nC + s.E0 - fsp[s.r]),
                                        rk[i], espd[i], W, s.r, (int32_t* const*)gspeers[i],
                                        (uint8_t* const*)grpeers[i], remote[i], local_mode));
    }
    PHFEM_TRY(fence(R));
    if (!no_remote) PHFEM_TRY(stat_windows(R, remote, 5));
  tr("start");
    // 4. children, fine elem_edge, midpoints of the own elements' edges
    for (int i = 0; i < nl; ++i) {
      RS& s = S[i];
      const int n = own(s);
      int32_t *kids = nullptr, *fee = nullptr;
      PHFEM_TRY(dalloc(ctx[i], &kids, 12 * (int64_t)std::max(n, 1)));
      PHFEM_TRY(dalloc(ctx[i], &fee, 12 * (int64_t)std::max(n, 1)));
      // midpoints of the edges this rank owns: written by its level kernel
      PHFEM_TRY(phfem_dist_children_slots_ex(ctx[i], s.elements, s.ee, n, (const int32_t*)gsbuf[i],
                                             (const uint8_t*)grbuf[i], (int32_t)nC, E0s[s.r], E0s[s.r + 1],
                                             local_mode ? fpart[i].node_edge_start : nullptr,
                                             (int32_t)(nC + s.E0 - fsp[s.r]), rk[i], cfine[i], kids, fee));
      phfem_topology_release(ctx[i], &s.part);
      s.part = fpart[i];
      dfree(ctx[i], rk[i]);
      dfree(ctx[i], edgesp[i]);
      if (s.own_elements) dfree(ctx[i], s.elements);
      if (s.own_ee) dfree(ctx[i], s.ee);
      s.elements = kids;
      s.own_elements = true;
      s.ee = fee;
      s.own_ee = true;
      s.elo *= 4;
      s.ehi *= 4;
    }
  tr("children");
    // boundary lists bisected (refine.cpp:39-50)
    {
      std::vector<int32_t> nd, nn;
      nd.reserve(2 * hdir.size());
      nn.reserve(2 * hneu.size());
      for (int k = 0; k < nD; ++k) {
        const int32_t m = (int32_t)(nC + ids[k]);
        nd.insert(nd.end(), {hdir[2 * k], m, m, hdir[2 * k + 1]});
      }
      for (int k = 0; k < nN; ++k) {
        const int32_t m = (int32_t)(nC + ids[nD + k]);
        nn.insert(nn.end(), {hneu[2 * k], m, m, hneu[2 * k + 1]});
      }
      hdir.swap(nd);
      hneu.swap(nn);
    }
    // coordinates: replicated again (owned midpoints all-gathered) unless last
    if (last) {
      for (int i = 0; i < nl; ++i) {
        RS& s = S[i];
        if (s.own_coords) dfree(ctx[i], s.coords);
        s.coords = cfine[i];
        s.own_coords = true;
        s.nc_parent = (int32_t)nC;
        s.mid_lo = nC + E0s[s.r];
        s.mid_hi = nC + E0s[s.r + 1];
      }
    } else {
      int64_t mx = 1;
      for (int r = 0; r < W; ++r) mx = std::max<int64_t>(mx, (int64_t)E0s[r + 1] - E0s[r]);
      std::vector<double*> pad(nl), gat(nl);
      for (int i = 0; i < nl; ++i) {
        RS& s = S[i];
        PHFEM_TRY(dalloc(ctx[i], &pad[i], 2 * mx));
        PHFEM_TRY(dalloc(ctx[i], &gat[i], 2 * mx * W));
        PHFEM_CUDA(ctx[i], cudaMemcpyAsync(pad[i], cfine[i] + 2 * (nC + E0s[s.r]),
                                           sizeof(double) * 2 * ((int64_t)E0s[s.r + 1] - E0s[s.r]),
                                           cudaMemcpyDeviceToDevice, R.st(i)));
      }
      PHFEM_TRY(allgather_dev(R, std::vector<const void*>(pad.begin(), pad.end()), sizeof(double) * 2 * mx,
                              std::vector<void*>(gat.begin(), gat.end())));
      for (int i = 0; i < nl; ++i) {
        RS& s = S[i];
        for (int r = 0; r < W; ++r)
          PHFEM_CUDA(ctx[i], cudaMemcpyAsync(cfine[i] + 2 * (nC + E0s[r]), gat[i] + 2 * mx * r,
                                             sizeof(double) * 2 * ((int64_t)E0s[r + 1] - E0s[r]),
                                             cudaMemcpyDeviceToDevice, R.st(i)));
        dfree(ctx[i], pad[i]);
        dfree(ctx[i], gat[i]);
        if (s.own_coords) dfree(ctx[i], s.coords);
        s.coords = cfine[i];
        s.own_coords = true;
      }
    }
    for (int r = 0; r <= W; ++r) splits[r] = (int32_t)fsp[r];
    nC += Etot;
    nE *= 4;
    for (int r = 0; r <= W; ++r) esp[r] *= 4;
    for (int i = 0; i < nl; ++i) {
      RS& s = S[i];
      s.E0 = fE0s[s.r];
      s.B0 = fB0s[s.r];
      dfree(ctx[i], espd[i]);
      PHFEM_TRY(upload(ctx[i], esp, &espd[i]));
    }
    E0s = fE0s;
    Etot = fE0s[W];
    Btot = fB0s[W];
  }

  tr("levels done");
  // ---- last level: classification, C, bD, blocks, load = b + LN
  PHFEM_TRY(resolve_enqueue());
  const int nD = (int)hdir.size() / 2, nN = (int)hneu.size() / 2;
  // the blocks + load next: the host waits for the ids and enqueues the
  // classification / bD / Neumann tables while the element pass runs
  std::vector<phfem_mesh> mv(nl);
  for (int i = 0; i < nl; ++i) {
    RS& s = S[i];
    phfem_dist_rank_out& o = outs[i];
    memset(&mv[i], 0, sizeof(phfem_mesh));
    mv[i].coords = s.coords;
    mv[i].elements = s.elements;
    mv[i].nC = (int32_t)nC;
    mv[i].nE = own(s);
    const int64_t n = std::max<int64_t>(own(s), 1);
    PHFEM_TRY(dalloc(ctx[i], &o.B, 9 * n));
    PHFEM_TRY(dalloc(ctx[i], &o.D, 9 * n));
    PHFEM_TRY(dalloc(ctx[i], &o.M, 9 * n));
    PHFEM_TRY(dalloc(ctx[i], &o.M0, 9 * n));
    PHFEM_TRY(dalloc(ctx[i], &o.load, 3 * n));
    if (own(s)) PHFEM_TRY(phfem_dist_volume_start(ctx[i], &mv[i], coeffs, f, t, o.B, o.D, o.M, o.M0, o.load));
    if (c->local && nl > 1 && own(s))  // emulated ranks share contexts: one error block each time
      PHFEM_TRY(phfem_dist_volume_finish(ctx[i]));
  }
  tr("volume enqueued");
  std::vector<int32_t> ids;
  PHFEM_TRY(resolve_wait(ids));
  // the rank's id lists and Neumann table positions
  std::vector<std::vector<int32_t>> dl(nl), neu_loc(nl);
  std::vector<int32_t*> dld(nl), nld(nl), fulld(nl);
  for (int i = 0; i < nl; ++i) {
    RS& s = S[i];
    const int Er = s.part.E;
    std::vector<int32_t> full(std::max(nN, 1), -1);
    for (int k = 0; k < nD; ++k)
      if (ids[k] >= 0 && ids[k] - s.E0 >= 0 && ids[k] - s.E0 < Er) dl[i].push_back(ids[k] - s.E0);
    for (int k = 0; k < nN; ++k) {
      const int v = ids[nD + k];
      if (v >= 0 && v - s.E0 >= 0 && v - s.E0 < Er) {
        neu_loc[i].push_back(v - s.E0);
        full[k] = v - s.E0;
      }
    }
    PHFEM_TRY(upload(ctx[i], dl[i], &dld[i]));
    PHFEM_TRY(upload(ctx[i], neu_loc[i], &nld[i]));
    PHFEM_TRY(upload(ctx[i], full, &fulld[i]));
  }
  tr("lists");
  bool dup = false;  // a Neumann pair listed twice (global list; phfem_dist_neumann_apply's order)
  {
    std::vector<int32_t> nv(ids.begin() + nD, ids.end());
    std::sort(nv.begin(), nv.end());
    dup = std::adjacent_find(nv.begin(), nv.end()) != nv.end();
  }
  std::vector<std::vector<int64_t>> Lv(nl);
  std::vector<phfem_classification> cls(nl);
  for (int i = 0; i < nl; ++i) {
    RS& s = S[i];
    memset(&cls[i], 0, sizeof(phfem_classification));
    if (s.rpos) {  // retained arrays from the fused level kernel
      PHFEM_TRY(phfem_dist_classify_given(ctx[i], &s.part, dld[i], (int32_t)dl[i].size(), nld[i],
                                          (int32_t)neu_loc[i].size(), s.rpos, s.redges, s.Lr, &cls[i]));
      s.rpos = s.redges = nullptr;  // owned by the classification now
      cls[i].flags = dup ? PHFEM_CLS_DUP_NEUMANN : 0;
    } else {
      PHFEM_TRY(phfem_dist_classify_ex(ctx[i], &s.part, s.E0, dld[i], (int32_t)dl[i].size(), nld[i],
                                       (int32_t)neu_loc[i].size(), 0, 0, &cls[i]));
    }
    outs[i].cls = cls[i];  // owned by the output from here (released with it on error)
    dfree(ctx[i], dld[i]);
    dfree(ctx[i], nld[i]);
    Lv[i] = {cls[i].L};
  }
  tr("classified");
  std::vector<int64_t> Lg;
  PHFEM_TRY(allgather_host(R, Lv, Lg));
  int64_t Ltot = 0;
  for (int r = 0; r < W; ++r) Ltot += Lg[r];
  std::vector<void*> tables(nl);
  for (int i = 0; i < nl; ++i) {
    RS& s = S[i];
    phfem_dist_rank_out& o = outs[i];
    int64_t R0 = 0;
    for (int r = 0; r < s.r; ++r) R0 += Lg[r];
    const int64_t N0 = s.E0 - R0;                        // Neumann edges before the rank
    const int64_t nnz0 = 4 * R0 - 2 * ((int64_t)s.B0 - N0);  // retained boundary rows hold 2 entries
    if (s.R0 >= 0 && s.R0 != R0)
      return set_error(ctx[i], PHFEM_ERR_MISMATCH, "dist: level offsets disagree with the classification");
    if (!s.have_C) {  // no refinement: C from the sort-built part (columns 3 m, m global)
      phfem_mesh mc = mv[i];
      mc.nE = (int32_t)nE;
      PHFEM_TRY(phfem_assemble_constraint(ctx[i], &mc, &s.part, &cls[i], &s.C));
      s.have_C = true;
    }
    PHFEM_TRY(dalloc(ctx[i], &o.bd, std::max(cls[i].L, 1)));
    PHFEM_TRY(phfem_dist_dirichlet(ctx[i], &mv[i], &s.part, &cls[i], uD, t, s.R0 >= 0 ? s.R0 : 0, o.bd));
    if (s.R0 < 0) {  // rank-local positions, edges, row pointers -> global
      if (cls[i].E && R0) PHFEM_TRY(phfem_dist_add_offset(ctx[i], cls[i].retained_pos, cls[i].E, (int32_t)R0, 1));
      if (cls[i].L && s.E0) PHFEM_TRY(phfem_dist_add_offset(ctx[i], cls[i].retained_edges, cls[i].L, s.E0, 0));
      if (nnz0) PHFEM_TRY(phfem_dist_add_offset(ctx[i], s.C.row_ptr, (int64_t)s.C.rows + 1, (int32_t)nnz0, 0));
    }
    // Neumann: the owners publish {a, b, t_plus, led}; element owners add b + LN
    int32_t* tb = nullptr;
    PHFEM_TRY(dalloc(ctx[i], &tb, 4 * (int64_t)std::max(nN, 1)));
    PHFEM_CUDA(ctx[i], cudaMemsetAsync(tb, 0, sizeof(int32_t) * 4 * std::max(nN, 1), R.st(i)));
    if (nN) PHFEM_TRY(phfem_dist_neumann_table(ctx[i], &s.part, 0, fulld[i], nN, tb));
    dfree(ctx[i], fulld[i]);
    tables[i] = tb;
  }
  tr("bd+tables");
  if (nN) PHFEM_TRY(allreduce_dev(R, tables, 4 * (int64_t)nN, kSum));
  if (!(c->local && nl > 1))  // the element pass's errors (degenerate element, non-finite load)
    for (int i = 0; i < nl; ++i)
      if (own(S[i])) PHFEM_TRY(phfem_dist_volume_finish(ctx[i]));
  for (int i = 0; i < nl; ++i) {
    RS& s = S[i];
    phfem_dist_rank_out& o = outs[i];
    if (nN && own(s))
      PHFEM_TRY(phfem_dist_neumann_apply(ctx[i], &mv[i], (const int32_t*)tables[i], nN, dup ? 1 : 0, s.elo, s.ehi, g,
                                         t, o.load));
    int32_t* tb = (int32_t*)tables[i];
    dfree(ctx[i], tb);
    // outputs (ownership moves to the rank's phfem_dist_rank_out)
    o.part = s.part;
    memset(&s.part, 0, sizeof s.part);
    o.C = s.C;
    memset(&s.C, 0, sizeof s.C);
    if (s.own_ee) {
      o.elem_edge = s.ee;
    } else {
      PHFEM_TRY(dalloc(ctx[i], &o.elem_edge, 3 * (int64_t)std::max(own(s), 1)));
      PHFEM_CUDA(ctx[i], cudaMemcpyAsync(o.elem_edge, s.ee, 12 * (size_t)own(s), cudaMemcpyDeviceToDevice, R.st(i)));
    }
    s.ee = nullptr;
    s.own_ee = false;
    if (s.own_elements) {
      o.elements = s.elements;
    } else {  // no refinement: a copy (the input stays the caller's)
      PHFEM_TRY(dalloc(ctx[i], &o.elements, 3 * (int64_t)std::max(own(s), 1)));
      PHFEM_CUDA(ctx[i], cudaMemcpyAsync(o.elements, s.elements, 12 * (size_t)own(s), cudaMemcpyDeviceToDevice,
                                         R.st(i)));
    }
    s.elements = nullptr;
    s.own_elements = false;
    if (s.own_coords) {
      o.coords = s.coords;
    } else {
      PHFEM_TRY(dalloc(ctx[i], &o.coords, 2 * nC));
      PHFEM_CUDA(ctx[i], cudaMemcpyAsync(o.coords, s.coords, sizeof(double) * 2 * nC, cudaMemcpyDeviceToDevice,
                                         R.st(i)));
    }
    s.coords = nullptr;
    s.own_coords = false;
    o.coords_all = levels == 0 ? 1 : 0;
    o.nc_parent = levels == 0 ? (int32_t)nC : s.nc_parent;
    o.mid_lo = s.mid_lo;
    o.mid_hi = s.mid_hi;
    o.elo = s.elo;
    o.ehi = s.ehi;
    o.E0 = s.E0;
    o.E = (int32_t)Etot;
    o.n_boundary = (int32_t)Btot;
    o.L = (int32_t)Ltot;
    o.nC = (int32_t)nC;
    o.nE = (int32_t)nE;
    o.nD = nD;
    o.nN = nN;
    PHFEM_TRY(upload(ctx[i], hdir, &o.dirichlet));
    PHFEM_TRY(upload(ctx[i], hneu, &o.neumann));
    dfree(ctx[i], bspd[i]);
    dfree(ctx[i], espd[i]);
    dfree(ctx[i], remote[i]);
  }
  for (int i = 0; i < nl; ++i) {
    int64_t R0 = 0;
    for (int r = 0; r < S[i].r; ++r) R0 += Lg[r];
    outs[i].R0 = (int32_t)R0;
  }
  tr("outputs");
  const phfem_status st = R.sync_all();
  tr("synchronised");
  return st;
}

}  // namespace

PHFEM_API phfem_status phfem_dist_pipeline(phfem_dist_comm* c, phfem_ctx** ctxs, const phfem_mesh* meshes,
                                           int32_t nC_all, int32_t nE_all, int32_t levels,
                                           const phfem_coeffs* coeffs, const phfem_field* f, const phfem_field* g,
                                           const phfem_field* uD, double t, int32_t hist_sample, int32_t flags,
                                           phfem_dist_rank_out* outs) {
  if (!c || !ctxs || !meshes || !coeffs || !f || !g || !uD || !outs || levels < 0 || levels > 8)
    return PHFEM_ERR_INVALID_ARGUMENT;
  Ranks R;
  R.c = c;
  R.ctx.assign(ctxs, ctxs + (c->local ? c->world : 1));
  for (phfem_ctx* x : R.ctx)
    if (!x) return PHFEM_ERR_INVALID_ARGUMENT;
  for (int i = 0; i < R.n(); ++i) memset(&outs[i], 0, sizeof(outs[i]));
  std::vector<RS> S(R.n());
  for (RS& s : S) {
    memset(&s.part, 0, sizeof s.part);
    memset(&s.C, 0, sizeof s.C);
  }
  const phfem_status st =
      dist_pipeline(R, meshes, nC_all, nE_all, levels, coeffs, f, g, uD, t, hist_sample, flags, outs, S);
  if (st != PHFEM_OK) {
    // leave nothing behind: partial per-rank state and outputs
    cudaDeviceSynchronize();
    for (int i = 0; i < R.n(); ++i) {
      RS& s = S[i];
      phfem_topology_release(R.ctx[i], &s.part);
      phfem_csr_release(R.ctx[i], &s.C);
      if (s.own_ee) dfree(R.ctx[i], s.ee);
      if (s.own_elements) dfree(R.ctx[i], s.elements);
      if (s.own_coords) dfree(R.ctx[i], s.coords);
      dfree(R.ctx[i], s.rpos);
      dfree(R.ctx[i], s.redges);
      phfem_dist_rank_out_release(R.ctx[i], &outs[i]);
    }
    if (!c->message.empty() && R.ctx[0]->message.empty()) R.ctx[0]->message = c->message;
  }
  return st;
}
