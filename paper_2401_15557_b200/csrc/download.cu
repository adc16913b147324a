// download.cu — phfem_pipeline_download: every output of the fused pipeline
// into the caller's host buffers in the reference's layouts (the drop-in /
// e2e path).  PCIe is the bottleneck (65.5 GB of outputs at L13), so the
// redundant parts are not sent twice:
//   * B is symmetric (6 distinct of 9 per block), D column-constant (3), M and
//     M0 hold two values (diagonal, off-diagonal) — assembly.cpp:59-75,
//     134-140: 13 doubles per element cross the bus instead of 36;
//   * C's values are +-|E|/2 per row and its pattern follows from the edge
//     arrays (assembly.cpp:144-168): one double per row crosses the bus;
//   * local_in_tplus / local_in_tminus travel as one byte per edge;
//   * interior_edges, retained_edges, retained_pos and bD do not travel at
//     all: they follow from the (small) boundary, Neumann and Dirichlet id
//     lists (edge_topology.cpp:104-113, 165-173: ascending complements and
//     running positions; assembly.cpp:230-242: bD is zero outside the
//     Dirichlet rows, whose values come along gathered).
// A device pack kernel writes the compact form, chunks of it are copied into
// a pinned staging buffer (kept in the ctx), and host threads expand each
// chunk into the caller's buffers as soon as its copy event fires, while the
// copy engine streams the next chunk and then the arrays sent as they are.
// The expansion only copies bits, so the host buffers equal the device
// outputs exactly.
#include <algorithm>
#include <climits>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <thread>
#include <vector>

#include <emmintrin.h>  // SSE2 streaming stores (baseline x86-64)

#include "common.cuh"

namespace phfem {

__global__ void k_pack_blocks(const double* __restrict__ B, const double* __restrict__ D,
                              const double* __restrict__ M, const double* __restrict__ M0, int64_t e0,
                              int64_t n, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = e0 + i;
    const double* b = B + 9 * m;
    double* o = out + 13 * i;
    // upper triangle of B (column-major index 3j + i)
    o[0] = b[0];
    o[1] = b[3];
    o[2] = b[6];
    o[3] = b[4];
    o[4] = b[7];
    o[5] = b[8];
    o[6] = D[9 * m];
    o[7] = D[9 * m + 3];
    o[8] = D[9 * m + 6];
    o[9] = M[9 * m];
    o[10] = M[9 * m + 1];
    o[11] = M0[9 * m];
    o[12] = M0[9 * m + 1];
  }
}

__global__ void k_pack_c(const int32_t* __restrict__ row_ptr, const double* __restrict__ vals, int L,
                         double* __restrict__ out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < L;
       r += (int64_t)gridDim.x * blockDim.x)
    out[r] = vals[row_ptr[r]];  // the T+ value |E|/2 (T- entries are its negation)
}

__global__ void k_pack_locals(const int32_t* __restrict__ ltp, const int32_t* __restrict__ ltm, int E,
                              uint8_t* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x)
    out[e] = (uint8_t)(ltp[e] | (ltm[e] + 1) << 2);
}

// bD at the Dirichlet rows (list order; rows of Neumann edges give 0, unused)
__global__ void k_pack_bd(const double* __restrict__ bd, const int32_t* __restrict__ rpos,
                          const int32_t* __restrict__ dir_ids, int n, double* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int r = rpos[dir_ids[i]];
    out[i] = r >= 0 ? bd[r] : 0.0;
  }
}

struct HostPool {
  int n;
  explicit HostPool(int threads) : n(threads) {}
  template <typename Fn>
  void run(int64_t count, Fn fn) {  // fn(begin, end) over [0, count)
    if (count <= 0) return;
    const int t = (int)std::max<int64_t>(1, std::min<int64_t>(n, count / 65536 + 1));
    std::vector<std::thread> th;
    for (int k = 0; k < t; ++k)
      th.emplace_back([&, k] { fn(count * k / t, count * (k + 1) / t); });
    for (auto& x : th) x.join();
  }
};

static phfem_status staging(phfem_ctx* ctx, size_t bytes, void** p) {
  static thread_local std::vector<std::pair<phfem_ctx*, std::pair<void*, size_t>>> cache;
  for (auto& c : cache)
    if (c.first == ctx) {
      if (c.second.second >= bytes) {
        *p = c.second.first;
        return PHFEM_OK;
      }
      cudaFreeHost(c.second.first);
      c.second = {nullptr, 0};
      PHFEM_CUDA(ctx, cudaHostAlloc(&c.second.first, bytes, cudaHostAllocDefault));
      c.second.second = bytes;
      *p = c.second.first;
      return PHFEM_OK;
    }
  void* q = nullptr;
  PHFEM_CUDA(ctx, cudaHostAlloc(&q, bytes, cudaHostAllocDefault));
  cache.push_back({ctx, {q, bytes}});
  *p = q;
  return PHFEM_OK;
}

}  // namespace phfem

using namespace phfem;

namespace {
struct Piece {
  void* dst;
  const void* src;
  size_t bytes;
};
}  // namespace

PHFEM_API int64_t phfem_pipeline_download_bytes(const phfem_pipeline_out* o,
                                                const phfem_pipeline_host* d) {
  // bytes crossing PCIe with the compact encodings
  const int64_t nC = o->mesh.nC, nE = o->mesh.nE, E = o->topo.E, L = o->cls.L;
  int64_t b = 0;
  auto add = [&](const void* dst, int64_t bytes) {
    if (dst) b += bytes;
  };
  add(d->coords, 16 * nC);
  add(d->elements, 12 * nE);
  add(d->dirichlet, 8 * (int64_t)o->mesh.nD);
  add(d->neumann, 8 * (int64_t)o->mesh.nN);
  add(d->edge_nodes, 8 * E);
  add(d->edge_elements, 8 * E);
  if (d->local_in_tplus || d->local_in_tminus) b += E;
  add(d->boundary_edges, 4 * (int64_t)o->topo.n_boundary);
  // interior / retained arrays and bD are derived on the host from id lists
  if (d->interior_edges) b += 4 * (int64_t)o->topo.n_boundary;
  if (d->retained_pos || d->retained_edges || d->bd || d->C_row_ptr || d->C_col_idx || d->C_values)
    b += 4 * (int64_t)o->cls.nN;
  if (d->bd) b += 12 * (int64_t)o->cls.nD;
  add(d->elem_edge, 12 * nE);
  add(d->dirichlet_edge_ids, 4 * (int64_t)o->cls.nD);
  add(d->neumann_edge_ids, 4 * (int64_t)o->cls.nN);
  if (d->C_row_ptr || d->C_col_idx || d->C_values) b += 8 * L;
  if (d->B || d->D || d->M || d->M0) b += 104 * nE;
  add(d->load, 24 * nE);
  return b;
}

PHFEM_API phfem_status phfem_pipeline_download(phfem_ctx* ctx, const phfem_pipeline_out* o,
                                               const phfem_pipeline_host* d) {
  if (!ctx || !o || !d) return PHFEM_ERR_INVALID_ARGUMENT;
  const bool trace = std::getenv("PHFEM_DL_TRACE") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  auto tick = [&](const char* what) {
    if (trace)
      fprintf(stderr, "[download] %-18s %8.1f ms\n", what,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  };
  const int64_t nC = o->mesh.nC, nE = o->mesh.nE, E = o->topo.E, L = o->cls.L;
  const bool want_blocks = d->B || d->D || d->M || d->M0;
  const bool want_c = d->C_row_ptr || d->C_col_idx || d->C_values;
  const bool want_loc = d->local_in_tplus || d->local_in_tminus;
  // C is rebuilt from the edge arrays: they must come along
  std::vector<int32_t> tmp_el, tmp_re;
  std::vector<uint8_t> dummy;
  int32_t* h_el = d->edge_elements;
  int32_t* h_re = d->retained_edges;
  if (want_c && !h_el) {
    tmp_el.resize(2 * E);
    h_el = tmp_el.data();
  }
  if (want_c && !h_re) {
    tmp_re.resize(L);
    h_re = tmp_re.data();
  }
  // the id lists the host derives interior / retained arrays and bD from
  const bool want_bd = d->bd != nullptr;
  const bool need_neu = d->retained_pos || h_re || want_bd;
  const int64_t nB = o->topo.n_boundary, nNc = o->cls.nN, nDc = o->cls.nD;
  std::vector<int32_t> hb(d->interior_edges ? nB : 0), hn(need_neu ? nNc : 0), hd(want_bd ? nDc : 0);
  std::vector<double> hbv(want_bd ? nDc : 0);
  if (!hb.empty())
    PHFEM_CUDA(ctx, cudaMemcpyAsync(hb.data(), o->topo.boundary_edges, 4 * hb.size(), cudaMemcpyDeviceToHost,
                                    ctx->stream));
  if (!hn.empty())
    PHFEM_CUDA(ctx, cudaMemcpyAsync(hn.data(), o->cls.neumann_edge_ids, 4 * hn.size(), cudaMemcpyDeviceToHost,
                                    ctx->stream));
  double* dbv = nullptr;
  if (!hd.empty()) {
    PHFEM_TRY(dalloc(ctx, &dbv, nDc));
    PHFEM_LAUNCH(ctx, "k_pack_bd", k_pack_bd<<<grid_for(nDc, 256, ctx->num_sms * 4), 256, 0, ctx->stream>>>(
        o->bd, o->cls.retained_pos, o->cls.dirichlet_edge_ids, (int)nDc, dbv));
    PHFEM_CUDA(ctx, cudaMemcpyAsync(hd.data(), o->cls.dirichlet_edge_ids, 4 * hd.size(), cudaMemcpyDeviceToHost,
                                    ctx->stream));
    PHFEM_CUDA(ctx, cudaMemcpyAsync(hbv.data(), dbv, 8 * hbv.size(), cudaMemcpyDeviceToHost, ctx->stream));
  }
  if (!hb.empty() || !hn.empty() || !hd.empty()) PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  // elements per block chunk (416 MB compact).  Measured e2e at L13: chunks of
  // 2^22 / 2^20 / 2^18 / 2^16 elements 0.85-0.91 / 0.92 / 1.73-1.86 / 4.50 s
  // per step — small chunks do not keep the DMA'd data cache-resident for the
  // expansion, they only add per-chunk synchronisation
  const int64_t CH = int64_t(1) << 22;
  const int64_t nchunks = want_blocks ? (nE + CH - 1) / CH : 0;
  const size_t bytes_blocks = want_blocks ? (size_t)104 * nE : 0;
  const size_t bytes_c = (want_c ? 8 * (size_t)L : 0) + ((want_c || want_loc) ? (size_t)E : 0);
  void* stage = nullptr;
  PHFEM_TRY(staging(ctx, std::max<size_t>(bytes_blocks + bytes_c + 64, 64), &stage));
  double* sb = reinterpret_cast<double*>(stage);
  double* sc = sb + 13 * (want_blocks ? nE : 0);
  uint8_t* sl = reinterpret_cast<uint8_t*>(sc + (want_c ? L : 0));

  // device scratch for the compact forms
  double* dpk = nullptr;
  PHFEM_TRY(dalloc(ctx, &dpk, std::max<int64_t>(13 * std::min(nE, CH) * (nchunks > 1 ? 2 : 1), 1)));
  std::vector<cudaEvent_t> ev(nchunks + 1);
  for (auto& e : ev) PHFEM_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (int64_t c = 0; c < nchunks; ++c) {
    const int64_t e0 = c * CH, n = std::min(CH, nE - e0);
    double* dbuf = dpk + 13 * CH * (c & 1);
    PHFEM_LAUNCH(ctx, "k_pack_blocks", k_pack_blocks<<<grid_for(n, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
        o->B, o->D, o->M, o->M0, e0, n, dbuf));
    PHFEM_CUDA(ctx, cudaMemcpyAsync(sb + 13 * e0, dbuf, 104 * (size_t)n, cudaMemcpyDeviceToHost, ctx->stream));
    PHFEM_CUDA(ctx, cudaEventRecord(ev[c], ctx->stream));
  }
  // C values + packed locals (small), then everything sent as it is
  double* dcv = nullptr;
  uint8_t* dloc = nullptr;
  if (want_c && L > 0) {
    PHFEM_TRY(dalloc(ctx, &dcv, L));
    PHFEM_LAUNCH(ctx, "k_pack_c", k_pack_c<<<grid_for(L, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
        o->C.row_ptr, o->C.values, (int)L, dcv));
    PHFEM_CUDA(ctx, cudaMemcpyAsync(sc, dcv, 8 * (size_t)L, cudaMemcpyDeviceToHost, ctx->stream));
  }
  if ((want_c || want_loc) && E > 0) {
    PHFEM_TRY(dalloc(ctx, &dloc, E));
    PHFEM_LAUNCH(ctx, "k_pack_locals", k_pack_locals<<<grid_for(E, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
        o->topo.local_in_tplus, o->topo.local_in_tminus, (int)E, dloc));
    PHFEM_CUDA(ctx, cudaMemcpyAsync(sl, dloc, (size_t)E, cudaMemcpyDeviceToHost, ctx->stream));
  }
  Piece p[24];
  int np = 0;
  auto add = [&](void* dst, const void* src, size_t bytes) {
    if (dst && bytes) p[np++] = Piece{dst, src, bytes};
  };
  add(h_el, o->topo.edge_elements, 8 * (size_t)E);
  for (int i = 0; i < np; ++i)
    PHFEM_CUDA(ctx, cudaMemcpyAsync(p[i].dst, p[i].src, p[i].bytes, cudaMemcpyDeviceToHost, ctx->stream));
  PHFEM_CUDA(ctx, cudaEventRecord(ev[nchunks], ctx->stream));  // C inputs ready
  np = 0;
  add(d->coords, o->mesh.coords, 16 * (size_t)nC);
  add(d->elements, o->mesh.elements, 12 * (size_t)nE);
  add(d->dirichlet, o->mesh.dirichlet, 8 * (size_t)o->mesh.nD);
  add(d->neumann, o->mesh.neumann, 8 * (size_t)o->mesh.nN);
  add(d->edge_nodes, o->topo.edge_nodes, 8 * (size_t)E);
  add(d->boundary_edges, o->topo.boundary_edges, 4 * (size_t)o->topo.n_boundary);
  add(d->elem_edge, o->topo.elem_edge, 12 * (size_t)nE);
  add(d->dirichlet_edge_ids, o->cls.dirichlet_edge_ids, 4 * (size_t)o->cls.nD);
  add(d->neumann_edge_ids, o->cls.neumann_edge_ids, 4 * (size_t)o->cls.nN);
  add(d->load, o->load, 24 * (size_t)nE);
  for (int i = 0; i < np; ++i)
    PHFEM_CUDA(ctx, cudaMemcpyAsync(p[i].dst, p[i].src, p[i].bytes, cudaMemcpyDeviceToHost, ctx->stream));

  tick("issued");
  // host expansion, chunk by chunk, overlapping the copies still in flight
  // host threads for the expansion (PHFEM_DL_THREADS overrides; default: 2 per
  // core, measured 1-3 % faster than one per core on the 16-core host)
  static const int hw = [] {
    const char* e = std::getenv("PHFEM_DL_THREADS");
    if (e && atoi(e) > 0) return atoi(e);
    return (int)std::max(1u, std::min(64u, 2 * std::thread::hardware_concurrency()));
  }();
  HostPool pool(hw);
  for (int64_t c = 0; c < nchunks; ++c) {
    PHFEM_CUDA(ctx, cudaEventSynchronize(ev[c]));
    const int64_t e0 = c * CH, n = std::min(CH, nE - e0);
    // element pairs (2 x 9 doubles = 9 aligned 16-B lines): non-temporal
    // stores, so the host writes its outputs once instead of read-for-ownership
    // + write (host memory bandwidth, not PCIe, bounds this path)
    const bool nt = ((uintptr_t)d->B | (uintptr_t)d->D | (uintptr_t)d->M | (uintptr_t)d->M0) % 16 == 0;
    pool.run((n + 1) / 2, [&](int64_t a, int64_t b) {
      for (int64_t pi = a; pi < b; ++pi) {
        const int64_t m0 = e0 + 2 * pi;
        const int cnt = (m0 + 1 < e0 + n) ? 2 : 1;
        double x[4][18];
        for (int h = 0; h < cnt; ++h) {
          const double* u = sb + 13 * (m0 + h);
          double* xb = x[0] + 9 * h;
          xb[0] = u[0]; xb[1] = u[1]; xb[2] = u[2];
          xb[3] = u[1]; xb[4] = u[3]; xb[5] = u[4];
          xb[6] = u[2]; xb[7] = u[4]; xb[8] = u[5];
          double* xd = x[1] + 9 * h;
          xd[0] = xd[1] = xd[2] = u[6];
          xd[3] = xd[4] = xd[5] = u[7];
          xd[6] = xd[7] = xd[8] = u[8];
          double* xm = x[2] + 9 * h;
          xm[0] = xm[4] = xm[8] = u[9];
          xm[1] = xm[2] = xm[3] = xm[5] = xm[6] = xm[7] = u[10];
          double* xz = x[3] + 9 * h;
          xz[0] = xz[4] = xz[8] = u[11];
          xz[1] = xz[2] = xz[3] = xz[5] = xz[6] = xz[7] = u[12];
        }
        double* dsts[4] = {d->B, d->D, d->M, d->M0};
        for (int w = 0; w < 4; ++w) {
          if (!dsts[w]) continue;
          double* out = dsts[w] + 9 * m0;
          if (nt && cnt == 2) {
            for (int q = 0; q < 9; ++q) _mm_stream_pd(out + 2 * q, _mm_loadu_pd(x[w] + 2 * q));
          } else {
            for (int q = 0; q < 9 * cnt; ++q) out[q] = x[w][q];
          }
        }
      }
    });
  }
  _mm_sfence();
  tick("blocks expanded");
  // retained set = edges minus the (sorted, unique) Neumann ids: retained_edges
  // ascending, retained_pos the running position (edge_topology.cpp:165-173)
  std::sort(hn.begin(), hn.end());
  hn.erase(std::unique(hn.begin(), hn.end()), hn.end());
  auto below = [](const std::vector<int32_t>& v, int64_t x) {  // #entries < x
    return (int64_t)(std::lower_bound(v.begin(), v.end(), (int32_t)std::min<int64_t>(x, INT32_MAX)) - v.begin());
  };
  if (h_re || d->retained_pos) {
    int32_t* rpos = d->retained_pos;
    pool.run(E, [&](int64_t a, int64_t b) {
      int64_t k = below(hn, a), q = a - k;
      for (int64_t e = a; e < b; ++e) {
        // non-temporal stores: written once, never read back here
        if (k < (int64_t)hn.size() && hn[k] == e) {
          if (rpos) _mm_stream_si32(rpos + e, -1);
          ++k;
        } else {
          if (h_re) _mm_stream_si32(h_re + q, (int)e);
          if (rpos) _mm_stream_si32(rpos + e, (int)q);
          ++q;
        }
      }
      _mm_sfence();
    });
  }
  if (d->interior_edges) {  // ascending complement of the boundary list (edge_topology.cpp:104-113)
    int32_t* in = d->interior_edges;
    pool.run(E, [&](int64_t a, int64_t b) {
      int64_t k = below(hb, a), q = a - k;
      for (int64_t e = a; e < b; ++e) {
        if (k < (int64_t)hb.size() && hb[k] == e) ++k;
        else _mm_stream_si32(in + q++, (int)e);
      }
      _mm_sfence();
    });
  }
  if (want_bd) {  // zero outside the Dirichlet rows (assembly.cpp:230-242)
    double* bd = d->bd;
    pool.run(L, [&](int64_t a, int64_t b) {
      for (int64_t i = a; i < b; ++i) _mm_stream_si64(reinterpret_cast<long long*>(bd + i), 0);
      _mm_sfence();
    });
    for (int64_t i = 0; i < nDc; ++i) {
      const int64_t e = hd[i];
      const int64_t k = below(hn, e);
      if (k < (int64_t)hn.size() && hn[k] == e) continue;  // a Neumann edge has no row
      bd[e - k] = hbv[i];
    }
  }
  tick("lists derived");
  PHFEM_CUDA(ctx, cudaEventSynchronize(ev[nchunks]));
  tick("C inputs arrived");
  if (want_loc) {
    pool.run(E, [&](int64_t a, int64_t b) {
      for (int64_t e = a; e < b; ++e) {
        if (d->local_in_tplus) d->local_in_tplus[e] = sl[e] & 3;
        if (d->local_in_tminus) d->local_in_tminus[e] = (sl[e] >> 2) - 1;
      }
    });
  }
  if (want_c) {
    // rows r: cols 3 tp + c (c != ltp), then 3 tm + c (c != ltm); values v, v, -v, -v
    const bool ntc = (uintptr_t)d->C_values % 16 == 0 && (uintptr_t)d->C_col_idx % 8 == 0;
    // row ranges per thread: count boundary rows (2 entries) in parallel, prefix, fill
    const int t = (int)std::max<int64_t>(1, std::min<int64_t>(hw, L / 65536 + 1));
    std::vector<int64_t> off(t + 1, 0);
    {
      std::vector<std::thread> th;
      for (int k = 0; k < t; ++k)
        th.emplace_back([&, k] {
          const int64_t a = L * k / t, b = L * (k + 1) / t;
          int64_t bd = 0;
          for (int64_t r = a; r < b; ++r) bd += h_el[2 * (int64_t)h_re[r] + 1] < 0;
          off[k + 1] = 4 * (b - a) - 2 * bd;
        });
      for (auto& x : th) x.join();
      for (int k = 0; k < t; ++k) off[k + 1] += off[k];
    }
    std::vector<std::thread> th;
    for (int k = 0; k < t; ++k)
      th.emplace_back([&, k] {
        const int64_t a = L * k / t, b = L * (k + 1) / t;
        int64_t q = off[k];
        for (int64_t r = a; r < b; ++r) {
          const int64_t e = h_re[r];
          const int tp = h_el[2 * e], tm = h_el[2 * e + 1];
          const int lp = sl[e] & 3, lm = (sl[e] >> 2) - 1;
          const double v = sc[r];
          if (d->C_row_ptr) d->C_row_ptr[r] = (int32_t)q;
          // q is even (rows hold 2 or 4 entries): 16-B aligned value pairs,
          // 8-B aligned column pairs -> streaming stores
          const int cp0 = lp == 0 ? 1 : 0, cp1 = lp == 2 ? 1 : 2;
          const int cm0 = lm == 0 ? 1 : 0, cm1 = lm == 2 ? 1 : 2;
          const int nq = tm >= 0 ? 4 : 2;
          const int32_t cols[4] = {3 * tp + cp0, 3 * tp + cp1, 3 * tm + cm0, 3 * tm + cm1};
          if (ntc) {
            if (d->C_col_idx)
              for (int h = 0; h < nq; h += 2)
                _mm_stream_si64(reinterpret_cast<long long*>(d->C_col_idx + q + h),
                                (long long)(uint32_t)cols[h] | (long long)(uint32_t)cols[h + 1] << 32);
            if (d->C_values) {
              _mm_stream_pd(d->C_values + q, _mm_set1_pd(v));
              if (nq == 4) _mm_stream_pd(d->C_values + q + 2, _mm_set1_pd(-v));
            }
          } else {
            for (int h = 0; h < nq; ++h) {
              if (d->C_col_idx) d->C_col_idx[q + h] = cols[h];
              if (d->C_values) d->C_values[q + h] = h < 2 ? v : -v;
            }
          }
          q += nq;
        }
        if (k == t - 1 && d->C_row_ptr) d->C_row_ptr[L] = (int32_t)q;
        _mm_sfence();
      });
    for (auto& x : th) x.join();
  }
  tick("C expanded");
  PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  tick("all copies done");
  for (auto& e : ev) cudaEventDestroy(e);
  dfree(ctx, dpk);
  dfree(ctx, dcv);
  dfree(ctx, dloc);
  dfree(ctx, dbv);
  return PHFEM_OK;
}
