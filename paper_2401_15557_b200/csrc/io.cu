// io.cu — SURVEY §8(f3): the reference's on-disk formats at scale.
//
//  * load_mesh (mesh.cpp:114-150; read_rows / parse_double / parse_index /
//    read_boundary / normalize_against_cycles :17-98): 4 text files ->
//    device mesh, every validation with the reference's message and order;
//  * save_mesh (mesh.cpp:170-180): `%.17g` coordinates, 1-based ids;
//  * the CLI's topology CSV (tools/main.cpp:302-323).
//
// Integer files (elements, boundary pairs) are parsed ON THE DEVICE: newline
// positions by a count / scan / scatter over 4 KB chunks, one thread per
// line for the tokens (the reference's whitespace set, blank lines skipped,
// strtol semantics incl. sign and 64-bit overflow), the signed-area check of
// each element fused into the same pass, and the boundary-pair normalisation
// against the element cycles as one streaming pass over the elements with a
// small hash set of the pairs.  All output text is FORMATTED on the device
// (line lengths, 64-bit scan, bytes, one copy back): ids, and the
// coordinates / CSV lengths through fmt.cuh's exact "%.<P>g" (128-bit
// scaling, big-integer fallback; byte-identical to glibc's printf).  Parsing
// floating-point text (exact decimal -> binary) runs on host threads through
// std::from_chars (correctly rounded like strtod); any token outside the plain
// decimal grammar or whose value is not a normal number goes through
// std::stod itself, so hex floats, inf/nan and ERANGE behave exactly as in
// the reference.  The first
// error in the reference's order (file, row, check) is found as a minimum
// over per-row keys; its message is rebuilt on the host from the text.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <system_error>
#include <thread>
#include <vector>

#include "common.cuh"
#include "fmt.cuh"

namespace phfem {

// ---------------------------------------------------------------- device side
constexpr int kIoChunk = 4096;   // bytes per block in the newline passes
constexpr int kIoThreads = 256;  // 16 bytes per thread

__device__ __forceinline__ bool io_space(unsigned char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

__global__ void __launch_bounds__(kIoThreads) k_nl_count(const char* __restrict__ s, int64_t n,
                                                         int32_t* __restrict__ cnt) {
  __shared__ int32_t sm[33];
  const int64_t base = (int64_t)blockIdx.x * kIoChunk + threadIdx.x * 16;
  int c = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) c += (base + k < n && s[base + k] == '\n');
  int32_t tot;
  block_exclusive_scan(c, sm, &tot);
  if (threadIdx.x == 0) cnt[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kIoThreads) k_nl_pos(const char* __restrict__ s, int64_t n,
                                                       const int32_t* __restrict__ off,
                                                       int64_t* __restrict__ pos) {
  __shared__ int32_t sm[33];
  const int64_t base = (int64_t)blockIdx.x * kIoChunk + threadIdx.x * 16;
  int c = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) c += (base + k < n && s[base + k] == '\n');
  int32_t tot;
  int ex = block_exclusive_scan(c, sm, &tot) + off[blockIdx.x];
#pragma unroll
  for (int k = 0; k < 16; ++k)
    if (base + k < n && s[base + k] == '\n') pos[ex++] = base + k;
}

struct Lines {
  const char* s;
  int64_t n;
  const int64_t* nl;  // newline positions
  int32_t n_nl, nlines;
  __device__ void span(int k, int64_t* a, int64_t* b) const {
    *a = k == 0 ? 0 : nl[k - 1] + 1;
    *b = k < n_nl ? nl[k] : n;
  }
};

__global__ void k_line_nonblank(Lines L, int32_t* __restrict__ flag) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < L.nlines;
       k += (int64_t)gridDim.x * blockDim.x) {
    int64_t a, b;
    L.span((int)k, &a, &b);
    int f = 0;
    for (int64_t i = a; i < b && !f; ++i) f = !io_space((unsigned char)L.s[i]);
    flag[k] = f;
  }
}

// One text row of K indices -> out[row][K] (0-based), the smallest failing
// (row << 3 | check) into *err: check 0 = entry count, 1 + 2j / 2 + 2j = token
// j not an index / out of range, 7 = non-positive signed area (elements).
template <int K>
__global__ void k_parse_index_rows(Lines L, const int32_t* __restrict__ row_of, int node_count,
                                   const double2* __restrict__ coords, int32_t* __restrict__ out,
                                   unsigned long long* __restrict__ err) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < L.nlines;
       k += (int64_t)gridDim.x * blockDim.x) {
    int64_t a, b;
    L.span((int)k, &a, &b);
    const int64_t r = row_of[k];
    int ntok = 0;
    int64_t ts[K], te[K];
    for (int64_t i = a; i < b;) {
      while (i < b && io_space((unsigned char)L.s[i])) ++i;
      if (i >= b) break;
      const int64_t t0 = i;
      while (i < b && !io_space((unsigned char)L.s[i])) ++i;
      if (ntok < K) {
        ts[ntok] = t0;
        te[ntok] = i;
      }
      ++ntok;
    }
    if (ntok == 0) continue;  // blank line: not a row
    unsigned long long key = ~0ull;
    int v[K];
    if (ntok != K) {
      key = (unsigned long long)r << 3;
    } else {
      for (int j = 0; j < K && key == ~0ull; ++j) {
        // std::stol: [+-]?[0-9]+ consuming the whole token, fits in a long
        int64_t i = ts[j];
        bool neg = false;
        if (L.s[i] == '+' || L.s[i] == '-') neg = L.s[i++] == '-';
        unsigned long long acc = 0;
        bool ok = i < te[j], over = false;
        for (; i < te[j]; ++i) {
          const unsigned d = (unsigned char)L.s[i] - '0';
          if (d > 9) {
            ok = false;
            break;
          }
          if (acc > (~0ull - d) / 10) over = true;
          else acc = acc * 10 + d;
        }
        const unsigned long long lim = neg ? (1ull << 63) : (1ull << 63) - 1;
        if (!ok || over || acc > lim) {
          key = (unsigned long long)r << 3 | (unsigned long long)(1 + 2 * j);
        } else if (neg || acc < 1 || acc > (unsigned long long)node_count) {
          key = (unsigned long long)r << 3 | (unsigned long long)(2 + 2 * j);
        } else {
          v[j] = (int)acc - 1;
        }
      }
      if (key == ~0ull) {
#pragma unroll
        for (int j = 0; j < K; ++j) out[K * r + j] = v[j];
        if (coords) {  // element_area > 0 (mesh.cpp:140-142; signed_area2 :104-106)
          const double2 p0 = coords[v[0]], p1 = coords[v[1]], p2 = coords[v[2 % K]];
          const double area = 0.5 * ((p1.x - p0.x) * (p2.y - p0.y) - (p1.y - p0.y) * (p2.x - p0.x));
          if (!(area > 0.0)) key = (unsigned long long)r << 3 | 7ull;
        }
      }
    }
    if (key != ~0ull) atomicMin(err, key);
  }
}

// ---- boundary pairs vs the element cycles (normalize_against_cycles) -------
__device__ __forceinline__ uint32_t pair_hash(unsigned long long key, int cap) {
  return (uint32_t)((key * 0x9E3779B97F4A7C15ull) >> 32) & (uint32_t)(cap - 1);
}

__global__ void k_pair_insert(const int32_t* __restrict__ pairs, int n, int cap,
                              unsigned long long* __restrict__ keys) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned long long key =
        (unsigned long long)(uint32_t)pairs[2 * i] << 32 | (uint32_t)pairs[2 * i + 1];
    uint32_t h = pair_hash(key, cap);
    while (true) {
      const unsigned long long prev = atomicCAS(keys + h, ~0ull, key);
      if (prev == ~0ull || prev == key) break;
      h = (h + 1) & (uint32_t)(cap - 1);
    }
  }
}

__device__ __forceinline__ int pair_find(const unsigned long long* __restrict__ keys, int cap,
                                         unsigned long long key) {
  uint32_t h = pair_hash(key, cap);
  while (true) {
    const unsigned long long k = keys[h];
    if (k == key) return (int)h;
    if (k == ~0ull) return -1;
    h = (h + 1) & (uint32_t)(cap - 1);
  }
}

// bit 1: some element has the directed pair (a, b); bit 2: some has (b, a)
__global__ void k_pair_mark(const int32_t* __restrict__ elements, int nE, int cap,
                            const unsigned long long* __restrict__ keys, uint32_t* __restrict__ flag) {
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < nE;
       m += (int64_t)gridDim.x * blockDim.x) {
    const int t[3] = {elements[3 * m], elements[3 * m + 1], elements[3 * m + 2]};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const uint32_t u = (uint32_t)t[k], w = (uint32_t)t[(k + 1) % 3];
      const int f = pair_find(keys, cap, (unsigned long long)u << 32 | w);
      if (f >= 0 && !(flag[f] & 1u)) atomicOr(flag + f, 1u);
      const int r = pair_find(keys, cap, (unsigned long long)w << 32 | u);
      if (r >= 0 && !(flag[r] & 2u)) atomicOr(flag + r, 2u);
    }
  }
}

__global__ void k_pair_apply(int32_t* __restrict__ pairs, int n, int cap,
                             const unsigned long long* __restrict__ keys,
                             const uint32_t* __restrict__ flag) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int a = pairs[2 * i], b = pairs[2 * i + 1];
    const int s = pair_find(keys, cap, (unsigned long long)(uint32_t)a << 32 | (uint32_t)b);
    const uint32_t f = s >= 0 ? flag[s] : 0u;
    if (!(f & 1u) && (f & 2u)) {  // only the flipped direction is a cycle pair
      pairs[2 * i] = b;
      pairs[2 * i + 1] = a;
    }
  }
}

// ---- formatting of index rows: "i+1 j+1 ...\n" ------------------------------
__device__ __forceinline__ int ndigits(uint32_t v) {
  int d = 1;
  while (v >= 10) {
    v /= 10;
    ++d;
  }
  return d;
}

template <int K>
__global__ void k_fmt_len(const int32_t* __restrict__ ids, int64_t rows, int64_t* __restrict__ len) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    int l = K;  // K-1 separators + '\n'
#pragma unroll
    for (int j = 0; j < K; ++j) l += ndigits((uint32_t)(ids[K * r + j] + 1));
    len[r] = l;
  }
}

template <int K>
__global__ void k_fmt_write(const int32_t* __restrict__ ids, int64_t rows, const int64_t* __restrict__ off,
                            char* __restrict__ out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    char* p = out + off[r];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      uint32_t v = (uint32_t)(ids[K * r + j] + 1);
      const int d = ndigits(v);
      for (int q = d - 1; q >= 0; --q) {
        p[q] = (char)('0' + v % 10);
        v /= 10;
      }
      p += d;
      *p++ = j + 1 < K ? ' ' : '\n';
    }
  }
}

// "%.17g %.17g\n" per node (save_mesh / format_g17, mesh.cpp:95-99, 172-173)
__global__ void k_fmt_coords_len(const double* __restrict__ xy, int64_t rows, int64_t* __restrict__ len) {
  char buf[32];
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x)
    len[r] = fmt_g(xy[2 * r], 17, buf) + fmt_g(xy[2 * r + 1], 17, buf) + 2;
}

__global__ void k_fmt_coords_write(const double* __restrict__ xy, int64_t rows, const int64_t* __restrict__ off,
                                   char* __restrict__ out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    char* p = out + off[r];
    p += fmt_g(xy[2 * r], 17, p);
    *p++ = ' ';
    p += fmt_g(xy[2 * r + 1], 17, p);
    *p = '\n';
  }
}

// the CLI's topology CSV row (tools/main.cpp:315-318): 1-based ids, 0 for no
// t_minus, fmt(length) = "%.10g"
__device__ __forceinline__ int put_uint(char* p, uint32_t v) {
  const int d = ndigits(v);
  for (int q = d - 1; q >= 0; --q) {
    p[q] = (char)('0' + v % 10);
    v /= 10;
  }
  return d;
}

template <bool kWrite>
__global__ void k_fmt_csv(const int32_t* __restrict__ edge_nodes, const int32_t* __restrict__ edge_elements,
                          const int32_t* __restrict__ ltp, const int32_t* __restrict__ ltm,
                          const double2* __restrict__ coords, int64_t E, int64_t* __restrict__ len_off,
                          char* __restrict__ out) {
  char buf[96];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int2 ab = reinterpret_cast<const int2*>(edge_nodes)[e];
    const int2 el = reinterpret_cast<const int2*>(edge_elements)[e];
    const double2 pa = coords[ab.x], pb = coords[ab.y];
    const double dx = pb.x - pa.x, dy = pb.y - pa.y;
    const double len = sqrt(dx * dx + dy * dy);  // edge_lengths, edge_topology.cpp:183
    char* p = kWrite ? out + len_off[e] : buf;
    char* q = p;
    q += put_uint(q, (uint32_t)(e + 1));
    *q++ = ',';
    q += put_uint(q, (uint32_t)(ab.x + 1));
    *q++ = ',';
    q += put_uint(q, (uint32_t)(ab.y + 1));
    *q++ = ',';
    q += put_uint(q, (uint32_t)(el.x + 1));
    *q++ = ',';
    q += put_uint(q, (uint32_t)(el.y + 1));
    *q++ = ',';
    q += put_uint(q, (uint32_t)(ltp[e] + 1));
    *q++ = ',';
    q += put_uint(q, (uint32_t)(el.y >= 0 ? ltm[e] + 1 : 0));
    *q++ = ',';
    q += fmt_g(len, 10, q);
    *q++ = '\n';
    if (!kWrite) len_off[e] = q - p;
  }
}

// test entry: "%.<P>g" of n device doubles into 32-byte slots + lengths
__global__ void k_fmt_g_test(const double* __restrict__ v, int64_t n, int P, char* __restrict__ out,
                             int32_t* __restrict__ lens) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    lens[i] = fmt_g(v[i], P, out + 32 * i);
}

// ---------------------------------------------------------------- host side
namespace {

int io_threads() {
  if (const char* e = getenv("PHFEM_IO_THREADS")) {
    const int v = atoi(e);
    if (v > 0) return v;
  }
  return (int)std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
}

template <class F>
void parallel_for(int n, F&& f) {
  std::vector<std::thread> th;
  for (int i = 1; i < n; ++i) th.emplace_back(f, i);
  f(0);
  for (auto& t : th) t.join();
}

inline bool host_space(char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

// chunk boundaries at line starts
std::vector<size_t> line_chunks(const char* s, size_t n, int parts) {
  std::vector<size_t> b((size_t)parts + 1, n);
  b[0] = 0;
  for (int i = 1; i < parts; ++i) {
    size_t p = std::max(b[i - 1], n / parts * (size_t)i);
    while (p < n && p > 0 && s[p - 1] != '\n') ++p;
    b[i] = p;
  }
  return b;
}

// tokens of line [p, q)
template <class F>
int for_tokens(const char* p, const char* q, F&& f) {
  int n = 0;
  while (p < q) {
    while (p < q && host_space(*p)) ++p;
    if (p >= q) break;
    const char* t = p;
    while (p < q && !host_space(*p)) ++p;
    f(n++, t, p);
  }
  return n;
}

// parse_double (mesh.cpp:31-44): std::stod consuming the whole token, finite
bool parse_double_tok(const char* p, const char* q, double* v) {
  const char* r = p;
  if (r < q && *r == '-') ++r;
  bool nonzero = false;
  int nd = 0;
  while (r < q && *r >= '0' && *r <= '9') nonzero |= *r++ != '0', ++nd;
  if (r < q && *r == '.') {
    ++r;
    while (r < q && *r >= '0' && *r <= '9') nonzero |= *r++ != '0', ++nd;
  }
  bool plain = nd > 0;
  if (plain && r < q && (*r == 'e' || *r == 'E')) {
    ++r;
    if (r < q && (*r == '+' || *r == '-')) ++r;
    int ne = 0;
    while (r < q && *r >= '0' && *r <= '9') ++r, ++ne;
    plain = ne > 0;
  }
  if (plain && r == q) {
    double x = 0.0;
    const auto res = std::from_chars(p, q, x);
    // correctly rounded like strtod; normal results (or an exact zero) cannot
    // have raised ERANGE there
    if (res.ec == std::errc() && res.ptr == q && (std::isnormal(x) || (x == 0.0 && !nonzero))) {
      *v = x;
      return true;
    }
  }
  const std::string tok(p, q);
  size_t pos = 0;
  double x = 0.0;
  try {
    x = std::stod(tok, &pos);
  } catch (const std::exception&) {
    pos = 0;
  }
  if (pos != tok.size() || !std::isfinite(x)) return false;
  *v = x;
  return true;
}

struct RowError {
  int64_t row = -1;  // 0-based row of the first error, -1 none
  int check = 0;     // 0 count, 1/2 token 0/1 not finite
  int ntok = 0;
  std::string tok;
};

// coordinates file: count pass, then parse pass into out[2 * rows]
phfem_status parse_coords(phfem_ctx* ctx, const char* s, size_t n, std::vector<double>& out) {
  const int T = n < (1u << 20) ? 1 : io_threads();
  const auto b = line_chunks(s, n, T);
  std::vector<int64_t> rows((size_t)T + 1, 0);
  parallel_for(T, [&](int t) {
    int64_t c = 0;
    const char* p = s + b[t];
    const char* e = s + b[t + 1];
    while (p < e) {
      const char* q = (const char*)memchr(p, '\n', (size_t)(e - p));
      if (!q) q = e;
      for (const char* i = p; i < q; ++i)
        if (!host_space(*i)) {
          ++c;
          break;
        }
      p = q + 1;
    }
    rows[t + 1] = c;
  });
  for (int t = 0; t < T; ++t) rows[t + 1] += rows[t];
  out.assign(2 * (size_t)rows[T], 0.0);
  std::vector<RowError> errs((size_t)T);
  parallel_for(T, [&](int t) {
    int64_t r = rows[t];
    const char* p = s + b[t];
    const char* e = s + b[t + 1];
    RowError& er = errs[t];
    while (p < e && er.row < 0) {
      const char* q = (const char*)memchr(p, '\n', (size_t)(e - p));
      if (!q) q = e;
      const char* ts[2] = {nullptr, nullptr};
      const char* te[2] = {nullptr, nullptr};
      const int nt = for_tokens(p, q, [&](int k, const char* a, const char* z) {
        if (k < 2) {
          ts[k] = a;
          te[k] = z;
        }
      });
      if (nt > 0) {
        if (nt != 2) {
          er.row = r;
          er.check = 0;
          er.ntok = nt;
        } else {
          for (int k = 0; k < 2 && er.row < 0; ++k)
            if (!parse_double_tok(ts[k], te[k], &out[2 * r + k])) {
              er.row = r;
              er.check = 1 + k;
              er.tok.assign(ts[k], te[k]);
            }
        }
        ++r;
      }
      p = q + 1;
    }
  });
  for (const RowError& er : errs) {
    if (er.row < 0) continue;
    if (er.check == 0)
      return set_error(ctx, PHFEM_ERR_RUNTIME, "coordinates: row %lld: expected 2 entries, got %d",
                       (long long)er.row + 1, er.ntok);
    return set_error(ctx, PHFEM_ERR_RUNTIME, "coordinates: row %lld: not a finite number: '%s'",
                     (long long)er.row + 1, er.tok.c_str());
  }
  return PHFEM_OK;
}

// the message of index-row error `key` of `what`, rebuilt from the host text
phfem_status index_row_error(phfem_ctx* ctx, const char* what, const char* s, size_t n,
                             unsigned long long key, int node_count) {
  const int64_t row = (int64_t)(key >> 3);
  const int check = (int)(key & 7);
  if (check == 7)
    return set_error(ctx, PHFEM_ERR_RUNTIME, "%s: element %lld has non-positive signed area (not CCW)", what,
                     (long long)row + 1);
  // find the row's tokens
  int64_t r = -1;
  const char* p = s;
  const char* e = s + n;
  std::vector<std::string> toks;
  while (p < e) {
    const char* q = (const char*)memchr(p, '\n', (size_t)(e - p));
    if (!q) q = e;
    std::vector<std::string> t;
    for_tokens(p, q, [&](int, const char* a, const char* z) { t.emplace_back(a, z); });
    if (!t.empty() && ++r == row) {
      toks = std::move(t);
      break;
    }
    p = q + 1;
  }
  if (check == 0)
    return set_error(ctx, PHFEM_ERR_RUNTIME, "%s: row %lld: expected %d entries, got %d", what,
                     (long long)row + 1, strcmp(what, "elements") == 0 ? 3 : 2, (int)toks.size());
  const int j = (check - 1) / 2;
  const std::string tok = j < (int)toks.size() ? toks[j] : std::string();
  if (check % 2 == 1)
    return set_error(ctx, PHFEM_ERR_RUNTIME, "%s: row %lld: not an index: '%s'", what, (long long)row + 1,
                     tok.c_str());
  const long v = std::stol(tok);
  return set_error(ctx, PHFEM_ERR_RUNTIME, "%s: row %lld: node index %ld out of range 1..%d", what,
                   (long long)row + 1, v, node_count);
}

}  // namespace

// Device parse of an index file -> out (library-allocated, [rows][K]).
template <int K>
static phfem_status parse_index_file(phfem_ctx* ctx, const char* what, const char* s, size_t n, int node_count,
                                     const double2* coords, int32_t** out, int32_t* nrows) {
  *out = nullptr;
  *nrows = 0;
  if (n == 0) return PHFEM_OK;
  if (n >= (size_t(1) << 40)) return set_error(ctx, PHFEM_ERR_INVALID_ARGUMENT, "%s: file too large", what);
  char* d = nullptr;
  PHFEM_TRY(dalloc(ctx, &d, n));
  PHFEM_CUDA(ctx, cudaMemcpyAsync(d, s, n, cudaMemcpyHostToDevice, ctx->stream));
  const int64_t nblk = ((int64_t)n + kIoChunk - 1) / kIoChunk;
  int32_t* cnt = nullptr;
  PHFEM_TRY(dalloc(ctx, &cnt, nblk + 1));
  PHFEM_LAUNCH(ctx, "k_nl_count", k_nl_count<<<(unsigned)nblk, kIoThreads, 0, ctx->stream>>>(d, (int64_t)n, cnt));
  PHFEM_CUDA(ctx, cudaMemsetAsync(cnt + nblk, 0, sizeof(int32_t), ctx->stream));
  int32_t* total = nullptr;
  PHFEM_TRY(dalloc(ctx, &total, 2));
  PHFEM_TRY(scan_exclusive_i32(ctx, cnt, cnt, nblk + 1, total));
  int32_t n_nl = 0;
  char last = 0;
  PHFEM_CUDA(ctx, cudaMemcpyAsync(&n_nl, total, sizeof n_nl, cudaMemcpyDeviceToHost, ctx->stream));
  PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  last = s[n - 1];
  Lines L;
  L.s = d;
  L.n = (int64_t)n;
  L.n_nl = n_nl;
  L.nlines = n_nl + (last != '\n' ? 1 : 0);
  int64_t* nl = nullptr;
  PHFEM_TRY(dalloc(ctx, &nl, std::max(n_nl, 1)));
  L.nl = nl;
  PHFEM_LAUNCH(ctx, "k_nl_pos", k_nl_pos<<<(unsigned)nblk, kIoThreads, 0, ctx->stream>>>(d, (int64_t)n, cnt, nl));
  int32_t* rowi = nullptr;
  PHFEM_TRY(dalloc(ctx, &rowi, (int64_t)L.nlines + 1));
  const int g = grid_for(L.nlines, 256, ctx->num_sms * 8);
  PHFEM_LAUNCH(ctx, "k_line_nonblank", k_line_nonblank<<<g, 256, 0, ctx->stream>>>(L, rowi));
  PHFEM_CUDA(ctx, cudaMemsetAsync(rowi + L.nlines, 0, sizeof(int32_t), ctx->stream));
  PHFEM_TRY(scan_exclusive_i32(ctx, rowi, rowi, (int64_t)L.nlines + 1, total));
  int32_t rows = 0;
  PHFEM_CUDA(ctx, cudaMemcpyAsync(&rows, total, sizeof rows, cudaMemcpyDeviceToHost, ctx->stream));
  PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  int32_t* o = nullptr;
  PHFEM_TRY(dalloc(ctx, &o, (int64_t)K * std::max(rows, 1)));
  unsigned long long* err = nullptr;
  PHFEM_TRY(dalloc(ctx, &err, 1));
  PHFEM_CUDA(ctx, cudaMemsetAsync(err, 0xff, sizeof(unsigned long long), ctx->stream));
  PHFEM_LAUNCH(ctx, "k_parse_index_rows", k_parse_index_rows<K><<<g, 256, 0, ctx->stream>>>(L, rowi, node_count,
                                                                                           coords, o, err));
  unsigned long long herr = 0;
  PHFEM_CUDA(ctx, cudaMemcpyAsync(&herr, err, sizeof herr, cudaMemcpyDeviceToHost, ctx->stream));
  PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  dfree(ctx, err);
  dfree(ctx, rowi);
  dfree(ctx, nl);
  dfree(ctx, total);
  dfree(ctx, cnt);
  dfree(ctx, d);
  if (herr != ~0ull) {
    dfree(ctx, o);
    return index_row_error(ctx, what, s, n, herr, node_count);
  }
  *out = o;
  *nrows = rows;
  return PHFEM_OK;
}

static phfem_status normalize_pairs(phfem_ctx* ctx, const phfem_mesh* m) {
  const int nB = m->nD + m->nN;
  if (nB == 0 || m->nE == 0) return PHFEM_OK;
  int cap = 64;
  while (cap < 2 * nB) cap <<= 1;
  unsigned long long* keys = nullptr;
  uint32_t* flag = nullptr;
  PHFEM_TRY(dalloc(ctx, &keys, cap));
  PHFEM_TRY(dalloc(ctx, &flag, cap));
  PHFEM_CUDA(ctx, cudaMemsetAsync(keys, 0xff, sizeof(unsigned long long) * cap, ctx->stream));
  PHFEM_CUDA(ctx, cudaMemsetAsync(flag, 0, sizeof(uint32_t) * cap, ctx->stream));
  if (m->nD)
    PHFEM_LAUNCH(ctx, "k_pair_insert", k_pair_insert<<<grid_for(m->nD, 256, ctx->num_sms), 256, 0, ctx->stream>>>(
        m->dirichlet, m->nD, cap, keys));
  if (m->nN)
    PHFEM_LAUNCH(ctx, "k_pair_insert", k_pair_insert<<<grid_for(m->nN, 256, ctx->num_sms), 256, 0, ctx->stream>>>(
        m->neumann, m->nN, cap, keys));
  PHFEM_LAUNCH(ctx, "k_pair_mark", k_pair_mark<<<grid_for(m->nE, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
      m->elements, m->nE, cap, keys, flag));
  if (m->nD)
    PHFEM_LAUNCH(ctx, "k_pair_apply", k_pair_apply<<<grid_for(m->nD, 256, ctx->num_sms), 256, 0, ctx->stream>>>(
        m->dirichlet, m->nD, cap, keys, flag));
  if (m->nN)
    PHFEM_LAUNCH(ctx, "k_pair_apply", k_pair_apply<<<grid_for(m->nN, 256, ctx->num_sms), 256, 0, ctx->stream>>>(
        m->neumann, m->nN, cap, keys, flag));
  dfree(ctx, keys);
  dfree(ctx, flag);
  return PHFEM_OK;
}

static phfem_status load_text(phfem_ctx* ctx, const char* c, size_t nc, const char* e, size_t ne,
                              const char* dir, size_t nd, const char* neu, size_t nn, phfem_mesh* out) {
  memset(out, 0, sizeof(*out));
  std::vector<double> xy;
  PHFEM_TRY(parse_coords(ctx, c, nc, xy));
  if (xy.size() / 2 >= (size_t(1) << 31))
    return set_error(ctx, PHFEM_ERR_INVALID_ARGUMENT, "coordinates: too many nodes for int ids");
  phfem_mesh m;
  memset(&m, 0, sizeof m);
  m.owned = 1;
  m.nC = (int32_t)(xy.size() / 2);
  PHFEM_TRY(dalloc(ctx, &m.coords, std::max<size_t>(xy.size(), 2)));
  if (!xy.empty())
    PHFEM_CUDA(ctx, cudaMemcpyAsync(m.coords, xy.data(), sizeof(double) * xy.size(), cudaMemcpyHostToDevice,
                                    ctx->stream));
  phfem_status st = parse_index_file<3>(ctx, "elements", e, ne, m.nC, (const double2*)m.coords, &m.elements, &m.nE);
  if (st == PHFEM_OK) st = parse_index_file<2>(ctx, "dirichlet", dir, nd, m.nC, nullptr, &m.dirichlet, &m.nD);
  if (st == PHFEM_OK) st = parse_index_file<2>(ctx, "neumann", neu, nn, m.nC, nullptr, &m.neumann, &m.nN);
  if (st == PHFEM_OK) st = normalize_pairs(ctx, &m);
  if (st != PHFEM_OK) {
    phfem_mesh_release(ctx, &m);
    return st;
  }
  *out = m;
  return PHFEM_OK;
}

// whole file into malloc'd memory (no zero fill), large files by parallel pread
struct FileBuf {
  char* p = nullptr;
  size_t n = 0;
  ~FileBuf() { free(p); }
};

static bool read_file(const std::string& path, FileBuf* b) {
  const int fd = open(path.c_str(), O_RDONLY);
  if (fd < 0) return false;
  struct stat st;
  if (fstat(fd, &st) != 0) {
    close(fd);
    return false;
  }
  const size_t sz = (size_t)st.st_size;
  b->p = (char*)malloc(sz ? sz : 1);
  if (!b->p) {
    close(fd);
    return false;
  }
  const int T = sz < (size_t(64) << 20) ? 1 : std::min(8, io_threads());
  std::vector<size_t> got((size_t)T, 0);
  parallel_for(T, [&](int t) {
    size_t a = sz * t / T;
    const size_t e = sz * (t + 1) / T;
    while (a < e) {
      const ssize_t r = pread(fd, b->p + a, e - a, (off_t)a);
      if (r <= 0) break;
      a += (size_t)r;
      got[t] += (size_t)r;
    }
  });
  close(fd);
  size_t total = 0;
  for (size_t g : got) total += g;
  b->n = total;  // (a short read ends the text there, like the stream would)
  return true;
}

// ---- formatting --------------------------------------------------------------
// Device -> pageable host copy of a large buffer: through a cached pinned
// ring (2 x 32 MB per ctx and thread), the host threads copying chunk i - 1
// out (first touch of the destination pages included) while the copy engine
// brings chunk i — a plain pageable copy into fresh memory ran at ~2 GB/s.
static phfem_status d2h_large(phfem_ctx* ctx, char* dst, const char* src, size_t bytes) {
  constexpr size_t kCh = size_t(32) << 20;
  if (bytes <= kCh) {
    PHFEM_CUDA(ctx, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return PHFEM_OK;
  }
  struct Ring {
    phfem_ctx* ctx;
    char* buf;
    cudaEvent_t ev[2];
  };
  static thread_local std::vector<Ring> rings;
  Ring* r = nullptr;
  for (auto& x : rings)
    if (x.ctx == ctx) r = &x;
  if (!r) {
    Ring x{ctx, nullptr, {nullptr, nullptr}};
    PHFEM_CUDA(ctx, cudaHostAlloc((void**)&x.buf, 2 * kCh, cudaHostAllocDefault));
    for (auto& e : x.ev) PHFEM_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    rings.push_back(x);
    r = &rings.back();
  }
  const size_t nch = (bytes + kCh - 1) / kCh;
  const int T = std::min(8, io_threads());
  auto drain = [&](size_t i) -> phfem_status {
    PHFEM_CUDA(ctx, cudaEventSynchronize(r->ev[i & 1]));
    const size_t off = i * kCh, n = std::min(kCh, bytes - off);
    const char* slot = r->buf + (i & 1) * kCh;
    parallel_for(T, [&](int t) {
      const size_t a = n * t / T, b = n * (t + 1) / T;
      memcpy(dst + off + a, slot + a, b - a);
    });
    return PHFEM_OK;
  };
  for (size_t i = 0; i < nch; ++i) {
    const size_t off = i * kCh, n = std::min(kCh, bytes - off);
    PHFEM_CUDA(ctx, cudaMemcpyAsync(r->buf + (i & 1) * kCh, src + off, n, cudaMemcpyDeviceToHost, ctx->stream));
    PHFEM_CUDA(ctx, cudaEventRecord(r->ev[i & 1], ctx->stream));
    if (i > 0) PHFEM_TRY(drain(i - 1));  // (slot (i+1)&1 is free once chunk i-1 is out)
  }
  return drain(nch - 1);
}

// Text: one malloc'd buffer (handed to the caller as is by the *_format /
// *_csv entry points; free with phfem_text_free), the optional header first.
struct Text {
  std::string head;
  char* buf = nullptr;
  size_t n = 0;
  Text() = default;
  Text(const Text&) = delete;
  Text& operator=(const Text&) = delete;
  ~Text() { free(buf); }
  char* release() {
    char* p = buf;
    buf = nullptr;
    return p;
  }
};

// Exclusive scan of the int64 line lengths (text offsets pass 2^31 bytes at
// L12): tile sums, a one-CTA scan of them, downsweep -- the shape of
// scan_exclusive_i32 (ctx.cu) over 64-bit values.
constexpr int kScan64Threads = 1024;
constexpr int kScan64Per = 4;
constexpr int kScan64Tile = kScan64Threads * kScan64Per;

__global__ void __launch_bounds__(kScan64Threads) k_scan64_tile_sums(const int64_t* __restrict__ in, int64_t n,
                                                                     int64_t* __restrict__ sums) {
  __shared__ int64_t sm[33];
  const int64_t base = (int64_t)blockIdx.x * kScan64Tile;
  int64_t v = 0;
#pragma unroll
  for (int k = 0; k < kScan64Per; ++k) {
    const int64_t i = base + (int64_t)k * kScan64Threads + threadIdx.x;
    if (i < n) v += in[i];
  }
  int64_t tot;
  block_exclusive_scan(v, sm, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScan64Threads) k_scan64_sums(int64_t* sums, int64_t n) {
  __shared__ int64_t sm[33];
  int64_t carry = 0;
  for (int64_t base = 0; base < n; base += kScan64Threads) {
    const int64_t i = base + threadIdx.x;
    const int64_t v = i < n ? sums[i] : 0;
    int64_t tot;
    const int64_t ex = block_exclusive_scan(v, sm, &tot);
    if (i < n) sums[i] = carry + ex;
    carry += tot;
  }
}

__global__ void __launch_bounds__(kScan64Threads) k_scan64_down(const int64_t* __restrict__ in,
                                                                int64_t* __restrict__ out, int64_t n,
                                                                const int64_t* __restrict__ sums) {
  __shared__ int64_t sm[33];
  const int64_t base = (int64_t)blockIdx.x * kScan64Tile + (int64_t)threadIdx.x * kScan64Per;
  int64_t v[kScan64Per];
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScan64Per; ++k) {
    const int64_t i = base + k;
    v[k] = i < n ? in[i] : 0;
    s += v[k];
  }
  int64_t tot;
  int64_t ex = block_exclusive_scan(s, sm, &tot) + sums[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScan64Per; ++k) {
    const int64_t i = base + k;
    if (i < n) out[i] = ex;
    ex += v[k];
  }
}

static phfem_status scan_exclusive_i64(phfem_ctx* ctx, const int64_t* in, int64_t* out, int64_t n) {
  if (n <= 0) return PHFEM_OK;
  const int64_t tiles = (n + kScan64Tile - 1) / kScan64Tile;
  int64_t* sums = nullptr;
  PHFEM_TRY(dalloc(ctx, &sums, tiles));
  k_scan64_tile_sums<<<(unsigned)tiles, kScan64Threads, 0, ctx->stream>>>(in, n, sums);
  PHFEM_CHECK_LAUNCH(ctx);
  k_scan64_sums<<<1, kScan64Threads, 0, ctx->stream>>>(sums, tiles);
  PHFEM_CHECK_LAUNCH(ctx);
  k_scan64_down<<<(unsigned)tiles, kScan64Threads, 0, ctx->stream>>>(in, out, n, sums);
  PHFEM_CHECK_LAUNCH(ctx);
  dfree(ctx, sums);
  return PHFEM_OK;
}

// Device text: line lengths (int64), one 64-bit scan, the bytes, one D2H.
template <class LenFn, class WriteFn>
static phfem_status device_text(phfem_ctx* ctx, int64_t rows, LenFn launch_len, WriteFn launch_write, Text* out) {
  free(out->buf);
  out->buf = nullptr;
  out->n = 0;
  const size_t hn = out->head.size();
  int64_t total = 0;
  char* d = nullptr;
  int64_t* len = nullptr;
  int64_t* off = nullptr;
  if (rows > 0) {
    PHFEM_TRY(dalloc(ctx, &len, rows + 1));
    PHFEM_TRY(dalloc(ctx, &off, rows + 1));
    PHFEM_TRY(launch_len(len));
    PHFEM_CUDA(ctx, cudaMemsetAsync(len + rows, 0, sizeof(int64_t), ctx->stream));
    PHFEM_TRY(scan_exclusive_i64(ctx, len, off, rows + 1));
    PHFEM_CUDA(ctx, cudaMemcpyAsync(&total, off + rows, sizeof total, cudaMemcpyDeviceToHost, ctx->stream));
    PHFEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    PHFEM_TRY(dalloc(ctx, &d, std::max<int64_t>(total, 1)));
    PHFEM_TRY(launch_write(off, d));
  }
  out->buf = (char*)malloc(hn + (size_t)total + 1);
  if (!out->buf) return set_error(ctx, PHFEM_ERR_OOM, "out of host memory (%zu bytes)", hn + (size_t)total);
  memcpy(out->buf, out->head.data(), hn);
  out->n = hn + (size_t)total;
  if (total > 0) PHFEM_TRY(d2h_large(ctx, out->buf + hn, d, (size_t)total));
  dfree(ctx, d);
  dfree(ctx, len);
  dfree(ctx, off);
  return PHFEM_OK;
}

template <int K>
static phfem_status format_index_rows(phfem_ctx* ctx, const int32_t* ids, int64_t rows, Text* out) {
  const int g = grid_for(rows, 256, ctx->num_sms * 8);
  return device_text(
      ctx, rows,
      [&](int64_t* len) -> phfem_status {
        PHFEM_LAUNCH(ctx, "k_fmt_len", k_fmt_len<K><<<g, 256, 0, ctx->stream>>>(ids, rows, len));
        return PHFEM_OK;
      },
      [&](const int64_t* off, char* d) -> phfem_status {
        PHFEM_LAUNCH(ctx, "k_fmt_write", k_fmt_write<K><<<g, 256, 0, ctx->stream>>>(ids, rows, off, d));
        return PHFEM_OK;
      },
      out);
}

static phfem_status mesh_text(phfem_ctx* ctx, const phfem_mesh* m, int which, Text* out) {
  switch (which) {
    case 0: {  // format_g17 (mesh.cpp:95-99) on the device (fmt.cuh, exact)
      const int64_t rows = m->nC;
      const int g = grid_for(rows, 256, ctx->num_sms * 8);
      return device_text(
          ctx, rows,
          [&](int64_t* len) -> phfem_status {
            PHFEM_LAUNCH(ctx, "k_fmt_coords_len", k_fmt_coords_len<<<g, 256, 0, ctx->stream>>>(m->coords, rows, len));
            return PHFEM_OK;
          },
          [&](const int64_t* off, char* d) -> phfem_status {
            PHFEM_LAUNCH(ctx, "k_fmt_coords_write", k_fmt_coords_write<<<g, 256, 0, ctx->stream>>>(m->coords, rows,
                                                                                              off, d));
            return PHFEM_OK;
          },
          out);
    }
    case 1: return format_index_rows<3>(ctx, m->elements, m->nE, out);
    case 2: return format_index_rows<2>(ctx, m->dirichlet, m->nD, out);
    case 3: return format_index_rows<2>(ctx, m->neumann, m->nN, out);
    default: return PHFEM_ERR_INVALID_ARGUMENT;
  }
}

// tools/main.cpp:302-323 (cmd_topology): header + one row per edge on the
// device (lengths as edge_lengths computes them, "%.10g" exact)
static phfem_status topology_csv(phfem_ctx* ctx, const phfem_mesh* m, const phfem_topology* t, Text* out) {
  const int64_t E = t->E;
  const int g = grid_for(E, 256, ctx->num_sms * 8);
  const double2* c = (const double2*)m->coords;
  out->head = "edge,node_start,node_end,t_plus,t_minus,led,led_tn,length\n";
  PHFEM_TRY(device_text(
      ctx, E,
      [&](int64_t* len) -> phfem_status {
        PHFEM_LAUNCH(ctx, "k_fmt_csv", (k_fmt_csv<false><<<g, 256, 0, ctx->stream>>>(
            t->edge_nodes, t->edge_elements, t->local_in_tplus, t->local_in_tminus, c, E, len, nullptr)));
        return PHFEM_OK;
      },
      [&](const int64_t* off, char* d) -> phfem_status {
        PHFEM_LAUNCH(ctx, "k_fmt_csv", (k_fmt_csv<true><<<g, 256, 0, ctx->stream>>>(
            t->edge_nodes, t->edge_elements, t->local_in_tplus, t->local_in_tminus, c, E,
            const_cast<int64_t*>(off), d)));
        return PHFEM_OK;
      },
      out));
  return PHFEM_OK;
}

static phfem_status to_buffer(phfem_ctx* ctx, Text& t, char** out, size_t* len) {
  (void)ctx;
  *len = t.n;
  *out = t.release();
  return PHFEM_OK;
}

static phfem_status write_file(phfem_ctx* ctx, const std::string& path, const Text& t) {
  FILE* f = fopen(path.c_str(), "wb");
  if (!f) return set_error(ctx, PHFEM_ERR_RUNTIME, "cannot write %s", path.c_str());
  bool ok = t.n == 0 || fwrite(t.buf, 1, t.n, f) == t.n;
  ok = (fclose(f) == 0) && ok;
  if (!ok) return set_error(ctx, PHFEM_ERR_RUNTIME, "cannot write %s", path.c_str());
  return PHFEM_OK;
}

}  // namespace phfem

using namespace phfem;

PHFEM_API phfem_status phfem_mesh_load_text(phfem_ctx* ctx, const char* coordinates, size_t coordinates_len,
                                            const char* elements, size_t elements_len, const char* dirichlet,
                                            size_t dirichlet_len, const char* neumann, size_t neumann_len,
                                            phfem_mesh* out) {
  if (!ctx || !out || (coordinates_len && !coordinates) || (elements_len && !elements) ||
      (dirichlet_len && !dirichlet) || (neumann_len && !neumann))
    return PHFEM_ERR_INVALID_ARGUMENT;
  return load_text(ctx, coordinates, coordinates_len, elements, elements_len, dirichlet, dirichlet_len, neumann,
                   neumann_len, out);
}

PHFEM_API phfem_status phfem_mesh_load_dir(phfem_ctx* ctx, const char* dir, phfem_mesh* out) {
  if (!ctx || !dir || !out) return PHFEM_ERR_INVALID_ARGUMENT;
  memset(out, 0, sizeof(*out));
  const std::string d(dir);
  FileBuf c, e, di, ne;
  if (!read_file(d + "/coordinates.dat", &c))
    return set_error(ctx, PHFEM_ERR_RUNTIME, "cannot open %s/coordinates.dat", dir);
  if (!read_file(d + "/elements.dat", &e)) return set_error(ctx, PHFEM_ERR_RUNTIME, "cannot open %s/elements.dat", dir);
  read_file(d + "/dirichlet.dat", &di);  // optional (mesh.cpp:162-163)
  read_file(d + "/neumann.dat", &ne);
  return load_text(ctx, c.p, c.n, e.p, e.n, di.p, di.n, ne.p, ne.n, out);
}

PHFEM_API phfem_status phfem_mesh_format(phfem_ctx* ctx, const phfem_mesh* mesh, int which, char** out,
                                         size_t* len) {
  if (!ctx || !mesh || !out || !len || which < 0 || which > 3) return PHFEM_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  Text s;
  PHFEM_TRY(mesh_text(ctx, mesh, which, &s));
  return to_buffer(ctx, s, out, len);
}

PHFEM_API void phfem_text_free(char* p) { free(p); }

PHFEM_API phfem_status phfem_mesh_save_dir(phfem_ctx* ctx, const phfem_mesh* mesh, const char* dir) {
  if (!ctx || !mesh || !dir) return PHFEM_ERR_INVALID_ARGUMENT;
  static const char* names[4] = {"coordinates.dat", "elements.dat", "dirichlet.dat", "neumann.dat"};
  // save_mesh_dir opens all four files before writing any (mesh.cpp:182-191)
  for (int w = 0; w < 4; ++w) {
    const std::string path = std::string(dir) + "/" + names[w];
    FILE* f = fopen(path.c_str(), "wb");
    if (!f) return set_error(ctx, PHFEM_ERR_RUNTIME, "cannot write %s", path.c_str());
    fclose(f);
  }
  for (int w = 0; w < 4; ++w) {
    Text s;
    PHFEM_TRY(mesh_text(ctx, mesh, w, &s));
    PHFEM_TRY(write_file(ctx, std::string(dir) + "/" + names[w], s));
  }
  return PHFEM_OK;
}

PHFEM_API phfem_status phfem_topology_csv(phfem_ctx* ctx, const phfem_mesh* mesh, const phfem_topology* topo,
                                          char** out, size_t* len) {
  if (!ctx || !mesh || !topo || !out || !len) return PHFEM_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  Text s;
  PHFEM_TRY(topology_csv(ctx, mesh, topo, &s));
  return to_buffer(ctx, s, out, len);
}

PHFEM_API phfem_status phfem_topology_csv_file(phfem_ctx* ctx, const phfem_mesh* mesh, const phfem_topology* topo,
                                               const char* path) {
  if (!ctx || !mesh || !topo || !path) return PHFEM_ERR_INVALID_ARGUMENT;
  Text s;
  PHFEM_TRY(topology_csv(ctx, mesh, topo, &s));
  return write_file(ctx, path, s);
}

// test entry: "%.<precision>g" of n device doubles into 32-byte slots (device)
PHFEM_API phfem_status phfem_format_g(phfem_ctx* ctx, const double* vals, int64_t n, int precision, char* out,
                                      int32_t* lens) {
  if (!ctx || precision < 1 || precision > 17 || (n > 0 && (!vals || !out || !lens)))
    return PHFEM_ERR_INVALID_ARGUMENT;
  if (n > 0)
    PHFEM_LAUNCH(ctx, "k_fmt_g_test", k_fmt_g_test<<<grid_for(n, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
        vals, n, precision, out, lens));
  return PHFEM_OK;
}

// the same formatter on the host (no device needed): the CPU tests pin it to
// glibc's printf over millions of doubles; the kernels run this very code
PHFEM_API int phfem_format_g_host(double v, int precision, char* out) {
  if (precision < 1 || precision > 17 || !out) return -1;
  return fmt_g(v, precision, out);
}
