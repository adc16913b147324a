// fmt.cuh — printf("%.<P>g") of fp64 on the device, exact (P <= 17): the
// same bytes as glibc for every double (round-half-even on the exact binary
// value; infinities / NaNs as "inf" / "nan" with their sign).
//
// Digits: D = round(|v| * 10^(P-1-X)) with v = m 2^e.  For the common
// exponent range the product m * 5^p fits 128 bits (p <= 27), or, for large
// values, m 2^e fits 128 bits and 10^q one 64-bit word — both exact with one
// 128-bit shift / division.  Everything else (|v| below ~1e-11 or above
// ~1e22 at P = 17) takes a small 32-bit-limb big integer: m * 5^p shifted
// right with a sticky bit, or m 2^e divided by 10^q in 10^9 steps — exact
// too, only slower.
#pragma once

#include <math.h>
#include <stdint.h>
#include <string.h>

// host and device: the same code formats on the GPU and in the CPU tests
#define PHFEM_FMT_HD __host__ __device__ __forceinline__

namespace phfem {

PHFEM_FMT_HD uint64_t pow10_u64(int k) {  // k <= 19
  uint64_t r = 1;
  for (int i = 0; i < k; ++i) r *= 10;
  return r;
}

PHFEM_FMT_HD uint64_t pow5_u64(int k) {  // k <= 27
  uint64_t r = 1;
  for (int i = 0; i < k; ++i) r *= 5;
  return r;
}

// round-half-even of N / 2^s (N exact, 128 bits, 0 < s < 128)
PHFEM_FMT_HD unsigned __int128 shr_rne(unsigned __int128 N, int s) {
  const unsigned __int128 q = N >> s;
  const unsigned __int128 rem = N - (q << s);
  const unsigned __int128 half = (unsigned __int128)1 << (s - 1);
  return (rem > half || (rem == half && (q & 1))) ? q + 1 : q;
}

// Big integer fallback: little-endian 32-bit limbs.
struct FmtBig {
  uint32_t w[40];  // m 2^e < 2^1077; m 5^p (p <= 342) < 2^850
  int n;
};

PHFEM_FMT_HD void big_set_u64(FmtBig& b, uint64_t v) {
  b.w[0] = (uint32_t)v;
  b.w[1] = (uint32_t)(v >> 32);
  b.n = b.w[1] ? 2 : (b.w[0] ? 1 : 0);
}

PHFEM_FMT_HD void big_mul_u32(FmtBig& b, uint32_t k) {
  uint64_t c = 0;
  for (int i = 0; i < b.n; ++i) {
    const uint64_t t = (uint64_t)b.w[i] * k + c;
    b.w[i] = (uint32_t)t;
    c = t >> 32;
  }
  if (c) b.w[b.n++] = (uint32_t)c;
}

PHFEM_FMT_HD void big_shl(FmtBig& b, int s) {
  const int ws = s >> 5, bs = s & 31;
  if (bs) {
    uint32_t c = 0;
    for (int i = 0; i < b.n; ++i) {
      const uint32_t x = b.w[i];
      b.w[i] = (x << bs) | c;
      c = x >> (32 - bs);
    }
    if (c) b.w[b.n++] = c;
  }
  if (ws) {
    for (int i = b.n - 1; i >= 0; --i) b.w[i + ws] = b.w[i];
    for (int i = 0; i < ws; ++i) b.w[i] = 0;
    b.n += ws;
  }
}

// b /= k, returns the remainder
PHFEM_FMT_HD uint32_t big_div_u32(FmtBig& b, uint32_t k) {
  uint64_t r = 0;
  for (int i = b.n - 1; i >= 0; --i) {
    const uint64_t t = (r << 32) | b.w[i];
    b.w[i] = (uint32_t)(t / k);
    r = t % k;
  }
  while (b.n > 0 && b.w[b.n - 1] == 0) --b.n;
  return (uint32_t)r;
}

PHFEM_FMT_HD uint64_t big_u64(const FmtBig& b) {
  return (b.n > 0 ? b.w[0] : 0) | ((uint64_t)(b.n > 1 ? b.w[1] : 0) << 32);
}

// bit i of b (0 beyond the top)
PHFEM_FMT_HD uint32_t big_bit(const FmtBig& b, int i) {
  return (i >> 5) < b.n ? (b.w[i >> 5] >> (i & 31)) & 1u : 0u;
}

// D = round-half-even(m 2^e 10^p), exact; D < 10^18 expected by the caller
PHFEM_FMT_HD uint64_t fmt_scaled(uint64_t m, int e, int p) {
  if (p >= 0) {
    const int s = e + p;  // m 5^p 2^s
    if (p <= 27 && s > -128 && s <= 8) {
      const unsigned __int128 N = (unsigned __int128)m * pow5_u64(p);  // < 2^117
      if (s >= 0) return (uint64_t)(N << s);
      return (uint64_t)shr_rne(N, -s);
    }
    FmtBig b;
    big_set_u64(b, m);
    for (int k = p; k > 0; k -= 13) big_mul_u32(b, (uint32_t)pow5_u64(k < 13 ? k : 13));
    if (s >= 0) {
      big_shl(b, s);
      return big_u64(b);
    }
    const int sh = -s, hb = sh - 1;  // quotient from bit sh, half bit hb, sticky below it
    const bool half = big_bit(b, hb);
    bool sticky = false;
    for (int i = 0; i < (hb >> 5) && i < b.n; ++i) sticky |= b.w[i] != 0;
    if ((hb & 31) && (hb >> 5) < b.n) sticky |= (b.w[hb >> 5] & ((1u << (hb & 31)) - 1u)) != 0;
    uint64_t q = 0;
    for (int i = 0; i < 64; ++i) q |= (uint64_t)big_bit(b, sh + i) << i;
    return (half && (sticky || (q & 1))) ? q + 1 : q;
  }
  // p < 0: m 2^e / 10^q, q = -p.  With e < 0, m 2^e = m 5^-e / 10^-e: the
  // numerator N = m 5^-e over 10^(q - e); otherwise N = m 2^e over 10^q.
  const int q = -p;
  const int k10 = e < 0 ? q - e : q;  // decimal exponent of the denominator
  if ((e >= 0 && e <= 74 && q <= 19) || (e < 0 && -e <= 27 && k10 <= 38)) {
    const unsigned __int128 N =
        e >= 0 ? (unsigned __int128)m << e : (unsigned __int128)m * pow5_u64(-e);
    unsigned __int128 d = 1;
    for (int i = 0; i < k10; ++i) d *= 10;
    const unsigned __int128 Q = N / d;
    const unsigned __int128 twice = (N - Q * d) * 2;
    return (uint64_t)((twice > d || (twice == d && (Q & 1))) ? Q + 1 : Q);
  }
  FmtBig b;
  big_set_u64(b, m);
  if (e > 0) big_shl(b, e);
  if (e < 0)
    for (int k = -e; k > 0; k -= 13) big_mul_u32(b, (uint32_t)pow5_u64(k < 13 ? k : 13));
  // divide by 10^(k10-1) noting any nonzero remainder, then the last digit decides
  bool sticky = false;
  int k = k10 - 1;
  while (k >= 9) {
    sticky |= big_div_u32(b, 1000000000u) != 0;
    k -= 9;
  }
  if (k > 0) sticky |= big_div_u32(b, (uint32_t)pow10_u64(k)) != 0;
  const uint32_t last = big_div_u32(b, 10u);
  const uint64_t Q = big_u64(b);
  return (last > 5 || (last == 5 && (sticky || (Q & 1)))) ? Q + 1 : Q;
}

// printf("%.Pg", v) into out (>= 32 bytes for P <= 17); returns the length
PHFEM_FMT_HD int fmt_g(double v, int P, char* out) {
  int n = 0;
  uint64_t bits;
  memcpy(&bits, &v, sizeof bits);
  const bool neg = bits >> 63;
  const int bexp = (int)((bits >> 52) & 0x7ff);
  uint64_t frac = bits & ((1ull << 52) - 1);
  if (bexp == 0x7ff) {
    if (neg) out[n++] = '-';
    if (frac) { out[n++] = 'n'; out[n++] = 'a'; out[n++] = 'n'; }
    else { out[n++] = 'i'; out[n++] = 'n'; out[n++] = 'f'; }
    return n;
  }
  if (neg) out[n++] = '-';
  if (bexp == 0 && frac == 0) {
    out[n++] = '0';
    return n;
  }
  uint64_t m;
  int e;
  if (bexp == 0) {  // subnormal
    m = frac;
    e = -1074;
  } else {
    m = frac | (1ull << 52);
    e = bexp - 1075;
  }
  // X = floor(log10(|v|)), estimated then corrected against the digits
  const double av = fabs(v);
  int X = (int)floor(log10(av));
  uint64_t D = fmt_scaled(m, e, P - 1 - X);
  const uint64_t lo = pow10_u64(P - 1), hi = pow10_u64(P);
  if (D >= hi) {  // estimate one too small (or rounded up to 10^P)
    ++X;
    D = fmt_scaled(m, e, P - 1 - X);
  } else if (D < lo) {  // estimate one too large
    --X;
    D = fmt_scaled(m, e, P - 1 - X);
  }
  if (D >= hi) {  // rounding carried into a new digit: 10^P -> 10^(P-1)
    D = lo;
    ++X;
  }
  if (D == lo) {  // 10^(P-1) may also be the rounded-up value of the smaller exponent
    const uint64_t D2 = fmt_scaled(m, e, P - X);
    if (D2 < hi) {
      D = D2;
      --X;
    }
  }
  char dig[20];
  for (int i = P - 1; i >= 0; --i) {
    dig[i] = (char)('0' + D % 10);
    D /= 10;
  }
  int nd = P;  // significant digits after removing trailing zeros
  while (nd > 1 && dig[nd - 1] == '0') --nd;
  if (X >= -4 && X < P) {  // style f
    if (X >= 0) {
      for (int i = 0; i <= X; ++i) out[n++] = dig[i];
      if (nd > X + 1) {
        out[n++] = '.';
        for (int i = X + 1; i < nd; ++i) out[n++] = dig[i];
      }
    } else {
      out[n++] = '0';
      out[n++] = '.';
      for (int i = 0; i < -X - 1; ++i) out[n++] = '0';
      for (int i = 0; i < nd; ++i) out[n++] = dig[i];
    }
  } else {  // style e
    out[n++] = dig[0];
    if (nd > 1) {
      out[n++] = '.';
      for (int i = 1; i < nd; ++i) out[n++] = dig[i];
    }
    out[n++] = 'e';
    int x = X;
    out[n++] = x < 0 ? '-' : '+';
    if (x < 0) x = -x;
    if (x >= 100) {
      out[n++] = (char)('0' + x / 100);
      x %= 100;
      out[n++] = (char)('0' + x / 10);
      out[n++] = (char)('0' + x % 10);
    } else {
      out[n++] = (char)('0' + x / 10);
      out[n++] = (char)('0' + x % 10);
    }
  }
  return n;
}

}  // namespace phfem
