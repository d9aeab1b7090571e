// TEST INFRASTRUCTURE ONLY -- part of the CPU oracle (see oracle/README.md).
// Never linked into the product library.
//
// Exact big-integer arithmetic used by the oracle's exact predicate
// fallbacks.  It restates the reference's exact path
// (/root/reference/pkg/src/tetrefine/predicates.py:45-126): every double is
// scaled to an integer over a common power of two (frexp mantissa * 2^53,
// shifted by its exponent above the minimum exponent) and determinants are
// evaluated in unbounded integer arithmetic.  Rational constructions
// (geometry.py:74-98 circumsphere fallback, geometry.py:168-194 equatorial
// comparison, plc.py point-in-polygon) use the same integers.
#pragma once
#include <cstdint>
#include <cmath>
#include <vector>
#include <algorithm>
#include <limits>

namespace orc {

struct BigInt {
  int sign = 0;                  // -1, 0, +1
  std::vector<uint32_t> mag;     // little-endian magnitude, no leading zeros

  BigInt() {}
  explicit BigInt(int64_t v) {
    if (v == 0) return;
    sign = v < 0 ? -1 : 1;
    uint64_t m = v < 0 ? (uint64_t)(-(v + 1)) + 1u : (uint64_t)v;
    while (m) { mag.push_back((uint32_t)m); m >>= 32; }
  }
  void trim() {
    while (!mag.empty() && mag.back() == 0) mag.pop_back();
    if (mag.empty()) sign = 0;
  }
  bool is_zero() const { return sign == 0; }
};

inline int cmp_mag(const std::vector<uint32_t>& a, const std::vector<uint32_t>& b) {
  if (a.size() != b.size()) return a.size() < b.size() ? -1 : 1;
  for (size_t i = a.size(); i-- > 0;) {
    if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
  }
  return 0;
}

inline std::vector<uint32_t> add_mag(const std::vector<uint32_t>& a, const std::vector<uint32_t>& b) {
  std::vector<uint32_t> r(std::max(a.size(), b.size()) + 1, 0);
  uint64_t c = 0;
  for (size_t i = 0; i < r.size(); ++i) {
    uint64_t s = c;
    if (i < a.size()) s += a[i];
    if (i < b.size()) s += b[i];
    r[i] = (uint32_t)s;
    c = s >> 32;
  }
  while (!r.empty() && r.back() == 0) r.pop_back();
  return r;
}

// a - b with |a| >= |b|
inline std::vector<uint32_t> sub_mag(const std::vector<uint32_t>& a, const std::vector<uint32_t>& b) {
  std::vector<uint32_t> r(a.size(), 0);
  int64_t br = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    int64_t s = (int64_t)a[i] - br - (i < b.size() ? (int64_t)b[i] : 0);
    if (s < 0) { s += ((int64_t)1 << 32); br = 1; } else br = 0;
    r[i] = (uint32_t)s;
  }
  while (!r.empty() && r.back() == 0) r.pop_back();
  return r;
}

inline BigInt operator-(const BigInt& a) { BigInt r = a; r.sign = -r.sign; return r; }

inline BigInt operator+(const BigInt& a, const BigInt& b) {
  if (a.sign == 0) return b;
  if (b.sign == 0) return a;
  BigInt r;
  if (a.sign == b.sign) {
    r.mag = add_mag(a.mag, b.mag);
    r.sign = a.sign;
  } else {
    int c = cmp_mag(a.mag, b.mag);
    if (c == 0) return BigInt();
    if (c > 0) { r.mag = sub_mag(a.mag, b.mag); r.sign = a.sign; }
    else { r.mag = sub_mag(b.mag, a.mag); r.sign = b.sign; }
  }
  r.trim();
  return r;
}
inline BigInt operator-(const BigInt& a, const BigInt& b) { return a + (-b); }

inline BigInt operator*(const BigInt& a, const BigInt& b) {
  BigInt r;
  if (a.sign == 0 || b.sign == 0) return r;
  r.mag.assign(a.mag.size() + b.mag.size(), 0);
  for (size_t i = 0; i < a.mag.size(); ++i) {
    uint64_t c = 0;
    for (size_t j = 0; j < b.mag.size(); ++j) {
      uint64_t t = (uint64_t)a.mag[i] * b.mag[j] + r.mag[i + j] + c;
      r.mag[i + j] = (uint32_t)t;
      c = t >> 32;
    }
    size_t k = i + b.mag.size();
    while (c) {
      uint64_t t = (uint64_t)r.mag[k] + c;
      r.mag[k] = (uint32_t)t;
      c = t >> 32;
      ++k;
    }
  }
  r.sign = a.sign * b.sign;
  r.trim();
  return r;
}

inline BigInt shl(const BigInt& a, int64_t bits) {
  if (a.sign == 0 || bits == 0) return a;
  BigInt r;
  size_t words = (size_t)(bits / 32);
  int rem = (int)(bits % 32);
  r.mag.assign(words, 0);
  uint32_t carry = 0;
  for (size_t i = 0; i < a.mag.size(); ++i) {
    uint64_t v = ((uint64_t)a.mag[i] << rem) | carry;
    r.mag.push_back((uint32_t)v);
    carry = rem ? (uint32_t)(v >> 32) : 0;
  }
  if (carry) r.mag.push_back(carry);
  r.sign = a.sign;
  r.trim();
  return r;
}

inline int cmp(const BigInt& a, const BigInt& b) {
  BigInt d = a - b;
  return d.sign;
}

inline int64_t bitlen(const BigInt& a) {
  if (a.sign == 0) return 0;
  uint32_t top = a.mag.back();
  int b = 0;
  while (top) { ++b; top >>= 1; }
  return (int64_t)(a.mag.size() - 1) * 32 + b;
}

inline bool test_bit(const BigInt& a, int64_t i) {
  size_t w = (size_t)(i / 32);
  if (w >= a.mag.size()) return false;
  return (a.mag[w] >> (i % 32)) & 1u;
}

// scaled integers: x_i = m_i * 2^(e_i - emin) where frexp(x_i) = (m_i/2^53, e_i)
// (predicates.py:55-63)
inline void scaled_ints(const double* xs, int n, BigInt* out) {
  int es[64];
  int64_t ms[64];
  int emin = std::numeric_limits<int>::max();
  for (int i = 0; i < n; ++i) {
    int e;
    double m = std::frexp(xs[i], &e);
    ms[i] = (int64_t)(m * 9007199254740992.0);  // exact: m has <= 53 bits
    es[i] = e;
    emin = std::min(emin, e);
  }
  for (int i = 0; i < n; ++i) out[i] = shl(BigInt(ms[i]), es[i] - emin);
}
// same, also returning the common scale exponent: x_i = out_i * 2^(emin-53)
inline int scaled_ints_exp(const double* xs, int n, BigInt* out) {
  int emin = std::numeric_limits<int>::max();
  for (int i = 0; i < n; ++i) { int e; std::frexp(xs[i], &e); emin = std::min(emin, e); }
  scaled_ints(xs, n, out);
  return emin - 53;
}

// Correctly rounded (round-half-even) conversion of num/den * 2^exp2 to
// double, as Python's float(Fraction) does.  Returns +-inf on overflow.
inline double rat_to_double(const BigInt& num, const BigInt& den, int64_t exp2) {
  if (num.sign == 0) return 0.0;
  int sgn = num.sign * den.sign;
  BigInt n = num; n.sign = 1;
  BigInt d = den; d.sign = 1;
  // choose k so that q = floor(n*2^k/d) has at least 55 bits
  int64_t k = 56 - (bitlen(n) - bitlen(d));
  BigInt nn = k >= 0 ? shl(n, k) : n;
  BigInt dd = k >= 0 ? d : shl(d, -k);
  // binary long division: q = floor(nn/dd), rem sticky
  int64_t qbits = bitlen(nn) - bitlen(dd) + 1;
  uint64_t q = 0;
  BigInt r = nn;
  for (int64_t i = qbits - 1; i >= 0; --i) {
    BigInt t = shl(dd, i);
    q <<= 1;
    if (cmp(r, t) >= 0) { r = r - t; q |= 1; }
  }
  bool sticky = r.sign != 0;
  // value = q * 2^(exp2 - k) (+ sticky), q in [2^55, 2^58)
  int64_t e = exp2 - k;
  // normalise q to exactly 55..57 bits; compute unbiased exponent of msb
  int qb = 0;
  { uint64_t t = q; while (t) { ++qb; t >>= 1; } }
  int64_t msb_exp = e + qb - 1;     // value in [2^msb_exp, 2^(msb_exp+1))
  if (msb_exp > 1023) return sgn * std::numeric_limits<double>::infinity();
  // number of mantissa bits available (subnormals below 2^-1022)
  int64_t lsb_exp = std::max<int64_t>(msb_exp - 52, -1074);
  int64_t drop = lsb_exp - e;      // bits of q to drop
  uint64_t mant;
  if (drop <= 0) {
    mant = q << (-drop);
  } else if (drop >= 64) {
    mant = 0;
    // everything dropped: round to 0 or to the smallest subnormal
    bool half_or_more = (drop == 64) ? ((q >> 63) & 1) : false;
    (void)half_or_more;
    return sgn * 0.0;
  } else {
    uint64_t kept = q >> drop;
    uint64_t rest = q & ((drop == 64) ? ~0ull : ((1ull << drop) - 1));
    uint64_t half = 1ull << (drop - 1);
    bool round_up = false;
    if (rest > half) round_up = true;
    else if (rest == half) round_up = sticky ? true : (kept & 1);
    else round_up = false;
    mant = kept + (round_up ? 1 : 0);
  }
  double v = std::ldexp((double)mant, (int)lsb_exp);
  return sgn * v;
}

}  // namespace orc
