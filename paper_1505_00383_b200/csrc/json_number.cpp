// json_number.cpp -- doubles printed exactly as nlohmann::json 3.11 dump() prints them, so that the
// JSON-lines records of pp_solutions_jsonl are byte-identical to the reference CLI's
// (polypath_main.cpp:133-189, which serialises with nlohmann::json).
//
// nlohmann prints a finite double with Grisu2 (F. Loitsch, "Printing floating-point numbers
// quickly and accurately with integers", PLDI 2010): the digits come from a 64-bit approximation
// of v * 10^-k, generated inside the rounding interval of v shrunk by one unit on each side, and
// the last digit is nudged toward v.  The result round-trips but is not always the shortest or
// the closest representation, so std::to_chars cannot stand in for it.  The digits are then laid
// out in fixed notation for decimal exponents in [-4, 15) (with ".0" on integers) and in
// scientific notation with an at least two-digit exponent otherwise; +-0 prints as "0.0" / "-0.0"
// and non-finite values as null.
#include "json_number.hpp"

#include <cmath>
#include <cstdint>
#include <cstring>

namespace pp {
namespace {

// f * 2^e
struct Fp {
  uint64_t f;
  int e;
};

// upper 64 bits of the 128-bit product, rounded half up
Fp fp_mul(Fp a, Fp b) {
  const unsigned __int128 p = static_cast<unsigned __int128>(a.f) * b.f + (static_cast<unsigned __int128>(1) << 63);
  return Fp{static_cast<uint64_t>(p >> 64), a.e + b.e + 64};
}

Fp fp_normalize(Fp x) {
  const int s = __builtin_clzll(x.f);
  return Fp{x.f << s, x.e - s};
}

struct Pow10 {
  uint64_t f;
  int e;
  int k;
};
constexpr Pow10 kPow10[] = {
#include "pow10_table.inc"
};

// digits of a positive finite v into buf; returns the count, *dexp = decimal exponent of the last digit
int grisu2_digits(double v, char* buf, int* dexp) {
  uint64_t bits;
  std::memcpy(&bits, &v, sizeof bits);
  const uint64_t frac = bits & ((uint64_t{1} << 52) - 1), bexp = bits >> 52;
  const Fp w = bexp == 0 ? Fp{frac, -1074} : Fp{frac | (uint64_t{1} << 52), static_cast<int>(bexp) - 1075};
  // rounding interval [m-, m+] of v: the midpoints to its neighbours (the lower one is closer when
  // v is a power of two above the smallest normal)
  const Fp mp = fp_normalize(Fp{2 * w.f + 1, w.e - 1});
  Fp mm = (frac == 0 && bexp > 1) ? Fp{4 * w.f - 1, w.e - 2} : Fp{2 * w.f - 1, w.e - 1};
  mm = Fp{mm.f << (mm.e - mp.e), mp.e};
  const Fp wn = fp_normalize(w);

  // cached power c ~= 10^-k so that the scaled binary exponent lands in [-60, -32]
  const int t = -61 - mp.e;
  const int k = (t * 78913) / (1 << 18) + (t > 0 ? 1 : 0);
  const Pow10& c = kPow10[(300 + k + 7) / 8];
  const Fp cw{c.f, c.e};
  const Fp sv = fp_mul(wn, cw), slo = fp_mul(mm, cw), shi = fp_mul(mp, cw);
  const Fp lo{slo.f + 1, slo.e}, hi{shi.f - 1, shi.e};  // shrunk by one unit: inside the true interval
  *dexp = -c.k;

  const int sh = -hi.e;
  const uint64_t one = uint64_t{1} << sh;
  uint64_t delta = hi.f - lo.f;  // width of the interval
  uint64_t dist = hi.f - sv.f;   // distance from the upper end to v
  uint32_t integral = static_cast<uint32_t>(hi.f >> sh);
  uint64_t fraction = hi.f & (one - 1);
  int len = 0;

  // nudge the last digit down while that moves the value closer to v and stays in the interval
  auto round_toward_v = [&](uint64_t rest, uint64_t unit) {
    while (rest < dist && delta - rest >= unit && (rest + unit < dist || dist - rest > rest + unit - dist)) {
      --buf[len - 1];
      rest += unit;
    }
  };

  uint32_t p10 = 1;
  int n = 1;
  while (n < 10 && integral >= p10 * 10u) {
    p10 *= 10;
    ++n;
  }
  while (n > 0) {
    buf[len++] = static_cast<char>('0' + integral / p10);
    integral %= p10;
    --n;
    const uint64_t rest = (static_cast<uint64_t>(integral) << sh) + fraction;
    if (rest <= delta) {  // enough digits: the rest lies inside the interval
      *dexp += n;
      round_toward_v(rest, static_cast<uint64_t>(p10) << sh);
      return len;
    }
    p10 /= 10;
  }
  int m = 0;
  for (;;) {
    fraction *= 10;
    buf[len++] = static_cast<char>('0' + (fraction >> sh));
    fraction &= one - 1;
    ++m;
    delta *= 10;
    dist *= 10;
    if (fraction <= delta) break;
  }
  *dexp -= m;
  round_toward_v(fraction, one);
  return len;
}

}  // namespace

void json_double(std::string& out, double v) {
  if (!std::isfinite(v)) {
    out += "null";
    return;
  }
  if (std::signbit(v)) {
    out += '-';
    v = -v;
  }
  if (v == 0.0) {
    out += "0.0";
    return;
  }
  char d[32];
  int dexp = 0;
  const int k = grisu2_digits(v, d, &dexp);
  const int n = k + dexp;  // position of the decimal point relative to the first digit
  constexpr int kMinExp = -4, kMaxExp = 15;
  if (k <= n && n <= kMaxExp) {  // integral: digits, zeros, ".0"
    out.append(d, k);
    out.append(static_cast<size_t>(n - k), '0');
    out += ".0";
  } else if (0 < n && n <= kMaxExp) {  // dig.its
    out.append(d, n);
    out += '.';
    out.append(d + n, k - n);
  } else if (kMinExp < n && n <= 0) {  // 0.[000]digits
    out += "0.";
    out.append(static_cast<size_t>(-n), '0');
    out.append(d, k);
  } else {  // d[.igits]e+NN
    out += d[0];
    if (k > 1) {
      out += '.';
      out.append(d + 1, k - 1);
    }
    int e = n - 1;
    out += 'e';
    out += e < 0 ? '-' : '+';
    if (e < 0) e = -e;
    if (e < 10) out += '0';
    out += std::to_string(e);
  }
}

}  // namespace pp
