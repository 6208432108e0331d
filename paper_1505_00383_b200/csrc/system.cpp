// system.cpp -- polynomial systems: text grammar, printing, cyclic-n generator, decimal I/O at
// the three levels, start-solution text, and the gamma constant.
//
// Behaviour (accepted language, merge rules, error positions, and the exact binary64 limbs a
// decimal literal turns into) follows the reference: polysys.cpp:117-252 (parse_system),
// :273-313 (print_system), :315-336 (cyclic_system), :381-425 (parse_solutions),
// xprec_io.cpp:11-193 (decimal I/O), homotopy.cpp:24-40 (random_gamma).  Coefficients are parsed
// at quad-double level so that narrowing to d/dd gives the reference's plan coefficients bit for
// bit.

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>

#include "host.hpp"

namespace pp {

void System::refresh_degrees() {
  degrees.assign(polys.size(), 0);
  for (size_t i = 0; i < polys.size(); ++i)
    for (const Term& t : polys[i]) degrees[i] = std::max(degrees[i], t.mono.degree());
}

uint64_t System::monomial_count() const {
  uint64_t n = 0;
  for (const auto& p : polys) n += p.size();
  return n;
}

// ---------------------------------------------------------------------------------------------
// decimal I/O
// ---------------------------------------------------------------------------------------------
namespace {

// 10^k by binary powering at level R; negative k via 1/10^|k| (xprec_io.cpp:11-23)
template <class R>
R pow10_level(long k) {
  unsigned long e = k < 0 ? static_cast<unsigned long>(-k) : static_cast<unsigned long>(k);
  R base = rfrom<R>(10.0), acc = rfrom<R>(1.0);
  for (; e != 0; e >>= 1) {
    if (e & 1u) acc = rmul(acc, base);
    base = rmul(base, base);
  }
  return k < 0 ? rdiv(rfrom<R>(1.0), acc) : acc;
}

// digits are folded into the accumulator 15 at a time as exact doubles
// (val = val * 10^len + chunk, level-times-double then level-plus-double)
template <class R>
bool parse_decimal_level(std::string_view s, R& out) {
  size_t i = 0, end = s.size();
  while (i < end && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
  while (end > i && std::isspace(static_cast<unsigned char>(s[end - 1]))) --end;
  if (i >= end) return false;
  bool neg = false;
  if (s[i] == '+' || s[i] == '-') neg = s[i++] == '-';

  R val = rfrom<R>(0.0);
  long frac = 0;
  bool any = false, point = false;
  int clen = 0;
  double chunk = 0.0;
  auto fold = [&] {
    if (clen == 0) return;
    val = radd(rmuld(val, pow10_level<double>(clen)), chunk);
    chunk = 0.0;
    clen = 0;
  };
  for (; i < end; ++i) {
    char c = s[i];
    if (c >= '0' && c <= '9') {
      chunk = chunk * 10.0 + (c - '0');
      if (++clen == 15) fold();
      if (point) ++frac;
      any = true;
    } else if (c == '.') {
      if (point) return false;
      point = true;
    } else if (c == 'e' || c == 'E') {
      break;
    } else {
      return false;
    }
  }
  fold();
  if (!any) return false;
  long e10 = 0;
  if (i < end) {  // exponent
    ++i;
    bool eneg = false;
    if (i < end && (s[i] == '+' || s[i] == '-')) eneg = s[i++] == '-';
    if (i >= end) return false;
    long ev = 0;
    for (; i < end; ++i) {
      if (s[i] < '0' || s[i] > '9') return false;
      ev = ev * 10 + (s[i] - '0');
      if (ev > 100000) return false;
    }
    e10 = eneg ? -ev : ev;
  }
  long scale = e10 - frac;
  if (scale > 350 || scale < -350) return false;
  if (scale > 0) val = rmul(val, pow10_level<R>(scale));
  if (scale < 0) val = rdiv(val, pow10_level<R>(-scale));
  out = neg ? rneg(val) : val;
  return true;
}

// repeated multiply-by-ten digit extraction with carry repair and rounding on one extra digit
// (xprec_io.cpp:31-108); 32 / 64 significant digits for dd / qd
template <class R>
std::string to_decimal_level(R x, int digits) {
  double head = level<R>::get(x, 0);
  if (std::isnan(head)) return "nan";
  if (std::isinf(head)) return head > 0 ? "inf" : "-inf";
  bool neg = head < 0.0;
  R r = rabs(x);
  if (level<R>::get(r, 0) == 0.0 && rtod(r) == 0.0) {
    std::string z = "0.";
    z.append(static_cast<size_t>(digits - 1), '0');
    return z + "e+00";
  }
  int e10 = static_cast<int>(std::floor(std::log10(std::fabs(head))));
  r = rmul(r, pow10_level<R>(-e10));
  if (rcmp(r, rfrom<R>(10.0)) >= 0) {
    r = rdiv(r, rfrom<R>(10.0));
    ++e10;
  } else if (rcmp(r, rfrom<R>(1.0)) < 0) {
    r = rmul(r, rfrom<R>(10.0));
    --e10;
  }
  const int nd = digits + 1;
  std::vector<int> dig(static_cast<size_t>(nd));
  for (int i = 0; i < nd; ++i) {
    int d = static_cast<int>(level<R>::get(r, 0));
    dig[static_cast<size_t>(i)] = d;
    r = rmuld(radd(r, -static_cast<double>(d)), 10.0);
  }
  for (int i = nd - 1; i > 0; --i) {
    if (dig[i] < 0) {
      dig[i - 1] -= 1;
      dig[i] += 10;
    } else if (dig[i] > 9) {
      dig[i - 1] += 1;
      dig[i] -= 10;
    }
  }
  if (dig[nd - 1] >= 5) {
    dig[nd - 2] += 1;
    for (int i = nd - 2; i > 0 && dig[i] > 9; --i) {
      dig[i] -= 10;
      dig[i - 1] += 1;
    }
  }
  if (dig[0] > 9) {
    ++e10;
    dig[0] = 1;
    for (int i = 1; i < digits; ++i) dig[i] = 0;
  }
  std::string out = neg ? "-" : "";
  out += static_cast<char>('0' + dig[0]);
  out += '.';
  for (int i = 1; i < digits; ++i) out += static_cast<char>('0' + dig[i]);
  char buf[16];
  std::snprintf(buf, sizeof buf, "e%c%02d", e10 < 0 ? '-' : '+', e10 < 0 ? -e10 : e10);
  return out + buf;
}

}  // namespace

bool parse_decimal_qd(std::string_view s, qd_t& out) { return parse_decimal_level<qd_t>(s, out); }
bool parse_decimal_dd(std::string_view s, dd_t& out) { return parse_decimal_level<dd_t>(s, out); }
bool parse_decimal_d(std::string_view s, double& out) {
  std::string tmp(s);
  char* ep = nullptr;
  double v = std::strtod(tmp.c_str(), &ep);
  if (ep == tmp.c_str()) return false;
  for (; *ep != '\0'; ++ep)
    if (!std::isspace(static_cast<unsigned char>(*ep))) return false;
  if (std::isnan(v) || std::isinf(v)) return false;
  out = v;
  return true;
}
std::string to_decimal_qd(qd_t x) { return to_decimal_level<qd_t>(x, 64); }
std::string to_decimal_dd(dd_t x) { return to_decimal_level<dd_t>(x, 32); }
std::string to_decimal_d(double x) {
  if (std::isnan(x)) return "nan";
  if (std::isinf(x)) return x > 0 ? "inf" : "-inf";
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.16e", x);
  return buf;
}

// ---------------------------------------------------------------------------------------------
// system grammar
// ---------------------------------------------------------------------------------------------
namespace {

class Lexer {
 public:
  explicit Lexer(std::string_view t) : text_(t) {}

  [[noreturn]] void fail(const std::string& msg) const { throw ParseFailure(msg, line_, col_); }
  bool eof() const { return pos_ >= text_.size(); }
  char peek() const { return text_[pos_]; }
  size_t line() const { return line_; }
  size_t col() const { return col_; }

  void next() {
    if (text_[pos_] == '\n') {
      ++line_;
      col_ = 1;
    } else {
      ++col_;
    }
    ++pos_;
  }

  void blanks() {
    while (!eof()) {
      char c = peek();
      if (c == '#') {
        while (!eof() && peek() != '\n') next();
      } else if (c == ' ' || c == '\t' || c == '\r' || c == '\n') {
        next();
      } else {
        break;
      }
    }
  }

  bool eat(char c) {
    blanks();
    if (!eof() && peek() == c) {
      next();
      return true;
    }
    return false;
  }

  void need(char c, const char* what) {
    if (!eat(c)) fail(std::string("expected '") + c + "' (" + what + ")");
  }

  uint64_t unsigned_int(const char* what) {
    blanks();
    if (eof() || !std::isdigit(static_cast<unsigned char>(peek()))) fail(std::string("expected ") + what);
    uint64_t v = 0;
    while (!eof() && std::isdigit(static_cast<unsigned char>(peek()))) {
      v = v * 10 + static_cast<uint64_t>(peek() - '0');
      if (v > (1ull << 40)) fail(std::string(what) + " out of range");
      next();
    }
    return v;
  }

  // optionally signed decimal literal, parsed at quad-double level
  qd_t real(const char* what) {
    blanks();
    size_t start = pos_;
    bool neg = false;
    if (!eof() && (peek() == '+' || peek() == '-')) {
      neg = peek() == '-';
      next();
    }
    size_t digits = pos_;
    while (!eof() && (std::isdigit(static_cast<unsigned char>(peek())) || peek() == '.')) next();
    if (pos_ == digits) fail(std::string("expected ") + what);
    if (!eof() && (peek() == 'e' || peek() == 'E')) {
      next();
      if (!eof() && (peek() == '+' || peek() == '-')) next();
      if (eof() || !std::isdigit(static_cast<unsigned char>(peek()))) fail("malformed exponent in number");
      while (!eof() && std::isdigit(static_cast<unsigned char>(peek()))) next();
    }
    size_t skip = neg ? 1 : 0;
    qd_t v;
    if (!parse_decimal_qd(text_.substr(start + skip, pos_ - start - skip), v))
      fail(std::string("malformed number in ") + what);
    return neg ? rneg(v) : v;
  }

  struct Mark {
    size_t pos, line, col;
  };
  Mark mark() const { return {pos_, line_, col_}; }
  void reset(const Mark& m) {
    pos_ = m.pos;
    line_ = m.line;
    col_ = m.col;
  }

 private:
  std::string_view text_;
  size_t pos_ = 0, line_ = 1, col_ = 1;
};

bool cx_is_zero(const cqd& c) {
  return rcmp(c.re, qd_make(0.0)) == 0 && rcmp(c.im, qd_make(0.0)) == 0;
}

}  // namespace

System parse_system(std::string_view text) {
  Lexer lx(text);
  System sys;
  lx.blanks();
  sys.dim = static_cast<uint32_t>(lx.unsigned_int("dimension"));
  if (sys.dim == 0) lx.fail("dimension must be >= 1");
  lx.eat(';');
  lx.blanks();
  while (!lx.eof()) {
    std::vector<Monomial> order;  // first-occurrence order of monomials
    std::map<Monomial, cqd> sum;
    bool first = true;
    for (;;) {
      lx.blanks();
      if (lx.eof()) lx.fail("unterminated polynomial (missing ';')");
      int sign = 1;
      bool signed_term = false;
      for (;;) {
        if (lx.eat('+')) {
          signed_term = true;
        } else if (lx.eat('-')) {
          sign = -sign;
          signed_term = true;
        } else {
          break;
        }
      }
      if (!first && !signed_term) lx.fail("expected '+', '-' or ';' between terms");
      first = false;
      lx.blanks();
      if (lx.eof()) lx.fail("unterminated polynomial (missing ';')");
      const size_t tl = lx.line(), tc = lx.col();

      cqd coeff{qd_make(1.0), qd_make(0.0)};
      bool explicit_coeff = false;
      char c = lx.peek();
      if (c == '(') {
        lx.next();
        qd_t re = lx.real("real part");
        lx.need(',', "complex coefficient");
        qd_t im = lx.real("imaginary part");
        lx.need(')', "complex coefficient");
        coeff = {re, im};
        explicit_coeff = true;
      } else if (std::isdigit(static_cast<unsigned char>(c)) || c == '.') {
        coeff = {lx.real("coefficient"), qd_make(0.0)};
        explicit_coeff = true;
      } else if (c != 'x') {
        lx.fail("expected a coefficient or a variable factor");
      }

      Monomial mono;
      bool star_needed = explicit_coeff;
      for (;;) {
        lx.blanks();
        if (star_needed) {
          Lexer::Mark m = lx.mark();
          if (!lx.eat('*')) break;
          lx.blanks();
          if (lx.eof() || lx.peek() != 'x') {
            lx.reset(m);
            break;
          }
        } else if (lx.eof() || lx.peek() != 'x') {
          break;
        }
        lx.next();  // 'x'
        const size_t vl = lx.line(), vc = lx.col();
        uint64_t v = lx.unsigned_int("variable index");
        if (v >= sys.dim) throw ParseFailure("variable index out of range", vl, vc);
        uint32_t e = 1;
        if (lx.eat('^')) {
          lx.blanks();
          if (!lx.eof() && (lx.peek() == '-' || lx.peek() == '+')) lx.fail("exponent must be a positive integer");
          uint64_t ev = lx.unsigned_int("exponent");
          if (ev == 0) lx.fail("exponent must be >= 1");
          if (ev > 1000) lx.fail("exponent out of range");
          e = static_cast<uint32_t>(ev);
        }
        bool merged = false;
        for (auto& f : mono.factors)
          if (f.first == v) {
            f.second += e;
            merged = true;
            break;
          }
        if (!merged) mono.factors.emplace_back(static_cast<uint32_t>(v), e);
        star_needed = true;
      }
      std::sort(mono.factors.begin(), mono.factors.end());
      if (explicit_coeff && cx_is_zero(coeff)) throw ParseFailure("zero coefficient term", tl, tc);
      if (sign < 0) coeff = cneg(coeff);
      auto it = sum.find(mono);
      if (it == sum.end()) {
        sum.emplace(mono, coeff);
        order.push_back(mono);
      } else {
        it->second = cadd(it->second, coeff);
      }
      lx.blanks();
      if (lx.eat(';')) break;
    }
    std::vector<Term> poly;
    for (const Monomial& m : order) {
      const cqd& cf = sum[m];
      if (!cx_is_zero(cf)) poly.push_back(Term{cf, m});
    }
    sys.polys.push_back(std::move(poly));
    lx.blanks();
  }
  if (sys.polys.empty()) throw ParseFailure("system has no polynomials", lx.line(), lx.col());
  sys.refresh_degrees();
  return sys;
}

namespace {

std::string real_text(const qd_t& v) {
  double d = rtod(v);
  if (std::rint(d) == d && std::fabs(d) < 9.0e15 && rcmp(qd_make(d), v) == 0) {
    char buf[32];
    std::snprintf(buf, sizeof buf, "%.0f", d);
    return buf;
  }
  return to_decimal_qd(v);
}

std::string coeff_text(const cqd& c) {
  if (rcmp(c.im, qd_make(0.0)) == 0) return real_text(c.re);
  return "(" + real_text(c.re) + "," + real_text(c.im) + ")";
}

}  // namespace

std::string print_system(const System& s) {
  std::string out = std::to_string(s.dim) + ";\n";
  for (const auto& poly : s.polys) {
    if (poly.empty()) out += "0";
    bool first = true;
    for (const Term& t : poly) {
      cqd c = t.coeff;
      bool neg_real = rcmp(c.im, qd_make(0.0)) == 0 && rcmp(c.re, qd_make(0.0)) < 0;
      if (neg_real) c = cneg(c);
      if (first)
        out += neg_real ? "-" : "";
      else
        out += neg_real ? " - " : " + ";
      first = false;
      bool unit = rcmp(c.im, qd_make(0.0)) == 0 && rcmp(c.re, qd_make(1.0)) == 0;
      bool implied = unit && !t.mono.factors.empty();
      if (!implied) out += coeff_text(c);
      bool lead = implied;
      for (const auto& [v, e] : t.mono.factors) {
        if (!lead) out += "*";
        lead = false;
        out += "x" + std::to_string(v);
        if (e > 1) out += "^" + std::to_string(e);
      }
    }
    out += ";\n";
  }
  return out;
}

System cyclic_system(uint32_t n) {
  if (n < 2) throw InvalidArgument("cyclic_system: n must be >= 2");
  System sys;
  sys.dim = n;
  const cqd one{qd_make(1.0), qd_make(0.0)};
  for (uint32_t k = 1; k < n; ++k) {
    std::vector<Term> poly;
    for (uint32_t i = 0; i < n; ++i) {
      Monomial m;
      for (uint32_t j = i; j < i + k; ++j) m.factors.emplace_back(j % n, 1u);
      std::sort(m.factors.begin(), m.factors.end());
      poly.push_back(Term{one, std::move(m)});
    }
    sys.polys.push_back(std::move(poly));
  }
  Monomial full;
  for (uint32_t v = 0; v < n; ++v) full.factors.emplace_back(v, 1u);
  sys.polys.push_back({Term{one, std::move(full)}, Term{cqd{qd_make(-1.0), qd_make(0.0)}, Monomial{}}});
  sys.refresh_degrees();
  return sys;
}

std::vector<std::vector<cqd>> parse_solutions(std::string_view text, uint32_t dim) {
  std::vector<std::vector<cqd>> sols;
  size_t lineno = 0, pos = 0;
  while (pos < text.size()) {
    size_t eol = text.find('\n', pos);
    if (eol == std::string_view::npos) eol = text.size();
    std::string_view line = text.substr(pos, eol - pos);
    pos = eol + 1;
    ++lineno;
    if (size_t h = line.find('#'); h != std::string_view::npos) line = line.substr(0, h);
    if (std::all_of(line.begin(), line.end(), [](char c) { return std::isspace(static_cast<unsigned char>(c)); }))
      continue;
    std::vector<qd_t> reals;
    size_t fpos = 0;
    while (fpos < line.size()) {
      size_t comma = line.find(',', fpos);
      std::string_view field =
          line.substr(fpos, comma == std::string_view::npos ? std::string_view::npos : comma - fpos);
      fpos = comma == std::string_view::npos ? line.size() : comma + 1;
      std::string cleaned;
      for (char c : field)
        if (c != '(' && c != ')') cleaned += c;
      qd_t v;
      if (!parse_decimal_qd(cleaned, v)) throw ParseFailure("malformed number in solution", lineno, fpos);
      reals.push_back(v);
    }
    if (reals.size() != 2ull * dim) throw ParseFailure("solution has wrong number of components", lineno, 1);
    std::vector<cqd> sol(dim);
    for (uint32_t i = 0; i < dim; ++i) sol[i] = cqd{reals[2 * i], reals[2 * i + 1]};
    sols.push_back(std::move(sol));
  }
  return sols;
}

void random_gamma(uint64_t seed, double& re, double& im) {
  auto mix = [](uint64_t& state) {
    state += 0x9e3779b97f4a7c15ULL;
    uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  };
  uint64_t s = seed;
  (void)mix(s);  // small seeds decorrelated by one discarded draw
  double u = static_cast<double>(mix(s) >> 11) * 0x1p-53;
  double theta = 2.0 * M_PI * u;
  re = std::cos(theta);
  im = std::sin(theta);
}

}  // namespace pp
