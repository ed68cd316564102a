// Exact floating-point expansion arithmetic for the stencil predicates (R13, R29).
//
// A value is a nonoverlapping expansion x = Σ t[k] of doubles in increasing
// magnitude (zero-free); sums and products of doubles are represented exactly
// with the error-free transformations two_sum / two_prod (fma).  Every result is
// re-compressed so expansions stay a few terms long.  Used only when a
// floating-point filter cannot certify a sign: orientation of a cell, the sign of
// a barycentric coordinate (cone membership), equality of squared distances,
// affine independence of sector barycentres.
#pragma once

#include <cmath>
#include <stdexcept>

namespace cwr {
namespace exact {

constexpr int CAP = 96;

struct Ex {
  int n = 0;
  double t[CAP];
  Ex() = default;
  explicit Ex(double a) { if (a != 0.0) { t[0] = a; n = 1; } }
};

inline void two_sum(double a, double b, double& x, double& y) {
  x = a + b;
  double bv = x - a;
  double av = x - bv;
  y = (a - av) + (b - bv);
}

inline void fast_two_sum(double a, double b, double& x, double& y) {  // |a| >= |b|
  x = a + b;
  y = b - (x - a);
}

inline void two_prod(double a, double b, double& x, double& y) {
  x = a * b;
  y = std::fma(a, b, -x);
}

inline void push(Ex& h, double v) {
  if (h.n >= CAP) throw std::runtime_error("exact expansion overflow");
  h.t[h.n++] = v;
}

// e += b in place (Shewchuk, Grow-Expansion with zero elimination)
inline void grow_inplace(Ex& e, double b) {
  double Q = b;
  int k = 0;
  for (int i = 0; i < e.n; ++i) {
    double Qn, hh;
    two_sum(Q, e.t[i], Qn, hh);
    Q = Qn;
    if (hh != 0.0) e.t[k++] = hh;
  }
  if (Q != 0.0 || k == 0) {
    if (k >= CAP) throw std::runtime_error("exact expansion overflow");
    e.t[k++] = Q;
  }
  e.n = k;
  if (e.n == 1 && e.t[0] == 0.0) e.n = 0;
}

inline Ex grow(const Ex& e, double b) {
  Ex h;
  h.n = e.n;
  for (int i = 0; i < e.n; ++i) h.t[i] = e.t[i];
  grow_inplace(h, b);
  return h;
}

// Compression to a short nonoverlapping expansion, in place (Shewchuk, Compress)
inline void compress_inplace(Ex& e) {
  if (e.n <= 1) return;
  double g[CAP];
  int bottom = e.n - 1;
  double Q = e.t[bottom];
  for (int i = e.n - 2; i >= 0; --i) {
    double Qn, q;
    fast_two_sum(Q, e.t[i], Qn, q);
    if (q != 0.0) {
      g[bottom--] = Qn;
      Q = q;
    } else {
      Q = Qn;
    }
  }
  int top = 0;
  for (int i = bottom + 1; i < e.n; ++i) {
    double Qn, q;
    fast_two_sum(g[i], Q, Qn, q);
    if (q != 0.0) e.t[top++] = q;
    Q = Qn;
  }
  if (Q != 0.0 || top == 0) e.t[top++] = Q;
  e.n = top;
  if (e.n == 1 && e.t[0] == 0.0) e.n = 0;
}

inline Ex compress(const Ex& e) {
  Ex h;
  h.n = e.n;
  for (int i = 0; i < e.n; ++i) h.t[i] = e.t[i];
  compress_inplace(h);
  return h;
}

inline void add_into(Ex& acc, const Ex& b) {  // acc += b, compressed
  for (int i = 0; i < b.n; ++i) grow_inplace(acc, b.t[i]);
  compress_inplace(acc);
}

inline Ex add(const Ex& a, const Ex& b) {
  Ex h;
  h.n = a.n;
  for (int i = 0; i < a.n; ++i) h.t[i] = a.t[i];
  add_into(h, b);
  return h;
}

inline Ex neg(const Ex& a) {
  Ex h;
  h.n = a.n;
  for (int i = 0; i < h.n; ++i) h.t[i] = -a.t[i];
  return h;
}

inline Ex sub(const Ex& a, const Ex& b) {
  Ex h;
  h.n = a.n;
  for (int i = 0; i < a.n; ++i) h.t[i] = a.t[i];
  for (int i = 0; i < b.n; ++i) grow_inplace(h, -b.t[i]);
  compress_inplace(h);
  return h;
}

// h = e * b   (Shewchuk, Scale-Expansion with zero elimination)
inline void scale_into(const Ex& e, double b, Ex& h) {
  h.n = 0;
  if (e.n == 0 || b == 0.0) return;
  double Q, hh;
  two_prod(e.t[0], b, Q, hh);
  if (hh != 0.0) push(h, hh);
  for (int i = 1; i < e.n; ++i) {
    double p1, p0, s;
    two_prod(e.t[i], b, p1, p0);
    two_sum(Q, p0, s, hh);
    if (hh != 0.0) push(h, hh);
    fast_two_sum(p1, s, Q, hh);
    if (hh != 0.0) push(h, hh);
  }
  if (Q != 0.0 || h.n == 0) push(h, Q);
  if (h.n == 1 && h.t[0] == 0.0) h.n = 0;
}

inline Ex scale(const Ex& e, double b) {
  Ex h;
  scale_into(e, b, h);
  return h;
}

inline Ex mul(const Ex& a, const Ex& b) {
  Ex acc, tmp;
  for (int i = 0; i < b.n; ++i) {
    scale_into(a, b.t[i], tmp);
    add_into(acc, tmp);
  }
  return acc;
}

inline int sign(const Ex& a) {
  for (int i = a.n - 1; i >= 0; --i)
    if (a.t[i] != 0.0) return a.t[i] > 0 ? 1 : -1;
  return 0;
}

inline double approx(const Ex& a) {
  double s = 0.0;
  for (int i = 0; i < a.n; ++i) s += a.t[i];
  return s;
}

// Exact orientation determinant of d+1 points (expansions), d ∈ {2,3}.
inline int orient_sign(int d, const Ex* const* p) {
  if (d == 2) {
    Ex ax = sub(p[1][0], p[0][0]), ay = sub(p[1][1], p[0][1]);
    Ex bx = sub(p[2][0], p[0][0]), by = sub(p[2][1], p[0][1]);
    return sign(sub(mul(ax, by), mul(ay, bx)));
  }
  Ex u[3], v[3], w[3];
  for (int k = 0; k < 3; ++k) {
    u[k] = sub(p[1][k], p[0][k]);
    v[k] = sub(p[2][k], p[0][k]);
    w[k] = sub(p[3][k], p[0][k]);
  }
  Ex c0 = sub(mul(v[1], w[2]), mul(v[2], w[1]));
  Ex c1 = sub(mul(v[2], w[0]), mul(v[0], w[2]));
  Ex c2 = sub(mul(v[0], w[1]), mul(v[1], w[0]));
  return sign(add(add(mul(u[0], c0), mul(u[1], c1)), mul(u[2], c2)));
}

}  // namespace exact
}  // namespace cwr
