// Orthonormal Dubiner basis on the reference simplex T_E (reading R8)
// and the universal oscillation-indicator matrix Σ.
//
// ψ is evaluated with the homogenised Jacobi three-term recurrence, which has no
// division, so it is valid at points outside T_E (stencil cells lie outside the
// owner's reference element):
//   2D ψ_pq  = c · H_p^{(0,0)}(2ξ+η−1, 1−η) · P_q^{(2p+1,0)}(2η−1)
//   3D ψ_pqr = c · H_p^{(0,0)}(2ξ+η+ζ−1, 1−η−ζ) · H_q^{(2p+1,0)}(2η+ζ−1, 1−ζ)
//                · P_r^{(2p+2q+2,0)}(2ζ−1)
// with H_n^{(α,β)}(num, den) = den^n P_n^{(α,β)}(num/den) and the
// normalisation c making ∫_{T_E} ψ_l ψ_m = δ_lm.  Σ is integrated with a
// collapsed Gauss-Legendre rule from the monomial form of the derivatives.
#include <array>
#include <cmath>
#include <vector>

#include "internal.hpp"

namespace cwr {

namespace {

// dense polynomial in up to 3 variables, exponents < P per variable
struct Poly {
  int P = 0;
  std::vector<double> a;  // a[(i*P + j)*P + k]  ξ^i η^j ζ^k
  explicit Poly(int P_ = 0, double c = 0.0) : P(P_), a(size_t(P_) * P_ * P_, 0.0) {
    if (P_ > 0) a[0] = c;
  }
  double& at(int i, int j, int k) { return a[(size_t(i) * P + j) * P + k]; }
  double at(int i, int j, int k) const { return a[(size_t(i) * P + j) * P + k]; }
};
Poly operator+(const Poly& x, const Poly& y) {
  Poly r(x.P);
  for (size_t t = 0; t < r.a.size(); ++t) r.a[t] = x.a[t] + y.a[t];
  return r;
}
Poly operator*(double s, const Poly& x) {
  Poly r(x.P);
  for (size_t t = 0; t < r.a.size(); ++t) r.a[t] = s * x.a[t];
  return r;
}
Poly operator*(const Poly& x, const Poly& y) {
  const int P = x.P;
  Poly r(P);
  for (int i = 0; i < P; ++i)
    for (int j = 0; j < P; ++j)
      for (int k = 0; k < P; ++k) {
        double v = x.at(i, j, k);
        if (v == 0.0) continue;
        for (int i2 = 0; i2 < P; ++i2)
          for (int j2 = 0; j2 < P; ++j2)
            for (int k2 = 0; k2 < P; ++k2) {
              double w = y.at(i2, j2, k2);
              if (w == 0.0) continue;
              if (i + i2 >= P || j + j2 >= P || k + k2 >= P) throw Error(CWRECO_EINVAL, "poly degree overflow");
              r.at(i + i2, j + j2, k + k2) += v * w;
            }
      }
  return r;
}

// homogenised Jacobi H_n^{(al,0)}(num, den) for any number-like T
template <class T>
T hjacobi(int n, double al, const T& num, const T& den, const T& one) {
  if (n == 0) return one;
  const double be = 0.0;
  T h0 = one;
  T h1 = 0.5 * ((al + be + 2.0) * num + (al - be) * den);
  for (int m = 2; m <= n; ++m) {
    const double s = 2.0 * m + al + be;
    const double a1 = 2.0 * m * (m + al + be) * (s - 2.0);
    const double a2 = (s - 1.0) * (al * al - be * be);
    const double a3 = (s - 2.0) * (s - 1.0) * s;
    const double a4 = 2.0 * (m + al - 1.0) * (m + be - 1.0) * s;
    T h2 = (1.0 / a1) * ((a2 * den + a3 * num) * h1 + (-a4) * ((den * den) * h0));
    h0 = h1;
    h1 = h2;
  }
  return h1;
}

template <class T>
void dubiner(int d, int M, const T* x, const T& one, std::vector<T>& out) {
  out.clear();
  if (d == 2) {
    const T& xi = x[0];
    const T& eta = x[1];
    T n1 = 2.0 * xi + eta + (-1.0) * one, d1 = one + (-1.0) * eta;
    T n2 = 2.0 * eta + (-1.0) * one;
    for (int n = 0; n <= M; ++n)
      for (int q = 0; q <= n; ++q) {
        const int p = n - q;
        const double c = std::sqrt(double((2 * p + 1) * (2 * p + 2 * q + 2)));
        out.push_back(c * (hjacobi(p, 0.0, n1, d1, one) * hjacobi(q, 2.0 * p + 1, n2, one, one)));
      }
  } else {
    const T& xi = x[0];
    const T& eta = x[1];
    const T& zeta = x[2];
    T n1 = 2.0 * xi + eta + zeta + (-1.0) * one, d1 = one + (-1.0) * eta + (-1.0) * zeta;
    T n2 = 2.0 * eta + zeta + (-1.0) * one, d2 = one + (-1.0) * zeta;
    T n3 = 2.0 * zeta + (-1.0) * one;
    for (int n = 0; n <= M; ++n)
      for (int r = 0; r <= n; ++r)
        for (int q = 0; q <= n - r; ++q) {
          const int p = n - q - r;
          const double c = std::sqrt(double((2 * p + 1) * (2 * p + 2 * q + 2) * (2 * p + 2 * q + 2 * r + 3)));
          out.push_back(c * ((hjacobi(p, 0.0, n1, d1, one) * hjacobi(q, 2.0 * p + 1, n2, d2, one)) *
                             hjacobi(r, 2.0 * p + 2 * q + 2, n3, one, one)));
        }
  }
}

Poly deriv(const Poly& f, int var) {
  Poly r(f.P);
  for (int i = 0; i < f.P; ++i)
    for (int j = 0; j < f.P; ++j)
      for (int k = 0; k < f.P; ++k) {
        int e = var == 0 ? i : var == 1 ? j : k;
        if (e == 0) continue;
        double v = f.at(i, j, k) * e;
        if (var == 0) r.at(i - 1, j, k) += v;
        else if (var == 1) r.at(i, j - 1, k) += v;
        else r.at(i, j, k - 1) += v;
      }
  return r;
}

double peval(const Poly& f, const double* x, int d) {
  double s = 0.0;
  for (int i = 0; i < f.P; ++i)
    for (int j = 0; j < f.P; ++j)
      for (int k = 0; k < f.P; ++k) {
        double v = f.at(i, j, k);
        if (v == 0.0) continue;
        s += v * std::pow(x[0], i) * std::pow(x[1], j) * (d == 3 ? std::pow(x[2], k) : (k == 0 ? 1.0 : 0.0));
      }
  return s;
}

}  // namespace

// ψ_l(ξ) for l < ℳ (any ξ, inside or outside T_E)
void basis_eval(int d, int M, const double* xi, double* out) {
  thread_local std::vector<double> v;
  dubiner<double>(d, M, xi, 1.0, v);
  for (size_t l = 0; l < v.size(); ++l) out[l] = v[l];
}

void gauss_legendre01(int n, std::vector<double>& x, std::vector<double>& w) {
  x.assign(n, 0);
  w.assign(n, 0);
  for (int i = 0; i < n; ++i) {
    double z = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = z;
      for (int k = 2; k <= n; ++k) {
        double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      double pn = n == 1 ? z : p1, pnm1 = n == 1 ? 1.0 : p0;
      double dp = n * (z * pn - pnm1) / (z * z - 1.0);
      double dz = pn / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    double p0 = 1.0, p1 = z;
    for (int k = 2; k <= n; ++k) {
      double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
      p0 = p1;
      p1 = p2;
    }
    double pn = n == 1 ? z : p1, pnm1 = n == 1 ? 1.0 : p0;
    double dp = n * (z * pn - pnm1) / (z * z - 1.0);
    x[i] = 0.5 * (1.0 - z);
    w[i] = 1.0 / ((1.0 - z * z) * dp * dp);  // 2/((1-z^2)P'^2) on [-1,1], halved
  }
}

// Monomial form of the basis: exps [nmono][3] (ζ exponent 0 for d=2, total degree
// <= M, graded order) and coef [ℳ][nmono] with ψ_l = Σ_e coef[l][e] ξ^e.
void basis_monomials(int d, int M, std::vector<int>& exps, std::vector<double>& coef) {
  const int nm = n_modes(M, d);
  const int P = M + 1;
  Poly one(P, 1.0);
  Poly vars[3] = {Poly(P), Poly(P), Poly(P)};
  vars[0].at(1, 0, 0) = 1.0;
  if (P > 1) vars[1].at(0, 1, 0) = 1.0;
  if (d == 3 && P > 1) vars[2].at(0, 0, 1) = 1.0;
  std::vector<Poly> psi;
  dubiner<Poly>(d, M, vars, one, psi);
  exps.clear();
  for (int n = 0; n <= M; ++n)
    for (int i = n; i >= 0; --i)
      for (int j = n - i; j >= 0; --j) {
        const int k = n - i - j;
        if (d == 2 && k != 0) continue;
        exps.push_back(i);
        exps.push_back(j);
        exps.push_back(k);
      }
  const int ne = (int)exps.size() / 3;
  coef.assign(size_t(nm) * ne, 0.0);
  for (int l = 0; l < nm; ++l)
    for (int e = 0; e < ne; ++e) coef[size_t(l) * ne + e] = psi[l].at(exps[3 * e], exps[3 * e + 1], exps[3 * e + 2]);
}

// Gauss-Jacobi nodes/weights for the weight (1-x)^alpha on [-1,1] (beta = 0), mapped
// to t = (1+x)/2 ∈ [0,1] (weights not normalised).  Newton with deflation.
void gauss_jacobi01(int n, double alpha, std::vector<double>& t, std::vector<double>& w) {
  const double beta = 0.0;
  auto jac = [&](int m, double al, double be, double x) {  // P_m^{(al,be)}(x)
    if (m == 0) return 1.0;
    double p0 = 1.0, p1 = 0.5 * ((al + be + 2.0) * x + (al - be));
    for (int k = 2; k <= m; ++k) {
      const double s = 2.0 * k + al + be;
      const double a1 = 2.0 * k * (k + al + be) * (s - 2.0);
      const double a2 = (s - 1.0) * (al * al - be * be);
      const double a3 = (s - 2.0) * (s - 1.0) * s;
      const double a4 = 2.0 * (k + al - 1.0) * (k + be - 1.0) * s;
      const double p2 = ((a2 + a3 * x) * p1 - a4 * p0) / a1;
      p0 = p1;
      p1 = p2;
    }
    return p1;
  };
  auto djac = [&](double x) { return 0.5 * (n + alpha + beta + 1.0) * jac(n - 1, alpha + 1.0, beta + 1.0, x); };
  std::vector<double> x(n);
  for (int k = 0; k < n; ++k) {
    double r = -std::cos((2.0 * k + 1.0) * M_PI / (2.0 * n));
    if (k > 0) r = 0.5 * (r + x[k - 1]);
    for (int it = 0; it < 100; ++it) {
      double s = 0.0;
      for (int i = 0; i < k; ++i) s += 1.0 / (r - x[i]);
      const double p = jac(n, alpha, beta, r);
      const double delta = -p / (djac(r) - s * p);
      r += delta;
      if (std::fabs(delta) < 1e-16) break;
    }
    x[k] = r;
  }
  t.assign(n, 0.0);
  w.assign(n, 0.0);
  for (int k = 0; k < n; ++k) {
    const double dp = djac(x[k]);
    t[k] = 0.5 * (1.0 + x[k]);
    w[k] = 1.0 / ((1.0 - x[k] * x[k]) * dp * dp);  // ∝ Gauss-Jacobi weight (constant factor dropped)
  }
}

std::vector<double> sigma_matrix(int d, int M) {
  const int nm = n_modes(M, d);
  const int P = M + 1;
  Poly one(P, 1.0);
  Poly vars[3] = {Poly(P), Poly(P), Poly(P)};
  vars[0].at(1, 0, 0) = 1.0;
  if (P > 1) vars[1].at(0, 1, 0) = 1.0;
  if (d == 3 && P > 1) vars[2].at(0, 0, 1) = 1.0;
  std::vector<Poly> psi;
  dubiner<Poly>(d, M, vars, one, psi);
  // derivatives ∂^α ψ_l for 1 <= |α| <= M, each multi-index once (R9)
  std::vector<std::vector<Poly>> D(nm);
  for (int l = 0; l < nm; ++l) {
    for (int a0 = 0; a0 <= M; ++a0)
      for (int a1 = 0; a1 <= M; ++a1)
        for (int a2 = 0; a2 <= (d == 3 ? M : 0); ++a2) {
          int s = a0 + a1 + a2;
          if (s < 1 || s > M) continue;
          Poly f = psi[l];
          for (int t = 0; t < a0; ++t) f = deriv(f, 0);
          for (int t = 0; t < a1; ++t) f = deriv(f, 1);
          for (int t = 0; t < a2; ++t) f = deriv(f, 2);
          D[l].push_back(f);
        }
  }
  // collapsed Gauss-Legendre on T_E
  std::vector<double> gx, gw;
  gauss_legendre01(M + 3, gx, gw);
  std::vector<std::array<double, 3>> pts;
  std::vector<double> wts;
  const int n = (int)gx.size();
  if (d == 2) {
    for (int a = 0; a < n; ++a)
      for (int b = 0; b < n; ++b) {
        pts.push_back({gx[a] * (1 - gx[b]), gx[b], 0.0});
        wts.push_back(gw[a] * gw[b] * (1 - gx[b]));
      }
  } else {
    for (int a = 0; a < n; ++a)
      for (int b = 0; b < n; ++b)
        for (int c = 0; c < n; ++c) {
          pts.push_back({gx[a] * (1 - gx[b]) * (1 - gx[c]), gx[b] * (1 - gx[c]), gx[c]});
          wts.push_back(gw[a] * gw[b] * gw[c] * (1 - gx[b]) * (1 - gx[c]) * (1 - gx[c]));
        }
  }
  const size_t na = D[0].size();
  std::vector<double> val(nm * na * pts.size());
  for (int l = 0; l < nm; ++l)
    for (size_t t = 0; t < na; ++t)
      for (size_t q = 0; q < pts.size(); ++q) val[(l * na + t) * pts.size() + q] = peval(D[l][t], pts[q].data(), d);
  std::vector<double> S(nm * nm, 0.0);
  for (int l = 0; l < nm; ++l)
    for (int m = 0; m < nm; ++m) {
      double s = 0.0;
      for (size_t t = 0; t < na; ++t)
        for (size_t q = 0; q < pts.size(); ++q)
          s += wts[q] * val[(l * na + t) * pts.size() + q] * val[(m * na + t) * pts.size() + q];
      S[l * nm + m] = s;
    }
  for (int l = 0; l < nm; ++l) {  // exact structure: constant ψ_1 has no derivatives
    S[l] = 0.0;
    S[l * nm] = 0.0;
  }
  for (int l = 0; l < nm; ++l)  // symmetrise the rounding
    for (int m = l + 1; m < nm; ++m) {
      double v = 0.5 * (S[l * nm + m] + S[m * nm + l]);
      S[l * nm + m] = S[m * nm + l] = v;
    }
  return S;
}

// Face quadrature (NEXT-3): M+1 points per direction, exact for degree 2M+1 on the
// face; barycentric weights lam [nq][d] over the face's d vertices (in the caller's
// canonical order), weights normalised to 1 (face average).  2-D: Gauss–Legendre
// on the edge; 3-D: collapsed Gauss–Jacobi on the triangle (u, v) ↦ (u(1−v), v).
void face_rule(int d, int M, std::vector<double>& lam, std::vector<double>& w) {
  lam.clear();
  w.clear();
  const int n = M + 1;
  std::vector<double> ua, wa, vb, wb;
  gauss_jacobi01(n, 0.0, ua, wa);
  if (d == 2) {
    for (int a = 0; a < n; ++a) {
      lam.push_back(1.0 - ua[a]);
      lam.push_back(ua[a]);
      w.push_back(wa[a]);
    }
  } else {
    gauss_jacobi01(n, 1.0, vb, wb);
    for (int a = 0; a < n; ++a)
      for (int b = 0; b < n; ++b) {
        const double x = ua[a] * (1.0 - vb[b]), y = vb[b];
        lam.push_back(1.0 - x - y);
        lam.push_back(x);
        lam.push_back(y);
        w.push_back(wa[a] * wb[b]);
      }
  }
  double s = 0.0;
  for (double x : w) s += x;
  for (double& x : w) x /= s;
}

}  // namespace cwr

