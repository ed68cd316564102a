// Host side of the local space-time Galerkin predictor (paper §2.2, P:235-320;
// SURVEY §8(f) NEXT-2): the nodal space-time basis on T_E × [0,1], the matrices of
// Eq. cgPDE, and the per-cell inverse Jacobians.  Readings R32-R36:
//   nodes (R32): uniform lattice of the (d+1)-simplex {ξ ≥ 0, τ ≥ 0, Σξ + τ ≤ 1},
//     spacing 1/M, ordered known (τ = 0) first, then by (τ level, integer tuple);
//   test functions (R33): θ_k of the unknown (τ > 0) nodes — a square system;
//   Ĥ_l = ∇_x·F_h at node l (R34); Picard from q̂ = w(ξ_l), stop at
//   max|Δq̂| ≤ 1e-12·max(1, max|q̂⁰|) or 2(M+1) iterations (R35).
// The oracle builds the same matrices from exact rationals; here they come from a
// floating-point Vandermonde inverse and tensor Gauss quadrature (degree 2M).
#include <algorithm>
#include <cmath>
#include <cstring>

#include "internal.hpp"

namespace cwr {

namespace {

// Dense LU with partial pivoting; solves A X = B in place (B: n × m, row-major).
void lu_solve(int n, std::vector<double> A, std::vector<double>& B, int m) {
  std::vector<int> piv(n);
  for (int k = 0; k < n; ++k) {
    int p = k;
    for (int i = k + 1; i < n; ++i)
      if (std::fabs(A[i * n + k]) > std::fabs(A[p * n + k])) p = i;
    if (A[p * n + k] == 0.0) fail(CWRECO_ESINGULAR, "predictor: singular space-time system");
    if (p != k) {
      for (int j = 0; j < n; ++j) std::swap(A[k * n + j], A[p * n + j]);
      for (int j = 0; j < m; ++j) std::swap(B[k * m + j], B[p * m + j]);
    }
    for (int i = k + 1; i < n; ++i) {
      const double f = A[i * n + k] / A[k * n + k];
      if (f == 0.0) continue;
      for (int j = k; j < n; ++j) A[i * n + j] -= f * A[k * n + j];
      for (int j = 0; j < m; ++j) B[i * m + j] -= f * B[k * m + j];
    }
  }
  for (int k = n - 1; k >= 0; --k)
    for (int j = 0; j < m; ++j) {
      double s = B[k * m + j];
      for (int i = k + 1; i < n; ++i) s -= A[k * n + i] * B[i * m + j];
      B[k * m + j] = s / A[k * n + k];
    }
}

}  // namespace

void st_nodes(int d, int M, std::vector<std::vector<int>>& nodes) {
  nodes.clear();
  std::vector<int> e(d + 1, 0);
  std::function<void(int, int)> rec = [&](int a, int left) {
    if (a == d + 1) {
      nodes.push_back(e);
      return;
    }
    for (int v = 0; v <= left; ++v) {
      e[a] = v;
      rec(a + 1, left - v);
    }
  };
  rec(0, M);
  std::stable_sort(nodes.begin(), nodes.end(), [&](const std::vector<int>& a, const std::vector<int>& b) {
    const int ta = a[d], tb = b[d];
    if ((ta > 0) != (tb > 0)) return ta == 0;
    if (ta != tb) return ta < tb;
    return a < b;
  });
}

void predictor_matrices(int d, int M, PredictorHost& h) {
  std::vector<std::vector<int>> nodes, monos;
  st_nodes(d, M, nodes);
  st_nodes(d, M, monos);  // the same exponent set serves as monomial basis
  const int L = (int)nodes.size(), nk = n_modes(M, d), nu = L - nk;
  h.L = L;
  h.nk = nk;
  h.nodes.assign(size_t(L) * (d + 1), 0.0);
  for (int l = 0; l < L; ++l)
    for (int a = 0; a <= d; ++a) h.nodes[l * (d + 1) + a] = double(nodes[l][a]) / M;
  auto mono = [&](int j, const double* x) {
    double v = 1.0;
    for (int a = 0; a <= d; ++a)
      for (int p = 0; p < monos[j][a]; ++p) v *= x[a];
    return v;
  };
  auto dmono = [&](int j, int b, const double* x) {  // ∂/∂x_b of monomial j
    if (monos[j][b] == 0) return 0.0;
    double v = monos[j][b];
    for (int a = 0; a <= d; ++a)
      for (int p = 0; p < monos[j][a] - (a == b ? 1 : 0); ++p) v *= x[a];
    return v;
  };
  // Lagrange coefficients: V C = I with V[i][j] = mono_j(node_i)  (θ_l = Σ_j C[j][l] mono_j)
  std::vector<double> Vm(size_t(L) * L), C(size_t(L) * L, 0.0);
  for (int i = 0; i < L; ++i)
    for (int j = 0; j < L; ++j) Vm[i * L + j] = mono(j, &h.nodes[i * (d + 1)]);
  for (int i = 0; i < L; ++i) C[i * L + i] = 1.0;
  lu_solve(L, Vm, C, L);
  auto theta = [&](int l, const double* x) {
    double s = 0.0;
    for (int j = 0; j < L; ++j) s += C[j * L + l] * mono(j, x);
    return s;
  };
  auto dtheta = [&](int l, int b, const double* x) {
    double s = 0.0;
    for (int j = 0; j < L; ++j) s += C[j * L + l] * dmono(j, b, x);
    return s;
  };
  // prism quadrature: simplex rule of degree 2M (weights normalised to average → × |T_E|)
  // × Gauss-Legendre in τ with M+1 points (degree 2M+1)
  std::vector<double> sp, sw, tp, tw;
  simplex_rule(d, 2 * M, sp, sw);
  gauss_legendre01(M + 1, tp, tw);
  double vol = 1.0;
  for (int a = 2; a <= d; ++a) vol /= a;
  std::vector<double> Mm(size_t(L) * L, 0.0), Kt(size_t(L) * L, 0.0);
  std::vector<double> x(d + 1), th(L), dth(L);
  for (size_t q = 0; q < sw.size(); ++q)
    for (size_t t = 0; t < tw.size(); ++t) {
      for (int a = 0; a < d; ++a) x[a] = sp[q * d + a];
      x[d] = tp[t];
      const double w = sw[q] * vol * tw[t];
      for (int l = 0; l < L; ++l) {
        th[l] = theta(l, x.data());
        dth[l] = dtheta(l, d, x.data());
      }
      for (int k = 0; k < L; ++k)
        for (int l = 0; l < L; ++l) {
          Mm[k * L + l] += w * th[k] * th[l];
          Kt[k * L + l] += w * th[k] * dth[l];
        }
    }
  // unknown rows (test functions θ_k, k ≥ nk): K_uu X = [M_u D_b | K_uk]
  std::vector<double> Kuu(size_t(nu) * nu);
  for (int i = 0; i < nu; ++i)
    for (int j = 0; j < nu; ++j) Kuu[i * nu + j] = Kt[(nk + i) * L + nk + j];
  const int ncol = d * L + nk;
  std::vector<double> rhs(size_t(nu) * ncol, 0.0);
  for (int b = 0; b < d; ++b)
    for (int l = 0; l < L; ++l) {  // column l of M_u D_b: Σ_m M[nk+i][m] D_b[m][l]
      for (int i = 0; i < nu; ++i) {
        double s = 0.0;
        for (int m = 0; m < L; ++m) s += Mm[(nk + i) * L + m] * dtheta(l, b, &h.nodes[m * (d + 1)]);
        rhs[i * ncol + b * L + l] = s;
      }
    }
  for (int i = 0; i < nu; ++i)
    for (int j = 0; j < nk; ++j) rhs[i * ncol + d * L + j] = Kt[(nk + i) * L + j];
  lu_solve(nu, Kuu, rhs, ncol);
  // A_b [nu][L] = K_uu⁻¹ M_u D_b;  C0 [nu][nk] = K_uu⁻¹ K_uk;  Phi [L][ℳ] = ψ_m(ξ_l)
  h.A.assign(size_t(d) * nu * L, 0.0);
  for (int b = 0; b < d; ++b)
    for (int i = 0; i < nu; ++i)
      for (int l = 0; l < L; ++l) h.A[(b * nu + i) * L + l] = rhs[i * ncol + b * L + l];
  h.C0.assign(size_t(nu) * nk, 0.0);
  for (int i = 0; i < nu; ++i)
    for (int j = 0; j < nk; ++j) h.C0[i * nk + j] = rhs[i * ncol + d * L + j];
  h.Phi.assign(size_t(L) * nk, 0.0);
  for (int l = 0; l < L; ++l) basis_eval(d, M, &h.nodes[l * (d + 1)], &h.Phi[l * nk]);
}

// ∂ξ/∂x of every owned cell in LOCAL order: x = X0 + J ξ, Jinv = J⁻¹
void predictor_jinv(const cwreco_ctx* c, std::vector<double>& jinv) {
  const int d = c->d;
  jinv.assign(size_t(c->n_owned) * d * d, 0.0);
  for (int64_t li = 0; li < c->n_owned; ++li) {
    const int64_t g = c->local2global[li];
    const double* X = &c->X[g * (d + 1) * d];
    double J[9];
    for (int e = 0; e < d; ++e)
      for (int k = 0; k < d; ++k) J[e * d + k] = X[(k + 1) * d + e] - X[e];
    std::vector<double> A(J, J + d * d), I(size_t(d) * d, 0.0);
    for (int e = 0; e < d; ++e) I[e * d + e] = 1.0;
    lu_solve(d, A, I, d);
    std::copy(I.begin(), I.end(), jinv.begin() + li * d * d);
  }
}

}  // namespace cwr
