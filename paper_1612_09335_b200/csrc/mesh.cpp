// Mesh ingest: validation, periodic unwrap (R16), orientation fix (R28),
// IEEE barycentres and Morton order (R29), face / node adjacency.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <numeric>
#include <parallel/algorithm>

#include "exact.hpp"
#include "internal.hpp"

namespace cwr {

namespace {

// Exact sign of the orientation of a cell from its unwrapped vertex doubles.
int cell_orientation(int d, const double* X) {
  // filter: double determinant with a generous error bound
  double e[3][3];
  for (int k = 0; k < d; ++k)
    for (int a = 0; a < d; ++a) e[k][a] = X[(k + 1) * d + a] - X[a];
  double det, perm;
  if (d == 2) {
    double t1 = e[0][0] * e[1][1], t2 = e[0][1] * e[1][0];
    det = t1 - t2;
    perm = std::fabs(t1) + std::fabs(t2);
  } else {
    double c0 = e[1][1] * e[2][2] - e[1][2] * e[2][1];
    double c1 = e[1][2] * e[2][0] - e[1][0] * e[2][2];
    double c2 = e[1][0] * e[2][1] - e[1][1] * e[2][0];
    det = e[0][0] * c0 + e[0][1] * c1 + e[0][2] * c2;
    perm = std::fabs(e[0][0]) * (std::fabs(e[1][1] * e[2][2]) + std::fabs(e[1][2] * e[2][1])) +
           std::fabs(e[0][1]) * (std::fabs(e[1][2] * e[2][0]) + std::fabs(e[1][0] * e[2][2])) +
           std::fabs(e[0][2]) * (std::fabs(e[1][0] * e[2][1]) + std::fabs(e[1][1] * e[2][0]));
  }
  if (std::fabs(det) > 1e-10 * perm) return det > 0 ? 1 : -1;
  exact::Ex P[4][3];
  const exact::Ex* pp[4];
  for (int k = 0; k <= d; ++k) {
    for (int a = 0; a < d; ++a) P[k][a] = exact::Ex(X[k * d + a]);
    pp[k] = P[k];
  }
  return exact::orient_sign(d, pp);
}

uint64_t spread_bits(uint64_t q, int d, int k) {
  uint64_t key = 0;
  for (int t = 0; t < k; ++t) key |= ((q >> t) & 1ull) << (uint64_t)(d * t);
  return key;
}

}  // namespace

void set_mesh(cwreco_ctx* c, int64_t n_nodes, const double* xyz, int64_t n_cells,
              const int64_t* cells_in, const double* period) {
  const int d = c->d, nv = d + 1;
  if (n_nodes <= 0 || n_cells <= 0 || !xyz || !cells_in) fail(CWRECO_EINVAL, "set_mesh: empty mesh or NULL array");
  if (n_cells > INT32_MAX - 1) fail(CWRECO_EUNSUPPORTED, "set_mesh: more than 2^31-2 cells");
  c->has_mesh = c->has_stencils = c->has_blocks = false;
  c->N = n_cells;
  c->Nn = n_nodes;
  c->periodic = period != nullptr;
  for (int a = 0; a < d; ++a) {
    c->L[a] = period ? period[a] : 0.0;
    if (period && !(period[a] > 0)) fail(CWRECO_EINVAL, "set_mesh: period must be > 0");
  }
  for (int64_t i = 0; i < n_nodes * d; ++i)
    if (!std::isfinite(xyz[i])) fail(CWRECO_EMESH, "set_mesh: non-finite node coordinate");
  c->has_bc = false;
  c->bc_ids.clear();
  for (int a = 0; a < d; ++a) {
    c->box_lo[a] = c->box_hi[a] = xyz[a];
    for (int64_t n = 1; n < n_nodes; ++n) {
      c->box_lo[a] = std::min(c->box_lo[a], xyz[n * d + a]);
      c->box_hi[a] = std::max(c->box_hi[a], xyz[n * d + a]);
    }
  }

  const int64_t N = n_cells;
  std::vector<int64_t> cn(cells_in, cells_in + N * nv);
  std::vector<double> X(N * nv * d);
  int bad = 0;
  // unwrap (R16) + orientation fix (R28)
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (int64_t i = 0; i < N; ++i) {
    int64_t* v = &cn[i * nv];
    for (int k = 0; k < nv; ++k) {
      if (v[k] < 0 || v[k] >= n_nodes) { bad |= 1; continue; }
      for (int q = 0; q < k; ++q)
        if (v[q] == v[k]) bad |= 2;
    }
    if (bad) continue;
    double* x = &X[i * nv * d];
    for (int k = 0; k < nv; ++k)
      for (int a = 0; a < d; ++a) x[k * d + a] = xyz[v[k] * d + a];
    if (c->periodic) {
      for (int k = 1; k < nv; ++k)
        for (int a = 0; a < d; ++a) {
          const double Lh = 0.5 * c->L[a];
          double delta = x[k * d + a] - x[a];
          if (delta > Lh) x[k * d + a] = x[k * d + a] - c->L[a];
          else if (delta < -Lh) x[k * d + a] = x[k * d + a] + c->L[a];
        }
    }
    int s = cell_orientation(d, x);
    if (s == 0) { bad |= 4; continue; }
    if (s < 0) {
      std::swap(v[d - 1], v[d]);
      for (int a = 0; a < d; ++a) std::swap(x[(d - 1) * d + a], x[d * d + a]);
    }
  }
  if (bad & 1) fail(CWRECO_EINVAL, "set_mesh: cell references a missing node");
  if (bad & 2) fail(CWRECO_EMESH, "set_mesh: cell with repeated vertex");
  if (bad & 4) fail(CWRECO_EMESH, "set_mesh: zero-volume cell");

  // barycentres b = ((X0+X1)+X2[+X3])/(d+1), IEEE, left to right (R29)
  std::vector<double> B(N * d);
  const double inv = double(d + 1);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i)
    for (int a = 0; a < d; ++a) {
      const double* x = &X[i * nv * d];
      double s = x[0 * d + a] + x[1 * d + a];
      s = s + x[2 * d + a];
      if (d == 3) s = s + x[3 * d + a];
      B[i * d + a] = s / inv;
    }

  // Morton key (R29)
  const int kb = d == 2 ? 31 : 21;
  double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  if (!c->periodic) {
    for (int a = 0; a < d; ++a) { lo[a] = xyz[a]; hi[a] = xyz[a]; }
    for (int64_t n = 0; n < n_nodes; ++n)
      for (int a = 0; a < d; ++a) {
        lo[a] = std::min(lo[a], xyz[n * d + a]);
        hi[a] = std::max(hi[a], xyz[n * d + a]);
      }
  }
  std::vector<uint64_t> key(N);
  const double scale = double(1ull << kb);
  const double qmax = double((1ull << kb) - 1);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i) {
    uint64_t k = 0;
    for (int a = 0; a < d; ++a) {
      double u;
      if (c->periodic) {
        u = B[i * d + a] / c->L[a];
        u = u - std::floor(u);
      } else {
        u = (B[i * d + a] - lo[a]) / (hi[a] - lo[a]);
      }
      double q = std::floor(u * scale);
      if (q < 0) q = 0;
      if (q > qmax) q = qmax;
      k |= spread_bits((uint64_t)q, d, kb) << a;
    }
    key[i] = k;
  }
  std::vector<int64_t> perm(N);
  std::iota(perm.begin(), perm.end(), 0);
  __gnu_parallel::stable_sort(perm.begin(), perm.end(), [&](int64_t a, int64_t b) { return key[a] < key[b]; });

  c->perm = perm;
  c->cell_nodes.assign(N * nv, 0);
  c->X.assign(N * nv * d, 0);
  c->bary.assign(N * d, 0);
#pragma omp parallel for schedule(static)
  for (int64_t s = 0; s < N; ++s) {
    const int64_t i = perm[s];
    std::memcpy(&c->cell_nodes[s * nv], &cn[i * nv], sizeof(int64_t) * nv);
    std::memcpy(&c->X[s * nv * d], &X[i * nv * d], sizeof(double) * nv * d);
    std::memcpy(&c->bary[s * d], &B[i * d], sizeof(double) * d);
  }

  // face adjacency via sorted node tuples
  struct Face {
    int64_t n[3];
    int64_t cell;
    int f;
  };
  std::vector<Face> F(N * nv);
#pragma omp parallel for schedule(static)
  for (int64_t s = 0; s < N; ++s)
    for (int f = 0; f < nv; ++f) {
      Face& fc = F[s * nv + f];
      int q = 0;
      for (int k = 0; k < nv; ++k)
        if (k != f) fc.n[q++] = c->cell_nodes[s * nv + k];
      if (d == 2) fc.n[2] = -1;
      std::sort(fc.n, fc.n + d);
      fc.cell = s;
      fc.f = f;
    }
  auto less = [](const Face& a, const Face& b) {
    if (a.n[0] != b.n[0]) return a.n[0] < b.n[0];
    if (a.n[1] != b.n[1]) return a.n[1] < b.n[1];
    if (a.n[2] != b.n[2]) return a.n[2] < b.n[2];
    return a.cell < b.cell;
  };
  __gnu_parallel::sort(F.begin(), F.end(), less);
  auto same = [](const Face& a, const Face& b) { return a.n[0] == b.n[0] && a.n[1] == b.n[1] && a.n[2] == b.n[2]; };
  c->nbr.assign(N * nv, -1);
  for (size_t k = 0; k < F.size();) {
    size_t e = k + 1;
    while (e < F.size() && same(F[k], F[e])) ++e;
    if (e - k > 2) fail(CWRECO_EMESH, "set_mesh: non-manifold face (shared by > 2 cells)");
    if (e - k == 2) {
      if (F[k].cell == F[k + 1].cell) fail(CWRECO_EMESH, "set_mesh: degenerate cell");
      c->nbr[F[k].cell * nv + F[k].f] = F[k + 1].cell;
      c->nbr[F[k + 1].cell * nv + F[k + 1].f] = F[k].cell;
    }
    k = e;
  }
  // duplicate cells (same node set)
  {
    std::vector<std::array<int64_t, 4>> srt(N);
    for (int64_t s = 0; s < N; ++s) {
      std::array<int64_t, 4> t{-1, -1, -1, -1};
      for (int k = 0; k < nv; ++k) t[k] = c->cell_nodes[s * nv + k];
      std::sort(t.begin(), t.begin() + nv);
      srt[s] = t;
    }
    __gnu_parallel::sort(srt.begin(), srt.end());
    for (int64_t s = 1; s < N; ++s)
      if (srt[s] == srt[s - 1]) fail(CWRECO_EMESH, "set_mesh: duplicate cell");
  }
  // node -> cells CSR (ascending SFC ids)
  c->nc_ptr.assign(n_nodes + 1, 0);
  for (int64_t s = 0; s < N * nv; ++s) c->nc_ptr[c->cell_nodes[s] + 1]++;
  for (int64_t n = 0; n < n_nodes; ++n) c->nc_ptr[n + 1] += c->nc_ptr[n];
  c->nc_idx.assign(N * nv, 0);
  std::vector<int64_t> fill(c->nc_ptr.begin(), c->nc_ptr.end() - 1);
  for (int64_t s = 0; s < N; ++s)
    for (int k = 0; k < nv; ++k) c->nc_idx[fill[c->cell_nodes[s * nv + k]]++] = s;

  c->has_mesh = true;
  c->own_lo = (c->rank * N) / c->nranks;
  c->own_hi = ((c->rank + 1) * N) / c->nranks;
}

}  // namespace cwr
