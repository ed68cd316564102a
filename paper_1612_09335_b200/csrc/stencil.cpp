// Central and sectorial CWENO stencils with exact predicates,
// then ghosts and the local numbering (owned interior | owned boundary | ghosts).
//
// Readings: R11 face neighbours drive the recursion (node neighbours
// only as the sector fallback), R12 layers sorted by (squared barycentre
// distance, SFC id) with the last layer truncated, R13 open cone of owner vertex
// v = {λ_w > 0 ∀ w ≠ v}, R14 sector fallback / invalid sectors, R16 periodic
// minimum image chosen by the IEEE recipe on barycentres.
//
// Every geometric decision is exact for the given doubles: an interval filter
// certifies the sign in double precision, otherwise expansion arithmetic decides.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "exact.hpp"
#include "internal.hpp"

namespace cwr {

// ---------------------------------------------------------------- boundary ghosts (R37)
// Ghost id N + s·N + k is the mirror image of real cell k across box side s (plane
// x_a = c, a = s / 2): vertices X'_a = c + (c − X_a) (IEEE double), last two swapped
// (orientation, R28).  A real boundary face lying exactly on an active side s borders
// the mirror of its own cell; a ghost's faces border the mirrors (same side) of its
// source's face neighbours, its mirrored face on s borders the source, and faces on
// other sides border nothing (no double reflection).
static double side_plane(const cwreco_ctx* c, int s) { return (s & 1) ? c->box_hi[s / 2] : c->box_lo[s / 2]; }

static int face_side(const cwreco_ctx* c, int64_t k, int f) {
  if (!c->has_bc) return -1;
  const int d = c->d;
  const double* X = &c->X[k * (d + 1) * d];
  for (int s = 0; s < 2 * d; ++s) {
    if (!c->bc[s]) continue;
    const int a = s / 2;
    const double pl = side_plane(c, s);
    bool on = true;
    for (int v = 0; v <= d && on; ++v)
      if (v != f) on = X[v * d + a] == pl;
    if (on) return s;
  }
  return -1;
}

const double* cell_X(const cwreco_ctx* c, int64_t j, double* buf) {
  const int d = c->d;
  if (j < c->N) return &c->X[j * (d + 1) * d];
  const int64_t s = (j - c->N) / c->N, k = (j - c->N) % c->N;
  const int a = int(s / 2);
  const double pl = side_plane(c, int(s));
  const double* X = &c->X[k * (d + 1) * d];
  for (int v = 0; v <= d; ++v) {
    const int src = v == d - 1 ? d : v == d ? d - 1 : v;  // last two swapped
    for (int e = 0; e < d; ++e) buf[v * d + e] = e == a ? pl + (pl - X[src * d + e]) : X[src * d + e];
  }
  return buf;
}

void cell_bary(const cwreco_ctx* c, int64_t j, double* out) {
  const int d = c->d;
  if (j < c->N) {
    for (int a = 0; a < d; ++a) out[a] = c->bary[j * d + a];
    return;
  }
  double buf[12];
  const double* X = cell_X(c, j, buf);
  for (int a = 0; a < d; ++a) {  // R29 order
    double s = X[a] + X[d + a];
    s = s + X[2 * d + a];
    if (d == 3) s = s + X[3 * d + a];
    out[a] = s / double(d + 1);
  }
}

int cell_neighbours(const cwreco_ctx* c, int64_t j, int64_t* out) {
  const int d = c->d;
  const int64_t N = c->N;
  int n = 0;
  if (j < N) {
    for (int f = 0; f <= d; ++f) {
      const int64_t nb = c->nbr[j * (d + 1) + f];
      if (nb >= 0) {
        out[n++] = nb;
      } else {
        const int s = face_side(c, j, f);
        if (s >= 0) out[n++] = N + s * N + j;
      }
    }
    return n;
  }
  const int64_t s = (j - N) / N, k = (j - N) % N;
  for (int f = 0; f <= d; ++f) {
    const int64_t nb = c->nbr[k * (d + 1) + f];
    if (nb >= 0)
      out[n++] = N + s * N + nb;
    else if (face_side(c, k, f) == s)
      out[n++] = k;
  }
  return n;
}

namespace {

constexpr double U = 1.1102230246251565e-16;  // 2^-53

// value with an absolute error radius (sound filter for sign decisions)
struct IV {
  double v, r;
};
inline IV iv_add(IV a, IV b) {
  double s = a.v + b.v;
  return {s, (a.r + b.r + U * std::fabs(s)) * (1 + 4 * U)};
}
inline IV iv_sub(IV a, IV b) { return iv_add(a, {-b.v, b.r}); }
inline IV iv_mul(IV a, IV b) {
  double p = a.v * b.v;
  return {p, (std::fabs(a.v) * b.r + std::fabs(b.v) * a.r + a.r * b.r + U * std::fabs(p)) * (1 + 4 * U)};
}
inline IV iv_exact(double x) { return {x, 0.0}; }

IV iv_orient(int d, const IV* const* p) {
  if (d == 2) {
    IV ax = iv_sub(p[1][0], p[0][0]), ay = iv_sub(p[1][1], p[0][1]);
    IV bx = iv_sub(p[2][0], p[0][0]), by = iv_sub(p[2][1], p[0][1]);
    return iv_sub(iv_mul(ax, by), iv_mul(ay, bx));
  }
  IV u[3], v[3], w[3];
  for (int k = 0; k < 3; ++k) {
    u[k] = iv_sub(p[1][k], p[0][k]);
    v[k] = iv_sub(p[2][k], p[0][k]);
    w[k] = iv_sub(p[3][k], p[0][k]);
  }
  IV c0 = iv_sub(iv_mul(v[1], w[2]), iv_mul(v[2], w[1]));
  IV c1 = iv_sub(iv_mul(v[2], w[0]), iv_mul(v[0], w[2]));
  IV c2 = iv_sub(iv_mul(v[0], w[1]), iv_mul(v[1], w[0]));
  return iv_add(iv_add(iv_mul(u[0], c0), iv_mul(u[1], c1)), iv_mul(u[2], c2));
}

// Geometry of one owner cell i, in coordinates scaled by (d+1) and centred on
// the owner's barycentre: W_k = (d+1) X_{i,k} − S_i, and for a cell j
// D_j = S_j + (d+1) n L − S_i  (S_c = Σ_k X_{c,k}; n the periodic image shift).
struct ExData {  // exact displacement and squared distance of one candidate
  exact::Ex De[3];
  exact::Ex keye;
};

struct Owner {
  const cwreco_ctx* c;
  int d;
  int64_t i;
  IV Wiv[4][3];
  exact::Ex Si[3];
  exact::Ex W[4][3];
  bool have_exactW = false;
  std::vector<ExData> pool;  // exact data of candidates that needed it

  Owner(const cwreco_ctx* c_, int64_t i_) : c(c_), d(c_->d), i(i_) {
    const double* X = &c->X[i * (d + 1) * d];
    for (int a = 0; a < d; ++a) {
      IV s = iv_exact(X[a]);
      for (int k = 1; k <= d; ++k) s = iv_add(s, iv_exact(X[k * d + a]));
      for (int k = 0; k <= d; ++k) Wiv[k][a] = iv_sub(iv_mul(iv_exact(double(d + 1)), iv_exact(X[k * d + a])), s);
    }
  }
  void ensure_exactW() {
    if (have_exactW) return;
    const double* X = &c->X[i * (d + 1) * d];
    for (int a = 0; a < d; ++a) {
      exact::Ex s;
      for (int k = 0; k <= d; ++k) s = exact::grow(s, X[k * d + a]);
      Si[a] = exact::compress(s);
      for (int k = 0; k <= d; ++k) W[k][a] = exact::sub(exact::scale(exact::Ex(X[k * d + a]), double(d + 1)), Si[a]);
    }
    have_exactW = true;
  }
};

struct Cand {
  int64_t j;
  int n[3];     // periodic shift
  IV D[3];      // filter value of D_j
  IV key;       // Σ D_a²
  int ex = -1;  // index into Owner::pool once the exact values were needed
  int8_t lam[4] = {2, 2, 2, 2};  // cached signs of the owner barycentric coordinates (2 = unknown)
};

void shift_of(const cwreco_ctx* c, int64_t i, int64_t j, int* n) {
  const int d = c->d;
  for (int a = 0; a < d; ++a) {
    n[a] = 0;
    if (!c->periodic) continue;
    const double L = c->L[a];
    double r = c->bary[j * d + a] - c->bary[i * d + a];
    while (r > 0.5 * L) { r -= L; n[a] -= 1; }
    while (r < -0.5 * L) { r += L; n[a] += 1; }
  }
}

void make_cand(Owner& o, int64_t j, Cand& cd) {
  const cwreco_ctx* c = o.c;
  const int d = o.d;
  cd.j = j;
  cd.ex = -1;
  shift_of(c, o.i, j, cd.n);
  const double* Xi = &c->X[o.i * (d + 1) * d];
  double xb[12];
  const double* Xj = cell_X(c, j, xb);
  IV key{0.0, 0.0};
  for (int a = 0; a < d; ++a) {
    IV sj = iv_exact(Xj[a]), si = iv_exact(Xi[a]);
    for (int k = 1; k <= d; ++k) {
      sj = iv_add(sj, iv_exact(Xj[k * d + a]));
      si = iv_add(si, iv_exact(Xi[k * d + a]));
    }
    IV sh = iv_mul(iv_exact(double((d + 1) * cd.n[a])), iv_exact(c->periodic ? c->L[a] : 0.0));
    cd.D[a] = iv_sub(iv_add(sj, sh), si);
    key = a == 0 ? iv_mul(cd.D[a], cd.D[a]) : iv_add(key, iv_mul(cd.D[a], cd.D[a]));
  }
  cd.key = key;
}

const ExData& ensure_exact(Owner& o, Cand& cd) {
  if (cd.ex >= 0) return o.pool[cd.ex];
  o.ensure_exactW();
  const cwreco_ctx* c = o.c;
  const int d = o.d;
  double xb[12];
  const double* Xj = cell_X(c, cd.j, xb);
  ExData x;
  for (int a = 0; a < d; ++a) {
    exact::Ex s;
    for (int k = 0; k <= d; ++k) s = exact::grow(s, Xj[k * d + a]);
    s = exact::compress(s);
    if (c->periodic && cd.n[a] != 0) s = exact::add(s, exact::scale(exact::Ex(c->L[a]), double((d + 1) * cd.n[a])));
    x.De[a] = exact::sub(s, o.Si[a]);
    x.keye = exact::add(x.keye, exact::mul(x.De[a], x.De[a]));
  }
  cd.ex = (int)o.pool.size();
  o.pool.push_back(x);
  return o.pool[cd.ex];
}

// strict-weak "less" by (exact squared distance, id)
bool key_less(Owner& o, Cand& a, Cand& b) {
  IV df = iv_sub(a.key, b.key);
  if (std::fabs(df.v) > df.r) return df.v < 0;
  ensure_exact(o, a);
  ensure_exact(o, b);
  int s = exact::sign(exact::sub(o.pool[a.ex].keye, o.pool[b.ex].keye));
  if (s != 0) return s < 0;
  return a.j < b.j;
}

// sign of the owner barycentric coordinate λ_w at D (orientation with W_w -> D)
int lambda_sign(Owner& o, Cand& cd, int w) {
  if (cd.lam[w] != 2) return cd.lam[w];
  const int d = o.d;
  const IV* p[4];
  for (int k = 0; k <= d; ++k) p[k] = (k == w) ? cd.D : o.Wiv[k];
  IV det = iv_orient(d, p);
  int sg;
  if (std::fabs(det.v) > det.r) {
    sg = det.v > 0 ? 1 : -1;
  } else {
    const ExData& x = ensure_exact(o, cd);
    const exact::Ex* pe[4];
    for (int k = 0; k <= d; ++k) pe[k] = (k == w) ? x.De : o.W[k];
    sg = exact::orient_sign(d, pe);
  }
  cd.lam[w] = (int8_t)sg;
  return sg;
}

bool in_cone(Owner& o, Cand& cd, int v) {  // R13: λ_w > 0 for all w != v
  for (int w = 0; w <= o.d; ++w) {
    if (w == v) continue;
    if (lambda_sign(o, cd, w) <= 0) return false;
  }
  return true;
}

// candidate cache of one owner (shared by the central and the d+1 sector searches)
struct Cache {
  Owner& o;
  std::vector<Cand> cs;
  explicit Cache(Owner& o_) : o(o_) { cs.reserve(256); }
  int get(int64_t j) {
    for (size_t q = 0; q < cs.size(); ++q)
      if (cs[q].j == j) return (int)q;
    cs.emplace_back();
    make_cand(o, j, cs.back());
    return (int)cs.size() - 1;
  }
  void sort(std::vector<int>& idx) {
    std::sort(idx.begin(), idx.end(), [&](int a, int b) { return key_less(o, cs[a], cs[b]); });
  }
};

bool affinely_independent(Cache& cc, const std::vector<int>& idx) {
  Owner& o = cc.o;
  const int d = o.d;
  IV zero[3] = {{0, 0}, {0, 0}, {0, 0}};
  const IV* p[4];
  p[0] = zero;
  for (int k = 0; k < d; ++k) p[k + 1] = cc.cs[idx[k]].D;
  IV det = iv_orient(d, p);
  if (std::fabs(det.v) > det.r) return true;
  exact::Ex ze[3];
  const exact::Ex* pe[4];
  pe[0] = ze;
  for (int k = 0; k < d; ++k) ensure_exact(o, cc.cs[idx[k]]);  // pool may grow: take pointers after
  for (int k = 0; k < d; ++k) pe[k + 1] = o.pool[cc.cs[idx[k]].ex].De;
  return exact::orient_sign(d, pe) != 0;
}

inline bool contains(const std::vector<int64_t>& v, int64_t x) {
  return std::find(v.begin(), v.end(), x) != v.end();
}

// returns false if exhausted
bool central_stencil(Cache& cc, int32_t* out) {
  const cwreco_ctx* c = cc.o.c;
  const int d = c->d, ne = c->ne;
  const int64_t i = cc.o.i;
  std::vector<int64_t> S{i}, frontier{i}, cand;
  std::vector<int> idx;
  while ((int)S.size() < ne) {
    cand.clear();
    for (int64_t f : frontier) {
      int64_t nbs[4];
      const int nn = cell_neighbours(c, f, nbs);
      for (int k = 0; k < nn; ++k)
        if (!contains(S, nbs[k]) && !contains(cand, nbs[k])) cand.push_back(nbs[k]);
    }
    if (cand.empty()) return false;
    idx.clear();
    for (int64_t x : cand) idx.push_back(cc.get(x));
    cc.sort(idx);
    const size_t take = std::min(idx.size(), size_t(ne) - S.size());
    frontier.clear();
    for (size_t q = 0; q < take; ++q) {
      S.push_back(cc.cs[idx[q]].j);
      frontier.push_back(cc.cs[idx[q]].j);
    }
  }
  for (int k = 0; k < ne; ++k) out[k] = (int32_t)S[k];
  return true;
}

bool in_cone_idx(Cache& cc, int q, int v) { return in_cone(cc.o, cc.cs[q], v); }

// P:156 + R14.  out: d+1 entries (self first, -1 padded); returns validity.
bool sector_stencil(Cache& cc, int v, int32_t* out) {
  const cwreco_ctx* c = cc.o.c;
  const int d = c->d;
  const int64_t i = cc.o.i;
  std::vector<int64_t> S{i}, seen{i}, frontier{i}, cand;
  std::vector<int> taken, acc;
  while ((int)S.size() < d + 1) {
    cand.clear();
    for (int64_t f : frontier) {
      int64_t nbs[4];
      const int nn = cell_neighbours(c, f, nbs);
      for (int k = 0; k < nn; ++k)
        if (!contains(seen, nbs[k]) && !contains(cand, nbs[k])) cand.push_back(nbs[k]);
    }
    for (int64_t x : cand) seen.push_back(x);
    acc.clear();
    for (int64_t x : cand) {
      const int q = cc.get(x);
      if (in_cone_idx(cc, q, v)) acc.push_back(q);
    }
    if (acc.empty()) {
      // fallback: node (Voronoi) neighbours of all selected sector cells
      cand.clear();
      for (int64_t s : S) {
        if (s >= c->N) continue;  // ghosts contribute no node neighbours (R37)
        const int64_t* nd = &c->cell_nodes[s * (d + 1)];
        for (int k = 0; k <= d; ++k)
          for (int64_t q = c->nc_ptr[nd[k]]; q < c->nc_ptr[nd[k] + 1]; ++q) {
            int64_t x = c->nc_idx[q];
            if (!contains(S, x) && !contains(cand, x)) cand.push_back(x);
          }
      }
      for (int64_t x : cand) {
        const int q = cc.get(x);
        if (in_cone_idx(cc, q, v)) acc.push_back(q);
      }
      if (acc.empty()) break;
    }
    cc.sort(acc);
    const size_t take = std::min(acc.size(), size_t(d + 1) - S.size());
    frontier.clear();
    for (size_t q = 0; q < take; ++q) {
      const int64_t j = cc.cs[acc[q]].j;
      S.push_back(j);
      if (!contains(seen, j)) seen.push_back(j);
      frontier.push_back(j);
      taken.push_back(acc[q]);
    }
  }
  for (int k = 0; k <= d; ++k) out[k] = k < (int)S.size() ? (int32_t)S[k] : -1;
  if ((int)S.size() < d + 1) return false;
  return affinely_independent(cc, taken);
}

int owner_rank(const cwreco_ctx* c, int64_t g) {
  // rank r owns [floor(r N / P), floor((r+1) N / P))
  int r = int((g * c->nranks) / c->N);
  while (r > 0 && (r * c->N) / c->nranks > g) --r;
  while (r + 1 < c->nranks && ((r + 1) * c->N) / c->nranks <= g) ++r;
  return r;
}

}  // namespace

void build_stencils(cwreco_ctx* c) {
  if (!c->has_mesh) fail(CWRECO_ESTATE, "build_stencils: no mesh");
  if (c->has_bc && c->nranks > 1)
    fail(CWRECO_EUNSUPPORTED, "build_stencils: boundary ghost cells are supported on one rank");
  const int d = c->d, ne = c->ne, nv = d + 1;
  const int64_t lo = c->own_lo, hi = c->own_hi, n_own = hi - lo;
  c->central.assign(n_own * ne, -1);
  c->sectors.assign(n_own * nv * nv, -1);
  c->valid.assign(n_own * nv, 0);
  int64_t exhausted = -1;
  std::string err;
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t q = 0; q < n_own; ++q) {
    const int64_t i = lo + q;
    try {
      Owner o(c, i);
      Cache cc(o);
      if (!central_stencil(cc, &c->central[q * ne])) {
#pragma omp critical
        exhausted = std::max<int64_t>(exhausted, i);
        continue;
      }
      for (int v = 0; v < nv; ++v)
        c->valid[q * nv + v] = sector_stencil(cc, v, &c->sectors[(q * nv + v) * nv]) ? 1 : 0;
    } catch (const std::exception& e) {
#pragma omp critical
      err = e.what();
    }
  }
  if (!err.empty()) fail(CWRECO_EINVAL, "build_stencils: " + err);
  if (exhausted >= 0)
    fail(CWRECO_ESTENCIL, "build_stencils: central stencil exhausted (cell " + std::to_string(exhausted) + ")");

  finalize_stencils(c);
}

// Ghosts, interior/boundary split, local numbering, extras and gather length of the
// stencils in c->central / c->sectors / c->valid (built or uploaded).
void finalize_stencils(cwreco_ctx* c) {
  const int d = c->d, ne = c->ne, nv = d + 1;
  const int64_t lo = c->own_lo, hi = c->own_hi, n_own = hi - lo;
  std::vector<uint8_t> is_bnd(n_own, 0);
  std::vector<int64_t> ghosts;
  std::vector<int64_t> bcg;
  for (int64_t q = 0; q < n_own; ++q) {
    bool b = false;
    for (int k = 0; k < ne; ++k) {
      int64_t g = c->central[q * ne + k];
      if (g >= c->N) bcg.push_back(g);
      else if (g < lo || g >= hi) { b = true; ghosts.push_back(g); }
    }
    for (int k = 0; k < nv * nv; ++k) {
      int64_t g = c->sectors[q * nv * nv + k];
      if (g >= c->N) bcg.push_back(g);
      else if (g >= 0 && (g < lo || g >= hi)) { b = true; ghosts.push_back(g); }
    }
    is_bnd[q] = b;
  }
  std::sort(bcg.begin(), bcg.end());
  bcg.erase(std::unique(bcg.begin(), bcg.end()), bcg.end());
  c->bc_ids = bcg;
  std::sort(ghosts.begin(), ghosts.end());
  ghosts.erase(std::unique(ghosts.begin(), ghosts.end()), ghosts.end());
  c->n_owned = n_own;
  c->n_ghost = (int64_t)ghosts.size();
  c->local2global.clear();
  c->local2global.reserve(n_own + c->n_ghost);
  for (int64_t q = 0; q < n_own; ++q)
    if (!is_bnd[q]) c->local2global.push_back(lo + q);
  c->n_interior = (int64_t)c->local2global.size();
  for (int64_t q = 0; q < n_own; ++q)
    if (is_bnd[q]) c->local2global.push_back(lo + q);
  for (int64_t g : ghosts) c->local2global.push_back(g);
  c->ghost_counts.assign(c->nranks, 0);
  for (int64_t g : ghosts) c->ghost_counts[owner_rank(c, g)]++;
  c->send_counts.assign(c->nranks, 0);
  c->send_local.clear();

  // extras (sector cells outside the central stencil, R15) and invalid sectors
  int64_t n_extra = 0, n_inv = 0;
  int max_extra = 0;
  for (int64_t q = 0; q < n_own; ++q) {
    int ex = 0;
    std::vector<int32_t> seen;
    for (int k = 0; k < nv * nv; ++k) {
      int32_t g = c->sectors[q * nv * nv + k];
      if (g < 0) continue;
      bool in = false;
      for (int m = 0; m < ne && !in; ++m) in = c->central[q * ne + m] == g;
      if (!in && std::find(seen.begin(), seen.end(), g) == seen.end()) { seen.push_back(g); ++ex; }
    }
    n_extra += ex;
    max_extra = std::max(max_extra, ex);
    for (int v = 0; v < nv; ++v) n_inv += c->valid[q * nv + v] ? 0 : 1;
  }
  c->n_extra = n_extra;
  c->n_invalid = n_inv;
  // gather positions: sector cells first ((d+1)·d slots), then the rest of S_i^0 (R15)
  c->G = std::max(nv * d, (ne - 1) + max_extra);
  c->has_stencils = true;
  c->has_blocks = false;
}

void install_send_lists(cwreco_ctx* c, const int64_t* send_counts, const int64_t* send_ids) {
  int64_t tot = 0;
  for (int r = 0; r < c->nranks; ++r) {
    if (send_counts[r] < 0) fail(CWRECO_EINVAL, "set_send_lists: negative count");
    tot += send_counts[r];
  }
  if (tot > 0 && !send_ids) fail(CWRECO_EINVAL, "set_send_lists: NULL ids");
  std::vector<int32_t> own2local(c->own_hi - c->own_lo, -1);
  for (int64_t li = 0; li < c->n_owned; ++li) own2local[c->local2global[li] - c->own_lo] = (int32_t)li;
  std::vector<int64_t> loc(tot);
  for (int64_t k = 0; k < tot; ++k) {
    const int64_t g = send_ids[k];
    if (g < c->own_lo || g >= c->own_hi) fail(CWRECO_EINVAL, "set_send_lists: id not owned by this rank");
    loc[k] = own2local[g - c->own_lo];
  }
  c->send_counts.assign(send_counts, send_counts + c->nranks);
  c->send_local = loc;
  dev_set_send(c);
}

}  // namespace cwr
