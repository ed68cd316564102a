// Per-cell reconstruction matrices (Eulerian pre-processing) packed into
// the tiled HBM stream consumed by the kernels.
//
//  A[k][l] = average over stencil cell j(k) (periodic image nearest the owner) of
//            ψ_l(ξ_i(x)), the basis in the OWNER's reference coordinates;
//            collapsed Gauss-Legendre quadrature exact for degree M (R19).
//  Constrained LSQ (R10): the owner row fixes p̂_1 = Q_i/ψ_1 (only ψ_1
//  has a non-zero mean on T_E), leaving the reduced problem
//      min ‖A[1:,1:] p − (Q_j − Q_i)‖₂,
//  whose pseudo-inverse B⁺ = R⁻¹Qᵀ comes from a Householder QR.
//  Sectors: the linear modes averaged over a cell equal their value at
//  the cell barycentre, so A_s[m][l] = ψ_{l+1}(ξ_i(b_{j_m})); S_s = A_s⁻¹ (d×d).
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <unordered_map>

#include "internal.hpp"

namespace cwr {

static inline int64_t r16(int64_t x) { return (x + 15) & ~int64_t(15); }

static Layout layout_with(int d, int M, int V, int G, int T, int KC, int Umax, int kind, int nsc = 1) {
  Layout L;
  L.kind = kind;
  L.VP = kind == KIND_ROWBLK ? V + (V & 1) : V;
  L.d = d;
  L.M = M;
  L.V = V;
  L.nm = n_modes(M, d);
  L.R = L.nm - 1;
  L.K = d * L.nm - 1;
  L.G = G;
  L.T = T;
  L.KC = KC;
  L.Umax = Umax;
  L.kslice_bytes = int64_t(T) * L.R * 8;
  L.NCH = (G + KC - 1) / KC;
  L.off_idx = r16(int64_t(Umax) * 4);
  L.idx_bytes = r16(int64_t(kind == KIND_ROWBLK ? (G + 1) & ~1 : G) * T * 2);
  L.u_bytes = L.off_idx + L.idx_bytes;
  L.ids_bytes = 0;
  L.chunk_bytes = int64_t(KC) * L.kslice_bytes;
  L.off_sector = r16(L.off_chunk(L.NCH - 1) + L.chunk_size(L.NCH - 1));
  L.NSC = nsc;
  L.TSC = (T + nsc - 1) / nsc;
  L.srec = (d + 1) * d * d + (kind == KIND_ROWBLK ? L.R : 0);
  L.sinv_bytes = int64_t(L.TSC) * L.srec * 8;
  L.sector_bytes = r16(L.sinv_bytes + L.TSC);
  L.tile_bytes = L.off_sector + nsc * L.sector_bytes;
  return L;
}

void rowblk_plan(const Layout& L, int max_smem, int max_ctas, int& ctas, int& stages) {
  // one warp-specialised CTA per SM: the deepest stage ring that fits
  (void)max_ctas;
  ctas = 0;
  stages = 0;
  for (int s = kRbMaxStages; s >= kRbMinStages; --s)
    if (rb_smem(L, s) <= max_smem) {
      ctas = 1;
      stages = s;
      return;
    }
}

Layout make_layout(int d, int M, int V, int G, int max_smem, const std::function<int(int)>& umax_for,
                   int family, int max_tile) {
  auto capped = [&](int T) { return max_tile > 0 && T > max_tile ? std::max(2, max_tile & ~1) : T; };
  const int nm = n_modes(M, d);
  // family (cwreco_set_option CWRECO_OPT_FAMILY): -1 = default, 0 = cell-variable,
  // 1 = row-block where instantiated
  const bool want_rb = family >= 0 ? family == 1 : rb_default(d, nm - 1, V);
  if (want_rb && rowblk_supported(d, M, V)) {
    // k_rowblk: T = consumers / NG cells per tile (halved while the CTA does not fit);
    // KC positions per chunk: ~10 KB of B⁺ per stage, KC ∈ {1, 2, 4} (compiled sizes)
    const int R = nm - 1;
    // T even: a position slice T·R doubles must stay a multiple of 16 bytes (TMA bulk sizes)
    for (int T = capped(rb_tfull(R, V)); T >= 2; T = (T / 2) & ~1) {
      // the whole sector chunk of a tile goes to its own buffer: one piece
      Layout L = layout_with(d, M, V, G, T, kRbKC, umax_for(T), KIND_ROWBLK, 1);
      int ctas, stages;
      rowblk_plan(L, max_smem, 1, ctas, stages);
      if (ctas > 0) return L;
    }
  }
  // one tile = T cells × V variables = one consumer thread each
  int T0 = (cons_threads(nm) / V) & ~1;
  if (T0 < 2) T0 = 2;
  T0 = capped(T0);
  // positions per streamed chunk: ~10 KB of B⁺ per chunk (measured best: larger
  // chunks lengthen the gather bursts, smaller ones add per-chunk synchronisation),
  // even (the kernel reads position pairs with 16-byte shared loads), a compiled
  // size (1-6, 8), such that the chunks holding the (d+1)·d sector positions are
  // full (their ΔQ is captured with static indices) and kMinStages stages fit.
  // A tile whose sector chunk alone is too large (small ℳ, V = 1) is halved.
  const int64_t budget = pipe_budget(nm, max_smem);
#ifdef CWRECO_EXPERIMENTS
  const char* force = std::getenv("CWRECO_KC");  // tuning experiments only (tools/sweep.py)
#else
  const char* force = nullptr;
#endif
  Layout best;
  bool found = false;
  for (int T = T0; T >= 2; T = (T / 2) & ~1) {
    const int Umax = umax_for(T);
    const int64_t kslice = int64_t(T) * (nm - 1) * 8;
    int want = std::max<int>(1, int(10240 / kslice));
    want = std::min(want, 8);
    want = (want + 1) & ~1;
    if (want == 7) want = 6;
    for (int KC = force ? std::atoi(force) : want; KC >= 1; --KC) {
      if (KC == 7 || KC > G || ((d + 1) * d + KC - 1) / KC * KC > G) continue;
      Layout L = layout_with(d, M, V, G, T, KC, Umax, KIND_CELLVAR);
      if (pipe_smem(L, kMinStages) <= budget) return L;
      if (!found || pipe_smem(L, kMinStages) < pipe_smem(best, kMinStages)) best = L, found = true;
    }
  }
  return best;
}

namespace {

void shift_of(const cwreco_ctx* c, int64_t i, int64_t j, double* sh) {
  const int d = c->d;
  for (int a = 0; a < d; ++a) {
    int n = 0;
    if (c->periodic) {
      const double L = c->L[a];
      double r = c->bary[j * d + a] - c->bary[i * d + a];
      while (r > 0.5 * L) { r -= L; n -= 1; }
      while (r < -0.5 * L) { r += L; n += 1; }
    }
    sh[a] = c->periodic ? n * c->L[a] : 0.0;
  }
}

bool inv_small(int d, const double* A, double* Ainv) {
  if (d == 2) {
    double det = A[0] * A[3] - A[1] * A[2];
    if (det == 0.0 || !std::isfinite(det)) return false;
    Ainv[0] = A[3] / det;
    Ainv[1] = -A[1] / det;
    Ainv[2] = -A[2] / det;
    Ainv[3] = A[0] / det;
    return true;
  }
  double c00 = A[4] * A[8] - A[5] * A[7], c01 = A[5] * A[6] - A[3] * A[8], c02 = A[3] * A[7] - A[4] * A[6];
  double det = A[0] * c00 + A[1] * c01 + A[2] * c02;
  if (det == 0.0 || !std::isfinite(det)) return false;
  Ainv[0] = c00 / det;
  Ainv[1] = (A[2] * A[7] - A[1] * A[8]) / det;
  Ainv[2] = (A[1] * A[5] - A[2] * A[4]) / det;
  Ainv[3] = c01 / det;
  Ainv[4] = (A[0] * A[8] - A[2] * A[6]) / det;
  Ainv[5] = (A[2] * A[3] - A[0] * A[5]) / det;
  Ainv[6] = c02 / det;
  Ainv[7] = (A[1] * A[6] - A[0] * A[7]) / det;
  Ainv[8] = (A[0] * A[4] - A[1] * A[3]) / det;
  return true;
}

// Householder QR of Ared (m×n, column-major, overwritten), returns B⁺ = R⁻¹Q₁ᵀ
// (n×m, row-major).  Q₁ is accumulated explicitly (backward), then one triangular
// solve per column.
bool pinv_qr(int m, int n, std::vector<double>& A, std::vector<double>& Bp, double& cond) {
  thread_local std::vector<double> V, beta, Q1;
  V.assign(size_t(m) * n, 0.0);
  beta.assign(n, 0.0);
  double rmax = 0.0, rmin = 1e300;
  for (int j = 0; j < n; ++j) {
    double* a = &A[size_t(j) * m];
    double nrm = 0.0;
    for (int r = j; r < m; ++r) nrm += a[r] * a[r];
    nrm = std::sqrt(nrm);
    if (nrm == 0.0) return false;
    const double alpha = a[j] > 0 ? -nrm : nrm;
    double* v = &V[size_t(j) * m];
    for (int r = j; r < m; ++r) v[r] = a[r];
    v[j] -= alpha;
    double vn = 0.0;
    for (int r = j; r < m; ++r) vn += v[r] * v[r];
    beta[j] = vn > 0 ? 2.0 / vn : 0.0;
    a[j] = alpha;
    for (int r = j + 1; r < m; ++r) a[r] = 0.0;
    for (int cidx = j + 1; cidx < n; ++cidx) {
      double* ac = &A[size_t(cidx) * m];
      double s = 0.0;
      for (int r = j; r < m; ++r) s += v[r] * ac[r];
      s *= beta[j];
      for (int r = j; r < m; ++r) ac[r] -= s * v[r];
    }
    rmax = std::max(rmax, std::fabs(alpha));
    rmin = std::min(rmin, std::fabs(alpha));
  }
  if (!(rmin > 1e-12 * rmax)) return false;
  cond = rmax / rmin;
  // Q₁ = H_0 H_1 … H_{n-1} [I_n; 0]  (m×n, column-major)
  Q1.assign(size_t(m) * n, 0.0);
  for (int c = 0; c < n; ++c) Q1[size_t(c) * m + c] = 1.0;
  for (int j = n - 1; j >= 0; --j) {
    const double* v = &V[size_t(j) * m];
    for (int c = j; c < n; ++c) {
      double* q = &Q1[size_t(c) * m];
      double s = 0.0;
      for (int r = j; r < m; ++r) s += v[r] * q[r];
      s *= beta[j];
      for (int r = j; r < m; ++r) q[r] -= s * v[r];
    }
  }
  // B⁺ = R⁻¹ Q₁ᵀ: for each k solve R x = (Q₁ᵀ)_{:,k}
  Bp.assign(size_t(n) * m, 0.0);
  for (int k = 0; k < m; ++k) {
    for (int j = n - 1; j >= 0; --j) {
      double s = Q1[size_t(j) * m + k];
      for (int q = j + 1; q < n; ++q) s -= A[size_t(q) * m + j] * Bp[size_t(q) * m + k];
      Bp[size_t(j) * m + k] = s / A[size_t(j) * m + j];
    }
  }
  return true;
}

}  // namespace

namespace {

// Gather order of owned local cell li (precompute's layout):
// positions s·d+m hold member m of sector s (invalid sectors: other S_i^0 cells,
// else the cell itself), then the rest of S_i^0; lid[p] local ids (padded with
// the cell itself up to G), col[p] = B⁺ column (index into S_i^0 ∖ i) or -1.
// Returns the number of positions used, -1 if a cell is missing locally.
template <class ToLocal>
int gather_order(const cwreco_ctx* c, int64_t li, int G, const ToLocal& to_local, int32_t* lid, int* col) {
  const int d = c->d, ne = c->ne, nv = d + 1;
  const int64_t g = c->local2global[li];
  const int64_t q = g - c->own_lo;
  const int32_t* cen = &c->central[q * ne];
  const int32_t* sec = &c->sectors[q * nv * nv];
  const uint8_t* val = &c->valid[q * nv];
  int64_t gglob[256];
  bool used[256] = {false};
  const int front = nv * d;
  for (int p = 0; p < front; ++p) { gglob[p] = -1; col[p] = -1; }
  for (int s = 0; s < nv; ++s) {
    if (!val[s]) continue;
    for (int m = 0; m < d; ++m) {
      const int64_t x = sec[s * nv + 1 + m];
      gglob[s * d + m] = x;
      for (int k = 1; k < ne; ++k)
        if (cen[k] == x) { col[s * d + m] = k - 1; used[k] = true; break; }
    }
  }
  int ng = front, next = 1;  // next unused central cell for invalid-sector fillers
  for (int p = 0; p < front; ++p) {
    if (gglob[p] >= 0) continue;
    while (next < ne && used[next]) ++next;
    if (next < ne) {
      gglob[p] = cen[next];
      col[p] = next - 1;
      used[next] = true;
    } else {
      gglob[p] = g;  // self: ΔQ = 0
    }
  }
  for (int k = 1; k < ne; ++k)
    if (!used[k]) { gglob[ng] = cen[k]; col[ng] = k - 1; ++ng; }
  if (ng > G) return -1;
  for (int p = 0; p < G; ++p) {
    lid[p] = (int32_t)li;
    if (p < ng && gglob[p] != g) {
      lid[p] = to_local(gglob[p]);
      if (lid[p] < 0) return -1;
    }
    if (p >= ng) col[p] = -1;
  }
  return ng;
}

// Stencil union of tile t (tiles of T cells): own cells [t·T, min((t+1)·T, n_owned))
// first (padded with the tile's first cell up to T), then the other gathered cells
// ascending.  Returns false if a gather list is invalid.
template <class ToLocal>
bool tile_union(const cwreco_ctx* c, int64_t t, int T, int G, const ToLocal& to_local, std::vector<int32_t>& u) {
  const int64_t lo = t * T, hi = std::min(c->n_owned, lo + T);
  std::vector<int32_t> others;
  int32_t lid[256];
  int col[256];
  for (int64_t li = lo; li < hi; ++li) {
    if (gather_order(c, li, G, to_local, lid, col) < 0) return false;
    for (int p = 0; p < G; ++p)
      if (lid[p] < lo || lid[p] >= hi) others.push_back(lid[p]);
  }
  std::sort(others.begin(), others.end());
  others.erase(std::unique(others.begin(), others.end()), others.end());
  u.clear();
  for (int k = 0; k < T; ++k) u.push_back((int32_t)(lo + k < hi ? lo + k : lo));
  u.insert(u.end(), others.begin(), others.end());
  return true;
}

}  // namespace

// Conical-product Gauss-Jacobi rule on T_E exact for degree M (R19); points [nq][d],
// weights normalised to 1.  Shared by the packed precompute and the matrix-free setup.
void simplex_rule(int d, int M, std::vector<double>& qp, std::vector<double>& qw) {
  qp.clear();
  qw.clear();
  // collapsed coordinates (u, v, w), Jacobian (1-v)(1-w)^2 absorbed by Jacobi weights
  // (1-x)^1 and (1-x)^2, ceil((M+1)/2) points per direction; normalised to average.
  {
    const int n = (M + 2) / 2;
    std::vector<double> ua, wa, vb, wb, wc, wcw;
    gauss_jacobi01(n, 0.0, ua, wa);
    gauss_jacobi01(n, 1.0, vb, wb);
    gauss_jacobi01(n, 2.0, wc, wcw);
    if (d == 2) {
      for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) {
          qp.push_back(ua[a] * (1 - vb[b]));
          qp.push_back(vb[b]);
          qw.push_back(wa[a] * wb[b]);
        }
    } else {
      for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b)
          for (int e = 0; e < n; ++e) {
            qp.push_back(ua[a] * (1 - vb[b]) * (1 - wc[e]));
            qp.push_back(vb[b] * (1 - wc[e]));
            qp.push_back(wc[e]);
            qw.push_back(wa[a] * wb[b] * wcw[e]);
          }
    }
    double wsum = 0.0;
    for (double w : qw) wsum += w;
    for (double& w : qw) w /= wsum;
  }
}

// Build the packed tiles for local owned cells [0, n_owned) and hand them to the
// device (or keep them on the host for a host-only context).
void precompute(cwreco_ctx* c) {
  if (!c->has_stencils) fail(CWRECO_ESTATE, "precompute: call cwreco_build_stencils first");
  const int d = c->d, M = c->M, nm = c->nm, ne = c->ne, nv = d + 1;
  const int R = nm - 1, K = ne - 1;

  // global -> local map
  const int64_t n_loc = c->n_owned + c->n_ghost;
  std::vector<int32_t> own2local(c->own_hi - c->own_lo, -1);
  for (int64_t li = 0; li < c->n_owned; ++li) own2local[c->local2global[li] - c->own_lo] = (int32_t)li;
  auto to_local = [&](int64_t g) -> int32_t {
    if (g >= c->own_lo && g < c->own_hi) return own2local[g - c->own_lo];
    if (g >= c->N) {  // boundary ghost (R37): local ids after the halo ghosts
      auto it = std::lower_bound(c->bc_ids.begin(), c->bc_ids.end(), g);
      if (it == c->bc_ids.end() || *it != g) return -1;
      return (int32_t)(n_loc + (it - c->bc_ids.begin()));
    }
    auto b = c->local2global.begin() + c->n_owned, e = c->local2global.begin() + n_loc;
    auto it = std::lower_bound(b, e, g);
    if (it == e || *it != g) return -1;
    return (int32_t)(it - c->local2global.begin());
  };
  const int G = c->G;
  // largest stencil union of tiles of T cells (sizes the union chunk and Q_u)
  auto umax_for = [&](int T) {
    const int64_t nt = (c->n_owned + T - 1) / T;
    int umax = T, bad = 0;
#pragma omp parallel reduction(max : umax) reduction(| : bad)
    {
      std::vector<int32_t> u;
#pragma omp for schedule(dynamic, 64)
      for (int64_t t = 0; t < nt; ++t) {
        if (!tile_union(c, t, T, G, to_local, u)) { bad |= 1; continue; }
        umax = std::max(umax, (int)u.size());
      }
    }
    if (bad) fail(CWRECO_EINVAL, "precompute: stencil cell missing from the local numbering");
    if ((int64_t)umax * (c->V + (c->V & 1)) > 65535)
      fail(CWRECO_EUNSUPPORTED, "precompute: tile stencil union × nvars exceeds the 16-bit offsets");
    return umax;
  };
  c->lay = make_layout(d, M, c->V, G, c->device >= 0 ? dev_max_smem(c) : 227 * 1024, umax_for, c->family, (int)c->max_tile);
  const Layout& L = c->lay;
  const int T = L.T;
  c->n_tiles = (c->n_owned + T - 1) / T;
  c->n_int_tiles = (c->n_interior == c->n_owned) ? c->n_tiles : c->n_interior / T;
  c->sigma = sigma_matrix(d, M);
  {
    double xi[3] = {0.25, 0.25, 0.25}, psi[64];
    basis_eval(d, M, xi, psi);
    c->psi1 = psi[0];
  }

  std::vector<double> qp, qw;  // points [nq][d], weights normalised to 1
  simplex_rule(d, M, qp, qw);
  const int nq = (int)qw.size();
  // monomial form of the basis: A row of stencil cell j = coef · (monomial averages over T_j)
  std::vector<int> mexp;
  std::vector<double> mcoef;
  basis_monomials(d, M, mexp, mcoef);
  const int nmono = (int)mexp.size() / 3;

  const int64_t TILES_PER_BATCH = std::max<int64_t>(1, (int64_t(256) << 20) / L.tile_bytes);
  const bool keep_host = c->device < 0;
  if (keep_host) c->host_blocks.assign(size_t(c->n_tiles) * L.tile_bytes, 0);
  std::vector<unsigned char> batch;
  if (!keep_host) dev_alloc_blocks(c, c->n_tiles * L.tile_bytes);
  int bad_singular = 0, bad_local = 0;
  double cond_max = 0.0;

  for (int64_t t0 = 0; t0 < c->n_tiles; t0 += TILES_PER_BATCH) {
    const int64_t t1 = std::min(c->n_tiles, t0 + TILES_PER_BATCH);
    unsigned char* base;
    if (keep_host) {
      base = c->host_blocks.data() + size_t(t0) * L.tile_bytes;
    } else {
      batch.assign(size_t(t1 - t0) * L.tile_bytes, 0);
      base = batch.data();
    }
#pragma omp parallel for schedule(dynamic, 16) reduction(| : bad_singular, bad_local) reduction(max : cond_max)
    for (int64_t tile = t0; tile < t1; ++tile) {
      unsigned char* tb = base + size_t(tile - t0) * L.tile_bytes;
      std::vector<int32_t> uni;
      if (!tile_union(c, tile, T, G, to_local, uni) || (int)uni.size() > L.Umax) { bad_local |= 1; continue; }
      int32_t* uid = (int32_t*)tb;
      for (int k = 0; k < L.Umax; ++k) uid[k] = k < (int)uni.size() ? uni[k] : uni[0];
      const int64_t lo = tile * T, hi = std::min(c->n_owned, lo + T);
      auto uindex = [&](int32_t lid) -> int {
        if (lid >= lo && lid < hi) return int(lid - lo);
        auto it = std::lower_bound(uni.begin() + T, uni.end(), lid);
        return int(it - uni.begin());
      };
      const int nvdd = nv * d * d;
      for (int64_t li = lo; li < hi; ++li) {
        const int ct = int(li - lo);
        const int64_t g = c->local2global[li];
        const int64_t q = g - c->own_lo;
        const int32_t* cen = &c->central[q * ne];
        const int32_t* sec = &c->sectors[q * nv * nv];
        const uint8_t* val = &c->valid[q * nv];

        // owner affine map x = X0 + J ξ
        const double* Xi = &c->X[g * nv * d];
        double J[9], Ji[9];
        for (int a = 0; a < d; ++a)
          for (int k = 0; k < d; ++k) J[a * d + k] = Xi[(k + 1) * d + a] - Xi[a];
        if (!inv_small(d, J, Ji)) { bad_singular |= 1; continue; }

        int32_t lid[256];
        int col[256];
        if (gather_order(c, li, G, to_local, lid, col) < 0) { bad_local |= 1; continue; }
        for (int p = 0; p < G; ++p)
          ((uint16_t*)(tb + L.off_idx))[idx_elem(L.kind, T, p, ct)] =
              (uint16_t)(uindex(lid[p]) * L.VP);  // element offset of the cell's row in Q_u
        uint8_t vm = 0;
        for (int s = 0; s < nv; ++s) vm |= val[s] ? uint8_t(1u << s) : 0;

        // central reduced LSQ matrix A[1:,1:] (column-major, K rows)
        thread_local std::vector<double> A;
        A.assign(size_t(K) * R, 0.0);
        double psi[64], xi[3], sh[3];
        for (int k = 1; k < ne; ++k) {
          const int64_t j = cen[k];
          double xb[12];
          const double* Xj = cell_X(c, j, xb);
          shift_of(c, g, j, sh);
          // ξ = t + C ξ' with t = J⁻¹(X_j0 + sh − X_i0), C = J⁻¹ J_j
          double t[3], Cm[9], Jj[9];
          for (int a = 0; a < d; ++a)
            for (int e = 0; e < d; ++e) Jj[a * d + e] = Xj[(e + 1) * d + a] - Xj[a];
          for (int a = 0; a < d; ++a) {
            double s = 0.0;
            for (int e = 0; e < d; ++e) s += Ji[a * d + e] * (Xj[e] + sh[e] - Xi[e]);
            t[a] = s;
            for (int e = 0; e < d; ++e) {
              double s2 = 0.0;
              for (int f = 0; f < d; ++f) s2 += Ji[a * d + f] * Jj[f * d + e];
              Cm[a * d + e] = s2;
            }
          }
          // monomial averages over the stencil cell, ξ = t + C ξ'_q (quadrature exact for degree M)
          double mom[64] = {0};
          for (int qq = 0; qq < nq; ++qq) {
            double pw[3][8];
            for (int a = 0; a < d; ++a) {
              double s = t[a];
              for (int e = 0; e < d; ++e) s += Cm[a * d + e] * qp[qq * d + e];
              pw[a][0] = 1.0;
              for (int p = 1; p <= M; ++p) pw[a][p] = pw[a][p - 1] * s;
            }
            if (d == 2) pw[2][0] = 1.0;
            const double wq = qw[qq];
            for (int e = 0; e < nmono; ++e)
              mom[e] += wq * (pw[0][mexp[3 * e]] * pw[1][mexp[3 * e + 1]] * pw[2][mexp[3 * e + 2]]);
          }
          for (int l = 1; l < nm; ++l) {
            double s = 0.0;
            const double* cl = &mcoef[size_t(l) * nmono];
            for (int e = 0; e < nmono; ++e) s += cl[e] * mom[e];
            A[size_t(l - 1) * K + (k - 1)] = s;
          }
        }
        thread_local std::vector<double> Bp;
        double cond = 0.0;
        if (!pinv_qr(K, R, A, Bp, cond)) { bad_singular |= 1; continue; }
        cond_max = std::max(cond_max, cond);
        // B chunks: chunk ch holds positions p in [ch·KC, ch·KC + kc) as [T][R][kc]
        for (int p = 0; p < G; ++p) {
          const int ch = p / L.KC, kk = p % L.KC;
          const int kc = L.kc_of(ch);
          double* chb = (double*)(tb + L.off_chunk(ch) + L.ids_bytes);
          const int k = col[p];
          for (int l = 0; l < R; ++l) chb[chunk_elem(L.kind, kc, R, L.V, T, l, ct, kk)] = k >= 0 ? Bp[size_t(l) * K + k] : 0.0;
        }
        if (L.kind == KIND_ROWBLK) {  // rs[l] = Σ_p B⁺[l][p] (positions in gather order)
          double* rs = (double*)(tb + sector_sinv_off(L.off_sector, L.sector_bytes, L.TSC, L.srec, ct)) + nvdd;
          for (int l = 0; l < R; ++l) {
            double t = 0.0;
            for (int p = 0; p < G; ++p) t += col[p] >= 0 ? Bp[size_t(l) * K + col[p]] : 0.0;
            rs[l] = t;
          }
        }

        // sector inverses
        for (int s = 0; s < nv; ++s) {
          double* Sd = (double*)(tb + sector_sinv_off(L.off_sector, L.sector_bytes, L.TSC, L.srec, ct)) + s * d * d;
          for (int e = 0; e < d * d; ++e) Sd[e] = 0.0;
          if (!val[s]) continue;
          double As[9];
          for (int m = 0; m < d; ++m) {
            const int64_t j = sec[s * nv + 1 + m];
            shift_of(c, g, j, sh);
            double bj[3];
            cell_bary(c, j, bj);
            for (int a = 0; a < d; ++a) {
              double s2 = 0.0;
              for (int e = 0; e < d; ++e) s2 += Ji[a * d + e] * (bj[e] + sh[e] - Xi[e]);
              xi[a] = s2;
            }
            basis_eval(d, 1, xi, psi);
            for (int l = 0; l < d; ++l) As[m * d + l] = psi[l + 1];
          }
          // p_l = Σ_m S[l][m] ΔQ_m with S = As⁻¹ where As[m][l]
          double Ai[9];
          if (!inv_small(d, As, Ai)) {
            vm &= uint8_t(~(1u << s));
            continue;
          }
          for (int e = 0; e < d * d; ++e) Sd[e] = Ai[e];
        }
        *(tb + sector_mask_off(L.off_sector, L.sector_bytes, L.sinv_bytes, L.TSC, ct)) = vm;
      }
    }
    if (bad_singular || bad_local) break;
    if (!keep_host) dev_upload_blocks(c, t0 * L.tile_bytes, batch.data(), int64_t(t1 - t0) * L.tile_bytes);
  }
  if (bad_singular) fail(CWRECO_ESINGULAR, "precompute: rank-deficient least-squares system or degenerate cell");
  if (bad_local) fail(CWRECO_EINVAL, "precompute: stencil cell missing from the local numbering");
  (void)cond_max;
  if (!keep_host) dev_upload_aux(c);
  c->has_blocks = true;
}

// Matrix-free mode (SURVEY §8(f) NEXT-1, P:230 ALE remark): instead of the packed
// B⁺ stream the device gets the geometry and stencils and solves each cell's
// constrained least-squares problem in the pass (matfree.cu).  Host part: local
// geometry, stencils as local ids with periodic image codes (2 bits per axis:
// 0 → 0, 1 → +L, 2 → −L, R16), the basis in monomial form and the quadrature rule.
void matfree_prepare(cwreco_ctx* c, MatfreeHost& h) {
  if (!c->has_stencils) fail(CWRECO_ESTATE, "prepare_matrixfree: call cwreco_build_stencils first");
  if (c->has_bc) fail(CWRECO_EUNSUPPORTED, "prepare_matrixfree: boundary ghost cells are not supported");
  const int d = c->d, ne = c->ne, nv = d + 1;
  const int64_t n_loc = c->n_owned + c->n_ghost;
  std::vector<int32_t> own2local(c->own_hi - c->own_lo, -1);
  for (int64_t li = 0; li < c->n_owned; ++li) own2local[c->local2global[li] - c->own_lo] = (int32_t)li;
  auto to_local = [&](int64_t g) -> int32_t {
    if (g >= c->own_lo && g < c->own_hi) return own2local[g - c->own_lo];
    auto b = c->local2global.begin() + c->n_owned, e = c->local2global.begin() + n_loc;
    auto it = std::lower_bound(b, e, g);
    if (it == e || *it != g) return -1;
    return (int32_t)(it - c->local2global.begin());
  };
  h.X.assign(n_loc * nv * d, 0.0);
  h.B.assign(n_loc * d, 0.0);
  for (int64_t li = 0; li < n_loc; ++li) {
    const int64_t g = c->local2global[li];
    std::memcpy(&h.X[li * nv * d], &c->X[g * nv * d], sizeof(double) * nv * d);
    std::memcpy(&h.B[li * d], &c->bary[g * d], sizeof(double) * d);
  }
  const int K = ne - 1;
  h.st.assign(c->n_owned * K, 0);
  h.sh.assign(c->n_owned * K, 0);
  h.sec.assign(c->n_owned * nv * d, -1);
  h.secsh.assign(c->n_owned * nv * d, 0);
  h.vmask.assign(c->n_owned, 0);
  int bad = 0;
  auto code_of = [&](int64_t gi, int64_t gj) -> uint8_t {
    double sh[3];
    shift_of(c, gi, gj, sh);
    uint8_t code = 0;
    for (int a = 0; a < d; ++a) {
      const double n = c->periodic ? sh[a] / c->L[a] : 0.0;
      if (n > 0.5) code |= uint8_t(1u << (2 * a));
      else if (n < -0.5) code |= uint8_t(2u << (2 * a));
      if (std::fabs(n) > 1.5) bad |= 2;  // stencils never span more than one period
    }
    return code;
  };
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (int64_t li = 0; li < c->n_owned; ++li) {
    const int64_t g = c->local2global[li], q = g - c->own_lo;
    for (int k = 1; k < ne; ++k) {
      const int64_t j = c->central[q * ne + k];
      const int32_t lj = to_local(j);
      if (lj < 0) bad |= 1;
      h.st[li * K + k - 1] = lj;
      h.sh[li * K + k - 1] = code_of(g, j);
    }
    uint8_t vm = 0;
    for (int s = 0; s < nv; ++s) {
      if (!c->valid[q * nv + s]) continue;
      vm |= uint8_t(1u << s);
      for (int m = 0; m < d; ++m) {
        const int64_t j = c->sectors[(q * nv + s) * nv + 1 + m];
        const int32_t lj = to_local(j);
        if (lj < 0) bad |= 1;
        h.sec[(li * nv + s) * d + m] = lj;
        h.secsh[(li * nv + s) * d + m] = code_of(g, j);
      }
    }
    h.vmask[li] = vm;
  }
  if (bad & 1) fail(CWRECO_EINVAL, "prepare_matrixfree: stencil cell missing from the local numbering");
  if (bad & 2) fail(CWRECO_EUNSUPPORTED, "prepare_matrixfree: stencil spans more than one period");
  basis_monomials(d, c->M, h.mexp, h.mcoef);
  simplex_rule(d, c->M, h.qp, h.qw);
  if (c->sigma.empty()) c->sigma = sigma_matrix(d, c->M);
  if (c->psi1 == 0.0) {
    double xi[3] = {0.25, 0.25, 0.25}, psi[64];
    basis_eval(d, c->M, xi, psi);
    c->psi1 = psi[0];
  }
}

}  // namespace cwr

