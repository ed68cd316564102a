// k_matfree: matrix-free CWENO reconstruction.
//
// The fixed-mesh path streams precomputed per-cell pseudo-inverses ("in the
// Eulerian case the matrices can be precomputed"); on a moving (ALE) mesh they must
// be rebuilt every step, and on large meshes they dominate the memory.
// This kernel builds and solves each cell's systems in the pass, from the geometry:
//   A[k][l] = average over stencil cell j(k) of ψ_l(ξ_i(x))
//   p̂_opt[1..] = argmin ‖A[1:,1:] p − (Q_j − Q_i)‖₂ (constrained LSQ, R10)
//   p̂_s = A_s⁻¹ ΔQ_s, A_s[m][l] = ψ_{l+1}(ξ_i(b_{j_m}))
// then the same fused epilogue as the other kernels (P0, σ, ω, blend).
//
// One warp per cell (persistent grid, 4-warp CTAs):
//   1. lane L assembles rows k = L, L+32 of X = [mom | ΔQ] in shared memory: the
//      stencil cell's vertices in the owner's reference frame, its monomial moments in
//      closed form (Dirichlet formula, exact for polynomials: equal to the degree-M
//      quadrature of R19 up to rounding);
//   1b. the basis transform A = mom·Cᵀ (C: the modes' monomial coefficients) on the fp64
//      tensor cores (mma.sync m8n8k4), one 8-row tile at a time, in place;
//   2. Gram [AᵀA | AᵀΔQ] = XᵀX on the fp64 tensor cores, upper block tiles only;
//   3. normal equations (R38): Cholesky AᵀA = UᵀU, lane k holding column k, the pivot
//      rows broadcast through shared memory, the V right-hand sides forward-substituted
//      in the same sweep; back substitution per variable (lane v) with Uᵀ rows;
//   4. lanes 0..d solve the sector systems; lanes 0..V−1 run cweno_epilogue.
// fp64-ALU bound, HBM traffic ≈ geometry + stencil ids + Q + w per cell.  Results agree
// with the oracle within the parity tolerance (not bitwise with the matrix kernels:
// a different solve).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "kcommon.cuh"

namespace cwr {

#define MCK(x)                                                                                 \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) fail(CWRECO_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#ifndef CWR_MF_V2
#define CWR_MF_V2 1  // unrolled basis transform, rsqrt pivots, column back substitution
#endif
#ifndef CWR_MF_TC
#define CWR_MF_TC 1  // basis transform A = mom·Cᵀ on the fp64 tensor cores (else scalar FMAs)
#endif
#ifndef CWR_MF_CHOL_SMEM
#define CWR_MF_CHOL_SMEM 1  // Cholesky rows broadcast through shared memory (else shuffles)
#endif
#ifndef CWR_MF_FAST_RSQ
#define CWR_MF_FAST_RSQ 1  // rsqrt.approx + two Newton steps (else the library rsqrt)
#endif
#ifndef CWR_MF_PF
#define CWR_MF_PF 0  // prefetch the next cell's stencil vertices / averages (1: L1, 2: L2)
#endif
#ifndef CWR_MF_UNROLL
#define CWR_MF_UNROLL 0  // basis transform fully unrolled (register pressure: spills at 4 CTAs/SM)
#endif
// resident 4-warp CTAs per SM the register allocation must allow (3-D M = 3 with many
// variables: 3, i.e. 168 registers; otherwise 4, i.e. 128)
__host__ __device__ constexpr int mf_minb(int D, int M, int V) { return D == 3 && M == 3 && V > 6 ? 3 : 4; }

// Basis (monomial form) and quadrature tables of every supported (d, M), each in its
// own slot of the constant bank, so contexts of different (d, M) on one device never
// overwrite each other's tables (the tables depend only on (d, M)).
constexpr int kMfMaxQ = 64;
__host__ __device__ constexpr int mf_slot(int D, int M) { return (D - 2) * 3 + (M - 1); }  // M ≤ 3
__host__ __device__ constexpr int mf_coef_off(int D, int M) {
  int off = 0;
  for (int s = 0; s < mf_slot(D, M); ++s) {
    const int n = nmodes(s % 3 + 1, s / 3 + 2);
    off += n * n;
  }
  return off;
}
static __constant__ double c_mcoef[mf_coef_off(3, 3) + 20 * 20];

// Monomial exponents in basis_monomials' graded order (basis.cpp): for n, for i = n..0,
// for j = n−i..0, k = n−i−j (2-D: k = 0 only) — compile-time, so the powers index
// registers, not local memory.
struct MonoTab {
  int e[64][3];
};
__host__ __device__ constexpr MonoTab mono_tab(int D, int M) {
  MonoTab t{};
  int c = 0;
  for (int n = 0; n <= M; ++n)
    for (int i = n; i >= 0; --i)
      for (int j = n - i; j >= 0; --j) {
        const int k = n - i - j;
        if (D == 2 && k != 0) continue;
        t.e[c][0] = i;
        t.e[c][1] = j;
        t.e[c][2] = k;
        ++c;
      }
  return t;
}

struct MfArgs {
  const double* X;       // [n_local][d+1][d]
  const double* B;       // [n_local][d]
  const int32_t* st;     // [n_owned][K]
  const uint8_t* sh;     // [n_owned][K]
  const int32_t* sec;    // [n_owned][d+1][d]
  const uint8_t* secsh;  // [n_owned][d+1][d]
  const uint8_t* vmask;  // [n_owned]
  double L[3];
  int nq, nmono;
  int64_t cell_begin, cell_end;
};

struct MfState {
  double *X = nullptr, *B = nullptr;
  int32_t *st = nullptr, *sec = nullptr;
  uint8_t *sh = nullptr, *secsh = nullptr, *vmask = nullptr;
  int nq = 0, nmono = 0;
};

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

template <int D>
__device__ __forceinline__ void shift_vec(uint8_t code, const double (&L)[3], double (&s)[D]) {
#pragma unroll
  for (int a = 0; a < D; ++a) {
    // branch-free: code 1 → +L, 2 → −L, 0 → 0 (mask the bits of L, flip its sign bit)
    const int c = (code >> (2 * a)) & 3;
    const long long keep = (c == 1 || c == 2) ? -1LL : 0LL, sign = (long long)(c == 2) << 63;
    s[a] = __longlong_as_double((__double_as_longlong(L[a]) & keep) ^ sign);
  }
}

// 3×3 / 2×2 inverse by cofactors (as the host's sector inverse); false if det = 0
template <int D>
__device__ __forceinline__ bool inv_small_d(const double (&A)[D][D], double (&Ai)[D][D]) {
  if constexpr (D == 2) {
    const double det = A[0][0] * A[1][1] - A[0][1] * A[1][0];
    if (det == 0.0 || !isfinite(det)) return false;
    const double r = 1.0 / det;
    Ai[0][0] = A[1][1] * r;
    Ai[0][1] = -A[0][1] * r;
    Ai[1][0] = -A[1][0] * r;
    Ai[1][1] = A[0][0] * r;
    return true;
  } else {
    const double c00 = A[1][1] * A[2][2] - A[1][2] * A[2][1], c01 = A[1][2] * A[2][0] - A[1][0] * A[2][2],
                 c02 = A[1][0] * A[2][1] - A[1][1] * A[2][0];
    const double det = A[0][0] * c00 + A[0][1] * c01 + A[0][2] * c02;
    if (det == 0.0 || !isfinite(det)) return false;
    const double r = 1.0 / det;
    Ai[0][0] = c00 * r;
    Ai[0][1] = (A[0][2] * A[2][1] - A[0][1] * A[2][2]) * r;
    Ai[0][2] = (A[0][1] * A[1][2] - A[0][2] * A[1][1]) * r;
    Ai[1][0] = c01 * r;
    Ai[1][1] = (A[0][0] * A[2][2] - A[0][2] * A[2][0]) * r;
    Ai[1][2] = (A[0][2] * A[1][0] - A[0][0] * A[1][2]) * r;
    Ai[2][0] = c02 * r;
    Ai[2][1] = (A[0][1] * A[2][0] - A[0][0] * A[2][1]) * r;
    Ai[2][2] = (A[0][0] * A[1][1] - A[0][1] * A[1][0]) * r;
    return true;
  }
}

// Row stride of X in doubles.  The assembly writes X row-per-lane (lane k, row k: a
// 64-bit store of 16 lanes is conflict-free only if 16 consecutive rows fall in 16
// different bank pairs, i.e. the stride is odd — NCP itself, a multiple of 8, put
// every row of a half-warp in 2 bank pairs: 8-way conflicts, 4.9e9 per C5 pass); the
// Gram fragments read rows lane%4 × columns lane/4, conflict-free only for strides
// ≡ 4, 12 (mod 16): an odd stride with stride mod 16 ∉ {1, 15} keeps those 2-way.
__host__ __device__ constexpr int mf_xs(int ncp) {
  int s = ncp | 1;
  while (s % 16 == 1 || s % 16 == 15) s += 2;
  return s;
}

// Row stride of G / U: even (16-byte aligned rows: the Cholesky reads row pairs with
// one 128-bit broadcast load) in the shared-memory Cholesky, else NCP + 1.
__host__ __device__ constexpr int mf_gs(int ncp) { return CWR_MF_CHOL_SMEM ? ncp + 2 : ncp + 1; }
// monomials of degree ≤ deg(ψ_l) (the basis transform's sum length for mode l)
__host__ __device__ constexpr int mf_hi_of_mode(int D, int l) {
  int n = 0;
  while (nmodes(n, D) <= l) ++n;
  return nmodes(n, D);
}
// k-steps (4 monomials each) the transform's 8-column tile nt needs: its columns are
// modes 8nt+1 .. min(8nt+8, R), of degree ≤ that of the last one
__host__ __device__ constexpr int mf_nk_tile(int D, int M, int nt) {
  const int R = nmodes(M, D) - 1, l = 8 * nt + 8 < R ? 8 * nt + 8 : R;
  return (mf_hi_of_mode(D, l) + 3) / 4;
}

// Per-warp shared scratch (doubles): X = [A | ΔQ] with KR rows of stride XS (the
// Gram matrix and then the Cholesky factor reuse its first rows), then the sector
// products [NV][D][V]; per CTA after the warps' scratch: the transform's B fragments.
template <int D, int M, int V>
struct MfShape {
  static constexpr int NM = nmodes(M, D), R = NM - 1, NV = D + 1, K = D * NM - 1;
  static constexpr int KP = (K + 3) & ~3;            // rows padded to whole k-steps of 4 (Gram)
  static constexpr int KR = (K + 7) & ~7;            // rows padded to whole 8-row tiles (transform)
  static constexpr int NC = R + V;                   // columns of [A | ΔQ]
  static constexpr int NCP = (NC + 7) & ~7;          // padded to whole 8-column blocks
  static constexpr int NB = NCP / 8;                 // column blocks (DMMA tiles per side)
  static constexpr int NK = (NM + 3) / 4;            // transform k-steps (monomials)
  static constexpr int NT = (R + 7) / 8;             // transform column tiles
  static constexpr int GS = mf_gs(NCP);              // row stride of G and U in the scratch
  static constexpr int XS = mf_xs(NCP);              // row stride of X (see mf_xs)
  static constexpr int XR = CWR_MF_TC ? KR : KP;     // rows of X held
  static constexpr int G_DBL = (CWR_MF_CHOL_SMEM ? 2 : 1) * NCP * GS;   // G / U (+ Uᵀ)
  static constexpr int X_DBL = XR * XS > G_DBL ? XR * XS : G_DBL;         // X, then G / U
  static constexpr int PS_DBL = NV * D * V;
  static constexpr int SCR = (X_DBL + PS_DBL + 1) & ~1;  // even: every warp's X 16-byte aligned
  static constexpr int BF_DBL = CWR_MF_TC ? NT * NK * 32 : 0;
  static_assert(NC <= 32, "one lane per column of [G | AᵀΔQ]");
  static_assert(4 * NK <= NCP, "the monomial moments fit in a row of X");
};
__host__ __device__ constexpr int mf_scr_doubles(int D, int M, int V) {
  const int k = D * nmodes(M, D) - 1, kp = (k + 3) & ~3, kr = (k + 7) & ~7, xr = CWR_MF_TC ? kr : kp;
  const int ncp = (nmodes(M, D) - 1 + V + 7) & ~7, xs = mf_xs(ncp), gs = mf_gs(ncp);
  const int g = (CWR_MF_CHOL_SMEM ? 2 : 1) * ncp * gs;
  return ((xr * xs > g ? xr * xs : g) + (D + 1) * D * V + 1) & ~1;
}
__host__ __device__ constexpr int mf_bf_doubles(int D, int M) {
  return CWR_MF_TC ? ((nmodes(M, D) - 1 + 7) / 8) * ((nmodes(M, D) + 3) / 4) * 32 : 0;
}

// 1/√x: the SFU approximation refined by two Newton steps (relative error at the
// rounding level; NaN for x ≤ 0 as the library's rsqrt, so a rank-deficient stencil
// still yields NaN, not a silent result)
__device__ __forceinline__ double mf_rsqrt(double x) {
#if CWR_MF_FAST_RSQ
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    const double h = x * y;
    const double r = fma(-h, y, 1.0);
    y = fma(0.5 * y, r, y);
  }
  return y;
#else
  return rsqrt(x);
#endif
}

// Moments of the monomials of degree ≤ 3 over a simplex with vertices y_0..y_D, in
// closed form (exact for polynomials, so equal to the degree-M quadrature of R19 up
// to rounding): with λ ~ Dirichlet(1,…,1), E[λ^β] = D!·β!/(D+|β|)!, hence with
// s_a = Σ_m y_m[a], S_ab = Σ_m y_m[a]y_m[b], T_abc = Σ_m y_m[a]y_m[b]y_m[c]:
//   E[ξ_a] = s_a/(D+1),   E[ξ_aξ_b] = (S_ab + s_a s_b)/((D+1)(D+2)),
//   E[ξ_aξ_bξ_c] = (2T_abc + S_ab s_c + S_ac s_b + S_bc s_a + s_a s_b s_c)/((D+1)(D+2)(D+3)).
struct MonoIdx {  // per monomial: degree and its sorted coordinate multiset
  int deg[64], a[64], b[64], c[64];
};
__host__ __device__ constexpr MonoIdx mono_idx(int D, int M) {
  MonoIdx t{};
  const MonoTab mt = mono_tab(D, M);
  for (int e = 0; e < nmodes(M, D); ++e) {
    int lst[3] = {0, 0, 0}, n = 0;
    for (int ax = 0; ax < 3; ++ax)
      for (int p = 0; p < mt.e[e][ax]; ++p) lst[n++] = ax;
    t.deg[e] = n;
    t.a[e] = lst[0];
    t.b[e] = lst[1];
    t.c[e] = lst[2];
  }
  return t;
}
// moment of monomial E (compile time: no runtime-indexed arrays) from the power sums
template <int D, int M, int E>
__device__ __forceinline__ double mono_moment(const double (&sv)[D], const double (&S2)[D][D],
                                              const double (&T3)[D * D * D]) {
  constexpr MonoIdx MI = mono_idx(D, M);
  constexpr int dg = MI.deg[E], ea = MI.a[E], eb = MI.b[E], ec = MI.c[E];
  constexpr double c1 = 1.0 / (D + 1), c2 = 1.0 / ((D + 1) * (D + 2)), c3 = 1.0 / ((D + 1) * (D + 2) * (D + 3));
  if constexpr (dg == 0) {
    return 1.0;
  } else if constexpr (dg == 1) {
    return sv[ea] * c1;
  } else if constexpr (dg == 2) {
    return (S2[ea][eb] + sv[ea] * sv[eb]) * c2;
  } else {
    return (2.0 * T3[(ea * D + eb) * D + ec] + S2[ea][eb] * sv[ec] + S2[ea][ec] * sv[eb] + S2[eb][ec] * sv[ea] +
            sv[ea] * sv[eb] * sv[ec]) *
           c3;
  }
}
template <int D, int M, int NM, int... E>
__device__ __forceinline__ void mono_moments(double (&mom)[NM], const double (&sv)[D], const double (&S2)[D][D],
                                             const double (&T3)[D * D * D], std::integer_sequence<int, E...>) {
  ((mom[E] = mono_moment<D, M, E>(sv, S2, T3)), ...);
}

// One warp per cell (persistent grid):
//  1. assembly: lane L builds rows k = L, L+32 of X = [A | ΔQ] (A[k][l−1] = average of
//     ψ_l(ξ_i(x)) over stencil cell j(k): closed-form simplex moments of the
//     monomials, then the basis coefficients of mode l over the monomials of degree
//     ≤ deg(l)) into shared memory;
//  2. Gram: [AᵀA | AᵀΔQ] = XᵀX on the fp64 tensor cores (mma.sync m8n8k4: both operand
//     fragments are X[k0 + lane%4][8·blk + lane/4]);
//  3. the normal equations of the reduced LSQ (R10; R38): Cholesky of AᵀA in
//     registers (lane k owns column k of [AᵀA | AᵀΔQ], pivot rows by shuffles), which
//     also forward-substitutes the V right-hand sides; lanes v < V back-substitute;
//  4. lanes 0..d solve the sector systems; lanes 0..V−1 run the fused
//     epilogue and store w.
// fp64-ALU bound; HBM per cell ≈ geometry + stencil ids + Q + w.
template <int D, int M, int V>
__global__ void __launch_bounds__(128, mf_minb(D, M, V)) k_matfree(MfArgs m, KArgs a) {
  using S = MfShape<D, M, V>;
  constexpr int NM = S::NM, R = S::R, NV = S::NV, K = S::K, KP = S::KP, KR = S::KR, NC = S::NC, NCP = S::NCP,
                NB = S::NB, XS = S::XS, GS = S::GS;
  constexpr int KPL = (K + 31) / 32;  // rows of X per lane

  const int lane = threadIdx.x & 31;
  const double* mcoef = c_mcoef + mf_coef_off(D, M);
  extern __shared__ __align__(16) double mf_smem[];
  double* X = mf_smem + (threadIdx.x >> 5) * S::SCR;  // [KP][XS], later G / U [NCP][GS]
  double* PSs = X + S::X_DBL;                          // [NV][D][V] sector products
#if CWR_MF_TC
  // B fragments of the basis transform, Cᵀ[k][n] = C[n+1][k] (lane L holds k = 4ks + L%4,
  // n = 8nt + L/4), in fragment order after the warps' scratch: one conflict-free load each
  double* Bs = mf_smem + (blockDim.x >> 5) * S::SCR;
  for (int t = threadIdx.x; t < S::BF_DBL; t += blockDim.x) {
    const int ln = t & 31, ks = (t >> 5) % S::NK, nt = (t >> 5) / S::NK;
    const int kk = 4 * ks + (ln & 3), n = 8 * nt + (ln >> 2);
    Bs[t] = (n < R && kk < NM) ? mcoef[(n + 1) * NM + kk] : 0.0;
  }
  __syncthreads();
#endif
  const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  // stencil ids and image codes of this lane's rows, loaded one cell ahead (the vertex
  // gathers then depend on one global load, not two)
  int32_t jn[KPL];
  uint8_t cn[KPL];
  auto load_ids = [&](int64_t ic) {
#pragma unroll
    for (int r = 0; r < KPL; ++r) {
      const int k = lane + 32 * r;
      const bool ok = ic < m.cell_end && k < K;
      jn[r] = ok ? m.st[ic * K + k] : 0;
      cn[r] = ok ? m.sh[ic * K + k] : 0;
    }
  };
  load_ids(m.cell_begin + w0);
  for (int64_t i = m.cell_begin + w0; i < m.cell_end; i += nw) {
    int32_t jc[KPL];
    uint8_t cc[KPL];
#pragma unroll
    for (int r = 0; r < KPL; ++r) {
      jc[r] = jn[r];
      cc[r] = cn[r];
    }
    load_ids(i + nw);
    // ---- owner geometry x = X0 + J ξ, J⁻¹
    double X0[D], J[D][D], Ji[D][D];
    {
      const double* Xi = m.X + i * NV * D;
#pragma unroll
      for (int e = 0; e < D; ++e) X0[e] = Xi[e];
#pragma unroll
      for (int e = 0; e < D; ++e)
#pragma unroll
        for (int k = 0; k < D; ++k) J[e][k] = Xi[(k + 1) * D + e] - Xi[e];
      inv_small_d<D>(J, Ji);
    }
    double qi[V];
#pragma unroll
    for (int v = 0; v < V; ++v) qi[v] = a.Q[i * a.acs + v * a.avs];

    // ---- 1. rows of X = [A | ΔQ]
#if CWR_MF_UNROLL
#pragma unroll 1  // one row at a time: the unrolled basis transform keeps one row's moments live
#else
#pragma unroll
#endif
    for (int r = 0; r < KPL; ++r) {
      const int k = lane + 32 * r;
      if (k >= S::XR) continue;
      double* xr = X + k * XS;
      if (k >= K) {  // zero rows up to a whole k-step
#pragma unroll
        for (int l = 0; l < NCP; ++l) xr[l] = 0.0;
        continue;
      }
      int32_t j = jc[0];
      uint8_t jcode = cc[0];
#pragma unroll
      for (int rr = 1; rr < KPL; ++rr)  // selects, not a runtime-indexed register array
        if (r == rr) j = jc[rr], jcode = cc[rr];
      double sh[D];
      shift_vec<D>(jcode, m.L, sh);
      const double* Xj = m.X + int64_t(j) * NV * D;
      // vertices y_v of T_j in ξ_i coordinates, y_0 = J⁻¹(X_j0 + shift − X0),
      // y_v = y_0 + J⁻¹(X_jv − X_j0), accumulated into the power sums as they are formed
      double sv[D], S2[D][D], T3[D * D * D], y0[D];
      {
        double d0[D];
#pragma unroll
        for (int f = 0; f < D; ++f) d0[f] = Xj[f] + sh[f] - X0[f];
#pragma unroll
        for (int e = 0; e < D; ++e) {
          double s0 = 0.0;
#pragma unroll
          for (int f = 0; f < D; ++f) s0 = fma(Ji[e][f], d0[f], s0);
          y0[e] = s0;
        }
      }
#pragma unroll
      for (int v2 = 0; v2 < NV; ++v2) {
        double y[D];
        if (v2 == 0) {
#pragma unroll
          for (int e = 0; e < D; ++e) y[e] = y0[e];
        } else {
          double dv[D];
#pragma unroll
          for (int f = 0; f < D; ++f) dv[f] = Xj[v2 * D + f] - Xj[f];
#pragma unroll
          for (int e = 0; e < D; ++e) {
            double s1 = y0[e];
#pragma unroll
            for (int f = 0; f < D; ++f) s1 = fma(Ji[e][f], dv[f], s1);
            y[e] = s1;
          }
        }
#pragma unroll
        for (int e = 0; e < D; ++e) {
          sv[e] = v2 == 0 ? y[e] : sv[e] + y[e];
#pragma unroll
          for (int f = e; f < D; ++f) {
            const double pef = y[e] * y[f];
            S2[e][f] = v2 == 0 ? pef : S2[e][f] + pef;
            if constexpr (M >= 3) {
#pragma unroll
              for (int g2 = f; g2 < D; ++g2)
                T3[(e * D + f) * D + g2] = v2 == 0 ? pef * y[g2] : fma(pef, y[g2], T3[(e * D + f) * D + g2]);
            }
          }
        }
      }
      double mom[NM];
      mono_moments<D, M, NM>(mom, sv, S2, T3, std::make_integer_sequence<int, NM>{});
#if CWR_MF_TC
      // the row's monomial moments (zero-padded to whole k-steps); the transform to
      // the basis runs on the tensor cores below
#pragma unroll
      for (int e = 0; e < 4 * S::NK; ++e) xr[e] = e < NM ? mom[e] : 0.0;
    }
#else
      // A[k][l−1] = Σ_e C[l][e]·mom[e] over the monomials of degree ≤ deg(ψ_l): rows in
      // blocks of one degree n (compile-time bounds), each block's row loop rolled
#pragma unroll
      for (int n = 1; n <= M; ++n) {
        const int lo = D == 2 ? n * (n + 1) / 2 : n * (n + 1) * (n + 2) / 6;
        const int hi = D == 2 ? (n + 1) * (n + 2) / 2 : (n + 1) * (n + 2) * (n + 3) / 6;
#if CWR_MF_UNROLL
#pragma unroll  // compile-time offsets: the coefficients are constant-bank operands of the FMAs
#else
#pragma unroll 1
#endif
        for (int l = lo; l < hi; ++l) {
#if CWR_MF_V2
          // four interleaved partial sums: the dependent chain is hi/4 FMAs, not hi
          double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
          for (int e = 0; e < hi; ++e) s4[e & 3] = fma(mcoef[l * NM + e], mom[e], s4[e & 3]);
          xr[l - 1] = (s4[0] + s4[1]) + (s4[2] + s4[3]);
#else
          double s2 = 0.0;
#pragma unroll
          for (int e = 0; e < hi; ++e) s2 = fma(mcoef[l * NM + e], mom[e], s2);
          xr[l - 1] = s2;
#endif
        }
      }
#pragma unroll
      for (int v = 0; v < V; ++v) xr[R + v] = a.Q[int64_t(j) * a.acs + v * a.avs] - qi[v];
#pragma unroll
      for (int l = NC; l < NCP; ++l) xr[l] = 0.0;
    }
#endif
#if CWR_MF_TC
    // ---- 1b. A = mom·Cᵀ on the fp64 tensor cores, one 8-row tile at a time, in place:
    // A[k][l−1] = Σ_e C[l][e]·mom[k][e] (mode l uses the monomials of degree ≤ deg ψ_l,
    // so column tile nt stops after mf_nk_tile k-steps)
    {
      double dq[KPL][V];
#pragma unroll
      for (int r = 0; r < KPL; ++r)
#pragma unroll
        for (int v = 0; v < V; ++v) dq[r][v] = lane + 32 * r < K ? a.Q[int64_t(jc[r]) * a.acs + v * a.avs] - qi[v] : 0.0;
      __syncwarp();
#pragma unroll 1
      for (int t = 0; t < KR / 8; ++t) {
        double* xt = X + (8 * t + (lane >> 2)) * XS;
        double af[S::NK];
#pragma unroll
        for (int ks = 0; ks < S::NK; ++ks) af[ks] = xt[4 * ks + (lane & 3)];
        double dd[S::NT][2];
#pragma unroll
        for (int nt = 0; nt < S::NT; ++nt) {
          dd[nt][0] = dd[nt][1] = 0.0;
#pragma unroll
          for (int ks = 0; ks < mf_nk_tile(D, M, nt); ++ks)
            dmma884(dd[nt][0], dd[nt][1], af[ks], Bs[(nt * S::NK + ks) * 32 + lane]);
        }
        __syncwarp();  // every lane's fragments of this tile are read before it is overwritten
#pragma unroll
        for (int nt = 0; nt < S::NT; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = 8 * nt + 2 * (lane & 3) + e;
            if (col < R) xt[col] = dd[nt][e];
          }
      }
      __syncwarp();
      // ΔQ columns and their zero padding (rows ≥ K are zero already)
#pragma unroll
      for (int r = 0; r < KPL; ++r) {
        const int k = lane + 32 * r;
        if (k < K) {
          double* xr = X + k * XS;
#pragma unroll
          for (int v = 0; v < V; ++v) xr[R + v] = dq[r][v];
#pragma unroll
          for (int l = NC; l < NCP; ++l) xr[l] = 0.0;
        }
      }
    }
#endif

#if CWR_MF_PF
    // the next cell's stencil vertices and averages (ids loaded at the top of this cell)
    // towards the SM while the Gram / Cholesky phases run
    if (i + nw < m.cell_end) {
#pragma unroll
      for (int r = 0; r < KPL; ++r)
        if (lane + 32 * r < K) {
          const double* xp = m.X + int64_t(jn[r]) * NV * D;
          const double* qp = a.Q + int64_t(jn[r]) * a.acs;
#if CWR_MF_PF == 1
          asm volatile("prefetch.global.L1 [%0];" ::"l"(xp));
          if (D == 3) asm volatile("prefetch.global.L1 [%0];" ::"l"(xp + 8));
          asm volatile("prefetch.global.L1 [%0];" ::"l"(qp));
#else
          asm volatile("prefetch.global.L2 [%0];" ::"l"(xp));
          if (D == 3) asm volatile("prefetch.global.L2 [%0];" ::"l"(xp + 8));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(qp));
#endif
        }
    }
#endif

    // ---- 4a. sectors: lane s < d+1 solves sector s for all variables
    bool vs = false;
    if (lane < NV && ((m.vmask[i] >> lane) & 1)) {
      double As[D][D], Si[D][D], dq[D][V];
#pragma unroll
      for (int mm = 0; mm < D; ++mm) {
        const int32_t j = m.sec[(i * NV + lane) * D + mm];
        double sh[D], xi[D];
        shift_vec<D>(m.secsh[(i * NV + lane) * D + mm], m.L, sh);
#pragma unroll
        for (int e = 0; e < D; ++e) {
          double s = 0.0;
#pragma unroll
          for (int f = 0; f < D; ++f) s += Ji[e][f] * (m.B[int64_t(j) * D + f] + sh[f] - X0[f]);
          xi[e] = s;
        }
        // linear modes ψ_1..ψ_d at ξ: monomials 1, ξ, η(, ζ) are e = 0..d
#pragma unroll
        for (int l = 0; l < D; ++l) {
          double s = mcoef[(l + 1) * NM + 0];
#pragma unroll
          for (int e = 0; e < D; ++e) s += mcoef[(l + 1) * NM + 1 + e] * xi[e];
          As[mm][l] = s;
        }
#pragma unroll
        for (int v = 0; v < V; ++v) dq[mm][v] = a.Q[int64_t(j) * a.acs + v * a.avs] - qi[v];
      }
      if (inv_small_d<D>(As, Si)) {  // p_l = Σ_m S[l][m] ΔQ_m with S = As⁻¹ (As[m][l])
        vs = true;
#pragma unroll
        for (int l = 0; l < D; ++l)
#pragma unroll
          for (int v = 0; v < V; ++v) {
            double s = 0.0;
#pragma unroll
            for (int mm = 0; mm < D; ++mm) s += Si[l][mm] * dq[mm][v];
            PSs[(lane * D + l) * V + v] = s;
          }
      }
    }
    if (lane < NV && !vs) {
#pragma unroll
      for (int l = 0; l < D; ++l)
#pragma unroll
        for (int v = 0; v < V; ++v) PSs[(lane * D + l) * V + v] = 0.0;
    }
    const unsigned vbits = __ballot_sync(0xffffffffu, vs);
    __syncwarp();

    // ---- 2. Gram [AᵀA | AᵀΔQ] = XᵀX, upper block tiles (I ≤ J) on the fp64 tensor cores
    double gc[NB][NB][2];
#pragma unroll
    for (int I = 0; I < NB; ++I)
#pragma unroll
      for (int J2 = 0; J2 < NB; ++J2) gc[I][J2][0] = gc[I][J2][1] = 0.0;
    {
      const double* xf = X + (lane & 3) * XS + (lane >> 2);
#pragma unroll 5
      for (int k0 = 0; k0 < KP; k0 += 4) {
        double fr[NB];
#pragma unroll
        for (int b = 0; b < NB; ++b) fr[b] = xf[k0 * XS + 8 * b];
#pragma unroll
        for (int I = 0; I < NB; ++I)
#pragma unroll
          for (int J2 = I; J2 < NB; ++J2) dmma884(gc[I][J2][0], gc[I][J2][1], fr[I], fr[J2]);
      }
    }
    __syncwarp();  // X is dead: G takes its place
    double* G = X;  // [NCP][GS]: G[r][c] for r < R (both triangles of AᵀA), c < NC
    double* GT = X + NCP * GS;  // [NCP][GS]: Uᵀ (CWR_MF_CHOL_SMEM)
    (void)GT;
    {
      const int gr = lane >> 2, gcol = 2 * (lane & 3);
#pragma unroll
      for (int I = 0; I < NB; ++I)
#pragma unroll
        for (int J2 = I; J2 < NB; ++J2)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r0 = 8 * I + gr, c0 = 8 * J2 + gcol + e;
            G[r0 * GS + c0] = gc[I][J2][e];
            if (I != J2) G[c0 * GS + r0] = gc[I][J2][e];
          }
    }
    __syncwarp();

    // ---- 3. Cholesky AᵀA = UᵀU on [AᵀA | AᵀΔQ]: lane k holds column k; step c scales
    // row c by 1/√G[c][c] and updates rows j > c with the broadcast U[c][j]; on the
    // right-hand-side lanes (k = R + v) this is the forward substitution Uᵀy = AᵀΔQ.
    double g[R];
#pragma unroll
    for (int j = 0; j < R; ++j) g[j] = lane < NC ? G[j * GS + lane] : 0.0;
#if CWR_MF_CHOL_SMEM
    // row c of U goes straight to its final place in G (the g registers were loaded
    // before), and the update reads it back as 128-bit broadcast loads of row pairs
    __syncwarp();
#pragma unroll
    for (int c = 0; c < R; ++c) {
      const double dcc = __shfl_sync(0xffffffffu, g[c], c);
      const double inv = mf_rsqrt(dcc);  // NaN for a rank-deficient stencil (no silent result)
      const double u = g[c] * inv;
      g[c] = u;
      if (lane < NC) G[c * GS + lane] = u;    // U[c][k] (k ≥ c), y[c] for k ≥ R
      if (lane < R) GT[lane * GS + c] = u;    // Uᵀ: column k of U as a row (back substitution)
      if (lane == c) G[c * GS + NCP] = inv;  // 1/U[c][c] in the padding column
      __syncwarp();
      const double* uc = G + c * GS;
      int j = c + 1;
      if (j & 1) {
        if (j < R) g[j] = fma(-uc[j], u, g[j]);
        ++j;
      }
#pragma unroll
      for (; j + 1 < R; j += 2) {
        const double2 p = *reinterpret_cast<const double2*>(uc + j);
        g[j] = fma(-p.x, u, g[j]);
        g[j + 1] = fma(-p.y, u, g[j + 1]);
      }
      if (j < R) g[j] = fma(-uc[j], u, g[j]);
    }
    __syncwarp();
#else
#pragma unroll
    for (int c = 0; c < R; ++c) {
      const double dcc = __shfl_sync(0xffffffffu, g[c], c);
#if CWR_MF_V2
      const double inv = mf_rsqrt(dcc);  // one op on the serial chain; NaN for a rank-deficient stencil
#else
      const double inv = 1.0 / sqrt(dcc);  // NaN for a rank-deficient stencil (no silent result)
#endif
      const double u = g[c] * inv;
      g[c] = u;
      if (lane == c) G[c * GS + NCP] = inv;  // 1/U[c][c] in the padding column
#pragma unroll
      for (int j = c + 1; j < R; ++j) g[j] = fma(-__shfl_sync(0xffffffffu, u, j), u, g[j]);
    }
    __syncwarp();
    if (lane < NC) {
#pragma unroll
      for (int c = 0; c < R; ++c) G[c * GS + lane] = g[c];  // U[c][k] (k ≥ c), y[c] for k ≥ R
    }
    __syncwarp();
#endif

    // ---- per variable (lane v): back substitution U p = y, gather, fused epilogue
    double acc[R], ps[NV][D];
    bool valid[NV];
#pragma unroll
    for (int s2 = 0; s2 < NV; ++s2) valid[s2] = (vbits >> s2) & 1;
    if (lane < V) {
#if CWR_MF_V2
      // column-oriented: once p[c] is known it updates every row above it (independent
      // FMAs), so the dependent chain is R steps long instead of R²/2
      double t[R];
#pragma unroll
      for (int c = 0; c < R; ++c) t[c] = G[c * GS + R + lane];
#pragma unroll
      for (int c = R - 1; c >= 0; --c) {
        acc[c] = t[c] * G[c * GS + NCP];
#if CWR_MF_CHOL_SMEM
        // U[j][c], j < c, is row c of Uᵀ: 128-bit broadcast loads of pairs
        const double* ut = GT + c * GS;
        int j = 0;
#pragma unroll
        for (; j + 1 < c; j += 2) {
          const double2 p = *reinterpret_cast<const double2*>(ut + j);
          t[j] = fma(-p.x, acc[c], t[j]);
          t[j + 1] = fma(-p.y, acc[c], t[j + 1]);
        }
        if (j < c) t[j] = fma(-ut[j], acc[c], t[j]);
#else
#pragma unroll
        for (int j = 0; j < c; ++j) t[j] = fma(-G[j * GS + c], acc[c], t[j]);
#endif
      }
#else
#pragma unroll
      for (int c = R - 1; c >= 0; --c) {
        double t = G[c * GS + R + lane];
#pragma unroll
        for (int mm = c + 1; mm < R; ++mm) t = fma(-G[c * GS + mm], acc[mm], t);
        acc[c] = t * G[c * GS + NCP];
      }
#endif
#pragma unroll
      for (int s2 = 0; s2 < NV; ++s2)
#pragma unroll
        for (int l = 0; l < D; ++l) ps[s2][l] = PSs[(s2 * D + l) * V + lane];
      double q = 0.0;
#pragma unroll
      for (int v = 0; v < V; ++v)
        if (lane == v) q = qi[v];
      double w[NM];
      cweno_epilogue<D, NM>(q, acc, ps, valid, a, w, nullptr, nullptr);
      double* o = a.out + i * a.ccs + lane * a.cvs;
#pragma unroll
      for (int l = 0; l < NM; ++l) o[l] = w[l];
    }
    __syncwarp();  // the scratch is rewritten by the next cell
  }
}

using MfFn = void (*)(MfArgs, KArgs);
template <int D, int M>
static MfFn mf_fn_v(int V) {
  switch (V) {
    case 1: return k_matfree<D, M, 1>;
    case 2: return k_matfree<D, M, 2>;
    case 3: return k_matfree<D, M, 3>;
    case 4: return k_matfree<D, M, 4>;
    case 5: return k_matfree<D, M, 5>;
    case 6: return k_matfree<D, M, 6>;
    case 7: return k_matfree<D, M, 7>;
    case 8: return k_matfree<D, M, 8>;
    case 9: return k_matfree<D, M, 9>;
    default: return nullptr;
  }
}
static MfFn mf_fn(int d, int M, int V) {
  MfFn f = nullptr;
  if (d == 2 && M == 1) f = mf_fn_v<2, 1>(V);
  if (d == 2 && M == 2) f = mf_fn_v<2, 2>(V);
  if (d == 2 && M == 3) f = mf_fn_v<2, 3>(V);
  if (d == 3 && M == 1) f = mf_fn_v<3, 1>(V);
  if (d == 3 && M == 2) f = mf_fn_v<3, 2>(V);
  if (d == 3 && M == 3) f = mf_fn_v<3, 3>(V);
  if (!f) fail(CWRECO_EUNSUPPORTED, "matrix-free kernel: (d, M, nvars) not instantiated (M ≤ 3, nvars ≤ 9)");
  return f;
}

template <class T>
static void upload(T*& dst, const std::vector<T>& src) {
  cudaFree(dst);
  dst = nullptr;
  const size_t bytes = std::max<size_t>(1, src.size()) * sizeof(T);
  if (cudaMalloc(&dst, bytes) != cudaSuccess) {
    cudaGetLastError();
    fail(CWRECO_ENOMEM, "matrix-free: device allocation failed");
  }
  if (!src.empty()) MCK(cudaMemcpy(dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice));
}

void dev_matfree_destroy(cwreco_ctx* c) {
  MfState* s = (MfState*)c->mf;
  if (!s) return;
  DeviceGuard dg(c->device);
  cudaFree(s->X);
  cudaFree(s->B);
  cudaFree(s->st);
  cudaFree(s->sh);
  cudaFree(s->sec);
  cudaFree(s->secsh);
  cudaFree(s->vmask);
  delete s;
  c->mf = nullptr;
}

void dev_matfree_upload(cwreco_ctx* c, const MatfreeHost& h) {
  if (c->device < 0) fail(CWRECO_ECUDA, "prepare_matrixfree: context has no device (no CPU fallback)");
  mf_fn(c->d, c->M, c->V);  // EUNSUPPORTED early
  DeviceGuard dg(c->device);
  const int nmono = (int)h.mexp.size() / 3, nq = (int)h.qw.size();
  if (nq > kMfMaxQ || nmono != c->nm || c->M > 3) fail(CWRECO_EUNSUPPORTED, "matrix-free: basis too large");
  {  // the kernel's compile-time monomial order must be the library's
    int cnt = 0;
    for (int n = 0; n <= c->M; ++n)
      for (int i = n; i >= 0; --i)
        for (int j = n - i; j >= 0; --j) {
          const int k = n - i - j;
          if (c->d == 2 && k != 0) continue;
          if (h.mexp[3 * cnt] != i || h.mexp[3 * cnt + 1] != j || h.mexp[3 * cnt + 2] != k)
            fail(CWRECO_EUNSUPPORTED, "matrix-free: monomial order mismatch");
          ++cnt;
        }
  }
  if (!c->mf) c->mf = new MfState();
  MfState* s = (MfState*)c->mf;
  upload(s->X, h.X);
  upload(s->B, h.B);
  upload(s->st, h.st);
  upload(s->sh, h.sh);
  upload(s->sec, h.sec);
  upload(s->secsh, h.secsh);
  upload(s->vmask, h.vmask);
  s->nq = nq;
  s->nmono = nmono;
  // the basis over the monomials: mode l of degree n may use only monomials of degree
  // ≤ n (the kernel's sums stop there)
  for (int l = 0; l < c->nm; ++l)
    for (int e = 0; e < c->nm; ++e) {
      const int de = h.mexp[3 * e] + h.mexp[3 * e + 1] + h.mexp[3 * e + 2];
      int deg_l = 0;
      for (int n = 0, cnt = 0; n <= c->M; ++n) {
        cnt += c->d == 2 ? n + 1 : (n + 1) * (n + 2) / 2;
        if (l < cnt) {
          deg_l = n;
          break;
        }
      }
      if (de > deg_l && h.mcoef[size_t(l) * c->nm + e] != 0.0)
        fail(CWRECO_EUNSUPPORTED, "matrix-free: basis mode uses a monomial above its degree");
    }
  // constants of this translation unit: basis coefficients, packed Σ
  MCK(cudaMemcpyToSymbol(c_mcoef, h.mcoef.data(), sizeof(double) * h.mcoef.size(),
                         sizeof(double) * mf_coef_off(c->d, c->M)));
  const int nm = c->nm;
  std::vector<double> packed;
  for (int l = 1; l < nm; ++l)
    for (int m = l; m < nm; ++m) packed.push_back((l == m ? 1.0 : 2.0) * c->sigma[l * nm + m]);
  MCK(cudaMemcpyToSymbol(c_sig, packed.data(), sizeof(double) * packed.size(), sizeof(double) * sig_off(c->d, c->M)));
}

void dev_matfree_reconstruct(cwreco_ctx* c, const double* avgs, int64_t acs, int64_t avs, double* coeffs,
                             int64_t ccs, int64_t cvs, int64_t cell_begin, int64_t cell_end, void* stream) {
  MfState* s = (MfState*)c->mf;
  if (!s) fail(CWRECO_ESTATE, "matrix-free kernel: call cwreco_prepare_matrixfree first");
  if (cell_end <= cell_begin) return;
  DeviceGuard dg(c->device);
  MfArgs m;
  m.X = s->X;
  m.B = s->B;
  m.st = s->st;
  m.sh = s->sh;
  m.sec = s->sec;
  m.secsh = s->secsh;
  m.vmask = s->vmask;
  for (int e = 0; e < 3; ++e) m.L[e] = c->periodic ? c->L[e] : 0.0;
  m.nq = s->nq;
  m.nmono = s->nmono;
  m.cell_begin = cell_begin;
  m.cell_end = cell_end;
  KArgs a;
  std::memset(&a, 0, sizeof(a));
  a.V = c->V;
  a.n_owned = c->n_owned;
  a.Q = avgs;
  a.acs = acs;
  a.avs = avs;
  a.out = coeffs;
  a.ccs = ccs;
  a.cvs = cvs;
  a.eps = c->prm.eps;
  a.psi1 = c->psi1;
  a.r = c->prm.r;
  for (int n = 0; n <= c->d + 1; ++n) {
    const double denom = c->prm.lambda0 + n * c->prm.lambda_s;  // R5
    a.l0[n] = c->prm.lambda0 / denom;
    a.inv_l0[n] = 1.0 / a.l0[n];
    a.ls[n] = c->prm.lambda_s / denom;
  }
  int nsm = 148;
  MCK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
  MfFn f = mf_fn(c->d, c->M, c->V);
  constexpr int kWarps = 4;  // warps (cells in flight) per CTA
  const size_t smem =
      (size_t(kWarps) * mf_scr_doubles(c->d, c->M, c->V) + mf_bf_doubles(c->d, c->M)) * sizeof(double);
  MCK(cudaFuncSetAttribute((const void*)f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 1;
  MCK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)f, 32 * kWarps, smem));
  const int64_t warps = cell_end - cell_begin;
  int64_t grid = std::max<int64_t>(1, std::min<int64_t>((warps + kWarps - 1) / kWarps, (int64_t)nsm * std::max(1, occ)));
  if (c->max_ctas > 0) grid = std::min<int64_t>(grid, c->max_ctas);  // CWRECO_OPT_MAX_CTAS
  f<<<(unsigned)grid, 32 * kWarps, smem, (cudaStream_t)stream>>>(m, a);
  MCK(cudaGetLastError());
}

}  // namespace cwr
