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
// One warp per cell (persistent grid): lane L holds the rows k = L, L+32 of A and
// ΔQ (assembled by monomial quadrature exact for degree M, R19); Householder QR
// with warp reductions (shuffle butterflies) applied to the V right-hand sides;
// back substitution with the solution broadcast row by row; lanes 0..d solve the
// sector systems; lanes 0..V−1 then gather their variable's coefficients and run
// cweno_epilogue.  fp64-ALU bound (≈ 2·(n_e−1)·(ℳ−1)² FMAs per cell for the QR),
// HBM traffic ≈ geometry + stencil ids + Q + w per cell.
// Results agree with the oracle within the parity tolerance (not bitwise with the
// matrix kernels: different QR order).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "kcommon.cuh"

namespace cwr {

#define MCK(x)                                                                                 \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) fail(CWRECO_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

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
constexpr int kMfSlots = 6;
static __constant__ double c_mcoef[mf_coef_off(3, 3) + 20 * 20];
static __constant__ double c_qp[kMfSlots * kMfMaxQ * 3];
static __constant__ double c_qw[kMfSlots * kMfMaxQ];

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
    const int c = (code >> (2 * a)) & 3;
    s[a] = c == 1 ? L[a] : c == 2 ? -L[a] : 0.0;
  }
}

// 3×3 / 2×2 inverse by cofactors (as the host's sector inverse); false if det = 0
template <int D>
__device__ __forceinline__ bool inv_small_d(const double (&A)[D][D], double (&Ai)[D][D]) {
  if (D == 2) {
    const double det = A[0][0] * A[1][1] - A[0][1] * A[1][0];
    if (det == 0.0 || !isfinite(det)) return false;
    Ai[0][0] = A[1][1] / det;
    Ai[0][1] = -A[0][1] / det;
    Ai[1][0] = -A[1][0] / det;
    Ai[1][1] = A[0][0] / det;
    return true;
  } else {
    const double c00 = A[1][1] * A[2][2] - A[1][2] * A[2][1], c01 = A[1][2] * A[2][0] - A[1][0] * A[2][2],
                 c02 = A[1][0] * A[2][1] - A[1][1] * A[2][0];
    const double det = A[0][0] * c00 + A[0][1] * c01 + A[0][2] * c02;
    if (det == 0.0 || !isfinite(det)) return false;
    Ai[0][0] = c00 / det;
    Ai[0][1] = (A[0][2] * A[2][1] - A[0][1] * A[2][2]) / det;
    Ai[0][2] = (A[0][1] * A[1][2] - A[0][2] * A[1][1]) / det;
    Ai[1][0] = c01 / det;
    Ai[1][1] = (A[0][0] * A[2][2] - A[0][2] * A[2][0]) / det;
    Ai[1][2] = (A[0][2] * A[1][0] - A[0][0] * A[1][2]) / det;
    Ai[2][0] = c02 / det;
    Ai[2][1] = (A[0][1] * A[2][0] - A[0][0] * A[2][1]) / det;
    Ai[2][2] = (A[0][0] * A[1][1] - A[0][1] * A[1][0]) / det;
    return true;
  }
}

// per-warp shared scratch: R factor, Qᵀ ΔQ, diag(R), sector products
__host__ __device__ constexpr int mf_scr_doubles(int D, int M, int V) {
  return (nmodes(M, D) - 1) * (nmodes(M, D) - 1 + V + 1) + (D + 1) * D * V;
}

template <int D, int M, int V>
__global__ void __launch_bounds__(256) k_matfree(MfArgs m, KArgs a) {
  constexpr int NM = nmodes(M, D), R = NM - 1, NV = D + 1, NE = D * NM, K = NE - 1;
  constexpr int KPL = (K + 31) / 32;  // rows of A per lane

  const int lane = threadIdx.x & 31;
  const double* qp = c_qp + mf_slot(D, M) * kMfMaxQ * 3;  // this (d, M)'s tables
  const double* qw = c_qw + mf_slot(D, M) * kMfMaxQ;
  const double* mcoef = c_mcoef + mf_coef_off(D, M);
  extern __shared__ __align__(16) double mf_smem[];
  double* scr = mf_smem + (threadIdx.x >> 5) * mf_scr_doubles(D, M, V);
  const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = m.cell_begin + w0; i < m.cell_end; i += nw) {
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

    // ---- rows of the reduced system: A[k][l-1] = avg_{T_j} ψ_l(ξ_i(x)), rhs = ΔQ
    double A[KPL][R], rhs[KPL][V];
#pragma unroll
    for (int r = 0; r < KPL; ++r) {
      const int k = lane + 32 * r;
#pragma unroll
      for (int l = 0; l < R; ++l) A[r][l] = 0.0;
#pragma unroll
      for (int v = 0; v < V; ++v) rhs[r][v] = 0.0;
      if (k < K) {
        const int32_t j = m.st[i * K + k];
        double sh[D];
        shift_vec<D>(m.sh[i * K + k], m.L, sh);
        const double* Xj = m.X + int64_t(j) * NV * D;
        double t[D], C[D][D];
#pragma unroll
        for (int e = 0; e < D; ++e) {
          double s = 0.0;
#pragma unroll
          for (int f = 0; f < D; ++f) s += Ji[e][f] * (Xj[f] + sh[f] - X0[f]);
          t[e] = s;
#pragma unroll
          for (int f = 0; f < D; ++f) {
            double s2 = 0.0;
#pragma unroll
            for (int g = 0; g < D; ++g) s2 += Ji[e][g] * (Xj[(f + 1) * D + g] - Xj[g]);
            C[e][f] = s2;
          }
        }
        double mom[NM];  // monomial averages over T_j (ℳ monomials of degree ≤ M)
#pragma unroll
        for (int e = 0; e < NM; ++e) mom[e] = 0.0;
        for (int q = 0; q < m.nq; ++q) {
          double pw[3][M + 1];
#pragma unroll
          for (int e = 0; e < D; ++e) {
            double s = t[e];
#pragma unroll
            for (int f = 0; f < D; ++f) s += C[e][f] * qp[q * D + f];
            pw[e][0] = 1.0;
#pragma unroll
            for (int p = 1; p <= M; ++p) pw[e][p] = pw[e][p - 1] * s;
          }
          if (D == 2) {
#pragma unroll
            for (int p = 0; p <= M; ++p) pw[2][p] = p == 0 ? 1.0 : 0.0;
          }
          const double wq = qw[q];
          constexpr MonoTab MT = mono_tab(D, M);
#pragma unroll
          for (int e = 0; e < NM; ++e) mom[e] += wq * (pw[0][MT.e[e][0]] * pw[1][MT.e[e][1]] * pw[2][MT.e[e][2]]);
        }
#pragma unroll
        for (int l = 1; l < NM; ++l) {
          double s = 0.0;
#pragma unroll
          for (int e = 0; e < NM; ++e) s += mcoef[l * NM + e] * mom[e];
          A[r][l - 1] = s;
        }
#pragma unroll
        for (int v = 0; v < V; ++v) rhs[r][v] = a.Q[int64_t(j) * a.acs + v * a.avs] - qi[v];
      }
    }

    // ---- Householder QR of A (K × R) applied to rhs; R factor left in rows 0..R−1.
    // Per column c: the R+V dot products vᵀ[A|ΔQ] are reduced with a butterfly
    // reduce-scatter (after the xor-o step a lane keeps the half selected by bit o,
    // so lane L ends with column L's full sum: 31 shuffles instead of 5·(R+V)), then
    // all-gathered for the rank-1 update.  The column loop is not unrolled (code size).
    static_assert(R + V <= 32, "one lane per column of A|ΔQ");
    constexpr int NP = R + V <= 16 ? 16 : 32;  // padded column count of the reduce-scatter
    auto qr_step = [&](const int c) {
      double x[KPL];
      double part = 0.0;
#pragma unroll
      for (int r = 0; r < KPL; ++r) {
        const int k = lane + 32 * r;
        double ak = 0.0;
#pragma unroll
        for (int mm = 0; mm < R; ++mm)
          if (mm == c) ak = A[r][mm];
        x[r] = (k >= c && k < K) ? ak : 0.0;
        part += x[r] * x[r];
      }
      const double nrm2 = warp_sum(part);
      const double xc = __shfl_sync(0xffffffffu, x[0], c);  // row c is slot 0 of lane c
      const double alpha = xc >= 0.0 ? -sqrt(nrm2) : sqrt(nrm2);
      const double vtv = 2.0 * (nrm2 - alpha * xc);
      const double tau = vtv > 0.0 ? 2.0 / vtv : 0.0;
      if (lane == c) x[0] -= alpha;
      double dd[NP];
#pragma unroll
      for (int mm = 0; mm < NP; ++mm) {
        double s2 = 0.0;
        if (mm < R + V) {
#pragma unroll
          for (int r = 0; r < KPL; ++r) s2 += x[r] * (mm < R ? A[r][mm] : rhs[r][mm < R ? 0 : mm - R]);
        }
        dd[mm] = s2;
      }
#pragma unroll
      for (int o = NP / 2; o > 0; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i2 = 0; i2 < o; ++i2) {
          const double keep = up ? dd[i2 + o] : dd[i2];
          const double send = up ? dd[i2] : dd[i2 + o];
          dd[i2] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      if (NP == 16) dd[0] += __shfl_xor_sync(0xffffffffu, dd[0], 16);
      const double fl = tau * dd[0];  // lane L: τ·(vᵀ column L mod NP)
#pragma unroll
      for (int mm = 0; mm < R + V; ++mm) {
        const double f = __shfl_sync(0xffffffffu, fl, mm);
        if (mm > c) {
#pragma unroll
          for (int r = 0; r < KPL; ++r) {
            if (mm < R)
              A[r][mm] -= f * x[r];
            else
              rhs[r][mm - R] -= f * x[r];
          }
        }
      }
      if (lane == c) {
#pragma unroll
        for (int mm = 0; mm < R; ++mm)
          if (mm == c) A[0][mm] = alpha;
      }
    };
    if constexpr (R <= 9) {  // small: fully unrolled (column selects fold away)
#pragma unroll
      for (int c = 0; c < R; ++c) qr_step(c);
    } else {  // ℳ ≥ 15: a rolled column loop keeps the code in the instruction cache
#pragma unroll 1
      for (int c = 0; c < R; ++c) qr_step(c);
    }
    // ---- R factor and Qᵀ ΔQ to this warp's shared scratch: lane v < V then solves
    // R p = (Qᵀ ΔQ)[0:R] for its variable, keeping p̂_opt in registers
    double* Rs = scr;                 // [R][R] upper triangle of R
    double* Ys = Rs + R * R;          // [R][V]
    double* Ri = Ys + R * V;          // [R] diagonal of R
    double* PSs = Ri + R;             // [NV][D][V] sector products
    if (lane < R) {
#pragma unroll
      for (int mm = 0; mm < R; ++mm)
        if (mm >= lane) Rs[lane * R + mm] = A[0][mm];
#pragma unroll
      for (int v = 0; v < V; ++v) Ys[lane * V + v] = rhs[0][v];
#pragma unroll
      for (int mm = 0; mm < R; ++mm)
        if (mm == lane) Ri[lane] = A[0][mm];
    }
    // ---- sectors: lane s < d+1 solves sector s for all variables
    double psl[D][V];
    bool vs = false;
#pragma unroll
    for (int l = 0; l < D; ++l)
#pragma unroll
      for (int v = 0; v < V; ++v) psl[l][v] = 0.0;
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
            psl[l][v] = s;
          }
      }
    }

    // ---- per variable (lane v): back substitution, gather, fused epilogue
    if (lane < NV) {
#pragma unroll
      for (int l = 0; l < D; ++l)
#pragma unroll
        for (int v = 0; v < V; ++v) PSs[(lane * D + l) * V + v] = psl[l][v];
    }
    const unsigned vbits = __ballot_sync(0xffffffffu, vs);
    __syncwarp();
    double acc[R], ps[NV][D];
    bool valid[NV];
#pragma unroll
    for (int s2 = 0; s2 < NV; ++s2) valid[s2] = (vbits >> s2) & 1;
    if (lane < V) {
#pragma unroll
      for (int c = R - 1; c >= 0; --c) {
        double t = Ys[c * V + lane];
#pragma unroll
        for (int mm = c + 1; mm < R; ++mm) t -= Rs[c * R + mm] * acc[mm];
        acc[c] = t / Ri[c];
      }
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
  // constants of this translation unit: monomials, basis, rule, packed Σ
  std::vector<double> qp3(nq * 3, 0.0);
  for (int q = 0; q < nq; ++q)
    for (int e = 0; e < c->d; ++e) qp3[q * c->d + e] = h.qp[q * c->d + e];
  const int slot = mf_slot(c->d, c->M);
  MCK(cudaMemcpyToSymbol(c_mcoef, h.mcoef.data(), sizeof(double) * h.mcoef.size(),
                         sizeof(double) * mf_coef_off(c->d, c->M)));
  MCK(cudaMemcpyToSymbol(c_qp, qp3.data(), sizeof(double) * qp3.size(), sizeof(double) * slot * kMfMaxQ * 3));
  MCK(cudaMemcpyToSymbol(c_qw, h.qw.data(), sizeof(double) * h.qw.size(), sizeof(double) * slot * kMfMaxQ));
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
  const size_t smem = size_t(8) * mf_scr_doubles(c->d, c->M, c->V) * sizeof(double);
  MCK(cudaFuncSetAttribute((const void*)f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 1;
  MCK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)f, 256, smem));
  const int64_t warps = cell_end - cell_begin;
  int64_t grid = std::max<int64_t>(1, std::min<int64_t>((warps + 7) / 8, (int64_t)nsm * std::max(1, occ)));
  if (c->max_ctas > 0) grid = std::min<int64_t>(grid, c->max_ctas);  // CWRECO_OPT_MAX_CTAS
  f<<<(unsigned)grid, 256, smem, (cudaStream_t)stream>>>(m, a);
  MCK(cudaGetLastError());
}

}  // namespace cwr
