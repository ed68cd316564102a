// k_predictor: the element-local space-time Galerkin predictor on sm_100a (paper
// §2.2), Eulerian (fixed mesh), Euler equations.
//
// Per owned cell, from the reconstruction polynomial w (cwreco_reconstruct's
// output, Dubiner modes) and Δt:
//   q̂_l = w(ξ_l) at all 𝓛 space-time nodes (initial guess, R35; the τ = 0 ones
//   stay: the known DOFs q̂⁰);
//   Picard (Eq. CGfinal, test functions of the unknown nodes, R33):
//       F̂_l = F(q̂_l) (Eq. PDEterm), Ĝ_b,l = Σ_a (∂ξ_b/∂x_a) F̂_a,l,
//       q̂¹ = −Δt Σ_b A_b Ĝ_b − C0 q̂⁰      A_b = K_uu⁻¹ M_u D_b, C0 = K_uu⁻¹ K_uk
//   until max|Δq̂¹| ≤ 1e-12·max(1, max|q̂⁰|) or 2(M+1) iterations (R35; at the cap
//   an update ≤ 1e-8·max(1, max|q̂⁰|) still counts as converged).
// Output: q̂ [n_owned][𝓛][V] (nodes in the order of cwreco_predictor_nodes) and,
// optionally, per cell the iteration count (negative: not converged or an
// inadmissible state ρ ≤ 0 / p ≤ 0 met at a node).
//
// Layout: a CTA holds CB cells; shared memory q̂[CB][𝓛][V] and Ĝ[CB][d][𝓛][V].
// Flux phase: one thread per (cell, node) evaluates the Euler flux and its
// contravariant components.  Update phase: one thread per (cell, variable) forms
// all NU = 𝓛 − ℳ unknown rows; the universal matrices A_b and C0 live in the
// constant bank (warp-uniform operands), Ĝ is read from shared memory.  A cell
// that has converged is frozen (its iteration count is that of the oracle).
// fp64-ALU bound: ≈ d·NU·𝓛·V FMAs per cell and iteration.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "devguard.cuh"
#include "kcommon.cuh"

namespace cwr {

#define PCK(x)                                                                                 \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) fail(CWRECO_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// 𝓛 = ℳ(M, d+1) space-time nodes, ℳ(M, d) of them known (τ = 0)
__host__ __device__ constexpr int pr_L(int D, int M) {
  return D == 2 ? (M + 1) * (M + 2) * (M + 3) / 6 : (M + 1) * (M + 2) * (M + 3) * (M + 4) / 24;
}
__host__ __device__ constexpr int pr_nk(int D, int M) { return nmodes(M, D); }
__host__ __device__ constexpr int pr_len(int D, int M) {  // doubles of the (D, M) tables: A, C0, Phi
  return D * (pr_L(D, M) - pr_nk(D, M)) * pr_L(D, M) + (pr_L(D, M) - pr_nk(D, M)) * pr_nk(D, M) +
         pr_L(D, M) * pr_nk(D, M);
}
__host__ __device__ constexpr int pr_off(int D, int M) {
  int off = 0;
  for (int dd = 2; dd <= 3; ++dd)
    for (int mm = 1; mm <= 3; ++mm) {
      if (dd == D && mm == M) return off;
      off += pr_len(dd, mm);
    }
  return off;
}
static __constant__ double c_pred[pr_off(4, 1)];

// Update phase as one CTA-wide GEMM on the fp64 tensor cores: -1 = for 3-D M = 3 only
// (C5 51.3 vs 67.2 ms; the smaller shapes pad NU to 8-row tiles and measured slower:
// C3 3.10 vs 2.78, C2 3.39 vs 2.31 ms), 0 = never, 1 = always
#ifndef CWR_PRED_MMA
#define CWR_PRED_MMA -1
#endif
// Tensor-core form of the update (CWR_PRED_MMA): per CTA and iteration
//   U[k][n] = Σ_j A'[k][j] Ĝ[j][n],  j = b·𝓛 + l ∈ [0, d·𝓛),  n = cell·V + v ∈ [0, 32·V)
// with A'[k][b·𝓛 + l] = A_b[k][l] the SAME for every cell: m8n8k4 DMMA tiles, rows k
// padded to MT·8, j to KS·4 (zero), the 32·V/8 column tiles dealt to V·pr_wm warps.
// A' and C0 are stored per lane in fragment order ([k-step][m-tile][lane]) so a lane's
// fragment is one coalesced load (L1-resident tables of ≤ 14 KB).
// cells per CTA (the CTA runs (d+2)·pr_wm warps): CWR_PRED_CB3 for the tensor-core shape
// 3-D M = 3 (5.6 KB of shared state per cell: 32 cells = one CTA per SM, 16 = two)
#ifndef CWR_PRED_CB3
#define CWR_PRED_CB3 32
#endif
__host__ __device__ constexpr int pr_cb(int D, int M) { return D == 3 && M == 3 ? CWR_PRED_CB3 : 32; }
// warps per variable of the tensor-core shape (3-D M = 3): the CB·V/8 column tiles of the
// update GEMM are dealt to (d+2)·pr_wm warps
// (measured, profiles/r02w_predictor_wm_variants.log: C5 37.8 ms with 5 warps, 29.3 ms with 10)
#ifndef CWR_PRED_WM3
#define CWR_PRED_WM3 2
#endif
__host__ __device__ constexpr int pr_wm(int D, int M) { return D == 3 && M == 3 ? CWR_PRED_WM3 : 1; }
__host__ __device__ constexpr int pr_mt(int D, int M) { return (pr_L(D, M) - pr_nk(D, M) + 7) / 8; }
__host__ __device__ constexpr int pr_ks(int D, int M) { return (D * pr_L(D, M) + 3) / 4; }
__host__ __device__ constexpr int pr_ks0(int D, int M) { return (pr_nk(D, M) + 3) / 4; }

struct PredArgs {
  const double* fa;    // A' fragments [KS][MT][32]
  const double* fc;    // C0 fragments [KS0][MT][32]
  const double* w;     // coefficients: (c, v, m) at w[c·ccs + v·cvs + m]
  int64_t ccs, cvs;
  const double* jinv;  // [n_owned][d][d]  ∂ξ_b/∂x_a at [b·d + a]
  double* q;           // [n_owned][𝓛][V]
  int32_t* iters;      // [n_owned] or nullptr
  int64_t n;
  double dt, gamma, tol;
  int maxit;
};

template <int D, int M>
__global__ void __launch_bounds__(pr_wm(D, M) > 1 ? 32 * (D + 2) * pr_wm(D, M) : 256) k_predictor(PredArgs p) {
  constexpr int V = D + 2, L = pr_L(D, M), NK = pr_nk(D, M), NU = L - NK;
  constexpr int CB = pr_cb(D, M);  // cells per CTA
  constexpr int OA = pr_off(D, M), OC = OA + D * NU * L, OP = OC + NU * NK;
  constexpr bool kMma = CWR_PRED_MMA < 0 ? (D == 3 && M == 3) : CWR_PRED_MMA > 0;
  extern __shared__ __align__(16) double psm[];
  double* Q = psm;                                   // [CB][L][V]
  double* G = Q + CB * L * V;                        // [CB][D][L][V]
  double* Ji = G + CB * D * L * V;                   // [CB][D][D]
  double* dl = Ji + CB * D * D;                      // [CB][V] update norms
  double* sc = dl + CB * V;                          // [CB] scales
  int* flag = (int*)(sc + CB);                       // [CB] 0 active, 1 converged; bit 2: inadmissible
  int* its = flag + CB;                              // [CB]
  const int tid = threadIdx.x, nth = blockDim.x;
  for (int64_t c0 = int64_t(blockIdx.x) * CB; c0 < p.n; c0 += int64_t(gridDim.x) * CB) {
    const int nc = (int)(p.n - c0 < CB ? p.n - c0 : CB);
    // ---- initial guess q̂_l = Σ_m Φ[l][m] w_m (every node), per (cell, variable)
    for (int it = tid; it < nc * V; it += nth) {
      const int cl = it / V, v = it - cl * V;
      const double* wp = p.w + (c0 + cl) * p.ccs + v * p.cvs;
      double wm[NK];
#pragma unroll
      for (int m = 0; m < NK; ++m) wm[m] = wp[m];
#pragma unroll
      for (int l = 0; l < L; ++l) {
        double s = 0.0;
#pragma unroll
        for (int m = 0; m < NK; ++m) s = __fma_rn(c_pred[OP + l * NK + m], wm[m], s);
        Q[(cl * L + l) * V + v] = s;
      }
    }
    for (int it = tid; it < nc * D * D; it += nth) Ji[it] = p.jinv[c0 * D * D + it];
    for (int it = tid; it < CB; it += nth) {
      flag[it] = it < nc ? 0 : 1;
      its[it] = 0;
    }
    __syncthreads();
    for (int it = tid; it < nc; it += nth) {  // scale = max(1, max|q̂⁰|)
      double s = 1.0;
      for (int e = 0; e < NK * V; ++e) s = fmax(s, fabs(Q[it * L * V + e]));
      sc[it] = s;
    }
    constexpr int MT = pr_mt(D, M), KS = pr_ks(D, M), KS0 = pr_ks0(D, M), DL = D * L;
    constexpr int NTW = CB / 8 / pr_wm(D, M);  // column tiles per warp: CB·V columns / 8 / (V·pr_wm warps)
    const int lane = tid & 31, warp = tid >> 5;
    int nb[NTW];
    double basef[MT][NTW][2];
    // scalar form: C0 q̂⁰ is fixed: kept in registers by the update threads (≤ 1 item per thread)
    const int ui = tid;
    const bool upd = ui < nc * V;
    const int ucl = upd ? ui / V : 0, uv = upd ? ui - (ui / V) * V : 0;
    double base[NU];
    if constexpr (kMma) {
      // this lane's B-fragment column n = (nt0 + t)·8 + lane/4 and its element offset
#pragma unroll
      for (int t = 0; t < NTW; ++t) {
        const int n = (warp * NTW + t) * 8 + (lane >> 2), cl = n / V;
        nb[t] = cl * (D * L * V) + (n - cl * V);
      }
      // C0 q̂⁰ (fixed over the iterations) in accumulator layout (q̂¹ = −Δt·U − basef)
      {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int t = 0; t < NTW; ++t) basef[mt][t][0] = basef[mt][t][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < KS0; ++ks) {
          const int j = ks * 4 + (lane & 3);
          double fb[NTW];
#pragma unroll
          for (int t = 0; t < NTW; ++t) {  // Q⁰[cell][j][v] = Q[(cell·L + j)·V + v], n-offset as for Ĝ
            const int n = (warp * NTW + t) * 8 + (lane >> 2), cl = n / V;
            fb[t] = j < NK ? Q[(cl * L + j) * V + (n - cl * V)] : 0.0;
          }
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            const double fa = __ldg(p.fc + (ks * MT + mt) * 32 + lane);
#pragma unroll
            for (int t = 0; t < NTW; ++t) dmma884(basef[mt][t][0], basef[mt][t][1], fa, fb[t]);
          }
        }
      }
    } else {
      if (upd) {
#pragma unroll
        for (int k = 0; k < NU; ++k) {
          double s = 0.0;
#pragma unroll
          for (int j = 0; j < NK; ++j) s = __fma_rn(c_pred[OC + k * NK + j], Q[(ucl * L + j) * V + uv], s);
          base[k] = -s;
        }
      }
    }
    for (int iter = 0; iter < p.maxit; ++iter) {
      __syncthreads();
      // ---- flux phase: (cell, node) → Ĝ_b = Σ_a Jinv[b][a] F_a(q̂)
      for (int it = tid; it < nc * L; it += nth) {
        const int cl = it / L, l = it - cl * L;
        if (flag[cl] & 1) continue;
        const double* qn = Q + (cl * L + l) * V;
        double q[V];
#pragma unroll
        for (int v = 0; v < V; ++v) q[v] = qn[v];
        const double rho = q[0], E = q[D + 1];
        const double ir = 1.0 / rho;
        double u[D], ke = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          u[a] = q[1 + a] * ir;
          ke = __fma_rn(q[1 + a], u[a], ke);
        }
        const double pr = (p.gamma - 1.0) * (E - 0.5 * ke);
        if (!(rho > 0.0) || !(pr > 0.0)) atomicOr(&flag[cl], 4);
        double F[D][V];
#pragma unroll
        for (int a = 0; a < D; ++a) {
          F[a][0] = q[1 + a];
#pragma unroll
          for (int b = 0; b < D; ++b) F[a][1 + b] = q[1 + a] * u[b] + (a == b ? pr : 0.0);
          F[a][D + 1] = u[a] * (E + pr);
        }
        const double* J = Ji + cl * D * D;
#pragma unroll
        for (int b = 0; b < D; ++b)
#pragma unroll
          for (int v = 0; v < V; ++v) {
            double s = 0.0;
#pragma unroll
            for (int a = 0; a < D; ++a) s = __fma_rn(J[b * D + a], F[a][v], s);
            G[((cl * D + b) * L + l) * V + v] = s;
          }
      }
      __syncthreads();
      // ---- update phase: (cell, variable) → the NU unknown rows
      if constexpr (kMma) {
        {
          double acc[MT][NTW][2];
#pragma unroll
          for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int t = 0; t < NTW; ++t) acc[mt][t][0] = acc[mt][t][1] = 0.0;
#pragma unroll 3
          for (int ks = 0; ks < KS; ++ks) {
            const int j = ks * 4 + (lane & 3);
            double fb[NTW], fa[MT];
#pragma unroll
            for (int t = 0; t < NTW; ++t) fb[t] = j < DL ? G[nb[t] + j * V] : 0.0;
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) fa[mt] = __ldg(p.fa + (ks * MT + mt) * 32 + lane);
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
              for (int t = 0; t < NTW; ++t) dmma884(acc[mt][t][0], acc[mt][t][1], fa[mt], fb[t]);
          }
          // q̂¹ = −Δt·U − C0 q̂⁰ on the lane's elements (row k = mt·8 + lane/4, columns
          // n = tile·8 + 2·(lane%4) + e); frozen cells keep their state
          double dm[NTW][2];
#pragma unroll
          for (int t = 0; t < NTW; ++t) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int n = (warp * NTW + t) * 8 + 2 * (lane & 3) + e, cl = n / V, v = n - cl * V;
              const bool live = cl < nc && !(flag[cl] & 1);
              double mx = 0.0;
#pragma unroll
              for (int mt = 0; mt < MT; ++mt) {
                const int k = mt * 8 + (lane >> 2);
                if (live && k < NU) {
                  double* qk = Q + (cl * L + NK + k) * V + v;
                  const double nv = __fma_rn(-p.dt, acc[mt][t][e], -basef[mt][t][e]);
                  mx = fmax(mx, fabs(nv - *qk));
                  *qk = nv;
                }
              }
              dm[t][e] = mx;
            }
          }
          // max over the rows k: lanes with the same lane%4 hold the same columns
#pragma unroll
          for (int t = 0; t < NTW; ++t)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              double x = dm[t][e];
              x = fmax(x, __shfl_xor_sync(0xffffffffu, x, 4));
              x = fmax(x, __shfl_xor_sync(0xffffffffu, x, 8));
              x = fmax(x, __shfl_xor_sync(0xffffffffu, x, 16));
              const int n = (warp * NTW + t) * 8 + 2 * (lane & 3) + e;
              if ((lane >> 2) == 0 && n < nc * V) dl[n] = x;
            }
        }
      } else {
        if (upd && !(flag[ucl] & 1)) {
          double acc[NU];
#pragma unroll
          for (int k = 0; k < NU; ++k) acc[k] = 0.0;
          const double* Gc = G + (ucl * D * L) * V + uv;
#pragma unroll
          for (int b = 0; b < D; ++b)
#pragma unroll
            for (int l = 0; l < L; ++l) {
              const double g = Gc[(b * L + l) * V];
#pragma unroll
              for (int k = 0; k < NU; ++k) acc[k] = __fma_rn(c_pred[OA + (b * NU + k) * L + l], g, acc[k]);
            }
          double dmax = 0.0;
          double* qu = Q + (ucl * L + NK) * V + uv;
#pragma unroll
          for (int k = 0; k < NU; ++k) {
            const double nv = __fma_rn(-p.dt, acc[k], base[k]);
            dmax = fmax(dmax, fabs(nv - qu[k * V]));
            qu[k * V] = nv;
          }
          dl[ucl * V + uv] = dmax;
        }
      }
      __syncthreads();
      int active = 0;
      for (int cl = tid; cl < nc; cl += nth) {
        if (flag[cl] & 1) continue;
        its[cl] = iter + 1;
        double dm = 0.0;
        for (int v = 0; v < V; ++v) dm = fmax(dm, dl[cl * V + v]);
        if (dm <= p.tol * sc[cl])
          flag[cl] |= 1;
        else if (iter + 1 == p.maxit)
          flag[cl] |= dm <= 1e-8 * sc[cl] ? 8 : 0;  // R35: acceptable update at the cap
        else
          active = 1;
      }
      if (!__syncthreads_or(active)) break;
    }
    __syncthreads();
    // ---- the last iterate's states: admissibility of the final q̂ (as the oracle)
    for (int it = tid; it < nc * L; it += nth) {
      const int cl = it / L, l = it - cl * L;
      const double* qn = Q + (cl * L + l) * V;
      double ke = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) ke = __fma_rn(qn[1 + a], qn[1 + a] / qn[0], ke);
      const double pr = (p.gamma - 1.0) * (qn[D + 1] - 0.5 * ke);
      if (!(qn[0] > 0.0) || !(pr > 0.0)) atomicOr(&flag[cl], 4);
    }
    __syncthreads();
    // ---- store q̂ (contiguous [cell][L][V] rows) and the iteration counts
    double* qo = p.q + c0 * L * V;
    for (int e = tid; e < nc * L * V; e += nth) qo[e] = Q[e];
    if (p.iters)
      for (int cl = tid; cl < nc; cl += nth)
        p.iters[c0 + cl] = ((flag[cl] & 9) && !(flag[cl] & 4)) ? its[cl] : -its[cl] - 1;
    __syncthreads();
  }
}

using PredFn = void (*)(PredArgs);
static PredFn pred_fn(int d, int M) {
#define PC(DD, MM) \
  if (d == DD && M == MM) return k_predictor<DD, MM>;
  PC(2, 1) PC(2, 2) PC(2, 3) PC(3, 1) PC(3, 2) PC(3, 3)
#undef PC
  fail(CWRECO_EUNSUPPORTED, "predictor: (d, M) not instantiated (M ≤ 3)");
}
static size_t pred_smem(int d, int M) {
  const int L = pr_L(d, M), V = d + 2, CB = pr_cb(d, M);
  return sizeof(double) * (size_t(CB) * L * V * (1 + d) + CB * d * d + CB * V + CB) + 2 * sizeof(int) * CB;
}

struct PredState {
  double* frag = nullptr;  // A' fragments, then C0 fragments (CWR_PRED_MMA)
  double* jinv = nullptr;
  double gamma = 1.4;
  int L = 0;
};

void dev_predictor_setup(cwreco_ctx* c, const PredictorHost& h, const std::vector<double>& jinv, double gamma) {
  if (c->device < 0) fail(CWRECO_ECUDA, "predictor_setup: host-only context (no CUDA device)");
  if (c->V != c->d + 2) fail(CWRECO_EUNSUPPORTED, "predictor: the Euler system needs nvars = dim + 2");
  PredFn f = pred_fn(c->d, c->M);
  DeviceGuard dg(c->device);
  if (pr_L(c->d, c->M) != h.L || pr_nk(c->d, c->M) != h.nk) fail(CWRECO_EUNSUPPORTED, "predictor: table shape");
  std::vector<double> tab;
  tab.insert(tab.end(), h.A.begin(), h.A.end());
  tab.insert(tab.end(), h.C0.begin(), h.C0.end());
  tab.insert(tab.end(), h.Phi.begin(), h.Phi.end());
  if ((int)tab.size() != pr_len(c->d, c->M)) fail(CWRECO_EUNSUPPORTED, "predictor: table length");
  PCK(cudaMemcpyToSymbol(c_pred, tab.data(), tab.size() * sizeof(double), sizeof(double) * pr_off(c->d, c->M)));
  PCK(cudaFuncSetAttribute((const void*)f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pred_smem(c->d, c->M)));
  auto* s = (PredState*)c->pred;
  if (!s) c->pred = s = new PredState();
  cudaFree(s->jinv);
  s->jinv = nullptr;
  // A'[k][b·L + l] = A_b[k][l] and C0[k][j] in DMMA A-fragment order [ks][mt][lane]:
  // lane holds row mt·8 + lane/4, column ks·4 + lane%4 (zero outside the matrix)
  {
    const int d = c->d, L = h.L, nk = h.nk, nu = L - nk;
    const int mt = (nu + 7) / 8, ks = (d * L + 3) / 4, ks0 = (nk + 3) / 4;
    std::vector<double> fr(size_t(ks + ks0) * mt * 32, 0.0);
    for (int a = 0; a < ks; ++a)
      for (int m = 0; m < mt; ++m)
        for (int ln = 0; ln < 32; ++ln) {
          const int k = m * 8 + ln / 4, j = a * 4 + ln % 4;
          if (k < nu && j < d * L) fr[(size_t(a) * mt + m) * 32 + ln] = h.A[(size_t(j / L) * nu + k) * L + j % L];
        }
    const size_t o0 = size_t(ks) * mt * 32;
    for (int a = 0; a < ks0; ++a)
      for (int m = 0; m < mt; ++m)
        for (int ln = 0; ln < 32; ++ln) {
          const int k = m * 8 + ln / 4, j = a * 4 + ln % 4;
          if (k < nu && j < nk) fr[o0 + (size_t(a) * mt + m) * 32 + ln] = h.C0[size_t(k) * nk + j];
        }
    cudaFree(s->frag);
    s->frag = nullptr;
    PCK(cudaMalloc(&s->frag, fr.size() * sizeof(double)));
    PCK(cudaMemcpy(s->frag, fr.data(), fr.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  PCK(cudaMalloc(&s->jinv, std::max<size_t>(1, jinv.size()) * sizeof(double)));
  if (!jinv.empty()) PCK(cudaMemcpy(s->jinv, jinv.data(), jinv.size() * sizeof(double), cudaMemcpyHostToDevice));
  s->gamma = gamma;
  s->L = h.L;
}

void dev_predictor_destroy(cwreco_ctx* c) {
  auto* s = (PredState*)c->pred;
  if (!s) return;
  DeviceGuard dg(c->device);
  cudaFree(s->jinv);
  cudaFree(s->frag);
  delete s;
  c->pred = nullptr;
}

void dev_predict(cwreco_ctx* c, const double* w, int64_t ccs, int64_t cvs, double dt, double* q, int32_t* iters,
                 void* stream) {
  auto* s = (PredState*)c->pred;
  if (!s) fail(CWRECO_ESTATE, "predict: call cwreco_predictor_setup first");
  DeviceGuard dg(c->device);
  PredArgs a;
  a.fa = s->frag;
  a.fc = s->frag + size_t(pr_ks(c->d, c->M)) * pr_mt(c->d, c->M) * 32;
  a.w = w;
  a.ccs = ccs;
  a.cvs = cvs;
  a.jinv = s->jinv;
  a.q = q;
  a.iters = iters;
  a.n = c->n_owned;
  a.dt = dt;
  a.gamma = s->gamma;
  a.tol = 1e-12;
  a.maxit = 2 * (c->M + 1);
  if (a.n == 0) return;
  PredFn f = pred_fn(c->d, c->M);
  int occ = 1, nsm = 148;
  const size_t smem = pred_smem(c->d, c->M);
  PCK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)f, 32 * (c->d + 2) * pr_wm(c->d, c->M), smem));
  PCK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
  const int64_t blocks = (a.n + pr_cb(c->d, c->M) - 1) / pr_cb(c->d, c->M);
  int64_t grid = std::min<int64_t>(blocks, (int64_t)nsm * std::max(1, occ));
  if (c->max_ctas > 0) grid = std::min<int64_t>(grid, c->max_ctas);
  f<<<(unsigned)grid, 32 * (c->d + 2) * pr_wm(c->d, c->M), smem, (cudaStream_t)stream>>>(a);
  PCK(cudaGetLastError());
}

}  // namespace cwr
