// Face traces of the reconstruction polynomials:
// the values w_i(x) of every owned cell's blended polynomial at the quadrature
// points of its d+1 faces — the left/right states q_h^∓ a Rusanov-type flux
// (Eq. rusanov) consumes.
//
// Face rule: Gauss–Legendre on an edge (2-D) / collapsed Gauss–Jacobi on a
// triangle (3-D), M+1 points per direction (exact for degree 2M+1 on the face),
// given as barycentric weights over the face's vertices SORTED BY GLOBAL NODE ID,
// so the two cells sharing a face evaluate at the same physical points in the same
// order.  In cell i's reference coordinates a face point is Σ_a λ_a ξ(vertex_a)
// with ξ(vertex 0) = 0, ξ(vertex k) = e_k: the basis values Φ[code][q][l] depend
// only on which local vertices the sorted face vertices are (24 orders in 3-D, 6 in
// 2-D), so one table serves every cell; persistent blocks keep it in shared memory.  traces[i][f][q][v] = Σ_l w[i][v][l] Φ[code(i,f)][q][l].
// HBM-bound: read w (ℳ·V doubles per cell, L1-shared by the cell's (d+1)·nq threads),
// write (d+1)·nq·V doubles per cell.
#include <cuda_runtime.h>

#include <cstdlib>
#include <string>
#include <vector>

#include "devguard.cuh"
#include "internal.hpp"

namespace cwr {

#define TCK(x)                                                                                 \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) fail(CWRECO_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct TraceState {
  double* phi = nullptr;     // [(d+1)^d][nq][ℳ]
  uint8_t* code = nullptr;   // [n_owned][d+1]
  int nq = 0;
  int ncc = 0;  // compact vertex-order codes (table rows / nq)
};

// A block handles CB consecutive cells.  Work unit = (cell, face, block of QB points):
// a V × QB register tile streamed over the ℳ modes (per mode V coefficient loads and
// QB table loads feed V·QB FMAs, so a cell's coefficients are read (d+1)·nq/QB
// times, not (d+1)·nq).  The tiles land in shared memory in the output layout and
// the block's contiguous output region is written with coalesced stores.
template <int NM, int V, int QB>
__global__ void __launch_bounds__(256) k_traces(const double* __restrict__ w, int64_t ccs, int64_t cvs,
                                                const double* __restrict__ phi, int phi_n,
                                                const uint8_t* __restrict__ code, int nf, int nq, int cb,
                                                int64_t n_owned, double* __restrict__ out) {
  extern __shared__ __align__(16) double tr_smem[];  // [phi_n] table, then [cb][nf][nq][V] staging
  double* ph_s = tr_smem;
  double* st = tr_smem + ((phi_n + 1) & ~1);
  for (int k = threadIdx.x; k < phi_n; k += blockDim.x) ph_s[k] = phi[k];  // once per persistent block
  const int nb = nq / QB, units = nf * nb;
  const int64_t ngroups = (n_owned + cb - 1) / cb;
  for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    __syncthreads();  // table loaded / staging free again
    const int64_t c0 = grp * cb;
    const int ncell = (int)min((int64_t)cb, n_owned - c0);
    const int u = threadIdx.x;
    if (u < ncell * units) {
      const int cl = u / units, fb = u - cl * units, f = fb / nb, q0 = (fb - f * nb) * QB;
      const int64_t i = c0 + cl;
      const double* p = ph_s + (int(code[i * nf + f]) * nq + q0) * NM;
      const double* wi = w + i * ccs;
      double acc[V][QB];
#pragma unroll
      for (int v = 0; v < V; ++v)
#pragma unroll
        for (int b = 0; b < QB; ++b) acc[v][b] = 0.0;
#pragma unroll
      for (int l = 0; l < NM; ++l) {
        double ph[QB], wv[V];
#pragma unroll
        for (int b = 0; b < QB; ++b) ph[b] = p[b * NM + l];
#pragma unroll
        for (int v = 0; v < V; ++v) wv[v] = __ldg(wi + v * cvs + l);
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
          for (int b = 0; b < QB; ++b) acc[v][b] = __fma_rn(wv[v], ph[b], acc[v][b]);
      }
      double* o = st + ((cl * nf + f) * nq + q0) * V;
#pragma unroll
      for (int b = 0; b < QB; ++b)
#pragma unroll
        for (int v = 0; v < V; ++v) o[b * V + v] = acc[v][b];
    }
    __syncthreads();
    const int n = ncell * nf * nq * V;
    double* dst = out + c0 * nf * nq * V;
    for (int k = threadIdx.x; k < n; k += blockDim.x) dst[k] = st[k];
  }
}

using TrFn = void (*)(const double*, int64_t, int64_t, const double*, int, const uint8_t*, int, int, int, int64_t,
                      double*);
template <int NM, int QB>
static TrFn tr_fn_v(int V) {
  switch (V) {
    case 1: return k_traces<NM, 1, QB>;
    case 2: return k_traces<NM, 2, QB>;
    case 3: return k_traces<NM, 3, QB>;
    case 4: return k_traces<NM, 4, QB>;
    case 5: return k_traces<NM, 5, QB>;
    case 6: return k_traces<NM, 6, QB>;
    case 7: return k_traces<NM, 7, QB>;
    case 8: return k_traces<NM, 8, QB>;
    case 9: return k_traces<NM, 9, QB>;
    default: return nullptr;
  }
}
// points per work unit (measured, tools/traces_bench.py with CWRECO_TRACE_QB, table in
// shared memory): 3 for the 9-point faces of 3-D M = 2 (C3 1.08 ms), 2 for ℳ = 20 (C5:
// 15.5 ms at 1, 13.9 at 2, 20.5 at 4), otherwise 1 (C2: 0.134 ms at 1, 0.145 at 2)
static int tr_qb(int nq, int nm) { return (nq % 3 == 0 && nm <= 10) ? 3 : (nm >= 20 && nq % 2 == 0) ? 2 : 1; }
static TrFn tr_fn(int nm, int V, int qb) {
  TrFn f = nullptr;
#define TRC(NMV)                                   \
  case NMV:                                        \
    f = qb == 4   ? tr_fn_v<NMV, 4>(V)             \
        : qb == 3 ? tr_fn_v<NMV, 3>(V)             \
        : qb == 2 ? tr_fn_v<NMV, 2>(V)             \
                  : tr_fn_v<NMV, 1>(V);            \
    break;
  switch (nm) {
    TRC(3)
    TRC(4)
    TRC(6)
    TRC(10)
    TRC(15)
    TRC(20)
  }
#undef TRC
  if (!f) fail(CWRECO_EUNSUPPORTED, "face traces: nvars must be ≤ 9");
  return f;
}

void dev_traces_destroy(cwreco_ctx* c) {
  TraceState* t = (TraceState*)c->tr;
  if (!t) return;
  DeviceGuard dg(c->device);
  cudaFree(t->phi);
  cudaFree(t->code);
  delete t;
  c->tr = nullptr;
}

// Host: the table Φ and the per-(cell, face) codes (owned cells, local order).
static void traces_prepare(cwreco_ctx* c) {
  const int d = c->d, nv = d + 1, nm = c->nm;
  std::vector<double> lam, wts;
  face_rule(d, c->M, lam, wts);
  const int nq = (int)wts.size();
  int ncode = 1;
  for (int a = 0; a < d; ++a) ncode *= nv;
  // compact ids of the codes whose d vertices are distinct (24 in 3-D, 6 in 2-D)
  std::vector<int> compact(ncode, -1), full_of;
  for (int code = 0; code < ncode; ++code) {
    int loc[3], x = code, ok = 1;
    for (int a = 0; a < d; ++a) {
      loc[a] = x % nv;
      x /= nv;
      for (int b = 0; b < a; ++b) ok &= loc[b] != loc[a];
    }
    if (ok) {
      compact[code] = (int)full_of.size();
      full_of.push_back(code);
    }
  }
  const int ncc = (int)full_of.size();
  std::vector<double> phi(size_t(ncc) * nq * nm, 0.0);
  for (int cc = 0; cc < ncc; ++cc) {
    const int code = full_of[cc];
    int loc[3], x = code;
    for (int a = 0; a < d; ++a) {
      loc[a] = x % nv;
      x /= nv;
    }
    for (int q = 0; q < nq; ++q) {
      double xi[3] = {0.0, 0.0, 0.0};
      for (int a = 0; a < d; ++a)
        if (loc[a] > 0) xi[loc[a] - 1] += lam[q * d + a];
      basis_eval(d, c->M, xi, &phi[(size_t(cc) * nq + q) * nm]);
    }
  }
  std::vector<uint8_t> codes(c->n_owned * nv, 0);
  for (int64_t li = 0; li < c->n_owned; ++li) {
    const int64_t g = c->local2global[li];
    for (int f = 0; f < nv; ++f) {
      int loc[3], n = 0;
      for (int k = 0; k < nv; ++k)
        if (k != f) loc[n++] = k;
      // sort the face's local vertices by global node id (ascending)
      for (int a = 1; a < d; ++a)
        for (int b = a; b > 0 && c->cell_nodes[g * nv + loc[b]] < c->cell_nodes[g * nv + loc[b - 1]]; --b)
          std::swap(loc[b], loc[b - 1]);
      int code = 0, p = 1;
      for (int a = 0; a < d; ++a, p *= nv) code += loc[a] * p;
      codes[li * nv + f] = (uint8_t)compact[code];
    }
  }
  if (!c->tr) c->tr = new TraceState();
  TraceState* t = (TraceState*)c->tr;
  cudaFree(t->phi);
  cudaFree(t->code);
  t->phi = nullptr;
  t->code = nullptr;
  TCK(cudaMalloc(&t->phi, phi.size() * sizeof(double)));
  TCK(cudaMalloc(&t->code, std::max<size_t>(1, codes.size())));
  TCK(cudaMemcpy(t->phi, phi.data(), phi.size() * sizeof(double), cudaMemcpyHostToDevice));
  if (!codes.empty()) TCK(cudaMemcpy(t->code, codes.data(), codes.size(), cudaMemcpyHostToDevice));
  t->nq = nq;
  t->ncc = ncc;
}

void dev_face_traces(cwreco_ctx* c, const double* coeffs, int64_t ccs, int64_t cvs, double* traces, void* stream) {
  DeviceGuard dg(c->device);
  if (!c->tr) traces_prepare(c);
  TraceState* t = (TraceState*)c->tr;
  const int nv = c->d + 1;
  int qb = tr_qb(t->nq, c->nm);
#ifdef CWRECO_EXPERIMENTS
  if (const char* e = std::getenv("CWRECO_TRACE_QB")) {  // tuning experiments only
    const int x = std::atoi(e);
    if (x >= 1 && x <= 4 && t->nq % x == 0) qb = x;
  }
#endif
  const int units = nv * (t->nq / qb);
  const int cb = std::max(1, 256 / units);
  const int64_t groups = (c->n_owned + cb - 1) / cb;
  if (groups == 0) return;
  const int phi_n = t->ncc * t->nq * c->nm;
  const size_t smem = (size_t((phi_n + 1) & ~1) + size_t(cb) * nv * t->nq * c->V) * sizeof(double);
  TrFn f = tr_fn(c->nm, c->V, qb);
  TCK(cudaFuncSetAttribute((const void*)f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 1, nsm = 148;
  TCK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)f, 256, smem));
  TCK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
  const int64_t grid = std::min<int64_t>(groups, (int64_t)nsm * std::max(1, occ));
  f<<<(unsigned)grid, 256, smem, (cudaStream_t)stream>>>(coeffs, ccs, cvs, t->phi, phi_n, t->code, nv, t->nq, cb,
                                                         c->n_owned, traces);
  TCK(cudaGetLastError());
}

}  // namespace cwr
