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
// only on which local vertices the sorted face vertices are (code = Σ_a loc_a·(d+1)^a),
// so one table serves every cell.  traces[i][f][q][v] = Σ_l w[i][v][l] Φ[code(i,f)][q][l].
// HBM-bound: read w (ℳ·V doubles per cell, L1-shared by the cell's (d+1)·nq threads),
// write (d+1)·nq·V doubles per cell.
#include <cuda_runtime.h>

#include <string>
#include <vector>

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
};

template <int NM, int V>
__global__ void __launch_bounds__(256) k_traces(const double* __restrict__ w, int64_t ccs, int64_t cvs,
                                                const double* __restrict__ phi, const uint8_t* __restrict__ code,
                                                int nf, int nq, int64_t n_owned, double* __restrict__ out) {
  const int64_t gid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;  // (cell, face, point)
  const int64_t per = int64_t(nf) * nq;
  if (gid >= n_owned * per) return;
  const int64_t i = gid / per;
  const int fq = int(gid - i * per), f = fq / nq, q = fq - f * nq;
  const double* p = phi + (int64_t(code[i * nf + f]) * nq + q) * NM;
  double ph[NM];
#pragma unroll
  for (int l = 0; l < NM; ++l) ph[l] = p[l];
  const double* wi = w + i * ccs;
  double* o = out + gid * V;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    double t = 0.0;
#pragma unroll
    for (int l = 0; l < NM; ++l) t = __fma_rn(wi[v * cvs + l], ph[l], t);
    o[v] = t;
  }
}

using TrFn = void (*)(const double*, int64_t, int64_t, const double*, const uint8_t*, int, int, int64_t, double*);
template <int NM>
static TrFn tr_fn_v(int V) {
  switch (V) {
    case 1: return k_traces<NM, 1>;
    case 2: return k_traces<NM, 2>;
    case 3: return k_traces<NM, 3>;
    case 4: return k_traces<NM, 4>;
    case 5: return k_traces<NM, 5>;
    case 6: return k_traces<NM, 6>;
    case 7: return k_traces<NM, 7>;
    case 8: return k_traces<NM, 8>;
    case 9: return k_traces<NM, 9>;
    default: return nullptr;
  }
}
static TrFn tr_fn(int nm, int V) {
  TrFn f = nullptr;
  switch (nm) {
    case 3: f = tr_fn_v<3>(V); break;
    case 4: f = tr_fn_v<4>(V); break;
    case 6: f = tr_fn_v<6>(V); break;
    case 10: f = tr_fn_v<10>(V); break;
    case 15: f = tr_fn_v<15>(V); break;
    case 20: f = tr_fn_v<20>(V); break;
  }
  if (!f) fail(CWRECO_EUNSUPPORTED, "face traces: nvars must be ≤ 9");
  return f;
}

void dev_traces_destroy(cwreco_ctx* c) {
  TraceState* t = (TraceState*)c->tr;
  if (!t) return;
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
  std::vector<double> phi(size_t(ncode) * nq * nm, 0.0);
  for (int code = 0; code < ncode; ++code) {
    int loc[3], x = code;
    for (int a = 0; a < d; ++a) {
      loc[a] = x % nv;
      x /= nv;
    }
    for (int q = 0; q < nq; ++q) {
      double xi[3] = {0.0, 0.0, 0.0};
      for (int a = 0; a < d; ++a)
        if (loc[a] > 0) xi[loc[a] - 1] += lam[q * d + a];
      basis_eval(d, c->M, xi, &phi[(size_t(code) * nq + q) * nm]);
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
      codes[li * nv + f] = (uint8_t)code;
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
}

void dev_face_traces(cwreco_ctx* c, const double* coeffs, int64_t ccs, int64_t cvs, double* traces, void* stream) {
  TCK(cudaSetDevice(c->device));
  if (!c->tr) traces_prepare(c);
  TraceState* t = (TraceState*)c->tr;
  const int nv = c->d + 1;
  const int64_t threads = c->n_owned * nv * t->nq;
  if (threads == 0) return;
  TrFn f = tr_fn(c->nm, c->V);
  f<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(coeffs, ccs, cvs, t->phi, t->code, nv, t->nq,
                                                                          c->n_owned, traces);
  TCK(cudaGetLastError());
}

}  // namespace cwr
