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

#include "kcommon.cuh"

#ifndef CWR_TR_V2
#define CWR_TR_V2 1  // staged-block kernel k_traces2 (else the register-tile kernel k_traces)
#endif

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

// ---- k_traces2: a block of cb consecutive cells per step (persistent grid), the cells'
// coefficients double-buffered in shared memory (one TMA bulk copy per step, the next
// step's issued before this step's arithmetic), the basis table transposed to
// Φ[code][l][q] so a thread's P consecutive points are 128-bit loads, every coefficient
// pair a 128-bit broadcast load; a thread computes a P × V tile (points × variables)
// of one face, the tiles land in shared memory in output order and the block's
// contiguous output leaves in one bulk store that drains during the next step.
template <int D, int M, int V>
struct TrShape {
  static constexpr int NM = nmodes(M, D), NF = D + 1, NQ = D == 2 ? M + 1 : (M + 1) * (M + 1);
  static constexpr int P = NQ % 4 == 0 ? 4 : NQ % 3 == 0 ? 3 : NQ % 2 == 0 ? 2 : 1;  // points per thread
  static constexpr int UN = NF * NQ / P;        // threads per cell
  static constexpr int NMP = (NM + 1) & ~1;     // staged coefficient row (even: pair loads)
  static constexpr int WC = V * NMP;            // staged doubles per cell
  static constexpr int OUTC = NF * NQ * V;      // output doubles per cell
  static constexpr int TMAX = V > 6 ? 352 : 512;  // threads per CTA (P × V accumulators: 184 registers for V > 6)
};

template <int D, int M, int V>
__global__ void __launch_bounds__(TrShape<D, M, V>::TMAX) k_traces2(const double* __restrict__ w, int64_t ccs, int64_t cvs,
                                                 const double* __restrict__ phi, int ncc,
                                                 const uint8_t* __restrict__ code, int cb, int64_t n_owned,
                                                 double* __restrict__ out, int bulk_in, int bulk_out, int ng) {
  using S = TrShape<D, M, V>;
  constexpr int NM = S::NM, NF = S::NF, NQ = S::NQ, P = S::P, NMP = S::NMP, WC = S::WC, OUTC = S::OUTC;
  // 16-point faces (3-D M = 3): a thread owns the point pairs t and t+4 of the row's 8
  // and reads them in face-parity order, so the two faces of a quarter-warp touch
  // disjoint banks on every 128-bit Φ load (4 threads of a face read 64 of a row's 128
  // bytes; with q0 = 4t ownership both faces hit the same 16 banks: 2-way conflicts on
  // the load that bounds this kernel); the output pieces land conflict-free as well
#ifndef CWR_TR_SWZ
#define CWR_TR_SWZ 1
#endif
  constexpr bool SWZ = CWR_TR_SWZ && NQ == 16 && P == 4;
  extern __shared__ __align__(16) double tr2_smem[];
  __shared__ __align__(8) uint64_t bars[2][2];
  // ng thread groups share the table Φ and walk their own blocks of cells with their own
  // buffers, mbarriers and named barrier: one group's arithmetic overlaps the other's
  // output staging and waits (the phases of a single group run one after the other)
  const int bd = blockDim.x / ng, grp_id = threadIdx.x / bd, tid = threadIdx.x - grp_id * bd;
  const int phn = (ncc * NM * NQ + 1) & ~1;
  double* ph = tr2_smem;                                          // [ncc][NM][NQ]
  double* wb0 = ph + phn + grp_id * ((cb * (2 * WC + OUTC) + 1) & ~1);  // 2 × [cb][V][NMP]
  double* ob = wb0 + 2 * cb * WC;                                 // [cb][NF][NQ][V]
  uint64_t* bar = bars[grp_id];
  auto group_sync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(1 + grp_id), "r"(bd) : "memory"); };
  for (int k = threadIdx.x; k < ncc * NQ * NM; k += blockDim.x) {  // global table is [code][q][l]
    const int cc = k / (NQ * NM), r = k - cc * (NQ * NM), q = r / NM, l = r - q * NM;
    ph[(cc * NM + l) * NQ + q] = phi[k];
  }
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const int64_t ngroups = (n_owned + cb - 1) / cb;
  const int64_t first = (int64_t)blockIdx.x * ng + grp_id, step = (int64_t)gridDim.x * ng;
  auto issue = [&](int64_t grp, int buf) {
    const int64_t c0 = grp * cb;
    const int ncell = (int)min((int64_t)cb, n_owned - c0);
    double* wb = wb0 + buf * cb * WC;
    if (bulk_in) {
      if (tid == 0) {
        const uint32_t bytes = uint32_t(ncell) * WC * 8;
        mbar_expect_tx(&bar[buf], bytes);
        bulk_g2s(wb, w + c0 * ccs, bytes, &bar[buf]);
      }
    } else {
      for (int k = tid; k < ncell * V * NM; k += bd) {
        const int cl = k / (V * NM), r = k - cl * (V * NM), v = r / NM, l = r - v * NM;
        cp_async8(wb + cl * WC + v * NMP + l, w + (c0 + cl) * ccs + v * cvs + l);
      }
      cp_async_commit();
    }
  };
  int j = 0;
  if (first < ngroups) issue(first, 0);
  // a thread keeps its (cell slot, face, point pairs) over the steps; its face's code byte
  // comes from global memory (1 byte per face, streamed: a DRAM-latency load), fetched one
  // step ahead so that no step waits for it
  const int u = tid;
  const int cl = u / S::UN, f = (u - cl * S::UN) / (NQ / P), t = u - cl * S::UN - f * (NQ / P), q0 = t * P;
  int qo[(P + 1) / 2];  // row offset of the thread's k-th point pair
#pragma unroll
  for (int k = 0; k < (P + 1) / 2; ++k) qo[k] = SWZ ? 2 * (t + 4 * ((k + f) & 1)) : q0 + 2 * k;
  auto load_code = [&](int64_t grp) -> int {
    const int64_t c0 = grp * cb;
    return (grp < ngroups && c0 + cl < n_owned && cl < cb) ? int(code[(c0 + cl) * NF + f]) : 0;
  };
  int fcode_next = load_code(first);
  for (int64_t grp = first; grp < ngroups; grp += step, ++j) {
    const int buf = j & 1;
    const bool more = grp + step < ngroups;
    if (more) issue(grp + step, buf ^ 1);  // buffer buf^1 was released by the last step's barrier
    const int fcode = fcode_next;
    fcode_next = load_code(grp + step);
    const int64_t c0 = grp * cb;
    const int ncell = (int)min((int64_t)cb, n_owned - c0);
    const double* wb = wb0 + buf * cb * WC;
    double acc[P][V];
    const bool act = u < ncell * S::UN;
    if (bulk_in) {
      mbar_wait(&bar[buf], (j >> 1) & 1);
    } else {
      if (more) cp_async_wait<1>();
      else cp_async_wait<0>();
      group_sync();
    }
    if (act) {
      const double* pp = ph + fcode * NM * NQ;
      const double* wc = wb + cl * WC;
#pragma unroll
      for (int p2 = 0; p2 < P; ++p2)
#pragma unroll
        for (int v = 0; v < V; ++v) acc[p2][v] = 0.0;
#pragma unroll
      for (int l = 0; l < NM; l += 2) {
        const bool two = l + 1 < NM;
        double w0[V], w1[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const double2 t = *reinterpret_cast<const double2*>(wc + v * NMP + l);
          w0[v] = t.x;
          w1[v] = t.y;
        }
        double f0[P], f1[P];
        if constexpr (P % 2 == 0) {
#pragma unroll
          for (int p2 = 0; p2 < P; p2 += 2) {
            const double2 a0 = *reinterpret_cast<const double2*>(pp + l * NQ + qo[p2 / 2]);
            f0[p2] = a0.x;
            f0[p2 + 1] = a0.y;
            if (two) {
              const double2 a1 = *reinterpret_cast<const double2*>(pp + (l + 1) * NQ + qo[p2 / 2]);
              f1[p2] = a1.x;
              f1[p2 + 1] = a1.y;
            }
          }
        } else {
#pragma unroll
          for (int p2 = 0; p2 < P; ++p2) {
            f0[p2] = pp[l * NQ + q0 + p2];
            if (two) f1[p2] = pp[(l + 1) * NQ + q0 + p2];
          }
        }
#pragma unroll
        for (int p2 = 0; p2 < P; ++p2)
#pragma unroll
          for (int v = 0; v < V; ++v) {
            acc[p2][v] = __fma_rn(w0[v], f0[p2], acc[p2][v]);
            if (two) acc[p2][v] = __fma_rn(w1[v], f1[p2], acc[p2][v]);
          }
      }
    }
    if (bulk_out && tid == 0) bulk_wait_read();  // the last step's output has left ob
    group_sync();
    if (act) {
      double* o = ob + ((cl * NF + f) * NQ + q0) * V;  // the tile's P·V outputs are contiguous
      if constexpr (SWZ) {
#pragma unroll
        for (int k = 0; k < P / 2; ++k) {  // two pieces of 2·V outputs (point pairs qo[k])
          double* ok = ob + ((cl * NF + f) * NQ + qo[k]) * V;
#pragma unroll
          for (int e = 0; e < 2 * V; e += 2)
            *reinterpret_cast<double2*>(ok + e) =
                make_double2(acc[2 * k + e / V][e % V], acc[2 * k + (e + 1) / V][(e + 1) % V]);
        }
      } else if constexpr ((P * V) % 2 == 0 && (NQ * V) % 2 == 0) {
#pragma unroll
        for (int k = 0; k < P * V; k += 2)
          *reinterpret_cast<double2*>(o + k) = make_double2(acc[k / V][k % V], acc[(k + 1) / V][(k + 1) % V]);
      } else {
#pragma unroll
        for (int k = 0; k < P * V; ++k) o[k] = acc[k / V][k % V];
      }
    }
    if (bulk_out) fence_proxy_async();  // generic-proxy writes of ob before the bulk store reads them
    group_sync();
    if (bulk_out) {
      if (tid == 0) bulk_s2g(out + c0 * OUTC, ob, uint32_t(ncell) * OUTC * 8);
    } else {
      double* dst = out + c0 * OUTC;
      for (int k = tid; k < ncell * OUTC; k += bd) dst[k] = ob[k];
    }
  }
  if (bulk_out && tid == 0) bulk_wait_all();
}

using Tr2Fn = void (*)(const double*, int64_t, int64_t, const double*, int, const uint8_t*, int, int64_t, double*,
                       int, int, int);
template <int D, int M>
static Tr2Fn tr2_fn_v(int V) {
  switch (V) {
    case 1: return k_traces2<D, M, 1>;
    case 2: return k_traces2<D, M, 2>;
    case 3: return k_traces2<D, M, 3>;
    case 4: return k_traces2<D, M, 4>;
    case 5: return k_traces2<D, M, 5>;
    case 6: return k_traces2<D, M, 6>;
    case 7: return k_traces2<D, M, 7>;
    case 8: return k_traces2<D, M, 8>;
    case 9: return k_traces2<D, M, 9>;
    default: return nullptr;
  }
}
static Tr2Fn tr2_fn(int d, int M, int V) {
  Tr2Fn f = nullptr;
  if (d == 2 && M == 1) f = tr2_fn_v<2, 1>(V);
  if (d == 2 && M == 2) f = tr2_fn_v<2, 2>(V);
  if (d == 2 && M == 3) f = tr2_fn_v<2, 3>(V);
  if (d == 3 && M == 1) f = tr2_fn_v<3, 1>(V);
  if (d == 3 && M == 2) f = tr2_fn_v<3, 2>(V);
  if (d == 3 && M == 3) f = tr2_fn_v<3, 3>(V);
  if (!f) fail(CWRECO_EUNSUPPORTED, "face traces: (d, M, nvars) not instantiated (M ≤ 3, nvars ≤ 9)");
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
#if CWR_TR_V2
  if (c->M <= 3) {
    const int d = c->d, M = c->M, V = c->V, nm = c->nm, nq = t->nq;
    const int P = nq % 4 == 0 ? 4 : nq % 3 == 0 ? 3 : nq % 2 == 0 ? 2 : 1, un = nv * nq / P;
    const int nmp = (nm + 1) & ~1, wc = V * nmp, outc = nv * nq * V;
    const int phn = (t->ncc * nm * nq + 1) & ~1;
    int dev_smem = 0, nsm = 148;
    TCK(cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
    TCK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
    const int64_t budget = int64_t(dev_smem) - 64 - int64_t(phn) * 8;  // 64: the static mbarriers
    // thread groups per CTA (see the kernel): two when each still has ≥ 2 warps of work;
    // measured (profiles/r02q_traces_variants.log): C3 0.763 vs 0.778 ms with one group,
    // C2 equal, but C5 4.88 vs 4.78 ms — ℳ = 20 stays on one group
#ifndef CWR_TR_NG
#define CWR_TR_NG (nm >= 20 ? 1 : 2)
#endif
    int ng = CWR_TR_NG;
    int cb = 0;
    for (; ng >= 1; --ng) {
      cb = std::min<int64_t>((((V > 6 ? 352 : 512) / ng) & ~31) / un,  // whole warps per group within TMAX
                             (budget - 16 * ng) / (int64_t(ng) * (2 * wc + outc) * 8));
      if (ng == 1 || cb * un >= 64) break;
    }
    if (cb < 1) fail(CWRECO_EUNSUPPORTED, "face traces: shape does not fit in shared memory");
    const int64_t groups = (c->n_owned + cb - 1) / cb;
    if (groups == 0) return;
    const int threads = ng * ((cb * un + 31) & ~31);
    const size_t smem = (size_t(phn) + size_t(ng) * ((size_t(cb) * (2 * wc + outc) + 1) & ~size_t(1))) * sizeof(double);
    // bulk copies need the dense layout (coefficients [cell][v][l] with an even ℳ) and
    // 16-byte alignment; otherwise per-element cp.async in, thread-copied out
    const int bulk_in = (cvs == nm && ccs == int64_t(V) * nm && nm % 2 == 0 && (uintptr_t(coeffs) & 15) == 0) ? 1 : 0;
    const int bulk_out = (outc % 2 == 0 && (uintptr_t(traces) & 15) == 0) ? 1 : 0;
    Tr2Fn f = tr2_fn(d, M, V);
    TCK(cudaFuncSetAttribute((const void*)f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 1;
    TCK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)f, threads, smem));
    int64_t grid = std::min<int64_t>((groups + ng - 1) / ng, (int64_t)nsm * std::max(1, occ));
    if (c->max_ctas > 0) grid = std::min<int64_t>(grid, c->max_ctas);  // CWRECO_OPT_MAX_CTAS (tests)
    f<<<(unsigned)grid, threads, smem, (cudaStream_t)stream>>>(coeffs, ccs, cvs, t->phi, t->ncc, t->code, cb,
                                                               c->n_owned, traces, bulk_in, bulk_out, ng);
    TCK(cudaGetLastError());
    return;
  }
#endif
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
