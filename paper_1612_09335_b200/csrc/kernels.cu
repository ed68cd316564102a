// sm_100a kernels of libcwreco: the CWENO reconstruction pass over the
// packed per-cell matrix stream, plus the halo pack.
//
//  k_simple     one thread per (cell, variable), plain global loads.  Reference
//               kernel and debug tap (writes the intermediates).
//  k_pipelined  persistent, warp-specialised: one producer lane streams each tile
//               (header + K-chunks of B⁺) into a ring of shared-memory stages with
//               1-D TMA bulk copies (cp.async.bulk + mbarrier complete_tx); the
//               consumer warps (one thread per (cell, variable)) gather Q_j through
//               L1/L2, accumulate B⁺ΔQ in registers, run the fused
//               sector / P0 / σ / ω / blend epilogue, stage the tile's output in
//               shared memory and write it back with one bulk store.
// Both compute exactly the same arithmetic in the same order.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "internal.hpp"

namespace cwr {

struct DeviceState {
  unsigned char* blocks = nullptr;
  int64_t blocks_bytes = 0;
  double* sigma = nullptr;  // packed upper triangle of Σ[1:,1:], doubled off-diagonals
  int64_t* send = nullptr;
  int64_t n_send = 0;
  int num_sms = 148;
  int max_smem = 227 * 1024;
  double* dbg = nullptr;
  int64_t dbg_bytes = 0;
  int64_t* dbg_cells = nullptr;
  int64_t dbg_ncells = 0;
};

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) fail(CWRECO_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct KArgs {
  const unsigned char* blocks;
  int64_t tile_bytes, off_ids, off_sinv, off_slots, off_chunks;
  int T, G, K, KC, NCH, V;
  int64_t n_owned, tile_begin, tile_end;
  const double* Q;
  int64_t acs, avs;
  double* out;
  int64_t ccs, cvs;
  int dense_out;
  const double* sig;  // packed Σ' (global)
  double lam0, lams, eps, psi1;
  int r;
};

struct DbgOut {
  double *popt, *psec, *sigma, *omega, *w;
  const int64_t* cells;
  int64_t n;
};

__host__ __device__ constexpr int nmodes(int M, int d) {
  return d == 2 ? (M + 1) * (M + 2) / 2 : (M + 1) * (M + 2) * (M + 3) / 6;
}

__device__ __forceinline__ double powr(double t, int r) {
  if (r == 4) {
    double t2 = t * t;
    return t2 * t2;
  }
  double p = 1.0;
  for (int i = 0; i < r; ++i) p *= t;
  return p;
}

// The fused epilogue: P0, σ, ω, blend.  acc[l-1] = p̂_opt[l], l >= 1;
// ps[s][l-1] = p̂_s[l], l = 1..D; valid[s].  Σ' is the packed upper triangle of
// Σ[1:,1:] with doubled off-diagonal entries (Σ is symmetric, row/col 0 zero).
template <int D, int NM>
__device__ __forceinline__ void cweno_epilogue(double qi, double* acc, const double (&ps)[D + 1][D],
                                               const bool (&valid)[D + 1], const KArgs& a,
                                               const double* __restrict__ sig, double* w,
                                               double* sigma_out, double* omega_out) {
  constexpr int R = NM - 1;
  const double p0 = qi / a.psi1;
  int nval = 0;
#pragma unroll
  for (int s = 0; s <= D; ++s) nval += valid[s] ? 1 : 0;
  const double denom = a.lam0 + nval * a.lams;
  const double l0 = a.lam0 / denom, ls = a.lams / denom;
  // P0 = (P_opt − Σ λ̄_s P_s)/λ̄0, in place in acc
#pragma unroll
  for (int l = 0; l < D; ++l) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q <= D; ++q) s += valid[q] ? ps[q][l] : 0.0;
    acc[l] = (acc[l] - ls * s) / l0;
  }
#pragma unroll
  for (int l = D; l < R; ++l) acc[l] = acc[l] / l0;
  // σ0 = P0ᵀ Σ P0
  double sg0 = 0.0;
  {
    int idx = 0;
#pragma unroll
    for (int l = 0; l < R; ++l) {
      double t = 0.0;
#pragma unroll
      for (int m = l; m < R; ++m) t += sig[idx + m - l] * acc[m];
      idx += R - l;
      sg0 += acc[l] * t;
    }
  }
  double sgs[D + 1];
#pragma unroll
  for (int s = 0; s <= D; ++s) {
    double v = 0.0;
    int idx = 0;
#pragma unroll
    for (int l = 0; l < D; ++l) {
      double t = 0.0;
#pragma unroll
      for (int m = l; m < D; ++m) t += sig[idx + m - l] * ps[s][m];
      idx += R - l;
      v += ps[s][l] * t;
    }
    sgs[s] = v;
  }
  // nonlinear weights
  double wt0 = l0 / powr(sg0 + a.eps, a.r);
  double wts[D + 1];
  double sum = wt0;
#pragma unroll
  for (int s = 0; s <= D; ++s) {
    wts[s] = valid[s] ? ls / powr(sgs[s] + a.eps, a.r) : 0.0;
    sum += wts[s];
  }
  const double om0 = wt0 / sum;
  double oms[D + 1];
#pragma unroll
  for (int s = 0; s <= D; ++s) oms[s] = wts[s] / sum;
  // blend; w[0] := Q_i/ψ1 (R17)
  w[0] = p0;
#pragma unroll
  for (int l = 0; l < D; ++l) {
    double v = om0 * acc[l];
#pragma unroll
    for (int s = 0; s <= D; ++s) v += oms[s] * ps[s][l];
    w[l + 1] = v;
  }
#pragma unroll
  for (int l = D; l < R; ++l) w[l + 1] = om0 * acc[l];
  if (sigma_out) {
    sigma_out[0] = sg0;
    omega_out[0] = om0;
#pragma unroll
    for (int s = 0; s <= D; ++s) {
      sigma_out[s + 1] = valid[s] ? sgs[s] : 0.0;
      omega_out[s + 1] = oms[s];
    }
  }
}

// ---------------------------------------------------------------- simple kernel
template <int D, int M, bool DEBUG>
__global__ void __launch_bounds__(256) k_simple(KArgs a, DbgOut dbg) {
  constexpr int NM = nmodes(M, D), R = NM - 1, NV = D + 1;
  const int64_t gid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t item = gid / a.V;
  const int v = int(gid % a.V);
  int64_t c;
  if (DEBUG) {
    if (item >= dbg.n) return;
    c = dbg.cells[item];
  } else {
    c = a.tile_begin * a.T + item;
    if (c >= a.n_owned || c >= a.tile_end * a.T) return;
  }
  const int64_t tile = c / a.T;
  const int ct = int(c % a.T);
  const unsigned char* tb = a.blocks + tile * a.tile_bytes;
  const int32_t* ids = (const int32_t*)(tb + a.off_ids);
  const double* sinv = (const double*)(tb + a.off_sinv) + size_t(ct) * NV * D * D;
  const uint8_t* slots = (const uint8_t*)(tb + a.off_slots) + size_t(ct) * NV * D;
  const double* B = (const double*)(tb + a.off_chunks);
  const double* Qv = a.Q + v * a.avs;
  const double qi = Qv[c * a.acs];

  double acc[R];
#pragma unroll
  for (int l = 0; l < R; ++l) acc[l] = 0.0;
  for (int k = 0; k < a.K; ++k) {
    const int32_t j = ids[size_t(k) * a.T + ct];
    const double dq = Qv[int64_t(j) * a.acs] - qi;
    const double* b = B + (size_t(k) * a.T + ct) * R;
#pragma unroll
    for (int l = 0; l < R; ++l) acc[l] += b[l] * dq;
  }
  double ps[NV][D];
  bool valid[NV];
#pragma unroll
  for (int s = 0; s < NV; ++s) {
    valid[s] = slots[s * D] != 255;
    double dq[D];
#pragma unroll
    for (int m = 0; m < D; ++m) {
      const int g = valid[s] ? slots[s * D + m] : 0;
      const int32_t j = ids[size_t(g) * a.T + ct];
      dq[m] = valid[s] ? Qv[int64_t(j) * a.acs] - qi : 0.0;
    }
#pragma unroll
    for (int l = 0; l < D; ++l) {
      double t = 0.0;
#pragma unroll
      for (int m = 0; m < D; ++m) t += sinv[(s * D + l) * D + m] * dq[m];
      ps[s][l] = t;
    }
  }
  if (DEBUG) {
    double* po = dbg.popt + (item * a.V + v) * NM;
    po[0] = qi / a.psi1;
    for (int l = 0; l < R; ++l) po[l + 1] = acc[l];
    for (int s = 0; s < NV; ++s) {
      double* pp = dbg.psec + ((item * NV + s) * a.V + v) * NV;
      pp[0] = valid[s] ? qi / a.psi1 : 0.0;
      for (int l = 0; l < D; ++l) pp[l + 1] = ps[s][l];
    }
  }
  double w[NM];
  double sg[NV + 1], om[NV + 1];
  cweno_epilogue<D, NM>(qi, acc, ps, valid, a, a.sig, w, DEBUG ? sg : nullptr, DEBUG ? om : nullptr);
  if (DEBUG) {
    for (int s = 0; s <= NV; ++s) {
      dbg.sigma[(item * (NV + 1) + s) * a.V + v] = sg[s];
      dbg.omega[(item * (NV + 1) + s) * a.V + v] = om[s];
    }
    double* wo = dbg.w + (item * a.V + v) * NM;
    for (int l = 0; l < NM; ++l) wo[l] = w[l];
  } else {
    double* o = a.out + c * a.ccs + v * a.cvs;
#pragma unroll
    for (int l = 0; l < NM; ++l) o[l] = w[l];
  }
}

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

constexpr int KCMAX = 8;

struct PipeCfg {
  int stages;
  int64_t stage_bytes, hdr_bytes, out_bytes, sig_bytes;
  int64_t off_hdr, off_stage, off_out, off_sig, off_bar, smem;
  int ncw;  // consumer warps
};

// ---------------------------------------------------------------- pipelined kernel
template <int D, int M>
__global__ void __launch_bounds__(11 * 32, 1) k_pipelined(KArgs a, PipeCfg pc) {
  constexpr int NM = nmodes(M, D), R = NM - 1, NV = D + 1;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* hdr = smem + pc.off_hdr;
  unsigned char* stg = smem + pc.off_stage;
  double* outs = (double*)(smem + pc.off_out);
  double* sig = (double*)(smem + pc.off_sig);
  uint64_t* bars = (uint64_t*)(smem + pc.off_bar);
  uint64_t* hdr_full = bars;            // [2]
  uint64_t* hdr_empty = bars + 2;       // [2]
  uint64_t* ch_full = bars + 4;         // [S]
  uint64_t* ch_empty = bars + 4 + pc.stages;  // [S]
  const int S = pc.stages;
  const int ncons = pc.ncw * 32;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&hdr_full[b], 1);
      mbar_init(&hdr_empty[b], pc.ncw);
    }
    for (int s = 0; s < S; ++s) {
      mbar_init(&ch_full[s], 1);
      mbar_init(&ch_empty[s], pc.ncw);
    }
    fence_barrier_init();
  }
  // Σ' into shared memory
  const int nsig = R * (R + 1) / 2;
  for (int i = tid; i < nsig; i += blockDim.x) sig[i] = a.sig[i];
  __syncthreads();

  if (warp == pc.ncw) {
    // ------------------------------------------------ producer warp
    if (lane == 0) {
      uint32_t gc = 0;
      int it = 0;
      for (int64_t tile = a.tile_begin + blockIdx.x; tile < a.tile_end; tile += gridDim.x, ++it) {
        const unsigned char* tb = a.blocks + tile * a.tile_bytes;
        const int hb = it & 1;
        mbar_wait(&hdr_empty[hb], ((it >> 1) & 1) ^ 1);
        mbar_expect_tx(&hdr_full[hb], (uint32_t)pc.hdr_bytes);
        bulk_g2s(hdr + hb * pc.hdr_bytes, tb, (uint32_t)pc.hdr_bytes, &hdr_full[hb]);
        for (int ch = 0; ch < a.NCH; ++ch, ++gc) {
          const int st = gc % S;
          const int kc = min(a.KC, a.K - ch * a.KC);
          const uint32_t bytes = (uint32_t)(kc * (int64_t)a.T * R * 8);
          mbar_wait(&ch_empty[st], ((gc / S) & 1) ^ 1);
          mbar_expect_tx(&ch_full[st], bytes);
          bulk_g2s(stg + st * pc.stage_bytes, tb + a.off_chunks + (int64_t)ch * a.KC * a.T * R * 8, bytes,
                   &ch_full[st]);
        }
      }
    }
    return;
  }

  // -------------------------------------------------- consumer warps
  const bool active = tid < a.T * a.V;
  const int ct = active ? tid / a.V : 0;
  const int v = active ? tid % a.V : 0;
  const double* Qv = a.Q + v * a.avs;
  uint32_t gc = 0;
  int it = 0;
  for (int64_t tile = a.tile_begin + blockIdx.x; tile < a.tile_end; tile += gridDim.x, ++it) {
    const int hb = it & 1;
    const int64_t c = tile * a.T + ct;
    const bool live = active && c < a.n_owned;
    const double qi = live ? Qv[c * a.acs] : 0.0;
    mbar_wait(&hdr_full[hb], (it >> 1) & 1);
    const unsigned char* hb_p = hdr + hb * pc.hdr_bytes;
    const int32_t* ids = (const int32_t*)(hb_p + a.off_ids);

    double acc[R];
#pragma unroll
    for (int l = 0; l < R; ++l) acc[l] = 0.0;
    for (int ch = 0; ch < a.NCH; ++ch, ++gc) {
      const int st = gc % S;
      const int kc = min(a.KC, a.K - ch * a.KC);
      // gather this chunk's ΔQ first (KC loads in flight), then wait for B
      double dq[KCMAX];
#pragma unroll
      for (int kk = 0; kk < KCMAX; ++kk) {
        dq[kk] = 0.0;
        if (kk < kc && live) {
          const int32_t j = ids[(size_t)(ch * a.KC + kk) * a.T + ct];
          dq[kk] = __ldg(Qv + int64_t(j) * a.acs) - qi;
        }
      }
      mbar_wait(&ch_full[st], (gc / S) & 1);
      const double* Bs = (const double*)(stg + st * pc.stage_bytes);
#pragma unroll
      for (int kk = 0; kk < KCMAX; ++kk) {
        if (kk < kc) {
          const double* b = Bs + ((size_t)kk * a.T + ct) * R;
#pragma unroll
          for (int l = 0; l < R; ++l) acc[l] += b[l] * dq[kk];
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&ch_empty[st]);
    }

    // sectors
    const double* sinv = (const double*)(hb_p + a.off_sinv) + size_t(ct) * NV * D * D;
    const uint8_t* slots = (const uint8_t*)(hb_p + a.off_slots) + size_t(ct) * NV * D;
    double ps[NV][D];
    bool valid[NV];
#pragma unroll
    for (int s = 0; s < NV; ++s) {
      valid[s] = slots[s * D] != 255;
      double dqs[D];
#pragma unroll
      for (int m = 0; m < D; ++m) {
        const int g = valid[s] ? slots[s * D + m] : 0;
        const int32_t j = ids[size_t(g) * a.T + ct];
        dqs[m] = (valid[s] && live) ? __ldg(Qv + int64_t(j) * a.acs) - qi : 0.0;
      }
#pragma unroll
      for (int l = 0; l < D; ++l) {
        double t = 0.0;
#pragma unroll
        for (int m = 0; m < D; ++m) t += sinv[(s * D + l) * D + m] * dqs[m];
        ps[s][l] = t;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&hdr_empty[hb]);

    double w[NM];
    cweno_epilogue<D, NM>(qi, acc, ps, valid, a, sig, w, nullptr, nullptr);

    if (a.dense_out) {
      if (tid == 0) bulk_wait_read();  // previous tile's store has read outs
      named_bar(1, ncons);
      if (live) {
        double* o = outs + (size_t)(ct * a.V + v) * NM;
#pragma unroll
        for (int l = 0; l < NM; ++l) o[l] = w[l];
      }
      fence_proxy_async();
      named_bar(1, ncons);
      if (tid == 0) {
        const int64_t c0 = tile * a.T;
        const int64_t ncell = min((int64_t)a.T, a.n_owned - c0);
        bulk_s2g(a.out + c0 * a.ccs, outs, (uint32_t)(ncell * a.V * NM * 8));
      }
    } else if (live) {
      double* o = a.out + c * a.ccs + v * a.cvs;
#pragma unroll
      for (int l = 0; l < NM; ++l) o[l] = w[l];
    }
  }
  if (tid == 0) bulk_wait_all();
}

// ---------------------------------------------------------------- halo pack
__global__ void k_halo_pack(const double* __restrict__ Q, int64_t acs, int64_t avs, int V,
                            const int64_t* __restrict__ send, int64_t n, double* __restrict__ buf) {
  const int64_t gid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gid >= n * V) return;
  const int64_t k = gid / V;
  const int v = int(gid % V);
  buf[gid] = Q[send[k] * acs + v * avs];
}

// ---------------------------------------------------------------- dispatch
template <bool DEBUG>
void launch_simple(int d, int M, dim3 g, dim3 b, cudaStream_t st, const KArgs& a, const DbgOut& o) {
#define CASE(DD, MM) \
  if (d == DD && M == MM) { k_simple<DD, MM, DEBUG><<<g, b, 0, st>>>(a, o); return; }
  CASE(2, 1) CASE(2, 2) CASE(2, 3) CASE(2, 4) CASE(3, 1) CASE(3, 2) CASE(3, 3)
#undef CASE
  fail(CWRECO_EUNSUPPORTED, "unsupported (d, M)");
}

using PipeFn = void (*)(KArgs, PipeCfg);
PipeFn pipe_fn(int d, int M) {
#define CASE(DD, MM) \
  if (d == DD && M == MM) return k_pipelined<DD, MM>;
  CASE(2, 1) CASE(2, 2) CASE(2, 3) CASE(2, 4) CASE(3, 1) CASE(3, 2) CASE(3, 3)
#undef CASE
  fail(CWRECO_EUNSUPPORTED, "unsupported (d, M)");
}

static KArgs make_args(const cwreco_ctx* c, const double* avgs, int64_t acs, int64_t avs, double* out,
                       int64_t ccs, int64_t cvs) {
  const Layout& L = c->lay;
  KArgs a;
  a.blocks = c->dev->blocks;
  a.tile_bytes = L.tile_bytes;
  a.off_ids = L.off_ids;
  a.off_sinv = L.off_sinv;
  a.off_slots = L.off_slots;
  a.off_chunks = L.off_chunks;
  a.T = L.T;
  a.G = L.G;
  a.K = L.K;
  a.KC = L.KC;
  a.NCH = L.NCH;
  a.V = c->V;
  a.n_owned = c->n_owned;
  a.tile_begin = 0;
  a.tile_end = c->n_tiles;
  a.Q = avgs;
  a.acs = acs;
  a.avs = avs;
  a.out = out;
  a.ccs = ccs;
  a.cvs = cvs;
  a.dense_out = 0;
  a.sig = c->dev->sigma;
  a.lam0 = c->prm.lambda0;
  a.lams = c->prm.lambda_s;
  a.eps = c->prm.eps;
  a.psi1 = c->psi1;
  a.r = c->prm.r;
  return a;
}

static PipeCfg pipe_cfg(const cwreco_ctx* c) {
  const Layout& L = c->lay;
  PipeCfg p;
  p.ncw = (L.T * c->V + 31) / 32;
  p.hdr_bytes = L.header_bytes;
  p.stage_bytes = (int64_t)L.KC * L.kslice_bytes;
  p.out_bytes = ((int64_t)L.T * c->V * c->nm * 8 + 127) & ~int64_t(127);
  p.sig_bytes = ((int64_t)(c->nm - 1) * c->nm / 2 * 8 + 127) & ~int64_t(127);
  auto r128 = [](int64_t x) { return (x + 127) & ~int64_t(127); };
  int best = 2;
  for (int s = 6; s >= 2; --s) {
    int64_t tot = r128(2 * p.hdr_bytes) + r128(s * p.stage_bytes) + p.out_bytes + p.sig_bytes + 256;
    if (tot <= c->dev->max_smem) { best = s; break; }
  }
  p.stages = best;
  p.off_hdr = 0;
  p.off_stage = r128(2 * p.hdr_bytes);
  p.off_out = p.off_stage + r128(best * p.stage_bytes);
  p.off_sig = p.off_out + p.out_bytes;
  p.off_bar = p.off_sig + p.sig_bytes;
  p.smem = p.off_bar + 8 * (4 + 2 * best);
  return p;
}

void dev_create(cwreco_ctx* c) {
  if (c->device < 0) return;
  c->dev = new DeviceState();
  CK(cudaSetDevice(c->device));
  CK(cudaDeviceGetAttribute(&c->dev->num_sms, cudaDevAttrMultiProcessorCount, c->device));
  CK(cudaDeviceGetAttribute(&c->dev->max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
}

void dev_destroy(cwreco_ctx* c) {
  if (!c->dev) return;
  cudaSetDevice(c->device);
  cudaFree(c->dev->blocks);
  cudaFree(c->dev->sigma);
  cudaFree(c->dev->send);
  cudaFree(c->dev->dbg);
  cudaFree(c->dev->dbg_cells);
  delete c->dev;
  c->dev = nullptr;
}

void dev_alloc_blocks(cwreco_ctx* c, int64_t bytes) {
  CK(cudaSetDevice(c->device));
  if (c->dev->blocks) CK(cudaFree(c->dev->blocks));
  c->dev->blocks = nullptr;
  c->dev->blocks_bytes = 0;
  cudaError_t e = cudaMalloc(&c->dev->blocks, (size_t)bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(CWRECO_ENOMEM, "cudaMalloc of " + std::to_string(bytes) + " bytes of matrix blocks failed");
  }
  c->dev->blocks_bytes = bytes;
}

void dev_upload_blocks(cwreco_ctx* c, int64_t offset, const unsigned char* host, int64_t bytes) {
  CK(cudaMemcpy(c->dev->blocks + offset, host, (size_t)bytes, cudaMemcpyHostToDevice));
}

void dev_upload_aux(cwreco_ctx* c) {
  const int nm = c->nm, R = nm - 1;
  std::vector<double> packed;
  for (int l = 1; l < nm; ++l)
    for (int m = l; m < nm; ++m) packed.push_back((l == m ? 1.0 : 2.0) * c->sigma[l * nm + m]);
  if (c->dev->sigma) CK(cudaFree(c->dev->sigma));
  CK(cudaMalloc(&c->dev->sigma, sizeof(double) * (packed.size() + 1)));
  CK(cudaMemcpy(c->dev->sigma, packed.data(), sizeof(double) * packed.size(), cudaMemcpyHostToDevice));
  (void)R;
  PipeCfg p = pipe_cfg(c);
  PipeFn f = pipe_fn(c->d, c->M);
  CK(cudaFuncSetAttribute((const void*)f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
}

void dev_download_tile(const cwreco_ctx* c, int64_t tile, unsigned char* host) {
  CK(cudaSetDevice(c->device));
  CK(cudaMemcpy(host, c->dev->blocks + tile * c->lay.tile_bytes, (size_t)c->lay.tile_bytes, cudaMemcpyDeviceToHost));
}

int64_t dev_bytes(const cwreco_ctx* c) {
  if (!c->dev) return 0;
  return c->dev->blocks_bytes + c->dev->dbg_bytes + c->dev->n_send * 8;
}

void dev_reconstruct(cwreco_ctx* c, const double* avgs, int64_t acs, int64_t avs, double* coeffs, int64_t ccs,
                     int64_t cvs, int part, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  KArgs a = make_args(c, avgs, acs, avs, coeffs, ccs, cvs);
  if (part == CWRECO_PART_INTERIOR) {
    a.tile_end = c->n_int_tiles;
  } else if (part == CWRECO_PART_BOUNDARY) {
    a.tile_begin = c->n_int_tiles;
  }
  if (a.tile_end <= a.tile_begin) return;
  const int nm = c->nm;
  if (c->kernel == CWRECO_KERNEL_SIMPLE) {
    const int64_t cells = std::min(a.tile_end * a.T, c->n_owned) - a.tile_begin * a.T;
    const int64_t threads = cells * c->V;
    dim3 b(256), g((unsigned)((threads + 255) / 256));
    DbgOut o{};
    launch_simple<false>(c->d, c->M, g, b, st, a, o);
  } else {
    a.dense_out = (cvs == nm && ccs == (int64_t)c->V * nm && (((uintptr_t)coeffs) & 15) == 0 &&
                   ((int64_t)c->V * nm) % 2 == 0)
                      ? 1
                      : 0;
    PipeCfg p = pipe_cfg(c);
    const int64_t ntiles = a.tile_end - a.tile_begin;
    const int per_sm = std::max<int>(1, int(c->dev->max_smem / std::max<int64_t>(p.smem, 1)));
    const int64_t grid = std::min<int64_t>(ntiles, (int64_t)c->dev->num_sms * std::min(per_sm, 2));
    dim3 b((p.ncw + 1) * 32), g((unsigned)grid);
    pipe_fn(c->d, c->M)<<<g, b, p.smem, st>>>(a, p);
  }
  CK(cudaGetLastError());
}

void dev_debug(cwreco_ctx* c, const double* avgs, int64_t acs, int64_t avs, int64_t n_sel, const int64_t* cells,
               double* popt, double* psec, double* sigma, double* omega, double* w, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int V = c->V, nm = c->nm, NV = c->d + 1;
  const int64_t n_popt = n_sel * V * nm, n_psec = n_sel * NV * V * NV, n_sig = n_sel * (NV + 1) * V;
  const int64_t total = n_popt + n_psec + 2 * n_sig + n_popt;
  const int64_t bytes = total * 8;
  if (bytes > c->dev->dbg_bytes) {
    cudaFree(c->dev->dbg);
    CK(cudaMalloc(&c->dev->dbg, bytes));
    c->dev->dbg_bytes = bytes;
  }
  if (n_sel > c->dev->dbg_ncells) {
    cudaFree(c->dev->dbg_cells);
    CK(cudaMalloc(&c->dev->dbg_cells, n_sel * 8));
    c->dev->dbg_ncells = n_sel;
  }
  CK(cudaMemcpyAsync(c->dev->dbg_cells, cells, n_sel * 8, cudaMemcpyHostToDevice, st));
  DbgOut o;
  o.popt = c->dev->dbg;
  o.psec = o.popt + n_popt;
  o.sigma = o.psec + n_psec;
  o.omega = o.sigma + n_sig;
  o.w = o.omega + n_sig;
  o.cells = c->dev->dbg_cells;
  o.n = n_sel;
  KArgs a = make_args(c, avgs, acs, avs, nullptr, 0, 0);
  const int64_t threads = n_sel * V;
  dim3 b(256), g((unsigned)((threads + 255) / 256));
  launch_simple<true>(c->d, c->M, g, b, st, a, o);
  CK(cudaGetLastError());
  std::vector<double> h(total);
  CK(cudaMemcpyAsync(h.data(), c->dev->dbg, bytes, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const double* p = h.data();
  if (popt) std::memcpy(popt, p, n_popt * 8);
  p += n_popt;
  if (psec) std::memcpy(psec, p, n_psec * 8);
  p += n_psec;
  if (sigma) std::memcpy(sigma, p, n_sig * 8);
  p += n_sig;
  if (omega) std::memcpy(omega, p, n_sig * 8);
  p += n_sig;
  if (w) std::memcpy(w, p, n_popt * 8);
}

void dev_set_send(cwreco_ctx* c) {
  if (!c->dev) return;
  CK(cudaSetDevice(c->device));
  cudaFree(c->dev->send);
  c->dev->send = nullptr;
  c->dev->n_send = (int64_t)c->send_local.size();
  if (c->dev->n_send == 0) return;
  CK(cudaMalloc(&c->dev->send, c->dev->n_send * 8));
  CK(cudaMemcpy(c->dev->send, c->send_local.data(), c->dev->n_send * 8, cudaMemcpyHostToDevice));
}

void dev_halo_pack(cwreco_ctx* c, const double* avgs, int64_t acs, int64_t avs, double* sendbuf, void* stream) {
  const int64_t n = c->dev->n_send;
  if (n == 0) return;
  const int64_t threads = n * c->V;
  k_halo_pack<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(avgs, acs, avs, c->V, c->dev->send,
                                                                                     n, sendbuf);
  CK(cudaGetLastError());
}

}  // namespace cwr
