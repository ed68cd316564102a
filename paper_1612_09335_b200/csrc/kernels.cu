// sm_100a kernels of libcwreco: the CWENO reconstruction pass over the
// packed per-cell matrix stream, plus the halo pack.
//
//  k_simple     one thread per (cell, variable), plain global loads.  Reference
//               kernel and debug tap (writes the intermediates).
//  k_pipelined  persistent and warp-specialised.  One producer lane streams each
//               tile (header + K-chunks of B⁺) into a ring of shared-memory stages
//               with 1-D TMA bulk copies (cp.async.bulk, mbarrier complete_tx);
//               two gather warps copy the stencil averages Q_j of each chunk into
//               the same stage with cp.async; the consumer warps (one thread per
//               (cell, variable)) accumulate B⁺ΔQ in registers, run the fused
//               sector / P0 / σ / ω / blend epilogue (Σ from the constant bank) and
//               write their outputs back with per-warp bulk stores.
// Both kernels perform the same floating-point operations in the same order, so
// their outputs are bitwise identical (tested).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "kcommon.cuh"

namespace cwr {

struct DeviceState {
  unsigned char* blocks = nullptr;
  int64_t blocks_bytes = 0;
  int64_t* send = nullptr;
  int64_t n_send = 0;
  int num_sms = 148;
  int max_smem = 227 * 1024;
  double* dbg = nullptr;
  int64_t dbg_bytes = 0;
  int64_t* dbg_cells = nullptr;
  int64_t dbg_ncells = 0;
  int64_t* bc_src = nullptr;  // boundary ghosts (R37): local id of the source cell
  int32_t* bc_neg = nullptr;  //   variable negated (wall side), −1 none
  double* Qbc = nullptr;      //   their averages [n_bc][V], filled before every pass
  int64_t n_bc = 0;
  double* h_avgs = nullptr;  // device buffers of cwreco_reconstruct_host (lazy)
  double* h_coeffs = nullptr;
  int64_t h_avgs_n = 0, h_coeffs_n = 0;
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t> piece_done;
  bool have_cfg = false;  // launch shape of the pipelined kernel, fixed at precompute
  PipeCfg cfg{};
  int cfg_ctas = 1;
};

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) fail(CWRECO_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ---------------------------------------------------------------- simple kernel
template <int D, int M, bool DEBUG>
__global__ void __launch_bounds__(256) k_simple(KArgs a, DbgOut dbg) {
  constexpr int NM = nmodes(M, D), R = NM - 1, NV = D + 1, NCAP = NV * D;
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
  const double* sinv = (const double*)(tb + sector_sinv_off(a.off_sector, a.sector_bytes, a.TSC, a.srec, ct));
  const uint8_t vmask = *(tb + sector_mask_off(a.off_sector, a.sector_bytes, a.sinv_bytes, a.TSC, ct));
  const double* Qv = a.Q + v * a.avs;
  const double qi = Qv[c * a.acs];

  double acc[R];
#pragma unroll
  for (int l = 0; l < R; ++l) acc[l] = 0.0;
  double dqs[NCAP];
  for (int ch = 0; ch < a.NCH; ++ch) {
    const int kc = min(a.KC, a.G - ch * a.KC);
    const unsigned char* cb = tb + a.u_bytes + ch * a.chunk_bytes;
    const uint16_t* idx = (const uint16_t*)(tb + a.off_idx);  // idx_elem layout
    const double* Bc = (const double*)(cb + a.ids_bytes);   // chunk_elem layout
    for (int kk = 0; kk < kc; ++kk) {
      const int p = ch * a.KC + kk;
      const int32_t j = ((const int32_t*)tb)[idx[idx_elem(a.kind, a.T, p, ct)] / a.VP];  // union chunk
      const double qj = *qptr(a, j, v);
      const double dq = qj - qi;
#pragma unroll
      for (int q = 0; q < NCAP; ++q)
        if (p == q) dqs[q] = dq;
      // ROWBLK family: B⁺Q accumulated on the raw averages, B⁺ΔQ = B⁺Q − rs·Q_i after
      // the loop (row sums rs from the sector record; k_rowblk's arithmetic)
      const double x = a.kind == KIND_ROWBLK ? qj : dq;
#pragma unroll
      for (int l = 0; l < R; ++l) acc[l] = __fma_rn(Bc[chunk_elem(a.kind, kc, R, a.V, a.T, l, ct, kk)], x, acc[l]);
    }
  }
  if (a.kind == KIND_ROWBLK) {
#pragma unroll
    for (int l = 0; l < R; ++l) acc[l] = __fma_rn(-sinv[NV * D * D + l], qi, acc[l]);
  }
  bool valid[NV];
#pragma unroll
  for (int s = 0; s < NV; ++s) valid[s] = (vmask >> s) & 1;
  double ps[NV][D];
  sector_apply<D>(sinv, dqs, ps);
  if (DEBUG) {
    double* po = dbg.popt + (item * a.V + v) * NM;
    po[0] = qi / a.psi1;
    for (int l = 0; l < R; ++l) po[l + 1] = acc[l];
    for (int s = 0; s < NV; ++s) {
      double* pp = dbg.psec + ((item * NV + s) * a.V + v) * NV;
      pp[0] = valid[s] ? qi / a.psi1 : 0.0;
      for (int l = 0; l < D; ++l) pp[l + 1] = valid[s] ? ps[s][l] : 0.0;
    }
  }
  double sg[NV + 1], om[NV + 1];
  double* wout = DEBUG ? dbg.w + (item * a.V + v) * NM : a.out + c * a.ccs + v * a.cvs;
  cweno_epilogue<D, NM>(qi, acc, ps, valid, a, wout, DEBUG ? sg : nullptr, DEBUG ? om : nullptr);
  if (DEBUG) {
    for (int s = 0; s <= NV; ++s) {
      dbg.sigma[(item * (NV + 1) + s) * a.V + v] = sg[s];
      dbg.omega[(item * (NV + 1) + s) * a.V + v] = om[s];
    }
  }
}

// (must agree with cons_threads / ctas_per_sm in internal.hpp)
__host__ __device__ constexpr int cons_target(int D, int M) { return nmodes(M, D) >= 20 ? 320 : 160; }
__host__ __device__ constexpr int min_blocks(int D, int M) { return nmodes(M, D) >= 20 ? 1 : 2; }
// consumers + one producer warp
__host__ __device__ constexpr int max_threads(int D, int M) { return cons_target(D, M) + 32; }
// ---------------------------------------------------------------- pipelined kernel
// Persistent, warp-specialised.  Warp roles: [0, ncw) consumers, thread
// tid ↔ (ct, v) = (tid / V, tid % V); warp ncw: TMA producer (lane 0) — streams,
// per tile t, the union chunk of the CTA's NEXT tile, then t's position chunks
// (union indices + B⁺ columns) and sector chunk (sector inverses + validity) into
// a ring of S shared-memory stages with 1-D bulk copies completing on mbarrier
// transaction counts.
// Stencil averages are gathered once per tile: at the start of tile t the
// consumers read the next tile's union chunk and cp.async-copy the V averages of
// every cell of that union into the other half of a double-buffered Q_u; a
// whole tile of work hides the gather.  Per position the consumers then read
// Q_u[idx][v] from shared memory.  Gather positions [0, (D+1)·D) are the sector
// cells (precompute.cpp), so their ΔQ is captured from the first chunks.
template <int D, int M, int KC>
__global__ void __launch_bounds__(max_threads(D, M), min_blocks(D, M)) k_pipelined(KArgs a, PipeCfg pc) {
  constexpr int NM = nmodes(M, D), R = NM - 1, NV = D + 1;
  constexpr int NCAP = NV * D, NCAPCH = (NCAP + KC - 1) / KC;  // captured positions / chunks
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* stg = smem + pc.off_stage;
  double* outs = (double*)(smem + pc.off_out);
  double* Qu = (double*)(smem + pc.off_q);  // [2][Umax][V]
  uint16_t* Ix = (uint16_t*)(smem + pc.off_q + ((2 * (int64_t)a.Umax * a.V * 8 + 127) & ~int64_t(127)));  // [2][G][T]
  uint64_t* bars = (uint64_t*)(smem + pc.off_bar);
  const int S = pc.stages;
  uint64_t* full = bars;       // [S]
  uint64_t* empty = bars + S;  // [S]
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int TV = a.T * a.V;
  const int64_t t0 = a.tile_begin + blockIdx.x;  // this CTA's tiles: t0, t0 + grid, …

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], pc.ncw);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == pc.ncw) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      Ring rg;
      auto issue = [&](const unsigned char* src, uint32_t bytes) {
        mbar_wait_sleep(&empty[rg.st], rg.ph ^ 1);
        mbar_expect_tx(&full[rg.st], bytes);
        bulk_g2s(stg + rg.st * pc.stage_bytes, src, bytes, &full[rg.st]);
        rg.next(S);
      };
      if (t0 < a.tile_end) issue(a.blocks + t0 * a.tile_bytes, (uint32_t)a.u_bytes);
      for (int64_t tile = t0; tile < a.tile_end; tile += gridDim.x) {
        const unsigned char* tb = a.blocks + tile * a.tile_bytes;
        if (tile + gridDim.x < a.tile_end) issue(tb + gridDim.x * a.tile_bytes, (uint32_t)a.u_bytes);
        for (int ch = 0; ch < a.NCH; ++ch)
          issue(tb + a.u_bytes + ch * a.chunk_bytes, (uint32_t)(min(KC, a.G - ch * KC) * a.kslice_bytes));
        issue(tb + a.off_sector, (uint32_t)a.sector_bytes);
      }
    }
    return;
  }

  // -------------------------------------------------- consumer warps
  const int nct = pc.ncw * 32;  // consumer threads
  const bool active = tid < TV;
  const int ct = active ? tid / a.V : 0;
  const int v = active ? tid % a.V : 0;
  double* outw = outs + (size_t)warp * 32 * NM;  // output staging
  Ring rg;
  // gather the union of tile `tile` (its union chunk is the current stage) into
  // Q_u[buf] and copy its position → union-offset table into Ix[buf]
  auto gather_union = [&](int64_t tile, int buf) {
    mbar_wait(&full[rg.st], rg.ph);
    const unsigned char* ub = stg + rg.st * pc.stage_bytes;
    const int32_t* uid = (const int32_t*)ub;
    {
      const uint4* src = (const uint4*)(ub + a.off_idx);
      uint4* dsti = (uint4*)((unsigned char*)Ix + buf * a.idx_bytes);
      for (int i = tid; i < (int)(a.idx_bytes / 16); i += nct) dsti[i] = src[i];
    }
    double* dst = Qu + (size_t)buf * a.Umax * a.V;
    if (!EXP(a, 1)) {
      // element e = u·V + vv, e = tid, tid + nct, …: (u, vv) stepped without divisions
      int u = tid / a.V, vv = tid - (tid / a.V) * a.V;
      const int du = nct / a.V, dv = nct - du * a.V;
      for (int e = tid; e < a.Umax * a.V; e += nct) {
        cp_async8(dst + e, qptr(a, uid[u], vv));
        u += du;
        vv += dv;
        if (vv >= a.V) {
          vv -= a.V;
          ++u;
        }
      }
    }
    cp_async_commit();
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[rg.st]);
    rg.next(S);
  };
  if (t0 < a.tile_end) gather_union(t0, 0);

  int buf = 0;
  for (int64_t tile = t0; tile < a.tile_end; tile += gridDim.x, buf ^= 1) {
    const int64_t c = tile * a.T + ct;
    const bool live = active && c < a.n_owned;
    cp_async_wait<0>();
    consumer_bar(nct);  // Q_u[buf] complete and visible; every consumer is done with tile t−1
    if (tile + gridDim.x < a.tile_end) gather_union(tile + gridDim.x, buf ^ 1);
    const double* Qb = Qu + (size_t)buf * a.Umax * a.V + v;
    const uint16_t* ix = (const uint16_t*)((const unsigned char*)Ix + buf * a.idx_bytes) + ct;  // [G][T]
    const double qi = Qb[ct * a.V];  // the tile's own cells lead its union (padded past n_owned)

    double acc[R];
#pragma unroll
    for (int l = 0; l < R; ++l) acc[l] = 0.0;
    double dqs[NCAP];
    // one chunk: ΔQ of kc positions, B⁺ columns accumulated in registers.  FULL:
    // kc == KC (static); CAP: capture the sector ΔQ (positions < NCAP; only the
    // first NCAPCH chunks, which make_layout guarantees to be full).
    auto chunk = [&](int ch, auto full_t, auto cap) {
      constexpr bool FULL = decltype(full_t)::value;
      const int kc = FULL ? KC : a.G - ch * KC;
      // ΔQ does not depend on the stage: formed before waiting for it
      const uint16_t* ic = ix + (size_t)ch * KC * a.T;
      double dq[KC];
#pragma unroll
      for (int kk = 0; kk < KC; ++kk) dq[kk] = (FULL || kk < kc) ? Qb[ic[kk * a.T]] - qi : 0.0;
      mbar_wait(&full[rg.st], rg.ph);
      const double* Bs = (const double*)(stg + rg.st * pc.stage_bytes);  // chunk_elem layout
      if (EXP(a, 2)) {
        acc[0] += dq[0];
      } else if (FULL) {
        if (decltype(cap)::value) {
#pragma unroll
          for (int kk = 0; kk < KC; ++kk)
            if (ch * KC + kk < NCAP) dqs[ch * KC + kk] = dq[kk];
        }
        // position pairs: 16-byte loads, the T cells of a (pair, row) adjacent
        const double2* b2 = reinterpret_cast<const double2*>(Bs) + ct;
#pragma unroll
        for (int l = 0; l < R; ++l) {
#pragma unroll
          for (int p = 0; p < KC / 2; ++p) {
            const double2 bb = b2[(p * R + l) * a.T];
            acc[l] = __fma_rn(bb.x, dq[2 * p], acc[l]);
            acc[l] = __fma_rn(bb.y, dq[2 * p + 1], acc[l]);
          }
        }
        if (KC % 2) {  // odd chunk size: the last position is stored [R][T]
          const double* b1 = Bs + (KC / 2) * R * a.T * 2 + ct;
#pragma unroll
          for (int l = 0; l < R; ++l) acc[l] = __fma_rn(b1[l * a.T], dq[KC - 1], acc[l]);
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < KC; ++kk) {
          if (kk < kc) {
#pragma unroll
            for (int l = 0; l < R; ++l) acc[l] = __fma_rn(Bs[chunk_elem(KIND_CELLVAR, kc, R, a.V, a.T, l, ct, kk)], dq[kk], acc[l]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[rg.st]);
      rg.next(S);
    };
    // first chunks (sector positions): fully unrolled so dqs[] stays in registers
#pragma unroll
    for (int ch = 0; ch < NCAPCH; ++ch) chunk(ch, std::true_type{}, std::true_type{});
    const int nfull = a.G / KC;
    for (int ch = NCAPCH; ch < nfull; ++ch) chunk(ch, std::true_type{}, std::false_type{});
    if (nfull < a.NCH) chunk(nfull, std::false_type{}, std::false_type{});

    // sector chunk: sector inverses + validity
    mbar_wait(&full[rg.st], rg.ph);
    const unsigned char* sb = stg + rg.st * pc.stage_bytes;
    const uint8_t vmask = sb[a.sinv_bytes + ct];
    bool valid[NV];
#pragma unroll
    for (int s = 0; s < NV; ++s) valid[s] = (vmask >> s) & 1;
    double ps[NV][D];
    sector_apply<D>((const double*)sb + size_t(ct) * NV * D * D, dqs, ps);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[rg.st]);
    rg.next(S);

    if (a.dense_out) {
      // per-warp staging + one bulk store of the warp's contiguous output rows
      const int64_t first = tile * (int64_t)TV + warp * 32;  // (cell·V + v) index of lane 0
      const int64_t lim = min((int64_t)TV, (a.n_owned - tile * a.T) * a.V) - warp * 32;
      const int nlive = (int)max((int64_t)0, min((int64_t)32, lim));
      if (lane == 0) bulk_wait_read();  // the staging rows are free again
      __syncwarp();
      if (EXP(a, 16)) {
        outw[lane * NM] = acc[0] + ps[0][0];
      } else {
        cweno_epilogue<D, NM>(qi, acc, ps, valid, a, outw + lane * NM, nullptr, nullptr);
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0 && nlive > 0) bulk_s2g(a.out + first * NM, outw, (uint32_t)(nlive * NM * 8));
    } else {
      double w[NM];
      cweno_epilogue<D, NM>(qi, acc, ps, valid, a, w, nullptr, nullptr);
      if (live) {
        double* o = a.out + c * a.ccs + v * a.cvs;
#pragma unroll
        for (int l = 0; l < NM; ++l) o[l] = w[l];
      }
    }
  }
  cp_async_wait<0>();
  if (lane == 0) bulk_wait_all();
}

// ---------------------------------------------------------------- boundary ghosts (R37)
__global__ void k_bc_fill(const double* __restrict__ Q, int64_t acs, int64_t avs, int V,
                          const int64_t* __restrict__ src, const int32_t* __restrict__ neg, int64_t n,
                          double* __restrict__ Qbc) {
  const int64_t gid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gid >= n * V) return;
  const int64_t g = gid / V;
  const int v = int(gid % V);
  const double x = Q[src[g] * acs + v * avs];
  Qbc[gid] = v == neg[g] ? -x : x;  // transmissive: copy; wall: −ρu_normal
}

static void bc_fill(cwreco_ctx* c, const double* avgs, int64_t acs, int64_t avs, cudaStream_t st) {
  DeviceState* ds = c->dev;
  if (ds->n_bc == 0) return;
  const int64_t th = ds->n_bc * c->V;
  k_bc_fill<<<(unsigned)((th + 255) / 256), 256, 0, st>>>(avgs, acs, avs, c->V, ds->bc_src, ds->bc_neg, ds->n_bc,
                                                          ds->Qbc);
  CK(cudaGetLastError());
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

template <int D, int M>
PipeFn pipe_fn_kc(int KC) {
  switch (KC) {
    case 1: return k_pipelined<D, M, 1>;
    case 2: return k_pipelined<D, M, 2>;
    case 3: return k_pipelined<D, M, 3>;
    case 4: return k_pipelined<D, M, 4>;
    case 5: return k_pipelined<D, M, 5>;
    case 6: return k_pipelined<D, M, 6>;
    case 8: return k_pipelined<D, M, 8>;
    default: fail(CWRECO_EUNSUPPORTED, "unsupported chunk size " + std::to_string(KC));
  }
}
PipeFn pipe_fn(int d, int M, int KC) {
#define CASE(DD, MM) \
  if (d == DD && M == MM) return pipe_fn_kc<DD, MM>(KC);
  CASE(2, 1) CASE(2, 2) CASE(2, 3) CASE(2, 4) CASE(3, 1) CASE(3, 2) CASE(3, 3)
#undef CASE
  fail(CWRECO_EUNSUPPORTED, "unsupported (d, M)");
}

static KArgs make_args(const cwreco_ctx* c, const double* avgs, int64_t acs, int64_t avs, double* out, int64_t ccs,
                       int64_t cvs) {
  const Layout& L = c->lay;
  KArgs a;
  std::memset(&a, 0, sizeof(a));
  a.blocks = c->dev->blocks;
  a.tile_bytes = L.tile_bytes;
  a.u_bytes = L.u_bytes;
  a.off_idx = L.off_idx;
  a.idx_bytes = L.idx_bytes;
  a.Umax = L.Umax;
  a.ids_bytes = L.ids_bytes;
  a.chunk_bytes = L.chunk_bytes;
  a.kslice_bytes = L.kslice_bytes;
  a.off_sector = L.off_sector;
  a.sinv_bytes = L.sinv_bytes;
  a.sector_bytes = L.sector_bytes;
  a.NSC = L.NSC;
  a.TSC = L.TSC;
  a.srec = L.srec;
  a.T = L.T;
  a.G = L.G;
  a.K = L.K;
  a.KC = L.KC;
  a.NCH = L.NCH;
  a.V = c->V;
  a.VP = L.VP;
  a.kind = L.kind;
  a.n_owned = c->n_owned;
  a.tile_begin = 0;
  a.tile_end = c->n_tiles;
  a.Q = avgs;
  a.acs = acs;
  a.avs = avs;
  a.n_local = c->n_owned + c->n_ghost;
  a.Qbc = c->dev ? c->dev->Qbc : nullptr;
  a.out = out;
  a.ccs = ccs;
  a.cvs = cvs;
  a.dense_out = 0;
#ifdef CWRECO_EXPERIMENTS
  {
    const char* e = std::getenv("CWRECO_EXP_FLAGS");  // bottleneck experiments (tools/exp_bench.py)
    a.exp_flags = e ? std::atoi(e) : 0;
  }
#endif
  a.eps = c->prm.eps;
  a.psi1 = c->psi1;
  a.r = c->prm.r;
  for (int n = 0; n <= c->d + 1; ++n) {
    const double denom = c->prm.lambda0 + n * c->prm.lambda_s;  // R5: λ normalised over valid stencils
    a.l0[n] = c->prm.lambda0 / denom;
    a.inv_l0[n] = 1.0 / a.l0[n];
    a.ls[n] = c->prm.lambda_s / denom;
  }
  return a;
}

bool rowblk_supported(int d, int M, int V) {
  return (d == 2 ? rowblk_fn_2d(M, V, true) : d == 3 ? rowblk_fn_3d(M, V, true) : nullptr) != nullptr;
}
static PipeFn rowblk_fn(const cwreco_ctx* c) {
  const bool full = c->lay.T == rb_tfull(c->lay.R, c->lay.V);
  PipeFn f = c->d == 2 ? rowblk_fn_2d(c->M, c->V, full) : rowblk_fn_3d(c->M, c->V, full);
  if (!f) fail(CWRECO_EUNSUPPORTED, "row-block kernel not instantiated for (d, M, V)");
  return f;
}

static PipeCfg pipe_cfg(const cwreco_ctx* c, int* ctas = nullptr) {
#ifdef CWRECO_EXPERIMENTS
  const char* kcap = std::getenv("CWRECO_CTAS");        // tuning experiments only
  const char* cap = std::getenv("CWRECO_MAX_STAGES");   // tuning experiments only (tools/sweep.py)
#else
  const char* kcap = nullptr;
  const char* cap = nullptr;
#endif
  if (c->dev->have_cfg && !cap && !kcap) {
    if (ctas) *ctas = c->dev->cfg_ctas;
    return c->dev->cfg;
  }
  const Layout& L = c->lay;
  PipeCfg p{};
  p.stage_bytes = pipe_stage_bytes(L);
  p.q_bytes = pipe_q_bytes(L);
  p.out_bytes = pipe_out_bytes(L);
  if (L.kind == KIND_ROWBLK) {
    // warp-specialised row-block kernel: one CTA per SM, the deepest stage ring that fits
    int k = 0, st = 0;
    rowblk_plan(L, c->dev->max_smem, 1, k, st);
    if (cap) st = std::max(kRbMinStages, std::min(st, std::atoi(cap)));
    if (!k) fail(CWRECO_EUNSUPPORTED, "row-block kernel: tile does not fit in shared memory");
    if (ctas) *ctas = 1;
    // the CTA keeps its compiled shape whatever T is (setmaxnreg acts per warp group:
    // the 4 main warps must fill warp group 0); main threads tid ≥ T·NG idle in the loop
    p.ncw = rb_main_warps(rb_tfull(L.R, L.V), rb_ng(L.R, L.V));
    p.eww = rb_ew(L.R, L.V);
    p.stages = st;
    p.stage_bytes = round128(L.chunk_bytes);
    p.ubuf_bytes = rb_ubuf_bytes(L);
    p.sbuf_bytes = rb_sbuf_bytes(L);
    p.q_bytes = round128(2 * int64_t(L.Umax) * L.VP * 8);
    p.out_bytes = round128(int64_t(L.T) * L.V * L.nm * 8);
    p.off_stage = 0;
    p.off_ubuf = st * p.stage_bytes;
    p.off_sbuf = p.off_ubuf + 3 * p.ubuf_bytes;
    p.off_q = p.off_sbuf + 2 * p.sbuf_bytes;
    p.off_out = p.off_q + p.q_bytes;
    p.off_bar = p.off_out + p.out_bytes;
    p.smem = p.off_bar + 8 * (2 * st + 12);
    if (p.smem != rb_smem(L, st)) fail(CWRECO_EUNSUPPORTED, "row-block kernel: shared-memory model mismatch");
    (void)kcap;
    return p;
  }
  if (ctas) *ctas = ctas_per_sm(c->nm);
  p.ncw = (L.T * c->V + 31) / 32;
  // as many stages as fit the per-CTA budget (ctas_per_sm CTAs/SM); a tile too
  // large for that budget runs at 1 CTA/SM with the whole shared memory.  The
  // prefetch cursor runs up to PF + 1 stages ahead of the consumers.
  int st = 0;
  const int smax = cap ? std::max(kMinStages, std::atoi(cap)) : kMaxStages;
  for (int64_t budget : {pipe_budget(c->nm, c->dev->max_smem), (int64_t)c->dev->max_smem}) {
    for (int s = smax; s >= kMinStages; --s)
      if (pipe_smem(L, s) <= budget) {
        st = s;
        break;
      }
    if (st) break;
  }
  if (!st) fail(CWRECO_EUNSUPPORTED, "pipelined kernel: tile does not fit in shared memory");
  p.stages = st;
  p.off_stage = 0;
  p.off_q = st * p.stage_bytes;
  p.off_out = p.off_q + p.q_bytes;
  p.off_bar = p.off_out + p.out_bytes;
  p.smem = p.off_bar + 16 * st;
  return p;
}

int dev_max_smem(const cwreco_ctx* c) { return c->dev ? c->dev->max_smem : 227 * 1024; }

void dev_create(cwreco_ctx* c) {
  if (c->device < 0) return;
  c->dev = new DeviceState();
  DeviceGuard dg(c->device);
  CK(cudaDeviceGetAttribute(&c->dev->num_sms, cudaDevAttrMultiProcessorCount, c->device));
  CK(cudaDeviceGetAttribute(&c->dev->max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
}

void dev_destroy(cwreco_ctx* c) {
  if (!c->dev) return;
  DeviceGuard dg(c->device);
  cudaFree(c->dev->blocks);
  cudaFree(c->dev->send);
  cudaFree(c->dev->dbg);
  cudaFree(c->dev->dbg_cells);
  cudaFree(c->dev->h_avgs);
  cudaFree(c->dev->h_coeffs);
  cudaFree(c->dev->bc_src);
  cudaFree(c->dev->bc_neg);
  cudaFree(c->dev->Qbc);
  for (cudaEvent_t e : c->dev->piece_done) cudaEventDestroy(e);
  if (c->dev->copy_stream) cudaStreamDestroy(c->dev->copy_stream);
  delete c->dev;
  c->dev = nullptr;
}

void dev_alloc_blocks(cwreco_ctx* c, int64_t bytes) {
  DeviceGuard dg(c->device);
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
  DeviceGuard dg(c->device);
  CK(cudaMemcpy(c->dev->blocks + offset, host, (size_t)bytes, cudaMemcpyHostToDevice));
}

void dev_upload_aux(cwreco_ctx* c) {
  const int nm = c->nm;
  {  // boundary ghosts (R37): source local ids and the negated (wall) variable
    DeviceGuard dg0(c->device);
    DeviceState* ds = c->dev;
    cudaFree(ds->bc_src);
    cudaFree(ds->bc_neg);
    cudaFree(ds->Qbc);
    ds->bc_src = nullptr;
    ds->bc_neg = nullptr;
    ds->Qbc = nullptr;
    ds->n_bc = (int64_t)c->bc_ids.size();
    if (ds->n_bc > 0) {
      std::vector<int64_t> own2local(c->own_hi - c->own_lo, -1);
      for (int64_t li = 0; li < c->n_owned; ++li) own2local[c->local2global[li] - c->own_lo] = li;
      std::vector<int64_t> src(ds->n_bc);
      std::vector<int32_t> neg(ds->n_bc);
      for (int64_t g = 0; g < ds->n_bc; ++g) {
        const int64_t id = c->bc_ids[g], s = (id - c->N) / c->N, k = (id - c->N) % c->N;
        src[g] = own2local[k - c->own_lo];
        neg[g] = (c->bc[s] == 2 && c->mom0 >= 0) ? int32_t(c->mom0 + s / 2) : -1;
      }
      CK(cudaMalloc(&ds->bc_src, ds->n_bc * 8));
      CK(cudaMalloc(&ds->bc_neg, ds->n_bc * 4));
      CK(cudaMalloc(&ds->Qbc, ds->n_bc * c->V * 8));
      CK(cudaMemcpy(ds->bc_src, src.data(), ds->n_bc * 8, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(ds->bc_neg, neg.data(), ds->n_bc * 4, cudaMemcpyHostToDevice));
    }
  }
  std::vector<double> packed;
  for (int l = 1; l < nm; ++l)
    for (int m = l; m < nm; ++m) packed.push_back((l == m ? 1.0 : 2.0) * c->sigma[l * nm + m]);
  DeviceGuard dg(c->device);
  const size_t sb = sizeof(double) * packed.size(), so = sizeof(double) * sig_off(c->d, c->M);
  CK(cudaMemcpyToSymbol(c_sig, packed.data(), sb, so));
  CK(rowblk_upload_sigma_2d(packed.data(), sb, so));
  CK(rowblk_upload_sigma_3d(packed.data(), sb, so));
  PipeFn f = c->lay.kind == KIND_ROWBLK ? rowblk_fn(c) : pipe_fn(c->d, c->M, c->lay.KC);
  CK(cudaFuncSetAttribute((const void*)f, cudaFuncAttributeMaxDynamicSharedMemorySize, c->dev->max_smem));
  c->dev->have_cfg = false;
  c->dev->cfg = pipe_cfg(c, &c->dev->cfg_ctas);
  c->dev->have_cfg = true;
}

void dev_download_tile(const cwreco_ctx* c, int64_t tile, unsigned char* host) {
  DeviceGuard dg(c->device);
  CK(cudaMemcpy(host, c->dev->blocks + tile * c->lay.tile_bytes, (size_t)c->lay.tile_bytes, cudaMemcpyDeviceToHost));
}

int64_t dev_bytes(const cwreco_ctx* c) {
  if (!c->dev) return 0;
  return c->dev->blocks_bytes + c->dev->dbg_bytes + c->dev->n_send * 8 + (c->dev->h_avgs_n + c->dev->h_coeffs_n) * 8;
}

// One launch of the reconstruction over owned tiles [tile_begin, tile_end).
static void launch_range(cwreco_ctx* c, const double* avgs, int64_t acs, int64_t avs, double* coeffs, int64_t ccs,
                         int64_t cvs, int64_t tile_begin, int64_t tile_end, cudaStream_t st) {
  KArgs a = make_args(c, avgs, acs, avs, coeffs, ccs, cvs);
  a.tile_begin = tile_begin;
  a.tile_end = tile_end;
  if (a.tile_end <= a.tile_begin) return;
  const int nm = c->nm;
  if (c->kernel == CWRECO_KERNEL_SIMPLE) {
    const int64_t cells = std::min(a.tile_end * a.T, c->n_owned) - a.tile_begin * a.T;
    const int64_t threads = cells * c->V;
    dim3 b(256), g((unsigned)((threads + 255) / 256));
    DbgOut o{};
    launch_simple<false>(c->d, c->M, g, b, st, a, o);
  } else {
    a.dense_out = (cvs == nm && ccs == (int64_t)c->V * nm && (((uintptr_t)coeffs) & 15) == 0 && nm % 2 == 0) ? 1 : 0;
    int per_sm = 1;
    PipeCfg p = pipe_cfg(c, &per_sm);
    const int64_t ntiles = a.tile_end - a.tile_begin;
    int64_t grid = std::min<int64_t>(ntiles, (int64_t)c->dev->num_sms * per_sm);
    if (c->max_ctas > 0) grid = std::min<int64_t>(grid, c->max_ctas);  // CWRECO_OPT_MAX_CTAS
    dim3 b((p.ncw + (c->lay.kind == KIND_ROWBLK ? p.eww : 0) + 1) * 32), g((unsigned)grid);
    PipeFn f = c->lay.kind == KIND_ROWBLK ? rowblk_fn(c) : pipe_fn(c->d, c->M, c->lay.KC);
    f<<<g, b, p.smem, st>>>(a, p);
  }
  CK(cudaGetLastError());
}

void dev_reconstruct(cwreco_ctx* c, const double* avgs, int64_t acs, int64_t avs, double* coeffs, int64_t ccs,
                     int64_t cvs, int part, void* stream) {
  DeviceGuard dg(c->device);
  if (c->kernel == CWRECO_KERNEL_MATRIXFREE) {  // cells, not tiles: interior first in local order
    const int64_t c0 = part == CWRECO_PART_BOUNDARY ? c->n_interior : 0;
    const int64_t c1 = part == CWRECO_PART_INTERIOR ? c->n_interior : c->n_owned;
    dev_matfree_reconstruct(c, avgs, acs, avs, coeffs, ccs, cvs, c0, c1, stream);
    return;
  }
  bc_fill(c, avgs, acs, avs, (cudaStream_t)stream);
  int64_t t0 = 0, t1 = c->n_tiles;
  if (part == CWRECO_PART_INTERIOR) {
    t1 = c->n_int_tiles;
  } else if (part == CWRECO_PART_BOUNDARY) {
    t0 = c->n_int_tiles;
  }
  launch_range(c, avgs, acs, avs, coeffs, ccs, cvs, t0, t1, (cudaStream_t)stream);
}

// cwreco_reconstruct_host: H2D of the averages, n_pieces tile ranges on `stream`,
// each range's D2H on the copy stream as soon as its event fires.
void dev_reconstruct_host(cwreco_ctx* c, const double* h_avgs, double* h_coeffs, int n_pieces, void* stream) {
  DeviceState* ds = c->dev;
  cudaStream_t st = (cudaStream_t)stream;
  DeviceGuard dg(c->device);
  const int V = c->V, nm = c->nm;
  const int64_t na = (c->n_owned + c->n_ghost) * V, nc = c->n_owned * V * nm;
  auto grow = [&](double*& p, int64_t& have, int64_t need_n) {
    if (have >= need_n) return;
    cudaFree(p);
    p = nullptr;
    have = 0;
    if (cudaMalloc(&p, std::max<int64_t>(1, need_n) * 8) != cudaSuccess) {
      cudaGetLastError();
      fail(CWRECO_ENOMEM, "reconstruct_host: device buffer allocation failed");
    }
    have = need_n;
  };
  grow(ds->h_avgs, ds->h_avgs_n, na);
  grow(ds->h_coeffs, ds->h_coeffs_n, nc);
  if (!ds->copy_stream) CK(cudaStreamCreateWithFlags(&ds->copy_stream, cudaStreamNonBlocking));
  while ((int)ds->piece_done.size() < n_pieces) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ds->piece_done.push_back(e);
  }
  CK(cudaMemcpyAsync(ds->h_avgs, h_avgs, na * 8, cudaMemcpyHostToDevice, st));
  if (c->kernel != CWRECO_KERNEL_MATRIXFREE) bc_fill(c, ds->h_avgs, V, 1, st);
  const bool mf = c->kernel == CWRECO_KERNEL_MATRIXFREE;  // pieces of cells instead of tiles
  const int64_t nt = mf ? c->n_owned : c->n_tiles, T = mf ? 1 : c->lay.T, row = (int64_t)V * nm;
  for (int k = 0; k < n_pieces; ++k) {
    const int64_t a = nt * k / n_pieces, b = nt * (k + 1) / n_pieces;
    if (b <= a) continue;
    if (mf)
      dev_matfree_reconstruct(c, ds->h_avgs, V, 1, ds->h_coeffs, row, nm, a, b, st);
    else
      launch_range(c, ds->h_avgs, V, 1, ds->h_coeffs, row, nm, a, b, st);
    CK(cudaEventRecord(ds->piece_done[k], st));
    CK(cudaStreamWaitEvent(ds->copy_stream, ds->piece_done[k], 0));
    const int64_t c0 = a * T, c1 = std::min(c->n_owned, b * T);
    CK(cudaMemcpyAsync(h_coeffs + c0 * row, ds->h_coeffs + c0 * row, (c1 - c0) * row * 8, cudaMemcpyDeviceToHost,
                       ds->copy_stream));
  }
  CK(cudaStreamSynchronize(ds->copy_stream));
  CK(cudaStreamSynchronize(st));
}

void dev_debug(cwreco_ctx* c, const double* avgs, int64_t acs, int64_t avs, int64_t n_sel, const int64_t* cells,
               double* popt, double* psec, double* sigma, double* omega, double* w, void* stream) {
  DeviceGuard dg(c->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int V = c->V, nm = c->nm, NV = c->d + 1;
  const int64_t n_popt = n_sel * V * nm, n_psec = n_sel * NV * V * NV, n_sig = n_sel * (NV + 1) * V;
  const int64_t total = n_popt + n_psec + 2 * n_sig + n_popt;
  const int64_t bytes = total * 8;
  if (bytes > c->dev->dbg_bytes) {
    cudaFree(c->dev->dbg);
    c->dev->dbg = nullptr;
    CK(cudaMalloc(&c->dev->dbg, bytes));
    c->dev->dbg_bytes = bytes;
  }
  if (n_sel > c->dev->dbg_ncells) {
    cudaFree(c->dev->dbg_cells);
    c->dev->dbg_cells = nullptr;
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
  bc_fill(c, avgs, acs, avs, st);
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
  DeviceGuard dg(c->device);
  cudaFree(c->dev->send);
  c->dev->send = nullptr;
  c->dev->n_send = (int64_t)c->send_local.size();
  if (c->dev->n_send == 0) return;
  CK(cudaMalloc(&c->dev->send, c->dev->n_send * 8));
  CK(cudaMemcpy(c->dev->send, c->send_local.data(), c->dev->n_send * 8, cudaMemcpyHostToDevice));
}

void dev_halo_pack(cwreco_ctx* c, const double* avgs, int64_t acs, int64_t avs, double* sendbuf, void* stream) {
  dev_halo_pack_rows(c, avgs, acs, avs, c->V, sendbuf, stream);
}

void dev_halo_pack_rows(cwreco_ctx* c, const double* rows, int64_t rs, int64_t es, int width, double* sendbuf,
                        void* stream) {
  DeviceGuard dg(c->device);
  const int64_t n = c->dev->n_send;
  if (n == 0) return;
  const int64_t threads = n * width;
  k_halo_pack<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(rows, rs, es, width, c->dev->send,
                                                                                     n, sendbuf);
  CK(cudaGetLastError());
}

}  // namespace cwr
