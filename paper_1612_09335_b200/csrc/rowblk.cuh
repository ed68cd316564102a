// k_rowblk: the row-block CWENO reconstruction kernel (sm_100a), for ℳ ≥ 10.
//
// The central LSQ apply is, per cell, the small product
//     p̂_opt[1..R][v] = B⁺[R][G] · ΔQ[G][V]      (R = ℳ−1 reduced rows, G positions).
// k_pipelined gives every (cell, variable) its own thread, so each B⁺ element is
// read from shared memory by V lanes (a broadcast that still costs a full
// wavefront per quarter-warp: ncu counts ~4 wavefronts per LDS.128, and the
// shared-memory pipe saturates at ~83 % on C4).  Here a thread owns one cell and
// a group of RB rows for ALL V variables: each B⁺ element is loaded once and used
// V times from registers, and only the V averages of a position are broadcast
// (NG threads per cell).  Shared-memory wavefronts per cell and position drop
// from V·(R+1)·8/128 to (R + NG·V)·8/128 (C4: 11.3 → 3.4).
//
// Pipeline (persistent, warp-specialised, as k_pipelined):
//  - producer warp (one elected lane): per tile, the union chunk of the CTA's
//    NEXT tile, then the position chunks, then the sector chunk, into a ring of S
//    stages with 1-D TMA bulk copies completing on mbarrier transaction counts;
//  - consumers (T cells × NG row groups): at tile start they cp.async the V
//    averages of every cell of the next tile's stencil union into the other half
//    of a double-buffered Q_u[2][Umax][VP]; per position: acc[r][v] +=
//    B⁺[row r][p]·Q_u[idx][v] for the thread's rows and all V (B⁺ΔQ = B⁺Q − rs·Q_i
//    is completed in the epilogue with the stored row sums rs); after the
//    last chunk the row groups write p̂_opt into the tile's output rows
//    O[T][V][ℳ] (slots 1..R), and one thread per (cell, variable) runs the fused
//    sector / P0 / σ / ω / blend epilogue in place (reading its sector ΔQ back
//    from Q_u) — the tile's output block is then written with one bulk store.
// Arithmetic per (cell, variable) and its order are those of k_simple (bitwise
// identical results, tested).
#pragma once
#include "kcommon.cuh"

namespace cwr {

constexpr int KC = kRbKC;                       // positions per chunk (compile time)

template <int D, int M, int V>
__global__ void __launch_bounds__(rb_consumers(nmodes(M, D) - 1, V) + 32, 1) k_rowblk(KArgs a, PipeCfg pc) {
  constexpr int NM = nmodes(M, D), R = NM - 1, NV = D + 1, NCAP = NV * D;
  constexpr int NG = rb_ng(R, V), RB = rb_rb(R, V), NF = rb_nfull(R, V);
  constexpr int VP = V + (V & 1);
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* stg = smem + pc.off_stage;
  double* O = (double*)(smem + pc.off_out);  // [T][V][ℳ] output rows of the tile
  double* Qu = (double*)(smem + pc.off_q);   // [2][Umax][VP] gathered averages
  uint16_t* Ix = (uint16_t*)(smem + pc.off_q + ((2 * (int64_t)a.Umax * VP * 8 + 127) & ~int64_t(127)));  // [2][G][T]
  uint64_t* bars = (uint64_t*)(smem + pc.off_bar);
  const int S = pc.stages;
  uint64_t* full = bars;       // [S]
  uint64_t* empty = bars + S;  // [S]
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int T = a.T;
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
          issue(tb + a.u_bytes + ch * a.chunk_bytes, (uint32_t)(min(a.KC, a.G - ch * a.KC) * a.kslice_bytes));
        for (int j = 0; j < a.NSC; ++j) issue(tb + a.off_sector + j * a.sector_bytes, (uint32_t)a.sector_bytes);
      }
    }
    return;
  }

  // -------------------------------------------------- consumer warps
  const int nct = pc.ncw * 32;  // T·NG main-loop threads (+ epilogue-only warps, rb_cons_for)
  const bool mainthr = tid < T * NG;
  const int ct = mainthr ? tid / NG : 0, g = mainthr ? tid % NG : 0;
  // offsets of this thread's B⁺ entries inside a row slot (chunk_elem, KIND_ROWBLK):
  // slots r < RB−1 hold all NG groups, the last one the first NF (a group without a
  // row there reads a neighbour's entry into an accumulator that is never written out)
  const int bfull = ct * NG + g, bpart = ct * NF + min(g, NF - 1);
  Ring rg;
  // gather the union of the next tile (its union chunk is the current stage) into
  // Q_u[bufn] and copy its position → union-offset table into Ix[bufn]
  auto gather_union = [&](int bufn) {
    mbar_wait(&full[rg.st], rg.ph);
    const unsigned char* ub = stg + rg.st * pc.stage_bytes;
    const int32_t* uid = (const int32_t*)ub;
    {
      const uint4* src = (const uint4*)(ub + a.off_idx);
      uint4* dsti = (uint4*)((unsigned char*)Ix + bufn * a.idx_bytes);
      for (int i = tid; i < (int)(a.idx_bytes / 16); i += nct) dsti[i] = src[i];
    }
    double* dst = Qu + (size_t)bufn * a.Umax * VP;
    if (EXP(a, 1)) {  // experiment: no gather (timing only)
      cp_async_commit();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[rg.st]);
      rg.next(S);
      return;
    }
    // element e = u·V + vv, e = tid, tid + nct, …: (u, vv) stepped without divisions
    int u = tid / V, vv = tid - (tid / V) * V;
    const int du = nct / V, dv = nct - du * V;
    for (int e = tid; e < a.Umax * V; e += nct) {
      cp_async8(dst + u * VP + vv, a.Q + int64_t(uid[u]) * a.acs + vv * a.avs);
      u += du;
      vv += dv;
      if (vv >= V) {
        vv -= V;
        ++u;
      }
    }
    cp_async_commit();
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[rg.st]);
    rg.next(S);
  };
  auto store_tile = [&](int64_t tile) {  // one bulk store of the tile's live output rows
    const int64_t nlive = min((int64_t)T, a.n_owned - tile * T);
    if (nlive > 0) bulk_s2g(a.out + tile * T * (int64_t)(V * NM), O, (uint32_t)(nlive * V * NM * 8));
  };
  if (t0 < a.tile_end) gather_union(0);

  int buf = 0;
  int64_t prev = -1;
  for (int64_t tile = t0; tile < a.tile_end; tile += gridDim.x, buf ^= 1) {
    cp_async_wait<0>();
    consumer_bar(nct);  // Q_u[buf] complete and visible; tile t−1 fully done (O written, Q_u[buf^1] free)
    if (a.dense_out && tid == 0 && prev >= 0) store_tile(prev);
    if (tile + gridDim.x < a.tile_end) gather_union(buf ^ 1);
    const double* Qb = Qu + (size_t)buf * a.Umax * VP;
    const uint16_t* ixb = (const uint16_t*)((const unsigned char*)Ix + buf * a.idx_bytes);

    double acc[RB][V];
#pragma unroll
    for (int r = 0; r < RB; ++r)
#pragma unroll
      for (int v = 0; v < V; ++v) acc[r][v] = 0.0;
    // Main loop over chunks of KC = 2 positions, software-pipelined: the averages of
    // chunk ch+1 and the union offsets of chunk ch+2 are loaded while chunk ch's
    // FMAs run (they do not depend on the stage ring); the B⁺ entries of chunk ch+1
    // are loaded right after its stage arrives, before chunk ch's stage is released.
    // Ping-pong buffers (qa/qb, ba/bb) avoid register moves.  A trailing odd
    // position (G odd) is peeled.
    static_assert(KC % 2 == 0, "row-block chunks hold whole position pairs");
    constexpr int PPS = KC / 2;  // position pairs per stage
    const int G = a.G, nfc = G / 2, npr = (G + 1) / 2;  // full pairs; pairs incl. a trailing single
    const uint32_t* ix2 = reinterpret_cast<const uint32_t*>(ixb) + ct;  // [pair][T] offset pairs
    auto ldq = [&](int off, double (&d)[V]) {
      const double* q = Qb + off;
#pragma unroll
      for (int v = 0; v + 1 < V; v += 2) {
        const double2 x = *reinterpret_cast<const double2*>(q + v);
        d[v] = x.x;
        d[v + 1] = x.y;
      }
      if (V & 1) d[V - 1] = q[V - 1];
    };
    auto ldq2 = [&](uint32_t pr, double (&d)[2][V]) {
      ldq(int(pr & 0xffffu), d[0]);
      ldq(int(pr >> 16), d[1]);
    };
    auto ldb = [&](const double* Bs, double (&b)[2][RB]) {  // Bs: the pair's first position
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int r = 0; r < RB; ++r) b[k][r] = Bs[(k * R + r * NG) * T + (r < RB - 1 ? bfull : bpart)];
    };
    // B⁺Q on the raw averages (no per-lane ΔQ subtractions); B⁺ΔQ = B⁺Q − rs·Q_i is
    // formed in the epilogue with the row sums rs of the sector record (|B⁺| rows sum
    // to < 1 on the configs, so the cancellation costs ~1e-16·max|Q|, far inside R25)
    auto fma_pos = [&](const double (&q)[V], const double (&b)[RB]) {
#pragma unroll
      for (int r = 0; r < RB; ++r)
#pragma unroll
        for (int v = 0; v < V; ++v) acc[r][v] = __fma_rn(b[r], q[v], acc[r][v]);
    };
    auto stage_ptr = [&]() { return (const double*)(stg + rg.st * pc.stage_bytes); };
    auto release = [&]() {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[rg.st]);
      rg.next(S);
    };
    if (!mainthr) {  // epilogue-only warps (warp-uniform): walk the ring, no math
      for (int c2 = 0; c2 < a.NCH; ++c2) {
        mbar_wait(&full[rg.st], rg.ph);
        release();
      }
    } else {
    double qa[2][V], qb[2][V], ba[2][RB], bb[2][RB];
    ldq2(ix2[0], qa);
    uint32_t ipn = ix2[min(1, npr - 1) * T];
    mbar_wait(&full[rg.st], rg.ph);
    ldb(stage_ptr(), ba);
    // one full pair pp: q/b hold its averages and B⁺ entries; qn/bn receive pair pp+1's
    // (from the same stage, or from the next one, which releases the current stage)
    auto pair = [&](int pp, const double (&q)[2][V], const double (&b)[2][RB], double (&qn)[2][V],
                    double (&bn)[2][RB]) {
      ldq2(ipn, qn);
      ipn = ix2[min(pp + 2, npr - 1) * T];
      fma_pos(q[0], b[0]);
      fma_pos(q[1], b[1]);
      const int nx = pp + 1;
      if (nx >= npr) {
        release();
      } else if (nx % PPS == 0) {  // next stage (a tail pair reads past kc into the stage: unused)
        Ring nr = rg;
        nr.next(S);
        mbar_wait(&full[nr.st], nr.ph);
        ldb((const double*)(stg + nr.st * pc.stage_bytes), bn);
        release();
      } else {
        ldb(stage_ptr() + (nx % PPS) * 2 * R * T, bn);
      }
    };
    int pp = 0;
    for (; pp + 1 < nfc; pp += 2) {
      pair(pp, qa, ba, qb, bb);
      pair(pp + 1, qb, bb, qa, ba);
    }
    const bool odd_pair = pp < nfc;
    if (odd_pair) pair(pp, qa, ba, qb, bb);
    if (G & 1) {  // the last position alone (its stage already waited for)
      fma_pos(odd_pair ? qb[0] : qa[0], odd_pair ? bb[0] : ba[0]);
      release();
    }
    }  // main-loop threads

    // (after the previous tile's bulk store has read O)
    if (tid == 0) bulk_wait_read();
    consumer_bar(nct);
    const Ring rs = rg;  // the sector pieces: NSC consecutive stages
    for (int j = 0; j < a.NSC; ++j) {
      mbar_wait(&full[rg.st], rg.ph);
      rg.next(S);
    }
    // ---- per-item epilogue: p̂_opt rows → O[ct][v][1 + row], then one thread per
    // (cell, variable) runs cweno_epilogue in place
    if (mainthr) {
      double* Oc = O + (size_t)ct * V * NM + 1 + g;  // row l = r·NG + g
#pragma unroll
      for (int r = 0; r < RB; ++r)
        if (r < RB - 1 || g < NF)
#pragma unroll
          for (int v = 0; v < V; ++v) Oc[v * NM + r * NG] = acc[r][v];
    }
    consumer_bar(nct);
    for (int item = tid; item < (EXP(a, 16) ? 0 : T * V); item += nct) {  // flag 16: no epilogue
      const int c2 = item / V, v2 = item - (item / V) * V;
      const int j = c2 / a.TSC, cl = c2 - j * a.TSC;
      const int sst = rs.st + j < S ? rs.st + j : rs.st + j - S;
      const unsigned char* sb = stg + sst * pc.stage_bytes;
      const double q2 = Qb[c2 * VP + v2];
      double* row = O + (size_t)item * NM;
      const double* srec = (const double*)sb + size_t(cl) * a.srec;  // sector inverses, then rs
      double accr[R];
#pragma unroll
      for (int l = 0; l < R; ++l) accr[l] = __fma_rn(-srec[NV * D * D + l], q2, row[1 + l]);
      double dqs[NCAP];
#pragma unroll
      for (int p = 0; p < NCAP; ++p) dqs[p] = Qb[ixb[idx_elem(KIND_ROWBLK, T, p, c2)] + v2] - q2;
      const uint8_t vmask = sb[a.sinv_bytes + cl];
      bool valid[NV];
#pragma unroll
      for (int q = 0; q < NV; ++q) valid[q] = (vmask >> q) & 1;
      double ps[NV][D];
      sector_apply<D>(srec, dqs, ps);
      if (a.dense_out) {
        cweno_epilogue<D, NM>(q2, accr, ps, valid, a, row, nullptr, nullptr);
      } else {
        double w[NM];
        cweno_epilogue<D, NM>(q2, accr, ps, valid, a, w, nullptr, nullptr);
        const int64_t c = tile * T + c2;
        if (c < a.n_owned) {
          double* o = a.out + c * a.ccs + v2 * a.cvs;
#pragma unroll
          for (int l = 0; l < NM; ++l) o[l] = w[l];
        }
      }
    }
    __syncwarp();
    if (lane == 0) {
      int sst = rs.st;
      for (int j = 0; j < a.NSC; ++j) {
        mbar_arrive(&empty[sst]);
        if (++sst == S) sst = 0;
      }
    }
    if (a.dense_out) fence_proxy_async();  // O rows → visible to the bulk store after the next barrier
    prev = tile;
  }
  consumer_bar(nct);
  if (a.dense_out && tid == 0 && prev >= 0) {
    store_tile(prev);
    bulk_wait_all();
  }
  cp_async_wait<0>();
}

// Instantiations per translation unit (rowblk_2d.cu, rowblk_3d.cu)
template <int D, int M>
PipeFn rowblk_fn_v(int V) {
  switch (V) {
    case 1: return k_rowblk<D, M, 1>;
    case 2: return k_rowblk<D, M, 2>;
    case 3: return k_rowblk<D, M, 3>;
    case 4: return k_rowblk<D, M, 4>;
    case 5: return k_rowblk<D, M, 5>;
    case 6: return k_rowblk<D, M, 6>;
    case 7: return k_rowblk<D, M, 7>;
    case 8: return k_rowblk<D, M, 8>;
    case 9: return k_rowblk<D, M, 9>;
    default: return nullptr;
  }
}

}  // namespace cwr
