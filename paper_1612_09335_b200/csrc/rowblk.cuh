// k_rowblk: the row-block CWENO reconstruction kernel (sm_100a), for ℳ ≥ 10.
//
// The central LSQ apply is, per cell, the small product
//     p̂_opt[1..R][v] = B⁺[R][G] · Q[G][V]      (R = ℳ−1 reduced rows, G positions).
// A thread owns one cell and a group of RB rows for ALL V variables: each B⁺
// element is loaded from shared memory once and used V times from registers;
// only the V averages of a position are broadcast to the NG threads of the cell.
//
// Warp specialisation (persistent, one CTA per SM), three roles:
//  - producer warp (one elected lane): streams, with 1-D TMA bulk copies completing
//    on mbarrier transaction counts, per tile t_k of the CTA: its position chunks
//    into a ring of S stages; the union chunk of t_{k+2} (stencil-union cell ids +
//    position → union offsets) into one of 3 union buffers; the sector chunk of
//    t_{k+1} (sector inverses, B⁺ row sums, validity) into one of 2 sector buffers.
//  - main warps (T cells × NG row groups): per tile, wait for the tile's gathered
//    averages Q_u[k%2], run the B⁺·Q main loop over the ring (software-pipelined
//    over position pairs), then hand the p̂_opt rows to the epilogue warps through
//    the output block O[T][V][ℳ] (named barriers OFREE / OFULL) and go straight on
//    to the next tile.
//  - epilogue warps: per tile, one thread per (cell, variable) runs the fused
//    sector / P0 / σ / ω / blend epilogue in place in O, one bulk store
//    writes the tile's rows, the buffers of the tile are released, and the stencil
//    averages of tile t_{k+2} are gathered into Q_u[k%2] with cp.async (completion
//    on an mbarrier) — all of it while the main warps stream tile t_{k+1}.
// So the epilogue and the gather no longer serialise with the B⁺ stream (round 1:
// one thread set did both, and the stream stalled during every epilogue).
// Arithmetic per (cell, variable) and its order are those of k_simple (bitwise
// identical results, tested).
#pragma once
#include "kcommon.cuh"

namespace cwr {

constexpr int KC = kRbKC;  // positions per chunk (compile time)

// Timeline probes of CTA 0 (tuning builds with -DCWR_TRACE only; tools/c4_iter.py --trace)
#ifdef CWR_TRACE
static __device__ long long g_rb_trace[64][16];
#define RB_TRACE(k, slot)                                              \
  do {                                                                 \
    if (blockIdx.x == 0 && (k) < 64) g_rb_trace[k][slot] = clock64(); \
  } while (0)
#else
#define RB_TRACE(k, slot) \
  do {                    \
  } while (0)
#endif
constexpr int RB_BAR_OFULL = 1, RB_BAR_OFREE = 2, RB_BAR_EW = 3;
#ifndef CWR_RB_PAIR
#define CWR_RB_PAIR 0  // epilogue items computed two at a time (measured slower: registers)
#endif
#ifndef CWR_RB_PF
#define CWR_RB_PF 0  // B⁺ of the next pair loaded per position between the FMAs (see pair())
#endif
// Whole-stage main loop without the per-pair stage / end tests: -1 = for ℳ = 20 only
// (measured, same box: C4 proxy 0.841 vs 0.760, C5 shape 1.055 vs 1.040; 3-D M = 2 on
// C3 0.712 vs 0.725), 0 = never, 1 = always
#ifndef CWR_RB_STATIC
#define CWR_RB_STATIC -1
#endif
#ifndef CWR_RB_L2PF
#define CWR_RB_L2PF 0  // producer: L2 prefetch this many position chunks ahead (0: none)
#endif
#ifndef CWR_RB_TT
#define CWR_RB_TT 1  // instantiate the full tile size T as a compile-time constant
#endif
#ifndef CWR_RB_LOOK1
#define CWR_RB_LOOK1 0  // main loop with a one-position lookahead instead of the pair ping-pong
#endif

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// TT > 0: the tile holds TT cells (compile time: the B⁺ slot offsets (r·NG + kk·R)·T
// become immediates of the shared loads); TT = 0: a.T (a layout whose tile was halved)
template <int D, int M, int V, int TT>
__global__ void __launch_bounds__(rb_threads(nmodes(M, D) - 1, V), 1) k_rowblk(KArgs a, PipeCfg pc) {
  constexpr int NM = nmodes(M, D), R = NM - 1, NV = D + 1, NCAP = NV * D;
  constexpr int NG = rb_ng(R, V), RB = rb_rb(R, V), NF = rb_nfull(R, V);
  constexpr int VP = V + (V & 1);
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* stg = smem + pc.off_stage;
  double* O = (double*)(smem + pc.off_out);  // [T][V][ℳ] output rows of the tile
  double* Qu = (double*)(smem + pc.off_q);   // [2][Umax][VP] gathered averages
  unsigned char* ubuf = smem + pc.off_ubuf;  // [3] union chunks (uid int32[Umax] | idx)
  unsigned char* sbuf = smem + pc.off_sbuf;  // [2] sector chunks
  uint64_t* bars = (uint64_t*)(smem + pc.off_bar);
  const int S = pc.stages;
  uint64_t* full = bars;        // [S] ring
  uint64_t* empty = bars + S;   // [S]
  uint64_t* ufull = bars + 2 * S;   // [3]
  uint64_t* uempty = ufull + 3;     // [3]
  uint64_t* sfull = uempty + 3;     // [2]
  uint64_t* sempty = sfull + 2;     // [2]
  uint64_t* qfull = sempty + 2;     // [2] gather of Q_u[b] complete
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int T = TT > 0 ? TT : a.T;
  const int MW = pc.ncw * 32, EW = pc.eww * 32, NB = MW + EW;  // main / epilogue threads
  const int64_t t0 = a.tile_begin + blockIdx.x;                 // this CTA's tiles: t0 + k·grid
  const int nk = t0 < a.tile_end ? int((a.tile_end - 1 - t0) / gridDim.x + 1) : 0;
  auto tile_of = [&](int k) { return t0 + int64_t(k) * gridDim.x; };

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], pc.ncw);
    }
    for (int s = 0; s < 3; ++s) {
      mbar_init(&ufull[s], 1);
      mbar_init(&uempty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sfull[s], 1);
      mbar_init(&sempty[s], 1);
      mbar_init(&qfull[s], EW);
    }
    fence_barrier_init();
  }
  __syncthreads();

  // register rebalancing between the warp groups (setmaxnreg): warp group 0 = the main
  // warps takes MAINREG registers per thread, the epilogue / producer groups give theirs
  // back (the increase must be covered by what the other two release, else it waits)
  constexpr int MAINREG = rb_mainreg(R, V), OTHERREG = rb_otherreg(R, V);
  static_assert(!MAINREG || (rb_main(R, V) == 128 && rb_threads(R, V) == 384), "setmaxnreg: 3 warp groups");
  auto reg_main = [] {
    if constexpr (MAINREG > 0) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(MAINREG));
  };
  auto reg_other = [] {
    if constexpr (MAINREG > 0) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(OTHERREG));
  };
  if (warp == pc.ncw + pc.eww) {
    // ------------------------------------------------ TMA producer
    reg_other();
    if (lane == 0) {
      Ring rg;
      auto load_union = [&](int k) {  // union chunk of tile k → ubuf[k%3]
        const int s = k % 3;
        mbar_wait_sleep(&uempty[s], ((k / 3) & 1) ^ 1);
        mbar_expect_tx(&ufull[s], (uint32_t)a.u_bytes);
        bulk_g2s(ubuf + s * pc.ubuf_bytes, a.blocks + tile_of(k) * a.tile_bytes, (uint32_t)a.u_bytes, &ufull[s]);
      };
      auto load_sector = [&](int k) {  // all sector pieces of tile k → sbuf[k%2]
        const int s = k & 1;
        const uint32_t bytes = (uint32_t)(a.NSC * a.sector_bytes);
        mbar_wait_sleep(&sempty[s], ((k >> 1) & 1) ^ 1);
        mbar_expect_tx(&sfull[s], bytes);
        bulk_g2s(sbuf + s * pc.sbuf_bytes, a.blocks + tile_of(k) * a.tile_bytes + a.off_sector, bytes, &sfull[s]);
      };
      for (int k = 0; k < nk && k < 2; ++k) load_union(k);
      if (nk > 0) load_sector(0);
#if CWR_RB_L2PF > 0
      // L2 prefetch of the position chunks CWR_RB_L2PF chunks beyond the one being
      // loaded into the ring: more bytes in flight than the ring's shared memory holds,
      // so a stage's bulk copy finds its chunk in L2
      int pfk = 0, pfc = 0;  // next chunk to prefetch (tile k of this CTA, chunk)
      auto prefetch_to = [&](int k, int ch) {
        const int64_t lim = int64_t(k) * a.NCH + ch + CWR_RB_L2PF;
        while (pfk < nk && int64_t(pfk) * a.NCH + pfc <= lim) {
          const uint32_t bytes = (uint32_t)(min(a.KC, a.G - pfc * a.KC) * a.kslice_bytes);
          bulk_prefetch_l2(a.blocks + tile_of(pfk) * a.tile_bytes + a.u_bytes + pfc * a.chunk_bytes, bytes);
          if (++pfc == a.NCH) {
            pfc = 0;
            ++pfk;
          }
        }
      };
#endif
      for (int k = 0; k < nk; ++k) {
        RB_TRACE(k, 9);
        const unsigned char* tb = a.blocks + tile_of(k) * a.tile_bytes;
        for (int ch = 0; ch < a.NCH; ++ch) {
#if CWR_RB_L2PF > 0
          prefetch_to(k, ch);
#endif
          mbar_wait_sleep(&empty[rg.st], rg.ph ^ 1);
          const uint32_t bytes = (uint32_t)(min(a.KC, a.G - ch * a.KC) * a.kslice_bytes);
          mbar_expect_tx(&full[rg.st], bytes);
          bulk_g2s(stg + rg.st * pc.stage_bytes, tb + a.u_bytes + ch * a.chunk_bytes, bytes, &full[rg.st]);
          rg.next(S);
        }
        RB_TRACE(k, 10);
        if (k + 2 < nk) load_union(k + 2);
        RB_TRACE(k, 11);
        if (k + 1 < nk) load_sector(k + 1);
        RB_TRACE(k, 12);
      }
    }
    return;
  }

  const bool is_main = warp < pc.ncw;
  // union gather of tile k into Q_u[k%2] by the epilogue threads (cp.async, completion
  // counted on qfull[k%2] by every epilogue thread)
  auto gather = [&](int k, int etid) {
    const int s = k % 3;
    mbar_wait(&ufull[s], (k / 3) & 1);
    const int32_t* uid = (const int32_t*)(ubuf + s * pc.ubuf_bytes);
    double* dst = Qu + (size_t)(k & 1) * a.Umax * VP;
    if (!EXP(a, 1)) {
      // element e = u·V + vv, e = etid, etid + EW, …: (u, vv) stepped without divisions
      int u = etid / V, vv = etid - (etid / V) * V;
      const int du = EW / V, dv = EW - du * V;
      for (int e = etid; e < a.Umax * V; e += EW) {
        cp_async8(dst + u * VP + vv, qptr(a, uid[u], vv));
        u += du;
        vv += dv;
        if (vv >= V) {
          vv -= V;
          ++u;
        }
      }
    }
    cp_async_mbar_arrive_noinc(&qfull[k & 1]);
  };

  if (is_main) {
    // -------------------------------------------------- main warps
    reg_main();
    const bool mainthr = tid < T * NG;
    const int ct = mainthr ? tid / NG : 0, g = mainthr ? tid % NG : 0;
    // offsets of this thread's B⁺ entries inside a row slot (chunk_elem, KIND_ROWBLK):
    // slots r < RB−1 hold all NG groups, the last one the first NF (a group without a
    // row there reads a neighbour's entry into an accumulator that is never written out)
    const int bfull = ct * NG + g, bpart = ct * NF + min(g, NF - 1);
    Ring rg;
    for (int k = 0; k < nk; ++k) {
      if (tid == 0) RB_TRACE(k, 0);
      mbar_wait(&qfull[k & 1], (k >> 1) & 1);  // Q_u[k%2] gathered
      mbar_wait(&ufull[k % 3], (k / 3) & 1);   // its position → union offsets
      if (tid == 0) RB_TRACE(k, 1);
      const double* Qb = Qu + (size_t)(k & 1) * a.Umax * VP;
      const uint16_t* ixb = (const uint16_t*)(ubuf + (k % 3) * pc.ubuf_bytes + a.off_idx);

      double acc[RB][V];
#pragma unroll
      for (int r = 0; r < RB; ++r)
#pragma unroll
        for (int v = 0; v < V; ++v) acc[r][v] = 0.0;
      // Main loop over position pairs, software-pipelined: the averages of pair pp+1
      // and the union offsets of pair pp+2 are loaded while pair pp's FMAs run; the
      // B⁺ entries of pair pp+1 are loaded as soon as its stage arrives, before pair
      // pp's stage is released.  Ping-pong registers (qa/qb, ba/bb).  A trailing odd
      // position (G odd) is peeled.
      static_assert(KC % 2 == 0, "row-block chunks hold whole position pairs");
      constexpr int PPS = KC / 2;  // position pairs per stage
      const int G = a.G, nfc = G / 2, npr = (G + 1) / 2;
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
        for (int kk = 0; kk < 2; ++kk)
#pragma unroll
          for (int r = 0; r < RB; ++r) b[kk][r] = Bs[(kk * R + r * NG) * T + (r < RB - 1 ? bfull : bpart)];
      };
      // B⁺Q on the raw averages; B⁺ΔQ = B⁺Q − rs·Q_i is formed in the epilogue with
      // the row sums rs of the sector record
      auto fma_pos = [&](const double (&q)[V], const double (&b)[RB]) {
        if (EXP(a, 2)) return;
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
#if CWR_RB_LOOK1
      // One-position lookahead (half the operand registers of the pair ping-pong, so
      // that RB = 4 rows × V = 9 accumulators fit): the averages and B⁺ entries of
      // position p+1 are loaded while position p's FMAs run.
      auto ldb1 = [&](const double* Bs, int kk, double (&b)[RB]) {
#pragma unroll
        for (int r = 0; r < RB; ++r) b[r] = Bs[(kk * R + r * NG) * T + (r < RB - 1 ? bfull : bpart)];
      };
      double q0[V], q1[V], b0[RB], b1[RB];
      uint32_t ipc = ix2[0], ipn = ix2[min(1, npr - 1) * T];
      mbar_wait(&full[rg.st], rg.ph);
      ldq(int(ipc & 0xffffu), q0);
      ldb1(stage_ptr(), 0, b0);
      for (int pp = 0; pp < npr; ++pp) {
        const int p = 2 * pp, kk = p % KC;
        if (p + 1 < G) {
          ldq(int(ipc >> 16), q1);
          ldb1(stage_ptr(), kk + 1, b1);
          fma_pos(q0, b0);
          if (p + 2 < G) {
            if ((p + 2) % KC == 0) {  // position p+2 opens the next stage
              Ring nr = rg;
              nr.next(S);
              mbar_wait(&full[nr.st], nr.ph);
              ldq(int(ipn & 0xffffu), q0);
              ldb1((const double*)(stg + nr.st * pc.stage_bytes), 0, b0);
              fma_pos(q1, b1);
              release();
            } else {
              ldq(int(ipn & 0xffffu), q0);
              ldb1(stage_ptr(), kk + 2, b0);
              fma_pos(q1, b1);
            }
            ipc = ipn;
            ipn = ix2[min(pp + 2, npr - 1) * T];
          } else {
            fma_pos(q1, b1);
            release();
          }
        } else {  // G odd: the last position alone
          fma_pos(q0, b0);
          release();
        }
      }
#else
      double qa[2][V], qb[2][V], ba[2][RB], bb[2][RB];
      ldq2(ix2[0], qa);
      uint32_t ipn = ix2[min(1, npr - 1) * T];
      mbar_wait(&full[rg.st], rg.ph);
      ldb(stage_ptr(), ba);
#if CWR_RB_PF
      // B⁺ of the next pair one position at a time, each right after the FMAs that free
      // its registers: position 0's entries are loaded while this pair's position 1 runs,
      // position 1's while the next pair's position 0 runs — every B⁺ load has a
      // position of FMAs in front of it (no extra registers at the peak)
      auto ldb1 = [&](const double* Bs, int kk, double (&b)[RB]) {
#pragma unroll
        for (int r = 0; r < RB; ++r) b[r] = Bs[(kk * R + r * NG) * T + (r < RB - 1 ? bfull : bpart)];
      };
      auto pair = [&](int pp, const double (&q)[2][V], const double (&b)[2][RB], double (&qn)[2][V],
                      double (&bn)[2][RB]) {
        ldq2(ipn, qn);
        ipn = ix2[min(pp + 2, npr - 1) * T];
        fma_pos(q[0], b[0]);
        const int nx = pp + 1;
        const bool more = nx < npr, nstage = more && nx % PPS == 0;
        const double* nb = stage_ptr() + (nx % PPS) * 2 * R * T;
        if (nstage) {  // next stage (a tail pair reads past kc into the stage: unused)
          Ring nr = rg;
          nr.next(S);
          mbar_wait(&full[nr.st], nr.ph);
          nb = (const double*)(stg + nr.st * pc.stage_bytes);
        }
        if (more) ldb1(nb, 0, bn[0]);
        fma_pos(q[1], b[1]);
        if (more) ldb1(nb, 1, bn[1]);
        if (!more || nstage) release();
      };
#else
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
#endif
      int pp = 0;
      constexpr bool kStatic = CWR_RB_STATIC < 0 ? R > 14 : CWR_RB_STATIC > 0;
      if constexpr (kStatic) {
        // whole stages while the successor pair exists: the first pair of a stage stays in
        // it, the second opens the next stage — no per-pair stage / end tests
        static_assert(PPS == 2, "static stage loop: 2 position pairs per stage");
        auto pair_in = [&](int pp, const double (&q)[2][V], const double (&b)[2][RB], double (&qn)[2][V],
                           double (&bn)[2][RB]) {
          ldq2(ipn, qn);
          ipn = ix2[(pp + 2) * T];
          fma_pos(q[0], b[0]);
          fma_pos(q[1], b[1]);
          ldb(stage_ptr() + 2 * R * T, bn);
        };
        auto pair_out = [&](int pp, const double (&q)[2][V], const double (&b)[2][RB], double (&qn)[2][V],
                            double (&bn)[2][RB]) {
          ldq2(ipn, qn);
          ipn = ix2[min(pp + 2, npr - 1) * T];
          fma_pos(q[0], b[0]);
          fma_pos(q[1], b[1]);
          Ring nr = rg;
          nr.next(S);
          mbar_wait(&full[nr.st], nr.ph);
          ldb((const double*)(stg + nr.st * pc.stage_bytes), bn);
          release();
        };
        for (; pp + 2 < npr && pp + 1 < nfc; pp += 2) {
          pair_in(pp, qa, ba, qb, bb);
          pair_out(pp + 1, qb, bb, qa, ba);
        }
      }
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
#endif
      // hand the p̂_opt rows to the epilogue warps: O[ct][v][1 + row], row l = r·NG + g
      if (tid == 0) RB_TRACE(k, 2);
      named_sync(RB_BAR_OFREE, NB);  // the epilogue of the previous tile is done with O
      if (tid == 0) RB_TRACE(k, 3);
      if (mainthr) {
        double* Oc = O + (size_t)ct * V * NM + 1 + g;
#pragma unroll
        for (int r = 0; r < RB; ++r)
          if (r < RB - 1 || g < NF)
#pragma unroll
            for (int v = 0; v < V; ++v) Oc[v * NM + r * NG] = acc[r][v];
      }
      named_arrive(RB_BAR_OFULL, NB);
    }
    return;
  }

  // -------------------------------------------------- epilogue warps
  reg_other();
  const int etid = tid - MW;
  if (nk > 0) gather(0, etid);
  if (nk > 1) gather(1, etid);
  if (nk > 0) named_arrive(RB_BAR_OFREE, NB);  // O starts free
  for (int k = 0; k < nk; ++k) {
    const int64_t tile = tile_of(k);
    named_sync(RB_BAR_OFULL, NB);  // p̂_opt rows of tile k are in O
    if (etid == 0) RB_TRACE(k, 4);
    mbar_wait(&sfull[k & 1], (k >> 1) & 1);
    if (etid == 0) RB_TRACE(k, 5);
    const double* Qb = Qu + (size_t)(k & 1) * a.Umax * VP;
    const uint16_t* ixb = (const uint16_t*)(ubuf + (k % 3) * pc.ubuf_bytes + a.off_idx);
    const unsigned char* sb0 = sbuf + (k & 1) * pc.sbuf_bytes;
    // one (cell, variable) item → its blended coefficients w (registers); two items per
    // thread are computed before either is stored, so their dependency chains interleave
    auto item_w = [&](int item, double (&w)[NM]) {
      const int c2 = item / V, v2 = item - (item / V) * V;
      const int j = c2 / a.TSC, cl = c2 - j * a.TSC;
      const unsigned char* sb = sb0 + j * a.sector_bytes;
      const double q2 = Qb[c2 * VP + v2];
      const double* row = O + (size_t)item * NM;
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
      cweno_epilogue<D, NM>(q2, accr, ps, valid, a, w, nullptr, nullptr);
    };
    auto item_store = [&](int item, const double (&w)[NM]) {
      if (a.dense_out) {
        double* row = O + (size_t)item * NM;
#pragma unroll
        for (int l = 0; l < NM; ++l) row[l] = w[l];
      } else {
        const int c2 = item / V, v2 = item - (item / V) * V;
        const int64_t c = tile * T + c2;
        if (c < a.n_owned) {
          double* o = a.out + c * a.ccs + v2 * a.cvs;
#pragma unroll
          for (int l = 0; l < NM; ++l) o[l] = w[l];
        }
      }
    };
    const int n_items = EXP(a, 16) ? 0 : T * V;  // flag 16: no epilogue
#if CWR_RB_PAIR
    for (int i0 = etid; i0 < n_items; i0 += 2 * EW) {
      const int i1 = i0 + EW < n_items ? i0 + EW : i0;
      double w0[NM], w1[NM];
      item_w(i0, w0);
      item_w(i1, w1);
      item_store(i0, w0);
      if (i1 != i0) item_store(i1, w1);
    }
#else
    for (int i0 = etid; i0 < n_items; i0 += EW) {
      double w0[NM];
      item_w(i0, w0);
      item_store(i0, w0);
    }
#endif
    named_sync(RB_BAR_EW, EW);  // every item of the tile is done; Q_u[k%2] no longer read
    if (etid == 0) RB_TRACE(k, 6);
    if (etid == 0 && a.dense_out) {
      fence_proxy_async();  // O rows → visible to the bulk store
      const int64_t nlive = min((int64_t)T, a.n_owned - tile * T);
      if (nlive > 0) bulk_s2g(a.out + tile * T * (int64_t)(V * NM), O, (uint32_t)(nlive * V * NM * 8));
    }
    if (k + 2 < nk) gather(k + 2, etid);  // Q_u[k%2] is free: main warps are past tile k
    if (etid == 0) RB_TRACE(k, 7);
    if (etid == 0) {
      if (a.dense_out) bulk_wait_read();  // O may be overwritten once the store has read it
      mbar_arrive(&sempty[k & 1]);
      mbar_arrive(&uempty[k % 3]);
    }
    if (etid == 0) RB_TRACE(k, 8);
    if (k + 1 < nk) named_arrive(RB_BAR_OFREE, NB);  // (completes only once etid 0 has arrived)
  }
  if (etid == 0) bulk_wait_all();
  cp_async_wait<0>();
}

// Instantiations per translation unit (rowblk_2d.cu, rowblk_3d.cu): full_tile = the
// layout kept the full tile (rb_tfull), else the runtime-T instantiation
template <int D, int M, int V>
PipeFn rowblk_fn_t(bool full_tile) {
  constexpr int TF = CWR_RB_TT ? rb_tfull(nmodes(M, D) - 1, V) : 0;
  return full_tile ? k_rowblk<D, M, V, TF> : k_rowblk<D, M, V, 0>;
}
template <int D, int M>
PipeFn rowblk_fn_v(int V, bool full_tile) {
  switch (V) {
    case 1: return rowblk_fn_t<D, M, 1>(full_tile);
    case 2: return rowblk_fn_t<D, M, 2>(full_tile);
    case 3: return rowblk_fn_t<D, M, 3>(full_tile);
    case 4: return rowblk_fn_t<D, M, 4>(full_tile);
    case 5: return rowblk_fn_t<D, M, 5>(full_tile);
    case 6: return rowblk_fn_t<D, M, 6>(full_tile);
    case 7: return rowblk_fn_t<D, M, 7>(full_tile);
    case 8: return rowblk_fn_t<D, M, 8>(full_tile);
    case 9: return rowblk_fn_t<D, M, 9>(full_tile);
    default: return nullptr;
  }
}

}  // namespace cwr
