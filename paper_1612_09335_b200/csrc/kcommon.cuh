// Device code shared by the sm_100a kernels of libcwreco (kernels.cu, rowblk_*.cu):
// kernel arguments, the fused CWENO epilogue, the sector products
// and the PTX helpers of the TMA / mbarrier pipelines.  Each
// translation unit gets its own copy of the constant-bank Σ (static), uploaded by
// its own upload function.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "devguard.cuh"
#include "internal.hpp"

namespace cwr {

__host__ __device__ constexpr int nmodes(int M, int d) {
  return d == 2 ? (M + 1) * (M + 2) / 2 : (M + 1) * (M + 2) * (M + 3) / 6;
}

// Universal Σ depends only on (d, M): the packed upper triangle of Σ[1:,1:]
// (off-diagonals doubled) of every supported (d, M) lives in the constant bank, so
// the σ quadratic forms use it as DFMA constant operands.
__host__ __device__ constexpr int sig_len(int D, int M) { return (nmodes(M, D) - 1) * nmodes(M, D) / 2; }
__host__ __device__ constexpr int sig_off(int D, int M) {
  int off = 0;
  for (int dd = 2; dd <= 3; ++dd)
    for (int mm = 1; mm <= 4; ++mm) {
      if (dd == D && mm == M) return off;
      off += sig_len(dd, mm);
    }
  return off;
}
constexpr int SIG_TOTAL = sig_off(4, 1);
static __constant__ double c_sig[SIG_TOTAL];


struct KArgs {
  const unsigned char* blocks;
  int64_t tile_bytes, u_bytes, off_idx, idx_bytes, ids_bytes, chunk_bytes, kslice_bytes, off_sector, sinv_bytes,
      sector_bytes;
  int Umax;
  int T, G, K, KC, NCH, V, VP, kind, NSC, TSC, srec;
  int64_t n_owned, tile_begin, tile_end;
  const double* Q;
  int64_t acs, avs;
  int64_t n_local;     // local ids ≥ n_local are boundary ghosts (R37): rows of Qbc [n_bc][V]
  const double* Qbc;
  double* out;
  int64_t ccs, cvs;
  int dense_out;
  int exp_flags;  // bottleneck experiments only (CWRECO_EXP_FLAGS, read only by a library built
                 // with -DCWRECO_EXPERIMENTS): 1 no gather, 2 no B⁺ FMAs, 16 no epilogue
                 // (timing only: results are wrong).  The product build compiles these
                 // branches out (EXP() is constant false).
  double eps, psi1;
  int r;
  // normalised linear weights (R5, R14) indexed by the number of valid sectors
  double l0[5], inv_l0[5], ls[5];
};

#ifdef CWRECO_EXPERIMENTS
#define EXP(a, bit) (((a).exp_flags & (bit)) != 0)
#else
#define EXP(a, bit) false
#endif

// address of the average (local cell j, variable v): caller rows, or a boundary ghost row
__device__ __forceinline__ const double* qptr(const KArgs& a, int64_t j, int v) {
  return j < a.n_local ? a.Q + j * a.acs + v * a.avs : a.Qbc + (j - a.n_local) * a.V + v;
}

struct DbgOut {
  double *popt, *psec, *sigma, *omega, *w;
  const int64_t* cells;
  int64_t n;
};

__device__ __forceinline__ double powr(double t, int r) {
  if (r == 4) {
    const double t2 = __dmul_rn(t, t);
    return __dmul_rn(t2, t2);
  }
  double p = 1.0;
  for (int i = 0; i < r; ++i) p = __dmul_rn(p, t);
  return p;
}

template <int D, int NM>
struct ModeOf {  // M from (D, ℳ)
  static constexpr int M = D == 2 ? (NM == 3 ? 1 : NM == 6 ? 2 : NM == 10 ? 3 : 4) : (NM == 4 ? 1 : NM == 10 ? 2 : 3);
};

// Fused epilogue.  acc[l-1] = p̂_opt[l] (l >= 1); ps[s][l-1] = p̂_s[l]
// (l = 1..D).  The blended coefficients are written to w[0..NM) as they are formed
// (w may be shared or global memory).
template <int D, int NM>
__device__ __forceinline__ void cweno_epilogue(double qi, double* acc, const double (&ps)[D + 1][D],
                                               const bool (&valid)[D + 1], const KArgs& a, double* w,
                                               double* sigma_out, double* omega_out) {
  constexpr int R = NM - 1;
  constexpr int SO = sig_off(D, ModeOf<D, NM>::M);
  const double p0 = qi / a.psi1;
  int nval = 0;
#pragma unroll
  for (int s = 0; s <= D; ++s) nval += valid[s] ? 1 : 0;
  const double l0 = a.l0[nval], il0 = a.inv_l0[nval], ls = a.ls[nval];
  // P0 = (P_opt − Σ_s λ̄_s P_s)/λ̄0 is kept unscaled: acc := λ̄0·P0 (only the
  // first d modes change; modes above d are P_opt), and the factor 1/λ̄0 goes into σ_0
  // (× 1/λ̄0²) and into the blend weight (ω0/λ̄0) — ℳ−1 fewer multiplications
#pragma unroll
  for (int l = 0; l < D; ++l) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q <= D; ++q) s = __dadd_rn(s, valid[q] ? ps[q][l] : 0.0);
    acc[l] = __fma_rn(-ls, s, acc[l]);
  }
  // σ_0 = P0ᵀ Σ P0 and σ_s = P_sᵀ Σ P_s; explicit roundings (here and in
  // every kernel) so that all kernels perform the same operations bit for bit
  double sg0 = 0.0;
  {
    int idx = SO;
#pragma unroll
    for (int l = 0; l < R; ++l) {
      double t = 0.0;
#pragma unroll
      for (int m = l; m < R; ++m) t = __fma_rn(c_sig[idx + m - l], acc[m], t);
      idx += R - l;
      sg0 = __fma_rn(acc[l], t, sg0);
    }
  }
  double sgs[D + 1];
#pragma unroll
  for (int s = 0; s <= D; ++s) {
    double v = 0.0;
    int idx = SO;
#pragma unroll
    for (int l = 0; l < D; ++l) {
      double t = 0.0;
#pragma unroll
      for (int m = l; m < D; ++m) t = __fma_rn(c_sig[idx + m - l], ps[s][m], t);
      idx += R - l;
      v = __fma_rn(ps[s][l], t, v);
    }
    sgs[s] = v;
  }
  // ω̃_s = λ̄_s/(σ_s+ε)^r, ω_s = ω̃_s/Σ ω̃; invalid sectors get 0 (R14)
  // reciprocals instead of divisions (one extra rounding, far inside the 1e-11 bar)
  sg0 = __dmul_rn(sg0, __dmul_rn(il0, il0));  // σ_0 of P0 = σ(λ̄0·P0)/λ̄0²
  const double wt0 = __dmul_rn(l0, __drcp_rn(powr(__dadd_rn(sg0, a.eps), a.r)));
  double wts[D + 1];
  double sum = wt0;
#pragma unroll
  for (int s = 0; s <= D; ++s) {
    wts[s] = valid[s] ? __dmul_rn(ls, __drcp_rn(powr(__dadd_rn(sgs[s], a.eps), a.r))) : 0.0;
    sum = __dadd_rn(sum, wts[s]);
  }
  const double isum = __drcp_rn(sum);
  const double om0 = __dmul_rn(wt0, isum);
  double oms[D + 1];
#pragma unroll
  for (int s = 0; s <= D; ++s) oms[s] = __dmul_rn(wts[s], isum);
  // w = Σ_s ω_s P_s;  w[0] := Q_i/ψ1 (R17)
  w[0] = p0;
  const double om0s = __dmul_rn(om0, il0);  // ω0 · P0 = (ω0/λ̄0) · acc
#pragma unroll
  for (int l = 0; l < D; ++l) {
    double v = __dmul_rn(om0s, acc[l]);
#pragma unroll
    for (int s = 0; s <= D; ++s) v = __fma_rn(oms[s], ps[s][l], v);
    w[l + 1] = v;
  }
#pragma unroll
  for (int l = D; l < R; ++l) w[l + 1] = __dmul_rn(om0s, acc[l]);
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

template <int D>
__device__ __forceinline__ void sector_apply(const double* sinv, const double (&dqs)[(D + 1) * D],
                                             double (&ps)[D + 1][D]) {
#pragma unroll
  for (int s = 0; s <= D; ++s)
#pragma unroll
    for (int l = 0; l < D; ++l) {
      double t = 0.0;
#pragma unroll
      for (int m = 0; m < D; ++m) t = __fma_rn(sinv[(s * D + l) * D + m], dqs[s * D + m], t);
      ps[s][l] = t;
    }
}

// ---------------------------------------------------------------- PTX helpers
// fp64 tensor-core MMA, D = A·B + D with A 8×4 (row), B 4×8 (col): lane L holds
// A[L/4][L%4], B[L%4][L/4] and D[L/4][2(L%4) + {0, 1}]
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
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
// Blocking wait with a long suspend-time hint: the waiting thread sleeps until the
// phase completes instead of re-polling (used by the producer lane, whose spin
// otherwise steals issue slots from the consumers on its SM sub-partition).
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
        : "memory");
  }
}
// Non-blocking probe of a phase (result consumed later, so its latency overlaps work).
__device__ __forceinline__ uint32_t mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return done;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// L2 prefetch of a contiguous global range (bulk; bytes a multiple of 16): no shared
// memory, no completion — a later bulk copy of the range then hits L2
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
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
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

struct PipeCfg {
  int stages;
  int64_t stage_bytes, q_bytes, out_bytes;
  int64_t off_stage, off_q, off_out, off_bar, smem;
  int ncw;  // consumer warps (k_rowblk: main warps)
  // k_rowblk only: epilogue warps, union / sector chunk buffers
  int eww;
  int64_t off_ubuf, off_sbuf, ubuf_bytes, sbuf_bytes;
};

using PipeFn = void (*)(KArgs, PipeCfg);

// row-block kernels (rowblk_2d.cu, rowblk_3d.cu): nullptr if (M, V) is not instantiated
PipeFn rowblk_fn_2d(int M, int V, bool full_tile);
PipeFn rowblk_fn_3d(int M, int V, bool full_tile);
cudaError_t rowblk_upload_sigma_2d(const double* packed, size_t bytes, size_t offset);
cudaError_t rowblk_upload_sigma_3d(const double* packed, size_t bytes, size_t offset);

struct Ring {  // slot index + mbarrier phase of a ring of S slots
  int st = 0;
  uint32_t ph = 0;
  __device__ __forceinline__ void next(int S) {
    if (++st == S) {
      st = 0;
      ph ^= 1u;
    }
  }
};

__device__ __forceinline__ void consumer_bar(int nthreads) {  // named barrier 1: consumer warps only
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

}  // namespace cwr
