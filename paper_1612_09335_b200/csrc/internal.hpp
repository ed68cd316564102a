// Internal declarations of libcwreco (not part of the ABI; see include/cwreco.h).
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "cwreco.h"

namespace cwr {

// Error carrying a status code; converted to cwreco_status at the ABI boundary.
struct Error : std::runtime_error {
  cwreco_status code;
  Error(cwreco_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(cwreco_status c, const std::string& m) { throw Error(c, m); }

inline int n_modes(int M, int d) {  // ℳ(M,d) = (1/d!) Π_{l=1..d} (M+l)
  long num = 1, den = 1;
  for (int l = 1; l <= d; ++l) { num *= (M + l); den *= l; }
  return int(num / den);
}

// Layout of one packed tile of the matrix stream: the
// tile's T cells are streamed as a union chunk, NCH position chunks and a sector
// chunk, each a contiguous 16-byte-aligned block (one 1-D bulk copy):
//   union chunk: uid int32  [Umax]    local ids of every cell the tile's stencils touch:
//                                     the tile's own T cells first, then the others
//                                     ascending (padded to Umax entries)
//                idx uint16 [G][T]    (at off_idx) union index × VP of the cell gathered
//                                     at each position: positions [0, (d+1)d) hold
//                                     sector s, member m at s·d+m (R15; fillers if the
//                                     sector is invalid), then the rest of S_i^0, then
//                                     the cell itself as padding
//   chunk ch, positions p ∈ [ch·KC, ch·KC+kc) (kc = KC except a shorter last one):
//     B     double  reduced pseudo-inverse columns in gather order (0 for positions
//                   outside S_i^0), in the family's layout (chunk_elem below)
//   sector chunk (at off_sector), in NSC pieces of TSC cells (stride sector_bytes; one
//   piece unless a whole sector chunk would outgrow a stage, ROWBLK only), each:
//     sinv  double [T][d+1][d][d]  sector inverses
//     vmask uint8  [T]             bit s = sector s valid (R14)
#if defined(__CUDACC__)
#define CWR_HD __host__ __device__
#else
#define CWR_HD
#endif

// Kernel families, each with its own B⁺ chunk layout:
//  KIND_CELLVAR  one consumer thread per (cell, variable) (k_pipelined): position
//                pairs first, [kc/2][R][T][2], then an odd last position as [R][T]
//  KIND_ROWBLK   one consumer thread per (cell, row group) holding every variable
//                (k_rowblk): the R reduced rows are dealt round-robin to NG groups,
//                row l = r·NG + g (slot r of group g); the first nfull groups hold RB
//                rows, the others RB−1.  A position slice is [r][ct][g] over the row
//                slots r < RB, slot r holding the ngr(r) groups that have a row
//                there, so the lanes (ct, g) of a warp read consecutive doubles.
enum { KIND_CELLVAR = 0, KIND_ROWBLK = 1 };
// NG for ℳ = 20: 4 groups of ≤ 5 rows (20 slots for 19 rows) on 4 main warps that take
// 200 registers each through setmaxnreg (k_rowblk); the B⁺ loads per FMA stay, the
// average loads per FMA drop to 4/7 of the 7-group shape (C4-shape proxy under the
// power cap: 0.719 vs 0.667; 7 groups of ≤ 3 rows was the 168-register design)
#ifndef CWR_RB_NG20
#define CWR_RB_NG20 4
#endif
#ifndef CWR_RB_NG10
#define CWR_RB_NG10 2  // ℳ = 10 (R = 9 rows): 2 groups of ≤ 5 rows (C3 shape 0.783 vs 0.724 for 3 × 3)
#endif
CWR_HD constexpr int rb_ng(int R, int V) { return (void)V, R > 14 ? CWR_RB_NG20 : CWR_RB_NG10; }
CWR_HD constexpr int rb_rb(int R, int V) { return (R + rb_ng(R, V) - 1) / rb_ng(R, V); }
CWR_HD constexpr int rb_nfull(int R, int V) { return R - (rb_rb(R, V) - 1) * rb_ng(R, V); }
CWR_HD constexpr int rb_ngr(int R, int V, int r) { return r < rb_rb(R, V) - 1 ? rb_ng(R, V) : rb_nfull(R, V); }

// Entry (position p, cell ct) of the union-offset table (uint16, in the union chunk):
// CELLVAR [G][T]; ROWBLK position pairs interleaved, [⌈G/2⌉][T][2], so one 32-bit load
// gives a cell the offsets of both positions of a chunk.
CWR_HD inline int64_t idx_elem(int kind, int T, int p, int ct) {
  if (kind == KIND_ROWBLK) return (int64_t(p >> 1) * T + ct) * 2 + (p & 1);
  return int64_t(p) * T + ct;
}

// Element (row l, cell ct, position kk) of a B⁺ chunk holding kc positions.
CWR_HD inline int64_t chunk_elem(int kind, int kc, int R, int V, int T, int l, int ct, int kk) {
  if (kind == KIND_ROWBLK) {
    const int NG = rb_ng(R, V), r = l / NG, g = l % NG;
    return (int64_t(kk) * R + r * NG) * T + int64_t(ct) * rb_ngr(R, V, r) + g;
  }
  const int np = kc / 2;
  if (kk < 2 * np) return ((int64_t(kk / 2) * R + l) * T + ct) * 2 + (kk & 1);
  return int64_t(np) * R * T * 2 + int64_t(l) * T + ct;
}

// Byte offsets (from the tile start) of cell ct's sector record (srec doubles: the
// sector inverses, then for ROWBLK the B⁺ row sums) and validity byte.
CWR_HD inline int64_t sector_sinv_off(int64_t off_sector, int64_t sector_bytes, int TSC, int srec, int ct) {
  const int j = ct / TSC;
  return off_sector + j * sector_bytes + int64_t(ct - j * TSC) * srec * 8;
}
CWR_HD inline int64_t sector_mask_off(int64_t off_sector, int64_t sector_bytes, int64_t sinv_bytes, int TSC, int ct) {
  const int j = ct / TSC;
  return off_sector + j * sector_bytes + sinv_bytes + (ct - j * TSC);
}

struct Layout {
  int d = 0, M = 0, V = 0, nm = 0, R = 0, K = 0, G = 0, T = 0, KC = 0, NCH = 0, Umax = 0;
  int kind = KIND_CELLVAR;   // kernel family (chunk layout)
  int VP = 0;                // row stride of the gathered averages Q_u (V, rounded up to even for ROWBLK)
  int64_t kslice_bytes = 0;  // T·R·8: one position of B⁺ for the whole tile
  int64_t off_idx = 0;       // r16(Umax·4): the idx table inside the union chunk
  int64_t idx_bytes = 0;     // r16(G·T·2) (ROWBLK: G rounded up to even)
  int64_t u_bytes = 0;       // off_idx + idx_bytes: the union chunk
  int64_t ids_bytes = 0;     // 0 (position chunks hold only B⁺)
  int64_t chunk_bytes = 0;   // stride of full chunks: KC·kslice_bytes
  int64_t sinv_bytes = 0, sector_bytes = 0, off_sector = 0, tile_bytes = 0;
  int NSC = 1, TSC = 0;      // sector pieces per tile, cells per piece
  int srec = 0;              // doubles per cell in a sector piece: sector inverses (d+1)·d²,
                             // then (ROWBLK) the row sums rs[R] of B⁺
  int kc_of(int ch) const { return KC < G - ch * KC ? KC : G - ch * KC; }
  int64_t off_chunk(int ch) const { return u_bytes + int64_t(ch) * chunk_bytes; }
  int64_t chunk_size(int ch) const { return ids_bytes + int64_t(kc_of(ch)) * kslice_bytes; }
};

// Pipelined-kernel shape (kernels.cu), shared with make_layout's chunk choice.
constexpr int kMinStages = 4;             // stage ring depth floor
inline int cons_threads(int nm) { return nm >= 20 ? 320 : 160; }  // consumer threads per CTA
inline int ctas_per_sm(int nm) { return nm >= 20 ? 1 : 2; }
inline int64_t round128(int64_t x) { return (x + 127) & ~int64_t(127); }
// shared memory of one pipelined CTA: S stages + the consumers' private gather rings
inline int64_t pipe_stage_bytes(const Layout& L) {
  int64_t m = L.chunk_bytes > L.sector_bytes ? L.chunk_bytes : L.sector_bytes;  // (one sector piece)
  return round128(m > L.u_bytes ? m : L.u_bytes);
}
inline int64_t pipe_q_bytes(const Layout& L) {  // double-buffered Q_u [Umax][V] and idx [G][T]
  return round128(2 * int64_t(L.Umax) * L.VP * 8) + round128(2 * L.idx_bytes);
}
inline int64_t pipe_out_bytes(const Layout& L) {
  if (L.kind == KIND_ROWBLK) return round128(int64_t(L.T) * L.V * L.nm * 8);  // the tile's [T][V][ℳ] rows
  return round128(int64_t((L.T * L.V + 31) / 32) * 32 * L.nm * 8);           // per-warp staging
}
inline int64_t pipe_smem(const Layout& L, int stages) {
  return stages * pipe_stage_bytes(L) + pipe_q_bytes(L) + pipe_out_bytes(L) + 16 * stages;
}
constexpr int kMaxStages = 8;  // deeper rings measured no faster (tools/sweep.py); the rest is L1
inline int64_t pipe_budget(int nm, int max_smem) {
  return ctas_per_sm(nm) == 1 ? max_smem : (max_smem + 1024) / ctas_per_sm(nm) - 1024;
}

// max_smem: opt-in shared memory per block of the device (227 KB on B200);
// umax_for(T): the largest per-tile stencil union for tiles of T cells.
// max_tile (CWRECO_OPT_MAX_TILE): upper bound on the cells per tile (0: none).
Layout make_layout(int d, int M, int V, int G, int max_smem, const std::function<int(int)>& umax_for,
                   int family = -1, int max_tile = 0);
// k_rowblk (warp-specialised, rowblk.cuh): a CTA of kRbThreads threads = main warps
// (T = kRbMainThreads / NG cells × NG row groups, rounded up to whole warps), kRbEW
// epilogue warps and one producer warp; one CTA per SM.
// ℳ = 20: 4 main warps (T = 32 cells × 4 row groups, 200 registers by setmaxnreg) + 7
// epilogue warps (C4-shape proxy under the power cap: 0.719; the 168-register shapes
// 7 main / 4 epilogue 0.667, 4 main / 3 epilogue at 8 warps 0.698, 5 / 6 0.648, 4 / 2
// 0.539: the epilogue needs the warps); ℳ = 10 (3 groups of 3 rows): 6 main
// warps (T = 64) + 5 epilogue warps (C3 data: 0.708; 224/4 0.636, 96/8 0.632)
#ifndef CWR_RB_MAIN
#define CWR_RB_MAIN 128
#endif
#ifndef CWR_RB_EW
#define CWR_RB_EW 7
#endif
#ifndef CWR_RB_MAINREG20
#define CWR_RB_MAINREG20 200  // main-warp registers for ℳ = 20 (0: no setmaxnreg)
#endif
#ifndef CWR_RB_MAIN10
#define CWR_RB_MAIN10 128  // ℳ = 10: main threads (T = CWR_RB_MAIN10 / NG cells; was 192 / 3)
#endif
#ifndef CWR_RB_EW10
#define CWR_RB_EW10 7  // ℳ = 10: epilogue warps (was 5)
#endif
CWR_HD constexpr int rb_main(int R, int V) { return (void)V, R > 14 ? CWR_RB_MAIN : CWR_RB_MAIN10; }
CWR_HD constexpr int rb_ew(int R, int V) { return (void)V, R > 14 ? CWR_RB_EW : CWR_RB_EW10; }
CWR_HD constexpr int rb_main_warps(int T, int NG) { return (T * NG + 31) / 32; }
// the full row-block tile: main threads / row groups, even (T·R·8 a multiple of 16 bytes)
CWR_HD constexpr int rb_tfull(int R, int V) { return (rb_main(R, V) / rb_ng(R, V)) & ~1; }
// threads of a row-block CTA (main + epilogue + producer warp): the kernel's launch bound
CWR_HD constexpr int rb_threads(int R, int V) { return 32 * ((rb_main(R, V) + 31) / 32 + rb_ew(R, V) + 1); }
// setmaxnreg split (3 warp groups of 128 threads launched at 168 registers): the main
// group's increase must be covered by what the two others release, else it waits forever
CWR_HD constexpr int rb_mainreg(int R, int V) { return (void)V, R > 14 ? CWR_RB_MAINREG20 : 0; }
CWR_HD constexpr int rb_otherreg(int R, int V) { return ((168 * 3 - rb_mainreg(R, V)) / 2) & ~7; }
static_assert(CWR_RB_MAINREG20 == 0 || CWR_RB_MAINREG20 - 168 <= 2 * (168 - ((168 * 3 - CWR_RB_MAINREG20) / 2 & ~7)),
              "setmaxnreg increase not covered by the released registers");
// default family choice (tools/gpu_families.sh proxies, then the configs): the
// warp-specialised row-block kernel for ℳ = 20 (3-D M = 3: V = 9 0.75 vs 0.60, V = 5 1.00
// vs 0.81 of the copy peak on the proxy; C5 0.904 vs 0.775); the cell-variable kernel for
// 2-D ℳ = 10 (C2 0.847 vs 0.69) and the small shapes; 3-D M = 2 on the row-block kernel with
// 6 main / 5 epilogue warps (C3 data 0.708 vs 0.640)
CWR_HD constexpr bool rb_default(int d, int R, int V) { return (R > 14 && V >= 3) || (d == 3 && R == 9 && V >= 5); }
#ifndef CWR_RB_KC
#define CWR_RB_KC 4
#endif
constexpr int kRbKC = CWR_RB_KC;  // positions per streamed chunk of the row-block layout (2 pairs)
constexpr int kRbMaxStages = 32;  // row-block stage ring: as deep as shared memory allows
// row-block ring floor: 2 stages of KC positions before the tile is halved.  The ring
// depth barely matters to the row-block kernel (C4 proxy: 3 stages 0.722, 7 stages of
// half the size 0.710), halving T does (a partitioned C4 rank whose boundary tiles
// raise the union maximum from 371 to 399 cells lost the 4th stage and fell to T = 16:
// 1.48x the time per cell, tools/rank_projection.py)
constexpr int kRbMinStages = 2;
// shared memory of a row-block CTA with S ring stages: ring (position chunks),
// 3 union-chunk buffers, 2 sector-chunk buffers, Q_u[2][Umax][VP], O[T][V][ℳ], barriers
inline int64_t rb_ubuf_bytes(const Layout& L) { return round128(L.u_bytes); }
inline int64_t rb_sbuf_bytes(const Layout& L) { return round128(int64_t(L.NSC) * L.sector_bytes); }
inline int64_t rb_smem(const Layout& L, int S) {
  return int64_t(S) * round128(L.chunk_bytes) + 3 * rb_ubuf_bytes(L) + 2 * rb_sbuf_bytes(L) +
         round128(2 * int64_t(L.Umax) * L.VP * 8) + round128(int64_t(L.T) * L.V * L.nm * 8) + 8 * (2 * S + 12);
}
bool rowblk_supported(int d, int M, int V);
// CTAs per SM (≤ max_ctas, by shared memory) and stage-ring depth of a ROWBLK
// layout (0 CTAs: does not fit)
void rowblk_plan(const Layout& L, int max_smem, int max_ctas, int& ctas, int& stages);

struct DeviceState;  // kernels.cu

// Host arrays of the matrix-free mode (precompute.cpp: matfree_prepare)
struct MatfreeHost {
  std::vector<double> X, B;          // local cells: vertices [n_local][d+1][d], barycentres [n_local][d]
  std::vector<int32_t> st;           // [n_owned][n_e−1] central stencil members (local ids, self excluded)
  std::vector<uint8_t> sh;           // [n_owned][n_e−1] periodic image codes
  std::vector<int32_t> sec;          // [n_owned][d+1][d] sector members (local ids, −1 if invalid)
  std::vector<uint8_t> secsh;        // [n_owned][d+1][d]
  std::vector<uint8_t> vmask;        // [n_owned] bit s = sector s valid (stencil level)
  std::vector<int> mexp;             // monomial exponents [nmono][3]
  std::vector<double> mcoef;         // basis in monomial form [ℳ][nmono]
  std::vector<double> qp, qw;        // quadrature rule on T_E (exact for degree M)
};

}  // namespace cwr

struct cwreco_ctx {
  int d = 0, M = 0, V = 0, nm = 0, ne = 0;
  cwreco_params prm{1e5, 1.0, 1e-14, 4};
  int device = -1;
  int kernel = CWRECO_KERNEL_PIPELINED;
  int family = -1;       // CWRECO_OPT_FAMILY (-1: default per shape)
  int64_t max_ctas = 0;  // CWRECO_OPT_MAX_CTAS (0: every SM)
  int64_t max_tile = 0;  // CWRECO_OPT_MAX_TILE (0: the largest tile that fits)

  // ---- mesh, SFC order (set_mesh)
  bool has_mesh = false;
  int64_t N = 0, Nn = 0;
  bool periodic = false;
  double L[3] = {0, 0, 0};
  std::vector<int64_t> perm;        // sfc -> input id
  std::vector<int64_t> cell_nodes;  // [N][d+1], orientation fixed
  std::vector<double> X;            // [N][d+1][d] unwrapped vertex coordinates
  std::vector<double> bary;         // [N][d] IEEE barycentres (R29)
  std::vector<int64_t> nbr;         // [N][d+1] face neighbours, -1 none
  std::vector<int64_t> nc_ptr, nc_idx;  // node -> cells (SFC ids, ascending)

  double box_lo[3] = {0, 0, 0}, box_hi[3] = {0, 0, 0};  // bounding box of the nodes

  // ---- boundary ghost cells by reflection (R37, cwreco_set_boundary; open meshes)
  bool has_bc = false;
  int bc[6] = {0, 0, 0, 0, 0, 0};  // per box side s = 2·axis + (0 low, 1 high): 0 none, 1 transmissive, 2 wall
  int mom0 = -1;                   // index of ρu_1 among the variables (wall sides negate ρu_axis)
  std::vector<int64_t> bc_ids;     // ghost ids N + s·N + k referenced by owned stencils, ascending

  // ---- partition
  int rank = 0, nranks = 1;
  int64_t own_lo = 0, own_hi = 0;

  // ---- stencils (build_stencils), owned cells in SFC order (index = sfc - own_lo)
  bool has_stencils = false;
  std::vector<int32_t> central;  // [n_own][ne] global SFC ids
  std::vector<int32_t> sectors;  // [n_own][d+1][d+1] global, -1 padded
  std::vector<uint8_t> valid;    // [n_own][d+1]

  // ---- local numbering
  int64_t n_owned = 0, n_ghost = 0, n_interior = 0;
  std::vector<int64_t> local2global;   // [n_owned + n_ghost]
  std::vector<int64_t> ghost_counts;   // [nranks]
  std::vector<int64_t> send_counts;    // [nranks]
  std::vector<int64_t> send_local;     // local ids of owned cells to send
  int G = 0;                           // gather length
  int64_t n_extra = 0, n_invalid = 0;

  // ---- packed blocks
  bool has_blocks = false;
  cwr::Layout lay;
  int64_t n_tiles = 0, n_int_tiles = 0;
  std::vector<unsigned char> host_blocks;  // kept only for host-only contexts
  std::vector<double> sigma;               // ℳ×ℳ universal Σ
  double psi1 = 0;                         // constant basis function value

  cwr::DeviceState* dev = nullptr;
  void* mf = nullptr;  // matrix-free device state (matfree.cu), after cwreco_prepare_matrixfree
  void* tr = nullptr;  // face-trace tables (traces.cu), built on the first cwreco_face_traces
  void* halo = nullptr;  // multi-rank transport (halo.cu), after cwreco_set_partition with an id
  void* pred = nullptr;  // space-time predictor tables (predictor.cu), after cwreco_predictor_setup
};

namespace cwr {
// mesh.cpp
void set_mesh(cwreco_ctx* c, int64_t n_nodes, const double* xyz, int64_t n_cells,
              const int64_t* cells, const double* period);
// stencil.cpp
void build_stencils(cwreco_ctx* c);
void finalize_stencils(cwreco_ctx* c);  // local numbering etc. of c->central/sectors/valid
// basis.cpp
void basis_eval(int d, int M, const double* xi, double* out);  // ψ_l(ξ), l < ℳ
std::vector<double> sigma_matrix(int d, int M);                  // Σ by quadrature
void basis_monomials(int d, int M, std::vector<int>& exps, std::vector<double>& coef);
void gauss_legendre01(int n, std::vector<double>& x, std::vector<double>& w);
void gauss_jacobi01(int n, double alpha, std::vector<double>& t, std::vector<double>& w);
// precompute.cpp
void precompute(cwreco_ctx* c);
void simplex_rule(int d, int M, std::vector<double>& qp, std::vector<double>& qw);
void matfree_prepare(cwreco_ctx* c, MatfreeHost& h);
// matfree.cu
void dev_matfree_upload(cwreco_ctx* c, const MatfreeHost& h);
void dev_matfree_reconstruct(cwreco_ctx* c, const double* avgs, int64_t acs, int64_t avs, double* coeffs,
                             int64_t ccs, int64_t cvs, int64_t cell_begin, int64_t cell_end, void* stream);
void dev_matfree_destroy(cwreco_ctx* c);
// basis.cpp / traces.cu: face quadrature and face traces (NEXT-3)
void face_rule(int d, int M, std::vector<double>& lam, std::vector<double>& w);
void dev_face_traces(cwreco_ctx* c, const double* coeffs, int64_t ccs, int64_t cvs, double* traces, void* stream);
void dev_traces_destroy(cwreco_ctx* c);
// predictor.cpp / predictor.cu: the local space-time Galerkin predictor (NEXT-2)
struct PredictorHost {
  int L = 0, nk = 0;                 // space-time nodes, known (τ = 0) nodes
  std::vector<double> nodes;         // [L][d+1]
  std::vector<double> A, C0, Phi;    // [d][L−nk][L], [L−nk][nk], [L][nk]
};
void st_nodes(int d, int M, std::vector<std::vector<int>>& nodes);
void predictor_matrices(int d, int M, PredictorHost& h);
void predictor_jinv(const cwreco_ctx* c, std::vector<double>& jinv);
void dev_predictor_setup(cwreco_ctx* c, const PredictorHost& h, const std::vector<double>& jinv, double gamma);
void dev_predictor_destroy(cwreco_ctx* c);
void dev_predict(cwreco_ctx* c, const double* w, int64_t ccs, int64_t cvs, double dt, double* q, int32_t* iters,
                 void* stream);
// stencil.cpp: real and boundary-ghost cells (R37): vertices, barycentre, face neighbours
const double* cell_X(const cwreco_ctx* c, int64_t j, double* buf);  // [d+1][d]; buf ≥ 12 doubles
void cell_bary(const cwreco_ctx* c, int64_t j, double* out);
int cell_neighbours(const cwreco_ctx* c, int64_t j, int64_t* out);  // out ≥ d+1 entries; returns count
// stencil.cpp: send lists (owned cells requested by each peer, SFC ids) → local ids
void install_send_lists(cwreco_ctx* c, const int64_t* send_counts, const int64_t* send_ids);
// halo.cu: multi-rank transport (NCCL or in-process loopback) and the exchange
void halo_unique_id_nccl(uint8_t* id);
void halo_unique_id_loopback(int nranks, uint8_t* id);
void halo_set_transport(cwreco_ctx* c, const uint8_t* id);  // id == nullptr: none
bool halo_has_transport(const cwreco_ctx* c);
void halo_plan_exchange(cwreco_ctx* c);                       // collective, after the stencils
void halo_exchange(cwreco_ctx* c, double* rows, int64_t rs, int64_t es, int width, void* stream);
void halo_reconstruct_overlap(cwreco_ctx* c, double* avgs, int64_t acs, int64_t avs, double* coeffs, int64_t ccs,
                              int64_t cvs, void* stream);
void halo_destroy(cwreco_ctx* c);
// kernels.cu (device side; all return cudaError_t as int)
void dev_create(cwreco_ctx* c);
void dev_destroy(cwreco_ctx* c);
void dev_alloc_blocks(cwreco_ctx* c, int64_t bytes);
void dev_upload_blocks(cwreco_ctx* c, int64_t offset, const unsigned char* host, int64_t bytes);
void dev_upload_aux(cwreco_ctx* c);
void dev_download_tile(const cwreco_ctx* c, int64_t tile, unsigned char* host);
void dev_reconstruct(cwreco_ctx* c, const double* avgs, int64_t acs, int64_t avs, double* coeffs,
                     int64_t ccs, int64_t cvs, int part, void* stream);
void dev_reconstruct_host(cwreco_ctx* c, const double* h_avgs, double* h_coeffs, int n_pieces, void* stream);
void dev_debug(cwreco_ctx* c, const double* avgs, int64_t acs, int64_t avs, int64_t n_sel,
               const int64_t* cells, double* popt, double* psec, double* sigma, double* omega,
               double* w, void* stream);
void dev_halo_pack(cwreco_ctx* c, const double* avgs, int64_t acs, int64_t avs, double* sendbuf,
                   void* stream);
void dev_halo_pack_rows(cwreco_ctx* c, const double* rows, int64_t row_stride, int64_t elem_stride, int width,
                        double* sendbuf, void* stream);
int64_t dev_bytes(const cwreco_ctx* c);
int dev_max_smem(const cwreco_ctx* c);
void dev_set_send(cwreco_ctx* c);
}  // namespace cwr
