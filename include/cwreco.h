/*
 * cwreco.h — C ABI of libcwreco: B200-native CWENO reconstruction on unstructured
 * triangular (d=2) / tetrahedral (d=3) meshes, arXiv 1612.09335 §2.1.
 *
 * Citations "P:L" are lines of the paper's LaTeX source; "R<n>" are the
 * readings listed in DESIGN.md.  Everything here is plain C: pointers, sizes and
 * status codes; no C++ or torch types cross the boundary.
 *
 * Operation (per owned cell i and conserved variable v, fp64):
 *   gather Q_j for the central stencil S_i^0 (n_e = d·ℳ cells) and
 *   the d+1 sectorial stencils S_i^s (d+1 cells each);
 *   p̂_opt = constrained-LSQ polynomial of degree M (Eq. CWENO:Popt),
 *   applied as p̂_opt[0] = Q_i/ψ_1, p̂_opt[1..ℳ-1] = B⁺ (Q_j − Q_i)_{j∈S_i^0∖i};
 *   p̂_s = linear interpolant on S_i^s (Eq. CWENO:Ps);
 *   P_0 = (P_opt − Σ_s λ̄_s P_s)/λ̄_0 (Eq. CWENO:P0);
 *   σ_s = p̂_sᵀ Σ p̂_s with the universal Σ;
 *   ω_s = (λ̄_s/(σ_s+ε)^r) / Σ_m (λ̄_m/(σ_m+ε)^r);
 *   w = Σ_s ω_s P_s, w[0] := Q_i/ψ_1 (R17).
 * Output: modal coefficients in the orthonormal Dubiner basis of the owner's
 * reference element (ordering R8).
 *
 * Conventions
 *   - Indices are 0-based.  After cwreco_set_mesh, cells are renumbered along a
 *     Morton space-filling curve ("SFC ids", R29); cwreco_get_permutation maps
 *     SFC id -> input id.
 *   - LOCAL numbering (what d_avgs / d_coeffs are indexed by): owned cells first
 *     (interior cells, whose stencils are fully owned, then boundary cells, each
 *     group in SFC order), then ghost cells ordered by (owner rank, SFC id).  With
 *     nranks == 1 local == SFC order and there are no ghosts.
 *   - Host arrays passed in are copied during the call and never retained.
 *     Device pointers (d_*) are owned by the caller; the library owns the mesh,
 *     stencils, per-cell matrix blocks and its scratch.
 *   - Calls that take a stream are asynchronous on it; kernel faults surface as
 *     CWRECO_ECUDA at a later call.  No exception crosses the ABI.  A context is
 *     not thread-safe.
 *   - Every call returns a status; on failure cwreco_last_error() describes it.
 *   - There is NO CPU fallback: a context created with cuda_device < 0 can do the
 *     host-side setup (mesh, stencils, matrices) but every compute call returns
 *     CWRECO_ECUDA.
 */
#ifndef CWRECO_H
#define CWRECO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cwreco_ctx cwreco_ctx;
typedef void* cwreco_stream; /* a cudaStream_t (NULL = legacy default stream) */

typedef enum {
  CWRECO_OK = 0,
  CWRECO_EINVAL = 1,      /* bad argument (NULL pointer, negative size, bad stride) */
  CWRECO_ENOMEM = 2,      /* host or device allocation failed */
  CWRECO_ECUDA = 3,       /* CUDA runtime error, or no device for a compute call */
  CWRECO_EMESH = 4,       /* invalid mesh: repeated vertex, duplicate cell,
                             non-manifold face, zero-volume cell */
  CWRECO_ESTENCIL = 5,    /* central stencil exhausted (component has < n_e cells) */
  CWRECO_ESINGULAR = 6,   /* rank-deficient central least-squares system */
  CWRECO_ESTATE = 7,      /* call out of order (e.g. reconstruct before precompute) */
  CWRECO_EUNSUPPORTED = 8, /* (d, M, V) outside the compiled range */
  CWRECO_ENCCL = 9         /* NCCL could not be loaded, or an NCCL call failed */
} cwreco_status;

/* Linear weights and WENO parameters.  Defaults: lambda0 = 1e5,
 * lambda_s = 1, eps = 1e-14, r = 4.  The λ are normalised per cell over the
 * valid stencils before use (R5, R14). */
typedef struct {
  double lambda0;
  double lambda_s;
  double eps;
  int r;
} cwreco_params;

/* Kernel variant for cwreco_reconstruct. */
enum {
  CWRECO_KERNEL_PIPELINED = 0, /* default: TMA-bulk pipelined streaming kernel */
  CWRECO_KERNEL_SIMPLE = 1,    /* one thread per (cell, variable), plain loads */
  CWRECO_KERNEL_MATRIXFREE = 2 /* no precomputed matrices: each pass assembles and solves
                                  every cell's least-squares systems from the geometry
                                  (moving meshes); needs cwreco_prepare_matrixfree */
};

/* Which owned cells a cwreco_reconstruct call processes (for halo overlap). */
enum {
  CWRECO_PART_ALL = 0,
  CWRECO_PART_INTERIOR = 1, /* tiles made only of interior cells: needs no ghost data */
  CWRECO_PART_BOUNDARY = 2  /* the remaining tiles: run after the ghost exchange */
};

/* Sizes and layout facts of a context (valid after cwreco_precompute). */
typedef struct {
  int32_t dim, degree_M, nvars, n_modes; /* ℳ(M,d) = (1/d!) Π (M+l) */
  int32_t n_e;                           /* d·ℳ */
  int32_t gather_len;                    /* gather positions per cell: max((d+1)·d, n_e − 1 +
                                            extra sector cells outside S_i^0) */
  int32_t tile_cells;                    /* cells per tile of the packed matrix stream */
  int32_t chunk_k;                       /* stencil columns per streamed chunk */
  int64_t n_cells;                       /* global cells */
  int64_t n_owned, n_ghost, n_interior;
  int64_t n_tiles, n_interior_tiles;
  int64_t tile_bytes;                    /* packed bytes per tile */
  int64_t device_bytes;                  /* device memory held by the context */
  int64_t algorithmic_bytes_per_cell;    /* SURVEY §8(d) B_cell */
  int64_t n_invalid_sectors;             /* sectors flagged invalid (R14) */
  int64_t n_extra_gather;                /* sector cells outside S_i^0 (R15) */
  int64_t union_max;                     /* largest per-tile stencil union (cells whose
                                            averages a tile gathers once into shared memory) */
  int32_t kernel_family;                 /* layout of the packed stream after precompute:
                                            0 = cell-variable (k_pipelined),
                                            1 = row-block (k_rowblk); -1 before */
  int32_t reserved_;
  int64_t n_boundary_ghosts;             /* mirror cells (R37) referenced by the owned stencils */
} cwreco_info;

/* ---------------------------------------------------------------- lifecycle */
/* dim ∈ {2,3}; degree_M ∈ [1,4] (d=2) or [1,3] (d=3); 1 ≤ nvars ≤ 16.
 * params may be NULL (defaults).  cuda_device < 0: host-only context.
 * *out receives the context (NULL on failure). */
cwreco_status cwreco_create(int dim, int degree_M, int nvars, const cwreco_params* params,
                            int cuda_device, cwreco_ctx** out);
void cwreco_destroy(cwreco_ctx* ctx);
/* Message of the last failing call on this thread (never NULL). */
const char* cwreco_last_error(void);
const char* cwreco_version(void);
cwreco_status cwreco_get_info(const cwreco_ctx* ctx, cwreco_info* out);
/* CWRECO_KERNEL_* */
cwreco_status cwreco_set_kernel(cwreco_ctx* ctx, int variant);

/* Launch / layout options (cwreco_set_option).  None changes any result: every
 * family and grid size computes the same operations in the same order (tested
 * bitwise).
 *   CWRECO_OPT_FAMILY    packed-stream layout and kernel family chosen by the next
 *                        cwreco_precompute: -1 = default per shape (row-block where
 *                        ℳ = 20 and nvars ≥ 7, else cell-variable), 0 = cell-variable
 *                        (k_pipelined), 1 = row-block (k_rowblk, where instantiated).
 *                        Setting it drops the packed matrices (ESTATE until the next
 *                        cwreco_precompute).
 *   CWRECO_OPT_MAX_CTAS  upper bound on the CTAs of the persistent reconstruction
 *                        kernels (0 = one wave over every SM, the default).  A small
 *                        bound makes each CTA walk many tiles (tests of the multi-tile
 *                        pipeline) or leaves SMs free for concurrent work.
 *   CWRECO_OPT_MAX_TILE  upper bound on the cells per tile of the packed layout chosen by
 *                        the next cwreco_precompute (0 = the largest tile that fits, the
 *                        default; rounded down to even, ≥ 2).  A smaller tile runs the
 *                        kernels' runtime-tile-size instantiations (tests) and trades
 *                        stage-ring depth for tile width.  Setting it drops the packed
 *                        matrices (ESTATE until the next cwreco_precompute).
 * EINVAL for an unknown option or a value out of range. */
enum { CWRECO_OPT_FAMILY = 1, CWRECO_OPT_MAX_CTAS = 2, CWRECO_OPT_MAX_TILE = 3 };
cwreco_status cwreco_set_option(cwreco_ctx* ctx, int option, int64_t value);

/* ---------------------------------------------------------------- mesh / setup */
/* xyz: [n_nodes][dim] fp64; cell_nodes: [n_cells][dim+1] int64 (any orientation);
 * period: [dim] box lengths of a periodic box, or NULL for an open domain
 * (coordinates of a periodic box must lie in [0, period)).  Validates (EMESH),
 * unwraps periodic images (R16), fixes orientation (R28), computes barycentres
 * and the Morton order (R29), builds face and node adjacency. */
cwreco_status cwreco_set_mesh(cwreco_ctx* ctx, int64_t n_nodes, const double* xyz, int64_t n_cells,
                              const int64_t* cell_nodes, const double* period);
/* Physical boundaries of an OPEN mesh by reflected ghost cells (R37; the paper is
 * silent on boundary stencils): side_bc [2·dim], side s = 2·axis + (0 low,
 * 1 high) of the nodes' bounding box: 0 none (stencils grow inward, sectors may
 * starve), 1 transmissive, 2 wall.  Stencil searches cross every boundary face that
 * lies exactly on an active side into the mirror image of the domain across it
 * (ghost id N + s·N + k = cell k mirrored, vertices X'_a = c + (c − X_a)); ghosts
 * enter through face adjacency only (the R14 node-neighbour fallback stays on real
 * cells) and are never reflected twice.  A ghost's averages are its source's, with
 * ρu_axis (index mom0 + axis, mom0 ≥ 0) negated on wall sides; the library fills
 * them before every pass.  Call after cwreco_set_mesh, before the stencils (drops
 * them); one rank only (EUNSUPPORTED at cwreco_build_stencils otherwise); not with
 * the matrix-free mode.  EINVAL for a periodic mesh, codes outside 0..2 or a mom0
 * that leaves no room for dim momenta.  side_bc == NULL clears the boundaries. */
cwreco_status cwreco_set_boundary(cwreco_ctx* ctx, const int* side_bc, int mom0);
/* sfc_to_input: [n_cells] out. */
cwreco_status cwreco_get_permutation(const cwreco_ctx* ctx, int64_t* sfc_to_input);
/* Ownership: rank owns SFC ids [floor(r·N/P), floor((r+1)·N/P)) (contiguous Morton
 * ranges).  Optional; default rank 0 of 1.  Must precede cwreco_build_stencils.
 * id: NULL (no transport: the caller moves ghost data itself with cwreco_halo_plan /
 * cwreco_set_send_lists / cwreco_halo_pack), or 128 bytes from
 *   cwreco_nccl_unique_id   (one process per rank; every rank passes the SAME bytes,
 *                            made by one rank and broadcast by the caller): the
 *                            context creates an NCCL communicator over the ranks
 *                            (ncclCommInitRank — COLLECTIVE, blocks until all ranks
 *                            join; needs a CUDA device; ENCCL if libnccl cannot be
 *                            loaded or fails), or
 *   cwreco_loopback_unique_id (all ranks in ONE process, one host thread per rank,
 *                            each with its own context): peer transfers are device
 *                            copies (tests on one GPU; the plan exchange also works
 *                            host-only).
 * With a transport, cwreco_build_stencils / cwreco_set_stencils become collective:
 * after the stencils every rank sends each owner the ids of the ghosts it needs and
 * installs what it must send (the send lists), so cwreco_halo_exchange and
 * cwreco_reconstruct_overlap need no further setup.  Re-partitioning destroys the
 * previous transport.  EINVAL for a bad rank / nranks / unknown loopback id. */
cwreco_status cwreco_set_partition(cwreco_ctx* ctx, int rank, int nranks, const uint8_t* id);
/* id[128] ← a fresh NCCL unique id (ncclGetUniqueId) for cwreco_set_partition;
 * ENCCL if libnccl.so.2 cannot be loaded. */
cwreco_status cwreco_nccl_unique_id(uint8_t* id);
/* id[128] ← a fresh in-process loopback group of nranks ranks for cwreco_set_partition. */
cwreco_status cwreco_loopback_unique_id(int nranks, uint8_t* id);
/* Central and sectorial stencils of every owned cell (R11-R15),
 * exact geometric predicates; then ghosts and the local numbering. */
cwreco_status cwreco_build_stencils(cwreco_ctx* ctx);
/* Stencils of the owned cells in LOCAL order, entries as global SFC ids:
 * central [n_owned][n_e] (self first), sectors [n_owned][dim+1][dim+1] (self first,
 * -1 padded when starved), sector_valid [n_owned][dim+1] (0/1).  Any may be NULL. */
cwreco_status cwreco_get_stencils(const cwreco_ctx* ctx, int32_t* central, int32_t* sectors,
                                  uint8_t* sector_valid);
/* Upload external stencils instead of cwreco_build_stencils (S:194-211 interface):
 * OWNED cells in SFC order (row q = SFC id own_lo + q), global SFC ids:
 *   central [n_own][n_e]         the cell itself first, n_e distinct cells;
 *   sectors [n_own][dim+1][dim+1] sector s of the cell: itself first, then dim
 *                                 distinct members (ignored if not valid);
 *   valid   [n_own][dim+1]        1 = sector usable, 0 = invalid (ω_s = 0, R14).
 * Arrays are copied.  EINVAL on a malformed stencil, ESTATE without a mesh.
 * (cwreco_get_stencils returns LOCAL order; cwreco_get_local_cells maps it.) */
cwreco_status cwreco_set_stencils(cwreco_ctx* ctx, const int32_t* central, const int32_t* sectors,
                                  const uint8_t* valid);
/* local_to_global: [n_owned + n_ghost] SFC ids of the local cells. */
cwreco_status cwreco_get_local_cells(const cwreco_ctx* ctx, int64_t* local_to_global);
/* Per-cell matrices (B⁺ by Householder QR of the reduced LSQ system, sector
 * inverses), packed into tiles and uploaded to the device (host-only context:
 * kept on the host).  ESINGULAR if a central system is rank deficient. */
cwreco_status cwreco_precompute(cwreco_ctx* ctx);
/* The universal oscillation matrix Σ [ℳ][ℳ] as used by the kernels. */
cwreco_status cwreco_get_sigma(const cwreco_ctx* ctx, double* out);
/* Export the packed matrices of selected owned cells (local ids) for tests.
 * gather [n][gather_len]: local ids in gather order — positions s·dim+m hold
 * member m of sector s (fillers from S_i^0 or the cell itself when the sector is
 * invalid), then the remaining cells of S_i^0, then the cell itself as padding;
 * bplus [n][ℳ-1][gather_len]: the reduced pseudo-inverse B⁺ with its columns in
 * gather order (zero for positions outside S_i^0), so p̂_opt[1..] = B⁺ (Q_g − Q_i);
 * sinv [n][dim+1][dim][dim]; slots [n][dim+1][dim]: gather position of each
 * sector member, 255 = invalid sector.  Any output may be NULL. */
cwreco_status cwreco_get_blocks(const cwreco_ctx* ctx, int64_t n_sel, const int64_t* cells,
                                double* bplus, double* sinv, int32_t* gather, uint8_t* slots);

/* Matrix-free mode: upload the local geometry, the stencils
 * (as local ids with periodic image codes), the basis in monomial form and the
 * quadrature rule to the device, for cwreco_set_kernel(CWRECO_KERNEL_MATRIXFREE).
 * Needs cwreco_build_stencils (or cwreco_set_stencils); cwreco_precompute is not
 * needed.  The pass then builds A and solves the constrained LSQ
 * and the sector systems per cell on the GPU.  ECUDA
 * without a device; EUNSUPPORTED for M > 3 or nvars > 9. */
cwreco_status cwreco_prepare_matrixfree(cwreco_ctx* ctx);

/* ---------------------------------------------------------------- multi-rank halo */
/* Lower-level pieces of the exchange, for callers that move the bytes themselves
 * (no transport id): recv_counts [nranks]: ghosts owned by each rank; recv_ids [n_ghost]: their SFC
 * ids in local ghost order (grouped by owner rank, ascending id). */
cwreco_status cwreco_halo_plan(const cwreco_ctx* ctx, int64_t* recv_counts, int64_t* recv_ids);
/* Install what this rank sends: send_counts [nranks], send_ids [Σ counts] = SFC ids
 * of OWNED cells requested by each peer (peer order, each ascending).  EINVAL if an
 * id is not owned. */
cwreco_status cwreco_set_send_lists(cwreco_ctx* ctx, const int64_t* send_counts, const int64_t* send_ids);
cwreco_status cwreco_send_total(const cwreco_ctx* ctx, int64_t* total);
/* The installed send lists (by cwreco_set_send_lists or the transport's plan
 * exchange): send_counts [nranks], send_ids [send_total] as SFC ids, peer order.
 * Either may be NULL. */
cwreco_status cwreco_get_send_lists(const cwreco_ctx* ctx, int64_t* send_counts, int64_t* send_ids);
/* Pack the requested owned rows of d_avgs into d_sendbuf [send_total][nvars]
 * (contiguous, peer order) on `stream`.  The caller moves d_sendbuf to the peers'
 * ghost rows (e.g. NCCL all-to-all-v) before CWRECO_PART_BOUNDARY. */
cwreco_status cwreco_halo_pack(cwreco_ctx* ctx, const double* d_avgs, int64_t a_cell_stride,
                               int64_t a_var_stride, double* d_sendbuf, cwreco_stream stream);

/* The second exchange of the scheme (reconstruction polynomials after
 * the pass): pack `width` contiguous doubles of each requested owned row of d_rows
 * (row stride in doubles; e.g. the coefficients [n_local][nvars][ℳ] with width =
 * row_stride = nvars·ℳ) into d_sendbuf [send_total][width], peer order — the same
 * send lists as the averages.  The caller moves the buffer into the peers' ghost
 * rows (rows n_owned.. of their [n_local][width] array). */
cwreco_status cwreco_halo_pack_rows(cwreco_ctx* ctx, const double* d_rows, int64_t row_stride, int width,
                                    double* d_sendbuf, cwreco_stream stream);

/* ---------------------------------------------------------------- hot path */
/* d_avgs: cell averages of the LOCAL cells, element (c, v) at
 *   d_avgs[c·a_cell_stride + v·a_var_stride]  (n_owned + n_ghost rows);
 * d_coeffs: output for the owned cells, coefficient l of (c, v) at
 *   d_coeffs[c·c_cell_stride + v·c_var_stride + l], l < ℳ.
 * Strides are in elements (doubles); the fast path wants c_var_stride == ℳ and
 * c_cell_stride == nvars·ℳ (dense) and 16-byte aligned pointers; other strides
 * use per-thread stores.  part: CWRECO_PART_*.  Asynchronous on `stream`. */
cwreco_status cwreco_reconstruct(cwreco_ctx* ctx, const double* d_avgs, int64_t a_cell_stride,
                                 int64_t a_var_stride, double* d_coeffs, int64_t c_cell_stride,
                                 int64_t c_var_stride, int part, cwreco_stream stream);
/* The first exchange of the scheme ("exchange of the cell averages
 * before the reconstruction"): fill the ghost rows n_owned.. of d_avgs (strides as
 * cwreco_reconstruct) with the owners' averages, through the transport of
 * cwreco_set_partition: on the library's comm stream, after the work already on
 * `stream`, pack (one kernel) → NCCL send/recv per peer (or loopback copies) into
 * the ghost rows (directly when d_avgs is dense [n_local][nvars], else staged and
 * scattered by a kernel); `stream` then waits for it.  Asynchronous.  nranks == 1:
 * no-op.  ESTATE without a transport; ECUDA without a device.  Every rank must make
 * the same sequence of exchange calls. */
cwreco_status cwreco_halo_exchange(cwreco_ctx* ctx, double* d_avgs, int64_t a_cell_stride, int64_t a_var_stride,
                                   cwreco_stream stream);
/* The second exchange (the reconstruction polynomials after the pass):
 * rows of `width` contiguous doubles, row stride row_stride (e.g. the coefficients
 * [n_local][nvars][ℳ]: width = row_stride = nvars·ℳ); ghost rows n_owned.. are
 * filled from the owners' rows.  As cwreco_halo_exchange otherwise. */
cwreco_status cwreco_halo_exchange_rows(cwreco_ctx* ctx, double* d_rows, int64_t row_stride, int width,
                                        cwreco_stream stream);
/* One overlapped multi-rank pass (SURVEY §8(b) overlap_halo): the exchange of
 * cwreco_halo_exchange on the comm stream, the INTERIOR tiles (stencils fully owned,
 * no ghost reads) on `stream` concurrently, then — after the exchange event — the
 * BOUNDARY tiles.  Writes the ghost rows of d_avgs and all owned rows of d_coeffs;
 * results are bitwise those of a single-rank pass.  nranks == 1: a plain
 * cwreco_reconstruct.  Errors as cwreco_reconstruct / cwreco_halo_exchange. */
cwreco_status cwreco_reconstruct_overlap(cwreco_ctx* ctx, double* d_avgs, int64_t a_cell_stride,
                                         int64_t a_var_stride, double* d_coeffs, int64_t c_cell_stride,
                                         int64_t c_var_stride, cwreco_stream stream);
/* End-to-end pass on HOST buffers (the whole hot path behind one call):
 *   h_avgs   [n_owned + n_ghost][nvars] dense row-major, local order (ghost rows
 *            already filled by the caller when nranks > 1);
 *   h_coeffs [n_owned][nvars][ℳ] dense, written before the call returns.
 * The library copies h_avgs into its own device buffers (allocated on first use,
 * kept until cwreco_destroy), reconstructs in n_pieces consecutive tile ranges on
 * `stream`, and copies each range's coefficients back on an internal copy stream as
 * soon as that range is done, so the device→host transfer overlaps the remaining
 * ranges.  Page-locked host buffers (cudaHostAlloc / cudaHostRegister, torch
 * pin_memory) give asynchronous copies; pageable buffers work but serialise.
 * (cells, in matrix-free mode).  n_pieces ≤ 0 selects the default (4).  Synchronous: returns after h_coeffs is
 * complete.  Errors as cwreco_reconstruct; ENOMEM if the device buffers cannot be
 * allocated. */
cwreco_status cwreco_reconstruct_host(cwreco_ctx* ctx, const double* h_avgs, double* h_coeffs, int n_pieces,
                                      cwreco_stream stream);

/* ---------------------------------------------------------------- face traces (NEXT-3) */
/* Face quadrature used by cwreco_face_traces: *nq points; lam [nq][dim]
 * barycentric weights over the face's dim vertices SORTED BY ASCENDING GLOBAL NODE ID
 * (so both cells of a face use the same physical points in the same order);
 * weights [nq] sum to 1 (multiply by the face measure for integrals).  Exact for
 * polynomials of degree 2M+1 on the face.  lam / weights may be NULL. */
cwreco_status cwreco_face_rule(const cwreco_ctx* ctx, int* nq, double* lam, double* weights);
/* nbr [n_owned][dim+1]: local id of the cell across face f (the face opposite local
 * vertex f of the orientation-fixed cell), −1 on an open boundary.  Face neighbours
 * are always local (they belong to the central stencil).  ESTATE before stencils. */
cwreco_status cwreco_face_neighbors(const cwreco_ctx* ctx, int64_t* nbr);
/* d_traces [n_owned][dim+1][nq][nvars] (dense) ← the blended polynomial w of each owned
 * cell (d_coeffs as written by cwreco_reconstruct, strides in doubles) at its faces'
 * quadrature points.  Asynchronous on `stream`; tables built on the first call. */
cwreco_status cwreco_face_traces(cwreco_ctx* ctx, const double* d_coeffs, int64_t c_cell_stride,
                                 int64_t c_var_stride, double* d_traces, cwreco_stream stream);

/* ---------------------------------------------------------------- space-time predictor (NEXT-2) */
/* The element-local space-time Galerkin predictor of the ADER scheme (paper §2.2,
 * P:235-320), Eulerian (fixed mesh), compressible Euler equations (nvars = dim + 2:
 * ρ, ρu_1..ρu_dim, E; p = (γ−1)(E − ½ρ|u|²)).  Per owned cell the
 * reconstruction polynomial w is evolved into a space-time polynomial of degree M,
 * q_h = Σ_l θ_l(ξ, τ) q̂_l on T_E × [0,1] (τ = (t − tⁿ)/Δt), with nodal basis θ_l on
 * the uniform lattice of the (dim+1)-simplex (R32), by the Picard iteration of Eq.
 * CGfinal with the test functions of the unknown τ > 0 nodes (R33), the
 * nodal flux interpolant of Eq. PDEterm (R34), from q̂_l = w(ξ_l), until
 * max|Δq̂| ≤ 1e-12·max(1, max|q̂⁰|) or 2(M+1) iterations (R35).  No neighbour data.
 *
 * Setup (after the stencils: local numbering): the universal space-time matrices
 * (K_τ, M of Eq. cgPDE, by quadrature) to the constant bank, the owned cells'
 * inverse Jacobians to the device.  gamma > 1 (1.4: P:754).  ESTATE before the
 * stencils; EUNSUPPORTED unless nvars = dim + 2 and M ≤ 3; ECUDA host-only. */
cwreco_status cwreco_predictor_setup(cwreco_ctx* ctx, double gamma);
/* *n_nodes = 𝓛 = ℳ(M, dim+1), *n_known = ℳ(M, dim) (the τ = 0 nodes, first);
 * nodes [𝓛][dim+1] (may be NULL): (ξ_1..ξ_dim, τ) of each node in output order
 * (known nodes first, then by τ level, then by the lattice tuple). */
cwreco_status cwreco_predictor_nodes(const cwreco_ctx* ctx, int* n_nodes, int* n_known, double* nodes);
/* d_coeffs: the reconstruction of the owned cells, (c, v, l) at
 * d_coeffs[c·c_cell_stride + v·c_var_stride + l] (cwreco_reconstruct's output);
 * dt ≥ 0 the time step; d_qhat [n_owned][𝓛][nvars] dense ← the nodal space-time
 * degrees of freedom; d_iters [n_owned] (may be NULL) ← Picard iterations per cell,
 * or −(iterations + 1) if the cell did not converge or met ρ ≤ 0 / p ≤ 0 at a node.
 * Asynchronous on `stream`.  ESTATE before cwreco_predictor_setup. */
cwreco_status cwreco_predict(cwreco_ctx* ctx, const double* d_coeffs, int64_t c_cell_stride, int64_t c_var_stride,
                             double dt, double* d_qhat, int32_t* d_iters, cwreco_stream stream);

/* Debug tap (tests): intermediates of n_sel owned cells (local ids), computed by
 * the SIMPLE kernel and copied to host (synchronises `stream`):
 *   popt [n][nvars][ℳ], psec [n][dim+1][nvars][dim+1], sigma [n][dim+2][nvars],
 *   omega [n][dim+2][nvars], w [n][nvars][ℳ].  Any output may be NULL. */
cwreco_status cwreco_reconstruct_debug(cwreco_ctx* ctx, const double* d_avgs, int64_t a_cell_stride,
                                       int64_t a_var_stride, int64_t n_sel, const int64_t* cells,
                                       double* popt, double* psec, double* sigma, double* omega,
                                       double* w, cwreco_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* CWRECO_H */
