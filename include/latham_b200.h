/* include/latham_b200.h — C-ABI drop-in boundary of the B200-native core-Hamiltonian path.
 *
 * The reference (arXiv 1408.3839 C++ reference, "latham") has no plugin or FFI
 * layer: its boundary is the free-function C++ API under
 * proj/core/include/latham/ headers. Each entry point below replaces one of those
 * functions (cited file:line); include/latham_b200.hpp wraps them back into the
 * reference's C++ call shapes. Plain pointers and sizes only; no exceptions cross
 * the ABI; every function returns an lt_status whose message is lt_last_error().
 *
 * Layout conventions
 *   - matrices are column-major (Eigen's default storage, as in the reference);
 *   - an m0 x m0 block is stored column-major: entry (mu, nu) at mu + nu*m0;
 *   - k-points are lexicographic, lin = (k1*L2 + k2)*L3 + k3 (spectrum.hpp:27-29),
 *     eigenvalues ascending within each k-point;
 *   - periodic generating blocks are listed in std::map order of their kidx
 *     (block_circulant.hpp:47 iteration order).
 *
 * All heavy work runs on the GPU bound to the context; the host only does O(M0+m0)
 * integer planning (window starts, grid extents) between stages.
 */
#ifndef LATHAM_B200_H
#define LATHAM_B200_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error classes of latham/errors.hpp:10-43 */
typedef enum lt_status {
    LT_OK = 0,
    LT_EDIM = 1,      /* DimensionError    */
    LT_EBOUNDS = 2,   /* BoundsError       */
    LT_ESTRUCT = 3,   /* StructureError    */
    LT_EDEFINITE = 4, /* DefinitenessError (message names the k-point) */
    LT_ECAP = 5,      /* ResourceCapError  */
    LT_EGENERIC = 6,  /* latham::Error     */
    LT_ECUDA = 7      /* device / driver failure (no reference counterpart) */
} lt_status;

/* LatticeSystem (galerkin.hpp:17-35) + NucleiSet (newton_kernel.hpp:12-28) +
 * GtoBasis (gto_basis.hpp:12-29), with per-direction n / nbar (the reference's
 * scalar n is n[0]=n[1]=n[2]). Coordinates are cell-centred in [-b/2, b/2]. */
typedef struct lt_system {
    double b;
    int64_t L[3];
    int64_t n[3];
    int64_t nbar[3];
    int64_t quad_M;
    double eps_ov;
    int64_t n_nuclei;
    const double* nuc_pos;    /* [n_nuclei][3] */
    const double* nuc_charge; /* [n_nuclei]    */
    int64_t m0;
    const double* bf_center;  /* [m0][3] */
    const double* bf_alpha;   /* [m0]    */
    const int32_t* bf_deg;    /* [m0][3] */
} lt_system;

typedef enum lt_kind { LT_LAPLACE = 0, LT_MASS = 1, LT_NUCLEAR = 2 } lt_kind; /* galerkin.hpp:37 */

typedef struct lt_ctx lt_ctx;           /* device, stream, solver handle, cached buffers */
typedef struct lt_operator lt_operator; /* AssembledOperator (galerkin.hpp:43-54), device-resident */
typedef struct lt_sysdev lt_sysdev;     /* a system description uploaded to the device */

/* ---- context ---------------------------------------------------------------- */
lt_status lt_create(int device, lt_ctx** out);
void lt_destroy(lt_ctx* ctx);
const char* lt_last_error(void);
/* stream the context launches on (cudaStream_t as void*); 0 until created */
void* lt_stream(lt_ctx* ctx);
/* stream ordering for callers that own device buffers on their own stream (cudaStream_t as
   void*): lt_stream_wait — work the context enqueues after this call waits for everything
   enqueued on `stream` so far; lt_stream_join — `stream` waits for everything the context
   enqueued so far. Device-pointer entry points (lt_*_dev) write caller buffers on the
   context stream, so a caller brackets them with wait / join. */
lt_status lt_stream_wait(lt_ctx* ctx, void* stream);
lt_status lt_stream_join(lt_ctx* ctx, void* stream);
/* number of kernels this context launched so far (for the bench's gpu_launches) */
int64_t lt_launch_count(lt_ctx* ctx);
/* per-kernel CUDA-event timing on the context stream (off by default; resets totals) */
lt_status lt_set_stage_timing(lt_ctx* ctx, int on);
/* diagnostics (off by default): phase events between graph launches (accumulated into the
   stage totals as phase_l0/phase_gap/phase_post) and host-side timestamps (printed to stderr
   by lt_destroy) */
#define LT_DIAG_PHASE_TIMING 1
#define LT_DIAG_HOST_TIMING 2
lt_status lt_set_diagnostics(lt_ctx* ctx, int flags);
int64_t lt_stage_count(lt_ctx* ctx);
lt_status lt_stage_get(lt_ctx* ctx, int64_t idx, char* name, int64_t cap, double* ms, int64_t* launches);
/* per-launch timeline of the last timed solve: stream 0 main, 1-2 side branches; ms from solve start */
int64_t lt_stage_timeline_count(lt_ctx* ctx);
lt_status lt_stage_timeline_get(lt_ctx* ctx, int64_t idx, char* name, int64_t cap, int* stream, double* t0,
                                double* t1);

/* ---- whole path: LatticeSystem -> eigenvalues ------------------------------- *
 * Replaces assemble_core (tools/commands.cpp:51-59: H = combine(0.5, Laplace,
 * -1.0, Nuclear), S = Mass) followed by solve_periodic (eigensolver.cpp:124-141)
 * or solve_box_dense (eigensolver.cpp:12-35, eigenvalues only, cap 4096).
 * eig: periodic -> [L1*L2*L3][m0] ascending per k; box -> [N_b] ascending.
 * info (optional, 8 int64): L0, band[3], R_tot, N_b, k_count, 0. */
lt_status lt_solve_core(lt_ctx* ctx, const lt_system* sys, int periodic, double* eig_host, int64_t* info);

/* Same path with the system already resident on the device and eigenvalues left on
 * the device (eig_dev: device pointer). k-points may be sharded: this call solves
 * the pencils of k in [k_begin, k_end) only (k_end < 0: all) and writes them at
 * eig_dev + k_begin*m0. Box systems ignore the range. */
lt_status lt_sys_upload(lt_ctx* ctx, const lt_system* sys, lt_sysdev** out);
void lt_sys_free(lt_sysdev* s);
lt_status lt_solve_core_dev(lt_ctx* ctx, const lt_sysdev* sys, int periodic, double* eig_dev, int64_t k_begin,
                            int64_t k_end, int64_t* info);
/* lt_solve_core_dev ordered against a caller stream in one call (= lt_stream_wait(stream),
 * lt_solve_core_dev, lt_stream_join(stream)): the low-latency form for callers that own a
 * stream (a framework's current stream). */
lt_status lt_solve_core_dev_on(lt_ctx* ctx, const lt_sysdev* sys, int periodic, double* eig_dev, int64_t k_begin,
                               int64_t k_end, int64_t* info, void* stream);

/* ---- several GPUs of one process (parallel.hpp:15-32) ------------------ *
 * lt_mctx: one lt_ctx per listed device and an in-process NCCL communicator over them
 * (ncclCommInitAll; NCCL is loaded at creation). lt_solve_core_multi = lt_solve_core on
 * all devices:
 *   LT_SPLIT_KPOINTS   every device assembles H, S and solves its contiguous k-range
 *                      (eigensolver.cpp:95-120); one ncclAllGather of the eigenvalues;
 *   LT_SPLIT_RANKTERMS device q assembles the nuclear rank terms of its range
 *                      (galerkin.cpp:275-283) into a partial H (device 0 adds 0.5 Laplace),
 *                      one ncclAllReduce (sum) completes H; then the k-range solves and the
 *                      all-gather. Box systems: device 0 solves the dense pencil.
 * Eigenvalues land on the host in the single-device order (identical values for the
 * k-point split). lt_multi_ctx(m, i) exposes device i's context for the other entries. */
typedef struct lt_mctx lt_mctx;
#define LT_SPLIT_KPOINTS 0
#define LT_SPLIT_RANKTERMS 1
lt_status lt_create_multi(const int* devices, int ndev, lt_mctx** out);
void lt_destroy_multi(lt_mctx* m);
int lt_multi_ndev(const lt_mctx* m);
lt_ctx* lt_multi_ctx(lt_mctx* m, int i);
lt_status lt_solve_core_multi(lt_mctx* m, const lt_system* sys, int periodic, int split, double* eig_host,
                              int64_t* info);

/* ---- multi-GPU: assembly sharded by rank terms ---------------------- *
 * The nuclear operator is a rank-R_tot sum (galerkin.cpp:275-283: sum_r w_r prod_l T_l);
 * a shard assembles the terms r in [r_begin, r_end) (r_end < 0: all) and, with_kinetic != 0,
 * 0.5 Laplace, so the shards' H sum to H = 0.5 Laplace - Nuclear (one all-reduce); S = Mass
 * is complete on every shard. Buffers are device pointers of lt_core_layout's size:
 * periodic -> [nblocks][m0*m0] generating blocks in std::map order of kidx, box -> N_b x N_b
 * column-major. lt_spectrum_dev then solves the k-points [k_begin, k_end) of the reduced
 * pencil (eigenvalues at eig_dev + k_begin*m0; box: all N_b).
 * info (8 int64): L0, nblocks (0 for box), N_b, K, m0, R_tot, doubles per operator,
 * eigenvalues per k-point; kidx (optional, periodic): [nblocks][3]. */
lt_status lt_core_layout(lt_ctx* ctx, const lt_sysdev* sys, int periodic, int64_t* info, int64_t* kidx);
lt_status lt_assemble_core_dev(lt_ctx* ctx, const lt_sysdev* sys, int periodic, int64_t r_begin, int64_t r_end,
                               int with_kinetic, double* H_dev, double* S_dev);
lt_status lt_spectrum_dev(lt_ctx* ctx, const lt_sysdev* sys, int periodic, const double* H_dev, const double* S_dev,
                          double* eig_dev, int64_t k_begin, int64_t k_end);

/* ---- assembly (galerkin.hpp:70, :74; eigensolver.hpp:23-24) ------------------ */
lt_status lt_assemble(lt_ctx* ctx, const lt_system* sys, int periodic, lt_kind kind, lt_operator** out);
/* fused Laplace+Nuclear+Mass assembly: H = 0.5 Laplace - Nuclear, S = Mass */
lt_status lt_assemble_core(lt_ctx* ctx, const lt_system* sys, int periodic, lt_operator** H, lt_operator** S);
lt_status lt_combine(lt_ctx* ctx, double wa, const lt_operator* a, double wb, const lt_operator* b,
                     lt_operator** out);
void lt_op_free(lt_operator* op);
/* info (12 int64): periodic, m0, L[3], overlap_L0, coefficient_rank, stored blocks, N_b, band[3] */
void lt_op_info(const lt_operator* op, int64_t* info);
lt_status lt_op_dense(const lt_operator* op, double* out);                  /* box: N_b*N_b col-major */
lt_status lt_op_blocks(const lt_operator* op, int64_t* kidx, double* blocks); /* periodic */

/* ---- spectrum ------------------------------------------------------------------ */
/* eigensolver.hpp:32-33 (AssembledOperator overload) */
lt_status lt_solve_periodic_ops(lt_ctx* ctx, const lt_operator* H, const lt_operator* S, double* eig);
/* eigensolver.hpp:29-31 (GeneratingBlockTensor overload); host generating tensors */
lt_status lt_solve_periodic(lt_ctx* ctx, const int64_t* dims, int64_t m0, int64_t nH, const int64_t* kH,
                            const double* bH, int64_t nS, const int64_t* kS, const double* bS, double* eig);
/* block_circulant.hpp:86: out = k_count blocks of m0*m0 complex (re,im interleaved), col-major */
lt_status lt_block_diagonalize(lt_ctx* ctx, const int64_t* dims, int64_t m0, int64_t nblk, const int64_t* kidx,
                               const double* blocks, double* out);
/* eigensolver.hpp:17-18 (eigenvalues only): host H, S column-major */
lt_status lt_solve_box_dense(lt_ctx* ctx, int64_t n, const double* H, const double* S, int64_t cap, double* eig);
/* batch of Hermitian-definite pencils (eigensolver.cpp:72-93); complex interleaved col-major */
lt_status lt_pencil_eig(lt_ctx* ctx, int64_t count, int64_t m0, const double* Hc, const double* Sc, double* eig);

/* ---- eigenvectors (want_vectors = true; eigensolver.cpp:29-32, :88-92) ------------ *
 * Box: vec = N_b x N_b col-major, S-orthonormal columns X = L^-T Z (DenseSpectrum::eigenvectors).
 * Periodic / pencils: vec = K blocks of m0 x m0 complex (re,im interleaved, col-major), block j
 * = KPointSpectrum::eigenvectors[j] (columns u_{j,m}, S_j-orthonormal). Columns are defined up
 * to sign (box) or a unit phase (periodic), and within degenerate eigenspaces up to rotation. */
lt_status lt_solve_box_dense_vectors(lt_ctx* ctx, int64_t n, const double* H, const double* S, int64_t cap,
                                     double* eig, double* vec);
lt_status lt_pencil_eigvec(lt_ctx* ctx, int64_t count, int64_t m0, const double* Hc, const double* Sc, double* eig,
                           double* vec);
lt_status lt_solve_periodic_ops_vectors(lt_ctx* ctx, const lt_operator* H, const lt_operator* S, double* eig,
                                        double* vec);
lt_status lt_solve_periodic_vectors(lt_ctx* ctx, const int64_t* dims, int64_t m0, int64_t nH, const int64_t* kH,
                                    const double* bH, int64_t nS, const int64_t* kS, const double* bS, double* eig,
                                    double* vec);
lt_status lt_solve_periodic_factorized_vectors(lt_ctx* ctx, const lt_operator* H, const lt_operator* S,
                                               double metadata_tol, double* eig, double* vec);
/* reconstruct_eigenvectors (eigensolver.hpp; eigensolver.cpp:164-175): out = N x N complex
 * col-major, N = K m0, column (j m0 + m) = bc_full_eigenvector(j, m); N > cap -> LT_ECAP */
lt_status lt_reconstruct_eigenvectors(lt_ctx* ctx, const int64_t* dims, int64_t m0, const double* vec, int64_t cap,
                                      double* out);
/* bc_full_eigenvector (block_circulant.hpp; block_circulant.cpp:267-289): out = N complex */
lt_status lt_bc_full_eigenvector(lt_ctx* ctx, const int64_t* dims, int64_t m0, const double* vec, int64_t j,
                                 int64_t m, double* out);

/* ---- separable metadata and the factorized Fourier path -------------------------- *
 * Periodic operators carry their rank metadata (galerkin.cpp:394-423; combine scales level 0
 * and concatenates, eigensolver.cpp:57-64). Layout of a term list: [t][level l][L_l][m0*m0]
 * (SeparableTerm::level_blocks, factorized_diag.hpp). */
int64_t lt_op_separable_count(const lt_operator* op); /* doubles lt_op_separable writes; 0: none */
lt_status lt_op_separable(const lt_operator* op, double* out);
/* separable_residual (galerkin.hpp): max |gen_k - expanded_k| over the lattice */
lt_status lt_separable_residual(lt_ctx* ctx, const lt_operator* op, double* resid);
/* solve_periodic_factorized (eigensolver.hpp): metadata residual above metadata_tol is a
 * StructureError; then 1D DFTs per level and per-k Hadamard sums, batched pencils */
lt_status lt_solve_periodic_factorized(lt_ctx* ctx, const lt_operator* H, const lt_operator* S, double metadata_tol,
                                       double* eig);
/* the same from host generating tensors and host term lists (tH / tS terms each) */
lt_status lt_solve_periodic_factorized_gen(lt_ctx* ctx, const int64_t* dims, int64_t m0, int64_t nH, const int64_t* kH,
                                           const double* bH, int64_t tH, const double* termsH, int64_t nS,
                                           const int64_t* kS, const double* bS, int64_t tS, const double* termsS,
                                           double metadata_tol, double* eig);
/* factorized_block_diagonalize (factorized_diag.hpp): out = K blocks, complex interleaved */
lt_status lt_factorized_block_diagonalize(lt_ctx* ctx, int levels, const int64_t* dims, int64_t m0, int64_t nterms,
                                          const double* terms, double* out);

/* box_circulant_defect (galerkin.hpp:76-83): nuclear box matrix minus the dense expansion of
 * the periodic circulant; rel_fro = ||defect||_F / ||box||_F; defect (optional) N_b*N_b col-major */
lt_status lt_box_circulant_defect(lt_ctx* ctx, const lt_system* sys, double* rel_fro, double* defect);

/* ---- stage entry points for unit parity tests ---------------------------------- */
lt_status lt_sinc_quadrature(lt_ctx* ctx, int64_t M, double* nodes, double* weights); /* sinc_quadrature.cpp:9-29 */
lt_status lt_overlap_constant(lt_ctx* ctx, const lt_system* sys, int64_t* L0);         /* gto_basis.cpp:87-126 */
/* newton_kernel.cpp:22-45 on one centred grid: out ncells x (2M+1) col-major */
lt_status lt_newton_master(lt_ctx* ctx, int64_t ncells, double h, int64_t M, double* out);
/* the potential panels assembly uses (galerkin.cpp:151-198), margin in unit cells:
 * rows[3], tiled[3]; panels: direction-major, each rows_l x R_tot col-major; weights R_tot.
 * Call with panels == NULL to query rows. */
lt_status lt_potential(lt_ctx* ctx, const lt_system* sys, int periodic, int64_t margin, int64_t* rows,
                       int64_t* tiled, double* panels, double* weights, int64_t panels_cap);
/* assembled_window_sum (canonical_tensor.hpp:97-99) on one panel */
lt_status lt_assembled_window_sum(lt_ctx* ctx, int64_t mrows, int64_t R, const double* master, int64_t nsh,
                                  const int64_t* shifts, int64_t size, double* out);
/* sample_gto_1d (gto_basis.hpp:47-49) for every basis function and direction of the
 * assembly grids at the given margin: pwc and pwl profiles with their supports.
 * lo/hi: [2][3][m0] (0 = pwc, 1 = pwl); values: for each (kind, l, mu) a full-grid
 * vector of length grid_l (zero outside [lo, hi)), packed in that order. */
lt_status lt_profiles(lt_ctx* ctx, const lt_system* sys, int64_t margin, int64_t* grid, int64_t* lo, int64_t* hi,
                      double* values, int64_t values_cap);

#ifdef __cplusplus
}
#endif
#endif
