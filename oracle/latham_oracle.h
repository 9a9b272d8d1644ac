/* oracle/latham_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * C ABI of Oracle-X, the clean-room CPU restatement of the reference's hot path
 * (arXiv 1408.3839 C++ reference, /root/reference/proj/core). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load it, and only as the checker or the timed CPU baseline — never as part of
 * the product path (the product is paper_1408_3839_b200/, which has no CPU
 * fallback).
 *
 * The system struct has the same layout as lt_system in include/latham_b200.h so a
 * single host-side description feeds both. Per-direction n/nbar generalise the
 * reference's scalar grid; with n[0]=n[1]=n[2] every
 * function reduces to the reference exactly.
 */
#ifndef LATHAM_ORACLE_H
#define LATHAM_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct or_system {
    double b;
    int64_t L[3];
    int64_t n[3];
    int64_t nbar[3];
    int64_t quad_M;
    double eps_ov;
    int64_t n_nuclei;
    const double* nuc_pos;    /* [n_nuclei][3] cell-centred */
    const double* nuc_charge; /* [n_nuclei] */
    int64_t m0;
    const double* bf_center;  /* [m0][3] cell-centred */
    const double* bf_alpha;   /* [m0] */
    const int32_t* bf_deg;    /* [m0][3] */
} or_system;

/* status codes mirror latham/errors.hpp:10-43 */
enum { OR_OK = 0, OR_EDIM = 1, OR_EBOUNDS = 2, OR_ESTRUCT = 3, OR_EDEFINITE = 4, OR_ECAP = 5, OR_EGENERIC = 6 };

typedef struct or_op or_op; /* AssembledOperator (galerkin.hpp:43-54) */

/* kind: 0 Laplace, 1 Mass, 2 Nuclear (galerkin.hpp:37) */
int or_assemble(const or_system* sys, int periodic, int kind, or_op** out);
int or_combine(double wa, const or_op* a, double wb, const or_op* b, or_op** out);
void or_op_free(or_op* op);
/* info: [0] periodic [1] m0 [2..4] L [5] overlap_L0 [6] coefficient_rank
 *       [7] stored block count (periodic) [8] N_b [9..11] band  */
void or_op_info(const or_op* op, int64_t* info);
void or_op_dense(const or_op* op, double* out);                 /* N_b*N_b col-major */
void or_op_blocks(const or_op* op, int64_t* kidx, double* blk); /* map order; blocks col-major */
/* separable metadata (galerkin.cpp:394-423): rank terms x 3 levels x L_l blocks */
void or_op_separable(const or_op* op, double* out);             /* [rank][3][L_l][m0*m0] packed */

/* eigensolver.cpp:124-141: eigenvalues [k_count][m0], ascending per k */
int or_solve_periodic_ops(const or_op* H, const or_op* S, int64_t threads, double* eig);
/* generic generating tensors (block_circulant.hpp:18-48) */
int or_solve_periodic(const int64_t* dims, int64_t m0, int64_t nH, const int64_t* kH, const double* bH,
                      int64_t nS, const int64_t* kS, const double* bS, int64_t threads, double* eig);
int or_solve_periodic_factorized_ops(const or_op* H, const or_op* S, int64_t threads, double* eig);
/* block_circulant.cpp:184-196: out [k_count][m0*m0] complex (re,im interleaved), col-major blocks */
int or_block_diagonalize(const int64_t* dims, int64_t m0, int64_t nblk, const int64_t* kidx,
                         const double* blocks, double* out);
/* eigensolver.cpp:12-35, eigenvalues only */
int or_solve_box_dense(int64_t n, const double* H, const double* S, int64_t cap, double* eig);
/* one Hermitian-definite pencil (eigensolver.cpp:72-93): complex interleaved col-major */
int or_solve_pencil(int64_t m0, const double* Hc, const double* Sc, int64_t j, double* eig);

/* ---- stage entry points for unit parity tests ---- */
void or_sinc_quadrature(int64_t M, double* nodes, double* weights);
int64_t or_overlap_constant(const or_system* sys);
/* newton_kernel.cpp:22-45 one direction: ncells x R col-major */
void or_newton_master_column(int64_t ncells, double h, int64_t M, double* out);
/* box/periodic lattice potential as used by assembly (galerkin.cpp:151-198):
 * rows[3] filled, panels [l] rows_l x R_tot col-major concatenated; weights R_tot */
int or_potential(const or_system* sys, int periodic, int64_t margin, int64_t* rows, int64_t* tiled,
                 double* panels, double* weights, int64_t panels_cap);
/* canonical_tensor.cpp:123-164 on a single panel: master (mrows x R col-major) */
int or_assembled_window_sum(int64_t mrows, int64_t R, const double* master, int64_t nsh,
                            const int64_t* shifts, int64_t size, double* out);
/* gto_basis.cpp:31-47: returns support length; offset in *off; values (full grid_n buffer) */
int64_t or_sample_gto_1d(const double* center, double alpha, const int32_t* deg, int dir,
                         int64_t grid_n, double step, int64_t cell_index, int64_t per_cell,
                         double b, double align, double eps, int64_t* off, double* values);
/* fem1d.cpp:19-32 supported tri form */
double or_tri_form(int64_t uoff, int64_t ulen, const double* u, int64_t voff, int64_t vlen,
                   const double* v, double lo, double diag);

const char* or_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
