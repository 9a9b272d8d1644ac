// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (Oracle-R).
//
// C ABI over the reference's own library code (/root/reference/proj/core/src/*.cpp,
// compiled where it lies against oracle/eigen_shim by `make -C oracle ref`). Same
// functions and layouts as Oracle-X (latham_oracle.h) with the prefix ref_, so
// oracle/binding.py can drive either. The reference grid is isotropic: systems with
// n[0] != n[1] != n[2] are refused (DimensionError).
#include <algorithm>
#include <array>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "latham/block_circulant.hpp"
#include "latham/eigensolver.hpp"
#include "latham/factorized_diag.hpp"
#include "latham/galerkin.hpp"
#include "latham_oracle.h"

using namespace latham;

namespace {

thread_local std::string g_err;

struct Op {
    AssembledOperator op;
};

int code_of(const std::exception& e) {
    if (dynamic_cast<const DimensionError*>(&e)) return OR_EDIM;
    if (dynamic_cast<const BoundsError*>(&e)) return OR_EBOUNDS;
    if (dynamic_cast<const StructureError*>(&e)) return OR_ESTRUCT;
    if (dynamic_cast<const DefinitenessError*>(&e)) return OR_EDEFINITE;
    if (dynamic_cast<const ResourceCapError*>(&e)) return OR_ECAP;
    return OR_EGENERIC;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        g_err.clear();
        return OR_OK;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

LatticeSystem to_sys(const or_system* s) {
    if (s->n[0] != s->n[1] || s->n[1] != s->n[2] || s->nbar[0] != s->nbar[1] || s->nbar[1] != s->nbar[2])
        throw DimensionError("ref_driver: the reference grid is isotropic (n and nbar must agree per direction)");
    LatticeSystem sys;
    sys.b = s->b;
    sys.L = {s->L[0], s->L[1], s->L[2]};
    sys.n = s->n[0];
    sys.nbar = s->nbar[0];
    sys.quad_M = s->quad_M;
    sys.eps_ov = s->eps_ov;
    sys.nuclei.cell_size = s->b;
    for (int64_t i = 0; i < s->n_nuclei; ++i)
        sys.nuclei.nuclei.push_back(
            Nucleus{{s->nuc_pos[3 * i], s->nuc_pos[3 * i + 1], s->nuc_pos[3 * i + 2]}, s->nuc_charge[i]});
    for (int64_t m = 0; m < s->m0; ++m) {
        GtoFunction f;
        for (int l = 0; l < 3; ++l) {
            f.center[l] = s->bf_center[3 * m + l];
            f.degrees[l] = s->bf_deg[3 * m + l];
        }
        f.exponent = s->bf_alpha[m];
        sys.basis.functions.push_back(f);
    }
    return sys;
}

GeneratingBlockTensor gen_from(const int64_t* dims, int64_t m0, int64_t nblk, const int64_t* k, const double* b) {
    int levels = dims[2] > 1 ? 3 : dims[1] > 1 ? 2 : 1;
    GeneratingBlockTensor g(levels, {dims[0], dims[1], dims[2]}, m0);
    for (int64_t i = 0; i < nblk; ++i) {
        Eigen::MatrixXd blk(m0, m0);
        std::memcpy(blk.data(), b + i * m0 * m0, sizeof(double) * m0 * m0);
        g.set_block({k[3 * i], k[3 * i + 1], k[3 * i + 2]}, blk);
    }
    return g;
}

}  // namespace

struct or_op {
    AssembledOperator op;
};

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_assemble(const or_system* s, int periodic, int kind, or_op** out) {
    return guarded([&] {
        const LatticeSystem sys = to_sys(s);
        const OperatorKind k = kind == 0 ? OperatorKind::Laplace : kind == 1 ? OperatorKind::Mass : OperatorKind::Nuclear;
        auto o = std::make_unique<or_op>();
        o->op = periodic ? assemble_periodic(sys, k) : assemble_box(sys, k);
        *out = o.release();
    });
}

int ref_combine(double wa, const or_op* a, double wb, const or_op* b, or_op** out) {
    return guarded([&] {
        auto o = std::make_unique<or_op>();
        o->op = combine(wa, a->op, wb, b->op);
        *out = o.release();
    });
}

void ref_op_free(or_op* op) { delete op; }

void ref_op_info(const or_op* o, int64_t* info) {
    const AssembledOperator& op = o->op;
    info[0] = op.periodic;
    info[1] = op.m0;
    for (int l = 0; l < 3; ++l) info[2 + l] = op.L[l];
    info[5] = op.overlap_L0;
    info[6] = op.coefficient_rank;
    info[7] = op.periodic ? op.gen.stored_count() : 0;
    info[8] = op.m0 * op.L[0] * op.L[1] * op.L[2];
    for (int l = 0; l < 3; ++l) info[9 + l] = std::min<int64_t>(op.overlap_L0, op.L[l] - 1);
}

void ref_op_dense(const or_op* o, double* out) {
    std::memcpy(out, o->op.dense.data(), sizeof(double) * o->op.dense.size());
}

void ref_op_blocks(const or_op* o, int64_t* kidx, double* blk) {
    int64_t i = 0;
    const int64_t mm = o->op.m0 * o->op.m0;
    for (const auto& [k, b] : o->op.gen.stored()) {
        for (int l = 0; l < 3; ++l) kidx[3 * i + l] = k[l];
        std::memcpy(blk + i * mm, b.data(), sizeof(double) * mm);
        ++i;
    }
}

int ref_solve_periodic_ops(const or_op* H, const or_op* S, int64_t threads, double* eig) {
    return guarded([&] {
        const KPointSpectrum spec = solve_periodic(H->op, S->op, false, threads);
        for (int64_t j = 0; j < spec.k_count(); ++j)
            for (int64_t m = 0; m < spec.m0; ++m) eig[j * spec.m0 + m] = spec.eigenvalues[j][m];
    });
}

int ref_solve_periodic_factorized_ops(const or_op* H, const or_op* S, int64_t threads, double* eig) {
    return guarded([&] {
        const KPointSpectrum spec = solve_periodic_factorized(H->op, S->op, false, threads);
        for (int64_t j = 0; j < spec.k_count(); ++j)
            for (int64_t m = 0; m < spec.m0; ++m) eig[j * spec.m0 + m] = spec.eigenvalues[j][m];
    });
}

int ref_solve_periodic(const int64_t* dims, int64_t m0, int64_t nH, const int64_t* kH, const double* bH, int64_t nS,
                       const int64_t* kS, const double* bS, int64_t threads, double* eig) {
    return guarded([&] {
        const KPointSpectrum spec =
            solve_periodic(gen_from(dims, m0, nH, kH, bH), gen_from(dims, m0, nS, kS, bS), false, threads);
        for (int64_t j = 0; j < spec.k_count(); ++j)
            for (int64_t m = 0; m < spec.m0; ++m) eig[j * spec.m0 + m] = spec.eigenvalues[j][m];
    });
}

int ref_block_diagonalize(const int64_t* dims, int64_t m0, int64_t nblk, const int64_t* kidx, const double* blocks,
                          double* out) {
    return guarded([&] {
        const BlockDiagonalForm bd = bc_block_diagonalize(BlockCirculant{gen_from(dims, m0, nblk, kidx, blocks)});
        int64_t at = 0;
        for (const auto& b : bd.blocks)
            for (int64_t i = 0; i < b.size(); ++i) {
                out[at++] = b[i].real();
                out[at++] = b[i].imag();
            }
    });
}

int ref_solve_box_dense(int64_t n, const double* H, const double* S, int64_t cap, double* eig) {
    return guarded([&] {
        Eigen::MatrixXd h(n, n), s(n, n);
        std::memcpy(h.data(), H, sizeof(double) * n * n);
        std::memcpy(s.data(), S, sizeof(double) * n * n);
        const DenseSpectrum ds = solve_box_dense(h, s, false, cap);
        for (int64_t i = 0; i < n; ++i) eig[i] = ds.eigenvalues[i];
    });
}

// want_vectors = true (eigensolver.cpp:31-32): vec = n x n col-major
int ref_solve_box_dense_vec(int64_t n, const double* H, const double* S, int64_t cap, double* eig, double* vec) {
    return guarded([&] {
        Eigen::MatrixXd h(n, n), s(n, n);
        std::memcpy(h.data(), H, sizeof(double) * n * n);
        std::memcpy(s.data(), S, sizeof(double) * n * n);
        const DenseSpectrum ds = solve_box_dense(h, s, true, cap);
        for (int64_t i = 0; i < n; ++i) eig[i] = ds.eigenvalues[i];
        std::memcpy(vec, ds.eigenvectors.data(), sizeof(double) * n * n);
    });
}

static void put_vectors(const KPointSpectrum& spec, double* eig, double* vec) {
    const int64_t mm = spec.m0 * spec.m0;
    for (int64_t j = 0; j < spec.k_count(); ++j) {
        for (int64_t m = 0; m < spec.m0; ++m) eig[j * spec.m0 + m] = spec.eigenvalues[j][m];
        const auto& v = spec.eigenvectors[j];
        for (int64_t i = 0; i < mm; ++i) {
            vec[2 * (j * mm + i)] = v.data()[i].real();
            vec[2 * (j * mm + i) + 1] = v.data()[i].imag();
        }
    }
}

// solve_periodic(gen, gen, want_vectors = true): vec = K blocks m0 x m0 complex interleaved
int ref_solve_periodic_vec(const int64_t* dims, int64_t m0, int64_t nH, const int64_t* kH, const double* bH,
                           int64_t nS, const int64_t* kS, const double* bS, int64_t threads, double* eig,
                           double* vec) {
    return guarded([&] {
        put_vectors(solve_periodic(gen_from(dims, m0, nH, kH, bH), gen_from(dims, m0, nS, kS, bS), true, threads), eig,
                    vec);
    });
}

static KPointSpectrum spec_from(const int64_t* dims, int64_t m0, const double* vec) {
    KPointSpectrum spec;
    spec.dims = {dims[0], dims[1], dims[2]};
    spec.m0 = m0;
    const int64_t mm = m0 * m0;
    for (int64_t j = 0; j < spec.k_count(); ++j) {
        spec.eigenvalues.push_back(Eigen::VectorXd::Zero(m0));
        Eigen::MatrixXcd v(m0, m0);
        for (int64_t i = 0; i < mm; ++i) v.data()[i] = {vec[2 * (j * mm + i)], vec[2 * (j * mm + i) + 1]};
        spec.eigenvectors.push_back(v);
    }
    return spec;
}

// reconstruct_eigenvectors (eigensolver.cpp:164-175): out = N x N complex col-major
int ref_reconstruct_eigenvectors(const int64_t* dims, int64_t m0, const double* vec, int64_t cap, double* out) {
    return guarded([&] {
        const Eigen::MatrixXcd U = reconstruct_eigenvectors(spec_from(dims, m0, vec), cap);
        for (int64_t i = 0; i < U.size(); ++i) {
            out[2 * i] = U.data()[i].real();
            out[2 * i + 1] = U.data()[i].imag();
        }
    });
}

// bc_full_eigenvector (block_circulant.cpp:267-289)
int ref_bc_full_eigenvector(const int64_t* dims, int64_t m0, const double* vec, int64_t j, int64_t m, double* out) {
    return guarded([&] {
        const Eigen::VectorXcd u = bc_full_eigenvector(spec_from(dims, m0, vec), j, m);
        for (int64_t i = 0; i < u.size(); ++i) {
            out[2 * i] = u[i].real();
            out[2 * i + 1] = u[i].imag();
        }
    });
}

void ref_sinc_quadrature(int64_t M, double* nodes, double* weights) {
    const SincQuadrature q = build_sinc_quadrature(M);
    for (int64_t i = 0; i < q.rank(); ++i) {
        nodes[i] = q.nodes[i];
        weights[i] = q.weights[i];
    }
}

int64_t ref_overlap_constant(const or_system* s) {
    try {
        const LatticeSystem sys = to_sys(s);
        return overlap_constant(sys.basis, sys.b, sys.n, sys.eps_ov);
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

void ref_newton_master_column(int64_t ncells, double h, int64_t M, double* out) {
    const Grid1D g = Grid1D::centered_cells(ncells, h);
    const CanonicalTensor3 t = newton_master_tensor({g, g, g}, build_sinc_quadrature(M));
    std::memcpy(out, t.factor(0).data(), sizeof(double) * t.factor(0).size());
}

// the potential panels the assembly uses (galerkin.cpp:151-198) built from the public
// newton_kernel.hpp functions
int ref_potential(const or_system* s, int periodic, int64_t margin, int64_t* rows, int64_t* tiled, double* panels,
                  double* weights, int64_t panels_cap) {
    return guarded([&] {
        const LatticeSystem sys = to_sys(s);
        const SincQuadrature quad = build_sinc_quadrature(sys.quad_M);
        const double h = sys.h();
        std::array<Eigen::MatrixXd, 3> pot;
        Eigen::VectorXd w;
        if (!periodic) {
            const auto grids = master_grids_box(sys.n, h, sys.L, margin);
            const CanonicalTensor3 lat =
                lattice_potential_box(newton_master_tensor(grids, quad), sys.nuclei, sys.L, sys.n, h, margin);
            for (int l = 0; l < 3; ++l) {
                pot[l] = lat.factor(l);
                tiled[l] = 0;
            }
            w = lat.weights();
        } else {
            const CanonicalTensor3 cell = lattice_potential_periodic_cell(
                newton_master_tensor(master_grids_periodic(sys.n, h, sys.L), quad), sys.nuclei, sys.L, sys.n, h);
            const std::array<Index, 3> ones{1, 1, 1};
            const CanonicalTensor3 open = lattice_potential_box(
                newton_master_tensor(master_grids_box(sys.n, h, ones, margin), quad), sys.nuclei, ones, sys.n, h, margin);
            for (int l = 0; l < 3; ++l) {
                pot[l] = sys.L[l] > 1 ? cell.factor(l) : open.factor(l);
                tiled[l] = sys.L[l] > 1;
            }
            w = cell.weights();
        }
        int64_t need = 0;
        for (int l = 0; l < 3; ++l) {
            rows[l] = pot[l].rows();
            need += pot[l].size();
        }
        if (!panels || need > panels_cap) return;
        int64_t at = 0;
        for (int l = 0; l < 3; ++l) {
            std::memcpy(panels + at, pot[l].data(), sizeof(double) * pot[l].size());
            at += pot[l].size();
        }
        std::memcpy(weights, w.data(), sizeof(double) * w.size());
    });
}

int ref_assembled_window_sum(int64_t mrows, int64_t R, const double* master, int64_t nsh, const int64_t* shifts,
                             int64_t size, double* out) {
    return guarded([&] {
        std::array<Eigen::MatrixXd, 3> f;
        f[0] = Eigen::MatrixXd(mrows, R);
        std::memcpy(f[0].data(), master, sizeof(double) * mrows * R);
        f[1] = Eigen::MatrixXd::Ones(1, R);
        f[2] = Eigen::MatrixXd::Ones(1, R);
        const CanonicalTensor3 m(f, Eigen::VectorXd::Ones(R));
        std::array<std::vector<Index>, 3> sh;
        sh[0].assign(shifts, shifts + nsh);
        sh[1] = {0};
        sh[2] = {0};
        const CanonicalTensor3 r = assembled_window_sum(m, sh, {size, 1, 1});
        std::memcpy(out, r.factor(0).data(), sizeof(double) * size * R);
    });
}

int64_t ref_sample_gto_1d(const double* center, double alpha, const int32_t* deg, int dir, int64_t grid_n, double step,
                          int64_t cell_index, int64_t per_cell, double b, double align, double eps, int64_t* off,
                          double* values) {
    GtoFunction fn;
    for (int l = 0; l < 3; ++l) {
        fn.center[l] = center[l];
        fn.degrees[l] = deg[l];
    }
    fn.exponent = alpha;
    const Supported1D s = sample_gto_1d(fn, dir, grid_n, step, cell_index, per_cell, b, align, eps);
    *off = s.offset;
    std::memcpy(values, s.values.data(), sizeof(double) * s.values.size());
    return s.values.size();
}

// the supported tri_form through the public Fem1D forms: (lo, diag) identify the form
double ref_tri_form(int64_t uoff, int64_t ulen, const double* u, int64_t voff, int64_t vlen, const double* v, double lo,
                    double diag) {
    Supported1D a{uoff, Eigen::VectorXd(ulen)}, bb{voff, Eigen::VectorXd(vlen)};
    std::memcpy(a.values.data(), u, sizeof(double) * ulen);
    std::memcpy(bb.values.data(), v, sizeof(double) * vlen);
    const Index n = std::max(a.end(), bb.end()) + 2;
    if (lo < 0) {  // stiffness: lo = -1/h, diag = 2/h
        const Fem1D fem = fem_1d(n, -1.0 / lo);
        return fem.stiffness_form(a, bb);
    }
    const Fem1D fem = fem_1d(n, 6.0 * lo);  // mass: lo = h/6
    return fem.mass_form(a, bb);
}

}  // extern "C"
