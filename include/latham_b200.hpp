// include/latham_b200.hpp — header-only C++ mirror of the reference's public API
// (proj/core/include/latham/*.hpp) over the C-ABI in latham_b200.h.
//
// Same type names, field names, argument meaning and exception classes as the reference,
// in namespace latham_b200 so it can live next to `latham` in one binary:
//
//   reference (latham::)                                    here (latham_b200::)
//   LatticeSystem, NucleiSet, Nucleus, GtoBasis,           same (n / nbar per direction;
//     GtoFunction (galerkin.hpp:17-35, newton_kernel.hpp,    set_grid(n, nbar) sets all three)
//     gto_basis.hpp)
//   OperatorKind (galerkin.hpp:37)                          same
//   AssembledOperator (galerkin.hpp:43-54)                  same fields; payload on the device,
//                                                            dense() / generating_blocks() copy out
//   assemble_box / assemble_periodic (galerkin.hpp:70,74)   same, plus a Context argument
//   combine (eigensolver.hpp:23-24)                         same
//   solve_periodic (eigensolver.hpp:32-33)                  same (eigenvalues; want_vectors = false)
//   solve_box_dense (eigensolver.hpp:17-18)                 same (eigenvalues only)
//   KPointSpectrum / DenseSpectrum (spectrum.hpp,           same fields (std::vector instead of
//     eigensolver.hpp)                                       Eigen vectors)
//   Error, DimensionError, BoundsError, StructureError,     same classes, same messages
//     DefinitenessError, ResourceCapError (errors.hpp)
//
// plus solve_core_periodic / solve_core_box: the whole path of tools/commands.cpp:51-59
// (H = 0.5 Laplace - Nuclear, S = Mass) followed by the spectrum, in one device pass.
#pragma once

#include <algorithm>
#include <array>
#include <complex>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "latham_b200.h"

namespace latham_b200 {

using Index = std::int64_t;

// ---- errors (errors.hpp:10-43) -------------------------------------------------
class Error : public std::runtime_error {
public:
    explicit Error(const std::string& msg) : std::runtime_error(msg) {}
};
class DimensionError : public Error {
public:
    using Error::Error;
};
class BoundsError : public Error {
public:
    using Error::Error;
};
class StructureError : public Error {
public:
    using Error::Error;
};
class DefinitenessError : public Error {
public:
    using Error::Error;
};
class ResourceCapError : public Error {
public:
    using Error::Error;
};
/// Device or driver failure (no reference counterpart).
class DeviceError : public Error {
public:
    using Error::Error;
};

inline void check(lt_status st) {
    if (st == LT_OK) return;
    const std::string msg = lt_last_error();
    switch (st) {
        case LT_EDIM: throw DimensionError(msg);
        case LT_EBOUNDS: throw BoundsError(msg);
        case LT_ESTRUCT: throw StructureError(msg);
        case LT_EDEFINITE: throw DefinitenessError(msg);
        case LT_ECAP: throw ResourceCapError(msg);
        case LT_ECUDA: throw DeviceError(msg);
        default: throw Error(msg);
    }
}

// ---- system description ----------------------------------------------------------
struct Nucleus {  // newton_kernel.hpp:12-16
    std::array<double, 3> position{0.0, 0.0, 0.0};
    double charge = 1.0;
};

struct NucleiSet {  // newton_kernel.hpp:19-28
    double cell_size = 0.0;
    std::vector<Nucleus> nuclei;
    Index count() const { return static_cast<Index>(nuclei.size()); }
};

struct GtoFunction {  // gto_basis.hpp:12-22
    std::array<double, 3> center{0.0, 0.0, 0.0};
    double exponent = 1.0;
    std::array<int, 3> degrees{0, 0, 0};
};

struct GtoBasis {  // gto_basis.hpp:24-29
    std::vector<GtoFunction> functions;
    Index m0() const { return static_cast<Index>(functions.size()); }
};

struct LatticeSystem {  // galerkin.hpp:17-35, with per-direction n / nbar
    double b = 0.0;
    std::array<Index, 3> L{1, 1, 1};
    std::array<Index, 3> n{0, 0, 0};
    std::array<Index, 3> nbar{0, 0, 0};
    Index quad_M = 20;
    NucleiSet nuclei;
    GtoBasis basis;
    double eps_ov = 1e-8;

    /// The reference's scalar grid (n = n[0] = n[1] = n[2]).
    void set_grid(Index n_all, Index nbar_all) {
        n = {n_all, n_all, n_all};
        nbar = {nbar_all, nbar_all, nbar_all};
    }
    Index m0() const { return basis.m0(); }
    Index lattice_count() const { return L[0] * L[1] * L[2]; }
    Index basis_count() const { return m0() * lattice_count(); }
};

enum class OperatorKind { Laplace, Mass, Nuclear };  // galerkin.hpp:37

/// Flat POD view of a LatticeSystem for the C-ABI (owns the packed arrays).
class SystemView {
public:
    explicit SystemView(const LatticeSystem& s) {
        for (const auto& nu : s.nuclei.nuclei) {
            pos_.insert(pos_.end(), nu.position.begin(), nu.position.end());
            z_.push_back(nu.charge);
        }
        for (const auto& f : s.basis.functions) {
            center_.insert(center_.end(), f.center.begin(), f.center.end());
            alpha_.push_back(f.exponent);
            for (int d : f.degrees) deg_.push_back(static_cast<int32_t>(d));
        }
        c_.b = s.b;
        for (int l = 0; l < 3; ++l) {
            c_.L[l] = s.L[l];
            c_.n[l] = s.n[l];
            c_.nbar[l] = s.nbar[l];
        }
        c_.quad_M = s.quad_M;
        c_.eps_ov = s.eps_ov;
        c_.n_nuclei = static_cast<int64_t>(z_.size());
        c_.nuc_pos = pos_.data();
        c_.nuc_charge = z_.data();
        c_.m0 = static_cast<int64_t>(alpha_.size());
        c_.bf_center = center_.data();
        c_.bf_alpha = alpha_.data();
        c_.bf_deg = deg_.data();
    }
    const lt_system* get() const { return &c_; }

private:
    std::vector<double> pos_, z_, center_, alpha_;
    std::vector<int32_t> deg_;
    lt_system c_{};
};

// ---- device context ----------------------------------------------------------------
/// One GPU: stream, solver handle, cached device buffers and CUDA graphs.
class Context {
public:
    explicit Context(int device = 0) { check(lt_create(device, &h_)); }
    ~Context() { lt_destroy(h_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    lt_ctx* get() const { return h_; }

private:
    lt_ctx* h_ = nullptr;
};

/// Several GPUs of one process (lt_mctx): one Context per device + an in-process NCCL
/// communicator; the device-parallel analogue of parallel_for (parallel.hpp:15-32).
class MultiContext {
public:
    explicit MultiContext(const std::vector<int>& devices) {
        check(lt_create_multi(devices.data(), static_cast<int>(devices.size()), &h_));
    }
    ~MultiContext() { lt_destroy_multi(h_); }
    MultiContext(const MultiContext&) = delete;
    MultiContext& operator=(const MultiContext&) = delete;
    lt_mctx* get() const { return h_; }
    int devices() const { return lt_multi_ndev(h_); }

private:
    lt_mctx* h_ = nullptr;
};

// ---- assembled operators (galerkin.hpp:43-54) ---------------------------------------
class AssembledOperator {
public:
    OperatorKind which = OperatorKind::Mass;
    bool periodic = false;
    Index m0 = 0;
    std::array<Index, 3> L{1, 1, 1};
    Index coefficient_rank = 0;
    Index overlap_L0 = 0;

    AssembledOperator() = default;
    explicit AssembledOperator(lt_operator* op, OperatorKind kind) : which(kind), h_(op, lt_op_free) {
        int64_t info[12] = {};
        lt_op_info(op, info);
        periodic = info[0] != 0;
        m0 = info[1];
        L = {info[2], info[3], info[4]};
        overlap_L0 = info[5];
        coefficient_rank = info[6];
        stored_ = info[7];
        nb_ = info[8];
    }
    const lt_operator* handle() const { return h_.get(); }
    Index basis_count() const { return nb_; }
    Index stored_count() const { return stored_; }

    /// Box payload: N_b x N_b column-major (galerkin.hpp:50 `dense`).
    std::vector<double> dense() const {
        std::vector<double> out(static_cast<size_t>(nb_ * nb_));
        check(lt_op_dense(h_.get(), out.data()));
        return out;
    }
    /// Periodic payload: the stored generating blocks keyed by kidx (block_circulant.hpp
    /// GeneratingBlockTensor::stored()), each m0 x m0 column-major.
    std::map<std::array<Index, 3>, std::vector<double>> generating_blocks() const {
        std::vector<int64_t> kidx(static_cast<size_t>(3 * stored_));
        std::vector<double> blocks(static_cast<size_t>(stored_ * m0 * m0));
        check(lt_op_blocks(h_.get(), kidx.data(), blocks.data()));
        std::map<std::array<Index, 3>, std::vector<double>> out;
        for (Index b = 0; b < stored_; ++b)
            out[{kidx[3 * b], kidx[3 * b + 1], kidx[3 * b + 2]}] =
                std::vector<double>(blocks.begin() + b * m0 * m0, blocks.begin() + (b + 1) * m0 * m0);
        return out;
    }

private:
    std::shared_ptr<lt_operator> h_;
    Index stored_ = 0, nb_ = 0;
};

inline lt_kind to_kind(OperatorKind k) {
    return k == OperatorKind::Laplace ? LT_LAPLACE : (k == OperatorKind::Mass ? LT_MASS : LT_NUCLEAR);
}

/// galerkin.hpp:70
inline AssembledOperator assemble_box(Context& ctx, const LatticeSystem& sys, OperatorKind which) {
    SystemView v(sys);
    lt_operator* op = nullptr;
    check(lt_assemble(ctx.get(), v.get(), 0, to_kind(which), &op));
    return AssembledOperator(op, which);
}

/// galerkin.hpp:74 (StructureError unless L_l > 2 L0 in every lattice direction)
inline AssembledOperator assemble_periodic(Context& ctx, const LatticeSystem& sys, OperatorKind which) {
    SystemView v(sys);
    lt_operator* op = nullptr;
    check(lt_assemble(ctx.get(), v.get(), 1, to_kind(which), &op));
    return AssembledOperator(op, which);
}

/// eigensolver.hpp:23-24
inline AssembledOperator combine(Context& ctx, double wa, const AssembledOperator& a, double wb,
                                 const AssembledOperator& b) {
    lt_operator* op = nullptr;
    check(lt_combine(ctx.get(), wa, a.handle(), wb, b.handle(), &op));
    AssembledOperator out(op, a.which);
    return out;
}

// ---- spectra (spectrum.hpp, eigensolver.hpp) ------------------------------------------
struct KPointSpectrum {
    std::array<Index, 3> dims{1, 1, 1};
    Index m0 = 0;
    std::string solver_path;
    std::vector<std::vector<double>> eigenvalues;  ///< per k-point (lexicographic), ascending
    /// per k-point m0 x m0 column-major blocks (columns u_{j,m}); empty unless requested
    std::vector<std::vector<std::complex<double>>> eigenvectors;
    Index k_count() const { return dims[0] * dims[1] * dims[2]; }
    bool has_vectors() const { return !eigenvectors.empty(); }
    std::array<Index, 3> k_multi(Index lin) const {
        return {lin / (dims[1] * dims[2]), (lin / dims[2]) % dims[1], lin % dims[2]};
    }
    std::vector<double> sorted_all() const {
        std::vector<double> out;
        for (const auto& ev : eigenvalues) out.insert(out.end(), ev.begin(), ev.end());
        std::sort(out.begin(), out.end());
        return out;
    }
};

struct DenseSpectrum {
    std::vector<double> eigenvalues;   ///< ascending
    std::vector<double> eigenvectors;  ///< n x n column-major, S-orthonormal; empty unless requested
};

// per-k blocks from the C-ABI's interleaved layout
inline void put_vectors(KPointSpectrum& s, const std::vector<double>& flat) {
    const Index mm = s.m0 * s.m0;
    s.eigenvectors.assign(static_cast<size_t>(s.k_count()), std::vector<std::complex<double>>(static_cast<size_t>(mm)));
    for (Index k = 0; k < s.k_count(); ++k)
        for (Index i = 0; i < mm; ++i)
            s.eigenvectors[static_cast<size_t>(k)][static_cast<size_t>(i)] = {flat[2 * (k * mm + i)],
                                                                             flat[2 * (k * mm + i) + 1]};
}

inline std::vector<double> flat_vectors(const KPointSpectrum& s) {
    std::vector<double> flat;
    flat.reserve(static_cast<size_t>(2 * s.k_count() * s.m0 * s.m0));
    for (const auto& blk : s.eigenvectors)
        for (const auto& z : blk) {
            flat.push_back(z.real());
            flat.push_back(z.imag());
        }
    return flat;
}

inline KPointSpectrum make_spectrum(const std::array<Index, 3>& dims, Index m0, const std::vector<double>& flat,
                                    const char* path) {
    KPointSpectrum s;
    s.dims = dims;
    s.m0 = m0;
    s.solver_path = path;
    const Index K = s.k_count();
    for (Index k = 0; k < K; ++k) s.eigenvalues.emplace_back(flat.begin() + k * m0, flat.begin() + (k + 1) * m0);
    return s;
}

/// eigensolver.hpp:32-33 (the k-point loop runs as one batched launch)
inline KPointSpectrum solve_periodic(Context& ctx, const AssembledOperator& H, const AssembledOperator& S,
                                     bool want_vectors = false) {
    const Index K = H.L[0] * H.L[1] * H.L[2];
    std::vector<double> flat(static_cast<size_t>(K * H.m0));
    if (!want_vectors) {
        check(lt_solve_periodic_ops(ctx.get(), H.handle(), S.handle(), flat.data()));
        return make_spectrum(H.L, H.m0, flat, "b200-fft-batched-pencil");
    }
    std::vector<double> vec(static_cast<size_t>(2 * K * H.m0 * H.m0));
    check(lt_solve_periodic_ops_vectors(ctx.get(), H.handle(), S.handle(), flat.data(), vec.data()));
    KPointSpectrum s = make_spectrum(H.L, H.m0, flat, "b200-fft-batched-pencil");
    put_vectors(s, vec);
    return s;
}

/// eigensolver.hpp:17-18 (H, S column-major n x n); the reference's default want_vectors
inline DenseSpectrum solve_box_dense(Context& ctx, const std::vector<double>& H, const std::vector<double>& S,
                                     Index n, Index cap = 4096, bool want_vectors = false) {
    if (static_cast<Index>(H.size()) != n * n || static_cast<Index>(S.size()) != n * n)
        throw DimensionError("solve_box_dense: H and S must be n x n");
    DenseSpectrum d;
    d.eigenvalues.resize(static_cast<size_t>(n));
    if (!want_vectors) {
        check(lt_solve_box_dense(ctx.get(), n, H.data(), S.data(), cap, d.eigenvalues.data()));
        return d;
    }
    d.eigenvectors.resize(static_cast<size_t>(n * n));
    check(lt_solve_box_dense_vectors(ctx.get(), n, H.data(), S.data(), cap, d.eigenvalues.data(),
                                     d.eigenvectors.data()));
    return d;
}

/// eigensolver.hpp reconstruct_eigenvectors: N x N complex column-major, N = K m0
inline std::vector<std::complex<double>> reconstruct_eigenvectors(Context& ctx, const KPointSpectrum& spec,
                                                                  Index cap = 4096) {
    if (!spec.has_vectors()) throw StructureError("reconstruct_eigenvectors: spectrum carries no eigenvectors");
    const Index N = spec.k_count() * spec.m0;
    const std::vector<double> u = flat_vectors(spec);
    std::vector<double> out(static_cast<size_t>(N <= cap ? 2 * N * N : 2));
    check(lt_reconstruct_eigenvectors(ctx.get(), spec.dims.data(), spec.m0, u.data(), cap, out.data()));
    std::vector<std::complex<double>> z(static_cast<size_t>(N * N));
    for (size_t i = 0; i < z.size(); ++i) z[i] = {out[2 * i], out[2 * i + 1]};
    return z;
}

/// block_circulant.hpp bc_full_eigenvector
inline std::vector<std::complex<double>> bc_full_eigenvector(Context& ctx, const KPointSpectrum& spec, Index j,
                                                             Index m) {
    if (!spec.has_vectors()) throw StructureError("bc_full_eigenvector: no eigenvectors stored");
    const Index N = spec.k_count() * spec.m0;
    const std::vector<double> u = flat_vectors(spec);
    std::vector<double> out(static_cast<size_t>(2 * N));
    check(lt_bc_full_eigenvector(ctx.get(), spec.dims.data(), spec.m0, u.data(), j, m, out.data()));
    std::vector<std::complex<double>> z(static_cast<size_t>(N));
    for (size_t i = 0; i < z.size(); ++i) z[i] = {out[2 * i], out[2 * i + 1]};
    return z;
}

/// eigensolver.hpp solve_periodic_factorized: rank metadata validated against the
/// generating blocks (StructureError above metadata_tol), 1D DFTs per level, per-k sums.
inline KPointSpectrum solve_periodic_factorized(Context& ctx, const AssembledOperator& H, const AssembledOperator& S,
                                                double metadata_tol = 1e-10, bool want_vectors = false) {
    const Index K = H.L[0] * H.L[1] * H.L[2];
    std::vector<double> flat(static_cast<size_t>(K * H.m0));
    if (!want_vectors) {
        check(lt_solve_periodic_factorized(ctx.get(), H.handle(), S.handle(), metadata_tol, flat.data()));
        return make_spectrum(H.L, H.m0, flat, "periodic_factorized");
    }
    std::vector<double> vec(static_cast<size_t>(2 * K * H.m0 * H.m0));
    check(lt_solve_periodic_factorized_vectors(ctx.get(), H.handle(), S.handle(), metadata_tol, flat.data(),
                                               vec.data()));
    KPointSpectrum s = make_spectrum(H.L, H.m0, flat, "periodic_factorized");
    put_vectors(s, vec);
    return s;
}

/// galerkin.hpp separable_residual
inline double separable_residual(Context& ctx, const AssembledOperator& op) {
    double r = 0.0;
    check(lt_separable_residual(ctx.get(), op.handle(), &r));
    return r;
}

struct DefectReport {  // galerkin.hpp:76-83
    std::vector<double> defect;  ///< N_b x N_b column-major
    double relative_fro = 0.0;
};

/// galerkin.hpp box_circulant_defect
inline DefectReport box_circulant_defect(Context& ctx, const LatticeSystem& sys) {
    SystemView v(sys);
    DefectReport d;
    d.defect.resize(static_cast<size_t>(sys.basis_count() * sys.basis_count()));
    check(lt_box_circulant_defect(ctx.get(), v.get(), &d.relative_fro, d.defect.data()));
    return d;
}

struct BandStructure {  // spectrum.hpp
    Index m0 = 0;
    std::vector<std::vector<double>> bands;  ///< m0 bands, each of length k_count
    std::vector<double> band_min, band_max;
};

/// eigensolver.hpp spectral_bands
inline BandStructure spectral_bands(const KPointSpectrum& spec) {
    BandStructure bs;
    bs.m0 = spec.m0;
    bs.bands.assign(static_cast<size_t>(spec.m0), std::vector<double>(static_cast<size_t>(spec.k_count())));
    for (Index m = 0; m < spec.m0; ++m) {
        for (Index j = 0; j < spec.k_count(); ++j)
            bs.bands[static_cast<size_t>(m)][static_cast<size_t>(j)] =
                spec.eigenvalues[static_cast<size_t>(j)][static_cast<size_t>(m)];
        const auto& b = bs.bands[static_cast<size_t>(m)];
        bs.band_min.push_back(*std::min_element(b.begin(), b.end()));
        bs.band_max.push_back(*std::max_element(b.begin(), b.end()));
    }
    return bs;
}

/// eigensolver.hpp average_energy_per_cell
inline double average_energy_per_cell(const std::vector<double>& sorted_eigenvalues, Index cells, Index n_occ) {
    const Index take = n_occ * cells;
    if (take < 0 || take > static_cast<Index>(sorted_eigenvalues.size()))
        throw DimensionError("average_energy_per_cell: occupation exceeds spectrum size");
    double s = 0.0;
    for (Index i = 0; i < take; ++i) s += sorted_eigenvalues[static_cast<size_t>(i)];
    return s / static_cast<double>(cells);
}

/// tools/commands.cpp:51-59 + solve_periodic, fused on the device.
inline KPointSpectrum solve_core_periodic(Context& ctx, const LatticeSystem& sys, int64_t* info = nullptr) {
    SystemView v(sys);
    std::vector<double> flat(static_cast<size_t>(sys.basis_count()));
    check(lt_solve_core(ctx.get(), v.get(), 1, flat.data(), info));
    return make_spectrum(sys.L, sys.m0(), flat, "b200-core");
}

/// The whole path across the devices of `mctx` (split: LT_SPLIT_KPOINTS or LT_SPLIT_RANKTERMS);
/// the same KPointSpectrum as solve_core_periodic on one device.
inline KPointSpectrum solve_core_periodic(MultiContext& mctx, const LatticeSystem& sys, int split = LT_SPLIT_KPOINTS,
                                          int64_t* info = nullptr) {
    SystemView v(sys);
    std::vector<double> flat(static_cast<size_t>(sys.basis_count()));
    check(lt_solve_core_multi(mctx.get(), v.get(), 1, split, flat.data(), info));
    return make_spectrum(sys.L, sys.m0(), flat, "b200-core-multi");
}

/// tools/commands.cpp:51-59 + solve_box_dense, fused on the device.
inline DenseSpectrum solve_core_box(Context& ctx, const LatticeSystem& sys, int64_t* info = nullptr) {
    SystemView v(sys);
    DenseSpectrum d;
    d.eigenvalues.resize(static_cast<size_t>(sys.basis_count()));
    check(lt_solve_core(ctx.get(), v.get(), 0, d.eigenvalues.data(), info));
    return d;
}

}  // namespace latham_b200
