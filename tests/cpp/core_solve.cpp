// A reference-style client of the C++ mirror (include/latham_b200.hpp): the calls
// tools/commands.cpp makes for `latham solve` (assemble Laplace / Nuclear / Mass,
// H = combine(0.5, Lap, -1, Nuc), S = Mass, then the spectrum), plus the fused
// whole-path entry and the reference's error classes. Prints one line per result:
//   <tag> <count> <v1> <v2> ...   (%.17g)
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>

#include "latham_b200.hpp"

using namespace latham_b200;

static LatticeSystem chain(Index Lx, bool two_nuclei) {
    LatticeSystem s;
    s.b = 2.0;
    s.L = {Lx, 1, 1};
    s.set_grid(32, 32);
    s.quad_M = 8;
    s.nuclei.cell_size = s.b;
    if (two_nuclei) {
        s.nuclei.nuclei.push_back({{-0.5, 0.0, 0.0}, 1.0});
        s.nuclei.nuclei.push_back({{0.5, 0.0, 0.0}, 1.0});
    } else {
        s.nuclei.nuclei.push_back({{0.0, 0.0, 0.0}, 1.0});
    }
    for (const auto& nu : s.nuclei.nuclei) {
        s.basis.functions.push_back({nu.position, 1.3, {0, 0, 0}});
        s.basis.functions.push_back({nu.position, 3.1, {0, 0, 0}});
    }
    return s;
}

static void print(const std::string& tag, const std::vector<double>& v) {
    std::printf("%s %zu", tag.c_str(), v.size());
    for (double x : v) std::printf(" %.17g", x);
    std::printf("\n");
}

int main() {
    Context ctx(0);
    // periodic: reference-shaped calls
    const LatticeSystem per = chain(16, true);
    auto lap = assemble_periodic(ctx, per, OperatorKind::Laplace);
    auto nuc = assemble_periodic(ctx, per, OperatorKind::Nuclear);
    auto S = assemble_periodic(ctx, per, OperatorKind::Mass);
    auto H = combine(ctx, 0.5, lap, -1.0, nuc);
    print("periodic_ops", solve_periodic(ctx, H, S).sorted_all());
    print("periodic_core", solve_core_periodic(ctx, per).sorted_all());
    {
        // the multi-device entry over the devices of this box (one on the test box)
        MultiContext mctx({0});
        print("periodic_multi_k", solve_core_periodic(mctx, per, LT_SPLIT_KPOINTS).sorted_all());
        print("periodic_multi_r", solve_core_periodic(mctx, per, LT_SPLIT_RANKTERMS).sorted_all());
    }
    print("periodic_factorized", solve_periodic_factorized(ctx, H, S).sorted_all());
    std::printf("residual %.3g\n", separable_residual(ctx, H));
    // want_vectors: per-k blocks; one reconstructed column against bc_full_eigenvector
    const KPointSpectrum vs = solve_periodic(ctx, H, S, true);
    print("periodic_vec_eig", vs.sorted_all());
    const auto U = reconstruct_eigenvectors(ctx, vs);
    const auto u0 = bc_full_eigenvector(ctx, vs, 3, 1);
    double dev = 0.0;
    const Index N = vs.k_count() * vs.m0;
    for (Index i = 0; i < N; ++i) dev = std::max(dev, std::abs(U[static_cast<size_t>(i + (3 * vs.m0 + 1) * N)] - u0[static_cast<size_t>(i)]));
    std::printf("recon_col_dev %.3g\n", dev);
    // box
    const LatticeSystem box = chain(6, false);
    auto blap = assemble_box(ctx, box, OperatorKind::Laplace);
    auto bnuc = assemble_box(ctx, box, OperatorKind::Nuclear);
    auto bS = assemble_box(ctx, box, OperatorKind::Mass);
    auto bH = combine(ctx, 0.5, blap, -1.0, bnuc);
    print("box_ops", solve_box_dense(ctx, bH.dense(), bS.dense(), bH.basis_count()).eigenvalues);
    print("box_core", solve_core_box(ctx, box).eigenvalues);
    const DenseSpectrum bv = solve_box_dense(ctx, bH.dense(), bS.dense(), bH.basis_count(), 4096, true);
    print("box_vec_eig", bv.eigenvalues);
    print("box_vec", bv.eigenvectors);
    // errors: alias guard (galerkin.cpp:294-302) and the dense cap (eigensolver.cpp:17-19)
    try {
        assemble_periodic(ctx, chain(3, true), OperatorKind::Mass);
        std::printf("error_alias none\n");
    } catch (const StructureError& e) {
        std::printf("error_alias StructureError %s\n", e.what());
    }
    try {
        solve_box_dense(ctx, bH.dense(), bS.dense(), bH.basis_count(), 4);
        std::printf("error_cap none\n");
    } catch (const ResourceCapError& e) {
        std::printf("error_cap ResourceCapError %s\n", e.what());
    }
    return 0;
}
