// plan.cpp — host-side planning: validation and the integer bookkeeping of the
// reference's AssemblyContext (galerkin.cpp:19-30, :287-307), grid extents
// (newton_kernel.cpp:54-73), window starts and bounds (newton_kernel.cpp:81-95,
// :120-151). O(M0 + m0) integer work; every O(grid) step runs on the device.
#include <algorithm>
#include <cmath>
#include <string>

#include "lt_internal.cuh"

namespace lt {

HostSys host_sys_from(const lt_system* s) {
    if (!s) fail(LT_EDIM, "null system");
    HostSys h;
    h.b = s->b;
    for (int l = 0; l < 3; ++l) {
        h.L[l] = s->L[l];
        h.n[l] = s->n[l];
        h.nbar[l] = s->nbar[l];
    }
    h.quad_M = s->quad_M;
    h.eps_ov = s->eps_ov;
    if (s->n_nuclei < 0 || s->m0 < 0) fail(LT_EDIM, "LatticeSystem: negative counts");
    h.pos.assign(s->nuc_pos, s->nuc_pos + 3 * s->n_nuclei);
    h.Z.assign(s->nuc_charge, s->nuc_charge + s->n_nuclei);
    h.center.assign(s->bf_center, s->bf_center + 3 * s->m0);
    h.alpha.assign(s->bf_alpha, s->bf_alpha + s->m0);
    h.deg.assign(s->bf_deg, s->bf_deg + 3 * s->m0);
    return h;
}

// galerkin.cpp:19-30 with NucleiSet::validate (newton_kernel.cpp:5-20) and
// GtoBasis::validate (gto_basis.cpp:16-23); same order and messages
void validate(const HostSys& s) {
    if (s.b <= 0.0) fail(LT_EDIM, "LatticeSystem: b must be positive");
    for (int l = 0; l < 3; ++l)
        if (s.n[l] < 1 || s.nbar[l] < 1) fail(LT_EDIM, "LatticeSystem: n and nbar must be >= 1");
    if (s.quad_M < 1) fail(LT_EDIM, "LatticeSystem: quadrature half-count must be >= 1");
    for (int l = 0; l < 3; ++l)
        if (s.L[l] < 1) fail(LT_EDIM, "LatticeSystem: lattice counts must be >= 1");
    if (s.eps_ov <= 0.0) fail(LT_EDIM, "LatticeSystem: eps_ov must be positive");
    if (s.Z.empty()) fail(LT_ESTRUCT, "NucleiSet: no nuclei");
    for (size_t i = 0; i < s.Z.size(); ++i) {
        if (s.Z[i] <= 0.0) fail(LT_ESTRUCT, "NucleiSet: charges must be positive");
        for (int l = 0; l < 3; ++l)
            if (std::abs(s.pos[3 * i + l]) > 0.5 * s.b) fail(LT_EBOUNDS, "NucleiSet: nucleus outside the unit cell");
    }
    if (s.alpha.empty()) fail(LT_ESTRUCT, "GtoBasis: no functions");
    for (size_t m = 0; m < s.alpha.size(); ++m) {
        if (s.alpha[m] <= 0.0) fail(LT_ESTRUCT, "GtoBasis: exponents must be positive");
        for (int l = 0; l < 3; ++l)
            if (s.deg[3 * m + l] < 0) fail(LT_ESTRUCT, "GtoBasis: monomial degrees must be >= 0");
    }
}

Index master_rows_box(Index n, Index L, Index margin) {
    const Index NL = n * L;
    const Index win = NL + 2 * margin * n;
    const Index shift_range = (NL + 1) / 2 + n;
    return win + 2 * shift_range;
}

Index master_rows_periodic(Index n, Index L) { return n + 2 * (n * (L / 2) + n); }

Index window_start(Index master_n, Index win_n, double a, double h) {
    if ((master_n - win_n) % 2 != 0)
        fail(LT_ESTRUCT, "window_start: master and window sizes differ by an odd count");
    const double offset = a / h;
    const auto rounded = static_cast<Index>(std::llround(offset));
    return (master_n - win_n) / 2 - rounded;
}

static void check_window(Index start, Index win_n, Index master_n, const char* what) {
    if (start < 0 || start + win_n > master_n)
        fail(LT_EBOUNDS, std::string(what) + ": window [" + std::to_string(start) + ", " +
                             std::to_string(start + win_n) + ") outside master extent " + std::to_string(master_n));
}

void plan_after_L0(const HostSys& s, bool periodic, Index L0, Plan& p, bool need_potential, bool check_alias) {
    p.periodic = periodic;
    p.m0 = s.m0();
    p.nnuc = s.nnuc();
    p.M = s.quad_M;
    p.RN = 2 * s.quad_M + 1;
    p.Rtot = p.RN * p.nnuc;
    p.L0 = L0;
    p.margin = L0 + 2;  // galerkin.cpp:293
    if (periodic && check_alias)
        for (int l = 0; l < 3; ++l) {
            const Index Ll = s.L[l];
            if (Ll > 1 && Ll <= 2 * L0)
                fail(LT_ESTRUCT, "assemble_periodic: L" + std::to_string(l + 1) + " = " + std::to_string(Ll) +
                                     " must exceed 2*L0 = " + std::to_string(2 * L0) +
                                     " or generating blocks alias their wrap images");
        }
    p.cells = s.cells();
    p.Nb = p.m0 * p.cells;
    p.K = periodic ? p.cells : 1;
    p.nontrivial = 0;
    p.nblocks = 1;
    for (int l = 0; l < 3; ++l) {
        DirPlan& d = p.d[l];
        d.L = s.L[l];
        d.n = s.n[l];
        d.nbar = s.nbar[l];
        d.h = s.h(l);
        d.hbar = s.hbar(l);
        d.band = std::min(L0, d.L - 1);  // galerkin.cpp:15, :205
        d.width = 2 * d.band + 1;
        d.G = (d.L + 2 * p.margin) * d.n;
        d.Gbar = (d.L + 2 * p.margin) * d.nbar;
        if (d.L > 1) ++p.nontrivial;
        p.nblocks *= d.width;
        const bool wrapped = periodic && d.L > 1;
        d.tiled = wrapped;
        d.mode = d.L == 1 ? TM_TRIVIAL : (periodic ? TM_FOLD : TM_BOXDIR);
        d.npairs = d.mode == TM_TRIVIAL ? 1 : (d.mode == TM_FOLD ? d.width : d.L * d.width);
        // potential panel (galerkin.cpp:151-198; newton_kernel.cpp:120-181)
        const Index Lsum = wrapped ? d.L : (periodic ? 1 : d.L);
        d.nsum = Lsum;
        if (wrapped) {
            d.mrows = master_rows_periodic(d.n, d.L);
            d.pot_rows = d.n;
        } else {
            d.mrows = master_rows_box(d.n, Lsum, p.margin);
            d.pot_rows = d.n * Lsum + 2 * p.margin * d.n;
        }
        d.s0.clear();
        if (need_potential) {
            const char* what = wrapped ? "lattice_potential_periodic_cell" : "lattice_potential_box";
            for (Index v = 0; v < p.nnuc; ++v) {
                double base_a = s.pos[3 * v + l];
                Index k_lo = 0;
                if (wrapped) k_lo = -(Lsum / 2);
                else base_a -= 0.5 * static_cast<double>(Lsum - 1) * static_cast<double>(d.n) * d.h;
                const Index base = window_start(d.mrows, d.pot_rows, base_a, d.h);
                Index smin = base - d.n * k_lo, smax = smin;
                for (Index k = 0; k < Lsum; ++k) {
                    const Index sk = base - d.n * (k_lo + k);
                    smin = std::min(smin, sk);
                    smax = std::max(smax, sk);
                }
                check_window(smin, d.pot_rows, d.mrows, what);
                check_window(smax, d.pot_rows, d.mrows, what);
                d.s0.push_back(smin);
            }
        }
    }
    p.s2_dir = -1;
    if (!periodic && p.nontrivial == 1)
        for (int l = 0; l < 3; ++l)
            if (p.d[l].L > 1) p.s2_dir = l;
}

}  // namespace lt
