// oracle/latham_oracle.cpp — TEST INFRASTRUCTURE ONLY (Oracle-X).
//
// Clean-room CPU restatement of the reference hot path (arXiv 1408.3839 C++
// reference under /root/reference/proj/core), used by tests/ as the parity checker
// and by bench.py as the CPU baseline. It is never linked into the product.
// Every function cites the reference file:line it restates. Arithmetic is kept in
// the reference's evaluation order wherever the order changes the rounding.
//
// Generalisation: the grid counts n, nbar are per
// direction; h_l = b / n_l. With isotropic n every step reduces to the reference.
// L0 is the reference scan with direction l sampled on its own n_l grid
// (gto_basis.cpp:87-126 evaluated per direction, max over directions inside the
// same s loop).
#include "latham_oracle.h"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <numbers>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "linalg.hpp"

namespace orc {

using Index = std::int64_t;
using Cplx = std::complex<double>;

// errors.hpp:10-43
struct Err : std::runtime_error {
    int code;
    Err(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void fail(int code, const std::string& m) { throw Err(code, m); }

// column-major dense matrix (Eigen::MatrixXd default storage)
struct Mat {
    Index rows = 0, cols = 0;
    std::vector<double> a;
    Mat() = default;
    Mat(Index r, Index c) : rows(r), cols(c), a(static_cast<size_t>(r * c), 0.0) {}
    double& operator()(Index i, Index j) { return a[static_cast<size_t>(i + j * rows)]; }
    double operator()(Index i, Index j) const { return a[static_cast<size_t>(i + j * rows)]; }
};

struct Gto {
    std::array<double, 3> c{};
    double alpha = 1.0;
    std::array<int, 3> deg{};
    // gto_basis.cpp:9-14
    double eval1d(int dir, double x) const {
        const double d = x - c[dir];
        double mono = 1.0;
        for (int p = 0; p < deg[dir]; ++p) mono *= d;
        return mono * std::exp(-alpha * d * d);
    }
};

struct Sys {
    double b = 0;
    std::array<Index, 3> L{1, 1, 1}, n{}, nbar{};
    Index M = 0;
    double eps_ov = 1e-8;
    std::vector<std::array<double, 3>> pos;
    std::vector<double> Z;
    std::vector<Gto> basis;
    double h(int l) const { return b / static_cast<double>(n[l]); }
    double hbar(int l) const { return b / static_cast<double>(nbar[l]); }
    Index m0() const { return static_cast<Index>(basis.size()); }
    Index cells() const { return L[0] * L[1] * L[2]; }
};

Sys from_c(const or_system* s) {
    Sys o;
    o.b = s->b;
    for (int l = 0; l < 3; ++l) {
        o.L[l] = s->L[l];
        o.n[l] = s->n[l];
        o.nbar[l] = s->nbar[l];
    }
    o.M = s->quad_M;
    o.eps_ov = s->eps_ov;
    for (Index i = 0; i < s->n_nuclei; ++i) {
        o.pos.push_back({s->nuc_pos[3 * i], s->nuc_pos[3 * i + 1], s->nuc_pos[3 * i + 2]});
        o.Z.push_back(s->nuc_charge[i]);
    }
    for (Index i = 0; i < s->m0; ++i) {
        Gto g;
        for (int l = 0; l < 3; ++l) {
            g.c[l] = s->bf_center[3 * i + l];
            g.deg[l] = s->bf_deg[3 * i + l];
        }
        g.alpha = s->bf_alpha[i];
        o.basis.push_back(g);
    }
    return o;
}

// galerkin.cpp:19-30 + newton_kernel.cpp:5-20 + gto_basis.cpp:16-23
void validate(const Sys& s) {
    if (s.b <= 0.0) fail(OR_EDIM, "LatticeSystem: b must be positive");
    for (int l = 0; l < 3; ++l)
        if (s.n[l] < 1 || s.nbar[l] < 1) fail(OR_EDIM, "LatticeSystem: n and nbar must be >= 1");
    if (s.M < 1) fail(OR_EDIM, "LatticeSystem: quadrature half-count must be >= 1");
    for (Index l : s.L)
        if (l < 1) fail(OR_EDIM, "LatticeSystem: lattice counts must be >= 1");
    if (s.eps_ov <= 0.0) fail(OR_EDIM, "LatticeSystem: eps_ov must be positive");
    if (s.pos.empty()) fail(OR_ESTRUCT, "NucleiSet: no nuclei");
    for (size_t i = 0; i < s.pos.size(); ++i) {
        if (s.Z[i] <= 0.0) fail(OR_ESTRUCT, "NucleiSet: charges must be positive");
        for (double a : s.pos[i])
            if (std::abs(a) > 0.5 * s.b) fail(OR_EBOUNDS, "NucleiSet: nucleus outside the unit cell");
    }
    if (s.basis.empty()) fail(OR_ESTRUCT, "GtoBasis: no functions");
    for (const auto& g : s.basis) {
        if (g.alpha <= 0.0) fail(OR_ESTRUCT, "GtoBasis: exponents must be positive");
        for (int d : g.deg)
            if (d < 0) fail(OR_ESTRUCT, "GtoBasis: monomial degrees must be >= 0");
    }
}

// ---------------------------------------------------------------------------
// sinc_quadrature.cpp:9-29
// ---------------------------------------------------------------------------
void sinc(Index M, std::vector<double>& t, std::vector<double>& w) {
    if (M < 1) fail(OR_EDIM, "build_sinc_quadrature: M must be >= 1");
    double step = std::log(static_cast<double>(M)) / static_cast<double>(M);
    if (M == 1) step = 0.5;
    const Index R = 2 * M + 1;
    t.resize(R);
    w.resize(R);
    const double c = 2.0 * step / std::sqrt(std::numbers::pi);
    for (Index i = 0; i < R; ++i) {
        const double u = static_cast<double>(i - M) * step;
        const double eu = std::exp(-u);
        t[i] = std::exp(u - eu);
        w[i] = c * (t[i] + std::exp(-eu));
    }
}

// ---------------------------------------------------------------------------
// newton_kernel.cpp:22-45 on one centred cell grid (grid.hpp:28-38)
// ---------------------------------------------------------------------------
void master_column(Index ncells, double h, double t, double* f) {
    const double origin = -0.5 * static_cast<double>(ncells) * h;
    const double c = std::sqrt(std::numbers::pi) / (2.0 * t);
    double e_left = std::erf(t * (origin + static_cast<double>(0) * h));
    for (Index i = 0; i < ncells; ++i) {
        const double e_right = std::erf(t * (origin + static_cast<double>(i + 1) * h));
        f[i] = c * (e_right - e_left);
        e_left = e_right;
    }
}

Mat master_panel(Index ncells, double h, const std::vector<double>& t) {
    Mat m(ncells, static_cast<Index>(t.size()));
    for (size_t q = 0; q < t.size(); ++q) master_column(ncells, h, t[q], &m.a[q * ncells]);
    return m;
}

// newton_kernel.cpp:54-64 (one direction)
Index master_rows_box(Index n, Index L, Index margin) {
    const Index NL = n * L;
    const Index win = NL + 2 * margin * n;
    const Index shift_range = (NL + 1) / 2 + n;
    return win + 2 * shift_range;
}
// newton_kernel.cpp:66-73 (one direction)
Index master_rows_periodic(Index n, Index L) { return n + 2 * (n * (L / 2) + n); }

// newton_kernel.cpp:81-95
Index window_start(Index master_n, Index win_n, double a, double h) {
    if ((master_n - win_n) % 2 != 0)
        fail(OR_ESTRUCT, "window_start: master and window sizes differ by an odd count");
    const double offset = a / h;
    const auto rounded = static_cast<Index>(std::llround(offset));
    return (master_n - win_n) / 2 - rounded;
}
void check_window(Index start, Index win_n, Index master_n, const char* what) {
    if (start < 0 || start + win_n > master_n)
        fail(OR_EBOUNDS, std::string(what) + ": window [" + std::to_string(start) + ", " +
                             std::to_string(start + win_n) + ") outside master extent " +
                             std::to_string(master_n));
}

// canonical_tensor.cpp:112-164 (one direction; uniform progressions by running sums)
Mat assembled_window_sum(const Mat& m, const std::vector<Index>& sh, Index size) {
    if (sh.empty()) fail(OR_ESTRUCT, "assembled_window_sum: empty shift set");
    for (Index s : sh)
        if (s < 0 || s + size > m.rows)
            fail(OR_EBOUNDS, "assembled_window_sum: shift " + std::to_string(s) + " outside master extent " +
                                 std::to_string(m.rows));
    Mat acc(size, m.cols);
    bool uniform = sh.size() >= 2;
    Index step = 0;
    if (uniform) {
        step = sh[1] - sh[0];
        if (step <= 0) uniform = false;
        for (size_t i = 2; uniform && i < sh.size(); ++i)
            if (sh[i] - sh[i - 1] != step) uniform = false;
    }
    if (uniform) {
        const Index s0 = sh.front();
        const Index nsh = static_cast<Index>(sh.size());
        for (Index q = 0; q < m.cols; ++q) {
            for (Index i = 0; i < std::min(step, size); ++i) {
                double sum = 0.0;
                for (Index k = 0; k < nsh; ++k) sum += m(s0 + i + k * step, q);
                acc(i, q) = sum;
            }
            for (Index i = step; i < size; ++i)
                acc(i, q) = acc(i - step, q) + m(s0 + i + (nsh - 1) * step, q) - m(s0 + i - step, q);
        }
    } else {
        for (Index s : sh)
            for (Index q = 0; q < m.cols; ++q)
                for (Index i = 0; i < size; ++i) acc(i, q) += m(s + i, q);
    }
    return acc;
}

// newton_kernel.cpp:120-151, one direction of one nucleus
Mat assemble_nucleus_dir(const Mat& master, double a, Index L, Index n, double h, Index win_n,
                         bool centered, const char* what) {
    double base_a = a;
    Index k_lo = 0;
    if (centered) k_lo = -(L / 2);
    else base_a -= 0.5 * static_cast<double>(L - 1) * static_cast<double>(n) * h;
    const Index base = window_start(master.rows, win_n, base_a, h);
    std::vector<Index> s(static_cast<size_t>(L));
    for (Index k = 0; k < L; ++k) s[k] = base - n * (k_lo + k);
    std::sort(s.begin(), s.end());
    check_window(s.front(), win_n, master.rows, what);
    check_window(s.back(), win_n, master.rows, what);
    return assembled_window_sum(master, s, win_n);
}

// concat_sum (canonical_tensor.cpp:166-187) of per-nucleus panels for direction l
Mat concat_cols(const std::vector<Mat>& parts) {
    Index cols = 0;
    for (const auto& p : parts) cols += p.cols;
    Mat out(parts.front().rows, cols);
    Index at = 0;
    for (const auto& p : parts) {
        std::copy(p.a.begin(), p.a.end(), out.a.begin() + at * out.rows);
        at += p.cols;
    }
    return out;
}

// ---------------------------------------------------------------------------
// gto_basis.cpp:31-47
// ---------------------------------------------------------------------------
struct Supp {
    Index offset = 0;
    std::vector<double> v;
    Index end() const { return offset + static_cast<Index>(v.size()); }
};

Supp sample_gto_1d(const Gto& fn, int dir, Index grid_n, double step, Index cell_index, Index per_cell,
                   double b, double align, double eps) {
    std::vector<double> full(static_cast<size_t>(grid_n));
    const Index base = cell_index * per_cell;
    for (Index i = 0; i < grid_n; ++i) {
        const double x = (static_cast<double>(i - base) + align) * step - 0.5 * b;
        full[i] = fn.eval1d(dir, x);
    }
    Index lo = 0, hi = grid_n;
    while (lo < hi && std::abs(full[lo]) < eps) ++lo;
    while (hi > lo && std::abs(full[hi - 1]) < eps) --hi;
    if (lo == hi) return Supp{0, {}};
    return Supp{lo, std::vector<double>(full.begin() + lo, full.begin() + hi)};
}

// gto_basis.cpp:87-126, per-direction grids
Index overlap_constant(const Sys& s) {
    const Index m0 = s.m0();
    constexpr Index kMaxL0 = 256;
    std::vector<std::array<Supp, 3>> prof(static_cast<size_t>(m0));
    for (Index m = 0; m < m0; ++m)
        for (int l = 0; l < 3; ++l) {
            const Index width = 2 * (kMaxL0 + 2) * s.n[l];
            prof[m][l] = sample_gto_1d(s.basis[m], l, width, s.h(l), kMaxL0 + 2, s.n[l], s.b, 0.5, 0.0);
        }
    Index L0 = 0, misses = 0;
    for (Index sft = 1; sft <= kMaxL0 && misses < 2; ++sft) {
        double worst = 0.0;
        for (Index mu = 0; mu < m0; ++mu)
            for (Index nu = 0; nu < m0; ++nu)
                for (int l = 0; l < 3; ++l) {
                    const Supp& a = prof[mu][l];
                    const Supp& c = prof[nu][l];
                    const Index off = c.offset + sft * s.n[l];
                    const Index lo = std::max(a.offset, off);
                    const Index hi = std::min(a.end(), off + static_cast<Index>(c.v.size()));
                    for (Index i = lo; i < hi; ++i)
                        worst = std::max(worst, std::abs(a.v[i - a.offset] * c.v[i - off]));
                }
        if (worst >= s.eps_ov) {
            L0 = sft;
            misses = 0;
        } else {
            ++misses;
        }
    }
    return L0;
}

// fem1d.cpp:19-32
double tri_form(const Supp& u, const Supp& v, double lo, double diag) {
    const Index lo_i = std::max(u.offset, v.offset - 1);
    const Index hi_i = std::min(u.end(), v.end() + 1);
    double s = 0.0;
    for (Index i = lo_i; i < hi_i; ++i) {
        const double ui = u.v[i - u.offset];
        double row = 0.0;
        if (i - 1 >= v.offset && i - 1 < v.end()) row += lo * v.v[i - 1 - v.offset];
        if (i >= v.offset && i < v.end()) row += diag * v.v[i - v.offset];
        if (i + 1 >= v.offset && i + 1 < v.end()) row += lo * v.v[i + 1 - v.offset];
        s += ui * row;
    }
    return s;
}

// ---------------------------------------------------------------------------
// galerkin.cpp: assembly
// ---------------------------------------------------------------------------
constexpr double kTrimEps = 1e-280;  // galerkin.cpp:13
enum Kind { Laplace = 0, Mass = 1, Nuclear = 2 };

struct Ctx {
    const Sys* sys = nullptr;
    bool periodic = false;
    Index L0 = 0, margin = 0;
    std::array<Index, 3> band{};
    std::vector<std::array<Supp, 3>> pwc, pwl;
    std::array<double, 3> fem_h{};
    std::array<Mat, 3> pot;
    std::array<bool, 3> tiled{};
    std::vector<double> pot_w;
    std::array<std::vector<Mat>, 3> massT, stiffT, nucT;
    Index pair_index(int l, Index k, Index d) const {
        const Index width = 2 * band[l] + 1;
        return periodic ? (d + band[l]) : (k * width + d + band[l]);
    }
};

// galerkin.cpp:109-125
double dot3(const Supp& a, Index shA, const Supp& b, Index shB, const Mat& p, Index col, bool tiled,
            Index tile_n) {
    const Index offA = a.offset + shA, offB = b.offset + shB;
    Index lo = std::max(offA, offB);
    Index hi = std::min(offA + static_cast<Index>(a.v.size()), offB + static_cast<Index>(b.v.size()));
    if (!tiled) {
        lo = std::max<Index>(lo, 0);
        hi = std::min<Index>(hi, p.rows);
    }
    double s = 0.0;
    for (Index i = lo; i < hi; ++i) {
        const double pv = tiled ? p(i % tile_n, col) : p(i, col);
        s += a.v[i - offA] * b.v[i - offB] * pv;
    }
    return s;
}

// galerkin.cpp:127-149
void build_profiles(Ctx& c) {
    const Sys& s = *c.sys;
    c.pwc.resize(s.m0());
    c.pwl.resize(s.m0());
    for (Index m = 0; m < s.m0(); ++m)
        for (int l = 0; l < 3; ++l) {
            const Index cells = s.L[l] + 2 * c.margin;
            c.pwc[m][l] = sample_gto_1d(s.basis[m], l, cells * s.n[l], s.h(l), c.margin, s.n[l], s.b, 0.5, kTrimEps);
            c.pwl[m][l] =
                sample_gto_1d(s.basis[m], l, cells * s.nbar[l], s.hbar(l), c.margin, s.nbar[l], s.b, 0.0, kTrimEps);
        }
    for (int l = 0; l < 3; ++l) c.fem_h[l] = s.hbar(l);
}

// galerkin.cpp:151-198 (+ newton_kernel.cpp:155-181)
void build_potential(Ctx& c) {
    const Sys& s = *c.sys;
    std::vector<double> t, w;
    sinc(s.M, t, w);
    const Index nn = static_cast<Index>(s.pos.size());
    for (int l = 0; l < 3; ++l) {
        const double h = s.h(l);
        const Index n = s.n[l];
        std::vector<Mat> parts;
        if (!c.periodic || s.L[l] == 1) {
            // box lattice (or the open direction of a periodic system: unit lattice)
            const Index Ll = c.periodic ? 1 : s.L[l];
            const Index mrows = master_rows_box(n, Ll, c.margin);
            const Mat master = master_panel(mrows, h, t);
            const Index win = n * Ll + 2 * c.margin * n;
            for (Index v = 0; v < nn; ++v)
                parts.push_back(assemble_nucleus_dir(master, s.pos[v][l], Ll, n, h, win, false, "lattice_potential_box"));
            c.tiled[l] = false;
        } else {
            const Index mrows = master_rows_periodic(n, s.L[l]);
            const Mat master = master_panel(mrows, h, t);
            for (Index v = 0; v < nn; ++v)
                parts.push_back(assemble_nucleus_dir(master, s.pos[v][l], s.L[l], n, h, n, true,
                                                     "lattice_potential_periodic_cell"));
            c.tiled[l] = true;
        }
        c.pot[l] = concat_cols(parts);
    }
    // weights: nucleus-major Z_nu * w_q (canonical_tensor.cpp:40-44 scaled, :166-187)
    c.pot_w.clear();
    for (Index v = 0; v < nn; ++v)
        for (double wq : w) c.pot_w.push_back(wq * s.Z[v]);
}

// galerkin.cpp:200-250
void build_tables(Ctx& c, Kind which) {
    const Sys& s = *c.sys;
    const Index m0 = s.m0();
    for (int l = 0; l < 3; ++l) {
        c.band[l] = std::min(c.L0, s.L[l] - 1);
        const Index width = 2 * c.band[l] + 1;
        if (which != Nuclear) {
            const double h = c.fem_h[l];
            const double mlo = h / 6.0, mdiag = 4.0 * h / 6.0, slo = -1.0 / h, sdiag = 2.0 / h;
            c.massT[l].assign(width, Mat(m0, m0));
            c.stiffT[l].assign(width, Mat(m0, m0));
            for (Index d = -c.band[l]; d <= c.band[l]; ++d) {
                Mat ms(m0, m0), st(m0, m0);
                for (Index mu = 0; mu < m0; ++mu)
                    for (Index nu = 0; nu < m0; ++nu) {
                        const Supp& a = c.pwl[mu][l];
                        Supp bb = c.pwl[nu][l];
                        bb.offset += d * s.nbar[l];
                        ms(mu, nu) = tri_form(a, bb, mlo, mdiag);
                        st(mu, nu) = tri_form(a, bb, slo, sdiag);
                    }
                c.massT[l][d + c.band[l]] = ms;
                c.stiffT[l][d + c.band[l]] = st;
            }
        } else {
            const Index rank = static_cast<Index>(c.pot_w.size());
            const Index kk = c.periodic ? 1 : s.L[l];
            c.nucT[l].assign(kk * width * rank, Mat(m0, m0));
            for (Index k = 0; k < kk; ++k)
                for (Index d = -c.band[l]; d <= c.band[l]; ++d) {
                    const Index m_cell = k + d;
                    if (!c.periodic && (m_cell < 0 || m_cell >= s.L[l])) continue;
                    const Index pair = c.pair_index(l, k, d);
                    for (Index r = 0; r < rank; ++r) {
                        Mat blk(m0, m0);
                        for (Index mu = 0; mu < m0; ++mu)
                            for (Index nu = 0; nu < m0; ++nu)
                                blk(mu, nu) = dot3(c.pwc[mu][l], (c.periodic ? 0 : k) * s.n[l], c.pwc[nu][l],
                                                   (c.periodic ? d : m_cell) * s.n[l], c.pot[l], r, c.tiled[l], s.n[l]);
                        c.nucT[l][pair * rank + r] = blk;
                    }
                }
        }
    }
}

// galerkin.cpp:252-285
Mat combine_block(const Ctx& c, Kind which, const std::array<Index, 3>& k, const std::array<Index, 3>& d) {
    const Index m0 = c.sys->m0();
    Mat out(m0, m0);
    if (which == Mass) {
        const Mat& a = c.massT[0][d[0] + c.band[0]];
        const Mat& b = c.massT[1][d[1] + c.band[1]];
        const Mat& e = c.massT[2][d[2] + c.band[2]];
        for (size_t i = 0; i < out.a.size(); ++i) out.a[i] = a.a[i] * b.a[i] * e.a[i];
        return out;
    }
    if (which == Laplace) {
        for (int dir = 0; dir < 3; ++dir) {
            std::vector<double> term(out.a.size(), 1.0);
            for (int l = 0; l < 3; ++l) {
                const Mat& t = (l == dir ? c.stiffT[l] : c.massT[l])[d[l] + c.band[l]];
                for (size_t i = 0; i < term.size(); ++i) term[i] = term[i] * t.a[i];
            }
            for (size_t i = 0; i < term.size(); ++i) out.a[i] += term[i];
        }
        return out;
    }
    const Index rank = static_cast<Index>(c.pot_w.size());
    for (Index r = 0; r < rank; ++r) {
        const Mat& t1 = c.nucT[0][c.pair_index(0, k[0], d[0]) * rank + r];
        const Mat& t2 = c.nucT[1][c.pair_index(1, k[1], d[1]) * rank + r];
        const Mat& t3 = c.nucT[2][c.pair_index(2, k[2], d[2]) * rank + r];
        const double w = c.pot_w[r];
        for (size_t i = 0; i < out.a.size(); ++i) out.a[i] += w * (t1.a[i] * t2.a[i] * t3.a[i]);
    }
    return out;
}

// galerkin.cpp:287-307
Ctx make_context(const Sys& s, bool periodic, Kind which) {
    validate(s);
    Ctx c;
    c.sys = &s;
    c.periodic = periodic;
    c.L0 = overlap_constant(s);
    c.margin = c.L0 + 2;
    if (periodic)
        for (int l = 0; l < 3; ++l) {
            const Index Ll = s.L[l];
            if (Ll > 1 && Ll <= 2 * c.L0)
                fail(OR_ESTRUCT, "assemble_periodic: L" + std::to_string(l + 1) + " = " + std::to_string(Ll) +
                                     " must exceed 2*L0 = " + std::to_string(2 * c.L0) +
                                     " or generating blocks alias their wrap images");
        }
    build_profiles(c);
    if (which == Nuclear) build_potential(c);
    build_tables(c, which);
    return c;
}

using GenMap = std::map<std::array<Index, 3>, Mat>;  // block_circulant.hpp:47

struct Op {
    int which = 0;
    bool periodic = false;
    Index m0 = 0;
    std::array<Index, 3> L{1, 1, 1};
    std::array<Index, 3> band{};
    Mat dense;
    GenMap gen;
    std::vector<std::array<std::vector<Mat>, 3>> separable;
    Index coefficient_rank = 0, L0 = 0;
};

// galerkin.cpp:311-358
Op assemble_box(const Sys& s, Kind which) {
    Ctx c = make_context(s, false, which);
    const Index m0 = s.m0(), cells = s.cells(), Nb = m0 * cells;
    Op op;
    op.which = which;
    op.periodic = false;
    op.m0 = m0;
    op.L = s.L;
    op.band = c.band;
    op.L0 = c.L0;
    op.coefficient_rank = which == Mass ? 1 : which == Laplace ? 3 : static_cast<Index>(c.pot_w.size());
    op.dense = Mat(Nb, Nb);
    const Index max_row_blocks = (2 * c.L0 + 1) * (2 * c.L0 + 1) * (2 * c.L0 + 1);
    for (Index lin = 0; lin < cells; ++lin) {
        const std::array<Index, 3> k{lin / (s.L[1] * s.L[2]), (lin / s.L[2]) % s.L[1], lin % s.L[2]};
        Index row_blocks = 0;
        std::array<Index, 3> d{};
        for (d[0] = -c.band[0]; d[0] <= c.band[0]; ++d[0])
            for (d[1] = -c.band[1]; d[1] <= c.band[1]; ++d[1])
                for (d[2] = -c.band[2]; d[2] <= c.band[2]; ++d[2]) {
                    std::array<Index, 3> m{};
                    bool in_range = true;
                    for (int l = 0; l < 3; ++l) {
                        m[l] = k[l] + d[l];
                        in_range = in_range && m[l] >= 0 && m[l] < s.L[l];
                    }
                    if (!in_range) continue;
                    const Index mlin = (m[0] * s.L[1] + m[1]) * s.L[2] + m[2];
                    const Mat blk = combine_block(c, which, k, d);
                    for (Index j = 0; j < m0; ++j)
                        for (Index i = 0; i < m0; ++i) op.dense(lin * m0 + i, mlin * m0 + j) = blk(i, j);
                    ++row_blocks;
                }
        if (row_blocks > max_row_blocks)
            fail(OR_ESTRUCT, "assemble_box: block row " + std::to_string(lin) + " exceeds the (2 L0 + 1)^3 band bound");
    }
    return op;
}

// galerkin.cpp:360-425
Op assemble_periodic(const Sys& s, Kind which) {
    Ctx c = make_context(s, true, which);
    const Index m0 = s.m0();
    Op op;
    op.which = which;
    op.periodic = true;
    op.m0 = m0;
    op.L = s.L;
    op.band = c.band;
    op.L0 = c.L0;
    std::array<Index, 3> d{};
    Index distinct = 0;
    for (d[0] = -c.band[0]; d[0] <= c.band[0]; ++d[0])
        for (d[1] = -c.band[1]; d[1] <= c.band[1]; ++d[1])
            for (d[2] = -c.band[2]; d[2] <= c.band[2]; ++d[2]) {
                Mat blk = combine_block(c, which, {0, 0, 0}, d);
                std::array<Index, 3> kidx{};
                for (int l = 0; l < 3; ++l) kidx[l] = ((d[l] % s.L[l]) + s.L[l]) % s.L[l];
                if (d[0] >= 0 && d[1] >= 0 && d[2] >= 0) ++distinct;
                op.gen[kidx] = blk;
            }
    const Index bound = (c.L0 + 1) * (c.L0 + 1) * (c.L0 + 1);
    if (distinct > bound) fail(OR_ESTRUCT, "assemble_periodic: distinct offset magnitudes exceed the (L0+1)^3 bound");
    const Index rank = which == Mass ? 1 : which == Laplace ? 3 : static_cast<Index>(c.pot_w.size());
    op.coefficient_rank = rank;
    for (Index r = 0; r < rank; ++r) {
        std::array<std::vector<Mat>, 3> term;
        for (int l = 0; l < 3; ++l) {
            const Index Ll = s.L[l];
            term[l].assign(Ll, Mat(m0, m0));
            for (Index dd = -c.band[l]; dd <= c.band[l]; ++dd) {
                if (Ll == 1 && dd != 0) continue;
                const Index kidx = ((dd % Ll) + Ll) % Ll;
                Mat blk;
                if (which == Mass) blk = c.massT[l][dd + c.band[l]];
                else if (which == Laplace) blk = (l == static_cast<int>(r) ? c.stiffT : c.massT)[l][dd + c.band[l]];
                else {
                    blk = c.nucT[l][c.pair_index(l, 0, dd) * static_cast<Index>(c.pot_w.size()) + r];
                    if (l == 0)
                        for (double& x : blk.a) x *= c.pot_w[r];
                }
                term[l][kidx] = blk;
            }
        }
        op.separable.push_back(std::move(term));
    }
    return op;
}

// eigensolver.cpp:37-67
Op combine(double wa, const Op& a, double wb, const Op& b) {
    if (a.periodic != b.periodic || a.m0 != b.m0 || a.L != b.L)
        fail(OR_ESTRUCT, "combine: operators have different layouts");
    Op out;
    out.which = a.which;
    out.periodic = a.periodic;
    out.m0 = a.m0;
    out.L = a.L;
    out.band = a.band;
    out.L0 = std::max(a.L0, b.L0);
    out.coefficient_rank = a.coefficient_rank + b.coefficient_rank;
    if (!a.periodic) {
        out.dense = Mat(a.dense.rows, a.dense.cols);
        for (size_t i = 0; i < out.dense.a.size(); ++i) out.dense.a[i] = wa * a.dense.a[i] + wb * b.dense.a[i];
        return out;
    }
    for (const auto& [k, blk] : a.gen) {
        Mat o(a.m0, a.m0);
        auto it = b.gen.find(k);
        for (size_t i = 0; i < o.a.size(); ++i) o.a[i] = wa * blk.a[i] + wb * (it == b.gen.end() ? 0.0 : it->second.a[i]);
        out.gen[k] = o;
    }
    for (const auto& [k, blk] : b.gen)
        if (!a.gen.count(k)) {
            Mat o(a.m0, a.m0);
            for (size_t i = 0; i < o.a.size(); ++i) o.a[i] = wb * blk.a[i];
            out.gen[k] = o;
        }
    auto scaled = [&](double w, const Op& op) {
        for (auto t : op.separable) {
            for (auto& blk : t[0])
                for (double& x : blk.a) x *= w;
            out.separable.push_back(std::move(t));
        }
    };
    scaled(wa, a);
    scaled(wb, b);
    return out;
}

// ---------------------------------------------------------------------------
// block_circulant.cpp:82-112, :184-196
// ---------------------------------------------------------------------------
using CBlocks = std::vector<std::vector<Cplx>>;  // [k][m0*m0] col-major

void fft_levels(CBlocks& blk, const std::array<Index, 3>& dims, Index m0) {
    std::vector<Cplx> line;
    for (int axis = 0; axis < 3; ++axis) {
        const Index L = dims[axis];
        if (L == 1) continue;
        Index stride = 1;
        for (int l = axis + 1; l < 3; ++l) stride *= dims[l];
        const Index lines = dims[0] * dims[1] * dims[2] / L;
        line.resize(L);
        for (Index ln = 0; ln < lines; ++ln) {
            const Index inner = ln % stride, outer = ln / stride;
            const Index base = outer * stride * L + inner;
            for (Index e = 0; e < m0 * m0; ++e) {
                for (Index k = 0; k < L; ++k) line[k] = blk[base + k * stride][e];
                orla::fft_forward(line);
                for (Index k = 0; k < L; ++k) blk[base + k * stride][e] = line[k];
            }
        }
    }
}

CBlocks block_diagonalize(const GenMap& gen, const std::array<Index, 3>& dims, Index m0) {
    const Index total = dims[0] * dims[1] * dims[2];
    CBlocks bd(total, std::vector<Cplx>(m0 * m0, Cplx(0, 0)));
    for (const auto& [k, blk] : gen) {
        const Index lin = (k[0] * dims[1] + k[1]) * dims[2] + k[2];
        for (Index e = 0; e < m0 * m0; ++e) bd[lin][e] = Cplx(blk.a[e], 0.0);
    }
    fft_levels(bd, dims, m0);
    return bd;
}

// eigensolver.cpp:72-93
void solve_pencil(Index m0, const std::vector<Cplx>& Hj, const std::vector<Cplx>& Sj, Index j, double* values) {
    double hmax = 0.0, smax = 0.0, hdev = 0.0, sdev = 0.0;
    for (Index c = 0; c < m0; ++c)
        for (Index r = 0; r < m0; ++r) {
            hmax = std::max(hmax, std::abs(Hj[r + c * m0]));
            smax = std::max(smax, std::abs(Sj[r + c * m0]));
            hdev = std::max(hdev, std::abs(Hj[r + c * m0] - std::conj(Hj[c + r * m0])));
            sdev = std::max(sdev, std::abs(Sj[r + c * m0] - std::conj(Sj[c + r * m0])));
        }
    const double hscale = std::max(1.0, hmax), sscale = std::max(1.0, smax);
    if (hdev > 1e-10 * hscale || sdev > 1e-10 * sscale)
        fail(OR_EGENERIC, "solve_periodic: non-Hermitian diagonal block at k-point " + std::to_string(j));
    std::vector<Cplx> Hs(m0 * m0), Ss(m0 * m0);
    for (Index c = 0; c < m0; ++c)
        for (Index r = 0; r < m0; ++r) {
            Hs[r + c * m0] = 0.5 * (Hj[r + c * m0] + std::conj(Hj[c + r * m0]));
            Ss[r + c * m0] = 0.5 * (Sj[r + c * m0] + std::conj(Sj[c + r * m0]));
        }
    std::vector<Cplx> A;
    if (!orla::reduce_pencil<Cplx>(m0, Hs.data(), Ss.data(), A))
        fail(OR_EDEFINITE,
             "solve_periodic: overlap block at k-point " + std::to_string(j) + " is not positive definite");
    std::vector<Cplx> As(m0 * m0);
    for (Index c = 0; c < m0; ++c)
        for (Index r = 0; r < m0; ++r) As[r + c * m0] = 0.5 * (A[r + c * m0] + std::conj(A[c + r * m0]));
    orla::jacobi_eigenvalues<Cplx>(m0, As.data(), values);
}

// eigensolver.cpp:95-120 with parallel.hpp:15-32
void solve_blocks(const CBlocks& Hb, const std::function<std::vector<Cplx>(Index)>& Sblock, Index m0,
                  Index threads, double* eig) {
    const Index total = static_cast<Index>(Hb.size());
    std::vector<std::string> failures(total);
    std::vector<int> codes(total, 0);
    auto body = [&](Index j) {
        try {
            solve_pencil(m0, Hb[j], Sblock(j), j, eig + j * m0);
        } catch (const std::exception& e) {
            failures[j] = e.what();
        }
    };
    if (threads <= 1 || total < 2) {
        for (Index j = 0; j < total; ++j) body(j);
    } else {
        const Index nt = std::min(threads, total);
        std::vector<std::thread> pool;
        for (Index t = 0; t < nt; ++t)
            pool.emplace_back([&, t] {
                const Index chunk = (total + nt - 1) / nt;
                const Index lo = t * chunk, hi = std::min(total, lo + chunk);
                for (Index j = lo; j < hi; ++j) body(j);
            });
        for (auto& th : pool) th.join();
    }
    for (const auto& f : failures)
        if (!f.empty()) fail(OR_EDEFINITE, f);
}

void solve_periodic(const GenMap& H, const GenMap& S, const std::array<Index, 3>& dims, Index m0, Index threads,
                    double* eig) {
    const CBlocks Hb = block_diagonalize(H, dims, m0);
    const CBlocks Sb = block_diagonalize(S, dims, m0);
    solve_blocks(Hb, [&](Index j) { return Sb[j]; }, m0, threads, eig);
}

// factorized_diag.cpp:12-71 (per-level 1D FFTs + per-k Hadamard sums)
CBlocks factorized_blocks(const std::vector<std::array<std::vector<Mat>, 3>>& terms, const std::array<Index, 3>& dims,
                          Index m0) {
    std::vector<std::array<CBlocks, 3>> tr(terms.size());
    std::vector<Cplx> line;
    for (size_t t = 0; t < terms.size(); ++t)
        for (int l = 0; l < 3; ++l) {
            const Index Ll = static_cast<Index>(terms[t][l].size());
            tr[t][l].assign(Ll, std::vector<Cplx>(m0 * m0));
            line.resize(Ll);
            for (Index e = 0; e < m0 * m0; ++e) {
                for (Index k = 0; k < Ll; ++k) line[k] = Cplx(terms[t][l][k].a[e], 0.0);
                if (Ll > 1) orla::fft_forward(line);
                for (Index k = 0; k < Ll; ++k) tr[t][l][k][e] = line[k];
            }
        }
    const Index total = dims[0] * dims[1] * dims[2];
    CBlocks out(total, std::vector<Cplx>(m0 * m0, Cplx(0, 0)));
    for (Index j = 0; j < total; ++j) {
        const Index j1 = j / (dims[1] * dims[2]), j2 = (j / dims[2]) % dims[1], j3 = j % dims[2];
        for (const auto& t : tr)
            for (Index e = 0; e < m0 * m0; ++e) out[j][e] += t[0][j1][e] * t[1][j2][e] * t[2][j3][e];
    }
    return out;
}

// eigensolver.cpp:12-35 (eigenvalues only)
void solve_box_dense(Index n, const double* H, const double* S, Index cap, double* eig) {
    if (n > cap)
        fail(OR_ECAP, "solve_box_dense: size " + std::to_string(n) + " exceeds dense cap " + std::to_string(cap));
    std::vector<double> A;
    if (!orla::reduce_pencil<double>(n, H, S, A))
        fail(OR_EDEFINITE, "solve_box_dense: overlap matrix is not positive definite (near-linear-dependent basis?)");
    std::vector<double> As(n * n);
    for (Index c = 0; c < n; ++c)
        for (Index r = 0; r < n; ++r) As[r + c * n] = 0.5 * (A[r + c * n] + A[c + r * n]);
    orla::symmetric_eigenvalues(n, As.data(), eig);
}

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        g_err.clear();
        return OR_OK;
    } catch (const Err& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return OR_EGENERIC;
    }
}

GenMap gen_from_c(int64_t nblk, const int64_t* kidx, const double* b, Index m0) {
    GenMap g;
    for (int64_t i = 0; i < nblk; ++i) {
        Mat m(m0, m0);
        std::copy(b + i * m0 * m0, b + (i + 1) * m0 * m0, m.a.begin());
        g[{kidx[3 * i], kidx[3 * i + 1], kidx[3 * i + 2]}] = m;
    }
    return g;
}

}  // namespace orc

struct or_op {
    orc::Op op;
};

using namespace orc;

extern "C" {

const char* or_last_error(void) { return g_err.c_str(); }

int or_assemble(const or_system* csys, int periodic, int kind, or_op** out) {
    return guarded([&] {
        const Sys s = from_c(csys);
        auto* o = new or_op;
        try {
            o->op = periodic ? assemble_periodic(s, static_cast<Kind>(kind)) : assemble_box(s, static_cast<Kind>(kind));
        } catch (...) {
            delete o;
            throw;
        }
        *out = o;
    });
}

int or_combine(double wa, const or_op* a, double wb, const or_op* b, or_op** out) {
    return guarded([&] {
        auto* o = new or_op;
        try {
            o->op = combine(wa, a->op, wb, b->op);
        } catch (...) {
            delete o;
            throw;
        }
        *out = o;
    });
}

void or_op_free(or_op* op) { delete op; }

void or_op_info(const or_op* o, int64_t* info) {
    const Op& op = o->op;
    info[0] = op.periodic;
    info[1] = op.m0;
    for (int l = 0; l < 3; ++l) info[2 + l] = op.L[l];
    info[5] = op.L0;
    info[6] = op.coefficient_rank;
    info[7] = static_cast<int64_t>(op.gen.size());
    info[8] = op.m0 * op.L[0] * op.L[1] * op.L[2];
    for (int l = 0; l < 3; ++l) info[9 + l] = op.band[l];
}

void or_op_dense(const or_op* o, double* out) { std::copy(o->op.dense.a.begin(), o->op.dense.a.end(), out); }

void or_op_blocks(const or_op* o, int64_t* kidx, double* blk) {
    Index i = 0;
    const Index mm = o->op.m0 * o->op.m0;
    for (const auto& [k, b] : o->op.gen) {
        for (int l = 0; l < 3; ++l) kidx[3 * i + l] = k[l];
        std::copy(b.a.begin(), b.a.end(), blk + i * mm);
        ++i;
    }
}

void or_op_separable(const or_op* o, double* out) {
    const Index mm = o->op.m0 * o->op.m0;
    Index at = 0;
    for (const auto& t : o->op.separable)
        for (int l = 0; l < 3; ++l)
            for (const auto& b : t[l]) {
                std::copy(b.a.begin(), b.a.end(), out + at);
                at += mm;
            }
}

int or_solve_periodic_ops(const or_op* H, const or_op* S, int64_t threads, double* eig) {
    return guarded([&] {
        if (!H->op.periodic || !S->op.periodic)
            fail(OR_ESTRUCT, "solve_periodic: operators must be periodic assemblies");
        if (H->op.L != S->op.L || H->op.m0 != S->op.m0) fail(OR_ESTRUCT, "solve_periodic: H and S layouts differ");
        solve_periodic(H->op.gen, S->op.gen, H->op.L, H->op.m0, threads, eig);
    });
}

int or_solve_periodic(const int64_t* dims, int64_t m0, int64_t nH, const int64_t* kH, const double* bH, int64_t nS,
                      const int64_t* kS, const double* bS, int64_t threads, double* eig) {
    return guarded([&] {
        const std::array<Index, 3> d{dims[0], dims[1], dims[2]};
        solve_periodic(gen_from_c(nH, kH, bH, m0), gen_from_c(nS, kS, bS, m0), d, m0, threads, eig);
    });
}

int or_solve_periodic_factorized_ops(const or_op* H, const or_op* S, int64_t threads, double* eig) {
    return guarded([&] {
        if (!H->op.periodic || !S->op.periodic)
            fail(OR_ESTRUCT, "solve_periodic_factorized: operators must be periodic assemblies");
        if (H->op.separable.empty() || S->op.separable.empty())
            fail(OR_ESTRUCT, "solve_periodic_factorized: rank metadata missing");
        const CBlocks Hb = factorized_blocks(H->op.separable, H->op.L, H->op.m0);
        const CBlocks Sb = factorized_blocks(S->op.separable, S->op.L, S->op.m0);
        solve_blocks(Hb, [&](Index j) { return Sb[j]; }, H->op.m0, threads, eig);
    });
}

int or_block_diagonalize(const int64_t* dims, int64_t m0, int64_t nblk, const int64_t* kidx, const double* blocks,
                         double* out) {
    return guarded([&] {
        const std::array<Index, 3> d{dims[0], dims[1], dims[2]};
        const CBlocks bd = block_diagonalize(gen_from_c(nblk, kidx, blocks, m0), d, m0);
        Index at = 0;
        for (const auto& b : bd)
            for (const auto& z : b) {
                out[at++] = z.real();
                out[at++] = z.imag();
            }
    });
}

int or_solve_box_dense(int64_t n, const double* H, const double* S, int64_t cap, double* eig) {
    return guarded([&] { solve_box_dense(n, H, S, cap, eig); });
}

int or_solve_pencil(int64_t m0, const double* Hc, const double* Sc, int64_t j, double* eig) {
    return guarded([&] {
        std::vector<Cplx> H(m0 * m0), S(m0 * m0);
        for (int64_t i = 0; i < m0 * m0; ++i) {
            H[i] = Cplx(Hc[2 * i], Hc[2 * i + 1]);
            S[i] = Cplx(Sc[2 * i], Sc[2 * i + 1]);
        }
        solve_pencil(m0, H, S, j, eig);
    });
}

void or_sinc_quadrature(int64_t M, double* nodes, double* weights) {
    std::vector<double> t, w;
    sinc(M, t, w);
    std::copy(t.begin(), t.end(), nodes);
    std::copy(w.begin(), w.end(), weights);
}

int64_t or_overlap_constant(const or_system* csys) {
    const Sys s = from_c(csys);
    return overlap_constant(s);
}

void or_newton_master_column(int64_t ncells, double h, int64_t M, double* out) {
    std::vector<double> t, w;
    sinc(M, t, w);
    for (size_t q = 0; q < t.size(); ++q) master_column(ncells, h, t[q], out + q * ncells);
}

int or_potential(const or_system* csys, int periodic, int64_t margin, int64_t* rows, int64_t* tiled, double* panels,
                 double* weights, int64_t panels_cap) {
    return guarded([&] {
        const Sys s = from_c(csys);
        Ctx c;
        c.sys = &s;
        c.periodic = periodic != 0;
        c.margin = margin;
        build_potential(c);
        Index need = 0;
        for (int l = 0; l < 3; ++l) need += static_cast<Index>(c.pot[l].a.size());
        for (int l = 0; l < 3; ++l) {
            rows[l] = c.pot[l].rows;
            tiled[l] = c.tiled[l];
        }
        if (panels == nullptr || need > panels_cap) return;
        Index at = 0;
        for (int l = 0; l < 3; ++l) {
            std::copy(c.pot[l].a.begin(), c.pot[l].a.end(), panels + at);
            at += static_cast<Index>(c.pot[l].a.size());
        }
        std::copy(c.pot_w.begin(), c.pot_w.end(), weights);
    });
}

int or_assembled_window_sum(int64_t mrows, int64_t R, const double* master, int64_t nsh, const int64_t* shifts,
                            int64_t size, double* out) {
    return guarded([&] {
        Mat m(mrows, R);
        std::copy(master, master + mrows * R, m.a.begin());
        std::vector<Index> sh(shifts, shifts + nsh);
        const Mat acc = assembled_window_sum(m, sh, size);
        std::copy(acc.a.begin(), acc.a.end(), out);
    });
}

int64_t or_sample_gto_1d(const double* center, double alpha, const int32_t* deg, int dir, int64_t grid_n, double step,
                         int64_t cell_index, int64_t per_cell, double b, double align, double eps, int64_t* off,
                         double* values) {
    Gto g;
    for (int l = 0; l < 3; ++l) {
        g.c[l] = center[l];
        g.deg[l] = deg[l];
    }
    g.alpha = alpha;
    const Supp s = sample_gto_1d(g, dir, grid_n, step, cell_index, per_cell, b, align, eps);
    *off = s.offset;
    std::copy(s.v.begin(), s.v.end(), values);
    return static_cast<int64_t>(s.v.size());
}

double or_tri_form(int64_t uoff, int64_t ulen, const double* u, int64_t voff, int64_t vlen, const double* v, double lo,
                   double diag) {
    Supp a{uoff, std::vector<double>(u, u + ulen)};
    Supp b{voff, std::vector<double>(v, v + vlen)};
    return tri_form(a, b, lo, diag);
}

}  // extern "C"
