// latham_b200 — command-line front end of the B200 path with the reference CLI's wire
// formats: the flat `key = value` experiment file (tools/config.cpp:74-230),
// the four commands (tools/commands.cpp) and the CSV outputs with the resolved-config
// provenance header and %.17g numbers (tools/output.hpp:15-50), exit codes 2 / 3 / 4
// (tools/main.cpp:20-50).
//
//   latham_b200 {kernel|solve|bench|energy} --config FILE --out DIR
//
// All numerics run on the GPU through include/latham_b200.hpp. `solve.eigenvectors = true`
// writes eigenvectors_box.csv / eigenvectors_periodic.csv like commands.cpp:183-205 (box:
// S-orthonormal columns of the dense pencil; periodic: reconstruct_eigenvectors under
// caps.dense).
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <functional>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "latham_b200.hpp"

namespace fs = std::filesystem;
using namespace latham_b200;

namespace {

constexpr Index kDenseCap = 4096;            // block_circulant.hpp:76
constexpr Index kMaterializeCap = Index(1) << 24;  // canonical_tensor.hpp:76

struct ConfigError : Error {
    using Error::Error;
};

enum class Boundary { Box, Periodic, Both };

// ---------------------------------------------------------------------------
// experiment file
// ---------------------------------------------------------------------------
struct Experiment {
    double b = 8.0;
    Index n = 8, nbar = 8, n0 = 8, quad_M = 20;
    std::array<Index, 3> L{1, 1, 1};
    Boundary boundary = Boundary::Both;
    NucleiSet nuclei;
    GtoBasis basis;
    double eps_ov = 1e-8;
    Index n_occ = 1, threads = 1;
    Index cap_dense = kDenseCap, cap_materialize = kMaterializeCap;
    bool cap_ack = false, eigenvectors = false;
    std::vector<Index> bench_L, energy_L;
    std::vector<std::pair<std::string, std::string>> resolved;  // provenance header

    LatticeSystem system(const std::array<Index, 3>& Lx) const {
        LatticeSystem s;
        s.b = b;
        s.L = Lx;
        s.set_grid(n, nbar);
        s.quad_M = quad_M;
        s.nuclei = nuclei;
        s.basis = basis;
        s.eps_ov = eps_ov;
        return s;
    }
};

std::string strip(const std::string& s) {
    const size_t a = s.find_first_not_of(" \t\r\n");
    if (a == std::string::npos) return {};
    return s.substr(a, s.find_last_not_of(" \t\r\n") - a + 1);
}

std::vector<std::string> words(const std::string& s) {
    std::vector<std::string> w;
    std::istringstream is(s);
    for (std::string t; is >> t;) w.push_back(t);
    return w;
}

double number(const std::string& key, const std::string& v) {
    size_t used = 0;
    double d = 0.0;
    bool ok = true;
    try {
        d = std::stod(v, &used);
    } catch (const std::exception&) {
        ok = false;
    }
    if (!ok || used != v.size())
        throw ConfigError("config: key '" + key + "': expected a number, got '" + v + "'");
    return d;
}

Index integer(const std::string& key, const std::string& v) {
    const double d = number(key, v);
    const Index i = static_cast<Index>(d);
    if (static_cast<double>(i) != d)
        throw ConfigError("config: key '" + key + "': expected an integer, got '" + v + "'");
    return i;
}

bool boolean(const std::string& key, const std::string& v) {
    if (v == "true" || v == "1" || v == "yes") return true;
    if (v == "false" || v == "0" || v == "no") return false;
    throw ConfigError("config: key '" + key + "': expected true/false, got '" + v + "'");
}

std::vector<Index> integers(const std::string& key, const std::string& v) {
    std::vector<Index> out;
    for (const std::string& t : words(v)) out.push_back(integer(key, t));
    if (out.empty()) throw ConfigError("config: key '" + key + "': empty list");
    return out;
}

std::string shortest(double v) {  // default ostream formatting, as the resolved view prints doubles
    std::ostringstream os;
    os << v;
    return os.str();
}

Experiment read_experiment(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw ConfigError("config: cannot open '" + path + "'");
    Experiment x;
    std::map<std::string, std::string> scalars;
    std::string line;
    for (Index no = 1; std::getline(in, line); ++no) {
        line = strip(line.substr(0, line.find('#')));
        if (line.empty()) continue;
        const size_t eq = line.find('=');
        if (eq == std::string::npos)
            throw ConfigError("config: line " + std::to_string(no) + ": expected key = value");
        const std::string key = strip(line.substr(0, eq)), val = strip(line.substr(eq + 1));
        if (key.empty() || val.empty())
            throw ConfigError("config: line " + std::to_string(no) + ": empty key or value");
        if (key == "nucleus" || key == "basis") {  // repeated entity lines
            const auto f = words(val);
            if (key == "nucleus") {
                if (f.size() != 4)
                    throw ConfigError("config: line " + std::to_string(no) + ": nucleus wants 'x y z Z'");
                Nucleus nu;
                for (int i = 0; i < 3; ++i) nu.position[static_cast<size_t>(i)] = number(key, f[static_cast<size_t>(i)]);
                nu.charge = number(key, f[3]);
                x.nuclei.nuclei.push_back(nu);
            } else {
                if (f.size() != 4 && f.size() != 7)
                    throw ConfigError("config: line " + std::to_string(no) +
                                      ": basis wants 'x y z alpha [dx dy dz]'");
                GtoFunction g;
                for (int i = 0; i < 3; ++i) g.center[static_cast<size_t>(i)] = number(key, f[static_cast<size_t>(i)]);
                g.exponent = number(key, f[3]);
                if (f.size() == 7)
                    for (int i = 0; i < 3; ++i)
                        g.degrees[static_cast<size_t>(i)] = static_cast<int>(integer(key, f[static_cast<size_t>(4 + i)]));
                x.basis.functions.push_back(g);
            }
            x.resolved.emplace_back(key, val);
            continue;
        }
        if (!scalars.emplace(key, val).second)
            throw ConfigError("config: line " + std::to_string(no) + ": duplicate key '" + key + "'");
    }
    auto pop = [&](const std::string& key, const std::function<void(const std::string&)>& use) {
        auto it = scalars.find(key);
        if (it == scalars.end()) return false;
        use(it->second);
        scalars.erase(it);
        return true;
    };
    pop("cell.b", [&](const std::string& v) { x.b = number("cell.b", v); });
    pop("grid.n", [&](const std::string& v) { x.n = integer("grid.n", v); });
    pop("grid.nbar", [&](const std::string& v) { x.nbar = integer("grid.nbar", v); });
    pop("grid.n0", [&](const std::string& v) { x.n0 = integer("grid.n0", v); });
    pop("quad.M", [&](const std::string& v) { x.quad_M = integer("quad.M", v); });
    pop("lattice.L", [&](const std::string& v) {
        const auto f = integers("lattice.L", v);
        if (f.size() != 3) throw ConfigError("config: lattice.L wants three integers");
        x.L = {f[0], f[1], f[2]};
    });
    pop("boundary", [&](const std::string& v) {
        if (v == "box") x.boundary = Boundary::Box;
        else if (v == "periodic") x.boundary = Boundary::Periodic;
        else if (v == "both") x.boundary = Boundary::Both;
        else throw ConfigError("config: boundary must be box, periodic or both");
    });
    pop("eps_ov", [&](const std::string& v) { x.eps_ov = number("eps_ov", v); });
    pop("n_occ", [&](const std::string& v) { x.n_occ = integer("n_occ", v); });
    const bool threads_set = pop("threads", [&](const std::string& v) { x.threads = integer("threads", v); });
    pop("caps.dense", [&](const std::string& v) { x.cap_dense = integer("caps.dense", v); });
    pop("caps.materialize", [&](const std::string& v) { x.cap_materialize = integer("caps.materialize", v); });
    pop("caps.acknowledge", [&](const std::string& v) { x.cap_ack = boolean("caps.acknowledge", v); });
    pop("solve.eigenvectors", [&](const std::string& v) { x.eigenvectors = boolean("solve.eigenvectors", v); });
    pop("bench.L_list", [&](const std::string& v) { x.bench_L = integers("bench.L_list", v); });
    pop("energy.L_list", [&](const std::string& v) { x.energy_L = integers("energy.L_list", v); });
    if (!scalars.empty()) throw ConfigError("config: unknown key '" + scalars.begin()->first + "'");

    if (x.threads <= 0) throw ConfigError("config: threads must be positive");
    if (const char* env = std::getenv("LATHAM_THREADS"); env && !threads_set) {
        char* end = nullptr;
        const long t = std::strtol(env, &end, 10);
        if (end == env || *end) throw ConfigError("config: LATHAM_THREADS is not an integer");
        x.threads = std::max<Index>(1, t);
    }
    if (x.b <= 0.0) throw ConfigError("config: cell.b must be positive");
    if (x.n < 1 || x.nbar < 1) throw ConfigError("config: grid sizes must be >= 1");
    if (2 * x.n0 < x.n) throw ConfigError("config: grid.n0 must be at least n/2");
    if (x.quad_M < 1) throw ConfigError("config: quad.M must be >= 1");
    for (Index l : x.L)
        if (l < 1) throw ConfigError("config: lattice.L entries must be >= 1");
    if (x.nuclei.nuclei.empty()) throw ConfigError("config: at least one nucleus line required");
    if (x.basis.functions.empty()) throw ConfigError("config: at least one basis line required");
    if (x.eps_ov <= 0.0) throw ConfigError("config: eps_ov must be positive");
    if (x.n_occ < 1 || x.n_occ > x.basis.m0()) throw ConfigError("config: n_occ must be in [1, m0]");
    x.nuclei.cell_size = x.b;
    // NucleiSet / GtoBasis validation (newton_kernel.cpp, gto_basis.cpp)
    for (const auto& nu : x.nuclei.nuclei) {
        if (!(nu.charge > 0.0)) throw ConfigError("config: NucleiSet: charges must be positive");
        for (double p : nu.position)
            if (std::abs(p) > 0.5 * x.b) throw ConfigError("config: NucleiSet: nucleus outside the cell");
    }
    for (const auto& g : x.basis.functions) {
        if (!(g.exponent > 0.0)) throw ConfigError("config: GtoBasis: exponents must be positive");
        for (int d : g.degrees)
            if (d < 0) throw ConfigError("config: GtoBasis: monomial degrees must be >= 0");
    }
    if ((x.cap_dense != kDenseCap || x.cap_materialize != kMaterializeCap) &&
        (x.cap_dense > kDenseCap || x.cap_materialize > kMaterializeCap) && !x.cap_ack)
        throw ConfigError("config: raising caps.dense or caps.materialize requires caps.acknowledge = true");

    auto put = [&](const char* k, const std::string& v) { x.resolved.emplace_back(k, v); };
    put("cell.b", shortest(x.b));
    put("grid.n", std::to_string(x.n));
    put("grid.nbar", std::to_string(x.nbar));
    put("grid.n0", std::to_string(x.n0));
    put("quad.M", std::to_string(x.quad_M));
    put("lattice.L", std::to_string(x.L[0]) + " " + std::to_string(x.L[1]) + " " + std::to_string(x.L[2]));
    put("boundary", x.boundary == Boundary::Box ? "box" : (x.boundary == Boundary::Periodic ? "periodic" : "both"));
    put("eps_ov", shortest(x.eps_ov));
    put("n_occ", std::to_string(x.n_occ));
    put("threads", std::to_string(x.threads));
    put("caps.dense", std::to_string(x.cap_dense));
    put("caps.materialize", std::to_string(x.cap_materialize));
    return x;
}

// ---------------------------------------------------------------------------
// outputs: provenance header, LF endings, atomic landing (temp + rename)
// ---------------------------------------------------------------------------
class Sheet {
public:
    Sheet(const fs::path& dir, const std::string& name, const std::string& command, const Experiment& x)
        : path_(dir / name) {
        buf_ << "# latham " << command << "\n";
        for (const auto& kv : x.resolved) buf_ << "# " << kv.first << " = " << kv.second << "\n";
    }
    template <class T>
    Sheet& operator<<(const T& v) {
        buf_ << v;
        return *this;
    }
    static std::string num(double v) {
        char s[64];
        std::snprintf(s, sizeof s, "%.17g", v);
        return s;
    }
    void land() {
        const fs::path tmp = path_.string() + ".tmp";
        {
            std::ofstream f(tmp, std::ios::binary | std::ios::trunc);
            if (!f) throw Error("cannot write " + tmp.string());
            f << buf_.str();
        }
        fs::rename(tmp, path_);
    }

private:
    fs::path path_;
    std::ostringstream buf_;
};

double wall_seconds(const std::function<void()>& fn) {
    const auto a = std::chrono::steady_clock::now();
    fn();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
}

// the reference's timed_median: 1, 3 or 5 runs by the length of the first
double median_seconds(const std::function<void()>& fn) {
    std::vector<double> t{wall_seconds(fn)};
    const int reps = t[0] > 10.0 ? 1 : (t[0] > 1.0 ? 3 : 5);
    while (static_cast<int>(t.size()) < reps) t.push_back(wall_seconds(fn));
    std::sort(t.begin(), t.end());
    return t[t.size() / 2];
}

double loglog_slope(const std::vector<double>& x, const std::vector<double>& y) {
    double sx = 0, sy = 0, sxx = 0, sxy = 0;
    for (size_t i = 0; i < x.size(); ++i) {
        const double a = std::log(x[i]), b = std::log(y[i]);
        sx += a;
        sy += b;
        sxx += a * a;
        sxy += a * b;
    }
    const double n = static_cast<double>(x.size());
    return (n * sxy - sx * sy) / (n * sxx - sx * sx);
}

// box bands: ascending spectrum cut into m0 runs of PiL values (tools/commands.cpp box_bands)
BandStructure chunk_bands(const std::vector<double>& sorted, Index m0, Index cells) {
    BandStructure bs;
    bs.m0 = m0;
    for (Index m = 0; m < m0; ++m) {
        bs.bands.emplace_back(sorted.begin() + m * cells, sorted.begin() + (m + 1) * cells);
        const auto& b = bs.bands.back();
        bs.band_min.push_back(*std::min_element(b.begin(), b.end()));
        bs.band_max.push_back(*std::max_element(b.begin(), b.end()));
    }
    return bs;
}

void bands_sheet(const fs::path& out, const char* name, const Experiment& x, const BandStructure& bs) {
    Sheet f(out, name, "solve", x);
    f << "band,k_linear,eigenvalue\n";
    for (Index m = 0; m < bs.m0; ++m)
        for (size_t j = 0; j < bs.bands[static_cast<size_t>(m)].size(); ++j)
            f << m << "," << j << "," << Sheet::num(bs.bands[static_cast<size_t>(m)][j]) << "\n";
    f.land();
}

// ---------------------------------------------------------------------------
// commands
// ---------------------------------------------------------------------------
void run_kernel(Context& ctx, const Experiment& x, const fs::path& out) {
    const Index R = 2 * x.quad_M + 1;
    std::vector<double> t(static_cast<size_t>(R)), w(static_cast<size_t>(R));
    check(lt_sinc_quadrature(ctx.get(), x.quad_M, t.data(), w.data()));
    auto quad = [&](double z) {  // SincQuadrature::evaluate
        double s = 0.0;
        for (Index i = 0; i < R; ++i) s += w[static_cast<size_t>(i)] * std::exp(-(t[static_cast<size_t>(i)] * z) * (t[static_cast<size_t>(i)] * z));
        return s;
    };
    // the lattice-summed potential of the box supercell without margin, on the device
    const LatticeSystem sys = x.system(x.L);
    SystemView v(sys);
    int64_t rows[3] = {0, 0, 0}, tiled[3] = {0, 0, 0};
    Index rank = 0;
    const double secs = wall_seconds([&] {
        check(lt_potential(ctx.get(), v.get(), 0, 0, rows, tiled, nullptr, nullptr, 0));
        const Index Rt = R * x.nuclei.count();
        std::vector<double> panels(static_cast<size_t>((rows[0] + rows[1] + rows[2]) * Rt)), wts(static_cast<size_t>(Rt));
        check(lt_potential(ctx.get(), v.get(), 0, 0, rows, tiled, panels.data(), wts.data(),
                           static_cast<int64_t>(panels.size())));
        rank = Rt;
    });
    double worst = 0.0;
    Sheet acc(out, "kernel_accuracy.csv", "kernel", x);
    acc << "z,quadrature,exact,rel_error\n";
    for (double z : {0.5, 0.75, 1.0, 2.0, 5.0, 10.0, 20.0}) {
        const double q = quad(z), rel = std::abs(q - 1.0 / z) * z;
        worst = std::max(worst, rel);
        acc << Sheet::num(z) << "," << Sheet::num(q) << "," << Sheet::num(1.0 / z) << "," << Sheet::num(rel) << "\n";
    }
    acc.land();
    Sheet rep(out, "kernel_report.csv", "kernel", x);
    rep << "M,R,rank,rank_bound,quad_rel_err_z1,quad_rel_err_max,assembly_seconds\n";
    rep << x.quad_M << "," << R << "," << rank << "," << x.nuclei.count() * R << ","
        << Sheet::num(std::abs(quad(1.0) - 1.0)) << "," << Sheet::num(worst) << "," << Sheet::num(secs) << "\n";
    rep.land();
}

void run_solve(Context& ctx, const Experiment& x, const fs::path& out) {
    const LatticeSystem sys = x.system(x.L);
    const bool box = x.boundary != Boundary::Periodic, per = x.boundary != Boundary::Box;
    std::vector<double> box_sorted;
    KPointSpectrum spec;
    if (box) {
        if (sys.basis_count() > x.cap_dense)
            throw ResourceCapError("solve_box_dense: size " + std::to_string(sys.basis_count()) +
                                   " exceeds dense cap " + std::to_string(x.cap_dense));
        DenseSpectrum ds;
        if (x.eigenvectors) {  // commands.cpp:176-178 with want_vectors
            SystemView v(sys);
            lt_operator *hp = nullptr, *sp = nullptr;
            check(lt_assemble_core(ctx.get(), v.get(), 0, &hp, &sp));
            AssembledOperator Hb(hp, OperatorKind::Laplace), Sb(sp, OperatorKind::Mass);
            ds = solve_box_dense(ctx, Hb.dense(), Sb.dense(), sys.basis_count(), x.cap_dense, true);
        } else {
            ds = solve_core_box(ctx, sys);
        }
        box_sorted = ds.eigenvalues;
        Sheet f(out, "spectrum_box.csv", "solve", x);
        f << "k1,k2,k3,band,eigenvalue\n";
        for (size_t i = 0; i < box_sorted.size(); ++i) f << "-1,-1,-1," << i << "," << Sheet::num(box_sorted[i]) << "\n";
        f.land();
        bands_sheet(out, "bands_box.csv", x, chunk_bands(box_sorted, sys.m0(), sys.lattice_count()));
        if (x.eigenvectors) {  // commands.cpp:183-190
            const Index nb = sys.basis_count();
            Sheet ev(out, "eigenvectors_box.csv", "solve", x);
            ev << "index,component,value\n";
            for (Index c = 0; c < nb; ++c)
                for (Index r = 0; r < nb; ++r)
                    ev << c << "," << r << "," << Sheet::num(ds.eigenvectors[static_cast<size_t>(c * nb + r)]) << "\n";
            ev.land();
        }
    }
    if (per) {
        if (x.eigenvectors) {  // commands.cpp:192-194 with want_vectors
            SystemView v(sys);
            lt_operator *hp = nullptr, *sp = nullptr;
            check(lt_assemble_core(ctx.get(), v.get(), 1, &hp, &sp));
            AssembledOperator H(hp, OperatorKind::Laplace), S(sp, OperatorKind::Mass);
            spec = solve_periodic(ctx, H, S, true);
        } else {
            spec = solve_core_periodic(ctx, sys);
        }
        Sheet f(out, "spectrum_periodic.csv", "solve", x);
        f << "k1,k2,k3,band,eigenvalue\n";
        for (Index j = 0; j < spec.k_count(); ++j) {
            const auto k = spec.k_multi(j);
            for (Index m = 0; m < spec.m0; ++m)
                f << k[0] << "," << k[1] << "," << k[2] << "," << m << ","
                  << Sheet::num(spec.eigenvalues[static_cast<size_t>(j)][static_cast<size_t>(m)]) << "\n";
        }
        f.land();
        bands_sheet(out, "bands_periodic.csv", x, spectral_bands(spec));
        if (x.eigenvectors) {  // commands.cpp:197-205
            const Index N = spec.k_count() * spec.m0;
            const std::vector<std::complex<double>> U = reconstruct_eigenvectors(ctx, spec, x.cap_dense);
            Sheet ev(out, "eigenvectors_periodic.csv", "solve", x);
            ev << "index,component,re,im\n";
            for (Index c = 0; c < N; ++c)
                for (Index r = 0; r < N; ++r) {
                    const auto z = U[static_cast<size_t>(c * N + r)];
                    ev << c << "," << r << "," << Sheet::num(z.real()) << "," << Sheet::num(z.imag()) << "\n";
                }
            ev.land();
        }
    }
    if (box && per) {
        const DefectReport d = box_circulant_defect(ctx, sys);
        const BandStructure pb = spectral_bands(spec), bb = chunk_bands(box_sorted, sys.m0(), sys.lattice_count());
        Sheet f(out, "defect.csv", "solve", x);
        f << "L1,L2,L3,nuclear_defect_rel_fro,band,band_max_discrepancy\n";
        for (Index m = 0; m < sys.m0(); ++m) {
            auto a = pb.bands[static_cast<size_t>(m)], c = bb.bands[static_cast<size_t>(m)];
            std::sort(a.begin(), a.end());
            std::sort(c.begin(), c.end());
            double disc = 0.0;
            for (size_t i = 0; i < a.size(); ++i) disc = std::max(disc, std::abs(a[i] - c[i]));
            f << sys.L[0] << "," << sys.L[1] << "," << sys.L[2] << "," << Sheet::num(d.relative_fro) << "," << m << ","
              << Sheet::num(disc) << "\n";
        }
        f.land();
    }
    Sheet g(out, "bands.gp", "solve", x);
    g << "set datafile separator ','\nset xlabel 'k (linear index)'\nset ylabel 'eigenvalue'\nplot ";
    if (per) g << "'bands_periodic.csv' using 2:3 with points title 'periodic'";
    if (per && box) g << ", ";
    if (box) g << "'bands_box.csv' using 2:3 with points title 'box'";
    g << "\n";
    g.land();
}

// times the spectrum stage with prebuilt operators, like the reference's bench
void run_bench(Context& ctx, const Experiment& x, const fs::path& out) {
    if (x.bench_L.empty()) throw ConfigError("bench: bench.L_list must list the lattice sizes to sweep");
    Sheet f(out, "bench.csv", "bench", x);
    f << "Nb,path,seconds\n";
    std::vector<double> nd, td, nf, tf;
    for (Index Lx : x.bench_L) {
        const LatticeSystem sys = x.system({Lx, 1, 1});
        const Index Nb = sys.basis_count();
        SystemView v(sys);
        lt_operator *hp = nullptr, *sp = nullptr;
        check(lt_assemble_core(ctx.get(), v.get(), 1, &hp, &sp));
        AssembledOperator H(hp, OperatorKind::Laplace), S(sp, OperatorKind::Mass);
        const double tp = median_seconds([&] { (void)solve_periodic(ctx, H, S); });
        f << Nb << ",fft," << Sheet::num(tp) << "\n";
        nf.push_back(static_cast<double>(Nb));
        tf.push_back(tp);
        if (Nb <= x.cap_dense) {
            check(lt_assemble_core(ctx.get(), v.get(), 0, &hp, &sp));
            AssembledOperator Hb(hp, OperatorKind::Laplace), Sb(sp, OperatorKind::Mass);
            const std::vector<double> hd = Hb.dense(), sd = Sb.dense();
            const double tb = median_seconds([&] { (void)solve_box_dense(ctx, hd, sd, Nb, x.cap_dense); });
            f << Nb << ",dense," << Sheet::num(tb) << "\n";
            nd.push_back(static_cast<double>(Nb));
            td.push_back(tb);
        }
    }
    f.land();
    Sheet e(out, "bench_exponents.csv", "bench", x);
    e << "path,points,fitted_exponent\n";
    if (nd.size() >= 2) e << "dense," << nd.size() << "," << Sheet::num(loglog_slope(nd, td)) << "\n";
    if (nf.size() >= 2) e << "fft," << nf.size() << "," << Sheet::num(loglog_slope(nf, tf)) << "\n";
    e.land();
    Sheet g(out, "bench.gp", "bench", x);
    g << "set datafile separator ','\nset logscale xy\nset xlabel 'N_b'\nset ylabel 'seconds'\n"
      << "plot '< grep dense bench.csv' using 1:3 with linespoints title 'dense', \\\n"
      << "     '< grep fft bench.csv' using 1:3 with linespoints title 'fft'\n";
    g.land();
}

void run_energy(Context& ctx, const Experiment& x, const fs::path& out) {
    if (x.energy_L.empty()) throw ConfigError("energy: energy.L_list must list the lattice sizes to sweep");
    const bool box = x.boundary != Boundary::Periodic, per = x.boundary != Boundary::Box;
    Sheet f(out, "energy.csv", "energy", x);
    f << "L1,L2,L3,boundary,E_per_cell\n";
    for (Index Lx : x.energy_L) {
        const LatticeSystem sys = x.system({Lx, 1, 1});
        if (box) {
            if (sys.basis_count() > x.cap_dense)
                throw ResourceCapError("solve_box_dense: size " + std::to_string(sys.basis_count()) +
                                       " exceeds dense cap " + std::to_string(x.cap_dense));
            const auto ev = solve_core_box(ctx, sys).eigenvalues;
            f << Lx << ",1,1,box," << Sheet::num(average_energy_per_cell(ev, sys.lattice_count(), x.n_occ)) << "\n";
        }
        if (per) {
            const auto ev = solve_core_periodic(ctx, sys).sorted_all();
            f << Lx << ",1,1,periodic," << Sheet::num(average_energy_per_cell(ev, sys.lattice_count(), x.n_occ))
              << "\n";
        }
    }
    f.land();
    Sheet g(out, "energy.gp", "energy", x);
    g << "set datafile separator ','\nset xlabel 'L'\nset ylabel 'E per cell'\n"
      << "plot '< grep box energy.csv' using 1:5 with linespoints title 'box', \\\n"
      << "     '< grep periodic energy.csv' using 1:5 with linespoints title 'periodic'\n";
    g.land();
}

int usage() {
    std::fprintf(stderr, "usage: latham_b200 {kernel|solve|bench|energy} --config FILE --out DIR\n");
    return 2;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage();
    const std::string cmd = argv[1];
    if (cmd != "kernel" && cmd != "solve" && cmd != "bench" && cmd != "energy") return usage();
    std::string config, outdir;
    for (int i = 2; i + 1 < argc; i += 2) {
        const std::string opt = argv[i];
        if (opt == "--config") config = argv[i + 1];
        else if (opt == "--out") outdir = argv[i + 1];
        else return usage();
    }
    if (config.empty() || outdir.empty() || argc % 2 != 0) return usage();
    try {
        const Experiment x = read_experiment(config);
        fs::create_directories(outdir);
        Context ctx(0);
        if (cmd == "kernel") run_kernel(ctx, x, outdir);
        else if (cmd == "solve") run_solve(ctx, x, outdir);
        else if (cmd == "bench") run_bench(ctx, x, outdir);
        else run_energy(ctx, x, outdir);
        return 0;
    } catch (const ConfigError& e) {
        std::fprintf(stderr, "config error: %s\n", e.what());
        return 2;
    } catch (const ResourceCapError& e) {
        std::fprintf(stderr, "resource cap: %s\n", e.what());
        return 4;
    } catch (const Error& e) {
        std::fprintf(stderr, "numerical error: %s\n", e.what());
        return 3;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 3;
    }
}
