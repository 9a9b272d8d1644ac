// k_profiles.cu — GTO profiles on the assembly grids and the 1D FEM form tables.
//
//   launch_profiles    gto_basis.cpp:31-47 (sample_gto_1d with the assembly trim
//                      kTrimEps = 1e-280, galerkin.cpp:13, :127-149): values on the
//                      extended grid of (L + 2 margin) cells; support [lo, hi) is the
//                      first/last index with |v| >= eps (the reference's tail trim), and
//                      entries outside it are zeroed so the dense vector equals the
//                      reference's zero-extended Supported1D.
//   launch_fem_tables  fem1d.cpp:19-32 (supported tri_form) via galerkin.cpp:208-223:
//                      massT/stiffT[d][mu + nu m0] = <A u_mu, u_nu(. - d nbar)>, P1 mass
//                      (h/6){1,4,1} and stiffness (1/h){-1,2,-1}, open (not wrapped).
#include "lt_device.cuh"
#include "lt_internal.cuh"

namespace lt {

constexpr int kMaxProfileJobs = 6;
struct ProfileJobs {
    ProfileJob j[kMaxProfileJobs];
};

// One CTA per (job, function) over its whole grid: samples, the support [lo, hi) (first /
// last index with |v| >= eps, the reference's tail trim) from a block reduction, and the
// trimmed values in the same pass: a sample below eps is written as 0. That equals the
// zero-extended Supported1D wherever sub-eps samples occur only in the tails — for a
// Gaussian times (x - c)^deg a non-zero sample below 1e-280 away from the tails would need
// |x - c| < 1e-280^(1/deg), i.e. a grid point on the centre, where the sample is exactly 0.
__global__ void __launch_bounds__(512) k_profiles(DevSys s, ProfileJobs jobs, double eps) {
    const ProfileJob& jb = jobs.j[blockIdx.y];
    const Index mu = blockIdx.x;
    const Index base = jb.cell_index * jb.per_cell;
    long long lo = jb.grid, hi = -1;
    for (Index i = threadIdx.x; i < jb.grid; i += blockDim.x) {
        const double x =
            __dsub_rn(__dmul_rn(__dadd_rn(static_cast<double>(i - base), jb.align), jb.step), __dmul_rn(0.5, s.b));
        const double v = gto_eval1d(s, mu, jb.dir, x);
        const bool keep = !(fabs(v) < eps);
        jb.values[mu * jb.grid + i] = keep ? v : 0.0;
        if (keep) {
            lo = min(lo, static_cast<long long>(i));
            hi = max(hi, static_cast<long long>(i));
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    __shared__ long long slo[16], shi[16];
    if ((threadIdx.x & 31) == 0) {
        slo[threadIdx.x >> 5] = lo;
        shi[threadIdx.x >> 5] = hi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) {
            lo = min(lo, slo[w]);
            hi = max(hi, shi[w]);
        }
        const bool empty = hi < 0;  // Supported1D{0, empty}
        jb.lo[mu] = empty ? 0ull : static_cast<unsigned long long>(lo);
        jb.hi[mu] = empty ? 0ull : static_cast<unsigned long long>(hi + 1);
    }
}

void launch_profiles(const Launch& L, const DevSys& s, const ProfileJob* jobs, int njobs, double eps) {
    if (njobs > kMaxProfileJobs) fail(LT_EGENERIC, "launch_profiles: too many jobs");
    ProfileJobs pj{};
    for (int k = 0; k < njobs; ++k) pj.j[k] = jobs[k];
    dim3 grid(static_cast<unsigned>(s.m0), static_cast<unsigned>(njobs));
    Stage st_(L, "profiles");
    k_profiles<<<grid, 512, 0, L.st>>>(s, pj, eps);
    LT_CU(cudaGetLastError());
    L.tick();
}

// ---------------------------------------------------------------------------
// FEM tables: one warp per (d, mu, nu)
// ---------------------------------------------------------------------------
__global__ void k_fem_tables(Index m0, Index band, Index nbar, double hbar, Index Gbar, const double* __restrict__ pwl,
                             const unsigned long long* __restrict__ plo, const unsigned long long* __restrict__ phi,
                             double* __restrict__ massT, double* __restrict__ stiffT) {
    const int lane = threadIdx.x & 31;
    const Index task = static_cast<Index>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const Index width = 2 * band + 1;
    if (task >= width * m0 * m0) return;
    const Index di = task / (m0 * m0);
    const Index e = task % (m0 * m0);
    const Index mu = e % m0, nu = e / m0;
    const Index d = di - band;
    const Index sh = d * nbar;
    const Index ulo = static_cast<Index>(plo[mu]), uhi = static_cast<Index>(phi[mu]);
    const Index vlo = static_cast<Index>(plo[nu]) + sh, vhi = static_cast<Index>(phi[nu]) + sh;
    const Index lo_i = max(ulo, vlo - 1), hi_i = min(uhi, vhi + 1);
    const double* u = pwl + mu * Gbar;
    const double* vv = pwl + nu * Gbar;
    const double mlo = hbar / 6.0, mdiag = (4.0 * hbar) / 6.0;
    const double slo = -1.0 / hbar, sdiag = 2.0 / hbar;
    double sm = 0.0, ss = 0.0;
    for (Index i = lo_i + lane; i < hi_i; i += 32) {
        const double ui = u[i];
        double rm = 0.0, rs = 0.0;
        if (i - 1 >= vlo && i - 1 < vhi) {
            const double x = vv[i - 1 - sh];
            rm = __dadd_rn(rm, __dmul_rn(mlo, x));
            rs = __dadd_rn(rs, __dmul_rn(slo, x));
        }
        if (i >= vlo && i < vhi) {
            const double x = vv[i - sh];
            rm = __dadd_rn(rm, __dmul_rn(mdiag, x));
            rs = __dadd_rn(rs, __dmul_rn(sdiag, x));
        }
        if (i + 1 >= vlo && i + 1 < vhi) {
            const double x = vv[i + 1 - sh];
            rm = __dadd_rn(rm, __dmul_rn(mlo, x));
            rs = __dadd_rn(rs, __dmul_rn(slo, x));
        }
        sm = __dadd_rn(sm, __dmul_rn(ui, rm));
        ss = __dadd_rn(ss, __dmul_rn(ui, rs));
    }
    sm = warp_sum(sm);
    ss = warp_sum(ss);
    if (lane == 0) {
        massT[di * m0 * m0 + e] = sm;
        stiffT[di * m0 * m0 + e] = ss;
    }
}

void launch_fem_tables(const Launch& L, Index m0, Index band, Index nbar, double hbar, Index Gbar, const double* pwl,
                       const unsigned long long* lo, const unsigned long long* hi, double* massT, double* stiffT) {
    const Index tasks = (2 * band + 1) * m0 * m0;
    const int wpb = 8;
    Stage st_(L, "fem_tables");
    k_fem_tables<<<static_cast<unsigned>((tasks + wpb - 1) / wpb), wpb * 32, 0, L.st>>>(m0, band, nbar, hbar, Gbar,
                                                                                       pwl, lo, hi, massT, stiffT);
    LT_CU(cudaGetLastError());
    L.tick();
}

}  // namespace lt
