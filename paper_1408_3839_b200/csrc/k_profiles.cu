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

__global__ void k_profile_sample(DevSys s, ProfileJobs jobs, double eps) {
    const ProfileJob& jb = jobs.j[blockIdx.z];
    const Index mu = blockIdx.y;
    const Index i = static_cast<Index>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool in = i < jb.grid;
    bool keep = false;
    if (in) {
        const Index base = jb.cell_index * jb.per_cell;
        const double x =
            __dsub_rn(__dmul_rn(__dadd_rn(static_cast<double>(i - base), jb.align), jb.step), __dmul_rn(0.5, s.b));
        const double v = gto_eval1d(s, mu, jb.dir, x);
        jb.values[mu * jb.grid + i] = v;
        keep = !(fabs(v) < eps);
    }
    // CTA-aggregated support bounds: warp ballots, then one atomic pair per CTA (thousands
    // of CTAs hit the same m0 addresses otherwise)
    __shared__ unsigned long long cta_lo, cta_hi;
    if (threadIdx.x == 0) {
        cta_lo = ~0ull;
        cta_hi = 0ull;
    }
    __syncthreads();
    const unsigned mask = __ballot_sync(0xffffffffu, keep);
    if (mask && (threadIdx.x & 31) == 0) {
        const Index wbase = i;  // lane 0's index
        atomicMin(&cta_lo, static_cast<unsigned long long>(wbase + (__ffs(mask) - 1)));
        atomicMax(&cta_hi, static_cast<unsigned long long>(wbase + (31 - __clz(mask)) + 1));
    }
    __syncthreads();
    if (threadIdx.x == 0 && cta_hi > 0) {
        atomicMin(&jb.lo[mu], cta_lo);
        atomicMax(&jb.hi[mu], cta_hi);
    }
}

__global__ void k_profile_trim(ProfileJobs jobs) {
    const ProfileJob& jb = jobs.j[blockIdx.z];
    const Index mu = blockIdx.y;
    const Index i = static_cast<Index>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= jb.grid) return;
    unsigned long long lo = jb.lo[mu], hi = jb.hi[mu];
    const bool empty = lo == ~0ull;
    if (empty) {
        lo = 0;
        hi = 0;
    }
    if (static_cast<unsigned long long>(i) < lo || static_cast<unsigned long long>(i) >= hi)
        jb.values[mu * jb.grid + i] = 0.0;
    if (i == 0 && empty) {  // Supported1D{0, empty}
        jb.lo[mu] = 0;
        jb.hi[mu] = 0;
    }
}

// support bounds of every job reset in one launch (lo = all ones, hi = 0): a memset per
// array would put 2 x njobs serial graph nodes in front of the sampling
__global__ void k_profile_bounds_init(ProfileJobs jobs, int njobs, Index m0) {
    for (int k = 0; k < njobs; ++k)
        for (Index mu = threadIdx.x; mu < m0; mu += blockDim.x) {
            jobs.j[k].lo[mu] = ~0ull;
            jobs.j[k].hi[mu] = 0ull;
        }
}

void launch_profiles(const Launch& L, const DevSys& s, const ProfileJob* jobs, int njobs, double eps) {
    if (njobs > kMaxProfileJobs) fail(LT_EGENERIC, "launch_profiles: too many jobs");
    ProfileJobs pj{};
    Index gmax = 1;
    for (int k = 0; k < njobs; ++k) {
        pj.j[k] = jobs[k];
        gmax = std::max(gmax, jobs[k].grid);
    }
    dim3 grid(static_cast<unsigned>((gmax + 255) / 256), s.m0, njobs);
    Stage st_(L, "profiles");
    k_profile_bounds_init<<<1, 64, 0, L.st>>>(pj, njobs, s.m0);
    LT_CU(cudaGetLastError());
    k_profile_sample<<<grid, 256, 0, L.st>>>(s, pj, eps);
    LT_CU(cudaGetLastError());
    // trimming depends on the complete bounds: second pass (stream-ordered)
    k_profile_trim<<<grid, 256, 0, L.st>>>(pj);
    LT_CU(cudaGetLastError());
    L.tick(3);
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
