// k_fold.cu — residue-class correlations on DMMA, shared by the FEM tables and the
// periodic nuclear fold.
//
// For profiles a_mu, b_nu on a grid of J*n points (n points per unit cell) and an
// offset d in cells, the reference's 1D forms are sums over grid points i of
// a_mu(i) b_nu(i - d n). Splitting i = t + j n by residue t in [0, n):
//     C_t[d](mu, nu) = sum_j a_mu(t + j n) b_nu(t + (j - d) n)
// is, for each t, a set of (m0 x J)(J x m0) products (m8n8k4 DMMA tiles); the table is
// sum_t C_t[d] (FEM, nuclear of trivial-free paths) or sum_t V(t) C_t[d] (nuclear fold
// weighted by the effective potential). One CTA per residue t (and d-chunk) stages the
// t-strided profiles in shared memory.
//
// FEM (fem1d.cpp:19-32 via galerkin.cpp:208-223): a = pwl_mu, b = T pwl_nu where
// T = tridiag{lo, diag, lo}; each row value (T v)_i equals the reference's `row`
// bit for bit (absent neighbours add +0.0), so every term u_i * row_i is the
// reference's term; only the summation order differs.
#include <cstdlib>

#include "dmma.cuh"
#include "lt_device.cuh"
#include "lt_internal.cuh"

namespace lt {

// w_mass[nu][i+1], w_stiff[nu][i+1] = (T v_nu)(i) for i in [-1, Gbar]: one guard point
// each side, because a support touching the grid edge has (T v)(-1) = lo v(0) != 0 and the
// reference's supported tri_form (fem1d.cpp:19-32) runs to v.offset - 1 and v.end + 1.
__global__ void k_fem_apply(FemApplyJobs jobs, int m0) {
    const FemApplyJob& J = jobs.j[blockIdx.z];
    const int nu = blockIdx.y;
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x - 1;
    if (i > J.Gbar) return;
    const long long vlo = static_cast<long long>(J.lo[nu]), vhi = static_cast<long long>(J.hi[nu]);
    const double* v = J.pwl + nu * J.Gbar;
    const double h = J.hbar;
    const double mlo = h / 6.0, mdiag = (4.0 * h) / 6.0, slo = -1.0 / h, sdiag = 2.0 / h;
    double rm = 0.0, rs = 0.0;
    if (i - 1 >= vlo && i - 1 < vhi) {
        const double x = v[i - 1];
        rm = __dadd_rn(rm, __dmul_rn(mlo, x));
        rs = __dadd_rn(rs, __dmul_rn(slo, x));
    }
    if (i >= vlo && i < vhi) {
        const double x = v[i];
        rm = __dadd_rn(rm, __dmul_rn(mdiag, x));
        rs = __dadd_rn(rs, __dmul_rn(sdiag, x));
    }
    if (i + 1 >= vlo && i + 1 < vhi) {
        const double x = v[i + 1];
        rm = __dadd_rn(rm, __dmul_rn(mlo, x));
        rs = __dadd_rn(rs, __dmul_rn(slo, x));
    }
    J.wm[nu * (J.Gbar + 2) + i + 1] = rm;
    J.ws[nu * (J.Gbar + 2) + i + 1] = rs;
}

void launch_fem_apply(const Launch& L, const FemApplyJobs& jobs, int njobs, int m0) {
    long long gmax = 1;
    for (int k = 0; k < njobs; ++k) gmax = std::max(gmax, jobs.j[k].Gbar + 2);
    dim3 grid(static_cast<unsigned>((gmax + 255) / 256), m0, njobs);
    Stage st_(L, "fem_apply");
    k_fem_apply<<<grid, 256, 0, L.st>>>(jobs, m0);
    LT_CU(cudaGetLastError());
    L.tick();
}

// Residue-major slabs: slab[t][s][mu][c] with s = 0 the a-profiles (column c = j) and
// s = 1.. the b-profiles (column c = j' + 1, j' in [-1, J]); 32x32 tiles of (t, j) so the
// stride-n gathers become coalesced reads and writes.
__global__ void k_resfold_prep(ResFold f) {
    __shared__ double tile[32][33];
    const long long J = f.J, ldj = resfold_ldj(J);
    const int m0p = (f.m0 + 7) / 8 * 8;
    const int src = blockIdx.z / m0p, mu = blockIdx.z % m0p;
    const long long t0 = static_cast<long long>(blockIdx.x) * 32;
    const long long c0 = static_cast<long long>(blockIdx.y) * 32;  // slab column
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;        // 32 x 8 threads
    const long long gb = f.bguard ? f.G + 2 : f.G;
    const double* bsrc = src == 2 ? f.b[1] : f.b[0];
    for (int r = ty; r < 32; r += 8) {
        const long long c = c0 + r, t = t0 + tx;
        double v = 0.0;
        if (mu < f.m0 && t < f.n) {
            if (src == 0) {
                if (c < J) v = f.a[mu * f.G + t + (c + f.jw0) * f.n];
            } else {
                const long long gi = t + (c - 1 + f.jw0) * f.n;  // j' = c - 1
                if (c < J + 2) {
                    if (f.bguard) {
                        if (gi >= -1 && gi <= f.G) v = bsrc[mu * gb + gi + 1];
                    } else if (gi >= 0 && gi < f.G) {
                        v = bsrc[mu * gb + gi];
                    }
                }
            }
        }
        tile[r][tx] = v;
    }
    __syncthreads();
    const int ns = 1 + f.nb;
    for (int r = ty; r < 32; r += 8) {
        const long long t = t0 + r, c = c0 + tx;
        if (t < f.n && c < ldj) f.slab[((t * ns + src) * m0p + mu) * ldj + c] = tile[tx][r];
    }
}

// CTA per (residue t, d-chunk). out[q][(t*nd + di)*mm + e] = weight * C_t[d](mu, nu) for
// each b-source q, with di = d - dlo over [dlo, dhi]; weight = V[e][t] (mode 1) or 1.
// The slab is zero beyond the stored columns (resfold_ldj leaves >= 3 spare), so the
// k-steps run without bounds checks; two accumulator sets alternate to halve the DMMA
// dependency chain.
template <int NB>
__global__ void __launch_bounds__(256) k_resfold(ResFold f) {
    extern __shared__ double sh[];
    const long long t = blockIdx.x;
    const int dc = blockIdx.y;
    const int J = static_cast<int>(f.J);
    const int ldj = static_cast<int>(resfold_ldj(f.J));
    const int m0p = (f.m0 + 7) / 8 * 8;
    const double* As = sh;                // [m0p][ldj]
    const double* Bs = sh + m0p * ldj;    // [NB][m0p][ldj], column j' + 1 for j' in [-1, J]
    const long long tot = static_cast<long long>(1 + NB) * m0p * ldj;
    double* Vs = sh + tot;                // fused weights V[e] for this residue (f.W set)
    // the supports are needed after the staging below: their loads go first, so they share its
    // round trip to L2 instead of adding one between two barriers
    long long sup_l = 0, sup_h = 0;
    if (f.sup_lo && threadIdx.x < f.m0) {
        sup_l = static_cast<long long>(f.sup_lo[threadIdx.x]);
        sup_h = static_cast<long long>(f.sup_hi[threadIdx.x]);
    }
    if (f.slab) {
        const double2* srcp = reinterpret_cast<const double2*>(f.slab + t * tot);
        double2* dstp = reinterpret_cast<double2*>(sh);
        for (int idx = threadIdx.x; idx < tot / 2; idx += blockDim.x) dstp[idx] = srcp[idx];
    } else {
        // short residue classes: gather the strided rows directly (same values as the slab);
        // U addresses per thread first, then U loads in flight, then the stores
        const long long gb = f.bguard ? f.G + 2 : f.G;
        constexpr int U = 8;
        const int itot = static_cast<int>(tot), plane = m0p * ldj;
        for (int i0 = threadIdx.x; i0 < itot; i0 += U * blockDim.x) {
            const double* ptr[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int idx = i0 + u * static_cast<int>(blockDim.x);
                ptr[u] = nullptr;
                if (idx >= itot) continue;
                const int src = idx / plane, rem = idx % plane;
                const int mu = rem / ldj, c = rem % ldj;
                if (mu >= f.m0) continue;
                if (src == 0) {
                    if (c < J) ptr[u] = f.a + mu * f.G + t + (c + f.jw0) * f.n;
                } else if (c < J + 2) {
                    const double* bsrc = src == 2 ? f.b[1] : f.b[0];
                    const long long gi = t + (c - 1 + f.jw0) * f.n;
                    if (f.bguard) {
                        if (gi >= -1 && gi <= f.G) ptr[u] = bsrc + mu * gb + gi + 1;
                    } else if (gi >= 0 && gi < f.G) {
                        ptr[u] = bsrc + mu * gb + gi;
                    }
                }
            }
            double v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = ptr[u] ? __ldg(ptr[u]) : 0.0;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int idx = i0 + u * static_cast<int>(blockDim.x);
                if (idx < itot) sh[idx] = v[u];
            }
        }
    }
    if (f.W) {
        // V[e][t] = sum_r W[r][e] P[r][t] (the rank sum folded into an effective potential):
        // every thread takes one (e, rank part) with four independent accumulators so the
        // loads of a part are in flight together; parts are summed in fixed order below
        const int mme = f.m0 * f.m0;
        const int parts = max(1, static_cast<int>(blockDim.x) / mme);
        double* Vp = Vs + mme;  // [parts][mme]
        for (int idx = threadIdx.x; idx < mme * parts; idx += blockDim.x) {
            const int e = idx % mme, part = idx / mme;
            const int r0 = (f.Rtot * part) / parts, r1 = (f.Rtot * (part + 1)) / parts;
            double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
            int r = r0;
            // eight (W, P) pairs in flight per round trip, four accumulators
            for (; r + 7 < r1; r += 8) {
                double w[8], pv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    w[u] = f.W[(r + u) * mme + e];
                    pv[u] = f.P[(r + u) * f.prow + t];
                }
                v0 = fma(w[0], pv[0], v0);
                v1 = fma(w[1], pv[1], v1);
                v2 = fma(w[2], pv[2], v2);
                v3 = fma(w[3], pv[3], v3);
                v0 = fma(w[4], pv[4], v0);
                v1 = fma(w[5], pv[5], v1);
                v2 = fma(w[6], pv[6], v2);
                v3 = fma(w[7], pv[7], v3);
            }
            for (; r + 3 < r1; r += 4) {
                v0 = fma(f.W[(r + 0) * mme + e], f.P[(r + 0) * f.prow + t], v0);
                v1 = fma(f.W[(r + 1) * mme + e], f.P[(r + 1) * f.prow + t], v1);
                v2 = fma(f.W[(r + 2) * mme + e], f.P[(r + 2) * f.prow + t], v2);
                v3 = fma(f.W[(r + 3) * mme + e], f.P[(r + 3) * f.prow + t], v3);
            }
            for (; r < r1; ++r) v0 = fma(f.W[r * mme + e], f.P[r * f.prow + t], v0);
            Vp[part * mme + e] = (v0 + v1) + (v2 + v3);
        }
        __syncthreads();
        for (int e = threadIdx.x; e < mme; e += blockDim.x) {
            double v = Vp[e];
            for (int part = 1; part < parts; ++part) v += Vp[part * mme + e];
            Vs[e] = v;
        }
    }
    __shared__ long long slo[32], shi[32];
    if (f.sup_lo && threadIdx.x < f.m0) {
        slo[threadIdx.x] = sup_l;
        shi[threadIdx.x] = sup_h;
    }
    __syncthreads();  // the staged rows, V and the supports
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, tq = lane & 3;
    const int ntile = m0p / 8;
    const int nd = f.dhi - f.dlo + 1;
    const int dlo = f.dlo + dc * f.dchunk;
    const int dhi = min(f.dhi, dlo + f.dchunk - 1);
    const int tasks = (dhi - dlo + 1) * ntile * ntile;
    const int mm = f.m0 * f.m0;
    // j - d must stay in the stored range: [0, J) or, with guards, [-1, J]
    const int glo = f.bguard ? -1 : 0, ghi = f.bguard ? J + 1 : J;
    // per 8-function tile: the j range of residue t where some function of the tile is
    // non-zero (a side: t + j n in [lo, hi); b side: t + j' n in [lo - w, hi + w))
    __shared__ int tja[2][4], tjb[2][4];
    if (threadIdx.x < 2 * ntile && threadIdx.x < 8) {
        const int side = threadIdx.x / ntile, tile = threadIdx.x % ntile;
        int jl = 1 << 30, jh = -(1 << 30);
        if (f.sup_lo) {
            const long long w = side ? f.bwiden : 0;
            for (int u = 0; u < 8; ++u) {
                const int mu = tile * 8 + u;
                if (mu >= f.m0) break;
                if (slo[mu] >= shi[mu]) continue;
                const long long lo = slo[mu] - w;
                const long long hi = shi[mu] + w;
                auto cdiv = [&](long long x) { return x >= 0 ? (x + f.n - 1) / f.n : -((-x) / f.n); };
                jl = min(jl, static_cast<int>(cdiv(lo - t) - f.jw0));
                jh = max(jh, static_cast<int>(cdiv(hi - t) - f.jw0));
            }
        } else {
            jl = -1;
            jh = J + 1;
        }
        (side ? tjb : tja)[0][tile] = jl;
        (side ? tjb : tja)[1][tile] = jh;
    }
    __syncthreads();
    for (int task = warp; task < tasks; task += blockDim.x >> 5) {
        const int d = dlo + task / (ntile * ntile);
        const int mt = (task / ntile) % ntile, nt = task % ntile;
        double c0[NB][2], c1[NB][2];
#pragma unroll
        for (int q = 0; q < NB; ++q) c0[q][0] = c0[q][1] = c1[q][0] = c1[q][1] = 0.0;
        const int j0 = max(max(0, d + glo), max(tja[0][mt], tjb[0][nt] + d));
        const int j1 = max(j0, min(min(J, d + ghi), min(tja[1][mt], tjb[1][nt] + d)));
        const double* ap = As + (mt * 8 + g) * ldj + j0 + tq;
        const double* bp = Bs + (nt * 8 + g) * ldj + j0 + tq - d + 1;
        const int steps = (j1 - j0 + 3) >> 2;
        int s = 0;
        for (; s + 1 < steps; s += 2) {
            const double a0 = ap[4 * s], a1 = ap[4 * s + 4];
#pragma unroll
            for (int q = 0; q < NB; ++q) {
                dmma_m8n8k4(c0[q], a0, bp[q * m0p * ldj + 4 * s]);
                dmma_m8n8k4(c1[q], a1, bp[q * m0p * ldj + 4 * s + 4]);
            }
        }
        if (s < steps) {
            const double a0 = ap[4 * s];
#pragma unroll
            for (int q = 0; q < NB; ++q) dmma_m8n8k4(c0[q], a0, bp[q * m0p * ldj + 4 * s]);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int mu = mt * 8 + g, nu = nt * 8 + 2 * tq + i;
            if (mu >= f.m0 || nu >= f.m0) continue;
            const int e = mu + nu * f.m0;
            const double wgt = f.W ? Vs[e] : (f.V ? f.V[e * f.n + t] : 1.0);
            const long long o = (t * nd + (d - f.dlo)) * static_cast<long long>(mm) + e;
            f.out[0][o] = wgt * (c0[0][i] + c1[0][i]);
            if (NB == 2) f.out[1][o] = wgt * (c0[NB - 1][i] + c1[NB - 1][i]);
        }
    }
}

// warp per (q, di, e): sum over residues t in fixed lane order; optional mirror (d -> -d,
// (mu,nu) -> (nu,mu)) for symmetric folds computed on d >= 0 only
__global__ void k_resfold_reduce(ResFold f, int mirror) {
    const int lane = threadIdx.x & 31;
    const long long w = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int mm = f.m0 * f.m0;
    const int nd = f.dhi - f.dlo + 1;
    if (w >= static_cast<long long>(f.nb) * nd * mm) return;
    const int q = static_cast<int>(w / (static_cast<long long>(nd) * mm));
    const int di = static_cast<int>((w / mm) % nd), e = static_cast<int>(w % mm);
    double s = 0.0;
    const double* src = q ? f.out[1] : f.out[0];
    double* dst = q ? f.res[1] : f.res[0];
    for (long long t = lane; t < f.n; t += 32) s += src[(t * nd + di) * static_cast<long long>(mm) + e];
    s = warp_sum(s);
    if (lane == 0) {
        const int d = f.dlo + di;
        dst[(d + f.band) * static_cast<long long>(mm) + e] = s;
        if (mirror && d > 0) {
            const int mu = e % f.m0, nu = e / f.m0;
            dst[(f.band - d) * static_cast<long long>(mm) + nu + mu * f.m0] = s;
        }
    }
}

void launch_resfold(const Launch& L, const ResFold& f_in, bool reduce, bool mirror, const char* name) {
    ResFold f = f_in;
    const int m0p = (f.m0 + 7) / 8 * 8;
    const size_t mme = static_cast<size_t>(f.m0) * f.m0;
    const size_t vparts = f.W ? std::max<size_t>(1, 256 / mme) : 0;
    const size_t smem = sizeof(double) * (static_cast<size_t>(m0p) * resfold_ldj(f.J) * (1 + f.nb) +
                                          (f.W ? mme * (1 + vparts) : 0));
    static size_t attr[2] = {0, 0};
    if (f.nb < 1 || f.nb > 2) fail(LT_EGENERIC, "residue fold: nb must be 1 or 2");
    if (smem > 48 * 1024 && smem > attr[f.nb - 1] && smem <= 227 * 1024) {
        if (f.nb == 1)
            LT_CU(cudaFuncSetAttribute(k_resfold<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        else
            LT_CU(cudaFuncSetAttribute(k_resfold<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        attr[f.nb - 1] = smem;
    }
    const int nd = f.dhi - f.dlo + 1;
    const int nchunks = (nd + f.dchunk - 1) / f.dchunk;
    if (smem > 227 * 1024)
        fail(LT_EGENERIC, "residue fold: one residue class (" + std::to_string(smem) +
                              " bytes) exceeds the 227 KB shared-memory limit");
    if (f.slab) {
        Stage st_(L, "fold_prep");
        dim3 gp(static_cast<unsigned>((f.n + 31) / 32), static_cast<unsigned>((resfold_ldj(f.J) + 31) / 32), (1 + f.nb) * m0p);
        k_resfold_prep<<<gp, 256, 0, L.st>>>(f);
        LT_CU(cudaGetLastError());
        L.tick();
    }
    dim3 grid(static_cast<unsigned>(f.n), nchunks);
    {
        Stage st_(L, name);
        if (f.nb == 1) k_resfold<1><<<grid, 256, smem, L.st>>>(f);
        else k_resfold<2><<<grid, 256, smem, L.st>>>(f);
        LT_CU(cudaGetLastError());
        L.tick();
    }
    if (reduce) {
        const long long warps = static_cast<long long>(f.nb) * nd * f.m0 * f.m0;
        Stage st2_(L, "resfold_reduce");
        k_resfold_reduce<<<static_cast<unsigned>((warps + 7) / 8), 256, 0, L.st>>>(f, mirror ? 1 : 0);
        LT_CU(cudaGetLastError());
        L.tick();
    }
}

}  // namespace lt
