// k_assemble.cu — block combine and placement (galerkin.cpp:252-285, :311-358, :360-425)
// fused with the core-Hamiltonian combine H = 0.5 Laplace - 1.0 Nuclear, S = Mass
// (tools/commands.cpp:51-59, eigensolver.cpp:37-67).
//
// Per block (k, d) and entry e = mu + nu m0:
//   mass = (M0 * M1) * M2
//   lap  = ((S0*M1)*M2 + (M0*S1)*M2) + (M0*M1)*S2            (Laplace = A x S x S + ...)
//   nuc  = sum_r w_r ((T0 * T1) * T2)   or the S2 block N[k][d]
//   H    = 0.5*lap + (-1.0)*nuc,  S = mass
// Box blocks land in the dense N_b x N_b column-major matrix at (k m0 + mu, (k+d) m0 + nu);
// periodic blocks land in std::map order of kidx = ((d mod L) + L) mod L.
#include "lt_device.cuh"
#include "lt_internal.cuh"

namespace lt {

struct FillDev {
    Index m0, Rtot, L[3], band[3], width[3];
    const double* massT[3];
    const double* stiffT[3];
    const double* T[3];
    const double* potw;
    const double* N;
    const double* Npart;
    Index Nres, Nnd;
    int s2_dir, mode, periodic, nuc_mode;
    double kin;
    double* out0;
    double* out1;
    int64_t* kidx;
    Index Nb;
};

__device__ __forceinline__ Index pair_index(const FillDev& f, int l, Index k, Index d) {
    return f.periodic ? (d + f.band[l]) : (k * f.width[l] + d + f.band[l]);
}

// grid: x = block index (box: cell*nd + dlin ; periodic: dlin), threads over e
__global__ void k_fill(FillDev f) {
    const Index nd = f.width[0] * f.width[1] * f.width[2];
    const Index bidx = blockIdx.x;
    const Index dlin = bidx % nd;
    const Index lin = f.periodic ? 0 : bidx / nd;
    Index d[3], k[3], m[3];
    d[0] = dlin / (f.width[1] * f.width[2]) - f.band[0];
    d[1] = (dlin / f.width[2]) % f.width[1] - f.band[1];
    d[2] = dlin % f.width[2] - f.band[2];
    k[0] = lin / (f.L[1] * f.L[2]);
    k[1] = (lin / f.L[2]) % f.L[1];
    k[2] = lin % f.L[2];
    for (int l = 0; l < 3; ++l) {
        m[l] = k[l] + d[l];
        if (!f.periodic && (m[l] < 0 || m[l] >= f.L[l])) return;
    }
    const Index mm = f.m0 * f.m0;
    const bool want_ms = f.mode == 0 || f.mode == 1 || f.mode == 2 || f.mode == 5;
    const bool want_nuc = f.mode == 0 || f.mode == 3 || f.mode == 5;
    Index pidx[3];
    for (int l = 0; l < 3; ++l) pidx[l] = pair_index(f, l, k[l], d[l]);
    for (Index e = threadIdx.x; e < mm; e += blockDim.x) {
        double mass = 0.0, lap = 0.0, nuc = 0.0;
        if (want_ms) {
            const double M0 = f.massT[0][(d[0] + f.band[0]) * mm + e];
            const double M1 = f.massT[1][(d[1] + f.band[1]) * mm + e];
            const double M2 = f.massT[2][(d[2] + f.band[2]) * mm + e];
            const double S0 = f.stiffT[0][(d[0] + f.band[0]) * mm + e];
            const double S1 = f.stiffT[1][(d[1] + f.band[1]) * mm + e];
            const double S2 = f.stiffT[2][(d[2] + f.band[2]) * mm + e];
            mass = __dmul_rn(__dmul_rn(M0, M1), M2);
            const double t0 = __dmul_rn(__dmul_rn(S0, M1), M2);
            const double t1 = __dmul_rn(__dmul_rn(M0, S1), M2);
            const double t2 = __dmul_rn(__dmul_rn(M0, M1), S2);
            lap = __dadd_rn(__dadd_rn(t0, t1), t2);
        }
        if (want_nuc) {
            if (f.nuc_mode == 1 && f.Npart) {
                // periodic residue-fold partials summed here in t order (d < 0: the
                // (mu,nu)-transposed mirror of |d|)
                const int l = f.s2_dir;
                const Index ad = d[l] < 0 ? -d[l] : d[l];
                const Index ee = d[l] < 0 ? (e / f.m0) + (e % f.m0) * f.m0 : e;
                double acc = 0.0;
                const double* src = f.Npart + ad * mm + ee;
                const Index step = f.Nnd * mm;
                Index t = 0;
                for (; t + 7 < f.Nres; t += 8) {  // eight loads in flight, summed in t order
                    double v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) v[u] = src[(t + u) * step];
#pragma unroll
                    for (int u = 0; u < 8; ++u) acc += v[u];
                }
                for (; t < f.Nres; ++t) acc += src[t * step];
                nuc = acc;
            } else if (f.nuc_mode == 1) {
                const int l = f.s2_dir;
                nuc = f.N[(k[l] * f.width[l] + d[l] + f.band[l]) * mm + e];
            } else if (f.nuc_mode == 2) {
                nuc = f.N[dlin * mm + e];
            } else {
                double acc = 0.0;
                const double* T0 = f.T[0] + pidx[0] * f.Rtot * mm + e;
                const double* T1 = f.T[1] + pidx[1] * f.Rtot * mm + e;
                const double* T2 = f.T[2] + pidx[2] * f.Rtot * mm + e;
                for (Index r = 0; r < f.Rtot; ++r)
                    acc = __dadd_rn(acc, __dmul_rn(f.potw[r], __dmul_rn(__dmul_rn(T0[r * mm], T1[r * mm]), T2[r * mm])));
                nuc = acc;
            }
        }
        double v0 = 0.0, v1 = 0.0;
        switch (f.mode) {
            case 0: v0 = __dadd_rn(__dmul_rn(f.kin, lap), __dmul_rn(-1.0, nuc)); v1 = mass; break;
            case 5: v0 = __dadd_rn(__dmul_rn(f.kin, lap), __dmul_rn(-1.0, nuc)); break;  // H only
            case 1: v0 = lap; break;
            case 2: v0 = mass; break;
            default: v0 = nuc; break;
        }
        if (f.periodic) {
            Index slot = 0;
            for (int l = 0; l < 3; ++l) slot = slot * f.width[l] + (d[l] >= 0 ? d[l] : f.width[l] + d[l]);
            f.out0[slot * mm + e] = v0;
            if (f.mode == 0) f.out1[slot * mm + e] = v1;
            if (e == 0)
                for (int l = 0; l < 3; ++l) f.kidx[3 * slot + l] = ((d[l] % f.L[l]) + f.L[l]) % f.L[l];
        } else {
            const Index mu = e % f.m0, nu = e / f.m0;
            const Index mlin = (m[0] * f.L[1] + m[1]) * f.L[2] + m[2];
            const Index row = lin * f.m0 + mu, col = mlin * f.m0 + nu;
            f.out0[row + col * f.Nb] = v0;
            if (f.mode == 0) f.out1[row + col * f.Nb] = v1;
        }
    }
}

void launch_fill(const Launch& L, const FillArgs& a, Index Nb, Index nblocks) {
    FillDev f{};
    f.m0 = a.m0;
    f.Rtot = a.Rtot;
    for (int l = 0; l < 3; ++l) {
        f.L[l] = a.L[l];
        f.band[l] = a.band[l];
        f.width[l] = a.width[l];
        f.massT[l] = a.massT[l];
        f.stiffT[l] = a.stiffT[l];
        f.T[l] = a.T[l];
    }
    f.potw = a.potw;
    f.N = a.N;
    f.Npart = a.Npart;
    f.Nres = a.Nres;
    f.Nnd = a.Nnd;
    f.s2_dir = a.s2_dir;
    f.nuc_mode = a.nuc_mode;
    f.mode = a.mode;
    f.kin = a.kin;
    f.periodic = a.periodic ? 1 : 0;
    f.out0 = a.out0;
    f.out1 = a.out1;
    f.kidx = a.kidx;
    f.Nb = Nb;
    const Index mm = a.m0 * a.m0;
    const int th = static_cast<int>(std::min<Index>(256, ((mm + 31) / 32) * 32));
    Stage st_(L, "fill");
    k_fill<<<static_cast<unsigned>(nblocks), th, 0, L.st>>>(f);
    LT_CU(cudaGetLastError());
    L.tick();
}

// out[i][e] = wa a[ia[i]][e] + wb b[ib[i]][e]  (missing index -> 0), eigensolver.cpp:48-51, :60-64
__global__ void k_axpby_map(Index nout, Index mm, double wa, const double* __restrict__ a, const int64_t* __restrict__ ia,
                            double wb, const double* __restrict__ b, const int64_t* __restrict__ ib,
                            double* __restrict__ out) {
    const Index idx = static_cast<Index>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= nout * mm) return;
    const Index i = idx / mm, e = idx % mm;
    const Index xa = ia ? ia[i] : i;
    const Index xb = ib ? ib[i] : i;
    const bool has_a = xa >= 0, has_b = xb >= 0;
    const double va = has_a ? a[xa * mm + e] : 0.0;
    const double vb = has_b ? b[xb * mm + e] : 0.0;
    double r;
    if (has_a) r = __dadd_rn(__dmul_rn(wa, va), __dmul_rn(wb, vb));  // wa*blk + wb*block_or_zero
    else r = __dmul_rn(wb, vb);                                      // wb*blk for b-only keys
    out[idx] = r;
}

void launch_axpby_map(const Launch& L, Index nout, Index mm, double wa, const double* a, const int64_t* ia, double wb,
                      const double* b, const int64_t* ib, double* out) {
    const Index tot = nout * mm;
    Stage st_(L, "axpby");
    k_axpby_map<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, L.st>>>(nout, mm, wa, a, ia, wb, b, ib, out);
    LT_CU(cudaGetLastError());
    L.tick();
}

}  // namespace lt
