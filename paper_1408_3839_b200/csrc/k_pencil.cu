// k_pencil.cu — batched Hermitian-definite pencil eigensolver (eigensolver.cpp:72-93).
//
// Per k-point (or per dense box pencil with N_b <= 32):
//   1. Hermitian check at 1e-10 max(1, max|.|) and symmetrisation of H and S
//      (periodic path only, as in solve_pencil; solve_box_dense has neither);
//   2. S = L L^H, right-looking Cholesky with Eigen's pivot test (x <= 0 fails);
//   3. A = L^-1 H L^-H through the explicit triangular inverse, A symmetrised;
//   4. complex Householder tridiagonalisation (zhetd2 scheme, real sub-diagonal);
//   5. all eigenvalues of the real tridiagonal by parallel multisection: P threads
//      per eigenvalue evaluate Sturm counts (LDL^T pivots with LAPACK's pivmin guard)
//      at P interior points per iteration, shrinking the bracket (P+1)-fold.
// Eigenvalues come out ascending by construction. Results agree with the reference's
// SelfAdjointEigenSolver to O(eps ||A||).
//
// Layout: a group of G threads per pencil; m0 padded to NM in {8, 16, 32} (the
// padding is an exactly decoupled block, H_pad = 0, S_pad = I, never touched by
// steps 4-5 which run on the leading m0 x m0 block); compile-time index maps.
#include "lt_device.cuh"
#include "lt_internal.cuh"

namespace lt {

namespace {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // conj(a) * b
    return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double s, double2 a) { return make_double2(s * a.x, s * a.y); }
__device__ __forceinline__ double cabs2(double2 a) { return a.x * a.x + a.y * a.y; }
__device__ __forceinline__ double cabs_(double2 a) { return sqrt(a.x * a.x + a.y * a.y); }

template <int G>
__device__ __forceinline__ void gsync(int slot) {
    if constexpr (G == 32) {
        __syncwarp();
    } else if constexpr (G >= 256) {
        __syncthreads();
    } else {
        asm volatile("bar.sync %0, %1;" ::"r"(slot + 1), "r"(G) : "memory");
    }
}

template <int NM>
struct PSmem {
    double2 A[NM][NM + 1];
    double2 B[NM][NM + 1];
    double2 C[NM][NM + 1];
    double2 v[NM], w[NM];
    double d[NM], e2[NM], e[NM];
    double red[8];
    double2 tau;
    double scal[4];
};

template <int G, bool MAX>
__device__ __forceinline__ double greduce(double v, double* red, int t, int slot) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double w = __shfl_xor_sync(0xffffffffu, v, o);
        v = MAX ? fmax(v, w) : v + w;
    }
    if constexpr (G == 32) {
        return __shfl_sync(0xffffffffu, v, 0);
    } else {
        if ((t & 31) == 0) red[t >> 5] = v;
        gsync<G>(slot);
        double r = red[0];
#pragma unroll
        for (int w = 1; w < G / 32; ++w) r = MAX ? fmax(r, red[w]) : r + red[w];
        gsync<G>(slot);
        return r;
    }
}

// number of eigenvalues of the symmetric tridiagonal (d, e^2) strictly below x
__device__ __forceinline__ int sturm_count(const double* d, const double* e2, int n, double x, double pivmin) {
    int cnt = 0;
    double q = d[0] - x;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
    for (int i = 1; i < n; ++i) {
        q = (d[i] - x) - e2[i - 1] / q;
        if (fabs(q) < pivmin) q = -pivmin;
        cnt += q < 0.0;
    }
    return cnt;
}

}  // namespace

template <int NM, int G>
__global__ void __launch_bounds__(256) k_pencil(Index count, int m0, const double2* __restrict__ Hb,
                                                const double2* __restrict__ Sb, double* __restrict__ eig,
                                                unsigned long long* fail_key, int periodic_checks) {
    constexpr int PPC = (G >= 256) ? 1 : 256 / G;
    constexpr int EPT = (NM * NM + G - 1) / G;  // matrix entries per thread
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PSmem<NM>* all = reinterpret_cast<PSmem<NM>*>(smem_raw);
    const int slot = threadIdx.x / G;
    const int t = threadIdx.x % G;
    const Index k = static_cast<Index>(blockIdx.x) * PPC + slot;
    if (k >= count) return;
    PSmem<NM>& sm = all[slot];
    auto& A = sm.A;
    auto& B = sm.B;
    auto& C = sm.C;
    const int n = m0;
    const int mm = m0 * m0;
#pragma unroll
    for (int u = 0; u < EPT; ++u) {
        const int e = t + G * u;
        if (e < NM * NM) {
            const int r = e % NM, c = e / NM;
            if (r < m0 && c < m0) {
                A[r][c] = Hb[k * mm + r + c * m0];
                B[r][c] = Sb[k * mm + r + c * m0];
            } else {
                A[r][c] = make_double2(0.0, 0.0);
                B[r][c] = make_double2(r == c ? 1.0 : 0.0, 0.0);
            }
        }
    }
    gsync<G>(slot);
    int code = 0;
    if (periodic_checks) {
        double hmax = 0.0, smax = 0.0, hdev = 0.0, sdev = 0.0;
        double2 va[EPT], vb[EPT];
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
            const int e = t + G * u;
            if (e < NM * NM) {
                const int r = e % NM, c = e / NM;
                const double2 a = A[r][c], at = A[c][r], b = B[r][c], bt = B[c][r];
                hmax = fmax(hmax, cabs_(a));
                smax = fmax(smax, cabs_(b));
                hdev = fmax(hdev, cabs_(csub(a, cconj(at))));
                sdev = fmax(sdev, cabs_(csub(b, cconj(bt))));
                va[u] = cscale(0.5, cadd(a, cconj(at)));
                vb[u] = cscale(0.5, cadd(b, cconj(bt)));
            }
        }
        hmax = greduce<G, true>(hmax, sm.red, t, slot);
        smax = greduce<G, true>(smax, sm.red, t, slot);
        hdev = greduce<G, true>(hdev, sm.red, t, slot);
        sdev = greduce<G, true>(sdev, sm.red, t, slot);
        if (hdev > 1e-10 * fmax(1.0, hmax) || sdev > 1e-10 * fmax(1.0, smax)) code = 1;
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
            const int e = t + G * u;
            if (e < NM * NM) {
                A[e % NM][e / NM] = va[u];
                B[e % NM][e / NM] = vb[u];
            }
        }
        gsync<G>(slot);
    }
    // 2. right-looking Cholesky of B (lower triangle)
    if (code == 0) {
        for (int kk = 0; kk < n; ++kk) {
            const double x = B[kk][kk].x;
            if (!(x > 0.0)) {
                code = 2;
                break;
            }
            const double dd = sqrt(x);
            const double inv = 1.0 / dd;
            gsync<G>(slot);
            for (int i = kk + 1 + t; i < n; i += G) B[i][kk] = cscale(inv, B[i][kk]);
            if (t == 0) B[kk][kk] = make_double2(dd, 0.0);
            gsync<G>(slot);
#pragma unroll
            for (int u = 0; u < EPT; ++u) {
                const int e = t + G * u;
                if (e < NM * NM) {
                    const int r = e % NM, c = e / NM;
                    if (c > kk && r >= c && r < n) B[r][c] = csub(B[r][c], cmul(B[r][kk], cconj(B[c][kk])));
                }
            }
            gsync<G>(slot);
        }
    }
    if (code != 0) {
        if (t == 0) atomicMin(fail_key, static_cast<unsigned long long>(k) * 4ull + static_cast<unsigned long long>(code));
        return;
    }
    // 3. C = L^-1 (thread c owns column c), then A = C H C^H, symmetrised, into A
    for (int c = t; c < n; c += G) {
        for (int i = 0; i < n; ++i) {
            if (i < c) {
                C[i][c] = make_double2(0.0, 0.0);
                continue;
            }
            double2 s = make_double2(i == c ? 1.0 : 0.0, 0.0);
            for (int j = c; j < i; ++j) s = csub(s, cmul(B[i][j], C[j][c]));
            C[i][c] = cscale(1.0 / B[i][i].x, s);
        }
    }
    gsync<G>(slot);
    {
        double2 y[EPT];
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
            const int e = t + G * u;
            if (e < NM * NM) {
                const int r = e % NM, c = e / NM;
                double2 s = make_double2(0.0, 0.0);
                if (r < n && c < n)
                    for (int a = 0; a <= r; ++a) s = cadd(s, cmul(C[r][a], A[a][c]));
                y[u] = s;
            }
        }
        gsync<G>(slot);
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
            const int e = t + G * u;
            if (e < NM * NM) B[e % NM][e / NM] = y[u];  // B := L^-1 H  (L no longer needed)
        }
        gsync<G>(slot);
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
            const int e = t + G * u;
            if (e < NM * NM) {
                const int r = e % NM, c = e / NM;
                double2 s = make_double2(0.0, 0.0);
                if (r < n && c < n)
                    for (int b = 0; b <= c; ++b) s = cadd(s, cmul(B[r][b], cconj(C[c][b])));
                y[u] = s;
            }
        }
        gsync<G>(slot);
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
            const int e = t + G * u;
            if (e < NM * NM) A[e % NM][e / NM] = y[u];
        }
        gsync<G>(slot);
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
            const int e = t + G * u;
            if (e < NM * NM) {
                const int r = e % NM, c = e / NM;
                y[u] = cscale(0.5, cadd(A[r][c], cconj(A[c][r])));
            }
        }
        gsync<G>(slot);
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
            const int e = t + G * u;
            if (e < NM * NM) A[e % NM][e / NM] = y[u];
        }
        gsync<G>(slot);
    }
    // 4. Householder tridiagonalisation of the leading n x n block (zhetd2, lower)
    for (int kk = 0; kk + 1 < n; ++kk) {
        const int m = n - kk - 1;  // reflector length (rows kk+1 .. n-1)
        // zlarfg on x = A[kk+1 .. n-1][kk]
        double xn2 = 0.0;
        for (int i = kk + 2 + t; i < n; i += G) xn2 += cabs2(A[i][kk]);
        xn2 = greduce<G, false>(xn2, sm.red, t, slot);
        const double2 x0 = A[kk + 1][kk];
        double beta;
        double2 tau;
        double2 scal;  // 1 / (x0 - beta)
        if (xn2 == 0.0 && x0.y == 0.0) {
            tau = make_double2(0.0, 0.0);
            beta = x0.x;
            scal = make_double2(0.0, 0.0);
        } else {
            const double nrm = sqrt(x0.x * x0.x + x0.y * x0.y + xn2);
            beta = x0.x >= 0.0 ? -nrm : nrm;
            tau = make_double2((beta - x0.x) / beta, -x0.y / beta);
            const double2 den = make_double2(x0.x - beta, x0.y);
            const double id = 1.0 / (den.x * den.x + den.y * den.y);
            scal = make_double2(den.x * id, -den.y * id);
        }
        // v (index 0 <-> row kk+1)
        for (int i = t; i < m; i += G) sm.v[i] = i == 0 ? make_double2(1.0, 0.0) : cmul(A[kk + 1 + i][kk], scal);
        gsync<G>(slot);
        if (tau.x != 0.0 || tau.y != 0.0) {
            // y = A22 v, then w = tau y - 1/2 |tau|^2 (v^H y) v
            double2 yi = make_double2(0.0, 0.0);
            const int i = t;
            if (i < m) {
                for (int j = 0; j < m; ++j) yi = cadd(yi, cmul(A[kk + 1 + i][kk + 1 + j], sm.v[j]));
            }
            double part = i < m ? cmulc(sm.v[i], yi).x : 0.0;  // Re(v^H y); v^H A v is real
            const double vy = greduce<G, false>(part, sm.red, t, slot);
            const double half = 0.5 * (tau.x * tau.x + tau.y * tau.y) * vy;
            if (i < m) sm.w[i] = csub(cmul(tau, yi), cscale(half, sm.v[i]));
            gsync<G>(slot);
            // A22 -= w v^H + v w^H
#pragma unroll
            for (int u = 0; u < EPT; ++u) {
                const int e = t + G * u;
                if (e < NM * NM) {
                    const int r = e % NM - kk - 1, c = e / NM - kk - 1;
                    if (r >= 0 && c >= 0 && r < m && c < m) {
                        const double2 upd = cadd(cmul(sm.w[r], cconj(sm.v[c])), cmul(sm.v[r], cconj(sm.w[c])));
                        A[r + kk + 1][c + kk + 1] = csub(A[r + kk + 1][c + kk + 1], upd);
                    }
                }
            }
        }
        if (t == 0) {
            sm.d[kk] = A[kk][kk].x;
            sm.e[kk] = beta;
        }
        gsync<G>(slot);
    }
    if (t == 0) {
        sm.d[n - 1] = A[n - 1][n - 1].x;
        double emax = 0.0;
        for (int i = 0; i + 1 < n; ++i) {
            sm.e2[i] = sm.e[i] * sm.e[i];
            emax = fmax(emax, sm.e2[i]);
        }
        // Gershgorin bracket, widened, and LAPACK's pivmin = safmin * max(1, max e^2)
        double lo = 1e300, hi = -1e300;
        for (int i = 0; i < n; ++i) {
            const double r = (i > 0 ? fabs(sm.e[i - 1]) : 0.0) + (i + 1 < n ? fabs(sm.e[i]) : 0.0);
            lo = fmin(lo, sm.d[i] - r);
            hi = fmax(hi, sm.d[i] + r);
        }
        const double wid = fmax(hi - lo, fmax(fabs(lo), fabs(hi))) * 4.4e-16 * n + 1e-300;
        sm.scal[0] = lo - wid;
        sm.scal[1] = hi + wid;
        sm.scal[2] = 2.2250738585072014e-308 * fmax(1.0, emax);
    }
    gsync<G>(slot);
    // 5. parallel multisection: P threads per eigenvalue (same warp, contiguous lanes)
    int P = 1;
    while (P * 2 <= 32 && P * 2 * n <= G) P *= 2;
    const double pivmin = sm.scal[2];
    const int per_round = G / P;  // eigenvalues handled concurrently
    for (int base = 0; base < n; base += per_round) {
        const int mi = base + t / P;   // eigenvalue index of this thread
        const int sub = t % P;
        const bool active = mi < n;
        double a = sm.scal[0], b = sm.scal[1];
        const unsigned lane = threadIdx.x & 31;
        const unsigned gmask = (P == 32) ? 0xffffffffu : (((1u << P) - 1u) << (lane & ~static_cast<unsigned>(P - 1)));
        for (int it = 0; it < 80; ++it) {
            const double x = a + (b - a) * (static_cast<double>(sub + 1) / static_cast<double>(P + 1));
            const int cnt = active ? sturm_count(sm.d, sm.e2, n, x, pivmin) : 0;
            const unsigned bal = __ballot_sync(0xffffffffu, active && cnt > mi) & gmask;
            // x values of the group are increasing with sub: the first x with count > mi
            // bounds the eigenvalue above, its predecessor (or a) below. Shuffles are
            // executed unconditionally by the whole warp (groups may take different cases).
            const int gb = static_cast<int>(lane & ~static_cast<unsigned>(P - 1));
            const int j = bal ? (__ffs(bal) - 1 - gb) : P;  // P: none of the points is above
            const double xb = __shfl_sync(0xffffffffu, x, gb + min(j, P - 1));
            const double xa = __shfl_sync(0xffffffffu, x, gb + max(min(j, P) - 1, 0));
            double na, nb;
            if (j == P) {
                na = xb;  // last point
                nb = b;
            } else {
                nb = xb;
                na = j > 0 ? xa : a;
            }
            const bool done = !(nb - na > 2.2e-16 * fmax(fabs(na), fabs(nb))) || (na == a && nb == b);
            a = na;
            b = nb;
            if (__all_sync(0xffffffffu, done || !active)) break;
        }
        if (active && sub == 0) eig[k * m0 + mi] = 0.5 * (a + b);
    }
}

template <int NM, int G>
static void run_pencil(const Launch& L, Index count, Index m0, const double2* H, const double2* S, double* eig,
                       unsigned long long* fail_key, bool checks) {
    constexpr int PPC = (G >= 256) ? 1 : 256 / G;
    const size_t smem = sizeof(PSmem<NM>) * PPC;
    static bool attr = false;
    if (!attr) {
        LT_CU(cudaFuncSetAttribute(k_pencil<NM, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        attr = true;
    }
    const Index blocks = (count + PPC - 1) / PPC;
    Stage st_(L, "pencil");
    k_pencil<NM, G><<<static_cast<unsigned>(blocks), 256, smem, L.st>>>(count, static_cast<int>(m0), H, S, eig,
                                                                         fail_key, checks ? 1 : 0);
    LT_CU(cudaGetLastError());
    L.tick();
}

void launch_pencil(const Launch& L, Index count, Index m0, const double2* H, const double2* S, double* eig,
                   unsigned long long* fail_key, bool periodic_checks) {
    if (count <= 0) return;
    if (m0 <= 8) run_pencil<8, 32>(L, count, m0, H, S, eig, fail_key, periodic_checks);
    else if (m0 <= 16) run_pencil<16, 64>(L, count, m0, H, S, eig, fail_key, periodic_checks);
    else if (m0 <= 32) run_pencil<32, 256>(L, count, m0, H, S, eig, fail_key, periodic_checks);
    else fail(LT_EDIM, "pencil_eig: block size m0 > 32 is not supported by the batched solver");
}

}  // namespace lt
