// k_pencil.cu — batched Hermitian-definite pencil eigensolver (eigensolver.cpp:72-93).
//
// Per k-point (or per dense box pencil with N_b <= 32):
//   1. Hermitian check at 1e-10 max(1, max|.|) and symmetrisation of H and S
//      (periodic path only, as in solve_pencil; solve_box_dense has neither);
//   2. S = L L^H, right-looking Cholesky with Eigen's pivot test (x <= 0 fails);
//   3. A = L^-1 H L^-H through the explicit triangular inverse, A symmetrised;
//   4. complex Householder tridiagonalisation (zhetd2 scheme, real sub-diagonal);
//   5. all eigenvalues of the real tridiagonal by parallel multisection: P threads
//      per eigenvalue evaluate Sturm counts (the three-term recurrence of sturm3 on T
//      scaled by a power of two: one FMA per step, no reciprocal on the chain) at Q
//      points each per iteration, shrinking the bracket (P Q + 1)-fold.
// Eigenvalues come out ascending by construction. Results agree with the reference's
// SelfAdjointEigenSolver to O(eps ||A||).
//
// Vector mode (want_vectors, eigensolver.cpp:88-92): steps 4-5 are replaced by a parallel
// cyclic Jacobi on A (round-robin pair ordering, n/2 disjoint complex rotations per round,
// the rotation and stopping rule of a one-sided-phase Jacobi: phase a_pq to real, then the
// real rotation t = sign(tau) / (|tau| + sqrt(1 + tau^2))), which yields eigenvalues and an
// orthonormal Z together and is robust to degenerate eigenvalues; columns are sorted
// ascending and back-transformed X = L^-H Z (llt.matrixU().solve(Z)).
//
// Layout: a group of G threads per pencil; m0 padded to NM in {8, 16, 32} (the
// padding is an exactly decoupled block, H_pad = 0, S_pad = I, never touched by
// steps 4-5 which run on the leading m0 x m0 block); compile-time index maps.
#include "lt_device.cuh"
#include "lt_internal.cuh"

// Optional phase clocks (tools/pencil_phases.cu): group leader of pencil k records
// clock64() at phase boundaries into lt_pencil_prof[k][0..7].
#ifdef LT_PENCIL_PROFILE
__device__ long long lt_pencil_prof[8192][8];
__device__ long long lt_ms_prof[2];  // multisection of pencil 0, thread 0: cycles in Sturm counts, rounds
#define PPROF(i) \
    if (t == 0 && k < 8192) lt_pencil_prof[k][i] = clock64();
#else
#define PPROF(i)
#endif

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
// real-arithmetic variants (RE: a real symmetric pencil carried in the complex layout with
// zero imaginary parts, the box path): the same formulas without the imaginary terms
template <bool RE> __device__ __forceinline__ double2 cmul_(double2 a, double2 b) {
    if constexpr (RE) return make_double2(a.x * b.x, 0.0); else return cmul(a, b);
}
template <bool RE> __device__ __forceinline__ double2 cmulc_(double2 a, double2 b) {
    if constexpr (RE) return make_double2(a.x * b.x, 0.0); else return cmulc(a, b);
}
template <bool RE> __device__ __forceinline__ double2 cadd_(double2 a, double2 b) {
    if constexpr (RE) return make_double2(a.x + b.x, 0.0); else return cadd(a, b);
}
template <bool RE> __device__ __forceinline__ double2 csub_(double2 a, double2 b) {
    if constexpr (RE) return make_double2(a.x - b.x, 0.0); else return csub(a, b);
}
template <bool RE> __device__ __forceinline__ double2 cconj_(double2 a) {
    if constexpr (RE) return make_double2(a.x, 0.0); else return cconj(a);
}
template <bool RE> __device__ __forceinline__ double2 cscale_(double sc, double2 a) {
    if constexpr (RE) return make_double2(sc * a.x, 0.0); else return cscale(sc, a);
}
template <bool RE> __device__ __forceinline__ double cabs2_(double2 a) {
    if constexpr (RE) return a.x * a.x; else return cabs2(a);
}
template <bool RE> __device__ __forceinline__ double cabsr_(double2 a) {
    if constexpr (RE) return fabs(a.x); else return cabs_(a);
}

// Fused lattice DFT of one entry (single wrapped axis): F = sum_c w_c G[blk[c]] at offset
// `off` of the m0 x m0 generating blocks, c ascending (k_dft_axis2's first-axis sum); block
// indices from shared memory and eight (H, S) loads in flight per batch.
template <bool RE>
__device__ __forceinline__ void fused_dft_entry(const PencilDft& dft, const double2* tw, const int* blk, int mm,
                                                Index off, double2& ah, double2& as) {
    ah = make_double2(0.0, 0.0);
    as = make_double2(0.0, 0.0);
    int q = 0;
    for (; q + 7 < dft.nc; q += 8) {
        double vh[8], vs[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int b = blk[q + u];
            vh[u] = b >= 0 ? dft.GH[static_cast<Index>(b) * mm + off] : 0.0;
            vs[u] = b >= 0 ? dft.GS[static_cast<Index>(b) * mm + off] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            ah = cadd_<RE>(ah, cmul_<RE>(tw[q + u], make_double2(vh[u], 0.0)));
            as = cadd_<RE>(as, cmul_<RE>(tw[q + u], make_double2(vs[u], 0.0)));
        }
    }
    for (; q < dft.nc; ++q) {
        const int b = blk[q];
        const double vh = b >= 0 ? dft.GH[static_cast<Index>(b) * mm + off] : 0.0;
        const double vs = b >= 0 ? dft.GS[static_cast<Index>(b) * mm + off] : 0.0;
        ah = cadd_<RE>(ah, cmul_<RE>(tw[q], make_double2(vh, 0.0)));
        as = cadd_<RE>(as, cmul_<RE>(tw[q], make_double2(vs, 0.0)));
    }
}

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
    static_assert(kPencilDftMax > 0, "");
    double2 A[NM][NM + 1];
    double2 B[NM][NM + 1];
    double2 C[NM][NM + 1];
    double2 v[NM], w[NM];
    double d[NM], e2[NM], e[NM];
    double ix[NM], invd[NM];  // 1 / pivot, 1 / sqrt(pivot)
    double red[4][32];
    double scal[4];
    double2 tw[kPencilDftMax];  // fused DFT: twiddles of this k-point
    int blk[kPencilDftMax];     // fused DFT: stored block of each compressed offset (-1: none)
    // vector mode (parallel Jacobi): rotation of pair i = (jp[i], jq[i]); pair of index x
    double jc[NM / 2 + 1], js[NM / 2 + 1], jtr[NM / 2 + 1];
    double2 jph[NM / 2 + 1];
    int jp[NM / 2 + 1], jq[NM / 2 + 1], jrot[NM / 2 + 1], jpair[NM + 1], perm[NM];
    int rot[2];
};

// group reduction of NV values at once (one pair of barriers for all of them)
template <int G, int NV, bool MAX>
__device__ __forceinline__ void greduce(double (&v)[NV], double (*red)[32], int t, int slot) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            const double w = __shfl_xor_sync(0xffffffffu, v[q], o);
            v[q] = MAX ? fmax(v[q], w) : v[q] + w;
        }
    if constexpr (G > 32) {
        if ((t & 31) == 0)
#pragma unroll
            for (int q = 0; q < NV; ++q) red[q][t >> 5] = v[q];
        gsync<G>(slot);
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            double r = red[q][0];
#pragma unroll
            for (int w = 1; w < G / 32; ++w) r = MAX ? fmax(r, red[q][w]) : r + red[q][w];
            v[q] = r;
        }
        gsync<G>(slot);
    }
}

// 1/q: MUFU reciprocal seed + two Newton steps (within an ulp or two of 1/q) instead of
// the IEEE division subroutine on the dependent chains. Needs DBL_MIN <= |q| < 2^1022
// (safe_rcp falls back to the IEEE division outside that range).
__device__ __forceinline__ double fast_rcp(double q) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    double t = fma(-q, r, 1.0);
    r = fma(r, t, r);
    t = fma(-q, r, 1.0);
    return fma(r, t, r);
}
// 1/sqrt(x), 1/q: MUFU seed (2^-20) and one cubic correction, for normal arguments
__device__ __forceinline__ double pencil_rsqrt(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-x * y, y, 1.0);
    return fma(y * e, fma(e, 0.375, 0.5), y);
}
__device__ __forceinline__ double pencil_rcp(double q) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    const double e = fma(-q, r, 1.0);
    return fma(r, fma(e, e, e), r);
}
__device__ __forceinline__ double safe_rcp(double q) {
    const double a = fabs(q);
    return (a >= 1e-300 && a <= 1e300) ? fast_rcp(q) : 1.0 / q;
}

// Vector mode on the reduced matrix A (leading n x n): parallel cyclic Jacobi with the
// eigenvectors accumulated in C, then ascending order and X = L^-H Z (B holds the unscaled
// Cholesky factor, L[r][i] = B[r][i] invd[i]). Writes eig[k*n ..] and vec[k*n*n ..]
// (column-major, complex).
template <int NM, int G, int EPT>
__device__ void pencil_vectors(PSmem<NM>& sm, int n, int t, int slot, Index k, double* __restrict__ eig,
                               double2* __restrict__ vec) {
    auto& A = sm.A;
    auto& B = sm.B;
    auto& C = sm.C;
    // C = I; the stopping floor 1e-17 ||A||_F
    double fro[1] = {0.0};
#pragma unroll
    for (int u = 0; u < EPT; ++u) {
        const int e = t + G * u;
        if (e < NM * NM) {
            const int r = e % NM, c = e / NM;
            C[r][c] = make_double2(r == c ? 1.0 : 0.0, 0.0);
            if (r < n && c < n) fro[0] += cabs2(A[r][c]);
        }
    }
    if (t < 2) sm.rot[t] = 0;
    greduce<G, 1, false>(fro, sm.red, t, slot);  // also orders C and rot
    const double floor_abs = 1e-17 * sqrt(fro[0]);
    const int n2 = n + (n & 1);  // round-robin over an even count (index n: the idle slot)
    const int npair = n2 / 2;
    for (int sweep = 0; sweep < 60 && n > 1; ++sweep) {
        const int cur = sweep & 1;
        for (int round = 0; round < n2 - 1; ++round) {
            if (t < npair) {
                const int a = t, b = n2 - 1 - t;
                const int ia = a == 0 ? 0 : 1 + (a - 1 + round) % (n2 - 1);
                const int ib = b == 0 ? 0 : 1 + (b - 1 + round) % (n2 - 1);
                const int p = min(ia, ib), q = max(ia, ib);
                double c = 1.0, sn = 0.0, tr = 0.0;
                int rotated = 0;
                double2 cph = make_double2(1.0, 0.0);
                if (q < n) {
                    const double2 apq = A[p][q];
                    const double r = cabs_(apq);
                    const double app = A[p][p].x, aqq = A[q][q].x;
                    if (r > floor_abs && r > 1.1102230246251565e-16 * sqrt(fabs(app * aqq))) {
                        const double ir = 1.0 / r;
                        cph = make_double2(apq.x * ir, -apq.y * ir);  // conj(a_pq / r)
                        const double tau = (aqq - app) / (2.0 * r);
                        const double tt = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                        c = 1.0 / sqrt(1.0 + tt * tt);
                        sn = tt * c;
                        tr = tt * r;
                        rotated = 1;
                        sm.rot[cur] = 1;
                    }
                }
                sm.jp[t] = p;
                sm.jq[t] = q;
                sm.jc[t] = c;
                sm.js[t] = sn;
                sm.jtr[t] = tr;
                sm.jrot[t] = rotated;
                sm.jph[t] = cph;
                sm.jpair[p] = t;
                sm.jpair[q] = t;
            }
            gsync<G>(slot);
            // the next sweep's flag: every thread has passed this one's read of it
            if (round == 0 && t == 0) sm.rot[cur ^ 1] = 0;
            // J = D R per pair: J[p][p] = c, J[p][q] = s, J[q][p] = -s cph, J[q][q] = c cph;
            // A' = J^H A J entrywise from the 2 x 2 block of the two pairs, V' = V J
            double2 na[EPT], nv[EPT];
#pragma unroll
            for (int u = 0; u < EPT; ++u) {
                const int e = t + G * u;
                if (e < NM * NM) {
                    const int x = e % NM, y = e / NM;
                    if (x < n && y < n) {
                        const int P = sm.jpair[x], Q = sm.jpair[y];
                        const int xp = sm.jp[P], xq = sm.jq[P], yp = sm.jp[Q], yq = sm.jq[Q];
                        const double cx = sm.jc[P], sx = sm.js[P], cy = sm.jc[Q], sy = sm.js[Q];
                        const double2 phx = sm.jph[P], phy = sm.jph[Q];
                        // column x of J_P: (J[xp][x], J[xq][x]); column y of J_Q
                        double2 jx0, jx1, jy0, jy1;
                        if (x == xp) {
                            jx0 = make_double2(cx, 0.0);
                            jx1 = cscale(-sx, phx);
                        } else {
                            jx0 = make_double2(sx, 0.0);
                            jx1 = cscale(cx, phx);
                        }
                        if (y == yp) {
                            jy0 = make_double2(cy, 0.0);
                            jy1 = cscale(-sy, phy);
                        } else {
                            jy0 = make_double2(sy, 0.0);
                            jy1 = cscale(cy, phy);
                        }
                        const bool xin = xq < n, yin = yq < n;  // idle-slot partners carry J = 1
                        if (!xin) {
                            jx0 = make_double2(1.0, 0.0);
                            jx1 = make_double2(0.0, 0.0);
                        }
                        if (!yin) {
                            jy0 = make_double2(1.0, 0.0);
                            jy1 = make_double2(0.0, 0.0);
                        }
                        const int rx0 = xin ? xp : x, rx1 = xin ? xq : x, cy0 = yin ? yp : y, cy1 = yin ? yq : y;
                        // A' = sum conj(J[x'][x]) A[x'][y'] J[y'][y]
                        const double2 t0 = cadd(cmul(A[rx0][cy0], jy0), cmul(A[rx0][cy1], jy1));
                        const double2 t1 = cadd(cmul(A[rx1][cy0], jy0), cmul(A[rx1][cy1], jy1));
                        double2 r = cadd(cmulc(jx0, t0), cmulc(jx1, t1));
                        if (P == Q && sm.jrot[P]) {  // the rotated diagonal block, exactly
                            r = (x == y) ? make_double2(A[x][x].x + (x == xp ? -sm.jtr[P] : sm.jtr[P]), 0.0)
                                         : make_double2(0.0, 0.0);
                        }
                        na[u] = r;
                        nv[u] = cadd(cmul(C[x][cy0], jy0), cmul(C[x][cy1], jy1));
                    } else if (y < n) {
                        nv[u] = make_double2(0.0, 0.0);
                    }
                }
            }
            gsync<G>(slot);
#pragma unroll
            for (int u = 0; u < EPT; ++u) {
                const int e = t + G * u;
                if (e < NM * NM) {
                    const int x = e % NM, y = e / NM;
                    if (x < n && y < n) {
                        A[x][y] = na[u];
                        C[x][y] = nv[u];
                    }
                }
            }
            gsync<G>(slot);
        }
        if (sm.rot[cur] == 0) break;
    }
    // ascending order (ties by index): rank of each diagonal entry
    if (t < n) {
        const double dx = A[t][t].x;
        int rank = 0;
        for (int y = 0; y < n; ++y) {
            const double dy = A[y][y].x;
            rank += (dy < dx) || (dy == dx && y < t);
        }
        sm.perm[rank] = t;
        sm.d[rank] = dx;
    }
    gsync<G>(slot);
    // Z (sorted columns of C) into A
#pragma unroll
    for (int u = 0; u < EPT; ++u) {
        const int e = t + G * u;
        if (e < NM * NM) {
            const int r = e % NM, c = e / NM;
            if (r < n && c < n) A[r][c] = C[r][sm.perm[c]];
        }
    }
    gsync<G>(slot);
    // X = L^-H Z: row r final before step r; rows i < r take -= conj(L[r][i]) x_r with
    // x_r = A[r][.] invd[r]; the row scaling by invd is applied at the end
    for (int r = n - 1; r >= 1; --r) {
        const double ir = sm.invd[r];
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
            const int e = t + G * u;
            if (e < NM * NM) {
                const int i = e % NM, c = e / NM;
                if (i < r && c < n)
                    A[i][c] = csub(A[i][c], cscale(sm.invd[i] * ir, cmulc(B[r][i], A[r][c])));
            }
        }
        gsync<G>(slot);
    }
    const Index mmo = static_cast<Index>(n) * n;
#pragma unroll
    for (int u = 0; u < EPT; ++u) {
        const int e = t + G * u;
        if (e < NM * NM) {
            const int i = e % NM, c = e / NM;
            if (i < n && c < n) vec[k * mmo + i + c * n] = cscale(sm.invd[i], A[i][c]);
        }
    }
    for (int i = t; i < n; i += G) eig[k * n + i] = sm.d[i];
}

// Tridiagonal T (d, e) of an n x n pencil (n <= 32) -> the multisection's inputs, in place,
// one entry per lane of a full warp: exact power-of-two scale (max |d|, |e| in [0.5, 1)) for
// the three-term Sturm counts (the eigenvalues are unscaled exactly), e2 = e^2, the widened
// Gershgorin bracket scal[0..1], 1/scale in scal[2] and the absolute tolerance
// ulp * ||T|| (LAPACK dstebz's default ABSTOL) in scal[3]. Max / min reductions are exact,
// so the values equal those of a serial sweep.
__device__ void tridiag_prepare_warp(double* d, double* e, double* e2, double* scal, int n, int lane) {
    const bool in = lane < n, ine = lane + 1 < n;
    double dc = in ? d[lane] : 0.0, ec = ine ? e[lane] : 0.0;
    double mx = in ? fmax(fabs(dc), fabs(ec)) : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    int ex = mx > 0.0 ? static_cast<int>((__double_as_longlong(mx) >> 52) & 0x7ff) - 1022 : 0;
    ex = max(-1000, min(1000, ex));
    const double sc = __longlong_as_double(static_cast<long long>(1023 - ex) << 52);
    dc *= sc;
    ec *= sc;
    const double eprev = __shfl_up_sync(0xffffffffu, ec, 1);
    const double rad = (lane > 0 ? fabs(eprev) : 0.0) + (ine ? fabs(ec) : 0.0);
    double lo = in ? dc - rad : 1e300, hi = in ? dc + rad : -1e300;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    __syncwarp();
    if (in) d[lane] = dc;
    if (ine) {
        e[lane] = ec;
        e2[lane] = ec * ec;
    }
    if (lane == 0) {
        const double wid = fmax(hi - lo, fmax(fabs(lo), fabs(hi))) * 4.4e-16 * n + 1e-300;
        scal[0] = lo - wid;
        scal[1] = hi + wid;
        scal[2] = __longlong_as_double(static_cast<long long>(1023 + ex) << 52);  // 1 / sc
        scal[3] = 2.2e-16 * fmax(fabs(lo), fabs(hi));
    }
}

// Sturm counts of the scaled tridiagonal at Q shifts: sturm3<Q, 2>'s three-term recurrence
// p_{i+1} = (d_i - x) p_i - e2_{i-1} p_{i-1}, unrolled over the compile-time bound NM <= 32
// (steps i >= n run on padding and are masked out). The signs of p_1 .. p_n go into a bit
// mask and the sign changes are counted once per chain (tools/sturm_probe.cu: an integer
// count update per step costs more than the recurrence itself).
template <int Q, int NM>
__device__ __forceinline__ void sturm_fixed(const double* sd, const double* se2, int n, const double (&x)[Q],
                                            int (&cnt)[Q]) {
    static_assert(NM <= 32, "sign mask");
    double pv[Q], cv[Q];
    unsigned sg[Q];
#pragma unroll
    for (int j = 0; j < Q; ++j) {
        pv[j] = 1.0;
        cv[j] = sd[0] - x[j];
        sg[j] = static_cast<unsigned>(__double2hiint(cv[j])) >> 31;
    }
#pragma unroll
    for (int i = 1; i < NM; ++i) {
        const double di = sd[i], ei = se2[i - 1];
#pragma unroll
        for (int j = 0; j < Q; ++j) {
            const double nx = fma(di - x[j], cv[j], -ei * pv[j]);
            sg[j] |= (static_cast<unsigned>(__double2hiint(nx)) >> 31) << i;
            pv[j] = cv[j];
            cv[j] = nx;
        }
        if ((i & 3) == 0) {
#pragma unroll
            for (int j = 0; j < Q; ++j) {
                const int ex = ((__double2hiint(cv[j]) >> 20) & 0x7ff) - 1023;
                if (ex > 400 || ex < -400) {  // rare: exact power-of-two rescale of (cur, prev)
                    const double scl = __longlong_as_double(static_cast<long long>(1023 - ex) << 52);
                    cv[j] *= scl;
                    pv[j] *= scl;
                }
            }
        }
    }
    // bit b of sg: sign of p_{b+1}; sign changes of p_0 = 1, p_1, ..., p_n
    const unsigned live = n >= 32 ? 0xffffffffu : ((1u << n) - 1u);
#pragma unroll
    for (int j = 0; j < Q; ++j) cnt[j] = __popc((sg[j] ^ (sg[j] << 1)) & live);
}

// Parallel multisection over the G threads of a pencil group (t = 0 .. G-1, contiguous
// lanes): all n eigenvalues of the prepared tridiagonal, ascending, into eig[k m0 + i].
template <int G, int NM>
__device__ void pencil_multisection(const double* d, const double* e2, const double* scal, int n, int t, Index k,
                                    int m0, double* __restrict__ eig) {
    // 5. parallel multisection: P threads (contiguous lanes) x Q shifts per thread and
    //    eigenvalue; the bracket shrinks (P Q + 1)-fold per round.
#ifndef LT_PENCIL_Q
#define LT_PENCIL_Q 2  // shifts per thread: measured best (Q = 1, 4, 8 slower on the FP64 pipe)
#endif
    constexpr int Q = LT_PENCIL_Q;
    int P = 1;
    while (P * 2 <= 32 && P * 2 * n <= G) P *= 2;
    const double unscale = scal[2];
    const double atol = scal[3];
    const int per_round = G / P;  // eigenvalues handled concurrently
    const double inv_pts = 1.0 / static_cast<double>(P * Q + 1);
    for (int base = 0; base < n; base += per_round) {
        const int mi = base + t / P;  // eigenvalue index of this thread
        const int sub = t % P;
        const bool active = mi < n;
        double a = scal[0], b = scal[1];
        const unsigned lane = threadIdx.x & 31;
        const int gb = static_cast<int>(lane & ~static_cast<unsigned>(P - 1));
        const unsigned gmask = (P == 32) ? 0xffffffffu : (((1u << P) - 1u) << gb);
        for (int it = 0; it < 80; ++it) {
            double x[Q];
            int cnt[Q];
#pragma unroll
            for (int j = 0; j < Q; ++j) x[j] = a + (b - a) * (static_cast<double>(sub * Q + j + 1) * inv_pts);
#ifdef LT_PENCIL_PROFILE
            const long long c0 = clock64();
#endif
            if (active) {
                sturm_fixed<Q, NM>(d, e2, n, x, cnt);
            } else {
#pragma unroll
                for (int j = 0; j < Q; ++j) cnt[j] = 0;
            }
#ifdef LT_PENCIL_PROFILE
            if (t == 0 && k == 0) {
                long long c1;
                asm volatile("mov.u64 %0, %%clock64;" : "=l"(c1) : "r"(cnt[0]), "r"(cnt[Q - 1]) : "memory");
                lt_ms_prof[0] += c1 - c0;
                lt_ms_prof[1] += 1;
            }
#endif
            // first shift (in group order sub*Q + j, increasing x) whose count exceeds mi
            int fq = Q;
#pragma unroll
            for (int j = Q - 1; j >= 0; --j)
                if (cnt[j] > mi) fq = j;
            // candidate bracket if this thread holds the first such shift
            const double prev_last = __shfl_up_sync(0xffffffffu, x[Q - 1], 1);
            double clo = (sub > 0) ? prev_last : a, chi = x[0];
#pragma unroll
            for (int j = 1; j < Q; ++j)
                if (fq == j) {
                    clo = x[j - 1];
                    chi = x[j];
                }
            const unsigned bal = __ballot_sync(0xffffffffu, active && fq < Q) & gmask;
            const int src = bal ? (__ffs(bal) - 1) : (gb + P - 1);
            const double slo = __shfl_sync(0xffffffffu, clo, src);
            const double shi = __shfl_sync(0xffffffffu, chi, src);
            const double last = __shfl_sync(0xffffffffu, x[Q - 1], gb + P - 1);
            double na, nb;
            if (bal) {
                na = slo;
                nb = shi;
            } else {
                na = last;  // every shift is below the eigenvalue
                nb = b;
            }
            const bool done = !(nb - na > 2.2e-16 * fmax(fabs(na), fabs(nb)) + atol) || (na == a && nb == b);
            a = na;
            b = nb;
            if (__all_sync(0xffffffffu, done || !active)) {
#ifdef LT_PENCIL_PROFILE
                if (t == 0 && k < 8192) lt_pencil_prof[k][7] = it + 1;  // multisection rounds
#endif
                break;
            }
        }
        if (active && sub == 0) eig[k * m0 + mi] = 0.5 * (a + b) * unscale;
    }
}

}  // namespace

// Threads of a group own matrix entries e = t + G*u (row e % NM, column e / NM); the
// Householder mat-vec uses TPR = G / NM threads per row.
template <int NM, int G, int BS, bool VEC, bool RE = false>
__global__ void __launch_bounds__(BS) k_pencil(Index count, int m0, const double2* __restrict__ Hb,
                                                const double2* __restrict__ Sb, double* __restrict__ eig,
                                                unsigned long long* fail_key, int periodic_checks, PencilDft dft,
                                                double2* __restrict__ vec, PencilReadback rb) {
    constexpr int PPC = BS / G;                 // pencils per CTA
    constexpr int EPT = (NM * NM + G - 1) / G;  // matrix entries per thread
    constexpr int TPR = G / NM;                 // mat-vec threads per row
    static_assert(TPR >= 1 && TPR <= 32 && (TPR & (TPR - 1)) == 0, "row split");
    static_assert(G >= 32, "the tridiagonal preparation runs on the first warp of the group");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PSmem<NM>* all = reinterpret_cast<PSmem<NM>*>(smem_raw);
    const int slot = threadIdx.x / G;
    const int t = threadIdx.x % G;
    const Index k = static_cast<Index>(blockIdx.x) * PPC + slot;
    if (k >= count) return;
    PSmem<NM>& sm = all[slot];
    PPROF(0);
    auto& A = sm.A;
    auto& B = sm.B;
    auto& C = sm.C;
    const int n = m0;
    const int mm = m0 * m0;
    if (dft.nc > 0) {
        // fused lattice DFT (single wrapped axis): F[k] = sum_c w^(k comp[c] mod L) G[blk[c]],
        // c ascending, the sum of k_dft_axis2's first axis
        const Index j = dft.k0 + k;
        for (int c = t; c < dft.nc; c += G) {
            const Index mres = (j * dft.comp[c]) % dft.L;
            double sn, co;
            sincospi(-2.0 * static_cast<double>(mres) / static_cast<double>(dft.L), &sn, &co);
            sm.tw[c] = make_double2(co, sn);
            sm.blk[c] = static_cast<int>(dft.blk[c]);
        }
        gsync<G>(slot);
    }
#pragma unroll
    for (int u = 0; u < EPT; ++u) {
        const int e = t + G * u;
        if (e < NM * NM) {
            const int r = e % NM, c = e / NM;
            if (r < m0 && c < m0) {
                if (dft.nc > 0) {
                    double2 ah, as;
                    fused_dft_entry<RE>(dft, sm.tw, sm.blk, mm, r + c * m0, ah, as);
                    A[r][c] = ah;
                    B[r][c] = as;
                } else {
                    A[r][c] = Hb[k * mm + r + c * m0];
                    B[r][c] = Sb[k * mm + r + c * m0];
                }
            } else {
                A[r][c] = make_double2(0.0, 0.0);
                B[r][c] = make_double2(r == c ? 1.0 : 0.0, 0.0);
            }
        }
    }
    gsync<G>(slot);
    PPROF(1);
    int code = 0;
    if (periodic_checks) {
        double red4[4] = {0.0, 0.0, 0.0, 0.0};  // hmax, smax, hdev, sdev
        double2 va[EPT], vb[EPT];
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
            const int e = t + G * u;
            if (e < NM * NM) {
                const int r = e % NM, c = e / NM;
                const double2 a = A[r][c], at = A[c][r], b = B[r][c], bt = B[c][r];
                red4[0] = fmax(red4[0], cabsr_<RE>(a));
                red4[1] = fmax(red4[1], cabsr_<RE>(b));
                red4[2] = fmax(red4[2], cabsr_<RE>(csub_<RE>(a, cconj_<RE>(at))));
                red4[3] = fmax(red4[3], cabsr_<RE>(csub_<RE>(b, cconj_<RE>(bt))));
                va[u] = cscale_<RE>(0.5, cadd_<RE>(a, cconj_<RE>(at)));
                vb[u] = cscale_<RE>(0.5, cadd_<RE>(b, cconj_<RE>(bt)));
            }
        }
        greduce<G, 4, true>(red4, sm.red, t, slot);  // its barriers also order the reads above
        if (red4[2] > 1e-10 * fmax(1.0, red4[0]) || red4[3] > 1e-10 * fmax(1.0, red4[1])) code = 1;
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
    PPROF(2);
    // 2. right-looking Cholesky S = L L^H, unscaled: step kk subtracts
    //    B[r][kk] conj(B[c][kk]) / x_kk from the trailing lower triangle and leaves column kk
    //    unscaled, so one barrier per step suffices (L[r][kk] = B[r][kk] / sqrt(x_kk),
    //    applied implicitly below). Pivot test as Eigen's LLT: x <= 0 fails.
    if (code == 0) {
        for (int kk = 0; kk < n; ++kk) {
            const double x = B[kk][kk].x;
            if (!(x > 0.0)) {
                code = 2;
                break;
            }
            const double ixk = safe_rcp(x);
#pragma unroll
            for (int u = 0; u < EPT; ++u) {
                const int e = t + G * u;
                if (e < NM * NM) {
                    const int r = e % NM, c = e / NM;
                    if (c > kk && r >= c && r < n)
                        B[r][c] = csub_<RE>(B[r][c], cscale_<RE>(ixk, cmul_<RE>(B[r][kk], cconj_<RE>(B[c][kk]))));
                }
            }
            if (t == 0) sm.ix[kk] = ixk;
            gsync<G>(slot);
        }
    }
    if (code != 0) {
        if (t == 0) {
            atomicMin(fail_key, static_cast<unsigned long long>(k) * 4ull + static_cast<unsigned long long>(code));
            group_done(rb, count);
        }
        return;
    }
    for (int i = t; i < n; i += G) sm.invd[i] = 1.0 / sqrt(B[i][i].x);
    PPROF(3);
    // 3. A = L^-1 H L^-H by two right-looking forward substitutions (one barrier per step):
    //    Y = L^-1 H in place in A, then Z = L^-1 Y^H in C; A = Z^H, symmetrised.
    //    With L[r][i] = B[r][i] invd[i]: cur_r -= B[r][i] ix[i] cur_i, then y_r = cur_r invd[r].
    for (int i = 0; i + 1 < n; ++i) {
        const double ixi = sm.ix[i];
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
            const int e = t + G * u;
            if (e < NM * NM) {
                const int r = e % NM, c = e / NM;
                if (r > i && r < n && c < n) A[r][c] = csub_<RE>(A[r][c], cscale_<RE>(ixi, cmul_<RE>(B[r][i], A[i][c])));
            }
        }
        gsync<G>(slot);
    }
    gsync<G>(slot);  // sm.invd visible (n == 1 runs no step above)
#pragma unroll
    for (int u = 0; u < EPT; ++u) {
        const int e = t + G * u;
        if (e < NM * NM) {
            const int r = e % NM, c = e / NM;
            C[r][c] = (r < n && c < n) ? cscale_<RE>(sm.invd[c], cconj_<RE>(A[c][r])) : make_double2(0.0, 0.0);
        }
    }
    gsync<G>(slot);
    for (int i = 0; i + 1 < n; ++i) {
        const double ixi = sm.ix[i];
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
            const int e = t + G * u;
            if (e < NM * NM) {
                const int r = e % NM, c = e / NM;
                if (r > i && r < n && c < n) C[r][c] = csub_<RE>(C[r][c], cscale_<RE>(ixi, cmul_<RE>(B[r][i], C[i][c])));
            }
        }
        gsync<G>(slot);
    }
    {
        // A = Z^H with Z[r][c] = C[r][c] invd[r]; symmetrised: A_sym = (Z + Z^H) / 2
        double2 y[EPT];
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
            const int e = t + G * u;
            if (e < NM * NM) {
                const int r = e % NM, c = e / NM;
                y[u] = (r < n && c < n)
                           ? cscale_<RE>(0.5, cadd_<RE>(cscale_<RE>(sm.invd[r], C[r][c]), cconj_<RE>(cscale_<RE>(sm.invd[c], C[c][r]))))
                           : make_double2(0.0, 0.0);
            }
        }
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
            const int e = t + G * u;
            if (e < NM * NM) A[e % NM][e / NM] = y[u];
        }
        gsync<G>(slot);
    }
    PPROF(4);
    if constexpr (VEC) {
        pencil_vectors<NM, G, EPT>(sm, n, t, slot, k, eig, vec);
        if (t == 0) group_done(rb, count);
        return;
    }
    // 4. Householder tridiagonalisation of the leading n x n block (zhetd2, lower)
    const int row = t / TPR, part = t % TPR;
    for (int kk = 0; kk + 1 < n; ++kk) {
        const int m = n - kk - 1;  // reflector length (rows kk+1 .. n-1)
        // zlarfg on x = A[kk+1 .. n-1][kk]
        double xr[1] = {0.0};
        for (int i = kk + 2 + t; i < n; i += G) xr[0] += cabs2_<RE>(A[i][kk]);
        greduce<G, 1, false>(xr, sm.red, t, slot);
        const double xn2 = xr[0];
        const double2 x0 = A[kk + 1][kk];
        double beta;
        double2 tau;
        double2 scal;  // 1 / (x0 - beta)
        if (xn2 == 0.0 && x0.y == 0.0) {
            tau = make_double2(0.0, 0.0);
            beta = x0.x;
            scal = make_double2(0.0, 0.0);
        } else {
            // 1/nrm and 1/|x0 - beta|^2 from the MUFU seeds with one cubic correction each
            // (the step's dependent chain; IEEE sqrt / division outside the normal range)
            const double q = fma(x0.x, x0.x, fma(x0.y, x0.y, xn2));
            const bool nq = q >= 1e-290 && q <= 1e290;
            const double rq = nq ? pencil_rsqrt(q) : 1.0 / sqrt(q);
            const double nrm = q * rq;
            beta = x0.x >= 0.0 ? -nrm : nrm;
            const double ib = x0.x >= 0.0 ? -rq : rq;  // 1 / beta
            tau = make_double2((beta - x0.x) * ib, -x0.y * ib);
            const double2 den = make_double2(x0.x - beta, x0.y);
            const double dq = fma(den.x, den.x, den.y * den.y);
            const double id = nq ? pencil_rcp(dq) : 1.0 / dq;
            scal = make_double2(den.x * id, -den.y * id);
        }
        // v (index 0 <-> row kk+1)
        for (int i = t; i < m; i += G) sm.v[i] = i == 0 ? make_double2(1.0, 0.0) : cmul_<RE>(A[kk + 1 + i][kk], scal);
        gsync<G>(slot);
        if (tau.x != 0.0 || tau.y != 0.0) {
            // y = A22 v (TPR threads per row), then w = tau y - 1/2 |tau|^2 (v^H y) v
            double2 yi = make_double2(0.0, 0.0);
            if (row < m)
                for (int j = part; j < m; j += TPR) yi = cadd_<RE>(yi, cmul_<RE>(A[kk + 1 + row][kk + 1 + j], sm.v[j]));
#pragma unroll
            for (int o = TPR / 2; o > 0; o >>= 1) {
                yi.x += __shfl_xor_sync(0xffffffffu, yi.x, o);
                yi.y += __shfl_xor_sync(0xffffffffu, yi.y, o);
            }
            double vr[1] = {(row < m && part == 0) ? cmulc_<RE>(sm.v[row], yi).x : 0.0};  // Re(v^H y)
            greduce<G, 1, false>(vr, sm.red, t, slot);
            const double half = 0.5 * (tau.x * tau.x + tau.y * tau.y) * vr[0];
            if (row < m && part == 0) sm.w[row] = csub_<RE>(cmul_<RE>(tau, yi), cscale_<RE>(half, sm.v[row]));
            gsync<G>(slot);
            // A22 -= w v^H + v w^H
#pragma unroll
            for (int u = 0; u < EPT; ++u) {
                const int e = t + G * u;
                if (e < NM * NM) {
                    const int r = e % NM - kk - 1, c = e / NM - kk - 1;
                    if (r >= 0 && c >= 0 && r < m && c < m) {
                        const double2 upd = cadd_<RE>(cmul_<RE>(sm.w[r], cconj_<RE>(sm.v[c])), cmul_<RE>(sm.v[r], cconj_<RE>(sm.w[c])));
                        A[r + kk + 1][c + kk + 1] = csub_<RE>(A[r + kk + 1][c + kk + 1], upd);
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
    if (t == 0) sm.d[n - 1] = A[n - 1][n - 1].x;
    gsync<G>(slot);
    if (t < 32) tridiag_prepare_warp(sm.d, sm.e, sm.e2, sm.scal, n, t);
    gsync<G>(slot);
    PPROF(5);
    pencil_multisection<G, NM>(sm.d, sm.e2, sm.scal, n, t, k, m0, eig);
    PPROF(6);
    if (t == 0) group_done(rb, count);
}

template <int NM, int G, int BS, bool VEC, bool RE = false>
static void run_pencil(const Launch& L, Index count, Index m0, const double2* H, const double2* S, double* eig,
                       unsigned long long* fail_key, bool checks, const PencilDft& dft, double2* vec,
                       const PencilReadback& rb) {
    static_assert(BS % G == 0 && (G <= 32 || G % 32 == 0), "group layout");
    constexpr int PPC = BS / G;
    const size_t smem = sizeof(PSmem<NM>) * PPC;
    static bool attr = false;
    if (!attr) {
        LT_CU(cudaFuncSetAttribute(k_pencil<NM, G, BS, VEC, RE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
        attr = true;
    }
    const Index blocks = (count + PPC - 1) / PPC;
    Stage st_(L, "pencil");
    k_pencil<NM, G, BS, VEC, RE><<<static_cast<unsigned>(blocks), BS, smem, L.st>>>(
        count, static_cast<int>(m0), H, S, eig, fail_key, checks ? 1 : 0, dft, vec, rb);
    LT_CU(cudaGetLastError());
    L.tick();
}

// Group size per pencil (measured with tools/pencil_phases.cu): more threads per pencil
// only pay off for m0 <= 8 batches that cannot fill the GPU (16 multisection points per
// eigenvalue instead of 4); for larger blocks the extra threads lengthen every barrier of
// the Cholesky/Householder chains more than they shorten the bisection.
template <bool VEC>
static void dispatch_pencil(const Launch& L, Index count, Index m0, const double2* H, const double2* S, double* eig,
                            unsigned long long* fail_key, bool periodic_checks, const PencilDft& dft, double2* vec,
                            const PencilReadback& rb) {
    if (m0 <= 8) {
        // one pencil per 64-thread CTA while the batch is small (more SMs, fewer warps per
        // SM sharing the FP64 pipe), warp-per-pencil in 128-thread CTAs for large batches
        if (count <= 1184) run_pencil<8, 64, 64, VEC>(L, count, m0, H, S, eig, fail_key, periodic_checks, dft, vec, rb);
        else run_pencil<8, 32, 128, VEC>(L, count, m0, H, S, eig, fail_key, periodic_checks, dft, vec, rb);
    } else if (m0 <= 16) {
        run_pencil<16, 64, 256, VEC>(L, count, m0, H, S, eig, fail_key, periodic_checks, dft, vec, rb);
    } else if (m0 <= 32) {
        run_pencil<32, 256, 256, VEC>(L, count, m0, H, S, eig, fail_key, periodic_checks, dft, vec, rb);
    } else {
        fail(LT_EDIM, "pencil_eig: block size m0 > 32 is not supported by the batched solver");
    }
}

// a one-offset "lattice DFT" (offset 0, block 0, twiddle 1): lets a real dense pencil be
// read straight from its double arrays through the fused-DFT load path (no conversion launch)
__device__ const int64_t kPencilZeroComp[1] = {0};
__device__ const int kPencilZeroBlk[1] = {0};
PencilDft pencil_identity_source(const double* H, const double* S) {
    // symbol addresses resolved once per device (the first call runs eagerly, before any
    // capture of this path), not inside stream capture
    static void* pc[64] = {};
    static void* pb[64] = {};
    int dev = 0;
    LT_CU(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) fail(LT_EGENERIC, "pencil_identity_source: device index out of range");
    if (!pc[dev]) {
        LT_CU(cudaGetSymbolAddress(&pb[dev], kPencilZeroBlk));
        LT_CU(cudaGetSymbolAddress(&pc[dev], kPencilZeroComp));
    }
    PencilDft f;
    f.nc = 1;
    f.L = 1;
    f.k0 = 0;
    f.comp = static_cast<const int64_t*>(pc[dev]);
    f.blk = static_cast<const int*>(pb[dev]);
    f.GH = H;
    f.GS = S;
    return f;
}

void launch_pencil(const Launch& L, Index count, Index m0, const double2* H, const double2* S, double* eig,
                   unsigned long long* fail_key, bool periodic_checks, const PencilDft& dft, double2* vec,
                   const PencilReadback& rb, bool real) {
    if (count <= 0) return;
    if (real && !vec) {
        // real symmetric pencils (box, N_b <= 32): real arithmetic in the complex layout
        if (m0 <= 8) run_pencil<8, 64, 64, false, true>(L, count, m0, H, S, eig, fail_key, periodic_checks, dft, nullptr, rb);
        else if (m0 <= 16) run_pencil<16, 64, 256, false, true>(L, count, m0, H, S, eig, fail_key, periodic_checks, dft, nullptr, rb);
        else if (m0 <= 32) run_pencil<32, 256, 256, false, true>(L, count, m0, H, S, eig, fail_key, periodic_checks, dft, nullptr, rb);
        else fail(LT_EDIM, "pencil_eig: block size m0 > 32 is not supported by the batched solver");
        return;
    }
    if (dft.nc > kPencilDftMax) fail(LT_EGENERIC, "pencil_eig: fused DFT supports at most 64 stored offsets");
    if (vec) dispatch_pencil<true>(L, count, m0, H, S, eig, fail_key, periodic_checks, dft, vec, rb);
    else dispatch_pencil<false>(L, count, m0, H, S, eig, fail_key, periodic_checks, dft, nullptr, rb);
}

}  // namespace lt
