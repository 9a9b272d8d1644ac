// k_pencil_lane.cu — batched 8 x 8 Hermitian-definite pencils for batches that fill the GPU
// on their own (c5: 4096 k-points): solve_pencil, eigensolver.cpp:72-93.
//
// The group-per-pencil kernel (k_pencil.cu) spends its issue slots on the reductions,
// shuffles and barriers that coordinate 32 threads around one small pencil (c5, ncu: 8.5 k
// warp instructions per pencil, issue-active 67 %). Here a CTA of four warps owns 32 pencils
// with the pencil index in the LANE: every warp instruction advances 32 pencils, and the four
// warps split each pencil's work by columns (warp q: columns q and q + 4), exchanging only
// through shared memory at a few CTA barriers:
//   load      cp.async of the 2 x 64 complex entries of the 32 pencils (all in flight)
//   check     |X - X^H| <= 1e-10 max(1, max|X|) for H and S (on squared magnitudes) and the
//             symmetrisation 0.5 (X + X^H) (H into the working matrix, S into registers)
//   Cholesky  S = L L^H, right-looking, in registers, by every warp (pivot test x <= 0 as
//             Eigen's LLT); each warp needs all of L for its columns below
//   reduce    Y = L^-1 H (warp q: columns q, q + 4, in place), barrier, Z = L^-1 Y^H
//             (= L^-1 H L^-H; warp q: columns q, q + 4, from rows of Y) -> A, registers
//   tridiag   zhetd2 (lower) Householder reduction of A to a real tridiagonal (d, e): the
//             columns meet in shared memory and warp q reduces pencils 8q .. 8q+7 on its own
//             (a dependent chain of 7 steps per pencil: no barriers inside it)
//   eig       Sturm bisection on (d, e^2) scaled by a power of two: thread (q, lane) finds
//             eigenvalues q and q + 4 of pencil `lane` (the three-term recurrence of
//             lt_device.cuh's sturm3, no division on the chain), a fixed 53 rounds (enough
//             for k_pencil's absolute tolerance from any Gershgorin bracket); ascending by
//             construction
// Shared memory is slot-major ([slot][lane], 32 consecutive doubles per slot): conflict-free.
//
// Input blocks are read at H[k * ks + e * es] (complex, entry e = r + c N column-major):
// ks = N^2, es = 1 for the k-major layout of the lattice DFT; ks = 1, es = K for the
// entry-major layout k_dft_fused writes for this kernel (coalesced across the warp).
#include "lt_device.cuh"
#include "lt_internal.cuh"

// Optional phase clocks (tools/lane_phases.cu): thread 0 of CTA b records clock64() at the
// phase boundaries into lt_lane_prof[b][0..7].
#ifdef LT_LANE_PROFILE
__device__ long long lt_lane_prof[1024][8];
#define LPROF(i) \
    if (threadIdx.x == 0 && blockIdx.x < 1024) lt_lane_prof[blockIdx.x][i] = clock64();
#else
#define LPROF(i)
#endif

namespace lt {

#ifndef LT_LANE_WARPS
#define LT_LANE_WARPS 8
#endif
constexpr int kLaneWarps = LT_LANE_WARPS;  // warps per CTA (32 pencils); warp q owns columns q + kLaneWarps h
constexpr int kLaneCols = 8 / kLaneWarps;

namespace {

// 1/sqrt(x) and 1/q from the MUFU approximations (2^-20 relative, measured on B200) and one
// cubic correction each: y (1 + e/2 + 3e^2/8), e = 1 - x y^2; r (1 + e + e^2), e = 1 - q r
// (|e| <= 2^-20: error ~2^-59 before rounding). Arguments must be normal (ftz).
__device__ __forceinline__ double lane_rsqrt(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-x * y, y, 1.0);
    return fma(y * e, fma(e, 0.375, 0.5), y);
}

__device__ __forceinline__ double lane_rcp(double q) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    const double e = fma(-q, r, 1.0);
    return fma(r, fma(e, e, e), r);
}

__device__ __forceinline__ void lane_cp16(void* dst, const void* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}

// shared memory plan (doubles, each slot x 32 lanes)
template <int N>
struct LaneSmem {
    static constexpr int kRaw = 0;                   // 2 N^2 complex: raw H then raw S; later A
    static constexpr int kY = kRaw + 4 * N * N;      // N^2 complex (Re plane, Im plane): H -> Y
    static constexpr int kD = kY + 2 * N * N;        // d[N]
    static constexpr int kE = kD + N;                // e[N] (beta)
    static constexpr int kHc = kE + N;               // kLaneWarps x (hmax2, hdev2)
    static constexpr int kSc = kHc + 2 * kLaneWarps;  // kLaneWarps x (smax2, sdev2)
    static constexpr int kSlots = kSc + 2 * kLaneWarps;
};

}  // namespace

template <int N>
__global__ void __launch_bounds__(32 * kLaneWarps) k_pencil_lane(Index count, const double2* __restrict__ Hs,
                                                                 const double2* __restrict__ Ss, Index ks, Index es,
                                                                 double* __restrict__ eig,
                                                                 unsigned long long* fail_key, PencilReadback rb,
                                                                 Index ngroups) {
    static_assert(N == kLaneWarps * kLaneCols, "column split");
    using SM = LaneSmem<N>;
    extern __shared__ __align__(16) double lane_sm[];
    const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
    const Index k = static_cast<Index>(blockIdx.x) * 32 + lane;
    const bool valid = k < count;
    const Index kk = valid ? k : count - 1;  // idle lanes recompute a valid pencil; results dropped
    double* sl = lane_sm + lane;             // slot s of this lane's pencil: sl[s * 32]
#define SLOT(s) sl[(s) * 32]
#define YR(r, c) SLOT(SM::kY + (r) + (c) * N)
#define YI(r, c) SLOT(SM::kY + N * N + (r) + (c) * N)
    const double2* raw = reinterpret_cast<const double2*>(lane_sm) + lane;  // raw[e * 32]
    LPROF(0);
    // ---- load: warp q issues entries q, q + 4, ... of H and S -------------------------------
    {
        const double2* hp = Hs + kk * ks;
        const double2* sp = Ss + kk * ks;
        double2* dst = reinterpret_cast<double2*>(lane_sm) + lane;
#pragma unroll 8
        for (int e = q; e < N * N; e += kLaneWarps) {
            lane_cp16(dst + e * 32, hp + e * es);
            lane_cp16(dst + (N * N + e) * 32, sp + e * es);
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    LPROF(1);
    // ---- check + symmetrisation: H columns q, q + 4 by this warp; all of S by every warp ---
    {
        double hmax2 = 0.0, hdev2 = 0.0;
#pragma unroll
        for (int h = 0; h < kLaneCols; ++h) {
            const int c = q + kLaneWarps * h;
#pragma unroll
            for (int r = 0; r < N; ++r) {
                if (r < c) continue;
                const double2 a = raw[(r + c * N) * 32], at = raw[(c + r * N) * 32];
                hmax2 = fmax(hmax2, fmax(fma(a.x, a.x, a.y * a.y), fma(at.x, at.x, at.y * at.y)));
                const double hx = a.x - at.x, hy = a.y + at.y;
                hdev2 = fmax(hdev2, fma(hx, hx, hy * hy));
                const double hr = 0.5 * (a.x + at.x), hi = 0.5 * (a.y - at.y);
                YR(r, c) = hr;
                YI(r, c) = r == c ? 0.0 : hi;
                if (r != c) {
                    YR(c, r) = hr;
                    YI(c, r) = -hi;
                }
            }
        }
        SLOT(SM::kHc + 2 * q) = hmax2;
        SLOT(SM::kHc + 2 * q + 1) = hdev2;
    }
    {
        double smax2 = 0.0, sdev2 = 0.0;
#pragma unroll
        for (int h = 0; h < kLaneCols; ++h) {
            const int c = q + kLaneWarps * h;
#pragma unroll
            for (int r = 0; r < N; ++r) {
                if (r < c) continue;
                const double2 b = raw[(N * N + r + c * N) * 32], bt = raw[(N * N + c + r * N) * 32];
                smax2 = fmax(smax2, fmax(fma(b.x, b.x, b.y * b.y), fma(bt.x, bt.x, bt.y * bt.y)));
                const double sx = b.x - bt.x, sy = b.y + bt.y;
                sdev2 = fmax(sdev2, fma(sx, sx, sy * sy));
            }
        }
        SLOT(SM::kSc + 2 * q) = smax2;
        SLOT(SM::kSc + 2 * q + 1) = sdev2;
    }
    double lr[N][N], li[N][N];  // lower triangle of S, then of L (r > c)
#pragma unroll
    for (int c = 0; c < N; ++c)
#pragma unroll
        for (int r = c; r < N; ++r) {
            const double2 b = raw[(N * N + r + c * N) * 32], bt = raw[(N * N + c + r * N) * 32];
            lr[r][c] = 0.5 * (b.x + bt.x);
            li[r][c] = r == c ? 0.0 : 0.5 * (b.y - bt.y);
        }
    int code = 0;  // 2: Cholesky pivot (here); 1: non-Hermitian H or S (from the partials, at the end)
    LPROF(2);
    // ---- Cholesky S = L L^H (every warp) -------------------------------------------------------
    double idg[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
        double x = lr[j][j];
        if (!(x > 0.0)) code = 2;
        if (!(x > 0.0)) x = 1.0;  // keep a dropped pencil's arithmetic finite
        const double id = lane_rsqrt(x);
        idg[j] = id;
#pragma unroll
        for (int r = j + 1; r < N; ++r) {
            lr[r][j] *= id;
            li[r][j] *= id;
        }
#pragma unroll
        for (int c = j + 1; c < N; ++c)
#pragma unroll
            for (int r = c; r < N; ++r) {  // S_rc -= L_rj conj(L_cj)
                lr[r][c] = fma(-lr[r][j], lr[c][j], fma(-li[r][j], li[c][j], lr[r][c]));
                if (r != c) li[r][c] = fma(-li[r][j], lr[c][j], fma(lr[r][j], li[c][j], li[r][c]));
            }
    }
    __syncthreads();  // symmetrised H complete
    LPROF(3);
    // ---- Y = L^-1 H, columns q and q + 4 (right-looking: independent rows per step) ----------
#pragma unroll
    for (int h = 0; h < kLaneCols; ++h) {
        const int c = q + kLaneWarps * h;
        double yr[N], yi[N];
#pragma unroll
        for (int i = 0; i < N; ++i) {
            yr[i] = YR(i, c);
            yi[i] = YI(i, c);
        }
#pragma unroll
        for (int j = 0; j < N; ++j) {
            yr[j] *= idg[j];
            yi[j] *= idg[j];
#pragma unroll
            for (int i = j + 1; i < N; ++i) {  // y_i -= L_ij y_j
                yr[i] = fma(-lr[i][j], yr[j], fma(li[i][j], yi[j], yr[i]));
                yi[i] = fma(-lr[i][j], yi[j], fma(-li[i][j], yr[j], yi[i]));
            }
        }
#pragma unroll
        for (int i = 0; i < N; ++i) {
            YR(i, c) = yr[i];
            YI(i, c) = yi[i];
        }
    }
    __syncthreads();
    LPROF(4);
    // ---- A = lower(L^-1 Y^H), columns q and q + 4: L z = conj(Y[c][.]) ------------------------
    // owned columns in registers: a[h][r] = A[r][q + 4h], r >= q + 4h
    double ar[kLaneCols][N], ai[kLaneCols][N];
#pragma unroll
    for (int h = 0; h < kLaneCols; ++h) {
        const int c = q + kLaneWarps * h;
        double zr[N], zi[N];
#pragma unroll
        for (int i = 0; i < N; ++i) {
            zr[i] = YR(c, i);
            zi[i] = -YI(c, i);
        }
#pragma unroll
        for (int j = 0; j < N; ++j) {
            zr[j] *= idg[j];
            zi[j] *= idg[j];
#pragma unroll
            for (int i = j + 1; i < N; ++i) {
                zr[i] = fma(-lr[i][j], zr[j], fma(li[i][j], zi[j], zr[i]));
                zi[i] = fma(-lr[i][j], zi[j], fma(-li[i][j], zr[j], zi[i]));
            }
        }
#pragma unroll
        for (int r = 0; r < N; ++r) {
            ar[h][r] = zr[r];
            ai[h][r] = zi[r];
        }
    }
    LPROF(5);
    // ---- Householder tridiagonalisation (zhetd2, lower) --------------------------------------
    // The reduction is a chain of dependent steps; split by columns it would need two CTA
    // barriers per step. Instead the owned columns go to shared memory (the raw blocks are
    // dead) and warp q reduces pencils 8q .. 8q+7 alone, one pencil per lane (lanes >= 8
    // repeat lanes 0-7 and write nothing): no barriers, all four SMSPs busy.
    {
        double* al = lane_sm;  // A lower, slot-major [2 N^2][32] in the raw area
#pragma unroll
        for (int h = 0; h < kLaneCols; ++h) {
            const int c = q + kLaneWarps * h;
#pragma unroll
            for (int r = 0; r < N; ++r) {
                if (r < c) continue;
                al[(r + c * N) * 32 + lane] = ar[h][r];
                al[(N * N + r + c * N) * 32 + lane] = ai[h][r];
            }
        }
    }
    __syncthreads();
    {
        constexpr int kPer = 32 / kLaneWarps;  // pencils per warp
        const int pp = q * kPer + (lane & (kPer - 1));
        const double* al = lane_sm + pp;
        double xr[N][N], xi[N][N];  // lower triangle of A (r >= c)
#pragma unroll
        for (int c = 0; c < N; ++c)
#pragma unroll
            for (int r = c; r < N; ++r) {
                xr[r][c] = al[(r + c * N) * 32];
                xi[r][c] = r == c ? 0.0 : al[(N * N + r + c * N) * 32];
            }
        double dd[N], ee[N];
#pragma unroll
        for (int kq = 0; kq + 1 < N; ++kq) {
            double x2[N];
#pragma unroll
            for (int i = 0; i < N; ++i) x2[i] = i >= kq + 2 ? fma(xr[i][kq], xr[i][kq], xi[i][kq] * xi[i][kq]) : 0.0;
            const double xn2 = ((x2[0] + x2[1]) + (x2[2] + x2[3])) + ((x2[4] + x2[5]) + (x2[6] + x2[7]));
            const double a0r = xr[kq + 1][kq], a0i = xi[kq + 1][kq];
            dd[kq] = xr[kq][kq];
            double taur = 0.0, taui = 0.0, beta = a0r, scr = 0.0, sci = 0.0;
            const bool triv = xn2 == 0.0 && a0i == 0.0;
            if (!triv) {
                const double qq = fma(a0r, a0r, fma(a0i, a0i, xn2));
                const bool nq = qq >= 1e-290 && qq <= 1e290;  // fast reciprocals in range
                const double rq = nq ? lane_rsqrt(qq) : 1.0 / sqrt(qq);
                const double nrm = qq * rq;
                beta = a0r >= 0.0 ? -nrm : nrm;
                const double ib = a0r >= 0.0 ? -rq : rq;  // 1 / beta
                taur = (beta - a0r) * ib;
                taui = -a0i * ib;
                const double dr = a0r - beta, di = a0i;
                const double dq = fma(dr, dr, di * di);
                const double idn = nq ? lane_rcp(dq) : 1.0 / dq;
                scr = dr * idn;
                sci = -di * idn;  // 1 / (alpha - beta)
            }
            ee[kq] = beta;
            double vr[N], vi[N];
            vr[kq + 1] = 1.0;
            vi[kq + 1] = 0.0;
#pragma unroll
            for (int i = kq + 2; i < N; ++i) {
                vr[i] = fma(xr[i][kq], scr, -xi[i][kq] * sci);
                vi[i] = fma(xr[i][kq], sci, xi[i][kq] * scr);
            }
            // p = tau A22 v (two accumulators per row), w = p - 1/2 tau (p^H v) v
            double pr[N], pim[N];
#pragma unroll
            for (int i = kq + 1; i < N; ++i) {
                double s0r = 0.0, s0i = 0.0, s1r = 0.0, s1i = 0.0;
#pragma unroll
                for (int j = kq + 1; j < N; ++j) {
                    const double ar_ = i >= j ? xr[i][j] : xr[j][i];
                    const double ai_ = i == j ? 0.0 : (i > j ? xi[i][j] : -xi[j][i]);
                    if (j & 1) {
                        s0r = fma(ar_, vr[j], fma(-ai_, vi[j], s0r));
                        s0i = fma(ar_, vi[j], fma(ai_, vr[j], s0i));
                    } else {
                        s1r = fma(ar_, vr[j], fma(-ai_, vi[j], s1r));
                        s1i = fma(ar_, vi[j], fma(ai_, vr[j], s1i));
                    }
                }
                const double sr = s0r + s1r, si = s0i + s1i;
                pr[i] = fma(taur, sr, -taui * si);
                pim[i] = fma(taur, si, taui * sr);
            }
            double hr = 0.0, hi = 0.0, hr2 = 0.0, hi2 = 0.0;  // p^H v
#pragma unroll
            for (int i = kq + 1; i < N; ++i) {
                if ((i - kq) & 1) {
                    hr = fma(pr[i], vr[i], fma(pim[i], vi[i], hr));
                    hi = fma(pr[i], vi[i], fma(-pim[i], vr[i], hi));
                } else {
                    hr2 = fma(pr[i], vr[i], fma(pim[i], vi[i], hr2));
                    hi2 = fma(pr[i], vi[i], fma(-pim[i], vr[i], hi2));
                }
            }
            hr += hr2;
            hi += hi2;
            const double alr = -0.5 * fma(taur, hr, -taui * hi), ali = -0.5 * fma(taur, hi, taui * hr);
            double wr[N], wi[N];
#pragma unroll
            for (int i = kq + 1; i < N; ++i) {
                wr[i] = fma(alr, vr[i], fma(-ali, vi[i], pr[i]));
                wi[i] = fma(alr, vi[i], fma(ali, vr[i], pim[i]));
            }
            if (!triv) {  // A22 -= v w^H + w v^H (lower); tau = 0 leaves A22 unchanged
#pragma unroll
                for (int j = kq + 1; j < N; ++j)
#pragma unroll
                    for (int i = j; i < N; ++i) {
                        xr[i][j] -= fma(vr[i], wr[j], fma(vi[i], wi[j], fma(wr[i], vr[j], wi[i] * vi[j])));
                        if (i != j) xi[i][j] -= fma(vi[i], wr[j], fma(-vr[i], wi[j], fma(wi[i], vr[j], -wr[i] * vi[j])));
                    }
            }
        }
        dd[N - 1] = xr[N - 1][N - 1];
        if (lane < kPer) {
            double* dl = lane_sm + pp;
#pragma unroll
            for (int i = 0; i < N; ++i) {
                dl[(SM::kD + i) * 32] = dd[i];
                if (i + 1 < N) dl[(SM::kE + i) * 32] = ee[i];
            }
        }
    }
    __syncthreads();
    LPROF(6);
    // ---- eigenvalues: power-of-two scaling, Gershgorin bracket, Sturm bisection ------------------
    double d[N], e2[N];
    double mx = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        d[i] = SLOT(SM::kD + i);
        e2[i] = i + 1 < N ? SLOT(SM::kE + i) : 0.0;  // beta for now
        mx = fmax(mx, fmax(fabs(d[i]), fabs(e2[i])));
    }
    int ex = mx > 0.0 ? static_cast<int>((__double_as_longlong(mx) >> 52) & 0x7ff) - 1022 : 0;
    ex = max(-1000, min(1000, ex));
    const double sc = __longlong_as_double(static_cast<long long>(1023 - ex) << 52);
    const double unscale = __longlong_as_double(static_cast<long long>(1023 + ex) << 52);
    double lo = 1e300, hi = -1e300;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        d[i] *= sc;
        e2[i] *= sc;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const double r = (i > 0 ? fabs(e2[i - 1]) : 0.0) + (i + 1 < N ? fabs(e2[i]) : 0.0);
        lo = fmin(lo, d[i] - r);
        hi = fmax(hi, d[i] + r);
    }
#pragma unroll
    for (int i = 0; i < N; ++i) e2[i] *= e2[i];
    const double wid = fmax(hi - lo, fmax(fabs(lo), fabs(hi))) * 4.4e-16 * N + 1e-300;
    lo -= wid;
    hi += wid;
    const double atol = 2.2e-16 * fmax(fabs(lo), fabs(hi));
    // eigenvalues q and q + 4 of this pencil (0-based, ascending): count(a) <= i < count(b);
    // LQ interior points per eigenvalue and round (the bracket shrinks LQ + 1-fold)
#ifndef LT_LANE_Q
#define LT_LANE_Q 1  // measured best (2 and 3 points per round issue more than they save)
#endif
    constexpr int LQ = LT_LANE_Q;
    // a fixed round count: the bracket starts at most 2 max(|lo|, |hi|) wide and shrinks
    // (LQ + 1)-fold per round, so ceil(log_{LQ+1}(2 / 2.2e-16)) rounds reach the absolute
    // tolerance atol (k_pencil's stopping rule never needs more); no per-round vote
    constexpr int kRounds = LQ == 1 ? 53 : (LQ == 2 ? 34 : (LQ == 3 ? 27 : 23));
    double a[kLaneCols], b[kLaneCols];
#pragma unroll
    for (int h = 0; h < kLaneCols; ++h) {
        a[h] = lo;
        b[h] = hi;
    }
    for (int it = 0; it < kRounds; ++it) {
        double x[kLaneCols][LQ], cv[kLaneCols][LQ], pv[kLaneCols][LQ];
        int cn[kLaneCols][LQ];
#pragma unroll
        for (int h = 0; h < kLaneCols; ++h)
#pragma unroll
            for (int u = 0; u < LQ; ++u) {
                x[h][u] = fma(b[h] - a[h], static_cast<double>(u + 1) / static_cast<double>(LQ + 1), a[h]);
                pv[h][u] = 1.0;
                cv[h][u] = d[0] - x[h][u];
                cn[h][u] = static_cast<int>(static_cast<unsigned>(__double2hiint(cv[h][u])) >> 31);
            }
#pragma unroll
        for (int i = 1; i < N; ++i) {
#pragma unroll
            for (int h = 0; h < kLaneCols; ++h)
#pragma unroll
                for (int u = 0; u < LQ; ++u) {
                    const double nx = fma(d[i] - x[h][u], cv[h][u], -e2[i - 1] * pv[h][u]);
                    cn[h][u] += static_cast<int>(static_cast<unsigned>(__double2hiint(nx) ^ __double2hiint(cv[h][u])) >> 31);
                    pv[h][u] = cv[h][u];
                    cv[h][u] = nx;
                }
            if (i == 4) {
                // |p_i| <= 4.3^i cannot overflow; a chain shrinking below 2^-500 is lifted by the
                // exact power 2^500 (ratios and signs unchanged) so it cannot underflow
#pragma unroll
                for (int h = 0; h < kLaneCols; ++h)
#pragma unroll
                    for (int u = 0; u < LQ; ++u)
                        if (fabs(cv[h][u]) < 0x1p-500 && fabs(pv[h][u]) < 0x1p-500) {
                            cv[h][u] *= 0x1p500;
                            pv[h][u] *= 0x1p500;
                        }
            }
        }
#pragma unroll
        for (int h = 0; h < kLaneCols; ++h) {
            const int mi = q + kLaneWarps * h;
            // the first point whose count exceeds mi bounds the bracket from above
            double na = a[h], nb = b[h];
#pragma unroll
            for (int u = LQ - 1; u >= 0; --u)
                if (cn[h][u] > mi) nb = x[h][u];
#pragma unroll
            for (int u = 0; u < LQ; ++u)
                if (cn[h][u] <= mi) na = x[h][u];
            a[h] = na;
            b[h] = nb;
        }
    }
    // failure code: S (every warp), Cholesky pivots (every warp), H from the per-warp partials
    {
        double hm = 0.0, hd = 0.0;
#pragma unroll
        for (int w = 0; w < kLaneWarps; ++w) {
            hm = fmax(hm, SLOT(SM::kHc + 2 * w));
            hd = fmax(hd, SLOT(SM::kHc + 2 * w + 1));
        }
        double sm2 = 0.0, sd = 0.0;
#pragma unroll
        for (int w = 0; w < kLaneWarps; ++w) {
            sm2 = fmax(sm2, SLOT(SM::kSc + 2 * w));
            sd = fmax(sd, SLOT(SM::kSc + 2 * w + 1));
        }
        if (hd > 1e-20 * fmax(1.0, hm) || sd > 1e-20 * fmax(1.0, sm2)) code = 1;
    }
    LPROF(7);
    if (valid) {
        if (code == 0) {
#pragma unroll
            for (int h = 0; h < kLaneCols; ++h) eig[k * N + q + kLaneWarps * h] = 0.5 * (a[h] + b[h]) * unscale;
        } else if (q == 0) {
            atomicMin(fail_key, static_cast<unsigned long long>(k) * 4ull + static_cast<unsigned long long>(code));
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) group_done(rb, ngroups);
#undef SLOT
#undef YR
#undef YI
}

bool pencil_lane_supported(Index m0) { return m0 == 8; }

size_t pencil_lane_smem() { return sizeof(double) * 32 * LaneSmem<8>::kSlots; }

void launch_pencil_lane(const Launch& L, Index count, Index m0, const double2* H, const double2* S, Index ks, Index es,
                        double* eig, unsigned long long* fail_key, const PencilReadback& rb) {
    if (count <= 0) return;
    if (m0 != 8) fail(LT_EDIM, "pencil_lane: block size must be 8");
    constexpr int N = 8;
    const size_t smem = pencil_lane_smem();
    static bool attr = false;
    if (!attr) {
        LT_CU(cudaFuncSetAttribute(k_pencil_lane<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        attr = true;
    }
    const Index blocks = (count + 31) / 32;
    Stage st_(L, "pencil");
    k_pencil_lane<N><<<static_cast<unsigned>(blocks), 32 * kLaneWarps, smem, L.st>>>(count, H, S, ks, es, eig, fail_key,
                                                                                     rb, blocks);
    LT_CU(cudaGetLastError());
    L.tick();
}

}  // namespace lt
