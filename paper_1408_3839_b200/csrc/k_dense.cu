// k_dense.cu — dense box pencil beyond the library eigensolver (eigensolver.cpp:12-35,
// eigenvalues): after the Cholesky reduction A = L^-1 H L^-T (symmetrised as the reference
// does, 0.5 (A + A^T)), A is reduced to tridiagonal form by one persistent kernel and the
// eigenvalues of the tridiagonal come from parallel Sturm multisection.
//
//   k_sytrd        Householder tridiagonalisation (dsytd2, lower) in ONE cooperative launch:
//                  columns are distributed cyclically over the CTAs and stay in shared
//                  memory for the whole reduction. Step k needs one grid-wide exchange: every
//                  CTA publishes p_j = (A v)_j for its own columns (plus, by the owner,
//                  column k+1), then every CTA rebuilds w = tau p - tau^2/2 (v.p) v, applies
//                  the rank-2 update to its own columns, and recomputes the next reflector
//                  from column k+1 redundantly — no second barrier for the reflector.
//   k_sytrd_reg    the same with the own columns in registers (n <= 1024): the fused
//                  update + next-dot pass reads no matrix data from shared memory.
//   k_tridiag_eig3 eigenvalues of the tridiagonal (d, e): G lanes x Q shifts per eigenvalue of
//                  three-term Sturm counts (no division on the chain), the bracket shrinks
//                  G Q + 1-fold per round; ascending by construction.
#include "lt_device.cuh"
#include "lt_internal.cuh"

#include <cstdio>
#include <cstdlib>

namespace lt {

namespace {

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// grid-wide barrier over a monotone counter: CTA arrives once per step
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        while (ld_acquire(bar) < target) {
        }
        __threadfence();
    }
    __syncthreads();
}

__device__ __forceinline__ double fast_rcp(double q) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    double t = fma(-q, r, 1.0);
    r = fma(r, t, r);
    t = fma(-q, r, 1.0);
    return fma(r, t, r);
}

// dlarfg coefficients from alpha = a0 and sigma = |x|^2 (sigma != 0): beta, tau and
// 1 / (a0 - beta), on the step's dependent chain: MUFU reciprocal square root / reciprocal
// with one cubic correction each (within an ulp or two) in the normal range, IEEE otherwise
__device__ __forceinline__ void house_coeffs(double a0, double sigma, double& beta, double& tau, double& scal) {
    const double q = fma(a0, a0, sigma);
    if (q >= 1e-290 && q <= 1e290) {
        double y;
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(q));
        const double ey = fma(-q * y, y, 1.0);
        y = fma(y * ey, fma(ey, 0.375, 0.5), y);  // 1 / nrm
        const double nrm = q * y;
        beta = a0 >= 0.0 ? -nrm : nrm;
        tau = (beta - a0) * (a0 >= 0.0 ? -y : y);  // (beta - a0) / beta
        const double dn = a0 - beta;                // |a0| + nrm: no cancellation
        double r;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(dn));
        const double er = fma(-dn, r, 1.0);
        scal = fma(r, fma(er, er, er), r);
    } else {
        const double nrm = sqrt(q);
        beta = a0 >= 0.0 ? -nrm : nrm;
        tau = (beta - a0) / beta;
        scal = 1.0 / (a0 - beta);
    }
}

}  // namespace

// smem: A[cols][n] (own columns j = b + s P), v[2][n] (ping-pong reflectors), w[n], c[n],
// pown[cols] (p of own columns for the next exchange)
//
// Step k (trailing rows / columns r0 = k+1 .. n-1), every CTA holding v = v_k, tau_k and
// p_j = (A^(k) v)_j of its own columns j >= r0:
//   exchange   publish p_j (and, by the owner, column r0 of A^(k)); grid barrier
//   w, c       load p, column r0; w = tau p - tau^2/2 (v.p) v; column r0 of A^(k+1):
//              c = col - v w_r0 - w (v_r0 = 1); d_r0 = c_r0
//   reflector  of c[r0+1 ..] (dlarfg): v', tau', e_r0 = beta
//   fused pass own columns j > r0: A -= v w^T + w v^T and p'_j = A^(k+1)[.][j] . v' in one
//              sweep (warp per column); the owner of column r0+1 publishes it
template <int NT>
__global__ void __launch_bounds__(NT) k_sytrd(int n, int P, int cols, const double* __restrict__ C, double* d,
                                              double* e, double* pbuf, double* cbuf, unsigned* bar, long long* prof) {
    // optional phase clocks of CTA 0 (LT_SYTRD_PROFILE): fused pass, barrier, loads + v.p,
    // w/c + sigma, reflector
    long long tacc[6] = {0, 0, 0, 0, 0, 0};
    long long tl = clock64();
    const bool pr = prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
#define SYPROF(i)                       \
    if (pr) {                           \
        const long long tn = clock64(); \
        tacc[i] += tn - tl;             \
        tl = tn;                        \
    }
    extern __shared__ __align__(16) double sm[];
    double* A = sm;
    double* sv = A + static_cast<size_t>(cols) * n;
    double* svn = sv + n;
    double* sw = svn + n;
    double* sc = sw + n;
    double* pown = sc + n;
    __shared__ double red[2][NT / 32];
    const int b = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ncol = (n - b + P - 1) / P;  // own columns: j = b + s P, s < ncol
    auto first_own = [&](int r) { return r > b ? (r - b + P - 1) / P : 0; };  // first s with b + s P >= r
    auto bsum = [&](double v, int slot) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[slot][warp] = v;
        __syncthreads();
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) s += red[slot][w];
        return s;
    };
    for (int s = 0; s < ncol; ++s) {
        const double* src = C + static_cast<size_t>(b + s * P) * n;
        for (int i = threadIdx.x; i < n; i += NT) A[static_cast<size_t>(s) * n + i] = src[i];
    }
    // column 0 from the input, redundantly: d_0 and the first reflector
    double tau = 0.0;
    if (b == 0 && threadIdx.x == 0) d[0] = C[0];
    if (n > 1) {
        double sg = 0.0;
        for (int i = 2 + threadIdx.x; i < n; i += NT) sg += C[i] * C[i];
        const double sigma = bsum(sg, 0);
        const double a0 = C[1];
        double beta = a0, scal = 0.0;
        if (sigma != 0.0) {
            const double nrm = sqrt(a0 * a0 + sigma);
            beta = a0 >= 0.0 ? -nrm : nrm;
            tau = (beta - a0) / beta;
            scal = 1.0 / (a0 - beta);
        }
        for (int i = 1 + threadIdx.x; i < n; i += NT) sv[i] = (i == 1) ? 1.0 : C[i] * scal;
        if (b == 0 && threadIdx.x == 0) e[0] = beta;
    }
    __syncthreads();
    // p of own columns j >= 1 with v_0
    for (int s = first_own(1) + warp; s < ncol; s += NT / 32) {
        const double* col = A + static_cast<size_t>(s) * n;
        double a0 = 0.0, a1 = 0.0;
        if (tau != 0.0)
            for (int i = 1 + lane; i < n; i += 64) {
                a0 = fma(col[i], sv[i], a0);
                if (i + 32 < n) a1 = fma(col[i + 32], sv[i + 32], a1);
            }
        a0 += a1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a0 += __shfl_xor_sync(0xffffffffu, a0, o);
        if (lane == 0) pbuf[b + s * P] = a0;
    }
    if (n > 1 && 1 % P == b) {
        const double* col = A + static_cast<size_t>(1 / P) * n;
        for (int i = 1 + threadIdx.x; i < n; i += NT) cbuf[i] = col[i];
    }
    for (int k = 0; k + 1 < n; ++k) {
        const int r0 = k + 1;
        const double* pb = pbuf + static_cast<size_t>(k & 1) * n;
        const double* cb = cbuf + static_cast<size_t>(k & 1) * n;
        double* pbn = pbuf + static_cast<size_t>((k + 1) & 1) * n;
        double* cbn = cbuf + static_cast<size_t>((k + 1) & 1) * n;
        SYPROF(0);
        // grid barrier: every CTA's p (and column r0) published
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
            const unsigned target = static_cast<unsigned>(k + 1) * static_cast<unsigned>(P);
            while (ld_acquire(bar) < target) {
            }
        }
        __syncthreads();
        SYPROF(1);
        // loads and v.p
        double part = 0.0;
        for (int i = r0 + threadIdx.x; i < n; i += NT) {
            const double p = __ldcg(pb + i);
            sw[i] = p;
            sc[i] = __ldcg(cb + i);
            part = fma(sv[i], p, part);
        }
        const double p0 = __ldcg(pb + r0);
        const double vp = bsum(part, k & 1);
        SYPROF(2);
        const double half = 0.5 * tau * tau * vp;
        const double w0 = tau * p0 - half;  // v_r0 = 1
        double sg = 0.0;
        for (int i = r0 + threadIdx.x; i < n; i += NT) {
            const double w = tau * sw[i] - half * sv[i];
            sw[i] = w;
            const double c = sc[i] - fma(sv[i], w0, w);
            sc[i] = c;
            if (i >= r0 + 2) sg = fma(c, c, sg);
        }
        if (b == 0 && threadIdx.x == 0) d[r0] = sc[r0];  // row r0 is thread 0's
        const double sigma = bsum(sg, (k + 1) & 1);
        SYPROF(3);
        double taun = 0.0;
        if (r0 + 1 < n) {
            const double a0 = sc[r0 + 1];
            double beta = a0, scal = 0.0;
            if (sigma != 0.0) house_coeffs(a0, sigma, beta, taun, scal);
            for (int i = r0 + 1 + threadIdx.x; i < n; i += NT) svn[i] = (i == r0 + 1) ? 1.0 : sc[i] * scal;
            if (b == 0 && threadIdx.x == 0) e[r0] = beta;
        }
        __syncthreads();
        SYPROF(4);
        // fused pass over own columns j > r0
        for (int s = first_own(r0 + 1) + warp; s < ncol; s += NT / 32) {
            const int j = b + s * P;
            const double wj = sw[j], vj = sv[j];
            double* col = A + static_cast<size_t>(s) * n;
            double a0 = 0.0, a1 = 0.0;
            for (int i = r0 + lane; i < n; i += 64) {
                const double x = col[i] - fma(sv[i], wj, sw[i] * vj);
                col[i] = x;
                if (i > r0) a0 = fma(x, svn[i], a0);
                const int i2 = i + 32;
                if (i2 < n) {
                    const double x2 = col[i2] - fma(sv[i2], wj, sw[i2] * vj);
                    col[i2] = x2;
                    a1 = fma(x2, svn[i2], a1);
                }
            }
            a0 += a1;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) a0 += __shfl_xor_sync(0xffffffffu, a0, o);
            if (lane == 0) pbn[j] = taun != 0.0 ? a0 : 0.0;
            if (j == r0 + 1) {  // the next step's column, published by its owner
                __syncwarp();
                for (int i = r0 + 1 + lane; i < n; i += 32) cbn[i] = col[i];
            }
        }
        double* t = sv;
        sv = svn;
        svn = t;
        tau = taun;
        SYPROF(5);
    }
    if (pr)
        for (int i = 0; i < 6; ++i) prof[i] = tacc[i];
#undef SYPROF
}

// ---- register-resident variant: own columns in registers (thread t holds rows t + NT u),
// the same one-barrier exchange as k_sytrd.
// smem: v[2][n], w[n], c[n]; exchange: pbuf[2][n], cbuf[2][n]
template <int NT, int R, int CM>
__global__ void __launch_bounds__(NT) k_sytrd_reg(int n, int P, const double* __restrict__ C, double* d, double* e,
                                                  double* pbuf, double* cbuf, unsigned* bar, long long* prof) {
    long long tacc[6] = {0, 0, 0, 0, 0, 0};
    long long tl = clock64();
    const bool pr = prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
#define SYPROF(i)                       \
    if (pr) {                           \
        const long long tn = clock64(); \
        tacc[i] += tn - tl;             \
        tl = tn;                        \
    }
    extern __shared__ __align__(16) double sm[];
    double* sv = sm;
    double* svn = sv + n;
    double* sw = svn + n;
    double* sc = sw + n;
    __shared__ double red[2][NT / 32];
    __shared__ double cred[NT / 32][CM];
    const int b = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    auto bsum = [&](double v, int slot) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[slot][warp] = v;
        __syncthreads();
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) s += red[slot][w];
        return s;
    };
    // own columns j = b + s P into registers
    double a[R][CM];
#pragma unroll
    for (int s = 0; s < CM; ++s) {
        const int j = b + s * P;
#pragma unroll
        for (int u = 0; u < R; ++u) {
            const int i = threadIdx.x + NT * u;
            a[u][s] = (j < n && i < n) ? C[static_cast<size_t>(j) * n + i] : 0.0;
        }
    }
    // column 0 redundantly: d_0, the first reflector
    double tau = 0.0;
    if (b == 0 && threadIdx.x == 0) d[0] = C[0];
    if (n > 1) {
        double sg = 0.0;
        for (int i = 2 + threadIdx.x; i < n; i += NT) sg += C[i] * C[i];
        const double sigma = bsum(sg, 0);
        const double a0 = C[1];
        double beta = a0, scal = 0.0;
        if (sigma != 0.0) {
            const double nrm = sqrt(a0 * a0 + sigma);
            beta = a0 >= 0.0 ? -nrm : nrm;
            tau = (beta - a0) / beta;
            scal = 1.0 / (a0 - beta);
        }
        for (int i = 1 + threadIdx.x; i < n; i += NT) sv[i] = (i == 1) ? 1.0 : C[i] * scal;
        if (b == 0 && threadIdx.x == 0) e[0] = beta;
    }
    __syncthreads();
    // reduce the per-thread column partials and publish p (and the next column)
    auto publish = [&](const double (&part)[CM], int rfirst, double taun, int rnext, double* pdst, double* cdst) {
        // column rnext (rows >= rnext) by its owner, straight from the registers
        if (rnext < n && rnext % P == b) {
            const int sn = rnext / P;
#pragma unroll
            for (int s = 0; s < CM; ++s)
                if (s == sn)
#pragma unroll
                    for (int u = 0; u < R; ++u) {
                        const int i = threadIdx.x + NT * u;
                        if (i >= rnext && i < n) cdst[i] = a[u][s];
                    }
        }
        // warp transpose-reduction: CM - 1 exchanges leave lane l with column l % CM summed over
        // its CM-lane group, the remaining offsets add the groups (instead of 5 CM shuffles)
        double pt[CM];
#pragma unroll
        for (int s = 0; s < CM; ++s) pt[s] = part[s];
#pragma unroll
        for (int off = CM / 2; off >= 1; off >>= 1) {
            const bool up = (lane & off) != 0;
#pragma unroll
            for (int i = 0; i < off; ++i) {
                const double send = up ? pt[i] : pt[i + off];
                const double keep = up ? pt[i + off] : pt[i];
                pt[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
            }
        }
#pragma unroll
        for (int o = CM; o < 32; o <<= 1) pt[0] += __shfl_xor_sync(0xffffffffu, pt[0], o);
        if (lane < CM) cred[warp][lane] = pt[0];
        __syncthreads();
        if (static_cast<int>(threadIdx.x) < CM) {
            const int s = threadIdx.x;
            const int j = b + s * P;
            if (j >= rfirst && j < n) {
                double t = 0.0;
#pragma unroll
                for (int w = 0; w < NT / 32; ++w) t += cred[w][s];
                pdst[j] = taun != 0.0 ? t : 0.0;
            }
        }
    };
    {
        double part[CM];
#pragma unroll
        for (int s = 0; s < CM; ++s) {
            part[s] = 0.0;
#pragma unroll
            for (int u = 0; u < R; ++u) {
                const int i = threadIdx.x + NT * u;
                if (i >= 1 && i < n) part[s] = fma(a[u][s], sv[i], part[s]);
            }
        }
        publish(part, 1, tau, 1, pbuf, cbuf);
    }
    for (int k = 0; k + 1 < n; ++k) {
        const int r0 = k + 1;
        const double* pb = pbuf + static_cast<size_t>(k & 1) * n;
        const double* cb = cbuf + static_cast<size_t>(k & 1) * n;
        double* pbn = pbuf + static_cast<size_t>((k + 1) & 1) * n;
        double* cbn = cbuf + static_cast<size_t>((k + 1) & 1) * n;
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
            const unsigned target = static_cast<unsigned>(k + 1) * static_cast<unsigned>(P);
            while (ld_acquire(bar) < target) {
            }
        }
        __syncthreads();
        SYPROF(1);
        double part = 0.0;
        for (int i = r0 + threadIdx.x; i < n; i += NT) {
            const double p = __ldcg(pb + i);
            sw[i] = p;
            sc[i] = __ldcg(cb + i);
            part = fma(sv[i], p, part);
        }
        const double p0 = __ldcg(pb + r0);  // (sw[r0] is rewritten below by thread 0)
        const double vp = bsum(part, k & 1);
        SYPROF(2);
        const double half = 0.5 * tau * tau * vp;
        const double w0 = tau * p0 - half;
        double sg = 0.0;
        for (int i = r0 + threadIdx.x; i < n; i += NT) {
            const double w = tau * sw[i] - half * sv[i];
            sw[i] = w;
            const double c = sc[i] - fma(sv[i], w0, w);
            sc[i] = c;
            if (i >= r0 + 2) sg = fma(c, c, sg);
        }
        if (b == 0 && threadIdx.x == 0) d[r0] = sc[r0];
        const double sigma = bsum(sg, (k + 1) & 1);
        SYPROF(3);
        double taun = 0.0;
        if (r0 + 1 < n) {
            const double a0 = sc[r0 + 1];
            double beta = a0, scal = 0.0;
            if (sigma != 0.0) house_coeffs(a0, sigma, beta, taun, scal);
            for (int i = r0 + 1 + threadIdx.x; i < n; i += NT) svn[i] = (i == r0 + 1) ? 1.0 : sc[i] * scal;
            if (b == 0 && threadIdx.x == 0) e[r0] = beta;
        }
        __syncthreads();
        SYPROF(4);
        // fused pass: own columns j > r0 in registers
        double vi[R], wi[R], vni[R];
#pragma unroll
        for (int u = 0; u < R; ++u) {
            const int i = threadIdx.x + NT * u;
            const bool in = i >= r0 && i < n;
            vi[u] = in ? sv[i] : 0.0;
            wi[u] = in ? sw[i] : 0.0;
            vni[u] = (i > r0 && i < n) ? svn[i] : 0.0;
        }
        double cp[CM];
        // groups of 4 columns: a group whose columns are all reduced is skipped (uniform branch);
        // inside a group the arithmetic is branch-free (reduced columns get w_j = v_j = 0), so the
        // shared-memory loads and the FP64 chains of the columns overlap
#pragma unroll
        for (int g4 = 0; g4 < CM; g4 += 4) {
            if (b + (g4 + 3) * P > r0) {
                double wj[4], vj[4];
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    const int j = b + (g4 + s) * P;
                    const bool ok = j > r0 && j < n;
                    wj[s] = ok ? sw[j] : 0.0;
                    vj[s] = ok ? sv[j] : 0.0;
                }
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    double c0 = 0.0;
#pragma unroll
                    for (int u = 0; u < R; ++u) {
                        a[u][g4 + s] -= fma(vi[u], wj[s], wi[u] * vj[s]);  // rows < r0 carry v = w = 0
                        c0 = fma(a[u][g4 + s], vni[u], c0);
                    }
                    cp[g4 + s] = c0;
                }
            } else {
#pragma unroll
                for (int s = 0; s < 4; ++s) cp[g4 + s] = 0.0;
            }
        }
        SYPROF(0);
        publish(cp, r0 + 1, taun, r0 + 1, pbn, cbn);
        double* t = sv;
        sv = svn;
        svn = t;
        tau = taun;
        SYPROF(5);
    }
    if (pr)
        for (int i = 0; i < 6; ++i) prof[i] = tacc[i];
#undef SYPROF
}

// G lanes per eigenvalue, Q shifts per lane; T scaled by 2^-s (max |d|, |e| < 1) internally;
// GUARD: lt_device.cuh's sturm3 guard mode
template <int Q, int G, int BS, int GUARD = 0>
__global__ void __launch_bounds__(BS) k_tridiag_eig3(int n, const double* __restrict__ d, const double* __restrict__ e,
                                                     double* __restrict__ eig) {
    extern __shared__ __align__(16) double ts[];
    double* sd = ts;
    double* se2 = ts + n;
    constexpr int NW = BS / 32;
    __shared__ double red[NW][3];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double mx = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        mx = fmax(mx, fabs(d[i]));
        if (i + 1 < n) mx = fmax(mx, fabs(e[i]));
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) red[warp][0] = mx;
    __syncthreads();
    mx = red[0][0];
    for (int w = 1; w < NW; ++w) mx = fmax(mx, red[w][0]);
    __syncthreads();
    // exact power-of-two scale: max |entry| * sc in [0.5, 1)
    int ex = mx > 0.0 ? static_cast<int>((__double_as_longlong(mx) >> 52) & 0x7ff) - 1022 : 0;
    ex = max(-1000, min(1000, ex));
    const double sc = __longlong_as_double(static_cast<long long>(1023 - ex) << 52);
    double lo = 1e300, hi = -1e300;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double di = d[i] * sc;
        const double ei = i + 1 < n ? e[i] * sc : 0.0;
        sd[i] = di;
        se2[i] = ei * ei;
        const double r = (i > 0 ? fabs(e[i - 1] * sc) : 0.0) + fabs(ei);
        lo = fmin(lo, di - r);
        hi = fmax(hi, di + r);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) {
        red[warp][1] = lo;
        red[warp][2] = hi;
    }
    __syncthreads();
    lo = red[0][1];
    hi = red[0][2];
    for (int w = 1; w < NW; ++w) {
        lo = fmin(lo, red[w][1]);
        hi = fmax(hi, red[w][2]);
    }
    const double wid = fmax(hi - lo, fmax(fabs(lo), fabs(hi))) * 4.4e-16 * n + 1e-300;
    lo -= wid;
    hi += wid;
    const double atol = 2.2e-16 * fmax(fabs(lo), fabs(hi));
    const int mi = (blockIdx.x * blockDim.x + threadIdx.x) / G;
    const int sub = threadIdx.x % G;
    const bool active = mi < n;
    const int gb = lane & ~(G - 1);
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << gb);
    double a = lo, bnd = hi;
    const double inv_pts = 1.0 / static_cast<double>(G * Q + 1);
    for (int it = 0; it < 80; ++it) {
        double x[Q];
        int cnt[Q];
#pragma unroll
        for (int j = 0; j < Q; ++j) x[j] = a + (bnd - a) * (static_cast<double>(sub * Q + j + 1) * inv_pts);
        if (active) {
            sturm3<Q, GUARD>(sd, se2, n, x, cnt);
        } else {
#pragma unroll
            for (int j = 0; j < Q; ++j) cnt[j] = 0;
        }
        int fq = Q;
#pragma unroll
        for (int j = Q - 1; j >= 0; --j)
            if (cnt[j] > mi) fq = j;
        const double prev_last = __shfl_up_sync(0xffffffffu, x[Q - 1], 1);
        double clo = sub > 0 ? prev_last : a, chi = x[0];
#pragma unroll
        for (int j = 1; j < Q; ++j)
            if (fq == j) {
                clo = x[j - 1];
                chi = x[j];
            }
        const unsigned bal = __ballot_sync(0xffffffffu, active && fq < Q) & gmask;
        const int src = bal ? (__ffs(bal) - 1) : (gb + G - 1);
        const double slo = __shfl_sync(0xffffffffu, clo, src);
        const double shi = __shfl_sync(0xffffffffu, chi, src);
        const double last = __shfl_sync(0xffffffffu, x[Q - 1], gb + G - 1);
        double na, nb;
        if (bal) {
            na = slo;
            nb = shi;
        } else {
            na = last;
            nb = bnd;
        }
        const bool done = !(nb - na > 2.2e-16 * fmax(fabs(na), fabs(nb)) + atol) || (na == a && nb == bnd);
        a = na;
        bnd = nb;
        if (__all_sync(0xffffffffu, done || !active)) break;
    }
    if (active && sub == 0) eig[mi] = 0.5 * (a + bnd) / sc;
}

// A = 0.5 (A + A^T) in place: CTA per tile pair (bi >= bj), 32 x 32 tiles

#ifdef LT_SYTRD_PROF
long long* lt_sytrd_prof_ptr = nullptr;
#endif
static size_t sytrd_smem(int n, int cols) {
    return sizeof(double) * (static_cast<size_t>(cols) * n + 4 * static_cast<size_t>(n) + cols);
}

int sytrd_ctas(int n) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int P = std::min(n, sms);
    const int cols = (n + P - 1) / P;
    return sytrd_smem(n, cols) <= 227 * 1024 - 1024 ? P : 0;
}

template <int NT, int R, int CM>
static bool try_sytrd_reg(const Launch& L, int n, int P, const double* C, double* d, double* e, double* work,
                          unsigned* bar, long long* prof) {
    if (n > NT * R || (n + P - 1) / P > CM) return false;
    const size_t smem = sizeof(double) * 4 * static_cast<size_t>(n);
    LT_CU(cudaFuncSetAttribute(k_sytrd_reg<NT, R, CM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
    LT_CU(cudaMemsetAsync(bar, 0, sizeof(unsigned), L.st));
    double* pbuf = work;
    double* cbuf = work + 2 * static_cast<size_t>(n);
    int nn = n, PP = P;
    void* args[] = {&nn, &PP, &C, &d, &e, &pbuf, &cbuf, &bar, &prof};
    Stage st_(L, "sytrd");
    LT_CU(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_sytrd_reg<NT, R, CM>), dim3(P), dim3(NT), args,
                                      smem, L.st));
    L.tick();
    return true;
}

// work: 4 n doubles (p and column exchange buffers, double-buffered)
void launch_sytrd(const Launch& L, int n, const double* C, double* d, double* e, double* work, unsigned* bar) {
    constexpr int NT = 256;
    const int P = sytrd_ctas(n);
    if (P == 0) fail(LT_EGENERIC, "sytrd: matrix too large for the shared-memory resident reduction");
    long long* pp = nullptr;  // per-phase cycle counters (tools/sytrd_phases.cu only)
#ifdef LT_SYTRD_PROF
    pp = lt_sytrd_prof_ptr;
#endif
    // own columns in registers when they fit (n <= 256 R, ceil(n / P) <= CM), else in shared memory
    const bool reg = (try_sytrd_reg<256, 2, 4>(L, n, P, C, d, e, work, bar, pp) ||
                                    try_sytrd_reg<256, 4, 8>(L, n, P, C, d, e, work, bar, pp));
    if (!reg) {
        const int cols = (n + P - 1) / P;
        const size_t smem = sytrd_smem(n, cols);
        LT_CU(cudaFuncSetAttribute(k_sytrd<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        LT_CU(cudaMemsetAsync(bar, 0, sizeof(unsigned), L.st));
        double* pbuf = work;
        double* cbuf = work + 2 * static_cast<size_t>(n);
        int nn = n, PP = P, cc = cols;
        void* args[] = {&nn, &PP, &cc, &C, &d, &e, &pbuf, &cbuf, &bar, &pp};
        Stage st_(L, "sytrd");
        LT_CU(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_sytrd<NT>), dim3(P), dim3(NT), args, smem,
                                          L.st));
        L.tick();
    }
}

template <int Q, int G, int BS, int GUARD>
static void run_eig3(const Launch& L, int n, const double* d, const double* e, double* eig, size_t smem) {
    LT_CU(cudaFuncSetAttribute(k_tridiag_eig3<Q, G, BS, GUARD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
    const unsigned blocks = static_cast<unsigned>((static_cast<size_t>(n) * G + BS - 1) / BS);
    k_tridiag_eig3<Q, G, BS, GUARD><<<blocks, BS, smem, L.st>>>(n, d, e, eig);
}

void launch_tridiag_eig(const Launch& L, int n, const double* d, const double* e, double* eig) {
    const size_t smem = sizeof(double) * 2 * static_cast<size_t>(n);
    Stage st_(L, "tridiag_eig");
    // 32 lanes x 1 shift per eigenvalue (33-fold bracket shrink per round) in 64-thread CTAs,
    // the three-term counts without the per-step guard (sturm3 GUARD 2: one FMA per step on
    // the chain; the power-of-two rescale every 4 steps keeps it normal, |p_i| <= 4.3^i
    // between rescales): n = 1024 415 -> 249 us on B200 (tools/eig3_probe.cu: the guard's
    // compare/select on the chain, not the counts, set the round time; 2 shifts per lane,
    // fewer lanes and the LDL^T-ratio counts were slower)
    run_eig3<1, 32, 64, 2>(L, n, d, e, eig, smem);
    LT_CU(cudaGetLastError());
    L.tick();
}

}  // namespace lt
