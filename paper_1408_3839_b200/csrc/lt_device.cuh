// lt_device.cuh — device helpers shared by the kernels.
//
// Expressions that decide integers or trimming in the reference (grid coordinates,
// Gaussian arguments, erf arguments) are written with explicit round-to-nearest
// intrinsics so nvcc cannot contract them into FMAs: the host reference compiles
// without FMA contraction, and these values must round identically.
#pragma once

#include <cuda_runtime.h>

#include "lt_internal.cuh"

namespace lt {

// gto_basis.cpp:9-14: (x-c)^deg * exp(-alpha (x-c)^2), evaluated left to right
__device__ __forceinline__ double gto_eval1d(const DevSys& s, Index mu, int l, double x) {
    const double d = __dsub_rn(x, s.center[3 * mu + l]);
    double mono = 1.0;
    const int dg = s.deg[3 * mu + l];
    for (int p = 0; p < dg; ++p) mono = __dmul_rn(mono, d);
    const double arg = __dmul_rn(__dmul_rn(-s.alpha[mu], d), d);
    // exp(arg) rounds to exactly 0 below -745.14; skipping it for arg < -746 is exact and
    // avoids the slow underflow path of the FP64 exp on the (many) far-tail samples
    return __dmul_rn(mono, arg < -746.0 ? 0.0 : exp(arg));
}

// sinc_quadrature.cpp:9-29: node t_q of the 2M+1-point rule (k_sinc's arithmetic)
__device__ __forceinline__ double sinc_node(int q, int M) {
    double step = log(static_cast<double>(M)) / static_cast<double>(M);
    if (M == 1) step = 0.5;
    const double u = __dmul_rn(static_cast<double>(q - M), step);
    const double eu = exp(-u);
    return exp(__dsub_rn(u, eu));
}

// newton_kernel.cpp:22-45: master cell j of column t_q on the centred grid of mrows cells,
// sqrt(pi)/(2 t_q) (erf(t_q x_{j+1}) - erf(t_q x_j)), x_j = -mrows h / 2 + j h
__device__ __forceinline__ double master_cell(Index j, Index mrows, double h, double tq) {
    const double origin = __dmul_rn(__dmul_rn(-0.5, static_cast<double>(mrows)), h);
    const double xl = __dadd_rn(origin, __dmul_rn(static_cast<double>(j), h));
    const double xr = __dadd_rn(origin, __dmul_rn(static_cast<double>(j + 1), h));
    const double c = __ddiv_rn(sqrt(3.141592653589793), __dmul_rn(2.0, tq));
    const double el = erf(__dmul_rn(tq, xl));
    const double er = erf(__dmul_rn(tq, xr));
    return __dmul_rn(c, __dsub_rn(er, el));
}

// the two halves of master_cell: erf(t_q x_j) and the cell from its two edge values (the
// same arithmetic, so cells assembled from shared edge values are bitwise master_cell's)
__device__ __forceinline__ double master_edge(Index j, Index mrows, double h, double tq) {
    const double origin = __dmul_rn(__dmul_rn(-0.5, static_cast<double>(mrows)), h);
    return erf(__dmul_rn(tq, __dadd_rn(origin, __dmul_rn(static_cast<double>(j), h))));
}
__device__ __forceinline__ double master_from_edges(double el, double er, double tq) {
    const double c = __ddiv_rn(sqrt(3.141592653589793), __dmul_rn(2.0, tq));
    return __dmul_rn(c, __dsub_rn(er, el));
}

__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_max(double v) {
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Sturm counts by the three-term (continuant) recurrence p_i = (d_i - x) p_{i-1} - e_{i-1}^2
// p_{i-2} (Wilkinson's bisection form): the count of eigenvalues below x is the number of
// negative ratios q_i = p_i / p_{i-1}, the LDL^T pivots, without a division on the
// dependent chain (one FMA per step instead of a reciprocal). T is pre-scaled by a power of
// two to max |entry| < 1; a ratio with |q_i| < 2^-100 is replaced by -2^-100 (the pivmin rule
// of the ratio form, a perturbation of d_i far below eps ||T||), and (p_i, p_{i-1}) are
// rescaled by an exact power of two every 4 steps, which keeps them normal (|q| <= 4).
// GUARD 1: integer-pipe guard (below); 0: the same rule on the FP64 pipe; 2: no per-step
// guard (the batched pencils and the dense tridiagonal): with T scaled to max |entry| < 1
// and x inside the Gershgorin bracket, |p_i| grows at most 4.3-fold per step and cannot
// overflow between the every-4-steps power-of-two rescales, which also keep the chain
// normal; an exact p_i = 0 counts as non-negative (the next term -e^2 p_{i-2} restores the
// sign-change count). Measured: the guard's compare/select on the dependent chain set the
// round time of the long dense chains (n = 1024: 415 -> 249 us without it).
template <int Q, int GUARD = 1>
__device__ __forceinline__ void sturm3(const double* sd, const double* se2, int n, const double (&x)[Q],
                                       int (&cnt)[Q]) {
    constexpr bool INTGUARD = GUARD == 1;
    if constexpr (GUARD == 2) {
        // short chains: plain registers, no lambda (keeps x / cnt out of local memory)
        double xv[Q], pv[Q], cv[Q];
        int cn[Q];
#pragma unroll
        for (int j = 0; j < Q; ++j) {
            xv[j] = x[j];
            pv[j] = 1.0;
            cv[j] = sd[0] - xv[j];
            cn[j] = static_cast<int>(static_cast<unsigned>(__double2hiint(cv[j])) >> 31);
        }
        for (int i = 1; i < n; ++i) {
            const double di = sd[i], ei = se2[i - 1];
#pragma unroll
            for (int j = 0; j < Q; ++j) {
                const double nx = fma(di - xv[j], cv[j], -ei * pv[j]);
                cn[j] += static_cast<int>(static_cast<unsigned>(__double2hiint(nx) ^ __double2hiint(cv[j])) >> 31);
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
#pragma unroll
        for (int j = 0; j < Q; ++j) cnt[j] = cn[j];
        return;
    }
    constexpr double kDelta = 7.888609052210118e-31;  // 2^-100
    double prev[Q], cur[Q];
#pragma unroll
    for (int j = 0; j < Q; ++j) {
        prev[j] = 1.0;
        cur[j] = sd[0] - x[j];
        if (GUARD != 2 && fabs(cur[j]) < kDelta) cur[j] = -kDelta;
        cnt[j] = static_cast<int>(static_cast<unsigned>(__double2hiint(cur[j])) >> 31);
    }
    // INTGUARD: the guard and the sign count run on the integer pipe (the FP64 pipe then
    // carries only the DADD, DMUL and DFMA of the recurrence; measured faster for the batched
    // pencils, slower for the long dense chains, which keep the FP64 form): |nx| below
    // 2^-100 |cur| is detected from the exponent fields and nx replaced by the power of two
    // 2^(e(cur) - 100) (within a factor 2 of 2^-100 |cur|) of the sign opposite to cur.
    // The rescaling keeps e(cur) in [623, 1423], so the replacement stays normal.
    auto step = [&](double di, double ei) {
#pragma unroll
        for (int j = 0; j < Q; ++j) {
            double nx = fma(di - x[j], cur[j], -ei * prev[j]);
            if constexpr (GUARD == 2) {
                cnt[j] += static_cast<int>(static_cast<unsigned>(__double2hiint(nx) ^ __double2hiint(cur[j])) >> 31);
                prev[j] = cur[j];
                cur[j] = nx;
                continue;
            }
            if constexpr (!INTGUARD) {  // the same rule on the FP64 pipe (exact 2^-100 |cur|)
                const double thr = kDelta * fabs(cur[j]);
                if (fabs(nx) < thr) nx = cur[j] < 0.0 ? thr : -thr;
                cnt[j] += (nx < 0.0) != (cur[j] < 0.0);
                prev[j] = cur[j];
                cur[j] = nx;
                continue;
            }
            const int hn = __double2hiint(nx), hc = __double2hiint(cur[j]);
            const int ec = (hc >> 20) & 0x7ff;
            if (((hn >> 20) & 0x7ff) < ec - 100)
                nx = __hiloint2double(static_cast<int>((~hc & 0x80000000u) | static_cast<unsigned>((ec - 100) << 20)), 0);
            cnt[j] += static_cast<int>(static_cast<unsigned>(__double2hiint(nx) ^ hc) >> 31);
            prev[j] = cur[j];
            cur[j] = nx;
        }
    };
    int i = 1;
    // blocks of 4 steps: the 8 shared-memory loads are issued ahead of the dependent chain
    for (; i + 3 < n; i += 4) {
        const double d0 = sd[i], d1 = sd[i + 1], d2 = sd[i + 2], d3 = sd[i + 3];
        const double e0 = se2[i - 1], e1 = se2[i], e2 = se2[i + 1], e3 = se2[i + 2];
        step(d0, e0);
        step(d1, e1);
        step(d2, e2);
        step(d3, e3);
#pragma unroll
        for (int j = 0; j < Q; ++j) {
            const int ex = ((__double2hiint(cur[j]) >> 20) & 0x7ff) - 1023;
            if (ex > 400 || ex < -400) {  // rare: exact power-of-two rescale of (cur, prev)
                const double sc = __longlong_as_double(static_cast<long long>(1023 - ex) << 52);
                cur[j] *= sc;
                prev[j] *= sc;
            }
        }
    }
    for (; i < n; ++i) step(sd[i], se2[i - 1]);
}

// pencil kernels: called once per finished group (a group of threads per pencil, or a
// warp of one-thread pencils) by its leader on every exit path; the last of `count` groups
// copies the 8-int result block (L0 state, failure key) to pinned host memory
__device__ __forceinline__ void group_done(const PencilReadback& rb, Index count) {
    if (rb.done == nullptr) return;
    __threadfence();  // this group's failure key update before its arrival
    if (atomicAdd(rb.done, 1u) == static_cast<unsigned>(count - 1)) {
        __threadfence();
        const volatile int* src = rb.ret_dev;
        for (int i = 0; i < 8; ++i) rb.ret_host[i] = src[i];
        *rb.done = 0u;  // ready for the next launch or graph replay
    }
}

}  // namespace lt
