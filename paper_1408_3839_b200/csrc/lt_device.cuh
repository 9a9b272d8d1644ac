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

__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_max(double v) {
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

}  // namespace lt
