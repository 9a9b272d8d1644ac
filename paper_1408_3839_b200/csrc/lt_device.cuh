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

__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_max(double v) {
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

}  // namespace lt
