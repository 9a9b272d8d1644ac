// dmma.cuh — FP64 tensor-core (DMMA) building blocks for sm_100a.
//
// FP64 has no tcgen05 kind (ptxas rejects .kind::f64), so the FP64 tensor path on
// Blackwell is warp-level mma.sync .f64, which lowers to DMMA.8x8x4 in SASS. Measured on
// this B200: 37.1 TFLOP/s DMMA vs 34.2 TFLOP/s DFMA (profiles/fp64_peak.json); fragment
// layouts verified by tools/fp64_peak.cu.
//
//   m16n8k4: A 16x4 (row): a[i] -> (g + 8i, t)   B 4x8 (col): b -> (t, g)
//            C 16x8: c[i] -> (g + 8(i>>1), 2t + (i&1))            g = lane>>2, t = lane&3
//   m8n8k4 : A 8x4: a -> (g, t)   B 4x8: b -> (t, g)   C 8x8: c[i] -> (g, 2t + i)
#pragma once

#include <cuda_runtime.h>

namespace lt {

__device__ __forceinline__ void dmma_m16n8k4(double (&d)[4], double a0, double a1, double b0) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                 : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
                 : "d"(a0), "d"(a1), "d"(b0));
}

__device__ __forceinline__ void dmma_m8n8k4(double (&d)[2], double a0, double b0) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a0), "d"(b0));
}

// CTA tile GEMM, 256 threads: C[64 x 64] += sum_{k in [k0,k1)} A(m, k) B(k, n).
// Warps 4 (m) x 2 (n), warp tile 16 x 32 (4 m16n8 tiles). Shared tiles BK = 16 deep,
// double-buffered through registers. Loaders return 0 outside their domain; the tile
// loads walk k fastest (coalesced for k-contiguous operands).
constexpr int kGBM = 64, kGBN = 64, kGBK = 16;
constexpr int kGLDA = kGBK + 4;  // A smem row stride (doubles): conflict-free fragment reads
constexpr int kGLDB = kGBN + 8;  // B smem row stride

struct GemmSmem {
    double A[kGBM * kGLDA];
    double B[kGBK * kGLDB];
};

template <class LA, class LB>
__device__ __forceinline__ void cta_gemm_64x64(const LA& loadA, const LB& loadB, long long k0, long long k1,
                                               double (&acc)[4][4], GemmSmem& sm) {
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int wm = warp & 3, wn = warp >> 2;
    const int g = lane >> 2, t = lane & 3;
    double ra[4], rb[4];
    auto fetch = [&](long long kb) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = tid + 256 * u;
            const int am = e >> 4, ak = e & 15;  // A tile: k fastest
            ra[u] = (kb + ak < k1) ? loadA(am, kb + ak) : 0.0;
            const int bn = e >> 4, bk = e & 15;  // B tile: k fastest
            rb[u] = (kb + bk < k1) ? loadB(kb + bk, bn) : 0.0;
        }
    };
    if (k0 >= k1) return;
    fetch(k0);
    for (long long kb = k0; kb < k1; kb += kGBK) {
        __syncthreads();
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = tid + 256 * u;
            sm.A[(e >> 4) * kGLDA + (e & 15)] = ra[u];
            sm.B[(e & 15) * kGLDB + (e >> 4)] = rb[u];
        }
        __syncthreads();
        if (kb + kGBK < k1) fetch(kb + kGBK);  // overlap the next tile's loads with the MMAs
#pragma unroll
        for (int ks = 0; ks < kGBK; ks += 4) {
            const double a0 = sm.A[(wm * 16 + g) * kGLDA + ks + t];
            const double a1 = sm.A[(wm * 16 + g + 8) * kGLDA + ks + t];
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
                const double b0 = sm.B[(ks + t) * kGLDB + wn * 32 + nt * 8 + g];
                dmma_m16n8k4(acc[nt], a0, a1, b0);
            }
        }
    }
}

// accumulator element -> (m, n) inside the 64 x 64 tile
__device__ __forceinline__ void acc_coord(int nt, int i, int& m, int& n) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = warp & 3, wn = warp >> 2;
    const int g = lane >> 2, t = lane & 3;
    m = wm * 16 + g + 8 * (i >> 1);
    n = wn * 32 + nt * 8 + 2 * t + (i & 1);
}

}  // namespace lt
