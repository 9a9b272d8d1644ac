// k_nuclear.cu — Galerkin nuclear-attraction contraction (galerkin.cpp:109-125, :224-247, :273-284).
//
// The reference computes, per direction l and (cell k, offset d, rank term r),
// the table T_l[k,d,r](mu,nu) = sum_i g_mu(i - s_A) g_nu(i - s_B) p_r(i) (dot3), then
// combines H_nuc[k,d](mu,nu) = sum_r w_r prod_l T_l. Two generic device strategies live here:
//
//   direct   (launch_nuc_direct)  the table itself, for trivial directions (L_l = 1,
//            one (k,d) pair) and for box lattices with several non-trivial directions;
//   fold     (launch_nuc_fold)    periodic wrapped directions address p(i mod n), so
//            T[d,r](mu,nu) = sum_{t<n} p_r(t) Qf_d(mu,nu)(t) with the folded product
//            Qf_d(t) = sum_{i = t mod n} g_mu(i) g_nu(i - d n): the contraction shrinks
//            from the support length to n before meeting the R rank columns;
// (box chains with one non-trivial direction use the DMMA Hankel path in k_nuclear2.cu.)
// Each is the same sum as the reference, reassociated; see DESIGN.md for the flop counts.
#include "lt_device.cuh"
#include "lt_internal.cuh"

namespace lt {

// ---------------------------------------------------------------------------
// direct tables: CTA per (e, pair, r-chunk)
// ---------------------------------------------------------------------------
constexpr int kRChunk = 16;
constexpr int kDirThreads = 128;

__global__ void __launch_bounds__(kDirThreads) k_nuc_direct(Index m0, Index Rtot, Index L, Index n, Index band,
                                                            Index rows, int periodic, int tiled,
                                                            const double* __restrict__ pwc, Index G,
                                                            const unsigned long long* __restrict__ plo,
                                                            const unsigned long long* __restrict__ phi,
                                                            const double* __restrict__ pot, double* __restrict__ T) {
    const Index e = blockIdx.x;
    const Index pair = blockIdx.y;
    const Index r0 = static_cast<Index>(blockIdx.z) * kRChunk;
    const Index mu = e % m0, nu = e / m0;
    const Index width = 2 * band + 1;
    Index k = 0, d = 0;
    if (periodic) {
        d = pair - band;
    } else {
        k = pair / width;
        d = pair % width - band;
        if (k + d < 0 || k + d >= L) return;
    }
    const Index shA = (periodic ? 0 : k) * n;
    const Index shB = (periodic ? d : k + d) * n;
    const Index offA = static_cast<Index>(plo[mu]) + shA, endA = static_cast<Index>(phi[mu]) + shA;
    const Index offB = static_cast<Index>(plo[nu]) + shB, endB = static_cast<Index>(phi[nu]) + shB;
    Index lo = max(offA, offB), hi = min(endA, endB);
    if (!tiled) {
        lo = max(lo, Index(0));
        hi = min(hi, rows);
    }
    const double* a = pwc + mu * G;
    const double* b = pwc + nu * G;
    const Index nr = min(Index(kRChunk), Rtot - r0);
    double acc[kRChunk];
#pragma unroll
    for (int q = 0; q < kRChunk; ++q) acc[q] = 0.0;
    for (Index i = lo + threadIdx.x; i < hi; i += kDirThreads) {
        const double ab = a[i - shA] * b[i - shB];
        const Index pi = tiled ? (i % n) : i;
#pragma unroll
        for (int q = 0; q < kRChunk; ++q)
            if (q < nr) acc[q] += ab * pot[(r0 + q) * rows + pi];
    }
    __shared__ double red[kDirThreads / 32][kRChunk];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < kRChunk; ++q) {
        const double v = warp_sum(acc[q]);
        if (lane == 0) red[w][q] = v;
    }
    __syncthreads();
    if (threadIdx.x < nr) {
        double s = 0.0;
        for (int ww = 0; ww < kDirThreads / 32; ++ww) s += red[ww][threadIdx.x];
        T[(pair * Rtot + r0 + threadIdx.x) * m0 * m0 + e] = s;
    }
}

void launch_nuc_direct(const Launch& L, Index m0, Index Rtot, const DirPlan& d, bool periodic, const double* pwc,
                       const unsigned long long* lo, const unsigned long long* hi, const double* pot, double* T) {
    dim3 grid(static_cast<unsigned>(m0 * m0), static_cast<unsigned>(d.npairs),
              static_cast<unsigned>((Rtot + kRChunk - 1) / kRChunk));
    Stage st_(L, "nuc_direct");
    k_nuc_direct<<<grid, kDirThreads, 0, L.st>>>(m0, Rtot, d.L, d.n, d.band, d.pot_rows, periodic ? 1 : 0,
                                                 d.tiled ? 1 : 0, pwc, d.G, lo, hi, pot, T);
    LT_CU(cudaGetLastError());
    L.tick();
}

// ---------------------------------------------------------------------------
// periodic fold
// ---------------------------------------------------------------------------
__global__ void k_fold(Index m0, Index n, Index band, const double* __restrict__ pwc, Index G,
                       const unsigned long long* __restrict__ plo, const unsigned long long* __restrict__ phi,
                       double* __restrict__ Qf) {
    const Index e = blockIdx.x;
    const Index di = blockIdx.y;
    const Index mu = e % m0, nu = e / m0;
    const Index d = di - band;
    const Index shB = d * n;
    const Index lo = max(static_cast<Index>(plo[mu]), static_cast<Index>(plo[nu]) + shB);
    const Index hi = min(static_cast<Index>(phi[mu]), static_cast<Index>(phi[nu]) + shB);
    const double* a = pwc + mu * G;
    const double* b = pwc + nu * G;
    for (Index t = threadIdx.x; t < n; t += blockDim.x) {
        double acc = 0.0;
        if (lo < hi) {
            Index i = lo + (((t - lo) % n) + n) % n;
            for (; i < hi; i += n) acc += a[i] * b[i - shB];
        }
        Qf[(di * m0 * m0 + e) * n + t] = acc;
    }
}

// T[d][r][e] = sum_t P[r][t] Qf[d][e][t]; CTA per (d, r), threads over e
__global__ void k_fold_gemm(Index m0, Index Rtot, Index n, const double* __restrict__ pot,
                            const double* __restrict__ Qf, double* __restrict__ T) {
    const Index di = blockIdx.x, r = blockIdx.y;
    extern __shared__ double ps[];
    for (Index t = threadIdx.x; t < n; t += blockDim.x) ps[t] = pot[r * n + t];
    __syncthreads();
    const Index mm = m0 * m0;
    for (Index e = threadIdx.x; e < mm; e += blockDim.x) {
        const double* q = Qf + (di * mm + e) * n;
        double acc = 0.0;
        for (Index t = 0; t < n; ++t) acc += ps[t] * q[t];
        T[(di * Rtot + r) * mm + e] = acc;
    }
}

void launch_nuc_fold(const Launch& L, Index m0, Index Rtot, const DirPlan& d, const double* pwc,
                     const unsigned long long* lo, const unsigned long long* hi, const double* pot, double* Qf,
                     double* T) {
    dim3 g1(static_cast<unsigned>(m0 * m0), static_cast<unsigned>(d.width));
    const int th = static_cast<int>(std::min<Index>(256, ((d.n + 31) / 32) * 32));
    Stage st_(L, "nuc_fold");
    k_fold<<<g1, th, 0, L.st>>>(m0, d.n, d.band, pwc, d.G, lo, hi, Qf);
    LT_CU(cudaGetLastError());
    dim3 g2(static_cast<unsigned>(d.width), static_cast<unsigned>(Rtot));
    const size_t smem = sizeof(double) * d.n;
    if (smem > 48 * 1024) LT_CU(cudaFuncSetAttribute(k_fold_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_fold_gemm<<<g2, 128, smem, L.st>>>(m0, Rtot, d.n, pot, Qf, T);
    LT_CU(cudaGetLastError());
    L.tick(2);
}

}  // namespace lt
