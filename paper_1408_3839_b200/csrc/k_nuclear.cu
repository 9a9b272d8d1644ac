// k_nuclear.cu — Galerkin nuclear-attraction contraction (galerkin.cpp:109-125, :224-247, :273-284).
//
// The reference computes, per direction l and (cell k, offset d, rank term r),
// the table T_l[k,d,r](mu,nu) = sum_i g_mu(i - s_A) g_nu(i - s_B) p_r(i) (dot3), then
// combines H_nuc[k,d](mu,nu) = sum_r w_r prod_l T_l. Three device strategies cover it:
//
//   direct   (launch_nuc_direct)  the table itself, for trivial directions (L_l = 1,
//            one (k,d) pair) and for box lattices with several non-trivial directions;
//   fold     (launch_nuc_fold)    periodic wrapped directions address p(i mod n), so
//            T[d,r](mu,nu) = sum_{t<n} p_r(t) Qf_d(mu,nu)(t) with the folded product
//            Qf_d(t) = sum_{i = t mod n} g_mu(i) g_nu(i - d n): the contraction shrinks
//            from the support length to n before meeting the R rank columns;
//   box S2   (launch_box_*)       a box chain with one non-trivial direction l*: the
//            trivial directions' tables and the weights fold into W[r](mu,nu), the rank
//            sum into an effective potential V(mu,nu)(i) = sum_r W[r] p_r(i), and
//            H_nuc[k,d] = sum_j Q_d(j) V(j + k n) with Q_d(j) = g_mu(j) g_nu(j - d n):
//            a Hankel-operand GEMM (M = L cells, N = 2b+1 offsets, K = support) per pair.
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

// ---------------------------------------------------------------------------
// box chain (S2)
// ---------------------------------------------------------------------------
__global__ void k_box_w(Index mm, Index Rtot, const double* __restrict__ potw, const double* __restrict__ Ta,
                        const double* __restrict__ Tb, double* __restrict__ W) {
    const Index idx = static_cast<Index>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= mm * Rtot) return;
    const Index r = idx / mm;
    W[idx] = potw[r] * (Ta[idx] * Tb[idx]);
}

void launch_box_w(const Launch& L, Index m0, Index Rtot, const double* potw, const double* Ta, const double* Tb,
                  double* W) {
    const Index tot = m0 * m0 * Rtot;
    Stage st_(L, "box_w");
    k_box_w<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, L.st>>>(m0 * m0, Rtot, potw, Ta, Tb, W);
    LT_CU(cudaGetLastError());
    L.tick();
}

// V[e][i] = sum_r W[r][e] P[r][i]
__global__ void k_box_v(Index mm, Index Rtot, Index G, const double* __restrict__ W, const double* __restrict__ pot,
                        double* __restrict__ V) {
    const Index i = static_cast<Index>(blockIdx.x) * blockDim.x + threadIdx.x;
    const Index e = blockIdx.y;
    if (i >= G) return;
    double acc = 0.0;
    for (Index r = 0; r < Rtot; ++r) acc += W[r * mm + e] * pot[r * G + i];
    V[e * G + i] = acc;
}

void launch_box_v(const Launch& L, Index m0, Index Rtot, Index G, const double* W, const double* pot, double* V) {
    dim3 grid(static_cast<unsigned>((G + 255) / 256), static_cast<unsigned>(m0 * m0));
    Stage st_(L, "box_v");
    k_box_v<<<grid, 256, 0, L.st>>>(m0 * m0, Rtot, G, W, pot, V);
    LT_CU(cudaGetLastError());
    L.tick();
}

// Hankel GEMM per pair e: C[k][d] = sum_j Q_d(j) Vpad(j + k n)
constexpr int kCK = 64;   // k tile
constexpr int kCD = 32;   // d tile
constexpr int kCJ = 32;   // j step

__global__ void __launch_bounds__(256) k_box_corr(Index m0, Index L, Index n, Index band, Index G,
                                                  const double* __restrict__ pwc,
                                                  const unsigned long long* __restrict__ plo,
                                                  const unsigned long long* __restrict__ phi,
                                                  const double* __restrict__ V, double* __restrict__ part,
                                                  int nsplit) {
    const Index e = blockIdx.y;
    const Index mu = e % m0, nu = e / m0;
    const Index width = 2 * band + 1;
    const Index nkt = (L + kCK - 1) / kCK;
    const Index kt = blockIdx.x % nkt, dt = blockIdx.x / nkt;
    const Index k0 = kt * kCK, d0 = dt * kCD;  // d index (0..width-1)
    const int split = blockIdx.z;
    const Index alo = static_cast<Index>(plo[mu]), ahi = static_cast<Index>(phi[mu]);
    const Index blo = static_cast<Index>(plo[nu]), bhi = static_cast<Index>(phi[nu]);
    const Index dmin = d0 - band, dmax = min(d0 + kCD, width) - 1 - band;
    Index jlo = max(alo, blo + dmin * n), jhi = min(ahi, bhi + dmax * n);
    __shared__ double Qs[kCD][kCJ + 1];
    __shared__ double Vs[kCK][kCJ + 1];
    const int tx = threadIdx.x & 15;  // d pair
    const int ty = threadIdx.x >> 4;  // k quad
    double acc[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
    if (jlo < jhi) {
        const Index len = jhi - jlo;
        const Index per = ((len + nsplit - 1) / nsplit + kCJ - 1) / kCJ * kCJ;
        const Index js = jlo + split * per;
        const Index je = min(jhi, js + per);
        const double* a = pwc + mu * G;
        const double* b = pwc + nu * G;
        const double* v = V + e * G;
        for (Index j0 = js; j0 < je; j0 += kCJ) {
            for (int idx = threadIdx.x; idx < kCD * kCJ; idx += 256) {
                const int dd = idx / kCJ, jj = idx % kCJ;
                const Index j = j0 + jj;
                const Index d = d0 + dd - band;
                double q = 0.0;
                const Index jb = j - d * n;
                if (d0 + dd < width && j < je && j >= alo && j < ahi && jb >= blo && jb < bhi) q = a[j] * b[jb];
                Qs[dd][jj] = q;
            }
            for (int idx = threadIdx.x; idx < kCK * kCJ; idx += 256) {
                const int kk = idx / kCJ, jj = idx % kCJ;
                const Index j = j0 + jj;
                const Index gi = j + (k0 + kk) * n;
                Vs[kk][jj] = (j < je && k0 + kk < L && gi < G) ? v[gi] : 0.0;
            }
            __syncthreads();
#pragma unroll 8
            for (int jj = 0; jj < kCJ; ++jj) {
                const double q0 = Qs[2 * tx][jj], q1 = Qs[2 * tx + 1][jj];
#pragma unroll
                for (int a4 = 0; a4 < 4; ++a4) {
                    const double vv = Vs[ty * 4 + a4][jj];
                    acc[a4][0] += vv * q0;
                    acc[a4][1] += vv * q1;
                }
            }
            __syncthreads();
        }
    }
    // partial [split][e][k][d]
#pragma unroll
    for (int a4 = 0; a4 < 4; ++a4) {
        const Index k = k0 + ty * 4 + a4;
        if (k >= L) continue;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const Index di = d0 + 2 * tx + c;
            if (di >= width) continue;
            part[((static_cast<Index>(split) * m0 * m0 + e) * L + k) * width + di] = acc[a4][c];
        }
    }
}

// N[k][d][e] = sum_split part[split][e][k][d] (fixed order)
__global__ void k_box_reduce(Index mm, Index L, Index width, int nsplit, const double* __restrict__ part,
                             double* __restrict__ N) {
    const Index idx = static_cast<Index>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= mm * L * width) return;
    const Index e = idx % mm;
    const Index kd = idx / mm;  // k*width + d
    double s = 0.0;
    for (int sp = 0; sp < nsplit; ++sp) s += part[(static_cast<Index>(sp) * mm + e) * L * width + kd];
    N[idx] = s;
}

void launch_box_corr(const Launch& L, Index m0, const DirPlan& d, const double* pwc, const unsigned long long* lo,
                     const unsigned long long* hi, const double* V, double* Npart, double* N, int nsplit) {
    const Index nkt = (d.L + kCK - 1) / kCK;
    const Index ndt = (d.width + kCD - 1) / kCD;
    dim3 grid(static_cast<unsigned>(nkt * ndt), static_cast<unsigned>(m0 * m0), static_cast<unsigned>(nsplit));
    {
        Stage st_(L, "box_corr");
        k_box_corr<<<grid, 256, 0, L.st>>>(m0, d.L, d.n, d.band, d.G, pwc, lo, hi, V, Npart, nsplit);
        LT_CU(cudaGetLastError());
    }
    const Index tot = m0 * m0 * d.L * d.width;
    Stage st2_(L, "box_reduce");
    k_box_reduce<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, L.st>>>(m0 * m0, d.L, d.width, nsplit, Npart, N);
    LT_CU(cudaGetLastError());
    L.tick(2);
}

}  // namespace lt
