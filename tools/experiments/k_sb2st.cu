// k_sb2st.cu — two-stage tridiagonalisation of the dense box pencil's reduced matrix
// A = L^-1 H L^-T (eigensolver.cpp:20-28; the eigenvalues of SelfAdjointEigenSolver),
// replacing the one-stage reduction's n - 1 dependent grid-wide exchanges.
//
// Stage 1 (dense -> band of half-bandwidth KD), per panel of KD columns c0 .. c0+KD-1:
//   k_sb_panel   one CTA: Householder QR of the panel below its diagonal block (dgeqr2, rows
//                in registers, block reductions), the block reflector's T (dlarft, forward
//                columnwise), V T; R and the diagonal block's lower band go to the band buffer
//   k_sb_symm    W = A22 (V T): the trailing matrix (L2-resident) times a skinny operand, and
//                per-CTA partial products V^T W of the CTA's rows
//   k_sb_z       Z = W - 1/2 V (T^T V^T W), the partials summed in a fixed order
//   update       A22 -= [V Z] [Z V]^T: TMA-fed DMMA GEMM (k_dgemm_tn), lower tiles mirrored
//   (the two-sided update Q^T A22 Q, Q = I - V T V^T, of dsytrd_sy2sb)
// Stage 2 (band -> tridiagonal), k_sb2st: the band in shared memory (diagonals 0 .. 2 KD, the
//   upper half for the bulges), one sweep per column chased down by Householder reflectors of
//   length KD (the task sequence of LAPACK dsb2st_kernels: type 1, then alternating type 2 -
//   right-apply the previous reflector to the block below, generate the next one from its first
//   column, left-apply it - and type 3 - two-sided apply to the next diagonal block). Sweeps
//   are pipelined over the CTA's warps: sweep s runs task t once sweep s - 1 has finished task
//   t + 3 (their index windows are then disjoint).
// The tridiagonal (d, e) goes to the Sturm multisection of k_dense.cu.
#include "dmma.cuh"
#include "lt_internal.cuh"

// MEASURED DEAD END (kept out of the product build). B200, n = 1024,
// KD = 12 (tools/experiments/sb_probe.cu): stage 1 12.7 ms (85 panels x ~150 us: one-CTA panel
// QR 64 us, skinny TMA GEMMs 28 us each - a 4-stage ring cannot cover L2 latency along a
// 1000-long K in 1-16 CTAs), stage 2 17.8-20.9 ms (the chase is issue-bound on one SM:
// ~1k warp instructions per task x 87k tasks). The one-stage reduction takes 4.2 ms.
namespace lt {
struct SbBufs {
    double *band, *U1, *U2, *Vt, *VTt, *Wt, *M, *T;
};
int sb2st_kd(int n);
void launch_two_stage_tridiag(const Launch& L, int n, double* A, long long ld, const SbBufs& b, double* d, double* e);
}  // namespace lt

#include <algorithm>

#ifdef LT_SB_PROFILE
__device__ long long lt_sb_prof[4096][2];  // per sweep: clock64 at start, at end
#endif

namespace lt {

namespace {


// block-wide sum of NV values (result in every thread); red: >= NV * 33 doubles. Warps
// reduce by shuffles, warp 0 sums the per-warp partials (fixed order), one broadcast.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int q = 0; q < NV; ++q)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
    __syncthreads();  // red free (previous readers done)
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < NV; ++q) red[q * 32 + warp] = v[q];
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            double x = lane < nw ? red[q * 32 + lane] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            if (lane == 0) red[NV * 32 + q] = x;
        }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NV; ++q) v[q] = red[NV * 32 + q];
}

}  // namespace

// ---------------------------------------------------------------------------------------
// stage 1: panel QR
// ---------------------------------------------------------------------------------------
constexpr int kPanelThreads = 256;

// rows per thread: m <= 1024 at KD = 12, m <= 2048 at KD = 8
template <int KD>
__host__ __device__ constexpr int panel_rows() { return KD > 8 ? 4 : 8; }

// Householder QR of P = A[r0 .. n-1][c0 .. c0+KD-1] (r0 = c0 + KD, m = n - r0 rows, rows
// rho = tid + 256 q in registers). Column g: the reflector (dlarfg), then ONE block reduction
// carries both w_j = v_g^T P[:, j] (j > g) for the update and the Gram entries V[:, i]^T v_g
// (i < g) for the block reflector's T (dlarft, forward columnwise), computed by thread 0.
// Outputs: V into U1[:, 0:KD] and U2[:, KD:2KD] (row-major m x 2KD), V^T and (V T)^T row-major
// KD x mp (the GEMM operands), T (KD x KD), and the band (diagonals 0 .. KD, pitch n) of the
// panel's columns: the diagonal block's lower band and R.
template <int KD>
__global__ void __launch_bounds__(kPanelThreads) k_sb_panel(int n, const double* __restrict__ A, long long ld, int c0,
                                                           int mp, double* __restrict__ band, double* __restrict__ U1,
                                                           double* __restrict__ U2, double* __restrict__ Vt,
                                                           double* __restrict__ VTt, double* __restrict__ Tg) {
    constexpr int R = panel_rows<KD>();
    constexpr int NR = KD - 1;  // reduction width
    __shared__ double red[(NR + 1) * 33];
    __shared__ double sG[KD][KD];  // Gram: sG[g][i] = V[:, i]^T v_g (i < g)
    __shared__ double sT[KD][KD];
    __shared__ double sbc;
    const int r0 = c0 + KD, m = n - r0;
    const int tid = threadIdx.x;
    double p[R][KD];
#pragma unroll
    for (int q = 0; q < R; ++q) {
        const int rho = tid + kPanelThreads * q;
#pragma unroll
        for (int g = 0; g < KD; ++g) p[q][g] = rho < m ? A[static_cast<long long>(c0 + g) * ld + r0 + rho] : 0.0;
    }
    double tau[KD];
#pragma unroll
    for (int g = 0; g < KD; ++g) {
        double xs[1] = {0.0};
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const int rho = tid + kPanelThreads * q;
            if (rho > g && rho < m) xs[0] = fma(p[q][g], p[q][g], xs[0]);
            if (rho == g) sbc = p[q][g];
        }
        block_sum<1>(xs, red);  // its barriers publish sbc
        const double alpha = sbc, xn2 = xs[0];
        double t = 0.0, beta = alpha, scal = 0.0;
        if (xn2 != 0.0) {
            const double nrm = sqrt(fma(alpha, alpha, xn2));
            beta = alpha >= 0.0 ? -nrm : nrm;
            t = (beta - alpha) / beta;
            scal = 1.0 / (alpha - beta);
        }
        tau[g] = t;
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const int rho = tid + kPanelThreads * q;
            if (rho > g) p[q][g] *= scal;  // v below the unit entry
            if (rho == g) p[q][g] = beta;  // R(g, g)
        }
        if (g == 0 && KD == 1) continue;
        // r[j - 1] = v_g^T P[:, j] (j > g); r[i] = V[:, i]^T v_g (i < g)
        double r[NR];
#pragma unroll
        for (int j = 0; j < NR; ++j) r[j] = 0.0;
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const int rho = tid + kPanelThreads * q;
            if (rho < g || rho >= m) continue;
            const double vg = rho == g ? 1.0 : p[q][g];
#pragma unroll
            for (int j = g + 1; j < KD; ++j) r[j - 1] = fma(vg, p[q][j], r[j - 1]);
#pragma unroll
            for (int i = 0; i < g; ++i) r[i] = fma(rho == i ? 1.0 : p[q][i], vg, r[i]);  // rho >= g > i
        }
        block_sum<NR>(r, red);
        if (tid == 0)
#pragma unroll
            for (int i = 0; i < g; ++i) sG[g][i] = r[i];
        if (t != 0.0)
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const int rho = tid + kPanelThreads * q;
                if (rho < g || rho >= m) continue;
                const double vg = rho == g ? 1.0 : p[q][g];
#pragma unroll
                for (int j = g + 1; j < KD; ++j) p[q][j] = fma(-t * vg, r[j - 1], p[q][j]);
            }
    }
    // T[j][j] = tau_j, T[0:j][j] = -tau_j T[0:j][0:j] G[0:j][j]
    if (tid == 0) {
        for (int j = 0; j < KD; ++j) {
            for (int i = j + 1; i < KD; ++i) sT[i][j] = 0.0;
            sT[j][j] = tau[j];
            for (int i = 0; i < j; ++i) {
                double acc = 0.0;
                for (int k = i; k < j; ++k) acc = fma(sT[i][k], sG[j][k], acc);
                sT[i][j] = -tau[j] * acc;
            }
        }
        for (int i = 0; i < KD * KD; ++i) Tg[i] = sT[i / KD][i % KD];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < R; ++q) {
        const int rho = tid + kPanelThreads * q;
        if (rho >= m) continue;
        double v[KD];
#pragma unroll
        for (int i = 0; i < KD; ++i) v[i] = rho == i ? 1.0 : (rho > i ? p[q][i] : 0.0);
        const long long ro = static_cast<long long>(rho) * 2 * KD;
#pragma unroll
        for (int i = 0; i < KD; ++i) {
            U1[ro + i] = v[i];
            U2[ro + KD + i] = v[i];
            Vt[static_cast<long long>(i) * mp + rho] = v[i];
        }
#pragma unroll
        for (int c = 0; c < KD; ++c) {
            double acc = 0.0;
#pragma unroll
            for (int i = 0; i <= c; ++i) acc = fma(v[i], sT[i][c], acc);
            VTt[static_cast<long long>(c) * mp + rho] = acc;
        }
        // R(rho, g), rho <= g: row r0 + rho of column c0 + g, diagonal KD + rho - g
        if (rho < KD)
#pragma unroll
            for (int g = 0; g < KD; ++g)
                if (rho <= g) band[static_cast<long long>(KD + rho - g) * n + c0 + g] = p[q][g];
    }
    // the diagonal block's lower band (diagonals 0 .. KD - 1 - g of column c0 + g)
    for (int idx = tid; idx < KD * KD; idx += blockDim.x) {
        const int g = idx / KD, d = idx % KD;
        if (c0 + g + d < r0) band[static_cast<long long>(d) * n + c0 + g] = A[static_cast<long long>(c0 + g) * ld + c0 + g + d];
    }
}

// Z = W - V X, X = 1/2 T^T M (M = V^T W): Z -> U1[:, KD:2KD] and U2[:, 0:KD]; W from W^T (KD x mp)
template <int KD>
__global__ void __launch_bounds__(256) k_sb_z(int m, int mp, const double* __restrict__ M, const double* __restrict__ Tg,
                                              const double* __restrict__ Wt, double* __restrict__ U1,
                                              double* __restrict__ U2) {
    __shared__ double X[KD * KD];
    for (int idx = threadIdx.x; idx < KD * KD; idx += blockDim.x) {
        const int i = idx / KD, j = idx % KD;
        double acc = 0.0;
        for (int k = 0; k <= i; ++k) acc = fma(Tg[k * KD + i], M[k * KD + j], acc);  // (T^T M)[i][j], T upper
        X[idx] = 0.5 * acc;
    }
    __syncthreads();
    const int rho = blockIdx.x * blockDim.x + threadIdx.x;
    if (rho >= m) return;
    const long long ro = static_cast<long long>(rho) * 2 * KD;
    double v[KD];
#pragma unroll
    for (int i = 0; i < KD; ++i) v[i] = U1[ro + i];
#pragma unroll
    for (int j = 0; j < KD; ++j) {
        double acc = Wt[static_cast<long long>(j) * mp + rho];
#pragma unroll
        for (int i = 0; i < KD; ++i) acc = fma(-v[i], X[i * KD + j], acc);
        U1[ro + KD + j] = acc;
        U2[ro + j] = acc;
    }
}

// lower band of the trailing block A[j0 ..][j0 ..] (every entry of it lies within KD)
__global__ void k_sb_tail(int n, int kd, const double* __restrict__ A, long long ld, int j0, double* __restrict__ band) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    const int cols = n - j0;
    if (idx >= cols * (kd + 1)) return;
    const int j = j0 + idx / (kd + 1), d = idx % (kd + 1);
    band[static_cast<long long>(d) * n + j] = j + d < n ? A[static_cast<long long>(j) * ld + j + d] : 0.0;
}

// ---------------------------------------------------------------------------------------
// stage 2: band -> tridiagonal (one CTA, the band in shared memory)
// ---------------------------------------------------------------------------------------
constexpr int kChaseWarps = 32;

// shared-memory pitch of the band: P = 2 (mod 16) doubles, so that lanes walking one column
// (stride P) and lanes walking one row through the symmetric image (stride P - 1) both hit
// distinct 8-byte banks (at most 2-way for 12 lanes)
__host__ __device__ inline int chase_pitch(int n) { return n + (18 - n % 16) % 16; }

// dlarfg on x (length lm, x[0] = alpha) held one entry per lane (lanes < lm); v in the lanes
// (v[0] = 1), tau, beta
__device__ __forceinline__ void warp_larfg(int lm, double x, int lane, double& v, double& tau, double& beta) {
    double xs = (lane > 0 && lane < lm) ? x * x : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) xs += __shfl_xor_sync(0xffffffffu, xs, o);
    const double alpha = __shfl_sync(0xffffffffu, x, 0);
    tau = 0.0;
    beta = alpha;
    v = lane == 0 ? 1.0 : 0.0;
    if (lm > 1 && xs != 0.0) {
        const double nrm = sqrt(fma(alpha, alpha, xs));
        beta = alpha >= 0.0 ? -nrm : nrm;
        tau = (beta - alpha) / beta;
        const double scal = 1.0 / (alpha - beta);
        if (lane > 0 && lane < lm) v = x * scal;
    }
}

template <int KD>
__global__ void __launch_bounds__(32 * kChaseWarps, 1) k_sb2st(int n, const double* __restrict__ band,
                                                               double* __restrict__ dout, double* __restrict__ eout) {
    extern __shared__ double csm[];
    const int P = chase_pitch(n);
    double* ab = csm;  // diagonal d of column j at ab[d * P + j], d in [0, 2 KD]
    int* prog = reinterpret_cast<int*>(ab + static_cast<size_t>(2 * KD + 1) * P);
    double* scratch = reinterpret_cast<double*>(prog + ((n + 1) / 2) * 2);  // [warp][2][32]
    for (int idx = threadIdx.x; idx < (2 * KD + 1) * P; idx += blockDim.x) {
        const int d = idx / P, j = idx % P;
        ab[idx] = (d <= KD && j + d < n) ? band[static_cast<long long>(d) * n + j] : 0.0;
    }
    for (int s = threadIdx.x; s < n; s += blockDim.x) prog[s] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* wv = scratch + warp * 64;  // v (32) and w (32) of this warp
    constexpr int kDone = 1 << 30;
    // address of element (i, j) of the symmetric band (either triangle)
    auto sym = [&](int i, int j) -> int { return i >= j ? (i - j) * P + j : (j - i) * P + i; };
    for (int s = warp; s < n - 2; s += kChaseWarps) {
        volatile int* pv = prog;
        auto wait_for = [&](int t) {  // sweep s - 1 has finished task t + 3 (or all of it)
            if (s == 0) return;
            if (lane == 0)
                while (pv[s - 1] < t + 3) {
                }
            __syncwarp();
            __threadfence_block();
        };
        auto publish = [&](int t) {
            __threadfence_block();
            __syncwarp();
            if (lane == 0) pv[s] = t;
        };
        // two-sided symmetric update of the block [st, st+l) with (v, tau) (dlarfy, lower):
        // lane r owns row r: w = tau A v, w += -1/2 tau (w^T v) v, A -= v w^T + w v^T
        auto larfy = [&](int st, int l, double v, double tau) {
            if (tau == 0.0) return;
            wv[lane] = v;
            __syncwarp();
            double a[KD];
            double w0 = 0.0, w1 = 0.0;
            if (lane < l) {
#pragma unroll
                for (int j = 0; j < KD; ++j) a[j] = j < l ? ab[sym(st + lane, st + j)] : 0.0;
#pragma unroll
                for (int j = 0; j < KD; j += 2) w0 = fma(a[j], wv[j], w0);
#pragma unroll
                for (int j = 1; j < KD; j += 2) w1 = fma(a[j], wv[j], w1);
            }
            double w = tau * (w0 + w1);
            double h = lane < l ? w * v : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
            w = fma(-0.5 * tau * h, v, w);
            wv[32 + lane] = w;
            __syncwarp();
            if (lane < l)
#pragma unroll
                for (int j = 0; j < KD; ++j)
                    if (j <= lane && j < l) ab[(lane - j) * P + st + j] = fma(-v, wv[32 + j], fma(-w, wv[j], a[j]));
            __syncwarp();
        };
        // task 1: reflector of column s (rows s+1 .. s+lb), two-sided to the diagonal block
        int t = 1;
        wait_for(t);
#ifdef LT_SB_PROFILE
        if (lane == 0 && s < 4096) lt_sb_prof[s][0] = clock64();
#endif
        int st = s + 1, ed = min(s + KD, n - 1);
        double v, tau, beta;
        {
            const int lm = ed - st + 1;
            const double x = lane < lm ? ab[sym(st + lane, s)] : 0.0;
            warp_larfg(lm, x, lane, v, tau, beta);
            if (lane < lm && tau != 0.0) ab[sym(st + lane, s)] = lane == 0 ? beta : 0.0;
            __syncwarp();
            larfy(st, lm, v, tau);
        }
        publish(t);
        while (true) {
            const int ln = ed - st + 1;
            const int j1 = ed + 1, j2 = min(ed + KD, n - 1), lm = j2 - j1 + 1;
            if (lm <= 0) break;
            // type 2: C = A[j1 .. j2][st .. ed] (below the band's diagonal: C[r][c] at
            // ((j1 + r) - (st + c)) P + st + c) <- C H (right); the reflector of C's first
            // column, left-applied to C's other columns
            ++t;
            wait_for(t);
            double c[KD];  // lane r: row r of C
            if (lane < lm)
#pragma unroll
                for (int cc = 0; cc < KD; ++cc) c[cc] = cc < ln ? ab[(j1 + lane - st - cc) * P + st + cc] : 0.0;
            if (tau != 0.0) {
                wv[lane] = v;
                __syncwarp();
                double w0 = 0.0, w1 = 0.0;
                if (lane < lm) {
#pragma unroll
                    for (int cc = 0; cc < KD; cc += 2) w0 = fma(c[cc], wv[cc], w0);
#pragma unroll
                    for (int cc = 1; cc < KD; cc += 2) w1 = fma(c[cc], wv[cc], w1);
                }
                const double tw = tau * (w0 + w1);
#pragma unroll
                for (int cc = 0; cc < KD; ++cc) c[cc] = fma(-tw, wv[cc], c[cc]);
                __syncwarp();
            }
            warp_larfg(lm, c[0], lane, v, tau, beta);
            if (tau != 0.0) c[0] = lane == 0 ? beta : 0.0;
            if (tau != 0.0 && ln > 1) {
                // w_c = sum_r v_r C[r][c] (warp sums), C[r][c] -= tau v_r w_c
#pragma unroll
                for (int cc = 1; cc < KD; ++cc) {
                    double x = (lane < lm && cc < ln) ? v * c[cc] : 0.0;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
                    c[cc] = fma(-tau * v, x, c[cc]);
                }
            }
            if (lane < lm)
#pragma unroll
                for (int cc = 0; cc < KD; ++cc)
                    if (cc < ln) ab[(j1 + lane - st - cc) * P + st + cc] = c[cc];
            __syncwarp();
            publish(t);
            // type 3: two-sided to the diagonal block [j1, j2]
            ++t;
            wait_for(t);
            larfy(j1, lm, v, tau);
            publish(t);
            st = j1;
            ed = j2;
        }
        __threadfence_block();
        __syncwarp();
        if (lane == 0) pv[s] = kDone;
#ifdef LT_SB_PROFILE
        if (lane == 0 && s < 4096) lt_sb_prof[s][1] = clock64();
#endif
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        dout[i] = ab[i];
        if (i + 1 < n) eout[i] = ab[P + i];
    }
}

// ---------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------
static size_t sb2st_smem(int n, int kd) {
    return sizeof(double) * (2 * kd + 1) * static_cast<size_t>(chase_pitch(n)) + sizeof(int) * ((n + 1) / 2) * 2 +
           sizeof(double) * 64 * kChaseWarps;
}

int sb2st_kd(int n) {
    // the band (2 KD + 1 diagonals) and the per-warp scratch must fit one SM's shared memory;
    // the panel's rows must fit the panel kernel's registers
    if (n < 4 || n % 2) return 0;  // even n: 16-byte TMA row pitches
    if (n - 12 <= kPanelThreads * panel_rows<12>() && sb2st_smem(n, 12) <= 227 * 1024) return 12;
    if (n - 8 <= kPanelThreads * panel_rows<8>() && sb2st_smem(n, 8) <= 227 * 1024) return 8;
    return 0;
}

template <int KD>
static void run_two_stage(const Launch& L, int n, double* A, long long ld, const SbBufs& b, double* d, double* e) {
    int c0 = 0;
    for (; n - c0 - KD >= 2; c0 += KD) {
        const int r0 = c0 + KD, m = n - r0, mp = (m + 1) / 2 * 2;  // even pitch (TMA: 16-byte rows)
        {
            Stage st_(L, "sb_panel");
            k_sb_panel<KD><<<1, kPanelThreads, 0, L.st>>>(n, A, ld, c0, mp, b.band, b.U1, b.U2, b.Vt, b.VTt, b.T);
            LT_CU(cudaGetLastError());
            L.tick();
        }
        // W^T = ((A22 (V T))^T): A22 is symmetric, so its column-major storage read as rows is A22
        {
            const DgemmOperand a22{A + static_cast<long long>(r0) * ld + r0, m, m, ld}, vt{b.VTt, KD, m, mp};
            DgemmArgs g;
            g.M = m;
            g.N = KD;
            g.K = m;
            g.c1 = b.Wt;
            g.ldc = mp;
            g.flags = DG_C1_COLMAJOR;
            launch_dgemm_tn(L, a22, vt, g, 1, "sb_symm");
        }
        // M = V^T W (KD x KD)
        {
            const DgemmOperand vt{b.Vt, KD, m, mp}, wt{b.Wt, KD, m, mp};
            DgemmArgs g;
            g.M = KD;
            g.N = KD;
            g.K = m;
            g.c0 = b.M;
            g.ldc = KD;
            launch_dgemm_tn(L, vt, wt, g, 1, "sb_vtw");
        }
        {
            Stage st_(L, "sb_z");
            k_sb_z<KD><<<(m + 255) / 256, 256, 0, L.st>>>(m, mp, b.M, b.T, b.Wt, b.U1, b.U2);
            LT_CU(cudaGetLastError());
            L.tick();
        }
        // A22 -= [V Z] [Z V]^T (lower tiles, mirrored)
        const DgemmOperand u1{b.U1, m, 2 * KD, 2 * KD}, u2{b.U2, m, 2 * KD, 2 * KD};
        DgemmArgs g;
        g.M = m;
        g.N = m;
        g.K = 2 * KD;
        g.c0 = A + static_cast<long long>(r0) * ld + r0;
        g.ldc = ld;
        g.alpha = -1.0;
        g.beta_one = 1;
        g.flags = DG_C0_COLMAJOR | DG_LOWER | DG_MIRROR;
        launch_dgemm_tn(L, u1, u2, g, 1, "sb_update");
    }
    {
        Stage st_(L, "sb_tail");
        const int cols = n - c0;
        k_sb_tail<<<(cols * (KD + 1) + 255) / 256, 256, 0, L.st>>>(n, KD, A, ld, c0, b.band);
        LT_CU(cudaGetLastError());
        L.tick();
    }
    const size_t smem = sb2st_smem(n, KD);
    LT_CU(cudaFuncSetAttribute(k_sb2st<KD>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    Stage st_(L, "sb2st");
    k_sb2st<KD><<<1, 32 * kChaseWarps, smem, L.st>>>(n, b.band, d, e);
    LT_CU(cudaGetLastError());
    L.tick();
}

void launch_two_stage_tridiag(const Launch& L, int n, double* A, long long ld, const SbBufs& b, double* d, double* e) {
    const int kd = sb2st_kd(n);
    if (kd == 12) run_two_stage<12>(L, n, A, ld, b, d, e);
    else if (kd == 8) run_two_stage<8>(L, n, A, ld, b, d, e);
    else fail(LT_EGENERIC, "two-stage tridiagonalisation: size out of range");
}

}  // namespace lt
