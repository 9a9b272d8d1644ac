// k_dense2.cu — front end of the dense box pencil (eigensolver.cpp:12-35):
//
//   LLT<MatrixXd> llt(S);  A = L^-1 H L^-T;  SelfAdjointEigenSolver(0.5 (A + A^T))
//
// on the device without library calls:
//   1. blocked right-looking Cholesky, 64-column panels. k_potf_leaf factors the diagonal
//      block in shared memory (one barrier per column: the trailing update uses the unscaled
//      column and 1 / pivot, Eigen's pivot test x <= 0 -> not positive definite) and inverts
//      it; the panel L_ij = S_ij L_jj^-T and the trailing update S_il -= L_ij L_lj^T are
//      TMA-fed DMMA GEMMs (k_dgemm.cu). L is kept row-major in place of S (S is symmetric,
//      so its column-major input is also its row-major form): every product reads K-major.
//   2. L^-1 by recursive doubling from the 64 x 64 leaf inverses: for block pairs of size s,
//      X21 = -L22^-1 (L21 L11^-1), both GEMMs batched over the pairs of a level; L^-1 is
//      written row-major (Li) and column-major (Lic), the layouts its two uses read K-major.
//   3. W^T = H L^-T (W stored row-major), A = W L^-T on the lower tiles, mirrored: A is
//      exactly symmetric, which is what 0.5 (A + A^T) produces from a rounding-symmetric A.
// The triangular operands' zero parts are skipped at tile granularity (L^-1 row n has
// k <= n only).
#include "dmma.cuh"
#include "lt_internal.cuh"

namespace lt {

constexpr int kLeaf = 64;

__device__ __forceinline__ double leaf_rsqrt(double x) {  // 1/sqrt(x) within an ulp
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double hx = 0.5 * x;
    y = y * fma(-hx * y, y, 1.5);
    y = y * fma(-hx * y, y, 1.5);
    return y * fma(-hx * y, y, 1.5);
}

// Cholesky + inverse of diagonal block j (rows/cols b0 .. b0 + m) of the row-major S in shared
// memory (padded to 64 with the identity), blocked by 8 columns:
//   A. lanes 0-7 of warp 0 factor the 8 x 8 diagonal block, a row per lane (shuffles; Eigen's
//      pivot test x <= 0 -> not positive definite), then invert it, a column per lane;
//   B. the panel below, L_r = A_r D^-T, a row per thread (reads and writes its own row only);
//   C. the trailing lower part A -= L_p L_p^T as m8n8k4 DMMA tiles spread over the warps.
// Then X = L^-1 from the eight 8 x 8 inverses by recursive doubling, X21 = -X22 (L21 X11),
// block pairs of 8, 16 and 32 as DMMA tiles.
constexpr int kLB = 8;
constexpr int kLL = 65;  // smem row stride

#ifdef LT_LEAF_PROFILE
__device__ long long lt_leaf_prof[64];
#define LPROF(i) \
    if (threadIdx.x == 0) lt_leaf_prof[i] = clock64();
#else
#define LPROF(i)
#endif

// C (tile rows r0.., cols c0..) += sgn * A(r0.., k0..k0+K) B(c0.., k0..k0+K)^T as one m8n8k4 tile
// (A, B, C in row-major smem with stride kLL); acc initialised from C when `acc_from_c`
__device__ __forceinline__ void leaf_tile(const double* A, int ar0, int ak0, const double* B, int br0, int bk0, int K,
                                          double* C, int cr0, int cc0, double sgn, bool acc_from_c) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    double acc[2];
    acc[0] = acc_from_c ? C[(cr0 + g) * kLL + cc0 + 2 * t] : 0.0;
    acc[1] = acc_from_c ? C[(cr0 + g) * kLL + cc0 + 2 * t + 1] : 0.0;
    for (int ks = 0; ks < K; ks += 4)
        dmma_m8n8k4(acc, sgn * A[(ar0 + g) * kLL + ak0 + ks + t], B[(br0 + g) * kLL + bk0 + ks + t]);
    C[(cr0 + g) * kLL + cc0 + 2 * t] = acc[0];
    C[(cr0 + g) * kLL + cc0 + 2 * t + 1] = acc[1];
}

__global__ void __launch_bounds__(256) k_potf_leaf(int n, long long ld, double* __restrict__ S, double* __restrict__ Li,
                                                   double* __restrict__ Lic, int j, unsigned long long* fail) {
    extern __shared__ double leaf_smem[];
    double* sA = leaf_smem;                    // [64][kLL]: the block -> L (lower)
    double* sX = leaf_smem + 64 * kLL;         // [64][kLL]: X = L^-1 (lower)
    double* sT = leaf_smem + 2 * 64 * kLL;     // [64][kLL]: X^T staging / merge temporaries
    __shared__ double srd[64];                 // 1 / L_rr
    __shared__ int bad;
    if (*fail != ~0ull) return;
    const int b0 = j * kLeaf, m = min(kLeaf, n - b0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int idx = tid; idx < 64 * 64; idx += 256) {
        const int r = idx >> 6, c = idx & 63;
        sA[r * kLL + c] = (r < m && c <= r) ? S[static_cast<long long>(b0 + r) * ld + b0 + c] : (r == c ? 1.0 : 0.0);
        sX[r * kLL + c] = 0.0;
    }
    if (tid == 0) bad = 0;
    LPROF(0);
    __syncthreads();
    LPROF(1);
    for (int kb = 0; kb < 64 / kLB; ++kb) {
        const int c0 = kb * kLB, r1 = c0 + kLB;
        // A: 8 x 8 factor (row per lane) and its inverse (column per lane)
        if (warp == 0) {
            double a[kLB];
            const int rl = lane & 7;
#pragma unroll
            for (int q = 0; q < kLB; ++q) a[q] = q <= rl ? sA[(c0 + rl) * kLL + c0 + q] : 0.0;
            int ok = 1;
#pragma unroll
            for (int q = 0; q < kLB; ++q) {
                const double piv = __shfl_sync(0xffffffffu, a[q], q);
                if (!(piv > 0.0)) ok = 0;
                const double rs = leaf_rsqrt(piv > 0.0 ? piv : 1.0);
                if (rl == q) {
                    a[q] = piv * rs;
                    srd[c0 + q] = rs;
                } else if (rl > q) {
                    a[q] *= rs;
                }
#pragma unroll
                for (int c = q + 1; c < kLB; ++c) {
                    const double lc = __shfl_sync(0xffffffffu, a[q], c);  // L[c][q]
                    if (rl >= c) a[c] = fma(-a[q], lc, a[c]);
                }
            }
            if (lane < kLB)
#pragma unroll
                for (int q = 0; q < kLB; ++q)
                    if (q <= lane) sA[(c0 + lane) * kLL + c0 + q] = a[q];
            if (!ok && lane == 0) {
                atomicMin(fail, 2ull);
                bad = 1;
            }
            __syncwarp();
            if (lane < kLB) {  // column `lane` of D^-1 by forward substitution
                double x[kLB];
#pragma unroll
                for (int r = 0; r < kLB; ++r) {
                    if (r < lane) {
                        x[r] = 0.0;
                        continue;
                    }
                    double acc = r == lane ? 1.0 : 0.0;
#pragma unroll
                    for (int k = 0; k < r; ++k)
                        if (k >= lane) acc = fma(-sA[(c0 + r) * kLL + c0 + k], x[k], acc);
                    x[r] = acc * srd[c0 + r];
                }
#pragma unroll
                for (int r = 0; r < kLB; ++r) sX[(c0 + r) * kLL + c0 + lane] = x[r];
            }
        }
        __syncthreads();
        LPROF(2 + 3 * kb);
        if (bad) return;
        // B: panel rows r1 .. 63, one row per thread: L[r][c0+q] = sum_{t <= q} A[r][c0+t] Dinv[q][t]
        if (tid < 64 - r1) {
            const int r = r1 + tid;
            double ar[kLB], lr[kLB];
#pragma unroll
            for (int t = 0; t < kLB; ++t) ar[t] = sA[r * kLL + c0 + t];
#pragma unroll
            for (int q = 0; q < kLB; ++q) {
                double acc = 0.0;
#pragma unroll
                for (int t = 0; t <= q; ++t) acc = fma(ar[t], sX[(c0 + q) * kLL + c0 + t], acc);
                lr[q] = acc;
            }
#pragma unroll
            for (int q = 0; q < kLB; ++q) sA[r * kLL + c0 + q] = lr[q];
        }
        __syncthreads();
        LPROF(3 + 3 * kb);
        // C: trailing lower part rows/cols >= r1: A -= L_p L_p^T (K = 8), 8 x 8 tiles on the warps
        {
            const int nt = (64 - r1) / 8;
            const int ntiles = nt * (nt + 1) / 2;
            for (int tile = warp; tile < ntiles; tile += 8) {
                int ti = 0, rem = tile;  // lower-triangular tile (ti, tj), tj <= ti
                while (rem > ti) {
                    rem -= ti + 1;
                    ++ti;
                }
                const int tj = rem;
                leaf_tile(sA, r1 + 8 * ti, c0, sA, r1 + 8 * tj, c0, kLB, sA, r1 + 8 * ti, r1 + 8 * tj, -1.0, true);
            }
        }
        __syncthreads();
        LPROF(4 + 3 * kb);
    }
    // X = L^-1 by recursive doubling: X21 = -X22 (L21 X11) for block pairs of size s = 8, 16, 32
    for (int sz = kLB; sz < 64; sz *= 2) {
        const int npair = 64 / (2 * sz), tpb = (sz / 8) * (sz / 8);  // 8 x 8 tiles per s x s block
        // T = L21 X11 -> sT rows o+s.., cols o.. (X11 lower: k >= col tile start)
        for (int w = warp; w < npair * tpb; w += 8) {
            const int pr = w / tpb, tt = w % tpb, o = pr * 2 * sz;
            const int ti = tt / (sz / 8), tj = tt % (sz / 8);
            // T[i][jj] = sum_k L[o+s+i][o+k] X[o+k][o+jj]: B operand rows = X^T -> use X11^T staged
            // in sT's upper area? X11[k][jj] read as B(jj, k) = X11^T[jj][k]: a strided read of sX
            const int lane2 = lane, g = lane2 >> 2, t = lane2 & 3;
            double acc[2] = {0.0, 0.0};
            for (int ks = 8 * tj; ks < sz; ks += 4)  // X11[k][jj] = 0 for k < jj (tile granularity)
                dmma_m8n8k4(acc, sA[(o + sz + 8 * ti + g) * kLL + o + ks + t], sX[(o + ks + t) * kLL + o + 8 * tj + g]);
            sT[(o + sz + 8 * ti + g) * kLL + o + 8 * tj + 2 * t] = acc[0];
            sT[(o + sz + 8 * ti + g) * kLL + o + 8 * tj + 2 * t + 1] = acc[1];
        }
        __syncthreads();
        // X21 = -X22 T (X22 lower: k <= row tile end)
        for (int w = warp; w < npair * tpb; w += 8) {
            const int pr = w / tpb, tt = w % tpb, o = pr * 2 * sz;
            const int ti = tt / (sz / 8), tj = tt % (sz / 8);
            const int g = lane >> 2, t = lane & 3;
            double acc[2] = {0.0, 0.0};
            for (int ks = 0; ks < 8 * (ti + 1); ks += 4)
                dmma_m8n8k4(acc, -sX[(o + sz + 8 * ti + g) * kLL + o + sz + ks + t], sT[(o + sz + ks + t) * kLL + o + 8 * tj + g]);
            sX[(o + sz + 8 * ti + g) * kLL + o + 8 * tj + 2 * t] = acc[0];
            sX[(o + sz + 8 * ti + g) * kLL + o + 8 * tj + 2 * t + 1] = acc[1];
        }
        __syncthreads();
    }
    LPROF(30);
    for (int idx = tid; idx < 64 * 64; idx += 256) {
        const int r = idx >> 6, c = idx & 63;  // consecutive threads: consecutive columns (row-major)
        if (r < m && c < m) {
            Li[static_cast<long long>(b0 + r) * ld + b0 + c] = r >= c ? sX[r * kLL + c] : 0.0;
            if (c <= r) S[static_cast<long long>(b0 + r) * ld + b0 + c] = sA[r * kLL + c];
        }
        const int cc = idx >> 6, rr = idx & 63;  // column-major: consecutive rows
        if (rr < m && cc < m) Lic[static_cast<long long>(b0 + cc) * ld + b0 + rr] = rr >= cc ? sX[rr * kLL + cc] : 0.0;
    }
}

static void launch_potf_leaf(const Launch& L, int n, long long ld, double* S, double* Li, double* Lic, int j,
                             unsigned long long* fail) {
    const int smem = static_cast<int>(sizeof(double) * 3 * 64 * kLL);
    static bool attr = false;
    if (!attr) {
        LT_CU(cudaFuncSetAttribute(k_potf_leaf, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr = true;
    }
    Stage st_(L, "potf_leaf");
    k_potf_leaf<<<1, 256, smem, L.st>>>(n, ld, S, Li, Lic, j, fail);
    LT_CU(cudaGetLastError());
    L.tick();
}

static void trtri_merges(const Launch& L, int n, long long ld, const DenseReduceBufs& b) {
    const DgemmOperand S{b.S, n, n, ld}, Li{b.Li, n, n, ld}, Lic{b.Lic, n, n, ld};
    const DgemmOperand T{b.T, n, n, ld};
    // 2. L^-1: X21 = -L22^-1 (L21 L11^-1) per block pair of size s
    for (int s = kLeaf; s < n; s *= 2) {
        const int full = n / (2 * s);
        for (int pass = 0; pass < 2; ++pass) {
            const int r0 = pass == 0 ? 0 : full * 2 * s;
            const int m2 = pass == 0 ? s : n - r0 - s;
            const int batches = pass == 0 ? full : (m2 > 0 ? 1 : 0);
            if (batches <= 0 || m2 <= 0) continue;
            const long long zs = 2LL * s;
            DgemmArgs t;  // T = L21 L11^-1 (column-major into T at the L21 block position)
            t.M = m2;
            t.N = s;
            t.K = s;
            t.a_row0 = r0 + s;
            t.a_col0 = r0;
            t.b_row0 = r0;
            t.b_col0 = r0;
            t.a_zrow = t.a_zcol = t.b_zrow = t.b_zcol = zs;
            t.c0 = b.T + static_cast<long long>(r0) * ld + r0 + s;
            t.ldc = ld;
            t.c_zoff = zs * ld + zs;
            t.flags = DG_K_GE_N | DG_C0_COLMAJOR;
            t.fail = b.fail;
            launch_dgemm_tn(L, S, Lic, t, batches, "trtri_merge");
            DgemmArgs x;  // X21 = -L22^-1 T -> Li (row-major) and Lic (column-major)
            x.M = m2;
            x.N = s;
            x.K = m2;
            x.a_row0 = r0 + s;
            x.a_col0 = r0 + s;
            x.b_row0 = r0;
            x.b_col0 = r0 + s;
            x.a_zrow = x.a_zcol = x.b_zrow = x.b_zcol = zs;
            x.c0 = b.Li + static_cast<long long>(r0 + s) * ld + r0;
            x.c1 = b.Lic + static_cast<long long>(r0) * ld + r0 + s;
            x.ldc = ld;
            x.c_zoff = zs * ld + zs;
            x.alpha = -1.0;
            x.flags = DG_K_LE_M | DG_C1_COLMAJOR;
            x.fail = b.fail;
            launch_dgemm_tn(L, Li, T, x, batches, "trtri_merge");
        }
    }
}

void dense_factor(const Launch& L, int n, long long ld, const DenseReduceBufs& b) {

    const DgemmOperand S{b.S, n, n, ld}, Li{b.Li, n, n, ld}, Lic{b.Lic, n, n, ld};
    const DgemmOperand T{b.T, n, n, ld};
    const int nblk = (n + kLeaf - 1) / kLeaf;
    // 1. Cholesky
    for (int j = 0; j < nblk; ++j) {
        launch_potf_leaf(L, n, ld, b.S, b.Li, b.Lic, j, b.fail);
        const int c0 = j * kLeaf, w = std::min(kLeaf, n - c0), r0 = c0 + w, rows = n - r0;
        if (rows <= 0) break;
        DgemmArgs p;  // L_ij = S_ij L_jj^-T (in place)
        p.M = rows;
        p.N = w;
        p.K = w;
        p.a_row0 = r0;
        p.a_col0 = c0;
        p.b_row0 = c0;
        p.b_col0 = c0;
        p.c0 = b.S + static_cast<long long>(r0) * ld + c0;
        p.ldc = ld;
        p.fail = b.fail;
        launch_dgemm_tn(L, S, Li, p, 1, "potrf_panel");
        DgemmArgs u;  // S_il -= L_ij L_lj^T, lower tiles
        u.M = rows;
        u.N = rows;
        u.K = w;
        u.a_row0 = r0;
        u.a_col0 = c0;
        u.b_row0 = r0;
        u.b_col0 = c0;
        u.c0 = b.S + static_cast<long long>(r0) * ld + r0;
        u.ldc = ld;
        u.alpha = -1.0;
        u.beta_one = 1;
        u.flags = DG_LOWER;
        u.fail = b.fail;
        launch_dgemm_tn(L, S, S, u, 1, "potrf_update");
    }
    trtri_merges(L, n, ld, b);
}

void dense_transform(const Launch& L, int n, long long ld, const DenseReduceBufs& b) {
    const DgemmOperand Li{b.Li, n, n, ld}, H{b.H, n, n, ld}, W{b.W, n, n, ld};
    // 3. W^T = H L^-T (W row-major), A = W L^-T (lower tiles, mirrored) into H
    DgemmArgs w;
    w.M = n;
    w.N = n;
    w.K = n;
    w.c0 = b.W;
    w.ldc = ld;
    w.flags = DG_K_LE_N | DG_C0_COLMAJOR;
    w.fail = b.fail;
    launch_dgemm_tn(L, H, Li, w, 1, "reduce_gemm");
    DgemmArgs a;
    a.M = n;
    a.N = n;
    a.K = n;
    a.c0 = b.H;
    a.ldc = ld;
    a.flags = DG_K_LE_N | DG_LOWER | DG_MIRROR;
    a.fail = b.fail;
    launch_dgemm_tn(L, W, Li, a, 1, "reduce_gemm");
}

void dense_reduce(const Launch& L, int n, long long ld, const DenseReduceBufs& b) {
    dense_factor(L, n, ld, b);
    dense_transform(L, n, ld, b);
}

void dense_back_transform(const Launch& L, int n, long long ld, const double* Lic, const double* Z, double* X,
                          const unsigned long long* fail) {
    // X(m, c) = sum_{k >= m} L^-1(k, m) Z(k, c): A(m, k) = Lic[m][k], B(c, k) = Z column c
    const DgemmOperand A{Lic, n, n, ld}, B{Z, n, n, ld};
    DgemmArgs x;
    x.M = n;
    x.N = n;
    x.K = n;
    x.c0 = X;
    x.ldc = ld;
    x.flags = DG_K_GE_M | DG_C0_COLMAJOR;
    x.fail = fail;
    launch_dgemm_tn(L, A, B, x, 1, "back_transform");
}

}  // namespace lt
