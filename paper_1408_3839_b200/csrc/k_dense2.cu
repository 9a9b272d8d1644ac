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

// Cholesky + inverse of diagonal block j (rows/cols b0 .. b0 + m) of the row-major S, in
// shared memory, blocked by 8 columns (8 steps of three barriers instead of 64 of one):
//   A. one warp factors the 8 x 8 diagonal block (lane per row, shuffles; Eigen's pivot
//      test x <= 0 -> not positive definite) and inverts it;
//   B. the panel below: L_r = A_r D^-T;
//   C. the trailing lower part: A_rc -= sum_t L_rt L_ct (t in the block).
// Then X = L^-1 by blocked column elimination: X_b <- D_b^-1 X_b, X_r -= L_rb X_b (r below).
constexpr int kLB = 8;

#ifdef LT_LEAF_PROFILE
__device__ long long lt_leaf_prof[64];
#define LPROF(i) \
    if (threadIdx.x == 0) lt_leaf_prof[i] = clock64();
#else
#define LPROF(i)
#endif

// one thread: Cholesky of the mb x mb (mb <= 8) diagonal block at (c0, c0) in registers, its
// inverse, both written back (factor into sA's lower part, inverse into sD)
__device__ __forceinline__ void leaf_chol8(double (*sA)[65], double (*sD)[9], int c0, int mb,
                                           unsigned long long* fail, int* bad) {
    double a[kLB][kLB];
#pragma unroll
    for (int r = 0; r < kLB; ++r)
#pragma unroll
        for (int c = 0; c < kLB; ++c) a[r][c] = (r < mb && c <= r) ? sA[c0 + r][c0 + c] : (r == c ? 1.0 : 0.0);
    int ok = 1;
    double rd[kLB];
#pragma unroll
    for (int t = 0; t < kLB; ++t) {
        const double x = a[t][t];
        if (t < mb && !(x > 0.0)) ok = 0;
        const double is = leaf_rsqrt(x);
        rd[t] = is;
        a[t][t] = x * is;  // sqrt(x)
#pragma unroll
        for (int r = t + 1; r < kLB; ++r) a[r][t] *= is;
#pragma unroll
        for (int c = t + 1; c < kLB; ++c)
#pragma unroll
            for (int r = c; r < kLB; ++r) a[r][c] = fma(-a[r][t], a[c][t], a[r][c]);
    }
    // X = L^-1 by forward substitution (1 / L_rr = rd[r])
    double x[kLB][kLB];
#pragma unroll
    for (int c = 0; c < kLB; ++c)
#pragma unroll
        for (int r = 0; r < kLB; ++r) {
            if (r < c) {
                x[r][c] = 0.0;
                continue;
            }
            double acc = r == c ? 1.0 : 0.0;
#pragma unroll
            for (int k = c; k < r; ++k) acc = fma(-a[r][k], x[k][c], acc);
            x[r][c] = acc * rd[r];
        }
    if (!ok) {
        atomicMin(fail, 2ull);
        *bad = 1;
    }
#pragma unroll
    for (int r = 0; r < kLB; ++r)
#pragma unroll
        for (int c = 0; c < kLB; ++c) {
            if (r < mb && c <= r) sA[c0 + r][c0 + c] = a[r][c];
            sD[r][c] = (c <= r) ? x[r][c] : 0.0;
        }
}

__global__ void __launch_bounds__(256) k_potf_leaf(int n, long long ld, double* __restrict__ S, double* __restrict__ Li,
                                                   double* __restrict__ Lic, int j, unsigned long long* fail) {
    extern __shared__ double leaf_smem[];
    double(*sA)[65] = reinterpret_cast<double(*)[65]>(leaf_smem);            // the block: lower part -> L
    double(*sX)[65] = reinterpret_cast<double(*)[65]>(leaf_smem + 64 * 65);  // X = L^-1
    double(*sDall)[kLB][9] = reinterpret_cast<double(*)[kLB][9]>(leaf_smem + 2 * 64 * 65);  // 8 x 8 inverses
    __shared__ int bad;
    if (*fail != ~0ull) return;
    const int b0 = j * kLeaf, m = min(kLeaf, n - b0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int idx = tid; idx < 64 * 64; idx += 256) {
        const int r = idx >> 6, c = idx & 63;
        sA[r][c] = (r < m && c <= r) ? S[static_cast<long long>(b0 + r) * ld + b0 + c] : 0.0;
        sX[r][c] = (r == c && r < m) ? 1.0 : 0.0;
    }
    if (tid == 0) bad = 0;
    __syncthreads();
    LPROF(0);
    const int nb = (m + kLB - 1) / kLB;
    for (int kb = 0; kb < nb; ++kb) {
        const int c0 = kb * kLB, mb = min(kLB, m - c0), r1 = c0 + mb;
        double (*sD)[9] = sDall[kb];
        LPROF(1 + 4 * kb);
        if (tid == 0) leaf_chol8(sA, sD, c0, mb, fail, &bad);
        __syncthreads();
        LPROF(2 + 4 * kb);
        if (bad) return;
        // B: panel rows r >= r1: L_r,. = A_r,. D^-T (8 columns of the block); results held in
        // registers until every thread has read the block's rows
        double pv[2] = {0.0, 0.0};
        int cnt = 0;
        for (int idx = tid; idx < (m - r1) * kLB; idx += 256, ++cnt) {
            const int r = r1 + idx / kLB, c = idx % kLB;
            double acc = 0.0;
#pragma unroll
            for (int t = 0; t < kLB; ++t)
                if (t <= c && c < mb) acc = fma(sA[r][c0 + t], sD[c][t], acc);
            pv[cnt] = acc;
        }
        __syncthreads();
        cnt = 0;
        for (int idx = tid; idx < (m - r1) * kLB; idx += 256, ++cnt) {
            const int r = r1 + idx / kLB, c = idx % kLB;
            sA[r][c0 + c] = pv[cnt];
        }
        __syncthreads();
        // C: trailing lower part A_rc -= sum_t L_rt L_ct, r >= c >= r1
        {
            const int ty = tid >> 4, tx = tid & 15;  // 16 x 16 threads over the trailing square
            double lc[4][kLB];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int c = r1 + tx + 16 * v;
#pragma unroll
                for (int t = 0; t < kLB; ++t) lc[v][t] = c < m ? sA[c][c0 + t] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int r = r1 + ty + 16 * u;
                if (r >= m) break;
                double lr[kLB];
#pragma unroll
                for (int t = 0; t < kLB; ++t) lr[t] = sA[r][c0 + t];
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const int c = r1 + tx + 16 * v;
                    if (c > r) continue;
                    double acc = sA[r][c];
#pragma unroll
                    for (int t = 0; t < kLB; ++t) acc = fma(-lr[t], lc[v][t], acc);
                    sA[r][c] = acc;
                }
            }
        }
        __syncthreads();
        LPROF(3 + 4 * kb);
    }
    LPROF(40);
    // X = L^-1: for each 8-block b: X_b <- D_b^-1 X_b (rows of block b), then X_r -= L_rb X_b
    for (int kb = 0; kb < nb; ++kb) {
        const int c0 = kb * kLB, mb = min(kLB, m - c0), r1 = c0 + mb;
        const double (*sD)[9] = sDall[kb];
        // rows of block b: X_b,c = sum_t Dinv[r][t] X_{c0+t},c  (c <= r: columns up to r1)
        double xb[2] = {0.0, 0.0};
        int cnt = 0;
        for (int idx = tid; idx < mb * r1; idx += 256, ++cnt) {
            const int r = idx / r1, c = idx % r1;
            double acc = 0.0;
#pragma unroll
            for (int t = 0; t < kLB; ++t)
                if (t <= r) acc = fma(sD[r][t], sX[c0 + t][c], acc);
            xb[cnt] = acc;
        }
        __syncthreads();
        cnt = 0;
        for (int idx = tid; idx < mb * r1; idx += 256, ++cnt) {
            const int r = idx / r1, c = idx % r1;
            sX[c0 + r][c] = xb[cnt];
        }
        __syncthreads();
        // rows below: X_r,c -= sum_t L[r][c0+t] X[c0+t][c]
        const int rows = m - r1;
        for (int idx = tid; idx < rows * r1; idx += 256) {
            const int r = r1 + idx / r1, c = idx % r1;
            double acc = sX[r][c];
#pragma unroll
            for (int t = 0; t < kLB; ++t)
                if (t < mb) acc = fma(-sA[r][c0 + t], sX[c0 + t][c], acc);
            sX[r][c] = acc;
        }
        __syncthreads();
    }
    LPROF(41);
    for (int idx = tid; idx < 64 * 64; idx += 256) {
        const int r = idx >> 6, c = idx & 63;  // consecutive threads: consecutive columns (row-major)
        if (r < m && c < m) {
            Li[static_cast<long long>(b0 + r) * ld + b0 + c] = r >= c ? sX[r][c] : 0.0;
            if (c <= r) S[static_cast<long long>(b0 + r) * ld + b0 + c] = sA[r][c];
        }
        const int cc = idx >> 6, rr = idx & 63;  // column-major: consecutive rows
        if (rr < m && cc < m) Lic[static_cast<long long>(b0 + cc) * ld + b0 + rr] = rr >= cc ? sX[rr][cc] : 0.0;
    }
}

static void launch_potf_leaf(const Launch& L, int n, long long ld, double* S, double* Li, double* Lic, int j,
                             unsigned long long* fail) {
    const int smem = static_cast<int>(sizeof(double) * (2 * 64 * 65 + (kLeaf / kLB) * kLB * 9));
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
