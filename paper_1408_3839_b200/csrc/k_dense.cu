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
//   k_tridiag_eig  eigenvalues of the tridiagonal (d, e): one warp per eigenvalue, Q shifts
//                  per lane of LDL^T Sturm counts (LAPACK's pivmin guard), the bracket
//                  shrinks 32 Q + 1-fold per round; ascending by construction.
//   k_symmetrize   A = 0.5 (A + A^T) in place (tiles through shared memory).
#include "lt_device.cuh"
#include "lt_internal.cuh"

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

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();  // red reuse
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) s += red[w];
    return s;
}

__device__ __forceinline__ double fast_rcp(double q) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    double t = fma(-q, r, 1.0);
    r = fma(r, t, r);
    t = fma(-q, r, 1.0);
    return fma(r, t, r);
}

}  // namespace

// Householder reflector of x = c[r0 .. n-1] (dlarfg, real): beta, tau, and v (v[r0] = 1) in
// sv; all threads get beta / tau. c, sv in shared memory.
template <int NT>
__device__ __forceinline__ void reflector(const double* c, double* sv, int r0, int n, double* red, double& beta,
                                          double& tau) {
    double s = 0.0;
    for (int i = r0 + 1 + threadIdx.x; i < n; i += NT) s += c[i] * c[i];
    const double sigma = block_sum<NT>(s, red);
    const double a0 = c[r0];
    double scal;
    if (sigma == 0.0) {
        tau = 0.0;
        beta = a0;
        scal = 0.0;
    } else {
        const double nrm = sqrt(a0 * a0 + sigma);
        beta = a0 >= 0.0 ? -nrm : nrm;
        tau = (beta - a0) / beta;
        scal = 1.0 / (a0 - beta);
    }
    for (int i = r0 + threadIdx.x; i < n; i += NT) sv[i] = (i == r0) ? 1.0 : c[i] * scal;
    __syncthreads();
}

// smem: A[cols][n] (own columns, j = blockIdx.x + s P), v[n], w[n], c[n], red[NT/32]
template <int NT>
__global__ void __launch_bounds__(NT) k_sytrd(int n, int P, int cols, const double* __restrict__ C, double* d,
                                              double* e, double* pbuf, double* cbuf, unsigned* bar) {
    extern __shared__ __align__(16) double sm[];
    double* A = sm;
    double* sv = A + static_cast<size_t>(cols) * n;
    double* sw = sv + n;
    double* sc = sw + n;
    __shared__ double red[NT / 32];
    const int b = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ncol = (n - b + P - 1) / P;  // own columns: j = b + s P, s < ncol
    for (int s = 0; s < ncol; ++s) {
        const double* src = C + static_cast<size_t>(b + s * P) * n;
        for (int i = threadIdx.x; i < n; i += NT) A[static_cast<size_t>(s) * n + i] = src[i];
    }
    // column 0 from the input, redundantly: d_0 and the first reflector
    for (int i = threadIdx.x; i < n; i += NT) sc[i] = C[i];
    __syncthreads();
    double beta = 0.0, tau = 0.0;
    if (b == 0 && threadIdx.x == 0) d[0] = sc[0];
    if (n > 1) {
        reflector<NT>(sc, sv, 1, n, red, beta, tau);
        if (b == 0 && threadIdx.x == 0) e[0] = beta;
    }
    for (int k = 0; k + 1 < n; ++k) {
        const int r0 = k + 1;  // trailing rows / columns r0 .. n-1
        double* pb = pbuf + static_cast<size_t>(k & 1) * n;
        double* cb = cbuf + static_cast<size_t>(k & 1) * n;
        // phase 1: p_j = sum_i A[i][j] v_i for own columns j >= r0 (warp per column)
        const int s0 = (r0 - b + P - 1) / P > 0 ? (r0 - b + P - 1) / P : 0;  // first own column >= r0
        for (int s = s0 + warp; s < ncol; s += NT / 32) {
            const double* col = A + static_cast<size_t>(s) * n;
            double acc = 0.0;
            if (tau != 0.0)
                for (int i = r0 + lane; i < n; i += 32) acc = fma(col[i], sv[i], acc);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) pb[b + s * P] = acc;
        }
        if (r0 % P == b) {  // owner of column r0 publishes it (rows r0 ..)
            const double* col = A + static_cast<size_t>(r0 / P) * n;
            for (int i = r0 + threadIdx.x; i < n; i += NT) cb[i] = col[i];
        }
        grid_sync(bar, static_cast<unsigned>(k + 1) * static_cast<unsigned>(P));
        // phase 2: w = tau p - tau^2 / 2 (v.p) v
        double part = 0.0;
        for (int i = r0 + threadIdx.x; i < n; i += NT) {
            const double p = __ldcg(pb + i);
            sw[i] = p;
            part = fma(sv[i], p, part);
            sc[i] = __ldcg(cb + i);
        }
        const double vp = block_sum<NT>(part, red);
        const double half = 0.5 * tau * tau * vp;
        for (int i = r0 + threadIdx.x; i < n; i += NT) sw[i] = tau * sw[i] - half * sv[i];
        __syncthreads();
        // phase 3: own columns j > r0 (column r0 is rebuilt from cb below): A -= v w^T + w v^T
        if (tau != 0.0) {
            const int s1 = (r0 + 1 - b + P - 1) / P > 0 ? (r0 + 1 - b + P - 1) / P : 0;
            for (int s = s1; s < ncol; ++s) {
                const int j = b + s * P;
                const double wj = sw[j], vj = sv[j];
                double* col = A + static_cast<size_t>(s) * n;
                for (int i = r0 + threadIdx.x; i < n; i += NT) col[i] -= fma(sv[i], wj, sw[i] * vj);
            }
        }
        // phase 4: column r0 of the updated matrix, d_{r0}, the next reflector
        const double w0 = sw[r0];  // v_{r0} = 1
        for (int i = r0 + threadIdx.x; i < n; i += NT) sc[i] -= fma(sv[i], w0, sw[i]);
        __syncthreads();
        if (b == 0 && threadIdx.x == 0) d[r0] = sc[r0];
        if (r0 + 1 < n) {
            reflector<NT>(sc, sv, r0 + 1, n, red, beta, tau);
            if (b == 0 && threadIdx.x == 0) e[r0] = beta;
        }
    }
}

// one warp per eigenvalue index; multisection with Q shifts per lane
template <int Q>
__global__ void __launch_bounds__(256) k_tridiag_eig(int n, const double* __restrict__ d, const double* __restrict__ e,
                                                     double* __restrict__ eig) {
    extern __shared__ __align__(16) double ts[];
    double* sd = ts;
    double* se2 = ts + n;
    __shared__ double red[8][3];
    double lo = 1e300, hi = -1e300, emax = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double di = d[i];
        const double ei = i + 1 < n ? e[i] : 0.0;
        sd[i] = di;
        se2[i] = ei * ei;
        const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + fabs(ei);
        lo = fmin(lo, di - r);
        hi = fmax(hi, di + r);
        emax = fmax(emax, ei * ei);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, o));
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        red[warp][0] = lo;
        red[warp][1] = hi;
        red[warp][2] = emax;
    }
    __syncthreads();
    lo = red[0][0];
    hi = red[0][1];
    emax = red[0][2];
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) {
        lo = fmin(lo, red[w][0]);
        hi = fmax(hi, red[w][1]);
        emax = fmax(emax, red[w][2]);
    }
    const double wid = fmax(hi - lo, fmax(fabs(lo), fabs(hi))) * 4.4e-16 * n + 1e-300;
    lo -= wid;
    hi += wid;
    const double pivmin = 2.2250738585072014e-308 * fmax(1.0, emax);
    const double atol = 2.2e-16 * fmax(fabs(lo), fabs(hi));
    const int mi = blockIdx.x * (blockDim.x >> 5) + warp;
    if (mi >= n) return;
    double a = lo, bnd = hi;
    const double inv_pts = 1.0 / static_cast<double>(32 * Q + 1);
    for (int it = 0; it < 80; ++it) {
        double x[Q], q[Q];
        int cnt[Q];
#pragma unroll
        for (int j = 0; j < Q; ++j) {
            x[j] = a + (bnd - a) * (static_cast<double>(lane * Q + j + 1) * inv_pts);
            q[j] = sd[0] - x[j];
            if (fabs(q[j]) < pivmin) q[j] = -pivmin;
            cnt[j] = q[j] < 0.0;
        }
        for (int i = 1; i < n; ++i) {
            const double di = sd[i], ei = se2[i - 1];
#pragma unroll
            for (int j = 0; j < Q; ++j) {
                q[j] = (di - x[j]) - ei * fast_rcp(q[j]);
                if (fabs(q[j]) < pivmin) q[j] = -pivmin;
                cnt[j] += q[j] < 0.0;
            }
        }
        // first shift (lane-major order) whose count exceeds mi
        int fq = Q;
#pragma unroll
        for (int j = Q - 1; j >= 0; --j)
            if (cnt[j] > mi) fq = j;
        const double prev_last = __shfl_up_sync(0xffffffffu, x[Q - 1], 1);
        double clo = lane > 0 ? prev_last : a, chi = x[0];
#pragma unroll
        for (int j = 1; j < Q; ++j)
            if (fq == j) {
                clo = x[j - 1];
                chi = x[j];
            }
        const unsigned bal = __ballot_sync(0xffffffffu, fq < Q);
        double na, nb;
        if (bal) {
            const int src = __ffs(bal) - 1;
            na = __shfl_sync(0xffffffffu, clo, src);
            nb = __shfl_sync(0xffffffffu, chi, src);
        } else {
            na = __shfl_sync(0xffffffffu, x[Q - 1], 31);
            nb = bnd;
        }
        const bool done = !(nb - na > 2.2e-16 * fmax(fabs(na), fabs(nb)) + atol) || (na == a && nb == bnd);
        a = na;
        bnd = nb;
        if (done) break;
    }
    if (lane == 0) eig[mi] = 0.5 * (a + bnd);
}

// A = 0.5 (A + A^T) in place: CTA per tile pair (bi >= bj), 32 x 32 tiles
__global__ void k_symmetrize(int n, double* A) {
    __shared__ double t1[32][33], t2[32][33];
    const int bi = blockIdx.x, bj = blockIdx.y;
    if (bi < bj) return;
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    for (int r = ty; r < 32; r += 8) {
        const int i1 = bi * 32 + tx, j1 = bj * 32 + r;  // tile (bi, bj), column j1
        const int i2 = bj * 32 + tx, j2 = bi * 32 + r;  // tile (bj, bi)
        t1[r][tx] = (i1 < n && j1 < n) ? A[static_cast<size_t>(j1) * n + i1] : 0.0;
        t2[r][tx] = (i2 < n && j2 < n) ? A[static_cast<size_t>(j2) * n + i2] : 0.0;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const int i1 = bi * 32 + tx, j1 = bj * 32 + r;
        const int i2 = bj * 32 + tx, j2 = bi * 32 + r;
        // (i1, j1) pairs with (j1, i1) = tile (bj, bi) entry [row j1 - bj*32][col i1 - bi*32]
        const double s1 = 0.5 * (t1[r][tx] + t2[tx][r]);
        const double s2 = 0.5 * (t2[r][tx] + t1[tx][r]);
        if (i1 < n && j1 < n) A[static_cast<size_t>(j1) * n + i1] = s1;
        if (i2 < n && j2 < n) A[static_cast<size_t>(j2) * n + i2] = s2;
    }
}

static size_t sytrd_smem(int n, int cols) { return sizeof(double) * (static_cast<size_t>(cols) * n + 3 * n); }

int sytrd_ctas(int n) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int P = std::min(n, sms);
    const int cols = (n + P - 1) / P;
    return sytrd_smem(n, cols) <= 227 * 1024 - 1024 ? P : 0;
}

void launch_sytrd(const Launch& L, int n, const double* C, double* d, double* e, double* work, unsigned* bar) {
    constexpr int NT = 256;
    const int P = sytrd_ctas(n);
    if (P == 0) fail(LT_EGENERIC, "sytrd: matrix too large for the shared-memory resident reduction");
    const int cols = (n + P - 1) / P;
    const size_t smem = sytrd_smem(n, cols);
    LT_CU(cudaFuncSetAttribute(k_sytrd<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    LT_CU(cudaMemsetAsync(bar, 0, sizeof(unsigned), L.st));
    double* pbuf = work;
    double* cbuf = work + 2 * static_cast<size_t>(n);
    int nn = n, PP = P, cc = cols;
    void* args[] = {&nn, &PP, &cc, &C, &d, &e, &pbuf, &cbuf, &bar};
    Stage st_(L, "sytrd");
    LT_CU(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_sytrd<NT>), dim3(P), dim3(NT), args, smem, L.st));
    L.tick();
}

void launch_tridiag_eig(const Launch& L, int n, const double* d, const double* e, double* eig) {
    const size_t smem = sizeof(double) * 2 * static_cast<size_t>(n);
    LT_CU(cudaFuncSetAttribute(k_tridiag_eig<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    Stage st_(L, "tridiag_eig");
    k_tridiag_eig<4><<<static_cast<unsigned>((n + 7) / 8), 256, smem, L.st>>>(n, d, e, eig);
    LT_CU(cudaGetLastError());
    L.tick();
}

void launch_symmetrize(const Launch& L, int n, double* A) {
    const unsigned t = static_cast<unsigned>((n + 31) / 32);
    Stage st_(L, "symmetrize");
    k_symmetrize<<<dim3(t, t), dim3(32, 8), 0, L.st>>>(n, A);
    LT_CU(cudaGetLastError());
    L.tick();
}

}  // namespace lt
