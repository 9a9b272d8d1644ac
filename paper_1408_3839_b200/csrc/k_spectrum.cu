// k_spectrum.cu — block diagonalisation over lattice indices and batched pencil eigensolves.
//
//   launch_scatter_gen / launch_dft_axis
//       bc_block_diagonalize + fft_levels (block_circulant.cpp:82-112, :184-196):
//       unnormalised forward DFT, omega = exp(-2 pi i / L), axis 0 then 1 then 2, for every
//       block entry. Only the stored generating blocks are non-zero, so each axis is a
//       sparse DFT from the compressed set of stored kidx values to all L frequencies
//       (exact same sum as the zero-padded FFT; K = (2b+1) terms per output instead of
//       log L butterflies over mostly zeros).
//   launch_pencil
//       solve_pencil (eigensolver.cpp:72-93): Hermitian check at 1e-10 max(1, max|.|),
//       symmetrise, Cholesky of S, A = L^-1 H L^-H, symmetrise, eigenvalues ascending.
//       One warp per k-point, matrices in shared memory, parallel (round-robin) cyclic
//       complex Jacobi. The first failing k-point (in k order) is reported with its kind.
#include "lt_device.cuh"
#include "lt_internal.cuh"

namespace lt {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double s, double2 a) { return make_double2(s * a.x, s * a.y); }
__device__ __forceinline__ double cabs2(double2 a) { return a.x * a.x + a.y * a.y; }
__device__ __forceinline__ double cabs_(double2 a) { return hypot(a.x, a.y); }

// ---------------------------------------------------------------------------
// DFT over lattice indices
// ---------------------------------------------------------------------------
__global__ void k_scatter_gen(Index nblk, Index mm, const int64_t* __restrict__ kslot, const double* __restrict__ blocks,
                              double2* __restrict__ dense) {
    const Index idx = static_cast<Index>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= nblk * mm) return;
    const Index b = idx / mm, e = idx % mm;
    dense[kslot[b] * mm + e] = make_double2(blocks[idx], 0.0);
}

void launch_scatter_gen(const Launch& L, Index nblk, Index mm, const int64_t* kslot_dev, const double* blocks,
                        double2* dense) {
    const Index tot = nblk * mm;
    if (tot == 0) return;
    Stage st_(L, "scatter_gen");
    k_scatter_gen<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, L.st>>>(nblk, mm, kslot_dev, blocks, dense);
    LT_CU(cudaGetLastError());
    L.tick();
}

__global__ void k_twiddles(Index Lax, Index ncomp, const int64_t* __restrict__ comp, double2* __restrict__ tw) {
    const Index idx = static_cast<Index>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= Lax * ncomp) return;
    const Index j = idx / ncomp, c = idx % ncomp;
    const Index m = (j * comp[c]) % Lax;
    double s, co;
    sincospi(-2.0 * static_cast<double>(m) / static_cast<double>(Lax), &s, &co);
    tw[idx] = make_double2(co, s);
}

void launch_twiddles(const Launch& L, Index Lax, Index ncomp, const int64_t* comp_dev, double2* tw) {
    const Index tot = Lax * ncomp;
    Stage st_(L, "twiddles");
    k_twiddles<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, L.st>>>(Lax, ncomp, comp_dev, tw);
    LT_CU(cudaGetLastError());
    L.tick();
}

struct Ext3 {
    Index in[3], out[3];
};

__global__ void k_dft_axis(int axis, Ext3 x, Index mm, const double2* __restrict__ in, double2* __restrict__ out,
                           const double2* __restrict__ tw, Index ncomp) {
    const Index total = x.out[0] * x.out[1] * x.out[2] * mm;
    const Index idx = static_cast<Index>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= total) return;
    const Index e = idx % mm;
    Index pos = idx / mm;
    Index o[3];
    o[2] = pos % x.out[2];
    pos /= x.out[2];
    o[1] = pos % x.out[1];
    o[0] = pos / x.out[1];
    const Index j = o[axis];
    Index stride = mm;
    for (int l = 2; l > axis; --l) stride *= x.in[l];
    Index base = 0;
    for (int l = 0; l < 3; ++l) base = base * x.in[l] + (l == axis ? 0 : o[l]);
    base = base * mm + e;
    double2 acc = make_double2(0.0, 0.0);
    const double2* t = tw + j * ncomp;
    for (Index c = 0; c < ncomp; ++c) acc = cadd(acc, cmul(t[c], in[base + c * stride]));
    out[idx] = acc;
}

void launch_dft_axis(const Launch& L, int axis, const Index* in_ext, const Index* out_ext, Index mm, const double2* in,
                     double2* out, const double2* tw, Index ncomp, Index /*Lax*/) {
    Ext3 x;
    for (int l = 0; l < 3; ++l) {
        x.in[l] = in_ext[l];
        x.out[l] = out_ext[l];
    }
    const Index tot = out_ext[0] * out_ext[1] * out_ext[2] * mm;
    Stage st_(L, "dft_axis");
    k_dft_axis<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, L.st>>>(axis, x, mm, in, out, tw, ncomp);
    LT_CU(cudaGetLastError());
    L.tick();
}

// ---------------------------------------------------------------------------
// batched pencils: one warp per pencil
// ---------------------------------------------------------------------------
template <int NM>
struct PencilSmem {
    double2 A[NM][NM + 1];
    double2 B[NM][NM + 1];
    double cpar[NM / 2 + 1];
    double spar[NM / 2 + 1];
    double2 ppar[NM / 2 + 1];
    double dp[NM / 2 + 1];
    double dq[NM / 2 + 1];
    int flag[NM / 2 + 1];
};

template <int NM, int WPC>
__global__ void __launch_bounds__(32 * WPC) k_pencil(Index count, int m0, const double2* __restrict__ Hb,
                                                     const double2* __restrict__ Sb, double* __restrict__ eig,
                                                     unsigned long long* fail_key, int periodic_checks) {
    __shared__ PencilSmem<NM> sm_all[WPC];
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const Index k = static_cast<Index>(blockIdx.x) * WPC + w;
    if (k >= count) return;
    PencilSmem<NM>& sm = sm_all[w];
    auto& A = sm.A;
    auto& B = sm.B;
    const int mm = m0 * m0;
    for (int idx = lane; idx < mm; idx += 32) {
        const int r = idx % m0, c = idx / m0;
        A[r][c] = Hb[k * mm + idx];
        B[r][c] = Sb[k * mm + idx];
    }
    __syncwarp();
    int code = 0;
    if (periodic_checks) {
        double hmax = 0.0, smax = 0.0, hdev = 0.0, sdev = 0.0;
        for (int idx = lane; idx < mm; idx += 32) {
            const int r = idx % m0, c = idx / m0;
            hmax = fmax(hmax, cabs_(A[r][c]));
            smax = fmax(smax, cabs_(B[r][c]));
            hdev = fmax(hdev, cabs_(csub(A[r][c], cconj(A[c][r]))));
            sdev = fmax(sdev, cabs_(csub(B[r][c], cconj(B[c][r]))));
        }
        hmax = __shfl_sync(0xffffffffu, warp_max(hmax), 0);
        smax = __shfl_sync(0xffffffffu, warp_max(smax), 0);
        hdev = __shfl_sync(0xffffffffu, warp_max(hdev), 0);
        sdev = __shfl_sync(0xffffffffu, warp_max(sdev), 0);
        if (hdev > 1e-10 * fmax(1.0, hmax) || sdev > 1e-10 * fmax(1.0, smax)) code = 1;
        __syncwarp();
        // H <- (H + H^H)/2, S <- (S + S^H)/2
        for (int idx = lane; idx < mm; idx += 32) {
            const int r = idx % m0, c = idx / m0;
            if (r > c) continue;
            const double2 va = cscale(0.5, cadd(A[r][c], cconj(A[c][r])));
            const double2 vb = cscale(0.5, cadd(B[r][c], cconj(B[c][r])));
            A[r][c] = va;
            A[c][r] = cconj(va);
            B[r][c] = vb;
            B[c][r] = cconj(vb);
        }
        __syncwarp();
    }
    // left-looking Cholesky of B (lower triangle), lane i owns row i
    if (code == 0) {
        for (int kk = 0; kk < m0; ++kk) {
            double x = B[kk][kk].x;
            for (int j = 0; j < kk; ++j) x -= cabs2(B[kk][j]);
            if (!(x > 0.0)) {
                code = 2;
                break;
            }
            const double dkk = sqrt(x);
            __syncwarp();
            for (int i = kk + 1 + lane; i < m0; i += 32) {
                double2 s = B[i][kk];
                for (int j = 0; j < kk; ++j) s = csub(s, cmul(B[i][j], cconj(B[kk][j])));
                B[i][kk] = cscale(1.0 / dkk, s);
            }
            if (lane == 0) B[kk][kk] = make_double2(dkk, 0.0);
            __syncwarp();
        }
    }
    if (code != 0) {
        if (lane == 0) atomicMin(fail_key, static_cast<unsigned long long>(k) * 4ull + static_cast<unsigned long long>(code));
        return;
    }
    // Y = L^-1 H (lane c owns column c)
    for (int c = lane; c < m0; c += 32) {
        for (int i = 0; i < m0; ++i) {
            double2 s = A[i][c];
            for (int j = 0; j < i; ++j) s = csub(s, cmul(B[i][j], A[j][c]));
            A[i][c] = cscale(1.0 / B[i][i].x, s);
        }
    }
    __syncwarp();
    // A = (L^-1 Y^H)^H (lane c owns row c)
    for (int c = lane; c < m0; c += 32) {
        for (int i = 0; i < m0; ++i) {
            double2 s = cconj(A[c][i]);
            for (int j = 0; j < i; ++j) s = csub(s, cmul(B[i][j], cconj(A[c][j])));
            A[c][i] = cconj(cscale(1.0 / B[i][i].x, s));
        }
    }
    __syncwarp();
    for (int idx = lane; idx < mm; idx += 32) {
        const int r = idx % m0, c = idx / m0;
        if (r > c) continue;
        const double2 v = cscale(0.5, cadd(A[r][c], cconj(A[c][r])));
        A[r][c] = v;
        A[c][r] = cconj(v);
    }
    __syncwarp();
    // parallel cyclic Jacobi (circle-method pairing)
    const int N = (m0 % 2) ? m0 + 1 : m0;
    const int np = N / 2;
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0.0, dg = 0.0;
        for (int idx = lane; idx < mm; idx += 32) {
            const int r = idx % m0, c = idx / m0;
            if (r == c) dg += cabs2(A[r][c]);
            else off += cabs2(A[r][c]);
        }
        off = __shfl_sync(0xffffffffu, warp_sum(off), 0);
        dg = __shfl_sync(0xffffffffu, warp_sum(dg), 0);
        if (off == 0.0 || off <= 1e-32 * (off + dg)) break;
        for (int rd = 0; rd < N - 1; ++rd) {
            if (lane < np) {
                int a, b;
                if (lane == 0) {
                    a = rd;
                    b = N - 1;
                } else {
                    a = (rd + lane) % (N - 1);
                    b = (rd - lane + (N - 1)) % (N - 1);
                }
                const int p = min(a, b), q = max(a, b);
                int fl = 0;
                if (q < m0) {
                    const double2 apq = A[p][q];
                    const double r = cabs_(apq);
                    const double app = A[p][p].x, aqq = A[q][q].x;
                    if (r != 0.0) {
                        if (r <= 1e-18 * sqrt(fabs(app * aqq))) {
                            fl = 2;
                        } else {
                            fl = 1;
                            const double tau = (aqq - app) / (2.0 * r);
                            const double t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                            const double c = 1.0 / sqrt(1.0 + t * t);
                            sm.cpar[lane] = c;
                            sm.spar[lane] = t * c;
                            sm.ppar[lane] = make_double2(apq.x / r, apq.y / r);
                            sm.dp[lane] = app - t * r;
                            sm.dq[lane] = aqq + t * r;
                        }
                    }
                }
                sm.flag[lane] = fl;
            }
            __syncwarp();
            // columns: A <- A (D J)
            for (int task = lane; task < np * m0; task += 32) {
                const int pi = task / m0, kk = task % m0;
                if (sm.flag[pi] != 1) continue;
                int a, b;
                if (pi == 0) {
                    a = rd;
                    b = N - 1;
                } else {
                    a = (rd + pi) % (N - 1);
                    b = (rd - pi + (N - 1)) % (N - 1);
                }
                const int p = min(a, b), q = max(a, b);
                const double c = sm.cpar[pi], s = sm.spar[pi];
                const double2 akp = A[kk][p];
                const double2 akq = cmul(A[kk][q], cconj(sm.ppar[pi]));
                A[kk][p] = csub(cscale(c, akp), cscale(s, akq));
                A[kk][q] = cadd(cscale(s, akp), cscale(c, akq));
            }
            __syncwarp();
            // rows: A <- (D J)^H A
            for (int task = lane; task < np * m0; task += 32) {
                const int pi = task / m0, kk = task % m0;
                if (sm.flag[pi] != 1) continue;
                int a, b;
                if (pi == 0) {
                    a = rd;
                    b = N - 1;
                } else {
                    a = (rd + pi) % (N - 1);
                    b = (rd - pi + (N - 1)) % (N - 1);
                }
                const int p = min(a, b), q = max(a, b);
                const double c = sm.cpar[pi], s = sm.spar[pi];
                const double2 apk = A[p][kk];
                const double2 aqk = cmul(sm.ppar[pi], A[q][kk]);
                A[p][kk] = csub(cscale(c, apk), cscale(s, aqk));
                A[q][kk] = cadd(cscale(s, apk), cscale(c, aqk));
            }
            __syncwarp();
            if (lane < np && sm.flag[lane] != 0) {
                int a, b;
                if (lane == 0) {
                    a = rd;
                    b = N - 1;
                } else {
                    a = (rd + lane) % (N - 1);
                    b = (rd - lane + (N - 1)) % (N - 1);
                }
                const int p = min(a, b), q = max(a, b);
                if (sm.flag[lane] == 1) {
                    // exact post-rotation diagonals from the pre-rotation entries
                    A[p][p] = make_double2(sm.dp[lane], 0.0);
                    A[q][q] = make_double2(sm.dq[lane], 0.0);
                }
                A[p][q] = make_double2(0.0, 0.0);
                A[q][p] = make_double2(0.0, 0.0);
            }
            __syncwarp();
        }
    }
    // ascending sort by rank
    for (int i = lane; i < m0; i += 32) {
        const double wi = A[i][i].x;
        int rank = 0;
        for (int j = 0; j < m0; ++j) {
            const double wj = A[j][j].x;
            rank += (wj < wi || (wj == wi && j < i)) ? 1 : 0;
        }
        eig[k * m0 + rank] = wi;
    }
}

template <int NM, int WPC>
static void run_pencil(const Launch& L, Index count, Index m0, const double2* H, const double2* S, double* eig,
                       unsigned long long* fail_key, bool checks) {
    const Index blocks = (count + WPC - 1) / WPC;
    Stage st_(L, "pencil");
    k_pencil<NM, WPC><<<static_cast<unsigned>(blocks), 32 * WPC, 0, L.st>>>(count, static_cast<int>(m0), H, S, eig,
                                                                             fail_key, checks ? 1 : 0);
    LT_CU(cudaGetLastError());
    L.tick();
}

void launch_pencil(const Launch& L, Index count, Index m0, const double2* H, const double2* S, double* eig,
                   unsigned long long* fail_key, bool periodic_checks) {
    if (count <= 0) return;
    if (m0 <= 8) run_pencil<8, 8>(L, count, m0, H, S, eig, fail_key, periodic_checks);
    else if (m0 <= 16) run_pencil<16, 4>(L, count, m0, H, S, eig, fail_key, periodic_checks);
    else if (m0 <= 32) run_pencil<32, 1>(L, count, m0, H, S, eig, fail_key, periodic_checks);
    else fail(LT_EDIM, "pencil_eig: block size m0 > 32 is not supported on the warp path");
}

}  // namespace lt
