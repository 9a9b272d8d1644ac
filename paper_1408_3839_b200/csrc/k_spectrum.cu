// k_spectrum.cu — block diagonalisation over lattice indices and batched pencil eigensolves.
//
//   launch_dft_axis2
//       bc_block_diagonalize + fft_levels (block_circulant.cpp:82-112, :184-196):
//       unnormalised forward DFT, omega = exp(-2 pi i / L), axis 0 then 1 then 2, for every
//       block entry. Only the stored generating blocks are non-zero, so each axis is a
//       sparse DFT from the compressed set of stored kidx values to all L frequencies
//       (the zero-padded FFT's values from (2b+1) terms per output instead of log L
//       butterflies over mostly zeros).
// The batched pencil eigensolver is in k_pencil.cu.
#include "lt_device.cuh"
#include "lt_internal.cuh"

#include <cmath>

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
// fused axis DFT: one launch per transformed axis for up to two operators (H, S). CTA
// (j, op, chunk): output frequency j along the axis; its twiddles w^(j comp[c] mod L)
// are computed once into shared memory (same sincospi argument as k_twiddles). The
// first axis reads the real generating blocks directly through slot -> block (-1:
// absent block, i.e. zero), so no scatter / memset / twiddle launches remain. The sum
// runs over the compressed indices c in ascending order, as in k_dft_axis.
// ---------------------------------------------------------------------------
__global__ void k_dft_axis2(DftAxisArgs a) {
    extern __shared__ double2 tws[];
    const Index j = blockIdx.x;
    const int op = blockIdx.y;
    for (Index c = threadIdx.x; c < a.ncomp; c += blockDim.x) {
        const Index m = (j * a.comp[c]) % a.Lax;
        double s, co;
        sincospi(-2.0 * static_cast<double>(m) / static_cast<double>(a.Lax), &s, &co);
        tws[c] = make_double2(co, s);
    }
    __syncthreads();
    const Index mm = a.mm;
    const Index o0 = a.out[0], o1 = a.out[1], o2 = a.out[2];
    const Index i1 = a.in[1], i2 = a.in[2];
    const Index others = (o0 * o1 * o2 / (a.axis == 0 ? o0 : (a.axis == 1 ? o1 : o2))) * mm;
    const double* gen = op ? a.gen[1] : a.gen[0];
    const double2* in = op ? a.in_buf[1] : a.in_buf[0];
    double2* out = op ? a.out_buf[1] : a.out_buf[0];
    for (Index q = static_cast<Index>(blockIdx.z) * blockDim.x + threadIdx.x; q < others;
         q += static_cast<Index>(gridDim.z) * blockDim.x) {
        const Index e = q % mm, r = q / mm;
        Index ipos0, istride, opos;  // input position of c = 0, stride per c, output position
        if (a.axis == 0) {
            const Index u = r / o2, w = r % o2;
            ipos0 = u * i2 + w;
            istride = i1 * i2;
            opos = (j * o1 + u) * o2 + w;
        } else if (a.axis == 1) {
            const Index u = r / o2, w = r % o2;
            ipos0 = u * i1 * i2 + w;
            istride = i2;
            opos = (u * o1 + j) * o2 + w;
        } else {
            const Index u = r / o1, w = r % o1;
            ipos0 = (u * i1 + w) * i2;
            istride = 1;
            opos = (u * o1 + w) * o2 + j;
        }
        double2 acc = make_double2(0.0, 0.0);
        if (gen) {
#pragma unroll 4
            for (Index c = 0; c < a.ncomp; ++c) {
                const int b = a.slot2blk[ipos0 + c * istride];
                const double v = b >= 0 ? gen[static_cast<Index>(b) * mm + e] : 0.0;
                acc = cadd(acc, cmul(tws[c], make_double2(v, 0.0)));
            }
        } else {
#pragma unroll 4
            for (Index c = 0; c < a.ncomp; ++c) acc = cadd(acc, cmul(tws[c], in[(ipos0 + c * istride) * mm + e]));
        }
        out[opos * mm + e] = acc;
    }
}

void launch_dft_axis2(const Launch& L, const DftAxisArgs& a, int nops) {
    const Index others = (a.out[0] * a.out[1] * a.out[2] / a.Lax) * a.mm;
    const Index chunks = std::max<Index>(1, std::min<Index>((others + 1023) / 1024, 64));
    dim3 grid(static_cast<unsigned>(a.Lax), nops, static_cast<unsigned>(chunks));
    Stage st_(L, "dft_axis");
    k_dft_axis2<<<grid, 256, sizeof(double2) * a.ncomp, L.st>>>(a);
    LT_CU(cudaGetLastError());
    L.tick();
}

// ---------------------------------------------------------------------------
// Multi-axis lattice DFT in one launch: CTA per (block entry e, operator). The entry's
// compressed generating cube (at most (2b+1)^3 stored offsets) is gathered once into shared
// memory and every wrapped axis is transformed there in turn (same twiddles and the same
// ascending-c accumulation per output as k_dft_axis2); only the last axis writes to global
// memory. The per-axis kernel re-reads its input once per output frequency (L-fold L2
// traffic) and runs one launch per axis; this reads the cube once.
// ---------------------------------------------------------------------------
// One pass along axis AX (n: input extents, updated to the output extents). A thread takes
// (line, chunk of JT outputs): its nc inputs are read once, the twiddles are read as
// broadcasts (chunks vary slowest across threads), and the JT accumulators stay in
// registers. Compile-time AX and scalar extents keep every index in registers (a
// dynamically indexed extent array would live in local memory).
template <int AX>
__device__ __forceinline__ void dft_pass(unsigned& n0, unsigned& n1, unsigned& n2, unsigned L, unsigned nc,
                                         const double2* __restrict__ t, const double2* in, double2* outs,
                                         double2* __restrict__ outg, Index sq, Index oe) {
    constexpr unsigned JT = 8;
    const unsigned o0 = AX == 0 ? L : n0, o1 = AX == 1 ? L : n1, o2 = AX == 2 ? L : n2;
    const unsigned uext = AX == 0 ? n1 : n0, wext = AX == 2 ? n1 : n2;
    const unsigned nlines = uext * wext;
    const unsigned sin_ = AX == 0 ? n1 * n2 : (AX == 1 ? n2 : 1u);
    const unsigned sout = AX == 0 ? o1 * o2 : (AX == 1 ? o2 : 1u);
    const unsigned nch = (L + JT - 1) / JT;
    for (unsigned task = threadIdx.x; task < nlines * nch; task += blockDim.x) {
        const unsigned line = task % nlines, ch = task / nlines;
        const unsigned u = line / wext, w = line % wext;
        unsigned bin, bout;
        if (AX == 0) {
            bin = u * n2 + w;
            bout = u * o2 + w;
        } else if (AX == 1) {
            bin = u * n1 * n2 + w;
            bout = u * o1 * o2 + w;
        } else {
            bin = (u * n1 + w) * n2;
            bout = (u * o1 + w) * o2;
        }
        const unsigned j0 = ch * JT;
        double2 acc[JT];
#pragma unroll
        for (unsigned jj = 0; jj < JT; ++jj) acc[jj] = make_double2(0.0, 0.0);
        for (unsigned c = 0; c < nc; ++c) {
            const double2 x = in[bin + c * sin_];
#pragma unroll
            for (unsigned jj = 0; jj < JT; ++jj)
                if (j0 + jj < L) acc[jj] = cadd(acc[jj], cmul(t[(j0 + jj) * nc + c], x));
        }
#pragma unroll
        for (unsigned jj = 0; jj < JT; ++jj) {
            if (j0 + jj >= L) break;
            const unsigned q = bout + (j0 + jj) * sout;
            if (outg) outg[static_cast<Index>(q) * sq + oe] = acc[jj];
            else outs[q] = acc[jj];
        }
    }
    n0 = o0;
    n1 = o1;
    n2 = o2;
}

// Power-of-two axes (L = 2^LOG <= 16): each line is zero-filled to L points from its
// compressed inputs (cmap: position -> compressed index or -1) and transformed in registers
// by a radix-2 decimation-in-frequency FFT (L/2 log2 L butterflies instead of L nc
// multiply-adds); the output of slot j is X[bitrev(j)]. tw: w^m = e^{-2 pi i m / L}, m < L/2.
template <int AX, int LOG>
__device__ __forceinline__ void fft_pass(unsigned& n0, unsigned& n1, unsigned& n2, const int* __restrict__ cmap,
                                         const double2* __restrict__ tw, const double2* in, double2* outs,
                                         double2* __restrict__ outg, Index sq, Index oe) {
    constexpr unsigned L = 1u << LOG;
    const unsigned o0 = AX == 0 ? L : n0, o1 = AX == 1 ? L : n1, o2 = AX == 2 ? L : n2;
    const unsigned uext = AX == 0 ? n1 : n0, wext = AX == 2 ? n1 : n2;
    const unsigned nlines = uext * wext;
    const unsigned sin_ = AX == 0 ? n1 * n2 : (AX == 1 ? n2 : 1u);
    const unsigned sout = AX == 0 ? o1 * o2 : (AX == 1 ? o2 : 1u);
    double2 w[L / 2];
#pragma unroll
    for (unsigned m = 0; m < L / 2; ++m) w[m] = tw[m];
    for (unsigned line = threadIdx.x; line < nlines; line += blockDim.x) {
        const unsigned u = line / wext, v = line % wext;
        unsigned bin, bout;
        if (AX == 0) {
            bin = u * n2 + v;
            bout = u * o2 + v;
        } else if (AX == 1) {
            bin = u * n1 * n2 + v;
            bout = u * o1 * o2 + v;
        } else {
            bin = (u * n1 + v) * n2;
            bout = (u * o1 + v) * o2;
        }
        double2 x[L];
#pragma unroll
        for (unsigned p = 0; p < L; ++p) {
            const int c = cmap[p];
            x[p] = c >= 0 ? in[bin + static_cast<unsigned>(c) * sin_] : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (unsigned span = L / 2; span >= 1; span >>= 1) {
#pragma unroll
            for (unsigned b = 0; b < L; b += 2 * span)
#pragma unroll
                for (unsigned i = 0; i < span; ++i) {
                    const double2 a = x[b + i], c = x[b + i + span];
                    x[b + i] = cadd(a, c);
                    x[b + i + span] = cmul(csub(a, c), w[i * (L / (2 * span))]);
                }
        }
#pragma unroll
        for (unsigned j = 0; j < L; ++j) {
            unsigned r = 0;
#pragma unroll
            for (int bit = 0; bit < LOG; ++bit) r |= ((j >> bit) & 1u) << (LOG - 1 - bit);
            const unsigned q = bout + j * sout;
            if (outg) outg[static_cast<Index>(q) * sq + oe] = x[r];
            else outs[q] = x[r];
        }
    }
    n0 = o0;
    n1 = o1;
    n2 = o2;
}

__global__ void __launch_bounds__(256) k_dft_fused(DftFusedArgs a) {
    extern __shared__ double2 fsm[];
    const Index e = blockIdx.x;
    const int op = blockIdx.y;
    const Index mm = a.mm;
    // output element (k, e): k-major [K][mm] (q mm + e), or entry-major [mm][K] (e K + q)
    const Index osq = a.emajor ? 1 : mm;
    const Index ooe = a.emajor ? e * (a.dims[0] * a.dims[1] * a.dims[2]) : e;
    // per wrapped axis in pass order: DFT twiddles (L x nc), or for power-of-two L <= 16 the
    // FFT twiddles (L/2) and the position -> compressed-index map (L ints, 8-byte slots);
    // then two cube buffers
    unsigned twoff = 0;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        const Index L = a.dims[ax], nc = a.ncomp[ax];
        if (L == 1) continue;
        if (dft_fft_log(L) > 0) {
            for (Index q = threadIdx.x; q < L / 2; q += blockDim.x) {
                double sn, cs;
                sincospi(-2.0 * static_cast<double>(q) / static_cast<double>(L), &sn, &cs);
                fsm[twoff + q] = make_double2(cs, sn);
            }
            int* cm = reinterpret_cast<int*>(fsm + twoff + L / 2);
            for (Index q = threadIdx.x; q < L; q += blockDim.x) cm[q] = -1;
            __syncthreads();
            for (Index c = threadIdx.x; c < nc; c += blockDim.x) cm[a.comp[ax][c]] = static_cast<int>(c);
            twoff += static_cast<unsigned>(L / 2 + L);
        } else {
            for (Index q = threadIdx.x; q < L * nc; q += blockDim.x) {
                const Index j = q / nc, c = q % nc;
                const Index m = (j * a.comp[ax][c]) % L;
                double sn, cs;
                sincospi(-2.0 * static_cast<double>(m) / static_cast<double>(L), &sn, &cs);
                fsm[twoff + q] = make_double2(cs, sn);
            }
            twoff += static_cast<unsigned>(L * nc);
        }
    }
    double2* buf0 = fsm + twoff;
    double2* buf1 = buf0 + a.maxsz;
    const double* gen = a.gen[op];
    const unsigned ncube = static_cast<unsigned>(a.ext[0] * a.ext[1] * a.ext[2]);
    if (a.ident && a.gen_emajor) {
        // every cube position stored, in order, entry-major: the entry's cube is one contiguous
        // row; eight independent loads in flight per thread (one or two round trips in all)
        const double* row = gen + e * a.nblocks;
        constexpr unsigned U = 8;
        for (unsigned q0 = threadIdx.x; q0 < ncube; q0 += U * blockDim.x) {
            double v[U];
#pragma unroll
            for (unsigned u = 0; u < U; ++u) {
                const unsigned q = q0 + u * blockDim.x;
                v[u] = q < ncube ? row[q] : 0.0;
            }
#pragma unroll
            for (unsigned u = 0; u < U; ++u) {
                const unsigned q = q0 + u * blockDim.x;
                if (q < ncube) buf0[q] = make_double2(v[u], 0.0);
            }
        }
    } else {
        // gather the entry's stored values: block indices first, then the values, four
        // independent loads in flight per thread
        constexpr unsigned U = 4;
        for (unsigned q0 = threadIdx.x; q0 < ncube; q0 += U * blockDim.x) {
            int bi[U];
#pragma unroll
            for (unsigned u = 0; u < U; ++u) {
                const unsigned q = q0 + u * blockDim.x;
                bi[u] = q < ncube ? a.slot2blk[q] : -1;
            }
            double v[U];
#pragma unroll
            for (unsigned u = 0; u < U; ++u)
                v[u] = bi[u] >= 0 ? gen[a.gen_emajor ? e * a.nblocks + bi[u] : static_cast<Index>(bi[u]) * mm + e] : 0.0;
#pragma unroll
            for (unsigned u = 0; u < U; ++u) {
                const unsigned q = q0 + u * blockDim.x;
                if (q < ncube) buf0[q] = make_double2(v[u], 0.0);
            }
        }
    }
    __syncthreads();
    unsigned n0 = static_cast<unsigned>(a.ext[0]), n1 = static_cast<unsigned>(a.ext[1]),
             n2 = static_cast<unsigned>(a.ext[2]);
    const double2* t = fsm;
    double2* cur = buf0;
    double2* nxt = buf1;
    int done = 0;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        const unsigned L = static_cast<unsigned>(a.dims[ax]), nc = static_cast<unsigned>(a.ncomp[ax]);
        if (L == 1) continue;
        ++done;
        double2* og = done == a.nax ? a.out[op] : nullptr;
        const int lg = dft_fft_log(L);
        if (lg > 0) {
            const int* cm = reinterpret_cast<const int*>(t + L / 2);
#define LT_FFT_CASE(LG)                                                                            \
    case LG:                                                                                       \
        if (ax == 0) fft_pass<0, LG>(n0, n1, n2, cm, t, cur, nxt, og, osq, ooe);                      \
        else if (ax == 1) fft_pass<1, LG>(n0, n1, n2, cm, t, cur, nxt, og, osq, ooe);                 \
        else fft_pass<2, LG>(n0, n1, n2, cm, t, cur, nxt, og, osq, ooe);                              \
        break;
            switch (lg) {
                LT_FFT_CASE(1)
                LT_FFT_CASE(2)
                LT_FFT_CASE(3)
                LT_FFT_CASE(4)
            }
#undef LT_FFT_CASE
            t += L / 2 + L;
        } else {
            if (ax == 0) dft_pass<0>(n0, n1, n2, L, nc, t, cur, nxt, og, osq, ooe);
            else if (ax == 1) dft_pass<1>(n0, n1, n2, L, nc, t, cur, nxt, og, osq, ooe);
            else dft_pass<2>(n0, n1, n2, L, nc, t, cur, nxt, og, osq, ooe);
            t += L * nc;
        }
        double2* tmp = cur;
        cur = nxt;
        nxt = tmp;
        __syncthreads();
    }
}

size_t dft_fused_smem(const DftFusedArgs& a) {
    size_t tw = 0;
    for (int i = 0; i < a.nax; ++i) {
        const Index L = a.dims[a.axes[i]];
        tw += static_cast<size_t>(dft_fft_log(L) > 0 ? L / 2 + L : L * a.ncomp[a.axes[i]]);
    }
    return sizeof(double2) * (tw + 2 * static_cast<size_t>(a.maxsz));
}

void launch_dft_fused(const Launch& L, const DftFusedArgs& a, int nops) {
    const size_t smem = dft_fused_smem(a);
    static size_t attr = 0;
    if (smem > attr) {
        LT_CU(cudaFuncSetAttribute(k_dft_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        attr = smem;
    }
    Stage st_(L, "dft_fused");
    k_dft_fused<<<dim3(static_cast<unsigned>(a.mm), nops), 256, smem, L.st>>>(a);
    LT_CU(cudaGetLastError());
    L.tick();
}

// Full-space eigenvectors (block_circulant.cpp:267-289, eigensolver.cpp:164-175):
// out[(i m0 + r) + col N] = L^-1/2 e^{i phi(i, j)} u_{j,m}[r] for columns col = j m0 + m in
// [c0, c0 + ncols), phi = sum_l 2 pi (i_l j_l) / L_l accumulated as the reference does.
// One thread per output entry, rows fastest (coalesced column writes).
__global__ void k_reconstruct(Index d0, Index d1, Index d2, Index m0, const double2* __restrict__ u, Index c0,
                              Index ncols, double norm, double2* __restrict__ out) {
    const Index N = d0 * d1 * d2 * m0;
    const Index e = static_cast<Index>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= N * ncols) return;
    const Index row = e % N, col = c0 + e / N;
    const Index i = row / m0, r = row % m0, j = col / m0, m = col % m0;
    const Index mi[3] = {i / (d1 * d2), (i / d2) % d1, i % d2};
    const Index jm[3] = {j / (d1 * d2), (j / d2) % d1, j % d2};
    const Index dims[3] = {d0, d1, d2};
    const double two_pi = 6.283185307179586;
    double phase = 0.0;
    for (int l = 0; l < 3; ++l)
        phase += two_pi * static_cast<double>(mi[l] * jm[l]) / static_cast<double>(dims[l]);
    double sn, cs;
    sincos(phase, &sn, &cs);
    const double2 f = make_double2(norm * cs, norm * sn);
    const double2 v = u[j * m0 * m0 + r + m * m0];
    out[e] = make_double2(f.x * v.x - f.y * v.y, f.x * v.y + f.y * v.x);
}

void launch_reconstruct(const Launch& L, const Index* dims, Index m0, const double2* u, Index c0, Index ncols,
                        double2* out) {
    const Index N = dims[0] * dims[1] * dims[2] * m0;
    const Index total = N * ncols;
    if (total <= 0) return;
    double norm = 1.0;
    for (int l = 0; l < 3; ++l) norm *= static_cast<double>(dims[l]);
    norm = 1.0 / std::sqrt(norm);
    Stage st_(L, "reconstruct");
    k_reconstruct<<<static_cast<unsigned>((total + 255) / 256), 256, 0, L.st>>>(dims[0], dims[1], dims[2], m0, u, c0,
                                                                                 ncols, norm, out);
    LT_CU(cudaGetLastError());
    L.tick();
}

}  // namespace lt
