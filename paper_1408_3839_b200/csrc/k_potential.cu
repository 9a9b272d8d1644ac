// k_potential.cu — Newton-kernel master panels and the assembled lattice sum.
//
//   launch_master      newton_kernel.cpp:22-45: f(i,q) = sqrt(pi)/(2 t_q) (erf(t_q x_{i+1}) - erf(t_q x_i))
//                      on the centred cell grid x_i = -n h/2 + i h (grid.hpp:28-38)
//   launch_window_sum  canonical_tensor.cpp:123-164: out[i] = sum_k m[s0 + i + k*step] over the
//                      lattice shifts. Uniform progressions (k_window_sum_staged): a CTA bulk-copies
//                      (cp.async.bulk + mbarrier) the master range its output chunk reads into
//                      shared memory once, then every residue class of the chunk is cut into
//                      segments: the segment head is a direct K-term sum, the rest follows by the
//                      reference's recurrence out[i] = out[i-step] + m[s0+i+(K-1)step] - m[s0+i-step]
//                      (restarted every segment, so the rounding differs from the reference's one
//                      long chain by a few ulps of the largest term). Ranges that do not fit shared
//                      memory keep one thread per residue class (k_window_sum_uniform).
//
// Window kernels read the master panel (MasterArray) or, where every cell would be read
// exactly once (one nucleus, one window), evaluate the cells in place (MasterFused, the
// same arithmetic as k_master, so the panel is bitwise that of the two-step form).
//
// Layout: panels are column-major, column q contiguous (Eigen default), column index
// of the concatenated lattice tensor = v*R_N + q (nucleus-major, canonical_tensor.cpp:166-187).
#include "lt_device.cuh"
#include "lt_internal.cuh"
#include "tma.cuh"

#include <type_traits>

namespace lt {

// t == null: the node t_q is evaluated in place (sinc_node, k_sinc's arithmetic), so the
// master does not wait for the sinc kernel. A cell needs erf at its two edges and shares each
// with a neighbour: a CTA evaluates the kMasterC * 256 + 1 edges of its cells once into shared
// memory (one erf per cell instead of two; the extra edge by one warp) and differences them.
constexpr int kMasterC = 4;
__global__ void __launch_bounds__(256) k_master(Index mrows, double h, Index RN, const double* __restrict__ t, int M,
                                                double* __restrict__ out) {
    __shared__ double se[kMasterC * 256 + 1];
    const Index j0 = static_cast<Index>(blockIdx.x) * (kMasterC * 256);
    const Index q = blockIdx.y;
    const double tq = t ? t[q] : sinc_node(static_cast<int>(q), M);
    const int cells = static_cast<int>(min(static_cast<Index>(kMasterC * 256), mrows - j0));
#pragma unroll
    for (int u = 0; u < kMasterC; ++u) {
        const int i = threadIdx.x + 256 * u;
        if (i <= cells) se[i] = master_edge(j0 + i, mrows, h, tq);
    }
    if (threadIdx.x == 0 && cells == kMasterC * 256) se[cells] = master_edge(j0 + cells, mrows, h, tq);
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kMasterC; ++u) {
        const int i = threadIdx.x + 256 * u;
        if (i < cells) out[q * mrows + j0 + i] = master_from_edges(se[i], se[i + 1], tq);
    }
}

// the sinc nodes alone (k_sinc's t_q), for the master panel of a long lattice sum
__global__ void k_sinc_nodes(int M, double* t) {
    for (int q = threadIdx.x; q <= 2 * M; q += blockDim.x) t[q] = sinc_node(q, M);
}

void launch_sinc_nodes(const Launch& L, Index M, double* t) {
    Stage st_(L, "sinc");
    k_sinc_nodes<<<1, 128, 0, L.st>>>(static_cast<int>(M), t);
    LT_CU(cudaGetLastError());
    L.tick();
}

void launch_master(const Launch& L, Index mrows, double h, Index RN, const double* t, double* out, Index M) {
    dim3 grid(static_cast<unsigned>((mrows + kMasterC * 256 - 1) / (kMasterC * 256)), static_cast<unsigned>(RN));
    Stage st_(L, "master");
    k_master<<<grid, 256, 0, L.st>>>(mrows, h, RN, t, static_cast<int>(M), out);
    LT_CU(cudaGetLastError());
    L.tick();
}

struct MasterArray {  // caller-provided master panel [q][mrows]
    const double* m;
    Index mrows;
    __device__ double operator()(Index j, Index q, double) const { return m[q * mrows + j]; }
    __device__ double tq(Index) const { return 0.0; }
};

struct MasterFused {  // master cells evaluated on demand
    Index mrows;
    double h;
    int M;
    __device__ double operator()(Index j, Index, double tq) const { return master_cell(j, mrows, h, tq); }
    __device__ double tq(Index q) const { return sinc_node(static_cast<int>(q), M); }
};

// uniform progression: one thread per (v, q, residue r)
template <class Src>
__global__ void k_window_sum_uniform(Src src, Index RN, Index nnuc, const Index* __restrict__ s0v, Index K, Index step,
                                     Index size, double* __restrict__ out) {
    const Index nres = min(step, size);
    const Index tid = static_cast<Index>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= nnuc * RN * nres) return;
    const Index r = tid % nres;
    const Index q = (tid / nres) % RN;
    const Index v = tid / (nres * RN);
    const double tq = src.tq(q);
    double* o = out + (v * RN + q) * size;
    const Index s0 = s0v[v];
    double acc = 0.0;
    for (Index k = 0; k < K; ++k) acc = __dadd_rn(acc, src(s0 + r + k * step, q, tq));
    o[r] = acc;
    for (Index i = r + step; i < size; i += step) {
        acc = __dsub_rn(__dadd_rn(acc, src(s0 + i + (K - 1) * step, q, tq)), src(s0 + i - step, q, tq));
        o[i] = acc;
    }
}

// uniform progression staged through shared memory: CTA = (output chunk [i0, i0 + chunk), column
// v*RN + q). Lanes run along the residue r (coalesced stores, conflict-free shared loads),
// segments of Tl consecutive lattice steps along the rest of the CTA.
constexpr int kWsNT = 512;
constexpr Index kWsMaxSpan = 26000;  // doubles of master range per CTA (208 KB)
__global__ void __launch_bounds__(kWsNT) k_window_sum_staged(const double* __restrict__ m, Index mrows, Index RN,
                                                             const Index* __restrict__ s0v, int K, int step, Index size,
                                                             int chunk, int Tl, double* __restrict__ out) {
    extern __shared__ __align__(16) double ws_sm[];
    __shared__ uint64_t bar;
    const Index col = blockIdx.y;
    const Index v = col / RN, q = col % RN;
    const Index i0 = static_cast<Index>(blockIdx.x) * chunk;
    const int cnt = static_cast<int>(min(static_cast<Index>(chunk), size - i0));
    const int span = cnt + (K - 1) * step;
    const Index A0 = q * mrows + s0v[v] + i0;  // first master element of this CTA
    double* s = ws_sm + (A0 & 1);               // s[j] = m[A0 + j]; even master elements 16-byte aligned
    const Index Ab = (A0 + 1) & ~static_cast<Index>(1), Ae = (A0 + span) & ~static_cast<Index>(1);
    const bool bulk = Ae > Ab;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x == 0 && bulk) {
        mbar_arrive_expect_tx(&bar, static_cast<unsigned>((Ae - Ab) * 8));
        for (Index a = Ab; a < Ae; a += 4096) {
            const Index nb = min(static_cast<Index>(4096), Ae - a);
            tma_bulk_1d(s + (a - A0), m + a, static_cast<unsigned>(nb * 8), &bar);
        }
    }
    // the odd ends of the range (the bulk copy moves 16-byte units)
    if (threadIdx.x == 32 && (A0 & 1)) s[0] = m[A0];
    if (threadIdx.x == 64 && ((A0 + span) & 1)) s[span - 1] = m[A0 + span - 1];
    if (bulk) mbar_wait(&bar, 0);
    __syncthreads();
    const int nres = min(step, cnt);
    const int T = (cnt + step - 1) / step;
    const int S = (T + Tl - 1) / Tl;
    double* o = out + col * size + i0;
    // block sums over Tl consecutive lattice steps (one shared load per staged element): a
    // segment head is then K / Tl block sums plus the K mod Tl remaining terms
    const int nfull = Tl >= 2 ? K / Tl : 0;
    double* bs = ws_sm + ((span + 3) & ~1);  // [NB][nres]
    if (nfull > 0) {
        const int NB = (T + K - 1 + Tl - 1) / Tl;
        for (int item = threadIdx.x; item < nres * NB; item += kWsNT) {
            const int r = item % nres, c = item / nres;
            int j = r + c * Tl * step;
            double a0 = 0.0;
            for (int u = 0; u < Tl && j < span; ++u, j += step) a0 += s[j];  // past the span: no output reads it
            bs[item] = a0;
        }
        __syncthreads();
    }
    for (int item = threadIdx.x; item < nres * S; item += kWsNT) {
        const int r = item % nres, seg = item / nres;
        const int t0 = seg * Tl, t1 = min(T, t0 + Tl);
        const double* p = s + r + static_cast<size_t>(t0) * step;
        int i = r + t0 * step;
        if (i >= cnt) continue;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        {
            const double* b = bs + static_cast<size_t>(seg) * nres + r;
            int c = 0;
            for (; c + 3 < nfull; c += 4) {
                a0 += b[static_cast<size_t>(c) * nres];
                a1 += b[static_cast<size_t>(c + 1) * nres];
                a2 += b[static_cast<size_t>(c + 2) * nres];
                a3 += b[static_cast<size_t>(c + 3) * nres];
            }
            for (; c < nfull; ++c) a0 += b[static_cast<size_t>(c) * nres];
        }
        int k = nfull * Tl;
        for (; k + 3 < K; k += 4) {
            a0 += p[static_cast<size_t>(k) * step];
            a1 += p[static_cast<size_t>(k + 1) * step];
            a2 += p[static_cast<size_t>(k + 2) * step];
            a3 += p[static_cast<size_t>(k + 3) * step];
        }
        for (; k < K; ++k) a0 += p[static_cast<size_t>(k) * step];
        double acc = (a0 + a1) + (a2 + a3);
        o[i] = acc;
        for (int t = t0 + 1; t < t1; ++t) {
            i += step;
            if (i >= cnt) break;
            const int u = t - t0;
            acc = __dsub_rn(__dadd_rn(acc, p[static_cast<size_t>(u + K - 1) * step]), p[static_cast<size_t>(u - 1) * step]);
            o[i] = acc;
        }
    }
}

// size <= step (the periodic cell window: every residue class holds one output): no
// running-sum recurrence. CTA = 8 warps over 32 consecutive outputs r (coalesced reads
// along r); warp w sums the k-slice k = w, w+8, ...; the 8 slice sums are added in warp
// order (a fixed order, instead of the serial K-term chain)
template <class Src>
__global__ void __launch_bounds__(256) k_window_sum_short(Src src, Index RN, Index nnuc, const Index* __restrict__ s0v,
                                                          Index K, Index step, Index size, double* __restrict__ out) {
    __shared__ double part[8][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const Index rblocks = (size + 31) / 32;
    const Index col = blockIdx.x / rblocks;  // v*RN + q
    const Index r = (blockIdx.x % rblocks) * 32 + lane;
    const Index v = col / RN, q = col % RN;
    const double tq = src.tq(q);
    const Index s0 = s0v[v];
    double acc = 0.0;
    if (r < size)
        for (Index k = warp; k < K; k += 8) acc += src(s0 + r + k * step, q, tq);
    part[warp][lane] = acc;
    __syncthreads();
    if (warp == 0 && r < size) {
        double t = part[0][lane];
        for (int w = 1; w < 8; ++w) t += part[w][lane];
        out[col * size + r] = t;
    }
}

// single shift (non-uniform branch with one window): out = 0 + m[s0 + i]
template <class Src>
__global__ void k_window_copy(Src src, Index RN, Index nnuc, const Index* __restrict__ s0v, Index size,
                              double* __restrict__ out) {
    const Index i = static_cast<Index>(blockIdx.x) * blockDim.x + threadIdx.x;
    const Index col = blockIdx.y;  // v*RN + q
    if (i >= size) return;
    const Index v = col / RN, q = col % RN;
    out[col * size + i] = src(s0v[v] + i, q, src.tq(q));
}

template <class Src>
static void window_sum(const Launch& L, const Src& src, Index RN, Index nnuc, const Index* s0_dev, Index nsum,
                       Index step, Index size, double* out) {
    Stage st_(L, "window_sum");
    if (nsum >= 8 && size <= step) {
        const Index blocks = nnuc * RN * ((size + 31) / 32);
        k_window_sum_short<<<static_cast<unsigned>(blocks), 256, 0, L.st>>>(src, RN, nnuc, s0_dev, nsum, step, size,
                                                                              out);
    } else if (nsum >= 2) {
        if constexpr (std::is_same_v<Src, MasterArray>) {
            const Index ov = (nsum - 1) * step;
            if (ov + std::min(size, step) + 8 <= kWsMaxSpan && nsum < (1 << 20) && step < (1 << 20)) {
                // chunks of whole lattice steps: about one CTA per SM (every chunk re-reads the
                // (K - 1) step halo, so fewer, larger chunks move less), segments of Tl steps with
                // Tl ~ sqrt(K / 2) balancing the K / Tl block sums of a head against its 2 Tl updates
                const Index cols = nnuc * RN;
                Index nchunks = std::max<Index>(1, std::min<Index>(148 / std::max<Index>(cols, 1), (size + 4 * step - 1) / (4 * step)));
                Index chunk = size, Tl = 1;
                size_t smem = 0;
                for (;; ++nchunks) {
                    chunk = size <= step ? size : ((size + nchunks - 1) / nchunks + step - 1) / step * step;
                    const Index T = (chunk + step - 1) / step, nres = std::min(step, chunk);
                    const Index S = std::max<Index>(1, std::min<Index>(T, kWsNT / std::min<Index>(nres, kWsNT)));
                    Index root = 1;
                    while (2 * (root + 1) * (root + 1) <= nsum) ++root;
                    Tl = std::max((T + S - 1) / S, std::min(T, root));
                    const Index NB = Tl >= 2 ? (T + nsum - 1 + Tl - 1) / Tl : 0;
                    smem = sizeof(double) * static_cast<size_t>(chunk + ov + 6 + NB * nres);
                    if (smem <= sizeof(double) * (kWsMaxSpan + 2) || chunk <= step) break;
                }
                if (smem > sizeof(double) * (kWsMaxSpan + 2)) Tl = 1, smem = sizeof(double) * static_cast<size_t>(chunk + ov + 6);
                nchunks = (size + chunk - 1) / chunk;
                static bool attr = false;
                if (!attr) {
                    LT_CU(cudaFuncSetAttribute(k_window_sum_staged, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(sizeof(double) * (kWsMaxSpan + 8))));
                    attr = true;
                }
                dim3 grid(static_cast<unsigned>(nchunks), static_cast<unsigned>(cols));
                k_window_sum_staged<<<grid, kWsNT, smem, L.st>>>(src.m, src.mrows, RN, s0_dev, static_cast<int>(nsum),
                                                                  static_cast<int>(step), size, static_cast<int>(chunk),
                                                                  static_cast<int>(Tl), out);
                LT_CU(cudaGetLastError());
                L.tick();
                return;
            }
        }
        const Index nres = std::min(step, size);
        const Index threads = nnuc * RN * nres;
        k_window_sum_uniform<<<static_cast<unsigned>((threads + 127) / 128), 128, 0, L.st>>>(src, RN, nnuc, s0_dev,
                                                                                              nsum, step, size, out);
    } else {
        dim3 grid(static_cast<unsigned>((size + 255) / 256), static_cast<unsigned>(nnuc * RN));
        k_window_copy<<<grid, 256, 0, L.st>>>(src, RN, nnuc, s0_dev, size, out);
    }
    LT_CU(cudaGetLastError());
    L.tick();
}

void launch_window_sum(const Launch& L, const double* master, Index mrows, Index RN, Index nnuc, const Index* s0_dev,
                       Index nsum, Index step, Index size, double* out) {
    window_sum(L, MasterArray{master, mrows}, RN, nnuc, s0_dev, nsum, step, size, out);
}

void launch_potential_fused(const Launch& L, Index mrows, double h, Index M, Index RN, Index nnuc, const Index* s0_dev,
                            Index nsum, Index step, Index size, double* out) {
    window_sum(L, MasterFused{mrows, h, static_cast<int>(M)}, RN, nnuc, s0_dev, nsum, step, size, out);
}

}  // namespace lt
