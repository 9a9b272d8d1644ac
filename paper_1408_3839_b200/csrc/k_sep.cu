// k_sep.cu — separable coefficient metadata and the factorized Fourier path
// (galerkin.cpp:394-423, :427-444; factorized_diag.cpp:12-101; eigensolver.cpp:143-162).
//
// Metadata of an operator: rank terms t, each a Hadamard product over the three levels of
// per-level block sequences A^(l,t)_{k_l}. Stored band-compressed on the device:
//     vals[t][l][s][e],  slot s of level l holds the block at lattice index kid_l[s]
// (slots absent from a level are zero blocks). The factorized path applies one 1D DFT per
// level and term, X^(l,t)_j = sum_s w_l^(j kid_l[s]) A^(l,t)_s, and forms every k-point
// block as sum_t (X^(0,t)_{k0} o X^(1,t)_{k1}) o X^(2,t)_{k2} (FactorizedDiagonalizer::block).
#include "lt_device.cuh"
#include "lt_internal.cuh"

namespace lt {

namespace {
__device__ __forceinline__ double2 zmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
}  // namespace

// metadata from assembly tables (galerkin.cpp:398-421):
//   kind 1 (Mass):    term 0, level l, slot s: massT_l[s]
//   kind 0 (Laplace): term t, level l: (l == t ? stiffT_l : massT_l)[s]
//   kind 2 (Nuclear): term r, level l: T_l[s][r] (the per-pair table), times w_r on level 0
__global__ void k_sep_from_tables(SepBuild b) {
    const Index mm = b.mm;
    const Index e = static_cast<Index>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int l = blockIdx.y;
    const Index ts = blockIdx.z;  // t * S + s
    const Index t = ts / b.S, s = ts % b.S;
    if (e >= mm || s >= b.nslot[l]) return;
    double v = 0.0;
    if (b.kind == 1) {
        v = b.mass[l][s * mm + e];
    } else if (b.kind == 0) {
        v = (l == t ? b.stiff[l] : b.mass[l])[s * mm + e];
    } else {
        v = b.T[l][(s * b.R + t) * mm + e];
        if (l == 0) v = __dmul_rn(v, b.potw[t]);  // blk *= pot_weights[r] on level 0
    }
    b.out[((t * 3 + l) * b.S + s) * mm + e] = v;
}

void launch_sep_from_tables(const Launch& L, const SepBuild& b, Index terms) {
    dim3 grid(static_cast<unsigned>((b.mm + 127) / 128), 3, static_cast<unsigned>(terms * b.S));
    Stage st_(L, "sep_build");
    k_sep_from_tables<<<grid, 128, 0, L.st>>>(b);
    LT_CU(cudaGetLastError());
    L.tick();
}

// dst[(t0 + t)][l][map_l[s]][e] = (l == 0 ? w : 1) * src[t][l][s][e]   (combine: scaled
// concatenation of the term lists, eigensolver.cpp:57-64, with the slot sets re-indexed)
__global__ void k_sep_scale_copy(SepCopy c) {
    const Index e = static_cast<Index>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int l = blockIdx.y;
    const Index ts = blockIdx.z;
    const Index t = ts / c.Ssrc, s = ts % c.Ssrc;
    if (e >= c.mm || s >= c.nslot[l]) return;
    const double v = c.src[((t * 3 + l) * c.Ssrc + s) * c.mm + e];
    c.dst[(((c.t0 + t) * 3 + l) * c.Sdst + c.map[l][s]) * c.mm + e] = l == 0 ? __dmul_rn(c.w, v) : v;
}

void launch_sep_scale_copy(const Launch& L, const SepCopy& c, Index terms) {
    dim3 grid(static_cast<unsigned>((c.mm + 127) / 128), 3, static_cast<unsigned>(terms * c.Ssrc));
    Stage st_(L, "sep_copy");
    k_sep_scale_copy<<<grid, 128, 0, L.st>>>(c);
    LT_CU(cudaGetLastError());
    L.tick();
}

// per-level 1D DFTs: X[t][l][j][e] = sum_s w^(j kid_l[s] mod L_l) vals[t][l][s][e]
__global__ void k_sep_dft(SepDft d) {
    const Index mm = d.mm;
    const Index e = static_cast<Index>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int l = blockIdx.y;
    const Index tj = blockIdx.z;  // t * Lmax + j
    const Index t = tj / d.Lmax, j = tj % d.Lmax;
    const Index Ll = d.L[l];
    if (e >= mm || j >= Ll) return;
    double2 acc = make_double2(0.0, 0.0);
    for (Index s = 0; s < d.nslot[l]; ++s) {
        const Index m = (j * d.kid[l][s]) % Ll;
        double sn, co;
        sincospi(-2.0 * static_cast<double>(m) / static_cast<double>(Ll), &sn, &co);
        const double v = d.vals[((t * 3 + l) * d.S + s) * mm + e];
        acc.x += co * v;
        acc.y += sn * v;
    }
    d.out[((t * 3 + l) * d.Lmax + j) * mm + e] = acc;
}

void launch_sep_dft(const Launch& L, const SepDft& d, Index terms) {
    dim3 grid(static_cast<unsigned>((d.mm + 127) / 128), 3, static_cast<unsigned>(terms * d.Lmax));
    Stage st_(L, "sep_dft");
    k_sep_dft<<<grid, 128, 0, L.st>>>(d);
    LT_CU(cudaGetLastError());
    L.tick();
}

// k-point blocks: F[k][e] = sum_t (X0[k0] o X1[k1]) o X2[k2]
__global__ void k_sep_blocks(SepBlocks b) {
    const Index mm = b.mm;
    const Index idx = static_cast<Index>(blockIdx.x) * blockDim.x + threadIdx.x;
    const Index K = b.L[0] * b.L[1] * b.L[2];
    if (idx >= K * mm) return;
    const Index k = idx / mm, e = idx % mm;
    const Index k0 = k / (b.L[1] * b.L[2]), k1 = (k / b.L[2]) % b.L[1], k2 = k % b.L[2];
    double2 acc = make_double2(0.0, 0.0);
    for (Index t = 0; t < b.terms; ++t) {
        const double2* X = b.X + t * 3 * b.Lmax * mm;
        const double2 p = zmul(zmul(X[(0 * b.Lmax + k0) * mm + e], X[(1 * b.Lmax + k1) * mm + e]),
                               X[(2 * b.Lmax + k2) * mm + e]);
        acc.x += p.x;
        acc.y += p.y;
    }
    b.out[idx] = acc;
}

void launch_sep_blocks(const Launch& L, const SepBlocks& b) {
    const Index tot = b.L[0] * b.L[1] * b.L[2] * b.mm;
    Stage st_(L, "sep_blocks");
    k_sep_blocks<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, L.st>>>(b);
    LT_CU(cudaGetLastError());
    L.tick();
}

// residual max_k max_e |gen_k - sum_t prod_l A^(l,t)_{k_l}| over every lattice point
// (separable_residual, galerkin.cpp:427-444); non-negative doubles order like their bits
__global__ void k_sep_residual(SepResid r) {
    const Index mm = r.mm;
    const Index idx = static_cast<Index>(blockIdx.x) * blockDim.x + threadIdx.x;
    const Index K = r.L[0] * r.L[1] * r.L[2];
    double diff = 0.0;
    if (idx < K * mm) {
        const Index k = idx / mm, e = idx % mm;
        const Index kk[3] = {k / (r.L[1] * r.L[2]), (k / r.L[2]) % r.L[1], k % r.L[2]};
        const int s0 = r.slot_of[0][kk[0]], s1 = r.slot_of[1][kk[1]], s2 = r.slot_of[2][kk[2]];
        double ex = 0.0;
        if (s0 >= 0 && s1 >= 0 && s2 >= 0)
            for (Index t = 0; t < r.terms; ++t) {
                const double a = r.vals[((t * 3 + 0) * r.S + s0) * mm + e];
                const double b = r.vals[((t * 3 + 1) * r.S + s1) * mm + e];
                const double c = r.vals[((t * 3 + 2) * r.S + s2) * mm + e];
                ex += (a * b) * c;
            }
        const int gb = r.gen_of[k];
        const double g = gb >= 0 ? r.gen[static_cast<Index>(gb) * mm + e] : 0.0;
        diff = fabs(g - ex);
    }
    diff = warp_max(diff);
    if ((threadIdx.x & 31) == 0 && diff > 0.0)
        atomicMax(r.out, static_cast<unsigned long long>(__double_as_longlong(diff)));
}

void launch_sep_residual(const Launch& L, const SepResid& r) {
    const Index tot = r.L[0] * r.L[1] * r.L[2] * r.mm;
    Stage st_(L, "sep_residual");
    k_sep_residual<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, L.st>>>(r);
    LT_CU(cudaGetLastError());
    L.tick();
}

}  // namespace lt

namespace lt {

// box_circulant_defect (galerkin.cpp:445-454): defect = box - bc_to_dense(periodic) where
// block (i, j) of the circulant is gen[(m_i - m_j) mod L] (block_circulant.cpp:128-149).
// Writes the defect (optional) and per-CTA partial sums of defect^2 and box^2; the host
// adds the partials in CTA order (deterministic).
__global__ void k_circ_defect(CircDefect d) {
    __shared__ double s_def[8], s_box[8];
    const Index nb = d.Nb, m0 = d.m0;
    double acc_d = 0.0, acc_b = 0.0;
    for (Index idx = static_cast<Index>(blockIdx.x) * blockDim.x + threadIdx.x; idx < nb * nb;
         idx += static_cast<Index>(gridDim.x) * blockDim.x) {
        const Index row = idx % nb, col = idx / nb;  // column-major
        const Index i = row / m0, j = col / m0, mu = row % m0, nu = col % m0;
        Index k[3];
        const Index iv[3] = {i / (d.L[1] * d.L[2]), (i / d.L[2]) % d.L[1], i % d.L[2]};
        const Index jv[3] = {j / (d.L[1] * d.L[2]), (j / d.L[2]) % d.L[1], j % d.L[2]};
#pragma unroll
        for (int l = 0; l < 3; ++l) k[l] = ((iv[l] - jv[l]) % d.L[l] + d.L[l]) % d.L[l];
        const int b = d.gen_of[(k[0] * d.L[1] + k[1]) * d.L[2] + k[2]];
        const double per = b >= 0 ? d.gen[static_cast<Index>(b) * m0 * m0 + mu + nu * m0] : 0.0;
        const double box = d.box[idx];
        const double df = box - per;
        if (d.defect) d.defect[idx] = df;
        acc_d = fma(df, df, acc_d);
        acc_b = fma(box, box, acc_b);
    }
    for (int o = 16; o > 0; o >>= 1) {
        acc_d += __shfl_xor_sync(0xffffffffu, acc_d, o);
        acc_b += __shfl_xor_sync(0xffffffffu, acc_b, o);
    }
    if ((threadIdx.x & 31) == 0) {
        s_def[threadIdx.x >> 5] = acc_d;
        s_box[threadIdx.x >> 5] = acc_b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, bsum = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
            a += s_def[w];
            bsum += s_box[w];
        }
        d.partial[2 * blockIdx.x] = a;
        d.partial[2 * blockIdx.x + 1] = bsum;
    }
}

void launch_circ_defect(const Launch& L, const CircDefect& d, int blocks) {
    Stage st_(L, "circ_defect");
    k_circ_defect<<<blocks, 256, 0, L.st>>>(d);
    LT_CU(cudaGetLastError());
    L.tick();
}

}  // namespace lt
