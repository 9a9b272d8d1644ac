// k_spectrum.cu — block diagonalisation over lattice indices and batched pencil eigensolves.
//
//   launch_scatter_gen / launch_dft_axis
//       bc_block_diagonalize + fft_levels (block_circulant.cpp:82-112, :184-196):
//       unnormalised forward DFT, omega = exp(-2 pi i / L), axis 0 then 1 then 2, for every
//       block entry. Only the stored generating blocks are non-zero, so each axis is a
//       sparse DFT from the compressed set of stored kidx values to all L frequencies
//       (exact same sum as the zero-padded FFT; K = (2b+1) terms per output instead of
//       log L butterflies over mostly zeros).
// The batched pencil eigensolver is in k_pencil.cu.
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

}  // namespace lt
