// k_potential.cu — Newton-kernel master panels and the assembled lattice sum.
//
//   launch_master      newton_kernel.cpp:22-45: f(i,q) = sqrt(pi)/(2 t_q) (erf(t_q x_{i+1}) - erf(t_q x_i))
//                      on the centred cell grid x_i = -n h/2 + i h (grid.hpp:28-38)
//   launch_window_sum  canonical_tensor.cpp:123-164: out[i] = sum_k m[s_k + i] over the sorted
//                      lattice shifts s_k = s0 + k*step; uniform progressions use the
//                      reference's running sum out[i] = out[i-step] + m[s0+i+(K-1)step] - m[s0+i-step]
//                      (same recurrence, same rounding), one thread per residue class.
//
// Layout: panels are column-major, column q contiguous (Eigen default), column index
// of the concatenated lattice tensor = v*R_N + q (nucleus-major, canonical_tensor.cpp:166-187).
#include "lt_device.cuh"
#include "lt_internal.cuh"

namespace lt {

__global__ void k_master(Index mrows, double h, Index RN, const double* __restrict__ t, double* __restrict__ out) {
    const Index j = static_cast<Index>(blockIdx.x) * blockDim.x + threadIdx.x;
    const Index q = blockIdx.y;
    if (j >= mrows) return;
    const double tq = t[q];
    const double origin = __dmul_rn(__dmul_rn(-0.5, static_cast<double>(mrows)), h);
    const double xl = __dadd_rn(origin, __dmul_rn(static_cast<double>(j), h));
    const double xr = __dadd_rn(origin, __dmul_rn(static_cast<double>(j + 1), h));
    const double c = __ddiv_rn(sqrt(3.141592653589793), __dmul_rn(2.0, tq));
    const double el = erf(__dmul_rn(tq, xl));
    const double er = erf(__dmul_rn(tq, xr));
    out[q * mrows + j] = __dmul_rn(c, __dsub_rn(er, el));
}

void launch_master(const Launch& L, Index mrows, double h, Index RN, const double* t, double* out) {
    dim3 grid(static_cast<unsigned>((mrows + 255) / 256), static_cast<unsigned>(RN));
    Stage st_(L, "master");
    k_master<<<grid, 256, 0, L.st>>>(mrows, h, RN, t, out);
    LT_CU(cudaGetLastError());
    L.tick();
}

// uniform progression: one thread per (v, q, residue r)
__global__ void k_window_sum_uniform(const double* __restrict__ m, Index mrows, Index RN, Index nnuc,
                                     const Index* __restrict__ s0v, Index K, Index step, Index size,
                                     double* __restrict__ out) {
    const Index nres = min(step, size);
    const Index tid = static_cast<Index>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= nnuc * RN * nres) return;
    const Index r = tid % nres;
    const Index q = (tid / nres) % RN;
    const Index v = tid / (nres * RN);
    const double* col = m + q * mrows;
    double* o = out + (v * RN + q) * size;
    const Index s0 = s0v[v];
    double acc = 0.0;
    for (Index k = 0; k < K; ++k) acc = __dadd_rn(acc, col[s0 + r + k * step]);
    o[r] = acc;
    for (Index i = r + step; i < size; i += step) {
        acc = __dsub_rn(__dadd_rn(acc, col[s0 + i + (K - 1) * step]), col[s0 + i - step]);
        o[i] = acc;
    }
}

// single shift (non-uniform branch with one window): out = 0 + m[s0 + i]
__global__ void k_window_copy(const double* __restrict__ m, Index mrows, Index RN, Index nnuc,
                              const Index* __restrict__ s0v, Index size, double* __restrict__ out) {
    const Index i = static_cast<Index>(blockIdx.x) * blockDim.x + threadIdx.x;
    const Index col = blockIdx.y;  // v*RN + q
    if (i >= size) return;
    const Index v = col / RN, q = col % RN;
    out[col * size + i] = m[q * mrows + s0v[v] + i];
}

void launch_window_sum(const Launch& L, const double* master, Index mrows, Index RN, Index nnuc, const Index* s0_dev,
                       Index nsum, Index step, Index size, double* out) {
    Stage st_(L, "window_sum");
    if (nsum >= 2) {
        const Index nres = std::min(step, size);
        const Index threads = nnuc * RN * nres;
        k_window_sum_uniform<<<static_cast<unsigned>((threads + 127) / 128), 128, 0, L.st>>>(
            master, mrows, RN, nnuc, s0_dev, nsum, step, size, out);
    } else {
        dim3 grid(static_cast<unsigned>((size + 255) / 256), static_cast<unsigned>(nnuc * RN));
        k_window_copy<<<grid, 256, 0, L.st>>>(master, mrows, RN, nnuc, s0_dev, size, out);
    }
    LT_CU(cudaGetLastError());
    L.tick();
}

}  // namespace lt
