// k_setup.cu — sinc quadrature and the overlap constant L0.
//
//   launch_sinc            sinc_quadrature.cpp:9-29 (+ weights Z_v w_q, newton_kernel.cpp:150,
//                          canonical_tensor.cpp:166-187 nucleus-major concatenation)
//   launch_overlap_*       gto_basis.cpp:87-126 (per-direction grids)
//
// The L0 scan is an exact block-max-pruned search: for each shift s and pair
// (mu, nu, l) the reference takes worst = max_i |a_i c_{i-sn}| and compares it with
// eps_ov. Rounding is monotone, so fl(max|a|_blk * max|c|_blk) < eps proves every
// product of that block pair is < eps; only blocks whose bound reaches eps are
// scanned element by element. The resulting L0 is identical to the full scan.
#include <cfloat>

#include "lt_device.cuh"
#include "lt_internal.cuh"

namespace lt {

// potw[r] = Z_v w_q for rank terms r = v R + q in [r0, r1), 0 outside (a rank-term shard of
// the multi-GPU assembly: the shards' nuclear parts sum to the full one)
__global__ void k_sinc(int M, int nnuc, const double* __restrict__ Z, double* t, double* w, double* potw, long long r0,
                       long long r1) {
    const int R = 2 * M + 1;
    double step = log(static_cast<double>(M)) / static_cast<double>(M);
    if (M == 1) step = 0.5;
    const double c = (2.0 * step) / sqrt(3.141592653589793);
    for (int i = threadIdx.x; i < R; i += blockDim.x) {
        const double u = __dmul_rn(static_cast<double>(i - M), step);
        const double eu = exp(-u);
        const double ti = sinc_node(i, M);  // exp(u - e^-u), shared with the fused potential
        const double wi = __dmul_rn(c, __dadd_rn(ti, exp(-eu)));
        t[i] = ti;
        w[i] = wi;
        for (int v = 0; v < nnuc; ++v) {
            const long long r = static_cast<long long>(v) * R + i;
            potw[r] = (r >= r0 && r < r1) ? __dmul_rn(wi, Z[v]) : 0.0;
        }
    }
}

void launch_sinc(const Launch& L, Index M, const DevSys& s, double* t, double* w, double* potw, Index r0, Index r1) {
    Stage st_(L, "sinc");
    k_sinc<<<1, 128, 0, L.st>>>(static_cast<int>(M), s.nnuc, s.Z, t, w, potw, r0, r1 < 0 ? (1LL << 62) : r1);
    LT_CU(cudaGetLastError());
    L.tick();
}

// ---------------------------------------------------------------------------
// overlap constant
// ---------------------------------------------------------------------------
constexpr int kMaxL0 = 256;

struct Dir3 {
    Index n[3], off[3], boff[3];
    int nl;          // active (de-duplicated) directions
    int dir[3];      // their indices
    Index tcum[4];   // sample tasks: cumulative m0 * nblk over the active directions
};

__device__ __forceinline__ double l0_x(Index i, Index base, double h, double b) {
    return __dsub_rn(__dmul_rn(__dadd_rn(static_cast<double>(i - base), 0.5), h), __dmul_rn(0.5, b));
}

// Samples the untrimmed L0 profiles (gto_basis.cpp:95-97: width 2 (256+2) n, the
// function in cell 258) and their block maxima. One warp per 128-point block in a
// grid-stride loop. A block whose nearest point to the centre already has
// fl(fl(alpha d) d) > 746 is all zeros without evaluation: d = fl(x - c) and the
// products are monotone in |d|, so every point of it takes gto_eval1d's exact zero
// shortcut. Values are stored only for blocks with a non-zero maximum (the scan treats
// the others as zero); the first/last non-zero block of each profile is recorded.
__global__ void __launch_bounds__(256) k_l0_sample(DevSys s, Dir3 d, double* __restrict__ prof,
                                                   double* __restrict__ bmax, unsigned* __restrict__ nz) {
    const int lane = threadIdx.x & 31;
    const Index nwarps = static_cast<Index>(gridDim.x) * (blockDim.x >> 5);
    for (Index task = static_cast<Index>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); task < d.tcum[d.nl];
         task += nwarps) {
        int k = 0;
        while (task >= d.tcum[k + 1]) ++k;
        const int l = d.dir[k];
        const Index n = d.n[l];
        const Index width = 2 * (kMaxL0 + 2) * n;
        const Index nblk = (width + kL0Block - 1) / kL0Block;
        const Index rem = task - d.tcum[k];
        const int mu = static_cast<int>(rem / nblk);
        const Index blk = rem % nblk;
        const double h = s.b / static_cast<double>(n);
        const Index base = (kMaxL0 + 2) * n;
        const Index i0 = blk * kL0Block, i1 = min(i0 + kL0Block, width) - 1;
        const double c = s.center[3 * mu + l];
        const double x0 = l0_x(i0, base, h, s.b), x1 = l0_x(i1, base, h, s.b);
        const double dmin = c < x0 ? __dsub_rn(x0, c) : (c > x1 ? __dsub_rn(c, x1) : 0.0);
        double* bm = bmax + d.boff[l] + mu * nblk + blk;
        if (__dmul_rn(__dmul_rn(s.alpha[mu], dmin), dmin) > 746.0) {
            if (lane == 0) *bm = 0.0;
            continue;
        }
        double v[kL0Block / 32];
        double av = 0.0;
#pragma unroll
        for (int q = 0; q < kL0Block / 32; ++q) {
            const Index i = i0 + lane + 32 * q;
            v[q] = i <= i1 ? gto_eval1d(s, mu, l, l0_x(i, base, h, s.b)) : 0.0;
            av = fmax(av, fabs(v[q]));
        }
        const double m = warp_max(av);  // exact: max is order independent
        if (m > 0.0) {
            double* out = prof + d.off[l] + mu * width;
#pragma unroll
            for (int q = 0; q < kL0Block / 32; ++q)
                if (i0 + lane + 32 * q <= i1) out[i0 + lane + 32 * q] = v[q];
        }
        if (lane == 0) {
            *bm = m;
            if (m > 0.0) {
                atomicMin(&nz[(l * s.m0 + mu) * 2], static_cast<unsigned>(blk));
                atomicMax(&nz[(l * s.m0 + mu) * 2 + 1], static_cast<unsigned>(blk));
            }
        }
    }
}

static Dir3 make_dir3(const DevSys& s, const Index* n3, const Index* off3, const Index* boff3, const int* active) {
    Dir3 d{};
    d.nl = 0;
    d.tcum[0] = 0;
    for (int l = 0; l < 3; ++l) {
        d.n[l] = n3[l];
        d.off[l] = off3[l];
        d.boff[l] = boff3[l];
        if (!active[l]) continue;
        const Index width = 2 * (kMaxL0 + 2) * n3[l];
        d.dir[d.nl] = l;
        d.tcum[d.nl + 1] = d.tcum[d.nl] + static_cast<Index>(s.m0) * ((width + kL0Block - 1) / kL0Block);
        ++d.nl;
    }
    for (int k = d.nl; k < 3; ++k) d.tcum[k + 1] = d.tcum[k];
    return d;
}

void launch_overlap_profiles(const Launch& L, const DevSys& s, const Index* n3, const Index* off3, const Index* boff3,
                             const int* active, OverlapBufs b) {
    const Dir3 d = make_dir3(s, n3, off3, boff3, active);
    const Index blocks = std::min<Index>((d.tcum[d.nl] + 7) / 8, 148 * 8);
    Stage st_(L, "l0_sample");
    k_l0_sample<<<static_cast<unsigned>(std::max<Index>(1, blocks)), 256, 0, L.st>>>(s, d, b.prof, b.bmax, b.nz);
    LT_CU(cudaGetLastError());
    L.tick();
}

__global__ void k_l0_init(int* found, int* state, unsigned* nz, int nnz) {
    for (int i = threadIdx.x; i <= kMaxL0; i += blockDim.x) found[i] = 0;
    for (int i = threadIdx.x; i < nnz; i += blockDim.x) nz[i] = (i & 1) ? 0u : 0xffffffffu;
    if (threadIdx.x == 0) {
        state[0] = 0;  // L0
        state[1] = 0;  // misses
        state[2] = 1;  // next s
        state[3] = 0;  // done
        state[4] = 0;  // finished-block counter of the fused scan/finalize
        state[6] = -1;  // ints 6-7: the pencil failure key (~0 = none) of the read-back block
        state[7] = -1;
    }
}

void launch_overlap_init(const Launch& L, OverlapBufs b, int m0) {
    Stage st_(L, "l0_init");
    k_l0_init<<<1, 256, 0, L.st>>>(b.found, b.state, b.nz, 3 * m0 * 2);
    LT_CU(cudaGetLastError());
    L.tick();
}

// the reference's sequential rule: L0 = last s with worst >= eps; stop after 2 misses
__device__ void l0_finalize(const int* found, int* state, int s_end) {
    int L0 = state[0], misses = state[1], sft = state[2];
    for (; sft <= kMaxL0 && sft < s_end && misses < 2; ++sft) {
        if (__ldcg(&found[sft])) {
            L0 = sft;
            misses = 0;
        } else {
            ++misses;
        }
    }
    state[0] = L0;
    state[1] = misses;
    state[2] = sft;
    state[3] = (misses >= 2 || sft > kMaxL0) ? 1 : 0;
}

// One warp per (s, l, mu, nu) over the active directions (a duplicated direction has the
// same profiles, so its answers are identical): is there an i with |a_i c_{i-sn}| >= eps_ov?
// Only blocks where both profiles are non-zero are visited; a block pair is scanned
// element-wise only if fl(max|a|_blk * max|c|_blk) >= eps (exact pruning: rounding is
// monotone). Lanes test the bounds of 32 blocks at once; each candidate block is then
// scanned by the whole warp. The last CTA to finish applies the sequential L0 rule.
__global__ void k_l0_scan(DevSys s, Dir3 d, const double* __restrict__ prof, const double* __restrict__ bmax,
                          const unsigned* __restrict__ nz, int* found, int* state, int s_begin, int ns, int s_end,
                          int finalize) {
    const int lane = threadIdx.x & 31;
    const Index task = static_cast<Index>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const Index m0 = s.m0;
    const Index per_s = static_cast<Index>(d.nl) * m0 * m0;
    bool hit = false;
    int sft = 0;
    if (task < per_s * ns) {
        sft = s_begin + static_cast<int>(task / per_s);
        Index rem = task % per_s;
        const int l = d.dir[rem / (m0 * m0)];
        rem %= m0 * m0;
        const Index mu = rem / m0, nu = rem % m0;
        const Index n = d.n[l];
        const Index width = 2 * (kMaxL0 + 2) * n;
        const Index nblk = (width + kL0Block - 1) / kL0Block;
        const Index sn = static_cast<Index>(sft) * n;
        const Index alo = nz[(l * m0 + mu) * 2], ahi = nz[(l * m0 + mu) * 2 + 1];
        const Index clo = nz[(l * m0 + nu) * 2], chi = nz[(l * m0 + nu) * 2 + 1];
        Index jlo = max(alo, sn / kL0Block);
        jlo = max(jlo, (clo * kL0Block + sn) / kL0Block);
        Index jhi = min(ahi, nblk - 1);
        jhi = min(jhi, (chi * kL0Block + kL0Block - 1 + sn) / kL0Block);
        if (!__ldcg(&found[sft]) && sn < width && alo <= ahi && clo <= chi) {
            const double* a = prof + d.off[l] + mu * width;
            const double* c = prof + d.off[l] + nu * width;
            const double* am = bmax + d.boff[l] + mu * nblk;
            const double* cm = bmax + d.boff[l] + nu * nblk;
            const double eps = s.eps_ov;
            for (Index ja0 = jlo; ja0 <= jhi && !hit; ja0 += 32) {
                const Index ja = ja0 + lane;
                Index ilo = 0, ihi = 0;
                bool cand = false;
                if (ja <= jhi) {
                    ilo = max(ja * kL0Block, sn);
                    ihi = min(ja * kL0Block + kL0Block, width);
                    if (ilo < ihi) {
                        const Index cb0 = (ilo - sn) / kL0Block, cb1 = (ihi - 1 - sn) / kL0Block;
                        cand = am[ja] * fmax(cm[cb0], cm[cb1]) >= eps;
                    }
                }
                unsigned mask = __ballot_sync(0xffffffffu, cand);
                while (mask && !hit) {
                    const int src = __ffs(mask) - 1;
                    mask &= mask - 1;
                    const Index blo = __shfl_sync(0xffffffffu, ilo, src), bhi = __shfl_sync(0xffffffffu, ihi, src);
                    const double amx = am[(blo) / kL0Block];
                    bool h = false;
                    for (Index i = blo + lane; i < bhi; i += 32) {
                        const Index ci = i - sn;
                        const double av = amx > 0.0 ? a[i] : 0.0;
                        const double cv = cm[ci / kL0Block] > 0.0 ? c[ci] : 0.0;
                        h |= fabs(av * cv) >= eps;
                    }
                    hit = __any_sync(0xffffffffu, h);
                }
            }
        }
    }
    if (hit && lane == 0) atomicExch(&found[sft], 1);
    if (!finalize) return;
    // fused finalize: the last CTA to finish applies the sequential rule
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&state[4], 1) == static_cast<int>(gridDim.x) - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        l0_finalize(found, state, s_end);
        state[4] = 0;
    }
}

void launch_overlap_scan(const Launch& L, const DevSys& s, const Index* n3, const Index* off3, const Index* boff3,
                         const int* active, OverlapBufs b, int s_begin, int s_end, bool finalize) {
    const Dir3 d = make_dir3(s, n3, off3, boff3, active);
    const int ns = s_end - s_begin;
    const Index tasks = static_cast<Index>(ns) * d.nl * s.m0 * s.m0;
    const int wpb = 8;
    const Index blocks = std::max<Index>(1, (tasks + wpb - 1) / wpb);
    Stage st_(L, "l0_scan");
    k_l0_scan<<<static_cast<unsigned>(blocks), wpb * 32, 0, L.st>>>(s, d, b.prof, b.bmax, b.nz, b.found, b.state,
                                                                    s_begin, ns, s_end, finalize ? 1 : 0);
    LT_CU(cudaGetLastError());
    L.tick();
}

// Degree-0 directions: every profile is a sampled Gaussian exp(-alpha (x_i - c)^2) with
// x_i affine in i, so log|a_i c_{i-sn}| is a concave quadratic in i whose continuous
// maximiser is i* (x* = (alpha c_mu + beta (c_nu + s b)) / (alpha + beta)). The discrete
// maximum over the valid range is at round(i*) clipped to the range, so an 8-point window
// around it, evaluated with the same device arithmetic as the sampled scan, yields the
// scan's maximum (neighbouring products differ by a relative (alpha+beta) h^2 >> ulp).
// A window maximum just below eps (relative 1e-12) is re-checked by a full scan of that
// (s, mu, nu), so the decision equals the exhaustive one. Eight lanes per (s, l, mu, nu);
// the last CTA applies the sequential rule when `finalize`.
__global__ void k_l0_peak(DevSys s, Dir3 d, int* found, int* state, int s_begin, int ns, int s_end, int finalize) {
    // 8 lanes per (s, l, mu, nu): one window point each, max by shuffles within the group
    const Index gtid = static_cast<Index>(blockIdx.x) * blockDim.x + threadIdx.x;
    const Index task = gtid >> 3;
    const int sub = static_cast<int>(threadIdx.x & 7);
    const Index m0 = s.m0;
    const Index per_s = static_cast<Index>(d.nl) * m0 * m0;
    bool valid = task < per_s * ns;
    int sft = 0, l = 0, mu = 0, nu = 0;
    Index base = 0, sn = 0, lo = 0, hi = -1, i0 = 0;
    double h = 1.0;
    if (valid) {
        sft = s_begin + static_cast<int>(task / per_s);
        Index rem = task % per_s;
        l = d.dir[rem / (m0 * m0)];
        rem %= m0 * m0;
        mu = static_cast<int>(rem / m0);
        nu = static_cast<int>(rem % m0);
        const Index n = d.n[l];
        base = (kMaxL0 + 2) * n;
        const Index width = 2 * base;
        sn = static_cast<Index>(sft) * n;
        valid = !__ldcg(&found[sft]) && sn < width;
        if (valid) {
            h = s.b / static_cast<double>(n);
            const double al = s.alpha[mu], be = s.alpha[nu];
            const double xs = (al * s.center[3 * mu + l] + be * (s.center[3 * nu + l] + sft * s.b)) / (al + be);
            const double is = (xs + 0.5 * s.b) / h + static_cast<double>(base) - 0.5;
            lo = sn;
            hi = width - 1;  // j = i - sn >= 0
            const double isc = fmin(fmax(is, static_cast<double>(lo)), static_cast<double>(hi));
            i0 = static_cast<Index>(floor(isc)) - 3;
            i0 = max(lo, min(i0, hi - 7));
        }
    }
    double p = 0.0;
    const Index i = i0 + sub;
    if (valid && i <= hi)
        p = fabs(gto_eval1d(s, mu, l, l0_x(i, base, h, s.b)) * gto_eval1d(s, nu, l, l0_x(i - sn, base, h, s.b)));
    for (int o = 4; o > 0; o >>= 1) p = fmax(p, __shfl_xor_sync(0xffffffffu, p, o));
    if (valid && sub == 0) {
        bool hit = p >= s.eps_ov;
        if (!hit && p >= s.eps_ov * (1.0 - 1e-12))  // at the threshold: exhaustive
            for (Index k = lo; k <= hi && !hit; ++k)
                hit = fabs(gto_eval1d(s, mu, l, l0_x(k, base, h, s.b)) *
                           gto_eval1d(s, nu, l, l0_x(k - sn, base, h, s.b))) >= s.eps_ov;
        if (hit) atomicExch(&found[sft], 1);
    }
    if (!finalize) return;
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&state[4], 1) == static_cast<int>(gridDim.x) - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        l0_finalize(found, state, s_end);
        state[4] = 0;
    }
}

void launch_overlap_peak(const Launch& L, const DevSys& s, const Index* n3, const int* active, OverlapBufs b,
                         int s_begin, int s_end, bool finalize) {
    const Index zero3[3] = {0, 0, 0};
    const Dir3 d = make_dir3(s, n3, zero3, zero3, active);
    const int ns = s_end - s_begin;
    const Index tasks = static_cast<Index>(ns) * d.nl * s.m0 * s.m0;
    const Index blocks = std::max<Index>(1, (8 * tasks + 127) / 128);
    Stage st_(L, "l0_peak");
    k_l0_peak<<<static_cast<unsigned>(blocks), 128, 0, L.st>>>(s, d, b.found, b.state, s_begin, ns, s_end,
                                                              finalize ? 1 : 0);
    LT_CU(cudaGetLastError());
    L.tick();
}

}  // namespace lt
