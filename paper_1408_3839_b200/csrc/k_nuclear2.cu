// k_nuclear2.cu — the nuclear-attraction contraction on FP64 tensor cores (DMMA).
//
// Reference (galerkin.cpp:109-125, :224-247, :273-284):
//   T_l[k,d,r](mu,nu) = sum_i g_mu(i - s_A) g_nu(i - s_B) p_r(i)          (dot3)
//   H_nuc[k,d](mu,nu) = sum_r w_r T_0[.] T_1[.] T_2[.]                    (combine_block)
// Reassociated here so each product is a dense GEMM over the grid:
//   trivial direction (L_l = 1, one (k,d) pair):  T_l[r][e] = sum_i P[r][i] (g_mu g_nu)(i)
//       -> GEMM M = R_tot, N = sym pairs (mu <= nu; T is symmetric in (mu, nu) exactly),
//          K = grid; split-K over CTAs, fixed-order reduction; W[r][e] = w_r prod_l T_l.
//   V[e][i] = sum_r W[r][e] P_l*[r][i]  (rank sum folded into an effective potential)
//       -> GEMM M = m0^2, N = rows, K = R_tot.
//   box chain (one non-trivial direction l*):  N[k][d][e] = sum_j Q_d(j) V_e(j + k n)
//       -> per e a Hankel-operand GEMM M = L cells, N = 2b+1 offsets, K = support.
//   periodic wrapped direction:  Qf_t[d](mu,nu) = sum_j a_mu(t + j n) a_nu(t + (j-d) n)
//       -> per residue t in [0,n) and d >= 0 an (m0 x J)(J x m0) product (m8n8k4 tiles);
//          Qf[-d](nu,mu) = Qf[d](mu,nu) exactly (same terms, same order).
//       single non-trivial direction: N[d][e] = sum_t V_e(t) Qf_t[d](e);
//       several: T_l[d][r][e] = sum_t P_l[r][t] Qf_t[d](e) (GEMM) and
//                N[d0,d1,d2][e] = sum_r W[r][e] prod_l T_l[d_l][r][e] (Khatri-Rao combine).
#include "dmma.cuh"
#include "lt_device.cuh"
#include "lt_internal.cuh"
#include "tma.cuh"

namespace lt {

// symmetric pair index e_s (mu <= nu), row-major over mu: e_s = mu*m0 - mu(mu-1)/2 + (nu - mu)
__device__ __forceinline__ void sym_pair(int es, int m0, int& mu, int& nu) {
    int m = 0, base = 0;
    while (es >= base + (m0 - m)) {
        base += m0 - m;
        ++m;
    }
    mu = m;
    nu = m + (es - base);
}

constexpr int kTrivTK = 32, kTrivStages = 3;

// cp.async of one double into shared memory; src-size 0 (ok = false) writes a zero
__device__ __forceinline__ void cp_async8_zfill(double* dst, const double* src, bool ok) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(ok ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------------------
// trivial-direction tables: split-K DMMA GEMM over the symmetric pairs
// ---------------------------------------------------------------------------
// ASYNC: kTrivStages-deep cp.async pipeline (long K per CTA); else one stage with the next
// stage prefetched in registers (short K, many CTAs per SM)
template <bool ASYNC>
__global__ void __launch_bounds__(256) k_triv_gemm(TrivJobs jobs, int m0, int Rtot, int nsym, int splits,
                                                   double* __restrict__ part) {
    // 32-deep stages, kTrivStages of them in flight through cp.async: potential rows
    // As[st][64][32 + 4], profile rows Gs[st][m0 <= 32][32 + 1]; the product tile
    // Bs[32][64 + 8] (b(k, n) = g_mu(k) g_nu(k)) is formed once per stage by the CTA
    constexpr int TK = kTrivTK, TLA = TK + 4, TLG = TK + 1, TLB = kGBN + 8, NST = ASYNC ? kTrivStages : 1;
    extern __shared__ double tsm_dyn[];
    double* As = tsm_dyn;                      // [NST][kGBM * TLA]
    double* Gs = As + NST * kGBM * TLA;        // [NST][32 * TLG]
    double* Bs = Gs + NST * 32 * TLG;          // [TK * TLB]
    const int job = blockIdx.z / splits, split = blockIdx.z % splits;
    const TrivJob& J = jobs.j[job];
    const int r0 = blockIdx.x * kGBM, e0 = blockIdx.y * kGBN;
    // union of the supports (products vanish outside every pair's overlap): one parallel
    // load per function and a warp reduction instead of a serial chain of m0 loads
    __shared__ long long sk[2];
    __shared__ double tqs[kGBM];    // in-place potential: t_q of each tile row
    __shared__ long long s0s[kGBM];  // and its window start s0[v]
    if (threadIdx.x < 32) {
        long long lo = J.G, hi = 0;
        for (int m = threadIdx.x; m < m0; m += 32) {
            lo = min(lo, static_cast<long long>(J.lo[m]));
            hi = max(hi, static_cast<long long>(J.hi[m]));
        }
        for (int o = 16; o > 0; o >>= 1) {
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (threadIdx.x == 0) {
            sk[0] = lo;
            sk[1] = hi;
        }
    }
    if (threadIdx.x < kGBM) {
        const int r = r0 + static_cast<int>(threadIdx.x);
        if (!J.pot && r < Rtot) {
            tqs[threadIdx.x] = sinc_node(r % J.RN, J.M);
            s0s[threadIdx.x] = J.s0[r / J.RN];
        }
    }
    __syncthreads();
    const long long klo = sk[0];
    const long long khi = min(sk[1], static_cast<long long>(J.rows));
    const long long len = khi > klo ? khi - klo : 0;
    const long long per = ((len + splits - 1) / splits + TK - 1) / TK * TK;
    const long long k0 = klo + split * per, k1 = min(khi, k0 + per);
    const double* P = J.pot;
    const double* g = J.pwc;
    const long long G = J.G, rows = J.rows;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wm = warp & 3, wn = warp >> 2, gg = lane >> 2, tq = lane & 3;
    // product-tile column of this thread (fixed): pair (pmu, pnu) of column bn, rows bk0 + 4u
    const int bn = tid & 63, bk0 = tid >> 6;
    const bool bok = e0 + bn < nsym;
    int pmu = 0, pnu = 0;
    if (bok) sym_pair(e0 + bn, m0, pmu, pnu);
    double acc[4][4] = {};
    if constexpr (ASYNC) {
    // stage kb into buffer st: 8-byte cp.async copies, zero-filled outside the tile
    auto issue = [&](long long kb, int st) {
        double* as = As + st * kGBM * TLA;
        double* gs = Gs + st * 32 * TLG;
        if (kb < k1) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = tid + 256 * u;
                const int am = e >> 5, ak = e & 31;  // k fastest: contiguous rows of P
                const long long k = kb + ak;
                const bool ok = k < k1 && r0 + am < Rtot;
                cp_async8_zfill(as + am * TLA + ak, ok ? P + (r0 + am) * rows + k : P, ok);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e = tid + 256 * u;
                const int gm = e >> 5, gk = e & 31;
                const long long k = kb + gk;
                const bool ok = gm < m0 && k < k1;
                cp_async8_zfill(gs + gm * TLG + gk, ok ? g + gm * G + k : g, ok);
            }
        }
        cp_async_commit();
    };
    if (k0 < k1) {
#pragma unroll
        for (int st = 0; st < NST - 1; ++st) issue(k0 + st * TK, st);
        int it = 0;
        for (long long kb = k0; kb < k1; kb += TK, ++it) {
            const int st = it % NST;
            cp_async_wait<NST - 2>();  // this thread's copies of stage `it` have landed
            __syncthreads();           // everyone's copies; every warp is past the MMAs of it - 1
            issue(kb + (NST - 1) * TK, (it + NST - 1) % NST);
            const double* as = As + st * kGBM * TLA;
            const double* gs = Gs + st * 32 * TLG;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int k = bk0 + 4 * u;
                Bs[k * TLB + bn] = bok ? gs[pmu * TLG + k] * gs[pnu * TLG + k] : 0.0;
            }
            __syncthreads();
#pragma unroll
            for (int ks = 0; ks < TK; ks += 4) {
                const double a0 = as[(wm * 16 + gg) * TLA + ks + tq];
                const double a1 = as[(wm * 16 + gg + 8) * TLA + ks + tq];
#pragma unroll
                for (int nt = 0; nt < 4; ++nt)
                    dmma_m16n8k4(acc[nt], a0, a1, Bs[(ks + tq) * TLB + wn * 32 + nt * 8 + gg]);
            }
        }
        cp_async_wait<0>();
    }
    } else {
    double ra[8], rg[4];
    auto fetch = [&](long long kb) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = tid + 256 * u;
            const int am = e >> 5, ak = e & 31;  // k fastest: contiguous rows of P
            const long long k = kb + ak;
            double v = 0.0;
            if (k < k1 && r0 + am < Rtot)
                v = P ? P[(r0 + am) * rows + k] : master_cell(s0s[am] + k, J.mrows, J.h, tqs[am]);
            ra[u] = v;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = tid + 256 * u;
            const int gm = e >> 5, gk = e & 31;
            const long long k = kb + gk;
            rg[u] = (gm < m0 && k < k1) ? g[gm * G + k] : 0.0;
        }
    };
    if (k0 < k1) {
        fetch(k0);
        for (long long kb = k0; kb < k1; kb += TK) {
            __syncthreads();
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = tid + 256 * u;
                As[(e >> 5) * TLA + (e & 31)] = ra[u];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e = tid + 256 * u;
                Gs[(e >> 5) * TLG + (e & 31)] = rg[u];
            }
            __syncthreads();
            if (kb + TK < k1) fetch(kb + TK);  // next stage's loads overlap the products and MMAs
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int k = bk0 + 4 * u;
                Bs[k * TLB + bn] = bok ? Gs[pmu * TLG + k] * Gs[pnu * TLG + k] : 0.0;
            }
            __syncthreads();
#pragma unroll
            for (int ks = 0; ks < TK; ks += 4) {
                const double a0 = As[(wm * 16 + gg) * TLA + ks + tq];
                const double a1 = As[(wm * 16 + gg + 8) * TLA + ks + tq];
#pragma unroll
                for (int nt = 0; nt < 4; ++nt)
                    dmma_m16n8k4(acc[nt], a0, a1, Bs[(ks + tq) * TLB + wn * 32 + nt * 8 + gg]);
            }
        }
    }
    }
    double* out = part + (static_cast<long long>(job) * splits + split) * Rtot * nsym;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            int m, n;
            acc_coord(nt, i, m, n);
            if (r0 + m < Rtot && e0 + n < nsym) out[(r0 + m) * nsym + e0 + n] = acc[nt][i];
        }
}

// W[r][e] = w_r * prod over trivial directions of T_l[r][e] (T_l reduced over splits in
// fixed order); e over all m0^2 ordered pairs (mirror of the symmetric index)
__device__ __forceinline__ void triv_finish(const double (&tj)[3], int njobs, const WSpec& ws, int m0, int Rtot, int r,
                                            int mu, int nu, const double* __restrict__ potw, double* __restrict__ W,
                                            double* __restrict__ Tout) {
    const int mm = m0 * m0;
    double prod = 1.0;  // product in direction order (directions may share a job)
    bool first = true;
    for (int l = 0; l < 3; ++l) {
        if (ws.job_of_dir[l] < 0) continue;
        const double v = ws.job_of_dir[l] == 0 ? tj[0] : (ws.job_of_dir[l] == 1 ? tj[1] : tj[2]);
        prod = first ? v : prod * v;
        first = false;
    }
    const double wv = potw[r] * prod;
    W[r * mm + mu + nu * m0] = wv;
    W[r * mm + nu + mu * m0] = wv;
    if (Tout)
        for (int j = 0; j < njobs; ++j) {
            const double v = j == 0 ? tj[0] : (j == 1 ? tj[1] : tj[2]);
            Tout[(static_cast<long long>(j) * Rtot + r) * mm + mu + nu * m0] = v;
            Tout[(static_cast<long long>(j) * Rtot + r) * mm + nu + mu * m0] = v;
        }
}

// few outputs, many splits: one warp per (r, symmetric pair), lanes over the splits
__global__ void k_triv_reduce_w_warp(const double* __restrict__ part, int njobs, WSpec ws, int m0, int Rtot, int nsym,
                                     int splits, const double* __restrict__ potw, double* __restrict__ W,
                                     double* __restrict__ Tout) {
    const int lane = threadIdx.x & 31;
    const long long wid = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (wid >= static_cast<long long>(Rtot) * nsym) return;
    const int r = static_cast<int>(wid / nsym), es = static_cast<int>(wid % nsym);
    int mu, nu;
    sym_pair(es, m0, mu, nu);
    double tj[3] = {1.0, 1.0, 1.0};
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        if (j >= njobs) break;
        double sacc = 0.0;
        for (int sp = lane; sp < splits; sp += 32)
            sacc += part[((static_cast<long long>(j) * splits + sp) * Rtot + r) * nsym + es];
        tj[j] = __shfl_sync(0xffffffffu, warp_sum(sacc), 0);
    }
    if (lane == 0) triv_finish(tj, njobs, ws, m0, Rtot, r, mu, nu, potw, W, Tout);
}

// many outputs: one thread per (r, symmetric pair), consecutive threads over consecutive
// pairs (each split row read coalesced), four partial sums over the splits
__global__ void k_triv_reduce_w(const double* __restrict__ part, int njobs, WSpec ws, int m0, int Rtot, int nsym,
                                int splits, const double* __restrict__ potw, double* __restrict__ W,
                                double* __restrict__ Tout) {
    const long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= static_cast<long long>(Rtot) * nsym) return;
    const int r = static_cast<int>(tid / nsym), es = static_cast<int>(tid % nsym);
    int mu, nu;
    sym_pair(es, m0, mu, nu);
    double tj[3] = {1.0, 1.0, 1.0};
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        if (j >= njobs) break;
        const double* pj = part + (static_cast<long long>(j) * splits * Rtot + r) * nsym + es;
        const long long stride = static_cast<long long>(Rtot) * nsym;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int sp = 0;
        for (; sp + 3 < splits; sp += 4) {
            s0 += pj[(sp + 0) * stride];
            s1 += pj[(sp + 1) * stride];
            s2 += pj[(sp + 2) * stride];
            s3 += pj[(sp + 3) * stride];
        }
        for (; sp < splits; ++sp) s0 += pj[sp * stride];
        tj[j] = (s0 + s1) + (s2 + s3);
    }
    triv_finish(tj, njobs, ws, m0, Rtot, r, mu, nu, potw, W, Tout);
}

void launch_triv_tables(const Launch& L, const TrivJobs& jobs, int njobs, const WSpec& ws, int m0, int Rtot,
                        const double* potw, double* part, int splits, double* W, double* Tout, bool async) {
    const int nsym = m0 * (m0 + 1) / 2;
    if (njobs > 0) {
        dim3 grid((Rtot + kGBM - 1) / kGBM, (nsym + kGBN - 1) / kGBN, njobs * splits);
        auto smem_of = [](int nst) {
            return static_cast<int>(sizeof(double)) *
                   (nst * (kGBM * (kTrivTK + 4) + 32 * (kTrivTK + 1)) + kTrivTK * (kGBN + 8));
        };
        static bool attr = false;
        if (!attr) {
            LT_CU(cudaFuncSetAttribute(k_triv_gemm<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       smem_of(kTrivStages)));
            attr = true;
        }
        Stage st_(L, "triv_gemm");
        if (async) {
            k_triv_gemm<true><<<grid, 256, smem_of(kTrivStages), L.st>>>(jobs, m0, Rtot, nsym, splits, part);
        } else {
            k_triv_gemm<false><<<grid, 256, smem_of(1), L.st>>>(jobs, m0, Rtot, nsym, splits, part);
        }
        LT_CU(cudaGetLastError());
        L.tick();
    }
    const long long outs = static_cast<long long>(Rtot) * nsym;
    Stage st2_(L, "triv_reduce_w");
    if (outs < 8192)
        k_triv_reduce_w_warp<<<static_cast<unsigned>((outs + 7) / 8), 256, 0, L.st>>>(part, njobs, ws, m0, Rtot, nsym,
                                                                                      splits, potw, W, Tout);
    else
        k_triv_reduce_w<<<static_cast<unsigned>((outs + 127) / 128), 128, 0, L.st>>>(part, njobs, ws, m0, Rtot, nsym,
                                                                                   splits, potw, W, Tout);
    LT_CU(cudaGetLastError());
    L.tick();
}

// ---------------------------------------------------------------------------
// V[e][i] = sum_r W[r][e] P[r][i]
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_vgemm(int mm, int Rtot, long long rows, const double* __restrict__ W,
                                               const double* __restrict__ P, double* __restrict__ V) {
    __shared__ GemmSmem sm;
    const int e0 = blockIdx.y * kGBM;
    const long long i0 = static_cast<long long>(blockIdx.x) * kGBN;
    auto loadA = [&](int m, long long k) -> double { return e0 + m < mm ? W[k * mm + e0 + m] : 0.0; };
    auto loadB = [&](long long k, int n) -> double { return i0 + n < rows ? P[k * rows + i0 + n] : 0.0; };
    double acc[4][4] = {};
    cta_gemm_64x64(loadA, loadB, 0, Rtot, acc, sm);
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            int m, n;
            acc_coord(nt, i, m, n);
            if (e0 + m < mm && i0 + n < rows) V[(e0 + m) * rows + i0 + n] = acc[nt][i];
        }
}

// V[e][t] = sum_r W[r][e] P[r][t] for a periodic cell panel (rows = n residues): four
// lanes per (e, t) split the rank sum (r = lane4, lane4 + 4, ...), combined by shuffles;
// lanes of a warp cover 8 consecutive e (coalesced W reads, P broadcast)
__global__ void k_vdot(int mm, int Rtot, long long rows, const double* __restrict__ W, const double* __restrict__ P,
                       double* __restrict__ V) {
    const long long gid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int part = static_cast<int>(gid & 3);
    const long long idx = gid >> 2;
    const bool ok = idx < static_cast<long long>(mm) * rows;
    const int e = static_cast<int>(idx % mm);
    const long long t = idx / mm;
    double v = 0.0;
    if (ok) {
        // eight (W, P) pairs in flight per round trip; the sum stays in r order
        int r = part;
        for (; r + 28 < Rtot; r += 32) {
            double w[8], p[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                w[u] = W[(r + 4 * u) * mm + e];
                p[u] = P[(r + 4 * u) * rows + t];
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) v = fma(w[u], p[u], v);
        }
        for (; r < Rtot; r += 4) v = fma(W[r * mm + e], P[r * rows + t], v);
    }
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    if (ok && part == 0) V[static_cast<long long>(e) * rows + t] = v;
}

void launch_vdot(const Launch& L, int mm, int Rtot, long long rows, const double* W, const double* P, double* V) {
    const long long tot = 4LL * mm * rows;
    Stage st_(L, "vgemm");
    k_vdot<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, L.st>>>(mm, Rtot, rows, W, P, V);
    LT_CU(cudaGetLastError());
    L.tick();
}

void launch_vgemm(const Launch& L, int mm, int Rtot, long long rows, const double* W, const double* P, double* V) {
    dim3 grid(static_cast<unsigned>((rows + kGBN - 1) / kGBN), (mm + kGBM - 1) / kGBM);
    Stage st_(L, "vgemm");
    k_vgemm<<<grid, 256, 0, L.st>>>(mm, Rtot, rows, W, P, V);
    LT_CU(cudaGetLastError());
    L.tick();
}

// ---------------------------------------------------------------------------
// box chain: per pair e, C[k][d] = sum_j Q_d(j) V_e(j + k n)   (Hankel A operand)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_hankel(int m0, long long Lc, long long n, int band, long long G,
                                                const double* __restrict__ pwc,
                                                const unsigned long long* __restrict__ plo,
                                                const unsigned long long* __restrict__ phi,
                                                const double* __restrict__ V, double* __restrict__ part, int splits) {
    __shared__ GemmSmem sm;
    const int width = 2 * band + 1;
    const int nkt = static_cast<int>((Lc + kGBM - 1) / kGBM);
    const int kt = blockIdx.x % nkt, dt = blockIdx.x / nkt;
    const int e = blockIdx.y;
    const int split = blockIdx.z;
    const int mu = e % m0, nu = e / m0;
    const long long k0c = static_cast<long long>(kt) * kGBM;
    const int d0 = dt * kGBN;  // offset index (d + band)
    const long long alo = static_cast<long long>(plo[mu]), ahi = static_cast<long long>(phi[mu]);
    const long long blo = static_cast<long long>(plo[nu]), bhi = static_cast<long long>(phi[nu]);
    const long long dmin = d0 - band, dmax = min(d0 + kGBN, width) - 1 - band;
    const long long jlo = max(alo, blo + dmin * n), jhi = min(ahi, bhi + dmax * n);
    const long long len = jhi > jlo ? jhi - jlo : 0;
    const long long per = ((len + splits - 1) / splits + kGBK - 1) / kGBK * kGBK;
    const long long j0 = jlo + split * per, j1 = min(jhi, j0 + per);
    const double* a = pwc + mu * G;
    const double* b = pwc + nu * G;
    const double* v = V + static_cast<long long>(e) * G;
    auto loadA = [&](int m, long long j) -> double {
        const long long kc = k0c + m;
        const long long gi = j + kc * n;
        return (kc < Lc && gi < G) ? v[gi] : 0.0;
    };
    auto loadB = [&](long long j, int nn) -> double {
        const int di = d0 + nn;
        if (di >= width) return 0.0;
        const long long jb = j - static_cast<long long>(di - band) * n;
        return (j >= alo && j < ahi && jb >= blo && jb < bhi) ? a[j] * b[jb] : 0.0;
    };
    double acc[4][4] = {};
    cta_gemm_64x64(loadA, loadB, j0, j1, acc, sm);
    double* out = part + (static_cast<long long>(split) * m0 * m0 + e) * Lc * width;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            int m, nn;
            acc_coord(nt, i, m, nn);
            if (k0c + m < Lc && d0 + nn < width) out[(k0c + m) * width + d0 + nn] = acc[nt][i];
        }
}

// The same product with the operands RESIDENT in shared memory. As per-stage tiles,
// A(k, j) = V_e[j + k n] re-reads every element of V_e once per cell k (128-fold at c3; measured:
// tile loads by TMA boxes or by plain loads both run at the L2 -> SM rate, 141-145 us at c3).
// Here a CTA loads the part of V_e its (cell tile, j range) touches ONCE, as the row-major
// [rows][n] reshaping of the vector: n / 16 TMA box loads (cp.async.bulk.tensor, SWIZZLE_128B
// boxes of 16 columns x RV rows) through a tensor map of pitch n over the flat array, and the
// same for the Toeplitz view of the profile b_nu (rows reversed so the pitch is positive):
//   A(k, jj)   = Vt[k + jj / n][jj % n]            Vt[r][c] = V_e[jA + (k0 + r) n + c]
//   B(rho, jj) = bt[rho - rho0 + jj / n][jj % n]   bt[r][c] = b_nu[jA + (rho0 + r - band) n + c]
// times a_mu[jA + jj] (a plain shared array) in registers; rho = width - 1 - (d + band). Every
// DMMA fragment is a conflict-free read of a swizzled box; no barrier inside the j loop.
// Elements a view reads outside [0, G) of its function (the next pair's V, a neighbouring
// profile, the slack the caller leaves around the arrays) are masked by per-thread j limits.
// CTA = 8 warps, warp w owns cells 16 w .. 16 w + 15 of the 128-cell tile and NBLK 8-offset
// blocks; a CTA covers a fixed quota of `per` grid points of one pair's support overlap.
namespace {
constexpr int kHkM = 128, kHkN = 64;
struct HankelShape {
    int per_max = 0;    // j quota of one CTA (multiple of 16)
    int RV = 0, RB = 0; // box rows of the V and profile tiles (multiples of 8, <= 256)
    size_t smem = 0;    // bytes (incl. 1 KB alignment slack)
};
// shared-memory plan for row length n, `live` offsets per tile; per_max = 0 when nothing fits
HankelShape hankel_shape(long long n, int live) {
    HankelShape h;
    if (n % 16 != 0 || n > 1024) return h;
    const int nblk = (live + 7) / 8;
    // the longest quota with two CTAs per SM (<= 110 KB each), else the longest that fits one
    for (const size_t cap : {110u * 1024u, 200u * 1024u})
        for (const int per : {640, 512, 384, 256, 128}) {
            const long long RV = (kHkM + (per + n - 1) / n + 1 + 7) / 8 * 8;
            const long long RB = (8 * nblk + (per + n - 1) / n + 1 + 7) / 8 * 8;
            const size_t bytes = sizeof(double) * static_cast<size_t>((RV + RB) * n + per + 24) + 1024 + 64;
            if (RV <= 256 && RB <= 256 && bytes <= cap) {
                h.per_max = per;
                h.RV = static_cast<int>(RV);
                h.RB = static_cast<int>(RB);
                h.smem = bytes;
                return h;
            }
        }
    return h;
}
}  // namespace

#ifdef LT_HK_PROF
__device__ unsigned long long lt_hk_prof[8];
extern "C" void lt_debug_hk_prof(unsigned long long* out) {
    cudaMemcpyFromSymbol(out, lt_hk_prof, sizeof(lt_hk_prof));
    unsigned long long z[8] = {};
    cudaMemcpyToSymbol(lt_hk_prof, z, sizeof(z));
}
#endif
template <int NBLK>  // live 8-offset blocks of the tile, ceil(live / 8)
__global__ void __launch_bounds__(256) k_hankel_res(const __grid_constant__ CUtensorMap tv,
                                                    const __grid_constant__ CUtensorMap tb, int m0, long long Lc, int n,
                                                    int band, long long G, const double* __restrict__ pwc,
                                                    const unsigned long long* __restrict__ plo,
                                                    const unsigned long long* __restrict__ phi,
                                                    double* __restrict__ part, int per, int RV, int RB) {
    extern __shared__ __align__(1024) unsigned char hk_raw[];
    double* hk_sm = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(hk_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    __shared__ uint64_t bar;
    const int width = 2 * band + 1;
    const int nkt = static_cast<int>((Lc + kHkM - 1) / kHkM);
    const int kt = blockIdx.x % nkt, dt = blockIdx.x / nkt;
    const int e = blockIdx.y, split = blockIdx.z;
    const int mu = e % m0, nu = e / m0;
    const long long k0c = static_cast<long long>(kt) * kHkM;
    const int rho0 = dt * kHkN;
    const int live = min(kHkN, width - rho0);
    const long long dmax = width - 1 - rho0 - band, dmin = width - 1 - (rho0 + live - 1) - band;
    const long long alo = static_cast<long long>(plo[mu]), ahi = static_cast<long long>(phi[mu]);
    const long long blo = static_cast<long long>(plo[nu]), bhi = static_cast<long long>(phi[nu]);
    const long long jlo = max(alo, blo + dmin * n), jhi = min(ahi, bhi + dmax * n);
    // fixed quota of `per` grid points per CTA: a pair with a long support overlap takes more
    // CTAs (splits = ceil(G / per) slots exist; the unused ones only write zeros)
    const long long j0 = jlo + static_cast<long long>(split) * per, j1 = min(jhi, j0 + per);
    const long long jA = j0 & ~1LL;  // box columns start on 16-byte boundaries
    const int Lj = j1 > j0 ? static_cast<int>(j1 - jA) : 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int nbox = n / 16;
    double* Vs = hk_sm;                                      // [nbox][RV][16] swizzled
    double* bs = Vs + static_cast<size_t>(nbox) * RV * 16;   // [nbox][RB][16] swizzled
    double* as = bs + static_cast<size_t>(nbox) * RB * 16;   // [per + 24]
    double acc[NBLK][4];
#pragma unroll
    for (int j = 0; j < NBLK; ++j)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[j][q] = 0.0;
#ifdef LT_HK_PROF
    const long long tp0 = clock64();
    long long tp1 = tp0;
#endif
    if (Lj > 0) {
        if (threadIdx.x == 0) {
            mbar_init(&bar, 1);
            mbar_fence_init();
            mbar_arrive_expect_tx(&bar, static_cast<unsigned>((RV + RB) * n * 8));
            for (int b = 0; b < nbox; ++b) {
                tma_load_2d(Vs + static_cast<size_t>(b) * RV * 16, &tv, &bar, static_cast<int>(e * G + jA + 16 * b),
                            static_cast<int>(k0c));
                tma_load_2d(bs + static_cast<size_t>(b) * RB * 16, &tb, &bar, static_cast<int>(nu * G + jA + 16 * b), rho0);
            }
        }
        {
            const double* am = pwc + static_cast<long long>(mu) * G;
            for (int x = threadIdx.x; x < Lj + 16; x += 256) {
                const long long j = jA + x;
                as[x] = (j >= j0 && j < j1) ? am[j] : 0.0;  // trims the range to [j0, j1); zero tail
            }
        }
        __syncthreads();  // the barrier is initialised, as[] written
        mbar_wait(&bar, 0);
#ifdef LT_HK_PROF
        tp1 = clock64();
#endif
        if (k0c + warp * 16 < Lc) {
            // per-thread j limits (relative to jA) inside which the views read their own function
            auto clampi = [](long long v) { return static_cast<int>(max(-(1LL << 30), min(1LL << 30, v))); };
            const int rA = warp * 16 + g;
            const int limA0 = clampi(G - jA - (k0c + rA) * n), limA1 = clampi(G - jA - (k0c + rA + 8) * n);
            int loB[NBLK], hiB[NBLK];
#pragma unroll
            for (int jn = 0; jn < NBLK; ++jn) {
                const long long o = jA + static_cast<long long>(rho0 + jn * 8 + g - band) * n;  // b index at jj = 0
                loB[jn] = clampi(-o);
                hiB[jn] = clampi(G - o);
            }
            const int nrow = (Lj + n - 1) / n;
            for (int row = 0; row < nrow; ++row) {
                const int rsw = (g + row) & 7;  // the swizzle row phase, common to the A and B rows
                int off[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) off[q] = ((((4 * q + t) >> 1) ^ rsw) << 1) + (t & 1);
                const double* pa = Vs + (rA + row) * 16;
                const double* pb = bs + (g + row) * 16;
                const int xe = min(n, Lj - row * n);
                for (int xb = 0; xb * 16 < xe; ++xb) {
                    const double* pab = pa + static_cast<size_t>(xb) * RV * 16;
                    const double* pbb = pb + static_cast<size_t>(xb) * RB * 16;
                    const int jj0 = row * n + xb * 16 + t;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int jj = jj0 + 4 * q;
                        const double aj = as[jj];  // zero outside [j0, j1)
                        const double a0 = jj < limA0 ? pab[off[q]] : 0.0;
                        const double a1 = jj < limA1 ? pab[off[q] + 128] : 0.0;
#pragma unroll
                        for (int jn = 0; jn < NBLK; ++jn) {
                            const double b0 = (jj >= loB[jn] && jj < hiB[jn]) ? pbb[off[q] + jn * 128] * aj : 0.0;
                            dmma_m16n8k4(acc[jn], a0, a1, b0);
                        }
                    }
                }
            }
        }
    }
#ifdef LT_HK_PROF
    if (threadIdx.x == 0 && Lj > 0) {
        const long long tp2 = clock64();
        atomicAdd(&lt_hk_prof[0], static_cast<unsigned long long>(tp1 - tp0));
        atomicAdd(&lt_hk_prof[1], static_cast<unsigned long long>(tp2 - tp1));
        atomicAdd(&lt_hk_prof[2], 1ull);
        atomicAdd(&lt_hk_prof[3], static_cast<unsigned long long>(Lj));
        atomicMax(&lt_hk_prof[4], static_cast<unsigned long long>(tp2 - tp0));
    }
#endif
    if (k0c + warp * 16 >= Lc) return;
    if (Lj == 0 && width <= kHkN) return;  // an unused quota slot: k_split_reduce_quota skips it
    double* out = part + (static_cast<long long>(split) * m0 * m0 + e) * Lc * width;
#pragma unroll
    for (int jn = 0; jn < NBLK; ++jn)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const long long kc = k0c + warp * 16 + g + 8 * (q >> 1);
            const int rl = jn * 8 + 2 * t + (q & 1);
            const int di = width - 1 - rho0 - rl;
            if (kc < Lc && rl < live) out[kc * width + di] = acc[jn][q];
        }
}

// splits the resident kernel needs so that a CTA's j range fits its shared-memory plan (0: the
// shape does not fit, the tile-loading k_hankel runs with the caller's splits)
int hankel_res_splits(const DirPlan& d) {
    if (d.L < 32) return 0;  // few cells: the 64-row tile kernel wastes less
    const HankelShape h = hankel_shape(d.n, static_cast<int>(std::min<Index>(kHkN, d.width)));
    if (h.per_max == 0) return 0;
    return static_cast<int>((d.G + h.per_max - 1) / h.per_max);
}

// N[(k*width + d)][e] = sum_split part[split][e][k][d]
__global__ void k_split_reduce(long long mm, long long kd, int splits, const double* __restrict__ part,
                               double* __restrict__ N) {
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= mm * kd) return;
    const long long e = idx % mm, q = idx / mm;
    double s = 0.0;
    for (int sp = 0; sp < splits; ++sp) s += part[(sp * mm + e) * kd + q];
    N[idx] = s;
}

// splits: hankel_res_splits(d) when that is non-zero (the resident kernel), else the caller's.
// padded: band * n doubles of slack lie on both sides of pwc and L * n behind V (the TMA views
// of the resident kernel touch them; their contents are never used).
// the same for the resident kernel with one offset tile (width <= 64): pair e filled the first
// ceil(len_e / per) quota slots (k_hankel_res's own range arithmetic), the rest were not written
__global__ void k_split_reduce_quota(int m0, long long mm, long long kd, int splits, int per, long long n, int band,
                                     const unsigned long long* __restrict__ plo,
                                     const unsigned long long* __restrict__ phi, const double* __restrict__ part,
                                     double* __restrict__ N) {
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= mm * kd) return;
    const long long e = idx % mm, q = idx / mm;
    const int mu = static_cast<int>(e % m0), nu = static_cast<int>(e / m0);
    const long long alo = static_cast<long long>(plo[mu]), ahi = static_cast<long long>(phi[mu]);
    const long long blo = static_cast<long long>(plo[nu]), bhi = static_cast<long long>(phi[nu]);
    const long long jlo = max(alo, blo - band * n), jhi = min(ahi, bhi + band * n);
    const long long len = jhi > jlo ? jhi - jlo : 0;
    const int used = static_cast<int>(min(static_cast<long long>(splits), (len + per - 1) / per));
    double s = 0.0;
    for (int sp = 0; sp < used; ++sp) s += part[(sp * mm + e) * kd + q];
    N[idx] = s;
}

void launch_hankel(const Launch& L, int m0, const DirPlan& d, const double* pwc, const unsigned long long* lo,
                   const unsigned long long* hi, const double* V, double* part, double* N, int splits, bool padded) {
    const long long mm = m0 * m0, kd = d.L * d.width;
    const int rs = padded ? hankel_res_splits(d) : 0;
    const HankelShape h = hankel_shape(d.n, static_cast<int>(std::min<Index>(kHkN, d.width)));
    CUtensorMap tv, tb;
    bool res = rs > 0 && rs == splits && mm * d.G + d.G < (1LL << 31);
    // V as rows of pitch n over the flat array (row k, column e G + j -> V_e[j + k n]); the
    // profiles as rows of pitch n starting band n before pwc (row rho, column nu G + j)
    if (res)
        res = tma_try_map_2d(&tv, V, d.L + h.RV, mm * d.G, d.n, h.RV) &&
              tma_try_map_2d(&tb, pwc - d.band * d.n, d.width + h.RB, static_cast<long long>(m0) * d.G, d.n, h.RB);
    if (res) {
        const int nkt = static_cast<int>((d.L + kHkM - 1) / kHkM);
        const int ndt = static_cast<int>((d.width + kHkN - 1) / kHkN);
        dim3 grid(nkt * ndt, m0 * m0, splits);
        Stage st_(L, "hankel_gemm");
        // every offset tile of a launch runs the same instantiation: the block count of the
        // fullest tile (tiles with fewer live offsets compute on masked rows)
        const int nblk = static_cast<int>((std::min<Index>(kHkN, d.width) + 7) / 8);
        auto run = [&](auto kern) {
            static size_t attr = 0;
            if (h.smem > attr) {
                LT_CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(h.smem)));
                attr = h.smem;
            }
            kern<<<grid, 256, h.smem, L.st>>>(tv, tb, m0, d.L, static_cast<int>(d.n), static_cast<int>(d.band), d.G, pwc, lo,
                                              hi, part, h.per_max, h.RV, h.RB);
        };
        switch (nblk) {
            case 1: run(k_hankel_res<1>); break;
            case 2: run(k_hankel_res<2>); break;
            case 3: run(k_hankel_res<3>); break;
            case 4: run(k_hankel_res<4>); break;
            case 5: run(k_hankel_res<5>); break;
            case 6: run(k_hankel_res<6>); break;
            case 7: run(k_hankel_res<7>); break;
            default: run(k_hankel_res<8>); break;
        }
        LT_CU(cudaGetLastError());
    } else {
        const int nkt = static_cast<int>((d.L + kGBM - 1) / kGBM);
        const int ndt = static_cast<int>((d.width + kGBN - 1) / kGBN);
        dim3 grid(nkt * ndt, m0 * m0, splits);
        Stage st_(L, "hankel_gemm");
        k_hankel<<<grid, 256, 0, L.st>>>(m0, d.L, d.n, static_cast<int>(d.band), d.G, pwc, lo, hi, V, part, splits);
        LT_CU(cudaGetLastError());
    }
    Stage st2_(L, "split_reduce");
    if (res && d.width <= kHkN)
        k_split_reduce_quota<<<static_cast<unsigned>((mm * kd + 255) / 256), 256, 0, L.st>>>(
            m0, mm, kd, splits, h.per_max, d.n, static_cast<int>(d.band), lo, hi, part, N);
    else
        k_split_reduce<<<static_cast<unsigned>((mm * kd + 255) / 256), 256, 0, L.st>>>(mm, kd, splits, part, N);
    LT_CU(cudaGetLastError());
    L.tick(2);
}

// ---------------------------------------------------------------------------
// several wrapped directions: T[d][e][r] = sum_t P[r][t] Qf[d][e][t] (d >= 0), DMMA GEMM
// ---------------------------------------------------------------------------
constexpr int kFgemmK = 64;          // K (residues per cell) staged whole up to this
constexpr int kFgemmLDA = kFgemmK + 4;  // conflict-free m16n8k4 fragment reads
constexpr int kFgemmLDB = 64 + 8;
__global__ void __launch_bounds__(256) k_fgemm(int mm, int Rtot, long long n, int ncols, const double* __restrict__ P,
                                               const double* __restrict__ Qf, double* __restrict__ T) {
    const int r0 = blockIdx.y * kGBM;
    const int c0 = blockIdx.x * kGBN;  // column = d*mm + e
    double acc[4][4] = {};
    if (n <= kFgemmK) {
        // the whole K range at once (one load latency instead of one per 16-deep stage):
        // A[m][k] = P[r0+m][k], B[k][nn] = Qf[k][c0+nn] (Qf layout [t][d][e], k_resfold)
        extern __shared__ double fsm[];
        double* As = fsm;                  // [64][kFgemmLDA]
        double* Bs = fsm + kGBM * kFgemmLDA;  // [kFgemmK][kFgemmLDB]
        const int K = static_cast<int>(n);
        {
            // every element load in flight before the first store (16 + 16 per thread)
            constexpr int kPer = kGBM * kFgemmK / 256;
            double va[kPer], vb[kPer];
#pragma unroll
            for (int u = 0; u < kPer; ++u) {
                const int e = threadIdx.x + 256 * u;
                const int m = e / kFgemmK, k = e % kFgemmK;  // A: k fastest
                va[u] = (k < K && r0 + m < Rtot) ? P[static_cast<long long>(r0 + m) * n + k] : 0.0;
                const int kb = e / kGBN, nn = e % kGBN;      // B: n fastest
                vb[u] = (kb < K && c0 + nn < ncols) ? Qf[static_cast<long long>(kb) * ncols + c0 + nn] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kPer; ++u) {
                const int e = threadIdx.x + 256 * u;
                As[(e / kFgemmK) * kFgemmLDA + e % kFgemmK] = va[u];
                Bs[(e / kGBN) * kFgemmLDB + e % kGBN] = vb[u];
            }
        }
        const int Kp = (K + 3) & ~3;  // columns K .. Kp-1 were loaded as zeros
        __syncthreads();
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        const int wm = warp & 3, wn = warp >> 2;
        const int g = lane >> 2, t = lane & 3;
        for (int ks = 0; ks < Kp; ks += 4) {
            const double a0 = As[(wm * 16 + g) * kFgemmLDA + ks + t];
            const double a1 = As[(wm * 16 + g + 8) * kFgemmLDA + ks + t];
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) dmma_m16n8k4(acc[nt], a0, a1, Bs[(ks + t) * kFgemmLDB + wn * 32 + nt * 8 + g]);
        }
    } else {
        __shared__ GemmSmem sm;
        auto loadA = [&](int m, long long k) -> double { return r0 + m < Rtot ? P[(r0 + m) * n + k] : 0.0; };
        auto loadB = [&](long long k, int nn) -> double { return c0 + nn < ncols ? Qf[k * ncols + c0 + nn] : 0.0; };
        cta_gemm_64x64(loadA, loadB, 0, n, acc, sm);
    }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            int m, nn;
            acc_coord(nt, i, m, nn);
            if (r0 + m < Rtot && c0 + nn < ncols) {
                const int col = c0 + nn;
                const int dd = col / mm, e = col % mm;
                T[(static_cast<long long>(dd) * mm + e) * Rtot + r0 + m] = acc[nt][i];  // [d][e][r]
            }
        }
}

// K <= kFgemmK (residues per cell): 32 x 32 output tiles on 128 threads (4 warps of 16 x 16),
// the whole K staged at once. At c5 (Rtot ~ 100, 7 x 64 columns) the 64 x 64 tiles make only
// 14 CTAs, each walking 64 x 64 x K on DMMA; the quarter tiles spread the same work over 4x
// the SMs and finish in roughly a quarter of the time.
constexpr int kFsBM = 32, kFsBN = 32;
constexpr int kFsLDA = kFgemmK + 4;  // conflict-free m16n8k4 A-fragment reads
constexpr int kFsLDB = kFsBN + 8;    // conflict-free B-fragment reads
__global__ void __launch_bounds__(128) k_fgemm_s(int mm, int Rtot, int K, int ncols, const double* __restrict__ P,
                                                 const double* __restrict__ Qf, double* __restrict__ T) {
    __shared__ double As[kFsBM * kFsLDA];    // [m][k]
    __shared__ double Bs[kFgemmK * kFsLDB];  // [k][n]
    const int r0 = blockIdx.y * kFsBM;
    const int c0 = blockIdx.x * kFsBN;
    {
        constexpr int kPer = kFsBM * kFgemmK / 128;
        double va[kPer], vb[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int e = threadIdx.x + 128 * u;
            const int m = e / kFgemmK, k = e % kFgemmK;  // A: k fastest
            va[u] = (k < K && r0 + m < Rtot) ? P[static_cast<long long>(r0 + m) * K + k] : 0.0;
            const int kb = e / kFsBN, nn = e % kFsBN;  // B: n fastest
            vb[u] = (kb < K && c0 + nn < ncols) ? Qf[static_cast<long long>(kb) * ncols + c0 + nn] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int e = threadIdx.x + 128 * u;
            As[(e / kFgemmK) * kFsLDA + e % kFgemmK] = va[u];
            Bs[(e / kFsBN) * kFsLDB + e % kFsBN] = vb[u];
        }
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wm = warp & 1, wn = warp >> 1;
    const int g = lane >> 2, t = lane & 3;
    double acc[2][4] = {};
    const int Kp = (K + 3) & ~3;  // columns K .. Kp-1 were loaded as zeros
    for (int ks = 0; ks < Kp; ks += 4) {
        const double a0 = As[(wm * 16 + g) * kFsLDA + ks + t];
        const double a1 = As[(wm * 16 + g + 8) * kFsLDA + ks + t];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) dmma_m16n8k4(acc[nt], a0, a1, Bs[(ks + t) * kFsLDB + wn * 16 + nt * 8 + g]);
    }
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int m = wm * 16 + g + 8 * (i >> 1), nn = wn * 16 + nt * 8 + 2 * t + (i & 1);
            if (r0 + m < Rtot && c0 + nn < ncols) {
                const int col = c0 + nn;
                const int dd = col / mm, e = col % mm;
                T[(static_cast<long long>(dd) * mm + e) * Rtot + r0 + m] = acc[nt][i];  // [d][e][r]
            }
        }
}

void launch_fgemm(const Launch& L, int m0, int Rtot, const DirPlan& d, const double* P, const double* Qf, double* T) {
    const int mm = m0 * m0;
    const int ncols = static_cast<int>(d.band + 1) * mm;
    if (d.n <= kFgemmK) {
        Stage st_(L, "fold_gemm");
        k_fgemm_s<<<dim3((ncols + kFsBN - 1) / kFsBN, (Rtot + kFsBM - 1) / kFsBM), 128, 0, L.st>>>(
            mm, Rtot, static_cast<int>(d.n), ncols, P, Qf, T);
        LT_CU(cudaGetLastError());
        L.tick();
        return;
    }
    dim3 grid((ncols + kGBN - 1) / kGBN, (Rtot + kGBM - 1) / kGBM);
    const size_t smem = d.n <= kFgemmK ? sizeof(double) * (kGBM * kFgemmLDA + kFgemmK * kFgemmLDB) : 0;
    static bool attr = false;
    if (smem && !attr) {
        LT_CU(cudaFuncSetAttribute(k_fgemm, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        attr = true;
    }
    Stage st_(L, "fold_gemm");
    k_fgemm<<<grid, 256, smem, L.st>>>(mm, Rtot, d.n, ncols, P, Qf, T);
    LT_CU(cudaGetLastError());
    L.tick();
}

// Khatri-Rao combine: N[d0,d1,d2][e] = sum_r W[r][e] prod_{l wrapped} T_l[d_l][e][r]
// (T_l stored for d >= 0 with r contiguous, so a CTA's table gathers are coalesced;
// T_l[-d][(mu,nu)][r] = T_l[d][(nu,mu)][r]). CTA per (e, d0): u[d1][r] = W[r][e] T_0[d0][e][r]
// T_1[d1][e][r] and t2[d2][r] = T_2[d2][e][r] in shared memory, then the (width1 x width2)
// block N[d0][., .][e] = u t2^T as m8n8k4 DMMA tiles over r (one 8 x 8 tile per warp).
__host__ __device__ inline int kr_ldk(int Rtot) {
    const int kp = (Rtot + 3) & ~3;
    return kp + (20 - kp % 16) % 16;  // = 4 (mod 16): conflict-free fragment reads
}

__global__ void k_kr_combine(KRArgs a) {
    extern __shared__ double sh[];
    const int e = blockIdx.x;
    const int i0 = blockIdx.y;  // d0 index in [0, width0)
    const int mm = a.m0 * a.m0;
    const int mu = e % a.m0, nu = e / a.m0;
    const int eT = nu + mu * a.m0;
    const int K = a.Rtot, Kp = (K + 3) & ~3, ldk = kr_ldk(K);
    const int w1 = a.width[1], w2 = a.width[2];
    const int W1p = (w1 + 7) & ~7, W2p = (w2 + 7) & ~7;
    double* u = sh;                // [W1p][ldk]
    double* t2 = u + W1p * ldk;    // [W2p][ldk]
    double* w0 = t2 + W2p * ldk;   // [Kp]
    auto tab = [&](int l, int di, int r) -> double {
        if (!a.T[l]) return 1.0;
        const int d = di - a.band[l];
        const int ad = d < 0 ? -d : d;
        const int ee = d < 0 ? eT : e;
        return a.T[l][(static_cast<long long>(ad) * mm + ee) * a.Rtot + r];  // [d][e][r]: r contiguous
    };
    // w0[r] = W[r][e] T_0[d0][e][r] of this lane's ranks r = lane + 32 x in registers (the same
    // rounded product every row is scaled by): no shared staging, so the loads of both slabs
    // below are in flight together with these (one round trip to L2 for the whole prologue)
    (void)w0;
    double w0r[4];
    {
        const int ln = static_cast<int>(threadIdx.x) & 31;
#pragma unroll
        for (int x = 0; x < 4; ++x) {
            const int r = ln + 32 * x;
            w0r[x] = r < K ? a.W[r * mm + e] * tab(0, i0, r) : 0.0;
        }
    }
    // the two table slabs (zero padded): rows split over the warps, r over the lanes (no
    // index division), the row's d sign and transposed entry resolved once per row
    auto gather = [&](int l, int w, int wp, double* dst, bool scale) {
        const int nw = static_cast<int>(blockDim.x) >> 5, wl = static_cast<int>(threadIdx.x) >> 5;
        const int ln = static_cast<int>(threadIdx.x) & 31;
        for (int row = wl; row < wp; row += nw) {
            const double* src = nullptr;
            if (row < w && a.T[l]) {
                const int d = row - a.band[l];
                const int ad = d < 0 ? -d : d;
                src = a.T[l] + (static_cast<long long>(ad) * mm + (d < 0 ? eT : e)) * a.Rtot;
            }
            double v[4];
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                const int r = ln + 32 * x;
                v[x] = r < K ? (src ? src[r] : (row < w ? 1.0 : 0.0)) : 0.0;
            }
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                const int r = ln + 32 * x;
                if (r < Kp) dst[row * ldk + r] = scale ? v[x] * w0r[x] : v[x];
            }
        }
    };
    gather(1, w1, W1p, u, true);
    gather(2, w2, W2p, t2, false);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int nt2 = W2p / 8, ntiles = (W1p / 8) * nt2;
    for (int tile = warp; tile < ntiles; tile += nwarp) {
        const int mt = tile / nt2, nt = tile % nt2;
        double acc[2] = {0.0, 0.0};
        const double* ua = u + (mt * 8 + g) * ldk + t;
        const double* tb = t2 + (nt * 8 + g) * ldk + t;
        // the fill's FEM factors of this thread's two outputs: loaded ahead of the DMMA loop
        double Mv[2][3] = {}, Sv[2][3] = {};
        if (a.H) {
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int ii[3] = {i0, mt * 8 + g, nt * 8 + 2 * t + i};
                if (ii[1] < w1 && ii[2] < w2) {
#pragma unroll
                    for (int l = 0; l < 3; ++l) {
                        Mv[i][l] = a.massT[l][static_cast<long long>(ii[l]) * mm + e];
                        Sv[i][l] = a.stiffT[l][static_cast<long long>(ii[l]) * mm + e];
                    }
                }
            }
        }
        for (int ks = 0; ks < Kp; ks += 4) dmma_m8n8k4(acc, ua[ks], tb[ks]);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int i1 = mt * 8 + g, i2 = nt * 8 + 2 * t + i;
            if (i1 < w1 && i2 < w2) {
                if (!a.H) {
                    const long long dlin = (static_cast<long long>(i0) * w1 + i1) * w2 + i2;
                    a.N[dlin * mm + e] = acc[i];
                    continue;
                }
                // k_fill's combine for this block (the same rounded products and sums, so
                // the blocks equal the two-kernel form bit for bit), entry-major
                const int ii[3] = {i0, i1, i2};
                double M[3], St[3];
                long long slot = 0;
#pragma unroll
                for (int l = 0; l < 3; ++l) {
                    M[l] = Mv[i][l];
                    St[l] = Sv[i][l];
                    const int d = ii[l] - a.band[l];
                    slot = slot * a.width[l] + (d >= 0 ? d : a.width[l] + d);
                }
                const double mass = __dmul_rn(__dmul_rn(M[0], M[1]), M[2]);
                const double t0 = __dmul_rn(__dmul_rn(St[0], M[1]), M[2]);
                const double t1 = __dmul_rn(__dmul_rn(M[0], St[1]), M[2]);
                const double t2 = __dmul_rn(__dmul_rn(M[0], M[1]), St[2]);
                const double lap = __dadd_rn(__dadd_rn(t0, t1), t2);
                a.H[e * a.nblocks + slot] = __dadd_rn(__dmul_rn(a.kin, lap), __dmul_rn(-1.0, acc[i]));
                a.S[e * a.nblocks + slot] = mass;
                if (e == 0)
#pragma unroll
                    for (int l = 0; l < 3; ++l) {
                        const long long d = ii[l] - a.band[l];
                        a.kidx[3 * slot + l] = ((d % a.L[l]) + a.L[l]) % a.L[l];
                    }
            }
        }
    }
}

void launch_kr_combine(const Launch& L, const KRArgs& a) {
    if (a.Rtot > 128) fail(LT_EGENERIC, "kr_combine: more than 128 rank terms");
    const int W1p = (a.width[1] + 7) & ~7, W2p = (a.width[2] + 7) & ~7;
    const size_t smem = sizeof(double) * (static_cast<size_t>(W1p + W2p) * kr_ldk(a.Rtot) + ((a.Rtot + 3) & ~3));
    static size_t attr = 0;
    if (smem > 48 * 1024 && smem > attr) {
        LT_CU(cudaFuncSetAttribute(k_kr_combine, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        attr = smem;
    }
    dim3 grid(a.m0 * a.m0, a.width[0]);
    Stage st_(L, "kr_combine");
    k_kr_combine<<<grid, 128, smem, L.st>>>(a);
    LT_CU(cudaGetLastError());
    L.tick();
}

}  // namespace lt
