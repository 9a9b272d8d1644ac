// k_dgemm.cu — TMA-fed FP64 tensor-core GEMM for the dense box pencil (eigensolver.cpp:12-35).
//
//   C(m, n) = beta C(m, n) + alpha sum_{k in [k_lo, k_hi)} A(m, k) B(n, k)
//
// Both operands are K-major ("TN"): A(m, k) = TA[a_row0 + m][a_col0 + k] and
// B(n, k) = TB[b_row0 + n][b_col0 + k] of row-major 2D tensors, which is how every product
// of the pencil reduction reads (S, H symmetric; L, L^-1 kept row-major and, for L^-1, also
// column-major; see k_dense2.cu). A 64 x 64 tile per CTA: one producer warp issues
// cp.async.bulk.tensor loads of 64 x 16 boxes of A and B into a 4-stage ring (SWIZZLE_128B,
// full/empty mbarriers), eight consumer warps (4 x 2, 16 x 32 each) run m16n8k4 DMMA from
// the swizzled stages. Per tile the K range can be clipped to a triangular operand's
// non-zero part (k <= m, k <= n, k >= m, k >= n at tile granularity), tiles above the
// diagonal can be skipped (symmetric / triangular results) and mirrored, and the result
// stored row- or column-major (optionally both, into two buffers). Batches (grid.z) shift
// the operand coordinates and the output offsets by fixed strides.
#include "dmma.cuh"
#include "lt_internal.cuh"
#include "tma.cuh"

#include <cudaTypedefs.h>

#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

namespace lt {

namespace {
constexpr int kTM = 64, kTN = 64, kTK = 16, kStages = 4;
constexpr int kStageDoubles = (kTM + kTN) * kTK;  // A box then B box
constexpr unsigned kStageBytes = kStageDoubles * sizeof(double);
constexpr int kConsumerWarps = 8;  // 4 (m) x 2 (n), 16 x 32 each
constexpr int kThreads = 32 * (kConsumerWarps + 1);  // + 1 producer warp

struct alignas(1024) DgemmSmem {
    double stage[kStages][kStageDoubles];
    uint64_t full[kStages];
    uint64_t empty[kStages];
};
}  // namespace

__global__ void __launch_bounds__(kThreads) k_dgemm_tn(const __grid_constant__ CUtensorMap ta,
                                                       const __grid_constant__ CUtensorMap tb, DgemmArgs a) {
    extern __shared__ __align__(1024) unsigned char dg_raw[];
    DgemmSmem& sm = *reinterpret_cast<DgemmSmem*>(
        (reinterpret_cast<uintptr_t>(dg_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    if (a.fail && *a.fail != ~0ull) return;
    const int mt0 = blockIdx.x * kTM, nt0 = blockIdx.y * kTN;
    const int z = blockIdx.z;
    if (mt0 >= a.M || nt0 >= a.N) return;
    if ((a.flags & DG_LOWER) && nt0 > mt0 + kTM - 1) return;
    // K range of this tile
    long long klo = 0, khi = a.K;
    if (a.flags & DG_K_LE_M) khi = min(khi, static_cast<long long>(mt0 + kTM));
    if (a.flags & DG_K_LE_N) khi = min(khi, static_cast<long long>(nt0 + kTN));
    if (a.flags & DG_K_GE_M) klo = max(klo, static_cast<long long>(mt0));
    if (a.flags & DG_K_GE_N) klo = max(klo, static_cast<long long>(nt0));
    const int nk = khi > klo ? static_cast<int>((khi - klo + kTK - 1) / kTK) : 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], kConsumerWarps);
        }
        mbar_fence_init();
    }
    __syncthreads();
    const long long arow = a.a_row0 + static_cast<long long>(z) * a.a_zrow + mt0;
    const long long acol = a.a_col0 + static_cast<long long>(z) * a.a_zcol + klo;
    const long long brow = a.b_row0 + static_cast<long long>(z) * a.b_zrow + nt0;
    const long long bcol = a.b_col0 + static_cast<long long>(z) * a.b_zcol + klo;
    if (warp == kConsumerWarps) {
        // producer: one elected lane issues the TMA loads of every stage
        if (lane == 0) {
            tma_prefetch_desc(&ta);
            tma_prefetch_desc(&tb);
            for (int it = 0; it < nk; ++it) {
                const int s = it % kStages;
                if (it >= kStages) mbar_wait(&sm.empty[s], ((it / kStages) - 1) & 1);
                mbar_arrive_expect_tx(&sm.full[s], kStageBytes);
                tma_load_2d(&sm.stage[s][0], &ta, &sm.full[s], static_cast<int>(acol + it * kTK), static_cast<int>(arow));
                tma_load_2d(&sm.stage[s][kTM * kTK], &tb, &sm.full[s], static_cast<int>(bcol + it * kTK),
                            static_cast<int>(brow));
            }
        }
        return;
    }
    // consumers: warp (wm, wn) owns rows wm*16 .. +16, cols wn*32 .. +32
    const int wm = warp & 3, wn = warp >> 2;
    const int g = lane >> 2, t = lane & 3;
    double acc[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[j][q] = 0.0;
    for (int it = 0; it < nk; ++it) {
        const int s = it % kStages;
        mbar_wait(&sm.full[s], (it / kStages) & 1);
        const double* As = &sm.stage[s][0];
        const double* Bs = &sm.stage[s][kTM * kTK];
        const long long kbase = klo + static_cast<long long>(it) * kTK;
#pragma unroll
        for (int ks = 0; ks < kTK; ks += 4) {
            const bool kv = kbase + ks + t < khi;  // partial last stage: columns past k_hi are other data
            const int r = wm * 16 + g;
            const double a0 = kv ? As[swz128(r, ks + t)] : 0.0;
            const double a1 = kv ? As[swz128(r + 8, ks + t)] : 0.0;
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma_m16n8k4(acc[j], a0, a1, Bs[swz128(wn * 32 + j * 8 + g, ks + t)]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[s]);
    }
    // epilogue
    const long long coff0 = static_cast<long long>(z) * a.c_zoff;
    const bool diag_tile = (a.flags & DG_LOWER) && (mt0 == nt0);
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int m = mt0 + wm * 16 + g + 8 * (q >> 1);
                const int n = nt0 + wn * 32 + j * 8 + 2 * t + (q & 1);
                if (m >= a.M || n >= a.N) continue;
                if (diag_tile && n > m) continue;
                const double v = a.alpha * acc[j][q];
#pragma unroll
                for (int o = 0; o < 2; ++o) {
                    double* C = o == 0 ? a.c0 : a.c1;
                    if (!C) continue;
                    const bool cm = (a.flags & (o == 0 ? DG_C0_COLMAJOR : DG_C1_COLMAJOR)) != 0;
                    const long long idx = coff0 + (cm ? (m + static_cast<long long>(n) * a.ldc)
                                                      : (static_cast<long long>(m) * a.ldc + n));
                    C[idx] = a.beta_one ? C[idx] + v : v;
                    if ((a.flags & DG_MIRROR) && m != n) {
                        const long long idt = coff0 + (cm ? (n + static_cast<long long>(m) * a.ldc)
                                                          : (static_cast<long long>(n) * a.ldc + m));
                        C[idt] = a.beta_one ? C[idt] + v : v;
                    }
                }
            }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
bool tma_try_map_2d(CUtensorMap* out, const double* base, long long rows, long long cols, long long ld, int box_rows) {
    static std::mutex mu;
    static std::map<std::tuple<const double*, long long, long long, long long, int, int>, CUtensorMap> cache;
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    int dev = 0;
    LT_CU(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_tuple(base, rows, cols, ld, box_rows, dev);
    auto it = cache.find(key);
    if (it != cache.end()) {
        *out = it->second;
        return true;
    }
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        LT_CU(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !fn) fail(LT_ECUDA, "cuTensorMapEncodeTiled unavailable");
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    if ((reinterpret_cast<uintptr_t>(base) & 15) || (ld * 8) % 16) return false;
    CUtensorMap m;
    std::memset(&m, 0, sizeof(m));
    const cuuint64_t gdim[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t gstride[1] = {static_cast<cuuint64_t>(ld * 8)};
    const cuuint32_t box[2] = {16, static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), gdim, gstride, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    if (cache.size() > 4096) cache.clear();
    cache.emplace(key, m);
    *out = m;
    return true;
}

CUtensorMap tma_map_2d(const double* base, long long rows, long long cols, long long ld, int box_rows) {
    CUtensorMap m;
    if (!tma_try_map_2d(&m, base, rows, cols, ld, box_rows))
        fail(LT_EGENERIC, "tma_map_2d: base must be 16-byte aligned, the row pitch a multiple of 16 bytes and the "
                          "shape encodable (cuTensorMapEncodeTiled)");
    return m;
}

void launch_dgemm_tn(const Launch& L, const DgemmOperand& A, const DgemmOperand& B, const DgemmArgs& args, int batches,
                     const char* stage) {
    if (args.M <= 0 || args.N <= 0 || batches <= 0) return;
    const CUtensorMap ta = tma_map_2d(A.base, A.rows, A.cols, A.ld, kTM);
    const CUtensorMap tb = tma_map_2d(B.base, B.rows, B.cols, B.ld, kTN);
    const size_t smem = sizeof(DgemmSmem) + 1024;
    static bool attr = false;
    if (!attr) {
        LT_CU(cudaFuncSetAttribute(k_dgemm_tn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        attr = true;
    }
    dim3 grid(static_cast<unsigned>((args.M + kTM - 1) / kTM), static_cast<unsigned>((args.N + kTN - 1) / kTN),
              static_cast<unsigned>(batches));
    Stage st_(L, stage);
    k_dgemm_tn<<<grid, kThreads, smem, L.st>>>(ta, tb, args);
    LT_CU(cudaGetLastError());
    L.tick();
}

}  // namespace lt
