// tma.cuh — Tensor Memory Accelerator (cp.async.bulk.tensor) + mbarrier building blocks for
// sm_100a, and the host-side tensor-map cache.
//
// FP64 operands are staged global -> shared memory by TMA 2D tile loads (SWIZZLE_128B: a
// box row is 16 doubles = 128 B; the 16-byte chunks of row r are XOR-permuted by r mod 8, so
// the DMMA fragment reads of 8 rows x 4 k-columns hit 8 distinct chunks), signalled on an
// mbarrier with the transaction byte count (complete_tx). Consumers release a stage through a
// second mbarrier (one arrival per consumer warp).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace lt {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

// make the initialised barriers visible to the async (TMA) proxy
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// wait until the barrier's phase with parity `parity` has completed
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "LT_MBAR_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra LT_MBAR_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// 2D tile load: box at tensor coordinates (c0 = inner/column, c1 = row) into smem `dst`
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
        ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// 1D bulk copy global -> shared (cp.async.bulk): src, dst 16-byte aligned, bytes a multiple of 16
__device__ __forceinline__ void tma_bulk_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// element (r, c) of a SWIZZLE_128B box whose rows are 16 doubles (128 B), in doubles
__device__ __forceinline__ int swz128(int r, int c) { return r * 16 + ((((c >> 1) ^ (r & 7))) << 1) + (c & 1); }

// Host: a 2D row-major FP64 tensor map (rows x cols, row pitch ld doubles; ld * 8 must be a
// multiple of 16 and the base 16-byte aligned) with box {16 columns, box_rows rows},
// SWIZZLE_128B, out-of-bounds elements read as zero. Cached by (base, rows, cols, ld, box).
CUtensorMap tma_map_2d(const double* base, long long rows, long long cols, long long ld, int box_rows);
// the same, returning false instead of failing when the driver rejects the shape (rows may
// overlap: a pitch smaller than the row length gives the Hankel / Toeplitz views of k_hankel_tma)
bool tma_try_map_2d(CUtensorMap* out, const double* base, long long rows, long long cols, long long ld, int box_rows);

}  // namespace lt
