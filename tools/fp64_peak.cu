// tools/fp64_peak.cu — measured FP64 peaks on this B200 (roofline denominators) and a
// correctness check of the DMMA fragment layouts used by the engine.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
//   tools/fp64_peak  -> one JSON line {dfma_tflops, dmma_tflops (best shape), per-shape, layout_ok}
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e = (x);                                                               \
        if (e != cudaSuccess) {                                                            \
            std::printf("{\"error\": \"%s line %d\"}\n", cudaGetErrorString(e), __LINE__); \
            return 1;                                                                      \
        }                                                                                  \
    } while (0)

__global__ void k_dfma(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
}

// D = A*B + C with mma.sync .f64, shapes m8n8k4 / m16n8k4 / m16n8k8 / m16n8k16
__device__ __forceinline__ void mma_m8n8k4(double& d0, double& d1, double a0, double b0) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a0), "d"(b0));
}
__device__ __forceinline__ void mma_m16n8k4(double* d, const double* a, const double* b) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                 : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
                 : "d"(a[0]), "d"(a[1]), "d"(b[0]));
}
__device__ __forceinline__ void mma_m16n8k8(double* d, const double* a, const double* b) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ void mma_m16n8k16(double* d, const double* a, const double* b) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
        "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
        : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
          "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int SHAPE>
__global__ void k_dmma(double* out, int iters) {
    double acc[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[j][i] = 0.0;
    double a[8], b[4];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = 1.0 + 1e-9 * (threadIdx.x + i);
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] = 1.0 - 1e-9 * (threadIdx.x + i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (SHAPE == 0) mma_m8n8k4(acc[j][0], acc[j][1], a[j], b[j]);
            if (SHAPE == 1) mma_m16n8k4(acc[j], a, b);
            if (SHAPE == 2) mma_m16n8k8(acc[j], a, b);
            if (SHAPE == 3) mma_m16n8k16(acc[j], a, b);
        }
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i) s += acc[j][i];
    if (s == 12345.678) out[0] = s;
}

// layout check: one warp computes D = A(16xK) * B(Kx8) for K = 4, 8, 16 from the
// documented fragment maps (groupID = lane>>2, tig = lane&3):
//   A: a[i] -> row = g + 8*(i&1), col = tig + 4*(i>>1)     B: b[i] -> row = tig + 4*i, col = g
//   C: c[i] -> row = g + 8*(i>>1), col = 2*tig + (i&1)
template <int K>
__global__ void k_layout(const double* A, const double* B, double* D) {
    const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
    double a[8] = {0}, b[4] = {0}, d[4] = {0, 0, 0, 0};
    for (int i = 0; i < K / 2; ++i) a[i] = A[(g + 8 * (i & 1)) * K + t + 4 * (i >> 1)];
    for (int i = 0; i < K / 4; ++i) b[i] = B[(t + 4 * i) * 8 + g];
    if (K == 4) mma_m16n8k4(d, a, b);
    if (K == 8) mma_m16n8k8(d, a, b);
    if (K == 16) mma_m16n8k16(d, a, b);
    for (int i = 0; i < 4; ++i) D[(g + 8 * (i >> 1)) * 8 + 2 * t + (i & 1)] = d[i];
}

template <int K>
static bool check_layout() {
    std::vector<double> A(16 * K), B(K * 8), D(128), R(128, 0.0);
    for (int i = 0; i < 16 * K; ++i) A[i] = std::sin(1.0 + i);
    for (int i = 0; i < K * 8; ++i) B[i] = std::cos(2.0 + i);
    for (int r = 0; r < 16; ++r)
        for (int c = 0; c < 8; ++c)
            for (int k = 0; k < K; ++k) R[r * 8 + c] += A[r * K + k] * B[k * 8 + c];
    double *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 8);
    cudaMalloc(&dB, B.size() * 8);
    cudaMalloc(&dD, 128 * 8);
    cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice);
    k_layout<K><<<1, 32>>>(dA, dB, dD);
    cudaMemcpy(D.data(), dD, 128 * 8, cudaMemcpyDeviceToHost);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
    double err = 0;
    for (int i = 0; i < 128; ++i) err = std::fmax(err, std::fabs(D[i] - R[i]));
    return err < 1e-13;
}

int main() {
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    double* out;
    CK(cudaMalloc(&out, 8));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int threads = 256, blocks = sms * 8;
    const int iters = 20000;
    float ms = 0;
    double best = 0;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(out, iters, 1.0000001, 1e-7);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::fmax(best, 2.0 * 8 * iters * double(blocks) * threads / (ms * 1e-3) / 1e12);
    }
    const double dfma = best;
    const int flops_per_mma[4] = {2 * 8 * 8 * 4, 2 * 16 * 8 * 4, 2 * 16 * 8 * 8, 2 * 16 * 8 * 16};
    const char* names[4] = {"m8n8k4", "m16n8k4", "m16n8k8", "m16n8k16"};
    double shape_tf[4];
    const int miters = 4000;
    for (int s = 0; s < 4; ++s) {
        best = 0;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            if (s == 0) k_dmma<0><<<blocks, threads>>>(out, miters);
            if (s == 1) k_dmma<1><<<blocks, threads>>>(out, miters);
            if (s == 2) k_dmma<2><<<blocks, threads>>>(out, miters);
            if (s == 3) k_dmma<3><<<blocks, threads>>>(out, miters);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            cudaEventElapsedTime(&ms, e0, e1);
            const double warps = double(blocks) * threads / 32;
            best = std::fmax(best, warps * miters * 4.0 * flops_per_mma[s] / (ms * 1e-3) / 1e12);
        }
        shape_tf[s] = best;
    }
    double dmma = 0;
    for (double v : shape_tf) dmma = std::fmax(dmma, v);
    const bool ok4 = check_layout<4>(), ok8 = check_layout<8>(), ok16 = check_layout<16>();
    std::printf("{\"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f", dfma, dmma);
    for (int s = 0; s < 4; ++s) std::printf(", \"%s_tflops\": %.3f", names[s], shape_tf[s]);
    std::printf(", \"layout_m16n8k4_ok\": %s, \"layout_m16n8k8_ok\": %s, \"layout_m16n8k16_ok\": %s, \"sms\": %d}\n",
                ok4 ? "true" : "false", ok8 ? "true" : "false", ok16 ? "true" : "false", sms);
    return 0;
}
