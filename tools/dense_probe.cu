// Microbenchmark of the dense-pencil front-end kernels (k_potf_leaf, k_dgemm_tn) outside the
// engine: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include
//   -I paper_1408_3839_b200/csrc tools/dense_probe.cu paper_1408_3839_b200/csrc/k_dense2.cu
//   paper_1408_3839_b200/csrc/k_dgemm.cu -o tools/dense_probe
#include <cstdio>
#include <vector>
#include "lt_internal.cuh"
namespace lt { extern __device__ long long lt_leaf_prof[64]; }

using namespace lt;
void lt::StageTimer::begin(cudaStream_t, const char*) {}
void lt::StageTimer::end(cudaStream_t) {}

int main() {
    const int n = 1024;
    const long long ld = n;
    std::vector<double> h(static_cast<size_t>(n) * n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) h[static_cast<size_t>(i) * n + j] = (i == j ? n : 0.0) + 1.0 / (1 + i + j);
    double *S, *Li, *Lic, *W, *T, *H;
    unsigned long long* fail;
    for (double** p : {&S, &Li, &Lic, &W, &T, &H}) cudaMalloc(p, sizeof(double) * n * n);
    cudaMalloc(&fail, 8);
    cudaMemset(fail, 0xff, 8);
    cudaStream_t st;
    cudaStreamCreate(&st);
    Launch L{st, nullptr, nullptr};
    DenseReduceBufs b{S, H, Li, Lic, W, T, fail};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemcpy(S, h.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
        cudaMemcpy(H, h.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
        cudaEventRecord(e0, st);
        dense_factor(L, n, ld, b);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        std::printf("dense_factor n=%d: %.1f us\n", n, ms * 1e3);
        cudaEventRecord(e0, st);
        dense_transform(L, n, ld, b);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        std::printf("dense_transform n=%d: %.1f us\n", n, ms * 1e3);
    }
    // one leaf alone, 20 times
    cudaMemcpy(S, h.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
    cudaEventRecord(e0, st);
    for (int i = 0; i < 20; ++i) {
        DenseReduceBufs bb = b;
        dense_factor(L, 64, ld, bb);  // n = 64: exactly one leaf
    }
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    std::printf("leaf (n=64) x20: %.2f us each\n", ms * 1e3 / 20);
    // individual GEMM shapes, 50 back-to-back launches each
    auto time_gemm = [&](const char* name, int M, int N, long long K, int flags, unsigned long long* fl) {
        const DgemmOperand A{S, n, n, ld}, B{H, n, n, ld};
        DgemmArgs g;
        g.M = M;
        g.N = N;
        g.K = K;
        g.c0 = W;
        g.ldc = ld;
        g.flags = flags;
        g.fail = fl;
        launch_dgemm_tn(L, A, B, g, 1, "probe");
        cudaEventRecord(e0, st);
        for (int i = 0; i < 50; ++i) launch_dgemm_tn(L, A, B, g, 1, "probe");
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double fl2 = 2.0 * M * N * K;
        std::printf("gemm %-22s M=%d N=%d K=%lld: %8.2f us each, %.2f TFLOP/s (full-box flops)\n", name, M, N, K,
                    ms * 1e3 / 50, fl2 / (ms * 1e-3 / 50) / 1e12);
    };
    time_gemm("panel", 960, 64, 64, 0, fail);
    time_gemm("panel-nofail", 960, 64, 64, 0, nullptr);
    time_gemm("update", 960, 960, 64, DG_LOWER, fail);
    time_gemm("square", 1024, 1024, 1024, 0, nullptr);
    time_gemm("square-lower", 1024, 1024, 1024, DG_LOWER, nullptr);
    time_gemm("tiny", 64, 64, 64, 0, nullptr);
#ifdef LT_LEAF_PROFILE
    {
        long long pr[64];
        cudaMemcpyFromSymbol(pr, lt_leaf_prof, sizeof(pr));
        std::printf("leaf phases (cycles from start):");
        for (int i = 1; i <= 30; ++i) std::printf(" %d:%lld", i, pr[i] - pr[0]);
        std::printf("\n");
    }
#endif
    unsigned long long f;
    cudaMemcpy(&f, fail, 8, cudaMemcpyDeviceToHost);
    std::printf("fail key %llx, err %s\n", f, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
