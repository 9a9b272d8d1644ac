// Sturm-multisection variants for the dense tridiagonal eigenvalues (k_tridiag_eig3):
// lanes per eigenvalue G, shifts per lane Q, on a random n x n tridiagonal.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -Ipaper_1408_3839_b200/csrc \
//        tools/eig3_probe.cu -Lpaper_1408_3839_b200/_lib -llatham_b200 -o tools/eig3_probe
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "../paper_1408_3839_b200/csrc/k_dense.cu"

template <int Q, int G, int BS, int GU = 0>
static float run(int n, const double* d, const double* e, double* eig) {
    const size_t smem = sizeof(double) * 2 * n;
    cudaFuncSetAttribute(lt::k_tridiag_eig3<Q, G, BS, GU>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const unsigned blocks = (unsigned)((size_t(n) * G + BS - 1) / BS);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        lt::k_tridiag_eig3<Q, G, BS, GU><<<blocks, BS, smem>>>(n, d, e, eig);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = std::min(best, ms);
    }
    return best * 1e3f;
}

int main() {
    const int n = 1024;
    std::mt19937_64 rng(5);
    std::normal_distribution<double> nd;
    std::vector<double> hd(n), he(n);
    for (int i = 0; i < n; ++i) {
        hd[i] = nd(rng) * 3.0;
        he[i] = nd(rng);
    }
    double *d, *e, *e0, *e1;
    cudaMalloc(&d, n * 8);
    cudaMalloc(&e, n * 8);
    cudaMalloc(&e0, n * 8);
    cudaMalloc(&e1, n * 8);
    cudaMemcpy(d, hd.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(e, he.data(), n * 8, cudaMemcpyHostToDevice);
    std::vector<double> ref(n), got(n);
    const float t0 = run<2, 16, 64>(n, d, e, e0);
    cudaMemcpy(ref.data(), e0, n * 8, cudaMemcpyDeviceToHost);
    std::printf("Q2 G16 BS64 (current): %.1f us\n", t0);
    auto chk = [&](const char* name, float t) {
        cudaMemcpy(got.data(), e1, n * 8, cudaMemcpyDeviceToHost);
        double md = 0;
        for (int i = 0; i < n; ++i) md = std::max(md, std::fabs(got[i] - ref[i]));
        std::printf("%-14s %.1f us  max|d| %.2e\n", name, t, md);
    };
    chk("Q1 G32 g2 64", run<1, 32, 64, 2>(n, d, e, e1));
    chk("Q1 G32 g2 128", run<1, 32, 128, 2>(n, d, e, e1));
    chk("Q1 G32 g2 256", run<1, 32, 256, 2>(n, d, e, e1));
    chk("Q2 G32 g2 64", run<2, 32, 64, 2>(n, d, e, e1));
    chk("Q1 G32 g0 64", run<1, 32, 64, 0>(n, d, e, e1));
    chk("Q1 G32 g1 64", run<1, 32, 64, 1>(n, d, e, e1));
    chk("Q1 G16 g2 32", run<1, 16, 32, 2>(n, d, e, e1));
    return 0;
}
