// Phase clocks of the cluster tridiagonalisation (k_sytrd_cl) outside the engine:
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DLT_CL_PROF -I include
//   -I paper_1408_3839_b200/csrc tools/experiments/sytrd_cluster_probe.cu -o tools/experiments/sytrd_cluster_probe
#include <cstdio>
#include <vector>
#include "../../paper_1408_3839_b200/csrc/k_dense.cu"
using namespace lt;
void lt::StageTimer::begin(cudaStream_t, const char*) {}
void lt::StageTimer::end(cudaStream_t) {}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 512;
    std::vector<double> h(static_cast<size_t>(n) * n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) h[static_cast<size_t>(i) * n + j] = (i == j ? 2.0 : 0.0) + 1.0 / (1 + i + j) + 0.01 * ((i * 7 + j * 7) % 13);
    double *C, *d, *e, *work, *tail;
    unsigned* bar;
    cudaMalloc(&C, sizeof(double) * n * n);
    cudaMalloc(&d, sizeof(double) * n);
    cudaMalloc(&e, sizeof(double) * n);
    cudaMalloc(&work, sizeof(double) * 4 * n);
    cudaMalloc(&tail, sizeof(double) * 512 * 512);
    cudaMalloc(&bar, 4096);
    cudaMemcpy(C, h.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
    cudaStream_t st;
    cudaStreamCreate(&st);
    Launch L{st, nullptr, nullptr};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    for (int rep = 0; rep < 3; ++rep) {
        long long z[8] = {};
        cudaMemcpyToSymbol(lt_cl_prof, z, sizeof(z));
        cudaEventRecord(e0, st);
        launch_sytrd(L, n, C, d, e, work, bar, tail);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        long long pr[8];
        cudaMemcpyFromSymbol(pr, lt_cl_prof, sizeof(pr));
        std::printf("sytrd n=%d: %.1f us (%s)\n", n, ms * 1e3, cudaGetErrorString(cudaGetLastError()));
        const int steps = n > 512 ? 511 : n - 1;
        std::printf("  cluster cycles/step: sync %.0f  pull+vp %.0f  w/c+sigma %.0f  reflector %.0f  update %.0f  publish %.0f\n",
                    double(pr[0]) / steps, double(pr[1]) / steps, double(pr[2]) / steps, double(pr[3]) / steps,
                    double(pr[4]) / steps, double(pr[5]) / steps);
    }
    std::vector<double> hd(n), he(n);
    cudaMemcpy(hd.data(), d, sizeof(double) * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(he.data(), e, sizeof(double) * n, cudaMemcpyDeviceToHost);
    double tr = 0, tr0 = 0;
    for (int i = 0; i < n; ++i) tr += hd[i], tr0 += h[static_cast<size_t>(i) * n + i];
    std::printf("trace %.12g vs %.12g\n", tr, tr0);
    return 0;
}
