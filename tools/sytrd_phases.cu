// Phase clocks (CTA 0) of the persistent tridiagonalisation k_sytrd_reg outside the engine:
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DLT_SYTRD_PROF -I include
//   -I paper_1408_3839_b200/csrc tools/sytrd_phases.cu -o tools/sytrd_phases
#include <cstdio>
#include <vector>
#include "../paper_1408_3839_b200/csrc/k_dense.cu"
using namespace lt;
void lt::StageTimer::begin(cudaStream_t, const char*) {}
void lt::StageTimer::end(cudaStream_t) {}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 1024;
    std::vector<double> h(static_cast<size_t>(n) * n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            h[static_cast<size_t>(i) * n + j] = (i == j ? 2.0 : 0.0) + 1.0 / (1 + i + j) + 0.01 * ((i * 7 + j * 7) % 13);
    double *C, *d, *e, *work;
    unsigned* bar;
    long long* prof;
    cudaMalloc(&C, sizeof(double) * n * n);
    cudaMalloc(&d, sizeof(double) * n);
    cudaMalloc(&e, sizeof(double) * n);
    cudaMalloc(&work, sizeof(double) * 4 * n);
    cudaMalloc(&bar, 8192);
    cudaMalloc(&prof, 64);
    lt_sytrd_prof_ptr = prof;
    cudaMemcpy(C, h.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
    cudaStream_t st;
    cudaStreamCreate(&st);
    Launch L{st, nullptr, nullptr};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0, st);
        launch_sytrd(L, n, C, d, e, work, bar);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        long long pr[6];
        cudaMemcpy(pr, prof, sizeof(pr), cudaMemcpyDeviceToHost);
        std::printf("sytrd n=%d: %.1f us (%s)\n", n, ms * 1e3, cudaGetErrorString(cudaGetLastError()));
        const double st_ = n - 1;
        std::printf("  cycles/step: barrier %.0f  loads+vp %.0f  w/c+sigma %.0f  reflector %.0f  update %.0f  publish %.0f\n",
                    pr[1] / st_, pr[2] / st_, pr[3] / st_, pr[4] / st_, pr[0] / st_, pr[5] / st_);
    }
    std::vector<double> hd(n);
    cudaMemcpy(hd.data(), d, sizeof(double) * n, cudaMemcpyDeviceToHost);
    double tr = 0, tr0 = 0;
    for (int i = 0; i < n; ++i) tr += hd[i], tr0 += h[static_cast<size_t>(i) * n + i];
    std::printf("trace %.12g vs %.12g\n", tr, tr0);
    return 0;
}
