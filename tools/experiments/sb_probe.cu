// Two-stage tridiagonalisation probe (k_sb2st.cu built with LT_SB_PROFILE): a random symmetric
// matrix through stage 1 + stage 2 + the Sturm eigenvalues, against the one-stage reduction
// (k_dense.cu), with per-sweep start / end clocks of the bulge chase.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DLT_SB_PROFILE -Ipaper_1408_3839_b200/csrc \
//        -Iinclude tools/experiments/sb_probe.cu -Lpaper_1408_3839_b200/_lib -llatham_b200 -o tools/experiments/sb_probe
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "k_sb2st.cu"

int main(int argc, char** argv) {
    const int n = argc > 1 ? std::atoi(argv[1]) : 1024;
    std::mt19937_64 rng(11);
    std::normal_distribution<double> nd;
    std::vector<double> A(static_cast<size_t>(n) * n);
    for (int j = 0; j < n; ++j)
        for (int i = j; i < n; ++i) A[static_cast<size_t>(j) * n + i] = A[static_cast<size_t>(i) * n + j] = nd(rng);
    double *dA, *dA2, *d1, *e1, *d2, *e2, *ev1, *ev2, *tw;
    unsigned* bar;
    const int kd = lt::sb2st_kd(n);
    lt::SbBufs b;
    auto alloc = [](double** p, size_t cnt) { cudaMalloc(p, cnt * sizeof(double)); };
    alloc(&dA, A.size());
    alloc(&dA2, A.size());
    alloc(&d1, n); alloc(&e1, n); alloc(&d2, n); alloc(&e2, n); alloc(&ev1, n); alloc(&ev2, n); alloc(&tw, 4 * n);
    cudaMalloc(&bar, 8 * 160 * 4);
    alloc(&b.band, (kd + 1) * n); alloc(&b.U1, 2 * kd * n); alloc(&b.U2, 2 * kd * n); alloc(&b.Vt, kd * n);
    alloc(&b.VTt, kd * n); alloc(&b.Wt, kd * n); alloc(&b.M, kd * kd); alloc(&b.T, kd * kd);
    cudaMemcpy(dA2, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
    cudaStream_t st;
    cudaStreamCreate(&st);
    lt::Launch L{st, nullptr, nullptr};
    cudaEvent_t a, c, f;
    cudaEventCreate(&a); cudaEventCreate(&c); cudaEventCreate(&f);
    float t1 = 0, t2 = 0;
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemcpyAsync(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice, st);
        cudaEventRecord(a, st);
        lt::launch_two_stage_tridiag(L, n, dA, n, b, d1, e1);
        cudaEventRecord(c, st);
        lt::launch_tridiag_eig(L, n, d1, e1, ev1);
        lt::launch_sytrd(L, n, dA2, d2, e2, tw, bar);
        lt::launch_tridiag_eig(L, n, d2, e2, ev2);
        cudaEventRecord(f, st);
        cudaEventSynchronize(f);
        cudaEventElapsedTime(&t1, a, c);
    }
    std::vector<double> h1(n), h2(n);
    cudaMemcpy(h1.data(), ev1, n * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2.data(), ev2, n * 8, cudaMemcpyDeviceToHost);
    double md = 0, mx = 0;
    for (int i = 0; i < n; ++i) {
        md = std::max(md, std::fabs(h1[i] - h2[i]));
        mx = std::max(mx, std::fabs(h2[i]));
    }
    std::vector<long long> pr(4096 * 2);
    cudaMemcpyFromSymbol(pr.data(), lt_sb_prof, pr.size() * 8);
    long long t0 = pr[0];
    std::printf("n %d kd %d: two-stage %.3f ms; max |dlambda| %.3e (max |lambda| %.3e) %s\n", n, kd, t1, md, mx,
                cudaGetErrorString(cudaGetLastError()));
    for (int s : {0, 1, 2, 3, 31, 32, 33, 100, 500, n - 10})
        if (s < n - 2) std::printf("  sweep %5d: start %9lld end %9lld (len %lld)\n", s, pr[2 * s] - t0, pr[2 * s + 1] - t0, pr[2 * s + 1] - pr[2 * s]);
    return 0;
}
