// Per-phase cycle counts of the one-thread-per-pencil kernel (k_pencil_lane.cu built with
// LT_LANE_PROFILE), and its time against the group kernel on the same random pencils.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DLT_LANE_PROFILE -DLT_PENCIL_PROFILE \
//        -Ipaper_1408_3839_b200/csrc -Iinclude tools/lane_phases.cu -o tools/lane_phases
// Phases: 0 load, 1 check, 2 Cholesky, 3 Y = L^-1 H, 4 Z = L^-1 Y^H, 5 Householder, 6 bisection.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "../paper_1408_3839_b200/csrc/k_pencil.cu"
#include "../paper_1408_3839_b200/csrc/k_pencil_lane.cu"
void lt::StageTimer::begin(cudaStream_t, const char*) {}
void lt::StageTimer::end(cudaStream_t) {}

int main(int argc, char** argv) {
    const int count = argc > 1 ? std::atoi(argv[1]) : 4096;
    constexpr int N = 8, mm = 64;
    std::mt19937_64 rng(7);
    std::normal_distribution<double> nd;
    std::vector<double2> H(static_cast<size_t>(count) * mm), S(H.size()), He(H.size()), Se(H.size());
    for (int k = 0; k < count; ++k) {
        std::vector<double2> A(mm), B(mm);
        for (auto& z : A) z = make_double2(nd(rng), nd(rng));
        for (auto& z : B) z = make_double2(nd(rng), nd(rng));
        for (int r = 0; r < N; ++r)
            for (int c = 0; c < N; ++c) {
                const double2 a = A[r + c * N], at = A[c + r * N];
                H[k * mm + r + c * N] = make_double2(a.x + at.x, a.y - at.y);
                double2 s = make_double2(r == c ? N : 0.0, 0.0);
                for (int q = 0; q < N; ++q) {
                    const double2 x = B[r + q * N], y = B[c + q * N];
                    s.x += x.x * y.x + x.y * y.y;
                    s.y += x.y * y.x - x.x * y.y;
                }
                S[k * mm + r + c * N] = s;
            }
    }
    for (int k = 0; k < count; ++k)
        for (int e = 0; e < mm; ++e) {
            He[static_cast<size_t>(e) * count + k] = H[k * mm + e];
            Se[static_cast<size_t>(e) * count + k] = S[k * mm + e];
        }
    double2 *dH, *dS, *dHe, *dSe;
    double *e1, *e2;
    unsigned long long* fk;
    cudaMalloc(&dH, H.size() * 16);
    cudaMalloc(&dS, H.size() * 16);
    cudaMalloc(&dHe, H.size() * 16);
    cudaMalloc(&dSe, H.size() * 16);
    cudaMalloc(&e1, count * N * 8);
    cudaMalloc(&e2, count * N * 8);
    cudaMalloc(&fk, 8);
    cudaMemcpy(dH, H.data(), H.size() * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(dS, S.data(), H.size() * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(dHe, He.data(), H.size() * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(dSe, Se.data(), H.size() * 16, cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int smemg = sizeof(lt::PSmem<8>) * 4;
    cudaFuncSetAttribute(lt::k_pencil<8, 32, 128, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smemg);
    cudaFuncSetAttribute(lt::k_pencil_lane<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lt::pencil_lane_smem());
    float tg = 1e30f, tl = 1e30f;
    const int lb = (count + 31) / 32;
    for (int rep = 0; rep < 5; ++rep) {
        cudaMemset(fk, 0xff, 8);
        cudaEventRecord(a);
        lt::k_pencil<8, 32, 128, false><<<(count + 3) / 4, 128, smemg>>>(count, N, dH, dS, e1, fk, 1, lt::PencilDft{},
                                                                        nullptr, lt::PencilReadback{});
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        tg = std::min(tg, ms);
        cudaEventRecord(a);
        lt::k_pencil_lane<N><<<lb, 32 * lt::kLaneWarps, lt::pencil_lane_smem()>>>(count, dHe, dSe, 1, count, e2, fk, lt::PencilReadback{}, lb);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        tl = std::min(tl, ms);
    }
    std::vector<double> g(count * N), l(count * N);
    cudaMemcpy(g.data(), e1, g.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(l.data(), e2, l.size() * 8, cudaMemcpyDeviceToHost);
    double md = 0, mx = 0;
    for (size_t i = 0; i < g.size(); ++i) {
        md = std::max(md, std::fabs(g[i] - l[i]));
        mx = std::max(mx, std::fabs(g[i]));
    }
    std::vector<long long> prof(1024 * 8);
    cudaMemcpyFromSymbol(prof.data(), lt_lane_prof, prof.size() * 8);
    double ph[7] = {0};
    const int nw = std::min(lb, 1024);
    for (int w = 0; w < nw; ++w)
        for (int i = 0; i < 7; ++i) ph[i] += double(prof[w * 8 + i + 1] - prof[w * 8 + i]) / nw;
    std::printf("count %d: group kernel %.1f us, lane kernel %.1f us, max |dlambda| %.3e (max |lambda| %.3e) err %s\n",
                count, tg * 1e3, tl * 1e3, md, mx, cudaGetErrorString(cudaGetLastError()));
    std::printf("lane cycles: load %.0f check %.0f chol %.0f Y %.0f Z %.0f hh %.0f eig %.0f\n", ph[0], ph[1], ph[2], ph[3],
                ph[4], ph[5], ph[6]);
    return 0;
}
