// Per-phase cycle counts of the batched pencil kernel (k_pencil.cu built with
// LT_PENCIL_PROFILE). Build (after `make` in paper_1408_3839_b200/csrc):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DLT_PENCIL_PROFILE \
//        -Ipaper_1408_3839_b200/csrc -Iinclude tools/pencil_phases.cu \
//        -Lpaper_1408_3839_b200/_lib -llatham_b200 -Xlinker -rpath=$PWD/paper_1408_3839_b200/_lib \
//        -o tools/pencil_phases
// Phases: 0 load, 1 Hermitian check, 2 Cholesky, 3 reduction L^-1 H L^-H,
//         4 Householder tridiagonalisation, 5 multisection.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "../paper_1408_3839_b200/csrc/k_pencil.cu"

template <int NM, int G, int BS, bool VEC = false, bool RE = false>
static void run(int count, int m0, int reps) {
    std::mt19937_64 rng(count * 131 + m0);
    std::normal_distribution<double> nd;
    const int mm = m0 * m0;
    std::vector<double2> H(static_cast<size_t>(count) * mm), S(H.size());
    for (int k = 0; k < count; ++k) {
        std::vector<double2> A(mm), B(mm);
        for (auto& z : A) z = make_double2(nd(rng), RE ? 0.0 : nd(rng));
        for (auto& z : B) z = make_double2(nd(rng), RE ? 0.0 : nd(rng));
        for (int r = 0; r < m0; ++r)
            for (int c = 0; c < m0; ++c) {
                const double2 a = A[r + c * m0], at = A[c + r * m0];
                H[k * mm + r + c * m0] = make_double2(a.x + at.x, a.y - at.y);
                double2 s = make_double2(r == c ? m0 : 0.0, 0.0);
                for (int q = 0; q < m0; ++q) {  // B B^H
                    const double2 x = B[r + q * m0], y = B[c + q * m0];
                    s.x += x.x * y.x + x.y * y.y;
                    s.y += x.y * y.x - x.x * y.y;
                }
                S[k * mm + r + c * m0] = s;
            }
    }
    double2 *dH, *dS;
    double* de;
    unsigned long long* fk;
    cudaMalloc(&dH, H.size() * sizeof(double2));
    cudaMalloc(&dS, S.size() * sizeof(double2));
    cudaMalloc(&de, static_cast<size_t>(count) * m0 * sizeof(double));
    cudaMalloc(&fk, sizeof(unsigned long long));
    double2* dv = nullptr;
    if (VEC) cudaMalloc(&dv, static_cast<size_t>(count) * m0 * m0 * sizeof(double2));
    cudaMemcpy(dH, H.data(), H.size() * sizeof(double2), cudaMemcpyHostToDevice);
    cudaMemcpy(dS, S.data(), S.size() * sizeof(double2), cudaMemcpyHostToDevice);
    constexpr int PPC = BS / G;
    const size_t smem = sizeof(lt::PSmem<NM>) * PPC;
    cudaFuncSetAttribute(lt::k_pencil<NM, G, BS, VEC, RE>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    const int blocks = (count + PPC - 1) / PPC;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        {
            long long z[2] = {0, 0};
            cudaMemcpyToSymbol(lt_ms_prof, z, sizeof(z));
        }
        cudaMemset(fk, 0xff, sizeof(unsigned long long));
        cudaEventRecord(e0);
        lt::k_pencil<NM, G, BS, VEC, RE><<<blocks, BS, smem>>>(count, m0, dH, dS, de, fk, 1, lt::PencilDft{}, dv,
                                                             lt::PencilReadback{});
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    std::vector<long long> prof(8192 * 8);
    cudaMemcpyFromSymbol(prof.data(), lt_pencil_prof, prof.size() * sizeof(long long));
    double ph[6] = {0, 0, 0, 0, 0, 0}, rounds = 0;
    const int nk = count < 8192 ? count : 8192;
    for (int k = 0; k < nk; ++k)
        for (int i = 0; i < 6; ++i) ph[i] += static_cast<double>(prof[k * 8 + i + 1] - prof[k * 8 + i]) / nk;
    for (int k = 0; k < nk; ++k) rounds += static_cast<double>(prof[k * 8 + 7]) / nk;
    long long ms[2];
    cudaMemcpyFromSymbol(ms, lt_ms_prof, sizeof(ms));
    std::printf("   multisection of pencil 0: %.0f cycles per Sturm call over %lld calls\n", ms[1] ? double(ms[0]) / ms[1] : 0.0, ms[1]);
    std::printf("%s count %5d m0 %2d NM %2d G %4d BS %4d: kernel %8.1f us | cycles load %7.0f herm %7.0f chol %7.0f "
                "reduce %7.0f hh %7.0f bisect %7.0f rounds %4.1f | err %s\n",
                VEC ? "vec" : (RE ? "real" : "val"), count, m0, NM, G, BS, best * 1e3, ph[0], ph[1], ph[2], ph[3], ph[4], ph[5], rounds,
                cudaGetErrorString(cudaGetLastError()));
    cudaFree(dH);
    cudaFree(dS);
    cudaFree(de);
    cudaFree(fk);
}

int main() {
    run<8, 32, 64>(32, 8, 5);
    run<8, 64, 64>(32, 8, 5);
    run<8, 128, 128>(32, 8, 5);
    run<8, 32, 64>(4096, 8, 5);
    run<8, 32, 128>(4096, 8, 5);
    run<8, 32, 256>(4096, 8, 5);
    run<8, 64, 128>(4096, 8, 5);
    run<16, 64, 256>(512, 16, 5);
    run<16, 64, 128>(512, 16, 5);
    run<16, 128, 128>(512, 16, 5);
    run<16, 32, 128>(512, 16, 5);
    run<32, 256, 256, false, true>(1, 32, 5);
    run<32, 512, 512, false, true>(1, 32, 5);
    run<32, 128, 128, false, true>(1, 32, 5);
    return 0;
}
