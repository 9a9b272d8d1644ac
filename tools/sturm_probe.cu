// Cycles per step of Sturm-count recurrence variants in one warp (and 4 / 8 warps per SM):
// where the multisection's per-step cost comes from. Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/sturm_probe.cu -o tools/sturm_probe
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 32;

template <int V, int Q>
__global__ void k(const double* d, const double* e2, double x0, int reps, long long* out, int* sink) {
    __shared__ double sd[N], se[N];
    if (threadIdx.x < N) {
        sd[threadIdx.x] = d[threadIdx.x];
        se[threadIdx.x] = e2[threadIdx.x];
    }
    __syncthreads();
    double dr[N], er[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
        dr[i] = sd[i];
        er[i] = se[i];
    }
    double x[Q];
#pragma unroll
    for (int j = 0; j < Q; ++j) x[j] = x0 + 1e-3 * (threadIdx.x * Q + j);
    int tot = 0;
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        double pv[Q], cv[Q];
        int cn[Q];
#pragma unroll
        for (int j = 0; j < Q; ++j) {
            pv[j] = 1.0;
            cv[j] = dr[0] - x[j];
            cn[j] = 0;
        }
#pragma unroll
        for (int i = 1; i < N; ++i) {
#pragma unroll
            for (int j = 0; j < Q; ++j) {
                double nx;
                if (V == 0) {  // DFMA chain only (two-term), no count
                    nx = fma(dr[i] - x[j], cv[j], -er[i - 1]);
                } else if (V == 1) {  // three-term, no count
                    nx = fma(dr[i] - x[j], cv[j], -er[i - 1] * pv[j]);
                } else if (V == 2) {  // three-term + hi-word sign count (current)
                    nx = fma(dr[i] - x[j], cv[j], -er[i - 1] * pv[j]);
                    cn[j] += static_cast<int>(static_cast<unsigned>(__double2hiint(nx) ^ __double2hiint(cv[j])) >> 31);
                } else if (V == 3) {  // three-term + FP64 compare count
                    nx = fma(dr[i] - x[j], cv[j], -er[i - 1] * pv[j]);
                    cn[j] += ((nx < 0.0) != (cv[j] < 0.0)) ? 1 : 0;
                } else if (V == 5) {  // three-term, sign count of the previous pair after the new DFMA
                    nx = fma(dr[i] - x[j], cv[j], -er[i - 1] * pv[j]);
                    cn[j] += static_cast<int>(static_cast<unsigned>(__double2hiint(pv[j]) ^ __double2hiint(cv[j])) >> 31);
                } else if (V == 6) {  // sign bits collected into a mask, counted once per chain
                    nx = fma(dr[i] - x[j], cv[j], -er[i - 1] * pv[j]);
                    cn[j] |= static_cast<int>(static_cast<unsigned>(__double2hiint(cv[j])) >> 31) << i;
                } else {  // two-term ratio form with MUFU rcp: q = d - x - e2 / q
                    double r;
                    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(cv[j]));
                    nx = fma(-er[i - 1], r, dr[i] - x[j]);
                    cn[j] += static_cast<int>(static_cast<unsigned>(__double2hiint(nx)) >> 31);
                }
                pv[j] = cv[j];
                cv[j] = nx;
            }
        }
#pragma unroll
        for (int j = 0; j < Q; ++j) {
            if (V == 6) cn[j] = __popc(cn[j] ^ (cn[j] << 1));
            tot += cn[j] + (cv[j] > 1e300 ? 1 : 0);
            x[j] += (cn[j] & 1) ? 1e-12 : ((__double2hiint(cv[j]) & 1) ? -1e-12 : 2e-12);  // the next round depends on this one
        }
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = t1 - t0;
    if (tot == -1) *sink = tot;
}

template <int V, int Q>
static void run(const char* name, int threads, double* d, double* e, long long* out, int* sink) {
    const int reps = 200;
    k<V, Q><<<1, threads>>>(d, e, -0.3, 10, out, sink);
    k<V, Q><<<1, threads>>>(d, e, -0.3, reps, out, sink);
    long long c;
    cudaMemcpy(&c, out, sizeof(c), cudaMemcpyDeviceToHost);
    std::printf("%-34s Q=%d threads %4d: %6.1f cycles per step (per Q-batch)\n", name, Q, threads, double(c) / reps / (N - 1));
}

int main() {
    double hd[N], he[N];
    for (int i = 0; i < N; ++i) {
        hd[i] = 0.3 * ((i * 7919) % 13 - 6) / 6.0;
        he[i] = 0.1 + 0.05 * ((i * 104729) % 7) / 7.0;
    }
    double *d, *e;
    long long* out;
    int* sink;
    cudaMalloc(&d, sizeof(hd));
    cudaMalloc(&e, sizeof(he));
    cudaMalloc(&out, 8);
    cudaMalloc(&sink, 4);
    cudaMemcpy(d, hd, sizeof(hd), cudaMemcpyHostToDevice);
    cudaMemcpy(e, he, sizeof(he), cudaMemcpyHostToDevice);
    for (int th : {32, 256}) {
        run<0, 1>("dfma chain", th, d, e, out, sink);
        run<1, 1>("three-term", th, d, e, out, sink);
        run<2, 1>("three-term + hi-word count", th, d, e, out, sink);
        run<3, 1>("three-term + compare count", th, d, e, out, sink);
        run<4, 1>("ratio + MUFU rcp", th, d, e, out, sink);
        run<1, 2>("three-term", th, d, e, out, sink);
        run<2, 2>("three-term + hi-word count", th, d, e, out, sink);
        run<3, 2>("three-term + compare count", th, d, e, out, sink);
        run<2, 4>("three-term + hi-word count", th, d, e, out, sink);
        run<5, 2>("three-term + delayed count", th, d, e, out, sink);
        run<6, 2>("three-term + sign mask", th, d, e, out, sink);
        run<5, 4>("three-term + delayed count", th, d, e, out, sink);
        run<6, 4>("three-term + sign mask", th, d, e, out, sink);
        run<5, 1>("three-term + delayed count", th, d, e, out, sink);
    }
    std::printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
