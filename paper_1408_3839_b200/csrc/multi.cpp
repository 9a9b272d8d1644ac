// multi.cpp — several GPUs of one process behind the C-ABI.
//
// The reference's only parallelism is parallel_for over the k-points of the periodic
// spectrum (parallel.hpp:15-32, eigensolver.cpp:95-120) and results must not depend on the
// worker count (test_eigensolver.cpp:125-131). lt_mctx holds one lt_ctx per device and an
// in-process NCCL communicator over them (ncclCommInitAll). lt_solve_core_multi runs the
// whole path with
//   LT_SPLIT_KPOINTS   : every device assembles H, S (small, latency-bound) and solves its
//                        contiguous k-range; one ncclAllGather of the padded eigenvalue
//                        shards restores the k-lexicographic spectrum;
//   LT_SPLIT_RANKTERMS : the nuclear operator is a rank-R_tot sum (galerkin.cpp:275-283):
//                        device q assembles the terms of its range (device 0 adds 0.5
//                        Laplace) into a partial H, one ncclAllReduce (sum) completes
//                        H = 0.5 Lap - Nuc, S = Mass is complete everywhere; then the
//                        k-point shards and the all-gather as above.
// Box systems do not shard their spectrum (one dense pencil): device 0 solves it (after
// the all-reduce in the rank-term split). Eigenvalues are bitwise identical to one device
// for the k-point split (each k-point is solved by the same kernel on some device).
// NCCL is loaded at lt_create_multi time (dlopen), so single-GPU use never touches it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "latham_b200.h"

namespace {

struct Nccl {
    void* h = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            n.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (n.h) break;
        }
        if (!n.h) return;
        n.CommInitAll = reinterpret_cast<decltype(n.CommInitAll)>(dlsym(n.h, "ncclCommInitAll"));
        n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(dlsym(n.h, "ncclCommDestroy"));
        n.AllGather = reinterpret_cast<decltype(n.AllGather)>(dlsym(n.h, "ncclAllGather"));
        n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(dlsym(n.h, "ncclAllReduce"));
        n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(dlsym(n.h, "ncclGroupStart"));
        n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(dlsym(n.h, "ncclGroupEnd"));
        n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(dlsym(n.h, "ncclGetErrorString"));
    });
    return n;
}

struct Fail : std::runtime_error {
    lt_status code;
    Fail(lt_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

}  // namespace
extern "C" void lt_internal_set_error(const char* msg);  // engine.cu: lt_last_error() of this thread
namespace {

void ck(lt_status s) {
    if (s != LT_OK) throw Fail(s, lt_last_error());
}
void cu(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Fail(LT_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
void nc(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        const char* m = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
        throw Fail(LT_ECUDA, std::string(what) + ": " + m);
    }
}

template <class F>
lt_status guarded(F&& f) {
    try {
        f();
        return LT_OK;
    } catch (const Fail& e) {
        lt_internal_set_error(e.what());
        return e.code;
    } catch (const std::exception& e) {
        lt_internal_set_error(e.what());
        return LT_EGENERIC;
    }
}

// contiguous k-range [begin, end) of shard q of world (sizes differ by at most one)
void shard(int64_t K, int q, int world, int64_t& b, int64_t& e) {
    const int64_t base = K / world, extra = K % world;
    b = q * base + std::min<int64_t>(q, extra);
    e = b + base + (q < extra ? 1 : 0);
}

// run f(i) on one host thread per device (the per-device calls synchronise their stream)
template <class F>
void per_device(int ndev, F&& f) {
    std::vector<std::thread> th;
    std::vector<std::string> err(static_cast<size_t>(ndev));
    std::vector<lt_status> code(static_cast<size_t>(ndev), LT_OK);
    for (int i = 0; i < ndev; ++i)
        th.emplace_back([&, i] {
            try {
                f(i);
            } catch (const Fail& e) {
                code[static_cast<size_t>(i)] = e.code;
                err[static_cast<size_t>(i)] = e.what();
            } catch (const std::exception& e) {
                code[static_cast<size_t>(i)] = LT_EGENERIC;
                err[static_cast<size_t>(i)] = e.what();
            }
        });
    for (auto& t : th) t.join();
    for (int i = 0; i < ndev; ++i)  // the lowest failing device reports (deterministic)
        if (code[static_cast<size_t>(i)] != LT_OK) throw Fail(code[static_cast<size_t>(i)], err[static_cast<size_t>(i)]);
}

}  // namespace

struct lt_mctx {
    std::vector<int> devices;
    std::vector<lt_ctx*> ctx;
    std::vector<ncclComm_t> comm;
};

extern "C" {

lt_status lt_create_multi(const int* devices, int ndev, lt_mctx** out) {
    return guarded([&] {
        if (!devices || ndev < 1 || !out) throw Fail(LT_EDIM, "lt_create_multi: need at least one device");
        Nccl& n = nccl();
        if (!n.CommInitAll || !n.AllGather || !n.AllReduce || !n.GroupStart || !n.GroupEnd)
            throw Fail(LT_ECUDA, "lt_create_multi: NCCL (libnccl.so.2) could not be loaded");
        auto m = std::make_unique<lt_mctx>();
        m->devices.assign(devices, devices + ndev);
        try {
            for (int i = 0; i < ndev; ++i) {
                lt_ctx* c = nullptr;
                ck(lt_create(devices[i], &c));
                m->ctx.push_back(c);
            }
            m->comm.assign(static_cast<size_t>(ndev), nullptr);
            nc(n.CommInitAll(m->comm.data(), ndev, devices), "ncclCommInitAll");
        } catch (...) {
            for (auto* c : m->ctx) lt_destroy(c);
            throw;
        }
        *out = m.release();
    });
}

void lt_destroy_multi(lt_mctx* m) {
    if (!m) return;
    for (auto& c : m->comm)
        if (c && nccl().CommDestroy) nccl().CommDestroy(c);
    for (auto* c : m->ctx) lt_destroy(c);
    delete m;
}

int lt_multi_ndev(const lt_mctx* m) { return m ? static_cast<int>(m->ctx.size()) : 0; }

lt_ctx* lt_multi_ctx(lt_mctx* m, int i) {
    return (m && i >= 0 && i < static_cast<int>(m->ctx.size())) ? m->ctx[static_cast<size_t>(i)] : nullptr;
}

lt_status lt_solve_core_multi(lt_mctx* m, const lt_system* sys, int periodic, int split, double* eig_host,
                              int64_t* info) {
    return guarded([&] {
        if (!m || !sys || !eig_host) throw Fail(LT_EDIM, "solve_core_multi: null argument");
        if (split != LT_SPLIT_KPOINTS && split != LT_SPLIT_RANKTERMS)
            throw Fail(LT_EDIM, "solve_core_multi: unknown split");
        const int P = static_cast<int>(m->ctx.size());
        Nccl& n = nccl();
        std::vector<lt_sysdev*> sd(static_cast<size_t>(P), nullptr);
        std::vector<int64_t> lay(8 * static_cast<size_t>(P), 0);
        struct Bufs {
            double* H = nullptr;
            double* S = nullptr;
            double* eig = nullptr;   // full-size eigenvalue buffer (k-points at their global offset)
            double* send = nullptr;  // padded shard
            double* recv = nullptr;  // [P][slot] gathered shards
        };
        std::vector<Bufs> bufs(static_cast<size_t>(P));
        auto cleanup = [&] {
            for (int i = 0; i < P; ++i) {
                cudaSetDevice(m->devices[static_cast<size_t>(i)]);
                Bufs& b = bufs[static_cast<size_t>(i)];
                for (double* p : {b.H, b.S, b.eig, b.send, b.recv})
                    if (p) cudaFree(p);
                if (sd[static_cast<size_t>(i)]) lt_sys_free(sd[static_cast<size_t>(i)]);
            }
        };
        try {
            // layout (L0, blocks, N_b, K, m0, R_tot, doubles per operator, eigenvalues per k)
            per_device(P, [&](int i) {
                cu(cudaSetDevice(m->devices[static_cast<size_t>(i)]), "cudaSetDevice");
                ck(lt_sys_upload(m->ctx[static_cast<size_t>(i)], sys, &sd[static_cast<size_t>(i)]));
                ck(lt_core_layout(m->ctx[static_cast<size_t>(i)], sd[static_cast<size_t>(i)], periodic,
                                  lay.data() + 8 * i, nullptr));
            });
            const int64_t K = periodic ? lay[3] : 1, per_k = lay[7], count = lay[6], Rtot = lay[5];
            const int64_t total = K * per_k;
            int64_t slot = 0;
            for (int q = 0; q < P; ++q) {
                int64_t b, e;
                shard(K, q, P, b, e);
                slot = std::max(slot, e - b);
            }
            const size_t slot_n = static_cast<size_t>(slot * per_k);
            per_device(P, [&](int i) {
                cu(cudaSetDevice(m->devices[static_cast<size_t>(i)]), "cudaSetDevice");
                Bufs& b = bufs[static_cast<size_t>(i)];
                cu(cudaMalloc(&b.eig, sizeof(double) * static_cast<size_t>(total)), "cudaMalloc");
                cu(cudaMalloc(&b.send, sizeof(double) * std::max<size_t>(1, slot_n)), "cudaMalloc");
                cu(cudaMalloc(&b.recv, sizeof(double) * std::max<size_t>(1, slot_n * static_cast<size_t>(P))),
                   "cudaMalloc");
                if (split == LT_SPLIT_RANKTERMS) {
                    cu(cudaMalloc(&b.H, sizeof(double) * static_cast<size_t>(count)), "cudaMalloc");
                    cu(cudaMalloc(&b.S, sizeof(double) * static_cast<size_t>(count)), "cudaMalloc");
                }
            });
            if (split == LT_SPLIT_RANKTERMS) {
                // partial H per device (rank terms of its range, 0.5 Laplace on device 0)
                per_device(P, [&](int i) {
                    cu(cudaSetDevice(m->devices[static_cast<size_t>(i)]), "cudaSetDevice");
                    int64_t r0, r1;
                    shard(Rtot, i, P, r0, r1);
                    Bufs& b = bufs[static_cast<size_t>(i)];
                    ck(lt_assemble_core_dev(m->ctx[static_cast<size_t>(i)], sd[static_cast<size_t>(i)], periodic, r0,
                                            r1, i == 0 ? 1 : 0, b.H, b.S));
                });
                nc(n.GroupStart(), "ncclGroupStart");
                for (int i = 0; i < P; ++i) {
                    Bufs& b = bufs[static_cast<size_t>(i)];
                    nc(n.AllReduce(b.H, b.H, static_cast<size_t>(count), ncclFloat64, ncclSum,
                                   m->comm[static_cast<size_t>(i)],
                                   static_cast<cudaStream_t>(lt_stream(m->ctx[static_cast<size_t>(i)]))),
                       "ncclAllReduce");
                }
                nc(n.GroupEnd(), "ncclGroupEnd");
            }
            // spectrum: k-point shards (box: device 0 solves the dense pencil)
            per_device(P, [&](int i) {
                cu(cudaSetDevice(m->devices[static_cast<size_t>(i)]), "cudaSetDevice");
                lt_ctx* c = m->ctx[static_cast<size_t>(i)];
                Bufs& b = bufs[static_cast<size_t>(i)];
                int64_t kb = 0, ke = K;
                if (periodic) shard(K, i, P, kb, ke);
                const bool solves = periodic ? (kb < ke) : (i == 0);
                if (solves) {
                    if (split == LT_SPLIT_RANKTERMS)
                        ck(lt_spectrum_dev(c, sd[static_cast<size_t>(i)], periodic, b.H, b.S, b.eig, kb, ke));
                    else
                        ck(lt_solve_core_dev(c, sd[static_cast<size_t>(i)], periodic, b.eig, kb, ke,
                                             i == 0 ? info : nullptr));
                }
                const cudaStream_t st = static_cast<cudaStream_t>(lt_stream(c));
                cu(cudaMemsetAsync(b.send, 0, sizeof(double) * std::max<size_t>(1, slot_n), st), "cudaMemsetAsync");
                if (solves && periodic)
                    cu(cudaMemcpyAsync(b.send, b.eig + kb * per_k, sizeof(double) * static_cast<size_t>((ke - kb) * per_k),
                                       cudaMemcpyDeviceToDevice, st),
                       "cudaMemcpyAsync");
                else if (solves)
                    cu(cudaMemcpyAsync(b.send, b.eig, sizeof(double) * static_cast<size_t>(total),
                                       cudaMemcpyDeviceToDevice, st),
                       "cudaMemcpyAsync");
            });
            // one all-gather of the padded shards (every device ends with the whole spectrum)
            nc(n.GroupStart(), "ncclGroupStart");
            for (int i = 0; i < P; ++i) {
                Bufs& b = bufs[static_cast<size_t>(i)];
                nc(n.AllGather(b.send, b.recv, std::max<size_t>(1, slot_n), ncclFloat64, m->comm[static_cast<size_t>(i)],
                               static_cast<cudaStream_t>(lt_stream(m->ctx[static_cast<size_t>(i)]))),
                   "ncclAllGather");
            }
            nc(n.GroupEnd(), "ncclGroupEnd");
            cu(cudaSetDevice(m->devices[0]), "cudaSetDevice");
            std::vector<double> g(slot_n * static_cast<size_t>(P));
            const cudaStream_t st0 = static_cast<cudaStream_t>(lt_stream(m->ctx[0]));
            cu(cudaMemcpyAsync(g.data(), bufs[0].recv, sizeof(double) * g.size(), cudaMemcpyDeviceToHost, st0),
               "cudaMemcpyAsync");
            cu(cudaStreamSynchronize(st0), "cudaStreamSynchronize");
            if (periodic) {
                for (int q = 0; q < P; ++q) {
                    int64_t b, e;
                    shard(K, q, P, b, e);
                    std::memcpy(eig_host + b * per_k, g.data() + static_cast<size_t>(q) * slot_n,
                                sizeof(double) * static_cast<size_t>((e - b) * per_k));
                }
            } else {
                std::memcpy(eig_host, g.data(), sizeof(double) * static_cast<size_t>(total));
            }
            if (info && split == LT_SPLIT_RANKTERMS) {
                info[0] = lay[0];
                info[4] = Rtot;
                info[5] = lay[2];
                info[6] = lay[3];
            }
        } catch (...) {
            cleanup();
            throw;
        }
        cleanup();
    });
}

}  // extern "C"
