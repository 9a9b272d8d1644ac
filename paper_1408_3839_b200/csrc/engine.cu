// engine.cu — context, device memory, pipeline orchestration and the C-ABI
// (include/latham_b200.h). The pipeline for one system:
//
//   L0 scan (device) -> 1 small D2H -> host integer plan ->
//   sinc | master panels + lattice window sums | pwc/pwl profiles | FEM tables |
//   nuclear contraction (direct / fold / box S2) | fused combine into H, S ->
//   periodic: sparse lattice DFT of H and S, batched pencils ; box: dense pencil
//
// All of it is stream-ordered on the context's stream; the only host
// synchronisations are the L0 read-back and the final D2H of the results.
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <chrono>
#include <array>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <numeric>
#include <set>
#include <string>
#include <vector>

#include "lt_internal.cuh"

namespace lt {

static thread_local std::string g_err;

Arena::~Arena() {
    for (auto& kv : bufs_)
        if (kv.second.p) cudaFree(kv.second.p);
}

void* Arena::raw(const std::string& key, size_t bytes) {
    Buf& b = bufs_[key];
    if (b.cap < bytes) {
        if (b.p) LT_CU(cudaFree(b.p));
        b.p = nullptr;
        size_t cap = std::max<size_t>(bytes, 256);
        cap = cap + cap / 4;
        LT_CU(cudaMalloc(&b.p, cap));
        b.cap = cap;
        ++gen_;
    }
    return b.p;
}

size_t Arena::bytes() const {
    size_t s = 0;
    for (auto& kv : bufs_) s += kv.second.cap;
    return s;
}

StageTimer::~StageTimer() {
    if (ref_) cudaEventDestroy(ref_);
    for (cudaEvent_t e : pool_) cudaEventDestroy(e);
}

cudaEvent_t StageTimer::get() {
    if (owned) {
        cudaEvent_t e;
        LT_CU(cudaEventCreate(&e));
        owned->push_back(e);
        return e;
    }
    if (used_ == pool_.size()) {
        cudaEvent_t e;
        LT_CU(cudaEventCreate(&e));
        pool_.push_back(e);
    }
    return pool_[used_++];
}

// while capturing, timing events must be external event-record nodes (a plain record
// inside a capture only expresses a dependency and cannot be timed afterwards)
static void record_timing_event(cudaEvent_t e, cudaStream_t st, bool capturing) {
    if (capturing) LT_CU(cudaEventRecordWithFlags(e, st, cudaEventRecordExternal));
    else LT_CU(cudaEventRecord(e, st));
}

void StageTimer::begin(cudaStream_t st, const char* name) {
    open_ = get();
    open_name_ = name;
    record_timing_event(open_, st, owned != nullptr);
}

void StageTimer::end(cudaStream_t st) {
    cudaEvent_t b = get();
    record_timing_event(b, st, owned != nullptr);
    pending_.push_back({open_name_, open_, b, st, ref_});
}

void StageTimer::mark_ref(cudaStream_t st) {
    if (!on) return;
    if (!ref_) LT_CU(cudaEventCreate(&ref_));
    LT_CU(cudaEventRecord(ref_, st));
    timeline.clear();
}

void StageTimer::collect() {
    for (auto& p : pending_) {
        float ms = 0.f;
        LT_CU(cudaEventSynchronize(p.b));
        LT_CU(cudaEventElapsedTime(&ms, p.a, p.b));
        auto& t = totals[p.name];
        t.first += ms;
        t.second += 1;
        if (p.ref) {
            float t0 = 0.f, t1 = 0.f;
            LT_CU(cudaEventElapsedTime(&t0, p.ref, p.a));
            LT_CU(cudaEventElapsedTime(&t1, p.ref, p.b));
            timeline.push_back({p.name, p.st, t0, t1});
        }
    }
    pending_.clear();
    used_ = 0;
}

void StageTimer::reset() {
    collect();
    totals.clear();
}

}  // namespace lt

using namespace lt;

struct GraphCache {
    cudaGraphExec_t exec = nullptr;
    std::vector<int64_t> key, seen;
    int64_t launches = 0;
    // stage-timing events captured as graph nodes (timed graphs only)
    std::vector<cudaEvent_t> events;
    std::vector<StageTimer::Pending> timing;
    void drop_events() {
        for (cudaEvent_t e : events) cudaEventDestroy(e);
        events.clear();
        timing.clear();
    }
    ~GraphCache() {
        if (exec) cudaGraphExecDestroy(exec);
        drop_events();
    }
};

// Dense block-diagonal form [K][mm] (complex) of a generating tensor: compressed per-axis
// index sets and the slot map (device) prepared on the host by prepare_dft.
struct DftPrep {
    Index dims[3]{1, 1, 1};
    Index ext[3]{1, 1, 1};
    Index ncomp[3]{1, 1, 1};
    Index nblk = 0, m0 = 0, maxsz = 0;
    int* slot2blk = nullptr;  // compressed position -> stored block (-1: zero block)
    bool ident = false;       // slot2blk[q] == q for every q
    int64_t* comp[3]{nullptr, nullptr, nullptr};
    std::string tag;
};

// host-side products of one (system, periodic, L0): plan, uploaded window starts and DFT
// index maps (device pointers), valid while prep_epoch and the arena generation match
struct CorePrep {
    bool valid = false;
    std::vector<int64_t> key;
    Plan p;
    DftPrep dp;
    int64_t* s0d = nullptr;
    uint64_t epoch = 0, gen = 0;
};

struct lt_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cusolverDnHandle_t solver = nullptr;
    cublasHandle_t blas = nullptr;
    unsigned* pencil_done = nullptr;  // self-resetting arrival counter of the in-kernel read-back
    Arena arena;
    int64_t launches = 0;
    StageTimer timer;
    // CUDA graphs of the L0 sequence and of the post-L0 launch sequence
    bool graphs = true;
    GraphCache l0graph, coregraph, fullgraph;  // fullgraph: L0 + post-L0 under speculation
    GraphCache asmgraph, specgraph;            // multi-GPU phases: assembly shard, spectrum
    int* pinned = nullptr;  // small pinned read-back buffer
    // side streams for independent branches of the assembly (captured into the same graph
    // as parallel branches) and the fork/join events between them
    // 0, 1: assembly branches; 2: L0 check under speculation; 3: second FEM fold
    cudaStream_t aux[4]{nullptr, nullptr, nullptr, nullptr};
    // fork/join points of run_assembly (0-5, 9-12), the L0 branch (6-7), external streams (8)
    cudaEvent_t ev[13]{};
    // pinned staging for the small per-call host<->device copies (system, window starts,
    // DFT index maps, eigenvalue read-back): async copies instead of pageable round trips.
    // Valid between stage_begin() (stream idle) and the end of the API call.
    char* stage = nullptr;
    size_t stage_cap = 0, stage_off = 0;
    bool stage_on = false;
    void stage_begin(size_t hint) {
        LT_CU(cudaStreamSynchronize(stream));
        stage_off = 0;
        stage_on = true;
        if (stage_cap < hint) {
            if (stage) LT_CU(cudaFreeHost(stage));
            stage_cap = std::max<size_t>(4u << 20, size_t(1) << (64 - __builtin_clzll(hint)));
            LT_CU(cudaHostAlloc(reinterpret_cast<void**>(&stage), stage_cap, cudaHostAllocDefault));
        }
    }
    void stage_end() { stage_on = false; }
    void* stage_alloc(size_t n) {
        if (!stage_on || stage_off + n > stage_cap) return nullptr;
        void* p = stage + stage_off;
        stage_off += (n + 255) / 256 * 256;
        return p;
    }
    // plan-table uploads (window starts, DFT maps) bump the epoch; solve_core_dev reuses
    // its uploaded tables while the epoch and the arena generation are unchanged
    uint64_t prep_epoch = 0;
    // the last lattice-DFT index maps per buffer tag: they depend on the lattice and the stored
    // offsets only (not on the basis exponents), so a scan over systems of one shape re-uses them
    struct DftCache {
        std::vector<std::array<Index, 3>> kidx;
        Index dims[3] = {0, 0, 0}, m0 = 0;
        uint64_t gen = 0;
        DftPrep P;
    };
    std::map<std::string, DftCache> dft_cache;
    CorePrep prep;
    // speculation on L0: the last (system, L0) pair the device computed
    std::vector<int64_t> spec_key;
    Index spec_L0 = -1;
    bool spec_active = false;  // the running solve uses a predicted L0
    // optional host-side timestamps (lt_set_diagnostics LT_DIAG_HOST_TIMING): enter / launched / synced / exit
    bool host_timing = false;
    double host_acc[4] = {0, 0, 0, 0};
    double graph_launch_us = 0.0, key_us = 0.0;
    int64_t n_replay = 0, n_capture = 0, n_eager = 0;
    int64_t host_n = 0;
    std::chrono::steady_clock::time_point host_t[5];
    void host_mark(int i) {
        if (host_timing) host_t[i] = std::chrono::steady_clock::now();
    }
    void host_collect() {
        if (!host_timing) return;
        for (int i = 0; i < 4; ++i)
            host_acc[i] += std::chrono::duration<double, std::micro>(host_t[i + 1] - host_t[i]).count();
        ++host_n;
    }
    // optional phase markers (lt_set_diagnostics LT_DIAG_PHASE_TIMING): events between the graph launches,
    // accumulated into the stage totals as phase_l0 / phase_gap / phase_post
    bool phase_timing = false;
    cudaEvent_t pev[4]{};
    void phase_mark(int i) {
        if (phase_timing) LT_CU(cudaEventRecord(pev[i], stream));
    }
    void phase_collect() {
        if (!phase_timing) return;
        LT_CU(cudaEventSynchronize(pev[3]));
        const char* names[3] = {"phase_l0", "phase_gap", "phase_post"};
        for (int i = 0; i < 3; ++i) {
            float ms = 0.f;
            LT_CU(cudaEventElapsedTime(&ms, pev[i], pev[i + 1]));
            auto& t = timer.totals[names[i]];
            t.first += ms;
            t.second += 1;
        }
    }
    Launch L() { return Launch{stream, &launches, &timer}; }
    Launch LA(int i) { return Launch{aux[i], &launches, &timer}; }
    // `to` waits for everything enqueued on `from` so far
    void join(int e, cudaStream_t from, cudaStream_t to) {
        LT_CU(cudaEventRecord(ev[e], from));
        LT_CU(cudaStreamWaitEvent(to, ev[e], 0));
    }
    int* pinned_state() {
        if (!pinned) LT_CU(cudaHostAlloc(reinterpret_cast<void**>(&pinned), 64 * sizeof(int), cudaHostAllocDefault));
        return pinned;
    }
};

// RAII: pinned staging valid for the duration of one API call
struct StageScope {
    lt_ctx* c;
    StageScope(lt_ctx* ctx, size_t hint) : c(ctx) { c->stage_begin(hint); }
    ~StageScope() { c->stage_end(); }
};

namespace lt {
// Replay a captured launch sequence when the key (every host-derived parameter, pointer
// and the arena generation) matches; capture on the second identical call (the first runs
// eagerly so the arena is sized and no allocation happens inside a capture).
template <class K, class F>
static void run_cached(lt_ctx* c, GraphCache& g, K&& keyfn, F&& enqueue) {
    // stage timing is captured too (event nodes inside the graph), keyed separately, so the
    // per-stage times come from the same graph execution as the untimed solve
    const bool allow = c->graphs;
    const auto tk = std::chrono::steady_clock::now();
    std::vector<int64_t> key = keyfn();
    if (c->host_timing)
        c->key_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - tk).count();
    key.push_back(c->timer.on ? 1 : 0);
    if (allow && g.exec && key == g.key) {
        const auto t0 = std::chrono::steady_clock::now();
        LT_CU(cudaGraphLaunch(g.exec, c->stream));
        if (c->host_timing)
            c->graph_launch_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
        ++c->n_replay;
        c->launches += g.launches;
        if (c->timer.on) c->timer.add_pending(g.timing);
        return;
    }
    if (allow && key == g.seen) {
        const int64_t l0 = c->launches;
        cudaGraph_t graph = nullptr;
        if (g.exec) cudaGraphExecDestroy(g.exec);
        g.exec = nullptr;
        g.drop_events();
        const size_t p0 = c->timer.pending_size();
        c->timer.owned = &g.events;
        LT_CU(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        try {
            enqueue();
        } catch (...) {
            c->timer.owned = nullptr;
            cudaStreamEndCapture(c->stream, &graph);
            if (graph) cudaGraphDestroy(graph);
            c->timer.take_pending(p0);
            throw;
        }
        c->timer.owned = nullptr;
        LT_CU(cudaStreamEndCapture(c->stream, &graph));
        g.timing = c->timer.take_pending(p0);
        const cudaError_t e = cudaGraphInstantiate(&g.exec, graph, 0);
        cudaGraphDestroy(graph);
        LT_CU(e);
        g.key = key;
        g.launches = c->launches - l0;
        LT_CU(cudaGraphLaunch(g.exec, c->stream));
        if (c->timer.on) c->timer.add_pending(g.timing);
        ++c->n_capture;
        return;
    }
    ++c->n_eager;
    enqueue();
    g.seen = keyfn();  // after the eager run: it may have grown the arena (new generation)
    g.seen.push_back(c->timer.on ? 1 : 0);
}
}  // namespace lt

struct lt_sysdev {
    HostSys hs;
    DevSys ds;
    void* mem = nullptr;
};

// separable coefficient metadata of a periodic operator (galerkin.hpp:52 `separable`),
// band-compressed: level l keeps slots s with lattice index kid[l][s]; vals[t][l][s][mm]
struct SepMeta {
    Index terms = 0, m0 = 0, S = 1;
    Index L[3]{1, 1, 1};
    std::vector<Index> kid[3];
    double* vals = nullptr;
    SepMeta() = default;
    SepMeta(const SepMeta&) = delete;
    SepMeta& operator=(const SepMeta&) = delete;
    ~SepMeta() {
        if (vals) cudaFree(vals);
    }
    size_t count() const { return static_cast<size_t>(terms * 3 * S * m0 * m0); }
};

struct lt_operator {
    int which = 0;  // 0 Laplace 1 Mass 2 Nuclear; core H uses 0 (Laplace first operand)
    bool periodic = false;
    Index m0 = 0;
    Index L[3]{1, 1, 1};
    Index band[3]{0, 0, 0};
    Index L0 = 0, coefficient_rank = 0, Nb = 0;
    std::vector<std::array<Index, 3>> kidx;  // periodic, std::map order
    double* data = nullptr;                  // device: dense Nb*Nb or nblk*m0*m0
    size_t count = 0;
    std::unique_ptr<SepMeta> sep;            // periodic: rank metadata
    ~lt_operator() {
        if (data) cudaFree(data);
    }
};

namespace lt {

template <class F>
static lt_status guarded(F&& f) {
    try {
        f();
        g_err.clear();
        return LT_OK;
    } catch (const Error& e) {
        g_err = e.what();
        return static_cast<lt_status>(e.code);
    } catch (const std::exception& e) {
        g_err = e.what();
        return LT_EGENERIC;
    }
}

static void upload(lt_ctx* c, void* dst, const void* src, size_t bytes) {
    if (!bytes) return;
    if (void* pin = c->stage_alloc(bytes)) {
        std::memcpy(pin, src, bytes);
        src = pin;
    }
    LT_CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
}

// pack the system arrays into one device block; dst (optional) is a caller-owned buffer
// of at least sysdev_bytes(); the H2D copy is stream-ordered on `st`
static size_t sysdev_bytes(const HostSys& h) {
    const size_t m0 = h.alpha.size(), nn = h.Z.size();
    size_t bytes = 16;
    for (size_t nb : {3 * nn * 8, nn * 8, 3 * m0 * 8, m0 * 8, 3 * m0 * 4}) bytes += (nb + 15) / 16 * 16;
    return bytes;
}

static lt_sysdev* make_sysdev(const lt_system* s, void* dst = nullptr, lt_ctx* c = nullptr) {
    auto sd = std::make_unique<lt_sysdev>();
    sd->hs = host_sys_from(s);
    const HostSys& h = sd->hs;
    const size_t m0 = h.alpha.size(), nn = h.Z.size();
    const size_t bytes = sysdev_bytes(h);
    if (dst) sd->mem = dst;
    else LT_CU(cudaMalloc(&sd->mem, bytes));
    char* p = static_cast<char*>(sd->mem);
    std::vector<char> host(bytes, 0);
    size_t at = 0;
    auto put = [&](const void* src, size_t nb) {
        std::memcpy(host.data() + at, src, nb);
        void* d = p + at;
        at += (nb + 15) / 16 * 16;
        return d;
    };
    sd->ds.m0 = static_cast<int>(m0);
    sd->ds.nnuc = static_cast<int>(nn);
    sd->ds.b = h.b;
    sd->ds.eps_ov = h.eps_ov;
    sd->ds.pos = static_cast<const double*>(put(h.pos.data(), 3 * nn * 8));
    sd->ds.Z = static_cast<const double*>(put(h.Z.data(), nn * 8));
    sd->ds.center = static_cast<const double*>(put(h.center.data(), 3 * m0 * 8));
    sd->ds.alpha = static_cast<const double*>(put(h.alpha.data(), m0 * 8));
    sd->ds.deg = static_cast<const int*>(put(h.deg.data(), 3 * m0 * 4));
    if (dst) upload(c, sd->mem, host.data(), at);
    else LT_CU(cudaMemcpy(sd->mem, host.data(), at, cudaMemcpyHostToDevice));
    return sd.release();
}

static std::vector<int64_t> graph_key(const HostSys& h, const Plan& p, bool periodic, Index kb, Index ke,
                                      const void* eig, const void* sysmem, uint64_t gen);

// ---------------------------------------------------------------------------
// L0 (gto_basis.cpp:87-126)
// ---------------------------------------------------------------------------
// L0 work of one system: direction classes, device buffers, and the launches of a shift
// chunk [s_begin, s_end) (init + per-direction sampling only with the first chunk)
struct L0Work {
    const lt_sysdev* sd = nullptr;
    int m0 = 0;
    Index n3[3]{}, off3[3]{}, boff3[3]{};
    int act_peak[3] = {0, 0, 0}, act_scan[3] = {0, 0, 0};
    bool any_peak = false, any_scan = false;
    OverlapBufs b;
    void init(const Launch& L) const { launch_overlap_init(L, b, m0); }
    void enqueue(const Launch& L, int s_begin, int s_end, bool first) const {
        if (first) launch_overlap_init(L, b, m0);
        if (any_scan) {
            if (first) launch_overlap_profiles(L, sd->ds, n3, off3, boff3, act_scan, b);
            launch_overlap_scan(L, sd->ds, n3, off3, boff3, act_scan, b, s_begin, s_end, !any_peak);
        }
        if (any_peak) launch_overlap_peak(L, sd->ds, n3, act_peak, b, s_begin, s_end, true);
    }
};

static L0Work l0_setup(lt_ctx* c, const lt_sysdev* sd) {
    const HostSys& h = sd->hs;
    L0Work w;
    w.sd = sd;
    w.m0 = static_cast<int>(h.m0());
    const Index m0 = h.m0();
    Index tot = 0, btot = 0;
    for (int l = 0; l < 3; ++l) {
        w.n3[l] = h.n[l];
        const Index width = 2 * 258 * h.n[l];
        w.off3[l] = tot;
        w.boff3[l] = btot;
        tot += m0 * width;
        btot += m0 * ((width + kL0Block - 1) / kL0Block);
    }
    // a direction whose grid, centres and degrees repeat an earlier one has identical
    // profiles: its scan answers are the same, so it is skipped (found[] is an OR over l)
    int active[3] = {1, 1, 1};
    for (int l = 1; l < 3; ++l)
        for (int q = 0; q < l && active[l]; ++q) {
            if (!active[q] || h.n[q] != h.n[l]) continue;
            bool same = true;
            for (Index mu = 0; mu < m0 && same; ++mu)
                same = std::memcmp(&h.center[3 * mu + q], &h.center[3 * mu + l], sizeof(double)) == 0 &&
                       h.deg[3 * mu + q] == h.deg[3 * mu + l];
            if (same) active[l] = 0;
        }
    // directions whose functions are all degree 0 take the exact peak-window search
    // (k_l0_peak); the others sample the profiles and scan them
    for (int l = 0; l < 3; ++l) {
        if (!active[l]) continue;
        bool deg0 = true;
        for (Index mu = 0; mu < m0; ++mu) deg0 = deg0 && h.deg[3 * mu + l] == 0;
        (deg0 ? w.act_peak : w.act_scan)[l] = 1;
        (deg0 ? w.any_peak : w.any_scan) = true;
    }
    w.b.prof = w.any_scan ? c->arena.get<double>("l0.prof", tot) : nullptr;
    w.b.bmax = w.any_scan ? c->arena.get<double>("l0.bmax", btot) : nullptr;
    w.b.nz = c->arena.get<unsigned>("l0.nz", 6 * m0);
    w.b.found = c->arena.get<int>("l0.found", 260);
    w.b.state = c->arena.get<int>("l0.state", 8);
    return w;
}

// L0 with the host reading it: the first 16-shift chunk (it decides L0 <= 14) as a
// replayable graph ending in the read-back, further chunks only if the rule is not done
static Index compute_L0(lt_ctx* c, const lt_sysdev* sd) {
    const L0Work w = l0_setup(c, sd);
    const Launch L = c->L();
    const int chunk = 16;
    int* st = c->pinned_state();
    run_cached(
        c, c->l0graph,
        [&]() { return graph_key(sd->hs, Plan{}, false, chunk, -1, st, sd->mem, c->arena.generation()); },
        [&]() {
            w.enqueue(L, 1, 1 + chunk, true);
            LT_CU(cudaMemcpyAsync(st, w.b.state, 4 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        });
    c->phase_mark(1);
    LT_CU(cudaStreamSynchronize(c->stream));
    int s_begin = 1 + chunk;
    while (!st[3] && s_begin < 257) {
        const int s_end = std::min(257, s_begin + chunk);
        w.enqueue(L, s_begin, s_end, false);
        LT_CU(cudaMemcpyAsync(st, w.b.state, 4 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        LT_CU(cudaStreamSynchronize(c->stream));
        s_begin = s_end;
    }
    return st[0];
}

// ---------------------------------------------------------------------------
// assembly
// ---------------------------------------------------------------------------
struct AsmOut {
    double* out0 = nullptr;  // H / single operator
    double* out1 = nullptr;  // S
    int64_t* kidx = nullptr;
};

enum Need : int { NEED_MS = 1, NEED_NUC = 2 };

// one assembly shard of the multi-GPU path: the nuclear rank terms
// [r0, r1) (weights outside are 0) and the Laplace part with weight kin (0.5 on the
// leading shard, 0 elsewhere); the shards' H sum to the full H, S is complete on each
struct CoreShard {
    Index r0 = 0, r1 = -1;
    double kin = 0.5;
};

// solve_core_dev phases: 0 assembly + spectrum (one graph), 1 assembly only into caller
// buffers (H, S), 2 spectrum only from caller buffers
struct CoreOpts {
    int phase = 0;
    CoreShard shard;
    double* H = nullptr;
    double* S = nullptr;
};


struct Work {
    double *t = nullptr, *w = nullptr, *potw = nullptr;
    double* pot[3]{};
    double* pwc[3]{};
    double* pwl[3]{};
    unsigned long long *pwc_lo[3]{}, *pwc_hi[3]{}, *pwl_lo[3]{}, *pwl_hi[3]{};
    double *massT[3]{}, *stiffT[3]{}, *T[3]{};
    double* N = nullptr;
};

// Directions whose every input is bitwise identical (grid counts, lattice extent, every
// nucleus and basis-centre coordinate, monomial degrees) produce bitwise identical
// panels, profiles and tables; they are computed once (src[l] = first such direction).
static void direction_sources(const HostSys& h, int src[3]) {
    for (int l = 0; l < 3; ++l) {
        src[l] = l;
        for (int q = 0; q < l; ++q) {
            if (src[q] != q) continue;
            bool same = h.n[l] == h.n[q] && h.nbar[l] == h.nbar[q] && h.L[l] == h.L[q];
            for (size_t v = 0; same && v < h.Z.size(); ++v) same = h.pos[3 * v + l] == h.pos[3 * v + q];
            for (size_t m = 0; same && m < h.alpha.size(); ++m)
                same = h.center[3 * m + l] == h.center[3 * m + q] && h.deg[3 * m + l] == h.deg[3 * m + q];
            if (same) {
                src[l] = q;
                break;
            }
        }
    }
}

// split-K factor: aim for ~4 CTAs per SM while keeping >= 32 contraction steps (two
// 16-deep tiles) per CTA: these GEMMs are load-latency bound, so more CTAs with fewer
// dependent tile loads each finish sooner; the fixed-order split reduction absorbs it
static int splits_for(long long tiles, long long len, int waves = 4) {
    int s = 1;
    while (tiles * s < waves * 148 && len / (s * 2) >= 32 && s < 512) s *= 2;
    return s;
}

// window starts of every (direction, nucleus) to the device (host part; not capturable)
static int64_t* upload_s0(lt_ctx* c, const Plan& p) {
    std::vector<int64_t> s0all;
    for (int l = 0; l < 3; ++l)
        for (Index v : p.d[l].s0) s0all.push_back(v);
    int64_t* s0d = c->arena.get<int64_t>("pot.s0", s0all.size() + 1);
    upload(c, s0d, s0all.data(), s0all.size() * sizeof(int64_t));
    ++c->prep_epoch;
    return s0d;
}

// flags: AS_GENERAL_NUC forces the per-direction nuclear tables (w.T, the reference's
// nucT layout) instead of the fused reassociations; AS_NO_FILL stops after the tables.
// AS_EMAJOR (periodic, several wrapped axes, mode 0): the Khatri-Rao combine writes H, S
// itself, entry-major ([mm][nblocks], for the fused lattice DFT), after the FEM join; no fill
enum AsmFlags : unsigned { AS_GENERAL_NUC = 1u, AS_NO_FILL = 2u, AS_BOX_SPLIT = 4u, AS_EMAJOR = 8u };
// AS_BOX_SPLIT (box, mode 0): S = Mass is filled on the FEM branch as soon as the mass tables
// exist and `s_hook` runs right after it on that branch (the dense pencil's Cholesky and
// L^-1 overlap the nuclear contraction); the main-stream fill writes H only.
using BranchHook = std::function<void(const Launch&)>;

// Cells [j0, j0 + J) of direction l's extended grid that hold every sampled support (pwl:
// nbar grid, align 0; pwc: n grid, align 0.5; functions sit in cell `margin`, galerkin.cpp:
// 127-149). A sample |x - c|^deg exp(-alpha (x - c)^2) survives the 1e-280 trim (k_profiles)
// only if alpha r^2 <= 644.8 + deg ln r, so r <= sqrt((650 + deg ln(max(1, extent))) / alpha)
// bounds it; one spare cell each side. The residue folds cover only this window: for long
// periodic chains the extended grid is (L + 2 margin) cells, almost all of them empty.
static void support_window(const HostSys& s, const Plan& p, int l, bool pwl, long long& j0, long long& J) {
    const DirPlan& d = p.d[l];
    const Index per = pwl ? d.nbar : d.n;
    const double step = pwl ? d.hbar : d.h;
    const long long cells = (pwl ? d.Gbar : d.G) / per;
    const double align = pwl ? 0.0 : 0.5;
    const double extent = step * static_cast<double>(cells * per) + s.b;
    const double base = static_cast<double>(p.margin * per);
    long long lo = cells, hi = -1;
    auto fdiv = [&](long long x) { return x >= 0 ? x / per : -((-x + per - 1) / per); };
    for (Index mu = 0; mu < s.m0(); ++mu) {
        const double r = std::sqrt((650.0 + s.deg[3 * mu + l] * std::log(std::max(1.0, extent))) / s.alpha[mu]);
        const double ic = (s.center[3 * mu + l] + 0.5 * s.b) / step + base - align;
        const double ilo = std::floor(ic - r / step) - 2.0, ihi = std::ceil(ic + r / step) + 2.0;
        lo = std::min(lo, ilo < -1e15 ? -1 : fdiv(static_cast<long long>(ilo)));
        hi = std::max(hi, ihi > 1e15 ? cells : fdiv(static_cast<long long>(ihi)));
    }
    lo = std::max(0LL, lo - 1);
    hi = std::min(cells - 1, hi + 1);
    if (hi < lo) {  // no function reaches this grid: an empty one-cell window
        lo = 0;
        hi = 0;
    }
    j0 = lo;
    J = hi - lo + 1;
}

static void run_assembly(lt_ctx* c, const lt_sysdev* sd, const Plan& p, int need, int mode, AsmOut out,
                         Work* wout = nullptr, const int64_t* s0_dev = nullptr, unsigned flags = 0,
                         const CoreShard& shard = CoreShard{}, const BranchHook* s_hook = nullptr,
                         const BranchHook* root_hook = nullptr) {
    // Three concurrent branches (parallel branches of the captured graph):
    //   main   : sinc -> potential of the 1st, 3rd distinct direction -> nuclear -> fill
    //   aux[1] : potential of the 2nd distinct direction (joins main before the nuclear part)
    //   aux[0] : profiles -> FEM tables (profiles join main before the nuclear part, the
    //            tables before the fill)
    const Launch L = c->L();
    // stage-timing mode runs the branches back to back on the main stream, so each stage's
    // events bracket that kernel alone (concurrent branches would share SMs)
    const bool serial = c->timer.on;
    // the FEM branch normally runs on the low-priority side stream; when it feeds the box
    // pencil's Cholesky (AS_BOX_SPLIT: the S side is then the critical path) it takes the
    // high-priority one and the second potential the low-priority one
    const bool fem_hi = (flags & AS_BOX_SPLIT) && !p.periodic;
    const int fi = fem_hi ? 1 : 0, pi = fem_hi ? 0 : 1;
    const Launch LF = serial ? L : c->LA(fi), LP = serial ? L : c->LA(pi);
    const Index m0 = p.m0, mm = m0 * m0, RN = p.RN, Rtot = p.Rtot;
    Arena& A = c->arena;
    int src[3];
    direction_sources(sd->hs, src);
    Work w{};
    const int64_t* s0d = nullptr;
    const bool nuc = need & NEED_NUC, ms = need & NEED_MS;
    if (nuc) s0d = s0_dev ? s0_dev : upload_s0(c, p);
    // Trivial-direction panels could be evaluated inside k_triv_gemm (TrivJob.pot = null):
    // measured slower (erf pairs in the GEMM loader, repeated per N tile), so every panel is
    // materialised by the master-free window kernels.
    constexpr bool fused_nuc = false;
    // profiles (galerkin.cpp:127-149), distinct directions only. Every branch forks after one
    // root kernel: measured on B200, a second root branch of this graph starts 7-11 us late
    // (whichever is captured second), a branch forked after the root does not
    ProfileJob jobs[6];
    int nj = 0;
    for (int l = 0; l < 3; ++l) {
        if (src[l] != l) continue;
        const DirPlan& d = p.d[l];
        if (nuc) {
            ProfileJob j;
            j.grid = d.G;
            j.per_cell = d.n;
            j.cell_index = p.margin;
            j.step = d.h;
            j.align = 0.5;
            j.dir = l;
            // slack on both sides: the Toeplitz TMA view of the resident Hankel kernel
            const Index pad = d.band * d.n, padb = (d.band + 260) * d.n;
            j.values = w.pwc[l] = A.get<double>("prof.pwc" + std::to_string(l), m0 * d.G + pad + padb) + pad;
            j.lo = w.pwc_lo[l] = A.get<unsigned long long>("prof.pwc_lo" + std::to_string(l), m0);
            j.hi = w.pwc_hi[l] = A.get<unsigned long long>("prof.pwc_hi" + std::to_string(l), m0);
            jobs[nj++] = j;
        }
        if (ms) {
            ProfileJob j;
            j.grid = d.Gbar;
            j.per_cell = d.nbar;
            j.cell_index = p.margin;
            j.step = d.hbar;
            j.align = 0.0;
            j.dir = l;
            j.values = w.pwl[l] = A.get<double>("prof.pwl" + std::to_string(l), m0 * d.Gbar);
            j.lo = w.pwl_lo[l] = A.get<unsigned long long>("prof.pwl_lo" + std::to_string(l), m0);
            j.hi = w.pwl_hi[l] = A.get<unsigned long long>("prof.pwl_hi" + std::to_string(l), m0);
            jobs[nj++] = j;
        }
    }
    for (int l = 0; l < 3; ++l)
        if (src[l] != l) {
            w.pwc[l] = w.pwc[src[l]];
            w.pwc_lo[l] = w.pwc_lo[src[l]];
            w.pwc_hi[l] = w.pwc_hi[src[l]];
            w.pwl[l] = w.pwl[src[l]];
            w.pwl_lo[l] = w.pwl_lo[src[l]];
            w.pwl_hi[l] = w.pwl_hi[src[l]];
        }
    w.t = A.get<double>("sinc.t", RN);
    w.w = A.get<double>("sinc.w", RN);
    w.potw = A.get<double>("sinc.potw", Rtot);
    // nodes and weights Z_v w_q: the graph's single root (the master kernels evaluate their
    // nodes in place; the weights are first needed by the nuclear part)
    // The graph's single root heads the longer chain: lattices with several wrapped axes spend
    // longest in the FEM folds and the per-axis nuclear folds, both behind the profiles (c5:
    // 148 vs 160 us with the sinc first); otherwise the potentials' masters are the long head
    // (c4: 238 vs 250 us with the profiles first). Measured on B200 (tools/ab.sh).
    int nwrap = 0;
    for (int l = 0; l < 3; ++l) nwrap += p.d[l].L > 1;
    const bool prof_root = p.periodic && nwrap >= 2;
    if (prof_root) launch_profiles(L, sd->ds, jobs, nj, 1e-280);
    else launch_sinc(L, p.M, sd->ds, w.t, w.w, w.potw, shard.r0, shard.r1);
    c->join(0, c->stream, c->aux[fi]);
    c->join(1, c->stream, c->aux[pi]);
    if (root_hook) (*root_hook)(L);  // the L0 check under speculation: its own branch
    // (with the profiles as the root the sinc kernel goes ahead of the FEM chain, which has slack:
    // on the second potential's stream it delayed that master and its lattice sum, the head of
    // the nuclear chain, by its own 2 us)
    if (prof_root) launch_sinc(LF, p.M, sd->ds, w.t, w.w, w.potw, shard.r0, shard.r1);
    else launch_profiles(LF, sd->ds, jobs, nj, 1e-280);
    if (nuc) {
        int nth = 0;
        for (int l = 0; l < 3; ++l) {
            if (src[l] != l) {
                w.pot[l] = w.pot[src[l]];
                continue;
            }
            const DirPlan& d = p.d[l];
            if (fused_nuc && d.L == 1) {  // consumed by k_triv_gemm straight from the master cells
                w.pot[l] = nullptr;
                continue;
            }
            const Launch& LL = (nth++ == 1) ? LP : L;
            w.pot[l] = A.get<double>("pot.panel" + std::to_string(l), d.pot_rows * Rtot);
            if ((d.nsum == 1 && p.nnuc == 1) || (d.nsum >= 8 && d.pot_rows <= d.n && p.nnuc <= 2)) {
                // a single window copy of one nucleus: each master cell is read once, so it
                // is evaluated in the copy kernel instead of being materialised first. The
                // periodic cell window (one output per residue class) of <= 2 nuclei reads each
                // cell at most twice: evaluating in place costs less than a serial master node
                launch_potential_fused(LL, d.mrows, d.h, p.M, RN, p.nnuc, s0d + l * p.nnuc, d.nsum, d.n,
                                       d.pot_rows, w.pot[l]);
            } else {
                // the master panel once (massively parallel), then the windows read it: a cell
                // serves every nucleus and, for lattice sums, two running-sum updates
                double* master = A.get<double>("pot.master" + std::to_string(l), d.mrows * RN);
                launch_master(LL, d.mrows, d.h, RN, nullptr, master, p.M);
                launch_window_sum(LL, master, d.mrows, RN, p.nnuc, s0d + l * p.nnuc, d.nsum, d.n, d.pot_rows,
                                  w.pot[l]);
            }
        }
    }
    c->join(2, c->aux[pi], c->stream);
    c->join(3, c->aux[fi], c->stream);  // nuclear part needs the profiles
    if (ms) {
        // FEM-applied profiles (T v) for every distinct direction, then the tables as
        // residue-class correlations <u_mu, (T v_nu)(. - d nbar)> on DMMA
        FemApplyJobs fj{};
        int nfj = 0;
        double *wm[3] = {}, *wsf[3] = {};
        for (int l = 0; l < 3; ++l) {
            if (src[l] != l) continue;
            const DirPlan& d = p.d[l];
            FemApplyJob& J = fj.j[nfj++];
            J.pwl = w.pwl[l];
            J.Gbar = d.Gbar;
            J.hbar = d.hbar;
            J.lo = w.pwl_lo[l];
            J.hi = w.pwl_hi[l];
            J.wm = wm[l] = A.get<double>("fem.wm" + std::to_string(l), m0 * (d.Gbar + 2));
            J.ws = wsf[l] = A.get<double>("fem.ws" + std::to_string(l), m0 * (d.Gbar + 2));
        }
        launch_fem_apply(LF, fj, nfj, static_cast<int>(m0));
        // the distinct directions' folds are independent: the second runs on its own branch
        // (c5: the two folds were the longest chain before the Khatri-Rao combine)
        const bool fem_fork = nfj >= 2 && !serial;
        const Launch LF2 = fem_fork ? c->LA(3) : LF;
        if (fem_fork) c->join(11, c->aux[fi], c->aux[3]);
        int nfold = 0;
        for (int l = 0; l < 3; ++l) {
            if (src[l] != l) {
                w.massT[l] = w.massT[src[l]];
                w.stiffT[l] = w.stiffT[src[l]];
                continue;
            }
            const Launch& LFd = nfold++ == 1 ? LF2 : LF;
            const DirPlan& d = p.d[l];
            w.massT[l] = A.get<double>("fem.mass" + std::to_string(l), d.width * mm);
            w.stiffT[l] = A.get<double>("fem.stiff" + std::to_string(l), d.width * mm);
            ResFold f;
            f.m0 = static_cast<int>(m0);
            f.n = d.nbar;
            f.G = d.Gbar;
            support_window(sd->hs, p, l, true, f.jw0, f.J);
            f.a = w.pwl[l];
            f.b[0] = wm[l];
            f.b[1] = wsf[l];
            f.nb = 2;
            f.bguard = 1;
            f.band = static_cast<int>(d.band);
            // <u_mu, T v_nu(. - d nbar)> = <T u_mu(. + d nbar), v_nu>: the d < 0 half is the
            // (mu, nu)-transposed mirror of d > 0 (T symmetric), so only d >= 0 is folded
            f.dlo = 0;
            f.dhi = f.band;
            f.dchunk = std::max(1, (f.band + 1 + 3) / 4);
            f.out[0] = A.get<double>("fem.pm" + std::to_string(l), d.nbar * (d.band + 1) * mm);
            f.out[1] = A.get<double>("fem.ps" + std::to_string(l), d.nbar * (d.band + 1) * mm);
            f.res[0] = w.massT[l];
            f.res[1] = w.stiffT[l];
            f.slab = f.J <= kResfoldDirectJ ? nullptr : A.get<double>("fem.slab" + std::to_string(l), resfold_slab_doubles(f));
            f.sup_lo = w.pwl_lo[l];  // b = T v: one point wider on each side
            f.sup_hi = w.pwl_hi[l];
            f.bwiden = 1;
            launch_resfold(LFd, f, true, true, "fem_fold");
        }
        if (fem_fork) c->join(12, c->aux[3], c->aux[fi]);
    }
    // nuclear contraction: choose the reassociation (k_nuclear2.cu header)
    KRArgs kr_fused;  // the combine deferred to the fill point (AS_EMAJOR)
    bool kr_pending = false;
    int nuc_mode = 0, ndir = -1;
    const double* npart = nullptr;  // periodic single-direction fold partials (summed in fill)
    Index npart_res = 0, npart_nd = 0;
    if (nuc) {
        std::vector<int> wrapped;
        for (int l = 0; l < 3; ++l)
            if (p.d[l].L > 1) wrapped.push_back(l);
        const bool dmma_ok = m0 <= 32 && !(flags & AS_GENERAL_NUC);
        if (dmma_ok && wrapped.size() == 1) nuc_mode = 1;
        else if (dmma_ok && p.periodic && wrapped.size() >= 2) nuc_mode = 2;
        if (nuc_mode != 0) {
            // trivial directions -> W[r][e] = w_r prod_l T_l[r][e]
            TrivJobs tj{};
            WSpec ws{};
            int njobs = 0;
            int job_of_src[3] = {-1, -1, -1};
            for (int l = 0; l < 3; ++l) {
                if (p.d[l].L > 1) continue;
                const int s = src[l];
                if (job_of_src[s] < 0) {
                    job_of_src[s] = njobs;
                    TrivJob& J = tj.j[njobs++];
                    J.pot = w.pot[s];
                    J.rows = p.d[s].pot_rows;
                    J.mrows = p.d[s].mrows;
                    J.h = p.d[s].h;
                    J.M = static_cast<int>(p.M);
                    J.RN = static_cast<int>(RN);
                    J.s0 = s0d + s * p.nnuc;
                    J.pwc = w.pwc[s];
                    J.G = p.d[s].G;
                    J.lo = w.pwc_lo[s];
                    J.hi = w.pwc_hi[s];
                }
                ws.job_of_dir[l] = job_of_src[s];
            }
            const int nsym = static_cast<int>(m0 * (m0 + 1) / 2);
            long long maxG = 1;
            for (int j = 0; j < njobs; ++j) maxG = std::max(maxG, tj.j[j].G);
            const int tiles = static_cast<int>(((Rtot + 63) / 64) * ((nsym + 63) / 64));
            // split-K: one wave of CTAs on the cp.async pipeline when each CTA still gets >= 8
            // stages (long grids, c4: 43 + 12 us at four waves, 35 + 5 us at one), else four
            // waves of short register-prefetched CTAs (a short K is latency-bound: c2)
            int splits = 1;
            bool triv_async = false;
            if (njobs) {
                const int s1 = splits_for(tiles * njobs, maxG, 1);
                triv_async = maxG / s1 >= 8 * 32;
                const int w = triv_async ? 1 : 4;
                splits = splits_for(tiles * njobs, maxG, w);
            }
            double* part = A.get<double>("nuc.tpart", std::max<size_t>(1, static_cast<size_t>(njobs) * splits * Rtot * nsym));
            double* W = A.get<double>("nuc.W", Rtot * mm);
            launch_triv_tables(L, tj, njobs, ws, static_cast<int>(m0), static_cast<int>(Rtot), w.potw, part, splits, W,
                               nullptr, triv_async);
            if (nuc_mode == 1) {
                ndir = wrapped[0];
                const DirPlan& d = p.d[ndir];
                double* V = nullptr;
                if (!p.periodic) {  // periodic: V is formed per residue inside the fold
                    V = A.get<double>("nuc.V", mm * d.pot_rows + (d.L + 260) * d.n);  // + the Hankel TMA view's slack
                    launch_vgemm(L, static_cast<int>(mm), static_cast<int>(Rtot), d.pot_rows, W, w.pot[ndir], V);
                }
                w.N = A.get<double>("nuc.N", d.L * d.width * mm);
                if (!p.periodic) {
                    const int nt = static_cast<int>(((d.L + 63) / 64) * ((d.width + 63) / 64) * mm);
                    const int rs = d.pot_rows == d.G ? hankel_res_splits(d) : 0;  // the resident kernel's quota slots
                    const int sp = rs > 0 ? rs : splits_for(nt, d.G);
                    double* hp = A.get<double>("nuc.hpart", static_cast<size_t>(sp) * mm * d.L * d.width);
                    launch_hankel(L, static_cast<int>(m0), d, w.pwc[ndir], w.pwc_lo[ndir], w.pwc_hi[ndir], V, hp, w.N,
                                  sp, d.pot_rows == d.G);
                } else {
                    ResFold f;
                    f.m0 = static_cast<int>(m0);
                    f.n = d.n;
                    f.G = d.G;
                    support_window(sd->hs, p, ndir, false, f.jw0, f.J);
                    f.a = f.b[0] = w.pwc[ndir];
                    f.nb = 1;
                    f.band = static_cast<int>(d.band);
                    f.dlo = 0;
                    f.dhi = f.band;
                    f.dchunk = std::max(1, (f.band + 1 + 3) / 4);
                    if (mm * Rtot <= 8192) {
                        // small W: every fold CTA forms its residue's V column itself
                        f.W = W;
                        f.P = w.pot[ndir];
                        f.Rtot = static_cast<int>(Rtot);
                        f.prow = d.pot_rows;
                    } else {
                        // large W (read by every CTA otherwise): V once, then the weighted fold
                        double* V = A.get<double>("nuc.V", mm * d.pot_rows);
                        launch_vdot(L, static_cast<int>(mm), static_cast<int>(Rtot), d.pot_rows, W, w.pot[ndir], V);
                        f.V = V;
                    }
                    f.out[0] = A.get<double>("nuc.fpart", d.n * (d.band + 1) * mm);
                    f.res[0] = w.N;
                    f.slab = f.J <= kResfoldDirectJ ? nullptr : A.get<double>("nuc.slab", resfold_slab_doubles(f));
                    f.sup_lo = w.pwc_lo[ndir];
                    f.sup_hi = w.pwc_hi[ndir];
                    if (f.n <= 32) {
                        // few residues: the fill sums them (no reduce launch)
                        launch_resfold(L, f, false, false, "nuc_fold");
                        npart = f.out[0];
                        npart_res = f.n;
                        npart_nd = f.dhi - f.dlo + 1;
                    } else {
                        launch_resfold(L, f, true, true, "nuc_fold");
                    }
                }
            } else {
                KRArgs kr;
                kr.m0 = static_cast<int>(m0);
                kr.Rtot = static_cast<int>(Rtot);
                kr.W = W;
                double* Tl[3] = {nullptr, nullptr, nullptr};
                // the per-direction chains (fold -> fold GEMM) are independent: the second
                // distinct direction runs on the potential side stream (idle by now)
                int nchain = 0, ndist = 0;
                for (int l = 0; l < 3; ++l) ndist += p.d[l].L > 1 && src[l] == l;
                const bool forked = ndist >= 2 && !serial;
                if (forked) c->join(9, c->stream, c->aux[pi]);  // fork before the first chain
                for (int l = 0; l < 3; ++l) {
                    kr.width[l] = static_cast<int>(p.d[l].width);
                    kr.band[l] = static_cast<int>(p.d[l].band);
                    if (p.d[l].L == 1) continue;
                    const int s = src[l];
                    if (!Tl[s]) {
                        const bool side = nchain++ == 1 && forked;
                        const Launch& LC = side ? LP : L;
                        const DirPlan& d = p.d[s];
                        double* Qf = A.get<double>("nuc.Qf" + std::to_string(s), (d.band + 1) * mm * d.n);
                        Tl[s] = A.get<double>("nuc.T" + std::to_string(s), (d.band + 1) * Rtot * mm);
                        ResFold f;
                        f.m0 = static_cast<int>(m0);
                        f.n = d.n;
                        f.G = d.G;
                        support_window(sd->hs, p, s, false, f.jw0, f.J);
                        f.a = f.b[0] = w.pwc[s];
                        f.nb = 1;
                        f.band = static_cast<int>(d.band);
                        f.dlo = 0;
                        f.dhi = f.band;
                        f.dchunk = std::max(1, (f.band + 1 + 3) / 4);
                        f.out[0] = Qf;  // [t][d][e]
                        f.slab = f.J <= kResfoldDirectJ ? nullptr : A.get<double>("nuc.slab" + std::to_string(s), resfold_slab_doubles(f));
                        f.sup_lo = w.pwc_lo[s];
                        f.sup_hi = w.pwc_hi[s];
                        launch_resfold(LC, f, false, false, "nuc_fold");
                        launch_fgemm(LC, static_cast<int>(m0), static_cast<int>(Rtot), d, w.pot[s], Qf, Tl[s]);
                    }
                    kr.T[l] = Tl[s];
                }
                if (forked) c->join(10, c->aux[pi], c->stream);
                if ((flags & AS_EMAJOR) && p.periodic && mode == 0 && !(flags & AS_NO_FILL)) {
                    kr_fused = kr;
                    kr_pending = true;
                } else {
                    w.N = A.get<double>("nuc.N", p.nblocks * mm);
                    kr.N = w.N;
                    launch_kr_combine(L, kr);
                }
            }
        } else {
            // general path: per-direction tables by direct contraction, combined in the fill
            for (int l = 0; l < 3; ++l) {
                const DirPlan& d = p.d[l];
                if (src[l] != l) {
                    w.T[l] = w.T[src[l]];
                    continue;
                }
                w.T[l] = A.get<double>("nuc.T" + std::to_string(l), d.npairs * Rtot * mm);
                if (d.mode == TM_FOLD) {
                    double* Qf = A.get<double>("nuc.Qf" + std::to_string(l), d.width * mm * d.n);
                    launch_nuc_fold(L, m0, Rtot, d, w.pwc[l], w.pwc_lo[l], w.pwc_hi[l], w.pot[l], Qf, w.T[l]);
                } else {
                    if (d.mode == TM_BOXDIR)  // tables of pairs with k+d outside the lattice stay unused
                        LT_CU(cudaMemsetAsync(w.T[l], 0, sizeof(double) * d.npairs * Rtot * mm, c->stream));
                    launch_nuc_direct(L, m0, Rtot, d, p.periodic, w.pwc[l], w.pwc_lo[l], w.pwc_hi[l], w.pot[l],
                                      w.T[l]);
                }
            }
        }
    }
    const bool split = (flags & AS_BOX_SPLIT) && !p.periodic && mode == 0 && !(flags & AS_NO_FILL);
    if (split) {
        // S = Mass on the FEM branch (only the mass tables), then the hook there
        FillArgs fs;
        fs.m0 = m0;
        fs.Rtot = Rtot;
        for (int l = 0; l < 3; ++l) {
            fs.L[l] = p.d[l].L;
            fs.band[l] = p.d[l].band;
            fs.width[l] = p.d[l].width;
            fs.massT[l] = w.massT[l];
            fs.stiffT[l] = w.stiffT[l];
        }
        fs.mode = 2;
        fs.periodic = false;
        fs.out0 = out.out1;
        LT_CU(cudaMemsetAsync(out.out1, 0, sizeof(double) * p.Nb * p.Nb, LF.st));
        launch_fill(LF, fs, p.Nb, p.cells * p.d[0].width * p.d[1].width * p.d[2].width);
        if (s_hook) (*s_hook)(LF);
    }
    c->join(4, c->aux[fi], c->stream);  // FEM tables (and the S branch) before the fill
    if (flags & AS_NO_FILL) {
        if (wout) *wout = w;
        return;
    }
    if (kr_pending) {
        // Khatri-Rao combine + fill in one launch, H and S entry-major
        for (int l = 0; l < 3; ++l) {
            kr_fused.massT[l] = w.massT[l];
            kr_fused.stiffT[l] = w.stiffT[l];
            kr_fused.L[l] = p.d[l].L;
        }
        kr_fused.kin = shard.kin;
        kr_fused.H = out.out0;
        kr_fused.S = out.out1;
        kr_fused.kidx = out.kidx;
        kr_fused.nblocks = p.nblocks;
        launch_kr_combine(L, kr_fused);
        if (wout) *wout = w;
        return;
    }
    // fused combine + placement
    FillArgs fa;
    fa.m0 = m0;
    fa.Rtot = Rtot;
    for (int l = 0; l < 3; ++l) {
        fa.L[l] = p.d[l].L;
        fa.band[l] = p.d[l].band;
        fa.width[l] = p.d[l].width;
        fa.massT[l] = w.massT[l];
        fa.stiffT[l] = w.stiffT[l];
        fa.T[l] = w.T[l];
    }
    fa.potw = w.potw;
    fa.N = w.N;
    fa.Npart = npart;
    fa.Nres = npart_res;
    fa.Nnd = npart_nd;
    fa.s2_dir = ndir;
    fa.nuc_mode = nuc_mode;
    fa.mode = mode;
    fa.kin = shard.kin;
    fa.periodic = p.periodic;
    fa.out0 = out.out0;
    fa.out1 = out.out1;
    fa.kidx = out.kidx;
    Index nblocks;
    if (p.periodic) {
        nblocks = p.nblocks;
    } else {
        nblocks = p.cells * p.d[0].width * p.d[1].width * p.d[2].width;
        LT_CU(cudaMemsetAsync(out.out0, 0, sizeof(double) * p.Nb * p.Nb, c->stream));
        if (mode == 0 && !split) LT_CU(cudaMemsetAsync(out.out1, 0, sizeof(double) * p.Nb * p.Nb, c->stream));
        if (split) fa.mode = 5;
    }
    launch_fill(L, fa, p.Nb, nblocks);
    if (wout) *wout = w;
}

static std::vector<std::array<Index, 3>> periodic_kidx(const Plan& p) {
    std::vector<std::array<Index, 3>> out;
    std::vector<Index> ax[3];
    for (int l = 0; l < 3; ++l) {
        const DirPlan& d = p.d[l];
        for (Index r = 0; r < d.width; ++r) {
            const Index dd = r <= d.band ? r : r - d.width;
            ax[l].push_back(((dd % d.L) + d.L) % d.L);
        }
    }
    for (Index a : ax[0])
        for (Index b : ax[1])
            for (Index cc : ax[2]) out.push_back({a, b, cc});
    return out;
}

// ---------------------------------------------------------------------------
// spectrum
// ---------------------------------------------------------------------------
// Dense block-diagonal form [K][mm] (complex) of a generating tensor given by the
// stored kidx (host) and its blocks (device, std::map order): see DftPrep above.

// host part of the block diagonalisation: compressed per-axis index sets and the
// slot map, uploaded (not capturable, so done before any graph capture)
static DftPrep prepare_dft(lt_ctx* c, const Index dims[3], Index m0, const std::vector<std::array<Index, 3>>& kidx,
                           const std::string& tag) {
    {
        auto it = c->dft_cache.find(tag);
        if (it != c->dft_cache.end()) {
            const lt_ctx::DftCache& e = it->second;
            if (e.gen == c->arena.generation() && e.m0 == m0 && e.dims[0] == dims[0] && e.dims[1] == dims[1] &&
                e.dims[2] == dims[2] && e.kidx == kidx)
                return e.P;  // the device tables of this tag still hold exactly these maps
        }
    }
    DftPrep P;
    P.m0 = m0;
    P.tag = tag;
    P.nblk = static_cast<Index>(kidx.size());
    std::vector<Index> comp[3];
    for (int l = 0; l < 3; ++l) {
        P.dims[l] = dims[l];
        std::set<Index> s;
        for (auto& k : kidx) s.insert(k[l]);
        if (s.empty()) s.insert(0);
        comp[l].assign(s.begin(), s.end());
        P.ext[l] = P.ncomp[l] = static_cast<Index>(comp[l].size());
        if (dims[l] == 1) {
            if (comp[l].size() != 1 || comp[l][0] != 0) fail(LT_EBOUNDS, "GeneratingBlockTensor: index out of range");
        } else {
            for (Index v : comp[l])
                if (v < 0 || v >= dims[l]) fail(LT_EBOUNDS, "GeneratingBlockTensor: index out of range");
        }
    }
    std::vector<int> slot2blk(static_cast<size_t>(P.ext[0] * P.ext[1] * P.ext[2]), -1);
    for (size_t b = 0; b < kidx.size(); ++b) {
        Index pos = 0;
        for (int l = 0; l < 3; ++l) {
            const Index ci = std::lower_bound(comp[l].begin(), comp[l].end(), kidx[b][l]) - comp[l].begin();
            pos = pos * P.ext[l] + ci;
        }
        slot2blk[pos] = static_cast<int>(b);
    }
    P.maxsz = P.ext[0] * P.ext[1] * P.ext[2];
    Index e2[3] = {P.ext[0], P.ext[1], P.ext[2]};
    for (int a = 0; a < 3; ++a) {
        if (dims[a] > 1) e2[a] = dims[a];
        P.maxsz = std::max(P.maxsz, e2[0] * e2[1] * e2[2]);
    }
    P.ident = true;
    for (size_t q = 0; q < slot2blk.size(); ++q) P.ident = P.ident && slot2blk[q] == static_cast<int>(q);
    ++c->prep_epoch;
    P.slot2blk = c->arena.get<int>("dft.slot" + tag, slot2blk.size());
    upload(c, P.slot2blk, slot2blk.data(), slot2blk.size() * sizeof(int));
    for (int a = 0; a < 3; ++a) {
        P.comp[a] = c->arena.get<int64_t>("dft.comp" + tag + std::to_string(a), comp[a].size());
        upload(c, P.comp[a], comp[a].data(), comp[a].size() * sizeof(int64_t));
    }
    lt_ctx::DftCache& e = c->dft_cache[tag];
    e.kidx = kidx;
    for (int l = 0; l < 3; ++l) e.dims[l] = dims[l];
    e.m0 = m0;
    e.gen = c->arena.generation();  // after the allocations above (a grown arena is a new generation)
    e.P = P;
    return P;
}

// the multi-axis transform runs as one fused launch (an entry's cube fits shared memory)
static bool dft_fused_ok(const DftPrep& P) {
    DftFusedArgs f;
    f.mm = P.m0 * P.m0;
    f.maxsz = P.maxsz;
    for (int l = 0; l < 3; ++l) {
        f.dims[l] = P.dims[l];
        f.ncomp[l] = P.ncomp[l];
        if (P.dims[l] > 1) f.axes[f.nax++] = l;
    }
    return f.nax >= 2 && dft_fused_smem(f) <= 200 * 1024;
}

// device part (kernels only: capturable). Transforms nops operators that share the
// stored kidx (blocks[op] on device, std::map order); out[op] receives [K][mm] complex.
// With want_emajor, the fused multi-axis launch writes [mm][K] instead (entry-major, for the
// one-thread-per-pencil kernel); returns whether it did.
static bool launch_dft(lt_ctx* c, const DftPrep& P, int nops, const double* const* blocks, double2** out,
                       bool want_emajor = false, bool gen_emajor = false) {
    const Launch L = c->L();
    const Index mm = P.m0 * P.m0;
    double2* buf[2][2];
    for (int op = 0; op < nops; ++op) {
        buf[op][0] = c->arena.get<double2>("dft.a" + P.tag + std::to_string(op), P.maxsz * mm);
        buf[op][1] = c->arena.get<double2>("dft.b" + P.tag + std::to_string(op), P.maxsz * mm);
    }
    {
        // two or more wrapped axes: one fused launch when an entry's cube fits shared memory
        DftFusedArgs f;
        f.mm = mm;
        f.maxsz = P.maxsz;
        f.slot2blk = P.slot2blk;
        f.ident = P.ident ? 1 : 0;
        for (int l = 0; l < 3; ++l) {
            f.dims[l] = P.dims[l];
            f.ext[l] = P.ext[l];
            f.ncomp[l] = P.ncomp[l];
            f.comp[l] = P.comp[l];
            if (P.dims[l] > 1) f.axes[f.nax++] = l;
        }
        if (f.nax >= 2 && dft_fused_smem(f) <= 200 * 1024) {
            for (int op = 0; op < nops; ++op) {
                f.gen[op] = blocks[op];
                f.out[op] = out[op] = buf[op][1];
            }
            f.emajor = want_emajor ? 1 : 0;
            f.gen_emajor = gen_emajor ? 1 : 0;
            f.nblocks = P.nblk;
            launch_dft_fused(L, f, nops);
            return want_emajor;
        }
    }
    if (gen_emajor) fail(LT_EGENERIC, "lattice DFT: entry-major generating blocks need the fused transform");
    DftAxisArgs a;
    a.mm = mm;
    for (int l = 0; l < 3; ++l) a.in[l] = P.ext[l];
    int nax = 0, cur = 0;
    for (int ax = 0; ax < 3; ++ax) {
        if (P.dims[ax] == 1) continue;
        a.axis = ax;
        for (int l = 0; l < 3; ++l) a.out[l] = a.in[l];
        a.out[ax] = P.dims[ax];
        a.ncomp = P.ncomp[ax];
        a.Lax = P.dims[ax];
        a.comp = P.comp[ax];
        for (int op = 0; op < nops; ++op) {
            a.gen[op] = nax == 0 ? blocks[op] : nullptr;
            a.in_buf[op] = nax == 0 ? nullptr : buf[op][cur];
            a.out_buf[op] = buf[op][cur ^ 1];
        }
        a.slot2blk = P.slot2blk;
        launch_dft_axis2(L, a, nops);
        cur ^= 1;
        ++nax;
        for (int l = 0; l < 3; ++l) a.in[l] = a.out[l];
    }
    if (nax == 0) {
        // K = 1 (all L_l = 1): a single generating block; real -> complex copy
        DftAxisArgs z = a;
        z.axis = 0;
        z.ncomp = 1;
        z.Lax = 1;
        z.comp = P.comp[0];
        for (int op = 0; op < nops; ++op) {
            z.gen[op] = blocks[op];
            z.out_buf[op] = buf[op][1];
        }
        z.slot2blk = P.slot2blk;
        launch_dft_axis2(L, z, nops);
        cur = 1;
    }
    for (int op = 0; op < nops; ++op) out[op] = buf[op][cur];
    return false;
}

static double2* block_diag_device(lt_ctx* c, const Index dims[3], Index m0,
                                  const std::vector<std::array<Index, 3>>& kidx, const double* blocks_dev,
                                  const std::string& tag) {
    const DftPrep P = prepare_dft(c, dims, m0, kidx, tag);
    double2* out = nullptr;
    launch_dft(c, P, 1, &blocks_dev, &out);
    return out;
}

// key = 4 k + code with k local to the launched pencil range; k0 = the range's first global
// k-point, so the message names the global lexicographic index like eigensolver.cpp:79-86
static void raise_fail_key(unsigned long long key, bool periodic, Index k0 = 0) {
    if (key == ~0ull) return;
    const Index k = k0 + static_cast<Index>(key / 4);
    const int code = static_cast<int>(key % 4);
    if (!periodic)
        fail(LT_EDEFINITE, "solve_box_dense: overlap matrix is not positive definite (near-linear-dependent basis?)");
    if (code == 1)
        fail(LT_EDEFINITE, "solve_periodic: non-Hermitian diagonal block at k-point " + std::to_string(k));
    fail(LT_EDEFINITE, "solve_periodic: overlap block at k-point " + std::to_string(k) + " is not positive definite");
}

__global__ void k_real_to_complex(Index n, const double* __restrict__ a, double2* __restrict__ out) {
    const Index i = static_cast<Index>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = make_double2(a[i], 0.0);
}

__global__ void k_complex_real(Index n, const double2* __restrict__ a, double* __restrict__ out) {
    const Index i = static_cast<Index>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = a[i].x;
}

__global__ void k_pad_copy(int n, long long lds, const double* __restrict__ src, long long ldd, double* __restrict__ dst) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<long long>(n) * n) return;
    const long long r = i % n, c = i / n;
    dst[c * ldd + r] = src[c * lds + r];
}

static void pad_copy(const Launch& L, int n, long long lds, const double* src, long long ldd, double* dst) {
    Stage st_(L, "pad_copy");
    k_pad_copy<<<static_cast<unsigned>((static_cast<long long>(n) * n + 255) / 256), 256, 0, L.st>>>(n, lds, src, ldd,
                                                                                                   dst);
    LT_CU(cudaGetLastError());
    L.tick();
}

// The box pencil's reduction to a standard problem on the device (k_dense2.cu), in two
// halves so the S side can run as soon as S exists: box_factor (S = L L^T, L^-1 row- and
// column-major) and box_transform (A = L^-1 H L^-T, exactly symmetric, left in H, n x n
// pitch n). TMA needs a row pitch that is a multiple of 16 bytes: odd n works on padded
// copies. Failures (S not positive definite) land in fail_dev; no host synchronisation
// (graph-capturable).
static DenseReduceBufs box_bufs(lt_ctx* c, Index n, long long* ld_out) {
    const long long ld = (n % 2 == 0) ? n : n + 1;
    DenseReduceBufs b;
    b.Li = c->arena.get<double>("box.Li", n * ld);
    b.Lic = c->arena.get<double>("box.Lic", n * ld);
    b.W = c->arena.get<double>("box.W", n * ld);
    b.T = c->arena.get<double>("box.T", n * ld);
    if (ld != n) {
        b.S = c->arena.get<double>("box.Sp", n * ld);
        b.H = c->arena.get<double>("box.Hp", n * ld);
    }
    *ld_out = ld;
    return b;
}

static void box_factor(lt_ctx* c, const Launch& L, Index n, double* S, unsigned long long* fail_dev) {
    long long ld = 0;
    DenseReduceBufs b = box_bufs(c, n, &ld);
    b.fail = fail_dev;
    if (ld == n) b.S = S;
    else pad_copy(L, static_cast<int>(n), n, S, ld, b.S);
    dense_factor(L, static_cast<int>(n), ld, b);
}

static void box_transform(lt_ctx* c, const Launch& L, Index n, double* H, unsigned long long* fail_dev) {
    long long ld = 0;
    DenseReduceBufs b = box_bufs(c, n, &ld);
    b.fail = fail_dev;
    if (ld == n) b.H = H;
    else pad_copy(L, static_cast<int>(n), n, H, ld, b.H);
    dense_transform(L, static_cast<int>(n), ld, b);
    if (ld != n) pad_copy(L, static_cast<int>(n), ld, b.H, n, H);
}

// eigenvalues of the reduced box pencil (A in H): the persistent tridiagonalisation and
// the Sturm multisection (k_dense.cu)
static void box_tridiag_eig(lt_ctx* c, const Launch& L, Index n, const double* A, double* eig_dev) {
    const int ni = static_cast<int>(n);
    double* d = c->arena.get<double>("box.td", n);
    double* e = c->arena.get<double>("box.te", n);
    double* tw = c->arena.get<double>("box.tw", 4 * n);
    unsigned* bar = c->arena.get<unsigned>("box.bar", 8 * 160);  // per-CTA flags, 32 B apart
    launch_sytrd(L, ni, A, d, e, tw, bar);
    launch_tridiag_eig(L, ni, d, e, eig_dev);
}

static void box_eig_tridiag(lt_ctx* c, Index n, double* H, double* S, double* eig_dev, unsigned long long* fail_dev) {
    const Launch L = c->L();
    box_factor(c, L, n, S, fail_dev);
    box_transform(c, L, n, H, fail_dev);
    box_tridiag_eig(c, L, n, H, eig_dev);
}

// Box pencil on device buffers H, S (n x n col-major; both may be overwritten).
// Eigenvalues -> eig_dev; with vec_dev, the S-orthonormal eigenvectors X = L^-T Z (n x n
// col-major, eigensolver.cpp:31-32). Returns the failure key through *fail (device) for
// the batched-pencil path.
static void box_eig_device(lt_ctx* c, Index n, double* H, double* S, double* eig_dev, unsigned long long* fail_dev,
                           double* vec_dev = nullptr, const PencilReadback& rb = PencilReadback{}) {
    const Launch L = c->L();
    if (n <= 32 && !vec_dev) {  // real pencil straight from H, S (no conversion launches)
        launch_pencil(L, 1, n, nullptr, nullptr, eig_dev, fail_dev, false, pencil_identity_source(H, S), nullptr, rb,
                      true);
        return;
    }
    if (n <= 32) {
        double2* hc = c->arena.get<double2>("box.hc", n * n);
        double2* sc = c->arena.get<double2>("box.sc", n * n);
        {
            Stage st_(L, "r2c");
            k_real_to_complex<<<static_cast<unsigned>((n * n + 255) / 256), 256, 0, c->stream>>>(n * n, H, hc);
            k_real_to_complex<<<static_cast<unsigned>((n * n + 255) / 256), 256, 0, c->stream>>>(n * n, S, sc);
            LT_CU(cudaGetLastError());
            L.tick(2);
        }
        double2* vc = vec_dev ? c->arena.get<double2>("box.vc", n * n) : nullptr;
        launch_pencil(L, 1, n, hc, sc, eig_dev, fail_dev, false, PencilDft{}, vc, rb, true);
        if (vec_dev) {  // real symmetric input: the Jacobi rotations stay real
            Stage st_(L, "c2r");
            k_complex_real<<<static_cast<unsigned>((n * n + 255) / 256), 256, 0, c->stream>>>(n * n, vc, vec_dev);
            LT_CU(cudaGetLastError());
            L.tick();
        }
        return;
    }
    if (!vec_dev && sytrd_ctas(static_cast<int>(n)) > 0) {
        box_eig_tridiag(c, n, H, S, eig_dev, fail_dev);
        return;
    }
    // eigenvectors (want_vectors) or N_b beyond the on-chip tridiagonalisation: the same device
    // reduction A = L^-1 H L^-T (k_dense2.cu), the standard symmetric eigenproblem of A by the
    // library (cusolverDnDsyevd), then the back-transform X = L^-T Z on DMMA (eigensolver.cpp:
    // 29-32: llt.matrixU().solve(Z)); X^T S X = I.
    box_factor(c, L, n, S, fail_dev);
    box_transform(c, L, n, H, fail_dev);
    unsigned long long fkey = ~0ull;
    LT_CU(cudaMemcpyAsync(&fkey, fail_dev, sizeof(fkey), cudaMemcpyDeviceToHost, c->stream));
    LT_CU(cudaStreamSynchronize(c->stream));
    if (fkey != ~0ull)
        fail(LT_EDEFINITE, "solve_box_dense: overlap matrix is not positive definite (near-linear-dependent basis?)");
    if (!c->solver) {
        if (cusolverDnCreate(&c->solver) != CUSOLVER_STATUS_SUCCESS) fail(LT_ECUDA, "cusolverDnCreate failed");
    }
    cusolverDnSetStream(c->solver, c->stream);
    const cusolverEigMode_t mode = vec_dev ? CUSOLVER_EIG_MODE_VECTOR : CUSOLVER_EIG_MODE_NOVECTOR;
    const int ni = static_cast<int>(n);
    int lwork = 0;
    if (cusolverDnDsyevd_bufferSize(c->solver, mode, CUBLAS_FILL_MODE_LOWER, ni, H, ni, eig_dev, &lwork) !=
        CUSOLVER_STATUS_SUCCESS)
        fail(LT_ECUDA, "cusolverDnDsyevd_bufferSize failed");
    double* work = c->arena.get<double>("box.work", static_cast<size_t>(lwork) + 1);
    int* info = c->arena.get<int>("box.info", 1);
    {
        Stage st_(L, "syevd");
        if (cusolverDnDsyevd(c->solver, mode, CUBLAS_FILL_MODE_LOWER, ni, H, ni, eig_dev, work, lwork, info) !=
            CUSOLVER_STATUS_SUCCESS)
            fail(LT_ECUDA, "cusolverDnDsyevd failed");
    }
    int hinfo = 0;
    LT_CU(cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    LT_CU(cudaStreamSynchronize(c->stream));
    if (hinfo != 0) fail(LT_EGENERIC, "solve_box_dense: eigensolver failed");
    if (!vec_dev) return;
    long long ld = 0;
    const DenseReduceBufs b = box_bufs(c, n, &ld);
    if (ld == n) {
        dense_back_transform(L, ni, ld, b.Lic, H, vec_dev, fail_dev);
    } else {  // odd n: TMA row pitches on padded copies
        pad_copy(L, ni, n, H, ld, b.W);
        dense_back_transform(L, ni, ld, b.Lic, b.W, b.T, fail_dev);
        pad_copy(L, ni, ld, b.T, n, vec_dev);
    }
}

// graph-cache key: everything the captured launches bake in (host-derived parameters of
// the system and plan, device pointers, arena generation)
static std::vector<int64_t> graph_key(const HostSys& h, const Plan& p, bool periodic, Index kb, Index ke,
                                      const void* eig, const void* sysmem, uint64_t gen) {
    std::vector<int64_t> k;
    auto put_d = [&](double v) {
        int64_t b;
        std::memcpy(&b, &v, sizeof(b));
        k.push_back(b);
    };
    k.push_back(periodic);
    k.push_back(kb);
    k.push_back(ke);
    k.push_back(reinterpret_cast<int64_t>(eig));
    k.push_back(reinterpret_cast<int64_t>(sysmem));
    k.push_back(static_cast<int64_t>(gen));
    k.push_back(p.L0);
    put_d(h.b);
    put_d(h.eps_ov);
    k.push_back(h.quad_M);
    for (int l = 0; l < 3; ++l) {
        k.push_back(h.L[l]);
        k.push_back(h.n[l]);
        k.push_back(h.nbar[l]);
    }
    for (double v : h.pos) put_d(v);
    for (double v : h.Z) put_d(v);
    for (double v : h.center) put_d(v);
    for (double v : h.alpha) put_d(v);
    for (int v : h.deg) k.push_back(v);
    return k;
}

// the part of a system an exponent / geometry scan leaves unchanged (lattice, grids, counts,
// polynomial degrees): systems of one shape are likely to share L0
static std::vector<int64_t> shape_key(const HostSys& h, bool periodic) {
    std::vector<int64_t> k;
    auto put_d = [&](double v) {
        int64_t b;
        std::memcpy(&b, &v, sizeof(b));
        k.push_back(b);
    };
    k.push_back(periodic);
    put_d(h.b);
    put_d(h.eps_ov);
    k.push_back(h.quad_M);
    for (int l = 0; l < 3; ++l) {
        k.push_back(h.L[l]);
        k.push_back(h.n[l]);
        k.push_back(h.nbar[l]);
    }
    k.push_back(static_cast<int64_t>(h.Z.size()));
    k.push_back(static_cast<int64_t>(h.alpha.size()));
    for (int v : h.deg) k.push_back(v);
    return k;
}

static void solve_core_dev_body(lt_ctx* c, const lt_sysdev* sd, bool periodic, double* eig_dev, Index k_begin,
                                Index k_end, int64_t* info, double* eig_host, bool allow_spec, const CoreOpts& opt);

// full path on device; eigenvalues -> eig_dev (device). An error raised while the solve ran on
// a PREDICTED L0 may be the prediction's (a too large L0 trips the alias guard of a valid
// system): the solve is repeated without the prediction, which then decides.
static void solve_core_dev(lt_ctx* c, const lt_sysdev* sd, bool periodic, double* eig_dev, Index k_begin,
                           Index k_end, int64_t* info, double* eig_host = nullptr, bool allow_spec = true,
                           const CoreOpts& opt = CoreOpts{}) {
    c->spec_active = false;
    try {
        solve_core_dev_body(c, sd, periodic, eig_dev, k_begin, k_end, info, eig_host, allow_spec, opt);
    } catch (const lt::Error&) {
        if (!c->spec_active) throw;
        c->spec_active = false;
        c->spec_L0 = -1;
        c->prep.valid = false;
        cudaStreamSynchronize(c->stream);
        solve_core_dev_body(c, sd, periodic, eig_dev, k_begin, k_end, info, eig_host, false, opt);
    }
}

static void solve_core_dev_body(lt_ctx* c, const lt_sysdev* sd, bool periodic, double* eig_dev, Index k_begin,
                                Index k_end, int64_t* info, double* eig_host, bool allow_spec, const CoreOpts& opt) {
    const int phase = opt.phase;
    if (phase != 0) allow_spec = false;
    c->host_mark(0);
    validate(sd->hs);
    c->phase_mark(0);
    c->timer.mark_ref(c->stream);
    // L0 speculation: L0 is a function of the system alone; when the previous call solved this
    // system — or another one of the same shape (an exponent or geometry scan) — its L0 is the
    // prediction: the post-L0 work is launched right behind the L0 check (no host round trip)
    // and the device-computed L0 is compared after the final sync (a miss redoes the solve).
    std::vector<int64_t> skey = shape_key(sd->hs, periodic);
    // no host sync inside the post-L0 work: periodic systems, and box pencils solved on the
    // device (the batched pencil, or the dense reduction + on-chip tridiagonalisation)
    const Index nb_box = sd->hs.m0() * sd->hs.cells();
    const bool spec_ok_path = periodic || nb_box <= 32 || sytrd_ctas(static_cast<int>(nb_box)) > 0;
    const bool spec = allow_spec && spec_ok_path && c->graphs && !c->timer.on && c->spec_L0 >= 0 &&
                      c->spec_L0 <= 14 && skey == c->spec_key;
    Index L0;
    L0Work l0w;
    c->spec_active = spec;
    if (spec) {
        // L0 runs inside the same graph as the rest (shifts 1 .. L0 + 2, exactly those the
        // rule needs to confirm the prediction); its state is read back with the results
        l0w = l0_setup(c, sd);
        L0 = c->spec_L0;
        c->phase_mark(1);  // no separate L0 phase: it is part of the single graph
    } else {
        L0 = compute_L0(c, sd);
    }
    // plan products (host integer planning + small table uploads), reused while unchanged
    std::vector<int64_t> pkey = graph_key(sd->hs, Plan{}, periodic, -2, -2, nullptr, sd->mem, 0);
    pkey.push_back(L0);
    CorePrep& cp = c->prep;
    if (!(cp.valid && cp.key == pkey && cp.epoch == c->prep_epoch && cp.gen == c->arena.generation())) {
        cp.valid = false;
        plan_after_L0(sd->hs, periodic, L0, cp.p, true);
        if (!periodic && cp.p.Nb > 4096)
            fail(LT_ECAP, "solve_box_dense: size " + std::to_string(cp.p.Nb) + " exceeds dense cap 4096");
        cp.s0d = upload_s0(c, cp.p);
        if (periodic) {
            const auto kidx = periodic_kidx(cp.p);
            const Index dims[3] = {cp.p.d[0].L, cp.p.d[1].L, cp.p.d[2].L};
            cp.dp = prepare_dft(c, dims, cp.p.m0, kidx, "HS");
        }
        cp.key = pkey;
    }
    const Plan& p = cp.p;
    const Index mm = p.m0 * p.m0;
    if (k_end < 0 || k_end > p.K) k_end = p.K;
    if (k_begin < 0) k_begin = 0;
    AsmOut out;
    // read-back block: L0 state (ints 0-3, written by the L0 finalize) and the pencil
    // failure key (ints 6-7), fetched with one copy at the end of the graph
    int* ret = c->arena.get<int>("l0.state", 8);
    auto* fk = reinterpret_cast<unsigned long long*>(ret + 6);
    const Index ocount = periodic ? p.nblocks * mm : p.Nb * p.Nb;
    if (phase == 1 || (phase == 2 && periodic)) {  // caller buffers (the DFT only reads them)
        out.out0 = opt.H;
        out.out1 = opt.S;
    } else {
        out.out0 = c->arena.get<double>("core.H", ocount);
        out.out1 = c->arena.get<double>("core.S", ocount);
    }
    if (periodic) out.kidx = c->arena.get<int64_t>("core.kidx", p.nblocks * 3);
    const bool small_box = !periodic && p.Nb <= 32;
    // box pencils on the device path (batched pencil kernel or the dense reduction +
    // persistent tridiagonalisation) need no host step: they run inside the graph
    const bool graph_box = !periodic && (small_box || sytrd_ctas(static_cast<int>(p.Nb)) > 0);
    const bool inline_readback = periodic || graph_box;  // no host step after the graph
    const size_t ebytes = sizeof(double) * (periodic ? p.K * p.m0 : p.Nb);
    void* epin = eig_host ? c->stage_alloc(ebytes) : nullptr;  // pinned: capturable copy target
    int* rpin = c->pinned_state();
    const int64_t* s0d = cp.s0d;
    const DftPrep& dp = cp.dp;
    // device work after L0 (with L0 in front under speculation): kernels and memsets only
    // eigenvalues straight into the pinned staging buffer (host API) and the result block
    // copied by the pencil kernel's last group: no copy nodes at the end of the graph
    double* eig_out = epin ? static_cast<double*>(epin) : eig_dev;
    const bool kernel_readback = phase != 1 && inline_readback && (small_box || (periodic && k_begin < k_end));
    PencilReadback rb;
    if (kernel_readback) rb = PencilReadback{ret, rpin, c->pencil_done};
    auto enqueue = [&]() {
        // k_l0_init resets the failure key: in front of this graph under speculation, else in
        // the L0 graph that just ran. Under speculation the L0 check runs as its own branch
        // forked after the assembly's root kernel (its result is only read back at the end)
        // and joins before the spectrum, whose failure key it resets and whose read-back
        // carries its state. Large box pencils factor S on the FEM branch (the S side of the
        // dense reduction overlaps the nuclear contraction) and write the failure key there:
        // then k_l0_init goes first, ahead of every branch, and only the checks fork.
        const bool box_split = graph_box && !small_box && phase == 0;
        const bool fork_l0 = spec && !c->timer.on && phase != 2;
        const bool par_l0 = spec && !c->timer.on;
        if (spec && !fork_l0) {
            if (par_l0) {
                c->join(6, c->stream, c->aux[2]);
                l0w.enqueue(c->LA(2), 1, static_cast<int>(L0) + 3, true);
            } else {
                l0w.enqueue(c->L(), 1, static_cast<int>(L0) + 3, true);
            }
        }
        const bool init_first = fork_l0 && box_split;
        if (init_first) l0w.init(c->L());
        const BranchHook l0_fork = [&](const Launch&) {
            c->join(6, c->stream, c->aux[2]);
            l0w.enqueue(c->LA(2), 1, static_cast<int>(L0) + 3, !init_first);
        };
        // generating blocks entry-major straight from the Khatri-Rao combine when the fused
        // lattice DFT consumes them (the solve's internal buffers only)
        const bool gen_emajor = periodic && phase == 0 && dft_fused_ok(dp) && p.m0 <= 32;
        const BranchHook s_hook = [&](const Launch& LF) { box_factor(c, LF, p.Nb, out.out1, fk); };
        if (phase != 2)
            run_assembly(c, sd, p, NEED_MS | NEED_NUC, 0, out, nullptr, s0d,
                         (box_split ? AS_BOX_SPLIT : 0u) | (gen_emajor ? AS_EMAJOR : 0u), opt.shard,
                         box_split ? &s_hook : nullptr, fork_l0 ? &l0_fork : nullptr);
        if (par_l0) c->join(7, c->aux[2], c->stream);
        if (phase == 2 && !periodic) {  // the box pencil factorises in place: work on copies
            LT_CU(cudaMemcpyAsync(out.out0, opt.H, sizeof(double) * ocount, cudaMemcpyDeviceToDevice, c->stream));
            LT_CU(cudaMemcpyAsync(out.out1, opt.S, sizeof(double) * ocount, cudaMemcpyDeviceToDevice, c->stream));
        }
        if (phase == 1) {
            LT_CU(cudaMemcpyAsync(rpin, ret, 8 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
            return;
        }
        if (periodic) {
            int wrapped = 0, ax = -1;
            for (int l = 0; l < 3; ++l)
                if (dp.dims[l] > 1) {
                    ++wrapped;
                    ax = l;
                }
            // single wrapped axis and a small transform (K nc m0^2 terms): the lattice DFT is
            // fused into the pencil load stage (one launch less); larger ones keep the
            // separate DFT kernel, whose parallelism beats per-pencil sums
            if (wrapped == 1 && dp.ncomp[ax] <= kPencilDftMax &&
                (k_end - k_begin) * dp.ncomp[ax] * mm <= (Index(1) << 20)) {
                PencilDft f;
                f.nc = static_cast<int>(dp.ncomp[ax]);
                f.L = dp.dims[ax];
                f.k0 = k_begin;
                f.comp = dp.comp[ax];
                f.blk = dp.slot2blk;
                f.GH = out.out0;
                f.GS = out.out1;
                if (k_begin < k_end)
                    launch_pencil(c->L(), k_end - k_begin, p.m0, nullptr, nullptr, eig_out + k_begin * p.m0, fk, true,
                                  f, nullptr, rb);
            } else {
                const double* blocks[2] = {out.out0, out.out1};
                double2* bd[2];
                const Index nk = k_end - k_begin;
                // the kernel choice depends on the whole lattice (not the shard): every k-point
                // shard then reproduces the full solve bitwise
                const bool lane = pencil_lane_supported(p.m0) &&
                                  dp.dims[0] * dp.dims[1] * dp.dims[2] >= kPencilLaneMin;
                const bool emajor = launch_dft(c, dp, 2, blocks, bd, lane, gen_emajor);
                double2* Hb = bd[0];
                double2* Sb = bd[1];
                if (lane && nk > 0) {
                    const Index K = dp.dims[0] * dp.dims[1] * dp.dims[2];
                    launch_pencil_lane(c->L(), nk, p.m0, Hb + k_begin * (emajor ? 1 : mm),
                                       Sb + k_begin * (emajor ? 1 : mm), emajor ? 1 : mm, emajor ? K : 1,
                                       eig_out + k_begin * p.m0, fk, rb);
                } else if (!lane && nk > 0) {
                    launch_pencil(c->L(), nk, p.m0, Hb + k_begin * mm, Sb + k_begin * mm,
                                  eig_out + k_begin * p.m0, fk, true, PencilDft{}, nullptr, rb);
                }
            }
        } else if (box_split) {
            box_transform(c, c->L(), p.Nb, out.out0, fk);
            box_tridiag_eig(c, c->L(), p.Nb, out.out0, eig_out);
        } else if (graph_box) {
            box_eig_device(c, p.Nb, out.out0, out.out1, eig_out, fk, nullptr, rb);
        }
        if (inline_readback && !kernel_readback)  // (an empty k-point shard launches no pencil)
            LT_CU(cudaMemcpyAsync(rpin, ret, 8 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        if (inline_readback && epin && eig_out != epin)
            LT_CU(cudaMemcpyAsync(epin, eig_dev, ebytes, cudaMemcpyDeviceToHost, c->stream));
    };
    c->phase_mark(2);
    c->host_mark(1);
    run_cached(
        c, spec ? c->fullgraph : (phase == 1 ? c->asmgraph : (phase == 2 ? c->specgraph : c->coregraph)),
        [&]() {
            auto k = graph_key(sd->hs, p, periodic, k_begin, k_end, eig_dev, sd->mem, c->arena.generation());
            k.push_back(spec ? 1 : 0);
            k.push_back(reinterpret_cast<int64_t>(epin));
            k.push_back(reinterpret_cast<int64_t>(rpin));
            k.push_back(phase);
            k.push_back(opt.shard.r0);
            k.push_back(opt.shard.r1);
            int64_t kb;
            std::memcpy(&kb, &opt.shard.kin, sizeof(kb));
            k.push_back(kb);
            k.push_back(reinterpret_cast<int64_t>(opt.H));
            k.push_back(reinterpret_cast<int64_t>(opt.S));
            return k;
        },
        enqueue);
    if (!inline_readback && phase != 1) {
        box_eig_device(c, p.Nb, out.out0, out.out1, eig_dev, fk);
        LT_CU(cudaMemcpyAsync(rpin, ret, 8 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        if (epin) LT_CU(cudaMemcpyAsync(epin, eig_dev, ebytes, cudaMemcpyDeviceToHost, c->stream));
    }
    c->phase_mark(3);
    // one synchronisation for the failure key, the L0 state and (host API) the eigenvalues
    if (eig_host && !epin) LT_CU(cudaMemcpyAsync(eig_host, eig_dev, ebytes, cudaMemcpyDeviceToHost, c->stream));
    c->host_mark(2);
    LT_CU(cudaStreamSynchronize(c->stream));
    c->host_mark(3);
    unsigned long long fkey;
    std::memcpy(&fkey, rpin + 6, sizeof(fkey));
    cp.epoch = c->prep_epoch;
    cp.gen = c->arena.generation();
    cp.valid = true;
    if (spec) {
        const int* st = c->pinned_state();
        if (!(st[3] && st[0] == L0)) {  // misprediction: discard and redo without speculation
            c->spec_L0 = -1;
            cp.valid = false;
            solve_core_dev(c, sd, periodic, eig_dev, k_begin, k_end, info, eig_host, false);
            return;
        }
    }
    c->spec_key = std::move(skey);
    c->spec_L0 = L0;
    if (eig_host && epin && fkey == ~0ull) std::memcpy(eig_host, epin, ebytes);
    c->phase_collect();
    c->timer.collect();
    if (info) {
        info[0] = p.L0;
        for (int l = 0; l < 3; ++l) info[1 + l] = p.d[l].band;
        info[4] = p.Rtot;
        info[5] = p.Nb;
        info[6] = p.K;
        info[7] = fkey == ~0ull ? -1 : static_cast<int64_t>(fkey + (periodic ? 4ull * static_cast<unsigned long long>(k_begin) : 0ull));
    }
    c->host_mark(4);
    c->host_collect();
    raise_fail_key(fkey, periodic, periodic ? k_begin : 0);
}

static lt_operator* new_op(const Plan& p, int which, Index coefficient_rank) {
    auto* op = new lt_operator;
    op->which = which;
    op->periodic = p.periodic;
    op->m0 = p.m0;
    for (int l = 0; l < 3; ++l) {
        op->L[l] = p.d[l].L;
        op->band[l] = p.d[l].band;
    }
    op->L0 = p.L0;
    op->coefficient_rank = coefficient_rank;
    op->Nb = p.Nb;
    if (p.periodic) {
        op->kidx = periodic_kidx(p);
        op->count = p.nblocks * p.m0 * p.m0;
    } else {
        op->count = p.Nb * p.Nb;
    }
    if (cudaMalloc(&op->data, sizeof(double) * std::max<size_t>(op->count, 1)) != cudaSuccess) {
        delete op;
        fail(LT_ECUDA, "cudaMalloc failed for operator");
    }
    return op;
}

// ordered union of two kidx lists with index maps (eigensolver.cpp:60-64 semantics)
static void union_maps(const lt_operator* a, const lt_operator* b, std::vector<std::array<Index, 3>>& keys,
                       std::vector<int64_t>& ia, std::vector<int64_t>& ib) {
    std::map<std::array<Index, 3>, std::pair<int64_t, int64_t>> u;
    for (size_t i = 0; i < a->kidx.size(); ++i) u[a->kidx[i]].first = static_cast<int64_t>(i) + 1;
    for (size_t i = 0; i < b->kidx.size(); ++i) u[b->kidx[i]].second = static_cast<int64_t>(i) + 1;
    for (auto& kv : u) {
        keys.push_back(kv.first);
        ia.push_back(kv.second.first - 1);
        ib.push_back(kv.second.second - 1);
    }
}

}  // namespace lt

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* lt_last_error(void) { return lt::g_err.c_str(); }

// (not in the public header) the multi-device layer (multi.cpp) reports through lt_last_error
void lt_internal_set_error(const char* msg) { lt::g_err = msg ? msg : ""; }


// ---------------------------------------------------------------------------
// separable metadata and the factorized Fourier path (k_sep.cu)
// ---------------------------------------------------------------------------
// metadata of one assembly from its per-direction tables (galerkin.cpp:394-423)
static std::unique_ptr<SepMeta> build_sep(lt_ctx* c, const Plan& p, int kind, const Work& w) {
    auto m = std::make_unique<SepMeta>();
    m->m0 = p.m0;
    m->terms = kind == LT_MASS ? 1 : (kind == LT_LAPLACE ? 3 : p.Rtot);
    SepBuild b;
    b.kind = kind;
    b.mm = p.m0 * p.m0;
    b.R = p.Rtot;
    for (int l = 0; l < 3; ++l) {
        const DirPlan& d = p.d[l];
        m->L[l] = d.L;
        m->S = std::max(m->S, d.width);
        for (Index sl = 0; sl < d.width; ++sl) {
            const Index dd = sl - d.band;
            m->kid[l].push_back(((dd % d.L) + d.L) % d.L);
        }
        b.nslot[l] = d.width;
        b.mass[l] = w.massT[l];
        b.stiff[l] = w.stiffT[l];
        b.T[l] = w.T[l];
    }
    b.S = m->S;
    b.potw = w.potw;
    LT_CU(cudaMalloc(&m->vals, sizeof(double) * std::max<size_t>(1, m->count())));
    LT_CU(cudaMemsetAsync(m->vals, 0, sizeof(double) * m->count(), c->stream));
    b.out = m->vals;
    launch_sep_from_tables(c->L(), b, m->terms);
    return m;
}

// scaled concatenation a (level 0 times wa) ++ b (level 0 times wb), slot sets united
// (combine, eigensolver.cpp:57-64)
static std::unique_ptr<SepMeta> sep_combine(lt_ctx* c, const SepMeta& a, double wa, const SepMeta& b, double wb) {
    auto m = std::make_unique<SepMeta>();
    m->m0 = a.m0;
    m->terms = a.terms + b.terms;
    std::vector<Index> mapa[3], mapb[3];
    for (int l = 0; l < 3; ++l) {
        m->L[l] = a.L[l];
        m->kid[l] = a.kid[l];
        for (size_t q = 0; q < a.kid[l].size(); ++q) mapa[l].push_back(static_cast<Index>(q));
        for (Index k : b.kid[l]) {
            auto it = std::find(m->kid[l].begin(), m->kid[l].end(), k);
            if (it == m->kid[l].end()) {
                mapb[l].push_back(static_cast<Index>(m->kid[l].size()));
                m->kid[l].push_back(k);
            } else {
                mapb[l].push_back(static_cast<Index>(it - m->kid[l].begin()));
            }
        }
        m->S = std::max<Index>(m->S, static_cast<Index>(m->kid[l].size()));
    }
    LT_CU(cudaMalloc(&m->vals, sizeof(double) * std::max<size_t>(1, m->count())));
    LT_CU(cudaMemsetAsync(m->vals, 0, sizeof(double) * m->count(), c->stream));
    const Index mm = a.m0 * a.m0;
    for (int side = 0; side < 2; ++side) {
        const SepMeta& src = side ? b : a;
        SepCopy cp;
        cp.mm = mm;
        cp.Ssrc = src.S;
        cp.Sdst = m->S;
        cp.t0 = side ? a.terms : 0;
        cp.w = side ? wb : wa;
        cp.src = src.vals;
        cp.dst = m->vals;
        for (int l = 0; l < 3; ++l) {
            const auto& mp = side ? mapb[l] : mapa[l];
            Index* d = c->arena.get<Index>("sep.map" + std::to_string(side) + std::to_string(l), mp.size() + 1);
            upload(c, d, mp.data(), mp.size() * sizeof(Index));
            cp.map[l] = d;
            cp.nslot[l] = static_cast<Index>(mp.size());
        }
        if (src.terms > 0) launch_sep_scale_copy(c->L(), cp, src.terms);
    }
    return m;
}

// metadata given as full level sequences [t][l][L_l][m0*m0] (reference SeparableTerm)
static std::unique_ptr<SepMeta> sep_from_full(lt_ctx* c, Index m0, const Index L[3], Index terms, const double* full) {
    auto m = std::make_unique<SepMeta>();
    m->m0 = m0;
    m->terms = terms;
    const Index mm = m0 * m0;
    for (int l = 0; l < 3; ++l) {
        m->L[l] = L[l];
        for (Index k = 0; k < L[l]; ++k) m->kid[l].push_back(k);
        m->S = std::max(m->S, L[l]);
    }
    std::vector<double> host(m->count(), 0.0);
    const Index per_term = (L[0] + L[1] + L[2]) * mm;
    for (Index t = 0; t < terms; ++t) {
        Index off = t * per_term;
        for (int l = 0; l < 3; ++l)
            for (Index k = 0; k < L[l]; ++k, off += mm)
                std::memcpy(&host[static_cast<size_t>(((t * 3 + l) * m->S + k) * mm)], full + off, sizeof(double) * mm);
    }
    LT_CU(cudaMalloc(&m->vals, sizeof(double) * std::max<size_t>(1, m->count())));
    LT_CU(cudaMemcpy(m->vals, host.data(), sizeof(double) * host.size(), cudaMemcpyHostToDevice));
    return m;
}

// max over every lattice point of |gen_k - expanded_k| (separable_residual)
static double sep_residual(lt_ctx* c, const SepMeta& m, const std::vector<std::array<Index, 3>>& kidx,
                           const double* gen_dev, const std::string& tag) {
    SepResid r;
    r.mm = m.m0 * m.m0;
    r.terms = m.terms;
    r.S = m.S;
    for (int l = 0; l < 3; ++l) {
        r.L[l] = m.L[l];
        std::vector<int> so(static_cast<size_t>(m.L[l]), -1);
        for (size_t q = 0; q < m.kid[l].size(); ++q) so[static_cast<size_t>(m.kid[l][q])] = static_cast<int>(q);
        int* d = c->arena.get<int>("sep.slot" + tag + std::to_string(l), so.size());
        upload(c, d, so.data(), so.size() * sizeof(int));
        r.slot_of[l] = d;
    }
    const Index K = m.L[0] * m.L[1] * m.L[2];
    std::vector<int> go(static_cast<size_t>(K), -1);
    for (size_t b = 0; b < kidx.size(); ++b)
        go[static_cast<size_t>((kidx[b][0] * m.L[1] + kidx[b][1]) * m.L[2] + kidx[b][2])] = static_cast<int>(b);
    int* gd = c->arena.get<int>("sep.gen" + tag, go.size());
    upload(c, gd, go.data(), go.size() * sizeof(int));
    r.gen_of = gd;
    r.vals = m.vals;
    r.gen = gen_dev;
    r.out = c->arena.get<unsigned long long>("sep.resid" + tag, 1);
    LT_CU(cudaMemsetAsync(r.out, 0, sizeof(unsigned long long), c->stream));
    launch_sep_residual(c->L(), r);
    unsigned long long bits = 0;
    LT_CU(cudaMemcpyAsync(&bits, r.out, sizeof(bits), cudaMemcpyDeviceToHost, c->stream));
    LT_CU(cudaStreamSynchronize(c->stream));
    double v;
    std::memcpy(&v, &bits, sizeof(v));
    return v;
}

// k-point blocks [K][m0*m0] (complex) by per-level 1D DFTs and per-k Hadamard sums
static double2* sep_fourier(lt_ctx* c, const SepMeta& m, const std::string& tag) {
    const Index mm = m.m0 * m.m0;
    const Index Lmax = std::max(m.L[0], std::max(m.L[1], m.L[2]));
    SepDft d;
    d.mm = mm;
    d.S = m.S;
    d.Lmax = Lmax;
    d.vals = m.vals;
    for (int l = 0; l < 3; ++l) {
        d.L[l] = m.L[l];
        d.nslot[l] = static_cast<Index>(m.kid[l].size());
        Index* k = c->arena.get<Index>("sep.kid" + tag + std::to_string(l), m.kid[l].size() + 1);
        upload(c, k, m.kid[l].data(), m.kid[l].size() * sizeof(Index));
        d.kid[l] = k;
    }
    d.out = c->arena.get<double2>("sep.X" + tag, static_cast<size_t>(m.terms * 3 * Lmax * mm));
    launch_sep_dft(c->L(), d, m.terms);
    SepBlocks b;
    b.mm = mm;
    b.terms = m.terms;
    b.Lmax = Lmax;
    for (int l = 0; l < 3; ++l) b.L[l] = m.L[l];
    b.X = d.out;
    b.out = c->arena.get<double2>("sep.F" + tag, static_cast<size_t>(m.L[0] * m.L[1] * m.L[2] * mm));
    launch_sep_blocks(c->L(), b);
    return b.out;
}

// batched pencils on device blocks (solve_blocks, eigensolver.cpp:95-121): eigenvalues and,
// when vec != null, the per-k eigenvector blocks (complex, column-major) to the host
static void pencils_to_host(lt_ctx* c, Index K, Index m0, const double2* Hb, const double2* Sb, double* eig,
                            double* vec, bool periodic_checks = true) {
    double* e = c->arena.get<double>("solve.eig", K * m0);
    double2* v = vec ? c->arena.get<double2>("solve.vec", K * m0 * m0) : nullptr;
    unsigned long long* fk = c->arena.get<unsigned long long>("solve.fail", 1);
    LT_CU(cudaMemsetAsync(fk, 0xff, sizeof(unsigned long long), c->stream));
    launch_pencil(c->L(), K, m0, Hb, Sb, e, fk, periodic_checks, PencilDft{}, v);
    unsigned long long key = ~0ull;
    LT_CU(cudaMemcpyAsync(&key, fk, sizeof(key), cudaMemcpyDeviceToHost, c->stream));
    LT_CU(cudaMemcpyAsync(eig, e, sizeof(double) * K * m0, cudaMemcpyDeviceToHost, c->stream));
    if (vec) LT_CU(cudaMemcpyAsync(vec, v, sizeof(double2) * K * m0 * m0, cudaMemcpyDeviceToHost, c->stream));
    LT_CU(cudaStreamSynchronize(c->stream));
    raise_fail_key(key, periodic_checks);
}

// eigenvalues (and vectors) of the factorized pencils (solve_blocks with the factorized blocks)
static void sep_solve(lt_ctx* c, const SepMeta& H, const SepMeta& S, double* eig, double* vec = nullptr) {
    const Index K = H.L[0] * H.L[1] * H.L[2];
    double2* Hb = sep_fourier(c, H, "H");
    double2* Sb = sep_fourier(c, S, "S");
    pencils_to_host(c, K, H.m0, Hb, Sb, eig, vec);
}

static void sep_check_resid(double resid, double tol) {
    if (resid > tol)
        fail(LT_ESTRUCT, "solve_periodic_factorized: factorization residual " + std::to_string(resid) +
                             " exceeds tolerance");
}

lt_status lt_create(int device, lt_ctx** out) {
    return guarded([&] {
        auto c = std::make_unique<lt_ctx>();
        c->device = device;
        LT_CU(cudaSetDevice(device));
        // priorities: the main stream carries the critical path (potential -> nuclear chain ->
        // fill -> pencils); side branch 0 (profiles -> FEM folds) has slack and, its folds
        // filling every SM's shared memory, must not hold SMs the main stream waits for
        int prio_lo = 0, prio_hi = 0;
        LT_CU(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
        LT_CU(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio_hi));
        LT_CU(cudaStreamCreateWithPriority(&c->aux[0], cudaStreamNonBlocking, prio_hi));
        LT_CU(cudaStreamCreateWithPriority(&c->aux[1], cudaStreamNonBlocking, prio_hi));
        LT_CU(cudaStreamCreateWithPriority(&c->aux[2], cudaStreamNonBlocking, prio_hi));
        LT_CU(cudaStreamCreateWithPriority(&c->aux[3], cudaStreamNonBlocking, prio_hi));
        for (auto& e : c->ev) LT_CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        LT_CU(cudaMalloc(&c->pencil_done, sizeof(unsigned)));
        LT_CU(cudaMemset(c->pencil_done, 0, sizeof(unsigned)));
        for (auto& e : c->pev) LT_CU(cudaEventCreate(&e));
        *out = c.release();
    });
}

void lt_destroy(lt_ctx* c) {
    if (!c) return;
    if (c->host_timing && c->host_n)
        std::fprintf(stderr,
                     "host timing over %lld solves (us): prep %.2f launch %.2f (key %.2f, cudaGraphLaunch %.2f) "
                     "wait %.2f finish %.2f; run_cached replay %lld capture %lld eager %lld\n",
                     static_cast<long long>(c->host_n), c->host_acc[0] / c->host_n, c->host_acc[1] / c->host_n,
                     c->key_us / c->host_n, c->graph_launch_us / c->host_n, c->host_acc[2] / c->host_n,
                     c->host_acc[3] / c->host_n, static_cast<long long>(c->n_replay),
                     static_cast<long long>(c->n_capture), static_cast<long long>(c->n_eager));
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->solver) cusolverDnDestroy(c->solver);
    if (c->blas) cublasDestroy(c->blas);
    if (c->pencil_done) cudaFree(c->pencil_done);
    if (c->pinned) cudaFreeHost(c->pinned);
    for (auto& a : c->aux)
        if (a) {
            cudaStreamSynchronize(a);
            cudaStreamDestroy(a);
        }
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : c->pev)
        if (e) cudaEventDestroy(e);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

void* lt_stream(lt_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

lt_status lt_stream_wait(lt_ctx* c, void* stream) {
    return guarded([&] {
        LT_CU(cudaSetDevice(c->device));
        c->join(8, static_cast<cudaStream_t>(stream), c->stream);
    });
}

lt_status lt_stream_join(lt_ctx* c, void* stream) {
    return guarded([&] {
        LT_CU(cudaSetDevice(c->device));
        c->join(8, c->stream, static_cast<cudaStream_t>(stream));
    });
}
int64_t lt_launch_count(lt_ctx* c) { return c ? c->launches : 0; }

lt_status lt_set_diagnostics(lt_ctx* c, int flags) {
    return guarded([&] {
        LT_CU(cudaStreamSynchronize(c->stream));
        c->phase_timing = (flags & LT_DIAG_PHASE_TIMING) != 0;
        c->host_timing = (flags & LT_DIAG_HOST_TIMING) != 0;
    });
}

lt_status lt_set_stage_timing(lt_ctx* c, int on) {
    return guarded([&] {
        LT_CU(cudaStreamSynchronize(c->stream));
        c->timer.reset();
        c->timer.on = on != 0;
    });
}

int64_t lt_stage_count(lt_ctx* c) {
    cudaStreamSynchronize(c->stream);
    c->timer.collect();
    return static_cast<int64_t>(c->timer.totals.size());
}

lt_status lt_stage_get(lt_ctx* c, int64_t idx, char* name, int64_t cap, double* ms, int64_t* launches) {
    return guarded([&] {
        if (idx < 0 || idx >= static_cast<int64_t>(c->timer.totals.size())) fail(LT_EBOUNDS, "stage index");
        auto it = c->timer.totals.begin();
        std::advance(it, idx);
        std::snprintf(name, static_cast<size_t>(cap), "%s", it->first.c_str());
        *ms = it->second.first;
        *launches = it->second.second;
    });
}

int64_t lt_stage_timeline_count(lt_ctx* c) {
    cudaStreamSynchronize(c->stream);
    c->timer.collect();
    return static_cast<int64_t>(c->timer.timeline.size());
}

lt_status lt_stage_timeline_get(lt_ctx* c, int64_t idx, char* name, int64_t cap, int* stream, double* t0,
                                double* t1) {
    return guarded([&] {
        if (idx < 0 || idx >= static_cast<int64_t>(c->timer.timeline.size())) fail(LT_EBOUNDS, "timeline index");
        const auto& sp = c->timer.timeline[static_cast<size_t>(idx)];
        std::snprintf(name, static_cast<size_t>(cap), "%s", sp.name.c_str());
        *stream = sp.stream == c->stream ? 0 : (sp.stream == c->aux[0] ? 1 : (sp.stream == c->aux[1] ? 2 : 3));
        *t0 = sp.t0;
        *t1 = sp.t1;
    });
}

lt_status lt_sys_upload(lt_ctx* c, const lt_system* s, lt_sysdev** out) {
    return guarded([&] {
        LT_CU(cudaSetDevice(c->device));
        *out = make_sysdev(s);
    });
}

void lt_sys_free(lt_sysdev* s) {
    if (!s) return;
    if (s->mem) cudaFree(s->mem);
    delete s;
}

lt_status lt_solve_core_dev(lt_ctx* c, const lt_sysdev* s, int periodic, double* eig_dev, int64_t k_begin,
                            int64_t k_end, int64_t* info) {
    return guarded([&] {
        LT_CU(cudaSetDevice(c->device));
        StageScope ss(c, 1 << 20);
        solve_core_dev(c, s, periodic != 0, eig_dev, k_begin, k_end, info);
    });
}

lt_status lt_solve_core_dev_on(lt_ctx* c, const lt_sysdev* s, int periodic, double* eig_dev, int64_t k_begin,
                               int64_t k_end, int64_t* info, void* stream) {
    return guarded([&] {
        LT_CU(cudaSetDevice(c->device));
        const cudaStream_t ext = static_cast<cudaStream_t>(stream);
        c->join(8, ext, c->stream);
        StageScope ss(c, 1 << 20);
        solve_core_dev(c, s, periodic != 0, eig_dev, k_begin, k_end, info);
        c->join(8, c->stream, ext);
    });
}

lt_status lt_core_layout(lt_ctx* c, const lt_sysdev* s, int periodic, int64_t* info, int64_t* kidx) {
    return guarded([&] {
        LT_CU(cudaSetDevice(c->device));
        validate(s->hs);
        const Index L0 = compute_L0(c, s);
        Plan p;
        plan_after_L0(s->hs, periodic != 0, L0, p, true);
        if (!periodic && p.Nb > 4096)
            fail(LT_ECAP, "solve_box_dense: size " + std::to_string(p.Nb) + " exceeds dense cap 4096");
        const Index mm = p.m0 * p.m0;
        info[0] = p.L0;
        info[1] = periodic ? p.nblocks : 0;
        info[2] = p.Nb;
        info[3] = p.K;
        info[4] = p.m0;
        info[5] = p.Rtot;
        info[6] = periodic ? p.nblocks * mm : p.Nb * p.Nb;
        info[7] = periodic ? p.m0 : p.Nb;  // eigenvalues per k-point
        if (kidx && periodic) {
            const auto k = periodic_kidx(p);
            for (size_t b = 0; b < k.size(); ++b)
                for (int l = 0; l < 3; ++l) kidx[3 * b + l] = k[b][static_cast<size_t>(l)];
        }
    });
}

lt_status lt_assemble_core_dev(lt_ctx* c, const lt_sysdev* s, int periodic, int64_t r_begin, int64_t r_end,
                               int with_kinetic, double* H_dev, double* S_dev) {
    return guarded([&] {
        LT_CU(cudaSetDevice(c->device));
        if (!H_dev || !S_dev) fail(LT_EDIM, "assemble_core_dev: H and S device buffers are required");
        StageScope ss(c, 1 << 20);
        CoreOpts o;
        o.phase = 1;
        o.shard.r0 = std::max<int64_t>(0, r_begin);
        o.shard.r1 = r_end;
        o.shard.kin = with_kinetic ? 0.5 : 0.0;
        o.H = H_dev;
        o.S = S_dev;
        solve_core_dev(c, s, periodic != 0, nullptr, 0, 0, nullptr, nullptr, false, o);
    });
}

lt_status lt_spectrum_dev(lt_ctx* c, const lt_sysdev* s, int periodic, const double* H_dev, const double* S_dev,
                          double* eig_dev, int64_t k_begin, int64_t k_end) {
    return guarded([&] {
        LT_CU(cudaSetDevice(c->device));
        if (!H_dev || !S_dev || !eig_dev) fail(LT_EDIM, "spectrum_dev: H, S and eigenvalue buffers are required");
        StageScope ss(c, 1 << 20);
        CoreOpts o;
        o.phase = 2;
        o.H = const_cast<double*>(H_dev);  // read only (box: copied before the in-place factorisation)
        o.S = const_cast<double*>(S_dev);
        solve_core_dev(c, s, periodic != 0, eig_dev, k_begin, k_end, nullptr, nullptr, false, o);
    });
}

lt_status lt_solve_core(lt_ctx* c, const lt_system* s, int periodic, double* eig_host, int64_t* info) {
    return guarded([&] {
        LT_CU(cudaSetDevice(c->device));
        // the system is copied host -> device on every call, into a context-owned buffer
        const HostSys hs = host_sys_from(s);
        const Index count = hs.m0() * hs.cells();
        StageScope ss(c, (1 << 20) + 2 * sizeof(double) * static_cast<size_t>(count));
        void* dst = c->arena.get<char>("sys.mem", sysdev_bytes(hs));
        std::unique_ptr<lt_sysdev> sd(make_sysdev(s, dst, c));
        double* eig = c->arena.get<double>("solve.eig", count);
        solve_core_dev(c, sd.get(), periodic != 0, eig, 0, -1, info, eig_host);
    });
}

lt_status lt_assemble(lt_ctx* c, const lt_system* s, int periodic, lt_kind kind, lt_operator** out) {
    return guarded([&] {
        LT_CU(cudaSetDevice(c->device));
        std::unique_ptr<lt_sysdev, void (*)(lt_sysdev*)> sd(make_sysdev(s), lt_sys_free);
        validate(sd->hs);
        const Index L0 = compute_L0(c, sd.get());
        Plan p;
        const bool nuc = kind == LT_NUCLEAR;
        plan_after_L0(sd->hs, periodic != 0, L0, p, nuc);
        const Index crank = kind == LT_MASS ? 1 : kind == LT_LAPLACE ? 3 : p.Rtot;
        std::unique_ptr<lt_operator> op(new_op(p, static_cast<int>(kind), crank));
        AsmOut o;
        o.out0 = op->data;
        o.kidx = p.periodic ? c->arena.get<int64_t>("op.kidx", p.nblocks * 3) : nullptr;
        const int mode = kind == LT_LAPLACE ? 1 : kind == LT_MASS ? 2 : 3;
        // periodic: the per-direction tables are kept (nuclear in the reference's nucT form)
        // and become the operator's separable metadata
        Work w{};
        run_assembly(c, sd.get(), p, nuc ? NEED_NUC : NEED_MS, mode, o, &w, nullptr,
                     p.periodic && nuc ? AS_GENERAL_NUC : 0u);
        if (p.periodic) op->sep = build_sep(c, p, static_cast<int>(kind), w);
        LT_CU(cudaStreamSynchronize(c->stream));
        *out = op.release();
    });
}

lt_status lt_assemble_core(lt_ctx* c, const lt_system* s, int periodic, lt_operator** H, lt_operator** S) {
    return guarded([&] {
        LT_CU(cudaSetDevice(c->device));
        std::unique_ptr<lt_sysdev, void (*)(lt_sysdev*)> sd(make_sysdev(s), lt_sys_free);
        validate(sd->hs);
        const Index L0 = compute_L0(c, sd.get());
        Plan p;
        plan_after_L0(sd->hs, periodic != 0, L0, p, true);
        std::unique_ptr<lt_operator> h(new_op(p, 0, 3 + p.Rtot));
        std::unique_ptr<lt_operator> sop(new_op(p, 1, 1));
        AsmOut o;
        o.out0 = h->data;
        o.out1 = sop->data;
        o.kidx = p.periodic ? c->arena.get<int64_t>("op.kidx", p.nblocks * 3) : nullptr;
        Work w{};
        run_assembly(c, sd.get(), p, NEED_MS | NEED_NUC, 0, o, &w);
        if (p.periodic) {
            // metadata: assemble_core's H = combine(0.5, Laplace, -1, Nuclear) and S = Mass;
            // the nuclear part needs the per-direction tables of the general contraction
            Work wn{};
            run_assembly(c, sd.get(), p, NEED_NUC, 3, AsmOut{}, &wn, nullptr, AS_GENERAL_NUC | AS_NO_FILL);
            auto lap = build_sep(c, p, LT_LAPLACE, w);
            auto nucm = build_sep(c, p, LT_NUCLEAR, wn);
            h->sep = sep_combine(c, *lap, 0.5, *nucm, -1.0);
            sop->sep = build_sep(c, p, LT_MASS, w);
            LT_CU(cudaStreamSynchronize(c->stream));
        }
        LT_CU(cudaStreamSynchronize(c->stream));
        *H = h.release();
        *S = sop.release();
    });
}

lt_status lt_combine(lt_ctx* c, double wa, const lt_operator* a, double wb, const lt_operator* b, lt_operator** out) {
    return guarded([&] {
        if (a->periodic != b->periodic || a->m0 != b->m0 || a->L[0] != b->L[0] || a->L[1] != b->L[1] ||
            a->L[2] != b->L[2])
            fail(LT_ESTRUCT, "combine: operators have different layouts");
        LT_CU(cudaSetDevice(c->device));
        auto op = std::make_unique<lt_operator>();
        op->which = a->which;
        op->periodic = a->periodic;
        op->m0 = a->m0;
        for (int l = 0; l < 3; ++l) {
            op->L[l] = a->L[l];
            op->band[l] = std::max(a->band[l], b->band[l]);
        }
        op->L0 = std::max(a->L0, b->L0);
        op->coefficient_rank = a->coefficient_rank + b->coefficient_rank;
        op->Nb = a->Nb;
        const Index mm = a->m0 * a->m0;
        if (!a->periodic) {
            op->count = a->count;
            LT_CU(cudaMalloc(&op->data, sizeof(double) * op->count));
            launch_axpby_map(c->L(), static_cast<Index>(op->count), 1, wa, a->data, nullptr, wb, b->data, nullptr,
                             op->data);
        } else {
            std::vector<int64_t> ia, ib;
            union_maps(a, b, op->kidx, ia, ib);
            op->count = op->kidx.size() * mm;
            LT_CU(cudaMalloc(&op->data, sizeof(double) * std::max<size_t>(op->count, 1)));
            int64_t* d = c->arena.get<int64_t>("combine.maps", 2 * ia.size() + 1);
            std::vector<int64_t> both(ia);
            both.insert(both.end(), ib.begin(), ib.end());
            upload(c, d, both.data(), both.size() * sizeof(int64_t));
            launch_axpby_map(c->L(), static_cast<Index>(op->kidx.size()), mm, wa, a->data, d, wb, b->data,
                             d + ia.size(), op->data);
            if (a->sep && b->sep) op->sep = sep_combine(c, *a->sep, wa, *b->sep, wb);
        }
        LT_CU(cudaStreamSynchronize(c->stream));
        *out = op.release();
    });
}

void lt_op_free(lt_operator* op) { delete op; }

void lt_op_info(const lt_operator* op, int64_t* info) {
    info[0] = op->periodic;
    info[1] = op->m0;
    for (int l = 0; l < 3; ++l) info[2 + l] = op->L[l];
    info[5] = op->L0;
    info[6] = op->coefficient_rank;
    info[7] = static_cast<int64_t>(op->kidx.size());
    info[8] = op->Nb;
    for (int l = 0; l < 3; ++l) info[9 + l] = op->band[l];
}

lt_status lt_op_dense(const lt_operator* op, double* out) {
    return guarded([&] {
        if (op->periodic) fail(LT_ESTRUCT, "lt_op_dense: periodic operator carries no dense payload");
        LT_CU(cudaMemcpy(out, op->data, sizeof(double) * op->count, cudaMemcpyDeviceToHost));
    });
}

lt_status lt_op_blocks(const lt_operator* op, int64_t* kidx, double* blocks) {
    return guarded([&] {
        if (!op->periodic) fail(LT_ESTRUCT, "lt_op_blocks: box operator carries no generating tensor");
        for (size_t i = 0; i < op->kidx.size(); ++i)
            for (int l = 0; l < 3; ++l) kidx[3 * i + l] = op->kidx[i][l];
        LT_CU(cudaMemcpy(blocks, op->data, sizeof(double) * op->count, cudaMemcpyDeviceToHost));
    });
}

static void solve_periodic_ops(lt_ctx* c, const lt_operator* H, const lt_operator* S, double* eig, double* vec) {
    if (!H->periodic || !S->periodic) fail(LT_ESTRUCT, "solve_periodic: operators must be periodic assemblies");
    if (H->m0 != S->m0 || H->L[0] != S->L[0] || H->L[1] != S->L[1] || H->L[2] != S->L[2])
        fail(LT_ESTRUCT, "solve_periodic: H and S layouts differ");
    LT_CU(cudaSetDevice(c->device));
    const Index K = H->L[0] * H->L[1] * H->L[2];
    double2* Hb = block_diag_device(c, H->L, H->m0, H->kidx, H->data, "H");
    double2* Sb = block_diag_device(c, S->L, S->m0, S->kidx, S->data, "S");
    pencils_to_host(c, K, H->m0, Hb, Sb, eig, vec);
}

lt_status lt_solve_periodic_ops(lt_ctx* c, const lt_operator* H, const lt_operator* S, double* eig) {
    return guarded([&] { solve_periodic_ops(c, H, S, eig, nullptr); });
}

lt_status lt_solve_periodic_ops_vectors(lt_ctx* c, const lt_operator* H, const lt_operator* S, double* eig,
                                        double* vec) {
    return guarded([&] { solve_periodic_ops(c, H, S, eig, vec); });
}

static void gen_to_device(lt_ctx* c, int64_t nblk, const int64_t* k, const double* b, Index m0,
                          std::vector<std::array<Index, 3>>& keys, double** dev, const std::string& tag) {
    // std::map order (block_circulant.hpp:47); later duplicates overwrite earlier ones (set_block)
    std::map<std::array<Index, 3>, int64_t> order;
    for (int64_t i = 0; i < nblk; ++i) order[{k[3 * i], k[3 * i + 1], k[3 * i + 2]}] = i;
    const Index mm = m0 * m0;
    std::vector<double> host;
    host.reserve(order.size() * mm);
    for (auto& kv : order) {
        keys.push_back(kv.first);
        host.insert(host.end(), b + kv.second * mm, b + (kv.second + 1) * mm);
    }
    *dev = c->arena.get<double>("gen." + tag, host.size() + 1);
    upload(c, *dev, host.data(), host.size() * sizeof(double));
}

static void check_gen_dims(const int64_t* dims, int64_t m0) {
    for (int l = 0; l < 3; ++l)
        if (dims[l] < 1) fail(LT_EDIM, "GeneratingBlockTensor: level extents must be >= 1");
    if (m0 < 1) fail(LT_EDIM, "GeneratingBlockTensor: m0 must be >= 1");
}

static void solve_periodic_gen(lt_ctx* c, const int64_t* dims, int64_t m0, int64_t nH, const int64_t* kH,
                               const double* bH, int64_t nS, const int64_t* kS, const double* bS, double* eig,
                               double* vec) {
    LT_CU(cudaSetDevice(c->device));
    check_gen_dims(dims, m0);
    std::vector<std::array<Index, 3>> keysH, keysS;
    double *dH = nullptr, *dS = nullptr;
    gen_to_device(c, nH, kH, bH, m0, keysH, &dH, "H");
    gen_to_device(c, nS, kS, bS, m0, keysS, &dS, "S");
    const Index d3[3] = {dims[0], dims[1], dims[2]};
    const Index K = d3[0] * d3[1] * d3[2];
    double2* Hb = block_diag_device(c, d3, m0, keysH, dH, "H");
    double2* Sb = block_diag_device(c, d3, m0, keysS, dS, "S");
    pencils_to_host(c, K, m0, Hb, Sb, eig, vec);
}

lt_status lt_solve_periodic(lt_ctx* c, const int64_t* dims, int64_t m0, int64_t nH, const int64_t* kH, const double* bH,
                            int64_t nS, const int64_t* kS, const double* bS, double* eig) {
    return guarded([&] { solve_periodic_gen(c, dims, m0, nH, kH, bH, nS, kS, bS, eig, nullptr); });
}

lt_status lt_solve_periodic_vectors(lt_ctx* c, const int64_t* dims, int64_t m0, int64_t nH, const int64_t* kH,
                                    const double* bH, int64_t nS, const int64_t* kS, const double* bS, double* eig,
                                    double* vec) {
    return guarded([&] { solve_periodic_gen(c, dims, m0, nH, kH, bH, nS, kS, bS, eig, vec); });
}

lt_status lt_block_diagonalize(lt_ctx* c, const int64_t* dims, int64_t m0, int64_t nblk, const int64_t* kidx,
                               const double* blocks, double* out) {
    return guarded([&] {
        LT_CU(cudaSetDevice(c->device));
        check_gen_dims(dims, m0);
        std::vector<std::array<Index, 3>> keys;
        double* d = nullptr;
        gen_to_device(c, nblk, kidx, blocks, m0, keys, &d, "B");
        const Index d3[3] = {dims[0], dims[1], dims[2]};
        const Index K = d3[0] * d3[1] * d3[2];
        double2* bd = block_diag_device(c, d3, m0, keys, d, "B");
        LT_CU(cudaMemcpyAsync(out, bd, sizeof(double2) * K * m0 * m0, cudaMemcpyDeviceToHost, c->stream));
        LT_CU(cudaStreamSynchronize(c->stream));
    });
}

static void solve_box_dense_host(lt_ctx* c, int64_t n, const double* H, const double* S, int64_t cap, double* eig,
                                 double* vec) {
    if (n > cap)
        fail(LT_ECAP, "solve_box_dense: size " + std::to_string(n) + " exceeds dense cap " + std::to_string(cap));
    LT_CU(cudaSetDevice(c->device));
    double* dH = c->arena.get<double>("boxapi.H", n * n);
    double* dS = c->arena.get<double>("boxapi.S", n * n);
    double* e = c->arena.get<double>("boxapi.eig", n);
    double* dv = vec ? c->arena.get<double>("boxapi.vec", n * n) : nullptr;
    unsigned long long* fk = c->arena.get<unsigned long long>("solve.fail", 1);
    LT_CU(cudaMemsetAsync(fk, 0xff, sizeof(unsigned long long), c->stream));
    upload(c, dH, H, sizeof(double) * n * n);
    upload(c, dS, S, sizeof(double) * n * n);
    box_eig_device(c, n, dH, dS, e, fk, dv);
    unsigned long long key = ~0ull;
    LT_CU(cudaMemcpyAsync(&key, fk, sizeof(key), cudaMemcpyDeviceToHost, c->stream));
    LT_CU(cudaMemcpyAsync(eig, e, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    if (vec) LT_CU(cudaMemcpyAsync(vec, dv, sizeof(double) * n * n, cudaMemcpyDeviceToHost, c->stream));
    LT_CU(cudaStreamSynchronize(c->stream));
    raise_fail_key(key, false);
}

lt_status lt_solve_box_dense(lt_ctx* c, int64_t n, const double* H, const double* S, int64_t cap, double* eig) {
    return guarded([&] { solve_box_dense_host(c, n, H, S, cap, eig, nullptr); });
}

lt_status lt_solve_box_dense_vectors(lt_ctx* c, int64_t n, const double* H, const double* S, int64_t cap, double* eig,
                                     double* vec) {
    return guarded([&] { solve_box_dense_host(c, n, H, S, cap, eig, vec); });
}

static void pencil_eig_host(lt_ctx* c, int64_t count, int64_t m0, const double* Hc, const double* Sc, double* eig,
                            double* vec) {
    LT_CU(cudaSetDevice(c->device));
    const Index mm = m0 * m0;
    double2* dH = c->arena.get<double2>("pen.H", count * mm);
    double2* dS = c->arena.get<double2>("pen.S", count * mm);
    upload(c, dH, Hc, sizeof(double2) * count * mm);
    upload(c, dS, Sc, sizeof(double2) * count * mm);
    pencils_to_host(c, count, m0, dH, dS, eig, vec);
}

lt_status lt_pencil_eig(lt_ctx* c, int64_t count, int64_t m0, const double* Hc, const double* Sc, double* eig) {
    return guarded([&] { pencil_eig_host(c, count, m0, Hc, Sc, eig, nullptr); });
}

lt_status lt_pencil_eigvec(lt_ctx* c, int64_t count, int64_t m0, const double* Hc, const double* Sc, double* eig,
                           double* vec) {
    return guarded([&] { pencil_eig_host(c, count, m0, Hc, Sc, eig, vec); });
}

// reconstruct_eigenvectors (eigensolver.cpp:164-175): N x N complex, N = K m0 <= cap
lt_status lt_reconstruct_eigenvectors(lt_ctx* c, const int64_t* dims, int64_t m0, const double* vec, int64_t cap,
                                      double* out) {
    return guarded([&] {
        check_gen_dims(dims, m0);
        const Index d3[3] = {dims[0], dims[1], dims[2]};
        const Index K = d3[0] * d3[1] * d3[2], N = K * m0;
        if (N > cap) fail(LT_ECAP, "reconstruct_eigenvectors: size exceeds cap");
        LT_CU(cudaSetDevice(c->device));
        double2* u = c->arena.get<double2>("rec.u", K * m0 * m0);
        double2* o = c->arena.get<double2>("rec.out", N * N);
        upload(c, u, vec, sizeof(double2) * K * m0 * m0);
        launch_reconstruct(c->L(), d3, m0, u, 0, N, o);
        LT_CU(cudaMemcpyAsync(out, o, sizeof(double2) * N * N, cudaMemcpyDeviceToHost, c->stream));
        LT_CU(cudaStreamSynchronize(c->stream));
    });
}

// bc_full_eigenvector (block_circulant.cpp:267-289): column (j, m), N complex
lt_status lt_bc_full_eigenvector(lt_ctx* c, const int64_t* dims, int64_t m0, const double* vec, int64_t j, int64_t m,
                                 double* out) {
    return guarded([&] {
        check_gen_dims(dims, m0);
        const Index d3[3] = {dims[0], dims[1], dims[2]};
        const Index K = d3[0] * d3[1] * d3[2], N = K * m0;
        if (j < 0 || j >= K || m < 0 || m >= m0) fail(LT_EBOUNDS, "bc_full_eigenvector: (k-point, band) out of range");
        LT_CU(cudaSetDevice(c->device));
        double2* u = c->arena.get<double2>("rec.u", K * m0 * m0);
        double2* o = c->arena.get<double2>("rec.col", N);
        upload(c, u, vec, sizeof(double2) * K * m0 * m0);
        launch_reconstruct(c->L(), d3, m0, u, j * m0 + m, 1, o);
        LT_CU(cudaMemcpyAsync(out, o, sizeof(double2) * N, cudaMemcpyDeviceToHost, c->stream));
        LT_CU(cudaStreamSynchronize(c->stream));
    });
}

lt_status lt_sinc_quadrature(lt_ctx* c, int64_t M, double* nodes, double* weights) {
    return guarded([&] {
        if (M < 1) fail(LT_EDIM, "build_sinc_quadrature: M must be >= 1");
        LT_CU(cudaSetDevice(c->device));
        const Index R = 2 * M + 1;
        double* t = c->arena.get<double>("sinc.t", R);
        double* w = c->arena.get<double>("sinc.w", R);
        double* pw = c->arena.get<double>("sinc.potw", R);
        double* one = c->arena.get<double>("sinc.one", 1);
        const double h1 = 1.0;
        upload(c, one, &h1, sizeof(double));
        DevSys s{};
        s.nnuc = 1;
        s.Z = one;
        launch_sinc(c->L(), M, s, t, w, pw);
        LT_CU(cudaMemcpyAsync(nodes, t, sizeof(double) * R, cudaMemcpyDeviceToHost, c->stream));
        LT_CU(cudaMemcpyAsync(weights, w, sizeof(double) * R, cudaMemcpyDeviceToHost, c->stream));
        LT_CU(cudaStreamSynchronize(c->stream));
    });
}

lt_status lt_overlap_constant(lt_ctx* c, const lt_system* s, int64_t* L0) {
    return guarded([&] {
        LT_CU(cudaSetDevice(c->device));
        std::unique_ptr<lt_sysdev, void (*)(lt_sysdev*)> sd(make_sysdev(s), lt_sys_free);
        // overlap_constant validates the basis and (n, b) only (gto_basis.cpp:88-89)
        const HostSys& h = sd->hs;
        if (h.alpha.empty()) fail(LT_ESTRUCT, "GtoBasis: no functions");
        for (size_t m = 0; m < h.alpha.size(); ++m)
            if (h.alpha[m] <= 0.0) fail(LT_ESTRUCT, "GtoBasis: exponents must be positive");
        for (int l = 0; l < 3; ++l)
            if (h.n[l] < 1 || h.b <= 0.0) fail(LT_EDIM, "overlap_constant: need n >= 1, b > 0");
        *L0 = compute_L0(c, sd.get());
    });
}

lt_status lt_newton_master(lt_ctx* c, int64_t ncells, double h, int64_t M, double* out) {
    return guarded([&] {
        LT_CU(cudaSetDevice(c->device));
        const Index R = 2 * M + 1;
        double* t = c->arena.get<double>("sinc.t", R);
        double* w = c->arena.get<double>("sinc.w", R);
        double* pw = c->arena.get<double>("sinc.potw", R);
        double* one = c->arena.get<double>("sinc.one", 1);
        const double h1 = 1.0;
        upload(c, one, &h1, sizeof(double));
        DevSys s{};
        s.nnuc = 1;
        s.Z = one;
        launch_sinc(c->L(), M, s, t, w, pw);
        double* m = c->arena.get<double>("api.master", ncells * R);
        launch_master(c->L(), ncells, h, R, t, m);
        LT_CU(cudaMemcpyAsync(out, m, sizeof(double) * ncells * R, cudaMemcpyDeviceToHost, c->stream));
        LT_CU(cudaStreamSynchronize(c->stream));
    });
}

lt_status lt_potential(lt_ctx* c, const lt_system* s, int periodic, int64_t margin, int64_t* rows, int64_t* tiled,
                       double* panels, double* weights, int64_t panels_cap) {
    return guarded([&] {
        LT_CU(cudaSetDevice(c->device));
        std::unique_ptr<lt_sysdev, void (*)(lt_sysdev*)> sd(make_sysdev(s), lt_sys_free);
        validate(sd->hs);
        // margin given directly: plan with L0 = margin - 2 and no alias guard (stage call)
        Plan q;
        plan_after_L0(sd->hs, periodic != 0, margin - 2, q, true, false);
        Index need = 0;
        for (int l = 0; l < 3; ++l) {
            rows[l] = q.d[l].pot_rows;
            tiled[l] = q.d[l].tiled;
            need += q.d[l].pot_rows * q.Rtot;
        }
        if (!panels || need > panels_cap) return;
        const Launch L = c->L();
        double* t = c->arena.get<double>("sinc.t", q.RN);
        double* w = c->arena.get<double>("sinc.w", q.RN);
        double* pw = c->arena.get<double>("sinc.potw", q.Rtot);
        launch_sinc(L, q.M, sd->ds, t, w, pw);
        std::vector<int64_t> s0all;
        for (int l = 0; l < 3; ++l)
            for (Index v : q.d[l].s0) s0all.push_back(v);
        int64_t* s0d = c->arena.get<int64_t>("pot.s0", s0all.size());
        upload(c, s0d, s0all.data(), s0all.size() * sizeof(int64_t));
        Index at = 0;
        for (int l = 0; l < 3; ++l) {
            const DirPlan& d = q.d[l];
            double* master = c->arena.get<double>("pot.master" + std::to_string(l), d.mrows * q.RN);
            double* pan = c->arena.get<double>("api.panel" + std::to_string(l), d.pot_rows * q.Rtot);
            launch_master(L, d.mrows, d.h, q.RN, t, master);
            launch_window_sum(L, master, d.mrows, q.RN, q.nnuc, s0d + l * q.nnuc, d.nsum, d.n, d.pot_rows, pan);
            LT_CU(cudaMemcpyAsync(panels + at, pan, sizeof(double) * d.pot_rows * q.Rtot, cudaMemcpyDeviceToHost,
                                  c->stream));
            at += d.pot_rows * q.Rtot;
        }
        LT_CU(cudaMemcpyAsync(weights, pw, sizeof(double) * q.Rtot, cudaMemcpyDeviceToHost, c->stream));
        LT_CU(cudaStreamSynchronize(c->stream));
    });
}

lt_status lt_assembled_window_sum(lt_ctx* c, int64_t mrows, int64_t R, const double* master, int64_t nsh,
                                  const int64_t* shifts, int64_t size, double* out) {
    return guarded([&] {
        if (nsh < 1) fail(LT_ESTRUCT, "assembled_window_sum: empty shift set");
        for (int64_t i = 0; i < nsh; ++i)
            if (shifts[i] < 0 || shifts[i] + size > mrows)
                fail(LT_EBOUNDS, "assembled_window_sum: shift " + std::to_string(shifts[i]) +
                                     " in direction 0 outside master extent " + std::to_string(mrows));
        // the device kernel covers the uniform progression and the single-shift case
        // (the only shapes the lattice sums produce); canonical_tensor.cpp:112-119
        bool uniform = nsh >= 2;
        const int64_t step = nsh >= 2 ? shifts[1] - shifts[0] : 0;
        if (uniform && step <= 0) uniform = false;
        for (int64_t i = 2; uniform && i < nsh; ++i)
            if (shifts[i] - shifts[i - 1] != step) uniform = false;
        if (nsh >= 2 && !uniform) fail(LT_EGENERIC, "assembled_window_sum: non-uniform shift sets are not supported on the device");
        LT_CU(cudaSetDevice(c->device));
        double* m = c->arena.get<double>("aws.m", mrows * R);
        double* o = c->arena.get<double>("aws.o", size * R);
        int64_t* s0 = c->arena.get<int64_t>("aws.s0", 1);
        upload(c, m, master, sizeof(double) * mrows * R);
        upload(c, s0, shifts, sizeof(int64_t));
        launch_window_sum(c->L(), m, mrows, R, 1, s0, nsh, step, size, o);
        LT_CU(cudaMemcpyAsync(out, o, sizeof(double) * size * R, cudaMemcpyDeviceToHost, c->stream));
        LT_CU(cudaStreamSynchronize(c->stream));
    });
}

lt_status lt_profiles(lt_ctx* c, const lt_system* s, int64_t margin, int64_t* grid, int64_t* lo, int64_t* hi,
                      double* values, int64_t values_cap) {
    return guarded([&] {
        LT_CU(cudaSetDevice(c->device));
        std::unique_ptr<lt_sysdev, void (*)(lt_sysdev*)> sd(make_sysdev(s), lt_sys_free);
        validate(sd->hs);
        const HostSys& h = sd->hs;
        const Index m0 = h.m0();
        Index need = 0;
        for (int kind = 0; kind < 2; ++kind)
            for (int l = 0; l < 3; ++l) {
                const Index g = (h.L[l] + 2 * margin) * (kind == 0 ? h.n[l] : h.nbar[l]);
                grid[kind * 3 + l] = g;
                need += g * m0;
            }
        if (!values || need > values_cap) return;
        ProfileJob jobs[6];
        for (int kind = 0; kind < 2; ++kind)
            for (int l = 0; l < 3; ++l) {
                ProfileJob& j = jobs[kind * 3 + l];
                j.grid = grid[kind * 3 + l];
                j.per_cell = kind == 0 ? h.n[l] : h.nbar[l];
                j.cell_index = margin;
                j.step = kind == 0 ? h.h(l) : h.hbar(l);
                j.align = kind == 0 ? 0.5 : 0.0;
                j.dir = l;
                j.values = c->arena.get<double>("api.prof" + std::to_string(kind * 3 + l), m0 * j.grid);
                j.lo = c->arena.get<unsigned long long>("api.plo" + std::to_string(kind * 3 + l), m0);
                j.hi = c->arena.get<unsigned long long>("api.phi" + std::to_string(kind * 3 + l), m0);
            }
        launch_profiles(c->L(), sd->ds, jobs, 6, 1e-280);
        Index at = 0;
        for (int k = 0; k < 6; ++k) {
            LT_CU(cudaMemcpyAsync(values + at, jobs[k].values, sizeof(double) * m0 * jobs[k].grid,
                                  cudaMemcpyDeviceToHost, c->stream));
            at += m0 * jobs[k].grid;
            LT_CU(cudaMemcpyAsync(lo + k * m0, jobs[k].lo, sizeof(int64_t) * m0, cudaMemcpyDeviceToHost, c->stream));
            LT_CU(cudaMemcpyAsync(hi + k * m0, jobs[k].hi, sizeof(int64_t) * m0, cudaMemcpyDeviceToHost, c->stream));
        }
        LT_CU(cudaStreamSynchronize(c->stream));
    });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// factorized path entry points (eigensolver.hpp solve_periodic_factorized,
// factorized_diag.hpp factorized_block_diagonalize, galerkin.hpp separable_residual)
// ---------------------------------------------------------------------------
int64_t lt_op_separable_count(const lt_operator* op) {
    if (!op || !op->sep) return 0;
    return op->sep->terms * (op->L[0] + op->L[1] + op->L[2]) * op->m0 * op->m0;
}

lt_status lt_op_separable(const lt_operator* op, double* out) {
    return guarded([&] {
        if (!op->periodic) fail(LT_ESTRUCT, "separable_residual: box operators carry no metadata");
        if (!op->sep) fail(LT_ESTRUCT, "separable_residual: no metadata present");
        const SepMeta& m = *op->sep;
        const Index mm = m.m0 * m.m0;
        std::vector<double> v(m.count());
        LT_CU(cudaMemcpy(v.data(), m.vals, sizeof(double) * v.size(), cudaMemcpyDeviceToHost));
        const Index per_term = (m.L[0] + m.L[1] + m.L[2]) * mm;
        std::fill(out, out + m.terms * per_term, 0.0);
        for (Index t = 0; t < m.terms; ++t) {
            Index loff = 0;
            for (int l = 0; l < 3; ++l) {
                for (size_t q = 0; q < m.kid[l].size(); ++q)
                    std::memcpy(out + t * per_term + loff + m.kid[l][q] * mm,
                                &v[static_cast<size_t>(((t * 3 + l) * m.S + static_cast<Index>(q)) * mm)],
                                sizeof(double) * mm);
                loff += m.L[l] * mm;
            }
        }
    });
}

lt_status lt_separable_residual(lt_ctx* c, const lt_operator* op, double* resid) {
    return guarded([&] {
        if (!op->periodic) fail(LT_ESTRUCT, "separable_residual: box operators carry no metadata");
        if (!op->sep) fail(LT_ESTRUCT, "separable_residual: no metadata present");
        LT_CU(cudaSetDevice(c->device));
        *resid = sep_residual(c, *op->sep, op->kidx, op->data, "R");
    });
}

static void solve_factorized_ops(lt_ctx* c, const lt_operator* H, const lt_operator* S, double metadata_tol,
                                 double* eig, double* vec) {
    if (!H->periodic || !S->periodic)
        fail(LT_ESTRUCT, "solve_periodic_factorized: operators must be periodic assemblies");
    if (!H->sep || !S->sep || H->sep->terms == 0 || S->sep->terms == 0)
        fail(LT_ESTRUCT, "solve_periodic_factorized: rank metadata missing");
    LT_CU(cudaSetDevice(c->device));
    sep_check_resid(sep_residual(c, *H->sep, H->kidx, H->data, "H"), metadata_tol);
    sep_check_resid(sep_residual(c, *S->sep, S->kidx, S->data, "S"), metadata_tol);
    sep_solve(c, *H->sep, *S->sep, eig, vec);
}

lt_status lt_solve_periodic_factorized(lt_ctx* c, const lt_operator* H, const lt_operator* S, double metadata_tol,
                                       double* eig) {
    return guarded([&] { solve_factorized_ops(c, H, S, metadata_tol, eig, nullptr); });
}

lt_status lt_solve_periodic_factorized_vectors(lt_ctx* c, const lt_operator* H, const lt_operator* S,
                                               double metadata_tol, double* eig, double* vec) {
    return guarded([&] { solve_factorized_ops(c, H, S, metadata_tol, eig, vec); });
}

static void check_levels(int levels, const int64_t* dims, Index nterms) {
    if (levels < 1 || levels > 3) fail(LT_ESTRUCT, "FactorizedDiagonalizer: levels must be 1, 2 or 3");
    if (nterms <= 0) fail(LT_ESTRUCT, "FactorizedDiagonalizer: no separable terms");
    for (int l = levels; l < 3; ++l)
        if (dims[l] != 1)
            fail(LT_ESTRUCT, "FactorizedDiagonalizer: level " + std::to_string(l) + " sequence must have 1 blocks");
}

lt_status lt_factorized_block_diagonalize(lt_ctx* c, int levels, const int64_t* dims, int64_t m0, int64_t nterms,
                                          const double* terms, double* out) {
    return guarded([&] {
        check_levels(levels, dims, nterms);
        check_gen_dims(dims, m0);
        LT_CU(cudaSetDevice(c->device));
        const Index L[3] = {dims[0], dims[1], dims[2]};
        auto m = sep_from_full(c, m0, L, nterms, terms);
        double2* F = sep_fourier(c, *m, "B");
        const Index K = L[0] * L[1] * L[2];
        LT_CU(cudaMemcpyAsync(out, F, sizeof(double2) * K * m0 * m0, cudaMemcpyDeviceToHost, c->stream));
        LT_CU(cudaStreamSynchronize(c->stream));
    });
}

lt_status lt_solve_periodic_factorized_gen(lt_ctx* c, const int64_t* dims, int64_t m0, int64_t nH, const int64_t* kH,
                                           const double* bH, int64_t tH, const double* termsH, int64_t nS,
                                           const int64_t* kS, const double* bS, int64_t tS, const double* termsS,
                                           double metadata_tol, double* eig) {
    return guarded([&] {
        check_gen_dims(dims, m0);
        if (tH <= 0 || tS <= 0) fail(LT_ESTRUCT, "solve_periodic_factorized: rank metadata missing");
        LT_CU(cudaSetDevice(c->device));
        std::vector<std::array<Index, 3>> keysH, keysS;
        double *dH = nullptr, *dS = nullptr;
        gen_to_device(c, nH, kH, bH, m0, keysH, &dH, "H");
        gen_to_device(c, nS, kS, bS, m0, keysS, &dS, "S");
        const Index L[3] = {dims[0], dims[1], dims[2]};
        auto mH = sep_from_full(c, m0, L, tH, termsH);
        auto mS = sep_from_full(c, m0, L, tS, termsS);
        sep_check_resid(sep_residual(c, *mH, keysH, dH, "H"), metadata_tol);
        sep_check_resid(sep_residual(c, *mS, keysS, dS, "S"), metadata_tol);
        sep_solve(c, *mH, *mS, eig);
    });
}

// box_circulant_defect (galerkin.cpp:445-454): Nuclear assembled both ways, the periodic
// circulant expanded densely; rel_fro = ||box - per|| / ||box||. defect (optional): Nb*Nb.
lt_status lt_box_circulant_defect(lt_ctx* c, const lt_system* s, double* rel_fro, double* defect) {
    return guarded([&] {
        LT_CU(cudaSetDevice(c->device));
        lt_operator* bo = nullptr;
        lt_operator* po = nullptr;
        lt_status st = lt_assemble(c, s, 0, LT_NUCLEAR, &bo);
        if (st != LT_OK) fail(static_cast<int>(st), lt_last_error());
        std::unique_ptr<lt_operator> box(bo);
        st = lt_assemble(c, s, 1, LT_NUCLEAR, &po);
        if (st != LT_OK) fail(static_cast<int>(st), lt_last_error());
        std::unique_ptr<lt_operator> per(po);
        const Index K = per->L[0] * per->L[1] * per->L[2];
        std::vector<int> go(static_cast<size_t>(K), -1);
        for (size_t b = 0; b < per->kidx.size(); ++b)
            go[static_cast<size_t>((per->kidx[b][0] * per->L[1] + per->kidx[b][1]) * per->L[2] + per->kidx[b][2])] =
                static_cast<int>(b);
        StageScope ss(c, 1 << 20);
        int* gd = c->arena.get<int>("defect.gen", go.size());
        upload(c, gd, go.data(), go.size() * sizeof(int));
        CircDefect d;
        d.Nb = box->Nb;
        d.m0 = box->m0;
        for (int l = 0; l < 3; ++l) d.L[l] = per->L[l];
        d.box = box->data;
        d.gen = per->data;
        d.gen_of = gd;
        d.defect = defect ? c->arena.get<double>("defect.out", d.Nb * d.Nb) : nullptr;
        const int blocks = static_cast<int>(std::min<Index>(148 * 4, (d.Nb * d.Nb + 255) / 256));
        d.partial = c->arena.get<double>("defect.part", 2 * blocks);
        launch_circ_defect(c->L(), d, blocks);
        std::vector<double> part(static_cast<size_t>(2 * blocks));
        LT_CU(cudaMemcpyAsync(part.data(), d.partial, sizeof(double) * part.size(), cudaMemcpyDeviceToHost, c->stream));
        if (defect)
            LT_CU(cudaMemcpyAsync(defect, d.defect, sizeof(double) * d.Nb * d.Nb, cudaMemcpyDeviceToHost, c->stream));
        LT_CU(cudaStreamSynchronize(c->stream));
        double sd = 0.0, sb = 0.0;
        for (int b = 0; b < blocks; ++b) {
            sd += part[static_cast<size_t>(2 * b)];
            sb += part[static_cast<size_t>(2 * b + 1)];
        }
        *rel_fro = std::sqrt(sd) / std::sqrt(sb);
    });
}
