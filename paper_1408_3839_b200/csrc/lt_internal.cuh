// lt_internal.cuh — shared declarations of the B200-native core-Hamiltonian engine.
//
// Host planning structures (Plan/DirPlan), the device-side system view (DevSys),
// error plumbing and the launch wrappers of every kernel. See DESIGN.md for the
// data layout in HBM and the roofline of each kernel.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "latham_b200.h"

namespace lt {

using Index = std::int64_t;

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& m) { throw Error(code, m); }

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(LT_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define LT_CU(x) ::lt::cuda_check((x), #x)

// ---------------------------------------------------------------------------
// Device view of one LatticeSystem (all arrays device-resident)
// ---------------------------------------------------------------------------
struct DevSys {
    int m0 = 0, nnuc = 0;
    double b = 0.0, eps_ov = 0.0;
    const double* pos = nullptr;    // [nnuc][3]
    const double* Z = nullptr;      // [nnuc]
    const double* center = nullptr; // [m0][3]
    const double* alpha = nullptr;  // [m0]
    const int* deg = nullptr;       // [m0][3]
};

// Host copy of the system (validated), reference field names (galerkin.hpp:17-35)
struct HostSys {
    double b = 0.0;
    Index L[3]{1, 1, 1}, n[3]{}, nbar[3]{};
    Index quad_M = 0;
    double eps_ov = 1e-8;
    std::vector<double> pos, Z, center, alpha;
    std::vector<int> deg;
    Index m0() const { return static_cast<Index>(alpha.size()); }
    Index nnuc() const { return static_cast<Index>(Z.size()); }
    Index cells() const { return L[0] * L[1] * L[2]; }
    double h(int l) const { return b / static_cast<double>(n[l]); }
    double hbar(int l) const { return b / static_cast<double>(nbar[l]); }
};

HostSys host_sys_from(const lt_system* s);
void validate(const HostSys& s);

// table modes of the nuclear contraction per direction
enum TableMode : int { TM_TRIVIAL = 0, TM_FOLD = 1, TM_BOXDIR = 2 };

struct DirPlan {
    Index L = 1, n = 0, nbar = 0;
    double h = 0.0, hbar = 0.0;
    Index band = 0, width = 1;    // band = min(L0, L-1), width = 2 band + 1
    Index G = 0, Gbar = 0;        // pwc / pwl extended grid sizes
    Index pot_rows = 0;           // rows of the potential panel
    bool tiled = false;           // periodic wrapped direction (p addressed mod n)
    Index mrows = 0;              // master grid cells
    Index nsum = 1;               // lattice copies in the window sum
    std::vector<Index> s0;        // per nucleus: smallest sorted window start
    int mode = TM_TRIVIAL;
    Index npairs = 1;             // table pairs: box L*width, periodic width, trivial 1
};

struct Plan {
    bool periodic = false;
    Index m0 = 0, nnuc = 0, RN = 0, Rtot = 0, M = 0;
    Index L0 = 0, margin = 0;
    DirPlan d[3];
    Index cells = 1, Nb = 0, K = 1;
    int nontrivial = 0;       // directions with L > 1
    int s2_dir = -1;          // box: the single nontrivial direction folded by rank (S2)
    Index nblocks = 0;        // periodic: stored generating blocks = prod(width)
};

// planning (host integer bookkeeping; reference semantics, galerkin.cpp:287-307,
// newton_kernel.cpp:54-151). Throws lt::Error with the reference's messages.
void plan_after_L0(const HostSys& s, bool periodic, Index L0, Plan& p, bool need_potential, bool check_alias = true);
Index master_rows_box(Index n, Index L, Index margin);
Index master_rows_periodic(Index n, Index L);
Index window_start(Index master_n, Index win_n, double a, double h);

// ---------------------------------------------------------------------------
// Device buffer arena (grow-only, keyed)
// ---------------------------------------------------------------------------
class Arena {
public:
    ~Arena();
    void* raw(const std::string& key, size_t bytes);
    template <class T>
    T* get(const std::string& key, size_t count) {
        return static_cast<T*>(raw(key, count * sizeof(T) + 16));
    }
    size_t bytes() const;
    uint64_t generation() const { return gen_; }  // bumps on every (re)allocation

private:
    struct Buf {
        void* p = nullptr;
        size_t cap = 0;
    };
    std::map<std::string, Buf> bufs_;
    uint64_t gen_ = 0;
};

// ---------------------------------------------------------------------------
// kernel launch wrappers (each increments the launch counter)
// ---------------------------------------------------------------------------
// Optional per-kernel CUDA-event timing on the launching stream (bench roofline).
class StageTimer {
public:
    ~StageTimer();
    bool on = false;
    void begin(cudaStream_t st, const char* name);
    void end(cudaStream_t st);
    // resolve pending event pairs (call after a stream synchronisation)
    void collect();
    void reset();
    std::map<std::string, std::pair<double, int64_t>> totals;  // name -> (ms, launches)
    // per-launch timeline relative to the last mark_ref() (stage-timing mode only)
    struct Span {
        std::string name;
        cudaStream_t stream;
        double t0, t1;
    };
    std::vector<Span> timeline;
    void mark_ref(cudaStream_t st);
    // graph capture with timing on: events come from `owned` (kept alive by the graph) and
    // the begin/end pairs of the captured launches are replayed into pending_ per launch
    struct Pending {
        std::string name;
        cudaEvent_t a, b;
        cudaStream_t st;
        cudaEvent_t ref;
    };
    std::vector<cudaEvent_t>* owned = nullptr;
    size_t pending_size() const { return pending_.size(); }
    std::vector<Pending> take_pending(size_t from) {
        std::vector<Pending> out(pending_.begin() + static_cast<std::ptrdiff_t>(from), pending_.end());
        pending_.resize(from);
        return out;
    }
    void add_pending(const std::vector<Pending>& v) {
        for (Pending p : v) {
            p.ref = ref_;
            pending_.push_back(p);
        }
    }

private:
    cudaEvent_t get();
    std::vector<cudaEvent_t> pool_;
    size_t used_ = 0;
    cudaEvent_t ref_ = nullptr;
    std::vector<Pending> pending_;
    std::string open_name_;
    cudaEvent_t open_ = nullptr;
};

struct Launch {
    cudaStream_t st = nullptr;
    int64_t* counter = nullptr;
    StageTimer* timer = nullptr;
    void tick(int n = 1) const {
        if (counter) *counter += n;
    }
};

// RAII stage scope: events around the kernel(s) launched inside it when timing is on
struct Stage {
    const Launch& L;
    bool active;
    Stage(const Launch& l, const char* name) : L(l), active(l.timer && l.timer->on) {
        if (active) L.timer->begin(L.st, name);
    }
    ~Stage() {
        if (active) L.timer->end(L.st);
    }
};

// sinc quadrature (sinc_quadrature.cpp:9-29) and the nuclear weights Z_v w_q
// rank terms outside [r0, r1) get weight 0 (r1 < 0: all)
void launch_sinc(const Launch& L, Index M, const DevSys& s, double* t, double* w, double* potw, Index r0 = 0,
                 Index r1 = -1);

// overlap constant (gto_basis.cpp:87-126)
struct OverlapBufs {
    double* prof = nullptr;   // [3][m0][width_l] packed per direction (non-zero blocks only)
    double* bmax = nullptr;   // [3][m0][nblk_l]
    unsigned* nz = nullptr;   // [3][m0][2]: first / last non-zero block
    int* found = nullptr;     // [257]
    int* state = nullptr;     // [5]: L0, misses, s_next, done, finished-CTA counter
};
constexpr int kL0Block = 128;
// active[l] = 0 skips a direction whose (n, centre, degree) columns duplicate an earlier one
void launch_overlap_profiles(const Launch& L, const DevSys& s, const Index* n3, const Index* off3,
                             const Index* boff3, const int* active, OverlapBufs b);
// scan of shifts [s_begin, s_end) with the sequential L0 rule fused into the last CTA
void launch_overlap_scan(const Launch& L, const DevSys& s, const Index* n3, const Index* off3, const Index* boff3,
                         const int* active, OverlapBufs b, int s_begin, int s_end, bool finalize);
// degree-0 directions: exact peak-window search instead of sampling + scanning
void launch_overlap_peak(const Launch& L, const DevSys& s, const Index* n3, const int* active, OverlapBufs b,
                         int s_begin, int s_end, bool finalize);
void launch_overlap_init(const Launch& L, OverlapBufs b, int m0);

// master tensor (newton_kernel.cpp:22-45) and assembled window sums (canonical_tensor.cpp:123-164)
// t == null: nodes evaluated in place from M (no dependency on the sinc kernel)
void launch_master(const Launch& L, Index mrows, double h, Index RN, const double* t, double* out, Index M = 0);
void launch_sinc_nodes(const Launch& L, Index M, double* t);
// window sums with the master cells evaluated in place (no master panel)
void launch_potential_fused(const Launch& L, Index mrows, double h, Index M, Index RN, Index nnuc, const Index* s0_dev,
                            Index nsum, Index step, Index size, double* out);
void launch_window_sum(const Launch& L, const double* master, Index mrows, Index RN, Index nnuc, const Index* s0_dev,
                       Index nsum, Index step, Index size, double* out);

// GTO profiles (gto_basis.cpp:31-47) with trimming
struct ProfileJob {
    Index grid = 0, per_cell = 0, cell_index = 0;
    double step = 0.0, align = 0.0;
    int dir = 0;
    double* values = nullptr;  // [m0][grid]
    unsigned long long* lo = nullptr;  // [m0]
    unsigned long long* hi = nullptr;  // [m0]
};
void launch_profiles(const Launch& L, const DevSys& s, const ProfileJob* jobs, int njobs, double eps);

// 1D FEM tables (fem1d.cpp:19-32 via galerkin.cpp:208-223)
void launch_fem_tables(const Launch& L, Index m0, Index band, Index nbar, double hbar, Index Gbar, const double* pwl,
                       const unsigned long long* lo, const unsigned long long* hi, double* massT, double* stiffT);

// nuclear tables by direct contraction (galerkin.cpp:109-125, :224-247)
void launch_nuc_direct(const Launch& L, Index m0, Index Rtot, const DirPlan& d, bool periodic, const double* pwc,
                       const unsigned long long* lo, const unsigned long long* hi, const double* pot, double* T);
// periodic fold: Qf[d][e][t] then T[d][r][e] = sum_t P[r][t] Qf[d][e][t]
void launch_nuc_fold(const Launch& L, Index m0, Index Rtot, const DirPlan& d, const double* pwc,
                     const unsigned long long* lo, const unsigned long long* hi, const double* pot, double* Qf,
                     double* T);

// ---- DMMA nuclear contraction (k_nuclear2.cu) ----
struct TrivJob {
    const double* pot = nullptr;  // potential panel [Rtot][rows]; null: evaluated in place
    long long rows = 0;
    // in-place potential (pot == null): P[v RN + q][i] = master_cell(s0[v] + i, mrows, h, t_q)
    long long mrows = 0;
    double h = 0.0;
    int M = 0, RN = 0;
    const Index* s0 = nullptr;
    const double* pwc = nullptr;  // profiles [m0][G]
    long long G = 0;
    const unsigned long long* lo = nullptr;
    const unsigned long long* hi = nullptr;
};
struct TrivJobs {
    TrivJob j[3];
};
struct WSpec {
    int job_of_dir[3] = {-1, -1, -1};  // trivial direction -> job (directions may share one)
};
struct KRArgs {
    int m0 = 0, Rtot = 0;
    int width[3] = {1, 1, 1}, band[3] = {0, 0, 0};
    const double* T[3] = {nullptr, nullptr, nullptr};  // [d>=0][r][e] per wrapped direction
    const double* W = nullptr;
    double* N = nullptr;
    // fused fill (the periodic spectrum path): H = kin Lap - N and S = Mass of every block
    // written entry-major, H[e][slot] (slot = k_fill's periodic slot), with kidx; N unused
    double* H = nullptr;
    double* S = nullptr;
    int64_t* kidx = nullptr;
    const double* massT[3] = {nullptr, nullptr, nullptr};
    const double* stiffT[3] = {nullptr, nullptr, nullptr};
    double kin = 0.5;
    long long L[3] = {1, 1, 1};
    long long nblocks = 0;
};
void launch_triv_tables(const Launch& L, const TrivJobs& jobs, int njobs, const WSpec& ws, int m0, int Rtot,
                        const double* potw, double* part, int splits, double* W, double* Tout, bool async = false);
// V = W^T P on a periodic cell panel, one thread per output (large W; small ones fuse into the fold)
void launch_vdot(const Launch& L, int mm, int Rtot, long long rows, const double* W, const double* P, double* V);
void launch_vgemm(const Launch& L, int mm, int Rtot, long long rows, const double* W, const double* P, double* V);
void launch_hankel(const Launch& L, int m0, const DirPlan& d, const double* pwc, const unsigned long long* lo,
                   const unsigned long long* hi, const double* V, double* part, double* N, int splits, bool padded = false);
int hankel_res_splits(const DirPlan& d);
// ---- residue-class correlations on DMMA (k_fold.cu) ----
struct FemApplyJob {
    const double* pwl = nullptr;  // [m0][Gbar]
    long long Gbar = 0;
    double hbar = 0.0;
    const unsigned long long* lo = nullptr;
    const unsigned long long* hi = nullptr;
    double* wm = nullptr;  // [m0][Gbar] mass-applied profiles
    double* ws = nullptr;  // [m0][Gbar] stiffness-applied profiles
};
struct FemApplyJobs {
    FemApplyJob j[3];
};
void launch_fem_apply(const Launch& L, const FemApplyJobs& jobs, int njobs, int m0);
struct ResFold {
    int m0 = 0;
    long long J = 0, n = 0, G = 0;  // cells, points per cell (residues), grid = J*n
    const double* a = nullptr;      // [m0][G]
    const double* b[2] = {nullptr, nullptr};  // [m0][G], or [m0][G+2] with one guard each side
    int nb = 1;
    int bguard = 0;
    int dlo = 0, dhi = 0, dchunk = 1, band = 0;
    const double* V = nullptr;      // optional weight V[e][t]
    double* out[2] = {nullptr, nullptr};  // [t][d - dlo][e]
    double* res[2] = {nullptr, nullptr};  // reduced [d + band][e]
    double* slab = nullptr;               // workspace [n][1+nb][m0p][ldj] (residue-major); null: direct gather
    // fused weight (instead of V): wgt(e, t) = sum_r W[r][e] P[r][t], P rows of length prow
    const double* W = nullptr;
    const double* P = nullptr;
    int Rtot = 0;
    long long prow = 0;
    // supports [lo, hi) in grid index of the a- and b-profiles (b: the a support widened by
    // bwiden on each side, e.g. 1 for T v); when set, each (tile, d) task sweeps only the j
    // range where both tiles have non-zero values
    const unsigned long long* sup_lo = nullptr;
    const unsigned long long* sup_hi = nullptr;
    int bwiden = 0;
    // window: the fold covers grid cells [jw0, jw0 + J) (J counts window cells); every
    // profile is zero outside it (support_window in engine.cu), so long periodic chains do
    // not stage the empty cells of the extended grid
    long long jw0 = 0;
};
// slab row stride: >= J + 5 (two guard columns plus zero padding for the unchecked last
// k-step), == 4 mod 16 so the 8 rows x 4 columns of an m8n8k4 fragment hit distinct banks
__host__ __device__ inline long long resfold_ldj(long long J) { return (J + 16) / 16 * 16 + 4; }
// residue classes this short are gathered directly by the fold (no transpose launch)
constexpr long long kResfoldDirectJ = 128;
inline size_t resfold_slab_doubles(const ResFold& f) {
    const size_t m0p = (static_cast<size_t>(f.m0) + 7) / 8 * 8;
    return static_cast<size_t>(f.n) * (1 + f.nb) * m0p * static_cast<size_t>(resfold_ldj(f.J));
}
void launch_resfold(const Launch& L, const ResFold& f, bool reduce, bool mirror, const char* name);
void launch_fgemm(const Launch& L, int m0, int Rtot, const DirPlan& d, const double* P, const double* Qf, double* T);
void launch_kr_combine(const Launch& L, const KRArgs& a);

// fill H/S (box dense, periodic generating blocks); mode 0 core (H,S), 1 Laplace, 2 Mass, 3 Nuclear, 5 core H only
struct FillArgs {
    Index m0 = 0, Rtot = 0, L[3]{1, 1, 1}, band[3]{}, width[3]{1, 1, 1};
    const double* massT[3]{};
    const double* stiffT[3]{};
    const double* T[3]{};      // nuclear tables [pair][r][e]
    const double* potw = nullptr;
    const double* N = nullptr; // nuclear blocks: [k][d][e] along s2_dir, or [dlin][e] (nuc_mode 2)
    // periodic nuc_mode 1 without the reduce launch: N[d][e] = sum_t Npart[t][|d|][e or e^T]
    const double* Npart = nullptr;
    Index Nres = 0, Nnd = 0;
    int s2_dir = -1;
    int nuc_mode = 0;          // 0 tables, 1 N along s2_dir, 2 N by dlin
    int mode = 0;
    double kin = 0.5;          // mode 0: H = kin Laplace - Nuclear (0 on the non-leading assembly shards)
    bool periodic = false;
    double* out0 = nullptr;    // H (or single operator)
    double* out1 = nullptr;    // S
    int64_t* kidx = nullptr;   // periodic: [nblk][3]
};
void launch_fill(const Launch& L, const FillArgs& a, Index Nb, Index nblocks);

// block diagonalisation over lattice indices (block_circulant.cpp:82-112, :184-196)
struct DftPlan {
    Index dims[3]{1, 1, 1};
    Index ncomp[3]{1, 1, 1};   // compressed extents
    std::vector<Index> comp[3];  // compressed kidx values per axis (ascending)
};
// separable metadata and the factorized Fourier path (k_sep.cu); vals[t][l][s][e]
struct SepBuild {
    int kind = 0;  // 0 Laplace, 1 Mass, 2 Nuclear
    Index mm = 0, S = 0, R = 0;
    Index nslot[3]{1, 1, 1};
    const double* mass[3]{};
    const double* stiff[3]{};
    const double* T[3]{};  // nuclear per-pair tables [slot][R][mm]
    const double* potw = nullptr;
    double* out = nullptr;
};
void launch_sep_from_tables(const Launch& L, const SepBuild& b, Index terms);
struct SepCopy {
    Index mm = 0, Ssrc = 0, Sdst = 0, t0 = 0;
    Index nslot[3]{1, 1, 1};
    const Index* map[3]{};  // device: source slot -> destination slot
    double w = 1.0;
    const double* src = nullptr;
    double* dst = nullptr;
};
void launch_sep_scale_copy(const Launch& L, const SepCopy& c, Index terms);
struct SepDft {
    Index mm = 0, S = 0, Lmax = 1;
    Index L[3]{1, 1, 1};
    Index nslot[3]{1, 1, 1};
    const Index* kid[3]{};  // device: lattice index of each slot
    const double* vals = nullptr;
    double2* out = nullptr;  // [t][l][Lmax][mm]
};
void launch_sep_dft(const Launch& L, const SepDft& d, Index terms);
struct SepBlocks {
    Index mm = 0, terms = 0, Lmax = 1;
    Index L[3]{1, 1, 1};
    const double2* X = nullptr;
    double2* out = nullptr;  // [K][mm]
};
void launch_sep_blocks(const Launch& L, const SepBlocks& b);
struct SepResid {
    Index mm = 0, terms = 0, S = 0;
    Index L[3]{1, 1, 1};
    const int* slot_of[3]{};  // device: lattice index -> slot (-1 none)
    const int* gen_of = nullptr;  // device: lattice index -> stored generating block (-1 none)
    const double* vals = nullptr;
    const double* gen = nullptr;
    unsigned long long* out = nullptr;
};
void launch_sep_residual(const Launch& L, const SepResid& r);

struct CircDefect {
    Index Nb = 0, m0 = 0;
    Index L[3]{1, 1, 1};
    const double* box = nullptr;  // dense Nb x Nb, column-major
    const double* gen = nullptr;  // periodic generating blocks [stored][m0*m0]
    const int* gen_of = nullptr;  // lattice index -> stored block (-1 none)
    double* defect = nullptr;     // optional output
    double* partial = nullptr;    // [blocks][2]: sum defect^2, sum box^2
};
void launch_circ_defect(const Launch& L, const CircDefect& d, int blocks);

// fused per-axis DFT for one or two operators (k_spectrum.cu)
struct DftAxisArgs {
    int axis = 0;
    Index in[3]{1, 1, 1}, out[3]{1, 1, 1};
    Index mm = 0, ncomp = 0, Lax = 1;
    const int64_t* comp = nullptr;                 // compressed indices along the axis
    const double* gen[2] = {nullptr, nullptr};     // first axis: real generating blocks
    const int* slot2blk = nullptr;                 // first axis: compressed position -> block (-1: none)
    const double2* in_buf[2] = {nullptr, nullptr};  // later axes: complex input
    double2* out_buf[2] = {nullptr, nullptr};
};
void launch_dft_axis2(const Launch& L, const DftAxisArgs& a, int nops);
// all wrapped axes in one launch (k_spectrum.cu): CTA per (entry, operator), the entry's
// cube in shared memory (two buffers of maxsz complex + twiddles; dft_fused_smem bytes)
struct DftFusedArgs {
    Index dims[3]{1, 1, 1}, ext[3]{1, 1, 1}, ncomp[3]{1, 1, 1};
    Index mm = 0, maxsz = 0;
    int nax = 0, axes[3]{0, 0, 0};
    const int64_t* comp[3]{nullptr, nullptr, nullptr};
    const int* slot2blk = nullptr;
    const double* gen[2] = {nullptr, nullptr};
    double2* out[2] = {nullptr, nullptr};
    int emajor = 0;     // 1: out [mm][K] (entry-major, for the one-thread-per-pencil kernel)
    int gen_emajor = 0;  // 1: gen [mm][nblocks] (entry-major generating blocks, k_kr_combine's fused fill)
    Index nblocks = 0;
    int ident = 0;  // 1: slot2blk is the identity (every cube position stored, in order): no index loads
};
// log2 L for the register FFT of power-of-two axes 2 <= L <= 16 (0: DFT pass); LT_DFT_NO_FFT
// at compile time forces the DFT pass
__host__ __device__ inline int dft_fft_log(Index L) {
#ifdef LT_DFT_NO_FFT
    (void)L;
    return 0;
#else
    for (int lg = 1; lg <= 4; ++lg)
        if (L == (Index(1) << lg)) return lg;
    return 0;
#endif
}
size_t dft_fused_smem(const DftFusedArgs& a);
void launch_dft_fused(const Launch& L, const DftFusedArgs& a, int nops);
// TMA-fed DMMA GEMM (k_dgemm.cu): C(m, n) = [C +] alpha sum_k A(m, k) B(n, k), operands
// K-major rows of row-major 2D tensors (see the kernel header)
enum DgemmFlags : int {
    DG_LOWER = 1,        // tiles entirely above the diagonal are skipped (diagonal tiles: n <= m)
    DG_MIRROR = 2,       // also store C(n, m) (symmetric result from its lower triangle)
    DG_K_LE_M = 4,       // per tile: k < m_tile_end (A(m, k) lower triangular)
    DG_K_LE_N = 8,       // k < n_tile_end (B(n, k) lower triangular)
    DG_K_GE_M = 16,      // k >= m_tile_begin
    DG_K_GE_N = 32,      // k >= n_tile_begin
    DG_C0_COLMAJOR = 64, // c0 stored column-major (C[m + n ldc]); else row-major (C[m ldc + n])
    DG_C1_COLMAJOR = 128,
};
struct DgemmOperand {
    const double* base = nullptr;  // row-major tensor: rows x cols, pitch ld (doubles)
    long long rows = 0, cols = 0, ld = 0;
};
struct DgemmArgs {
    int M = 0, N = 0;
    long long K = 0;
    long long a_row0 = 0, a_col0 = 0, b_row0 = 0, b_col0 = 0;
    long long a_zrow = 0, a_zcol = 0, b_zrow = 0, b_zcol = 0;  // per-batch coordinate shifts
    double* c0 = nullptr;
    double* c1 = nullptr;  // optional second output (other layout)
    long long ldc = 0, c_zoff = 0;
    double alpha = 1.0;
    int beta_one = 0;  // 1: C += alpha AB, 0: C = alpha AB
    int flags = 0;
    const unsigned long long* fail = nullptr;  // skip when *fail != ~0 (an earlier stage failed)
};
void launch_dgemm_tn(const Launch& L, const DgemmOperand& A, const DgemmOperand& B, const DgemmArgs& args, int batches,
                     const char* stage);

// dense box pencil front end (k_dense2.cu): blocked Cholesky S = L L^T (row-major L in
// place of S, Eigen's pivot test; failure -> atomicMin(fail, 2)), L^-1 (row- and
// column-major) by 64 x 64 leaf inverses and recursive doubling, then A = L^-1 H L^-T into H
// (symmetric, both triangles). ld: row pitch of every n x n buffer (multiple of 2).
struct DenseReduceBufs {
    double* S = nullptr;    // in: S (symmetric); out: L row-major (lower)
    double* H = nullptr;    // in: H (symmetric); out: A = L^-1 H L^-T
    double* Li = nullptr;   // out: L^-1 row-major
    double* Lic = nullptr;  // out: L^-1 column-major
    double* W = nullptr;    // scratch n x n
    double* T = nullptr;    // scratch n x n
    unsigned long long* fail = nullptr;
};
void dense_reduce(const Launch& L, int n, long long ld, const DenseReduceBufs& b);
// the two halves: the S side (Cholesky + L^-1; S, Li, Lic, T) and the H side (W, A into H)
void dense_factor(const Launch& L, int n, long long ld, const DenseReduceBufs& b);
void dense_transform(const Launch& L, int n, long long ld, const DenseReduceBufs& b);
// X = L^-T Z (eigenvectors, eigensolver.cpp:31-32): Z, X column-major with pitch ld
void dense_back_transform(const Launch& L, int n, long long ld, const double* Lic, const double* Z, double* X,
                          const unsigned long long* fail);

// dense box pencil (k_dense.cu): CTAs of the shared-memory resident tridiagonalisation (0:
// too large), the reduction itself (work: 4 n doubles, bar: one zeroed counter), the
// tridiagonal eigenvalues and the in-place symmetrisation 0.5 (A + A^T)
int sytrd_ctas(int n);
void launch_sytrd(const Launch& L, int n, const double* C, double* d, double* e, double* work, unsigned* bar);
void launch_tridiag_eig(const Launch& L, int n, const double* d, const double* e, double* eig);
// full-space eigenvector columns [c0, c0 + ncols) from the per-k blocks u (K m0 x m0 complex)
void launch_reconstruct(const Launch& L, const Index* dims, Index m0, const double2* u, Index c0, Index ncols,
                        double2* out);

// batched Hermitian-definite pencils (eigensolver.cpp:72-93)
// fused lattice DFT in the pencil load stage (single wrapped axis): generating blocks
// GH/GS [nblocks][m0^2] (real), stored offsets comp[c] (ascending kidx) -> block blk[c]
constexpr int kPencilDftMax = 64;
struct PencilDft {
    int nc = 0;  // 0: H, S are the Fourier blocks already
    Index L = 1, k0 = 0;
    const int64_t* comp = nullptr;
    const int* blk = nullptr;
    const double* GH = nullptr;
    const double* GS = nullptr;
};
// real dense pencil read directly from column-major double arrays through the fused-DFT load
PencilDft pencil_identity_source(const double* H, const double* S);
// In-kernel read-back: the last pencil group to finish copies the 8-int result block
// (L0 state, failure key) to pinned host memory, replacing a device-to-host copy node at
// the end of the graph; `done` is a zeroed counter the kernel resets itself.
struct PencilReadback {
    const int* ret_dev = nullptr;
    int* ret_host = nullptr;
    unsigned* done = nullptr;
};
void launch_pencil(const Launch& L, Index count, Index m0, const double2* H, const double2* S, double* eig,
                   unsigned long long* fail_key, bool periodic_checks, const PencilDft& dft = PencilDft{},
                   double2* vec = nullptr,  // vec: K m0 x m0 complex eigenvector blocks (vector mode)
                   const PencilReadback& rb = PencilReadback{}, bool real = false);

// one thread per 8 x 8 pencil (k_pencil_lane.cu): blocks at H[k ks + e es], e = r + c m0
bool pencil_lane_supported(Index m0);
size_t pencil_lane_smem();
constexpr Index kPencilLaneMin = 256;  // lattices below: the group-per-pencil kernel (DFT fused into its load)
void launch_pencil_lane(const Launch& L, Index count, Index m0, const double2* H, const double2* S, Index ks, Index es,
                        double* eig, unsigned long long* fail_key, const PencilReadback& rb = PencilReadback{});

// combine (eigensolver.cpp:37-67) on device buffers with index maps
void launch_axpby_map(const Launch& L, Index nout, Index mm, double wa, const double* a, const int64_t* ia, double wb,
                      const double* b, const int64_t* ib, double* out);

}  // namespace lt
