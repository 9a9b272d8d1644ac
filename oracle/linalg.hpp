// oracle/linalg.hpp — TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// Self-contained dense linear algebra for the CPU oracle and for the Eigen-subset
// shim that compiles the reference sources in place (oracle/eigen_shim). The
// reference delegates these steps to Eigen3 (version unpinned, ">= 3.3",
// /root/reference/proj/core/CMakeLists.txt:1), which is absent from this image:
//
//   * LLT (Cholesky, lower)           — eigensolver.cpp:20, :80 (Eigen::LLT)
//   * SelfAdjointEigenSolver          — eigensolver.cpp:27, :86 (values ascending)
//   * Eigen::FFT<double>::fwd         — block_circulant.cpp:83-112 (kissfft backend;
//                                       unnormalised forward, omega = exp(-2 pi i/L))
//
// The restatements follow the published algorithms: column Cholesky with the
// Eigen pivot test `x <= 0` on the real part of the diagonal; cyclic two-sided
// Jacobi for complex Hermitian matrices; Householder tridiagonalisation followed
// by implicit QL with Wilkinson shifts for large real symmetric matrices; an
// iterative radix-2 FFT (powers of two) or a direct DFT (other lengths).
// Results agree with Eigen to round-off (eigenvalues to ~1e-15 relative), which is
// far inside the north-star tolerance (eigenvalues within 1e-9 absolute).
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <numbers>
#include <vector>

namespace orla {

using Index = std::int64_t;
using Cplx = std::complex<double>;

// ---------------------------------------------------------------------------
// Cholesky: A (n x n, column-major, only the lower triangle is read) -> L in
// place (lower). Returns false on a non-positive pivot, like Eigen's LLT.
// ---------------------------------------------------------------------------
template <class T>
inline double real_part(const T& v) { return std::real(v); }

template <class T>
inline T conj_of(const T& v) {
    if constexpr (std::is_same_v<T, double>) return v;
    else return std::conj(v);
}

// Right-looking, column-oriented (contiguous column updates); the pivot x is the
// Schur-complement diagonal, tested like Eigen's llt_inplace (x <= 0 fails).
template <class T>
bool cholesky_lower(Index n, T* a) {
    auto A = [&](Index i, Index j) -> T& { return a[i + j * n]; };
    for (Index k = 0; k < n; ++k) {
        const double x = real_part(A(k, k));
        if (!(x > 0.0)) return false;
        const double dkk = std::sqrt(x);
        A(k, k) = T(dkk);
        const double inv = 1.0 / dkk;
        T* ck = &A(0, k);
        for (Index i = k + 1; i < n; ++i) ck[i] *= inv;
        for (Index j = k + 1; j < n; ++j) {
            const T f = conj_of(ck[j]);
            T* cj = &A(0, j);
            for (Index i = j; i < n; ++i) cj[i] -= ck[i] * f;
        }
        for (Index j = k + 1; j < n; ++j) A(k, j) = T(0);
    }
    return true;
}

// Solve L X = B in place (B: n x m column-major), L lower from cholesky_lower
// (column-oriented forward substitution).
template <class T>
void lower_solve(Index n, const T* l, Index m, T* b) {
    for (Index c = 0; c < m; ++c) {
        T* x = b + c * n;
        for (Index j = 0; j < n; ++j) {
            x[j] /= l[j + j * n];
            const T xj = x[j];
            const T* lj = l + j * n;
            for (Index i = j + 1; i < n; ++i) x[i] -= lj[i] * xj;
        }
    }
}

// Reduce the pencil (H, S) to standard form A = L^{-1} H L^{-H} where S = L L^H,
// following eigensolver.cpp:79-80 / :138-139: Y = L^{-1} H, A = (L^{-1} Y^H)^H.
// Returns false if S is not positive definite. H and S are n x n column-major;
// both are read in full. Output A is n x n (not yet symmetrised).
template <class T>
bool reduce_pencil(Index n, const T* h, const T* s, std::vector<T>& a_out) {
    std::vector<T> l(s, s + n * n);
    if (!cholesky_lower(n, l.data())) return false;
    std::vector<T> y(h, h + n * n);
    lower_solve(n, l.data(), n, y.data());
    std::vector<T> yh(n * n);
    for (Index i = 0; i < n; ++i)
        for (Index j = 0; j < n; ++j) yh[j + i * n] = conj_of(y[i + j * n]);
    lower_solve(n, l.data(), n, yh.data());
    a_out.assign(n * n, T(0));
    for (Index i = 0; i < n; ++i)
        for (Index j = 0; j < n; ++j) a_out[j + i * n] = conj_of(yh[i + j * n]);
    return true;
}

// ---------------------------------------------------------------------------
// Cyclic two-sided Jacobi for a Hermitian (or real symmetric) matrix;
// eigenvalues ascending. a is overwritten.
// ---------------------------------------------------------------------------
// Rotation rule (Demmel-Veselic threshold with an absolute floor): rotate (p,q) iff
// |a_pq| > max(2^-53 sqrt(|a_pp a_qq|), 1e-17 ||A||_F); converged after a sweep with
// no rotation. Left-over off-diagonal entries move eigenvalues by O(eps ||A||).
template <class T>
void jacobi_eigenvalues(Index n, T* a, double* w) {
    auto A = [&](Index i, Index j) -> T& { return a[i + j * n]; };
    double fro = 0.0;
    for (Index k = 0; k < n * n; ++k) fro += std::norm(a[k]);
    const double floor_abs = 1e-17 * std::sqrt(fro);
    for (int sweep = 0; sweep < 60; ++sweep) {
        bool rotated = false;
        for (Index p = 0; p < n - 1; ++p) {
            for (Index q = p + 1; q < n; ++q) {
                const T apq = A(p, q);
                const double r = std::abs(apq);
                const double app = real_part(A(p, p)), aqq = real_part(A(q, q));
                if (!(r > floor_abs) || r <= 1.1102230246251565e-16 * std::sqrt(std::abs(app * aqq))) continue;
                rotated = true;
                // make a_pq real: column q *= conj(phase), row q *= phase
                T ph = apq / r;  // e^{i phi}
                if constexpr (!std::is_same_v<T, double>) {
                    const T cph = std::conj(ph);
                    for (Index k = 0; k < n; ++k) A(k, q) *= cph;
                    for (Index k = 0; k < n; ++k) A(q, k) *= ph;
                } else {
                    if (ph < 0) {
                        for (Index k = 0; k < n; ++k) A(k, q) = -A(k, q);
                        for (Index k = 0; k < n; ++k) A(q, k) = -A(q, k);
                    }
                }
                const double tau = (aqq - app) / (2.0 * r);
                const double t = (tau >= 0 ? 1.0 : -1.0) / (std::abs(tau) + std::sqrt(1.0 + tau * tau));
                const double c = 1.0 / std::sqrt(1.0 + t * t);
                const double s = t * c;
                for (Index k = 0; k < n; ++k) {  // columns: A J
                    const T akp = A(k, p), akq = A(k, q);
                    A(k, p) = c * akp - s * akq;
                    A(k, q) = s * akp + c * akq;
                }
                for (Index k = 0; k < n; ++k) {  // rows: J^T (A J)
                    const T apk = A(p, k), aqk = A(q, k);
                    A(p, k) = c * apk - s * aqk;
                    A(q, k) = s * apk + c * aqk;
                }
                A(p, q) = T(0);
                A(q, p) = T(0);
                A(p, p) = T(app - t * r);
                A(q, q) = T(aqq + t * r);
            }
        }
        if (!rotated) break;
    }
    for (Index i = 0; i < n; ++i) w[i] = real_part(A(i, i));
    std::sort(w, w + n);
}

// ---------------------------------------------------------------------------
// Real symmetric eigenvalues via Householder tridiagonalisation + implicit QL
// (O(n^3), used for the large dense box pencil). a (n x n, column-major) is
// overwritten; only symmetric input is meaningful.
// ---------------------------------------------------------------------------
inline void symmetric_eigenvalues(Index n, double* a, double* w) {
    if (n <= 0) return;
    if (n <= 48) { jacobi_eigenvalues<double>(n, a, w); return; }
    // symmetric input: address the transposed storage so the row sweeps of the
    // (row-oriented) Householder scheme run over contiguous memory
    auto A = [&](Index i, Index j) -> double& { return a[j + i * n]; };
    std::vector<double> d(n), e(n, 0.0);
    // Householder: annihilate row i left of the subdiagonal, i = n-1 .. 1
    for (Index i = n - 1; i > 0; --i) {
        const Index l = i - 1;
        double scale = 0.0, h = 0.0;
        for (Index k = 0; k <= l; ++k) scale += std::abs(A(i, k));
        if (l == 0 || scale == 0.0) {
            e[i] = A(i, l);
            d[i] = 0.0;
            continue;
        }
        for (Index k = 0; k <= l; ++k) {
            A(i, k) /= scale;
            h += A(i, k) * A(i, k);
        }
        const double f = A(i, l);
        const double g = f >= 0.0 ? -std::sqrt(h) : std::sqrt(h);
        e[i] = scale * g;
        h -= f * g;
        A(i, l) = f - g;
        // p = A u / h, stored in e[0..l]
        double kdot = 0.0;
        for (Index j = 0; j <= l; ++j) {
            double s = 0.0;
            for (Index k = 0; k <= j; ++k) s += A(j, k) * A(i, k);
            for (Index k = j + 1; k <= l; ++k) s += A(k, j) * A(i, k);
            e[j] = s / h;
            kdot += e[j] * A(i, j);
        }
        const double hh = kdot / (h + h);
        for (Index j = 0; j <= l; ++j) {
            const double fj = A(i, j);
            const double gj = e[j] - hh * fj;
            e[j] = gj;
            for (Index k = 0; k <= j; ++k) A(j, k) -= (fj * e[k] + gj * A(i, k));
        }
        d[i] = h;
    }
    for (Index i = 0; i < n; ++i) d[i] = A(i, i);
    // implicit QL with Wilkinson shifts on (d, e); e[i] couples i-1 and i
    for (Index i = 1; i < n; ++i) e[i - 1] = e[i];
    e[n - 1] = 0.0;
    for (Index l = 0; l < n; ++l) {
        int iter = 0;
        while (true) {
            Index m = l;
            for (; m < n - 1; ++m) {
                const double dd = std::abs(d[m]) + std::abs(d[m + 1]);
                if (std::abs(e[m]) <= 2.220446049250313e-16 * dd) break;
            }
            if (m == l) break;
            if (++iter > 200) break;
            double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
            double r = std::hypot(g, 1.0);
            g = d[m] - d[l] + e[l] / (g + (g >= 0.0 ? r : -r));
            double s = 1.0, c = 1.0, p = 0.0;
            bool underflow = false;
            for (Index i = m - 1; i >= l; --i) {
                double f = s * e[i];
                const double bb = c * e[i];
                r = std::hypot(f, g);
                e[i + 1] = r;
                if (r == 0.0) {
                    d[i + 1] -= p;
                    e[m] = 0.0;
                    underflow = true;
                    break;
                }
                s = f / r;
                c = g / r;
                g = d[i + 1] - p;
                r = (d[i] - g) * s + 2.0 * c * bb;
                p = s * r;
                d[i + 1] = g + p;
                g = c * r - bb;
            }
            if (underflow) continue;
            d[l] -= p;
            e[l] = g;
            e[m] = 0.0;
        }
    }
    for (Index i = 0; i < n; ++i) w[i] = d[i];
    std::sort(w, w + n);
}

// ---------------------------------------------------------------------------
// Unnormalised forward DFT, omega = exp(-2 pi i / L) (block_circulant.cpp:80-112,
// PAPER.md:1346). Radix-2 for powers of two, direct sum otherwise.
// ---------------------------------------------------------------------------
inline Cplx twiddle(Index jk, Index L) {
    const Index r = jk % L;
    const double ang = -2.0 * std::numbers::pi * static_cast<double>(r) / static_cast<double>(L);
    return Cplx(std::cos(ang), std::sin(ang));
}

inline void fft_forward(std::vector<Cplx>& x) {
    const Index L = static_cast<Index>(x.size());
    if (L <= 1) return;
    if ((L & (L - 1)) != 0) {
        std::vector<Cplx> out(L);
        for (Index j = 0; j < L; ++j) {
            Cplx s(0.0, 0.0);
            for (Index k = 0; k < L; ++k) s += x[k] * twiddle(j * k, L);
            out[j] = s;
        }
        x.swap(out);
        return;
    }
    // bit reversal
    for (Index i = 1, j = 0; i < L; ++i) {
        Index bit = L >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) std::swap(x[i], x[j]);
    }
    for (Index len = 2; len <= L; len <<= 1) {
        const Index half = len / 2;
        for (Index i = 0; i < L; i += len)
            for (Index k = 0; k < half; ++k) {
                const Cplx w = twiddle(k * (L / len), L);
                const Cplx u = x[i + k], v = x[i + k + half] * w;
                x[i + k] = u + v;
                x[i + k + half] = u - v;
            }
    }
}

}  // namespace orla
