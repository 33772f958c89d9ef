// Host fp64 small dense linear algebra of libtpo (d x d, b x b, k x k matrices only).
//   * QR by classical Gram-Schmidt with one re-orthogonalisation pass (CGS2): R has a
//     positive diagonal by construction, which is the sign convention of the Haar
//     rotation (Alg. 1 L7; unique QR with diag(R) > 0).
//   * Symmetric eigensolver: Householder tridiagonalisation + implicit-shift QL with
//     eigenvector accumulation (EISPACK tred2/tql2 scheme), used for the Rayleigh-Ritz
//     matrices of the subspace iteration (b x b) and for D x D when b = D.
//   * Cholesky (upper) and triangular inverse for CholeskyQR2.
#include <math.h>
#include <string.h>

#include <algorithm>
#include <numeric>
#include <vector>

#include "tpo_internal.cuh"

namespace tpo {

void host_qr_positive(int64_t rows, int64_t cols, const double *A, double *Q, double *R) {
    // Q (rows x cols) row-major; columns built one by one.
    std::vector<double> q((size_t)rows * cols, 0.0), r((size_t)cols * cols, 0.0), v(rows);
    for (int64_t j = 0; j < cols; ++j) {
        for (int64_t i = 0; i < rows; ++i) v[i] = A[i * cols + j];
        for (int pass = 0; pass < 2; ++pass) {
            std::vector<double> c(j, 0.0);
            for (int64_t p = 0; p < j; ++p) {
                double s = 0.0;
                for (int64_t i = 0; i < rows; ++i) s += q[i * cols + p] * v[i];
                c[p] = s;
            }
            for (int64_t p = 0; p < j; ++p) {
                for (int64_t i = 0; i < rows; ++i) v[i] -= c[p] * q[i * cols + p];
                r[p * cols + j] += c[p];
            }
        }
        double nr = 0.0;
        for (int64_t i = 0; i < rows; ++i) nr += v[i] * v[i];
        nr = sqrt(nr);
        if (!(nr > 0.0)) throw Error(TPO_ENUMERIC, "QR: rank-deficient input");
        r[j * cols + j] = nr;
        for (int64_t i = 0; i < rows; ++i) q[i * cols + j] = v[i] / nr;
    }
    memcpy(Q, q.data(), sizeof(double) * q.size());
    if (R) memcpy(R, r.data(), sizeof(double) * r.size());
}

namespace {

// Householder tridiagonalisation of symmetric a (n x n, row-major, full storage): T = Q^T A Q
// with Q = H_0 H_1 ... H_{n-3}, H_k = I - beta_k v_k v_k^T acting on rows / columns k+1 .. n-1.
// d = diag(T), e[i] couples i-1 and i (e[0] = 0); zt = Q^T (row i of zt = column i of Q), the
// transposed start of the QL eigenvector accumulation.  Every inner loop runs over contiguous
// rows (the symmetric rank-2 update keeps the full matrix), so it vectorises and stays in cache.
void tridiagonalise(int n, std::vector<double> &a, std::vector<double> &d, std::vector<double> &e,
                    std::vector<double> &zt) {
    auto A = [&](int i, int j) -> double & { return a[(size_t)i * n + j]; };
    std::vector<double> v(n), p(n), w(n), beta(n, 0.0), V((size_t)n * n, 0.0);   // V row k: v_k
    e[0] = 0.0;
    for (int k = 0; k + 2 < n; ++k) {
        const int m0 = k + 1;
        double *x = &A(k, m0);                         // row k right of the diagonal = column k below it
        double scale = 0.0;
        for (int i = 0; i < n - m0; ++i) scale = std::max(scale, fabs(x[i]));
        d[k] = A(k, k);
        if (scale == 0.0) {
            e[m0] = 0.0;
            continue;
        }
        double sig = 0.0;
        for (int i = 0; i < n - m0; ++i) {
            v[i] = x[i] / scale;
            sig += v[i] * v[i];
        }
        const double nrm = sqrt(sig);
        const double alpha = v[0] >= 0.0 ? -nrm : nrm;       // H x = alpha scale e_0
        v[0] -= alpha;
        const double vtv = sig - 2.0 * alpha * (v[0] + alpha) + alpha * alpha;   // |x/scale - alpha e0|^2
        const double b = 2.0 / vtv;
        e[m0] = alpha * scale;
        beta[k] = b;
        const int m = n - m0;
        // p = b A22 v (rows of A22 contiguous)
        double pv = 0.0;
        for (int i = 0; i < m; ++i) {
            const double *ri = &A(m0 + i, m0);
            double acc = 0.0;
            for (int j = 0; j < m; ++j) acc += ri[j] * v[j];
            p[i] = b * acc;
            pv += p[i] * v[i];
        }
        const double K = 0.5 * b * pv;
        for (int i = 0; i < m; ++i) w[i] = p[i] - K * v[i];
        // A22 -= v w^T + w v^T
        for (int i = 0; i < m; ++i) {
            double *ri = &A(m0 + i, m0);
            const double vi = v[i], wi = w[i];
            for (int j = 0; j < m; ++j) ri[j] -= vi * w[j] + wi * v[j];
        }
        double *vk = &V[(size_t)k * n + m0];
        for (int i = 0; i < m; ++i) vk[i] = v[i];
    }
    if (n >= 2) {
        d[n - 2] = A(n - 2, n - 2);
        e[n - 1] = A(n - 1, n - 2);
    }
    d[n - 1] = A(n - 1, n - 1);
    // zt = Q^T = H_{n-3} ... H_1 H_0: start from I, apply H_0 first (each H_k changes rows k+1..)
    std::fill(zt.begin(), zt.end(), 0.0);
    for (int i = 0; i < n; ++i) zt[(size_t)i * n + i] = 1.0;
    std::vector<double> y(n);
    for (int k = 0; k + 2 < n; ++k) {
        if (beta[k] == 0.0) continue;
        const int m0 = k + 1;
        const double *vk = &V[(size_t)k * n];
        std::fill(y.begin(), y.end(), 0.0);                // y^T = v^T M (rows m0..n-1 of M)
        for (int i = m0; i < n; ++i) {
            const double vi = vk[i];
            const double *mi = &zt[(size_t)i * n];
            for (int j = 0; j < n; ++j) y[j] += vi * mi[j];
        }
        for (int i = m0; i < n; ++i) {
            const double c = beta[k] * vk[i];
            double *mi = &zt[(size_t)i * n];
            for (int j = 0; j < n; ++j) mi[j] -= c * y[j];
        }
    }
}

// sqrt(a^2 + b^2) without libm's hypot (which dominated the QL sweeps: one call per rotation);
// rescaled only when a square could over- or underflow
inline double fast_hypot(double a, double b) {
    const double fa = fabs(a), fb = fabs(b);
    const double m = fa > fb ? fa : fb;
    if (m > 1e150 || (m < 1e-150 && m > 0.0)) return hypot(a, b);
    return sqrt(a * a + b * b);
}

// (zi, zi1) <- (c zi - s zi1, s zi + c zi1): two distinct rows (restrict: vectorised)
inline void rotate_rows(double *__restrict__ zi, double *__restrict__ zi1, int n, double c, double s) {
    for (int k = 0; k < n; ++k) {
        const double f = zi1[k], g = zi[k];
        zi1[k] = s * g + c * f;
        zi[k] = c * g - s * f;
    }
}

// Implicit-shift QL on the tridiagonal (d, e), accumulating rotations into z (n x n, TRANSPOSED:
// z[i * n + k] = component k of vector i).
void tridiag_ql(int n, std::vector<double> &d, std::vector<double> &e, std::vector<double> &z) {
    for (int i = 1; i < n; ++i) e[i - 1] = e[i];
    e[n - 1] = 0.0;
    for (int l = 0; l < n; ++l) {
        int iter = 0, m;
        do {
            for (m = l; m < n - 1; ++m) {
                const double dd = fabs(d[m]) + fabs(d[m + 1]);
                if (fabs(e[m]) <= 1e-300 || fabs(e[m]) + dd == dd) break;
            }
            if (m != l) {
                if (iter++ == 200) throw Error(TPO_ENUMERIC, "tridiagonal QL did not converge");
                double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
                double r = fast_hypot(g, 1.0);
                g = d[m] - d[l] + e[l] / (g + (g >= 0.0 ? fabs(r) : -fabs(r)));
                double s = 1.0, c = 1.0, p = 0.0;
                int i;
                for (i = m - 1; i >= l; --i) {
                    double f = s * e[i];
                    const double b = c * e[i];
                    e[i + 1] = (r = fast_hypot(f, g));
                    if (r == 0.0) {
                        d[i + 1] -= p;
                        e[m] = 0.0;
                        break;
                    }
                    s = f / r;
                    c = g / r;
                    g = d[i + 1] - p;
                    r = (d[i] - g) * s + 2.0 * c * b;
                    d[i + 1] = g + (p = s * r);
                    g = c * r - b;
                    // z is held transposed (row i = eigenvector column i): contiguous rows
                    rotate_rows(&z[(size_t)i * n], &z[(size_t)(i + 1) * n], n, c, s);
                }
                if (r == 0.0 && i >= l) continue;
                d[l] -= p;
                e[l] = g;
                e[m] = 0.0;
            }
        } while (m != l);
    }
}

}  // namespace

void host_sym_eig_top(int64_t D, const double *Ain, int64_t nvec, double *w, double *V) {
    const int n = (int)D;
    std::vector<double> a(Ain, Ain + (size_t)n * n), d(n), e(n);
    // symmetrise defensively (inputs are symmetric up to rounding of the reduction)
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < i; ++j) {
            const double s = 0.5 * (a[(size_t)i * n + j] + a[(size_t)j * n + i]);
            a[(size_t)i * n + j] = a[(size_t)j * n + i] = s;
        }
    if (n == 1) {
        w[0] = a[0];
        if (nvec > 0) V[0] = 1.0;
        return;
    }
    std::vector<double> zt((size_t)n * n);                  // the transform, transposed for tridiag_ql
    tridiagonalise(n, a, d, e, zt);
    tridiag_ql(n, d, e, zt);
    for (int r = 0; r < n; ++r)
        for (int c = 0; c < n; ++c) a[(size_t)r * n + c] = zt[(size_t)c * n + r];
    std::vector<int> ord(n);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return d[x] > d[y]; });
    for (int i = 0; i < n; ++i) w[i] = d[ord[i]];
    for (int64_t c = 0; c < nvec; ++c)
        for (int r = 0; r < n; ++r) V[(size_t)r * nvec + c] = a[(size_t)r * n + ord[c]];
}

bool host_cholesky_upper(int64_t k, const double *A, double *C) {
    for (int64_t i = 0; i < k * k; ++i) C[i] = 0.0;
    for (int64_t j = 0; j < k; ++j) {
        double s = A[j * k + j];
        for (int64_t p = 0; p < j; ++p) s -= C[p * k + j] * C[p * k + j];
        if (!(s > 0.0) || !std::isfinite(s)) return false;
        const double cjj = sqrt(s);
        C[j * k + j] = cjj;
        for (int64_t i = j + 1; i < k; ++i) {
            double t = A[j * k + i];
            for (int64_t p = 0; p < j; ++p) t -= C[p * k + j] * C[p * k + i];
            C[j * k + i] = t / cjj;
        }
    }
    return true;
}

void host_upper_inverse(int64_t k, const double *C, double *Ci) {
    for (int64_t i = 0; i < k * k; ++i) Ci[i] = 0.0;
    for (int64_t j = 0; j < k; ++j) {
        Ci[j * k + j] = 1.0 / C[j * k + j];
        for (int64_t i = j - 1; i >= 0; --i) {
            double s = 0.0;
            for (int64_t p = i + 1; p <= j; ++p) s += C[i * k + p] * Ci[p * k + j];
            Ci[i * k + j] = -s / C[i * k + i];
        }
    }
}

}  // namespace tpo
