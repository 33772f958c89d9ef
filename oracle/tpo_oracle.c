/*
 * tpo_oracle.c -- plain, slow, fp64 CPU oracle of the TPO hot path (arXiv 2405.11922).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or helper with the CUDA library under paper_2405_11922_b200/csrc/.
 *
 * Every function follows the paper's definition or algorithm in the paper's order,
 * in fp64, on fp32 inputs widened to double.  OpenMP loops only split independent
 * outputs across threads: every sum is accumulated by one thread in its serial order,
 * so the results do not depend on the thread count.  Citations are PAPER.md line numbers
 * (LaTeX source) plus the equation / algorithm label.  Readings of silent or garbled
 * passages are the ones listed in DESIGN.md "Readings" (R1..R12).
 *
 * Parity status: every function here is pinned by tests/test_oracle_pins.py except
 * where a header comment says "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EPS_ONMF 1e-12      /* R9: epsilon in the ONMF denominators */
#define FLOOR_DINV 1e-12    /* R6: floor before the square root of Eq. Ri */

static double *dalloc(size_t cnt) { return (double *)calloc(cnt ? cnt : 1, sizeof(double)); }

/* ------------------------------------------------------------------------------------
 * a1: degrees.  D_U[i] = sum of weights of edges incident to u_i, same for V
 * (PAPER.md:173).  1/sqrt(0) := 0 for isolated nodes (R3).
 * ------------------------------------------------------------------------------------ */
void oracle_degree_scales(int64_t n, int64_t m, const int64_t *rowptr, const int32_t *col,
                          const float *val, double *s_u, double *s_v) {
    double *dv = dalloc((size_t)m);
    for (int64_t u = 0; u < n; ++u) {
        double du = 0.0;
        for (int64_t e = rowptr[u]; e < rowptr[u + 1]; ++e) {
            double w = val ? (double)val[e] : 1.0;
            du += w;
            dv[col[e]] += w;
        }
        s_u[u] = du > 0.0 ? 1.0 / sqrt(du) : 0.0;
    }
    for (int64_t v = 0; v < m; ++v) s_v[v] = dv[v] > 0.0 ? 1.0 / sqrt(dv[v]) : 0.0;
    free(dv);
}

/* ------------------------------------------------------------------------------------
 * a1-a3: MSA propagation, Lemma 1 / Eq. PX truncated at gamma = T,
 * with L = D_U^{-1/2} B D_V^{-1/2} (Eq. L), evaluated by the hop
 * update of Eq. update-Z bracketed as L (L^T Z):
 *      Z_0 = c X,   Z <- c X + alpha * L (L^T Z)   (T times),
 * c = (1 - alpha) (R1: Lemma 1's prefactor; c = 1 at alpha = 1, the Alg. 1 limit).
 * Then Zhat = row-L2-normalised Z (Eq. Z), zero rows stay zero (R4).
 * Only CSR(B) is used: for L^T Z the oracle builds its own transposed edge list of B by a
 * stable counting sort (each v's incident edges in ascending u order) and sums
 * Y[v] = sum_u L[u,v] Z[u] in that order -- the order a serial scatter over B's rows adds
 * them in -- so it never reads the caller's CSR(B^T).
 * Z, Zhat: n x d row-major doubles (Zhat may be NULL).
 * ------------------------------------------------------------------------------------ */
void oracle_propagate(int64_t n, int64_t m, const int64_t *rowptr, const int32_t *col,
                      const float *val, const float *X, int64_t d, double alpha, int32_t T,
                      double *Z, double *Zhat) {
    double *s_u = dalloc((size_t)n), *s_v = dalloc((size_t)m);
    oracle_degree_scales(n, m, rowptr, col, val, s_u, s_v);
    const double c = (alpha < 1.0) ? (1.0 - alpha) : 1.0;
    for (int64_t i = 0; i < n * d; ++i) Z[i] = c * (double)X[i];
    /* transposed edge list: for each v, (u, L[u,v]) in ascending u */
    const int64_t E = rowptr[n];
    int64_t *tptr = (int64_t *)calloc((size_t)(m + 1), sizeof(int64_t));
    int64_t *tu = (int64_t *)malloc(sizeof(int64_t) * (size_t)(E ? E : 1));
    double *tL = dalloc((size_t)E);
    for (int64_t e = 0; e < E; ++e) tptr[col[e] + 1]++;
    for (int64_t v = 0; v < m; ++v) tptr[v + 1] += tptr[v];
    {
        int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(m ? m : 1));
        for (int64_t v = 0; v < m; ++v) fill[v] = tptr[v];
        for (int64_t u = 0; u < n; ++u)
            for (int64_t e = rowptr[u]; e < rowptr[u + 1]; ++e) {
                const int64_t v = col[e];
                tu[fill[v]] = u;
                tL[fill[v]] = (val ? (double)val[e] : 1.0) * s_u[u] * s_v[v];
                fill[v]++;
            }
        free(fill);
    }
    double *Y = dalloc((size_t)(m * d));
    for (int32_t t = 0; t < T; ++t) {
        /* Y = L^T Z :  Y[v] = sum_u L[u,v] * Z[u] */
#pragma omp parallel for schedule(static)
        for (int64_t v = 0; v < m; ++v) {
            double *yv = Y + v * d;
            for (int64_t j = 0; j < d; ++j) yv[j] = 0.0;
            for (int64_t q = tptr[v]; q < tptr[v + 1]; ++q) {
                const double L = tL[q];
                const double *zu = Z + tu[q] * d;
                for (int64_t j = 0; j < d; ++j) yv[j] += L * zu[j];
            }
        }
        /* Z = c X + alpha * L Y */
#pragma omp parallel for schedule(static)
        for (int64_t u = 0; u < n; ++u) {
            double *zu = Z + u * d;
            for (int64_t j = 0; j < d; ++j) zu[j] = 0.0;
            for (int64_t e = rowptr[u]; e < rowptr[u + 1]; ++e) {
                const int64_t v = col[e];
                const double L = (val ? (double)val[e] : 1.0) * s_u[u] * s_v[v];
                const double *yv = Y + v * d;
                for (int64_t j = 0; j < d; ++j) zu[j] += L * yv[j];
            }
            for (int64_t j = 0; j < d; ++j) zu[j] = c * (double)X[u * d + j] + alpha * zu[j];
        }
    }
    free(tptr); free(tu); free(tL);
    if (Zhat) {
        for (int64_t u = 0; u < n; ++u) {
            double s = 0.0;
            for (int64_t j = 0; j < d; ++j) s += Z[u * d + j] * Z[u * d + j];
            const double nr = sqrt(s);
            for (int64_t j = 0; j < d; ++j) Zhat[u * d + j] = nr > 0.0 ? Z[u * d + j] / nr : 0.0;
        }
    }
    free(Y); free(s_u); free(s_v);
}

/* ------------------------------------------------------------------------------------
 * Householder QR of a rows x cols (rows >= cols) row-major matrix A (overwritten).
 * Returns the thin Q (rows x cols) with the sign convention diag(R) > 0 (R8-style:
 * Q <- Q diag(sign(diag R))), and R (cols x cols) if R != NULL.
 * ------------------------------------------------------------------------------------ */
static void householder_qr(int64_t rows, int64_t cols, double *A, double *Q, double *R) {
    double *V = dalloc((size_t)(rows * cols));      /* Householder vectors, column j in V[:, j] */
    double *rdiag = dalloc((size_t)cols);
    for (int64_t j = 0; j < cols; ++j) {
        double nrm = 0.0;
        for (int64_t i = j; i < rows; ++i) nrm += A[i * cols + j] * A[i * cols + j];
        nrm = sqrt(nrm);
        const double x0 = A[j * cols + j];
        const double a = (x0 >= 0.0) ? -nrm : nrm;      /* R[j,j] = a */
        rdiag[j] = a;
        double vn = 0.0;
        for (int64_t i = j; i < rows; ++i) {
            const double vi = A[i * cols + j] - (i == j ? a : 0.0);
            V[i * cols + j] = vi;
            vn += vi * vi;
        }
        if (vn > 0.0) {
            const double inv = 1.0 / sqrt(vn);
            for (int64_t i = j; i < rows; ++i) V[i * cols + j] *= inv;
#pragma omp parallel for schedule(static)
            for (int64_t c2 = j; c2 < cols; ++c2) {           /* A[j:, j:] <- (I - 2 v v^T) A */
                double s = 0.0;
                for (int64_t i = j; i < rows; ++i) s += V[i * cols + j] * A[i * cols + c2];
                for (int64_t i = j; i < rows; ++i) A[i * cols + c2] -= 2.0 * V[i * cols + j] * s;
            }
        }
    }
    if (R) {
        for (int64_t i = 0; i < cols; ++i)
            for (int64_t j = 0; j < cols; ++j) R[i * cols + j] = (j >= i) ? A[i * cols + j] : 0.0;
        for (int64_t i = 0; i < cols; ++i) R[i * cols + i] = rdiag[i];
    }
    /* Q = H_0 H_1 ... H_{cols-1} [I; 0] : apply reflectors in reverse order */
    for (int64_t i = 0; i < rows; ++i)
        for (int64_t j = 0; j < cols; ++j) Q[i * cols + j] = (i == j) ? 1.0 : 0.0;
    for (int64_t j = cols - 1; j >= 0; --j)
#pragma omp parallel for schedule(static)
        for (int64_t c2 = 0; c2 < cols; ++c2) {
            double s = 0.0;
            for (int64_t i = j; i < rows; ++i) s += V[i * cols + j] * Q[i * cols + c2];
            for (int64_t i = j; i < rows; ++i) Q[i * cols + c2] -= 2.0 * V[i * cols + j] * s;
        }
    /* sign fix: make diag(R) positive */
    for (int64_t j = 0; j < cols; ++j)
        if (rdiag[j] < 0.0) {
            for (int64_t i = 0; i < rows; ++i) Q[i * cols + j] = -Q[i * cols + j];
            if (R) for (int64_t c2 = 0; c2 < cols; ++c2) R[j * cols + c2] = -R[j * cols + c2];
        }
    free(V); free(rdiag);
}

/* a4: Alg. 1 L6-7: Q from the QR decomposition of the Gaussian G,
 * sign-fixed so that diag(R) > 0 (Haar-distributed). */
void oracle_haar_q(int64_t d, const double *G, double *Q) {
    double *A = dalloc((size_t)(d * d));
    memcpy(A, G, sizeof(double) * (size_t)(d * d));
    householder_qr(d, d, A, Q, NULL);
    free(A);
}

/* generic thin QR exported for tests (orthonormal basis, diag(R) > 0) */
void oracle_qr(int64_t rows, int64_t cols, const double *A_in, double *Q, double *R) {
    double *A = dalloc((size_t)(rows * cols));
    memcpy(A, A_in, sizeof(double) * (size_t)(rows * cols));
    householder_qr(rows, cols, A, Q, R);
    free(A);
}

/* ------------------------------------------------------------------------------------
 * a5: random features, Eq. R-prime and Eq. Ri:
 *   Zo = sqrt(d) * Zhat * Q^T ;  R' = sqrt(e/d) * ( sin(Zo) || cos(Zo) )   (n x 2d)
 *   r  = sum_l R'[l] ;  dinv_i = 1 / sqrt(max(R'[i] . r, 1e-12))           (R6)
 * so that R = diag(dinv) R'.  e = exp(1).  Rp: n x 2d doubles; dinv: n; r: 2d.
 * ------------------------------------------------------------------------------------ */
void oracle_features(int64_t n, int64_t d, const float *Zhat, const float *Q, double *Rp,
                     double *dinv, double *r) {
    const double sd = sqrt((double)d), amp = sqrt(exp(1.0) / (double)d);
    const int64_t D = 2 * d;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t j = 0; j < d; ++j) {
            double s = 0.0;
            for (int64_t l = 0; l < d; ++l) s += (double)Zhat[i * d + l] * (double)Q[j * d + l];
            const double zo = sd * s;
            Rp[i * D + j] = amp * sin(zo);
            Rp[i * D + d + j] = amp * cos(zo);
        }
    }
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < D; ++j) {
        double rj = 0.0;
        for (int64_t i = 0; i < n; ++i) rj += Rp[i * D + j];
        r[j] = rj;
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double t = 0.0;
        for (int64_t j = 0; j < D; ++j) t += Rp[i * D + j] * r[j];
        dinv[i] = 1.0 / sqrt(t > FLOOR_DINV ? t : FLOOR_DINV);
    }
}

/* ------------------------------------------------------------------------------------
 * a6: implicit affinity product  out = R (R^T Y) = dinv . R'( R'^T (dinv . Y) )
 * (R R^T approximates S, Theorem 1; the n x n matrix is never formed,
 * PAPER.md:564).  Inputs fp32 R' (n x D), dinv (n); Y, out: n x b doubles.
 * ------------------------------------------------------------------------------------ */
void oracle_affinity_matvec(int64_t n, int64_t D, const float *Rp, const float *dinv,
                            const double *Y, int64_t b, double *out) {
    double *W = dalloc((size_t)(D * b));
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < D; ++j)
        for (int64_t i = 0; i < n; ++i) {
            const double rij = (double)dinv[i] * (double)Rp[i * D + j];
            for (int64_t c = 0; c < b; ++c) W[j * b + c] += rij * Y[i * b + c];
        }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
        for (int64_t c = 0; c < b; ++c) {
            double s = 0.0;
            for (int64_t j = 0; j < D; ++j) s += (double)Rp[i * D + j] * W[j * b + c];
            out[i * b + c] = (double)dinv[i] * s;
        }
    free(W);
}

/* ------------------------------------------------------------------------------------
 * Cyclic Jacobi eigensolver for a symmetric D x D matrix A (overwritten).  Eigenvalues
 * in w (unsorted), eigenvectors in the columns of V.  Textbook two-sided rotations.
 * ------------------------------------------------------------------------------------ */
static void jacobi_eig(int64_t D, double *A, double *w, double *V) {
    for (int64_t i = 0; i < D; ++i)
        for (int64_t j = 0; j < D; ++j) V[i * D + j] = (i == j) ? 1.0 : 0.0;
    double fro = 0.0;
    for (int64_t i = 0; i < D * D; ++i) fro += A[i] * A[i];
    fro = sqrt(fro);
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0;
        for (int64_t p = 0; p < D; ++p)
            for (int64_t q = p + 1; q < D; ++q) off += A[p * D + q] * A[p * D + q];
        if (sqrt(2.0 * off) <= 1e-15 * fro || off == 0.0) break;
        for (int64_t p = 0; p < D - 1; ++p)
            for (int64_t q = p + 1; q < D; ++q) {
                const double apq = A[p * D + q];
                if (fabs(apq) <= 1e-300) continue;
                const double app = A[p * D + p], aqq = A[q * D + q];
                const double theta = (aqq - app) / (2.0 * apq);
                const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
                for (int64_t k = 0; k < D; ++k) {          /* columns p, q */
                    const double akp = A[k * D + p], akq = A[k * D + q];
                    A[k * D + p] = c * akp - s * akq;
                    A[k * D + q] = s * akp + c * akq;
                }
                for (int64_t k = 0; k < D; ++k) {          /* rows p, q */
                    const double apk = A[p * D + k], aqk = A[q * D + k];
                    A[p * D + k] = c * apk - s * aqk;
                    A[q * D + k] = s * apk + c * aqk;
                }
                for (int64_t k = 0; k < D; ++k) {
                    const double vkp = V[k * D + p], vkq = V[k * D + q];
                    V[k * D + p] = c * vkp - s * vkq;
                    V[k * D + q] = s * vkp + c * vkq;
                }
            }
    }
    for (int64_t i = 0; i < D; ++i) w[i] = A[i * D + i];
}

void oracle_sym_eig(int64_t D, const double *A_in, double *w, double *V) {
    double *A = dalloc((size_t)(D * D));
    memcpy(A, A_in, sizeof(double) * (size_t)(D * D));
    jacobi_eig(D, A, w, V);
    free(A);
}

/* R8 sign rule for one column pair: flip so that sum_i Gamma[i,l] >= 0; if
 * |sum| < 1e-6 * ||Gamma[:,l]||_1 use the sign of the largest-magnitude entry
 * (smallest index among ties). */
static int sign_rule(int64_t n, int64_t k, const double *Gamma, int64_t l) {
    double s = 0.0, l1 = 0.0, best = -1.0;
    int64_t arg = 0;
    for (int64_t i = 0; i < n; ++i) {
        const double g = Gamma[i * k + l];
        s += g;
        l1 += fabs(g);
        if (fabs(g) > best) { best = fabs(g); arg = i; }
    }
    if (fabs(s) < 1e-6 * l1) return Gamma[arg * k + l] < 0.0 ? -1 : 1;
    return s < 0.0 ? -1 : 1;
}

/* ------------------------------------------------------------------------------------
 * a7: the exact top-k singular triplets (Gamma, Sigma, Psi) of R = diag(dinv) R'
 * -- "the top-k left and right singular vectors of R" of Eq. init-HY
 * (PAPER.md:571-574), R7 reading (exact, not the randomised approximation):
 *   1. G = R^T R (D x D) with fp64 products of the widened fp32 inputs;
 *   2. cyclic Jacobi eigendecomposition of G, eigenpairs sorted descending;
 *      Psi = top-k eigenvectors, sigma = sqrt(max(lambda, 0));
 *   3. Gamma = R Psi Sigma^{-1}; re-orthonormalised by Householder QR (diag(R) > 0);
 *   4. sign rule R8 applied to each pair (Gamma[:,l], Psi[:,l]).
 * Gamma: n x k, sigma: k, Psi: D x k (doubles).  Returns 0, or -5 if sigma_k == 0.
 * Optionally returns all D eigenvalues of G (descending) in lam_all.
 * ------------------------------------------------------------------------------------ */
/* G = R^T R with R = diag(dinv) R' (fp64 products of the widened fp32 inputs), step 1 of
 * oracle_topk; exported on its own for the parity test of the GPU Gram. */
void oracle_gram(int64_t n, int64_t D, const float *Rp, const float *dinv, double *G) {
    /* row a of the upper triangle per thread; each entry summed over i in ascending order */
#pragma omp parallel for schedule(static, 1)
    for (int64_t a = 0; a < D; ++a) {
        double *g = G + a * D;
        for (int64_t b = a; b < D; ++b) g[b] = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            const double di = (double)dinv[i];
            const double ra = di * (double)Rp[i * D + a];
            for (int64_t b = a; b < D; ++b) g[b] += ra * (di * (double)Rp[i * D + b]);
        }
    }
    for (int64_t a = 0; a < D; ++a)
        for (int64_t b = a + 1; b < D; ++b) G[b * D + a] = G[a * D + b];
}

/* Steps 2 (sorting) to 4 of oracle_topk from a given eigendecomposition of G = R^T R:
 * w (D eigenvalues, any order) and V (D x D, eigenvector j in column j).  Exported so that a
 * test may supply the eigenpairs of G from LAPACK (a library eigensolver, pinned against
 * jacobi_eig by the tests) where the O(D^3)-per-sweep Jacobi would be too slow (D = 2000). */
int oracle_topk_from_eig(int64_t n, int64_t D, const float *Rp, const float *dinv, int32_t k,
                         const double *w, const double *V, double *Gamma, double *sigma, double *Psi,
                         double *lam_all) {
    int64_t *ord = (int64_t *)malloc(sizeof(int64_t) * (size_t)D);
    for (int64_t i = 0; i < D; ++i) ord[i] = i;
    for (int64_t i = 1; i < D; ++i) {                 /* insertion sort, descending */
        int64_t x = ord[i], j = i - 1;
        while (j >= 0 && w[ord[j]] < w[x]) { ord[j + 1] = ord[j]; --j; }
        ord[j + 1] = x;
    }
    if (lam_all) for (int64_t i = 0; i < D; ++i) lam_all[i] = w[ord[i]];
    int rc = 0;
    for (int32_t l = 0; l < k; ++l) {
        const double lam = w[ord[l]];
        sigma[l] = sqrt(lam > 0.0 ? lam : 0.0);
        for (int64_t j = 0; j < D; ++j) Psi[j * k + l] = V[j * D + ord[l]];
        if (!(sigma[l] > 0.0)) rc = -5;
    }
    double *Gm = dalloc((size_t)(n * k));
    if (rc == 0) {
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i)
            for (int32_t l = 0; l < k; ++l) {
                double s = 0.0;
                for (int64_t j = 0; j < D; ++j) s += (double)Rp[i * D + j] * Psi[j * k + l];
                Gm[i * k + l] = (double)dinv[i] * s / sigma[l];
            }
        oracle_qr(n, k, Gm, Gamma, NULL);
        for (int32_t l = 0; l < k; ++l)
            if (sign_rule(n, k, Gamma, l) < 0) {
                for (int64_t i = 0; i < n; ++i) Gamma[i * k + l] = -Gamma[i * k + l];
                for (int64_t j = 0; j < D; ++j) Psi[j * k + l] = -Psi[j * k + l];
            }
    }
    free(Gm); free(ord);
    return rc;
}

int oracle_topk(int64_t n, int64_t D, const float *Rp, const float *dinv, int32_t k,
                double *Gamma, double *sigma, double *Psi, double *lam_all) {
    double *G = dalloc((size_t)(D * D));
    oracle_gram(n, D, Rp, dinv, G);
    double *w = dalloc((size_t)D), *V = dalloc((size_t)(D * D));
    jacobi_eig(D, G, w, V);
    const int rc = oracle_topk_from_eig(n, D, Rp, dinv, k, w, V, Gamma, sigma, Psi, lam_all);
    free(V); free(w); free(G);
    return rc;
}

/* ------------------------------------------------------------------------------------
 * f1: SVD-based attribute dimension reduction, Sec. 3.2.1 Eq. Xd:
 *   X' = Gamma Sigma  for the exact top-d SVD X ~ Gamma Sigma Psi^T of the n x d_U matrix X
 * (R14: the exact top-d, the unique result the paper's randomised SVD approximates, as R7),
 * evaluated as X' = X Psi, because X Psi = Gamma Sigma Psi^T Psi = Gamma Sigma for the exact
 * right singular vectors Psi = the top-d eigenvectors of X^T X.  The sign of each column pair is
 * fixed by R8 (column sum of X' >= 0, near-zero sums by the largest-magnitude entry), since
 * X' columns = sigma_l * Gamma columns.  d >= d_U is the pass-through X' = X.
 * oracle_svd_reduce_from_eig takes the eigendecomposition of X^T X (w: d_U eigenvalues in any
 * order, V: eigenvector j in column j); oracle_svd_reduce forms X^T X (fp64 products of the
 * widened fp32 X) and uses the cyclic Jacobi solver.  Xr: n x d doubles; sigma: d (descending).
 * ------------------------------------------------------------------------------------ */
void oracle_svd_reduce_from_eig(int64_t n, int64_t dU, const float *X, int64_t d, const double *w,
                                const double *V, double *Xr, double *sigma) {
    if (d >= dU) {
        for (int64_t i = 0; i < n * dU; ++i) Xr[i] = (double)X[i];
        return;
    }
    int64_t *ord = (int64_t *)malloc(sizeof(int64_t) * (size_t)dU);
    for (int64_t i = 0; i < dU; ++i) ord[i] = i;
    for (int64_t i = 1; i < dU; ++i) {                /* insertion sort, descending */
        int64_t x = ord[i], j = i - 1;
        while (j >= 0 && w[ord[j]] < w[x]) { ord[j + 1] = ord[j]; --j; }
        ord[j + 1] = x;
    }
    for (int64_t l = 0; l < d; ++l) sigma[l] = sqrt(w[ord[l]] > 0.0 ? w[ord[l]] : 0.0);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
        for (int64_t l = 0; l < d; ++l) {
            double s = 0.0;
            for (int64_t j = 0; j < dU; ++j) s += (double)X[i * dU + j] * V[j * dU + ord[l]];
            Xr[i * d + l] = s;
        }
    for (int64_t l = 0; l < d; ++l)
        if (sign_rule(n, d, Xr, l) < 0)
            for (int64_t i = 0; i < n; ++i) Xr[i * d + l] = -Xr[i * d + l];
    free(ord);
}

void oracle_svd_reduce(int64_t n, int64_t dU, const float *X, int64_t d, double *Xr, double *sigma) {
    if (d >= dU) {
        oracle_svd_reduce_from_eig(n, dU, X, d, NULL, NULL, Xr, sigma);
        return;
    }
    float *ones = (float *)malloc(sizeof(float) * (size_t)(n ? n : 1));
    for (int64_t i = 0; i < n; ++i) ones[i] = 1.0f;
    double *G = dalloc((size_t)(dU * dU)), *w = dalloc((size_t)dU), *V = dalloc((size_t)(dU * dU));
    oracle_gram(n, dU, X, ones, G);                  /* X^T X (dinv = 1) */
    jacobi_eig(dU, G, w, V);
    oracle_svd_reduce_from_eig(n, dU, X, d, w, V, Xr, sigma);
    free(ones); free(G); free(w); free(V);
}

/* ------------------------------------------------------------------------------------
 * a8: greedy orthogonal NMF, Alg. 2, from the exact singular
 * triplets of R (Eq. init-HY) with the R9 clamps:
 *   Ups = max(Gamma, 0) + eps,  H = max(Psi Sigma, 0) + eps
 *   repeat Tf times (H first, then Ups):
 *     H   <- H   . max(R^T Ups, 0) / (H (Ups^T Ups) + eps)                 (Eq. update-Q)
 *     Ups <- Ups . sqrt( max(R H, 0) / (max(Ups (Ups^T (R H)), 0) + eps) )  (Eq. update-Y)
 * products bracketed as PAPER.md:564 orders them.  R = diag(dinv) R'.
 * Gamma (n x k) and Psi (D x k) are fp32, sigma fp64, as the CUDA path receives them.
 * Ups: n x k doubles out, H: D x k doubles out.
 * ------------------------------------------------------------------------------------ */
void oracle_onmf(int64_t n, int64_t D, int32_t k, const float *Rp, const float *dinv,
                 const float *Gamma, const double *sigma, const float *Psi, int32_t Tf,
                 double *Ups, double *H) {
    for (int64_t i = 0; i < n; ++i)
        for (int32_t l = 0; l < k; ++l) {
            const double g = (double)Gamma[i * k + l];
            Ups[i * k + l] = (g > 0.0 ? g : 0.0) + EPS_ONMF;
        }
    for (int64_t j = 0; j < D; ++j)
        for (int32_t l = 0; l < k; ++l) {
            const double h = (double)Psi[j * k + l] * sigma[l];
            H[j * k + l] = (h > 0.0 ? h : 0.0) + EPS_ONMF;
        }
    double *RtU = dalloc((size_t)(D * k)), *UtU = dalloc((size_t)(k * k));
    double *HUU = dalloc((size_t)(D * k)), *RH = dalloc((size_t)(n * k));
    double *M = dalloc((size_t)(k * k)), *den = dalloc((size_t)(n * k));
    for (int32_t t = 0; t < Tf; ++t) {
        /* R^T Ups and Ups^T Ups */
        memset(RtU, 0, sizeof(double) * (size_t)(D * k));
        memset(UtU, 0, sizeof(double) * (size_t)(k * k));
#pragma omp parallel for schedule(static)
        for (int64_t j = 0; j < D; ++j)
            for (int64_t i = 0; i < n; ++i) {
                const double rij = (double)dinv[i] * (double)Rp[i * D + j];
                for (int32_t l = 0; l < k; ++l) RtU[j * k + l] += rij * Ups[i * k + l];
            }
#pragma omp parallel for schedule(static)
        for (int32_t a = 0; a < k; ++a)
            for (int64_t i = 0; i < n; ++i)
                for (int32_t b = 0; b < k; ++b) UtU[a * k + b] += Ups[i * k + a] * Ups[i * k + b];
        /* H (Ups^T Ups) then the H update (Eq. update-Q) */
        for (int64_t j = 0; j < D; ++j)
            for (int32_t l = 0; l < k; ++l) {
                double s = 0.0;
                for (int32_t a = 0; a < k; ++a) s += H[j * k + a] * UtU[a * k + l];
                HUU[j * k + l] = s;
            }
        for (int64_t j = 0; j < D * k; ++j) {
            const double num = RtU[j] > 0.0 ? RtU[j] : 0.0;
            H[j] = H[j] * num / (HUU[j] + EPS_ONMF);
        }
        /* R H */
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i)
            for (int32_t l = 0; l < k; ++l) {
                double s = 0.0;
                for (int64_t j = 0; j < D; ++j) s += (double)Rp[i * D + j] * H[j * k + l];
                RH[i * k + l] = (double)dinv[i] * s;
            }
        /* M = Ups^T (R H) */
        memset(M, 0, sizeof(double) * (size_t)(k * k));
#pragma omp parallel for schedule(static)
        for (int32_t a = 0; a < k; ++a)
            for (int64_t i = 0; i < n; ++i)
                for (int32_t b = 0; b < k; ++b) M[a * k + b] += Ups[i * k + a] * RH[i * k + b];
        /* den = Ups M ; Ups update (Eq. update-Y) */
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i)
            for (int32_t l = 0; l < k; ++l) {
                double s = 0.0;
                for (int32_t a = 0; a < k; ++a) s += Ups[i * k + a] * M[a * k + l];
                den[i * k + l] = s;
            }
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n * k; ++i) {
            const double num = RH[i] > 0.0 ? RH[i] : 0.0;
            const double dd = (den[i] > 0.0 ? den[i] : 0.0) + EPS_ONMF;
            Ups[i] = Ups[i] * sqrt(num / dd);
        }
    }
    free(RtU); free(UtU); free(HUU); free(RH); free(M); free(den);
}

/* ------------------------------------------------------------------------------------
 * a9: NCI generation, Alg. 3, R10 reading:
 *   Phi = I;  repeat Tg times:
 *     l*_i = argmax_l Ups[i] . Phi[:, l]   (Eq. ell-ast; ties -> smallest l)
 *     Y[i] = e_{l*}                         (Eq. Y-update)
 *     columns of Y scaled to unit L2 norm   (Eq. y-norm; empty -> zero)
 *     Phi = Ups^T Y
 *   early stop when the labels repeat (result-neutral).  R13: each score (Ups Phi)[i,l] is
 *   accumulated over a = 0..k-1 with one correctly rounded fused multiply-add per term (C99
 *   fma(); the paper fixes no rounding), the same operation the GPU argmax uses, so near-tie
 *   rows are decided identically.  labels: n int32;
 *   *iters_used = iterations run.
 * ------------------------------------------------------------------------------------ */
void oracle_nci(int64_t n, int32_t k, const double *Ups, int32_t Tg, int32_t *labels,
                int32_t *iters_used) {
    double *Phi = dalloc((size_t)(k * k));
    int64_t *cnt = (int64_t *)calloc((size_t)k, sizeof(int64_t));
    for (int32_t a = 0; a < k; ++a) Phi[a * k + a] = 1.0;
    for (int64_t i = 0; i < n; ++i) labels[i] = -1;
    int32_t it = 0;
    for (int32_t t = 0; t < Tg; ++t) {
        int changed = 0;
#pragma omp parallel for schedule(static) reduction(|:changed)
        for (int64_t i = 0; i < n; ++i) {
            int32_t best = 0;
            double bv = 0.0;
            for (int32_t l = 0; l < k; ++l) {
                double s = 0.0;
                for (int32_t a = 0; a < k; ++a) s = fma(Ups[i * k + a], Phi[a * k + l], s);   /* R13 */
                if (l == 0 || s > bv) { bv = s; best = l; }
            }
            if (labels[i] != best) changed = 1;
            labels[i] = best;
        }
        it = t + 1;
        if (!changed) break;
        for (int32_t l = 0; l < k; ++l) cnt[l] = 0;
        for (int64_t i = 0; i < n; ++i) cnt[labels[i]]++;
        memset(Phi, 0, sizeof(double) * (size_t)(k * k));
        for (int64_t i = 0; i < n; ++i) {
            const int32_t l = labels[i];
            const double y = 1.0 / sqrt((double)cnt[l]);
            for (int32_t a = 0; a < k; ++a) Phi[a * k + l] += Ups[i * k + a] * y;
        }
    }
    *iters_used = it;
    free(Phi); free(cnt);
}
