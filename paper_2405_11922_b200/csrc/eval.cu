// Evaluation and monitors on the device.
//
//  * Clustering metrics (Evaluation Metrics): the k_pred x k_true contingency
//    table |C_i intersect C*_j| is counted on the device (per-block shared-memory histograms,
//    integer atomics: exact, order-independent), then ACC (Hungarian matching of predicted to
//    ground-truth labels, Kuhn 1955), NMI and ARI are evaluated from the table on
//    the host in fp64.  NMI reading R15: the printed formula drops |U| inside the logarithm of the
//    numerator (it would not be normalised); the standard Strehl-Ghosh form
//    sum n_ij log(n n_ij / (a_i b_j)) / sqrt(sum a_i log(a_i/n) * sum b_j log(b_j/n)) is used.
//  * Lemma 4 monitor (Eq. obj5): for the NCI matrix Y of a labelling (columns
//    1/sqrt|C_l| on C_l, empty clusters zero) ||R^T Y||_F^2 = Tr(Y^T R R^T Y) -- the quantity
//    the discretisation maximises, bounded above by sum_{l<=k} sigma_l^2 (Ky Fan, E3) -- and,
//    given Ups, ||R^T Ups||_F^2, so that |Tr((Y Y^T - Ups Ups^T) R R^T)| = | ||R^T Y||^2 -
//    ||R^T Ups||^2 |.  R^T Y is formed as R'^T (dinv . Y) by the same fp64 pass as Alg. 2's R^T Ups.
#include <math.h>

#include <algorithm>
#include <limits>
#include <vector>

#include "tpo_internal.cuh"

namespace tpo {
namespace {

constexpr int CT_THREADS = 256;

// counts[a * kb + b] += #{i : pred[i] = a, truth[i] = b}; *bad = 1 for a label out of range
__global__ void contingency_kernel(const int32_t *__restrict__ pa, const int32_t *__restrict__ pb, int64_t n, int ka,
                                   int kb, unsigned long long *__restrict__ counts, int *__restrict__ bad) {
    extern __shared__ unsigned int hist[];
    const int cells = ka * kb;
    for (int i = threadIdx.x; i < cells; i += blockDim.x) hist[i] = 0u;
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int a = pa[i], b = pb[i];
        if (a < 0 || a >= ka || b < 0 || b >= kb) {
            *bad = 1;
            continue;
        }
        atomicAdd(hist + a * kb + b, 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < cells; i += blockDim.x)
        if (hist[i]) atomicAdd(counts + i, (unsigned long long)hist[i]);
}

// Y[i, l] = 1/sqrt(|C_l|) if labels[i] == l else 0 (n x k fp64)
__global__ void nci_matrix_kernel(const int32_t *__restrict__ labels, int64_t n, int k,
                                  const unsigned long long *__restrict__ sizes, double *__restrict__ Y) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n * k) return;
    const int64_t row = i / k;
    const int l = (int)(i - row * k);
    Y[i] = labels[row] == l ? 1.0 / sqrt((double)sizes[l]) : 0.0;
}

// sizes[l] = #{i : labels[i] = l}
__global__ void label_sizes_kernel(const int32_t *__restrict__ labels, int64_t n, int k,
                                   unsigned long long *__restrict__ sizes, int *__restrict__ bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int l = labels[i];
    if (l < 0 || l >= k) {
        *bad = 1;
        return;
    }
    atomicAdd(sizes + l, 1ull);
}

__global__ void frob2_kernel(const double *__restrict__ A, int64_t len, double *__restrict__ out) {
    // one block: fixed-order strided sums, then a fixed tree
    __shared__ double sh[1024];
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < len; i += blockDim.x) s += A[i] * A[i];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int o = blockDim.x / 2; o; o >>= 1) {
        if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sh[0];
}

// Hungarian algorithm (Kuhn-Munkres with potentials), maximising the matched counts of the
// ka x kb contingency table: returns the maximum total of a one-to-one label matching.
int64_t max_matching(const std::vector<int64_t> &ct, int ka, int kb) {
    const int n = std::max(ka, kb);
    const int64_t big = 0;
    // square cost matrix (minimise -count), padded with zeros
    std::vector<double> cost((size_t)(n + 1) * (n + 1), 0.0);
    for (int i = 0; i < ka; ++i)
        for (int j = 0; j < kb; ++j) cost[(size_t)(i + 1) * (n + 1) + (j + 1)] = -(double)ct[(size_t)i * kb + j];
    const double INF = std::numeric_limits<double>::infinity();
    std::vector<double> u(n + 1, 0.0), v(n + 1, 0.0), minv(n + 1);
    std::vector<int> p(n + 1, 0), way(n + 1, 0);
    std::vector<char> used(n + 1);
    for (int i = 1; i <= n; ++i) {
        p[0] = i;
        int j0 = 0;
        std::fill(minv.begin(), minv.end(), INF);
        std::fill(used.begin(), used.end(), 0);
        do {
            used[j0] = 1;
            const int i0 = p[j0];
            double delta = INF;
            int j1 = 0;
            for (int j = 1; j <= n; ++j)
                if (!used[j]) {
                    const double cur = cost[(size_t)i0 * (n + 1) + j] - u[i0] - v[j];
                    if (cur < minv[j]) { minv[j] = cur; way[j] = j0; }
                    if (minv[j] < delta) { delta = minv[j]; j1 = j; }
                }
            for (int j = 0; j <= n; ++j)
                if (used[j]) { u[p[j]] += delta; v[j] -= delta; }
                else minv[j] -= delta;
            j0 = j1;
        } while (p[j0] != 0);
        do {
            const int j1 = way[j0];
            p[j0] = p[j1];
            j0 = j1;
        } while (j0);
    }
    int64_t tot = big;
    for (int j = 1; j <= n; ++j) {
        const int i = p[j];
        if (i >= 1 && i <= ka && j <= kb) tot += ct[(size_t)(i - 1) * kb + (j - 1)];
    }
    return tot;
}

}  // namespace

size_t eval_ws_bytes(int32_t ka, int32_t kb) {
    return align_up(sizeof(unsigned long long) * (size_t)ka * kb) + 256 + 256;
}

void eval_impl(const int32_t *pred, const int32_t *truth, int64_t n, int32_t ka, int32_t kb, double *metrics, Arena &ar,
               cudaStream_t st) {
    unsigned long long *counts = ar.take<unsigned long long>((size_t)ka * kb);
    int *bad = ar.take<int>(1);
    TPO_CUDA(cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * (size_t)ka * kb, st));
    TPO_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
    const size_t smem = sizeof(unsigned int) * (size_t)ka * kb;
    if (smem > 48 * 1024)
        TPO_CUDA(cudaFuncSetAttribute(contingency_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (n > 0) {
        const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, CT_THREADS), 2 * 148));
        contingency_kernel<<<grid, CT_THREADS, smem, st>>>(pred, truth, n, ka, kb, counts, bad);
        TPO_LAUNCH_CHECK();
    }
    std::vector<unsigned long long> h((size_t)ka * kb);
    int hb = 0;
    TPO_CUDA(cudaMemcpyAsync(h.data(), counts, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost, st));
    TPO_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    TPO_CUDA(cudaStreamSynchronize(st));
    if (hb) throw Error(TPO_EINVAL, "tpo_eval: a label lies outside [0, k)");
    std::vector<int64_t> ct(h.begin(), h.end());
    std::vector<double> a(ka, 0.0), b(kb, 0.0);
    for (int i = 0; i < ka; ++i)
        for (int j = 0; j < kb; ++j) {
            a[i] += (double)ct[(size_t)i * kb + j];
            b[j] += (double)ct[(size_t)i * kb + j];
        }
    const double N = (double)n;
    auto c2 = [](double x) { return x * (x - 1.0) / 2.0; };
    // ARI
    double sij = 0.0, sa = 0.0, sb = 0.0;
    for (size_t i = 0; i < ct.size(); ++i) sij += c2((double)ct[i]);
    for (double x : a) sa += c2(x);
    for (double x : b) sb += c2(x);
    const double tot = c2(N);
    const double expv = tot > 0.0 ? sa * sb / tot : 0.0, mx = 0.5 * (sa + sb);
    metrics[0] = mx == expv ? 1.0 : (sij - expv) / (mx - expv);
    // NMI (reading R15)
    double mi = 0.0, ha = 0.0, hbv = 0.0;
    for (int i = 0; i < ka; ++i)
        for (int j = 0; j < kb; ++j) {
            const double nij = (double)ct[(size_t)i * kb + j];
            if (nij > 0.0) mi += nij * log(N * nij / (a[i] * b[j]));
        }
    for (double x : a) if (x > 0.0) ha += x * log(x / N);
    for (double x : b) if (x > 0.0) hbv += x * log(x / N);
    metrics[1] = (ha == 0.0 || hbv == 0.0) ? ((ha == 0.0 && hbv == 0.0) ? 1.0 : 0.0) : mi / sqrt(ha * hbv);
    // ACC: Hungarian matching of predicted to ground-truth labels
    metrics[2] = n > 0 ? (double)max_matching(ct, ka, kb) / N : 0.0;
}

size_t objective_ws_bytes(int64_t n, int64_t D, int32_t k) {
    return align_up(sizeof(double) * (size_t)n * k) + align_up(sizeof(double) * (size_t)D * k) +
           align_up(sizeof(unsigned long long) * k) + onmf_ws_bytes(n, D, k) + 4 * 256;
}

void objective_impl(const float *Rp, const float *dinv, int64_t n, int64_t D, int32_t k, const int32_t *labels,
                    const double *Ups, double *out, Arena &ar, cudaStream_t st) {
    double *Y = ar.take<double>((size_t)n * k), *RtY = ar.take<double>((size_t)D * k), *f = ar.take<double>(2);
    unsigned long long *sizes = ar.take<unsigned long long>(k);
    int *bad = ar.take<int>(1);
    TPO_CUDA(cudaMemsetAsync(sizes, 0, sizeof(unsigned long long) * k, st));
    TPO_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
    if (n > 0) {
        label_sizes_kernel<<<cdiv(n, 256), 256, 0, st>>>(labels, n, k, sizes, bad);
        TPO_LAUNCH_CHECK();
        nci_matrix_kernel<<<cdiv(n * k, 256), 256, 0, st>>>(labels, n, k, sizes, Y);
        TPO_LAUNCH_CHECK();
    }
    const size_t mark = ar.off;
    onmf_rtu(Rp, n, D, dinv, Y, k, RtY, ar, st);          // R^T Y = R'^T (dinv . Y)
    ar.off = mark;
    frob2_kernel<<<1, 1024, 0, st>>>(RtY, D * k, f);
    TPO_LAUNCH_CHECK();
    if (Ups) {
        onmf_rtu(Rp, n, D, dinv, Ups, k, RtY, ar, st);    // R^T Ups
        ar.off = mark;
        frob2_kernel<<<1, 1024, 0, st>>>(RtY, D * k, f + 1);
        TPO_LAUNCH_CHECK();
    }
    int hb = 0;
    TPO_CUDA(cudaMemcpyAsync(out, f, sizeof(double) * (Ups ? 2 : 1), cudaMemcpyDeviceToHost, st));
    TPO_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    TPO_CUDA(cudaStreamSynchronize(st));
    if (hb) throw Error(TPO_EINVAL, "tpo_objective: a label lies outside [0, k)");
}

}  // namespace tpo
