// Device-side initial data, error norms and finiteness scan.
//
// init:   reference problems.py:150-175 -- every DOF is the sum over separable
//         terms of a3[m3][n3] * a2[m2][n2] * a1[m1][n1] (per-axis scaled-derivative
//         tables built on the host, problems.py:47-54).  Accumulated term by term
//         from zero with the product formed left to right, as the host einsum does.
// errors: reference problems.py:202-213 -- l_inf and volume-weighted l2 of
//         node values (DOF n = 0) against sum_t e3[t][m3] e2[t][m2] e1[t][m1].
//         Two-stage deterministic reduction (no float atomics).
// finite: reference pipeline.py:210-215 -- first non-finite node in C order.
#include <cstdlib>

#include "h3_launch.h"

namespace h3 {

int band_width(int dflt) {
#ifdef H3_MEASURE
    static const int v = [] {  // tools library only: H3_BAND overrides every launcher's default
        const char* e = getenv("H3_BAND");
        return e ? atoi(e) : -1;
    }();
    return v >= 0 ? v : dflt;
#else
    return dflt;
#endif
}

int num_sms() {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess)
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms > 0 ? sms : 148;
}

__global__ void init_separable_kernel(double* __restrict__ dst, int64_t M1, int64_t M2, int64_t M3,
                                      int n, int nterms, const double* __restrict__ t1,
                                      const double* __restrict__ t2, const double* __restrict__ t3) {
    const int64_t n3 = (int64_t)n * n * n;
    const int64_t total = M1 * M2 * M3 * n3;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t node = e / n3;
        const int dof = (int)(e - node * n3);
        const int j1 = dof % n, j2 = (dof / n) % n, j3 = dof / (n * n);
        const int64_t m1 = node % M1, m2 = (node / M1) % M2, m3 = node / (M1 * M2);
        double acc = 0.0;
        for (int t = 0; t < nterms; ++t) {
            const double a3 = t3[(t * M3 + m3) * n + j3];
            const double a2 = t2[(t * M2 + m2) * n + j2];
            const double a1 = t1[(t * M1 + m1) * n + j1];
            acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(a3, a2), a1));
        }
        dst[e] = acc;
    }
}

int init_separable_launch(double* dst, int64_t M1, int64_t M2, int64_t M3, int order_n, int nterms,
                          const double* t1, const double* t2, const double* t3, cudaStream_t st) {
    const int n = order_n + 1;
    const int64_t total = M1 * M2 * M3 * n * n * n;
    if (total <= 0) return 0;
    int64_t blocks = (total + 255) / 256;
    const int64_t cap = (int64_t)num_sms() * 16;
    if (blocks > cap) blocks = cap;
    init_separable_kernel<<<(unsigned)blocks, 256, 0, st>>>(dst, M1, M2, M3, n, nterms, t1, t2, t3);
    return (int)cudaGetLastError();
}

// stage 1: per-block (max |diff|, sum diff^2) over node values
__global__ void error_partials_kernel(const double* __restrict__ field, int64_t M1, int64_t M2,
                                      int64_t M3, int64_t n3, int nterms,
                                      const double* __restrict__ e1, const double* __restrict__ e2,
                                      const double* __restrict__ e3, double* __restrict__ partials) {
    __shared__ double smax[256], ssum[256];
    const int64_t nodes = M1 * M2 * M3;
    double mx = 0.0, sm = 0.0;
    for (int64_t node = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; node < nodes;
         node += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m1 = node % M1, m2 = (node / M1) % M2, m3 = node / (M1 * M2);
        double ex = 0.0;
        for (int t = 0; t < nterms; ++t)
            ex += e1[t * M1 + m1] * e2[t * M2 + m2] * e3[t * M3 + m3];
        const double diff = field[node * n3] - ex;
        mx = fmax(mx, fabs(diff));
        sm = fma(diff, diff, sm);
        if (diff != diff) mx = diff;  // propagate NaN
    }
    smax[threadIdx.x] = mx;
    ssum[threadIdx.x] = sm;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            const double o = smax[threadIdx.x + w];
            smax[threadIdx.x] = (o != o) ? o : fmax(smax[threadIdx.x], o);
            ssum[threadIdx.x] += ssum[threadIdx.x + w];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = smax[0];
        partials[2 * blockIdx.x + 1] = ssum[0];
    }
}

__global__ void error_final_kernel(const double* __restrict__ partials, int nblocks, double* out) {
    __shared__ double smax[256], ssum[256];
    double mx = 0.0, sm = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += blockDim.x) {
        const double o = partials[2 * b];
        mx = (o != o) ? o : fmax(mx, o);
        sm += partials[2 * b + 1];
    }
    smax[threadIdx.x] = mx;
    ssum[threadIdx.x] = sm;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            const double o = smax[threadIdx.x + w];
            smax[threadIdx.x] = (o != o) ? o : fmax(smax[threadIdx.x], o);
            ssum[threadIdx.x] += ssum[threadIdx.x + w];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[0] = smax[0];
        out[1] = ssum[0];
    }
}

int error_norms_launch(const double* field, int64_t M1, int64_t M2, int64_t M3, int order_n,
                       int nterms, const double* e1, const double* e2, const double* e3,
                       double* d_partials, int64_t n_partials, double* d_out, cudaStream_t st) {
    const int64_t n = order_n + 1;
    const int64_t nodes = M1 * M2 * M3;
    int64_t blocks = (nodes + 255) / 256;
    if (blocks > n_partials) blocks = n_partials;
    if (blocks > 4096) blocks = 4096;
    if (blocks < 1) return (int)cudaErrorInvalidValue;
    error_partials_kernel<<<(unsigned)blocks, 256, 0, st>>>(field, M1, M2, M3, n * n * n, nterms,
                                                             e1, e2, e3, d_partials);
    error_final_kernel<<<1, 256, 0, st>>>(d_partials, (int)blocks, d_out);
    return (int)cudaGetLastError();
}

__global__ void check_finite_kernel(const double* __restrict__ field, int64_t nodes, int n3,
                                    unsigned long long* first_bad) {
    for (int64_t node = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; node < nodes;
         node += (int64_t)gridDim.x * blockDim.x) {
        bool bad = false;
        for (int k = 0; k < n3; ++k) bad |= !isfinite(field[node * n3 + k]);
        if (bad) flag_bad(first_bad, node);
    }
}

int check_finite_launch(const double* field, int64_t M1, int64_t M2, int64_t M3, int order_n,
                        unsigned long long* first_bad, cudaStream_t st) {
    const int n = order_n + 1;
    const int64_t nodes = M1 * M2 * M3;
    if (nodes <= 0) return 0;
    int64_t blocks = (nodes + 255) / 256;
    const int64_t cap = (int64_t)num_sms() * 16;
    if (blocks > cap) blocks = cap;
    check_finite_kernel<<<(unsigned)blocks, 256, 0, st>>>(field, nodes, n * n * n, first_bad);
    return (int)cudaGetLastError();
}

}  // namespace h3
