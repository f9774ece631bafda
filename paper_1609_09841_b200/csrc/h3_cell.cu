// Per-cell kernels of the reference's per-cell API (pkg/src/hermite3d/kernels.py:73-191):
// reconstruction sweeps, the advection derivative, the q-stage Horner evolution, the
// space-time coefficient tensor, its evaluation at a time fraction, and the space-time
// identity residual.  These are the semantic spec of the grid kernels, exposed by the
// reference package for single cells; here each runs on the device for a batch of cells.
//
// Arithmetic is the reference's numpy arithmetic operation for operation: separate
// round-to-nearest multiplies and adds (no FMA contraction), the same summation order and
// the same typed zeros, in the caller's precision (float or double), so every result is
// bit-identical to the reference for the same inputs (tests/test_gpu_cell_api.py pins the
// reference's golden digests).  Sizes are tiny (one cell is (2N+2)^3 values): one CTA per
// cell, grid-stride over the cell's entries, a barrier between dependent stages.
#include "../../include/h3b200.h"
#include "h3_launch.h"

namespace h3 {
namespace cell {

__device__ __forceinline__ double radd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double rmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double rsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float radd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float rmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float rsub(float a, float b) { return __fsub_rn(a, b); }

struct Shape {
    int n3, n2, n1;
    __device__ int size() const { return n3 * n2 * n1; }
};

// advect_time_derivative (kernels.py:99-108): out = s1; out += s2; out += s3, where
// s_k[i] = w[i + e_k] * fac_k[i_k] below the top index of axis k and +0 at it
// (_axis_shift_scale, kernels.py:90-96: zeros_like, then the shifted product).
template <typename T>
__device__ __forceinline__ T advect_at(const T* w, int e, const Shape& s, const T* f1, const T* f2,
                                       const T* f3) {
    const int i1 = e % s.n1, i2 = (e / s.n1) % s.n2, i3 = e / (s.n1 * s.n2);
    const T z = T(0);
    const T s1 = i1 < s.n1 - 1 ? rmul(w[e + 1], f1[i1]) : z;
    const T s2 = i2 < s.n2 - 1 ? rmul(w[e + s.n1], f2[i2]) : z;
    const T s3 = i3 < s.n3 - 1 ? rmul(w[e + s.n1 * s.n2], f3[i3]) : z;
    return radd(radd(s1, s2), s3);
}

// apply_along_axis (operators.py:127-151) as used by reconstruct_cell (kernels.py:73-87):
// out[.., i, ..] = 0 + m[i][0] x[.., 0, ..] + m[i][1] x[.., 1, ..] + ... (ascending k,
// accumulated from a zero array).
template <typename T>
__global__ void apply_axis_kernel(const T* __restrict__ in, T* __restrict__ out, Shape s,
                                  const T* __restrict__ mat, int axis) {
    const int size = s.size();
    const T* x = in + (int64_t)blockIdx.x * size;
    T* y = out + (int64_t)blockIdx.x * size;
    const int len = axis == 1 ? s.n1 : axis == 2 ? s.n2 : s.n3;
    const int stride = axis == 1 ? 1 : axis == 2 ? s.n1 : s.n1 * s.n2;
    for (int e = threadIdx.x; e < size; e += blockDim.x) {
        const int i = (e / stride) % len;
        const T* line = x + (e - i * stride);
        T acc = T(0);
        for (int k = 0; k < len; ++k) acc = radd(acc, rmul(mat[i * len + k], line[k * stride]));
        y[e] = acc;
    }
}

template <typename T>
__global__ void advect_kernel(const T* __restrict__ w, T* __restrict__ out, Shape s,
                              const T* __restrict__ f1, const T* __restrict__ f2,
                              const T* __restrict__ f3) {
    const int size = s.size();
    const T* wc = w + (int64_t)blockIdx.x * size;
    T* oc = out + (int64_t)blockIdx.x * size;
    for (int e = threadIdx.x; e < size; e += blockDim.x) oc[e] = advect_at(wc, e, s, f1, f2, f3);
}

// taylor_evolve_horner (kernels.py:111-128): w = b; for k = q..1: w = b + c_k * L(w), two-phase
// (each stage reads the whole previous w).  c_k = (T)(step / k), precomputed by the caller.
// `out` and `tmp` are the ping-pong buffers; the result ends in `out`.
template <typename T>
__global__ void horner_kernel(const T* __restrict__ b, T* out, T* tmp, Shape s, const T* __restrict__ f1,
                              const T* __restrict__ f2, const T* __restrict__ f3,
                              const T* __restrict__ cst, int q) {
    const int size = s.size();
    const int64_t base = (int64_t)blockIdx.x * size;
    const T* bc = b + base;
    // the buffer written by the last stage must be `out`: start in the other one when q is odd
    T* cur = (q & 1) ? tmp + base : out + base;
    T* nxt = (q & 1) ? out + base : tmp + base;
    for (int e = threadIdx.x; e < size; e += blockDim.x) cur[e] = bc[e];
    __syncthreads();
    for (int k = q; k >= 1; --k) {
        const T c = cst[k - 1];
        for (int e = threadIdx.x; e < size; e += blockDim.x)
            nxt[e] = radd(bc[e], rmul(c, advect_at(cur, e, s, f1, f2, f3)));
        __syncthreads();
        T* t = cur;
        cur = nxt;
        nxt = t;
    }
}

// space_time_tensor (kernels.py:131-142): st[0] = b, st[j+1] = c_j * L(st[j]), c_j = (T)(dt/(j+1)).
// st layout: [cell][j = 0..q][entry].
template <typename T>
__global__ void space_time_kernel(const T* __restrict__ b, T* __restrict__ st, Shape s,
                                  const T* __restrict__ f1, const T* __restrict__ f2,
                                  const T* __restrict__ f3, const T* __restrict__ cst, int q) {
    const int size = s.size();
    const T* bc = b + (int64_t)blockIdx.x * size;
    T* sc = st + (int64_t)blockIdx.x * (q + 1) * size;
    for (int e = threadIdx.x; e < size; e += blockDim.x) sc[e] = bc[e];
    __syncthreads();
    for (int j = 0; j < q; ++j) {
        const T c = cst[j];
        const T* cur = sc + (int64_t)j * size;
        T* nxt = sc + (int64_t)(j + 1) * size;
        for (int e = threadIdx.x; e < size; e += blockDim.x) nxt[e] = rmul(c, advect_at(cur, e, s, f1, f2, f3));
        __syncthreads();
    }
}

// taylor_evolve_recursion's sum (kernels.py:157-164): acc = st[0]; acc += st[j] * t_j for j = 1..q,
// t_j = (T)(tau^j) with tau^j formed by repeated multiplication in double by the caller.
template <typename T>
__global__ void time_sum_kernel(const T* __restrict__ st, T* __restrict__ out, int size,
                                const T* __restrict__ tpow, int q) {
    const T* sc = st + (int64_t)blockIdx.x * (q + 1) * size;
    T* oc = out + (int64_t)blockIdx.x * size;
    for (int e = threadIdx.x; e < size; e += blockDim.x) {
        T acc = sc[e];
        for (int j = 1; j <= q; ++j) acc = radd(acc, rmul(sc[(int64_t)j * size + e], tpow[j - 1]));
        oc[e] = acc;
    }
}

// verify_space_time_identity (kernels.py:167-191): residual_j = c_j st[j+1] - L(st[j]) (j < q),
// -L(st[q]) at the top; c_j = (T)((j+1) / dt).  The max |residual| over the cell(s) is exact in
// any order: non-negative doubles order like their bit patterns, so one atomicMax suffices.
template <typename T>
__global__ void identity_kernel(const T* __restrict__ st, Shape s, const T* __restrict__ f1,
                                const T* __restrict__ f2, const T* __restrict__ f3,
                                const T* __restrict__ coef, int q, unsigned long long* worst) {
    const int size = s.size();
    const T* sc = st + (int64_t)blockIdx.x * (q + 1) * size;
    unsigned long long mine = 0;
    for (int j = 0; j <= q; ++j) {
        const T* cur = sc + (int64_t)j * size;
        for (int e = threadIdx.x; e < size; e += blockDim.x) {
            const T spatial = advect_at(cur, e, s, f1, f2, f3);
            const T r = j < q ? rsub(rmul(coef[j], cur[size + e]), spatial) : -spatial;
            const double a = fabs((double)r);
            const unsigned long long bits = (unsigned long long)__double_as_longlong(a);
            mine = bits > mine ? bits : mine;
        }
    }
    atomicMax(worst, mine);
}

static bool shape_ok(int64_t batch, int n3, int n2, int n1) {
    return batch >= 0 && batch < (1ll << 31) && n3 >= 1 && n2 >= 1 && n1 >= 1 &&
           (int64_t)n3 * n2 * n1 < (1ll << 28);
}

constexpr int kThreads = 256;

}  // namespace cell
}  // namespace h3

using namespace h3::cell;

template <typename T>
static int apply_axis_t(const void* in, void* out, int64_t batch, int n3, int n2, int n1, const void* mat,
                        int axis, cudaStream_t st) {
    if (batch == 0) return 0;
    apply_axis_kernel<T><<<(unsigned)batch, kThreads, 0, st>>>((const T*)in, (T*)out, Shape{n3, n2, n1},
                                                               (const T*)mat, axis);
    return (int)cudaGetLastError();
}

extern "C" int h3_cell_apply_axis(const void* in, void* out, int64_t batch, int n3, int n2, int n1,
                                  const void* mat, int axis, int single, void* stream) {
    if (!in || !out || !mat || !shape_ok(batch, n3, n2, n1) || axis < 1 || axis > 3) return H3_ERR_ARG;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    return single ? apply_axis_t<float>(in, out, batch, n3, n2, n1, mat, axis, st)
                  : apply_axis_t<double>(in, out, batch, n3, n2, n1, mat, axis, st);
}

extern "C" int h3_cell_advect(const void* w, void* out, int64_t batch, int n3, int n2, int n1,
                              const void* f1, const void* f2, const void* f3, int single, void* stream) {
    if (!w || !out || !f1 || !f2 || !f3 || !shape_ok(batch, n3, n2, n1)) return H3_ERR_ARG;
    if (batch == 0) return 0;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const Shape s{n3, n2, n1};
    if (single)
        advect_kernel<float><<<(unsigned)batch, kThreads, 0, st>>>((const float*)w, (float*)out, s, (const float*)f1,
                                                                   (const float*)f2, (const float*)f3);
    else
        advect_kernel<double><<<(unsigned)batch, kThreads, 0, st>>>((const double*)w, (double*)out, s,
                                                                    (const double*)f1, (const double*)f2,
                                                                    (const double*)f3);
    return (int)cudaGetLastError();
}

extern "C" int h3_cell_horner(const void* b, void* out, void* tmp, int64_t batch, int n3, int n2, int n1,
                              const void* f1, const void* f2, const void* f3, const void* cstage, int q,
                              int single, void* stream) {
    if (!b || !out || !tmp || !f1 || !f2 || !f3 || !cstage || !shape_ok(batch, n3, n2, n1)) return H3_ERR_ARG;
    if (q < 1) return H3_ERR_STAGES;
    if (batch == 0) return 0;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const Shape s{n3, n2, n1};
    if (single)
        horner_kernel<float><<<(unsigned)batch, kThreads, 0, st>>>((const float*)b, (float*)out, (float*)tmp, s,
                                                                   (const float*)f1, (const float*)f2,
                                                                   (const float*)f3, (const float*)cstage, q);
    else
        horner_kernel<double><<<(unsigned)batch, kThreads, 0, st>>>((const double*)b, (double*)out, (double*)tmp, s,
                                                                    (const double*)f1, (const double*)f2,
                                                                    (const double*)f3, (const double*)cstage, q);
    return (int)cudaGetLastError();
}

extern "C" int h3_cell_space_time(const void* b, void* st_out, int64_t batch, int n3, int n2, int n1,
                                  const void* f1, const void* f2, const void* f3, const void* cstage, int q,
                                  int single, void* stream) {
    if (!b || !st_out || !f1 || !f2 || !f3 || !cstage || !shape_ok(batch, n3, n2, n1)) return H3_ERR_ARG;
    if (q < 0) return H3_ERR_STAGES;
    if (batch == 0) return 0;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const Shape s{n3, n2, n1};
    if (single)
        space_time_kernel<float><<<(unsigned)batch, kThreads, 0, st>>>((const float*)b, (float*)st_out, s,
                                                                       (const float*)f1, (const float*)f2,
                                                                       (const float*)f3, (const float*)cstage, q);
    else
        space_time_kernel<double><<<(unsigned)batch, kThreads, 0, st>>>((const double*)b, (double*)st_out, s,
                                                                        (const double*)f1, (const double*)f2,
                                                                        (const double*)f3, (const double*)cstage, q);
    return (int)cudaGetLastError();
}

extern "C" int h3_cell_time_sum(const void* st_in, void* out, int64_t batch, int64_t size, const void* tpow, int q,
                                int single, void* stream) {
    if (!st_in || !out || !tpow || batch < 0 || size < 1 || size >= (1ll << 28)) return H3_ERR_ARG;
    if (q < 0) return H3_ERR_STAGES;
    if (batch == 0) return 0;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (single)
        time_sum_kernel<float><<<(unsigned)batch, kThreads, 0, st>>>((const float*)st_in, (float*)out, (int)size,
                                                                     (const float*)tpow, q);
    else
        time_sum_kernel<double><<<(unsigned)batch, kThreads, 0, st>>>((const double*)st_in, (double*)out, (int)size,
                                                                      (const double*)tpow, q);
    return (int)cudaGetLastError();
}

extern "C" int h3_cell_identity_residual(const void* st_in, int64_t batch, int n3, int n2, int n1, const void* f1,
                                         const void* f2, const void* f3, const void* coef, int q,
                                         unsigned long long* d_worst, int single, void* stream) {
    if (!st_in || !f1 || !f2 || !f3 || !coef || !d_worst || !shape_ok(batch, n3, n2, n1)) return H3_ERR_ARG;
    if (q < 0) return H3_ERR_STAGES;
    if (batch == 0) return 0;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const Shape s{n3, n2, n1};
    if (single)
        identity_kernel<float><<<(unsigned)batch, kThreads, 0, st>>>((const float*)st_in, s, (const float*)f1,
                                                                     (const float*)f2, (const float*)f3,
                                                                     (const float*)coef, q, d_worst);
    else
        identity_kernel<double><<<(unsigned)batch, kThreads, 0, st>>>((const double*)st_in, s, (const double*)f1,
                                                                      (const double*)f2, (const double*)f3,
                                                                      (const double*)coef, q, d_worst);
    return (int)cudaGetLastError();
}
