/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle for the Hermite half-step.
 *
 * This file is a plain-C restatement of the reference's grid kernels
 * (reference: pkg/src/hermite3d/gridkernels.py).  It is compiled into
 * oracle/_build/libh3oracle.so and is loaded ONLY by tests/, by
 * __graft_entry__.smoke() (as the checker) and by bench.py's cpu_baseline /
 * --impl reference legs.  The product (paper_1609_09841_b200) never links,
 * imports or calls it.
 *
 * Bit-exactness contract: every output element is produced by the same
 * sequence of IEEE binary64 (or binary32) multiplies and adds, in the same
 * order, as the reference's numba code, which itself matches the numpy
 * per-cell path (reference: pkg/src/hermite3d/kernels.py:73-128).  Build
 * with -ffp-contract=off and without -ffast-math so no FMA is formed.
 * Results were checked bit-for-bit against the imported reference
 * (tests/golden/make_golden.py -> tests/golden/golden.json).
 *
 * Per-cell stages (all indices [z][y][x] = [n3][n2][n1], side s = 2N+2):
 *   gather      gridkernels.py:42-55   8 vertex blocks, periodic wrap, offset `off`
 *   reconstruct gridkernels.py:58-83   H sweeps x1, x2, x3; c = H[i,0]u0; c += H[i,k]uk
 *   evolve      gridkernels.py:86-110  q-stage Horner, two-phase (dsum then w)
 *   scatter     gridkernels.py:113-118 low n^3 block -> dst[c3,c2,c1]
 * Drivers: fused_pass 121-139, recon_pass 142-160, evolve_pass 163-182.
 * Tiling (make_tiles, 28-39) does not affect results and is replaced by an
 * OpenMP loop over (c3, c2) lines.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define IDX3(s, z, y, x) ((((size_t)(z)) * (s) + (y)) * (s) + (x))

static int64_t wrapi(int64_t v, int64_t m) {
    int64_t r = v % m;
    return r < 0 ? r + m : r;
}

#define DEFINE_ORACLE(T, SUF)                                                         \
static void gather_##SUF(const T* src, int64_t M1, int64_t M2, int64_t M3,            \
                         int64_t c1, int64_t c2, int64_t c3, int off, int n, T* u) {  \
    const int s = 2 * n;                                                              \
    const size_t blk = (size_t)n * n * n;                                             \
    for (int a3 = 0; a3 < 2; ++a3) {                                                  \
        int64_t g3 = wrapi(c3 + off + a3, M3);                                        \
        for (int a2 = 0; a2 < 2; ++a2) {                                              \
            int64_t g2 = wrapi(c2 + off + a2, M2);                                    \
            for (int a1 = 0; a1 < 2; ++a1) {                                          \
                int64_t g1 = wrapi(c1 + off + a1, M1);                                \
                const T* node = src + ((size_t)((g3 * M2 + g2) * M1 + g1)) * blk;     \
                for (int j3 = 0; j3 < n; ++j3)                                        \
                    for (int j2 = 0; j2 < n; ++j2)                                    \
                        for (int j1 = 0; j1 < n; ++j1)                                \
                            u[IDX3(s, a3 * n + j3, a2 * n + j2, a1 * n + j1)] =       \
                                node[(j3 * n + j2) * n + j1];                         \
            }                                                                         \
        }                                                                             \
    }                                                                                 \
}                                                                                     \
                                                                                      \
/* three sweeps; u is clobbered (ping-pong), result lands in ru */                    \
static void reconstruct_##SUF(const T* H, int s, T* u, T* ru) {                       \
    for (int z = 0; z < s; ++z)                                                       \
        for (int y = 0; y < s; ++y)                                                   \
            for (int i = 0; i < s; ++i) {                                             \
                T c = H[i * s] * u[IDX3(s, z, y, 0)];                                 \
                for (int k = 1; k < s; ++k) c += H[i * s + k] * u[IDX3(s, z, y, k)];  \
                ru[IDX3(s, z, y, i)] = c;                                             \
            }                                                                         \
    for (int z = 0; z < s; ++z)                                                       \
        for (int i = 0; i < s; ++i)                                                   \
            for (int x = 0; x < s; ++x) {                                             \
                T c = H[i * s] * ru[IDX3(s, z, 0, x)];                                \
                for (int k = 1; k < s; ++k) c += H[i * s + k] * ru[IDX3(s, z, k, x)]; \
                u[IDX3(s, z, i, x)] = c;                                              \
            }                                                                         \
    for (int i = 0; i < s; ++i)                                                       \
        for (int y = 0; y < s; ++y)                                                   \
            for (int x = 0; x < s; ++x) {                                             \
                T c = H[i * s] * u[IDX3(s, 0, y, x)];                                 \
                for (int k = 1; k < s; ++k) c += H[i * s + k] * u[IDX3(s, k, y, x)];  \
                ru[IDX3(s, i, y, x)] = c;                                             \
            }                                                                         \
}                                                                                     \
                                                                                      \
static void evolve_##SUF(const T* ru, const T* f1, const T* f2, const T* f3,          \
                         const T* cf, int q, int s, T* w, T* d) {                     \
    const size_t vol = (size_t)s * s * s;                                             \
    memcpy(w, ru, vol * sizeof(T));                                                   \
    for (int k = q; k >= 1; --k) {                                                    \
        const T c = cf[k - 1];                                                        \
        for (int z = 0; z < s; ++z)                                                   \
            for (int y = 0; y < s; ++y)                                               \
                for (int x = 0; x < s; ++x) {                                         \
                    T acc = f1[s - 1]; /* the reference's typed zero */               \
                    if (x < s - 1) acc += f1[x] * w[IDX3(s, z, y, x + 1)];            \
                    if (y < s - 1) acc += f2[y] * w[IDX3(s, z, y + 1, x)];            \
                    if (z < s - 1) acc += f3[z] * w[IDX3(s, z + 1, y, x)];            \
                    d[IDX3(s, z, y, x)] = acc;                                        \
                }                                                                     \
        for (size_t e = 0; e < vol; ++e) w[e] = ru[e] + c * d[e];                     \
    }                                                                                 \
}                                                                                     \
                                                                                      \
static void scatter_##SUF(const T* w, int n, int s, T* node) {                        \
    for (int j3 = 0; j3 < n; ++j3)                                                    \
        for (int j2 = 0; j2 < n; ++j2)                                                \
            for (int j1 = 0; j1 < n; ++j1)                                            \
                node[(j3 * n + j2) * n + j1] = w[IDX3(s, j3, j2, j1)];                \
}                                                                                     \
                                                                                      \
int h3o_fused_pass_##SUF(const T* src, T* dst, int64_t M1, int64_t M2, int64_t M3,    \
                         int order_n, const T* H, const T* f1, const T* f2,           \
                         const T* f3, const T* cf, int q, int off, int nthreads) {    \
    const int n = order_n + 1, s = 2 * n;                                             \
    const size_t vol = (size_t)s * s * s, blk = (size_t)n * n * n;                    \
    int err = 0;                                                                      \
    _Pragma("omp parallel num_threads(nthreads > 0 ? nthreads : omp_get_max_threads())") \
    {                                                                                 \
        T* buf = (T*)malloc(4 * vol * sizeof(T));                                     \
        if (!buf) { _Pragma("omp atomic write") err = 1; }                            \
        else {                                                                        \
            T *u = buf, *ru = buf + vol, *w = buf + 2 * vol, *d = buf + 3 * vol;      \
            _Pragma("omp for schedule(static)")                                       \
            for (int64_t line = 0; line < M3 * M2; ++line) {                          \
                int64_t c3 = line / M2, c2 = line % M2;                               \
                for (int64_t c1 = 0; c1 < M1; ++c1) {                                 \
                    gather_##SUF(src, M1, M2, M3, c1, c2, c3, off, n, u);             \
                    reconstruct_##SUF(H, s, u, ru);                                   \
                    evolve_##SUF(ru, f1, f2, f3, cf, q, s, w, d);                     \
                    scatter_##SUF(w, n, s, dst + ((size_t)(line * M1 + c1)) * blk);   \
                }                                                                     \
            }                                                                         \
            free(buf);                                                                \
        }                                                                             \
    }                                                                                 \
    return err;                                                                       \
}                                                                                     \
                                                                                      \
int h3o_recon_pass_##SUF(const T* src, T* coeff, int64_t M1, int64_t M2, int64_t M3,  \
                         int order_n, const T* H, int off, int nthreads) {            \
    const int n = order_n + 1, s = 2 * n;                                             \
    const size_t vol = (size_t)s * s * s;                                             \
    int err = 0;                                                                      \
    _Pragma("omp parallel num_threads(nthreads > 0 ? nthreads : omp_get_max_threads())") \
    {                                                                                 \
        T* buf = (T*)malloc(2 * vol * sizeof(T));                                     \
        if (!buf) { _Pragma("omp atomic write") err = 1; }                            \
        else {                                                                        \
            _Pragma("omp for schedule(static)")                                       \
            for (int64_t line = 0; line < M3 * M2; ++line) {                          \
                int64_t c3 = line / M2, c2 = line % M2;                               \
                for (int64_t c1 = 0; c1 < M1; ++c1) {                                 \
                    gather_##SUF(src, M1, M2, M3, c1, c2, c3, off, n, buf);           \
                    reconstruct_##SUF(H, s, buf, buf + vol);                          \
                    memcpy(coeff + ((size_t)(line * M1 + c1)) * vol, buf + vol,       \
                           vol * sizeof(T));                                          \
                }                                                                     \
            }                                                                         \
            free(buf);                                                                \
        }                                                                             \
    }                                                                                 \
    return err;                                                                       \
}                                                                                     \
                                                                                      \
int h3o_evolve_pass_##SUF(const T* coeff, T* dst, int64_t M1, int64_t M2, int64_t M3, \
                          int order_n, const T* f1, const T* f2, const T* f3,         \
                          const T* cf, int q, int nthreads) {                         \
    const int n = order_n + 1, s = 2 * n;                                             \
    const size_t vol = (size_t)s * s * s, blk = (size_t)n * n * n;                    \
    int err = 0;                                                                      \
    _Pragma("omp parallel num_threads(nthreads > 0 ? nthreads : omp_get_max_threads())") \
    {                                                                                 \
        T* buf = (T*)malloc(2 * vol * sizeof(T));                                     \
        if (!buf) { _Pragma("omp atomic write") err = 1; }                            \
        else {                                                                        \
            _Pragma("omp for schedule(static)")                                       \
            for (int64_t cell = 0; cell < M3 * M2 * M1; ++cell) {                     \
                evolve_##SUF(coeff + (size_t)cell * vol, f1, f2, f3, cf, q, s, buf,   \
                             buf + vol);                                              \
                scatter_##SUF(buf, n, s, dst + (size_t)cell * blk);                   \
            }                                                                         \
            free(buf);                                                                \
        }                                                                             \
    }                                                                                 \
    return err;                                                                       \
}

DEFINE_ORACLE(double, f64)
DEFINE_ORACLE(float, f32)

int h3o_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
