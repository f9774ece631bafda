/* A C host driving the B200 step through the C ABI alone (include/h3b200.h, libh3b200.so):
 * no Python, no torch.  m = 3 plane wave on a 16^3 periodic grid, 4 full steps of the fused
 * separable half step, node-value error against the exact advected solution, compared with the
 * reference's golden value (N=3, 16^3, 4 steps, l_inf = 2.385797115e-10).
 *
 * The inputs are the reference's own kernel arguments: H (its interpolation matrix, exact
 * rationals rounded once -- embedded here as hex floats), fac_k[i] = (i+1) * (1/h_k),
 * cfac[k-1] = delta / k (reference pipeline.py:197-207), the gather offset 0 / -1 per half step.
 *
 * build: gcc -O2 examples/c_host_step.c -Iinclude -Lpaper_1609_09841_b200 -lh3b200 \
 *            -L/usr/local/cuda/lib64 -lcudart -lm -Wl,-rpath,'$ORIGIN/../paper_1609_09841_b200'
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "h3b200.h"

#define N 3
#define NP (N + 1)
#define S (2 * N + 2)
#define M 16
#define STEPS 4
#define TERMS 4

static const double H[S * S] = {0x1.0000000000000p-1, 0x1.6000000000000p-3, 0x1.8000000000000p-5, 0x1.0000000000000p-7, 0x1.0000000000000p-1, -0x1.6000000000000p-3, 0x1.8000000000000p-5, -0x1.0000000000000p-7, -0x1.1800000000000p+1, -0x1.3000000000000p-1, -0x1.0000000000000p-3, -0x1.0000000000000p-6, 0x1.1800000000000p+1, -0x1.3000000000000p-1, 0x1.0000000000000p-3, -0x1.0000000000000p-6, 0x0.0p+0, -0x1.e000000000000p-1, -0x1.c000000000000p-2, -0x1.8000000000000p-4, 0x0.0p+0, 0x1.e000000000000p-1, -0x1.c000000000000p-2, 0x1.8000000000000p-4, 0x1.1800000000000p+3, 0x1.1800000000000p+2, 0x1.4000000000000p+0, 0x1.8000000000000p-3, -0x1.1800000000000p+3, 0x1.1800000000000p+2, -0x1.4000000000000p+0, 0x1.8000000000000p-3, 0x0.0p+0, 0x1.4000000000000p+0, 0x1.4000000000000p+0, 0x1.8000000000000p-2, 0x0.0p+0, -0x1.4000000000000p+0, 0x1.4000000000000p+0, -0x1.8000000000000p-2, -0x1.5000000000000p+4, -0x1.5000000000000p+3, -0x1.0000000000000p+2, -0x1.8000000000000p-1, 0x1.5000000000000p+4, -0x1.5000000000000p+3, 0x1.0000000000000p+2, -0x1.8000000000000p-1, 0x0.0p+0, -0x1.0000000000000p+0, -0x1.0000000000000p+0, -0x1.0000000000000p-1, 0x0.0p+0, 0x1.0000000000000p+0, -0x1.0000000000000p+0, 0x1.0000000000000p-1, 0x1.4000000000000p+4, 0x1.4000000000000p+3, 0x1.0000000000000p+2, 0x1.0000000000000p+0, -0x1.4000000000000p+4, 0x1.4000000000000p+3, -0x1.0000000000000p+2, 0x1.0000000000000p+0};

#define CHECK(x)                                                                             \
    do {                                                                                     \
        int rc_ = (int)(x);                                                                  \
        if (rc_) {                                                                           \
            fprintf(stderr, "%s failed: %d (%s)\n", #x, rc_, h3_error_string(rc_));         \
            return 1;                                                                        \
        }                                                                                    \
    } while (0)

/* plane wave sin(2 pi (x1 + x2 + x3)): four separable terms, (amplitude, phase) per axis */
static const double AMP[TERMS][3] = {{1, 1, 1}, {1, 1, 1}, {1, 1, 1}, {-1, 1, 1}};
static const int QUARTER[TERMS][3] = {{0, 1, 1}, {1, 0, 1}, {1, 1, 0}, {0, 0, 0}};

int main(void) {
    const double h = 1.0 / M, dt = 0.9 * h, delta = dt / 2, w = 2 * M_PI;
    const int q = 3 * (2 * N + 1);
    double fac[S], cfac[3 * (2 * N + 1)];
    for (int i = 0; i < S; ++i) fac[i] = i < S - 1 ? (i + 1) * (1.0 / h) : 0.0;
    for (int k = 1; k <= q; ++k) cfac[k - 1] = delta / k;

    /* per-axis scaled-derivative tables [term][m][j] and exact-solution tables [term][m] */
    static double tab[TERMS * M * NP], ex[TERMS * M];
    const size_t nodes = (size_t)M * M * M, dofs = nodes * NP * NP * NP;
    double *d_a, *d_b, *d_tab[3], *d_ex[3], *d_part, *d_out;
    unsigned long long* d_flag;
    CHECK(cudaMalloc((void**)&d_a, dofs * sizeof(double)));
    CHECK(cudaMalloc((void**)&d_b, dofs * sizeof(double)));
    CHECK(cudaMalloc((void**)&d_part, 2 * 256 * sizeof(double)));
    CHECK(cudaMalloc((void**)&d_out, 2 * sizeof(double)));
    CHECK(cudaMalloc((void**)&d_flag, sizeof(unsigned long long)));
    CHECK(cudaMemset(d_flag, 0xff, sizeof(unsigned long long))); /* H3_NO_BAD_NODE */
    for (int axis = 0; axis < 3; ++axis) {
        for (int t = 0; t < TERMS; ++t)
            for (int m = 0; m < M; ++m) {
                const double phase = QUARTER[t][axis] * M_PI / 2, x = m * h;
                double fact = 1.0;
                for (int j = 0; j < NP; ++j) {
                    if (j) fact *= j;
                    tab[(t * M + m) * NP + j] =
                        (pow(h, j) / fact) * AMP[t][axis] * pow(w, j) * sin(w * x + phase + j * M_PI / 2);
                }
                ex[t * M + m] = AMP[t][axis] * sin(w * fmod(x + STEPS * dt, 1.0) + phase);
            }
        CHECK(cudaMalloc((void**)&d_tab[axis], sizeof tab));
        CHECK(cudaMalloc((void**)&d_ex[axis], sizeof ex));
        CHECK(cudaMemcpy(d_tab[axis], tab, sizeof tab, cudaMemcpyHostToDevice));
        CHECK(cudaMemcpy(d_ex[axis], ex, sizeof ex, cudaMemcpyHostToDevice));
    }
    CHECK(h3_init_separable(d_a, M, M, M, N, TERMS, d_tab[0], d_tab[1], d_tab[2], NULL));

    for (int step = 0; step < STEPS; ++step) { /* primary -> dual (off 0), dual -> primary (off -1) */
        CHECK(h3_fused_pass(d_a, d_b, M, M, M, N, H, fac, fac, fac, cfac, q, 0, 0, M, 1,
                            H3_VARIANT_SEPARABLE, NULL, d_flag, NULL));
        CHECK(h3_fused_pass(d_b, d_a, M, M, M, N, H, fac, fac, fac, cfac, q, -1, 0, M, 1,
                            H3_VARIANT_SEPARABLE, NULL, d_flag, d_flag));
    }
    CHECK(h3_error_norms(d_a, M, M, M, N, TERMS, d_ex[0], d_ex[1], d_ex[2], d_part, 256, d_out, NULL));
    double norms[2];
    unsigned long long bad;
    CHECK(cudaMemcpy(norms, d_out, sizeof norms, cudaMemcpyDeviceToHost));
    CHECK(cudaMemcpy(&bad, d_flag, sizeof bad, cudaMemcpyDeviceToHost));
    const double l_inf = norms[0], l2 = sqrt(h * h * h * norms[1]), golden = 2.385797115422861e-10;
    printf("%s  N=%d %d^3 %d steps  l_inf=%.10e  l2=%.10e  (reference %.10e)\n", h3_version(), N, M, STEPS,
           l_inf, l2, golden);
    if (bad != H3_NO_BAD_NODE || fabs(l_inf / golden - 1.0) > 1e-3) {
        fprintf(stderr, "mismatch with the reference\n");
        return 1;
    }
    return 0;
}
