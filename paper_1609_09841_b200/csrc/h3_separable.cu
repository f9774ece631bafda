// Separable (node-factorised) Hermite half-step kernels -- the B200 fast path.
//
// For q >= 3(2N+1) stages the reference's local evolution is exact
// (kernels.py:30-35; pinned by the reference's
// test_exact_local_evolution_matches_shift, pkg/tests/test_kernels.py:184-199),
// so reconstruct+evolve+truncate of one cell equals the exact translation
//     out(c) = sum_{a in {0,1}^3} (A3^{a3} (x) A2^{a2} (x) A1^{a1}) u(c + off + a),
// with A_k = S_k[0:n, :] H (n x 2n), S_k[m][j] = C(j,m) (delta/h_k)^(j-m).
// Applied axis by axis that is 6 n^4 FMAs per node instead of the literal
// ~q s^3 * 8: 3 flop/B at N=3, i.e. HBM-bound on B200.
//
// sep_fused_kernel: CTA = TX x TY cells in (x1, x2), marching along x3 over a
// chunk of cell planes.  Per node plane:
//   1. the (TX+1) x (TY+1) node tile is staged into shared memory with
//      cp.async (double-buffered: plane p+1 streams in while p is computed);
//   2. pass x1 (smem -> smem): W[ly][ix] = A1^0 U[ly][ix] + A1^1 U[ly][ix+1];
//   3. pass x2 (smem -> registers) and pass x3 (registers, "register
//      rolling" across planes as in the paper): each thread owns
//      one (cell, m1) column and accumulates the two x3 contributions of the
//      plane into the finishing cell (a3 = 1) and the next cell (a3 = 0);
//   4. the finished cell plane is stored with a fused finiteness check.
// HBM traffic: each node block is read once and written once per half step
// (32 B per DOF-update); the tile halo is re-read from L2.
#include <cstdlib>
#include <cstring>

#include "h3_launch.h"

namespace h3 {

template <int N> struct SepTile;
// TX, TY: cells per CTA.  Shared-memory layouts (doubles), chosen by
// tools/smem_layout_search.py so that every hot shared access of the kernel is
// bank-conflict free (or as close as the tile allows):
//   U node [j3][j2][j1]: j3 stride UJ, node stride UNS  (staged input plane)
//   W node [j3][m1][j2]: j3 stride WJ, node stride WNS  (pass-x1 output)
template <> struct SepTile<0> { static constexpr int TX = 32, TY = 8, UJ = 1, UNS = 1, WJ = 1, WNS = 1; };
template <> struct SepTile<1> { static constexpr int TX = 16, TY = 8, UJ = 4, UNS = 8, WJ = 6, WNS = 12; };
template <> struct SepTile<2> { static constexpr int TX = 8, TY = 8, UJ = 9, UNS = 27, WJ = 12, WNS = 41; };
template <> struct SepTile<3> { static constexpr int TX = 8, TY = 8, UJ = 18, UNS = 72, WJ = 20, WNS = 82; };
template <> struct SepTile<4> { static constexpr int TX = 8, TY = 4, UJ = 25, UNS = 125, WJ = 27, WNS = 137; };
template <> struct SepTile<5> { static constexpr int TX = 8, TY = 4, UJ = 36, UNS = 216, WJ = 38, WNS = 228; };

template <int N>
struct SepGeom {
    using L = SepTile<N>;
    static constexpr int TX = L::TX, TY = L::TY;
    static constexpr int n = N + 1, n2 = n * n, n3 = n2 * n;
    static constexpr int NX = TX + 1, NY = TY + 1;
    static constexpr int UJ = L::UJ, UNS = L::UNS, WJ = L::WJ, WNS = L::WNS;
    static constexpr int THREADS = TX * TY * n;
    static constexpr int VEC = (n % 2 == 0) ? 2 : 1;    // doubles per shared vector access
    static constexpr int FVEC = (n3 % 2 == 0 && UJ % 2 == 0 && UNS % 2 == 0 && n2 % 2 == 0) ? 2 : 1;
    static constexpr int CPN = n3 / FVEC;                 // cp.async pieces per node
    static constexpr int NCOPY = NY * NX * CPN;
    static constexpr int L1 = NY * TX * n2;              // pass-x1 lines
    static constexpr int R1 = (L1 + THREADS - 1) / THREADS;
    static constexpr size_t U_DOUBLES = (size_t)NY * NX * UNS;
    static constexpr size_t W_DOUBLES = (size_t)NY * TX * WNS;
    static constexpr size_t SMEM = (2 * U_DOUBLES + W_DOUBLES) * sizeof(double) + NY * NX * sizeof(int);
};

template <int CNT, int VEC>
__device__ __forceinline__ void lds_vec(double (&dst)[CNT], const double* src) {
    if constexpr (VEC == 2) {
#pragma unroll
        for (int j = 0; j < CNT; j += 2) {
            const double2 v = *reinterpret_cast<const double2*>(src + j);
            dst[j] = v.x;
            dst[j + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int j = 0; j < CNT; ++j) dst[j] = src[j];
    }
}

template <int N>
__global__ void __launch_bounds__(SepGeom<N>::THREADS)
sep_fused_kernel(const double* __restrict__ src, double* __restrict__ dst, Dims d, int off,
                 int zchunk, const __grid_constant__ SepOps<N> p,
                 unsigned long long* first_bad, const unsigned long long* guard) {
    using G = SepGeom<N>;
    constexpr int TX = G::TX, n = G::n, n2 = G::n2, n3 = G::n3, NX = G::NX;
    constexpr int UJ = G::UJ, UNS = G::UNS, WJ = G::WJ, WNS = G::WNS;
    if (guarded_out(guard, first_bad)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* U0 = reinterpret_cast<double*>(smem_raw);
    double* U1 = U0 + G::U_DOUBLES;
    double* W = U1 + G::U_DOUBLES;

    const int tid = threadIdx.x;
    const int M1 = (int)d.M1, M2 = (int)d.M2;
    const int cx0 = blockIdx.x * TX, cy0 = blockIdx.y * G::TY;
    const int64_t zc0 = d.z_begin + (int64_t)blockIdx.z * zchunk;
    const int64_t zc1 = min(zc0 + (int64_t)zchunk, d.z_end);
    const int P = (int)(zc1 - zc0) + 1;  // node planes touched by this chunk
    const int64_t plane_elems = (int64_t)M1 * M2 * n3;

    // Global offset (doubles, relative to the plane base) of every tile node: the
    // periodic wrap is resolved once per CTA, so the per-plane copy loop is just
    // table lookup + LDGSTS.
    int* nodeoff = reinterpret_cast<int*>(W + G::W_DOUBLES);
    for (int node = tid; node < G::NY * NX; node += G::THREADS) {
        const int ly = node / NX, lx = node - (node / NX) * NX;
        int gx = cx0 + off + lx, gy = cy0 + off + ly;
        gx %= M1; if (gx < 0) gx += M1;
        gy %= M2; if (gy < 0) gy += M2;
        nodeoff[node] = (gy * M1 + gx) * n3;
    }
    __syncthreads();

    auto issue = [&](int pl, double* Ub) {
        const int64_t gz = zplane(zc0 + off + pl, d.M3, d.periodic_z);
        const double* base = src + gz * plane_elems;
        if constexpr (G::THREADS % G::CPN == 0) {
            // each thread always copies the same piece of successive nodes
            constexpr int STEP = G::THREADS / G::CPN;
            const int pc = tid % G::CPN;
            const int dbl = pc * G::FVEC;
            const int soff = (dbl / n2) * UJ + dbl % n2;
#pragma unroll 4
            for (int node = tid / G::CPN; node < G::NY * NX; node += STEP) {
                const double* g = base + nodeoff[node] + dbl;
                double* sp = Ub + node * UNS + soff;
                if (G::FVEC == 2) cp_async16(sp, g); else cp_async8(sp, g);
            }
        } else {
            for (int e = tid; e < G::NCOPY; e += G::THREADS) {
                const int node = e / G::CPN;
                const int dbl = (e - node * G::CPN) * G::FVEC;
                const double* g = base + nodeoff[node] + dbl;
                double* sp = Ub + node * UNS + (dbl / n2) * UJ + dbl % n2;
                if (G::FVEC == 2) cp_async16(sp, g); else cp_async8(sp, g);
            }
        }
    };

    // pass x2/x3 ownership: (m1, ix, iy)
    const int m1 = tid % n;
    const int ix = (tid / n) % TX;
    const int iy = tid / (n * TX);
    const int cx = cx0 + ix, cy = cy0 + iy;
    const bool owns = (cx < M1) && (cy < M2);

    double accP[n][n];  // cell finishing at this plane (a3 = 1 contribution pending)
#pragma unroll
    for (int a = 0; a < n; ++a)
#pragma unroll
        for (int b = 0; b < n; ++b) accP[a][b] = 0.0;

    issue(0, U0);
    cp_async_commit();
    for (int pl = 0; pl < P; ++pl) {
        const double* Ub = (pl & 1) ? U1 : U0;
        if (pl + 1 < P) issue(pl + 1, (pl & 1) ? U0 : U1);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();

        // ---- pass x1: W[ly][ix][j3][m1][j2] = A1^0 U[ly][ix] + A1^1 U[ly][ix+1] ------------
#pragma unroll
        for (int r = 0; r < G::R1; ++r) {
            const int l = tid + r * G::THREADS;
            if (G::L1 % G::THREADS == 0 || l < G::L1) {
                const int j32 = l % n2;
                const int rest = l / n2;
                const int lix = rest % TX, ly = rest / TX;
                const int j3 = j32 / n, j2 = j32 - (j32 / n) * n;
                const double* u0 = Ub + (ly * NX + lix) * UNS + j3 * UJ + j2 * n;
                double a[n], b[n];
                lds_vec<n, G::VEC>(a, u0);
                lds_vec<n, G::VEC>(b, u0 + UNS);
                double* wout = W + (ly * TX + lix) * WNS + j3 * WJ + j2;
#pragma unroll
                for (int m = 0; m < n; ++m) {
                    double acc = p.A[0][m][0] * a[0];
#pragma unroll
                    for (int j = 1; j < n; ++j) acc = fma(p.A[0][m][j], a[j], acc);
#pragma unroll
                    for (int j = 0; j < n; ++j) acc = fma(p.A[0][m][n + j], b[j], acc);
                    wout[m * n] = acc;
                }
            }
        }
        __syncthreads();

        // ---- pass x2 + x3 ----------------------------------------------------------------
        {
            const double* w0 = W + (iy * TX + ix) * WNS + m1 * n;
            const double* w1 = w0 + TX * WNS;
            double accN[n][n];
#pragma unroll
            for (int j3 = 0; j3 < n; ++j3) {
                double a[n], b[n];
                lds_vec<n, G::VEC>(a, w0 + j3 * WJ);
                lds_vec<n, G::VEC>(b, w1 + j3 * WJ);
                double v[n];
#pragma unroll
                for (int m = 0; m < n; ++m) {
                    double acc = p.A[1][m][0] * a[0];
#pragma unroll
                    for (int j = 1; j < n; ++j) acc = fma(p.A[1][m][j], a[j], acc);
#pragma unroll
                    for (int j = 0; j < n; ++j) acc = fma(p.A[1][m][n + j], b[j], acc);
                    v[m] = acc;
                }
#pragma unroll
                for (int m3 = 0; m3 < n; ++m3)
#pragma unroll
                    for (int m2 = 0; m2 < n; ++m2) {
                        accP[m3][m2] = fma(p.A[2][m3][n + j3], v[m2], accP[m3][m2]);
                        accN[m3][m2] = j3 == 0 ? p.A[2][m3][0] * v[m2]
                                               : fma(p.A[2][m3][j3], v[m2], accN[m3][m2]);
                    }
            }
            if (pl > 0 && owns) {
                const int64_t c3 = zc0 + pl - 1;
                const int64_t node = (c3 * M2 + cy) * (int64_t)M1 + cx;
                double* o = dst + node * n3 + m1;
                bool bad = false;
#pragma unroll
                for (int m3 = 0; m3 < n; ++m3)
#pragma unroll
                    for (int m2 = 0; m2 < n; ++m2) {
                        o[(m3 * n + m2) * n] = accP[m3][m2];
                        bad |= !isfinite(accP[m3][m2]);
                    }
                if (bad) flag_bad(first_bad, node);
            }
#pragma unroll
            for (int a = 0; a < n; ++a)
#pragma unroll
                for (int b = 0; b < n; ++b) accP[a][b] = accN[a][b];
        }
        __syncthreads();
    }
}

template <int N>
static int sep_fused_n(const double* src, double* dst, const Dims& d, const double* A, int off,
                       cudaStream_t st, unsigned long long* first_bad,
                       const unsigned long long* guard) {
    using G = SepGeom<N>;
    const int64_t nz = d.z_end - d.z_begin;
    if (nz <= 0 || d.M1 <= 0 || d.M2 <= 0) return 0;
    if (d.M1 * d.M2 * G::n3 >= (int64_t(1) << 31)) return (int)cudaErrorInvalidValue;  // int32 plane offsets
    SepOps<N> ops;
    for (int k = 0; k < 3; ++k)
        for (int m = 0; m < G::n; ++m)
            for (int c = 0; c < 2 * G::n; ++c) {
                ops.A[k][m][c] = A[(k * G::n + m) * 2 * G::n + c];
                ops.Sh[k][m][c] = 0.0;
            }
    auto kern = sep_fused_kernel<N>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM);
    if (e != cudaSuccess) return (int)e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, G::THREADS, G::SMEM);
    if (e != cudaSuccess) return (int)e;
    const int64_t gx = (d.M1 + G::TX - 1) / G::TX, gy = (d.M2 + G::TY - 1) / G::TY;
    // enough CTAs for ~4 waves; split the z march only when the x-y tiling is too coarse
    const int64_t zchunk = choose_zchunk(gx * gy, nz, (int64_t)num_sms() * (per_sm > 0 ? per_sm : 1));
    const int64_t gz = (nz + zchunk - 1) / zchunk;
    dim3 grid((unsigned)gx, (unsigned)gy, (unsigned)gz);
    kern<<<grid, G::THREADS, G::SMEM, st>>>(src, dst, d, off, (int)zchunk, ops, first_bad, guard);
    return (int)cudaGetLastError();
}

// H3_FUSED_IMPL=dfma runs the DFMA kernel at N = 3, 5 too: only in the tools library
// (-DH3_MEASURE), which backs the "DMMA only where ncu shows compute-bound" comparison.
#ifdef H3_MEASURE
static bool use_dfma_ab() {
    static const bool v = [] {
        const char* e = getenv("H3_FUSED_IMPL");
        return e && strcmp(e, "dfma") == 0;
    }();
    return v;
}
#endif

int sep_fused_launch(const double* src, double* dst, const Dims& d, int order_n, const double* A,
                     int off, cudaStream_t st, unsigned long long* first_bad,
                     const unsigned long long* guard) {
    switch (order_n) {
        case 0: return sep_fused_n<0>(src, dst, d, A, off, st, first_bad, guard);
        case 1: return sep_fused_n<1>(src, dst, d, A, off, st, first_bad, guard);
        case 2: return sep_fused_n<2>(src, dst, d, A, off, st, first_bad, guard);
        case 3:
            // FP64 tensor-core kernel (h3_dmma.cu); the DFMA kernel is the tools library's A/B
#ifdef H3_MEASURE
            if (use_dfma_ab()) return sep_fused_n<3>(src, dst, d, A, off, st, first_bad, guard);
#endif
            return sep_fused_dmma3_launch(src, dst, d, A, off, st, first_bad, guard);
        case 4: return sep_fused_n<4>(src, dst, d, A, off, st, first_bad, guard);
        case 5:
            // FP64 tensor-core cell-pair kernel (h3_dmma5.cu)
#ifdef H3_MEASURE
            if (use_dfma_ab()) return sep_fused_n<5>(src, dst, d, A, off, st, first_bad, guard);
#endif
            return sep_fused_dmma5_launch(src, dst, d, A, off, st, first_bad, guard);
    }
    return (int)cudaErrorInvalidValue;
}

// ---------------------------------------------------------------------------------------
// Separable evolution of a materialised coefficient field (two-kernel fast path):
// out[m3][m2][m1] = sum S3[m3][i3] S2[m2][i2] S1[m1][i1] coeff[i3][i2][i1], applied axis by
// axis (s^3 n + s^2 n^2 + s n^3 FMAs per cell).  S_k are the exact shift rows of
// exp(delta d/dx_k); equal to the reference's q-stage Horner for q >= 3(2N+1).
//
// Streaming design: one CTA per group of CPB consecutive cells; one thread per
// (cell, x1-line) reads its s contiguous coefficients straight from HBM into registers
// (16-B loads; a warp reads 2 KB contiguous), contracts them to n values (pass x1), and the
// small x2/x3 passes run through shared memory.  Many small CTAs per SM keep the loads
// in flight.
template <int N>
constexpr int ev_cpb() { return (2 * N + 2) * (2 * N + 2) >= 256 ? 1 : 256 / ((2 * N + 2) * (2 * N + 2)); }

template <int N, int CPB, int GPC>
__global__ void __launch_bounds__(CPB*(2 * N + 2) * (2 * N + 2))
sep_evolve_kernel(const double* __restrict__ coeff, double* __restrict__ dst, Dims d,
                  const __grid_constant__ SepOps<N> p, unsigned long long* first_bad,
                  const unsigned long long* guard) {
    constexpr int n = N + 1, S = 2 * n, S2 = S * S, S3 = S2 * S, n2 = n * n, n3 = n2 * n;
    constexpr int THREADS = CPB * S2;
    // shared layouts T1[c][i3][i2][m1] = c T1S + i3 A3 + i2 A2 + m1 and T2[c][i3][m2][m1] =
    // c T2S + i3 B3 + m2 B2 + m1; at N = 3 the strides come from tools/evolve_layout_search.py
    // (64 instead of 168 shared wavefronts per cell: every x1 store and x3 load conflict-free)
    constexpr int A2 = N == 3 ? 5 : n, A3 = N == 3 ? 40 : S * n;
    constexpr int B2 = n, B3 = N == 3 ? 20 : n2;
    constexpr int T1S = S * A3 + 1;  // per-cell strides (odd: spreads banks across cells)
    constexpr int T2S = S * B3 + 1;
    __shared__ double T1[CPB * T1S];  // [c][i3][i2][m1]
    __shared__ double T2[CPB * T2S];  // [c][i3][m2][m1]

    const int64_t nxy = d.M1 * d.M2;
    const int64_t total = (d.z_end - d.z_begin) * nxy;
    const int64_t groups = (total + CPB - 1) / CPB;
    const int tid = threadIdx.x;
    const int c = tid / S2, line = tid - (tid / S2) * S2;  // x1 task: (cell, line (i3, i2))

    // GPC consecutive groups per CTA, all loads issued up front (the later groups' loads are
    // in flight while the earlier ones are contracted), then the guard read (overlapped too)
    double u[GPC][S];
#pragma unroll
    for (int gi = 0; gi < GPC; ++gi) {
        const int64_t grp = (int64_t)blockIdx.x * GPC + gi;
        const int64_t cell = grp * CPB + c;
        if (grp < groups && cell < total) {
            const double2* g2 = reinterpret_cast<const double2*>(coeff + cell * S3 + line * S);
#pragma unroll
            for (int k = 0; k < S / 2; ++k) {
                const double2 v = __ldcs(g2 + k);
                u[gi][2 * k] = v.x;
                u[gi][2 * k + 1] = v.y;
            }
        } else {
#pragma unroll
            for (int k = 0; k < S; ++k) u[gi][k] = 0.0;
        }
    }
    if (guarded_out(guard, first_bad)) return;
#pragma unroll
    for (int gi = 0; gi < GPC; ++gi) {
        const int64_t grp = (int64_t)blockIdx.x * GPC + gi;
        if (grp >= groups) break;
        if (gi > 0) __syncthreads();  // T1/T2 reuse
        // pass x1 (registers): T1[c][i3][i2][m1] = sum_i1 S1[m1][i1] u[i1]
#pragma unroll
        for (int m = 0; m < n; ++m) {
            double acc = p.Sh[0][m][0] * u[gi][0];
#pragma unroll
            for (int k = 1; k < S; ++k) acc = fma(p.Sh[0][m][k], u[gi][k], acc);
            T1[c * T1S + (line / S) * A3 + (line % S) * A2 + m] = acc;
        }
        __syncthreads();
        // pass x2: (c, i3, m1) -> n outputs m2
        for (int l = tid; l < CPB * S * n; l += THREADS) {
            const int cc = l / (S * n), r = l - cc * (S * n), i3 = r / n, mm1 = r - (r / n) * n;
            double a[S];
#pragma unroll
            for (int k = 0; k < S; ++k) a[k] = T1[cc * T1S + i3 * A3 + k * A2 + mm1];
#pragma unroll
            for (int m = 0; m < n; ++m) {
                double acc = p.Sh[1][m][0] * a[0];
#pragma unroll
                for (int k = 1; k < S; ++k) acc = fma(p.Sh[1][m][k], a[k], acc);
                T2[cc * T2S + i3 * B3 + m * B2 + mm1] = acc;
            }
        }
        __syncthreads();
        // pass x3: (c, m2, m1) -> n outputs m3, stored to the destination node
        for (int l = tid; l < CPB * n2; l += THREADS) {
            const int cc = l / n2, r = l - cc * n2;
            const int64_t cell = grp * CPB + cc;
            if (cell >= total) continue;
            double a[S];
#pragma unroll
            for (int k = 0; k < S; ++k) a[k] = T2[cc * T2S + k * B3 + r];
            const int64_t crel3 = cell / nxy, rem = cell - crel3 * nxy;
            const int64_t node = ((d.z_begin + crel3) * d.M2 + rem / d.M1) * d.M1 + rem % d.M1;
            double* o = dst + node * n3 + r;
            bool bad = false;
#pragma unroll
            for (int m = 0; m < n; ++m) {
                double acc = p.Sh[2][m][0] * a[0];
#pragma unroll
                for (int k = 1; k < S; ++k) acc = fma(p.Sh[2][m][k], a[k], acc);
                __stcs(o + m * n2, acc);
                bad |= !isfinite(acc);
            }
            if (bad) flag_bad(first_bad, node);
        }
    }
}


template <int N, int CPB, int GPC = 1>
static int sep_evolve_nc(const double* coeff, double* dst, const Dims& d, const double* Sh,
                        cudaStream_t st, unsigned long long* first_bad,
                        const unsigned long long* guard) {
    constexpr int n = N + 1, S = 2 * n, S2 = S * S;
    const int64_t total = (d.z_end - d.z_begin) * d.M1 * d.M2;
    if (total <= 0) return 0;
    SepOps<N> ops;
    for (int k = 0; k < 3; ++k)
        for (int m = 0; m < n; ++m)
            for (int c = 0; c < S; ++c) {
                ops.Sh[k][m][c] = Sh[(k * n + m) * S + c];
                ops.A[k][m][c] = 0.0;
            }
    auto kern = sep_evolve_kernel<N, CPB, GPC>;
    const int64_t groups = (total + CPB - 1) / CPB;
    kern<<<(unsigned)((groups + GPC - 1) / GPC), CPB * S2, 0, st>>>(coeff, dst, d, ops, first_bad, guard);
    return (int)cudaGetLastError();
}

template <int N>
static int sep_evolve_n(const double* coeff, double* dst, const Dims& d, const double* Sh,
                        cudaStream_t st, unsigned long long* first_bad,
                        const unsigned long long* guard) {
    if constexpr (N == 3) {
#ifdef H3_MEASURE
        static const int cpb = [] {  // tools library only: cells per CTA for A/B runs
            const char* e = getenv("H3_EVOLVE_CPB");
            return e ? atoi(e) : 0;
        }();
        if (cpb == 4) return sep_evolve_nc<3, 4>(coeff, dst, d, Sh, st, first_bad, guard);
        if (cpb == 2) return sep_evolve_nc<3, 2>(coeff, dst, d, Sh, st, first_bad, guard);
        if (cpb == 42) return sep_evolve_nc<3, 4, 2>(coeff, dst, d, Sh, st, first_bad, guard);
        if (cpb == 8) return sep_evolve_nc<3, 8>(coeff, dst, d, Sh, st, first_bad, guard);
#endif
        // one cell (64 threads) per CTA: 32 independent CTAs per SM overlap their load and
        // contraction phases best (measured 4.7 vs 4.2 TB/s for 2-8 cells per CTA)
        return sep_evolve_nc<3, 1>(coeff, dst, d, Sh, st, first_bad, guard);
    }
    return sep_evolve_nc<N, ev_cpb<N>()>(coeff, dst, d, Sh, st, first_bad, guard);
}

int sep_evolve_launch(const double* coeff, double* dst, const Dims& d, int order_n,
                      const double* Sh, cudaStream_t st, unsigned long long* first_bad,
                      const unsigned long long* guard) {
    switch (order_n) {
        case 0: return sep_evolve_n<0>(coeff, dst, d, Sh, st, first_bad, guard);
        case 1: return sep_evolve_n<1>(coeff, dst, d, Sh, st, first_bad, guard);
        case 2: return sep_evolve_n<2>(coeff, dst, d, Sh, st, first_bad, guard);
        case 3: return sep_evolve_n<3>(coeff, dst, d, Sh, st, first_bad, guard);
        case 4: return sep_evolve_n<4>(coeff, dst, d, Sh, st, first_bad, guard);
        case 5: return sep_evolve_n<5>(coeff, dst, d, Sh, st, first_bad, guard);
    }
    return (int)cudaErrorInvalidValue;
}

}  // namespace h3
