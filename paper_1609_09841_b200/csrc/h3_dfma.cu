// FP64-FMA (DFMA) node-factorised kernels whose operators live in the CONSTANT bank.
//
// The per-axis operators (H for reconstruction) are small dense matrices used as one operand of
// every DFMA.  Passed as kernel parameters, the compiler hoists all of them into registers
// (144 doubles at N = 5) and spills; here they sit in a __constant__ ring (h3_cops.cuh) and
// each use is a `ld.const` with an immediate address that ptxas turns into a uniform-register
// operand (LDCU.128 feeds two DFMAs), so the registers hold only data.
//
// recon_sep_kernel: reconstruction pass of the two-kernel step, any order.
//   coeff(c)[i3][i2][i1] = sum_a (H^a3 (x) H^a2 (x) H^a1) u(c + off + a),  H^a = H[:, a n : a n + n]
// (gridkernels.py:58-83 computes the same tensor by three dense H sweeps of the gathered s^3
// block, 3 s^4 MACs per cell).  Applied axis by axis on the nodes of a tile it costs
// 2 s n^3 + 2 s^2 n^2 + 2 s^3 n MACs per cell (36,288 instead of 62,208 at N = 5, SURVEY
// Appendix B), and the coefficient field -- 89 % of the two-kernel traffic at N = 5 -- is
// written exactly once with coalesced streaming stores.
//
// CTA = TX x TY cells in (x1, x2) marching along x3 over a chunk of cell planes.  Per node
// plane (staged with cp.async, STAGES-deep ring):
//   x1: line (node row ly, cell cx, j3, j2): W = H^0 u(ly, cx) + H^1 u(ly, cx + 1)     [s outputs]
//   x2: line (cell cy, cell cx, j3, i1):    V = H^0 W(cy) + H^1 W(cy + 1)             [s outputs]
//   x3: each thread owns K3 columns (cell, i2, i1) across planes ("register rolling",
//       PAPER.md:147): the pending cell (node plane p is its right vertex) completes with
//       H^1 V and is stored; the next cell starts with H^0 V.
#include "h3_cops.cuh"
#include "h3_launch.h"

namespace h3 {

template <int N> struct RcTile;
//                                  TX  TY  THREADS  MINB
template <> struct RcTile<0> { static constexpr int TX = 16, TY = 8, THREADS = 256, MINB = 4; };
template <> struct RcTile<1> { static constexpr int TX = 8, TY = 8, THREADS = 256, MINB = 2; };
template <> struct RcTile<2> { static constexpr int TX = 8, TY = 4, THREADS = 384, MINB = 1; };
template <> struct RcTile<3> { static constexpr int TX = 8, TY = 4, THREADS = 512, MINB = 1; };
template <> struct RcTile<4> { static constexpr int TX = 4, TY = 2, THREADS = 800, MINB = 1; };
template <> struct RcTile<5> { static constexpr int TX = 4, TY = 2, THREADS = 384, MINB = 1; };

template <int N>
struct RcGeom {
    using T = RcTile<N>;
    static constexpr int n = N + 1, n2 = n * n, n3 = n2 * n, S = 2 * n, S2 = S * S, S3 = S2 * S;
    static constexpr int TX = T::TX, TY = T::TY, NX = TX + 1, NY = TY + 1, NNODE = NX * NY;
    static constexpr int THREADS = T::THREADS, MINB = T::MINB, STAGES = 3;
    static constexpr bool V16 = (n3 % 2) == 0;   // node blocks 16-B aligned: 16-B copies
    static constexpr int UNS = n3;               // U node stride (dense, = global block)
    static constexpr int WI = n2 | 1;            // W [cell][i1][j3 j2]: odd i1 stride
    static constexpr int WCS = S * WI;
    static constexpr int VJ = S2, VCS = n * VJ;  // V [cell][j3][i2 i1]
    static constexpr int L1 = NY * TX * n2;      // x1 lines
    static constexpr int L2 = TY * TX * n * S;   // x2 lines
    static constexpr int COLS = TY * TX * S2;    // x3 columns
    static constexpr int K3 = COLS / THREADS;
    static_assert(COLS % THREADS == 0, "x3 columns must divide evenly among threads");
    static constexpr int PIECES = NNODE * n3 / (V16 ? 2 : 1);
    static constexpr size_t U_D = (size_t)NNODE * UNS;
    static constexpr size_t W_D = (size_t)NY * TX * WCS;
    static constexpr size_t V_D = (size_t)TY * TX * VCS;
    static constexpr size_t SMEM = (STAGES * U_D + W_D + V_D) * sizeof(double) + NNODE * sizeof(int);
};

// c = sum_{j < K} H[row][col0 + j] * a[j], H row-major with S columns at constant offset HB
template <int HB, int S, int ROW, int COL0, int K, class A>
__device__ __forceinline__ double cdot(const A& a) {
    double c = cop<HB + ROW * S + COL0>() * a[0];
    sfor<K - 1>([&](auto jm) {
        constexpr int j = decltype(jm)::value + 1;
        c = fma(cop<HB + ROW * S + COL0 + j>(), a[j], c);
    });
    return c;
}
template <int HB, int S, int ROW, int COL0, int K, class A>
__device__ __forceinline__ double cdot_acc(double c, const A& a) {
    sfor<K>([&](auto jj) {
        constexpr int j = decltype(jj)::value;
        c = fma(cop<HB + ROW * S + COL0 + j>(), a[j], c);
    });
    return c;
}

template <int N, int SLOT>
__global__ void __launch_bounds__(RcGeom<N>::THREADS, RcGeom<N>::MINB)
recon_sep_kernel(const double* __restrict__ src, double* __restrict__ coeff, Dims d, int off,
                 int zchunk, const unsigned long long* guard) {
    using G = RcGeom<N>;
    constexpr int n = G::n, n2 = G::n2, n3 = G::n3, S = G::S, S2 = G::S2, S3 = G::S3;
    constexpr int TX = G::TX, NX = G::NX, THREADS = G::THREADS, STAGES = G::STAGES;
    constexpr int UNS = G::UNS, WI = G::WI, WCS = G::WCS, VJ = G::VJ, VCS = G::VCS, K3 = G::K3;
    constexpr int HB = SLOT * COP_SLOT;  // H (S x S, row-major) in the constant ring
    if (guarded_out(guard, nullptr)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* U = reinterpret_cast<double*>(smem_raw);
    double* W = U + STAGES * G::U_D;
    double* V = W + G::W_D;
    int* nodeoff = reinterpret_cast<int*>(V + G::V_D);

    const int tid = threadIdx.x;
    const int M1 = (int)d.M1, M2 = (int)d.M2;
    const int cx0 = blockIdx.x * TX, cy0 = blockIdx.y * G::TY;
    const int64_t zc0 = d.z_begin + (int64_t)blockIdx.z * zchunk;
    const int64_t zc1 = min(zc0 + (int64_t)zchunk, d.z_end);
    const int P = (int)(zc1 - zc0) + 1;  // node planes touched by this chunk
    const int64_t plane_elems = (int64_t)M1 * M2 * n3;
    const int64_t cplane = (int64_t)M1 * M2 * S3;

    // global offset (doubles, within a node plane) of every tile node, periodic in x1/x2
    for (int node = tid; node < G::NNODE; node += THREADS) {
        const int ly = node / NX, lx = node - (node / NX) * NX;
        int gx = cx0 + off + lx, gy = cy0 + off + ly;
        gx %= M1; if (gx < 0) gx += M1;
        gy %= M2; if (gy < 0) gy += M2;
        nodeoff[node] = (gy * M1 + gx) * n3;
    }
    __syncthreads();

    int64_t gz_next = d.periodic_z ? wrap(zc0 + off, d.M3) : zc0 + off;
    int issued = 0;
    auto issue = [&]() {
        if (issued < P) {
            const double* base = plane_base(src, gz_next, plane_elems, d);
            double* Ub = U + (issued % STAGES) * G::U_D;
            constexpr int PER = G::V16 ? 2 : 1, PPN = n3 / PER;  // pieces per node
#pragma unroll 1
            for (int e = tid; e < G::PIECES; e += THREADS) {
                const int node = e / PPN, k = (e - node * PPN) * PER;
                if (G::V16) cp_async16(Ub + node * UNS + k, base + nodeoff[node] + k);
                else cp_async8(Ub + node * UNS + k, base + nodeoff[node] + k);
            }
            ++gz_next;
            if (d.periodic_z && gz_next == d.M3) gz_next = 0;
            ++issued;
        }
        cp_async_commit();
    };
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) issue();

    // x3 columns owned by this thread: col = tid + THREADS k -> (cell, r = i2 s + i1)
    int64_t cbase[K3];
    int vbase[K3];
#pragma unroll
    for (int k = 0; k < K3; ++k) {
        const int col = tid + THREADS * k;
        const int cell = col / S2, r = col - (col / S2) * S2;
        const int cx = cx0 + cell % TX, cy = cy0 + cell / TX;
        vbase[k] = cell * VCS + r;
        cbase[k] = (cx < M1 && cy < M2)
                       ? ((zc0 - d.z_begin) * M2 * (int64_t)M1 + (int64_t)cy * M1 + cx) * S3 + r
                       : -1;
    }
    double acc[K3][S];
#pragma unroll
    for (int k = 0; k < K3; ++k)
#pragma unroll
        for (int i = 0; i < S; ++i) acc[k][i] = 0.0;

#pragma unroll 1
    for (int pl = 0; pl < P; ++pl) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        issue();  // refills the stage read in the previous iteration (all threads passed the barrier)
        const double* Ub = U + (pl % STAGES) * G::U_D;

        // ---- x1: line (ly, cx, j3 j2) -> W[ly][cx][i1][j3 j2] ---------------------------------
#pragma unroll 1
        for (int l = tid; l < G::L1; l += THREADS) {
            const int jj = l % n2, rest = l / n2;
            const int cx = rest % TX, ly = rest / TX;
            const double* ua = Ub + (ly * NX + cx) * UNS + jj * n;
            double a[2 * n];
#pragma unroll
            for (int j = 0; j < n; ++j) {
                a[j] = ua[j];
                a[n + j] = ua[UNS + j];
            }
            double* w = W + (ly * TX + cx) * WCS + jj;
            sfor<S>([&](auto ii) {
                constexpr int i = decltype(ii)::value;
                w[i * WI] = cdot<HB, S, i, 0, S>(a);
            });
        }
        __syncthreads();

        // ---- x2: line (cy, cx, j3, i1) -> V[cell][j3][i2][i1] ---------------------------------
#pragma unroll 1
        for (int l = tid; l < G::L2; l += THREADS) {
            const int i1 = l % S, rest = l / S;
            const int j3 = rest % n, cell = rest / n;  // cell = cy TX + cx
            const double* wa = W + cell * WCS + i1 * WI + j3 * n;
            double a[2 * n];
#pragma unroll
            for (int j = 0; j < n; ++j) {
                a[j] = wa[j];
                a[n + j] = wa[TX * WCS + j];
            }
            double* v = V + cell * VCS + j3 * VJ + i1;
            sfor<S>([&](auto ii) {
                constexpr int i = decltype(ii)::value;
                v[i * S] = cdot<HB, S, i, 0, S>(a);
            });
        }
        __syncthreads();

        // ---- x3: columns across planes; the completed cell plane goes straight to HBM --------
        {
            const int64_t plane_off = (int64_t)(pl - 1) * cplane;
#pragma unroll
            for (int k = 0; k < K3; ++k) {
                double v[n];
#pragma unroll
                for (int j = 0; j < n; ++j) v[j] = V[vbase[k] + j * VJ];
                if (pl > 0 && cbase[k] >= 0) {
                    double* o = coeff + cbase[k] + plane_off;
                    sfor<S>([&](auto ii) {
                        constexpr int i = decltype(ii)::value;
                        __stcs(o + i * S2, cdot_acc<HB, S, i, n, n>(acc[k][i], v));
                    });
                }
                sfor<S>([&](auto ii) {
                    constexpr int i = decltype(ii)::value;
                    acc[k][i] = cdot<HB, S, i, 0, n>(v);
                });
            }
        }
    }
    cp_async_wait<0>();
}

template <int N, int SLOT>
static int recon_sep_ns(const double* src, double* coeff, const Dims& d, int off, cudaStream_t st,
                        const unsigned long long* guard) {
    using G = RcGeom<N>;
    const int64_t nz = d.z_end - d.z_begin;
    auto kern = recon_sep_kernel<N, SLOT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM);
    if (e != cudaSuccess) return (int)e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, G::THREADS, G::SMEM);
    if (e != cudaSuccess) return (int)e;
    const int64_t gx = (d.M1 + G::TX - 1) / G::TX, gy = (d.M2 + G::TY - 1) / G::TY;
    const int64_t zchunk = choose_zchunk(gx * gy, nz, (int64_t)num_sms() * (per_sm > 0 ? per_sm : 1));
    const int64_t gz = (nz + zchunk - 1) / zchunk;
    kern<<<dim3((unsigned)gx, (unsigned)gy, (unsigned)gz), G::THREADS, G::SMEM, st>>>(
        src, coeff, d, off, (int)zchunk, guard);
    return (int)cudaGetLastError();
}

template <int N>
static int recon_sep_n(const double* src, double* coeff, const Dims& d, const double* h_mat, int off,
                       cudaStream_t st, const unsigned long long* guard) {
    using G = RcGeom<N>;
    if (d.z_end - d.z_begin <= 0) return 0;
    if (d.M1 * d.M2 * G::n3 >= (int64_t(1) << 31)) return (int)cudaErrorInvalidValue;  // int32 plane offsets
    int slot = 0;
    int rc = cop_acquire(h_mat, G::S2, st, &slot);
    if (rc) return rc;
    switch (slot) {
        case 0: rc = recon_sep_ns<N, 0>(src, coeff, d, off, st, guard); break;
        case 1: rc = recon_sep_ns<N, 1>(src, coeff, d, off, st, guard); break;
        case 2: rc = recon_sep_ns<N, 2>(src, coeff, d, off, st, guard); break;
        default: rc = recon_sep_ns<N, 3>(src, coeff, d, off, st, guard); break;
    }
    const int rc2 = cop_release(slot, st);
    return rc ? rc : rc2;
}

int recon_sep_launch(const double* src, double* coeff, const Dims& d, int order_n, const double* h_mat,
                     int off, cudaStream_t st, const unsigned long long* guard) {
    switch (order_n) {
        case 0: return recon_sep_n<0>(src, coeff, d, h_mat, off, st, guard);
        case 1: return recon_sep_n<1>(src, coeff, d, h_mat, off, st, guard);
        case 2: return recon_sep_n<2>(src, coeff, d, h_mat, off, st, guard);
        case 4: return recon_sep_n<4>(src, coeff, d, h_mat, off, st, guard);
#ifdef H3_MEASURE
        // N = 3, 5 reconstruct on the FP64 tensor cores (h3_dmma.cu, h3_dmma5.cu); the DFMA
        // kernels for them are A/B references of the tools library (H3_RECON_IMPL=sep)
        case 3: return recon_sep_n<3>(src, coeff, d, h_mat, off, st, guard);
        case 5: return recon_sep_n<5>(src, coeff, d, h_mat, off, st, guard);
#endif
    }
    return (int)cudaErrorInvalidValue;
}

// ---------------------------------------------------------------------------------------------
// (constant-operator ring: h3_cops.cuh)
// sets; a kernel is instantiated per slot so every operator read is an immediate constant-bank
// address.  Identical operator sets share a slot; a slot is only overwritten after every kernel
// that used it has completed (the overwriting stream waits on their events), so concurrent
// streams with different operators stay correct.
// ---------------------------------------------------------------------------------------------


}  // namespace h3
