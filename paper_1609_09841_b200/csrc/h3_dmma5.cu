// FP64 tensor-core (DMMA m8n8k4) fused half step for orders with 2n % 4 == 0 (N = 5: n = 6).
//
// Same exact separable local evolution as the other fused kernels,
//     out(c) = sum_a (A3^a3 (x) A2^a2 (x) A1^a1) u(c + off + a),
// applied as three 1-D passes, but in "cell-pair" form: a line of a pass gathers its cell's two
// vertex blocks (2n = 12 inputs, both nodes along the pass axis) and contracts them with
// [A^0 | A^1] (n x 2n) into the cell's n outputs.  As a GEMM: D[line][m] = sum_k X[line][k] B[k][m]
// with K = 2n = 12 = three m8n8k4 k-steps and N = n = 6 of the 8 columns (75 % of the MMA is
// useful).  The alternative, node-factorised form (K = n = 6, N = 2n = 12) would fill only
// 56 %; DFMA with the operators in registers spills (255 registers, 36 % of HBM measured).
// Nothing is carried between MMAs, so there is no per-lane bookkeeping: every pass is
// "3 x LDS, 3 x DMMA, 2 x store" per 8 lines.
//
// CTA = TX x TY cells in (x1, x2), 16 warps, marching along x3 over a chunk of cell planes.
// Per node plane p (staged by TMA bulk row copies, 3-stage mbarrier ring):
//   x1: line (node row ly, cell cx, j3 j2)   U(p) -> W[ly][cx][m1][j3 j2]
//   x2: line (cell, j3, m1)                  W    -> V[p & 1][cell][j3][m2 m1]
//   x3: line (cell, m2 m1), planes p-1 and p V[(p-1) & 1], V[p & 1] -> dst (cell plane p-1)
// V is double-buffered so x3 pairs the planes without a register accumulator.
#include <cstdlib>

#include "h3_launch.h"
#include "h3_tma.cuh"

namespace h3 {

namespace cp5 {

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}
using tma::bulk_g2s;
using tma::fence_proxy_async_smem;
using tma::mbar_arrive_expect_tx;
using tma::mbar_fence_init;
using tma::mbar_init;
using tma::mbar_wait;

// K order of the N = 5 fused passes: the input c = a n + j (vertex a, component j) that lane q
// reads at k-step ks, per pass (x1, x2, x3).  Found by tools/cp5_korder_search.py: a half-warp's
// 4 lines x 4 k-lanes then fall on distinct bank pairs (x1) or fewer wavefronts (x2),
// where the natural order k = 4 ks + q is 2-way on every load.  Packed 4 bits per lane q.
// LAYOUT2 (tools/cp5_smem_model.py, validated against ncu's per-instruction wavefronts): W cell
// stride n(n^2+1) + 1, V j3 stride n^2 with the second V buffer 8 doubles further, and the x2 order
// below: modelled wavefronts per plane 2724 -> 2112 (x3 loads 4 -> 2 per instruction).
template <int LAYOUT2 = 0>
__device__ __forceinline__ int korder5(int ax, int ks, int q) {
    constexpr unsigned T[3][3] = {{0x7610u, 0x9832u, 0xba54u},   // x1: (q >> 1, 2 ks + (q & 1))
                                  {0xa640u, 0xb751u, 0x9832u},   // x2
                                  {0x3210u, 0x7654u, 0xba98u}};  // x3: natural (the searched
                                  // conflict-free 0x6210 0xa843 0xb975 measured 4 % slower)
    constexpr unsigned T2[3] = {0x64a0u, 0x1b57u, 0x3892u};      // x2 under LAYOUT2
    const unsigned t = ((LAYOUT2 & 2) && ax == 1) ? T2[ks] : T[ax][ks];
    return (int)((t >> (4 * q)) & 15u);
}

// group `warp + WARPS * it` of a pass with G groups of 8 lines exists (warp-uniform; constant
// true when the groups divide evenly, so the unrolled loops keep no test)
template <int G, int WARPS>
__device__ __forceinline__ bool live(int warp, int it) {
    return G % WARPS == 0 || warp + WARPS * it < G;
}

template <int N_, int TX_, int TY_, int WARPS_ = 16, int STAGES_ = 3, int MINB_ = 1, bool ILP_ = false,
          int LAYOUT2_ = 0>
struct Cfg {
    // LAYOUT2 bit 0: the V layout (x3 loads); bit 1: the W layout + x2 K order (x2 loads)
    static constexpr int LAYOUT2 = LAYOUT2_;
    // ILP: issue a pass's DMMAs k-step-major (all line groups of the warp at k-step 0, then 1, 2),
    // so consecutive DMMAs are independent, instead of one group's 3-deep accumulation chain
    static constexpr bool ILP = ILP_;
    static constexpr int N = N_, n = N + 1, n2 = n * n, n3 = n2 * n, K2 = 2 * n;
    static constexpr int KS = K2 / 4;  // m8n8k4 k-steps per line
    static_assert(K2 % 4 == 0, "cell-pair form needs 2n divisible by 4");
    static_assert(n <= 8, "n outputs must fit the 8 MMA columns");
    static constexpr int TX = TX_, TY = TY_, NX = TX + 1, NY = TY + 1, NNODE = NX * NY;
    static constexpr int WARPS = WARPS_, THREADS = 32 * WARPS, STAGES = STAGES_, MINB = MINB_;
    static constexpr int UNS = n3;                   // U: dense node blocks [j3][j2][j1]
    static constexpr int WM = n2 + 1, WCS = n * WM + ((LAYOUT2 & 2) ? 1 : 0);  // W: [node row][cell][m1][j3 j2]
    static constexpr int VJ = (LAYOUT2 & 1) ? n2 : n2 + 1, VCS = n * VJ;       // V: [cell][j3][m2 m1]
    static constexpr int G1 = (NY * TX * n2 + 7) / 8;  // x1 line groups of 8
    static constexpr int G2 = (TY * TX * n2 + 7) / 8;  // x2 line groups
    static constexpr int G3 = (TY * TX * n2 + 7) / 8;  // x3 line groups
    static constexpr size_t U_D = (size_t)NNODE * UNS;
    static constexpr size_t W_D = (size_t)NY * TX * WCS;
    static constexpr size_t V_D = (size_t)TY * TX * VCS + ((LAYOUT2 & 1) ? 8 : 0);  // one V buffer (+ bank shift)
    static constexpr size_t SMEM_DATA = (STAGES * U_D + W_D + 2 * V_D) * sizeof(double);
    static constexpr size_t SMEM = SMEM_DATA + STAGES * sizeof(uint64_t);
    static_assert(NY <= WARPS, "one loader warp per tile row");
};

}  // namespace cp5

template <class C>
__global__ void __launch_bounds__(C::THREADS, C::MINB)
sep_fused_dmma_cp_kernel(const double* __restrict__ src, double* __restrict__ dst, Dims d, int off, int zchunk,
                         const __grid_constant__ SepOps<C::N> p, unsigned long long* first_bad,
                         const unsigned long long* guard) {
    using namespace cp5;
    constexpr int n = C::n, n2 = C::n2, n3 = C::n3, KS = C::KS, TX = C::TX, TY = C::TY, NX = C::NX, NY = C::NY;
    constexpr int WARPS = C::WARPS, STAGES = C::STAGES, UNS = C::UNS, WM = C::WM, WCS = C::WCS;
    constexpr int VJ = C::VJ, VCS = C::VCS;
    constexpr int L1 = NY * TX * n2, L2 = TY * TX * n2;
    if (guarded_out(guard, first_bad)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* U = reinterpret_cast<double*>(smem_raw);
    double* W = U + STAGES * C::U_D;
    double* V = W + C::W_D;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + C::SMEM_DATA);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q = lane & 3, g = lane >> 2;
    const int M1 = (int)d.M1, M2 = (int)d.M2;
    const int cx0 = blockIdx.x * TX, cy0 = blockIdx.y * TY;
    const int64_t zc0 = d.z_begin + (int64_t)blockIdx.z * zchunk;
    const int64_t zc1 = min(zc0 + (int64_t)zchunk, d.z_end);
    const int P = (int)(zc1 - zc0) + 1;
    const int64_t plane_elems = (int64_t)M1 * M2 * n3;

    // B fragments: lane holds B[k = 4 ks + q][col = g] = A_axis[g][k] (zero for g >= n)
    double bop[3][KS];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax)
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            // x1 orders its K inputs as (vertex q >> 1, component 2 ks + (q & 1)) instead of
            // k = 4 ks + q: with the 6-double line rows of a node block this puts the 16 lanes of a
            // half-warp on 16 distinct bank pairs (found by search; the natural order is 2-way)
            const int kc = C::N == 5 ? korder5<C::LAYOUT2>(ax, ks, q) : 4 * ks + q;
            bop[ax][ks] = g < n ? p.A[ax][g < n ? g : 0][kc] : 0.0;
        }

    // loader: lane 0 of warp ly < NY copies tile row ly of every plane
    int rowoff = 0, gx0 = 0;
    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
        mbar_fence_init();
    }
    if (lane == 0 && warp < NY) {
        int gy = (cy0 + off + warp) % M2; if (gy < 0) gy += M2;
        gx0 = (cx0 + off) % M1; if (gx0 < 0) gx0 += M1;
        rowoff = gy * M1;
    }
    __syncthreads();
    int64_t gz_next = d.periodic_z ? wrap(zc0 + off, d.M3) : zc0 + off;
    int issued = 0;
    auto issue = [&]() {
        if (issued < P) {
            if (lane == 0 && warp < NY) {
                const int s = issued % STAGES;
                fence_proxy_async_smem();
                if (warp == 0) mbar_arrive_expect_tx(&bars[s], (unsigned)(C::NNODE * UNS * sizeof(double)));
                const double* base = plane_base(src, gz_next, plane_elems, d) + (int64_t)rowoff * n3;
                double* Ub = U + s * C::U_D + warp * NX * UNS;
                int got = 0, gx = gx0;
                while (got < NX) {
                    const int len = min(NX - got, M1 - gx);
                    bulk_g2s(Ub + got * UNS, base + (int64_t)gx * n3, (unsigned)(len * UNS * sizeof(double)), &bars[s]);
                    got += len;
                    gx = 0;
                }
            }
            ++gz_next;
            if (d.periodic_z && gz_next == d.M3) gz_next = 0;
            ++issued;
        }
    };
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) issue();

    // Per-lane addressing, computed once: A-fragment input k = 4 ks + q -> (vertex a, component j);
    // per pass and unrolled group iteration the lane's smem read/write offsets.  Lines past the
    // end of a pass (ragged last group) read a clamped line and store nothing.
    constexpr int I1 = (C::G1 + WARPS - 1) / WARPS, I2 = (C::G2 + WARPS - 1) / WARPS;
    constexpr int I3 = (C::G3 + WARPS - 1) / WARPS;
    int k1[KS], k2[KS], k3[KS], ka[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
        // per pass, the (vertex a, component j) this lane's k-slot reads (korder5: N = 5)
        const int c1 = C::N == 5 ? korder5<C::LAYOUT2>(0, ks, q) : 4 * ks + q;
        const int c2 = C::N == 5 ? korder5<C::LAYOUT2>(1, ks, q) : 4 * ks + q;
        const int c3 = C::N == 5 ? korder5<C::LAYOUT2>(2, ks, q) : 4 * ks + q;
        k1[ks] = (c1 / n) * UNS + c1 % n;       // x1: node cx + a along the row
        k2[ks] = (c2 / n) * TX * WCS + c2 % n;  // x2: cell row cy + a
        ka[ks] = c3 / n;                        // x3: plane p - 1 + a ...
        k3[ks] = (c3 % n) * VJ;                 //     ... its j3 slot
    }
    const bool qout = 2 * q < n;  // this lane's output columns 2q, 2q + 1 are real outputs
    int r1[I1], w1[I1], r2[I2], w2[I2], r3[I3], o3[I3];
#pragma unroll
    for (int it = 0; it < I1; ++it) {
        const int l = (warp + WARPS * it) * 8 + g, lc = l < L1 ? l : L1 - 1;
        const int rc = lc / n2, jj = lc - rc * n2, ly = rc / TX, cx = rc - ly * TX;  // rc = ly TX + cx
        r1[it] = (ly * NX + cx) * UNS + jj * n;
        w1[it] = (l < L1 && qout) ? rc * WCS + (2 * q) * WM + jj : -1;
    }
#pragma unroll
    for (int it = 0; it < I2; ++it) {
        const int l = (warp + WARPS * it) * 8 + g, lc = l < L2 ? l : L2 - 1;
        const int cell = lc / n2, r = lc - cell * n2, j3 = r / n, m1 = r - j3 * n;
        r2[it] = cell * WCS + m1 * WM + j3 * n;
        w2[it] = (l < L2 && qout) ? cell * VCS + j3 * VJ + (2 * q) * n + m1 : -1;
    }
#pragma unroll
    for (int it = 0; it < I3; ++it) {
        const int l = (warp + WARPS * it) * 8 + g, lc = l < L2 ? l : L2 - 1;
        const int cell = lc / n2, r = lc - cell * n2;
        const int cx = cx0 + cell % TX, cy = cy0 + cell / TX;
        r3[it] = cell * VCS + r;
        // output offset within a node plane (int32: M1 M2 n^3 < 2^31 is checked at launch)
        o3[it] = (l < L2 && qout && cx < M1 && cy < M2) ? (cy * M1 + cx) * n3 + (2 * q) * n2 + r : -1;
    }

    // x3 of cell plane p-2 shares a barrier interval with x1 of node plane p (2 barriers per plane)
    for (int pl = 0; pl <= P; ++pl) {
        if (pl < P) {
            __syncthreads();
            issue();  // refills the stage read in iteration pl - 1
            mbar_wait(&bars[pl % STAGES], (unsigned)((pl / STAGES) & 1));
        } else {
            __syncthreads();
        }
        // ---- x3: line cell n^2 + (m2 n + m1), V planes p-1 and p -> dst (cell plane p-1) --------
        if (pl >= 2) {
            const int cp = pl - 2;  // cell plane (node planes cp, cp + 1)
            const double* vk[KS];
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) vk[ks] = V + ((cp + ka[ks]) & 1) * C::V_D + k3[ks];
            double* oplane = dst + (zc0 + cp) * plane_elems;
            double d[I3][2];
            if constexpr (C::ILP) {
#pragma unroll
                for (int it = 0; it < I3; ++it) d[it][0] = d[it][1] = 0.0;
#pragma unroll
                for (int ks = 0; ks < KS; ++ks)
#pragma unroll
                    for (int it = 0; it < I3; ++it)
                        if (live<C::G3, WARPS>(warp, it)) dmma(d[it][0], d[it][1], vk[ks][r3[it]], bop[2][ks]);
            } else {
#pragma unroll
            for (int it = 0; it < I3; ++it) {
                d[it][0] = d[it][1] = 0.0;
                if (!live<C::G3, WARPS>(warp, it)) continue;  // warp-uniform: no dummy DMMAs
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) dmma(d[it][0], d[it][1], vk[ks][r3[it]], bop[2][ks]);
            }
            }
#pragma unroll
            for (int it = 0; it < I3; ++it)
                if (live<C::G3, WARPS>(warp, it) && o3[it] >= 0) {
                    __stcs(oplane + o3[it], d[it][0]);
                    __stcs(oplane + o3[it] + n2, d[it][1]);
                    if (!isfinite(d[it][0]) || !isfinite(d[it][1]))
                        flag_bad(first_bad, (zc0 + cp) * M2 * (int64_t)M1 + o3[it] / n3);
                }
        }
        if (pl < P) {
            const double* Ub = U + (pl % STAGES) * C::U_D;
        // ---- x1: line (ly TX + cx) n^2 + jj:  U(p) -> W ------------------------------------------
        {
            double d[I1][2];
            if constexpr (C::ILP) {
#pragma unroll
                for (int it = 0; it < I1; ++it) d[it][0] = d[it][1] = 0.0;
#pragma unroll
                for (int ks = 0; ks < KS; ++ks)
#pragma unroll
                    for (int it = 0; it < I1; ++it)
                        if (live<C::G1, WARPS>(warp, it)) dmma(d[it][0], d[it][1], Ub[r1[it] + k1[ks]], bop[0][ks]);
            } else {
#pragma unroll
            for (int it = 0; it < I1; ++it) {
                d[it][0] = d[it][1] = 0.0;
                if (!live<C::G1, WARPS>(warp, it)) continue;
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) dmma(d[it][0], d[it][1], Ub[r1[it] + k1[ks]], bop[0][ks]);
            }
            }
#pragma unroll
            for (int it = 0; it < I1; ++it)
                if (live<C::G1, WARPS>(warp, it) && w1[it] >= 0) {
                    W[w1[it]] = d[it][0];
                    W[w1[it] + WM] = d[it][1];
                }
        }
        }
        __syncthreads();
        if (pl < P) {
            double* Vc = V + (pl & 1) * C::V_D;
        // ---- x2: line cell n^2 + j3 n + m1:  W -> V[p & 1] ---------------------------------------
        {
            double d[I2][2];
            if constexpr (C::ILP) {
#pragma unroll
                for (int it = 0; it < I2; ++it) d[it][0] = d[it][1] = 0.0;
#pragma unroll
                for (int ks = 0; ks < KS; ++ks)
#pragma unroll
                    for (int it = 0; it < I2; ++it)
                        if (live<C::G2, WARPS>(warp, it)) dmma(d[it][0], d[it][1], W[r2[it] + k2[ks]], bop[1][ks]);
            } else {
#pragma unroll
            for (int it = 0; it < I2; ++it) {
                d[it][0] = d[it][1] = 0.0;
                if (!live<C::G2, WARPS>(warp, it)) continue;
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) dmma(d[it][0], d[it][1], W[r2[it] + k2[ks]], bop[1][ks]);
            }
            }
#pragma unroll
            for (int it = 0; it < I2; ++it)
                if (live<C::G2, WARPS>(warp, it) && w2[it] >= 0) {
                    Vc[w2[it]] = d[it][0];
                    Vc[w2[it] + n] = d[it][1];
                }
        }
        }
    }
}

template <class C>
static int launch_cp(const double* src, double* dst, const Dims& d, const double* A, int off, cudaStream_t st,
                     unsigned long long* first_bad, const unsigned long long* guard) {
    const int64_t nz = d.z_end - d.z_begin;
    if (nz <= 0) return 0;
    if (d.M1 * d.M2 * C::n3 >= (int64_t(1) << 31)) return (int)cudaErrorInvalidValue;
    SepOps<C::N> ops;
    for (int k = 0; k < 3; ++k)
        for (int m = 0; m < C::n; ++m)
            for (int c = 0; c < 2 * C::n; ++c) {
                ops.A[k][m][c] = A[(k * C::n + m) * 2 * C::n + c];
                ops.Sh[k][m][c] = 0.0;
            }
    auto kern = sep_fused_dmma_cp_kernel<C>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return (int)e;
    const int64_t gx = (d.M1 + C::TX - 1) / C::TX, gy = (d.M2 + C::TY - 1) / C::TY;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::THREADS, C::SMEM);
    if (e != cudaSuccess) return (int)e;
    const int64_t zchunk = choose_zchunk(gx * gy, nz, (int64_t)num_sms() * (per_sm > 0 ? per_sm : 1));
    const int64_t gz = (nz + zchunk - 1) / zchunk;
    kern<<<dim3((unsigned)gx, (unsigned)gy, (unsigned)gz), C::THREADS, C::SMEM, st>>>(src, dst, d, off, (int)zchunk,
                                                                                   ops, first_bad, guard);
    return (int)cudaGetLastError();
}

int sep_fused_dmma5_launch(const double* src, double* dst, const Dims& d, const double* A, int off, cudaStream_t st,
                           unsigned long long* first_bad, const unsigned long long* guard) {
#ifdef H3_MEASURE
    static const int cfg = [] {  // tools library only: alternative tile shapes for tools/ab.sh
        const char* e = getenv("H3_DMMA5_CFG");
        return e ? atoi(e) : 0;
    }();
    if (cfg >= 20) return sep_fused_dmma5_ws_launch(src, dst, d, A, off, st, first_bad, guard, cfg - 20);
    if (cfg == 1) return launch_cp<cp5::Cfg<5, 4, 2, 8, 2, 2>>(src, dst, d, A, off, st, first_bad, guard);
    if (cfg == 2) return launch_cp<cp5::Cfg<5, 4, 2, 8, 3, 1>>(src, dst, d, A, off, st, first_bad, guard);
    if (cfg == 3) return launch_cp<cp5::Cfg<5, 4, 4, 16, 3, 1, true>>(src, dst, d, A, off, st, first_bad, guard);
    if (cfg == 4) return launch_cp<cp5::Cfg<5, 4, 4, 16, 2, 1>>(src, dst, d, A, off, st, first_bad, guard);
    if (cfg == 5) return launch_cp<cp5::Cfg<5, 2, 8, 16, 2, 1>>(src, dst, d, A, off, st, first_bad, guard);
    if (cfg == 6) return launch_cp<cp5::Cfg<5, 2, 8, 16, 2, 1, true>>(src, dst, d, A, off, st, first_bad, guard);
    if (cfg == 7) return launch_cp<cp5::Cfg<5, 3, 6, 16, 2, 1>>(src, dst, d, A, off, st, first_bad, guard);
    if (cfg == 8) return launch_cp<cp5::Cfg<5, 4, 5, 16, 2, 1>>(src, dst, d, A, off, st, first_bad, guard);
    if (cfg == 9) return launch_cp<cp5::Cfg<5, 4, 4, 16, 3, 1, false, 3>>(src, dst, d, A, off, st, first_bad, guard);
    if (cfg == 10) return launch_cp<cp5::Cfg<5, 4, 4, 16, 2, 1, false, 3>>(src, dst, d, A, off, st, first_bad, guard);
    if (cfg == 11) return launch_cp<cp5::Cfg<5, 4, 4, 16, 3, 1, false, 1>>(src, dst, d, A, off, st, first_bad, guard);
    if (cfg == 12) return launch_cp<cp5::Cfg<5, 4, 4, 16, 3, 1, false, 2>>(src, dst, d, A, off, st, first_bad, guard);
    if (cfg == 13) return launch_cp<cp5::Cfg<5, 4, 4>>(src, dst, d, A, off, st, first_bad, guard);  // r01 default
#endif
    // the warp-specialised pipeline (h3_dmma5ws.cu) replaces this lock-step march (r02: +15 %)
    return sep_fused_dmma5_ws_launch(src, dst, d, A, off, st, first_bad, guard, 0);
}

// ---------------------------------------------------------------------------------------------
// Reconstruction pass of the two-kernel step in the same cell-pair DMMA form (N = 5):
//   coeff(c) = sum_a (H^a3 (x) H^a2 (x) H^a1) u(c + off + a),  H^a = H[:, a n : a n + n],
// a pass line gathers its cell's two vertex blocks (K = 2n = 12) and produces s = 12 outputs
// (two 8-column blocks, 12 of 16 used).  H is the same for all three axes, so the whole operator
// is 6 registers per lane.  x3 writes the (2N+2)^3 coefficient block of each cell straight to HBM
// (the two-kernel intermediate, gridkernels.py:142-160 layout [i3][i2][i1]).
// ---------------------------------------------------------------------------------------------
namespace rcp {
template <int N_, int TX_, int TY_, int STAGES_>
struct Cfg {
    static constexpr int N = N_, n = N + 1, n2 = n * n, n3 = n2 * n, S = 2 * n, S2 = S * S, S3 = S2 * S;
    static constexpr int KS = S / 4, CB = (S + 7) / 8;  // k-steps, 8-column output blocks
    static_assert(S % 4 == 0, "cell-pair form needs 2n divisible by 4");
    static constexpr int TX = TX_, TY = TY_, NX = TX + 1, NY = TY + 1, NNODE = NX * NY;
    static constexpr int WARPS = 16, THREADS = 32 * WARPS, STAGES = STAGES_;
    static constexpr int UNS = n3;
    static constexpr int WI = n2 + 1, WCS = S * WI;  // W: [node row][cell][i1][j3 j2]
    // V: [cell][j3][i2 i1]; j3 stride = 4 (mod 16 doubles) so the x3 A-fragment loads (8 lines x 4
    // k of one cell) fall on 16 distinct bank pairs per half-warp (S2 + 1 gave 8-way conflicts)
    static constexpr int VJ = S2 + 4, VCS = n * VJ;
    static constexpr int L1 = NY * TX * n2, L2 = TY * TX * n * S, L3 = TY * TX * S2;
    static constexpr int G1 = (L1 + 7) / 8, G2 = (L2 + 7) / 8, G3 = (L3 + 7) / 8;
    static constexpr size_t U_D = (size_t)NNODE * UNS;
    static constexpr size_t W_D = (size_t)NY * TX * WCS;
    static constexpr size_t V_D = (size_t)TY * TX * VCS;
    static constexpr size_t SMEM_DATA = (STAGES * U_D + W_D + 2 * V_D) * sizeof(double);
    static constexpr size_t SMEM = SMEM_DATA + STAGES * sizeof(uint64_t);
    static_assert(NY <= WARPS, "one loader warp per tile row");
};
}  // namespace rcp

template <class C>
__global__ void __launch_bounds__(C::THREADS, 1)
recon_dmma_cp_kernel(const double* __restrict__ src, double* __restrict__ coeff, Dims d, int off, int zchunk,
                     const __grid_constant__ LitOps<double, C::N> hp, const unsigned long long* guard) {
    using namespace cp5;
    constexpr int n = C::n, n2 = C::n2, n3 = C::n3, S = C::S, S2 = C::S2, S3 = C::S3, KS = C::KS, CB = C::CB;
    constexpr int TX = C::TX, NX = C::NX, NY = C::NY, WARPS = C::WARPS, STAGES = C::STAGES, UNS = C::UNS;
    constexpr int WI = C::WI, WCS = C::WCS, VJ = C::VJ, VCS = C::VCS, L1 = C::L1, L2 = C::L2, L3 = C::L3;
    constexpr int I1 = (C::G1 + WARPS - 1) / WARPS, I2 = (C::G2 + WARPS - 1) / WARPS;
    constexpr int I3 = (C::G3 + WARPS - 1) / WARPS;
    if (guarded_out(guard, nullptr)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* U = reinterpret_cast<double*>(smem_raw);
    double* W = U + STAGES * C::U_D;
    double* V = W + C::W_D;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + C::SMEM_DATA);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q = lane & 3, g = lane >> 2;
    const int M1 = (int)d.M1, M2 = (int)d.M2;
    const int cx0 = blockIdx.x * TX, cy0 = blockIdx.y * C::TY;
    const int64_t zc0 = d.z_begin + (int64_t)blockIdx.z * zchunk;
    const int64_t zc1 = min(zc0 + (int64_t)zchunk, d.z_end);
    const int P = (int)(zc1 - zc0) + 1;
    const int64_t plane_elems = (int64_t)M1 * M2 * n3;
    const int64_t cplane = (int64_t)M1 * M2 * S3;

    // B fragments (all axes): lane holds B[k = 4 ks + q][col = 8 cb + g] = H[8 cb + g][k]
    double bop[KS][CB];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
        for (int cb = 0; cb < CB; ++cb) {
            const int col = 8 * cb + g;
            bop[ks][cb] = col < S ? hp.H[(col < S ? col : 0) * S + 4 * ks + q] : 0.0;
        }

    int rowoff = 0, gx0 = 0;
    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
        mbar_fence_init();
    }
    if (lane == 0 && warp < NY) {
        int gy = (cy0 + off + warp) % M2; if (gy < 0) gy += M2;
        gx0 = (cx0 + off) % M1; if (gx0 < 0) gx0 += M1;
        rowoff = gy * M1;
    }
    __syncthreads();
    int64_t gz_next = d.periodic_z ? wrap(zc0 + off, d.M3) : zc0 + off;
    int issued = 0;
    auto issue = [&]() {
        if (issued < P) {
            if (lane == 0 && warp < NY) {
                const int s = issued % STAGES;
                fence_proxy_async_smem();
                if (warp == 0) mbar_arrive_expect_tx(&bars[s], (unsigned)(C::NNODE * UNS * sizeof(double)));
                const double* base = plane_base(src, gz_next, plane_elems, d) + (int64_t)rowoff * n3;
                double* Ub = U + s * C::U_D + warp * NX * UNS;
                int got = 0, gx = gx0;
                while (got < NX) {
                    const int len = min(NX - got, M1 - gx);
                    bulk_g2s(Ub + got * UNS, base + (int64_t)gx * n3, (unsigned)(len * UNS * sizeof(double)), &bars[s]);
                    got += len;
                    gx = 0;
                }
            }
            ++gz_next;
            if (d.periodic_z && gz_next == d.M3) gz_next = 0;
            ++issued;
        }
    };
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) issue();

    int k1[KS], k2[KS], k3[KS], ka[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
        const int k = 4 * ks + q, a = k / n, j = k % n;
        ka[ks] = a;
        k1[ks] = a * UNS + j;
        k2[ks] = a * TX * WCS + j;
        k3[ks] = j * VJ;
    }
    // output columns of this lane: 8 cb + 2q (+1); the last block is partial when S % 8 != 0
    const bool cout1 = 8 * (CB - 1) + 2 * q < S;
    int r1[I1], w1[I1], r2[I2], w2[I2], r3[I3], o3[I3];
#pragma unroll
    for (int it = 0; it < I1; ++it) {
        const int l = (warp + WARPS * it) * 8 + g, lc = l < L1 ? l : L1 - 1;
        const int rc = lc / n2, jj = lc - rc * n2, ly = rc / TX, cx = rc - ly * TX;
        r1[it] = (ly * NX + cx) * UNS + jj * n;
        w1[it] = l < L1 ? rc * WCS + (2 * q) * WI + jj : -1;  // + 8 cb WI
    }
#pragma unroll
    for (int it = 0; it < I2; ++it) {
        const int l = (warp + WARPS * it) * 8 + g, lc = l < L2 ? l : L2 - 1;
        const int cell = lc / (n * S), r = lc - cell * (n * S), j3 = r / S, i1 = r - j3 * S;
        r2[it] = cell * WCS + i1 * WI + j3 * n;
        w2[it] = l < L2 ? cell * VCS + j3 * VJ + (2 * q) * S + i1 : -1;  // + 8 cb S
    }
#pragma unroll
    for (int it = 0; it < I3; ++it) {
        const int l = (warp + WARPS * it) * 8 + g, lc = l < L3 ? l : L3 - 1;
        const int cell = lc / S2, r = lc - cell * S2;
        const int cx = cx0 + cell % TX, cy = cy0 + cell / C::TX;
        r3[it] = cell * VCS + r;
        // relative to the tile's first cell (int32 up to M1 < 2^31 / (TY S^3)): the coefficient
        // plane itself (M1 M2 S^3 doubles) may exceed 2^31 elements
        o3[it] = (l < L3 && cx < M1 && cy < M2) ? ((cy - cy0) * M1 + (cx - cx0)) * S3 + (2 * q) * S2 + r : -1;  // + 8 cb S2
    }

    // x3 of cell plane p-2 shares a barrier interval with x1 of node plane p (2 barriers per plane)
    for (int pl = 0; pl <= P; ++pl) {
        if (pl < P) {
            __syncthreads();
            issue();  // refills the stage read in iteration pl - 1
            mbar_wait(&bars[pl % STAGES], (unsigned)((pl / STAGES) & 1));
        } else {
            __syncthreads();
        }
        // ---- x3: V planes p-1, p -> coeff (cell plane p-1), streaming stores ------------------
        if (pl >= 2) {
            const int cp = pl - 2;  // cell plane (node planes cp, cp + 1)
            const double* vk[KS];
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) vk[ks] = V + ((cp + ka[ks]) & 1) * C::V_D + k3[ks];
            double* oplane = coeff + (zc0 - d.z_begin + cp) * cplane + ((int64_t)cy0 * M1 + cx0) * S3;
#pragma unroll
            for (int it = 0; it < I3; ++it) {
                if (!live<C::G3, WARPS>(warp, it)) continue;  // warp-uniform: no dummy DMMAs
                double a[KS];
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) a[ks] = vk[ks][r3[it]];
#pragma unroll
                for (int cb = 0; cb < CB; ++cb) {
                    double d0 = 0.0, d1 = 0.0;
#pragma unroll
                    for (int ks = 0; ks < KS; ++ks) dmma(d0, d1, a[ks], bop[ks][cb]);
                    if (o3[it] >= 0 && (cb < CB - 1 || cout1)) {
                        __stcs(oplane + o3[it] + 8 * cb * S2, d0);
                        __stcs(oplane + o3[it] + (8 * cb + 1) * S2, d1);
                    }
                }
            }
        }
        if (pl < P) {
            const double* Ub = U + (pl % STAGES) * C::U_D;
        // ---- x1: U(p) -> W[row][cell][i1][j3 j2] ----------------------------------------------
#pragma unroll
        for (int it = 0; it < I1; ++it) {
            if (!live<C::G1, WARPS>(warp, it)) continue;
            double a[KS];
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) a[ks] = Ub[r1[it] + k1[ks]];
#pragma unroll
            for (int cb = 0; cb < CB; ++cb) {
                double d0 = 0.0, d1 = 0.0;
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) dmma(d0, d1, a[ks], bop[ks][cb]);
                if (w1[it] >= 0 && (cb < CB - 1 || cout1)) {
                    W[w1[it] + 8 * cb * WI] = d0;
                    W[w1[it] + (8 * cb + 1) * WI] = d1;
                }
            }
        }
        }
        __syncthreads();
        if (pl < P) {
            double* Vc = V + (pl & 1) * C::V_D;
        // ---- x2: W -> V[p & 1][cell][j3][i2 i1] -------------------------------------------------
#pragma unroll
        for (int it = 0; it < I2; ++it) {
            if (!live<C::G2, WARPS>(warp, it)) continue;
            double a[KS];
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) a[ks] = W[r2[it] + k2[ks]];
#pragma unroll
            for (int cb = 0; cb < CB; ++cb) {
                double d0 = 0.0, d1 = 0.0;
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) dmma(d0, d1, a[ks], bop[ks][cb]);
                if (w2[it] >= 0 && (cb < CB - 1 || cout1)) {
                    Vc[w2[it] + 8 * cb * S] = d0;
                    Vc[w2[it] + (8 * cb + 1) * S] = d1;
                }
            }
        }
        }
    }
}

int recon_dmma5_launch(const double* src, double* coeff, const Dims& d, const double* h_mat, int off,
                       cudaStream_t st, const unsigned long long* guard) {
    // the warp-specialised pipeline (h3_recon5ws.cu) is the product kernel; the lock-step kernel
    // below stays in the tools library as its A/B baseline (H3_RECON5_WS=-1)
#ifdef H3_MEASURE
    static const int ws = [] {  // tools library only: H3_RECON5_WS=k selects a variant
        const char* e = getenv("H3_RECON5_WS");
        return e ? atoi(e) : 0;
    }();
    if (ws >= 0) return recon_dmma5_ws_launch(src, coeff, d, h_mat, off, st, guard, ws);
    using C = rcp::Cfg<5, 4, 2, 2>;
    const int64_t nz = d.z_end - d.z_begin;
    if (nz <= 0) return 0;
    if (d.M1 * d.M2 * C::n3 >= (int64_t(1) << 31) || d.M1 * C::TY * C::S3 >= (int64_t(1) << 31))
        return (int)cudaErrorInvalidValue;  // int32 node-plane / tile-relative output offsets
    LitOps<double, 5> hp;
    for (int i = 0; i < C::S2; ++i) hp.H[i] = h_mat[i];
    for (int i = 0; i < C::S; ++i) hp.f1[i] = hp.f2[i] = hp.f3[i] = 0.0;
    for (int i = 0; i < H3_MAX_STAGES; ++i) hp.cf[i] = 0.0;
    hp.q = 0;
    auto kern = recon_dmma_cp_kernel<C>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return (int)e;
    const int64_t gx = (d.M1 + C::TX - 1) / C::TX, gy = (d.M2 + C::TY - 1) / C::TY;
    const int64_t zchunk = choose_zchunk(gx * gy, nz, num_sms());  // one CTA per SM
    const int64_t gz = (nz + zchunk - 1) / zchunk;
    kern<<<dim3((unsigned)gx, (unsigned)gy, (unsigned)gz), C::THREADS, C::SMEM, st>>>(src, coeff, d, off, (int)zchunk,
                                                                                   hp, guard);
    return (int)cudaGetLastError();
#else
    return recon_dmma5_ws_launch(src, coeff, d, h_mat, off, st, guard, 0);
#endif
}

}  // namespace h3
