// Warp-specialised FP64 tensor-core fused half step for N = 5 (n = 6): the cell-pair DMMA form of
// h3_dmma5.cu (same operators, same K orders, same shared layouts), reorganised as a producer /
// consumer pipeline over node planes instead of a lock-step march with CTA-wide barriers.
//
//   warp 0            TMA producer: bulk-copies tile rows of node plane t into U[t % SU]
//   warps 1 .. N1     x1: U[t % SU]          -> W[t % NWB]     (line = node row, cell, j3 j2)
//   next N2 warps     x2: W[t % NWB]         -> V[t % NVB]     (line = cell, j3, m1)
//   last N3 warps     x3: V[c % NVB], V[(c+1) % NVB] -> dst plane c (line = cell, m2 m1)
//
// Every hand-off is an mbarrier pair (full / empty) per buffer, so each role runs as soon as its
// input is ready and its output buffer is free: x1 of plane t, x2 of plane t-1 and x3 of cell plane
// t-3 overlap, and no warp ever waits at a CTA-wide barrier.  The lock-step kernel keeps the DMMA
// pipe ~59 % busy (ncu, r01/r02): with all 16 warps in the same pass, each barrier interval
// drains and refills the pipe.  Here the SM's warps always hold a mix of passes: 75 % DMMA pipe
// (profiles/r02_fused5_256_sep_fused_summary.json), against a ceiling of the FP64 tensor pipe itself
// (42.75 DMMAs per cell at 75 % column fill = 171 pipe cycles vs 153 cycles of HBM traffic per cell).
//
// Phases: the k-th use of a buffer waits for the k-th completion of its "full" barrier (parity
// k & 1); a producer's first wait on an "empty" barrier passes at once (parity 1 on a fresh
// barrier), later ones wait for the consumer's release of the use two / three planes back.
#include "h3_launch.h"
#include "h3_tma.cuh"

#ifndef H3_WS5_BAND
#define H3_WS5_BAND 8
#endif

namespace h3 {
namespace ws5 {

using tma::bulk_g2s;
using tma::fence_proxy_async_smem;
using tma::mbar_arrive_expect_tx;
using tma::mbar_fence_init;
using tma::mbar_init;
using tma::mbar_wait;

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}

// K orders (see h3_dmma5.cu korder5): x1 (vertex q >> 1, component 2 ks + (q & 1)), x2 searched,
// x3 natural
__device__ __forceinline__ int korder(int ax, int ks, int q, bool vl = false) {
    constexpr unsigned T[3][3] = {{0x7610u, 0x9832u, 0xba54u}, {0xa640u, 0xb751u, 0x9832u},
                                  {0x3210u, 0x7654u, 0xba98u}};
    constexpr unsigned T3[3] = {0x2530u, 0x16b4u, 0x978au};  // x3 under VL
    return (int)((((vl && ax == 2) ? T3[ks] : T[ax][ks]) >> (4 * q)) & 15u);
}
// lane row g -> line of its group of 8 (x3 under VL)
__device__ __forceinline__ int x3_line(int g, bool vl) {
    constexpr unsigned P = 0x27413065u;  // 5 6 0 3 1 4 7 2
    return vl ? (int)((P >> (4 * g)) & 15u) : g;
}

// Per-tile-shape W layout and x2 lane orders (tools/ws5_smem_model.py search: x1 loads and
// stores conflict-free, x2 at 2.67 wavefronts per instruction): W m1 stride, W cell padding,
// x2 K order (4 bits per lane q, per k-step) and x2 lane -> line order (4 bits per lane row g).
template <int TX, int TY>
struct Lay {
    static constexpr int WM = 37, WPAD = 0;
    static constexpr unsigned P2 = 0x76543210u;
    __device__ static constexpr unsigned k2(int ks) { return ks == 0 ? 0xa640u : ks == 1 ? 0xb751u : 0x9832u; }
};
template <>
struct Lay<3, 4> {
    static constexpr int WM = 38, WPAD = 4;
    static constexpr unsigned P2 = 0x46751203u;
    __device__ static constexpr unsigned k2(int ks) { return ks == 0 ? 0x54abu : ks == 1 ? 0x7106u : 0x2398u; }
};
template <>
struct Lay<2, 6> {
    static constexpr int WM = 37, WPAD = 6;
    static constexpr unsigned P2 = 0x47561032u;
    __device__ static constexpr unsigned k2(int ks) { return ks == 0 ? 0x4a60u : ks == 1 ? 0x51b7u : 0x8923u; }
};

template <int TX_, int TY_, int N1_, int N2_, int N3_, int SU_, int B_ = 0, bool VL_ = false, int NWB_ = 2,
          int NVB_ = 3>
struct Cfg {
    // NWB / NVB: ring lengths of the W and V buffers (>= 2 and >= 3): deeper rings decouple the
    // roles further; a V ring of 4 also keeps every x3 buffer pair 8 doubles apart in bank terms
    static constexpr int NWB = NWB_, NVB = NVB_;
    static_assert(NWB >= 2 && NVB >= 3, "x2 reads W(t) while x1 writes W(t+1); x3 reads 2 V planes");
    // VL: the x3-side layout of tools/ws5_smem_model.py -- V j3 stride n^2, V buffers 8 doubles
    // apart in bank terms, a searched x3 K order and lane -> line order: modelled x3 load
    // wavefronts 4 -> 2.0 / 2.67 per instruction (the wrap-around buffer pair keeps some conflicts)
    static constexpr bool VL = VL_;
    // B: line groups per batch within a pass (loads, DMMAs and stores of B groups at a time; 0 = all
    // of the warp's groups at once) -- trades in-flight DMMAs for accumulator registers
    static constexpr int N = 5, n = 6, n2 = 36, n3 = 216, KS = 3;
    static constexpr int TX = TX_, TY = TY_, NX = TX + 1, NY = TY + 1, NNODE = NX * NY;
    static constexpr int N1 = N1_, N2 = N2_, N3 = N3_, SU = SU_;
    static constexpr int WARPS = 1 + N1 + N2 + N3, THREADS = 32 * WARPS;
    static constexpr int UNS = n3;
    using LY = Lay<(VL_ ? TX_ : 0), (VL_ ? TY_ : 0)>;  // (the r02 layouts come with VL)
    static constexpr int WM = LY::WM, WCS = n * WM + LY::WPAD;  // W: [node row][cell][m1][j3 j2]
    static constexpr int VJ = VL ? n2 : n2 + 1, VCS = n * VJ;  // V: [cell][j3][m2 m1]
    static constexpr int L1 = NY * TX * n2, L2 = TY * TX * n2;
    static constexpr int G1 = (L1 + 7) / 8, G2 = (L2 + 7) / 8;
    static constexpr int I1 = (G1 + N1 - 1) / N1, I2 = (G2 + N2 - 1) / N2, I3 = (G2 + N3 - 1) / N3;
    static constexpr int B1 = B_ ? B_ : I1, B2 = B_ ? B_ : I2, B3 = B_ ? B_ : I3;
    static constexpr size_t U_D = (size_t)NNODE * UNS;
    static constexpr size_t W_D = (size_t)NY * TX * WCS;
    static constexpr size_t V_D = (size_t)TY * TX * VCS + (VL ? 8 : 0);  // V buffer stride
    static constexpr int NBAR = 2 * SU + 2 * NWB + 2 * NVB;
    static constexpr size_t SMEM_DATA = (SU * U_D + NWB * W_D + NVB * V_D) * sizeof(double);
    static constexpr size_t SMEM = SMEM_DATA + NBAR * sizeof(uint64_t);
    static_assert(NY <= 32, "one producer lane per tile row");
};

template <int G, int NW>
__device__ __forceinline__ bool live(int w, int it) {
    return G % NW == 0 || w + NW * it < G;
}

}  // namespace ws5

template <class C>
__global__ void __launch_bounds__(C::THREADS, 1)
sep_fused_dmma_ws_kernel(const double* __restrict__ src, double* __restrict__ dst, Dims d, int off, int zchunk,
                         const __grid_constant__ SepOps<5> p, unsigned long long* first_bad,
                         const unsigned long long* guard) {
    using namespace ws5;
    constexpr int n = C::n, n2 = C::n2, n3 = C::n3, KS = C::KS, TX = C::TX, NX = C::NX, NY = C::NY;
    constexpr int SU = C::SU, UNS = C::UNS, WM = C::WM, WCS = C::WCS, VJ = C::VJ, VCS = C::VCS;
    constexpr int L1 = C::L1, L2 = C::L2;
    if (guarded_out(guard, first_bad)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* U = reinterpret_cast<double*>(smem_raw);
    double* W = U + SU * C::U_D;
    double* V = W + C::NWB * C::W_D;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + C::SMEM_DATA);
    uint64_t* u_full = bars;
    uint64_t* u_empty = bars + SU;
    uint64_t* w_full = bars + 2 * SU;
    uint64_t* w_empty = w_full + C::NWB;
    uint64_t* v_full = w_empty + C::NWB;
    uint64_t* v_empty = v_full + C::NVB;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q = lane & 3, g = lane >> 2;
    const int M1 = (int)d.M1, M2 = (int)d.M2;
    int tbx, tby;
    band_tile(d.band, 1, tbx, tby);
    const int cx0 = tbx * TX, cy0 = tby * C::TY;
    const int64_t zc0 = d.z_begin + (int64_t)blockIdx.z * zchunk;
    const int64_t zc1 = min(zc0 + (int64_t)zchunk, d.z_end);
    const int P = (int)(zc1 - zc0) + 1;  // node planes of this chunk
    const int64_t plane_elems = (int64_t)M1 * M2 * n3;

    if (tid == 0) {
        // consumer hand-offs count every thread of the releasing role: each lane's own arrive (one
        // warp-wide instruction) releases its own shared-memory writes / reads
        for (int s = 0; s < SU; ++s) {
            mbar_init(&u_full[s], 1);
            mbar_init(&u_empty[s], 32 * C::N1);
        }
        for (int b = 0; b < C::NWB; ++b) {
            mbar_init(&w_full[b], 32 * C::N1);
            mbar_init(&w_empty[b], 32 * C::N2);
        }
        for (int b = 0; b < C::NVB; ++b) {
            mbar_init(&v_full[b], 32 * C::N2);
            mbar_init(&v_empty[b], 32 * C::N3);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (warp == 0) {
        // ---- producer: TMA bulk row copies of node plane t into U[t % SU] ------------------------
        int rowoff = 0, gx0 = (cx0 + off) % M1;
        if (gx0 < 0) gx0 += M1;
        if (lane < NY) {
            int gy = (cy0 + off + lane) % M2;
            if (gy < 0) gy += M2;
            rowoff = gy * M1;
        }
        int64_t gz = d.periodic_z ? wrap(zc0 + off, d.M3) : zc0 + off;
        for (int t = 0; t < P; ++t) {
            const int s = t % SU;
            mbar_wait(&u_empty[s], (unsigned)(((t / SU) & 1) ^ 1));
            if (lane == 0) {
                fence_proxy_async_smem();
                mbar_arrive_expect_tx(&u_full[s], (unsigned)(C::NNODE * UNS * sizeof(double)));
            }
            __syncwarp();
            if (lane < NY) {
                const double* base = plane_base(src, gz, plane_elems, d) + (int64_t)rowoff * n3;
                double* Ub = U + s * C::U_D + lane * NX * UNS;
                int got = 0, gx = gx0;
                while (got < NX) {
                    const int len = min(NX - got, M1 - gx);
                    bulk_g2s(Ub + got * UNS, base + (int64_t)gx * n3, (unsigned)(len * UNS * sizeof(double)),
                             &u_full[s]);
                    got += len;
                    gx = 0;
                }
            }
            ++gz;
            if (d.periodic_z && gz == d.M3) gz = 0;
        }
        return;
    }

    const bool qout = 2 * q < n;  // this lane's output columns 2q, 2q + 1 are real outputs
    if (warp <= C::N1) {
        // ---- x1: line (ly TX + cx) n^2 + jj : U(t) -> W[t & 1] ------------------------------------
        constexpr int NW = C::N1, I = C::I1;
        const int w = warp - 1;
        double bop[KS];
        int kk[KS];
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            const int c = korder(0, ks, q);
            bop[ks] = g < n ? p.A[0][g < n ? g : 0][c] : 0.0;
            kk[ks] = (c / n) * UNS + c % n;
        }
        int rd[I], wr[I];
#pragma unroll
        for (int it = 0; it < I; ++it) {
            const int l = (w + NW * it) * 8 + g, lc = l < L1 ? l : L1 - 1;
            const int rc = lc / n2, jj = lc - rc * n2, ly = rc / TX, cx = rc - ly * TX;
            rd[it] = (ly * NX + cx) * UNS + jj * n;
            wr[it] = (l < L1 && qout) ? rc * WCS + (2 * q) * WM + jj : -1;
        }
        for (int t = 0; t < P; ++t) {
            const int s = t % SU, b = t % C::NWB;
            mbar_wait(&u_full[s], (unsigned)((t / SU) & 1));
            mbar_wait(&w_empty[b], (unsigned)(((t / C::NWB) & 1) ^ 1));
            const double* Ub = U + s * C::U_D;
            double* Wb = W + b * C::W_D;
#pragma unroll
            for (int i0 = 0; i0 < I; i0 += C::B1) {
                double acc[C::B1][2];
#pragma unroll
                for (int j = 0; j < C::B1; ++j) {
                    const int it = i0 + j;
                    acc[j][0] = acc[j][1] = 0.0;
                    if (it >= I || !live<C::G1, NW>(w, it)) continue;
#pragma unroll
                    for (int ks = 0; ks < KS; ++ks) dmma(acc[j][0], acc[j][1], Ub[rd[it] + kk[ks]], bop[ks]);
                }
#pragma unroll
                for (int j = 0; j < C::B1; ++j) {
                    const int it = i0 + j;
                    if (it < I && live<C::G1, NW>(w, it) && wr[it] >= 0) {
                        Wb[wr[it]] = acc[j][0];
                        Wb[wr[it] + WM] = acc[j][1];
                    }
                }
            }
            mbar_arrive(&u_empty[s]);
            mbar_arrive(&w_full[b]);
        }
    } else if (warp <= C::N1 + C::N2) {
        // ---- x2: line cell n^2 + j3 n + m1 : W[t & 1] -> V[t % 3] ----------------------------------
        constexpr int NW = C::N2, I = C::I2;
        const int w = warp - 1 - C::N1;
        double bop[KS];
        int kk[KS];
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            const int c = (int)((C::LY::k2(ks) >> (4 * q)) & 15u);
            bop[ks] = g < n ? p.A[1][g < n ? g : 0][c] : 0.0;
            kk[ks] = (c / n) * TX * WCS + c % n;
        }
        int rd[I], wr[I];
#pragma unroll
        for (int it = 0; it < I; ++it) {
            const int l = (w + NW * it) * 8 + (int)((C::LY::P2 >> (4 * g)) & 15u), lc = l < L2 ? l : L2 - 1;
            const int cell = lc / n2, r = lc - cell * n2, j3 = r / n, m1 = r - j3 * n;
            rd[it] = cell * WCS + m1 * WM + j3 * n;
            wr[it] = (l < L2 && qout) ? cell * VCS + j3 * VJ + (2 * q) * n + m1 : -1;
        }
        for (int t = 0; t < P; ++t) {
            const int b = t % C::NWB, v = t % C::NVB;
            mbar_wait(&w_full[b], (unsigned)((t / C::NWB) & 1));
            mbar_wait(&v_empty[v], (unsigned)(((t / C::NVB) & 1) ^ 1));
            const double* Wb = W + b * C::W_D;
            double* Vb = V + v * C::V_D;
#pragma unroll
            for (int i0 = 0; i0 < I; i0 += C::B2) {
                double acc[C::B2][2];
#pragma unroll
                for (int j = 0; j < C::B2; ++j) {
                    const int it = i0 + j;
                    acc[j][0] = acc[j][1] = 0.0;
                    if (it >= I || !live<C::G2, NW>(w, it)) continue;
#pragma unroll
                    for (int ks = 0; ks < KS; ++ks) dmma(acc[j][0], acc[j][1], Wb[rd[it] + kk[ks]], bop[ks]);
                }
#pragma unroll
                for (int j = 0; j < C::B2; ++j) {
                    const int it = i0 + j;
                    if (it < I && live<C::G2, NW>(w, it) && wr[it] >= 0) {
                        Vb[wr[it]] = acc[j][0];
                        Vb[wr[it] + n] = acc[j][1];
                    }
                }
            }
            mbar_arrive(&w_empty[b]);
            mbar_arrive(&v_full[v]);
        }
    } else {
        // ---- x3: line cell n^2 + (m2 n + m1) : V(c), V(c+1) -> dst cell plane c --------------------
        constexpr int NW = C::N3, I = C::I3;
        const int w = warp - 1 - C::N1 - C::N2;
        double bop[KS];
        int kk[KS], ka[KS];
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            const int c = korder(2, ks, q, C::VL);
            bop[ks] = g < n ? p.A[2][g < n ? g : 0][c] : 0.0;
            ka[ks] = c / n;
            kk[ks] = (c % n) * VJ;
        }
        int rd[I], wo[I];
#pragma unroll
        for (int it = 0; it < I; ++it) {
            const int l = (w + NW * it) * 8 + x3_line(g, C::VL), lc = l < L2 ? l : L2 - 1;
            const int cell = lc / n2, r = lc - cell * n2;
            const int cx = cx0 + cell % TX, cy = cy0 + cell / TX;
            rd[it] = cell * VCS + r;
            // output offset within a node plane (int32: M1 M2 n^3 < 2^31 is checked at launch)
            wo[it] = (l < L2 && qout && cx < M1 && cy < M2) ? (cy * M1 + cx) * n3 + (2 * q) * n2 + r : -1;
        }
        mbar_wait(&v_full[0], 0u);
        int v0 = 0;  // buffer of V(c)
        for (int c = 0; c + 1 < P; ++c) {
            const int v1 = v0 == C::NVB - 1 ? 0 : v0 + 1;
            mbar_wait(&v_full[v1], (unsigned)(((c + 1) / C::NVB) & 1));
            const double* vk[KS];
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) vk[ks] = V + (ka[ks] ? v1 : v0) * C::V_D + kk[ks];
            double* oplane = dst + (zc0 + c) * plane_elems;
#pragma unroll
            for (int i0 = 0; i0 < I; i0 += C::B3) {
                double acc[C::B3][2];
#pragma unroll
                for (int j = 0; j < C::B3; ++j) {
                    const int it = i0 + j;
                    acc[j][0] = acc[j][1] = 0.0;
                    if (it >= I || !live<C::G2, NW>(w, it)) continue;
#pragma unroll
                    for (int ks = 0; ks < KS; ++ks) dmma(acc[j][0], acc[j][1], vk[ks][rd[it]], bop[ks]);
                }
                if (i0 + C::B3 >= I) mbar_arrive(&v_empty[v0]);  // V(c) read: release it (V(c+1) at c+1)
#pragma unroll
                for (int j = 0; j < C::B3; ++j) {
                    const int it = i0 + j;
                    if (it < I && live<C::G2, NW>(w, it) && wo[it] >= 0) {
                        __stcs(oplane + wo[it], acc[j][0]);
                        __stcs(oplane + wo[it] + n2, acc[j][1]);
                        if (!isfinite(acc[j][0]) || !isfinite(acc[j][1]))
                            flag_bad(first_bad, (zc0 + c) * M2 * (int64_t)M1 + wo[it] / n3);
                    }
                }
            }
            v0 = v1;
        }
    }
}

template <class C>
static int launch_ws(const double* src, double* dst, const Dims& d, const double* A, int off, cudaStream_t st,
                     unsigned long long* first_bad, const unsigned long long* guard) {
    const int64_t nz = d.z_end - d.z_begin;
    if (nz <= 0) return 0;
    if (d.M1 * d.M2 * C::n3 >= (int64_t(1) << 31)) return (int)cudaErrorInvalidValue;
    SepOps<5> ops;
    for (int k = 0; k < 3; ++k)
        for (int m = 0; m < C::n; ++m)
            for (int c = 0; c < 2 * C::n; ++c) {
                ops.A[k][m][c] = A[(k * C::n + m) * 2 * C::n + c];
                ops.Sh[k][m][c] = 0.0;
            }
    auto kern = sep_fused_dmma_ws_kernel<C>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return (int)e;
    const int64_t gx = (d.M1 + C::TX - 1) / C::TX, gy = (d.M2 + C::TY - 1) / C::TY;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::THREADS, C::SMEM);
    if (e != cudaSuccess) return (int)e;
    const int64_t zchunk = choose_zchunk(gx * gy, nz, (int64_t)num_sms() * (per_sm > 0 ? per_sm : 1));
    const int64_t gz = (nz + zchunk - 1) / zchunk;
    Dims db = d;
    db.band = band_width(H3_WS5_BAND);  // tile rasterisation (band_tile, h3_launch.h)
    kern<<<dim3((unsigned)gx, (unsigned)gy, (unsigned)gz), C::THREADS, C::SMEM, st>>>(src, dst, db, off, (int)zchunk,
                                                                                   ops, first_bad, guard);
    return (int)cudaGetLastError();
}

int sep_fused_dmma5_ws_launch(const double* src, double* dst, const Dims& d, const double* A, int off,
                              cudaStream_t st, unsigned long long* first_bad, const unsigned long long* guard,
                              int variant) {
#ifdef H3_MEASURE
    // tools library only (tools/ab.sh, H3_DMMA5_CFG = 20 + variant): the configurations of the r02
    // search, profiles/r02_m5_fused_variants.txt
    switch (variant) {
        case 1: return launch_ws<ws5::Cfg<4, 3, 8, 6, 6, 3, 3>>(src, dst, d, A, off, st, first_bad, guard);
        case 2: return launch_ws<ws5::Cfg<4, 3, 7, 6, 6, 3>>(src, dst, d, A, off, st, first_bad, guard);
        case 3: return launch_ws<ws5::Cfg<4, 3, 6, 5, 5, 3>>(src, dst, d, A, off, st, first_bad, guard);
        case 4: return launch_ws<ws5::Cfg<4, 3, 12, 9, 9, 2>>(src, dst, d, A, off, st, first_bad, guard);
        case 5: return launch_ws<ws5::Cfg<4, 3, 7, 6, 6, 3, 3>>(src, dst, d, A, off, st, first_bad, guard);
        case 6: return launch_ws<ws5::Cfg<4, 3, 9, 7, 7, 3, 3>>(src, dst, d, A, off, st, first_bad, guard);
        case 13: return launch_ws<ws5::Cfg<4, 3, 8, 6, 6, 3, 3, true>>(src, dst, d, A, off, st, first_bad, guard);
        case 16: return launch_ws<ws5::Cfg<3, 4, 8, 6, 6, 3, 3, true>>(src, dst, d, A, off, st, first_bad, guard);
        case 20: return launch_ws<ws5::Cfg<2, 6, 8, 6, 6, 2, 3, true, 2, 4>>(src, dst, d, A, off, st, first_bad, guard);
        case 21: return launch_ws<ws5::Cfg<2, 6, 8, 6, 6, 2, 3, true, 3, 3>>(src, dst, d, A, off, st, first_bad, guard);
        case 22: return launch_ws<ws5::Cfg<2, 6, 8, 6, 6, 3, 2, true>>(src, dst, d, A, off, st, first_bad, guard);
        case 23: return launch_ws<ws5::Cfg<2, 6, 8, 6, 6, 2, 3, true>>(src, dst, d, A, off, st, first_bad, guard);
        case 24: return launch_ws<ws5::Cfg<3, 4, 8, 6, 6, 2, 3, true, 2, 4>>(src, dst, d, A, off, st, first_bad, guard);
        case 25: return launch_ws<ws5::Cfg<2, 6, 7, 6, 6, 2, 3, true, 2, 4>>(src, dst, d, A, off, st, first_bad, guard);
        case 26: return launch_ws<ws5::Cfg<3, 4, 7, 6, 6, 2, 3, true, 2, 4>>(src, dst, d, A, off, st, first_bad, guard);
        case 27: return launch_ws<ws5::Cfg<2, 6, 7, 6, 6, 2, 0, true, 2, 4>>(src, dst, d, A, off, st, first_bad, guard);
        case 28: return launch_ws<ws5::Cfg<2, 6, 7, 6, 6, 2, 5, true, 2, 4>>(src, dst, d, A, off, st, first_bad, guard);
        case 29: return launch_ws<ws5::Cfg<2, 6, 7, 6, 6, 2, 1, true, 2, 4>>(src, dst, d, A, off, st, first_bad, guard);
        case 30: return launch_ws<ws5::Cfg<2, 6, 7, 6, 6, 2, 2, true, 2, 4>>(src, dst, d, A, off, st, first_bad, guard);
        // more x3 warps: the r02 ncu capture shows x1 and x2 waiting on their "empty" barriers
        // (343M / 304M retries) and x3 rarely waiting -- x3 paces the pipeline
        case 32: return launch_ws<ws5::Cfg<2, 6, 7, 6, 7, 2, 2, true, 2, 4>>(src, dst, d, A, off, st, first_bad, guard);
        case 33: return launch_ws<ws5::Cfg<2, 6, 7, 5, 7, 2, 2, true, 2, 4>>(src, dst, d, A, off, st, first_bad, guard);
        case 34: return launch_ws<ws5::Cfg<2, 6, 6, 6, 7, 2, 2, true, 2, 4>>(src, dst, d, A, off, st, first_bad, guard);
        case 35: return launch_ws<ws5::Cfg<2, 6, 7, 6, 8, 2, 2, true, 2, 4>>(src, dst, d, A, off, st, first_bad, guard);
        case 36: return launch_ws<ws5::Cfg<2, 6, 7, 7, 7, 2, 2, true, 2, 4>>(src, dst, d, A, off, st, first_bad, guard);
        case 37: return launch_ws<ws5::Cfg<2, 6, 7, 6, 9, 2, 2, true, 2, 4>>(src, dst, d, A, off, st, first_bad, guard);
        case 17: return launch_ws<ws5::Cfg<2, 6, 8, 6, 6, 3, 3, true>>(src, dst, d, A, off, st, first_bad, guard);
        case 18: return launch_ws<ws5::Cfg<3, 4, 9, 6, 6, 3, 3, true>>(src, dst, d, A, off, st, first_bad, guard);
        case 19: return launch_ws<ws5::Cfg<2, 6, 8, 7, 7, 3, 3, true>>(src, dst, d, A, off, st, first_bad, guard);
        case 14: return launch_ws<ws5::Cfg<4, 3, 8, 6, 6, 3, 2, true>>(src, dst, d, A, off, st, first_bad, guard);
        case 15: return launch_ws<ws5::Cfg<4, 3, 9, 6, 8, 3, 3, true>>(src, dst, d, A, off, st, first_bad, guard);
        case 7: return launch_ws<ws5::Cfg<4, 3, 9, 7, 7, 3, 2>>(src, dst, d, A, off, st, first_bad, guard);
        case 8: return launch_ws<ws5::Cfg<4, 3, 8, 6, 6, 3, 2>>(src, dst, d, A, off, st, first_bad, guard);
        case 9: return launch_ws<ws5::Cfg<4, 3, 8, 6, 6, 3, 4>>(src, dst, d, A, off, st, first_bad, guard);
        case 10: return launch_ws<ws5::Cfg<4, 3, 11, 8, 8, 3, 2>>(src, dst, d, A, off, st, first_bad, guard);
        case 11: return launch_ws<ws5::Cfg<4, 3, 8, 7, 7, 3, 3>>(src, dst, d, A, off, st, first_bad, guard);
        case 12: return launch_ws<ws5::Cfg<4, 3, 9, 6, 8, 3, 3>>(src, dst, d, A, off, st, first_bad, guard);
        case 99: return launch_ws<ws5::Cfg<4, 3, 8, 6, 6, 3>>(src, dst, d, A, off, st, first_bad, guard);
        default: break;
    }
#else
    (void)variant;
#endif
    // 2 x 6 cell tiles (x1 halo rows 7/6), 7 x1 + 6 x2 + 7 x3 warps + the TMA producer (x3 paces
    // the pipeline: 6 x3 warps 1 % slower), 2 TMA stages, W ring of 2, V ring of 4, 2 line groups
    // per batch (3: 1 % slower), the searched layouts: 14.8 ms per half step at 256^3 vs 17.6 ms
    // for the lock-step kernel (r02)
    return launch_ws<ws5::Cfg<2, 6, 7, 6, 7, 2, 2, true, 2, 4>>(src, dst, d, A, off, st, first_bad, guard);
}

}  // namespace h3
