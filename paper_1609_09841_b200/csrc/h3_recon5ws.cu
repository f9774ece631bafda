// Warp-specialised FP64 tensor-core reconstruction pass of the two-kernel step for N = 5 (n = 6):
// the cell-pair DMMA form of recon_dmma_cp_kernel (h3_dmma5.cu: K = 2n = 12 = three m8n8k4 k-steps,
// s = 12 outputs in two 8-column blocks, H shared by all axes) reorganised as a producer / consumer
// pipeline over node planes, like the fused N = 5 kernel of h3_dmma5ws.cu:
//
//   warp 0            TMA producer: tile rows of node plane t -> U[t % SU]
//   warps 1 .. N1     x1: line (node row, cell, j3 j2)  U[t % SU] -> W[t % NWB][row][cell][i1][j3 j2]
//   next N2 warps     x2: line (cell, j3, i1)           W[t % NWB] -> V[t % NVB][cell][j3][i2 i1]
//   last N3 warps     x3: line (cell, i2 i1)            V(c), V(c+1) -> coefficient cell plane c (HBM)
//
// The reconstruction is DMMA-bound (202 DMMAs per cell against 15.6 KB of HBM traffic: 810 pipe
// cycles vs ~690 memory cycles per cell per SM at 1.96 GHz); the lock-step kernel keeps the DMMA
// pipe ~70 % busy because every CTA barrier drains it; here the three passes of consecutive planes
// overlap (77 %, profiles/r02_two5_128_recon_dmma_ws_summary.json).  Layouts: x1 reads K in the
// searched conflict-free order of the fused kernel; the V ring stride is 8 (mod 16) doubles so the
// x3 k-steps that straddle V(c) and V(c+1) stay on distinct bank pairs
// (tools/rcp5_ws_layout_search.py).
//
// Phases as in h3_dmma5ws.cu: "full" waits use parity (use / ring) & 1, first "empty" waits pass at
// once; every lane of a releasing role arrives.
#include "h3_launch.h"
#include "h3_tma.cuh"

#ifndef H3_RWS5_BAND
#define H3_RWS5_BAND 0
#endif

namespace h3 {
namespace rws5 {

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

// x1 K order (vertex q >> 1, component 2 ks + (q & 1)): a half-warp's loads on 16 bank pairs
__device__ __forceinline__ int korder_x1(int ks, int q) {
    constexpr unsigned T[3] = {0x7610u, 0x9832u, 0xba54u};
    return (int)((T[ks] >> (4 * q)) & 15u);
}

template <int TX_, int TY_, int N1_, int N2_, int N3_, int SU_, int NWB_, int NVB_, int B_ = 3>
struct Cfg {
    static constexpr int N = 5, n = 6, n2 = 36, n3 = 216, S = 12, S2 = 144, S3 = 1728, KS = 3, CB = 2;
    static constexpr int TX = TX_, TY = TY_, NX = TX + 1, NY = TY + 1, NNODE = NX * NY;
    static constexpr int N1 = N1_, N2 = N2_, N3 = N3_, SU = SU_, NWB = NWB_, NVB = NVB_, B = B_;
    static constexpr int WARPS = 1 + N1 + N2 + N3, THREADS = 32 * WARPS;
    static constexpr int UNS = n3;
    static constexpr int WI = n2 + 1, WCS = S * WI;  // W: [node row][cell][i1][j3 j2]
    static constexpr int VJ = S2 + 4, VCS = n * VJ;  // V: [cell][j3][i2 i1] (j3 stride 4 mod 16)
    static constexpr int L1 = NY * TX * n2, L2 = TY * TX * n * S, L3 = TY * TX * S2;
    static constexpr int G1 = (L1 + 7) / 8, G2 = (L2 + 7) / 8, G3 = (L3 + 7) / 8;
    static constexpr int I1 = (G1 + N1 - 1) / N1, I2 = (G2 + N2 - 1) / N2, I3 = (G3 + N3 - 1) / N3;
    static constexpr size_t U_D = (size_t)NNODE * UNS;
    static constexpr size_t W_D = (size_t)NY * TX * WCS;
    // V ring stride: == 8 (mod 16) doubles, so V(c) and V(c+1) sit half a bank row apart (NVB even
    // keeps the wrap-around pair apart too)
    static constexpr size_t V_D = ((size_t)TY * TX * VCS + 15) / 16 * 16 + 8;
    static constexpr int NBAR = 2 * (SU + NWB + NVB);
    static constexpr size_t SMEM_DATA = (SU * U_D + NWB * W_D + NVB * V_D) * sizeof(double);
    static constexpr size_t SMEM = SMEM_DATA + NBAR * sizeof(uint64_t);
    static_assert(NY <= 32, "one producer lane per tile row");
    static_assert(NWB >= 1 && NVB >= 2 && NVB % 2 == 0, "x3 reads two V planes; even ring keeps banks apart");
    static_assert(SMEM <= 232448, "shared memory per CTA");
};

template <int G, int NW>
__device__ __forceinline__ bool live(int w, int it) {
    return G % NW == 0 || w + NW * it < G;
}

}  // namespace rws5

template <class C>
__global__ void __launch_bounds__(C::THREADS, 1)
recon_dmma_ws_kernel(const double* __restrict__ src, double* __restrict__ coeff, Dims d, int off, int zchunk,
                     const __grid_constant__ LitOps<double, 5> hp, const unsigned long long* guard) {
    using namespace rws5;
    constexpr int n = C::n, n2 = C::n2, n3 = C::n3, S = C::S, S2 = C::S2, S3 = C::S3, KS = C::KS, CB = C::CB;
    constexpr int TX = C::TX, NX = C::NX, NY = C::NY, SU = C::SU, NWB = C::NWB, NVB = C::NVB, UNS = C::UNS;
    constexpr int WI = C::WI, WCS = C::WCS, VJ = C::VJ, VCS = C::VCS, L1 = C::L1, L2 = C::L2, L3 = C::L3;
    constexpr int B = C::B;
    if (guarded_out(guard, nullptr)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* U = reinterpret_cast<double*>(smem_raw);
    double* W = U + SU * C::U_D;
    double* V = W + NWB * C::W_D;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + C::SMEM_DATA);
    uint64_t* u_full = bars;
    uint64_t* u_empty = u_full + SU;
    uint64_t* w_full = u_empty + SU;
    uint64_t* w_empty = w_full + NWB;
    uint64_t* v_full = w_empty + NWB;
    uint64_t* v_empty = v_full + NVB;

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
    const int64_t cplane = (int64_t)M1 * M2 * S3;

    if (tid == 0) {
        for (int s = 0; s < SU; ++s) {
            mbar_init(&u_full[s], 1);
            mbar_init(&u_empty[s], 32 * C::N1);
        }
        for (int b = 0; b < NWB; ++b) {
            mbar_init(&w_full[b], 32 * C::N1);
            mbar_init(&w_empty[b], 32 * C::N2);
        }
        for (int b = 0; b < NVB; ++b) {
            mbar_init(&v_full[b], 32 * C::N2);
            mbar_init(&v_empty[b], 32 * C::N3);
        }
        mbar_fence_init();
    }
    __syncthreads();

    // output columns of this lane: 8 cb + 2q (+1); the second block holds 4 of its 8 columns
    const bool cout1 = 8 * (CB - 1) + 2 * q < S;
    // B fragment: lane holds B[k][col = 8 cb + g] = H[8 cb + g][k] (zero for col >= s)
    auto hfrag = [&](int cb, int k) {
        const int col = 8 * cb + g;
        return col < S ? hp.H[(col < S ? col : 0) * S + k] : 0.0;
    };

    if (warp == 0) {
        // ---- producer -----------------------------------------------------------------------------
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

    if (warp <= C::N1) {
        // ---- x1: U(t) -> W ------------------------------------------------------------------------
        constexpr int NW = C::N1, I = C::I1;
        const int w = warp - 1;
        double bop[KS][CB];
        int kk[KS];
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            const int c = korder_x1(ks, q);
            kk[ks] = (c / n) * UNS + c % n;
#pragma unroll
            for (int cb = 0; cb < CB; ++cb) bop[ks][cb] = hfrag(cb, c);
        }
        int rd[I], wr[I];
#pragma unroll
        for (int it = 0; it < I; ++it) {
            const int l = (w + NW * it) * 8 + g, lc = l < L1 ? l : L1 - 1;
            const int rc = lc / n2, jj = lc - rc * n2, ly = rc / TX, cx = rc - ly * TX;
            rd[it] = (ly * NX + cx) * UNS + jj * n;
            wr[it] = l < L1 ? rc * WCS + (2 * q) * WI + jj : -1;
        }
        for (int t = 0; t < P; ++t) {
            const int s = t % SU, b = t % NWB;
            mbar_wait(&u_full[s], (unsigned)((t / SU) & 1));
            mbar_wait(&w_empty[b], (unsigned)(((t / NWB) & 1) ^ 1));
            const double* Ub = U + s * C::U_D;
            double* Wb = W + b * C::W_D;
#pragma unroll
            for (int i0 = 0; i0 < I; i0 += B) {
                double acc[B][CB][2];
#pragma unroll
                for (int j = 0; j < B; ++j) {
                    const int it = i0 + j;
#pragma unroll
                    for (int cb = 0; cb < CB; ++cb) acc[j][cb][0] = acc[j][cb][1] = 0.0;
                    if (it >= I || !live<C::G1, NW>(w, it)) continue;
                    double a[KS];
#pragma unroll
                    for (int ks = 0; ks < KS; ++ks) a[ks] = Ub[rd[it] + kk[ks]];
#pragma unroll
                    for (int cb = 0; cb < CB; ++cb)
#pragma unroll
                        for (int ks = 0; ks < KS; ++ks) dmma(acc[j][cb][0], acc[j][cb][1], a[ks], bop[ks][cb]);
                }
#pragma unroll
                for (int j = 0; j < B; ++j) {
                    const int it = i0 + j;
                    if (it >= I || !live<C::G1, NW>(w, it) || wr[it] < 0) continue;
#pragma unroll
                    for (int cb = 0; cb < CB; ++cb)
                        if (cb < CB - 1 || cout1) {
                            Wb[wr[it] + 8 * cb * WI] = acc[j][cb][0];
                            Wb[wr[it] + (8 * cb + 1) * WI] = acc[j][cb][1];
                        }
                }
            }
            mbar_arrive(&u_empty[s]);
            mbar_arrive(&w_full[b]);
        }
    } else if (warp <= C::N1 + C::N2) {
        // ---- x2: W -> V[t % NVB] -------------------------------------------------------------------
        constexpr int NW = C::N2, I = C::I2;
        const int w = warp - 1 - C::N1;
        double bop[KS][CB];
        int kk[KS];
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            const int c = 4 * ks + q;
            kk[ks] = (c / n) * TX * WCS + c % n;
#pragma unroll
            for (int cb = 0; cb < CB; ++cb) bop[ks][cb] = hfrag(cb, c);
        }
        int rd[I], wr[I];
#pragma unroll
        for (int it = 0; it < I; ++it) {
            const int l = (w + NW * it) * 8 + g, lc = l < L2 ? l : L2 - 1;
            const int cell = lc / (n * S), r = lc - cell * (n * S), j3 = r / S, i1 = r - j3 * S;
            rd[it] = cell * WCS + i1 * WI + j3 * n;
            wr[it] = l < L2 ? cell * VCS + j3 * VJ + (2 * q) * S + i1 : -1;
        }
        for (int t = 0; t < P; ++t) {
            const int b = t % NWB, v = t % NVB;
            mbar_wait(&w_full[b], (unsigned)((t / NWB) & 1));
            mbar_wait(&v_empty[v], (unsigned)(((t / NVB) & 1) ^ 1));
            const double* Wb = W + b * C::W_D;
            double* Vb = V + v * C::V_D;
#pragma unroll
            for (int i0 = 0; i0 < I; i0 += B) {
                double acc[B][CB][2];
#pragma unroll
                for (int j = 0; j < B; ++j) {
                    const int it = i0 + j;
#pragma unroll
                    for (int cb = 0; cb < CB; ++cb) acc[j][cb][0] = acc[j][cb][1] = 0.0;
                    if (it >= I || !live<C::G2, NW>(w, it)) continue;
                    double a[KS];
#pragma unroll
                    for (int ks = 0; ks < KS; ++ks) a[ks] = Wb[rd[it] + kk[ks]];
#pragma unroll
                    for (int cb = 0; cb < CB; ++cb)
#pragma unroll
                        for (int ks = 0; ks < KS; ++ks) dmma(acc[j][cb][0], acc[j][cb][1], a[ks], bop[ks][cb]);
                }
#pragma unroll
                for (int j = 0; j < B; ++j) {
                    const int it = i0 + j;
                    if (it >= I || !live<C::G2, NW>(w, it) || wr[it] < 0) continue;
#pragma unroll
                    for (int cb = 0; cb < CB; ++cb)
                        if (cb < CB - 1 || cout1) {
                            Vb[wr[it] + 8 * cb * S] = acc[j][cb][0];
                            Vb[wr[it] + (8 * cb + 1) * S] = acc[j][cb][1];
                        }
                }
            }
            mbar_arrive(&w_empty[b]);
            mbar_arrive(&v_full[v]);
        }
    } else {
        // ---- x3: V(c), V(c+1) -> coefficient cell plane c ------------------------------------------
        constexpr int NW = C::N3, I = C::I3;
        const int w = warp - 1 - C::N1 - C::N2;
        double bop[KS][CB];
        int kk[KS], ka[KS];
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            const int c = 4 * ks + q;
            ka[ks] = c / n;
            kk[ks] = (c % n) * VJ;
#pragma unroll
            for (int cb = 0; cb < CB; ++cb) bop[ks][cb] = hfrag(cb, c);
        }
        int rd[I], wo[I];
#pragma unroll
        for (int it = 0; it < I; ++it) {
            const int l = (w + NW * it) * 8 + g, lc = l < L3 ? l : L3 - 1;
            const int cell = lc / S2, r = lc - cell * S2;
            const int cx = cell % TX, cy = cell / TX;
            rd[it] = cell * VCS + r;
            // relative to the tile's first cell (int32 up to M1 < 2^31 / (TY S^3)): the coefficient
            // plane itself (M1 M2 S^3 doubles) may exceed 2^31 elements
            wo[it] = (l < L3 && cx0 + cx < M1 && cy0 + cy < M2) ? (cy * M1 + cx) * S3 + (2 * q) * S2 + r : -1;
        }
        mbar_wait(&v_full[0], 0u);
        int v0 = 0;  // buffer of V(c)
        for (int c = 0; c + 1 < P; ++c) {
            const int v1 = v0 == NVB - 1 ? 0 : v0 + 1;
            mbar_wait(&v_full[v1], (unsigned)(((c + 1) / NVB) & 1));
            const double* vk[KS];
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) vk[ks] = V + (ka[ks] ? v1 : v0) * C::V_D + kk[ks];
            double* oplane = coeff + (zc0 - d.z_begin + c) * cplane + ((int64_t)cy0 * M1 + cx0) * S3;
#pragma unroll
            for (int i0 = 0; i0 < I; i0 += B) {
                double acc[B][CB][2];
                double a[B][KS];
#pragma unroll
                for (int j = 0; j < B; ++j) {
                    const int it = i0 + j;
                    if (it >= I || !live<C::G3, NW>(w, it)) continue;
#pragma unroll
                    for (int ks = 0; ks < KS; ++ks) a[j][ks] = vk[ks][rd[it]];
                }
                if (i0 + B >= I) mbar_arrive(&v_empty[v0]);  // last reads of V(c) issued
#pragma unroll
                for (int j = 0; j < B; ++j) {
                    const int it = i0 + j;
#pragma unroll
                    for (int cb = 0; cb < CB; ++cb) acc[j][cb][0] = acc[j][cb][1] = 0.0;
                    if (it >= I || !live<C::G3, NW>(w, it)) continue;
#pragma unroll
                    for (int cb = 0; cb < CB; ++cb)
#pragma unroll
                        for (int ks = 0; ks < KS; ++ks) dmma(acc[j][cb][0], acc[j][cb][1], a[j][ks], bop[ks][cb]);
                }
#pragma unroll
                for (int j = 0; j < B; ++j) {
                    const int it = i0 + j;
                    if (it >= I || !live<C::G3, NW>(w, it) || wo[it] < 0) continue;
#pragma unroll
                    for (int cb = 0; cb < CB; ++cb)
                        if (cb < CB - 1 || cout1) {
                            __stcs(oplane + wo[it] + 8 * cb * S2, acc[j][cb][0]);
                            __stcs(oplane + wo[it] + (8 * cb + 1) * S2, acc[j][cb][1]);
                        }
                }
            }
            v0 = v1;
        }
    }
}

template <class C>
static int launch_rws5(const double* src, double* coeff, const Dims& d, const double* h_mat, int off,
                       cudaStream_t st, const unsigned long long* guard) {
    const int64_t nz = d.z_end - d.z_begin;
    if (nz <= 0) return 0;
    if (d.M1 * d.M2 * C::n3 >= (int64_t(1) << 31) || d.M1 * C::TY * C::S3 >= (int64_t(1) << 31))
        return (int)cudaErrorInvalidValue;  // int32 node-plane / tile-relative output offsets
    LitOps<double, 5> hp;
    for (int i = 0; i < C::S2; ++i) hp.H[i] = h_mat[i];
    for (int i = 0; i < C::S; ++i) hp.f1[i] = hp.f2[i] = hp.f3[i] = 0.0;
    for (int i = 0; i < H3_MAX_STAGES; ++i) hp.cf[i] = 0.0;
    hp.q = 0;
    auto kern = recon_dmma_ws_kernel<C>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return (int)e;
    const int64_t gx = (d.M1 + C::TX - 1) / C::TX, gy = (d.M2 + C::TY - 1) / C::TY;
    const int64_t zchunk = choose_zchunk(gx * gy, nz, num_sms());  // one CTA per SM
    const int64_t gz = (nz + zchunk - 1) / zchunk;
    Dims db = d;
    db.band = band_width(H3_RWS5_BAND);  // tile rasterisation (band_tile, h3_launch.h)
    kern<<<dim3((unsigned)gx, (unsigned)gy, (unsigned)gz), C::THREADS, C::SMEM, st>>>(src, coeff, db, off, (int)zchunk,
                                                                                   hp, guard);
    return (int)cudaGetLastError();
}

int recon_dmma5_ws_launch(const double* src, double* coeff, const Dims& d, const double* h_mat, int off,
                          cudaStream_t st, const unsigned long long* guard, int variant) {
    using rws5::Cfg;
#ifdef H3_MEASURE
    // tools library only (H3_RECON5_WS=k): the r02 search, profiles/r02_m5_recon_ws.txt
    switch (variant) {
        // TX, TY, N1, N2, N3, SU, NWB, NVB, B
        case 1: return launch_rws5<Cfg<2, 2, 3, 4, 8, 2, 2, 4>>(src, coeff, d, h_mat, off, st, guard);
        case 3: return launch_rws5<Cfg<2, 2, 3, 4, 8, 2, 2, 4, 2>>(src, coeff, d, h_mat, off, st, guard);
        case 8: return launch_rws5<Cfg<2, 4, 3, 4, 8, 2, 1, 2, 2>>(src, coeff, d, h_mat, off, st, guard);
        case 9: return launch_rws5<Cfg<2, 2, 3, 4, 8, 3, 2, 4, 2>>(src, coeff, d, h_mat, off, st, guard);
        case 10: return launch_rws5<Cfg<2, 2, 6, 8, 16, 2, 2, 4, 1>>(src, coeff, d, h_mat, off, st, guard);
        default: break;
    }
#else
    (void)variant;
#endif
    // 2 x 2 cell tiles, 3 x1 + 4 x2 + 8 x3 warps (9 line groups each per plane) + the TMA producer,
    // 2 TMA stages, W ring of 2, V ring of 4, one line group per batch: 4.3 % faster m=5 two-kernel
    // step than the lock-step reconstruction at 256^3, DMMA pipe 70 -> 74 % (r02)
    return launch_rws5<Cfg<2, 2, 3, 4, 8, 2, 2, 4, 1>>(src, coeff, d, h_mat, off, st, guard);
}

}  // namespace h3
