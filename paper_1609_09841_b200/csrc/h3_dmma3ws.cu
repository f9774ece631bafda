// Warp-specialised FP64 tensor-core fused half step for N = 3 (n = 4): the node-factorised,
// alternating-column rolling DMMA form of h3_dmma.cu (same operators, same shared layouts, same
// per-pass lane code), reorganised as a producer / consumer pipeline over node planes instead of a
// lock-step march with CTA-wide barriers (the m = 5 kernel h3_dmma5ws.cu does the same for the
// cell-pair form).
//
//   warp 0            TMA producer: bulk-copies the tile rows of node plane t into U[t % SU]
//   warps 1 .. N1     x1: (node row, line half) chains walk their row      U[t % SU] -> W[t % NWB]
//   next N2 warps     x2: (cell column, line half) chains walk their column W[t % NWB] -> V[t % NVB]
//   last N3 warps     x3: (cell, line half) chains carried across planes    V[t % NVB] -> dst plane t-1
//
// Each consumer loads its whole input for the plane into registers first and releases the buffer
// at once (an mbarrier "empty" arrive), then runs its DMMA chains and writes its output buffer,
// released to the next role by a "full" arrive.  So x1 of plane t, x2 of plane t-1 and x3 of
// plane t-2 overlap, and the DMMA pipe sees a steady mix of the three passes instead of draining
// at every CTA barrier (lock-step kernel: DMMA pipe 48 % busy, issue 43 %, top stalls wait /
// short-scoreboard / math-pipe-throttle in bursts, profiles/r01_sep_fused_dmma3_512_summary.json).
//
// Phases: the k-th use of a buffer waits for the k-th completion of its "full" barrier (parity
// k & 1); a producer's first wait on an "empty" barrier passes at once (parity 1 of a fresh
// barrier).  Every lane of a releasing role arrives (counts 32 x warps), so each lane's own
// shared-memory accesses are ordered by its own release.
// Measurement-only (tools build, -DH3_MEASURE): measured slower than the lock-step kernel, see
// profiles/r02_m3_fused_variants.txt; the product library does not contain it.
#ifdef H3_MEASURE
#include "h3_launch.h"
#include "h3_tma.cuh"

namespace h3 {
namespace ws3 {

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

// ~hi(x) & 0x7ff00000 in one LOP3: zero iff x is Inf/NaN (exponent all ones)
__device__ __forceinline__ unsigned exp_gap(double x) {
    unsigned r;
    asm("lop3.b32 %0, %1, 0x7ff00000, 0, 0x0c;" : "=r"(r) : "r"((unsigned)__double2hiint(x)));
    return r;
}

template <int TY_, int N1_, int N2_, int N3_, int SU_, int NWB_, int NVB_, int B3_ = 4>
struct Cfg {
    static constexpr int B3 = B3_;  // x3 chains per batch
    static constexpr int n = 4, n3 = 64;
    static constexpr int TX = 8, TY = TY_, NX = TX + 1, NY = TY + 1, NCOL = NX * NY;
    static constexpr int N1 = N1_, N2 = N2_, N3 = N3_, SU = SU_, NWB = NWB_, NVB = NVB_;
    static constexpr int WARPS = 1 + N1 + N2 + N3, THREADS = 32 * WARPS;
    static constexpr int UNS = 64;                           // U node stride (dense [j3][j2][j1])
    static constexpr int WRS = 20, WCS = 84;                 // W [j3][m1][j2]: j3 stride, cell stride
    static constexpr int VRS = 17, VCS = 68, VROW = TX * VCS + 1;  // V [m2][m1][j3]; cell row stride
    static constexpr int T1 = 2 * NY, K1 = (T1 + N1 - 1) / N1;     // x1 (row, half) tasks per warp
    static constexpr int T2 = 2 * TX, K2 = (T2 + N2 - 1) / N2;     // x2 (column, half) tasks per warp
    static constexpr int T3 = 2 * TX * TY, K3 = (T3 + N3 - 1) / N3;  // x3 chains per warp
    static constexpr size_t U_D = (size_t)NCOL * UNS;
    static constexpr size_t W_D = (size_t)NY * TX * WCS;
    static constexpr size_t V_D = (size_t)TY * VROW;
    static constexpr int NBAR = 2 * (SU + NWB + NVB);
    static constexpr size_t SMEM_DATA = (SU * U_D + NWB * W_D + NVB * V_D) * sizeof(double);
    static constexpr size_t SMEM = SMEM_DATA + NBAR * sizeof(uint64_t);
    static_assert(NY <= 32, "one producer lane per tile row");
    static_assert(SU >= 2 && NWB >= 1 && NVB >= 1, "ring lengths");
    static_assert(SMEM <= 232448, "shared memory per CTA");
};

}  // namespace ws3

template <class C>
__global__ void __launch_bounds__(C::THREADS, 1)
sep_fused_dmma3_ws_kernel(const double* __restrict__ src, double* __restrict__ dst, Dims d, int off, int zchunk,
                          const __grid_constant__ SepOps<3> p, unsigned long long* first_bad,
                          const unsigned long long* guard) {
    using namespace ws3;
    constexpr int n = C::n, n3 = C::n3, TX = C::TX, NX = C::NX, NY = C::NY;
    constexpr int SU = C::SU, NWB = C::NWB, NVB = C::NVB, UNS = C::UNS;
    constexpr int WRS = C::WRS, WCS = C::WCS, VRS = C::VRS, VCS = C::VCS, VROW = C::VROW;
    if (guarded_out(guard, first_bad)) return;
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
    const int q = lane & 3, g = lane >> 2, par = q >> 1;  // fragment coordinates
    const int M1 = (int)d.M1, M2 = (int)d.M2;
    const int cx0 = blockIdx.x * TX, cy0 = blockIdx.y * C::TY;
    const int64_t zc0 = d.z_begin + (int64_t)blockIdx.z * zchunk;
    const int64_t zc1 = min(zc0 + (int64_t)zchunk, d.z_end);
    const int P = (int)(zc1 - zc0) + 1;  // node planes of this chunk
    const int64_t plane_elems = (int64_t)M1 * M2 * n3;

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

    // operator fragment of an axis: lane holds B[k = q][col = g] for both column orders
    auto frag = [&](int ax, double& b0, double& b1) {
        const int m = g & 3, hi = g >> 2;
        b0 = hi ? p.A[ax][m][n + q] : p.A[ax][m][q];
        b1 = hi ? p.A[ax][m][q] : p.A[ax][m][n + q];
    };

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
                mbar_arrive_expect_tx(&u_full[s], (unsigned)(C::NCOL * UNS * sizeof(double)));
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
        // ---- x1: (row ly, half h) chains walk the NX nodes of their row -------------------------
        // Completed cells alternate between the lane halves; an even cell's values are held one
        // node longer so both halves store together (full-warp STS).
        constexpr int NW = C::N1, K1 = C::K1;
        const int w = warp - 1;
        double b0, b1;
        frag(0, b0, b1);
        int ua[K1], wrow[K1];
        bool live[K1];
#pragma unroll
        for (int j = 0; j < K1; ++j) {
            const int t = w + NW * j;
            live[j] = C::T1 % NW == 0 || t < C::T1;
            const int ly = live[j] ? t >> 1 : 0, h = t & 1;
            const int L = 8 * h + g;  // line (j3, j2) = (L >> 2, L & 3)
            ua[j] = ly * NX * UNS + L * 4 + q;
            wrow[j] = ly * TX * WCS + (2 * h + (g >> 2)) * WRS + (g & 3) + (2 * (q & 1)) * 4;
        }
        for (int t = 0; t < P; ++t) {
            const int s = t % SU, b = t % NWB;
            mbar_wait(&u_full[s], (unsigned)((t / SU) & 1));
            const double* Ub = U + s * C::U_D;
            double a[K1][NX];
#pragma unroll
            for (int j = 0; j < K1; ++j)
#pragma unroll
                for (int lx = 0; lx < NX; ++lx) a[j][lx] = live[j] ? Ub[ua[j] + lx * UNS] : 0.0;
            mbar_arrive(&u_empty[s]);
            mbar_wait(&w_empty[b], (unsigned)(((t / NWB) & 1) ^ 1));
            double* Wb = W + b * C::W_D;
            double r[K1][2], sv[K1][2];
#pragma unroll
            for (int j = 0; j < K1; ++j) r[j][0] = r[j][1] = sv[j][0] = sv[j][1] = 0.0;
#pragma unroll
            for (int lx = 0; lx < NX; ++lx) {
                const bool done = par == ((lx + 1) & 1);  // cell lx-1 completed in these lanes
#pragma unroll
                for (int j = 0; j < K1; ++j) {
                    dmma(r[j][0], r[j][1], a[j][lx], (lx & 1) ? b1 : b0);
                    if (lx & 1) {
                        sv[j][0] = r[j][0];
                        sv[j][1] = r[j][1];
                    } else if (lx > 0 && live[j]) {
                        double* wp = Wb + wrow[j] + (lx - 1 - (par ^ 1)) * WCS;
                        wp[0] = par ? r[j][0] : sv[j][0];
                        wp[4] = par ? r[j][1] : sv[j][1];
                    }
                    r[j][0] = done ? 0.0 : r[j][0];
                    r[j][1] = done ? 0.0 : r[j][1];
                }
            }
            mbar_arrive(&w_full[b]);
        }
    } else if (warp <= C::N1 + C::N2) {
        // ---- x2: (column ix, half h) chains walk the NY rows of their column --------------------
        constexpr int NW = C::N2, K2 = C::K2;
        const int w = warp - 1 - C::N1;
        double b0, b1;
        frag(1, b0, b1);
        int wa[K2], vcol[K2];
        bool live[K2];
#pragma unroll
        for (int j = 0; j < K2; ++j) {
            const int t = w + NW * j;
            live[j] = C::T2 % NW == 0 || t < C::T2;
            const int ix = live[j] ? t >> 1 : 0, h = t & 1;
            const int L = 8 * h + g;  // line (j3, m1) = (L >> 2, L & 3)
            wa[j] = ix * WCS + (L >> 2) * WRS + (L & 3) * 4 + q;
            vcol[j] = ix * VCS + (L & 3) * 4 + (L >> 2) + (2 * (q & 1)) * VRS;
        }
        for (int t = 0; t < P; ++t) {
            const int b = t % NWB, v = t % NVB;
            mbar_wait(&w_full[b], (unsigned)((t / NWB) & 1));
            const double* Wb = W + b * C::W_D;
            double a[K2][NY];
#pragma unroll
            for (int j = 0; j < K2; ++j)
#pragma unroll
                for (int ly = 0; ly < NY; ++ly) a[j][ly] = live[j] ? Wb[wa[j] + ly * TX * WCS] : 0.0;
            mbar_arrive(&w_empty[b]);
            mbar_wait(&v_empty[v], (unsigned)(((t / NVB) & 1) ^ 1));
            double* Vb = V + v * C::V_D;
            double r[K2][2], sv[K2][2];
#pragma unroll
            for (int j = 0; j < K2; ++j) r[j][0] = r[j][1] = sv[j][0] = sv[j][1] = 0.0;
#pragma unroll
            for (int ly = 0; ly < NY; ++ly) {
                const bool done = par == ((ly + 1) & 1);
#pragma unroll
                for (int j = 0; j < K2; ++j) {
                    dmma(r[j][0], r[j][1], a[j][ly], (ly & 1) ? b1 : b0);
                    if (ly & 1) {
                        if (ly == NY - 1) {  // lone last cell row: half-warp store
                            if (done && live[j]) {
                                double* vp = Vb + vcol[j] + (ly - 1) * VROW;
                                vp[0] = r[j][0];
                                vp[VRS] = r[j][1];
                            }
                        } else {
                            sv[j][0] = r[j][0];
                            sv[j][1] = r[j][1];
                        }
                    } else if (ly > 0 && live[j]) {
                        double* vp = Vb + vcol[j] + (ly - 1 - (par ^ 1)) * VROW;
                        vp[0] = par ? r[j][0] : sv[j][0];
                        vp[VRS] = par ? r[j][1] : sv[j][1];
                    }
                    r[j][0] = done ? 0.0 : r[j][0];
                    r[j][1] = done ? 0.0 : r[j][1];
                }
            }
            mbar_arrive(&v_full[v]);
        }
    } else {
        // ---- x3: each warp advances its chains by one plane per node plane ----------------------
        constexpr int NW = C::N3, K3 = C::K3;
        const int w = warp - 1 - C::N1 - C::N2;
        double b0, b1;
        frag(2, b0, b1);
        int va[K3], ooff[K3];
#pragma unroll
        for (int k = 0; k < K3; ++k) {
            const int t = w + NW * k;
            const bool lv = C::T3 % NW == 0 || t < C::T3;
            const int cell = lv ? t >> 1 : 0, h = t & 1;
            const int L = 8 * h + g;  // line (m2, m1) = (L >> 2, L & 3)
            va[k] = (cell / TX) * VROW + (cell % TX) * VCS + (L >> 2) * VRS + (L & 3) * 4 + q;
            const int cx = cx0 + (cell % TX), cy = cy0 + cell / TX;
            // the lane's output offset within a node plane (int32: M1 M2 64 < 2^31 checked at launch)
            ooff[k] = (lv && cx < M1 && cy < M2) ? (cy * M1 + cx) * n3 + (2 * (q & 1)) * 16 + 8 * h + g : -1;
        }
        double acc[K3][2];
#pragma unroll
        for (int k = 0; k < K3; ++k) acc[k][0] = acc[k][1] = 0.0;
        for (int t = 0; t < P; ++t) {
            const int v = t % NVB;
            mbar_wait(&v_full[v], (unsigned)((t / NVB) & 1));
            const double* Vb = V + v * C::V_D;
            double* oplane = dst + (zc0 + t - 1) * plane_elems;
            asm volatile("" : "+l"(oplane));  // one 64-bit plane base, 32-bit lane offsets
            unsigned screen = 0x7ff00000u;
            // chains in batches of B3 (bounds the live temporaries); chain k runs with column phase
            // (t + k) & 1, so the completed cell plane t-1 sits in the lanes with par == (t+k+1) & 1
#pragma unroll
            for (int k0 = 0; k0 < K3; k0 += C::B3) {
                constexpr int B = C::B3;
                double a[B], o0[B], o1[B];
#pragma unroll
                for (int b = 0; b < B; ++b)
                    if (k0 + b < K3) a[b] = Vb[va[k0 + b]];
                if (k0 + B >= K3) mbar_arrive(&v_empty[v]);  // last reads of V(t) issued
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    const int k = k0 + b;
                    if (k >= K3) continue;
                    dmma(acc[k][0], acc[k][1], a[b], ((t + k) & 1) ? b1 : b0);
                    const bool done = par == ((t + k + 1) & 1);
                    o0[b] = acc[k][0];
                    o1[b] = acc[k][1];
                    acc[k][0] = done ? 0.0 : acc[k][0];
                    acc[k][1] = done ? 0.0 : acc[k][1];
                }
                if (t > 0) {
#pragma unroll
                    for (int b = 0; b < B; ++b) {
                        const int k = k0 + b;
                        if (k >= K3) continue;
                        const bool done = par == ((t + k + 1) & 1);
                        if (done && ooff[k] >= 0) {
                            __stcs(oplane + ooff[k], o0[b]);
                            __stcs(oplane + ooff[k] + 16, o1[b]);
                            screen = min(screen, min(exp_gap(o0[b]), exp_gap(o1[b])));
                        }
                    }
                }
            }
            if (screen == 0u) {  // rare: a finished value is Inf/NaN -- locate it exactly
                // (this thread's own stores, read back in program order)
#pragma unroll
                for (int k = 0; k < K3; ++k) {
                    const bool done = par == ((t + k + 1) & 1);
                    if (done && ooff[k] >= 0 &&
                        (!isfinite(oplane[ooff[k]]) || !isfinite(oplane[ooff[k] + 16])))
                        flag_bad(first_bad, (zc0 + t - 1) * M2 * (int64_t)M1 + ooff[k] / n3);
                }
            }
        }
    }
}

template <class C>
static int launch_ws3(const double* src, double* dst, const Dims& d, const SepOps<3>& ops, int off,
                      cudaStream_t st, unsigned long long* first_bad, const unsigned long long* guard,
                      int cluster_y) {
    const int64_t nz = d.z_end - d.z_begin;
    auto kern = sep_fused_dmma3_ws_kernel<C>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return (int)e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::THREADS, C::SMEM);
    if (e != cudaSuccess) return (int)e;
    const int64_t gx = (d.M1 + C::TX - 1) / C::TX, gy = (d.M2 + C::TY - 1) / C::TY;
    const int64_t zchunk = choose_zchunk(gx * gy, nz, (int64_t)num_sms() * (per_sm > 0 ? per_sm : 1));
    const int64_t gz = (nz + zchunk - 1) / zchunk;
    if (cluster_y > 1 && gy % cluster_y == 0) {
        // clusters of y-adjacent tiles: co-scheduled, so their shared node row stays in L2
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3((unsigned)gx, (unsigned)gy, (unsigned)gz);
        lc.blockDim = dim3(C::THREADS);
        lc.dynamicSmemBytes = C::SMEM;
        lc.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 1;
        at[0].val.clusterDim.y = cluster_y;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        return (int)cudaLaunchKernelEx(&lc, kern, src, dst, d, off, (int)zchunk, ops, first_bad, guard);
    }
    kern<<<dim3((unsigned)gx, (unsigned)gy, (unsigned)gz), C::THREADS, C::SMEM, st>>>(src, dst, d, off, (int)zchunk,
                                                                                   ops, first_bad, guard);
    return (int)cudaGetLastError();
}

int sep_fused_dmma3_ws_launch(const double* src, double* dst, const Dims& d, const SepOps<3>& ops, int off,
                              cudaStream_t st, unsigned long long* first_bad, const unsigned long long* guard,
                              int variant) {
    using ws3::Cfg;
    switch (variant) {
        // TY, N1, N2, N3, SU, NWB, NVB, B3
        case 1: return launch_ws3<Cfg<7, 4, 4, 7, 3, 1, 2>>(src, dst, d, ops, off, st, first_bad, guard, 2);
        case 2: return launch_ws3<Cfg<7, 4, 4, 7, 2, 2, 2>>(src, dst, d, ops, off, st, first_bad, guard, 2);
        case 3: return launch_ws3<Cfg<7, 4, 4, 7, 3, 1, 1>>(src, dst, d, ops, off, st, first_bad, guard, 2);
        case 4: return launch_ws3<Cfg<7, 4, 4, 7, 3, 1, 2, 8>>(src, dst, d, ops, off, st, first_bad, guard, 2);
        case 5: return launch_ws3<Cfg<5, 4, 4, 5, 4, 1, 2>>(src, dst, d, ops, off, st, first_bad, guard, 2);
        case 6: return launch_ws3<Cfg<7, 8, 8, 7, 3, 1, 2, 2>>(src, dst, d, ops, off, st, first_bad, guard, 2);
        case 7: return launch_ws3<Cfg<7, 4, 4, 7, 3, 1, 2>>(src, dst, d, ops, off, st, first_bad, guard, 1);
        case 8: return launch_ws3<Cfg<3, 4, 4, 3, 4, 2, 2>>(src, dst, d, ops, off, st, first_bad, guard, 2);
        default: break;
    }
    return launch_ws3<Cfg<7, 4, 4, 7, 3, 1, 2>>(src, dst, d, ops, off, st, first_bad, guard, 2);
}

}  // namespace h3
#endif  // H3_MEASURE
