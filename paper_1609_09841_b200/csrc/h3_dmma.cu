// FP64 tensor-core (DMMA m8n8k4) fused half step for order N = 3 (n = 4).
//
// Same algorithm as sep_fused_kernel (h3_separable.cu): the exact separable local
// evolution out(c) = sum_a (A3^a3 (x) A2^a2 (x) A1^a1) u(c + off + a), applied as
// three node-factorised 1-D passes.  Each pass is a batch of tiny GEMMs
//     D[line][col] = sum_k data[line][k] * B[k][col]        (8 lines x 4 k x 8 cols)
// issued as mma.sync.m8n8k4.f64: one instruction does 256 FMAs, so the FP64 work
// costs 1/8 of the issue slots of DFMA and the operator never leaves registers
// (each lane holds one B element per operator).  B200's FP64 tensor rate equals its
// FP64 FMA rate (measured 37 TFLOP/s for both, tools/micro), so this is about issue
// efficiency, not peak flops.
//
// n = 4 outputs per line fill only half of the 8 columns, so the columns carry both
// roles of a node: its contribution to the cell on its right (A^0) and on its left
// (A^1).  Walking along an axis, consecutive nodes alternate the column order, so the
// two contributions to one cell land in the SAME lanes and are summed by the MMA's
// own accumulator -- no shuffles:
//     node parity 0: cols 0-3 = A^0 (cell p, pending)   cols 4-7 = A^1 (cell p-1, completes)
//     node parity 1: cols 0-3 = A^1 (cell p-1, completes) cols 4-7 = A^0 (cell p, pending)
// After each MMA the completed half of the lanes is stored and zeroed.
//
// CTA: 8 x 7 cells in (x1, x2), 16 warps, marching along x3 ("register rolling" in
// x3).  Per node plane:
//   x1: warp (row ly, line-half h) walks the 9 nodes of its row        (9 MMAs)
//   x2: warp (column ix, line-half h) walks the 8 rows of its column    (8 MMAs)
//   x3: warp owns 7 (cell, line-half) chains across planes             (7 MMAs)
// Input planes stream in with cp.async (3 stages); the pass results are exchanged
// through bank-conflict-free shared-memory layouts.
#include <cstdlib>

#include "h3_launch.h"
#include "h3_tma.cuh"

namespace h3 {

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}

template <int ABL>
__device__ __forceinline__ void dmma_abl(double& d0, double& d1, double a, double b) {
    if constexpr (ABL & 8) {  // energy ablation: the same dependencies through integer XORs only
        d0 = __longlong_as_double(__double_as_longlong(d0) ^ __double_as_longlong(a));
        d1 = __longlong_as_double(__double_as_longlong(d1) ^ __double_as_longlong(b));
    } else if constexpr (ABL & 4) {
        d0 += a;
        d1 -= b;
    } else {
        dmma884(d0, d1, a, b);
    }
}

// TMA bulk copies + mbarriers: h3_tma.cuh
using tma::bulk_g2s;
using tma::fence_proxy_async_smem;
using tma::mbar_arrive_expect_tx;
using tma::mbar_fence_init;
using tma::mbar_init;
using tma::mbar_wait;

// Tile / pipeline configuration of the DMMA kernel.
// TMA: input planes arrive as one bulk copy per tile row (9 contiguous node blocks, split at
// the periodic wrap) issued by lane 0 of warps 0..NY-1 and tracked by an mbarrier per stage, instead
// of 16-B cp.async by every thread (which cost ~50 address instructions per warp per plane).
// ABL (measurement-only ablations, results are garbage): bit 0 skips the global stores,
// bit 1 the input copies, bit 2 replaces every DMMA by a register update (two DADDs), bit 3 by
// two 64-bit integer XORs (same dependencies, no floating-point work: the energy ablation).
template <int TY_, int WARPS_, int STAGES_, bool VALIAS_, int MINB_ = 1, int ABL_ = 0, bool TMA_ = false,
          bool LEAN_ = false, int PIPE_ = 0, bool CF_ = false, bool FI_ = false>
struct Dm3Cfg {
    // FI: the per-plane TMA issue and mbarrier wait use shared addresses, source offsets and the
    // periodic-wrap split of the tile row precomputed once per CTA (the loader lanes' issue sits on
    // the path between the two CTA barriers of a plane)
    static constexpr bool FI = FI_;
    // CF: W cell stride 84 and an odd V row stride, so the paired stores of x1 / x2 (the two lane
    // halves write neighbouring cells / cell rows) hit distinct banks (80 and 8 x 68 are 0 mod 16)
    static constexpr bool CF = CF_;
    // PIPE 1: x3 of plane p-1 shares a barrier interval with x1 of plane p (2 barriers/plane).
    // (A 1-barrier variant -- x3(p-2), x2(p-1), x1(p) with W and V doubled -- measured 17 % slower.)
    static constexpr int PIPE = PIPE_;
    static constexpr int ABL = ABL_;
    static constexpr bool TMA = TMA_;
    // LEAN: x3 stores each chain's finished lanes with predicated half-warp stores at 32-bit
    // offsets from a per-plane base, and screens for non-finite values with one integer min
    // per value (the exact node is located on a rare path).
    static constexpr bool LEAN = LEAN_;
    static constexpr int MINB = MINB_;  // CTAs per SM the register budget is sized for
    static constexpr int n = 4, n3 = 64;
    static constexpr int TX = 8, TY = TY_, NX = TX + 1, NY = TY + 1, NCOL = NX * NY;
    static constexpr int WARPS = WARPS_, THREADS = 32 * WARPS, STAGES = STAGES_;
    static constexpr bool VALIAS = VALIAS_;  // x2 output reuses the consumed input stage
    static constexpr int UNS = 64;            // U node stride (dense [j3][j2][j1])
    static constexpr int WRS = 20, WCS = CF ? 84 : 80;  // W  [j3][m1][j2]: j3-row stride, cell stride
    static constexpr int VRS = 17, VCS = 68;  // V  [m2][m1][j3]: m2-row stride, cell stride
    static constexpr int VROW = TX * VCS + (CF ? 1 : 0);  // V cell-row stride
    static constexpr int T1 = 2 * NY, K1 = (T1 + WARPS - 1) / WARPS;  // x1 (row, half) tasks
    static constexpr int T2 = 2 * TX, K2 = (T2 + WARPS - 1) / WARPS;  // x2 (column, half) tasks
    static constexpr int T3 = 2 * TX * TY, K3 = T3 / WARPS;           // x3 (cell, half) chains
    static constexpr int CPW = (NCOL + WARPS - 1) / WARPS;            // node copies per warp
    static constexpr size_t U_D = (size_t)NCOL * UNS;
    static constexpr size_t W_D = (size_t)NY * TX * WCS;
    static constexpr size_t V_D = (size_t)TY * VROW;
    static constexpr size_t SMEM_DATA =
        (STAGES * U_D + W_D + (VALIAS ? 0 : V_D)) * sizeof(double);
    static constexpr size_t SMEM = SMEM_DATA + (TMA ? STAGES * sizeof(uint64_t) : 0);
    static_assert(!TMA || NY <= WARPS, "one loader warp per tile row");
    static_assert(T3 % WARPS == 0, "x3 chains must divide evenly among warps");
    static_assert(!VALIAS || V_D <= U_D, "aliased V must fit in one input stage");
    static_assert(STAGES >= 2, "need at least double buffering");
};

// ~hi(x) & 0x7ff00000 in one LOP3: zero iff x is Inf/NaN (exponent all ones)
__device__ __forceinline__ unsigned exp_gap(double x) {
    unsigned r;
    asm("lop3.b32 %0, %1, 0x7ff00000, 0, 0x0c;" : "=r"(r) : "r"((unsigned)__double2hiint(x)));
    return r;
}

template <class C>
__global__ void __launch_bounds__(C::THREADS, C::MINB)
sep_fused_dmma3_kernel(const double* __restrict__ src, double* __restrict__ dst, Dims d, int off,
                       int zchunk, int band, int cy, const __grid_constant__ SepOps<3> p,
                       unsigned long long* first_bad, const unsigned long long* guard) {
    constexpr int n = C::n, n3 = C::n3, TX = C::TX, TY = C::TY, NX = C::NX, NY = C::NY;
    constexpr int NCOL = C::NCOL, WARPS = C::WARPS, STAGES = C::STAGES, UNS = C::UNS;
    constexpr int WRS = C::WRS, WCS = C::WCS, VRS = C::VRS, VCS = C::VCS, VROW = C::VROW;
    constexpr int K1 = C::K1, K2 = C::K2, K3 = C::K3;
    if (guarded_out(guard, first_bad)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* U = reinterpret_cast<double*>(smem_raw);
    double* W = U + STAGES * C::U_D;
    double* Vfix = W + C::W_D;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q = lane & 3, g = lane >> 2, par = q >> 1;  // fragment coordinates
    const int M1 = (int)d.M1, M2 = (int)d.M2;
    int tbx, tby;
    band_tile(band, cy, tbx, tby);
    const int cx0 = tbx * TX, cy0 = tby * TY;
    const int64_t zc0 = d.z_begin + (int64_t)blockIdx.z * zchunk;
    const int64_t zc1 = min(zc0 + (int64_t)zchunk, d.z_end);
    const int P = (int)(zc1 - zc0) + 1;
    const int64_t plane_elems = (int64_t)M1 * M2 * n3;

    // operator fragments: lane holds B[k = q][col = g] for both column orders
    double bop[3][2];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        const int m = g & 3, hi = g >> 2;
        bop[ax][0] = hi ? p.A[ax][m][n + q] : p.A[ax][m][q];
        bop[ax][1] = hi ? p.A[ax][m][q] : p.A[ax][m][n + q];
    }

    // global offsets of the nodes this warp copies (node = warp + WARPS * j); the periodic
    // wrap is resolved once; each lane copies 16 B of the 512-B node block
    int nodeoff[C::TMA ? 1 : C::CPW];
    if constexpr (!C::TMA) {
#pragma unroll
        for (int j = 0; j < C::CPW; ++j) {
            const int c = warp + WARPS * j;
            const int ly = c / NX, lx = c - (c / NX) * NX;
            int gx = cx0 + off + lx, gy = cy0 + off + ly;
            gx %= M1; if (gx < 0) gx += M1;
            gy %= M2; if (gy < 0) gy += M2;
            nodeoff[j] = (gy * M1 + gx) * n3 + 2 * lane;
        }
    }
    // TMA loader: warp 0, lane ly < NY copies tile row ly (rowoff: its x2 row, gx0: first node)
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + C::SMEM_DATA);
    int rowoff = 0, gx0 = 0;
    if constexpr (C::TMA) {
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
    }
    // node plane of the next copy, wrapped incrementally
    int64_t gz_next = d.periodic_z ? wrap(zc0 + off, d.M3) : zc0 + off;
    int issued = 0;
    // FI: precomputed loader state (lane 0 of warp < NY): tile row split at the periodic wrap into
    // at most two bulk copies, their shared destinations in stage 0, the barrier address
    const uint32_t bar_u32 = smem_u32(bars);
    uint32_t sdst0 = 0, bytes1 = 0, bytes2 = 0;
    int64_t soff1 = 0, soff2 = 0;
    if constexpr (C::FI) {
        if (lane == 0 && warp < NY) {
            // a row narrower than the tile (M1 < NX) wraps more than once: the second piece is
            // clamped to the row (columns 0 .. gx0, all the in-grid cells need); the node slots
            // past it belong to out-of-grid cells only, whose outputs are never stored
            const int len1 = min(NX, M1 - gx0), len2 = min(NX - len1, M1);
            sdst0 = smem_u32(U + warp * NX * UNS);
            soff1 = ((int64_t)rowoff + gx0) * n3;
            soff2 = (int64_t)rowoff * n3;
            bytes1 = (unsigned)(len1 * UNS * sizeof(double));
            bytes2 = (unsigned)(len2 * UNS * sizeof(double));
        }
    }
    auto issue = [&]() {
        if constexpr (C::TMA && C::FI) {
            if (issued < P) {
                if (lane == 0 && warp < NY) {
                    const int s = issued % STAGES;
                    const uint32_t bar = bar_u32 + 8u * (unsigned)s;
                    const uint32_t sd = sdst0 + (uint32_t)(s * C::U_D * sizeof(double));
                    fence_proxy_async_smem();
                    // every loader row copies the same bytes1 + bytes2 (same gx0)
                    if (warp == 0) tma::mbar_arrive_expect_tx_u32(bar, (unsigned)NY * (bytes1 + bytes2));
                    const double* base = plane_base(src, gz_next, plane_elems, d);
                    tma::bulk_g2s_u32(sd, base + soff1, bytes1, bar);
                    if (bytes2) tma::bulk_g2s_u32(sd + bytes1, base + soff2, bytes2, bar);
                }
                ++gz_next;
                if (d.periodic_z && gz_next == d.M3) gz_next = 0;
                ++issued;
            }
        } else if constexpr (C::TMA) {
            if (issued < P) {
                // lane 0 of warp ly < NY copies tile row ly; warp 0 also posts the byte count
                // (the mbarrier tx-count may run ahead of it: the phase cannot complete before
                // the single arrival)
                if (lane == 0 && warp < NY) {
                    const int s = issued % STAGES;
                    fence_proxy_async_smem();
                    if (warp == 0) mbar_arrive_expect_tx(&bars[s], (unsigned)(NCOL * UNS * sizeof(double)));
                    if (!(C::ABL & 2)) {
                        const double* base = plane_base(src, gz_next, plane_elems, d) + (int64_t)rowoff * n3;
                        double* Ub = U + s * C::U_D + warp * NX * UNS;
                        int got = 0, gx = gx0;
                        while (got < NX) {
                            const int len = min(NX - got, M1 - gx);
                            bulk_g2s(Ub + got * UNS, base + (int64_t)gx * n3, (unsigned)(len * UNS * sizeof(double)),
                                     &bars[s]);
                            got += len;
                            gx = 0;
                        }
                    }
                }
                ++gz_next;
                if (d.periodic_z && gz_next == d.M3) gz_next = 0;
                ++issued;
            }
        } else {
            if (issued < P) {
                const double* base = plane_base(src, gz_next, plane_elems, d);
                double* Ub = U + (issued % STAGES) * C::U_D + 2 * lane;
#pragma unroll
                for (int j = 0; j < C::CPW; ++j)
                    if (NCOL % WARPS == 0 || warp + WARPS * j < NCOL)
                        if (!(C::ABL & 2)) cp_async16(Ub + (warp + WARPS * j) * UNS, base + nodeoff[j]);
                ++gz_next;
                if (d.periodic_z && gz_next == d.M3) gz_next = 0;
                ++issued;
            }
            cp_async_commit();
        }
    };
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) issue();

    // x3 chains: t = warp + WARPS * k -> (cell t >> 1, half t & 1).  obase: the lane's output
    // offset in cell plane zc0 (m3 = 2 (q & 1) + i, line L), or -1 outside the grid.
    int64_t obase[K3];
#pragma unroll
    for (int k = 0; k < K3; ++k) {
        const int t = warp + WARPS * k;
        const int cell = t >> 1, h = t & 1;
        const int cx = cx0 + (cell % TX), cy = cy0 + cell / TX;
        obase[k] = (cx < M1 && cy < M2)
                       ? ((zc0 * M2 + cy) * (int64_t)M1 + cx) * n3 + (2 * (q & 1)) * 16 + 8 * h + g
                       : -1;
    }
    // LEAN: the lane's output offset within a node plane (int32; M1 M2 64 < 2^31 checked at launch)
    int ooff[C::LEAN ? K3 : 1];
    if constexpr (C::LEAN) {
#pragma unroll
        for (int k = 0; k < K3; ++k) {
            const int t = warp + WARPS * k;
            const int cell = t >> 1, h = t & 1;
            const int cx = cx0 + (cell % TX), cy = cy0 + cell / TX;
            ooff[k] = (cx < M1 && cy < M2) ? (cy * M1 + cx) * n3 + (2 * (q & 1)) * 16 + 8 * h + g : -1;
        }
    }
    double acc[K3][2];
#pragma unroll
    for (int k = 0; k < K3; ++k) acc[k][0] = acc[k][1] = 0.0;

    // three passes per node plane; PIPE overlaps x3 of plane p-1 with x1 of plane p in one
    // barrier interval (2 barriers per plane instead of 3; needs the non-aliased V buffer)
    auto x1_pass = [&](const double* Ub, double* W) {
        // ---- x1: (row ly, half h) chains walk the nodes of their row ------------------------
        // Completed cells alternate between the lane halves; an even cell's values are
        // held one node longer so both halves store together (full-warp STS).
        {
            const double* ua[K1];
            double* wrow[K1];
            bool live[K1];
#pragma unroll
            for (int j = 0; j < K1; ++j) {
                const int t = warp + WARPS * j;
                live[j] = C::T1 % WARPS == 0 || t < C::T1;
                const int ly = live[j] ? t >> 1 : 0, h = t & 1;
                const int L = 8 * h + g;  // line (j3, j2) = (L >> 2, L & 3)
                ua[j] = Ub + ly * NX * UNS + L * 4 + q;
                wrow[j] = W + ly * TX * WCS + (2 * h + (g >> 2)) * WRS + (g & 3) + (2 * (q & 1)) * 4;
            }
            double a[K1][NX];
#pragma unroll
            for (int j = 0; j < K1; ++j)
#pragma unroll
                for (int lx = 0; lx < NX; ++lx) a[j][lx] = live[j] ? ua[j][lx * UNS] : 0.0;
            double r[K1][2], sv[K1][2];
#pragma unroll
            for (int j = 0; j < K1; ++j) r[j][0] = r[j][1] = sv[j][0] = sv[j][1] = 0.0;
#pragma unroll
            for (int lx = 0; lx < NX; ++lx) {
                const bool done = par == ((lx + 1) & 1);  // cell lx-1 completed in these lanes
#pragma unroll
                for (int j = 0; j < K1; ++j) {
                    dmma_abl<C::ABL>(r[j][0], r[j][1], a[j][lx], bop[0][lx & 1]);
                    if (lx & 1) {
                        sv[j][0] = r[j][0];
                        sv[j][1] = r[j][1];
                    } else if (lx > 0 && live[j]) {
                        double* w = wrow[j] + (lx - 1 - (par ^ 1)) * WCS;
                        w[0] = par ? r[j][0] : sv[j][0];
                        w[4] = par ? r[j][1] : sv[j][1];
                    }
                    r[j][0] = done ? 0.0 : r[j][0];
                    r[j][1] = done ? 0.0 : r[j][1];
                }
            }
        }
    };
    auto x2_pass = [&](const double* W, double* V) {
        // ---- x2: (column ix, half h) chains walk the rows of their column -----------------
        {
            const double* wa[K2];
            double* vcol[K2];
            bool live[K2];
#pragma unroll
            for (int j = 0; j < K2; ++j) {
                const int t = warp + WARPS * j;
                live[j] = C::T2 % WARPS == 0 || t < C::T2;
                const int ix = live[j] ? t >> 1 : 0, h = t & 1;
                const int L = 8 * h + g;  // line (j3, m1) = (L >> 2, L & 3)
                wa[j] = W + ix * WCS + (L >> 2) * WRS + (L & 3) * 4 + q;
                vcol[j] = V + ix * VCS + (L & 3) * 4 + (L >> 2) + (2 * (q & 1)) * VRS;
            }
            double a[K2][NY];
#pragma unroll
            for (int j = 0; j < K2; ++j)
#pragma unroll
                for (int ly = 0; ly < NY; ++ly) a[j][ly] = live[j] ? wa[j][ly * TX * WCS] : 0.0;
            double r[K2][2], sv[K2][2];
#pragma unroll
            for (int j = 0; j < K2; ++j) r[j][0] = r[j][1] = sv[j][0] = sv[j][1] = 0.0;
#pragma unroll
            for (int ly = 0; ly < NY; ++ly) {
                const bool done = par == ((ly + 1) & 1);
#pragma unroll
                for (int j = 0; j < K2; ++j) {
                    dmma_abl<C::ABL>(r[j][0], r[j][1], a[j][ly], bop[1][ly & 1]);
                    if (ly & 1) {
                        if (ly == NY - 1) {  // lone last cell row: half-warp store
                            if (done && live[j]) {
                                double* v = vcol[j] + (ly - 1) * VROW;
                                v[0] = r[j][0];
                                v[VRS] = r[j][1];
                            }
                        } else {
                            sv[j][0] = r[j][0];
                            sv[j][1] = r[j][1];
                        }
                    } else if (ly > 0 && live[j]) {
                        double* v = vcol[j] + (ly - 1 - (par ^ 1)) * VROW;
                        v[0] = par ? r[j][0] : sv[j][0];
                        v[VRS] = par ? r[j][1] : sv[j][1];
                    }
                    r[j][0] = done ? 0.0 : r[j][0];
                    r[j][1] = done ? 0.0 : r[j][1];
                }
            }
        }
    };
    auto x3_pass = [&](const double* V, const int pp) {
        // ---- x3: each warp advances its chains by one plane ---------------------------------
        // Chain k runs with column phase (k & 1), so chains 2j and 2j+1 complete in opposite
        // lane halves and share one full-warp store.
        {
            const int64_t plane_off = (int64_t)(pp - 1) * plane_elems;
            double v0[K3], v1[K3];
#pragma unroll
            for (int k = 0; k < K3; ++k) {
                const int t = warp + WARPS * k;
                const int cell = t >> 1, h = t & 1;
                const int L = 8 * h + g;  // line (m2, m1) = (L >> 2, L & 3)
                const double a = V[(cell / TX) * VROW + (cell % TX) * VCS + (L >> 2) * VRS + (L & 3) * 4 + q];
                const int ph = (pp + k) & 1;
                dmma_abl<C::ABL>(acc[k][0], acc[k][1], a, ph ? bop[2][1] : bop[2][0]);
                const bool done = par == ((pp + k + 1) & 1);
                v0[k] = acc[k][0];
                v1[k] = acc[k][1];
                acc[k][0] = done ? 0.0 : acc[k][0];
                acc[k][1] = done ? 0.0 : acc[k][1];
            }
            if constexpr (C::LEAN) {
                if (pp > 0) {
                    double* oplane = dst + (zc0 + pp - 1) * plane_elems;
                    // opaque to the optimiser: one 64-bit plane pointer, then one IMAD.WIDE per
                    // store pair (instead of re-deriving dst + plane + offset per store)
                    asm volatile("" : "+l"(oplane));
                    unsigned screen = 0x7ff00000u;
#pragma unroll
                    for (int k = 0; k < K3; ++k) {
                        const bool done = par == ((pp + k + 1) & 1);
                        if (done && ooff[k] >= 0) {
                            if (!(C::ABL & 1)) {
                                __stcs(oplane + ooff[k], v0[k]);
                                __stcs(oplane + ooff[k] + 16, v1[k]);
                            }
                        }
                        screen = min(screen, min(exp_gap(v0[k]), exp_gap(v1[k])));
                    }
                    if (screen == 0u) {  // rare: some lane holds Inf/NaN (finished or partial)
#pragma unroll
                        for (int k = 0; k < K3; ++k) {
                            const bool done = par == ((pp + k + 1) & 1);
                            if (done && ooff[k] >= 0 && (!isfinite(v0[k]) || !isfinite(v1[k])))
                                flag_bad(first_bad, (zc0 + pp - 1) * M2 * (int64_t)M1 + ooff[k] / n3);
                        }
                    }
                }
            } else if (pp > 0) {
#pragma unroll
                for (int k = 0; k < K3; k += 2) {
                    // lanes with par == ((pp + k + 1) & 1) hold chain k, the others chain k+1
                    const bool mine = par == ((pp + k + 1) & 1);
                    const bool pair = k + 1 < K3;
                    if (!pair && !mine) continue;  // odd chain count: lone last chain
                    const int k2 = pair ? k + 1 : k;
                    const double o0 = mine ? v0[k] : v0[k2];
                    const double o1 = mine ? v1[k] : v1[k2];
                    const int64_t base = mine ? obase[k] : obase[k2];
                    const bool bad = !isfinite(o0) || !isfinite(o1);
                    if (base >= 0) {
                        double* o = dst + base + plane_off;
                        if (!(C::ABL & 1)) {
                            __stcs(o, o0);
                            __stcs(o + 16, o1);
                        }
                        if (bad) flag_bad(first_bad, (base + plane_off) / n3);
                    }
                }
            }
        }
    };
    auto top = [&](int pl) {
        if constexpr (C::TMA) {
            __syncthreads();
            issue();  // the stage it fills was last read before the barrier above
            if constexpr (C::FI)
                tma::mbar_wait_u32(bar_u32 + 8u * (unsigned)(pl % STAGES), (unsigned)((pl / STAGES) & 1));
            else if (!(C::ABL & 2))
                mbar_wait(&bars[pl % STAGES], (unsigned)((pl / STAGES) & 1));
        } else {
            cp_async_wait<STAGES - 2>();
            __syncthreads();
            issue();  // the stage it fills was last read before the barrier above
        }
    };
    if constexpr (C::PIPE == 1) {
        static_assert(!C::VALIAS, "PIPE keeps V(p-1) while stage p is refilled");
        for (int pl = 0; pl <= P; ++pl) {
            if (pl < P) top(pl);
            else __syncthreads();
            if (pl >= 1) x3_pass(Vfix, pl - 1);
            if (pl < P) x1_pass(U + (pl % STAGES) * C::U_D, W);
            __syncthreads();
            if (pl < P) x2_pass(W, Vfix);
        }
    } else {
        for (int pl = 0; pl < P; ++pl) {
            top(pl);
            double* V = C::VALIAS ? U + (pl % STAGES) * C::U_D : Vfix;
            x1_pass(U + (pl % STAGES) * C::U_D, W);
            __syncthreads();
            x2_pass(W, V);
            __syncthreads();
            x3_pass(V, pl);
        }
    }
    cp_async_wait<0>();
}

// column-band widths of the tile rasterisation (band_tile, h3_launch.h)
#ifndef H3_DMMA3_BAND
#define H3_DMMA3_BAND 8
#endif

template <class C>
static int launch_dm3(const double* src, double* dst, const Dims& d, const SepOps<3>& ops, int off,
                      cudaStream_t st, unsigned long long* first_bad,
                      const unsigned long long* guard) {
    const int64_t nz = d.z_end - d.z_begin;
    auto kern = sep_fused_dmma3_kernel<C>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return (int)e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::THREADS, C::SMEM);
    if (e != cudaSuccess) return (int)e;
    const int64_t gx = (d.M1 + C::TX - 1) / C::TX, gy = (d.M2 + C::TY - 1) / C::TY;
    const int64_t zchunk = choose_zchunk(gx * gy, nz, (int64_t)num_sms() * (per_sm > 0 ? per_sm : 1));
    const int64_t gz = (nz + zchunk - 1) / zchunk;
    // Thread-block clusters of 2 tiles along x2: y-adjacent tiles share a node row;
    // co-scheduling them keeps that row in L2 for the second reader (DRAM over-read 14% ->
    // measured +4.5% throughput at 512^3).
#ifdef H3_MEASURE
    static const int cy = [] {  // tools library only: H3_DMMA_CLUSTER_Y (1 = off)
        const char* e = getenv("H3_DMMA_CLUSTER_Y");
        return e ? atoi(e) : 2;
    }();
    static const int cx = [] {  // tools library only: H3_DMMA_CLUSTER_X
        const char* e = getenv("H3_DMMA_CLUSTER_X");
        return e ? atoi(e) : 1;
    }();
    static const int band = [] {  // tools library only: H3_DMMA_BAND (0 = plain row order)
        const char* e = getenv("H3_DMMA_BAND");
        return e ? atoi(e) : H3_DMMA3_BAND;
    }();
#else
    constexpr int cy = 2, cx = 1, band = H3_DMMA3_BAND;
#endif
    const bool clustered = (cy > 1 || cx > 1) && gy % cy == 0 && gx % cx == 0;
    const int cy_eff = clustered ? cy : 1;
    const int band_eff = cx > 1 ? 0 : band;  // the band map keeps y clusters only
    if (clustered) {
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3((unsigned)gx, (unsigned)gy, (unsigned)gz);
        lc.blockDim = dim3(C::THREADS);
        lc.dynamicSmemBytes = C::SMEM;
        lc.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cx;
        at[0].val.clusterDim.y = cy;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        e = cudaLaunchKernelEx(&lc, kern, src, dst, d, off, (int)zchunk, band_eff, cy_eff, ops, first_bad, guard);
        return (int)e;
    }
    kern<<<dim3((unsigned)gx, (unsigned)gy, (unsigned)gz), C::THREADS, C::SMEM, st>>>(
        src, dst, d, off, (int)zchunk, band_eff, cy_eff, ops, first_bad, guard);
    return (int)cudaGetLastError();
}

int sep_fused_dmma3_launch(const double* src, double* dst, const Dims& d, const double* A, int off,
                           cudaStream_t st, unsigned long long* first_bad,
                           const unsigned long long* guard) {
    const int64_t nz = d.z_end - d.z_begin;
    if (nz <= 0) return 0;
    if (d.M1 * d.M2 * 64 >= (int64_t(1) << 31)) return (int)cudaErrorInvalidValue;
    SepOps<3> ops;
    for (int k = 0; k < 3; ++k)
        for (int m = 0; m < 4; ++m)
            for (int c = 0; c < 8; ++c) {
                ops.A[k][m][c] = A[(k * 4 + m) * 8 + c];
                ops.Sh[k][m][c] = 0.0;
            }
#ifdef H3_MEASURE
    // tools library only: H3_DMMA_CFG=k selects the measurement variants of tools/ab.sh
    // (ablations 11/14/15 skip stores / replace the DMMAs and produce garbage on purpose)
    static const int cfg = [] {
        const char* e = getenv("H3_DMMA_CFG");
        return e ? atoi(e) : 0;
    }();
    if (cfg >= 200) return sep_fused_dmma3x_launch(src, dst, d, ops, off, st, first_bad, guard, cfg - 200);
    if (cfg >= 100) return sep_fused_dmma3_ws_launch(src, dst, d, ops, off, st, first_bad, guard, cfg - 100);
    switch (cfg) {
        case 6: return launch_dm3<Dm3Cfg<7, 16, 3, true>>(src, dst, d, ops, off, st, first_bad, guard);  // cp.async loads
        case 11: return launch_dm3<Dm3Cfg<7, 16, 3, true, 1, 1, true>>(src, dst, d, ops, off, st, first_bad, guard);
        case 14: return launch_dm3<Dm3Cfg<7, 16, 3, true, 1, 4, true>>(src, dst, d, ops, off, st, first_bad, guard);
        case 15: return launch_dm3<Dm3Cfg<7, 16, 3, true, 1, 5, true>>(src, dst, d, ops, off, st, first_bad, guard);
        case 16: return launch_dm3<Dm3Cfg<7, 16, 3, true, 1, 0, true>>(src, dst, d, ops, off, st, first_bad, guard);
        case 31: return launch_dm3<Dm3Cfg<7, 16, 3, false, 1, 0, true, true, 1, false>>(src, dst, d, ops, off, st, first_bad, guard);  // bank-conflicted W/V
        case 33: return launch_dm3<Dm3Cfg<7, 8, 3, false, 1, 0, true, true, 1, true, true>>(src, dst, d, ops, off, st, first_bad, guard);  // 8 warps, 2 tasks each
        case 34: return launch_dm3<Dm3Cfg<7, 16, 3, false, 1, 8, true, true, 1, true, true>>(src, dst, d, ops, off, st, first_bad, guard);  // product with XOR for DMMA (energy ablation)
        case 35: return launch_dm3<Dm3Cfg<7, 16, 3, false, 1, 1, true, true, 1, true, true>>(src, dst, d, ops, off, st, first_bad, guard);  // product without the global stores
        case 36: return launch_dm3<Dm3Cfg<7, 16, 3, false, 1, 9, true, true, 1, true, true>>(src, dst, d, ops, off, st, first_bad, guard);  // neither
        // taller tiles (fewer halo DMMAs: 6.72 / 6.64 vs 6.86 per cell) with 2 TMA stages to fit 227 KB
        case 37: return launch_dm3<Dm3Cfg<9, 16, 2, false, 1, 0, true, true, 1, true, true>>(src, dst, d, ops, off, st, first_bad, guard);
        case 38: return launch_dm3<Dm3Cfg<11, 16, 2, false, 1, 0, true, true, 1, true, true>>(src, dst, d, ops, off, st, first_bad, guard);
        case 39: return launch_dm3<Dm3Cfg<7, 16, 2, false, 1, 0, true, true, 1, true, true>>(src, dst, d, ops, off, st, first_bad, guard);
        case 32: return launch_dm3<Dm3Cfg<7, 16, 3, false, 1, 0, true, true, 1, true, true>>(src, dst, d, ops, off, st, first_bad, guard);  // precomputed issue
        default: break;
    }
#endif
    // TMA row loads with a precomputed issue (r02: -0.6 %), x3(p-1) pipelined with x1(p) (2 barriers
    // per plane), lean x3 stores, conflict-free W / V strides
    return launch_dm3<Dm3Cfg<7, 16, 3, false, 1, 0, true, true, 1, true, true>>(src, dst, d, ops, off, st, first_bad, guard);
}


// ---------------------------------------------------------------------------------------
// Reconstruction pass of the two-kernel step for N = 3 on the FP64 tensor cores.
//
// coeff(c)[i3][i2][i1] = sum_a (H^a3 (x) H^a2 (x) H^a1) u(c + off + a), H^a = H[:, 4a:4a+4]
// (gridkernels.py:58-83 computes the same tensor by three dense sweeps of the gathered
// 8^3 block).  Node-factorised: x1 and x2 in the plane, x3 rolled across planes.  Each
// pass contracts 4 inputs of a node into 8 outputs, so a node's two roles (left vertex,
// H^0; right vertex, H^1) are two full 8-column MMAs and the rolling accumulator needs
// no lane tricks: W(cell c) = H^1 u(c+1) accumulated onto H^0 u(c).
// CTA: 8 x 4 cells, 16 warps; per node plane x1 (10 row chains), x2 (32 column chains),
// x3 (16 chains per warp, 8 line groups per cell, carried across planes).
namespace rc3 {
constexpr int n3 = 64, S3 = 512;
constexpr int TX = 8, TY = 4, NX = TX + 1, NY = TY + 1, NCOL = NX * NY;
constexpr int WARPS = 16, THREADS = 32 * WARPS, STAGES = 3;
constexpr int UNS = 64;
constexpr int WJ = 36, WCS = 4 * WJ;  // W [j3][i1 (+gap at i1 = 4)][j2]
constexpr int VCS = 256;               // V [i2][i1][j3 rotated by (i2 >> 1)]
constexpr int T1 = 2 * NY;             // x1 chains (row, line group)
constexpr int T2 = 4 * TX;             // x2 chains (column, j3)
constexpr int K2 = (T2 + WARPS - 1) / WARPS;
constexpr int T3 = 8 * TX * TY;        // x3 chains (cell, i2)
constexpr int K3 = T3 / WARPS;
constexpr int CPW = (NCOL + WARPS - 1) / WARPS;
constexpr size_t U_D = (size_t)NCOL * UNS, W_D = (size_t)NY * TX * WCS, V_D = (size_t)TX * TY * VCS;
constexpr size_t SMEM = (STAGES * U_D + W_D + V_D) * sizeof(double);
static_assert(T3 % WARPS == 0, "x3 chains must divide evenly");
__device__ __forceinline__ int wpos(int i1, int j2) { return 4 * (i1 + (i1 >> 2)) + j2; }
__device__ __forceinline__ int vpos(int i2, int i1, int j3) { return (i2 * 8 + i1) * 4 + ((j3 + (i2 >> 1)) & 3); }
}  // namespace rc3

template <bool PIPE>
__global__ void __launch_bounds__(rc3::THREADS, 1)
recon_dmma3_kernel(const double* __restrict__ src, double* __restrict__ coeff, Dims d, int off,
                   int zchunk, const __grid_constant__ LitOps<double, 3> hp,
                   const unsigned long long* guard) {
    using namespace rc3;
    if (guarded_out(guard, nullptr)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* U = reinterpret_cast<double*>(smem_raw);
    double* W = U + STAGES * U_D;
    double* V = W + W_D;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q = lane & 3, g = lane >> 2;
    const int M1 = (int)d.M1, M2 = (int)d.M2;
    const int cx0 = blockIdx.x * TX, cy0 = blockIdx.y * TY;
    const int64_t zc0 = d.z_begin + (int64_t)blockIdx.z * zchunk;
    const int64_t zc1 = min(zc0 + (int64_t)zchunk, d.z_end);
    const int P = (int)(zc1 - zc0) + 1;
    const int64_t plane_elems = (int64_t)M1 * M2 * n3;
    const int64_t cplane = (int64_t)M1 * M2 * S3;  // one cell plane of the coefficient field

    // B fragments: lane holds B[k = q][col = g]; H^0: H[i][j], H^1: H[i][4 + j]
    const double b0 = hp.H[g * 8 + q], b1 = hp.H[g * 8 + 4 + q];

    int nodeoff[CPW];
#pragma unroll
    for (int j = 0; j < CPW; ++j) {
        const int c = min(warp + WARPS * j, NCOL - 1);
        const int ly = c / NX, lx = c - (c / NX) * NX;
        int gx = cx0 + off + lx, gy = cy0 + off + ly;
        gx %= M1; if (gx < 0) gx += M1;
        gy %= M2; if (gy < 0) gy += M2;
        nodeoff[j] = (gy * M1 + gx) * n3 + 2 * lane;
    }
    int64_t gz_next = d.periodic_z ? wrap(zc0 + off, d.M3) : zc0 + off;
    int issued = 0;
    auto issue = [&]() {
        if (issued < P) {
            const double* base = plane_base(src, gz_next, plane_elems, d);
            double* Ub = U + (issued % STAGES) * U_D + 2 * lane;
#pragma unroll
            for (int j = 0; j < CPW; ++j)
                if (warp + WARPS * j < NCOL) cp_async16(Ub + (warp + WARPS * j) * UNS, base + nodeoff[j]);
            ++gz_next;
            if (d.periodic_z && gz_next == d.M3) gz_next = 0;
            ++issued;
        }
        cp_async_commit();
    };
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) issue();

    // x3 chains: t = warp + WARPS * k -> cell t >> 3 = (warp >> 3) + 2k, i2 = t & 7 = warp & 7.
    // Output offset of the lane in cell plane zc0 relative to the tile origin; per chain the
    // cell adds (cell % TX) + (cell / TX) * M1 cells.
    static_assert(WARPS == 16 && TX == 8, "chain -> cell mapping assumes 16 warps, 8-wide tiles");
    const int64_t obase0 = ((zc0 - d.z_begin) * M2 * (int64_t)M1 + (int64_t)cy0 * M1 + cx0) * S3 +
                           (2 * q) * 64 + (warp & 7) * 8 + g;
    double acc[K3][2];
#pragma unroll
    for (int k = 0; k < K3; ++k) acc[k][0] = acc[k][1] = 0.0;

    // the three passes of one node plane; PIPE runs x3 of plane p-1 in the barrier interval of x1
    // of plane p (2 barriers per plane instead of 3, and the warps without an x1 task -- 10 tasks
    // for 16 warps -- start on x3 at once); single W and V buffers suffice: V(p-1) is read in the
    // interval before x2(p) rewrites it, W(p) is written after x2(p-1) read it
    auto x1_pass = [&](const double* Ub) {
        // ---- x1: (row, line group) chains along x1 -----------------------------------------
        if (warp < T1) {
            const int ly = warp >> 1, G = warp & 1;
            const int L = 8 * G + g;  // line (j3, j2)
            const double* ua = Ub + ly * NX * UNS + L * 4 + q;
            double* wrow = W + ly * TX * WCS + (L >> 2) * WJ + (L & 3);
            double a[NX];
#pragma unroll
            for (int lx = 0; lx < NX; ++lx) a[lx] = ua[lx * UNS];
            double r0 = 0.0, r1 = 0.0;
#pragma unroll
            for (int lx = 0; lx < NX; ++lx) {
                if (lx > 0) {
                    dmma884(r0, r1, a[lx], b1);  // completes cell lx-1
                    double* w = wrow + (lx - 1) * WCS;
                    w[wpos(2 * q, 0)] = r0;
                    w[wpos(2 * q + 1, 0)] = r1;
                }
                if (lx < NX - 1) {
                    r0 = r1 = 0.0;
                    dmma884(r0, r1, a[lx], b0);
                }
            }
        }
    };
    auto x2_pass = [&]() {
        // ---- x2: (column, j3) chains along x2 ------------------------------------------------
#pragma unroll
        for (int j = 0; j < K2; ++j) {
            const int t = warp + WARPS * j;
            if (T2 % WARPS == 0 || t < T2) {
                const int ix = t >> 2, j3 = t & 3;
                const double* wa = W + ix * WCS + j3 * WJ + wpos(g, q);  // line (j3, i1 = g), k = j2
                double a[NY];
#pragma unroll
                for (int ly = 0; ly < NY; ++ly) a[ly] = wa[ly * TX * WCS];
                double r0 = 0.0, r1 = 0.0;
#pragma unroll
                for (int ly = 0; ly < NY; ++ly) {
                    if (ly > 0) {
                        dmma884(r0, r1, a[ly], b1);  // completes cell row ly-1: [j3][i2][i1=g]
                        double* v = V + ((ly - 1) * TX + ix) * VCS;
                        v[vpos(2 * q, g, j3)] = r0;
                        v[vpos(2 * q + 1, g, j3)] = r1;
                    }
                    if (ly < NY - 1) {
                        r0 = r1 = 0.0;
                        dmma884(r0, r1, a[ly], b0);
                    }
                }
            }
        }
    };
    auto x3_pass = [&](const int pl) {
        // ---- x3: chains across planes; completed cell planes go straight to HBM ----------------
        {
            const int64_t plane_off = (int64_t)(pl - 1) * cplane;
            constexpr int B = 4;  // chains per batch: bounds the live temporaries
#pragma unroll
            for (int k0 = 0; k0 < K3; k0 += B) {
                double a[B], o0[B], o1[B];
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    const int t = warp + WARPS * (k0 + b);
                    a[b] = V[(t >> 3) * VCS + vpos(t & 7, g, q)];  // line (i2, i1 = g), k = j3
                }
                // completions are computed into copies so the accumulators restart at once
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    o0[b] = acc[k0 + b][0];
                    o1[b] = acc[k0 + b][1];
                    dmma884(o0[b], o1[b], a[b], b1);
                    acc[k0 + b][0] = acc[k0 + b][1] = 0.0;
                    dmma884(acc[k0 + b][0], acc[k0 + b][1], a[b], b0);
                }
                if (pl > 0) {
#pragma unroll
                    for (int b = 0; b < B; ++b) {
                        const int cell = (warp >> 3) + 2 * (k0 + b);
                        const int cx = cell % TX, cy = cell / TX;
                        if (cx0 + cx < M1 && cy0 + cy < M2) {
                            double* o = coeff + obase0 + plane_off + ((int64_t)cy * M1 + cx) * S3;
                            __stcs(o, o0[b]);
                            __stcs(o + 64, o1[b]);
                        }
                    }
                }
            }
        }
        };
    if constexpr (PIPE) {
        for (int pl = 0; pl <= P; ++pl) {
            if (pl < P) {
                cp_async_wait<STAGES - 2>();
                __syncthreads();
                issue();
            } else {
                __syncthreads();
            }
            if (pl >= 1) x3_pass(pl - 1);
            if (pl < P) x1_pass(U + (pl % STAGES) * U_D);
            __syncthreads();
            if (pl < P) x2_pass();
        }
    } else {
        for (int pl = 0; pl < P; ++pl) {
            cp_async_wait<STAGES - 2>();
            __syncthreads();
            issue();
            x1_pass(U + (pl % STAGES) * U_D);
            __syncthreads();
            x2_pass();
            __syncthreads();
            x3_pass(pl);
        }
    }
    cp_async_wait<0>();
}

#ifndef H3_RC3_PIPE_DEFAULT
// x3 of plane p-1 pipelined with x1 of plane p: 0.7 % faster m=3 two-kernel step (r02)
#define H3_RC3_PIPE_DEFAULT true
#endif

int recon_dmma3_launch(const double* src, double* coeff, const Dims& d, const double* h_mat, int off,
                       cudaStream_t st, const unsigned long long* guard) {
    using namespace rc3;
    const int64_t nz = d.z_end - d.z_begin;
    if (nz <= 0) return 0;
    if (d.M1 * d.M2 * n3 >= (int64_t(1) << 31)) return (int)cudaErrorInvalidValue;
    LitOps<double, 3> hp;
    for (int i = 0; i < 64; ++i) hp.H[i] = h_mat[i];
    for (int i = 0; i < 8; ++i) hp.f1[i] = hp.f2[i] = hp.f3[i] = 0.0;
    for (int i = 0; i < H3_MAX_STAGES; ++i) hp.cf[i] = 0.0;
    hp.q = 0;
#ifdef H3_MEASURE
    static const bool pipe = [] {  // tools library only: H3_RC3_PIPE=0/1
        const char* e = getenv("H3_RC3_PIPE");
        return e ? atoi(e) != 0 : H3_RC3_PIPE_DEFAULT;
    }();
    auto kern = pipe ? recon_dmma3_kernel<true> : recon_dmma3_kernel<false>;
#else
    auto kern = recon_dmma3_kernel<H3_RC3_PIPE_DEFAULT>;
#endif
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
    if (e != cudaSuccess) return (int)e;
    const int64_t gx = (d.M1 + TX - 1) / TX, gy = (d.M2 + TY - 1) / TY;
    const int64_t zchunk = choose_zchunk(gx * gy, nz, num_sms());  // one CTA per SM
    const int64_t gz = (nz + zchunk - 1) / zchunk;
    // (plain row order: the band rasterisation measured neutral to slightly slower here,
    // profiles/r02_tuning_ab.txt)
    kern<<<dim3((unsigned)gx, (unsigned)gy, (unsigned)gz), THREADS, SMEM, st>>>(
        src, coeff, d, off, (int)zchunk, hp, guard);
    return (int)cudaGetLastError();
}

}  // namespace h3
