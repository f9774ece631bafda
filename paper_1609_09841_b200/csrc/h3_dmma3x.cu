// FP64 tensor-core fused half step for N = 3 (n = 4) with the x1 and x2 passes chained in
// registers: one shared-memory round trip per node plane instead of two.
//
// Same exact separable local evolution as h3_dmma.cu, out(c) = sum_a (A3^a3 (x) A2^a2 (x) A1^a1)
// u(c + off + a), applied as three node-factorised rolling DMMA passes (mma.sync.m8n8k4.f64).
// What changes is the fragment orientation of the x1 pass.  An m8n8k4 fragment pins the
// contraction index k to the lane's quad position q (A: lane (g, q) = A[g][q]; B: lane (g, q) =
// B[q][g]) and puts the two outputs of a lane at columns 2q, 2q+1 of row g.  The lock-step kernel
// runs every pass "data as A" (D[line][out] = data[line][k] * Op[k][out]): the outputs land on q,
// so every pass must go through shared memory to bring the next contraction index back onto q.
// Here x1 runs "data as B": D[out][line] = Op[out][k] * data[k][line].  With the x1 lines of a
// fragment chosen as (j2, node-row slot) -- line = 2 j2 + slot -- the lane holding x1 output
// (m1, line 2q + i) holds j2 = q and row slot i: exactly x2's A fragment (line = m1 (+ cell of the
// pair), k = j2 = q), one fragment per node row.  x1's rolling alternation completes even cells in
// lanes g < 4 and odd cells in lanes g >= 4, so two neighbouring cells of a row form one x2 A
// fragment (8 lines = cell pair x m1) with one select per value, no shuffle.  Only x2 -> x3 (j3 must
// reach q) goes through shared memory (V).  Per node plane: shared wavefronts 288 (TMA) + 320 (x1
// loads) + 224 (V stores) + 224 (V loads) against 288 + 288 + 256 + 256 + 224 + 224 in the
// lock-step kernel, and no W buffer.
//
// CTA: 8 x TY cells (TY odd, so the NY = TY + 1 node rows pair up), 16 warps:
//   warps 0..7   "x12": warp (j3 = w & 3, segment = w >> 2) runs x1 along its 4-cell row
//                segment (5 nodes) for each node-row pair, feeding x2 chains (one per cell pair of
//                the segment) that roll down the node rows; finished x2 cell rows go to V.
//   warps 8..15  "x3": 2 TX TY / 8 (cell, line-half) chains rolled across planes (lock-step
//                kernel's x3, LEAN stores).
// One CTA barrier per plane: x12 of plane p writes V[p & 1] while x3 finishes plane p - 1 from
// V[(p - 1) & 1].  Input planes arrive by TMA bulk row copies into a 3-stage mbarrier ring; the
// tile rows are padded to 584 doubles so the two node rows of an x1 fragment hit disjoint bank
// halves.
// Measurement-only (tools build, -DH3_MEASURE): measured slower than the lock-step kernel, see
// profiles/r02_m3_fused_variants.txt; the product library does not contain it.
#ifdef H3_MEASURE
#include "h3_launch.h"
#include "h3_tma.cuh"

namespace h3 {
namespace x12 {

using tma::bulk_g2s;
using tma::fence_proxy_async_smem;
using tma::mbar_arrive_expect_tx;
using tma::mbar_fence_init;
using tma::mbar_init;
using tma::mbar_wait;

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

template <int TY_, int STAGES_ = 3, int B3_ = 7, int NX3_ = 8, bool SPLIT_ = false>
struct Cfg {
    // SPLIT: x1 of all node-row pairs first (4 independent chains, interleaved), then the two x2
    // chains -- a shorter dependency path per plane than row pair after row pair
    static constexpr bool SPLIT = SPLIT_;
    static constexpr int n = 4, n3 = 64;
    static constexpr int TX = 8, TY = TY_, NX = TX + 1, NY = TY + 1;
    static constexpr int NSEG = TX / 4;                 // 4-cell row segments
    static constexpr int NX12 = 4 * NSEG;              // x12 warps: (j3, segment)
    static constexpr int NX3 = NX3_, WARPS = NX12 + NX3, THREADS = 32 * WARPS;
    static constexpr int STAGES = STAGES_, B3 = B3_;
    static constexpr int URS = NX * n3 + 8;            // U tile-row stride (== 8 mod 16 doubles)
    static constexpr int VCS = 64, VROW = TX * VCS + 2;  // V [cy][cx][m2][m1][(j3 + (m2 >> 1)) & 3]
    static constexpr int T3 = 2 * TX * TY, K3 = T3 / NX3;
    static constexpr size_t U_D = (size_t)NY * URS;
    static constexpr size_t V_D = (size_t)TY * VROW;
    static constexpr size_t SMEM_DATA = (STAGES * U_D + 2 * V_D) * sizeof(double);
    static constexpr size_t SMEM = SMEM_DATA + STAGES * sizeof(uint64_t);
    static_assert(NY % 2 == 0, "x1 fragments pair node rows: TY must be odd");
    static_assert(T3 % NX3 == 0, "x3 chains must divide evenly among the x3 warps");
    static_assert(NY <= NX12, "one TMA lane per tile row among the x12 warps");
    static_assert(SMEM <= 232448, "shared memory per CTA");
};

}  // namespace x12

template <class C>
__global__ void __launch_bounds__(C::THREADS, 1)
sep_fused_dmma3x_kernel(const double* __restrict__ src, double* __restrict__ dst, Dims d, int off, int zchunk,
                        const __grid_constant__ SepOps<3> p, unsigned long long* first_bad,
                        const unsigned long long* guard) {
    using namespace x12;
    constexpr int n = C::n, n3 = C::n3, TX = C::TX, NX = C::NX, NY = C::NY, STAGES = C::STAGES;
    constexpr int URS = C::URS, VCS = C::VCS, VROW = C::VROW, K3 = C::K3;
    if (guarded_out(guard, first_bad)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* U = reinterpret_cast<double*>(smem_raw);
    double* V = U + STAGES * C::U_D;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + C::SMEM_DATA);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q = lane & 3, g = lane >> 2, par = q >> 1, hi = g >> 2;
    const int M1 = (int)d.M1, M2 = (int)d.M2;
    const int cx0 = blockIdx.x * TX, cy0 = blockIdx.y * C::TY;
    const int64_t zc0 = d.z_begin + (int64_t)blockIdx.z * zchunk;
    const int64_t zc1 = min(zc0 + (int64_t)zchunk, d.z_end);
    const int P = (int)(zc1 - zc0) + 1;
    const int64_t plane_elems = (int64_t)M1 * M2 * n3;

    // operator fragments, both column (row) orders: lane holds Op[g][q] = B_DA[q][g]
    auto frag = [&](int ax, double& f0, double& f1) {
        const int m = g & 3;
        f0 = hi ? p.A[ax][m][n + q] : p.A[ax][m][q];
        f1 = hi ? p.A[ax][m][q] : p.A[ax][m][n + q];
    };

    // ---- TMA loader: lane 0 of warp ly < NY copies tile row ly (split at the periodic wrap) ------
    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
        mbar_fence_init();
    }
    int rowoff = 0, gx0 = 0;
    if (lane == 0 && warp < NY) {
        int gy = (cy0 + off + warp) % M2;
        if (gy < 0) gy += M2;
        gx0 = (cx0 + off) % M1;
        if (gx0 < 0) gx0 += M1;
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
                if (warp == 0) mbar_arrive_expect_tx(&bars[s], (unsigned)(NY * NX * n3 * sizeof(double)));
                const double* base = plane_base(src, gz_next, plane_elems, d) + (int64_t)rowoff * n3;
                double* Ub = U + s * C::U_D + warp * URS;
                int got = 0, gx = gx0;
                while (got < NX) {
                    const int len = min(NX - got, M1 - gx);
                    bulk_g2s(Ub + got * n3, base + (int64_t)gx * n3, (unsigned)(len * n3 * sizeof(double)), &bars[s]);
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

    if (warp < C::NX12) {
        // =========================== x12 warps =====================================================
        const int j3 = warp & 3, seg = warp >> 2;
        double o1[2], o2[2];
        frag(0, o1[0], o1[1]);
        frag(1, o2[0], o2[1]);
        // x1 B fragment: lane (g, q) = data[j1 = q][line g = (j2 = g >> 1, row slot = g & 1)]
        const int uoff = (g & 1) * URS + (4 * seg) * n3 + j3 * 16 + (g >> 1) * 4 + q;
        // V store of x2 output (line (cell 2s + hi, m1 = g & 3), cols m2 = 2 (q & 1) + i):
        // [cy][cx][m2][m1][(j3 + (m2 >> 1)) & 3]; the row cy = 2k + par is added per store
        const int voff = (4 * seg + hi) * VCS + (2 * (q & 1)) * 16 + (g & 3) * 4 + ((j3 + (q & 1)) & 3);
        for (int pl = 0; pl < P; ++pl) {
            __syncthreads();
            issue();  // the stage it fills was last read before the barrier above
            mbar_wait(&bars[pl % STAGES], (unsigned)((pl / STAGES) & 1));
            const double* Ub = U + (pl % STAGES) * C::U_D + uoff;
            double* Vb = V + (pl & 1) * C::V_D + voff;
            double x2r[2][2], sv2[2][2];
#pragma unroll
            for (int s = 0; s < 2; ++s) x2r[s][0] = x2r[s][1] = sv2[s][0] = sv2[s][1] = 0.0;
            // x2 step of cell pair s at node row ly with A fragment xa; completed cell rows to V
            auto x2_step = [&](int s, int ly, double xa) {
                dmma(x2r[s][0], x2r[s][1], xa, o2[ly & 1]);
                // x2 completion: cell row ly - 1 in the lanes with par == (ly + 1) & 1
                if (ly & 1) {
                    if (ly == NY - 1) {  // lone last cell row: half-warp store
                        if (par == 0) {
                            double* v = Vb + (ly - 1) * VROW + s * 2 * VCS;
                            v[0] = x2r[s][0];
                            v[16] = x2r[s][1];
                        }
                    } else {
                        sv2[s][0] = x2r[s][0];
                        sv2[s][1] = x2r[s][1];
                    }
                } else if (ly > 0) {
                    // rows ly-2 (par 0, saved) and ly-1 (par 1) in one full-warp store
                    double* v = Vb + (ly - 2 + par) * VROW + s * 2 * VCS;
                    v[0] = par ? x2r[s][0] : sv2[s][0];
                    v[16] = par ? x2r[s][1] : sv2[s][1];
                }
                const bool d2 = par == ((ly + 1) & 1);
                x2r[s][0] = d2 ? 0.0 : x2r[s][0];
                x2r[s][1] = d2 ? 0.0 : x2r[s][1];
            };
            if constexpr (C::SPLIT) {
                constexpr int R = NY / 2;
                double r1[R][2], sv[R][2], xd[R][2][2];
#pragma unroll
                for (int r = 0; r < R; ++r) r1[r][0] = r1[r][1] = sv[r][0] = sv[r][1] = 0.0;
#pragma unroll
                for (int k = 0; k < 5; ++k) {
                    const bool done = hi == ((k + 1) & 1);
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        dmma(r1[r][0], r1[r][1], o1[k & 1], Ub[2 * r * URS + k * n3]);
                        if (k & 1) {
                            sv[r][0] = r1[r][0];
                            sv[r][1] = r1[r][1];
                        } else if (k > 0) {
                            const int s = (k - 2) >> 1;
                            xd[r][s][0] = hi ? r1[r][0] : sv[r][0];
                            xd[r][s][1] = hi ? r1[r][1] : sv[r][1];
                        }
                        r1[r][0] = done ? 0.0 : r1[r][0];
                        r1[r][1] = done ? 0.0 : r1[r][1];
                    }
                }
#pragma unroll
                for (int ly = 0; ly < NY; ++ly)
#pragma unroll
                    for (int s = 0; s < 2; ++s) x2_step(s, ly, xd[ly >> 1][s][ly & 1]);
            } else {
#pragma unroll
            for (int r = 0; r < NY / 2; ++r) {
                double a[5];
#pragma unroll
                for (int k = 0; k < 5; ++k) a[k] = Ub[2 * r * URS + k * n3];
                double r1[2] = {0.0, 0.0}, sv[2] = {0.0, 0.0};
#pragma unroll
                for (int k = 0; k < 5; ++k) {
                    // local node 4 seg + k (even at k = 0): parity k & 1
                    dmma(r1[0], r1[1], o1[k & 1], a[k]);
                    const bool done = hi == ((k + 1) & 1);  // lanes that just completed cell k-1
                    if (k & 1) {
                        sv[0] = r1[0];
                        sv[1] = r1[1];
                    } else if (k > 0) {
                        // cell pair s = (k - 2) / 2 of the segment is complete (even cell in g < 4
                        // from sv, odd cell in g >= 4): two x2 steps, node rows 2r (i = 0), 2r+1
                        const int s = (k - 2) >> 1;
#pragma unroll
                        for (int i = 0; i < 2; ++i) x2_step(s, 2 * r + i, hi ? r1[i] : sv[i]);
                    }
                    r1[0] = done ? 0.0 : r1[0];
                    r1[1] = done ? 0.0 : r1[1];
                }
            }
            }
        }
        __syncthreads();  // matches the x3 warps' final iteration
    } else {
        // =========================== x3 warps ======================================================
        const int w = warp - C::NX12;
        double b0, b1;
        frag(2, b0, b1);
        // chain k = (cell c0 + (NX3 / 2) k, half h) with c0 = w >> 1 < NX3 / 2: cell row
        // cyk(k), column c0 + cxk(k); line L = 8h + g = (m2, m1), k = j3 = q.  Offsets are a per-lane
        // base plus a compile-time term per chain.
        static_assert(TX == 8 && (C::NX3 == 8 || C::NX3 == 16), "x3 chain -> cell map: 8-wide tiles, 8 or 16 x3 warps");
        constexpr int CS = C::NX3 / 2;  // cell stride between a warp's chains
        auto cxk = [](int k) { return (CS * k) % TX; };
        auto cyk = [](int k) { return (CS * k) / TX; };
        const int c0 = w >> 1, h = w & 1, L = 8 * h + g;
        const int vbase = c0 * VCS + L * 4 + ((q + h) & 3);
        const int obase = (cy0 * M1 + cx0 + c0) * n3 + (2 * (q & 1)) * 16 + L;  // int32: M1 M2 64 < 2^31
        const int rowstep = M1 * n3;
        unsigned live = 0;  // chains whose cell lies inside the grid
#pragma unroll
        for (int k = 0; k < K3; ++k)
            if (cx0 + c0 + cxk(k) < M1 && cy0 + cyk(k) < M2) live |= 1u << k;
        auto va = [&](int k) { return cyk(k) * VROW + cxk(k) * VCS; };  // + vbase
        auto ooff = [&](int k) { return obase + cyk(k) * rowstep + cxk(k) * n3; };
        double acc[K3][2];
#pragma unroll
        for (int k = 0; k < K3; ++k) acc[k][0] = acc[k][1] = 0.0;
        for (int pl = 0; pl <= P; ++pl) {
            __syncthreads();
            if (pl == 0) continue;
            const int t = pl - 1;  // node plane whose V this iteration contracts
            const double* Vb = V + (t & 1) * C::V_D + vbase;
            double* ob = dst + (zc0 + t - 1) * plane_elems + obase;
            // chain k completes cell plane t-1 in the lanes with par == (t + k + 1) & 1
            const bool de = par == ((t + 1) & 1);  // even chains
            unsigned screen = 0x7ff00000u;
            double a[K3];
#pragma unroll
            for (int k = 0; k < K3; ++k) a[k] = Vb[va(k)];
#pragma unroll
            for (int k = 0; k < K3; ++k) {
                const bool done = (k & 1) ? !de : de;
                dmma(acc[k][0], acc[k][1], a[k], ((t + k) & 1) ? b1 : b0);
                if (t > 0) {
                    if (done && (live >> k & 1u)) {  // finished lanes of live chains
                        double* o = ob + (cyk(k) * rowstep + cxk(k) * n3);
                        __stcs(o, acc[k][0]);
                        __stcs(o + 16, acc[k][1]);
                    }
                    screen = min(screen, min(exp_gap(acc[k][0]), exp_gap(acc[k][1])));
                }
                acc[k][0] = done ? 0.0 : acc[k][0];
                acc[k][1] = done ? 0.0 : acc[k][1];
            }
            if (t > 0 && screen == 0u) {  // rare: some lane holds Inf/NaN -- locate it exactly
                double* oplane = dst + (zc0 + t - 1) * plane_elems;
#pragma unroll
                for (int k = 0; k < K3; ++k) {
                    const bool done = (k & 1) ? !de : de;
                    if (done && (live >> k & 1u) &&
                        (!isfinite(oplane[ooff(k)]) || !isfinite(oplane[ooff(k) + 16])))
                        flag_bad(first_bad, (zc0 + t - 1) * M2 * (int64_t)M1 + ooff(k) / n3);
                }
            }
        }
    }
}

template <class C>
static int launch_x12(const double* src, double* dst, const Dims& d, const SepOps<3>& ops, int off,
                      cudaStream_t st, unsigned long long* first_bad, const unsigned long long* guard,
                      int cluster_y) {
    const int64_t nz = d.z_end - d.z_begin;
    auto kern = sep_fused_dmma3x_kernel<C>;
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

int sep_fused_dmma3x_launch(const double* src, double* dst, const Dims& d, const SepOps<3>& ops, int off,
                            cudaStream_t st, unsigned long long* first_bad, const unsigned long long* guard,
                            int variant) {
    using x12::Cfg;
    switch (variant) {
        case 1: return launch_x12<Cfg<7, 3, 7, 16>>(src, dst, d, ops, off, st, first_bad, guard, 2);
        case 2: return launch_x12<Cfg<7, 4, 7, 16>>(src, dst, d, ops, off, st, first_bad, guard, 2);
        case 3: return launch_x12<Cfg<7, 3, 4, 16>>(src, dst, d, ops, off, st, first_bad, guard, 2);
        case 4: return launch_x12<Cfg<7, 3, 2, 8>>(src, dst, d, ops, off, st, first_bad, guard, 2);
        case 5: return launch_x12<Cfg<7, 3, 7, 16>>(src, dst, d, ops, off, st, first_bad, guard, 1);
        case 6: return launch_x12<Cfg<7, 3, 7, 16, true>>(src, dst, d, ops, off, st, first_bad, guard, 2);
        case 7: return launch_x12<Cfg<7, 4, 7, 16, true>>(src, dst, d, ops, off, st, first_bad, guard, 2);
        case 8: return launch_x12<Cfg<7, 3, 7, 8, true>>(src, dst, d, ops, off, st, first_bad, guard, 2);
        default: break;
    }
    return launch_x12<Cfg<7, 3, 7>>(src, dst, d, ops, off, st, first_bad, guard, 2);
}

}  // namespace h3
#endif  // H3_MEASURE
