// Literal Hermite half-step kernels: the reference's per-cell arithmetic
// (gather -> three H sweeps -> q-stage Horner -> scatter), operation for
// operation, so the result is bit-identical to the reference
// (pkg/src/hermite3d/gridkernels.py:42-182).
//
// Layout: one CTA holds CPB cells; each cell is worked on by s^2 threads, one
// per (outer, middle) line of the s^3 local tensor, with two s^3 buffers in
// shared memory.  Multiplies and adds use __dmul_rn/__dadd_rn (never
// contracted to FMA) unless FAST is set, in which case the same sweeps use
// FMA (the two-kernel fast path's reconstruction).
//
// These kernels are FP64-issue bound (the reference algorithm does
// 3s^4 + q(3s^2(s-1)+s^3) MACs per cell); they are the
// parity path and the paper-faithful comparison, not the headline kernel.
#include "h3_launch.h"

namespace h3 {

template <typename T, bool FAST>
struct Arith {
    static __device__ __forceinline__ T mul(T a, T b) { return RN<T>::mul(a, b); }
    static __device__ __forceinline__ T mac(T acc, T a, T b) { return RN<T>::add(acc, RN<T>::mul(a, b)); }
};
template <typename T>
struct Arith<T, true> {
    static __device__ __forceinline__ T mul(T a, T b) { return a * b; }
    static __device__ __forceinline__ T mac(T acc, T a, T b) { return fma(a, b, acc); }
};

template <int N>
constexpr int lit_cpb() {
    constexpr int s2 = (2 * N + 2) * (2 * N + 2);
    return s2 >= 256 ? 1 : (256 / s2 < 1 ? 1 : 256 / s2);
}

// mode 0: fused  (src nodes -> dst nodes)
// mode 1: recon  (src nodes -> coeff cells of the slab chunk [z_begin, z_end))
// mode 2: evolve (coeff cells of the chunk -> dst nodes)
template <typename T, int N, int CPB, int MODE, bool FAST>
__global__ void __launch_bounds__(CPB*(2 * N + 2) * (2 * N + 2))
literal_kernel(const T* __restrict__ in, T* __restrict__ out, Dims d, int off,
               const __grid_constant__ LitOps<T, N> p, unsigned long long* first_bad,
               const unsigned long long* guard) {
    constexpr int n = N + 1, S = 2 * n, S2 = S * S, S3 = S2 * S, n3 = n * n * n;
    // shared tensors [a][b][c] with the innermost stride padded to SP = S + 1: the lanes of every
    // sweep and of the Horner stages then hit distinct banks (an unpadded 8-double row stride put
    // 8 lanes of a half-warp on the same bank pair at N = 3)
    constexpr int SP = S + 1, SB = S2 * SP;
    using A = Arith<T, FAST>;
    if (guarded_out(guard, first_bad)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* sm = reinterpret_cast<T*>(smem_raw);

    const int local = threadIdx.x / S2;
    const int t = threadIdx.x % S2;
    T* bufA = sm + (size_t)local * 2 * SB;
    T* bufB = bufA + SB;

    const int64_t nxy = d.M1 * d.M2;
    const int64_t total = (d.z_end - d.z_begin) * nxy;
    const int64_t cell = (int64_t)blockIdx.x * CPB + local;
    const bool valid = cell < total;
    const int64_t crel3 = valid ? cell / nxy : 0;
    const int64_t rem = valid ? cell - crel3 * nxy : 0;
    const int64_t c3 = d.z_begin + crel3, c2 = rem / d.M1, c1 = rem - (rem / d.M1) * d.M1;

    if (MODE != 2) {
        // ---- gather (gridkernels.py:42-55) -------------------------------------
        if (valid) {
            for (int e = t; e < S3; e += S2) {
                const int zz = e / S2, yy = (e / S) % S, xx = e % S;
                const int a3 = zz / n, j3 = zz % n, a2 = yy / n, j2 = yy % n, a1 = xx / n, j1 = xx % n;
                const int64_t g3 = zplane(c3 + off + a3, d.M3, d.periodic_z);
                const int64_t g2 = wrap(c2 + off + a2, d.M2);
                const int64_t g1 = wrap(c1 + off + a1, d.M1);
                bufA[(zz * S + yy) * SP + xx] = in[((g3 * d.M2 + g2) * d.M1 + g1) * n3 + (j3 * n + j2) * n + j1];
            }
        }
        __syncthreads();
        // ---- reconstruct (gridkernels.py:58-83): sweeps x1, x2, x3 ---------------
        {
            const int o = t / S, m = t % S;  // (z, y)
            T u[S];
#pragma unroll
            for (int k = 0; k < S; ++k) u[k] = bufA[(o * S + m) * SP + k];
#pragma unroll
            for (int i = 0; i < S; ++i) {
                T c = A::mul(p.H[i * S], u[0]);
#pragma unroll
                for (int k = 1; k < S; ++k) c = A::mac(c, p.H[i * S + k], u[k]);
                bufB[(o * S + m) * SP + i] = c;
            }
        }
        __syncthreads();
        {
            const int o = t / S, x = t % S;  // (z, x)
            T u[S];
#pragma unroll
            for (int k = 0; k < S; ++k) u[k] = bufB[(o * S + k) * SP + x];
#pragma unroll
            for (int i = 0; i < S; ++i) {
                T c = A::mul(p.H[i * S], u[0]);
#pragma unroll
                for (int k = 1; k < S; ++k) c = A::mac(c, p.H[i * S + k], u[k]);
                bufA[(o * S + i) * SP + x] = c;
            }
        }
        __syncthreads();
        {
            const int y = t / S, x = t % S;  // (y, x)
            T u[S];
#pragma unroll
            for (int k = 0; k < S; ++k) u[k] = bufA[(k * S + y) * SP + x];
#pragma unroll
            for (int i = 0; i < S; ++i) {
                T c = A::mul(p.H[i * S], u[0]);
#pragma unroll
                for (int k = 1; k < S; ++k) c = A::mac(c, p.H[i * S + k], u[k]);
                bufB[(i * S + y) * SP + x] = c;
            }
        }
        __syncthreads();
        if (MODE == 1) {
            if (valid) {
                T* dstc = out + (size_t)cell * S3;  // chunk-relative cell index
                for (int e = t; e < S3; e += S2) dstc[e] = bufB[(e / S) * SP + e % S];
            }
            return;
        }
    } else {
        if (valid) {
            const T* srcc = in + (size_t)cell * S3;
            for (int e = t; e < S3; e += S2) bufB[(e / S) * SP + e % S] = srcc[e];
        }
        __syncthreads();
    }

    // ---- evolve (gridkernels.py:86-110): q-stage Horner, two-phase --------------
    // Stage k reads the neighbours' stage-(k-1) values from `cur` and writes its own to `nxt`
    // (the two buffers alternate), so one barrier per stage orders both the reads after the
    // writes and the next overwrite after the reads.  When a cell's threads are whole warps
    // (N = 3: 64 threads) the barrier is the cell's own named barrier, not the CTA's.
    auto cell_sync = [&]() {
        if constexpr (CPB > 1 && S2 % 32 == 0)
            asm volatile("bar.sync %0, %1;" ::"r"(1 + local), "n"(S2) : "memory");
        else
            __syncthreads();
    };
    const int z = t / S, y = t % S;
    T ru[S], w[S];
#pragma unroll
    for (int x = 0; x < S; ++x) {
        ru[x] = bufB[(z * S + y) * SP + x];
        w[x] = ru[x];
        bufA[(z * S + y) * SP + x] = ru[x];
    }
    __syncthreads();
    T* cur = bufA;
    T* nxt = bufB;
    // this thread's y / z factors are stage-invariant: load them once (a per-thread index into the
    // parameter bank would otherwise be re-read, serialised across the warp, every stage)
    const T f2y = p.f2[y], f3z = p.f3[z], zero = p.f1[S - 1];
    for (int k = p.q; k >= 1; --k) {
        const T c = p.cf[k - 1];
        T nw[S];
#pragma unroll
        for (int x = 0; x < S; ++x) {
            T acc = zero;  // the reference's typed zero
            if (x < S - 1) acc = RN<T>::add(acc, RN<T>::mul(p.f1[x], w[x + 1]));
            if (y < S - 1) acc = RN<T>::add(acc, RN<T>::mul(f2y, cur[(z * S + y + 1) * SP + x]));
            if (z < S - 1) acc = RN<T>::add(acc, RN<T>::mul(f3z, cur[((z + 1) * S + y) * SP + x]));
            nw[x] = RN<T>::add(ru[x], RN<T>::mul(c, acc));
        }
#pragma unroll
        for (int x = 0; x < S; ++x) {
            w[x] = nw[x];
            nxt[(z * S + y) * SP + x] = nw[x];
        }
        cell_sync();
        T* const tmp = cur;
        cur = nxt;
        nxt = tmp;
    }
    // ---- scatter (gridkernels.py:113-118) -----------------------------------------
    if (valid && z < n && y < n) {
        const int64_t node = (c3 * d.M2 + c2) * d.M1 + c1;
        T* dn = out + node * n3 + (z * n + y) * n;
        bool bad = false;
#pragma unroll
        for (int x = 0; x < n; ++x) {
            dn[x] = w[x];
            bad |= !finite(w[x]);
        }
        if (bad) flag_bad(first_bad, node);
    }
}

template <typename T, int N, int MODE, bool FAST>
static int launch_one(const T* in, T* out, const Dims& d, const LitOps<T, N>& ops, int off,
                      cudaStream_t st, unsigned long long* first_bad,
                      const unsigned long long* guard) {
    constexpr int S = 2 * N + 2, S2 = S * S, CPB = lit_cpb<N>(), SB = S2 * (S + 1);
    const int64_t total = (d.z_end - d.z_begin) * d.M1 * d.M2;
    if (total <= 0) return 0;
    const size_t smem = (size_t)CPB * 2 * SB * sizeof(T);
    auto kern = literal_kernel<T, N, CPB, MODE, FAST>;
    // per-device attribute; cheap and idempotent, so set on every launch
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    const int64_t blocks = (total + CPB - 1) / CPB;
    kern<<<(unsigned)blocks, CPB * S2, smem, st>>>(in, out, d, off, ops, first_bad, guard);
    return (int)cudaGetLastError();
}

template <typename T, int N>
static int dispatch_mode(int mode, bool fast, const T* in, T* out, const Dims& d, const T* H,
                         const T* f1, const T* f2, const T* f3, const T* cf, int q, int off,
                         cudaStream_t st, unsigned long long* first_bad,
                         const unsigned long long* guard) {
    constexpr int S = 2 * N + 2;
    LitOps<T, N> ops;
    for (int i = 0; i < S * S; ++i) ops.H[i] = H ? H[i] : T(0);
    for (int i = 0; i < S; ++i) {
        ops.f1[i] = f1 ? f1[i] : T(0);
        ops.f2[i] = f2 ? f2[i] : T(0);
        ops.f3[i] = f3 ? f3[i] : T(0);
    }
    for (int i = 0; i < H3_MAX_STAGES; ++i) ops.cf[i] = (cf && i < q) ? cf[i] : T(0);
    ops.q = q;
    switch (mode) {
        case 0:
            return launch_one<T, N, 0, false>(in, out, d, ops, off, st, first_bad, guard);
        case 1:
#ifdef H3_MEASURE
            // the FMA per-cell sweeps (H3_RECON_IMPL=fma) exist in the tools library only
            if (fast) return launch_one<T, N, 1, true>(in, out, d, ops, off, st, first_bad, guard);
#else
            (void)fast;
#endif
            return launch_one<T, N, 1, false>(in, out, d, ops, off, st, first_bad, guard);
        case 2:
            return launch_one<T, N, 2, false>(in, out, d, ops, off, st, first_bad, guard);
    }
    return (int)cudaErrorInvalidValue;
}

template <typename T>
int literal_launch(int mode, bool fast, const T* in, T* out, const Dims& d, int order_n,
                   const T* H, const T* f1, const T* f2, const T* f3, const T* cf, int q,
                   int off, cudaStream_t st, unsigned long long* first_bad,
                   const unsigned long long* guard) {
    switch (order_n) {
#define H3_CASE(NN) \
    case NN: return dispatch_mode<T, NN>(mode, fast, in, out, d, H, f1, f2, f3, cf, q, off, st, first_bad, guard);
        H3_CASE(0) H3_CASE(1) H3_CASE(2) H3_CASE(3) H3_CASE(4) H3_CASE(5)
#undef H3_CASE
    }
    return (int)cudaErrorInvalidValue;
}

template int literal_launch<double>(int, bool, const double*, double*, const Dims&, int,
                                    const double*, const double*, const double*, const double*,
                                    const double*, int, int, cudaStream_t, unsigned long long*,
                                    const unsigned long long*);
template int literal_launch<float>(int, bool, const float*, float*, const Dims&, int,
                                   const float*, const float*, const float*, const float*,
                                   const float*, int, int, cudaStream_t, unsigned long long*,
                                   const unsigned long long*);

}  // namespace h3
