// Shared device helpers for the Hermite half-step kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define H3_MAX_ORDER 5
#define H3_MAX_STAGES 128
#define H3_NO_BAD 0xFFFFFFFFFFFFFFFFull

namespace h3 {

// Periodic wrap of a (possibly slightly negative) index.
__device__ __forceinline__ int64_t wrap(int64_t v, int64_t m) {
    int64_t r = v % m;
    return r < 0 ? r + m : r;
}

// Node-plane index along x3: wrapped when the field is periodic in z, used
// as-is (ghost planes just outside [0, M3)) when the slab is part of a
// distributed field whose neighbour planes were received by the halo exchange.
__device__ __forceinline__ int64_t zplane(int64_t v, int64_t m3, int periodic_z) {
    return periodic_z ? wrap(v, m3) : v;
}

// Round-to-nearest multiply/add that the compiler may never contract into an
// FMA: the literal (parity) kernels reproduce the reference's separate
// multiply-then-add sequence bit for bit (gridkernels.py:58-110).
template <typename T> struct RN;
template <> struct RN<double> {
    static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
};
template <> struct RN<float> {
    static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
    static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
};

template <typename T> __device__ __forceinline__ bool finite(T v) { return isfinite(v); }

// First non-finite node in C order (m3, m2, m1): the reference reports the
// first offending node of the destination scan (pipeline.py:210-215).
__device__ __forceinline__ void flag_bad(unsigned long long* first_bad, int64_t lin) {
    if (first_bad) atomicMin(first_bad, (unsigned long long)lin);
}

// A kernel given a guard pointer skips all work when the guard already holds a
// bad node: the reference raises after the first half step and never runs the
// second one, so the destination of the second half step stays untouched.
// A skipped call copies the guard into its own flag so that a chain of half
// steps (each guarded by its predecessor's flag) stays skipped after a failure.
__device__ __forceinline__ bool guarded_out(const unsigned long long* guard,
                                            unsigned long long* first_bad) {
    if (guard == nullptr) return false;
    const unsigned long long g = *((volatile const unsigned long long*)guard);
    if (g == H3_NO_BAD) return false;
    if (first_bad && threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0)
        atomicMin(first_bad, g);
    return true;
}

// ---- cp.async (LDGSTS) helpers --------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(smem)), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

}  // namespace h3
