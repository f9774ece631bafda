// Ceiling of the fused kernel's memory access pattern without its compute: per CTA an 8x7-cell
// tile marches along x3; every node plane (9x8 node blocks of 512 B, periodic) arrives by TMA bulk
// row copies into a 3-stage mbarrier ring, and the 8x7 cell blocks of the previous plane leave
// with the same per-lane 8-byte streaming stores as sep_fused_dmma3_kernel (or 16-byte stores).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <nvml.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void expect(uint64_t* b, unsigned n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void waitp(uint64_t* b, unsigned ph) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void g2s(void* s, const void* g, unsigned n, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(s)), "l"(g), "r"(n), "r"(su32(b)) : "memory");
}

__device__ __forceinline__ void s2g(void* g, const void* s, unsigned n) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(su32(s)), "r"(n) : "memory");
}

// 0: 8-B stores like the kernel, 1: 16-B stores, 2: no stores, 3: TMA bulk stores (one 4-KB
// cell row per copy, straight from the staged plane)
template <int MODE>
__global__ void __launch_bounds__(512, 1) tile_stream(const double* src, double* dst, int M, int nz) {
    constexpr int TX = 8, TY = 7, NX = 9, NY = 8, ST = 3, UD = NX * NY * 64;
    extern __shared__ __align__(16) unsigned char sm[];
    double* U = (double*)sm;
    uint64_t* bars = (uint64_t*)(sm + ST * UD * 8);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, q = lane & 3, g = lane >> 2;
    const int cx0 = blockIdx.x * TX, cy0 = blockIdx.y * TY;
    const long plane = (long)M * M * 64;
    if (tid == 0) { for (int s = 0; s < ST; ++s) mbar_init(&bars[s], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncthreads();
    auto issue = [&](int p) {
        if (p < nz + 1 && lane == 0 && warp < NY) {
            const int s = p % ST;
            if (warp == 0) expect(&bars[s], UD * 8);
            const int gy = (cy0 + warp) % M;
            const double* base = src + (long)(p % nz) * plane + (long)gy * M * 64;
            int got = 0, gx = cx0;
            while (got < NX) { int len = min(NX - got, M - gx); g2s(U + s * UD + (warp * NX + got) * 64, base + (long)gx * 64, len * 512, &bars[s]); got += len; gx = 0; }
        }
    };
    issue(0); issue(1);
    for (int p = 0; p <= nz; ++p) {
        if (MODE == 3 && tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncthreads();
        issue(p + 2);
        waitp(&bars[p % ST], (p / ST) & 1);
        const double* Ub = U + (p % ST) * UD;
        if (p > 0 && MODE == 3) {
            if (tid == 0) {
                double* op = dst + (long)(p - 1) * plane;
                for (int cy = 0; cy < TY && cy0 + cy < M; ++cy)
                    s2g(op + ((long)(cy0 + cy) * M + cx0) * 64, Ub + cy * NX * 64, min(TX, M - cx0) * 512);
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        } else if (p > 0 && MODE != 2) {
            double* op = dst + (long)(p - 1) * plane;
            for (int k = 0; k < 7; ++k) {
                const int t = warp + 16 * k, cell = t >> 1, h = t & 1;
                const int cx = cell % TX, cy = cell / TX;
                if (cy0 + cy >= M) continue;
                const double* s = Ub + (cy * NX + cx) * 64;
                double* o = op + ((long)(cy0 + cy) * M + cx0 + cx) * 64;
                if (MODE == 0) {
                    const int pos = (2 * (q & 1)) * 16 + 8 * h + g;
                    if (((p + k) & 1) == (q >> 1)) { __stcs(o + pos, s[pos]); __stcs(o + pos + 16, s[pos + 16]); }
                } else if (h == 0 && ((p + k) & 1) == 0) {  // whole 512-B block, 16 B per lane
                    __stcs((double2*)(o + 2 * lane), *(const double2*)(s + 2 * lane));
                } else if (h == 0) {
                    __stcs((double2*)(o + 2 * lane), *(const double2*)(s + 2 * lane));
                }
            }
        }
    }
}

int main() {
    const int M = 512, nz = 512;
    const size_t n = (size_t)M * M * nz * 64;
    double *a, *b;
    if (cudaMalloc(&a, n * 8) || cudaMalloc(&b, n * 8)) { printf("alloc failed\n"); return 1; }
    cudaMemset(a, 0, n * 8);
    const int smem = 3 * 72 * 64 * 8 + 64;
    cudaFuncSetAttribute(tile_stream<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(tile_stream<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(tile_stream<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(tile_stream<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    dim3 grid(M / 8, (M + 6) / 7);
    nvmlDevice_t dev;
    const bool nv = nvmlInit() == NVML_SUCCESS && nvmlDeviceGetHandleByIndex(0, &dev) == NVML_SUCCESS;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const char* names[] = {"8-B lane stores", "16-B stores", "loads only", "TMA bulk stores"};
    const int reps = 12;
    for (int mode : {0, 3, 1, 2, 0, 3})
        {
            auto launch = [&] {
                if (mode == 0) tile_stream<0><<<grid, 512, smem>>>(a, b, M, nz);
                if (mode == 1) tile_stream<1><<<grid, 512, smem>>>(a, b, M, nz);
                if (mode == 2) tile_stream<2><<<grid, 512, smem>>>(a, b, M, nz);
                if (mode == 3) tile_stream<3><<<grid, 512, smem>>>(a, b, M, nz);
            };
            launch();
            cudaDeviceSynchronize();
            unsigned long long j0 = 0, j1 = 0;
            if (nv) nvmlDeviceGetTotalEnergyConsumption(dev, &j0);
            cudaEventRecord(e0);
            for (int r = 0; r < reps; ++r) launch();
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            if (nv) nvmlDeviceGetTotalEnergyConsumption(dev, &j1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            ms /= reps;
            const double bytes = (mode == 2 ? 1.0 : 2.0) * n * 8;
            printf("mode %d (%s): %.2f ms, %.0f GB/s (algorithmic %s), %.2f J per pass, %.0f W\n", mode, names[mode], ms,
                   bytes / ms / 1e6, mode == 2 ? "read" : "read+write", (j1 - j0) / 1e3 / reps,
                   (j1 - j0) / 1e3 / reps / (ms / 1e3));
        }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
