// Microbenchmark: dependent-chain latency of DMMA.8x8x4 and DFMA on one SM, and
// throughput vs independent chains per warp / warps per SM.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void dmma_chain(double* out, int iters, long long* cycles) {
    double a = threadIdx.x * 1e-3, b = 0.5;
    double c[CH][2] = {};
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < CH; ++j)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
    }
    long long t1 = clock64();
    double s = 0;
    for (int j = 0; j < CH; ++j) s += c[j][0] + c[j][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = t1 - t0;
}

// chain with the fused kernel's rolling-accumulation pattern: half the lanes zero their
// accumulator between dependent DMMAs (alternating halves)
template <int CH>
__global__ void dmma_chain_sel(double* out, int iters, long long* cycles) {
    double a = threadIdx.x * 1e-3, b = 0.5;
    double c[CH][2] = {};
    const bool hi = (threadIdx.x & 3) >= 2;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < CH; ++j) {
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
            const bool z = hi ^ (i & 1);
#ifdef ZASM
            asm volatile("{.reg .pred p; setp.ne.u32 p, %2, 0; @p mov.b64 %0, 0; @p mov.b64 %1, 0;}"
                         : "+d"(c[j][0]), "+d"(c[j][1]) : "r"((unsigned)z));
#else
            c[j][0] = z ? 0.0 : c[j][0];
            c[j][1] = z ? 0.0 : c[j][1];
#endif
        }
    }
    long long t1 = clock64();
    double s = 0;
    for (int j = 0; j < CH; ++j) s += c[j][0] + c[j][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = t1 - t0;
}

template <int CH>
__global__ void dfma_chain(double* out, int iters, long long* cycles) {
    double c[CH];
    for (int j = 0; j < CH; ++j) c[j] = threadIdx.x + j;
    const double b = 0.999999, d = 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < CH; ++j) c[j] = fma(c[j], b, d);
    }
    long long t1 = clock64();
    double s = 0;
    for (int j = 0; j < CH; ++j) s += c[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = t1 - t0;
}

template <int CH>
void run(double* out, long long* cyc, int warps) {
    long long h;
    int iters = 2000;
    dmma_chain<CH><<<1, 32 * warps>>>(out, iters, cyc);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DMMA chains/warp %d warps/SM %2d: %.1f cycles per chain step (%.2f DMMA/clk/SM)\n", CH, warps,
           (double)h / iters, (double)CH * warps * iters / h);
    dmma_chain_sel<CH><<<1, 32 * warps>>>(out, iters, cyc);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DMMA+FSEL chains/warp %d warps/SM %2d: %.1f cycles per chain step (%.2f DMMA/clk/SM)\n", CH, warps,
           (double)h / iters, (double)CH * warps * iters / h);
    dfma_chain<CH><<<1, 32 * warps>>>(out, iters * 4, cyc);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA chains/warp %d warps/SM %2d: %.1f cycles per chain step (%.2f warp-DFMA/clk/SM)\n", CH, warps,
           (double)h / (iters * 4), (double)CH * warps * iters * 4 / h);
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 1 << 20);
    cudaMalloc(&cyc, 8);
    for (int w : {1, 4, 8, 16, 32}) {
        run<1>(out, cyc, w);
        run<2>(out, cyc, w);
        run<4>(out, cyc, w);
    }
    return 0;
}
