// Microbenchmark: does DMMA (mma.sync m8n8k4 f64) share issue/pipe capacity with DADD, DMUL,
// DFMA and 32-bit selects?  Each variant runs 4 independent DMMA chains per warp plus X extra
// instructions per DMMA; the printed DMMA rate shows how much the extras slow the tensor pipe.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE, int X>
__global__ void mix(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 0.5;
    double c[4][2] = {};
    double e[8];
    for (int j = 0; j < 8; ++j) e[j] = threadIdx.x * 1e-7 + j;
    const double f = 1.0000001, g = 1e-12;
    int sel = threadIdx.x & 1;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                             : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
#pragma unroll
                for (int x = 0; x < X; ++x) {
                    double& v = e[(j * X + x) & 7];
                    if (MODE == 1) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(v) : "d"(g));
                    if (MODE == 2) asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(v) : "d"(f));
                    if (MODE == 3) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(v) : "d"(f), "d"(g));
                    if (MODE == 4) {
                        int lo = __double2loint(v);
                        asm volatile("{.reg .pred p; setp.ne.s32 p, %1, 0; selp.b32 %0, %0, 0, p;}" : "+r"(lo) : "r"(sel));
                        v = __hiloint2double(__double2hiint(v), lo);
                    }
                }
            }
        }
    }
    double s = 0;
    for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
    for (int j = 0; j < 8; ++j) s += e[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE, int X>
void run(const char* name, double* out, int sms, int threads) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 2048;
    mix<MODE, X><<<sms, threads>>>(out, 16);
    cudaEventRecord(e0);
    mix<MODE, X><<<sms, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double dmma = (double)sms * (threads / 32) * iters * 32;
    printf("%-22s threads %4d: DMMA %.2f TFLOP/s, %.2f ns per DMMA per SMSP\n", name, threads,
           2.0 * 256 * dmma / ms / 1e9, ms * 1e6 / (dmma / (sms * 4)));
}

int main() {
    double* out;
    cudaMalloc(&out, 148 * 1024 * sizeof(double));
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int threads : {128, 512}) {
        run<0, 0>("dmma only", out, sms, threads);
        run<1, 2>("dmma + 2 dadd", out, sms, threads);
        run<1, 4>("dmma + 4 dadd", out, sms, threads);
        run<2, 2>("dmma + 2 dmul", out, sms, threads);
        run<3, 2>("dmma + 2 dfma", out, sms, threads);
        run<3, 8>("dmma + 8 dfma", out, sms, threads);
        run<4, 4>("dmma + 4 selp.b32", out, sms, threads);
        run<4, 8>("dmma + 8 selp.b32", out, sms, threads);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
