// Micro-benchmark: per-SM issue rate of DFMA, F2F.F64.F32, MUFU.RCP64H, I2F.F64 on this GPU.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(double* out, float* fout, int iters) {
    double a = threadIdx.x * 1e-3 + 1.0, b = 1.0000001, c = 1e-9;
    double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
    float f = threadIdx.x * 1e-3f + 1.f;
    int iv = threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        if (OP == 0) {            // DFMA, 8 independent chains
            x0 = fma(x0, b, c); x1 = fma(x1, b, c); x2 = fma(x2, b, c); x3 = fma(x3, b, c);
            x4 = fma(x4, b, c); x5 = fma(x5, b, c); x6 = fma(x6, b, c); x7 = fma(x7, b, c);
        } else if (OP == 1) {     // F2F.F64.F32
            x0 += (double)(f + 1.f); x1 += (double)(f + 2.f); x2 += (double)(f + 3.f); x3 += (double)(f + 4.f);
            f += 1e-7f;
        } else if (OP == 2) {     // MUFU.RCP64H
            double r0, r1, r2, r3;
            asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r0) : "d"(x0));
            asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r1) : "d"(x1));
            asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r2) : "d"(x2));
            asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r3) : "d"(x3));
            x0 = r0 + 1.0; x1 = r1 + 1.0; x2 = r2 + 1.0; x3 = r3 + 1.0;
        } else if (OP == 3) {     // I2F.F64
            x0 += (double)(iv + i); x1 += (double)(iv - i); x2 += (double)(iv ^ i); x3 += (double)(iv + 2 * i);
        } else {                  // FFMA fp32 reference, 8 chains
            float y0 = (float)x0;
            for (int q = 0; q < 1; ++q) f = fmaf(f, 1.0000001f, 1e-9f);
            x0 = y0;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    fout[blockIdx.x * blockDim.x + threadIdx.x] = f;
}

template <int OP>
void run(const char* name, int ops_per_iter, double* d, float* fo) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 20000, threads = 1024, blocks = sms;
    k<OP><<<blocks, threads>>>(d, fo, 10);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<OP><<<blocks, threads>>>(d, fo, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double cycles = ms * 1e-3 * clk * 1e3;
    double thread_ops = (double)threads * iters * ops_per_iter;   // per SM
    printf("%-14s %7.2f thread-ops/clk/SM  (%.3f ms)\n", name, thread_ops / cycles, ms);
}

int main() {
    double* d; float* fo;
    cudaMalloc(&d, 1 << 24); cudaMalloc(&fo, 1 << 24);
    run<0>("DFMA", 8, d, fo);
    run<1>("F2F.F64.F32", 4, d, fo);
    run<2>("MUFU.RCP64H", 4, d, fo);
    run<3>("I2F.F64", 4, d, fo);
    return 0;
}
