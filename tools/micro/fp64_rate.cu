// DFMA / MUFU.RCP64H / F2F throughput per SM (cycles per warp instruction), 32 warps per SM
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double* out, float* fin, long long* cyc, int iters) {
    double a0 = threadIdx.x * 1e-3 + 1.0, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double b = 1.0000001, c = 1e-9;
    float f = fin[threadIdx.x];
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (MODE == 0) {
            a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
            a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
        } else if (MODE == 1) {
            asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(a0)); asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(a1));
            asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(a2)); asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(a3));
            asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(a4)); asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(a5));
            asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(a6)); asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(a7));
        } else {
            a0 += (double)f; f += 1.0f; a1 += (double)f; f += 1.0f; a2 += (double)f; f += 1.0f; a3 += (double)f; f += 1.0f;
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 + f;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    double* out; float* fin; long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 8); cudaMalloc(&fin, 4096); cudaMemset(fin, 0, 4096); cudaMalloc(&cyc, 148 * 8);
    const int iters = 4096;
    long long h[148];
    const char* names[3] = {"DFMA", "MUFU.RCP64H", "F2F.F64.F32 + DADD (+FADD)"};
    for (int m = 0; m < 3; ++m) {
        if (m == 0) k<0><<<148, 1024>>>(out, fin, cyc, iters);
        if (m == 1) k<1><<<148, 1024>>>(out, fin, cyc, iters);
        if (m == 2) k<2><<<148, 1024>>>(out, fin, cyc, iters);
        cudaDeviceSynchronize();
        cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        const int per = m == 2 ? 4 : 8;
        printf("%s: %.2f cycles per warp instruction per SM (32 warps) -> %.1f lanes/clk/SM\n", names[m],
               (double)h[0] / (iters * per * 32.0), 32.0 * iters * per * 32.0 / h[0]);
    }
    return 0;
}
