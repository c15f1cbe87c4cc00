// Issue-rate microbenchmark behind the encoder's roofline (K1):
// per-SM throughput of the instruction classes the nearest-centroid scan is
// made of.  8 independent chains per thread, 2 CTAs x 512 threads per SM.
//   ffma    : fma.rn.f32 with three register operands
//   ffma2   : fma.rn.f32x2 (two lanes' worth per instruction)
//   fadd    : add.f32
//   imnmx   : min.u32
//   lop3    : (a & mask) | b
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fma_peak fma_peak.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

constexpr int ITERS = 8192, CH = 8;

template <int MODE>
__global__ void __launch_bounds__(512) k(float *out, float s) {
    float a[CH];
    uint32_t u[CH];
    unsigned long long p[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        a[c] = s * (threadIdx.x + c);
        u[c] = threadIdx.x * 7u + c;
        asm("mov.b64 %0, {%1,%1};" : "=l"(p[c]) : "f"(a[c]));
    }
    const float b = s * 0.999f, cc = s * 1e-3f;
    unsigned long long bb, cc2;
    asm("mov.b64 %0, {%1,%1};" : "=l"(bb) : "f"(b));
    asm("mov.b64 %0, {%1,%1};" : "=l"(cc2) : "f"(cc));
    const uint32_t m = ~0xffu, v = threadIdx.x & 0xff;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            if (MODE == 0) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[c]) : "f"(b), "f"(cc));
            if (MODE == 1)
                asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[c]) : "l"(bb), "l"(cc2));
            if (MODE == 2) asm volatile("add.f32 %0, %0, %1;" : "+f"(a[c]) : "f"(b));
            if (MODE == 3) asm volatile("min.u32 %0, %0, %1;" : "+r"(u[c]) : "r"(v + it));
            if (MODE == 4)
                asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(u[c]) : "r"(m), "r"(v));
        }
    }
    float r = 0.f;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        float x, y;
        asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(p[c]));
        r += a[c] + (float)u[c] + x + y;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = 2 * sms, threads = 512;
    float *out;
    cudaMalloc(&out, blocks * threads * 4);
    const char *names[] = {"ffma (3-reg)", "ffma2 (f32x2)", "fadd", "imnmx (min.u32)", "lop3"};
    const double per_inst[] = {2, 4, 1, 1, 1};  // flops (or ops) per lane per instruction
    void (*ks[])(float *, float) = {k<0>, k<1>, k<2>, k<3>, k<4>};
    for (int mo = 0; mo < 5; ++mo) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        ks[mo]<<<blocks, threads>>>(out, 1.0f);
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) ks[mo]<<<blocks, threads>>>(out, 1.0f + r);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double inst = 5.0 * blocks * threads * (double)ITERS * CH;  // lane-instructions
        const double s = ms * 1e-3;
        printf("%-18s %8.3f ms  %7.1f lane-inst/clk/SM (at 1.965 GHz)  %8.2f T ops/s\n", names[mo],
               ms / 5, inst / s / sms / 1.965e9, inst * per_inst[mo] / s / 1e12);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
