// Microbenchmark behind the value-path design (K2): the paper's
// per-(subspace, centroid) shared-memory bins vs this kernel's register
// gather.  One persistent 512-thread CTA per SM; every lane touches a distinct
// subspace (bank) per step, as the decode layout guarantees, with random
// codes.  Per value code:
//   bins_f32  : atomicAdd(float) into bins[i][code]  (sm_100: LDS + ATOMS.CAST.SPIN loop)
//   bins_u32  : atomicAdd(uint32) fixed point        (native ATOMS.ADD)
//   gather64  : acc += p * C_V[i][code] (LDS.64 + FFMA2), the decode kernel
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bins_vs_gather bins_vs_gather.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

constexpr int ITERS = 4096;

__device__ __forceinline__ uint32_t hash(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(float *out, uint32_t seed) {
    extern __shared__ __align__(16) unsigned char sm[];
    float *bins = reinterpret_cast<float *>(sm);             // [32][256] (one half-table)
    uint32_t *ubins = reinterpret_cast<uint32_t *>(sm);
    float2 *cv = reinterpret_cast<float2 *>(sm + 32 * 256 * 4);  // [256][32] float2
    for (int i = threadIdx.x; i < 32 * 256; i += blockDim.x) { bins[i] = 0.f; cv[i] = make_float2(i, -i); }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    uint32_t h = hash(seed ^ (blockIdx.x * 512 + threadIdx.x));
    float p = 1e-3f * (lane + 1);
    float2 acc = make_float2(0.f, 0.f);
    for (int it = 0; it < ITERS; ++it) {
        h = hash(h);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t code = (h >> (8 * j)) & 255;
            const int i = (lane + j) & 31;  // distinct subspace per lane
            if (MODE == 0) atomicAdd(&bins[i * 256 + code], p);
            if (MODE == 1) atomicAdd(&ubins[i * 256 + code], 1234u);
            if (MODE == 2) {
                const float2 c = cv[code * 32 + i];
                acc.x = fmaf(p, c.x, acc.x);
                acc.y = fmaf(p, c.y, acc.y);
            }
        }
    }
    __syncthreads();
    if (MODE == 2) out[blockIdx.x * 512 + threadIdx.x] = acc.x + acc.y;
    else if (threadIdx.x == 0) out[blockIdx.x] = bins[threadIdx.x];
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out; cudaMalloc(&out, sms * 512 * 4);
    const size_t smem = 32 * 256 * 4 + 32 * 256 * 8;
    const char *names[] = {"bins_f32 (atomicAdd float)", "bins_u32 (fixed-point atomicAdd)", "gather64 (LDS.64 + FMA)"};
    void (*ks[])(float *, uint32_t) = {k<0>, k<1>, k<2>};
    for (int m = 0; m < 3; ++m) {
        cudaFuncSetAttribute(ks[m], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        ks[m]<<<sms, 512, smem>>>(out, 1);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) ks[m]<<<sms, 512, smem>>>(out, r + 2);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        const double codes = 5.0 * sms * 512.0 * ITERS * 4;
        printf("%-34s %8.3f ms  %7.2f G codes/s  %6.2f codes/clk/SM (at 1.965 GHz)\n", names[m], ms / 5,
               codes / (ms * 1e-3) / 1e9, codes / (ms * 1e-3) / sms / 1.965e9);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
