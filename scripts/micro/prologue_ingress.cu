// Microbenchmark: time for every SM (1 CTA x 512 threads each) to pull the
// decode prologue's tables into the SM -- 128 KiB by TMA bulk copy and/or
// 128 KiB by per-thread 16-byte loads -- from a buffer that all CTAs share
// (the L2 hot-spot pattern of the value / key codebooks).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__global__ void __launch_bounds__(512, 1) k(const char *src, int mode, int nchunks, unsigned long long *t, float *sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm);
    uint32_t bar = sb + 200 * 1024;
    unsigned long long t0 = gtime();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if ((mode & 1) && threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(nchunks * 16384) : "memory");
        for (int c = 0; c < nchunks; ++c)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];"
                         ::"r"(sb + c * 16384), "l"(src + c * 16384), "r"(bar) : "memory");
    }
    float acc = 0.f;
    if (mode & 2) {
        const float4 *s4 = reinterpret_cast<const float4 *>(src + (mode & 4 ? 0 : 131072));
        float4 v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = __ldg(s4 + threadIdx.x + i * 512);
#pragma unroll
        for (int i = 0; i < 16; ++i) acc += v[i].x + v[i].y + v[i].z + v[i].w;
    }
    if (mode & 1) {
        asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(bar) : "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) { t[blockIdx.x * 2] = t0; t[blockIdx.x * 2 + 1] = gtime(); }
    if (acc == 12345.f) sink[0] = acc;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    char *src; cudaMalloc(&src, 1 << 20); cudaMemset(src, 1, 1 << 20);
    unsigned long long *t; cudaMalloc(&t, sms * 16); float *sink; cudaMalloc(&sink, 4);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 201 * 1024);
    unsigned long long *h = new unsigned long long[sms * 2];
    const char *names[] = {"", "TMA 128K", "LDG 128K", "TMA 128K + LDG 128K (other)", "", "", "", ""};
    for (int mode : {1, 2, 3, 1, 3}) {
        for (int ctas : {sms, 1}) {
            for (int rep = 0; rep < 3; ++rep) k<<<ctas, 512, 201 * 1024>>>(src, mode, 8, t, sink);
            cudaDeviceSynchronize();
            cudaMemcpy(h, t, ctas * 16, cudaMemcpyDeviceToHost);
            unsigned long long mn = ~0ull, mx = 0, sum = 0;
            for (int i = 0; i < ctas; ++i) { unsigned long long d = h[2*i+1] - h[2*i]; mn = d < mn ? d : mn; mx = d > mx ? d : mx; sum += d; }
            printf("%-30s ctas=%3d  per-CTA us: min %.2f avg %.2f max %.2f\n", names[mode], ctas, mn / 1e3, sum / 1e3 / ctas, mx / 1e3);
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
