// Microbenchmark: how fast can one persistent CTA per SM stream a code buffer
// from HBM, as a function of the load structure?  (Design evidence for the
// decode kernel's code stream.)
//   reg<D>   : 16 warps, each lane keeps D units of 4 x 16-byte loads in a
//              static register ring (the decode kernel's structure, D = 2)
//   tma<S,B> : one producer thread fills an S-stage shared-memory ring of
//              B-byte stages with cp.async.bulk; 16 consumer warps read it
//              with 16-byte LDS and release the stage (full/empty mbarriers)
// Each kernel XOR-reduces what it reads so nothing is dead code.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_bw stream_bw.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint4 ldg_stream(const uint8_t *p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

// unit = 2048 B per warp (4 loads x 512 B); a CTA round = 16 warps x 2048 B = 32 KiB
template <int D>
__global__ void __launch_bounds__(512, 1) reg_ring(const uint8_t *buf, int64_t bytes, uint32_t *sink) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t per_cta = bytes / gridDim.x;
    const uint8_t *base = buf + per_cta * blockIdx.x + lane * 16;
    const int64_t units = per_cta / 2048;
    uint4 r[D][4];
    uint32_t acc = 0;
#pragma unroll
    for (int d = 0; d < D; ++d) {
        const int64_t u = warp + d * 16;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (u < units) r[d][k] = ldg_stream(base + u * 2048 + k * 512);
    }
    for (int64_t u = warp; u < units; u += 16 * D) {
#pragma unroll
        for (int d = 0; d < D; ++d) {
            const int64_t uu = u + d * 16;
            if (uu < units) {
#pragma unroll
                for (int k = 0; k < 4; ++k) acc ^= r[d][k].x ^ r[d][k].y ^ r[d][k].z ^ r[d][k].w;
                const int64_t un = uu + 16 * D;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (un < units) r[d][k] = ldg_stream(base + un * 2048 + k * 512);
            }
        }
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

// the decode kernel's pattern: two streams per CTA (K codes and V codes of a
// head, in different halves of the buffer); a unit = 2 x 512 B of each
template <int D>
__global__ void __launch_bounds__(512, 1) reg_ring_kv(const uint8_t *buf, int64_t bytes, uint32_t *sink) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t half = bytes / 2;
    const int64_t per_cta = half / gridDim.x;
    const uint8_t *kb = buf + per_cta * blockIdx.x + lane * 16;
    const uint8_t *vb = kb + half;
    const int64_t units = per_cta / 1024;
    uint4 r[D][4];
    uint32_t acc = 0;
#pragma unroll
    for (int d = 0; d < D; ++d) {
        const int64_t u = warp + d * 16;
        if (u < units) {
            r[d][0] = ldg_stream(kb + u * 1024); r[d][1] = ldg_stream(vb + u * 1024);
            r[d][2] = ldg_stream(kb + u * 1024 + 512); r[d][3] = ldg_stream(vb + u * 1024 + 512);
        }
    }
    for (int64_t u = warp; u < units; u += 16 * D) {
#pragma unroll
        for (int d = 0; d < D; ++d) {
            const int64_t uu = u + d * 16;
            if (uu < units) {
#pragma unroll
                for (int k = 0; k < 4; ++k) acc ^= r[d][k].x ^ r[d][k].y ^ r[d][k].z ^ r[d][k].w;
                const int64_t un = uu + 16 * D;
                if (un < units) {
                    r[d][0] = ldg_stream(kb + un * 1024); r[d][1] = ldg_stream(vb + un * 1024);
                    r[d][2] = ldg_stream(kb + un * 1024 + 512); r[d][3] = ldg_stream(vb + un * 1024 + 512);
                }
            }
        }
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

// CTA pair (2c, 2c+1) shares a chunk; rank r reads 32-byte half r of every
// 64-byte row (lane l: row l >> 1 of a 16-row group, 16 bytes at 32r + 16(l & 1))
template <int D>
__global__ void __launch_bounds__(512, 1) reg_ring_half(const uint8_t *buf, int64_t bytes, uint32_t *sink) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int r = blockIdx.x & 1;
    const int64_t per_pair = bytes / (gridDim.x / 2);
    const uint8_t *base = buf + per_pair * (blockIdx.x >> 1) + (lane >> 1) * 64 + r * 32 + (lane & 1) * 16;
    const int64_t units = per_pair / 4096;
    uint4 rr[D][4];
    uint32_t acc = 0;
#pragma unroll
    for (int d = 0; d < D; ++d) {
        const int64_t u = warp + d * 16;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (u < units) rr[d][k] = ldg_stream(base + u * 4096 + k * 1024);
    }
    for (int64_t u = warp; u < units; u += 16 * D) {
#pragma unroll
        for (int d = 0; d < D; ++d) {
            const int64_t uu = u + d * 16;
            if (uu < units) {
#pragma unroll
                for (int k = 0; k < 4; ++k) acc ^= rr[d][k].x ^ rr[d][k].y ^ rr[d][k].z ^ rr[d][k].w;
                const int64_t un = uu + 16 * D;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (un < units) rr[d][k] = ldg_stream(base + un * 4096 + k * 1024);
            }
        }
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(bar), "r"(phase) : "memory");
}

template <int S, int B>
__global__ void __launch_bounds__(544, 1) tma_ring(const uint8_t *buf, int64_t bytes, uint32_t *sink) {
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t full = sb + S * B, empty = full + 8 * S;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int64_t per_cta = bytes / gridDim.x;
    const uint8_t *src = buf + per_cta * blockIdx.x;
    const int64_t stages = per_cta / B;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(full + 8 * s, 1); mbar_init(empty + 8 * s, 16); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 16) {  // producer warp
        if ((tid & 31) == 0) {
            for (int64_t i = 0; i < stages; ++i) {
                const int s = (int)(i % S);
                if (i >= S) mbar_wait(empty + 8 * s, (uint32_t)(((i / S) - 1) & 1));
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full + 8 * s), "r"(B) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(sb + s * B), "l"(src + i * B), "r"(B), "r"(full + 8 * s) : "memory");
            }
        }
        return;
    }
    uint32_t acc = 0;
    for (int64_t i = 0; i < stages; ++i) {
        const int s = (int)(i % S);
        mbar_wait(full + 8 * s, (uint32_t)((i / S) & 1));
        for (int off = tid * 16; off < B; off += 512 * 16) {
            const uint4 v = *reinterpret_cast<const uint4 *>(smem + s * B + off);
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
        __syncwarp();
        if ((tid & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty + 8 * s) : "memory");
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

template <typename K>
static float time_it(K kern, int threads, size_t smem, const uint8_t *buf, int64_t bytes, uint32_t *sink, int sms) {
    if (smem) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int w = 0; w < 3; ++w) kern<<<sms, threads, smem>>>(buf, bytes, sink);
    const int reps = 20;
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) kern<<<sms, threads, smem>>>(buf + (r & 1) * bytes, bytes, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return ms / reps;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t bytes = (int64_t)sms * 64 * 32768 * 32;  // ~310 MB per launch (> L2), 2 buffers alternate
    uint8_t *buf; CK(cudaMalloc(&buf, 2 * bytes)); CK(cudaMemset(buf, 7, 2 * bytes));
    uint32_t *sink; CK(cudaMalloc(&sink, 4));
    auto rep = [&](const char *name, float ms) { printf("%-24s %8.1f us  %7.0f GB/s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9); };
    rep("reg_ring<1>", time_it(reg_ring<1>, 512, 0, buf, bytes, sink, sms));
    rep("reg_ring<2>", time_it(reg_ring<2>, 512, 0, buf, bytes, sink, sms));
    rep("reg_ring<3>", time_it(reg_ring<3>, 512, 0, buf, bytes, sink, sms));
    rep("reg_ring<4>", time_it(reg_ring<4>, 512, 0, buf, bytes, sink, sms));
    rep("reg_ring_kv<1>", time_it(reg_ring_kv<1>, 512, 0, buf, bytes, sink, sms));
    rep("reg_ring_kv<2>", time_it(reg_ring_kv<2>, 512, 0, buf, bytes, sink, sms));
    rep("reg_ring_half<2>", time_it(reg_ring_half<2>, 512, 0, buf, bytes, sink, sms));
    rep("reg_ring_half<4>", time_it(reg_ring_half<4>, 512, 0, buf, bytes, sink, sms));
    rep("tma<4,8K>", time_it(tma_ring<4, 8192>, 544, 4 * 8192 + 256, buf, bytes, sink, sms));
    rep("tma<4,16K>", time_it(tma_ring<4, 16384>, 544, 4 * 16384 + 256, buf, bytes, sink, sms));
    rep("tma<8,8K>", time_it(tma_ring<8, 8192>, 544, 8 * 8192 + 256, buf, bytes, sink, sms));
    rep("tma<4,32K>", time_it(tma_ring<4, 32768>, 544, 4 * 32768 + 256, buf, bytes, sink, sms));
    rep("tma<6,32K>", time_it(tma_ring<6, 32768>, 544, 6 * 32768 + 256, buf, bytes, sink, sms));
    rep("tma<2,16K>", time_it(tma_ring<2, 16384>, 544, 2 * 16384 + 256, buf, bytes, sink, sms));
    rep("tma<3,8K>", time_it(tma_ring<3, 8192>, 544, 3 * 8192 + 256, buf, bytes, sink, sms));
    return 0;
}
