// Paged code store: virtually contiguous, physically paged device memory for
// the growing PQ code stores (LayerKVCache, ServingCache).
//
// The reference grows a head's code store by doubling and copying
// (kv_cache.py:74-76, 217-228).  Here a store is one reservation of virtual
// address space split into equal regions (one per (layer, sequence, KV head,
// kind) stream of code rows); growth maps more physical pages at the end of
// every region (cuMemCreate + cuMemMap through the CUDA VMM API), so rows
// never move and the decode kernel keeps reading each head's codes as one
// contiguous run -- the GPU's page tables are the store's page table, and
// nothing on the hot path indirects through a software one.  Physical pages
// come in the allocation granularity (2 MiB on B200: 32 Ki rows of 64 B).
//
// The driver entry points are resolved through cudaGetDriverEntryPoint, so
// the library does not link libcuda (and still loads on a host without a
// driver, as the CPU test suite needs).
#include <cuda.h>
#include <cuda_runtime.h>

#include <vector>

#include "common.cuh"

namespace pqkv {
namespace {

struct Driver {
    CUresult (*get_granularity)(size_t *, const CUmemAllocationProp *,
                                CUmemAllocationGranularity_flags) = nullptr;
    CUresult (*reserve)(CUdeviceptr *, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
    CUresult (*address_free)(CUdeviceptr, size_t) = nullptr;
    CUresult (*create)(CUmemGenericAllocationHandle *, size_t, const CUmemAllocationProp *,
                       unsigned long long) = nullptr;
    CUresult (*release)(CUmemGenericAllocationHandle) = nullptr;
    CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle,
                    unsigned long long) = nullptr;
    CUresult (*unmap)(CUdeviceptr, size_t) = nullptr;
    CUresult (*set_access)(CUdeviceptr, size_t, const CUmemAccessDesc *, size_t) = nullptr;
    bool ok = false;
};

template <typename F>
bool entry(const char *name, F *fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || p == nullptr)
        return false;
    *fn = reinterpret_cast<F>(p);
    return true;
}

const Driver &driver() {
    static Driver d = [] {
        Driver x;
        x.ok = entry("cuMemGetAllocationGranularity", &x.get_granularity) &&
               entry("cuMemAddressReserve", &x.reserve) &&
               entry("cuMemAddressFree", &x.address_free) && entry("cuMemCreate", &x.create) &&
               entry("cuMemRelease", &x.release) && entry("cuMemMap", &x.map) &&
               entry("cuMemUnmap", &x.unmap) && entry("cuMemSetAccess", &x.set_access);
        return x;
    }();
    return d;
}

CUmemAllocationProp device_prop(int dev) {
    CUmemAllocationProp p = {};
    p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    p.location.id = dev;
    return p;
}

}  // namespace
}  // namespace pqkv

using namespace pqkv;

struct pqkv_vstore {
    int device;
    CUdeviceptr base;
    int64_t n_regions, region_bytes, granularity;
    int64_t mapped;  // bytes mapped at the start of every region
    struct Piece {
        CUdeviceptr va;
        size_t bytes;
        CUmemGenericAllocationHandle h;
    };
    std::vector<Piece> pieces;
};

static int drv_fail(const char *what, CUresult r) {
    return fail(PQKV_ECUDA, "%s failed (CUresult %d)", what, (int)r);
}

extern "C" int64_t pqkv_vstore_granularity(int device) {
    const Driver &d = driver();
    if (!d.ok) return -1;
    CUmemAllocationProp p = device_prop(device);
    size_t g = 0;
    if (d.get_granularity(&g, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS) return -1;
    return (int64_t)g;
}

extern "C" int pqkv_vstore_create(int device, int64_t n_regions, int64_t region_bytes,
                                  pqkv_vstore **out, void **base) {
    PQKV_CHECK_ARG(out && base && n_regions > 0 && region_bytes > 0,
                   "pqkv_vstore_create: bad arguments");
    const Driver &d = driver();
    if (!d.ok) return fail(PQKV_ECUDA, "pqkv_vstore_create: CUDA VMM entry points unavailable");
    const int64_t g = pqkv_vstore_granularity(device);
    if (g <= 0) return fail(PQKV_ECUDA, "pqkv_vstore_create: no allocation granularity");
    const int64_t rb = (region_bytes + g - 1) / g * g;
    PQKV_CHECK_ARG(rb <= ((int64_t)1 << 46) / n_regions, "pqkv_vstore_create: reservation too large");
    CUdeviceptr va = 0;
    CUresult r = d.reserve(&va, (size_t)(rb * n_regions), (size_t)g, 0, 0);
    if (r != CUDA_SUCCESS) return drv_fail("cuMemAddressReserve", r);
    pqkv_vstore *vs = new pqkv_vstore{device, va, n_regions, rb, g, 0, {}};
    *out = vs;
    *base = reinterpret_cast<void *>(va);
    return PQKV_OK;
}

// Map pages so that every region holds at least `bytes` mapped bytes (grown
// geometrically, at most to the region size); mapped pages never move.
extern "C" int pqkv_vstore_ensure(pqkv_vstore *vs, int64_t bytes) {
    PQKV_CHECK_ARG(vs != nullptr && bytes >= 0, "pqkv_vstore_ensure: bad arguments");
    if (bytes <= vs->mapped) return PQKV_OK;
    PQKV_CHECK_ARG(bytes <= vs->region_bytes,
                   "pqkv_vstore_ensure: %lld bytes exceed the region's reservation (%lld)",
                   (long long)bytes, (long long)vs->region_bytes);
    const Driver &d = driver();
    const int64_t g = vs->granularity;
    int64_t want = bytes > 2 * vs->mapped ? bytes : 2 * vs->mapped;
    want = (want + g - 1) / g * g;
    if (want > vs->region_bytes) want = vs->region_bytes;
    const size_t grow = (size_t)(want - vs->mapped);
    CUmemAllocationProp p = device_prop(vs->device);
    CUmemAccessDesc acc = {};
    acc.location = p.location;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    for (int64_t r = 0; r < vs->n_regions; ++r) {
        CUdeviceptr va = vs->base + (CUdeviceptr)(r * vs->region_bytes + vs->mapped);
        CUmemGenericAllocationHandle h;
        CUresult e = d.create(&h, grow, &p, 0);
        if (e != CUDA_SUCCESS) return drv_fail("cuMemCreate", e);
        e = d.map(va, grow, 0, h, 0);
        if (e != CUDA_SUCCESS) {
            d.release(h);
            return drv_fail("cuMemMap", e);
        }
        vs->pieces.push_back({va, grow, h});
        e = d.set_access(va, grow, &acc, 1);
        if (e != CUDA_SUCCESS) return drv_fail("cuMemSetAccess", e);
    }
    vs->mapped = want;
    return PQKV_OK;
}

extern "C" int64_t pqkv_vstore_mapped(const pqkv_vstore *vs) { return vs ? vs->mapped : -1; }
extern "C" int64_t pqkv_vstore_region_bytes(const pqkv_vstore *vs) {
    return vs ? vs->region_bytes : -1;
}

extern "C" int pqkv_vstore_destroy(pqkv_vstore *vs) {
    if (vs == nullptr) return PQKV_OK;
    const Driver &d = driver();
    int rc = PQKV_OK;
    int cur = 0;  // no kernel may still read the pages
    cudaGetDevice(&cur);
    cudaSetDevice(vs->device);
    cudaDeviceSynchronize();
    cudaSetDevice(cur);
    for (auto &pc : vs->pieces) {
        if (d.unmap(pc.va, pc.bytes) != CUDA_SUCCESS) rc = PQKV_ECUDA;
        if (d.release(pc.h) != CUDA_SUCCESS) rc = PQKV_ECUDA;
    }
    if (d.address_free(vs->base, (size_t)(vs->region_bytes * vs->n_regions)) != CUDA_SUCCESS)
        rc = PQKV_ECUDA;
    delete vs;
    return rc == PQKV_OK ? rc : fail(rc, "pqkv_vstore_destroy: unmap/release failed");
}
