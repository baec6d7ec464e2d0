// mem_pool.cu — the engines' device memory: every DevBuf comes from one
// stream-ordered caching pool per device.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

#include "engine.h"

namespace tsom {

// Device memory comes from one stream-ordered pool per device that keeps freed
// blocks cached (like torch's caching allocator): an engine created after
// another one reuses its memory instead of paying cudaMalloc/cudaFree (tens to
// hundreds of ms for GB-sized buffers).  Allocations are made on a private,
// otherwise idle stream and synchronised, so a block is usable from every
// stream on return; frees follow a device synchronisation (cudaFree's own
// semantics), so no queued work can still touch a block the pool hands out
// again.  tsom_release_cached_memory() trims the pool.
struct DevicePool {
    cudaMemPool_t pool = nullptr;
    cudaStream_t st = nullptr;
};

static std::mutex g_pool_mu;
static DevicePool g_pools[64];

static cudaError_t device_pool(DevicePool** out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lk(g_pool_mu);
    DevicePool& dp = g_pools[dev];
    if (!dp.pool) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        if ((e = cudaMemPoolCreate(&dp.pool, &props)) != cudaSuccess) return e;
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(dp.pool, cudaMemPoolAttrReleaseThreshold, &keep);
        if ((e = cudaStreamCreateWithFlags(&dp.st, cudaStreamNonBlocking)) != cudaSuccess) {
            cudaMemPoolDestroy(dp.pool);
            dp.pool = nullptr;
            return e;
        }
    }
    *out = &dp;
    return cudaSuccess;
}

void release_cached_memory() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (g_pools[dev].pool) {
        cudaStreamSynchronize(g_pools[dev].st);
        cudaMemPoolTrimTo(g_pools[dev].pool, 0);
    }
}

static bool pool_disabled() {  // TSOM_NO_POOL=1: plain cudaMalloc/cudaFree (diagnostics)
    static const bool off = [] {
        const char* v = getenv("TSOM_NO_POOL");
        return v && v[0] == '1';
    }();
    return off;
}

cudaError_t DevBuf::ensure(size_t need) {
    if (need <= bytes && p) return cudaSuccess;
    release();
    if (need == 0) return cudaSuccess;
    if (pool_disabled()) {
        cudaError_t e = cudaMalloc(&p, need);
        if (e != cudaSuccess) {
            p = nullptr;
            bytes = 0;
            return e;
        }
        bytes = need;
        owned = true;
        return cudaSuccess;
    }
    DevicePool* dp = nullptr;
    cudaError_t e = device_pool(&dp);
    if (e == cudaSuccess) {
        e = cudaMallocFromPoolAsync(&p, need, dp->pool, dp->st);
        if (e == cudaErrorMemoryAllocation) {  // cached blocks may be in the way
            cudaGetLastError();
            release_cached_memory();
            e = cudaMallocFromPoolAsync(&p, need, dp->pool, dp->st);
        }
        if (e == cudaSuccess) {
            // debug: TSOM_POISON_ALLOC=<hex byte> fills new blocks with it so a
            // kernel that relies on zeroed memory fails deterministically
            static const int poison = [] {
                const char* v = getenv("TSOM_POISON_ALLOC");
                return v && v[0] ? (int)strtol(v, nullptr, 16) : -1;
            }();
            if (poison >= 0) e = cudaMemsetAsync(p, poison & 0xFF, need, dp->st);
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(dp->st);
    }
    if (e != cudaSuccess) {
        p = nullptr;
        bytes = 0;
        return e;
    }
    bytes = need;
    owned = true;
    return cudaSuccess;
}

cudaError_t DevBuf::ensure_on(size_t need, cudaStream_t st) {
    if (need <= bytes && p) return cudaSuccess;
    if (pool_disabled()) return ensure(need);
    release_on(st);
    DevicePool* dp = nullptr;
    cudaError_t e = device_pool(&dp);
    if (e == cudaSuccess) e = cudaMallocFromPoolAsync(&p, need, dp->pool, st);
    if (e == cudaErrorMemoryAllocation) {  // cached blocks may be in the way
        cudaGetLastError();
        release_cached_memory();
        e = cudaMallocFromPoolAsync(&p, need, dp->pool, st);
    }
    if (e != cudaSuccess) {
        p = nullptr;
        bytes = 0;
        return e;
    }
    bytes = need;
    owned = true;
    return cudaSuccess;
}

void DevBuf::release_on(cudaStream_t st) {
    if (p && owned) {
        if (pool_disabled()) {
            cudaStreamSynchronize(st);
            cudaFree(p);
        } else {
            cudaFreeAsync(p, st);
        }
    }
    p = nullptr;
    bytes = 0;
    owned = true;
}

void DevBuf::release(bool synced) {
    if (p && owned) {
        DevicePool* dp = nullptr;
        if (pool_disabled()) {
            cudaFree(p);
        } else {
            if (!synced) cudaDeviceSynchronize();
            if (device_pool(&dp) == cudaSuccess) cudaFreeAsync(p, dp->st);
        }
    }
    p = nullptr;
    bytes = 0;
    owned = true;
}

// Kernel attributes are per device (context): one cache entry per
// (kernel, device), so a second engine on another GPU of the same process
// sets them for its own device too.
cudaError_t ensure_smem_attr(const void* func, size_t bytes, bool* newly_set) {
    if (newly_set) *newly_set = false;
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    size_t& have = done[{func, dev}];
    if (have >= bytes) return cudaSuccess;
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) {
        have = bytes;
        if (newly_set) *newly_set = true;
    }
    return e;
}

}  // namespace tsom
