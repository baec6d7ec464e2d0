// capi_internal.h — shared by the engine's host translation units (capi.cu,
// host_staging.cu): the error plumbing of the guarded C-ABI calls and the
// host-side row staging.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <string>

#include "engine.h"
#include "tsom_b200.h"

namespace tsom {

// NVTX range over a host-side phase (enqueue of an epoch's steps, binds,
// refreshes); header-only NVTX 3, free when no tool is attached
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// a failed CU / REQUIRE inside a guarded call: the status it returns
struct Fail {
    int code;
};

#define CU(expr)                                                                          \
    do {                                                                                  \
        cudaError_t _e = (expr);                                                          \
        if (_e != cudaSuccess) {                                                          \
            eng->last_error = std::string("cuda: ") + cudaGetErrorString(_e) + " at " #expr; \
            throw ::tsom::Fail{TSOM_ERR_CUDA};                                            \
        }                                                                                 \
    } while (0)

#define REQUIRE(cond, code, msg)        \
    do {                                \
        if (!(cond)) {                  \
            eng->last_error = (msg);    \
            throw ::tsom::Fail{code};   \
        }                               \
    } while (0)

namespace host {

// FSOMSHRD files of a shard bind
void close_shards(Engine* eng);
// two pinned staging slots of at least `rows` rows (blocks cached process-wide)
void ensure_pinned(Engine* eng, uint64_t rows);
void pinned_give(void* p, size_t bytes);
// host pointer of rows [r0, r1) the copy engine can read (slot s when staged)
const float* host_chunk_source(Engine* eng, uint64_t r0, uint64_t r1, int s);
void note_pinned_copy(Engine* eng, int s);

}  // namespace host
}  // namespace tsom
