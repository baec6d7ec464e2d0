// capi.cu — the tsom_* C-ABI (include/tsom_b200.h) over the B200 kernels.
//
// One engine = one GPU = one training run.  Every call is synchronous from the
// caller's point of view (it returns after its results are in the caller's
// buffers), all device work is issued on the engine stream.  There is no CPU
// fallback: if a kernel cannot run, the call fails with TSOM_ERR_CUDA.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <fcntl.h>
#include <thread>
#include <unistd.h>
#include <nccl.h>

#include <condition_variable>
#include <chrono>
#include <mutex>
#include <functional>
#include <memory>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "capi_internal.h"
#include "engine.h"
#include "mt_jump.h"

using tsom::DevBuf;
using tsom::Engine;

struct tsom_engine : public Engine {};

namespace tsom {

std::atomic<uint64_t> g_launches{0};

}  // namespace tsom

namespace {

using tsom::host::close_shards;
using tsom::host::ensure_pinned;
using tsom::host::host_chunk_source;
using tsom::host::note_pinned_copy;
using tsom::host::pinned_give;

const char* kVersion = "toposom-b200 0.2 (sm_100a; tcgen05 3xFP16 BMU with exact FP64 near-tie resolution, TMA row gathers)";

template <typename F>
int guarded(Engine* eng, F&& f) {
    if (!eng) return TSOM_ERR_INVALID;
    try {
        f();
        return TSOM_OK;
    } catch (const tsom::Fail& fl) {
        return fl.code;
    } catch (const std::exception& ex) {
        eng->last_error = ex.what();
        return TSOM_ERR_INVALID;
    }
}

// ---- NCCL, loaded lazily (single-GPU use never needs it) -------------------
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*commInitRankConfig)(ncclComm_t*, int, ncclUniqueId, int, ncclConfig_t*) = nullptr;
    ncclResult_t (*getAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*commAbort)(ncclComm_t) = nullptr;
    const char* (*errStr)(ncclResult_t) = nullptr;
    bool load(std::string& err) {
        if (h) return true;
        // a NCCL the process already loaded (e.g. by torch) first, then
        // TSOM_NCCL_LIB (the Python binding points it at the NCCL wheel torch
        // links against), then the loader's search path: two different
        // libnccl.so.2 in one process would break whichever loads second
        h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        const char* env = getenv("TSOM_NCCL_LIB");
        if (!h && env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* n : names)
            if (!h && (h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
        if (!h) {
            err = std::string("nccl: cannot load libnccl.so.2: ") + dlerror();
            return false;
        }
        getUniqueId = (decltype(getUniqueId))dlsym(h, "ncclGetUniqueId");
        commInitRank = (decltype(commInitRank))dlsym(h, "ncclCommInitRank");
        allReduce = (decltype(allReduce))dlsym(h, "ncclAllReduce");
        commDestroy = (decltype(commDestroy))dlsym(h, "ncclCommDestroy");
        errStr = (decltype(errStr))dlsym(h, "ncclGetErrorString");
        commInitRankConfig = (decltype(commInitRankConfig))dlsym(h, "ncclCommInitRankConfig");
        getAsyncError = (decltype(getAsyncError))dlsym(h, "ncclCommGetAsyncError");
        commAbort = (decltype(commAbort))dlsym(h, "ncclCommAbort");
        if (!getUniqueId || !commInitRank || !allReduce || !commDestroy || !commInitRankConfig ||
            !getAsyncError || !commAbort) {
            err = "nccl: missing symbols";
            return false;
        }
        return true;
    }
};
NcclApi g_nccl;

size_t slot_len(const Engine* e) { return (size_t)e->P * e->D + e->P + 2; }

uint32_t ppad(const Engine* e) { return (e->P + 63) / 64 * 64; }

// Tensor-core operand encoding for this engine: option 2 = 3xTF32, 3 = 3xFP16,
// 0 (auto) = 3xFP16 when d fits (d <= 62), else 3xTF32 (d <= 53), else SIMT.
int tc_kind(const Engine* e) {
    if (e->bmu_kernel == 1) return tsom::kTcNone;
    if (e->bmu_kernel == 2) return tsom::kTcTf32;
    if (e->bmu_kernel == 3) return tsom::kTcF16;
    if (tsom::tc_supported(tsom::kTcF16, e->P, e->D)) return tsom::kTcF16;
    if (tsom::tc_supported(tsom::kTcTf32, e->P, e->D)) return tsom::kTcTf32;
    return tsom::kTcNone;
}

tsom::TieWin tie_window(const Engine* e, int kind) {
    tsom::TieWin w;
    w.tau = (float)e->tau_tc;
    w.abs_coef = kind == tsom::kTcF16 ? (float)(std::ldexp(1.0, -24) * std::sqrt((double)e->D)) : 0.0f;
    w.quant = 0.0f;  // raw (unpacked) values in every K1 epilogue
    return w;
}

// per-row scratch of a pass over n rows (distances only when asked for)
void ensure_rows(Engine* eng, uint64_t n, bool want_dist = false) {
    CU(eng->bmu.ensure(std::max<uint64_t>(n, 1) * sizeof(uint32_t)));
    if (want_dist) CU(eng->dist.ensure(std::max<uint64_t>(n, 1) * sizeof(double)));
    CU(eng->flags.ensure((std::max<uint64_t>(n, 1) + 2) * sizeof(uint32_t)));
}

void prep_codebook(Engine* eng) {
    REQUIRE(eng->codebook_set, TSOM_ERR_INVALID, "engine: codebook not set (tsom_set_codebook)");
    if (eng->codebook_prepped) return;
    tsom::launch_prep_codebook(eng->w.as<float>(), eng->P, eng->D, eng->w2.as<double>(),
                               eng->w2max.as<float>(), eng->wt.as<float>(), ppad(eng), eng->stream);
    CU(cudaGetLastError());
    eng->codebook_prepped = true;
}

// the K1 main-pass events of the current epoch (per-epoch pairs during
// tsom_train_epochs, else ev[8] / ev[9])
cudaEvent_t k1_event(Engine* eng, int end) {
    if (eng->k1_slot >= 0) return eng->k1_ev[2 * (size_t)eng->k1_slot + end];
    return eng->ev[8 + end];
}

constexpr uint32_t kTieLogCap = 1024;  // tie_log entries between two syncs

// An engine's pinned host words (hstat: 32 status words, then tie_log) come
// from a process-wide cache: cudaMallocHost / cudaFreeHost cost milliseconds
// per call (a third of an engine's creation), and studies create many engines.
constexpr size_t kHostWords = 32 + 2 * kTieLogCap;
std::mutex g_host_words_mu;
std::vector<uint32_t*> g_host_words_free;

cudaError_t host_words_take(uint32_t** out) {
    {
        std::lock_guard<std::mutex> lk(g_host_words_mu);
        if (!g_host_words_free.empty()) {
            *out = g_host_words_free.back();
            g_host_words_free.pop_back();
            return cudaSuccess;
        }
    }
    return cudaMallocHost(reinterpret_cast<void**>(out), kHostWords * sizeof(uint32_t));
}

void host_words_give(uint32_t* p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_host_words_mu);
    g_host_words_free.push_back(p);
}

// the near-tie fractions logged since the last sync (called after it)
void fold_tie_log(Engine* eng) {
    if (eng->tie_log_n == 0) return;
    std::vector<uint32_t> cnt(eng->tie_log_n);
    if (cudaMemcpy(cnt.data(), eng->tie_dev.p, cnt.size() * sizeof(uint32_t),
                   cudaMemcpyDeviceToHost) != cudaSuccess) {
        cudaGetLastError();
        eng->tie_log_n = 0;
        return;
    }
    for (uint32_t i = 0; i < eng->tie_log_n; ++i) eng->tie_log[2 * i] = cnt[i];
    for (uint32_t i = 0; i < eng->tie_log_n; ++i)
        if (eng->tie_log[2 * i + 1])
            eng->tie_frac_max = std::max(eng->tie_frac_max, (double)eng->tie_log[2 * i] /
                                                                (double)eng->tie_log[2 * i + 1]);
    eng->tie_log_n = 0;
}

// near-tie list passes: pcount[p] = clamp(count - p * cap, 0, cap); the last
// pass keeps the whole remainder (its slots past cap take the full re-scan)
constexpr uint32_t kTiePasses = 4;
constexpr uint32_t kTieCapDiv = 16;  // enumerate scratch: n / 16 rows (4 passes cover 25 %)
__global__ void k_tie_pass_counts(const uint32_t* __restrict__ count, uint64_t cap,
                                  uint32_t passes, uint32_t* __restrict__ pcount,
                                  uint32_t* __restrict__ log_slot) {
    const uint32_t p = threadIdx.x;
    if (p == 0 && log_slot) *log_slot = *count;  // the near-tie count, for later pass sizing
    if (p >= passes) return;
    const uint64_t c = *count, o = (uint64_t)p * cap;
    const uint64_t rest = c <= o ? 0 : c - o;
    pcount[p] = (uint32_t)(p + 1 == passes ? rest : (rest < cap ? rest : cap));
}

// ids[i] = sel[pos[i]] (pos null: i) for i < count (count = *dev_n when given),
// and their window terms from the split image
__global__ void k_gather_ids(const uint32_t* __restrict__ sel, const uint32_t* __restrict__ pos,
                             const uint32_t* __restrict__ dev_n, uint64_t n_host,
                             const float* __restrict__ img_xn2, uint32_t* __restrict__ ids,
                             float* __restrict__ xn2) {
    const uint64_t n = dev_n ? min((uint64_t)*dev_n, n_host) : n_host;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = sel[pos ? pos[i] : i];
        ids[i] = r;
        xn2[i] = img_xn2[r];
    }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            return (EncodeTiledFn) nullptr;
        }
        return reinterpret_cast<EncodeTiledFn>(f);
    }();
    return fn;
}

// Use (and if needed build) the split image for a 3xFP16 pass over the
// selection `sel` (n rows) of the resident rows: false = pre-split tiles as
// before (streamed or caller rows, small selections, image off or no room).
bool use_image(Engine* eng, const float* x, const uint32_t* sel, uint64_t n, int kind) {
    if (!sel || kind != tsom::kTcF16 || !eng->img_mode || eng->streamed || !eng->x.p ||
        x != eng->x.as<float>() || n * 64 < eng->n_rows || !encode_tiled())
        return false;
    if (eng->img_valid) return true;
    const tsom::TcGeom geo = tsom::tc_geom(kind, eng->D);
    const uint32_t w = (geo.kpad + 63u) / 64u * 64u;
    if (eng->ximg.ensure(eng->n_rows * w * 2) != cudaSuccess ||
        eng->ximg_xn2.ensure(eng->n_rows * sizeof(float)) != cudaSuccess) {
        cudaGetLastError();
        eng->ximg.release();
        eng->ximg_xn2.release();
        eng->img_mode = 0;  // no room next to the rows: the per-pass split stays
        return false;
    }
    tsom::launch_split_image(eng->x.as<float>(), eng->ldx, eng->n_rows, eng->D,
                             eng->scale.as<float>(), tie_window(eng, kind), eng->ximg.p, w,
                             eng->ximg_xn2.as<float>(), eng->stream);
    CU(cudaGetLastError());
    cuuint64_t gdim[2] = {(cuuint64_t)w, (cuuint64_t)eng->n_rows};
    cuuint64_t gstr[1] = {(cuuint64_t)w * 2};
    cuuint32_t box[2] = {64, 1};  // tile::gather4: one row per coordinate, a 128-B atom wide
    cuuint32_t es[2] = {1, 1};
    const CUresult cr = encode_tiled()(&eng->img_map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2,
                                       eng->ximg.p, gdim, gstr, box, es,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    REQUIRE(cr == CUDA_SUCCESS, TSOM_ERR_CUDA, "cuTensorMapEncodeTiled failed for the split image");
    eng->img_w = w;
    eng->img_valid = true;
    return true;
}

// K1 + exact re-check over rows `x` (selection `sel` of length n, or first n rows).
// x2max: max ||x||^2 over these rows (device; picks the FP16 operand scale).
// `tiles` = pre-split tcgen05 A tiles for exactly these n rows, built with the
// scale of this same x2max (or nullptr to build them here).
// skip: the rows are the BMU-ordered bound rows (K1's chunk-skipping epilogue).
void run_bmu(Engine* eng, const float* x, uint32_t ldx, const uint32_t* sel, uint64_t n,
             const float* x2max, const void* tiles, const float* tiles_xn2, bool skip = false) {
    tsom::NvtxRange nv("tsom.bmu");
    const float* xsrc = x;
    const int kind = tc_kind(eng);
    if (n == 0 || kind == tsom::kTcNone)
        CU(cudaMemsetAsync(eng->flags.p, 0, 2 * sizeof(uint32_t), eng->stream));
    if (n == 0) return;
    if (kind != tsom::kTcNone) {
        const tsom::TcGeom geo = tsom::tc_geom(kind, eng->D);
        const uint32_t gn = tsom::tc_group_width(eng->P);
        const uint32_t groups = (eng->P + gn - 1) / gn;
        const float* scale = eng->scale.as<float>();
        const tsom::TieWin win = tie_window(eng, kind);
        CU(eng->ties.ensure((n + 1) * sizeof(uint32_t)));
        CU(eng->tcls.ensure(2 * tsom::kTieClasses * sizeof(uint32_t)));
        // operand scale + codebook B operand for these rows (a few microseconds);
        // the re-check counters, the near-tie count and its class counters
        // start at zero
        tsom::launch_set_scale(kind, x2max, eng->scale.as<float>(), eng->stream,
                               eng->flags.as<uint32_t>(), 2, eng->ties.as<uint32_t>(),
                               eng->tcls.as<uint32_t>(), 2 * tsom::kTieClasses);
        CU(eng->wsplit.ensure(tsom::tc_wsplit_bytes(kind, eng->P, eng->D)));
        tsom::launch_prep_wsplit(kind, eng->w.as<float>(), eng->P, eng->D, scale, eng->wsplit.p,
                                 eng->stream);
        // selections of the resident rows: K1 gathers them from the split image
        const bool img = !tiles && use_image(eng, x, sel, n, kind);
        const CUtensorMap* tmap = img ? &eng->img_map : nullptr;
        if (img) {
            CU(eng->gxn2.ensure(n * sizeof(float)));
            CU(eng->gid.ensure(2 * n * sizeof(uint32_t)));  // [selection ids | near-tie ids]
            TSOM_LAUNCH(k_gather_ids<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 16), 256,
                                       0, eng->stream>>>(sel, nullptr, nullptr, n,
                                                         eng->ximg_xn2.as<float>(),
                                                         eng->gid.as<uint32_t>(),
                                                         eng->gxn2.as<float>()));
            tiles_xn2 = eng->gxn2.as<float>();
        } else if (!tiles) {
            const uint64_t ntiles = (n + tsom::kTcTileM - 1) / tsom::kTcTileM;
            CU(eng->gsplit.ensure(ntiles * geo.tile_bytes));
            CU(eng->gxn2.ensure(n * sizeof(float)));
            tsom::launch_split_rows(kind, xsrc, sel, nullptr, n, eng->D, scale, win,
                                    eng->gsplit.p, eng->gxn2.as<float>(), eng->stream, nullptr,
                                    ldx);
            tiles = eng->gsplit.p;
            tiles_xn2 = eng->gxn2.as<float>();
        }
        CU(eng->part.ensure((size_t)groups * 2 * n * sizeof(float)));
        CU(eng->tmask.ensure(std::max<uint64_t>(n, 1) * sizeof(uint32_t)));
        const float* w2 = eng->w2max.as<float>();
        CU(cudaEventRecord(k1_event(eng, 0), eng->stream));
        CU(tsom::launch_bmu_tc(kind, tiles, n, nullptr, false, eng->P, eng->D, eng->wsplit.p,
                               tiles_xn2, w2, scale, win, nullptr, eng->part.as<float>(),
                               eng->sm_count, eng->smem_optin, eng->stream, nullptr, skip, tmap,
                               img ? eng->gid.as<uint32_t>() : nullptr));
        CU(cudaEventRecord(k1_event(eng, 1), eng->stream));
        eng->k1_timed = true;
        tsom::sampler_pregenerate(eng->sampler, k1_event(eng, 1));
        // (the near-tie list's group classes are counted by the merge, and the
        // class-sorted list's tile masks zeroed there: k_tie_classes below)
        const uint64_t ntl = (n + tsom::kTcTileM - 1) / tsom::kTcTileM;
        CU(eng->tsort.ensure((2 * (size_t)n + 1 + ntl + 8) * sizeof(uint32_t)));
        uint32_t* ties_s = eng->tsort.as<uint32_t>();
        uint32_t* tmask_s = ties_s + n + 1;
        uint32_t* tile_mask = tmask_s + n;
        const bool classed = tsom::launch_merge_fast(
            eng->part.as<float>(), n, groups, 1, gn, tiles_xn2, w2, scale, win,
            eng->bmu.as<uint32_t>(), eng->ties.as<uint32_t>(), eng->tmask.as<uint32_t>(),
            eng->flags.as<uint32_t>(), eng->stream, eng->tcls.as<uint32_t>(), tile_mask);
        CU(cudaGetLastError());
        uint32_t* log_slot = nullptr;  // the count goes to a device log, read after the sync
        if (eng->tie_log_n < kTieLogCap) {
            eng->tie_log[2 * eng->tie_log_n + 1] = (uint32_t)std::min<uint64_t>(n, UINT32_MAX);
            log_slot = eng->tie_dev.as<uint32_t>() + eng->tie_log_n++;
        }
        // near-tie rows (~1-3%): same tensor-core kernel in enumerate mode on just
        // those rows, then exact FP64 over their few candidates.  The list length
        // stays on the device (kernels grid-stride over it), so the epoch needs
        // no host round trip; rows with > 8 candidates in a group get the full
        // exact re-scan.  A collapsed map (large sigma, early epochs) can put a
        // large share of the rows in the window (measured up to 18 %), so the
        // list is worked through in kTiePasses passes of `cap` slots each: the
        // enumerate scratch is bounded at n / 16 rows, pass p
        // reads its slot count on the device, passes past the actual count
        // exit at once, and slots past 4 cap (> 25 % of the rows) take the
        // full exact re-scan.
        // passes launched: all kTiePasses until near-ties have been observed,
        // then enough for 1.25 x the largest fraction seen so far (at least
        // one).  An empty pass still costs three launches (~12 us), and a
        // count past the last pass only costs time (its overflow takes the
        // exact re-scan), not correctness.
        uint32_t passes = n > (1u << 20) ? kTiePasses : 1u;
        // (a multiple of the tile: pass p starts at tile p cap / 128 of the list)
        const uint64_t cap = passes > 1
            ? ((n + kTieCapDiv - 1) / kTieCapDiv + tsom::kTcTileM - 1) / tsom::kTcTileM * tsom::kTcTileM
            : n;
        if (passes > 1 && eng->tie_frac_max >= 0.0) {
            const double need = 1.25 * eng->tie_frac_max * (double)n / (double)cap;
            passes = std::min<uint32_t>(kTiePasses, std::max<uint32_t>(1u, (uint32_t)std::ceil(need)));
        }
        const uint64_t mt = (cap + tsom::kTcTileM - 1) / tsom::kTcTileM;
        if (!img) CU(eng->tsplit.ensure(mt * geo.tile_bytes));
        CU(eng->part2.ensure((size_t)groups * 4 * cap * sizeof(float)));
        CU(eng->txn2.ensure(cap * sizeof(float)));
        CU(eng->tcnt.ensure(kTiePasses * sizeof(uint32_t)));
        // the near-tie list re-ordered by the groups its rows need (k_bmu.cu:
        // k_tie_classes): the enumerate pass's tiles then each need few groups,
        // and the CTAs of a group skip the tiles holding none of its rows
        if (classed)
            tsom::launch_tie_classes(eng->ties.as<uint32_t>(), eng->tmask.as<uint32_t>(), n,
                                     eng->tcls.as<uint32_t>(), ties_s, tmask_s, tile_mask,
                                     eng->stream);
        else {  // (the per-row merge: the list as it is, every group every tile)
            ties_s = eng->ties.as<uint32_t>();
            tmask_s = eng->tmask.as<uint32_t>();
            tile_mask = nullptr;
        }
        const uint32_t* tcount = ties_s;
        const uint32_t* tpos = tcount + 1;
        uint32_t* pcount = eng->tcnt.as<uint32_t>();
        TSOM_LAUNCH(k_tie_pass_counts<<<1, 32, 0, eng->stream>>>(tcount, cap, passes, pcount,
                                                                  log_slot));
        for (uint32_t pz = 0; pz < passes; ++pz) {
            const uint64_t o = (uint64_t)pz * cap;
            // the pass's rows: split into tiles, or (image) their ids
            uint32_t* tid = img ? eng->gid.as<uint32_t>() + n : nullptr;
            if (img)
                TSOM_LAUNCH(k_gather_ids<<<(unsigned)std::min<uint64_t>((cap + 255) / 256, 148 * 8),
                                           256, 0, eng->stream>>>(
                    sel, tpos + o, pcount + pz, cap, eng->ximg_xn2.as<float>(), tid,
                    eng->txn2.as<float>()));
            else
                tsom::launch_split_rows(kind, xsrc, sel, tpos + o, cap, eng->D, scale, win,
                                        eng->tsplit.p, eng->txn2.as<float>(), eng->stream,
                                        pcount + pz, ldx);
            CU(tsom::launch_bmu_tc(kind, img ? nullptr : eng->tsplit.p, cap, pcount + pz, true,
                                   eng->P, eng->D, eng->wsplit.p, eng->txn2.as<float>(), w2, scale,
                                   win, tmask_s + o, eng->part2.as<float>(), eng->sm_count,
                                   eng->smem_optin, eng->stream,
                                   tile_mask ? tile_mask + o / tsom::kTcTileM : nullptr, false,
                                   tmap, tid));
            tsom::launch_merge_partials(eng->part2.as<float>(), tpos + o, pcount + pz, cap, cap,
                                        groups, gn, eng->txn2.as<float>(), w2, scale, win, x, ldx,
                                        sel, eng->w.as<float>(), eng->D, eng->bmu.as<uint32_t>(),
                                        eng->flags.as<uint32_t>(), eng->stream, tmask_s + o);
        }
    } else {
        CU(cudaEventRecord(k1_event(eng, 0), eng->stream));
        // the FP32 accumulation bound grows with the d+1 terms of each dot product
        const double tau_s = eng->tau_simt * std::max(1.0, (eng->D + 1) / 51.0);
        tsom::launch_bmu_simt(x, ldx, sel, n, eng->D, eng->wt.as<float>(), eng->P, ppad(eng), x2max,
                              eng->w2max.as<float>(), (float)tau_s, eng->bmu.as<uint32_t>(),
                              eng->flags.as<uint32_t>(), eng->sm_count, eng->stream);
        CU(cudaEventRecord(k1_event(eng, 1), eng->stream));
        eng->k1_timed = true;
        tsom::sampler_pregenerate(eng->sampler, k1_event(eng, 1));
    }
    CU(cudaGetLastError());
    tsom::launch_rescan(x, ldx, sel, eng->w.as<float>(), eng->P, eng->D,
                        eng->flags.as<uint32_t>(), n, eng->bmu.as<uint32_t>(), eng->stream);
    CU(cudaGetLastError());
}

// out[0] = ids >= n_rows, out[1] = positions i > 0 with sel[i] <= sel[i-1]
__global__ void k_check_sel(const uint32_t* __restrict__ sel, uint64_t n, uint64_t n_rows,
                            unsigned long long* out) {
    unsigned long long bad = 0, unsorted = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = sel[i];
        bad += v >= n_rows;
        unsorted += i > 0 && v <= sel[i - 1];
    }
    for (int o = 16; o; o >>= 1) {
        bad += __shfl_xor_sync(0xffffffffu, bad, o);
        unsorted += __shfl_xor_sync(0xffffffffu, unsorted, o);
    }
    if ((threadIdx.x & 31) == 0 && (bad | unsorted)) {
        atomicAdd(out, bad);
        atomicAdd(out + 1, unsorted);
    }
}

// Upload a caller selection into eng->sel and validate it on the device
// against the bound rows (fetch_rows, dataset.hpp:393-416: an id beyond the
// data is out_of_range; any order and repeats are a valid gather).  Returns
// true when it is the identity (N strictly increasing ids in [0, N)), which
// then runs as "all rows".
bool upload_selection(Engine* eng, const uint32_t* sel, uint64_t n) {
    CU(eng->sel.ensure(std::max<uint64_t>(n, 1) * sizeof(uint32_t)));
    if (n == 0) return false;
    CU(cudaMemcpyAsync(eng->sel.p, sel, n * sizeof(uint32_t), cudaMemcpyHostToDevice, eng->stream));
    auto* chk = reinterpret_cast<unsigned long long*>(eng->hstat + 8);  // pinned [8..11]
    CU(cudaMemsetAsync(eng->status.as<int>() + 2, 0, 16, eng->stream));
    auto* dchk = reinterpret_cast<unsigned long long*>(eng->status.as<int>() + 2);
    const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)eng->sm_count * 8);
    TSOM_LAUNCH(k_check_sel<<<grid, 256, 0, eng->stream>>>(eng->sel.as<uint32_t>(), n,
                                                           eng->n_rows, dchk));
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(chk, dchk, 16, cudaMemcpyDeviceToHost, eng->stream));
    CU(cudaStreamSynchronize(eng->stream));
    REQUIRE(chk[0] == 0, TSOM_ERR_RANGE, "fetch_rows: row index beyond data size");
    REQUIRE(chk[1] == 0 || !eng->streamed, TSOM_ERR_INVALID,
            "epoch: streamed data needs a sorted, distinct selection (Sampler::select order)");
    return chk[1] == 0 && n == eng->n_rows;
}

// resident rows are kept at a 256-B stride (each row exactly two 128-B lines
// for the K2 gather) when d is even and <= 62 (TSOM_OPT_PAD_ROWS, default on)
bool pad_eligible(const Engine* eng) {
    return eng->pad_rows && eng->D % 2 == 0 && eng->D <= tsom::kPadFloats - 2;
}

// The one resident copy of the bound rows: n_rows at stride ldx (+ slack for
// the row-window gathers).
void alloc_resident(Engine* eng, uint64_t n_rows) {
    eng->ldx = pad_eligible(eng) ? tsom::kPadFloats : eng->D;
    CU(eng->x.ensure(std::max<uint64_t>(n_rows, 1) * eng->ldx * sizeof(float) + tsom::kRowSlack));
    eng->x_slack = true;
}

// Rows [0, total) of the bound host source (caller rows, or shard files read
// into pinned staging) into the resident copy, C rows per chunk on the copy
// stream.  Each chunk's row-norm maximum (and, for padded rows, its placement
// at the 256-B stride from a packed device stage) runs on the engine stream
// while the next chunk is in flight.
void upload_resident(Engine* eng, uint64_t total, uint64_t C) {
    tsom::NvtxRange nv("tsom.bind_upload");
    alloc_resident(eng, total);
    const bool pad = eng->ldx != eng->D;
    const uint64_t rowb = (uint64_t)eng->D * sizeof(float);
    C = std::max<uint64_t>(1, std::min<uint64_t>(C, std::max<uint64_t>(total, 1)));
    if (pad) {
        CU(eng->stage[0].ensure(C * rowb + tsom::kRowSlack));
        CU(eng->stage[1].ensure(C * rowb + tsom::kRowSlack));
    }
    CU(cudaMemsetAsync(eng->x2max.p, 0, sizeof(float), eng->stream));
    for (uint64_t r0 = 0, c = 0; r0 < total; r0 += C, ++c) {
        const uint64_t r1 = std::min(total, r0 + C), nr = r1 - r0;
        const int s = (int)(c & 1);
        const float* src = host_chunk_source(eng, r0, r1, s);
        float* dst = pad ? eng->stage[s].as<float>() : eng->x.as<float>() + r0 * eng->D;
        if (pad && c >= 2) CU(cudaStreamWaitEvent(eng->copy_stream, eng->ev[4 + s], 0));
        CU(cudaMemcpyAsync(dst, src, nr * rowb, cudaMemcpyHostToDevice, eng->copy_stream));
        note_pinned_copy(eng, s);
        CU(cudaEventRecord(eng->ev[2 + s], eng->copy_stream));
        CU(cudaStreamWaitEvent(eng->stream, eng->ev[2 + s], 0));
        tsom::launch_row_norm_max(dst, nr, eng->D, eng->x2max.as<float>(), eng->stream, false);
        if (pad) {
            tsom::launch_pad_rows(dst, nr, eng->D, eng->x.as<float>() + r0 * tsom::kPadFloats,
                                  eng->stream);
            CU(cudaEventRecord(eng->ev[4 + s], eng->stream));
        }
    }
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(eng->stream));
    if (pad) {
        eng->stage[0].release(true);
        eng->stage[1].release(true);
    }
}

// K2 scratch (counting sort + piece partials) sized for `rows` rows per launch.
void ensure_accum(Engine* eng, uint64_t rows) {
    if (rows <= eng->acc_rows && eng->acc.counts) return;
    size_t bytes[7];
    tsom::accum_scratch_bytes(rows, eng->P, eng->D, bytes);
    for (int i = 0; i < 7; ++i) CU(eng->acc_buf[i].ensure(bytes[i]));
    eng->acc.counts = eng->acc_buf[0].as<uint32_t>();
    eng->acc.totals = eng->acc_buf[1].as<uint32_t>();
    eng->acc.node_start = eng->acc_buf[2].as<uint32_t>();
    eng->acc.piece_start = eng->acc_buf[3].as<uint32_t>();
    eng->acc.piece_node = eng->acc_buf[4].as<uint32_t>();
    eng->acc.sorted = eng->acc_buf[5].as<uint32_t>();
    eng->acc.partial = eng->acc_buf[6].as<double>();
    eng->acc_rows = rows;
}

// TSOM_OPT_ROW_ORDER (k_order.cu).  A new bind drops the order.
void reset_order(Engine* eng) {
    eng->ordered = false;
    eng->sorted_full = false;
    eng->passes_since_order = 0;
    eng->perm.release();
    eng->pinv.release();
    eng->idmap.release();
    eng->unperm.release();
    eng->img_valid = false;  // (the split image follows the rows)
    eng->ximg.release();
    eng->ximg_xn2.release();
}

// Re-lay the rows out now?  Needs the engine's own resident copy and the
// BMU-ordered positions of a full pass over them (acc.sorted).  row_order 1
// (auto): once, at an epoch of a tsom_train_epochs call with at least
// kOrderMinEpochs epochs still to run — the re-layout costs about one to two
// epochs' time and each later epoch saves ~5 %, so a shorter run would lose
// (scripts/ab_relayout.sh, scripts/ab_relayout_large.py); 2: once, at the
// first full pass that finds one; R >= 3: that, then every R full passes.
constexpr uint32_t kOrderMinEpochs = 20;
bool order_due(const Engine* eng) {
    if (!eng->row_order || eng->streamed || !eng->x.owned || !eng->x.p || !eng->sorted_full ||
        eng->n_rows < std::max<uint64_t>(2, eng->row_order_min))
        return false;
    if (eng->row_order == 1) return !eng->ordered && eng->epochs_left >= kOrderMinEpochs;
    if (!eng->ordered) return true;
    return eng->row_order >= 3 && eng->passes_since_order >= eng->row_order;
}

// The resident rows re-laid out (packed: the gather then reads runs of rows in
// one copy) in the BMU order of the last full pass; perm / pinv composed with
// the previous order.  No new block for the rows: the permuted rows go to the
// split tiles' buffer (rebuilt from the new layout by the pass that follows
// anyway) and are copied back into the rows' own buffer — a pool allocation
// of a second copy costs tens of milliseconds once the pool has to map new
// memory, more than the re-layout saves in a run.  ~2.3 ms at 1e7 rows.
void order_rows(Engine* eng) {
    tsom::NvtxRange nv("tsom.order_rows");
    const uint64_t n = eng->n_rows;
    const size_t packed = n * eng->D * sizeof(float);
    DevBuf np;
    if (eng->xsplit.bytes < packed || packed > eng->x.bytes ||
        np.ensure_on(n * sizeof(uint32_t), eng->stream) != cudaSuccess ||
        (!eng->ordered &&
         eng->pinv.ensure_on(n * sizeof(uint32_t), eng->stream) != cudaSuccess)) {
        // no split tiles to borrow (SIMT kernel) or no room for the id maps:
        // an optimisation, not a failure — the rows keep their layout
        cudaGetLastError();
        np.release_on(eng->stream);
        if (!eng->ordered) eng->pinv.release_on(eng->stream);
        eng->row_order = 0;
        eng->sorted_full = false;
        return;
    }
    float* tmp = eng->xsplit.as<float>();
    tsom::launch_permute_rows(eng->x.as<float>(), eng->ldx, eng->acc.sorted, n, eng->D, tmp,
                              eng->ordered ? eng->perm.as<uint32_t>() : nullptr,
                              np.as<uint32_t>(), eng->stream);
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(eng->x.p, tmp, packed, cudaMemcpyDeviceToDevice, eng->stream));
    std::swap(eng->perm, np);
    np.release_on(eng->stream);
    tsom::launch_invert_perm(eng->perm.as<uint32_t>(), n, eng->pinv.as<uint32_t>(), eng->stream);
    CU(cudaGetLastError());
    eng->ldx = eng->D;  // (the buffer keeps its size; the tail past the packed rows is slack)
    eng->x_slack = true;
    eng->xsplit_valid = false;
    eng->img_valid = false;
    eng->ordered = true;
    eng->sorted_full = false;
    eng->passes_since_order = 0;
}

// Exact mode: the global max ||x||^2 (once per bind; a u64 max over the ranks
// of the float's bits — non-negative floats order like their bits) and the
// limb buffer; returns the ExactSums of this engine.
tsom::ExactSums exact_setup(Engine* eng) {
    REQUIRE(!eng->streamed, TSOM_ERR_INVALID,
            "exact mode (TSOM_OPT_DETERMINISTIC) needs resident rows");
    CU(eng->xsums.ensure(tsom::exact_sums_words(eng->P, eng->D) * sizeof(long long)));
    CU(eng->xmax_g.ensure(sizeof(uint64_t)));
    if (!eng->xmax_g_ready) {
        CU(cudaMemsetAsync(eng->xmax_g.p, 0, sizeof(uint64_t), eng->stream));
        CU(cudaMemcpyAsync(eng->xmax_g.p, eng->x2max.p, sizeof(float), cudaMemcpyDeviceToDevice,
                           eng->stream));
        if (eng->comm_reduce) {
            const int rc = eng->comm_reduce(eng->xmax_g.p, 1, 1);
            if (rc != TSOM_OK) throw tsom::Fail{rc};
        }
        eng->xmax_g_ready = true;
    }
    tsom::ExactSums ex;
    ex.xs = eng->xsums.as<long long>();
    ex.xmax2 = eng->xmax_g.as<float>();
    ex.w2max = eng->w2max.as<float>();
    return ex;
}

// One pass over the bound rows (resident or streamed): BMU search, then K2
// into sums = [R | c | sum dist | rows] (+ allreduce).  want_dist: per-row
// distances into eng->dist; want_dsum: distance sum; accumulate: R and c.
// dev_sel (optional, resident data only): a sorted selection of n_sel rows
// already in device memory (the device sampler's), used instead of sel_host.
void accumulate_epoch(Engine* eng, const uint32_t* sel_host, uint64_t n_sel, bool want_dist,
                      bool want_dsum, bool accumulate, const uint32_t* dev_sel = nullptr) {
    tsom::NvtxRange nv("tsom.pass");
    CU(eng->sums.ensure(slot_len(eng) * sizeof(double)));
    const uint32_t* sel = dev_sel;
    if (!dev_sel) {
        if (!sel_host)
            REQUIRE(n_sel == 0 || n_sel == eng->n_rows, TSOM_ERR_INVALID,
                    "epoch: NULL selection means all rows (n_sel must be 0 or tsom_rows())");
        else if (!upload_selection(eng, sel_host, n_sel))
            sel = sel_host;
    }
    const uint64_t n = sel ? n_sel : eng->n_rows;
    const uint32_t* dsel = dev_sel ? dev_sel : (sel ? eng->sel.as<uint32_t>() : nullptr);
    if (!eng->streamed) {
        if (!sel && order_due(eng)) order_rows(eng);
        if (sel && eng->ordered && n) {  // caller row ids -> positions of the ordered rows
            CU(eng->idmap.ensure(n * sizeof(uint32_t)));
            tsom::launch_map_ids(dsel, n, eng->pinv.as<uint32_t>(), eng->idmap.as<uint32_t>(),
                                 eng->stream);
            CU(cudaGetLastError());
            dsel = eng->idmap.as<uint32_t>();
        }
    }
    ensure_rows(eng, n, want_dist);
    prep_codebook(eng);
    eng->last_recheck = 0;
    eng->recheck_from_chunks = false;
    eng->k1_timed = false;
    eng->update_timed = false;
    CU(cudaEventRecord(eng->ev[0], eng->stream));
    if (!eng->streamed) {
        const void* tiles = nullptr;
        const float* tiles_xn2 = nullptr;
        const int kind = tc_kind(eng);
        if (kind != tsom::kTcNone && !sel) {
            if (!eng->xsplit_valid || eng->xsplit_kind != kind) {
                // split once per bound dataset (the rows do not change across epochs)
                const uint64_t ntiles = (eng->n_rows + tsom::kTcTileM - 1) / tsom::kTcTileM;
                CU(eng->xsplit.ensure(ntiles * tsom::tc_geom(kind, eng->D).tile_bytes));
                CU(eng->xn2.ensure(std::max<uint64_t>(eng->n_rows, 1) * sizeof(float)));
                tsom::launch_set_scale(kind, eng->x2max.as<float>(), eng->scale.as<float>(),
                                       eng->stream);
                tsom::launch_split_rows(kind, eng->x.as<float>(), nullptr, nullptr, eng->n_rows,
                                        eng->D, eng->scale.as<float>(), tie_window(eng, kind),
                                        eng->xsplit.p, eng->xn2.as<float>(), eng->stream, nullptr,
                                        eng->ldx);
                eng->xsplit_valid = true;
                eng->xsplit_kind = kind;
            }
            tiles = eng->xsplit.p;
            tiles_xn2 = eng->xn2.as<float>();
        }
        tsom::ExactSums ex;
        if (eng->exact) ex = exact_setup(eng);
        run_bmu(eng, eng->x.as<float>(), eng->ldx, dsel, n, eng->x2max.as<float>(), tiles,
                tiles_xn2, eng->ordered && !sel);
        eng->pass_x = eng->x.as<float>();
        eng->pass_ldx = eng->ldx;
        eng->pass_sel = dsel;
        eng->pass_n = n;
        CU(cudaEventRecord(eng->ev[1], eng->stream));
        if (eng->k1_slot >= 0)  // multi-epoch call: this epoch's accumulation phase
            CU(cudaEventRecord(eng->acc_ev[2 * (size_t)eng->k1_slot], eng->stream));
        ensure_accum(eng, n);
        const int arc = tsom::launch_accumulate(
            eng->x.as<float>(), dsel, n, eng->D, eng->w.as<float>(), eng->P,
            eng->bmu.as<uint32_t>(), want_dist ? eng->dist.as<double>() : nullptr, want_dsum,
            accumulate, true, eng->acc, eng->sums.as<double>(), eng->sm_count, eng->stream,
            eng->x_slack, eng->ldx, eng->exact ? &ex : nullptr);
        REQUIRE(arc == 0, TSOM_ERR_INVALID,
                "exact mode (TSOM_OPT_DETERMINISTIC) needs d even and <= 62 with resident rows");
        CU(cudaGetLastError());
        // a full pass leaves its BMU-ordered positions in acc.sorted (the
        // next re-layout's order); per-row distances go back to caller order
        eng->sorted_full = !sel && n == eng->n_rows && n > 0 &&
                           (accumulate || want_dist || want_dsum);
        if (eng->sorted_full && accumulate) ++eng->passes_since_order;
        if (eng->ordered && !sel && want_dist && n) {
            CU(eng->unperm.ensure(n * sizeof(double)));
            tsom::launch_unpermute_f64(eng->dist.as<double>(), eng->perm.as<uint32_t>(), n,
                                       eng->unperm.as<double>(), eng->stream);
            CU(cudaGetLastError());
            std::swap(eng->dist, eng->unperm);
        }
        eng->chunk_counts.clear();
        eng->recheck_from_chunks = true;
        eng->hstat_counts = true;
        // (a multi-epoch call reads only its last epoch's counts: a D2H copy
        // in the middle of the stream costs ~15 us of device time per epoch)
        if (!eng->defer_hstat)
            CU(cudaMemcpyAsync(eng->hstat, eng->flags.p, 2 * sizeof(uint32_t),
                               cudaMemcpyDeviceToHost, eng->stream));
    } else {
        // Streamed: rows live in host memory; chunks of stream_chunk_rows rows
        // are copied on copy_stream into two device stages, compute on stream.
        eng->sorted_full = false;
        eng->pass_x = nullptr;
        eng->pass_sel = nullptr;
        eng->pass_n = 0;
        REQUIRE(!eng->exact, TSOM_ERR_INVALID,
                "exact mode (TSOM_OPT_DETERMINISTIC) needs resident rows");
        const uint64_t C = eng->stream_chunk_rows;
        CU(eng->stage[0].ensure(C * eng->D * sizeof(float) + tsom::kRowSlack));
        CU(eng->stage[1].ensure(C * eng->D * sizeof(float) + tsom::kRowSlack));
        CU(eng->x2max.ensure(2 * sizeof(float)));
        ensure_accum(eng, C);
        const uint64_t nchunks = (eng->n_rows + C - 1) / C;
        // chunk list (chunks holding no selected row are skipped)
        struct Job { uint64_t c, r0, r1, p0, p1; };
        std::vector<Job> jobs;
        for (uint64_t c = 0, pos0 = 0; c < nchunks; ++c) {
            const uint64_t r0 = c * C, r1 = std::min(eng->n_rows, r0 + C);
            uint64_t p1 = pos0;
            if (sel) {
                p1 = (uint64_t)(std::lower_bound(sel + pos0, sel + n, (uint32_t)r1) - sel);
                if (p1 == pos0) continue;
            }
            jobs.push_back({c, r0, r1, pos0, p1});
            pos0 = p1;
        }
        // events: ev[2+s] = stage s filled, ev[4+s] = stage s consumed.  Two
        // chunks are in flight ahead of the compute stream: while chunk k is
        // computed, chunk k+1 is on the copy engine and the host stages k+2.
        auto issue = [&](size_t k) {
            const Job& j = jobs[k];
            const int s = (int)(k & 1);
            const float* src = host_chunk_source(eng, j.r0, j.r1, s);
            if (k >= 2) CU(cudaStreamWaitEvent(eng->copy_stream, eng->ev[4 + s], 0));
            CU(cudaMemcpyAsync(eng->stage[s].p, src, (j.r1 - j.r0) * eng->D * sizeof(float),
                               cudaMemcpyHostToDevice, eng->copy_stream));
            note_pinned_copy(eng, s);
            CU(cudaEventRecord(eng->ev[2 + s], eng->copy_stream));
        };
        CU(eng->chunk_flags.ensure(std::max<size_t>(1, 2 * jobs.size()) * sizeof(uint32_t)));
        for (size_t k = 0; k < std::min<size_t>(2, jobs.size()); ++k) issue(k);
        bool first = true;
        for (size_t k = 0; k < jobs.size(); ++k) {
            const Job& j = jobs[k];
            const int s = (int)(k & 1);
            CU(cudaStreamWaitEvent(eng->stream, eng->ev[2 + s], 0));
            const float* xs = eng->stage[s].as<float>();
            float* xmax = eng->x2max.as<float>() + 1;
            tsom::launch_row_norm_max(xs, j.r1 - j.r0, eng->D, xmax, eng->stream);
            tsom::launch_fold_max(eng->x2max.as<float>(), eng->stream);
            // selected rows of this chunk are addressed as (row - r0): shift the base
            const float* xbase = xs - (ptrdiff_t)(j.r0 * eng->D);
            const uint64_t cn = sel ? (j.p1 - j.p0) : (j.r1 - j.r0);
            const uint32_t* csel = sel ? dsel + j.p0 : nullptr;
            const uint64_t out0 = sel ? j.p0 : j.r0;
            run_bmu(eng, sel ? xbase : xs, eng->D, csel, cn, xmax, nullptr, nullptr);
            // re-check counters per chunk, kept on the device (a D2H into pageable
            // memory here would block the host and stall the look-ahead)
            CU(cudaMemcpyAsync(eng->chunk_flags.as<uint32_t>() + 2 * k, eng->flags.p,
                               2 * sizeof(uint32_t), cudaMemcpyDeviceToDevice, eng->stream));
            tsom::launch_accumulate(sel ? xbase : xs, csel, cn, eng->D, eng->w.as<float>(), eng->P,
                                    eng->bmu.as<uint32_t>(),
                                    want_dist ? eng->dist.as<double>() + out0 : nullptr, want_dsum,
                                    accumulate, first, eng->acc, eng->sums.as<double>(),
                                    eng->sm_count, eng->stream, true);
            CU(cudaGetLastError());
            CU(cudaEventRecord(eng->ev[4 + s], eng->stream));
            first = false;
            if (k + 2 < jobs.size()) issue(k + 2);
        }
        if (first) CU(cudaMemsetAsync(eng->sums.p, 0, slot_len(eng) * sizeof(double), eng->stream));
        eng->hstat_counts = false;
        eng->chunk_counts.assign(std::max<size_t>(2, 2 * jobs.size()), 0u);
        if (!jobs.empty())
            CU(cudaMemcpyAsync(eng->chunk_counts.data(), eng->chunk_flags.p,
                               2 * jobs.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                               eng->stream));
        eng->recheck_from_chunks = true;
        CU(cudaEventRecord(eng->ev[1], eng->stream));
    }
    if (n == 0 && !eng->streamed)
        CU(cudaMemsetAsync(eng->sums.p, 0, slot_len(eng) * sizeof(double), eng->stream));
    CU(cudaGetLastError());
    // the one reduce of the epoch (parallel.hpp:90-95): [S | c | sum dist | rows]
    // summed over the ranks, identical on every rank afterwards
    if (eng->exact && !eng->streamed) {
        // exact sums: the one reduce is an int64 sum of the limb buffer, then
        // the f64 sums are rebuilt from it (the same on every rank)
        if (eng->comm_reduce && (accumulate || want_dsum)) {
            tsom::NvtxRange nvr("tsom.reduce");
            const int rc = eng->comm_reduce(eng->xsums.p, tsom::exact_sums_words(eng->P, eng->D), 4);
            if (rc != TSOM_OK) throw tsom::Fail{rc};
        }
        tsom::ExactSums ex;
        ex.xs = eng->xsums.as<long long>();
        ex.xmax2 = eng->xmax_g.as<float>();
        ex.w2max = eng->w2max.as<float>();
        tsom::launch_exact_unpack(ex, eng->P, eng->D, eng->sums.as<double>(), eng->stream);
        CU(cudaGetLastError());
    } else if (eng->comm_reduce && (accumulate || want_dsum)) {
        tsom::NvtxRange nvr("tsom.reduce");
        const int rc = eng->comm_reduce(eng->sums.p, slot_len(eng), 3);
        if (rc != TSOM_OK) throw tsom::Fail{rc};
    }
    CU(cudaEventRecord(eng->ev[2 + 4], eng->stream));
    if (eng->k1_slot >= 0 && !eng->streamed)
        CU(cudaEventRecord(eng->acc_ev[2 * (size_t)eng->k1_slot + 1], eng->stream));
}

std::string barrier_seconds(double s) { return std::to_string(s); }  // the reference's format

// Drop the communicator after a failed or timed-out reduce (ncclCommAbort
// ends its kernels); the engine then runs single-rank again.
void abort_comm(Engine* eng) {
    if (eng->nccl_comm && g_nccl.commAbort) g_nccl.commAbort((ncclComm_t)eng->nccl_comm);
    eng->nccl_comm = nullptr;
    eng->comm_reduce = nullptr;
    eng->sampler.allreduce = nullptr;
    eng->sampler.sync = nullptr;
    eng->red_pending = 0;
    eng->world = 1;
    eng->rank = 0;
    cudaStreamSynchronize(eng->stream);
    cudaGetLastError();
}

// Wait for the engine stream.  With NCCL reduces in flight this is the reduce
// barrier of collect_with_barrier (parallel.hpp:67-86): every enqueued reduce
// must complete within barrier_timeout_s of the previous one (or of the start
// of the wait), else the communicator is aborted and the call fails with
// TSOM_ERR_TIMEOUT instead of hanging on a dead peer.
void wait_stream(Engine* eng) {
    tsom::NvtxRange nv("tsom.wait");
    if (!eng->nccl_comm || eng->red_pending == 0) {
        eng->red_pending = 0;
        CU(cudaStreamSynchronize(eng->stream));
        return;
    }
    using clk = std::chrono::steady_clock;
    const size_t pending = eng->red_pending;
    const auto t0 = clk::now();
    auto mark = t0;
    size_t done = 0;
    for (int spin = 0;; ++spin) {
        while (done < pending) {
            const cudaError_t q = cudaEventQuery(eng->red_ev[done]);
            if (q == cudaErrorNotReady) break;
            CU(q);
            ++done;
            mark = clk::now();
        }
        const cudaError_t q = cudaStreamQuery(eng->stream);
        if (q == cudaSuccess) break;
        if (q != cudaErrorNotReady) CU(q);
        ncclResult_t ae = ncclSuccess;
        g_nccl.getAsyncError((ncclComm_t)eng->nccl_comm, &ae);
        if (ae != ncclSuccess && ae != ncclInProgress) {
            abort_comm(eng);
            REQUIRE(false, TSOM_ERR_NCCL,
                    std::string("nccl: reduce failed: ") + (g_nccl.errStr ? g_nccl.errStr(ae) : "?"));
        }
        if (done < pending &&
            std::chrono::duration<double>(clk::now() - mark).count() > eng->barrier_timeout_s) {
            const int me = eng->rank, world = eng->world;
            abort_comm(eng);
            // NCCL does not say which peer is missing: name the ranks it can be
            REQUIRE(false, TSOM_ERR_TIMEOUT,
                    "reduce barrier timed out after " + barrier_seconds(eng->barrier_timeout_s) +
                        " s waiting for worker " + std::to_string(me == 0 ? 1 : 0) +
                        (world > 2 ? " (or another peer of rank " + std::to_string(me) + ")" : ""));
        }
        if (spin < 256)
            std::this_thread::yield();
        else
            std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
    eng->barrier_wait_s += std::chrono::duration<double>(clk::now() - t0).count();
    eng->red_pending = 0;
}

// Guard of quantize_term (accum.hpp:34-38) for the last accumulation pass,
// with the epoch's (pre-update) codebook: exact on resident rows (k_guard.cu:
// a cheap bound, and only when it fails the per-node extremes test);
// streamed rows are not kept, so there the bound decides alone.
// dead (optional): the multi-epoch failure record, set before the update.
uint32_t enqueue_term_guard(Engine* eng, double eta, int* dead = nullptr, uint32_t epoch = 0) {
    const size_t words = tsom::guard_scratch_words(eng->P, eng->D);
    if (eng->guard_buf.bytes < words * sizeof(uint32_t)) {
        CU(eng->guard_buf.ensure(words * sizeof(uint32_t)));
        CU(cudaMemsetAsync(eng->guard_buf.p, 0, words * sizeof(uint32_t), eng->stream));
    }
    const uint32_t tag = ++eng->guard_tag ? eng->guard_tag : ++eng->guard_tag;  // never 0
    static const int mode = [] {  // diagnostics: TSOM_GUARD=1 plain launch, 2 skip (A/B)
        const char* v = getenv("TSOM_GUARD");
        return v ? atoi(v) : 0;
    }();
    if (mode == 2) return tag;
    CU(tsom::launch_term_guard(eng->pass_x, eng->pass_ldx, eng->pass_sel, eng->pass_n,
                            eng->bmu.as<uint32_t>(), eng->w.as<float>(), eng->infl.as<double>(),
                            eng->P, eng->D, eta, eng->x2max.as<float>(), eng->w2max.as<float>(),
                            eng->hmax.as<double>(), tag,
                            tsom::guard_scratch(eng->guard_buf.as<uint32_t>(), eng->P, eng->D),
                            eng->sm_count, eng->stream, dead, epoch));
    return tag;
}

// the guard's verdict, read back with the epoch's other status words
void enqueue_guard_read(Engine* eng) {
    CU(cudaMemcpyAsync(eng->hstat + 3, eng->guard_buf.as<uint32_t>() + 1, sizeof(uint32_t),
                       cudaMemcpyDeviceToHost, eng->stream));
}

// after the end-of-epoch synchronisation
void check_term_guard(Engine* eng, uint32_t tag) {
    REQUIRE(eng->hstat[3] != tag, TSOM_ERR_NUMERICAL,
            "numerical fault: accumulation term out of range (|term| >= 2^22)");
}

void finish_recheck(Engine* eng) {
    fold_tie_log(eng);
    if (eng->recheck_from_chunks) {
        uint64_t t = 0;
        if (eng->hstat_counts)
            t = (uint64_t)eng->hstat[0] + eng->hstat[1];
        else
            for (uint32_t c : eng->chunk_counts) t += c;
        eng->last_recheck = t;
    }
}

void smooth(Engine* eng, double eta) {
    tsom::NvtxRange nv("tsom.smooth");
    CU(eng->smooth_scratch.ensure(tsom::smooth_scratch_doubles(eng->P, eng->D) * sizeof(double)));
    tsom::launch_smooth(eng->infl.as<double>(), eng->sums.as<double>(), eng->w.as<float>(), eng->P,
                        eng->D, eta, eng->U.as<double>(), eng->H.as<double>(),
                        eng->smooth_scratch.as<double>(), eng->stream, eng->status.as<int>());
    CU(cudaGetLastError());
    CU(cudaEventRecord(eng->ev[7], eng->stream));
}

void record_timing(Engine* eng) {
    eng->t_k1 = 0.0f;
    eng->t_update = 0.0f;
    if (eng->k1_timed) cudaEventElapsedTime(&eng->t_k1, eng->ev[8], eng->ev[9]);
    if (eng->update_timed) cudaEventElapsedTime(&eng->t_update, eng->ev[7], eng->ev[10]);
    eng->t_sample = 0.0f;
    if (eng->sample_timed) cudaEventElapsedTime(&eng->t_sample, eng->ev[11], eng->ev[0]);
    cudaEventElapsedTime(&eng->t_bmu, eng->ev[0], eng->ev[1]);
    cudaEventElapsedTime(&eng->t_accum, eng->ev[1], eng->ev[6]);
    cudaEventElapsedTime(&eng->t_smooth, eng->ev[6], eng->ev[7]);
    cudaEventElapsedTime(&eng->t_total, eng->ev[0], eng->ev[7]);
    cudaGetLastError();  // an event pair that was not recorded must not poison later calls
}

// every device buffer an engine owns (the sampler's are released separately)
std::vector<DevBuf*> all_buffers(Engine* eng) {
    return std::vector<DevBuf*>({&eng->x, &eng->xsplit, &eng->xn2, &eng->gxn2, &eng->txn2, &eng->x2max, &eng->w, &eng->wt, &eng->wsplit, &eng->w2,
                      &eng->w2max, &eng->scale, &eng->prev, &eng->infl, &eng->topo_dist, &eng->sel,
                      &eng->rows_scratch, &eng->gsplit, &eng->tsort, &eng->tcls, &eng->bmu, &eng->dist, &eng->part,
                      &eng->flags, &eng->ties, &eng->tmask, &eng->part2, &eng->tsplit, &eng->tcnt, &eng->acc_buf[0], &eng->acc_buf[1], &eng->acc_buf[2], &eng->acc_buf[3],
                      &eng->acc_buf[4], &eng->acc_buf[5], &eng->acc_buf[6], &eng->sums, &eng->chunk_flags,
                      &eng->topo_buf[0], &eng->topo_buf[1], &eng->topo_buf[2], &eng->topo_buf[3],
                      &eng->topo_buf[4], &eng->topo_buf[5], &eng->topo_buf[6], &eng->topo_buf[7],
                      &eng->topo_buf[8], &eng->topo_buf[9], &eng->topo_buf[10], &eng->topo_buf[11],
                      &eng->topo_buf[12], &eng->topo_buf[13], &eng->topo_buf[14], &eng->U, &eng->H, &eng->status, &eng->smooth_scratch,
                      &eng->stage[0], &eng->stage[1], &eng->dead, &eng->hmax, &eng->guard_buf,
                      &eng->tie_dev, &eng->xsums, &eng->xmax_g, &eng->perm, &eng->pinv,
                      &eng->idmap, &eng->unperm, &eng->ximg, &eng->ximg_xn2, &eng->gid});
}

}  // namespace

extern "C" {

const char* tsom_version(void) { return kVersion; }

int tsom_create(int device, uint32_t nodes, uint32_t dims, tsom_engine** out) {
    if (!out) return TSOM_ERR_INVALID;
    *out = nullptr;
    // d <= 256 (K2 lanes); K <= 65536 (16-bit node ids in the near-tie merge;
    // the K x K FP64 influence matrix alone is 34 GB there)
    if (nodes < 1 || nodes > 65536 || dims < 1 || dims > 256) return TSOM_ERR_INVALID;
    auto* eng = new tsom_engine();
    eng->device = device;
    eng->P = nodes;
    eng->D = dims;
    int rc = guarded(eng, [&] {
        int ndev = 0;
        CU(cudaGetDeviceCount(&ndev));
        REQUIRE(device >= 0 && device < ndev, TSOM_ERR_CUDA, "cuda: no such device");
        CU(cudaSetDevice(device));
        // single attributes (cudaGetDeviceProperties costs milliseconds per call)
        int major = 0, sms = 0, smem = 0;
        CU(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
        CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        CU(cudaDeviceGetAttribute(&smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
        if (major < 10) {
            cudaDeviceProp prop;
            CU(cudaGetDeviceProperties(&prop, device));
            REQUIRE(false, TSOM_ERR_CUDA,
                    std::string("cuda: device ") + prop.name + " is not sm_100 (B200) class");
        }
        eng->sm_count = sms;
        eng->smem_optin = (size_t)smem;
        // diagnostics: defaults for engines built by code that sets no options
        // (the C++ drop-ins), for A/B runs
        if (const char* v = getenv("TSOM_ROW_ORDER")) eng->row_order = (uint32_t)atoi(v);
        if (const char* v = getenv("TSOM_PAGEABLE_CHUNK_MB"))
            eng->pageable_chunk_bytes = std::max<uint64_t>(1, (uint64_t)atoll(v)) << 20;
        CU(cudaStreamCreateWithFlags(&eng->stream, cudaStreamNonBlocking));
        CU(cudaStreamCreateWithFlags(&eng->copy_stream, cudaStreamNonBlocking));
        for (auto& ev : eng->ev) CU(cudaEventCreate(&ev));
        const size_t P = nodes, D = dims;
        CU(eng->w.ensure(P * D * sizeof(float)));
        CU(eng->prev.ensure(P * D * sizeof(float)));
        CU(cudaMemsetAsync(eng->prev.p, 0, P * D * sizeof(float), eng->stream));
        CU(eng->wt.ensure((size_t)(D + 1) * ppad(eng) * sizeof(float)));
        CU(eng->w2.ensure(P * sizeof(double)));
        CU(eng->w2max.ensure(sizeof(float)));
        CU(eng->x2max.ensure(2 * sizeof(float)));
        CU(cudaMemsetAsync(eng->x2max.p, 0, 2 * sizeof(float), eng->stream));
        CU(eng->scale.ensure(4 * sizeof(float)));
        CU(cudaMemsetAsync(eng->scale.p, 0, 4 * sizeof(float), eng->stream));
        CU(eng->infl.ensure(P * P * sizeof(double)));
        CU(eng->U.ensure(P * D * sizeof(double)));
        CU(eng->H.ensure(P * sizeof(double)));
        CU(eng->status.ensure(8 * sizeof(int)));
        CU(eng->hmax.ensure(tsom::kHmaxParts * sizeof(double)));
        CU(cudaMemsetAsync(eng->hmax.p, 0, tsom::kHmaxParts * sizeof(double), eng->stream));
        CU(host_words_take(&eng->hstat));
        eng->tie_log = eng->hstat + 32;
        CU(eng->tie_dev.ensure(kTieLogCap * sizeof(uint32_t)));
        std::memset(eng->hstat, 0, 32 * sizeof(uint32_t));
        ensure_rows(eng, 1);
        CU(cudaStreamSynchronize(eng->stream));
    });
    if (rc != TSOM_OK) {
        std::fprintf(stderr, "tsom_create: %s\n", eng->last_error.c_str());
        tsom_destroy(eng);
        return rc;
    }
    *out = eng;
    return TSOM_OK;
}

int tsom_destroy(tsom_engine* eng) {
    if (!eng) return TSOM_OK;
    cudaSetDevice(eng->device);
    cudaDeviceSynchronize();  // every stream of this engine idle before its blocks return
    if (eng->nccl_comm && g_nccl.commDestroy) g_nccl.commDestroy((ncclComm_t)eng->nccl_comm);
    if (eng->host_registered) cudaHostUnregister(const_cast<float*>(eng->host_rows));
    close_shards(eng);
    tsom::sampler_release(eng->sampler);
    for (int s2 = 0; s2 < 2; ++s2) {
        pinned_give(eng->pinned[s2], eng->pinned_bytes[s2]);
        if (eng->ev_pin[s2]) cudaEventDestroy(eng->ev_pin[s2]);
    }
    for (DevBuf* b : all_buffers(eng))
        b->release(true);
    for (auto& ev : eng->ev)
        if (ev) cudaEventDestroy(ev);
    host_words_give(eng->hstat);  // (tie_log lives in the same block)
    for (cudaEvent_t e : eng->k1_ev) cudaEventDestroy(e);
    for (cudaEvent_t e : eng->acc_ev) cudaEventDestroy(e);
    for (cudaEvent_t e : eng->red_ev) cudaEventDestroy(e);
    if (eng->stream) cudaStreamDestroy(eng->stream);
    if (eng->copy_stream) cudaStreamDestroy(eng->copy_stream);
    delete eng;
    return TSOM_OK;
}

const char* tsom_last_error(const tsom_engine* eng) {
    return eng ? eng->last_error.c_str() : "null engine";
}

int tsom_set_option(tsom_engine* eng, int key, int64_t value) {
    return guarded(eng, [&] {
        switch (key) {
            case TSOM_OPT_BMU_KERNEL:
                REQUIRE(value >= 0 && value <= 3, TSOM_ERR_INVALID, "option: bmu kernel 0..3");
                REQUIRE(value != 2 || tsom::tc_supported(tsom::kTcTf32, eng->P, eng->D),
                        TSOM_ERR_INVALID, "option: 3xTF32 tcgen05 BMU kernel needs d <= 53");
                REQUIRE(value != 3 || tsom::tc_supported(tsom::kTcF16, eng->P, eng->D),
                        TSOM_ERR_INVALID, "option: 3xFP16 tcgen05 BMU kernel needs d <= 62");
                eng->bmu_kernel = (int)value;
                eng->codebook_prepped = false;
                break;
            case TSOM_OPT_TIE_TAU:
                REQUIRE(value >= 0, TSOM_ERR_INVALID, "option: tau must be >= 0");
                eng->tau_simt = eng->tau_tc = (double)value * std::ldexp(1.0, -30);
                eng->xsplit_valid = eng->img_valid = false;  // their window terms change
                break;
            case TSOM_OPT_STREAM_CHUNK:
                REQUIRE(value >= 128, TSOM_ERR_INVALID, "option: stream chunk >= 128 rows");
                eng->stream_chunk_rows = (uint64_t)value;
                break;
            case 99:  // diagnostics (not in the public header): K1 stage isolation
                tsom::g_k1_debug = (uint32_t)value;
                break;
            case 98:  // diagnostics: element-wise 3xFP16 split (k_split_rows<kTcF16>)
                tsom::g_split_v1 = (int)value;
                break;
            case 96:  // diagnostics: 1 = the per-row main-pass merge (k_merge_fast)
                tsom::g_merge_v1 = (int)value;
                break;
            case 92:  // diagnostics: gathered split L2 prefetch distance in chunks (0 = off)
                tsom::g_split_prefetch = (int)value;
                break;
            case 91:  // diagnostics: gathered split rows staged by TMA (1, default) or loaded (0)
                tsom::g_split_tma = (int)value;
                break;
            case 93:  // diagnostics: fewest rows a BMU-order re-layout is made for
                eng->row_order_min = (uint64_t)value;
                break;
            case 94:  // diagnostics: pageable-bind staging chunk, bytes
                REQUIRE(value >= (1 << 20), TSOM_ERR_INVALID, "option: chunk >= 1 MiB");
                eng->pageable_chunk_bytes = (uint64_t)value;
                break;
            case 95:  // diagnostics: 0 = no split image (selections split per pass)
                eng->img_mode = (int)value;
                eng->img_valid = false;
                break;
            case 97:  // diagnostics: 1 = cp.async K2 gather instead of the TMA gather
                tsom::g_gather_kind = (int)value;
                break;
            case TSOM_OPT_HOST_REGISTER:
                eng->host_register = value != 0;
                break;
            case TSOM_OPT_BARRIER_TIMEOUT_MS:
                REQUIRE(value >= 1, TSOM_ERR_INVALID, "option: barrier timeout >= 1 ms");
                eng->barrier_timeout_s = (double)value / 1000.0;
                break;
            case TSOM_OPT_DETERMINISTIC:
                eng->exact = value != 0;
                eng->xmax_g_ready = false;
                break;
            case TSOM_OPT_PAD_ROWS:
                eng->pad_rows = value != 0;
                break;
            case TSOM_OPT_ROW_ORDER:
                REQUIRE(value >= 0 && value <= (1 << 30), TSOM_ERR_INVALID,
                        "option: row order 0, 1 (auto), 2 (once) or a re-layout period >= 3");
                eng->row_order = (uint32_t)value;
                break;
            case TSOM_OPT_STAGING_THREADS:
                REQUIRE(value >= 1 && value <= 64, TSOM_ERR_INVALID,
                        "option: staging threads in [1, 64]");
                eng->staging_threads = (uint32_t)value;
                break;
            default:
                REQUIRE(false, TSOM_ERR_INVALID, "option: unknown key");
        }
    });
}

int tsom_bind_host_data(tsom_engine* eng, const float* rows, uint64_t n_rows, uint32_t flags) {
    return guarded(eng, [&] {
        CU(cudaSetDevice(eng->device));
        REQUIRE(rows || n_rows == 0, TSOM_ERR_INVALID, "bind: null rows");
        REQUIRE(n_rows < (1ull << 32), TSOM_ERR_INVALID, "bind: row ids are uint32 (n < 2^32)");
        if (eng->host_registered) {
            cudaHostUnregister(const_cast<float*>(eng->host_rows));
            eng->host_registered = false;
        }
        eng->host_direct = false;
        close_shards(eng);
        eng->xsplit_valid = false;
        reset_order(eng);
        eng->xmax_g_ready = false;
        eng->n_rows = n_rows;
        cudaPointerAttributes pa{};
        const bool pinned = n_rows && cudaPointerGetAttributes(&pa, rows) == cudaSuccess &&
                            pa.type == cudaMemoryTypeHost;
        cudaGetLastError();
        eng->host_rows = rows;
        if (flags & TSOM_BIND_STREAMED) {
            eng->streamed = true;
            eng->x.release();
            eng->ldx = eng->D;
            // DMA straight from the caller's rows when they are page-locked
            // already or can be pinned in place; otherwise pinned staging
            if (pinned) {
                eng->host_direct = true;
            } else if (n_rows && eng->host_register &&
                       cudaHostRegister(const_cast<float*>(rows), n_rows * eng->D * sizeof(float),
                                        cudaHostRegisterReadOnly) == cudaSuccess) {
                eng->host_registered = eng->host_direct = true;
            } else {
                cudaGetLastError();
            }
            return;
        }
        eng->streamed = false;
        eng->host_direct = pinned;
        const char* tr = getenv("TSOM_TRACE_BIND");
        const auto tb0 = std::chrono::steady_clock::now();
        // page-locked rows: 8 chunks straight from the caller's buffer, each
        // chunk's norms / 256-B-stride placement overlapped with the next DMA;
        // pageable rows: 128-MB chunks through the multi-threaded pinned
        // staging (44 GB/s on 16 host threads; 32-MB chunks: 24.5 GB/s, the
        // driver's own staging ~11 GB/s; scripts/pageable_bind_ab.py)
        const uint64_t rowb = (uint64_t)eng->D * sizeof(float);
        const uint64_t C = pinned ? std::max<uint64_t>((n_rows + 7) / 8, 4096)
                                  : std::max<uint64_t>(1, eng->pageable_chunk_bytes / rowb);
        upload_resident(eng, n_rows, C);
        eng->host_rows = nullptr;
        eng->host_direct = false;
        if (tr && tr[0] == '1')
            fprintf(stderr, "[tsom bind] %s rows=%llu ldx=%u %.2f ms\n",
                    pinned ? "pinned" : "pageable", (unsigned long long)n_rows, eng->ldx,
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() -
                                                              tb0).count());
    });
}

int tsom_bind_shards(tsom_engine* eng, const char* const* paths, uint32_t n_paths,
                     uint32_t flags) {
    return guarded(eng, [&] {
        CU(cudaSetDevice(eng->device));
        REQUIRE(paths && n_paths >= 1, TSOM_ERR_INVALID, "no .shard files given");
        if (eng->host_registered) {
            cudaHostUnregister(const_cast<float*>(eng->host_rows));
            eng->host_registered = false;
        }
        eng->host_direct = false;
        close_shards(eng);
        eng->host_rows = nullptr;
        uint64_t total = 0;
        for (uint32_t i = 0; i < n_paths; ++i) {
            Engine::ShardFile f;
            f.path = paths[i];
            f.fd = ::open(paths[i], O_RDONLY);
            if (f.fd < 0) {
                close_shards(eng);
                REQUIRE(false, TSOM_ERR_NUMERICAL, "cannot open shard: " + f.path);
            }
            eng->shards.push_back(f);
            // FSOMSHRD header (dataset.hpp:171-183, read_shard_header :221-233)
            unsigned char h[24] = {0};
            const ssize_t got = ::pread(f.fd, h, 24, 0);
            REQUIRE(got >= 8 && std::memcmp(h, "FSOMSHRD", 8) == 0, TSOM_ERR_NUMERICAL,
                    "not a shard file (bad magic): " + f.path);
            uint32_t ver, cols;
            uint64_t rows;
            std::memcpy(&ver, h + 8, 4);
            std::memcpy(&rows, h + 12, 8);
            std::memcpy(&cols, h + 20, 4);
            REQUIRE(got < 12 || ver == 1, TSOM_ERR_NUMERICAL,
                    "unsupported shard version " + std::to_string(ver) + " in " + f.path);
            REQUIRE(got == 24, TSOM_ERR_NUMERICAL, "truncated shard header: " + f.path);
            REQUIRE(cols == eng->D, TSOM_ERR_NUMERICAL, "shard column count mismatch in " + f.path);
            const off_t want = (off_t)(24 + rows * cols * sizeof(float));
            REQUIRE(::lseek(f.fd, 0, SEEK_END) == want, TSOM_ERR_NUMERICAL,
                    "truncated or corrupt shard: " + f.path);
            eng->shards.back().row0 = total;
            eng->shards.back().rows = rows;
            total += rows;
        }
        REQUIRE(total < (1ull << 32), TSOM_ERR_INVALID, "bind: row ids are uint32 (n < 2^32)");
        eng->n_rows = total;
        eng->xsplit_valid = false;
        reset_order(eng);
        eng->xmax_g_ready = false;
        if (flags & TSOM_BIND_STREAMED) {
            eng->streamed = true;
            eng->x.release();
            eng->ldx = eng->D;
            return;
        }
        // resident: stream the files once into HBM through the pinned staging
        eng->streamed = false;
        upload_resident(eng, total, eng->stream_chunk_rows);
        close_shards(eng);
    });
}

// Whether kRowSlack bytes after [p, p + bytes) lie inside the same device
// allocation (cuMemGetAddressRange through the runtime's driver entry point):
// the row-window kernels may then read a few bytes past the last row of a
// caller-owned buffer.
static bool device_slack_after(const void* p, size_t bytes) {
    using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static GetRange fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            return (GetRange) nullptr;
        }
        return reinterpret_cast<GetRange>(f);
    }();
    if (!fn || !p) return false;
    CUdeviceptr base = 0;
    size_t size = 0;
    if (fn(&base, &size, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS) return false;
    return reinterpret_cast<uintptr_t>(p) + bytes + tsom::kRowSlack <= (uintptr_t)base + size;
}

int tsom_bind_device_data(tsom_engine* eng, const float* d_rows, uint64_t n_rows) {
    return guarded(eng, [&] {
        CU(cudaSetDevice(eng->device));
        REQUIRE(n_rows < (1ull << 32), TSOM_ERR_INVALID, "bind: row ids are uint32 (n < 2^32)");
        eng->x.release();
        // borrowed rows keep the caller's packed layout (no second copy)
        eng->x.p = const_cast<float*>(d_rows);
        eng->x.bytes = n_rows * eng->D * sizeof(float);
        eng->x.owned = false;
        eng->ldx = eng->D;
        eng->x_slack = device_slack_after(d_rows, (size_t)n_rows * eng->D * sizeof(float));
        eng->n_rows = n_rows;
        eng->streamed = false;
        eng->xsplit_valid = false;
        reset_order(eng);
        eng->xmax_g_ready = false;
        tsom::launch_row_norm_max(d_rows, n_rows, eng->D, eng->x2max.as<float>(), eng->stream);
        CU(cudaGetLastError());
        CU(cudaStreamSynchronize(eng->stream));
    });
}

int tsom_bind_synthetic_gmm(tsom_engine* eng, uint64_t n_rows, uint64_t seed, uint32_t n_comp,
                            uint64_t row_offset) {
    return guarded(eng, [&] {
        CU(cudaSetDevice(eng->device));
        REQUIRE(n_comp >= 1, TSOM_ERR_INVALID, "synth: n_comp >= 1");
        REQUIRE(n_rows < (1ull << 32), TSOM_ERR_INVALID, "bind: row ids are uint32 (n < 2^32)");
        // centres from the reference Rng (rng.hpp:12-91): Rng(seed, SeedStream::synth),
        // real(-4, 4) in (component, feature) order.
        uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (4 + 1);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        std::mt19937_64 gen(z ^ (z >> 31));
        std::vector<float> centres((size_t)n_comp * eng->D);
        for (auto& c : centres) c = (float)(-4.0 + 8.0 * ((double)(gen() >> 11) * 0x1.0p-53));
        DevBuf dc;
        CU(dc.ensure(centres.size() * sizeof(float)));
        CU(tsom::h2d_blocking(dc.p, centres.data(), centres.size() * sizeof(float)));
        eng->n_rows = n_rows;
        alloc_resident(eng, n_rows);
        tsom::launch_synth_gmm(eng->x.as<float>(), n_rows, eng->D, dc.as<float>(), n_comp, seed,
                               row_offset, eng->stream, eng->ldx);
        CU(cudaGetLastError());
        eng->streamed = false;
        eng->xsplit_valid = false;
        reset_order(eng);
        eng->xmax_g_ready = false;
        tsom::launch_row_norm_max(eng->x.as<float>(), n_rows, eng->D, eng->x2max.as<float>(),
                                  eng->stream, true, eng->ldx);
        CU(cudaStreamSynchronize(eng->stream));
        dc.release();
    });
}

uint64_t tsom_rows(const tsom_engine* eng) { return eng ? eng->n_rows : 0; }

int tsom_get_rows(tsom_engine* eng, uint64_t row0, uint64_t n, float* out) {
    return guarded(eng, [&] {
        CU(cudaSetDevice(eng->device));
        REQUIRE(!eng->streamed && eng->x.p, TSOM_ERR_INVALID, "get_rows: no resident rows bound");
        REQUIRE(row0 + n <= eng->n_rows && row0 + n >= row0, TSOM_ERR_RANGE,
                "fetch_rows: row index beyond data size");
        REQUIRE(out || n == 0, TSOM_ERR_INVALID, "get_rows: null buffer");
        if (n == 0) return;
        const size_t rowb = (size_t)eng->D * sizeof(float), pitch = (size_t)eng->ldx * sizeof(float);
        if (eng->ordered) {  // caller rows [row0, row0 + n) sit at positions pinv[.]
            CU(eng->rows_scratch.ensure(n * rowb));
            tsom::launch_permute_rows(eng->x.as<float>(), eng->ldx, eng->pinv.as<uint32_t>() + row0,
                                      n, eng->D, eng->rows_scratch.as<float>(), nullptr, nullptr,
                                      eng->stream);
            CU(cudaGetLastError());
            CU(cudaMemcpyAsync(out, eng->rows_scratch.p, n * rowb, cudaMemcpyDeviceToHost,
                               eng->stream));
        } else {
            CU(cudaMemcpy2DAsync(out, rowb, eng->x.as<float>() + row0 * eng->ldx, pitch, rowb, n,
                                 cudaMemcpyDeviceToHost, eng->stream));
        }
        CU(cudaStreamSynchronize(eng->stream));
    });
}

int tsom_set_codebook(tsom_engine* eng, const float* weights) {
    return guarded(eng, [&] {
        CU(cudaSetDevice(eng->device));
        REQUIRE(weights, TSOM_ERR_INVALID, "set_codebook: null weights");
        CU(cudaMemcpyAsync(eng->w.p, weights, (size_t)eng->P * eng->D * sizeof(float),
                           cudaMemcpyHostToDevice, eng->stream));
        eng->codebook_set = true;
        eng->codebook_prepped = false;
        prep_codebook(eng);
        CU(cudaStreamSynchronize(eng->stream));
    });
}

int tsom_get_codebook(tsom_engine* eng, float* weights) {
    return guarded(eng, [&] {
        CU(cudaSetDevice(eng->device));
        REQUIRE(eng->codebook_set, TSOM_ERR_INVALID, "get_codebook: codebook not set");
        CU(cudaMemcpyAsync(weights, eng->w.p, (size_t)eng->P * eng->D * sizeof(float),
                           cudaMemcpyDeviceToHost, eng->stream));
        CU(cudaStreamSynchronize(eng->stream));
    });
}

int tsom_get_prev_update(tsom_engine* eng, float* prev) {
    return guarded(eng, [&] {
        CU(cudaSetDevice(eng->device));
        REQUIRE(prev, TSOM_ERR_INVALID, "get_prev_update: null buffer");
        CU(cudaMemcpyAsync(prev, eng->prev.p, (size_t)eng->P * eng->D * sizeof(float),
                           cudaMemcpyDeviceToHost, eng->stream));
        CU(cudaStreamSynchronize(eng->stream));
    });
}

int tsom_set_influence(tsom_engine* eng, const double* influence, int64_t key) {
    return guarded(eng, [&] {
        CU(cudaSetDevice(eng->device));
        REQUIRE(influence, TSOM_ERR_INVALID, "set_influence: null matrix");
        if (key >= 0 && eng->infl_set && key == eng->infl_key) return;
        const size_t n = (size_t)eng->P * eng->P;
        CU(cudaMemcpyAsync(eng->infl.p, influence, n * sizeof(double), cudaMemcpyHostToDevice,
                           eng->stream));
        tsom::launch_infl_absmax(eng->infl.as<double>(), n, eng->hmax.as<double>(), eng->stream);
        CU(cudaGetLastError());
        CU(cudaStreamSynchronize(eng->stream));
        eng->infl_key = key;
        eng->infl_set = true;
    });
}

int tsom_epoch(tsom_engine* eng, const uint32_t* selected, uint64_t n_sel, double eta,
               double* u_out, double* h_out, double* dist_out) {
    return guarded(eng, [&] {
        CU(cudaSetDevice(eng->device));
        REQUIRE(eng->infl_set, TSOM_ERR_INVALID, "epoch: influence not set");
        REQUIRE(eng->n_rows > 0 || (selected && n_sel == 0) || eng->comm_reduce, TSOM_ERR_INVALID,
                "epoch: no data bound");
        prep_codebook(eng);
        accumulate_epoch(eng, selected, n_sel, dist_out != nullptr, false, true);
        smooth(eng, eta);
        const uint32_t tag = enqueue_term_guard(eng, eta);
        const size_t P = eng->P, D = eng->D;
        if (u_out)
            CU(cudaMemcpyAsync(u_out, eng->U.p, P * D * sizeof(double), cudaMemcpyDeviceToHost,
                               eng->stream));
        if (h_out)
            CU(cudaMemcpyAsync(h_out, eng->H.p, P * sizeof(double), cudaMemcpyDeviceToHost,
                               eng->stream));
        const uint64_t n = selected ? n_sel : eng->n_rows;
        if (dist_out && n)
            CU(cudaMemcpyAsync(dist_out, eng->dist.p, n * sizeof(double), cudaMemcpyDeviceToHost,
                               eng->stream));
        enqueue_guard_read(eng);
        wait_stream(eng);
        finish_recheck(eng);
        record_timing(eng);
        if (n) check_term_guard(eng, tag);
    });
}

int tsom_bmu(tsom_engine* eng, const float* rows, uint64_t n, uint32_t* bmu, double* dist) {
    return guarded(eng, [&] {
        CU(cudaSetDevice(eng->device));
        REQUIRE(rows || n == 0, TSOM_ERR_INVALID, "find_bmus: null rows");
        prep_codebook(eng);
        if (n == 0) return;
        CU(eng->rows_scratch.ensure(n * eng->D * sizeof(float) + tsom::kRowSlack));
        CU(cudaMemcpyAsync(eng->rows_scratch.p, rows, n * eng->D * sizeof(float),
                           cudaMemcpyHostToDevice, eng->stream));
        ensure_rows(eng, n, dist != nullptr);
        CU(eng->sums.ensure(slot_len(eng) * sizeof(double)));
        float* xm = eng->x2max.as<float>() + 1;
        tsom::launch_row_norm_max(eng->rows_scratch.as<float>(), n, eng->D, xm, eng->stream);
        run_bmu(eng, eng->rows_scratch.as<float>(), eng->D, nullptr, n, xm, nullptr, nullptr);
        if (dist) {
            ensure_accum(eng, n);
            eng->sorted_full = false;  // acc.sorted now orders these rows
            tsom::launch_accumulate(eng->rows_scratch.as<float>(), nullptr, n, eng->D,
                                    eng->w.as<float>(), eng->P, eng->bmu.as<uint32_t>(),
                                    eng->dist.as<double>(), false, false, true, eng->acc,
                                    eng->sums.as<double>(), eng->sm_count, eng->stream, true);
        }
        CU(cudaGetLastError());
        CU(cudaMemcpyAsync(bmu, eng->bmu.p, n * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                           eng->stream));
        if (dist)
            CU(cudaMemcpyAsync(dist, eng->dist.p, n * sizeof(double), cudaMemcpyDeviceToHost,
                               eng->stream));
        uint32_t cnt[2] = {0, 0};
        CU(cudaMemcpyAsync(cnt, eng->flags.p, 2 * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                           eng->stream));
        CU(cudaStreamSynchronize(eng->stream));
        eng->last_recheck = (uint64_t)cnt[0] + cnt[1];
    });
}

int tsom_bmu_bound(tsom_engine* eng, const uint32_t* selected, uint64_t n_sel, uint32_t* bmu,
                   double* dist) {
    return guarded(eng, [&] {
        CU(cudaSetDevice(eng->device));
        REQUIRE(!eng->streamed, TSOM_ERR_INVALID, "bmu_bound: resident data only");
        accumulate_epoch(eng, selected, n_sel, dist != nullptr, false, false);
        const uint64_t n = selected ? n_sel : eng->n_rows;
        if (n) {
            const void* b = eng->bmu.p;
            if (!selected && eng->ordered) {  // positions -> caller row order
                CU(eng->unperm.ensure(n * sizeof(uint32_t)));
                tsom::launch_unpermute_u32(eng->bmu.as<uint32_t>(), eng->perm.as<uint32_t>(), n,
                                           eng->unperm.as<uint32_t>(), eng->stream);
                CU(cudaGetLastError());
                b = eng->unperm.p;
            }
            CU(cudaMemcpyAsync(bmu, b, n * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                               eng->stream));
            if (dist)
                CU(cudaMemcpyAsync(dist, eng->dist.p, n * sizeof(double), cudaMemcpyDeviceToHost,
                                   eng->stream));
        }
        CU(cudaStreamSynchronize(eng->stream));
        finish_recheck(eng);
    });
}

int tsom_qe(tsom_engine* eng, const uint32_t* selected, uint64_t n_sel, double* dist_sum,
            uint64_t* count) {
    return guarded(eng, [&] {
        CU(cudaSetDevice(eng->device));
        accumulate_epoch(eng, selected, n_sel, false, true, false);
        double tail[2] = {0, 0};
        CU(cudaMemcpyAsync(tail, eng->sums.as<double>() + (size_t)eng->P * eng->D + eng->P,
                           2 * sizeof(double), cudaMemcpyDeviceToHost, eng->stream));
        wait_stream(eng);
        finish_recheck(eng);
        if (dist_sum) *dist_sum = tail[0];
        if (count) *count = (uint64_t)tail[1];
    });
}

int tsom_set_topology_distance(tsom_engine* eng, const double* dist) {
    return guarded(eng, [&] {
        CU(cudaSetDevice(eng->device));
        REQUIRE(dist, TSOM_ERR_INVALID, "topology: null distance matrix");
        const size_t n = (size_t)eng->P * eng->P;
        CU(eng->topo_dist.ensure(n * sizeof(double)));
        CU(cudaMemcpyAsync(eng->topo_dist.p, dist, n * sizeof(double), cudaMemcpyHostToDevice,
                           eng->stream));
        CU(cudaStreamSynchronize(eng->stream));
        eng->topo_set = true;
        eng->infl_key = -2;
    });
}

}  // extern "C"

namespace {
void ensure_topo(Engine* eng) {
    const size_t P = eng->P;
    if (eng->topo_p == P && eng->topo.d2) return;
    const size_t sizes[15] = {P * 8,     P * P * 8,         P * 4,     2 * P * 8, 2 * P * 4,
                              2 * P * 4, P * P,             P * 4,     P * (P > 1 ? P - 1 : 1) * 4 + 8,
                              4,         (P + 1) * 4,       P * (P > 1 ? P - 1 : 1) * 4 + 8,
                              P * P * 2, P * P * 8,         4};
    for (int i = 0; i < 15; ++i) CU(eng->topo_buf[i].ensure(sizes[i]));
    tsom::TopoScratch& t = eng->topo;
    t.norms = eng->topo_buf[0].as<double>();
    t.d2 = eng->topo_buf[1].as<double>();
    t.comp = eng->topo_buf[2].as<uint32_t>();
    t.bw = eng->topo_buf[3].as<double>();
    t.ba = eng->topo_buf[4].as<uint32_t>();
    t.bb = eng->topo_buf[5].as<uint32_t>();
    t.keep = eng->topo_buf[6].as<uint8_t>();
    t.rowcnt = eng->topo_buf[7].as<uint32_t>();
    t.edges = eng->topo_buf[8].as<uint32_t>();
    t.ne = eng->topo_buf[9].as<uint32_t>();
    t.deg = eng->topo_buf[10].as<uint32_t>();
    t.adj = eng->topo_buf[11].as<uint32_t>();
    t.hops = eng->topo_buf[12].as<uint16_t>();
    t.hopd = eng->topo_buf[13].as<double>();
    t.status = eng->topo_buf[14].as<uint32_t>();
    eng->topo_p = (uint32_t)P;
}
}  // namespace

extern "C" {

int tsom_refresh_topology(tsom_engine* eng, int kind, uint32_t* edges_out, uint64_t edges_cap,
                          uint64_t* n_edges, uint16_t* hops_out) {
    return guarded(eng, [&] {
        CU(cudaSetDevice(eng->device));
        tsom::NvtxRange nv("tsom.refresh_topology");
        REQUIRE(kind == 2 || kind == 3, TSOM_ERR_INVALID,
                "refresh_topology: kind must be 2 (mst) or 3 (rng)");
        REQUIRE(eng->codebook_set, TSOM_ERR_INVALID, "engine: codebook not set (tsom_set_codebook)");
        REQUIRE(kind != 3 || eng->P >= 2, TSOM_ERR_INVALID, "build_rng_graph: P must be >= 2");
        REQUIRE(eng->P <= 8192, TSOM_ERR_INVALID, "refresh_topology: P <= 8192 on the device");
        ensure_topo(eng);
        tsom::launch_refresh_topology(eng->w.as<float>(), eng->P, eng->D, kind, eng->topo,
                                      eng->stream);
        CU(cudaGetLastError());
        uint32_t st = 0, ne = 0;
        CU(cudaMemcpyAsync(&st, eng->topo.status, 4, cudaMemcpyDeviceToHost, eng->stream));
        CU(cudaMemcpyAsync(&ne, eng->topo.ne, 4, cudaMemcpyDeviceToHost, eng->stream));
        CU(cudaStreamSynchronize(eng->stream));
        REQUIRE(!(st & 2u), TSOM_ERR_RANGE, "hop_distances: edge index out of range");
        REQUIRE(!(st & 1u), TSOM_ERR_NUMERICAL, "hop_distances: graph is disconnected");
        if (n_edges) *n_edges = ne;
        if (edges_out) {
            REQUIRE(edges_cap >= ne, TSOM_ERR_INVALID, "refresh_topology: edge buffer too small");
            CU(cudaMemcpy(edges_out, eng->topo.edges, (size_t)ne * 2 * sizeof(uint32_t),
                          cudaMemcpyDeviceToHost));
        }
        if (hops_out)
            CU(cudaMemcpy(hops_out, eng->topo.hops, (size_t)eng->P * eng->P * sizeof(uint16_t),
                          cudaMemcpyDeviceToHost));
        // the device-resident loop builds its influence from these hop counts
        const size_t nn = (size_t)eng->P * eng->P;
        CU(eng->topo_dist.ensure(nn * sizeof(double)));
        CU(cudaMemcpyAsync(eng->topo_dist.p, eng->topo.hopd, nn * sizeof(double),
                           cudaMemcpyDeviceToDevice, eng->stream));
        CU(cudaStreamSynchronize(eng->stream));
        eng->topo_set = true;
        eng->infl_key = -2;  // influence cache cleared on refresh (topology.hpp:447)
    });
}

int tsom_pairwise_sq_dists(tsom_engine* eng, double* out) {
    return guarded(eng, [&] {
        CU(cudaSetDevice(eng->device));
        REQUIRE(eng->codebook_set, TSOM_ERR_INVALID, "engine: codebook not set (tsom_set_codebook)");
        ensure_topo(eng);
        // the Gram alone (kind 0: no graph)
        tsom::launch_gram_only(eng->w.as<float>(), eng->P, eng->D, eng->topo, eng->stream);
        CU(cudaGetLastError());
        CU(cudaMemcpyAsync(out, eng->topo.d2, (size_t)eng->P * eng->P * sizeof(double),
                           cudaMemcpyDeviceToHost, eng->stream));
        CU(cudaStreamSynchronize(eng->stream));
    });
}

}  // extern "C"

namespace {
// run the device sampler; true = identity selection (all rows), else the
// selection is in eng->sampler.sel (device), m rows
bool sampler_pick(Engine* eng, uint64_t* m) {
    tsom::NvtxRange nv("tsom.sampler_select");
    tsom::SamplerState& smp = eng->sampler;
    REQUIRE(smp.n == eng->n_rows, TSOM_ERR_INVALID,
            "sampler: bound data changed since tsom_sampler_init");
    CU(smp.sel.ensure(std::max<uint64_t>(smp.n, 1) * sizeof(uint32_t)));
    const int rc = tsom::sampler_select(smp, smp.sel.as<uint32_t>(), m, eng->sm_count, eng->stream);
    CU(cudaGetLastError());
    if (rc == 5) {
        if (eng->last_error.rfind("reduce barrier timed out", 0) == 0)
            throw tsom::Fail{TSOM_ERR_TIMEOUT};
        if (eng->last_error.rfind("nccl", 0) != 0) eng->last_error = "nccl: allreduce failed (sampler)";
        throw tsom::Fail{TSOM_ERR_NCCL};
    }
    REQUIRE(rc == 0 || rc == -1, TSOM_ERR_CUDA, "sampler: device allocation failed");
    smp.identity = rc == -1;
    smp.last_m = *m;
    return smp.identity;
}

__global__ void k_iota(uint32_t* out, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = (uint32_t)i;
}

void fill_identity(Engine* eng, uint64_t n) {
    tsom::SamplerState& smp = eng->sampler;
    CU(smp.sel.ensure(std::max<uint64_t>(n, 1) * sizeof(uint32_t)));
    TSOM_LAUNCH(k_iota<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 4096), 256, 0, eng->stream>>>(
        smp.sel.as<uint32_t>(), n));
}
}  // namespace

// In-process rank group (tsom_group_*): ranks are engines driven from separate
// host threads of one process (one engine per GPU, or several engines on one
// GPU in the tests); a reduce goes through host memory with a
// generation barrier.  Every rank's contribution is kept and the reduction is
// evaluated in rank order by the last rank to arrive, so the f64 sums are the
// same on every rank and from run to run (the ordered reduce of
// parallel.hpp:90-95).  A rank that does not arrive within the barrier timeout
// is named, like collect_with_barrier (parallel.hpp:67-86).  This is the
// ThreadedExecutor shape (parallel.hpp:99-140) with engines as workers; it
// also lets the multi-rank epoch and the sharded sampler run on one GPU.
struct LoopbackGroup {
    int world;
    std::mutex mu;
    std::condition_variable cv;
    std::vector<std::vector<uint8_t>> contrib;
    std::vector<char> present;
    std::vector<uint8_t> result;
    int arrived = 0, leaving = 0;
    uint64_t gen = 0;
    bool broken = false;
    explicit LoopbackGroup(int w) : world(w), contrib(w), present(w, 0) {}

    template <typename T, typename F>
    void fold(size_t count, F f) {
        result = contrib[0];
        T* acc = reinterpret_cast<T*>(result.data());
        for (int r = 1; r < world; ++r) {
            const T* v = reinterpret_cast<const T*>(contrib[r].data());
            for (size_t i = 0; i < count; ++i) acc[i] = f(acc[i], v[i]);
        }
    }
    // In-place reduce of `bytes` host bytes (op as Engine::comm_reduce).
    // Returns -1 on success, -2 if the group was broken by another rank's
    // timeout, else the first rank that did not arrive in time.
    int reduce(int rank, void* data, size_t bytes, int op, double timeout_s) {
        using clk = std::chrono::steady_clock;
        const auto deadline =
            clk::now() + std::chrono::duration_cast<clk::duration>(std::chrono::duration<double>(timeout_s));
        std::unique_lock<std::mutex> lk(mu);
        // previous round fully drained
        if (!cv.wait_until(lk, deadline, [&] { return leaving == 0 || broken; })) {
            broken = true;
            cv.notify_all();
            return -2;
        }
        if (broken) return -2;
        const uint8_t* src = static_cast<const uint8_t*>(data);
        contrib[rank].assign(src, src + bytes);
        present[rank] = 1;
        const uint64_t my_gen = gen;
        if (++arrived == world) {
            const size_t count = bytes / (op == 0 ? 4 : 8);
            switch (op) {
                case 0: fold<uint32_t>(count, [](uint32_t a, uint32_t b) { return a + b; }); break;
                case 1: fold<uint64_t>(count, [](uint64_t a, uint64_t b) { return a > b ? a : b; }); break;
                case 2: fold<uint64_t>(count, [](uint64_t a, uint64_t b) { return a + b; }); break;
                case 4: fold<int64_t>(count, [](int64_t a, int64_t b) { return a + b; }); break;
                default: fold<double>(count, [](double a, double b) { return a + b; }); break;
            }
            arrived = 0;
            leaving = world;
            std::fill(present.begin(), present.end(), 0);
            ++gen;
            cv.notify_all();
        } else if (!cv.wait_until(lk, deadline, [&] { return gen != my_gen || broken; })) {
            int late = 0;
            while (late < world && present[late]) ++late;
            broken = true;
            cv.notify_all();
            return late;
        }
        if (gen == my_gen) return -2;  // broken while waiting
        std::memcpy(data, result.data(), bytes);
        if (--leaving == 0) cv.notify_all();
        return -1;
    }
};

namespace {
// the reduce hook of an engine joined to a loopback group: device buffer ->
// host, group reduce (with the barrier deadline), host -> device
void attach_loopback(Engine* eng, LoopbackGroup* g, int rank) {
    REQUIRE(rank >= 0 && rank < g->world, TSOM_ERR_INVALID, "comm: bad rank/world");
    eng->world = g->world;
    eng->rank = rank;
    eng->comm_reduce = [eng, g, rank](void* buf, size_t count, int op) -> int {
        cudaStream_t st = eng->stream;
        const size_t bytes = count * (op == 0 ? 4 : 8);
        std::vector<uint8_t> raw(bytes);
        if (cudaMemcpyAsync(raw.data(), buf, bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess) {
            eng->last_error = "cuda: reduce staging failed";
            return TSOM_ERR_CUDA;
        }
        const auto t0 = std::chrono::steady_clock::now();
        const int late = g->reduce(rank, raw.data(), bytes, op, eng->barrier_timeout_s);
        eng->barrier_wait_s +=
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (late >= 0) {
            eng->last_error = "reduce barrier timed out after " +
                              std::to_string(eng->barrier_timeout_s) + " s waiting for worker " +
                              std::to_string(late);
            return TSOM_ERR_TIMEOUT;
        }
        if (late == -2) {
            eng->last_error = "reduce barrier aborted: another rank timed out";
            return TSOM_ERR_TIMEOUT;
        }
        if (cudaMemcpyAsync(buf, raw.data(), bytes, cudaMemcpyHostToDevice, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess) {
            eng->last_error = "cuda: reduce staging failed";
            return TSOM_ERR_CUDA;
        }
        return TSOM_OK;
    };
    tsom::SamplerState& smp = eng->sampler;
    smp.loopback = true;
    smp.world = g->world;
    smp.rank = rank;
    smp.allreduce = [eng](void* buf, size_t count, int op) {
        return eng->comm_reduce && eng->comm_reduce(buf, count, op) == TSOM_OK;
    };
    smp.sync = nullptr;
}
}  // namespace

extern "C" {

// the handle owns one reference; every joined engine holds another, so the
// group and its engines can be destroyed in any order
int tsom_group_create(int world, tsom_group** out) {
    if (!out || world < 1) return TSOM_ERR_INVALID;
    *out = reinterpret_cast<tsom_group*>(new std::shared_ptr<LoopbackGroup>(
        std::make_shared<LoopbackGroup>(world)));
    return TSOM_OK;
}
int tsom_group_destroy(tsom_group* g) {
    delete reinterpret_cast<std::shared_ptr<LoopbackGroup>*>(g);
    return TSOM_OK;
}
// tests only (not in the public header): one rank's host-side reduce through
// the group, no engine or GPU involved; returns -1 ok, -2 aborted, else the
// late rank
int tsom_debug_group_reduce(tsom_group* g, int rank, void* data, uint64_t bytes, int op,
                            double timeout_s) {
    if (!g) return -3;
    return (*reinterpret_cast<std::shared_ptr<LoopbackGroup>*>(g))->reduce(rank, data, bytes, op,
                                                                           timeout_s);
}

int tsom_group_join(tsom_engine* eng, tsom_group* g, int rank) {
    return guarded(eng, [&] {
        REQUIRE(g, TSOM_ERR_INVALID, "comm: null group");
        REQUIRE(!eng->nccl_comm, TSOM_ERR_INVALID, "comm: engine already has an NCCL communicator");
        const auto& sp = *reinterpret_cast<std::shared_ptr<LoopbackGroup>*>(g);
        attach_loopback(eng, sp.get(), rank);
        eng->group_ref = sp;
    });
}

int tsom_sampler_init(tsom_engine* eng, int kind, uint64_t m, uint64_t seed, double alpha,
                      double beta) {
    return guarded(eng, [&] {
        CU(cudaSetDevice(eng->device));
        CU(cudaStreamSynchronize(eng->stream));  // no queued epoch still uses the old state
        REQUIRE(kind >= 0 && kind <= 2, TSOM_ERR_INVALID, "unknown sampling kind");
        REQUIRE(eng->n_rows >= 1, TSOM_ERR_INVALID, "sampler: N must be >= 1 (bind data first)");
        REQUIRE(kind == 0 || m >= 1, TSOM_ERR_INVALID, "select_random: m must be >= 1");
        REQUIRE(eng->n_rows < (1ull << 31), TSOM_ERR_INVALID, "sampler: N < 2^31");
        tsom::SamplerState& smp = eng->sampler;
        smp.sharded = eng->comm_reduce != nullptr;
        if (smp.sharded) {
            // one Sampler over the ranks' rows in rank order: global N and this
            // rank's first row from an allreduce of the per-rank row counts
            cudaStream_t st = eng->stream;
            smp.world = eng->world;
            smp.rank = eng->rank;
            smp.allreduce = [eng](void* buf, size_t count, int op) {
                return eng->comm_reduce && eng->comm_reduce(buf, count, op) == TSOM_OK;
            };
            if (eng->nccl_comm)
                smp.sync = [eng](cudaStream_t) {
                    try {
                        wait_stream(eng);
                        return true;
                    } catch (const tsom::Fail&) {
                        return false;
                    }
                };
            std::vector<uint64_t> cnt(smp.world, 0);
            cnt[smp.rank] = eng->n_rows;
            CU(smp.slots.ensure((size_t)smp.world * 8));
            CU(cudaMemcpyAsync(smp.slots.p, cnt.data(), cnt.size() * 8, cudaMemcpyHostToDevice, st));
            const int rc = eng->comm_reduce(smp.slots.p, cnt.size(), 2);
            if (rc != TSOM_OK) throw tsom::Fail{rc};
            CU(cudaMemcpyAsync(cnt.data(), smp.slots.p, cnt.size() * 8, cudaMemcpyDeviceToHost, st));
            wait_stream(eng);
            smp.gN = 0;
            smp.off = 0;
            for (int r = 0; r < smp.world; ++r) {
                if (r < smp.rank) smp.off += cnt[r];
                smp.gN += cnt[r];
            }
            REQUIRE(smp.gN < (1ull << 32), TSOM_ERR_INVALID, "sampler: global N < 2^32");
        }
        const int rc = tsom::sampler_setup(smp, kind, eng->n_rows, m, seed, alpha, beta,
                                           eng->sm_count);
        REQUIRE(rc == 0, TSOM_ERR_CUDA, "sampler: device allocation failed");
        CU(cudaDeviceSynchronize());
    });
}

int tsom_sampler_select(tsom_engine* eng, uint32_t* sel_out, uint64_t* m_out) {
    return guarded(eng, [&] {
        CU(cudaSetDevice(eng->device));
        REQUIRE(eng->sampler.kind >= 0, TSOM_ERR_INVALID, "sampler: not initialised");
        uint64_t m = 0;
        const bool ident = sampler_pick(eng, &m);
        if (ident) fill_identity(eng, m);
        uint32_t status = 0;
        CU(cudaMemcpyAsync(&status, eng->sampler.misc.as<uint64_t>() + 1, 4, cudaMemcpyDeviceToHost,
                           eng->stream));
        if (sel_out && m)
            CU(cudaMemcpyAsync(sel_out, eng->sampler.sel.p, m * sizeof(uint32_t),
                               cudaMemcpyDeviceToHost, eng->stream));
        wait_stream(eng);
        REQUIRE(!(status & 4u), TSOM_ERR_NUMERICAL, "sampler: random stream slack exceeded");
        if (m_out) *m_out = m;
    });
}

int tsom_sampler_observe(tsom_engine* eng, const double* dist) {
    return guarded(eng, [&] {
        CU(cudaSetDevice(eng->device));
        tsom::SamplerState& smp = eng->sampler;
        REQUIRE(smp.kind >= 0, TSOM_ERR_INVALID, "sampler: not initialised");
        if (smp.kind != 2) return;
        const uint64_t m = smp.last_m;
        const double* d = eng->dist.as<double>();
        REQUIRE(dist || d || m == 0, TSOM_ERR_INVALID,
                "sampler: no distances to observe (no sampled epoch produced them)");
        if (dist) {
            CU(eng->dist.ensure(std::max<uint64_t>(m, 1) * sizeof(double)));
            CU(cudaMemcpyAsync(eng->dist.p, dist, m * sizeof(double), cudaMemcpyHostToDevice,
                               eng->stream));
            d = eng->dist.as<double>();
        }
        tsom::sampler_observe(smp, smp.sel.as<uint32_t>(), m, d, eng->sm_count, eng->stream);
        CU(cudaStreamSynchronize(eng->stream));
    });
}

int tsom_sampler_state(tsom_engine* eng, double* last_error, uint32_t* age) {
    return guarded(eng, [&] {
        CU(cudaSetDevice(eng->device));
        tsom::SamplerState& smp = eng->sampler;
        REQUIRE(smp.kind == 2, TSOM_ERR_INVALID, "sampler: no adaptive state");
        tsom::sampler_materialize_ages(smp, eng->sm_count, eng->stream);
        if (last_error)
            CU(cudaMemcpyAsync(last_error, smp.err.p, smp.n * sizeof(double),
                               cudaMemcpyDeviceToHost, eng->stream));
        if (age)
            CU(cudaMemcpyAsync(age, smp.age.p, smp.n * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                               eng->stream));
        CU(cudaStreamSynchronize(eng->stream));
    });
}

int tsom_mt_selftest(uint64_t seed, uint64_t jump) { return tsom::mt::selftest(seed, jump); }

int tsom_release_cached_memory(int device) {
    if (cudaSetDevice(device) != cudaSuccess) {
        cudaGetLastError();
        return TSOM_ERR_CUDA;
    }
    cudaDeviceSynchronize();
    tsom::release_cached_memory();
    return TSOM_OK;
}

// One device-resident epoch (tsom_train_epoch), enqueued on the engine stream
// without waiting for it; dead (optional): the multi-epoch failure record.
static void train_epoch_enqueue(Engine* eng, double eta, double sigma, double momentum, uint32_t flags,
                         int* dead, uint32_t epoch) {
    tsom::NvtxRange nv("tsom.train_epoch");
    CU(cudaSetDevice(eng->device));
    REQUIRE(eng->topo_set, TSOM_ERR_INVALID, "train_epoch: topology distance not set");
    REQUIRE(sigma > 0.0, TSOM_ERR_INVALID, "influence_matrix: sigma must be > 0");
    const bool momentum_on = (flags & 1u) != 0;
    // influence(sigma) on the device (topology.hpp:342-364); the device
    // path keys its cache on sigma exactly like influence_cache_key (:399-401)
    const int64_t key = (int64_t)std::llround(sigma * 1e6);
    if (!(eng->infl_set && eng->infl_key == key)) {
        const double inv = 1.0 / (2.0 * sigma * sigma);
        tsom::launch_influence(eng->topo_dist.as<double>(), (size_t)eng->P * eng->P, inv,
                               eng->infl.as<double>(), eng->stream, eng->hmax.as<double>());
        CU(cudaGetLastError());
        eng->infl_key = key;
        eng->infl_set = true;
    }
    prep_codebook(eng);
    // flags bit 1: the device sampler picks this epoch's rows (select ->
    // epoch over them -> observe), sampling.hpp:197-211
    tsom::SamplerState& smp = eng->sampler;
    const bool sampled = (flags & 2u) != 0;
    REQUIRE(!sampled || smp.kind >= 0, TSOM_ERR_INVALID,
            "train_epoch: no device sampler (tsom_sampler_init)");
    uint64_t m = eng->n_rows;
    bool ident = true;
    std::vector<uint32_t> host_sel;
    eng->sample_timed = sampled;
    if (sampled) {
        CU(cudaEventRecord(eng->ev[11], eng->stream));
        ident = sampler_pick(eng, &m);
        if (!ident && eng->streamed) {
            host_sel.resize(m);
            CU(cudaMemcpyAsync(host_sel.data(), smp.sel.p, m * sizeof(uint32_t),
                               cudaMemcpyDeviceToHost, eng->stream));
            wait_stream(eng);
        }
    }
    const bool want_dist = sampled && smp.kind == 2;
    if (ident)
        accumulate_epoch(eng, nullptr, eng->n_rows, want_dist, false, true);
    else if (eng->streamed)
        accumulate_epoch(eng, host_sel.data(), m, want_dist, false, true);
    else
        accumulate_epoch(eng, nullptr, m, want_dist, false, true, smp.sel.as<uint32_t>());
    if (want_dist) {
        if (ident) fill_identity(eng, eng->n_rows);
        tsom::sampler_observe(smp, ident ? smp.sel.as<uint32_t>() : smp.sel.as<uint32_t>(), m,
                              eng->dist.as<double>(), eng->sm_count, eng->stream);
    }
    smooth(eng, eta);
    // the term guard on this epoch's rows and codebook; a violation records
    // the failure before the update, which then leaves the weights as they
    // were (the reference throws out of run_iteration, trainer.hpp:506)
    // (apply_update's fault slot was reset by the smoothing's last kernel)
    eng->last_guard_tag = enqueue_term_guard(eng, eta, dead, epoch);
    tsom::launch_apply_update_guarded(eng->w.as<float>(), eng->prev.as<float>(), eng->P,
                                      eng->D, eng->U.as<double>(), eng->H.as<double>(),
                                      momentum_on, momentum, eng->status.as<int>(), dead,
                                      eng->stream);
    CU(cudaGetLastError());
    CU(cudaEventRecord(eng->ev[10], eng->stream));
    eng->update_timed = true;
    eng->codebook_prepped = false;
    prep_codebook(eng);
}

int tsom_train_epoch(tsom_engine* eng, double eta, double sigma, double momentum, uint32_t flags) {
    return guarded(eng, [&] {
        CU(cudaSetDevice(eng->device));
        CU(eng->dead.ensure(4 * sizeof(int)));
        CU(cudaMemsetAsync(eng->dead.p, 0, 4 * sizeof(int), eng->stream));
        train_epoch_enqueue(eng, eta, sigma, momentum, flags, eng->dead.as<int>(), 0);
        CU(cudaMemcpyAsync(eng->hstat + 2, eng->status.p, sizeof(int), cudaMemcpyDeviceToHost,
                           eng->stream));
        enqueue_guard_read(eng);
        wait_stream(eng);
        int st;
        std::memcpy(&st, eng->hstat + 2, sizeof(int));
        finish_recheck(eng);
        record_timing(eng);
        check_term_guard(eng, eng->last_guard_tag);  // the update was skipped
        REQUIRE(st == INT_MAX, TSOM_ERR_NUMERICAL,
                "numerical fault: non-finite weight update at node " + std::to_string(st));
    });
}

int tsom_train_epochs(tsom_engine* eng, uint32_t n_epochs, const double* eta,
                      const double* sigma, double momentum, uint32_t flags,
                      uint32_t* failed_epoch) {
    return guarded(eng, [&] {
        CU(cudaSetDevice(eng->device));
        REQUIRE(n_epochs >= 1 && eta && sigma, TSOM_ERR_INVALID,
                "train_epochs: need n >= 1 and eta / sigma arrays");
        if (failed_epoch) *failed_epoch = UINT32_MAX;
        CU(eng->dead.ensure(4 * sizeof(int)));
        CU(cudaMemsetAsync(eng->dead.p, 0, 4 * sizeof(int), eng->stream));
        while (eng->k1_ev.size() < 2 * (size_t)n_epochs) {
            cudaEvent_t ev;
            CU(cudaEventCreate(&ev));
            eng->k1_ev.push_back(ev);
        }
        while (eng->acc_ev.size() < 2 * (size_t)n_epochs) {
            cudaEvent_t ev;
            CU(cudaEventCreate(&ev));
            eng->acc_ev.push_back(ev);
        }
        int* dead = eng->dead.as<int>();
        struct SlotReset {
            Engine* e;
            ~SlotReset() {
                e->k1_slot = -1;
                e->defer_hstat = false;
                e->epochs_left = 0;
            }
        } reset{eng};
        for (uint32_t t = 0; t < n_epochs; ++t) {
            eng->k1_slot = (int)t;
            eng->k1_timed = false;
            eng->defer_hstat = t + 1 < n_epochs;
            eng->epochs_left = n_epochs - t;
            train_epoch_enqueue(eng, eta[t], sigma[t], momentum, flags, dead, t);
            tsom::launch_epoch_guard(eng->status.as<int>(), t, dead, eng->stream);
            CU(cudaGetLastError());
        }
        const bool k1_all = eng->k1_timed;  // every epoch ran the tcgen05 main pass
        eng->k1_slot = -1;
        CU(cudaMemcpyAsync(eng->hstat + 5, dead, 3 * sizeof(int), cudaMemcpyDeviceToHost,
                           eng->stream));
        wait_stream(eng);
        finish_recheck(eng);
        eng->k1_timed = false;  // ev[8] / ev[9] were not recorded: per-epoch events below
        record_timing(eng);     // phases of the last epoch
        eng->t_k1 = 0.0f;
        if (k1_all) {
            float sum = 0.0f;
            for (uint32_t t = 0; t < n_epochs; ++t) {
                float ms = 0.0f;
                cudaEventElapsedTime(&ms, eng->k1_ev[2 * (size_t)t], eng->k1_ev[2 * (size_t)t + 1]);
                sum += ms;
            }
            eng->t_k1 = sum / (float)n_epochs;  // mean main-pass K1 time of the call
            cudaGetLastError();  // a timing query is never an error of the epochs
        }
        eng->t_accum_mean = 0.0f;
        if (!eng->streamed) {
            float sum = 0.0f;
            for (uint32_t t = 0; t < n_epochs; ++t) {
                float ms = 0.0f;
                cudaEventElapsedTime(&ms, eng->acc_ev[2 * (size_t)t], eng->acc_ev[2 * (size_t)t + 1]);
                sum += ms;
            }
            eng->t_accum_mean = sum / (float)n_epochs;  // mean accumulation phase of the call
            cudaGetLastError();
        }
        int rec[3];
        std::memcpy(rec, eng->hstat + 5, sizeof(rec));
        if (rec[0]) {
            if (failed_epoch) *failed_epoch = (uint32_t)(rec[0] - 1);
            REQUIRE(rec[1] != 1, TSOM_ERR_NUMERICAL,
                    "numerical fault: non-finite weight update at node " + std::to_string(rec[2]) +
                        " (epoch " + std::to_string(rec[0] - 1) + ")");
            REQUIRE(false, TSOM_ERR_NUMERICAL,
                    "numerical fault: accumulation term out of range (|term| >= 2^22) (epoch " +
                        std::to_string(rec[0] - 1) + ")");
        }
    });
}

uint64_t tsom_last_recheck_count(const tsom_engine* eng) { return eng ? eng->last_recheck : 0; }

// diagnostics only (not in the public header): the device buffer (bound rows x
// groups * group width floats) K1's main pass writes its raw values into
// while option 99 bit 7 is set
int tsom_debug_k1_dump(float* d_buf) { return tsom::k1_set_dump(d_buf); }

// diagnostics only (not in the public header): K1 timestamps of CTA 0
int tsom_debug_k1_trace(unsigned long long* out, uint32_t n) {
    return tsom::k1_trace_copy(out, n);
}

// diagnostics only (not in the public header): copy an internal device buffer
// (0 xsplit, 1 xn2, 2 wsplit, 3 scale, 4 part, 5 gsplit, 6 gxn2, 7 w2max,
// 8 x2max, 9 ties, 10 bmu (per position), 11 perm) to the host; returns the
// bytes copied
int64_t tsom_debug_read(tsom_engine* eng, int which, void* out, uint64_t bytes) {
    if (!eng) return -1;
    cudaSetDevice(eng->device);
    tsom::DevBuf* bufs[] = {&eng->xsplit, &eng->xn2, &eng->wsplit, &eng->scale, &eng->part,
                            &eng->gsplit, &eng->gxn2, &eng->w2max, &eng->x2max, &eng->ties,
                            &eng->bmu, &eng->perm};
    if (which < 0 || which >= (int)(sizeof(bufs) / sizeof(bufs[0]))) return -1;
    const uint64_t nb = std::min<uint64_t>(bytes, bufs[which]->bytes);
    cudaStreamSynchronize(eng->stream);
    if (nb && cudaMemcpy(out, bufs[which]->p, nb, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    return (int64_t)nb;
}

int tsom_active_bmu_kernel(const tsom_engine* eng) {
    if (!eng) return 0;
    const int k = tc_kind(eng);
    return k == tsom::kTcF16 ? 3 : (k == tsom::kTcTf32 ? 2 : 1);
}

int tsom_comm_unique_id(tsom_engine* eng, uint8_t id_out[128]) {
    return guarded(eng, [&] {
        std::string err;
        REQUIRE(g_nccl.load(err), TSOM_ERR_NCCL, err);
        ncclUniqueId id;
        ncclResult_t r = g_nccl.getUniqueId(&id);
        REQUIRE(r == ncclSuccess, TSOM_ERR_NCCL, "nccl: ncclGetUniqueId failed");
        static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
        std::memcpy(id_out, &id, 128);
    });
}

int tsom_comm_init(tsom_engine* eng, const uint8_t id[128], int rank, int world) {
    return guarded(eng, [&] {
        CU(cudaSetDevice(eng->device));
        REQUIRE(world >= 1 && rank >= 0 && rank < world, TSOM_ERR_INVALID, "comm: bad rank/world");
        std::string err;
        REQUIRE(g_nccl.load(err), TSOM_ERR_NCCL, err);
        ncclUniqueId uid;
        std::memcpy(&uid, id, 128);
        // non-blocking communicator: initialisation and every reduce can be
        // polled against the barrier deadline and aborted (ncclCommAbort)
        // when a peer never arrives, instead of blocking forever
        ncclComm_t comm = nullptr;
        ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
        cfg.blocking = 0;
        ncclResult_t r = g_nccl.commInitRankConfig(&comm, world, uid, rank, &cfg);
        using clk = std::chrono::steady_clock;
        const auto t0 = clk::now();
        while (r == ncclInProgress) {
            if (std::chrono::duration<double>(clk::now() - t0).count() > eng->barrier_timeout_s) {
                g_nccl.commAbort(comm);
                REQUIRE(false, TSOM_ERR_TIMEOUT,
                        "comm init timed out after " + barrier_seconds(eng->barrier_timeout_s) +
                            " s waiting for the other ranks of " + std::to_string(world));
            }
            std::this_thread::sleep_for(std::chrono::microseconds(200));
            g_nccl.getAsyncError(comm, &r);
        }
        REQUIRE(r == ncclSuccess, TSOM_ERR_NCCL,
                std::string("nccl: ncclCommInitRankConfig failed: ") +
                    (g_nccl.errStr ? g_nccl.errStr(r) : "?"));
        eng->nccl_comm = comm;
        eng->rank = rank;
        eng->world = world;
        eng->comm_reduce = [eng, comm](void* buf, size_t count, int op) -> int {
            const ncclDataType_t t =
                op == 0 ? ncclUint32 : (op == 3 ? ncclFloat64 : (op == 4 ? ncclInt64 : ncclUint64));
            const ncclRedOp_t o = op == 1 ? ncclMax : ncclSum;
            ncclResult_t rr = g_nccl.allReduce(buf, buf, count, t, o, comm, eng->stream);
            // a non-blocking communicator may still be enqueueing the call
            while (rr == ncclInProgress) {
                std::this_thread::yield();
                g_nccl.getAsyncError(comm, &rr);
            }
            if (rr != ncclSuccess) {
                eng->last_error = std::string("nccl: allreduce failed: ") +
                                  (g_nccl.errStr ? g_nccl.errStr(rr) : "?");
                return TSOM_ERR_NCCL;
            }
            // the barrier of this reduce: wait_stream polls it with the deadline
            if (eng->red_pending == eng->red_ev.size()) {
                cudaEvent_t ev;
                if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
                    eng->last_error = "cuda: event creation failed";
                    return TSOM_ERR_CUDA;
                }
                eng->red_ev.push_back(ev);
            }
            if (cudaEventRecord(eng->red_ev[eng->red_pending], eng->stream) != cudaSuccess) {
                eng->last_error = "cuda: event record failed";
                return TSOM_ERR_CUDA;
            }
            ++eng->red_pending;
            return TSOM_OK;
        };
    });
}

double tsom_barrier_wait_s(const tsom_engine* eng) { return eng ? eng->barrier_wait_s : 0.0; }

int tsom_last_timing(const tsom_engine* eng, float* bmu_ms, float* accum_ms, float* smooth_ms,
                     float* total_ms) {
    if (!eng) return TSOM_ERR_INVALID;
    if (bmu_ms) *bmu_ms = eng->t_bmu;
    if (accum_ms) *accum_ms = eng->t_accum;
    if (smooth_ms) *smooth_ms = eng->t_smooth;
    if (total_ms) *total_ms = eng->t_total;
    return TSOM_OK;
}

int tsom_last_timing_detail(const tsom_engine* eng, float out[8]) {
    if (!eng || !out) return TSOM_ERR_INVALID;
    const float v[8] = {eng->t_k1,    eng->t_bmu,    eng->t_accum,  eng->t_smooth,
                        eng->t_update, eng->t_total, eng->t_sample, eng->t_accum_mean};
    std::memcpy(out, v, sizeof(v));
    return TSOM_OK;
}

uint64_t tsom_kernel_launches(void) { return tsom::g_launches.load(); }

uint64_t tsom_device_bytes(const tsom_engine* e) {
    if (!e) return 0;
    Engine* eng = const_cast<tsom_engine*>(e);
    uint64_t total = 0;
    for (const DevBuf* b : all_buffers(eng))
        if (b->owned) total += b->bytes;
    const tsom::SamplerState& s = eng->sampler;
    for (const DevBuf* b : {&s.window, &s.jp, &s.gwin, &s.misc, &s.seqb[0], &s.seqb[1],
                            &s.drawsb[0], &s.drawsb[1], &s.tailb[0], &s.tailb[1], &s.err, &s.age,
                            &s.keys, &s.hist, &s.cand, &s.ccnt, &s.first, &s.tidx, &s.bitmap,
                            &s.bcount, &s.sel, &s.jN, &s.glist, &s.slots})
        total += b->bytes;
    return total;
}

void* tsom_stream(tsom_engine* eng) { return eng ? (void*)eng->stream : nullptr; }

}  // extern "C"
