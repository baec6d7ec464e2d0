// host_staging.cu — host side of the out-of-core and pageable-row paths:
// FSOMSHRD reads, a process-wide cache of pinned staging blocks, and the
// persistent worker pool that fills them while the copy engine drains the
// other slot.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "capi_internal.h"

namespace tsom {
namespace host {

using tsom::Fail;

// Host side of one streamed chunk [r0, r1): returns a host pointer the copy
// engine can DMA from.  Registered caller memory is used in place; shard files
// (pread) and pageable caller memory go through the two pinned staging
// buffers, reusing slot s only after its previous H2D has completed.
void close_shards(Engine* eng) {
    for (auto& f : eng->shards)
        if (f.fd >= 0) ::close(f.fd);
    eng->shards.clear();
}

// Pinned staging blocks are cached process-wide (cudaMallocHost of tens of MB
// costs tens of ms): engines take a block at least as large as they need and
// return it on destroy.
struct PinnedBlock {
    void* p;
    size_t bytes;
};
static std::mutex g_pinned_mu;
static std::vector<PinnedBlock> g_pinned_free;

cudaError_t pinned_take(size_t bytes, void** out, size_t* got) {
    {
        std::lock_guard<std::mutex> lk(g_pinned_mu);
        for (size_t i = 0; i < g_pinned_free.size(); ++i)
            if (g_pinned_free[i].bytes >= bytes) {
                *out = g_pinned_free[i].p;
                *got = g_pinned_free[i].bytes;
                g_pinned_free.erase(g_pinned_free.begin() + (std::ptrdiff_t)i);
                return cudaSuccess;
            }
    }
    *got = bytes;
    return cudaMallocHost(out, bytes);
}

void pinned_give(void* p, size_t bytes) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    g_pinned_free.push_back({p, bytes});
    if (g_pinned_free.size() > 8) {  // bound the cache: drop the oldest
        cudaFreeHost(g_pinned_free.front().p);
        g_pinned_free.erase(g_pinned_free.begin());
    }
}

void ensure_pinned(Engine* eng, uint64_t rows) {
    if (eng->pinned_rows >= rows && eng->pinned[0]) return;
    for (int s = 0; s < 2; ++s) {
        if (eng->pin_busy[s]) CU(cudaEventSynchronize(eng->ev_pin[s]));
        pinned_give(eng->pinned[s], eng->pinned_bytes[s]);
        eng->pinned[s] = nullptr;
        void* p = nullptr;
        CU(pinned_take(rows * eng->D * sizeof(float), &p, &eng->pinned_bytes[s]));
        eng->pinned[s] = static_cast<float*>(p);
        if (!eng->ev_pin[s]) CU(cudaEventCreateWithFlags(&eng->ev_pin[s], cudaEventDisableTiming));
        eng->pin_busy[s] = false;
    }
    eng->pinned_rows = rows;
}

// returns "" or the failing shard's error message (called from staging threads)
std::string read_shard_rows(const Engine* eng, uint64_t r0, uint64_t r1, float* dst) {
    const size_t rowb = (size_t)eng->D * sizeof(float);
    for (const auto& f : eng->shards) {
        const uint64_t a = std::max(r0, f.row0), b = std::min(r1, f.row0 + f.rows);
        if (a >= b) continue;
        char* out = reinterpret_cast<char*>(dst + (a - r0) * eng->D);
        size_t left = (b - a) * rowb;
        off_t off = (off_t)(24 + (a - f.row0) * rowb);
        while (left) {
            const ssize_t got = ::pread(f.fd, out, left, off);
            if (got <= 0) return "shard read failed: " + f.path;
            out += got;
            off += got;
            left -= (size_t)got;
        }
    }
    return std::string();
}

// Persistent host workers for the staging fills (a fork-join per chunk;
// spawning threads per chunk cost ~1 ms of every 32-MB chunk).  The calling
// thread works too; concurrent callers (engines on several threads) take
// turns.  Workers only copy host memory / read files.
class StagingPool {
public:
    explicit StagingPool(unsigned n) {
        for (unsigned i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
    }
    void run(uint32_t n, const std::function<void(uint32_t)>& fn) {
        std::lock_guard<std::mutex> turn(run_mu_);
        std::unique_lock<std::mutex> lk(mu_);
        job_ = &fn;
        njobs_ = n;
        next_ = 0;
        finished_ = 0;
        ++gen_;
        cv_.notify_all();
        while (next_ < njobs_) {
            const uint32_t i = next_++;
            lk.unlock();
            fn(i);
            lk.lock();
            ++finished_;
        }
        done_.wait(lk, [&] { return finished_ == njobs_; });
        job_ = nullptr;
    }

private:
    void loop() {
        std::unique_lock<std::mutex> lk(mu_);
        uint64_t seen = 0;
        for (;;) {
            cv_.wait(lk, [&] { return gen_ != seen && job_ && next_ < njobs_; });
            seen = gen_;
            while (job_ && next_ < njobs_) {
                const uint32_t i = next_++;
                const std::function<void(uint32_t)>* fn = job_;
                lk.unlock();
                (*fn)(i);
                lk.lock();
                if (++finished_ == njobs_) done_.notify_all();
            }
        }
    }
    std::mutex run_mu_, mu_;
    std::condition_variable cv_, done_;
    std::vector<std::thread> workers_;
    const std::function<void(uint32_t)>* job_ = nullptr;
    uint32_t njobs_ = 0, next_ = 0, finished_ = 0;
    uint64_t gen_ = 0;
};

StagingPool& staging_pool() {
    // leaked on purpose: blocked workers need no joining at process exit
    static StagingPool* pool =
        new StagingPool(std::max(1u, std::min(16u, std::thread::hardware_concurrency())) - 1);
    return *pool;
}

const float* host_chunk_source(Engine* eng, uint64_t r0, uint64_t r1, int s) {
    if (eng->shards.empty() && eng->host_direct) return eng->host_rows + r0 * eng->D;
    ensure_pinned(eng, std::max<uint64_t>(r1 - r0, eng->pinned_rows));
    if (eng->pin_busy[s]) CU(cudaEventSynchronize(eng->ev_pin[s]));
    float* dst = eng->pinned[s];
    // one host thread streams ~10 GB/s; split the fill so staging keeps up
    // with the PCIe copy engine
    auto fill = [&](uint64_t a, uint64_t b) -> std::string {
        if (!eng->shards.empty()) return read_shard_rows(eng, a, b, dst + (a - r0) * eng->D);
        std::memcpy(dst + (a - r0) * eng->D, eng->host_rows + a * eng->D,
                    (b - a) * eng->D * sizeof(float));
        return std::string();
    };
    const uint64_t bytes = (r1 - r0) * eng->D * sizeof(float);
    static const uint32_t host_threads = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const uint32_t T = (uint32_t)std::min<uint64_t>(eng->staging_threads ? eng->staging_threads
                                                                         : host_threads,
                                                    std::max<uint64_t>(1, bytes >> 22));
    if (T <= 1) {
        const std::string e = fill(r0, r1);
        REQUIRE(e.empty(), TSOM_ERR_NUMERICAL, e);
    } else {
        std::vector<std::string> errs(T);
        const uint64_t per = (r1 - r0 + T - 1) / T;
        staging_pool().run(T, [&](uint32_t t) {
            const uint64_t a = std::min(r1, r0 + t * per), b = std::min(r1, a + per);
            errs[t] = fill(a, b);
        });
        for (const auto& e : errs) REQUIRE(e.empty(), TSOM_ERR_NUMERICAL, e);
    }
    return dst;
}

void note_pinned_copy(Engine* eng, int s) {
    if (eng->shards.empty() && eng->host_direct) return;
    CU(cudaEventRecord(eng->ev_pin[s], eng->copy_stream));
    eng->pin_busy[s] = true;
}

// Copy rows [0, total) of the bound host source (shard files or caller rows)
// into eng->x: staging threads fill one pinned slot while the copy engine
// drains the other.
}  // namespace host
}  // namespace tsom
