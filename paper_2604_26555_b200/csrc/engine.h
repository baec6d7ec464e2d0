// engine.h — internal state of the B200 batch-SOM epoch engine.
//
// Data layout in HBM:
//   x        n_rows x d   f32 row-major   bound samples (resident mode)
//   xs       tiles of 128 rows, [hi|lo] x [14 k-cores][128 rows][4 f32]
//            pre-split TF32 operands for the tcgen05 BMU kernel (k1_bmu_tc.cu)
//   w        P x d        f32             codebook (updated in place by the
//                                         device-resident loop)
//   wt       (d+1) x Ppad f32             SIMT operand: -2 w^T and ||w||^2 row
//   ws       ceil(P/gn) groups of [hi|lo] x [14][gn][4] f32  tcgen05 B operand (gn <= 256)
//   infl     P x P        f64             influence h[b][j]
//   sorted   n u32                        row positions in BMU order (counting sort)
//   partial  pieces x (d+1) f64           per-piece (<= 256 rows) FP64 row sums
//   sums     P*d + P + 2  f64             reduced [S | c | sum dist | count]
//                                         (the one allreduce buffer)
//   U, H     P*d, P       f64             smoothed accumulators (K3 output)
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "../../include/tsom_b200.h"

namespace tsom {

// Kernel launches issued by this library (tsom_kernel_launches): the bench
// reports it so a silent host fallback would be visible.
extern std::atomic<uint64_t> g_launches;
#define TSOM_LAUNCH(...) (++::tsom::g_launches, __VA_ARGS__)

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    bool owned = true;
    cudaError_t ensure(size_t need);
    void release(bool synced = false);  // synced: the device is known idle
    // stream-ordered variants (no synchronisation): the block is usable by
    // work queued on st after the call / returned once st's queued work is done
    cudaError_t ensure_on(size_t need, cudaStream_t st);
    void release_on(cudaStream_t st);
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

void release_cached_memory();  // trim the device pool DevBuf allocates from
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize, >= bytes) once per (kernel, device)
// (newly_set: true when this call set it, i.e. first use on this device)
cudaError_t ensure_smem_attr(const void* func, size_t bytes, bool* newly_set = nullptr);

// Host-to-device copy that is complete on return.  cudaMemcpy from pageable
// memory may return once the data is staged, before the DMA lands; kernels on
// the engine's non-blocking streams are not ordered after it.
inline cudaError_t h2d_blocking(void* dst, const void* src, size_t bytes) {
    cudaError_t e = cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaStreamSynchronize(0);
    return e;
}

struct Error {
    int code;
    std::string msg;
};

// Threshold for the exact FP64 re-check of near-ties (see k1 kernels):
// a row is re-scanned when second_best - best <= tau * (max||x||^2 + max||w||^2).
constexpr double kDefaultTauSimt = 1.0 / 65536.0;   // 2^-16
constexpr double kDefaultTauTc = 1.0 / 16384.0;     // 2^-14 (3xTF32 error is larger)

constexpr int kTcTileM = 128;   // samples per tcgen05 tile (TMEM lanes)
constexpr int kTcGroupN = 256;  // nodes per CTA-resident codebook group
constexpr int kTcKPad = 56;     // tf32 operand: d + 3 augmented columns padded to 7 k-steps
constexpr uint32_t kTcF16MaxK = 192;  // f16 operand: 3d + 5 columns padded to 16 (d <= 62)
constexpr uint32_t kCandOverflow = 15u;  // enumerate pass: > 8 candidates in a group

// Tensor-core operand encodings of K1 (k1_bmu_tc.cu)
enum TcKind : int { kTcNone = 0, kTcTf32 = 1, kTcF16 = 2 };
struct TcGeom {
    int kind;
    uint32_t kpad;        // K elements per row (tf32: per half)
    uint32_t ksteps;      // MMA k-steps (tf32: x3 products each)
    uint32_t tile_bytes;  // one 128-row A tile
    uint32_t row_bytes;   // one node row of the B operand
};
__host__ __device__ inline TcGeom tc_geom(int kind, uint32_t D) {
    TcGeom g{kind, 0, 0, 0, 0};
    if (kind == kTcTf32) {
        g.kpad = kTcKPad;
        g.ksteps = kTcKPad / 8;
        g.tile_bytes = 2u * kTcTileM * kTcKPad * 4u;
        g.row_bytes = 2u * kTcKPad * 4u;
    } else if (kind == kTcF16) {
        g.kpad = (3u * D + 5u + 15u) / 16u * 16u;
        g.ksteps = g.kpad / 16u;
        g.tile_bytes = kTcTileM * g.kpad * 2u;
        g.row_bytes = g.kpad * 2u;
    }
    return g;
}

// Error window of the tensor-core BMU values (scaled units, S = s^2): a row whose
// computed best/second-best gap exceeds
//   thr = tau S (||x||^2 + max||w||^2) + abs_coef (sqrt(S ||x||^2) + 2 sqrt(S max||w||^2))
// has a unique exact argmin equal to the computed one.  The row
// part (tie_xpart) is computed once per split row and stored in place of
// ||x||^2; the codebook part (tie_wpart) once per kernel.
struct TieWin {
    float tau;       // relative bound of the split-precision products + FP32 accumulation
    float abs_coef;  // absolute floor (FP16 subnormal spacing): 2^-24 sqrt(d), 0 for tf32
    float quant;     // (unused: every epilogue compares raw values)
};
__host__ __device__ inline float tie_sqrt_up(float v) {
    return v > 0.0f ? sqrtf(v) * 1.000001f : 0.0f;
}
// both parts rounded up (the window only has to be an upper bound)
__host__ __device__ inline float tie_xpart(float xn2, float S, TieWin w) {
    return (w.tau * S * xn2 + w.abs_coef * tie_sqrt_up(S * xn2)) * 1.000001f;
}
__host__ __device__ inline float tie_wpart(float w2max, float S, TieWin w) {
    return (w.tau * S * w2max + 2.0f * w.abs_coef * tie_sqrt_up(S * w2max)) * 1.000001f;
}

// K2: counting sort by BMU + per-piece FP64 gather accumulation (k_accum.cu).
struct AccumScratch {
    uint32_t* counts = nullptr;      // [nblk][P] histograms -> offsets
    uint32_t* totals = nullptr;      // [P]
    uint32_t* node_start = nullptr;  // [P+1]
    uint32_t* piece_start = nullptr; // [P+1]
    uint32_t* piece_node = nullptr;  // [pieces]
    uint32_t* sorted = nullptr;      // [n] positions in BMU order
    double* partial = nullptr;       // [pieces][d+1]
};
// Topology refresh scratch (k_topology.cu), P x P arrays on the device.
struct TopoScratch {
    double* norms = nullptr;   // [P]
    double* d2 = nullptr;      // [P*P] pairwise squared distances (FP64 Gram)
    uint32_t* comp = nullptr;  // [P]
    double* bw = nullptr;      // [2P]
    uint32_t* ba = nullptr;    // [2P]
    uint32_t* bb = nullptr;    // [2P]
    uint8_t* keep = nullptr;   // [P*P] edge mask (a < b)
    uint32_t* rowcnt = nullptr;// [P]
    uint32_t* edges = nullptr; // [P*(P-1)] (i, j) pairs, lexicographic
    uint32_t* ne = nullptr;    // [1]
    uint32_t* deg = nullptr;   // [P+1] CSR offsets
    uint32_t* adj = nullptr;   // [2 * edges]
    uint16_t* hops = nullptr;  // [P*P]
    double* hopd = nullptr;    // [P*P] hop counts widened (influence input)
    uint32_t* status = nullptr;// bit0 disconnected, bit1 edge out of range
};
// refresh_topology (topology.hpp:439-451) for kind 2 (MST) / 3 (RNG)
int launch_refresh_topology(const float* w, uint32_t P, uint32_t D, int kind, TopoScratch& s,
                            cudaStream_t st);
void launch_gram_only(const float* w, uint32_t P, uint32_t D, TopoScratch& s, cudaStream_t st);

// Device sampler (k_sampler.cu, sampling.hpp:183-221)
struct SamplerState {
    int kind = -1;  // -1 none, 0 full, 1 random, 2 adaptive
    uint64_t n = 0, m = 0;
    double alpha = 1.0, beta = 1.0;
    uint64_t draws_per_epoch = 0;  // nominal draws (m random, n adaptive)
    uint32_t G = 0;                // generators per epoch
    uint64_t L = 0;                // draws per generator
    uint64_t tail0 = 0;
    uint32_t tail_len = 0;
    uint64_t last_m = 0;           // size of the last selection
    bool identity = false;         // last selection = all rows
    DevBuf window, jp, gwin, misc;              // stream state, jump polynomials, generator windows
    // draws are double-buffered: while an epoch trains on buffer `cur`, the
    // next epoch's draws are generated into the other one on `side`
    DevBuf seqb[2], drawsb[2], tailb[2];
    int cur = 0;
    bool pre = false;       // buffer `cur` already holds (or is receiving) this epoch's draws
    bool want_gen = false;  // buffer `cur` still to be generated (after the next BMU kernel)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_adv = nullptr, ev_gen = nullptr;
    DevBuf err, age, keys, hist, cand, cidx, ccnt;  // adaptive (cand, cidx: first-digit bucket)
    bool age_pending = false;  // observe marked rows; +1 / 0 applied at the next select
    DevBuf first, tidx;                         // random
    DevBuf bitmap, bcount, sel;                 // selection
    // Sharded (a communicator attached): this rank holds rows [off, off + n) of
    // the gN rows the one reference Sampler covers; allreduce(buf, count, op)
    // runs on the engine stream, op 0 = u32 sum, 1 = u64 max, 2 = u64 sum.
    bool sharded = false;
    bool loopback = false;         // tests: in-process rank group instead of NCCL
    uint64_t gN = 0, off = 0;
    int world = 1, rank = 0;
    int jump0 = 0;                 // generator 0 starts at a jumped offset (off > 0)
    std::function<bool(void*, size_t, int)> allreduce;
    // waits for the engine stream after a sharded selection (the engine's
    // reduce barrier with its deadline); false = the barrier failed
    std::function<bool(cudaStream_t)> sync;
    DevBuf jN, glist, slots;       // jump by gN (adaptive), global selection, per-rank counts
};
int sampler_setup(SamplerState& s, int kind, uint64_t n, uint64_t m, uint64_t seed, double alpha,
                  double beta, int sm_count);
// 0: selection written to `out` (device), -1: identity (all rows), else error
int sampler_select(SamplerState& s, uint32_t* out, uint64_t* m_out, int sm_count, cudaStream_t st);
void sampler_observe(SamplerState& s, const uint32_t* sel, uint64_t m, const double* dist,
                     int sm_count, cudaStream_t st);
// apply the pending "+1 / observed rows 0" age update (before reading ages)
void sampler_materialize_ages(SamplerState& s, int sm_count, cudaStream_t st);
void sampler_release(SamplerState& s);
// start generating the next epoch's draws on the sampler's side stream once
// `after` (recorded on the engine stream) completes
void sampler_pregenerate(SamplerState& s, cudaEvent_t after);

struct Engine {
    int device = 0;
    uint32_t P = 0, D = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;
    std::string last_error;
    int sm_count = 148;
    size_t smem_optin = 0;

    // options
    int bmu_kernel = 0;  // 0 auto, 1 simt, 2 tc
    double tau_simt = kDefaultTauSimt;
    double tau_tc = kDefaultTauTc;
    uint64_t stream_chunk_rows = 1u << 20;

    // bound data
    DevBuf x;           // resident rows, row stride ldx floats
    uint32_t ldx = 0;   // D (packed), or kPadFloats: each row on its own two 128-B lines
    bool pad_rows = true;  // TSOM_OPT_PAD_ROWS
    // TSOM_OPT_DETERMINISTIC: exact (order-independent) sums, k_accum.cu
    bool exact = false;
    DevBuf xsums;         // exact_sums_words int64: the epoch's reduce buffer in exact mode
    DevBuf xmax_g;        // max ||x||^2 over all ranks' rows (float; u64 slot for the reduce)
    bool xmax_g_ready = false;
    uint64_t n_rows = 0;
    bool x_slack = false;  // kRowSlack bytes readable after the last resident row
    bool streamed = false;
    const float* host_rows = nullptr;  // streamed mode source
    bool host_registered = false;
    DevBuf xsplit;      // pre-split tcgen05 A tiles of all rows (encoding xsplit_kind)
    int xsplit_kind = 0;
    DevBuf scale;       // {s, s^2, overflow} of the operands currently in wsplit
    DevBuf xn2, gxn2, txn2;  // per-row ||x||^2 for xsplit / gsplit / tsplit rows
    bool xsplit_valid = false;
    DevBuf x2max;       // float: max ||x||^2 over bound rows
    // TSOM_OPT_ROW_ORDER (k_order.cu): the resident rows re-laid out in the BMU
    // order of an earlier full pass — position q holds caller row perm[q],
    // pinv is the inverse; every call still takes and returns caller row ids
    uint32_t row_order = 1;     // 0 off, 1 auto (long multi-epoch calls), 2 once, R >= 3 periodic
    uint32_t epochs_left = 0;   // tsom_train_epochs: epochs of the call from this one on
    uint64_t row_order_min = 1u << 18;  // fewer rows: not worth a re-layout
    bool ordered = false;
    DevBuf perm, pinv, idmap;   // idmap: a selection mapped to positions
    DevBuf unperm;              // per-row outputs scattered back to caller order
    bool sorted_full = false;   // acc.sorted = the last full pass's BMU-ordered positions
    uint32_t passes_since_order = 0;
    // 3xFP16 split image of the resident rows (row-major, img_w halves per
    // row) + per-row window terms: the gather source of K1 for selections
    // (kGather), built on the first selection pass that covers >= 1/64 of
    // the rows (launch_split_image).  Diagnostics option 95 = 1 turns it on;
    // off by default: measured slower than splitting the selection per pass
    // (TMA gather4 of 128-B row segments is op-rate bound)
    DevBuf ximg, ximg_xn2, gid;
    bool img_valid = false;
    int img_mode = 0;
    uint32_t img_w = 0;
    alignas(64) CUtensorMap img_map{};

    // codebook
    DevBuf w, wt, wsplit, w2, w2max, prev;
    bool codebook_set = false;
    bool codebook_prepped = false;

    // influence
    DevBuf infl;
    int64_t infl_key = -1;
    bool infl_set = false;
    DevBuf topo_dist;
    bool topo_set = false;
    DevBuf topo_buf[15];
    tsom::TopoScratch topo;
    uint32_t topo_p = 0;  // P the scratch was sized for

    // per-epoch scratch
    DevBuf sel;
    DevBuf rows_scratch;   // caller rows for tsom_bmu / gathered split tiles
    DevBuf gsplit;         // split tiles of a gathered selection
    DevBuf tsort, tcls;    // near-tie list by group class + tile masks; class counters
    DevBuf bmu;
    DevBuf dist;
    DevBuf part;           // tcgen05 per-group partial top-2 [groups][n] (b1, i1, b2)
    DevBuf flags;          // [0] full re-scan count, [1] exact-candidate count, then positions
    DevBuf ties;           // [0] near-tie count, then positions (enumerate pass input)
    DevBuf tmask;          // per near-tie row: bitmask of groups inside the window
    DevBuf part2;          // enumerate-pass partials
    DevBuf tsplit;         // split tiles of the near-tie rows (one pass of them)
    DevBuf tcnt;           // per-pass near-tie counts
    DevBuf acc_buf[7];     // AccumScratch arrays
    tsom::AccumScratch acc;
    uint64_t acc_rows = 0; // capacity the scratch was sized for
    DevBuf sums;
    DevBuf U, H;
    DevBuf smooth_scratch;   // saug + split-b GEMM partials
    DevBuf status;         // device error word(s)
    DevBuf stage[2];       // streamed-mode device chunks
    DevBuf chunk_flags;    // streamed mode: re-check counters per chunk
    float* pinned[2] = {nullptr, nullptr};  // host staging for shard / pageable sources
    size_t pinned_rows = 0;
    size_t pinned_bytes[2] = {0, 0};  // sizes of the (possibly larger) cached blocks
    cudaEvent_t ev_pin[2] = {nullptr, nullptr};  // H2D from pinned[s] finished
    bool pin_busy[2] = {false, false};
    bool host_register = true;  // TSOM_OPT_HOST_REGISTER
    bool host_direct = false;   // streamed host rows are DMA-able (pinned)
    uint32_t staging_threads = 0;  // TSOM_OPT_STAGING_THREADS (0: min(16, host cores))
    uint64_t pageable_chunk_bytes = (uint64_t)128 << 20;  // pageable bind staging chunk
    struct ShardFile {
        std::string path;
        int fd = -1;
        uint64_t row0 = 0, rows = 0;
    };
    std::vector<ShardFile> shards;  // FSOMSHRD files (dataset.hpp:171-344)
    cudaEvent_t ev[12] = {};  // 0 start, 1 bmu end, 6 accum end, 7 smooth end, 8/9 K1 kernel, 10 update end
    // tsom_train_epochs: per-epoch K1 start/end events (the main pass of epoch t
    // records k1_ev[2t], k1_ev[2t+1] instead of ev[8], ev[9]) and the device
    // failure record [epoch + 1, kind (1 non-finite update, 2 term guard), node]
    std::vector<cudaEvent_t> k1_ev;
    std::vector<cudaEvent_t> acc_ev;  // the same for the accumulation phase (resident passes)
    float t_accum_mean = 0.0f;        // mean accumulation phase of the last multi-epoch call
    int k1_slot = -1;
    DevBuf dead;
    uint64_t last_recheck = 0;
    std::vector<uint32_t> chunk_counts;  // per-chunk re-check counts (streamed epochs)
    // pinned per-epoch status words, read back asynchronously before the one
    // end-of-epoch synchronisation: [0..1] re-check counts (resident epochs),
    // [2] update status, [3] max ||x||^2 and [4] max ||w||^2 (term guard)
    uint32_t* hstat = nullptr;
    // near-tie list lengths of the main passes since the last sync ([count,
    // rows] pairs, pinned, read back asynchronously); their largest fraction
    // sizes the enumerate passes of later epochs (run_bmu)
    uint32_t* tie_log = nullptr;
    DevBuf tie_dev;  // the counts themselves, written by k_tie_pass_counts
    uint32_t tie_log_n = 0;
    double tie_frac_max = -1.0;  // < 0: nothing observed yet
    bool defer_hstat = false;  // tsom_train_epochs: skip the count copy but for the last epoch
    bool hstat_counts = false;  // [0..1] hold this epoch's re-check counts
    bool recheck_from_chunks = false;
    // term guard (k_guard.cu): max |h| of the influence (device double), the
    // zero-initialised extremes scratch, the invocation tag, and the row set
    // of the last accumulation pass (x == nullptr: streamed, bound only)
    DevBuf hmax, guard_buf;
    uint32_t guard_tag = 0, last_guard_tag = 0;
    const float* pass_x = nullptr;
    uint32_t pass_ldx = 0;
    const uint32_t* pass_sel = nullptr;
    uint64_t pass_n = 0;
    float t_bmu = 0, t_accum = 0, t_smooth = 0, t_total = 0, t_k1 = 0, t_update = 0;
    float t_sample = 0;  // device sampler before the epoch (sampled tsom_train_epoch)
    bool k1_timed = false, update_timed = false, sample_timed = false;

    // device sampler
    SamplerState sampler;

    // multi-GPU
    void* nccl_comm = nullptr;
    int rank = 0, world = 1;
    // The reduce step of an epoch (and of the sharded sampler): the NCCL
    // communicator, or (tests) an in-process loopback group of engines.
    // op 0 = u32 sum, 1 = u64 max, 2 = u64 sum, 3 = f64 sum, 4 = i64 sum, in place on the
    // device buffer; returns a TSOM status with last_error set on failure.
    std::function<int(void*, size_t, int)> comm_reduce;
    // collect_with_barrier's deadline (parallel.hpp:24, 67-86): a rank that
    // does not reach the reduce within this many seconds fails the call with
    // TSOM_ERR_TIMEOUT instead of hanging it
    double barrier_timeout_s = 60.0;
    std::shared_ptr<void> group_ref;  // keeps a joined in-process rank group alive
    double barrier_wait_s = 0.0;   // seconds spent waiting in reduces (ThreadedExecutor::barrier_wait_s)
    std::vector<cudaEvent_t> red_ev;  // one per enqueued NCCL reduce of the current call
    size_t red_pending = 0;
};

// ---------------------------------------------------------------------------
// Kernel launchers (all asynchronous on `st`)
// ---------------------------------------------------------------------------

// codebook prep: w2 (f64 ||w_j||^2), w2max, SIMT operand wt
void launch_prep_codebook(const float* w, uint32_t P, uint32_t D, double* w2, float* w2max,
                          float* wt, uint32_t Ppad, cudaStream_t st);
// max ||x||^2 over rows (f32 atomic max on non-negative floats)
void launch_row_norm_max(const float* x, uint64_t n, uint32_t D, float* out, cudaStream_t st,
                         bool reset = true,  // reset = false: fold into *out (atomicMax)
                         uint32_t ldx = 0);  // row stride in floats (0: D)
// a[0] = max(a[0], a[1])
void launch_fold_max(float* a, cudaStream_t st);
// split rows (optionally gathered through sel, and/or through a position list
// idx: split row f = position idx[f]) into tcgen05 A tiles of encoding `kind`
// tx[f] (optional) = tie_xpart of the row: its share of the error window
void launch_split_rows(int kind, const float* x, const uint32_t* sel, const uint32_t* idx,
                       uint64_t n, uint32_t D, const float* scale, TieWin win, void* tiles,
                       float* tx, cudaStream_t st, const uint32_t* dev_n = nullptr,
                       uint32_t ldx = 0);
// The 3xFP16 split of rows [0, n) as a row-major image: row r at img + r * img_w
// halves (img_w = 64 * atoms >= kpad; columns past kpad are not written), the
// gather source of K1's kGather mode; xn2[r] = the row's window term.
void launch_split_image(const float* x, uint32_t ldx, uint64_t n, uint32_t D, const float* scale,
                        TieWin win, void* img, uint32_t img_w, float* xn2, cudaStream_t st);  // row stride in floats (0: D)
bool tc_supported(int kind, uint32_t P, uint32_t D);
size_t tc_wsplit_bytes(int kind, uint32_t P, uint32_t D);
// scale = {s, s^2, overflow flag}: kTcF16 picks s = 2^e from max ||x||^2 (x2max[0])
// zero[0..nzero) and *zero2 (optional) are cleared first: the counters of the pass
void launch_set_scale(int kind, const float* x2max, float* scale, cudaStream_t st,
                      uint32_t* zero = nullptr, uint32_t nzero = 0, uint32_t* zero2 = nullptr,
                      uint32_t* zero3 = nullptr, uint32_t nzero3 = 0);
// tcgen05 B operand of the codebook (per group, core-matrix order)
void launch_prep_wsplit(int kind, const float* w, uint32_t P, uint32_t D, const float* scale,
                        void* wsplit, cudaStream_t st);
// nodes per CTA-resident codebook group (multiple of 32, <= 256)
__host__ __device__ inline uint32_t tc_group_width(uint32_t P) {
    return P >= (uint32_t)kTcGroupN ? (uint32_t)kTcGroupN : (P + 31u) / 32u * 32u;
}

// K1: BMU candidates.  SIMT variant writes final bmu + flags directly.
void launch_bmu_simt(const float* x, uint32_t ldx, const uint32_t* sel, uint64_t n, uint32_t D,
                     const float* wt, uint32_t P, uint32_t Ppad, const float* x2max,
                     const float* w2max, float tau, uint32_t* bmu, uint32_t* flags, int sm_count,
                     cudaStream_t st);
// tcgen05 variant: per-group partials (enumerate = candidate lists; dev_n =
// optional device row count; skip: the main pass over BMU-ordered rows, whose
// epilogue skips the column chunks no row of a warp needs; tmap: 3xFP16 rows
// gathered by id (grow[pos]) from the split image instead of tiles).
cudaError_t launch_bmu_tc(int kind, const void* tiles, uint64_t n, const uint32_t* dev_n,
                          bool enumerate, uint32_t P, uint32_t D, const void* wsplit,
                          const float* xn2, const float* w2max, const float* scale, TieWin win,
                          const uint32_t* rmask, float* part, int sm_count, size_t smem_optin,
                          cudaStream_t st, const uint32_t* tile_mask = nullptr, bool skip = false,
                          const CUtensorMap* tmap = nullptr, const uint32_t* grow = nullptr);
extern uint32_t g_k1_debug;
extern int g_split_v1;
extern int g_split_prefetch;
extern int g_split_tma;
extern int g_gather_kind;
extern int g_merge_v1;
int k1_trace_copy(unsigned long long* out, uint32_t n);
int k1_set_dump(float* d_buf);  // diagnostics: option 99 bit 7 target (rows x groups*gn floats)  // diagnostics  // diagnostics: bit0 skip epilogue math, bit1 skip MMAs
// main-pass merge: bmu for rows with a clear winner, near-tie positions -> ties
constexpr uint32_t kTcEpiSets = 2;  // K1 main pass: partial results per group (sub-groups)
// returns true when the near-tie rows' group classes were counted into cls
bool launch_merge_fast(const float* part, uint64_t n, uint32_t groups, uint32_t sets, uint32_t gn,
                       const float* xn2, const float* w2max, const float* scale, TieWin win,
                       uint32_t* bmu, uint32_t* ties, uint32_t* tmask, uint32_t* flags,
                       cudaStream_t st, uint32_t* cls = nullptr, uint32_t* tile_mask = nullptr);
// enumerate-pass merge over the near-tie rows: candidates -> exact FP64 -> bmu;
// overflow -> flags list for the full re-scan.
// ties: near-tie positions, dev_count: their number (device); rows past `cap`
// are sent to the full re-scan; n_max bounds the count (grid sizing)
// rmask (optional): per row the groups enumerated for it (the others skipped)
void launch_merge_partials(const float* part, const uint32_t* ties, const uint32_t* dev_count,
                           uint64_t cap, uint64_t n_max, uint32_t groups, uint32_t gn,
                           const float* xn2, const float* w2max, const float* scale, TieWin win,
                           const float* x, uint32_t ldx, const uint32_t* sel, const float* w,
                           uint32_t D, uint32_t* bmu, uint32_t* flags, cudaStream_t st,
                           const uint32_t* rmask = nullptr);
// near-tie list re-ordered by the groups each row needs (k_bmu.cu)
constexpr uint32_t kTieClasses = 9;
#ifdef __CUDACC__
__device__ inline uint32_t tie_class(uint32_t mask) {  // one group alone, or several
    const uint32_t c = __popc(mask) == 1 ? (uint32_t)(__ffs(mask) - 1) : kTieClasses - 1;
    return c < kTieClasses - 1 ? c : kTieClasses - 1;
}
#endif
void launch_tie_classes(const uint32_t* ties, const uint32_t* tmask, uint64_t n_max, uint32_t* cls,
                        uint32_t* ties_s, uint32_t* tmask_s, uint32_t* tile_mask, cudaStream_t st);
// exact FP64 re-scan of flagged rows (reference loop order)
void launch_rescan(const float* x, uint32_t ldx, const uint32_t* sel, const float* w, uint32_t P,
                   uint32_t D, const uint32_t* flags, uint64_t n, uint32_t* bmu, cudaStream_t st);

void accum_scratch_bytes(uint64_t n, uint32_t P, uint32_t D, size_t out[7]);
// sums = [R (P*d) | c (P) | sum dist | rows]; first=false adds to it (streamed chunks).
// accumulate=false -> distances / distance sum only (QE, find_bmus).
// Exact mode (TSOM_OPT_DETERMINISTIC): the epoch's sums on fixed-point grids
// given by the data's global bounds, in int64 limbs — independent of chunks,
// pieces and ranks (k_accum.cu).  xs: exact_sums_words(P, D) int64 =
// [S limbs (3 P d) | sum-dist limbs (3) | counts (P) | rows (1)]; the one
// reduce is an int64 sum of it; launch_exact_unpack writes the f64 sums.
struct ExactSums {
    long long* xs = nullptr;
    const float* xmax2 = nullptr;  // max ||x||^2 over every rank's rows
    const float* w2max = nullptr;  // max ||w||^2 of the epoch's codebook
};
// the grids: x values at 2^L with max|x| 2^L <= 2^53 (<= 256 rows a piece stay
// below 2^61), distances at the scale of max||x|| + max||w|| the same way
__host__ __device__ inline void exact_scales(const float* xmax2, const float* w2max, double* sx,
                                             double* sd) {
    const double xm = sqrt((double)*xmax2), dm = xm + sqrt((double)*w2max);
    const int ex = xm > 0.0 ? ilogb(xm) + 1 : 0;
    const int ed = dm > 0.0 ? ilogb(dm) + 1 : 0;
    *sx = ldexp(1.0, 53 - (ex < -900 ? -900 : ex));
    *sd = ldexp(1.0, 53 - (ed < -900 ? -900 : ed));
}
size_t exact_sums_words(uint32_t P, uint32_t D);
void launch_exact_unpack(const ExactSums& ex, uint32_t P, uint32_t D, double* sums,
                         cudaStream_t st);
// returns 1 when `exact` is asked for on a path without the TMA gather, else 0
int launch_accumulate(const float* x, const uint32_t* sel, uint64_t n, uint32_t D,
                       const float* w, uint32_t P, const uint32_t* bmu, double* dist_out,
                       bool want_dist_sum, bool accumulate, bool first, const AccumScratch& s,
                       double* sums, int sm_count, cudaStream_t st, bool x_slack = false,
                       uint32_t ldx = 0,  // row stride in floats (0: D; kPadFloats: padded rows)
                       const ExactSums* exact = nullptr);
// resident rows at a 256-byte stride (kPadFloats floats per row, zero tail):
// the K2 gather's rows are then exactly two 128-byte lines
constexpr uint32_t kPadFloats = 64;
void launch_pad_rows(const float* x, uint64_t n, uint32_t D, float* xpad, cudaStream_t st);
// BMU-ordered residency (k_order.cu): dst[q] = src[sorted[q]] packed, perm_out[q]
// = perm_in[sorted[q]] (perm_in null: identity); pinv = perm^-1; out[i] =
// pinv[sel[i]]; out[perm[q]] = v[q]
void launch_permute_rows(const float* src, uint32_t ldx, const uint32_t* sorted, uint64_t n,
                         uint32_t D, float* dst, const uint32_t* perm_in, uint32_t* perm_out,
                         cudaStream_t st);
void launch_invert_perm(const uint32_t* perm, uint64_t n, uint32_t* pinv, cudaStream_t st);
void launch_map_ids(const uint32_t* sel, uint64_t n, const uint32_t* pinv, uint32_t* out,
                    cudaStream_t st);
void launch_unpermute_u32(const uint32_t* v, const uint32_t* perm, uint64_t n, uint32_t* out,
                          cudaStream_t st);
void launch_unpermute_f64(const double* v, const uint32_t* perm, uint64_t n, double* out,
                          cudaStream_t st);
// bytes of slack the engine allocates after resident rows (TMA row gathers read
// up to 16 bytes past a row)
constexpr size_t kRowSlack = 64;

// K3: smoothing num = H^T S, den = H^T c; U = eta (num - w den), H = den
// status (optional): apply_update's fault slot, reset to INT_MAX here
void launch_smooth(const double* infl, const double* sums, const float* w, uint32_t P, uint32_t D,
                   double eta, double* U, double* H, double* scratch, cudaStream_t st,
                   int* status = nullptr);
size_t smooth_scratch_doubles(uint32_t P, uint32_t D);
// apply_update on device (trainer.hpp:341-369); status[0] = first bad node + 1
void launch_apply_update(float* w, float* prev, uint32_t P, uint32_t D, const double* U,
                         const double* H, bool use_momentum, double momentum, int* status,
                         cudaStream_t st);
// status[0] = INT_MAX (no failing node) before launch_apply_update
void launch_status_reset(int* status, cudaStream_t st);
// multi-epoch runs: skip the update once dead[0] != 0; after an epoch, record
// a failed update (status) or a violated term guard in dead[]
void launch_apply_update_guarded(float* w, float* prev, uint32_t P, uint32_t D, const double* U,
                                 const double* H, bool use_momentum, double momentum, int* status,
                                 const int* dead, cudaStream_t st);
// after an epoch's update: a non-finite update recorded in dead[]
void launch_epoch_guard(const int* status, uint32_t epoch, int* dead, cudaStream_t st);
// The accumulation-term guard of quantize_term (accum.hpp:34-38), exact
// (k_guard.cu): flag[1] == tag iff the reference would throw for this epoch's
// rows, BMUs and (pre-update) codebook.  Zero-initialised scratch of
// guard_scratch_words() u32; dead (optional): multi-epoch failure record.
struct GuardScratch {
    uint32_t* flag = nullptr;  // [2]
    uint32_t* seen = nullptr;  // [P]
    uint32_t* mn = nullptr;    // [P * D]
    uint32_t* mx = nullptr;    // [P * D]
};
size_t guard_scratch_words(uint32_t P, uint32_t D);
GuardScratch guard_scratch(uint32_t* base, uint32_t P, uint32_t D);
cudaError_t launch_term_guard(const float* x, uint32_t ldx, const uint32_t* sel, uint64_t n,
                       const uint32_t* bmu, const float* w, const double* infl, uint32_t P,
                       uint32_t D, double eta, const float* x2max, const float* w2max,
                       const double* hmax, uint32_t tag, GuardScratch g, int sm_count,
                       cudaStream_t st, int* dead = nullptr, uint32_t epoch = 0);
// max |h| of an influence matrix as kHmaxParts per-block maxima (no reset
// needed: every block writes its slot; the guard folds them)
constexpr unsigned kHmaxParts = 592;
void launch_infl_absmax(const double* infl, size_t n, double* hpart, cudaStream_t st);
// block-wide max of a non-negative double (NaN wins) into out[blockIdx.x]
__device__ __forceinline__ void block_max_to(double m, double* out) {
    __shared__ double s_bm[32];
    for (int o = 16; o; o >>= 1) {
        const double v = __shfl_xor_sync(0xffffffffu, m, o);
        m = v > m || v != v ? v : m;
    }
    if ((threadIdx.x & 31) == 0) s_bm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (unsigned w = 1; w < (blockDim.x + 31) / 32; ++w)
            m = s_bm[w] > m || s_bm[w] != s_bm[w] ? s_bm[w] : m;
        out[blockIdx.x] = m;
    }
}
// influence_matrix (topology.hpp:342-364) from a P x P distance matrix
// (hpart: kHmaxParts per-block maxima of |h| for the term guard)
void launch_influence(const double* dist, size_t n, double inv_two_sigma_sq, double* out,
                      cudaStream_t st, double* hpart);
// synthetic Gaussian mixture rows
void launch_synth_gmm(float* x, uint64_t n, uint32_t D, const float* centres, uint32_t n_comp,
                      uint64_t seed, uint64_t row_offset, cudaStream_t st, uint32_t ldx = 0);

}  // namespace tsom
