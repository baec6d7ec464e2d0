/*
 * tsom_b200.h — C-ABI of the B200-native batch-SOM epoch engine.
 *
 * This is the drop-in boundary for the hot path of the toposom reference
 * (paths below are relative to /root/reference/proj/include/toposom).  The
 * reference's only seam is the Executor concept consumed by
 * train_with_executor<Executor> (trainer.hpp:466-470, called at :506-508):
 *
 *     IterationAccumulators run_iteration(selected, weights, influence, eta,
 *                                         n_chunks, distances);
 *
 * include/toposom_b200/cuda_executor.hpp implements that concept on top of
 * the functions declared here, so the reference training loop runs unchanged
 * with every per-epoch data pass on the GPU.  The free functions find_bmus /
 * map_samples / mean_bmu_distance / quantization_error map onto tsom_bmu and
 * tsom_qe.
 *
 * Conventions:
 *   - every call returns an int status (TSOM_OK .. TSOM_ERR_TIMEOUT);
 *     tsom_last_error() holds the message, whose prefix matches the
 *     reference's exception text so the C++ adapter can rethrow the same type;
 *   - plain pointers and sizes only; host buffers are borrowed for the call;
 *   - the engine owns all device memory, streams and the NCCL communicator;
 *   - an engine is not re-entrant (one training run, one thread).
 *
 * Layouts: samples and codebooks are row-major float32 (DataMatrix,
 * matrix.hpp:12-29); influence is P x P float64 row-major, row b = influence
 * of BMU b on every node (trainer.hpp:326); accumulators U (P x d) and H (P)
 * are float64 values of the IterationAccumulators (accum.hpp:45-69).
 */
#ifndef TSOM_B200_H
#define TSOM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes. */
#define TSOM_OK 0
#define TSOM_ERR_INVALID 1   /* std::invalid_argument */
#define TSOM_ERR_NUMERICAL 2 /* std::runtime_error "numerical fault: ..." */
#define TSOM_ERR_RANGE 3     /* std::out_of_range */
#define TSOM_ERR_CUDA 4
#define TSOM_ERR_NCCL 5
#define TSOM_ERR_TIMEOUT 6

/* tsom_bind_host_data flags */
#define TSOM_BIND_COPY 0u      /* copy rows into HBM once (resident mode)      */
#define TSOM_BIND_STREAMED 1u  /* keep rows in (pinned) host memory; every epoch
                                  streams them through double-buffered chunks */

/* tsom_set_option keys */
#define TSOM_OPT_BMU_KERNEL 1      /* 0 = auto, 1 = SIMT, 2 = tcgen05 3xTF32 (d <= 53),
                                      3 = tcgen05 3xFP16 (d <= 62); auto = 3, else 2, else 1 */
#define TSOM_OPT_TIE_TAU 2         /* value*2^-30: relative tie window for the exact re-check */
#define TSOM_OPT_STREAM_CHUNK 3    /* rows per streamed chunk */
#define TSOM_OPT_DETERMINISTIC 4   /* 1 = exact sums: every row's features and distance on
                                      fixed-point grids set by the data's global bounds, summed
                                      in int64 limbs and reduced as integers, so an epoch's
                                      results are bit-identical for any rank count, chunking or
                                      selection order (the reference's guarantee,
                                      accum.hpp:12-20; parallel.hpp:17-21).  Resident rows,
                                      d even and <= 62.  Default 0: FP64 sums (they agree to
                                      summation order) */
#define TSOM_OPT_HOST_REGISTER 5   /* streamed host rows: 1 (default) page-lock the caller's
                                      buffer for direct DMA, 0 copy through pinned staging */
#define TSOM_OPT_STAGING_THREADS 6 /* host threads filling the pinned staging (default: min(16, cores)) */
#define TSOM_OPT_PAD_ROWS 8          /* resident rows at a 256-B stride (d even, <= 62):
                                        1 (default) or 0 = packed d-float rows */
#define TSOM_OPT_ROW_ORDER 9          /* resident rows kept in BMU order (rows that share a
                                         BMU adjacent: K1 skips the column chunks no row of a warp
                                         needs, K2 copies runs of rows): 0 = bind order; 1
                                         (default, auto) = re-laid out (packed) once, in the BMU
                                         order of the last full pass, at an epoch of a
                                         tsom_train_epochs call with >= 20 epochs still to run (a
                                         shorter run does not win back the re-layout); 2 = once, at
                                         the first full pass after one; R >= 3 = that, then every R
                                         full training passes.  Row ids in every call stay the
                                         caller's */
#define TSOM_OPT_BARRIER_TIMEOUT_MS 7 /* reduce-barrier deadline, ms (default 60000 =
                                         kDefaultBarrierTimeoutS, parallel.hpp:24); a rank that
                                         misses it fails the call with TSOM_ERR_TIMEOUT
                                         "reduce barrier timed out after X s waiting for worker g"
                                         (collect_with_barrier, parallel.hpp:67-86) */

typedef struct tsom_engine tsom_engine;
typedef struct tsom_group tsom_group;

/* Engine lifetime ---------------------------------------------------------- */

/* Create an engine for a P-node, d-dimensional codebook on CUDA `device`
 * (1 <= P <= 65536, 1 <= d <= 256; the tensor-core BMU kernels cover d <= 62,
 * larger d uses the SIMT kernel). */
int tsom_create(int device, uint32_t nodes, uint32_t dims, tsom_engine** out);
int tsom_destroy(tsom_engine* eng);
const char* tsom_last_error(const tsom_engine* eng);
const char* tsom_version(void);
int tsom_set_option(tsom_engine* eng, int key, int64_t value);

/* Data binding (DataSourceRef, dataset.hpp:362-421) ------------------------ */

/* Bind n_rows x dims row-major float32 host rows.  TSOM_BIND_COPY uploads once
 * and keeps the rows resident in HBM; TSOM_BIND_STREAMED re-streams them from
 * host memory every epoch (the caller keeps `rows` alive until rebind/destroy).
 * Replaces the executor's DataSourceRef (trainer.hpp:442, parallel.hpp:101). */
int tsom_bind_host_data(tsom_engine* eng, const float* rows, uint64_t n_rows, uint32_t flags);
/* Bind FSOMSHRD shard files (dataset.hpp:171-344: 24-byte header "FSOMSHRD",
 * u32 version 1, u64 rows, u32 cols, then row-major f32), rows in the order of
 * `paths` (open_shards sorts part-*.shard by name, :277-301).  TSOM_BIND_COPY
 * reads them once into HBM; TSOM_BIND_STREAMED keeps them on disk and every
 * epoch preads chunks into pinned staging, overlapped with the GPU work of the
 * previous chunk (the out-of-core path; replaces ChunkReader :305-344 and the
 * per-chunk rescans of DataSourceRef::fetch_rows :400-415).  Header errors keep
 * the reference's messages ("not a shard file (bad magic): ...", "truncated or
 * corrupt shard: ...", "shard column count mismatch in ..."). */
int tsom_bind_shards(tsom_engine* eng, const char* const* paths, uint32_t n_paths,
                     uint32_t flags);
/* Bind rows that already live in this device's memory (borrowed). */
int tsom_bind_device_data(tsom_engine* eng, const float* d_rows, uint64_t n_rows);
/* Fill the bound dataset with the SURVEY.md §8(d) Gaussian mixture generated
 * on the device (centres from the reference Rng on the host, noise from a
 * counter-based generator).  Used for throughput runs at N >= 1e7. */
int tsom_bind_synthetic_gmm(tsom_engine* eng, uint64_t n_rows, uint64_t seed, uint32_t n_comp,
                            uint64_t row_offset);
uint64_t tsom_rows(const tsom_engine* eng);
/* Copy resident rows [row0, row0 + n) back to the host as n x d row-major
 * f32 (DataSourceRef::fetch_rows of a contiguous range, dataset.hpp:393-399). */
int tsom_get_rows(tsom_engine* eng, uint64_t row0, uint64_t n, float* out);

/* Per-epoch state ---------------------------------------------------------- */

/* Codebook P x d (SomModel::weights, trainer.hpp:106). */
int tsom_set_codebook(tsom_engine* eng, const float* weights);
int tsom_get_codebook(tsom_engine* eng, float* weights);
/* SomModel::prev_update (trainer.hpp:108): the momentum memory the device
 * update keeps (all zero when momentum is off), P x d f32. */
int tsom_get_prev_update(tsom_engine* eng, float* prev);
/* Influence P x P float64 (cached_influence, topology.hpp:406-418).  key is the
 * caller's cache key (e.g. influence_cache_key(sigma) mixed with the topology
 * refresh count); an unchanged non-negative key skips the upload. */
int tsom_set_influence(tsom_engine* eng, const double* influence, int64_t key);

/*
 * One iteration's accumulation pass: Executor::run_iteration
 * (trainer.hpp:446-453, parallel.hpp:107-130) plus the single reduce.
 *   selected : sorted distinct row ids, or NULL for all bound rows
 *   u_out    : P x d float64 U_j = eta * sum_i h[b_i][j] (x_i - w_j)  (may be NULL)
 *   h_out    : P float64     H_j = sum_i h[b_i][j]                    (may be NULL)
 *   dist_out : one BMU distance per selected row, selection order (may be NULL)
 * With a communicator attached (tsom_comm_init) each rank passes its own
 * rows/selection and receives the globally reduced U/H.
 */
int tsom_epoch(tsom_engine* eng, const uint32_t* selected, uint64_t n_sel, double eta,
               double* u_out, double* h_out, double* dist_out);

/* BMU search on caller rows (find_bmus trainer.hpp:282-308 / map_samples
 * :534-541).  bmu: n uint32; dist: n float64 or NULL. */
int tsom_bmu(tsom_engine* eng, const float* rows, uint64_t n, uint32_t* bmu, double* dist);
/* BMU search over the bound rows (or a selection of them). */
int tsom_bmu_bound(tsom_engine* eng, const uint32_t* selected, uint64_t n_sel, uint32_t* bmu,
                   double* dist);
/* Quantisation error over bound rows (mean_bmu_distance trainer.hpp:377-398,
 * quantization_error metrics.hpp:28-30): returns the distance sum and count. */
int tsom_qe(tsom_engine* eng, const uint32_t* selected, uint64_t n_sel, double* dist_sum,
            uint64_t* count);

/* Device-resident training (no per-epoch host traffic) -------------------- */

/* Static neighbourhood distances P x P (lattice_dist topology.hpp:137-149, or
 * hop counts topology.hpp:292-325 widened to float64); the influence for each
 * sigma is then built on the device exactly as influence_matrix (:342-364). */
int tsom_set_topology_distance(tsom_engine* eng, const double* dist);
/* One full epoch on the device: influence(sigma) -> BMU -> accumulate ->
 * (allreduce) -> smoothing -> apply_update (trainer.hpp:341-369) with the
 * reference's H floor, momentum and non-finite guards.  flags bit0 = momentum
 * on; bit1 = rows picked by the device sampler (tsom_sampler_init), which then
 * observes their distances (trainer.hpp:495, 511).  Weights stay on the device
 * (read with tsom_get_codebook). */
int tsom_train_epoch(tsom_engine* eng, double eta, double sigma, double momentum,
                     uint32_t flags);
/* n_epochs consecutive tsom_train_epoch calls (the epoch loop of
 * train_with_executor, trainer.hpp:486-520, with the schedules eta[t], sigma[t]
 * precomputed by the caller) enqueued back to back with no host round trip
 * between epochs.  The per-epoch checks run on the device: after a failing
 * epoch the later ones leave the weights unchanged, and the call returns
 * TSOM_ERR_NUMERICAL with *failed_epoch (optional) = the failing epoch.
 * tsom_last_timing_detail then reports the last epoch's phases and the mean
 * K1 time of the call. */
int tsom_train_epochs(tsom_engine* eng, uint32_t n_epochs, const double* eta,
                      const double* sigma, double momentum, uint32_t flags,
                      uint32_t* failed_epoch);
/* Topology refresh on the device (refresh_topology topology.hpp:439-451) from
 * the engine's current codebook: FP64 Gram (pairwise_sq_dists :81-108), then
 * kind 2 = MST (build_mst :192-220) or 3 = RNG (build_rng_graph :229-258), then
 * all-pairs hop counts (hop_distances :292-325) which become the distance
 * matrix of the device-resident loop.  edges_out (optional): (i, j) pairs, i < j,
 * lexicographic; hops_out (optional): P x P uint16.  Errors: "hop_distances:
 * graph is disconnected" (TSOM_ERR_NUMERICAL). */
int tsom_refresh_topology(tsom_engine* eng, int kind, uint32_t* edges_out, uint64_t edges_cap,
                          uint64_t* n_edges, uint16_t* hops_out);
/* pairwise_sq_dists (topology.hpp:81-108) of the current codebook, P x P f64. */
int tsom_pairwise_sq_dists(tsom_engine* eng, double* out);
/* Rows of the last BMU pass whose winner was decided in exact FP64 (several
 * candidates inside the FP32 error window, or a full re-scan). */
uint64_t tsom_last_recheck_count(const tsom_engine* eng);
/* The BMU kernel the engine runs for its shape and options: 1 = SIMT FP32,
 * 2 = tcgen05 3xTF32, 3 = tcgen05 3xFP16 (TSOM_OPT_BMU_KERNEL values). */
int tsom_active_bmu_kernel(const tsom_engine* eng);

/* Device samplers (Sampler, sampling.hpp:183-221) ------------------------ */

/* Per-epoch row selection on the device, identical to toposom::Sampler(kind,
 * budget, N = tsom_rows(), seed, alpha, beta) for the same seed: kind 0 = full
 * (select_full :46-51), 1 = random (Floyd, select_random :56-73), 2 = adaptive
 * (select_adaptive :101-139 with update_adaptive :143-157).  m = the resolved
 * budget (resolve_budget :30-40).  The random stream is the reference's
 * mt19937_64 (Rng(seed, SeedStream::sampler), rng.hpp:21-37), produced by many
 * device generators started with jump-ahead polynomials.  Errors:
 * "select_random: m must be >= 1". */
int tsom_sampler_init(tsom_engine* eng, int kind, uint64_t m, uint64_t seed, double alpha,
                      double beta);
/* Sampler::select(): the next sorted selection (kept on the device for the
 * next sampled epoch); sel_out (optional) receives m_out row ids. */
int tsom_sampler_select(tsom_engine* eng, uint32_t* sel_out, uint64_t* m_out);
/* Sampler::observe(selected, distances) for the last selection: dist = one
 * distance per selected row in selection order, or NULL for the distances of
 * the last sampled tsom_train_epoch.  No-op unless adaptive. */
int tsom_sampler_observe(tsom_engine* eng, const double* dist);
/* AdaptiveSamplerState (sampling.hpp:83-92): last_error (N f64) and age (N u32). */
int tsom_sampler_state(tsom_engine* eng, double* last_error, uint32_t* age);
/* The SURVEY.md §8(d) synthetic rows on the host (no GPU), value-identical to
 * the reference's generator: Rng(seed, SeedStream::synth) (rng.hpp:21-37),
 * n_comp x d centres real(-4, 4), then per row m = index(n_comp) and
 * x_k = f32(mu[m][k] + gaussian()) (rng.hpp:64-76).  `threads` host threads
 * (0 = all cores), each jumping the mt19937_64 stream to its first row.
 * out: rows [row0, row0 + n) of the stream, n x d row-major f32 (a rank's
 * contiguous share of a dataset generated once). */
int tsom_synth_gmm_host(float* out, uint64_t row0, uint64_t n, uint32_t d, uint64_t seed,
                        uint32_t n_comp, uint32_t threads);
/* Host-only check of the jump-ahead (no GPU): 0 when the state jumped by `jump`
 * draws from mt19937_64(seed) equals sequential generation. */
int tsom_mt_selftest(uint64_t seed, uint64_t jump);
/* Return the device memory cached by destroyed engines to the driver (engines
 * allocate from a per-device caching pool; cf. torch.cuda.empty_cache). */
int tsom_release_cached_memory(int device);

/* Multi-GPU (one process per GPU) ---------------------------------------- */

/* 128-byte ncclUniqueId produced by rank 0 and broadcast by the caller. */
int tsom_comm_unique_id(tsom_engine* eng, uint8_t id_out[128]);
/* Attach an NCCL communicator (non-blocking: initialisation and every reduce
 * are polled against TSOM_OPT_BARRIER_TIMEOUT_MS and aborted with
 * ncclCommAbort -> TSOM_ERR_TIMEOUT when a peer never arrives); every epoch then
 * ends with exactly one ncclAllReduce(sum, float64) of the packed
 * [S | c | sum dist | count] buffer (parallel.hpp:90-95 reduce). */
int tsom_comm_init(tsom_engine* eng, const uint8_t id[128], int rank, int world);
/* In-process rank group: `world` engines driven from separate threads of one
 * process (one per GPU, the ThreadedExecutor shape of parallel.hpp:99-140, or
 * several on one GPU) joined by a host-memory reduce instead of NCCL.  Each
 * rank's contribution is kept and the reduce is evaluated in rank order
 * (parallel.hpp:90-95), so every rank gets the same sums; a rank that misses
 * the barrier deadline is named ("reduce barrier timed out after X s waiting
 * for worker g", TSOM_ERR_TIMEOUT).  The sharded device sampler uses the same
 * group.  Destroy the group after its engines. */
int tsom_group_create(int world, tsom_group** out);
int tsom_group_join(tsom_engine* eng, tsom_group* group, int rank);
int tsom_group_destroy(tsom_group* group);
/* Seconds this engine has spent in reduce barriers
 * (ThreadedExecutor::barrier_wait_s, parallel.hpp:136). */
double tsom_barrier_wait_s(const tsom_engine* eng);

/* Timing of the last epoch (device events), milliseconds. */
int tsom_last_timing(const tsom_engine* eng, float* bmu_ms, float* accum_ms, float* smooth_ms,
                     float* total_ms);
/* Detail of the last epoch (ms): [0] BMU kernel (K1) alone, [1] BMU phase incl.
 * merge + exact re-check, [2] accumulation + reduce (+ allreduce), [3] smoothing,
 * [4] device update (tsom_train_epoch), [5] total (sampler excluded), [6] device sampler
 * (sampled tsom_train_epoch), [7] mean accumulation phase over the epochs of the last
 * tsom_train_epochs call (resident rows; per-epoch events). */
int tsom_last_timing_detail(const tsom_engine* eng, float out[8]);
/* Device memory this engine holds (bytes of its buffers, sampler included). */
uint64_t tsom_device_bytes(const tsom_engine* eng);
/* Number of CUDA kernels this library has launched in this process. */
uint64_t tsom_kernel_launches(void);
/* The CUDA stream all engine work is issued on (cudaStream_t as void*). */
void* tsom_stream(tsom_engine* eng);

#ifdef __cplusplus
}
#endif

#endif /* TSOM_B200_H */
