// cuda_executor.hpp — B200 drop-in for the toposom Executor seam.
//
// The reference training loop train_with_executor<Executor>
// (toposom/trainer.hpp:466-523) calls executor.run_iteration(...) exactly once
// per epoch (:506-508) and applies the returned IterationAccumulators with
// apply_update (:510).  CudaExecutor satisfies that concept (same signature as
// SerialExecutor, trainer.hpp:440-460, and ThreadedExecutor,
// parallel.hpp:99-140) and runs the whole data pass — BMU search,
// accumulation, reduce, neighbourhood smoothing — on a B200 through the C-ABI
// in tsom_b200.h.  A maintainer switches a run to the GPU with
//
//     #include <toposom_b200/cuda_executor.hpp>
//     auto [model, log] = toposom_b200::train_cuda(config, data, sampler);
//
// exactly where they would call toposom::train / train_parallel.  Exceptions
// keep the reference's types and message prefixes.
#pragma once

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <future>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "toposom/metrics.hpp"
#include "toposom/parallel.hpp"
#include "toposom/trainer.hpp"
#include "toposom/tune.hpp"
#include "tsom_b200.h"

namespace toposom_b200 {

using toposom::DataMatrix;
using toposom::DataSourceRef;
using toposom::IterationAccumulators;

/// Map a C-ABI status to the reference's exception types.
inline void throw_status(int status, const char* msg) {
    const std::string m = msg ? msg : "";
    switch (status) {
        case TSOM_OK: return;
        case TSOM_ERR_INVALID: throw std::invalid_argument(m);
        case TSOM_ERR_RANGE: throw std::out_of_range(m);
        case TSOM_ERR_NUMERICAL: throw std::runtime_error(m);
        case TSOM_ERR_TIMEOUT: throw std::runtime_error(m);  // collect_with_barrier's error
        default: throw std::runtime_error("toposom_b200: " + m);
    }
}

struct Engine {
    tsom_engine* h = nullptr;
    Engine(int device, std::size_t nodes, std::size_t dims) {
        const int st = tsom_create(device, static_cast<uint32_t>(nodes), static_cast<uint32_t>(dims), &h);
        if (st) throw_status(st, "tsom_create failed (no sm_100 device?)");
    }
    ~Engine() { tsom_destroy(h); }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;
    void check(int st) const { throw_status(st, tsom_last_error(h)); }
};

/// Whether run_iteration fills the per-row distance vector (the adaptive
/// sampler needs it, trainer.hpp:511; full/random sampling ignores it).
enum class Distances { always, never };

struct CudaOptions {
    int device = 0;
    // more than one entry: one engine per entry, each owning a contiguous
    // slice of the rows (assign_shards, parallel.hpp:28-41), joined by an
    // in-process rank group with one ordered reduce per epoch — the
    // ThreadedExecutor shape (parallel.hpp:99-140) with GPUs as workers.  The
    // same device may repeat (several engines on one GPU).
    std::vector<int> devices;
    bool streamed = false;            // keep rows in host memory, stream every epoch
    Distances distances = Distances::always;
    int bmu_kernel = 0;               // 0 auto (tcgen05), 1 SIMT, 2 tcgen05
    double barrier_timeout_s = toposom::kDefaultBarrierTimeoutS;  // parallel.hpp:24
    // exact sums (TSOM_OPT_DETERMINISTIC): results bit-identical for any number
    // of engines, like the reference's for any worker count (parallel.hpp:17-21)
    bool exact = false;
    // TSOM_OPT_ROW_ORDER for the engines (-1: the engine's auto mode, which
    // re-lays the rows out only in device calls of >= 20 epochs; train_cuda
    // and train_device ask for 2 (once) when config.n_iters >= 20, since the
    // reference loop calls the executor one epoch at a time)
    int row_order = -1;
};

/// G engines joined by an in-process rank group (tsom_group_*): each owns
/// rows [slice.first, slice.second) of the data.  for_each runs a step on
/// every engine from its own thread and rethrows the first failure in engine
/// order, like collect_with_barrier (parallel.hpp:67-86); a rank that misses
/// the reduce deadline fails its peers' reduce with TSOM_ERR_TIMEOUT.
class EngineSet {
public:
    EngineSet(const DataSourceRef& data, std::size_t nodes, const CudaOptions& opts) {
        std::vector<int> devs = opts.devices;
        if (devs.empty()) devs.push_back(opts.device);
        const std::size_t G = devs.size();
        if (G > 1 && !data.in_memory())
            throw std::invalid_argument(
                "CudaExecutor: several devices need an in-memory DataMatrix (shard sources bind "
                "to one engine)");
        slices_ = toposom::assign_shards(data.rows(), G);
        if (G > 1) {
            const int st = tsom_group_create(static_cast<int>(G), &group_);
            if (st) throw_status(st, "tsom_group_create failed");
        }
        for (std::size_t g = 0; g < G; ++g) {
            engines_.push_back(std::make_unique<Engine>(devs[g], nodes, data.cols()));
            Engine& e = *engines_.back();
            if (opts.bmu_kernel)
                e.check(tsom_set_option(e.h, TSOM_OPT_BMU_KERNEL, opts.bmu_kernel));
            e.check(tsom_set_option(e.h, TSOM_OPT_BARRIER_TIMEOUT_MS,
                                    std::max<std::int64_t>(1, std::llround(opts.barrier_timeout_s * 1e3))));
            if (opts.exact) e.check(tsom_set_option(e.h, TSOM_OPT_DETERMINISTIC, 1));
            if (opts.row_order >= 0) e.check(tsom_set_option(e.h, TSOM_OPT_ROW_ORDER, opts.row_order));
            if (group_) e.check(tsom_group_join(e.h, group_, static_cast<int>(g)));
        }
        const std::uint32_t flags = opts.streamed ? TSOM_BIND_STREAMED : TSOM_BIND_COPY;
        if (data.in_memory()) {
            const DataMatrix* rows = data.matrix();
            for_each([&](std::size_t g, tsom_engine* h) {
                const auto& sl = slices_[g];
                return tsom_bind_host_data(h, rows->values.data() + sl.first * rows->cols,
                                           sl.second - sl.first, flags);
            });
        } else {
            // Shard-backed source: the engine reads the FSOMSHRD files itself
            // (copied once into HBM, or streamed from disk every epoch through
            // pinned staging), replacing the per-epoch rescans of
            // DataSourceRef::fetch_rows (dataset.hpp:400-415).
            std::vector<std::string> names;
            for (const auto& p : data.shards()->shard_paths) names.push_back(p.string());
            std::vector<const char*> cpaths;
            for (const auto& n : names) cpaths.push_back(n.c_str());
            engines_[0]->check(tsom_bind_shards(engines_[0]->h, cpaths.data(),
                                                (std::uint32_t)cpaths.size(), flags));
        }
    }
    ~EngineSet() {
        engines_.clear();
        if (group_) tsom_group_destroy(group_);
    }
    EngineSet(const EngineSet&) = delete;
    EngineSet& operator=(const EngineSet&) = delete;

    std::size_t size() const { return engines_.size(); }
    tsom_engine* handle(std::size_t g) const { return engines_[g]->h; }
    const std::pair<std::size_t, std::size_t>& slice(std::size_t g) const { return slices_[g]; }

    /// f(g, engine) -> C-ABI status, on every engine concurrently (inline when G = 1)
    template <typename F>
    void for_each(F&& f) {
        const std::size_t G = engines_.size();
        if (G == 1) {
            engines_[0]->check(f(std::size_t{0}, engines_[0]->h));
            return;
        }
        std::vector<std::future<int>> fut;
        fut.reserve(G);
        for (std::size_t g = 0; g < G; ++g)
            fut.push_back(std::async(std::launch::async, [&f, g, this] { return f(g, engines_[g]->h); }));
        std::vector<int> st(G);
        for (std::size_t g = 0; g < G; ++g) st[g] = fut[g].get();
        // the first failure in worker order; a peer's "aborted" follows a timeout
        for (int pass = 0; pass < 2; ++pass)
            for (std::size_t g = 0; g < G; ++g)
                if (st[g] != TSOM_OK) {
                    const char* m = tsom_last_error(engines_[g]->h);
                    if (pass == 0 && std::strncmp(m, "reduce barrier aborted", 22) == 0) continue;
                    throw_status(st[g], m);
                }
    }

private:
    std::vector<std::pair<std::size_t, std::size_t>> slices_;
    tsom_group* group_ = nullptr;
    std::vector<std::unique_ptr<Engine>> engines_;
};

/// Convert the engine's float64 U/H into the reference's fixed-point
/// accumulators (accum.hpp:45-53): value * 2^40 rounded to nearest.
inline toposom::AccumInt to_fixed(double v) {
    if (!std::isfinite(v))
        throw std::runtime_error("numerical fault: accumulation term out of range (|term| >= 2^22)");
    const double q = std::nearbyint(v * toposom::kAccumScale);
    return static_cast<toposom::AccumInt>(q);
}

class CudaExecutor {
public:
    CudaExecutor(const DataSourceRef& data, std::size_t nodes, const CudaOptions& opts = {})
        : opts_(opts), set_(data, nodes, opts), nodes_(nodes), dims_(data.cols()) {}

    /// Executor::run_iteration (trainer.hpp:446-453): one accumulation pass
    /// plus the single reduce.  n_chunks is result-invariant by contract
    /// (test_trainer.cpp:315-333) and therefore not used.  With several
    /// engines the sorted selection is split by row owner (each engine gets
    /// the ids in its slice, made local), every engine runs its pass from its
    /// own thread, the ranks' sums meet in one ordered reduce, and the
    /// distances land in selection order (the slices are contiguous).
    IterationAccumulators run_iteration(const std::vector<std::uint32_t>& selected,
                                        const DataMatrix& weights,
                                        const std::vector<double>& influence, double eta,
                                        std::size_t /*n_chunks*/, std::vector<double>& distances) {
        if (weights.rows != nodes_ || weights.cols != dims_)
            throw std::invalid_argument("accumulate: accumulator shape mismatch");
        if (influence.size() != nodes_ * nodes_)
            throw std::invalid_argument("accumulate: influence shape mismatch");
        const std::size_t G = set_.size();
        // the reference's loop hands in cached_influence(...) (topology.hpp:406-418):
        // upload only when its content changed (compared, not keyed by address)
        const bool new_infl = influence != infl_;
        if (new_infl) infl_ = influence;
        for (std::uint32_t id : selected)
            if (id >= set_.slice(G - 1).second)
                throw std::out_of_range("fetch_rows: row index beyond data size");
        u_.resize(nodes_ * dims_);
        h_.resize(nodes_);
        distances.clear();
        const bool want_dist = opts_.distances == Distances::always;
        if (want_dist) distances.resize(selected.size());
        // selection split by owner (sorted ids: one lower_bound per slice)
        std::vector<std::size_t> p(G + 1, selected.size());
        p[0] = 0;
        for (std::size_t g = 1; g < G; ++g)
            p[g] = static_cast<std::size_t>(
                std::lower_bound(selected.begin(), selected.end(),
                                 static_cast<std::uint32_t>(set_.slice(g).first)) -
                selected.begin());
        local_.resize(G);
        set_.for_each([&](std::size_t g, tsom_engine* h) {
            int st = tsom_set_codebook(h, weights.values.data());
            if (!st && new_infl) st = tsom_set_influence(h, influence.data(), -1);
            if (st) return st;
            static const std::uint32_t kNone = 0;  // non-null + n_sel 0 = empty selection
            const std::uint32_t* sel = &kNone;
            const std::size_t n = p[g + 1] - p[g];
            if (G == 1) {
                if (n) sel = selected.data();
            } else if (n) {
                const std::uint32_t o = static_cast<std::uint32_t>(set_.slice(g).first);
                local_[g].assign(selected.begin() + p[g], selected.begin() + p[g + 1]);
                for (auto& v : local_[g]) v -= o;
                sel = local_[g].data();
            }
            return tsom_epoch(h, sel, n, eta, g == 0 ? u_.data() : nullptr,
                              g == 0 ? h_.data() : nullptr,
                              want_dist ? distances.data() + p[g] : nullptr);
        });
        IterationAccumulators acc(nodes_, dims_);
        for (std::size_t i = 0; i < u_.size(); ++i) acc.u[i] = to_fixed(u_[i]);
        for (std::size_t j = 0; j < nodes_; ++j) acc.h[j] = to_fixed(h_[j]);
        return acc;
    }

    std::size_t workers() const { return set_.size(); }
    /// seconds rank 0 spent waiting in the reduce (ThreadedExecutor::barrier_wait_s)
    double barrier_wait_s() const { return tsom_barrier_wait_s(set_.handle(0)); }
    tsom_engine* engine() const { return set_.handle(0); }
    EngineSet& engines() { return set_; }

private:
    CudaOptions opts_;
    EngineSet set_;
    std::size_t nodes_, dims_;
    std::vector<double> u_, h_, infl_;
    std::vector<std::vector<std::uint32_t>> local_;
};

/// GPU analogue of toposom::train / train_parallel (trainer.hpp:526-530,
/// parallel.hpp:145-152).  Distances are only produced when the sampler needs
/// them (adaptive), unless the caller forces them.
inline std::pair<toposom::SomModel, toposom::RunLog> train_cuda(
    const toposom::SomConfig& config, const DataSourceRef& data, toposom::Sampler& sampler,
    CudaOptions opts = {}, const toposom::TrainOptions& options = {}) {
    if (sampler.kind() != toposom::SamplingKind::adaptive) opts.distances = Distances::never;
    if (data.rows() < 1) throw std::invalid_argument("train: empty training data");
    if (opts.row_order < 0 && config.n_iters >= 20) opts.row_order = 2;  // a long run
    CudaExecutor executor(data, config.nodes(), opts);
    return toposom::train_with_executor(config, data, sampler, executor, options);
}

/// The sampler of a device-resident run: the arguments of toposom::Sampler
/// (sampling.hpp:185-191) except n (the data's rows) and the seed (the
/// config's, as train_with_executor's callers use it).
struct DeviceSampling {
    toposom::SamplingKind kind = toposom::SamplingKind::full;
    toposom::SamplingBudget budget{};
    double alpha = 1.0;
    double beta = 1.0;
};

/// train_with_executor (trainer.hpp:466-523) with every step of every epoch
/// on the device: init_weights and the lattice distances on the host as the
/// reference builds them, then selection (device sampler), topology refresh
/// on the reference's schedule (device MST / RNG graph and hop counts),
/// influence, BMU, accumulation, smoothing and apply_update.  The epochs
/// between two refreshes go to the engine as one tsom_train_epochs call (no
/// host round trip between them); with options.log_qe each epoch is its own
/// call followed by the device QE.  options.timeout_s is checked between
/// calls.  Returns the reference's (SomModel, RunLog): weights, momentum
/// memory, topology state (edges, hop counts and refresh counters of the last
/// refresh for graphs) and one log entry per epoch.  With opts.devices the
/// rows are split over several engines (EngineSet) that run every step in
/// lockstep from their own threads: one ordered reduce per epoch, one sharded
/// device sampler over all rows, identical refreshes and updates on every
/// engine (the multi-GPU epoch of SURVEY.md §8(e)).
inline std::pair<toposom::SomModel, toposom::RunLog> train_device(
    const toposom::SomConfig& config, const DataSourceRef& data, DeviceSampling sampling = {},
    CudaOptions opts = {}, const toposom::TrainOptions& options = {}) {
    config.validate();
    if (data.rows() < 1) throw std::invalid_argument("train: empty training data");
    toposom::SomModel model;
    model.weights = toposom::init_weights(config, data);
    model.prev_update = DataMatrix(config.nodes(), data.cols());
    model.topology_state = toposom::build_topology(config.topology);
    opts.distances = Distances::never;
    if (opts.row_order < 0 && config.n_iters >= 20) opts.row_order = 2;  // a long run
    EngineSet es(data, config.nodes(), opts);  // engines + their rows (resident or streamed)
    tsom_engine* h = es.handle(0);
    auto check = [h](int st) { throw_status(st, tsom_last_error(h)); };
    toposom::TopologyState& ts = model.topology_state;
    const bool lattice = toposom::is_lattice(config.topology.kind);
    const bool sampled = sampling.kind != toposom::SamplingKind::full;
    const std::uint64_t m_sel = sampled ? toposom::resolve_budget(sampling.budget, data.rows()) : 0;
    es.for_each([&](std::size_t, tsom_engine* e) {
        int st = tsom_set_codebook(e, model.weights.values.data());
        if (!st && lattice) st = tsom_set_topology_distance(e, ts.lattice_distances.data());
        // one Sampler over all rows; with several engines it is sharded over them
        if (!st && sampled)
            st = tsom_sampler_init(e, static_cast<int>(sampling.kind), m_sel, config.seed,
                                   sampling.alpha, sampling.beta);
        return st;
    });
    // schedules and refresh points depend only on t; the refresh counters are
    // advanced exactly as refresh_topology does (topology.hpp:442-451)
    const toposom::RefreshPolicy policy = config.resolved_refresh();
    const double sigma0 = config.resolved_sigma0();
    const std::size_t total = config.n_iters;
    std::vector<double> etas(total), sigmas(total);
    std::vector<char> refresh(total, 0);
    for (std::size_t t = 0; t < total; ++t) {
        etas[t] = toposom::schedule_value(config.eta0, config.lr_decay, t, total,
                                          toposom::kEtaFloor);
        sigmas[t] = toposom::schedule_value(sigma0, config.radius_decay, t, total,
                                            config.sigma_min);
        if (toposom::should_refresh(policy, t, ts)) {
            refresh[t] = 1;
            ts.last_refresh_iter = static_cast<std::int64_t>(t);
            ++ts.refresh_count;
            if (t >= policy.warmup_iters) ++ts.post_warmup_refreshes;
        }
    }
    const std::size_t P = config.nodes();
    std::vector<std::uint32_t> edges(lattice ? 0 : P * (P - 1));
    std::vector<std::uint16_t> hops(lattice ? 0 : P * P);
    std::uint64_t n_edges = 0;
    const std::uint32_t flags = (config.use_momentum ? 1u : 0u) | (sampled ? 2u : 0u);
    toposom::RunLog log;
    const auto run_start = std::chrono::steady_clock::now();
    for (std::size_t t = 0; t < total;) {
        if (options.timeout_s > 0.0) {
            const std::chrono::duration<double> el = std::chrono::steady_clock::now() - run_start;
            if (el.count() > options.timeout_s)
                throw toposom::TrainTimeoutError("training run exceeded timeout of " +
                                                 std::to_string(options.timeout_s) +
                                                 " s at iteration " + std::to_string(t));
        }
        if (refresh[t])
            es.for_each([&](std::size_t g, tsom_engine* e) {
                return g == 0 ? tsom_refresh_topology(e, static_cast<int>(config.topology.kind),
                                                      edges.data(), edges.size() / 2, &n_edges,
                                                      hops.data())
                              : tsom_refresh_topology(e, static_cast<int>(config.topology.kind),
                                                      nullptr, 0, nullptr, nullptr);
            });
        std::size_t t1 = t + 1;
        if (!options.log_qe)
            while (t1 < total && !refresh[t1]) ++t1;
        es.for_each([&](std::size_t, tsom_engine* e) {
            std::uint32_t failed = 0;
            return tsom_train_epochs(e, static_cast<std::uint32_t>(t1 - t), etas.data() + t,
                                     sigmas.data() + t, config.momentum, flags, &failed);
        });
        for (std::size_t u = t; u < t1; ++u) {
            toposom::IterationLogEntry e;
            e.iter = u;
            e.eta = etas[u];
            e.sigma = sigmas[u];
            e.refreshed = refresh[u] != 0;
            log.iterations.push_back(e);
        }
        if (options.log_qe) {
            double sum = 0.0;
            std::uint64_t count = 0;
            es.for_each([&](std::size_t g, tsom_engine* e) {
                double s2 = 0.0;
                std::uint64_t c2 = 0;
                return g == 0 ? tsom_qe(e, nullptr, 0, &sum, &count) : tsom_qe(e, nullptr, 0, &s2, &c2);
            });
            log.iterations.back().qe_train = sum / static_cast<double>(count);
        }
        t = t1;
    }
    log.reduce_count = total;
    check(tsom_get_codebook(h, model.weights.values.data()));
    check(tsom_get_prev_update(h, model.prev_update.values.data()));
    if (!lattice) {
        ts.edges.clear();
        for (std::uint64_t k = 0; k < n_edges; ++k) ts.edges.emplace_back(edges[2 * k], edges[2 * k + 1]);
        ts.hop_dist = std::move(hops);
    }
    model.iter = total;
    return {std::move(model), std::move(log)};
}

/// find_bmus (trainer.hpp:282-308) on the GPU; bit-identical BMU indices.
inline void find_bmus_cuda(const DataMatrix& chunk, const DataMatrix& weights,
                           std::vector<std::uint32_t>& bmus, std::vector<double>& distances,
                           int device = 0) {
    if (chunk.cols != weights.cols) throw std::invalid_argument("find_bmus: dimension mismatch");
    bmus.resize(chunk.rows);
    distances.resize(chunk.rows);
    if (chunk.rows == 0) return;
    Engine eng(device, weights.rows, weights.cols);
    eng.check(tsom_set_codebook(eng.h, weights.values.data()));
    eng.check(tsom_bmu(eng.h, chunk.values.data(), chunk.rows, bmus.data(), distances.data()));
}

/// quantization_error (metrics.hpp:28-30) on the GPU.
inline double quantization_error_cuda(const toposom::SomModel& model, const DataMatrix& data,
                                      int device = 0) {
    if (data.cols != model.weights.cols)
        throw std::invalid_argument("mean_bmu_distance: dimension mismatch");
    if (data.rows == 0) throw std::invalid_argument("mean_bmu_distance: empty data");
    Engine eng(device, model.weights.rows, model.weights.cols);
    eng.check(tsom_set_codebook(eng.h, model.weights.values.data()));
    eng.check(tsom_bind_host_data(eng.h, data.values.data(), data.rows, TSOM_BIND_COPY));
    double sum = 0.0;
    uint64_t count = 0;
    eng.check(tsom_qe(eng.h, nullptr, 0, &sum, &count));
    return sum / static_cast<double>(count);
}

/// run_study (tune.hpp:125-159) with every trial trained by the GPU executor
/// and scored by the GPU QE.  Trials are the reference's (sample_trial with
/// Rng(mix_seed(seed, trial), SeedStream::trial), tune.hpp:77-93, 140-143) and
/// come back in the reference's order (seed-major); up to `concurrency` trials
/// run at once, each on its own engine and CUDA stream, so the many small
/// trainings of a search overlap on the device.  A failing trial records the
/// +infinity sentinel and the study continues, as in the reference.
inline std::vector<toposom::TrialRecord> run_study_cuda(
    const toposom::SearchSpace& space, const toposom::StudySpec& spec,
    const DataMatrix& train_data, const DataMatrix& holdout_data, unsigned concurrency = 4,
    CudaOptions opts = {}) {
    using Record = toposom::TrialRecord;
    if (spec.n_trials < 1) throw std::invalid_argument("run_study: n_trials must be >= 1");
    if (spec.seeds.empty()) throw std::invalid_argument("run_study: need at least one seed");
    space.validate();
    std::vector<Record> records;
    for (const std::uint64_t seed : spec.seeds)
        for (std::size_t trial = 0; trial < spec.n_trials; ++trial) {
            toposom::Rng trial_rng(toposom::mix_seed(seed, trial), toposom::SeedStream::trial);
            Record rec;
            rec.seed = seed;
            rec.trial_index = trial;
            rec.config = toposom::sample_trial(space, spec.base_config, trial_rng);
            rec.config.seed = seed;
            records.push_back(std::move(rec));
        }
    std::atomic<std::size_t> next{0};
    auto worker = [&] {
        for (std::size_t i = next++; i < records.size(); i = next++) {
            Record& rec = records[i];
            try {
                toposom::Sampler sampler(spec.sampling, spec.budget, train_data.rows, rec.seed,
                                         spec.sampler_alpha, spec.sampler_beta);
                auto result = train_cuda(rec.config, train_data, sampler, opts);
                rec.qe_train = quantization_error_cuda(result.first, train_data, opts.device);
                rec.qe_holdout = quantization_error_cuda(result.first, holdout_data, opts.device);
            } catch (const std::exception& e) {
                rec.failed = true;
                rec.failure = e.what();
                rec.qe_train = std::numeric_limits<double>::infinity();
                rec.qe_holdout = std::numeric_limits<double>::infinity();
            }
        }
    };
    std::vector<std::thread> pool;
    const unsigned T = std::max(1u, std::min<unsigned>(concurrency, (unsigned)records.size()));
    for (unsigned t = 1; t < T; ++t) pool.emplace_back(worker);
    worker();
    for (auto& th : pool) th.join();
    return records;
}

}  // namespace toposom_b200
