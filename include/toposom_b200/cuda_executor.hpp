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
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "toposom/metrics.hpp"
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
    bool streamed = false;            // keep rows in host memory, stream every epoch
    Distances distances = Distances::always;
    int bmu_kernel = 0;               // 0 auto (tcgen05), 1 SIMT, 2 tcgen05
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
        : opts_(opts), eng_(std::make_unique<Engine>(opts.device, nodes, data.cols())),
          nodes_(nodes), dims_(data.cols()) {
        if (opts.bmu_kernel) eng_->check(tsom_set_option(eng_->h, TSOM_OPT_BMU_KERNEL, opts.bmu_kernel));
        if (data.in_memory()) {
            rows_ = data.matrix();
            eng_->check(tsom_bind_host_data(eng_->h, rows_->values.data(), rows_->rows,
                                            opts.streamed ? TSOM_BIND_STREAMED : TSOM_BIND_COPY));
        } else {
            // Shard-backed source: the engine reads the FSOMSHRD files itself
            // (copied once into HBM, or streamed from disk every epoch through
            // pinned staging), replacing the per-epoch rescans of
            // DataSourceRef::fetch_rows (dataset.hpp:400-415).
            std::vector<std::string> names;
            for (const auto& p : data.shards()->shard_paths) names.push_back(p.string());
            std::vector<const char*> cpaths;
            for (const auto& n : names) cpaths.push_back(n.c_str());
            eng_->check(tsom_bind_shards(eng_->h, cpaths.data(), (std::uint32_t)cpaths.size(),
                                         opts.streamed ? TSOM_BIND_STREAMED : TSOM_BIND_COPY));
        }
    }

    /// Executor::run_iteration (trainer.hpp:446-453): one accumulation pass
    /// plus the single reduce.  n_chunks is result-invariant by contract
    /// (test_trainer.cpp:315-333) and therefore not used.
    IterationAccumulators run_iteration(const std::vector<std::uint32_t>& selected,
                                        const DataMatrix& weights,
                                        const std::vector<double>& influence, double eta,
                                        std::size_t /*n_chunks*/, std::vector<double>& distances) {
        if (weights.rows != nodes_ || weights.cols != dims_)
            throw std::invalid_argument("accumulate: accumulator shape mismatch");
        if (influence.size() != nodes_ * nodes_)
            throw std::invalid_argument("accumulate: influence shape mismatch");
        eng_->check(tsom_set_codebook(eng_->h, weights.values.data()));
        eng_->check(tsom_set_influence(eng_->h, influence.data(), -1));
        u_.resize(nodes_ * dims_);
        h_.resize(nodes_);
        distances.clear();
        double* dist_out = nullptr;
        if (opts_.distances == Distances::always) {
            distances.resize(selected.size());
            dist_out = distances.data();
        }
        static const std::uint32_t kNone = 0;  // non-null + n_sel 0 = empty selection
        const std::uint32_t* sel = selected.empty() ? &kNone : selected.data();
        eng_->check(tsom_epoch(eng_->h, sel, selected.size(), eta, u_.data(), h_.data(), dist_out));
        IterationAccumulators acc(nodes_, dims_);
        for (std::size_t i = 0; i < u_.size(); ++i) acc.u[i] = to_fixed(u_[i]);
        for (std::size_t j = 0; j < nodes_; ++j) acc.h[j] = to_fixed(h_[j]);
        return acc;
    }

    std::size_t workers() const { return 1; }
    double barrier_wait_s() const { return 0.0; }
    tsom_engine* engine() const { return eng_->h; }

private:
    CudaOptions opts_;
    std::unique_ptr<Engine> eng_;
    std::size_t nodes_, dims_;
    const DataMatrix* rows_ = nullptr;
    std::vector<double> u_, h_;
};

/// GPU analogue of toposom::train / train_parallel (trainer.hpp:526-530,
/// parallel.hpp:145-152).  Distances are only produced when the sampler needs
/// them (adaptive), unless the caller forces them.
inline std::pair<toposom::SomModel, toposom::RunLog> train_cuda(
    const toposom::SomConfig& config, const DataSourceRef& data, toposom::Sampler& sampler,
    CudaOptions opts = {}, const toposom::TrainOptions& options = {}) {
    if (sampler.kind() != toposom::SamplingKind::adaptive) opts.distances = Distances::never;
    if (data.rows() < 1) throw std::invalid_argument("train: empty training data");
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
/// refresh for graphs) and one log entry per epoch.
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
    CudaExecutor ex(data, config.nodes(), opts);  // engine + rows (resident or streamed)
    tsom_engine* h = ex.engine();
    auto check = [h](int st) { throw_status(st, tsom_last_error(h)); };
    check(tsom_set_codebook(h, model.weights.values.data()));
    toposom::TopologyState& ts = model.topology_state;
    const bool lattice = toposom::is_lattice(config.topology.kind);
    if (lattice) check(tsom_set_topology_distance(h, ts.lattice_distances.data()));
    const bool sampled = sampling.kind != toposom::SamplingKind::full;
    if (sampled)
        check(tsom_sampler_init(h, static_cast<int>(sampling.kind),
                                toposom::resolve_budget(sampling.budget, data.rows()), config.seed,
                                sampling.alpha, sampling.beta));
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
            check(tsom_refresh_topology(h, static_cast<int>(config.topology.kind), edges.data(),
                                        edges.size() / 2, &n_edges, hops.data()));
        std::size_t t1 = t + 1;
        if (!options.log_qe)
            while (t1 < total && !refresh[t1]) ++t1;
        std::uint32_t failed = 0;
        check(tsom_train_epochs(h, static_cast<std::uint32_t>(t1 - t), etas.data() + t,
                                sigmas.data() + t, config.momentum, flags, &failed));
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
            check(tsom_qe(h, nullptr, 0, &sum, &count));
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
