// dropin.cpp — the reference training loop driving the B200 engine.
//
// Built only where the reference headers exist (the maintainer's build): it
// instantiates toposom::train_with_executor (trainer.hpp:466-523) with
// toposom_b200::CudaExecutor (include/toposom_b200/cuda_executor.hpp) and
// exports a flat C entry with the same config layout as oracle/_ref's
// ref_train, so tests and bench.py can run the identical reference loop with
// the GPU executor swapped in.  No kernel code lives here.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>

#include "toposom_b200/cuda_executor.hpp"

using namespace toposom;

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 3;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}
}  // namespace

struct dropin_config {  // layout shared with oracle/_ref ref_config
    int topology;
    std::uint64_t grid_w, grid_h, nodes;
    std::uint64_t n_iters;
    double eta0;
    int lr_exponential;
    double sigma0;
    int radius_exponential;
    double sigma_min;
    int init_method;
    int use_momentum;
    double momentum;
    std::uint64_t refresh_warmup;
    double refresh_growth;
    std::uint64_t refresh_max_interval;
    std::uint64_t n_chunks;
    std::uint64_t seed;
    int sampling;
    int budget_fixed;
    std::uint64_t m0;
    double rho;
    double alpha, beta;
    int n_threads;
};

extern "C" {

const char* tsom_dropin_last_error() { return g_err.c_str(); }
std::size_t tsom_dropin_config_sizeof() { return sizeof(dropin_config); }

// flags: bit0 streamed, bits1-2 bmu kernel (0 auto, 1 simt, 2 tc), bit3 force distances
static SomConfig make_config(const dropin_config* rc) {
        SomConfig c;
        const auto kind = static_cast<TopologyKind>(rc->topology);
        c.topology = is_lattice(kind) ? TopologySpec::lattice(kind, rc->grid_w, rc->grid_h)
                                      : TopologySpec::graph(kind, rc->nodes);
        c.n_iters = rc->n_iters;
        c.eta0 = rc->eta0;
        c.lr_decay = rc->lr_exponential ? DecayKind::exponential : DecayKind::linear;
        c.sigma0 = rc->sigma0;
        c.radius_decay = rc->radius_exponential ? DecayKind::exponential : DecayKind::linear;
        c.sigma_min = rc->sigma_min;
        c.init_method = rc->init_method == 1 ? InitMethod::uniform_box
                        : rc->init_method == 2 ? InitMethod::pca_plane
                                               : InitMethod::sample_draw;
        c.use_momentum = rc->use_momentum != 0;
        c.momentum = rc->momentum;
        c.refresh.warmup_iters = rc->refresh_warmup;
        c.refresh.growth = rc->refresh_growth;
        c.refresh.max_interval = rc->refresh_max_interval;
        c.n_chunks = rc->n_chunks;
        c.seed = rc->seed;
        return c;
}

static Sampler make_sampler(const dropin_config* rc, std::size_t n, std::uint64_t seed) {
        SamplingBudget b;
        b.mode = rc->budget_fixed ? BudgetMode::fixed : BudgetMode::proportional;
        b.m0 = rc->m0;
        b.rho = rc->rho;
        return Sampler(static_cast<SamplingKind>(rc->sampling), b, n, seed, rc->alpha, rc->beta);
}

// Executor wrapper that times run_iteration (flags bit 4: profile breakdown)
struct TimedExecutor {
    toposom_b200::CudaExecutor& ex;
    double iter_s = 0.0;
    IterationAccumulators run_iteration(const std::vector<std::uint32_t>& selected,
                                        const DataMatrix& weights, const std::vector<double>& infl,
                                        double eta, std::size_t n_chunks,
                                        std::vector<double>& distances) {
        const auto t0 = std::chrono::steady_clock::now();
        auto acc = ex.run_iteration(selected, weights, infl, eta, n_chunks, distances);
        iter_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return acc;
    }
    std::size_t workers() const { return ex.workers(); }
    double barrier_wait_s() const { return ex.barrier_wait_s(); }
};

// train_with_executor + CudaExecutor over any DataSourceRef (in-memory or ShardSet)
static void run_train(const dropin_config* rc, const DataSourceRef& src, float* weights_out,
                      double* qe_log, std::uint8_t* refresh_log, int device, unsigned flags,
                      double* seconds_out) {
        SomConfig c = make_config(rc);
        Sampler sampler = make_sampler(rc, src.rows(), c.seed);
        toposom_b200::CudaOptions opts;
        opts.device = device;
        opts.streamed = (flags & 1u) != 0;
        opts.bmu_kernel = static_cast<int>((flags >> 1) & 3u);
        // bits 8-11: engines (one per row slice, all on `device`); 0 = 1
        const unsigned engines = (flags >> 8) & 15u;
        if (engines > 1) opts.devices.assign(engines, device);
        // bits 12-27: reduce-barrier timeout in ms (0 = the reference's 60 s)
        if ((flags >> 12) & 0xFFFFu) opts.barrier_timeout_s = ((flags >> 12) & 0xFFFFu) / 1000.0;
        opts.exact = (flags >> 28) & 1u;  // bit 28: exact sums
        TrainOptions to;
        to.log_qe = qe_log != nullptr;
        const auto t0 = std::chrono::steady_clock::now();
        std::pair<SomModel, RunLog> result;
        if (flags & 32u) {
            // every step on the device (toposom_b200::train_device)
            toposom_b200::DeviceSampling ds;
            ds.kind = static_cast<SamplingKind>(rc->sampling);
            ds.budget.mode = rc->budget_fixed ? BudgetMode::fixed : BudgetMode::proportional;
            ds.budget.m0 = rc->m0;
            ds.budget.rho = rc->rho;
            ds.alpha = rc->alpha;
            ds.beta = rc->beta;
            result = toposom_b200::train_device(c, src, ds, opts, to);
        } else if (flags & 16u) {
            // profile: seconds_out[1] = executor construction (bind), [2] = run_iteration
            if (sampler.kind() != SamplingKind::adaptive && !(flags & 8u))
                opts.distances = toposom_b200::Distances::never;
            toposom_b200::CudaExecutor ex(src, c.nodes(), opts);
            const auto t1 = std::chrono::steady_clock::now();
            TimedExecutor tex{ex};
            result = train_with_executor(c, src, sampler, tex, to);
            if (seconds_out) {
                seconds_out[1] = std::chrono::duration<double>(t1 - t0).count();
                seconds_out[2] = tex.iter_s;
            }
        } else if (flags & 8u) {
            opts.distances = toposom_b200::Distances::always;
            toposom_b200::CudaExecutor ex(src, c.nodes(), opts);
            result = train_with_executor(c, src, sampler, ex, to);
        } else {
            result = toposom_b200::train_cuda(c, src, sampler, opts, to);
        }
        const std::chrono::duration<double> dt = std::chrono::steady_clock::now() - t0;
        if (seconds_out) *seconds_out = dt.count();
        std::memcpy(weights_out, result.first.weights.values.data(),
                    result.first.weights.values.size() * sizeof(float));
        for (std::size_t t = 0; t < result.second.iterations.size(); ++t) {
            if (qe_log) qe_log[t] = *result.second.iterations[t].qe_train;
            if (refresh_log) refresh_log[t] = result.second.iterations[t].refreshed ? 1 : 0;
        }
}

int tsom_dropin_train(const dropin_config* rc, const float* data, std::size_t n, std::size_t d,
                      float* weights_out, double* qe_log, std::uint8_t* refresh_log, int device,
                      unsigned flags, double* seconds_out) {
    return guarded([&] {
        // DataMatrix over the caller's rows (one host copy, as DataSourceRef needs a matrix)
        DataMatrix mat(n, d, std::vector<float>(data, data + n * d));
        run_train(rc, mat, weights_out, qe_log, refresh_log, device, flags, seconds_out);
    });
}

// Same loop over a directory of part-*.shard files (open_shards, dataset.hpp:277-302)
int tsom_dropin_train_shards(const dropin_config* rc, const char* shard_dir, std::size_t chunk_rows,
                             float* weights_out, double* qe_log, std::uint8_t* refresh_log,
                             int device, unsigned flags, double* seconds_out) {
    return guarded([&] {
        ShardSet set = open_shards(shard_dir, chunk_rows);
        DataSourceRef src(set);
        run_train(rc, src, weights_out, qe_log, refresh_log, device, flags, seconds_out);
    });
}

// run_study (tune.hpp:125-159) with GPU trials: default SearchSpace, the base
// config and sampler from rc; records in the reference's order.
int tsom_dropin_run_study(const dropin_config* rc, std::size_t n_trials, const std::uint64_t* seeds,
                          std::size_t n_seeds, const float* train, std::size_t n,
                          const float* holdout, std::size_t nh, std::size_t d, int device,
                          unsigned concurrency, double* qe_train, double* qe_holdout,
                          std::uint8_t* failed, double* seconds_out) {
    return guarded([&] {
        DataMatrix tm(n, d, std::vector<float>(train, train + n * d));
        DataMatrix hm(nh, d, std::vector<float>(holdout, holdout + nh * d));
        StudySpec spec;
        spec.base_config = make_config(rc);
        spec.sampling = static_cast<SamplingKind>(rc->sampling);
        spec.budget.mode = rc->budget_fixed ? BudgetMode::fixed : BudgetMode::proportional;
        spec.budget.m0 = rc->m0;
        spec.budget.rho = rc->rho;
        spec.sampler_alpha = rc->alpha;
        spec.sampler_beta = rc->beta;
        spec.n_trials = n_trials;
        spec.seeds.assign(seeds, seeds + n_seeds);
        toposom_b200::CudaOptions opts;
        opts.device = device;
        const auto t0 = std::chrono::steady_clock::now();
        const auto recs = toposom_b200::run_study_cuda(SearchSpace{}, spec, tm, hm, concurrency, opts);
        const std::chrono::duration<double> dt = std::chrono::steady_clock::now() - t0;
        if (seconds_out) *seconds_out = dt.count();
        for (std::size_t i = 0; i < recs.size(); ++i) {
            qe_train[i] = recs[i].qe_train;
            qe_holdout[i] = recs[i].qe_holdout;
            failed[i] = recs[i].failed ? 1 : 0;
        }
    });
}

// write_shards (dataset.hpp:252-275), for tests and benches that need shard files
int tsom_dropin_write_shards(const float* data, std::size_t n, std::size_t d, const char* out_dir,
                             std::size_t n_shards) {
    return guarded([&] {
        DataMatrix mat(n, d, std::vector<float>(data, data + n * d));
        write_shards(mat, out_dir, n_shards, 4096);
    });
}

// find_bmus through the drop-in helper
int tsom_dropin_find_bmus(const float* x, std::size_t n, const float* w, std::size_t p,
                          std::size_t d, std::uint32_t* bmus, double* dists, int device) {
    return guarded([&] {
        DataMatrix chunk(n, d, std::vector<float>(x, x + n * d));
        DataMatrix weights(p, d, std::vector<float>(w, w + p * d));
        std::vector<std::uint32_t> b;
        std::vector<double> dd;
        toposom_b200::find_bmus_cuda(chunk, weights, b, dd, device);
        std::memcpy(bmus, b.data(), n * sizeof(std::uint32_t));
        std::memcpy(dists, dd.data(), n * sizeof(double));
    });
}

}  // extern "C"
