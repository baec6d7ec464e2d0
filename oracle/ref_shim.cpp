// ref_shim.cpp — C entry points over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY (see oracle/tsom_oracle.c header).  This file holds
// no reference code: it #includes the reference's own headers from
// /root/reference/proj/include at build time (oracle/Makefile) and exposes a
// flat C ABI so the Python tests and bench.py's CPU leg can run the reference
// itself.  The built library lands in oracle/_ref/ (git-ignored).
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "toposom/metrics.hpp"
#include "toposom/parallel.hpp"
#include "toposom/trainer.hpp"
#include "toposom/tune.hpp"

using namespace toposom;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, 1);
    } catch (const std::out_of_range& e) {
        return fail(e, 3);
    } catch (const std::runtime_error& e) {
        return fail(e, 2);
    } catch (const std::exception& e) {
        return fail(e, 9);
    }
}

DataMatrix make_matrix(const float* v, std::size_t rows, std::size_t cols) {
    return DataMatrix(rows, cols, std::vector<float>(v, v + rows * cols));
}
}  // namespace

// Same layout as orc_config in tsom_oracle.c.
struct ref_config {
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

const char* ref_last_error() { return g_err.c_str(); }
std::size_t ref_config_sizeof() { return sizeof(ref_config); }

int ref_find_bmus(const float* x, std::size_t n, const float* w, std::size_t p, std::size_t d,
                  std::uint32_t* bmus, double* dists) {
    return guarded([&] {
        const auto chunk = make_matrix(x, n, d);
        const auto weights = make_matrix(w, p, d);
        std::vector<std::uint32_t> b;
        std::vector<double> dd;
        find_bmus(chunk, weights, b, dd);
        std::memcpy(bmus, b.data(), n * sizeof(std::uint32_t));
        if (dists) std::memcpy(dists, dd.data(), n * sizeof(double));
    });
}

int ref_mean_bmu_distance(const float* x, std::size_t n, const float* w, std::size_t p,
                          std::size_t d, double* out) {
    return guarded([&] {
        const auto data = make_matrix(x, n, d);
        const auto weights = make_matrix(w, p, d);
        *out = mean_bmu_distance(DataSourceRef(data), weights);
    });
}

// One iteration through the reference executors (SerialExecutor for workers==1,
// ThreadedExecutor otherwise).  u_raw/h_raw: int128 as (hi, lo) int64 pairs.
int ref_run_iteration(const float* data, std::size_t n_rows, std::size_t d,
                      const std::uint32_t* sel, std::size_t n_sel, const float* w, std::size_t p,
                      const double* infl, double eta, std::size_t n_chunks, std::size_t workers,
                      double* u_out, double* h_out, std::int64_t* u_raw, std::int64_t* h_raw,
                      double* dist_out) {
    return guarded([&] {
        const auto mat = make_matrix(data, n_rows, d);
        const DataSourceRef src(mat);
        const auto weights = make_matrix(w, p, d);
        const std::vector<double> influence(infl, infl + p * p);
        const std::vector<std::uint32_t> selected(sel, sel + n_sel);
        std::vector<double> dist;
        IterationAccumulators acc;
        if (workers <= 1) {
            SerialExecutor ex(src);
            acc = ex.run_iteration(selected, weights, influence, eta, n_chunks, dist);
        } else {
            ThreadedExecutor ex(src, workers);
            acc = ex.run_iteration(selected, weights, influence, eta, n_chunks, dist);
        }
        for (std::size_t i = 0; i < p * d; ++i) {
            if (u_out) u_out[i] = acc.u_value(i / d, i % d);
            if (u_raw) {
                u_raw[2 * i] = static_cast<std::int64_t>(acc.u[i] >> 64);
                u_raw[2 * i + 1] = static_cast<std::int64_t>(static_cast<std::uint64_t>(acc.u[i]));
            }
        }
        for (std::size_t j = 0; j < p; ++j) {
            if (h_out) h_out[j] = acc.h_value(j);
            if (h_raw) {
                h_raw[2 * j] = static_cast<std::int64_t>(acc.h[j] >> 64);
                h_raw[2 * j + 1] = static_cast<std::int64_t>(static_cast<std::uint64_t>(acc.h[j]));
            }
        }
        if (dist_out) std::memcpy(dist_out, dist.data(), dist.size() * sizeof(double));
    });
}

// apply_update on exact int128 accumulators passed as (hi, lo) int64 pairs.
int ref_apply_update(float* w, float* prev, std::size_t p, std::size_t d, const std::int64_t* u_raw,
                     const std::int64_t* h_raw, int use_momentum, double momentum) {
    return guarded([&] {
        SomModel model;
        model.weights = make_matrix(w, p, d);
        model.prev_update = make_matrix(prev, p, d);
        IterationAccumulators acc(p, d);
        for (std::size_t i = 0; i < p * d; ++i)
            acc.u[i] = (static_cast<AccumInt>(u_raw[2 * i]) << 64) |
                       static_cast<AccumInt>(static_cast<std::uint64_t>(u_raw[2 * i + 1]));
        for (std::size_t j = 0; j < p; ++j)
            acc.h[j] = (static_cast<AccumInt>(h_raw[2 * j]) << 64) |
                       static_cast<AccumInt>(static_cast<std::uint64_t>(h_raw[2 * j + 1]));
        SomConfig c;
        c.topology = TopologySpec::graph(TopologyKind::mst, p);
        c.use_momentum = use_momentum != 0;
        c.momentum = momentum;
        apply_update(model, acc, c);
        std::memcpy(w, model.weights.values.data(), p * d * sizeof(float));
        std::memcpy(prev, model.prev_update.values.data(), p * d * sizeof(float));
    });
}

int ref_lattice_dist(int kind, std::size_t width, std::size_t height, double* out) {
    return guarded([&] {
        const auto dist = lattice_dist(lattice_coords(static_cast<TopologyKind>(kind), width, height));
        std::memcpy(out, dist.data(), dist.size() * sizeof(double));
    });
}

int ref_influence_from_dist(const double* dist, std::size_t n, double sigma, double* out) {
    return guarded([&] {
        const auto h = influence_matrix(std::vector<double>(dist, dist + n), sigma);
        std::memcpy(out, h.data(), n * sizeof(double));
    });
}

int ref_influence_from_hops(const std::uint16_t* hops, std::size_t n, double sigma, double* out) {
    return guarded([&] {
        const auto h = influence_matrix(std::vector<std::uint16_t>(hops, hops + n), sigma);
        std::memcpy(out, h.data(), n * sizeof(double));
    });
}

int ref_pairwise_sq_dists(const float* w, std::size_t p, std::size_t d, double* out) {
    return guarded([&] {
        const auto sq = pairwise_sq_dists(make_matrix(w, p, d), 256);
        std::memcpy(out, sq.data(), sq.size() * sizeof(double));
    });
}

// Edges out as (i, j) pairs; *n_edges in = capacity (pairs), out = count.
int ref_build_graph(int kind, const double* sq, std::size_t p, std::uint32_t* edges,
                    std::size_t* n_edges) {
    return guarded([&] {
        const std::vector<double> s(sq, sq + p * p);
        const auto e = kind == 2 ? build_mst(s, p) : build_rng_graph(s, p, 256);
        if (e.size() > *n_edges) throw std::invalid_argument("ref_build_graph: edge buffer too small");
        for (std::size_t i = 0; i < e.size(); ++i) {
            edges[2 * i] = e[i].first;
            edges[2 * i + 1] = e[i].second;
        }
        *n_edges = e.size();
    });
}

int ref_hop_distances(const std::uint32_t* edges, std::size_t n_edges, std::size_t p,
                      std::uint16_t* out) {
    return guarded([&] {
        std::vector<Edge> e(n_edges);
        for (std::size_t i = 0; i < n_edges; ++i) e[i] = {edges[2 * i], edges[2 * i + 1]};
        const auto h = hop_distances(e, p, 256);
        std::memcpy(out, h.data(), h.size() * sizeof(std::uint16_t));
    });
}

// Gaussian-mixture workload drawn with the reference's own Rng.
int ref_synth_gmm(float* out, std::size_t n, std::size_t d, std::uint64_t seed, std::size_t n_comp) {
    return guarded([&] {
        Rng rng(seed, SeedStream::synth);
        std::vector<double> mu(n_comp * d);
        for (auto& v : mu) v = rng.real(-4.0, 4.0);
        for (std::size_t i = 0; i < n; ++i) {
            const std::size_t m = rng.index(n_comp);
            for (std::size_t k = 0; k < d; ++k)
                out[i * d + k] = static_cast<float>(mu[m * d + k] + rng.gaussian());
        }
    });
}

int ref_synth_uniform(float* out, std::size_t n, std::size_t d, std::uint64_t seed) {
    return guarded([&] {
        const auto m = synth_uniform(n, d, seed);
        std::memcpy(out, m.values.data(), n * d * sizeof(float));
    });
}

int ref_synth_rings(float* out, std::size_t n, double noise, std::uint64_t seed) {
    return guarded([&] {
        const auto m = synth_rings(n, noise, seed);
        std::memcpy(out, m.values.data(), n * 2 * sizeof(float));
    });
}

int ref_rng_draws(std::uint64_t seed, std::uint64_t stream, std::size_t n, std::uint64_t* next_out,
                  double* gauss_out) {
    return guarded([&] {
        Rng a(seed, static_cast<SeedStream>(stream));
        for (std::size_t i = 0; i < n; ++i) next_out[i] = a.next();
        Rng b(seed, static_cast<SeedStream>(stream));
        for (std::size_t i = 0; i < n; ++i) gauss_out[i] = b.gaussian();
    });
}

// Sampler: `iters` successive selections of a Sampler, feeding back `dist`
// (constant per row, read from dist_by_row) for adaptive; out: iters*m indices.
int ref_sampler_run(int kind, int budget_fixed, std::uint64_t m0, double rho, std::size_t n,
                    std::uint64_t seed, double alpha, double beta, std::size_t iters,
                    const double* dist_by_row, std::uint32_t* out, std::size_t* m_out) {
    return guarded([&] {
        SamplingBudget b;
        b.mode = budget_fixed ? BudgetMode::fixed : BudgetMode::proportional;
        b.m0 = m0;
        b.rho = rho;
        Sampler s(static_cast<SamplingKind>(kind), b, n, seed, alpha, beta);
        std::size_t off = 0;
        for (std::size_t t = 0; t < iters; ++t) {
            const auto sel = s.select();
            std::vector<double> dist(sel.size());
            for (std::size_t i = 0; i < sel.size(); ++i) dist[i] = dist_by_row ? dist_by_row[sel[i]] : 0.0;
            s.observe(sel, dist);
            std::memcpy(out + off, sel.data(), sel.size() * sizeof(std::uint32_t));
            off += sel.size();
            m_out[t] = sel.size();
        }
    });
}

// SomConfig (trainer.hpp:58-99) from the flat config
static SomConfig to_config(const ref_config* rc) {
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

// run_study (tune.hpp:125-159), default SearchSpace, serial trials.
int ref_run_study(const ref_config* rc, std::size_t n_trials, const std::uint64_t* seeds,
                  std::size_t n_seeds, const float* train, std::size_t n, const float* holdout,
                  std::size_t nh, std::size_t d, double* qe_train, double* qe_holdout,
                  std::uint8_t* failed) {
    return guarded([&] {
        const auto tm = make_matrix(train, n, d);
        const auto hm = make_matrix(holdout, nh, d);
        StudySpec spec;
        spec.base_config = to_config(rc);
        spec.sampling = static_cast<SamplingKind>(rc->sampling);
        spec.budget.mode = rc->budget_fixed ? BudgetMode::fixed : BudgetMode::proportional;
        spec.budget.m0 = rc->m0;
        spec.budget.rho = rc->rho;
        spec.sampler_alpha = rc->alpha;
        spec.sampler_beta = rc->beta;
        spec.n_trials = n_trials;
        spec.seeds.assign(seeds, seeds + n_seeds);
        const auto recs = run_study(SearchSpace{}, spec, tm, hm);
        for (std::size_t i = 0; i < recs.size(); ++i) {
            qe_train[i] = recs[i].qe_train;
            qe_holdout[i] = recs[i].qe_holdout;
            failed[i] = recs[i].failed ? 1 : 0;
        }
    });
}

// Whole training run: train() for n_threads<=1, else train_parallel().
int ref_train(const ref_config* rc, const float* data, std::size_t n, std::size_t d,
              float* weights_out, double* qe_log, std::uint8_t* refresh_log) {
    return guarded([&] {
        SomConfig c = to_config(rc);
        SamplingBudget b;
        b.mode = rc->budget_fixed ? BudgetMode::fixed : BudgetMode::proportional;
        b.m0 = rc->m0;
        b.rho = rc->rho;
        Sampler sampler(static_cast<SamplingKind>(rc->sampling), b, n, c.seed, rc->alpha, rc->beta);
        const auto mat = make_matrix(data, n, d);
        TrainOptions opts;
        opts.log_qe = qe_log != nullptr;
        auto result = rc->n_threads <= 1
                          ? train(c, mat, sampler, opts)
                          : train_parallel(c, mat, sampler, static_cast<std::size_t>(rc->n_threads), opts);
        std::memcpy(weights_out, result.first.weights.values.data(),
                    result.first.weights.values.size() * sizeof(float));
        for (std::size_t t = 0; t < result.second.iterations.size(); ++t) {
            if (qe_log) qe_log[t] = *result.second.iterations[t].qe_train;
            if (refresh_log) refresh_log[t] = result.second.iterations[t].refreshed ? 1 : 0;
        }
    });
}

}  // extern "C"
