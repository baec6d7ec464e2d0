/*
 * tsom_oracle.c — CPU restatement of the toposom batch-SOM hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * engine: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
 * may load it.  The product path (paper_2604_26555_b200/) never links, calls
 * or falls back to it.
 *
 * Every function restates the reference algorithm and cites the reference
 * file:line it follows (paths relative to /root/reference/proj/include/toposom).
 * Parity of this restatement is pinned two ways (see tests/test_oracle.py):
 *   - the reference's own known-answer tests (test_trainer.cpp, test_parallel.cpp,
 *     test_metrics.cpp, test_rng.cpp) re-expressed as golden vectors;
 *   - bit-for-bit comparison against oracle/_ref/libtoposom_ref.so, which is
 *     the reference headers themselves compiled by oracle/Makefile.
 *
 * Arithmetic notes: compiled with -ffp-contract=off so FP64 sums are evaluated
 * exactly as the reference's Release build (x86-64 baseline ISA, no FMA).
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_INVALID 1
#define ORC_NUMERICAL 2
#define ORC_RANGE 3

typedef __int128 i128;

/* ------------------------------------------------------------------------ */
/* rng.hpp:12-91 — splitmix seed streams + mt19937_64 + hand-rolled draws    */
/* ------------------------------------------------------------------------ */

#define MT_NN 312
#define MT_MM 156
#define MT_MATRIX_A 0xB5026F5AA96619E9ULL
#define MT_UM 0xFFFFFFFF80000000ULL
#define MT_LM 0x7FFFFFFFULL

typedef struct {
    uint64_t mt[MT_NN];
    int mti;
    double cached;
    int has_cached;
} orc_rng;

/* rng.hpp:12-17 */
uint64_t orc_mix_seed(uint64_t seed, uint64_t stream) {
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (stream + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* std::mt19937_64 seeding (the standard's recurrence), rng.hpp:33 */
void orc_rng_init(orc_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_NN; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->mti = MT_NN;
    r->cached = 0.0;
    r->has_cached = 0;
}

/* rng.hpp:34-35 */
void orc_rng_init_stream(orc_rng* r, uint64_t seed, uint64_t stream) {
    orc_rng_init(r, orc_mix_seed(seed, stream));
}

uint64_t orc_rng_next(orc_rng* r) {
    uint64_t x;
    if (r->mti >= MT_NN) {
        int i;
        for (i = 0; i < MT_NN - MT_MM; ++i) {
            x = (r->mt[i] & MT_UM) | (r->mt[i + 1] & MT_LM);
            r->mt[i] = r->mt[i + MT_MM] ^ (x >> 1) ^ ((x & 1ULL) ? MT_MATRIX_A : 0ULL);
        }
        for (; i < MT_NN - 1; ++i) {
            x = (r->mt[i] & MT_UM) | (r->mt[i + 1] & MT_LM);
            r->mt[i] = r->mt[i + (MT_MM - MT_NN)] ^ (x >> 1) ^ ((x & 1ULL) ? MT_MATRIX_A : 0ULL);
        }
        x = (r->mt[MT_NN - 1] & MT_UM) | (r->mt[0] & MT_LM);
        r->mt[MT_NN - 1] = r->mt[MT_MM - 1] ^ (x >> 1) ^ ((x & 1ULL) ? MT_MATRIX_A : 0ULL);
        r->mti = 0;
    }
    x = r->mt[r->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

/* rng.hpp:40-49 — unbiased bounded draw by rejection */
uint64_t orc_rng_index(orc_rng* r, uint64_t n) {
    const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t x;
    do {
        x = orc_rng_next(r);
    } while (x >= limit);
    return x % n;
}

/* rng.hpp:52 */
double orc_rng_real01(orc_rng* r) { return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:54 */
double orc_rng_real(orc_rng* r, double lo, double hi) { return lo + (hi - lo) * orc_rng_real01(r); }

/* rng.hpp:62-76 — Box-Muller with cached pair */
double orc_rng_gaussian(orc_rng* r) {
    if (r->has_cached) {
        r->has_cached = 0;
        return r->cached;
    }
    const double u1 = 1.0 - orc_rng_real01(r);
    const double u2 = orc_rng_real01(r);
    const double rr = sqrt(-2.0 * log(u1));
    const double theta = 2.0 * 3.14159265358979323846 * u2;
    r->cached = rr * sin(theta);
    r->has_cached = 1;
    return rr * cos(theta);
}

size_t orc_rng_sizeof(void) { return sizeof(orc_rng); }

/* ------------------------------------------------------------------------ */
/* Synthetic data                                                            */
/* ------------------------------------------------------------------------ */

enum { STREAM_SPLIT = 1, STREAM_INIT = 2, STREAM_SAMPLER = 3, STREAM_SYNTH = 4 };

/* dataset.hpp:428-435 */
void orc_synth_uniform(float* out, size_t n, size_t d, uint64_t seed) {
    orc_rng r;
    orc_rng_init_stream(&r, seed, STREAM_SYNTH);
    for (size_t i = 0; i < n * d; ++i) out[i] = (float)orc_rng_real01(&r);
}

/* dataset.hpp:439-453 */
void orc_synth_rings(float* out, size_t n, double noise, uint64_t seed) {
    orc_rng r;
    orc_rng_init_stream(&r, seed, STREAM_SYNTH);
    const size_t n_outer = n / 2 + (n % 2);
    for (size_t i = 0; i < n; ++i) {
        const double radius = i < n_outer ? 1.0 : 0.5;
        const double theta = orc_rng_real01(&r) * 2.0 * 3.14159265358979323846;
        const double x = radius * cos(theta) + noise * orc_rng_gaussian(&r);
        const double y = radius * sin(theta) + noise * orc_rng_gaussian(&r);
        out[2 * i] = (float)x;
        out[2 * i + 1] = (float)y;
    }
}

/*
 * Gaussian-mixture workload of SURVEY.md §8(d): centres
 * mu_m ~ U[-4,4]^d drawn first from Rng(seed, synth), then per row
 * m = index(n_comp) and x = mu_m + N(0, I) via Rng::gaussian, stored f32.
 * Written with the reference's own Rng so both sides see identical inputs.
 */
void orc_synth_gmm(float* out, size_t n, size_t d, uint64_t seed, size_t n_comp,
                   double* centres_out) {
    orc_rng r;
    orc_rng_init_stream(&r, seed, STREAM_SYNTH);
    double* mu = (double*)malloc(sizeof(double) * n_comp * d);
    for (size_t m = 0; m < n_comp; ++m)
        for (size_t k = 0; k < d; ++k) mu[m * d + k] = orc_rng_real(&r, -4.0, 4.0);
    for (size_t i = 0; i < n; ++i) {
        const size_t m = (size_t)orc_rng_index(&r, n_comp);
        for (size_t k = 0; k < d; ++k) out[i * d + k] = (float)(mu[m * d + k] + orc_rng_gaussian(&r));
    }
    if (centres_out) memcpy(centres_out, mu, sizeof(double) * n_comp * d);
    free(mu);
}

/* ------------------------------------------------------------------------ */
/* accum.hpp:27-81 — Q23.40 fixed-point accumulators                          */
/* ------------------------------------------------------------------------ */

#define ACC_SCALE 1099511627776.0 /* 2^40, accum.hpp:28 */
#define ACC_MAX 4194304.0         /* 2^22, accum.hpp:29 */

/* accum.hpp:34-38; returns 0 on success, ORC_NUMERICAL on guard violation */
static inline int quantize_term(double term, int64_t* q) {
    if (!(fabs(term) < ACC_MAX)) return ORC_NUMERICAL;
    *q = llrint(term * ACC_SCALE);
    return ORC_OK;
}

int64_t orc_quantize_term(double term, int* status) {
    int64_t q = 0;
    *status = quantize_term(term, &q);
    return q;
}

/* accum.hpp:40-42 */
double orc_dequantize_parts(int64_t hi, uint64_t lo) {
    const i128 v = (i128)(((unsigned __int128)(uint64_t)hi << 64) | lo);
    return (double)v / ACC_SCALE;
}

/* ------------------------------------------------------------------------ */
/* trainer.hpp:282-308 — find_bmus                                           */
/* ------------------------------------------------------------------------ */

static inline void bmu_one(const float* x, const float* w, size_t p, size_t d, uint32_t* bmu,
                           double* best_out) {
    double best = INFINITY;
    uint32_t best_j = 0;
    for (size_t j = 0; j < p; ++j) {
        const float* wj = w + j * d;
        double acc = 0.0;
        for (size_t k = 0; k < d; ++k) {
            const double diff = (double)x[k] - (double)wj[k];
            acc += diff * diff;
        }
        if (acc < best) {
            best = acc;
            best_j = (uint32_t)j;
        }
    }
    *bmu = best_j;
    *best_out = best;
}

void orc_find_bmus(const float* x, size_t n, const float* w, size_t p, size_t d, uint32_t* bmus,
                   double* dists) {
    for (size_t i = 0; i < n; ++i) {
        double best;
        bmu_one(x + i * d, w, p, d, &bmus[i], &best);
        if (dists) dists[i] = sqrt(best > 0.0 ? best : 0.0);
    }
}

/* trainer.hpp:377-398 — mean Euclidean BMU distance (QE) */
double orc_mean_bmu_distance(const float* x, size_t n, const float* w, size_t p, size_t d) {
    double total = 0.0;
    for (size_t i = 0; i < n; ++i) {
        uint32_t b;
        double best;
        bmu_one(x + i * d, w, p, d, &b, &best);
        total += sqrt(best > 0.0 ? best : 0.0);
    }
    return total / (double)n;
}

/* ------------------------------------------------------------------------ */
/* trainer.hpp:318-336 — accumulate (every sample x every node, fixed point) */
/* ------------------------------------------------------------------------ */

static int accumulate_rows(const float* chunk, size_t rows, const uint32_t* bmus, const float* w,
                           size_t p, size_t d, const double* infl, double eta, i128* u, i128* h) {
    for (size_t i = 0; i < rows; ++i) {
        const float* x = chunk + i * d;
        const double* h_row = infl + (size_t)bmus[i] * p;
        for (size_t j = 0; j < p; ++j) {
            const double hv = h_row[j];
            const float* wj = w + j * d;
            int64_t q;
            if (quantize_term(hv, &q)) return ORC_NUMERICAL;
            h[j] += q;
            const double eh = eta * hv;
            for (size_t k = 0; k < d; ++k) {
                if (quantize_term(eh * ((double)x[k] - (double)wj[k]), &q)) return ORC_NUMERICAL;
                u[j * d + k] += q;
            }
        }
    }
    return ORC_OK;
}

/*
 * trainer.hpp:414-435 accumulate_selection, fanned out like parallel.hpp:99-140
 * (contiguous slices, exact int128 merge ⇒ result independent of n_threads).
 */
typedef struct {
    const float* data;
    size_t n_rows;
    const uint32_t* sel;
    size_t lo, hi;
    const float* w;
    size_t p, d;
    const double* infl;
    double eta;
    size_t n_chunks;
    i128* u;
    i128* h;
    double* dist; /* selection-order output, may be NULL */
    int status;
} acc_job;

static void* acc_worker(void* arg) {
    acc_job* jb = (acc_job*)arg;
    const size_t n_sel = jb->hi - jb->lo;
    const size_t nc = jb->n_chunks ? jb->n_chunks : 1;
    size_t chunk_rows = (n_sel + nc - 1) / nc;
    if (chunk_rows < 1) chunk_rows = 1;
    float* chunk = (float*)malloc(sizeof(float) * chunk_rows * jb->d + 1);
    uint32_t* bmus = (uint32_t*)malloc(sizeof(uint32_t) * chunk_rows + 1);
    jb->status = ORC_OK;
    for (size_t c0 = 0; c0 < n_sel && jb->status == ORC_OK; c0 += chunk_rows) {
        const size_t c1 = c0 + chunk_rows < n_sel ? c0 + chunk_rows : n_sel;
        /* dataset.hpp:393-398 fetch_rows gather */
        for (size_t i = c0; i < c1; ++i) {
            const uint32_t row = jb->sel[jb->lo + i];
            if (row >= jb->n_rows) {
                jb->status = ORC_RANGE;
                break;
            }
            memcpy(chunk + (i - c0) * jb->d, jb->data + (size_t)row * jb->d, sizeof(float) * jb->d);
        }
        if (jb->status) break;
        for (size_t i = c0; i < c1; ++i) {
            double best;
            bmu_one(chunk + (i - c0) * jb->d, jb->w, jb->p, jb->d, &bmus[i - c0], &best);
            if (jb->dist) jb->dist[jb->lo + i] = sqrt(best > 0.0 ? best : 0.0);
        }
        jb->status = accumulate_rows(chunk, c1 - c0, bmus, jb->w, jb->p, jb->d, jb->infl, jb->eta,
                                     jb->u, jb->h);
    }
    free(chunk);
    free(bmus);
    return NULL;
}

/*
 * One iteration's accumulation over a selection.  Outputs both the exact
 * int128 accumulators (as hi/lo int64 pairs, may be NULL) and their
 * dequantised doubles (IterationAccumulators::u_value/h_value, accum.hpp:64-69).
 */
int orc_accumulate_selection(const float* data, size_t n_rows, const uint32_t* sel, size_t n_sel,
                             const float* w, size_t p, size_t d, const double* infl, double eta,
                             size_t n_chunks, int n_threads, double* u_out, double* h_out,
                             int64_t* u_raw, int64_t* h_raw, double* dist_out) {
    if (n_threads < 1) n_threads = 1;
    acc_job* jobs = (acc_job*)calloc((size_t)n_threads, sizeof(acc_job));
    pthread_t* th = (pthread_t*)calloc((size_t)n_threads, sizeof(pthread_t));
    const size_t base = n_sel / (size_t)n_threads, extra = n_sel % (size_t)n_threads;
    size_t begin = 0;
    for (int g = 0; g < n_threads; ++g) { /* parallel.hpp:28-41 assign_shards */
        const size_t cnt = base + ((size_t)g < extra ? 1 : 0);
        acc_job* jb = &jobs[g];
        jb->data = data;
        jb->n_rows = n_rows;
        jb->sel = sel;
        jb->lo = begin;
        jb->hi = begin + cnt;
        jb->w = w;
        jb->p = p;
        jb->d = d;
        jb->infl = infl;
        jb->eta = eta;
        jb->n_chunks = n_chunks;
        jb->u = (i128*)calloc(p * d, sizeof(i128));
        jb->h = (i128*)calloc(p, sizeof(i128));
        jb->dist = dist_out;
        begin += cnt;
        if (n_threads > 1)
            pthread_create(&th[g], NULL, acc_worker, jb);
        else
            acc_worker(jb);
    }
    int status = ORC_OK;
    i128* u = (i128*)calloc(p * d, sizeof(i128));
    i128* h = (i128*)calloc(p, sizeof(i128));
    for (int g = 0; g < n_threads; ++g) { /* parallel.hpp:90-95 ordered reduce */
        if (n_threads > 1) pthread_join(th[g], NULL);
        if (jobs[g].status && !status) status = jobs[g].status;
        for (size_t i = 0; i < p * d; ++i) u[i] += jobs[g].u[i];
        for (size_t i = 0; i < p; ++i) h[i] += jobs[g].h[i];
        free(jobs[g].u);
        free(jobs[g].h);
    }
    for (size_t i = 0; i < p * d; ++i) {
        if (u_out) u_out[i] = (double)u[i] / ACC_SCALE;
        if (u_raw) {
            u_raw[2 * i] = (int64_t)(u[i] >> 64);
            u_raw[2 * i + 1] = (int64_t)(uint64_t)u[i];
        }
    }
    for (size_t i = 0; i < p; ++i) {
        if (h_out) h_out[i] = (double)h[i] / ACC_SCALE;
        if (h_raw) {
            h_raw[2 * i] = (int64_t)(h[i] >> 64);
            h_raw[2 * i + 1] = (int64_t)(uint64_t)h[i];
        }
    }
    free(u);
    free(h);
    free(jobs);
    free(th);
    return status;
}

/* ------------------------------------------------------------------------ */
/* trainer.hpp:341-369 — apply_update                                        */
/* ------------------------------------------------------------------------ */

int orc_apply_update(float* w, float* prev, size_t p, size_t d, const double* u, const double* h,
                     int use_momentum, double momentum, int64_t* bad_node) {
    const double kHFloor = 1e-12;
    for (size_t j = 0; j < p; ++j) {
        const double hv = h[j];
        float* wj = w + j * d;
        float* pj = prev + j * d;
        if (hv < kHFloor) {
            if (use_momentum)
                for (size_t k = 0; k < d; ++k) pj[k] = 0.0f;
            continue;
        }
        for (size_t k = 0; k < d; ++k) {
            double delta = u[j * d + k] / hv;
            if (use_momentum) delta += momentum * (double)pj[k];
            if (!isfinite(delta)) {
                if (bad_node) *bad_node = (int64_t)j;
                return ORC_NUMERICAL;
            }
            const double updated = (double)wj[k] + delta;
            if (!isfinite(updated)) {
                if (bad_node) *bad_node = (int64_t)j;
                return ORC_NUMERICAL;
            }
            wj[k] = (float)updated;
            if (use_momentum) pj[k] = (float)delta;
        }
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* trainer.hpp:132-139 — schedules                                           */
/* ------------------------------------------------------------------------ */

double orc_schedule_value(double v0, int exponential, size_t t, size_t total, double floor_v) {
    const double frac = (double)t / (double)total;
    const double v = exponential ? v0 * exp(-3.0 * frac) : v0 * (1.0 - frac);
    return v > floor_v ? v : floor_v;
}

/* ------------------------------------------------------------------------ */
/* topology.hpp — geometry, graphs, hops, influence                           */
/* ------------------------------------------------------------------------ */

enum { TOPO_RECT = 0, TOPO_HEX = 1, TOPO_MST = 2, TOPO_RNG = 3 };

/* topology.hpp:81-108 */
void orc_pairwise_sq_dists(const float* w, size_t p, size_t d, double* out) {
    double* norms = (double*)malloc(sizeof(double) * p);
    for (size_t i = 0; i < p; ++i) {
        double s = 0.0;
        for (size_t k = 0; k < d; ++k) s += (double)w[i * d + k] * (double)w[i * d + k];
        norms[i] = s;
    }
    for (size_t i = 0; i < p; ++i)
        for (size_t j = 0; j < p; ++j) {
            if (j == i) {
                out[i * p + j] = 0.0;
                continue;
            }
            double dot = 0.0;
            for (size_t k = 0; k < d; ++k) dot += (double)w[i * d + k] * (double)w[j * d + k];
            const double v = norms[i] + norms[j] - 2.0 * dot;
            out[i * p + j] = v > 0.0 ? v : 0.0;
        }
    free(norms);
}

/* topology.hpp:114-149 */
void orc_lattice_dist(int kind, size_t width, size_t height, double* out) {
    const size_t p = width * height;
    double* c = (double*)malloc(sizeof(double) * 2 * p);
    const double kHexRow = 0.86602540378443864676;
    size_t q = 0;
    for (size_t r = 0; r < height; ++r)
        for (size_t col = 0; col < width; ++col, ++q) {
            if (kind == TOPO_RECT) {
                c[2 * q] = (double)r;
                c[2 * q + 1] = (double)col;
            } else {
                c[2 * q] = (double)col + (r % 2 == 1 ? 0.5 : 0.0);
                c[2 * q + 1] = (double)r * kHexRow;
            }
        }
    for (size_t i = 0; i < p; ++i) out[i * p + i] = 0.0;
    for (size_t i = 0; i < p; ++i)
        for (size_t j = i + 1; j < p; ++j) {
            const double dx = c[2 * i] - c[2 * j], dy = c[2 * i + 1] - c[2 * j + 1];
            const double dist = sqrt(dx * dx + dy * dy);
            out[i * p + j] = dist;
            out[j * p + i] = dist;
        }
    free(c);
}

typedef struct {
    double w;
    uint32_t i, j;
} wedge;

static int wedge_cmp(const void* a, const void* b) {
    const wedge* x = (const wedge*)a;
    const wedge* y = (const wedge*)b;
    if (x->w != y->w) return x->w < y->w ? -1 : 1;
    if (x->i != y->i) return x->i < y->i ? -1 : 1;
    return x->j < y->j ? -1 : (x->j > y->j);
}

static uint32_t uf_find(uint32_t* parent, uint32_t x) {
    while (parent[x] != x) {
        parent[x] = parent[parent[x]];
        x = parent[x];
    }
    return x;
}

static int edge_cmp(const void* a, const void* b) {
    const uint32_t* x = (const uint32_t*)a;
    const uint32_t* y = (const uint32_t*)b;
    if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
    return x[1] < y[1] ? -1 : (x[1] > y[1]);
}

/* topology.hpp:192-220 Kruskal; edges_out has room for 2*(p-1); returns count */
size_t orc_build_mst(const double* sq, size_t p, uint32_t* edges_out) {
    if (p <= 1) return 0;
    const size_t m = p * (p - 1) / 2;
    wedge* all = (wedge*)malloc(sizeof(wedge) * m);
    size_t q = 0;
    for (uint32_t i = 0; i < p; ++i)
        for (uint32_t j = i + 1; j < p; ++j) all[q++] = (wedge){sq[(size_t)i * p + j], i, j};
    qsort(all, m, sizeof(wedge), wedge_cmp);
    uint32_t* parent = (uint32_t*)malloc(sizeof(uint32_t) * p);
    uint8_t* rank = (uint8_t*)calloc(p, 1);
    for (uint32_t i = 0; i < p; ++i) parent[i] = i;
    size_t ne = 0;
    for (size_t e = 0; e < m && ne < p - 1; ++e) {
        uint32_t a = uf_find(parent, all[e].i), b = uf_find(parent, all[e].j);
        if (a == b) continue;
        if (rank[a] < rank[b]) {
            uint32_t t = a;
            a = b;
            b = t;
        }
        parent[b] = a;
        if (rank[a] == rank[b]) ++rank[a];
        edges_out[2 * ne] = all[e].i;
        edges_out[2 * ne + 1] = all[e].j;
        ++ne;
    }
    qsort(edges_out, ne, 2 * sizeof(uint32_t), edge_cmp);
    free(all);
    free(parent);
    free(rank);
    return ne;
}

/* topology.hpp:229-258 RNG (strict blocker); edges_out room p*(p-1); returns count */
size_t orc_build_rng_graph(const double* sq, size_t p, uint32_t* edges_out) {
    size_t ne = 0;
    for (uint32_t a = 0; a < p; ++a)
        for (uint32_t b = a + 1; b < p; ++b) {
            const double dab = sq[(size_t)a * p + b];
            int blocked = 0;
            for (size_t r = 0; r < p && !blocked; ++r) {
                if (r == a || r == b) continue;
                const double dar = sq[(size_t)a * p + r], dbr = sq[(size_t)b * p + r];
                if ((dar > dbr ? dar : dbr) < dab) blocked = 1;
            }
            if (!blocked) {
                edges_out[2 * ne] = a;
                edges_out[2 * ne + 1] = b;
                ++ne;
            }
        }
    return ne;
}

/* topology.hpp:292-325 all-pairs hops (BFS gives identical shortest hop counts);
 * returns ORC_OK, or ORC_NUMERICAL when disconnected ("graph is disconnected"). */
int orc_hop_distances(const uint32_t* edges, size_t ne, size_t p, uint16_t* out) {
    size_t* deg = (size_t*)calloc(p + 1, sizeof(size_t));
    for (size_t e = 0; e < ne; ++e) {
        if (edges[2 * e] >= p || edges[2 * e + 1] >= p) {
            free(deg);
            return ORC_RANGE;
        }
        deg[edges[2 * e] + 1]++;
        deg[edges[2 * e + 1] + 1]++;
    }
    for (size_t i = 0; i < p; ++i) deg[i + 1] += deg[i];
    uint32_t* adj = (uint32_t*)malloc(sizeof(uint32_t) * (2 * ne + 1));
    size_t* fill = (size_t*)malloc(sizeof(size_t) * (p + 1));
    memcpy(fill, deg, sizeof(size_t) * (p + 1));
    for (size_t e = 0; e < ne; ++e) {
        adj[fill[edges[2 * e]]++] = edges[2 * e + 1];
        adj[fill[edges[2 * e + 1]]++] = edges[2 * e];
    }
    uint32_t* queue = (uint32_t*)malloc(sizeof(uint32_t) * p);
    int status = ORC_OK;
    for (size_t s = 0; s < p; ++s) {
        uint16_t* row = out + s * p;
        for (size_t i = 0; i < p; ++i) row[i] = 0xFFFF;
        row[s] = 0;
        size_t qh = 0, qt = 0;
        queue[qt++] = (uint32_t)s;
        while (qh < qt) {
            const uint32_t v = queue[qh++];
            for (size_t a = deg[v]; a < deg[v + 1]; ++a) {
                const uint32_t nb = adj[a];
                if (row[nb] == 0xFFFF) {
                    row[nb] = (uint16_t)(row[v] + 1);
                    queue[qt++] = nb;
                }
            }
        }
        if (qt != p) status = ORC_NUMERICAL;
    }
    free(deg);
    free(adj);
    free(fill);
    free(queue);
    return status;
}

/* topology.hpp:339-364 Gaussian influence with exp cut at 57.6 */
void orc_influence_from_dist(const double* dist, size_t n, double sigma, double* out) {
    const double inv = 1.0 / (2.0 * sigma * sigma);
    for (size_t i = 0; i < n; ++i) {
        const double z = (dist[i] * dist[i]) * inv;
        out[i] = z > 57.6 ? 0.0 : exp(-z);
    }
}

void orc_influence_from_hops(const uint16_t* hops, size_t n, double sigma, double* out) {
    const double inv = 1.0 / (2.0 * sigma * sigma);
    for (size_t i = 0; i < n; ++i) {
        const double dd = (double)hops[i];
        const double z = (dd * dd) * inv;
        out[i] = z > 57.6 ? 0.0 : exp(-z);
    }
}

/* ------------------------------------------------------------------------ */
/* sampling.hpp — selectors                                                  */
/* ------------------------------------------------------------------------ */

static int u32_cmp(const void* a, const void* b) {
    const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : (x > y);
}

/* open-addressing set for Floyd's algorithm (sampling.hpp:56-73 uses a hash set;
 * the selected SET is implementation-independent) */
typedef struct {
    uint32_t* keys;
    size_t cap;
} u32set;

static int set_insert(u32set* s, uint32_t k) {
    size_t h = ((uint64_t)k * 0x9E3779B97F4A7C15ULL) & (s->cap - 1);
    while (s->keys[h] != 0xFFFFFFFFu) {
        if (s->keys[h] == k) return 0;
        h = (h + 1) & (s->cap - 1);
    }
    s->keys[h] = k;
    return 1;
}

/* sampling.hpp:56-73; out has room for m (m < n) */
void orc_select_random(size_t n, size_t m, orc_rng* r, uint32_t* out) {
    if (m >= n) {
        for (size_t i = 0; i < n; ++i) out[i] = (uint32_t)i;
        return;
    }
    u32set s;
    s.cap = 1;
    while (s.cap < 4 * m + 4) s.cap <<= 1;
    s.keys = (uint32_t*)malloc(sizeof(uint32_t) * s.cap);
    memset(s.keys, 0xFF, sizeof(uint32_t) * s.cap);
    size_t q = 0;
    for (size_t j = n - m; j < n; ++j) {
        const uint32_t t = (uint32_t)orc_rng_index(r, j + 1);
        const uint32_t pick = set_insert(&s, t) ? t : (uint32_t)j;
        if (pick != t) set_insert(&s, pick);
        out[q++] = pick;
    }
    qsort(out, m, sizeof(uint32_t), u32_cmp);
    free(s.keys);
}

typedef struct {
    int seen;
    double key;
    uint32_t index;
} ranked;

static int ranked_cmp(const void* a, const void* b) {
    const ranked* x = (const ranked*)a;
    const ranked* y = (const ranked*)b;
    if (x->seen != y->seen) return x->seen ? 1 : -1; /* unseen first */
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return 0;
}

#define UNSEEN 1e30

/* sampling.hpp:101-139 exponential-key weighted selection */
void orc_select_adaptive(const double* last_error, const uint32_t* age, size_t n, double alpha,
                         double beta, size_t m, orc_rng* r, uint32_t* out) {
    if (m > n) m = n;
    double max_err = 0.0, max_age = 0.0;
    for (size_t i = 0; i < n; ++i) {
        if (last_error[i] > max_err) max_err = last_error[i];
        if ((double)age[i] > max_age) max_age = (double)age[i];
    }
    if (max_err < 1e-12) max_err = 1e-12;
    if (max_age < 1e-12) max_age = 1e-12;
    ranked* keys = (ranked*)malloc(sizeof(ranked) * n);
    for (size_t i = 0; i < n; ++i) {
        const double w = pow(last_error[i] / max_err, alpha) + pow((double)age[i] / max_age, beta);
        const double u = 1.0 - orc_rng_real01(r);
        const double key = w > 0.0 ? -log(u) / w : INFINITY;
        keys[i].seen = last_error[i] != UNSEEN;
        keys[i].key = key;
        keys[i].index = (uint32_t)i;
    }
    qsort(keys, n, sizeof(ranked), ranked_cmp);
    for (size_t i = 0; i < m; ++i) out[i] = keys[i].index;
    qsort(out, m, sizeof(uint32_t), u32_cmp);
    free(keys);
}

/* sampling.hpp:143-157 */
void orc_update_adaptive(double* last_error, uint32_t* age, size_t n, const uint32_t* sel,
                         size_t n_sel, const double* dist) {
    for (size_t i = 0; i < n; ++i) ++age[i];
    for (size_t i = 0; i < n_sel; ++i) {
        last_error[sel[i]] = dist[i];
        age[sel[i]] = 0;
    }
}

/* ------------------------------------------------------------------------ */
/* trainer.hpp:187-211 init_weights (sample_draw, uniform_box)               */
/* ------------------------------------------------------------------------ */

void orc_init_sample_draw(const float* data, size_t n, size_t d, size_t p, uint64_t seed,
                          float* w_out) {
    orc_rng r;
    orc_rng_init_stream(&r, seed, STREAM_INIT);
    uint32_t* picks = (uint32_t*)malloc(sizeof(uint32_t) * p);
    if (p <= n) {
        size_t q = 0;
        for (size_t j = n - p; j < n; ++j) {
            const uint32_t t = (uint32_t)orc_rng_index(&r, j + 1);
            int found = 0;
            for (size_t a = 0; a < q; ++a)
                if (picks[a] == t) {
                    found = 1;
                    break;
                }
            picks[q++] = found ? (uint32_t)j : t;
        }
    } else {
        for (size_t i = 0; i < p; ++i) picks[i] = (uint32_t)orc_rng_index(&r, n);
    }
    for (size_t i = 0; i < p; ++i) memcpy(w_out + i * d, data + (size_t)picks[i] * d, sizeof(float) * d);
    free(picks);
}

void orc_init_uniform_box(const float* data, size_t n, size_t d, size_t p, uint64_t seed,
                          float* w_out) {
    orc_rng r;
    orc_rng_init_stream(&r, seed, STREAM_INIT);
    double* lo = (double*)malloc(sizeof(double) * d);
    double* hi = (double*)malloc(sizeof(double) * d);
    for (size_t k = 0; k < d; ++k) {
        lo[k] = INFINITY;
        hi[k] = -INFINITY;
    }
    for (size_t i = 0; i < n; ++i)
        for (size_t k = 0; k < d; ++k) {
            const double v = data[i * d + k];
            if (v < lo[k]) lo[k] = v;
            if (v > hi[k]) hi[k] = v;
        }
    for (size_t j = 0; j < p; ++j)
        for (size_t k = 0; k < d; ++k)
            w_out[j * d + k] = (float)(lo[k] + orc_rng_real01(&r) * (hi[k] - lo[k]));
    free(lo);
    free(hi);
}

/* ------------------------------------------------------------------------ */
/* trainer.hpp:466-523 train_with_executor (serial executor)                 */
/* ------------------------------------------------------------------------ */

typedef struct {
    int topology;         /* TOPO_* */
    uint64_t grid_w, grid_h, nodes;
    uint64_t n_iters;
    double eta0;
    int lr_exponential;
    double sigma0; /* 0 = auto */
    int radius_exponential;
    double sigma_min;
    int init_method; /* 0 sample_draw, 1 uniform_box */
    int use_momentum;
    double momentum;
    uint64_t refresh_warmup; /* 0 = auto (n_iters/10) */
    double refresh_growth;
    uint64_t refresh_max_interval;
    uint64_t n_chunks;
    uint64_t seed;
    int sampling;         /* 0 full, 1 random, 2 adaptive */
    int budget_fixed;     /* 1 = fixed m0 */
    uint64_t m0;
    double rho;
    double alpha, beta;
    int n_threads;
} orc_config;

size_t orc_config_sizeof(void) { return sizeof(orc_config); }

/* trainer.hpp:75-80 */
static double resolved_sigma0(const orc_config* c) {
    if (c->sigma0 > 0.0) return c->sigma0;
    if (c->topology == TOPO_RECT || c->topology == TOPO_HEX) {
        const double side = (double)(c->grid_w > c->grid_h ? c->grid_w : c->grid_h) / 2.0;
        return side > 1.0 ? side : 1.0;
    }
    return 3.0;
}

/*
 * Full training run.  weights_out: P x d; qe_log (optional): per-iteration QE
 * after the update; returns status.  refresh_log (optional): 1 per refreshed
 * iteration.
 */
int orc_train(const orc_config* c, const float* data, size_t n, size_t d, float* weights_out,
              double* qe_log, uint8_t* refresh_log) {
    const size_t p = c->nodes;
    const int lattice = c->topology == TOPO_RECT || c->topology == TOPO_HEX;
    float* w = weights_out;
    if (c->init_method == 1)
        orc_init_uniform_box(data, n, d, p, c->seed, w);
    else
        orc_init_sample_draw(data, n, d, p, c->seed, w);
    float* prev = (float*)calloc(p * d, sizeof(float));
    double* dist_mat = NULL;
    uint16_t* hops = NULL;
    if (lattice) {
        dist_mat = (double*)malloc(sizeof(double) * p * p);
        orc_lattice_dist(c->topology, c->grid_w, c->grid_h, dist_mat);
    } else {
        hops = (uint16_t*)malloc(sizeof(uint16_t) * p * p);
    }
    const uint64_t warmup = c->refresh_warmup ? c->refresh_warmup : c->n_iters / 10;
    int64_t last_refresh = -1;
    uint64_t post_warmup = 0;
    const double sigma0 = resolved_sigma0(c);

    orc_rng srng;
    orc_rng_init_stream(&srng, c->seed, STREAM_SAMPLER);
    size_t m = n;
    if (c->sampling != 0) {
        if (c->budget_fixed)
            m = c->m0;
        else {
            m = (size_t)floor((double)n * c->rho);
            if (m < 1) m = 1;
        }
    }
    double* last_err = NULL;
    uint32_t* age = NULL;
    if (c->sampling == 2) {
        last_err = (double*)malloc(sizeof(double) * n);
        age = (uint32_t*)calloc(n, sizeof(uint32_t));
        for (size_t i = 0; i < n; ++i) last_err[i] = UNSEEN;
    }
    uint32_t* sel = (uint32_t*)malloc(sizeof(uint32_t) * (n > m ? n : m));
    double* dist = (double*)malloc(sizeof(double) * (n > m ? n : m));
    double* infl = (double*)malloc(sizeof(double) * p * p);
    double* u = (double*)malloc(sizeof(double) * p * d);
    double* h = (double*)malloc(sizeof(double) * p);
    double* sq = lattice ? NULL : (double*)malloc(sizeof(double) * p * p);
    uint32_t* edges = lattice ? NULL : (uint32_t*)malloc(sizeof(uint32_t) * p * (p > 1 ? p - 1 : 1) + 8);
    int status = ORC_OK;
    for (uint64_t t = 0; t < c->n_iters && status == ORC_OK; ++t) {
        /* sampling.hpp:197-204 */
        size_t n_sel;
        if (c->sampling == 0) {
            for (size_t i = 0; i < n; ++i) sel[i] = (uint32_t)i;
            n_sel = n;
        } else if (c->sampling == 1) {
            orc_select_random(n, m, &srng, sel);
            n_sel = m < n ? m : n;
        } else {
            orc_select_adaptive(last_err, age, n, c->alpha, c->beta, m, &srng, sel);
            n_sel = m < n ? m : n;
        }
        /* topology.hpp:423-451 */
        int refreshed = 0;
        if (!lattice) {
            int do_refresh;
            if (t < warmup)
                do_refresh = 1;
            else {
                const double raw = ceil(pow(c->refresh_growth, (double)post_warmup));
                const uint64_t interval = raw >= (double)c->refresh_max_interval
                                              ? c->refresh_max_interval
                                              : (uint64_t)raw;
                do_refresh = (int64_t)t - last_refresh >= (int64_t)interval;
            }
            if (do_refresh) {
                orc_pairwise_sq_dists(w, p, d, sq);
                size_t ne = c->topology == TOPO_MST ? orc_build_mst(sq, p, edges)
                                                    : orc_build_rng_graph(sq, p, edges);
                if (orc_hop_distances(edges, ne, p, hops)) {
                    status = ORC_NUMERICAL;
                    break;
                }
                last_refresh = (int64_t)t;
                if (t >= warmup) ++post_warmup;
                refreshed = 1;
            }
        }
        if (refresh_log) refresh_log[t] = (uint8_t)refreshed;
        const double eta = orc_schedule_value(c->eta0, c->lr_exponential, t, c->n_iters, 1e-4);
        const double sigma =
            orc_schedule_value(sigma0, c->radius_exponential, t, c->n_iters, c->sigma_min);
        if (lattice)
            orc_influence_from_dist(dist_mat, p * p, sigma, infl);
        else
            orc_influence_from_hops(hops, p * p, sigma, infl);
        status = orc_accumulate_selection(data, n, sel, n_sel, w, p, d, infl, eta, c->n_chunks,
                                          c->n_threads, u, h, NULL, NULL, dist);
        if (status) break;
        status = orc_apply_update(w, prev, p, d, u, h, c->use_momentum, c->momentum, NULL);
        if (status) break;
        if (c->sampling == 2) orc_update_adaptive(last_err, age, n, sel, n_sel, dist);
        if (qe_log) qe_log[t] = orc_mean_bmu_distance(data, n, w, p, d);
    }
    free(prev);
    free(dist_mat);
    free(hops);
    free(last_err);
    free(age);
    free(sel);
    free(dist);
    free(infl);
    free(u);
    free(h);
    free(sq);
    free(edges);
    return status;
}
