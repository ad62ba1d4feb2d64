/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference's online CF
 * completion + selection path, used as the CPU oracle by tests/ and as the
 * "port" CPU baseline.  Never linked into the product.
 *
 * Arithmetic follows either reference kernel lane op for op (ocgo_set_lane):
 * the scalar lane (kernels_scalar.cpp, baseline x86-64, no FMA) or the AVX2
 * lane as g++ compiles kernels_avx2.cpp; this file is compiled with
 * -ffp-contract=off so only the explicit fma() calls fuse.  exp() is the host
 * libm exp, exactly what the reference calls (nnkit.cpp:30, :41).
 *
 * Parity: pinned against oracle/_ref (the reference library itself) and the
 * goldens in tests/golden/ by tests/test_oracle.py. */
#include "ocg_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];
const char* ocgo_last_error(void) { return g_err; }
static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}
enum { E_OK = 0, E_INVALID = 1, E_LOGIC = 3, E_RANGE = 4, E_COLD = 5, E_DIVERGE = 6, E_NOMEM = 7 };

/* ------------------------------------------------------------------ rng --
 * Rng = std::mt19937_64 + hand-written transforms (rng.hpp:13-42). */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->idx = 312;
}

static uint64_t mt64_next(mt64* s) {
    if (s->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
        }
        s->idx = 0;
    }
    uint64_t x = s->mt[s->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

/* rng.hpp:22 */
static double rng_uniform01(mt64* s) { return (double)(mt64_next(s) >> 11) * 0x1.0p-53; }
/* rng.hpp:24 */
static double rng_uniform(mt64* s, double lo, double hi) { return lo + (hi - lo) * rng_uniform01(s); }
/* rng.hpp:27-30 */
static int64_t rng_uniform_int(mt64* s, int64_t lo, int64_t hi) {
    uint64_t span = (uint64_t)(hi - lo + 1);
    return lo + (int64_t)(mt64_next(s) % span);
}

/* rng.hpp:44-60 */
static uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
uint64_t ocgo_derive_seed(uint64_t root, const char* tag, uint64_t n) {
    uint64_t h = 0xcbf29ce484222325ULL;
    for (const unsigned char* c = (const unsigned char*)tag; *c; ++c) {
        h ^= *c;
        h *= 0x100000001b3ULL;
    }
    return splitmix64(root ^ splitmix64(h) ^ splitmix64(n * 0x9e3779b97f4a7c15ULL + 1));
}

void ocgo_rng_u64(uint64_t seed, uint64_t* out, size_t n) {
    mt64 s;
    mt64_seed(&s, seed);
    for (size_t i = 0; i < n; ++i) out[i] = mt64_next(&s);
}
void ocgo_rng_uniform(uint64_t seed, double lo, double hi, double* out, size_t n) {
    mt64 s;
    mt64_seed(&s, seed);
    for (size_t i = 0; i < n; ++i) out[i] = rng_uniform(&s, lo, hi);
}

/* ------------------------------------------------------------ selection --
 * policy::select_caps (policy.cpp:17-64).  Grid columns are the
 * lexicographic (cpu, gpu) product (core.cpp:59-65); baseline = last column. */
int ocgo_select_caps(const double* rows, int64_t nrows, const int32_t* cpu, int32_t ncpu,
                     const int32_t* gpu, int32_t ngpu, double gamma, int32_t* idx, double* saving,
                     double* loss_out, int32_t* ncand) {
    const int64_t n = (int64_t)ncpu * ngpu;
    if (!(gamma > 0.0 && gamma < 1.0)) return fail(E_INVALID, "select_caps: gamma must lie in (0, 1)");
    const int cb = cpu[ncpu - 1], gb = gpu[ngpu - 1];
    const double e_base = cb + gb; /* policy.cpp:31, int sum converted */
    for (int64_t r = 0; r < nrows; ++r) {
        const double* row = rows + r * n;
        for (int64_t j = 0; j < n; ++j)
            if (!isfinite(row[j]) || row[j] <= 0.0)
                return fail(E_INVALID, "select_caps: performance entries must be positive");
        const double p_base = row[n - 1];
        int have = 0, best_j = -1, cands = 0;
        double best_saving = 0.0, best_loss = 0.0, best_perf = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            const int c = cpu[j / ngpu], g = gpu[j % ngpu];
            const double p = row[j];
            const double loss = 1.0 - p / p_base;
            if (loss > gamma) continue;
            const double e_pred = (double)(c + g) / p;
            const double s = (e_base - e_pred) / e_base;
            ++cands;
            int better;
            if (!have) better = 1;
            else if (s != best_saving) better = s > best_saving;
            else if (p != best_perf) better = p > best_perf;
            else {
                const int bc = cpu[best_j / ngpu], bg = gpu[best_j % ngpu];
                const int sum = c + g, bsum = bc + bg;
                if (sum != bsum) better = sum < bsum;
                else better = (c < bc) || (c == bc && g < bg);
            }
            if (better) {
                best_j = (int)j;
                best_saving = s;
                best_loss = loss;
                best_perf = p;
                have = 1;
            }
        }
        if (!have) return fail(E_LOGIC, "select_caps: empty valid set");
        idx[r] = best_j;
        saving[r] = best_saving;
        loss_out[r] = best_loss;
        ncand[r] = cands;
    }
    return E_OK;
}

/* ProbePlan::default_plan (policy.cpp:66-82) as column indices */
int ocgo_default_plan(const int32_t* cpu, int32_t ncpu, const int32_t* gpu, int32_t ngpu,
                      int32_t* out_cols, int32_t* count) {
    (void)cpu;
    (void)gpu;
    const int32_t want_c[6] = {ncpu - 1, 0, 0, ncpu - 1, ncpu / 2, ncpu / 4};
    const int32_t want_g[6] = {ngpu - 1, 0, ngpu - 1, 0, ngpu / 2, ngpu / 4};
    int32_t k = 0;
    for (int w = 0; w < 6; ++w) {
        int32_t col = want_c[w] * ngpu + want_g[w];
        int dup = 0;
        for (int32_t q = 0; q < k; ++q) dup |= out_cols[q] == col;
        if (!dup) out_cols[k++] = col;
    }
    *count = k;
    return E_OK;
}

/* ------------------------------------------------------------------ ncf --
 * Model = app table (m x ka) + setting table (n x ks) + MLP
 * [ka+ks] -> hidden... -> 1, SELU hidden, identity out (cfcomplete.cpp:74-86).
 * Flat parameter layout = the reference's Adam block order
 * (cfcomplete.cpp:107-110, nnkit.cpp:91-98): app, setting, then per layer
 * W (out x in, row-major) and b. */
#define MAXL 9
#define MAXW 512
static const double kLambda = 1.0507009873554805, kAlpha = 1.6732632423543772; /* nnkit.hpp:20-21 */

typedef struct {
    int64_t m, n, ka, ks, nl;
    int64_t dims[MAXL + 1];
    int64_t off_w[MAXL], off_b[MAXL];
    int64_t total;
} layout;

static int make_layout(int64_t m, int64_t n, const ocgo_hyper* h, layout* L) {
    if (h->n_hidden < 0 || h->n_hidden > MAXL - 1) return fail(E_INVALID, "ncf: too many hidden layers");
    L->m = m;
    L->n = n;
    L->ka = h->app_dim;
    L->ks = h->setting_dim;
    L->nl = h->n_hidden + 1;
    L->dims[0] = h->app_dim + h->setting_dim;
    for (int64_t l = 0; l < h->n_hidden; ++l) L->dims[l + 1] = h->hidden[l];
    L->dims[L->nl] = 1;
    for (int64_t l = 0; l <= L->nl; ++l)
        if (L->dims[l] <= 0 || L->dims[l] > MAXW) return fail(E_INVALID, "mlp: bad layer width");
    int64_t off = m * h->app_dim + n * h->setting_dim;
    for (int64_t l = 0; l < L->nl; ++l) {
        L->off_w[l] = off;
        off += L->dims[l] * L->dims[l + 1];
        L->off_b[l] = off;
        off += L->dims[l + 1];
    }
    L->total = off;
    return E_OK;
}

int64_t ocgo_ncf_param_count(int64_t m, int64_t n, const ocgo_hyper* h) {
    layout L;
    if (make_layout(m, n, h, &L)) return -1;
    return L.total;
}

/* nnkit.cpp:27-45 */
static double act(int hidden, double z) {
    if (!hidden) return z;
    return z > 0 ? kLambda * z : kLambda * kAlpha * (exp(z) - 1.0);
}
static double act_grad(int hidden, double z) {
    if (!hidden) return 1.0;
    return z > 0 ? kLambda : kLambda * kAlpha * exp(z);
}

/* The reference's two kernel lanes (kern::Ops, kernels.hpp:12-26).
 * lane 0: kernels_scalar.cpp (baseline x86-64, no FMA).
 * lane 1: kernels_avx2.cpp as g++ -O3 -mavx2 -mfma compiles it: dot = four
 *   FMA partial sums over full 4-chunks, hsum (a0+a2)+(a1+a3), plus a tail
 *   that g++ vectorises as unfused products for the first two leftover
 *   elements and an FMA for a third/lone one; axpy = FMA everywhere;
 *   adam = FMA moment updates and p = fnma(lr, num/den, p) (g++ contracts the
 *   intrinsics' sub(p, mul(lr, q))) on full 4-chunks of each block, scalar
 *   formula on the block tail. */
static int g_lane = 0;
static double lane_dot(const double* w, const double* x, int64_t n) {
    if (g_lane == 0) {
        double acc = 0.0;
        for (int64_t i = 0; i < n; ++i) acc += w[i] * x[i];
        return acc;
    }
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int64_t i = 0;
    for (; i + 4 <= n; i += 4) {
        a0 = fma(w[i], x[i], a0);
        a1 = fma(w[i + 1], x[i + 1], a1);
        a2 = fma(w[i + 2], x[i + 2], a2);
        a3 = fma(w[i + 3], x[i + 3], a3);
    }
    double tail = 0.0;
    const int64_t r = n - i;
    if (r >= 2) {
        tail = tail + w[i] * x[i];
        tail = tail + w[i + 1] * x[i + 1];
        if (r == 3) tail = fma(w[i + 2], x[i + 2], tail);
    } else if (r == 1) {
        tail = fma(w[i], x[i], tail);
    }
    return ((a0 + a2) + (a1 + a3)) + tail;
}
static double lane_axpy(double y, double a, double x) { return g_lane == 0 ? y + a * x : fma(a, x, y); }
static void lane_adam(double* p, const double* g, double* m, double* v, int64_t n, double lr, double b1, double b2,
                      double eps, double b1p, double b2p) {
    const double mc = 1.0 / (1.0 - b1p), vc = 1.0 / (1.0 - b2p);
    const int64_t nvec = g_lane == 0 ? 0 : (n & ~(int64_t)3);
    for (int64_t i = 0; i < nvec; ++i) {
        m[i] = fma(b1, m[i], (1.0 - b1) * g[i]);
        v[i] = fma(b2, v[i], (1.0 - b2) * (g[i] * g[i]));
        const double num = m[i] * mc, den = sqrt(v[i] * vc) + eps;
        p[i] = fma(-lr, num / den, p[i]); /* g++ fuses sub(p, mul(lr, q)) into vfnmadd */
    }
    for (int64_t i = nvec; i < n; ++i) {
        m[i] = b1 * m[i] + (1.0 - b1) * g[i];
        v[i] = b2 * v[i] + (1.0 - b2) * g[i] * g[i];
        p[i] -= lr * (m[i] * mc) / (sqrt(v[i] * vc) + eps);
    }
}

/* forward with tape (nnkit.cpp:124-138); matvec = dot per row */
static double forward(const layout* L, const double* P, const double* x, double acts[][MAXW],
                      double pre[][MAXW]) {
    double a[MAXW], z[MAXW];
    memcpy(a, x, sizeof(double) * (size_t)L->dims[0]);
    for (int64_t l = 0; l < L->nl; ++l) {
        const int64_t in = L->dims[l], out = L->dims[l + 1];
        const double* W = P + L->off_w[l];
        const double* b = P + L->off_b[l];
        if (acts) memcpy(acts[l], a, sizeof(double) * (size_t)in);
        for (int64_t o = 0; o < out; ++o) {
            z[o] = lane_dot(W + o * in, a, in) + b[o];
        }
        if (pre) memcpy(pre[l], z, sizeof(double) * (size_t)out);
        const int hidden = l + 1 < L->nl;
        for (int64_t o = 0; o < out; ++o) a[o] = act(hidden, z[o]);
    }
    return a[0];
}

static void concat(const layout* L, const double* P, int64_t i, int64_t j, double* x) {
    memcpy(x, P + i * L->ka, sizeof(double) * (size_t)L->ka);
    memcpy(x + L->ka, P + L->m * L->ka + j * L->ks, sizeof(double) * (size_t)L->ks);
}

typedef struct {
    int64_t app, setting;
    double value;
} cell;

/* cells_mse (cfcomplete.cpp:34-43) */
static double cells_mse(const layout* L, const double* P, const cell* c, int64_t nc) {
    if (nc == 0) return 0.0;
    double acc = 0.0, x[MAXW];
    for (int64_t k = 0; k < nc; ++k) {
        concat(L, P, c[k].app, c[k].setting, x);
        const double err = forward(L, P, x, NULL, NULL) - c[k].value;
        acc += err * err;
    }
    return acc / (double)nc;
}

/* backprop_sample (nnkit.cpp:184-212) + embedding-grad scatter
 * (cfcomplete.cpp:170-174) accumulating into G (flat, same layout as P). */
static void backprop(const layout* L, const double* P, const cell* c, double scale, double* G) {
    double x[MAXW], acts[MAXL][MAXW], pre[MAXL][MAXW], delta[MAXW], nd[MAXW];
    concat(L, P, c->app, c->setting, x);
    const double out = forward(L, P, x, acts, pre);
    const double err = out - c->value;
    delta[0] = 2.0 * err * scale;
    for (int64_t l = L->nl - 1; l >= 0; --l) {
        const int64_t in = L->dims[l], outd = L->dims[l + 1];
        const int hidden = l + 1 < L->nl;
        const double* W = P + L->off_w[l];
        double* GW = G + L->off_w[l];
        double* Gb = G + L->off_b[l];
        for (int64_t o = 0; o < outd; ++o) delta[o] *= act_grad(hidden, pre[l][o]);
        for (int64_t r = 0; r < outd; ++r) /* outer_acc kernels_scalar.cpp:28-30 */
            for (int64_t q = 0; q < in; ++q) GW[r * in + q] = lane_axpy(GW[r * in + q], delta[r], acts[l][q]);
        for (int64_t o = 0; o < outd; ++o) Gb[o] += delta[o];
        for (int64_t q = 0; q < in; ++q) nd[q] = 0.0; /* matvec_t kernels_scalar.cpp:23-26 */
        for (int64_t r = 0; r < outd; ++r)
            for (int64_t q = 0; q < in; ++q) nd[q] = lane_axpy(nd[q], delta[r], W[r * in + q]);
        memcpy(delta, nd, sizeof(double) * (size_t)in);
    }
    for (int64_t k = 0; k < L->ka; ++k) G[c->app * L->ka + k] += delta[k];
    for (int64_t k = 0; k < L->ks; ++k) G[L->m * L->ka + c->setting * L->ks + k] += delta[L->ka + k];
}

void ocgo_set_lane(int lane) { g_lane = lane; }

int ocgo_ncf_fit(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col,
                 const double* val, const ocgo_hyper* h, uint64_t seed, double* P, ocgo_meta* meta,
                 uint8_t* app_seen, uint8_t* setting_seen) {
    /* cfcomplete.cpp:64-66 */
    if (h->app_dim == 0 || h->setting_dim == 0 || h->lr <= 0 || h->max_epochs <= 0 || h->batch_size <= 0 ||
        h->val_fraction < 0 || h->val_fraction >= 1)
        return fail(E_INVALID, "ncf: bad hyperparameters");
    layout L;
    int rc = make_layout(m, n, h, &L);
    if (rc) return rc;
    const int64_t nc = row_ptr[m];
    if (nc == 0) return fail(E_INVALID, "ncf: matrix has no observed entries");
    if (m == 0 || n == 0) return fail(E_INVALID, "embedding: zero shape");

    /* gather cells in row-major order (cfcomplete.cpp:68-71) */
    cell* cells = malloc(sizeof(cell) * (size_t)nc);
    for (int64_t i = 0; i < m; ++i)
        for (int64_t q = row_ptr[i]; q < row_ptr[i + 1]; ++q) cells[q] = (cell){i, col[q], val[q]};

    /* init (cfcomplete.cpp:74-86; nnkit.cpp:47-64, :253-262) */
    mt64 rng;
    mt64_seed(&rng, ocgo_derive_seed(seed, "ncf.fit", 0));
    {
        const double ba = sqrt(6.0 / (double)(m + L.ka));
        for (int64_t q = 0; q < m * L.ka; ++q) P[q] = rng_uniform(&rng, -ba, ba);
        const double bs = sqrt(6.0 / (double)(n + L.ks));
        for (int64_t q = 0; q < n * L.ks; ++q) P[m * L.ka + q] = rng_uniform(&rng, -bs, bs);
        for (int64_t l = 0; l < L.nl; ++l) {
            const double b = sqrt(6.0 / (double)(L.dims[l] + L.dims[l + 1]));
            for (int64_t q = 0; q < L.dims[l] * L.dims[l + 1]; ++q) P[L.off_w[l] + q] = rng_uniform(&rng, -b, b);
            for (int64_t q = 0; q < L.dims[l + 1]; ++q) P[L.off_b[l] + q] = 0.0;
        }
    }
    memset(app_seen, 0, (size_t)m);
    memset(setting_seen, 0, (size_t)n);
    for (int64_t q = 0; q < nc; ++q) {
        app_seen[cells[q].app] = 1;
        setting_seen[cells[q].setting] = 1;
    }

    /* validation split (cfcomplete.cpp:92-103) */
    int64_t* order = malloc(sizeof(int64_t) * (size_t)nc);
    for (int64_t q = 0; q < nc; ++q) order[q] = q;
    for (int64_t i = nc; i > 1; --i) {
        int64_t j = rng_uniform_int(&rng, 0, i - 1);
        int64_t t = order[i - 1];
        order[i - 1] = order[j];
        order[j] = t;
    }
    int64_t val_count = (int64_t)(h->val_fraction * (double)nc);
    cell* vset = malloc(sizeof(cell) * (size_t)nc);
    cell* tset = malloc(sizeof(cell) * (size_t)nc);
    int64_t nv = 0, nt = 0;
    for (int64_t q = 0; q < nc; ++q) {
        if (q < val_count) vset[nv++] = cells[order[q]];
        else tset[nt++] = cells[order[q]];
    }
    if (nt == 0) { /* std::swap(train, val) */
        cell* t = tset;
        tset = vset;
        vset = t;
        nt = nv;
        nv = 0;
    }
    const cell* mon = nv == 0 ? tset : vset;
    const int64_t nmon = nv == 0 ? nt : nv;

    const int64_t T = L.total;
    double* G = calloc((size_t)T, sizeof(double));
    double* M1 = calloc((size_t)T, sizeof(double));
    double* V1 = calloc((size_t)T, sizeof(double));
    double* best = malloc(sizeof(double) * (size_t)T);
    int64_t* idx = malloc(sizeof(int64_t) * (size_t)(nt > 0 ? nt : 1));

    meta->seed = seed;
    meta->initial_train_mse = cells_mse(&L, P, tset, nt);
    memcpy(best, P, sizeof(double) * (size_t)T);
    double best_val = cells_mse(&L, P, mon, nmon);
    int stale = 0;
    const double lr = h->lr, b1 = 0.9, b2 = 0.999, eps = 1e-8; /* nnkit.hpp:95 */
    double b1p = 1.0, b2p = 1.0;
    for (int64_t q = 0; q < nt; ++q) idx[q] = q;
    int epoch = 0;
    rc = E_OK;
    for (; epoch < h->max_epochs; ++epoch) {
        for (int64_t i = nt; i > 1; --i) { /* cfcomplete.cpp:153-154 */
            int64_t j = rng_uniform_int(&rng, 0, i - 1);
            int64_t t = idx[i - 1];
            idx[i - 1] = idx[j];
            idx[j] = t;
        }
        for (int64_t start = 0; start < nt; start += h->batch_size) {
            const int64_t end = start + h->batch_size < nt ? start + h->batch_size : nt;
            const double scale = 1.0 / (double)(end - start);
            memset(G, 0, sizeof(double) * (size_t)T);
            for (int64_t i = start; i < end; ++i) backprop(&L, P, &tset[idx[i]], scale, G);
            /* AdamState::step (nnkit.cpp:239-251): adam_update over every block, dense */
            b1p *= b1;
            b2p *= b2;
            lane_adam(P, G, M1, V1, m * L.ka, lr, b1, b2, eps, b1p, b2p);
            lane_adam(P + m * L.ka, G + m * L.ka, M1 + m * L.ka, V1 + m * L.ka, n * L.ks, lr, b1, b2, eps, b1p, b2p);
            for (int64_t l = 0; l < L.nl; ++l) {
                const int64_t ow = L.off_w[l], ob = L.off_b[l];
                lane_adam(P + ow, G + ow, M1 + ow, V1 + ow, ob - ow, lr, b1, b2, eps, b1p, b2p);
                lane_adam(P + ob, G + ob, M1 + ob, V1 + ob, L.dims[l + 1], lr, b1, b2, eps, b1p, b2p);
            }
        }
        const double vl = cells_mse(&L, P, mon, nmon); /* cfcomplete.cpp:179-188 */
        if (!isfinite(vl)) {
            rc = fail(E_DIVERGE, "ncf: divergence");
            break;
        }
        if (vl < best_val) {
            best_val = vl;
            memcpy(best, P, sizeof(double) * (size_t)T);
            stale = 0;
        } else if (++stale > h->patience) {
            ++epoch;
            break;
        }
    }
    if (rc == E_OK) {
        memcpy(P, best, sizeof(double) * (size_t)T); /* restore(best) :190 */
        meta->epochs_run = epoch;
        meta->best_val_mse = best_val;
        meta->final_train_mse = cells_mse(&L, P, tset, nt);
        for (int64_t l = 0; l < L.nl && rc == E_OK; ++l) /* check_finite nnkit.cpp:106-113 */
            for (int64_t q = L.off_w[l]; q < L.off_b[l] + L.dims[l + 1]; ++q)
                if (!isfinite(P[q])) {
                    rc = fail(3, "non-finite weight");
                    break;
                }
    }
    free(cells);
    free(order);
    free(vset);
    free(tset);
    free(G);
    free(M1);
    free(V1);
    free(best);
    free(idx);
    return rc;
}

/* NcfModel::predict (cfcomplete.cpp:47-58) */
int ocgo_ncf_predict(int64_t m, int64_t n, const ocgo_hyper* h, const double* P,
                     const uint8_t* app_seen, const uint8_t* setting_seen, const int64_t* rows,
                     const int64_t* cols, int64_t count, double* out) {
    layout L;
    int rc = make_layout(m, n, h, &L);
    if (rc) return rc;
    double x[MAXW];
    for (int64_t k = 0; k < count; ++k) {
        const int64_t i = rows[k], j = cols[k];
        if (i < 0 || i >= m) return fail(E_RANGE, "ncf: app index out of range");
        if (j < 0 || j >= n) return fail(E_RANGE, "ncf: setting index out of range");
        if (!app_seen[i]) return fail(E_COLD, "ncf: cold app row");
        if (!setting_seen[j]) return fail(E_COLD, "ncf: cold setting column");
        concat(&L, P, i, j, x);
        double v = forward(&L, P, x, NULL, NULL);
        out[k] = v < 0.01 ? 0.01 : (1.25 < v ? 1.25 : v); /* std::clamp, kPredictMin/kPerfMax */
    }
    return E_OK;
}

/* ------------------------------------------------------------------ als --
 * ALS matrix factorisation P ~ U V^T.  NO REFERENCE COUNTERPART: the
 * reference's only CF is NCF, so this oracle defines the semantics the GPU
 * path is checked against ("parity unpinned" vs the reference).
 *   init   V[j][0] = 1, V[j][f>0] = 0.01*(2u-1), u = splitmix64 stream
 *          (ocgo_als_init_value); U unused until the first row sweep
 *   sweep  rows:    u_i = (sum_j v_j v_j^T + lambda n_i I)^-1 sum_j r_ij v_j
 *          columns: v_j = (sum_i u_i u_i^T + lambda n_j I)^-1 sum_i r_ij u_i
 *          (weighted-lambda regularisation; empty row/col -> zero factor)
 *   solve  Cholesky (lower), forward + back substitution
 * FP64 throughout (the GPU runs FP32; tests compare within tolerance). */
double ocgo_als_init_value(uint64_t seed, int64_t j, int32_t f, int32_t k) {
    if (f == 0) return 1.0;
    const uint64_t h = splitmix64(seed ^ splitmix64((uint64_t)(j * k + f)));
    const double u = (double)(h >> 11) * 0x1.0p-53;
    return 0.01 * (2.0 * u - 1.0);
}

static void chol_solve(double* A, double* b, int k) {
    for (int c = 0; c < k; ++c) {
        double d = A[c * k + c];
        for (int q = 0; q < c; ++q) d -= A[c * k + q] * A[c * k + q];
        d = sqrt(d);
        A[c * k + c] = d;
        for (int r = c + 1; r < k; ++r) {
            double s = A[r * k + c];
            for (int q = 0; q < c; ++q) s -= A[r * k + q] * A[c * k + q];
            A[r * k + c] = s / d;
        }
    }
    for (int c = 0; c < k; ++c) { /* L y = b */
        double s = b[c];
        for (int q = 0; q < c; ++q) s -= A[c * k + q] * b[q];
        b[c] = s / A[c * k + c];
    }
    for (int c = k - 1; c >= 0; --c) { /* L^T x = y */
        double s = b[c];
        for (int q = c + 1; q < k; ++q) s -= A[q * k + c] * b[q];
        b[c] = s / A[c * k + c];
    }
}

static void als_half(int64_t nrows, const int64_t* ptr, const int32_t* idx, const float* val, const double* Y,
                     double* X, int k, double lambda) {
    double A[64 * 64], b[64];
    for (int64_t i = 0; i < nrows; ++i) {
        const int64_t cnt = ptr[i + 1] - ptr[i];
        if (cnt == 0) {
            for (int f = 0; f < k; ++f) X[i * k + f] = 0.0;
            continue;
        }
        memset(A, 0, sizeof(double) * (size_t)(k * k));
        memset(b, 0, sizeof(double) * (size_t)k);
        for (int64_t q = ptr[i]; q < ptr[i + 1]; ++q) {
            const double* y = Y + (int64_t)idx[q] * k;
            const double r = val[q];
            for (int a = 0; a < k; ++a) {
                b[a] += r * y[a];
                for (int c = 0; c <= a; ++c) A[a * k + c] += y[a] * y[c];
            }
        }
        for (int a = 0; a < k; ++a) A[a * k + a] += lambda * (double)cnt;
        chol_solve(A, b, k);
        for (int f = 0; f < k; ++f) X[i * k + f] = b[f];
    }
}

int ocgo_als_fit(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col, const float* val,
                 const int64_t* col_ptr, const int32_t* row_idx, const float* cval, int32_t k, double lambda,
                 int32_t sweeps, uint64_t seed, double* U, double* V) {
    if (k <= 0 || k > 64) return fail(E_INVALID, "als: rank must be in [1, 64]");
    for (int64_t j = 0; j < n; ++j)
        for (int32_t f = 0; f < k; ++f) V[j * k + f] = ocgo_als_init_value(seed, j, f, k);
    for (int32_t s = 0; s < sweeps; ++s) {
        als_half(m, row_ptr, col, val, V, U, k, lambda);
        als_half(n, col_ptr, row_idx, cval, U, V, k, lambda);
    }
    return E_OK;
}

/* Per-half pieces of ocgo_als_fit for the row-sharded (multi-rank) schedule:
 * row solves are local; column Gram records [k*k Gram | k rhs | count] are
 * summed across ranks, then every rank solves the same records. */
void ocgo_als_solve_rows(int64_t nrows, const int64_t* ptr, const int32_t* idx, const float* val, const double* Y,
                         double* X, int32_t k, double lambda) {
    als_half(nrows, ptr, idx, val, Y, X, k, lambda);
}

void ocgo_als_col_gram(int64_t ncols, const int64_t* col_ptr, const int32_t* row_idx, const float* cval,
                       const double* U, int32_t k, double* G) {
    const int64_t rec = (int64_t)k * k + k + 1;
    for (int64_t j = 0; j < ncols; ++j) {
        double* g = G + j * rec;
        memset(g, 0, sizeof(double) * (size_t)rec);
        for (int64_t q = col_ptr[j]; q < col_ptr[j + 1]; ++q) {
            const double* u = U + (int64_t)row_idx[q] * k;
            for (int a = 0; a < k; ++a) {
                g[k * k + a] += (double)cval[q] * u[a];
                for (int c = 0; c < k; ++c) g[a * k + c] += u[a] * u[c];
            }
        }
        g[k * k + k] = (double)(col_ptr[j + 1] - col_ptr[j]);
    }
}

void ocgo_als_solve_from_gram(int64_t ncols, const double* G, double* X, int32_t k, double lambda) {
    const int64_t rec = (int64_t)k * k + k + 1;
    double A[64 * 64], b[64];
    for (int64_t j = 0; j < ncols; ++j) {
        const double* g = G + j * rec;
        const double cnt = g[k * k + k];
        if (cnt == 0.0) {
            for (int f = 0; f < k; ++f) X[j * k + f] = 0.0;
            continue;
        }
        for (int a = 0; a < k; ++a) {
            for (int c = 0; c <= a; ++c) A[a * k + c] = g[a * k + c];
            b[a] = g[k * k + a];
            A[a * k + a] += lambda * cnt;
        }
        chol_solve(A, b, k);
        for (int f = 0; f < k; ++f) X[j * k + f] = b[f];
    }
}
