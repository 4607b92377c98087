/* pbkv_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path; it may be called only from tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py.  The product (libpbkv.so) never links or calls
 * it, and has no CPU fallback.
 *
 * Parity pin: validated against the reference itself (oracle/_ref/
 * libflowkv_ref.so, the reference headers compiled from /root/reference) on
 * random trees and on the reference tests' known-answer vectors
 * (tests/test_oracle.py); the reference's own 140 Catch2 tests are compiled
 * unmodified against a shim (oracle/Makefile, target ref-tests).
 *
 * It restates, on the struct-of-arrays view of a CacheTree (pbkv_tree_soa):
 *   - Forecast survival              forecast.hpp:35-41
 *   - Forecast::mass_on              forecast.hpp:64-69
 *   - single_step_value (Eq. 1)      scoring.hpp:41-45
 *   - multi_step_score (Eq. 2)       scoring.hpp:49-62
 *   - node_terms error               scoring.hpp:66-75
 *   - detail::select_victims         policies.hpp:50-83 (the greedy frontier
 *     itself -- NOT the closed form the GPU uses -- so the two are independent)
 *   - LRU / LAE / HE / KVFlow keys   policies.hpp:88-153
 *   - detail::plan_prefetch          policies.hpp:181-235
 * Arithmetic is IEEE binary64 with no contraction (-ffp-contract=off), in the
 * reference's exact evaluation order.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/pbkv.h"

#define ORC_ERRLEN 256
static char orc_err[ORC_ERRLEN];
const char* orc_last_error(void) { return orc_err; }

/* ---- forecasts --------------------------------------------------------------
 * n workflows, ids sorted ascending, p[n][H][V1].  surv[n][H] derived as in
 * the Forecast ctor (forecast.hpp:35-41). */
typedef struct {
    int64_t n;
    int H, V1;
    const int64_t* wf;
    const double* p;
    double* surv;
} orc_fc;

static int orc_fc_init(orc_fc* f, const int64_t* wf, int64_t n, int H, int V1, const double* p) {
    f->n = n;
    f->H = H;
    f->V1 = V1;
    f->wf = wf;
    f->p = p;
    f->surv = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1) * (size_t)(H > 0 ? H : 1));
    if (!f->surv) return 1;
    for (int64_t i = 0; i < n; ++i) {
        if (i > 0 && wf[i] <= wf[i - 1]) {
            snprintf(orc_err, ORC_ERRLEN, "oracle: forecast ids must be strictly ascending");
            return 1;
        }
        double s = 1.0;
        for (int k = 0; k < H; ++k) {
            f->surv[i * H + k] = s;
            s *= 1.0 - p[(i * H + k) * V1 + (V1 - 1)];
            if (s < 0.0) s = 0.0;
        }
    }
    return 0;
}

static int64_t orc_fc_find(const orc_fc* f, int64_t w) {
    int64_t lo = 0, hi = f->n;
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (f->wf[mid] < w)
            lo = mid + 1;
        else
            hi = mid;
    }
    return (lo < f->n && f->wf[lo] == w) ? lo : -1;
}

/* Forecast::mass_on (forecast.hpp:64-69) */
static double orc_mass_on(const orc_fc* f, int64_t i, int k, uint64_t bits) {
    double s = 0.0;
    const double* row = f->p + (i * f->H + k) * f->V1;
    for (int a = 0; a < f->V1 - 1; ++a)
        if (bits & (1ULL << a)) s += row[a];
    return s;
}

/* multi_step_score over node_terms (scoring.hpp:49-75).  Returns 0 ok, 1 error. */
static int orc_score_one(const pbkv_tree_soa* t, const orc_fc* f, int K, double gamma, int32_t id, double* out) {
    double total = 0.0;
    for (int64_t e = t->acc_off[id]; e < t->acc_off[id + 1]; ++e) {
        int64_t i = orc_fc_find(f, t->acc_wf[e]);
        if (i < 0) {
            snprintf(orc_err, ORC_ERRLEN, "missing forecast for active workflow %lld", (long long)t->acc_wf[e]);
            return 1;
        }
    }
    for (int64_t e = t->acc_off[id]; e < t->acc_off[id + 1]; ++e) {
        int64_t i = orc_fc_find(f, t->acc_wf[e]);
        if (f->H < K) {
            snprintf(orc_err, ORC_ERRLEN, "forecast horizon shorter than the scoring horizon");
            return 1;
        }
        double g = 1.0;
        for (int k = 0; k < K; ++k) {
            double gs = g * f->surv[i * f->H + k];
            double m = orc_mass_on(f, i, k, t->acc_bits[e]);
            total = total + gs * m;
            g *= gamma;
        }
    }
    *out = total;
    return 0;
}

static int orc_params_ok(int K, double gamma) {
    if (K < 1) {
        snprintf(orc_err, ORC_ERRLEN, "lookahead horizon must be >= 1");
        return 0;
    }
    if (!(gamma > 0.0 && gamma < 1.0)) {
        snprintf(orc_err, ORC_ERRLEN, "gamma must be in (0, 1)");
        return 0;
    }
    return 1;
}

/* Eq. 2 for the listed nodes (ids == NULL: all nodes 0..n-1). */
int orc_score_nodes(const pbkv_tree_soa* t, const int64_t* fwf, int64_t nf, int H, int V1, const double* P, int K,
                    double gamma, const int32_t* ids, int64_t n, double* out) {
    if (!orc_params_ok(K, gamma)) return 1;
    orc_fc f;
    if (orc_fc_init(&f, fwf, nf, H, V1, P)) {
        free(f.surv);
        return 1;
    }
    int rc = 0;
    for (int64_t j = 0; j < n && !rc; ++j) rc = orc_score_one(t, &f, K, gamma, ids ? ids[j] : (int32_t)j, &out[j]);
    free(f.surv);
    return rc;
}

/* single_step_value (Eq. 1) for the listed nodes. */
static int orc_value_one(const pbkv_tree_soa* t, const orc_fc* f, int32_t id, double* out) {
    double v = 0.0;
    for (int64_t e = t->acc_off[id]; e < t->acc_off[id + 1]; ++e) {
        int64_t i = orc_fc_find(f, t->acc_wf[e]);
        if (i < 0) {
            snprintf(orc_err, ORC_ERRLEN, "missing forecast for active workflow %lld", (long long)t->acc_wf[e]);
            return 1;
        }
    }
    for (int64_t e = t->acc_off[id]; e < t->acc_off[id + 1]; ++e) {
        int64_t i = orc_fc_find(f, t->acc_wf[e]);
        v += orc_mass_on(f, i, 0, t->acc_bits[e]);
    }
    *out = v;
    return 0;
}

int orc_value_nodes(const pbkv_tree_soa* t, const int64_t* fwf, int64_t nf, int H, int V1, const double* P,
                    const int32_t* ids, int64_t n, double* out) {
    orc_fc f;
    if (orc_fc_init(&f, fwf, nf, H, V1, P)) {
        free(f.surv);
        return 1;
    }
    int rc = 0;
    for (int64_t j = 0; j < n && !rc; ++j) rc = orc_value_one(t, &f, ids ? ids[j] : (int32_t)j, &out[j]);
    free(f.surv);
    return rc;
}

/* ---- victim selection: the greedy frontier of policies.hpp:50-83 ------------ */
typedef struct {
    int cls;
    double rank;
    uint64_t last;
    int32_t id;
} orc_key;

/* std::tie(cls, rank, last_access, id) < ... (policies.hpp:45-47) */
static int orc_key_less(const orc_key* a, const orc_key* b) {
    if (a->cls != b->cls) return a->cls < b->cls;
    if (a->rank < b->rank) return 1;
    if (b->rank < a->rank) return 0;
    if (a->last != b->last) return a->last < b->last;
    return a->id < b->id;
}

typedef struct {
    orc_key* a;
    int64_t n, cap;
} orc_heap;

static int orc_heap_push(orc_heap* h, orc_key k) {
    if (h->n == h->cap) {
        int64_t nc = h->cap ? h->cap * 2 : 64;
        orc_key* na = (orc_key*)realloc(h->a, sizeof(orc_key) * (size_t)nc);
        if (!na) return 1;
        h->a = na;
        h->cap = nc;
    }
    int64_t i = h->n++;
    h->a[i] = k;
    while (i > 0) {
        int64_t p = (i - 1) / 2;
        if (!orc_key_less(&h->a[i], &h->a[p])) break;
        orc_key tmp = h->a[i];
        h->a[i] = h->a[p];
        h->a[p] = tmp;
        i = p;
    }
    return 0;
}

static orc_key orc_heap_pop(orc_heap* h) {
    orc_key top = h->a[0];
    h->a[0] = h->a[--h->n];
    int64_t i = 0;
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < h->n && orc_key_less(&h->a[l], &h->a[m])) m = l;
        if (r < h->n && orc_key_less(&h->a[r], &h->a[m])) m = r;
        if (m == i) break;
        orc_key tmp = h->a[i];
        h->a[i] = h->a[m];
        h->a[m] = tmp;
        i = m;
    }
    return top;
}

static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

static int orc_locked(const int32_t* sorted, int64_t n, int32_t id) {
    return bsearch(&id, sorted, (size_t)n, sizeof(int32_t), cmp_i32) != NULL;
}

/* remaining sequences for KVFlow: workflows rw[nr] (any order), CSR roff/rseq */
typedef struct {
    const int64_t* wf;
    int64_t n;
    const int64_t* off;
    const int32_t* seq;
} orc_rem;

/* kvflow_distance (policies.hpp:121-139); returns 0 ok, 1 error. */
static int orc_kvflow_distance(const pbkv_tree_soa* t, const orc_rem* rem, int32_t id, double* out) {
    double best = INFINITY;
    for (int64_t e = t->acc_off[id]; e < t->acc_off[id + 1]; ++e) {
        int64_t w = t->acc_wf[e], r = -1;
        for (int64_t j = 0; j < rem->n; ++j)
            if (rem->wf[j] == w) {
                r = j;
                break;
            }
        if (r < 0) {
            snprintf(orc_err, ORC_ERRLEN, "kvflow needs a static remaining sequence for workflow %lld", (long long)w);
            return 1;
        }
        for (int64_t k = rem->off[r]; k < rem->off[r + 1]; ++k) {
            if (t->acc_bits[e] & (1ULL << rem->seq[k])) {
                double d = (double)(k - rem->off[r] + 1);
                if (d < best) best = d;
                break;
            }
        }
    }
    *out = best;
    return 0;
}

static int orc_key_of(const pbkv_tree_soa* t, int policy, const orc_rem* rem, int32_t id, orc_key* k) {
    k->last = t->last_access[id];
    k->id = id;
    double score = t->score ? t->score[id] : 0.0;
    switch (policy) {
        case PBKV_POLICY_LRU: /* policies.hpp:90-92 */
            k->cls = 0;
            k->rank = 0.0;
            return 0;
        case PBKV_POLICY_LAE: /* policies.hpp:99-103 */
            if (t->retired[id]) {
                k->cls = 0;
                k->rank = (double)t->ever_tagged[id];
            } else {
                k->cls = 1;
                k->rank = 0.0;
            }
            return 0;
        case PBKV_POLICY_HE: /* policies.hpp:110-114 */
            if (t->retired[id]) {
                k->cls = 0;
                k->rank = (double)t->ever_tagged[id];
            } else {
                k->cls = 1;
                k->rank = score;
            }
            return 0;
        case PBKV_POLICY_KVFLOW: { /* policies.hpp:147-152 */
            double d = INFINITY;
            if (!t->retired[id] && orc_kvflow_distance(t, rem, id, &d)) return 1;
            if (isinf(d)) {
                k->cls = 0;
                k->rank = 0.0;
            } else {
                k->cls = 1;
                k->rank = -d;
            }
            return 0;
        }
        default:
            snprintf(orc_err, ORC_ERRLEN, "unknown eviction policy");
            return 1;
    }
}

int orc_select(const pbkv_tree_soa* t, int policy, int64_t needed, const int32_t* locked, int64_t n_locked,
               const int64_t* rem_wf, int64_t n_rem, const int64_t* rem_off, const int32_t* rem_seq, int32_t* victims,
               int64_t cap, int64_t* n_victims, int64_t* freed, int* shortfall) {
    if (needed <= 0) {
        snprintf(orc_err, ORC_ERRLEN, "eviction request must free a positive amount");
        return 1;
    }
    if (policy == PBKV_POLICY_KVFLOW && !rem_wf) {
        snprintf(orc_err, ORC_ERRLEN, "kvflow selected without static sequences");
        return 1;
    }
    orc_rem rem = {rem_wf, n_rem, rem_off, rem_seq};
    const int64_t n = t->n_nodes;
    int32_t* lk = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_locked > 0 ? n_locked : 1));
    int32_t* dc = (int32_t*)calloc((size_t)n, sizeof(int32_t));
    int32_t* vdc = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    orc_heap h = {NULL, 0, 0};
    int rc = 0;
    if (!lk || !dc || !vdc) {
        snprintf(orc_err, ORC_ERRLEN, "oracle: out of memory");
        rc = 1;
        goto done;
    }
    if (n_locked > 0) memcpy(lk, locked, sizeof(int32_t) * (size_t)n_locked);
    qsort(lk, (size_t)n_locked, sizeof(int32_t), cmp_i32);
    /* device child counts from the tier image (cache.hpp:63 invariant, audited
     * at cache.hpp:370-377) */
    for (int64_t i = 1; i < n; ++i)
        if (t->tier[i] == PBKV_TIER_DEVICE && t->parent[i] >= 0) dc[t->parent[i]]++;
    for (int64_t i = 0; i < n; ++i) vdc[i] = -1;
    /* frontier = lru_leaves() minus locked (policies.hpp:56-63, cache.hpp:452) */
    for (int64_t i = 1; i < n; ++i) {
        if (t->tier[i] != PBKV_TIER_DEVICE || dc[i] != 0) continue;
        if (orc_locked(lk, n_locked, (int32_t)i)) continue;
        orc_key k;
        if (orc_key_of(t, policy, &rem, (int32_t)i, &k) || orc_heap_push(&h, k)) {
            rc = 1;
            goto done;
        }
    }
    int64_t nv = 0, fr = 0;
    while (fr < needed && h.n > 0) { /* policies.hpp:65-80 */
        orc_key top = orc_heap_pop(&h);
        int32_t id = top.id;
        if (nv < cap) victims[nv] = id;
        ++nv;
        fr += t->len[id];
        int32_t pid = t->parent[id];
        if (pid > 0 && t->tier[pid] == PBKV_TIER_DEVICE) {
            if (vdc[pid] < 0) vdc[pid] = dc[pid];
            if (--vdc[pid] == 0 && !orc_locked(lk, n_locked, pid)) {
                orc_key k;
                if (orc_key_of(t, policy, &rem, pid, &k) || orc_heap_push(&h, k)) {
                    rc = 1;
                    goto done;
                }
            }
        }
    }
    *n_victims = nv;
    *freed = fr;
    *shortfall = fr < needed; /* policies.hpp:81 */
    if (nv > cap) {
        snprintf(orc_err, ORC_ERRLEN, "oracle: victim capacity too small");
        rc = 2;
    }
done:
    free(lk);
    free(dc);
    free(vdc);
    free(h.a);
    return rc;
}

/* ---- prefetch plan: policies.hpp:181-235 ------------------------------------ */
typedef struct {
    int32_t id;
    double v;
} orc_cand;

static int cmp_cand(const void* a, const void* b) { /* value desc, id asc (policies.hpp:199-202) */
    const orc_cand* x = (const orc_cand*)a;
    const orc_cand* y = (const orc_cand*)b;
    if (x->v != y->v) return x->v > y->v ? -1 : 1;
    return (x->id > y->id) - (x->id < y->id);
}

typedef struct {
    uint64_t last;
    int32_t id;
} orc_hostkey;

static int cmp_hostkey(const void* a, const void* b) { /* host_index_ order (last_access, id), cache.hpp:434 */
    const orc_hostkey* x = (const orc_hostkey*)a;
    const orc_hostkey* y = (const orc_hostkey*)b;
    if (x->last != y->last) return x->last < y->last ? -1 : 1;
    return (x->id > y->id) - (x->id < y->id);
}

int orc_plan_prefetch(const pbkv_tree_soa* t, const int64_t* fwf, int64_t nf, int H, int V1, const double* P,
                      int64_t bandwidth, int step_duration, double rho, int32_t* cand_ids, double* cand_values,
                      int64_t cand_cap, int32_t* selected, int64_t sel_cap, pbkv_prefetch_plan* plan) {
    int64_t extra = 0;
    if (rho >= 0.0 || rho != rho) { /* aggressive (policies.hpp:228-235) */
        if (rho < 0.0 || rho > 1.0 || rho != rho) {
            snprintf(orc_err, ORC_ERRLEN, "rho must be in [0, 1]");
            return 1;
        }
        extra = (int64_t)(rho * (double)t->device_capacity);
    }
    orc_fc f;
    if (orc_fc_init(&f, fwf, nf, H, V1, P)) {
        free(f.surv);
        return 1;
    }
    memset(plan, 0, sizeof *plan);
    plan->budget_space = (t->device_capacity - t->device_used) + t->retired_device_tokens;
    plan->budget_bw = bandwidth * (int64_t)step_duration;
    plan->displacement_budget = extra;
    int64_t budget = plan->budget_space + extra;
    if (plan->budget_bw < budget) budget = plan->budget_bw;

    const int64_t n = t->n_nodes;
    orc_hostkey* hk = (orc_hostkey*)malloc(sizeof(orc_hostkey) * (size_t)(n > 0 ? n : 1));
    orc_cand* c = (orc_cand*)malloc(sizeof(orc_cand) * (size_t)(n > 0 ? n : 1));
    int rc = 0;
    int64_t nh = 0, nc = 0;
    if (!hk || !c) {
        snprintf(orc_err, ORC_ERRLEN, "oracle: out of memory");
        rc = 1;
        goto done;
    }
    for (int64_t i = 1; i < n; ++i)
        if (t->tier[i] == PBKV_TIER_HOST) {
            hk[nh].last = t->last_access[i];
            hk[nh].id = (int32_t)i;
            ++nh;
        }
    qsort(hk, (size_t)nh, sizeof(orc_hostkey), cmp_hostkey);
    for (int64_t j = 0; j < nh; ++j) { /* policies.hpp:190-198 */
        int32_t id = hk[j].id;
        if (t->tier[t->parent[id]] != PBKV_TIER_DEVICE) continue;
        double v;
        if (orc_value_one(t, &f, id, &v)) {
            rc = 1;
            goto done;
        }
        if (v <= 0.0) continue;
        c[nc].id = id;
        c[nc].v = v;
        ++nc;
    }
    qsort(c, (size_t)nc, sizeof(orc_cand), cmp_cand);
    plan->n_candidates = nc;
    for (int64_t j = 0; j < nc; ++j) {
        if (j < cand_cap) {
            if (cand_ids) cand_ids[j] = c[j].id;
            if (cand_values) cand_values[j] = c[j].v;
        }
        int64_t len = t->len[c[j].id];
        if (len <= budget - plan->selected_tokens) { /* policies.hpp:203-210 */
            if (plan->n_selected < sel_cap && selected) selected[plan->n_selected] = c[j].id;
            plan->n_selected++;
            plan->selected_tokens += len;
        }
    }
done:
    free(hk);
    free(c);
    free(f.surv);
    return rc;
}
