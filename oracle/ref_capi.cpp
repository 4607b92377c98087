// ref_capi.cpp -- C ABI over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY (oracle).  Compiled by oracle/Makefile from
// /root/reference/proj/include (never copied) into oracle/_ref/libflowkv_ref.so.
// Used by tests/ to (1) pin the C restatement (pbkv_oracle.c) and the product's
// host mirror against the real flowkv::CacheTree, and (2) by bench.py's
// cpu_baseline / --impl reference leg to time the reference policy code on the
// host cores.  Never linked or called by the product.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <span>
#include <string>
#include <vector>

#include "flowkv/cache.hpp"
#include "flowkv/forecast.hpp"
#include "flowkv/policies.hpp"
#include "flowkv/scoring.hpp"

// the shared op-stream / synthetic generator (same stream drives the product's
// RadixMirror, so the two trees can be compared field by field)
#include "../paper_2605_06472_b200/csrc/host/ops.hpp"
#include "../include/pbkv.h"

using namespace flowkv;

namespace {

struct RefHandle {
    CacheTree tree;
    std::map<WorkflowId, Forecast> forecasts;
    std::map<WorkflowId, std::vector<AgentId>> remaining;
    bool have_remaining = false;
    std::string err;
    RefHandle(std::int64_t d, std::int64_t h) : tree(d, h) {}
    ForecastProvider provider() const {
        return [this](WorkflowId w) -> const Forecast* {
            auto it = forecasts.find(w);
            return it == forecasts.end() ? nullptr : &it->second;
        };
    }
};

thread_local std::string g_err;

template <class F>
int guarded(RefHandle* h, F&& f) {
    try {
        f();
        return 0;
    } catch (const ValidationError& e) {
        (h ? h->err : g_err) = e.what();
        return 1;
    } catch (const std::exception& e) {
        (h ? h->err : g_err) = e.what();
        return 2;
    }
}

std::set<int> to_set(const std::int32_t* ids, std::int64_t n) {
    std::set<int> s;
    for (std::int64_t i = 0; i < n; ++i) s.insert(ids[i]);
    return s;
}

}  // namespace

extern "C" {

const char* fkref_last_error(void* h) { return h ? static_cast<RefHandle*>(h)->err.c_str() : g_err.c_str(); }

void* fkref_tree_new(std::int64_t device_capacity, std::int64_t host_capacity) {
    RefHandle* h = nullptr;
    guarded(nullptr, [&] { h = new RefHandle(device_capacity, host_capacity); });
    return h;
}

void fkref_tree_free(void* h) { delete static_cast<RefHandle*>(h); }

int fkref_apply_ops(void* hv, const std::int64_t* words, std::int64_t n) {
    auto* h = static_cast<RefHandle*>(hv);
    return guarded(h, [&] { pbkv::apply_ops(h->tree, words, n); });
}

int fkref_synth(void* hv, const pbkv_synth_params* p) {
    auto* h = static_cast<RefHandle*>(hv);
    return guarded(h, [&] {
        pbkv::SynthParams sp;
        sp.n_nodes = p->n_nodes;
        sp.n_workflows = p->n_workflows;
        sp.agents = p->agents;
        sp.group_size = p->group_size;
        sp.shared_len = p->shared_len;
        sp.group_len = p->group_len;
        sp.alphabet = p->alphabet;
        sp.max_rand_len = p->max_rand_len;
        sp.retired_frac = p->retired_frac;
        sp.host_every = p->host_every;
        sp.seed = p->seed;
        pbkv::synth_build(h->tree, sp);
    });
}

int fkref_shape(void* hv, pbkv_tree_soa* soa) {
    auto* h = static_cast<RefHandle*>(hv);
    const CacheTree& t = h->tree;
    soa->n_nodes = static_cast<std::int64_t>(t.node_count());
    std::int64_t e = 0;
    for (std::size_t i = 0; i < t.node_count(); ++i) e += static_cast<std::int64_t>(t.node(static_cast<int>(i)).access.size());
    soa->n_entries = e;
    soa->device_capacity = t.device_capacity();
    soa->device_used = t.device_used();
    soa->retired_device_tokens = t.retired_device_tokens();
    soa->host_capacity = t.host_capacity();
    soa->host_used = t.host_used();
    return 0;
}

int fkref_export(void* hv, pbkv_tree_soa* s) {
    auto* h = static_cast<RefHandle*>(hv);
    const CacheTree& t = h->tree;
    const std::size_t n = t.node_count();
    std::int64_t e = 0;
    for (std::size_t i = 0; i < n; ++i) {
        const auto& nd = t.node(static_cast<int>(i));
        if (s->parent) s->parent[i] = nd.parent;
        if (s->len) s->len[i] = static_cast<std::int32_t>(nd.len());
        if (s->tier) s->tier[i] = static_cast<std::uint8_t>(nd.tier);
        if (s->retired) s->retired[i] = nd.retired ? 1 : 0;
        if (s->last_access) s->last_access[i] = nd.last_access;
        if (s->ever_tagged) s->ever_tagged[i] = nd.ever_tagged;
        if (s->score) s->score[i] = nd.score;
        if (s->device_children) s->device_children[i] = nd.device_children;
        if (s->acc_off) s->acc_off[i] = e;
        for (const auto& [w, bits] : nd.access) {
            if (s->acc_wf) s->acc_wf[e] = w;
            if (s->acc_bits) s->acc_bits[e] = bits;
            ++e;
        }
    }
    if (s->acc_off) s->acc_off[n] = e;
    if (s->depth) {
        for (std::size_t i = 0; i < n; ++i) {
            int d = 0;
            for (int p = t.node(static_cast<int>(i)).parent; p >= 0; p = t.node(p).parent) ++d;
            s->depth[i] = d;
        }
    }
    return 0;
}

int fkref_set_forecasts(void* hv, const std::int64_t* wf, std::int64_t n, int horizon, int outcomes,
                        const double* p) {
    auto* h = static_cast<RefHandle*>(hv);
    return guarded(h, [&] {
        const std::size_t per = static_cast<std::size_t>(horizon) * static_cast<std::size_t>(outcomes);
        for (std::int64_t i = 0; i < n; ++i) {
            std::vector<double> steps(p + static_cast<std::size_t>(i) * per, p + static_cast<std::size_t>(i + 1) * per);
            h->forecasts.insert_or_assign(wf[i], Forecast(horizon, outcomes, std::move(steps)));
        }
    });
}

int fkref_drop_forecast(void* hv, std::int64_t w) {
    static_cast<RefHandle*>(hv)->forecasts.erase(w);
    return 0;
}

int fkref_set_remaining(void* hv, const std::int64_t* wf, std::int64_t n, const std::int64_t* off,
                        const std::int32_t* seq) {
    auto* h = static_cast<RefHandle*>(hv);
    h->remaining.clear();
    for (std::int64_t i = 0; i < n; ++i) h->remaining[wf[i]] = std::vector<AgentId>(seq + off[i], seq + off[i + 1]);
    h->have_remaining = true;
    return 0;
}

int fkref_set_score(void* hv, std::int32_t id, double s) {
    auto* h = static_cast<RefHandle*>(hv);
    h->tree.set_score(id, s);
    return 0;
}

/* refresh_scores (scoring.hpp:80-91): returns the count through *count. */
int fkref_refresh_scores(void* hv, std::int64_t w, int k, double gamma, std::int64_t* count) {
    auto* h = static_cast<RefHandle*>(hv);
    return guarded(h, [&] { *count = refresh_scores(h->tree, w, h->provider(), ScoreParams{k, gamma}); });
}

/* refresh_nodes (scoring.hpp:95-101) over ids (NULL -> all nodes). */
int fkref_refresh_nodes(void* hv, const std::int32_t* ids, std::int64_t n, int k, double gamma) {
    auto* h = static_cast<RefHandle*>(hv);
    return guarded(h, [&] {
        std::vector<int> v;
        if (ids)
            v.assign(ids, ids + n);
        else
            for (std::size_t i = 0; i < h->tree.node_count(); ++i) v.push_back(static_cast<int>(i));
        refresh_nodes(h->tree, v, h->provider(), ScoreParams{k, gamma});
    });
}

/* multi_step_score(node_terms(...)) without write-back (ids NULL -> all). */
int fkref_score_nodes(void* hv, const std::int32_t* ids, std::int64_t n, int k, double gamma, double* out) {
    auto* h = static_cast<RefHandle*>(hv);
    return guarded(h, [&] {
        auto prov = h->provider();
        ScoreParams sp{k, gamma};
        for (std::int64_t j = 0; j < n; ++j) {
            int id = ids ? ids[j] : static_cast<int>(j);
            out[j] = multi_step_score(node_terms(h->tree, id, prov), sp);
        }
    });
}

int fkref_value_nodes(void* hv, const std::int32_t* ids, std::int64_t n, double* out) {
    auto* h = static_cast<RefHandle*>(hv);
    return guarded(h, [&] {
        auto prov = h->provider();
        for (std::int64_t j = 0; j < n; ++j) out[j] = single_step_value(node_terms(h->tree, ids[j], prov));
    });
}

/* select_victims dispatcher (policies.hpp:155-168). */
int fkref_select(void* hv, int policy, std::int64_t needed, const std::int32_t* locked, std::int64_t n_locked,
                 std::int32_t* victims, std::int64_t cap, std::int64_t* n_victims, std::int64_t* freed,
                 int* shortfall) {
    auto* h = static_cast<RefHandle*>(hv);
    return guarded(h, [&] {
        std::set<int> lk = to_set(locked, n_locked);
        VictimSelection sel = select_victims(h->tree, static_cast<EvictionPolicy>(policy), needed,
                                             h->have_remaining ? &h->remaining : nullptr, lk);
        *n_victims = static_cast<std::int64_t>(sel.victims.size());
        *freed = sel.freed;
        *shortfall = sel.shortfall ? 1 : 0;
        for (std::size_t i = 0; i < sel.victims.size() && static_cast<std::int64_t>(i) < cap; ++i)
            victims[i] = sel.victims[i];
    });
}

/* plan_conservative_prefetch (rho < 0) / plan_aggressive_prefetch (policies.hpp:220-235). */
int fkref_plan(void* hv, std::int64_t bandwidth, int step, double rho, std::int32_t* cand_ids, double* cand_values,
               std::int64_t cand_cap, std::int32_t* selected, std::int64_t sel_cap, pbkv_prefetch_plan* out) {
    auto* h = static_cast<RefHandle*>(hv);
    return guarded(h, [&] {
        PrefetchPlan plan = rho < 0.0 ? plan_conservative_prefetch(h->tree, h->provider(), bandwidth, step)
                                      : plan_aggressive_prefetch(h->tree, h->provider(), bandwidth, rho, step);
        out->budget_space = plan.budget_space;
        out->budget_bw = plan.budget_bw;
        out->displacement_budget = plan.displacement_budget;
        out->selected_tokens = plan.selected_tokens;
        out->n_candidates = static_cast<std::int64_t>(plan.candidates.size());
        out->n_selected = static_cast<std::int64_t>(plan.selected.size());
        for (std::size_t i = 0; i < plan.candidates.size() && static_cast<std::int64_t>(i) < cand_cap; ++i) {
            if (cand_ids) cand_ids[i] = plan.candidates[i].first;
            if (cand_values) cand_values[i] = plan.candidates[i].second;
        }
        for (std::size_t i = 0; i < plan.selected.size() && static_cast<std::int64_t>(i) < sel_cap; ++i)
            if (selected) selected[i] = plan.selected[i];
    });
}

/* touched_nodes(w) (cache.hpp:101-104) */
int fkref_touched(void* hv, std::int64_t w, std::int32_t* ids, std::int64_t cap, std::int64_t* n) {
    auto* h = static_cast<RefHandle*>(hv);
    const std::vector<int>* t = h->tree.touched_nodes(w);
    *n = t ? static_cast<std::int64_t>(t->size()) : 0;
    if (t)
        for (std::size_t i = 0; i < t->size() && static_cast<std::int64_t>(i) < cap; ++i) ids[i] = (*t)[i];
    return 0;
}

}  // extern "C"
