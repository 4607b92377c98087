// flowkv_gpu.hpp -- C++ drop-in for the reference policy interface, on the
// pbkv C ABI (include/pbkv.h) and its sm_100a kernels.
//
// The reference (/root/reference/proj/include/flowkv) selects policies at
// call sites through inline free functions (no virtual interface, SURVEY.md
// §8(b)).  This header declares the same functions, with the same
// signatures, argument meaning and flowkv::ValidationError messages, in
// namespace flowkv::gpu:
//
//   reference                                          replaced by
//   refresh_scores            scoring.hpp:80-91        gpu::refresh_scores
//   refresh_nodes             scoring.hpp:95-101       gpu::refresh_nodes
//   select_victims            policies.hpp:155-168     gpu::select_victims
//   select_victims_lru        policies.hpp:88-93       gpu::select_victims_lru
//   select_victims_lae        policies.hpp:97-104      gpu::select_victims_lae
//   select_victims_hierarchical policies.hpp:108-115   gpu::select_victims_hierarchical
//   select_victims_kvflow     policies.hpp:144-153     gpu::select_victims_kvflow
//   plan_conservative_prefetch policies.hpp:220-224    gpu::plan_conservative_prefetch
//   plan_aggressive_prefetch  policies.hpp:228-235     gpu::plan_aggressive_prefetch
//   CallGraph::true_kstep_marginals callgraph.hpp:136  gpu::oracle_predict_batch
//   noisy_predict             predictor.hpp:25-35      gpu::oracle_predict_batch(.., lambda)
//   MarkovModel::predict      predictor.hpp:79-118     gpu::markov_predict_batch
//
// A caller switches by qualifying the call (or, for an unmodified
// simulator.hpp, by the macro interposition shown in INTEGRATION.md).
// Include the reference headers first; link libpbkv.so.
//
// Tree mirroring: a tree that is a TrackedCacheTree (tracked_tree.hpp --
// the reference CacheTree with a change log; an unmodified simulator.hpp
// holds one via `#define CacheTree TrackedCacheTree`) is
// mirrored incrementally: each call uploads only the nodes changed since
// that context last saw the tree (pbkv_mirror_delta).  A plain CacheTree has
// no change log, so its calls upload a full struct-of-arrays image (exact;
// SURVEY.md §7 hard part 9).  Forecasts are copied at
// call time (the provider's pointers are only valid during the call,
// SURVEY.md §8(b) "Ownership").  One pbkv context per thread and
// (K, gamma, A): scenario cells run on separate threads and share nothing
// (scenario.hpp:291-301).  There is no CPU fallback: a missing or non-sm_100
// device surfaces as std::runtime_error from the first call.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <set>
#include <span>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include <algorithm>
#include <deque>

#include "flowkv/cache.hpp"
#include "flowkv/errors.hpp"
#include "flowkv/forecast.hpp"
#include "flowkv/policies.hpp"
#include "flowkv/scoring.hpp"
#ifdef PBKV_WITH_PREDICTORS  // callgraph.hpp / predictor.hpp need nlohmann json.hpp
#include "flowkv/callgraph.hpp"
#include "flowkv/predictor.hpp"
#endif

#include "../pbkv.h"
#include "tracked_tree.hpp"

namespace flowkv::gpu {

namespace detail {

// Status -> exception: PBKV_EINVAL carries the reference's ValidationError
// message verbatim; everything else is a device / ABI failure.
inline void check(int rc, const pbkv_ctx* ctx) {
    if (rc == PBKV_OK) return;
    std::string msg = pbkv_last_error(ctx);
    if (rc == PBKV_EINVAL) throw ValidationError(msg);
    throw std::runtime_error("pbkv: " + msg);
}

inline int device_ordinal() {
    const char* s = std::getenv("PBKV_DEVICE");
    return s ? std::atoi(s) : 0;
}

// per-thread context cache keyed by the score parameters and agent count;
// each context remembers which tracked tree (uid) its mirror holds and the
// change-log position it has applied
class Contexts {
public:
    struct Entry {
        pbkv_ctx* ctx = nullptr;
        std::uint64_t uid = 0;
        std::int64_t pos = 0;
    };
    Entry& get(int k, double gamma, int agents) {
        auto key = std::make_tuple(k, gamma, agents);
        auto it = ctx_.find(key);
        if (it != ctx_.end()) return it->second.e;
        pbkv_cfg cfg{device_ordinal(), k, gamma, agents};
        pbkv_ctx* c = nullptr;
        check(pbkv_ctx_create(&c, &cfg), nullptr);
        Slot& s = ctx_[key];
        s.h.reset(c);
        s.e.ctx = c;
        return s.e;
    }

private:
    struct Del {
        void operator()(pbkv_ctx* c) const { pbkv_ctx_destroy(c); }
    };
    struct Slot {
        std::unique_ptr<pbkv_ctx, Del> h;
        Entry e;
    };
    std::map<std::tuple<int, double, int>, Slot> ctx_;
};

inline Contexts& contexts() {
    thread_local Contexts c;
    return c;
}

// Brings the context's device mirror up to date with `tree`: the changed
// nodes of a tracked tree, or a full image of a plain CacheTree.
inline void mirror(Contexts::Entry& e, const CacheTree& tree) {
    thread_local TreeImage img;
    thread_local DeltaBatch batch;
    thread_local std::vector<int> ids;
    if (const TrackedCacheTree* tt = tracked(tree)) {
        check(sync_mirror(e.ctx, *tt, e.uid, e.pos, ids, batch, img), e.ctx);
        return;
    }
    img.build(tree);
    e.uid = 0;
    check(pbkv_mirror_full(e.ctx, &img.soa), e.ctx);
}

// Uploads the forecasts of every workflow tagged on `ids`, grouped by
// horizon.  Returns the agent count of the first forecast (or `fallback`).
struct ForecastBatch {
    std::map<int, std::pair<std::vector<std::int64_t>, std::vector<double>>> by_horizon;
    int outcomes = 0;

    void add(WorkflowId w, const Forecast& f) {
        if (outcomes == 0) outcomes = f.outcomes();
        auto& [ids, p] = by_horizon[f.horizon()];
        ids.push_back(static_cast<std::int64_t>(w));
        for (int k = 0; k < f.horizon(); ++k)
            for (int a = 0; a < f.outcomes(); ++a) p.push_back(f.at(k, a));
    }
    void upload(pbkv_ctx* c) const {
        for (const auto& [h, v] : by_horizon)
            // rows of Forecast objects (validated by their constructor): no
            // synchronisation here, the next call reads the status word
            check(pbkv_forecast_put_async(c, v.first.data(), static_cast<std::int64_t>(v.first.size()), h, outcomes,
                                          v.second.data()),
                  c);
    }
};

// node_terms (scoring.hpp:66-75) + multi_step_score (scoring.hpp:49-62)
// preconditions for one node, in the reference's order: the first missing
// forecast, then params.validate(), then any short horizon.
inline const char* node_precheck(const CacheTree& tree, int id, const ForecastProvider& fp,
                                 const ScoreParams& params, std::string& msg, ForecastBatch* batch,
                                 std::set<WorkflowId>& seen) {
    const auto& acc = tree.node(id).access;
    for (const auto& [w, b] : acc) {
        (void)b;
        if (!fp(w)) {
            msg = "missing forecast for active workflow " + std::to_string(w);
            return msg.c_str();
        }
    }
    if (params.k < 1) return "lookahead horizon must be >= 1";
    if (!(params.gamma > 0.0 && params.gamma < 1.0)) return "gamma must be in (0, 1)";
    for (const auto& [w, b] : acc) {
        (void)b;
        const Forecast* f = fp(w);
        if (f->horizon() < params.k) return "forecast horizon shorter than the scoring horizon";
        if (batch && seen.insert(w).second) batch->add(w, *f);
    }
    return nullptr;
}

// Eq. 2 for `ids` on the device, written back with set_score in order; the
// first failing node raises after the nodes before it were written (as the
// reference loop does).
inline int score_ids(CacheTree& tree, std::span<const int> ids, const ForecastProvider& fp,
                     const ScoreParams& params) {
    ForecastBatch batch;
    std::set<WorkflowId> seen;
    std::string msg;
    const char* err = nullptr;
    std::size_t ok = 0;
    for (; ok < ids.size(); ++ok) {
        err = node_precheck(tree, ids[ok], fp, params, msg, &batch, seen);
        if (err) break;
    }
    if (ok > 0) {
        int agents = batch.outcomes ? batch.outcomes - 1 : 1;
        Contexts::Entry& e = contexts().get(params.k, params.gamma, agents);
        pbkv_ctx* c = e.ctx;
        mirror(e, tree);
        batch.upload(c);
        std::vector<double> out(ok);
        check(pbkv_score_nodes(c, ids.data(), static_cast<std::int64_t>(ok), out.data()), c);
        // a tracked tree logs the write-back (set_score is not virtual)
        if (const TrackedCacheTree* tt = tracked(tree)) {
            auto* wt = const_cast<TrackedCacheTree*>(tt);
            for (std::size_t i = 0; i < ok; ++i) wt->set_score(ids[i], out[i]);
        } else {
            for (std::size_t i = 0; i < ok; ++i) tree.set_score(ids[i], out[i]);
        }
    }
    if (err) throw ValidationError(err);
    return static_cast<int>(ok);
}

inline VictimSelection select(const CacheTree& tree, int policy, std::int64_t needed,
                              const std::map<WorkflowId, std::vector<AgentId>>* remaining,
                              const std::set<int>& locked) {
    // selection needs no forecasts; the context's score parameters are unused
    Contexts::Entry& e = contexts().get(3, 0.7, 63);
    pbkv_ctx* c = e.ctx;
    mirror(e, tree);
    if (policy == PBKV_POLICY_KVFLOW) {
        std::vector<std::int64_t> wf, off{0};
        std::vector<std::int32_t> seq;
        for (const auto& [w, s] : *remaining) {
            wf.push_back(static_cast<std::int64_t>(w));
            for (AgentId a : s) seq.push_back(static_cast<std::int32_t>(a));
            off.push_back(static_cast<std::int64_t>(seq.size()));
        }
        check(pbkv_set_remaining(c, wf.data(), static_cast<std::int64_t>(wf.size()), off.data(), seq.data()), c);
    }
    std::vector<std::int32_t> lk(locked.begin(), locked.end());
    VictimSelection sel;
    sel.victims.resize(tree.node_count());
    std::int64_t nv = 0, freed = 0;
    int shortfall = 0;
    check(pbkv_select(c, policy, PBKV_SCORE_CACHED, needed, lk.data(), static_cast<std::int64_t>(lk.size()),
                      sel.victims.data(), static_cast<std::int64_t>(sel.victims.size()), &nv, &freed, &shortfall),
          c);
    sel.victims.resize(static_cast<std::size_t>(nv));
    sel.freed = freed;
    sel.shortfall = shortfall != 0;
    return sel;
}

inline PrefetchPlan plan(const CacheTree& tree, const ForecastProvider& fp, std::int64_t bandwidth,
                         int step_duration, double rho) {
    // candidates: host nodes with a DEVICE parent (policies.hpp:190-193); the
    // first one (host_index_ order) with a missing forecast raises
    ForecastBatch batch;
    std::set<WorkflowId> seen;
    for (auto [last, id] : tree.host_nodes()) {
        (void)last;
        const CacheTree::Node& n = tree.node(id);
        if (tree.node(n.parent).tier != Tier::Device) continue;
        for (const auto& [w, b] : n.access) {
            (void)b;
            const Forecast* f = fp(w);
            if (!f) throw ValidationError("missing forecast for active workflow " + std::to_string(w));
            if (seen.insert(w).second) batch.add(w, *f);
        }
    }
    const int agents = batch.outcomes ? batch.outcomes - 1 : 1;
    // Eq. 1 reads step 0 only: any horizon >= 1 serves (context K = 1)
    Contexts::Entry& e = contexts().get(1, 0.7, agents);
    pbkv_ctx* c = e.ctx;
    mirror(e, tree);
    batch.upload(c);
    pbkv_prefetch_plan p{};
    check(pbkv_plan_prefetch(c, bandwidth, step_duration, rho, nullptr, nullptr, 0, nullptr, 0, &p), c);
    std::vector<std::int32_t> cid(static_cast<std::size_t>(p.n_candidates)), sel(static_cast<std::size_t>(p.n_selected));
    std::vector<double> cv(static_cast<std::size_t>(p.n_candidates));
    check(pbkv_plan_fetch(c, cid.data(), cv.data(), p.n_candidates, sel.data(), p.n_selected), c);
    PrefetchPlan out;
    out.budget_space = p.budget_space;
    out.budget_bw = p.budget_bw;
    out.displacement_budget = p.displacement_budget;
    out.selected_tokens = p.selected_tokens;
    out.candidates.reserve(static_cast<std::size_t>(p.n_candidates));
    for (std::int64_t i = 0; i < p.n_candidates; ++i)
        out.candidates.push_back({cid[static_cast<std::size_t>(i)], cv[static_cast<std::size_t>(i)]});
    out.selected.assign(sel.begin(), sel.begin() + p.n_selected);
    return out;
}

}  // namespace detail

// ---- scoring.hpp -------------------------------------------------------------
inline int refresh_scores(CacheTree& tree, WorkflowId changed_workflow, const ForecastProvider& forecasts,
                          const ScoreParams& params) {
    const std::vector<int>* touched = tree.touched_nodes(changed_workflow);
    if (!touched) return 0;
    const std::vector<int> ids = *touched;  // set_score never changes the list
    return detail::score_ids(tree, ids, forecasts, params);
}

inline void refresh_nodes(CacheTree& tree, std::span<const int> ids, const ForecastProvider& forecasts,
                          const ScoreParams& params) {
    detail::score_ids(tree, ids, forecasts, params);
}

// ---- policies.hpp ------------------------------------------------------------
inline VictimSelection select_victims_lru(const CacheTree& tree, std::int64_t needed,
                                          const std::set<int>& locked = {}) {
    return detail::select(tree, PBKV_POLICY_LRU, needed, nullptr, locked);
}

inline VictimSelection select_victims_lae(const CacheTree& tree, std::int64_t needed,
                                          const std::set<int>& locked = {}) {
    return detail::select(tree, PBKV_POLICY_LAE, needed, nullptr, locked);
}

inline VictimSelection select_victims_hierarchical(const CacheTree& tree, std::int64_t needed,
                                                   const std::set<int>& locked = {}) {
    return detail::select(tree, PBKV_POLICY_HE, needed, nullptr, locked);
}

inline VictimSelection select_victims_kvflow(const CacheTree& tree, std::int64_t needed,
                                             const std::map<WorkflowId, std::vector<AgentId>>& remaining,
                                             const std::set<int>& locked = {}) {
    return detail::select(tree, PBKV_POLICY_KVFLOW, needed, &remaining, locked);
}

inline VictimSelection select_victims(const CacheTree& tree, EvictionPolicy policy, std::int64_t needed,
                                      const std::map<WorkflowId, std::vector<AgentId>>* remaining,
                                      const std::set<int>& locked = {}) {
    switch (policy) {
        // qualified: argument-dependent lookup would also find flowkv::
        case EvictionPolicy::Lru: return gpu::select_victims_lru(tree, needed, locked);
        case EvictionPolicy::Lae: return gpu::select_victims_lae(tree, needed, locked);
        case EvictionPolicy::Hierarchical: return gpu::select_victims_hierarchical(tree, needed, locked);
        case EvictionPolicy::KvFlow:
            if (!remaining) throw ValidationError("kvflow selected without static sequences");
            return gpu::select_victims_kvflow(tree, needed, *remaining, locked);
    }
    throw ValidationError("unknown eviction policy");
}

inline PrefetchPlan plan_conservative_prefetch(const CacheTree& tree, const ForecastProvider& forecasts,
                                               std::int64_t bandwidth, int step_duration = 1) {
    return detail::plan(tree, forecasts, bandwidth, step_duration, -1.0);
}

inline PrefetchPlan plan_aggressive_prefetch(const CacheTree& tree, const ForecastProvider& forecasts,
                                             std::int64_t bandwidth, double rho, int step_duration = 1) {
    if (rho < 0.0 || rho > 1.0) throw ValidationError("rho must be in [0, 1]");
    return detail::plan(tree, forecasts, bandwidth, step_duration, rho);
}

#ifdef PBKV_WITH_PREDICTORS
// ---- predictor slot (simulator.hpp:414-421): the reference predictors, batched ----
// Both propagate alive mass over context states visited in std::map order.
// The state table is built on the host from the model's public interface
// (row_for_prefix / row_for) as the closure of the requested start contexts,
// sorted in the reference's map order; the device replays the propagation
// bit for bit (csrc/fmodel.cu).
namespace detail {

template <class Key>
struct StateTable {
    std::vector<Key> keys;  // sorted (the std::map order)
    std::vector<double> rows;
    std::vector<std::int32_t> next;

    template <class RowFn, class NextFn>
    void build(const std::vector<Key>& seeds, int A, RowFn&& row_of, NextFn&& next_of) {
        std::map<Key, std::vector<double>> rowmap;
        std::deque<Key> q(seeds.begin(), seeds.end());
        while (!q.empty()) {
            Key k = q.front();
            q.pop_front();
            if (rowmap.count(k)) continue;
            std::vector<double> r = row_of(k);
            for (int a = 0; a < A; ++a)
                if (r[static_cast<std::size_t>(a)] > 0.0) q.push_back(next_of(k, a));
            rowmap.emplace(std::move(k), std::move(r));
        }
        keys.clear();
        rows.clear();
        for (auto& [k, r] : rowmap) {
            keys.push_back(k);
            rows.insert(rows.end(), r.begin(), r.end());
        }
        next.assign(keys.size() * static_cast<std::size_t>(A), -1);
        for (std::size_t s = 0; s < keys.size(); ++s)
            for (int a = 0; a < A; ++a) {
                if (!(rows[s * (A + 1) + static_cast<std::size_t>(a)] > 0.0)) continue;
                auto it = std::lower_bound(keys.begin(), keys.end(), next_of(keys[s], a));
                next[s * A + static_cast<std::size_t>(a)] = static_cast<std::int32_t>(it - keys.begin());
            }
    }
    std::int32_t index(const Key& k) const {
        auto it = std::lower_bound(keys.begin(), keys.end(), k);
        return (it != keys.end() && *it == k) ? static_cast<std::int32_t>(it - keys.begin()) : -1;
    }
};

inline std::vector<Forecast> propagate(int A, const std::vector<double>& rows, const std::vector<std::int32_t>& next,
                                       const std::vector<std::int32_t>& start, int K, double lambda) {
    pbkv_ctx* c = contexts().get(K, 0.7, A).ctx;
    pbkv_fmodel m{A, static_cast<std::int64_t>(rows.size() / static_cast<std::size_t>(A + 1)), rows.data(),
                  next.data()};
    check(pbkv_fmodel_load(c, &m), c);
    const std::size_t n = start.size();
    std::vector<std::int64_t> wf(n);
    for (std::size_t i = 0; i < n; ++i) wf[i] = -1 - static_cast<std::int64_t>(i);  // scratch forecast slots
    std::vector<double> probs(n * static_cast<std::size_t>(K) * (A + 1));
    check(pbkv_forecast_propagate(c, wf.data(), static_cast<std::int64_t>(n), start.data(), K, lambda, probs.data()),
          c);
    std::vector<Forecast> out;
    out.reserve(n);
    const std::size_t per = static_cast<std::size_t>(K) * (A + 1);
    for (std::size_t i = 0; i < n; ++i)
        out.emplace_back(K, A + 1, std::vector<double>(probs.begin() + i * per, probs.begin() + (i + 1) * per));
    return out;
}

inline std::uint64_t encode_context(std::span<const AgentId> ctx) {  // callgraph.hpp:216-220
    std::uint64_t key = 0;
    for (AgentId a : ctx) key = key * 128 + static_cast<std::uint64_t>(a + 1);
    return key;
}

inline std::vector<AgentId> decode_context(std::uint64_t key) {
    std::vector<AgentId> ctx;
    while (key != 0) {
        ctx.push_back(static_cast<AgentId>(key % 128) - 1);
        key /= 128;
    }
    std::reverse(ctx.begin(), ctx.end());
    return ctx;
}

}  // namespace detail

// CallGraph::true_kstep_marginals for a batch of prefixes (callgraph.hpp:136-186),
// then noisy_predict (predictor.hpp:25-35) when lambda >= 0.
inline std::vector<Forecast> oracle_predict_batch(const CallGraph& g, std::span<const std::vector<AgentId>> prefixes,
                                                  int K, double lambda = -1.0) {
    if (K < 1) throw ValidationError("horizon must be >= 1");
    if (lambda >= 0.0 && lambda > 1.0) throw ValidationError("noise level must be in [0, 1]");
    const int A = g.num_agents(), n_ctx = g.context_order();
    auto ctx_of = [&](std::span<const AgentId> p) {
        const std::size_t n = std::min<std::size_t>(p.size(), static_cast<std::size_t>(n_ctx));
        return std::vector<AgentId>(p.end() - n, p.end());
    };
    std::vector<std::uint64_t> seeds;
    for (const auto& p : prefixes) {
        for (std::size_t i = 0; i + 1 < p.size(); ++i)
            if (!g.edges().count({p[i], p[i + 1]})) throw ValidationError("prefix contains a non-edge transition");
        if (!p.empty()) g.row_for_prefix(p);  // must be a known state (throws like the reference)
        seeds.push_back(detail::encode_context(ctx_of(p)));
    }
    detail::StateTable<std::uint64_t> t;
    t.build(
        seeds, A,
        [&](std::uint64_t k) {  // key 0: the entry state (empty context, entry row with END mass 0)
            const std::vector<AgentId> ctx = detail::decode_context(k);
            return g.row_for_prefix(ctx);
        },
        [&](std::uint64_t k, AgentId a) {
            std::vector<AgentId> ns = detail::decode_context(k);
            ns.push_back(a);
            return detail::encode_context(ctx_of(ns));
        });
    std::vector<std::int32_t> start;
    for (std::uint64_t k : seeds) start.push_back(t.index(k));
    return detail::propagate(A, t.rows, t.next, start, K, lambda);
}

// MarkovModel::predict for a batch of prefixes (predictor.hpp:79-118).
inline std::vector<Forecast> markov_predict_batch(const MarkovModel& m, std::span<const std::vector<AgentId>> prefixes,
                                                  int K) {
    if (K < 1) throw ValidationError("horizon must be >= 1");
    const int A = m.num_agents(), order = m.order();
    auto tail = [&](std::span<const AgentId> p) {
        const std::size_t n = std::min<std::size_t>(p.size(), static_cast<std::size_t>(order));
        return std::vector<AgentId>(p.end() - n, p.end());
    };
    std::vector<std::vector<AgentId>> seeds;
    for (const auto& p : prefixes) {
        if (p.empty()) throw ValidationError("markov prediction needs a non-empty prefix");
        seeds.push_back(tail(p));
    }
    detail::StateTable<std::vector<AgentId>> t;
    t.build(
        seeds, A, [&](const std::vector<AgentId>& k) { return m.row_for(k); },
        [&](const std::vector<AgentId>& k, AgentId a) {
            std::vector<AgentId> ns = k;
            ns.push_back(a);
            return tail(ns);
        });
    std::vector<std::int32_t> start;
    for (const auto& k : seeds) start.push_back(t.index(k));
    return detail::propagate(A, t.rows, t.next, start, K, -1.0);
}
#endif  // PBKV_WITH_PREDICTORS

}  // namespace flowkv::gpu
