// tracked_tree.hpp -- the reference flowkv::CacheTree with a change log, and
// the pbkv mirror images built from it (full snapshot / incremental delta).
//
// CacheTree (cache.hpp:52-612) has no change log: every mutation is private
// bookkeeping behind a handful of public members.  TrackedCacheTree derives
// from it and shadows exactly those public mutators -- calling the reference
// implementation, then logging the ids of every node whose mirrored fields
// (cache.hpp:54-69: parent, tokens.size(), tier, retired, last_access,
// score, access, ever_tagged) may have changed:
//
//   match_prefix            cache.hpp:121-153   the matched path + split halves
//   insert_suffix           cache.hpp:159-219   the path root..leaf + split halves
//   on_workflow_terminated  cache.hpp:224-250   the workflow's touched list
//   demote_to_host          cache.hpp:254-275   the node (+ its subtree when dropped)
//   promote_to_device       cache.hpp:278-291   the node
//   drop_host_node          cache.hpp:294-301   the node + its subtree
//   make_room_on_host       cache.hpp:305-318   every dropped node + subtree
//   set_score               cache.hpp:320-325   the node
//
// split() (cache.hpp:531-569) creates the lower half as a NEW node (id =
// node_count) that adopts the old children: every new node is logged with its
// parent, and a new node that has children had a subtree moved one level
// down -- the subtree is re-levelled and logged.  The class also keeps each
// node's depth (root = 0), which the device selection uses for chain
// distances.  Derived-to-base binding keeps every `const CacheTree&` reader
// (policies.hpp, scoring.hpp) unchanged; an unmodified simulator.hpp holds one
// through `#define CacheTree TrackedCacheTree`.
//
// A reference mutator that throws part-way leaves an unknown set of nodes
// changed: the log is then invalidated, so every consumer re-mirrors fully.
//
// Consumers (pbkv contexts) remember (uid, position) of the log they have
// applied.  changes_since(pos) returns the distinct ids logged after pos, or
// false when the log no longer reaches back (it is bounded: past
// max(2^16, 4 * node_count) entries it is dropped and consumers re-mirror).
#pragma once

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <set>
#include <span>
#include <unordered_map>
#include <vector>

#include "flowkv/cache.hpp"

#include "../pbkv.h"

namespace flowkv::gpu {

class TrackedCacheTree;

namespace detail {
// base-object address -> tracked tree: lets the drop-in (flowkv_gpu.hpp),
// which receives `const CacheTree&`, find the change log of a tracked tree
struct TrackedRegistry {
    std::mutex mu;
    std::unordered_map<const CacheTree*, const TrackedCacheTree*> map;
};
inline TrackedRegistry& tracked_registry() {
    static TrackedRegistry r;
    return r;
}
}  // namespace detail

class TrackedCacheTree : public CacheTree {
public:
    TrackedCacheTree(std::int64_t device_capacity, std::int64_t host_capacity)
        : CacheTree(device_capacity, host_capacity), uid_(next_uid()), depth_(1, 0) {
        enroll();
    }
    TrackedCacheTree(const TrackedCacheTree& o)
        : CacheTree(o), uid_(next_uid()), depth_(o.depth_), base_(0), log_() {
        enroll();
    }
    TrackedCacheTree& operator=(const TrackedCacheTree& o) {
        if (this != &o) {
            CacheTree::operator=(o);
            depth_ = o.depth_;
            invalidate();
            uid_ = next_uid();
        }
        return *this;
    }
    ~TrackedCacheTree() {
        auto& r = detail::tracked_registry();
        std::lock_guard<std::mutex> g(r.mu);
        r.map.erase(static_cast<const CacheTree*>(this));
    }

    /// Identity of this tree's log (unique per instance and per assignment).
    std::uint64_t uid() const { return uid_; }
    int depth(int id) const { return depth_[static_cast<std::size_t>(id)]; }
    const std::vector<int>& depths() const { return depth_; }

    /// End position of the change log.
    std::int64_t log_end() const { return base_ + static_cast<std::int64_t>(log_.size()); }

    /// Distinct ids logged after `pos`, ascending; false when the log has
    /// been truncated past `pos` (the consumer must re-mirror in full).
    bool changes_since(std::int64_t pos, std::vector<int>& out) const {
        out.clear();
        if (pos < base_ || pos > log_end()) return false;
        if (seen_.size() < node_count()) seen_.resize(node_count(), 0);
        if (++stamp_ == 0) {
            std::fill(seen_.begin(), seen_.end(), 0u);
            stamp_ = 1;
        }
        for (std::size_t i = static_cast<std::size_t>(pos - base_); i < log_.size(); ++i) {
            const int id = log_[i];
            if (seen_[static_cast<std::size_t>(id)] == stamp_) continue;
            seen_[static_cast<std::size_t>(id)] = stamp_;
            out.push_back(id);
        }
        std::sort(out.begin(), out.end());
        return true;
    }

    // ---- shadowed mutators (cache.hpp semantics, then the log) ---------------
    MatchResult match_prefix(std::span<const TokenId> tokens, WorkflowId w, int agent) {
        const std::size_t n0 = node_count();
        try {
            MatchResult r = CacheTree::match_prefix(tokens, w, agent);
            for (int id : r.path) log(id);
            after(n0);
            return r;
        } catch (...) {
            failed(n0);
            throw;
        }
    }

    InsertReport insert_suffix(std::span<const TokenId> tokens, WorkflowId w, int agent, std::int64_t budget = -1) {
        const std::size_t n0 = node_count();
        try {
            InsertReport r = CacheTree::insert_suffix(tokens, w, agent, budget);
            // touched / revived nodes are exactly the path root..leaf
            for (int v = r.leaf; v > 0; v = node(v).parent) log(v);
            after(n0);
            return r;
        } catch (...) {
            failed(n0);
            throw;
        }
    }

    std::vector<int> on_workflow_terminated(WorkflowId w, int* newly_retired = nullptr) {
        const std::size_t n0 = node_count();
        try {
            std::vector<int> affected = CacheTree::on_workflow_terminated(w, newly_retired);
            for (int id : affected) log(id);
            return affected;
        } catch (...) {
            failed(n0);
            throw;
        }
    }

    Tier demote_to_host(int id) {
        const std::size_t n0 = node_count();
        try {
            const Tier t = CacheTree::demote_to_host(id);
            log(id);
            if (t == Tier::Absent) log_subtree(id);  // drop_host_subtree (cache.hpp:571-585)
            return t;
        } catch (...) {
            failed(n0);
            throw;
        }
    }

    void promote_to_device(int id) {
        const std::size_t n0 = node_count();
        try {
            CacheTree::promote_to_device(id);
            log(id);
        } catch (...) {
            failed(n0);
            throw;
        }
    }

    void drop_host_node(int id) {
        const std::size_t n0 = node_count();
        try {
            CacheTree::drop_host_node(id);
            log_subtree(id);
        } catch (...) {
            failed(n0);
            throw;
        }
    }

    std::vector<int> make_room_on_host(std::int64_t need, const std::set<int>& keep = {}) {
        const std::size_t n0 = node_count();
        try {
            std::vector<int> dropped = CacheTree::make_room_on_host(need, keep);
            for (int id : dropped) log_subtree(id);
            return dropped;
        } catch (...) {
            failed(n0);
            throw;
        }
    }

    void set_score(int id, double score) {
        CacheTree::set_score(id, score);
        log(id);
    }

    /// Drops the log: every consumer re-mirrors in full at its next sync.
    void invalidate() {
        base_ = log_end() + 1;
        log_.clear();
    }

private:
    static std::uint64_t next_uid() {
        static std::atomic<std::uint64_t> ctr{0};
        return ++ctr;
    }

    void enroll() {
        auto& r = detail::tracked_registry();
        std::lock_guard<std::mutex> g(r.mu);
        r.map[static_cast<const CacheTree*>(this)] = this;
    }

    void log(int id) {
        log_.push_back(id);
        const std::size_t cap = std::max<std::size_t>(std::size_t(1) << 16, 4 * node_count());
        if (log_.size() > cap) invalidate();
    }

    // every node below `id` (children maps), logged; depths re-levelled
    void log_subtree(int id) {
        std::vector<int> stack{id};
        while (!stack.empty()) {
            const int v = stack.back();
            stack.pop_back();
            log(v);
            if (v != id) depth_[static_cast<std::size_t>(v)] = depth_[static_cast<std::size_t>(node(v).parent)] + 1;
            for (const auto& [tok, c] : node(v).children) {
                (void)tok;
                stack.push_back(c);
            }
        }
    }

    // new nodes [n0, node_count()): depth, the node and its parent (a split
    // shortened the parent); a new node with children is a split's lower half
    // that adopted a subtree one level deeper
    void after(std::size_t n0) {
        const std::size_t n1 = node_count();
        depth_.resize(n1, 0);
        for (std::size_t x = n0; x < n1; ++x) {
            const int p = node(static_cast<int>(x)).parent;
            depth_[x] = depth_[static_cast<std::size_t>(p)] + 1;
            log(p);
            if (node(static_cast<int>(x)).children.empty())
                log(static_cast<int>(x));
            else
                log_subtree(static_cast<int>(x));
        }
    }

    void failed(std::size_t n0) {
        after(n0);
        invalidate();
    }

    std::uint64_t uid_;
    std::vector<int> depth_;
    std::int64_t base_ = 0;
    std::vector<int> log_;
    mutable std::vector<std::uint32_t> seen_;
    mutable std::uint32_t stamp_ = 0;
};

/// The tracked tree behind `t`, if `t` is one.
inline const TrackedCacheTree* tracked(const CacheTree& t) {
    auto& r = detail::tracked_registry();
    std::lock_guard<std::mutex> g(r.mu);
    auto it = r.map.find(&t);
    return it == r.map.end() ? nullptr : it->second;
}

inline std::uint8_t tier_code(Tier t) {
    return t == Tier::Device ? PBKV_TIER_DEVICE : (t == Tier::Host ? PBKV_TIER_HOST : PBKV_TIER_ABSENT);
}

inline pbkv_tree_totals totals_of(const CacheTree& t) {
    return pbkv_tree_totals{t.device_capacity(), t.device_used(), t.retired_device_tokens(), t.host_capacity(),
                            t.host_used()};
}

/// Struct-of-arrays image of a whole CacheTree (read-side fields,
/// cache.hpp:54-69) for pbkv_mirror_full / pbkv_mirror_verify.  `depths`
/// (optional) is a TrackedCacheTree's depth table; without it the device
/// context derives depths from the parents.
struct TreeImage {
    std::vector<std::int32_t> parent, len, ever, dc, depth;
    std::vector<std::uint8_t> tier, retired;
    std::vector<std::uint64_t> last, bits;
    std::vector<double> score;
    std::vector<std::int64_t> off, wf;
    pbkv_tree_soa soa{};

    void build(const CacheTree& t, const std::vector<int>* depths = nullptr) {
        const std::size_t n = t.node_count();
        parent.resize(n);
        len.resize(n);
        ever.resize(n);
        dc.resize(n);
        tier.resize(n);
        retired.resize(n);
        last.resize(n);
        score.resize(n);
        off.resize(n + 1);
        wf.clear();
        bits.clear();
        for (std::size_t i = 0; i < n; ++i) {
            const CacheTree::Node& nd = t.node(static_cast<int>(i));
            parent[i] = nd.parent;
            len[i] = static_cast<std::int32_t>(nd.tokens.size());
            ever[i] = nd.ever_tagged;
            dc[i] = nd.device_children;
            tier[i] = tier_code(nd.tier);
            retired[i] = nd.retired ? 1 : 0;
            last[i] = nd.last_access;
            score[i] = nd.score;
            off[i] = static_cast<std::int64_t>(wf.size());
            for (const auto& [w, b] : nd.access) {  // std::map: ascending WorkflowId (cache.hpp:64)
                wf.push_back(static_cast<std::int64_t>(w));
                bits.push_back(b);
            }
        }
        off[n] = static_cast<std::int64_t>(wf.size());
        if (depths) depth.assign(depths->begin(), depths->begin() + static_cast<std::ptrdiff_t>(n));
        soa = pbkv_tree_soa{};
        soa.n_nodes = static_cast<std::int64_t>(n);
        soa.n_entries = static_cast<std::int64_t>(wf.size());
        soa.parent = parent.data();
        soa.len = len.data();
        soa.tier = tier.data();
        soa.retired = retired.data();
        soa.last_access = last.data();
        soa.ever_tagged = ever.data();
        soa.score = score.data();
        soa.device_children = dc.data();
        soa.depth = depths ? depth.data() : nullptr;
        soa.acc_off = off.data();
        soa.acc_wf = wf.data();
        soa.acc_bits = bits.data();
        const pbkv_tree_totals tt = totals_of(t);
        soa.device_capacity = tt.device_capacity;
        soa.device_used = tt.device_used;
        soa.retired_device_tokens = tt.retired_device_tokens;
        soa.host_capacity = tt.host_capacity;
        soa.host_used = tt.host_used;
    }
};

/// The pbkv_mirror_delta batch of a set of node ids: each node's current
/// fields and access entries.
struct DeltaBatch {
    std::vector<pbkv_node_delta> nodes;
    std::vector<std::int64_t> wf;
    std::vector<std::uint64_t> bits;
    pbkv_tree_totals totals{};

    void build(const TrackedCacheTree& t, std::span<const int> ids) {
        nodes.resize(ids.size());
        wf.clear();
        bits.clear();
        for (std::size_t k = 0; k < ids.size(); ++k) {
            if (k + kAhead < ids.size()) {  // scattered nodes: their lines (a Node spans three) in flight early
                const char* q = reinterpret_cast<const char*>(&t.node(ids[k + kAhead]));
                __builtin_prefetch(q);
                __builtin_prefetch(q + 64);
                __builtin_prefetch(q + 128);
                __builtin_prefetch(&t.depths()[static_cast<std::size_t>(ids[k + kAhead])]);
            }
            if (k + kAhead / 2 < ids.size()) {  // the first entry of the access map, once its header is cached
                const auto& acc = t.node(ids[k + kAhead / 2]).access;
                if (!acc.empty()) __builtin_prefetch(&*acc.begin());
            }
            const CacheTree::Node& nd = t.node(ids[k]);
            pbkv_node_delta& r = nodes[k];
            std::memset(&r, 0, sizeof r);
            r.id = ids[k];
            r.parent = nd.parent;
            r.len = static_cast<std::int32_t>(nd.tokens.size());
            r.ever_tagged = nd.ever_tagged;
            r.depth = t.depth(ids[k]);
            r.tier = tier_code(nd.tier);
            r.retired = nd.retired ? 1 : 0;
            r.last_access = nd.last_access;
            r.score = nd.score;
            r.acc_begin = static_cast<std::int64_t>(wf.size());
            for (const auto& [w, b] : nd.access) {
                wf.push_back(static_cast<std::int64_t>(w));
                bits.push_back(b);
            }
            r.acc_end = static_cast<std::int64_t>(wf.size());
        }
        totals = totals_of(t);
    }
    static constexpr std::size_t kAhead = 16;
};

/// Brings the context's mirror of `t` up to date.  (uid, pos) is the
/// consumer state the caller keeps per context: a delta when it matches this
/// tree and the log reaches back to pos, else a full upload.  Returns the
/// pbkv status and sets *full_upload accordingly.
inline int sync_mirror(pbkv_ctx* c, const TrackedCacheTree& t, std::uint64_t& uid, std::int64_t& pos,
                       std::vector<int>& ids, DeltaBatch& batch, TreeImage& img, bool* full_upload = nullptr) {
    if (uid == t.uid()) {
        static const bool prof = std::getenv("PBKV_PROFILE_SYNC") != nullptr;
        const auto t0 = std::chrono::steady_clock::now();
        if (t.changes_since(pos, ids)) {
            if (full_upload) *full_upload = false;
            const auto t1 = std::chrono::steady_clock::now();
            batch.build(t, ids);
            const auto t2 = std::chrono::steady_clock::now();
            const int rc = pbkv_mirror_delta(c, batch.nodes.data(), static_cast<std::int64_t>(batch.nodes.size()),
                                             batch.wf.data(), batch.bits.data(), &batch.totals);
            const auto t3 = std::chrono::steady_clock::now();
            if (prof) {
                auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
                std::fprintf(stderr, "[pbkv sync] ids=%zu entries=%zu log=%.1fus batch=%.1fus delta=%.1fus\n",
                             ids.size(), batch.wf.size(), us(t0, t1), us(t1, t2), us(t2, t3));
            }
            if (rc == PBKV_OK) pos = t.log_end();
            return rc;
        }
    }
    if (full_upload) *full_upload = true;
    img.build(t, &t.depths());
    const int rc = pbkv_mirror_full(c, &img.soa);
    if (rc == PBKV_OK) {
        uid = t.uid();
        pos = t.log_end();
    } else {
        uid = 0;
    }
    return rc;
}

}  // namespace flowkv::gpu

namespace flowkv {
// `#define CacheTree TrackedCacheTree` around an unmodified simulator.hpp
// resolves inside namespace flowkv
using gpu::TrackedCacheTree;
}  // namespace flowkv
