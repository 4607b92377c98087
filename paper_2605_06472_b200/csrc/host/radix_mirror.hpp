// Host-side radix-tree mirror: the caller-side tree whose read-side fields the
// GPU hot path consumes, kept directly in the SoA shape the device mirror uses.
//
// It follows the mutation semantics of the reference CacheTree
// (/root/reference/proj/include/flowkv/cache.hpp) so that a tree built through
// the same operation stream has identical node ids, parents, lengths, tiers,
// retired bits, last_access clocks, ever_tagged counts and per-node access
// maps:
//   match_prefix            cache.hpp:121-153
//   insert_suffix           cache.hpp:159-219
//   on_workflow_terminated  cache.hpp:224-250
//   demote_to_host          cache.hpp:254-275
//   promote_to_device       cache.hpp:278-291
//   drop_host_node          cache.hpp:294-301
//   set_score               cache.hpp:320-325 (no heap: the GPU selection never
//                           reads one, policies.hpp:60-63)
//   touch / revive / split  cache.hpp:479-569
// The candidate indexes of the reference (lru_leaves_, retired_leaves_,
// host_index_, ScoreHeap) are deliberately absent: every candidate set is
// derived on the device from the SoA fields.
//
// Storage is a vector of compact node records; children are a token-sorted
// vector (same iteration order as the reference's std::map), access entries a
// WorkflowId-sorted vector (same order as std::map<WorkflowId, uint64_t>,
// cache.hpp:64 -- the order Eq. 2 sums in).  Every mutated node id is recorded
// in a dirty list for incremental device sync.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

namespace pbkv {

enum class Tier : std::uint8_t { Device = 0, Host = 1, Absent = 2 };

/// Same role as flowkv::ValidationError (errors.hpp:24-26): the C-ABI maps it
/// to PBKV_EINVAL with the message preserved.
struct ValidationError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

class RadixMirror {
public:
    using TokenId = std::uint64_t;
    using WorkflowId = std::int64_t;

    struct Node {
        int id = 0;
        int parent = -1;
        Tier tier = Tier::Device;
        bool retired = false;
        std::uint64_t last_access = 0;
        double score = 0.0;
        int device_children = 0;
        int ever_tagged = 0;
        std::vector<TokenId> tokens;
        std::vector<std::pair<TokenId, int>> children;            // sorted by token
        std::vector<std::pair<WorkflowId, std::uint64_t>> access;  // sorted by workflow id
        std::int64_t len() const { return static_cast<std::int64_t>(tokens.size()); }
    };

    struct MatchResult {
        std::int64_t device_hit = 0, host_hit = 0, miss = 0;
        std::vector<int> path, host_path;
    };

    RadixMirror(std::int64_t device_capacity, std::int64_t host_capacity)
        : device_capacity_(device_capacity), host_capacity_(host_capacity) {
        if (device_capacity_ <= 0 || host_capacity_ < 0)
            throw ValidationError("cache capacities must be positive");
        nodes_.emplace_back();
        nodes_[0].id = 0;
        mark(0);
    }

    std::int64_t device_capacity() const { return device_capacity_; }
    std::int64_t host_capacity() const { return host_capacity_; }
    std::int64_t device_used() const { return device_used_; }
    std::int64_t host_used() const { return host_used_; }
    std::int64_t device_free() const { return device_capacity_ - device_used_; }
    std::int64_t host_free() const { return host_capacity_ - host_used_; }
    std::int64_t retired_device_tokens() const { return retired_device_tokens_; }
    std::uint64_t clock() const { return clock_; }
    std::size_t node_count() const { return nodes_.size(); }
    const Node& node(int id) const { return nodes_[static_cast<std::size_t>(id)]; }
    std::size_t entry_count() const {
        std::size_t e = 0;
        for (const Node& n : nodes_) e += n.access.size();
        return e;
    }

    const std::vector<int>* touched_nodes(WorkflowId w) const {
        auto it = workflows_.find(w);
        return it == workflows_.end() ? nullptr : &it->second.touched;
    }

    // ---- dirty tracking for incremental device sync --------------------------
    const std::vector<int>& dirty() const { return dirty_list_; }
    void clear_dirty() {
        for (int id : dirty_list_) dirty_flag_[static_cast<std::size_t>(id)] = 0;
        dirty_list_.clear();
    }

    // ---- mutation API (cache.hpp semantics) ----------------------------------

    MatchResult match_prefix(const std::vector<TokenId>& tokens, WorkflowId w, int agent) {
        if (tokens.empty()) throw ValidationError("match_prefix needs a non-empty token sequence");
        register_workflow(w);
        MatchResult r;
        int cur = 0;
        std::size_t i = 0;
        bool seen_host = false;
        while (i < tokens.size()) {
            int cid = child_of(cur, tokens[i]);
            if (cid < 0 || nodes_[cid].tier == Tier::Absent) break;
            std::size_t m = common_prefix(nodes_[cid].tokens, tokens, i);
            if (m < nodes_[cid].tokens.size()) split(cid, m);
            Node& ch = nodes_[cid];
            if (ch.tier == Tier::Device) {
                if (seen_host) throw ValidationError("device node below host node");
                r.device_hit += ch.len();
            } else {
                seen_host = true;
                r.host_hit += ch.len();
                r.host_path.push_back(cid);
            }
            touch(cid, w, agent);
            r.path.push_back(cid);
            i += m;
            cur = cid;
        }
        r.miss = static_cast<std::int64_t>(tokens.size() - i);
        return r;
    }

    /// Returns the deepest path node (InsertReport::leaf, cache.hpp:40).
    int insert_suffix(const std::vector<TokenId>& tokens, WorkflowId w, int agent,
                      std::int64_t budget = -1, std::int64_t* cached_out = nullptr) {
        if (tokens.empty()) throw ValidationError("insert_suffix needs a non-empty token sequence");
        register_workflow(w);
        if (budget < 0) {
            std::int64_t needed = probe_missing(tokens);
            if (needed > device_free())
                throw ValidationError("insert_suffix without room: caller must evict first");
            budget = needed;
        } else {
            budget = std::min(budget, device_free());
        }
        std::int64_t cached = 0;
        int cur = 0;
        std::size_t i = 0;
        bool on_device_path = true;
        while (i < tokens.size()) {
            int cid = child_of(cur, tokens[i]);
            if (cid < 0) break;
            std::size_t m = common_prefix(nodes_[cid].tokens, tokens, i);
            if (m < nodes_[cid].tokens.size()) split(cid, m);
            if (nodes_[cid].tier == Tier::Absent) {
                if (!on_device_path) break;
                if (budget < nodes_[cid].len()) {
                    if (budget > 0) {
                        split(cid, static_cast<std::size_t>(budget));
                        revive(cid, w, agent);
                        cached += budget;
                        budget = 0;
                        cur = cid;
                    }
                    if (cached_out) *cached_out = cached;
                    return cur;
                }
                budget -= nodes_[cid].len();
                cached += nodes_[cid].len();
                revive(cid, w, agent);
            } else {
                if (nodes_[cid].tier == Tier::Host) on_device_path = false;
                touch(cid, w, agent);
            }
            i += m;
            cur = cid;
        }
        if (i < tokens.size() && budget > 0 && on_device_path) {
            std::size_t take = std::min<std::size_t>(tokens.size() - i, static_cast<std::size_t>(budget));
            int nid = make_node(cur, std::vector<TokenId>(tokens.begin() + static_cast<std::ptrdiff_t>(i),
                                                          tokens.begin() + static_cast<std::ptrdiff_t>(i + take)),
                                Tier::Device);
            device_used_ += nodes_[nid].len();
            touch(nid, w, agent);
            cached += nodes_[nid].len();
            cur = nid;
        }
        if (cached_out) *cached_out = cached;
        return cur;
    }

    std::vector<int> on_workflow_terminated(WorkflowId w, int* newly_retired = nullptr) {
        if (newly_retired) *newly_retired = 0;
        auto it = workflows_.find(w);
        if (it == workflows_.end() || it->second.terminated) {
            ++unknown_workflow_warnings_;
            return {};
        }
        it->second.terminated = true;
        std::vector<int> affected = std::move(it->second.touched);
        it->second.touched.clear();
        int count = 0;
        for (int id : affected) {
            Node& n = nodes_[id];
            auto a = find_access(n, w);
            if (a == n.access.end() || a->first != w) continue;
            n.access.erase(a);
            mark(id);
            if (n.access.empty() && !n.retired) {
                n.retired = true;
                if (n.tier == Tier::Device) retired_device_tokens_ += n.len();
                ++count;
            }
        }
        if (newly_retired) *newly_retired = count;
        return affected;
    }

    Tier demote_to_host(int id) {
        check_id(id);
        Node& n = nodes_[id];
        if (id == 0 || n.tier != Tier::Device) throw ValidationError("demote needs a device node");
        if (n.device_children > 0) throw ValidationError("demote of an interior node with device descendants");
        device_used_ -= n.len();
        if (n.retired) retired_device_tokens_ -= n.len();
        Tier target;
        if (host_free() >= n.len()) {
            n.tier = Tier::Host;
            host_used_ += n.len();
            target = Tier::Host;
        } else {
            n.tier = Tier::Absent;
            drop_host_subtree(id);
            target = Tier::Absent;
        }
        mark(id);
        adjust_parent_device_children(id, -1);
        return target;
    }

    void promote_to_device(int id) {
        check_id(id);
        Node& n = nodes_[id];
        if (n.tier != Tier::Host) throw ValidationError("promote needs a host node");
        if (nodes_[n.parent].tier != Tier::Device) throw ValidationError("promote needs a device-resident parent");
        if (device_free() < n.len()) throw ValidationError("promote without device room");
        host_used_ -= n.len();
        n.tier = Tier::Device;
        device_used_ += n.len();
        if (n.retired) retired_device_tokens_ += n.len();
        mark(id);
        adjust_parent_device_children(id, +1);
    }

    void drop_host_node(int id) {
        check_id(id);
        Node& n = nodes_[id];
        if (n.tier != Tier::Host) throw ValidationError("drop needs a host node");
        host_used_ -= n.len();
        n.tier = Tier::Absent;
        mark(id);
        drop_host_subtree(id);
    }

    void set_score(int id, double score) {
        check_id(id);
        Node& n = nodes_[id];
        if (n.score == score) return;
        n.score = score;
        mark(id);
    }

    // ---- SoA export ----------------------------------------------------------
    // Layout matches pbkv_tree_soa (include/pbkv.h).
    void export_soa(std::int32_t* parent, std::int32_t* len, std::uint8_t* tier, std::uint8_t* retired,
                    std::uint64_t* last_access, std::int32_t* ever_tagged, double* score,
                    std::int32_t* device_children, std::int32_t* depth, std::int64_t* acc_off,
                    std::int64_t* acc_wf, std::uint64_t* acc_bits) const {
        std::int64_t e = 0;
        for (std::size_t i = 0; i < nodes_.size(); ++i) {
            const Node& n = nodes_[i];
            if (parent) parent[i] = n.parent;
            if (len) len[i] = static_cast<std::int32_t>(n.tokens.size());
            if (tier) tier[i] = static_cast<std::uint8_t>(n.tier);
            if (retired) retired[i] = n.retired ? 1 : 0;
            if (last_access) last_access[i] = n.last_access;
            if (ever_tagged) ever_tagged[i] = n.ever_tagged;
            if (score) score[i] = n.score;
            if (device_children) device_children[i] = n.device_children;
            if (acc_off) acc_off[i] = e;
            for (const auto& [w, bits] : n.access) {
                if (acc_wf) acc_wf[e] = w;
                if (acc_bits) acc_bits[e] = bits;
                ++e;
            }
        }
        if (acc_off) acc_off[nodes_.size()] = e;
        if (depth) compute_depth(depth);
    }

    void compute_depth(std::int32_t* depth) const {
        // parents can have larger ids than children after a split
        // (cache.hpp:531-569), so resolve depths by memoised walks.
        const std::size_t n = nodes_.size();
        for (std::size_t i = 0; i < n; ++i) depth[i] = -1;
        depth[0] = 0;
        std::vector<int> stack;
        for (std::size_t i = 1; i < n; ++i) {
            int v = static_cast<int>(i);
            while (depth[v] < 0) {
                stack.push_back(v);
                v = nodes_[v].parent;
            }
            int d = depth[v];
            while (!stack.empty()) {
                depth[stack.back()] = ++d;
                stack.pop_back();
            }
        }
    }

private:
    struct WorkflowEntry {
        bool terminated = false;
        std::vector<int> touched;
    };

    std::vector<Node> nodes_;
    std::int64_t device_capacity_, host_capacity_;
    std::int64_t device_used_ = 0, host_used_ = 0, retired_device_tokens_ = 0;
    std::int64_t unknown_workflow_warnings_ = 0;
    std::uint64_t clock_ = 0;
    std::unordered_map<WorkflowId, WorkflowEntry> workflows_;
    std::vector<std::uint8_t> dirty_flag_;
    std::vector<int> dirty_list_;

    void mark(int id) {
        std::size_t u = static_cast<std::size_t>(id);
        if (u >= dirty_flag_.size()) dirty_flag_.resize(std::max<std::size_t>(u + 1, dirty_flag_.size() * 2), 0);
        if (!dirty_flag_[u]) {
            dirty_flag_[u] = 1;
            dirty_list_.push_back(id);
        }
    }

    void check_id(int id) const {
        if (id < 0 || static_cast<std::size_t>(id) >= nodes_.size()) throw ValidationError("node id out of range");
    }

    static std::size_t common_prefix(const std::vector<TokenId>& seg, const std::vector<TokenId>& q,
                                     std::size_t off) {
        std::size_t n = std::min(seg.size(), q.size() - off);
        std::size_t i = 0;
        while (i < n && seg[i] == q[off + i]) ++i;
        return i;
    }

    int child_of(int id, TokenId tok) const {
        const auto& ch = nodes_[id].children;
        auto it = std::lower_bound(ch.begin(), ch.end(), tok,
                                   [](const std::pair<TokenId, int>& p, TokenId t) { return p.first < t; });
        return (it != ch.end() && it->first == tok) ? it->second : -1;
    }

    void set_child(int id, TokenId tok, int cid) {
        auto& ch = nodes_[id].children;
        auto it = std::lower_bound(ch.begin(), ch.end(), tok,
                                   [](const std::pair<TokenId, int>& p, TokenId t) { return p.first < t; });
        if (it != ch.end() && it->first == tok)
            it->second = cid;
        else
            ch.insert(it, {tok, cid});
    }

    static std::vector<std::pair<WorkflowId, std::uint64_t>>::iterator find_access(Node& n, WorkflowId w) {
        return std::lower_bound(n.access.begin(), n.access.end(), w,
                                [](const std::pair<WorkflowId, std::uint64_t>& p, WorkflowId x) {
                                    return p.first < x;
                                });
    }

    void register_workflow(WorkflowId w) {
        auto& e = workflows_[w];
        if (e.terminated) throw ValidationError("terminated workflow touched the cache again");
    }

    void touch(int id, WorkflowId w, int agent) {
        Node& n = nodes_[id];
        auto it = find_access(n, w);
        if (it == n.access.end() || it->first != w) {
            it = n.access.insert(it, {w, 0});
            ++n.ever_tagged;
            workflows_.at(w).touched.push_back(id);
        }
        it->second |= 1ULL << agent;
        if (n.retired) {
            n.retired = false;
            if (n.tier == Tier::Device) retired_device_tokens_ -= n.len();
        }
        n.last_access = ++clock_;
        mark(id);
    }

    void revive(int id, WorkflowId w, int agent) {
        Node& n = nodes_[id];
        n.tier = Tier::Device;
        device_used_ += n.len();
        if (n.retired) retired_device_tokens_ += n.len();
        adjust_parent_device_children(id, +1);
        touch(id, w, agent);
    }

    int make_node(int parent, std::vector<TokenId> tokens, Tier tier) {
        int id = static_cast<int>(nodes_.size());
        nodes_.emplace_back();
        Node& n = nodes_.back();
        n.id = id;
        n.parent = parent;
        n.tokens = std::move(tokens);
        n.tier = tier;
        set_child(parent, nodes_[id].tokens[0], id);
        mark(id);
        if (tier == Tier::Device) adjust_parent_device_children(id, +1);
        return id;
    }

    void adjust_parent_device_children(int id, int delta) {
        int pid = nodes_[id].parent;
        nodes_[pid].device_children += delta;
        mark(pid);
    }

    void split(int id, std::size_t offset) {
        if (offset == 0 || offset >= nodes_[id].tokens.size()) throw ValidationError("split offset out of range");
        int low_id = static_cast<int>(nodes_.size());
        nodes_.emplace_back();
        Node& up = nodes_[id];
        Node& low = nodes_.back();
        low.id = low_id;
        low.parent = id;
        low.tokens.assign(up.tokens.begin() + static_cast<std::ptrdiff_t>(offset), up.tokens.end());
        low.tier = up.tier;
        low.retired = up.retired;
        low.last_access = up.last_access;
        low.score = up.score;
        low.children = std::move(up.children);
        low.device_children = up.device_children;
        low.access = up.access;
        low.ever_tagged = up.ever_tagged;
        for (const auto& [tok, cid] : low.children) {
            (void)tok;
            nodes_[cid].parent = low_id;
            mark(cid);
        }
        up.tokens.resize(offset);
        up.children.clear();
        up.children.push_back({low.tokens[0], low_id});
        up.device_children = low.tier == Tier::Device ? 1 : 0;
        for (const auto& [w, bits] : low.access) {
            (void)bits;
            workflows_.at(w).touched.push_back(low_id);
        }
        mark(id);
        mark(low_id);
    }

    void drop_host_subtree(int id) {
        for (const auto& [tok, cid] : nodes_[id].children) {
            (void)tok;
            Node& c = nodes_[cid];
            if (c.tier == Tier::Device) throw ValidationError("device node stranded below a dropped node");
            if (c.tier == Tier::Host) {
                host_used_ -= c.len();
                c.tier = Tier::Absent;
                mark(cid);
                drop_host_subtree(cid);
            }
        }
    }

    std::int64_t probe_missing(const std::vector<TokenId>& tokens) const {
        int cur = 0;
        std::size_t i = 0;
        std::int64_t missing = 0;
        bool on_device_path = true;
        while (i < tokens.size()) {
            int cid = child_of(cur, tokens[i]);
            if (cid < 0) break;
            const Node& ch = nodes_[cid];
            std::size_t m = common_prefix(ch.tokens, tokens, i);
            if (ch.tier == Tier::Absent) {
                if (!on_device_path) return missing;
                missing += static_cast<std::int64_t>(m);
            } else if (ch.tier == Tier::Host) {
                on_device_path = false;
            }
            i += m;
            if (m < ch.tokens.size()) break;
            cur = cid;
        }
        if (on_device_path) missing += static_cast<std::int64_t>(tokens.size() - i);
        return missing;
    }
};

}  // namespace pbkv
