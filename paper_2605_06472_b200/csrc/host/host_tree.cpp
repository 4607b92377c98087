// Host trees of the C ABI (include/pbkv.h "host trees"): the reference
// flowkv::CacheTree itself (cache.hpp, compiled from the reference headers),
// wrapped in TrackedCacheTree for incremental device sync
// (include/pbkv/tracked_tree.hpp).  Used by the tests, the bench and Python
// callers; C++ callers use TrackedCacheTree directly.
#include <cstring>
#include <string>
#include <vector>

#include "internal_abi.h"
#include "ops.hpp"
#include "pbkv/tracked_tree.hpp"

struct pbkv_tree {
    flowkv::gpu::TrackedCacheTree tree;
    std::string err;
    // scratch of pbkv_mirror_sync
    std::vector<int> ids;
    flowkv::gpu::DeltaBatch batch;
    flowkv::gpu::TreeImage img;
    pbkv_tree(std::int64_t d, std::int64_t h) : tree(d, h) {}
};

namespace {

struct TreeError {
    int status;
    std::string msg;
};

template <class F>
int tree_api(pbkv_tree* t, F&& f) {
    std::string msg;
    int rc = PBKV_OK;
    try {
        if (!t) throw TreeError{PBKV_EARG, "null tree"};
        f();
        return PBKV_OK;
    } catch (const TreeError& e) {
        rc = e.status;
        msg = e.msg;
    } catch (const flowkv::ValidationError& e) {
        rc = PBKV_EINVAL;
        msg = e.what();
    } catch (const pbkv::OpStreamError& e) {
        rc = PBKV_EARG;
        msg = e.what();
    } catch (const std::bad_alloc&) {
        rc = PBKV_ENOMEM;
        msg = "host allocation failed";
    } catch (const std::exception& e) {
        rc = PBKV_EARG;
        msg = e.what();
    }
    if (t) t->err = msg;
    pbkv_internal_set_error(msg.c_str());
    return rc;
}

void need(bool ok, const char* what) {
    if (!ok) throw TreeError{PBKV_EARG, what};
}

}  // namespace

extern "C" {

int pbkv_tree_create(pbkv_tree** out, int64_t device_capacity, int64_t host_capacity) {
    if (!out) {
        pbkv_internal_set_error("null out");
        return PBKV_EARG;
    }
    try {
        *out = new pbkv_tree(device_capacity, host_capacity);
        return PBKV_OK;
    } catch (const flowkv::ValidationError& e) {
        pbkv_internal_set_error(e.what());
        return PBKV_EINVAL;
    } catch (const std::exception& e) {
        pbkv_internal_set_error(e.what());
        return PBKV_ENOMEM;
    }
}

int pbkv_tree_destroy(pbkv_tree* t) {
    delete t;
    return PBKV_OK;
}

int pbkv_tree_apply_ops(pbkv_tree* t, const int64_t* words, int64_t n_words) {
    return tree_api(t, [&] {
        need(n_words == 0 || words, "null words");
        pbkv::apply_ops(t->tree, words, n_words);
    });
}

int pbkv_tree_synth(pbkv_tree* t, const pbkv_synth_params* p) {
    return tree_api(t, [&] {
        need(p != nullptr, "null params");
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
        pbkv::synth_build(t->tree, sp);
    });
}

int pbkv_tree_shape(pbkv_tree* t, pbkv_tree_soa* s) {
    return tree_api(t, [&] {
        need(s != nullptr, "null soa");
        const auto& tr = t->tree;
        std::int64_t e = 0;
        for (std::size_t i = 0; i < tr.node_count(); ++i) e += static_cast<std::int64_t>(tr.node(static_cast<int>(i)).access.size());
        s->n_nodes = static_cast<std::int64_t>(tr.node_count());
        s->n_entries = e;
        const pbkv_tree_totals tt = flowkv::gpu::totals_of(tr);
        s->device_capacity = tt.device_capacity;
        s->device_used = tt.device_used;
        s->retired_device_tokens = tt.retired_device_tokens;
        s->host_capacity = tt.host_capacity;
        s->host_used = tt.host_used;
    });
}

int pbkv_tree_export(pbkv_tree* t, pbkv_tree_soa* s) {
    return tree_api(t, [&] {
        need(s != nullptr, "null soa");
        const auto& tr = t->tree;
        const std::size_t n = tr.node_count();
        std::int64_t e = 0;
        if (s->acc_off) s->acc_off[0] = 0;
        for (std::size_t i = 0; i < n; ++i) {
            const auto& nd = tr.node(static_cast<int>(i));
            if (s->parent) s->parent[i] = nd.parent;
            if (s->len) s->len[i] = static_cast<std::int32_t>(nd.tokens.size());
            if (s->tier) s->tier[i] = flowkv::gpu::tier_code(nd.tier);
            if (s->retired) s->retired[i] = nd.retired ? 1 : 0;
            if (s->last_access) s->last_access[i] = nd.last_access;
            if (s->ever_tagged) s->ever_tagged[i] = nd.ever_tagged;
            if (s->score) s->score[i] = nd.score;
            if (s->device_children) s->device_children[i] = nd.device_children;
            if (s->depth) s->depth[i] = tr.depth(static_cast<int>(i));
            for (const auto& [w, b] : nd.access) {
                if (s->acc_wf) s->acc_wf[e] = static_cast<std::int64_t>(w);
                if (s->acc_bits) s->acc_bits[e] = b;
                ++e;
            }
            if (s->acc_off) s->acc_off[i + 1] = e;
        }
    });
}

int pbkv_tree_touched(pbkv_tree* t, int64_t wf, int32_t* ids, int64_t cap, int64_t* n) {
    return tree_api(t, [&] {
        need(n != nullptr, "null out");
        const std::vector<int>* v = t->tree.touched_nodes(wf);
        *n = v ? static_cast<int64_t>(v->size()) : 0;
        if (v && ids)
            for (std::size_t i = 0; i < v->size() && static_cast<int64_t>(i) < cap; ++i) ids[i] = (*v)[i];
    });
}

int pbkv_tree_log(pbkv_tree* t, int64_t pos, int64_t* end, int32_t* ids, int64_t cap, int64_t* n_changed) {
    return tree_api(t, [&] {
        need(end && n_changed, "null out");
        *end = t->tree.log_end();
        if (!t->tree.changes_since(pos, t->ids)) {
            *n_changed = -1;
            return;
        }
        *n_changed = static_cast<int64_t>(t->ids.size());
        if (ids)
            for (std::size_t i = 0; i < t->ids.size() && static_cast<int64_t>(i) < cap; ++i) ids[i] = t->ids[i];
    });
}

int pbkv_mirror_tree(pbkv_ctx* c, pbkv_tree* t) {
    return tree_api(t, [&] {
        need(c != nullptr, "null ctx");
        uint64_t* uid = nullptr;
        int64_t* pos = nullptr;
        need(pbkv_internal_mirror_tag(c, &uid, &pos) == PBKV_OK, "null ctx");
        *uid = 0;  // forces the full upload
        const int rc = flowkv::gpu::sync_mirror(c, t->tree, *uid, *pos, t->ids, t->batch, t->img);
        if (rc != PBKV_OK) throw TreeError{rc, pbkv_last_error(c)};
    });
}

int pbkv_mirror_sync(pbkv_ctx* c, pbkv_tree* t) {
    return tree_api(t, [&] {
        need(c != nullptr, "null ctx");
        uint64_t* uid = nullptr;
        int64_t* pos = nullptr;
        need(pbkv_internal_mirror_tag(c, &uid, &pos) == PBKV_OK, "null ctx");
        const int rc = flowkv::gpu::sync_mirror(c, t->tree, *uid, *pos, t->ids, t->batch, t->img);
        if (rc != PBKV_OK) throw TreeError{rc, pbkv_last_error(c)};
    });
}

}  // extern "C"
