// Tree operation stream and the seeded synthetic-workload generator.
//
// Both are templated on the tree type so that the SAME stream drives the
// product's RadixMirror (radix_mirror.hpp) and, in the test oracle, the
// reference flowkv::CacheTree (cache.hpp) -- which is how the SoA export of the
// mirror is pinned against the reference (tests/test_mirror_parity.py).
//
// Op stream: flat int64 words.
//   PBKV_OP_INSERT    w agent budget ntok tok[ntok]   insert_suffix  (cache.hpp:159)
//   PBKV_OP_MATCH     w agent ntok tok[ntok]          match_prefix   (cache.hpp:121)
//   PBKV_OP_TERMINATE w                               on_workflow_terminated (cache.hpp:224)
//   PBKV_OP_DEMOTE    id                              demote_to_host (cache.hpp:254)
//   PBKV_OP_PROMOTE   id                              promote_to_device (cache.hpp:278)
//   PBKV_OP_DROP      id                              drop_host_node (cache.hpp:294)
//   PBKV_OP_SET_SCORE id bits(double)                 set_score      (cache.hpp:320)
// Tokens are uint64 TokenIds (types.hpp:11) carried bit-for-bit in int64 words.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

namespace pbkv {

enum : std::int64_t {
    PBKV_OP_INSERT = 1,
    PBKV_OP_MATCH = 2,
    PBKV_OP_TERMINATE = 3,
    PBKV_OP_DEMOTE = 4,
    PBKV_OP_PROMOTE = 5,
    PBKV_OP_DROP = 6,
    PBKV_OP_SET_SCORE = 7,
};

struct OpStreamError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

/// Applies an op stream.  Tree exceptions propagate to the caller unchanged.
template <class Tree>
void apply_ops(Tree& tree, const std::int64_t* w, std::int64_t n) {
    std::int64_t i = 0;
    std::vector<std::uint64_t> tok;
    auto need = [&](std::int64_t k) {
        if (i + k > n) throw OpStreamError("truncated op stream");
    };
    auto read_tokens = [&](std::int64_t cnt) {
        if (cnt < 0) throw OpStreamError("negative token count in op stream");
        need(cnt);
        tok.resize(static_cast<std::size_t>(cnt));
        for (std::int64_t j = 0; j < cnt; ++j) tok[static_cast<std::size_t>(j)] = static_cast<std::uint64_t>(w[i + j]);
        i += cnt;
    };
    while (i < n) {
        std::int64_t op = w[i++];
        switch (op) {
            case PBKV_OP_INSERT: {
                need(4);
                std::int64_t wf = w[i], agent = w[i + 1], budget = w[i + 2], cnt = w[i + 3];
                i += 4;
                read_tokens(cnt);
                tree.insert_suffix(tok, wf, static_cast<int>(agent), budget);
                break;
            }
            case PBKV_OP_MATCH: {
                need(3);
                std::int64_t wf = w[i], agent = w[i + 1], cnt = w[i + 2];
                i += 3;
                read_tokens(cnt);
                tree.match_prefix(tok, wf, static_cast<int>(agent));
                break;
            }
            case PBKV_OP_TERMINATE:
                need(1);
                tree.on_workflow_terminated(w[i++]);
                break;
            case PBKV_OP_DEMOTE:
                need(1);
                tree.demote_to_host(static_cast<int>(w[i++]));
                break;
            case PBKV_OP_PROMOTE:
                need(1);
                tree.promote_to_device(static_cast<int>(w[i++]));
                break;
            case PBKV_OP_DROP:
                need(1);
                tree.drop_host_node(static_cast<int>(w[i++]));
                break;
            case PBKV_OP_SET_SCORE: {
                need(2);
                int id = static_cast<int>(w[i]);
                double s;
                std::memcpy(&s, &w[i + 1], sizeof s);
                i += 2;
                tree.set_score(id, s);
                break;
            }
            default:
                throw OpStreamError("unknown op code " + std::to_string(op));
        }
    }
}

/// Parameters of the synthetic workload.
struct SynthParams {
    std::int64_t n_nodes = 10000;      // stop inserting once the tree has this many nodes
    std::int64_t n_workflows = 256;    // W
    int agents = 16;                   // A (agent bit per insert, uniform)
    int group_size = 16;               // workflows per group prefix
    int shared_len = 32;               // global shared prefix, tagged by every workflow
    int group_len = 8;                 // per-group prefix
    int alphabet = 4;                  // private random string alphabet
    int max_rand_len = 10;             // private random string length in [1, max]
    double retired_frac = 0.3;         // terminate workflow ids [0, retired_frac*W)
    int host_every = 10;               // demote every k-th active device leaf (0 = none)
    std::uint64_t seed = 12345;
};

/// splitmix64 stream: the generator's only source of randomness.
struct SplitMix64 {
    std::uint64_t s;
    explicit SplitMix64(std::uint64_t seed) : s(seed) {}
    std::uint64_t next() {
        std::uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    std::uint64_t below(std::uint64_t n) { return next() % n; }
};

/// Token namespaces: shared (1<<60|i), group (2<<60|g<<20|i), private root
/// (3<<60|w); private random-string tokens are 0..alphabet-1.
inline std::uint64_t synth_shared_token(std::int64_t i) { return (1ULL << 60) | static_cast<std::uint64_t>(i); }
inline std::uint64_t synth_group_token(std::int64_t g, std::int64_t i) {
    return (2ULL << 60) | (static_cast<std::uint64_t>(g) << 20) | static_cast<std::uint64_t>(i);
}
inline std::uint64_t synth_private_token(std::int64_t w) { return (3ULL << 60) | static_cast<std::uint64_t>(w); }

/// Builds the synthetic tree:
///  1. round-robin over workflows: insert shared ++ group(w/group_size) ++
///     private(w) ++ random string, agent uniform in [0, A), until n_nodes;
///  2. terminate workflow ids [0, floor(retired_frac * W));
///  3. demote every host_every-th active (non-retired) device leaf, scanning
///     node ids in ascending order (builds the host tier for stage 4).
template <class Tree>
void synth_build(Tree& tree, const SynthParams& p) {
    if (p.n_workflows < 1 || p.agents < 1 || p.agents > 63 || p.alphabet < 1 || p.max_rand_len < 1 ||
        p.group_size < 1 || p.shared_len < 1 || p.group_len < 0)
        throw OpStreamError("invalid synthetic parameters");
    SplitMix64 rng(p.seed);
    std::vector<std::uint64_t> tok;
    bool full = static_cast<std::int64_t>(tree.node_count()) >= p.n_nodes;
    while (!full) {
        for (std::int64_t w = 0; w < p.n_workflows; ++w) {
            tok.clear();
            for (int i = 0; i < p.shared_len; ++i) tok.push_back(synth_shared_token(i));
            std::int64_t g = w / p.group_size;
            for (int i = 0; i < p.group_len; ++i) tok.push_back(synth_group_token(g, i));
            tok.push_back(synth_private_token(w));
            int L = 1 + static_cast<int>(rng.below(static_cast<std::uint64_t>(p.max_rand_len)));
            for (int i = 0; i < L; ++i) tok.push_back(rng.below(static_cast<std::uint64_t>(p.alphabet)));
            int agent = static_cast<int>(rng.below(static_cast<std::uint64_t>(p.agents)));
            tree.insert_suffix(tok, w, agent, -1);
            if (static_cast<std::int64_t>(tree.node_count()) >= p.n_nodes) {
                full = true;
                break;
            }
        }
    }
    std::int64_t n_term = static_cast<std::int64_t>(std::floor(p.retired_frac * static_cast<double>(p.n_workflows)));
    for (std::int64_t w = 0; w < n_term; ++w) tree.on_workflow_terminated(w);
    if (p.host_every > 0) {
        std::vector<int> leaves;
        for (std::size_t i = 1; i < tree.node_count(); ++i) {
            const auto& n = tree.node(static_cast<int>(i));
            if (static_cast<int>(n.tier) == 0 && n.device_children == 0 && !n.retired)
                leaves.push_back(static_cast<int>(i));
        }
        for (std::size_t j = 0; j < leaves.size(); j += static_cast<std::size_t>(p.host_every))
            tree.demote_to_host(leaves[j]);
    }
}

}  // namespace pbkv
