// sim_interpose.cpp -- the UNMODIFIED reference simulator with its policy call
// sites redirected to the GPU drop-in (include/pbkv/flowkv_gpu.hpp).
//
// TEST INFRASTRUCTURE (parity harness for BASELINE configs 1 and 5).  Built by
// oracle/Makefile twice from this one file:
//   _ref/sim_cpu  -- plain reference build (no interposition): the oracle run
//   _ref/sim_gpu  -- -DPBKV_INTERPOSE: simulator.hpp:434, :464, :618, :636-637,
//                    :657 call flowkv::gpu::* (the product, libpbkv.so), and
//                    the simulator's CacheTree (:349) is a TrackedCacheTree,
//                    so the device mirror is updated incrementally
//   _ref/sim_gpu_fed -- also -DPBKV_DEVICE_PREDICT: the predictor slot
//                    (simulator.hpp:414-421) computes every forecast on the
//                    GPU, so the whole run is device-fed
// Technique: SURVEY.md App. A.4 -- the CPU definitions are included first
// (#pragma once), then the call-site names are macro-renamed only while
// simulator.hpp is parsed.  No reference source is edited or copied.
//
// Usage: sim_{cpu,gpu} <scenario.json> [cell-substring] [max-seeds]
// Prints one line per (cell, seed):
//   cell seed hit_rate evictions prefetch_tokens shortfalls events_fnv dump_fnv
// events_fnv / dump_fnv are FNV-1a 64 of events_to_log() (simulator.hpp:191)
// and of the final CacheTree::dump() (cache.hpp:330).
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>

#include <algorithm>
#include <type_traits>
#include <vector>

#include "flowkv/policies.hpp"
#include "flowkv/scoring.hpp"

// Per-call wall time of every policy call site, in both builds (printed to
// stderr as "timing <op> <calls> <p50_us> <p99_us> <total_ms>" after the runs,
// when PBKV_SIM_TIMING is set): the drop-in's per-call latency against the
// reference's on the same scenario (BASELINE configs 1 and 5).
namespace pbkv_sim {
enum Op { kSelect, kSelectHE, kPlan, kRefreshScores, kRefreshNodes, kPredict, kNumOps };
inline const char* op_name(int o) {
    static const char* n[] = {"select_victims", "select_victims_hierarchical", "plan_prefetch", "refresh_scores",
                              "refresh_nodes", "predict"};
    return n[o];
}
inline std::vector<double>& samples(int o) {
    static std::vector<double> v[kNumOps];
    return v[o];
}
template <class F>
inline auto timed(int op, F&& f) {
    const auto t0 = std::chrono::steady_clock::now();
    auto done = [&] {
        samples(op).push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
    };
    if constexpr (std::is_void_v<decltype(f())>) {
        f();
        done();
    } else {
        auto r = f();
        done();
        return r;
    }
}
inline void report() {
    for (int o = 0; o < kNumOps; ++o) {
        std::vector<double> v = samples(o);
        if (v.empty()) continue;
        std::sort(v.begin(), v.end());
        double tot = 0;
        for (double x : v) tot += x;
        std::fprintf(stderr, "timing %s %zu %.2f %.2f %.3f\n", op_name(o), v.size(), v[v.size() / 2],
                     v[std::min(v.size() - 1, static_cast<std::size_t>(0.99 * static_cast<double>(v.size())))],
                     tot * 1e-3);
    }
}
}  // namespace pbkv_sim
#ifdef PBKV_INTERPOSE
#define PBKV_NS ::flowkv::gpu
#else
#define PBKV_NS ::flowkv
#endif

#ifdef PBKV_INTERPOSE
#include "flowkv/callgraph.hpp"
#include "flowkv/csv.hpp"
#include "flowkv/predictor.hpp"
#include "flowkv/rng.hpp"
#include "pbkv/flowkv_gpu.hpp"
#ifdef PBKV_DEVICE_PREDICT
// Simulator::predict (simulator.hpp:414-421) fed by the device: the exact
// K-step marginals (callgraph.hpp:136-186) and the Markov propagation
// (predictor.hpp:79-118) run on the GPU (fmodel.cu, gpu::*_predict_batch);
// noisy_predict's (1-lambda) p + lambda / V1 mix (predictor.hpp:25-35) is
// applied by the slot to the device marginals.  The member calls are
// rewritten by function-like macros into a conditional whose both arms call
// the device (the condition only keeps the expression well formed).
namespace pbkv_sim {
inline flowkv::Forecast gpu_marginals(const flowkv::CallGraph& g, std::span<const flowkv::AgentId> p, int k) {
    const std::vector<std::vector<flowkv::AgentId>> one{std::vector<flowkv::AgentId>(p.begin(), p.end())};
    return timed(kPredict, [&] { return flowkv::gpu::oracle_predict_batch(g, one, k)[0]; });
}
inline flowkv::Forecast gpu_markov(const flowkv::MarkovModel& m, std::span<const flowkv::AgentId> p, int k) {
    const std::vector<std::vector<flowkv::AgentId>> one{std::vector<flowkv::AgentId>(p.begin(), p.end())};
    return timed(kPredict, [&] { return flowkv::gpu::markov_predict_batch(m, one, k)[0]; });
}
}  // namespace pbkv_sim
#define true_kstep_marginals(p, k) \
    edges().empty() ? ::pbkv_sim::gpu_marginals(g_, p, k) : ::pbkv_sim::gpu_marginals(g_, p, k)
#define PBKV_PRED_SEL(_1, _2, NAME, ...) NAME
#define PBKV_PRED1(x) predict(x)
#define PBKV_PRED2(p, k) \
    num_agents() < 0 ? ::pbkv_sim::gpu_markov(markov_, p, k) : ::pbkv_sim::gpu_markov(markov_, p, k)
#define predict(...) PBKV_PRED_SEL(__VA_ARGS__, PBKV_PRED2, PBKV_PRED1)(__VA_ARGS__)
#endif
// the simulator's tree carries a change log: every policy call mirrors only
// the nodes changed since the previous call (pbkv_mirror_delta)
#define CacheTree TrackedCacheTree
#endif
// the policy call sites (simulator.hpp:434, :464, :618, :636-637, :657):
// PBKV_NS::* -- flowkv::gpu::* (the drop-in) or flowkv::* (the reference)
#define select_victims(...) ::pbkv_sim::timed(::pbkv_sim::kSelect, [&] { return PBKV_NS::select_victims(__VA_ARGS__); })
#define select_victims_hierarchical(...) \
    ::pbkv_sim::timed(::pbkv_sim::kSelectHE, [&] { return PBKV_NS::select_victims_hierarchical(__VA_ARGS__); })
#define plan_conservative_prefetch(...) \
    ::pbkv_sim::timed(::pbkv_sim::kPlan, [&] { return PBKV_NS::plan_conservative_prefetch(__VA_ARGS__); })
#define plan_aggressive_prefetch(...) \
    ::pbkv_sim::timed(::pbkv_sim::kPlan, [&] { return PBKV_NS::plan_aggressive_prefetch(__VA_ARGS__); })
#define refresh_scores(...) ::pbkv_sim::timed(::pbkv_sim::kRefreshScores, [&] { return PBKV_NS::refresh_scores(__VA_ARGS__); })
#define refresh_nodes(...) ::pbkv_sim::timed(::pbkv_sim::kRefreshNodes, [&] { return PBKV_NS::refresh_nodes(__VA_ARGS__); })
#include "flowkv/simulator.hpp"
#undef select_victims
#undef select_victims_hierarchical
#undef plan_conservative_prefetch
#undef plan_aggressive_prefetch
#undef refresh_scores
#undef refresh_nodes
#ifdef PBKV_INTERPOSE
#undef CacheTree
#undef select_victims
#undef select_victims_hierarchical
#undef plan_conservative_prefetch
#undef plan_aggressive_prefetch
#undef refresh_scores
#undef refresh_nodes
#ifdef PBKV_DEVICE_PREDICT
#undef true_kstep_marginals
#undef predict
#endif
#endif
#include "flowkv/scenario.hpp"

static std::uint64_t fnv1a(const std::string& s) {
    std::uint64_t h = 1469598103934665603ull;
    for (unsigned char ch : s) {
        h ^= ch;
        h *= 1099511628211ull;
    }
    return h;
}

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s <scenario.json> [cell-substring] [max-seeds]\n", argv[0]);
        return 2;
    }
    try {
        flowkv::Scenario sc = flowkv::Scenario::from_file(argv[1]);
        const std::string filt = argc > 2 ? argv[2] : "";
        const std::size_t max_seeds = argc > 3 ? std::strtoul(argv[3], nullptr, 10) : sc.seeds.size();
        for (const auto& cell : sc.cells()) {
            if (!filt.empty() && cell.id.find(filt) == std::string::npos) continue;
            for (std::size_t s = 0; s < sc.seeds.size() && s < max_seeds; ++s) {
                flowkv::SimConfig cfg = sc.config_for(cell, sc.seeds[s]);
                auto t0 = std::chrono::steady_clock::now();
                flowkv::RunResult r = flowkv::run(cfg);
                double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                const auto& m = r.metrics;
                std::printf("%s %llu %s %lld %lld %lld %016llx %016llx %.3f\n", cell.id.c_str(),
                            static_cast<unsigned long long>(sc.seeds[s]), flowkv::fmt_double(m.hit_rate).c_str(),
                            static_cast<long long>(m.evictions), static_cast<long long>(m.prefetch_tokens),
                            static_cast<long long>(m.shortfalls),
                            static_cast<unsigned long long>(fnv1a(flowkv::events_to_log(r.events))),
                            static_cast<unsigned long long>(fnv1a(r.final_dump)), secs);
                std::fflush(stdout);
            }
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    if (std::getenv("PBKV_SIM_TIMING")) pbkv_sim::report();
    return 0;
}
