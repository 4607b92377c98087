// forecast_parity.cpp -- the reference predictors vs their batched GPU
// restatement (include/pbkv/flowkv_gpu.hpp -> csrc/fmodel.cu), bit for bit.
//
// TEST INFRASTRUCTURE (built by oracle/Makefile into _ref/forecast_parity where
// /root/reference exists; the binary travels to the GPU box).  For every
// bundled call graph (scenarios/graphs/*.json): sample workflows with the
// reference's own sampler, and for every prefix of every trace compare
//   CallGraph::true_kstep_marginals(prefix, K)      callgraph.hpp:136-186
//   noisy_predict(base, lambda)                     predictor.hpp:25-35
//   MarkovModel::predict(prefix, K) (trained with   predictor.hpp:79-118,
//     train_markov on reference-sampled traces)     :175-188
// against flowkv::gpu::{oracle,markov}_predict_batch.  Exit 0 iff every
// probability is bit-identical; prints one summary line per graph.
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#define PBKV_WITH_PREDICTORS
#include "flowkv/callgraph.hpp"
#include "flowkv/predictor.hpp"
#include "pbkv/flowkv_gpu.hpp"

using namespace flowkv;

static long long compare(const std::vector<Forecast>& a, const std::vector<Forecast>& b) {
    long long bad = 0;
    for (std::size_t i = 0; i < a.size(); ++i)
        for (int k = 0; k < a[i].horizon(); ++k)
            for (int o = 0; o < a[i].outcomes(); ++o) {
                const double x = a[i].at(k, o), y = b[i].at(k, o);
                if (std::memcmp(&x, &y, sizeof x) != 0) ++bad;
            }
    return bad;
}

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : "oracle/_ref/scenarios/graphs";
    const char* graphs[] = {"codegen_retry.json", "factcheck_loop.json", "report_pipeline.json"};
    long long total_bad = 0, total_vals = 0;
    for (const char* gname : graphs) {
        CallGraph g = CallGraph::from_file(dir + "/" + gname);
        std::vector<WorkflowTrace> traces;
        for (int i = 0; i < 300; ++i) traces.push_back(g.sample_workflow(1000 + i, i));
        std::vector<std::vector<AgentId>> prefixes{{}};
        for (int i = 0; i < 60; ++i)
            for (std::size_t t = 1; t <= traces[i].invocations.size(); ++t)
                prefixes.emplace_back(traces[i].invocations.begin(), traces[i].invocations.begin() + t);
        long long bad = 0, vals = 0;
        for (int K : {1, 3, 8}) {
            std::vector<Forecast> ref;
            for (const auto& p : prefixes) ref.push_back(g.true_kstep_marginals(p, K));
            auto gpu = gpu::oracle_predict_batch(g, prefixes, K);
            bad += compare(ref, gpu);
            vals += static_cast<long long>(ref.size()) * K * g.outcomes();
            for (double lambda : {0.0, 0.1, 0.5, 1.0}) {
                std::vector<Forecast> rn;
                for (const auto& b : ref) rn.push_back(noisy_predict(b, lambda));
                auto gn = gpu::oracle_predict_batch(g, prefixes, K, lambda);
                bad += compare(rn, gn);
                vals += static_cast<long long>(rn.size()) * K * g.outcomes();
            }
            std::vector<std::vector<AgentId>> nonempty(prefixes.begin() + 1, prefixes.end());
            for (int order : {1, 2, 3}) {
                MarkovModel mm = train_markov(std::span<const WorkflowTrace>(traces), g.num_agents(), order, 0.5);
                std::vector<Forecast> rm;
                for (const auto& p : nonempty) rm.push_back(mm.predict(p, K));
                auto gm = gpu::markov_predict_batch(mm, nonempty, K);
                bad += compare(rm, gm);
                vals += static_cast<long long>(rm.size()) * K * g.outcomes();
            }
        }
        std::printf("%s prefixes=%zu values=%lld mismatches=%lld\n", gname, prefixes.size(), vals, bad);
        total_bad += bad;
        total_vals += vals;
    }
    std::printf("total values=%lld mismatches=%lld\n", total_vals, total_bad);
    return total_bad == 0 ? 0 : 1;
}
