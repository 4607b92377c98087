// Batched forward-propagation forecasters on sm_100a, bit-exact with the
// reference predictors of the simulator's predictor slot (simulator.hpp:414-421):
//   CallGraph::true_kstep_marginals   callgraph.hpp:136-186  (oracle)
//   MarkovModel::predict              predictor.hpp:79-118
//   noisy_predict                     predictor.hpp:25-35   (lambda >= 0)
// Both predictors propagate alive mass over context states visited in the
// order of a std::map; the host flattens the model into a state table in that
// order (rows[s][0..V1), next[s][a]), so one thread per workflow replays the
// reference's loops exactly: states ascending, agents ascending,
//   alive += m;  outcome[a] += m*p;  next_mass[next(s,a)] += m*p;
// then outcome /= alive (or the absorbing END row when alive <= 1e-15).
// All in binary64 with __dadd_rn / __dmul_rn / __ddiv_rn (no contraction).
// The rows land in the forecast staging buffer; forecast_prepare_kernel
// validates them like the Forecast ctor and builds P / gs (score.cu).
#include "common.cuh"

namespace pbkv {

using namespace dev;

namespace {

__global__ void propagate_kernel(const double* rows, const int* next, int S, int A, const int* start,
                                 std::int64_t n, int H, double lambda, double* mass, double* stage,
                                 DevStatus* st) {
    const int V1 = A + 1;
    for (std::int64_t w = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; w < n;
         w += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        double* cur = mass + static_cast<std::size_t>(w) * 2 * S;
        double* nxt = cur + S;
        for (int s = 0; s < S; ++s) cur[s] = 0.0;
        const int s0 = start[w];
        if (s0 < 0 || s0 >= S) {
            set_error(st, PBKV_EINVAL, kErrModelState, w);
            continue;
        }
        cur[s0] = 1.0;
        double* out = stage + static_cast<std::size_t>(w) * H * V1;
        bool bad = false, lost = false;  // lost: positive mass sent to a state without a row
        for (int k = 0; k < H && !bad; ++k) {
            if (lost) {  // the reference fails when it visits that state (kernel_.at, callgraph.hpp:160)
                bad = true;
                break;
            }
            double* o = out + static_cast<std::size_t>(k) * V1;
            for (int a = 0; a < V1; ++a) o[a] = 0.0;
            for (int s = 0; s < S; ++s) nxt[s] = 0.0;
            double alive = 0.0;
            for (int s = 0; s < S; ++s) {
                const double m = cur[s];
                if (!(m > 0.0)) continue;  // m <= 0.0 (callgraph.hpp:157)
                alive = __dadd_rn(alive, m);
                const double* row = rows + static_cast<std::size_t>(s) * V1;
                for (int a = 0; a < V1; ++a) {
                    const double p = row[a];
                    if (!(p > 0.0)) continue;
                    const double mp = __dmul_rn(m, p);
                    o[a] = __dadd_rn(o[a], mp);
                    if (a != A) {
                        const int ns = next[static_cast<std::size_t>(s) * A + a];
                        if (ns < 0)
                            lost = lost || mp > 0.0;
                        else
                            nxt[ns] = __dadd_rn(nxt[ns], mp);
                    }
                }
            }
            if (alive <= 1e-15) {  // absorbed: degenerate at END from here on
                for (int a = 0; a < V1; ++a) o[a] = 0.0;
                o[A] = 1.0;
            } else {
                for (int a = 0; a < V1; ++a) o[a] = __ddiv_rn(o[a], alive);
            }
            double* t = cur;
            cur = nxt;
            nxt = t;
        }
        if (bad) {
            set_error(st, PBKV_EINVAL, kErrModelState, w);
            continue;
        }
        if (!(lambda >= 0.0)) continue;
        // noisy_predict: (1 - lambda) * P + lambda * (1 / V1), per entry
        const double keep = __dsub_rn(1.0, lambda);
        const double lu = __dmul_rn(lambda, __ddiv_rn(1.0, static_cast<double>(V1)));
        for (int i = 0; i < H * V1; ++i) out[i] = __dadd_rn(__dmul_rn(keep, out[i]), lu);
    }
}

}  // namespace

void launch_propagate(Context& c, const int* start_dev, std::int64_t n, int H, double lambda) {
    const int S = static_cast<int>(c.fm_states);
    c.fm_mass.reserve(static_cast<std::size_t>(n) * 2 * (S > 0 ? S : 1));
    propagate_kernel<<<grid_for(n, 128), 128, 0, c.stream>>>(c.fm_rows.p, c.fm_next.p, S, c.A, start_dev, n, H,
                                                             lambda, c.fm_mass.p, c.fstage.p, c.status.p);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

}  // namespace pbkv
