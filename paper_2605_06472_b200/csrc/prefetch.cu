// Stage 4 on sm_100a: conservative / aggressive prefetch candidate ranking
// (policies.hpp:181-235).  Candidates = host-tier nodes with a device parent
// and single-step value (Eq. 1, scoring.hpp:41-45) > 0, ranked by (value
// desc, id asc); the greedy-with-skip fill runs in one CTA.
#include <cub/device/device_radix_sort.cuh>

#include <cuda/std/tuple>

#include "common.cuh"

namespace pbkv {

using namespace dev;

ScoreArgs make_score_args(Context& c, double* out);

namespace {

unsigned int grid_cap(std::int64_t n, int block) {
    std::int64_t want = (n + block - 1) / block;
    const std::int64_t cap = 148LL * 16;
    if (want > cap) want = cap;
    return static_cast<unsigned int>(want < 1 ? 1 : want);
}

// Eq. 1 chain of a node, in access order (the reference sums the terms in
// WorkflowId order, scoring.hpp:43-44)
__device__ __forceinline__ double eq1(const ScoreArgs& s, unsigned int e0, unsigned int e1, bool* miss) {
    double v = 0.0;
    for (unsigned int e = e0; e < e1; ++e) {
        const int slot = __ldg(s.acc_slot + e);
        const unsigned long long b = __ldg(s.acc_bits + e) & s.amask;
        if (__ldg(s.fstate + slot) == 0) {
            *miss = true;
            continue;
        }
        v = __dadd_rn(v, mass_on(s.P + static_cast<std::size_t>(slot) * s.V1 * s.K, s.K, b));
    }
    return v;
}

__global__ void __launch_bounds__(256) prefetch_cand_kernel(ScoreArgs s, const int* parent, const std::uint8_t* flags,
                                                            const unsigned long long* last, CandKey* ck, double* cv,
                                                            unsigned long long* n_cand, DevStatus* st,
                                                            std::int64_t n_nodes) {
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    for (std::int64_t base = blockIdx.x * static_cast<std::int64_t>(blockDim.x); base < n_nodes; base += stride) {
        const std::int64_t i = base + threadIdx.x;
        const int n = static_cast<int>(i);
        bool take = false;
        double v = 0.0;
        if (i < n_nodes && n != 0 && (flags[n] & kFlagTierMask) == PBKV_TIER_HOST &&
            (flags[parent[n]] & kFlagTierMask) == PBKV_TIER_DEVICE) {
            bool miss = false;
            v = eq1(s, s.acc_rng[n].x, s.acc_rng[n].y, &miss);
            if (miss) {
                // the reference raises on the first host node in (last_access,
                // id) order (host_index_, cache.hpp:434): keep the minimum
                atomicCAS(&st->code, 0, PBKV_EINVAL);
                atomicCAS(&st->kind, 0, kErrMissingForecast);
                atomicMin(reinterpret_cast<unsigned long long*>(&st->aux), last[n]);
            } else {
                take = v > 0.0;
            }
        }
        const long long slot = warp_append(n_cand, take);
        if (take) {
            ck[slot] = CandKey{~enc_rank(v), static_cast<unsigned int>(n)};
            cv[slot] = v;
        }
    }
}

// error path: among host candidates with the minimal last_access that miss a
// forecast, the smallest id
__global__ void prefetch_err_id_kernel(ScoreArgs s, const int* parent, const std::uint8_t* flags,
                                       const unsigned long long* last, DevStatus* st, std::int64_t n_nodes) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n_nodes;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const int n = static_cast<int>(i);
        if (n == 0 || (flags[n] & kFlagTierMask) != PBKV_TIER_HOST) continue;
        if ((flags[parent[n]] & kFlagTierMask) != PBKV_TIER_DEVICE) continue;
        if (last[n] != static_cast<unsigned long long>(st->aux)) continue;
        bool miss = false;
        eq1(s, s.acc_rng[n].x, s.acc_rng[n].y, &miss);
        if (miss) atomicMin(&st->node, static_cast<long long>(n));
    }
}

// greedy fill with skip (policies.hpp:203-210): per round the block finds the
// first remaining candidate with len <= budget - selected_tokens, selects it
// and resumes after it
constexpr int kGreedyThreads = 1024;
__global__ void __launch_bounds__(kGreedyThreads) prefetch_greedy_kernel(const CandKey* sorted, const int* len,
                                                                         std::int64_t n, long long budget, int* sel,
                                                                         long long* counters) {
    using Red = cub::BlockReduce<long long, kGreedyThreads>;
    __shared__ typename Red::TempStorage tmp;
    __shared__ long long pick_sh, rem_sh, nsel_sh;
    if (threadIdx.x == 0) {
        rem_sh = budget;
        nsel_sh = 0;
    }
    __syncthreads();
    long long start = 0;
    while (start < n) {
        const long long rem = rem_sh;
        const long long i = start + threadIdx.x;
        long long mine = LLONG_MAX;
        if (i < n && static_cast<long long>(len[sorted[i].id]) <= rem) mine = i;
        long long pick = Red(tmp).Reduce(mine, cub::Min());
        if (threadIdx.x == 0) pick_sh = pick;
        __syncthreads();
        pick = pick_sh;
        if (pick == LLONG_MAX) {
            start += kGreedyThreads;
        } else {
            if (threadIdx.x == 0) {
                const int id = static_cast<int>(sorted[pick].id);
                sel[nsel_sh] = id;
                nsel_sh += 1;
                rem_sh -= len[id];
            }
            start = pick + 1;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        counters[1] = nsel_sh;
        counters[2] = budget - rem_sh;
    }
}

struct CandDecomposer {
    __host__ __device__ ::cuda::std::tuple<unsigned long long&, unsigned int&> operator()(CandKey& k) const {
        return {k.vdesc, k.id};
    }
};

}  // namespace

void launch_prefetch_candidates(Context& c, unsigned long long* n_cand_dev) {
    ScoreArgs s = make_score_args(c, nullptr);
    prefetch_cand_kernel<<<grid_cap(c.n, 256), 256, 0, c.stream>>>(s, c.parent.p, c.flags.p, c.last.p, c.ck_in.p,
                                                                   c.cv_in.p, n_cand_dev, c.status.p, c.n);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

void launch_prefetch_err_id(Context& c) {
    ScoreArgs s = make_score_args(c, nullptr);
    prefetch_err_id_kernel<<<grid_cap(c.n, 256), 256, 0, c.stream>>>(s, c.parent.p, c.flags.p, c.last.p, c.status.p,
                                                                     c.n);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

void launch_prefetch_sort_greedy(Context& c, std::int64_t n_cand, long long budget, long long* counters_dev) {
    std::size_t b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b, c.ck_in.p, c.ck_out.p, c.cv_in.p, c.cv_out.p, static_cast<int>(n_cand),
                                    CandDecomposer{});
    c.cub_tmp.reserve(b);
    ++c.lib_calls;
    PBKV_CUDA(cub::DeviceRadixSort::SortPairs(c.cub_tmp.p, b, c.ck_in.p, c.ck_out.p, c.cv_in.p, c.cv_out.p,
                                              static_cast<int>(n_cand), CandDecomposer{}, c.stream));
    prefetch_greedy_kernel<<<1, kGreedyThreads, 0, c.stream>>>(c.ck_out.p, c.len.p, n_cand, budget, c.sel.p,
                                                               counters_dev);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

}  // namespace pbkv
