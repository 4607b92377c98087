// Stage 2 on sm_100a: Eq. 2 (scoring.hpp:49-62) for every node, bit-exact.
//
// Nodes are split by their Eq. 2 chain length L = entries * K:
//   light  (entries <= 2)     one thread per node, chain in registers
//   medium (L <= 256)         one warp per node: products in parallel, the
//                             serial add chain from shared memory
//   heavy  (L > 256)          products for all heavy entries by the whole grid,
//                             then one CTA per node evaluates the serial
//                             rounding chain exactly in parallel per binade
// The heavy path runs on a side stream, overlapped with the light pass.
#include <climits>

#include "chain.cuh"
#include "common.cuh"

namespace pbkv {

using namespace dev;

namespace {

constexpr int kLightThreads = 256;
constexpr int kMediumWarps = 8;
constexpr int kMediumMaxElems = 256;
constexpr int kChainThreads = 256;

unsigned int grid_cap(std::int64_t n, int block) {
    std::int64_t want = (n + block - 1) / block;
    const std::int64_t cap = 148LL * 16;
    if (want > cap) want = cap;
    return static_cast<unsigned int>(want < 1 ? 1 : want);
}
constexpr int kChainEPT = 8;  // elements per thread per chunk
constexpr int kChainChunk = kChainThreads * kChainEPT;

// Eq. 2 of one access entry appended to `total` (scoring.hpp:56-59)
__device__ __forceinline__ void eq2_entry(const ScoreArgs& s, int slot, unsigned long long b, double& total) {
    const int K = s.K;
    const double* pw = s.P + static_cast<std::size_t>(slot) * s.V1 * K;
    const double* g = s.gs + static_cast<std::size_t>(slot) * K;
    for (int k = 0; k < K; ++k) total = __dadd_rn(total, __dmul_rn(__ldg(g + k), mass_on(pw + k, K, b)));
}

// One 32-byte global load (LDG.E.256, sm_100): a gathered row of 4 doubles
// costs one L1 wavefront per lane instead of two with 16-byte loads.
__device__ __forceinline__ void ldg4d(const double* p, double* v) {
    asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
        : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
        : "l"(p));
}

// kK doubles from a row aligned to min(kK, 4) * 8 bytes, widest loads first
template <int kK>
__device__ __forceinline__ void load_row(const double* p, double* v) {
    if constexpr (kK % 4 == 0) {
#pragma unroll
        for (int k = 0; k < kK; k += 4) ldg4d(p + k, v + k);
    } else if constexpr (kK % 2 == 0) {
#pragma unroll
        for (int k = 0; k < kK; k += 2) {
            const double2 t = __ldg(reinterpret_cast<const double2*>(p + k));
            v[k] = t.x;
            v[k + 1] = t.y;
        }
    } else {
#pragma unroll
        for (int k = 0; k < kK; ++k) v[k] = __ldg(p + k);
    }
}

// Eq. 2 of one access entry with the horizon known at compile time: the K
// step masses are accumulated agent by agent (ascending, forecast.hpp:66-67)
// in K independent registers, so the K row loads of each agent are in flight
// together; then total += gs[k] * m[k] in step order (scoring.hpp:56-57).
template <int kK>
__device__ __forceinline__ void eq2_entry_k(const ScoreArgs& s, int slot, unsigned long long b, double& total) {
    if (!b) {  // no agent inside [0, A): no row is read, so the slot's state is checked here
        if (__ldg(s.fstate + slot) != 1) total = CUDART_NAN;  // missing / short: raised like a poisoned row
        return;
    }
    if (!(b & (b - 1))) {  // one agent: the K terms are precomputed (Pg), one 64-byte line
        const double* row = s.Pg + (static_cast<std::size_t>(slot) * s.V1 + (__ffsll(static_cast<long long>(b)) - 1)) * kK;
        double v[kK];
        load_row<kK>(row, v);
#pragma unroll
        for (int k = 0; k < kK; ++k) total = __dadd_rn(total, v[k]);
        return;
    }
    const double* pw = s.P + static_cast<std::size_t>(slot) * s.V1 * kK;  // [agent][k]
    const double* g = s.gs + static_cast<std::size_t>(slot) * kK;
    double m[kK];
#pragma unroll
    for (int k = 0; k < kK; ++k) m[k] = 0.0;
    // agents in groups: all rows of a group are loaded before any is added
    // (one L2 round trip per group instead of per agent), then added in
    // ascending agent order (forecast.hpp:66-67)
    constexpr int kG = kK <= 4 ? 4 : 2;
    while (b) {
        const double* row[kG];
        int cnt = 0;
#pragma unroll
        for (int j = 0; j < kG; ++j) {
            row[j] = nullptr;
            if (b) {
                row[j] = pw + static_cast<std::size_t>(__ffsll(static_cast<long long>(b)) - 1) * kK;
                b &= b - 1;
                cnt = j + 1;
            }
        }
        double v[kG][kK];
#pragma unroll
        for (int j = 0; j < kG; ++j) {
            if (j >= cnt) continue;
            load_row<kK>(row[j], v[j]);
        }
#pragma unroll
        for (int j = 0; j < kG; ++j) {
            if (j >= cnt) continue;
#pragma unroll
            for (int k = 0; k < kK; ++k) m[k] = __dadd_rn(m[k], v[j][k]);
        }
    }
    double gv[kK];
    load_row<kK>(g, gv);
#pragma unroll
    for (int k = 0; k < kK; ++k) total = __dadd_rn(total, __dmul_rn(gv[k], m[k]));
}

// ---------------------------------------------------------------------------
// Light nodes (<= 2 entries): one thread per node, Eq. 2 and the stage-3 key
// in registers.  kK > 0: horizon specialised; kK == 0: any horizon.
template <bool kKeys, int kK>
#ifndef PBKV_LIGHT_MINB
#define PBKV_LIGHT_MINB 4  // CTAs/SM the registers are sized for (measured: 4 -> 38 us, 5 -> 52, 6 -> 73: spills)
#endif
__global__ void __launch_bounds__(kLightThreads, PBKV_LIGHT_MINB) score_light_kernel(ScoreArgs s, KeyArgs ka, std::int64_t n_nodes,
                                                                       int report_missing) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n_nodes;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const int n = static_cast<int>(i);
        // the node's (at most two) entries, node-indexed and coalesced
        const int2 ls = s.lslot[n];
        const ulonglong2 lb = s.lbits[n];
        // key inputs are independent of the Eq. 2 chain: issued up front
        std::uint8_t fl = 0;
        unsigned long long last = 0;
        int ever = 0;
        if constexpr (kKeys) {
            fl = ka.flags[n];
            last = ka.last[n];
            ever = ka.ever[n];
        }
        const bool light = ls.x != -2;
        double total = 0.0;
        bool miss = false, shorth = false;
        if (light) {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int slot = q == 0 ? ls.x : ls.y;
                if (slot < 0) break;
                const unsigned long long b = (q == 0 ? lb.x : lb.y) & s.amask;
                if constexpr (kK > 0) {
                    eq2_entry_k<kK>(s, slot, b, total);  // unusable slots hold NaN rows
                } else {
                    const std::uint8_t fs = __ldg(s.fstate + slot);
                    if (fs != 1) {
                        (fs == 2 ? shorth : miss) = true;
                        continue;
                    }
                    eq2_entry(s, slot, b, total);
                }
            }
            if constexpr (kK > 0) miss = isnan(total);  // the message is resolved from fstate on error
            s.out[n] = total;
            if (report_missing && (miss || shorth))
                set_error(s.st, PBKV_EINVAL, miss ? kErrMissingForecast : kErrShortHorizon, n);
        }
        if constexpr (kKeys) {
            ka.eff[n] = n;
            ka.sublock[n] = 0;
            ka.W[n] = 0;  // chain weight / size accumulators of the selection
            ka.C[n] = 0;
            const bool dev = n != 0 && (fl & kFlagTierMask) == PBKV_TIER_DEVICE;
            if (light) {
                ka.missing[n] = (miss || shorth) ? 1 : 0;
                if (dev) write_key_v(ka, n, total, fl, last, ever);
            }
            // every other node's key is defined too (zero): the selection's
            // batched loads read keys before they test the tier
            if (!dev) reinterpret_cast<ulonglong2*>(ka.keys)[n] = make_ulonglong2(0ull, 0ull);
        }
    }
}

template <bool kKeys>
void launch_light(Context& c, const ScoreArgs& s, const KeyArgs& ka, int rm) {
    const unsigned int g = grid_cap(c.n, kLightThreads);
    if (c.timing) {
        PBKV_CUDA(cudaEventRecord(c.kev[0], c.stream));
        c.kev_light = true;
    }
    struct After {
        Context& c;
        ~After() {
            if (c.timing) cudaEventRecord(c.kev[1], c.stream);
        }
    } after{c};
    switch (c.K) {
        case 1: score_light_kernel<kKeys, 1><<<g, kLightThreads, 0, c.stream>>>(s, ka, c.n, rm); break;
        case 2: score_light_kernel<kKeys, 2><<<g, kLightThreads, 0, c.stream>>>(s, ka, c.n, rm); break;
        case 3: score_light_kernel<kKeys, 3><<<g, kLightThreads, 0, c.stream>>>(s, ka, c.n, rm); break;
        case 4: score_light_kernel<kKeys, 4><<<g, kLightThreads, 0, c.stream>>>(s, ka, c.n, rm); break;
        case 8: score_light_kernel<kKeys, 8><<<g, kLightThreads, 0, c.stream>>>(s, ka, c.n, rm); break;
        default: score_light_kernel<kKeys, 0><<<g, kLightThreads, 0, c.stream>>>(s, ka, c.n, rm);
    }
}

// one warp per medium node: lane l forms products l, l+32, ... of the chain
// (element i = entry i/K, step i%K), lane 0 then adds them in order.
template <bool kKeys, bool kValueOnly>
__global__ void __launch_bounds__(kMediumWarps * 32) score_medium_kernel(ScoreArgs s, KeyArgs ka, const int* nodes,
                                                                         std::int64_t n_list, int report_missing,
                                                                         int report_per_node) {
    __shared__ double xs[kMediumWarps][kMediumMaxElems];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const std::int64_t w = blockIdx.x * static_cast<std::int64_t>(kMediumWarps) + warp;
    if (w >= n_list) return;
    const int n = nodes[w];
    const int K = kValueOnly ? 1 : s.K;
    const uint2 rg = s.acc_rng[n];
    const unsigned int e0 = rg.x, e1 = rg.y;
    const int L = static_cast<int>(e1 - e0) * K;
    int miss = 0;
    for (int i = lane; i < L; i += 32) {
        const unsigned int e = e0 + static_cast<unsigned int>(i / K);
        const int k = i % K;
        const int slot = __ldg(s.acc_slot + e);
        const unsigned long long b = __ldg(s.acc_bits + e) & s.amask;
        const std::uint8_t fs = __ldg(s.fstate + slot);
        double x = 0.0;
        if (kValueOnly ? fs == 0 : fs != 1) {
            miss |= (fs == 2 && !kValueOnly) ? 2 : 1;
        } else {
            const double* col = s.P + static_cast<std::size_t>(slot) * s.V1 * s.K + k;
            x = kValueOnly ? mass_on(col, s.K, b)
                           : __dmul_rn(__ldg(s.gs + static_cast<std::size_t>(slot) * s.K + k), mass_on(col, s.K, b));
        }
        xs[warp][i] = x;
    }
    miss = __reduce_or_sync(0xffffffffu, miss);
    __syncwarp();
    if (lane == 0) {
        double t = 0.0;
        for (int i = 0; i < L; ++i) t = __dadd_rn(t, xs[warp][i]);
        s.out[n] = t;
        if ((report_missing || report_per_node) && miss)
            set_error(s.st, PBKV_EINVAL, (miss & 1) ? kErrMissingForecast : kErrShortHorizon, n);
        if constexpr (kKeys) {
            ka.missing[n] = miss ? 1 : 0;
            if (n != 0 && (ka.flags[n] & kFlagTierMask) == PBKV_TIER_DEVICE) write_key(ka, n, t);
        }
    }
}

// products of every heavy entry: element j*K + k of the packed product array
// approx (optional, [2*heavy]): any-order sum and sum of |x| per heavy node,
// accumulated with one double atomic per warp run of the same node
__global__ void __launch_bounds__(256) heavy_products_kernel(ScoreArgs s, const unsigned int* hent,
                                                             const int* hent_node, std::int64_t n_hent, double* xs,
                                                             unsigned int* hmiss, double* approx, int n_heavy) {
    const int K = s.K;
    const std::int64_t total = n_hent * K;
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    const std::int64_t rounds = (total + stride - 1) / stride;  // uniform trip count: shuffles stay convergent
    for (std::int64_t r = 0; r < rounds; ++r) {
        const std::int64_t t = r * stride + blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
        const bool in = t < total;
        double x = 0.0;
        int node = -1;
        if (in) {
            const std::int64_t j = t / K;
            const int k = static_cast<int>(t - j * K);
            const unsigned int e = hent[j];
            const int slot = __ldg(s.acc_slot + e);
            const unsigned long long b = __ldg(s.acc_bits + e) & s.amask;
            const std::uint8_t fs = __ldg(s.fstate + slot);
            node = hent_node[j];
            if (fs != 1) {
                atomicOr(&hmiss[node], fs == 2 ? 2u : 1u);
            } else {
                const double* col = s.P + static_cast<std::size_t>(slot) * s.V1 * K + k;
                x = __dmul_rn(__ldg(s.gs + static_cast<std::size_t>(slot) * K + k), mass_on(col, K, b));
            }
            xs[t] = x;
        }
        if (approx == nullptr) continue;
        const unsigned same = __match_any_sync(0xffffffffu, node);
        double sx = 0.0, sa = 0.0;
        for (unsigned m = same; m; m &= m - 1) {
            const int src = __ffs(m) - 1;
            const double v = __shfl_sync(same, x, src);
            sx += v;
            sa += fabs(v);
        }
        if (node >= 0 && node < n_heavy && (threadIdx.x & 31) == __ffs(same) - 1) {
            atomicAdd(&approx[2 * node], sx);
            atomicAdd(&approx[2 * node + 1], sa);
        }
    }
}

struct SatAdd {
    __device__ __forceinline__ unsigned long long operator()(unsigned long long a, unsigned long long b) const {
        unsigned long long r = a + b;
        const unsigned long long cap = 1ull << 62;
        return (r > cap || r < a) ? cap : r;
    }
};

// The serial chain t <- RN(t + x_i), i = 0..L-1, evaluated exactly in
// parallel.  Inside one binade [2^(E-1), 2^E) with x_i >= 0,
// RN(t + x_i) = t + u * RN(x_i / u), u = ulp(t), unless x_i / u has a
// fractional part of exactly 1/2 (then the tie rounds to even, which depends
// on t).  So a run of steps is an integer prefix sum in units of u.  Binade
// crossings, exact ties and negative / NaN / huge x_i are "events", executed
// one at a time with __dadd_rn.  Bit-identical to scoring.hpp:52-60.
//
// kPre:  products read from `xs_g` (heavy path);
// !kPre: products formed in the CTA per chunk (id-list path: refresh_nodes).
template <bool kPre, bool kValueOnly, bool kKeys>
__global__ void __launch_bounds__(kChainThreads) chain_kernel(ScoreArgs s, KeyArgs ka, const int* nodes,
                                                              const long long* xs_start, const double* xs_g,
                                                              const unsigned int* hmiss, int report_missing) {
    using Scan = cub::BlockScan<unsigned long long, kChainThreads>;
    using RedI = cub::BlockReduce<int, kChainThreads>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ typename RedI::TempStorage red_tmp;
    __shared__ double xs[kChainChunk];
    __shared__ double t_sh;
    __shared__ int ev_sh;
    __shared__ unsigned long long pclean_sh;
    __shared__ int miss_sh;

    const int node = nodes[blockIdx.x];
    const int K = kValueOnly ? 1 : s.K;
    const uint2 rg = s.acc_rng[node];
    const unsigned int e0 = rg.x, e1 = rg.y;
    const long long L = static_cast<long long>(e1 - e0) * K;
    const int tid = threadIdx.x;
    if (tid == 0) {
        t_sh = 0.0;
        miss_sh = kPre ? static_cast<int>(hmiss[blockIdx.x]) : 0;
    }
    __syncthreads();

    for (long long c0 = 0; c0 < L; c0 += kChainChunk) {
        const int nc = static_cast<int>(min(static_cast<long long>(kChainChunk), L - c0));
        for (int i = tid; i < nc; i += kChainThreads) {
            if constexpr (kPre) {
                xs[i] = xs_g[xs_start[blockIdx.x] + c0 + i];
            } else {
                const long long gi = c0 + i;
                const unsigned int e = e0 + static_cast<unsigned int>(gi / K);
                const int k = static_cast<int>(gi % K);
                const int slot = __ldg(s.acc_slot + e);
                const unsigned long long b = __ldg(s.acc_bits + e) & s.amask;
                const std::uint8_t fs = __ldg(s.fstate + slot);
                double x = 0.0;
                if (kValueOnly ? fs == 0 : fs != 1) {
                    atomicOr(&miss_sh, (fs == 2 && !kValueOnly) ? 2 : 1);
                } else {
                    const double* col = s.P + static_cast<std::size_t>(slot) * s.V1 * s.K + k;
                    x = kValueOnly ? mass_on(col, s.K, b)
                                   : __dmul_rn(__ldg(s.gs + static_cast<std::size_t>(slot) * s.K + k),
                                               mass_on(col, s.K, b));
                }
                xs[i] = x;
            }
        }
        __syncthreads();
        int pos = 0;
        const int i0 = tid * kChainEPT;
        while (pos < nc) {
            const double t = t_sh;
            if (!(t > 0x1p-900 && t < 0x1p+1000)) {  // zero / tiny / huge running total: one serial step
                if (tid == 0) t_sh = __dadd_rn(t, xs[pos]);
                __syncthreads();
                ++pos;
                continue;
            }
            int E;
            frexp(t, &E);  // t = f * 2^E, f in [0.5, 1): ulp(t) = 2^(E-53)
            const double scale = ldexp(1.0, 53 - E);
            const unsigned long long T = static_cast<unsigned long long>(t * scale);  // in [2^52, 2^53)
            const unsigned long long room = (1ull << 53) - T;
            auto qof = [&](int i, unsigned long long& q) -> bool {
                const double y = xs[i] * scale;  // exact power-of-two scaling
                if (!(y >= 0.0) || y > 0x1p53) return false;
                if (fabs(y - trunc(y)) == 0.5) return false;  // exact tie
                q = static_cast<unsigned long long>(rint(y));
                return true;
            };
            unsigned long long local = 0;
            int first_bad = nc;
#pragma unroll
            for (int k = 0; k < kChainEPT; ++k) {
                const int i = i0 + k;
                if (i >= nc || i < pos || i >= first_bad) continue;
                unsigned long long q;
                if (!qof(i, q))
                    first_bad = i;
                else
                    local = SatAdd()(local, q);
            }
            unsigned long long excl;
            Scan(scan_tmp).ExclusiveScan(local, excl, 0ull, SatAdd());
            int my_ev = first_bad;
            unsigned long long run = excl;
#pragma unroll
            for (int k = 0; k < kChainEPT; ++k) {
                const int i = i0 + k;
                if (i >= nc || i < pos || i >= my_ev) continue;
                unsigned long long q = 0;
                qof(i, q);
                const unsigned long long nxt = SatAdd()(run, q);
                if (nxt > room)
                    my_ev = i;  // crossing at i
                else
                    run = nxt;
            }
            __syncthreads();
            const int blk_ev = RedI(red_tmp).Reduce(my_ev, cub::Min());
            if (tid == 0) ev_sh = blk_ev;
            __syncthreads();
            const int ev = ev_sh;
            if (ev > pos && tid == (ev - 1) / kChainEPT) {
                unsigned long long p = excl;
                for (int k = 0; k < kChainEPT; ++k) {
                    const int i = i0 + k;
                    if (i >= ev) break;
                    if (i < pos) continue;
                    unsigned long long q = 0;
                    qof(i, q);
                    p = SatAdd()(p, q);
                }
                pclean_sh = p;
            }
            __syncthreads();
            if (tid == 0) {
                const unsigned long long pc = ev > pos ? pclean_sh : 0ull;
                double tn = static_cast<double>(T + pc) / scale;  // exact: <= 2^53 units of ulp
                if (ev < nc) tn = __dadd_rn(tn, xs[ev]);        // the event step
                t_sh = tn;
            }
            __syncthreads();
            pos = ev < nc ? ev + 1 : nc;
        }
        __syncthreads();
    }
    if (tid == 0) {
        const double total = t_sh;
        s.out[node] = total;
        const int miss = miss_sh;
        if (report_missing && miss)
            set_error(s.st, PBKV_EINVAL, (miss & 1) ? kErrMissingForecast : kErrShortHorizon, node);
        if constexpr (kKeys) {
            ka.missing[node] = miss ? 1 : 0;
            if (node != 0 && (ka.flags[node] & kFlagTierMask) == PBKV_TIER_DEVICE) write_key(ka, node, total);
        }
    }
}

// Heavy nodes: one 1024-thread CTA per node runs the exact chain (chain.cuh)
// over the node's products (heavy_products_kernel).
template <bool kKeys>
__global__ void __launch_bounds__(kChainT) heavy_chain_kernel(ScoreArgs s, KeyArgs ka, const int* nodes,
                                                              const long long* xs_start, const double* xs_g,
                                                              const unsigned int* hmiss, int report_missing) {
    extern __shared__ __align__(16) unsigned char chain_raw[];
    ChainSmem& sm = *reinterpret_cast<ChainSmem*>(chain_raw);
    const int node = nodes[blockIdx.x];
    const long long L = static_cast<long long>(s.acc_rng[node].y - s.acc_rng[node].x) * s.K;
    const double total = chain_eval(xs_g + xs_start[blockIdx.x], L, sm);
    if (threadIdx.x == 0) {
        s.out[node] = total;
        const unsigned int miss = hmiss[blockIdx.x];
        if (report_missing && miss)
            set_error(s.st, PBKV_EINVAL, (miss & 1) ? kErrMissingForecast : kErrShortHorizon, node);
        if constexpr (kKeys) {
            ka.missing[node] = miss ? 1 : 0;
            if (node != 0 && (ka.flags[node] & kFlagTierMask) == PBKV_TIER_DEVICE) write_key(ka, node, total);
        }
    }
}

// Medium nodes (entries * K <= 256): one warp per node adds the node's
// products (heavy_products_kernel, combined index n_heavy + m) in order;
// lanes fetch 32 at a time, lane 0 folds them via shuffles.
template <bool kKeys>
__global__ void __launch_bounds__(256) medium_chain_kernel(ScoreArgs s, KeyArgs ka, const int* medium,
                                                           std::int64_t n_medium, std::int64_t n_heavy,
                                                           const long long* xs_start, const double* xs_g,
                                                           const unsigned int* hmiss, int report_missing) {
    const std::int64_t m = (blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (m >= n_medium) return;
    const int node = medium[m];
    const int L = static_cast<int>(s.acc_rng[node].y - s.acc_rng[node].x) * s.K;
    const double* x = xs_g + xs_start[n_heavy + m];
    double t = 0.0;
    for (int c0 = 0; c0 < L; c0 += 32) {
        const double v = c0 + lane < L ? __ldcg(x + c0 + lane) : 0.0;
        const int cnt = min(32, L - c0);
        for (int q = 0; q < cnt; ++q) t = __dadd_rn(t, __shfl_sync(0xffffffffu, v, q));
    }
    if (lane == 0) {
        s.out[node] = t;
        const unsigned int miss = hmiss[n_heavy + m];
        if (report_missing && miss)
            set_error(s.st, PBKV_EINVAL, (miss & 1) ? kErrMissingForecast : kErrShortHorizon, node);
        if constexpr (kKeys) {
            ka.missing[node] = miss ? 1 : 0;
            if (node != 0 && (ka.flags[node] & kFlagTierMask) == PBKV_TIER_DEVICE) write_key(ka, node, t);
        }
    }
}

// Generic exact chains: out[b] = the chain over x[off[b], off[b+1]) (the
// sharded spine score over all ranks' products, shard.cu).
__global__ void __launch_bounds__(kChainT) chain_sum_kernel(const double* x, const long long* off, double* out) {
    extern __shared__ __align__(16) unsigned char chain_raw[];
    ChainSmem& sm = *reinterpret_cast<ChainSmem*>(chain_raw);
    const double t = chain_eval(x + off[blockIdx.x], off[blockIdx.x + 1] - off[blockIdx.x], sm);
    if (threadIdx.x == 0) out[blockIdx.x] = t;
}

// Approximate Eq. 2 of each heavy node (the decision fast path): the sum and
// the sum of |terms| of its products in any order, accumulated by
// heavy_products_kernel.  The exact serial chain E and this sum A both lie
// within L * ulp(sum|x|) / 2 of the real sum, so |E - A| <= L * ulp(sum|x|).

__global__ void set_deferred_kernel(std::uint8_t* flags, Key2* keys, const int* nodes, int n, int on,
                                    const int* skip_if) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || (skip_if && *skip_if)) return;
    const int v = nodes[i];
    flags[v] = on ? (flags[v] | kFlagDeferred) : (flags[v] & ~kFlagDeferred);
    if (on) reinterpret_cast<ulonglong2*>(keys)[v] = make_ulonglong2(0ull, 0ull);  // out of every eff max
}

// First kernel of a decision: the status word reset (no host->device copy)
// and, with heavy deferral, the deferred flags / zero keys and the side
// stream's accumulators (hmiss, approx).
__global__ void decision_prologue_kernel(DevStatus* st, std::uint8_t* flags, Key2* keys, const int* heavy,
                                         int n_heavy, int defer, unsigned int* hmiss, int n_hmiss, double* approx) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0 && st) *st = DevStatus{0, 0, LLONG_MAX, LLONG_MAX};  // (kept when an async upload's is unread)
    if (!defer) return;
    if (i < n_heavy) {
        const int v = heavy[i];
        flags[v] = flags[v] | kFlagDeferred;
        reinterpret_cast<ulonglong2*>(keys)[v] = make_ulonglong2(0ull, 0ull);  // out of every eff max
        approx[2 * i] = 0.0;
        approx[2 * i + 1] = 0.0;
    }
    if (i < n_hmiss) hmiss[i] = 0u;
}

// Eq. 1 / Eq. 2 of an id list, one thread per short id (refresh_nodes path)
template <bool kValueOnly>
__global__ void __launch_bounds__(256) score_ids_kernel(ScoreArgs s, const int* ids, std::int64_t n, double* out) {
    for (std::int64_t j = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; j < n;
         j += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const int id = ids[j];
        const uint2 rg = s.acc_rng[id];
        const unsigned int e0 = rg.x, e1 = rg.y;
        double v = 0.0;
        bool miss = false, shorth = false;
        for (unsigned int e = e0; e < e1; ++e) {
            const int slot = __ldg(s.acc_slot + e);
            const unsigned long long b = __ldg(s.acc_bits + e) & s.amask;
            const std::uint8_t fs = __ldg(s.fstate + slot);
            if (kValueOnly) {
                if (fs == 0) {
                    miss = true;
                    continue;
                }
                v = __dadd_rn(v, mass_on(s.P + static_cast<std::size_t>(slot) * s.V1 * s.K, s.K, b));
            } else {
                if (fs != 1) {
                    (fs == 2 ? shorth : miss) = true;
                    continue;
                }
                eq2_entry(s, slot, b, v);
            }
        }
        out[id] = v;
        if (miss || shorth) set_error(s.st, PBKV_EINVAL, miss ? kErrMissingForecast : kErrShortHorizon, id);
    }
}

// survival + gs table + validation of uploaded forecast rows (Forecast ctor,
// forecast.hpp:19-42).  gs[k] = gamma^k * s(k) with gamma^k by repeated
// multiplication and the product taken in the reference order (g * s),
// scoring.hpp:56-58, so that gs[k] * m equals (g * s(k)) * m bit for bit.
__global__ void __launch_bounds__(256) forecast_prepare_kernel(const double* stage, const long long* slots,
                                                               std::int64_t n, int H, int V1, int K, double gamma,
                                                               double* P, double* Pg, double* gs,
                                                               std::uint8_t* fstate, DevStatus* st) {
    // one warp per forecast row: lane k validates step k (agent-ordered sum,
    // forecast.hpp:25-34), the warp transposes the row into the agent-major
    // table, lane 0 runs the survival / gamma chain (forecast.hpp:35-41)
    const int lane = threadIdx.x & 31;
    const std::int64_t nw = (static_cast<std::int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (std::int64_t j = (blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x) >> 5; j < n; j += nw) {
        const double* p = stage + static_cast<std::size_t>(j) * H * V1;
        const long long slot = slots[j];
        int bad = 0;
        for (int k = lane; k < H; k += 32) {
            double sum = 0.0;
            for (int a = 0; a < V1; ++a) {
                const double v = p[k * V1 + a];
                if (v < -1e-12) {
                    bad = 1;
                    break;
                }
                sum = __dadd_rn(sum, v);
            }
            if (!bad && fabs(__dsub_rn(sum, 1.0)) > 1e-9) bad = 2;
        }
        // the first failing step wins, as in the ctor's loop
        const unsigned neg = __ballot_sync(0xffffffffu, bad == 1), off = __ballot_sync(0xffffffffu, bad == 2);
        if (neg | off) {
            if (lane == 0) {
                const int first = __ffs(neg | off) - 1;
                set_error(st, PBKV_EINVAL, ((neg >> first) & 1u) ? kErrForecastNegative : kErrForecastSum, j);
            }
            continue;
        }
        double* dst = P + static_cast<std::size_t>(slot) * K * V1;
        for (int idx = lane; idx < K * V1; idx += 32) {  // dst[a][k], coalesced stores
            const int a = idx / K, k = idx % K;
            dst[idx] = k < H ? p[k * V1 + a] : CUDART_NAN;  // horizon < K: unusable (NaN rows)
        }
        double* g = gs + static_cast<std::size_t>(slot) * K;
        if (lane == 0) {
            double surv = 1.0, gk = 1.0;
            for (int k = 0; k < K; ++k) {
                if (k < H) {
                    g[k] = __dmul_rn(gk, surv);
                    surv = __dmul_rn(surv, __dsub_rn(1.0, p[k * V1 + V1 - 1]));
                    if (surv < 0.0) surv = 0.0;
                } else {
                    g[k] = 0.0;
                }
                gk = __dmul_rn(gk, gamma);
            }
            fstate[slot] = H >= K ? 1 : 2;
        }
        __syncwarp();
        // one-agent Eq. 2 terms: mass_on of a single bit is 0.0 + P (forecast.hpp:66-67)
        double* dg = Pg + static_cast<std::size_t>(slot) * K * V1;
        for (int idx = lane; idx < K * V1; idx += 32) {
            const int a = idx / K, k = idx % K;
            dg[idx] = k < H ? __dmul_rn(g[k], __dadd_rn(0.0, p[k * V1 + a])) : CUDART_NAN;
        }
    }
}

__global__ void gather_f64_kernel(const double* src, const int* ids, std::int64_t n, double* dst) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
        dst[i] = src[ids[i]];
}

std::size_t chain_smem_bytes() {
    static bool init = false;
    const std::size_t b = sizeof(ChainSmem);
    if (!init) {
        PBKV_CUDA(cudaFuncSetAttribute(heavy_chain_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(b)));
        PBKV_CUDA(cudaFuncSetAttribute(heavy_chain_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(b)));
        PBKV_CUDA(cudaFuncSetAttribute(chain_sum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(b)));
        init = true;
    }
    return b;
}


}  // namespace

ScoreArgs make_score_args(Context& c, double* out) {
    ScoreArgs s;
    s.acc_rng = c.acc_rng.p;
    s.acc_slot = c.acc_slot.p;
    s.acc_bits = c.acc_bits.p;
    s.P = c.P.p;
    s.Pg = c.Pg.p;
    s.lslot = c.lslot.p;
    s.lbits = c.lbits.p;
    s.gs = c.gs.p;
    s.fstate = c.fstate.p;
    s.K = c.K;
    s.V1 = c.V1;
    s.amask = c.A >= 64 ? ~0ull : ((1ull << c.A) - 1ull);
    s.out = out;
    s.st = c.status.p;
    return s;
}

KeyArgs make_key_args(Context& c, int policy) {
    KeyArgs k;
    k.parent = c.parent.p;
    k.len = c.len.p;
    k.flags = c.flags.p;
    k.last = c.last.p;
    k.ever = c.ever.p;
    k.score_cached = c.score.p;
    k.acc_rng = c.acc_rng.p;
    k.acc_slot = c.acc_slot.p;
    k.acc_bits = c.acc_bits.p;
    k.rem_off = c.rem_off.p;
    k.rem_seq = c.rem_seq.p;
    k.rem_has = c.rem_has.p;
    k.keys = c.keys.p;
    k.eff = c.eff.p;
    k.sublock = c.sublock.p;
    k.W = c.W.p;
    k.C = c.C.p;
    k.rank = c.rank.p;
    k.missing = c.missing.p;
    k.st = c.status.p;
    k.policy = policy;
    return k;
}

void launch_forecast_prepare(Context& c, const double* stage, const long long* slots, std::int64_t n, int H) {
    forecast_prepare_kernel<<<grid_cap(n * 32, 256), 256, 0, c.stream>>>(stage, slots, n, H, c.V1, c.K, c.gamma,
                                                                        c.P.p, c.Pg.p, c.gs.p, c.fstate.p,
                                                                        c.status.p);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

// Eq. 2 for every node.  With write_keys the stage-3 per-node state (keys,
// eff, W, C, rank, missing) is produced in the same passes.
void launch_score_all(Context& c, double* out, bool write_keys, int policy, bool report_missing) {
    ScoreArgs s = make_score_args(c, out);
    KeyArgs ka = make_key_args(c, policy);
    const int rm = report_missing ? 1 : 0;
    // medium + heavy products and chains on the side stream, overlapped with the light pass
    const bool side = c.n_heavy + c.n_medium > 0;
    if (side) {
        PBKV_CUDA(cudaEventRecord(c.ev_fork, c.stream));
        PBKV_CUDA(cudaStreamWaitEvent(c.side, c.ev_fork, 0));
        PBKV_CUDA(cudaMemsetAsync(c.hmiss.p, 0, static_cast<std::size_t>(c.n_heavy + c.n_medium) * sizeof(unsigned int),
                                  c.side));
        heavy_products_kernel<<<grid_cap(c.n_hent * c.K, 256), 256, 0, c.side>>>(
            s, c.hent.p, c.hent_node.p, c.n_hent, c.hxs.p, c.hmiss.p, nullptr, static_cast<int>(c.n_heavy));
        PBKV_CUDA(cudaGetLastError());
        ++c.launches;
        if (c.n_medium > 0) {
            const unsigned int g = static_cast<unsigned int>((c.n_medium * 32 + 255) / 256);
            if (write_keys)
                medium_chain_kernel<true><<<g, 256, 0, c.side>>>(s, ka, c.medium.p, c.n_medium, c.n_heavy, c.hstart.p,
                                                                 c.hxs.p, c.hmiss.p, rm);
            else
                medium_chain_kernel<false><<<g, 256, 0, c.side>>>(s, ka, c.medium.p, c.n_medium, c.n_heavy,
                                                                  c.hstart.p, c.hxs.p, c.hmiss.p, rm);
            PBKV_CUDA(cudaGetLastError());
            ++c.launches;
        }
        if (c.n_heavy > 0) {
            const unsigned int hb = static_cast<unsigned int>(c.n_heavy);
            if (write_keys)
                heavy_chain_kernel<true><<<hb, kChainT, chain_smem_bytes(), c.side>>>(s, ka, c.heavy.p, c.hstart.p,
                                                                                   c.hxs.p, c.hmiss.p, rm);
            else
                heavy_chain_kernel<false><<<hb, kChainT, chain_smem_bytes(), c.side>>>(s, ka, c.heavy.p, c.hstart.p,
                                                                                    c.hxs.p, c.hmiss.p, rm);
            PBKV_CUDA(cudaGetLastError());
            ++c.launches;
        }
        PBKV_CUDA(cudaEventRecord(c.ev_join, c.side));
    }
    if (write_keys)
        launch_light<true>(c, s, ka, rm);
    else
        launch_light<false>(c, s, ka, rm);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
    if (side) PBKV_CUDA(cudaStreamWaitEvent(c.stream, c.ev_join, 0));
}

// skip_if (device): the kernel does nothing when *skip_if != 0 (run_select
// enqueues the clear before its synchronisation, unless the host-sort
// fallback -- which still needs the flags -- was taken)
void launch_set_deferred(Context& c, bool on, const int* skip_if) {
    if (c.n_heavy == 0) return;
    const int n = static_cast<int>(c.n_heavy);
    set_deferred_kernel<<<(n + 127) / 128, 128, 0, c.stream>>>(c.flags.p, c.keys.p, c.heavy.p, n, on ? 1 : 0,
                                                                  skip_if);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

void launch_decision_prologue(Context& c, bool defer, cudaStream_t st) {
    const int nh = defer ? static_cast<int>(c.n_heavy) : 0;
    const int nm = defer ? static_cast<int>(c.n_heavy + c.n_medium) : 0;
    if (defer) c.happrox.reserve(static_cast<std::size_t>(2 * c.n_heavy) + 2);
    const int n = std::max(1, std::max(nh, nm));
    decision_prologue_kernel<<<(n + 255) / 256, 256, 0, st>>>(c.status_pending ? nullptr : c.status.p, c.flags.p,
                                                                      c.keys.p, c.heavy.p, nh, defer ? 1 : 0, c.hmiss.p,
                                                                      nm, c.happrox.p);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

// Eq. 2 + keys for a decision with the heavy chains deferred: heavy nodes
// carry the kFlagDeferred bit (zero key, out of the order); their products
// and approximate sums are formed on the side stream; the exact chains run
// only if the fast-path check in select_core cannot place them.
void launch_score_decision(Context& c, int policy) {
    ScoreArgs s = make_score_args(c, c.score_rc.p);
    KeyArgs ka = make_key_args(c, policy);
    const bool side = c.n_heavy + c.n_medium > 0;
    // the light pass is enqueued first (every API call before it delays its
    // start); the side stream forks off the same point, has the higher
    // priority for SM slots, and joins after it.  The decision's prologue
    // (status reset, the deferral marks, hmiss / approx zeroed) runs at the
    // head of the side stream: the light pass reads none of it (no status
    // writes at report_missing 0, no keys of heavy nodes), the side stream's
    // kernels and the selection (after the join) read all of it.
    if (side) {
        PBKV_CUDA(cudaEventRecord(c.ev_fork, c.stream));
    } else {
        launch_decision_prologue(c, true, c.stream);
    }
    launch_light<true>(c, s, ka, 0);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
    if (side) {
        PBKV_CUDA(cudaStreamWaitEvent(c.side, c.ev_fork, 0));
        launch_decision_prologue(c, true, c.side);
        heavy_products_kernel<<<grid_cap(c.n_hent * c.K, 256), 256, 0, c.side>>>(
            s, c.hent.p, c.hent_node.p, c.n_hent, c.hxs.p, c.hmiss.p, c.happrox.p, static_cast<int>(c.n_heavy));
        PBKV_CUDA(cudaGetLastError());
        ++c.launches;
        if (c.n_medium > 0) {
            const unsigned int g = static_cast<unsigned int>((c.n_medium * 32 + 255) / 256);
            medium_chain_kernel<true><<<g, 256, 0, c.side>>>(s, ka, c.medium.p, c.n_medium, c.n_heavy, c.hstart.p,
                                                             c.hxs.p, c.hmiss.p, 0);
            PBKV_CUDA(cudaGetLastError());
            ++c.launches;
        }
        PBKV_CUDA(cudaEventRecord(c.ev_join, c.side));
        PBKV_CUDA(cudaStreamWaitEvent(c.stream, c.ev_join, 0));
    }
}

// Eq. 2 / Eq. 1 of an id list, results scattered into out[id]
void launch_score_ids(Context& c, const int* ids_dev, const int* h_ids, std::int64_t n, double* out, bool value_only) {
    ScoreArgs s = make_score_args(c, out);
    KeyArgs ka = make_key_args(c, PBKV_POLICY_HE);
    // classify on the host: ids with long chains go to the CTA chain kernel
    std::vector<int> longs;
    std::vector<int> shorts;
    const int K = value_only ? 1 : c.K;
    for (std::int64_t j = 0; j < n; ++j) {
        const int id = h_ids[j];
        const std::int64_t L = static_cast<std::int64_t>(c.h_entries[static_cast<std::size_t>(id)]) * K;
        (L > kMediumMaxElems ? longs : shorts).push_back(id);
    }
    if (!shorts.empty()) {
        c.ids2.reserve(shorts.size());
        PBKV_CUDA(cudaMemcpyAsync(c.ids2.p, shorts.data(), shorts.size() * sizeof(int), cudaMemcpyHostToDevice,
                                  c.stream));
        const std::int64_t m = static_cast<std::int64_t>(shorts.size());
        if (value_only)
            score_ids_kernel<true><<<grid_cap(m, 256), 256, 0, c.stream>>>(s, c.ids2.p, m, out);
        else
            score_ids_kernel<false><<<grid_cap(m, 256), 256, 0, c.stream>>>(s, c.ids2.p, m, out);
        PBKV_CUDA(cudaGetLastError());
        ++c.launches;
    }
    if (!longs.empty()) {
        c.ids3.reserve(longs.size());
        PBKV_CUDA(cudaMemcpyAsync(c.ids3.p, longs.data(), longs.size() * sizeof(int), cudaMemcpyHostToDevice,
                                  c.stream));
        const unsigned int g = static_cast<unsigned int>(longs.size());
        if (value_only)
            chain_kernel<false, true, false><<<g, kChainThreads, 0, c.stream>>>(s, ka, c.ids3.p, nullptr, nullptr,
                                                                                nullptr, 1);
        else
            chain_kernel<false, false, false><<<g, kChainThreads, 0, c.stream>>>(s, ka, c.ids3.p, nullptr, nullptr,
                                                                                 nullptr, 1);
        PBKV_CUDA(cudaGetLastError());
        ++c.launches;
    }
    (void)ids_dev;
}

void launch_chain_sum(Context& c, const double* x, const long long* off, int n_seg, double* out) {
    chain_sum_kernel<<<static_cast<unsigned int>(n_seg), kChainT, chain_smem_bytes(), c.stream>>>(x, off, out);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

void launch_gather_f64(Context& c, const double* src, const int* ids, std::int64_t n, double* dst) {
    gather_f64_kernel<<<grid_cap(n, 256), 256, 0, c.stream>>>(src, ids, n, dst);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

// Eq. 1 for the host-tier candidates is evaluated inside prefetch.cu with the
// same helpers; this hook keeps the value path for id lists.
}  // namespace pbkv
