// Stage 3 on sm_100a: hierarchical victim selection (policies.hpp:50-115) via
// its closed form:
//   order(eligible device nodes) = sort by (eff(n), d(n)),
//   eff(n) = argmax key over n's device subtree, d(n) = depth(eff) - depth(n),
//   victims = shortest prefix with sum(len) >= needed.
// The nodes sharing one eff value h ("chain of head h") form a contiguous
// ancestor path starting at h, so the order is: heads sorted by key, each
// followed by its chain in d order.  Pipeline:
//   keys (score.cu or keys_cached) -> lock marks -> eff (CAS walk-up) ->
//   weights (W[h] tokens, C[h] nodes, head list) -> weighted MSD radix select
//   on the head keys -> sort of the selected heads only -> chain scatter.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <cuda/std/tuple>

#include "common.cuh"

namespace pbkv {

using namespace dev;

KeyArgs make_key_args(Context& c, int policy);

namespace {

constexpr int kThreads = 256;
constexpr int kDigitBits = 11;
constexpr int kBins = 1 << kDigitBits;

unsigned int grid_cap(std::int64_t n, int block) {
    std::int64_t want = (n + block - 1) / block;
    const std::int64_t cap = 148LL * 16;
    if (want > cap) want = cap;
    return static_cast<unsigned int>(want < 1 ? 1 : want);
}

__global__ void __launch_bounds__(kThreads) keys_cached_kernel(KeyArgs ka, std::int64_t n_nodes) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n_nodes;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const int n = static_cast<int>(i);
        init_select_state(ka, n, false);
        if (n != 0 && (ka.flags[n] & kFlagTierMask) == PBKV_TIER_DEVICE) write_key(ka, n, ka.score_cached[n]);
    }
}

// A locked DEVICE node makes itself and all of its ancestors ineligible: in
// the greedy frontier (policies.hpp:56-79) it is never pushed, so no
// ancestor's virtual device-child count can reach zero.
__global__ void lock_kernel(const int* locked, std::int64_t n_locked, const int* parent, const std::uint8_t* flags,
                            int* sublock, std::int64_t n_nodes) {
    for (std::int64_t j = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; j < n_locked;
         j += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        int v = locked[j];
        if (v <= 0 || v >= n_nodes) continue;
        if ((flags[v] & kFlagTierMask) != PBKV_TIER_DEVICE) continue;
        while (v > 0) {
            if (atomicExch(&sublock[v], 1) == 1) break;
            v = parent[v];
        }
    }
}

// eff: every device node walks its key up the ancestor chain, CAS-ing the
// ancestors' argmax id; a walk stops at the first ancestor already holding a
// larger key (its holder carries it further), so eff ends as the exact
// subtree maximum.
__global__ void __launch_bounds__(kThreads) eff_kernel(const int* parent, const std::uint8_t* flags,
                                                       const Key2* keys, int* eff, std::int64_t n_nodes) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n_nodes;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const int n = static_cast<int>(i);
        if (n == 0 || (flags[n] & kFlagTierMask) != PBKV_TIER_DEVICE) continue;
        const Key2 km = load_key(keys, n);
        int p = parent[n];
        while (p > 0) {
            int cur = *reinterpret_cast<volatile int*>(&eff[p]);
            bool advanced = false;
            for (;;) {
                const Key2 kc = load_key(keys, cur);
                if (!key_less(kc, cur, km, n)) break;
                const int old = atomicCAS(&eff[p], cur, n);
                if (old == cur) {
                    advanced = true;
                    break;
                }
                cur = old;
            }
            if (!advanced) break;
            p = parent[p];
        }
    }
}

// selection state shared by the select kernels (device memory)
struct SelState {
    unsigned long long need_rem;   // tokens still needed beyond the selected heads
    unsigned long long total_tok;  // all eligible tokens
    unsigned long long n_L, n_L2;  // candidate list sizes (current, next)
    unsigned long long n_S;        // selected heads
    unsigned long long or_L[3], and_L[3];    // bitwise OR / AND of the current candidates' keys
    unsigned long long or_L2[3], and_L2[3];  // ... of the next candidates
    unsigned long long or_S[3], and_S[3];    // ... of the selected heads
    int lo_bit;       // digit = key bits [lo_bit, lo_bit + kDigitBits)
    int bucket;       // chosen digit value
    int take_all;     // eligible total < needed: every head selected
    int done;
    unsigned long long n_victims, freed;
    int shortfall;
    int cut_head;
};

__device__ __forceinline__ unsigned long long key_word(const Key2& k, int id, int w) {
    return w == 0 ? k.w0 : (w == 1 ? k.w1 : static_cast<unsigned long long>(static_cast<unsigned int>(id)));
}

// bits [lo, lo+n) of the 160-bit key (w0:64 | w1:64 | id:32), bit 0 = id LSB
__device__ __forceinline__ unsigned int key_bits(const Key2& k, int id, int lo, int n) {
    unsigned long long out = 0;
    for (int b = 0; b < n; ++b) {
        const int pos = lo + b;
        unsigned long long bit;
        if (pos < 32)
            bit = (static_cast<unsigned int>(id) >> pos) & 1u;
        else if (pos < 96)
            bit = (k.w1 >> (pos - 32)) & 1ull;
        else
            bit = (k.w0 >> (pos - 96)) & 1ull;
        out |= bit << b;
    }
    return static_cast<unsigned int>(out);
}

template <class Op>
__device__ __forceinline__ unsigned long long block_reduce_bits(unsigned long long v, Op op,
                                                                unsigned long long* sh /*[32]*/) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    const int nw = (blockDim.x + 31) >> 5;
    if (warp == 0) {
        v = lane < nw ? sh[lane] : sh[0];
        for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    }
    __syncthreads();
    return v;  // valid in warp 0
}

struct OrOp {
    __device__ unsigned long long operator()(unsigned long long a, unsigned long long b) const { return a | b; }
};
struct AndOp {
    __device__ unsigned long long operator()(unsigned long long a, unsigned long long b) const { return a & b; }
};

// token weight and node count of every chain, head list, eligible tokens,
// OR/AND of the head keys (first radix pass)
__global__ void __launch_bounds__(kThreads) weights_kernel(const int* len, const std::uint8_t* flags,
                                                           const int* sublock, const int* eff,
                                                           const std::uint8_t* missing, const Key2* keys,
                                                           unsigned long long* W, unsigned int* C, int* heads,
                                                           SelState* ss, DevStatus* st, std::int64_t n_nodes,
                                                           int he_recompute) {
    __shared__ unsigned long long sh[32];
    unsigned long long tok = 0;
    unsigned long long or3[3] = {0, 0, 0}, and3[3] = {~0ull, ~0ull, ~0ull};
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    for (std::int64_t base = blockIdx.x * static_cast<std::int64_t>(blockDim.x); base < n_nodes; base += stride) {
        const std::int64_t i = base + threadIdx.x;
        const int n = static_cast<int>(i);
        bool elig = false;
        int h = -1;
        if (i < n_nodes && n != 0 && (flags[n] & kFlagTierMask) == PBKV_TIER_DEVICE && !sublock[n]) {
            elig = true;
            if (missing[n] == 2) set_error(st, PBKV_EINVAL, kErrKvflowMissing, n);
            if (he_recompute && missing[n] && !(flags[n] & kFlagRetired))
                set_error(st, PBKV_EINVAL, kErrMissingForecast, n);
            h = eff[n];
            atomicAdd(&W[h], static_cast<unsigned long long>(len[n]));
            atomicAdd(&C[h], 1u);
            tok += static_cast<unsigned long long>(len[n]);
        }
        const bool head = elig && h == n;
        const long long slot = warp_append(&ss->n_L, head);
        if (head) {
            heads[slot] = n;
            const Key2 k = load_key(keys, n);
            for (int w = 0; w < 3; ++w) {
                const unsigned long long x = key_word(k, n, w);
                or3[w] |= x;
                and3[w] &= x;
            }
        }
    }
    using Red = cub::BlockReduce<unsigned long long, kThreads>;
    __shared__ typename Red::TempStorage tmp;
    const unsigned long long blk = Red(tmp).Sum(tok);
    if (threadIdx.x == 0 && blk) atomicAdd(&ss->total_tok, blk);
    for (int w = 0; w < 3; ++w) {
        const unsigned long long o = block_reduce_bits(or3[w], OrOp(), sh);
        const unsigned long long a = block_reduce_bits(and3[w], AndOp(), sh);
        if (threadIdx.x == 0) {
            if (o) atomicOr(&ss->or_L[w], o);
            if (~a) atomicAnd(&ss->and_L[w], a);
        }
    }
}

__device__ __forceinline__ int top_varying_bit(const unsigned long long* o, const unsigned long long* a) {
    const unsigned long long v0 = o[0] ^ a[0], v1 = o[1] ^ a[1], v2 = (o[2] ^ a[2]) & 0xffffffffull;
    if (v0) return 96 + 63 - __clzll(static_cast<long long>(v0));
    if (v1) return 32 + 63 - __clzll(static_cast<long long>(v1));
    if (v2) return 63 - __clzll(static_cast<long long>(v2));
    return -1;
}

// weighted histogram of the next digit over the candidate list
__global__ void __launch_bounds__(kThreads) hist_kernel(const int* L, const Key2* keys, const unsigned long long* W,
                                                        SelState* ss, unsigned long long* hist) {
    __shared__ unsigned long long h[kBins];
    for (int b = threadIdx.x; b < kBins; b += blockDim.x) h[b] = 0;
    __syncthreads();
    const unsigned long long n = ss->n_L;
    const int top = top_varying_bit(ss->or_L, ss->and_L);
    const int lo = top - kDigitBits + 1 < 0 ? 0 : top - kDigitBits + 1;
    for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
        const int x = L[i];
        const unsigned int d = key_bits(load_key(keys, x), x, lo, kDigitBits);
        atomicAdd(&h[d], W[x]);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < kBins; b += blockDim.x)
        if (h[b]) atomicAdd(&hist[b], h[b]);
}

// single CTA: the bucket where the cumulative weight reaches need_rem
__global__ void __launch_bounds__(1024) pick_kernel(SelState* ss, unsigned long long* hist) {
    using Scan = cub::BlockScan<unsigned long long, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ int pick;
    const int top = top_varying_bit(ss->or_L, ss->and_L);
    const int lo = top - kDigitBits + 1 < 0 ? 0 : top - kDigitBits + 1;
    constexpr int kPer = kBins / 1024;
    unsigned long long v[kPer], sum = 0;
    for (int j = 0; j < kPer; ++j) {
        v[j] = hist[threadIdx.x * kPer + j];
        sum += v[j];
    }
    unsigned long long excl;
    Scan(tmp).ExclusiveSum(sum, excl);
    if (threadIdx.x == 0) pick = -1;
    __syncthreads();
    const unsigned long long need = ss->need_rem;
    unsigned long long run = excl;
    for (int j = 0; j < kPer; ++j) {
        if (run < need && run + v[j] >= need) {
            pick = threadIdx.x * kPer + j;
            ss->need_rem = need - run;
        }
        run += v[j];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        ss->lo_bit = lo;
        ss->bucket = pick;  // always found: total of L >= need_rem
        ss->n_L2 = 0;
        for (int w = 0; w < 3; ++w) {
            ss->or_L2[w] = 0;
            ss->and_L2[w] = ~0ull;
        }
    }
    for (int b = threadIdx.x; b < kBins; b += blockDim.x) hist[b] = 0;  // ready for the next pass
}

// split the candidates: below the bucket -> selected S, in the bucket -> L2
__global__ void __launch_bounds__(kThreads) compact_kernel(const int* L, const Key2* keys, SelState* ss, int* L2,
                                                           int* S) {
    __shared__ unsigned long long sh[32];
    const unsigned long long n = ss->n_L;
    const int lo = ss->lo_bit, b = ss->bucket;
    unsigned long long orS[3] = {0, 0, 0}, andS[3] = {~0ull, ~0ull, ~0ull};
    unsigned long long orL[3] = {0, 0, 0}, andL[3] = {~0ull, ~0ull, ~0ull};
    const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
    for (unsigned long long base = blockIdx.x * static_cast<unsigned long long>(blockDim.x); base < n;
         base += stride) {
        const unsigned long long i = base + threadIdx.x;
        bool below = false, same = false;
        int x = 0;
        Key2 k{0, 0};
        if (i < n) {
            x = L[i];
            k = load_key(keys, x);
            const int d = static_cast<int>(key_bits(k, x, lo, kDigitBits));
            below = d < b;
            same = d == b;
        }
        const long long s1 = warp_append(&ss->n_S, below);
        const long long s2 = warp_append(&ss->n_L2, same);
        if (below) {
            S[s1] = x;
            for (int w = 0; w < 3; ++w) {
                orS[w] |= key_word(k, x, w);
                andS[w] &= key_word(k, x, w);
            }
        }
        if (same) {
            L2[s2] = x;
            for (int w = 0; w < 3; ++w) {
                orL[w] |= key_word(k, x, w);
                andL[w] &= key_word(k, x, w);
            }
        }
    }
    for (int w = 0; w < 3; ++w) {
        unsigned long long v = block_reduce_bits(orS[w], OrOp(), sh);
        if (threadIdx.x == 0 && v) atomicOr(&ss->or_S[w], v);
        v = block_reduce_bits(andS[w], AndOp(), sh);
        if (threadIdx.x == 0 && ~v) atomicAnd(&ss->and_S[w], v);
        v = block_reduce_bits(orL[w], OrOp(), sh);
        if (threadIdx.x == 0 && v) atomicOr(&ss->or_L2[w], v);
        v = block_reduce_bits(andL[w], AndOp(), sh);
        if (threadIdx.x == 0 && ~v) atomicAnd(&ss->and_L2[w], v);
    }
}

// next pass: L2 -> L (swap of the OR/AND accumulators; lists swapped by host)
__global__ void advance_kernel(SelState* ss) {
    ss->n_L = ss->n_L2;
    for (int w = 0; w < 3; ++w) {
        ss->or_L[w] = ss->or_L2[w];
        ss->and_L[w] = ss->and_L2[w];
    }
}

// the last candidate is the cut head: append it to S
__global__ void finish_select_kernel(const int* L, const Key2* keys, SelState* ss, int* S) {
    const int x = L[0];
    const Key2 k = load_key(keys, x);
    S[ss->n_S] = x;
    ss->n_S += 1;
    for (int w = 0; w < 3; ++w) {
        ss->or_S[w] |= key_word(k, x, w);
        ss->and_S[w] &= key_word(k, x, w);
    }
    ss->cut_head = x;
}

// sort keys for the selected heads: the varying bits of (w0, w1, id) packed
// into one uint64 (order-preserving bit extraction) when they fit
__global__ void pack_keys_kernel(const int* S, const Key2* keys, const SelState* ss, unsigned long long* out,
                                 int* ids) {
    const unsigned long long n = ss->n_S;
    const unsigned long long v0 = ss->or_S[0] ^ ss->and_S[0];
    const unsigned long long v1 = ss->or_S[1] ^ ss->and_S[1];
    const unsigned long long v2 = (ss->or_S[2] ^ ss->and_S[2]) & 0xffffffffull;
    for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
        const int x = S[i];
        const Key2 k = load_key(keys, x);
        unsigned long long r = 0;
        auto ext = [&](unsigned long long word, unsigned long long mask) {
            while (mask) {
                const int b = 63 - __clzll(static_cast<long long>(mask));
                r = (r << 1) | ((word >> b) & 1ull);
                mask &= ~(1ull << b);
            }
        };
        ext(k.w0, v0);
        ext(k.w1, v1);
        ext(static_cast<unsigned long long>(static_cast<unsigned int>(x)), v2);
        out[i] = r;
        ids[i] = x;
    }
}

__global__ void gather_headkeys_kernel(const int* S, const Key2* keys, const SelState* ss, HeadKey* out) {
    const unsigned long long n = ss->n_S;
    for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
        const int x = S[i];
        const Key2 k = load_key(keys, x);
        out[i] = HeadKey{k.w0, k.w1, static_cast<unsigned int>(x)};
    }
}

__global__ void heads_from_hk_kernel(const HeadKey* hk, const SelState* ss, int* out) {
    const unsigned long long n = ss->n_S;
    for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<unsigned long long>(gridDim.x) * blockDim.x)
        out[i] = static_cast<int>(hk[i].id);
}

// rank of every selected head and its chain size in sorted order
__global__ void rank_kernel(const int* sorted, const unsigned int* C, const SelState* ss, int* rank,
                            unsigned long long* cnt) {
    const unsigned long long n = ss->n_S;
    for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
        const int h = sorted[i];
        rank[h] = static_cast<int>(i);
        cnt[i] = C[h];
    }
}

// every eligible node of a selected chain lands at start[rank(head)] + d
__global__ void __launch_bounds__(kThreads) scatter_kernel(const std::uint8_t* flags, const int* sublock,
                                                           const int* eff, const int* rank, const int* depth,
                                                           const unsigned long long* start, int* out,
                                                           std::int64_t n_nodes) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n_nodes;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const int n = static_cast<int>(i);
        if (n == 0 || (flags[n] & kFlagTierMask) != PBKV_TIER_DEVICE || sublock[n]) continue;
        const int h = eff[n];
        const int r = rank[h];
        if (r < 0) continue;
        out[start[r] + static_cast<unsigned long long>(depth[h] - depth[n])] = n;
    }
}

// the cut inside the last (cut) chain; freed / shortfall
__global__ void cut_kernel(const int* victims, const int* len, const unsigned long long* start,
                           const unsigned int* C, SelState* ss, long long needed, long long* result) {
    const unsigned long long nS = ss->n_S;
    if (ss->take_all) {
        const unsigned long long nv = start[nS - 1] + C[ss->cut_head];
        ss->n_victims = nv;
        ss->freed = ss->total_tok;
    } else {
        const unsigned long long s0 = start[nS - 1];
        const unsigned int c = C[ss->cut_head];
        const unsigned long long need = ss->need_rem;
        const unsigned long long below = static_cast<unsigned long long>(needed) - need;
        unsigned long long acc = 0, j = 0;
        for (; j < c; ++j) {
            acc += static_cast<unsigned long long>(len[victims[s0 + j]]);
            if (acc >= need) break;
        }
        ss->n_victims = s0 + j + 1;
        ss->freed = below + acc;
    }
    ss->shortfall = ss->freed < static_cast<unsigned long long>(needed) ? 1 : 0;
    result[0] = static_cast<long long>(ss->n_victims);
    result[1] = static_cast<long long>(ss->freed);
    result[2] = ss->shortfall;
}

__global__ void init_state_kernel(SelState* ss, long long needed) {
    SelState z{};
    z.need_rem = static_cast<unsigned long long>(needed);
    for (int w = 0; w < 3; ++w) {
        z.and_L[w] = ~0ull;
        z.and_L2[w] = ~0ull;
        z.and_S[w] = ~0ull;
    }
    z.cut_head = -1;
    *ss = z;
}

// take-all: every head is selected (eligible tokens < needed)
__global__ void take_all_kernel(SelState* ss) {
    ss->take_all = 1;
    ss->n_S = ss->n_L;
    for (int w = 0; w < 3; ++w) {
        ss->or_S[w] = ss->or_L[w];
        ss->and_S[w] = ss->and_L[w];
    }
}

// after sorting in take-all mode the cut head is the last head
__global__ void set_last_head_kernel(const int* sorted, SelState* ss) { ss->cut_head = sorted[ss->n_S - 1]; }

}  // namespace

struct HeadDecomposer {
    __host__ __device__ ::cuda::std::tuple<unsigned long long&, unsigned long long&, unsigned int&> operator()(
        HeadKey& k) const {
        return {k.w0, k.w1, k.id};
    }
};

std::size_t sel_state_bytes() { return sizeof(SelState); }

void launch_keys_cached(Context& c, int policy) {
    KeyArgs ka = make_key_args(c, policy);
    keys_cached_kernel<<<grid_cap(c.n, kThreads), kThreads, 0, c.stream>>>(ka, c.n);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

void launch_lock_eff(Context& c, const int* locked_dev, std::int64_t n_locked) {
    if (n_locked > 0) {
        lock_kernel<<<grid_for(n_locked, kThreads), kThreads, 0, c.stream>>>(locked_dev, n_locked, c.parent.p,
                                                                            c.flags.p, c.sublock.p, c.n);
        PBKV_CUDA(cudaGetLastError());
        ++c.launches;
    }
    eff_kernel<<<grid_cap(c.n, kThreads), kThreads, 0, c.stream>>>(c.parent.p, c.flags.p, c.keys.p, c.eff.p, c.n);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

// Runs weights -> radix select -> sort -> scatter -> cut.  Victims land in
// c.vid_out[0..n); result_dev gets {n_victims, freed, shortfall}.  Host
// synchronisations: one per radix pass (candidate count) and one before the
// head sort (its size).  Returns the device status checked by the caller.
SelectCounts run_select(Context& c, std::int64_t needed, bool he_recompute, long long* result_dev) {
    SelState* ss = reinterpret_cast<SelState*>(c.selstate.p);
    SelState* hs = reinterpret_cast<SelState*>(c.hselstate.p);
    init_state_kernel<<<1, 1, 0, c.stream>>>(ss, needed);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
    weights_kernel<<<grid_cap(c.n, kThreads), kThreads, 0, c.stream>>>(
        c.len.p, c.flags.p, c.sublock.p, c.eff.p, c.missing.p, c.keys.p, c.W.p, c.C.p, c.heads.p, ss, c.status.p, c.n,
        he_recompute ? 1 : 0);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
    PBKV_CUDA(cudaMemcpyAsync(hs, ss, sizeof(SelState), cudaMemcpyDeviceToHost, c.stream));
    check_status(c);  // synchronises
    SelectCounts out;
    if (hs->n_L == 0) {  // nothing evictable
        const long long z[3] = {0, 0, 1};
        PBKV_CUDA(cudaMemcpyAsync(c.hcounters.p + 8, z, sizeof z, cudaMemcpyHostToDevice, c.stream));
        if (result_dev)
            PBKV_CUDA(cudaMemcpyAsync(result_dev, c.hcounters.p + 8, sizeof z, cudaMemcpyHostToDevice, c.stream));
        out.n_victims = 0;
        out.freed = 0;
        out.shortfall = 1;
        return out;
    }
    int* L = c.heads.p;
    int* L2 = c.listB.p;
    int* S = c.listS.p;
    const bool take_all = hs->total_tok < static_cast<unsigned long long>(needed);
    if (take_all) {
        take_all_kernel<<<1, 1, 0, c.stream>>>(ss);
        PBKV_CUDA(cudaGetLastError());
        ++c.launches;
        S = L;
    } else {
        PBKV_CUDA(cudaMemsetAsync(c.hist.p, 0, kBins * sizeof(unsigned long long), c.stream));
        unsigned long long nL = hs->n_L;
        for (int pass = 0; pass < 32 && nL > 1; ++pass) {
            hist_kernel<<<grid_cap(static_cast<std::int64_t>(nL), kThreads), kThreads, 0, c.stream>>>(L, c.keys.p,
                                                                                                     c.W.p, ss,
                                                                                                     c.hist.p);
            pick_kernel<<<1, 1024, 0, c.stream>>>(ss, c.hist.p);
            compact_kernel<<<grid_cap(static_cast<std::int64_t>(nL), kThreads), kThreads, 0, c.stream>>>(
                L, c.keys.p, ss, L2, S);
            advance_kernel<<<1, 1, 0, c.stream>>>(ss);
            PBKV_CUDA(cudaGetLastError());
            c.launches += 4;
            PBKV_CUDA(cudaMemcpyAsync(&hs->n_L, &ss->n_L, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                      c.stream));
            PBKV_CUDA(cudaStreamSynchronize(c.stream));
            nL = hs->n_L;
            std::swap(L, L2);
        }
        finish_select_kernel<<<1, 1, 0, c.stream>>>(L, c.keys.p, ss, S);
        PBKV_CUDA(cudaGetLastError());
        ++c.launches;
    }
    PBKV_CUDA(cudaMemcpyAsync(hs, ss, sizeof(SelState), cudaMemcpyDeviceToHost, c.stream));
    PBKV_CUDA(cudaStreamSynchronize(c.stream));
    const std::int64_t nS = static_cast<std::int64_t>(hs->n_S);
    // ---- sort the selected heads by key ----------------------------------------
    int nbits = 0;
    for (int w = 0; w < 3; ++w) {
        unsigned long long v = hs->or_S[w] ^ hs->and_S[w];
        if (w == 2) v &= 0xffffffffull;
        nbits += __builtin_popcountll(v);
    }
    c.sortk_in.reserve(nS);
    c.sortk_out.reserve(nS);
    c.sorti_in.reserve(nS);
    c.sorti_out.reserve(nS);
    c.cnt.reserve(nS + 1);
    c.vid_out.reserve(c.n + 1);
    int* sorted = c.sorti_out.p;
    if (nS == 1) {
        PBKV_CUDA(cudaMemcpyAsync(sorted, S, sizeof(int), cudaMemcpyDeviceToDevice, c.stream));
    } else if (nbits <= 64) {
        pack_keys_kernel<<<grid_cap(nS, kThreads), kThreads, 0, c.stream>>>(S, c.keys.p, ss, c.sortk_in.p,
                                                                           c.sorti_in.p);
        PBKV_CUDA(cudaGetLastError());
        ++c.launches;
        std::size_t b = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, b, c.sortk_in.p, c.sortk_out.p, c.sorti_in.p, c.sorti_out.p,
                                        static_cast<int>(nS), 0, nbits > 0 ? nbits : 1);
        c.cub_tmp.reserve(b);
        ++c.lib_calls;
        PBKV_CUDA(cub::DeviceRadixSort::SortPairs(c.cub_tmp.p, b, c.sortk_in.p, c.sortk_out.p, c.sorti_in.p,
                                                  c.sorti_out.p, static_cast<int>(nS), 0, nbits > 0 ? nbits : 1,
                                                  c.stream));
    } else {
        c.hk_in.reserve(nS);
        c.hk_out.reserve(nS);
        gather_headkeys_kernel<<<grid_cap(nS, kThreads), kThreads, 0, c.stream>>>(S, c.keys.p, ss, c.hk_in.p);
        PBKV_CUDA(cudaGetLastError());
        ++c.launches;
        std::size_t b = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, b, c.hk_in.p, c.hk_out.p, static_cast<int>(nS), HeadDecomposer{});
        c.cub_tmp.reserve(b);
        ++c.lib_calls;
        PBKV_CUDA(cub::DeviceRadixSort::SortKeys(c.cub_tmp.p, b, c.hk_in.p, c.hk_out.p, static_cast<int>(nS),
                                                 HeadDecomposer{}, c.stream));
        heads_from_hk_kernel<<<grid_cap(nS, kThreads), kThreads, 0, c.stream>>>(c.hk_out.p, ss, sorted);
        PBKV_CUDA(cudaGetLastError());
        ++c.launches;
    }
    if (take_all) {
        set_last_head_kernel<<<1, 1, 0, c.stream>>>(sorted, ss);
        PBKV_CUDA(cudaGetLastError());
        ++c.launches;
    }
    // ---- chain placement ----------------------------------------------------------
    rank_kernel<<<grid_cap(nS, kThreads), kThreads, 0, c.stream>>>(sorted, c.C.p, ss, c.rank.p, c.cnt.p);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
    {
        std::size_t b = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, b, c.cnt.p, c.cnt.p, static_cast<int>(nS));
        c.cub_tmp.reserve(b);
        ++c.lib_calls;
        PBKV_CUDA(cub::DeviceScan::ExclusiveSum(c.cub_tmp.p, b, c.cnt.p, c.cnt.p, static_cast<int>(nS), c.stream));
    }
    scatter_kernel<<<grid_cap(c.n, kThreads), kThreads, 0, c.stream>>>(c.flags.p, c.sublock.p, c.eff.p, c.rank.p,
                                                                       c.depth.p, c.cnt.p, c.vid_out.p, c.n);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
    long long* res = result_dev ? result_dev : c.counters.p + 8;
    cut_kernel<<<1, 1, 0, c.stream>>>(c.vid_out.p, c.len.p, c.cnt.p, c.C.p, ss, needed, res);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
    PBKV_CUDA(cudaMemcpyAsync(c.hcounters.p + 8, res, 3 * sizeof(long long), cudaMemcpyDeviceToHost, c.stream));
    PBKV_CUDA(cudaStreamSynchronize(c.stream));
    out.n_victims = c.hcounters.p[8];
    out.freed = c.hcounters.p[9];
    out.shortfall = static_cast<int>(c.hcounters.p[10]);
    return out;
}

}  // namespace pbkv
