// Stage 3 on sm_100a: hierarchical victim selection (policies.hpp:50-115) via
// its closed form:
//   order(eligible device nodes) = sort by (eff(n), d(n)),
//   eff(n) = argmax key over n's device subtree, d(n) = depth(eff) - depth(n),
//   victims = shortest prefix with sum(len) >= needed.
// The nodes sharing one eff value h ("chain of head h") form a contiguous
// ancestor path starting at h, so the order is: heads sorted by key, each
// followed by its chain in d order.
//
// The whole selection after the keys is ONE persistent kernel (two 512-thread
// CTAs per SM, co-resident by cooperative launch, phases separated by grid
// barriers):
//   lock marks + eff (queued CAS walk-ups) + the small-cut bound from a node
//   sample -> chains (scatter-added weight W and size C per head) ->
//   small-cut path: the heads at or below the bound bucketed by one 9-bit
//   digit and ranked in place, each selected head scattering its own chain;
//   or the full radix path: weighted MSD radix select on the head keys
//   (11-bit digits at the top varying bit of the surviving candidates),
//   heads below the chosen digit placed into their digit's bucket of the
//   selected list S -> oversized buckets split in place (refine_buckets) ->
//   every bucket ranked (warp sorts <= 32, rank-counting tasks <= 256) ->
//   chain starts (scan of chain sizes) -> chain scatter -> cut.
// No host round trip.  The CUB device sort below the kernel is the last
// resort of a refinement round whose per-CTA slices would span more than
// kRfLoc buckets (tens of millions of selected heads).
#include <cooperative_groups.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <cuda/std/tuple>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace pbkv {

using namespace dev;

KeyArgs make_key_args(Context& c, int policy);

namespace {

constexpr int kThreads = 256;
constexpr int kPThreads = 512;  // persistent CTA (two per SM)
constexpr int kDigitBits = 11;
constexpr int kBins = 1 << kDigitBits;
constexpr int kMaxPasses = 16;
constexpr int kBucketCap = 4096;  // bucket sorted by one CTA in shared memory
constexpr int kScanIPT = 8;       // chain-start scan: items per thread per chunk
// small-cut path: a node sample bounds the cut from above;
// the low heads are bucketed by a 9-bit digit (one bin per thread of the
// layout scan)
constexpr int kSBits = 9;           // digit of the small path (512 bins, one per layout thread) ...
constexpr int kSBitsWide = 11;      // ... or 2048 bins when the low list is long
constexpr unsigned long long kSWideAt = 65536;  // low heads from which the wide digit is used
constexpr int kChunkS = 512 / 8;    // small-path rank task: 64 heads, 8 threads each (kPThreads = 512)
constexpr int kSamp = 2048;            // sample records (the eff phase appends ~1024)
constexpr unsigned int kSampTarget = 1024;
constexpr long long kSmallMax = 1 << 18;  // estimated heads below the bound for the small path

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
        ka.W[n] = 0;
        ka.C[n] = 0;
        if (n != 0 && (ka.flags[n] & kFlagTierMask) == PBKV_TIER_DEVICE) write_key(ka, n, ka.score_cached[n]);
        else reinterpret_cast<ulonglong2*>(ka.keys)[n] = make_ulonglong2(0ull, 0ull);  // defined for batched loads
    }
}

// selection state (device memory)
struct SelState {
    unsigned long long need_final;  // tokens needed from the cut chain
    unsigned long long total_tok;   // all eligible tokens
    unsigned long long n_L[2];      // candidate list sizes by pass parity
    unsigned long long or_L[2][3], and_L[2][3];
    unsigned long long n_S;
    unsigned int n_big;  // buckets of S sorted by chunked rank counting
    unsigned long long or_S[3], and_S[3];
    int n_pass, take_all, host_sort, s_is_heads;
    int cut_head, max_bucket;
    unsigned long long n_victims, freed;
    int shortfall, n_ts;
    unsigned int low_overflow;  // a CTA's low buffer overflowed: no small path
    unsigned int small_done;    // S1 CTAs finished (the last one lays out the buckets)
    unsigned long long n_heads_seen;  // heads counted by the chains phase in small-cut mode
    unsigned int small_ok;      // 1 the small path proceeds, 2 it is abandoned
    unsigned int n_task;        // rank tasks of the small path's big buckets
    int bound_id;               // small-cut bound (key, id); -1: no small path
    unsigned long long bound_w0, bound_w1;
    int path;                   // 0 full radix path, 1 small-cut path, 2 small path abandoned
    unsigned long long n_low;   // heads at or below the sample bound
    unsigned long long or_low[3], and_low[3];
    unsigned long long est_low; // the sample's estimate of n_low (diagnostics)
    unsigned int n_rf[2];       // oversized buckets being refined, by round parity
    unsigned int n_rsmall;      // pieces of <= 32 heads the refinement produced
    unsigned int rf_rounds;     // refinement rounds run (diagnostics)
    unsigned long long ts[40];  // %globaltimer after each phase (diagnostics)
    unsigned long long dbg[8];  // per-CTA maxima of phase work (diagnostics)
    unsigned long long dbg2[4]; // small path: S1 histogram (max CTA), S1 layout (last CTA) (diagnostics)
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// stores only (a load of the counter would stall thread 0 while the grid waits on it)
__device__ __forceinline__ void stamp(SelState* ss, int& nts) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && nts < 40) {
        ss->ts[nts] = gtimer();
        ss->n_ts = ++nts;
    }
}

__device__ __forceinline__ unsigned long long key_word(const Key2& k, int id, int w) {
    return w == 0 ? k.w0 : (w == 1 ? k.w1 : static_cast<unsigned long long>(static_cast<unsigned int>(id)));
}

// bits [lo, lo+n) of the 160-bit key (w0:64 | w1:64 | id:32), bit 0 = id LSB
__device__ __forceinline__ unsigned int key_bits(const Key2& k, int id, int lo, int n) {
    unsigned long long win;
    if (lo >= 96) {
        win = k.w0 >> (lo - 96);
    } else if (lo >= 32) {
        const int s = lo - 32;
        win = (k.w1 >> s) | (s ? (k.w0 << (64 - s)) : 0ull);
    } else {
        win = (static_cast<unsigned long long>(static_cast<unsigned int>(id)) >> lo) | (k.w1 << (32 - lo));
    }
    return static_cast<unsigned int>(win & ((1ull << n) - 1ull));
}

// cross-CTA state is read through L2 (ld.global.cg): the barrier orders the
// writes but does not invalidate L1
__device__ __forceinline__ int top_varying_bit_cg(const unsigned long long* o_, const unsigned long long* a_) {
    unsigned long long o[3], a[3];
    for (int w = 0; w < 3; ++w) {
        o[w] = __ldcg(o_ + w);
        a[w] = __ldcg(a_ + w);
    }
    const unsigned long long v0 = o[0] ^ a[0], v1 = o[1] ^ a[1], v2 = (o[2] ^ a[2]) & 0xffffffffull;
    if (v0) return 96 + 63 - __clzll(static_cast<long long>(v0));
    if (v1) return 32 + 63 - __clzll(static_cast<long long>(v1));
    if (v2) return 63 - __clzll(static_cast<long long>(v2));
    return -1;
}

template <class Op>
__device__ __forceinline__ unsigned long long block_reduce_bits(unsigned long long v, Op op,
                                                                unsigned long long* sh /*[32]*/) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    const int nw = (blockDim.x + 31) >> 5;
    if (warp == 0) {
        v = lane < nw ? sh[lane] : Op::identity();
        for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    }
    return v;  // valid in warp 0
}

struct OrOp {
    __device__ static unsigned long long identity() { return 0ull; }
    __device__ unsigned long long operator()(unsigned long long a, unsigned long long b) const { return a | b; }
};
struct AndOp {
    __device__ static unsigned long long identity() { return ~0ull; }
    __device__ unsigned long long operator()(unsigned long long a, unsigned long long b) const { return a & b; }
};
struct SumOp {
    __device__ static unsigned long long identity() { return 0ull; }
    __device__ unsigned long long operator()(unsigned long long a, unsigned long long b) const { return a + b; }
};
struct MaxOp {
    __device__ static unsigned long long identity() { return 0ull; }
    __device__ unsigned long long operator()(unsigned long long a, unsigned long long b) const { return a > b ? a : b; }
};

__device__ __forceinline__ void flush_orand(const unsigned long long* or3, const unsigned long long* and3,
                                            unsigned long long* gor, unsigned long long* gand,
                                            unsigned long long* sh) {
    for (int w = 0; w < 3; ++w) {
        const unsigned long long o = block_reduce_bits(or3[w], OrOp(), sh);
        if (threadIdx.x == 0 && o) atomicOr(&gor[w], o);
        const unsigned long long a = block_reduce_bits(and3[w], AndOp(), sh);
        if (threadIdx.x == 0 && ~a) atomicAnd(&gand[w], a);
    }
}

// CTA-aggregated append: one global atomic per CTA and call (a grid-wide
// stream of warp-level atomics on one counter serialises in its L2 slice).
// Must be called by every thread of the CTA.
__device__ __forceinline__ long long block_append(unsigned long long* counter, bool pred, unsigned int* wcount,
                                                  unsigned long long* base_sh) {
    const unsigned mask = __ballot_sync(0xffffffffu, pred);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane == 0) wcount[warp] = static_cast<unsigned int>(__popc(mask));
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int s = 0;
        for (int w = 0; w < nw; ++w) {
            const unsigned int c = wcount[w];
            wcount[w] = s;
            s += c;
        }
        *base_sh = s ? atomicAdd(counter, static_cast<unsigned long long>(s)) : 0ull;
    }
    __syncthreads();
    const long long slot =
        pred ? static_cast<long long>(*base_sh + wcount[warp] + __popc(mask & ((1u << lane) - 1u))) : -1;
    __syncthreads();
    return slot;
}

// exclusive prefix of one value per thread over the CTA; *total = the sum
__device__ __forceinline__ unsigned int block_excl_u32(unsigned int v, unsigned long long* sh, unsigned int* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    unsigned int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    __syncthreads();
    if (lane == 31) sh[w] = inc;
    __syncthreads();
    if (w == 0) {
        const unsigned int s = lane < nw ? static_cast<unsigned int>(sh[lane]) : 0u;
        unsigned int si = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned int t = __shfl_up_sync(0xffffffffu, si, o);
            if (lane >= o) si += t;
        }
        if (lane < nw) sh[lane] = si - s;
        if (lane == 31) sh[31] = si;
    }
    __syncthreads();
    const unsigned int r = static_cast<unsigned int>(sh[w]) + inc - v;
    if (total) *total = static_cast<unsigned int>(sh[31]);
    __syncthreads();
    return r;
}

// order-preserving packing of the varying bits of (w0, w1, id) into 64 bits;
// the masks are walked a run of consecutive set bits at a time (the varying
// bits are typically one or two runs per word: timestamp and id low bits)
__device__ __forceinline__ unsigned long long pack_key(const Key2& k, int id, unsigned long long v0,
                                                       unsigned long long v1, unsigned long long v2) {
    unsigned long long r = 0;
    auto ext = [&](unsigned long long word, unsigned long long mask) {
        while (mask) {
            const int hi = 63 - __clzll(static_cast<long long>(mask));
            // run of ones ending at bit hi (downward)
            const unsigned long long above_cleared = ~mask & ((hi == 63) ? ~0ull : ((1ull << (hi + 1)) - 1ull));
            const int lo = above_cleared ? 64 - __clzll(static_cast<long long>(above_cleared)) : 0;
            const int len = hi - lo + 1;
            const unsigned long long run = (len == 64) ? ~0ull : ((1ull << len) - 1ull);
            r = (len == 64 ? 0ull : (r << len)) | ((word >> lo) & run);
            mask &= ~(run << lo);
        }
    };
    ext(k.w0, v0);
    ext(k.w1, v1);
    ext(static_cast<unsigned long long>(static_cast<unsigned int>(id)), v2);
    return r;
}

// the same packing into 128 bits (hi, lo) for keys with 64..128 varying bits
__device__ __forceinline__ void pack_key2(const Key2& k, int id, unsigned long long v0, unsigned long long v1,
                                          unsigned long long v2, unsigned long long& hi, unsigned long long& lo) {
    hi = 0;
    lo = 0;
    auto ext = [&](unsigned long long word, unsigned long long mask) {
        while (mask) {
            const int h = 63 - __clzll(static_cast<long long>(mask));
            const unsigned long long above_cleared = ~mask & ((h == 63) ? ~0ull : ((1ull << (h + 1)) - 1ull));
            const int l = above_cleared ? 64 - __clzll(static_cast<long long>(above_cleared)) : 0;
            const int len = h - l + 1;
            const unsigned long long run = (len == 64) ? ~0ull : ((1ull << len) - 1ull);
            const unsigned long long bits = (word >> l) & run;
            if (len == 64) {
                hi = lo;
                lo = bits;
            } else {
                hi = (hi << len) | (lo >> (64 - len));
                lo = (lo << len) | bits;
            }
            mask &= ~(run << l);
        }
    };
    ext(k.w0, v0);
    ext(k.w1, v1);
    ext(static_cast<unsigned long long>(static_cast<unsigned int>(id)), v2);
}

// one sampled eligible node (eff phase): key, id, token length
struct SampRec {
    unsigned long long w0, w1;
    int id, len;
};

__device__ __forceinline__ unsigned int mix32(unsigned int x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

struct SelArgs {
    const int* parent;
    const int* len;
    const std::uint8_t* flags;
    const int* depth;
    const Key2* keys;
    int* eff;
    int* sublock;
    const std::uint8_t* missing;
    unsigned long long* W;
    unsigned int* C;
    int* rank;
    int* heads;
    int* listB;
    int* listS;
    int* listS2;        // S, sorted (rank-counting / warp sorts write here)
    ulonglong2* listSK;     // key of S[i] (written with S by the compaction: the sort reads it coalesced)
    unsigned int* listSC;   // chain size C of S[i]
    unsigned int* listSC2;  // chain size of S2[i]
    unsigned int* big;  // (offset, count) of the buckets with > 32 heads
    int* sorted;
    unsigned long long* start;
    int* victims;
    unsigned long long* hist_w;       // [kMaxPasses][kBins] weights (global atomics)
    unsigned int* hist_c;             // [kMaxPasses][kBins] counts
    unsigned int* seg_off;            // [kMaxPasses][kBins] bucket start in S
    unsigned int* seg_cnt;            // [kMaxPasses][kBins] bucket size
    unsigned int* cursor;             // [kMaxPasses][kBins] placement cursors
    SelState* ss;
    DevStatus* st;
    long long* result;
    const int* locked;
    long long n_locked;
    long long n_nodes;
    long long needed;
    int he_recompute;
    // deferred-heavy reports (report_deferred decisions; n_report = 0 otherwise),
    // written by otherwise idle CTAs during the sort phase and by do_cut (tail)
    int n_report;
    const int* heavy;
    const int* hch_off;
    const int* hch;
    const unsigned int* hmiss;
    HeavyReport* rep_out;   // pinned host memory
    const double* approx;
    double* approx_out;     // pinned host memory
    // small-cut path
    SampRec* samp;          // [kSamp]
    unsigned int samp_mask; // node n is sampled when hash(n) & mask == 0
    int* low;               // heads at or below the bound
    unsigned long long* gbar;  // grid barrier arrival counter (GridBar)
    unsigned int* sm_c;     // [kBins] counts, cursors, bucket offsets, big list [2*kBins]
    unsigned int* sm_cur;
    unsigned int* sm_off;
    unsigned int* sm_big;
    unsigned int* sm_task;  // [kBins] first rank task of each big bucket
    unsigned long long* sm_w;   // [kBins] weights, chain sizes, and their bucket prefixes
    unsigned long long* sm_cs;
    unsigned long long* sm_wpre;
    unsigned long long* sm_cpre;
    // the fused epilogue (select_epilogue): pinned host destinations
    DevStatus* h_st;
    SelState* h_ss;
    int* h_vict;                // null: the victims stay on the device
    long long h_cap;
    int no_refine;              // (tests) take the device-wide-sort fallback instead of refining
    std::uint8_t* flags_w;      // the deferral is cleared in place
    // oversized-bucket refinement (refine_buckets)
    unsigned int rf_cap;        // bucket descriptors per round parity
    unsigned int* rf_off;       // [2][rf_cap] bucket start in S
    unsigned int* rf_cnt;       // [2][rf_cap] bucket size
    unsigned int* rf_hist;      // [kRfSh][kBins] digit counts, then placement cursors (one window)
    unsigned long long* rf_orand;  // [2][rf_cap][6] OR / AND of the key words
    unsigned int* rf_small;     // [2 * n] (offset, count) of pieces with <= 32 heads
    ulonglong2* rf_tmpk;        // [n] keys in flight (the scatter's staging)
};

// Chain weight / size of head h: the members' scatter-adds (phase_chains)
// plus the head itself, which does not add to its own counters.
__device__ __forceinline__ unsigned long long chain_w(const SelArgs& a, int h) {
    return __ldcg(&a.W[h]) + static_cast<unsigned long long>(a.len[h]);
}
__device__ __forceinline__ unsigned int chain_c(const SelArgs& a, int h) { return __ldcg(&a.C[h]) + 1u; }


// record of heavy node j: max over its in-order device children's eff (the
// shared prefix has thousands of children), block-wide; eff / sublock read
// through L2 (written by other CTAs of the persistent kernel)
__device__ __forceinline__ void report_heavy_block(int j, const int* heavy, const int* ch_off, const int* ch,
                                                   const Key2* keys, const int* eff, const int* sublock,
                                                   const int* depth, const std::uint8_t* flags,
                                                   const unsigned int* hmiss, HeavyReport* out, const double* approx,
                                                   double* approx_out) {
    __shared__ unsigned long long s0[32], s1[32];
    __shared__ int se[32];
    int e = -1;
    Key2 best{0, 0};
    for (int q = ch_off[j] + threadIdx.x; q < ch_off[j + 1]; q += blockDim.x) {
        const int c = ch[q];
        if ((flags[c] & (kFlagTierMask | kFlagOutOfOrder)) != PBKV_TIER_DEVICE) continue;
        const int ec = __ldcg(&eff[c]);
        const Key2 k = load_key(keys, ec);
        if (e < 0 || key_less(best, e, k, ec)) {
            e = ec;
            best = k;
        }
    }
    for (int o = 16; o; o >>= 1) {
        const unsigned long long b0 = __shfl_xor_sync(0xffffffffu, best.w0, o);
        const unsigned long long b1 = __shfl_xor_sync(0xffffffffu, best.w1, o);
        const int be = __shfl_xor_sync(0xffffffffu, e, o);
        const Key2 bk{b0, b1};
        if (be >= 0 && (e < 0 || key_less(best, e, bk, be))) {
            e = be;
            best = bk;
        }
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) {
        s0[warp] = best.w0;
        s1[warp] = best.w1;
        se[warp] = e;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        e = -1;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
            const Key2 bk{s0[w], s1[w]};
            if (se[w] >= 0 && (e < 0 || key_less(best, e, bk, se[w]))) {
                e = se[w];
                best = bk;
            }
        }
        const int h = heavy[j];
        HeavyReport r{};
        r.w0 = e >= 0 ? best.w0 : 0ull;
        r.w1 = e >= 0 ? best.w1 : 0ull;
        r.eff = e;
        r.eff_depth = e >= 0 ? depth[e] : -1;
        r.sublock = __ldcg(&sublock[h]) ? 1 : 0;
        r.miss = static_cast<int>(hmiss[j]);
        out[j] = r;
        if (approx_out) {
            approx_out[2 * j] = approx[2 * j];
            approx_out[2 * j + 1] = approx[2 * j + 1];
        }
    }
}

// the record of the last victim (tail): its head's key and depths
__device__ __forceinline__ HeavyReport report_tail(const Key2* keys, const int* eff, const int* depth,
                                                  const int* victims, long long n) {
    HeavyReport r{};
    r.eff = -1;
    if (n > 0) {
        const int v = __ldcg(&victims[n - 1]);
        const int h = __ldcg(&eff[v]);
        const Key2 k = load_key(keys, h);
        r.w0 = k.w0;
        r.w1 = k.w1;
        r.eff = h;
        r.eff_depth = depth[h];
        r.depth_diff = depth[h] - depth[v];
    }
    return r;
}

// ---- phases ---------------------------------------------------------------------

// a locked DEVICE node makes itself and all of its ancestors ineligible: in the
// greedy frontier (policies.hpp:56-79) it is never pushed, so no ancestor's
// virtual device-child count can reach zero
__device__ __forceinline__ void phase_lock(const SelArgs& a, std::int64_t tid, std::int64_t nthr) {
    for (std::int64_t j = tid; j < a.n_locked; j += nthr) {
        int v = a.locked[j];
        if (v <= 0 || v >= a.n_nodes) continue;
        if ((a.flags[v] & kFlagTierMask) != PBKV_TIER_DEVICE) continue;
        while (v > 0) {
            if (atomicExch(&a.sublock[v], 1) == 1) break;
            v = a.parent[v];
        }
    }
    for (std::int64_t j = tid; j < static_cast<std::int64_t>(kMaxPasses) * kBins; j += nthr) {
        a.cursor[j] = 0;
        a.hist_w[j] = 0;
        a.hist_c[j] = 0;
    }
    for (std::int64_t j = tid; j < kBins; j += nthr) {
        a.sm_c[j] = 0;
        a.sm_cur[j] = 0;
        a.sm_w[j] = 0;
        a.sm_cs[j] = 0;
    }
}

// eff: every device node walks its key up the ancestor chain, CAS-ing the
// ancestors' argmax id; a walk stops at the first ancestor already holding a
// larger key (its holder carries it further), so eff ends as the exact
// subtree maximum
// (small-cut path) every head with key <= the bound joins the low list: collected
// per CTA in shared memory, appended with one global atomic per CTA
struct LowSink {
    bool on;
    Key2 tk;
    int tid;
    int* buf;                  // shared memory, kLowSh entries
    unsigned int* cnt;         // shared counter
    unsigned long long* orand; // shared [6]: OR, AND of the low keys' words
};
constexpr int kLowSh = 8192;

// One hop of a walker: n's key km is carried to ancestor p when it beats
// eff[p]'s key (plain read first, CAS only when it would win; a lost race
// re-reads next time).  Returns false when the walk is over.
__device__ __forceinline__ bool eff_hop(const SelArgs& a, int n, int& p, const Key2& km, int cur, const Key2& kc) {
    if (!key_less(kc, cur, km, n)) return false;  // a larger key holds p: its holder carries it
    if (atomicCAS(&a.eff[p], cur, n) == cur) {
        p = a.parent[p];
        return p > 0 && !(a.flags[p] & kFlagOutOfOrder);
    }
    return true;
}

// Per-CTA walk queue of the eff phase (shared memory, the sort union): the
// walker ids; parent and key are reloaded when a slot takes one (L2 hits)
struct WalkQueue {
    int* n;
    unsigned int* count;  // pushed
    unsigned int* head;   // popped
    int cap;
};

__device__ __forceinline__ void phase_eff(const SelArgs& a, std::int64_t tid, std::int64_t nthr, const WalkQueue& q) {
    // (1) every device node whose key beats its parent's own key starts a walk
    // (eff[p] >= key(p): below that it cannot change anything -- the common
    // case, HE keys grow toward the root).  kWalk nodes per thread have their
    // fields in flight together.  The walkers go to the CTA's queue.
    // (2) the CTA's threads drain the queue, kSlot walkers each, refilling a
    // slot as soon as its walk ends: the phase lasts about the longest walk
    // instead of the longest walk of every warp's lockstep group.
    constexpr int kWalk = 4;
    for (std::int64_t base = tid; base < a.n_nodes; base += kWalk * nthr) {
        int n[kWalk], p[kWalk];
        Key2 km[kWalk];
        bool act[kWalk];
        std::uint8_t fn[kWalk];
#pragma unroll
        for (int j = 0; j < kWalk; ++j) {  // own fields in one round trip (coalesced streams)
            const std::int64_t i = base + j * nthr;
            n[j] = static_cast<int>(i < a.n_nodes ? i : 0);
            fn[j] = a.flags[n[j]];
            p[j] = a.parent[n[j]];
            km[j] = load_key(a.keys, n[j]);
        }
#pragma unroll
        for (int j = 0; j < kWalk; ++j) {
            const std::int64_t i = base + j * nthr;
            act[j] = i < a.n_nodes && n[j] != 0 && (fn[j] & kFlagTierMask) == PBKV_TIER_DEVICE;
            // (out-of-order parents -- deferred heavy / spine -- are reduced
            // over their children lists instead: thousands of walkers CAS-ing
            // one hot word serialised in its L2 slice)
            act[j] = act[j] && p[j] > 0;
        }
        std::uint8_t fp[kWalk];
        Key2 kp[kWalk];
#pragma unroll
        for (int j = 0; j < kWalk; ++j) {  // the parent's flag and key in one round trip
            fp[j] = act[j] ? a.flags[p[j]] : std::uint8_t(0);
            kp[j] = act[j] ? load_key(a.keys, p[j]) : Key2{0, 0};
        }
#pragma unroll
        for (int j = 0; j < kWalk; ++j) {
            if (!(act[j] && !(fp[j] & kFlagOutOfOrder) && key_less(kp[j], p[j], km[j], n[j]))) continue;
            const unsigned int at = atomicAdd(q.count, 1u);
            if (at < static_cast<unsigned int>(q.cap)) {
                q.n[at] = n[j];
            } else {  // queue full (rare): walk here
                int pp = p[j];
                for (;;) {
                    const int cur = __ldcg(&a.eff[pp]);
                    if (!eff_hop(a, n[j], pp, km[j], cur, load_key(a.keys, cur))) break;
                }
            }
        }
    }
    __syncthreads();
    const unsigned int total = min(*q.count, static_cast<unsigned int>(q.cap));
    constexpr int kSlot = 4;
    int sn[kSlot], sp[kSlot];
    Key2 sk[kSlot];
    bool sa[kSlot];
#pragma unroll
    for (int j = 0; j < kSlot; ++j) sa[j] = false;
    bool more = true;  // the queue may still hold walkers
    for (;;) {
        if (more) {
#pragma unroll
            for (int j = 0; j < kSlot; ++j) {
                if (sa[j]) continue;
                const unsigned int at = atomicAdd(q.head, 1u);
                if (at >= total) {
                    more = false;
                    break;
                }
                sn[j] = q.n[at];
                sa[j] = true;
                sp[j] = -1;  // parent and key loaded below, together
            }
#pragma unroll
            for (int j = 0; j < kSlot; ++j)
                if (sa[j] && sp[j] < 0) {
                    sp[j] = a.parent[sn[j]];
                    sk[j] = load_key(a.keys, sn[j]);
                }
        }
        bool any = false;
        int cur[kSlot];
#pragma unroll
        for (int j = 0; j < kSlot; ++j) {
            cur[j] = sa[j] ? __ldcg(&a.eff[sp[j]]) : 0;
            any = any || sa[j];
        }
        if (!any) break;
        Key2 kc[kSlot];
#pragma unroll
        for (int j = 0; j < kSlot; ++j) kc[j] = sa[j] ? load_key(a.keys, cur[j]) : Key2{0, 0};
#pragma unroll
        for (int j = 0; j < kSlot; ++j)
            if (sa[j]) sa[j] = eff_hop(a, sn[j], sp[j], sk[j], cur[j], kc[j]);
    }
}

// the CTA's low heads: one global append, OR / AND into the selection state
__device__ __forceinline__ void low_flush(const SelArgs& a, const LowSink& lk) {
    __syncthreads();
    unsigned long long* sh = lk.orand + 8;  // a free word after the OR / AND
    const unsigned int c = *lk.cnt;
    if (threadIdx.x == 0) {
        if (c > static_cast<unsigned int>(kLowSh)) atomicOr(&a.ss->low_overflow, 1u);
        sh[0] = c ? atomicAdd(&a.ss->n_low, static_cast<unsigned long long>(min(c, static_cast<unsigned int>(kLowSh)))) : 0ull;
    }
    __syncthreads();
    const unsigned long long b0 = sh[0];
    for (unsigned int i = threadIdx.x; i < min(c, static_cast<unsigned int>(kLowSh)); i += blockDim.x) a.low[b0 + i] = lk.buf[i];
    if (threadIdx.x < 3 && c) {
        atomicOr(&a.ss->or_low[threadIdx.x], lk.orand[threadIdx.x]);
        atomicAnd(&a.ss->and_low[threadIdx.x], lk.orand[3 + threadIdx.x]);
    }
    __syncthreads();
}

// heads (eligible n with eff(n) == n) walk their own chain -- the contiguous
// eligible ancestors with the same eff -- for its token weight W and size C;
// head list, eligible tokens, OR/AND of the head keys (first radix pass)
__device__ __forceinline__ void phase_chains(const SelArgs& a, unsigned long long* sh, const LowSink& lk,
                                             bool build_list) {
    // Every eligible node n belongs to the chain of eff(n) (the closed form
    // orders eligible nodes by (eff, d); the nodes sharing an eff form a
    // contiguous eligible ancestor path from it), so the chain weight W[h] and
    // size C[h] are scatter-adds from the members -- no pointer-chasing walks.
    // Heads (eff(n) == n) are appended with one atomic per CTA and iteration.
    constexpr int kBatch = 4;
    SelState* ss = a.ss;
    unsigned long long tok = 0, n_seen = 0;
    unsigned long long or3[3] = {0, 0, 0}, and3[3] = {~0ull, ~0ull, ~0ull};
    const std::int64_t nthr = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    for (std::int64_t base = blockIdx.x * static_cast<std::int64_t>(blockDim.x); base < a.n_nodes;
         base += kBatch * nthr) {
        int n[kBatch], e[kBatch], ln[kBatch];
        bool elig[kBatch];
        std::uint8_t fl[kBatch], ms[kBatch];
        unsigned int cnt = 0;
        // every per-node field of the batch in one round trip (coalesced
        // streams; eligibility is decided after they arrive)
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
            const std::int64_t i = base + threadIdx.x + j * nthr;
            n[j] = static_cast<int>(i < a.n_nodes ? i : 0);
            fl[j] = a.flags[n[j]];
            elig[j] = !__ldcg(&a.sublock[n[j]]);
            e[j] = __ldcg(&a.eff[n[j]]);
            ms[j] = a.missing[n[j]];
            ln[j] = a.len[n[j]];
        }
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
            const std::int64_t i = base + threadIdx.x + j * nthr;
            elig[j] = elig[j] && i < a.n_nodes && n[j] != 0 &&
                      (fl[j] & (kFlagTierMask | kFlagOutOfOrder)) == PBKV_TIER_DEVICE;
            if (!elig[j]) {
                e[j] = -1;
                continue;
            }
            if (ms[j] == 2) set_error(a.st, PBKV_EINVAL, kErrKvflowMissing, n[j]);
            if (a.he_recompute && ms[j] && !(fl[j] & kFlagRetired))
                set_error(a.st, PBKV_EINVAL, kErrMissingForecast, n[j]);
            const unsigned long long l = static_cast<unsigned long long>(ln[j]);
            if (e[j] != n[j]) {  // a head's own length / count are implicit (chain_w / chain_c)
                atomicAdd(&a.W[e[j]], l);
                atomicAdd(&a.C[e[j]], 1u);
            }
            tok += l;
            cnt += e[j] == n[j] ? 1u : 0u;
        }
        if (!build_list) {  // small-cut mode: heads are counted; only the low ones are listed
            n_seen += cnt;
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                if (!elig[j] || e[j] != n[j]) continue;
                const int h = n[j];
                const Key2 k = load_key(a.keys, h);
                if (!key_less(lk.tk, lk.tid, k, h)) {  // a low head
                    const unsigned int q = atomicAdd(lk.cnt, 1u);
                    if (q < static_cast<unsigned int>(kLowSh)) lk.buf[q] = h;
                    for (int wd = 0; wd < 3; ++wd) {
                        const unsigned long long x = key_word(k, h, wd);
                        smem_or_u64(&lk.orand[wd], x);
                        smem_and_u64(&lk.orand[3 + wd], x);
                    }
                }
            }
            continue;
        }
        // CTA-wide exclusive offsets of the heads, one global atomic per CTA
        unsigned int* wcount = reinterpret_cast<unsigned int*>(sh);
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
        unsigned int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wcount[warp] = incl;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned int sum = 0;
            for (int w = 0; w < nw; ++w) {
                const unsigned int c = wcount[w];
                wcount[w] = sum;
                sum += c;
            }
            sh[31] = sum ? atomicAdd(&ss->n_L[0], static_cast<unsigned long long>(sum)) : 0ull;
        }
        __syncthreads();
        unsigned long long slot = sh[31] + wcount[warp] + (incl - cnt);
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
            if (!elig[j] || e[j] != n[j]) continue;
            const int h = n[j];
            a.heads[slot++] = h;
            const Key2 k = load_key(a.keys, h);
            for (int wd = 0; wd < 3; ++wd) {
                const unsigned long long x = key_word(k, h, wd);
                or3[wd] |= x;
                and3[wd] &= x;
            }
            if (lk.on && !key_less(lk.tk, lk.tid, k, h)) {  // a low head
                const unsigned int q = atomicAdd(lk.cnt, 1u);
                if (q < static_cast<unsigned int>(kLowSh)) lk.buf[q] = h;
                for (int wd = 0; wd < 3; ++wd) {
                    const unsigned long long x = key_word(k, h, wd);
                    smem_or_u64(&lk.orand[wd], x);
                    smem_and_u64(&lk.orand[3 + wd], x);
                }
            }
        }
    }
    const unsigned long long blk = block_reduce_bits(tok, SumOp(), sh);
    if (threadIdx.x == 0 && blk) atomicAdd(&ss->total_tok, blk);
    if (build_list) {
        flush_orand(or3, and3, ss->or_L[0], ss->and_L[0], sh);
    } else {
        const unsigned long long hs = block_reduce_bits(n_seen, SumOp(), sh);
        if (threadIdx.x == 0 && hs) atomicAdd(&ss->n_heads_seen, hs);
    }
    if (lk.on) low_flush(a, lk);
}

// The head list and its key OR / AND, for the full radix path when the
// chains phase ran in small-cut mode (it only counted the heads)
__device__ __forceinline__ void phase_heads(const SelArgs& a, unsigned long long* sh) {
    SelState* ss = a.ss;
    unsigned long long or3[3] = {0, 0, 0}, and3[3] = {~0ull, ~0ull, ~0ull};
    const std::int64_t nthr = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    for (std::int64_t base = blockIdx.x * static_cast<std::int64_t>(blockDim.x); base < a.n_nodes; base += nthr) {
        const std::int64_t i = base + threadIdx.x;
        const int n = static_cast<int>(i < a.n_nodes ? i : 0);
        const bool head = i < a.n_nodes && n != 0 &&
                          (a.flags[n] & (kFlagTierMask | kFlagOutOfOrder)) == PBKV_TIER_DEVICE &&
                          !__ldcg(&a.sublock[n]) && __ldcg(&a.eff[n]) == n;
        unsigned int* wcount = reinterpret_cast<unsigned int*>(sh);
        const long long slot = block_append(&ss->n_L[0], head, wcount, sh + 31);
        if (head) {
            a.heads[slot] = n;
            const Key2 k = load_key(a.keys, n);
            for (int wd = 0; wd < 3; ++wd) {
                const unsigned long long x = key_word(k, n, wd);
                or3[wd] |= x;
                and3[wd] &= x;
            }
        }
    }
    flush_orand(or3, and3, ss->or_L[0], ss->and_L[0], sh);
}

// per-CTA weight and count histograms of the next digit over the candidates
__device__ __forceinline__ void phase_hist(const SelArgs& a, const int* L, unsigned long long n_L, int lo, int pass,
                                           unsigned long long* hw, unsigned int* hc) {
    for (int b = threadIdx.x; b < kBins; b += blockDim.x) {
        hw[b] = 0;
        hc[b] = 0;
    }
    __syncthreads();
    const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
    const unsigned long long base0 = blockIdx.x * static_cast<unsigned long long>(blockDim.x);
    int xn = base0 + threadIdx.x < n_L ? __ldcg(&L[base0 + threadIdx.x]) : 0;  // next candidate, one ahead
    for (unsigned long long base = base0; base < n_L; base += stride) {
        const unsigned long long i = base + threadIdx.x;
        unsigned int d = 0xffffffffu;
        unsigned long long w = 0;
        const int x = xn;
        xn = i + stride < n_L ? __ldcg(&L[i + stride]) : 0;
        if (i < n_L) {
            d = key_bits(load_key(a.keys, x), x, lo, kDigitBits);
            w = chain_w(a, x);
        }
        // equal digits of a warp are summed first: skewed digit distributions
        // (e.g. every retired head in one bucket) would serialise on one bank
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        unsigned long long sum = 0;
        if (peers == 0xffffffffu) {  // one digit across the warp (the skewed case): butterfly
            sum = w;
#pragma unroll
            for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        } else {
            for (unsigned m = peers; m; m &= m - 1) sum += __shfl_sync(peers, w, __ffs(m) - 1);
        }
        if (d != 0xffffffffu && (threadIdx.x & 31) == __ffs(peers) - 1) {
            smem_add_u64(&hw[d], sum);
            atomicAdd(&hc[d], static_cast<unsigned int>(__popc(peers)));
        }
    }
    __syncthreads();
    // per-pass global histogram (zeroed at kernel start): one atomic per
    // non-empty bin per CTA, no partial arrays and no reduction phase
    unsigned long long* gw = a.hist_w + static_cast<std::size_t>(pass) * kBins;
    unsigned int* gc = a.hist_c + static_cast<std::size_t>(pass) * kBins;
    for (int b = threadIdx.x; b < kBins; b += blockDim.x) {
        const unsigned int c = hc[b];
        if (c) {
            atomicAdd(&gw[b], hw[b]);
            atomicAdd(&gc[b], c);
        }
    }
}

struct PickOut {
    int bucket;
    unsigned long long need;       // need remaining inside the bucket
    unsigned int below_cnt;        // heads placed into S by this pass
    unsigned int max_cnt;          // largest bucket below
};

// the digit bucket where the cumulative weight reaches `need`, and the bucket
// offsets of the heads below it.  Every CTA evaluates the same pick from the
// reduced histograms (no extra barrier); CTA 0 records the bucket layout.
__device__ __forceinline__ PickOut phase_pick(const SelArgs& a, unsigned long long need, int pass,
                                              unsigned long long s_base, void* tmp_raw, unsigned int* off_sh,
                                              PickOut* out_sh) {
    using ScanW = cub::BlockScan<unsigned long long, kPThreads>;
    constexpr int kPer = kBins / kPThreads;
    unsigned long long vw[kPer], sw = 0;
    unsigned int vc[kPer];
    unsigned long long sc = 0;
    for (int j = 0; j < kPer; ++j) {
        vw[j] = __ldcg(&a.hist_w[static_cast<std::size_t>(pass) * kBins + threadIdx.x * kPer + j]);
        vc[j] = __ldcg(&a.hist_c[static_cast<std::size_t>(pass) * kBins + threadIdx.x * kPer + j]);
        sw += vw[j];
        sc += vc[j];
    }
    unsigned long long ew, ec;
    ScanW(*reinterpret_cast<typename ScanW::TempStorage*>(tmp_raw)).ExclusiveSum(sw, ew);
    __syncthreads();
    ScanW(*reinterpret_cast<typename ScanW::TempStorage*>(tmp_raw)).ExclusiveSum(sc, ec);
    unsigned long long rw = ew, rc = ec;
    for (int j = 0; j < kPer; ++j) {
        const int d = threadIdx.x * kPer + j;
        off_sh[d] = static_cast<unsigned int>(s_base + rc);
        if (rw < need && rw + vw[j] >= need) {
            out_sh->bucket = d;
            out_sh->need = need - rw;
            out_sh->below_cnt = static_cast<unsigned int>(rc);
        }
        rw += vw[j];
        rc += vc[j];
    }
    __syncthreads();
    PickOut r = *out_sh;
    // largest bucket below the pick (for the sort-capacity decision)
    unsigned int mx = 0;
    for (int j = 0; j < kPer; ++j) {
        const int d = threadIdx.x * kPer + j;
        if (d < r.bucket) mx = max(mx, vc[j]);
    }
    mx = static_cast<unsigned int>(block_reduce_bits(mx, MaxOp(), reinterpret_cast<unsigned long long*>(tmp_raw)));
    __syncthreads();
    if (threadIdx.x == 0) out_sh->max_cnt = mx;
    if (blockIdx.x == 0) {
        unsigned int* so = a.seg_off + static_cast<std::size_t>(pass) * kBins;
        unsigned int* sc2 = a.seg_cnt + static_cast<std::size_t>(pass) * kBins;
        for (int j = 0; j < kPer; ++j) {
            const int d = threadIdx.x * kPer + j;
            so[d] = off_sh[d];
            sc2[d] = d < r.bucket ? vc[j] : 0u;
            if (d < r.bucket && vc[j] > 32u) {  // sorted by chunked rank counting
                const unsigned int q = atomicAdd(&a.ss->n_big, 1u);
                a.big[2 * q] = off_sh[d];
                a.big[2 * q + 1] = vc[j];
            }
        }
    }
    __syncthreads();
    r.max_cnt = out_sh->max_cnt;
    return r;
}

// below the bucket -> S at its digit's bucket; in the bucket -> next list
__device__ __forceinline__ void phase_compact(const SelArgs& a, const int* L, unsigned long long n_L, int* L2,
                                              int nx, int* S, int pass, int lo, int bucket,
                                              const unsigned int* off_sh, unsigned long long* sh) {
    SelState* ss = a.ss;
    unsigned int* cur = a.cursor + static_cast<std::size_t>(pass) * kBins;
    unsigned long long orS[3] = {0, 0, 0}, andS[3] = {~0ull, ~0ull, ~0ull};
    unsigned long long orL[3] = {0, 0, 0}, andL[3] = {~0ull, ~0ull, ~0ull};
    const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
    const unsigned long long base0 = blockIdx.x * static_cast<unsigned long long>(blockDim.x);
    int xn = base0 + threadIdx.x < n_L ? __ldcg(&L[base0 + threadIdx.x]) : 0;  // next candidate, one ahead
    for (unsigned long long base = base0; base < n_L; base += stride) {
        const unsigned long long i = base + threadIdx.x;
        int d = -1;
        const int x = xn;
        Key2 k{0, 0};
        xn = i + stride < n_L ? __ldcg(&L[i + stride]) : 0;
        if (i < n_L) {
            k = load_key(a.keys, x);
            d = static_cast<int>(key_bits(k, x, lo, kDigitBits));
        }
        const bool below = d >= 0 && d < bucket;
        const bool same = d == bucket;
        // placement into the digit's bucket: warp-aggregated cursor
        const unsigned peers = __match_any_sync(0xffffffffu, below ? d : -1);
        if (below) {
            const int lane = threadIdx.x & 31;
            const int leader = __ffs(peers) - 1;
            unsigned int basepos = 0;
            const unsigned int cx = chain_c(a, x);  // in flight with the cursor atomic
            if (lane == leader) basepos = atomicAdd(&cur[d], static_cast<unsigned int>(__popc(peers)));
            basepos = __shfl_sync(peers, basepos, leader);
            const unsigned int pos = off_sh[d] + basepos + __popc(peers & ((1u << lane) - 1u));
            S[pos] = x;
            a.listSK[pos] = make_ulonglong2(k.w0, k.w1);
            a.listSC[pos] = cx;
            for (int w = 0; w < 3; ++w) {
                orS[w] |= key_word(k, x, w);
                andS[w] &= key_word(k, x, w);
            }
        }
        const long long s2 = block_append(&ss->n_L[nx], same, reinterpret_cast<unsigned int*>(sh), sh + 31);
        if (same) {
            L2[s2] = x;
            for (int w = 0; w < 3; ++w) {
                orL[w] |= key_word(k, x, w);
                andL[w] &= key_word(k, x, w);
            }
        }
    }
    flush_orand(orS, andS, ss->or_S, ss->and_S, sh);
    flush_orand(orL, andL, ss->or_L[nx], ss->and_L[nx], sh);
}

// (w0, w1, id) order with padding (id < 0) after every real key
__device__ __forceinline__ bool sk_less(unsigned long long a0, unsigned long long a1, int av, unsigned long long b0,
                                        unsigned long long b1, int bv) {
    if (av < 0) return false;
    if (bv < 0) return true;
    if (a0 != b0) return a0 < b0;
    if (a1 != b1) return a1 < b1;
    return av < bv;
}

// small bucket (<= 32 heads): one warp, rank = number of smaller keys
__device__ __forceinline__ void warp_sort_bucket(const SelArgs& a, const int* S, int* S2, unsigned int off,
                                                 unsigned int cnt) {
    const int lane = threadIdx.x & 31;
    const bool in = static_cast<unsigned int>(lane) < cnt;
    const int x = in ? __ldcg(&S[off + lane]) : -1;
    Key2 k{0, 0};
    unsigned int cx = 0;
    if (in) {
        const ulonglong2 kk = __ldcg(&a.listSK[off + lane]);
        k = Key2{kk.x, kk.y};
        cx = __ldcg(&a.listSC[off + lane]);
    }
    int rank = 0;
    for (unsigned int j = 0; j < cnt; ++j) {
        const unsigned long long b0 = __shfl_sync(0xffffffffu, k.w0, j);
        const unsigned long long b1 = __shfl_sync(0xffffffffu, k.w1, j);
        const int bv = __shfl_sync(0xffffffffu, x, j);
        rank += sk_less(b0, b1, bv, k.w0, k.w1, x) ? 1 : 0;
    }
    if (in) {
        S2[off + rank] = x;
        a.listSC2[off + rank] = cx;
    }
}

// Buckets with > 32 heads (at most kRankCap): every element's rank is the
// number of smaller keys in its bucket, counted from shared memory by
// kRankParts threads per group of kRankQuad elements.  Tasks are (bucket, chunk of kRankChunk
// elements), task t on CTA t mod gridDim.x; a CTA finds its tasks through the
// chunk-count prefix of the bucket list, a tile of kPThreads buckets at a
// time.  The keys of a bucket are packed over the bucket's own varying bits
// into one word when they fit, else two (one or two compares per pair).
constexpr int kRankCap = 256;  // larger buckets are split first (refine_buckets)
static_assert(kRankCap + (3 * kPThreads) / 2 + 6 * (kPThreads / 32 + 1) <= kBucketCap, "rank scratch exceeds k0");
constexpr int kRankChunk = 128;
constexpr int kRankQuad = 4;                                   // elements ranked per thread
constexpr int kRankParts = kPThreads * kRankQuad / kRankChunk;  // threads per element group (16)
__device__ __forceinline__ void rank_sort_big(const SelArgs& a, const int* S, int* S2, unsigned int n_big,
                                              unsigned long long* k0, unsigned long long* k1, int* val,
                                              bool has_sk, unsigned long long* sh) {
    // the bucket arrays hold at most kRankCap keys: the tile of the bucket
    // list and the mask reduction live above them (no static shared memory:
    // the L1 share of the eff walk's gathers stays larger)
    unsigned int* tile_sh = reinterpret_cast<unsigned int*>(k0 + kRankCap);  // [3 * kPThreads]
    unsigned long long (*red_sh)[6] =
        reinterpret_cast<unsigned long long (*)[6]>(k0 + kRankCap + (3 * kPThreads) / 2);  // [kPThreads / 32 + 1][6]
    unsigned int* tp = tile_sh;
    unsigned int* toff = tile_sh + kPThreads;
    unsigned int* tcnt = tile_sh + 2 * kPThreads;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    unsigned int T = 0;  // first task of the tile
    for (unsigned int b0 = 0; b0 < n_big; b0 += blockDim.x) {
        const unsigned int bb = b0 + threadIdx.x;
        const unsigned int m = min(static_cast<unsigned int>(blockDim.x), n_big - b0);
        unsigned int off = 0, cnt = 0;
        if (bb < n_big) {
            off = __ldcg(&a.big[2 * bb]);
            cnt = __ldcg(&a.big[2 * bb + 1]);
        }
        unsigned int tile_tasks = 0;
        const unsigned int ex = block_excl_u32((cnt + kRankChunk - 1) / kRankChunk, sh, &tile_tasks);
        tp[threadIdx.x] = ex;
        toff[threadIdx.x] = off;
        tcnt[threadIdx.x] = cnt;
        __syncthreads();
        // this CTA's first task at or after T
        unsigned int t = T + (blockIdx.x + gridDim.x - T % gridDim.x) % gridDim.x;
        for (; t < T + tile_tasks; t += gridDim.x) {
            const unsigned int loc = t - T;
            unsigned int lo = 0, hi = m - 1;  // last bucket of the tile whose first task is <= loc
            while (lo < hi) {
                const unsigned int mid = (lo + hi + 1) >> 1;
                if (tp[mid] <= loc) lo = mid;
                else hi = mid - 1;
            }
            const unsigned int boff = toff[lo], bcnt = tcnt[lo], c = loc - tp[lo];
            const unsigned long long tl0 = gtimer();
            // the bucket's ids and keys: coalesced reads of S / SK (the head
            // list of take_all has no SK: gathered instead); OR / AND of the
            // key words on the way
            unsigned long long o[3] = {0, 0, 0}, n3[3] = {~0ull, ~0ull, ~0ull};
            for (unsigned int i = threadIdx.x; i < bcnt; i += blockDim.x) {
                const int x = __ldcg(&S[boff + i]);
                Key2 k;
                if (has_sk) {
                    const ulonglong2 kk = __ldcg(&a.listSK[boff + i]);
                    k = Key2{kk.x, kk.y};
                } else {
                    k = load_key(a.keys, x);
                }
                k0[i] = k.w0;
                k1[i] = k.w1;
                val[i] = x;
                for (int w = 0; w < 3; ++w) {
                    o[w] |= key_word(k, x, w);
                    n3[w] &= key_word(k, x, w);
                }
            }
            for (int w = 0; w < 3; ++w) {
#pragma unroll
                for (int q = 16; q > 0; q >>= 1) {
                    o[w] |= __shfl_xor_sync(0xffffffffu, o[w], q);
                    n3[w] &= __shfl_xor_sync(0xffffffffu, n3[w], q);
                }
            }
            if (lane == 0)
                for (int w = 0; w < 3; ++w) {
                    red_sh[warp][w] = o[w];
                    red_sh[warp][3 + w] = n3[w];
                }
            __syncthreads();
            if (threadIdx.x < 6) {
                unsigned long long r = threadIdx.x < 3 ? 0ull : ~0ull;
                for (int q = 0; q < nw; ++q) r = threadIdx.x < 3 ? (r | red_sh[q][threadIdx.x]) : (r & red_sh[q][threadIdx.x]);
                red_sh[kPThreads / 32][threadIdx.x] = r;
            }
            __syncthreads();
            const unsigned long long v0 = red_sh[kPThreads / 32][0] ^ red_sh[kPThreads / 32][3];
            const unsigned long long v1 = red_sh[kPThreads / 32][1] ^ red_sh[kPThreads / 32][4];
            const unsigned long long v2 = (red_sh[kPThreads / 32][2] ^ red_sh[kPThreads / 32][5]) & 0xffffffffull;
            const int vbits = __popcll(v0) + __popcll(v1) + __popcll(v2);
            const bool packed = vbits <= 64;               // one word; k1 carries the chain sizes
            const bool packed2 = !packed && vbits <= 128;  // two words (hi, lo)
            if (packed) {
                for (unsigned int i = threadIdx.x; i < bcnt; i += blockDim.x) {
                    const int x = val[i];
                    k0[i] = pack_key(Key2{k0[i], k1[i]}, x, v0, v1, v2);
                    k1[i] = has_sk ? __ldcg(&a.listSC[boff + i]) : chain_c(a, x);
                }
            } else if (packed2) {
                for (unsigned int i = threadIdx.x; i < bcnt; i += blockDim.x) {
                    unsigned long long h, l;
                    pack_key2(Key2{k0[i], k1[i]}, val[i], v0, v1, v2, h, l);
                    k0[i] = h;
                    k1[i] = l;
                }
            }
            __syncthreads();
            const unsigned long long tl1 = gtimer();
            if (threadIdx.x == 0) atomicMax(&a.ss->dbg[2], tl1 - tl0);
            {  // kRankQuad elements per thread group, each loaded key compared against all of them
                const unsigned int g = threadIdx.x / kRankParts, part = threadIdx.x % kRankParts;
                const unsigned int e0 = c * kRankChunk + g * kRankQuad;
                unsigned long long x0[kRankQuad], x1[kRankQuad];
                unsigned int r[kRankQuad];
#pragma unroll
                for (int j = 0; j < kRankQuad; ++j) {
                    const unsigned int e = e0 + j;
                    x0[j] = e < bcnt ? k0[e] : 0ull;
                    x1[j] = e < bcnt ? k1[e] : 0ull;
                    r[j] = 0;
                }
                if (packed) {  // distinct 64-bit order-preserving keys: one compare each
#pragma unroll 2
                    for (unsigned int q = part; q < bcnt; q += kRankParts) {
                        const unsigned long long h = k0[q];
#pragma unroll
                        for (int j = 0; j < kRankQuad; ++j) r[j] += h < x0[j] ? 1u : 0u;
                    }
                } else if (packed2) {  // distinct 128-bit keys, branch-free
#pragma unroll 2
                    for (unsigned int q = part; q < bcnt; q += kRankParts) {
                        const unsigned long long h = k0[q], l = k1[q];
#pragma unroll
                        for (int j = 0; j < kRankQuad; ++j) r[j] += (h < x0[j] || (h == x0[j] && l < x1[j])) ? 1u : 0u;
                    }
                } else {
                    for (unsigned int q = part; q < bcnt; q += kRankParts)
#pragma unroll
                        for (int j = 0; j < kRankQuad; ++j) {
                            const unsigned int e = e0 + j;
                            r[j] += e < bcnt && sk_less(k0[q], k1[q], val[q], x0[j], x1[j], val[e]) ? 1u : 0u;
                        }
                }
#pragma unroll
                for (int j = 0; j < kRankQuad; ++j)
#pragma unroll
                    for (int q = 1; q < kRankParts; q <<= 1) r[j] += __shfl_xor_sync(0xffffffffu, r[j], q);
                if (part == 0) {
#pragma unroll
                    for (int j = 0; j < kRankQuad; ++j) {
                        const unsigned int e = e0 + j;
                        if (e < bcnt) {
                            const int av = val[e];
                            S2[boff + r[j]] = av;
                            a.listSC2[boff + r[j]] = packed ? static_cast<unsigned int>(k1[e])
                                                            : (has_sk ? __ldcg(&a.listSC[boff + e]) : chain_c(a, av));
                        }
                    }
                }
            }
            if (threadIdx.x == 0) atomicMax(&a.ss->dbg[3], gtimer() - tl1);
            __syncthreads();  // the next task reloads the bucket arrays
        }
        T += tile_tasks;
        __syncthreads();  // the next tile overwrites the tile arrays
    }
}

// every eligible node of a selected chain lands at start[rank(head)] + d:
// each selected head walks its own chain (the contiguous eligible ancestors
// with eff == head, d = depth difference), O(victims) instead of a pass over
// every node
__device__ __forceinline__ void phase_scatter(const SelArgs& a, const int* S2, unsigned long long nS,
                                              std::int64_t tid, std::int64_t nthr) {
    for (std::int64_t pos = tid; pos < static_cast<std::int64_t>(nS); pos += nthr) {
        const int h = __ldcg(&S2[pos]);
        unsigned long long at = __ldcg(&a.start[pos]);
        int x = h;
        for (;;) {
            a.victims[at++] = x;
            x = a.parent[x];
            if (x <= 0) break;
            const bool ok = (a.flags[x] & (kFlagTierMask | kFlagOutOfOrder)) == PBKV_TIER_DEVICE &&
                            !__ldcg(&a.sublock[x]) && __ldcg(&a.eff[x]) == h;
            if (!ok) break;
        }
    }
}

// the cut inside the last (cut) chain; freed / shortfall
__device__ __forceinline__ void do_cut(const SelArgs& a) {
    SelState* ss = a.ss;
    const unsigned long long nS = __ldcg(&ss->n_S);
    const int cut = __ldcg(&ss->cut_head);
    const unsigned long long s0 = __ldcg(&a.start[nS - 1]);
    const unsigned int c = chain_c(a, cut);
    if (__ldcg(&ss->take_all)) {
        ss->n_victims = s0 + c;
        ss->freed = __ldcg(&ss->total_tok);
    } else {
        const unsigned long long need = __ldcg(&ss->need_final);
        const unsigned long long below = static_cast<unsigned long long>(a.needed) - need;
        unsigned long long acc = 0, j = 0;
        for (; j < c; ++j) {
            acc += static_cast<unsigned long long>(a.len[__ldcg(&a.victims[s0 + j])]);
            if (acc >= need) break;
        }
        ss->n_victims = s0 + j + 1;
        ss->freed = below + acc;
    }
    ss->shortfall = ss->freed < static_cast<unsigned long long>(a.needed) ? 1 : 0;
    a.result[0] = static_cast<long long>(ss->n_victims);
    a.result[1] = static_cast<long long>(ss->freed);
    a.result[2] = ss->shortfall;
    if (a.n_report > 0) {
        __threadfence();  // the victims of every CTA are in L2 (grid barrier before the cut)
        a.rep_out[a.n_report] = report_tail(a.keys, a.eff, a.depth, a.victims, static_cast<long long>(ss->n_victims));
    }
}

// ---- grid barrier ------------------------------------------------------------------------
// Arrival counter shared by every launch of the persistent kernel (64-bit,
// never reset): a CTA's arrival returns the running count, whose quotient by
// the grid size names the barrier.  The waiting CTAs back off with
// __nanosleep, so the tail of a phase -- often one CTA's serial work -- does
// not compete with 295 spinning loads for the memory system.
struct GridBar {
    unsigned long long* count;
    __device__ __forceinline__ void sync() const {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            const unsigned long long old = atomicAdd(count, 1ull);
            const unsigned long long target = (old / gridDim.x + 1ull) * gridDim.x;
            unsigned int ns = 32;
            for (;;) {
                unsigned long long v;
                asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(count) : "memory");
                if (v >= target) break;
                __nanosleep(ns);
                ns = ns < 128 ? ns * 2 : 128;
            }
        }
        __syncthreads();
    }
};

// ---- the persistent kernel --------------------------------------------------------------
struct PersistSmem {
    union {
        struct {
            unsigned long long w[kBins];
            unsigned int c[kBins];
            unsigned long long cs[kBins];  // small path: chain sizes per bucket
        } hist;
        typename cub::BlockScan<unsigned long long, kPThreads>::TempStorage scan;
        struct {
            unsigned long long k0[kBucketCap];
            unsigned long long k1[kBucketCap];
            int val[kBucketCap];
        } sort;
    } u;
    unsigned int off[kBins];
    unsigned long long sh[32];
    unsigned long long bc[4];  // broadcast of shared scalars
    unsigned int qctl[2];      // eff walk queue: pushed, popped
    PickOut pick;
};

// ---- small-cut path ------------------------------------------------
// A cut that takes a small share of the eligible tokens lies among the
// lowest keys.  During the lock phase CTA 0 reads a strided node sample (node
// j*R + jitter(j), ~1/R of the nodes: key, token length) and finds by a
// weighted MSD radix select over it the bound T: the sampled key at which R x
// the sampled tokens at or below it reach 2 x `needed` plus a sampling margin.
// The eff phase lists every device node with key <= T (the low list).  If the
// exact chain weight of the low list's heads reaches `needed` (checked from
// its histogram) the cut lies among them, and the rest of the decision is:
// one 11-bit MSD histogram of the low heads, placement into buckets, then
// every bucket ranked in place -- the rank count also sums the chain weights W
// and sizes C of the smaller keys, so with the per-bucket prefixes each head
// knows its cumulative token count and its victim offset: a selected head
// scatters its own chain, and the head whose count crosses `needed` scatters
// the cut.  Otherwise (the sample missed; rare) the full radix path below
// runs.  Results are identical either way.
struct SmallBound {
    Key2 k;
    int id;
    bool ok;
};

// one CTA: the bound T from the node sample (two samples per thread)
__device__ SmallBound small_bound(const SelArgs& a, PersistSmem& sm) {
    SmallBound r{{0, 0}, -1, false};
    const long long R = static_cast<long long>(a.samp_mask) + 1;
    const long long ns = (a.n_nodes + R - 1) / R;
    if (ns > 2 * kPThreads) return r;
    const unsigned long long tb0 = gtimer();
    Key2 k[2];
    int id[2];
    unsigned long long ln[2];
    bool alive[2];
    unsigned long long tok = 0, nv = 0;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const long long j = threadIdx.x + q * kPThreads;
        long long n = j * R + static_cast<long long>(mix32(static_cast<unsigned int>(j)) & a.samp_mask);
        if (n >= a.n_nodes) n = j * R;
        alive[q] = false;
        id[q] = -1;
        ln[q] = 0;
        k[q] = Key2{0, 0};
        if (j < ns && n != 0 && (a.flags[n] & (kFlagTierMask | kFlagOutOfOrder)) == PBKV_TIER_DEVICE) {
            k[q] = load_key(a.keys, static_cast<int>(n));
            id[q] = static_cast<int>(n);
            ln[q] = static_cast<unsigned long long>(a.len[n]);
            alive[q] = true;
            tok += ln[q];
            nv += 1;
        }
    }
    const unsigned long long T = block_reduce_bits(tok, SumOp(), sm.sh);
    if (threadIdx.x == 0) sm.bc[0] = T;
    __syncthreads();
    const unsigned long long stok = sm.bc[0];
    __syncthreads();
    const unsigned long long NV = block_reduce_bits(nv, SumOp(), sm.sh);
    if (threadIdx.x == 0) sm.bc[1] = NV;
    __syncthreads();
    const unsigned long long nvalid = sm.bc[1];
    __syncthreads();
    if (nvalid == 0 || stok == 0) return r;
    // sampled-token target: 2 x needed / R, plus 8 + 3 sqrt(count) samples' worth
    const double mean = static_cast<double>(stok) / static_cast<double>(nvalid);
    const double tgt = 2.0 * static_cast<double>(a.needed) / static_cast<double>(R);
    const double cnt_est = tgt / mean;
    unsigned long long rem =
        static_cast<unsigned long long>(ceil(tgt + (8.0 + 3.0 * sqrt(cnt_est + 1.0)) * mean));
    if (rem == 0) rem = 1;
    if (rem > stok) return r;
    const unsigned long long tb1 = gtimer();
    int n_pass = 0;
    unsigned long long below = 0;  // samples below the chosen bins
    unsigned int* hc = sm.u.hist.c;
    unsigned long long* hw = sm.u.hist.w;
    unsigned long long* orand = sm.u.hist.cs;  // [0..2] or, [3..5] and
    for (int pass = 0; pass < 24; ++pass) {
        // varying bits of the alive keys
        if (threadIdx.x < 3) {
            orand[threadIdx.x] = 0ull;
            orand[3 + threadIdx.x] = ~0ull;
        }
        __syncthreads();
        unsigned long long o3[3] = {0, 0, 0}, n3[3] = {~0ull, ~0ull, ~0ull};
#pragma unroll
        for (int q = 0; q < 2; ++q)
            if (alive[q])
                for (int w = 0; w < 3; ++w) {
                    const unsigned long long x = key_word(k[q], id[q], w);
                    o3[w] |= x;
                    n3[w] &= x;
                }
        for (int w = 0; w < 3; ++w) {
            for (int o = 16; o; o >>= 1) {
                o3[w] |= __shfl_xor_sync(0xffffffffu, o3[w], o);
                n3[w] &= __shfl_xor_sync(0xffffffffu, n3[w], o);
            }
            if ((threadIdx.x & 31) == 0) {
                smem_or_u64(&orand[w], o3[w]);
                smem_and_u64(&orand[3 + w], n3[w]);
            }
        }
        for (int b = threadIdx.x; b < 256; b += blockDim.x) {
            hc[b] = 0;
            hw[b] = 0;
        }
        __syncthreads();
        int top = -1;  // top varying bit of the alive keys (shared-memory words)
        {
            const unsigned long long x0 = orand[0] ^ orand[3], x1 = orand[1] ^ orand[4];
            const unsigned long long x2 = (orand[2] ^ orand[5]) & 0xffffffffull;
            if (x0) top = 96 + 63 - __clzll(static_cast<long long>(x0));
            else if (x1) top = 32 + 63 - __clzll(static_cast<long long>(x1));
            else if (x2) top = 63 - __clzll(static_cast<long long>(x2));
        }
        if (top < 0) break;  // one alive key left
        const int lo = top - 7 < 0 ? 0 : top - 7;
        const int nb = top - lo + 1;
        unsigned int dg[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            dg[q] = alive[q] ? key_bits(k[q], id[q], lo, nb) : 0u;
            // equal digits of a warp first (early passes put most samples in one bin)
            const unsigned peers = __match_any_sync(0xffffffffu, alive[q] ? dg[q] : 0xffffffffu);
            // (the sample's token weights only steer the bound: saturated at 2^26 per node)
            const unsigned long long sw =
                __reduce_add_sync(peers, static_cast<unsigned int>(ln[q] < (1ull << 26) ? ln[q] : (1ull << 26)));
            if (alive[q] && (threadIdx.x & 31) == __ffs(peers) - 1) {
                atomicAdd(&hc[dg[q]], static_cast<unsigned int>(__popc(peers)));
                smem_add_u64(&hw[dg[q]], sw);
            }
        }
        __syncthreads();
        if (threadIdx.x < 32) {  // the bin where the running sampled tokens reach rem
            const int lane = threadIdx.x;
            unsigned long long w8 = 0, c8 = 0;
            for (int j = 0; j < 8; ++j) {
                w8 += hw[lane * 8 + j];
                c8 += hc[lane * 8 + j];
            }
            unsigned long long wi = w8, ci = c8;
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, wi, o);
                const unsigned long long z = __shfl_up_sync(0xffffffffu, ci, o);
                if (lane >= o) {
                    wi += y;
                    ci += z;
                }
            }
            unsigned long long wb = wi - w8, cb = ci - c8;
            if (wb < rem && wi >= rem) {
                for (int j = 0; j < 8; ++j) {
                    const int d = lane * 8 + j;
                    if (wb + hw[d] >= rem) {
                        sm.bc[2] = static_cast<unsigned long long>(d);
                        sm.bc[3] = rem - wb;
                        sm.bc[0] = cb;
                        sm.bc[1] = hc[d];
                        break;
                    }
                    wb += hw[d];
                    cb += hc[d];
                }
            }
        }
        __syncthreads();
        const unsigned int pick = static_cast<unsigned int>(sm.bc[2]);
        rem = sm.bc[3];
        below += sm.bc[0];
        const unsigned long long left = sm.bc[1];
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 2; ++q) alive[q] = alive[q] && dg[q] == pick;
        ++n_pass;
        if (left == 1) break;
    }
#pragma unroll
    for (int q = 0; q < 2; ++q)
        if (alive[q]) {  // the bound (unique)
            sm.bc[0] = k[q].w0;
            sm.bc[1] = k[q].w1;
            sm.bc[2] = static_cast<unsigned long long>(id[q]);
        }
    __syncthreads();
    r.k = Key2{sm.bc[0], sm.bc[1]};
    r.id = static_cast<int>(sm.bc[2]);
    r.ok = (below + 1) * static_cast<unsigned long long>(R) <= static_cast<unsigned long long>(kSmallMax);
    if (threadIdx.x == 0) {
        a.ss->est_low = (below + 1) * static_cast<unsigned long long>(R);
        a.ss->dbg[0] = tb1 - tb0;
        a.ss->dbg[1] = gtimer() - tb1;
        a.ss->dbg[2] = static_cast<unsigned long long>(n_pass);
    }
    __syncthreads();
    return r;
}

// S1: histogram of the low heads (count, chain weight, chain size per 11-bit digit)
template <int kNBins>
__device__ __forceinline__ void small_hist(const SelArgs& a, unsigned long long n_low, int lo,
                                           unsigned long long v0, unsigned long long v1, unsigned long long v2,
                                           PersistSmem& sm) {
    constexpr int nbins = kNBins;
    const unsigned long long th0 = gtimer();
    for (int b = threadIdx.x; b < nbins; b += blockDim.x) {
        sm.u.hist.w[b] = 0;
        sm.u.hist.c[b] = 0;
        sm.u.hist.cs[b] = 0;
    }
    __syncthreads();
    const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
    for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x; i < n_low;
         i += stride) {
        const int x = __ldcg(&a.low[i]);
        const unsigned long long pk = pack_key(load_key(a.keys, x), x, v0, v1, v2);
        const unsigned int d = static_cast<unsigned int>(pk >> lo) & static_cast<unsigned int>(nbins - 1);
        smem_add_u64(&sm.u.hist.w[d], chain_w(a, x));
        atomicAdd(&sm.u.hist.c[d], 1u);
        atomicAdd(reinterpret_cast<unsigned int*>(sm.u.hist.cs) + d, chain_c(a, x));  // < 2^24 (nodes)
    }
    __syncthreads();
    // two global atomics per non-empty bin: the token weight, and the head
    // count with the chain-size sum packed in one word (both < 2^32: they
    // count nodes)
    const unsigned int* csum = reinterpret_cast<const unsigned int*>(sm.u.hist.cs);
    for (int b = threadIdx.x; b < nbins; b += blockDim.x) {
        const unsigned int c = sm.u.hist.c[b];
        if (c) {
            atomicAdd(&a.sm_w[b], sm.u.hist.w[b]);
            atomicAdd(&a.sm_cs[b], (static_cast<unsigned long long>(c) << 32) | csum[b]);
        }
    }
    // the last CTA to finish turns the histogram into the bucket layout once:
    // offsets, token / chain-size prefixes, the check that the cut lies among
    // the low heads, the list of buckets ranked by tiles and their first tasks
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        sm.bc[0] = atomicAdd(&a.ss->small_done, 1u);
        atomicMax(&a.ss->dbg2[0], gtimer() - th0);
    }
    __syncthreads();
    if (sm.bc[0] != gridDim.x - 1) return;
    const unsigned long long tl0 = gtimer();
    if constexpr (nbins == kPThreads) {  // the narrow digit: one bin per thread, in registers
        // one bin per thread: warp scans, the warps' totals
        // through shared memory -- two block barriers per scan stage, coalesced
        // loads and stores, a handful of registers
        __threadfence();
        const int d = threadIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        constexpr int kW = kPThreads / 32;
        unsigned long long* wt = sm.u.hist.w;  // [kW][4] warp totals (the histogram is no longer needed)
        const unsigned long long packed = __ldcg(&a.sm_cs[d]);
        const unsigned long long vw = __ldcg(&a.sm_w[d]);
        const unsigned int vc = static_cast<unsigned int>(packed >> 32);
        const unsigned long long vs = packed & 0xffffffffull;
        // stage 1: counts, tokens, chain sizes (exclusive prefixes), max count
        unsigned long long xc = vc, xw = vw, xs = vs;
        unsigned int mx = vc;
    #pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long yc = __shfl_up_sync(0xffffffffu, xc, o);
            const unsigned long long yw = __shfl_up_sync(0xffffffffu, xw, o);
            const unsigned long long ys = __shfl_up_sync(0xffffffffu, xs, o);
            if (lane >= o) {
                xc += yc;
                xw += yw;
                xs += ys;
            }
            mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (lane == 31) {
            wt[warp * 4 + 0] = xc;
            wt[warp * 4 + 1] = xw;
            wt[warp * 4 + 2] = xs;
            wt[warp * 4 + 3] = mx;
        }
        __syncthreads();
        unsigned long long pc = 0, pw = 0, ps = 0, tw = 0;
        unsigned int mxa = 0;
        for (int w = 0; w < kW; ++w) {
            if (w < warp) {
                pc += wt[w * 4 + 0];
                pw += wt[w * 4 + 1];
                ps += wt[w * 4 + 2];
            }
            tw += wt[w * 4 + 1];
            mxa = max(mxa, static_cast<unsigned int>(wt[w * 4 + 3]));
        }
        const unsigned long long ex_c = pc + xc - vc, ex_w = pw + xw - vw, ex_s = ps + xs - vs;
        const unsigned long long need = static_cast<unsigned long long>(a.needed);
        if (!(tw >= need && mxa <= static_cast<unsigned int>(kBucketCap))) {  // uniform
            if (threadIdx.x == 0) {
                a.ss->small_ok = 2;
                a.ss->path = tw >= need ? 4 : 3;  // bucket too large / bound too low
                a.ss->dbg[5] = tw;
                a.ss->dbg[6] = mxa;
            }
            return;
        }
        // stage 2: the buckets ranked by tiles (> 32 heads, not wholly after the
        // cut): their list positions and first rank tasks
        const bool big = vc > 32u && ex_w < need;
        const unsigned long long tk = big ? (vc + kChunkS - 1) / kChunkS : 0u;
        unsigned long long xb = big ? 1u : 0u, xt = tk;
    #pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long yb = __shfl_up_sync(0xffffffffu, xb, o);
            const unsigned long long yt = __shfl_up_sync(0xffffffffu, xt, o);
            if (lane >= o) {
                xb += yb;
                xt += yt;
            }
        }
        __syncthreads();  // wt is rewritten
        if (lane == 31) {
            wt[warp * 4 + 0] = xb;
            wt[warp * 4 + 1] = xt;
        }
        __syncthreads();
        unsigned long long pb = 0, pt = 0, tb = 0, tt = 0;
        for (int w = 0; w < kW; ++w) {
            if (w < warp) {
                pb += wt[w * 4 + 0];
                pt += wt[w * 4 + 1];
            }
            tb += wt[w * 4 + 0];
            tt += wt[w * 4 + 1];
        }
        a.sm_c[d] = vc;
        a.sm_off[d] = static_cast<unsigned int>(ex_c);
        a.sm_wpre[d] = ex_w;
        a.sm_cpre[d] = ex_s;
        if (big) {
            const unsigned long long q = pb + xb - 1u;
            a.sm_big[3 * q] = static_cast<unsigned int>(d);
            a.sm_big[3 * q + 1] = static_cast<unsigned int>(ex_c);
            a.sm_big[3 * q + 2] = vc;
            a.sm_task[q] = static_cast<unsigned int>(pt + xt - tk);
        }
        if (threadIdx.x == 0) {
            a.ss->n_big = static_cast<unsigned int>(tb);
            a.ss->n_task = static_cast<unsigned int>(tt);
            a.ss->small_ok = 1;
            a.ss->path = 1;
            a.ss->dbg2[1] = gtimer() - tl0;
        }
    } else {
    // kPer = nbins / kPThreads consecutive bins per thread (4): thread
    // sums, warp scans, the warps' totals through shared memory; the bins'
    // values are re-read from L2 in each pass (no per-bin register arrays)
    __threadfence();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int kPer = nbins / kPThreads;
    const int d0 = threadIdx.x * kPer;
    constexpr int kW = kPThreads / 32;
    // the CTA's own histogram is flushed: its shared arrays hold the global
    // bins (each thread its own, read once from L2) and the warp totals
    unsigned long long* bw_sh = sm.u.hist.w;   // [nbins] tokens
    unsigned long long* bcs_sh = sm.u.hist.cs;  // [nbins] count << 32 | chain sizes
    unsigned long long* wt = reinterpret_cast<unsigned long long*>(sm.u.hist.c);  // [kW][4] warp totals
    for (int i = 0; i < kPer; ++i) {
        bw_sh[d0 + i] = __ldcg(&a.sm_w[d0 + i]);
        bcs_sh[d0 + i] = __ldcg(&a.sm_cs[d0 + i]);
    }
    auto bin = [&](int d, unsigned long long& vc, unsigned long long& vw, unsigned long long& vs) {
        const unsigned long long packed = bcs_sh[d];
        vw = bw_sh[d];
        vc = packed >> 32;
        vs = packed & 0xffffffffull;
    };
    // stage 1: counts, tokens, chain sizes (exclusive prefixes), max count
    unsigned long long tc = 0, tw_ = 0, ts = 0;
    unsigned int mx = 0;
    for (int i = 0; i < kPer; ++i) {
        unsigned long long vc, vw, vs;
        bin(d0 + i, vc, vw, vs);
        tc += vc;
        tw_ += vw;
        ts += vs;
        mx = max(mx, static_cast<unsigned int>(vc));
    }
    unsigned long long xc = tc, xw = tw_, xs = ts;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long yc = __shfl_up_sync(0xffffffffu, xc, o);
        const unsigned long long yw = __shfl_up_sync(0xffffffffu, xw, o);
        const unsigned long long ys = __shfl_up_sync(0xffffffffu, xs, o);
        if (lane >= o) {
            xc += yc;
            xw += yw;
            xs += ys;
        }
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 31) {
        wt[warp * 4 + 0] = xc;
        wt[warp * 4 + 1] = xw;
        wt[warp * 4 + 2] = xs;
        wt[warp * 4 + 3] = mx;
    }
    __syncthreads();
    unsigned long long pc = 0, pw = 0, ps = 0, tw = 0;
    unsigned int mxa = 0;
    for (int w = 0; w < kW; ++w) {
        if (w < warp) {
            pc += wt[w * 4 + 0];
            pw += wt[w * 4 + 1];
            ps += wt[w * 4 + 2];
        }
        tw += wt[w * 4 + 1];
        mxa = max(mxa, static_cast<unsigned int>(wt[w * 4 + 3]));
    }
    const unsigned long long bc0 = pc + xc - tc, bw0 = pw + xw - tw_, bs0 = ps + xs - ts;  // the thread's first bin
    const unsigned long long need = static_cast<unsigned long long>(a.needed);
    if (!(tw >= need && mxa <= static_cast<unsigned int>(kBucketCap))) {  // uniform
        if (threadIdx.x == 0) {
            a.ss->small_ok = 2;
            a.ss->path = tw >= need ? 4 : 3;  // bucket too large / bound too low
            a.ss->dbg[5] = tw;
            a.ss->dbg[6] = mxa;
        }
        return;
    }
    // stage 2: the buckets ranked by tiles (> 32 heads, not wholly after the
    // cut): their list positions and first rank tasks
    unsigned long long nbt = 0, ntt = 0;
    {
        unsigned long long ew = bw0;
        for (int i = 0; i < kPer; ++i) {
            unsigned long long vc, vw, vs;
            bin(d0 + i, vc, vw, vs);
            if (vc > 32u && ew < need) {
                nbt += 1;
                ntt += (vc + kChunkS - 1) / kChunkS;
            }
            ew += vw;
        }
    }
    unsigned long long xb = nbt, xt = ntt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long yb = __shfl_up_sync(0xffffffffu, xb, o);
        const unsigned long long yt = __shfl_up_sync(0xffffffffu, xt, o);
        if (lane >= o) {
            xb += yb;
            xt += yt;
        }
    }
    __syncthreads();  // wt is rewritten
    if (lane == 31) {
        wt[warp * 4 + 0] = xb;
        wt[warp * 4 + 1] = xt;
    }
    __syncthreads();
    unsigned long long pb = 0, pt = 0, tb = 0, tt = 0;
    for (int w = 0; w < kW; ++w) {
        if (w < warp) {
            pb += wt[w * 4 + 0];
            pt += wt[w * 4 + 1];
        }
        tb += wt[w * 4 + 0];
        tt += wt[w * 4 + 1];
    }
    {
        unsigned long long ec = bc0, ew = bw0, es = bs0, q = pb + xb - nbt, tq = pt + xt - ntt;
        for (int i = 0; i < kPer; ++i) {
            const int d = d0 + i;
            unsigned long long vc, vw, vs;
            bin(d, vc, vw, vs);
            a.sm_c[d] = static_cast<unsigned int>(vc);
            a.sm_off[d] = static_cast<unsigned int>(ec);
            a.sm_wpre[d] = ew;
            a.sm_cpre[d] = es;
            if (vc > 32u && ew < need) {
                a.sm_big[3 * q] = static_cast<unsigned int>(d);
                a.sm_big[3 * q + 1] = static_cast<unsigned int>(ec);
                a.sm_big[3 * q + 2] = static_cast<unsigned int>(vc);
                a.sm_task[q] = static_cast<unsigned int>(tq);
                ++q;
                tq += (vc + kChunkS - 1) / kChunkS;
            }
            ec += vc;
            ew += vw;
            es += vs;
        }
    }
    if (threadIdx.x == 0) {
        a.ss->n_big = static_cast<unsigned int>(tb);
        a.ss->n_task = static_cast<unsigned int>(tt);
        a.ss->small_ok = 1;
        a.ss->path = 1;
        a.ss->dbg2[1] = gtimer() - tl0;
    }
    }
}

// a ranked low head: a selected one scatters its chain at its victim offset;
// the head whose running token count crosses `needed` scatters the cut part of
// its chain and finishes the decision (do_cut's work)
__device__ __forceinline__ void small_place_head(const SelArgs& a, int x, unsigned long long cw,
                                                 unsigned long long w_before, unsigned long long c_before) {
    const unsigned long long need = static_cast<unsigned long long>(a.needed);
    if (w_before >= need) return;
    const unsigned long long wx = cw >> 24;
    unsigned long long at = c_before;
    if (w_before + wx < need) {  // the whole chain
        int v = x;
        for (;;) {
            a.victims[at++] = v;
            v = a.parent[v];
            if (v <= 0) break;
            const bool ok = (a.flags[v] & (kFlagTierMask | kFlagOutOfOrder)) == PBKV_TIER_DEVICE &&
                            !__ldcg(&a.sublock[v]) && __ldcg(&a.eff[v]) == x;
            if (!ok) break;
        }
        return;
    }
    // the cut chain: its nodes until the running total reaches need
    const unsigned long long need_c = need - w_before;
    unsigned long long acc = 0;
    int v = x;
    for (;;) {
        a.victims[at++] = v;
        acc += static_cast<unsigned long long>(a.len[v]);
        if (acc >= need_c) break;
        v = a.parent[v];  // the chain holds >= need_c tokens: v stays in it
    }
    SelState* ss = a.ss;
    ss->n_S = 0;
    ss->cut_head = x;
    ss->need_final = need_c;
    ss->n_victims = at;
    ss->freed = w_before + acc;
    ss->shortfall = 0;
    a.result[0] = static_cast<long long>(at);
    a.result[1] = static_cast<long long>(w_before + acc);
    a.result[2] = 0;
    if (a.n_report > 0) a.rep_out[a.n_report] = report_tail(a.keys, a.eff, a.depth, a.victims, static_cast<long long>(at));
}

// S1..S3.  Returns false (uniformly) when the low list cannot hold the cut or
// does not fit the small path's limits; nothing has been written then.
__device__ bool small_path(const SelArgs& a, PersistSmem& sm, const GridBar& grid, int& nts,
                           unsigned long long total_tok) {
    SelState* ss = a.ss;
    if (threadIdx.x == 0) {
        sm.bc[0] = __ldcg(&ss->n_low);
        sm.bc[1] = __ldcg(&ss->or_low[0]) ^ __ldcg(&ss->and_low[0]);
        sm.bc[2] = __ldcg(&ss->or_low[1]) ^ __ldcg(&ss->and_low[1]);
        sm.bc[3] = (__ldcg(&ss->or_low[2]) ^ __ldcg(&ss->and_low[2])) & 0xffffffffull;
    }
    __syncthreads();
    const unsigned long long n_low = sm.bc[0];
    const unsigned long long v0 = sm.bc[1], v1 = sm.bc[2], v2 = sm.bc[3];
    const bool ovf = __ldcg(&ss->low_overflow) != 0u;
    __syncthreads();
    const int nbits = __popcll(v0) + __popcll(v1) + __popcll(v2);
    // packed keys, chain weight < 2^40 and chain size < 2^24 packed in one word
    if (n_low == 0 || ovf || nbits > 64 || total_tok >= (1ull << 40) || a.n_nodes >= (1ll << 24)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            ss->path = 2;
            ss->dbg[7] = static_cast<unsigned long long>(nbits);
        }
        return false;
    }
    const int sb = n_low > kSWideAt ? kSBitsWide : kSBits;  // uniform: every CTA read the same n_low
    const int nbins = 1 << sb;
    const int lo = nbits > sb ? nbits - sb : 0;
    if (sb == kSBits)
        small_hist<1 << kSBits>(a, n_low, lo, v0, v1, v2, sm);
    else
        small_hist<1 << kSBitsWide>(a, n_low, lo, v0, v1, v2, sm);
    grid.sync();
    stamp(ss, nts);
    // S2: the layout the last S1 CTA wrote; the check that the cut lies among
    // the low heads (uniform: every CTA reads the same flag)
    const unsigned long long s2t0 = gtimer();
    if (threadIdx.x == 0) sm.bc[0] = __ldcg(&ss->small_ok);
    __syncthreads();
    if (sm.bc[0] != 1) return false;
    {
        const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
        for (unsigned long long base = blockIdx.x * static_cast<unsigned long long>(blockDim.x); base < n_low;
             base += stride) {
            const unsigned long long i = base + threadIdx.x;
            int x = 0, d = -1;
            unsigned long long pk = 0, cw = 0;
            if (i < n_low) {
                x = __ldcg(&a.low[i]);
                pk = pack_key(load_key(a.keys, x), x, v0, v1, v2);
                d = static_cast<int>((pk >> lo) & static_cast<unsigned long long>(nbins - 1));
                cw = (chain_w(a, x) << 24) | static_cast<unsigned long long>(chain_c(a, x));
            }
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            if (d >= 0) {
                const int lane = threadIdx.x & 31, leader = __ffs(peers) - 1;
                unsigned int b = 0;
                if (lane == leader) b = atomicAdd(&a.sm_cur[d], static_cast<unsigned int>(__popc(peers)));
                b = __shfl_sync(peers, b, leader);
                const unsigned int pos = __ldcg(&a.sm_off[d]) + b + __popc(peers & ((1u << lane) - 1u));
                a.listS[pos] = x;
                a.listSK[pos] = make_ulonglong2(pk, cw);
            }
        }
    }
    if (threadIdx.x == 0) atomicMax(&ss->dbg[4], gtimer() - s2t0);  // S2 total, slowest CTA
    grid.sync();
    stamp(ss, nts);
    // S3: rank every bucket with the token / chain-size prefixes of the smaller
    // keys; selected heads scatter their chains, the crossing head the cut
    {
        const int lane = threadIdx.x & 31;
        const int gwarp = static_cast<int>((blockIdx.x * static_cast<unsigned int>(blockDim.x) + threadIdx.x) >> 5);
        const int nwarps = static_cast<int>((gridDim.x * static_cast<unsigned int>(blockDim.x)) >> 5);
        for (int d = gwarp; d < nbins; d += nwarps) {
            const unsigned int cnt = __ldcg(&a.sm_c[d]);
            if (cnt == 0u || cnt > 32u) continue;
            const unsigned long long wpre = __ldcg(&a.sm_wpre[d]);
            if (wpre >= static_cast<unsigned long long>(a.needed)) continue;  // wholly after the cut
            const unsigned int off = __ldcg(&a.sm_off[d]);
            const bool in = static_cast<unsigned int>(lane) < cnt;
            ulonglong2 kc = make_ulonglong2(0ull, 0ull);
            int x = 0;
            if (in) {
                kc = __ldcg(&a.listSK[off + lane]);
                x = __ldcg(&a.listS[off + lane]);
            }
            unsigned long long wb = 0, cb = 0;
            for (unsigned int j = 0; j < cnt; ++j) {
                const unsigned long long kj = __shfl_sync(0xffffffffu, kc.x, j);
                const unsigned long long cj = __shfl_sync(0xffffffffu, kc.y, j);
                if (kj < kc.x) {
                    wb += cj >> 24;
                    cb += cj & 0xffffffull;
                }
            }
            if (in) small_place_head(a, x, kc.y, wpre + wb, __ldcg(&a.sm_cpre[d]) + cb);
        }
        // larger buckets: rank counting from a shared-memory tile, 8 threads per
        // element; tasks (bucket, 64-element chunk) over every CTA, the first
        // task of every bucket precomputed by the last S1 CTA
        if (threadIdx.x == 0) {
            sm.bc[0] = __ldcg(&ss->n_big);
            sm.bc[1] = __ldcg(&ss->n_task);
        }
        __syncthreads();
        const unsigned int n_big = static_cast<unsigned int>(sm.bc[0]);
        const unsigned long long ttot = sm.bc[1];
        for (unsigned int q = threadIdx.x; q < n_big; q += blockDim.x) sm.off[q] = __ldcg(&a.sm_task[q]);
        __syncthreads();
        if (n_big > 0) {
            unsigned int held = ~0u;
            for (unsigned int t = blockIdx.x; t < static_cast<unsigned int>(ttot); t += gridDim.x) {
                unsigned int blo = 0, bhi = n_big - 1;  // last bucket whose first task is <= t
                while (blo < bhi) {
                    const unsigned int mid = (blo + bhi + 1) >> 1;
                    if (sm.off[mid] <= t) blo = mid;
                    else bhi = mid - 1;
                }
                const unsigned int b = blo, c = t - sm.off[b];
                const unsigned int dg = __ldcg(&a.sm_big[3 * b]), off = __ldcg(&a.sm_big[3 * b + 1]),
                                   cnt = __ldcg(&a.sm_big[3 * b + 2]);
                if (held != b) {
                    __syncthreads();
                    for (unsigned int q = threadIdx.x; q < cnt; q += blockDim.x) {
                        const ulonglong2 kc = __ldcg(&a.listSK[off + q]);
                        sm.u.sort.k0[q] = kc.x;
                        sm.u.sort.k1[q] = kc.y;
                    }
                    __syncthreads();
                    held = b;
                }
                const unsigned int e = c * kChunkS + threadIdx.x / 8, part = threadIdx.x % 8;
                const bool in = e < cnt;
                const unsigned long long mk = in ? sm.u.sort.k0[e] : 0ull;
                unsigned long long wb = 0, cb = 0;
                if (in) {
                    for (unsigned int q = part; q < cnt; q += 8) {
                        if (sm.u.sort.k0[q] < mk) {
                            const unsigned long long cq = sm.u.sort.k1[q];
                            wb += cq >> 24;
                            cb += cq & 0xffffffull;
                        }
                    }
                }
#pragma unroll
                for (int o = 1; o < 8; o <<= 1) {
                    wb += __shfl_xor_sync(0xffffffffu, wb, o);
                    cb += __shfl_xor_sync(0xffffffffu, cb, o);
                }
                if (in && part == 0)
                    small_place_head(a, __ldcg(&a.listS[off + e]), sm.u.sort.k1[e], __ldcg(&a.sm_wpre[dg]) + wb,
                                     __ldcg(&a.sm_cpre[dg]) + cb);
            }
        }
        // deferred-heavy reports by the CTAs at the top of the grid
        for (int j = static_cast<int>(gridDim.x) - 1 - static_cast<int>(blockIdx.x); j < a.n_report;
             j += static_cast<int>(gridDim.x))
            report_heavy_block(j, a.heavy, a.hch_off, a.hch, a.keys, a.eff, a.sublock, a.depth, a.flags, a.hmiss,
                               a.rep_out, a.approx, a.approx_out);
    }
    stamp(ss, nts);
    return true;
}

// ---- oversized buckets: MSD refinement ------------------------------
// Rank counting costs O(cnt^2) per bucket, so a bucket of S with more than
// kRankCap heads is split first: by a digit window (up to 11 bits) that
// starts at its own top varying key bit, sized for pieces of ~2^kRfPieceLog
// heads, round after round until every piece fits.  A round is OR/AND of the
// key words -> digit histogram -> piece offsets -> scatter -> copy back (five
// grid phases), with shared-memory aggregation per CTA (a CTA's contiguous
// slice of the round's heads covers one bucket or a few).  Pieces of <= 32
// heads go to the warp sorts, of <= kRankCap to the rank-counting sorts,
// larger ones to the next round.  A round consumes at least the bucket's top
// varying bit, and every live bucket holds more than kRankCap heads, so a
// round has at most n / (kRankCap + 1) buckets.
constexpr int kRfPieceLog = 7;                                 // digit width aimed at ~128-head pieces
constexpr int kRfSh = 8192;                                   // descriptors cached per CTA (prefix, offset)
constexpr int kRfLoc = 256;                                    // buckets one CTA's slice may span
static_assert(2 * kRfSh * 4 + kRfLoc * 13 * 4 <= static_cast<int>(sizeof(unsigned long long) * 2 * kBucketCap +
                                                                  sizeof(int) * kBucketCap),
              "refinement scratch exceeds the sort arrays");

// largest j with pre[j] <= v (pre strictly ascending, pre[0] = 0)
__device__ __forceinline__ unsigned int rf_find(const unsigned int* pre, unsigned int n, unsigned int v) {
    unsigned int lo = 0, hi = n - 1;
    while (lo < hi) {
        const unsigned int mid = (lo + hi + 1) >> 1;
        if (pre[mid] <= v) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ void rf_init_bucket(const SelArgs& a, int par, unsigned int q, unsigned int off,
                                               unsigned int cnt) {
    const std::size_t b = static_cast<std::size_t>(par) * a.rf_cap + q;
    a.rf_off[b] = off;
    a.rf_cnt[b] = cnt;
    for (int w = 0; w < 3; ++w) {
        a.rf_orand[b * 6 + w] = 0ull;
        a.rf_orand[b * 6 + 3 + w] = ~0ull;
    }
}

// Splits every bucket of S above kRankCap (all CTAs).  take_all: S is the
// unsorted head list (no keys listed yet), one bucket.  A round with more
// buckets than a CTA caches (kRfSh) runs window by window.  Returns false
// (grid-uniform) only when a CTA's slice would span more than kRfLoc
// buckets: the caller falls back to the device-wide sort.
__device__ bool refine_buckets(const SelArgs& a, PersistSmem& sm, const GridBar& grid, int& nts, bool take_all,
                               unsigned long long nS) {
    SelState* ss = a.ss;
    const std::int64_t tid = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
    const std::int64_t nthr = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    const int lane = threadIdx.x & 31;
    int* S = a.listS;
    if (take_all) {  // the head list with its keys and chain sizes, as the compaction lists S
        for (std::int64_t i = tid; i < static_cast<std::int64_t>(nS); i += nthr) {
            const int x = __ldcg(&a.heads[i]);
            const Key2 k = load_key(a.keys, x);
            S[i] = x;
            a.listSK[i] = make_ulonglong2(k.w0, k.w1);
            a.listSC[i] = chain_c(a, x);
        }
        if (tid == 0) {
            ss->s_is_heads = 0;
            ss->n_rf[0] = 1;
            rf_init_bucket(a, 0, 0, 0u, static_cast<unsigned int>(nS));
        }
    } else if (blockIdx.x == 0) {  // oversized buckets leave the rank-sort list (count 0: no tasks)
        const unsigned int nb = __ldcg(&ss->n_big);
        for (unsigned int q = threadIdx.x; q < nb; q += blockDim.x) {
            const unsigned int cnt = __ldcg(&a.big[2 * q + 1]);
            if (cnt > static_cast<unsigned int>(kRankCap)) {
                const unsigned int r = atomicAdd(&ss->n_rf[0], 1u);
                if (r < a.rf_cap) rf_init_bucket(a, 0, r, __ldcg(&a.big[2 * q]), cnt);
                a.big[2 * q + 1] = 0u;
            }
        }
    }
    grid.sync();
    stamp(ss, nts);
    unsigned int* pre = reinterpret_cast<unsigned int*>(&sm.u.sort);  // [kRfSh]
    unsigned int* offs = pre + kRfSh;                                  // [kRfSh]
    unsigned int* lo_sh = offs + kRfSh;  // [kRfLoc] (window low bit << 4) | width, per local bucket
    unsigned int (*oa_sh)[12] = reinterpret_cast<unsigned int (*)[12]>(lo_sh + kRfLoc);  // OR / AND halves
    unsigned int* hloc = sm.off;                                       // [kBins] this CTA's digit counts / cursors
    for (int par = 0;; par ^= 1) {
        const int nx = par ^ 1;
        if (threadIdx.x == 0) sm.bc[0] = __ldcg(&ss->n_rf[par]);
        __syncthreads();
        const unsigned int nr = static_cast<unsigned int>(sm.bc[0]);
        __syncthreads();
        if (nr == 0) break;
        if (nr > a.rf_cap) return false;
        // the round's buckets, a window of at most kRfSh at a time (the
        // descriptors a CTA caches; the histogram rows are per window)
        for (unsigned int jb = 0; jb < nr; jb += kRfSh) {
        const unsigned int n = min(static_cast<unsigned int>(kRfSh), nr - jb);
        const std::size_t rb = static_cast<std::size_t>(par) * a.rf_cap + jb;  // the window's descriptors
        // the window's descriptors and their prefix, per CTA
        unsigned int total = 0;
        for (unsigned int t0 = 0; t0 < n; t0 += blockDim.x) {
            const unsigned int j = t0 + threadIdx.x;
            const unsigned int c = j < n ? __ldcg(&a.rf_cnt[rb + j]) : 0u;
            unsigned int tile = 0;
            const unsigned int ex = block_excl_u32(c, sm.sh, &tile);
            if (j < n) {
                pre[j] = total + ex;
                offs[j] = __ldcg(&a.rf_off[rb + j]);
            }
            total += tile;
        }
        __syncthreads();
        if (threadIdx.x == 0 && blockIdx.x == 0 && jb == 0) {
            ss->n_rf[nx] = 0;
            ss->rf_rounds += 1;
        }
        // the window's histogram rows, zeroed (read after the next barrier)
        for (unsigned int j = blockIdx.x; j < n; j += gridDim.x)
            for (unsigned int d = threadIdx.x; d < static_cast<unsigned int>(kBins); d += blockDim.x)
                a.rf_hist[static_cast<std::size_t>(j) * kBins + d] = 0u;
        // this CTA's contiguous slice of the round's heads and the buckets it spans
        const unsigned int chunk = (total + gridDim.x - 1) / gridDim.x;
        if (chunk / (kRankCap + 1) + 2 > static_cast<unsigned int>(kRfLoc)) return false;
        const unsigned int v0 = min(total, blockIdx.x * chunk), v1 = min(total, v0 + chunk);
        const unsigned int j0 = v0 < v1 ? rf_find(pre, n, v0) : 0u;
        const unsigned int nloc = v0 < v1 ? rf_find(pre, n, v1 - 1) - j0 + 1 : 0u;
        const bool single = nloc == 1;
        for (unsigned int t = threadIdx.x; t < nloc * 12; t += blockDim.x)
            oa_sh[t / 12][t % 12] = (t % 12) < 6 ? 0u : ~0u;
        __syncthreads();
        // (A) OR / AND of the key words per bucket: warp, then CTA, then one
        // global atomic per word and bucket
        for (unsigned int vb = v0; vb < v1; vb += blockDim.x) {
            const unsigned int v = vb + threadIdx.x;
            const bool in = v < v1;
            unsigned int j = 0;
            Key2 k{0, 0};
            int x = 0;
            if (in) {
                j = rf_find(pre, n, v);
                const unsigned int i = offs[j] + (v - pre[j]);
                const ulonglong2 kk = __ldcg(&a.listSK[i]);
                k = Key2{kk.x, kk.y};
                x = __ldcg(&S[i]);
            }
            const unsigned peers = __match_any_sync(0xffffffffu, in ? j : 0xffffffffu);
            const bool lead = in && lane == __ffs(peers) - 1;
#pragma unroll
            for (int w = 0; w < 3; ++w) {
                const unsigned long long kw = key_word(k, x, w);
                const unsigned int ohi = __reduce_or_sync(peers, static_cast<unsigned int>(kw >> 32));
                const unsigned int olo = __reduce_or_sync(peers, static_cast<unsigned int>(kw));
                const unsigned int ahi = __reduce_and_sync(peers, static_cast<unsigned int>(kw >> 32));
                const unsigned int alo = __reduce_and_sync(peers, static_cast<unsigned int>(kw));
                if (lead) {
                    unsigned int* o = oa_sh[j - j0];
                    atomicOr(&o[2 * w], ohi);
                    atomicOr(&o[2 * w + 1], olo);
                    atomicAnd(&o[6 + 2 * w], ahi);
                    atomicAnd(&o[6 + 2 * w + 1], alo);
                }
            }
        }
        __syncthreads();
        for (unsigned int t = threadIdx.x; t < nloc * 6; t += blockDim.x) {
            const unsigned int jj = t / 6, w = t % 6;
            const unsigned long long val = (static_cast<unsigned long long>(oa_sh[jj][2 * w]) << 32) | oa_sh[jj][2 * w + 1];
            unsigned long long* g = a.rf_orand + (rb + j0 + jj) * 6 + w;
            if (w < 3) atomicOr(g, val);
            else atomicAnd(g, val);
        }
        grid.sync();
        stamp(ss, nts);
        // (B) each bucket's digit window from its top varying bit down, wide
        // enough for ~2^kRfPieceLog-head pieces; digit counts (in shared
        // memory when the slice lies in one bucket)
        for (unsigned int jj = threadIdx.x; jj < nloc; jj += blockDim.x) {
            const unsigned int j = j0 + jj;
            const int top = top_varying_bit_cg(a.rf_orand + (rb + j) * 6, a.rf_orand + (rb + j) * 6 + 3);
            const unsigned int cnt = (j + 1 < n ? pre[j + 1] : total) - pre[j];
            const int nb = min(kDigitBits, max(1, (32 - __clz(static_cast<int>(cnt - 1))) - kRfPieceLog));
            lo_sh[jj] = (static_cast<unsigned int>(max(0, top - nb + 1)) << 4) | static_cast<unsigned int>(nb);
        }
        if (single)
            for (unsigned int d = threadIdx.x; d < static_cast<unsigned int>(kBins); d += blockDim.x) hloc[d] = 0u;
        __syncthreads();
        for (unsigned int vb = v0; vb < v1; vb += blockDim.x) {
            const unsigned int v = vb + threadIdx.x;
            const bool in = v < v1;
            unsigned int key = 0xffffffffu, j = 0, d = 0;
            if (in) {
                j = rf_find(pre, n, v);
                const unsigned int i = offs[j] + (v - pre[j]);
                const ulonglong2 kk = __ldcg(&a.listSK[i]);
                const unsigned int lw = lo_sh[j - j0];
                d = key_bits(Key2{kk.x, kk.y}, __ldcg(&S[i]), static_cast<int>(lw >> 4), static_cast<int>(lw & 15u));
                key = (j << kDigitBits) | d;
            }
            const unsigned peers = __match_any_sync(0xffffffffu, key);
            if (in && lane == __ffs(peers) - 1) {
                if (single) atomicAdd(&hloc[d], static_cast<unsigned int>(__popc(peers)));
                else atomicAdd(&a.rf_hist[static_cast<std::size_t>(j) * kBins + d], static_cast<unsigned int>(__popc(peers)));
            }
        }
        __syncthreads();
        if (single)
            for (unsigned int d = threadIdx.x; d < static_cast<unsigned int>(kBins); d += blockDim.x)
                if (hloc[d]) atomicAdd(&a.rf_hist[static_cast<std::size_t>(j0) * kBins + d], hloc[d]);
        grid.sync();
        stamp(ss, nts);
        // (C) piece offsets (the histogram rows become placement cursors) and
        // the pieces' lists: warp sorts, rank sorts, next round
        for (unsigned int j = blockIdx.x; j < n; j += gridDim.x) {
            unsigned int* row = a.rf_hist + static_cast<std::size_t>(j) * kBins;
            constexpr int kPer = kBins / kPThreads;
            unsigned int c[kPer], s4 = 0;
#pragma unroll
            for (int q = 0; q < kPer; ++q) {
                c[q] = __ldcg(&row[threadIdx.x * kPer + q]);
                s4 += c[q];
            }
            unsigned int at = offs[j] + block_excl_u32(s4, sm.sh, nullptr);
#pragma unroll
            for (int q = 0; q < kPer; ++q) {
                row[threadIdx.x * kPer + q] = at;
                if (c[q] == 0u) {
                } else if (c[q] <= 32u) {
                    const unsigned int r = atomicAdd(&ss->n_rsmall, 1u);
                    a.rf_small[2 * r] = at;
                    a.rf_small[2 * r + 1] = c[q];
                } else if (c[q] <= static_cast<unsigned int>(kRankCap)) {
                    const unsigned int r = atomicAdd(&ss->n_big, 1u);
                    a.big[2 * r] = at;
                    a.big[2 * r + 1] = c[q];
                } else {
                    const unsigned int r = atomicAdd(&ss->n_rf[nx], 1u);
                    if (r < a.rf_cap) rf_init_bucket(a, nx, r, at, c[q]);
                }
                at += c[q];
            }
        }
        grid.sync();
        stamp(ss, nts);
        // (D) scatter into the pieces (staging: S2, the key buffer, SC2); a
        // one-bucket slice reserves its ranges with one atomic per digit
        if (single) {
            for (unsigned int d = threadIdx.x; d < static_cast<unsigned int>(kBins); d += blockDim.x)
                if (hloc[d]) hloc[d] = atomicAdd(&a.rf_hist[static_cast<std::size_t>(j0) * kBins + d], hloc[d]);
            __syncthreads();
        }
        for (unsigned int vb = v0; vb < v1; vb += blockDim.x) {
            const unsigned int v = vb + threadIdx.x;
            const bool in = v < v1;
            unsigned int key = 0xffffffffu, j = 0, d = 0, i = 0;
            Key2 k{0, 0};
            int x = 0;
            if (in) {
                j = rf_find(pre, n, v);
                i = offs[j] + (v - pre[j]);
                const ulonglong2 kk = __ldcg(&a.listSK[i]);
                k = Key2{kk.x, kk.y};
                x = __ldcg(&S[i]);
                const unsigned int lw = lo_sh[j - j0];
                d = key_bits(k, x, static_cast<int>(lw >> 4), static_cast<int>(lw & 15u));
                key = (j << kDigitBits) | d;
            }
            const unsigned peers = __match_any_sync(0xffffffffu, key);
            const int leader = __ffs(peers) - 1;
            unsigned int base = 0;
            if (in && lane == leader)
                base = single ? atomicAdd(&hloc[d], static_cast<unsigned int>(__popc(peers)))
                              : atomicAdd(&a.rf_hist[static_cast<std::size_t>(j) * kBins + d], static_cast<unsigned int>(__popc(peers)));
            base = __shfl_sync(peers, base, leader);
            if (in) {
                const unsigned int pos = base + __popc(peers & ((1u << lane) - 1u));
                a.listS2[pos] = x;
                a.rf_tmpk[pos] = make_ulonglong2(k.w0, k.w1);
                a.listSC2[pos] = __ldcg(&a.listSC[i]);
            }
        }
        grid.sync();
        stamp(ss, nts);
        // (E) copy back
        for (unsigned int vb = v0; vb < v1; vb += blockDim.x) {
            const unsigned int v = vb + threadIdx.x;
            if (v < v1) {
                const unsigned int j = rf_find(pre, n, v);
                const unsigned int i = offs[j] + (v - pre[j]);
                S[i] = __ldcg(&a.listS2[i]);
                a.listSK[i] = __ldcg(&a.rf_tmpk[i]);
                a.listSC[i] = __ldcg(&a.listSC2[i]);
            }
        }
        grid.sync();
        stamp(ss, nts);
        }  // window
    }
    return true;
}

__device__ __forceinline__ void select_body(const SelArgs& a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PersistSmem& sm = *reinterpret_cast<PersistSmem*>(smem_raw);
    const GridBar grid{a.gbar};
    SelState* ss = a.ss;
    const std::int64_t tid = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
    const std::int64_t nthr = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    int nts = 0;
    // initial selection state, written by CTA 0 before the first grid barrier
    // (no other CTA touches it earlier): no host->device copy per decision
    if (blockIdx.x == 0) {
        unsigned long long* w = reinterpret_cast<unsigned long long*>(ss);
        for (unsigned int i = threadIdx.x; i < sizeof(SelState) / 8; i += blockDim.x) w[i] = 0ull;
        __syncthreads();
        if (threadIdx.x == 0) {
            ss->need_final = static_cast<unsigned long long>(a.needed);
            for (int q = 0; q < 3; ++q) {
                ss->and_L[0][q] = ss->and_L[1][q] = ~0ull;
                ss->and_S[q] = ~0ull;
                ss->and_low[q] = ~0ull;
            }
            ss->cut_head = -1;
        }
    }

    stamp(ss, nts);
    // One phase: CTA 0 reads the node sample and sets the small-cut bound
    // while the other CTAs mark the locks and walk eff (independent: eff is
    // the subtree maximum of every device node, eligibility comes in the
    // chains phase).  Only CTA 0 touches the selection state before the
    // barrier (it initialised it above).
    // (a grid of one CTA -- small trees -- does the bound, then the walks)
    const bool solo = gridDim.x == 1;
    const unsigned long long tp0 = gtimer();
    if (blockIdx.x == 0) {
        const SmallBound b = small_bound(a, sm);
        if (threadIdx.x == 0) {
            ss->bound_w0 = b.k.w0;
            ss->bound_w1 = b.k.w1;
            ss->bound_id = b.ok ? b.id : -1;
            ss->dbg[5] = gtimer() - tp0;  // (diagnostics: the bound's time)
        }
    }
    if (blockIdx.x != 0 || solo) {
        if (threadIdx.x == 0) {
            sm.qctl[0] = 0u;
            sm.qctl[1] = 0u;
        }
        __syncthreads();
        // walkers queued per CTA: ~400 at C3, ~3 K at C4 on one GPU (overflow walks inline)
        constexpr int kQ = static_cast<int>(sizeof(sm.u.sort) / sizeof(int));
        const WalkQueue q{reinterpret_cast<int*>(&sm.u.sort), &sm.qctl[0], &sm.qctl[1], kQ};
        const std::int64_t t0 = solo ? tid : tid - kPThreads, nt = solo ? nthr : nthr - kPThreads;
        phase_lock(a, t0, nt);
        __syncthreads();
        if (threadIdx.x == 0) atomicMax(&ss->dbg[7], gtimer() - tp0);  // (diagnostics: the slowest lock marking)
        phase_eff(a, t0, nt, q);
        __syncthreads();
        if (threadIdx.x == 0) atomicMax(&ss->dbg[6], gtimer() - tp0);  // (diagnostics: the slowest walking CTA)
    }
    grid.sync();
    stamp(ss, nts);
    if (threadIdx.x == 0) {
        sm.bc[0] = __ldcg(&ss->bound_w0);
        sm.bc[1] = __ldcg(&ss->bound_w1);
        sm.bc[2] = static_cast<unsigned long long>(static_cast<long long>(__ldcg(&ss->bound_id)));
        reinterpret_cast<unsigned int*>(sm.u.sort.val)[0] = 0u;  // low-list counter
    }
    if (threadIdx.x < 6) sm.u.sort.k1[threadIdx.x] = threadIdx.x < 3 ? 0ull : ~0ull;  // low OR / AND
    __syncthreads();
    {
        const int bid = static_cast<int>(static_cast<long long>(sm.bc[2]));
        const LowSink lk{bid >= 0, Key2{sm.bc[0], sm.bc[1]}, bid, reinterpret_cast<int*>(sm.u.sort.k0),
                         reinterpret_cast<unsigned int*>(sm.u.sort.val), sm.u.sort.k1};
        __syncthreads();
        phase_chains(a, sm.sh, lk, !lk.on);
    }
    grid.sync();
    stamp(ss, nts);
    const bool listed = __ldcg(&ss->bound_id) < 0;  // the chains phase built the head list

    // shared scalars are read once per CTA and broadcast through shared memory
    // (thousands of threads reading one L2 line serialise on its slice)
    if (threadIdx.x == 0) {
        sm.bc[0] = listed ? __ldcg(&ss->n_L[0]) : __ldcg(&ss->n_heads_seen);
        sm.bc[1] = __ldcg(&ss->total_tok);
    }
    __syncthreads();
    const unsigned long long n_heads = sm.bc[0];
    const unsigned long long total_tok = sm.bc[1];
    __syncthreads();
    if (n_heads == 0) {  // nothing evictable
        if (tid == 0) {
            ss->n_victims = 0;
            ss->freed = 0;
            ss->shortfall = 1;
            a.result[0] = 0;
            a.result[1] = 0;
            a.result[2] = 1;
        }
        return;
    }
    const bool take_all = total_tok < static_cast<unsigned long long>(a.needed);
    if (!take_all && !listed && small_path(a, sm, grid, nts, total_tok)) return;
    if (!listed) {  // the small-cut path did not apply: the head list for the paths below
        phase_heads(a, sm.sh);
        grid.sync();
        stamp(ss, nts);
    }
    int* S = a.listS;
    unsigned long long nS = 0;
    unsigned int max_bucket = 0;
    int n_pass = 0;
    if (take_all) {
        // every head is a victim; S is the unsorted head list: one bucket
        S = a.heads;
        nS = n_heads;
        max_bucket = static_cast<unsigned int>(n_heads);
        if (tid == 0) {
            ss->take_all = 1;
            ss->s_is_heads = 1;
            ss->n_S = n_heads;
            for (int w = 0; w < 3; ++w) {
                ss->or_S[w] = __ldcg(&ss->or_L[0][w]);
                ss->and_S[w] = __ldcg(&ss->and_L[0][w]);
            }
        }
    } else {
        int* L = a.heads;
        int* L2 = a.listB;
        int cur = 0;
        unsigned long long need = static_cast<unsigned long long>(a.needed);
        for (; n_pass < kMaxPasses; ++n_pass) {
            if (threadIdx.x == 0) {
                sm.bc[0] = __ldcg(&ss->n_L[cur]);
                sm.bc[1] = static_cast<unsigned long long>(top_varying_bit_cg(ss->or_L[cur], ss->and_L[cur]) + 1);
            }
            __syncthreads();
            const unsigned long long nL = sm.bc[0];
            const int top = static_cast<int>(sm.bc[1]) - 1;
            __syncthreads();
            if (nL <= 1) break;
            const int lo = top - kDigitBits + 1 < 0 ? 0 : top - kDigitBits + 1;
            if (tid == 0) {  // the next candidate list's accumulators
                const int nx = cur ^ 1;
                ss->n_L[nx] = 0;
                for (int w = 0; w < 3; ++w) {
                    ss->or_L[nx][w] = 0;
                    ss->and_L[nx][w] = ~0ull;
                }
            }
            phase_hist(a, L, nL, lo, n_pass, sm.u.hist.w, sm.u.hist.c);
            grid.sync();
            stamp(ss, nts);
            const PickOut pk = phase_pick(a, need, n_pass, nS, &sm.u.scan, sm.off, &sm.pick);
            phase_compact(a, L, nL, L2, cur ^ 1, S, n_pass, lo, pk.bucket, sm.off, sm.sh);
            need = pk.need;
            nS += pk.below_cnt;
            max_bucket = max(max_bucket, pk.max_cnt);
            grid.sync();
            stamp(ss, nts);
            int* t = L;
            L = L2;
            L2 = t;
            cur ^= 1;
        }
        if (tid == 0) {  // the last candidate is the cut head (its own bucket)
            const int x = __ldcg(&L[0]);
            const Key2 k = load_key(a.keys, x);
            S[nS] = x;
            a.listSK[nS] = make_ulonglong2(k.w0, k.w1);
            a.listSC[nS] = chain_c(a, x);
            ss->n_S = nS + 1;
            ss->need_final = need;
            ss->n_pass = n_pass;
            for (int w = 0; w < 3; ++w) {
                ss->or_S[w] = __ldcg(&ss->or_S[w]) | key_word(k, x, w);
                ss->and_S[w] = __ldcg(&ss->and_S[w]) & key_word(k, x, w);
            }
            ss->cut_head = x;
        }
        nS += 1;
    }
    grid.sync();
    stamp(ss, nts);

    // ---- sort every bucket of S (rank counting over every CTA, warp sorts) ------------
    const bool refined = max_bucket > static_cast<unsigned int>(kRankCap);
    if (refined) {
        if (tid == 0) ss->max_bucket = static_cast<int>(max_bucket);
        if (a.no_refine || !refine_buckets(a, sm, grid, nts, take_all, nS)) {
            if (tid == 0) ss->host_sort = 1;  // device-wide sort driven from the host (> 16 M nodes)
            return;
        }
        S = a.listS;
    }
    int* S2 = a.listS2;
    if (take_all && !refined) {
        if (tid == 0 && nS > 0) {  // the whole head list is one bucket
            a.big[0] = 0u;
            a.big[1] = static_cast<unsigned int>(nS);
        }
        grid.sync();
        rank_sort_big(a, S, S2, nS > 0 ? 1u : 0u, sm.u.sort.k0, sm.u.sort.k1, sm.u.sort.val, false, sm.sh);
    } else {
        const unsigned long long t0 = gtimer();
        if (threadIdx.x == 0) sm.bc[3] = __ldcg(&ss->n_big);
        __syncthreads();
        const unsigned int n_big = static_cast<unsigned int>(sm.bc[3]);
        rank_sort_big(a, S, S2, n_big, sm.u.sort.k0, sm.u.sort.k1, sm.u.sort.val, true, sm.sh);
        const unsigned long long t1 = gtimer();
        if (threadIdx.x == 0) {
            atomicMax(&ss->dbg[0], t1 - t0);
            atomicMax(&ss->dbg[4], static_cast<unsigned long long>(n_big));
        }
        // small buckets: one warp each; singletons and the cut head are copied
        // (the compaction's buckets, then the refinement's pieces)
        if (threadIdx.x == 0) sm.bc[2] = refined ? __ldcg(&ss->n_rsmall) : 0ull;
        __syncthreads();
        const int nb = n_pass * kBins;
        const int nbr = nb + static_cast<int>(sm.bc[2]);
        const int gwarp = static_cast<int>((blockIdx.x * static_cast<unsigned int>(blockDim.x) + threadIdx.x) >> 5);
        const int nwarps = static_cast<int>((gridDim.x * static_cast<unsigned int>(blockDim.x)) >> 5);
        for (int j = gwarp; j < nbr; j += nwarps) {
            const unsigned int cnt = j < nb ? __ldcg(&a.seg_cnt[j]) : __ldcg(&a.rf_small[2 * (j - nb) + 1]);
            if (cnt == 0u || cnt > 32u) continue;
            const unsigned int off = j < nb ? __ldcg(&a.seg_off[j]) : __ldcg(&a.rf_small[2 * (j - nb)]);
            if (cnt == 1u) {
                if ((threadIdx.x & 31) == 0) {
                    S2[off] = __ldcg(&S[off]);
                    a.listSC2[off] = __ldcg(&a.listSC[off]);
                }
            } else {
                warp_sort_bucket(a, S, S2, off, cnt);
            }
        }
        if (tid == 0 && !take_all) {  // the cut head (its own bucket)
            S2[nS - 1] = __ldcg(&S[nS - 1]);
            a.listSC2[nS - 1] = __ldcg(&a.listSC[nS - 1]);
        }
        if ((threadIdx.x & 31) == 0) atomicMax(&ss->dbg[1], gtimer() - t1);
    }
    // deferred-heavy reports by the CTAs at the top of the grid (the bucket
    // sorts above occupy the bottom ones)
    for (int j = static_cast<int>(gridDim.x) - 1 - static_cast<int>(blockIdx.x); j < a.n_report;
         j += static_cast<int>(gridDim.x))
        report_heavy_block(j, a.heavy, a.hch_off, a.hch, a.keys, a.eff, a.sublock, a.depth, a.flags, a.hmiss,
                           a.rep_out, a.approx, a.approx_out);
    grid.sync();
    stamp(ss, nts);

    // ---- chain starts: start[p] = sum of the chain sizes before S2[p] ----------------
    // every CTA scans its own slice of S2.  The prefix before the slice is
    // recomputed redundantly by each CTA (sum of C over S2[0, c0)) for the
    // sizes a decision usually selects; above 64 K heads the slice sums go
    // through global memory instead (one more grid phase)
    {
        using Scan = cub::BlockScan<unsigned long long, kPThreads>;
        const bool spread = nS <= 65536ull;
        const unsigned long long per = (nS + gridDim.x - 1) / gridDim.x;
        const unsigned long long c0 = min(nS, blockIdx.x * per);
        const unsigned long long c1 = min(nS, c0 + per);
        unsigned long long carry = 0;
        if (!spread) {
            unsigned long long loc = 0;
            for (unsigned long long i = c0 + threadIdx.x; i < c1; i += blockDim.x) loc += __ldcg(&a.listSC2[i]);
            loc = block_reduce_bits(loc, SumOp(), sm.sh);
            if (threadIdx.x == 0) a.hist_w[blockIdx.x] = loc;  // (the radix passes' histograms are done)
            grid.sync();
            stamp(ss, nts);
            unsigned long long pre = 0;
            for (unsigned int q = threadIdx.x; q < blockIdx.x; q += blockDim.x) pre += __ldcg(&a.hist_w[q]);
            carry = block_reduce_bits(pre, SumOp(), sm.sh);
            if (threadIdx.x == 0) sm.bc[2] = carry;
            __syncthreads();
            carry = sm.bc[2];
            __syncthreads();
        } else if (c0 < c1) {
            unsigned long long pre = 0;
            // batches of 8 independent loads per thread (the prefix is L2-latency bound)
            for (unsigned long long i0 = static_cast<unsigned long long>(threadIdx.x) * 8; i0 < c0;
                 i0 += static_cast<unsigned long long>(blockDim.x) * 8) {
                int hb[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) hb[q] = i0 + q < c0 ? static_cast<int>(__ldcg(&a.listSC2[i0 + q])) : 0;
#pragma unroll
                for (int q = 0; q < 8; ++q) pre += static_cast<unsigned int>(hb[q]);
            }
            carry = block_reduce_bits(pre, SumOp(), sm.sh);
            if (threadIdx.x == 0) sm.bc[2] = carry;
            __syncthreads();
            carry = sm.bc[2];
        }
        for (unsigned long long b0 = c0; b0 < c1; b0 += static_cast<unsigned long long>(kPThreads) * kScanIPT) {
            unsigned long long cnt[kScanIPT], local = 0;
            int hv[kScanIPT];
            for (int j = 0; j < kScanIPT; ++j) {
                const unsigned long long pos = b0 + static_cast<unsigned long long>(threadIdx.x) * kScanIPT + j;
                cnt[j] = 0;
                hv[j] = -1;
                if (pos < c1) {
                    const int h = __ldcg(&S2[pos]);
                    hv[j] = h;
                    a.rank[h] = static_cast<int>(pos);
                    cnt[j] = __ldcg(&a.listSC2[pos]);
                }
                local += cnt[j];
            }
            unsigned long long excl, total;
            Scan(sm.u.scan).ExclusiveSum(local, excl, total);
            __syncthreads();
            excl += carry;
            for (int j = 0; j < kScanIPT; ++j) {
                const unsigned long long pos = b0 + static_cast<unsigned long long>(threadIdx.x) * kScanIPT + j;
                if (pos < c1) a.start[pos] = excl;
                excl += cnt[j];
                if (pos < c1 && pos == nS - 1 && take_all) ss->cut_head = hv[j];
            }
            carry += total;
        }
    }
    grid.sync();
    stamp(ss, nts);
    phase_scatter(a, a.listS2, nS, tid, nthr);
    grid.sync();
    stamp(ss, nts);
    if (tid == 0) do_cut(a);
    stamp(ss, nts);
}

// The decision's epilogue, after the last phase (every CTA): the victim ids
// (16-byte stores, when they fit h_cap; larger cuts are copied by DMA), the
// status word and the selection state straight into pinned host memory, and
// the heavy-node deferral cleared unless the host-sort fallback still needs it.
__device__ __forceinline__ void select_epilogue(const SelArgs& a) {
    const SelState* ss = a.ss;
    if (a.h_vict && !__ldcg(&ss->host_sort)) {
        const long long nv = static_cast<long long>(__ldcg(&ss->n_victims));
        if (nv <= a.h_cap) {
            const long long n4 = nv >> 2;
            const long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
            const long long nt = static_cast<long long>(gridDim.x) * blockDim.x;
            for (long long i = t; i < n4; i += nt)
                reinterpret_cast<int4*>(a.h_vict)[i] = __ldcg(reinterpret_cast<const int4*>(a.victims) + i);
            for (long long i = 4 * n4 + t; i < nv; i += nt) a.h_vict[i] = __ldcg(a.victims + i);
        }
    }
    if (blockIdx.x != 0) return;
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(ss);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(a.h_ss);
    for (unsigned int i = threadIdx.x; i < sizeof(SelState) / 8; i += blockDim.x) dst[i] = __ldcg(src + i);
    if (threadIdx.x == 0) *a.h_st = *a.st;
    if (__ldcg(&ss->host_sort)) return;
    for (int i = threadIdx.x; i < a.n_report; i += blockDim.x)
        a.flags_w[a.heavy[i]] &= static_cast<std::uint8_t>(~kFlagDeferred);
}

__global__ void __launch_bounds__(kPThreads, 2) select_persistent_kernel(SelArgs a) {
    select_body(a);
    const GridBar grid{a.gbar};
    grid.sync();  // every phase's writes (victims, result, state) before the epilogue reads them
    select_epilogue(a);
}

// ---- fallback path (a bucket larger than one CTA's sort) -----------------------------
__global__ void pack_keys_kernel(const int* S, const Key2* keys, const SelState* ss, unsigned long long* out,
                                 int* ids) {
    const unsigned long long n = ss->n_S;
    const unsigned long long v0 = ss->or_S[0] ^ ss->and_S[0];
    const unsigned long long v1 = ss->or_S[1] ^ ss->and_S[1];
    const unsigned long long v2 = (ss->or_S[2] ^ ss->and_S[2]) & 0xffffffffull;
    for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
        const int x = S[i];
        out[i] = pack_key(load_key(keys, x), x, v0, v1, v2);
        ids[i] = x;
    }
}

__global__ void gather_headkeys_kernel(const int* S, const Key2* keys, const SelState* ss, HeadKey* out) {
    const unsigned long long n = ss->n_S;
    for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
        const int x = S[i];
        const Key2 k = load_key(keys, x);
        out[i] = HeadKey{k.w0, k.w1, static_cast<unsigned int>(x), 0u};
    }
}

__global__ void heads_from_hk_kernel(const HeadKey* hk, const SelState* ss, int* out) {
    const unsigned long long n = ss->n_S;
    for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<unsigned long long>(gridDim.x) * blockDim.x)
        out[i] = static_cast<int>(hk[i].id);
}

__global__ void rank_kernel(const int* sorted, const unsigned int* C, SelState* ss, int* rank,
                            unsigned long long* cnt) {
    const unsigned long long n = ss->n_S;
    for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
        const int h = sorted[i];
        rank[h] = static_cast<int>(i);
        cnt[i] = C[h] + 1u;  // the head itself (see chain_c)
        if (i == n - 1 && ss->take_all) ss->cut_head = h;
    }
}

__global__ void __launch_bounds__(kThreads) scatter_kernel(SelArgs a) {
    phase_scatter(a, a.sorted, a.ss->n_S, blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x,
                  static_cast<std::int64_t>(gridDim.x) * blockDim.x);
}

__global__ void cut_kernel(SelArgs a) { do_cut(a); }

struct HeadDecomposer {
    __host__ __device__ ::cuda::std::tuple<unsigned long long&, unsigned long long&, unsigned int&> operator()(
        HeadKey& k) const {
        return {k.w0, k.w1, k.id};
    }
};

int persistent_grid(Context& c) {
    static int cached = 0;
    if (cached) return cached;
    int dev_sms = 0;
    PBKV_CUDA(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, c.device));
    const int smem = static_cast<int>(sizeof(PersistSmem));
    PBKV_CUDA(cudaFuncSetAttribute(select_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int per_sm = 0;
    PBKV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, select_persistent_kernel, kPThreads, smem));
    if (per_sm < 1) throw ApiError(PBKV_ECUDA, "persistent select kernel cannot be resident");
    cached = dev_sms * (per_sm >= 2 ? 2 : 1);
    return cached;
}

}  // namespace

std::size_t sel_state_bytes() { return sizeof(SelState); }

namespace {
// per deferred heavy node: max key over its non-deferred device descendants
// (eff after the walk; its own key is zeroed), lock status, missing
// forecasts; plus the record of the last victim of the cut (tail)
__global__ void __launch_bounds__(256) heavy_report_kernel(const int* heavy, int n_heavy, const int* ch_off,
                                                           const int* ch, const Key2* keys, const int* eff,
                                                           const int* sublock, const int* depth,
                                                           const std::uint8_t* flags, const unsigned int* hmiss,
                                                           const int* victims, const long long* result,
                                                           HeavyReport* out, const double* approx, double* approx_out) {
    // one CTA per heavy node; the last CTA writes the record of the last
    // victim (tail).  The persistent kernel does the same in place
    // (report_deferred decisions); this kernel serves the host-sort fallback.
    const int j = blockIdx.x;
    if (j < n_heavy)
        report_heavy_block(j, heavy, ch_off, ch, keys, eff, sublock, depth, flags, hmiss, out, approx, approx_out);
    else if (threadIdx.x == 0)
        out[j] = report_tail(keys, eff, depth, victims, result[0]);
}
}  // namespace

void launch_heavy_report(Context& c, long long* result_dev, HeavyReport* out, double* approx_out) {
    const int n = static_cast<int>(c.n_heavy);
    heavy_report_kernel<<<n + 1, 256, 0, c.stream>>>(c.heavy.p, n, c.hch_off.p, c.hch.p, c.keys.p,
                                                                   c.eff.p, c.sublock.p,
                                                                   c.depth.p, c.flags.p, c.hmiss.p, c.vid_out.p,
                                                                   result_dev, out, c.happrox.p, approx_out);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

void launch_keys_cached(Context& c, int policy) {
    KeyArgs ka = make_key_args(c, policy);
    keys_cached_kernel<<<grid_cap(c.n, kThreads), kThreads, 0, c.stream>>>(ka, c.n);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

// Runs lock -> eff -> chains -> select -> bucket sorts -> scan -> scatter ->
// cut.  Victims land in c.vid_out[0..n); result_dev (or an internal buffer)
// receives {n_victims, freed, shortfall}.  One host synchronisation at the end
// (plus the fallback sort's when a bucket exceeds one CTA's sort).
SelectCounts run_select(Context& c, const int* locked_dev, std::int64_t n_locked, std::int64_t needed,
                        bool he_recompute, long long* result_dev) {
    SelState* ss = reinterpret_cast<SelState*>(c.selstate.p);
    SelState* hs = reinterpret_cast<SelState*>(c.hselstate.p);
    // initial state from a pinned template (no kernel)
    // the initial state is written by the persistent kernel itself; the chain
    // weights / sizes (scatter-added in phase_chains) were zeroed by the keying
    // kernel (score_light_kernel / keys_cached_kernel)
    long long* res = result_dev ? result_dev : c.counters.p + 8;
    c.sorti_out.reserve(static_cast<std::size_t>(c.n) + 1);
    c.cnt.reserve(static_cast<std::size_t>(c.n) + 1);
    int grid = persistent_grid(c);
    {
        static const int forced = std::getenv("PBKV_SELECT_GRID") ? std::atoi(std::getenv("PBKV_SELECT_GRID")) : 0;
        if (forced > 0) grid = std::min(grid, forced);  // (experiments; measured: no gain at 10 K nodes)
    }
    c.hist_w.reserve(static_cast<std::size_t>(kMaxPasses) * kBins);
    c.hist_c.reserve(static_cast<std::size_t>(kMaxPasses) * kBins);
    c.seg_off.reserve(static_cast<std::size_t>(kMaxPasses) * kBins);
    c.seg_cnt.reserve(static_cast<std::size_t>(kMaxPasses) * kBins);
    c.cursor.reserve(static_cast<std::size_t>(kMaxPasses) * kBins);
    SelArgs a;
    a.parent = c.parent.p;
    a.len = c.len.p;
    a.flags = c.flags.p;
    a.depth = c.depth.p;
    a.keys = c.keys.p;
    a.eff = c.eff.p;
    a.sublock = c.sublock.p;
    a.missing = c.missing.p;
    a.W = c.W.p;
    a.C = c.C.p;
    a.rank = c.rank.p;
    a.heads = c.heads.p;
    a.listB = c.listB.p;
    a.listS = c.listS.p;
    a.listS2 = c.listS2.p;
    a.listSK = c.listSK.p;
    a.listSC = c.listSC.p;
    a.listSC2 = c.listSC2.p;
    a.big = c.big.p;
    a.sorted = c.sorti_out.p;
    a.start = c.cnt.p;
    a.victims = c.vid_out.p;
    a.hist_w = c.hist_w.p;
    a.hist_c = c.hist_c.p;
    a.seg_off = c.seg_off.p;
    a.seg_cnt = c.seg_cnt.p;
    a.cursor = c.cursor.p;
    a.ss = ss;
    a.st = c.status.p;
    a.result = res;
    a.locked = locked_dev;
    a.n_locked = n_locked;
    a.n_nodes = c.n;
    a.needed = needed;
    a.he_recompute = he_recompute ? 1 : 0;
    a.n_report = 0;
    {  // small-cut path: ~kSampTarget sampled nodes, its scratch
        unsigned int R = 1;
        while (static_cast<std::int64_t>(R) * kSampTarget < c.n) R <<= 1;
        a.samp_mask = R - 1;
        c.samp.reserve(kSamp * sizeof(SampRec));
        c.low.reserve(static_cast<std::size_t>(c.n) + 1);
        c.small_u32.reserve(7 * kBins);
        c.small_u64.reserve(4 * kBins);
        a.samp = reinterpret_cast<SampRec*>(c.samp.p);
        // the grid barrier's arrival counter: every launch leaves it at a
        // multiple of its grid size, so it is zeroed only when the grid changes
        c.gbar.reserve(1);
        if (c.gbar_grid != grid) {
            PBKV_CUDA(cudaMemsetAsync(c.gbar.p, 0, sizeof(unsigned long long), c.stream));
            c.gbar_grid = grid;
        }
        a.gbar = c.gbar.p;
        a.low = c.low.p;
        a.sm_c = c.small_u32.p;
        a.sm_cur = c.small_u32.p + kBins;
        a.sm_off = c.small_u32.p + 2 * kBins;
        a.sm_big = c.small_u32.p + 3 * kBins;
        a.sm_task = c.small_u32.p + 6 * kBins;
        a.sm_w = c.small_u64.p;
        a.sm_cs = c.small_u64.p + kBins;
        a.sm_wpre = c.small_u64.p + 2 * kBins;
        a.sm_cpre = c.small_u64.p + 3 * kBins;
    }
    {  // oversized-bucket refinement: a round has at most n / (kRankCap + 1) buckets
        // (descriptors for every bucket of a round; histogram rows for one
        // window of kRfSh buckets)
        const std::size_t cap = static_cast<std::size_t>(c.n) / (kRankCap + 1) + 2;
        c.rf_u32.reserve(4 * cap + static_cast<std::size_t>(kRfSh) * kBins);
        c.rf_orand.reserve(2 * cap * 6);
        c.rf_small.reserve(2 * static_cast<std::size_t>(c.n) + 2);
        c.rf_tmpk.reserve(static_cast<std::size_t>(c.n) + 1);
        a.rf_cap = static_cast<unsigned int>(cap);
        a.rf_off = c.rf_u32.p;
        a.rf_cnt = c.rf_u32.p + 2 * cap;
        a.rf_hist = c.rf_u32.p + 4 * cap;
        a.rf_orand = c.rf_orand.p;
        a.rf_small = c.rf_small.p;
        a.rf_tmpk = c.rf_tmpk.p;
    }
    if (c.report_deferred) {  // the deferred-heavy reports are written in place, to pinned memory
        const std::size_t nh = static_cast<std::size_t>(c.n_heavy);
        const std::size_t bytes = (nh + 1) * sizeof(HeavyReport);
        c.hreport_h.reserve(bytes + 2 * nh * sizeof(double));
        a.n_report = static_cast<int>(c.n_heavy);
        a.heavy = c.heavy.p;
        a.hch_off = c.hch_off.p;
        a.hch = c.hch.p;
        a.hmiss = c.hmiss.p;
        a.rep_out = reinterpret_cast<HeavyReport*>(c.hreport_h.p);
        a.approx = c.happrox.p;
        a.approx_out = reinterpret_cast<double*>(c.hreport_h.p + bytes);
    }
    {  // (tests: PBKV_SELECT_NO_REFINE=1 exercises the device-wide-sort fallback)
        const char* e = std::getenv("PBKV_SELECT_NO_REFINE");
        a.no_refine = e && e[0] == '1' ? 1 : 0;
    }
    a.h_st = c.hstatus.p;
    a.h_ss = hs;
    a.h_vict = c.epi_vict;
    a.h_cap = c.epi_cap;
    a.flags_w = c.flags.p;
    void* args[] = {&a};
    if (c.timing) {
        PBKV_CUDA(cudaEventRecord(c.kev[2], c.stream));
        c.kev_select = true;
    }
    PBKV_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(select_persistent_kernel), dim3(grid),
                                          dim3(kPThreads), args, sizeof(PersistSmem), c.stream));
    if (c.timing) PBKV_CUDA(cudaEventRecord(c.kev[3], c.stream));
    ++c.launches;
    // (the kernel's own epilogue stored the status, the selection state and
    // the victims into pinned memory and cleared the deferral)
    PBKV_CUDA(cudaStreamSynchronize(c.stream));
    {
        const DevStatus st = *c.hstatus.p;  // a copy: raising may reuse the pinned word
        raise_status(c, st);
    }
    c.deferred_cleared = c.report_deferred && !hs->host_sort;
    c.epi_vict_valid = c.epi_vict && !hs->host_sort && static_cast<long long>(hs->n_victims) <= c.epi_cap;
    SelectCounts out;
    c.phase_ns.assign(hs->ts, hs->ts + (hs->n_ts < 40 ? hs->n_ts : 40));
    if (std::getenv("PBKV_DEBUG_SELECT"))
        std::fprintf(stderr,
                     "[pbkv select] n_heads=%llu total_tok=%llu take_all=%d host_sort=%d n_S=%llu n_pass=%d "
                     "cut_head=%d need_final=%llu max_bucket=%d n_victims=%llu freed=%llu shortfall=%d grid=%d "
                     "path=%d low_ovf=%u n_low=%llu est_low=%llu n_big=%u rf_rounds=%u n_rsmall=%u "
                     "dbg(ns): sortCTA=%llu sortWarp=%llu loadpack=%llu rank=%llu nbig=%llu bound=%llu "
                     "walk_end=%llu lock_end=%llu s1_hist=%llu s1_layout=%llu\n",
                     hs->n_L[0], hs->total_tok, hs->take_all, hs->host_sort, hs->n_S, hs->n_pass, hs->cut_head,
                     hs->need_final, hs->max_bucket, hs->n_victims, hs->freed, hs->shortfall, grid, hs->path,
                     hs->low_overflow, hs->n_low, hs->est_low, hs->n_big, hs->rf_rounds, hs->n_rsmall, hs->dbg[0],
                     hs->dbg[1], hs->dbg[2], hs->dbg[3], hs->dbg[4], hs->dbg[5], hs->dbg[6], hs->dbg[7], hs->dbg2[0], hs->dbg2[1]);
    if (hs->host_sort) {
        // ---- fallback: device-wide sort of the selected heads -----------------------------
        const std::int64_t nS = static_cast<std::int64_t>(hs->n_S);
        const int* S = hs->s_is_heads ? c.heads.p : c.listS.p;
        int nbits = 0;
        for (int w = 0; w < 3; ++w) {
            unsigned long long v = hs->or_S[w] ^ hs->and_S[w];
            if (w == 2) v &= 0xffffffffull;
            nbits += __builtin_popcountll(v);
        }
        c.sortk_in.reserve(nS);
        c.sortk_out.reserve(nS);
        c.sorti_in.reserve(nS);
        int* sorted = c.sorti_out.p;
        if (nbits <= 64) {
            pack_keys_kernel<<<grid_cap(nS, kThreads), kThreads, 0, c.stream>>>(S, c.keys.p, ss, c.sortk_in.p,
                                                                               c.sorti_in.p);
            PBKV_CUDA(cudaGetLastError());
            ++c.launches;
            std::size_t b = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, b, c.sortk_in.p, c.sortk_out.p, c.sorti_in.p, sorted,
                                            static_cast<int>(nS), 0, nbits);
            c.cub_tmp.reserve(b);
            ++c.lib_calls;
            PBKV_CUDA(cub::DeviceRadixSort::SortPairs(c.cub_tmp.p, b, c.sortk_in.p, c.sortk_out.p, c.sorti_in.p,
                                                      sorted, static_cast<int>(nS), 0, nbits, c.stream));
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
        rank_kernel<<<grid_cap(nS, kThreads), kThreads, 0, c.stream>>>(sorted, c.C.p, ss, c.rank.p, c.cnt.p);
        PBKV_CUDA(cudaGetLastError());
        ++c.launches;
        std::size_t b = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, b, c.cnt.p, c.cnt.p, static_cast<int>(nS));
        c.cub_tmp.reserve(b);
        ++c.lib_calls;
        PBKV_CUDA(cub::DeviceScan::ExclusiveSum(c.cub_tmp.p, b, c.cnt.p, c.cnt.p, static_cast<int>(nS), c.stream));
        scatter_kernel<<<grid_cap(nS, kThreads), kThreads, 0, c.stream>>>(a);
        PBKV_CUDA(cudaGetLastError());
        cut_kernel<<<1, 1, 0, c.stream>>>(a);
        PBKV_CUDA(cudaGetLastError());
        c.launches += 2;
        PBKV_CUDA(cudaMemcpyAsync(hs, ss, sizeof(SelState), cudaMemcpyDeviceToHost, c.stream));
        if (c.report_deferred) {  // the persistent kernel stopped before its reports: all of them here
            const std::size_t nh = static_cast<std::size_t>(c.n_heavy);
            const std::size_t bytes = (nh + 1) * sizeof(HeavyReport);
            launch_heavy_report(c, reinterpret_cast<long long*>(res), reinterpret_cast<HeavyReport*>(c.hreport_h.p),
                                reinterpret_cast<double*>(c.hreport_h.p + bytes));
        }
        PBKV_CUDA(cudaStreamSynchronize(c.stream));
    }
    out.n_victims = static_cast<std::int64_t>(hs->n_victims);
    out.freed = static_cast<std::int64_t>(hs->freed);
    out.shortfall = hs->shortfall;
    return out;
}

}  // namespace pbkv
