// Stage 4 on sm_100a: conservative / aggressive prefetch planning
// (policies.hpp:181-235) as ONE cooperative kernel with no library calls and
// one host synchronisation per plan:
//   1. candidates: host-tier nodes whose parent is on the device, with the
//      single-step value v (Eq. 1, scoring.hpp:41-45, summed in entry order)
//      > 0 (policies.hpp:190-197).  A missing forecast raises on the first
//      host node in host_index_ order, i.e. least (last_access, id)
//      (cache.hpp:97);
//   2. (v desc, id asc) order (policies.hpp:199-202): the sort key
//      (~enc(v), id) has its varying bits packed order-preservingly into 64
//      bits; a 12-bit MSD histogram places every candidate into its digit's
//      bucket, then every bucket is ranked in place -- one warp for <= 32
//      elements, else rank counting from shared-memory tiles, (bucket, 64-
//      element chunk) tasks spread over every CTA;
//   3. greedy fill with skip (policies.hpp:203-210), exact and mostly
//      parallel: while the running token total of the sorted candidates stays
//      within the budget every candidate is taken, so the sort phase, which
//      knows each candidate's token prefix (bucket prefix from the histogram
//      + the lengths of the smaller keys in its bucket, summed by the rank
//      count), selects that whole prefix at once and marks the first
//      candidate that overflows it; one warp then continues from there with
//      the small remaining budget, skipping 32-candidate chunks whose shortest
//      length exceeds it and taking runs that fit by a warp prefix sum;
//   4. the plan (sorted candidates, values, selection, counters) is stored
//      straight into pinned host memory by the kernel.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace pbkv {

using namespace dev;

ScoreArgs make_score_args(Context& c, double* out);

namespace {

constexpr int kPT = 512;              // threads per CTA (two CTAs per SM)
constexpr int kPBits = 12;            // MSD digit
constexpr int kPBins = 1 << kPBits;
constexpr int kPer = kPBins / kPT;    // bins per thread in the offset scan
constexpr int kTile = 4096;           // rank-counting tile (keys in shared memory)
constexpr int kChunk = kPT / 8;       // elements per rank task (8 threads each)

struct PfState {
    unsigned long long n_cand;
    unsigned long long or_hi, and_hi;
    unsigned int or_id, and_id;
    int min_len;
    unsigned int n_big;
    unsigned long long f;      // sorted position of the first candidate overflowing the budget
    long long tok_f;           // tokens of the candidates before it (all selected)
    long long tot_len;         // tokens of all candidates
    unsigned long long ts[8];  // %globaltimer after each phase (CTA 0; diagnostics)
};

__device__ __forceinline__ void pf_stamp(PfState* ps, int i) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        ps->ts[i] = t;
    }
}

struct PfArgs {
    ScoreArgs s;
    const int* parent;
    const std::uint8_t* flags;
    const unsigned long long* last;
    const int* len;
    long long n_nodes;
    long long budget;
    unsigned long long* c_hi;  // candidates in append order: ~enc(v), id, len
    unsigned int* c_id;
    unsigned int* c_len;
    unsigned long long* b_key;  // bucketed: sort key (packed, or ~enc(v)), ~enc(v), id, len
    unsigned long long* b_hi;
    unsigned int* b_id;
    unsigned int* b_len;
    int* s_id;  // sorted ids, lengths and keys
    int* s_len;
    unsigned long long* s_hi;
    int* chunk_min;  // shortest length of every 32 sorted candidates
    unsigned int* hist;     // [kPBins] counts
    unsigned long long* hist_len;  // [kPBins] token sums
    unsigned int* cursor;   // [kPBins]
    unsigned int* seg_off;  // [kPBins] first sorted position of every bucket
    unsigned long long* seg_lpre;  // [kPBins] tokens of the buckets before it
    unsigned int* big;      // (bucket, offset, count) of the buckets ranked by tiles
    PfState* ps;
    DevStatus* st;
    int* h_cand;  // pinned host outputs
    double* h_val;
    int* h_sel;
    long long* h_ctr;  // n_candidates, n_selected, selected_tokens, error flag
};

struct PfSmem {
    union {
        struct {
            unsigned int c[kPBins];
            unsigned long long l[kPBins];
        } hist;
        struct {
            unsigned long long k[kTile];
            unsigned int id[kTile];
            unsigned int len[kTile];
        } tile;
        typename cub::BlockScan<unsigned int, kPT>::TempStorage scan;
        typename cub::BlockScan<unsigned long long, kPT>::TempStorage scan64;
        int queue[kPT / 32][512];  // phase 1: host-tier nodes per warp
    } u;
    unsigned int off[kPBins];
    unsigned long long red[32];
    unsigned long long bc[4];
};

// Eq. 1 of a node, in access order (scoring.hpp:43-44): mass on step 0
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

// a host node whose Eq. 1 is computed by the reference (parent on the device)
__device__ __forceinline__ bool host_candidate(const PfArgs& a, int n) {
    return n != 0 && (a.flags[n] & kFlagTierMask) == PBKV_TIER_HOST &&
           (a.flags[a.parent[n]] & kFlagTierMask) == PBKV_TIER_DEVICE;
}

// order-preserving extraction of the bits of `w` under `mask` (a run of set
// mask bits at a time, high to low)
__device__ __forceinline__ unsigned long long pext_runs(unsigned long long w, unsigned long long mask) {
    unsigned long long r = 0;
    while (mask) {
        const int hi = 63 - __clzll(static_cast<long long>(mask));
        const unsigned long long above_cleared = ~mask & ((hi == 63) ? ~0ull : ((1ull << (hi + 1)) - 1ull));
        const int lo = above_cleared ? 64 - __clzll(static_cast<long long>(above_cleared)) : 0;
        const int n = hi - lo + 1;
        const unsigned long long run = (n == 64) ? ~0ull : ((1ull << n) - 1ull);
        r = (n == 64 ? 0ull : (r << n)) | ((w >> lo) & run);
        mask &= ~(run << lo);
    }
    return r;
}

// the candidates' varying key bits: (~enc(v)) bits under vhi, then id bits
// under vid; packed when they fit 64 bits (the usual case), else the rank
// counting compares (hi, id) and the digit comes from the hi bits alone
struct Packer {
    unsigned long long vhi;
    unsigned int vid;
    int nhi, nid, nbits;
    int dbits;  // digit width: ~8 candidates per bucket, 4..kPBits bits
    bool packed;
    __device__ void init(const PfState* ps, unsigned long long n) {
        vhi = __ldcg(&ps->or_hi) ^ __ldcg(&ps->and_hi);
        vid = __ldcg(&ps->or_id) ^ __ldcg(&ps->and_id);
        nhi = __popcll(vhi);
        nid = __popc(vid);
        nbits = nhi + nid;
        packed = nbits <= 64;
        dbits = 4;
        while (dbits < kPBits && (8ull << dbits) < n) ++dbits;
        if (!packed && dbits > nhi) dbits = nhi;
    }
    __device__ int bins() const { return 1 << dbits; }
    __device__ unsigned long long key(unsigned long long hi, unsigned int id) const {
        if (!packed) return hi;
        const unsigned long long ph = pext_runs(hi, vhi), pi = pext_runs(id, vid);
        return (nid == 64 ? 0ull : (ph << nid)) | pi;
    }
    __device__ unsigned int digit(unsigned long long key) const {
        if (packed) return static_cast<unsigned int>(nbits <= dbits ? key : key >> (nbits - dbits));
        const unsigned long long ph = pext_runs(key, vhi);
        return static_cast<unsigned int>(ph >> (nhi - dbits));
    }
};

__device__ __forceinline__ bool pf_less(bool packed, unsigned long long ka, unsigned int ia, unsigned long long kb,
                                        unsigned int ib) {
    if (packed) return ka < kb;  // distinct ids: packed keys are distinct
    return ka != kb ? ka < kb : ia < ib;
}

__device__ __forceinline__ double dec_value(unsigned long long hi) {
    const unsigned long long e = ~hi;  // enc(v) (common.cuh enc_rank)
    const unsigned long long b = (e >> 63) ? (e & 0x7fffffffffffffffull) : ~e;
    return __longlong_as_double(static_cast<long long>(b));
}

template <class T, class Op>
__device__ __forceinline__ T block_all(T v, Op op, unsigned long long* sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int o = 16; o; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if (lane == 0) sh[warp] = static_cast<unsigned long long>(v);
    __syncthreads();
    T r = static_cast<T>(sh[0]);
    for (int w = 1; w < kPT / 32; ++w) r = op(r, static_cast<T>(sh[w]));
    __syncthreads();
    return r;
}

// ---- phase 1: candidates ------------------------------------------------------------
// Every thread reads the tier bytes of 16 consecutive nodes in one 16-byte
// load; the host-tier ones (a few percent) are queued per warp in shared
// memory and then evaluated 32 at a time, one per lane (parent tier, Eq. 1):
// the scan costs one coalesced load per 16 nodes, the per-candidate chains of
// dependent loads run on full warps.
__device__ __forceinline__ void pf_eval(const PfArgs& a, int n, bool valid, unsigned long long& or_hi,
                                        unsigned long long& and_hi, unsigned int& or_id, unsigned int& and_id,
                                        int& min_len) {
    bool take = false;
    double v = 0.0;
    if (valid) {
        const int p = a.parent[n];
        const uint2 rg = a.s.acc_rng[n];
        if ((a.flags[p] & kFlagTierMask) == PBKV_TIER_DEVICE) {
            bool miss = false;
            v = eq1(a.s, rg.x, rg.y, &miss);
            if (miss) {
                atomicCAS(&a.st->code, 0, PBKV_EINVAL);
                atomicCAS(&a.st->kind, 0, kErrMissingForecast);
                atomicMin(reinterpret_cast<unsigned long long*>(&a.st->aux), a.last[n]);
            } else {
                take = v > 0.0;  // policies.hpp:196
            }
        }
    }
    const long long slot = warp_append(&a.ps->n_cand, take);
    if (take) {
        const unsigned long long hi = ~enc_rank(v);
        const int ln = a.len[n];
        a.c_hi[slot] = hi;
        a.c_id[slot] = static_cast<unsigned int>(n);
        a.c_len[slot] = static_cast<unsigned int>(ln);
        or_hi |= hi;
        and_hi &= hi;
        or_id |= static_cast<unsigned int>(n);
        and_id &= static_cast<unsigned int>(n);
        min_len = min(min_len, ln);
    }
}

__device__ __forceinline__ void pf_candidates(const PfArgs& a, PfSmem& sm) {
    const long long tid = blockIdx.x * static_cast<long long>(kPT) + threadIdx.x;
    const long long nthr = static_cast<long long>(gridDim.x) * kPT;
    for (long long j = tid; j < kPBins; j += nthr) {
        a.hist[j] = 0;
        a.hist_len[j] = 0;
        a.cursor[j] = 0;
    }
    for (long long j = tid; j <= (a.n_nodes >> 5); j += nthr) a.chunk_min[j] = INT_MAX;
    unsigned long long or_hi = 0, and_hi = ~0ull;
    unsigned int or_id = 0, and_id = ~0u;
    int min_len = INT_MAX;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int* q = sm.u.queue[warp];
    for (long long base = blockIdx.x * static_cast<long long>(kPT) * 16; base < a.n_nodes; base += nthr * 16) {
        const long long i0 = base + threadIdx.x * 16ll;
        unsigned int hm = 0;  // host-tier bytes of this thread's 16 nodes
        if (i0 + 16 <= a.n_nodes) {
            const uint4 f = __ldg(reinterpret_cast<const uint4*>(a.flags + i0));
            const unsigned int w[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
            for (int b = 0; b < 16; ++b)
                hm |= (((w[b >> 2] >> (8 * (b & 3))) & kFlagTierMask) == PBKV_TIER_HOST ? 1u : 0u) << b;
        } else {
            for (int b = 0; b < 16; ++b)
                if (i0 + b < a.n_nodes && (a.flags[i0 + b] & kFlagTierMask) == PBKV_TIER_HOST) hm |= 1u << b;
        }
        if (i0 == 0) hm &= ~1u;  // the root is never a candidate
        // warp-wide queue of the host nodes (<= 512)
        const unsigned int cnt = __popc(hm);
        unsigned int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const unsigned int total = __shfl_sync(0xffffffffu, incl, 31);
        unsigned int at = incl - cnt;
        while (hm) {
            const int b = __ffs(hm) - 1;
            hm &= hm - 1;
            q[at++] = static_cast<int>(i0 + b);
        }
        __syncwarp();
        for (unsigned int k = 0; k < total; k += 32) {
            const bool valid = k + lane < total;
            pf_eval(a, valid ? q[k + lane] : 0, valid, or_hi, and_hi, or_id, and_id, min_len);
        }
        __syncwarp();
    }
    struct Or {
        __device__ unsigned long long operator()(unsigned long long x, unsigned long long y) const { return x | y; }
    };
    struct And {
        __device__ unsigned long long operator()(unsigned long long x, unsigned long long y) const { return x & y; }
    };
    struct Min {
        __device__ long long operator()(long long x, long long y) const { return x < y ? x : y; }
    };
    const unsigned long long bo = block_all<unsigned long long>(or_hi, Or(), sm.red);
    const unsigned long long ba = block_all<unsigned long long>(and_hi, And(), sm.red);
    const unsigned long long bio = block_all<unsigned long long>(or_id, Or(), sm.red);
    const unsigned long long bia = block_all<unsigned long long>(0xffffffff00000000ull | and_id, And(), sm.red);
    const long long bm = block_all<long long>(min_len, Min(), sm.red);
    if (threadIdx.x == 0) {
        if (bo) atomicOr(&a.ps->or_hi, bo);
        if (~ba) atomicAnd(&a.ps->and_hi, ba);
        if (bio) atomicOr(&a.ps->or_id, static_cast<unsigned int>(bio));
        if (static_cast<unsigned int>(bia) != ~0u) atomicAnd(&a.ps->and_id, static_cast<unsigned int>(bia));
        if (bm != INT_MAX) atomicMin(&a.ps->min_len, static_cast<int>(bm));
    }
}

// error path: among the host nodes with the least last_access that miss a
// forecast, the smallest id (the first raise of policies.hpp:190-195)
__device__ __forceinline__ void pf_error_id(const PfArgs& a) {
    const unsigned long long lmin = static_cast<unsigned long long>(__ldcg(&a.st->aux));
    const long long nthr = static_cast<long long>(gridDim.x) * kPT;
    for (long long i = blockIdx.x * static_cast<long long>(kPT) + threadIdx.x; i < a.n_nodes; i += nthr) {
        const int n = static_cast<int>(i);
        if (!host_candidate(a, n) || a.last[n] != lmin) continue;
        const uint2 rg = a.s.acc_rng[n];
        bool miss = false;
        eq1(a.s, rg.x, rg.y, &miss);
        if (miss) atomicMin(&a.st->node, static_cast<long long>(n));
    }
}

// ---- phase 2: digit histogram (counts and token sums) ----------------------------------
__device__ __forceinline__ void pf_hist(const PfArgs& a, const Packer& pk, unsigned long long n, PfSmem& sm) {
    for (int b = threadIdx.x; b < kPBins; b += kPT) {
        sm.u.hist.c[b] = 0;
        sm.u.hist.l[b] = 0;
    }
    __syncthreads();
    const unsigned long long nthr = static_cast<unsigned long long>(gridDim.x) * kPT;
    for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(kPT) + threadIdx.x; i < n; i += nthr) {
        const unsigned int d = pk.digit(pk.key(__ldcg(&a.c_hi[i]), __ldcg(&a.c_id[i])));
        atomicAdd(&sm.u.hist.c[d], 1u);
        smem_add_u64(&sm.u.hist.l[d], static_cast<unsigned long long>(__ldcg(&a.c_len[i])));
    }
    __syncthreads();
    for (int b = threadIdx.x; b < kPBins; b += kPT) {
        const unsigned int c = sm.u.hist.c[b];
        if (c) {
            atomicAdd(&a.hist[b], c);
            atomicAdd(&a.hist_len[b], sm.u.hist.l[b]);
        }
    }
}

// ---- phase 3: bucket offsets, scatter -------------------------------------------------
__device__ __forceinline__ void pf_scatter(const PfArgs& a, const Packer& pk, unsigned long long n, PfSmem& sm) {
    unsigned int v[kPer], s = 0;
    unsigned long long vl[kPer], sl = 0;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        v[j] = __ldcg(&a.hist[threadIdx.x * kPer + j]);
        vl[j] = __ldcg(&a.hist_len[threadIdx.x * kPer + j]);
        s += v[j];
        sl += vl[j];
    }
    unsigned int ex;
    cub::BlockScan<unsigned int, kPT>(sm.u.scan).ExclusiveSum(s, ex);
    unsigned long long exl = 0;
    if (blockIdx.x == 0) {
        __syncthreads();
        unsigned long long tl;
        cub::BlockScan<unsigned long long, kPT>(sm.u.scan64).ExclusiveSum(sl, exl, tl);
        if (threadIdx.x == 0) a.ps->tot_len = static_cast<long long>(tl);
    }
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        const int d = threadIdx.x * kPer + j;
        sm.off[d] = ex;
        if (blockIdx.x == 0) {
            a.seg_off[d] = ex;
            a.seg_lpre[d] = exl;
            if (v[j] > 32u) {
                const unsigned int q = atomicAdd(&a.ps->n_big, 1u);
                a.big[3 * q] = static_cast<unsigned int>(d);
                a.big[3 * q + 1] = ex;
                a.big[3 * q + 2] = v[j];
            }
        }
        ex += v[j];
        exl += vl[j];
    }
    __syncthreads();
    const unsigned long long nthr = static_cast<unsigned long long>(gridDim.x) * kPT;
    for (unsigned long long base = blockIdx.x * static_cast<unsigned long long>(kPT); base < n; base += nthr) {
        const unsigned long long i = base + threadIdx.x;
        const bool in = i < n;
        unsigned long long hi = 0, key = 0;
        unsigned int id = 0, ln = 0;
        int d = -1;
        if (in) {
            hi = __ldcg(&a.c_hi[i]);
            id = __ldcg(&a.c_id[i]);
            ln = __ldcg(&a.c_len[i]);
            key = pk.key(hi, id);
            d = static_cast<int>(pk.digit(key));
        }
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        if (in) {
            const int lane = threadIdx.x & 31, leader = __ffs(peers) - 1;
            unsigned int b = 0;
            if (lane == leader) b = atomicAdd(&a.cursor[d], static_cast<unsigned int>(__popc(peers)));
            b = __shfl_sync(peers, b, leader);
            const unsigned int pos = sm.off[d] + b + __popc(peers & ((1u << lane) - 1u));
            a.b_key[pos] = key;
            a.b_hi[pos] = hi;
            a.b_id[pos] = id;
            a.b_len[pos] = ln;
        }
    }
}

// a ranked candidate: its sorted position and the tokens of the candidates
// before it.  The plan arrays are written here; a candidate whose running
// total fits the budget is selected (no candidate before it was skipped), the
// first one past it is recorded for the greedy tail.
__device__ __forceinline__ void pf_place(const PfArgs& a, unsigned int pos, unsigned int id, unsigned long long hi,
                                         unsigned int ln, unsigned long long before) {
    a.s_id[pos] = static_cast<int>(id);
    a.s_len[pos] = static_cast<int>(ln);
    a.s_hi[pos] = hi;
    atomicMin(&a.chunk_min[pos >> 5], static_cast<int>(ln));
    const long long b = static_cast<long long>(before), e = b + static_cast<long long>(ln);
    if (e > a.budget && b <= a.budget) {
        a.ps->f = pos;
        a.ps->tok_f = b;
    }
}

// ---- phase 4: rank every bucket -------------------------------------------------------
__device__ __forceinline__ void pf_sort(const PfArgs& a, const Packer& pk, PfSmem& sm) {
    // buckets of 1..32: one warp each (rank and token prefix by shuffles)
    const int lane = threadIdx.x & 31;
    const int gwarp = static_cast<int>((blockIdx.x * static_cast<unsigned int>(kPT) + threadIdx.x) >> 5);
    const int nwarps = static_cast<int>((gridDim.x * static_cast<unsigned int>(kPT)) >> 5);
    for (int d = gwarp; d < pk.bins(); d += nwarps) {
        const unsigned int cnt = __ldcg(&a.hist[d]);
        if (cnt == 0u || cnt > 32u) continue;
        const unsigned int off = __ldcg(&a.seg_off[d]);
        const unsigned long long lpre = __ldcg(&a.seg_lpre[d]);
        const bool in = static_cast<unsigned int>(lane) < cnt;
        const unsigned long long k = in ? __ldcg(&a.b_key[off + lane]) : 0ull;
        const unsigned int id = in ? __ldcg(&a.b_id[off + lane]) : 0u;
        const unsigned int ln = in ? __ldcg(&a.b_len[off + lane]) : 0u;
        unsigned int r = 0;
        unsigned long long before = 0;
        for (unsigned int j = 0; j < cnt; ++j) {
            const unsigned long long kj = __shfl_sync(0xffffffffu, k, j);
            const unsigned int ij = __shfl_sync(0xffffffffu, id, j);
            const unsigned int lj = __shfl_sync(0xffffffffu, ln, j);
            if (pf_less(pk.packed, kj, ij, k, id)) {
                ++r;
                before += lj;
            }
        }
        if (in) pf_place(a, off + r, id, __ldcg(&a.b_hi[off + lane]), ln, lpre + before);
    }
    // larger buckets: rank = number of smaller keys, token prefix = their
    // lengths, counted from shared-memory tiles by 8 threads per element.
    // Tasks are (bucket, 64-element chunk); the first task of every bucket
    // comes from a block scan of the chunk counts (sm.off, free after the
    // scatter), task t -> CTA t % grid.
    if (threadIdx.x == 0) sm.bc[0] = __ldcg(&a.ps->n_big);
    __syncthreads();
    const unsigned int n_big = static_cast<unsigned int>(sm.bc[0]);
    if (n_big == 0) return;
    {
        unsigned int v[kPer], s = 0;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            const unsigned int b = threadIdx.x * kPer + j;
            v[j] = b < n_big ? (__ldcg(&a.big[3 * b + 2]) + kChunk - 1) / kChunk : 0u;
            s += v[j];
        }
        unsigned int ex, tot;
        __syncthreads();
        cub::BlockScan<unsigned int, kPT>(sm.u.scan).ExclusiveSum(s, ex, tot);
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            sm.off[threadIdx.x * kPer + j] = ex;
            ex += v[j];
        }
        if (threadIdx.x == 0) sm.bc[1] = tot;
        __syncthreads();
    }
    const unsigned int n_task = static_cast<unsigned int>(sm.bc[1]);
    unsigned int held = ~0u;  // bucket whose first tile is in shared memory
    for (unsigned int t = blockIdx.x; t < n_task; t += gridDim.x) {
        unsigned int lo = 0, hi = n_big - 1;  // last bucket with off[b] <= t
        while (lo < hi) {
            const unsigned int mid = (lo + hi + 1) >> 1;
            if (sm.off[mid] <= t) lo = mid;
            else hi = mid - 1;
        }
        const unsigned int b = lo, c = t - sm.off[b];
        const unsigned int dg = __ldcg(&a.big[3 * b]), off = __ldcg(&a.big[3 * b + 1]), cnt = __ldcg(&a.big[3 * b + 2]);
        const unsigned int e = c * kChunk + threadIdx.x / 8, part = threadIdx.x % 8;
        const bool in = e < cnt;
        const unsigned long long mk = in ? __ldcg(&a.b_key[off + e]) : 0ull;
        const unsigned int mi = in ? __ldcg(&a.b_id[off + e]) : 0u;
        unsigned int r = 0;
        unsigned long long before = 0;
        for (unsigned int t0 = 0; t0 < cnt; t0 += kTile) {
            const unsigned int tn = min(static_cast<unsigned int>(kTile), cnt - t0);
            if (!(t0 == 0 && held == b)) {
                __syncthreads();
                for (unsigned int q = threadIdx.x; q < tn; q += kPT) {
                    sm.u.tile.k[q] = __ldcg(&a.b_key[off + t0 + q]);
                    sm.u.tile.id[q] = __ldcg(&a.b_id[off + t0 + q]);
                    sm.u.tile.len[q] = __ldcg(&a.b_len[off + t0 + q]);
                }
                __syncthreads();
                held = t0 == 0 ? b : ~0u;
            }
            if (in) {
                if (pk.packed) {
#pragma unroll 4
                    for (unsigned int q = part; q < tn; q += 8) {
                        const bool lt = sm.u.tile.k[q] < mk;
                        r += lt ? 1u : 0u;
                        before += lt ? sm.u.tile.len[q] : 0u;
                    }
                } else {
                    for (unsigned int q = part; q < tn; q += 8) {
                        const bool lt = pf_less(false, sm.u.tile.k[q], sm.u.tile.id[q], mk, mi);
                        r += lt ? 1u : 0u;
                        before += lt ? sm.u.tile.len[q] : 0u;
                    }
                }
            }
        }
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            r += __shfl_xor_sync(0xffffffffu, r, o);
            before += __shfl_xor_sync(0xffffffffu, before, o);
        }
        if (in && part == 0)
            pf_place(a, off + r, mi, __ldcg(&a.b_hi[off + e]), __ldcg(&a.b_len[off + e]),
                     __ldcg(&a.seg_lpre[dg]) + before);
    }
}

// ---- phase 5: the greedy tail (one warp) ------------------------------------------------
// From the first candidate past the all-fitting prefix (skipped: it
// overflows), with the remaining budget: chunks of 32 sorted candidates whose
// shortest length exceeds the budget are skipped 32 chunks per step; inside a
// chunk a prefix sum takes every lane that still fits, the first that does
// not is skipped (policies.hpp:203-210).
__device__ __forceinline__ void pf_greedy_tail(const PfArgs& a, unsigned long long n) {
    const int lane = threadIdx.x & 31;
    const unsigned long long f = __ldcg(&a.ps->f);
    long long nsel, tok;
    if (f < n) {
        nsel = static_cast<long long>(f);
        tok = __ldcg(&a.ps->tok_f);
    } else if (a.budget >= 0) {  // every candidate fits
        nsel = static_cast<long long>(n);
        tok = __ldcg(&a.ps->tot_len);
    } else {
        nsel = 0;
        tok = 0;
    }
    long long rem = a.budget - tok;
    const long long min_len = __ldcg(&a.ps->min_len);
    unsigned long long c = f < n ? (f + 1) >> 5 : (n + 31) >> 5;
    unsigned int first = f < n ? static_cast<unsigned int>((f + 1) & 31u) : 0u;
    const unsigned long long n_chunks = (n + 31) >> 5;
    while (c < n_chunks && rem >= min_len) {
        // the next chunk that can hold a candidate of length <= rem
        const unsigned long long cc = c + lane;
        const int cm = cc < n_chunks ? __ldcg(&a.chunk_min[cc]) : 0;
        const unsigned m = __ballot_sync(0xffffffffu, cc >= n_chunks || cm <= rem);
        if (!m) {
            c += 32;
            first = 0;
            continue;
        }
        const int s = __ffs(m) - 1;
        if (s) first = 0;
        c += s;
        if (c >= n_chunks) break;
        const unsigned long long i = c * 32 + lane;
        const bool in = i < n && static_cast<unsigned int>(lane) >= first;
        const int id = in ? __ldcg(&a.s_id[i]) : 0;
        const long long l = in ? __ldcg(&a.s_len[i]) : 0;
        unsigned todo = __ballot_sync(0xffffffffu, in);
        while (todo) {
            // a lane longer than the remaining budget is skipped for good
            todo &= __ballot_sync(0xffffffffu, l <= rem);
            if (!todo) break;
            const bool mine = (todo >> lane) & 1u;
            long long x = mine ? l : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            // every lane whose running total still fits is taken (a prefix of todo)
            const bool fit = mine && x <= rem;
            const unsigned fm = __ballot_sync(0xffffffffu, fit);
            if (fit) a.h_sel[nsel + __popc(fm & ((1u << lane) - 1u))] = id;
            const long long used = fm ? __shfl_sync(0xffffffffu, x, 31 - __clz(fm)) : 0;
            rem -= used;
            tok += used;
            nsel += __popc(fm);
            todo &= ~fm;
            if (todo) todo &= todo - 1u;  // the first lane past them does not fit: skipped
        }
        ++c;
        first = 0;
    }
    if (lane == 0) {
        a.h_ctr[0] = static_cast<long long>(n);
        a.h_ctr[1] = nsel;
        a.h_ctr[2] = tok;
    }
}

__global__ void __launch_bounds__(kPT, 2) prefetch_plan_kernel(PfArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PfSmem& sm = *reinterpret_cast<PfSmem*>(smem_raw);
    cg::grid_group grid = cg::this_grid();
    pf_stamp(a.ps, 0);
    pf_candidates(a, sm);
    grid.sync();
    pf_stamp(a.ps, 1);
    if (threadIdx.x == 0) {
        sm.bc[0] = static_cast<unsigned long long>(__ldcg(&a.st->code));
        sm.bc[1] = __ldcg(&a.ps->n_cand);
    }
    __syncthreads();
    const bool err = sm.bc[0] != 0;
    const unsigned long long n = sm.bc[1];
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) a.h_ctr[3] = err ? 1 : 0;
    if (err) {
        pf_error_id(a);
        return;
    }
    if (n == 0) {
        if (blockIdx.x == 0 && threadIdx.x == 0) a.h_ctr[0] = a.h_ctr[1] = a.h_ctr[2] = 0;
        return;
    }
    Packer pk;
    pk.init(a.ps, n);
    pf_hist(a, pk, n, sm);
    grid.sync();
    pf_stamp(a.ps, 2);
    pf_scatter(a, pk, n, sm);
    grid.sync();
    pf_stamp(a.ps, 3);
    pf_sort(a, pk, sm);
    grid.sync();
    pf_stamp(a.ps, 4);
    if (blockIdx.x == 0 && threadIdx.x < 32) {
        pf_greedy_tail(a, n);
        pf_stamp(a.ps, 5);
        return;
    }
    // the sorted plan into pinned host memory with 16-byte stores: ids,
    // values, and the all-fitting prefix of the selection (= the first f ids)
    const long long t = blockIdx.x * static_cast<long long>(kPT) + threadIdx.x - 32;
    const long long nt = static_cast<long long>(gridDim.x) * kPT - 32;
    const long long nn = static_cast<long long>(n);
    const unsigned long long f = __ldcg(&a.ps->f);
    const long long nf = f < n ? static_cast<long long>(f) : (a.budget >= 0 ? nn : 0);
    for (long long i = t; i < (nn >> 2); i += nt) {
        const int4 v = __ldcg(reinterpret_cast<const int4*>(a.s_id) + i);
        reinterpret_cast<int4*>(a.h_cand)[i] = v;
    }
    for (long long i = t; i < (nn >> 1); i += nt) {
        const ulonglong2 h = __ldcg(reinterpret_cast<const ulonglong2*>(a.s_hi) + i);
        reinterpret_cast<double2*>(a.h_val)[i] = make_double2(dec_value(h.x), dec_value(h.y));
    }
    for (long long i = t; i < (nf >> 2); i += nt) {
        const int4 v = __ldcg(reinterpret_cast<const int4*>(a.s_id) + i);
        reinterpret_cast<int4*>(a.h_sel)[i] = v;
    }
    if (t < 4) {  // the ragged ends
        const long long ic = (nn & ~3ll) + t, iv = (nn & ~1ll) + t, is = (nf & ~3ll) + t;
        if (ic < nn) a.h_cand[ic] = __ldcg(&a.s_id[ic]);
        if (t < 2 && iv < nn) a.h_val[iv] = dec_value(__ldcg(&a.s_hi[iv]));
        if (is < nf) a.h_sel[is] = __ldcg(&a.s_id[is]);
    }
    __syncthreads();
    if (threadIdx.x == 32) {  // (diagnostics: the store phase's end, latest CTA)
        unsigned long long tnow;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
        atomicMax(&a.ps->ts[6], tnow);
    }
}

int plan_grid(Context& c, std::int64_t n_nodes) {
    static int per_sm = 0, sms = 0;
    if (!per_sm) {
        PBKV_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device));
        PBKV_CUDA(cudaFuncSetAttribute(prefetch_plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(sizeof(PfSmem))));
        PBKV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, prefetch_plan_kernel, kPT,
                                                                sizeof(PfSmem)));
        if (per_sm < 1) throw ApiError(PBKV_ECUDA, "prefetch plan kernel cannot be resident");
        per_sm = per_sm >= 2 ? 2 : 1;
    }
    // small trees: fewer CTAs (cheaper grid barriers); one node per thread
    // and pass up to the full co-resident grid
    const std::int64_t want = (n_nodes + 4LL * kPT - 1) / (4LL * kPT);
    const std::int64_t cap = static_cast<std::int64_t>(sms) * per_sm;
    return static_cast<int>(std::max<std::int64_t>(8, std::min(want, cap)));
}

}  // namespace

// One plan: status + state reset, the cooperative kernel, one synchronisation.
// The plan lands in pinned host memory: c.hplan = [ctr 3 x i64 | cand ids
// (cap) | values (cap) | selected (cap)].
void run_prefetch_plan(Context& c, long long budget, PrefetchOut* out) {
    const std::size_t n = static_cast<std::size_t>(c.n) + 1;
    c.pf_hi.reserve(n);
    c.pf_id.reserve(n);
    c.pf_len.reserve(n);
    c.pf_bkey.reserve(n);
    c.pf_bhi.reserve(n);
    c.pf_bid.reserve(n);
    c.pf_blen.reserve(n);
    c.pf_sid.reserve(n);
    c.pf_slen.reserve(n);
    c.pf_shi.reserve(n);
    c.pf_cmin.reserve((n >> 5) + 2);
    c.pf_hist.reserve(3 * kPBins);
    c.pf_hlen.reserve(2 * kPBins);
    c.pf_big.reserve(3 * kPBins);
    c.pf_state.reserve(sizeof(PfState));
    const std::size_t b_ctr = 4 * sizeof(long long), b_ids = ((n * 4 + 15) & ~std::size_t(15));
    const std::size_t b_val = n * 8;
    c.hplan.reserve(b_ctr + 2 * b_ids + b_val);
    unsigned char* hp = c.hplan.p;
    PfArgs a;
    a.s = make_score_args(c, nullptr);
    a.parent = c.parent.p;
    a.flags = c.flags.p;
    a.last = c.last.p;
    a.len = c.len.p;
    a.n_nodes = c.n;
    a.budget = budget;
    a.c_hi = c.pf_hi.p;
    a.c_id = c.pf_id.p;
    a.c_len = c.pf_len.p;
    a.b_key = c.pf_bkey.p;
    a.b_hi = c.pf_bhi.p;
    a.b_id = c.pf_bid.p;
    a.b_len = c.pf_blen.p;
    a.s_id = c.pf_sid.p;
    a.s_len = c.pf_slen.p;
    a.s_hi = c.pf_shi.p;
    a.chunk_min = c.pf_cmin.p;
    a.hist = c.pf_hist.p;
    a.cursor = c.pf_hist.p + kPBins;
    a.seg_off = c.pf_hist.p + 2 * kPBins;
    a.hist_len = c.pf_hlen.p;
    a.seg_lpre = c.pf_hlen.p + kPBins;
    a.big = c.pf_big.p;
    a.ps = reinterpret_cast<PfState*>(c.pf_state.p);
    a.st = c.status.p;
    a.h_ctr = reinterpret_cast<long long*>(hp);
    a.h_cand = reinterpret_cast<int*>(hp + b_ctr);
    a.h_sel = reinterpret_cast<int*>(hp + b_ctr + b_ids);
    a.h_val = reinterpret_cast<double*>(hp + b_ctr + 2 * b_ids);
    // initial state from the pinned template (and_* all ones, min_len max)
    PfState* init = reinterpret_cast<PfState*>(c.hplan_init.p);
    if (!init) {
        c.hplan_init.reserve(sizeof(PfState));
        init = reinterpret_cast<PfState*>(c.hplan_init.p);
        *init = PfState{0, 0, ~0ull, 0u, ~0u, INT_MAX, 0u, ~0ull, 0, 0, {}};
    }
    PBKV_CUDA(cudaMemcpyAsync(a.ps, init, sizeof(PfState), cudaMemcpyHostToDevice, c.stream));
    void* args[] = {&a};
    if (c.timing) {  // kernel_ms[1] (pbkv_ctx_kernel_timings): the plan kernel alone
        PBKV_CUDA(cudaEventRecord(c.kev[2], c.stream));
        c.kev_select = true;
    }
    PBKV_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(prefetch_plan_kernel), dim3(plan_grid(c, c.n)),
                                          dim3(kPT), args, sizeof(PfSmem), c.stream));
    if (c.timing) PBKV_CUDA(cudaEventRecord(c.kev[3], c.stream));
    ++c.launches;
    PBKV_CUDA(cudaStreamSynchronize(c.stream));
    if (a.h_ctr[3]) check_status(c);  // the error path: the full status word
    else c.status_pending = false;    // the kernel read a clear status word
    if (std::getenv("PBKV_DEBUG_PLAN")) {
        PfState h{};
        PBKV_CUDA(cudaMemcpy(&h, a.ps, sizeof h, cudaMemcpyDeviceToHost));
        std::fprintf(stderr, "[pbkv plan] grid=%d n_cand=%llu n_big=%u f=%llu min_len=%d us: cand %.1f hist %.1f "
                     "scatter %.1f sort %.1f tail %.1f store %.1f\n", plan_grid(c, c.n), h.n_cand, h.n_big, h.f, h.min_len,
                     (h.ts[1] - h.ts[0]) * 1e-3, (h.ts[2] - h.ts[1]) * 1e-3, (h.ts[3] - h.ts[2]) * 1e-3,
                     (h.ts[4] - h.ts[3]) * 1e-3, (h.ts[5] - h.ts[4]) * 1e-3,
                     h.ts[6] > h.ts[4] ? (h.ts[6] - h.ts[4]) * 1e-3 : 0.0);
    }
    out->ctr = a.h_ctr;
    out->cand = a.h_cand;
    out->val = a.h_val;
    out->sel = a.h_sel;
}

}  // namespace pbkv
