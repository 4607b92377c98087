// Device helpers shared by the score / select / prefetch kernels.
#pragma once

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/warp/warp_reduce.cuh>
#include <math_constants.h>

#include "pbkv_internal.cuh"

namespace pbkv {
namespace dev {

__device__ __forceinline__ void set_error(DevStatus* st, int code, int kind, long long node) {
    atomicCAS(&st->code, 0, code);
    if (st->code == code) {
        atomicCAS(&st->kind, 0, kind);
        atomicMin(&st->node, node);
    }
}

// Forecast::mass_on (forecast.hpp:64-69): sum over set agent bits in
// ascending agent order.  The resident forecast table is agent-major,
// P[slot][agent][k] (the K steps of one agent are one 64-byte line at K = 8),
// so step k of agent a is base[a * stride] with base = &P[slot][0][k] and
// stride = K.  Loads are issued in batches of 8 so their latency overlaps;
// the additions stay in the reference order.  A masked-out agent is skipped
// (not "+0.0"), so the result is the exact reference chain.
__device__ __forceinline__ double mass_on(const double* __restrict__ base, int stride, unsigned long long bits) {
    double m = 0.0;
    while (bits) {
        double v[8];
        int cnt = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (bits) {
                int a = __ffsll(static_cast<long long>(bits)) - 1;
                v[j] = __ldg(base + static_cast<std::size_t>(a) * stride);
                bits &= bits - 1;
                cnt = j + 1;
            }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (j < cnt) m = __dadd_rn(m, v[j]);
    }
    return m;
}

// order-preserving double -> uint64 (policies.hpp:46 compares ranks with <)
__device__ __forceinline__ unsigned long long enc_rank(double r) {
    if (r == 0.0) r = 0.0;  // -0.0 == +0.0 under std::tie
    unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(r));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ Key2 make_key(int cls, double rank, unsigned long long last) {
    unsigned long long e = enc_rank(rank);
    Key2 k;
    k.w0 = (static_cast<unsigned long long>(cls) << 63) | (e >> 1);
    k.w1 = ((e & 1ull) << 63) | last;
    return k;
}

__device__ __forceinline__ bool key_less(const Key2& a, int ia, const Key2& b, int ib) {
    if (a.w0 != b.w0) return a.w0 < b.w0;
    if (a.w1 != b.w1) return a.w1 < b.w1;
    return ia < ib;
}

__device__ __forceinline__ Key2 load_key(const Key2* keys, int i) {
    const ulonglong2 v = __ldcg(reinterpret_cast<const ulonglong2*>(keys) + i);
    return Key2{v.x, v.y};
}

// 64-bit shared-memory add / or / and through native 32-bit atomics (the
// 64-bit shared atomics compile to CAS spin loops on sm_100a).  The add is
// exact: the carry out of the low word is added to the high word.
__device__ __forceinline__ void smem_add_u64(unsigned long long* p, unsigned long long v) {
    unsigned int* w = reinterpret_cast<unsigned int*>(p);
    const unsigned int lo = static_cast<unsigned int>(v), hi = static_cast<unsigned int>(v >> 32);
    const unsigned int old = lo ? atomicAdd(w, lo) : 0u;
    const unsigned int up = hi + (static_cast<unsigned int>(old + lo) < old ? 1u : 0u);
    if (up) atomicAdd(w + 1, up);
}
__device__ __forceinline__ void smem_or_u64(unsigned long long* p, unsigned long long v) {
    unsigned int* w = reinterpret_cast<unsigned int*>(p);
    if (static_cast<unsigned int>(v)) atomicOr(w, static_cast<unsigned int>(v));
    if (v >> 32) atomicOr(w + 1, static_cast<unsigned int>(v >> 32));
}
__device__ __forceinline__ void smem_and_u64(unsigned long long* p, unsigned long long v) {
    unsigned int* w = reinterpret_cast<unsigned int*>(p);
    if (~static_cast<unsigned int>(v)) atomicAnd(w, static_cast<unsigned int>(v));
    if (~static_cast<unsigned int>(v >> 32)) atomicAnd(w + 1, static_cast<unsigned int>(v >> 32));
}

// warp-aggregated append: one atomic per warp; returns this lane's slot
__device__ __forceinline__ long long warp_append(unsigned long long* counter, bool pred) {
    const unsigned mask = __ballot_sync(0xffffffffu, pred);
    if (!mask) return -1;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(mask) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(counter, static_cast<unsigned long long>(__popc(mask)));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (!pred) return -1;
    return static_cast<long long>(base + __popc(mask & ((1u << lane) - 1u)));
}

// KVFlow steps-to-execution (policies.hpp:121-139): +inf when no tagged agent
// recurs; sets *missing when a tagged workflow has no remaining sequence.
__device__ __forceinline__ double kvflow_distance(const uint2* __restrict__ rng,
                                                  const int* __restrict__ slot,
                                                  const unsigned long long* __restrict__ bits,
                                                  const int* __restrict__ rem_off, const int* __restrict__ rem_seq,
                                                  const std::uint8_t* __restrict__ rem_has, int n, bool* missing) {
    double best = CUDART_INF;
    const uint2 rg = rng[n];
    for (unsigned int e = rg.x; e < rg.y; ++e) {
        int s = slot[e];
        if (!rem_has[s]) {
            *missing = true;
            return best;
        }
        unsigned long long b = bits[e];
        for (int k = rem_off[s]; k < rem_off[s + 1]; ++k) {
            int a = rem_seq[k];
            if (a >= 0 && a < 64 && ((b >> a) & 1ull)) {
                double d = static_cast<double>(k - rem_off[s] + 1);
                best = d < best ? d : best;
                break;
            }
        }
    }
    return best;
}

}  // namespace dev

// ---- kernel argument packs -------------------------------------------------------
struct ScoreArgs {
    const uint2* acc_rng;  // [n] {begin, end} of the node's entries in the pool
    const int* acc_slot;
    const unsigned long long* acc_bits;
    const double* P;
    const double* Pg;  // gs-premultiplied rows (one-agent entries)
    const int2* lslot;         // light nodes' entries, node-indexed
    const ulonglong2* lbits;
    const double* gs;
    const std::uint8_t* fstate;
    int K, V1;
    unsigned long long amask;
    double* out;
    DevStatus* st;
};

// per-node stage-3 state initialised by whichever kernel scores/keys the node
struct KeyArgs {
    const int* parent;
    const int* len;
    const std::uint8_t* flags;
    const unsigned long long* last;
    const int* ever;
    const double* score_cached;
    const uint2* acc_rng;
    const int* acc_slot;
    const unsigned long long* acc_bits;
    const int* rem_off;
    const int* rem_seq;
    const std::uint8_t* rem_has;
    Key2* keys;
    int* eff;
    int* sublock;
    unsigned long long* W;
    unsigned int* C;
    int* rank;
    std::uint8_t* missing;
    DevStatus* st;
    int policy;
};

namespace dev {

// key of policies.hpp:88-153 for device node n (HE uses `score`), node
// fields already loaded by the caller
__device__ __forceinline__ void write_key_v(const KeyArgs& a, int n, double score, std::uint8_t f,
                                            unsigned long long last, int ever) {
    const bool retired = (f & kFlagRetired) != 0;
    if (last >> 63) set_error(a.st, PBKV_EINVAL, kErrLastAccessRange, n);
    Key2 k;
    if (f & kFlagOutOfOrder) {  // sharded spine node (shard.cu) / deferred heavy node
        reinterpret_cast<ulonglong2*>(a.keys)[n] = make_ulonglong2(0ull, 0ull);
        return;
    }
    switch (a.policy) {
        case PBKV_POLICY_LRU:
            k = make_key(0, 0.0, last);
            break;
        case PBKV_POLICY_LAE:
            k = retired ? make_key(0, static_cast<double>(ever), last) : make_key(1, 0.0, last);
            break;
        case PBKV_POLICY_HE:
            k = retired ? make_key(0, static_cast<double>(ever), last) : make_key(1, score, last);
            break;
        default: {  // KVFLOW
            bool miss = false;
            double d = retired ? CUDART_INF
                               : kvflow_distance(a.acc_rng, a.acc_slot, a.acc_bits, a.rem_off, a.rem_seq, a.rem_has,
                                                 n, &miss);
            if (miss) a.missing[n] = 2;
            k = isinf(d) ? make_key(0, 0.0, last) : make_key(1, -d, last);
        }
    }
    reinterpret_cast<ulonglong2*>(a.keys)[n] = make_ulonglong2(k.w0, k.w1);
}

__device__ __forceinline__ void write_key(const KeyArgs& a, int n, double score) {
    write_key_v(a, n, score, a.flags[n], a.last[n], a.ever[n]);
}

// per-node scratch init for the selection (every node, device or not); the
// per-head fields (W, C, rank) are written by the selection kernel itself
__device__ __forceinline__ void init_select_state(const KeyArgs& a, int n, bool missing) {
    a.eff[n] = n;
    a.sublock[n] = 0;
    a.missing[n] = missing ? 1 : 0;
}

}  // namespace dev
}  // namespace pbkv
