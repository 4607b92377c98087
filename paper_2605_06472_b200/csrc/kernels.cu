// sm_100a kernels of the PBKV hot path: Eq. 2 / Eq. 1 scoring (stage 2),
// candidate keys + subtree-max reduction + token weights (stage 3), prefetch
// candidate filter + greedy-with-skip fill (stage 4).  See DESIGN.md §3 for
// the data layout, the closed form of the victim order and the roofline of
// each kernel.
//
// Floating point: every Eq. 1 / Eq. 2 operation is an explicit round-to-
// nearest __dmul_rn/__dadd_rn in the reference's evaluation order
// (scoring.hpp:49-62, forecast.hpp:64-69), so nvcc cannot contract into FMA
// and results are bit-identical to the CPU reference.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <cuda/std/tuple>
#include <math_constants.h>

#include "pbkv_internal.cuh"

namespace pbkv {

namespace {

__device__ __forceinline__ void set_error(DevStatus* st, int code, int kind, long long node) {
    atomicCAS(&st->code, 0, code);
    if (st->code == code) {
        atomicCAS(&st->kind, 0, kind);
        atomicMin(&st->node, node);
    }
}

// Forecast::mass_on (forecast.hpp:64-69): agents in ascending order.
__device__ __forceinline__ double mass_on(const double* __restrict__ row, unsigned long long bits) {
    double m = 0.0;
    while (bits) {
        int a = __ffsll(static_cast<long long>(bits)) - 1;
        m = __dadd_rn(m, __ldg(row + a));
        bits &= bits - 1;
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

// KVFlow steps-to-execution (policies.hpp:121-139): returns +inf or distance,
// or -1 when a tagged workflow has no remaining sequence.
__device__ double kvflow_distance(const unsigned int* __restrict__ off, const int* __restrict__ slot,
                                  const unsigned long long* __restrict__ bits, const int* __restrict__ rem_off,
                                  const int* __restrict__ rem_seq, const std::uint8_t* __restrict__ rem_has, int n,
                                  bool* missing) {
    double best = CUDART_INF;
    for (unsigned int e = off[n]; e < off[n + 1]; ++e) {
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

struct KeyArgs {
    const int* parent;
    const int* len;
    const std::uint8_t* flags;
    const unsigned long long* last;
    const int* ever;
    const double* score_cached;
    const unsigned int* acc_off;
    const int* acc_slot;
    const unsigned long long* acc_bits;
    const int* rem_off;
    const int* rem_seq;
    const std::uint8_t* rem_has;
    Key2* keys;
    int* eff;
    int* sublock;
    unsigned long long* W;
    std::uint8_t* missing;
    DevStatus* st;
    int policy;
};

// key of policies.hpp:88-153 for device node n with HE score `score`
__device__ __forceinline__ void write_key(const KeyArgs& a, int n, double score) {
    std::uint8_t f = a.flags[n];
    bool retired = (f & kFlagRetired) != 0;
    unsigned long long last = a.last[n];
    if (last >> 63) set_error(a.st, PBKV_EINVAL, kErrLastAccessRange, n);
    Key2 k;
    switch (a.policy) {
        case PBKV_POLICY_LRU:
            k = make_key(0, 0.0, last);
            break;
        case PBKV_POLICY_LAE:
            k = retired ? make_key(0, static_cast<double>(a.ever[n]), last) : make_key(1, 0.0, last);
            break;
        case PBKV_POLICY_HE:
            k = retired ? make_key(0, static_cast<double>(a.ever[n]), last) : make_key(1, score, last);
            break;
        default: {  // KVFLOW
            bool miss = false;
            double d = retired ? CUDART_INF
                               : kvflow_distance(a.acc_off, a.acc_slot, a.acc_bits, a.rem_off, a.rem_seq, a.rem_has,
                                                 n, &miss);
            if (miss) a.missing[n] = 2;
            k = isinf(d) ? make_key(0, 0.0, last) : make_key(1, -d, last);
        }
    }
    a.keys[n] = k;
}

// ---------------------------------------------------------------------------
// Stage 2, light nodes: one thread per node, the Eq. 2 chain in registers.
// Nodes with > kHeavyEntries entries are left to heavy_score_kernel.
struct ScoreArgs {
    const unsigned int* acc_off;
    const int* acc_slot;
    const unsigned long long* acc_bits;
    const double* P;
    const double* gs;
    const std::uint8_t* fstate;
    int K, V1;
    unsigned long long amask;
    double* out;
    DevStatus* st;
};

__device__ __forceinline__ double eq2_node(const ScoreArgs& s, unsigned int e0, unsigned int e1, bool* miss,
                                           bool* shorth) {
    double total = 0.0;
    const int K = s.K, V1 = s.V1;
    for (unsigned int e = e0; e < e1; ++e) {
        int slot = __ldg(s.acc_slot + e);
        unsigned long long b = __ldg(s.acc_bits + e) & s.amask;
        std::uint8_t fs = __ldg(s.fstate + slot);
        if (fs != 1) {
            if (fs == 2)
                *shorth = true;
            else
                *miss = true;
            continue;
        }
        const double* pw = s.P + static_cast<std::size_t>(slot) * K * V1;
        const double* g = s.gs + static_cast<std::size_t>(slot) * K;
        for (int k = 0; k < K; ++k) total = __dadd_rn(total, __dmul_rn(__ldg(g + k), mass_on(pw + k * V1, b)));
    }
    return total;
}

__device__ __forceinline__ double eq1_node(const ScoreArgs& s, unsigned int e0, unsigned int e1, bool* miss) {
    double v = 0.0;
    for (unsigned int e = e0; e < e1; ++e) {
        int slot = __ldg(s.acc_slot + e);
        unsigned long long b = __ldg(s.acc_bits + e) & s.amask;
        std::uint8_t fs = __ldg(s.fstate + slot);
        if (fs == 0) {
            *miss = true;
            continue;
        }
        v = __dadd_rn(v, mass_on(s.P + static_cast<std::size_t>(slot) * s.K * s.V1, b));
    }
    return v;
}

// score every light node; optionally build the stage-3 key/eff/W state in the
// same pass (the "score all, then select" fusion).
template <bool kKeys>
__global__ void __launch_bounds__(256) score_light_kernel(ScoreArgs s, KeyArgs ka, std::int64_t n_nodes,
                                                          int report_missing) {
    for (std::int64_t n = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; n < n_nodes;
         n += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        unsigned int e0 = s.acc_off[n], e1 = s.acc_off[n + 1];
        bool heavy = (e1 - e0) > static_cast<unsigned int>(kHeavyEntries);
        double total = 0.0;
        bool miss = false, shorth = false;
        if (!heavy) {
            total = eq2_node(s, e0, e1, &miss, &shorth);
            s.out[n] = total;
            if (report_missing && (miss || shorth))
                set_error(s.st, PBKV_EINVAL, miss ? kErrMissingForecast : kErrShortHorizon, n);
        }
        if constexpr (kKeys) {
            int ni = static_cast<int>(n);
            ka.eff[ni] = ni;
            ka.sublock[ni] = 0;
            ka.W[ni] = 0ull;
            ka.missing[ni] = (miss || shorth) ? 1 : 0;
            if (!heavy && ni != 0 && (ka.flags[ni] & kFlagTierMask) == PBKV_TIER_DEVICE) write_key(ka, ni, total);
        }
    }
}

// keys from the cached (mirrored) score
__global__ void __launch_bounds__(256) keys_cached_kernel(KeyArgs ka, std::int64_t n_nodes) {
    for (std::int64_t n = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; n < n_nodes;
         n += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        int ni = static_cast<int>(n);
        ka.eff[ni] = ni;
        ka.sublock[ni] = 0;
        ka.W[ni] = 0ull;
        ka.missing[ni] = 0;
        if (ni != 0 && (ka.flags[ni] & kFlagTierMask) == PBKV_TIER_DEVICE) write_key(ka, ni, ka.score_cached[ni]);
    }
}

// ---------------------------------------------------------------------------
// Stage 2, heavy nodes: one CTA per node.  The products x_i = gs*m are formed
// in parallel; the serial rounding chain t <- RN(t + x_i) is evaluated
// EXACTLY in parallel inside each binade: while t stays in [2^E, 2^(E+1)) and
// x_i >= 0, RN(t + x_i) = t + RN_u(x_i) with u = ulp(t) (rounding of x_i to a
// multiple of u is independent of t except at exact ties), so a run of steps
// is an integer prefix sum in units of u.  Binade crossings, exact ties,
// negative or huge x_i are "events" executed one at a time with __dadd_rn.
// Result: bit-identical to the sequential loop of scoring.hpp:52-60.
constexpr int kHeavyThreads = 256;
constexpr int kMaxK = 32;

struct SatAdd {
    __device__ __forceinline__ unsigned long long operator()(unsigned long long a, unsigned long long b) const {
        unsigned long long s = a + b;
        const unsigned long long cap = 1ull << 62;
        return (s > cap || s < a) ? cap : s;
    }
};

template <bool kValueOnly>
__global__ void __launch_bounds__(kHeavyThreads) heavy_score_kernel(ScoreArgs s, KeyArgs ka, const int* heavy,
                                                                    int write_keys, int report_missing) {
    using Scan = cub::BlockScan<unsigned long long, kHeavyThreads>;
    using RedI = cub::BlockReduce<int, kHeavyThreads>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ typename RedI::TempStorage red_tmp;
    extern __shared__ double xs[];  // kHeavyThreads * K products of the current chunk
    __shared__ double t_sh;
    __shared__ int ev_sh;
    __shared__ unsigned long long pclean_sh;
    __shared__ int miss_sh;

    const int node = heavy[blockIdx.x];
    const int K = kValueOnly ? 1 : s.K;
    const unsigned int e0 = s.acc_off[node], e1 = s.acc_off[node + 1];
    const int tid = threadIdx.x;
    if (tid == 0) {
        t_sh = 0.0;
        miss_sh = 0;
    }
    __syncthreads();

    for (unsigned int c0 = e0; c0 < e1; c0 += kHeavyThreads) {
        const int n_ent = static_cast<int>(min(static_cast<unsigned int>(kHeavyThreads), e1 - c0));
        const int nc = n_ent * K;
        // products, in chain order i = j*K + k (scoring.hpp:53-60)
        if (tid < n_ent) {
            unsigned int e = c0 + tid;
            int slot = __ldg(s.acc_slot + e);
            unsigned long long b = __ldg(s.acc_bits + e) & s.amask;
            std::uint8_t fs = __ldg(s.fstate + slot);
            bool ok = kValueOnly ? (fs != 0) : (fs == 1);
            if (!ok) {
                atomicOr(&miss_sh, fs == 2 ? 2 : 1);
                for (int k = 0; k < K; ++k) xs[tid * K + k] = 0.0;
            } else {
                const double* pw = s.P + static_cast<std::size_t>(slot) * s.K * s.V1;
                if (kValueOnly) {
                    xs[tid] = mass_on(pw, b);
                } else {
                    const double* g = s.gs + static_cast<std::size_t>(slot) * s.K;
                    for (int k = 0; k < K; ++k) xs[tid * K + k] = __dmul_rn(__ldg(g + k), mass_on(pw + k * s.V1, b));
                }
            }
        }
        __syncthreads();
        int pos = 0;
        while (pos < nc) {
            const double t = t_sh;
            int E = 0;
            bool fast = (t > 0x1p-900) && (t < 0x1p+1000);
            int ev = nc;
            unsigned long long pclean = 0;
            if (fast) {
                frexp(t, &E);  // t = f * 2^E, f in [0.5,1)  -> ulp(t) = 2^(E-53)
                const double scale = ldexp(1.0, 53 - E);  // x / ulp(t)
                const unsigned long long T = static_cast<unsigned long long>(t * scale);  // in [2^52, 2^53)
                const unsigned long long room = (1ull << 53) - T;
                // per-thread: the K elements of entry `tid`, chain order i0..i0+K-1
                auto qof = [&](int i, unsigned long long& q) -> bool {
                    double y = xs[i] * scale;  // exact: power-of-two scaling
                    if (!(y >= 0.0) || y > 0x1p53) return false;   // negative / NaN / crossing by itself
                    if (fabs(y - trunc(y)) == 0.5) return false;   // exact tie: depends on t's parity
                    q = static_cast<unsigned long long>(rint(y));
                    return true;
                };
                const int i0 = tid * K;
                unsigned long long local = 0;
                int my_first_bad = nc;
                for (int k = 0; k < K; ++k) {
                    int i = i0 + k;
                    if (tid >= n_ent || i < pos) continue;
                    unsigned long long q;
                    if (!qof(i, q)) {
                        my_first_bad = i;
                        break;
                    }
                    local = SatAdd()(local, q);
                }
                unsigned long long excl;
                Scan(scan_tmp).ExclusiveScan(local, excl, 0ull, SatAdd());
                // first crossing of the binade inside my run
                int my_ev = my_first_bad;
                unsigned long long run = excl;
                for (int k = 0; k < K; ++k) {
                    int i = i0 + k;
                    if (tid >= n_ent || i < pos) continue;
                    if (i >= my_first_bad) break;
                    unsigned long long q = 0;
                    qof(i, q);
                    unsigned long long nxt = SatAdd()(run, q);
                    if (nxt > room) {
                        my_ev = i;
                        break;
                    }
                    run = nxt;
                }
                __syncthreads();
                int blk_ev = RedI(red_tmp).Reduce(my_ev, cub::Min());
                if (tid == 0) ev_sh = blk_ev;
                __syncthreads();
                ev = ev_sh;
                // clean prefix = sum of q over [pos, ev): owner of element ev-1
                if (ev > pos && tid == (ev - 1) / K) {
                    unsigned long long p = excl;
                    for (int k = 0; k < K; ++k) {
                        int i = i0 + k;
                        if (i >= ev) break;
                        if (i < pos) continue;
                        unsigned long long q = 0;
                        qof(i, q);
                        p = SatAdd()(p, q);
                    }
                    pclean_sh = p;
                }
                __syncthreads();
                pclean = ev > pos ? pclean_sh : 0ull;
                if (tid == 0) {
                    double tn = static_cast<double>(T + pclean) / scale;  // exact: <= 2^53 units of ulp
                    if (ev < nc) {
                        tn = __dadd_rn(tn, xs[ev]);  // the event step, sequentially
                    }
                    t_sh = tn;
                }
                __syncthreads();
                pos = ev < nc ? ev + 1 : nc;
            } else {
                if (tid == 0) t_sh = __dadd_rn(t, xs[pos]);
                __syncthreads();
                pos += 1;
            }
        }
        __syncthreads();
    }
    if (tid == 0) {
        double total = t_sh;
        if (s.out) s.out[node] = total;
        bool miss = miss_sh != 0;
        if (report_missing && miss)
            set_error(s.st, PBKV_EINVAL, (miss_sh & 1) ? kErrMissingForecast : kErrShortHorizon, node);
        if (write_keys) {
            ka.missing[node] = miss ? 1 : 0;
            if ((ka.flags[node] & kFlagTierMask) == PBKV_TIER_DEVICE && node != 0) write_key(ka, node, total);
        }
    }
}

// Eq. 2 / Eq. 1 for an id list (refresh_nodes / single_step_value), light path
// per thread; heavy ids are flagged for the CTA path by the launcher.
template <bool kValueOnly>
__global__ void __launch_bounds__(256) score_ids_kernel(ScoreArgs s, const int* ids, std::int64_t n, int* heavy_out,
                                                        long long* n_heavy) {
    for (std::int64_t j = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; j < n;
         j += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        int id = ids[j];
        unsigned int e0 = s.acc_off[id], e1 = s.acc_off[id + 1];
        if (e1 - e0 > static_cast<unsigned int>(kHeavyEntries)) {
            long long slot = atomicAdd(reinterpret_cast<unsigned long long*>(n_heavy), 1ull);
            heavy_out[slot] = id;
            continue;
        }
        bool miss = false, shorth = false;
        double v = kValueOnly ? eq1_node(s, e0, e1, &miss) : eq2_node(s, e0, e1, &miss, &shorth);
        s.out[id] = v;
        if (miss || shorth) set_error(s.st, PBKV_EINVAL, miss ? kErrMissingForecast : kErrShortHorizon, id);
    }
}

// ---------------------------------------------------------------------------
// Stage 3: locked-subtree marks, subtree max of the candidate key.

// A locked DEVICE node makes itself and all its (device) ancestors ineligible:
// in the greedy frontier (policies.hpp:56-79) a locked node is never pushed,
// so no ancestor's virtual device-child count reaches 0.
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

// eff(n) = argmax of the key over n's device subtree.  Every device node walks
// its key up the ancestor chain with CAS on the ancestors' argmax id; a walk
// stops at the first ancestor already holding a larger key (whoever holds it
// carries it further), so the final eff is the exact subtree maximum.
__global__ void __launch_bounds__(256) eff_kernel(const int* parent, const std::uint8_t* flags, const Key2* keys,
                                                  int* eff, std::int64_t n_nodes) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n_nodes;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        int n = static_cast<int>(i);
        if (n == 0 || (flags[n] & kFlagTierMask) != PBKV_TIER_DEVICE) continue;
        const Key2 km = keys[n];
        int p = parent[n];
        while (p > 0) {
            int cur = *reinterpret_cast<volatile int*>(&eff[p]);
            bool advanced = false;
            for (;;) {
                Key2 kc = keys[cur];
                if (!key_less(kc, cur, km, n)) break;  // ancestor already holds >= my key
                int old = atomicCAS(&eff[p], cur, n);
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

// token weight of every head (chain), head list, total eligible tokens
__global__ void __launch_bounds__(256) weights_kernel(const int* len, const std::uint8_t* flags, const int* sublock,
                                                      const int* eff, const std::uint8_t* missing,
                                                      unsigned long long* W, int* heads, long long* counters,
                                                      DevStatus* st, std::int64_t n_nodes, int he_recompute) {
    unsigned long long tok = 0;
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n_nodes;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        int n = static_cast<int>(i);
        if (n == 0 || (flags[n] & kFlagTierMask) != PBKV_TIER_DEVICE || sublock[n]) continue;
        if (missing[n] == 2) set_error(st, PBKV_EINVAL, kErrKvflowMissing, n);
        if (he_recompute && missing[n] && !(flags[n] & kFlagRetired))
            set_error(st, PBKV_EINVAL, kErrMissingForecast, n);
        int h = eff[n];
        atomicAdd(&W[h], static_cast<unsigned long long>(len[n]));
        tok += static_cast<unsigned long long>(len[n]);
        if (h == n) {
            unsigned long long slot = atomicAdd(reinterpret_cast<unsigned long long*>(&counters[0]), 1ull);
            heads[slot] = n;
        }
    }
    using Red = cub::BlockReduce<unsigned long long, 256>;
    __shared__ typename Red::TempStorage tmp;
    unsigned long long blk = Red(tmp).Sum(tok);
    if (threadIdx.x == 0 && blk) atomicAdd(reinterpret_cast<unsigned long long*>(&counters[1]), blk);
}

__global__ void gather_heads_kernel(const int* heads, const Key2* keys, HeadKey* out, std::int64_t n) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        int h = heads[i];
        Key2 k = keys[h];
        out[i] = HeadKey{k.w0, k.w1, static_cast<unsigned int>(h)};
    }
}

__global__ void head_weights_kernel(const HeadKey* sorted, const unsigned long long* W, unsigned long long* w_sorted,
                                    int* rank, std::int64_t n) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        unsigned int h = sorted[i].id;
        w_sorted[i] = W[h];
        rank[h] = static_cast<int>(i);
    }
}

// first index whose inclusive prefix reaches `needed` (counters[2] = min index)
__global__ void find_cut_kernel(const unsigned long long* scan, std::int64_t n, long long needed, long long* out) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        unsigned long long prev = i ? scan[i - 1] : 0ull;
        if (scan[i] >= static_cast<unsigned long long>(needed) && prev < static_cast<unsigned long long>(needed))
            atomicMin(out, static_cast<long long>(i));
    }
}

// victim candidates: eligible nodes whose head ranks <= cut; sort key
// (rank, depth(head) - depth(n)) realises the (eff, d) order of the closed form
__global__ void __launch_bounds__(256) victim_keys_kernel(const std::uint8_t* flags, const int* sublock,
                                                          const int* eff, const int* rank, const int* depth,
                                                          long long cut, unsigned long long* vkey, int* vid,
                                                          long long* counter, std::int64_t n_nodes) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n_nodes;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        int n = static_cast<int>(i);
        if (n == 0 || (flags[n] & kFlagTierMask) != PBKV_TIER_DEVICE || sublock[n]) continue;
        int h = eff[n];
        int r = rank[h];
        if (r > cut) continue;
        unsigned long long d = static_cast<unsigned long long>(depth[h] - depth[n]);
        unsigned long long slot = atomicAdd(reinterpret_cast<unsigned long long*>(counter), 1ull);
        vkey[slot] = (static_cast<unsigned long long>(r) << 24) | d;
        vid[slot] = n;
    }
}

__global__ void victim_len_kernel(const int* vid, const int* len, unsigned long long* out, std::int64_t n) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
        out[i] = static_cast<unsigned long long>(len[vid[i]]);
}

// ---------------------------------------------------------------------------
// Stage 4: host-tier candidates with a device parent and Eq. 1 > 0
// (policies.hpp:190-198).
__global__ void __launch_bounds__(256) prefetch_cand_kernel(ScoreArgs s, const int* parent,
                                                            const std::uint8_t* flags,
                                                            const unsigned long long* last, CandKey* ck, double* cv,
                                                            long long* counters, DevStatus* st, std::int64_t n_nodes) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n_nodes;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        int n = static_cast<int>(i);
        if (n == 0 || (flags[n] & kFlagTierMask) != PBKV_TIER_HOST) continue;
        int p = parent[n];
        if ((flags[p] & kFlagTierMask) != PBKV_TIER_DEVICE) continue;
        unsigned int e0 = s.acc_off[n], e1 = s.acc_off[n + 1];
        bool miss = false;
        double v;
        if (e1 - e0 > static_cast<unsigned int>(kHeavyEntries)) {
            // rare: a popular host node; exact chain in-thread
            v = eq1_node(s, e0, e1, &miss);
        } else {
            v = eq1_node(s, e0, e1, &miss);
        }
        if (miss) {
            // the reference raises on the first host node in (last_access, id)
            // order (host_index_, cache.hpp:434): keep the minimum last_access
            atomicCAS(&st->code, 0, PBKV_EINVAL);
            atomicCAS(&st->kind, 0, kErrMissingForecast);
            atomicMin(reinterpret_cast<unsigned long long*>(&st->aux), last[n]);
            continue;
        }
        if (!(v > 0.0)) continue;
        unsigned long long slot = atomicAdd(reinterpret_cast<unsigned long long*>(&counters[0]), 1ull);
        unsigned long long e = enc_rank(v);
        ck[slot] = CandKey{~e, static_cast<unsigned int>(n)};
        cv[slot] = v;
    }
}

// among host nodes with the minimal last_access that miss a forecast, the
// smallest id (second pass, error path only)
__global__ void prefetch_err_id_kernel(ScoreArgs s, const int* parent, const std::uint8_t* flags,
                                       const unsigned long long* last, DevStatus* st, std::int64_t n_nodes) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n_nodes;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        int n = static_cast<int>(i);
        if (n == 0 || (flags[n] & kFlagTierMask) != PBKV_TIER_HOST) continue;
        if ((flags[parent[n]] & kFlagTierMask) != PBKV_TIER_DEVICE) continue;
        if (last[n] != static_cast<unsigned long long>(st->aux)) continue;
        bool miss = false;
        eq1_node(s, s.acc_off[n], s.acc_off[n + 1], &miss);
        if (miss) atomicMin(&st->node, static_cast<long long>(n));
    }
}

// greedy fill with skip (policies.hpp:203-210): one CTA walks the sorted
// candidates; per round it finds the first candidate that still fits
// (len <= budget - selected_tokens) with a block-wide min, selects it, and
// continues after it.
constexpr int kGreedyThreads = 1024;
__global__ void __launch_bounds__(kGreedyThreads) prefetch_greedy_kernel(const CandKey* sorted, const int* len,
                                                                         std::int64_t n, long long budget, int* sel,
                                                                         long long* counters) {
    using Red = cub::BlockReduce<long long, kGreedyThreads>;
    __shared__ typename Red::TempStorage tmp;
    __shared__ long long pick_sh;
    __shared__ long long rem_sh;
    __shared__ long long nsel_sh;
    if (threadIdx.x == 0) {
        rem_sh = budget;
        nsel_sh = 0;
    }
    __syncthreads();
    long long start = 0;
    while (start < n) {
        long long rem = rem_sh;
        long long i = start + threadIdx.x;
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
                int id = static_cast<int>(sorted[pick].id);
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

// survival + gs table + validation of uploaded forecast rows
// (Forecast ctor, forecast.hpp:19-42; gs[k] = gamma^k * s(k) with gamma^k by
// repeated multiplication exactly like scoring.hpp:56-58)
__global__ void forecast_prepare_kernel(const double* stage, const long long* slots, std::int64_t n, int H, int V1,
                                        int K, double gamma, double* P, double* gs, std::uint8_t* fstate,
                                        DevStatus* st) {
    for (std::int64_t j = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; j < n;
         j += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const double* p = stage + static_cast<std::size_t>(j) * H * V1;
        long long slot = slots[j];
        bool bad = false;
        for (int k = 0; k < H && !bad; ++k) {
            double s = 0.0;
            for (int a = 0; a < V1; ++a) {
                double v = p[k * V1 + a];
                if (v < -1e-12) {
                    set_error(st, PBKV_EINVAL, kErrForecastNegative, j);
                    bad = true;
                    break;
                }
                s = __dadd_rn(s, v);
            }
            if (!bad && fabs(__dsub_rn(s, 1.0)) > 1e-9) {
                set_error(st, PBKV_EINVAL, kErrForecastSum, j);
                bad = true;
            }
        }
        if (bad) continue;
        double* dst = P + static_cast<std::size_t>(slot) * K * V1;
        double* g = gs + static_cast<std::size_t>(slot) * K;
        double surv = 1.0, gk = 1.0;
        for (int k = 0; k < K; ++k) {
            if (k < H) {
                for (int a = 0; a < V1; ++a) dst[k * V1 + a] = p[k * V1 + a];
                g[k] = __dmul_rn(gk, surv);
                surv = __dmul_rn(surv, __dsub_rn(1.0, p[k * V1 + V1 - 1]));
                if (surv < 0.0) surv = 0.0;
            } else {
                for (int a = 0; a < V1; ++a) dst[k * V1 + a] = 0.0;
                g[k] = 0.0;
            }
            gk = __dmul_rn(gk, gamma);
        }
        fstate[slot] = H >= K ? 1 : 2;
    }
}

}  // namespace

// ---------------------------------------------------------------------------
// launchers

static ScoreArgs score_args(Context& c, double* out) {
    ScoreArgs s;
    s.acc_off = c.acc_off.p;
    s.acc_slot = c.acc_slot.p;
    s.acc_bits = c.acc_bits.p;
    s.P = c.P.p;
    s.gs = c.gs.p;
    s.fstate = c.fstate.p;
    s.K = c.K;
    s.V1 = c.V1;
    s.amask = c.A >= 64 ? ~0ull : ((1ull << c.A) - 1ull);
    s.out = out;
    s.st = c.status.p;
    return s;
}

static KeyArgs key_args(Context& c, int policy) {
    KeyArgs k;
    k.parent = c.parent.p;
    k.len = c.len.p;
    k.flags = c.flags.p;
    k.last = c.last.p;
    k.ever = c.ever.p;
    k.score_cached = c.score.p;
    k.acc_off = c.acc_off.p;
    k.acc_slot = c.acc_slot.p;
    k.acc_bits = c.acc_bits.p;
    k.rem_off = c.rem_off.p;
    k.rem_seq = c.rem_seq.p;
    k.rem_has = c.rem_has.p;
    k.keys = c.keys.p;
    k.eff = c.eff.p;
    k.sublock = c.sublock.p;
    k.W = c.W.p;
    k.missing = c.missing.p;
    k.st = c.status.p;
    k.policy = policy;
    return k;
}

static unsigned int sm_grid(Context&, std::int64_t n, int block) {
    // grid-stride kernels: enough CTAs for 148 SMs x 8 resident, capped by work
    std::int64_t want = (n + block - 1) / block;
    std::int64_t cap = 148LL * 8;
    if (want > cap) want = cap;
    return static_cast<unsigned int>(want < 1 ? 1 : want);
}

static std::size_t heavy_smem(int K) {
    static bool attr_set = false;
    if (!attr_set) {
        const int bytes = kHeavyThreads * kMaxK * static_cast<int>(sizeof(double));
        PBKV_CUDA(cudaFuncSetAttribute(heavy_score_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        PBKV_CUDA(cudaFuncSetAttribute(heavy_score_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        attr_set = true;
    }
    return static_cast<std::size_t>(kHeavyThreads) * static_cast<std::size_t>(K) * sizeof(double);
}

void reset_status(Context& c) {
    DevStatus z{0, 0, LLONG_MAX, LLONG_MAX};
    PBKV_CUDA(cudaMemcpyAsync(c.status.p, &z, sizeof z, cudaMemcpyHostToDevice, c.stream));
}

void launch_forecast_prepare(Context& c, const double* stage, const long long* slots, std::int64_t n, int H) {
    forecast_prepare_kernel<<<grid_for(n, 128), 128, 0, c.stream>>>(stage, slots, n, H, c.V1, c.K, c.gamma, c.P.p,
                                                                   c.gs.p, c.fstate.p, c.status.p);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

void launch_score_all(Context& c, double* out_dev, bool write_keys, int policy, bool want_missing) {
    ScoreArgs s = score_args(c, out_dev);
    KeyArgs ka = key_args(c, policy);
    if (c.n_heavy > 0) {
        heavy_score_kernel<false><<<static_cast<unsigned int>(c.n_heavy), kHeavyThreads, heavy_smem(c.K), c.stream>>>(
            s, ka, c.heavy.p, write_keys ? 1 : 0, want_missing ? 1 : 0);
        PBKV_CUDA(cudaGetLastError());
    ++c.launches;
    }
    if (write_keys)
        score_light_kernel<true><<<sm_grid(c, c.n, 256), 256, 0, c.stream>>>(s, ka, c.n, want_missing ? 1 : 0);
    else
        score_light_kernel<false><<<sm_grid(c, c.n, 256), 256, 0, c.stream>>>(s, ka, c.n, want_missing ? 1 : 0);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

void launch_score_ids(Context& c, const int* ids_dev, std::int64_t n, double* out_dev, bool value_only) {
    ScoreArgs s = score_args(c, out_dev);
    KeyArgs ka = key_args(c, PBKV_POLICY_HE);
    long long* nh = c.counters.p + 4;
    PBKV_CUDA(cudaMemsetAsync(nh, 0, sizeof(long long), c.stream));
    c.sel.reserve(static_cast<std::size_t>(n) + 1);
    if (value_only)
        score_ids_kernel<true><<<sm_grid(c, n, 256), 256, 0, c.stream>>>(s, ids_dev, n, c.sel.p, nh);
    else
        score_ids_kernel<false><<<sm_grid(c, n, 256), 256, 0, c.stream>>>(s, ids_dev, n, c.sel.p, nh);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
    PBKV_CUDA(cudaMemcpyAsync(c.hcounters.p + 4, nh, sizeof(long long), cudaMemcpyDeviceToHost, c.stream));
    PBKV_CUDA(cudaStreamSynchronize(c.stream));
    long long heavy = c.hcounters.p[4];
    if (heavy > 0) {
        if (value_only)
            heavy_score_kernel<true><<<static_cast<unsigned int>(heavy), kHeavyThreads, heavy_smem(1), c.stream>>>(
                s, ka, c.sel.p, 0, 1);
        else
            heavy_score_kernel<false><<<static_cast<unsigned int>(heavy), kHeavyThreads, heavy_smem(c.K), c.stream>>>(
                s, ka, c.sel.p, 0, 1);
        PBKV_CUDA(cudaGetLastError());
    ++c.launches;
    }
}

void launch_keys_cached(Context& c, int policy) {
    KeyArgs ka = key_args(c, policy);
    keys_cached_kernel<<<sm_grid(c, c.n, 256), 256, 0, c.stream>>>(ka, c.n);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

void launch_eff(Context& c, const int* locked_dev, std::int64_t n_locked) {
    if (n_locked > 0) {
        lock_kernel<<<grid_for(n_locked, 256), 256, 0, c.stream>>>(locked_dev, n_locked, c.parent.p, c.flags.p,
                                                                  c.sublock.p, c.n);
        PBKV_CUDA(cudaGetLastError());
    ++c.launches;
    }
    eff_kernel<<<sm_grid(c, c.n, 256), 256, 0, c.stream>>>(c.parent.p, c.flags.p, c.keys.p, c.eff.p, c.n);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

void launch_weights(Context& c, long long* counters_dev, bool he_recompute) {
    weights_kernel<<<sm_grid(c, c.n, 256), 256, 0, c.stream>>>(c.len.p, c.flags.p, c.sublock.p, c.eff.p, c.missing.p,
                                                              c.W.p, c.heads.p, counters_dev, c.status.p, c.n,
                                                              he_recompute ? 1 : 0);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

void launch_prefetch_candidates(Context& c, long long* counters_dev) {
    ScoreArgs s = score_args(c, nullptr);
    prefetch_cand_kernel<<<sm_grid(c, c.n, 256), 256, 0, c.stream>>>(s, c.parent.p, c.flags.p, c.last.p, c.ck_in.p,
                                                                     c.cv_in.p, counters_dev, c.status.p, c.n);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

void launch_prefetch_err_id(Context& c) {
    ScoreArgs s = score_args(c, nullptr);
    prefetch_err_id_kernel<<<sm_grid(c, c.n, 256), 256, 0, c.stream>>>(s, c.parent.p, c.flags.p, c.last.p, c.status.p,
                                                                       c.n);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

void launch_prefetch_greedy(Context& c, std::int64_t n_cand, long long budget, long long* counters_dev) {
    prefetch_greedy_kernel<<<1, kGreedyThreads, 0, c.stream>>>(c.ck_out.p, c.len.p, n_cand, budget, c.sel.p,
                                                               counters_dev);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

void launch_gather_heads(Context& c, std::int64_t n_heads) {
    gather_heads_kernel<<<sm_grid(c, n_heads, 256), 256, 0, c.stream>>>(c.heads.p, c.keys.p, c.hk_in.p, n_heads);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

void launch_head_weights(Context& c, std::int64_t n_heads) {
    head_weights_kernel<<<sm_grid(c, n_heads, 256), 256, 0, c.stream>>>(c.hk_out.p, c.W.p, c.wsorted.p, c.rank.p,
                                                                        n_heads);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

void launch_find_cut(Context& c, const unsigned long long* scan, std::int64_t n, long long needed, long long* out) {
    find_cut_kernel<<<sm_grid(c, n, 256), 256, 0, c.stream>>>(scan, n, needed, out);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

void launch_victim_keys(Context& c, long long cut, long long* counter) {
    victim_keys_kernel<<<sm_grid(c, c.n, 256), 256, 0, c.stream>>>(c.flags.p, c.sublock.p, c.eff.p, c.rank.p,
                                                                   c.depth.p, cut, c.vkey_in.p, c.vid_in.p, counter,
                                                                   c.n);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

void launch_victim_len(Context& c, std::int64_t n) {
    victim_len_kernel<<<sm_grid(c, n, 256), 256, 0, c.stream>>>(c.vid_out.p, c.len.p, c.vscan.p, n);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

namespace {
__global__ void gather_f64_kernel(const double* src, const int* ids, std::int64_t n, double* dst) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
        dst[i] = src[ids[i]];
}
}  // namespace

void launch_gather_f64(Context& c, const double* src, const int* ids, std::int64_t n, double* dst) {
    gather_f64_kernel<<<sm_grid(c, n, 256), 256, 0, c.stream>>>(src, ids, n, dst);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

// ---- CUB wrappers ---------------------------------------------------------------
struct HeadDecomposer {
    __host__ __device__ ::cuda::std::tuple<unsigned long long&, unsigned long long&, unsigned int&> operator()(
        HeadKey& k) const {
        return {k.w0, k.w1, k.id};
    }
};
struct CandDecomposer {
    __host__ __device__ ::cuda::std::tuple<unsigned long long&, unsigned int&> operator()(CandKey& k) const {
        return {k.vdesc, k.id};
    }
};

std::size_t cub_sort_heads_bytes(std::int64_t n) {
    std::size_t b = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, b, static_cast<HeadKey*>(nullptr), static_cast<HeadKey*>(nullptr),
                                   static_cast<int>(n), HeadDecomposer{});
    return b;
}

void cub_sort_heads(Context& c, std::int64_t n) {
    std::size_t b = cub_sort_heads_bytes(n);
    c.cub_tmp.reserve(b);
    ++c.lib_calls;
    PBKV_CUDA(cub::DeviceRadixSort::SortKeys(c.cub_tmp.p, b, c.hk_in.p, c.hk_out.p, static_cast<int>(n),
                                             HeadDecomposer{}, c.stream));
}

std::size_t cub_scan_bytes(std::int64_t n) {
    std::size_t b = 0;
    cub::DeviceScan::InclusiveSum(nullptr, b, static_cast<unsigned long long*>(nullptr),
                                  static_cast<unsigned long long*>(nullptr), static_cast<int>(n));
    return b;
}

void cub_scan_u64(Context& c, const unsigned long long* in, unsigned long long* out, std::int64_t n) {
    std::size_t b = cub_scan_bytes(n);
    c.cub_tmp.reserve(b);
    ++c.lib_calls;
    PBKV_CUDA(cub::DeviceScan::InclusiveSum(c.cub_tmp.p, b, in, out, static_cast<int>(n), c.stream));
}

std::size_t cub_sort_pairs_bytes(std::int64_t n) {
    std::size_t b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b, static_cast<unsigned long long*>(nullptr),
                                    static_cast<unsigned long long*>(nullptr), static_cast<int*>(nullptr),
                                    static_cast<int*>(nullptr), static_cast<int>(n));
    return b;
}

void cub_sort_pairs_u64(Context& c, std::int64_t n, int end_bit) {
    std::size_t b = cub_sort_pairs_bytes(n);
    c.cub_tmp.reserve(b);
    ++c.lib_calls;
    PBKV_CUDA(cub::DeviceRadixSort::SortPairs(c.cub_tmp.p, b, c.vkey_in.p, c.vkey_out.p, c.vid_in.p, c.vid_out.p,
                                              static_cast<int>(n), 0, end_bit, c.stream));
}

std::size_t cub_sort_cands_bytes(std::int64_t n) {
    std::size_t b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b, static_cast<CandKey*>(nullptr), static_cast<CandKey*>(nullptr),
                                    static_cast<double*>(nullptr), static_cast<double*>(nullptr), static_cast<int>(n),
                                    CandDecomposer{});
    return b;
}

void cub_sort_cands(Context& c, std::int64_t n) {
    std::size_t b = cub_sort_cands_bytes(n);
    c.cub_tmp.reserve(b);
    ++c.lib_calls;
    PBKV_CUDA(cub::DeviceRadixSort::SortPairs(c.cub_tmp.p, b, c.ck_in.p, c.ck_out.p, c.cv_in.p, c.cv_out.p,
                                              static_cast<int>(n), CandDecomposer{}, c.stream));
}

}  // namespace pbkv
