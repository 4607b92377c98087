// The serial FP64 rounding chain t <- RN(t + x_i), i = 0..L-1 (t_0 = +0.0),
// evaluated exactly by one CTA.  This is the inner loop of Eq. 2 for nodes
// tagged by thousands of workflows (scoring.hpp:52-60: total += term, in
// WorkflowId / step order, binary64, no FMA) -- SURVEY.md §7 hard part 1.
//
// Inside one binade [2^e, 2^(e+1)) with ulp u = 2^(e-52), and x_i >= 0,
//     RN(t + x_i) = t + u * rint(x_i / u)
// unless x_i / u has a fractional part of exactly 1/2 (the tie rounds to even,
// which depends on t).  So a run of steps that stays inside the binade is an
// integer prefix sum in units of u.  Per binade the CTA forms q_i =
// rint(x_i / u) for every remaining element of the window, scans them, and
// finds the first "event": the step that leaves the binade (prefix > 2^53 -
// t/u), an exact tie, or an abnormal x_i (negative, NaN, >= the binade width).
// The event step itself is executed with __dadd_rn on the exact value of t
// before it.  The number of scans is the number of binade crossings (about
// log2(total / first term), ~20 at C3) plus ties, independent of L.
// Bit-identical to the serial loop.
#pragma once

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

namespace pbkv {
namespace dev {

constexpr int kChainT = 512;               // threads of a chain CTA (128 registers each)
constexpr int kChainG = 24;                // elements per thread per window (in registers)
constexpr int kChainW = kChainT * kChainG;  // window: 12288 elements held in registers

struct ChainSatAdd {
    __device__ __forceinline__ unsigned long long operator()(unsigned long long a, unsigned long long b) const {
        const unsigned long long r = a + b;
        const unsigned long long cap = 1ull << 62;
        return (r > cap || r < a) ? cap : r;
    }
};

struct ChainSmem {
    typename cub::BlockScan<double, kChainT>::TempStorage scand;
    unsigned long long wsum[kChainT / 32];
    long long wmin[kChainT / 32];
    double t;
};

// q = rint(x * scale) when that is the exact in-binade increment; false for an event
__device__ __forceinline__ bool chain_q(double x, double scale, unsigned long long& q) {
    const double y = x * scale;  // exact: scale is a power of two and t >= 2^-900
    if (!(y >= 0.0) || y > 0x1p53) return false;
    const double r = rint(y);
    if (fabs(y - r) == 0.5) return false;  // exact tie: rounding depends on t's parity
    q = static_cast<unsigned long long>(r);
    return true;
}

// Two-level shuffle scan / min over the CTA (kChainT / 32 warps): far lower
// latency than a raking block scan for the one-value-per-thread case.
__device__ __forceinline__ unsigned long long chain_block_excl(unsigned long long v, unsigned long long* wsum,
                                                               unsigned long long& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    constexpr int kW = kChainT / 32;
    unsigned long long w = lane < kW ? wsum[lane] : 0ull;
#pragma unroll
    for (int o = 1; o < kW; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
    }
    const unsigned long long before = warp ? __shfl_sync(0xffffffffu, w, warp - 1) : 0ull;
    total = __shfl_sync(0xffffffffu, w, kW - 1);
    return before + x - v;
}

__device__ __forceinline__ long long chain_block_min(long long v, long long* wmin) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) v = min(v, static_cast<long long>(__shfl_xor_sync(0xffffffffu, v, o)));
    if (lane == 0) wmin[warp] = v;
    __syncthreads();
    constexpr int kW = kChainT / 32;
    long long w = lane < kW ? wmin[lane] : LLONG_MAX;
#pragma unroll
    for (int o = 16; o; o >>= 1) w = min(w, static_cast<long long>(__shfl_xor_sync(0xffffffffu, w, o)));
    return w;
}

// Evaluates the chain over xg[0, L) (global memory); returns t in every thread.
// Each thread keeps its contiguous run of kChainG elements of the window in
// registers.  A pass only does element work in the threads whose elements can
// lie before the next binade crossing: an approximate (plain FP64 scan) prefix
// of the window locates the crossing, and the first thread past it reports a
// "stop" event -- the pass ends exactly there (no step is taken) and the next
// pass resumes from it, so the estimate affects only speed, never the result.
// Integer prefixes use plain (wrapping) adds: up to the first index whose
// prefix exceeds `room` (< 2^53) they are exact, and nothing after it is used.
__device__ double chain_eval(const double* __restrict__ xg, long long L, ChainSmem& sm) {
    using ScanD = cub::BlockScan<double, kChainT>;
    const int tid = threadIdx.x;
    if (tid == 0) sm.t = 0.0;
#ifdef PBKV_CHAIN_DEBUG
    long long dbg_passes = 0, dbg_serial = 0, dbg_t0 = clock64();
    long long dbg_ph[6] = {0, 0, 0, 0, 0, 0}, dbg_c = 0;
#define PBKV_PH(i)                      \
    do {                                \
        long long now_ = clock64();     \
        dbg_ph[i] += now_ - dbg_c;      \
        dbg_c = now_;                   \
    } while (0)
#else
#define PBKV_PH(i) \
    do {           \
    } while (0)
#endif
    for (long long w0 = 0; w0 < L; w0 += kChainW) {
        const int nw = static_cast<int>(min(static_cast<long long>(kChainW), L - w0));
        const int a0 = tid * kChainG;
        double xr[kChainG];
        double lsum = 0.0;
#pragma unroll
        for (int k = 0; k < kChainG; ++k) {
            xr[k] = a0 + k < nw ? __ldcg(xg + w0 + a0 + k) : 0.0;
            lsum += fabs(xr[k]);
        }
        __syncthreads();  // sm.t of the previous window visible; scan storage free
        double sbefore;   // approximate running total before this thread's elements
        ScanD(sm.scand).ExclusiveSum(lsum, sbefore);
        sbefore += sm.t;
        int pos = 0;
        while (pos < nw) {
#ifdef PBKV_CHAIN_DEBUG
            dbg_c = clock64();
#endif
            __syncthreads();
            const double t = sm.t;
            PBKV_PH(0);
            if (!(t >= 0x1p-900 && t < 0x1p+1000)) {  // zero / tiny / huge / NaN: one serial step
#ifdef PBKV_CHAIN_DEBUG
                ++dbg_serial;
#endif
                __syncthreads();
                if (pos >= a0 && pos < a0 + kChainG) {
#pragma unroll
                    for (int k = 0; k < kChainG; ++k)
                        if (a0 + k == pos) sm.t = __dadd_rn(t, xr[k]);
                }
                ++pos;
                continue;
            }
#ifdef PBKV_CHAIN_DEBUG
            ++dbg_passes;
#endif
            const int e = static_cast<int>((__double_as_longlong(t) >> 52) & 0x7ff) - 1023;  // t in [2^e, 2^(e+1))
            const double scale = __longlong_as_double(static_cast<long long>(1023 + 52 - e) << 52);  // 2^(52-e)
            const unsigned long long T = static_cast<unsigned long long>(t * scale);                // [2^52, 2^53)
            const unsigned long long room = (1ull << 53) - T;
            const double unit = __longlong_as_double(static_cast<long long>(1023 + e - 52) << 52);  // ulp(t) = 1/scale
            // threads wholly past the (approximate) crossing do no element work
            const double limit = __longlong_as_double(static_cast<long long>(1023 + e + 1) << 52) * (1.0 + 0x1p-20);
            const bool mine = a0 + kChainG > pos && a0 < nw;
            const bool past = mine && a0 >= pos && sbefore > limit;
            const bool work = mine && !past;
            // Element loops are branch-free (selects only) and guarded by
            // warp-uniform votes, so the shuffles below stay convergent and
            // idle warps skip the bodies entirely.
            unsigned int ok = 0;  // bit k: element k is an in-binade step
            unsigned long long local = 0;
            int first_bad = INT_MAX;
            if (__any_sync(0xffffffffu, work)) {
#pragma unroll
                for (int k = 0; k < kChainG; ++k) {
                    const int i = a0 + k;
                    const bool in = work && i >= pos && i < nw;
                    const double y = xr[k] * scale;
                    const double r = rint(y);
                    const bool good = (y >= 0.0) && (y <= 0x1p53) && (fabs(y - r) != 0.5);
                    const unsigned long long q = good ? static_cast<unsigned long long>(r) : 0ull;
                    ok |= (in && good) ? (1u << k) : 0u;
                    first_bad = (in && !good && first_bad == INT_MAX) ? i : first_bad;
                    local += (in && first_bad == INT_MAX) ? q : 0ull;
                }
            }
            PBKV_PH(1);
            unsigned long long agg;
            const unsigned long long excl = chain_block_excl(local, sm.wsum, agg);
            PBKV_PH(2);
            long long ev = past ? 2ll * a0 + 1 : LLONG_MAX;  // 2*index (+1 for a stop event)
            unsigned long long run = excl;
            int evk = 0;
            const bool need2 = work && (first_bad != INT_MAX || excl + local > room);  // the event is in my range
            if (__any_sync(0xffffffffu, need2)) {
#pragma unroll
                for (int k = 0; k < kChainG; ++k) {
                    const int i = a0 + k;
                    const bool act = need2 && i >= pos && i < nw && ev == LLONG_MAX;
                    const bool good = (ok >> k) & 1u;
                    const double r = rint(xr[k] * scale);
                    const unsigned long long nxt = run + (good ? static_cast<unsigned long long>(r) : 0ull);
                    const bool hit = act && (!good || nxt > room);
                    ev = hit ? 2ll * i : ev;
                    evk = hit ? k : evk;
                    run = (act && !hit) ? nxt : run;
                }
            }
            PBKV_PH(3);
            const long long E = chain_block_min(ev, sm.wmin);
            PBKV_PH(4);
            if (E == LLONG_MAX) {
                if (tid == 0) sm.t = static_cast<double>(T + agg) * unit;  // exact (<= 2^53 units)
                pos = nw;
            } else if (E & 1) {  // stop: the run so far is exact; resume at the stop index
                if (ev == E) sm.t = static_cast<double>(T + run) * unit;
                pos = static_cast<int>(E >> 1);
            } else {
                if (ev == E) {  // the event step, on the exact value of t before it
                    double xe = 0.0;
#pragma unroll
                    for (int k = 0; k < kChainG; ++k)
                        if (k == evk) xe = xr[k];
                    sm.t = __dadd_rn(static_cast<double>(T + run) * unit, xe);
                }
                pos = static_cast<int>(E >> 1) + 1;
            }
            PBKV_PH(5);
        }
    }
    __syncthreads();
#ifdef PBKV_CHAIN_DEBUG
    if (tid == 0)
        printf("chain L=%lld passes=%lld serial=%lld cycles=%lld ph=%lld %lld %lld %lld %lld %lld\n", L, dbg_passes,
               dbg_serial, clock64() - dbg_t0, dbg_ph[0], dbg_ph[1], dbg_ph[2], dbg_ph[3], dbg_ph[4], dbg_ph[5]);
#endif
    return sm.t;
}

}  // namespace dev
}  // namespace pbkv
