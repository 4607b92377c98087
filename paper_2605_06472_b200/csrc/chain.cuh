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

constexpr int kChainT = 1024;              // threads of a chain CTA
constexpr int kChainG = 12;                // elements per thread per window
constexpr int kChainW = kChainT * kChainG;  // window: 12288 doubles (96 KB)

struct ChainSatAdd {
    __device__ __forceinline__ unsigned long long operator()(unsigned long long a, unsigned long long b) const {
        const unsigned long long r = a + b;
        const unsigned long long cap = 1ull << 62;
        return (r > cap || r < a) ? cap : r;
    }
};

struct ChainSmem {
    double x[kChainW];
    union {
        typename cub::BlockScan<unsigned long long, kChainT>::TempStorage scan;
        typename cub::BlockReduce<int, kChainT>::TempStorage red;
    } tmp;
    double t;
    int ev;
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

// Evaluates the chain over xg[0, L) (global memory); returns t in every thread.
__device__ double chain_eval(const double* __restrict__ xg, long long L, ChainSmem& sm) {
    using Scan = cub::BlockScan<unsigned long long, kChainT>;
    using Red = cub::BlockReduce<int, kChainT>;
    const int tid = threadIdx.x;
    if (tid == 0) sm.t = 0.0;
    for (long long w0 = 0; w0 < L; w0 += kChainW) {
        const int nw = static_cast<int>(min(static_cast<long long>(kChainW), L - w0));
        __syncthreads();  // previous window fully consumed
        for (int i = tid; i < nw; i += kChainT) sm.x[i] = __ldcg(xg + w0 + i);
        __syncthreads();
        const int a0 = tid * kChainG;
        int pos = 0;
        while (pos < nw) {
            const double t = sm.t;
            if (!(t >= 0x1p-900 && t < 0x1p+1000)) {  // zero / tiny / huge / NaN: one serial step
                __syncthreads();
                if (tid == 0) sm.t = __dadd_rn(t, sm.x[pos]);
                __syncthreads();
                ++pos;
                continue;
            }
            const int e = static_cast<int>((__double_as_longlong(t) >> 52) & 0x7ff) - 1023;  // t in [2^e, 2^(e+1))
            const double scale = __longlong_as_double(static_cast<long long>(1023 + 52 - e) << 52);  // 2^(52-e)
            const unsigned long long T = static_cast<unsigned long long>(t * scale);                // [2^52, 2^53)
            const unsigned long long room = (1ull << 53) - T;
            unsigned long long local = 0;
            int first_bad = INT_MAX;
#pragma unroll
            for (int k = 0; k < kChainG; ++k) {
                const int i = a0 + k;
                if (i < pos || i >= nw || first_bad != INT_MAX) continue;
                unsigned long long q;
                if (chain_q(sm.x[i], scale, q))
                    local = ChainSatAdd()(local, q);
                else
                    first_bad = i;
            }
            unsigned long long excl, agg;
            Scan(sm.tmp.scan).ExclusiveScan(local, excl, 0ull, ChainSatAdd(), agg);
            int ev = INT_MAX;
            unsigned long long run = excl;
#pragma unroll
            for (int k = 0; k < kChainG; ++k) {
                const int i = a0 + k;
                if (i < pos || i >= nw || ev != INT_MAX) continue;
                unsigned long long q = 0;
                if (i == first_bad) {
                    ev = i;
                    continue;
                }
                chain_q(sm.x[i], scale, q);
                const unsigned long long nxt = ChainSatAdd()(run, q);
                if (nxt > room)
                    ev = i;
                else
                    run = nxt;
            }
            __syncthreads();  // scan storage reused by the reduction
            const int EV = Red(sm.tmp.red).Reduce(ev, cub::Min());
            if (tid == 0) sm.ev = EV;
            __syncthreads();
            const int E = sm.ev;
            if (E == INT_MAX) {
                if (tid == 0) sm.t = static_cast<double>(T + agg) / scale;  // exact (<= 2^53 units)
                pos = nw;
            } else {
                if (ev == E) sm.t = __dadd_rn(static_cast<double>(T + run) / scale, sm.x[E]);  // the event step
                pos = E + 1;
            }
            __syncthreads();
        }
    }
    __syncthreads();
    return sm.t;
}

}  // namespace dev
}  // namespace pbkv
