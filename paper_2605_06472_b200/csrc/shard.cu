// Node-set sharding of stages 2-3 across GPUs (BASELINE config 4).
//
// A rank holds the subtrees below the shared "spine" that it owns, plus a
// copy of the spine itself (the ancestors whose subtrees span ranks).  Local
// node ids are increasing in global id, so local tie-breaks agree with global
// ones.  Spine nodes are flagged kFlagExcluded: they never enter the local
// order, their keys are zeroed so eff(spine) is the maximum over the rank's
// own descendants, and chains stop below them.  The global victim order is
// then the merge of the per-rank orders plus the spine records, cut at the
// shortest prefix with sum(len) >= needed:
//   - each rank's local cut (shortest local prefix reaching `needed`) bounds
//     its share of the global prefix, so exchanging only local cuts is exact;
//   - spine scores (HE) are exact chains over all ranks' products in global
//     WorkflowId order (ranks own contiguous WorkflowId blocks).
// Kernels: candidate records of the local cut, spine reports, spine products,
// merge-path rank merge of the exchanged runs, single-CTA cut.
#include <cub/block/block_scan.cuh>

#include <algorithm>

#include "common.cuh"

namespace pbkv {

using namespace dev;

namespace {

__device__ __forceinline__ bool cand_less(const pbkv_cand& a, const pbkv_cand& b) {
    if (a.w0 != b.w0) return a.w0 < b.w0;
    if (a.w1 != b.w1) return a.w1 < b.w1;
    if (a.eff_gid != b.eff_gid) return a.eff_gid < b.eff_gid;
    return a.d < b.d;
}

__global__ void mark_excluded_kernel(std::uint8_t* flags, const int* ids, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flags[ids[i]] |= kFlagExcluded;
}

// record of victim i of the local cut: the key of its chain head, the head's
// global id, its distance below the head, its length, its global id
__global__ void records_kernel(const int* victims, const long long* result, const Key2* keys, const int* eff,
                               const int* depth, const int* len, const int* gid, pbkv_cand* out) {
    const long long n = result[0];
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int v = victims[i];
        const int h = eff[v];
        const Key2 k = load_key(keys, h);
        pbkv_cand r;
        r.w0 = k.w0;
        r.w1 = k.w1;
        r.eff_gid = gid[h];
        r.gid = gid[v];
        r.d = depth[h] - depth[v];
        r.len = len[v];
        out[i] = r;
    }
}

// per spine node: the maximum key over the rank's device descendants (eff
// after the selection's walk) and whether a locked node lies below.  One CTA
// per spine node strides over its children (the shared prefix has a child
// per workflow group: a serial loop took 1 ms at config 4) and reduces.
__global__ void __launch_bounds__(256) spine_report_kernel(const int* spine, int n_spine, const int* ch_off,
                                                           const int* ch, const Key2* keys, const int* eff,
                                                           const int* sublock, const int* depth, const int* gid,
                                                           const std::uint8_t* flags, pbkv_spine_info* out) {
    const int j = blockIdx.x;
    if (j >= n_spine) return;
    const int s = spine[j];
    // max over the in-order device children's eff (the walk stops below the
    // spine; spine children are combined on the host, shard.py)
    int e = -1;
    Key2 best{0, 0};
    for (int q = ch_off[j] + static_cast<int>(threadIdx.x); q < ch_off[j + 1]; q += blockDim.x) {
        const int c = ch[q];
        if ((flags[c] & (kFlagTierMask | kFlagOutOfOrder)) != PBKV_TIER_DEVICE) continue;
        const int ec = eff[c];
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
    __shared__ unsigned long long s0[8], s1[8];
    __shared__ int se[8];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        s0[warp] = best.w0;
        s1[warp] = best.w1;
        se[warp] = e;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    e = -1;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
        const Key2 bk{s0[w], s1[w]};
        if (se[w] >= 0 && (e < 0 || key_less(best, e, bk, se[w]))) {
            e = se[w];
            best = bk;
        }
    }
    pbkv_spine_info r;
    r.has_eff = e >= 0 ? 1 : 0;
    r.w0 = e >= 0 ? best.w0 : 0ull;
    r.w1 = e >= 0 ? best.w1 : 0ull;
    r.eff_gid = e >= 0 ? gid[e] : -1;
    r.eff_depth = e >= 0 ? depth[e] : -1;
    r.sublock = sublock[s] ? 1 : 0;
    out[j] = r;
}

// Eq. 2 products (gs * mass_on, scoring.hpp:56-57) of the spine nodes' local
// entries, node-major, entries in WorkflowId order, K per entry
__global__ void spine_products_kernel(ScoreArgs s, const int* spine, const long long* base, int n_spine, double* out,
                                      unsigned int* miss) {
    const int j = blockIdx.y;
    if (j >= n_spine) return;
    const int node = spine[j];
    const uint2 rg = s.acc_rng[node];
    const unsigned int e0 = rg.x, e1 = rg.y;
    const long long L = static_cast<long long>(e1 - e0) * s.K;
    for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < L;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        const unsigned int e = e0 + static_cast<unsigned int>(t / s.K);
        const int k = static_cast<int>(t % s.K);
        const int slot = __ldg(s.acc_slot + e);
        const unsigned long long b = __ldg(s.acc_bits + e) & s.amask;
        double x = 0.0;
        if (__ldg(s.fstate + slot) != 1) {
            atomicOr(miss, 1u);
        } else {
            const double* col = s.P + static_cast<std::size_t>(slot) * s.V1 * s.K + k;
            x = __dmul_rn(__ldg(s.gs + static_cast<std::size_t>(slot) * s.K + k), mass_on(col, s.K, b));
        }
        out[base[j] + t] = x;
    }
}

// merge of sorted runs (disjoint unique keys): element i of run r lands at
// i + sum over other runs of their count of smaller keys
__global__ void merge_runs_kernel(const pbkv_cand* src, const long long* run_start, const long long* run_len,
                                  const long long* out_base, int n_runs, pbkv_cand* dst) {
    const int r = blockIdx.y;
    const long long n = run_len[r];
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const pbkv_cand x = src[run_start[r] + i];
        long long pos = i;
        for (int q = 0; q < n_runs; ++q) {
            if (q == r) continue;
            const pbkv_cand* b = src + run_start[q];
            long long lo = 0, hi = run_len[q];
            while (lo < hi) {
                const long long mid = (lo + hi) >> 1;
                if (cand_less(b[mid], x))
                    lo = mid + 1;
                else
                    hi = mid;
            }
            pos += lo;
        }
        dst[pos] = x;
        (void)out_base;
    }
}

// shortest prefix of the merged order with sum(len) >= needed (all if none),
// in two launches over every SM: the tokens of each CTA's chunk, then each
// CTA's prefix (the partial sums before it) and a block scan of its chunk --
// element i is a victim iff the tokens before it are < needed; the element
// that crosses `needed` (or the last CTA, when none does) writes the result
constexpr int kCutT = 512;
__global__ void __launch_bounds__(kCutT) cut_partials_kernel(const pbkv_cand* m, long long n, long long chunk,
                                                             long long* partial) {
    const long long b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
    long long s = 0;
    for (long long i = b0 + threadIdx.x; i < b1; i += kCutT) s += m[i].len;
    using Red = cub::BlockReduce<long long, kCutT>;
    __shared__ typename Red::TempStorage tmp;
    const long long t = Red(tmp).Sum(s);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

__global__ void __launch_bounds__(kCutT) cut_apply_kernel(const pbkv_cand* m, long long n, long long chunk,
                                                          const long long* partial, long long needed, int* victims,
                                                          long long* result) {
    using Scan = cub::BlockScan<long long, kCutT>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ long long pre_sh;
    if (threadIdx.x == 0) {
        long long p = 0;
        for (unsigned int g = 0; g < blockIdx.x; ++g) p += partial[g];
        pre_sh = p;
    }
    __syncthreads();
    long long carry = pre_sh;
    const long long b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
    if (carry >= needed) return;  // wholly after the cut
    for (long long c0 = b0; c0 < b1; c0 += kCutT) {
        const long long i = c0 + threadIdx.x;
        const long long v = i < b1 ? static_cast<long long>(m[i].len) : 0;
        long long excl, agg;
        Scan(tmp).ExclusiveSum(v, excl, agg);
        __syncthreads();
        excl += carry;
        if (i < b1 && excl < needed) {
            victims[i] = m[i].gid;
            if (excl + v >= needed) {  // the cut
                result[0] = i + 1;
                result[1] = excl + v;
                result[2] = 0;
            }
        }
        carry += agg;
        if (carry >= needed) return;
    }
    if (blockIdx.x == gridDim.x - 1) {  // nothing reached `needed`: every record
        result[0] = n;
        result[1] = carry;
        result[2] = carry < needed ? 1 : 0;
    }
}

unsigned int grid_for_cap(long long n, int block) {
    long long g = (n + block - 1) / block;
    if (g > 148 * 8) g = 148 * 8;
    return static_cast<unsigned int>(g < 1 ? 1 : g);
}

}  // namespace

void shard_apply_flags(Context& c) {
    if (c.spine.empty()) return;
    c.spine_dev.reserve(c.spine.size());
    PBKV_CUDA(cudaMemcpyAsync(c.spine_dev.p, c.spine.data(), c.spine.size() * sizeof(int), cudaMemcpyHostToDevice,
                              c.stream));
    const int n = static_cast<int>(c.spine.size());
    mark_excluded_kernel<<<(n + 127) / 128, 128, 0, c.stream>>>(c.flags.p, c.spine_dev.p, n);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

void shard_records(Context& c, long long* result_dev, pbkv_cand* out, long long cap_unused) {
    (void)cap_unused;
    records_kernel<<<grid_for_cap(c.n, 256), 256, 0, c.stream>>>(c.vid_out.p, result_dev, c.keys.p, c.eff.p,
                                                                 c.depth.p, c.len.p, c.gid.p, out);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

void shard_spine_report(Context& c, pbkv_spine_info* out) {
    const int n = static_cast<int>(c.spine.size());
    if (n == 0) return;
    spine_report_kernel<<<n, 256, 0, c.stream>>>(c.spine_dev.p, n, c.sch_off.p, c.sch.p, c.keys.p,
                                                               c.eff.p, c.sublock.p, c.depth.p, c.gid.p, c.flags.p,
                                                               out);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

ScoreArgs make_score_args(Context& c, double* out);

void shard_spine_products(Context& c, const long long* base_dev, long long max_len, double* out, unsigned int* miss) {
    const int n = static_cast<int>(c.spine.size());
    if (n == 0 || max_len == 0) return;
    ScoreArgs s = make_score_args(c, nullptr);
    dim3 grid(grid_for_cap(max_len, 256), static_cast<unsigned int>(n));
    spine_products_kernel<<<grid, 256, 0, c.stream>>>(s, c.spine_dev.p, base_dev, n, out, miss);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

void shard_merge_cut(Context& c, const pbkv_cand* src, const long long* run_start_dev, const long long* run_len_dev,
                     int n_runs, long long max_run, long long total, pbkv_cand* merged, long long needed,
                     int* victims, long long* result) {
    if (total > 0) {
        dim3 grid(grid_for_cap(max_run, 256), static_cast<unsigned int>(n_runs));
        merge_runs_kernel<<<grid, 256, 0, c.stream>>>(src, run_start_dev, run_len_dev, nullptr, n_runs, merged);
        PBKV_CUDA(cudaGetLastError());
        ++c.launches;
    }
    const long long chunk = std::max<long long>(4 * kCutT, (total + 295) / 296);
    const unsigned int g = static_cast<unsigned int>(std::max<long long>(1, (total + chunk - 1) / chunk));
    c.cut_partial.reserve(g);
    if (total == 0) {  // nothing to take: the empty cut
        PBKV_CUDA(cudaMemsetAsync(result, 0, 2 * sizeof(long long), c.stream));
        const long long one = needed > 0 ? 1 : 0;
        PBKV_CUDA(cudaMemcpyAsync(result + 2, &one, sizeof one, cudaMemcpyHostToDevice, c.stream));
        PBKV_CUDA(cudaStreamSynchronize(c.stream));
        return;
    }
    cut_partials_kernel<<<g, kCutT, 0, c.stream>>>(merged, total, chunk, c.cut_partial.p);
    cut_apply_kernel<<<g, kCutT, 0, c.stream>>>(merged, total, chunk, c.cut_partial.p, needed, victims, result);
    PBKV_CUDA(cudaGetLastError());
    c.launches += 2;
}


// ---- interval sums of the exchanged spine products (shard.py fast path) -------------
// Output j: the sum and the sum of magnitudes of x over its pieces
// [pieces[2q], pieces[2q+1]) for q in [out_off[j], out_off[j+1]), any order
// within a piece (block reduction), pieces in order: deterministic.  One CTA
// per output; the results go straight to pinned host memory.
namespace {
constexpr int kIsT = 256;
__global__ void __launch_bounds__(kIsT) interval_sums_kernel(const double* x, const long long* pieces,
                                                            const long long* out_off, double* out) {
    __shared__ double red[2][kIsT / 32];
    const int j = blockIdx.x;
    double s = 0.0, sa = 0.0;
    for (long long q = out_off[j]; q < out_off[j + 1]; ++q) {
        for (long long i = pieces[2 * q] + threadIdx.x; i < pieces[2 * q + 1]; i += kIsT) {
            const double v = __ldg(x + i);
            s += v;
            sa += fabs(v);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        sa += __shfl_xor_sync(0xffffffffu, sa, o);
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = s;
        red[1][threadIdx.x >> 5] = sa;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0, ta = 0.0;
        for (int w = 0; w < kIsT / 32; ++w) {
            t += red[0][w];
            ta += red[1][w];
        }
        out[2 * j] = t;
        out[2 * j + 1] = ta;
    }
}
}  // namespace

void launch_interval_sums(Context& c, const double* x, const long long* pieces, const long long* out_off, int n_out,
                          double* out_host) {
    interval_sums_kernel<<<n_out, kIsT, 0, c.stream>>>(x, pieces, out_off, out_host);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
}

}  // namespace pbkv
