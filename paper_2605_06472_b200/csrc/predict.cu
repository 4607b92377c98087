// Stage 1 on sm_100a: the batched multi-step predictor forward of
// PAPER.md:1040-1066 (no reference code exists).
//
//   H1 = ReLU([H0 | A H0] W1^T), H2 = ReLU([H1 | A H1] W2^T)
//   h_cur = H2[v_t];  a_i = softmax_i<t((Wq h_cur)^T H2[v_i] / sqrt(d))
//   h_path = sum_i a_i H2[v_i]
//   h_txt = ReLU(W_t x)
//   logits = W_m2 ReLU(W_m1 [h_cur | h_path | h_txt] + b1) + b2
//   P_w[k] = softmax(logits[k*V1 .. k*V1+V1)), END a regular class
//
// Kernels:
//   graph_kernel   once per weight load: H2 and the per-agent attention table
//                  QK[u][v] = (Wq H2[u]) . H2[v] / sqrt(d) (the query depends on
//                  the current agent only), fp32, one CTA
//   txt_gemm_kernel  h_txt pre-activation = x W_t^T: the one dense contraction
//                  (M = workflows, N = d, K = H).  TMA (128B swizzle) feeds a
//                  4-stage shared-memory ring (kStages); one elected thread issues
//                  tcgen05.mma kind::f16 (bf16 in, fp32 accumulate in TMEM);
//                  four epilogue warps drain TMEM with tcgen05.ld.  Split-K
//                  over blockIdx.y so every SM streams x (the GEMM is HBM-bound
//                  on x: ~1 flop per byte, SURVEY.md §7 hard part 10).
//   head_kernel    per 16 workflows: split-K sum + ReLU, attention over the
//                  prefix, the two-layer MLP (weights read once per CTA),
//                  per-step softmax, FP64 renormalisation, written straight
//                  into the forecast staging rows that forecast_prepare turns
//                  into P / survival / gs (score.cu).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstring>
#include <vector>

#include <cuda_bf16.h>

#include "common.cuh"

namespace pbkv {

namespace {

constexpr int BM = 128;  // workflows per MMA tile (UMMA M)
constexpr int BN = 64;   // = d (UMMA N)
constexpr int BK = 64;   // bf16 elements per 128-byte swizzle row
constexpr int kStages = 4;  // 96 KB ring: two CTAs per SM
constexpr int kABytes = BM * BK * 2;
constexpr int kBBytes = BN * BK * 2;
constexpr int kGemmThreads = 128;
constexpr int kHeadWf = 16;       // workflows per head CTA
constexpr int kRW = kHeadWf / 8;  // workflow rows per thread in the MLP tiles (8 thread rows)
constexpr int kHeadThreads = 256;
constexpr int kChunk1 = 32;  // W_m1^T rows staged in shared memory per pass
constexpr int kChunk2 = 16;  // W_m2^T rows staged per pass

struct GemmSmem {
    unsigned char a[kStages][kABytes];  // 1024-aligned (SW128 atoms)
    unsigned char b[kStages][kBBytes];
    unsigned long long full[kStages], empty[kStages], done;
    unsigned int tmem_base;
};

__device__ __forceinline__ unsigned int smem_u32(const void* p) {
    return static_cast<unsigned int>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned int bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned int parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, unsigned long long* bar, int c0,
                                            int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// K-major, 128-byte-swizzled operand tile (rows of 64 bf16 = 128 B, 8-row
// atoms of 1024 B): start >> 4, LBO 1 (unused when swizzled), SBO 1024 B,
// descriptor version 1 (sm_100), layout SWIZZLE_128B (2).
__device__ __forceinline__ unsigned long long umma_desc_sw128(const void* tile) {
    const unsigned long long start = (smem_u32(tile) & 0x3FFFFu) >> 4;
    return start | (1ull << 16) | (static_cast<unsigned long long>(1024 >> 4) << 32) | (1ull << 46) |
           (2ull << 61);
}

// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, N = BN, M = BM
constexpr unsigned int kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<unsigned int>(BN >> 3) << 17) |
                                (static_cast<unsigned int>(BM >> 4) << 24);

__device__ __forceinline__ void umma_bf16(unsigned int tmem_d, unsigned long long a, unsigned long long b,
                                          unsigned int accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(unsigned long long* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// h_txt partial sums: part[split][row][0..BN) = x[row, kslice] . W_t[:, kslice]
__global__ void __launch_bounds__(kGemmThreads, 2)
    txt_gemm_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmw, float* part,
                    int n_rows, int k_blocks, int kb_per_split) {
    extern __shared__ unsigned char smem_raw[];
    GemmSmem& sm = *reinterpret_cast<GemmSmem*>(
        (reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~static_cast<std::uintptr_t>(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.x * BM;
    const int kb0 = blockIdx.y * kb_per_split;
    const int nk = max(0, min(k_blocks, kb0 + kb_per_split) - kb0);

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], 1);
        }
        mbar_init(&sm.done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<unsigned long long>(&tmx)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<unsigned long long>(&tmw)) : "memory");
    }
    if (warp == 1) {  // TMEM: 128 lanes x 64 fp32 columns for the accumulator
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&sm.tmem_base))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned int tmem = sm.tmem_base;

    if (warp == 0 && lane == 0) {
        // ---- TMA producer ----
        for (int i = 0; i < nk; ++i) {
            const int s = i % kStages;
            if (i >= kStages) mbar_wait(&sm.empty[s], static_cast<unsigned int>((i / kStages - 1) & 1));
            mbar_expect_tx(&sm.full[s], kABytes + kBBytes);
            const int kc = (kb0 + i) * BK;
            tma_load_2d(sm.a[s], &tmx, &sm.full[s], kc, m0);
            tma_load_2d(sm.b[s], &tmw, &sm.full[s], kc, 0);
        }
    } else if (warp == 1 && lane == 0) {
        // ---- MMA issuer: 4 x (128x64x16) per k-block ----
        for (int i = 0; i < nk; ++i) {
            const int s = i % kStages;
            mbar_wait(&sm.full[s], static_cast<unsigned int>((i / kStages) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const unsigned long long da = umma_desc_sw128(sm.a[s]);
            const unsigned long long db = umma_desc_sw128(sm.b[s]);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)  // +32 bytes along K inside the swizzle row
                umma_bf16(tmem, da + 2ull * k, db + 2ull * k, (i > 0 || k > 0) ? 1u : 0u);
            umma_commit(&sm.empty[s]);
        }
        umma_commit(&sm.done);
    }
    __syncwarp();

    // ---- epilogue: TMEM lane r (warp 32w + lane) = output row m0 + r ----
    if (nk > 0) mbar_wait(&sm.done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int row = m0 + warp * 32 + lane;
    float* dst = part + (static_cast<std::size_t>(blockIdx.y) * n_rows + row) * BN;
#pragma unroll
    for (int c0 = 0; c0 < BN; c0 += 16) {
        unsigned int v[16];
        const unsigned int taddr = tmem + (static_cast<unsigned int>(warp * 32) << 16) + static_cast<unsigned int>(c0);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (row < n_rows) {
            float4* d4 = reinterpret_cast<float4*>(dst + c0);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                float4 f;
                f.x = nk > 0 ? __uint_as_float(v[4 * j + 0]) : 0.f;
                f.y = nk > 0 ? __uint_as_float(v[4 * j + 1]) : 0.f;
                f.z = nk > 0 ? __uint_as_float(v[4 * j + 2]) : 0.f;
                f.w = nk > 0 ? __uint_as_float(v[4 * j + 3]) : 0.f;
                d4[j] = f;
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem) : "memory");
}

// H2 and the attention table (fp32), one CTA of 256 threads.
__global__ void graph_kernel(const float* E, const float* Atr, const float* W1, const float* W2, const float* Wq,
                             int A, int d, float* H2, float* QK) {
    extern __shared__ float g_sm[];
    float* H = g_sm;          // [A][d]
    float* AH = H + A * d;    // [A][d]
    float* Hn = AH + A * d;   // [A][d]
    for (int i = threadIdx.x; i < A * d; i += blockDim.x) H[i] = E[i];
    __syncthreads();
    for (int layer = 0; layer < 2; ++layer) {
        const float* W = layer == 0 ? W1 : W2;
        for (int i = threadIdx.x; i < A * d; i += blockDim.x) {  // AH = A . H
            const int u = i / d, j = i % d;
            float s = 0.f;
            for (int v = 0; v < A; ++v) s = fmaf(Atr[u * A + v], H[v * d + j], s);
            AH[i] = s;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < A * d; i += blockDim.x) {  // ReLU([H | AH] W^T)
            const int u = i / d, j = i % d;
            float s = 0.f;
            for (int c = 0; c < d; ++c) s = fmaf(H[u * d + c], W[j * 2 * d + c], s);
            for (int c = 0; c < d; ++c) s = fmaf(AH[u * d + c], W[j * 2 * d + d + c], s);
            Hn[i] = fmaxf(s, 0.f);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < A * d; i += blockDim.x) H[i] = Hn[i];
        __syncthreads();
    }
    for (int i = threadIdx.x; i < A * d; i += blockDim.x) {  // AH <- q = Wq h (per agent)
        const int u = i / d, j = i % d;
        float s = 0.f;
        for (int c = 0; c < d; ++c) s = fmaf(Wq[j * d + c], H[u * d + c], s);
        AH[i] = s;
        H2[i] = H[i];
    }
    __syncthreads();
    const float inv = rsqrtf(static_cast<float>(d));
    for (int i = threadIdx.x; i < A * A; i += blockDim.x) {
        const int u = i / A, v = i % A;
        float s = 0.f;
        for (int c = 0; c < d; ++c) s = fmaf(AH[u * d + c], H[v * d + c], s);
        QK[i] = s * inv;
    }
}

__device__ __forceinline__ int head_wchunk_floats_dev(int h1, int KV) {
    return kChunk1 * h1 > kChunk2 * KV ? kChunk1 * h1 : kChunk2 * KV;
}

struct HeadArgs {
    const float* part;  // [splits][n][d]
    int splits;
    const float* H2;    // [A][d]
    const float* QK;    // [A][A]
    const float* Wm1T;  // [3d][h1]
    const float* b1;    // [h1]
    const float* Wm2T;  // [h1][KV]
    const float* b2;    // [KV]
    const int* pre_off; // [n+1]
    const int* pre;     // agents
    const long long* slots;  // [n] forecast slot of each workflow
    int n, A, d, h1, Kp, V1;
    // resident forecast store (score.cu layout): P[slot][K][V1], gs[slot][K], fstate[slot]
    double* P;
    double* Pg;
    double* gs;
    std::uint8_t* fstate;
    int K;               // scoring horizon of the context
    double gamma;
    double* probs_out;   // [n][Kp][V1] or null
};

// Shared memory: H2 [A][d] | QK [A][A] | z [32][3d] | hidden [32][h1] |
// logits [32][KV] (floats) | p [32][Kp][V1] (doubles, 8-aligned).
std::size_t head_wchunk_floats(int h1, int KV) {
    return static_cast<std::size_t>(kChunk1 * h1 > kChunk2 * KV ? kChunk1 * h1 : kChunk2 * KV);
}

// Shared memory: H2 [A][d] | QK [A][A] | z [32][3d] | hidden [32][h1] |
// logits [32][KV] | weight chunk (floats, each 16-aligned) | p [32][KV] (doubles).
std::size_t head_smem_bytes(int A, int d, int h1, int KV) {
    auto al4 = [](std::size_t f) { return (f + 3) & ~static_cast<std::size_t>(3); };
    std::size_t f = al4(static_cast<std::size_t>(A) * d) + al4(static_cast<std::size_t>(A) * A) +
                    al4(static_cast<std::size_t>(kHeadWf) * 3 * d) + al4(static_cast<std::size_t>(kHeadWf) * h1) +
                    al4(static_cast<std::size_t>(kHeadWf) * KV) + al4(head_wchunk_floats(h1, KV));
    return f * sizeof(float) + static_cast<std::size_t>(kHeadWf) * KV * sizeof(double);
}

__global__ void __launch_bounds__(kHeadThreads) head_kernel(HeadArgs a) {
    extern __shared__ __align__(16) float h_sm[];
    const int d = a.d, Z = 3 * d, KV = a.Kp * a.V1, h1 = a.h1;
    auto al4 = [](int f) { return (f + 3) & ~3; };
    float* sH2 = h_sm;
    float* sQK = sH2 + al4(a.A * d);
    float* z = sQK + al4(a.A * a.A);
    float* hid = z + al4(kHeadWf * Z);
    float* lg = hid + al4(kHeadWf * h1);
    float* wch = lg + al4(kHeadWf * KV);
    double* pp = reinterpret_cast<double*>(wch + al4(static_cast<int>(head_wchunk_floats_dev(h1, KV))));
    const int w0 = blockIdx.x * kHeadWf;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    for (int i = threadIdx.x; i < a.A * d; i += kHeadThreads) sH2[i] = a.H2[i];
    for (int i = threadIdx.x; i < a.A * a.A; i += kHeadThreads) sQK[i] = a.QK[i];
    __syncthreads();

    // ---- z = [h_cur | h_path | h_txt]: one warp per workflow ----
    for (int i = warp; i < kHeadWf; i += kHeadThreads / 32) {
        const int w = w0 + i;
        float* zi = z + i * Z;
        if (w >= a.n) {
            for (int j = lane; j < Z; j += 32) zi[j] = 0.f;
            continue;
        }
        const int p0 = a.pre_off[w], p1 = a.pre_off[w + 1];
        const int t = p1 - p0;  // >= 1 (validated on the host)
        const int cur = a.pre[p1 - 1];
        for (int j = lane; j < d; j += 32) zi[j] = sH2[cur * d + j];
        // attention over the strictly earlier prefix positions (i < t); lane
        // q owns positions q, q+32, ...
        float mx = -INFINITY;
        for (int q = lane; q < t - 1; q += 32) mx = fmaxf(mx, sQK[cur * a.A + a.pre[p0 + q]]);
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        float den = 0.f;
        for (int q = lane; q < t - 1; q += 32) den += expf(sQK[cur * a.A + a.pre[p0 + q]] - mx);
        for (int o = 16; o; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
        float acc0 = 0.f, acc1 = 0.f;  // dims lane and lane + 32 (d = 64)
        for (int q0 = 0; q0 < t - 1; q0 += 32) {
            const int q = q0 + lane;
            int v = 0;
            float al = 0.f;
            if (q < t - 1) {
                v = a.pre[p0 + q];
                al = expf(sQK[cur * a.A + v] - mx) / den;
            }
            const int m = min(32, t - 1 - q0);
            for (int u = 0; u < m; ++u) {
                const float au = __shfl_sync(0xffffffffu, al, u);
                const int vu = __shfl_sync(0xffffffffu, v, u);
                acc0 = fmaf(au, sH2[vu * d + lane], acc0);
                acc1 = fmaf(au, sH2[vu * d + lane + 32], acc1);
            }
        }
        zi[d + lane] = acc0;
        zi[d + lane + 32] = acc1;
        for (int j = lane; j < d; j += 32) {  // split-K partials, fixed order (deterministic)
            float s4[4] = {0.f, 0.f, 0.f, 0.f};
            const float* pj = a.part + static_cast<std::size_t>(w) * d + j;
            const std::size_t stride = static_cast<std::size_t>(a.n) * d;
            int sp = 0;
            for (; sp + 4 <= a.splits; sp += 4)
#pragma unroll
                for (int u = 0; u < 4; ++u) s4[u] += __ldcg(pj + (sp + u) * stride);
            for (; sp < a.splits; ++sp) s4[0] += __ldcg(pj + sp * stride);
            zi[2 * d + j] = fmaxf((s4[0] + s4[1]) + (s4[2] + s4[3]), 0.f);
        }
    }
    __syncthreads();

    // ---- hidden = ReLU(W_m1 z + b1): thread (ty, tx) -> kRW workflows x 4 neurons per pass ----
    const int ty = threadIdx.x >> 5, tx = threadIdx.x & 31;  // ty: 8 groups of kRW workflows
    for (int j0 = tx * 4; j0 - tx * 4 < h1; j0 += 128) {
        float acc[kRW][4] = {};
        for (int c0 = 0; c0 < Z; c0 += kChunk1) {
            const int rows = min(kChunk1, Z - c0);
            __syncthreads();  // previous chunk consumed
            for (int e = threadIdx.x * 4; e < rows * h1; e += kHeadThreads * 4) {
                if (e + 4 <= rows * h1 && (h1 & 3) == 0)
                    *reinterpret_cast<float4*>(wch + e) =
                        __ldg(reinterpret_cast<const float4*>(a.Wm1T + static_cast<std::size_t>(c0) * h1 + e));
                else
                    for (int q = 0; q < 4 && e + q < rows * h1; ++q) wch[e + q] = __ldg(a.Wm1T + static_cast<std::size_t>(c0) * h1 + e + q);
            }
            __syncthreads();
            if (j0 < h1) {
#pragma unroll 4
                for (int c = 0; c < rows; ++c) {
                    float wv[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) wv[q] = j0 + q < h1 ? wch[c * h1 + j0 + q] : 0.f;
#pragma unroll
                    for (int i = 0; i < kRW; ++i) {
                        const float zv = z[(ty * kRW + i) * Z + c0 + c];
#pragma unroll
                        for (int q = 0; q < 4; ++q) acc[i][q] = fmaf(wv[q], zv, acc[i][q]);
                    }
                }
            }
        }
        if (j0 < h1) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (j0 + q >= h1) break;
                const float bj = a.b1[j0 + q];
#pragma unroll
                for (int i = 0; i < kRW; ++i) hid[(ty * kRW + i) * h1 + j0 + q] = fmaxf(acc[i][q] + bj, 0.f);
            }
        }
    }
    __syncthreads();

    // ---- logits = W_m2 hidden + b2: thread -> kRW workflows x outputs tx, tx+32, ... ----
    for (int o0 = 0; o0 < KV; o0 += 32 * 5) {
        float acc[kRW][5] = {};
        for (int c0 = 0; c0 < h1; c0 += kChunk2) {
            const int rows = min(kChunk2, h1 - c0);
            __syncthreads();
            for (int e = threadIdx.x; e < rows * KV; e += kHeadThreads)
                wch[e] = __ldg(a.Wm2T + static_cast<std::size_t>(c0) * KV + e);
            __syncthreads();
#pragma unroll 4
            for (int c = 0; c < rows; ++c) {
                float wv[5];
#pragma unroll
                for (int m = 0; m < 5; ++m) {
                    const int o = o0 + tx + 32 * m;
                    wv[m] = o < KV ? wch[c * KV + o] : 0.f;
                }
#pragma unroll
                for (int i = 0; i < kRW; ++i) {
                    const float hv = hid[(ty * kRW + i) * h1 + c0 + c];
#pragma unroll
                    for (int m = 0; m < 5; ++m) acc[i][m] = fmaf(wv[m], hv, acc[i][m]);
                }
            }
        }
#pragma unroll
        for (int m = 0; m < 5; ++m) {
            const int o = o0 + tx + 32 * m;
            if (o >= KV) break;
            const float bo = a.b2[o];
#pragma unroll
            for (int i = 0; i < kRW; ++i) lg[(ty * kRW + i) * KV + o] = acc[i][m] + bo;
        }
    }
    __syncthreads();

    // ---- per-step softmax (END a regular class), FP64 renormalisation ----
    for (int task = threadIdx.x; task < kHeadWf * a.Kp; task += kHeadThreads) {
        const int i = task / a.Kp, k = task % a.Kp;
        const float* l = lg + i * KV + k * a.V1;
        double* out = pp + i * KV + k * a.V1;
        float mx = -INFINITY;
        for (int v = 0; v < a.V1; ++v) mx = fmaxf(mx, l[v]);
        float s = 0.f;
        for (int v = 0; v < a.V1; ++v) s += expf(l[v] - mx);
        double tot = 0.0;
        for (int v = 0; v < a.V1; ++v) {
            const double p = static_cast<double>(expf(l[v] - mx) / s);
            out[v] = p;
            tot += p;
        }
        for (int v = 0; v < a.V1; ++v) out[v] = out[v] / tot;
    }
    __syncthreads();

    // ---- store as resident forecasts (the Forecast ctor + gs table of
    //      forecast_prepare_kernel, score.cu: survival s_k = prod_{j<k}(1 - p_end(j))
    //      clamped at 0, gs[k] = gamma^k * s_k by repeated multiplication) ----
    const int nw = min(kHeadWf, a.n - w0);
    const int KK = a.K < a.Kp ? a.K : a.Kp;
    for (int idx = threadIdx.x; idx < nw * a.K * a.V1; idx += kHeadThreads) {
        const int i = idx / (a.K * a.V1), r = idx % (a.K * a.V1);
        const int k = r / a.V1, v = r % a.V1;  // agent-major store: P[slot][v][k]
        a.P[static_cast<std::size_t>(a.slots[w0 + i]) * a.K * a.V1 + static_cast<std::size_t>(v) * a.K + k] =
            k < KK ? pp[i * KV + r] : CUDART_NAN;  // horizon < K: unusable rows (see capi.cu poison_slot)
    }
    if (a.probs_out)
        for (int idx = threadIdx.x; idx < nw * KV; idx += kHeadThreads)
            a.probs_out[static_cast<std::size_t>(w0) * KV + idx] = pp[idx];
    if (threadIdx.x < nw) {
        const int i = threadIdx.x;
        const long long slot = a.slots[w0 + i];
        double surv = 1.0, gk = 1.0;
        for (int k = 0; k < a.K; ++k) {
            double g = 0.0;
            if (k < KK) {
                g = __dmul_rn(gk, surv);
                surv = __dmul_rn(surv, __dsub_rn(1.0, pp[i * KV + k * a.V1 + a.V1 - 1]));
                if (surv < 0.0) surv = 0.0;
            }
            a.gs[static_cast<std::size_t>(slot) * a.K + k] = g;
            gk = __dmul_rn(gk, a.gamma);
        }
        a.fstate[slot] = a.Kp >= a.K ? 1 : 2;
    }
    __syncthreads();
    // one-agent Eq. 2 terms gs[k] * (0.0 + P[a][k]) (see forecast_prepare_kernel)
    for (int idx = threadIdx.x; idx < nw * a.K * a.V1; idx += kHeadThreads) {
        const int i = idx / (a.K * a.V1), r = idx % (a.K * a.V1);
        const int v = r / a.K, k = r % a.K;  // agent-major position
        const std::size_t base = static_cast<std::size_t>(a.slots[w0 + i]) * a.K * a.V1;
        const double g = a.gs[static_cast<std::size_t>(a.slots[w0 + i]) * a.K + k];
        a.Pg[base + r] = k < KK ? __dmul_rn(g, __dadd_rn(0.0, pp[i * KV + k * a.V1 + v])) : CUDART_NAN;
    }
}

// ---------------------------------------------------------------------------
// head_mma_kernel: the MLP of the head on tcgen05, one
// CTA per 128 workflows (= one UMMA M tile, TMEM lane = workflow row).
//
// Precision: each fp32 operand is split into bf16 hi + lo (x = hi + lo up to
// 2^-16 relative) and every layer is the three products hi.hi + hi.lo + lo.hi
// accumulated in fp32 in TMEM ("bf16x3"): the error is that of an fp32 dot
// product, not of a bf16 one, so the tolerance of tests/test_predictor.py
// holds unchanged.  Operands sit in shared memory as K-major 128-byte-swizzled
// atoms (64 bf16 columns x rows, 8-row / 1024-byte groups); the weights arrive
// pre-split and pre-swizzled from the host (predictor_load).
//
// Shared memory: region A (96 KB) = z hi/lo (3 + 3 atoms), later hidden hi/lo
// (2 + 2 atoms); region W (96 KB) = W_m1 hi/lo (3 + 3 atoms of h1 rows), later
// W_m2 hi/lo (2 + 2 atoms of N2 rows, loaded while the layer-1 epilogue runs);
// after layer 2 both regions hold the logits [128][N2 + 1] fp32 for the
// softmax epilogue (the per-step column offsets k*V1 are not 16-aligned, so
// the rows go through shared memory rather than per-step tcgen05.ld).
constexpr int kMT = 128;          // workflows per CTA
constexpr int kMmaThreads = 512;  // 16 warps
constexpr int kMmaH1 = 128;       // hidden width of the MMA head
constexpr int kMmaMaxN2 = 192;    // 4 W_m2 atoms of N2 rows fit region W
constexpr std::size_t kAtomRows = 128;  // bytes per swizzled row
constexpr std::size_t kRegion = 6 * kMT * kAtomRows;  // 96 KB

__host__ __device__ constexpr std::size_t sw128_off(int r, int c) {  // (row, col) in a 64-column atom
    return static_cast<std::size_t>(r) * 128 + static_cast<std::size_t>(((c >> 3) ^ (r & 7)) << 4) +
           static_cast<std::size_t>((c & 7) * 2);
}

__device__ __forceinline__ unsigned int idesc_bf16_n(int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<unsigned int>(n >> 3) << 17) |
           (static_cast<unsigned int>(kMT >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16_n(unsigned int tmem_d, unsigned long long a, unsigned long long b,
                                            unsigned int idesc, unsigned int accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_ld16(unsigned int taddr, float* v) {
    unsigned int u[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]),
          "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(u[i]);
}

// 1-D bulk copy global -> shared (async proxy), completion on `bar` (tx bytes)
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned int bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(reinterpret_cast<unsigned long long>(src)), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// bf16 hi/lo split of x into two swizzled atoms sets (hi at `hi`, lo at `lo`)
__device__ __forceinline__ void put_split(unsigned char* hi, unsigned char* lo, std::size_t atom_bytes, int r, int col,
                                          float x) {
    const __nv_bfloat16 h = __float2bfloat16_rn(x);
    const __nv_bfloat16 l = __float2bfloat16_rn(x - __bfloat162float(h));
    const std::size_t o = (col >> 6) * atom_bytes + sw128_off(r, col & 63);
    *reinterpret_cast<__nv_bfloat16*>(hi + o) = h;
    *reinterpret_cast<__nv_bfloat16*>(lo + o) = l;
}

// layer: D[128 x N] (+)= A . B^T over `atoms` 64-column K atoms, bf16x3
__device__ __forceinline__ void issue_layer(unsigned int tmem_d, const unsigned char* a_hi, const unsigned char* a_lo,
                                            std::size_t a_atom, const unsigned char* b_hi, const unsigned char* b_lo,
                                            std::size_t b_atom, int atoms, unsigned int idesc) {
    unsigned int acc = 0;
    for (int kb = 0; kb < atoms; ++kb)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const unsigned long long ah = umma_desc_sw128(a_hi + kb * a_atom) + 2ull * k;
            const unsigned long long al = umma_desc_sw128(a_lo + kb * a_atom) + 2ull * k;
            const unsigned long long bh = umma_desc_sw128(b_hi + kb * b_atom) + 2ull * k;
            const unsigned long long bl = umma_desc_sw128(b_lo + kb * b_atom) + 2ull * k;
            umma_bf16_n(tmem_d, ah, bh, idesc, acc);
            acc = 1;
            umma_bf16_n(tmem_d, ah, bl, idesc, 1);
            umma_bf16_n(tmem_d, al, bh, idesc, 1);
        }
}

// PBKV_HEAD_PROF: block 0 prints the cycles of each phase (tools/head_prof.sh)
#ifdef PBKV_HEAD_PROF
#define HEAD_STAMP(n) \
    if (blockIdx.x == 0 && threadIdx.x == 0) tprof[n] = clock64();
#else
#define HEAD_STAMP(n)
#endif

__global__ void __launch_bounds__(kMmaThreads, 1)
    head_mma_kernel(HeadArgs a, const unsigned char* __restrict__ w1s, const unsigned char* __restrict__ w2s, int N2,
                    int rows) {
#ifdef PBKV_HEAD_PROF
    long long tprof[14];
#endif
    HEAD_STAMP(0);
    constexpr int D = 64, H1 = kMmaH1;
    constexpr std::size_t kAtomA = kMT * kAtomRows;   // 16 KB
    constexpr std::size_t kAtomW1 = H1 * kAtomRows;   // 16 KB
    const std::size_t atomW2 = static_cast<std::size_t>(N2) * kAtomRows;
    extern __shared__ unsigned char hm_raw[];
    unsigned char* rA =
        reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(hm_raw) + 1023) & ~std::uintptr_t(1023));
    unsigned char* rW = rA + kRegion;
    unsigned int* sCnt = reinterpret_cast<unsigned int*>(rW + kRegion);  // [128][32]: 16-bit agent counts, 2 per word
    int* sOff = reinterpret_cast<int*>(sCnt + kMT * 32);                    // [129] prefix offsets of the rows
    int* sCur = sOff + kMT + 1;                                             // [128] current agent
    float* sH2 = reinterpret_cast<float*>(sCur + kMT + 1);                  // [A <= 32][64]
    float* sQK = sH2 + 32 * D;                                              // [A][A]
    long long* sSlot = reinterpret_cast<long long*>(sQK + 32 * 32);         // [128] forecast slots
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(sSlot + kMT);
    unsigned int* tmem_sh = reinterpret_cast<unsigned int*>(bar + 4);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int w0 = blockIdx.x * rows;  // rows (32/64/96/128) of the M = 128 tile carry workflows
    const int V1 = a.V1, KV = a.Kp * V1;

    if (threadIdx.x == 0) {
#pragma unroll
        for (int b = 0; b < 4; ++b) mbar_init(&bar[b], 1);  // MMA1, MMA2 done; W_m1, W_m2 landed
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // W_m1 hi/lo (pre-swizzled) by the bulk-copy engine, overlapping the z rows
        mbar_expect_tx(&bar[2], static_cast<unsigned int>(6 * kAtomW1));
        for (int b = 0; b < 6; ++b)
            bulk_load(rW + b * kAtomW1, w1s + b * kAtomW1, static_cast<unsigned int>(kAtomW1), &bar[2]);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_sh))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    const int nw = min(rows, a.n - w0);
    for (int i = threadIdx.x; i <= nw; i += kMmaThreads) sOff[i] = a.pre_off[w0 + i];
    for (int i = threadIdx.x; i < nw; i += kMmaThreads) sSlot[i] = a.slots[w0 + i];
    for (int i = threadIdx.x; i < a.A * D; i += kMmaThreads) sH2[i] = __ldg(a.H2 + i);
    for (int i = threadIdx.x; i < a.A * a.A; i += kMmaThreads) sQK[i] = __ldg(a.QK + i);
    for (int i = threadIdx.x; i < rows * 32; i += kMmaThreads) sCnt[i] = 0u;
    __syncthreads();
    HEAD_STAMP(1);

    // ---- z = [h_cur | h_path | h_txt].  The attention logit of a prefix
    //      position depends on its agent only (the query is the current
    //      agent's): h_path = sum_v n_v e_v H2[v] / sum_v n_v e_v over the
    //      agents' counts n_v in the prefix. ----
    unsigned char* zlo = rA + 3 * kAtomA;
    {  // h_txt = ReLU(sum of the split-K partials, fixed order), every thread, coalesced
        const std::size_t stride = static_cast<std::size_t>(a.n) * D;
        // agent histogram over the rows' (contiguous) prefixes; the last position is the current
        // agent.  Four positions in flight per thread.
        const int q0 = sOff[0], q1 = sOff[nw];
        for (int pb = q0 + threadIdx.x; pb < q1; pb += 4 * kMmaThreads) {
            int vv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) vv[u] = pb + u * kMmaThreads < q1 ? __ldg(a.pre + pb + u * kMmaThreads) : 0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int p = pb + u * kMmaThreads;
                if (p >= q1) break;
                int lo = 0, hi = nw - 1;  // row: largest i with sOff[i] <= p
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (sOff[mid] <= p) lo = mid; else hi = mid - 1;
                }
                const int v = vv[u];
                if (p == sOff[lo + 1] - 1)
                    sCur[lo] = v;
                else
                    atomicAdd(&sCnt[lo * 32 + (v >> 1)], 1u << ((v & 1) * 16));
            }
        }
        HEAD_STAMP(10);
        const float* pbase = a.part + static_cast<std::size_t>(w0) * D;
        const int ne = nw * D;
        for (int e0 = threadIdx.x; e0 < rows * D; e0 += 4 * kMmaThreads) {  // 4 elements in flight per thread
            float z[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
            for (int sp = 0; sp < a.splits; ++sp)
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int e = e0 + u * kMmaThreads;
                    if (e < ne) z[u] += __ldcg(pbase + sp * stride + e);
                }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e = e0 + u * kMmaThreads;
                if (e < rows * D) put_split(rA, zlo, kAtomA, e >> 6, 128 + (e & 63), fmaxf(z[u], 0.f));
            }
        }
    }
    HEAD_STAMP(11);
    __syncthreads();
    HEAD_STAMP(12);
    for (int i = warp; i < rows; i += kMmaThreads / 32) {  // h_cur, h_path: one warp per row
        float zc0 = 0.f, zc1 = 0.f, zp0 = 0.f, zp1 = 0.f;  // dims lane, lane + 32
        if (i < nw) {
            const int cur = sCur[i];
            zc0 = sH2[cur * D + lane];
            zc1 = sH2[cur * D + lane + 32];
            const unsigned int wc = sCnt[i * 32 + (lane >> 1)];  // agents lane, lane + 32
            const unsigned int wc1 = sCnt[i * 32 + 16 + (lane >> 1)];
            const int c0 = lane < a.A ? static_cast<int>((wc >> ((lane & 1) * 16)) & 0xFFFFu) : 0;
            const int c1 = lane + 32 < a.A ? static_cast<int>((wc1 >> ((lane & 1) * 16)) & 0xFFFFu) : 0;
            const float l0 = c0 ? sQK[cur * a.A + lane] : -INFINITY;
            const float l1 = c1 ? sQK[cur * a.A + (lane + 32)] : -INFINITY;
            float mx = fmaxf(l0, l1);
            for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            const float e0 = c0 ? static_cast<float>(c0) * expf(l0 - mx) : 0.f;
            const float e1 = c1 ? static_cast<float>(c1) * expf(l1 - mx) : 0.f;
            float den = e0 + e1;
            for (int o = 16; o; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
            const float a0 = den > 0.f ? e0 / den : 0.f, a1 = den > 0.f ? e1 / den : 0.f;
            for (int v = 0; v < a.A; ++v) {
                const float av = __shfl_sync(0xffffffffu, v < 32 ? a0 : a1, v & 31);
                zp0 = fmaf(av, sH2[v * D + lane], zp0);
                zp1 = fmaf(av, sH2[v * D + lane + 32], zp1);
            }
        }
        put_split(rA, zlo, kAtomA, i, lane, zc0);
        put_split(rA, zlo, kAtomA, i, lane + 32, zc1);
        put_split(rA, zlo, kAtomA, i, 64 + lane, zp0);
        put_split(rA, zlo, kAtomA, i, 96 + lane, zp1);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy stores -> tensor core
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    HEAD_STAMP(2);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned int tmem = *tmem_sh;

    // ---- layer 1: D1[128 x H1] (TMEM columns 0..H1) ----
    if (threadIdx.x == 0) {
        mbar_wait(&bar[2], 0);
        issue_layer(tmem, rA, rA + 3 * kAtomA, kAtomA, rW, rW + 3 * kAtomW1, kAtomW1, 3, idesc_bf16_n(H1));
        umma_commit(&bar[0]);
    }
    __syncwarp();
    mbar_wait(&bar[0], 0);
    HEAD_STAMP(3);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x == 0) {  // W_m2 hi/lo into region W (layer 1 has consumed W_m1), overlapping epilogue 1
        mbar_expect_tx(&bar[3], static_cast<unsigned int>(4 * atomW2));
        for (int b = 0; b < 4; ++b)
            bulk_load(rW + b * atomW2, w2s + b * atomW2, static_cast<unsigned int>(atomW2), &bar[3]);
    }
    if ((warp & 3) * 32 < rows) {  // epilogue 1: warp -> TMEM lane quarter (warp % 4) x 32 columns (warp / 4)
        const int q = warp & 3, r = q * 32 + lane, c0 = (warp >> 2) * 32;
        float v[32];
        tmem_ld16(tmem + (static_cast<unsigned int>(q * 32) << 16) + static_cast<unsigned int>(c0), v);
        tmem_ld16(tmem + (static_cast<unsigned int>(q * 32) << 16) + static_cast<unsigned int>(c0 + 16), v + 16);
#pragma unroll
        for (int j = 0; j < 32; ++j)
            put_split(rA, rA + 2 * kAtomA, kAtomA, r, c0 + j, fmaxf(v[j] + __ldg(a.b1 + c0 + j), 0.f));
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    HEAD_STAMP(4);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    // ---- layer 2: D2[128 x N2] (TMEM columns H1..H1+N2) ----
    if (threadIdx.x == 0) {
        mbar_wait(&bar[3], 0);
        issue_layer(tmem + H1, rA, rA + 2 * kAtomA, kAtomA, rW, rW + 2 * atomW2, atomW2, 2, idesc_bf16_n(N2));
        umma_commit(&bar[1]);
    }
    __syncwarp();
    mbar_wait(&bar[1], 0);
    HEAD_STAMP(5);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // ---- logits + b2 -> shared [128][N2 + 1] (regions A and W are free now) ----
    float* lg = reinterpret_cast<float*>(rA);
    const int LS = N2 + 1;
    if ((warp & 3) * 32 < rows) {
        const int q = warp & 3, r = q * 32 + lane;
        for (int c0 = (warp >> 2) * 16; c0 < N2; c0 += 64) {
            float v[16];
            tmem_ld16(tmem + (static_cast<unsigned int>(q * 32) << 16) + static_cast<unsigned int>(H1 + c0), v);
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (c0 + j < KV) lg[r * LS + c0 + j] = v[j] + __ldg(a.b2 + c0 + j);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    HEAD_STAMP(6);
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");

    // ---- per-step softmax (END a regular class), FP64 renormalisation: task = (row, step).
    //      q_v = e_v / s (fp32) stays in place; sInv = 1 / sum_v double(q_v); every
    //      store below uses p = double(q_v) * sInv, so P, Pg and probs_out agree bitwise. ----
    const int KK = a.K < a.Kp ? a.K : a.Kp;
    double* sInv = reinterpret_cast<double*>(rA + 100 * 1024);  // [128][Kp] 1 / sum (past the logits)
    double* sGs = sInv + kMT * a.Kp;                             // [128][K]
    for (int task = threadIdx.x; task < nw * a.Kp; task += kMmaThreads) {
        const int i = task / a.Kp, k = task % a.Kp;
        float* l = lg + i * LS + k * V1;
        float mx = -INFINITY;
        for (int v = 0; v < V1; ++v) mx = fmaxf(mx, l[v]);
        float s = 0.f;
        for (int v = 0; v < V1; ++v) {
            const float e = expf(l[v] - mx);
            l[v] = e;
            s += e;
        }
        double tot = 0.0;
        for (int v = 0; v < V1; ++v) {
            const float qv = l[v] / s;
            l[v] = qv;
            tot += static_cast<double>(qv);
        }
        sInv[i * a.Kp + k] = 1.0 / tot;
    }
    __syncthreads();
    HEAD_STAMP(7);
    // ---- survival / gs chain per workflow (forecast_prepare_kernel semantics) ----
    if (threadIdx.x < nw) {
        const int i = threadIdx.x;
        const long long slot = sSlot[i];
        double surv = 1.0, gk = 1.0;
        for (int k = 0; k < a.K; ++k) {
            double g = 0.0;
            if (k < KK) {
                g = __dmul_rn(gk, surv);
                const double pend = static_cast<double>(lg[i * LS + k * V1 + V1 - 1]) * sInv[i * a.Kp + k];
                surv = __dmul_rn(surv, __dsub_rn(1.0, pend));
                if (surv < 0.0) surv = 0.0;
            }
            sGs[i * a.K + k] = g;
            a.gs[static_cast<std::size_t>(slot) * a.K + k] = g;
            gk = __dmul_rn(gk, a.gamma);
        }
        a.fstate[slot] = a.Kp >= a.K ? 1 : 2;
    }
    __syncthreads();
    HEAD_STAMP(8);
    // ---- coalesced stores, one warp per row: P[slot][v][k] and Pg = gs[k] * (0.0 + P)
    //      (NaN beyond the horizon), then probs_out[w][k][v] ----
    const int KV1 = a.K * V1;
    for (int i = warp; i < nw; i += kMmaThreads / 32) {
        const std::size_t base = static_cast<std::size_t>(sSlot[i]) * KV1;
        const float* li = lg + i * LS;
        const double* inv = sInv + i * a.Kp;
        const double* gsi = sGs + i * a.K;
        for (int r = lane; r < KV1; r += 32) {
            const int v = r / a.K, k = r - v * a.K;  // agent-major position
            double p = CUDART_NAN, pg = CUDART_NAN;
            if (k < KK) {
                p = static_cast<double>(li[k * V1 + v]) * inv[k];
                pg = __dmul_rn(gsi[k], __dadd_rn(0.0, p));
            }
            a.P[base + r] = p;
            a.Pg[base + r] = pg;
        }
        if (a.probs_out) {
            double* po = a.probs_out + static_cast<std::size_t>(w0 + i) * KV;
            for (int r = lane; r < KV; r += 32) po[r] = static_cast<double>(li[r]) * inv[r / V1];
        }
    }
    HEAD_STAMP(9);
#ifdef PBKV_HEAD_PROF
    if (blockIdx.x == 0 && threadIdx.x == 0)
        printf("head phases: tables %lld z %lld mma1 %lld epi1 %lld mma2 %lld logits %lld softmax %lld chain %lld store %lld\n",
               tprof[1] - tprof[0], tprof[2] - tprof[1], tprof[3] - tprof[2], tprof[4] - tprof[3], tprof[5] - tprof[4],
               tprof[6] - tprof[5], tprof[7] - tprof[6], tprof[8] - tprof[7], tprof[9] - tprof[8]);
    if (blockIdx.x == 0 && threadIdx.x == 0)
        printf("  z: txt %lld hist %lld sync %lld rows+sync %lld\n", tprof[10] - tprof[1], tprof[11] - tprof[10],
               tprof[12] - tprof[11], tprof[2] - tprof[12]);
#endif
}

std::size_t head_mma_smem() {
    return 1024 + 2 * kRegion + (kMT * 32 + 2 * (kMT + 1) + 32 * 64 + 32 * 32) * 4 + kMT * 8 + 64;
}

// rows x cols fp32 (row-major) -> bf16 hi atoms then lo atoms, K-major 128B-swizzled,
// `rows_pad` rows per atom (zero padding)
std::vector<unsigned char> split_swizzle(const float* src, int rows, int rows_pad, int cols) {
    const int atoms = cols / 64;
    const std::size_t atom = static_cast<std::size_t>(rows_pad) * kAtomRows;
    std::vector<unsigned char> out(2 * atoms * atom, 0);
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) {
            const float x = src[static_cast<std::size_t>(r) * cols + c];
            const __nv_bfloat16 h = __float2bfloat16_rn(x);
            const __nv_bfloat16 l = __float2bfloat16_rn(x - __bfloat162float(h));
            const std::size_t o = (c / 64) * atom + sw128_off(r, c % 64);
            std::memcpy(out.data() + o, &h, 2);
            std::memcpy(out.data() + atoms * atom + o, &l, 2);
        }
    return out;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        PBKV_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) throw ApiError(PBKV_ECUDA, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// row-major [rows][cols] bf16 matrix, box = BK columns x box_rows rows, 128B swizzle
CUtensorMap make_map(const void* base, std::int64_t rows, std::int64_t cols, int box_rows) {
    CUtensorMap m;
    std::memset(&m, 0, sizeof m);
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw ApiError(PBKV_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
    return m;
}

}  // namespace

struct PredictorState {
    pbkv_predictor_cfg cfg{};
    DevBuf<float> H2, QK, Wm1T, b1, Wm2T, b2, part;
    DevBuf<std::uint16_t> Wt;
    DevBuf<int> pre_off, pre;
    DevBuf<std::uint16_t> xbuf;
    DevBuf<unsigned char> w1s, w2s;  // head_mma_kernel operands (bf16 hi/lo, swizzled); empty: fp32 head
    int n2 = 0;
    CUtensorMap map_w{};
    int sms = 148;
};

pbkv_predictor_cfg predictor_cfg(const Context& c) { return c.pred->cfg; }

std::size_t gemm_smem_bytes() { return sizeof(GemmSmem) + 1024; }

void predictor_load(Context& c, const pbkv_predictor_cfg& cfg, const pbkv_predictor_weights& w) {
    auto st = std::make_shared<PredictorState>();
    st->cfg = cfg;
    const int A = cfg.num_agents, d = cfg.dim, h1 = cfg.hidden, H = cfg.text_dim, KV = cfg.horizon * (A + 1);
    cudaStream_t s = c.stream;
    auto up = [&](DevBuf<float>& dst, const float* src, std::size_t n) {
        dst.reserve(n);
        PBKV_CUDA(cudaMemcpyAsync(dst.p, src, n * sizeof(float), cudaMemcpyHostToDevice, s));
    };
    // transposed MLP weights: column reads become coalesced row reads
    std::vector<float> m1t(static_cast<std::size_t>(3 * d) * h1), m2t(static_cast<std::size_t>(h1) * KV);
    for (int j = 0; j < h1; ++j)
        for (int c2 = 0; c2 < 3 * d; ++c2) m1t[static_cast<std::size_t>(c2) * h1 + j] = w.mlp1[static_cast<std::size_t>(j) * 3 * d + c2];
    for (int o = 0; o < KV; ++o)
        for (int c2 = 0; c2 < h1; ++c2) m2t[static_cast<std::size_t>(c2) * KV + o] = w.mlp2[static_cast<std::size_t>(o) * h1 + c2];
    DevBuf<float> E, Atr, W1, W2, Wq;
    up(E, w.embed, static_cast<std::size_t>(A) * d);
    up(Atr, w.transition, static_cast<std::size_t>(A) * A);
    up(W1, w.sage1, static_cast<std::size_t>(d) * 2 * d);
    up(W2, w.sage2, static_cast<std::size_t>(d) * 2 * d);
    up(Wq, w.query, static_cast<std::size_t>(d) * d);
    up(st->Wm1T, m1t.data(), m1t.size());
    up(st->b1, w.mlp1_bias, static_cast<std::size_t>(h1));
    up(st->Wm2T, m2t.data(), m2t.size());
    up(st->b2, w.mlp2_bias, static_cast<std::size_t>(KV));
    // tcgen05 head: d = 64, h1 = 128, K*V1 <= 192 (else the fp32 head_kernel)
    if (d == 64 && h1 == kMmaH1 && KV <= kMmaMaxN2 && A <= 32 && cfg.horizon <= 16 && c.K <= 16 &&
        cfg.max_prefix < 65536) {
        st->n2 = (KV + 15) & ~15;
        const auto b1 = split_swizzle(w.mlp1, h1, h1, 3 * d);
        const auto b2 = split_swizzle(w.mlp2, KV, st->n2, h1);
        st->w1s.reserve(b1.size());
        st->w2s.reserve(b2.size());
        PBKV_CUDA(cudaMemcpyAsync(st->w1s.p, b1.data(), b1.size(), cudaMemcpyHostToDevice, s));
        PBKV_CUDA(cudaMemcpyAsync(st->w2s.p, b2.data(), b2.size(), cudaMemcpyHostToDevice, s));
        PBKV_CUDA(cudaFuncSetAttribute(head_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(head_mma_smem())));
    }
    st->Wt.reserve(static_cast<std::size_t>(d) * H);
    PBKV_CUDA(cudaMemcpyAsync(st->Wt.p, w.text, static_cast<std::size_t>(d) * H * 2, cudaMemcpyHostToDevice, s));
    st->H2.reserve(static_cast<std::size_t>(A) * d);
    st->QK.reserve(static_cast<std::size_t>(A) * A);
    const int gsm = static_cast<int>(3 * A * d * sizeof(float));
    PBKV_CUDA(cudaFuncSetAttribute(graph_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, gsm));
    graph_kernel<<<1, 256, gsm, s>>>(E.p, Atr.p, W1.p, W2.p, Wq.p, A, d, st->H2.p, st->QK.p);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
    st->map_w = make_map(st->Wt.p, d, H, BN);
    PBKV_CUDA(cudaDeviceGetAttribute(&st->sms, cudaDevAttrMultiProcessorCount, c.device));
    PBKV_CUDA(cudaFuncSetAttribute(txt_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(gemm_smem_bytes())));
    PBKV_CUDA(cudaStreamSynchronize(s));  // the temporaries above are freed on return
    c.pred = st;
}

// Forward for n workflows; the forecasts land in the resident store (P, gs,
// fstate) at slots_dev, and in probs_dev ([n][Kp][V1]) when non-null.
void predictor_run(Context& c, std::int64_t n, const int* pre_off_dev, const int* pre_dev, const void* x_dev,
                   const long long* slots_dev, double* probs_dev) {
    PredictorState& st = *c.pred;
    const pbkv_predictor_cfg& cfg = st.cfg;
    const int d = cfg.dim, H = cfg.text_dim, V1 = cfg.num_agents + 1;
    const int k_blocks = H / BK;
    const int m_tiles = static_cast<int>((n + BM - 1) / BM);
    // split K so that ~2 CTAs per SM stream x
    // one wave at 2 CTAs/SM, at least 4 k-blocks (256 columns of x) per split
    int splits = std::max(1, std::min((k_blocks + 3) / 4, (2 * st.sms) / m_tiles));
    const int kbs = (k_blocks + splits - 1) / splits;
    splits = (k_blocks + kbs - 1) / kbs;
    st.part.reserve(static_cast<std::size_t>(splits) * n * d);
    const CUtensorMap map_x = make_map(x_dev, n, H, BM);
    txt_gemm_kernel<<<dim3(m_tiles, splits), kGemmThreads, gemm_smem_bytes(), c.stream>>>(map_x, st.map_w, st.part.p,
                                                                                         static_cast<int>(n), k_blocks,
                                                                                         kbs);
    PBKV_CUDA(cudaGetLastError());
    HeadArgs a;
    a.part = st.part.p;
    a.splits = splits;
    a.H2 = st.H2.p;
    a.QK = st.QK.p;
    a.Wm1T = st.Wm1T.p;
    a.b1 = st.b1.p;
    a.Wm2T = st.Wm2T.p;
    a.b2 = st.b2.p;
    a.pre_off = pre_off_dev;
    a.pre = pre_dev;
    a.slots = slots_dev;
    a.n = static_cast<int>(n);
    a.A = cfg.num_agents;
    a.d = d;
    a.h1 = cfg.hidden;
    a.Kp = cfg.horizon;
    a.V1 = V1;
    a.P = c.P.p;
    a.Pg = c.Pg.p;
    a.gs = c.gs.p;
    a.fstate = c.fstate.p;
    a.K = c.K;
    a.gamma = c.gamma;
    a.probs_out = probs_dev;
    if (st.n2 > 0) {
        // rows per CTA: a multiple of 32 that spreads the batch over all SMs (the
        // MMA is nowhere near the bound; the per-row prefix attention is)
        const std::int64_t per = (n + st.sms - 1) / st.sms;
        const int rows = static_cast<int>(std::min<std::int64_t>(kMT, std::max<std::int64_t>(32, (per + 31) / 32 * 32)));
        head_mma_kernel<<<static_cast<unsigned int>((n + rows - 1) / rows), kMmaThreads,
                          head_mma_smem(), c.stream>>>(a, st.w1s.p, st.w2s.p, st.n2,
                                                                                     rows);
        PBKV_CUDA(cudaGetLastError());
        c.launches += 2;
        return;
    }
    const std::size_t hsm = head_smem_bytes(cfg.num_agents, d, cfg.hidden, cfg.horizon * V1);
    PBKV_CUDA(cudaFuncSetAttribute(head_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(hsm)));
    head_kernel<<<static_cast<unsigned int>((n + kHeadWf - 1) / kHeadWf), kHeadThreads, hsm, c.stream>>>(a);
    PBKV_CUDA(cudaGetLastError());
    c.launches += 2;
}

}  // namespace pbkv
