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
//                  6-stage shared-memory ring; one elected thread issues
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
    const std::size_t hsm = head_smem_bytes(cfg.num_agents, d, cfg.hidden, cfg.horizon * V1);
    PBKV_CUDA(cudaFuncSetAttribute(head_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(hsm)));
    head_kernel<<<static_cast<unsigned int>((n + kHeadWf - 1) / kHeadWf), kHeadThreads, hsm, c.stream>>>(a);
    PBKV_CUDA(cudaGetLastError());
    c.launches += 2;
}

}  // namespace pbkv
