// Microbenchmark: grid-wide barrier variants on B200 (148 co-resident CTAs).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/mb tools/microbench_barrier.cu
#include <cooperative_groups.h>
#include <cstdio>

namespace cg = cooperative_groups;

struct Bar {
    unsigned int count, gen;
};

__device__ __forceinline__ void bar_fence(Bar* b) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned int* gen = &b->gen;
        const unsigned int g = *gen;
        __threadfence();
        const unsigned int arrived = atomicAdd(&b->count, 1u);
        if (arrived == gridDim.x - 1) {
            b->count = 0;
            __threadfence();
            atomicAdd(&b->gen, 1u);
        } else {
            while (*gen == g) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned int atom_add_acqrel(unsigned int* p, unsigned int v) {
    unsigned int r;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory");
    return r;
}
__device__ __forceinline__ void st_release(unsigned int* p, unsigned int v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// arrive with acq_rel atomic, flip with release store, poll with acquire loads
__device__ __forceinline__ void bar_acqrel(Bar* b) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int g = ld_acquire(&b->gen);
        const unsigned int arrived = atom_add_acqrel(&b->count, 1u);
        if (arrived == gridDim.x - 1) {
            b->count = 0;
            st_release(&b->gen, g + 1);
        } else {
            while (ld_acquire(&b->gen) == g) {
            }
        }
    }
    __syncthreads();
}

template <int kVariant>
__global__ void __launch_bounds__(1024, 1) k_bar(Bar* b, int iters, unsigned long long* out) {
    cg::grid_group grid = cg::this_grid();
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (kVariant == 0) grid.sync();
        if (kVariant == 1) bar_fence(b);
        if (kVariant == 2) bar_acqrel(b);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

__global__ void __launch_bounds__(1024, 1) k_bitonic(unsigned long long* g_out, int n) {
    __shared__ unsigned long long key[4096];
    for (int i = threadIdx.x; i < n; i += blockDim.x) key[i] = (i * 2654435761u) & 0xffffffffffull;
    __syncthreads();
    for (int k = 2; k <= n; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const unsigned long long a = key[i], c = key[ixj];
                    if ((a > c) == ((i & k) == 0)) {
                        key[i] = c;
                        key[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    if (threadIdx.x == 0) g_out[0] = key[n - 1];
}

int main() {
    Bar* b;
    unsigned long long* out;
    cudaMalloc(&b, sizeof(Bar));
    cudaMalloc(&out, 64);
    cudaMemset(b, 0, sizeof(Bar));
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int iters = 2000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    void* args[] = {&b, &iters, &out};
    const char* names[] = {"cg grid.sync", "atomic+threadfence", "acq_rel atomics"};
    void* fns[] = {(void*)k_bar<0>, (void*)k_bar<1>, (void*)k_bar<2>};
    for (int v = 0; v < 3; ++v) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            cudaError_t err = cudaLaunchCooperativeKernel(fns[v], dim3(sms), dim3(1024), args, 0, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep) printf("%-22s %s: %.3f us per barrier (grid %d x 1024)\n", names[v], cudaGetErrorString(err),
                            1000.0 * ms / iters, sms);
        }
    }
    for (int n : {1024, 2048, 4096}) {
        cudaEventRecord(e0);
        k_bitonic<<<1, 1024>>>(out, n);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("bitonic one CTA n=%d: %.1f us\n", n, 1000.0 * ms);
    }
    return 0;
}
