// microbenchmark: dependent-chain latency of FP64 ops on the running GPU
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, double a, double b, int n) {
    double x = a;
    unsigned long long u = 3;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __dadd_rn(x, b);
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) x = __dmul_rn(x, b);
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) { u += static_cast<unsigned long long>(x * 1.0000001); x = static_cast<double>(u) * 1e-30 + a; }
    long long t3 = clock64();
    for (int i = 0; i < n; ++i) x = rint(x * 1.5) + b;
    long long t4 = clock64();
    float f = (float)a;
    for (int i = 0; i < n; ++i) f = f * 1.000001f + (float)b;
    long long t5 = clock64();
    out[threadIdx.x] = x + u + f;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; }
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMallocManaged(&c, 64);
    for (int threads : {32, 512}) {
        lat<<<1, threads>>>(o, c, 1.0, 1e-9, 1000);
        cudaDeviceSynchronize();
        printf("threads=%d per-op cycles: dadd %.1f dmul %.1f (f2i+i2f+dmul+dfma) %.1f (dmul+frnd+dadd) %.1f ffma %.1f\n", threads,
               c[0] / 1000.0, c[1] / 1000.0, c[2] / 1000.0, c[3] / 1000.0, c[4] / 1000.0);
    }
}
