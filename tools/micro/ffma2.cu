// Throughput of FFMA (3-register) vs FFMA2 (fma.rn.f32x2) vs FMUL2/FADD2 on one B200.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    unsigned long long d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d)
        : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
          "l"(*reinterpret_cast<unsigned long long*>(&c)));
    return *reinterpret_cast<float2*>(&d);
}
constexpr int kChains = 8, kIters = 4096;
__global__ void k_ffma(float* out, float a, float b) {
    float x[kChains];
    float y = b + threadIdx.x;
    for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x + c;
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(y), "f"(a));
    }
    float s = 0; for (int c = 0; c < kChains; ++c) s += x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2(float* out, float a, float b) {
    float2 x[kChains];
    float2 y = make_float2(b + threadIdx.x, b), aa = make_float2(a, a + 1);
    for (int c = 0; c < kChains; ++c) x[c] = make_float2(threadIdx.x + c, c);
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) x[c] = fma2(x[c], y, aa);
    }
    float s = 0; for (int c = 0; c < kChains; ++c) s += x[c].x + x[c].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// no operand reuse: every FFMA reads three different registers
__global__ void k_ffma_nr(float* out, float a, float b) {
    float x[kChains], y[kChains], z[kChains];
    for (int c = 0; c < kChains; ++c) { x[c] = threadIdx.x + c; y[c] = b + c * 0.001f; z[c] = a + c; }
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(x[c]) : "f"(y[c]), "f"(z[(c + 3) % kChains]));
    }
    float s = 0; for (int c = 0; c < kChains; ++c) s += x[c] + y[c] + z[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2_nr(float* out, float a, float b) {
    float2 x[kChains], y[kChains], z[kChains];
    for (int c = 0; c < kChains; ++c) { x[c] = make_float2(threadIdx.x + c, c); y[c] = make_float2(b + c * 0.001f, b); z[c] = make_float2(a + c, a); }
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) x[c] = fma2(y[c], z[(c + 3) % kChains], x[c]);
    }
    float s = 0; for (int c = 0; c < kChains; ++c) s += x[c].x + x[c].y + y[c].x + z[c].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    float* out; cudaMalloc(&out, 148 * 8 * 1024 * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        for (int k = 0; k < 4; ++k) {
            cudaEventRecord(e0);
            if (k == 0) k_ffma<<<148 * 8, 256>>>(out, 1.0001f, 0.5f);
            else if (k == 1) k_ffma2<<<148 * 8, 256>>>(out, 1.0001f, 0.5f);
            else if (k == 2) k_ffma_nr<<<148 * 8, 256>>>(out, 1.0001f, 0.5f);
            else k_ffma2_nr<<<148 * 8, 256>>>(out, 1.0001f, 0.5f);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double lanes = (double)148 * 8 * 256 * kIters * kChains * (k & 1 ? 2 : 1);
            printf("%s: %.3f ms  %.1f TFLOP/s (fma=2 flop)\n", (const char*[]){"FFMA ", "FFMA2", "FFMA  no-reuse", "FFMA2 no-reuse"}[k], ms, 2 * lanes / ms / 1e9);
        }
    }
    return 0;
}
