// peaks.cu -- libsdpeaks.so: in-run microbenchmarks for the roofline
// denominators that MEASURED_PEAKS.json does not carry (it has HBM copy and
// bf16 GEMM only): FP32 FFMA, FP64 DFMA and MUFU (ex2) issue throughput,
// measured on the same GPU, in the same process, right before the bench.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

constexpr int kChains = 8;
constexpr int kIters = 2048;

template <class T>
__global__ void fma_kernel(T* out, T a, T b) {
    T x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = T(threadIdx.x + c);
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
    }
    T s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c];
    if (s == T(-1234.5)) out[threadIdx.x] = s;  // defeat dead-code elimination
}

// packed fp32x2 FMA (FFMA2): two FMAs per instruction
__global__ void ffma2_kernel(float* out, float a, float b) {
    unsigned long long x[kChains];
    const float2 av = make_float2(a, a), bv = make_float2(b, b);
    const unsigned long long A = *reinterpret_cast<const unsigned long long*>(&av);
    const unsigned long long B = *reinterpret_cast<const unsigned long long*>(&bv);
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        const float2 v = make_float2(float(threadIdx.x + c), float(c));
        x[c] = *reinterpret_cast<const unsigned long long*>(&v);
    }
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[c]) : "l"(A), "l"(B));
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        const float2 v = *reinterpret_cast<const float2*>(&x[c]);
        s += v.x + v.y;
    }
    if (s == -1234.5f) out[threadIdx.x] = s;
}

__global__ void ex2_kernel(float* out, float a) {
    float x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = -1e-3f * float(threadIdx.x + c);
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            float y;
            asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[c]));
            x[c] = y * a;
        }
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c];
    if (s == -1234.5f) out[threadIdx.x] = s;
}

template <class F>
double time_ms(F&& launch, int reps) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();  // warm-up
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return double(ms) / reps;
}

}  // namespace

extern "C" {

// FFMA2 (packed fp32x2) rate in flop/s (each FFMA2 = 2 FMA = 4 flops).
int sd_measure_ffma2(double* ffma2_flops) {
    int sms = 0;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
    void* buf = nullptr;
    if (cudaMalloc(&buf, 4096) != cudaSuccess) return -1;
    const int threads = 256, blocks = sms * 8;
    const double work = double(blocks) * threads * kIters * kChains;
    const double ms = time_ms([&] { ffma2_kernel<<<blocks, threads>>>((float*)buf, 0.999f, 1e-3f); }, 10);
    *ffma2_flops = 4.0 * work / (ms * 1e-3);
    cudaFree(buf);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// Selects the device the measurements run on (this library has its own
// CUDA runtime state: it does not see the caller's current device).
int sd_peaks_set_device(int device) { return cudaSetDevice(device) == cudaSuccess ? 0 : -1; }

// Returns 0 on success. Rates in flop/s (FMA = 2 flops) and MUFU ops/s.
int sd_measure_peaks(double* ffma_flops, double* dfma_flops, double* mufu_ops) {
    int sms = 0;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
    void* buf = nullptr;
    if (cudaMalloc(&buf, 4096) != cudaSuccess) return -1;
    const int threads = 256, blocks = sms * 8;
    const double work = double(blocks) * threads * kIters * kChains;
    double ms = time_ms([&] { fma_kernel<float><<<blocks, threads>>>((float*)buf, 0.999f, 1e-3f); }, 10);
    *ffma_flops = 2.0 * work / (ms * 1e-3);
    ms = time_ms([&] { fma_kernel<double><<<blocks, threads>>>((double*)buf, 0.999, 1e-3); }, 5);
    *dfma_flops = 2.0 * work / (ms * 1e-3);
    ms = time_ms([&] { ex2_kernel<<<blocks, threads>>>((float*)buf, 0.999f); }, 10);
    *mufu_ops = work / (ms * 1e-3);
    cudaFree(buf);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // extern "C"
