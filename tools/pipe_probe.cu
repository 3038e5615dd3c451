// pipe_probe.cu -- issue / pipe throughput of the packed fp32x2 forms used by
// K1 on this GPU: FFMA2, FMUL2, FADD2, scalar FFMA, and mixes with ALU
// selects, as warp instructions per SM per cycle (independent chains, no
// memory). Does FMUL2 / FADD2 run at FFMA2's rate, and does an ALU op
// co-issue for free in the gap of a 2-cycle packed op?
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/pipe_probe.cu -o /tmp/pipe_probe && /tmp/pipe_probe
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;

#define PK(x) "l"(x)

template <int OP>
__global__ void probe(unsigned long long* out, unsigned long long a, unsigned long long b, float fa) {
    unsigned long long x[kChains];
    float y[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        x[c] = (unsigned long long)(threadIdx.x + c) * 0x100000001ull;
        y[c] = float(threadIdx.x + c);
    }
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            if constexpr (OP == 0) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[c]) : PK(a), PK(b));
            if constexpr (OP == 1) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(x[c]) : PK(a));
            if constexpr (OP == 2) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(x[c]) : PK(b));
            if constexpr (OP == 3) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(y[c]) : "f"(fa));
            if constexpr (OP == 4) {  // FFMA2 + an independent ALU select
                asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[c]) : PK(a), PK(b));
                asm volatile("{ .reg .pred p; setp.gt.f32 p, %0, %1; selp.f32 %0, %0, %1, p; }" : "+f"(y[c]) : "f"(fa));
            }
            if constexpr (OP == 5) {  // FFMA2 + FMUL2 alternating
                if (c & 1) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(x[c]) : PK(a));
                else asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[c]) : PK(a), PK(b));
            }
        }
    }
    unsigned long long s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c] + (unsigned long long)__float_as_uint(y[c]);
    if (s == 12345) out[threadIdx.x] = s;
}

template <int OP>
void run(const char* name, int instr_per_chain_step) {
    unsigned long long* out;
    cudaMalloc(&out, 1024 * 8);
    const float2 av = make_float2(0.999f, 0.999f), bv = make_float2(1e-3f, 1e-3f);
    const unsigned long long A = *reinterpret_cast<const unsigned long long*>(&av);
    const unsigned long long B = *reinterpret_cast<const unsigned long long*>(&bv);
    const int blocks = 148 * 8, threads = 256;
    probe<OP><<<blocks, threads>>>(out, A, B, 0.999f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) probe<OP><<<blocks, threads>>>(out, A, B, 0.999f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    int mhz = 0;
    cudaDeviceGetAttribute(&mhz, cudaDevAttrClockRate, 0);
    const double warp_instr = 5.0 * blocks * (threads / 32) * double(kIters) * kChains * instr_per_chain_step;
    const double cycles = ms * 1e-3 * 1965e6;  // SM clock under load (the bench's sampled 1965 MHz)
    printf("%-28s %7.3f ms  %6.3f warp-instr / SM / cycle\n", name, ms / 5, warp_instr / cycles / 148.0);
    cudaFree(out);
}

int main() {
    run<0>("FFMA2", 1);
    run<1>("FMUL2", 1);
    run<2>("FADD2", 1);
    run<3>("FFMA", 1);
    run<4>("FFMA2 + FSETP/FSEL", 2);
    run<5>("FFMA2 / FMUL2 alternating", 1);
    return 0;
}
