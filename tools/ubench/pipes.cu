// Pipe-throughput microbenchmark for sm_100a: packed f32x2 vs scalar FP32,
// immediate forms and MUFU.EX2 (tools/ubench/README: informs the radiator
// kernels' instruction mix).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long f2u(float2 a) {
    return (unsigned long long)__float_as_uint(a.x) | ((unsigned long long)__float_as_uint(a.y) << 32);
}
__device__ __forceinline__ float2 u2f(unsigned long long u) {
    return make_float2(__uint_as_float((unsigned)u), __uint_as_float((unsigned)(u >> 32)));
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    unsigned long long d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
    return u2f(d);
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
    unsigned long long d;
    asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(d);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    unsigned long long d;
    asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(d);
}
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float ffma_r(float a, float b, float c) {
    float d;
    asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ float fadd_r(float a, float b) {
    float d;
    asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}

constexpr int NIT = 2048;
constexpr int NC = 8;

template <int K>
__global__ void kbench(float* out, float s) {
    float2 a[NC], b = make_float2(s, s * 1.0001f), c = make_float2(s * 0.999f, s * 1.001f);
    float x[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) {
        a[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
        x[i] = threadIdx.x * 1e-4f + i * 0.01f;
    }
    for (int it = 0; it < NIT; ++it) {
#pragma unroll
        for (int i = 0; i < NC; ++i) {
            if (K == 0) a[i] = ffma2(a[i], b, c);                 // FFMA2 3-reg
            if (K == 1) a[i] = fmul2(a[i], b);                    // FMUL2
            if (K == 2) a[i] = fadd2(a[i], c);                    // FADD2
            if (K == 3) x[i] = ffma_r(x[i], b.x, c.x);            // FFMA 3-reg
            if (K == 4) x[i] = x[i] * 0.999f + 0.5f;              // FFMA imm
            if (K == 5) x[i] = ex2(-x[i]);                        // MUFU.EX2
            if (K == 6) x[i] = fadd_r(x[i], c.x);                 // FADD
            if (K == 7) { a[i] = ffma2(a[i], b, c); x[i] = ex2(-x[i]); }   // FFMA2 + MUFU
            if (K == 8) { a[i] = fmul2(a[i], b); x[i] = fadd_r(x[i], c.x); }  // FMUL2 + FADD (alu?)
        }
    }
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < NC; ++i) acc += a[i].x + a[i].y + x[i];
    if (acc == 1234.5f) out[threadIdx.x] = acc;
}

// Shared-memory read-modify-write of float2 (the forward's trace update):
// each warp owns a 2 KB trace, lane l updates samples 2l, 2l+1 of 64-sample
// steps (one conflict-free 256-byte LDS.64 + STS.64 per warp step).
__global__ void ksmem(float* out, float s) {
    __shared__ float2 tr[8][256];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    for (int i = l; i < 256; i += 32) tr[w][i] = make_float2(0.f, 0.f);
    __syncwarp();
    const float2 c = make_float2(s, s * 0.5f);
    for (int it = 0; it < NIT; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            float2* p = &tr[w][(k * 32 + l + it) & 255];   // address varies per iteration
            float2 t;
            asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(t.x), "=f"(t.y)
                         : "r"((unsigned)__cvta_generic_to_shared(p)));
            t.x += c.x;
            t.y += c.y;
            asm volatile("st.shared.v2.f32 [%0], {%1, %2};" :: "r"((unsigned)__cvta_generic_to_shared(p)),
                         "f"(t.x), "f"(t.y) : "memory");
        }
    }
    __syncwarp();
    float acc = 0.f;
    for (int i = l; i < 256; i += 32) acc += tr[w][i].x + tr[w][i].y;
    if (acc == 1234.5f) out[threadIdx.x] = acc;
}

void run_smem() {
    float* out;
    cudaMalloc(&out, 4096);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = nsm * 8, threads = 256;
    ksmem<<<blocks, threads>>>(out, 1.f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) ksmem<<<blocks, threads>>>(out, 1.f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    // samples updated: 2 per lane per RMW
    const double samples = 5.0 * blocks * threads * (double)NIT * 8 * 2;
    const double cycles = ms * 1e-3 * clk * 1e3;
    printf("%-28s %.3f samples/clk/SM  (%.3f ms)\n", "smem float2 RMW", samples / cycles / nsm, ms);
    cudaFree(out);
}

template <int K>
void run(const char* name, int ops_per_inner) {
    float* out;
    cudaMalloc(&out, 4096);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = nsm * 8, threads = 256;
    kbench<K><<<blocks, threads>>>(out, 1.f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) kbench<K><<<blocks, threads>>>(out, 1.f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double warp_instr = 5.0 * blocks * (threads / 32) * (double)NIT * NC * ops_per_inner;
    const double cycles = ms * 1e-3 * clk * 1e3;
    printf("%-28s %.3f warp-instr/clk/SMSP  (%.3f ms)\n", name, warp_instr / cycles / nsm / 4, ms);
    cudaFree(out);
}

int main() {
    run<0>("FFMA2 3-reg", 1);
    run<1>("FMUL2", 1);
    run<2>("FADD2", 1);
    run<3>("FFMA 3-reg", 1);
    run<4>("FFMA imm", 1);
    run<5>("MUFU.EX2", 1);
    run<6>("FADD", 1);
    run<7>("FFMA2+MUFU (pairs)", 2);
    run<8>("FMUL2+FADD (pairs)", 2);
    run_smem();
    return 0;
}
