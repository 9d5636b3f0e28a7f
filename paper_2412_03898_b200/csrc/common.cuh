// Shared device helpers for the pacloud_b200 sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "pacloud_b200.h"

#define PC_NUM_SMS_DEFAULT 148

namespace pc {

constexpr float kLog2e = 1.4426950408889634f;
constexpr double kCoincidenceEps = 1e-9;  // radiator.py:33 _COINCIDENCE_EPS

// MUFU ex2 (flush-to-zero). Arguments here are <= 0, results in [0, 1].
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Packed fp32x2 arithmetic (FFMA2 / FMUL2 / FADD2 on sm_100a): one issue slot
// and one FMA-pipe slot for two lanes' worth of work.
__device__ __forceinline__ unsigned long long f2u(float2 a) {
    return (unsigned long long)__float_as_uint(a.x) |
           ((unsigned long long)__float_as_uint(a.y) << 32);
}
__device__ __forceinline__ float2 u2f(unsigned long long u) {
    return make_float2(__uint_as_float((unsigned)u), __uint_as_float((unsigned)(u >> 32)));
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
    return u2f(d);
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(d);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(d);
}
__device__ __forceinline__ float2 ex2_2(float2 x) { return make_float2(ex2(x.x), ex2(x.y)); }
// 2^-xx per component (the negation folds into MUFU.EX2's operand)
__device__ __forceinline__ float2 ex2n_2(float2 xx) { return make_float2(ex2(-xx.x), ex2(-xx.y)); }
__device__ __forceinline__ float2 splat2(float v) { return make_float2(v, v); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

inline int status_of(cudaError_t e) { return e == cudaSuccess ? PC_OK : PC_ERR_CUDA; }

inline int last_status() { return status_of(cudaGetLastError()); }

inline int num_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
            n <= 0)
            n = PC_NUM_SMS_DEFAULT;
    }
    return n;
}

inline cudaStream_t as_stream(pc_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// Per-(ball, sensor) window and fp64 wavefront offsets, shared by forward
// and adjoint.  Follows radiator.py:93-112 with the reciprocals of v and dt
// hoisted (an edge sample can move only where (R +- 6a)/v lands exactly on a
// sample time; such samples weigh exp(-18) of the peak).
//
// Samples are evaluated in scaled units x = s * (R - v t), s = sqrt(log2 e /
// 2) / a0, so exp(-(R - v t)^2 / (2 a0^2)) = 2^(-x^2) is one FMUL + MUFU.EX2.
// X (and Y for the near-field R + v t term) are x at the window start, formed
// in fp64 and rounded once; per sample x = X - k * (s v dt) in fp32 with an
// exact integer k, so the error stays ~1e-7 of a0.
struct ArrayConsts {
    double v, t0, dt, inv_v, inv_dt, support;
    float vdt;
    int T;
    int exact;
};

constexpr float kHalfLog2e = 0.72134752044448170f;   // log2(e) / 2
constexpr float kKappa = 1.3862943611198906f;        // 2 / log2(e) = 1/(s a)^2

__device__ __forceinline__ float scale_of(float a0) { return sqrtf(kHalfLog2e) / a0; }

struct PairSetup {
    double R;
    int jl, jh;    // window clipped to [clip_lo, clip_hi)
    int jr;        // reference sample: nearest the (R - v t) wavefront, in window
    float X, Y;    // s (R -/+ v t_jr)
    bool near;     // the (R + v t) term exceeds exp(-50) of the peak somewhere
};

// Window and offsets of one pair.  R is refined from an fp32 estimate by one
// fp64 Newton step (|error| ~ 1e-16 R); the window bounds and the reference
// sample come from the fp32 wavefront position (an edge can move by one
// sample only within ~1e-3 sample of a boundary, where the Gaussian weighs
// exp(-18)); the wavefront offsets X, Y are differences formed in fp64.
__device__ __forceinline__ void pair_setup(double dx, double dy, double dz, float a0, float s,
                                           const ArrayConsts& ac, int clip_lo, int clip_hi,
                                           PairSetup& q) {
    const double R2 = fma(dx, dx, fma(dy, dy, dz * dz));
    const float r2f = (float)R2;
    const float rinv = rsqrtf(r2f);
    const float rf = r2f * rinv;
    const double R = r2f > 1e-30f
                         ? fma(fma(-(double)rf, (double)rf, R2), 0.5 * (double)rinv, (double)rf)
                         : sqrt(R2);
    q.R = R;
    int lo, hi;
    const float tc = ((float)R * (float)ac.inv_v - (float)ac.t0) * (float)ac.inv_dt;
    if (ac.exact) {
        lo = 0;
        hi = ac.T;
    } else {
        const float sa = (float)(ac.support * ac.inv_v * ac.inv_dt) * a0;
        const float flo = ceilf(tc - sa);
        const float fhi = floorf(tc + sa) + 1.f;
        lo = (int)fminf(fmaxf(flo, 0.f), (float)ac.T);
        hi = (int)fminf(fmaxf(fhi, 0.f), (float)ac.T);
    }
    q.jl = max(lo, clip_lo);
    q.jh = min(hi, clip_hi);
    const int rc = __float2int_rn(tc);
    q.jr = min(max(rc, q.jl), max(q.jh - 1, q.jl));
    const double vt = fma((double)q.jr, ac.v * ac.dt, ac.v * ac.t0);
    q.X = (float)(R - vt) * s;
    q.Y = (float)(R + vt) * s;
    q.near = (float)R + (float)(ac.v * ac.t0) + (float)(ac.v * ac.dt) * (float)q.jl <
             10.f * a0;
}

// Longest supported trace (sample indices stay in 30 bits).
constexpr int kMaxSamples = 1 << 30;

// register-run forward (fwd_run.cu)
int fwd_run_supported(const pc_array_t* array);
int fwd_run_samples_per_run();
size_t fwd_run_workspace_bytes(int32_t n_frames, const pc_array_t* array);
int fwd_run_launch(const double* mu_t, const float* a0_t, const float* p0_t, int64_t n_balls,
                   int32_t F, const pc_array_t* array, const ArrayConsts& ac,
                   const float* observed, float* out, double* loss_partial,
                   int64_t* coincident, cudaStream_t st);
// the same file compiled with TMA-staged ball tiles (PC_FWD_TMA=1 at run time)
namespace tma {
int fwd_run_supported(const pc_array_t* array);
int fwd_run_samples_per_run();
size_t fwd_run_workspace_bytes(int32_t n_frames, const pc_array_t* array);
int fwd_run_launch(const double* mu_t, const float* a0_t, const float* p0_t, int64_t n_balls,
                   int32_t F, const pc_array_t* array, const ArrayConsts& ac,
                   const float* observed, float* out, double* loss_partial,
                   int64_t* coincident, cudaStream_t st);
}  // namespace tma

}  // namespace pc
