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

// Per-(ball, sensor) window and fp64 offsets, shared by forward and adjoint.
// Follows radiator.py:93-112 with the reciprocals of v and dt hoisted (the
// window edge can move by one sample only where (R +- 6a)/v lands exactly on
// a sample time; those samples weigh exp(-18) of the peak).
struct PairGeom {
    double R;
    int jlo, jhi;  // clipped to [0, T)
    int jc;        // reference sample for the fp32 offsets (near the peak)
    float Dc;      // R - v*t(jc), fp32 of an fp64 difference
    float Uc;      // R + v*t(jc)
    bool near;     // the (R + v t) term matters somewhere in the window
};

struct ArrayConsts {
    double v, t0, dt, inv_v, inv_dt, support;
    float vdt;
    int T;
    int exact;
};

__device__ __forceinline__ void pair_geometry(double dx, double dy, double dz, float a0,
                                              const ArrayConsts& ac, PairGeom& g) {
    g.R = sqrt(dx * dx + dy * dy + dz * dz);
    const double R = g.R;
    int lo, hi;
    if (ac.exact) {
        lo = 0;
        hi = ac.T;
    } else {
        const double sa = ac.support * (double)a0;
        const double flo = ceil(((R - sa) * ac.inv_v - ac.t0) * ac.inv_dt);
        const double fhi = floor(((R + sa) * ac.inv_v - ac.t0) * ac.inv_dt) + 1.0;
        lo = flo < 0.0 ? 0 : (flo > (double)ac.T ? ac.T : (int)flo);
        hi = fhi > (double)ac.T ? ac.T : (fhi < 0.0 ? 0 : (int)fhi);
    }
    g.jlo = lo;
    g.jhi = hi;
    double fc = rint((R * ac.inv_v - ac.t0) * ac.inv_dt);
    int jc = fc < (double)lo ? lo : (fc > (double)(hi - 1) ? hi - 1 : (int)fc);
    if (hi <= lo) jc = lo;
    g.jc = jc;
    const double vt = ac.v * (ac.t0 + (double)jc * ac.dt);
    g.Dc = (float)(R - vt);
    g.Uc = (float)(R + vt);
    const double upmin = R + ac.v * (ac.t0 + (double)lo * ac.dt);
    g.near = upmin < 10.0 * (double)a0;
}

}  // namespace pc
