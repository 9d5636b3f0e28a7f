// Forward model, register-run formulation (sm_100a): the default
// pc_forward_traces path.
//
//   replaces pkg/src/pacloud/radiator.py:86-118 (_forward_traces),
//   :195-216 (forward_frame) and reconstruction.py:312-313 (residual, loss)
//
// CTA = one trace row (sensor m, frame f), looping over ball chunks of
// FR_CHUNK balls.  The row is cut into runs of RUN consecutive samples.  Per
// chunk:
//
//   setup   one thread per ball: the fp64 pair geometry of common.cuh
//           (R, window [jl, jh), wavefront offset X at the reference sample
//           jr) into a 16-byte record + the window word; per 32-ball group
//           the span of runs its windows touch.
//   runs    one warp per run at a time (dynamic, index order): the warp
//           scans the groups whose span holds the run; a group whose 32
//           balls all meet the run is swept directly (lane = ball), the
//           others' overlapping balls are compacted into a per-warp queue
//           (ball order kept) that is swept 32 balls at a time, ONE BALL PER
//           LANE: each lane sweeps
//           all RUN samples of its ball with the Gaussian-on-grid recurrence
//           (e <- e g, g <- g h over two packed f32x2 chains, re-seeded by
//           MUFU every 16 samples) into RUN accumulators held in REGISTERS.
//           The 32 lanes' partial runs are then summed per sample through a
//           shared-memory transpose in fixed lane order and added to the
//           row's trace in shared memory.
//   epilog  residual = trace - observed, the row's fp64 L2 partial, one
//           coalesced (vectorised when aligned) store of the row.
//
// There is no shared-memory read-modify-write per ball sample (the old
// kernel's 8 B/sample ceiling) and no chunk-partial traces in HBM: a sample's
// work is 4 FMA-pipe lane-ops (x step, e, g, accumulate) + 1/8 of a MUFU seed.
// Every sum has a fixed order (ball order within a lane, lane order within a
// run, chunk order across chunks): the result is deterministic.
//
// Numerics.  A lane may start a run up to RUN-1 samples before its ball's
// window, where 2^-x^2 would underflow fp32 and kill the recurrence; the
// chain therefore carries E = 2^(80 - x^2) (scaled by 2^80, exact) and the
// run sums are scaled back by 2^-80 before they meet the trace.  The
// recurrence is used while the seed point stays inside the scaled range
// (s v dt <= vs_max, i.e. a0 >~ 0.06 mm at 40 MHz, 1.5 mm/us); smaller balls,
// pairs that need the near-field (R + v t) term and exact mode take the
// direct path (MUFU per sample, exact window clip [jl, jh) as the reference).
// Samples the fast path adds outside a pair's +-6 sigma window weigh
// < e^-18 of its peak (the reference's fast path drops them).
#include <stdlib.h>

#include "common.cuh"

// The file is compiled twice into the library: as is (the default forward)
// and with -DPC_FR_NS=tma -DPC_FR_TMA=1 -DPC_FR_CHUNK=512 (the TMA-staged
// variant, selected at run time with PC_FWD_TMA=1), each in its own namespace.
namespace pc {
#ifdef PC_FR_NS
namespace PC_FR_NS {
#endif

#ifndef PC_FR_RUN
#define PC_FR_RUN 32
#endif
#ifndef PC_FR_CHUNK
#define PC_FR_CHUNK 1024
#endif
#ifndef PC_FR_DIRECT
#define PC_FR_DIRECT 1
#endif
// a partly-hit group with at least this many members on the run is swept
// directly (lane = ball, the other lanes idle) instead of through the queue
// (config 3 forward, radius-sorted layout: 32 / 28 / 24 / 16 -> 242.3 /
// 240.6 / 240.6 / 243.1 ms)
#ifndef PC_FR_DIRECT_MIN
#define PC_FR_DIRECT_MIN 24
#endif
// PC_FR_QDUMMY 1 (default): the queue push is an unconditional store
// (non-members write a per-lane dummy slot behind the queue) instead of a
// branch (config 3 forward 240.6 -> 239.7 ms, bit-identical)
#ifndef PC_FR_QDUMMY
#define PC_FR_QDUMMY 1
#endif
#ifndef PC_FR_CHAIN1
#define PC_FR_CHAIN1 0
#endif
// PC_FR_ORDER 1: warp 0 orders each chunk's runs by weight (longest first)
// between the chunk's barriers; 0 (default): runs taken in index order, no
// run-weight bookkeeping (config 3 forward, same box: 303.3 vs 309.7 ms).
// PC_FR_DIRECT 1 (default): a group whose 32 balls all meet the run is swept
// directly, lane = ball, without the queue round trip (with ORDER 0:
// 280.4 vs 303.3 ms).  PC_FR_CHAIN1 1: one recurrence chain per ball-run (4
// MUFU seeds instead of 8; 284.2 with ORDER 0 + DIRECT, parity 1.3e-6 vs
// 4.2e-7): off.
#ifndef PC_FR_ORDER
#define PC_FR_ORDER 0
#endif
#ifndef PC_FR_LPT
#define PC_FR_LPT 1
#endif
// 4 CTAs (32 warps) per SM: 64 registers (small spill) and the 9 KB
// transpose buffer (PC_FR_XQ 1) keep the CTA under 57 KB of shared memory
// (config 3 forward 273.1 ms vs 279.9 at 3 CTAs / 80 registers / 20 KB)
#ifndef PC_FR_MINB
#define PC_FR_MINB 4
#endif
// PC_FR_SEEDS 1: the fast path takes the per-ball constant u = 2^(-D^2)
// (D = 2 s v dt) from the setup pass (kept in the record's Y word, which only
// near-field pairs use): h = u^2 and g(x - s v dt) = g(x) u, so a ball-run
// seeds 10 MUFU instead of 13.
#ifndef PC_FR_SEEDS
#define PC_FR_SEEDS 0
#endif
// PC_FR_TMA 1: the chunk's raw ball tile (mu, a0, p0 of FR_CHUNK balls) is
// staged in shared memory by three cp.async.bulk (TMA) copies completing on
// an mbarrier; the copy of chunk c+1 is issued right after chunk c's setup
// pass has consumed the stage, so it lands while the runs of chunk c are
// swept (the stage and the record buffers are the two halves of the
// pipeline).  Chunks whose global addresses or byte counts are not 16-byte
// multiples fall back to plain loads.
#ifndef PC_FR_TMA
#define PC_FR_TMA 0
#endif
// PC_FR_DIET 1 (default): the setup pass without the libdevice range guards
// (raw rcp / rsqrt.approx.ftz: the operands are normal floats), chunk-local
// 32-bit indexing, and the chunk's run range reduced from the group spans
// after the barrier instead of two shared-memory atomics per group.
#ifndef PC_FR_DIET
#define PC_FR_DIET 1
#endif
#ifndef PC_FR_SETUP_UNROLL
#define PC_FR_SETUP_UNROLL 1
#endif
// PC_FR_PF 1: L1 prefetch of the next chunk's raw balls at the start of the
// chunk's runs (the no-shared-memory counterpart of PC_FR_TMA).
#ifndef PC_FR_PF
#define PC_FR_PF 0
#endif
constexpr int FR_SETUP_UNROLL = PC_FR_SETUP_UNROLL;
constexpr int FR_RUN = PC_FR_RUN;          // samples per run (register accumulators)
constexpr int FR_CHUNK = PC_FR_CHUNK;      // balls per setup chunk
#ifndef PC_FR_WARPS
#define PC_FR_WARPS 8
#endif
constexpr int FR_WARPS = PC_FR_WARPS;
constexpr int FR_THREADS = FR_WARPS * 32;
constexpr int FR_GROUPS = FR_CHUNK / 32;
constexpr int FR_QLEN = 64;                // per-warp ball queue (circular)
// Transpose of the 32 lanes' partial runs: PC_FR_XQ 0: 16 samples at a time
// through [32][20] float rows (float4 stores); 1: 8 samples at a time
// through [32][9] rows (scalar stores, conflict-free), 9 KB instead of 20 KB
// of shared memory per CTA.
#ifndef PC_FR_XQ
#define PC_FR_XQ 1
#endif
constexpr int FR_XPAD = PC_FR_XQ ? 9 : 20;  // transpose row stride (floats)
constexpr float FR_SCALE_EXP = 80.f;       // chains carry c 2^(80 - x^2)
#define FR_U(idx) (PC_FR_SEEDS ? recY[idx] : 0.f)

__device__ __forceinline__ float fr_rcp(float x) {
#if PC_FR_DIET
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
#else
    return __fdividef(1.f, x);
#endif
}
__device__ __forceinline__ float fr_rsqrt(float x) {
#if PC_FR_DIET
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
#else
    return rsqrtf(x);
#endif
}

struct FwdRunArgs {
    const double* mu;      // (F,B,3)
    const float* a0;       // (F,B)
    const float* p0;       // (F,B)
    const double* pos;     // (M,3)
    const float* obs;      // (F,M,T) or NULL
    float* out;            // (F,M,T)
    double* loss;          // (F*M) row partials or NULL
    long long* coinc;
    int64_t B;
    int F, M;
    ArrayConsts ac;
    float vs_max;          // recurrence bound on s v dt
    // coincidence word = ((frame_offset + f) B + b) n_sensors_total + sensor_offset + m
    long long frame_offset, sensor_offset, n_sensors_total;
    // host-precomputed constants of the pair setup (bit-identical to common.cuh)
    float inv_v_f, t0_f, inv_dt_f, sa_f, vt0_f, vdt_f;
    double vdt_d, vt0_d;
};

// shared-memory layout (bytes)
struct FrSmem {
    static constexpr size_t recA = 0;                                   // float4 [C]
    static constexpr size_t recB = recA + (size_t)FR_CHUNK * 16;         // u32 [C]: jl | jh << 16
    static constexpr size_t recY = recB + (size_t)FR_CHUNK * 4;          // f32 [C]: near-field Y
    static constexpr size_t gspan = recY + (size_t)FR_CHUNK * 4;         // u32 [C/32]
    static constexpr size_t gfull = gspan + (size_t)FR_GROUPS * 4;       // u32 [C/32]: runs every member meets
    static constexpr size_t queue = gfull + (size_t)FR_GROUPS * 4;       // u16 [W][QLEN]
    static constexpr size_t xbuf = queue + (size_t)FR_WARPS * (FR_QLEN + 32 * PC_FR_QDUMMY) * 2;   // f32 [W][32][XPAD]
    static constexpr size_t ctl = xbuf + (size_t)FR_WARPS * 32 * FR_XPAD * 4; // int [8]
    // TMA stage of the next chunk's raw balls: mu f64 [C][3] | a0 f32 [C] | p0 f32 [C]
    static constexpr size_t rawmu = ctl + 64;
    static constexpr size_t rawa = rawmu + (PC_FR_TMA ? (size_t)FR_CHUNK * 24 : 0);
    static constexpr size_t rawp = rawa + (PC_FR_TMA ? (size_t)FR_CHUNK * 4 : 0);
    static constexpr size_t trace = rawp + (PC_FR_TMA ? (size_t)FR_CHUNK * 4 : 0);   // f32 [Tpad]
};

// after the trace: run weights (int [Tp/RUN]), run order (u16 [Tp/RUN]),
// weight histogram (int [32])
static size_t fr_smem_bytes(int T) {
    const size_t tp = ((size_t)T + FR_RUN - 1) / FR_RUN * FR_RUN;
    const size_t nr = tp / FR_RUN;
    return FrSmem::trace + tp * sizeof(float) + (nr + 4) * 4 + ((nr * 2 + 15) / 16) * 16 + 32 * 4;
}

// One ball's run, fast path: two packed chains (samples k, k+1), stepped by
// 2 samples; re-seeded every 16 samples.  x0 = x at the run's first sample.
// The Gaussian chain E = 2^(80 - x^2) does not depend on the amplitude c;
// the other factor carries it (xc = c x, stepped by -c D), so doubling p0
// doubles every product exactly (radiator tests: p0 scaling / two identical
// balls are bit-exact).
__device__ __forceinline__ void fr_fast(float2 (&acc)[FR_RUN / 2], float x0, float vs, float cs,
                                        float u) {
    static_assert(FR_RUN == 32, "two interleaved 16-sample halves");
#if PC_FR_CHAIN1
    // one packed chain over the whole run: 4 MUFU seeds instead of 8 (the
    // seed may sit up to 31 samples before the window: fr_vs_max)
    {
        const float D = 2.f * vs;
        const float2 mcD = splat2(-cs * D);
        const float2 h2 = splat2(ex2(-2.f * D * D));
        const float2 xa = make_float2(x0, x0 - vs);
        const float2 xxa = fmul2(xa, xa);
        float2 ea = make_float2(ex2(FR_SCALE_EXP - xxa.x), ex2(FR_SCALE_EXP - xxa.y));
        float2 ga = ex2_2(ffma2(xa, splat2(2.f * D), splat2(-D * D)));
        float2 ca = fmul2(splat2(cs), xa);
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            acc[k] = ffma2(ca, ea, acc[k]);
            if (k < 15) {
                ea = fmul2(ea, ga);
                ga = fmul2(ga, h2);
                ca = fadd2(ca, mcD);
            }
        }
        return;
    }
#endif
    const float D = 2.f * vs;
    const float2 mcD = splat2(-cs * D);
#if PC_FR_SEEDS
    const float2 h2 = splat2(u * u);
#else
    const float2 h2 = splat2(ex2(-2.f * D * D));
    const float2 tD = splat2(2.f * D), mDD = splat2(-D * D);
#endif
    const float2 csc = splat2(cs);
    // the two halves' chains run interleaved (independent: ILP for the
    // 4-cycle FMA-pipe latency of each chain)
    const float2 xa = make_float2(x0, x0 - vs);
    const float2 xb = make_float2(fmaf(-16.f, vs, x0), fmaf(-17.f, vs, x0));
    const float2 xxa = fmul2(xa, xa), xxb = fmul2(xb, xb);
    float2 ea = make_float2(ex2(FR_SCALE_EXP - xxa.x), ex2(FR_SCALE_EXP - xxa.y));
    float2 eb = make_float2(ex2(FR_SCALE_EXP - xxb.x), ex2(FR_SCALE_EXP - xxb.y));
#if PC_FR_SEEDS
    const float gax = ex2(fmaf(xa.x, 2.f * D, -D * D)), gbx = ex2(fmaf(xb.x, 2.f * D, -D * D));
    float2 ga = make_float2(gax, gax * u), gb = make_float2(gbx, gbx * u);
#else
    float2 ga = ex2_2(ffma2(xa, tD, mDD));
    float2 gb = ex2_2(ffma2(xb, tD, mDD));
#endif
    float2 ca = fmul2(csc, xa), cb = fmul2(csc, xb);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        acc[k] = ffma2(ca, ea, acc[k]);
        acc[8 + k] = ffma2(cb, eb, acc[8 + k]);
        if (k < 7) {
            ea = fmul2(ea, ga);
            eb = fmul2(eb, gb);
            ga = fmul2(ga, h2);
            gb = fmul2(gb, h2);
            ca = fadd2(ca, mcD);
            cb = fadd2(cb, mcD);
        }
    }
}

// Direct path: MUFU per sample, the reference's window [jl, jh) (exact mode:
// [0, T)), the near-field term where the pair needs it.
__device__ __forceinline__ void fr_slow(float2 (&acc)[FR_RUN / 2], int j0, float X, float Y,
                                        float vs, float cs, int jr, int jl, int jh, bool near) {
#pragma unroll
    for (int k = 0; k < FR_RUN / 2; ++k) {
        const int j = j0 + 2 * k;
        const float d0 = (float)(j - jr);
        float2 v = splat2(0.f);
        const float xa = fmaf(-d0, vs, X), xb = fmaf(-(d0 + 1.f), vs, X);
        v.x = xa * ex2(-xa * xa);
        v.y = xb * ex2(-xb * xb);
        if (near) {
            const float ya = fmaf(d0, vs, Y), yb = fmaf(d0 + 1.f, vs, Y);
            v.x = fmaf(ya, ex2(-ya * ya), v.x);
            v.y = fmaf(yb, ex2(-yb * yb), v.y);
        }
        // scaled units (x 2^80) like the fast path
        const float sc = cs * 1.2089258196146292e24f;   // 2^80
        if (j >= jl && j < jh) acc[k].x = fmaf(sc, v.x, acc[k].x);
        if (j + 1 >= jl && j + 1 < jh) acc[k].y = fmaf(sc, v.y, acc[k].y);
    }
}

// Sum the 32 lanes' partial runs per sample in a fixed order and add the
// run to the row (scaled back by 2^-80).
__device__ __forceinline__ void fr_flush(const float2 (&acc)[FR_RUN / 2], float* xb, float* trace,
                                         int j0, int Tp) {
    const int lane = threadIdx.x & 31;
#if PC_FR_XQ
#pragma unroll
    for (int qq = 0; qq < FR_RUN / 8; ++qq) {
        __syncwarp();
        float* rowp = xb + lane * FR_XPAD;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            rowp[2 * u] = acc[4 * qq + u].x;
            rowp[2 * u + 1] = acc[4 * qq + u].y;
        }
        __syncwarp();
        // lane = column c (8) x row block p (4 blocks of 8 rows)
        const int col = lane & 7, r0 = (lane >> 3) * 8;
        float sacc = 0.f;
#pragma unroll
        for (int r = 0; r < 8; ++r) sacc += xb[(r0 + r) * FR_XPAD + col];
        sacc += __shfl_down_sync(0xffffffffu, sacc, 16);
        sacc += __shfl_down_sync(0xffffffffu, sacc, 8);
        if (lane < 8) {
            // chain a holds samples 0..15 (acc 0..7), chain b 16..31
            const int j = j0 + 8 * qq + col;
            if (j < Tp) trace[j] += sacc * 8.271806125530277e-25f;   // 2^-80
        }
    }
#else
#pragma unroll
    for (int hb = 0; hb < FR_RUN / 16; ++hb) {
        __syncwarp();
        float4* rowp = reinterpret_cast<float4*>(xb + lane * FR_XPAD);
#pragma unroll
        for (int k = 0; k < 4; ++k)
            rowp[k] = make_float4(acc[8 * hb + 2 * k].x, acc[8 * hb + 2 * k].y,
                                  acc[8 * hb + 2 * k + 1].x, acc[8 * hb + 2 * k + 1].y);
        __syncwarp();
        // lane c < 16 sums rows 0..15 of column c, lane 16 + c rows 16..31
        const int col = lane & 15, r0 = lane & 16;
        float sacc = 0.f;
#pragma unroll
        for (int r = 0; r < 16; ++r) sacc += xb[(r0 + r) * FR_XPAD + col];
        const float other = __shfl_down_sync(0xffffffffu, sacc, 16);
        if (lane < 16) {
            const int j = j0 + 16 * hb + col;
            if (j < Tp) trace[j] += (sacc + other) * 8.271806125530277e-25f;   // 2^-80
        }
    }
#endif
}

// Row epilogue shared by the forward kernels: relative tail threshold,
// residual against the observed row, the row's fp64 L2 partial, one
// (vectorised when aligned) store.
__device__ __forceinline__ void fr_epilogue(const FwdRunArgs& a, const float* trace, float* xbuf,
                                            int T, size_t row) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // Samples below 2^-60 of the row's peak are set to zero: the fast path
    // sums the far Gaussian tails outside each pair's window (the reference
    // drops them), where products leave fp32's normal range; a threshold
    // RELATIVE to the row keeps the output exactly linear in p0.
    float mx = 0.f;
    for (int j = tid; j < T; j += FR_THREADS) mx = fmaxf(mx, fabsf(trace[j]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float* redf = reinterpret_cast<float*>(xbuf);
    if (lane == 0) redf[warp] = mx;
    __syncthreads();
    mx = 0.f;
#pragma unroll
    for (int w = 0; w < FR_WARPS; ++w) mx = fmaxf(mx, redf[w]);
    const float thr = mx * 8.673617379884035e-19f;    // 2^-60
    const size_t base = row * (size_t)T;
    double lsum = 0.0;
    const bool vec = (T & 3) == 0 && ((reinterpret_cast<uintptr_t>(a.out) |
                                       reinterpret_cast<uintptr_t>(a.obs)) & 15) == 0;
    if (vec) {
        const int T4 = T >> 2;
        float4* o4 = reinterpret_cast<float4*>(a.out + base);
        const float4* t4 = reinterpret_cast<const float4*>(trace);
        if (a.obs) {
            const float4* b4 = reinterpret_cast<const float4*>(a.obs + base);
            for (int j = tid; j < T4; j += FR_THREADS) {
                float4 p = t4[j];
                const float4 ob = __ldcs(b4 + j);
                p.x = fabsf(p.x) < thr ? 0.f : p.x;
                p.y = fabsf(p.y) < thr ? 0.f : p.y;
                p.z = fabsf(p.z) < thr ? 0.f : p.z;
                p.w = fabsf(p.w) < thr ? 0.f : p.w;
                const float4 r = make_float4(p.x - ob.x, p.y - ob.y, p.z - ob.z, p.w - ob.w);
                lsum = fma((double)r.x, (double)r.x, lsum);
                lsum = fma((double)r.y, (double)r.y, lsum);
                lsum = fma((double)r.z, (double)r.z, lsum);
                lsum = fma((double)r.w, (double)r.w, lsum);
                o4[j] = r;
            }
        } else {
            for (int j = tid; j < T4; j += FR_THREADS) {
                float4 p = t4[j];
                p.x = fabsf(p.x) < thr ? 0.f : p.x;
                p.y = fabsf(p.y) < thr ? 0.f : p.y;
                p.z = fabsf(p.z) < thr ? 0.f : p.z;
                p.w = fabsf(p.w) < thr ? 0.f : p.w;
                o4[j] = p;
            }
        }
    } else {
        for (int j = tid; j < T; j += FR_THREADS) {
            float r = trace[j];
            r = fabsf(r) < thr ? 0.f : r;
            if (a.obs) {
                r -= a.obs[base + j];
                lsum = fma((double)r, (double)r, lsum);
            }
            a.out[base + j] = r;
        }
    }
    if (a.loss) {
        double* red = reinterpret_cast<double*>(xbuf);
        __syncthreads();
        lsum = warp_sum(lsum);
        if (lane == 0) red[warp] = lsum;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int w = 0; w < FR_WARPS; ++w) t += red[w];
            a.loss[row] = t;
        }
    }
}

#if PC_FR_TMA
__device__ __forceinline__ unsigned fr_smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void fr_mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(fr_smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fr_mbar_expect(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fr_smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void fr_mbar_wait(unsigned long long* bar, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(fr_smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void fr_bulk(void* dst, const void* src, unsigned bytes,
                                        unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(fr_smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(fr_smem_u32(bar))
        : "memory");
}
#endif

template <bool EXACT>
__global__ void __launch_bounds__(FR_THREADS, PC_FR_MINB) k_fwd_run(FwdRunArgs a) {
    extern __shared__ __align__(16) unsigned char sm[];
    float4* recA = reinterpret_cast<float4*>(sm + FrSmem::recA);
    unsigned* recB = reinterpret_cast<unsigned*>(sm + FrSmem::recB);
    float* recY = reinterpret_cast<float*>(sm + FrSmem::recY);
    unsigned* gspan = reinterpret_cast<unsigned*>(sm + FrSmem::gspan);
    unsigned* gfull = reinterpret_cast<unsigned*>(sm + FrSmem::gfull);
    unsigned short* queue = reinterpret_cast<unsigned short*>(sm + FrSmem::queue);
    float* xbuf = reinterpret_cast<float*>(sm + FrSmem::xbuf);
    int* ctl = reinterpret_cast<int*>(sm + FrSmem::ctl);
    float* trace = reinterpret_cast<float*>(sm + FrSmem::trace);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int T = a.ac.T;
    const int Tp = (T + FR_RUN - 1) / FR_RUN * FR_RUN;
    const int NR = Tp / FR_RUN;
    int* runw = reinterpret_cast<int*>(trace + Tp);                         // [NR]
    unsigned short* rorder = reinterpret_cast<unsigned short*>(runw + NR + 4);   // [NR]
    int* whist = reinterpret_cast<int*>(sm + FrSmem::trace + (size_t)Tp * 4 + (size_t)(NR + 4) * 4 +
                                        (((size_t)NR * 2 + 15) / 16) * 16);  // [32]
    const int f = blockIdx.x / a.M, m = blockIdx.x % a.M;
    const size_t row = (size_t)f * a.M + m;
    const double px = a.pos[3 * m], py = a.pos[3 * m + 1], pz = a.pos[3 * m + 2];
    const float vsup = a.sa_f;          // support / (v dt) in samples per mm of a0

    for (int j = tid; j < Tp; j += FR_THREADS) trace[j] = 0.f;
    for (int j = tid; j < NR + 4; j += FR_THREADS) runw[j] = 0;
    // ctl[0..2] chunk parity 0: next run, run lo, run hi; ctl[4..6] parity 1
    if (tid < 8) ctl[tid] = (tid == 1 || tid == 5) ? 0x7fffffff : (tid == 2 || tid == 6) ? -1 : 0;
    __syncthreads();

    const size_t fb = (size_t)f * a.B;
#if PC_FR_TMA
    const double* rawmu = reinterpret_cast<const double*>(sm + FrSmem::rawmu);
    const float* rawa = reinterpret_cast<const float*>(sm + FrSmem::rawa);
    const float* rawp = reinterpret_cast<const float*>(sm + FrSmem::rawp);
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(ctl + 8);
    // a chunk is staged when its three sources are 16-byte aligned whole
    // multiples of 16 bytes (always, for full chunks of aligned frames)
    auto stageable = [&](int64_t c) -> bool {
        const int64_t n = min((int64_t)FR_CHUNK, a.B - c);
        return ((reinterpret_cast<uintptr_t>(a.mu + 3 * (fb + c)) |
                 reinterpret_cast<uintptr_t>(a.a0 + fb + c) |
                 reinterpret_cast<uintptr_t>(a.p0 + fb + c)) & 15) == 0 && (n & 3) == 0;
    };
    auto stage = [&](int64_t c) {
        const unsigned n = (unsigned)min((int64_t)FR_CHUNK, a.B - c);
        fr_mbar_expect(bar, n * 32u);
        fr_bulk(sm + FrSmem::rawmu, a.mu + 3 * (fb + c), n * 24u, bar);
        fr_bulk(sm + FrSmem::rawa, a.a0 + fb + c, n * 4u, bar);
        fr_bulk(sm + FrSmem::rawp, a.p0 + fb + c, n * 4u, bar);
    };
    unsigned phase = 0;
    if (tid == 0) {
        fr_mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (a.B > 0 && stageable(0)) stage(0);
    }
    __syncthreads();
#endif
    const unsigned lt = (1u << lane) - 1u;
    unsigned short* Q = queue + warp * (FR_QLEN + 32 * PC_FR_QDUMMY);
    float* xb = xbuf + warp * 32 * FR_XPAD;
    int par = 0;
    for (int64_t c0 = 0; c0 < a.B; c0 += FR_CHUNK, par ^= 1) {
        int* cc = ctl + 4 * par;
        // ---------------------------------------------------------- setup
#if PC_FR_TMA
        const bool staged = stageable(c0);
        if (staged) {
            fr_mbar_wait(bar, phase);
            phase ^= 1u;
        }
#endif
        // chunk-local views: 32-bit indices inside the chunk
        const double* muc = a.mu + 3 * (fb + c0);
        const float* a0c = a.a0 + fb + c0;
        const float* p0c = a.p0 + fb + c0;
        const int nb = (int)min((int64_t)FR_CHUNK, a.B - c0);
#pragma unroll FR_SETUP_UNROLL
        for (int i = tid; i < FR_CHUNK; i += FR_THREADS) {
            unsigned wb = 0x0000ffffu;           // empty window (jl = 0xffff, jh = 0)
            float4 ra = make_float4(0.f, 0.f, 0.f, 0.f);
            float ry = 0.f;
            if (i < nb) {
#if PC_FR_TMA
                const double dx = (staged ? rawmu[3 * i] : muc[3 * i]) - px;
                const double dy = (staged ? rawmu[3 * i + 1] : muc[3 * i + 1]) - py;
                const double dz = (staged ? rawmu[3 * i + 2] : muc[3 * i + 2]) - pz;
                const float av = staged ? rawa[i] : a0c[i];
                const float pv = staged ? rawp[i] : p0c[i];
#else
                const double dx = muc[3 * i] - px, dy = muc[3 * i + 1] - py, dz = muc[3 * i + 2] - pz;
                const float av = a0c[i];
                const float pv = p0c[i];
#endif
#if PC_FR_DIET
                const float s = sqrtf(kHalfLog2e) * fr_rcp(av);
#else
                const float s = __fdividef(sqrtf(kHalfLog2e), av);
#endif
                const double R2 = fma(dx, dx, fma(dy, dy, dz * dz));
                const float r2f = (float)R2;
                const float rinv = fr_rsqrt(r2f);
                const float rf = r2f * rinv;
                const double R = r2f > 1e-30f
                                     ? fma(fma(-(double)rf, (double)rf, R2), 0.5 * (double)rinv,
                                           (double)rf)
                                     : sqrt(R2);
                if (R < kCoincidenceEps) {
                    atomicMin(a.coinc, ((a.frame_offset + f) * a.B + (c0 + i)) * a.n_sensors_total +
                                           a.sensor_offset + m);
                } else {
                    const float tc = ((float)R * a.inv_v_f - a.t0_f) * a.inv_dt_f;
                    int lo, hi;
                    if (EXACT) {
                        lo = 0;
                        hi = T;
                    } else {
                        const float sa = vsup * av;
                        lo = (int)fminf(fmaxf(ceilf(tc - sa), 0.f), (float)T);
                        hi = (int)fminf(fmaxf(floorf(tc + sa) + 1.f, 0.f), (float)T);
                    }
                    if (hi > lo) {
                        const int rc = __float2int_rn(tc);
                        const int jr = min(max(rc, lo), hi - 1);
                        const double vt = fma((double)jr, a.vdt_d, a.vt0_d);
                        const float X = (float)(R - vt) * s;
                        ry = (float)(R + vt) * s;
                        const bool near = (float)R + a.vt0_f + a.vdt_f * (float)lo < 10.f * av;
                        const float vs = a.vdt_f * s;
                        const bool fast = !EXACT && !near && vs <= a.vs_max;
#if PC_FR_DIET
                        const float cs = (0.5f * pv) * fr_rcp((float)R * s);
#else
                        const float cs = __fdividef(0.5f * pv, (float)R * s);
#endif
#if PC_FR_SEEDS
                        if (fast) ry = ex2(-4.f * vs * vs);   // u = 2^(-D^2), D = 2 vs
#endif
                        ra = make_float4(X, cs, vs,
                                         __int_as_float(jr | (fast ? 0 : 1 << 30) |
                                                        (near ? (int)0x80000000u : 0)));
                        wb = (unsigned)lo | ((unsigned)hi << 16);
                    }
                }
            }
            recA[i] = ra;
            recB[i] = wb;
            recY[i] = ry;
            // group span of runs (lanes of this warp = the group's 32 balls)
            const int jl = wb & 0xffff, jh = wb >> 16;
            const int q0 = __reduce_min_sync(0xffffffffu, jh > jl ? jl / FR_RUN : 0x7fff);
            const int q1 = __reduce_max_sync(0xffffffffu, jh > jl ? (jh - 1) / FR_RUN : -1);
            // runs that every member's window meets (all 32 live): [max q0, min q1]
            const int f0 = __reduce_max_sync(0xffffffffu, jh > jl ? jl / FR_RUN : 0x7fff);
            const int f1 = __reduce_min_sync(0xffffffffu, jh > jl ? (jh - 1) / FR_RUN : -1);
            const int g = i >> 5;
            if (lane == 0) {
                gspan[g] = q1 >= q0 ? ((unsigned)q0 | ((unsigned)q1 << 16)) : 0x0000ffffu;
                gfull[g] = f1 >= f0 ? ((unsigned)f0 | ((unsigned)f1 << 16)) : 0x0000ffffu;
                if (q1 >= q0) {
#if !PC_FR_DIET || PC_FR_ORDER
                    atomicMin(cc + 1, q0);
                    atomicMax(cc + 2, q1);
#endif
#if PC_FR_ORDER
                    // run weight (groups whose span holds the run, the task
                    // order's work proxy) as a difference array
                    atomicAdd(runw + q0, 1);
                    atomicAdd(runw + q1 + 1, -1);
#endif
                }
            }
        }
        if (tid == 0) {   // the other parity's counters, for the next chunk
            int* cn = ctl + 4 * (par ^ 1);
            cn[0] = 0;
            cn[1] = 0x7fffffff;
            cn[2] = -1;
        }
        __syncthreads();
#if PC_FR_TMA
        // the stage is consumed: start the next chunk's copy under this
        // chunk's runs
        if (tid == 0 && c0 + FR_CHUNK < a.B && stageable(c0 + FR_CHUNK)) stage(c0 + FR_CHUNK);
#endif
#if PC_FR_PF
        for (int i = tid; i < FR_CHUNK; i += FR_THREADS) {
            const int64_t b = c0 + FR_CHUNK + i;
            if (b < a.B) {
                asm volatile("prefetch.global.L1 [%0];" ::"l"(a.mu + 3 * (fb + b)));
                if ((i & 31) == 0) {
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(a.a0 + fb + b));
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(a.p0 + fb + b));
                }
            }
        }
#endif
#if PC_FR_DIET && !PC_FR_ORDER
        // the chunk's run range from the group spans (every warp reduces the
        // same FR_GROUPS words: no atomics in the setup, no extra barrier)
        int rlo, rhi;
        {
            int l = 0x7fff, h = -1;
            for (int g = lane; g < FR_GROUPS; g += 32) {
                const unsigned sp = gspan[g];
                const int s0 = (int)(sp & 0xffff), s1 = (int)(sp >> 16);
                if (s1 >= s0) {
                    l = min(l, s0);
                    h = max(h, s1);
                }
            }
            rlo = __reduce_min_sync(0xffffffffu, l);
            rhi = __reduce_max_sync(0xffffffffu, h);
        }
#else
        const int rlo = cc[1], rhi = cc[2];
#endif
        const int nrun = rhi - rlo + 1;
        // ---------------------------------------------------------- task order
        // warp 0: runs by descending weight (counting sort on min(w, 31)), so
        // the long runs start first and the chunk ends on short ones (the
        // order does not change any result: each run is summed by one warp)
        if (PC_FR_ORDER && warp == 0 && nrun > 0) {
            // weights: inclusive prefix of the difference array (runs 0..rhi;
            // runs below rlo hold 0), the array zeroed for the next chunk
            int carry = 0;
            for (int b0 = 0; b0 <= rhi + 1; b0 += 32) {
                const int i = b0 + lane;
                int v = i <= rhi + 1 ? runw[i] : 0;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(0xffffffffu, v, o);
                    if (lane >= o) v += t;
                }
                v += carry;
                carry = __shfl_sync(0xffffffffu, v, 31);
                if (i <= rhi + 1) runw[i] = i <= rhi ? v : 0;
            }
            whist[lane] = 0;
            __syncwarp();
            for (int i = lane; i < nrun; i += 32) atomicAdd(whist + min(runw[rlo + i], 31), 1);
            __syncwarp();
            const int h = whist[lane];
            int suf = h;                          // sum of hist[w'] for w' >= lane
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_down_sync(0xffffffffu, suf, o);
                if (lane + o < 32) suf += t;
            }
            __syncwarp();
            whist[lane] = suf - h;                // first slot of weight `lane`
            __syncwarp();
            for (int i = lane; i < nrun; i += 32) {
                const int p = atomicAdd(whist + min(runw[rlo + i], 31), 1);
                rorder[p] = (unsigned short)(rlo + i);
            }
            __syncwarp();
            for (int i = lane; i <= rhi; i += 32) runw[i] = 0;
        }
#if PC_FR_ORDER || !PC_FR_DIET
        __syncthreads();
#endif
        // ---------------------------------------------------------- runs
        while (nrun > 0) {
            int k = 0;
            if (lane == 0) k = atomicAdd(cc, 1);
            k = __shfl_sync(0xffffffffu, k, 0);
            if (k >= nrun) break;
            const int q = (PC_FR_ORDER && PC_FR_LPT) ? rorder[k] : rlo + k;
            const int j0 = q * FR_RUN;
            float2 acc[FR_RUN / 2];
#pragma unroll
            for (int k = 0; k < FR_RUN / 2; ++k) acc[k] = splat2(0.f);
            int qn = 0, qd = 0, nd = 0;   // nd: a full group went the direct way
            for (int gb = 0; gb < FR_GROUPS; gb += 32) {
                const unsigned sp = (FR_GROUPS % 32 == 0 || gb + lane < FR_GROUPS) ? gspan[gb + lane]
                                                                                : 0x0000ffffu;
                const bool gh = (int)(sp & 0xffff) <= q && q <= (int)(sp >> 16);
                unsigned gm = __ballot_sync(0xffffffffu, gh);
#if PC_FR_DIRECT
                {
                    // groups every member of which meets the run: swept
                    // directly without testing the members' windows
                    const unsigned fu = (FR_GROUPS % 32 == 0 || gb + lane < FR_GROUPS)
                                            ? gfull[gb + lane]
                                            : 0x0000ffffu;
                    const unsigned fm = __ballot_sync(
                        0xffffffffu, (int)(fu & 0xffff) <= q && q <= (int)(fu >> 16));
                    gm &= ~fm;
                    unsigned fl = fm;
                    while (fl) {
                        const int g = gb + __ffs(fl) - 1;
                        fl &= fl - 1;
                        const int i = g * 32 + lane;
                        const float4 r = recA[i];
                        const int w = __float_as_int(r.w);
                        if (!(w & (1 << 30))) {
                            fr_fast(acc, fmaf(-(float)(j0 - (w & 0xffff)), r.z, r.x), r.z, r.y,
                                    FR_U(i));
                        } else {
                            const unsigned wq = recB[i];
                            fr_slow(acc, j0, r.x, recY[i], r.z, r.y, w & 0xffff, wq & 0xffff,
                                    wq >> 16, w < 0);
                        }
                        nd = 1;
                    }
                }
#endif
                while (gm) {
                    const int g = gb + __ffs(gm) - 1;
                    gm &= gm - 1;
                    const int i = g * 32 + lane;
                    const unsigned wb = recB[i];
                    const unsigned hm = __ballot_sync(0xffffffffu, (int)(wb & 0xffff) < j0 + FR_RUN &&
                                                                       (int)(wb >> 16) > j0);
#if PC_FR_DIRECT && PC_FR_DIRECT_MIN < 32
                // (with the default threshold of 32 the per-group full-run
                // range above already took every such group)
                if (__popc(hm) >= PC_FR_DIRECT_MIN) {
                    // (nearly) the whole group meets the run: each lane takes
                    // its own ball directly (no queue round trip); lanes whose
                    // ball misses the run stay idle
                    if ((hm >> lane) & 1u) {
                        const float4 r = recA[i];
                        const int w = __float_as_int(r.w);
                        if (!(w & (1 << 30))) {
                            fr_fast(acc, fmaf(-(float)(j0 - (w & 0xffff)), r.z, r.x), r.z, r.y,
                                    FR_U(i));
                        } else {
                            fr_slow(acc, j0, r.x, recY[i], r.z, r.y, w & 0xffff, wb & 0xffff,
                                    wb >> 16, w < 0);
                        }
                    }
                    nd = 1;
                    continue;
                }
#endif
#if PC_FR_QDUMMY
                    Q[((hm >> lane) & 1u) ? ((qn + __popc(hm & lt)) & (FR_QLEN - 1)) : FR_QLEN + lane] =
                        (unsigned short)i;
#else
                    if ((hm >> lane) & 1u) Q[(qn + __popc(hm & lt)) & (FR_QLEN - 1)] = (unsigned short)i;
#endif
                    qn += __popc(hm);
                    if (qn - qd >= 32) {
                        __syncwarp();
                        const int e = Q[(qd + lane) & (FR_QLEN - 1)];
                        const float4 r = recA[e];
                        const int w = __float_as_int(r.w);
                        if (!(w & (1 << 30))) {
                            fr_fast(acc, fmaf(-(float)(j0 - (w & 0xffff)), r.z, r.x), r.z, r.y,
                                    FR_U(e));
                        } else {
                            const unsigned wq = recB[e];
                            fr_slow(acc, j0, r.x, recY[e], r.z, r.y, w & 0xffff, wq & 0xffff,
                                    wq >> 16, w < 0);
                        }
                        qd += 32;
                    }
                }
            }
            __syncwarp();
            if (lane < qn - qd) {
                const int e = Q[(qd + lane) & (FR_QLEN - 1)];
                const float4 r = recA[e];
                const int w = __float_as_int(r.w);
                if (!(w & (1 << 30))) {
                    fr_fast(acc, fmaf(-(float)(j0 - (w & 0xffff)), r.z, r.x), r.z, r.y,
                            FR_U(e));
                } else {
                    const unsigned wq = recB[e];
                    fr_slow(acc, j0, r.x, recY[e], r.z, r.y, w & 0xffff, wq & 0xffff, wq >> 16,
                            w < 0);
                }
            }
            if (qn == 0 && nd == 0) continue;
            // ---- sum the 32 lanes' partial runs per sample (fixed order)
            fr_flush(acc, xb, trace, j0, Tp);
        }
        __syncthreads();
    }
    fr_epilogue(a, trace, xbuf, T, row);
}

// recurrence bound: the seed x of a half run is at most the window edge
// x (support sqrt(log2 e / 2) + s v dt) plus 16 samples; 2^(80 - x^2) must
// stay a normal float: x^2 <= 196 (margin to 206)
static float fr_vs_max(double support) {
    const double xe = 0.8493218002880191 * support;
    const double v = (14.0 - xe) / (PC_FR_CHAIN1 ? 33.0 : 17.0);
    return v > 0 ? (float)v : 0.f;
}

int fwd_run_samples_per_run() { return FR_RUN; }

int fwd_run_supported(const pc_array_t* array) {
    return array->n_samples < 65535 && fr_smem_bytes(array->n_samples) <= 200 * 1024;
}

size_t fwd_run_workspace_bytes(int32_t n_frames, const pc_array_t* array) {
    return (size_t)n_frames * array->n_sensors * sizeof(double) + 256;
}

int fwd_run_launch(const double* mu_t, const float* a0_t, const float* p0_t, int64_t n_balls,
                   int32_t F, const pc_array_t* array, const ArrayConsts& ac,
                   const float* observed, float* out, double* loss_partial,
                   int64_t* coincident, cudaStream_t st) {
    FwdRunArgs a;
    a.mu = mu_t;
    a.a0 = a0_t;
    a.p0 = p0_t;
    a.pos = array->positions;
    a.obs = observed;
    a.out = out;
    a.loss = loss_partial;
    a.coinc = reinterpret_cast<long long*>(coincident);
    a.B = n_balls;
    a.F = F;
    a.M = array->n_sensors;
    a.ac = ac;
    a.vs_max = fr_vs_max(ac.support);
    a.frame_offset = array->frame_offset;
    a.sensor_offset = array->sensor_offset;
    a.n_sensors_total = array->n_sensors_total > 0 ? array->n_sensors_total : array->n_sensors;
    a.inv_v_f = (float)ac.inv_v;
    a.t0_f = (float)ac.t0;
    a.inv_dt_f = (float)ac.inv_dt;
    a.sa_f = (float)(ac.support * ac.inv_v * ac.inv_dt);
    a.vt0_f = (float)(ac.v * ac.t0);
    a.vdt_f = (float)(ac.v * ac.dt);
    a.vdt_d = ac.v * ac.dt;
    a.vt0_d = ac.v * ac.t0;
    const size_t smem = fr_smem_bytes(ac.T);
    static unsigned long long attr_set = 0;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return PC_ERR_CUDA;
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(attr_set & bit)) {
        const int mx = 200 * 1024;
        cudaFuncSetAttribute(k_fwd_run<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(k_fwd_run<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        attr_set |= bit;
    }
    const unsigned grid = (unsigned)F * (unsigned)a.M;
    if (ac.exact)
        k_fwd_run<true><<<grid, FR_THREADS, smem, st>>>(a);
    else
        k_fwd_run<false><<<grid, FR_THREADS, smem, st>>>(a);
    return last_status();
}

#ifdef PC_FR_NS
}  // namespace PC_FR_NS
#endif
}  // namespace pc
