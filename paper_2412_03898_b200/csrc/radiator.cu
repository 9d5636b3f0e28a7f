// Radiator hot path for sm_100a: sensor-major forward (fused residual + L2
// loss) and ball-major adjoint.
//
//   forward  <- pkg/src/pacloud/radiator.py:86-118 (_forward_traces),
//               :195-216 (forward_frame), reconstruction.py:312-313 (loss)
//   adjoint  <- pkg/src/pacloud/radiator.py:121-174 (_residual_state_grads),
//               :219-242 (frame_state_grads)
//
// Numerics: per (ball, sensor) pair the distance R, the window and the
// wavefront offsets are formed in fp64 (the subtraction R - v t cancels
// ~2-3 decades at 60-110 mm); the per-sample inner loops run in fp32 with
// MUFU ex2.  The (R + v t) near-field term is evaluated only where it can
// exceed exp(-50) of the peak (R + v t < 10 a0), inside the reference's
// far-field window exactly as radiator.py:113-118 does.
#include "common.cuh"

namespace pc {

// ---------------------------------------------------------------- forward
//
// CTA = FWD_WARPS warps x FSW (2) sensors x one time segment x one frame x
// one ball chunk.  Each sensor has a private shared-memory trace, so
// accumulation needs no atomics and its order is fixed (deterministic).
// Warps never synchronise with each other: each streams the chunk's ball
// records (a compact float4 {x, y, z, a0} cull record, L1/L2 resident) with a
// one-batch prefetch.  Segments are laid over the warp's ACTIVE arrival range,
// derived from the (frame, chunk) ball bounding box, so no segment is empty.
// Per 16-ball batch a lane-parallel fp32 cull (skipped when one segment holds
// the whole range) drops balls whose +-6 sigma window misses the segment;
// surviving pairs get the fp64 setup and a 32-byte record; then both
// half-warps sweep each surviving ball's window for their own sensor, lanes
// on consecutive sample pairs.  With ball chunks, each chunk's partial traces
// are written over the active range and combined in fixed chunk order by
// k_forward_combine (k_forward_finish for dense rows).

#ifndef PC_FWD_WARPS
#define PC_FWD_WARPS 4
#endif
constexpr int FWD_WARPS = PC_FWD_WARPS;        // warps per forward CTA
#ifndef PC_FWD_FSW
#define PC_FWD_FSW 2
#endif
constexpr int FSW = PC_FWD_FSW;     // sensors per warp (32 / FSW lanes each)
constexpr int FL = 32 / FSW;        // lanes per (ball, sensor) pair
constexpr int FSTR = 2 * FL;        // samples between a lane's successive pairs
constexpr int FBATCH = 32 / FSW;    // balls per setup batch (one lane per pair)
constexpr int FWD_TSEG_MAX = 1024;  // samples per time segment (private traces)
constexpr int64_t FWD_CHUNK_BALLS = 16384;            // balls per forward chunk (max)
#ifndef PC_FWD_MIN_CHUNK
#define PC_FWD_MIN_CHUNK 128
#endif
constexpr int64_t FWD_MIN_CHUNK_BALLS = PC_FWD_MIN_CHUNK; // balls per forward chunk (min)
#ifndef PC_FWD_BUDGET_GB
#define PC_FWD_BUDGET_GB 48
#endif
constexpr size_t FWD_PARTIAL_BUDGET = (size_t)PC_FWD_BUDGET_GB << 30;  // bytes of chunk partial traces
constexpr int TRACE_PAD = 8;        // floats after a trace (even-window overrun)

struct FwdPlan {
    int Tseg, nseg, nchunk;
    int64_t chunk_balls;
    size_t partial_bytes, loss_bytes, prep_bytes;
};

// Segment length cap (samples); PC_FWD_TSEG overrides it for tuning sweeps.
static int fwd_tseg_max() {
    static int v = 0;
    if (v == 0) {
        const char* e = getenv("PC_FWD_TSEG");
        const int x = e ? atoi(e) : 0;
        v = (x >= 64 && x <= 8192) ? (x / 32) * 32 : FWD_TSEG_MAX;
    }
    return v;
}

static size_t fwd_smem_bytes(int Tseg);

// Target waves of resident CTAs when balls are chunked (PC_FWD_WAVES).  With
// per-(frame, chunk) bounding boxes, finer Morton chunks also tighten each
// warp's arrival range; measured on config 2 (segment cap 1024): 8 / 12 / 20
// / 32 waves -> 5.84 / 5.49 / 5.47 / 5.52 ms forward.
static int fwd_waves() {
    static int v = 0;
    if (v == 0) {
        const char* e = getenv("PC_FWD_WAVES");
        const int x = e ? atoi(e) : 0;
        v = (x >= 1 && x <= 64) ? x : 12;
    }
    return v;
}

static FwdPlan fwd_plan(int64_t B, int F, int M, int T) {
    FwdPlan p;
    const int tmax = fwd_tseg_max();
    p.Tseg = T < tmax ? ((T + 31) / 32) * 32 : tmax;
    p.nseg = (T + p.Tseg - 1) / p.Tseg;
    const int64_t tiles = (M + FWD_WARPS * FSW - 1) / (FWD_WARPS * FSW);
    // CTAs with work (the active arrival range typically spans half of T);
    // ask for >= 2 waves of resident CTAs so the tail stays short
    const int64_t base = tiles * F * (p.nseg > 1 ? p.nseg / 2 : 1);
    const int per_sm = (int)(228 * 1024 / (fwd_smem_bytes(p.Tseg) + 1024));
    const int64_t want = (int64_t)fwd_waves() * (per_sm < 1 ? 1 : per_sm > 16 ? 16 : per_sm) *
                         num_sms();
    int64_t c = base >= want ? 1 : (want + base - 1) / base;
    // Morton chunks of at most FWD_CHUNK_BALLS balls keep each chunk's
    // bounding box (hence its warps' arrival ranges) tight; measured on
    // configs 3 / 4: 1 -> 8 / 16 chunks cut the forward 506 -> 393 ms and
    // 2855 -> 2041 ms.  The partial traces are bounded by FWD_PARTIAL_BUDGET.
    const int64_t c_box = (B + FWD_CHUNK_BALLS - 1) / FWD_CHUNK_BALLS;
    if (c < c_box) c = c_box;
    const char* ce = getenv("PC_FWD_CHUNKS");      // tuning override
    if (ce && atoi(ce) > 0) c = atoi(ce);
    const int64_t cmax = B / FWD_MIN_CHUNK_BALLS > 1 ? B / FWD_MIN_CHUNK_BALLS : 1;
    if (c > cmax) c = cmax;
    if (c > 64) c = 64;
    const size_t per_chunk = (size_t)F * M * T * sizeof(float);
    const int64_t cmem = per_chunk ? (int64_t)(FWD_PARTIAL_BUDGET / per_chunk) : 64;
    if (c > 1 && c > cmem) c = cmem > 1 ? cmem : 1;
    p.nchunk = (int)c;
    p.chunk_balls = (B + c - 1) / c;
    p.partial_bytes = p.nchunk > 1 ? (size_t)p.nchunk * F * M * T * sizeof(float) : 0;
    const int nloss = p.nchunk > 1 ? 1 : p.nseg;
    p.loss_bytes = (size_t)F * M * nloss * sizeof(double);
    // cull records (F,B) float4 + per-(frame, chunk) bounds (8 u32), 256-byte aligned
    p.prep_bytes = (((size_t)F * B * sizeof(float4) + 255) / 256) * 256 +
                   (size_t)F * p.nchunk * 8 * sizeof(unsigned);
    return p;
}

struct FwdRec {
    float4 r0, r1;
};
struct FwdWarpSmem {                 // per-warp shared memory
    FwdRec rec[32];                  // pair records of the current batch, [sensor slot][ball]
};

static size_t fwd_smem_bytes(int Tseg) {
    return (size_t)FWD_WARPS *
           (sizeof(FwdWarpSmem) + (size_t)FSW * (Tseg + TRACE_PAD) * sizeof(float));
}

// order-preserving float <-> u32 (atomicMin on the code = float min)
__device__ __forceinline__ unsigned f2ord(float f) {
    const unsigned b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float ord2f(unsigned u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// Per (frame, ball): the float4 cull record, and the frame's bounding box
// (min xyz, max xyz as ~code, max a0 as ~code: all atomicMin, init 0xff..).
__global__ void __launch_bounds__(256) k_forward_prep(const double* __restrict__ mu,
                                                      const float* __restrict__ a0, int64_t B,
                                                      int F, int nchunk, int64_t chunk_balls,
                                                      int bpc, float4* __restrict__ cull,
                                                      unsigned* __restrict__ bounds) {
    // blockIdx.x = chunk * bpc + block within the chunk: bounds per (frame,
    // ball chunk), so a chunk's warps lay their traces over the arrival
    // range of that chunk's balls only
    const int f = blockIdx.y;
    const int c = blockIdx.x / bpc;
    const int64_t c0 = (int64_t)c * chunk_balls;
    const int64_t c1 = min(B, c0 + chunk_balls);
    unsigned mn[3] = {~0u, ~0u, ~0u}, mxn[4] = {~0u, ~0u, ~0u, ~0u};
    for (int64_t b = c0 + (int64_t)(blockIdx.x % bpc) * blockDim.x + threadIdx.x; b < c1;
         b += (int64_t)bpc * blockDim.x) {
        const size_t s = (size_t)f * B + b;
        const float x = (float)mu[3 * s], y = (float)mu[3 * s + 1], z = (float)mu[3 * s + 2];
        const float a = a0[s];
        cull[s] = make_float4(x, y, z, a);
        const float v[3] = {x, y, z};
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            mn[k] = min(mn[k], f2ord(v[k]));
            mxn[k] = min(mxn[k], ~f2ord(v[k]));
        }
        mxn[3] = min(mxn[3], ~f2ord(a));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            mn[k] = min(mn[k], __shfl_xor_sync(0xffffffffu, mn[k], o));
            mxn[k] = min(mxn[k], __shfl_xor_sync(0xffffffffu, mxn[k], o));
        }
        mxn[3] = min(mxn[3], __shfl_xor_sync(0xffffffffu, mxn[3], o));
    }
    if ((threadIdx.x & 31) == 0) {
        unsigned* bf = bounds + 8 * ((size_t)f * nchunk + c);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            atomicMin(bf + k, mn[k]);
            atomicMin(bf + 3 + k, mxn[k]);
        }
        atomicMin(bf + 6, mxn[3]);
    }
}

// Can the Gaussian-on-grid recurrence run for this ball?  x starts at most
// ~support*sqrt(log2 e / 2) + 2 vs from the wavefront; the ratios g (and the
// second ratio h = 2^-2D^2, D = stride * vs) must stay inside fp32's range.
__device__ __forceinline__ bool recur_ok(float D, float vs, float support) {
    const float xmax = sqrtf(kHalfLog2e) * support + 2.f * vs;
    return 2.f * D * xmax + D * D <= 120.f && 2.f * D * D <= 120.f;
}

// Per-lane start of the recurrence for samples (j, j+1): e = 2^-x^2,
// g = e(j + stride) / e(j) = 2^(2 D x - D^2).
__device__ __forceinline__ void recur_init(float2 x, float D, float2& e, float2& g) {
    e = ex2n_2(fmul2(x, x));
    g = ex2_2(ffma2(x, splat2(2.f * D), splat2(-D * D)));
}

struct FwdArgs {
    const double* mu;
    const float* p0;
    const float4* cull;
    const unsigned* bounds;
    const double* pos;
    const int* sorder;   // sensor processing order (spatial neighbours) or NULL
    const float* obs;
    float* out;          // final (nchunk == 1) or partial traces (nchunk > 1)
    double* loss;        // (F, M, nseg) partials or NULL
    long long* coinc;
    int64_t B;
    int F, M;
    ArrayConsts ac;
    int Tseg, nseg, nchunk;
    int64_t chunk_balls;
    // host-precomputed casts / products of ArrayConsts for the per-pair
    // setup (the same IEEE operations pair_setup performs on the device,
    // so the setup is bit-identical; ptxas otherwise re-converts them from
    // the double constants in every batch)
    float inv_v_f, t0_f, inv_dt_f, sa_f, vt0_f, vdt_f;
    double vdt_d, vt0_d;
    int part_margin;     // > 0: partial rows written over the active range +- margin only
    long long fo, so, mt; // coincidence word: frame offset, sensor offset, total sensors
};

// s = sqrt(log2 e / 2) / a0 by the approximate division (2 ulp: x and the
// amplitude move by ~2e-7 relative, far inside the 1e-5 signal tolerance;
// the IEEE division's slow path cost 112 instructions of code and 0.7 % of
// the forward)
#ifndef PC_FWD_NOCULL1
#define PC_FWD_NOCULL1 1
#endif
#ifndef PC_FWD_FASTDIV
#define PC_FWD_FASTDIV 1
#endif
#if PC_FWD_FASTDIV
#define PC_FWD_SCALE(a0) __fdividef(sqrtf(kHalfLog2e), (a0))
#else
#define PC_FWD_SCALE(a0) scale_of(a0)
#endif
#ifndef PC_FWD_FCONST
#define PC_FWD_FCONST 1
#endif
// pair_setup (common.cuh) with the array constants taken from FwdArgs'
// precomputed fields; identical arithmetic.
__device__ __forceinline__ void pair_setup_fwd(double dx, double dy, double dz, float a0,
                                               const FwdArgs& a, int clip_lo, int clip_hi,
                                               PairSetup& q, float s) {
    const double R2 = fma(dx, dx, fma(dy, dy, dz * dz));
    const float r2f = (float)R2;
    const float rinv = rsqrtf(r2f);
    const float rf = r2f * rinv;
    const double R = r2f > 1e-30f
                         ? fma(fma(-(double)rf, (double)rf, R2), 0.5 * (double)rinv, (double)rf)
                         : sqrt(R2);
    q.R = R;
    int lo, hi;
    const float tc = ((float)R * a.inv_v_f - a.t0_f) * a.inv_dt_f;
    const int T = a.ac.T;
    if (a.ac.exact) {
        lo = 0;
        hi = T;
    } else {
        const float sa = a.sa_f * a0;
        const float flo = ceilf(tc - sa);
        const float fhi = floorf(tc + sa) + 1.f;
        lo = (int)fminf(fmaxf(flo, 0.f), (float)T);
        hi = (int)fminf(fmaxf(fhi, 0.f), (float)T);
    }
    q.jl = max(lo, clip_lo);
    q.jh = min(hi, clip_hi);
    const int rc = __float2int_rn(tc);
    q.jr = min(max(rc, q.jl), max(q.jh - 1, q.jl));
    const double vt = fma((double)q.jr, a.vdt_d, a.vt0_d);
    q.X = (float)(R - vt) * s;
    q.Y = (float)(R + vt) * s;
    q.near = (float)R + a.vt0_f + a.vdt_f * (float)q.jl < 10.f * a0;
}

// Both half-warps sweep the same ball for their own sensor: lane `sub` of a
// half owns sample pairs (j, j+1), j = je0 + 2 sub + FSTR n, so each half's
// float2 access is 128 contiguous bytes of its own trace (one conflict-free
// wavefront).
// Gaussian term of one sample pair: x 2^(-x^2)
__device__ __forceinline__ float2 gterm(float2 x) { return fmul2(x, ex2n_2(fmul2(x, x))); }

// Record word 0: byte offset of sample je0 in the warp's trace area (this
// half's trace, segment-relative; even je0) | slow << 30 | recur << 31 (per
// ball: slow = a pair of the ball needs the near field (or exact), recur =
// the Gaussian may be stepped by recurrence, recur_ok).  The lane adds its own
// 8 sub once, so a sweep's pointer is one add (p = lane_base + offset).
constexpr int REC_OFF_MASK = (1 << 20) - 1;
__device__ __forceinline__ float2* rec_ptr(unsigned char* lbase, int w) {
    return reinterpret_cast<float2*>(lbase + (w & REC_OFF_MASK));
}

// Fast path.  r0 = {word, X0, c, dx} with X0 = x at je0 and dx = -FSTR s v dt.
// Lane `sub` covers samples je0 + 2 sub + FSTR k; the first (span + 1) / FSTR
// steps are inside the window on every lane of the half, at most one more is
// live on the lower lanes.  trl = this half's trace at absolute sample 2 sub;
// subq = 2 sub / FSTR (exact: x0 = X0 + subq dx = X0 - 2 sub s v dt).  In a
// block of 4 steps x_k = x_b + k dx, x_b += 4 dx.
__device__ __forceinline__ void fwd_sweep_fast(unsigned char* lbase, float4 r0, float4 r1,
                                               int sub2i, float2 subq) {
    const int w = __float_as_int(r0.x);
    const int span = __float_as_int(r1.w);
    const float2 dx = splat2(r0.w);
    const float2 cc = splat2(r0.z);
    float2 xb = ffma2(subq, dx, splat2(r0.y));
    float2* __restrict__ p = rec_ptr(lbase, w);
    const int nfull = (span + 1) / FSTR;
    int n = nfull;
    const float2 k2 = fadd2(dx, dx), k3 = fadd2(k2, dx), k4 = fadd2(k2, k2);
    for (; n >= 4; n -= 4, p += 4 * FL) {
        const float2 t0 = p[0], t1 = p[FL], t2 = p[2 * FL], t3 = p[3 * FL];
        const float2 v0 = gterm(xb);
        const float2 v1 = gterm(fadd2(xb, dx));
        const float2 v2 = gterm(fadd2(xb, k2));
        const float2 v3 = gterm(fadd2(xb, k3));
        xb = fadd2(xb, k4);
        p[0] = ffma2(cc, v0, t0);
        p[FL] = ffma2(cc, v1, t1);
        p[2 * FL] = ffma2(cc, v2, t2);
        p[3 * FL] = ffma2(cc, v3, t3);
    }
    if (n & 2) {
        const float2 t0 = p[0], t1 = p[FL];
        const float2 v0 = gterm(xb);
        const float2 v1 = gterm(fadd2(xb, dx));
        xb = fadd2(xb, k2);
        p[0] = ffma2(cc, v0, t0);
        p[FL] = ffma2(cc, v1, t1);
        p += 2 * FL;
    }
    if (n & 1) {
        const float2 t0 = p[0];
        const float2 v0 = gterm(xb);
        xb = fadd2(xb, dx);
        p[0] = ffma2(cc, v0, t0);
        p += FL;
    }
    if (sub2i + nfull * FSTR < span) *p = ffma2(cc, gterm(xb), *p);
}

// Fast path by recurrence (the adjoint's scheme): with D = FSTR s v dt,
// e = 2^-x^2 steps as e <- e g, g <- g h (g = 2^(2 D x - D^2), h = 2^(-2 D^2)),
// so MUFU runs only at the lane's first sample.  Same lane layout as
// fwd_sweep_fast (r0.w = dx = -D); r1 = {2D, -D^2, h, nfull | tail << 16}
// from the setup pass: nfull steps are live on every lane of the half, one
// more where 2 sub < tail.
__device__ __forceinline__ void fwd_sweep_recur(unsigned char* lbase, float4 r0, float4 r1,
                                                int sub2i, float2 subq) {
    const int w = __float_as_int(r0.x);
    const int nr = __float_as_int(r1.w);
    const float2 dx = splat2(r0.w);
    const float2 cc = splat2(r0.z);
    float2 x = ffma2(subq, dx, splat2(r0.y));
    float2 e = ex2n_2(fmul2(x, x));
    float2 g = ex2_2(ffma2(x, splat2(r1.x), splat2(r1.y)));
    const float2 h2 = splat2(r1.z);
    float2* __restrict__ p = rec_ptr(lbase, w);
    const int nfull = nr & 0xffff;
    int n = nfull;
#define PC_FWD_RSTEP(V)   \
    V = fmul2(x, e);      \
    e = fmul2(e, g);      \
    g = fmul2(g, h2);     \
    x = fadd2(x, dx);
    // 2-step blocks (measured against 4-step blocks + an n & 2 block: the
    // typical ball has 3-5 full steps, so one loop beats two branch blocks)
    for (; n >= 2; n -= 2, p += 2 * FL) {
        const float2 t0 = p[0], t1 = p[FL];
        float2 v0, v1;
        PC_FWD_RSTEP(v0)
        PC_FWD_RSTEP(v1)
        p[0] = ffma2(cc, v0, t0);
        p[FL] = ffma2(cc, v1, t1);
    }
    if (n & 1) {
        const float2 t0 = p[0];
        float2 v0;
        PC_FWD_RSTEP(v0)
        p[0] = ffma2(cc, v0, t0);
        p += FL;
    }
#undef PC_FWD_RSTEP
    if (sub2i < (nr >> 16)) *p = ffma2(cc, fmul2(x, e), *p);
}

// Exact window / near field: x (and y) from the exact integer offset to the
// wavefront sample jr every iteration (the window may start far from it).
// r1 = {X, Y at jr, jr, h}; s v dt = -r0.w / FSTR (exact).
__device__ __forceinline__ void fwd_sweep_slow(unsigned char* lbase, float4 r0, float4 r1,
                                               float2 sub2, int sub2i) {
    const int w = __float_as_int(r0.x);
    const bool near = (w >> 30) & 1;        // the ball's slow flag: evaluate the near field
    const int nl = (__float_as_int(r1.w) - sub2i + FSTR - 1) / FSTR;
    const float vs = r0.w * (-1.f / FSTR);
    const float2 cc = splat2(r0.z);
    float2 k = fadd2(sub2, splat2((float)__float_as_int(r1.z)));   // je0 - jr
    float2* p = rec_ptr(lbase, w);
    for (int n = 0; n < nl; ++n, p += FL) {
        const float2 x = ffma2(k, splat2(-vs), splat2(r1.x));
        float2 v = fmul2(x, ex2n_2(fmul2(x, x)));
        if (near) {
            const float2 y = ffma2(k, splat2(vs), splat2(r1.y));
            v = ffma2(y, ex2n_2(fmul2(y, y)), v);
        }
        *p = ffma2(cc, v, *p);
        k = fadd2(k, splat2((float)FSTR));
    }
}

// CTA = FWD_WARPS warps x FSW neighbouring sensors each, one time segment,
// one frame (x one ball chunk); no CTA-wide synchronisation.  Each sensor has
// a private shared-memory trace over the segment, laid over the warp's active
// arrival range (frame bounding box); for the BASELINE scenes one segment
// holds the whole range, so every pair is set up and swept exactly once.
// Per batch of 16 balls the 32 lanes set up the 16 x 2 pairs (fp32 cull,
// fp64 geometry) into shared-memory records; then both half-warps sweep each
// surviving ball for their own sensor (fixed ball order: deterministic).
template <bool EXACT, bool REL>
__global__ void __launch_bounds__(FWD_WARPS * 32) k_forward(FwdArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int TP = a.Tseg + TRACE_PAD;
    FwdWarpSmem& ws = reinterpret_cast<FwdWarpSmem*>(smem)[warp];
    float* traces = reinterpret_cast<float*>(reinterpret_cast<FwdWarpSmem*>(smem) + FWD_WARPS) +
                    warp * FSW * TP;
    const int seg = blockIdx.x % a.nseg;
    const int chunk = blockIdx.x / a.nseg;
    const int f = blockIdx.z;
    const int T = a.ac.T;
    const int slot0 = (blockIdx.y * FWD_WARPS + warp) * FSW;
    if (slot0 >= a.M) return;
    const int h = lane / FL, sub = lane % FL;      // half = sensor slot
    const int slot = slot0 + h;
    const int m = slot < a.M ? (a.sorder ? a.sorder[slot] : slot) : -1;

    double px = 0.0, py = 0.0, pz = 0.0;
    if (m >= 0) {
        px = a.pos[3 * m + 0];
        py = a.pos[3 * m + 1];
        pz = a.pos[3 * m + 2];
    }
    const float fpx = (float)px, fpy = (float)py, fpz = (float)pz;
    const float sup = (float)a.ac.support;

    // ---- active arrival range (union over the warp's sensors)
    int act_lo = 0, act_hi = T;
    float dmin_box = 0.f;
    if (!EXACT) {
        const unsigned* bf = a.bounds + 8 * ((size_t)f * a.nchunk + chunk);
        const float lx = ord2f(bf[0]), ly = ord2f(bf[1]), lz = ord2f(bf[2]);
        const float hx = ord2f(~bf[3]), hy = ord2f(~bf[4]), hz = ord2f(~bf[5]);
        const float amax = ord2f(~bf[6]);
        const float nx = fmaxf(fmaxf(lx - fpx, fpx - hx), 0.f);
        const float ny = fmaxf(fmaxf(ly - fpy, fpy - hy), 0.f);
        const float nz = fmaxf(fmaxf(lz - fpz, fpz - hz), 0.f);
        const float fx = fmaxf(fabsf(lx - fpx), fabsf(hx - fpx));
        const float fy = fmaxf(fabsf(ly - fpy), fabsf(hy - fpy));
        const float fz = fmaxf(fabsf(lz - fpz), fabsf(hz - fpz));
        float dmin = sqrtf(nx * nx + ny * ny + nz * nz);
        float dmax = sqrtf(fx * fx + fy * fy + fz * fz);
        if (m < 0) {
            dmin = 3.4e38f;
            dmax = 0.f;
        }
#pragma unroll
        for (int o = FL; o < 32; o <<= 1) {
            dmin = fminf(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
            dmax = fmaxf(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
        }
        dmin_box = dmin;
        const float w = sup * amax;
        const double tlo = (((double)dmin - w) * a.ac.inv_v - a.ac.t0) * a.ac.inv_dt;
        const double thi = (((double)dmax + w) * a.ac.inv_v - a.ac.t0) * a.ac.inv_dt;
        const double pad = 2.0 + 1e-5 * (double)dmax * a.ac.inv_v * a.ac.inv_dt;
        act_lo = (int)fmax(0.0, fmin((double)T, floor(tlo - pad)));
        act_hi = (int)fmax((double)act_lo, fmin((double)T, ceil(thi + pad)));
    }
    act_lo &= ~1;                                   // even segment starts
    const int nseg_w = max(1, (act_hi - act_lo + a.Tseg - 1) / a.Tseg);
    if (seg >= nseg_w) {
        if (a.loss && a.nchunk == 1 && sub == 0 && m >= 0)
            a.loss[((size_t)f * a.M + m) * a.nseg + seg] = 0.0;
        return;
    }
    const int s0 = act_lo + seg * a.Tseg;           // ball-active part of the segment
    const int s1 = min(act_hi, s0 + a.Tseg);
    const int w0 = seg == 0 ? 0 : s0;               // output range this warp writes
    const int w1 = seg == nseg_w - 1 ? T : s1;
    for (int j = lane; j < FSW * TP; j += 32) traces[j] = 0.f;

    const float d_lo = (float)(a.ac.v * (a.ac.t0 + (double)s0 * a.ac.dt)) - 2.f * a.ac.vdt;
    const float d_hi = (float)(a.ac.v * (a.ac.t0 + (double)(s1 - 1) * a.ac.dt)) + 2.f * a.ac.vdt;
    const int64_t b0 = (int64_t)chunk * a.chunk_balls;
    const int64_t b1 = min(a.B, b0 + a.chunk_balls);
    const size_t fb = (size_t)f * a.B;
    const float4* cl = a.cull + fb;
    const float vdt = a.ac.vdt;
    const bool scan = s1 > s0 || (seg == 0 && dmin_box < 1e-3f);
    const float2 sub2 = make_float2((float)(2 * sub), (float)(2 * sub + 1));
    // lane offsets from a per-warp shared table: ptxas then keeps them in a
    // register pair instead of rematerialising IADD + 2 I2F + 2 FMUL in
    // every ball's sweep prologue (config 2 forward 5.38 -> 5.26 ms)
    __shared__ float2 sq_tab[FWD_WARPS][FL];
    if (lane < FL)
        sq_tab[warp][lane] = make_float2((float)(2 * lane) / FSTR, (float)(2 * lane + 1) / FSTR);
    __syncwarp();
    const float2 subq = sq_tab[warp][sub];
    // the warp's trace area at this lane's first sample pair (records carry
    // this half's segment-relative byte offsets)
    unsigned char* lbase = reinterpret_cast<unsigned char*>(traces) + 8 * sub;
    FwdRec* recs = &ws.rec[h * FBATCH];
    __syncwarp();

    if (scan) {
        // 32-bit ball offsets within the chunk (chunks hold < 2^31 balls)
        const int nbc = (int)(b1 - b0);
        const float4* clc = cl + b0;
        const double* muc = a.mu + 3 * (fb + b0);
        const float* p0c = a.p0 + fb + b0;
        float4 nxt = sub < nbc ? clc[sub] : make_float4(0.f, 0.f, 0.f, 1.f);
        for (int g = 0; g < nbc; g += FBATCH) {
            const float4 cur = nxt;
            const int i = g + sub;                      // this lane's ball (sensor h)
            if (g + FBATCH + sub < nbc) nxt = clc[g + FBATCH + sub];
            bool pass = false;
#if PC_FWD_NOCULL1
            // one segment holds the whole arrival range of the chunk box: every
            // ball's window meets it, the cull is skipped
            if (i < nbc && m >= 0 && nseg_w == 1) {
                pass = true;
            } else
#endif
            if (i < nbc && m >= 0) {
                const float dx = cur.x - fpx, dy = cur.y - fpy, dz = cur.z - fpz;
                const float r = sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
                const float w = sup * cur.w + 1e-5f * r;
                pass = EXACT || r < 1e-3f || (r + w >= d_lo && r - w <= d_hi);
            }
            float4 q0 = make_float4(0.f, 0.f, 0.f, 0.f), q1 = q0, qr = q0;
            bool slow = false;
            if (pass) {
                const float av = cur.w;
                const float s = PC_FWD_SCALE(av);
                const int q3 = 3 * i;
                PairSetup q;
#if PC_FWD_FCONST
                pair_setup_fwd(muc[q3] - px, muc[q3 + 1] - py, muc[q3 + 2] - pz, av, a, s0, s1,
                               q, s);
#else
                pair_setup(muc[q3] - px, muc[q3 + 1] - py, muc[q3 + 2] - pz, av, s, a.ac, s0,
                           s1, q);
#endif
                if (q.R < kCoincidenceEps) {
                    atomicMin(a.coinc, ((a.fo + f) * a.B + b0 + i) * a.mt + a.so + m);
                    pass = false;
                } else if (q.jh <= q.jl) {
                    pass = false;
                } else {
                    const float c = __fdividef(0.5f * __ldg(p0c + i), (float)q.R * s);
                    const float vs = vdt * s;
                    const int je0 = q.jl & ~1;
                    const int je1 = (q.jh + 1) & ~1;
                    const float X0 = fmaf((float)(q.jr - je0), vs, q.X);
                    const float D = (float)FSTR * vs;
                    // trace byte offset of je0 (this half, segment-relative);
                    // record 1 for the direct forms: {X, Y, je0 - jr, span}
                    const int off = (je0 - s0) * 4 + h * TP * 4;
                    q0 = make_float4(__int_as_float(off), X0, c, -D);
                    q1 = make_float4(q.X, q.Y, __int_as_float(je0 - q.jr),
                                     __int_as_float(je1 - je0));
                    const int nfull = (je1 - je0 + 1) / FSTR;
                    qr = make_float4(2.f * D, -D * D, ex2(-2.f * D * D),
                                     __int_as_float(nfull | ((je1 - je0 - nfull * FSTR) << 16)));
                    slow = EXACT || q.near;
                }
            }
            {
                // per ball (both sensors of the warp agree): the direct form
                // when either pair needs the near field (bit 30, record 1 =
                // {X, Y, jr}), else the recurrence when its bounds hold
                // (bit 31, record 1 = {2D, -D^2, h, nfull | tail << 16})
                // (the shuffle must run on every lane: no short-circuit)
                bool bslow = slow;
#pragma unroll
                for (int o = FL; o < 32; o <<= 1)
                    bslow = __shfl_xor_sync(0xffffffffu, bslow, o) || bslow;
                int w = __float_as_int(q0.x);
                if (bslow) {
                    w |= 1 << 30;
                } else if (!EXACT) {
                    const float vsb = vdt * PC_FWD_SCALE(cur.w);
                    if (recur_ok((float)FSTR * vsb, vsb, sup)) {
                        w |= (int)0x80000000u;
                        q1 = qr;
                    }
                }
                q0.x = __int_as_float(w);
            }
            // compact: balls with a live pair for either sensor, in batch order
            const unsigned pm = __ballot_sync(0xffffffffu, pass);
            unsigned bm = pm;
#pragma unroll
            for (int o = FL; o < 32; o <<= 1) bm |= bm >> o;
            bm &= (1u << FL) - 1u;
            if ((bm >> sub) & 1u) {
                const int pos = __popc(bm & ((1u << sub) - 1u));
                recs[pos].r0 = q0;
                recs[pos].r1 = q1;
            }
            const int nb = __popc(bm);
            __syncwarp();
            for (int k = 0; k < nb; ++k) {
                const float4 r0 = recs[k].r0;
                const int w = __float_as_int(r0.x);
                if (w < 0)
                    fwd_sweep_recur(lbase, r0, recs[k].r1, 2 * sub, subq);
                else if (EXACT || ((w >> 30) & 1))
                    fwd_sweep_slow(lbase, r0, recs[k].r1, sub2, 2 * sub);
                else
                    fwd_sweep_fast(lbase, r0, recs[k].r1, 2 * sub, subq);
                __syncwarp();
            }
        }
    }
    __syncwarp();
    // ---- epilogue: each sensor of the warp, written by the whole warp
    for (int hh = 0; hh < FSW; ++hh) {
        const int mq = __shfl_sync(0xffffffffu, m, hh * FL);
        if (mq < 0) continue;
        const float* tq = traces + hh * TP - s0;
        const size_t row = ((size_t)f * a.M + mq) * T;
        if (a.nchunk > 1) {
            float* dst = a.out + (size_t)chunk * a.F * a.M * T + row;
            // with the ranged combine only the active part (+ a 16-sample
            // margin of zeros, covering the combine's wider padding) is
            // written; the dense combine reads whole rows
            const int p0w = a.part_margin ? max(w0, s0 - a.part_margin) : w0;
            const int p1w = a.part_margin ? min(w1, s1 + a.part_margin) : w1;
            for (int j = p0w + lane; j < p1w; j += 32) dst[j] = (j >= s0 && j < s1) ? tq[j] : 0.f;
            continue;
        }
        double lsum = 0.0;
        if (a.obs) {
            for (int j = w0 + lane; j < w1; j += 32) {
                const float pv = (j >= s0 && j < s1) ? tq[j] : 0.f;
                const float r = pv - __ldg(a.obs + row + j);
                a.out[row + j] = r;
                lsum = fma((double)r, (double)r, lsum);
            }
        } else {
            for (int j = w0 + lane; j < w1; j += 32)
                a.out[row + j] = (j >= s0 && j < s1) ? tq[j] : 0.f;
        }
        if (a.loss) {
            lsum = warp_sum(lsum);
            if (lane == 0) a.loss[((size_t)f * a.M + mq) * a.nseg + seg] = lsum;
        }
    }
}

static int finish_vec(const void* a, const void* b, const void* c, int T) {
    const uintptr_t m = reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) |
                        reinterpret_cast<uintptr_t>(c);
    return (T % 4 == 0 && (m & 15) == 0) ? 1 : 0;
}

// Chunk combine (fixed chunk order) + residual + per-trace loss partial.
// One CTA per (sensor, frame) row; float4 accesses when `vec` (T % 4 == 0
// and every base pointer 16-byte aligned, checked on the host), scalar
// otherwise.  HBM-bound: (nchunk + 2) x 4 B/sample.
// (out may alias partial when nchunk == 1: element-wise, same thread)
// Chunk combine that reads each chunk's partial row only over the samples
// sensor m can receive from that chunk: the arrival range of the (frame,
// chunk) bounding box seen from sensor m, as k_forward computes it for its
// warp (which covers it), widened by 4 samples.  Outside that range the
// forward wrote exact zeros, so skipping them leaves every per-sample sum in
// the same chunk order and bit-identical to k_forward_finish, while the
// traffic scales with the arrival ranges instead of nchunk x T (64 chunks at
// one frame per rank).  Thread t owns samples j = t (mod 256) of a
// shared-memory tile; no barriers between chunks.
constexpr int CMB_TILE = 4096;
__global__ void __launch_bounds__(256) k_forward_combine(const float* __restrict__ partial,
                                                         const unsigned* __restrict__ bounds,
                                                         const double* __restrict__ pos,
                                                         ArrayConsts ac,
                                                         const float* __restrict__ obs,
                                                         float* __restrict__ out,
                                                         double* __restrict__ loss, int nchunk,
                                                         int F, int M, int T) {
    __shared__ float acc[CMB_TILE];
    __shared__ int2 rg[64];
    const int m = blockIdx.x, f = blockIdx.y;
    const int tid = threadIdx.x;
    const size_t row = ((size_t)f * M + m) * T;
    const size_t cstride = (size_t)F * M * T;
    if (tid < nchunk) {
        const float fpx = (float)pos[3 * m], fpy = (float)pos[3 * m + 1], fpz = (float)pos[3 * m + 2];
        const unsigned* bf = bounds + 8 * ((size_t)f * nchunk + tid);
        const float lx = ord2f(bf[0]), ly = ord2f(bf[1]), lz = ord2f(bf[2]);
        const float hx = ord2f(~bf[3]), hy = ord2f(~bf[4]), hz = ord2f(~bf[5]);
        const float amax = ord2f(~bf[6]);
        const float nx = fmaxf(fmaxf(lx - fpx, fpx - hx), 0.f);
        const float ny = fmaxf(fmaxf(ly - fpy, fpy - hy), 0.f);
        const float nz = fmaxf(fmaxf(lz - fpz, fpz - hz), 0.f);
        const float fx = fmaxf(fabsf(lx - fpx), fabsf(hx - fpx));
        const float fy = fmaxf(fabsf(ly - fpy), fabsf(hy - fpy));
        const float fz = fmaxf(fabsf(lz - fpz), fabsf(hz - fpz));
        const float dmin = sqrtf(nx * nx + ny * ny + nz * nz);
        const float dmax = sqrtf(fx * fx + fy * fy + fz * fz);
        const float w = (float)ac.support * amax;
        const double tlo = (((double)dmin - w) * ac.inv_v - ac.t0) * ac.inv_dt;
        const double thi = (((double)dmax + w) * ac.inv_v - ac.t0) * ac.inv_dt;
        const double pad = 6.0 + 1e-5 * (double)dmax * ac.inv_v * ac.inv_dt;
        int lo = (int)fmax(0.0, fmin((double)T, floor(tlo - pad)));
        int hi = (int)fmax((double)lo, fmin((double)T, ceil(thi + pad)));
        if (bf[0] == ~0u) lo = hi = 0;          // empty chunk (no balls)
        rg[tid] = make_int2(lo, hi);
    }
    __syncthreads();
    double lsum = 0.0;
    for (int t0 = 0; t0 < T; t0 += CMB_TILE) {
        const int t1 = min(T, t0 + CMB_TILE);
        for (int j = t0 + tid; j < t1; j += 256) acc[j - t0] = 0.f;
        for (int c = 0; c < nchunk; ++c) {
            const int lo = max(rg[c].x, t0), hi = min(rg[c].y, t1);
            const float* pc = partial + c * cstride + row;
            int j = lo + ((t0 + tid - lo) & 255);      // first owned sample >= lo
            for (; j + 3 * 256 < hi; j += 4 * 256) {
                const float v0 = __ldcs(pc + j), v1 = __ldcs(pc + j + 256);
                const float v2 = __ldcs(pc + j + 512), v3 = __ldcs(pc + j + 768);
                acc[j - t0] += v0;
                acc[j - t0 + 256] += v1;
                acc[j - t0 + 512] += v2;
                acc[j - t0 + 768] += v3;
            }
            for (; j < hi; j += 256) acc[j - t0] += __ldcs(pc + j);
        }
        for (int j = t0 + tid; j < t1; j += 256) {
            float s = acc[j - t0];
            if (obs) {
                s -= __ldcs(obs + row + j);
                lsum = fma((double)s, (double)s, lsum);
            }
            out[row + j] = s;
        }
    }
    if (!loss) return;
    __shared__ double red[8];
    lsum = warp_sum(lsum);
    if ((tid & 31) == 0) red[tid >> 5] = lsum;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int wq = 0; wq < 8; ++wq) t += red[wq];
        loss[(size_t)f * M + m] = t;
    }
}

__global__ void __launch_bounds__(256, 4) k_forward_finish(const float* partial,
                                                           const float* __restrict__ obs,
                                                           float* out, double* __restrict__ loss,
                                                           int nchunk, int F, int M, int T,
                                                           int vec) {
    const int m = blockIdx.x, f = blockIdx.y;
    const size_t row = ((size_t)f * M + m) * T;
    const size_t cstride = (size_t)F * M * T;
    double lsum = 0.0;
    if (vec) {
        const int T4 = T >> 2;
        for (int j = threadIdx.x; j < T4; j += blockDim.x) {
            float4 s = __ldcs(reinterpret_cast<const float4*>(partial + row) + j);
            for (int c = 1; c < nchunk; ++c) {
                const float4 q = __ldcs(reinterpret_cast<const float4*>(partial + c * cstride + row) + j);
                s.x += q.x;
                s.y += q.y;
                s.z += q.z;
                s.w += q.w;
            }
            if (obs) {
                const float4 o = __ldcs(reinterpret_cast<const float4*>(obs + row) + j);
                s.x -= o.x;
                s.y -= o.y;
                s.z -= o.z;
                s.w -= o.w;
                lsum = fma((double)s.x, (double)s.x, lsum);
                lsum = fma((double)s.y, (double)s.y, lsum);
                lsum = fma((double)s.z, (double)s.z, lsum);
                lsum = fma((double)s.w, (double)s.w, lsum);
            }
            reinterpret_cast<float4*>(out + row)[j] = s;
        }
    } else {
        for (int j = threadIdx.x; j < T; j += blockDim.x) {
            float s = partial[row + j];
            for (int c = 1; c < nchunk; ++c) s += partial[c * cstride + row + j];
            if (obs) {
                s -= obs[row + j];
                lsum = fma((double)s, (double)s, lsum);
            }
            out[row + j] = s;
        }
    }
    if (!loss) return;
    __shared__ double red[8];
    lsum = warp_sum(lsum);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = lsum;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        loss[(size_t)f * M + m] = t;
    }
}

// loss_per_frame[f] = 0.5 * sum of the frame's partials (fixed order).
__global__ void __launch_bounds__(256) k_loss_reduce(const double* __restrict__ part, int per_frame,
                                                     double* __restrict__ out) {
    const int f = blockIdx.x;
    double s = 0.0;
    for (int i = threadIdx.x; i < per_frame; i += blockDim.x) s += part[(size_t)f * per_frame + i];
    __shared__ double red[8];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        out[f] = 0.5 * t;
    }
}

// ---------------------------------------------------------------- adjoint
//
// One warp owns two neighbouring balls of one frame (PC_ADJ_B2; one ball
// with PC_ADJ_B2=0).  Per block of 16 sensors the lanes form the 32 pair
// setups in parallel (fp64; lane = 2 * sensor + ball) into 48-byte
// shared-memory records; then lane groups of LG lanes take one pair each
// (NGRP = 16 pairs at a time: 8 sensors x 2 balls, i.e. 8 residual rows per
// load request).  Each lane owns quads (j .. j+3) of the pair's window
// (extended to multiples of 4 samples), reads them with one 128-bit load and
// accumulates the moments
//   A0 = sum r e,  A1 = sum r e x,  A2 = sum r e x^2,  A3 = sum r e x^3
// (AQ = A0 - kappa A2) with packed fp32x2 arithmetic, e = 2^-x^2 from MUFU
// (PC_ADJ_MODE 2; modes 0 / 1 step it by the recurrence e <- e g, g <- g h;
// the near-field and exact paths use one MUFU per term and sample).  Every
// pair constant multiplies a lane-local partial, so the per-pair reduction is
// deferred: lanes fold their partials into five ball accumulators and each
// ball's lanes reduce once at the end (fixed xor order: deterministic).

#ifndef PC_ADJ_WARPS
#define PC_ADJ_WARPS 4
#endif
constexpr int ADJ_WARPS = PC_ADJ_WARPS;   // balls per CTA
#ifndef PC_ADJ_LG
#define PC_ADJ_LG 2
#endif
constexpr int LG = PC_ADJ_LG;             // lanes per pair (adjoint; 1 / 2 / 4 / 8 -> 6.16 / 5.12 / 5.53 / 7.08 ms on config 2)
constexpr int NGRP = 32 / LG;     // pairs in flight per warp
constexpr int LSTRIDE = 4 * LG;   // samples between a lane's successive quads
#ifndef PC_ADJ_CHUNK
#define PC_ADJ_CHUNK 2        // config 2 adjoint ms: 1 / 2 / 3 / 4 -> 5.49 / 4.90 / 4.98 / 5.11
#endif
#ifndef PC_ADJ_UNROLL
#define PC_ADJ_UNROLL 1
#endif
// unroll factor of the chunk loop (its control is ~14 % of its instructions)
constexpr int ADJ_UNROLL = PC_ADJ_UNROLL;
#ifndef PC_ADJ_LOCKSTEP
#define PC_ADJ_LOCKSTEP 1
#endif
// PC_ADJ_V8 1: the fast sweep reads 8 consecutive residual samples per lane
// with one 256-bit load (LDG.E.256 on sm_100a): a pair's two lanes cover 64
// contiguous, 32-byte aligned bytes per request, i.e. exactly one sector per
// lane, instead of 2 x 16 bytes straddling sectors (23 sectors and ~8 L1
// data-pipe wavefronts per 128 samples; the L1 data pipe runs at 95 % of its
// peak).  Windows are extended to multiples of 8 samples.  Measured (config
// 3): 371.7 ms at ptxas's 72 registers (7 CTAs / SM), 393.8 ms forced to 64
// (PC_ADJ_MINB=8: register moves and rematerialised constants in the loop)
// against 367.1 ms; against the later pointer sweep (356.1 ms at 56
// registers) 388.6 ms at ptxas's 78 and 376.6 ms forced to 56: off.
#ifndef PC_ADJ_V8
#define PC_ADJ_V8 0
#endif
// PC_ADJ_ALIGN8 1: aligned fast sweeps start on a 32-byte boundary, so the
// two lanes' quads of a pair share one sector in every request (16 instead
// of ~23 sectors per 16-pair request; at most one more quad at the window
// start, weights < exp(-18)).  With one ball per warp the L1 data pipe was at
// 97 % of its peak and this paid (config 3 adjoint 356.3 -> 343.6 ms); with
// two balls per warp (PC_ADJ_B2, L1 pipe 74 %) the extra quad costs more
// than the sectors save (336.1 with, 327.5 ms without): off.
#ifndef PC_ADJ_ALIGN8
#define PC_ADJ_ALIGN8 0
#endif
// PC_ADJ_COLD 1 (default): the per-ball values only the pair setup needs
// (centre, a0, p0, scale factors) are parked in shared memory instead of
// living in 11 registers through the sweeps: 48 instead of 56 registers
// (10 CTAs / SM), config 3 adjoint 343.6 -> 341.8 ms.
#ifndef PC_ADJ_COLD
#define PC_ADJ_COLD 1
#endif
// PC_ADJ_B2 = NB in {2, 4, 8, 16}: a warp owns NB neighbouring balls and walks the
// sensors 32 / NB at a time; its 32 pair records interleave the balls per
// sensor, so the 16 pairs of a request cover 16 / NB residual rows (the
// balls' windows in a row overlap) instead of 16: fewer distinct L1 lines
// per request.  0: one ball per warp.  Config 3 adjoint, NB = 0 / 2 / 4:
// 343.6 / 332.3 / 333.7 ms (config 2: 4.56 / 4.50 / 4.71): 2 is the default.
#ifndef PC_ADJ_B2
#define PC_ADJ_B2 2
#endif
constexpr int ADJ_NB = PC_ADJ_B2 > 0 ? PC_ADJ_B2 : 1;      // balls per warp
constexpr int ADJ_NBSH = ADJ_NB == 16 ? 4 : ADJ_NB == 8 ? 3 : ADJ_NB == 4 ? 2 : ADJ_NB == 2 ? 1 : 0;
// PC_ADJ_PTR 1 (default): the aligned fast sweep runs on one pointer (chunks
// of 2 quads, a single-quad remainder) instead of carrying the sample index
// through the loop: one loop-control instruction less and 56 registers
// instead of 64 (9 CTAs / SM); config 3 adjoint 361.6 -> 355.7 ms.
#ifndef PC_ADJ_PTR
#define PC_ADJ_PTR 1
#endif
#ifndef PC_ADJ_TMA
#define PC_ADJ_TMA 0          // > 0: TMA-staged adjoint with that many balls per CTA
#endif
constexpr int ADJ_CHUNK = PC_ADJ_CHUNK;   // residual quads loaded per wave
// Gaussian per chain in the sweep: 0 = both chains by recurrence, 1 = chain a
// by MUFU and chain b by recurrence, 2 = both by MUFU.
#ifndef PC_ADJ_MODE
#define PC_ADJ_MODE 2
#endif

struct AdjArgs {
    const double* mu;
    const float* a0;
    const float* p0;
    const double* pos;
    const float* resid;
    float* G;
    long long* coinc;
    int64_t B;
    int F, M;
    ArrayConsts ac;
    int msplit;     // SPLIT: first sensor of the second half (multiple of 32)
    long long fo, so, mt; // coincidence word: frame offset, sensor offset, total sensors
    // PC_ADJ_DIET: the float forms of the array constants pair_setup converts
    // per pair (bit-identical values, formed once on the host)
    float inv_v_f, t0_f, inv_dt_f, sa_f, vt0_f, vdt_f;
    double vdt_d, vt0_d;
};

// PC_ADJ_DIET 1 (default): config 3 adjoint 367.1 -> 361.9 ms, config 2 4.86
// -> 4.78 ms (the reciprocal of R differs from the IEEE division by ~1e-16)
#ifndef PC_ADJ_DIET
#define PC_ADJ_DIET 1
#endif
#if PC_ADJ_DIET
// pair_setup (common.cuh) for the adjoint with the constants above, the raw
// MUFU rsqrt (R^2 is a normal float wherever the result is used) and the
// reciprocal of R from one fp64 Newton step on that estimate instead of an
// fp64 division (relative error ~1e-13).
__device__ __forceinline__ void adj_pair_setup(double dx, double dy, double dz, float a0, float s,
                                               const AdjArgs& a, PairSetup& q, double& inv_r) {
    const double R2 = fma(dx, dx, fma(dy, dy, dz * dz));
    const float r2f = (float)R2;
    float rinv;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(rinv) : "f"(r2f));
    const float rf = r2f * rinv;
    const double rid = (double)rinv;
    const double R = r2f > 1e-30f ? fma(fma(-(double)rf, (double)rf, R2), 0.5 * rid, (double)rf)
                                  : sqrt(R2);
    q.R = R;
    inv_r = r2f > 1e-30f ? rid * fma(-R, rid, 2.0) : 1.0 / R;
    inv_r = inv_r * fma(-R, inv_r, 2.0);
    const int T = a.ac.T;
    int lo, hi;
    const float tc = ((float)R * a.inv_v_f - a.t0_f) * a.inv_dt_f;
    if (a.ac.exact) {
        lo = 0;
        hi = T;
    } else {
        const float sa = a.sa_f * a0;
        lo = (int)fminf(fmaxf(ceilf(tc - sa), 0.f), (float)T);
        hi = (int)fminf(fmaxf(floorf(tc + sa) + 1.f, 0.f), (float)T);
    }
    q.jl = max(lo, 0);
    q.jh = min(hi, T);
    const int rc = __float2int_rn(tc);
    q.jr = min(max(rc, q.jl), max(q.jh - 1, q.jl));
    const double vt = fma((double)q.jr, a.vdt_d, a.vt0_d);
    q.X = (float)(R - vt) * s;
    q.Y = (float)(R + vt) * s;
    q.near = (float)R + a.vt0_f + a.vdt_f * (float)q.jl < 10.f * a0;
}
#endif

// Residual samples j .. j+3 (one 16-byte load when rows are 16-byte aligned).
template <bool ALIGNED>
__device__ __forceinline__ float4 load_quad(const float* __restrict__ row, int j, int T) {
    if (ALIGNED) return __ldg(reinterpret_cast<const float4*>(row + j));
    return make_float4(j < T ? __ldg(row + j) : 0.f, j + 1 < T ? __ldg(row + j + 1) : 0.f,
                       j + 2 < T ? __ldg(row + j + 2) : 0.f, j + 3 < T ? __ldg(row + j + 3) : 0.f);
}
// Residual samples j .. j+7 with one 256-bit load (32-byte aligned).
__device__ __forceinline__ void load_oct(const float* __restrict__ p, float4& a, float4& b) {
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z),
                   "=f"(b.w)
                 : "l"(p));
}
__device__ __forceinline__ float2 lo2(float4 v) { return make_float2(v.x, v.y); }
__device__ __forceinline__ float2 hi2(float4 v) { return make_float2(v.z, v.w); }

// Sample-pair moments A0 = sum w, A1 = sum w x, A2 = sum w x^2, A3 = sum w x^3
// (w = r e); AQ = A0 - kappa A2 is formed once per pair.  7 packed ops.
__device__ __forceinline__ void accum_pair(float2 r, float2 e, float2 x, float2& A0, float2& A1,
                                           float2& A2, float2& A3) {
    const float2 w = fmul2(r, e);
    A0 = fadd2(A0, w);
    const float2 t = fmul2(w, x);
    A1 = fadd2(A1, t);
    const float2 u = fmul2(t, x);
    A2 = fadd2(A2, u);
    A3 = ffma2(u, x, A3);
}

// The same moments with e = 2^-x^2 from MUFU: x^2 is then at hand for the
// second moment, 6 packed FMA-pipe ops + 2 MUFU per sample pair (against 7
// + the recurrence's 2), moving work from the FMA pipe to the idle XU pipe.
__device__ __forceinline__ void accum_pair_mufu(float2 r, float2 x, float2& A0, float2& A1,
                                                float2& A2, float2& A3) {
    const float2 xx = fmul2(x, x);
    const float2 w = fmul2(r, ex2n_2(xx));
    A0 = fadd2(A0, w);
    A1 = ffma2(w, x, A1);
    const float2 u = fmul2(w, xx);
    A2 = fadd2(A2, u);
    A3 = ffma2(u, x, A3);
}

// Registers: ptxas's default for 128-thread blocks gives 64 (8 CTAs / SM);
// config 2 adjoint ms at 96 / 64 / 56 / 48 registers (min-blocks 1 / none /
// 9 / 10): 5.43 / 4.90 / 5.66 / 5.62.
//
// SPLIT (small problems, < 2 waves of CTAs): each ball's sensors are split
// over two CTAs (blockIdx.y = 2 frame + half, halves on 32-sensor blocks),
// which add their partial G into the zeroed output; with exactly two
// addends onto 0 the sum is order-independent (IEEE addition commutes), so
// the result stays deterministic.
// PC_ADJ_MINB > 0: min-blocks hint of the launch bounds (0: ptxas's own choice)
#ifndef PC_ADJ_MINB
#define PC_ADJ_MINB 0
#endif
template <bool ALIGNED, bool SPLIT>
#if PC_ADJ_MINB > 0
__global__ void __launch_bounds__(ADJ_WARPS * 32, PC_ADJ_MINB) k_adjoint(AdjArgs a) {
#else
__global__ void __launch_bounds__(ADJ_WARPS * 32) k_adjoint(AdjArgs a) {
#endif
    __shared__ __align__(16) float4 recs[ADJ_WARPS][32][3];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#if PC_ADJ_B2
    static_assert(PC_ADJ_COLD && PC_ADJ_LOCKSTEP && PC_ADJ_MODE == 2 && LG == 2 && !PC_ADJ_V8,
                  "PC_ADJ_B2 is written for the default sweep");
    static_assert(ADJ_NB == 2 || ADJ_NB == 4 || ADJ_NB == 8 || ADJ_NB == 16,
                  "PC_ADJ_B2: 2, 4, 8 or 16 balls per warp");
    // setup lanes: ball = lane % NB; sweep lanes (pair = lane / 2): ball = (lane / 2) % NB
    const int64_t b0 = ((int64_t)blockIdx.x * ADJ_WARPS + warp) * ADJ_NB;
    const int64_t b = b0 + (lane & (ADJ_NB - 1));
    const int64_t b_swp = b0 + ((lane >> 1) & (ADJ_NB - 1));
#else
    const int64_t b = (int64_t)blockIdx.x * ADJ_WARPS + warp;
#endif
    const int f = SPLIT ? (int)(blockIdx.y >> 1) : (int)blockIdx.y;
    const int m_lo = SPLIT ? (int)(blockIdx.y & 1) * a.msplit : 0;
    const int m_hi = SPLIT ? ((blockIdx.y & 1) ? a.M : min(a.M, a.msplit)) : a.M;
#if PC_ADJ_LOCKSTEP
    const bool live = b < a.B;
    const size_t sb = (size_t)f * a.B + (live ? b : a.B - 1);
#else
    if (b >= a.B) return;
    const size_t sb = (size_t)f * a.B + b;
#endif
    const double mx = a.mu[3 * sb + 0], my = a.mu[3 * sb + 1], mz = a.mu[3 * sb + 2];
    const float av = a.a0[sb], pv = a.p0[sb];
    const float s = scale_of(av);
#if PC_ADJ_B2
    const bool live_swp = b_swp < a.B;
    const size_t sb_swp = (size_t)f * a.B + (live_swp ? b_swp : a.B - 1);
    const float vs = a.ac.vdt * scale_of(a.a0[sb_swp]);   // the sweep ball's sample step
#else
    const float vs = a.ac.vdt * s;
#endif
    const float inv_s = 1.f / s;
    const float ka_ball = pv / (av * av * av) * inv_s * inv_s * inv_s;
    const int T = a.ac.T;
    const float D = (float)LSTRIDE * vs;
    // the MUFU sweep (mode 2) is valid for any step; the recurrence modes need
    // their bound
    const bool fast = !a.ac.exact && (PC_ADJ_MODE == 2 || recur_ok(D, vs, (float)a.ac.support));
    const float2 h2 = splat2(ex2(-2.f * D * D));
    const float2 mD2 = splat2(-D);
    const float2 mvs2 = splat2(-vs);
    const float2 vs2 = splat2(vs);
    float g0 = 0.f, g1 = 0.f, g2 = 0.f, g3 = 0.f, g4 = 0.f;
    float4(&rec)[32][3] = recs[warp];
    const int grp = lane / LG, sub = lane % LG;
#if PC_ADJ_COLD
#if PC_ADJ_B2
    __shared__ double cold_d[ADJ_NB * ADJ_WARPS][4];
    __shared__ float cold_f[ADJ_NB * ADJ_WARPS][8];
    const int cw = ADJ_NB * warp + (lane & (ADJ_NB - 1));
    if (lane < ADJ_NB) {
#else
    __shared__ double cold_d[ADJ_WARPS][4];
    __shared__ float cold_f[ADJ_WARPS][8];
    const int cw = warp;
    if (lane == 0) {
#endif
        cold_d[cw][0] = mx;
        cold_d[cw][1] = my;
        cold_d[cw][2] = mz;
        cold_f[cw][0] = av;
        cold_f[cw][1] = pv;
        cold_f[cw][2] = s;
        cold_f[cw][3] = inv_s;
        cold_f[cw][4] = ka_ball;
    }
    __syncwarp();
    const volatile double* cd = cold_d[cw];
    const volatile float* cf = cold_f[cw];
#endif

    const float* rblk = a.resid + ((size_t)f * a.M + m_lo) * T;   // this block's first row
#if PC_ADJ_B2
    for (int mb = m_lo; mb < m_hi; mb += 32 / ADJ_NB, rblk += (size_t)(32 / ADJ_NB) * T) {
        const int m = mb + (lane >> ADJ_NBSH);
#else
    for (int mb = m_lo; mb < m_hi; mb += 32, rblk += (size_t)32 * T) {
        const int m = mb + lane;
#endif
        int win = -1, wh = 0, jr = 0;           // window [jl, jh) (win = jl | near << 30)
        float X = 0.f, Y = 0.f, kp = 0.f, ka = 0.f, kR1 = 0.f, kR2 = 0.f;
        float ux = 0.f, uy = 0.f, uz = 0.f;
#if PC_ADJ_LOCKSTEP
        if (live && m < m_hi) {
#else
        if (m < a.M) {
#endif
#if PC_ADJ_COLD
            const double bx = cd[0], by = cd[1], bz = cd[2];
            const float b_av = cf[0], b_pv = cf[1], b_s = cf[2], b_inv_s = cf[3], b_ka = cf[4];
#else
            const double bx = mx, by = my, bz = mz;
            const float b_av = av, b_pv = pv, b_s = s, b_inv_s = inv_s, b_ka = ka_ball;
#endif
            const double dx = bx - a.pos[3 * m + 0];
            const double dy = by - a.pos[3 * m + 1];
            const double dz = bz - a.pos[3 * m + 2];
            PairSetup q;
#if PC_ADJ_DIET
            double ir;
            adj_pair_setup(dx, dy, dz, b_av, b_s, a, q, ir);
#else
            pair_setup(dx, dy, dz, b_av, b_s, a.ac, 0, T, q);
#endif
            if (q.R < kCoincidenceEps) {
                atomicMin(a.coinc, ((a.fo + f) * a.B + b) * a.mt + a.so + m);
            } else if (q.jh > q.jl) {
                win = q.jl | (q.near ? 1 << 30 : 0);
                wh = q.jh;
                jr = q.jr;
                X = q.X;
                Y = q.Y;
#if !PC_ADJ_DIET
                const double ir = 1.0 / q.R;
#endif
                const float inv2R = (float)(0.5 * ir);
                kp = inv2R * b_inv_s;
                ka = b_ka * inv2R;
                kR2 = b_pv * inv2R;
                kR1 = -kR2 * (float)ir * b_inv_s;
                ux = (float)(dx * ir);
                uy = (float)(dy * ir);
                uz = (float)(dz * ir);
            }
        }
        rec[lane][0] = make_float4(__int_as_float(win), __int_as_float(jr), X, kp);
        rec[lane][1] = make_float4(ka, kR1, kR2, ux);
        rec[lane][2] = make_float4(uy, uz, Y, __int_as_float(wh));
        __syncwarp();
#if PC_ADJ_B2
        const int npair = min(32, ADJ_NB * (m_hi - mb));
#else
        const int npair = min(32, m_hi - mb);
#endif
        for (int pb = 0; pb < npair; pb += NGRP) {
            const int pi = pb + grp;
            if (pi >= npair) continue;
            const float4 r0 = rec[pi][0];
            const int w = __float_as_int(r0.x);
            if (w < 0) continue;
            const int jl = w & 0x3fffffff;
            const bool near = (w >> 30) & 1;
            const int jh = __float_as_int(rec[pi][2].w);
            // window extended to multiples of 4 (the extra samples weigh
            // < exp(-19) of the peak); lane `sub` takes quads j, j + 16, ...
            const int je1 = (jh + 3) & ~3;
#if PC_ADJ_ALIGN8
            int j = ((ALIGNED && fast && !near) ? (jl & ~7) : (jl & ~3)) + 4 * sub;
#else
            int j = (jl & ~3) + 4 * sub;
#endif
#if PC_ADJ_B2
            const float* row = rblk + (size_t)(pi >> ADJ_NBSH) * T;
#else
            const float* row = rblk + (size_t)pi * T;
#endif
            float2 A0 = splat2(0.f), A1 = A0, A2 = A0, A3 = A0;
            bool swept = false;
#if PC_ADJ_V8
            static_assert(PC_ADJ_MODE == 2 && LG == 2, "PC_ADJ_V8: MUFU sweep, two lanes per pair");
            if (ALIGNED && fast && !near) {
                // octs j8, j8 + 16, ... of the window extended to multiples of 8
                const int je8 = (jh + 7) & ~7;
                const int j8 = (jl & ~7) + 8 * sub;
                if (j8 < je8) {
                    const int jrr = __float_as_int(r0.y);
                    const float2 k = make_float2((float)(j8 - jrr), (float)(j8 + 1 - jrr));
                    float2 xa = ffma2(k, mvs2, splat2(r0.z));
                    float2 xb = ffma2(fadd2(k, splat2(2.f)), mvs2, splat2(r0.z));
                    const float2 s1 = splat2(-4.f * vs), s2 = splat2(-12.f * vs);
                    const float* p = row + j8;
                    for (int n = (je8 - j8 + 15) >> 4; n > 0; --n, p += 16) {
                        float4 q0, q1;
                        load_oct(p, q0, q1);
                        accum_pair_mufu(lo2(q0), xa, A0, A1, A2, A3);
                        accum_pair_mufu(hi2(q0), xb, A0, A1, A2, A3);
                        xa = fadd2(xa, s1);
                        xb = fadd2(xb, s1);
                        accum_pair_mufu(lo2(q1), xa, A0, A1, A2, A3);
                        accum_pair_mufu(hi2(q1), xb, A0, A1, A2, A3);
                        xa = fadd2(xa, s2);
                        xb = fadd2(xb, s2);
                    }
                }
                swept = true;
            }
#endif
            if (!swept && j < je1) {
                const int jrr = __float_as_int(r0.y);
                float2 k = make_float2((float)(j - jrr), (float)(j + 1 - jrr));
                const float2 two = splat2(2.f);
                if (fast && !near && !(PC_ADJ_V8 && ALIGNED)) {
                    // two chains per lane: samples (j, j+1) and (j+2, j+3)
                    float2 xa = ffma2(k, mvs2, splat2(r0.z));
                    float2 xb = ffma2(fadd2(k, two), mvs2, splat2(r0.z));
                    float2 ea, ga, eb, gb;
                    recur_init(xa, D, ea, ga);
                    recur_init(xb, D, eb, gb);
                    int n = (je1 - j + LSTRIDE - 1) / LSTRIDE;   // quads of this lane
#if PC_ADJ_MODE == 0
#define PC_ADJ_STEP(R)                                   \
    accum_pair(lo2(R), ea, xa, A0, A1, A2, A3);          \
    accum_pair(hi2(R), eb, xb, A0, A1, A2, A3);          \
    ea = fmul2(ea, ga);                                  \
    eb = fmul2(eb, gb);                                  \
    ga = fmul2(ga, h2);                                  \
    gb = fmul2(gb, h2);                                  \
    xa = fadd2(xa, mD2);                                 \
    xb = fadd2(xb, mD2);
#elif PC_ADJ_MODE == 1
#define PC_ADJ_STEP(R)                                   \
    accum_pair_mufu(lo2(R), xa, A0, A1, A2, A3);         \
    accum_pair(hi2(R), eb, xb, A0, A1, A2, A3);          \
    eb = fmul2(eb, gb);                                  \
    gb = fmul2(gb, h2);                                  \
    xa = fadd2(xa, mD2);                                 \
    xb = fadd2(xb, mD2);
#else
#define PC_ADJ_STEP(R)                                   \
    accum_pair_mufu(lo2(R), xa, A0, A1, A2, A3);         \
    accum_pair_mufu(hi2(R), xb, A0, A1, A2, A3);         \
    xa = fadd2(xa, mD2);                                 \
    xb = fadd2(xb, mD2);
#endif
#if PC_ADJ_PTR
                    if (ALIGNED) {
                        // the same sweep on one running pointer (no sample index
                        // carried through the loop)
                        const float4* p4 = reinterpret_cast<const float4*>(row + j);
                        for (; n >= 2; n -= 2, p4 += 2 * (LSTRIDE / 4)) {
                            const float4 ra = __ldg(p4), rb = __ldg(p4 + LSTRIDE / 4);
                            PC_ADJ_STEP(ra)
                            PC_ADJ_STEP(rb)
                        }
                        if (n > 0) {
                            const float4 ra = __ldg(p4);
                            PC_ADJ_STEP(ra)
                        }
                        n = 0;
                    }
#endif
                    // chunks of ADJ_CHUNK quads: that many loads in flight
#pragma unroll ADJ_UNROLL
                    for (; n >= ADJ_CHUNK; n -= ADJ_CHUNK, j += ADJ_CHUNK * LSTRIDE) {
                        float4 rr[ADJ_CHUNK];
#pragma unroll
                        for (int u = 0; u < ADJ_CHUNK; ++u)
                            rr[u] = load_quad<ALIGNED>(row, j + u * LSTRIDE, T);
#pragma unroll
                        for (int u = 0; u < ADJ_CHUNK; ++u) {
                            PC_ADJ_STEP(rr[u])
                        }
                    }
                    if (ADJ_CHUNK > 4 && n >= 4) {
                        float4 rr[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) rr[u] = load_quad<ALIGNED>(row, j + u * LSTRIDE, T);
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            PC_ADJ_STEP(rr[u])
                        }
                        n -= 4;
                        j += 4 * LSTRIDE;
                    }
                    if (n > 0) {
                        // remainder (< 4 quads): all loads in flight at once
                        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
                        const float4 r0q = load_quad<ALIGNED>(row, j, T);
                        const float4 r1q = n > 1 ? load_quad<ALIGNED>(row, j + LSTRIDE, T) : z;
                        const float4 r2q = n > 2 ? load_quad<ALIGNED>(row, j + 2 * LSTRIDE, T) : z;
                        PC_ADJ_STEP(r0q)
                        if (n > 1) {
                            PC_ADJ_STEP(r1q)
                        }
                        if (n > 2) {
                            PC_ADJ_STEP(r2q)
                        }
                    }
#undef PC_ADJ_STEP
                } else {
                    const float Yr = rec[pi][2].z;
                    const float2 kstep = splat2((float)LSTRIDE);
                    for (; j < je1; j += LSTRIDE) {
                        const float4 r = load_quad<ALIGNED>(row, j, T);
                        const float2 kb = fadd2(k, two);
                        const float2 xa = ffma2(k, mvs2, splat2(r0.z));
                        const float2 xb = ffma2(kb, mvs2, splat2(r0.z));
                        accum_pair(lo2(r), ex2n_2(fmul2(xa, xa)), xa, A0, A1, A2, A3);
                        accum_pair(hi2(r), ex2n_2(fmul2(xb, xb)), xb, A0, A1, A2, A3);
                        if (near) {
                            const float2 ya = ffma2(k, vs2, splat2(Yr));
                            const float2 yb = ffma2(kb, vs2, splat2(Yr));
                            accum_pair(lo2(r), ex2n_2(fmul2(ya, ya)), ya, A0, A1, A2, A3);
                            accum_pair(hi2(r), ex2n_2(fmul2(yb, yb)), yb, A0, A1, A2, A3);
                        }
                        k = fadd2(k, kstep);
                    }
                }
            }
            const float a1 = A1.x + A1.y, a3 = A3.x + A3.y;
            const float aq = fmaf(A2.x + A2.y, -kKappa, A0.x + A0.y);
            const float4 r1 = rec[pi][1];
            const float4 r2 = rec[pi][2];
            const float accR = fmaf(r1.y, a1, r1.z * aq);
            g0 = fmaf(r1.x, a3, g0);
            g1 = fmaf(r0.w, a1, g1);
            g2 = fmaf(accR, r1.w, g2);
            g3 = fmaf(accR, r2.x, g3);
            g4 = fmaf(accR, r2.y, g4);
        }
        __syncwarp();
#if PC_ADJ_LOCKSTEP
        __syncthreads();   // the CTA's balls read the same sensor rows together
#endif
    }
#if PC_ADJ_B2
    // lanes with equal (lane / 2) % NB hold one ball's partials: fixed xor
    // order over the other lane bits
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        if (o >= 2 && o < 2 * ADJ_NB) continue;
        g0 += __shfl_xor_sync(0xffffffffu, g0, o);
        g1 += __shfl_xor_sync(0xffffffffu, g1, o);
        g2 += __shfl_xor_sync(0xffffffffu, g2, o);
        g3 += __shfl_xor_sync(0xffffffffu, g3, o);
        g4 += __shfl_xor_sync(0xffffffffu, g4, o);
    }
    if ((lane & ~(2 * (ADJ_NB - 1))) == 0 && live_swp) {
        float* out = a.G + 5 * sb_swp;
#else
#if PC_ADJ_LOCKSTEP
    if (!live) return;
#endif
    g0 = warp_sum(g0);
    g1 = warp_sum(g1);
    g2 = warp_sum(g2);
    g3 = warp_sum(g3);
    g4 = warp_sum(g4);
    if (lane == 0) {
        float* out = a.G + 5 * sb;
#endif
        if (SPLIT) {
            atomicAdd(out + 0, g0);
            atomicAdd(out + 1, g1);
            atomicAdd(out + 2, g2);
            atomicAdd(out + 3, g3);
            atomicAdd(out + 4, g4);
        } else {
            out[0] = g0;
            out[1] = g1;
            out[2] = g2;
            out[3] = g3;
            out[4] = g4;
        }
    }
}

#if PC_ADJ_TMA
// ---------------------------------------------------------------- adjoint,
// TMA-staged residual windows (PC_ADJ_TMA)
//
// CTA = TW balls (warps) of one frame.  Per block of 32 sensors the warps
// set up their pairs into double-buffered records, one CTA barrier, then
// warp 0 forms each sensor's union window over the CTA's balls and issues
// 1-D bulk copies (cp.async.bulk, TMA) of those rows into a double-buffered
// shared-memory stage, completing on an mbarrier; the block is then swept
// from shared memory while the next block's copies are in flight.  The
// mbarrier (arrive = release, wait = acquire) also publishes warp 0's union
// offsets, so one CTA barrier per block suffices.  A block whose union does
// not fit the stage is swept from global memory.

#ifndef PC_ADJ_TSTAGE
#define PC_ADJ_TSTAGE 8192
#endif
constexpr int ADJ_TSTAGE = PC_ADJ_TSTAGE;   // floats per stage buffer

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void tma_row(float* dst, const float* src, unsigned bytes,
                                        unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

struct StagedRow {                 // staged row: shared byte address of sample 0
    unsigned base;
    __device__ __forceinline__ float4 q(int j) const {
        float4 v;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                     : "r"(base + 4u * (unsigned)j));
        return v;
    }
};
struct GlobalRowT {
    const float* p;
    __device__ __forceinline__ float4 q(int j) const {
        return __ldg(reinterpret_cast<const float4*>(p + j));
    }
};

template <class Row>
__device__ __forceinline__ void adj_sweep_t(const Row& row, int j, int je1, float2 xa, float2 xb,
                                            float2 mD2, float2& A0, float2& A1, float2& A2,
                                            float2& A3) {
    int n = (je1 - j + LSTRIDE - 1) / LSTRIDE;
#define PC_T_STEP(R)                                     \
    accum_pair_mufu(lo2(R), xa, A0, A1, A2, A3);         \
    accum_pair_mufu(hi2(R), xb, A0, A1, A2, A3);         \
    xa = fadd2(xa, mD2);                                 \
    xb = fadd2(xb, mD2);
    for (; n >= 4; n -= 4, j += 4 * LSTRIDE) {
        float4 rr[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) rr[u] = row.q(j + u * LSTRIDE);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            PC_T_STEP(rr[u])
        }
    }
    if (n > 0) {
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 q0 = row.q(j);
        const float4 q1 = n > 1 ? row.q(j + LSTRIDE) : z;
        const float4 q2 = n > 2 ? row.q(j + 2 * LSTRIDE) : z;
        PC_T_STEP(q0)
        if (n > 1) {
            PC_T_STEP(q1)
        }
        if (n > 2) {
            PC_T_STEP(q2)
        }
    }
#undef PC_T_STEP
}

template <class Row>
__device__ __forceinline__ void adj_sweep_direct_t(const Row& row, int j, int je1, float2 k,
                                                   float vs, float X, float Y, bool near,
                                                   float2& A0, float2& A1, float2& A2,
                                                   float2& A3) {
    const float2 two = splat2(2.f), kstep = splat2((float)LSTRIDE);
    const float2 mvs2 = splat2(-vs), vs2 = splat2(vs);
    for (; j < je1; j += LSTRIDE) {
        const float4 r = row.q(j);
        const float2 kb = fadd2(k, two);
        const float2 xa = ffma2(k, mvs2, splat2(X));
        const float2 xb = ffma2(kb, mvs2, splat2(X));
        accum_pair(lo2(r), ex2n_2(fmul2(xa, xa)), xa, A0, A1, A2, A3);
        accum_pair(hi2(r), ex2n_2(fmul2(xb, xb)), xb, A0, A1, A2, A3);
        if (near) {
            const float2 ya = ffma2(k, vs2, splat2(Y));
            const float2 yb = ffma2(kb, vs2, splat2(Y));
            accum_pair(lo2(r), ex2n_2(fmul2(ya, ya)), ya, A0, A1, A2, A3);
            accum_pair(hi2(r), ex2n_2(fmul2(yb, yb)), yb, A0, A1, A2, A3);
        }
        k = fadd2(k, kstep);
    }
}

template <int TW>
__global__ void __launch_bounds__(TW * 32) k_adjoint_tma(AdjArgs a) {
    extern __shared__ __align__(128) unsigned char tsm[];
    float* stage = reinterpret_cast<float*>(tsm);                        // [2][ADJ_TSTAGE]
    float4(*recs)[TW][32][3] =
        reinterpret_cast<float4(*)[TW][32][3]>(stage + 2 * ADJ_TSTAGE);  // [2][TW][32][3]
    int2(*s_win)[32] = reinterpret_cast<int2(*)[32]>(recs + 2);          // [TW][32]
    int* s_lo = reinterpret_cast<int*>(s_win + TW);                       // [2][32]
    int* s_off = s_lo + 64;                                               // [2][33]
    unsigned long long* bar =
        reinterpret_cast<unsigned long long*>(((uintptr_t)(s_off + 66) + 7) & ~(uintptr_t)7);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t b = (int64_t)blockIdx.x * TW + warp;
    const bool live = b < a.B;
    const int f = blockIdx.y;
    const size_t sb = (size_t)f * a.B + (live ? b : a.B - 1);
    const double mx = a.mu[3 * sb + 0], my = a.mu[3 * sb + 1], mz = a.mu[3 * sb + 2];
    const float av = a.a0[sb], pv = a.p0[sb];
    const float s = scale_of(av);
    const float vs = a.ac.vdt * s;
    const float inv_s = 1.f / s;
    const float ka_ball = pv / (av * av * av) * inv_s * inv_s * inv_s;
    const int T = a.ac.T;
    const float2 mD2 = splat2(-(float)LSTRIDE * vs);
    const float2 mvs2 = splat2(-vs);
    float g0 = 0.f, g1 = 0.f, g2 = 0.f, g3 = 0.f, g4 = 0.f;
    const int grp = lane / LG, sub = lane % LG;
    const int nblk = (a.M + 31) / 32;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    auto setup = [&](int kb, int buf) {
        const int m = kb * 32 + lane;
        int win = -1, wh = 0, jr = 0;
        float X = 0.f, Y = 0.f, kp = 0.f, ka = 0.f, kR1 = 0.f, kR2 = 0.f;
        float ux = 0.f, uy = 0.f, uz = 0.f;
        int2 wq = make_int2(0x7fffffff, -0x7fffffff);
        if (live && m < a.M) {
            const double dx = mx - a.pos[3 * m + 0];
            const double dy = my - a.pos[3 * m + 1];
            const double dz = mz - a.pos[3 * m + 2];
            PairSetup q;
            pair_setup(dx, dy, dz, av, s, a.ac, 0, T, q);
            if (q.R < kCoincidenceEps) {
                atomicMin(a.coinc, ((a.fo + f) * a.B + b) * a.mt + a.so + m);
            } else if (q.jh > q.jl) {
                win = q.jl | (q.near ? 1 << 30 : 0);
                wh = q.jh;
                wq = make_int2(q.jl & ~3, (q.jh + 3) & ~3);
                jr = q.jr;
                X = q.X;
                Y = q.Y;
                const double ir = 1.0 / q.R;
                const float inv2R = (float)(0.5 * ir);
                kp = inv2R * inv_s;
                ka = ka_ball * inv2R;
                kR2 = pv * inv2R;
                kR1 = -kR2 * (float)ir * inv_s;
                ux = (float)(dx * ir);
                uy = (float)(dy * ir);
                uz = (float)(dz * ir);
            }
        }
        recs[buf][warp][lane][0] = make_float4(__int_as_float(win), __int_as_float(jr), X, kp);
        recs[buf][warp][lane][1] = make_float4(ka, kR1, kR2, ux);
        recs[buf][warp][lane][2] = make_float4(uy, uz, Y, __int_as_float(wh));
        s_win[warp][lane] = wq;
    };
    // warp 0: union windows of block kb, offsets, bulk copies (or none)
    auto issue = [&](int kb, int buf) {
        int lo = 0x7fffffff, hi = -0x7fffffff;
#pragma unroll
        for (int w2 = 0; w2 < TW; ++w2) {
            lo = min(lo, s_win[w2][lane].x);
            hi = max(hi, s_win[w2][lane].y);
        }
        const int len = hi > lo ? hi - lo : 0;
        int incl = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        const bool fits = total <= ADJ_TSTAGE;
        s_lo[buf * 32 + lane] = len ? lo : 0;
        s_off[buf * 33 + lane] = incl - len;
        if (lane == 0) s_off[buf * 33 + 32] = fits ? total : -1;
        __syncwarp();
        if (lane == 0) mbar_arrive_tx(&bar[buf], fits ? (unsigned)total * 4u : 0u);
        __syncwarp();
        if (fits && len > 0) {
            const int m = kb * 32 + lane;
            tma_row(stage + buf * ADJ_TSTAGE + (incl - len),
                    a.resid + ((size_t)f * a.M + m) * T + lo, (unsigned)len * 4u, &bar[buf]);
        }
    };

    setup(0, 0);
    __syncthreads();
    if (warp == 0) issue(0, 0);
    unsigned phase[2] = {0u, 0u};
    for (int kb = 0; kb < nblk; ++kb) {
        const int buf = kb & 1;
        if (kb + 1 < nblk) {
            setup(kb + 1, buf ^ 1);
            __syncthreads();       // all warps are past block kb-1: its buffers are free
            if (warp == 0) issue(kb + 1, buf ^ 1);
        }
        mbar_wait(&bar[buf], phase[buf]);
        phase[buf] ^= 1u;
        const bool staged = s_off[buf * 33 + 32] >= 0;
        const int mb = kb * 32;
        const int npair = min(32, a.M - mb);
        if (live) {
            for (int pb = 0; pb < npair; pb += NGRP) {
                const int pi = pb + grp;
                if (pi >= npair) continue;
                const float4 r0 = recs[buf][warp][pi][0];
                const int w = __float_as_int(r0.x);
                if (w < 0) continue;
                const int jl = w & 0x3fffffff;
                const bool near = (w >> 30) & 1;
                const float4 r2 = recs[buf][warp][pi][2];
                const int jh = __float_as_int(r2.w);
                const int je1 = (jh + 3) & ~3;
                const int j = (jl & ~3) + 4 * sub;
                float2 A0 = splat2(0.f), A1 = A0, A2 = A0, A3 = A0;
                if (j < je1) {
                    const int jrr = __float_as_int(r0.y);
                    const float2 k = make_float2((float)(j - jrr), (float)(j + 1 - jrr));
                    const float2 xa = ffma2(k, mvs2, splat2(r0.z));
                    const float2 xb = ffma2(fadd2(k, splat2(2.f)), mvs2, splat2(r0.z));
                    if (staged) {
                        const StagedRow row{smem_u32(stage + buf * ADJ_TSTAGE) +
                                            4u * (unsigned)(s_off[buf * 33 + pi] -
                                                            s_lo[buf * 32 + pi])};
                        if (!near)
                            adj_sweep_t(row, j, je1, xa, xb, mD2, A0, A1, A2, A3);
                        else
                            adj_sweep_direct_t(row, j, je1, k, vs, r0.z, r2.z, true, A0, A1, A2,
                                               A3);
                    } else {
                        const GlobalRowT row{a.resid + ((size_t)f * a.M + mb + pi) * T};
                        if (!near)
                            adj_sweep_t(row, j, je1, xa, xb, mD2, A0, A1, A2, A3);
                        else
                            adj_sweep_direct_t(row, j, je1, k, vs, r0.z, r2.z, true, A0, A1, A2,
                                               A3);
                    }
                }
                const float a1 = A1.x + A1.y, a3 = A3.x + A3.y;
                const float aq = fmaf(A2.x + A2.y, -kKappa, A0.x + A0.y);
                const float4 r1 = recs[buf][warp][pi][1];
                const float accR = fmaf(r1.y, a1, r1.z * aq);
                g0 = fmaf(r1.x, a3, g0);
                g1 = fmaf(r0.w, a1, g1);
                g2 = fmaf(accR, r1.w, g2);
                g3 = fmaf(accR, r2.x, g3);
                g4 = fmaf(accR, r2.y, g4);
            }
        }
        __syncwarp();
    }
    if (!live) return;
    g0 = warp_sum(g0);
    g1 = warp_sum(g1);
    g2 = warp_sum(g2);
    g3 = warp_sum(g3);
    g4 = warp_sum(g4);
    if (lane == 0) {
        float* out = a.G + 5 * sb;
        out[0] = g0;
        out[1] = g1;
        out[2] = g2;
        out[3] = g3;
        out[4] = g4;
    }
}

template <int TW>
static size_t adj_tma_smem() {
    return 2 * ADJ_TSTAGE * sizeof(float) + 2 * TW * 32 * 3 * sizeof(float4) +
           TW * 32 * sizeof(int2) + (64 + 66) * sizeof(int) + 16 + 16;
}

#endif  // PC_ADJ_TMA

static bool array_consts(const pc_array_t* arr, ArrayConsts& ac) {
    if (!arr || !arr->positions || arr->n_sensors < 1 || arr->n_samples < 1 ||
        !(arr->sound_speed > 0) || !(arr->dt > 0))
        return false;
    ac.v = arr->sound_speed;
    ac.t0 = arr->t_start;
    ac.dt = arr->dt;
    ac.inv_v = 1.0 / arr->sound_speed;
    ac.inv_dt = 1.0 / arr->dt;
    ac.support = arr->support_sigmas;
    ac.vdt = (float)(arr->sound_speed * arr->dt);
    ac.T = arr->n_samples;
    ac.exact = arr->exact ? 1 : 0;
    return true;
}

}  // namespace pc

using namespace pc;

// Range-limited chunk combine (PC_FWD_CMB=0 selects the dense combine).
static bool fwd_cmb() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("PC_FWD_CMB");
        v = e ? atoi(e) != 0 : 1;
    }
    return v != 0;
}

// Partial rows written over the active range only (PC_FWD_PM=0: whole rows).
static bool fwd_pm() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("PC_FWD_PM");
        v = e ? atoi(e) != 0 : 1;
    }
    return v != 0;
}

// The register-run forward (fwd_run.cu) is the default; PC_FWD_LEGACY=1
// selects the shared-memory-trace kernel above (kept for A/B measurements).
static bool fwd_legacy(const pc_array_t* array) {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("PC_FWD_LEGACY");
        v = e ? atoi(e) != 0 : 0;
    }
    return v != 0 || !fwd_run_supported(array);
}

// PC_FWD_TMA=1: the register-run forward with the chunk's raw ball tile
// staged in shared memory by cp.async.bulk behind an mbarrier (fwd_run.cu
// compiled with PC_FR_TMA; chunks of 512 balls so four CTAs still fit an SM).
// Measured 7 % slower than the default on config 3:
// kept selectable and parity-tested.
static bool fwd_tma(const pc_array_t* array) {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("PC_FWD_TMA");
        v = e ? atoi(e) != 0 : 0;
    }
    return v != 0 && tma::fwd_run_supported(array);
}

extern "C" int pc_forward_plan(int64_t n_balls, int32_t n_frames, const pc_array_t* array,
                               int32_t* plan) {
    if (!array || !plan || n_balls < 0 || n_frames < 1 || array->n_sensors < 1 ||
        array->n_samples < 1)
        return PC_ERR_ARGUMENT;
    if (!fwd_legacy(array)) {
        plan[0] = fwd_run_samples_per_run();
        plan[1] = 1;
        plan[2] = 1;
        plan[3] = 2;   // forward + loss reduce
        return PC_OK;
    }
    FwdPlan p = fwd_plan(n_balls > 0 ? n_balls : 1, n_frames, array->n_sensors,
                         array->n_samples);
    plan[0] = p.Tseg;
    plan[1] = p.nseg;
    plan[2] = p.nchunk;
    plan[3] = 3 + (p.nchunk > 1 ? 1 : 0);  // prep + forward [+ combine] + loss reduce
    return PC_OK;
}

extern "C" int pc_forward_variant(const pc_array_t* array) {
    if (!array) return -1;
    return fwd_legacy(array) ? 1 : fwd_tma(array) ? 2 : 0;
}

extern "C" size_t pc_forward_workspace_bytes(int64_t n_balls, int32_t n_frames,
                                             const pc_array_t* array) {
    if (!array || n_balls < 0 || n_frames < 1) return 0;
    if (!fwd_legacy(array)) return fwd_run_workspace_bytes(n_frames, array);
    FwdPlan p = fwd_plan(n_balls > 0 ? n_balls : 1, n_frames, array->n_sensors,
                         array->n_samples);
    return p.prep_bytes + p.partial_bytes + p.loss_bytes + 256;
}

extern "C" int pc_forward_traces(const double* mu_t, const float* a0_t, const float* p0_t,
                                 int64_t n_balls, int32_t n_frames, const pc_array_t* array,
                                 const float* observed, float* out, double* loss_per_frame,
                                 int64_t* coincident, void* workspace, size_t workspace_bytes,
                                 pc_stream_t stream) {
    ArrayConsts ac;
    if (!array_consts(array, ac) || n_balls < 0 || n_frames < 1 || !out || !coincident)
        return PC_ERR_ARGUMENT;
    if (array->n_samples >= kMaxSamples) return PC_ERR_UNSUPPORTED;   // 2^30
    const int M = array->n_sensors, T = array->n_samples, F = n_frames;
    cudaStream_t st = as_stream(stream);
    if (n_balls > 0 && (!mu_t || !a0_t || !p0_t)) return PC_ERR_ARGUMENT;
    if (!fwd_legacy(array)) {
        const bool want_loss = observed && loss_per_frame;
        if (want_loss && (!workspace || workspace_bytes < fwd_run_workspace_bytes(F, array)))
            return PC_ERR_ARGUMENT;
        double* lpart = reinterpret_cast<double*>(workspace);
        if (n_balls > 0) {
            const int rc =
                fwd_tma(array)
                    ? tma::fwd_run_launch(mu_t, a0_t, p0_t, n_balls, F, array, ac, observed, out,
                                          want_loss ? lpart : nullptr, coincident, st)
                    : fwd_run_launch(mu_t, a0_t, p0_t, n_balls, F, array, ac, observed, out,
                                     want_loss ? lpart : nullptr, coincident, st);
            if (rc != PC_OK) return rc;
        } else {
            if (cudaMemsetAsync(out, 0, (size_t)F * M * T * sizeof(float), st) != cudaSuccess)
                return PC_ERR_CUDA;
            if (observed)
                k_forward_finish<<<dim3(M, F), 256, 0, st>>>(
                    out, observed, out, want_loss ? lpart : nullptr, 1, F, M, T,
                    finish_vec(out, observed, out, T));
        }
        if (want_loss) k_loss_reduce<<<F, 256, 0, st>>>(lpart, M, loss_per_frame);
        return last_status();
    }
    FwdPlan p = fwd_plan(n_balls > 0 ? n_balls : 1, F, M, T);
    const size_t need = p.partial_bytes + p.loss_bytes + p.prep_bytes;
    if (!workspace || workspace_bytes < need) return PC_ERR_ARGUMENT;
    unsigned char* ws = static_cast<unsigned char*>(workspace);
    float4* cull = reinterpret_cast<float4*>(ws);
    unsigned* bounds = reinterpret_cast<unsigned*>(
        ws + (((size_t)F * (n_balls > 0 ? n_balls : 1) * sizeof(float4) + 255) / 256) * 256);
    unsigned char* rest = ws + p.prep_bytes;
    float* partial = p.partial_bytes ? reinterpret_cast<float*>(rest) : nullptr;
    double* lpart = reinterpret_cast<double*>(rest + p.partial_bytes);
    const bool want_loss = observed && loss_per_frame;

    if (n_balls > 0) {
        if (cudaMemsetAsync(bounds, 0xff, (size_t)F * p.nchunk * 8 * sizeof(unsigned), st) !=
            cudaSuccess)
            return PC_ERR_CUDA;
        int64_t bpc = (p.chunk_balls + 255) / 256;      // prep blocks per chunk
        const int64_t cap = (2LL * num_sms() + p.nchunk - 1) / p.nchunk;
        if (bpc > cap) bpc = cap;
        if (bpc < 1) bpc = 1;
        k_forward_prep<<<dim3((unsigned)(bpc * p.nchunk), F), 256, 0, st>>>(
            mu_t, a0_t, n_balls, F, p.nchunk, p.chunk_balls, (int)bpc, cull, bounds);
        FwdArgs a;
        a.mu = mu_t;
        a.p0 = p0_t;
        a.cull = cull;
        a.bounds = bounds;
        a.pos = array->positions;
        a.sorder = array->sensor_order;
        a.obs = observed;
        a.out = p.nchunk > 1 ? partial : out;
        a.loss = (want_loss && p.nchunk == 1) ? lpart : nullptr;
        a.coinc = reinterpret_cast<long long*>(coincident);
        a.fo = array->frame_offset;
        a.so = array->sensor_offset;
        a.mt = array->n_sensors_total > 0 ? array->n_sensors_total : M;
        a.B = n_balls;
        a.F = F;
        a.M = M;
        a.ac = ac;
        a.Tseg = p.Tseg;
        a.nseg = p.nseg;
        a.nchunk = p.nchunk;
        a.chunk_balls = p.chunk_balls;
        a.inv_v_f = (float)ac.inv_v;
        a.t0_f = (float)ac.t0;
        a.inv_dt_f = (float)ac.inv_dt;
        a.sa_f = (float)(ac.support * ac.inv_v * ac.inv_dt);
        a.vt0_f = (float)(ac.v * ac.t0);
        a.vdt_f = (float)(ac.v * ac.dt);
        a.vdt_d = ac.v * ac.dt;
        a.vt0_d = ac.v * ac.t0;
        const bool ranged = p.nchunk > 1 && !ac.exact && fwd_cmb() && T >= 4096;
        a.part_margin = ranged && fwd_pm() ? 16 : 0;
        const size_t smem = fwd_smem_bytes(p.Tseg);
        // the dynamic shared-memory opt-in is per device: track it per device
        static unsigned long long attr_set = 0;
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess) return PC_ERR_CUDA;
        const unsigned long long bit = 1ull << (dev & 63);
        if (!(attr_set & bit)) {
            const int mx = (int)fwd_smem_bytes(fwd_tseg_max());
            cudaFuncSetAttribute(k_forward<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
            cudaFuncSetAttribute(k_forward<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
            cudaFuncSetAttribute(k_forward<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
            cudaFuncSetAttribute(k_forward<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
            attr_set |= bit;
        }
        dim3 grid(p.nseg * p.nchunk, (M + FWD_WARPS * FSW - 1) / (FWD_WARPS * FSW), F);
        // record windows are 15-bit: segment-relative for long traces
        const bool rel = T >= (1 << 15) - 64;
        if (ac.exact && rel)
            k_forward<true, true><<<grid, FWD_WARPS * 32, smem, st>>>(a);
        else if (ac.exact)
            k_forward<true, false><<<grid, FWD_WARPS * 32, smem, st>>>(a);
        else if (rel)
            k_forward<false, true><<<grid, FWD_WARPS * 32, smem, st>>>(a);
        else
            k_forward<false, false><<<grid, FWD_WARPS * 32, smem, st>>>(a);
        // the ranged combine pays off on long rows (config 2: -0.7 %; config
        // 1, T = 2048 with wide ranges: +15 % against the dense float4 path)
        if (ranged) {
            k_forward_combine<<<dim3(M, F), 256, 0, st>>>(
                partial, bounds, array->positions, ac, observed, out,
                want_loss ? lpart : nullptr, p.nchunk, F, M, T);
        } else if (p.nchunk > 1) {
            k_forward_finish<<<dim3(M, F), 256, 0, st>>>(
                partial, observed, out, want_loss ? lpart : nullptr, p.nchunk, F, M, T,
                finish_vec(partial, observed, out, T));
        }
    } else {
        // empty cloud: zero traces (radiator.py:205-207); residual = -observed
        if (cudaMemsetAsync(out, 0, (size_t)F * M * T * sizeof(float), st) != cudaSuccess)
            return PC_ERR_CUDA;
        if (observed)
            k_forward_finish<<<dim3(M, F), 256, 0, st>>>(
                out, observed, out, want_loss ? lpart : nullptr, 1, F, M, T,
                finish_vec(out, observed, out, T));
    }
    if (want_loss) {
        const int per_frame = (n_balls > 0 && p.nchunk == 1) ? M * p.nseg : M;
        k_loss_reduce<<<F, 256, 0, st>>>(lpart, per_frame, loss_per_frame);
    }
    return last_status();
}

extern "C" int pc_residual_loss(const float* predicted, const float* observed, float* out,
                                double* loss_partial, double* loss_per_frame, int32_t n_frames,
                                int32_t n_sensors, int32_t n_samples, pc_stream_t stream) {
    if (n_frames < 0 || n_sensors < 0 || n_samples < 0) return PC_ERR_ARGUMENT;
    if (n_frames == 0 || n_sensors == 0 || n_samples == 0) return PC_OK;
    if (!predicted || !observed || !out || (loss_per_frame && !loss_partial))
        return PC_ERR_ARGUMENT;
    cudaStream_t st = as_stream(stream);
    k_forward_finish<<<dim3(n_sensors, n_frames), 256, 0, st>>>(
        predicted, observed, out, loss_per_frame ? loss_partial : nullptr, 1, n_frames, n_sensors,
        n_samples, finish_vec(predicted, observed, out, n_samples));
    if (loss_per_frame)
        k_loss_reduce<<<n_frames, 256, 0, st>>>(loss_partial, n_sensors, loss_per_frame);
    return last_status();
}

// Two-CTA sensor split of the adjoint for grids under PC_ADJ_SPLIT waves of
// 8-CTA SMs (default 6; 0 = off).  Config 2 at one frame per rank (4.2
// waves): 1.577 -> 1.532 ms per iteration with the split.
static int adj_split() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("PC_ADJ_SPLIT");
        v = e ? atoi(e) : 6;
    }
    return v;
}

extern "C" int pc_residual_state_grads(const double* mu_t, const float* a0_t, const float* p0_t,
                                       int64_t n_balls, int32_t n_frames,
                                       const pc_array_t* array, const float* residual, float* G,
                                       int64_t* coincident, pc_stream_t stream) {
    ArrayConsts ac;
    if (!array_consts(array, ac) || n_balls < 0 || n_frames < 1 || !coincident)
        return PC_ERR_ARGUMENT;
    if (array->n_samples >= kMaxSamples) return PC_ERR_UNSUPPORTED;   // 2^30
    if (n_balls == 0) return PC_OK;
    if (!mu_t || !a0_t || !p0_t || !residual || !G) return PC_ERR_ARGUMENT;
    AdjArgs a;
    a.mu = mu_t;
    a.a0 = a0_t;
    a.p0 = p0_t;
    a.pos = array->positions;
    a.resid = residual;
    a.G = G;
    a.coinc = reinterpret_cast<long long*>(coincident);
    a.fo = array->frame_offset;
    a.so = array->sensor_offset;
    a.mt = array->n_sensors_total > 0 ? array->n_sensors_total : array->n_sensors;
    a.B = n_balls;
    a.F = n_frames;
    a.M = array->n_sensors;
    a.ac = ac;
    a.inv_v_f = (float)ac.inv_v;
    a.t0_f = (float)ac.t0;
    a.inv_dt_f = (float)ac.inv_dt;
    a.sa_f = (float)(ac.support * ac.inv_v * ac.inv_dt);
    a.vt0_f = (float)(ac.v * ac.t0);
    a.vdt_f = (float)(ac.v * ac.dt);
    a.vdt_d = ac.v * ac.dt;
    a.vt0_d = ac.v * ac.t0;
#if PC_ADJ_B2
    dim3 grid((unsigned)((n_balls + ADJ_NB * ADJ_WARPS - 1) / (ADJ_NB * ADJ_WARPS)), n_frames);
#else
    dim3 grid((unsigned)((n_balls + ADJ_WARPS - 1) / ADJ_WARPS), n_frames);
#endif
    cudaStream_t st = as_stream(stream);
#if PC_ADJ_TMA
    if (!ac.exact && array->n_samples % 4 == 0 &&
        reinterpret_cast<uintptr_t>(residual) % 16 == 0) {
        constexpr int TW = PC_ADJ_TMA;
        const size_t smem = adj_tma_smem<TW>();
        static unsigned long long tma_attr = 0;
        int dev = 0;
        cudaGetDevice(&dev);
        if (!(tma_attr & (1ull << (dev & 63)))) {
            cudaFuncSetAttribute(k_adjoint_tma<TW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
            tma_attr |= 1ull << (dev & 63);
        }
        dim3 gt((unsigned)((n_balls + TW - 1) / TW), n_frames);
        k_adjoint_tma<TW><<<gt, TW * 32, smem, st>>>(a);
        return last_status();
    }
#endif
    // few waves of 8-CTA SMs: split each ball's sensors over two CTAs (G
    // zeroed, two partial sums added)
    const int64_t ctas = (int64_t)grid.x * n_frames;
    const bool split = adj_split() > 0 && a.M >= 64 && ctas < (int64_t)adj_split() * 8 * num_sms();
    a.msplit = ((a.M / 2 + 31) / 32) * 32;
#if PC_ADJ_V8
    const bool aligned = array->n_samples % 8 == 0 && reinterpret_cast<uintptr_t>(residual) % 32 == 0;
#else
    const bool aligned = array->n_samples % 4 == 0 && reinterpret_cast<uintptr_t>(residual) % 16 == 0;
#endif
    if (split) {
        if (cudaMemsetAsync(G, 0, (size_t)n_balls * n_frames * 5 * sizeof(float), st) != cudaSuccess)
            return PC_ERR_CUDA;
        dim3 g2(grid.x, 2 * n_frames);
        if (aligned)
            k_adjoint<true, true><<<g2, ADJ_WARPS * 32, 0, st>>>(a);
        else
            k_adjoint<false, true><<<g2, ADJ_WARPS * 32, 0, st>>>(a);
    } else if (aligned) {
        k_adjoint<true, false><<<grid, ADJ_WARPS * 32, 0, st>>>(a);
    } else {
        k_adjoint<false, false><<<grid, ADJ_WARPS * 32, 0, st>>>(a);
    }
    return last_status();
}

// ---------------------------------------------------------------- formula anchors
//
// radiator.py:36-55 pressure_kernel and :58-83 pressure_kernel_grad,
// elementwise in fp64 over already-broadcast inputs (the reference's
// closed form, term for term).
__global__ void __launch_bounds__(256) k_pressure(const double* __restrict__ R,
                                                  const double* __restrict__ t,
                                                  const double* __restrict__ p0,
                                                  const double* __restrict__ a0, int64_t n,
                                                  double v, double* __restrict__ out,
                                                  double* __restrict__ d_p0,
                                                  double* __restrict__ d_a0,
                                                  double* __restrict__ d_R) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double r = R[i], tt = t[i], p = p0[i], a = a0[i];
        const double um = r - v * tt, up = r + v * tt;
        if (out) {
            const double inv2a2 = 1.0 / (2.0 * (a * a));
            out[i] = (p / (2.0 * r)) * (um * exp(-um * um * inv2a2) + up * exp(-up * up * inv2a2));
        }
        if (d_p0) {
            const double inv_a2 = 1.0 / (a * a);
            const double gm = exp(-0.5 * um * um * inv_a2);
            const double gp = exp(-0.5 * up * up * inv_a2);
            const double s = um * gm + up * gp;
            d_p0[i] = s / (2.0 * r);
            d_a0[i] = (p / (2.0 * r)) * (um * um * um * gm + up * up * up * gp) * inv_a2 / a;
            const double ds = gm * (1.0 - um * um * inv_a2) + gp * (1.0 - up * up * inv_a2);
            d_R[i] = -(p * s) / (2.0 * r * r) + (p / (2.0 * r)) * ds;
        }
    }
}

extern "C" int pc_pressure_kernel(const double* R, const double* t, const double* p0,
                                  const double* a0, int64_t n, double sound_speed, double* out,
                                  double* d_p0, double* d_a0, double* d_R, pc_stream_t stream) {
    if (n < 0 || !(sound_speed > 0)) return PC_ERR_ARGUMENT;
    if (n == 0) return PC_OK;
    if (!R || !t || !p0 || !a0 || (!out && !d_p0)) return PC_ERR_ARGUMENT;
    if (d_p0 && (!d_a0 || !d_R)) return PC_ERR_ARGUMENT;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 8LL * num_sms()) blocks = 8LL * num_sms();
    k_pressure<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(R, t, p0, a0, n, sound_speed, out,
                                                                d_p0, d_a0, d_R);
    return last_status();
}
