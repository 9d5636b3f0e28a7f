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

constexpr int FWD_WARPS = 4;    // sensors per CTA (one warp owns one sensor)
constexpr int FWD_TILE = 128;   // balls staged per shared-memory tile
constexpr int FWD_TSEG_MAX = 2048;

struct FwdPlan {
    int Tseg, nseg, nchunk;
    int64_t chunk_balls;
    size_t partial_bytes, loss_bytes;
};

static FwdPlan fwd_plan(int64_t B, int F, int M, int T) {
    FwdPlan p;
    p.Tseg = T < FWD_TSEG_MAX ? ((T + 31) / 32) * 32 : FWD_TSEG_MAX;
    p.nseg = (T + p.Tseg - 1) / p.Tseg;
    const int64_t tiles = (M + FWD_WARPS - 1) / FWD_WARPS;
    const int64_t base = (int64_t)p.nseg * tiles * F;
    const int64_t want = 6LL * num_sms();
    int64_t c = base >= want ? 1 : (want + base - 1) / base;
    const int64_t cmax = B / 256 > 1 ? B / 256 : 1;
    if (c > cmax) c = cmax;
    if (c > 64) c = 64;
    p.nchunk = (int)c;
    p.chunk_balls = (B + c - 1) / c;
    p.partial_bytes = p.nchunk > 1 ? (size_t)p.nchunk * F * M * T * sizeof(float) : 0;
    const int nloss = p.nchunk > 1 ? 1 : p.nseg;
    p.loss_bytes = (size_t)F * M * nloss * sizeof(double);
    return p;
}

struct FwdArgs {
    const double* mu;
    const float* a0;
    const float* p0;
    const double* pos;
    const float* obs;
    float* out;       // final (nchunk == 1) or partial traces (nchunk > 1)
    double* loss;     // (F, M, nseg) partials or NULL
    long long* coinc;
    int64_t B;
    int F, M;
    ArrayConsts ac;
    int Tseg, nseg, nchunk;
    int64_t chunk_balls;
};

template <bool NEAR>
__device__ __forceinline__ void fwd_window(float* __restrict__ tr, int s0, int jl, int jh, int jc,
                                           float Dc, float Uc, float c, float nk, float vdt,
                                           int lane) {
    int j = jl + lane;
    float kf = (float)(j - jc);
    for (; j < jh; j += 32, kf += 32.f) {
        const float um = fmaf(-kf, vdt, Dc);
        float val = um * ex2(um * um * nk);
        if (NEAR) {
            const float up = fmaf(kf, vdt, Uc);
            val = fmaf(up, ex2(up * up * nk), val);
        }
        tr[j - s0] = fmaf(c, val, tr[j - s0]);
    }
}

__global__ void __launch_bounds__(FWD_WARPS * 32) k_forward(FwdArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* smx = reinterpret_cast<double*>(smem);
    double* smy = smx + FWD_TILE;
    double* smz = smy + FWD_TILE;
    float* sa0 = reinterpret_cast<float*>(smz + FWD_TILE);
    float* sp0 = sa0 + FWD_TILE;
    float* traces = sp0 + FWD_TILE;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int seg = blockIdx.x % a.nseg;
    const int chunk = blockIdx.x / a.nseg;
    const int m = blockIdx.y * FWD_WARPS + warp;
    const int f = blockIdx.z;
    const int T = a.ac.T;
    const int s0 = seg * a.Tseg;
    const int s1 = min(T, s0 + a.Tseg);
    const bool active = m < a.M;
    float* tr = traces + warp * a.Tseg;
    for (int j = lane; j < a.Tseg; j += 32) tr[j] = 0.f;

    double px = 0.0, py = 0.0, pz = 0.0;
    if (active) {
        px = a.pos[3 * m + 0];
        py = a.pos[3 * m + 1];
        pz = a.pos[3 * m + 2];
    }
    const int64_t b0 = (int64_t)chunk * a.chunk_balls;
    const int64_t b1 = min(a.B, b0 + a.chunk_balls);
    const size_t fb = (size_t)f * a.B;
    const float vdt = a.ac.vdt;

    for (int64_t tb = b0; tb < b1; tb += FWD_TILE) {
        const int n_in = (int)min((int64_t)FWD_TILE, b1 - tb);
        __syncthreads();
        for (int i = threadIdx.x; i < n_in; i += blockDim.x) {
            const size_t s = fb + tb + i;
            smx[i] = a.mu[3 * s + 0];
            smy[i] = a.mu[3 * s + 1];
            smz[i] = a.mu[3 * s + 2];
            sa0[i] = a.a0[s];
            sp0[i] = a.p0[s];
        }
        __syncthreads();
        if (!active) continue;
        for (int g = 0; g < n_in; g += 32) {
            const int i = g + lane;
            bool valid = i < n_in;
            int jl = 0, jh = 0, jc = 0, near = 0;
            float Dc = 0.f, Uc = 0.f, c = 0.f, nk = 0.f;
            if (valid) {
                const float av = sa0[i];
                PairGeom pg;
                pair_geometry(smx[i] - px, smy[i] - py, smz[i] - pz, av, a.ac, pg);
                if (pg.R < kCoincidenceEps) {
                    atomicMin(a.coinc, (long long)(tb + i) * a.M + m);
                    valid = false;
                } else {
                    jl = max(pg.jlo, s0);
                    jh = min(pg.jhi, s1);
                    valid = jh > jl;
                    jc = pg.jc;
                    Dc = pg.Dc;
                    Uc = pg.Uc;
                    near = pg.near;
                    c = sp0[i] * (0.5f / (float)pg.R);
                    nk = -0.5f * kLog2e / (av * av);
                }
            }
            unsigned mask = __ballot_sync(0xffffffffu, valid);
            while (mask) {
                const int src = __ffs(mask) - 1;
                mask &= mask - 1;
                const int bjl = __shfl_sync(0xffffffffu, jl, src);
                const int bjh = __shfl_sync(0xffffffffu, jh, src);
                const int bjc = __shfl_sync(0xffffffffu, jc, src);
                const int bnear = __shfl_sync(0xffffffffu, near, src);
                const float bDc = __shfl_sync(0xffffffffu, Dc, src);
                const float bc = __shfl_sync(0xffffffffu, c, src);
                const float bnk = __shfl_sync(0xffffffffu, nk, src);
                if (bnear) {
                    const float bUc = __shfl_sync(0xffffffffu, Uc, src);
                    fwd_window<true>(tr, s0, bjl, bjh, bjc, bDc, bUc, bc, bnk, vdt, lane);
                } else {
                    fwd_window<false>(tr, s0, bjl, bjh, bjc, bDc, 0.f, bc, bnk, vdt, lane);
                }
            }
        }
    }
    __syncwarp();
    if (!active) return;
    const size_t row = ((size_t)f * a.M + m) * T;
    if (a.nchunk > 1) {
        float* dst = a.out + (size_t)chunk * a.F * a.M * T + row;
        for (int j = s0 + lane; j < s1; j += 32) dst[j] = tr[j - s0];
        return;
    }
    double lsum = 0.0;
    if (a.obs) {
        for (int j = s0 + lane; j < s1; j += 32) {
            const float r = tr[j - s0] - __ldg(a.obs + row + j);
            a.out[row + j] = r;
            lsum = fma((double)r, (double)r, lsum);
        }
    } else {
        for (int j = s0 + lane; j < s1; j += 32) a.out[row + j] = tr[j - s0];
    }
    if (a.loss) {
        lsum = warp_sum(lsum);
        if (lane == 0) a.loss[((size_t)f * a.M + m) * a.nseg + seg] = lsum;
    }
}

// Chunk combine (fixed chunk order) + residual + per-trace loss partial.
__global__ void __launch_bounds__(256) k_forward_finish(const float* __restrict__ partial,
                                                        const float* __restrict__ obs,
                                                        float* __restrict__ out,
                                                        double* __restrict__ loss, int nchunk,
                                                        int F, int M, int T) {
    const int m = blockIdx.x, f = blockIdx.y;
    const size_t row = ((size_t)f * M + m) * T;
    const size_t cstride = (size_t)F * M * T;
    double lsum = 0.0;
    for (int j = threadIdx.x; j < T; j += blockDim.x) {
        float s = 0.f;
        for (int c = 0; c < nchunk; ++c) s += partial[c * cstride + row + j];
        if (obs) {
            s -= obs[row + j];
            lsum = fma((double)s, (double)s, lsum);
        }
        out[row + j] = s;
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

constexpr int ADJ_WARPS = 4;  // balls per CTA (one warp owns one (ball, frame))

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
};

enum { REC_VALID = 1, REC_NEAR = 2 };

// One pair's partial sums over the samples this lane owns.
template <int G, bool NEAR>
__device__ __forceinline__ void adj_window(const float* __restrict__ row, int j, int jh, float kf,
                                           float Dc, float Uc, float nk, float inv_a2, float vdt,
                                           float& A1, float& AQ, float& A3) {
    for (; j < jh; j += G, kf += (float)G) {
        const float r = __ldg(row + j);
        const float um = fmaf(-kf, vdt, Dc);
        const float u2 = um * um;
        const float w = r * ex2(u2 * nk);
        A1 = fmaf(w, um, A1);
        AQ = fmaf(w, fmaf(u2, -inv_a2, 1.f), AQ);
        A3 = fmaf(w * u2, um, A3);
        if (NEAR) {
            const float up = fmaf(kf, vdt, Uc);
            const float p2 = up * up;
            const float wp = r * ex2(p2 * nk);
            A1 = fmaf(wp, up, A1);
            AQ = fmaf(wp, fmaf(p2, -inv_a2, 1.f), AQ);
            A3 = fmaf(wp * p2, up, A3);
        }
    }
}

template <int G>
__global__ void __launch_bounds__(ADJ_WARPS * 32) k_adjoint(AdjArgs a) {
    __shared__ __align__(16) float4 recs[ADJ_WARPS][32][4];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t b = (int64_t)blockIdx.x * ADJ_WARPS + warp;
    const int f = blockIdx.y;
    if (b >= a.B) return;
    const size_t sb = (size_t)f * a.B + b;
    const double mx = a.mu[3 * sb + 0], my = a.mu[3 * sb + 1], mz = a.mu[3 * sb + 2];
    const float av = a.a0[sb], pv = a.p0[sb];
    const float inv_a2 = 1.f / (av * av);
    const float nk = -0.5f * kLog2e * inv_a2;
    const float vdt = a.ac.vdt;
    const int T = a.ac.T;
    float g0 = 0.f, g1 = 0.f, g2 = 0.f, g3 = 0.f, g4 = 0.f;
    float4(&rec)[32][4] = recs[warp];

    for (int mb = 0; mb < a.M; mb += 32) {
        const int m = mb + lane;
        int flags = 0;
        PairGeom pg;
        pg.jlo = pg.jhi = pg.jc = 0;
        pg.Dc = pg.Uc = 0.f;
        pg.R = 1.0;
        float ux = 0.f, uy = 0.f, uz = 0.f;
        if (m < a.M) {
            const double dx = mx - a.pos[3 * m + 0];
            const double dy = my - a.pos[3 * m + 1];
            const double dz = mz - a.pos[3 * m + 2];
            pair_geometry(dx, dy, dz, av, a.ac, pg);
            if (pg.R < kCoincidenceEps) {
                atomicMin(a.coinc, (long long)b * a.M + m);
            } else {
                flags = (pg.jhi > pg.jlo ? REC_VALID : 0) | (pg.near ? REC_NEAR : 0);
                const double ir = 1.0 / pg.R;
                ux = (float)(dx * ir);
                uy = (float)(dy * ir);
                uz = (float)(dz * ir);
            }
        }
        const float inv2R = (float)(0.5 / pg.R);
        const float kp = inv2R;
        const float ka = pv * inv2R * inv_a2 / av;
        const float kR2 = pv * inv2R;
        const float kR1 = -kR2 * (float)(1.0 / pg.R);
        rec[lane][0] = make_float4(__int_as_float(pg.jlo), __int_as_float(pg.jhi),
                                   __int_as_float(pg.jc), __int_as_float(flags));
        rec[lane][1] = make_float4(pg.Dc, pg.Uc, kp, ka);
        rec[lane][2] = make_float4(kR1, kR2, ux, uy);
        rec[lane][3] = make_float4(uz, 0.f, 0.f, 0.f);
        __syncwarp();
        const int npair = min(32, a.M - mb);
        for (int pb = 0; pb < npair; pb += 32 / G) {
            const int pi = pb + lane / G;
            const int s = lane % G;
            const float4 r0 = rec[pi][0];
            const int rflags = __float_as_int(r0.w);
            if (pi < npair && (rflags & REC_VALID)) {
                const float4 r1 = rec[pi][1];
                const int jl = __float_as_int(r0.x), jh = __float_as_int(r0.y);
                const int jc = __float_as_int(r0.z);
                const float* row = a.resid + ((size_t)f * a.M + mb + pi) * T;
                float A1 = 0.f, AQ = 0.f, A3 = 0.f;
                const int j = jl + s;
                const float kf = (float)(j - jc);
                if (rflags & REC_NEAR)
                    adj_window<G, true>(row, j, jh, kf, r1.x, r1.y, nk, inv_a2, vdt, A1, AQ, A3);
                else
                    adj_window<G, false>(row, j, jh, kf, r1.x, 0.f, nk, inv_a2, vdt, A1, AQ, A3);
                const float4 r2 = rec[pi][2];
                const float4 r3 = rec[pi][3];
                const float accR = fmaf(r2.x, A1, r2.y * AQ);
                g0 = fmaf(r1.w, A3, g0);
                g1 = fmaf(r1.z, A1, g1);
                g2 = fmaf(accR, r2.z, g2);
                g3 = fmaf(accR, r2.w, g3);
                g4 = fmaf(accR, r3.x, g4);
            }
        }
        __syncwarp();
    }
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

extern "C" int pc_forward_plan(int64_t n_balls, int32_t n_frames, const pc_array_t* array,
                               int32_t* plan) {
    if (!array || !plan || n_balls < 0 || n_frames < 1 || array->n_sensors < 1 ||
        array->n_samples < 1)
        return PC_ERR_ARGUMENT;
    FwdPlan p = fwd_plan(n_balls > 0 ? n_balls : 1, n_frames, array->n_sensors,
                         array->n_samples);
    plan[0] = p.Tseg;
    plan[1] = p.nseg;
    plan[2] = p.nchunk;
    plan[3] = 2 + (p.nchunk > 1 ? 1 : 0);  // forward [+ combine] + loss reduce
    return PC_OK;
}

extern "C" size_t pc_forward_workspace_bytes(int64_t n_balls, int32_t n_frames,
                                             const pc_array_t* array) {
    if (!array || n_balls < 0 || n_frames < 1) return 0;
    FwdPlan p = fwd_plan(n_balls, n_frames, array->n_sensors, array->n_samples);
    return p.partial_bytes + p.loss_bytes + 256;
}

extern "C" int pc_forward_traces(const double* mu_t, const float* a0_t, const float* p0_t,
                                 int64_t n_balls, int32_t n_frames, const pc_array_t* array,
                                 const float* observed, float* out, double* loss_per_frame,
                                 int64_t* coincident, void* workspace, size_t workspace_bytes,
                                 pc_stream_t stream) {
    ArrayConsts ac;
    if (!array_consts(array, ac) || n_balls < 0 || n_frames < 1 || !out || !coincident)
        return PC_ERR_ARGUMENT;
    const int M = array->n_sensors, T = array->n_samples, F = n_frames;
    cudaStream_t st = as_stream(stream);
    if (n_balls > 0 && (!mu_t || !a0_t || !p0_t)) return PC_ERR_ARGUMENT;
    FwdPlan p = fwd_plan(n_balls > 0 ? n_balls : 1, F, M, T);
    const size_t need = p.partial_bytes + p.loss_bytes;
    if (need > 0 && (!workspace || workspace_bytes < need)) return PC_ERR_ARGUMENT;
    unsigned char* ws = static_cast<unsigned char*>(workspace);
    float* partial = p.partial_bytes ? reinterpret_cast<float*>(ws) : nullptr;
    double* lpart = reinterpret_cast<double*>(ws + p.partial_bytes);
    const bool want_loss = observed && loss_per_frame;

    if (n_balls > 0) {
        FwdArgs a;
        a.mu = mu_t;
        a.a0 = a0_t;
        a.p0 = p0_t;
        a.pos = array->positions;
        a.obs = observed;
        a.out = p.nchunk > 1 ? partial : out;
        a.loss = (want_loss && p.nchunk == 1) ? lpart : nullptr;
        a.coinc = reinterpret_cast<long long*>(coincident);
        a.B = n_balls;
        a.F = F;
        a.M = M;
        a.ac = ac;
        a.Tseg = p.Tseg;
        a.nseg = p.nseg;
        a.nchunk = p.nchunk;
        a.chunk_balls = p.chunk_balls;
        const size_t smem = (size_t)FWD_TILE * (3 * sizeof(double) + 2 * sizeof(float)) +
                            (size_t)FWD_WARPS * p.Tseg * sizeof(float);
        static bool attr_set = false;
        if (!attr_set) {
            cudaFuncSetAttribute(k_forward, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 64 * 1024);
            attr_set = true;
        }
        dim3 grid(p.nseg * p.nchunk, (M + FWD_WARPS - 1) / FWD_WARPS, F);
        k_forward<<<grid, FWD_WARPS * 32, smem, st>>>(a);
        if (p.nchunk > 1) {
            k_forward_finish<<<dim3(M, F), 256, 0, st>>>(partial, observed, out,
                                                        want_loss ? lpart : nullptr, p.nchunk,
                                                        F, M, T);
        }
    } else {
        // empty cloud: zero traces (radiator.py:205-207); residual = -observed
        if (cudaMemsetAsync(out, 0, (size_t)F * M * T * sizeof(float), st) != cudaSuccess)
            return PC_ERR_CUDA;
        if (observed)
            k_forward_finish<<<dim3(M, F), 256, 0, st>>>(out, observed, out,
                                                        want_loss ? lpart : nullptr, 1, F, M, T);
    }
    if (want_loss) {
        const int per_frame = (n_balls > 0 && p.nchunk == 1) ? M * p.nseg : M;
        k_loss_reduce<<<F, 256, 0, st>>>(lpart, per_frame, loss_per_frame);
    }
    return last_status();
}

extern "C" int pc_residual_state_grads(const double* mu_t, const float* a0_t, const float* p0_t,
                                       int64_t n_balls, int32_t n_frames,
                                       const pc_array_t* array, const float* residual, float* G,
                                       int64_t* coincident, pc_stream_t stream) {
    ArrayConsts ac;
    if (!array_consts(array, ac) || n_balls < 0 || n_frames < 1 || !coincident)
        return PC_ERR_ARGUMENT;
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
    a.B = n_balls;
    a.F = n_frames;
    a.M = array->n_sensors;
    a.ac = ac;
    dim3 grid((unsigned)((n_balls + ADJ_WARPS - 1) / ADJ_WARPS), n_frames);
    cudaStream_t st = as_stream(stream);
    // lane-group width per pair from the typical window length 12 a0 / (v dt)
    k_adjoint<8><<<grid, ADJ_WARPS * 32, 0, st>>>(a);
    return last_status();
}
