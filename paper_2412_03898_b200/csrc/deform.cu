// Deformation forward / backward for sm_100a.
//
//   pc_deform_states   <- pkg/src/pacloud/deformation.py:184-204 (cloud_states_at)
//   pc_deform_jacobian <- deformation.py:219-267 (cloud_state_grads, materialised)
//   pc_assemble_grads  <- radiator.py:278-294 (accumulate_frame_grads' chain rule)
//   pc_deform_backward <- the same chain rule fused over frames
//                         (reconstruction.py:303-316), no Jacobian in HBM
//
// These kernels are HBM / latency bound and tiny next to the radiator; they
// run in fp64 so deformed centres keep the precision the radiator's fp64 pair
// geometry relies on.
#include "common.cuh"

namespace pc {

__device__ __forceinline__ void mode_rows(int mode, int rows[5]) {
    rows[0] = 0;
    rows[1] = 1;
    if (mode == PC_COORD_RADIAL) {
        rows[2] = rows[3] = rows[4] = 2;
    } else {
        rows[2] = 2;
        rows[3] = 3;
        rows[4] = 4;
    }
}

// Gaussian basis value and partials (deformation.py:93-99).
__device__ __forceinline__ void gauss_pieces(double t, double th, double sg, double& phi,
                                             double& dth, double& dsg) {
    const double u = (t - th) / sg;
    phi = exp(-0.5 * u * u);
    dth = phi * u / sg;
    dsg = phi * u * u / sg;
}

// Builder-defined poly+Fourier basis: [1, t, t^2, t^3, sin 2pi k t, cos 2pi k t].
__device__ __forceinline__ double pf_basis(int n, double t) {
    if (n == 0) return 1.0;
    if (n == 1) return t;
    if (n == 2) return t * t;
    if (n == 3) return t * t * t;
    const int k = (n - 4) / 2 + 1;
    const double x = 2.0 * (double)k * t;
    return ((n - 4) & 1) ? cospi(x) : sinpi(x);
}

struct CloudView {
    const double *p0, *a0, *mu, *theta, *sigma, *omega;
    int64_t B;
    int N, per_channel, kind;
};

static bool view_of(const pc_cloud_t* c, CloudView& v) {
    if (!c || c->n_balls < 0 || c->n_basis < 1) return false;
    if (c->n_balls > 0 && (!c->p0 || !c->a0 || !c->mu || !c->omega)) return false;
    if (c->basis_kind == PC_BASIS_GAUSS && c->n_balls > 0 && (!c->theta || !c->sigma))
        return false;
    if (c->basis_kind != PC_BASIS_GAUSS && c->basis_kind != PC_BASIS_POLYFOURIER) return false;
    if (c->basis_kind == PC_BASIS_POLYFOURIER && (c->n_basis < 4 || (c->n_basis - 4) % 2))
        return false;
    v.p0 = c->p0;
    v.a0 = c->a0;
    v.mu = c->mu;
    v.theta = c->theta;
    v.sigma = c->sigma;
    v.omega = c->omega;
    v.B = c->n_balls;
    v.N = c->n_basis;
    v.per_channel = c->per_channel;
    v.kind = c->basis_kind;
    return true;
}

// Channel sums H[c] = sum_n omega[b,c,n] phi_n(t) in fp64.
__device__ void channel_sums(const CloudView& c, int64_t b, double t, double H[5]) {
    for (int k = 0; k < 5; ++k) H[k] = 0.0;
    const int N = c.N;
    const double* om = c.omega + (size_t)b * 5 * N;
    for (int n = 0; n < N; ++n) {
        if (c.kind == PC_BASIS_POLYFOURIER) {
            const double ph = pf_basis(n, t);
#pragma unroll
            for (int k = 0; k < 5; ++k) H[k] = fma(om[k * N + n], ph, H[k]);
        } else if (!c.per_channel) {
            double ph, d1, d2;
            gauss_pieces(t, c.theta[(size_t)b * N + n], c.sigma[(size_t)b * N + n], ph, d1, d2);
#pragma unroll
            for (int k = 0; k < 5; ++k) H[k] = fma(om[k * N + n], ph, H[k]);
        } else {
#pragma unroll
            for (int k = 0; k < 5; ++k) {
                double ph, d1, d2;
                const size_t q = ((size_t)b * 5 + k) * N + n;
                gauss_pieces(t, c.theta[q], c.sigma[q], ph, d1, d2);
                H[k] = fma(om[k * N + n], ph, H[k]);
            }
        }
    }
}

// a0_floor NaN = no floor (a0_floor=None): x < NaN is false, so every
// non-NaN floor clamps exactly as deformation.py:202-203 (np.maximum).
// Hout[...,0] = NaN marks a clamped (frame, ball) for pc_deform_backward
// (the decision is taken here, in fp64).
template <typename ST>
__global__ void __launch_bounds__(128) k_deform_states(CloudView c, const double* __restrict__ tf,
                                                       int F, int mode, double a0_floor,
                                                       double* __restrict__ mu_t,
                                                       ST* __restrict__ a0_t,
                                                       ST* __restrict__ p0_t,
                                                       float* __restrict__ Hout) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= c.B * F) return;
    const int64_t b = idx / F;
    const int f = (int)(idx - b * F);
    double H[5];
    channel_sums(c, b, tf[f], H);
    const double a0raw = c.a0[b] * (1.0 + H[0]);
    const bool clamped = a0raw < a0_floor;
    const double a0 = clamped ? a0_floor : a0raw;
    const double p0 = c.p0[b] * (1.0 + H[1]);
    const size_t s = (size_t)f * c.B + b;
    for (int k = 0; k < 3; ++k) {
        const double mu = c.mu[3 * b + k];
        const double h = H[mode == PC_COORD_RADIAL ? 2 : 2 + k];
        mu_t[3 * s + k] = mode == PC_COORD_ADDITIVE ? mu + h : mu * (1.0 + h);
    }
    a0_t[s] = (ST)a0;
    p0_t[s] = (ST)p0;
    if (Hout) {
        for (int k = 0; k < 5; ++k) Hout[5 * s + k] = (float)H[k];
        if (clamped) Hout[5 * s] = __int_as_float(0x7fc00000);
    }
}

__global__ void __launch_bounds__(128) k_deform_jacobian(CloudView c, double t, int mode,
                                                         double a0_floor, double* d_base,
                                                         double* d_omega, double* d_theta,
                                                         double* d_sigma) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= c.B) return;
    const int N = c.N;
    int rows[5];
    mode_rows(mode, rows);
    double H[5];
    channel_sums(c, b, t, H);
    double factor[5] = {c.a0[b], c.p0[b], c.mu[3 * b], c.mu[3 * b + 1], c.mu[3 * b + 2]};
    double db[5];
    if (mode == PC_COORD_ADDITIVE) {
        factor[2] = factor[3] = factor[4] = 1.0;
        db[0] = 1.0 + H[0];
        db[1] = 1.0 + H[1];
        db[2] = db[3] = db[4] = 1.0;
    } else {
        for (int s = 0; s < 5; ++s) db[s] = 1.0 + H[rows[s]];
    }
    const bool clamped = c.a0[b] * (1.0 + H[0]) < a0_floor;   // strict; NaN floor: none
    if (clamped) db[0] = 0.0;
    for (int s = 0; s < 5; ++s) d_base[5 * b + s] = db[s];
    const double* om = c.omega + (size_t)b * 5 * N;
    for (int s = 0; s < 5; ++s) {
        const int r = rows[s];
        const double fs = (clamped && s == 0) ? 0.0 : factor[s];
        for (int n = 0; n < N; ++n) {
            double ph, d1 = 0.0, d2 = 0.0;
            if (c.kind == PC_BASIS_POLYFOURIER) {
                ph = pf_basis(n, t);
            } else {
                const size_t q = c.per_channel ? ((size_t)b * 5 + r) * N + n : (size_t)b * N + n;
                gauss_pieces(t, c.theta[q], c.sigma[q], ph, d1, d2);
            }
            const size_t o = ((size_t)b * 5 + s) * N + n;
            d_omega[o] = fs * ph;
            if (d_theta) d_theta[o] = fs * om[r * N + n] * d1;
            if (d_sigma) d_sigma[o] = fs * om[r * N + n] * d2;
        }
    }
}

__global__ void __launch_bounds__(128) k_assemble(const float* __restrict__ G, int64_t B, int N,
                                                  const double* __restrict__ d_base,
                                                  const double* __restrict__ d_omega,
                                                  const double* __restrict__ d_theta,
                                                  const double* __restrict__ d_sigma, int4 r03,
                                                  int r4, int shared, int with_ts, double* g_p0,
                                                  double* g_a0, double* g_mu, double* g_theta,
                                                  double* g_sigma, double* g_omega) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    const int rows[5] = {r03.x, r03.y, r03.z, r03.w, r4};
    double Gs[5];
    for (int s = 0; s < 5; ++s) Gs[s] = (double)G[5 * b + s];
    g_a0[b] = Gs[0] * d_base[5 * b + 0];
    g_p0[b] = Gs[1] * d_base[5 * b + 1];
    for (int k = 0; k < 3; ++k) g_mu[3 * b + k] = Gs[2 + k] * d_base[5 * b + 2 + k];
    for (int n = 0; n < N; ++n) {
        double om[5] = {0, 0, 0, 0, 0}, th[5] = {0, 0, 0, 0, 0}, sg[5] = {0, 0, 0, 0, 0};
        double ths = 0.0, sgs = 0.0;
        for (int s = 0; s < 5; ++s) {
            const size_t o = ((size_t)b * 5 + s) * N + n;
            om[rows[s]] += Gs[s] * d_omega[o];
            if (with_ts) {
                const double a = Gs[s] * d_theta[o];
                const double c = Gs[s] * d_sigma[o];
                th[rows[s]] += a;
                sg[rows[s]] += c;
                ths += a;
                sgs += c;
            }
        }
        for (int c = 0; c < 5; ++c) g_omega[((size_t)b * 5 + c) * N + n] = om[c];
        if (with_ts) {
            if (shared) {
                g_theta[(size_t)b * N + n] = ths;
                g_sigma[(size_t)b * N + n] = sgs;
            } else {
                for (int c = 0; c < 5; ++c) {
                    g_theta[((size_t)b * 5 + c) * N + n] = th[c];
                    g_sigma[((size_t)b * 5 + c) * N + n] = sg[c];
                }
            }
        }
    }
}

// Fused chain rule over frames: one warp per ball, lanes over basis index.
// Accumulators live in registers; parameters are re-read per frame through L1.
constexpr int BWD_MAX_SLOTS = 4;  // N <= 128

template <int NS, bool PC>
__global__ void __launch_bounds__(128) k_deform_backward(CloudView c, const double* __restrict__ tf,
                                                         int F, int mode, double a0_floor,
                                                         const float* __restrict__ G,
                                                         const float* __restrict__ Hs,
                                                         pc_cloud_grads_t g) {
    constexpr int NC = PC ? 5 : 1;
    const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (b >= c.B) return;
    const int N = c.N;
    const bool gauss = c.kind == PC_BASIS_GAUSS;
    int rows[5];
    mode_rows(mode, rows);
    const double a0 = c.a0[b], p0 = c.p0[b];
    double factor[5] = {a0, p0, c.mu[3 * b], c.mu[3 * b + 1], c.mu[3 * b + 2]};
    if (mode == PC_COORD_ADDITIVE) factor[2] = factor[3] = factor[4] = 1.0;
    const double* om = c.omega + (size_t)b * 5 * N;
    const double* th = gauss ? c.theta + (size_t)b * NC * N : nullptr;
    const double* sg = gauss ? c.sigma + (size_t)b * NC * N : nullptr;

    double aom[5][NS], ath[NC][NS], asg[NC][NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) {
#pragma unroll
        for (int ch = 0; ch < 5; ++ch) aom[ch][k] = 0.0;
#pragma unroll
        for (int ch = 0; ch < NC; ++ch) ath[ch][k] = asg[ch][k] = 0.0;
    }
    double gb[5] = {0, 0, 0, 0, 0};
    for (int f = 0; f < F; ++f) {
        const double t = tf[f];
        const size_t s5 = 5 * ((size_t)f * c.B + b);
        double Gs[5], H[5];
#pragma unroll
        for (int s = 0; s < 5; ++s) {
            Gs[s] = (double)G[s5 + s];
            H[s] = (double)Hs[s5 + s];
        }
        const bool clamped = isnan(H[0]);   // decided in fp64 by k_deform_states
        double db[5];
        if (mode == PC_COORD_ADDITIVE) {
            db[0] = 1.0 + H[0];
            db[1] = 1.0 + H[1];
            db[2] = db[3] = db[4] = 1.0;
        } else {
#pragma unroll
            for (int s = 0; s < 5; ++s) db[s] = 1.0 + H[rows[s]];
        }
        if (clamped) db[0] = 0.0;
        double W[5] = {0, 0, 0, 0, 0};
#pragma unroll
        for (int s = 0; s < 5; ++s) {
            gb[s] = fma(Gs[s], db[s], gb[s]);
            const double w = (clamped && s == 0) ? 0.0 : Gs[s] * factor[s];
            W[rows[s]] += w;
        }
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            const int n = lane + 32 * k;
            if (n >= N) continue;
            if (!gauss) {
                const double ph = pf_basis(n, t);
#pragma unroll
                for (int ch = 0; ch < 5; ++ch) aom[ch][k] = fma(W[ch], ph, aom[ch][k]);
            } else if (!PC) {
                double ph, d1, d2;
                gauss_pieces(t, th[n], sg[n], ph, d1, d2);
                double S = 0.0;
#pragma unroll
                for (int ch = 0; ch < 5; ++ch) {
                    aom[ch][k] = fma(W[ch], ph, aom[ch][k]);
                    S = fma(W[ch], om[ch * N + n], S);
                }
                ath[0][k] = fma(S, d1, ath[0][k]);
                asg[0][k] = fma(S, d2, asg[0][k]);
            } else {
#pragma unroll
                for (int ch = 0; ch < NC; ++ch) {
                    double ph, d1, d2;
                    gauss_pieces(t, th[ch * N + n], sg[ch * N + n], ph, d1, d2);
                    aom[ch][k] = fma(W[ch], ph, aom[ch][k]);
                    const double S = W[ch] * om[ch * N + n];
                    ath[ch][k] = fma(S, d1, ath[ch][k]);
                    asg[ch][k] = fma(S, d2, asg[ch][k]);
                }
            }
        }
    }
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        const int n = lane + 32 * k;
        if (n >= N) continue;
#pragma unroll
        for (int ch = 0; ch < 5; ++ch) g.omega[((size_t)b * 5 + ch) * N + n] = (float)aom[ch][k];
        if (gauss) {
#pragma unroll
            for (int ch = 0; ch < NC; ++ch) {
                g.theta[((size_t)b * NC + ch) * N + n] = (float)ath[ch][k];
                g.sigma[((size_t)b * NC + ch) * N + n] = (float)asg[ch][k];
            }
        }
    }
    if (lane == 0) {
        g.a0[b] = (float)gb[0];
        g.p0[b] = (float)gb[1];
        g.mu[3 * b + 0] = (float)gb[2];
        g.mu[3 * b + 1] = (float)gb[3];
        g.mu[3 * b + 2] = (float)gb[4];
    }
}

// Poly+Fourier chain rule: the basis depends on t only, so one CTA tabulates
// it per frame in shared memory; LPB lanes per ball (next power of two >= N),
// lane n owning basis index n: no transcendental per ball and no idle lanes
// (N = 8: 16 balls per 128-thread CTA).  Same fp64 arithmetic per lane as
// k_deform_backward.
template <int LPB>
__global__ void __launch_bounds__(128) k_deform_backward_pf(CloudView c,
                                                            const double* __restrict__ tf, int F,
                                                            int mode, double a0_floor,
                                                            const float* __restrict__ G,
                                                            const float* __restrict__ Hs,
                                                            pc_cloud_grads_t g) {
    extern __shared__ double table[];                // (F, N)
    const int N = c.N;
    for (int i = threadIdx.x; i < F * N; i += blockDim.x) table[i] = pf_basis(i % N, tf[i / N]);
    __syncthreads();
    const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPB;
    const int n = threadIdx.x % LPB;
    if (b >= c.B) return;
    int rows[5];
    mode_rows(mode, rows);
    const double a0 = c.a0[b], p0 = c.p0[b];
    double factor[5] = {a0, p0, c.mu[3 * b], c.mu[3 * b + 1], c.mu[3 * b + 2]};
    if (mode == PC_COORD_ADDITIVE) factor[2] = factor[3] = factor[4] = 1.0;
    double aom[5] = {0, 0, 0, 0, 0}, gb[5] = {0, 0, 0, 0, 0};
    for (int f = 0; f < F; ++f) {
        const size_t s5 = 5 * ((size_t)f * c.B + b);
        double Gs[5], H[5];
#pragma unroll
        for (int s = 0; s < 5; ++s) {
            Gs[s] = (double)G[s5 + s];
            H[s] = (double)Hs[s5 + s];
        }
        const bool clamped = isnan(H[0]);   // decided in fp64 by k_deform_states
        double db[5];
        if (mode == PC_COORD_ADDITIVE) {
            db[0] = 1.0 + H[0];
            db[1] = 1.0 + H[1];
            db[2] = db[3] = db[4] = 1.0;
        } else {
#pragma unroll
            for (int s = 0; s < 5; ++s) db[s] = 1.0 + H[rows[s]];
        }
        if (clamped) db[0] = 0.0;
        double W[5] = {0, 0, 0, 0, 0};
#pragma unroll
        for (int s = 0; s < 5; ++s) {
            gb[s] = fma(Gs[s], db[s], gb[s]);
            const double w = (clamped && s == 0) ? 0.0 : Gs[s] * factor[s];
            W[rows[s]] += w;
        }
        if (n < N) {
            const double ph = table[f * N + n];
#pragma unroll
            for (int ch = 0; ch < 5; ++ch) aom[ch] = fma(W[ch], ph, aom[ch]);
        }
    }
    if (n < N) {
#pragma unroll
        for (int ch = 0; ch < 5; ++ch) g.omega[((size_t)b * 5 + ch) * N + n] = (float)aom[ch];
    }
    if (n == 0) {
        g.a0[b] = (float)gb[0];
        g.p0[b] = (float)gb[1];
        g.mu[3 * b + 0] = (float)gb[2];
        g.mu[3 * b + 1] = (float)gb[3];
        g.mu[3 * b + 2] = (float)gb[4];
    }
}

template <bool PC>
static void launch_bwd(int ns, unsigned blocks, cudaStream_t st, const CloudView& c,
                       const double* tf, int F, int mode, double floor_, const float* G,
                       const float* H, const pc_cloud_grads_t& g) {
    switch (ns) {
        case 1: k_deform_backward<1, PC><<<blocks, 128, 0, st>>>(c, tf, F, mode, floor_, G, H, g); break;
        case 2: k_deform_backward<2, PC><<<blocks, 128, 0, st>>>(c, tf, F, mode, floor_, G, H, g); break;
        case 3: k_deform_backward<3, PC><<<blocks, 128, 0, st>>>(c, tf, F, mode, floor_, G, H, g); break;
        default: k_deform_backward<4, PC><<<blocks, 128, 0, st>>>(c, tf, F, mode, floor_, G, H, g); break;
    }
}

}  // namespace pc

using namespace pc;

extern "C" int pc_deform_states(const pc_cloud_t* cloud, const double* t_frames_dev,
                                int32_t n_frames, int32_t coord_mode, double a0_floor,
                                double* mu_t, float* a0_t, float* p0_t, float* H,
                                pc_stream_t stream) {
    CloudView c;
    if (!view_of(cloud, c) || n_frames < 1 || coord_mode < 0 || coord_mode > 2)
        return PC_ERR_ARGUMENT;
    if (c.B == 0) return PC_OK;
    if (!t_frames_dev || !mu_t || !a0_t || !p0_t) return PC_ERR_ARGUMENT;
    const int64_t n = c.B * n_frames;
    k_deform_states<float><<<(unsigned)((n + 127) / 128), 128, 0, as_stream(stream)>>>(
        c, t_frames_dev, n_frames, coord_mode, a0_floor, mu_t, a0_t, p0_t, H);
    return last_status();
}

extern "C" int pc_deform_states_f64(const pc_cloud_t* cloud, const double* t_frames_dev,
                                    int32_t n_frames, int32_t coord_mode, double a0_floor,
                                    double* mu_t, double* a0_t, double* p0_t,
                                    pc_stream_t stream) {
    CloudView c;
    if (!view_of(cloud, c) || n_frames < 1 || coord_mode < 0 || coord_mode > 2)
        return PC_ERR_ARGUMENT;
    if (c.B == 0) return PC_OK;
    if (!t_frames_dev || !mu_t || !a0_t || !p0_t) return PC_ERR_ARGUMENT;
    const int64_t n = c.B * n_frames;
    k_deform_states<double><<<(unsigned)((n + 127) / 128), 128, 0, as_stream(stream)>>>(
        c, t_frames_dev, n_frames, coord_mode, a0_floor, mu_t, a0_t, p0_t, nullptr);
    return last_status();
}

extern "C" int pc_deform_jacobian(const pc_cloud_t* cloud, double t, int32_t coord_mode,
                                  double a0_floor, double* d_base, double* d_omega,
                                  double* d_theta, double* d_sigma, pc_stream_t stream) {
    CloudView c;
    if (!view_of(cloud, c) || coord_mode < 0 || coord_mode > 2) return PC_ERR_ARGUMENT;
    if (c.B == 0) return PC_OK;
    if (!d_base || !d_omega) return PC_ERR_ARGUMENT;
    if (c.kind == PC_BASIS_GAUSS && (!d_theta || !d_sigma)) return PC_ERR_ARGUMENT;
    k_deform_jacobian<<<(unsigned)((c.B + 127) / 128), 128, 0, as_stream(stream)>>>(
        c, t, coord_mode, a0_floor, d_base, d_omega, d_theta, d_sigma);
    return last_status();
}

extern "C" int pc_assemble_grads(const float* G, int64_t n_balls, int32_t n_basis,
                                 const double* d_base, const double* d_omega,
                                 const double* d_theta, const double* d_sigma,
                                 const int32_t* omega_row_host, int32_t shared,
                                 int32_t with_theta_sigma, double* g_p0, double* g_a0,
                                 double* g_mu, double* g_theta, double* g_sigma, double* g_omega,
                                 pc_stream_t stream) {
    if (n_balls < 0 || n_basis < 1 || !omega_row_host) return PC_ERR_ARGUMENT;
    if (n_balls == 0) return PC_OK;
    for (int s = 0; s < 5; ++s)
        if (omega_row_host[s] < 0 || omega_row_host[s] > 4) return PC_ERR_ARGUMENT;
    if (!G || !d_base || !d_omega || !g_p0 || !g_a0 || !g_mu || !g_omega) return PC_ERR_ARGUMENT;
    if (with_theta_sigma && (!d_theta || !d_sigma || !g_theta || !g_sigma)) return PC_ERR_ARGUMENT;
    int4 r03 = make_int4(omega_row_host[0], omega_row_host[1], omega_row_host[2],
                         omega_row_host[3]);
    k_assemble<<<(unsigned)((n_balls + 127) / 128), 128, 0, as_stream(stream)>>>(
        G, n_balls, n_basis, d_base, d_omega, d_theta, d_sigma, r03, omega_row_host[4], shared,
        with_theta_sigma, g_p0, g_a0, g_mu, g_theta, g_sigma, g_omega);
    return last_status();
}

extern "C" int pc_deform_backward(const pc_cloud_t* cloud, const double* t_frames_dev,
                                  int32_t n_frames, int32_t coord_mode, double a0_floor,
                                  const float* G, const float* H, const pc_cloud_grads_t* grads,
                                  pc_stream_t stream) {
    CloudView c;
    if (!view_of(cloud, c) || n_frames < 1 || coord_mode < 0 || coord_mode > 2 || !grads)
        return PC_ERR_ARGUMENT;
    if (c.B == 0) return PC_OK;
    if (!t_frames_dev || !G || !H || !grads->p0 || !grads->a0 || !grads->mu || !grads->omega)
        return PC_ERR_ARGUMENT;
    if (c.kind == PC_BASIS_GAUSS && (!grads->theta || !grads->sigma)) return PC_ERR_ARGUMENT;
    const int ns = (c.N + 31) / 32;
    if (ns > BWD_MAX_SLOTS) return PC_ERR_UNSUPPORTED;
    const unsigned blocks = (unsigned)((c.B * 32 + 127) / 128);
    cudaStream_t st = as_stream(stream);
    pc_cloud_grads_t g = *grads;
    const size_t table_bytes = (size_t)n_frames * c.N * sizeof(double);
    if (c.kind == PC_BASIS_POLYFOURIER && c.N <= 16 && table_bytes <= 32768) {
        if (c.N <= 8)
            k_deform_backward_pf<8><<<(unsigned)((c.B * 8 + 127) / 128), 128, table_bytes, st>>>(
                c, t_frames_dev, n_frames, coord_mode, a0_floor, G, H, g);
        else
            k_deform_backward_pf<16><<<(unsigned)((c.B * 16 + 127) / 128), 128, table_bytes, st>>>(
                c, t_frames_dev, n_frames, coord_mode, a0_floor, G, H, g);
        return last_status();
    }
    if (c.kind == PC_BASIS_GAUSS && c.per_channel)
        launch_bwd<true>(ns, blocks, st, c, t_frames_dev, n_frames, coord_mode, a0_floor, G, H, g);
    else
        launch_bwd<false>(ns, blocks, st, c, t_frames_dev, n_frames, coord_mode, a0_floor, G, H, g);
    return last_status();
}

// ---------------------------------------------------------------- basis helpers
//
// deformation.py:57-70 eval_basis: exp(-(t - theta)^2 / (2 sigma^2)),
// elementwise over already-broadcast fp64 inputs; and :73-84 eval_H's
// weighted sum over one basis vector, in index order by one thread.
__global__ void __launch_bounds__(256) k_eval_basis(const double* __restrict__ t,
                                                    const double* __restrict__ theta,
                                                    const double* __restrict__ sigma, int64_t n,
                                                    double* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double d = (t[i] - theta[i]) / sigma[i];
        out[i] = exp(-0.5 * d * d);
    }
}

__global__ void k_basis_dot(double t, const double* __restrict__ omega,
                            const double* __restrict__ theta, const double* __restrict__ sigma,
                            int n, double* __restrict__ out) {
    double h = 0.0;
    for (int i = 0; i < n; ++i) {
        const double d = (t - theta[i]) / sigma[i];
        h = fma(omega[i], exp(-0.5 * d * d), h);
    }
    out[0] = h;
}

extern "C" int pc_eval_basis(const double* t, const double* theta, const double* sigma,
                             int64_t n, double* out, pc_stream_t stream) {
    if (n < 0) return PC_ERR_ARGUMENT;
    if (n == 0) return PC_OK;
    if (!t || !theta || !sigma || !out) return PC_ERR_ARGUMENT;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 8LL * num_sms()) blocks = 8LL * num_sms();
    k_eval_basis<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(t, theta, sigma, n, out);
    return last_status();
}

extern "C" int pc_eval_h(double t, const double* omega, const double* theta, const double* sigma,
                         int32_t n, double* out, pc_stream_t stream) {
    if (n < 0 || !out || (n > 0 && (!omega || !theta || !sigma))) return PC_ERR_ARGUMENT;
    k_basis_dot<<<1, 1, 0, as_stream(stream)>>>(t, omega, theta, sigma, n, out);
    return last_status();
}
