// Universal back-projection.
//
// Restates pacloud/reconstruction.py:352-417:
//   filter (ubp_reconstruct :397-398): b_m(t_j) = 2 p_m(t_j) - 2 t_j dp_m/dt,
//     dp/dt = numpy.gradient (central differences, one-sided at both ends),
//     t_j = t_start + j / sample_rate;
//   back-projection (_backproject :352-377): per voxel x
//     V(x) = (1/M) sum_m lerp(b_m, u),  u = (|x - s_m| / v - t0) / dt,
//     j = int(u) clamped to T - 2, frac = u - j.
//
// k_ubp_filter: one thread per sample, fp64 arithmetic, f32 output.
// k_backproject: one thread per voxel on 8 (z) x 8 (y) x 4 (x) tiles (the
// 256 voxels of a CTA see neighbouring times of flight, so the trace gathers
// hit L1); sensors in chunks of 256 staged in shared memory; the distance is
// the fp32 sqrt of the fp64 squared distance refined by one fp64 Newton
// step, so u (and j) carry the reference's fp64 precision; terms accumulate
// in fp32 in sensor order (deterministic), scaled by 1/M at the end.

#include "common.cuh"

namespace pc {

constexpr int BP_THREADS = 256;
constexpr int BP_CHUNK = 256;

__global__ void __launch_bounds__(256) k_ubp_filter(const double* __restrict__ traces, int M,
                                                    int T, double t0, double fs,
                                                    float* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)M * T) return;
    const int j = (int)(i % T);
    const double* p = traces + (i - j);
    const double dt = 1.0 / fs;
    double d;
    if (T < 2)
        d = 0.0;
    else if (j == 0)
        d = (p[1] - p[0]) / dt;
    else if (j == T - 1)
        d = (p[T - 1] - p[T - 2]) / dt;
    else
        d = (p[j + 1] - p[j - 1]) / (2.0 * dt);
    const double t = t0 + (double)j / fs;
    out[i] = (float)(2.0 * p[j] - 2.0 * t * d);
}

struct BpGrid {
    double ox, oy, oz, sp;
    int nx, ny, nz;
    int ntx, nty;   // tiles along x (4) and y (8); z tiles = rest
};

__global__ void __launch_bounds__(BP_THREADS) k_backproject(const float* __restrict__ filt,
                                                            const double* __restrict__ pos,
                                                            int M, int T, double v, double t0,
                                                            double dt, BpGrid g,
                                                            float* __restrict__ out) {
    __shared__ double sx[BP_CHUNK], sy[BP_CHUNK], sz[BP_CHUNK];
    const int tid = threadIdx.x;
    const int t = blockIdx.x;
    const int tx = t % g.ntx, ty = (t / g.ntx) % g.nty, tz = t / (g.ntx * g.nty);
    const int ix = tx * 4 + (tid >> 6), iy = ty * 8 + ((tid >> 3) & 7), iz = tz * 8 + (tid & 7);
    const bool live = ix < g.nx && iy < g.ny && iz < g.nz;
    const double x = g.ox + ix * g.sp, y = g.oy + iy * g.sp, z = g.oz + iz * g.sp;
    const double inv_v = 1.0 / v, inv_dt = 1.0 / dt;
    float acc = 0.f;
    for (int m0 = 0; m0 < M; m0 += BP_CHUNK) {
        const int n = min(BP_CHUNK, M - m0);
        __syncthreads();
        if (tid < n) {
            sx[tid] = pos[3 * (m0 + tid)];
            sy[tid] = pos[3 * (m0 + tid) + 1];
            sz[tid] = pos[3 * (m0 + tid) + 2];
        }
        __syncthreads();
        if (!live) continue;
        for (int k = 0; k < n; ++k) {
            const double dx = x - sx[k], dy = y - sy[k], dz = z - sz[k];
            const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
            const float r2f = (float)r2;
            const float rinv = rsqrtf(r2f);
            const float rf = r2f * rinv;
            const double r = r2f > 0.f
                                 ? fma(fma(-(double)rf, (double)rf, r2), 0.5 * (double)rinv,
                                       (double)rf)
                                 : 0.0;
            const double u = (r * inv_v - t0) * inv_dt;
            int j = (int)u;
            if (j >= T - 1) j = T - 2;
            const float fr = (float)(u - (double)j);
            const float* row = filt + (size_t)(m0 + k) * T + j;
            const float b0 = __ldg(row), b1 = __ldg(row + 1);
            acc += fmaf(fr, b1 - b0, b0);
        }
    }
    if (live) out[((size_t)ix * g.ny + iy) * g.nz + iz] = acc / (float)M;
}

}  // namespace pc

using namespace pc;

extern "C" int pc_ubp_filter(const double* traces, int32_t n_sensors, int32_t n_samples,
                             double t_start, double sample_rate, float* filtered,
                             pc_stream_t stream) {
    if (n_sensors < 0 || n_samples < 0 || !(sample_rate > 0)) return PC_ERR_ARGUMENT;
    const int64_t n = (int64_t)n_sensors * n_samples;
    if (n == 0) return PC_OK;
    if (!traces || !filtered) return PC_ERR_ARGUMENT;
    k_ubp_filter<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(
        traces, n_sensors, n_samples, t_start, sample_rate, filtered);
    return last_status();
}

extern "C" int pc_backproject(const float* filtered, const double* positions, int32_t n_sensors,
                              int32_t n_samples, double sound_speed, double t_start, double dt,
                              const double* origin, double spacing, const int32_t* dims,
                              float* out, pc_stream_t stream) {
    if (!filtered || !positions || !origin || !dims || !out || n_sensors < 1 || n_samples < 2 ||
        !(sound_speed > 0) || !(dt > 0) || !(spacing > 0) || dims[0] < 1 || dims[1] < 1 ||
        dims[2] < 1)
        return PC_ERR_ARGUMENT;
    BpGrid g;
    g.ox = origin[0];
    g.oy = origin[1];
    g.oz = origin[2];
    g.sp = spacing;
    g.nx = dims[0];
    g.ny = dims[1];
    g.nz = dims[2];
    g.ntx = (g.nx + 3) / 4;
    g.nty = (g.ny + 7) / 8;
    const long long tiles = (long long)g.ntx * g.nty * ((g.nz + 7) / 8);
    if (tiles > 0x7fffffffLL) return PC_ERR_ARGUMENT;
    k_backproject<<<(unsigned)tiles, BP_THREADS, 0, as_stream(stream)>>>(
        filtered, positions, n_sensors, n_samples, sound_speed, t_start, dt, g, out);
    return last_status();
}
