// Voxelisation of a ball cloud on a regular grid.
//
// Restates pacloud/evaluation.py:46-93 (_splat_balls / voxelize):
//   V(ix, iy, iz) = sum_b p0_b exp(-|x - mu_b|^2 / (2 a0_b^2)),
//   x = origin + i * spacing (fp64, per axis),
// with the fast path limited to each ball's support cube: along x the voxels
// with |x - mu_x| <= support a0 (:55-57), along y / z the index ranges
// ceil((mu - reach - o) / sp) .. floor((mu + reach - o) / sp) (:62-65).
//
// Layout: one CTA per 8 x 8 x 8 voxel tile, 256 threads x 2 z-adjacent
// voxels.  The CTA walks the balls in index order in chunks of 256, keeps the
// ones whose support cube meets the tile (order-preserving ballot
// compaction into shared memory), and accumulates them in that fixed order:
// deterministic, no atomics.  Offsets to the voxel centre in fp64, the
// Gaussian in fp32 (MUFU ex2), accumulation in fp32.
//
// Cost is O(tiles x balls) cull tests (16-byte coalesced reads of the ball
// ranges) plus the in-support evaluations; evaluation-size grids (<= 256^3,
// <= 1e6 balls) finish in milliseconds.

#include "common.cuh"

namespace pc {

constexpr int VT = 8;            // tile edge (voxels)
constexpr int VTHREADS = 256;    // 2 voxels per thread

struct VoxBall {                 // 64 bytes
    double mx, my, mz;
    float p0, k;                 // k = log2(e) / (2 a0^2)
    int lo[3], hi[3];            // support cube, voxel index ranges [lo, hi)
    int pad[2];
};

// Cull record: per axis lo | hi << 16 (dims <= 32767).
__device__ __forceinline__ int4 cull_of(const VoxBall& r) {
    return make_int4(r.lo[0] | (r.hi[0] << 16), r.lo[1] | (r.hi[1] << 16),
                     r.lo[2] | (r.hi[2] << 16), 0);
}
__device__ __forceinline__ bool meets(int v, int t0, int t1) {
    return (v & 0xffff) < t1 && (v >> 16) > t0;
}

struct VoxGrid {
    double ox, oy, oz, sp, support;
    int nx, ny, nz;
    int exact;
};

__device__ __forceinline__ int clampi(long long v, int lo, int hi) {
    return (int)(v < lo ? lo : (v > hi ? hi : v));
}

// Along x the reference tests |o + i sp - mu| > reach per voxel: find the
// first / last index passing that test exactly (fp64, same expression).
__device__ int x_lo(double mu, double reach, double o, double sp, int n) {
    long long i = (long long)ceil((mu - reach - o) / sp);
    int j = clampi(i, 0, n);
    while (j > 0 && fabs(o + (j - 1) * sp - mu) <= reach) --j;
    while (j < n && fabs(o + j * sp - mu) > reach) ++j;
    return j;
}
__device__ int x_hi(double mu, double reach, double o, double sp, int n, int lo) {
    long long i = (long long)floor((mu + reach - o) / sp) + 1;
    int j = clampi(i, lo, n);
    while (j < n && fabs(o + j * sp - mu) <= reach) ++j;
    while (j > lo && fabs(o + (j - 1) * sp - mu) > reach) --j;
    return j;
}

__global__ void __launch_bounds__(256) k_vox_prep(const double* __restrict__ mu,
                                                  const double* __restrict__ a0,
                                                  const double* __restrict__ p0, int64_t B,
                                                  VoxGrid g, VoxBall* __restrict__ out,
                                                  int4* __restrict__ cull, int* __restrict__ bad) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    VoxBall r;
    r.mx = mu[3 * b];
    r.my = mu[3 * b + 1];
    r.mz = mu[3 * b + 2];
    const double a = a0[b];
    if (!(a > 0)) atomicExch(bad, 1);
    r.p0 = (float)p0[b];
    r.k = (float)(1.0 / (2.0 * a * a) * 1.4426950408889634);
    if (g.exact) {
        r.lo[0] = r.lo[1] = r.lo[2] = 0;
        r.hi[0] = g.nx;
        r.hi[1] = g.ny;
        r.hi[2] = g.nz;
    } else {
        const double reach = g.support * a;
        r.lo[0] = x_lo(r.mx, reach, g.ox, g.sp, g.nx);
        r.hi[0] = x_hi(r.mx, reach, g.ox, g.sp, g.nx, r.lo[0]);
        r.lo[1] = clampi((long long)ceil((r.my - reach - g.oy) / g.sp), 0, g.ny);
        r.hi[1] = clampi((long long)floor((r.my + reach - g.oy) / g.sp) + 1, 0, g.ny);
        r.lo[2] = clampi((long long)ceil((r.mz - reach - g.oz) / g.sp), 0, g.nz);
        r.hi[2] = clampi((long long)floor((r.mz + reach - g.oz) / g.sp) + 1, 0, g.nz);
    }
    r.pad[0] = r.pad[1] = 0;
    out[b] = r;
    cull[b] = cull_of(r);
}

__global__ void __launch_bounds__(VTHREADS) k_vox_tiles(const VoxBall* __restrict__ balls,
                                                        const int4* __restrict__ cull, int64_t B,
                                                        VoxGrid g, int ntx, int nty,
                                                        float* __restrict__ out) {
    __shared__ VoxBall list[VTHREADS];
    __shared__ int wcount[VTHREADS / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int t = blockIdx.x;
    const int tx = t % ntx, ty = (t / ntx) % nty, tz = t / (ntx * nty);
    const int x0 = tx * VT, y0 = ty * VT, z0 = tz * VT;
    const int x1 = min(x0 + VT, g.nx), y1 = min(y0 + VT, g.ny), z1 = min(z0 + VT, g.nz);
    // this thread's voxels: (ix, iy, iz) and (ix, iy, iz + 1)
    const int ix = x0 + (tid >> 5), iy = y0 + ((tid >> 2) & 7), iz = z0 + 2 * (tid & 3);
    const double x = g.ox + ix * g.sp, y = g.oy + iy * g.sp;
    const double z = g.oz + iz * g.sp, z2 = g.oz + (iz + 1) * g.sp;
    float acc0 = 0.f, acc1 = 0.f;
    for (int64_t c = 0; c < B; c += VTHREADS) {
        const int64_t b = c + tid;
        bool hit = false;
        if (b < B) {
            const int4 q = __ldg(cull + b);
            hit = meets(q.x, x0, x1) && meets(q.y, y0, y1) && meets(q.z, z0, z1);
        }
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if (lane == 0) wcount[warp] = __popc(m);
        __syncthreads();
        int base = 0, n = 0;
#pragma unroll
        for (int w = 0; w < VTHREADS / 32; ++w) {
            const int cw = wcount[w];
            base += w < warp ? cw : 0;
            n += cw;
        }
        if (hit) list[base + __popc(m & ((1u << lane) - 1u))] = balls[b];
        __syncthreads();
        for (int k = 0; k < n; ++k) {
            const VoxBall& q = list[k];
            if (ix >= q.lo[0] && ix < q.hi[0] && iy >= q.lo[1] && iy < q.hi[1]) {
                const double dx = x - q.mx, dy = y - q.my;
                const double dxy = dx * dx + dy * dy;
                if (iz >= q.lo[2] && iz < q.hi[2]) {
                    const double dz = z - q.mz;
                    acc0 = fmaf(q.p0, ex2(-(float)(dxy + dz * dz) * q.k), acc0);
                }
                if (iz + 1 >= q.lo[2] && iz + 1 < q.hi[2]) {
                    const double dz = z2 - q.mz;
                    acc1 = fmaf(q.p0, ex2(-(float)(dxy + dz * dz) * q.k), acc1);
                }
            }
        }
        __syncthreads();
    }
    if (ix < x1 && iy < y1) {
        const size_t row = ((size_t)ix * g.ny + iy) * g.nz;
        if (iz < z1) out[row + iz] = acc0;
        if (iz + 1 < z1) out[row + iz + 1] = acc1;
    }
}

}  // namespace pc

using namespace pc;

extern "C" size_t pc_voxelize_workspace_bytes(int64_t n_balls) {
    const size_t n = (size_t)(n_balls > 0 ? n_balls : 0);
    return n * (sizeof(VoxBall) + sizeof(int4)) + 256;
}

extern "C" int pc_voxelize(const double* mu, const double* a0, const double* p0,
                           int64_t n_balls, const double* origin, double spacing,
                           const int32_t* dims, double support_sigmas, int32_t exact, float* out,
                           int32_t* bad_a0, void* workspace, size_t workspace_bytes,
                           pc_stream_t stream) {
    if (!origin || !dims || !out || n_balls < 0 || !(spacing > 0) || dims[0] < 1 ||
        dims[1] < 1 || dims[2] < 1 || dims[0] > 32767 || dims[1] > 32767 || dims[2] > 32767)
        return PC_ERR_ARGUMENT;
    if (n_balls > 0 && (!mu || !a0 || !p0 || !bad_a0)) return PC_ERR_ARGUMENT;
    if (workspace_bytes < pc_voxelize_workspace_bytes(n_balls) || (n_balls > 0 && !workspace))
        return PC_ERR_ARGUMENT;
    cudaStream_t st = as_stream(stream);
    VoxGrid g;
    g.ox = origin[0];
    g.oy = origin[1];
    g.oz = origin[2];
    g.sp = spacing;
    g.support = support_sigmas;
    g.nx = dims[0];
    g.ny = dims[1];
    g.nz = dims[2];
    g.exact = exact ? 1 : 0;
    const size_t nvox = (size_t)g.nx * g.ny * g.nz;
    if (n_balls == 0) return status_of(cudaMemsetAsync(out, 0, nvox * sizeof(float), st));
    VoxBall* balls = reinterpret_cast<VoxBall*>(
        (reinterpret_cast<uintptr_t>(workspace) + 127) & ~(uintptr_t)127);
    int4* cull = reinterpret_cast<int4*>(balls + n_balls);
    k_vox_prep<<<(unsigned)((n_balls + 255) / 256), 256, 0, st>>>(mu, a0, p0, n_balls, g, balls,
                                                                   cull, bad_a0);
    const int ntx = (g.nx + VT - 1) / VT, nty = (g.ny + VT - 1) / VT, ntz = (g.nz + VT - 1) / VT;
    const long long tiles = (long long)ntx * nty * ntz;
    if (tiles > 0x7fffffffLL) return PC_ERR_ARGUMENT;
    k_vox_tiles<<<(unsigned)tiles, VTHREADS, 0, st>>>(balls, cull, n_balls, g, ntx, nty, out);
    return last_status();
}
