// Loss, optimiser and compaction kernels (HBM-bound) for sm_100a.
//
//   pc_l2_loss          <- pkg/src/pacloud/reconstruction.py:28-35 (l2_loss)
//   pc_check_finite     <- reconstruction.py:60-61, 74-75 (non-finite guard)
//   pc_adam_segments    <- reconstruction.py:57-69 (adam_step) x the four
//                          ParamGroups (:320-327) + _clamp_floors (:153-157)
//   pc_sgd_segments     <- reconstruction.py:72-76 (sgd_step)
//   pc_prune_mask       <- reconstruction.py:217-220 (keep = p0 > thr*max p0)
//   pc_compact_index    <- reconstruction.py:95-100 (stable boolean gather)
//   pc_gather_rows      <- the gather itself, for params and Adam moments
//   pc_abs_quantile_f32 <- config-5 densify threshold: numpy.percentile(|g|,
//                          q, 'linear') by device radix select (builder rule)
//   pc_densify_masks / pc_densify_flags / pc_densify_apply <- config-5 split
//                          + absolute prune (builder-defined)
#include <math.h>

#include "common.cuh"

namespace pc {

// ---------------------------------------------------------------- l2 loss

__global__ void __launch_bounds__(1024) k_l2(const double* __restrict__ p,
                                             const double* __restrict__ o, int64_t n,
                                             double* __restrict__ out) {
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double d = p[i] - o[i];
        s = fma(d, d, s);
    }
    __shared__ double red[32];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        t = warp_sum(t);
        if (threadIdx.x == 0) out[0] = 0.5 * t;
    }
}

// ---------------------------------------------------------------- segments

struct SegTable {
    int64_t off[PC_MAX_SEGMENTS + 1];
    double lr[PC_MAX_SEGMENTS];
    double bc1[PC_MAX_SEGMENTS];
    double bc2[PC_MAX_SEGMENTS];
    double floor_[PC_MAX_SEGMENTS];
    int n;
};

template <typename GT>
__global__ void __launch_bounds__(256) k_finite(const GT* __restrict__ x, SegTable t,
                                                int* __restrict__ flags) {
    const int s = blockIdx.y;
    const int64_t lo = t.off[s], hi = t.off[s + 1];
    int bad = 0;
    for (int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi;
         i += (int64_t)gridDim.x * blockDim.x)
        bad |= !isfinite(x[i]);
    bad = __syncthreads_or(bad);
    if (bad && threadIdx.x == 0) atomicOr(flags + s, 1);
}

constexpr double kBeta1 = 0.9, kBeta2 = 0.999, kEps = 1e-8;  // reconstruction.py:23-25

template <typename GT>
__global__ void __launch_bounds__(256) k_adam(double* __restrict__ p, const GT* __restrict__ g,
                                              double* __restrict__ m, double* __restrict__ v,
                                              SegTable t) {
    const int s = blockIdx.y;
    const int64_t lo = t.off[s], hi = t.off[s + 1];
    const double lr = t.lr[s], bc1 = t.bc1[s], bc2 = t.bc2[s], fl = t.floor_[s];
    for (int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double gi = (double)g[i];
        double mi = m[i] * kBeta1;
        mi = mi + (1.0 - kBeta1) * gi;
        double vi = v[i] * kBeta2;
        vi = vi + (1.0 - kBeta2) * gi * gi;
        m[i] = mi;
        v[i] = vi;
        const double mh = mi / bc1;
        const double vh = vi / bc2;
        double pi = p[i] - lr * mh / (sqrt(vh) + kEps);
        p[i] = pi < fl ? fl : pi;
    }
}

template <typename GT>
__global__ void __launch_bounds__(256) k_sgd(double* __restrict__ p, const GT* __restrict__ g,
                                             SegTable t) {
    const int s = blockIdx.y;
    const int64_t lo = t.off[s], hi = t.off[s + 1];
    const double lr = t.lr[s], fl = t.floor_[s];
    for (int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double pi = p[i] - lr * (double)g[i];
        p[i] = pi < fl ? fl : pi;
    }
}

static bool seg_table(int n_seg, const int64_t* off, SegTable& t) {
    if (n_seg < 1 || n_seg > PC_MAX_SEGMENTS || !off) return false;
    t.n = n_seg;
    for (int s = 0; s <= n_seg; ++s) {
        t.off[s] = off[s];
        if (s > 0 && off[s] < off[s - 1]) return false;
    }
    if (off[0] < 0) return false;
    return true;
}

static unsigned seg_blocks(const SegTable& t) {
    int64_t widest = 0;
    for (int s = 0; s < t.n; ++s) widest = t.off[s + 1] - t.off[s] > widest ? t.off[s + 1] - t.off[s] : widest;
    int64_t b = (widest + 255) / 256;
    const int64_t cap = 8LL * num_sms();
    if (b > cap) b = cap;
    return (unsigned)(b < 1 ? 1 : b);
}

// ---------------------------------------------------------------- compaction

constexpr int CMP_BLOCK = 1024;

__global__ void __launch_bounds__(1024) k_max(const double* __restrict__ x, int64_t n,
                                              double* __restrict__ out) {
    double mx = 0.0;  // np.max(p0, initial=0.0)
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) mx = fmax(mx, x[i]);
    __shared__ double red[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = fmax(t, red[w]);
        out[0] = t;
    }
}

__global__ void __launch_bounds__(256) k_prune(const double* __restrict__ p0, int64_t n, double rel,
                                               const double* __restrict__ maxv,
                                               uint8_t* __restrict__ keep,
                                               unsigned long long* __restrict__ count) {
    const double thr = rel * maxv[0];
    int c = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t k = p0[i] > thr ? 1 : 0;
        keep[i] = k;
        c += k;
    }
    c = __syncthreads_count(c);
    if (threadIdx.x == 0 && c) atomicAdd(count, (unsigned long long)c);
}

__global__ void __launch_bounds__(CMP_BLOCK) k_block_counts(const uint8_t* __restrict__ keep,
                                                            const uint8_t* __restrict__ app,
                                                            int64_t n, int64_t* __restrict__ ck,
                                                            int64_t* __restrict__ ca) {
    const int64_t i = (int64_t)blockIdx.x * CMP_BLOCK + threadIdx.x;
    const int k = i < n && keep[i] ? 1 : 0;
    const int a = i < n && app && app[i] ? 1 : 0;
    const int sk = __syncthreads_count(k);
    const int sa = __syncthreads_count(a);
    if (threadIdx.x == 0) {
        ck[blockIdx.x] = sk;
        ca[blockIdx.x] = sa;
    }
}

// exclusive scan of the per-block counts (single block, fixed order)
__global__ void __launch_bounds__(1024) k_scan_counts(int64_t* __restrict__ ck,
                                                      int64_t* __restrict__ ca, int nblk,
                                                      int64_t* __restrict__ n_out) {
    __shared__ int64_t sk[1024], sa[1024];
    __shared__ int64_t carry_k, carry_a;
    if (threadIdx.x == 0) carry_k = carry_a = 0;
    __syncthreads();
    for (int base = 0; base < nblk; base += 1024) {
        const int i = base + threadIdx.x;
        sk[threadIdx.x] = i < nblk ? ck[i] : 0;
        sa[threadIdx.x] = i < nblk ? ca[i] : 0;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {  // Hillis-Steele inclusive scan
            int64_t xk = threadIdx.x >= o ? sk[threadIdx.x - o] : 0;
            int64_t xa = threadIdx.x >= o ? sa[threadIdx.x - o] : 0;
            __syncthreads();
            sk[threadIdx.x] += xk;
            sa[threadIdx.x] += xa;
            __syncthreads();
        }
        if (i < nblk) {
            const int64_t ek = (threadIdx.x ? sk[threadIdx.x - 1] : 0) + carry_k;
            const int64_t ea = (threadIdx.x ? sa[threadIdx.x - 1] : 0) + carry_a;
            ck[i] = ek;
            ca[i] = ea;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            carry_k += sk[1023];
            carry_a += sa[1023];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        n_out[0] = carry_k + carry_a;
        n_out[1] = carry_k;  // survivors (children start here)
    }
}

__global__ void __launch_bounds__(CMP_BLOCK) k_scatter_index(const uint8_t* __restrict__ keep,
                                                             const uint8_t* __restrict__ app,
                                                             int64_t n,
                                                             const int64_t* __restrict__ ck,
                                                             const int64_t* __restrict__ ca,
                                                             const int64_t* __restrict__ n_out,
                                                             int64_t* __restrict__ index) {
    __shared__ int wk[32], wa[32];
    const int64_t i = (int64_t)blockIdx.x * CMP_BLOCK + threadIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool k = i < n && keep[i];
    const bool a = i < n && app && app[i];
    const unsigned bk = __ballot_sync(0xffffffffu, k);
    const unsigned ba = __ballot_sync(0xffffffffu, a);
    if (lane == 0) {
        wk[warp] = __popc(bk);
        wa[warp] = __popc(ba);
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // exclusive scan over 32 warps
        int rk = 0, ra = 0;
        for (int w = 0; w < 32; ++w) {
            const int tk = wk[w], ta = wa[w];
            wk[w] = rk;
            wa[w] = ra;
            rk += tk;
            ra += ta;
        }
    }
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
    if (k) index[ck[blockIdx.x] + wk[warp] + __popc(bk & lt)] = i;
    if (a) index[n_out[1] + ca[blockIdx.x] + wa[warp] + __popc(ba & lt)] = i;
}

__global__ void __launch_bounds__(256) k_gather(const uint32_t* __restrict__ src,
                                                uint32_t* __restrict__ dst,
                                                const int64_t* __restrict__ index, int64_t rows,
                                                int64_t words) {
    const int64_t total = rows * words;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = q / words, w = q - r * words;
        dst[q] = src[index[r] * words + w];
    }
}

__global__ void __launch_bounds__(256) k_densify_masks(const double* __restrict__ p0,
                                                       const float* __restrict__ g, int64_t n,
                                                       double p0_min,
                                                       const double* __restrict__ thr_dev,
                                                       uint8_t* __restrict__ keep,
                                                       uint8_t* __restrict__ split,
                                                       unsigned long long* __restrict__ counts) {
    (void)counts;
    const double thr = *thr_dev;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t k = (p0[i] < p0_min) ? 0 : 1;
        const uint8_t s = (k && fabs((double)g[i]) > thr) ? 1 : 0;
        keep[i] = k;
        split[i] = s;
    }
}

__global__ void __launch_bounds__(256) k_count_u8(const uint8_t* __restrict__ a,
                                                  const uint8_t* __restrict__ b, int64_t n,
                                                  unsigned long long* __restrict__ counts) {
    unsigned long long ca = 0, cb = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        ca += a[i];
        cb += b[i];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ca += __shfl_xor_sync(0xffffffffu, ca, o);
        cb += __shfl_xor_sync(0xffffffffu, cb, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(counts, ca);
        atomicAdd(counts + 1, cb);
    }
}


// ------------------------------------------------ order statistic of |g|
// numpy.percentile(|g|, q, method='linear') on the device (config-5 densify
// threshold; numpy/lib/_function_base_impl.py _quantile + _lerp): the host
// passes numpy's virtual-index split k = floor((n-1) q), gamma = (n-1) q - k
// (it depends on n and q only); the device finds the order statistics
// x_(k), x_(k+1) of |g| by an MSB-first 8-bit radix select on the float
// bit patterns (non-negative floats order like their uint32 bits) and
// applies numpy's lerp with explicit round-to-nearest double operations.

struct QuantState {
    unsigned int prefix;     // selected high digits of x_(k)
    unsigned int mask;       // digits fixed so far
    long long rank;          // rank of x_(k) among the elements matching prefix
    unsigned int a_bits;     // x_(k) when done
    unsigned int min_gt;     // min |g| > x_(k)      (atomicMin)
    unsigned long long n_le; // #{|g| <= x_(k)}       (atomicAdd)
};

__device__ __forceinline__ unsigned int abs_bits(float x) {
    return __float_as_uint(x) & 0x7fffffffu;
}

__global__ void __launch_bounds__(256) k_radix_hist(const float* __restrict__ g, int64_t n,
                                                    const QuantState* __restrict__ st,
                                                    int shift,
                                                    unsigned int* __restrict__ hist) {
    __shared__ unsigned int h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const unsigned int prefix = st->prefix, mask = st->mask;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned int u = abs_bits(g[i]);
        if ((u & mask) == prefix) atomicAdd(&h[(u >> shift) & 0xffu], 1u);
    }
    __syncthreads();
    if (h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], h[threadIdx.x]);
}

// one block of 256: pick the digit holding `rank`, clear the histogram
__global__ void __launch_bounds__(256) k_radix_pick(QuantState* __restrict__ st, int shift,
                                                    unsigned int* __restrict__ hist) {
    __shared__ unsigned int c[256];
    const int t = threadIdx.x;
    c[t] = hist[t];
    hist[t] = 0;
    __syncthreads();
    // inclusive scan (Hillis-Steele; 256 entries)
    for (int o = 1; o < 256; o <<= 1) {
        const unsigned int v = t >= o ? c[t - o] : 0u;
        __syncthreads();
        c[t] += v;
        __syncthreads();
    }
    const long long r = st->rank;
    const unsigned long long lo = t ? c[t - 1] : 0u;
    if ((long long)lo <= r && r < (long long)c[t]) {
        st->prefix |= (unsigned int)t << shift;
        st->mask |= 0xffu << shift;
        st->rank = r - (long long)lo;
        if (shift == 0) {
            st->a_bits = st->prefix;
            st->min_gt = 0x7f800000u;   // +inf
            st->n_le = 0;
        }
    }
}

__global__ void __launch_bounds__(256) k_quant_next(const float* __restrict__ g, int64_t n,
                                                    QuantState* __restrict__ st) {
    const unsigned int a = st->a_bits;
    unsigned int mn = 0x7f800000u;
    unsigned long long le = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned int u = abs_bits(g[i]);
        if (u <= a) ++le;
        else mn = min(mn, u);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        le += __shfl_xor_sync(0xffffffffu, le, o);
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&st->n_le, le);
        atomicMin(&st->min_gt, mn);
    }
}

__global__ void k_quant_lerp(const QuantState* __restrict__ st, int64_t k, int64_t n,
                             double gamma, double* __restrict__ out) {
    const double a = (double)__uint_as_float(st->a_bits);
    // x_(k+1): x_(k) again while more than k+1 elements are <= x_(k)
    const bool same = k + 1 >= n || (long long)st->n_le > k + 1;
    const double b = same ? a : (double)__uint_as_float(st->min_gt);
    const double diff = __dsub_rn(b, a);
    // numpy _lerp: a + diff*t, replaced by b - diff*(1-t) where t >= 0.5
    out[0] = gamma >= 0.5 ? __dsub_rn(b, __dmul_rn(diff, __dsub_rn(1.0, gamma)))
                          : __dadd_rn(a, __dmul_rn(diff, gamma));
}

// ------------------------------------------------ densify flags
// After pc_compact_index(keep, split): index[0, n_keep) survivors,
// index[n_keep, n_out) children (parent ids).  has_child[b] marks parents
// whose child made it into [n_keep, n_out) (a max-balls cap truncates the
// children); halve[i] = parent of a child, or a child; child[i] = i >= n_keep.
__global__ void __launch_bounds__(256) k_mark_parents(const int64_t* __restrict__ index,
                                                      int64_t n_keep, int64_t n_out,
                                                      uint8_t* __restrict__ has_child) {
    for (int64_t r = n_keep + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_out;
         r += (int64_t)gridDim.x * blockDim.x)
        has_child[index[r]] = 1;
}

__global__ void __launch_bounds__(256) k_densify_flags(const int64_t* __restrict__ index,
                                                       int64_t n_keep, int64_t n_out,
                                                       const uint8_t* __restrict__ has_child,
                                                       uint8_t* __restrict__ halve,
                                                       uint8_t* __restrict__ child) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_out;
         i += (int64_t)gridDim.x * blockDim.x) {
        const bool c = i >= n_keep;
        child[i] = c ? 1 : 0;
        halve[i] = (c || has_child[index[i]]) ? 1 : 0;
    }
}

__global__ void __launch_bounds__(256) k_densify_apply(double* __restrict__ p0,
                                                       double* __restrict__ mu,
                                                       const double* __restrict__ a0,
                                                       const uint8_t* __restrict__ halve,
                                                       const uint8_t* __restrict__ child,
                                                       int64_t n, double shift) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (halve && halve[i]) p0[i] = 0.5 * p0[i];
        if (child[i]) mu[3 * i] = mu[3 * i] + shift * a0[i];
    }
}

}  // namespace pc

using namespace pc;

extern "C" size_t pc_abs_quantile_workspace_bytes(void) {
    return sizeof(QuantState) + 256 * sizeof(unsigned int) + 64;
}

extern "C" int pc_abs_quantile_f32(const float* g, int64_t n, int64_t k, double gamma,
                                   double* threshold, void* workspace, size_t workspace_bytes,
                                   pc_stream_t stream) {
    if (n < 1 || k < 0 || k >= n || !(gamma >= 0.0 && gamma < 1.0) || !g || !threshold ||
        !workspace || workspace_bytes < pc_abs_quantile_workspace_bytes())
        return PC_ERR_ARGUMENT;
    cudaStream_t st = as_stream(stream);
    QuantState* qs = reinterpret_cast<QuantState*>(workspace);
    unsigned int* hist = reinterpret_cast<unsigned int*>(
        reinterpret_cast<char*>(workspace) + ((sizeof(QuantState) + 63) / 64) * 64);
    QuantState init{};
    init.rank = k;
    if (cudaMemcpyAsync(qs, &init, sizeof(init), cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaMemsetAsync(hist, 0, 256 * sizeof(unsigned int), st) != cudaSuccess)
        return PC_ERR_CUDA;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 4LL * num_sms()) blocks = 4LL * num_sms();
    for (int shift = 24; shift >= 0; shift -= 8) {
        k_radix_hist<<<(unsigned)blocks, 256, 0, st>>>(g, n, qs, shift, hist);
        k_radix_pick<<<1, 256, 0, st>>>(qs, shift, hist);
    }
    k_quant_next<<<(unsigned)blocks, 256, 0, st>>>(g, n, qs);
    k_quant_lerp<<<1, 1, 0, st>>>(qs, k, n, gamma, threshold);
    return last_status();
}

extern "C" int pc_densify_flags(const int64_t* index, int64_t n_balls, int64_t n_keep,
                                int64_t n_out, uint8_t* has_child, uint8_t* halve,
                                uint8_t* child, pc_stream_t stream) {
    if (n_balls < 0 || n_keep < 0 || n_out < n_keep || n_out > 2 * n_balls)
        return PC_ERR_ARGUMENT;
    if (n_out == 0) return PC_OK;
    if (!index || !has_child || !halve || !child) return PC_ERR_ARGUMENT;
    cudaStream_t st = as_stream(stream);
    if (cudaMemsetAsync(has_child, 0, (size_t)n_balls, st) != cudaSuccess) return PC_ERR_CUDA;
    int64_t blocks = (n_out + 255) / 256;
    if (blocks > 8LL * num_sms()) blocks = 8LL * num_sms();
    if (n_out > n_keep)
        k_mark_parents<<<(unsigned)blocks, 256, 0, st>>>(index, n_keep, n_out, has_child);
    k_densify_flags<<<(unsigned)blocks, 256, 0, st>>>(index, n_keep, n_out, has_child, halve,
                                                      child);
    return last_status();
}

extern "C" int pc_densify_masks(const double* p0, const float* g, int64_t n_balls, double p0_min,
                                const double* threshold, uint8_t* keep, uint8_t* split,
                                int64_t* counts, pc_stream_t stream) {
    if (n_balls < 0 || !counts) return PC_ERR_ARGUMENT;
    cudaStream_t st = as_stream(stream);
    if (cudaMemsetAsync(counts, 0, 2 * sizeof(int64_t), st) != cudaSuccess) return PC_ERR_CUDA;
    if (n_balls == 0) return PC_OK;
    if (!p0 || !g || !keep || !split || !threshold) return PC_ERR_ARGUMENT;
    int64_t blocks = (n_balls + 255) / 256;
    if (blocks > 8LL * num_sms()) blocks = 8LL * num_sms();
    k_densify_masks<<<(unsigned)blocks, 256, 0, st>>>(p0, g, n_balls, p0_min, threshold, keep,
                                                      split, nullptr);
    k_count_u8<<<(unsigned)blocks, 256, 0, st>>>(keep, split, n_balls,
                                                 reinterpret_cast<unsigned long long*>(counts));
    return last_status();
}

extern "C" int pc_densify_apply(double* p0, double* mu, const double* a0, const uint8_t* halve,
                                const uint8_t* child, int64_t n_balls, double shift,
                                pc_stream_t stream) {
    if (n_balls < 0) return PC_ERR_ARGUMENT;
    if (n_balls == 0) return PC_OK;
    if (!p0 || !mu || !a0 || !child) return PC_ERR_ARGUMENT;
    int64_t blocks = (n_balls + 255) / 256;
    if (blocks > 8LL * num_sms()) blocks = 8LL * num_sms();
    k_densify_apply<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(p0, mu, a0, halve, child,
                                                                     n_balls, shift);
    return last_status();
}

extern "C" int pc_l2_loss(const double* predicted, const double* observed, int64_t n, double* out,
                          pc_stream_t stream) {
    if (n < 0 || !out || (n > 0 && (!predicted || !observed))) return PC_ERR_ARGUMENT;
    k_l2<<<1, 1024, 0, as_stream(stream)>>>(predicted, observed, n, out);
    return last_status();
}

template <typename GT>
static int check_finite_impl(const GT* x, int32_t n_seg, const int64_t* seg_off, int32_t* flags,
                             pc_stream_t stream) {
    SegTable t;
    if (!seg_table(n_seg, seg_off, t) || !flags) return PC_ERR_ARGUMENT;
    if (t.off[n_seg] > t.off[0] && !x) return PC_ERR_ARGUMENT;
    k_finite<GT><<<dim3(seg_blocks(t), n_seg), 256, 0, as_stream(stream)>>>(x, t, flags);
    return last_status();
}

extern "C" int pc_check_finite(const float* x, int32_t n_seg, const int64_t* seg_off,
                               int32_t* flags, pc_stream_t stream) {
    return check_finite_impl(x, n_seg, seg_off, flags, stream);
}

extern "C" int pc_check_finite_f64(const double* x, int32_t n_seg, const int64_t* seg_off,
                                   int32_t* flags, pc_stream_t stream) {
    return check_finite_impl(x, n_seg, seg_off, flags, stream);
}

template <typename GT>
static int adam_impl(double* params, const GT* grads, double* m, double* v, int32_t n_seg,
                     const int64_t* seg_off, const double* seg_lr, const int32_t* seg_step,
                     const double* seg_floor, pc_stream_t stream) {
    SegTable t;
    if (!seg_table(n_seg, seg_off, t) || !seg_lr || !seg_step) return PC_ERR_ARGUMENT;
    if (t.off[n_seg] > t.off[0] && (!params || !grads || !m || !v)) return PC_ERR_ARGUMENT;
    for (int s = 0; s < n_seg; ++s) {
        if (seg_step[s] < 1) return PC_ERR_ARGUMENT;
        t.lr[s] = seg_lr[s];
        t.bc1[s] = 1.0 - pow(kBeta1, (double)seg_step[s]);
        t.bc2[s] = 1.0 - pow(kBeta2, (double)seg_step[s]);
        t.floor_[s] = seg_floor ? seg_floor[s] : -INFINITY;
    }
    k_adam<GT><<<dim3(seg_blocks(t), n_seg), 256, 0, as_stream(stream)>>>(params, grads, m, v, t);
    return last_status();
}

extern "C" int pc_adam_segments(double* params, const float* grads, double* m, double* v,
                                int32_t n_seg, const int64_t* seg_off, const double* seg_lr,
                                const int32_t* seg_step, const double* seg_floor,
                                pc_stream_t stream) {
    return adam_impl(params, grads, m, v, n_seg, seg_off, seg_lr, seg_step, seg_floor, stream);
}

extern "C" int pc_adam_segments_f64(double* params, const double* grads, double* m, double* v,
                                    int32_t n_seg, const int64_t* seg_off, const double* seg_lr,
                                    const int32_t* seg_step, const double* seg_floor,
                                    pc_stream_t stream) {
    return adam_impl(params, grads, m, v, n_seg, seg_off, seg_lr, seg_step, seg_floor, stream);
}

// Guarded update (no host round trip between the gradient and the step):
// every block reads the non-finite flags, the iteration loss and the
// coincidence word from the device and applies the reference's semantics --
// a coincident pair or a non-finite loss raise before any update
// (radiator.py:186-192, reconstruction.py:317-318), a non-finite gradient
// raises after the groups before it were stepped (reconstruction.py:60-61,
// 320-327) -- so the host only reads the status once the step is done.
struct GuardTable {
    int64_t off[PC_MAX_SEGMENTS + 1];
    double floor_[PC_MAX_SEGMENTS];
    int group[PC_MAX_SEGMENTS];
    int n;
};

__global__ void __launch_bounds__(256) k_update_guarded(double* __restrict__ p,
                                                        const float* __restrict__ g,
                                                        double* __restrict__ m,
                                                        double* __restrict__ v, GuardTable t,
                                                        const double* __restrict__ hyper,
                                                        const int* __restrict__ flags,
                                                        const double* __restrict__ loss,
                                                        const long long* __restrict__ coinc,
                                                        int sgd) {
    const int s = blockIdx.y;
    // the guard decision and the bias corrections once per block (fp64 pow
    // per thread cost 2.5x the whole update)
    __shared__ double sh[3];
    if (threadIdx.x == 0) {
        int bad = t.n;                          // first segment with a non-finite gradient
        for (int k = t.n - 1; k >= 0; --k)
            if (flags[k]) bad = k;
        const bool go = isfinite(*loss) && *coinc == 0x7fffffffffffffffLL && s < bad;
        const double step = hyper[2 * s + 1];
        // floors only when every segment stepped: the reference raises out
        // of ParamGroup.step before _clamp_floors (reconstruction.py:320-328)
        sh[0] = go ? (bad == t.n ? 2.0 : 1.0) : 0.0;
        sh[1] = 1.0 - pow(kBeta1, step);
        sh[2] = 1.0 - pow(kBeta2, step);
    }
    __syncthreads();
    if (sh[0] == 0.0) return;
    const int64_t lo = t.off[s], hi = t.off[s + 1];
    const double lr = hyper[2 * s], fl = sh[0] == 2.0 ? t.floor_[s] : -INFINITY;
    const double bc1 = sh[1], bc2 = sh[2];
    for (int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double gi = (double)g[i];
        double pi;
        if (sgd) {
            pi = p[i] - lr * gi;
        } else {
            double mi = m[i] * kBeta1;
            mi = mi + (1.0 - kBeta1) * gi;
            double vi = v[i] * kBeta2;
            vi = vi + (1.0 - kBeta2) * gi * gi;
            m[i] = mi;
            v[i] = vi;
            pi = p[i] - lr * (mi / bc1) / (sqrt(vi / bc2) + kEps);
        }
        p[i] = pi < fl ? fl : pi;
    }
}

extern "C" int pc_update_guarded(double* params, const float* grads, double* m, double* v,
                                 int32_t n_seg, const int64_t* seg_off, const double* seg_floor,
                                 const int32_t* seg_group, const double* hyper_dev,
                                 const int32_t* flags_dev, const double* loss_dev,
                                 const int64_t* coincident_dev, int32_t optimizer,
                                 pc_stream_t stream) {
    SegTable st;
    if (!seg_table(n_seg, seg_off, st) || !seg_group || !hyper_dev || !flags_dev || !loss_dev ||
        !coincident_dev || (optimizer != 0 && optimizer != 1))
        return PC_ERR_ARGUMENT;
    if (st.off[n_seg] > st.off[0] && (!params || !grads || (optimizer == 0 && (!m || !v))))
        return PC_ERR_ARGUMENT;
    GuardTable t;
    t.n = n_seg;
    for (int k = 0; k <= n_seg; ++k) t.off[k] = seg_off[k];
    for (int k = 0; k < n_seg; ++k) {
        t.floor_[k] = seg_floor ? seg_floor[k] : -INFINITY;
        t.group[k] = seg_group[k];
    }
    k_update_guarded<<<dim3(seg_blocks(st), n_seg), 256, 0, as_stream(stream)>>>(
        params, grads, m, v, t, hyper_dev, flags_dev, loss_dev,
        reinterpret_cast<const long long*>(coincident_dev), optimizer);
    return last_status();
}

template <typename GT>
static int sgd_impl(double* params, const GT* grads, int32_t n_seg, const int64_t* seg_off,
                    const double* seg_lr, const double* seg_floor, pc_stream_t stream) {
    SegTable t;
    if (!seg_table(n_seg, seg_off, t) || !seg_lr) return PC_ERR_ARGUMENT;
    if (t.off[n_seg] > t.off[0] && (!params || !grads)) return PC_ERR_ARGUMENT;
    for (int s = 0; s < n_seg; ++s) {
        t.lr[s] = seg_lr[s];
        t.floor_[s] = seg_floor ? seg_floor[s] : -INFINITY;
        t.bc1[s] = t.bc2[s] = 1.0;
    }
    k_sgd<GT><<<dim3(seg_blocks(t), n_seg), 256, 0, as_stream(stream)>>>(params, grads, t);
    return last_status();
}

extern "C" int pc_sgd_segments(double* params, const float* grads, int32_t n_seg,
                               const int64_t* seg_off, const double* seg_lr,
                               const double* seg_floor, pc_stream_t stream) {
    return sgd_impl(params, grads, n_seg, seg_off, seg_lr, seg_floor, stream);
}

extern "C" int pc_sgd_segments_f64(double* params, const double* grads, int32_t n_seg,
                                   const int64_t* seg_off, const double* seg_lr,
                                   const double* seg_floor, pc_stream_t stream) {
    return sgd_impl(params, grads, n_seg, seg_off, seg_lr, seg_floor, stream);
}

extern "C" size_t pc_compact_workspace_bytes(int64_t n_balls) {
    const int64_t nblk = (n_balls + CMP_BLOCK - 1) / CMP_BLOCK + 1;
    return (size_t)(2 * nblk + 8) * sizeof(int64_t);
}

extern "C" int pc_prune_mask(const double* p0, int64_t n_balls, double rel_threshold,
                             uint8_t* keep, int64_t* n_keep, void* workspace,
                             size_t workspace_bytes, pc_stream_t stream) {
    if (n_balls < 0 || !keep || !n_keep || !workspace || workspace_bytes < 16)
        return PC_ERR_ARGUMENT;
    cudaStream_t st = as_stream(stream);
    if (cudaMemsetAsync(n_keep, 0, sizeof(int64_t), st) != cudaSuccess) return PC_ERR_CUDA;
    if (n_balls == 0) return PC_OK;
    if (!p0) return PC_ERR_ARGUMENT;
    double* maxv = static_cast<double*>(workspace);
    k_max<<<1, 1024, 0, st>>>(p0, n_balls, maxv);
    int64_t blocks = (n_balls + 255) / 256;
    if (blocks > 8LL * num_sms()) blocks = 8LL * num_sms();
    k_prune<<<(unsigned)blocks, 256, 0, st>>>(p0, n_balls, rel_threshold, maxv, keep,
                                              reinterpret_cast<unsigned long long*>(n_keep));
    return last_status();
}

extern "C" int pc_compact_index(const uint8_t* keep, const uint8_t* append, int64_t n_balls,
                                int64_t* index, int64_t* n_out, void* workspace,
                                size_t workspace_bytes, pc_stream_t stream) {
    if (n_balls < 0 || !n_out || !workspace ||
        workspace_bytes < pc_compact_workspace_bytes(n_balls))
        return PC_ERR_ARGUMENT;
    cudaStream_t st = as_stream(stream);
    if (n_balls == 0) {
        return status_of(cudaMemsetAsync(n_out, 0, sizeof(int64_t), st));
    }
    if (!keep || !index) return PC_ERR_ARGUMENT;
    const int64_t nblk = (n_balls + CMP_BLOCK - 1) / CMP_BLOCK;
    int64_t* ck = static_cast<int64_t*>(workspace);
    int64_t* ca = ck + nblk + 1;
    int64_t* tot = ca + nblk + 1;  // [n_out, n_keep]
    k_block_counts<<<(unsigned)nblk, CMP_BLOCK, 0, st>>>(keep, append, n_balls, ck, ca);
    k_scan_counts<<<1, 1024, 0, st>>>(ck, ca, (int)nblk, tot);
    k_scatter_index<<<(unsigned)nblk, CMP_BLOCK, 0, st>>>(keep, append, n_balls, ck, ca, tot,
                                                          index);
    if (cudaMemcpyAsync(n_out, tot, sizeof(int64_t), cudaMemcpyDeviceToDevice, st) !=
        cudaSuccess)
        return PC_ERR_CUDA;
    return last_status();
}

extern "C" int pc_gather_rows(const void* src, void* dst, const int64_t* index, int64_t n_rows,
                              int64_t row_bytes, pc_stream_t stream) {
    if (n_rows < 0 || row_bytes < 0 || (row_bytes & 3)) return PC_ERR_ARGUMENT;
    if (n_rows == 0 || row_bytes == 0) return PC_OK;
    if (!src || !dst || !index) return PC_ERR_ARGUMENT;
    const int64_t words = row_bytes / 4;
    int64_t blocks = (n_rows * words + 255) / 256;
    if (blocks > 16LL * num_sms()) blocks = 16LL * num_sms();
    k_gather<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(
        static_cast<const uint32_t*>(src), static_cast<uint32_t*>(dst), index, n_rows, words);
    return last_status();
}

extern "C" const char* pc_version(void) { return "pacloud_b200 0.1.0 (sm_100a)"; }
