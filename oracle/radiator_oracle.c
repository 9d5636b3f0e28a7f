/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle for the pacloud radiator hot path.
 *
 * Plain-C, float64 restatement of the reference's two numba kernels:
 *   oracle_forward_traces        <- pkg/src/pacloud/radiator.py:86-118  (_forward_traces)
 *   oracle_residual_state_grads  <- pkg/src/pacloud/radiator.py:121-174 (_residual_state_grads)
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
 * reference) may load this library, and only as the checker or the timed CPU
 * baseline.  The product path (paper_2412_03898_b200) never links it.
 *
 * Same loop nest and row ownership as the reference: the forward owns one
 * sensor row per thread and sums balls in index order; the adjoint owns one
 * ball row per thread and sums sensors then samples in order.  Results are
 * therefore deterministic for any OpenMP thread count, like numba's prange.
 * Pinned against the live reference by tests/test_oracle.py (golden vectors in
 * tests/golden/, made by tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define COINCIDENCE_EPS 1e-9 /* radiator.py:33 */

/* radiator.py:100-110: sample window [jlo, jhi) of one (ball, sensor) pair. */
static inline void pair_window(double R, double a0, double v, double t0,
                               double dt, int64_t n_samples, double support,
                               int exact, int64_t *jlo, int64_t *jhi)
{
    if (exact) {
        *jlo = 0;
        *jhi = n_samples;
        return;
    }
    double tlo = (R - support * a0) / v;
    double thi = (R + support * a0) / v;
    int64_t lo = (int64_t)ceil((tlo - t0) / dt);
    int64_t hi = (int64_t)floor((thi - t0) / dt) + 1;
    if (lo < 0) lo = 0;
    if (hi > n_samples) hi = n_samples;
    *jlo = lo;
    *jhi = hi;
}

/* out (M, T) is accumulated into (+=), like the numba kernel. */
void oracle_forward_traces(const double *mu_t, const double *a0_t,
                           const double *p0_t, int64_t n_balls,
                           const double *positions, int64_t n_sensors,
                           double v, double t0, double dt, int64_t n_samples,
                           double support, int exact, double *out,
                           int64_t *flag, int n_threads)
{
#ifdef _OPENMP
    if (n_threads > 0) omp_set_num_threads(n_threads);
#else
    (void)n_threads;
#endif
    int64_t m;
#pragma omp parallel for schedule(dynamic, 1)
    for (m = 0; m < n_sensors; ++m) {
        double *row = out + m * n_samples;
        for (int64_t b = 0; b < n_balls; ++b) {
            double dx = mu_t[3 * b + 0] - positions[3 * m + 0];
            double dy = mu_t[3 * b + 1] - positions[3 * m + 1];
            double dz = mu_t[3 * b + 2] - positions[3 * m + 2];
            double R = sqrt(dx * dx + dy * dy + dz * dz);
            if (R < COINCIDENCE_EPS) {
                flag[0] = 1;
                continue;
            }
            int64_t jlo, jhi;
            pair_window(R, a0_t[b], v, t0, dt, n_samples, support, exact,
                        &jlo, &jhi);
            double inv2a2 = 1.0 / (2.0 * a0_t[b] * a0_t[b]);
            double c = p0_t[b] / (2.0 * R);
            for (int64_t j = jlo; j < jhi; ++j) {
                double t = t0 + j * dt;
                double um = R - v * t;
                double up = R + v * t;
                row[j] += c * (um * exp(-um * um * inv2a2) +
                               up * exp(-up * up * inv2a2));
            }
        }
    }
}

/* G (B, 5) in state order (a0, p0, mu_x, mu_y, mu_z) is accumulated into. */
void oracle_residual_state_grads(const double *mu_t, const double *a0_t,
                                 const double *p0_t, int64_t n_balls,
                                 const double *positions, int64_t n_sensors,
                                 double v, double t0, double dt,
                                 const double *residual, int64_t n_samples,
                                 double support, int exact, double *G,
                                 int64_t *flag, int n_threads)
{
#ifdef _OPENMP
    if (n_threads > 0) omp_set_num_threads(n_threads);
#else
    (void)n_threads;
#endif
    int64_t b;
#pragma omp parallel for schedule(dynamic, 16)
    for (b = 0; b < n_balls; ++b) {
        double a0 = a0_t[b];
        double p0 = p0_t[b];
        double inv_a2 = 1.0 / (a0 * a0);
        for (int64_t m = 0; m < n_sensors; ++m) {
            double dx = mu_t[3 * b + 0] - positions[3 * m + 0];
            double dy = mu_t[3 * b + 1] - positions[3 * m + 1];
            double dz = mu_t[3 * b + 2] - positions[3 * m + 2];
            double R = sqrt(dx * dx + dy * dy + dz * dz);
            if (R < COINCIDENCE_EPS) {
                flag[0] = 1;
                continue;
            }
            int64_t jlo, jhi;
            pair_window(R, a0, v, t0, dt, n_samples, support, exact, &jlo,
                        &jhi);
            double inv2R = 1.0 / (2.0 * R);
            double acc_p = 0.0, acc_a = 0.0, acc_R = 0.0;
            const double *row = residual + m * n_samples;
            for (int64_t j = jlo; j < jhi; ++j) {
                double r = row[j];
                if (r == 0.0) continue;
                double t = t0 + j * dt;
                double um = R - v * t;
                double up = R + v * t;
                double gm = exp(-0.5 * um * um * inv_a2);
                double gp = exp(-0.5 * up * up * inv_a2);
                double s = um * gm + up * gp;
                double k1 = s * inv2R;
                acc_p += r * k1;
                acc_a += r * (um * um * um * gm + up * up * up * gp);
                acc_R += r * (-p0 * k1 / R +
                              p0 * inv2R *
                                  (gm * (1.0 - um * um * inv_a2) +
                                   gp * (1.0 - up * up * inv_a2)));
            }
            G[5 * b + 0] += acc_a * p0 * inv2R * inv_a2 / a0;
            G[5 * b + 1] += acc_p;
            G[5 * b + 2] += acc_R * dx / R;
            G[5 * b + 3] += acc_R * dy / R;
            G[5 * b + 4] += acc_R * dz / R;
        }
    }
}

/* radiator.py:103-110 window sizes: exact in-support sample count sum over
 * pairs, the algorithmic work unit of SURVEY.md section 8(d). */
int64_t oracle_support_samples(const double *mu_t, const double *a0_t,
                               int64_t n_balls, const double *positions,
                               int64_t n_sensors, double v, double t0,
                               double dt, int64_t n_samples, double support,
                               int exact, int n_threads)
{
#ifdef _OPENMP
    if (n_threads > 0) omp_set_num_threads(n_threads);
#else
    (void)n_threads;
#endif
    int64_t total = 0;
    int64_t b;
#pragma omp parallel for reduction(+ : total) schedule(static)
    for (b = 0; b < n_balls; ++b) {
        for (int64_t m = 0; m < n_sensors; ++m) {
            double dx = mu_t[3 * b + 0] - positions[3 * m + 0];
            double dy = mu_t[3 * b + 1] - positions[3 * m + 1];
            double dz = mu_t[3 * b + 2] - positions[3 * m + 2];
            double R = sqrt(dx * dx + dy * dy + dz * dz);
            if (R < COINCIDENCE_EPS) continue;
            int64_t jlo, jhi;
            pair_window(R, a0_t[b], v, t0, dt, n_samples, support, exact,
                        &jlo, &jhi);
            if (jhi > jlo) total += jhi - jlo;
        }
    }
    return total;
}

int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* evaluation.py:46-74 _splat_balls: out (nx,ny,nz) += p0 exp(-d^2/(2 a0^2))
 * over each ball's support cube (|x - mu_x| <= reach per x plane, ceil /
 * floor index ranges along y and z), every voxel when exact.  x planes in
 * parallel, balls in index order per plane, float64 throughout. */
void oracle_voxelize(const double *mu, const double *a0, const double *p0,
                     int64_t n_balls, double ox, double oy, double oz,
                     double sp, int64_t nx, int64_t ny, int64_t nz,
                     double support, int exact, double *out, int n_threads)
{
#ifdef _OPENMP
    if (n_threads > 0) omp_set_num_threads(n_threads);
#else
    (void)n_threads;
#endif
    int64_t ix;
#pragma omp parallel for schedule(static)
    for (ix = 0; ix < nx; ++ix) {
        const double x = ox + ix * sp;
        for (int64_t b = 0; b < n_balls; ++b) {
            const double reach = support * a0[b];
            const double mx = mu[3 * b], my = mu[3 * b + 1], mz = mu[3 * b + 2];
            if (!exact && fabs(x - mx) > reach) continue;
            int64_t ylo = 0, yhi = ny, zlo = 0, zhi = nz;
            if (!exact) {
                ylo = (int64_t)ceil((my - reach - oy) / sp);
                yhi = (int64_t)floor((my + reach - oy) / sp) + 1;
                zlo = (int64_t)ceil((mz - reach - oz) / sp);
                zhi = (int64_t)floor((mz + reach - oz) / sp) + 1;
                if (ylo < 0) ylo = 0;
                if (yhi > ny) yhi = ny;
                if (zlo < 0) zlo = 0;
                if (zhi > nz) zhi = nz;
            }
            const double k = 1.0 / (2.0 * a0[b] * a0[b]);
            const double dx2 = (x - mx) * (x - mx);
            for (int64_t iy = ylo; iy < yhi; ++iy) {
                const double y = oy + iy * sp;
                const double dy2 = (y - my) * (y - my);
                double *row = out + (ix * ny + iy) * nz;
                for (int64_t iz = zlo; iz < zhi; ++iz) {
                    const double z = oz + iz * sp;
                    const double dz2 = (z - mz) * (z - mz);
                    row[iz] += p0[b] * exp(-(dx2 + dy2 + dz2) * k);
                }
            }
        }
    }
}

/* reconstruction.py:352-377 _backproject (filtered traces given): out
 * (nx,ny,nz) = sum_m w * lerp(filtered_m, (|x - s_m| / v - t0) / dt),
 * w = 1/M, j = int(u) clamped to T - 2. */
void oracle_backproject(const double *filtered, const double *positions,
                        int64_t n_sensors, int64_t n_samples, double v,
                        double t0, double dt, double ox, double oy, double oz,
                        double sp, int64_t nx, int64_t ny, int64_t nz,
                        double *out, int n_threads)
{
#ifdef _OPENMP
    if (n_threads > 0) omp_set_num_threads(n_threads);
#else
    (void)n_threads;
#endif
    const double w = 1.0 / (double)n_sensors;
    int64_t ix;
#pragma omp parallel for schedule(static)
    for (ix = 0; ix < nx; ++ix) {
        const double x = ox + ix * sp;
        for (int64_t iy = 0; iy < ny; ++iy) {
            const double y = oy + iy * sp;
            for (int64_t iz = 0; iz < nz; ++iz) {
                const double z = oz + iz * sp;
                double acc = 0.0;
                for (int64_t m = 0; m < n_sensors; ++m) {
                    const double dx = x - positions[3 * m];
                    const double dy = y - positions[3 * m + 1];
                    const double dz = z - positions[3 * m + 2];
                    const double tof = sqrt(dx * dx + dy * dy + dz * dz) / v;
                    const double u = (tof - t0) / dt;
                    int64_t j = (int64_t)u;
                    if (j >= n_samples - 1) j = n_samples - 2;
                    const double fr = u - (double)j;
                    const double *f = filtered + m * n_samples;
                    acc += w * ((1.0 - fr) * f[j] + fr * f[j + 1]);
                }
                out[(ix * ny + iy) * nz + iz] = acc;
            }
        }
    }
}
