/*
 * ORACLE — test infrastructure only. Never linked into the product path.
 *
 * Plain-C restatement of the reference's only native kernel,
 * hqmq._kernels.nearest_scan (/root/reference/pkg/src/hqmq/_kernels.pyx:16-46):
 *
 *   for each direction u (row of dirs, n x 4, float64, C-contiguous):
 *       best = -2.0; best_j = 0
 *       for j in 0..m-1:
 *           s = ((u0*c[j,0] + u1*c[j,1]) + u2*c[j,2]) + u3*c[j,3]   (fp64, no FMA)
 *           if s > best: best = s; best_j = j                       (strict '>')
 *       idx[i] = best_j; cos[i] = best
 *
 * Must be compiled with -ffp-contract=off (the reference builds with
 * "-O3 -ffp-contract=off", /root/reference/pkg/setup.py:22-24) so the four
 * products and three sums round separately, exactly like numpy's
 * left-to-right evaluation in kernels.py:33-51.
 *
 * The optional `threads` argument splits rows across OpenMP threads; each row
 * is computed by exactly one thread with the same arithmetic, so the result
 * is independent of the thread count.
 */
#include <stdint.h>

void oracle_nearest_scan(const double *dirs, int64_t n, const double *cw,
                         int64_t m, int64_t *idx, double *cos_out,
                         int threads) {
    if (threads < 1) threads = 1;
#pragma omp parallel for num_threads(threads) schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const double u0 = dirs[4 * i + 0], u1 = dirs[4 * i + 1];
        const double u2 = dirs[4 * i + 2], u3 = dirs[4 * i + 3];
        double best = -2.0;
        int64_t best_j = 0;
        for (int64_t j = 0; j < m; ++j) {
            const double *c = cw + 4 * j;
            double s = u0 * c[0];
            s = s + u1 * c[1];
            s = s + u2 * c[2];
            s = s + u3 * c[3];
            if (s > best) {
                best = s;
                best_j = j;
            }
        }
        idx[i] = best_j;
        cos_out[i] = best;
    }
}
