/* Oracle helper kernels (TEST INFRASTRUCTURE ONLY -- never linked into the
 * product library, never on the measured path).
 *
 * hsw_ddot: restatement of the OpenBLAS 0.3.30 Haswell ddot kernel that numpy
 * reaches through np.linalg.norm / np.dot in the reference's power method
 * (reference nodal_amg.py:106-111, estimate_rho).  Sixteen independent FMA
 * chains over blocks of 16 elements (4 ymm accumulators x 4 lanes), a fixed
 * combine tree, then a non-fused scalar tail.  Verified bitwise against
 * numpy under OPENBLAS_CORETYPE=Haswell OPENBLAS_NUM_THREADS=1
 * (tests/test_oracle.py::test_hsw_ddot_matches_pinned_numpy).
 *
 * Build: oracle/Makefile  ->  oracle/_build/liboracle.so  (-ffp-contract=off)
 */
#include <math.h>

double oracle_hsw_ddot(long n, const double *x, const double *y)
{
    double acc[4][4] = {{0.0}};
    long n1 = n & -16L;
    for (long i = 0; i < n1; i += 16)
        for (int a = 0; a < 4; a++)
            for (int l = 0; l < 4; l++)
                acc[a][l] = fma(x[i + 4 * a + l], y[i + 4 * a + l], acc[a][l]);
    double dot = 0.0;
    if (n1) {
        double h[4][2];
        for (int a = 0; a < 4; a++) {
            h[a][0] = acc[a][0] + acc[a][2];
            h[a][1] = acc[a][1] + acc[a][3];
        }
        double u0 = (h[0][0] + h[1][0]) + (h[2][0] + h[3][0]);
        double u1 = (h[0][1] + h[1][1]) + (h[2][1] + h[3][1]);
        dot = u0 + u1;
    }
    for (long i = n1; i < n; i++) {
        double p = y[i] * x[i];
        dot = dot + p;
    }
    return dot;
}
