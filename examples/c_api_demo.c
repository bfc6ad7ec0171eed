/* c_api_demo.c -- the library used from plain C through include/wd.h (no
 * Python, no torch): builds a terrain-following mesh on the host, runs one
 * time step (assemble, RHS, solve to 1e-8, wind recovery) with HOST arrays
 * (the library stages them through device memory) and prints the solver
 * report and the mass-consistency diagnostics.
 *
 *   gcc -O2 -std=c11 examples/c_api_demo.c -Iinclude -Lpaper_2101_08453_b200 -lwd \
 *       -Wl,-rpath,$PWD/paper_2101_08453_b200 -lm -o c_api_demo && ./c_api_demo [nx ny nz]
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "wd.h"

#define CHECK(call)                                                                \
    do {                                                                           \
        int rc_ = (call);                                                          \
        if (rc_ != WD_OK && rc_ != WD_E_NOCONV) {                                  \
            fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, wd_last_error()); \
            return 1;                                                              \
        }                                                                          \
    } while (0)

int main(int argc, char** argv) {
    const int nx = argc > 1 ? atoi(argv[1]) : 48, ny = argc > 2 ? atoi(argv[2]) : 40,
              nz = argc > 3 ? atoi(argv[3]) : 8;
    const int n1 = nx + 1, n2 = ny + 1, n3 = nz + 1;
    const double dx = 30.0;
    const size_t N = (size_t)n1 * n2 * n3, E = (size_t)3 * nx * ny * nz;
    double* zs = malloc(sizeof(double) * n1 * n2);
    double* zeta = malloc(sizeof(double) * n3);
    double *X = malloc(sizeof(double) * N), *Y = malloc(sizeof(double) * N),
           *Z = malloc(sizeof(double) * N);
    double *u0 = malloc(sizeof(double) * E), *u = malloc(sizeof(double) * E);
    double* lam = calloc(N, sizeof(double));
    if (!zs || !zeta || !X || !Y || !Z || !u0 || !u || !lam) return 1;

    /* one Gaussian hill, levels stretched by 1.2 from 5 m, flat top (reading C13) */
    double zmax = 0.0;
    for (int j = 0; j < n2; j++)
        for (int i = 0; i < n1; i++) {
            const double x = i * dx - 0.5 * nx * dx, y = j * dx - 0.5 * ny * dx;
            zs[j * n1 + i] = 120.0 * exp(-(x * x + y * y) / (2.0 * 200.0 * 200.0));
            if (zs[j * n1 + i] > zmax) zmax = zs[j * n1 + i];
        }
    zeta[0] = 0.0;
    for (int k = 1; k < n3; k++) zeta[k] = zeta[k - 1] + 5.0 * pow(1.2, k - 1);
    CHECK(wd_build_mesh(zs, n1, n2, 0.0, 0.0, dx, dx, zeta, n3, zmax + zeta[n3 - 1], X, Y, Z,
                        NULL));

    /* uniform 5 m/s westerly at every element centre */
    for (size_t e = 0; e < E; e++) u0[e] = e < E / 3 ? 5.0 : 0.0;

    wd_options opt;
    wd_default_options(&opt);
    wd_ctx* ctx = NULL;
    CHECK(wd_assemble(X, Y, Z, n1, n2, n3, 1.0, 1.0, 1.0, &opt, NULL, &ctx));
    wd_report rep;
    CHECK(wd_downscale_step(ctx, u0, lam, 0, 1e-8, u, &rep, NULL));
    double d0[2], d1[2];
    CHECK(wd_mass_consistency(ctx, u0, d0, NULL));
    CHECK(wd_mass_consistency(ctx, u, d1, NULL));

    /* vertical wind at the lowest layer, windward and lee of the hill centre */
    const size_t plane = (size_t)nx * ny, wofs = 2 * (E / 3);
    const int jc = ny / 2, iw = nx / 2 - 4, il = nx / 2 + 3;
    printf("levels %d, cycles %d, rate %.3f, rel residual %.2e\n", rep.nlevels, rep.cycles,
           rep.rate, rep.rel_res_final);
    printf("|D1 u0| = %.4e  |D1 u| = %.4e\n", d0[0], d1[0]);
    printf("w windward %.4f  w lee %.4f\n", u[wofs + (size_t)jc * nx + iw],
           u[wofs + (size_t)jc * nx + il]);
    (void)plane;
    wd_destroy(ctx);
    free(zs); free(zeta); free(X); free(Y); free(Z); free(u0); free(u); free(lam);
    return rep.converged ? 0 : 2;
}
