/* Plain-C caller of the multi-GPU part of the C-ABI (one rank): the sequence
 * a reference-side driver runs per PR(2,2,2) stage on its x-slab —
 * communicator init, halo exchange, slab transport, scalar all-reduce. */
#include <cuda_runtime_api.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "hykin_b200.h"

#define CHECK(x)                                                      \
    do {                                                              \
        int st_ = (x);                                                \
        if (st_) {                                                    \
            fprintf(stderr, "%s failed with status %d\n", #x, st_);  \
            return 10 + st_;                                          \
        }                                                             \
    } while (0)

int main(void) {
    const int n = 8, nx = 4, ny = 3;
    const size_t nb = (size_t)n * n * n, cells = (size_t)nx * ny;
    hk_ctx ctx;
    CHECK(hk_ctx_create(0, &ctx));
    char id[HK_COMM_ID_BYTES];
    CHECK(hk_comm_unique_id(id));  /* rank 0; MPI_Bcast to the other ranks */
    CHECK(hk_ctx_comm_init(ctx, 1, 0, id));
    double* fh = malloc(sizeof(double) * cells * nb);
    for (size_t c = 0; c < cells; ++c)
        for (size_t k = 0; k < nb; ++k) fh[c * nb + k] = 0.5 + 0.4 * sin(0.7 * c + 0.013 * k);
    double *f, *left, *right, *out, *red;
    cudaMalloc((void**)&f, sizeof(double) * cells * nb);
    cudaMalloc((void**)&left, sizeof(double) * ny * 2 * nb);
    cudaMalloc((void**)&right, sizeof(double) * ny * 2 * nb);
    cudaMalloc((void**)&out, sizeof(double) * cells * nb);
    cudaMalloc((void**)&red, sizeof(double) * 3);
    cudaMemcpy(f, fh, sizeof(double) * cells * nb, cudaMemcpyHostToDevice);
    CHECK(hk_halo_exchange(ctx, n, f, nx, ny, left, right));
    CHECK(hk_transport_rhs_slab(ctx, n, 8.0, f, left, right, out, nx, ny, 1.0 / nx, 1.0 / ny, 1e-6));
    const double sums[3] = {1.0, -2.0, 3.5};
    cudaMemcpy(red, sums, sizeof sums, cudaMemcpyHostToDevice);
    CHECK(hk_allreduce_scalars(ctx, red, 3, HK_REDUCE_SUM));
    cudaDeviceSynchronize();
    double* lh = malloc(sizeof(double) * ny * 2 * nb);
    double* rh = malloc(sizeof(double) * ny * 2 * nb);
    double back[3];
    cudaMemcpy(lh, left, sizeof(double) * ny * 2 * nb, cudaMemcpyDeviceToHost);
    cudaMemcpy(rh, right, sizeof(double) * ny * 2 * nb, cudaMemcpyDeviceToHost);
    cudaMemcpy(back, red, sizeof back, cudaMemcpyDeviceToHost);
    double err = 0.0;
    for (int j = 0; j < ny; ++j)
        for (int h = 0; h < 2; ++h)
            for (size_t k = 0; k < nb; ++k) {
                /* one rank: periodic self-wrap */
                err = fmax(err, fabs(lh[(j * 2 + h) * nb + k] - fh[((size_t)j * nx + nx - 2 + h) * nb + k]));
                err = fmax(err, fabs(rh[(j * 2 + h) * nb + k] - fh[((size_t)j * nx + h) * nb + k]));
            }
    for (int i = 0; i < 3; ++i) err = fmax(err, fabs(back[i] - sums[i]));
    printf("{\"halo_and_allreduce_max_err\": %.3e}\n", err);
    hk_ctx_destroy(ctx);
    return err == 0.0 ? 0 : 1;
}
