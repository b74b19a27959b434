// hk_collision.cu — batched fast-spectral Boltzmann collision operator, sm_100a.
//
// Replaces spectral_collision (src/spectral.cpp:114-154) + FftWorkspace3d
// (src/fft.cpp:49-81) for a whole batch of cells.  One thread-block CLUSTER
// of C CTAs evaluates one cell at a time (persistent over the batch); the
// cell's spectrum F never leaves shared memory:
//
//   prologue  f (HBM) -> forward 3-D FFT split over the cluster -> F slab in SMEM
//             CTA r owns modes i1 in [rP, rP+P), P = N/C  ("slab")
//   round     phase A: per owned (i1,i2) pencil: X = F * weights (L2-resident
//                      tables, coalesced), inverse FFT over i3 in registers,
//                      scatter to the owner of j3 through DSMEM
//             phase B: per owned j3 plane (i1,i2): inverse FFT over i2, then
//                      over i1 (in place in SMEM), product + accumulate the
//                      gain in registers
//   epilogue  Q = jac (w gain - f loss)  -> HBM, per-cell verdict
//
// Two arithmetic modes:
//   EXACT (reference semantics): per direction two complex fields
//        ga = IFFT(alpha F), gb = IFFT(alpha' F);  gain += ga gb (complex).
//   FAST: since f is real, F is Hermitian; with the Hermitian-symmetrised
//        weights alpha_s the field IFFT(F (alpha_s + i alpha'_s)) = gs + i hs
//        carries BOTH real transforms, so one complex transform per direction
//        gives Re(ga gb) up to the Nyquist-plane term -Im ga Im gb, which a
//        per-cell rigorous bound (guard_kernel) checks; cells failing it are
//        recomputed on the EXACT path.  Two directions per round.
// Phase factors of src/fft.cpp:19-28 cancel between to_spectral and
// to_nodal (|phase| = 1) and are not applied.
#include <cstdio>

#include "hk_common.cuh"
#include "hk_internal.h"

namespace hk {

struct CollArgs {
    const double* f;
    double* q;
    int64_t ncells;
    const int64_t* list;    // optional cell list (rerouted cells)
    const int* list_count;  // device count for `list`
    const double* alpha;
    const double* alpha_p;
    const double* loss;
    const double2* wfast;
    int md;
    double mult0, jac, w;
    hk_cell_status* st;
    double* nyq;  // [cell][3][N][N] |F| on the Nyquist planes (FAST) or null
};

template <int N, int C>
struct Geo {
    static constexpr int P = N / C;
    static constexpr int ROW = N + 1;  // padded row: conflict-free column and row access
    static constexpr int PLANE = N * ROW;
    static constexpr int SLAB = P * PLANE;  // double2 per F slab / per received field
    static constexpr int NT = 256;
    static_assert(P * N == 128, "one pencil per thread per field");
    static constexpr size_t SMEM = size_t(3 * SLAB) * sizeof(double2) + 8 * 3 * sizeof(double);
};

template <int N, int C, bool EXACT>
__global__ void __launch_bounds__(256, 1) coll_kernel(CollArgs a) {
    using G = Geo<N, C>;
    constexpr int P = G::P, ROW = G::ROW, PLANE = G::PLANE, SLAB = G::SLAB;
    constexpr int64_t NB = (int64_t)N * N * N;
    extern __shared__ __align__(16) double2 smem[];
    double2* Fs = smem;
    double2* Rv0 = smem + SLAB;
    double2* Rv1 = smem + 2 * SLAB;
    double* red = reinterpret_cast<double*>(smem + 3 * SLAB);

    const unsigned r = cluster_rank();
    const unsigned cid = cluster_id_x();
    const unsigned ncl = n_clusters_x();
    const int t = threadIdx.x;
    const int phi = t >> 7;
    const int pp = t & 127;
    const int64_t count = a.list_count ? (int64_t)*a.list_count : a.ncells;

    double2* RvMine = phi ? Rv1 : Rv0;

    const int n_entries = a.md + 1;  // distinct directions + loss
    const int rounds = EXACT ? n_entries : (n_entries + 1) / 2;
    const int loss_phi = EXACT ? 0 : ((n_entries - 1) & 1);

    for (int64_t it = cid; it < count; it += ncl) {
        const int64_t cell = a.list ? a.list[it] : it;
        const double* fc = a.f + cell * NB;

        // ---------------- prologue: F = FFT(f) / N^3 ----------------
        for (int idx = t; idx < N * N * P; idx += 256) {  // f(j1, j2, j3 in my block)
            const int j3l = idx % P, j2 = (idx / P) % N, j1 = idx / (P * N);
            Rv0[j3l * PLANE + j1 * ROW + j2] = make_double2(fc[(j1 * N + j2) * N + r * P + j3l], 0.0);
        }
        __syncthreads();
        if (t < 128) {  // forward over j2 (rows)
            const int j3l = pp / N, j1 = pp % N;
            double2* row = Rv0 + j3l * PLANE + j1 * ROW;
            double2 x[N];
#pragma unroll
            for (int i = 0; i < N; ++i) x[i] = row[i];
            fft_reg<N, false>(x);
#pragma unroll
            for (int i = 0; i < N; ++i) row[i] = x[i];
        }
        __syncthreads();
        if (t < 128) {  // forward over j1 (columns) -> owner of k1
            const int j3l = pp / N, k2 = pp % N;
            const double2* col = Rv0 + j3l * PLANE + k2;
            double2 x[N];
#pragma unroll
            for (int i = 0; i < N; ++i) x[i] = col[i * ROW];
            fft_reg<N, false>(x);
            const int j3 = r * P + j3l;
#pragma unroll
            for (int dst = 0; dst < C; ++dst) {
                double2* rb = dsmem_ptr(Fs + k2 * ROW + j3, dst);
#pragma unroll
                for (int kl = 0; kl < P; ++kl) rb[kl * PLANE] = x[dst * P + kl];
            }
        }
        cluster_arrive();
        cluster_wait();
        if (t < 128) {  // forward over k3 (rows of the slab), scale 1/N^3
            const int pl = pp / N, k2 = pp % N;
            double2* row = Fs + pl * PLANE + k2 * ROW;
            double2 x[N];
#pragma unroll
            for (int i = 0; i < N; ++i) x[i] = row[i];
            fft_reg<N, false>(x);
            const double s = 1.0 / double(NB);
#pragma unroll
            for (int i = 0; i < N; ++i) row[i] = make_double2(x[i].x * s, x[i].y * s);
        }
        __syncthreads();
        if (!EXACT && a.nyq) {  // |F| on the three Nyquist planes for the guard
            double* ny = a.nyq + cell * 3 * N * N;
            constexpr int H = N / 2;
            for (int idx = t; idx < P * N; idx += 256) {
                const int pl = idx / N, c = idx % N;
                const int k1 = r * P + pl;
                const double2 v1 = Fs[pl * PLANE + H * ROW + c];  // (k1, H, k3=c)
                ny[1 * N * N + k1 * N + c] = sqrt(v1.x * v1.x + v1.y * v1.y);
                const double2 v2 = Fs[pl * PLANE + c * ROW + H];  // (k1, k2=c, H)
                ny[2 * N * N + k1 * N + c] = sqrt(v2.x * v2.x + v2.y * v2.y);
            }
            if (H / P == (int)r) {
                const int pl = H % P;
                for (int idx = t; idx < N * N; idx += 256) {
                    const double2 v = Fs[pl * PLANE + (idx / N) * ROW + (idx % N)];
                    ny[idx] = sqrt(v.x * v.x + v.y * v.y);
                }
            }
        }
        cluster_arrive();  // token: my Rv is free for round 0

        // ---------------- rounds over directions ----------------
        double gacc[N];
#pragma unroll
        for (int i = 0; i < N; ++i) gacc[i] = 0.0;

        for (int rd = 0; rd < rounds; ++rd) {
            const int e = EXACT ? rd : 2 * rd + phi;
            const bool valid = EXACT ? (rd < a.md || phi == 0) : (e < n_entries);
            const bool is_loss = (e == a.md);
            // ---- phase A: X = F * weights, inverse FFT over i3 ----
            const int pl = pp / N, i2 = pp % N, i1 = r * P + pl;
            double2 x[N];
            if (valid) {
                const double2* frow = Fs + pl * PLANE + i2 * ROW;
                if (EXACT) {
                    const double* wt = (is_loss ? a.loss : (phi ? a.alpha_p : a.alpha) + (int64_t)e * NB) +
                                       (int64_t)i1 * N * N + i2;
#pragma unroll
                    for (int i3 = 0; i3 < N; ++i3) {
                        const double wv = __ldg(wt + i3 * N);
                        const double2 F = frow[i3];
                        x[i3] = make_double2(F.x * wv, F.y * wv);
                    }
                } else {
                    const double2* wt = a.wfast + (int64_t)e * NB + (int64_t)i1 * N * N + i2;
#pragma unroll
                    for (int i3 = 0; i3 < N; ++i3) {
                        const double2 wv = __ldg(wt + i3 * N);
                        const double2 F = frow[i3];
                        x[i3] = make_double2(F.x * wv.x - F.y * wv.y, F.x * wv.y + F.y * wv.x);
                    }
                }
                fft_reg<N, true>(x);
            }
            cluster_wait();  // every rank has finished reading its Rv (previous round)
            if (valid) {
#pragma unroll
                for (int dst = 0; dst < C; ++dst) {
                    double2* rb = dsmem_ptr(RvMine + i1 * ROW + i2, dst);
#pragma unroll
                    for (int jl = 0; jl < P; ++jl) rb[jl * PLANE] = x[dst * P + jl];
                }
            }
            cluster_arrive();
            cluster_wait();  // my Rv now holds (all i1, all i2, my j3) of both fields

            // ---- phase B: inverse FFT over i2 (rows), then i1 (columns) ----
            const int j3l = pp / N;
            if (valid) {
                double2* row = RvMine + j3l * PLANE + (pp % N) * ROW;
                double2 y[N];
#pragma unroll
                for (int i = 0; i < N; ++i) y[i] = row[i];
                fft_reg<N, true>(y);
#pragma unroll
                for (int i = 0; i < N; ++i) row[i] = y[i];
            }
            __syncthreads();
            const int j2 = pp % N;
            if (valid) {
                double2* col = RvMine + j3l * PLANE + j2;
                double2 y[N];
#pragma unroll
                for (int i = 0; i < N; ++i) y[i] = col[i * ROW];
                fft_reg<N, true>(y);
                if (!EXACT && !is_loss) {
                    const double m = (e == 0) ? a.mult0 : 1.0;
#pragma unroll
                    for (int j1 = 0; j1 < N; ++j1) gacc[j1] += m * (y[j1].x * y[j1].y);
                } else {
#pragma unroll
                    for (int i = 0; i < N; ++i) col[i * ROW] = y[i];
                }
            }
            if (EXACT) {
                __syncthreads();
                if (rd < a.md) {  // gain += m * ga * gb on half the column per thread
                    const double m = (rd == 0) ? a.mult0 : 1.0;
#pragma unroll
                    for (int h = 0; h < N / 2; ++h) {
                        const int j1 = phi * (N / 2) + h;
                        const double2 ga = Rv0[j3l * PLANE + j1 * ROW + j2];
                        const double2 gb = Rv1[j3l * PLANE + j1 * ROW + j2];
                        gacc[2 * h] += m * (ga.x * gb.x - ga.y * gb.y);
                        gacc[2 * h + 1] += m * (ga.x * gb.y + ga.y * gb.x);
                    }
                }
            }
            if (rd + 1 < rounds) cluster_arrive();  // my Rv may be overwritten
        }

        // ---------------- epilogue: Q = jac (w gain - f loss) ----------------
        double2* Lbuf = loss_phi ? Rv1 : Rv0;
        double2* Free = loss_phi ? Rv0 : Rv1;
        {
            const int j3l = pp / N, j2 = pp % N;
            if (!EXACT) {
                double* Gd = reinterpret_cast<double*>(Free);
#pragma unroll
                for (int j1 = 0; j1 < N; ++j1) Gd[phi * N * N * P + (j1 * N + j2) * P + j3l] = gacc[j1];
            } else {
#pragma unroll
                for (int h = 0; h < N / 2; ++h) {
                    const int j1 = phi * (N / 2) + h;
                    Free[(j1 * N + j2) * P + j3l] = make_double2(gacc[2 * h], gacc[2 * h + 1]);
                }
            }
        }
        __syncthreads();
        double mre = 0.0, mim = 0.0, n2 = 0.0;
        double* qc = a.q + cell * NB;
        for (int idx = t; idx < N * N * P; idx += 256) {
            const int j3l = idx % P, j2 = (idx / P) % N, j1 = idx / (P * N);
            double gre, gim;
            if (!EXACT) {
                const double* Gd = reinterpret_cast<const double*>(Free);
                gre = Gd[idx] + Gd[N * N * P + idx];
                gim = 0.0;
            } else {
                const double2 g = Free[idx];
                gre = g.x;
                gim = g.y;
            }
            const double2 L = Lbuf[j3l * PLANE + j1 * ROW + j2];
            const int64_t gi = ((int64_t)j1 * N + j2) * N + r * P + j3l;
            const double fv = fc[gi];
            const double qre = a.jac * (a.w * gre - fv * L.x);
            qc[gi] = qre;
            mre = fmax(mre, fabs(qre));
            n2 += qre * qre;
            if (EXACT) mim = fmax(mim, fabs(a.jac * (a.w * gim - fv * L.y)));
        }
        // block reduction -> global atomics into the cell's verdict
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mre = fmax(mre, __shfl_xor_sync(0xffffffffu, mre, o));
            mim = fmax(mim, __shfl_xor_sync(0xffffffffu, mim, o));
            n2 += __shfl_xor_sync(0xffffffffu, n2, o);
        }
        const int warp = t >> 5, lane = t & 31;
        if (lane == 0) {
            red[warp] = mre;
            red[8 + warp] = mim;
            red[16 + warp] = n2;
        }
        __syncthreads();
        if (t == 0 && a.st) {
            double m1 = 0, m2 = 0, s = 0;
            for (int w = 0; w < 8; ++w) {
                m1 = fmax(m1, red[w]);
                m2 = fmax(m2, red[8 + w]);
                s += red[16 + w];
            }
            hk_cell_status* sc = a.st + cell;
            atomic_max_nonneg(&sc->max_re, m1);
            atomic_max_nonneg(&sc->max_im, m2);
            atomicAdd(&sc->q_norm2, s);
            if (EXACT && r == 0) atomicOr(&sc->flags, HK_CELL_EXACT);
        }
        cluster_arrive();
        cluster_wait();  // end of cell: Fs / Rv of every rank reusable
    }
}

// Rigorous bound of the dropped Nyquist term of the FAST path, per cell:
//   |Im ga_d(j)| <= A_d = sum_{k in S} |alpha_a,d(k)| |F(k)|,  likewise B_d,
//   ||dQ||_2 <= jac w sum_d m_d A_d B_d N^{3/2}.
// Cells with bound / ||Q||_2 > tau are appended to the reroute list.
__global__ void guard_kernel(int n, int md, double mult0, double jac, double w, double tau,
                             const double* __restrict__ nyq, const double* __restrict__ abs_a,
                             const double* __restrict__ abs_ap, int64_t ncells,
                             hk_cell_status* __restrict__ st, int64_t* __restrict__ list,
                             int* __restrict__ count) {
    const int64_t cell = blockIdx.x;
    if (cell >= ncells) return;
    const int nn3 = 3 * n * n;
    const double* F = nyq + cell * nn3;
    __shared__ double sA[8], sB[8];
    double bound = 0.0;
    for (int e = 0; e < md; ++e) {
        const double* pa = abs_a + (int64_t)e * nn3;
        const double* pb = abs_ap + (int64_t)e * nn3;
        double A = 0.0, B = 0.0;
        for (int i = threadIdx.x; i < nn3; i += blockDim.x) {
            const double fv = F[i];
            A += __ldg(pa + i) * fv;
            B += __ldg(pb + i) * fv;
        }
        for (int o = 16; o > 0; o >>= 1) {
            A += __shfl_xor_sync(0xffffffffu, A, o);
            B += __shfl_xor_sync(0xffffffffu, B, o);
        }
        if ((threadIdx.x & 31) == 0) {
            sA[threadIdx.x >> 5] = A;
            sB[threadIdx.x >> 5] = B;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double At = 0, Bt = 0;
            for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
                At += sA[k];
                Bt += sB[k];
            }
            bound += (e == 0 ? mult0 : 1.0) * At * Bt;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        hk_cell_status* sc = st + cell;
        const double qn = sqrt(sc->q_norm2);
        const double abs_bound = jac * w * bound * pow(double(n), 1.5);
        const double rel = qn > 0.0 ? abs_bound / qn : (abs_bound > 0.0 ? INFINITY : 0.0);
        sc->nyq_bound = rel;
        if (!(rel <= tau)) {
            const int slot = atomicAdd(count, 1);
            list[slot] = cell;
            sc->max_re = 0.0;
            sc->max_im = 0.0;
            sc->q_norm2 = 0.0;
            sc->flags |= HK_CELL_GUARD_REROUTED;
        }
    }
}

__global__ void residue_kernel(int64_t ncells, hk_cell_status* st) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncells) return;
    hk_cell_status* s = st + c;
    if ((s->flags & HK_CELL_EXACT) && s->max_im > 1e-10 * fmax(s->max_re, 1e-300))
        s->flags |= HK_CELL_RESIDUE;
}

namespace {

template <int N, int C, bool EXACT>
int launch_variant(hk_ctx ctx, const CollArgs& args, int64_t max_cells) {
    using G = Geo<N, C>;
    auto kern = coll_kernel<N, C, EXACT>;
    const int key = N * 100 + C * 2 + (EXACT ? 1 : 0);
    int st;
    if (!ctx->max_clusters.count(key)) {
        if ((st = check_cuda(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM),
                             "smem attribute")))
            return st;
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = C;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(C * 256);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = G::SMEM;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int ncl = 0;
        if ((st = check_cuda(ctx, cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg), "max active clusters")))
            return st;
        if (ncl < 1) return fail(ctx, HK_CUDA, "collision kernel cannot be resident (cluster occupancy 0)");
        ctx->max_clusters[key] = ncl;
    }
    int64_t ncl = ctx->max_clusters[key];
    if (max_cells < ncl) ncl = max_cells;
    if (ncl < 1) return HK_OK;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(unsigned(ncl * C));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = G::SMEM;
    cfg.stream = ctx->stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    st = check_cuda(ctx, cudaLaunchKernelEx(&cfg, kern, args), "collision kernel launch");
    ctx->launches++;
    return st;
}

template <int N, int C>
int run_size(hk_ctx ctx, hk_kernel k, const double* f, double* q, int64_t ncells, uint32_t flags,
             hk_cell_status* st) {
    const bool exact = (flags & (HK_COLL_EXACT | HK_COLL_STRICT)) != 0;
    const bool guard = !exact && !(flags & HK_COLL_NOGUARD);
    const int64_t nn3 = 3LL * N * N;
    // scratch: [nyq |F| planes][reroute list][count]
    const size_t st_bytes = st ? 0 : sizeof(hk_cell_status) * ncells;
    const size_t nyq_bytes = guard ? sizeof(double) * nn3 * ncells : 0;
    const size_t list_bytes = guard ? sizeof(int64_t) * ncells : 0;
    int s;
    if ((s = ensure_scratch(ctx, st_bytes + nyq_bytes + list_bytes + 64))) return s;
    char* base = static_cast<char*>(ctx->scratch);
    if (!st) st = reinterpret_cast<hk_cell_status*>(base);
    double* nyq = guard ? reinterpret_cast<double*>(base + st_bytes) : nullptr;
    int64_t* list = guard ? reinterpret_cast<int64_t*>(base + st_bytes + nyq_bytes) : nullptr;
    int* count = reinterpret_cast<int*>(base + st_bytes + nyq_bytes + list_bytes);
    cudaMemsetAsync(st, 0, sizeof(hk_cell_status) * ncells, ctx->stream);

    CollArgs a{};
    a.f = f;
    a.q = q;
    a.ncells = ncells;
    a.alpha = k->alpha;
    a.alpha_p = k->alpha_p;
    a.loss = k->loss;
    a.wfast = k->wfast;
    a.md = k->md;
    a.mult0 = k->mult0;
    a.jac = k->jac;
    a.w = k->weight;
    a.st = st;
    if (exact) {
        if ((s = launch_variant<N, C, true>(ctx, a, ncells))) return s;
    } else {
        a.nyq = nyq;
        if ((s = launch_variant<N, C, false>(ctx, a, ncells))) return s;
        if (guard) {
            cudaMemsetAsync(count, 0, sizeof(int), ctx->stream);
            guard_kernel<<<unsigned(ncells), 256, 0, ctx->stream>>>(N, k->md, k->mult0, k->jac, k->weight, 1e-11, nyq,
                                                                  k->abs_a, k->abs_ap, ncells, st, list, count);
            ctx->launches++;
            if ((s = check_cuda(ctx, cudaGetLastError(), "guard kernel"))) return s;
            CollArgs b = a;
            b.nyq = nullptr;
            b.list = list;
            b.list_count = count;
            if ((s = launch_variant<N, C, true>(ctx, b, ncells))) return s;
        }
    }
    {
        residue_kernel<<<unsigned((ncells + 255) / 256), 256, 0, ctx->stream>>>(ncells, st);
        ctx->launches++;
        if ((s = check_cuda(ctx, cudaGetLastError(), "residue kernel"))) return s;
    }
    return HK_OK;
}

}  // namespace

int collision_launch(hk_ctx ctx, hk_kernel k, const double* f, double* q, int64_t ncells,
                     uint32_t flags, hk_cell_status* st) {
    if (ncells <= 0) return HK_OK;
    switch (k->n) {
    case 16:
        return run_size<16, 2>(ctx, k, f, q, ncells, flags, st);
    case 32:
        return run_size<32, 8>(ctx, k, f, q, ncells, flags, st);
    default:
        return fail(ctx, HK_UNSUPPORTED, "collision path implemented for n = 16, 32");
    }
}

}  // namespace hk
