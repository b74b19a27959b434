// hk_nyqfix.cu — exact Nyquist correction of fast-path cells.
//
// The FAST collision kernels return Q_fast = jac (w sum_d m_d gs_d hs_d - f L)
// with gs + i hs = IFFT(F (alpha_s + i alpha'_s)).  The exact operator of
// spectral_collision (src/spectral.cpp:114-154) has Re(ga gb) = gs hs - ga_i hb_i,
// where ga_i = IFFT(alpha_a F) / i and hb_i = IFFT(alpha'_a F) / i come from the
// antisymmetric parts of the weights, which live on the three Nyquist sets only
// (S1: k1 = H;  S2: k2 = H, k1 != H;  S3: k3 = H, k1, k2 != H;  H = N/2).  A
// Nyquist set is a plane, so its 3-D inverse transform is a 2-D transform times
// a sign along the normal axis:
//     ga_i(j) = (-1)^j1 A1(j2, j3) + (-1)^j2 A2(j1, j3) + (-1)^j3 A3(j1, j2),
// with one complex 2-D transform per plane giving both A and B (hb_i) because
// each restricted input is anti-Hermitian:  IFFT2(Y_a + i Y_b) = -B + i A.
// Two kernels add  -jac w sum_d m_d ga_i,d hb_i,d  to Q for the cells on the
// guard's list, turning their fast result into the exact one (real part) at a
// few per cent of the cost of re-running the exact collision kernel:
//   nyq_planes_kernel: per (cell, direction) the three packed 2-D transforms
//                      (SMEM, in place) -> scratch [cell][d][3][N][N];
//   nyq_apply_kernel:  per (cell, slab of T j1-planes) the correction of every
//                      node accumulated over all directions in registers, then
//                      one read-modify-write of Q.
// The list is processed in chunks sized to bound the scratch (~2 GiB).
#include <type_traits>
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "hk_coll.cuh"
#include "hk_common.cuh"

namespace hk {

template <int N>
struct GeoFix {
    static constexpr int ROW = N + 1;
    static constexpr int PLANE = N * ROW;                          // double2, padded plane
    static constexpr int NN = N * N;
    static constexpr size_t SMEM1 = size_t(3) * (N <= 16 ? 4 : (N <= 32 ? 2 : 1)) * PLANE * sizeof(double2);
#ifndef HK_NYQ_APPLY_NT
#define HK_NYQ_APPLY_NT 256  // apply threads per CTA
#endif
#ifndef HK_NYQ_T32
#define HK_NYQ_T32 8  // j1 planes per apply item at N >= 32 (with 2 CTAs per SM; r02: 16 at 1 CTA per SM)
#endif
    // apply work item: T j1-planes x a B x B block of (j2, j3) pairs (B = N up to 32): its
    // three plane pieces per direction (B x B of plane 0, T x B of planes 1 and 2) are
    // 1/T + 2/B of a value per node (N = 64 with whole 64 x 64 planes and T = 4 re-staged
    // plane 0 sixteen times per cell: 72 -> 32 KiB per direction and item)
    static constexpr int T = N >= 32 ? HK_NYQ_T32 : 16;  // j1 planes per apply work item
    static constexpr int B = N < 32 ? N : 32;             // (j2, j3) block edge
    static constexpr int ANT = N >= 32 ? HK_NYQ_APPLY_NT : 256;  // apply threads per CTA
    static constexpr int MP = B * B / ANT;                // (j2, j3) pairs per apply thread
    static constexpr int NBLK = (N / B) * (N / B);        // blocks per plane
    static constexpr int STAGE = B * B + 2 * T * B;       // double2 per direction in SMEM
    static constexpr size_t SMEM2 = size_t(2) * STAGE * sizeof(double2) + 64 * sizeof(double);
};

// Inverse 1-D transforms of `npen` pencils in shared memory, in place, natural
// order: pencil p starts at base + (p / ppg) gstride + (p % ppg) pstride, its
// elements are estride apart.
#ifndef HK_NYQ_SPLIT32
#define HK_NYQ_SPLIT32 1  // N = 32 plane transforms on split pencils (64 data registers, 2 CTAs per SM)
#endif
template <int N>
__device__ __forceinline__ void smem_fft_pass(double2* base, int npen, int pstride, int estride, int ppg = 1 << 30,
                                              int gstride = 0) {
    auto at = [&](int p) { return base + (size_t)(p / ppg) * gstride + (size_t)(p % ppg) * pstride; };
    if constexpr (N <= (HK_NYQ_SPLIT32 ? 16 : 32)) {
        for (int p = threadIdx.x; p < npen; p += blockDim.x) {
            double2* x0 = at(p);
            double2 v[N];
#pragma unroll
            for (int i = 0; i < N; ++i) v[i] = x0[i * estride];
            fft_reg<N, true>(v);
#pragma unroll
            for (int i = 0; i < N; ++i) x0[i * estride] = v[i];
        }
    } else {  // N = 32, 64: one pencil per lane pair (l, l ^ 16), N / 2 values per thread
        constexpr int M = N / 2, Q = M / 2;
        const int lane = threadIdx.x & 31, h = lane >> 4;
        const int slot0 = (threadIdx.x >> 5) * 16 + (lane & 15);
        const int slots = blockDim.x / 2;
        for (int pb = 0; pb < npen; pb += slots) {  // uniform trip count: the pair shuffles
            const int p = pb + slot0;
            const bool on = p < npen;
            double2* x0 = at(on ? p : 0);
            double2 v[M];
#pragma unroll
            for (int j = 0; j < Q; ++j) {
                v[j] = on ? x0[(h * Q + j) * estride] : make_double2(0.0, 0.0);
                v[Q + j] = on ? x0[(M + h * Q + j) * estride] : make_double2(0.0, 0.0);
            }
            fftxh_dif<M, true>(v, h);
            __syncwarp();
            if (on) {
#pragma unroll
                for (int m = 0; m < M; ++m) x0[(2 * m + h) * estride] = v[m];
            }
            __syncwarp();
        }
    }
}

// Phase 1: Z_p = IFFT2((alpha_a + i alpha'_a) F |_{S_p}) = -B_p + i A_p for every
// (listed cell, direction) of the chunk -> planes[w][3][N][N], w = local cell * md + d.
// A work item takes DP directions of one cell at once (N = 32: 2, so the FFT
// passes keep 192 of the 256 threads busy instead of 96).
template <int N>
struct PlanesDP {
    static constexpr int DP = N <= 16 ? 4 : (N <= 32 ? 2 : 1);
    static constexpr int MINB = N == 32 && HK_NYQ_SPLIT32 ? 2 : 1;  // N = 32: split pencils, 2 CTAs per SM
#ifndef HK_NYQ_KB32
#define HK_NYQ_KB32 4  // N = 32 at 128 registers: 6 and 8 spill
#endif
    static constexpr int KB = N == 32 && HK_NYQ_SPLIT32 ? HK_NYQ_KB32 : 12;  // product entries per thread per batch
};
template <int N>
__global__ void __launch_bounds__(256, PlanesDP<N>::MINB) nyq_planes_kernel(const int64_t* __restrict__ list, const int* __restrict__ count,
                                                         int64_t chunk0, int64_t chunk_n, const double2* __restrict__ nyqF,
                                                         const double* __restrict__ ta, const double* __restrict__ tap,
                                                         int md, double2* __restrict__ planes) {
    using G = GeoFix<N>;
    constexpr int ROW = G::ROW, PLANE = G::PLANE, NN = G::NN, DP = PlanesDP<N>::DP;
    extern __shared__ __align__(16) double2 sm[];
    const int t = threadIdx.x;
    int64_t avail = (int64_t)*count - chunk0;
    if (avail > chunk_n) avail = chunk_n;
    const int groups = (md + DP - 1) / DP;  // direction groups per cell
    for (int64_t wi = blockIdx.x; wi < avail * groups; wi += gridDim.x) {
        const int64_t lc = wi / groups;
        const int d0 = (int)(wi % groups) * DP, nd = md - d0 < DP ? md - d0 : DP;
        const int64_t cell = list[chunk0 + lc];
        const double2* Fc = nyqF + cell * 3 * NN;
        __syncthreads();  // previous item's planes written out
        // the restricted products (alpha_a + i alpha'_a) F on the three planes of each
        // direction; the loads of a batch of KB entries per thread are issued together
        // (one L2 round trip per batch instead of one per entry)
        constexpr int KB = PlanesDP<N>::KB;
        const double* ta_d = ta + (int64_t)d0 * 3 * NN;
        const double* tap_d = tap + (int64_t)d0 * 3 * NN;
        const int tot = nd * 3 * NN;
        for (int i0 = 0; i0 < tot; i0 += KB * 256) {
            double av[KB], bv[KB];
            double2 Fv[KB];
#pragma unroll
            for (int k = 0; k < KB; ++k) {
                const int i = i0 + k * 256 + t;
                if (i < tot) {
                    av[k] = __ldg(ta_d + i);
                    bv[k] = __ldg(tap_d + i);
                    Fv[k] = Fc[i % (3 * NN)];
                }
            }
#pragma unroll
            for (int k = 0; k < KB; ++k) {
                const int i = i0 + k * 256 + t;
                if (i < tot)
                    sm[(i / NN) * PLANE + ((i % NN) / N) * ROW + (i % N)] =
                        make_double2(av[k] * Fv[k].x - bv[k] * Fv[k].y, av[k] * Fv[k].y + bv[k] * Fv[k].x);
            }
        }
        __syncthreads();
        smem_fft_pass<N>(sm, 3 * nd * N, ROW, 1);             // rows of the 3 nd planes
        __syncthreads();
        smem_fft_pass<N>(sm, 3 * nd * N, 1, ROW, N, PLANE);   // columns
        __syncthreads();
        double2* out = planes + (lc * md + d0) * 3 * NN;
        for (int i = t; i < tot; i += blockDim.x) out[i] = sm[(i / NN) * PLANE + ((i % NN) / N) * ROW + (i % N)];
    }
}

// Phase 2: per (listed cell, j1 slab, (j2, j3) block) accumulate -sum_d m_d ga_i hb_i
// over all directions in registers (thread: MP (j2, j3) pairs x T planes), then
// Q += jac w acc.
template <int N>
#ifndef HK_NYQ_APPLY_MINB
#define HK_NYQ_APPLY_MINB 2  // apply CTAs per SM (T = 8: <= 128 registers)
#endif
__global__ void __launch_bounds__(GeoFix<N>::ANT, HK_NYQ_APPLY_MINB) nyq_apply_kernel(const int64_t* __restrict__ list, const int* __restrict__ count,
                                                           int64_t chunk0, int64_t chunk_n,
                                                           const double2* __restrict__ planes, int md, double mult0,
                                                           double jac, double w, double* __restrict__ q,
                                                           hk_cell_status* __restrict__ st) {
    using G = GeoFix<N>;
    constexpr int NT = G::ANT;
    constexpr int NN = G::NN, T = G::T, B = G::B, MP = G::MP, STAGE = G::STAGE, SLABS = N / T, NBLK = G::NBLK;
    constexpr int64_t NB = (int64_t)N * N * N;
    extern __shared__ __align__(16) double2 sm[];
    double* red = reinterpret_cast<double*>(sm + 2 * STAGE);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    static_assert(NT % B == 0 && ((NT / B) % 2 == 0 || MP == 1) && T % 2 == 0 && N % B == 0,
                  "pair layout: j2 = j2b + t / B + (NT / B) m, j3 = j3b + t % B");
    const int j2l = t / B, j3l = t % B;  // this thread's pairs in the block: (j2l + (NT / B) m, j3l)
    int64_t avail = (int64_t)*count - chunk0;
    if (avail > chunk_n) avail = chunk_n;
    for (int64_t wi = blockIdx.x; wi < avail * SLABS * NBLK; wi += gridDim.x) {
        const int64_t lc = wi / (SLABS * NBLK);
        const int rem = (int)(wi % (SLABS * NBLK)), slab = rem / NBLK, blk = rem % NBLK;
        const int j1_0 = slab * T, j2b = (blk / (N / B)) * B, j3b = (blk % (N / B)) * B;
        const int j2_0 = j2b + j2l, j3 = j3b + j3l;
        const double s2 = (j2_0 & 1) ? -1.0 : 1.0, s3 = (j3 & 1) ? -1.0 : 1.0, tau = s2 * s3;
        const int64_t cell = list[chunk0 + lc];
        const double2* pc = planes + lc * md * 3 * NN;
        // stage direction d: the block of plane 0 ([j2][j3]), rows j1_0.. of planes 1
        // ([j1][j3], the block's j3 range) and 2 ([j1][j2], its j2 range), 16 B per copy
        auto stage = [&](int d, int buf) {
            const double2* src = pc + (int64_t)d * 3 * NN;
            const uint32_t dst = smem_u32(sm + buf * STAGE);
            for (int i = t; i < STAGE; i += blockDim.x) {
                const double2* g;
                if (i < B * B) {
                    g = src + (j2b + i / B) * N + j3b + i % B;
                } else if (i < B * B + T * B) {
                    const int k = i - B * B;
                    g = src + NN + (j1_0 + k / B) * N + j3b + k % B;
                } else {
                    const int k = i - B * B - T * B;
                    g = src + 2 * NN + (j1_0 + k / B) * N + j2b + k % B;
                }
                cp_async16(dst + i * 16, g);
            }
            cp_async_commit();
        };
        double acc[MP * T];
#pragma unroll
        for (int k = 0; k < MP * T; ++k) acc[k] = 0.0;
        __syncthreads();  // previous item done with both buffers
        stage(0, 0);
        for (int d = 0; d < md; ++d) {
            cp_async_wait_all();
            __syncthreads();  // direction d landed for every thread; buffer d+1 free
            if (d + 1 < md) stage(d + 1, (d + 1) & 1);
            const double2* P0 = sm + (d & 1) * STAGE;
            const double2* P1 = P0 + B * B;
            const double2* P2 = P1 + T * B;
            // A B with A = s1 z0.y + s2 z1.y + s3 z2.y (B: the .x parts) equals A' B' with
            // A' = s1 (s2 z0.y) + z1.y + (s2 s3) z2.y: s2 = (-1)^j2 and s3 = (-1)^j3 are fixed
            // per thread (j2 = j2b + t / B + (NT / B) m with NT / B even, j3 = j3b + t % B),
            // s1 = (-1)^j1 per plane tt.
            // z1 depends on (tt, j3) only: one load per plane for all MP pairs.
            double2 z0[MP];
#pragma unroll
            for (int m = 0; m < MP; ++m) {
                const double2 v = P0[t + NT * m];
                z0[m] = make_double2(s2 * v.x, s2 * v.y);
            }
            // direction 0 carries the multiplicity mult0; the others (1.0 * A == A)
            // take the same arithmetic without the multiply
            auto accumulate = [&](auto with_mu) {
#pragma unroll
                for (int tt = 0; tt < T; ++tt) {
                    const double2 z1 = P1[tt * B + j3l];
#pragma unroll
                    for (int m = 0; m < MP; ++m) {
                        const double2 z2 = P2[tt * B + j2l + (NT / B) * m];
                        const bool odd = ((j1_0 + tt) & 1) != 0;  // j1_0 is even: compile-time per tt
                        const double Aq = fma(tau, z2.y, odd ? z1.y - z0[m].y : z1.y + z0[m].y);
                        const double Bq = fma(tau, z2.x, odd ? z1.x - z0[m].x : z1.x + z0[m].x);  // = -hb_i
                        acc[m * T + tt] = fma(decltype(with_mu)::value ? mult0 * Aq : Aq, Bq,
                                              acc[m * T + tt]);  // += -m ga_i hb_i
                    }
                }
            };
            if (d == 0)
                accumulate(std::true_type{});
            else
                accumulate(std::false_type{});
        }
        double mre = 0.0, n2 = 0.0;
        double* qc = q + cell * NB;
#pragma unroll
        for (int m = 0; m < MP; ++m) {
            const int p = (j2_0 + (NT / B) * m) * N + j3;
#pragma unroll
            for (int tt = 0; tt < T; ++tt) {
                const int64_t gi = (int64_t)(j1_0 + tt) * NN + p;
                const double qv = qc[gi] + jac * w * acc[m * T + tt];
                qc[gi] = qv;
                mre = fmax(mre, fabs(qv));
                n2 += qv * qv;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mre = fmax(mre, __shfl_xor_sync(0xffffffffu, mre, o));
            n2 += __shfl_xor_sync(0xffffffffu, n2, o);
        }
        if (lane == 0) {
            red[warp] = mre;
            red[32 + warp] = n2;
        }
        __syncthreads();
        if (t == 0) {  // the guard cleared max_re / q_norm2 of listed cells
            double m1 = 0.0, s = 0.0;
            for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
                m1 = fmax(m1, red[k]);
                s += red[32 + k];
            }
            atomic_max_nonneg(&st[cell].max_re, m1);
            atomicAdd(&st[cell].q_norm2, s);
        }
    }
}

#ifndef HK_NYQ_CHUNK_BYTES
#define HK_NYQ_CHUNK_BYTES (size_t(2) << 30)  // plane scratch per chunk of listed cells
#endif

// Grows the plane scratch for up to max_cells listed cells.  Growing
// synchronises the device (cudaFree / cudaMalloc), so run_size reserves it
// BEFORE launching the collision kernel: a kernel waiting on host-fed flags
// (the streamed host path) must never sit behind an implicit synchronisation.
int nyq_fix_reserve(hk_ctx ctx, int n, int md, int64_t max_cells) {
    if (max_cells < 1) return HK_OK;
    const size_t per_cell = size_t(md) * 3 * n * n * sizeof(double2);
    int64_t chunk = int64_t(size_t(HK_NYQ_CHUNK_BYTES) / per_cell);
    if (chunk < 1) chunk = 1;
    if (chunk > max_cells) chunk = max_cells;
    const size_t need = per_cell * chunk;
    if (need > ctx->fix_bytes) {
        if (ctx->fix_scratch) {
            cudaStreamSynchronize(ctx->stream);
            cudaFree(ctx->fix_scratch);
            ctx->fix_scratch = nullptr;
            ctx->fix_bytes = 0;
        }
        int s = check_cuda(ctx, cudaMalloc(&ctx->fix_scratch, need), "nyq_fix scratch");
        if (s) return s;
        ctx->fix_bytes = need;
    }
    return HK_OK;
}

// Forces the lazy load of the correction kernels for size n (see preload_guard_kernels).
void nyq_fix_preload(int n) {
    cudaFuncAttributes fa;
    switch (n) {
    case 16: cudaFuncGetAttributes(&fa, nyq_planes_kernel<16>); cudaFuncGetAttributes(&fa, nyq_apply_kernel<16>); break;
    case 32: cudaFuncGetAttributes(&fa, nyq_planes_kernel<32>); cudaFuncGetAttributes(&fa, nyq_apply_kernel<32>); break;
    case 64: cudaFuncGetAttributes(&fa, nyq_planes_kernel<64>); cudaFuncGetAttributes(&fa, nyq_apply_kernel<64>); break;
    default: break;
    }
}

int launch_nyq_fix(hk_ctx ctx, int n, const int64_t* list, const int* count, int64_t max_cells, const double2* nyqF,
                   const double* ta, const double* tap, int md, double mult0, double jac, double w, double* q,
                   hk_cell_status* st) {
    if (max_cells < 1) return HK_OK;
    const size_t per_cell = size_t(md) * 3 * n * n * sizeof(double2);
    int64_t chunk = int64_t(size_t(HK_NYQ_CHUNK_BYTES) / per_cell);
    if (chunk < 1) chunk = 1;
    if (chunk > max_cells) chunk = max_cells;
    int s0 = nyq_fix_reserve(ctx, n, md, max_cells);
    if (s0) return s0;
    double2* planes = static_cast<double2*>(ctx->fix_scratch);
    // persistent grids of exactly the resident CTAs (registers / shared memory decide)
    auto run = [&](auto k1, size_t smem1, auto k2, size_t smem2, int nt2) -> int {
        int s;
        if ((s = check_cuda(ctx, cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1), "smem")) ||
            (s = check_cuda(ctx, cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2), "smem")))
            return s;
        int r1 = 0, r2 = 0;
        if ((s = check_cuda(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r1, k1, 256, smem1), "occupancy")) ||
            (s = check_cuda(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r2, k2, nt2, smem2), "occupancy")))
            return s;
        const unsigned g1 = unsigned(ctx->sm_count * std::max(r1, 1)), g2 = unsigned(ctx->sm_count * std::max(r2, 1));
        for (int64_t c0 = 0; c0 < max_cells; c0 += chunk) {
            k1<<<g1, 256, smem1, ctx->stream>>>(list, count, c0, chunk, nyqF, ta, tap, md, planes);
            k2<<<g2, nt2, smem2, ctx->stream>>>(list, count, c0, chunk, planes, md, mult0, jac, w, q, st);
            ctx->launches += 2;
            if ((s = check_cuda(ctx, cudaGetLastError(), "nyq_fix kernels"))) return s;
        }
        return HK_OK;
    };
    switch (n) {
    case 16: return run(nyq_planes_kernel<16>, GeoFix<16>::SMEM1, nyq_apply_kernel<16>, GeoFix<16>::SMEM2, GeoFix<16>::ANT);
    case 32: return run(nyq_planes_kernel<32>, GeoFix<32>::SMEM1, nyq_apply_kernel<32>, GeoFix<32>::SMEM2, GeoFix<32>::ANT);
    case 64: return run(nyq_planes_kernel<64>, GeoFix<64>::SMEM1, nyq_apply_kernel<64>, GeoFix<64>::SMEM2, GeoFix<64>::ANT);
    default: return fail(ctx, HK_UNSUPPORTED, "nyq_fix: n = 16, 32, 64");
    }
}

}  // namespace hk
