// hk_coll64.cu — collision operator at N = 64 (config 5), sm_100a.
//
// Same operator as hk_collision.cu (spectral_collision, src/spectral.cpp:114-154;
// FftWorkspace3d, src/fft.cpp:49-81), re-partitioned for a 64^3 cell whose
// spectrum (4 MiB complex) no longer fits one SM:
//
//   * a TEAM of C = 32 CTAs (one per SM, cooperative launch, 4 teams = 128
//     SMs) evaluates one cell at a time; CTA r owns P = 2 planes: i1 planes
//     rP..rP+1 of the spectrum (producer side) and j3 planes of the nodal
//     fields (consumer side);
//   * F for the CTA's two i1 planes lives in TMEM (256 of 512 columns), the
//     gain accumulators of its two j3 planes in the rest;
//   * every 64-point pencil is split over the lane pair (l, l ^ 16): a thread
//     holds 32 complex values (fftxh_dit / fftxh_dif), so one warp covers 16
//     pencils and four warps a whole plane;
//   * warps 0-3 produce (weights x F, inverse FFT over i3, 16-byte st.cg into
//     an L2 exchange slot), warps 4-7 consume one j3 plane at a time (cp.async
//     pull, double-buffered; inverse FFT over i2, then i1; product; gain);
//     producers and consumers of a team synchronise with per-slot ready/done
//     counters in global memory (release / relaxed-poll acquire, D slots).
//
// FAST (default): one Hermitian-packed transform per distinct direction,
// IFFT(F (alpha_s + i alpha'_s)) = gs + i hs, gain += m gs hs; the dropped
// Nyquist term is bounded per cell by guard_kernel and failing cells are
// recomputed by EXACT.  EXACT: the reference's arithmetic, two complex
// transforms per direction (alpha F, alpha' F) and a complex gain; the ga
// field is parked in its landing buffer until gb arrives.
#include <cstdio>
#include <cstdlib>

#include "hk_coll.cuh"
#include "hk_common.cuh"

namespace hk {

#ifndef HK_SLOTS64
#define HK_SLOTS64 2  // config 5 slab: D = 2 1609 ms, 3 1636, 4 1665
#endif
struct Geo64 {
    static constexpr int N = 64, C = 32, P = 2, M = 32, Q = 16;
    static constexpr int ROW = N + 1;           // padded SMEM row (conflict-free columns)
    static constexpr int PLANE = N * ROW;       // double2 per landing plane
    static constexpr int D = HK_SLOTS64;        // exchange slots per team
    static constexpr int64_t NB = (int64_t)N * N * N;
    static constexpr int BLK = P * N * N;       // double2 per destination CTA per field
    static constexpr int64_t SLOT = (int64_t)C * BLK;
    static constexpr unsigned ARR = C * 4;      // warp arrivals per slot use (each role)
    static constexpr uint32_t TM_COLS = 512;
    static constexpr size_t SMEM = size_t(3 * PLANE) * sizeof(double2) + 128;
    static constexpr size_t XCHG_PER_TEAM = size_t(D) * SLOT * sizeof(double2);
};
#ifndef HK_PULL_TMA64
#define HK_PULL_TMA64 1  // consumer plane pulls by TMA bulk row copies instead of per-thread cp.async
#endif
#ifndef HK_W_TMA64
#define HK_W_TMA64 1  // FAST producer weight planes by TMA bulk copy: 163 ms vs 198 ms per 1024 shock cells with per-thread cp.async (r02)
#endif

template <bool EXACT>
__global__ void __launch_bounds__(256, 1) coll64_kernel(CollArgs a) {
    using G = Geo64;
    constexpr int N = G::N, C = G::C, P = G::P, M = G::M, Q = G::Q, ROW = G::ROW, PLANE = G::PLANE, D = G::D;
    constexpr int64_t NB = G::NB;
    constexpr int BLK = G::BLK;
    constexpr int64_t SLOT = G::SLOT;
    constexpr unsigned ARR = G::ARR;
    constexpr int GCOLS = EXACT ? 128 : 64;  // TMEM columns of gain per plane
    extern __shared__ __align__(16) double2 smem[];
    double2* Rvb = smem;              // consumer landing planes [2][N][ROW]
    double2* Pw = smem + 2 * PLANE;   // producer: prologue plane / weight staging
    uint64_t* fbar = reinterpret_cast<uint64_t*>(smem + 3 * PLANE);  // [P] F-plane ready
    uint32_t* tslot = reinterpret_cast<uint32_t*>(fbar + P);

    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    const int rw = warp & 3;                 // role-local warp == TMEM lane quarter
    const int pp = 16 * rw + (lane & 15);    // pencil (row / column) within a plane
    const int h = lane >> 4;                 // half of the pencil
    const int u = t & 127;
    const bool producer = t < 128;
    const unsigned team = blockIdx.x / C, r = blockIdx.x % C, nteams = gridDim.x / C;
    const int64_t count = a.list_count ? (int64_t)*a.list_count : a.ncells;
    double2* X = a.xchg + (int64_t)team * D * SLOT;
    unsigned* ready = a.team_ctr + (int64_t)team * 2 * D;
    unsigned* done = ready + D;

    if (warp == 0) tmem_alloc(tslot, G::TM_COLS);
    if (t < P) mbar_init(smem_u32(fbar + t), 128);
    if (t == 0) asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const uint32_t tm = *tslot + ((uint32_t)(32 * rw) << 16);
    const uint32_t tmF = tm, tmG = tm + 256;  // F plane pl: +128 pl; gain plane pl: +GCOLS pl
    const int nfields = EXACT ? 2 * a.md + 1 : a.md + 1;
    unsigned g = 0, ncell = 0;

    if (producer) {
        // ================================ PRODUCERS ================================
        // Weight staging: thread-private slots [m][u] (interleaved: conflict-free).
        const uint32_t wb_s = smem_u32(Pw);
        auto issue_w = [&](int fi, int pl) {
            const int i1 = r * P + pl;
            if constexpr (!EXACT) {
                const double2* wt = a.wfast + (int64_t)fi * NB + (int64_t)i1 * N * N + pp;
#pragma unroll
                for (int m = 0; m < M; ++m) cp_async16(wb_s + (m * 128 + u) * 16, wt + (2 * m + h) * N);
            } else {
                const double* base = (fi == 2 * a.md) ? a.loss : ((fi & 1) ? a.alpha_p : a.alpha) + (int64_t)(fi >> 1) * NB;
                const double* wt = base + (int64_t)i1 * N * N + pp;
#pragma unroll
                for (int m = 0; m < M; ++m) cp_async8(wb_s + (m * 128 + u) * 8, wt + (2 * m + h) * N);
            }
            cp_async_commit();
        };
        auto acquire = [&](unsigned gg) {
            if (lane == 0) spin_geq(done + gg % D, ARR * (gg / D));
            __syncwarp();
        };
        auto publish = [&](unsigned gg) {
            __syncwarp();
            if (lane == 0) signal_add(ready + gg % D);
        };
        for (int64_t it = team; it < count; it += nteams, ++ncell) {
            const int64_t cell = a.list ? a.list[it] : it;
            const double* fc = a.f + cell * NB;
            // ---- prologue: per j3 plane, 2-D forward transform (j2 then j1) -> owner of k1 ----
            for (int pl = 0; pl < P; ++pl) {
                const int j3 = r * P + pl;
                named_bar(1, 128);  // Pw free
                for (int idx = u; idx < N * N; idx += 128)
                    Pw[(idx / N) * ROW + (idx % N)] = make_double2(__ldg(fc + (int64_t)idx * N + j3), 0.0);
                named_bar(1, 128);
                {  // rows j1 = pp over j2 (DIF), back in natural order
                    double2* row = Pw + pp * ROW;
                    double2 v[M];
#pragma unroll
                    for (int j = 0; j < Q; ++j) {
                        v[j] = row[h * Q + j];
                        v[Q + j] = row[M + h * Q + j];
                    }
                    fftxh_dif<M, false>(v, h);
                    __syncwarp();
#pragma unroll
                    for (int m = 0; m < M; ++m) row[2 * m + h] = v[m];
                }
                named_bar(1, 128);  // columns need every row
                {  // columns k2 = pp over j1 (DIT): v[j] = K1 index hQ + j, v[Q + j] = M + hQ + j
                    const double2* col = Pw + pp;
                    double2 v[M];
#pragma unroll
                    for (int m = 0; m < M; ++m) v[m] = col[(2 * m + h) * ROW];
                    fftxh_dit<M, false>(v, h);
                    if (pl == 0) acquire(g);
                    double2* Xs = X + (int64_t)(g % D) * SLOT;
#pragma unroll
                    for (int j = 0; j < Q; ++j) {
                        const int ka = h * Q + j, kb = M + h * Q + j;
                        st_cg16(Xs + (int64_t)(ka / P) * BLK + ((ka % P) * N + pp) * N + j3, v[j]);
                        st_cg16(Xs + (int64_t)(kb / P) * BLK + ((kb % P) * N + pp) * N + j3, v[Q + j]);
                    }
                }
            }
            publish(g);
            ++g;
            named_bar(1, 128);  // prologue reads of Pw done: weight staging may overwrite it
            issue_w(0, 0);
            // ---- phase A: X = F * weights, inverse FFT over i3, -> owner of j3 ----
            for (int fi = 0; fi < nfields; ++fi) {
#pragma unroll 1
                for (int pl = 0; pl < P; ++pl) {
                    if (fi == 0) {
                        mbar_wait_parity(smem_u32(fbar + pl), ncell & 1);  // consumers put F(plane) in TMEM
                        tmem_fence_after();
                    }
                    // F of this half-pencil (32 complex = 128 TMEM columns): four x32
                    // loads and ONE wait, overlapping the weight reads
                    double2 x[M];
                    {
                        uint32_t r0[32], r1[32], r2[32], r3[32];
                        tmem_ld32_nowait(tmF + 128 * pl, r0);
                        tmem_ld32_nowait(tmF + 128 * pl + 32, r1);
                        tmem_ld32_nowait(tmF + 128 * pl + 64, r2);
                        tmem_ld32_nowait(tmF + 128 * pl + 96, r3);
                        cp_async_wait_all();
                        __syncwarp();
                        tmem_wait_ld();
#pragma unroll
                        for (int m = 0; m < 8; ++m) {
                            x[m] = make_double2(tmem_pair(r0[4 * m], r0[4 * m + 1]), tmem_pair(r0[4 * m + 2], r0[4 * m + 3]));
                            x[8 + m] = make_double2(tmem_pair(r1[4 * m], r1[4 * m + 1]), tmem_pair(r1[4 * m + 2], r1[4 * m + 3]));
                            x[16 + m] = make_double2(tmem_pair(r2[4 * m], r2[4 * m + 1]), tmem_pair(r2[4 * m + 2], r2[4 * m + 3]));
                            x[24 + m] = make_double2(tmem_pair(r3[4 * m], r3[4 * m + 1]), tmem_pair(r3[4 * m + 2], r3[4 * m + 3]));
                        }
                    }
                    if constexpr (!EXACT) {
                        const double2* wb = Pw;
#pragma unroll
                        for (int m = 0; m < M; ++m) {
                            const double2 w = wb[m * 128 + u], v = x[m];
                            x[m] = make_double2(v.x * w.x - v.y * w.y, v.x * w.y + v.y * w.x);
                        }
                    } else {
                        const double* wb = reinterpret_cast<const double*>(Pw);
#pragma unroll
                        for (int m = 0; m < M; ++m) {
                            const double w = wb[m * 128 + u];
                            x[m] = make_double2(x[m].x * w, x[m].y * w);
                        }
                    }
                    __syncwarp();
                    if (pl + 1 < P)
                        issue_w(fi, pl + 1);
                    else if (fi + 1 < nfields)
                        issue_w(fi + 1, 0);
                    fftxh_dit<M, true>(x, h);  // x[j] = Y[hQ + j], x[Q + j] = Y[M + hQ + j]
                    if (pl == 0) acquire(g);
                    double2* Xs = X + (int64_t)(g % D) * SLOT;
                    const int i1 = r * P + pl;
#pragma unroll
                    for (int j = 0; j < Q; ++j) {
                        const int ja = h * Q + j, jb = M + h * Q + j;
                        st_cg16(Xs + (int64_t)(ja / P) * BLK + ((ja % P) * N + i1) * N + pp, x[j]);
                        st_cg16(Xs + (int64_t)(jb / P) * BLK + ((jb % P) * N + i1) * N + pp, x[Q + j]);
                    }
                }
                publish(g);
                ++g;
            }
        }
    } else {
        // ================================ CONSUMERS ================================
        // Units: (field, plane) pulls in a fixed order per cell; unit k lands in
        // Rvb[k & 1] (units per cell is even).  Field 0 is the prologue.
        const int upc = 2 * (1 + nfields);
        auto unit_of = [&](int k, int& fi, int& pl) {
            if (k < 2) {
                fi = 0;
                pl = k;
                return;
            }
            const int j = k - 2;
            if (EXACT && j < 4 * a.md) {  // (ga, p0) (gb, p0) (ga, p1) (gb, p1) per direction
                fi = 1 + 2 * (j >> 2) + (j & 1);
                pl = (j >> 1) & 1;
            } else {
                const int jj = EXACT ? j - 4 * a.md : j;
                fi = (EXACT ? 1 + 2 * a.md : 1) + (jj >> 1);
                pl = jj & 1;
            }
        };
        auto pull = [&](unsigned gs, int pl, int buf) {  // my 16 rows of (slot gs, plane pl)
            const double2* src = X + (int64_t)(gs % D) * SLOT + (int64_t)r * BLK + (int64_t)pl * N * N + 16 * rw * N;
            const uint32_t d0 = smem_u32(Rvb + buf * PLANE + 16 * rw * ROW);
#pragma unroll 4
            for (int k = 0; k < 16; ++k) {
                cp_async16(d0 + (k * ROW + lane) * 16, src + k * N + lane);
                cp_async16(d0 + (k * ROW + 32 + lane) * 16, src + k * N + 32 + lane);
            }
            cp_async_commit();
        };
        auto issue = [&](unsigned gs, int pl, int buf) {
            if (lane == 0) spin_geq(ready + gs % D, ARR * (gs / D + 1));
            __syncwarp();
            pull(gs, pl, buf);
        };
        auto try_issue = [&](unsigned gs, int pl, int buf) -> bool {  // pull only if already published
            unsigned v = 0;
            if (lane == 0) asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(ready + gs % D) : "memory");
            v = __shfl_sync(0xffffffffu, v, 0);
            if ((int)(v - ARR * (gs / D + 1)) < 0) return false;
            pull(gs, pl, buf);
            return true;
        };
        auto complete = [&](unsigned gs, int pl) {
            cp_async_wait_all();
            __syncwarp();
            if (pl == P - 1 && lane == 0) signal_add_relaxed(done + gs % D);  // last pull of this slot
            named_bar(2, 128);  // every warp's rows have landed; previous unit fully consumed
        };
        if ((int64_t)team < count) issue(0, 0, 0);
        for (int64_t it = team; it < count; it += nteams, ++ncell) {
            const int64_t cell = a.list ? a.list[it] : it;
            const double* fc = a.f + cell * NB;
            const unsigned gb = ncell * (1 + nfields);
            const bool more_cells = it + nteams < count;
            double mre = 0.0, mim = 0.0, n2 = 0.0, l2 = 0.0;
#pragma unroll 1
            for (int k = 0; k < upc; ++k) {
                int fi, pl;
                unit_of(k, fi, pl);
                const unsigned gs = gb + fi;
                const int buf = k & 1;
                double2* Rv = Rvb + buf * PLANE;
                complete(gs, pl);
                const bool has_next = (k + 1 < upc) || more_cells;
                unsigned gs2 = gb + 1 + nfields;
                int pl2 = 0;
                if (k + 1 < upc) {
                    int f2;
                    unit_of(k + 1, f2, pl2);
                    gs2 = gb + f2;
                }
                // Deferred successor: after the last prologue plane (the first field
                // needs F in TMEM) and, EXACT, after a gb unit (the other buffer holds ga).
                const bool defer = (fi == 0 && pl == P - 1) || (EXACT && fi >= 1 && fi <= 2 * a.md && ((fi - 1) & 1));
                // successor pull: now if published, else retried between the passes
                bool pending = has_next && !defer && !try_issue(gs2, pl2, buf ^ 1);
                if (fi == 0) {
                    // ---- prologue: forward over k3 of rows (k1 = rP + pl, k2 = pp) -> F (TMEM) ----
                    const double2* row = Rv + pp * ROW;
                    const int k1 = r * P + pl, k2 = pp;
                    double2 v[M];
#pragma unroll
                    for (int j = 0; j < Q; ++j) {
                        v[j] = row[h * Q + j];
                        v[Q + j] = row[M + h * Q + j];
                    }
                    fftxh_dif<M, false>(v, h);  // v[m] = F[k3 = 2m + h] (unscaled)
                    const double s = 1.0 / double(NB);
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        double w8[8];
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            w8[2 * i] = v[4 * c + i].x * s;
                            w8[2 * i + 1] = v[4 * c + i].y * s;
                        }
                        tmem_st16(tmF + 128 * pl + 16 * c, w8);
                    }
                    if (!EXACT && a.nyq) {
                        constexpr int H = N / 2;
                        double2* ny = a.nyq + cell * 3 * N * N;
                        if (h == 0) ny[2 * N * N + k1 * N + k2] = make_double2(s * v[H / 2].x, s * v[H / 2].y);
                        if (k2 == H) {
#pragma unroll
                            for (int m = 0; m < M; ++m)
                                ny[1 * N * N + k1 * N + 2 * m + h] = make_double2(s * v[m].x, s * v[m].y);
                        }
                        if (k1 == H) {
#pragma unroll
                            for (int m = 0; m < M; ++m) ny[k2 * N + 2 * m + h] = make_double2(s * v[m].x, s * v[m].y);
                        }
                    }
                    const double z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
                    for (int c = 0; c < GCOLS / 16; ++c) tmem_st16(tmG + GCOLS * pl + 16 * c, z);
                    tmem_wait_st();
                    tmem_fence_before();
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(fbar + pl)) : "memory");
                    if (pending) issue(gs2, pl2, buf ^ 1);
                } else {
                    // ---- field: inverse over i2 (rows i1 = pp), then i1 (columns j2 = pp) ----
                    {
                        double2* row = Rv + pp * ROW;
                        double2 v[M];
#pragma unroll
                        for (int j = 0; j < Q; ++j) {
                            v[j] = row[h * Q + j];
                            v[Q + j] = row[M + h * Q + j];
                        }
                        fftxh_dif<M, true>(v, h);
                        __syncwarp();
#pragma unroll
                        for (int m = 0; m < M; ++m) row[2 * m + h] = v[m];
                    }
                    if (pending) pending = !try_issue(gs2, pl2, buf ^ 1);
                    named_bar(2, 128);  // columns need every row
                    double2 y[M];       // y[j] = node j1 = hQ + j, y[Q + j] = node M + hQ + j
                    double2* col = Rv + pp;
#pragma unroll
                    for (int m = 0; m < M; ++m) y[m] = col[(2 * m + h) * ROW];
                    fftxh_dit<M, true>(y, h);
                    if (pending) issue(gs2, pl2, buf ^ 1);
                    const bool is_loss = EXACT ? (fi == 1 + 2 * a.md) : (fi == 1 + a.md);
                    const int j3 = r * P + pl;
                    if (!is_loss) {
                        if constexpr (!EXACT) {
                            const double mu = (fi == 1) ? a.mult0 : 1.0;
                            uint32_t g0[32], g1[32];  // 32 gain accumulators: two x32 loads, one wait
                            tmem_ld32_nowait(tmG + GCOLS * pl, g0);
                            tmem_ld32_nowait(tmG + GCOLS * pl + 32, g1);
                            tmem_wait_ld();
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                double gv[8];
#pragma unroll
                                for (int i = 0; i < 8; ++i) {
                                    const int k = 16 * (c & 1) + 2 * i;
                                    const double old = (c < 2) ? tmem_pair(g0[k], g0[k + 1]) : tmem_pair(g1[k], g1[k + 1]);
                                    gv[i] = old + mu * (y[8 * c + i].x * y[8 * c + i].y);
                                }
                                tmem_st16(tmG + GCOLS * pl + 16 * c, gv);
                            }
                            tmem_wait_st();
                        } else if (!((fi - 1) & 1)) {  // ga: park it in place for the gb unit
                            __syncwarp();
#pragma unroll
                            for (int j = 0; j < Q; ++j) {
                                col[(h * Q + j) * ROW] = y[j];
                                col[(M + h * Q + j) * ROW] = y[Q + j];
                            }
                        } else {  // gb: gain += m ga gb (complex), ga in the other buffer
                            const double mu = (fi == 2) ? a.mult0 : 1.0;
                            const double2* gcol = Rvb + (buf ^ 1) * PLANE + pp;
#pragma unroll
                            for (int c = 0; c < 8; ++c) {  // nodes jj = 4c .. 4c + 3
                                double gv[8];
                                tmem_ld16(tmG + GCOLS * pl + 16 * c, gv);
#pragma unroll
                                for (int i = 0; i < 4; ++i) {
                                    const int jj = 4 * c + i;
                                    const int j1 = jj < Q ? h * Q + jj : M + h * Q + (jj - Q);
                                    const double2 ga = gcol[j1 * ROW], gbv = y[jj];
                                    gv[2 * i] += mu * (ga.x * gbv.x - ga.y * gbv.y);
                                    gv[2 * i + 1] += mu * (ga.x * gbv.y + ga.y * gbv.x);
                                }
                                tmem_st16(tmG + GCOLS * pl + 16 * c, gv);
                            }
                            tmem_wait_st();
                        }
                    } else {
                        // ---- epilogue for plane pl: Q = jac (w gain - f loss) at (j1, pp, j3) ----
                        double* qc = a.q + cell * NB;
                        if constexpr (!EXACT) {
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                double gv[8];
                                tmem_ld16(tmG + GCOLS * pl + 16 * c, gv);
#pragma unroll
                                for (int i = 0; i < 8; ++i) {
                                    const int jj = 8 * c + i;
                                    const int j1 = jj < Q ? h * Q + jj : M + h * Q + (jj - Q);
                                    const int64_t gi = ((int64_t)j1 * N + pp) * N + j3;
                                    const double lt = __ldg(fc + gi) * y[jj].x;
                                    const double qre = a.jac * (a.w * gv[i] - lt);
                                    qc[gi] = qre;
                                    mre = fmax(mre, fabs(qre));
                                    n2 += qre * qre;
                                    l2 += lt * lt;
                                }
                            }
                        } else {
#pragma unroll
                            for (int c = 0; c < 8; ++c) {
                                double gv[8];
                                tmem_ld16(tmG + GCOLS * pl + 16 * c, gv);
#pragma unroll
                                for (int i = 0; i < 4; ++i) {
                                    const int jj = 4 * c + i;
                                    const int j1 = jj < Q ? h * Q + jj : M + h * Q + (jj - Q);
                                    const int64_t gi = ((int64_t)j1 * N + pp) * N + j3;
                                    const double fv = __ldg(fc + gi);
                                    const double qre = a.jac * (a.w * gv[2 * i] - fv * y[jj].x);
                                    const double qim = a.jac * (a.w * gv[2 * i + 1] - fv * y[jj].y);
                                    qc[gi] = qre;
                                    mre = fmax(mre, fabs(qre));
                                    mim = fmax(mim, fabs(qim));
                                    n2 += qre * qre;
                                }
                            }
                        }
                        if (pl == P - 1) {
#pragma unroll
                            for (int o = 16; o > 0; o >>= 1) {
                                mre = fmax(mre, __shfl_xor_sync(0xffffffffu, mre, o));
                                mim = fmax(mim, __shfl_xor_sync(0xffffffffu, mim, o));
                                n2 += __shfl_xor_sync(0xffffffffu, n2, o);
                                if (!EXACT) l2 += __shfl_xor_sync(0xffffffffu, l2, o);
                            }
                            if (lane == 0 && a.st) {
                                hk_cell_status* sc = a.st + cell;
                                atomic_max_nonneg(&sc->max_re, mre);
                                atomicAdd(&sc->q_norm2, n2);
                                if (!EXACT) atomicAdd(&sc->loss_norm2, a.jac * a.jac * l2);
                                if (EXACT) {
                                    atomic_max_nonneg(&sc->max_im, mim);
                                    if (r == 0 && rw == 0) atomicOr(&sc->flags, HK_CELL_EXACT);
                                }
                            }
                        }
                    }
                }
                if (has_next && defer) {
                    named_bar(2, 128);  // every warp is done with the other buffer
                    issue(gs2, pl2, buf ^ 1);
                }
            }
        }
    }
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    if (warp == 0) tmem_dealloc(*tslot, G::TM_COLS);
}

// FAST path with 12 warps: warps 0-3 produce exactly as in coll64_kernel,
// warps 4-11 are two consumer groups of four, group k owning j3 plane k
// (single landing buffer each), so both planes of a field are consumed
// concurrently: one producer and two consumers per scheduler, matching the
// 1 : 2 transform count of the roles (as coll_fast_w12_kernel at N = 32).
#ifndef HK_PROD_PHASES
#define HK_PROD_PHASES 0  // role phase timers (HK_PROF_SPIN report), profiling builds only
#endif
#if HK_PROD_PHASES
#define HK_PH_T(v) long long v = clock64()
#define HK_PH_ADD(k, v) do { const long long _t = clock64(); ph[k] += _t - v; v = _t; } while (0)
#else
#define HK_PH_T(v) do {} while (0)
#define HK_PH_ADD(k, v) do {} while (0)
#endif
__global__ void __launch_bounds__(384, 1) coll64_w12_kernel(CollArgs a) {
    constexpr bool EXACT = false;
    using G = Geo64;
    constexpr int N = G::N, C = G::C, P = G::P, M = G::M, Q = G::Q, ROW = G::ROW, PLANE = G::PLANE, D = G::D;
    constexpr int64_t NB = G::NB;
    constexpr int BLK = G::BLK;
    constexpr int64_t SLOT = G::SLOT;
    constexpr unsigned ARR = G::ARR;          // producer warp arrivals per slot (ready)
    constexpr unsigned ARR_C = 2 * G::ARR;    // consumer warp arrivals per slot (done)
    constexpr int GCOLS = EXACT ? 128 : 64;  // TMEM columns of gain per plane
    extern __shared__ __align__(16) double2 smem[];
    double2* Rvb = smem;              // consumer landing planes [group][N][ROW]
    double2* Pw = smem + 2 * PLANE;   // producer: prologue plane / weight staging
    uint64_t* fbar = reinterpret_cast<uint64_t*>(smem + 3 * PLANE);  // [P] F-plane ready
    uint32_t* tslot = reinterpret_cast<uint32_t*>(fbar + P);
    uint64_t* wbar = fbar + P + 1;  // weight-plane TMA barrier of the producer group
    uint64_t* cbar = fbar + P + 5;  // [8] consumer pull barriers (HK_PULL_TMA64)

    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    const int rw = warp & 3;                 // role-local warp == TMEM lane quarter
    const int pp = 16 * rw + (lane & 15);    // pencil (row / column) within a plane
    const int h = lane >> 4;                 // half of the pencil
    const int u = t & 127;
    const bool producer = t < 128;
    const unsigned team = blockIdx.x / C, r = blockIdx.x % C, nteams = gridDim.x / C;
    const int64_t count = a.list_count ? (int64_t)*a.list_count : a.ncells;
    double2* X = a.xchg + (int64_t)team * D * SLOT;
    unsigned* ready = a.team_ctr + (int64_t)team * 2 * D;
    unsigned* done = ready + D;

    if (warp == 0) tmem_alloc(tslot, G::TM_COLS);
    if (t < P) mbar_init(smem_u32(fbar + t), 128);
    if (HK_W_TMA64 && t >= 32 && t < 36) mbar_init(smem_u32(wbar + (t - 32)), 1);
    if (HK_PULL_TMA64 && t >= 64 && t < 72) mbar_init(smem_u32(cbar + (t - 64)), 1);
    if (t == 0) asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const uint32_t tm = *tslot + ((uint32_t)(32 * rw) << 16);
    const uint32_t tmF = tm, tmG = tm + 256;  // F plane pl: +128 pl; gain plane pl: +GCOLS pl
    const int nfields = EXACT ? 2 * a.md + 1 : a.md + 1;
    unsigned g = 0, ncell = 0;

    if (producer) {
        // ================================ PRODUCERS ================================
        // Weight staging: thread-private slots [m][u] (interleaved: conflict-free).
        const uint32_t wb_s = smem_u32(Pw);
#if HK_W_TMA64
        // each producer warp fetches its own 16 pencils' weights of the unit's plane,
        // one contiguous 16 KiB block of the warp-blocked table ([i1][i2/16][i3][i2%16],
        // hk_weights.cu), by one bulk copy completing on its own mbarrier: no barrier
        // across the producer warps
        const uint32_t wbar_s = smem_u32(wbar + rw);
        const uint32_t wq_s = wb_s + rw * (N * 16 * 16);
        unsigned wph = 0;
        auto issue_w = [&](int fi, int pl) {
            const int i1 = r * P + pl;
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // my reads of the block before the async write
            __syncwarp();
            if (lane == 0) {
                mbar_arrive_expect_tx(wbar_s, N * 16 * 16);
                bulk_g2s(wq_s, a.wfast + (int64_t)fi * NB + ((int64_t)i1 * 4 + rw) * (N * 16), N * 16 * 16, wbar_s);
            }
        };
        auto wait_w = [&]() {
            mbar_wait_parity(wbar_s, wph);
            wph ^= 1;
        };
#else
        auto wait_w = [&]() { cp_async_wait_all(); };
        auto issue_w = [&](int fi, int pl) {  // warp-blocked table: pencil pp's column in block rw
            const int i1 = r * P + pl;
            const double2* wt = a.wfast + (int64_t)fi * NB + ((int64_t)i1 * 4 + rw) * (N * 16) + (pp & 15);
#pragma unroll
            for (int m = 0; m < M; ++m) cp_async16(wb_s + (m * 128 + u) * 16, wt + (2 * m + h) * 16);
            cp_async_commit();
        };
#endif
        long long spin_cyc = 0;
        const long long t_start = clock64();
#if HK_PROD_PHASES
        long long ph[6] = {0, 0, 0, 0, 0, 0};
#endif
        auto acquire = [&](unsigned gg) {
            if (lane == 0) spin_cyc += spin_geq(done + gg % D, ARR_C * (gg / D));
            __syncwarp();
        };
        auto publish = [&](unsigned gg) {
            __syncwarp();
            if (lane == 0) signal_add(ready + gg % D);
        };
        for (int64_t it = team; it < count; it += nteams, ++ncell) {
            const int64_t cell = a.list ? a.list[it] : it;
            const double* fc = a.f + cell * NB;
            // ---- prologue: per j3 plane, 2-D forward transform (j2 then j1) -> owner of k1 ----
            for (int pl = 0; pl < P; ++pl) {
                const int j3 = r * P + pl;
                named_bar(1, 128);  // Pw free
                for (int idx = u; idx < N * N; idx += 128)
                    Pw[(idx / N) * ROW + (idx % N)] = make_double2(__ldg(fc + (int64_t)idx * N + j3), 0.0);
                named_bar(1, 128);
                {  // rows j1 = pp over j2 (DIF), back in natural order
                    double2* row = Pw + pp * ROW;
                    double2 v[M];
#pragma unroll
                    for (int j = 0; j < Q; ++j) {
                        v[j] = row[h * Q + j];
                        v[Q + j] = row[M + h * Q + j];
                    }
                    fftxh_dif<M, false>(v, h);
                    __syncwarp();
#pragma unroll
                    for (int m = 0; m < M; ++m) row[2 * m + h] = v[m];
                }
                named_bar(1, 128);  // columns need every row
                {  // columns k2 = pp over j1 (DIT): v[j] = K1 index hQ + j, v[Q + j] = M + hQ + j
                    const double2* col = Pw + pp;
                    double2 v[M];
#pragma unroll
                    for (int m = 0; m < M; ++m) v[m] = col[(2 * m + h) * ROW];
                    fftxh_dit<M, false>(v, h);
                    if (pl == 0) acquire(g);
                    double2* Xs = X + (int64_t)(g % D) * SLOT;
#pragma unroll
                    for (int j = 0; j < Q; ++j) {
                        const int ka = h * Q + j, kb = M + h * Q + j;
                        st_cg16(Xs + (int64_t)(ka / P) * BLK + ((ka % P) * N + pp) * N + j3, v[j]);
                        st_cg16(Xs + (int64_t)(kb / P) * BLK + ((kb % P) * N + pp) * N + j3, v[Q + j]);
                    }
                }
            }
            publish(g);
            ++g;
            named_bar(1, 128);  // prologue reads of Pw done: weight staging may overwrite it
            issue_w(0, 0);
            // ---- phase A: X = F * weights, inverse FFT over i3, -> owner of j3 ----
            for (int fi = 0; fi < nfields; ++fi) {
#pragma unroll 1
                for (int pl = 0; pl < P; ++pl) {
                    HK_PH_T(tA);
                    if (fi == 0) {
                        mbar_wait_parity(smem_u32(fbar + pl), ncell & 1);  // consumers put F(plane) in TMEM
                        tmem_fence_after();
                    }
                    // F of this half-pencil (32 complex = 128 TMEM columns): four x32
                    // loads and ONE wait, overlapping the weight reads
                    double2 x[M];
                    {
                        uint32_t r0[32], r1[32], r2[32], r3[32];
                        tmem_ld32_nowait(tmF + 128 * pl, r0);
                        tmem_ld32_nowait(tmF + 128 * pl + 32, r1);
                        tmem_ld32_nowait(tmF + 128 * pl + 64, r2);
                        tmem_ld32_nowait(tmF + 128 * pl + 96, r3);
                        wait_w();
                        __syncwarp();
                        tmem_wait_ld();
                        HK_PH_ADD(0, tA);
#pragma unroll
                        for (int m = 0; m < 8; ++m) {
                            x[m] = make_double2(tmem_pair(r0[4 * m], r0[4 * m + 1]), tmem_pair(r0[4 * m + 2], r0[4 * m + 3]));
                            x[8 + m] = make_double2(tmem_pair(r1[4 * m], r1[4 * m + 1]), tmem_pair(r1[4 * m + 2], r1[4 * m + 3]));
                            x[16 + m] = make_double2(tmem_pair(r2[4 * m], r2[4 * m + 1]), tmem_pair(r2[4 * m + 2], r2[4 * m + 3]));
                            x[24 + m] = make_double2(tmem_pair(r3[4 * m], r3[4 * m + 1]), tmem_pair(r3[4 * m + 2], r3[4 * m + 3]));
                        }
                    }
                    if constexpr (!EXACT) {
#ifndef HK_EXP_NOMUL
                        const double2* wb = Pw;
#pragma unroll
                        for (int m = 0; m < M; ++m) {
#if HK_W_TMA64
                            const double2 w = wb[rw * (N * 16) + (2 * m + h) * 16 + (pp & 15)], v = x[m];
#else
                            const double2 w = wb[m * 128 + u], v = x[m];
#endif
                            x[m] = make_double2(v.x * w.x - v.y * w.y, v.x * w.y + v.y * w.x);
                        }
#endif
                    } else {
                        const double* wb = reinterpret_cast<const double*>(Pw);
#pragma unroll
                        for (int m = 0; m < M; ++m) {
                            const double w = wb[m * 128 + u];
                            x[m] = make_double2(x[m].x * w, x[m].y * w);
                        }
                    }
                    __syncwarp();
#ifndef HK_EXP_NOISSUE
                    if (pl + 1 < P)
                        issue_w(fi, pl + 1);
                    else if (fi + 1 < nfields)
                        issue_w(fi + 1, 0);
#endif
                    HK_PH_ADD(1, tA);
                    fftxh_dit<M, true>(x, h);  // x[j] = Y[hQ + j], x[Q + j] = Y[M + hQ + j]
                    HK_PH_ADD(2, tA);
                    if (pl == 0) acquire(g);
                    HK_PH_ADD(3, tA);
                    double2* Xs = X + (int64_t)(g % D) * SLOT;
                    const int i1 = r * P + pl;
#pragma unroll
                    for (int j = 0; j < Q; ++j) {
                        const int ja = h * Q + j, jb = M + h * Q + j;
                        st_cg16(Xs + (int64_t)(ja / P) * BLK + ((ja % P) * N + i1) * N + pp, x[j]);
                        st_cg16(Xs + (int64_t)(jb / P) * BLK + ((jb % P) * N + i1) * N + pp, x[Q + j]);
                    }
                    HK_PH_ADD(4, tA);
                }
                HK_PH_T(tP);
                publish(g);
                HK_PH_ADD(5, tP);
                ++g;
            }
        }
        if (a.prof && lane == 0) {
            atomicAdd(&a.prof[0], (unsigned long long)spin_cyc);
            atomicAdd(&a.prof[2], (unsigned long long)(clock64() - t_start));
#if HK_PROD_PHASES
            for (int k = 0; k < 6; ++k) atomicAdd(&a.prof[8 + k], (unsigned long long)ph[k]);
#endif
        }
    } else {
        // ============================ CONSUMER GROUPS ============================
        const int grp = (warp - 4) >> 2;   // = my j3 / k1 plane (P = 2)
        const unsigned bar = 2 + grp;      // named barrier of my group (128 threads)
        double2* Rv = Rvb + grp * PLANE;
#if HK_PULL_TMA64
        // my 16 rows (1 KiB each) of plane grp by bulk copies, one per lane of the
        // first half-warp, into the padded landing rows; completion on this warp's mbarrier
        const uint32_t cbar_s = smem_u32(cbar + (warp - 4));
        unsigned cph = 0;
        auto pull = [&](unsigned gs) {
            const double2* src = X + (int64_t)(gs % D) * SLOT + (int64_t)r * BLK + (int64_t)grp * N * N + 16 * rw * N;
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            asm volatile("fence.proxy.async.global;\n" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive_expect_tx(cbar_s, 16 * N * 16);
            __syncwarp();
            if (lane < 16) bulk_g2s(smem_u32(Rv + (16 * rw + lane) * ROW), src + lane * N, N * 16, cbar_s);
        };
#else
        auto pull = [&](unsigned gs) {     // my 16 rows of plane grp of slot gs
            const double2* src = X + (int64_t)(gs % D) * SLOT + (int64_t)r * BLK + (int64_t)grp * N * N + 16 * rw * N;
            const uint32_t d0 = smem_u32(Rv + 16 * rw * ROW);
#pragma unroll 4
            for (int k = 0; k < 16; ++k) {
                cp_async16(d0 + (k * ROW + lane) * 16, src + k * N + lane);
                cp_async16(d0 + (k * ROW + 32 + lane) * 16, src + k * N + 32 + lane);
            }
            cp_async_commit();
        };
#endif
        long long spin_cyc = 0;
        const long long t_start = clock64();
#if HK_PROD_PHASES
        long long ph[6] = {0, 0, 0, 0, 0, 0};
#endif
        auto issue = [&](unsigned gs) {
            if (lane == 0) spin_cyc += spin_geq(ready + gs % D, ARR * (gs / D + 1));
            __syncwarp();
            pull(gs);
        };
        auto complete = [&](unsigned gs) {
#if HK_PULL_TMA64
            mbar_wait_parity(cbar_s, cph);
            cph ^= 1;
#else
            cp_async_wait_all();
#endif
            __syncwarp();
            if (lane == 0) signal_add_relaxed(done + gs % D);
            named_bar(bar, 128);  // every warp's rows of my plane have landed
        };
        if ((int64_t)team < count) issue(0);
        for (int64_t it = team; it < count; it += nteams, ++ncell) {
            const int64_t cell = a.list ? a.list[it] : it;
            const double* fc = a.f + cell * NB;
            const unsigned gb = ncell * (1 + nfields);
            const bool more_cells = it + nteams < count;
            // ---- prologue: forward over k3 of rows (k1 = rP + grp, k2 = pp), F -> TMEM ----
            complete(gb);
            {
                const double2* row = Rv + pp * ROW;
                const int k1 = r * P + grp, k2 = pp;
                double2 v[M];
#pragma unroll
                for (int j = 0; j < Q; ++j) {
                    v[j] = row[h * Q + j];
                    v[Q + j] = row[M + h * Q + j];
                }
                fftxh_dif<M, false>(v, h);  // v[m] = F[k3 = 2m + h] (unscaled)
                const double s = 1.0 / double(NB);
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    double w8[8];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        w8[2 * i] = v[4 * c + i].x * s;
                        w8[2 * i + 1] = v[4 * c + i].y * s;
                    }
                    tmem_st16(tmF + 128 * grp + 16 * c, w8);
                }
                if (a.nyq) {
                    constexpr int H = N / 2;
                    double2* ny = a.nyq + cell * 3 * N * N;
                    if (h == 0) ny[2 * N * N + k1 * N + k2] = make_double2(s * v[H / 2].x, s * v[H / 2].y);
                    if (k2 == H) {
#pragma unroll
                        for (int m = 0; m < M; ++m)
                            ny[1 * N * N + k1 * N + 2 * m + h] = make_double2(s * v[m].x, s * v[m].y);
                    }
                    if (k1 == H) {
#pragma unroll
                        for (int m = 0; m < M; ++m) ny[k2 * N + 2 * m + h] = make_double2(s * v[m].x, s * v[m].y);
                    }
                }
                const double z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
                for (int c = 0; c < GCOLS / 16; ++c) tmem_st16(tmG + GCOLS * grp + 16 * c, z);
                tmem_wait_st();
                tmem_fence_before();
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(fbar + grp)) : "memory");
            }
            named_bar(bar, 128);  // my group's reads of the buffer are done
            issue(gb + 1);        // field 1 (needs F of both planes: the other group publishes its own)
            double mre = 0.0, n2 = 0.0, l2 = 0.0;
            for (int fi = 1; fi <= nfields; ++fi) {
                const unsigned gs = gb + fi;
                HK_PH_T(tC);
                complete(gs);
                HK_PH_ADD(0, tC);
                {  // rows i1 = pp over i2 (DIF), back in natural order
                    double2* row = Rv + pp * ROW;
                    double2 v[M];
#pragma unroll
                    for (int j = 0; j < Q; ++j) {
                        v[j] = row[h * Q + j];
                        v[Q + j] = row[M + h * Q + j];
                    }
                    fftxh_dif<M, true>(v, h);
                    __syncwarp();
#pragma unroll
                    for (int m = 0; m < M; ++m) row[2 * m + h] = v[m];
                }
                HK_PH_ADD(1, tC);
                named_bar(bar, 128);  // columns need every row
                double2 y[M];
                const double2* col = Rv + pp;
#pragma unroll
                for (int m = 0; m < M; ++m) y[m] = col[(2 * m + h) * ROW];
                named_bar(bar, 128);  // buffer free: the next field's pull overlaps the transform
                HK_PH_ADD(2, tC);
                if (fi < nfields || more_cells) issue(gs + 1);
                HK_PH_ADD(3, tC);
                fftxh_dit<M, true>(y, h);  // y[j] = node hQ + j, y[Q + j] = node M + hQ + j
                HK_PH_ADD(4, tC);
                const int j3 = r * P + grp;
                if (fi < nfields) {
                    const double mu = (fi == 1) ? a.mult0 : 1.0;
                    uint32_t g0[32], g1[32];
                    tmem_ld32_nowait(tmG + GCOLS * grp, g0);
                    tmem_ld32_nowait(tmG + GCOLS * grp + 32, g1);
                    tmem_wait_ld();
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        double gv[8];
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const int k = 16 * (c & 1) + 2 * i;
                            const double old = (c < 2) ? tmem_pair(g0[k], g0[k + 1]) : tmem_pair(g1[k], g1[k + 1]);
                            gv[i] = old + mu * (y[8 * c + i].x * y[8 * c + i].y);
                        }
                        tmem_st16(tmG + GCOLS * grp + 16 * c, gv);
                    }
                    tmem_wait_st();
                } else {  // loss field: Q = jac (w gain - f loss) at (j1, pp, j3)
                    double* qc = a.q + cell * NB;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        double gv[8];
                        tmem_ld16(tmG + GCOLS * grp + 16 * c, gv);
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const int jj = 8 * c + i;
                            const int j1 = jj < Q ? h * Q + jj : M + h * Q + (jj - Q);
                            const int64_t gi = ((int64_t)j1 * N + pp) * N + j3;
                            const double lt = __ldg(fc + gi) * y[jj].x;
                            const double qre = a.jac * (a.w * gv[i] - lt);
                            qc[gi] = qre;
                            mre = fmax(mre, fabs(qre));
                            n2 += qre * qre;
                            l2 += lt * lt;
                        }
                    }
                }
                HK_PH_ADD(5, tC);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                mre = fmax(mre, __shfl_xor_sync(0xffffffffu, mre, o));
                n2 += __shfl_xor_sync(0xffffffffu, n2, o);
                l2 += __shfl_xor_sync(0xffffffffu, l2, o);
            }
            if (lane == 0 && a.st) {
                hk_cell_status* sc = a.st + cell;
                atomic_max_nonneg(&sc->max_re, mre);
                atomicAdd(&sc->q_norm2, n2);
                atomicAdd(&sc->loss_norm2, a.jac * a.jac * l2);
            }
        }
        if (a.prof && lane == 0) {
            atomicAdd(&a.prof[1], (unsigned long long)spin_cyc);
            atomicAdd(&a.prof[3], (unsigned long long)(clock64() - t_start));
#if HK_PROD_PHASES
            for (int k = 0; k < 6; ++k) atomicAdd(&a.prof[16 + k], (unsigned long long)ph[k]);
#endif
        }
    }
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    if (warp == 0) tmem_dealloc(*tslot, G::TM_COLS);
}

size_t coll64_xchg_bytes(hk_ctx ctx) {
    const int teams = ctx->sm_count / Geo64::C;
    return size_t(teams > 0 ? teams : 1) * Geo64::XCHG_PER_TEAM;
}

int launch_coll64(hk_ctx ctx, const CollArgs& args_in, bool exact, int64_t max_cells, int tag) {
    using G = Geo64;
    // FAST: the 12-warp kernel; EXACT: the 8-warp two-transform kernel.  (The
    // 8-warp FAST kernel was measured slower and is not launched.)
    auto kern = exact ? coll64_kernel<true> : coll64_w12_kernel;
    const int nthreads = exact ? 256 : 384;
    const int key = 6400 + (exact ? 1 : 2);
    int st;
    if (!ctx->max_clusters.count(key)) {
        if ((st = check_cuda(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM),
                             "smem attribute")))
            return st;
        int per_sm = 0;
        if ((st = check_cuda(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nthreads, G::SMEM), "occupancy")))
            return st;
        const int teams = per_sm >= 1 ? ctx->sm_count / G::C : 0;
        if (teams < 1) return fail(ctx, HK_CUDA, "N = 64 collision kernel cannot be resident");
        ctx->max_clusters[key] = teams;
    }
    int64_t teams = ctx->max_clusters[key];
    if (max_cells < teams) teams = max_cells;
    if (teams < 1) return HK_OK;
    CollArgs args = args_in;
    args.in_ready = nullptr;
    args.out_done = nullptr;
    if ((st = check_cuda(ctx, cudaMemsetAsync(args.team_ctr, 0, sizeof(unsigned) * 2 * G::D * teams, ctx->stream),
                         "team counters")))
        return st;
    static unsigned long long* prof = nullptr;
#if HK_PROFILING
    const bool profiling = !exact && getenv("HK_PROF_SPIN") != nullptr;  // profiling builds only
#else
    const bool profiling = false;
#endif
    if (profiling) {
        if (!prof) cudaMalloc(&prof, 256);
        cudaMemsetAsync(prof, 0, 256, ctx->stream);
        args.prof = prof;
    }
    void* params[] = {&args};
    timing_begin(ctx, tag);
    st = check_cuda(ctx, cudaLaunchCooperativeKernel((const void*)kern, dim3(unsigned(teams * G::C)), dim3(nthreads), params,
                                                     G::SMEM, ctx->stream),
                    "N = 64 collision kernel launch");
    timing_end(ctx);
    ctx->launches++;
    if (profiling) {
        unsigned long long h[32];
        cudaMemcpyAsync(h, prof, sizeof h, cudaMemcpyDeviceToHost, ctx->stream);
        cudaStreamSynchronize(ctx->stream);
        fprintf(stderr, "[hk prof] coll64 CTAs %lld: producer spin %.1f%%, consumer spin %.1f%%\n", (long long)(teams * G::C),
                100.0 * h[0] / (double)h[2], 100.0 * h[1] / (double)h[3]);
#if HK_PROD_PHASES
        fprintf(stderr, "[hk prof] producer phases (%% of producer time): ld+wait %.1f mul %.1f fft %.1f acquire %.1f "
                "store %.1f publish %.1f\n", 100.0 * h[8] / h[2], 100.0 * h[9] / h[2], 100.0 * h[10] / h[2],
                100.0 * h[11] / h[2], 100.0 * h[12] / h[2], 100.0 * h[13] / h[2]);
        fprintf(stderr, "[hk prof] consumer phases (%% of consumer time): complete %.1f rowfft %.1f colread %.1f "
                "issue %.1f colfft %.1f gain %.1f\n", 100.0 * h[16] / h[3], 100.0 * h[17] / h[3], 100.0 * h[18] / h[3],
                100.0 * h[19] / h[3], 100.0 * h[20] / h[3], 100.0 * h[21] / h[3]);
#endif
    }
    return st;
}

}  // namespace hk
