// hk_common.cuh — shared device helpers for the hykin B200 collision path.
//
// Register-resident complex FFTs (one pencil per thread, fully unrolled so
// every index is a compile-time constant and the pencil lives in registers),
// complex arithmetic on double2, and cluster/DSMEM helpers.  fp64 only: the
// reference path is double precision end to end (inc/spectral.hpp:15-33).
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#ifndef HK_PROFILING
#define HK_PROFILING 0  // 1: HK_PROF_SPIN / HK_HYB_PROF reports (profiling builds only)
#endif

namespace hk {

namespace cg = cooperative_groups;

// e^{-2 pi i k / 64}, k = 0..31, correctly rounded (generated with 50-digit
// arithmetic).  Radix-2 stages of an N-point transform (N | 64) index it with
// stride 64/N.
__device__ __constant__ double2 c_tw64[32] = {
    {1.0, 0.0},
    {0.9951847266721969, -0.0980171403295606},
    {0.9807852804032304, -0.19509032201612828},
    {0.9569403357322088, -0.2902846772544624},
    {0.9238795325112867, -0.3826834323650898},
    {0.881921264348355, -0.47139673682599764},
    {0.8314696123025452, -0.5555702330196022},
    {0.773010453362737, -0.6343932841636455},
    {0.7071067811865476, -0.7071067811865476},
    {0.6343932841636455, -0.773010453362737},
    {0.5555702330196022, -0.8314696123025452},
    {0.47139673682599764, -0.881921264348355},
    {0.3826834323650898, -0.9238795325112867},
    {0.2902846772544624, -0.9569403357322088},
    {0.19509032201612828, -0.9807852804032304},
    {0.0980171403295606, -0.9951847266721969},
    {0.0, -1.0},
    {-0.0980171403295606, -0.9951847266721969},
    {-0.19509032201612828, -0.9807852804032304},
    {-0.2902846772544624, -0.9569403357322088},
    {-0.3826834323650898, -0.9238795325112867},
    {-0.47139673682599764, -0.881921264348355},
    {-0.5555702330196022, -0.8314696123025452},
    {-0.6343932841636455, -0.773010453362737},
    {-0.7071067811865476, -0.7071067811865476},
    {-0.773010453362737, -0.6343932841636455},
    {-0.8314696123025452, -0.5555702330196022},
    {-0.881921264348355, -0.47139673682599764},
    {-0.9238795325112867, -0.3826834323650898},
    {-0.9569403357322088, -0.2902846772544624},
    {-0.9807852804032304, -0.19509032201612828},
    {-0.9951847266721969, -0.0980171403295606}};

__host__ __device__ constexpr int ilog2c(int n) { return n <= 1 ? 0 : 1 + ilog2c(n >> 1); }

template <int N>
__host__ __device__ constexpr int bitrev(int i) {
    int r = 0;
    for (int b = 0; b < ilog2c(N); ++b) r |= ((i >> b) & 1) << (ilog2c(N) - 1 - b);
    return r;
}

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// d * w_N^{k} with w = e^{-2 pi i / N} (forward) or its conjugate (inverse).
// k is a compile-time constant after unrolling; trivial twiddles fold away.
template <int N, bool INV>
__device__ __forceinline__ double2 twiddle(double2 d, int k) {
    if (k == 0) return d;
    if (4 * k == N) {  // w^{N/4} = -i (forward) / +i (inverse)
        return INV ? make_double2(-d.y, d.x) : make_double2(d.y, -d.x);
    }
    double2 w = c_tw64[k * (64 / N)];
    if (INV) w.y = -w.y;
    return cmul(d, w);
}

// In-register radix-2 decimation-in-frequency transform of N complex values,
// natural order in and out (the bit-reversal is a compile-time renaming).
// Unnormalised: forward = sum x_j e^{-2 pi i jk/N} (FFTW_FORWARD), inverse
// = sum x_j e^{+2 pi i jk/N} (FFTW_BACKWARD), as used by src/fft.cpp:49-81.
template <int N, bool INV>
__device__ __forceinline__ void fft_reg(double2 (&x)[N]) {
#pragma unroll
    for (int len = N; len >= 2; len >>= 1) {
        const int half = len >> 1;
#pragma unroll
        for (int i = 0; i < N; i += len) {
#pragma unroll
            for (int j = 0; j < half; ++j) {
                const double2 a = x[i + j], b = x[i + j + half];
                x[i + j] = cadd(a, b);
                x[i + j + half] = twiddle<N, INV>(csub(a, b), j * (N / len));
            }
        }
    }
    double2 y[N];
#pragma unroll
    for (int i = 0; i < N; ++i) y[bitrev<N>(i)] = x[i];
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = y[i];
}

// Same transform, radix-2 decimation in time with FMA butterflies: the
// twiddled butterfly (a + w b, a - w b) is o0 = fma(w, b, a) in 4 DFMA and
// o1 = 2a - o0 in 2 DFMA (6 fp64 instructions instead of 4 DADD + 2 DMUL +
// 2 DFMA); trivial twiddles (1, -+i) stay 4 DADD.  456 -> 388 fp64
// instructions per 32-point pencil.  Bit-reversed renaming on input.
template <int N, int LEN, bool INV>
__device__ __forceinline__ void fft_fma_stage(double2 (&y)[N]) {
    constexpr int HALF = LEN / 2;
#pragma unroll
    for (int i = 0; i < N; i += LEN) {
#pragma unroll
        for (int j = 0; j < HALF; ++j) {
            const int k = j * (N / LEN);
            const double2 a = y[i + j], b = y[i + j + HALF];
            if (k == 0) {
                y[i + j] = cadd(a, b);
                y[i + j + HALF] = csub(a, b);
            } else if (4 * k == N) {  // w = -i (forward) / +i (inverse)
                const double2 t = INV ? make_double2(-b.y, b.x) : make_double2(b.y, -b.x);
                y[i + j] = cadd(a, t);
                y[i + j + HALF] = csub(a, t);
            } else {
                // constant-bank twiddle operands; the conjugate (INV) flips register signs only
                const double2 w = c_tw64[k * (64 / N)];
                const double by = INV ? b.y : -b.y, bx = INV ? -b.x : b.x;
                const double2 o0 = make_double2(__fma_rn(w.x, b.x, __fma_rn(w.y, by, a.x)),
                                                __fma_rn(w.x, b.y, __fma_rn(w.y, bx, a.y)));
                y[i + j] = o0;
                y[i + j + HALF] = make_double2(__fma_rn(2.0, a.x, -o0.x), __fma_rn(2.0, a.y, -o0.y));
            }
        }
    }
    if constexpr (LEN < N) fft_fma_stage<N, 2 * LEN, INV>(y);
}

template <int N, bool INV>
__device__ __forceinline__ void fft_fma(double2 (&x)[N]) {
    double2 y[N];
#pragma unroll
    for (int i = 0; i < N; ++i) y[i] = x[bitrev<N>(i)];
    fft_fma_stage<N, 2, INV>(y);
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = y[i];
}

// Cluster barrier split into arrive (release) / wait (acquire) so that
// independent work can run between the two (PTX barrier.cluster).
__device__ __forceinline__ void cluster_arrive() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cluster_id_x() {
    unsigned r;
    asm volatile("mov.u32 %0, %%clusterid.x;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned n_clusters_x() {
    unsigned r;
    asm volatile("mov.u32 %0, %%nclusterid.x;\n" : "=r"(r));
    return r;
}

// Address of `p` (a pointer into this CTA's shared memory) in the shared
// memory of cluster rank `rank`, as a generic pointer (DSMEM window).
template <typename T>
__device__ __forceinline__ T* dsmem_ptr(T* p, unsigned rank) {
    return cg::this_cluster().map_shared_rank(p, rank);
}

// 32-bit shared::cluster address of `p` (this CTA's shared memory) in the
// shared window of cluster rank `rank`; stores through it are DSMEM stores.
__device__ __forceinline__ uint32_t dsmem_addr(const void* p, unsigned rank) {
    const uint32_t local = static_cast<uint32_t>(__cvta_generic_to_shared(p));
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(remote) : "r"(local), "r"(rank));
    return remote;
}
__device__ __forceinline__ void st_dsmem(uint32_t addr, double2 v) {
    asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};\n" ::"r"(addr), "d"(v.x), "d"(v.y) : "memory");
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// Remote (DSMEM) address of a local shared-memory address in cluster rank `rank`.
__device__ __forceinline__ uint32_t mapa_u32(uint32_t local, unsigned rank) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(remote) : "r"(local), "r"(rank));
    return remote;
}
// Asynchronous 16-byte store into a peer CTA's shared memory that completes
// `bytes` on the peer's mbarrier (no fence, no generic-proxy membar).
__device__ __forceinline__ void st_async16(uint32_t remote_addr, double2 v, uint32_t remote_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];\n" ::"r"(remote_addr),
                 "l"(__double_as_longlong(v.x)), "l"(__double_as_longlong(v.y)), "r"(remote_bar)
                 : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
// Local arrive that also raises the expected transaction bytes of the phase.
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
// 1-D bulk copy global -> this CTA's shared memory (TMA engine), completion
// counted on `bar` in bytes (pair with mbar_arrive_expect_tx).  16-byte
// aligned addresses, size a multiple of 16.
__device__ __forceinline__ void bulk_g2s(uint32_t smem_dst, const void* gsrc, unsigned bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_dst),
                 "l"(gsrc), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint32_t bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// Cluster barrier arrive without release semantics: used only to signal
// "my shared buffers may be overwritten" after a __syncthreads.
__device__ __forceinline__ void cluster_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
}

// 16-byte global -> shared async copy through L2 only (cp.async.cg, LDGSTS).
__device__ __forceinline__ void cp_async16(uint32_t smem_dst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_dst), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
// With an L2 eviction-priority policy (createpolicy).
__device__ __forceinline__ void cp_async16_hint(uint32_t smem_dst, const void* gsrc, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(smem_dst), "l"(gsrc), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
__device__ __forceinline__ void st_cg16_hint(double2* p, double2 v, uint64_t pol) {
    asm volatile("st.global.cg.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol)
                 : "memory");
}
// 8-byte variant (cp.async.ca: sizes below 16 B go through L1).
__device__ __forceinline__ void cp_async8(uint32_t smem_dst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_dst), "l"(gsrc) : "memory");
}
// L2-only 16-byte store (skip L1: the consumer is another SM).
__device__ __forceinline__ void st_cg16(double2* p, double2 v) {
    asm volatile("st.global.cg.v2.f64 [%0], {%1, %2};\n" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
// L2-only 16-byte load (the producer is another SM of the cluster).
__device__ __forceinline__ double2 ld_cg16(const double2* p) {
    double2 v;
    asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
    return v;
}

// Named barrier over `count` threads (role groups of a warp-specialised CTA).
__device__ __forceinline__ void named_bar(unsigned id, unsigned count) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Spin until *p >= target (acquire, GPU scope).  Polls with relaxed loads (no
// L1 invalidation per iteration) and an exponential __nanosleep backoff
// (HK_SPIN_NS0 doubling up to HK_SPIN_NSMAX): a waiting warp shares its
// scheduler with the warps it waits for, so every poll it does not issue is an
// issue slot for them.  One acquire load once the target is reached.  Traps
// instead of hanging if the producer never arrives (~2^24 polls, seconds).
#ifndef HK_SPIN_NS0
#define HK_SPIN_NS0 32
#endif
#ifndef HK_SPIN_NSMAX
#define HK_SPIN_NSMAX 256
#endif
__device__ __forceinline__ long long spin_geq(const unsigned* p, unsigned target) {
    const long long t0 = clock64();
    unsigned v;
    unsigned ns = HK_SPIN_NS0, polls = 0;
    for (;;) {
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
        if ((int)(v - target) >= 0) break;
        if (++polls > (1u << 24)) __trap();
        __nanosleep(ns);
        ns = ns < HK_SPIN_NSMAX ? 2 * ns : ns;
    }
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return clock64() - t0;
}
// WAR-only signal ("I have finished reading"): the reads it orders are
// already complete (cp.async.wait_group), so no fence is issued.
__device__ __forceinline__ void signal_add_relaxed(unsigned* p) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;\n" ::"l"(p) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_group0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
// RAW signal ("my stores are visible"): release at GPU scope.
__device__ __forceinline__ void signal_add(unsigned* p) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(p) : "memory");
}

// Non-negative double max via its ordered bit pattern.
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
    atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

}  // namespace hk

// ---------------------------------------------------------------------------
// Tensor memory (TMEM) as per-thread spill-free storage.  A CTA allocates a
// power-of-two number of columns; warp w (of the first four) owns lanes
// [32 (w % 4), 32 (w % 4) + 32), so thread t < 128 owns lane t.  Each thread
// only touches its own lane, so only the per-thread tcgen05.wait fences are
// needed (no cross-thread TMEM traffic).
// ---------------------------------------------------------------------------
namespace hk {

__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {  // one full warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(slot)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {  // same warp
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// 16 x 32-bit columns of this thread's lane <-> 8 doubles.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, double (&v)[8]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
    tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __hiloint2double((int)r[2 * i + 1], (int)r[2 * i]);
}
// 32 x 32-bit columns of this thread's lane, NO wait (issue several, then
// one tmem_wait_ld()); raw words, pair them with tmem_pair().
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ double tmem_pair(uint32_t lo, uint32_t hi) { return __hiloint2double((int)hi, (int)lo); }

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const double (&v)[8]) {
    uint32_t r[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        r[2 * i] = (uint32_t)__double2loint(v[i]);
        r[2 * i + 1] = (uint32_t)__double2hiint(v[i]);
    }
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

}  // namespace hk

// ---------------------------------------------------------------------------
// Split-pencil transforms: one pencil over the lane pair (l, l ^ 16), h = (lane
// >> 4) & 1 selects the half.  Unnormalised, forward = e^{-2 pi i}, INV =
// e^{+2 pi i}, like fft_reg.
// ---------------------------------------------------------------------------
namespace hk {

#ifndef HK_FFTXH_INNER
#define HK_FFTXH_INNER fft_fma  // per-half transform of the split pencils (fft_reg: DIF, no FMA butterflies)
#endif

__device__ __forceinline__ double2 shfl_xor16(double2 v) {
    return make_double2(__shfl_xor_sync(0xffffffffu, v.x, 16), __shfl_xor_sync(0xffffffffu, v.y, 16));
}

// Generic split-pencil transforms of length L = 2M over the lane pair
// (l, l ^ 16); each thread holds M values (M = 32 for the N = 64 kernels:
// 64 data registers pairs instead of 128).  Same contracts as fftx2_*, with
// 8 -> M/2 and 16 -> M:
//   fftxh_dit: in  v[m] = x[2m + h]                 out v[j] = X[hM/2 + j], v[M/2 + j] = X[M + hM/2 + j]
//   fftxh_dif: in  v[j] = x[hM/2 + j], v[M/2 + j] = x[M + hM/2 + j]    out v[m] = X[2m + h]
template <int M, bool INV>
__device__ __forceinline__ void fftxh_dit(double2 (&v)[M], int h) {
    constexpr int L = 2 * M, Q = M / 2;
    static_assert(64 % L == 0, "twiddle table covers L | 64");
    HK_FFTXH_INNER<M, INV>(v);  // E[k] (h = 0) or O[k] (h = 1)
    if (h) {
#pragma unroll
        for (int k = 1; k < M; ++k) {
            double2 w = c_tw64[k * (64 / L)];  // e^{-2 pi i k / L}
            if (INV) w.y = -w.y;
            v[k] = cmul(v[k], w);
        }
    }
#pragma unroll
    for (int j = 0; j < Q; ++j) {
        const double2 send = h ? v[j] : v[Q + j];  // h=0 sends E[Q+j], h=1 sends T[j]
        const double2 r = shfl_xor16(send);
        const double2 a = h ? r : v[j];            // E[hQ + j]
        const double2 b = h ? v[Q + j] : r;        // T[hQ + j]
        v[j] = cadd(a, b);                         // X[hQ + j]
        v[Q + j] = csub(a, b);                     // X[M + hQ + j]
    }
}

template <int M, bool INV>
__device__ __forceinline__ void fftxh_dif(double2 (&v)[M], int h) {
    constexpr int L = 2 * M, Q = M / 2;
    static_assert(64 % L == 0, "twiddle table covers L | 64");
#pragma unroll
    for (int j = 0; j < Q; ++j) {
        const double2 a = cadd(v[j], v[Q + j]);  // n = hQ + j
        double2 w = h ? c_tw64[(Q + j) * (64 / L)] : c_tw64[j * (64 / L)];
        if (INV) w.y = -w.y;
        const double2 b = cmul(csub(v[j], v[Q + j]), w);
        const double2 send = h ? a : b;  // h=0 sends b (n = j), h=1 sends a (n = Q + j)
        const double2 r = shfl_xor16(send);
        v[j] = h ? r : a;       // h=0: a[j];        h=1: b[j] (from h=0)
        v[Q + j] = h ? b : r;   // h=0: a[Q+j] (h=1); h=1: own b[Q+j]
    }
    HK_FFTXH_INNER<M, INV>(v);  // v[m] = X[2m + h]
}

}  // namespace hk
