// Skeleton of a cluster-resident stage solve (feasibility probe, not product
// code): a cell of n^3 doubles is split by k1 planes over a CL-CTA cluster,
// each CTA pulls its slice into shared memory by TMA bulk copies, reduces it
// (CTA + cluster through DSMEM), rescales it in place and writes it back by
// TMA bulk stores.  HBM traffic is exactly one read + one write of the field.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 stage_skel.cu -o stage_skel
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, unsigned bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_wait(uint32_t bar, unsigned parity) {
    asm volatile(
        "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ unsigned cl_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cl_id() {
    unsigned r;
    asm volatile("mov.u32 %0, %%clusterid.x;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cl_n() {
    unsigned r;
    asm volatile("mov.u32 %0, %%nclusterid.x;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ double ld_dsmem(const double* p, unsigned rank) {
    uint32_t a = smem_u32(p), r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];\n" : "=d"(v) : "r"(r) : "memory");
    return v;
}

template <int CL, int NT>
__global__ void __launch_bounds__(NT) skel(const double* __restrict__ f, double* __restrict__ out, int64_t ncells, int n) {
    extern __shared__ __align__(128) double sm[];
    const int nb = n * n * n, slice = nb / CL, plane = n * n;
    double* buf = sm;
    double* part = sm + slice;  // [2] partial sums (double-buffered by cell parity)
    __shared__ __align__(8) uint64_t bar;
    __shared__ double red[NT / 32];
    const int t = threadIdx.x;
    const unsigned r = cl_rank();
    if (t == 0) {
        mbar_init(smem_u32(&bar), 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    unsigned phase = 0;
    int it = 0;
    for (int64_t cell = cl_id(); cell < ncells; cell += cl_n(), ++it) {
        const double* src = f + cell * nb + (int64_t)r * slice;
        double* dst = out + cell * nb + (int64_t)r * slice;
        if (t == 0) {
            bulk_wait_read0();  // the previous cell's stores have read the buffer
            mbar_arrive_expect_tx(smem_u32(&bar), slice * 8);
            for (int p = 0; p < slice / plane; ++p)
                bulk_g2s(smem_u32(buf + p * plane), src + p * plane, plane * 8, smem_u32(&bar));
        }
        mbar_wait(smem_u32(&bar), phase);
        phase ^= 1;
        double s = 0.0;
        for (int i = 2 * t; i < slice; i += 2 * NT) {
            const double2 v = *reinterpret_cast<const double2*>(buf + i);
            s += v.x + v.y;
        }
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if ((t & 31) == 0) red[t >> 5] = s;
        __syncthreads();
        if (t == 0) {
            double a = 0;
            for (int w = 0; w < NT / 32; ++w) a += red[w];
            part[it & 1] = a;
        }
        cl_sync();
        double tot = 0;
        for (int q = 0; q < CL; ++q) tot += ld_dsmem(part + (it & 1), q);
        const double sc = 1.0 / (1.0 + 1e-9 * tot);
        for (int i = 2 * t; i < slice; i += 2 * NT) {
            double2 v = *reinterpret_cast<double2*>(buf + i);
            v.x *= sc;
            v.y *= sc;
            *reinterpret_cast<double2*>(buf + i) = v;
        }
        fence_proxy_async();
        __syncthreads();
        if (t == 0) {
            for (int p = 0; p < slice / plane; ++p) bulk_s2g(dst + p * plane, smem_u32(buf + p * plane), plane * 8);
            bulk_commit();
        }
    }
    if (t == 0) bulk_wait0();
    cl_sync();  // no CTA leaves while a peer may still read its partials
}

template <int CL, int NT>
float run(const double* f, double* o, int64_t ncells, int n, int per_sm, int sms) {
    auto k = skel<CL, NT>;
    const size_t smem = (size_t(n) * n * n / CL + 2) * 8;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(sms * per_sm / CL * CL));
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    cudaOccupancyMaxActiveClusters(&ncl, k, &cfg);
    cfg.gridDim = dim3(unsigned(ncl * CL));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaLaunchKernelEx(&cfg, k, f, o, ncells, n);
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) cudaLaunchKernelEx(&cfg, k, f, o, ncells, n);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("CL=%d NT=%d smem=%zu KB active clusters=%d (%d CTAs): %.3f ms per pass (%s)\n", CL, NT, smem >> 10, ncl,
           ncl * CL, ms / 5, cudaGetErrorString(cudaGetLastError()));
    return ms / 5;
}

int main() {
    const int n = 32;
    const int64_t ncells = 65536, nb = int64_t(n) * n * n;
    double *f, *o;
    cudaMalloc(&f, ncells * nb * 8);
    cudaMalloc(&o, ncells * nb * 8);
    cudaMemset(f, 0, ncells * nb * 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<4, 256>(f, o, ncells, n, 3, sms);
    run<4, 128>(f, o, ncells, n, 3, sms);
    run<8, 128>(f, o, ncells, n, 6, sms);
    run<8, 256>(f, o, ncells, n, 6, sms);
    run<2, 256>(f, o, ncells, n, 1, sms);
    printf("HBM bound (1 read + 1 write of %.1f GB) at 6.54 TB/s: %.3f ms\n", 2.0 * ncells * nb * 8 / 1e9,
           2.0 * ncells * nb * 8 / 6.54e12 * 1e3);
    return 0;
}
