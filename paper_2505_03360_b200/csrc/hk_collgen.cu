// hk_collgen.cu — collision operator for any velocity resolution n outside the
// specialised team kernels (n = 16, 32, 64), sm_100a.
//
// spectral_collision (src/spectral.cpp:114-154) accepts every n (FFTW plans any
// size); this path keeps that contract on the device with the reference's
// arithmetic (two complex transforms per direction, complex gain):
//   F  = FFT(f) / n^3,  ga_d = IFFT(alpha_d F),  gb_d = IFFT(alpha'_d F),
//   L  = IFFT(loss F),  Q = Re[jac (w sum_d m_d ga_d gb_d - f L)].
// Transforms are direct DFTs along each axis (any n, prime factors included):
// one thread per output element sums its pencil (n complex MACs, the pencil
// stays in L1), twiddles e^{-+2 pi i m / n} from sincospi in a table.  Cells run
// in chunks through five complex work fields [chunk][n^3] in HBM.  This is the
// completeness path (n = 8, 12, 24, 48, ...), not the performance path.
#include <algorithm>
#include <cmath>

#include "hk_coll.cuh"
#include "hk_common.cuh"

namespace hk {
namespace {

__global__ void twiddle_kernel(int n, double2* tw_fwd, double2* tw_bwd) {
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= n) return;
    double s, c;
    sincospi(2.0 * m / n, &s, &c);
    tw_fwd[m] = make_double2(c, -s);  // FFTW_FORWARD: e^{-2 pi i m / n}
    tw_bwd[m] = make_double2(c, s);   // FFTW_BACKWARD, unnormalised
}

__global__ void load_kernel(const double* __restrict__ f, double2* __restrict__ F, int64_t count) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        F[i] = make_double2(f[i], 0.0);
}

// out[.., k, ..] = scale * sum_j in[.., j, ..] tw[(j k) mod n] along axis `ax`
// (0 = i1, stride n^2; 1 = i2, stride n; 2 = i3, stride 1) of [cells][n][n][n].
__global__ void dft_axis_kernel(const double2* __restrict__ in, double2* __restrict__ out, int64_t ncells, int n,
                                int ax, const double2* __restrict__ tw, double scale) {
    const int64_t nb = (int64_t)n * n * n, total = ncells * nb;
    const int64_t stride = ax == 0 ? (int64_t)n * n : (ax == 1 ? n : 1);
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
        const int64_t idx = o % nb;
        const int k = int((idx / stride) % n);
        const double2* p = in + (o - (int64_t)k * stride);
        double re = 0.0, im = 0.0;
        int m = 0;  // (j k) mod n, advanced incrementally
        for (int j = 0; j < n; ++j) {
            const double2 x = p[(int64_t)j * stride], w = tw[m];
            re = fma(x.x, w.x, fma(-x.y, w.y, re));
            im = fma(x.x, w.y, fma(x.y, w.x, im));
            m += k;
            if (m >= n) m -= n;
        }
        out[o] = make_double2(scale * re, scale * im);
    }
}

// out = F * w with w real in the device table layout [i1][i3][i2] (entry plane)
__global__ void weight_kernel(const double2* __restrict__ F, const double* __restrict__ w, double2* __restrict__ out,
                              int64_t ncells, int n) {
    const int64_t nb = (int64_t)n * n * n, total = ncells * nb;
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
        const int64_t idx = o % nb;
        const int i3 = int(idx % n), i2 = int((idx / n) % n), i1 = int(idx / ((int64_t)n * n));
        const double s = __ldg(w + ((int64_t)i1 * n + i3) * n + i2);
        const double2 x = F[o];
        out[o] = make_double2(x.x * s, x.y * s);
    }
}

__global__ void gain_kernel(const double2* __restrict__ ga, const double2* __restrict__ gb, double2* __restrict__ gain,
                            int64_t count, double mu) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        const double2 a = ga[i], b = gb[i];
        double2 g = gain[i];
        g.x += mu * (a.x * b.x - a.y * b.y);
        g.y += mu * (a.x * b.y + a.y * b.x);
        gain[i] = g;
    }
}

// Q = Re[jac (w gain - f L)] and the per-cell verdict (src/spectral.cpp:142-153)
__global__ void final_kernel(const double* __restrict__ f, const double2* __restrict__ gain,
                             const double2* __restrict__ loss, double* __restrict__ q, int n, double jac, double w,
                             hk_cell_status* __restrict__ st) {
    const int64_t nb = (int64_t)n * n * n;
    const int64_t c = blockIdx.y;
    double mre = 0.0, mim = 0.0, n2 = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = c * nb + i;
        const double fv = f[o];
        const double re = jac * (w * gain[o].x - fv * loss[o].x);
        const double im = jac * (w * gain[o].y - fv * loss[o].y);
        q[o] = re;
        mre = fmax(mre, fabs(re));
        mim = fmax(mim, fabs(im));
        n2 += re * re;
    }
    for (int s = 16; s > 0; s >>= 1) {
        mre = fmax(mre, __shfl_xor_sync(0xffffffffu, mre, s));
        mim = fmax(mim, __shfl_xor_sync(0xffffffffu, mim, s));
        n2 += __shfl_xor_sync(0xffffffffu, n2, s);
    }
    if ((threadIdx.x & 31) == 0) {
        atomic_max_nonneg(&st[c].max_re, mre);
        atomic_max_nonneg(&st[c].max_im, mim);
        atomicAdd(&st[c].q_norm2, n2);
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&st[c].flags, HK_CELL_EXACT);
    }
}

unsigned grid_of(hk_ctx ctx, int64_t count) {
    const int64_t b = (count + 255) / 256, cap = int64_t(ctx->sm_count) * 16;
    return unsigned(std::max<int64_t>(1, std::min(b, cap)));
}

}  // namespace

int launch_coll_generic(hk_ctx ctx, hk_kernel k, const double* f, double* q, int64_t ncells, hk_cell_status* st) {
    const int n = k->n;
    const int64_t nb = (int64_t)n * n * n;
    // chunk: five complex work fields per cell within ~1 GiB of scratch
    const int64_t per_cell = 5 * nb * (int64_t)sizeof(double2);
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(ncells, (int64_t(1) << 30) / per_cell));
    const size_t tw_bytes = 2 * sizeof(double2) * n;
    int s;
    if ((s = ensure_scratch(ctx, size_t(chunk * per_cell) + tw_bytes + 256))) return s;
    double2* base = static_cast<double2*>(ctx->scratch);
    double2 *F = base, *T1 = F + chunk * nb, *T2 = T1 + chunk * nb, *GA = T2 + chunk * nb, *G = GA + chunk * nb;
    double2 *twf = G + chunk * nb, *twb = twf + n;
    cudaStream_t sm = ctx->stream;
    twiddle_kernel<<<(n + 127) / 128, 128, 0, sm>>>(n, twf, twb);
    ctx->launches++;
    const double inv = 1.0 / double(nb);
    // out-of-place passes src -> tmp -> src -> dst (dst must differ from src)
    auto dft3 = [&](double2* src, double2* tmp, double2* dst, int64_t nc, const double2* tw, double scale) {
        const unsigned gr = grid_of(ctx, nc * nb);
        dft_axis_kernel<<<gr, 256, 0, sm>>>(src, tmp, nc, n, 2, tw, 1.0);   // i3
        dft_axis_kernel<<<gr, 256, 0, sm>>>(tmp, src, nc, n, 1, tw, 1.0);   // i2
        dft_axis_kernel<<<gr, 256, 0, sm>>>(src, dst, nc, n, 0, tw, scale); // i1
        ctx->launches += 3;
    };
    timing_begin(ctx, 0);
    for (int64_t c0 = 0; c0 < ncells; c0 += chunk) {
        const int64_t nc = std::min(chunk, ncells - c0), cnt = nc * nb;
        const unsigned gr = grid_of(ctx, cnt);
        load_kernel<<<gr, 256, 0, sm>>>(f + c0 * nb, T1, cnt);
        ctx->launches++;
        dft3(T1, T2, F, nc, twf, inv);  // F = FFT(f) / n^3 (to_spectral without the phases that cancel)
        cudaMemsetAsync(G, 0, sizeof(double2) * cnt, sm);
        for (int e = 0; e < k->md; ++e) {
            weight_kernel<<<gr, 256, 0, sm>>>(F, k->alpha + (int64_t)e * nb, T1, nc, n);
            dft3(T1, T2, GA, nc, twb, 1.0);  // ga
            weight_kernel<<<gr, 256, 0, sm>>>(F, k->alpha_p + (int64_t)e * nb, T1, nc, n);
            dft3(T1, T2, T2, nc, twb, 1.0);  // gb (passes T1 -> T2 -> T1 -> T2)
            gain_kernel<<<gr, 256, 0, sm>>>(GA, T2, G, cnt, e == 0 ? k->mult0 : 1.0);
            ctx->launches += 3;
        }
        weight_kernel<<<gr, 256, 0, sm>>>(F, k->loss, T1, nc, n);
        dft3(T1, T2, GA, nc, twb, 1.0);  // loss field
        final_kernel<<<dim3(unsigned(std::min<int64_t>(64, (nb + 255) / 256)), unsigned(nc)), 256, 0, sm>>>(
            f + c0 * nb, G, GA, q + c0 * nb, n, k->jac, k->weight, st + c0);
        ctx->launches += 2;
        if ((s = check_cuda(ctx, cudaGetLastError(), "generic collision"))) break;
    }
    timing_end(ctx);
    return s;
}

}  // namespace hk
