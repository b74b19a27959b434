// hykin_b200.hpp — header-only C++20 mirror of the reference's operator
// interfaces over the C-ABI of hykin_b200.h.
//
// Same names, argument meaning and exceptions as namespace hykin
// (/root/reference/proj/core/include/hykin): a caller swaps
//     hykin::precompute_kernel / hykin::spectral_collision / ...
// for hykin_b200::... (or `namespace hykin = hykin_b200;` for these names)
// and links libhykin_b200.so.  Host spans are copied to the device inside the
// call (the e2e path); *_device variants take device pointers.  Errors are
// thrown as the reference's exception classes (inc/errors.hpp:9-61).
#pragma once

#include <cmath>
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "hykin_b200.h"

namespace hykin_b200 {

class error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class config_error : public error {
public:
    using error::error;
};
class aliasing_config_error : public config_error {
public:
    using config_error::config_error;
};
class degenerate_state_error : public error {
public:
    using error::error;
};
class positivity_error : public error {
public:
    using error::error;
};
class contract_violation : public error {
public:
    using error::error;
};
class numerical_consistency_error : public error {
public:
    using error::error;
};
class device_error : public error {
public:
    using error::error;
};

class Context {
public:
    explicit Context(int device = 0) {
        if (hk_ctx_create(device, &ctx_) != HK_OK) throw device_error("hk_ctx_create: no usable sm_100 device");
    }
    ~Context() { hk_ctx_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    hk_ctx get() const { return ctx_; }

    void check(int st) const {
        if (st == HK_OK) return;
        char msg[512];
        int64_t cell = -1;
        hk_last_error(ctx_, &cell, msg, sizeof msg);
        std::string m = msg;
        if (cell >= 0) m += " (cell " + std::to_string(cell) + ")";
        switch (st) {
        case HK_CONFIG: throw config_error(m);
        case HK_ALIASING: throw aliasing_config_error(m);
        case HK_DEGENERATE: throw degenerate_state_error(m);
        case HK_NUMERICAL_CONSISTENCY: throw numerical_consistency_error(m);
        case HK_CONTRACT: throw contract_violation(m);
        case HK_POSITIVITY: throw positivity_error(m);
        case HK_UNSUPPORTED: throw config_error(m);
        default: throw device_error(m);
        }
    }

    static Context& instance() {
        static Context c(0);
        return c;
    }

private:
    hk_ctx ctx_ = nullptr;
};

// inc/grid.hpp:45-56
struct VelocityGrid {
    int nv = 0;
    double vmax = 0, dv1 = 0, dv2 = 0, dv3 = 0, dvk = 0;
    std::vector<double> nodes;
    int size() const { return nv * nv * nv; }
    int index(int k1, int k2, int k3) const { return (k1 * nv + k2) * nv + k3; }
    double node(int k) const { return nodes[k]; }
};

// src/grid.cpp:18-33
inline VelocityGrid make_velocity_grid(int nv, double vmax) {
    if (nv < 2) throw config_error("velocity grid needs at least 2 nodes per axis, got " + std::to_string(nv));
    if (vmax <= 0.0) throw config_error("velocity cutoff must be positive");
    VelocityGrid g;
    g.nv = nv;
    g.vmax = vmax;
    g.dv1 = g.dv2 = g.dv3 = 2.0 * vmax / nv;
    g.dvk = g.dv1 * g.dv2 * g.dv3;
    g.nodes.resize(nv);
    for (int k = 0; k < nv; ++k) g.nodes[k] = -vmax + (k + 0.5) * g.dv1;
    return g;
}

// inc/spectral.hpp:15-33 — the tables live on the device.
struct SpectralKernel {
    int n = 0, a1 = 0, a2 = 0;
    double r_phys = 0, r = 0, jacobian = 1, weight = 0;
    std::shared_ptr<hk_kernel_s> handle;
    int dirs() const { return a1 * a2; }
    int modes() const { return n * n * n; }
};

// src/spectral.cpp:53-112
inline SpectralKernel precompute_kernel(const VelocityGrid& vgrid, int n, int a1, int a2, double r_phys,
                                        Context& ctx = Context::instance()) {
    if (n != vgrid.nv)
        throw config_error("spectral mode count must match the velocity grid (" + std::to_string(n) + " vs " +
                           std::to_string(vgrid.nv) + ")");
    hk_kernel k = nullptr;
    ctx.check(hk_kernel_create(ctx.get(), n, a1, a2, vgrid.vmax, r_phys, &k));
    SpectralKernel out;
    out.n = n;
    out.a1 = a1;
    out.a2 = a2;
    double info[6];
    hk_kernel_info(k, info);
    out.r = info[0];
    out.jacobian = info[1];
    out.weight = info[2];
    out.r_phys = info[3];
    out.handle = std::shared_ptr<hk_kernel_s>(k, [](hk_kernel p) { hk_kernel_destroy(p); });
    return out;
}

// src/spectral.cpp:114-154: Q(f) for one cell, throwing numerical_consistency_error
// after writing `out` when max|Im Q| > 1e-10 max|Re Q| (reference semantics).
inline void spectral_collision(std::span<const double> f, const SpectralKernel& kernel, std::span<double> out,
                               Context& ctx = Context::instance()) {
    if ((int64_t)f.size() != kernel.modes() || out.size() != f.size())
        throw contract_violation("spectral_collision: span sizes must equal n^3");
    ctx.check(hk_collision_batch_host(ctx.get(), kernel.handle.get(), f.data(), out.data(), 1, HK_COLL_STRICT,
                                      nullptr));
}

// Batched extension: ncells contiguous blocks, default (fast + guarded) path,
// no throw on the imaginary residue (per-cell verdicts in `status`).
inline void spectral_collision_batch(std::span<const double> f, const SpectralKernel& kernel, std::span<double> out,
                                     std::span<hk_cell_status> status = {}, Context& ctx = Context::instance()) {
    const int64_t nb = kernel.modes();
    if (f.size() % nb || out.size() != f.size()) throw contract_violation("spectral_collision_batch: bad sizes");
    const int64_t ncells = f.size() / nb;
    ctx.check(hk_collision_batch_host(ctx.get(), kernel.handle.get(), f.data(), out.data(), ncells, 0,
                                      status.empty() ? nullptr : status.data()));
}

}  // namespace hykin_b200
