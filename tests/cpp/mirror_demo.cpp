// Reference-style caller of every mirrored signature of include/hykin_b200.hpp
// (SURVEY §8(b)): reads the inputs tests/test_cpp_mirror.py wrote into <dir>
// as raw little-endian doubles, calls the hykin-style functions exactly as the
// reference's callers would (spans, Moments, DistributionField, ImexTableau,
// exceptions) and writes every result back as raw doubles for the test to
// compare with the golden fixtures / the oracle.
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "hykin_b200.hpp"

namespace hk = hykin_b200;
static std::string dir;

static std::vector<double> load(const std::string& name, size_t count) {
    std::vector<double> v(count);
    std::ifstream in(dir + "/" + name, std::ios::binary);
    in.read(reinterpret_cast<char*>(v.data()), std::streamsize(count * sizeof(double)));
    if (!in) throw std::runtime_error("cannot read " + name);
    return v;
}
static void save(const std::string& name, const std::vector<double>& v) {
    std::ofstream out(dir + "/" + name, std::ios::binary);
    out.write(reinterpret_cast<const char*>(v.data()), std::streamsize(v.size() * sizeof(double)));
}
template <typename T>
static void append(std::vector<double>& v, const T& span) {
    v.insert(v.end(), span.begin(), span.end());
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    dir = argv[1];
    const auto par = load("params.bin", 16);
    const double vmax = par[0], r_phys = par[1];
    const int a1 = int(par[2]), a2 = int(par[3]);

    // ---- collision + residual (N = 16, config-1 shapes): reference throw semantics ----
    {
        const int n = 16, nb = n * n * n, cells = 4;
        const auto f = load("coll_f.bin", size_t(cells) * nb);
        const hk::VelocityGrid vg = hk::make_velocity_grid(n, vmax);
        const hk::SpectralKernel kern = hk::precompute_kernel(vg, n, a1, a2, r_phys);
        std::vector<double> q, res, threw;
        for (int c = 0; c < cells; ++c) {
            std::span<const double> fc(f.data() + size_t(c) * nb, nb);
            std::vector<double> qc(nb), rc(nb);
            double t = 0.0;
            try {
                hk::spectral_collision(fc, kern, qc);
            } catch (const hk::numerical_consistency_error&) {
                t += 1.0;
            }
            try {
                hk::penalized_residual(fc, kern, vg, hk::PenalizationRule{}, rc);
            } catch (const hk::numerical_consistency_error&) {
                t += 2.0;
            }
            append(q, qc);
            append(res, rc);
            threw.push_back(t);
        }
        save("out_coll_q.bin", q);
        save("out_coll_res.bin", res);
        save("out_coll_threw.bin", threw);
    }
    // ---- moments family + stage solves (N = 16, config-3 shapes) ----
    {
        const int n = 16, nb = n * n * n, cells = 4;
        const auto f = load("mom_f.bin", size_t(cells) * nb);
        const auto sp = load("mom_params.bin", 4);  // a, eps, beta, nu_coeff
        const hk::VelocityGrid vg = hk::make_velocity_grid(n, vmax);
        std::vector<double> mom, real, l1, sigma, maxw, gauss, fb, matched, removed, esbgk, esfb, pen;
        for (int c = 0; c < cells; ++c) {
            std::span<const double> fc(f.data() + size_t(c) * nb, nb);
            const hk::Moments m = hk::moments_of(fc, vg);
            mom.insert(mom.end(), {m.rho, m.u(0), m.u(1), m.u(2), m.T});
            const hk::RealizabilityMatrix rm = hk::realizability_matrix(fc, vg, m);
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) real.push_back(rm.a_bar(i, j));
            real.insert(real.end(), {rm.b_bar(0), rm.b_bar(1), rm.b_bar(2), rm.c_bar});
            l1.push_back(hk::l1_distance_to_maxwellian(fc, vg));
            const hk::Matrix3 s = hk::second_moment(fc, vg);
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) sigma.push_back(s(i, j));
            append(maxw, hk::maxwellian(m, vg));
            std::vector<double> g(nb);
            bool fell = false;
            hk::anisotropic_gaussian(m, hk::stress_tensor(fc, vg, m), -0.5, vg, g, &fell);
            append(gauss, g);
            fb.push_back(fell ? 1.0 : 0.0);
            hk::match_moments(g, vg, m.rho, hk::Vector3(m.rho * m.u(0), m.rho * m.u(1), m.rho * m.u(2)), m.energy());
            append(matched, g);
            std::vector<double> qd(nb);
            for (int k = 0; k < nb; ++k) qd[k] = fc[k] - g[k];
            hk::remove_invariant_moments(qd, g, vg, m.u);
            append(removed, qd);
            std::vector<double> out(nb);
            const hk::EsbgkStageInfo info =
                hk::esbgk_stage_solve(fc, sp[0], sp[1], hk::EsbgkParams{sp[2], sp[3], 1e-6}, vg, out);
            append(esbgk, out);
            esfb.push_back(info.gaussian_fallback ? 1.0 : 0.0);
            hk::penalized_stage_solve(fc, sp[0], sp[1], hk::PenalizationRule{}, vg, out);
            append(pen, out);
        }
        save("out_mom.bin", mom);
        save("out_real.bin", real);
        save("out_l1.bin", l1);
        save("out_sigma.bin", sigma);
        save("out_maxw.bin", maxw);
        save("out_gauss.bin", gauss);
        save("out_gauss_fb.bin", fb);
        save("out_matched.bin", matched);
        save("out_removed.bin", removed);
        save("out_esbgk.bin", esbgk);
        save("out_esbgk_fb.bin", esfb);
        save("out_pen.bin", pen);
    }
    // ---- transport + PR(2,2,2) steps on a DistributionField (N = 8 torus) ----
    {
        const auto tp = load("tr_params.bin", 6);  // nx, ny, dx, dy, dt, n
        const int nx = int(tp[0]), ny = int(tp[1]), n = int(tp[5]), nb = n * n * n, cells = nx * ny;
        const double dx = tp[2], dy = tp[3], dt = tp[4];
        const auto f = load("tr_f.bin", size_t(cells) * nb);
        const auto eps = load("tr_eps.bin", cells);
        const hk::VelocityGrid vg = hk::make_velocity_grid(n, vmax);
        hk::DistributionField field(cells, nb), out;
        for (int c = 0; c < cells; ++c) std::copy(f.begin() + size_t(c) * nb, f.begin() + size_t(c + 1) * nb, field.ensure(c).begin());
        hk::kinetic_transport_rhs_periodic(field, nx, ny, vg, dx, dy, out);
        std::vector<double> rhs;
        for (int c = 0; c < cells; ++c) append(rhs, out[c]);
        save("out_tr_rhs.bin", rhs);
        // one cell from its stencils: (i, j) = (1, 2)
        const int i = 1, j = 2;
        std::array<const double*, 5> fxs, fys;
        for (int k = 0; k < 5; ++k) {
            fxs[k] = field[j * nx + ((i + k - 2 + nx) % nx)].data();
            fys[k] = field[((j + k - 2 + ny) % ny) * nx + i].data();
        }
        std::vector<double> cell(nb);
        hk::kinetic_transport_rhs_cell(fxs, fys, vg, dx, dy, 1e-6, cell.data());
        save("out_tr_cell.bin", cell);
        hk::DistributionField es = field, pb = field;
        hk::esbgk_imex_step(es, nx, ny, vg, dx, dy, dt, eps, hk::ImexTableau::pr222(), hk::EsbgkParams{});
        std::vector<double> v;
        for (int c = 0; c < cells; ++c) append(v, es[c]);
        save("out_esbgk_step.bin", v);
        (void)pb;
    }
    // ---- penalized PR(2,2,2) step on a DistributionField (N = 16, 4 x 3 torus) ----
    {
        const int n = 16, nb = n * n * n, nx = 4, ny = 3, cells = nx * ny;
        const auto f = load("pen_f.bin", size_t(cells) * nb);
        const auto eps = load("pen_eps.bin", cells);
        const hk::VelocityGrid vg = hk::make_velocity_grid(n, vmax);
        hk::DistributionField pb(cells, nb);
        for (int c = 0; c < cells; ++c) std::copy(f.begin() + size_t(c) * nb, f.begin() + size_t(c + 1) * nb, pb.ensure(c).begin());
        const hk::SpectralKernel kern = hk::precompute_kernel(vg, n, 2, 4, r_phys);
        hk::penalized_imex_step(pb, nx, ny, vg, kern, 0.25, 1.0 / 3.0, 1e-3, eps, hk::ImexTableau::pr222(),
                                hk::BoltzmannParams{});
        std::vector<double> v;
        for (int c = 0; c < cells; ++c) append(v, pb[c]);
        save("out_pen_step.bin", v);
        hk::ImexTableau bad = hk::ImexTableau::pr222();
        bad.a_im[1][1] = 0.5;
        double rejected = 0.0;
        try {
            hk::penalized_imex_step(pb, nx, ny, vg, kern, 0.25, 1.0 / 3.0, 1e-3, eps, bad, hk::BoltzmannParams{});
        } catch (const hk::contract_violation&) {
            rejected = 1.0;
        }
        save("out_tableau_rejected.bin", {rejected});
    }
    // ---- indicators + Algorithm 1 ----
    {
        const auto pr = load("ind_prim.bin", 20 + 3);  // 5 x (rho, ux, uy, T), dx, dy, eps
        auto pm = [&](int k) { return hk::PrimMoments{pr[4 * k], pr[4 * k + 1], pr[4 * k + 2], pr[4 * k + 3]}; };
        const hk::DerivativeBundle d = hk::spatial_derivatives(pm(0), pm(1), pm(2), pm(3), pm(4), pr[20], pr[21]);
        const hk::Eigenvalues lam = hk::v_eps1_eigenvalues(d, pm(0), pr[22], hk::TransportCoefficients{});
        save("out_ind.bin", {lam.a, lam.b, lam.c, hk::lambda_b_indicator(d, pm(0), pr[22])});
        const auto rows = load("regime_rows.bin", 256 * 8);  // r, has_lam, la, lb, lc, lambda_b (nan = none), l1 (nan = none), pad
        const hk::Thresholds th{1e-3, 1e-2, 1e-3};
        std::vector<double> res;
        for (int k = 0; k < 256; ++k) {
            const double* w = rows.data() + 8 * k;
            hk::IndicatorSet ind;
            if (w[1] != 0.0) ind.eigenvalues = hk::Eigenvalues{w[2], w[3], w[4]};
            if (w[5] == w[5]) ind.lambda_b = w[5];
            if (w[6] == w[6]) ind.l1_distance = w[6];
            try {
                res.push_back(hk::regime_update(int(w[0]), ind, th));
            } catch (const hk::contract_violation&) {
                res.push_back(-1.0);
            }
        }
        save("out_regime.bin", res);
    }
    std::printf("mirror_demo: done\n");
    return 0;
}
