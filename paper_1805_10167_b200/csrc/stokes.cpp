// P1-P1-PSPG Stokes on the device engine (see stokes.hpp). Reference:
// src/solvers.cpp:466-753.
#include "stokes.hpp"

#include <cmath>
#include <cstdio>

#include "coarse.hpp"

namespace hyb {

namespace {
constexpr uint8_t kSmoothMask = INNER | NEUMANN;
constexpr uint8_t kDirichletMask = DIRICHLET;

void check_state(StokesState& s, int level, const char* what) {
    s.u1->check_level(level, what);
    s.u2->check_level(level, what);
    s.p->check_level(level, what);
}
} // namespace

std::string solve_history(const std::vector<double>& residuals, bool breakdown) {
    std::string out;
    char line[96];
    for (size_t k = 0; k < residuals.size(); ++k) {
        if (k == 0) std::snprintf(line, sizeof line, "cycle %zu residual %.6e\n", k, residuals[k]);
        else {
            const double f = residuals[k - 1] > 0.0 ? residuals[k] / residuals[k - 1] : 0.0;
            std::snprintf(line, sizeof line, "cycle %zu residual %.6e factor %.4f\n", k, residuals[k], f);
        }
        out += line;
    }
    if (breakdown) out += "breakdown\n";
    return out;
}

StokesState::StokesState(Domain& d, const std::string& name, int min_level, int max_level,
                         const BoundaryMap& bc_velocity, const BoundaryMap& bc_pressure) {
    own_[0] = std::make_unique<Function>(d, name + ".u1", min_level, max_level, bc_velocity);
    own_[1] = std::make_unique<Function>(d, name + ".u2", min_level, max_level, bc_velocity);
    own_[2] = std::make_unique<Function>(d, name + ".p", min_level, max_level, bc_pressure);
    u1 = own_[0].get();
    u2 = own_[1].get();
    p = own_[2].get();
}

// ((dot u1 + dot u2) + dot p), each the reference's bitwise dot
double stokes_dot(StokesState& a, StokesState& b, int level) {
    return dot(*a.u1, *b.u1, level) + dot(*a.u2, *b.u2, level) + dot(*a.p, *b.p, level);
}

// src/solvers.cpp:486-504
StokesSystem::StokesSystem(Domain& d, int min_level, int max_level, const BoundaryMap& bcu, const BoundaryMap& bcp)
    : a_(d, LAPLACE, min_level, max_level, bcu), gx_(d, GRAD_X, min_level, max_level, bcu),
      gy_(d, GRAD_Y, min_level, max_level, bcu), bx_(d, DIV_X, min_level, max_level, bcp),
      by_(d, DIV_Y, min_level, max_level, bcp), c_(d, PSPG, min_level, max_level, bcp),
      tmp_u_(d, "stokes.tmp_u", min_level, max_level, bcu), mom_rhs_(d, "stokes.mom_rhs", min_level, max_level, bcu),
      tmp_p_(d, "stokes.tmp_p", min_level, max_level, bcp), res_p_(d, "stokes.res_p", min_level, max_level, bcp),
      diag_c_(d, "stokes.diag_c", min_level, max_level, bcp) {
    for (int l = min_level; l <= max_level; ++l) diagonal(c_, diag_c_, l);
}

// src/solvers.cpp:506-546
void uzawa_smooth(StokesSystem& S, StokesState& rhs, StokesState& x, int level, double omega) {
    check_state(rhs, level, "uzawa_smooth");
    check_state(x, level, "uzawa_smooth");
    // momentum: one forward hybrid Gauss-Seidel sweep per component against
    // the current pressure gradient
    apply(S.gx_, *x.p, S.tmp_u_, level, kSmoothMask);
    assign(1.0, *rhs.u1, -1.0, S.tmp_u_, S.mom_rhs_, level, kSmoothMask);
    assign(1.0, *rhs.u1, 0.0, *rhs.u1, S.mom_rhs_, level, kDirichletMask);
    smooth_gs(S.a_, S.mom_rhs_, *x.u1, level);
    apply(S.gy_, *x.p, S.tmp_u_, level, kSmoothMask);
    assign(1.0, *rhs.u2, -1.0, S.tmp_u_, S.mom_rhs_, level, kSmoothMask);
    assign(1.0, *rhs.u2, 0.0, *rhs.u2, S.mom_rhs_, level, kDirichletMask);
    smooth_gs(S.a_, S.mom_rhs_, *x.u2, level);
    // pressure: damped pointwise correction by the continuity residual
    apply(S.bx_, *x.u1, S.tmp_p_, level, kSmoothMask);
    assign(1.0, *rhs.p, -1.0, S.tmp_p_, S.res_p_, level, kSmoothMask);
    apply(S.by_, *x.u2, S.tmp_p_, level, kSmoothMask);
    add_scaled(S.res_p_, -1.0, S.tmp_p_, level, kSmoothMask);
    apply(S.c_, *x.p, S.tmp_p_, level, kSmoothMask);
    add_scaled(S.res_p_, -1.0, S.tmp_p_, level, kSmoothMask);
    if (zero_diagonal_row(S.c_, *x.p, level)) throw RuntimeError("uzawa_smooth: zero stabilization diagonal");
    Domain& d = S.domain();
    launch_blas1(3, d.level(level).t, x.p->flags(), omega, S.res_p_.data(level), 0.0, S.diag_c_.data(level),
                 x.p->data(level), kSmoothMask, d.stream());
}

// src/solvers.cpp:548-566 (r := rhs - S x blockwise; DIRICHLET rows rhs - x)
void stokes_residual(StokesSystem& S, StokesState& rhs, StokesState& x, StokesState& r, int level) {
    check_state(rhs, level, "stokes_residual");
    check_state(x, level, "stokes_residual");
    check_state(r, level, "stokes_residual");
    apply(S.a_, *x.u1, S.tmp_u_, level, kSmoothMask);
    assign(1.0, *rhs.u1, -1.0, S.tmp_u_, *r.u1, level, kSmoothMask);
    apply(S.gx_, *x.p, S.tmp_u_, level, kSmoothMask);
    add_scaled(*r.u1, -1.0, S.tmp_u_, level, kSmoothMask);
    assign(1.0, *rhs.u1, -1.0, *x.u1, *r.u1, level, kDirichletMask);
    apply(S.a_, *x.u2, S.tmp_u_, level, kSmoothMask);
    assign(1.0, *rhs.u2, -1.0, S.tmp_u_, *r.u2, level, kSmoothMask);
    apply(S.gy_, *x.p, S.tmp_u_, level, kSmoothMask);
    add_scaled(*r.u2, -1.0, S.tmp_u_, level, kSmoothMask);
    assign(1.0, *rhs.u2, -1.0, *x.u2, *r.u2, level, kDirichletMask);
    apply(S.bx_, *x.u1, S.tmp_p_, level, kSmoothMask);
    assign(1.0, *rhs.p, -1.0, S.tmp_p_, *r.p, level, kSmoothMask);
    apply(S.by_, *x.u2, S.tmp_p_, level, kSmoothMask);
    add_scaled(*r.p, -1.0, S.tmp_p_, level, kSmoothMask);
    apply(S.c_, *x.p, S.tmp_p_, level, kSmoothMask);
    add_scaled(*r.p, -1.0, S.tmp_p_, level, kSmoothMask);
    assign(1.0, *rhs.p, -1.0, *x.p, *r.p, level, kDirichletMask);
}

namespace {
int checked_min_level(int min_level, int max_level) {
    // check_hierarchy_levels (src/solvers.cpp:366-371)
    if (min_level < 1 || min_level > max_level)
        throw InvalidArgument("StokesMultigrid: need 1 <= min_level <= max_level, got [" + std::to_string(min_level) +
                              ", " + std::to_string(max_level) + "]");
    return min_level;
}
void check_cycle(int level, int lo, int hi, int nu_pre, int nu_post, const char* what) {
    if (level < lo || level > hi)
        throw OutOfRange(std::string(what) + ": level " + std::to_string(level) + " outside [" + std::to_string(lo) +
                         ", " + std::to_string(hi) + "]");
    if (nu_pre < 0 || nu_post < 0) throw InvalidArgument(std::string(what) + ": negative smoothing count");
}
} // namespace

// src/solvers.cpp:602-627
StokesMultigrid::StokesMultigrid(Domain& d, int min_level, int max_level, const BoundaryMap& bcu,
                                 const BoundaryMap& bcp, bool project, double omega)
    : dom_(&d), sys_(d, checked_min_level(min_level, max_level), max_level, bcu, bcp),
      r_(d, "stokes_mg.r", min_level, max_level, bcu, bcp), b_(d, "stokes_mg.b", min_level, max_level, bcu, bcp),
      e_(d, "stokes_mg.e", min_level, max_level, bcu, bcp), ones_(d, "stokes_mg.ones", min_level, max_level, bcp),
      omega_(omega), project_(project) {
    const MacroGraph& g = d.graph();
    const HostCsr csr = assemble_stokes_constrained(g, min_level, bcu, bcp);
    const int64_t n = csr.n / 3;
    const std::vector<int64_t> gidx = owned_global_index(g, d.placement(), min_level);
    const HostLayout lay = plan_layout(g, d.placement(), min_level);
    const std::vector<int64_t> pos = owned_positions(g, d.placement(), lay);
    std::vector<uint8_t> fu(gidx.size()), fp(gidx.size());
    for (size_t i = 0; i < gidx.size(); ++i) {
        fu[i] = csr.flag[size_t(gidx[i])];
        fp[i] = csr.flag[size_t(2 * n + gidx[i])];
    }
    coarse_.n = n;
    coarse_.nloc = int64_t(gidx.size());
    coarse_.max_iter = int(3 * n) * 3 + 200; // src/solvers.cpp:715
    coarse_.rowptr = upload_vec(csr.rowptr, d.stream());
    coarse_.col = upload_vec(csr.col, d.stream());
    coarse_.val = upload_vec(csr.val, d.stream());
    coarse_.gidx = upload_vec(gidx, d.stream());
    coarse_.pos = upload_vec(pos, d.stream());
    coarse_.flag_u = upload_vec(fu, d.stream());
    coarse_.flag_p = upload_vec(fp, d.stream());
    coarse_.vec = DevMem(size_t(6 * std::max<int64_t>(n, 1)) * 8);
    const size_t wd = coarse_minres_work_doubles(3 * n);
    if (wd) coarse_.work = DevMem(wd * 8);
    coarse_.status = DevMem(sizeof(CoarseStatus));
    coarse_.hist = DevMem(size_t(coarse_.max_iter + 1) * 8);
    for (int l = min_level; l <= max_level; ++l) fill_const(ones_, 1.0, l, ALL_FLAGS);
}

void StokesMultigrid::vcycle(StokesState& rhs, StokesState& x, int level, int nu_pre, int nu_post) {
    check_cycle(level, min_level(), max_level(), nu_pre, nu_post, "stokes vcycle");
    cycle(rhs, x, level, nu_pre, nu_post);
}

// src/solvers.cpp:635-672
void StokesMultigrid::cycle(StokesState& rhs, StokesState& x, int level, int nu_pre, int nu_post) {
    assign(1.0, *rhs.u1, 0.0, *rhs.u1, *x.u1, level, kDirichletMask);
    assign(1.0, *rhs.u2, 0.0, *rhs.u2, *x.u2, level, kDirichletMask);
    assign(1.0, *rhs.p, 0.0, *rhs.p, *x.p, level, kDirichletMask);
    if (level == min_level()) {
        coarse_correct(rhs, x);
        return;
    }
    for (int i = 0; i < nu_pre; ++i) uzawa_smooth(sys_, rhs, x, level, omega_);
    stokes_residual(sys_, rhs, x, r_, level);
    const int lc = level - 1;
    restrict_to_coarse(*r_.u1, *b_.u1, lc, ALL_FLAGS);
    restrict_to_coarse(*r_.u2, *b_.u2, lc, ALL_FLAGS);
    restrict_to_coarse(*r_.p, *b_.p, lc, ALL_FLAGS);
    fill_const(*b_.u1, 0.0, lc, kDirichletMask);
    fill_const(*b_.u2, 0.0, lc, kDirichletMask);
    fill_const(*b_.p, 0.0, lc, kDirichletMask);
    fill_const(*e_.u1, 0.0, lc, ALL_FLAGS);
    fill_const(*e_.u2, 0.0, lc, ALL_FLAGS);
    fill_const(*e_.p, 0.0, lc, ALL_FLAGS);
    cycle(b_, e_, lc, nu_pre, nu_post);
    // prolongate(e, r, lc, smooth) + add_scaled(x, 1, r, level, smooth): the
    // fused prolongate-add is bitwise the pair
    prolongate(*e_.u1, *x.u1, lc, kSmoothMask, true);
    prolongate(*e_.u2, *x.u2, lc, kSmoothMask, true);
    prolongate(*e_.p, *x.p, lc, kSmoothMask, true);
    for (int i = 0; i < nu_post; ++i) uzawa_smooth(sys_, rhs, x, level, omega_);
}

// src/solvers.cpp:702-726: residual, gather into the monolithic vector (one
// allreduce across processes: one owner per entry), MINRES on the device,
// x += e on the smooth mask. A failed MINRES throws the reference's message
// with the MINRES history, before x is touched.
void StokesMultigrid::coarse_correct(StokesState& rhs, StokesState& x) {
    const int L = min_level();
    Domain& d = *dom_;
    stokes_residual(sys_, rhs, x, r_, L);
    const int64_t n = coarse_.n;
    double* b = coarse_.vec.as<double>();
    double* cx = b + 3 * n;
    HYB_CUDA(cudaMemsetAsync(b, 0, size_t(3 * n) * 8, d.stream()));
    Function* comps[3] = {r_.u1, r_.u2, r_.p};
    for (int k = 0; k < 3; ++k)
        launch_coarse_gather(coarse_.nloc, coarse_.gidx.as<int64_t>(), coarse_.pos.as<int64_t>(), comps[k]->data(L),
                             b + k * n, d.stream());
    d.allreduce_sum(b, 3 * n);
    d.timer_begin("coarse_minres");
    launch_coarse_minres(3 * n, coarse_.rowptr.as<int32_t>(), coarse_.col.as<int32_t>(), coarse_.val.as<double>(), b,
                         cx, coarse_.work.as<double>(), 1e-12, coarse_.max_iter, project_ ? 2 * n : 0,
                         project_ ? 3 * n : 0, coarse_.status.as<CoarseStatus>(), coarse_.hist.as<double>(),
                         d.stream());
    d.timer_end();
    CoarseStatus st{};
    HYB_CUDA(cudaMemcpyAsync(&st, coarse_.status.as<void>(), sizeof st, cudaMemcpyDeviceToHost, d.stream()));
    HYB_CUDA(cudaStreamSynchronize(d.stream()));
    last_coarse_iterations = st.iterations;
    if (!st.converged) {
        std::vector<double> h(size_t(st.iterations) + 1);
        HYB_CUDA(cudaMemcpy(h.data(), coarse_.hist.as<void>(), h.size() * 8, cudaMemcpyDeviceToHost));
        throw RuntimeError("stokes vcycle: coarse MINRES did not converge\n" + solve_history(h, st.breakdown != 0));
    }
    Function* xs[3] = {x.u1, x.u2, x.p};
    for (int k = 0; k < 3; ++k)
        launch_coarse_scatter_add(coarse_.nloc, coarse_.gidx.as<int64_t>(), coarse_.pos.as<int64_t>(),
                                  (k < 2 ? coarse_.flag_u : coarse_.flag_p).as<uint8_t>(), kSmoothMask, cx + k * n,
                                  xs[k]->data(L), d.stream());
}

// src/solvers.cpp:728-731
double StokesMultigrid::residual_norm(StokesState& rhs, StokesState& x, int level) {
    stokes_residual(sys_, rhs, x, r_, level);
    return std::sqrt(stokes_dot(r_, r_, level));
}

// src/solvers.cpp:733-735
double StokesMultigrid::pressure_mean(Function& p, int level) {
    return dot(p, ones_, level) / dot(ones_, ones_, level);
}

// src/solvers.cpp:737-753
std::vector<double> StokesMultigrid::solve(StokesState& rhs, StokesState& x, int level, double tol, int max_cycles,
                                           int nu_pre, int nu_post, bool* converged) {
    check_cycle(level, min_level(), max_level(), nu_pre, nu_post, "stokes solve");
    std::vector<double> res{residual_norm(rhs, x, level)};
    const double r0 = res.front();
    const double target = r0 > 0.0 ? tol * r0 : tol;
    int it = 0;
    while (it < max_cycles && res.back() > target) {
        cycle(rhs, x, level, nu_pre, nu_post);
        ++it;
        res.push_back(residual_norm(rhs, x, level));
    }
    if (converged) *converged = res.back() <= target;
    if (project_) add_scaled(*x.p, -pressure_mean(*x.p, level), ones_, level, kSmoothMask);
    return res;
}

} // namespace hyb
