// Equal-order P1-P1-PSPG Stokes on the device engine (reference
// include/hytegrid/solvers.hpp:117-236, src/solvers.cpp:466-753):
//   StokesState      ~ StokesState: three functions u1, u2 (velocity BCs), p (pressure BCs)
//   StokesSystem     ~ StokesSystem: the Laplacian per velocity component, the
//                      GRAD_X/Y, DIV_X/Y pair and the PSPG block, plus scratch
//   uzawa_smooth     ~ uzawa_smooth: two hybrid Gauss-Seidel sweeps against the
//                      current pressure gradient, then p += omega (g - B u - C p) / diag C
//   stokes_residual  ~ stokes_residual
//   StokesMultigrid  ~ StokesMultigrid: Uzawa-smoothed V-cycles over the P1
//                      transfer pair, MINRES on the assembled monolithic
//                      min-level system (one CTA, bitwise the reference's)
// Every step is the reference's sequence of apply / assign / add_scaled /
// smooth_gs / restrict / prolongate calls on the bitwise kernels, so a sweep,
// a residual and a whole solve reproduce the reference bit for bit.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "domain.hpp"

namespace hyb {

struct StokesState {
    StokesState(Domain& d, const std::string& name, int min_level, int max_level, const BoundaryMap& bc_velocity,
                const BoundaryMap& bc_pressure);
    /// a state over existing functions (not owned)
    StokesState(Function& u1, Function& u2, Function& p) : u1(&u1), u2(&u2), p(&p) {}
    Function* u1;
    Function* u2;
    Function* p;

  private:
    std::unique_ptr<Function> own_[3];
};

/// sum of the three component dot products (src/solvers.cpp:482-484)
double stokes_dot(StokesState& a, StokesState& b, int level);

class StokesSystem {
  public:
    StokesSystem(Domain& d, int min_level, int max_level, const BoundaryMap& bc_velocity,
                 const BoundaryMap& bc_pressure);
    int min_level() const { return a_.min_level(); }
    int max_level() const { return a_.max_level(); }
    const BoundaryMap& bc_velocity() const { return a_.bc(); }
    const BoundaryMap& bc_pressure() const { return c_.bc(); }
    Domain& domain() const { return a_.domain(); }

    Operator a_, gx_, gy_, bx_, by_, c_;
    Function tmp_u_, mom_rhs_, tmp_p_, res_p_, diag_c_;
};

void uzawa_smooth(StokesSystem& S, StokesState& rhs, StokesState& x, int level, double omega);
void stokes_residual(StokesSystem& S, StokesState& rhs, StokesState& x, StokesState& r, int level);

class StokesMultigrid {
  public:
    StokesMultigrid(Domain& d, int min_level, int max_level, const BoundaryMap& bc_velocity,
                    const BoundaryMap& bc_pressure, bool project_pressure_mean, double omega);
    StokesSystem& system() { return sys_; }
    int min_level() const { return sys_.min_level(); }
    int max_level() const { return sys_.max_level(); }
    void vcycle(StokesState& rhs, StokesState& x, int level, int nu_pre, int nu_post);
    /// residual history; *converged as SolveReport::converged
    std::vector<double> solve(StokesState& rhs, StokesState& x, int level, double tol, int max_cycles, int nu_pre,
                              int nu_post, bool* converged);
    double residual_norm(StokesState& rhs, StokesState& x, int level);
    double pressure_mean(Function& p, int level);
    int last_coarse_iterations = 0;

  private:
    void cycle(StokesState& rhs, StokesState& x, int level, int nu_pre, int nu_post);
    void coarse_correct(StokesState& rhs, StokesState& x);

    Domain* dom_;
    StokesSystem sys_;
    StokesState r_, b_, e_;
    Function ones_;
    double omega_;
    bool project_;
    struct Coarse {
        int64_t n = 0, nloc = 0; // n: one block (the P1 min-level numbering); the system has 3n rows
        int max_iter = 0;
        DevMem rowptr, col, val;      // constrained monolithic CSR
        DevMem gidx, pos, flag_u, flag_p;
        DevMem vec;                   // b (3n), x (3n)
        DevMem work;                  // MINRES vectors when they do not fit in shared memory
        DevMem status, hist;
    } coarse_;
};

/// SolveReport::history() text (src/solvers.cpp:208-224)
std::string solve_history(const std::vector<double>& residuals, bool breakdown);

} // namespace hyb
