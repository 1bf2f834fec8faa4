// C++ drop-in check: the reference's usage pattern (cf. reference
// tests/test_operators.cpp, tests/test_solvers.cpp) against hytegrid_b200.hpp.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>

#include "hytegrid_b200.hpp"

using namespace hytegrid_b200;

#define EXPECT(cond)                                                                                \
    do {                                                                                            \
        if (!(cond)) {                                                                              \
            std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond);                  \
            return 1;                                                                               \
        }                                                                                           \
    } while (0)

int main() {
    const int level = 5;
    DistributedDomain dom(meshgen::square_ring8(), 2);
    Controller ctl(dom);
    ScalarFunction src("src", dom, 1, level), dst("dst", dom, 1, level);
    register_function(ctl, src);
    StencilOperator A(dom, Form::LAPLACE, 1, level);
    // linear fields are annihilated on interior rows (tests/test_operators.cpp:265-285)
    interpolate(src, [](double x, double y) { return 1.5 + 2.0 * x - 0.75 * y; }, level);
    apply(A, ctl, src, dst, level, flag_bit(DoFFlag::INNER));
    const auto y = dst.download(level);
    double m = 0;
    for (double v : y) m = std::fmax(m, std::fabs(v));
    EXPECT(m <= 1e-12);
    // misuse raises the reference's exception types (tests/test_operators.cpp:444-469)
    bool threw = false;
    try {
        apply(A, ctl, src, src, level);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    EXPECT(threw);
    threw = false;
    try {
        apply(A, ctl, src, dst, level + 1);
    } catch (const std::out_of_range&) {
        threw = true;
    }
    EXPECT(threw);
    // harmonic extension of linear Dirichlet data (tests/test_solvers.cpp:408-429)
    DistributedDomain sq(meshgen::unit_square(), 3);
    Controller c2(sq);
    GridHierarchy mg(sq, c2, Form::LAPLACE, 1, level);
    ScalarFunction rhs("rhs", sq, 1, level), x("x", sq, 1, level);
    interpolate(rhs, [](double a, double b) { return 1.5 + 2.0 * a - 0.75 * b; }, level,
                flag_bit(DoFFlag::DIRICHLET));
    // the same boundary data from a device-evaluated expression: bitwise the host callable's
    ScalarFunction rhs2("rhs2", sq, 1, level);
    interpolate(rhs2, Expr::poly2(1.5, 2.0, -0.75), level, flag_bit(DoFFlag::DIRICHLET));
    EXPECT(rhs2.download(level) == rhs.download(level));
    const SolveReport rep = mg.solve(rhs, x, level, 1e-12, 60);
    EXPECT(rep.converged);
    const auto xs = x.download(level);
    const auto xy = sq.coords(level);
    double err = 0;
    for (size_t i = 0; i < xs.size(); ++i)
        err = std::fmax(err, std::fabs(xs[i] - (1.5 + 2.0 * xy[2 * i] - 0.75 * xy[2 * i + 1])));
    EXPECT(err <= 1e-10);
    // partial-direction sync in the reference's full order == sync_all (function.hpp:79-81)
    sync(c2, x, level, {Direction::VERTEX_TO_EDGE, Direction::EDGE_TO_FACE, Direction::FACE_TO_EDGE,
                        Direction::EDGE_TO_VERTEX});
    // the exact solution is a fixed point of the reference's GS sweep (tests/test_operators.cpp:287-310)
    StencilOperator As(sq, Form::LAPLACE, level, level);
    smooth_gs(As, c2, rhs, x, level);
    const auto xg = x.download(level);
    double moved = 0;
    for (size_t i = 0; i < xs.size(); ++i) moved = std::fmax(moved, std::fabs(xg[i] - xs[i]));
    EXPECT(moved <= 1e-12);
    // the additions: weighted-Jacobi FMG and V(1,1)-preconditioned CG
    GridHierarchy mj(sq, c2, Form::LAPLACE, 1, level, {}, Smoother::JACOBI);
    ScalarFunction f("f", sq, 1, level), u("u", sq, 1, level);
    interpolate(f, [](double a, double b) { return a * (1 - a) + b; }, level, flag_bit(DoFFlag::INNER));
    const SolveReport fr = mj.fmg(f, u, level, 1e-8, 40);
    EXPECT(fr.converged && fr.residuals.back() <= 1e-8 * fr.residuals.front());
    const SolveReport pr = mj.pcg(f, u, level, 20);
    EXPECT(pr.residuals.size() == 21 && pr.residuals.back() <= 1e-9 * pr.residuals.front());
    // checkpoint records (DataCallbacks::serialize) of every primitive round-trip into a fresh
    // function. Records hold the state after a ghost refresh, so the comparison is made once every
    // owner has been restored (unit square: 4 vertices, 5 edges, 2 faces)
    ScalarFunction w("w", sq, 1, level);
    for (std::uint64_t p = 0; p < 11; ++p) w.deserialize(p, u.serialize(p));
    for (std::uint64_t p = 0; p < 11; ++p) EXPECT(w.serialize(p) == u.serialize(p));
    EXPECT(w.download(level) == u.download(level));
    // SolveReport::history() of the reference GridHierarchy's own cycle (smooth_gs, min level 1) on a
    // keyed U[-1,1] rhs (seed 5): tests/test_cpp_api.py prints the reference's text for the same solve
    {
        DistributedDomain hd(meshgen::unit_square(), 1);
        Controller hc(hd);
        GridHierarchy hg(hd, hc, Form::LAPLACE, 1, level);
        ScalarFunction hr("hr", hd, 1, level), hx("hx", hd, 1, level);
        EXPECT(hyb_interpolate_random(hr.handle(), level, 5, 0, -1.0, 1.0, HYB_ALL_FLAGS) == HYB_OK);
        const SolveReport hrep = hg.solve(hr, hx, level, 0.0, 6);
        std::printf("HISTORY_BEGIN\n%sHISTORY_END\n", hrep.history().c_str());
    }
    // P1-P1-PSPG Stokes: the reference's enclosed-cavity test (tests/test_solvers.cpp:689-719) through
    // the drop-in types: all-Dirichlet velocity, free pressure with its mean projected out
    {
        DistributedDomain sd(meshgen::unit_square(), 2);
        Controller scx(sd);
        BoundaryConditions free_p;
        for (int m = 1; m <= 3; ++m) free_p.marker_flag[m] = DoFFlag::NEUMANN;
        StokesMultigrid smg(sd, scx, 1, 3, {}, free_p, true);
        StokesState srhs("rhs", sd, 1, 3, {}, free_p), sx("x", sd, 1, 3, {}, free_p);
        register_state(scx, srhs);
        interpolate(srhs.u1, [](double a, double b) { return std::exp(0.3 * a - 0.2 * b) + 0.1 * a * b; }, 3,
                    flag_bit(DoFFlag::INNER) | flag_bit(DoFFlag::NEUMANN));
        const SolveReport srep = smg.solve(srhs, sx, 3, 1e-8, 20);
        EXPECT(srep.converged);
        EXPECT(std::fabs(smg.pressure_mean(sx.p, 3)) <= 1e-9);
        StokesState sr("r", sd, 1, 3, {}, free_p);
        stokes_residual(smg.system(), scx, srhs, sx, sr, 3);
        EXPECT(std::sqrt(stokes_dot(sr, sr, 3)) <= 1e-8 * srep.residuals.front());
        uzawa_smooth(smg.system(), scx, srhs, sx, 3);
    }
    // P2 through the reference's signatures: apply of the P2 Laplacian to a quadratic is exact
    // against the mass matrix times its (constant) negative Laplacian, checked as a zero row sum
    {
        DistributedDomain pd(meshgen::unit_square(), 2);
        Controller pc(pd);
        StencilOperator a2(pd, Form::LAPLACE, FunctionKind::P2, 2, 2);
        ScalarFunction one("one", pd, FunctionKind::P2, 2, 2, {}), y2("y2", pd, FunctionKind::P2, 2, 2, {});
        interpolate(one, [](double, double) { return 1.0; }, 2);
        apply(a2, pc, one, y2, 2, flag_bit(DoFFlag::INNER));
        const auto yv = y2.download(2);
        double m = 0;
        for (double v : yv) m = std::fmax(m, std::fabs(v));
        EXPECT(yv.size() == 81 && m <= 1e-12); // constants are in the kernel of the Laplacian
        smooth_gs(a2, pc, y2, one, 2);
        smooth_jacobi(a2, pc, y2, one, 0.8, 2);
    }
    // a user PackInfo plugin on the reference's Controller schedule: every face receives its three
    // edges' messages (E->F), in slot order
    {
        struct Count : PackInfo {
            mutable std::map<std::uint64_t, std::vector<std::uint64_t>> got;
            void pack(std::uint64_t s, std::uint64_t, Direction, int, std::vector<std::uint8_t>& out) const override {
                out.resize(8);
                std::memcpy(out.data(), &s, 8);
            }
            std::size_t unpack(std::uint64_t r, std::uint64_t, Direction, int, const std::uint8_t* in,
                               std::size_t len) const override {
                std::uint64_t s = 0;
                std::memcpy(&s, in, 8);
                got[r].push_back(s);
                return len;
            }
        };
        DistributedDomain cd(meshgen::unit_square(), 2);
        Controller cc(cd);
        auto info = std::make_shared<Count>();
        cc.register_pack_info(5, info);
        cc.sync(5, 2, {Direction::EDGE_TO_FACE});
        EXPECT(info->got.size() == 2 && info->got.begin()->second.size() == 3);
    }
    std::printf("cpp api ok: %d cycles, residual %.3e, error %.3e; fmg %d cycles, pcg %.1e\n", rep.iterations,
                rep.residuals.back(), err, fr.iterations, pr.residuals.back() / pr.residuals.front());
    return 0;
}
