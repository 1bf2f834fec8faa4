// hytegrid_b200.hpp -- C++ drop-in for the reference's multigrid hot-path API
// (arXiv 1805.10167 "hytegrid", /root/reference/proj/include/hytegrid/*.hpp),
// header-only over the C ABI in hyteg_b200.h. Same names, argument order and
// exception types as the reference:
//
//   reference                                   here
//   DistributedDomain(setup, assignment, P)     DistributedDomain(mesh_text, P[, assignment])
//   Controller(domain), register_function       Controller(domain), register_function (no-ops)
//   ScalarFunction(name, dom, kind, min, max, bc) same (kind P1 or P2; P1 when omitted)
//   StencilOperator(dom, form, kind, min, max, bc) same (kind P1 or P2; P1 when omitted)
//   apply / smooth_jacobi / smooth_gs / diagonal same (operators.hpp:108-125)
//   prolongate / restrict_to_coarse             same (solvers.hpp:26-33)
//   assign / add_scaled / dot / norm2 / max_abs same (function.hpp:60-74)
//   interpolate(f, expr, level, mask)           same; expr evaluated on the host at the
//                                               reference's DoF coordinates, then uploaded
//   sync_all(ctl, f, level)                     same
//   GridHierarchy(dom, ctl, form, min, max, bc) same (+ smoother choice, Jacobi weight, coarse tolerance;
//                                               default: the reference's Gauss-Seidel)
//   StokesState / StokesSystem / uzawa_smooth / same (solvers.hpp:117-236)
//   stokes_residual / stokes_dot / StokesMultigrid
//   f.values(id, level)                         f.download(level) / f.upload(level, v)
//                                               (GlobalDoFMap order, numbering.hpp:41-43)
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "hyteg_b200.h"

namespace hytegrid_b200 {

enum class DoFFlag : std::uint8_t { INNER = 1, DIRICHLET = 2, NEUMANN = 4 };
/// include/hytegrid/indexing.hpp:28 (DG0 is not provided)
enum class FunctionKind : int { P1 = HYB_P1, P2 = HYB_P2 };
constexpr std::uint8_t ALL_DOF_FLAGS = 7;
inline std::uint8_t flag_bit(DoFFlag f) { return static_cast<std::uint8_t>(f); }
enum class Form : int {
    LAPLACE = HYB_LAPLACE,
    MASS = HYB_MASS,
    DIV_X = HYB_DIV_X,
    DIV_Y = HYB_DIV_Y,
    GRAD_X = HYB_GRAD_X,
    GRAD_Y = HYB_GRAD_Y,
    PSPG = HYB_PSPG
};
/// GridHierarchy smoother: the reference always uses its hybrid Gauss-Seidel
/// (solvers.cpp:417, 427); weighted Jacobi and coloured GS are additions.
enum class Smoother : int { GAUSS_SEIDEL = HYB_SMOOTH_GS, JACOBI = HYB_SMOOTH_JACOBI, COLORED_GS = HYB_SMOOTH_COLORED_GS };

struct BoundaryConditions {
    std::map<int, DoFFlag> marker_flag;
};

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(int status) {
    if (status == HYB_OK) return;
    const std::string msg = hyb_last_error();
    switch (status) {
    case HYB_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case HYB_OUT_OF_RANGE: throw std::out_of_range(msg);
    case HYB_RUNTIME_ERROR: throw std::runtime_error(msg);
    case HYB_LOGIC_ERROR: throw std::logic_error(msg);
    default: throw CudaError(msg);
    }
}

namespace meshgen {
inline std::string gen(const char* kind, std::vector<double> p = {}) {
    int64_t len = 0;
    check(hyb_meshgen(kind, p.data(), int(p.size()), nullptr, 0, &len));
    std::string s(size_t(len) + 1, '\0');
    check(hyb_meshgen(kind, p.data(), int(p.size()), s.data(), len + 1, &len));
    s.resize(size_t(len));
    return s;
}
inline std::string unit_triangle() { return gen("unit_triangle"); }
inline std::string unit_square() { return gen("unit_square"); }
inline std::string unit_square_reversed() { return gen("unit_square_reversed"); }
inline std::string square_ring8() { return gen("square_ring8"); }
inline std::string channel(int nx, int ny, double w = 1.0, double h = 1.0) { return gen("channel", {double(nx), double(ny), w, h}); }
inline std::string annulus(int seg, int layers, double ri, double ro) {
    return gen("annulus", {double(seg), double(layers), ri, ro});
}
} // namespace meshgen

class DistributedDomain {
  public:
    /// P logical ranks, all driven by this process (the reference's model);
    /// assignment empty = partition_round_robin.
    DistributedDomain(const std::string& mesh_text, int ranks = 1, std::vector<int32_t> assignment = {},
                      int device = 0) {
        int64_t nv, ne, nf;
        check(hyb_mesh_counts(mesh_text.c_str(), &nv, &ne, &nf));
        if (assignment.empty()) {
            assignment.resize(size_t(nv + ne + nf));
            check(hyb_partition(mesh_text.c_str(), ranks, HYB_PARTITION_ROUND_ROBIN, 0, assignment.data()));
        }
        std::vector<int32_t> local(static_cast<size_t>(ranks));
        for (int r = 0; r < ranks; ++r) local[size_t(r)] = r;
        check(hyb_domain_create(mesh_text.c_str(), ranks, assignment.data(), local.data(), ranks, device, &h_));
    }
    ~DistributedDomain() { hyb_domain_destroy(h_); }
    DistributedDomain(const DistributedDomain&) = delete;
    DistributedDomain& operator=(const DistributedDomain&) = delete;
    hyb_domain* handle() const { return h_; }
    int64_t owned(int level) const {
        int64_t t = 0;
        check(hyb_domain_owned_count(h_, level, &t, nullptr));
        return t;
    }
    std::vector<double> coords(int level, int kind = HYB_P1) const {
        const int64_t n = owned(kind == HYB_P2 ? level + 1 : level);
        std::vector<double> xy(size_t(2 * n));
        check(hyb_owned_coords_kind(h_, kind, level, 1, xy.data(), n));
        return xy;
    }

  private:
    hyb_domain* h_ = nullptr;
};

class ScalarFunction;

enum class Direction : int { VERTEX_TO_EDGE = HYB_V2E, EDGE_TO_FACE = HYB_E2F, FACE_TO_EDGE = HYB_F2E,
                             EDGE_TO_VERTEX = HYB_E2V };

/// The reference's extension point (communication.hpp:24-34) for data the
/// caller keeps on the host: primitives are named by ID (the device owns the
/// field storage, so no Primitive object is handed out); unpack returns the
/// bytes it consumed (fewer than the message is the reference's logic_error).
class PackInfo {
  public:
    virtual ~PackInfo() = default;
    virtual void pack(std::uint64_t sender, std::uint64_t receiver, Direction dir, int level,
                      std::vector<std::uint8_t>& out) const = 0;
    virtual std::size_t unpack(std::uint64_t receiver, std::uint64_t sender, Direction dir, int level,
                               const std::uint8_t* in, std::size_t len) const = 0;
};

class Controller {
  public:
    explicit Controller(DistributedDomain& d) : domain_(&d) {}
    DistributedDomain& domain() { return *domain_; }
    /// Controller::register_pack_info / sync (communication.hpp:44-49)
    void register_pack_info(std::uint32_t channel, std::shared_ptr<const PackInfo> info) {
        if (!info) throw std::invalid_argument("register_pack_info: null PackInfo");
        check(hyb_register_pack_info(domain_->handle(), channel, &pack_cb, &unpack_cb,
                                     const_cast<PackInfo*>(info.get())));
        infos_[channel] = std::move(info);
    }
    void sync(std::uint32_t channel, int level, const std::vector<Direction>& dirs) {
        std::vector<int> d;
        for (Direction x : dirs) d.push_back(int(x));
        check(hyb_controller_sync(domain_->handle(), channel, level, d.data(), int(d.size())));
    }

  private:
    static int pack_cb(void* user, std::uint64_t s, std::uint64_t r, int dir, int level, std::uint8_t* out,
                       std::int64_t cap, std::int64_t* len) {
        try {
            std::vector<std::uint8_t> buf;
            static_cast<const PackInfo*>(user)->pack(s, r, Direction(dir), level, buf);
            *len = std::int64_t(buf.size());
            if (out && cap >= *len && !buf.empty()) std::memcpy(out, buf.data(), buf.size());
            return 0;
        } catch (...) {
            return 1;
        }
    }
    static int unpack_cb(void* user, std::uint64_t r, std::uint64_t s, int dir, int level, const std::uint8_t* in,
                         std::int64_t len, std::int64_t* used) {
        try {
            *used = std::int64_t(static_cast<const PackInfo*>(user)->unpack(r, s, Direction(dir), level, in,
                                                                            std::size_t(len)));
            return 0;
        } catch (...) {
            return 1;
        }
    }
    DistributedDomain* domain_;
    std::map<std::uint32_t, std::shared_ptr<const PackInfo>> infos_;
};

namespace detail {
inline void bc_arrays(const BoundaryConditions& bc, std::vector<int32_t>& m, std::vector<uint8_t>& f) {
    for (const auto& [k, v] : bc.marker_flag) {
        m.push_back(k);
        f.push_back(static_cast<uint8_t>(v));
    }
}
} // namespace detail

class ScalarFunction {
  public:
    ScalarFunction(const std::string& name, DistributedDomain& d, int min_level, int max_level,
                   BoundaryConditions bc = {})
        : ScalarFunction(name, d, FunctionKind::P1, min_level, max_level, std::move(bc)) {}
    /// the reference's signature (function.hpp:19-20)
    ScalarFunction(const std::string& name, DistributedDomain& d, FunctionKind kind, int min_level, int max_level,
                   BoundaryConditions bc = {})
        : dom_(&d), kind_(kind) {
        std::vector<int32_t> m;
        std::vector<uint8_t> f;
        detail::bc_arrays(bc, m, f);
        check(hyb_function_create_kind(d.handle(), name.c_str(), int(kind), min_level, max_level, m.data(), f.data(),
                                       int(m.size()), &h_));
    }
    FunctionKind kind() const { return kind_; }
    ~ScalarFunction() { hyb_function_destroy(h_); }
    ScalarFunction(const ScalarFunction&) = delete;
    ScalarFunction& operator=(const ScalarFunction&) = delete;
    hyb_function* handle() const { return h_; }
    DistributedDomain& domain() const { return *dom_; }
    std::vector<double> download(int level) const {
        // a P2 function at level L holds the DoF count of P1 at level L + 1
        std::vector<double> v(size_t(dom_->owned(kind_ == FunctionKind::P2 ? level + 1 : level)));
        check(hyb_function_download(h_, level, v.data(), int64_t(v.size()), 1));
        return v;
    }
    void upload(int level, const std::vector<double>& v, std::uint8_t mask = ALL_DOF_FLAGS) {
        check(hyb_function_upload(h_, level, v.data(), int64_t(v.size()), 1, mask));
    }
    /// the primitive's record as DataCallbacks::serialize writes it (field.cpp:157-175)
    std::vector<std::uint8_t> serialize(std::uint64_t prim) const {
        int64_t n = 0;
        check(hyb_function_serialize(h_, prim, nullptr, 0, &n));
        std::vector<std::uint8_t> out(static_cast<size_t>(n));
        check(hyb_function_serialize(h_, prim, out.data(), n, &n));
        return out;
    }
    /// DataCallbacks::deserialize into this function's slots of `prim`
    void deserialize(std::uint64_t prim, const std::vector<std::uint8_t>& record) {
        check(hyb_function_deserialize(h_, prim, record.data(), int64_t(record.size())));
    }

  private:
    DistributedDomain* dom_;
    FunctionKind kind_ = FunctionKind::P1;
    hyb_function* h_ = nullptr;
};

inline void register_function(Controller&, const ScalarFunction&) {}

class StencilOperator {
  public:
    StencilOperator(DistributedDomain& d, Form form, int min_level, int max_level, BoundaryConditions bc = {})
        : StencilOperator(d, form, FunctionKind::P1, min_level, max_level, std::move(bc)) {}
    /// the reference's signature (operators.hpp:76-88)
    StencilOperator(DistributedDomain& d, Form form, FunctionKind kind, int min_level, int max_level,
                    BoundaryConditions bc = {}) {
        std::vector<int32_t> m;
        std::vector<uint8_t> f;
        detail::bc_arrays(bc, m, f);
        check(hyb_operator_create_kind(d.handle(), int(form), int(kind), min_level, max_level, m.data(), f.data(),
                                       int(m.size()), &h_));
    }
    ~StencilOperator() { hyb_operator_destroy(h_); }
    StencilOperator(const StencilOperator&) = delete;
    StencilOperator& operator=(const StencilOperator&) = delete;
    hyb_operator* handle() const { return h_; }

  private:
    hyb_operator* h_ = nullptr;
};

inline void interpolate(ScalarFunction& f, const std::function<double(double, double)>& expr, int level,
                        std::uint8_t mask = ALL_DOF_FLAGS) {
    const std::vector<double> xy = f.domain().coords(level, int(f.kind()));
    std::vector<double> v(xy.size() / 2);
    for (size_t i = 0; i < v.size(); ++i) v[i] = expr(xy[2 * i], xy[2 * i + 1]);
    f.upload(level, v, mask);
}
/// an analytic expression evaluated on the device at the reference's DoF coordinates (no host round trip)
struct Expr {
    int kind = HYB_EXPR_POLY2;
    std::vector<double> params;
    static Expr poly2(double p0, double px, double py, double pxx = 0, double pxy = 0, double pyy = 0) {
        return {HYB_EXPR_POLY2, {p0, px, py, pxx, pxy, pyy}};
    }
    /// a sin(kx x + phx) sin(ky y + phy) + c
    static Expr sinsin(double a, double kx, double phx, double ky, double phy, double c = 0) {
        return {HYB_EXPR_SINSIN, {a, kx, phx, ky, phy, c}};
    }
};
inline void interpolate(ScalarFunction& f, const Expr& e, int level, std::uint8_t mask = ALL_DOF_FLAGS) {
    check(hyb_interpolate_expr(f.handle(), level, e.kind, e.params.data(), int(e.params.size()), mask));
}
inline void sync_all(Controller&, const ScalarFunction& f, int level) { check(hyb_sync(f.handle(), level)); }
/// the reference's Direction (transport.hpp:19-26)
/// sync(c, f, level, span<Direction>) (function.hpp:79-80): the directions in order
inline void sync(Controller&, const ScalarFunction& f, int level, const std::vector<Direction>& dirs) {
    std::vector<int> d;
    for (Direction x : dirs) d.push_back(int(x));
    check(hyb_sync_directions(f.handle(), level, d.data(), int(d.size())));
}
inline void apply(const StencilOperator& A, Controller&, const ScalarFunction& src, ScalarFunction& dst, int level,
                  std::uint8_t mask = ALL_DOF_FLAGS) {
    check(hyb_apply(A.handle(), src.handle(), dst.handle(), level, mask));
}
inline void smooth_jacobi(const StencilOperator& A, Controller&, const ScalarFunction& rhs, ScalarFunction& x,
                          double omega, int level) {
    check(hyb_smooth_jacobi(A.handle(), rhs.handle(), x.handle(), omega, level));
}
/// the reference's hybrid Gauss-Seidel sweep (operators.hpp:120-121), bitwise
inline void smooth_gs(const StencilOperator& A, Controller&, const ScalarFunction& rhs, ScalarFunction& x, int level) {
    check(hyb_smooth_gs(A.handle(), rhs.handle(), x.handle(), level));
}
/// coloured variant (faces by (c + 2r) mod 3, edges odd/even); no reference counterpart
inline void smooth_colored_gs(const StencilOperator& A, Controller&, const ScalarFunction& rhs, ScalarFunction& x,
                              int level) {
    check(hyb_smooth_cgs(A.handle(), rhs.handle(), x.handle(), level));
}
inline void diagonal(const StencilOperator& A, ScalarFunction& d, int level) {
    check(hyb_diagonal(A.handle(), d.handle(), level));
}
inline void prolongate(Controller&, const ScalarFunction& coarse, ScalarFunction& fine, int coarse_level,
                       std::uint8_t mask = ALL_DOF_FLAGS) {
    check(hyb_prolongate(coarse.handle(), fine.handle(), coarse_level, mask));
}
inline void restrict_to_coarse(Controller&, const ScalarFunction& fine, ScalarFunction& coarse, int coarse_level,
                               std::uint8_t mask = ALL_DOF_FLAGS) {
    check(hyb_restrict(fine.handle(), coarse.handle(), coarse_level, mask));
}
inline void assign(double alpha, const ScalarFunction& x1, double beta, const ScalarFunction& x2, ScalarFunction& dst,
                   int level, std::uint8_t mask = ALL_DOF_FLAGS) {
    check(hyb_assign(alpha, x1.handle(), beta, x2.handle(), dst.handle(), level, mask));
}
inline void add_scaled(ScalarFunction& dst, double gamma, const ScalarFunction& y, int level,
                       std::uint8_t mask = ALL_DOF_FLAGS) {
    check(hyb_add_scaled(dst.handle(), gamma, y.handle(), level, mask));
}
inline double dot(const ScalarFunction& a, const ScalarFunction& b, int level) {
    double out = 0;
    check(hyb_dot(a.handle(), b.handle(), level, &out));
    return out;
}
inline double norm2(const ScalarFunction& a, int level) { return std::sqrt(dot(a, a, level)); }
inline double max_abs(const ScalarFunction& a, int level) {
    double out = 0;
    check(hyb_max_abs(a.handle(), level, &out));
    return out;
}

struct SolveReport {
    bool converged = false;
    bool breakdown = false;
    int iterations = 0;
    std::vector<double> residuals;

    /// One "cycle <k> residual <norm> factor <reduction>" line per entry, the
    /// format of the reference's SolveReport::history (src/solvers.cpp:208-224).
    std::string history() const {
        std::string out;
        char line[96];
        for (std::size_t k = 0; k < residuals.size(); ++k) {
            if (k == 0) {
                std::snprintf(line, sizeof line, "cycle %zu residual %.6e\n", k, residuals[k]);
            } else {
                const double f = residuals[k - 1] > 0.0 ? residuals[k] / residuals[k - 1] : 0.0;
                std::snprintf(line, sizeof line, "cycle %zu residual %.6e factor %.4f\n", k, residuals[k], f);
            }
            out += line;
        }
        if (breakdown) out += "breakdown\n";
        return out;
    }
};

class GridHierarchy {
  public:
    GridHierarchy(DistributedDomain& d, Controller&, Form form, int min_level, int max_level,
                  BoundaryConditions bc = {}, Smoother smoother = Smoother::GAUSS_SEIDEL, double omega = 2.0 / 3.0,
                  double coarse_tol = 1e-12)
        : max_(max_level) {
        std::vector<int32_t> m;
        std::vector<uint8_t> f;
        detail::bc_arrays(bc, m, f);
        check(hyb_hierarchy_create(d.handle(), int(form), min_level, max_level, m.data(), f.data(), int(m.size()),
                                   int(smoother), omega, coarse_tol, -1, &h_));
    }
    ~GridHierarchy() { hyb_hierarchy_destroy(h_); }
    GridHierarchy(const GridHierarchy&) = delete;
    GridHierarchy& operator=(const GridHierarchy&) = delete;
    void vcycle(const ScalarFunction& rhs, ScalarFunction& x, int level, int nu_pre = 2, int nu_post = 2) {
        check(hyb_hierarchy_vcycle(h_, rhs.handle(), x.handle(), level, nu_pre, nu_post));
    }
    double residual_norm(const ScalarFunction& rhs, const ScalarFunction& x, int level) {
        double out = 0;
        check(hyb_hierarchy_residual_norm(h_, rhs.handle(), x.handle(), level, &out));
        return out;
    }
    SolveReport solve(const ScalarFunction& rhs, ScalarFunction& x, int level, double tol, int max_cycles,
                      int nu_pre = 2, int nu_post = 2) {
        SolveReport rep;
        rep.residuals.resize(size_t(max_cycles) + 1);
        int n = 0, conv = 0;
        check(hyb_hierarchy_solve(h_, rhs.handle(), x.handle(), level, tol, max_cycles, nu_pre, nu_post,
                                  rep.residuals.data(), &n, &conv));
        rep.residuals.resize(size_t(n));
        rep.iterations = n - 1;
        rep.converged = conv != 0;
        return rep;
    }
    /// full multigrid (rhs coarser levels are overwritten), see hyb_hierarchy_fmg
    SolveReport fmg(ScalarFunction& rhs, ScalarFunction& x, int level, double tol, int max_cycles, int nu_pre = 2,
                    int nu_post = 2, int cycles_per_level = 1) {
        SolveReport rep;
        rep.residuals.resize(size_t(max_cycles) + 2);
        int n = 0, conv = 0;
        check(hyb_hierarchy_fmg(h_, rhs.handle(), x.handle(), level, cycles_per_level, nu_pre, nu_post, tol,
                                max_cycles, rep.residuals.data(), &n, &conv));
        rep.residuals.resize(size_t(n));
        rep.iterations = n - 2;
        rep.converged = conv != 0;
        return rep;
    }
    /// V-cycle preconditioned CG from x = 0, see hyb_hierarchy_pcg
    SolveReport pcg(const ScalarFunction& rhs, ScalarFunction& x, int level, int max_iter, double tol = 0.0,
                    int nu_pre = 1, int nu_post = 1) {
        SolveReport rep;
        rep.residuals.resize(size_t(max_iter) + 1);
        int n = 0, conv = 0;
        check(hyb_hierarchy_pcg(h_, rhs.handle(), x.handle(), level, max_iter, nu_pre, nu_post, tol,
                                rep.residuals.data(), &n, &conv));
        rep.residuals.resize(size_t(n));
        rep.iterations = n - 1;
        rep.converged = conv != 0;
        return rep;
    }

  private:
    hyb_hierarchy* h_ = nullptr;
    int max_;
};

// ---- P1-P1-PSPG Stokes (reference include/hytegrid/solvers.hpp:117-236) ----

/// u1, u2 carry the velocity boundary conditions, p the pressure ones
struct StokesState {
    StokesState(const std::string& name, DistributedDomain& d, int min_level, int max_level,
                const BoundaryConditions& bc_velocity, const BoundaryConditions& bc_pressure)
        : u1(name + ".u1", d, min_level, max_level, bc_velocity), u2(name + ".u2", d, min_level, max_level, bc_velocity),
          p(name + ".p", d, min_level, max_level, bc_pressure) {}
    ScalarFunction u1, u2, p;
};

inline void register_state(Controller&, const StokesState&) {}

namespace detail {
struct State3 {
    hyb_function* f[3];
    explicit State3(const StokesState& s) : f{s.u1.handle(), s.u2.handle(), s.p.handle()} {}
};
} // namespace detail

inline double stokes_dot(const StokesState& a, const StokesState& b, int level) {
    double out = 0;
    check(hyb_stokes_dot(detail::State3(a).f, detail::State3(b).f, level, &out));
    return out;
}

class StokesSystem {
  public:
    StokesSystem(DistributedDomain& d, int min_level, int max_level, BoundaryConditions bc_velocity,
                 BoundaryConditions bc_pressure) {
        std::vector<int32_t> mu, mp;
        std::vector<uint8_t> fu, fp;
        detail::bc_arrays(bc_velocity, mu, fu);
        detail::bc_arrays(bc_pressure, mp, fp);
        check(hyb_stokes_create(d.handle(), min_level, max_level, mu.data(), fu.data(), int(mu.size()), mp.data(),
                                fp.data(), int(mp.size()), 0, 0, 0.3, &h_));
    }
    ~StokesSystem() {
        if (owner_) hyb_stokes_destroy(h_);
    }
    StokesSystem(const StokesSystem&) = delete;
    StokesSystem& operator=(const StokesSystem&) = delete;
    hyb_stokes* handle() const { return h_; }

  private:
    friend class StokesMultigrid;
    explicit StokesSystem(hyb_stokes* h) : h_(h), owner_(false) {}
    hyb_stokes* h_ = nullptr;
    bool owner_ = true;
};

inline void uzawa_smooth(StokesSystem& S, Controller&, const StokesState& rhs, StokesState& x, int level,
                         double omega = 0.3) {
    check(hyb_uzawa_smooth(S.handle(), detail::State3(rhs).f, detail::State3(x).f, level, omega));
}

inline void stokes_residual(StokesSystem& S, Controller&, const StokesState& rhs, const StokesState& x,
                            StokesState& r, int level) {
    check(hyb_stokes_residual(S.handle(), detail::State3(rhs).f, detail::State3(x).f, detail::State3(r).f, level));
}

class StokesMultigrid {
  public:
    StokesMultigrid(DistributedDomain& d, Controller&, int min_level, int max_level, BoundaryConditions bc_velocity,
                    BoundaryConditions bc_pressure, bool project_pressure_mean = false, double omega = 0.3)
        : h_(create(d, min_level, max_level, bc_velocity, bc_pressure, project_pressure_mean, omega)), sys_(h_),
          min_(min_level), max_(max_level) {}
    ~StokesMultigrid() { hyb_stokes_destroy(h_); }
    StokesMultigrid(const StokesMultigrid&) = delete;
    StokesMultigrid& operator=(const StokesMultigrid&) = delete;
    StokesSystem& system() { return sys_; }
    int min_level() const { return min_; }
    int max_level() const { return max_; }
    void vcycle(const StokesState& rhs, StokesState& x, int level, int nu_pre = 2, int nu_post = 2) {
        check(hyb_stokes_vcycle(h_, detail::State3(rhs).f, detail::State3(x).f, level, nu_pre, nu_post));
    }
    SolveReport solve(const StokesState& rhs, StokesState& x, int level, double tol, int max_cycles, int nu_pre = 2,
                      int nu_post = 2) {
        SolveReport rep;
        rep.residuals.resize(size_t(max_cycles) + 1);
        int n = 0, conv = 0;
        check(hyb_stokes_solve(h_, detail::State3(rhs).f, detail::State3(x).f, level, tol, max_cycles, nu_pre, nu_post,
                               rep.residuals.data(), &n, &conv));
        rep.residuals.resize(size_t(n));
        rep.iterations = n - 1;
        rep.converged = conv != 0;
        return rep;
    }
    double residual_norm(const StokesState& rhs, const StokesState& x, int level) {
        double out = 0;
        check(hyb_stokes_residual_norm(h_, detail::State3(rhs).f, detail::State3(x).f, level, &out));
        return out;
    }
    double pressure_mean(const ScalarFunction& p, int level) {
        double out = 0;
        check(hyb_stokes_pressure_mean(h_, p.handle(), level, &out));
        return out;
    }

  private:
    static hyb_stokes* create(DistributedDomain& d, int lo, int hi, const BoundaryConditions& bu,
                              const BoundaryConditions& bp, bool project, double omega) {
        std::vector<int32_t> mu, mp;
        std::vector<uint8_t> fu, fp;
        detail::bc_arrays(bu, mu, fu);
        detail::bc_arrays(bp, mp, fp);
        hyb_stokes* h = nullptr;
        check(hyb_stokes_create(d.handle(), lo, hi, mu.data(), fu.data(), int(mu.size()), mp.data(), fp.data(),
                                int(mp.size()), 1, project ? 1 : 0, omega, &h));
        return h;
    }
    hyb_stokes* h_;
    StokesSystem sys_;
    int min_, max_;
};

} // namespace hytegrid_b200
