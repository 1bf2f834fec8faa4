// TEST INFRASTRUCTURE ONLY -- never part of the product path.
//
// Plain-C adapter around the UNMODIFIED reference library (compiled from
// /root/reference/proj/src/*.cpp by oracle/Makefile with
// -Dhytegrid=hytegrid_ref, output only under oracle/_ref/). Used by tests/
// to pin the C restatement (oracle/hyteg_oracle.c), to generate the golden
// fixtures in tests/golden/, and by bench.py --impl reference as the CPU
// baseline. Values cross this boundary as owned-DoF vectors in GlobalDoFMap
// order (primitives by ID, each in for_each_owned order), filled per
// primitive so no global std::map is built.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "hytegrid/balancing.hpp"
#include "hytegrid/function.hpp"
#include "hytegrid/meshgen.hpp"
#include "hytegrid/numbering.hpp"
#include "hytegrid/operators.hpp"
#include "hytegrid/solvers.hpp"

using namespace hytegrid;

namespace {

thread_local std::string g_err;

template <class F> int guard(F&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 2;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 4;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 7;
    }
}

struct Session {
    SetupGraph setup;
    std::unique_ptr<DistributedDomain> dom;
    std::unique_ptr<Controller> ctl;
    BoundaryConditions bc;
    int min_level = 0, max_level = 0;
    FunctionKind kind = FunctionKind::P1;
    std::vector<std::unique_ptr<ScalarFunction>> f;
    std::unique_ptr<StencilOperator> A;
    // composed V-cycle scratch (GridHierarchy's r_, b_, e_)
    std::unique_ptr<ScalarFunction> r, b, e;
};

std::vector<PrimitiveID> ids_sorted(const DistributedDomain& dom) {
    std::vector<PrimitiveID> ids;
    for (int r = 0; r < dom.ranks(); ++r)
        for (const auto& [id, p] : dom.graph(r).local) ids.push_back(id);
    std::sort(ids.begin(), ids.end());
    return ids;
}

void move_owned(Session& s, int fi, int level, double* data, bool to_field) {
    ScalarFunction& fn = *s.f.at(size_t(fi));
    size_t pos = 0;
    for (const PrimitiveID id : ids_sorted(*s.dom)) {
        const Primitive& p = s.dom->primitive(id);
        auto& vals = fn.values(id, level);
        for_each_owned(fn.kind(), p.kind, p.info, level, fn.layout(), [&](std::size_t slot) {
            if (to_field) vals[slot] = data[pos];
            else data[pos] = vals[slot];
            ++pos;
        });
    }
}

const std::uint8_t kSmooth = flag_bit(DoFFlag::INNER) | flag_bit(DoFFlag::NEUMANN);
const std::uint8_t kDir = flag_bit(DoFFlag::DIRICHLET);

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_meshgen(const char* kind, const double* p, char* out, int64_t cap, int64_t* len) {
    return guard([&] {
        const std::string k(kind);
        std::string t;
        if (k == "unit_triangle") t = meshgen::unit_triangle();
        else if (k == "unit_square") t = meshgen::unit_square();
        else if (k == "unit_square_reversed") t = meshgen::unit_square_reversed();
        else if (k == "square_ring8") t = meshgen::square_ring8();
        else if (k == "channel") t = meshgen::channel(int(p[0]), int(p[1]), p[2], p[3]);
        else if (k == "annulus") t = meshgen::annulus(int(p[0]), int(p[1]), p[2], p[3]);
        else throw std::invalid_argument("unknown mesh kind");
        *len = int64_t(t.size());
        if (cap > int64_t(t.size())) std::memcpy(out, t.c_str(), t.size() + 1);
    });
}

// rank per primitive ID from the reference partitioners (src/balancing.cpp)
int ref_partition(const char* mesh, int ranks, int partitioner, int weight_level, int* out) {
    return guard([&] {
        const SetupGraph setup = build_setup_graph(parse_mesh_string(mesh));
        const Assignment a = partitioner == 1
                                 ? partition_greedy_edgecut(setup, weighted_graph(setup, FunctionKind::P1, weight_level),
                                                            ranks)
                                 : partition_round_robin(setup, ranks);
        for (const auto& [id, r] : a) out[id.value] = r;
    });
}

// partitioner: 0 round robin, 1 greedy edge cut (weights at weight_level)
int ref_create_kind(const char* mesh, int ranks, int partitioner, int weight_level, int min_level, int max_level,
                    const int* bc_markers, const uint8_t* bc_flags, int nbc, int nfuncs, int kind, void** out) {
    return guard([&] {
        auto s = std::make_unique<Session>();
        s->kind = FunctionKind(kind);
        s->setup = build_setup_graph(parse_mesh_string(mesh));
        const Assignment a = partitioner == 1
                                 ? partition_greedy_edgecut(s->setup,
                                                            weighted_graph(s->setup, FunctionKind::P1, weight_level),
                                                            ranks)
                                 : partition_round_robin(s->setup, ranks);
        s->dom = std::make_unique<DistributedDomain>(s->setup, a, ranks);
        s->ctl = std::make_unique<Controller>(*s->dom);
        for (int i = 0; i < nbc; ++i) s->bc.marker_flag[bc_markers[i]] = DoFFlag(bc_flags[i]);
        s->min_level = min_level;
        s->max_level = max_level;
        for (int i = 0; i < nfuncs; ++i) {
            s->f.push_back(std::make_unique<ScalarFunction>("f" + std::to_string(i), *s->dom, s->kind,
                                                            min_level, max_level, s->bc));
            register_function(*s->ctl, *s->f.back());
        }
        s->A = std::make_unique<StencilOperator>(*s->dom, Form::LAPLACE, s->kind, min_level, max_level, s->bc);
        *out = s.release();
    });
}

int ref_create(const char* mesh, int ranks, int partitioner, int weight_level, int min_level, int max_level,
               const int* bc_markers, const uint8_t* bc_flags, int nbc, int nfuncs, void** out) {
    return ref_create_kind(mesh, ranks, partitioner, weight_level, min_level, max_level, bc_markers, bc_flags, nbc,
                           nfuncs, 0, out);
}

void ref_destroy(void* s) { delete static_cast<Session*>(s); }

int64_t ref_owned(void* sp, int level) {
    Session& s = *static_cast<Session*>(sp);
    int64_t n = 0;
    for (const PrimitiveID id : ids_sorted(*s.dom)) {
        const Primitive& p = s.dom->primitive(id);
        for_each_owned(s.kind, p.kind, p.info, level, row_major_layout(), [&](std::size_t) { ++n; });
    }
    return n;
}

int ref_set(void* s, int fi, int level, const double* data) {
    return guard([&] { move_owned(*static_cast<Session*>(s), fi, level, const_cast<double*>(data), true); });
}
int ref_get(void* s, int fi, int level, double* data) {
    return guard([&] { move_owned(*static_cast<Session*>(s), fi, level, data, false); });
}
int ref_flags(void* sp, int fi, int level, uint8_t* out) {
    return guard([&] {
        Session& s = *static_cast<Session*>(sp);
        size_t pos = 0;
        for (const PrimitiveID id : ids_sorted(*s.dom)) {
            const Primitive& p = s.dom->primitive(id);
            const auto& fl = s.f.at(size_t(fi))->flags(id, level);
            for_each_owned(s.kind, p.kind, p.info, level, row_major_layout(),
                           [&](std::size_t slot) { out[pos++] = fl[slot]; });
        }
    });
}
// owned DoF coordinates (for_each_owned_coord), x/y interleaved
int ref_coords(void* sp, int level, double* xy) {
    return guard([&] {
        Session& s = *static_cast<Session*>(sp);
        size_t pos = 0;
        for (const PrimitiveID id : ids_sorted(*s.dom)) {
            const Primitive& p = s.dom->primitive(id);
            for_each_owned_coord(s.kind, p.kind, p.info, level, row_major_layout(),
                                 [&](std::size_t, double x, double y) {
                                     xy[2 * pos] = x;
                                     xy[2 * pos + 1] = y;
                                     ++pos;
                                 });
        }
    });
}

int ref_sync(void* sp, int fi, int level) {
    return guard([&] {
        Session& s = *static_cast<Session*>(sp);
        sync_all(*s.ctl, *s.f.at(size_t(fi)), level);
    });
}

// sync(c, f, level, directions) (src/function.cpp:234-237)
int ref_sync_dirs(void* sp, int fi, int level, const int* dirs, int n) {
    return guard([&] {
        Session& s = *static_cast<Session*>(sp);
        std::vector<Direction> d;
        for (int i = 0; i < n; ++i) d.push_back(Direction(dirs[i]));
        sync(*s.ctl, *s.f.at(size_t(fi)), level, std::span<const Direction>(d));
    });
}

// values(id, level): the primitive's raw slots; set writes them
int ref_values(void* sp, int fi, uint64_t prim, int level, double* out, int64_t cap, int64_t* len) {
    return guard([&] {
        Session& s = *static_cast<Session*>(sp);
        auto& v = s.f.at(size_t(fi))->values(PrimitiveID{prim}, level);
        *len = int64_t(v.size());
        if (out && cap >= int64_t(v.size())) std::memcpy(out, v.data(), v.size() * 8);
    });
}
int ref_set_values(void* sp, int fi, uint64_t prim, int level, const double* in, int64_t n) {
    return guard([&] {
        Session& s = *static_cast<Session*>(sp);
        auto& v = s.f.at(size_t(fi))->values(PrimitiveID{prim}, level);
        if (int64_t(v.size()) != n) throw std::invalid_argument("ref_set_values: size");
        std::memcpy(v.data(), in, size_t(n) * 8);
    });
}

// The reference's own DataCallbacks::serialize of one primitive's field data
// (src/field.cpp:157-166): the checkpoint / migration byte format.
int ref_serialize(void* sp, int fi, uint64_t prim, uint8_t* out, int64_t cap, int64_t* len) {
    return guard([&] {
        Session& s = *static_cast<Session*>(sp);
        ScalarFunction& fn = *s.f.at(size_t(fi));
        const Primitive& p = s.dom->primitive(PrimitiveID{prim});
        MessageBuffer buf;
        s.dom->callbacks(fn.handle()).serialize(primitive_data(p, fn.handle()), buf);
        *len = int64_t(buf.size());
        if (out && cap >= int64_t(buf.size())) std::memcpy(out, buf.bytes().data(), buf.size());
    });
}

// replace the session's operator by one of `form` (include/hytegrid/elements.hpp:17-25)
int ref_set_form(void* sp, int form) {
    return guard([&] {
        Session& s = *static_cast<Session*>(sp);
        if (form < 0 || form > 6) throw std::invalid_argument("ref_set_form: bad form");
        s.A = std::make_unique<StencilOperator>(*s.dom, Form(form), s.kind, s.min_level, s.max_level,
                                                s.bc);
    });
}

int ref_apply(void* sp, int src, int dst, int level, uint8_t mask) {
    return guard([&] {
        Session& s = *static_cast<Session*>(sp);
        apply(*s.A, *s.ctl, *s.f.at(size_t(src)), *s.f.at(size_t(dst)), level, mask);
    });
}

// r = rhs - A x, composed exactly as GridHierarchy (src/solvers.cpp:418-419)
int ref_residual(void* sp, int rhs, int x, int r, int level) {
    return guard([&] {
        Session& s = *static_cast<Session*>(sp);
        apply(*s.A, *s.ctl, *s.f.at(size_t(x)), *s.f.at(size_t(r)), level);
        assign(1.0, *s.f.at(size_t(rhs)), -1.0, *s.f.at(size_t(r)), *s.f.at(size_t(r)), level);
    });
}

int ref_jacobi(void* sp, int rhs, int x, double omega, int level) {
    return guard([&] {
        Session& s = *static_cast<Session*>(sp);
        smooth_jacobi(*s.A, *s.ctl, *s.f.at(size_t(rhs)), *s.f.at(size_t(x)), omega, level);
    });
}

int ref_gs(void* sp, int rhs, int x, int level) {
    return guard([&] {
        Session& s = *static_cast<Session*>(sp);
        smooth_gs(*s.A, *s.ctl, *s.f.at(size_t(rhs)), *s.f.at(size_t(x)), level);
    });
}

int ref_restrict(void* sp, int fine, int coarse, int lc, uint8_t mask) {
    return guard([&] {
        Session& s = *static_cast<Session*>(sp);
        restrict_to_coarse(*s.ctl, *s.f.at(size_t(fine)), *s.f.at(size_t(coarse)), lc, mask);
    });
}

int ref_prolongate(void* sp, int coarse, int fine, int lc, uint8_t mask) {
    return guard([&] {
        Session& s = *static_cast<Session*>(sp);
        prolongate(*s.ctl, *s.f.at(size_t(coarse)), *s.f.at(size_t(fine)), lc, mask);
    });
}

int ref_assign(void* sp, double alpha, int x1, double beta, int x2, int dst, int level, uint8_t mask) {
    return guard([&] {
        Session& s = *static_cast<Session*>(sp);
        assign(alpha, *s.f.at(size_t(x1)), beta, *s.f.at(size_t(x2)), *s.f.at(size_t(dst)), level, mask);
    });
}

int ref_add_scaled(void* sp, int dst, double gamma, int y, int level, uint8_t mask) {
    return guard([&] {
        Session& s = *static_cast<Session*>(sp);
        add_scaled(*s.f.at(size_t(dst)), gamma, *s.f.at(size_t(y)), level, mask);
    });
}

int ref_dot(void* sp, int a, int b, int level, double* out) {
    return guard([&] {
        Session& s = *static_cast<Session*>(sp);
        *out = dot(*s.f.at(size_t(a)), *s.f.at(size_t(b)), level);
    });
}

// stencil readback in the reference's table order; face: 7 terms + diag;
// edge: line terms + diag; vertex: terms + diag
int ref_stencil(void* sp, uint64_t id, int level, double* out, int* len) {
    return guard([&] {
        Session& s = *static_cast<Session*>(sp);
        const StencilTable& t = s.A->table(PrimitiveID{id}, level);
        int n = 0;
        const Primitive& p = s.dom->primitive(PrimitiveID{id});
        if (p.kind == PrimitiveKind::FACE) {
            for (const auto& e : t.face.at(DoFGroup::VERTEX)) out[n++] = e.coeff;
            out[n++] = t.face_diag.at(DoFGroup::VERTEX);
        } else if (p.kind == PrimitiveKind::EDGE) {
            for (const auto& e : t.edge_line) out[n++] = e.coeff;
            out[n++] = t.edge_line_diag;
        } else {
            for (const auto& e : t.vertex) out[n++] = e.coeff;
            out[n++] = t.vertex_diag;
        }
        *len = n;
    });
}

// Composed Jacobi V-cycle oracle: GridHierarchy::cycle
// (src/solvers.cpp:406-428) line by line with smooth_jacobi(omega) in place of
// smooth_gs, any min level (>= 0), coarse CG (cg_solve) to coarse_tol on the
// constrained assembled min-level matrix. residuals[0..ncycles] as in
// GridHierarchy::solve (src/solvers.cpp:451-465) with tol = 0.
namespace {
struct Composed {
    Session& s;
    int min_level;
    int nu1, nu2;
    double omega, tol;
    GlobalDoFMap cmap;
    std::vector<uint8_t> cflags;
    SparseMatrix cA;
    Composed(Session& s_, int minl, int a, int b, double w, double t)
        : s(s_), min_level(minl), nu1(a), nu2(b), omega(w), tol(t),
          cmap(*s_.dom, FunctionKind::P1, minl), cflags(cmap.gather_flags(*s_.r)),
          cA(assemble_global_sparse(*s_.A, minl, cmap)) {
        std::vector<double> zero(cA.rows(), 0.0);
        constrain_dirichlet(cA, zero, cflags);
    }
    void coarse(ScalarFunction& rhs, ScalarFunction& x) {
        const int L = min_level;
        apply(*s.A, *s.ctl, x, *s.r, L);
        assign(1.0, rhs, -1.0, *s.r, *s.r, L);
        const std::vector<double> b = cmap.gather(*s.r);
        std::vector<double> e(b.size(), 0.0);
        const SolveReport rep = cg_solve(cA, b, e, tol, static_cast<int>(b.size()) + 100);
        if (!rep.converged) throw std::runtime_error("vcycle: coarse CG did not converge\n" + rep.history());
        cmap.scatter(e, *s.r);
        add_scaled(x, 1.0, *s.r, L, kSmooth);
    }
    void cycle(ScalarFunction& rhs, ScalarFunction& x, int L) {
        assign(1.0, rhs, 0.0, rhs, x, L, kDir);
        if (L == min_level) {
            coarse(rhs, x);
            return;
        }
        for (int i = 0; i < nu1; ++i) smooth_jacobi(*s.A, *s.ctl, rhs, x, omega, L);
        apply(*s.A, *s.ctl, x, *s.r, L);
        assign(1.0, rhs, -1.0, *s.r, *s.r, L);
        restrict_to_coarse(*s.ctl, *s.r, *s.b, L - 1);
        interpolate(*s.b, [](double, double) { return 0.0; }, L - 1, kDir);
        interpolate(*s.e, [](double, double) { return 0.0; }, L - 1);
        cycle(*s.b, *s.e, L - 1);
        prolongate(*s.ctl, *s.e, *s.r, L - 1, kSmooth);
        add_scaled(x, 1.0, *s.r, L, kSmooth);
        for (int i = 0; i < nu2; ++i) smooth_jacobi(*s.A, *s.ctl, rhs, x, omega, L);
    }
    double resnorm(ScalarFunction& rhs, ScalarFunction& x, int L) {
        apply(*s.A, *s.ctl, x, *s.r, L);
        assign(1.0, rhs, -1.0, *s.r, *s.r, L);
        return norm2(*s.r, L);
    }
};
} // namespace

int ref_vcycle_jacobi(void* sp, int rhs, int x, int level, int nu1, int nu2, double omega, double coarse_tol,
                      int ncycles, double* residuals) {
    return guard([&] {
        Session& s = *static_cast<Session*>(sp);
        if (!s.r) {
            s.r = std::make_unique<ScalarFunction>("mg.r", *s.dom, FunctionKind::P1, s.min_level, s.max_level, s.bc);
            s.b = std::make_unique<ScalarFunction>("mg.b", *s.dom, FunctionKind::P1, s.min_level, s.max_level, s.bc);
            s.e = std::make_unique<ScalarFunction>("mg.e", *s.dom, FunctionKind::P1, s.min_level, s.max_level, s.bc);
            register_function(*s.ctl, *s.r);
            register_function(*s.ctl, *s.b);
            register_function(*s.ctl, *s.e);
        }
        Composed c(s, s.min_level, nu1, nu2, omega, coarse_tol);
        ScalarFunction& R = *s.f.at(size_t(rhs));
        ScalarFunction& X = *s.f.at(size_t(x));
        residuals[0] = c.resnorm(R, X, level);
        for (int k = 0; k < ncycles; ++k) {
            c.cycle(R, X, level);
            residuals[k + 1] = c.resnorm(R, X, level);
        }
    });
}

// the reference's own GridHierarchy (hybrid Gauss-Seidel, min level >= 1)
int ref_gridhierarchy_solve(void* sp, int rhs, int x, int level, double tol, int max_cycles, int nu1, int nu2,
                            double* residuals, int* n_out) {
    return guard([&] {
        Session& s = *static_cast<Session*>(sp);
        GridHierarchy mg(*s.dom, *s.ctl, Form::LAPLACE, s.min_level, s.max_level, s.bc);
        const SolveReport rep =
            mg.solve(*s.f.at(size_t(rhs)), *s.f.at(size_t(x)), level, tol, max_cycles, nu1, nu2);
        for (size_t i = 0; i < rep.residuals.size(); ++i) residuals[i] = rep.residuals[i];
        *n_out = int(rep.residuals.size());
    });
}

// keyed U[lo, hi] of the device generator (the restatement's og_keyed_uniform)
// written straight into function fi at `level` (no host vector in GlobalDoFMap
// order: config 2 at level 10 is 268 M DoFs)
namespace {
uint64_t kmix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
} // namespace
int ref_fill_keyed(void* sp, int fi, int level, uint64_t seed, uint64_t stream, double lo, double hi) {
    return guard([&] {
        Session& s = *static_cast<Session*>(sp);
        ScalarFunction& fn = *s.f.at(size_t(fi));
        const uint64_t sk = kmix(kmix(seed) ^ (stream * 0xD1B54A32D192ED03ull));
        const int n = 1 << level;
        auto u = [&](uint64_t key) { return lo + (hi - lo) * (double(kmix(sk ^ kmix(key)) >> 11) * 0x1p-53); };
        for (const PrimitiveID id : ids_sorted(*s.dom)) {
            const Primitive& p = s.dom->primitive(id);
            auto& vals = fn.values(id, level);
            const uint64_t base = uint64_t(id.value) << 40;
            int q = 1, r = 1, c = 1; // for_each_owned order: edges k = 1..n-1; faces r = 1..n-2, c = 1..n-1-r
            for_each_owned(FunctionKind::P1, p.kind, p.info, level, fn.layout(), [&](std::size_t slot) {
                if (p.kind == PrimitiveKind::VERTEX) {
                    vals[slot] = u(base);
                } else if (p.kind == PrimitiveKind::EDGE) {
                    vals[slot] = u(base ^ (uint64_t(q) << 20));
                    ++q;
                } else {
                    vals[slot] = u(base ^ (uint64_t(c) << 20) ^ uint64_t(r));
                    if (++c + r > n - 1) {
                        c = 1;
                        ++r;
                    }
                }
            });
        }
    });
}

// diagonal(A, d, level) (include/hytegrid/operators.hpp:125, src/operators.cpp:484-505)
// of a fresh StencilOperator of `form` (0 LAPLACE, 1 MASS) into function d
int ref_diagonal(void* sp, int form, int d, int level) {
    return guard([&] {
        Session& s = *static_cast<Session*>(sp);
        StencilOperator A(*s.dom, form == 1 ? Form::MASS : Form::LAPLACE, s.kind, s.min_level,
                          s.max_level, s.bc);
        diagonal(A, *s.f.at(size_t(d)), level);
    });
}

// The GridHierarchy coarse matrix (constrained_matrix, src/solvers.cpp:358-364):
// assemble_global_sparse + constrain_dirichlet at `level`, as COO in row then
// column order (SparseMatrix row maps); *nnz = entries (size query: cap 0).
int ref_coarse_matrix(void* sp, int level, int64_t* rows, int64_t* cols, double* vals, int64_t cap, int64_t* nnz) {
    return guard([&] {
        Session& s = *static_cast<Session*>(sp);
        GlobalDoFMap map(*s.dom, FunctionKind::P1, level);
        const std::vector<uint8_t> flags = map.gather_flags(*s.f.at(0));
        SparseMatrix M = assemble_global_sparse(*s.A, level, map);
        std::vector<double> zero(M.rows(), 0.0);
        constrain_dirichlet(M, zero, flags);
        int64_t k = 0;
        for (size_t r = 0; r < M.rows(); ++r)
            for (const auto& [c, v] : M.row(r)) {
                if (k < cap) {
                    rows[k] = int64_t(r);
                    cols[k] = int64_t(c);
                    vals[k] = v;
                }
                ++k;
            }
        *nnz = k;
    });
}


// ---- P1-P1-PSPG Stokes (src/solvers.cpp:466-753): the reference's own
// StokesMultigrid, uzawa_smooth and stokes_residual on states rhs (0), x (1)
// and r (2); component 0 u1, 1 u2, 2 p. Velocity and pressure have separate
// boundary conditions (marker -> flag). A solve whose coarse MINRES fails
// returns 3 (runtime_error) with the reference's message and history.
namespace {
struct StokesSession {
    SetupGraph setup;
    std::unique_ptr<DistributedDomain> dom;
    std::unique_ptr<Controller> ctl;
    BoundaryConditions bcu, bcp;
    int min_level = 1, max_level = 1;
    std::unique_ptr<StokesMultigrid> mg;
    std::vector<std::unique_ptr<StokesState>> st; // rhs, x, r
};
ScalarFunction& stokes_comp(StokesState& s, int comp) { return comp == 0 ? s.u1 : comp == 1 ? s.u2 : s.p; }
void stokes_move(StokesSession& s, int state, int comp, int level, double* data, bool to_field) {
    ScalarFunction& fn = stokes_comp(*s.st.at(size_t(state)), comp);
    size_t pos = 0;
    for (const PrimitiveID id : ids_sorted(*s.dom)) {
        const Primitive& p = s.dom->primitive(id);
        auto& vals = fn.values(id, level);
        for_each_owned(FunctionKind::P1, p.kind, p.info, level, fn.layout(), [&](std::size_t slot) {
            if (to_field) vals[slot] = data[pos];
            else data[pos] = vals[slot];
            ++pos;
        });
    }
}
} // namespace

int ref_stokes_create(const char* mesh, int ranks, int partitioner, int weight_level, int min_level, int max_level,
                      const int* bcu_markers, const uint8_t* bcu_flags, int nbcu, const int* bcp_markers,
                      const uint8_t* bcp_flags, int nbcp, int project, double omega, void** out) {
    return guard([&] {
        auto s = std::make_unique<StokesSession>();
        s->setup = build_setup_graph(parse_mesh_string(mesh));
        const Assignment a = partitioner == 1
                                 ? partition_greedy_edgecut(s->setup,
                                                            weighted_graph(s->setup, FunctionKind::P1, weight_level),
                                                            ranks)
                                 : partition_round_robin(s->setup, ranks);
        s->dom = std::make_unique<DistributedDomain>(s->setup, a, ranks);
        s->ctl = std::make_unique<Controller>(*s->dom);
        for (int i = 0; i < nbcu; ++i) s->bcu.marker_flag[bcu_markers[i]] = DoFFlag(bcu_flags[i]);
        for (int i = 0; i < nbcp; ++i) s->bcp.marker_flag[bcp_markers[i]] = DoFFlag(bcp_flags[i]);
        s->min_level = min_level;
        s->max_level = max_level;
        s->mg = std::make_unique<StokesMultigrid>(*s->dom, *s->ctl, min_level, max_level, s->bcu, s->bcp,
                                                  project != 0, omega);
        for (const char* nm : {"rhs", "x", "r"}) {
            s->st.push_back(std::make_unique<StokesState>(nm, *s->dom, min_level, max_level, s->bcu, s->bcp));
            register_state(*s->ctl, *s->st.back());
        }
        *out = s.release();
    });
}
void ref_stokes_destroy(void* s) { delete static_cast<StokesSession*>(s); }
int ref_stokes_set(void* s, int state, int comp, int level, const double* data) {
    return guard([&] {
        stokes_move(*static_cast<StokesSession*>(s), state, comp, level, const_cast<double*>(data), true);
    });
}
int ref_stokes_get(void* s, int state, int comp, int level, double* data) {
    return guard([&] { stokes_move(*static_cast<StokesSession*>(s), state, comp, level, data, false); });
}
int ref_stokes_uzawa(void* sp, int level, double omega) {
    return guard([&] {
        StokesSession& s = *static_cast<StokesSession*>(sp);
        uzawa_smooth(s.mg->system(), *s.ctl, *s.st[0], *s.st[1], level, omega);
    });
}
int ref_stokes_residual(void* sp, int level) {
    return guard([&] {
        StokesSession& s = *static_cast<StokesSession*>(sp);
        stokes_residual(s.mg->system(), *s.ctl, *s.st[0], *s.st[1], *s.st[2], level);
    });
}
int ref_stokes_vcycle(void* sp, int level, int nu1, int nu2) {
    return guard([&] {
        StokesSession& s = *static_cast<StokesSession*>(sp);
        s.mg->vcycle(*s.st[0], *s.st[1], level, nu1, nu2);
    });
}
// residuals: capacity max_cycles + 1; *n_out entries written (also on failure:
// the residuals recorded before the failing cycle)
int ref_stokes_solve(void* sp, int level, double tol, int max_cycles, int nu1, int nu2, double* residuals,
                     int* n_out, int* converged) {
    StokesSession& s = *static_cast<StokesSession*>(sp);
    *n_out = 0;
    return guard([&] {
        const SolveReport rep = s.mg->solve(*s.st[0], *s.st[1], level, tol, max_cycles, nu1, nu2);
        for (size_t i = 0; i < rep.residuals.size(); ++i) residuals[i] = rep.residuals[i];
        *n_out = int(rep.residuals.size());
        *converged = rep.converged ? 1 : 0;
    });
}
int ref_stokes_residual_norm(void* sp, int level, double* out) {
    return guard([&] {
        StokesSession& s = *static_cast<StokesSession*>(sp);
        *out = s.mg->residual_norm(*s.st[0], *s.st[1], level);
    });
}
int ref_stokes_pressure_mean(void* sp, int level, double* out) {
    return guard([&] {
        StokesSession& s = *static_cast<StokesSession*>(sp);
        *out = s.mg->pressure_mean(s.st[1]->p, level);
    });
}
// the assembled, constrained monolithic min-level matrix (constrained_stokes_matrix,
// src/solvers.cpp:578-592) as COO (size query: cap 0)
int ref_stokes_matrix(void* sp, int level, int64_t* rows, int64_t* cols, double* vals, int64_t cap, int64_t* nnz) {
    return guard([&] {
        StokesSession& s = *static_cast<StokesSession*>(sp);
        GlobalDoFMap map(*s.dom, FunctionKind::P1, level);
        const auto fu = map.gather_flags(s.st[0]->u1);
        const auto fp = map.gather_flags(s.st[0]->p);
        SparseMatrix M = assemble_stokes_sparse(s.mg->system(), level, map, fu, fp);
        std::vector<double> zero(M.rows(), 0.0);
        std::vector<std::uint8_t> f3(fu);
        f3.insert(f3.end(), fu.begin(), fu.end());
        f3.insert(f3.end(), fp.begin(), fp.end());
        constrain_dirichlet(M, zero, f3);
        int64_t k = 0;
        for (size_t r = 0; r < M.rows(); ++r)
            for (const auto& [c, v] : M.row(r)) {
                if (k < cap) {
                    rows[k] = int64_t(r);
                    cols[k] = int64_t(c);
                    vals[k] = v;
                }
                ++k;
            }
        *nnz = k;
    });
}
} // extern "C"

// ---- Controller::sync with a tracing PackInfo (src/communication.cpp:126-173) ----
// Every message is (sender, receiver, direction, level) as four u64; every
// unpack is logged as (receiver, sender, direction, level) + the message.
namespace {
struct TracePack : PackInfo {
    std::vector<int64_t>* log = nullptr;
    void pack(const Primitive& sender, PrimitiveID receiver, Direction dir, int level,
              MessageBuffer& out) const override {
        out.put_u64(sender.id.value);
        out.put_u64(receiver.value);
        out.put_u64(uint64_t(dir));
        out.put_u64(uint64_t(level));
    }
    void unpack(Primitive& receiver, PrimitiveID sender, Direction dir, int level, MessageBuffer& in) const override {
        const int64_t a = int64_t(in.get_u64()), b = int64_t(in.get_u64()), c = int64_t(in.get_u64()),
                      d = int64_t(in.get_u64());
        log->insert(log->end(), {int64_t(receiver.id.value), int64_t(sender.value), int64_t(dir), int64_t(level), a,
                                 b, c, d});
    }
};
} // namespace
extern "C" int ref_controller_trace(const char* mesh, int ranks, int partitioner, int weight_level, int level,
                                    const int* dirs, int n, int64_t* out, int64_t cap, int64_t* len) {
    return guard([&] {
        const SetupGraph setup = build_setup_graph(parse_mesh_string(mesh));
        const Assignment a = partitioner == 1
                                 ? partition_greedy_edgecut(setup, weighted_graph(setup, FunctionKind::P1, weight_level),
                                                            ranks)
                                 : partition_round_robin(setup, ranks);
        DistributedDomain dom(setup, a, ranks);
        Controller ctl(dom);
        std::vector<int64_t> log;
        auto info = std::make_shared<TracePack>();
        info->log = &log;
        ctl.register_pack_info(7, info);
        std::vector<Direction> d;
        for (int i = 0; i < n; ++i) d.push_back(Direction(dirs[i]));
        ctl.sync(7, level, std::span<const Direction>(d));
        *len = int64_t(log.size());
        for (int64_t i = 0; i < *len && i < cap; ++i) out[i] = log[size_t(i)];
    });
}
