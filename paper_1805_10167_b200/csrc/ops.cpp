// Operations on device-resident functions, with the reference's argument
// checks and exception types (reference src/operators.cpp:322-505,
// src/solvers.cpp:22-204, 385-465, src/function.cpp:11-241).
#include <cstdlib>
#include <algorithm>
#include <cmath>
#include <cstring>

#include "coarse.hpp"
#include "domain.hpp"

namespace hyb {

namespace {

constexpr uint8_t kSmoothMask = INNER | NEUMANN;
constexpr uint8_t kDirichletMask = DIRICHLET;

void check_op_function(const Operator& A, const Function& f, int level, const char* what, bool check_bc) {
    if (&f.domain() != &A.domain()) throw InvalidArgument(std::string(what) + ": function lives on a different domain");
    if (f.kind() != A.kind()) throw InvalidArgument(std::string(what) + ": function kind differs from the operator");
    if (level < f.min_level() || level > f.max_level() || level < A.min_level() || level > A.max_level())
        throw OutOfRange(std::string(what) + ": level " + std::to_string(level) + " outside the allocated range");
    if (check_bc && !(f.bc() == A.bc()))
        throw InvalidArgument(std::string(what) + ": boundary conditions differ from the operator's");
}

void check_pair(const char* op, const Function& a, const Function& b, int level) {
    a.check_level(level, op);
    b.check_level(level, op);
    if (&a.domain() != &b.domain())
        throw InvalidArgument(std::string(op) + ": '" + a.name() + "' and '" + b.name() + "' live on different domains");
    if (a.kind() != b.kind())
        throw InvalidArgument(std::string(op) + ": '" + a.name() + "' and '" + b.name() +
                              "' have different function kinds");
}

// operations this engine provides for P1 only (the reference's level
// transfers are P1-only too, src/solvers.cpp:24-25)
void require_p1(const Function& f, const char* what) {
    if (f.kind() != KIND_P1) throw InvalidArgument(std::string(what) + ": provided for P1 functions");
}

// zero diagonal on a P2 row a smoother would update (src/operators.cpp:457-458)
void check_diagonals_p2(const Operator& A, const Function& x, int level, const char* what) {
    Domain& d = A.domain();
    const MacroGraph& g = d.graph();
    const auto& h = A.host_p2_diag(level);
    size_t pos = 0;
    const int n = 1 << level;
    for (size_t i = 0; i < d.local_faces().size(); ++i, pos += 4)
        for (int k = 0; k < 4; ++k)
            if (n >= 2 && h[pos + size_t(k)] == 0.0) throw RuntimeError(std::string(what) + ": zero diagonal entry");
    for (size_t i = 0; i < d.local_edges().size(); ++i, pos += 2) {
        if (x.bc().flag_for(g.edges[g.edge_index(d.local_edges()[i])].marker) & DIRICHLET) continue;
        if ((n >= 2 && h[pos] == 0.0) || h[pos + 1] == 0.0)
            throw RuntimeError(std::string(what) + ": zero diagonal entry");
    }
    for (size_t i = 0; i < d.local_verts().size(); ++i, ++pos)
        if (!(x.bc().flag_for(g.vertices[d.local_verts()[i]].marker) & DIRICHLET) && h[pos] == 0.0)
            throw RuntimeError(std::string(what) + ": zero diagonal entry");
}

void check_transfer(const Function& coarse, const Function& fine, int lc, const char* what) {
    if (coarse.kind() != KIND_P1 || fine.kind() != KIND_P1) // reference src/solvers.cpp:24-25
        throw InvalidArgument(std::string(what) + ": level transfers are defined for P1");
    if (&coarse.domain() != &fine.domain())
        throw InvalidArgument(std::string(what) + ": functions live on different domains");
    if (lc < coarse.min_level() || lc > coarse.max_level() || lc + 1 < fine.min_level() || lc + 1 > fine.max_level())
        throw OutOfRange(std::string(what) + ": level pair (" + std::to_string(lc) + ", " + std::to_string(lc + 1) +
                         ") outside the functions' level ranges");
}

// zero diagonal on a row that a smoother would update -> runtime_error
// (reference src/operators.cpp:457-458)
bool zero_diagonal_row_impl(const Operator& A, const Function& x, int level) {
    Domain& d = A.domain();
    const MacroGraph& g = d.graph();
    const int n = 1 << level;
    const auto& hf = A.host_face_coef(level);
    if (n >= 3)
        for (size_t i = 0; i < d.local_faces().size(); ++i)
            if (hf[i * 8 + 7] == 0.0) return true;
    const auto& he = A.host_edge_coef(level);
    if (n >= 2)
        for (size_t i = 0; i < d.local_edges().size(); ++i)
            if (!(x.bc().flag_for(g.edges[g.edge_index(d.local_edges()[i])].marker) & DIRICHLET) && he[i * 8 + 7] == 0.0)
                return true;
    const auto& hv = A.host_vtx_coef(level);
    size_t pos = 0;
    for (uint64_t id : d.local_verts()) {
        const MacroVertex& v = g.vertices[id];
        pos += 1 + v.edges.size();
        if (!(x.bc().flag_for(v.marker) & DIRICHLET) && hv[pos] == 0.0)
            return true;
        pos += 1;
    }
    return false;
}

void check_diagonals(const Operator& A, const Function& x, int level, const char* what) {
    if (zero_diagonal_row_impl(A, x, level)) throw RuntimeError(std::string(what) + ": zero diagonal entry");
}

} // namespace

bool zero_diagonal_row(const Operator& A, const Function& x, int level) { return zero_diagonal_row_impl(A, x, level); }

namespace {
// The ghost refresh of x and one stencil launch. With other ranks' ghosts in
// play (Domain::overlap_active) the launch is split: primitives whose ghosts
// all have same-rank owners run while the transfers are in flight, the others
// after the receive half of the refresh (the paper's Algorithm 3; the
// reference itself syncs first, src/operators.cpp:390). Every row is
// computed from the same values either way: bitwise the unsplit launch.
// `timer` brackets the stencil launch(es) only, not the refresh (as before the split)
template <class Launch>
void synced_launch(Domain& d, Function& x, int level, const LevelTables& t, const char* timer, Launch launch) {
    if (!d.overlap_active(x, level)) {
        d.sync(x, level);
        d.timer_begin(timer);
        launch(t);
        d.timer_end();
        return;
    }
    d.sync_begin(x, level);
    d.timer_begin(timer);
    launch(d.overlap_tables(t, x, level, 0));
    d.sync_end(x, level);
    launch(d.overlap_tables(t, x, level, 1));
    d.timer_end();
}
} // namespace

void apply(const Operator& A, Function& src, Function& dst, int level, uint8_t mask) {
    check_op_function(A, src, level, "apply", false);
    check_op_function(A, dst, level, "apply", true);
    if (&src == &dst) throw InvalidArgument("apply: src and dst must be distinct functions");
    Domain& d = A.domain();
    if (A.kind() == KIND_P2) {
        d.sync(src, level); // full schedule first (reference src/operators.cpp:390)
        launch_p2(P2_APPLY, A.tables_p2(level), dst.flags(), src.data(level), src.data(level), dst.data(level), 0.0,
                  mask, d.stream());
        return;
    }
    const LevelTables t = A.tables(level);
    // face interiors, then edge/vertex rows as the same launch's trailing CTAs
    synced_launch(d, src, level, t, "apply", [&](const LevelTables& tt) {
        launch_stencil(ST_APPLY, tt, dst.flags(), src.data(level), src.data(level), dst.data(level), 0.0, mask,
                       d.stream(), 3);
    });
}

void residual(const Operator& A, Function& rhs, Function& x, Function& r, int level) {
    check_op_function(A, rhs, level, "residual", false);
    check_op_function(A, x, level, "residual", false);
    check_op_function(A, r, level, "residual", true);
    if (&x == &r || &rhs == &r) throw InvalidArgument("residual: r must be distinct from x and rhs");
    require_p1(x, "residual (fused)");
    Domain& d = A.domain();
    const LevelTables t = A.tables(level);
    synced_launch(d, x, level, t, "residual", [&](const LevelTables& tt) {
        launch_stencil(ST_RESIDUAL, tt, r.flags(), x.data(level), rhs.data(level), r.data(level), 0.0, ALL_FLAGS,
                       d.stream(), 3);
    });
}

void smooth_jacobi(const Operator& A, Function& rhs, Function& x, double omega, int level, double* dotp, int target) {
    check_op_function(A, rhs, level, "smooth_jacobi", true);
    check_op_function(A, x, level, "smooth_jacobi", true);
    if (&rhs == &x) throw InvalidArgument("smooth_jacobi: rhs and x must be distinct functions");
    if (A.kind() == KIND_P2) {
        if (dotp) throw InvalidArgument("smooth_jacobi: fused dot provided for P1");
        check_diagonals_p2(A, x, level, "smooth_jacobi");
        Domain& d = A.domain();
        d.sync(x, level);
        DevMem& next = d.jacobi_scratch(level, KIND_P2);
        launch_p2(P2_JACOBI, A.tables_p2(level), x.flags(), x.data(level), rhs.data(level), next.as<double>(), omega,
                  ALL_FLAGS, d.stream());
        x.arena(level).swap(next);
        return;
    }
    check_diagonals(A, x, level, "smooth_jacobi");
    Domain& d = A.domain();
    DevMem& next = target == 2 ? d.jacobi_scratch2(level) : d.jacobi_scratch(level);
    // pending write-back of the reference (src/operators.cpp:435-468) is a
    // second buffer here: read x, write x', swap.
    const LevelTables t = A.tables(level);
    synced_launch(d, x, level, t, "jacobi", [&](const LevelTables& tt) {
        launch_stencil(ST_JACOBI, tt, x.flags(), x.data(level), rhs.data(level), next.as<double>(), omega, ALL_FLAGS,
                       d.stream(), 3, dotp);
    });
    x.arena(level).swap(next);
}

namespace {
// measured on config 2, L10 (one B200): the pass 2.95 ms against 2.10 ms for two
// sweeps -- issue-bound (ncu: 2.5 IPC, 63% issue slots busy, ~480 instructions per
// warp and row step for x1 at three columns and x2 at two, 96 registers with
// spills), so it is off unless asked for (hyb_tuning("jacobi2_min_n", n))
int g_jacobi2_min_n = 1 << 30;
} // namespace

int jacobi2_min_n() { return g_jacobi2_min_n; }
namespace {
int64_t g_mega_dofs_per_cta = 16384;
}
int64_t mega_dofs_per_cta_default() { return g_mega_dofs_per_cta; }
void set_mega_dofs_per_cta_default(int64_t v) { g_mega_dofs_per_cta = v; }
void set_jacobi2_min_n(int n) { g_jacobi2_min_n = n; }

// Two sweeps, x0 -> x1 -> x2: the face pass forms x1 in registers and writes x2
// two or more away from every border plus x1 on the two layers next to the
// borders; the edges' and vertices' first sweep runs as its trailing CTAs into
// the scratch arena; after a ghost refresh of that arena the layer pass and the
// edges' / vertices' second sweep complete x2. Every value is computed from the
// same operands in the same order as by two smooth_jacobi calls: bitwise.
void smooth_jacobi2(const Operator& A, Function& rhs, Function& x, double omega, int level) {
    check_op_function(A, rhs, level, "smooth_jacobi", true);
    check_op_function(A, x, level, "smooth_jacobi", true);
    if (&rhs == &x) throw InvalidArgument("smooth_jacobi: rhs and x must be distinct functions");
    Domain& d = A.domain();
    if (A.kind() != KIND_P1 || (1 << level) < jacobi2_min_n()) {
        smooth_jacobi(A, rhs, x, omega, level);
        smooth_jacobi(A, rhs, x, omega, level, nullptr, 2); // lands where the pass would put it
        d.swap_scratch(level);
        return;
    }
    check_diagonals(A, x, level, "smooth_jacobi");
    d.sync(x, level);
    const LevelTables t = A.tables(level);
    DevMem& y1 = d.jacobi_scratch(level);
    DevMem& y2 = d.jacobi_scratch2(level);
    d.timer_begin("jacobi2");
    launch_jacobi2(t, x.flags(), x.data(level), rhs.data(level), y1.as<double>(), y2.as<double>(), omega, d.stream());
    d.sync_arena(KIND_P1, level, y1.as<double>());
    launch_jacobi2_finish(t, x.flags(), y1.as<double>(), rhs.data(level), y2.as<double>(), omega, d.stream());
    d.timer_end();
    x.arena(level).swap(y2);
}

namespace {
// per-primitive partials already in `part` (faces: `slots` CTA partials each
// in scratch) -> the reference's fold over the global vector -> host
void finish_dot_dev(Domain& d, const LevelTables& t, const double* u, const double* v, const double* scratch,
                    int slots, double* part, double* out) {
    launch_partials_finish(t, u, v, scratch, slots, part, d.stream());
    const int64_t np = int64_t(d.graph().size());
    d.allreduce_sum(part, np);
    launch_combine_tree(0, part, np, out, d.stream());
}
double to_host(Domain& d, const double* dev) {
    double out = 0.0;
    HYB_CUDA(cudaMemcpyAsync(&out, dev, 8, cudaMemcpyDeviceToHost, d.stream()));
    HYB_CUDA(cudaStreamSynchronize(d.stream()));
    return out;
}
} // namespace

// dst = A src and src.dst in one pass over the faces (PCG's p.Ap): the face
// partials come from the stencil kernel's CTAs (fixed shapes, so the result is
// deterministic and partition invariant, though not bitwise dot()'s order)
double apply_dot(const Operator& A, Function& src, Function& dst, int level) {
    apply_dot_dev(A, src, dst, level, A.domain().scalar_out());
    return to_host(A.domain(), A.domain().scalar_out());
}

void apply_dot_dev(const Operator& A, Function& src, Function& dst, int level, double* out) {
    check_op_function(A, src, level, "apply", false);
    check_op_function(A, dst, level, "apply", true);
    if (&src == &dst) throw InvalidArgument("apply: src and dst must be distinct functions");
    Domain& d = A.domain();
    d.sync(src, level);
    const LevelTables t = A.tables(level);
    const int slots = face_dot_slots(t);
    const int64_t np = int64_t(d.graph().size());
    double* buf = d.partials(np + int64_t(t.nfaces) * slots + 1);
    double* part = buf;
    double* scratch = buf + np;
    HYB_CUDA(cudaMemsetAsync(part, 0, size_t(np) * 8, d.stream()));
    d.timer_begin("apply");
    launch_stencil(ST_APPLY, t, dst.flags(), src.data(level), src.data(level), dst.data(level), 0.0, ALL_FLAGS,
                   d.stream(), 3, scratch);
    d.timer_end();
    finish_dot_dev(d, t, src.data(level), dst.data(level), scratch, slots, part, out);
}

// r = rhs - A x and r.r in one pass over the faces (a solve's residual norm after each cycle):
// the face partials come from the stencil kernel's CTAs, as apply_dot's do
double residual_dot(const Operator& A, Function& rhs, Function& x, Function& r, int level) {
    check_op_function(A, rhs, level, "residual", false);
    check_op_function(A, x, level, "residual", false);
    check_op_function(A, r, level, "residual", true);
    if (&x == &r || &rhs == &r) throw InvalidArgument("residual: r must be distinct from x and rhs");
    require_p1(x, "residual (fused)");
    Domain& d = A.domain();
    d.sync(x, level);
    const LevelTables t = A.tables(level);
    const int slots = face_dot_slots(t);
    const int64_t np = int64_t(d.graph().size());
    double* buf = d.partials(np + int64_t(t.nfaces) * slots + 1);
    double* part = buf;
    double* scratch = buf + np;
    HYB_CUDA(cudaMemsetAsync(part, 0, size_t(np) * 8, d.stream()));
    d.timer_begin("residual");
    launch_stencil(ST_RESIDUAL, t, r.flags(), x.data(level), rhs.data(level), r.data(level), 0.0, ALL_FLAGS,
                   d.stream(), 3, scratch);
    d.timer_end();
    finish_dot_dev(d, t, r.data(level), r.data(level), scratch, slots, part, d.scalar_out());
    return to_host(d, d.scalar_out());
}

// the first weighted-Jacobi sweep of a cycle whose x starts at zero (see
// ST_JACOBI_ZERO): x is neither synced nor read; Dirichlet rows take rhs,
// exactly what the cycle's assign would have put there
void smooth_jacobi_zero(const Operator& A, Function& rhs, Function& x, double omega, int level) {
    check_op_function(A, rhs, level, "smooth_jacobi", true);
    check_op_function(A, x, level, "smooth_jacobi", true);
    if (&rhs == &x) throw InvalidArgument("smooth_jacobi: rhs and x must be distinct functions");
    require_p1(x, "smooth_jacobi (from zero)");
    check_diagonals(A, x, level, "smooth_jacobi");
    Domain& d = A.domain();
    DevMem& next = d.jacobi_scratch(level);
    const LevelTables t = A.tables(level);
    d.timer_begin("jacobi_zero");
    launch_stencil(ST_JACOBI_ZERO, t, x.flags(), nullptr, rhs.data(level), next.as<double>(), omega, ALL_FLAGS,
                   d.stream(), 3);
    d.timer_end();
    x.arena(level).swap(next);
}

// hybrid Gauss-Seidel (reference smooth_gs, src/operators.cpp:423-482): one
// sync, then every primitive in place in lattice order with frozen halos;
// faces (wavefront tiles) and edges/vertices are independent, so the latter
// run on the side stream concurrently.
void smooth_gs(const Operator& A, Function& rhs, Function& x, int level) {
    check_op_function(A, rhs, level, "smooth_gs", true);
    check_op_function(A, x, level, "smooth_gs", true);
    if (&rhs == &x) throw InvalidArgument("smooth_gs: rhs and x must be distinct functions");
    if (A.kind() == KIND_P2) {
        check_diagonals_p2(A, x, level, "smooth_gs");
        Domain& d = A.domain();
        d.sync(x, level);
        launch_p2_gs(A.tables_p2(level), x.flags(), rhs.data(level), x.data(level), d.stream());
        return;
    }
    check_diagonals(A, x, level, "smooth_gs");
    Domain& d = A.domain();
    d.sync(x, level);
    const LevelTables t = A.tables(level);
    Domain::GsPlan& gp = d.gs_plan(level);
    d.fork();
    launch_gs_ev(t, x.flags(), rhs.data(level), x.data(level), d.aux_stream());
    if (gp.ntiles > 0) {
        HYB_CUDA(cudaMemsetAsync(gp.flags.as<void>(), 0, size_t(gp.nflags) * 4, d.stream()));
        HYB_CUDA(cudaMemsetAsync(gp.counter.as<void>(), 0, 16, d.stream()));
        d.timer_begin("gauss_seidel");
        launch_gs_faces(t, rhs.data(level), x.data(level), gp.tiles.as<int4>(), gp.ntiles, gp.ni, gp.nj,
                        gp.flags.as<int>(), gp.counter.as<int>(), d.stream());
        d.timer_end();
    }
    d.join();
}

// coloured hybrid Gauss-Seidel (configuration 3, see gauss_seidel.cuh)
void smooth_cgs(const Operator& A, Function& rhs, Function& x, int level) {
    check_op_function(A, rhs, level, "smooth_cgs", true);
    check_op_function(A, x, level, "smooth_cgs", true);
    if (&rhs == &x) throw InvalidArgument("smooth_cgs: rhs and x must be distinct functions");
    require_p1(x, "smooth_cgs");
    check_diagonals(A, x, level, "smooth_cgs");
    Domain& d = A.domain();
    d.sync(x, level);
    const LevelTables t = A.tables(level);
    // faces in column blocks (k_cgs_cols): one block per face sweeps in place;
    // several blocks per face sweep out of place into the Jacobi scratch arena,
    // with the edges and vertices, and the scratch is swapped in
    DevMem& next = d.jacobi_scratch(level);
    // the edges and vertices read only their own rows and their halo copies (frozen by the sync
    // above) and the faces only theirs, so the two run side by side, as in smooth_gs
    d.fork();
    d.timer_begin("coloured_gs");
    const bool oop = launch_cgs_faces_cols(t, rhs.data(level), x.data(level), next.as<double>(), d.stream());
    d.timer_end();
    if (oop) launch_cgs_ev_oop(t, x.flags(), rhs.data(level), x.data(level), next.as<double>(), d.aux_stream());
    else launch_cgs_ev(t, x.flags(), rhs.data(level), x.data(level), d.aux_stream());
    d.join();
    if (oop) x.arena(level).swap(next);
}

// `count` coloured sweeps; consecutive pairs run the faces' two sweeps in one pass
// (k_cgs_pair) where a tuned variant exists for the face size, every ghost is
// same-process and same-rank, and n >= cgs_pair_min_n(). The pass reproduces the
// ghost refresh between the two sweeps with two split gathers (face-boundary copies
// into the second scratch arena before, the edges' halo rows from the faces' sweep-1
// layer after), so the result is bitwise `count` smooth_cgs calls. Measured slower
// than single sweeps (k_cgs_pair), so off unless asked for (hyb_tuning("cgs_pair_min_n")).
int g_cgs_pair_min_n = 1 << 30;
int cgs_pair_min_n() { return g_cgs_pair_min_n; }
void set_cgs_pair_min_n(int n) { g_cgs_pair_min_n = n; }

static bool cgs_pair_usable(const Operator& A, Function& x, int level) {
    Domain& d = A.domain();
    if (A.kind() != KIND_P1 || x.kind() != KIND_P1 || (1 << level) < cgs_pair_min_n()) return false;
    if (cgs_pair_blocks(1 << level) == 0 || d.multi_process() || d.local_ranks().size() != 1) return false;
    const Exchange& X = d.level(level).xch;
    return X.ntotal == X.nlocal;
}

// One coloured sweep of x = 0 (a coarse-grid correction's first pre-smoothing sweep: the
// iterate and every ghost of it are zero on entry, and its Dirichlet rows -- x := rhs -- are
// zero because the cycle zeroes the coarse rhs there). x's face blocks are neither filled
// nor read (the face kernels sweep rows of zeros and write rows 1..n-2), the edge/vertex
// part of the arena, halos included, is zeroed with one memset, and no ghost refresh is
// needed: bitwise fill_const(x, 0) + smooth_cgs. Face rows 0, n-1 and n hold only ghosts;
// the next operation's refresh rewrites them. False where no variant exists (the caller
// then fills and sweeps).
bool g_cgs_zero_sweep = true; // hyb_tuning("cgs_zero_sweep", 0) fills and sweeps instead
bool cgs_zero_sweep() { return g_cgs_zero_sweep; }
void set_cgs_zero_sweep(bool on) { g_cgs_zero_sweep = on; }

bool smooth_cgs_zero(const Operator& A, Function& rhs, Function& x, int level) {
    check_op_function(A, rhs, level, "smooth_cgs", true);
    check_op_function(A, x, level, "smooth_cgs", true);
    if (&rhs == &x) throw InvalidArgument("smooth_cgs: rhs and x must be distinct functions");
    require_p1(x, "smooth_cgs");
    const LevelTables t = A.tables(level);
    if (!cgs_zero_supported(t) || (1 << level) >= cgs_pair_min_n()) return false;
    check_diagonals(A, x, level, "smooth_cgs");
    Domain& d = A.domain();
    double* xa = x.data(level);
    if (t.arena_size > t.faces_size)
        HYB_CUDA(cudaMemsetAsync(xa + t.faces_size, 0, size_t(t.arena_size - t.faces_size) * 8, d.stream()));
    d.fork(); // after the memset; edges/vertices beside the faces, as in smooth_cgs
    d.timer_begin("coloured_gs");
    launch_cgs_faces_zero(t, rhs.data(level), xa, d.stream());
    d.timer_end();
    launch_cgs_ev(t, x.flags(), rhs.data(level), xa, d.aux_stream());
    d.join();
    return true;
}

void smooth_cgs_n(const Operator& A, Function& rhs, Function& x, int level, int count) {
    if (count < 0) throw InvalidArgument("smooth_cgs: negative sweep count");
    check_op_function(A, rhs, level, "smooth_cgs", true);
    check_op_function(A, x, level, "smooth_cgs", true);
    if (&rhs == &x) throw InvalidArgument("smooth_cgs: rhs and x must be distinct functions");
    require_p1(x, "smooth_cgs");
    const bool pairs = count >= 2 && cgs_pair_usable(A, x, level);
    for (; pairs && count >= 2; count -= 2) {
        check_diagonals(A, x, level, "smooth_cgs");
        Domain& d = A.domain();
        d.sync(x, level);
        const LevelTables t = A.tables(level);
        const FlagTables fl = x.flags();
        const Exchange& X = d.level(level).xch;
        const bool oop = cgs_pair_blocks(t.n) > 1;
        DevMem& next = d.jacobi_scratch(level);
        double* xa = x.data(level);
        double* y = oop ? next.as<double>() : xa;
        double* g = d.jacobi_scratch2(level).as<double>();
        const double* b = rhs.data(level);
        // sweep 1 of the edges and vertices (their ghosts are the synced copies)
        if (oop) launch_cgs_ev_oop(t, fl, b, xa, y, d.stream());
        else launch_cgs_ev(t, fl, b, xa, d.stream());
        // the faces' boundary ghosts as sweep 2 sees them
        launch_gather_split(X.dst.as<void>(), X.src.as<void>(), X.idx32, X.nlocal, t.faces_size, 0, y, g, d.stream());
        d.timer_begin("coloured_gs_pair");
        launch_cgs_pair(t, b, xa, y, g, d.stream());
        d.timer_end();
        // the edges' halo rows (faces after sweep 1) and the vertex/edge cross copies
        launch_gather_split(X.dst.as<void>(), X.src.as<void>(), X.idx32, X.nlocal, t.faces_size, 1, y, g, d.stream());
        launch_cgs_ev(t, fl, b, y, d.stream()); // sweep 2 of the edges and vertices
        if (oop) x.arena(level).swap(next);
    }
    for (; count > 0; --count) smooth_cgs(A, rhs, x, level);
}

void diagonal(const Operator& A, Function& dst, int level) {
    check_op_function(A, dst, level, "diagonal", true);
    Domain& d = A.domain();
    const MacroGraph& g = d.graph();
    const int n = 1 << level;
    if (A.kind() == KIND_P2) { // packed in the P2 owned order (owned_positions_p2)
        const auto& h = A.host_p2_diag(level);
        std::vector<double> packed;
        packed.reserve(size_t(d.geom(KIND_P2, level).t.owned_local));
        const size_t nf = d.local_faces().size(), ne = d.local_edges().size();
        for (size_t i = 0; i < d.local_verts().size(); ++i)
            packed.push_back((dst.bc().flag_for(g.vertices[d.local_verts()[i]].marker) & DIRICHLET) ? 1.0
                                                                                                : h[4 * nf + 2 * ne + i]);
        for (size_t i = 0; i < ne; ++i) {
            const bool dir = dst.bc().flag_for(g.edges[g.edge_index(d.local_edges()[i])].marker) & DIRICHLET;
            for (int k = 1; k <= n - 1; ++k) packed.push_back(dir ? 1.0 : h[4 * nf + 2 * i]);
            for (int m = 0; m < n; ++m) packed.push_back(dir ? 1.0 : h[4 * nf + 2 * i + 1]);
        }
        // face groups EH, ED, EV, V (classes 1, 3, 2, 0)
        for (size_t i = 0; i < nf; ++i) {
            const double* fd = &h[4 * i];
            for (int r = 1; r <= n - 1; ++r)
                for (int c = 0; c + r <= n - 1; ++c) packed.push_back(fd[1]);
            for (int r = 0; r <= n - 2; ++r)
                for (int c = 0; c + r <= n - 2; ++c) packed.push_back(fd[3]);
            for (int r = 0; r <= n - 2; ++r)
                for (int c = 1; c + r <= n - 1; ++c) packed.push_back(fd[2]);
            for (int r = 1; r <= n - 2; ++r)
                for (int c = 1; c + r <= n - 1; ++c) packed.push_back(fd[0]);
        }
        upload(dst, level, packed.data(), int64_t(packed.size()), false, ALL_FLAGS);
        return;
    }
    std::vector<double> packed(size_t(d.owned_local(level)));
    size_t pos = 0;
    const auto& hv = A.host_vtx_coef(level);
    size_t cpos = 0;
    for (uint64_t id : d.local_verts()) {
        const MacroVertex& v = g.vertices[id];
        const double diag = hv[cpos + 1 + v.edges.size()];
        cpos += 2 + v.edges.size();
        packed[pos++] = (dst.bc().flag_for(v.marker) & DIRICHLET) ? 1.0 : diag;
    }
    const auto& he = A.host_edge_coef(level);
    for (size_t i = 0; i < d.local_edges().size(); ++i) {
        const bool dir = dst.bc().flag_for(g.edges[g.edge_index(d.local_edges()[i])].marker) & DIRICHLET;
        for (int k = 1; k <= n - 1; ++k) packed[pos++] = dir ? 1.0 : he[i * 8 + 7];
    }
    const auto& hf = A.host_face_coef(level);
    const size_t per_face = size_t(n - 1) * size_t(std::max(n - 2, 0)) / 2;
    for (size_t i = 0; i < d.local_faces().size(); ++i)
        for (size_t k = 0; k < per_face; ++k) packed[pos++] = hf[i * 8 + 7];
    upload(dst, level, packed.data(), int64_t(packed.size()), false, ALL_FLAGS);
}

void prolongate(Function& coarse, Function& fine, int lc, uint8_t mask, bool add) {
    check_transfer(coarse, fine, lc, "prolongate");
    Domain& d = fine.domain();
    d.sync(coarse, lc);
    d.timer_begin(add ? "prolongate_add" : "prolongate");
    launch_prolongate(d.level(lc).t, d.level(lc + 1).t, fine.flags(), coarse.data(lc), fine.data(lc + 1), mask, add,
                      d.stream());
    d.timer_end();
}

// prolongate(e -> x, smooth mask, add) followed by smooth_jacobi(A, rhs, x,
// omega, lc+1), fused on the faces (ST_JACOBI_PROLONG): edges, vertices and
// the face layer next to the borders take the correction in place, a sync
// refreshes the ghosts, and the face kernel forms x + P e on the fly for the
// remaining points, so the corrected face interiors are never stored.
// Bitwise the two operations in sequence.
void prolongate_add_jacobi(const Operator& A, Function& e, Function& rhs, Function& x, double omega, int lc,
                           double* dotp) {
    const int level = lc + 1;
    check_transfer(e, x, lc, "prolongate");
    check_op_function(A, rhs, level, "smooth_jacobi", true);
    check_op_function(A, x, level, "smooth_jacobi", true);
    if (&rhs == &x) throw InvalidArgument("smooth_jacobi: rhs and x must be distinct functions");
    if (A.kind() == KIND_P2) {
        if (dotp) throw InvalidArgument("smooth_jacobi: fused dot provided for P1");
        check_diagonals_p2(A, x, level, "smooth_jacobi");
        Domain& d = A.domain();
        d.sync(x, level);
        DevMem& next = d.jacobi_scratch(level, KIND_P2);
        launch_p2(P2_JACOBI, A.tables_p2(level), x.flags(), x.data(level), rhs.data(level), next.as<double>(), omega,
                  ALL_FLAGS, d.stream());
        x.arena(level).swap(next);
        return;
    }
    check_diagonals(A, x, level, "smooth_jacobi");
    Domain& d = A.domain();
    d.sync(e, lc);
    const LevelTables& tc = d.level(lc).t;
    const LevelTables t = A.tables(level);
    launch_prolongate(tc, t, x.flags(), e.data(lc), x.data(level), kSmoothMask, true, d.stream(), false);
    launch_prolongate_layer(tc, t, e.data(lc), x.data(level), d.stream());
    d.sync(x, level);
    DevMem& next = d.jacobi_scratch(level);
    d.timer_begin("prolongate_jacobi"); // edge/vertex Jacobi rows as the launch's trailing CTAs
    const FlagTables fl = x.flags();
    launch_jacobi_prolong_faces(tc, t, x.data(level), e.data(lc), rhs.data(level), next.as<double>(), omega, dotp,
                                d.stream(), &fl);
    d.timer_end();
    x.arena(level).swap(next);
}

// prolongate(e -> x, smooth mask, add) followed by smooth_cgs(A, rhs, x, lc+1), fused
// on the faces where a variant exists (k_cgs_cols<PRO>, faces of n >= 256): edges,
// vertices and the face layer next to the borders take the correction in place, a sync
// refreshes the ghosts, and the sweep adds the correction to the other face points as
// their rows enter its ring, so the corrected faces are never stored before the sweep.
// Bitwise the two calls in sequence. Measured slower than the two calls on B200
// (config 3, per level with the syncs: L9 10.59 vs 9.62 ms, L8 3.36 vs 2.99): the
// fused sweep needs 256-column blocks and corrector warps (9.57 ms, 6.3 G instructions,
// against 5.56 ms + 3.38 ms for the 512-column sweep and the prolongation), so the
// fusion is off unless asked for (hyb_tuning("cgs_prolong_fused", 1)).
bool g_cgs_prolong_fused = false;
bool cgs_prolong_fused() { return g_cgs_prolong_fused; }
void set_cgs_prolong_fused(bool on) { g_cgs_prolong_fused = on; }

void prolongate_add_cgs(const Operator& A, Function& e, Function& rhs, Function& x, int lc) {
    const int level = lc + 1;
    check_transfer(e, x, lc, "prolongate");
    check_op_function(A, rhs, level, "smooth_cgs", true);
    check_op_function(A, x, level, "smooth_cgs", true);
    if (&rhs == &x) throw InvalidArgument("smooth_cgs: rhs and x must be distinct functions");
    require_p1(x, "smooth_cgs");
    const LevelTables t = A.tables(level);
    if (!cgs_prolong_fused() || t.n < 256) {
        prolongate(e, x, lc, kSmoothMask, true);
        smooth_cgs(A, rhs, x, level);
        return;
    }
    check_diagonals(A, x, level, "smooth_cgs");
    Domain& d = A.domain();
    d.sync(e, lc);
    const LevelTables& tc = d.level(lc).t;
    launch_prolongate(tc, t, x.flags(), e.data(lc), x.data(level), kSmoothMask, true, d.stream(), false);
    launch_prolongate_layer(tc, t, e.data(lc), x.data(level), d.stream());
    d.sync(x, level);
    DevMem& next = d.jacobi_scratch(level);
    d.fork(); // edges/vertices beside the faces, as in smooth_cgs
    d.timer_begin("coloured_gs_prolong");
    const int oop = launch_cgs_prolong(tc, t, rhs.data(level), x.data(level), next.as<double>(), e.data(lc), d.stream());
    d.timer_end();
    if (oop) launch_cgs_ev_oop(t, x.flags(), rhs.data(level), x.data(level), next.as<double>(), d.aux_stream());
    else launch_cgs_ev(t, x.flags(), rhs.data(level), x.data(level), d.aux_stream());
    d.join();
    if (oop) x.arena(level).swap(next);
}

void restrict_to_coarse(Function& fine, Function& coarse, int lc, uint8_t mask) {
    check_transfer(coarse, fine, lc, "restrict_to_coarse");
    Domain& d = fine.domain();
    d.sync(fine, lc + 1);
    d.timer_begin("restrict");
    launch_restrict(d.level(lc).t, d.level(lc + 1).t, coarse.flags(), fine.data(lc + 1), coarse.data(lc), mask,
                    d.stream());
    d.timer_end();
}

// residual (reference solvers.cpp:418-419) + restrict_to_coarse (:420),
// fused on face interiors: the fine residual there is never stored
// (k_residual_restrict_faces); edges/vertices and the face layer next to the
// borders are computed as in residual(), synced, and restricted as usual.
void residual_restrict(const Operator& A, Function& rhs, Function& x, Function& r, Function& coarse, int lc) {
    const int level = lc + 1;
    check_op_function(A, rhs, level, "residual_restrict", false);
    check_op_function(A, x, level, "residual_restrict", false);
    check_op_function(A, r, level, "residual_restrict", true);
    check_transfer(coarse, r, lc, "residual_restrict");
    // coarse is written at coarse_level only, so it may be rhs or x (other levels)
    if (&x == &r || &rhs == &r || &coarse == &r)
        throw InvalidArgument("residual_restrict: r must be distinct from x, rhs and coarse");
    Domain& d = A.domain();
    // small faces: the two operations apart (the residual is then the thread-per-point kernel; the
    // fused tiled mode spends a pipeline stage per row however short: on 8192 faces 603 us at level 7,
    // 345 at level 6, 221 at level 5); bitwise the fused result
    static const int rr_unfused_max_n = [] {
        const char* e = std::getenv("HYB_RR_UNFUSED_MAX_N");
        return e ? std::atoi(e) : 128;
    }();
    if ((1 << level) <= rr_unfused_max_n) {
        residual(A, rhs, x, r, level);
        restrict_to_coarse(r, coarse, lc, ALL_FLAGS);
        return;
    }
    d.sync(x, level);
    const LevelTables t = A.tables(level);
    const LevelTables& tc = d.level(lc).t;
    // the faces' border layer and the edge/vertex rows of r on the side stream, beside the face kernel
    // (all three read x and rhs only and write disjoint parts of r / coarse)
    d.fork();
    d.timer_begin("residual_restrict");
    launch_residual_restrict_faces(tc, t, x.data(level), rhs.data(level), r.data(level), coarse.data(lc), d.stream(),
                                   d.aux_stream());
    d.timer_end();
    launch_stencil(ST_RESIDUAL, t, r.flags(), x.data(level), rhs.data(level), r.data(level), 0.0, ALL_FLAGS,
                   d.aux_stream(), 2);
    d.join();
    d.sync(r, level);
    launch_restrict_ev(tc, t, coarse.flags(), r.data(level), coarse.data(lc), ALL_FLAGS, d.stream());
}

void assign(double alpha, Function& x1, double beta, Function& x2, Function& dst, int level, uint8_t mask) {
    check_pair("assign", x1, x2, level);
    check_pair("assign", x1, dst, level);
    Domain& d = dst.domain();
    launch_blas1(0, d.geom(dst.kind(), level).t, dst.flags(), alpha, x1.data(level), beta, x2.data(level), dst.data(level), mask,
                 d.stream());
}

void add_scaled(Function& dst, double gamma, Function& y, int level, uint8_t mask) {
    check_pair("add_scaled", dst, y, level);
    Domain& d = dst.domain();
    launch_blas1(1, d.geom(dst.kind(), level).t, dst.flags(), gamma, y.data(level), 0.0, y.data(level), dst.data(level), mask,
                 d.stream());
}

void fill_const(Function& f, double value, int level, uint8_t mask) {
    f.check_level(level, "interpolate");
    Domain& d = f.domain();
    launch_blas1(2, d.geom(f.kind(), level).t, f.flags(), value, f.data(level), 0.0, f.data(level), f.data(level), mask,
                 d.stream());
}

void fill_random(Function& f, int level, uint64_t seed, uint64_t stream, double lo, double hi, uint8_t mask) {
    f.check_level(level, "interpolate");
    Domain& d = f.domain();
    launch_random(d.geom(f.kind(), level).t, f.flags(), seed, stream, lo, hi, f.data(level), mask, d.stream());
}

void fill_expr(Function& f, int level, const Expr& e, uint8_t mask) {
    f.check_level(level, "interpolate");
    if (e.kind != EXPR_POLY2 && e.kind != EXPR_SINSIN)
        throw InvalidArgument("interpolate: unknown expression kind " + std::to_string(e.kind));
    Domain& d = f.domain();
    launch_expr(d.geom(f.kind(), level).t, f.flags(), d.geometry(), e, f.data(level), mask, d.stream());
}

namespace {
void reduce_dev(int op, Function& a, Function& b, int level, double* out) {
    Domain& d = a.domain();
    const LevelTables& t = d.geom(a.kind(), level).t;
    const int64_t np = int64_t(d.graph().size());
    const int bands = t.n >= 3 ? (t.n - 2 + 31) / 32 : 0;
    double* buf = d.partials(2 * np + int64_t(t.nfaces) * bands + 1);
    double* part = buf;
    double* scratch = buf + 2 * np;
    HYB_CUDA(cudaMemsetAsync(part, 0, size_t(np) * 8, d.stream()));
    launch_partials(op, t, a.data(level), b.data(level), part, scratch, d.stream());
    d.allreduce_sum(part, np); // one non-zero entry per primitive: exact
    launch_combine_tree(op, part, np, out, d.stream());
}
double reduce(int op, Function& a, Function& b, int level) {
    reduce_dev(op, a, b, level, a.domain().scalar_out());
    return to_host(a.domain(), a.domain().scalar_out());
}
} // namespace

// x += alpha p; r -= alpha ap (add_scaled twice, bitwise) and return r.r
// (bitwise dot(r, r)) from one pass over the faces
double pcg_update(Function& x, Function& p, Function& r, Function& ap, double alpha, int level) {
    pcg_update_dev(x, p, r, ap, alpha, nullptr, level, x.domain().scalar_out());
    return to_host(x.domain(), x.domain().scalar_out());
}

void pcg_update_dev(Function& x, Function& p, Function& r, Function& ap, double alpha, const double* alpha_dev,
                    int level, double* rr_out) {
    check_pair("pcg_update", x, p, level);
    check_pair("pcg_update", r, ap, level);
    check_pair("pcg_update", x, r, level);
    Domain& d = x.domain();
    const LevelTables& t = d.level(level).t;
    const int64_t np = int64_t(d.graph().size());
    const int bands = t.n >= 3 ? (t.n - 2 + 31) / 32 : 0;
    double* buf = d.partials(2 * np + int64_t(t.nfaces) * bands + 1);
    double* part = buf;
    double* scratch = buf + 2 * np;
    HYB_CUDA(cudaMemsetAsync(part, 0, size_t(np) * 8, d.stream()));
    launch_pcg_update(t, r.flags(), x.data(level), p.data(level), r.data(level), ap.data(level), alpha, part, scratch,
                      d.stream(), alpha_dev);
    d.allreduce_sum(part, np);
    launch_combine_tree(0, part, np, rr_out, d.stream());
}

void dot_dev(Function& a, Function& b, int level, double* out) {
    check_pair("dot", a, b, level);
    reduce_dev(0, a, b, level, out);
}

double dot(Function& a, Function& b, int level) {
    check_pair("dot", a, b, level);
    return reduce(0, a, b, level);
}

double max_abs(Function& a, int level) {
    a.check_level(level, "max_abs");
    return reduce(1, a, a, level);
}

// ---------------------------------------------------------------- host <-> device
namespace {
// owned position of a local primitive's first DoF in the global ordering
struct GlobalOrder {
    int64_t nv, ne, n, per_face;
    int64_t vertex(uint64_t id) const { return int64_t(id); }
    int64_t edge(size_t ei) const { return nv + int64_t(ei) * (n - 1); }
    int64_t face(size_t fi) const { return nv + ne * (n - 1) + int64_t(fi) * per_face; }
};

bool all_local(const Domain& d) {
    return d.local_faces().size() == d.graph().nf() && d.local_edges().size() == d.graph().ne() &&
           d.local_verts().size() == d.graph().nv();
}

// copies between the global vector and the local packed vector
void global_local(Domain& d, int level, const double* src, double* dst, bool to_local) {
    const MacroGraph& g = d.graph();
    const int64_t n = int64_t(1) << level;
    const GlobalOrder go{int64_t(g.nv()), int64_t(g.ne()), n, (n - 1) * (n - 2) / 2};
    int64_t pos = 0;
    auto mv = [&](int64_t gpos, int64_t len) {
        if (len <= 0) return;
        if (to_local) std::memcpy(dst + pos, src + gpos, size_t(len) * 8);
        else std::memcpy(dst + gpos, src + pos, size_t(len) * 8);
        pos += len;
    };
    for (uint64_t id : d.local_verts()) mv(go.vertex(id), 1);
    for (uint64_t id : d.local_edges()) mv(go.edge(g.edge_index(id)), n - 1);
    for (uint64_t id : d.local_faces()) mv(go.face(g.face_index(id)), go.per_face);
}
} // namespace

void upload(Function& f, int level, const double* host, int64_t n, bool global_order, uint8_t mask) {
    f.check_level(level, "upload");
    Domain& d = f.domain();
    const LevelGeom& lg = d.geom(f.kind(), level);
    const LevelTables& t = lg.t;
    // a P2 level holds the owned set of P1 level + 1 (per primitive counts equal)
    const int olevel = f.kind() == KIND_P2 ? level + 1 : level;
    const int64_t want = global_order ? d.owned_total(olevel) : t.owned_local;
    if (n != want)
        throw InvalidArgument("upload: vector has " + std::to_string(n) + " entries, expected " + std::to_string(want));
    double* stage = d.staging(t.owned_local);
    if (!global_order || all_local(d)) {
        HYB_CUDA(cudaMemcpyAsync(stage, host, size_t(t.owned_local) * 8, cudaMemcpyHostToDevice, d.stream()));
    } else {
        std::vector<double> tmp(size_t(t.owned_local));
        global_local(d, olevel, host, tmp.data(), true);
        HYB_CUDA(cudaMemcpyAsync(stage, tmp.data(), tmp.size() * 8, cudaMemcpyHostToDevice, d.stream()));
        HYB_CUDA(cudaStreamSynchronize(d.stream()));
    }
    if (f.kind() == KIND_P2)
        launch_scatter_pos(t.owned_local, lg.owned_pos.as<int64_t>(), f.owned_flags(level), mask, stage, f.data(level),
                           d.stream());
    else
        launch_scatter_owned(t, f.flags(), stage, f.data(level), mask, d.stream());
}

// Stream-ordered transfers for pipelines (see Domain::h2d_stream): `host`
// holds this process's owned DoFs in local order (GlobalDoFMap order when the
// process owns every primitive); pinned memory makes the copies asynchronous.
void upload_async(Function& f, int level, const double* host, int64_t n, uint8_t mask) {
    f.check_level(level, "upload_async");
    require_p1(f, "upload_async");
    Domain& d = f.domain();
    const LevelTables& t = d.level(level).t;
    if (n != t.owned_local)
        throw InvalidArgument("upload_async: vector has " + std::to_string(n) + " entries, expected " +
                              std::to_string(t.owned_local));
    double* stage = d.stage_h2d(n);
    d.after_main(d.h2d_stream()); // earlier work may still read f
    HYB_CUDA(cudaMemcpyAsync(stage, host, size_t(n) * 8, cudaMemcpyHostToDevice, d.h2d_stream()));
    launch_scatter_owned(t, f.flags(), stage, f.raw(level), mask, d.h2d_stream());
    d.main_waits(d.h2d_stream()); // later work reads the new values
}

void download_async(Function& f, int level, double* host, int64_t n) {
    f.check_level(level, "download_async");
    require_p1(f, "download_async");
    Domain& d = f.domain();
    const LevelTables& t = d.level(level).t;
    if (n != t.owned_local)
        throw InvalidArgument("download_async: vector has " + std::to_string(n) + " entries, expected " +
                              std::to_string(t.owned_local));
    double* stage = d.stage_d2h(n);
    d.after_main(d.d2h_stream()); // the values f holds once the queued work is done
    launch_gather_owned(t, f.raw(level), stage, d.d2h_stream());
    HYB_CUDA(cudaMemcpyAsync(host, stage, size_t(n) * 8, cudaMemcpyDeviceToHost, d.d2h_stream()));
    d.download_issued();
}

void download(Function& f, int level, double* host, int64_t n, bool global_order) {
    f.check_level(level, "download");
    Domain& d = f.domain();
    const LevelGeom& lg = d.geom(f.kind(), level);
    const LevelTables& t = lg.t;
    const int olevel = f.kind() == KIND_P2 ? level + 1 : level;
    const int64_t want = global_order ? d.owned_total(olevel) : t.owned_local;
    if (n != want)
        throw InvalidArgument("download: vector has " + std::to_string(n) + " entries, expected " + std::to_string(want));
    double* stage = d.staging(t.owned_local);
    if (f.kind() == KIND_P2) launch_gather_pos(t.owned_local, lg.owned_pos.as<int64_t>(), f.data(level), stage, d.stream());
    else launch_gather_owned(t, f.data(level), stage, d.stream());
    if (!global_order || all_local(d)) {
        HYB_CUDA(cudaMemcpyAsync(host, stage, size_t(t.owned_local) * 8, cudaMemcpyDeviceToHost, d.stream()));
        HYB_CUDA(cudaStreamSynchronize(d.stream()));
    } else {
        std::vector<double> tmp(size_t(t.owned_local));
        HYB_CUDA(cudaMemcpyAsync(tmp.data(), stage, tmp.size() * 8, cudaMemcpyDeviceToHost, d.stream()));
        HYB_CUDA(cudaStreamSynchronize(d.stream()));
        global_local(d, olevel, tmp.data(), host, false);
    }
}

// ---------------------------------------------------------------- Hierarchy
Hierarchy::Hierarchy(Domain& d, Form form, int min_level, int max_level, BoundaryMap bc, int smoother, double omega,
                     double coarse_tol, int coarse_max_iter)
    : dom_(&d), a_(d, form, min_level, max_level, bc), r_(d, "mg.r", min_level, max_level, bc),
      b_(d, "mg.b", min_level, std::max(min_level, max_level - 1), bc),
      e_(d, "mg.e", min_level, std::max(min_level, max_level - 1), bc), smoother_(smoother),
      omega_(omega), coarse_tol_(coarse_tol), coarse_max_iter_(coarse_max_iter) {
    if (min_level < 0 || min_level > max_level)
        throw InvalidArgument("GridHierarchy: need 0 <= min_level <= max_level");
    mega_dofs_per_cta = mega_dofs_per_cta_default();
    if (smoother != SMOOTH_JACOBI && smoother != SMOOTH_GS && smoother != SMOOTH_CGS)
        throw InvalidArgument("GridHierarchy: unknown smoother");
    // min-level system: every rank holds the whole (small) constrained matrix
    const HostCsr csr = assemble_constrained(d.graph(), form, min_level, bc);
    if (coarse_max_iter_ < 0) coarse_max_iter_ = int(csr.n) + 100; // reference src/solvers.cpp:437
    const HostLayout lay = plan_layout(d.graph(), d.placement(), min_level);
    const std::vector<int64_t> gidx = owned_global_index(d.graph(), d.placement(), min_level);
    const std::vector<int64_t> pos = owned_positions(d.graph(), d.placement(), lay);
    std::vector<uint8_t> fl(gidx.size());
    for (size_t i = 0; i < gidx.size(); ++i) fl[i] = csr.flag[size_t(gidx[i])];
    coarse_.n = csr.n;
    for (int64_t i = 0; i < csr.n; ++i)
        coarse_.max_row_nnz = std::max(coarse_.max_row_nnz, csr.rowptr[size_t(i) + 1] - csr.rowptr[size_t(i)]);
    coarse_.nloc = int64_t(gidx.size());
    coarse_.rowptr = upload_vec(csr.rowptr, d.stream());
    coarse_.col = upload_vec(csr.col, d.stream());
    coarse_.val = upload_vec(csr.val, d.stream());
    coarse_.gidx = upload_vec(gidx, d.stream());
    coarse_.pos = upload_vec(pos, d.stream());
    coarse_.flag = upload_vec(fl, d.stream());
    coarse_.vec = DevMem(size_t(5 * std::max<int64_t>(csr.n, 1)) * 8);
    coarse_.status = DevMem(sizeof(CoarseStatus));
    HYB_CUDA(cudaMemsetAsync(coarse_.status.as<void>(), 0, sizeof(CoarseStatus), d.stream()));
    if (csr.n >= coarse_grid_min_rows()) { // whole-GPU CG: per-CTA partials + barrier words
        coarse_.grid = DevMem(size_t(4 * std::max(coarse_grid_blocks(), 1)) * 8 + 64);
        HYB_CUDA(cudaMemsetAsync(coarse_.grid.as<void>(), 0, coarse_.grid.bytes(), d.stream()));
    }
}

void Hierarchy::smooth(Function& rhs, Function& x, int level, double* dotp) {
    if (smoother_ == SMOOTH_GS) smooth_gs(a_, rhs, x, level); // the reference's own choice (solvers.cpp:417, 427)
    else if (smoother_ == SMOOTH_CGS) smooth_cgs(a_, rhs, x, level);
    else smooth_jacobi(a_, rhs, x, omega_, level, dotp);
}

void Hierarchy::vcycle(Function& rhs, Function& x, int level, int nu_pre, int nu_post) {
    if (level < a_.min_level() || level > a_.max_level())
        throw OutOfRange("vcycle: level " + std::to_string(level) + " outside [" + std::to_string(a_.min_level()) +
                         ", " + std::to_string(a_.max_level()) + "]");
    if (nu_pre < 0 || nu_post < 0) throw InvalidArgument("vcycle: negative smoothing count");
    run_cycle(rhs, x, level, nu_pre, nu_post);
}

Hierarchy::~Hierarchy() {
    for (auto& g : graphs_)
        if (g.exec) cudaGraphExecDestroy(g.exec);
}

std::vector<const void*> Hierarchy::graph_key(Function& rhs, Function& x, int level, int nu_pre, int nu_post,
                                              bool x_zero) {
    std::vector<const void*> k{&rhs, &x, rhs.data(level), x.data(level), reinterpret_cast<const void*>(intptr_t(level)),
                               reinterpret_cast<const void*>(intptr_t(nu_pre)),
                               reinterpret_cast<const void*>(intptr_t(nu_post)),
                               reinterpret_cast<const void*>(intptr_t(x_zero)), cycle_dot_,
                               reinterpret_cast<const void*>(intptr_t(cycle_dot_level_)), dom_->send_buffer(),
                               dom_->recv_buffer()};
    for (int l = a_.min_level(); l <= level; ++l) {
        k.push_back(r_.data(l));
        if (l < level) {
            k.push_back(b_.data(l));
            k.push_back(e_.data(l));
        }
        if (l > a_.min_level()) k.push_back(dom_->jacobi_scratch(l).as<void>());
        k.push_back(dom_->jacobi_scratch2_ptr(l));
    }
    return k;
}

// One cycle, replayed from a CUDA graph when possible: the first call with a
// given argument/arena state runs eagerly (allocations, plans), the second
// captures the whole cycle (kernels, copies, NCCL) and later calls replay it.
void Hierarchy::run_cycle(Function& rhs, Function& x, int level, int nu_pre, int nu_post, bool x_zero) {
    Domain& d = *dom_;
    const bool swaps_restore = smoother_ != SMOOTH_JACOBI || (nu_pre + nu_post) % 2 == 0; // GS works in place
    if (!use_graphs || !swaps_restore || d.profiling) {
        cycle(rhs, x, level, nu_pre, nu_post, x_zero);
        check_coarse();
        return;
    }
    const std::vector<const void*> key = graph_key(rhs, x, level, nu_pre, nu_post, x_zero);
    if (std::find(no_graph_.begin(), no_graph_.end(), key) != no_graph_.end()) {
        cycle(rhs, x, level, nu_pre, nu_post, x_zero);
        check_coarse();
        return;
    }
    for (const auto& g : graphs_)
        if (g.key == key) {
            HYB_CUDA(cudaGraphLaunch(g.exec, d.stream()));
            ++graph_replays;
            check_coarse();
            return;
        }
    if (std::find(warm_.begin(), warm_.end(), key) == warm_.end()) {
        cycle(rhs, x, level, nu_pre, nu_post, x_zero);
        check_coarse();
        warm_.push_back(key);
        return;
    }
    cudaGraph_t graph = nullptr;
    d.settle_transfers(); // no wait on an outside event inside the capture
    HYB_CUDA(cudaStreamBeginCapture(d.stream(), cudaStreamCaptureModeThreadLocal));
    try {
        cycle(rhs, x, level, nu_pre, nu_post, x_zero);
    } catch (...) {
        cudaStreamEndCapture(d.stream(), &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
    }
    HYB_CUDA(cudaStreamEndCapture(d.stream(), &graph));
    cudaGraphExec_t exec = nullptr;
    const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    HYB_CUDA(ie);
    if (graph_key(rhs, x, level, nu_pre, nu_post, x_zero) != key) {
        // the cycle leaves some arena swapped (an odd number of out-of-place sweeps on a
        // level): the captured kernels match the host state after this one call but no
        // later call, so run them once and keep this cycle eager from now on
        HYB_CUDA(cudaGraphLaunch(exec, d.stream()));
        cudaGraphExecDestroy(exec);
        no_graph_.push_back(key);
        check_coarse();
        return;
    }
    graphs_.push_back({key, exec});
    HYB_CUDA(cudaGraphLaunch(exec, d.stream()));
    ++graph_replays;
    check_coarse();
}

// reference src/solvers.cpp:406-428 with the smoother of the configuration.
// x_zero: x is known to be zero (a coarse correction, PCG's z); with Jacobi
// pre-smoothing the zero-fill, the Dirichlet assign and the first sweep's read
// of x are replaced by one zero-guess sweep (bitwise the same values).
// The coarse end of the cycle in one cooperative kernel (mega.cuh): weighted
// Jacobi, one process with one rank (every ghost same-rank), a one-CTA coarse
// CG, an even number of sweeps per level (the iterate ends in its own arena),
// no fused dot at these levels; bitwise the launched cycle.
bool Hierarchy::mega_usable(int level, int nu_pre, int nu_post) {
    Domain& d = *dom_;
    const int lmin = a_.min_level();
    if (mega_ == 0 || smoother_ != SMOOTH_JACOBI || d.profiling || (1 << level) > mega_max_n || level <= lmin)
        return false;
    if (mega_ < 0 && d.local_faces().size() > size_t(mega_auto_faces)) return false;
    if (nu_pre < 1 || (nu_pre + nu_post) % 2 != 0 || level - lmin + 1 > MC_MAX_LEVELS) return false;
    if (d.multi_process() || d.local_ranks().size() != 1 || coarse_.n >= coarse_grid_min_rows()) return false;
    if (cycle_dot_ && cycle_dot_level_ >= lmin && cycle_dot_level_ <= level) return false;
    for (int l = lmin; l <= level; ++l) {
        const Exchange& X = d.level(l).xch;
        if (X.ntotal != X.nlocal || X.npack) return false;
    }
    return true;
}

void Hierarchy::run_mega(Function& rhs, Function& x, int level, int nu_pre, int nu_post, bool x_zero) {
    Domain& d = *dom_;
    const int lmin = a_.min_level();
    std::vector<McLevel> lv;
    std::vector<const void*> key;
    for (int l = lmin; l <= level; ++l) {
        McLevel m{};
        m.t = a_.tables(l);
        Function& xf = l == level ? x : e_;
        Function& bf = l == level ? rhs : b_;
        m.fl = xf.flags();
        m.x = xf.data(l);
        m.s = d.jacobi_scratch(l).as<double>();
        m.rhs = bf.data(l);
        m.r = r_.data(l);
        const Exchange& X = d.level(l).xch;
        m.gdst = X.dst.as<void>();
        m.gsrc = X.src.as<void>();
        m.ng = X.nlocal;
        m.idx32 = X.idx32 ? 1 : 0;
        lv.push_back(m);
        key.insert(key.end(), {m.x, m.s, m.rhs, m.r, m.fl.edge_flag, m.fl.vtx_flag});
    }
    auto it = mega_tables_.find(key);
    if (it == mega_tables_.end()) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        HYB_CUDA(cudaStreamIsCapturing(d.stream(), &cs));
        if (cs != cudaStreamCaptureStatusNone) throw LogicError("vcycle: coarse-cycle tables missing during capture");
        it = mega_tables_.emplace(key, upload_vec(lv, d.stream())).first;
    }
    if (!mega_bar_.bytes()) {
        mega_bar_ = DevMem(64);
        HYB_CUDA(cudaMemsetAsync(mega_bar_.as<void>(), 0, 64, d.stream()));
    }
    McRun run;
    run.top = level;
    run.lmin = lmin;
    run.nu_pre = nu_pre;
    run.nu_post = nu_post;
    run.x_zero = x_zero ? 1 : 0;
    run.omega = omega_;
    run.cg.n = coarse_.n;
    run.cg.nloc = coarse_.nloc;
    run.cg.rowptr = coarse_.rowptr.as<int32_t>();
    run.cg.col = coarse_.col.as<int32_t>();
    run.cg.val = coarse_.val.as<double>();
    run.cg.gidx = coarse_.gidx.as<int64_t>();
    run.cg.pos = coarse_.pos.as<int64_t>();
    run.cg.flag = coarse_.flag.as<uint8_t>();
    run.cg.vec = coarse_.vec.as<double>();
    run.cg.st = coarse_.status.as<CoarseStatus>();
    run.cg.tol = coarse_tol_;
    run.cg.max_iter = coarse_max_iter_;
    run.bar = mega_bar_.as<unsigned>();
    run.cg_smem = size_t(5 * coarse_.n) * sizeof(double) <= 200 * 1024 ? 1 : 0;
    const int64_t dofs = d.owned_local(level);
    launch_vcycle_coarse(it->second.as<McLevel>(), run, int((dofs + mega_dofs_per_cta - 1) / mega_dofs_per_cta),
                         d.stream());
    ++mega_launches;
}

void Hierarchy::cycle(Function& rhs, Function& x, int level, int nu_pre, int nu_post, bool x_zero) {
    if (mega_usable(level, nu_pre, nu_post)) {
        run_mega(rhs, x, level, nu_pre, nu_post, x_zero);
        return;
    }
    const bool zero_sweep = x_zero && level > a_.min_level() && nu_pre > 0 && smoother_ == SMOOTH_JACOBI;
    // coloured GS: the first sweep of a correction (x = 0, Dirichlet rows of the coarse rhs
    // zeroed by the caller below) without the fill, the ghost refresh and the read of x
    int cgs_done = 0;
    if (x_zero && &rhs == &b_ && &x == &e_ && level > a_.min_level() && nu_pre > 0 && smoother_ == SMOOTH_CGS &&
        cgs_zero_sweep() && smooth_cgs_zero(a_, rhs, x, level))
        cgs_done = 1;
    if (x_zero && !zero_sweep && !cgs_done) fill_const(x, 0.0, level, ALL_FLAGS);
    if (!zero_sweep && !cgs_done) assign(1.0, rhs, 0.0, rhs, x, level, kDirichletMask);
    if (level == a_.min_level()) {
        coarse_correct(rhs, x);
        return;
    }
    // the pre-smoothing pair as one two-sweep pass (x's arena goes to the second
    // scratch arena); the post-smoothing's last sweep then writes the second scratch
    // arena, and a final exchange of the two scratch arenas leaves every arena as
    // the cycle found it (CUDA-graph replay)
    const bool pair = smoother_ == SMOOTH_JACOBI && temporal_ && !zero_sweep && nu_pre == 2 && nu_post >= 2 &&
                      (1 << level) >= jacobi2_min_n();
    if (pair) {
        smooth_jacobi2(a_, rhs, x, omega_, level);
    } else {
        if (smoother_ == SMOOTH_CGS) smooth_cgs_n(a_, rhs, x, level, nu_pre - cgs_done);
        else
            for (int i = 0; i < nu_pre; ++i) {
                if (i == 0 && zero_sweep) smooth_jacobi_zero(a_, rhs, x, omega_, level);
                else smooth(rhs, x, level);
            }
    }
    residual_restrict(a_, rhs, x, r_, b_, level - 1); // residual + restrict_to_coarse, fused
    fill_const(b_, 0.0, level - 1, kDirichletMask);
    cycle(b_, e_, level - 1, nu_pre, nu_post, true); // e = 0 on entry
    // prolongate(e -> r) + add_scaled(x, 1, r) on the smooth mask, fused; with
    // Jacobi post-smoothing also fused with the first sweep
    auto dot_for = [&](int i) { return (level == cycle_dot_level_ && i == nu_post - 1) ? cycle_dot_ : nullptr; };
    int i0 = 0;
    // (on small faces the correction and the sweep run apart: the sweep is then the thread-per-point
    // kernel, HYB_JP_UNFUSED_MAX_N)
    static const int jp_unfused_max_n = [] {
        const char* e = std::getenv("HYB_JP_UNFUSED_MAX_N");
        return e ? std::atoi(e) : 128;
    }();
    if (nu_post > 0 && smoother_ == SMOOTH_JACOBI && fuse_post_ && (1 << level) > jp_unfused_max_n) {
        prolongate_add_jacobi(a_, e_, rhs, x, omega_, level - 1, dot_for(0));
        i0 = 1;
    } else if (nu_post > 0 && smoother_ == SMOOTH_CGS && fuse_post_) {
        prolongate_add_cgs(a_, e_, rhs, x, level - 1);
        i0 = 1;
    } else {
        prolongate(e_, x, level - 1, kSmoothMask, true);
    }
    if (smoother_ == SMOOTH_CGS) {
        smooth_cgs_n(a_, rhs, x, level, nu_post - i0);
        i0 = nu_post;
    }
    for (int i = i0; i < nu_post; ++i) {
        if (pair && i == nu_post - 1) smooth_jacobi(a_, rhs, x, omega_, level, dot_for(i), 2);
        else smooth(rhs, x, level, dot_for(i));
    }
    // (x, s1, s2) went (X, Y, Z) -> (Z, Y, X) in the pass; nu_post - 1 exchanges with s1
    // and one with s2 bring x back; the scratch pair is swapped when that count is odd
    if (pair && (nu_post - 1) % 2 == 1) dom_->swap_scratch(level);
}

// reference src/solvers.cpp:430-442: residual, gather into the global coarse
// vector (one allreduce across processes), CG on the assembled constrained
// matrix (cg_solve :226-259) on the device, scatter-add on the smooth mask.
// No host synchronisation: convergence is checked after the cycle.
void Hierarchy::coarse_correct(Function& rhs, Function& x) {
    const int L = a_.min_level();
    Domain& d = *dom_;
    residual(a_, rhs, x, r_, L);
    const int64_t n = coarse_.n;
    double* b = coarse_.vec.as<double>();
    double* cx = b + n;
    HYB_CUDA(cudaMemsetAsync(b, 0, size_t(n) * 8, d.stream()));
    launch_coarse_gather(coarse_.nloc, coarse_.gidx.as<int64_t>(), coarse_.pos.as<int64_t>(), r_.data(L), b,
                         d.stream());
    d.allreduce_sum(b, n); // one owner per entry: exact
    d.timer_begin("coarse_cg");
    launch_coarse_cg(n, coarse_.rowptr.as<int32_t>(), coarse_.col.as<int32_t>(), coarse_.val.as<double>(), b, cx,
                     b + 2 * n, b + 3 * n, b + 4 * n, coarse_tol_, coarse_max_iter_,
                     coarse_.status.as<CoarseStatus>(), coarse_.grid_part(), coarse_.grid_bar(), coarse_.max_row_nnz,
                     d.stream());
    d.timer_end();
    launch_coarse_scatter_add(coarse_.nloc, coarse_.gidx.as<int64_t>(), coarse_.pos.as<int64_t>(),
                              coarse_.flag.as<uint8_t>(), kSmoothMask, cx, x.data(L), d.stream());
}

void Hierarchy::check_coarse() {
    CoarseStatus st{};
    HYB_CUDA(cudaMemcpyAsync(&st, coarse_.status.as<void>(), sizeof st, cudaMemcpyDeviceToHost, dom_->stream()));
    HYB_CUDA(cudaStreamSynchronize(dom_->stream()));
    last_coarse_iterations = st.iterations;
    if (!st.converged)
        throw RuntimeError("vcycle: coarse CG did not converge (" + std::to_string(st.iterations) +
                           " iterations, residual " + std::to_string(st.residual) + ", target " +
                           std::to_string(st.target) + ")");
}

double Hierarchy::residual_norm(Function& rhs, Function& x, int level) {
    if (a_.kind() == KIND_P1 && fuse_norm_) return std::sqrt(residual_dot(a_, rhs, x, r_, level));
    residual(a_, rhs, x, r_, level);
    return std::sqrt(dot(r_, r_, level));
}

std::vector<double> Hierarchy::solve(Function& rhs, Function& x, int level, double tol, int max_cycles, int nu_pre,
                                     int nu_post, bool* converged) {
    if (level < a_.min_level() || level > a_.max_level())
        throw OutOfRange("solve: level " + std::to_string(level) + " outside the hierarchy");
    if (nu_pre < 0 || nu_post < 0) throw InvalidArgument("solve: negative smoothing count");
    std::vector<double> res{residual_norm(rhs, x, level)};
    const double r0 = res.front();
    const double target = r0 > 0.0 ? tol * r0 : tol;
    int it = 0;
    while (it < max_cycles && res.back() > target) {
        run_cycle(rhs, x, level, nu_pre, nu_post);
        ++it;
        res.push_back(residual_norm(rhs, x, level));
    }
    if (converged) *converged = res.back() <= target;
    return res;
}

// Full multigrid (configuration 4; no reference counterpart). Restatement:
// oracle/hyteg_oracle.c og_fmg.
std::vector<double> Hierarchy::fmg(Function& rhs, Function& x, int level, int per_level, int nu_pre, int nu_post,
                                   double tol, int max_cycles, bool* converged) {
    const int lmin = a_.min_level();
    if (level < lmin || level > a_.max_level()) throw OutOfRange("fmg: level " + std::to_string(level) + " outside the hierarchy");
    if (nu_pre < 0 || nu_post < 0 || per_level < 0 || max_cycles < 0)
        throw InvalidArgument("fmg: negative smoothing or cycle count");
    for (Function* f : {&rhs, &x}) {
        f->check_level(lmin, "fmg");
        f->check_level(level, "fmg");
    }
    if (&rhs == &x) throw InvalidArgument("fmg: rhs and x must be distinct functions");
    for (int l = level; l > lmin; --l) {
        restrict_to_coarse(rhs, rhs, l - 1, ALL_FLAGS);
        fill_const(rhs, 0.0, l - 1, kDirichletMask);
    }
    fill_const(x, 0.0, level, ALL_FLAGS);
    std::vector<double> res{residual_norm(rhs, x, level)};
    const double target = tol * res.front();
    fill_const(x, 0.0, lmin, ALL_FLAGS);
    run_cycle(rhs, x, lmin, nu_pre, nu_post);
    for (int l = lmin + 1; l <= level; ++l) {
        fill_const(x, 0.0, l, ALL_FLAGS);
        prolongate(x, x, l - 1, kSmoothMask, false);
        for (int i = 0; i < per_level; ++i) run_cycle(rhs, x, l, nu_pre, nu_post);
    }
    res.push_back(residual_norm(rhs, x, level));
    for (int it = 0; it < max_cycles && res.back() > target; ++it) {
        run_cycle(rhs, x, level, nu_pre, nu_post);
        res.push_back(residual_norm(rhs, x, level));
    }
    if (converged) *converged = res.back() <= target;
    return res;
}

// CG preconditioned by one V-cycle from zero (configuration 5): cg_solve's
// recurrence (reference src/solvers.cpp:226-259) with apply / dot on the
// device. Ap is held in the hierarchy's finest residual r_, which the cycle
// only needs after Ap has been consumed. Restatement: og_pcg.
std::vector<double> Hierarchy::pcg(Function& rhs, Function& x, int level, int max_iter, int nu_pre, int nu_post,
                                   double tol, bool* converged) {
    if (level < a_.min_level() || level > a_.max_level())
        throw OutOfRange("pcg: level " + std::to_string(level) + " outside the hierarchy");
    if (nu_pre < 0 || nu_post < 0 || max_iter < 0) throw InvalidArgument("pcg: negative smoothing or iteration count");
    if (&rhs == &x) throw InvalidArgument("pcg: rhs and x must be distinct functions");
    rhs.check_level(level, "pcg");
    x.check_level(level, "pcg");
    Domain& d = *dom_;
    if (!pcg_r_ || pcg_r_->min_level() != level) {
        pcg_r_.reset();
        pcg_z_.reset();
        pcg_p_.reset();
        pcg_r_ = std::make_unique<Function>(d, "pcg.r", level, level, a_.bc());
        pcg_z_ = std::make_unique<Function>(d, "pcg.z", level, level, a_.bc());
        pcg_p_ = std::make_unique<Function>(d, "pcg.p", level, level, a_.bc());
    }
    Function &r = *pcg_r_, &z = *pcg_z_, &p = *pcg_p_, &ap = r_;
    // the scalar recurrence stays on the device (k_pcg_scalars): an iteration
    // queues its kernels without waiting for the host; only a positive tol
    // reads each residual back for the stopping test
    if (pcg_s_.bytes() < sizeof(PcgScalars)) pcg_s_ = DevMem(sizeof(PcgScalars));
    if (int64_t(pcg_res_.bytes() / 8) < int64_t(max_iter) + 1) pcg_res_ = DevMem(size_t(max_iter + 1) * 8);
    PcgScalars* S = pcg_s_.as<PcgScalars>();
    double* R = pcg_res_.as<double>();
    HYB_CUDA(cudaMemsetAsync(S, 0, sizeof(PcgScalars), d.stream()));
    fill_const(x, 0.0, level, ALL_FLAGS);
    residual(a_, rhs, x, r, level);
    std::vector<double> res{std::sqrt(dot(r, r, level))};
    const double target = tol * res.front();
    run_cycle(r, z, level, nu_pre, nu_post, true); // z = M r from z = 0
    assign(1.0, z, 0.0, z, p, level, ALL_FLAGS);
    dot_dev(r, z, level, &S->rz);
    // r.z from the cycle's last post-smoothing sweep when it is a Jacobi sweep
    // at this level (its partials land in dot_scratch_), else a separate dot
    const bool fused_rz = smoother_ == SMOOTH_JACOBI && nu_post > 0 && level > a_.min_level();
    const LevelTables tl = a_.tables(level);
    const int slots = face_dot_slots(tl);
    const int64_t np = int64_t(d.graph().size());
    if (fused_rz && int64_t(dot_scratch_.bytes() / 8) < np + int64_t(tl.nfaces) * slots + 1)
        dot_scratch_ = DevMem(size_t(np + int64_t(tl.nfaces) * slots + 1) * 8);
    DevScalars beta_dev;
    beta_dev.pb = &S->beta;
    int done = 0;
    for (int k = 0; k < max_iter && res.front() > target; ++k) {
        apply_dot_dev(a_, p, ap, level, &S->pap); // Ap and p.Ap in one pass
        launch_pcg_scalars(0, S, R, k, d.stream()); // alpha = r.z / p.Ap
        pcg_update_dev(x, p, r, ap, 0.0, &S->alpha, level, &S->rr); // x += alpha p, r -= alpha Ap, r.r
        if (fused_rz) {
            double* part = dot_scratch_.as<double>();
            HYB_CUDA(cudaMemsetAsync(part, 0, size_t(np) * 8, d.stream()));
            cycle_dot_ = part + np;
            cycle_dot_level_ = level;
            try {
                run_cycle(r, z, level, nu_pre, nu_post, true);
            } catch (...) {
                cycle_dot_ = nullptr;
                cycle_dot_level_ = -1;
                throw;
            }
            cycle_dot_ = nullptr;
            cycle_dot_level_ = -1;
            finish_dot_dev(d, tl, r.data(level), z.data(level), part + np, slots, part, &S->rz_new);
        } else {
            run_cycle(r, z, level, nu_pre, nu_post, true);
            dot_dev(r, z, level, &S->rz_new);
        }
        launch_pcg_scalars(1, S, R, k + 1, d.stream()); // beta, rz, ||r_k+1||
        launch_blas1(0, tl, p.flags(), 1.0, z.data(level), 0.0, p.data(level), p.data(level), ALL_FLAGS, d.stream(),
                     beta_dev); // p = z + beta p
        done = k + 1;
        if (target > 0.0 && to_host(d, R + k + 1) <= target) break;
    }
    if (done > 0) {
        res.resize(size_t(done) + 1);
        HYB_CUDA(cudaMemcpyAsync(res.data() + 1, R + 1, size_t(done) * 8, cudaMemcpyDeviceToHost, d.stream()));
    }
    PcgScalars host{};
    HYB_CUDA(cudaMemcpyAsync(&host, S, sizeof host, cudaMemcpyDeviceToHost, d.stream()));
    HYB_CUDA(cudaStreamSynchronize(d.stream()));
    if (host.bad != 0.0)
        throw RuntimeError("pcg: non-positive curvature p.Ap at iteration " + std::to_string(int(host.bad) - 1));
    if (converged) *converged = res.back() <= target;
    return res;
}

} // namespace hyb
