// Coarse-grid system assembly (see coarse.hpp).
#include "coarse.hpp"

#include <map>

namespace hyb {

HostRows assemble_rows(const MacroGraph& g, Form form, int L, const BoundaryMap& bc) {
    const int n = 1 << L, W = n + 1;
    HostRows m;
    m.n = int64_t(g.nv()) + int64_t(g.ne()) * (n - 1) + int64_t(g.nf()) * ((int64_t(n) - 1) * (n - 2) / 2);
    if (m.n > (int64_t(1) << 30)) throw InvalidArgument("coarse system too large for the device coarse solver");
    m.flag.assign(size_t(m.n), INNER);
    m.rows.resize(size_t(m.n));
    auto& rows = m.rows;
    auto gi = [&](const OwnerSlot& o) { return global_owned_index(g, o, n); };

    // vertex rows: own + one ghost per incident edge (src/operators.cpp:275-281)
    for (size_t v = 0; v < g.nv(); ++v) {
        const MacroVertex& mv = g.vertices[v];
        const int64_t row = gi({v, 0, 0});
        m.flag[size_t(row)] = bc.flag_for(mv.marker);
        const VertexStencil s = assemble_vertex_stencil(form, mv, L);
        auto& acc = rows[size_t(row)];
        acc[row] += s.c[0];
        for (size_t j = 0; j < mv.edges.size(); ++j) {
            const MacroEdge& e = g.edges[g.edge_index(mv.edges[j])];
            acc[gi(resolve_edge(g, mv.edges[j], e.v[0] == v ? 1 : n - 1, n))] += s.c[1 + j];
        }
    }
    // edge line rows: k-1, k, k+1, then per face halo row 1 at k-1, k (:283-292)
    for (size_t ei = 0; ei < g.ne() && n >= 2; ++ei) {
        const uint64_t eid = g.edge_id(ei);
        const MacroEdge& e = g.edges[ei];
        const EdgeStencil s = assemble_edge_stencil(form, g, e, L);
        const uint8_t fl = bc.flag_for(e.marker);
        for (int k = 1; k <= n - 1; ++k) {
            const int64_t row = gi({eid, k, 0});
            m.flag[size_t(row)] = fl;
            auto& acc = rows[size_t(row)];
            acc[gi(resolve_edge(g, eid, k - 1, n))] += s.c[0];
            acc[gi(resolve_edge(g, eid, k, n))] += s.c[1];
            acc[gi(resolve_edge(g, eid, k + 1, n))] += s.c[2];
            for (size_t j = 0; j < e.faces.size(); ++j) {
                const FaceSide& fs = e.faces[j];
                for (int t = 0; t < 2; ++t) {
                    const int q = k - 1 + t;                  // halo row 1 entry, edge order
                    const int w = fs.aligned ? q : n - 1 - q; // face walk position
                    const int c = fs.slot == 0 ? w : (fs.slot == 1 ? 1 : W - 2 - w);
                    const int r = fs.slot == 0 ? 1 : w;
                    acc[gi(resolve_face(g, fs.face, c, r, n))] += s.c[3 + 2 * j + t];
                }
            }
        }
    }
    // face rows: W NW S C N SE E (:308-316)
    static const int off[7][2] = {{-1, 0}, {-1, 1}, {0, -1}, {0, 0}, {0, 1}, {1, -1}, {1, 0}};
    for (size_t fi = 0; fi < g.nf(); ++fi) {
        const uint64_t fid = g.face_id(fi);
        const FaceStencil s = assemble_face_stencil(form, g.faces[fi], L);
        for (int r = 1; r <= n - 2; ++r)
            for (int c = 1; c + r <= n - 1; ++c) {
                const int64_t row = gi({fid, c, r});
                auto& acc = rows[size_t(row)];
                for (int t = 0; t < 7; ++t) acc[gi(resolve_face(g, fid, c + off[t][0], r + off[t][1], n))] += s.c[t];
            }
    }
    return m;
}

namespace {
// constrain_dirichlet (src/solvers.cpp:322-352) on rows whose DIRICHLET rows
// are already identities: DIRICHLET columns dropped from every other row
HostCsr constrained_csr(const std::vector<std::map<int64_t, double>>& rows, const std::vector<uint8_t>& flag) {
    HostCsr m;
    m.n = int64_t(rows.size());
    m.flag = flag;
    m.rowptr.push_back(0);
    for (int64_t row = 0; row < m.n; ++row) {
        if (m.flag[size_t(row)] & DIRICHLET) {
            m.col.push_back(int32_t(row));
            m.val.push_back(1.0);
        } else {
            for (const auto& [col, v] : rows[size_t(row)]) {
                if (m.flag[size_t(col)] & DIRICHLET) continue;
                m.col.push_back(int32_t(col));
                m.val.push_back(v);
            }
        }
        m.rowptr.push_back(int32_t(m.col.size()));
    }
    return m;
}
} // namespace

HostCsr assemble_constrained(const MacroGraph& g, Form form, int L, const BoundaryMap& bc) {
    const HostRows r = assemble_rows(g, form, L, bc);
    return constrained_csr(r.rows, r.flag);
}

// assemble_stokes_sparse (src/solvers.cpp:548-576) + constrain_dirichlet with
// the flags (u, u, p) (:578-592): blocks at offsets 0, N, 2N
HostCsr assemble_stokes_constrained(const MacroGraph& g, int L, const BoundaryMap& bc_u, const BoundaryMap& bc_p) {
    const HostRows A = assemble_rows(g, LAPLACE, L, bc_u);
    const HostRows Gx = assemble_rows(g, GRAD_X, L, bc_u);
    const HostRows Gy = assemble_rows(g, GRAD_Y, L, bc_u);
    const HostRows Bx = assemble_rows(g, DIV_X, L, bc_p);
    const HostRows By = assemble_rows(g, DIV_Y, L, bc_p);
    const HostRows C = assemble_rows(g, PSPG, L, bc_p);
    const int64_t n = A.n;
    if (3 * n > (int64_t(1) << 30)) throw InvalidArgument("coarse Stokes system too large for the device solver");
    std::vector<std::map<int64_t, double>> M(size_t(3 * n));
    std::vector<uint8_t> f3(size_t(3 * n));
    for (int64_t r = 0; r < n; ++r) {
        const uint8_t fu = A.flag[size_t(r)], fp = C.flag[size_t(r)];
        f3[size_t(r)] = fu;
        f3[size_t(n + r)] = fu;
        f3[size_t(2 * n + r)] = fp;
        if (fu & DIRICHLET) {
            M[size_t(r)][r] = 1.0;
            M[size_t(n + r)][n + r] = 1.0;
        } else {
            for (const auto& [c, v] : A.rows[size_t(r)]) {
                M[size_t(r)][c] += v;
                M[size_t(n + r)][n + c] += v;
            }
            for (const auto& [c, v] : Gx.rows[size_t(r)]) M[size_t(r)][2 * n + c] += v;
            for (const auto& [c, v] : Gy.rows[size_t(r)]) M[size_t(n + r)][2 * n + c] += v;
        }
        if (fp & DIRICHLET) {
            M[size_t(2 * n + r)][2 * n + r] = 1.0;
        } else {
            for (const auto& [c, v] : Bx.rows[size_t(r)]) M[size_t(2 * n + r)][c] += v;
            for (const auto& [c, v] : By.rows[size_t(r)]) M[size_t(2 * n + r)][n + c] += v;
            for (const auto& [c, v] : C.rows[size_t(r)]) M[size_t(2 * n + r)][2 * n + c] += v;
        }
    }
    return constrained_csr(M, f3);
}

} // namespace hyb
