// P2 stencil assembly (see p2.hpp). Restates the reference's P2 element
// matrices (src/elements.cpp:74-186) and its generic stencil assembly
// (src/operators.cpp:22-263) for FunctionKind::P2, term for term; only the
// storage position of each term is re-expressed in the level-(L+1) layout.
// Host code is compiled with -ffp-contract=off (every product and sum rounds
// separately, as in the reference's build).
#include "p2.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <tuple>

namespace hyb {

namespace {

// DoFGroup values of the reference (include/hytegrid/indexing.hpp:19-26)
enum Grp : int { GV = 0, GEH = 1, GED = 2, GEV = 3 };

struct Elem6 {
    double m[6][6] = {};
};

struct Geo {
    double area = 0;
    Vec2 grad[3];
};

Geo geometry(const std::array<Vec2, 3>& tri) {
    const Vec2 u1 = tri[1] - tri[0];
    const Vec2 u2 = tri[2] - tri[0];
    const double det = cross2(u1, u2);
    if (det == 0.0) throw InvalidArgument("local_stiffness: zero-area triangle");
    Geo g;
    g.area = std::abs(det) / 2.0;
    g.grad[1] = {u2.y / det, -u2.x / det};
    g.grad[2] = {-u1.y / det, u1.x / det};
    g.grad[0] = {-g.grad[1].x - g.grad[2].x, -g.grad[1].y - g.grad[2].y};
    return g;
}

// 6-point degree-4 rule (src/elements.cpp:78-96)
constexpr double kA1 = 0.44594849091596489;
constexpr double kW1 = 0.22338158967801147;
constexpr double kA2 = 0.091576213509770743;
constexpr double kW2 = 0.10995174365532187;
struct QP {
    double l[3];
    double w;
};
constexpr QP kQuad[6] = {
    {{1.0 - 2.0 * kA1, kA1, kA1}, kW1}, {{kA1, 1.0 - 2.0 * kA1, kA1}, kW1}, {{kA1, kA1, 1.0 - 2.0 * kA1}, kW1},
    {{1.0 - 2.0 * kA2, kA2, kA2}, kW2}, {{kA2, 1.0 - 2.0 * kA2, kA2}, kW2}, {{kA2, kA2, 1.0 - 2.0 * kA2}, kW2},
};

void p2_basis(const Geo& g, const double* l, double* phi, Vec2* grad) {
    for (int i = 0; i < 3; ++i) {
        phi[i] = l[i] * (2.0 * l[i] - 1.0);
        grad[i] = (4.0 * l[i] - 1.0) * g.grad[i];
    }
    static constexpr int pair[3][2] = {{0, 1}, {1, 2}, {2, 0}};
    for (int e = 0; e < 3; ++e) {
        const int i = pair[e][0], j = pair[e][1];
        phi[3 + e] = 4.0 * l[i] * l[j];
        grad[3 + e] = 4.0 * l[j] * g.grad[i] + 4.0 * l[i] * g.grad[j];
    }
}

Elem6 p2_matrix(Form form, const Geo& g) {
    Elem6 m;
    if (form == GRAD_X || form == GRAD_Y) {
        const Elem6 d = p2_matrix(form == GRAD_X ? DIV_X : DIV_Y, g);
        for (int i = 0; i < 6; ++i)
            for (int j = 0; j < 6; ++j) m.m[i][j] = d.m[j][i];
        return m;
    }
    const bool symmetric = form == LAPLACE || form == MASS || form == PSPG;
    const double scale = form == PSPG ? -(1.0 / 12.0) * 2.0 * g.area : 1.0;
    double phi[6];
    Vec2 grad[6];
    for (const QP& q : kQuad) {
        p2_basis(g, q.l, phi, grad);
        const double w = q.w * g.area * scale;
        for (int i = 0; i < 6; ++i) {
            const int jmax = symmetric ? i : 5;
            for (int j = 0; j <= jmax; ++j) {
                double integrand = 0;
                switch (form) {
                case LAPLACE:
                case PSPG: integrand = dot2(grad[i], grad[j]); break;
                case MASS: integrand = phi[i] * phi[j]; break;
                case DIV_X: integrand = -phi[i] * grad[j].x; break;
                case DIV_Y: integrand = -phi[i] * grad[j].y; break;
                default: throw InvalidArgument("local_stiffness: bad form");
                }
                m.m[i][j] += w * integrand;
            }
        }
    }
    if (symmetric)
        for (int i = 0; i < 6; ++i)
            for (int j = 0; j < i; ++j) m.m[j][i] = m.m[i][j];
    return m;
}

struct Mats {
    Elem6 up, down;
};
Mats micro_elements_p2(Form form, const std::array<Vec2, 3>& corners, int level) {
    const double inv = 1.0 / double(1 << level);
    const Vec2 u = inv * (corners[1] - corners[0]);
    const Vec2 v = inv * (corners[2] - corners[0]);
    return {p2_matrix(form, geometry({Vec2{0, 0}, u, v})), p2_matrix(form, geometry({u, v, u + v}))};
}

struct Dof {
    int g, dc, dr;
};
// cell_dofs (src/operators.cpp:24-42), element order v0, v1, v2, m01, m12, m20
constexpr Dof kUp[6] = {{GV, 0, 0}, {GV, 1, 0}, {GV, 0, 1}, {GEH, 0, 0}, {GED, 0, 0}, {GEV, 0, 0}};
constexpr Dof kDown[6] = {{GV, 1, 0}, {GV, 0, 1}, {GV, 1, 1}, {GED, 0, 0}, {GEH, 0, 1}, {GEV, 1, 0}};

struct Cell {
    bool up;
    int c, r;
};
// incident_cells (src/operators.cpp:50-62)
std::vector<Cell> incident(int g, int c, int r) {
    switch (g) {
    case GV:
        return {{true, c, r}, {true, c - 1, r}, {true, c, r - 1}, {false, c - 1, r}, {false, c, r - 1},
                {false, c - 1, r - 1}};
    case GEH: return {{true, c, r}, {false, c, r - 1}};
    case GED: return {{true, c, r}, {false, c, r}};
    default: return {{true, c, r}, {false, c - 1, r}};
    }
}
bool inside(const Cell& t, int n) { return t.c >= 0 && t.r >= 0 && t.c + t.r <= (t.up ? n - 1 : n - 2); }

int recv_index(const Cell& cell, int g, int c, int r) {
    const Dof* d = cell.up ? kUp : kDown;
    int irecv = -1;
    for (int i = 0; i < 6; ++i)
        if (d[i].g == g && cell.c + d[i].dc == c && cell.r + d[i].dr == r) irecv = i;
    if (irecv < 0) throw LogicError("P2 stencil assembly: receiving DoF missing from its cell");
    return irecv;
}

// fine-lattice position of a group DoF (group_lattice_coord x 2)
void fine(int g, int c, int r, int& fc, int& fr) {
    fc = 2 * c + ((g == GEH || g == GED) ? 1 : 0);
    fr = 2 * r + ((g == GED || g == GEV) ? 1 : 0);
}
int base_width(int g, int n) { return g == GV ? n + 1 : n; }
int parallel_group(int slot) { return slot == 0 ? GEH : slot == 1 ? GEV : GED; }
int border_offset(int g, int n, int slot, int c, int r) {
    return slot == 0 ? r : slot == 1 ? c : (base_width(g, n) - 1) - (c + r);
}
int walk(int slot, int c, int r) { return slot == 0 ? c : r; }
int row_length(int g, int n, int o) { return std::max(base_width(g, n) - o, 0); }

// the reference's P2 edge halo rows of a face at `slot` (src/layout.cpp:40-52)
std::vector<std::pair<int, int>> halo_rows(int slot) {
    const int par = parallel_group(slot);
    std::vector<std::pair<int, int>> rows{{GV, 0}, {par, 0}, {GV, 1}, {par, 1}};
    for (int g : {GEH, GED, GEV})
        if (g != par) rows.push_back({g, 0});
    return rows;
}
int halo_block(int n, int slot) {
    int s = 0;
    for (auto [g, o] : halo_rows(slot)) s += row_length(g, n, o);
    return s;
}
int halo_row_offset(int n, int slot, int g, int o) {
    int s = 0;
    for (auto [hg, ho] : halo_rows(slot)) {
        if (hg == g && ho == o) return s;
        s += row_length(hg, n, ho);
    }
    throw LogicError("P2 edge stencil: no halo row for the coupled DoF");
}

} // namespace

// assemble_face (src/operators.cpp:95-120), P2
P2FaceStencil assemble_p2_face(Form form, const MacroFace& f, int level) {
    const Mats E = micro_elements_p2(form, f.coord, level);
    P2FaceStencil s;
    for (int g : {GV, GEH, GED, GEV}) {
        std::map<std::tuple<int, int, int>, double> acc;
        for (const Cell& cell : incident(g, 0, 0)) {
            const Dof* d = cell.up ? kUp : kDown;
            const Elem6& M = cell.up ? E.up : E.down;
            const int irecv = recv_index(cell, g, 0, 0);
            for (int j = 0; j < 6; ++j) acc[{d[j].g, cell.c + d[j].dc, cell.r + d[j].dr}] += M.m[irecv][j];
        }
        int c0, r0;
        fine(g, 0, 0, c0, r0);
        const int cls = (c0 & 1) + 2 * (r0 & 1);
        for (const auto& [key, coeff] : acc) {
            const auto [ng, dc, dr] = key;
            int fc, fr;
            fine(ng, dc, dr, fc, fr);
            s.cls[cls].push_back({fc - c0, fr - r0, coeff});
        }
        s.diag[cls] = acc.at({g, 0, 0});
    }
    return s;
}

// assemble_edge + accumulate_edge_row + edge_position (src/operators.cpp:122-200), P2
P2EdgeStencil assemble_p2_edge(Form form, const MacroEdge& e, int level) {
    const int n = 1 << level, n2 = 2 * n;
    using Key = std::pair<long, long>;
    std::map<Key, double> line_acc, mid_acc;
    std::map<Key, std::pair<int, int>> line_pos, mid_pos; // reference key -> (base, dk) here
    const long ref_line = 2L * n + 1;                     // edge_line_size(P2)
    const long ref_mid = n + 1;                           // edge_midline_offset
    for (size_t fi = 0; fi < e.faces.size(); ++fi) {
        const FaceSide& nb = e.faces[fi];
        const Mats E = micro_elements_p2(form, nb.corners, level);
        long ref_halo = ref_line;
        for (size_t j = 0; j < fi; ++j) ref_halo += halo_block(n, e.faces[j].slot);
        auto row = [&](std::map<Key, double>& acc, std::map<Key, std::pair<int, int>>& pos, int rg, int w0, int k0,
                       int kf) {
            // receiving border DoF (border_dof, src/indexing.cpp:61-72)
            const int bw = base_width(rg, n);
            const int rc = nb.slot == 0 ? w0 : nb.slot == 1 ? 0 : (bw - 1) - w0;
            const int rr = nb.slot == 0 ? 0 : w0;
            for (const Cell& cell : incident(rg, rc, rr)) {
                if (!inside(cell, n)) continue;
                const Dof* d = cell.up ? kUp : kDown;
                const Elem6& M = cell.up ? E.up : E.down;
                const int irecv = recv_index(cell, rg, rc, rr);
                for (int j = 0; j < 6; ++j) {
                    const int g = d[j].g, c = cell.c + d[j].dc, r = cell.r + d[j].dr;
                    const int o = border_offset(g, n, nb.slot, c, r);
                    const int w = walk(nb.slot, c, r);
                    long base, entry;
                    if (g == GV && o == 0) {
                        base = 0;
                        entry = nb.aligned ? w : n - w;
                    } else if (g == parallel_group(nb.slot) && o == 0) {
                        base = ref_mid;
                        entry = nb.aligned ? w : (n - 1) - w;
                    } else {
                        const int len = row_length(g, n, o);
                        base = ref_halo + halo_row_offset(n, nb.slot, g, o);
                        entry = nb.aligned ? w : (len - 1) - w;
                    }
                    const Key key{base, entry - k0};
                    acc[key] += M.m[irecv][j];
                    // the same DoF in the fine layout
                    int fc, fr;
                    fine(g, c, r, fc, fr);
                    const int dist = nb.slot == 0 ? fr : nb.slot == 1 ? fc : n2 - (fc + fr);
                    const int fw = nb.slot == 0 ? fc : fr;
                    int mb, idx;
                    if (dist == 0) {
                        mb = 0;
                        idx = nb.aligned ? fw : n2 - fw;
                    } else if (dist == 1) {
                        mb = p2_edge_halo1(n2, int(fi));
                        idx = nb.aligned ? fw : (n2 - 1) - fw;
                    } else if (dist == 2) {
                        mb = p2_edge_halo2(n2, int(fi));
                        idx = nb.aligned ? fw : (n2 - 2) - fw;
                    } else {
                        throw LogicError("P2 edge stencil: coupling beyond fine halo row 2");
                    }
                    const std::pair<int, int> mine{mb, idx - kf};
                    const auto it = pos.find(key);
                    if (it == pos.end()) pos.emplace(key, mine);
                    else if (it->second != mine) throw LogicError("P2 edge stencil: inconsistent term position");
                }
            }
        };
        if (n >= 2) row(line_acc, line_pos, GV, nb.aligned ? 1 : n - 1, 1, 2);
        row(mid_acc, mid_pos, parallel_group(nb.slot), nb.aligned ? 0 : (n - 1), 0, 1);
    }
    P2EdgeStencil s;
    for (const auto& [key, coeff] : line_acc) s.line.push_back({line_pos[key].first, line_pos[key].second, coeff});
    for (const auto& [key, coeff] : mid_acc) s.mid.push_back({mid_pos[key].first, mid_pos[key].second, coeff});
    if (!line_acc.empty()) s.line_diag = line_acc.at({0, 0});
    s.mid_diag = mid_acc.at({ref_mid, 0});
    return s;
}

// assemble_vertex (src/operators.cpp:209-263), P2
P2VertexStencil assemble_p2_vertex(Form form, const MacroVertex& v, int level) {
    const int n = 1 << level;
    static constexpr int corner_slots[3][2] = {{0, 1}, {0, 2}, {1, 2}};
    std::map<size_t, double> acc;
    const size_t ne = v.edges.size();
    for (size_t fvi = 0; fvi < v.faces.size(); ++fvi) {
        const CornerFace& cf = v.faces[fvi];
        const Elem6 M = micro_elements_p2(form, cf.corners, level).up;
        const int ci = cf.corner;
        const Cell cell = ci == 0 ? Cell{true, 0, 0} : ci == 1 ? Cell{true, n - 1, 0} : Cell{true, 0, n - 1};
        for (int j = 0; j < 6; ++j) {
            const double coeff = M.m[ci][j];
            if (j == ci) {
                acc[0] += coeff;
                continue;
            }
            const int g = kUp[j].g, c = cell.c + kUp[j].dc, r = cell.r + kUp[j].dr;
            auto edge_slot = [&](int pick) {
                const uint64_t eid = cf.flank[pick == corner_slots[ci][0] ? 0 : 1];
                const auto it = std::find(v.edges.begin(), v.edges.end(), eid);
                if (it == v.edges.end()) throw LogicError("P2 vertex stencil: flank edge not incident");
                return 1 + 2 * size_t(it - v.edges.begin());
            };
            int pick = -1;
            if (g == GV) {
                for (int s : corner_slots[ci])
                    if (border_offset(g, n, s, c, r) == 0) {
                        pick = s;
                        break;
                    }
                if (pick < 0) throw LogicError("P2 vertex stencil: neighbour vertex off the flank borders");
                acc[edge_slot(pick)] += coeff;
                continue;
            }
            for (int s : corner_slots[ci])
                if (g == parallel_group(s) && border_offset(g, n, s, c, r) == 0) {
                    pick = s;
                    break;
                }
            if (pick >= 0) acc[edge_slot(pick) + 1] += coeff;
            else acc[1 + 2 * ne + fvi] += coeff;
        }
    }
    P2VertexStencil s;
    for (const auto& [slot, coeff] : acc) s.terms.push_back({int(slot), coeff});
    s.diag = acc.at(0);
    return s;
}

} // namespace hyb
