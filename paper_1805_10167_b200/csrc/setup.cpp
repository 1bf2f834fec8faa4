// Host setup: see setup.hpp for the reference anchors of every function here.
#include "setup.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numbers>
#include <set>
#include <sstream>

namespace hyb {

// =====================================================================
// Mesh text (reference src/mesh.cpp:22-83)
// =====================================================================
namespace {

struct LineReader {
    std::istringstream in;
    size_t lineno = 0;
    explicit LineReader(const std::string& t) : in(t) {}

    // Next non-blank line with comments removed; throws at end of input.
    std::string next(const char* expecting) {
        std::string raw;
        while (std::getline(in, raw)) {
            ++lineno;
            const auto h = raw.find('#');
            if (h != std::string::npos) raw.resize(h);
            if (raw.find_first_not_of(" \t\r\n") != std::string::npos) return raw;
        }
        throw InvalidArgument("mesh parse error, line " + std::to_string(lineno) +
                              ": unexpected end of input, expected " + expecting);
    }
    [[noreturn]] void fail(const std::string& what) const {
        throw InvalidArgument("mesh parse error, line " + std::to_string(lineno) + ": " + what);
    }
};

} // namespace

CoarseMesh parse_mesh_text(const std::string& text) {
    LineReader rd(text);
    CoarseMesh m;
    long long nv = 0, nt = 0;
    {
        std::istringstream ls(rd.next("header 'NV NT'"));
        if (!(ls >> nv >> nt) || nv < 0 || nt < 0) rd.fail("header must be two non-negative integers 'NV NT'");
    }
    m.pos.resize(size_t(nv));
    m.marker.resize(size_t(nv));
    for (long long i = 0; i < nv; ++i) {
        std::istringstream ls(rd.next("vertex line 'x y marker'"));
        if (!(ls >> m.pos[size_t(i)].x >> m.pos[size_t(i)].y >> m.marker[size_t(i)]))
            rd.fail("vertex line must be 'x y marker'");
    }
    std::set<std::array<int, 3>> seen;
    for (long long i = 0; i < nt; ++i) {
        std::istringstream ls(rd.next("triangle line 'v0 v1 v2 region'"));
        std::array<int, 3> t{};
        int region = 0;
        if (!(ls >> t[0] >> t[1] >> t[2] >> region)) rd.fail("triangle line must be 'v0 v1 v2 region'");
        for (int v : t)
            if (v < 0 || v >= nv) rd.fail("vertex index " + std::to_string(v) + " out of range");
        if (t[0] == t[1] || t[1] == t[2] || t[0] == t[2]) rd.fail("triangle references a vertex twice");
        const Vec2 a = m.pos[size_t(t[0])], b = m.pos[size_t(t[1])], c = m.pos[size_t(t[2])];
        const double area2 = cross2(b - a, c - a);
        if (area2 == 0.0) rd.fail("degenerate (zero-area) triangle");
        if (area2 < 0.0) std::swap(t[1], t[2]); // canonical CCW, v0 kept
        std::array<int, 3> key = t;
        std::sort(key.begin(), key.end());
        if (!seen.insert(key).second) rd.fail("duplicate triangle (same vertex set)");
        m.tri.push_back(t);
        m.region.push_back(region);
    }
    return m;
}

// =====================================================================
// Macro-primitive graph (reference src/mesh.cpp:97-263)
// =====================================================================
namespace {
// slot -> (first, second) local corner of the border walk
constexpr int kSlotCorner[3][2] = {{0, 1}, {0, 2}, {1, 2}};
// local corner -> the two slots meeting there
constexpr int kCornerSlots[3][2] = {{0, 1}, {0, 2}, {1, 2}};
} // namespace

MacroGraph build_macro_graph(const CoarseMesh& mesh) {
    MacroGraph g;
    const size_t nv = mesh.pos.size(), nf = mesh.tri.size();

    // Edge identity = sorted vertex pair; lexicographic pair order fixes IDs.
    std::map<std::pair<int, int>, std::vector<int>> incident;
    for (size_t ti = 0; ti < nf; ++ti) {
        const auto& t = mesh.tri[ti];
        for (int s = 0; s < 3; ++s) {
            const int a = t[size_t(kSlotCorner[s][0])], b = t[size_t(kSlotCorner[s][1])];
            incident[std::minmax(a, b)].push_back(int(ti));
        }
    }
    std::map<std::pair<int, int>, size_t> eidx;
    for (const auto& [pr, fl] : incident) {
        if (fl.size() > 2)
            throw InvalidArgument("non-manifold mesh: edge (" + std::to_string(pr.first) + "," +
                                  std::to_string(pr.second) + ") shared by " + std::to_string(fl.size()) +
                                  " triangles");
        const size_t i = eidx.size();
        eidx[pr] = i;
    }
    const size_t ne = eidx.size();
    g.vertices.resize(nv);
    g.edges.resize(ne);
    g.faces.resize(nf);
    const uint64_t ebase = nv, fbase = nv + ne;

    for (size_t ti = 0; ti < nf; ++ti) {
        const auto& t = mesh.tri[ti];
        MacroFace& f = g.faces[ti];
        for (int k = 0; k < 3; ++k) {
            f.v[size_t(k)] = uint64_t(t[size_t(k)]);
            f.coord[size_t(k)] = mesh.pos[size_t(t[size_t(k)])];
            f.vmarker[size_t(k)] = mesh.marker[size_t(t[size_t(k)])];
        }
        for (int s = 0; s < 3; ++s) {
            const int a = t[size_t(kSlotCorner[s][0])], b = t[size_t(kSlotCorner[s][1])];
            f.e[size_t(s)] = ebase + eidx.at(std::minmax(a, b));
            f.aligned[size_t(s)] = a < b; // intrinsic direction runs low -> high vertex ID
        }
    }

    for (const auto& [pr, fl] : incident) {
        const size_t ei = eidx.at(pr);
        const uint64_t id = ebase + ei;
        MacroEdge& e = g.edges[ei];
        e.v = {uint64_t(pr.first), uint64_t(pr.second)};
        e.coord = {mesh.pos[size_t(pr.first)], mesh.pos[size_t(pr.second)]};
        e.vmarker = {mesh.marker[size_t(pr.first)], mesh.marker[size_t(pr.second)]};
        // boundary iff one adjacent face and both ends flagged; larger flag wins
        e.marker = (fl.size() == 1 && e.vmarker[0] != 0 && e.vmarker[1] != 0)
                       ? std::max(e.vmarker[0], e.vmarker[1])
                       : 0;
        std::vector<int> sorted = fl;
        std::sort(sorted.begin(), sorted.end());
        for (int ti : sorted) {
            const MacroFace& f = g.faces[size_t(ti)];
            FaceSide side;
            side.face = fbase + uint64_t(ti);
            side.corners = f.coord;
            for (int s = 0; s < 3; ++s)
                if (f.e[size_t(s)] == id) {
                    side.slot = s;
                    side.aligned = f.aligned[size_t(s)];
                }
            e.faces.push_back(side);
        }
    }
    for (auto& f : g.faces)
        for (int s = 0; s < 3; ++s) f.emarker[size_t(s)] = g.edges[size_t(f.e[size_t(s)] - ebase)].marker;

    for (size_t v = 0; v < nv; ++v) {
        g.vertices[v].coord = mesh.pos[v];
        g.vertices[v].marker = mesh.marker[v];
    }
    for (size_t ei = 0; ei < ne; ++ei) { // edge-ID order keeps vertex edge lists sorted
        const MacroEdge& e = g.edges[ei];
        for (int end = 0; end < 2; ++end) {
            MacroVertex& mv = g.vertices[size_t(e.v[size_t(end)])];
            mv.edges.push_back(ebase + ei);
            mv.edge_marker.push_back(e.marker);
            mv.edge_far_marker.push_back(e.vmarker[size_t(1 - end)]);
        }
    }
    for (size_t ti = 0; ti < nf; ++ti) {
        const MacroFace& f = g.faces[ti];
        for (int k = 0; k < 3; ++k) {
            CornerFace cf;
            cf.face = fbase + ti;
            cf.corners = f.coord;
            cf.corner = k;
            cf.flank = {f.e[size_t(kCornerSlots[k][0])], f.e[size_t(kCornerSlots[k][1])]};
            g.vertices[size_t(f.v[size_t(k)])].faces.push_back(cf);
        }
    }
    return g;
}

// =====================================================================
// Fixture meshes (reference src/meshgen.cpp:50-141), emitted in the mesh
// text format with 17 significant digits so coordinates round-trip exactly.
// =====================================================================
namespace meshgen {
namespace {

struct TextMesh {
    std::vector<std::array<double, 2>> p;
    std::vector<int> mk;
    std::vector<std::array<int, 3>> t;

    int add(double x, double y, int marker) {
        p.push_back({x, y});
        mk.push_back(marker);
        return int(p.size()) - 1;
    }
    void tri(int a, int b, int c) { t.push_back({a, b, c}); }

    std::string text(const std::string& title) const {
        std::string s = "# " + title + "\n" + std::to_string(p.size()) + " " + std::to_string(t.size()) + "\n";
        char buf[96];
        for (size_t i = 0; i < p.size(); ++i) {
            std::snprintf(buf, sizeof buf, "%.17g %.17g %d\n", p[i][0], p[i][1], mk[i]);
            s += buf;
        }
        for (const auto& tr : t) {
            std::snprintf(buf, sizeof buf, "%d %d %d 0\n", tr[0], tr[1], tr[2]);
            s += buf;
        }
        return s;
    }
};

} // namespace

std::string unit_triangle() {
    TextMesh m;
    m.add(0, 0, 1);
    m.add(1, 0, 1);
    m.add(0, 1, 1);
    m.tri(0, 1, 2);
    return m.text("reference right triangle");
}

std::string unit_square() {
    TextMesh m;
    m.add(0, 0, 1);
    m.add(1, 0, 1);
    m.add(1, 1, 1);
    m.add(0, 1, 1);
    m.tri(0, 1, 2);
    m.tri(0, 2, 3);
    return m.text("unit square, two triangles");
}

std::string unit_square_reversed() {
    TextMesh m;
    m.add(0, 0, 1);
    m.add(1, 0, 1);
    m.add(1, 1, 1);
    m.add(0, 1, 1);
    m.tri(0, 1, 2);
    m.tri(2, 3, 0); // shared diagonal walked against its intrinsic direction
    return m.text("unit square, reversed shared-edge orientation");
}

std::string square_ring8() {
    TextMesh m;
    const double outer[4][2] = {{0, 0}, {3, 0}, {3, 3}, {0, 3}};
    const double inner[4][2] = {{1, 1}, {2, 1}, {2, 2}, {1, 2}};
    int o[4], in[4];
    for (int k = 0; k < 4; ++k) o[k] = m.add(outer[k][0], outer[k][1], 1);
    for (int k = 0; k < 4; ++k) in[k] = m.add(inner[k][0], inner[k][1], 2);
    // side k of the ring: outer k -> outer k+1, inner k+1, inner k
    const int nxt[4] = {1, 2, 3, 0};
    const int ia[4] = {1, 2, 3, 0}; // inner vertex across from outer side k's second corner
    const int ib[4] = {0, 1, 2, 3};
    for (int k = 0; k < 4; ++k) {
        m.tri(o[k], o[nxt[k]], in[ia[k]]);
        m.tri(o[k], in[ia[k]], in[ib[k]]);
    }
    return m.text("square ring of 8 triangles (one hole)");
}

std::string channel(int nx, int ny, double width, double height) {
    if (nx < 1 || ny < 1) throw InvalidArgument("channel: nx and ny must be >= 1");
    TextMesh m;
    for (int j = 0; j <= ny; ++j)
        for (int i = 0; i <= nx; ++i) {
            const int marker = i == 0 ? 1 : (j == 0 || j == ny) ? 2 : (i == nx ? 3 : 0);
            m.add(width * i / nx, height * j / ny, marker);
        }
    const auto at = [&](int i, int j) { return j * (nx + 1) + i; };
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            m.tri(at(i, j), at(i + 1, j), at(i + 1, j + 1));
            m.tri(at(i, j), at(i + 1, j + 1), at(i, j + 1));
        }
    return m.text("channel");
}

std::string annulus(int segments, int layers, double r_inner, double r_outer) {
    if (segments < 3 || layers < 1) throw InvalidArgument("annulus: need segments >= 3 and layers >= 1");
    if (!(0.0 < r_inner && r_inner < r_outer)) throw InvalidArgument("annulus: need 0 < r_inner < r_outer");
    TextMesh m;
    for (int ring = 0; ring <= layers; ++ring) {
        const double r = r_inner + (r_outer - r_inner) * ring / layers;
        const int marker = ring == 0 ? 1 : (ring == layers ? 2 : 0);
        for (int s = 0; s < segments; ++s) {
            const double a = 2.0 * std::numbers::pi * s / segments;
            m.add(r * std::cos(a), r * std::sin(a), marker);
        }
    }
    const auto at = [&](int ring, int s) { return ring * segments + (s % segments); };
    for (int ring = 0; ring < layers; ++ring)
        for (int s = 0; s < segments; ++s) {
            m.tri(at(ring, s), at(ring, s + 1), at(ring + 1, s + 1));
            m.tri(at(ring, s), at(ring + 1, s + 1), at(ring + 1, s));
        }
    return m.text("annulus " + std::to_string(segments) + "x" + std::to_string(layers));
}

namespace {
uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
double unit_pm1(uint64_t h) { return 2.0 * (double(h >> 11) * 0x1p-53) - 1.0; }
} // namespace

std::string perturb_interior(const std::string& mesh_text, double frac, uint64_t seed) {
    CoarseMesh m = parse_mesh_text(mesh_text);
    const size_t nv = m.pos.size();
    std::vector<double> h(nv, INFINITY);
    for (const auto& t : m.tri)
        for (int s = 0; s < 3; ++s) {
            const int a = t[size_t(kSlotCorner[s][0])], b = t[size_t(kSlotCorner[s][1])];
            const Vec2 d = m.pos[size_t(a)] - m.pos[size_t(b)];
            const double len = std::sqrt(dot2(d, d));
            h[size_t(a)] = std::min(h[size_t(a)], len);
            h[size_t(b)] = std::min(h[size_t(b)], len);
        }
    std::vector<Vec2> np = m.pos;
    for (size_t v = 0; v < nv; ++v) {
        if (m.marker[v] != 0 || !std::isfinite(h[v])) continue;
        const double dx = frac * h[v] * unit_pm1(mix64(mix64(seed) ^ (uint64_t(v) << 1)));
        const double dy = frac * h[v] * unit_pm1(mix64(mix64(seed) ^ ((uint64_t(v) << 1) | 1)));
        np[v] = {m.pos[v].x + dx, m.pos[v].y + dy};
    }
    TextMesh out;
    for (size_t v = 0; v < nv; ++v) out.add(np[v].x, np[v].y, m.marker[v]);
    for (const auto& t : m.tri) {
        const double a2 = cross2(np[size_t(t[1])] - np[size_t(t[0])], np[size_t(t[2])] - np[size_t(t[0])]);
        if (!(a2 > 0.0)) throw RuntimeError("perturb_interior: perturbation inverted a triangle");
        out.tri(t[0], t[1], t[2]);
    }
    return out.text("perturbed mesh");
}

} // namespace meshgen

// =====================================================================
// Partitioning (reference src/balancing.cpp:19-137)
// =====================================================================
std::vector<int> partition_round_robin(const MacroGraph& g, int ranks) {
    if (ranks < 1) throw InvalidArgument("partition_round_robin: need at least one rank");
    std::vector<int> a(g.size());
    for (size_t i = 0; i < g.nv(); ++i) a[i] = int(i % size_t(ranks));
    for (size_t i = 0; i < g.ne(); ++i) a[g.edge_id(i)] = int(i % size_t(ranks));
    for (size_t i = 0; i < g.nf(); ++i) a[g.face_id(i)] = int(i % size_t(ranks));
    return a;
}

namespace {
double owned_weight(Kind k, int level) {
    if (level < 1) throw InvalidArgument("owned_count: level must be >= 1");
    const double n = double(1 << level);
    switch (k) {
    case VERTEX: return 1.0;
    case EDGE: return n - 1.0;
    case FACE: return (n - 1.0) * (n - 2.0) / 2.0;
    }
    return 0.0;
}
} // namespace

std::vector<int> partition_greedy_edgecut(const MacroGraph& g, int ranks, int weight_level) {
    if (ranks < 1) throw InvalidArgument("partition_greedy_edgecut: need at least one rank");
    const size_t nf = g.nf();
    std::vector<std::vector<size_t>> adj(nf);
    for (const auto& e : g.edges)
        if (e.faces.size() == 2) {
            const size_t a = g.face_index(e.faces[0].face), b = g.face_index(e.faces[1].face);
            adj[a].push_back(b);
            adj[b].push_back(a);
        }
    // a face carries the edges / vertices that will be co-located with it
    std::vector<double> eff(nf, owned_weight(FACE, weight_level));
    for (const auto& e : g.edges) eff[g.face_index(e.faces.front().face)] += owned_weight(EDGE, weight_level);
    for (const auto& v : g.vertices)
        if (!v.faces.empty()) eff[g.face_index(v.faces.front().face)] += owned_weight(VERTEX, weight_level);

    double remaining = 0.0;
    std::set<size_t> open;
    for (size_t f = 0; f < nf; ++f) {
        open.insert(f);
        remaining += eff[f];
    }
    std::vector<int> face_rank(nf, ranks - 1);
    for (int r = 0; r + 1 < ranks && !open.empty(); ++r) {
        const double target = remaining / double(ranks - r);
        double grabbed = 0.0;
        std::set<size_t> front;
        while (!open.empty()) {
            size_t pick = 0;
            double best = 0.0;
            bool found = false;
            for (size_t f : front) {
                const double d = std::abs(grabbed + eff[f] - target);
                if (!found || d < best) {
                    pick = f;
                    best = d;
                    found = true;
                }
            }
            if (!found) {
                pick = *open.begin();
                best = std::abs(grabbed + eff[pick] - target);
            }
            if (grabbed > 0.0 && best >= std::abs(grabbed - target)) break;
            face_rank[pick] = r;
            grabbed += eff[pick];
            remaining -= eff[pick];
            open.erase(pick);
            front.erase(pick);
            for (size_t nb : adj[pick])
                if (open.count(nb)) front.insert(nb);
        }
    }
    std::vector<int> a(g.size());
    for (size_t f = 0; f < nf; ++f) a[g.face_id(f)] = face_rank[f];
    for (size_t i = 0; i < g.ne(); ++i) a[g.edge_id(i)] = face_rank[g.face_index(g.edges[i].faces.front().face)];
    for (size_t i = 0; i < g.nv(); ++i)
        a[i] = g.vertices[i].faces.empty() ? 0 : face_rank[g.face_index(g.vertices[i].faces.front().face)];
    return a;
}

// =====================================================================
// P1 element matrices (reference src/elements.cpp:17-76). Host code is
// compiled with -ffp-contract=off so every product/sum rounds separately,
// as in the reference's baseline x86-64 build.
// =====================================================================
Elem3 p1_element(Form form, const std::array<Vec2, 3>& tri) {
    const Vec2 u1 = tri[1] - tri[0], u2 = tri[2] - tri[0];
    const double det = cross2(u1, u2);
    if (det == 0.0) throw InvalidArgument("local_stiffness: zero-area triangle");
    const double area = std::abs(det) / 2.0;
    Vec2 gr[3];
    gr[1] = {u2.y / det, -u2.x / det};
    gr[2] = {-u1.y / det, u1.x / det};
    gr[0] = {-gr[1].x - gr[2].x, -gr[1].y - gr[2].y};
    Elem3 m{};
    switch (form) {
    case LAPLACE:
    case PSPG: {
        // PSPG: -delta h_T^2 (grad q, grad p), delta = 1/12, h_T^2 = 2|T| (elements.cpp:33-47)
        const double s = form == LAPLACE ? area : -(1.0 / 12.0) * 2.0 * area * area;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j <= i; ++j) {
                const double v = s * dot2(gr[i], gr[j]);
                m.m[i][j] = v;
                m.m[j][i] = v;
            }
        return m;
    }
    case MASS:
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) m.m[i][j] = i == j ? area / 6.0 : area / 12.0;
        return m;
    case DIV_X:
    case DIV_Y: // -(q, d* u): hat integral area/3 times the constant trial derivative (:54-63)
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) m.m[i][j] = -(area / 3.0) * (form == DIV_X ? gr[j].x : gr[j].y);
        return m;
    case GRAD_X:
    case GRAD_Y: { // the transpose of DIV (:64-71)
        const Elem3 d = p1_element(form == GRAD_X ? DIV_X : DIV_Y, tri);
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) m.m[i][j] = d.m[j][i];
        return m;
    }
    }
    throw InvalidArgument("local_stiffness: bad form");
}

// =====================================================================
// Stencil assembly (reference src/operators.cpp:22-263), P1 only.
// A stencil entry is the sum of element-matrix entries over the micro-cells
// containing both DoFs, accumulated in the reference's cell order so every
// coefficient is bitwise the reference's.
// =====================================================================
namespace {

struct Cell {
    bool up;
    int c, r;
};
struct Off {
    int dc, dr;
};
constexpr Off kUpDofs[3] = {{0, 0}, {1, 0}, {0, 1}};
constexpr Off kDownDofs[3] = {{1, 0}, {0, 1}, {1, 1}};

// cells whose element matrix couples the lattice vertex (c, r), in the
// reference's enumeration order (operators.cpp:50-54)
std::array<Cell, 6> vertex_cells(int c, int r) {
    return {{{true, c, r}, {true, c - 1, r}, {true, c, r - 1}, {false, c - 1, r}, {false, c, r - 1},
             {false, c - 1, r - 1}}};
}
bool cell_inside(const Cell& t, int n) { return t.c >= 0 && t.r >= 0 && t.c + t.r <= (t.up ? n - 1 : n - 2); }

struct CellMats {
    Elem3 up, down;
};
CellMats micro_elements(Form form, const std::array<Vec2, 3>& corners, int level) {
    const double inv = 1.0 / double(1 << level);
    const Vec2 u = inv * (corners[1] - corners[0]);
    const Vec2 v = inv * (corners[2] - corners[0]);
    return {p1_element(form, {Vec2{0, 0}, u, v}), p1_element(form, {u, v, u + v})};
}

int local_index(const Cell& cell, int c, int r) {
    const Off* d = cell.up ? kUpDofs : kDownDofs;
    int irecv = -1;
    for (int i = 0; i < 3; ++i)
        if (cell.c + d[i].dc == c && cell.r + d[i].dr == r) irecv = i;
    if (irecv < 0) throw LogicError("stencil assembly: receiving DoF missing from its cell");
    return irecv;
}

// distance of lattice vertex (c, r) from border `slot`, and walk coordinate
int border_distance(int slot, int n, int c, int r) { return slot == 0 ? r : slot == 1 ? c : n - (c + r); }
int walk_coordinate(int slot, int c, int r) { return slot == 0 ? c : r; }

} // namespace

FaceStencil assemble_face_stencil(Form form, const MacroFace& f, int level) {
    const CellMats E = micro_elements(form, f.coord, level);
    // key (dc, dr) -> reference map order index
    const auto slot_of = [](int dc, int dr) -> int {
        static const Off order[7] = {{-1, 0}, {-1, 1}, {0, -1}, {0, 0}, {0, 1}, {1, -1}, {1, 0}};
        for (int i = 0; i < 7; ++i)
            if (order[i].dc == dc && order[i].dr == dr) return i;
        throw LogicError("face stencil: coupling outside the 7-point pattern");
    };
    FaceStencil s{};
    for (const Cell& cell : vertex_cells(0, 0)) {
        const Elem3& M = cell.up ? E.up : E.down;
        const int irecv = local_index(cell, 0, 0);
        const Off* d = cell.up ? kUpDofs : kDownDofs;
        for (int j = 0; j < 3; ++j) s.c[slot_of(cell.c + d[j].dc, cell.r + d[j].dr)] += M.m[irecv][j];
    }
    s.diag = s.c[3];
    return s;
}

EdgeStencil assemble_edge_stencil(Form form, const MacroGraph& g, const MacroEdge& e, int level) {
    (void)g;
    const int n = 1 << level, W = n + 1;
    EdgeStencil s{};
    if (n < 2) return s; // no interior line DoFs on level 0
    // keys exactly as the reference forms them: (storage row base in the
    // reference edge layout, entry offset relative to k)
    std::map<std::pair<long, long>, double> acc;
    for (size_t fi = 0; fi < e.faces.size(); ++fi) {
        const FaceSide& nb = e.faces[fi];
        const CellMats E = micro_elements(form, nb.corners, level);
        const int k0 = 1;
        const int w0 = nb.aligned ? k0 : n - k0;
        int rc, rr; // receiving border DoF in the face frame
        if (nb.slot == 0) { rc = w0; rr = 0; }
        else if (nb.slot == 1) { rc = 0; rr = w0; }
        else { rc = n - w0; rr = w0; }
        const long halo_base = long(n + 1) + long(fi) * long(2 * n + 1);
        for (const Cell& cell : vertex_cells(rc, rr)) {
            if (!cell_inside(cell, n)) continue;
            const Elem3& M = cell.up ? E.up : E.down;
            const int irecv = local_index(cell, rc, rr);
            const Off* d = cell.up ? kUpDofs : kDownDofs;
            for (int j = 0; j < 3; ++j) {
                const int c = cell.c + d[j].dc, r = cell.r + d[j].dr;
                const int o = border_distance(nb.slot, n, c, r);
                const int w = walk_coordinate(nb.slot, c, r);
                long base, entry;
                if (o == 0) {
                    base = 0;
                    entry = nb.aligned ? w : n - w;
                } else {
                    if (o != 1) throw LogicError("edge stencil: coupling beyond halo row 1");
                    const int len = W - o;
                    base = halo_base + W; // row 1 follows row 0 (length W) in the reference block
                    entry = nb.aligned ? w : (len - 1) - w;
                }
                acc[{base, entry - k0}] += M.m[irecv][j];
            }
        }
    }
    // expected key set: line (-1,0,1), then per face row 1 (-1,0)
    std::vector<std::pair<long, long>> want = {{0, -1}, {0, 0}, {0, 1}};
    for (size_t fi = 0; fi < e.faces.size(); ++fi) {
        const long b = long(n + 1) + long(fi) * long(2 * n + 1) + W;
        want.push_back({b, -1});
        want.push_back({b, 0});
    }
    if (acc.size() != want.size()) throw LogicError("edge stencil: unexpected support size");
    size_t i = 0;
    for (const auto& [key, coeff] : acc) {
        if (key != want[i]) throw LogicError("edge stencil: unexpected support pattern");
        s.c[i++] = coeff;
    }
    s.nterms = int(i);
    s.diag = acc.at({0, 0});
    return s;
}

VertexStencil assemble_vertex_stencil(Form form, const MacroVertex& v, int level) {
    const int n = 1 << level;
    std::map<size_t, double> acc;
    for (const CornerFace& cf : v.faces) {
        const Elem3 M = micro_elements(form, cf.corners, level).up;
        const int ci = cf.corner;
        const Cell cell = ci == 0 ? Cell{true, 0, 0} : ci == 1 ? Cell{true, n - 1, 0} : Cell{true, 0, n - 1};
        for (int j = 0; j < 3; ++j) {
            const double coeff = M.m[ci][j];
            if (j == ci) {
                acc[0] += coeff;
                continue;
            }
            const int c = cell.c + kUpDofs[j].dc, r = cell.r + kUpDofs[j].dr;
            int pick = -1;
            for (int s : kCornerSlots[ci])
                if (border_distance(s, n, c, r) == 0) {
                    pick = s;
                    break;
                }
            if (pick < 0) throw LogicError("vertex stencil: neighbour off the flank borders");
            const uint64_t eid = cf.flank[pick == kCornerSlots[ci][0] ? 0 : 1];
            const auto it = std::find(v.edges.begin(), v.edges.end(), eid);
            if (it == v.edges.end()) throw LogicError("vertex stencil: flank edge not incident");
            acc[1 + size_t(it - v.edges.begin())] += coeff;
        }
    }
    VertexStencil s;
    if (acc.size() != 1 + v.edges.size()) throw LogicError("vertex stencil: unexpected support size");
    for (const auto& [slot, coeff] : acc) s.c.push_back(coeff);
    s.diag = acc.at(0);
    return s;
}

} // namespace hyb
