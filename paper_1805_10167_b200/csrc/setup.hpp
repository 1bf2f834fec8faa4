// Host-side setup for the B200 multigrid hot path: coarse mesh, macro-primitive
// graph, fixture meshes, partitioning, P1 stencil assembly and DoF flags.
//
// Everything here runs once per domain (O(#macro-primitives)); the conventions
// (dense ID blocks, border slots, `aligned`, derived edge markers, ID-sorted
// neighbour lists) are the ones the reference's storage and exchange rely on,
// so the device tables built from this graph address exactly the DoFs the
// reference addresses:
//   mesh file format / CCW canonicalisation   reference src/mesh.cpp:22-83
//   macro-primitive graph                     reference src/mesh.cpp:97-263
//   slot convention                           reference include/hytegrid/mesh.hpp:52-62
//   fixture generators                        reference src/meshgen.cpp:50-141
//   partitioners                              reference src/balancing.cpp:19-137
//   P1 element matrices                       reference src/elements.cpp:17-76
//   stencil assembly (face/edge/vertex)       reference src/operators.cpp:95-263
//   flags                                     reference src/field.cpp:15-120
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace hyb {

struct Vec2 {
    double x = 0.0, y = 0.0;
};
inline Vec2 operator+(Vec2 a, Vec2 b) { return {a.x + b.x, a.y + b.y}; }
inline Vec2 operator-(Vec2 a, Vec2 b) { return {a.x - b.x, a.y - b.y}; }
inline Vec2 operator*(double s, Vec2 a) { return {s * a.x, s * a.y}; }
inline double dot2(Vec2 a, Vec2 b) { return a.x * b.x + a.y * b.y; }
inline double cross2(Vec2 a, Vec2 b) { return a.x * b.y - a.y * b.x; }

// ---------------------------------------------------------------- errors
// One exception class per reference exception kind; the C ABI maps each to
// its own status code (see include/hyteg_b200.h).
struct InvalidArgument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct OutOfRange : std::out_of_range {
    using std::out_of_range::out_of_range;
};
struct RuntimeError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct LogicError : std::logic_error {
    using std::logic_error::logic_error;
};

// ---------------------------------------------------------------- mesh
struct CoarseMesh {
    std::vector<Vec2> pos;
    std::vector<int> marker;
    std::vector<std::array<int, 3>> tri; // CCW after parsing
    std::vector<int> region;
};

/// Parses the reference's ASCII mesh format ("NV NT", NV vertex lines
/// "x y marker", NT triangle lines "v0 v1 v2 region", '#' comments).
/// Clockwise triangles are flipped (v1<->v2) exactly as the reference does.
CoarseMesh parse_mesh_text(const std::string& text);

// ---------------------------------------------------------------- graph
enum Kind : uint8_t { VERTEX = 0, EDGE = 1, FACE = 2 };

struct FaceSide {            // what an edge knows about an adjacent face
    uint64_t face = 0;       // global primitive ID
    int slot = 0;            // border slot of the face occupied by the edge
    bool aligned = true;     // edge direction == face walk direction
    std::array<Vec2, 3> corners{};
};

struct CornerFace {          // what a vertex knows about an incident face
    uint64_t face = 0;
    std::array<Vec2, 3> corners{};
    int corner = 0;                   // local corner index of the vertex
    std::array<uint64_t, 2> flank{};  // the face's two edges meeting there
};

struct MacroVertex {
    Vec2 coord;
    int marker = 0;
    std::vector<uint64_t> edges;      // ID-sorted
    std::vector<int> edge_marker;     // derived marker of each edge
    std::vector<int> edge_far_marker; // marker of each edge's other endpoint
    std::vector<CornerFace> faces;    // ID-sorted
};

struct MacroEdge {
    std::array<uint64_t, 2> v{};      // end 0 = lower vertex ID
    std::array<Vec2, 2> coord{};
    std::array<int, 2> vmarker{};
    int marker = 0;                   // derived boundary marker
    std::vector<FaceSide> faces;      // 1 or 2, ID-sorted
};

struct MacroFace {
    std::array<uint64_t, 3> v{};      // CCW corners
    std::array<Vec2, 3> coord{};
    std::array<int, 3> vmarker{};
    std::array<uint64_t, 3> e{};      // by slot
    std::array<bool, 3> aligned{};
    std::array<int, 3> emarker{};
};

/// Dense IDs: vertices [0, nv), edges [nv, nv+ne), faces [nv+ne, nv+ne+nf).
struct MacroGraph {
    std::vector<MacroVertex> vertices;
    std::vector<MacroEdge> edges;
    std::vector<MacroFace> faces;

    size_t nv() const { return vertices.size(); }
    size_t ne() const { return edges.size(); }
    size_t nf() const { return faces.size(); }
    size_t size() const { return nv() + ne() + nf(); }
    Kind kind_of(uint64_t id) const {
        if (id < nv()) return VERTEX;
        if (id < nv() + ne()) return EDGE;
        if (id < size()) return FACE;
        throw OutOfRange("primitive id " + std::to_string(id) + " outside the graph");
    }
    uint64_t edge_id(size_t i) const { return nv() + i; }
    uint64_t face_id(size_t i) const { return nv() + ne() + i; }
    size_t edge_index(uint64_t id) const { return static_cast<size_t>(id - nv()); }
    size_t face_index(uint64_t id) const { return static_cast<size_t>(id - nv() - ne()); }
};

MacroGraph build_macro_graph(const CoarseMesh& mesh);

// ---------------------------------------------------------------- meshgen
namespace meshgen {
std::string unit_triangle();
std::string unit_square();
std::string unit_square_reversed();
std::string square_ring8();
std::string channel(int nx, int ny, double width, double height);
std::string annulus(int segments, int layers, double r_inner, double r_outer);
/// Same text with every marker-0 vertex moved by (dx, dy) ~ U[-frac, frac]*h_v
/// where h_v is its shortest incident coarse edge (counter-based RNG, `seed`).
std::string perturb_interior(const std::string& mesh_text, double frac, uint64_t seed);
} // namespace meshgen

// ---------------------------------------------------------------- partition
/// rank of every primitive, indexed by ID
std::vector<int> partition_round_robin(const MacroGraph& g, int ranks);
std::vector<int> partition_greedy_edgecut(const MacroGraph& g, int ranks, int weight_level);

// ---------------------------------------------------------------- flags
enum Flag : uint8_t { INNER = 1, DIRICHLET = 2, NEUMANN = 4 };
constexpr uint8_t ALL_FLAGS = 7;

struct BoundaryMap {
    std::map<int, uint8_t> marker_flag; // missing nonzero marker -> DIRICHLET
    uint8_t flag_for(int marker) const {
        if (marker == 0) return INNER;
        auto it = marker_flag.find(marker);
        return it == marker_flag.end() ? uint8_t(DIRICHLET) : it->second;
    }
    bool operator==(const BoundaryMap& o) const { return marker_flag == o.marker_flag; }
};

// ---------------------------------------------------------------- stencils
/// include/hytegrid/elements.hpp:17-25 (same values)
enum Form : uint8_t { LAPLACE = 0, MASS = 1, DIV_X = 2, DIV_Y = 3, GRAD_X = 4, GRAD_Y = 5, PSPG = 6 };

struct Elem3 {
    double m[3][3];
};
Elem3 p1_element(Form form, const std::array<Vec2, 3>& tri);

/// Face stencil in the reference's term order:
/// W(-1,0) NW(-1,+1) S(0,-1) C(0,0) N(0,+1) SE(+1,-1) E(+1,0).
struct FaceStencil {
    double c[7];
    double diag;
};
/// Edge line stencil: line k-1, k, k+1, then per adjacent face (ID order)
/// halo row 1 entries k-1, k.  nfaces in {1, 2}.
struct EdgeStencil {
    double c[7];
    int nterms;
    double diag;
};
/// Vertex stencil: own value, then one term per incident edge (ID order).
struct VertexStencil {
    std::vector<double> c;
    double diag;
};

FaceStencil assemble_face_stencil(Form form, const MacroFace& f, int level);
EdgeStencil assemble_edge_stencil(Form form, const MacroGraph& g, const MacroEdge& e, int level);
VertexStencil assemble_vertex_stencil(Form form, const MacroVertex& v, int level);

} // namespace hyb
