// P2 on the engine: the four-group quadratic stencils of the reference
// (src/operators.cpp:22-263 with FunctionKind::P2, src/elements.cpp:74-186)
// laid out on the level-(L+1) P1 lattice.
//
// A P2 function at level L has one DoF per lattice point of the once-refined
// lattice: group VERTEX (c, r) -> (2c, 2r), EDGE_HORIZONTAL -> (2c+1, 2r),
// EDGE_DIAGONAL -> (2c+1, 2r+1), EDGE_VERTICAL -> (2c, 2r+1) (the reference's
// own DoF coordinates, group_lattice_coord, src/indexing.cpp:85-95). So its
// faces are the closed level-(L+1) triangle of the P1 arena, its edge line is
// the level-(L+1) line (vertex DoFs at even, midline DoFs at odd positions),
// and its owned set is the P1 level-(L+1) owned set. What differs from P1:
//   * the stencil of a face DoF depends on its group = the parity class of
//     (c', r') (0 V, 1 EH, 2 EV, 3 ED: (c' & 1) + 2 (r' & 1)) and reaches two
//     rows / columns of the fine lattice (the vertex group's 19 points);
//   * edges keep two halo rows per face (fine rows 1 and 2: the reference's
//     P2 halo rows {V,1},{par,1},{non-par,0}, src/layout.cpp:40-52);
//   * vertices keep the reference's P2 ghosts: per incident edge the next
//     line vertex and the midpoint, per incident face the corner cell's
//     interior midpoint (src/layout.cpp:131-157).
// Stencils are assembled exactly as the reference does (same cells, same
// accumulation order, same std::map term order), then each term's storage
// position is re-expressed in this layout, so apply sums the same products in
// the same order: bitwise the reference.
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include "setup.hpp"

namespace hyb {

/// fine-lattice term of a face stencil: x(c' + dc, r' + dr)
struct P2FaceTerm {
    int dc, dr;
    double coeff;
};
struct P2FaceStencil {
    std::vector<P2FaceTerm> cls[4]; // by parity class (c' & 1) + 2 (r' & 1)
    double diag[4] = {0, 0, 0, 0};
};
/// edge term: storage position (P2 edge layout) base + k' + dk for the row at
/// fine line index k'
struct P2EdgeTerm {
    int base, dk;
    double coeff;
};
struct P2EdgeStencil {
    std::vector<P2EdgeTerm> line, mid; // vertex rows (even k'), midline rows (odd k')
    double line_diag = 0, mid_diag = 0;
};
/// vertex term: slot of the reference's P2 vertex layout (0 own, 1 + 2j next
/// line vertex on edge j, 2 + 2j midpoint on edge j, 1 + 2E + f face ghost)
struct P2VertexStencil {
    std::vector<std::pair<int, double>> terms;
    double diag = 0;
};

P2FaceStencil assemble_p2_face(Form form, const MacroFace& f, int level);
P2EdgeStencil assemble_p2_edge(Form form, const MacroEdge& e, int level);
P2VertexStencil assemble_p2_vertex(Form form, const MacroVertex& v, int level);

/// P2 edge storage at level L (n2 = 2^(L+1)): line [0, n2], then per adjacent
/// face j: fine halo row 1 (n2 entries, edge order) and row 2 (n2 - 1)
inline int p2_edge_halo1(int n2, int j) { return (n2 + 1) + j * (2 * n2 - 1); }
inline int p2_edge_halo2(int n2, int j) { return p2_edge_halo1(n2, j) + n2; }

} // namespace hyb
