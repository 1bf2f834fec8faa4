// Coarse-grid system of the V-cycle (reference GridHierarchy ctor and
// coarse_correct, src/solvers.cpp:358-364, 385-398, 430-442): the min-level
// operator assembled over the global owned numbering (assemble_global_sparse,
// src/operators.cpp:507-546), DIRICHLET rows/columns eliminated
// (constrain_dirichlet, src/solvers.cpp:322-352), rows in GlobalDoFMap order,
// columns ascending as in the reference's row maps.
#pragma once

#include <cstdint>
#include <map>
#include <vector>

#include "plan.hpp"
#include "setup.hpp"

namespace hyb {

struct HostCsr {
    int64_t n = 0;
    std::vector<int32_t> rowptr, col;
    std::vector<double> val;
    std::vector<uint8_t> flag; // per global DoF
};

/// assemble_global_sparse rows before constraining (every row holds its
/// stencil; flag = the DoF's flag under bc)
struct HostRows {
    int64_t n = 0;
    std::vector<std::map<int64_t, double>> rows;
    std::vector<uint8_t> flag;
};
HostRows assemble_rows(const MacroGraph& g, Form form, int L, const BoundaryMap& bc);

HostCsr assemble_constrained(const MacroGraph& g, Form form, int L, const BoundaryMap& bc);

/// StokesMultigrid's min-level matrix (constrained_stokes_matrix,
/// src/solvers.cpp:578-592): [[A,0,Gx],[0,A,Gy],[Bx,By,C]] over one P1
/// numbering, DIRICHLET rows identities, DIRICHLET columns dropped
HostCsr assemble_stokes_constrained(const MacroGraph& g, int L, const BoundaryMap& bc_u, const BoundaryMap& bc_p);

} // namespace hyb
